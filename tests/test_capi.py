"""The C-ABI library loads without a GPU and exports every declared symbol."""

import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "disctree_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dt_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared_functions()
    for need in ("dt_prefix_scan", "dt_sign_terms", "dt_build_tree", "dt_moments",
                 "dt_tree_phi_sum", "dt_tree_phi_sum_packed", "dt_phi_sum_direct"):
        assert need in names


def test_library_exports_every_symbol():
    from paper_1710_05781_b200 import _lib

    lib = _lib.load()  # dlopen works without a GPU (static cudart)
    names = declared_functions()
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (dt_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a_only():
    from paper_1710_05781_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_version_and_errors_without_gpu():
    from paper_1710_05781_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.dt_version()
    # argument validation happens before any device work
    rc = lib.dt_phi_sum_direct(None, None, 0, None, -1.0, None, 0, 1, 0, 0, None)
    assert rc == -1
    assert b"rd2" in lib.dt_last_error()
    # sharded upward pass: argument checks and slot sizes
    assert lib.dt_shard_plan(None, None, None, None, None, 0, None, 0, 1, 1 / 3, 4, 2, 0,
                             None, None) == -1
    assert lib.dt_shard_plan(1, 1, 1, 1, 1, 0, None, 0, 1, 1 / 3, 4, 2, 2, 1, None) == -1
    assert b"rank" in lib.dt_last_error()
    assert lib.dt_moments_partial(1, 1, 1, 1, 1, 1, 1, 1, 1, 32, 1, None, 34, 16, 1, 4096,
                                  None) == -1
    assert b"order <= 31" in lib.dt_last_error()
    assert lib.dt_shard_rows_bytes(-1, 30, 32) == 0
    assert lib.dt_shard_rows_bytes(4, 30, 32) == 16 * 32 * 8


def test_order_limits_checked_before_device_work():
    """The far-field tables cover orders 0..127: larger p, p_cap or moment
    strides are rejected (DT_ERR_ARG) instead of reading past them."""
    from paper_1710_05781_b200 import _lib

    lib = _lib.load()

    def call(p, p_cap, stride, adaptive=1):
        return lib.dt_tree_phi_sum(1, 1, 1, 1, 1, 1, 1, stride, 3, 1, 1, 4, 1e-4, 1 / 3, p,
                                   adaptive, 1e-10, p_cap, 1, 1, 64, 1, 1, 0, 0, 0, None, 0,
                                   None)

    assert call(128, 30, 256) == -1 and b"<= 127" in lib.dt_last_error()
    assert call(8, 128, 256) == -1 and b"<= 127" in lib.dt_last_error()
    assert call(8, 30, 130, adaptive=0) == -1 and b"<= 128" in lib.dt_last_error()
    # in range: the argument checks pass and the empty target range returns OK
    assert call(127, 127, 128) == 0


def test_no_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1710_05781_b200 as dt

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        dt.from_particles([(0.0, 1.0)])
