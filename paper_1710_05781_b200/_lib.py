"""ctypes binding of libdisctree_b200.so (include/disctree_b200.h).

The shared library holds every sm_100a kernel of the hot path.  There is no
CPU fallback: if the library is missing, or no B200 is visible, compute entry
points raise ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DISCTREE_B200_LIB", os.path.join(_HERE, "libdisctree_b200.so"))

DT_OK = 0
DT_PSEL_FAST = 0
DT_PSEL_EXACT = 1
DT_DIRECT_FP64 = 0
DT_DIRECT_FP32 = 1
DT_DIRECT_KAHAN = 2
DT_MAX_DEPTH = 60
DT_META_NODES = 0
DT_META_DEPTH = 1
DT_META_LEAVES = 2
DT_META_OVERFLOW = 3
DT_META_P2M_UPTO = 5
DT_META_LEVEL0 = 8
DT_META_WORDS = 72
DT_EVAL_COUNTER_BYTES = 65536
DT_MAX_WORLD = 64
DT_PLAN_CUT = 0
DT_PLAN_LEVEL_BEGIN = 1
DT_PLAN_LEVEL_END = 2
DT_PLAN_SRC_LO = 3
DT_PLAN_SRC_HI = 4
DT_PLAN_NEED_LO = 5
DT_PLAN_NEED_HI = 6
DT_PLAN_OWNER0 = 8
DT_PLAN_WORDS = DT_PLAN_OWNER0 + DT_MAX_WORLD + 1

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_SZ = C.c_size_t


class EvalStats(C.Structure):
    """dt_eval_stats: device pointers indexed by target (NULL allowed)."""

    _fields_ = [
        ("hash", _P),
        ("near_pairs", _P),
        ("n_far", _P),
        ("sum_p", _P),
        ("n_p0", _P),
        ("n_exact", _P),
        ("bound", _P),
        ("abs_prefix", _P),
    ]


# name -> (restype, argtypes); exactly the symbols of include/disctree_b200.h
SIGNATURES = {
    "dt_version": (C.c_char_p, []),
    "dt_last_error": (C.c_char_p, []),
    "dt_device_check": (C.c_int, []),
    "dt_prefix_scan_workspace": (_SZ, [_I64]),
    "dt_prefix_scan": (C.c_int, [_P, _P, _I64, _P, _SZ, _P]),
    "dt_sign_terms_workspace": (_SZ, [_I64]),
    "dt_sign_terms": (C.c_int, [_P, _P, _I64, _P, _P, _I64, _P, _SZ, _P]),
    "dt_sign_bracket": (C.c_int, [_P, _I64, _P, _I64, _P, _SZ, _P]),
    "dt_sign_terms_bracketed": (C.c_int, [_P, _P, _I64, _P, _P, _I64, _P, _SZ, _P]),
    "dt_check_values": (C.c_int, [_P, _I64, _P, _P]),
    "dt_unpack_pairs": (C.c_int, [_P, _I64, _P, _P, _P, _P]),
    "dt_density_nodes": (C.c_int, [_D, _D, _I64, _P, _I64, _I64, _P, _P, _D, _P, _P]),
    "dt_mirror_charges": (C.c_int, [_P, _P, _I64, _D, _D, _P, _P, _P, _P]),
    "dt_build_workspace": (_SZ, [_I64, _I64]),
    "dt_build_tree": (
        C.c_int,
        [_P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P],
    ),
    "dt_build_tree_p2m": (
        C.c_int,
        [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P,
         _I64, _P, _P, _SZ, _P],
    ),
    "dt_moments_workspace": (_SZ, [_I64]),
    "dt_moments": (
        C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _I64, _I64, _P, _SZ, _P],
    ),
    "dt_moments_pack": (
        C.c_int,
        [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _I64, _I64, _P, _P, _SZ, _P],
    ),
    "dt_moments_from_eval": (C.c_int, [_P, _I64, _I64, _I64, _P, _P]),
    "dt_sort_workspace": (_SZ, [_I64]),
    "dt_sort_stable": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "dt_permute": (C.c_int, [_P, _P, _I64, _P, C.c_int, _P]),
    "dt_compact_workspace": (_SZ, [_I64]),
    "dt_compact_pairs": (C.c_int, [_P, _P, _P, _I64, _P, _I64, _P, _P, _SZ, _P]),
    "dt_zero": (C.c_int, [_P, _SZ, _P]),
    "dt_shard_plan": (
        C.c_int,
        [_P, _P, _P, _P, _P, _I64, _P, _I64, C.c_int, _D, _I64, C.c_int, C.c_int, _P, _P],
    ),
    "dt_shard_rows_bytes": (_SZ, [_I64, _I64, _I64]),
    "dt_moments_partial": (
        C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _P, _P, _I64, _I64, _P, _SZ, _P],
    ),
    "dt_shard_pack": (C.c_int, [_P, C.c_int, _I64, _I64, _P, _P, _I64, _P, _P]),
    "dt_shard_finish": (
        C.c_int, [_P, C.c_int, _I64, _P, _P, _P, _P, _P, _I64, _P, _P, _I64, _P],
    ),
    "dt_pack_sources": (C.c_int, [_P, _P, _I64, _P, _P]),
    "dt_pack_tree": (C.c_int, [_P, _P, _P, _P, _P, _P, _I64, _P, _P]),
    "dt_tree_eval_workspace": (_SZ, [_I64, _I64, _I64]),
    "dt_tree_phi_sum": (
        C.c_int,
        [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _I64, _D, _D, _I64, C.c_int, _D,
         _I64, _P, _P, _I64, _P, _P, _I64, _I64, C.c_int, _P, _SZ, _P],
    ),
    "dt_tree_phi_sum_packed": (
        C.c_int,
        [_P, _I64, _P, _I64, _P, _I64, _D, _D, _I64, C.c_int, _D, _I64, _P, _P, _I64, _P,
         _P, _I64, _I64, C.c_int, C.c_int, C.POINTER(EvalStats), _P, _SZ, _P],
    ),
    "dt_tree_field_workspace": (_SZ, [_I64]),
    "dt_tree_field_packed": (
        C.c_int,
        [_P, _I64, _P, _I64, _P, _P, _P, _I64, _D, _D, _I64, C.c_int, _D, _I64, _P, _P, _I64,
         _P, _P, _I64, _I64, _P, _P, _SZ, _P],
    ),
    "dt_tree_eval_device": (
        C.c_int,
        [_P, _P, _I64, _P, _I64, _P, _I64, _D, _D, _I64, C.c_int, _D, _I64, _P, _P, _I64, _P,
         _P, _I64, _I64, C.c_int, _P, _SZ, _P],
    ),
    "dt_eval_prepare": (
        C.c_int,
        [_P, _P, _I64, _P, _I64, _P, _I64, _D, _D, _I64, C.c_int, _D, _I64, _P, _P, _I64, _P,
         _P, _I64, _I64, C.c_int, _P, _SZ, _P],
    ),
    "dt_tree_eval_device_prepared": (
        C.c_int,
        [_P, _P, _I64, _P, _I64, _P, _I64, _D, _D, _I64, C.c_int, _D, _I64, _P, _P, _I64, _P,
         _P, _I64, _I64, C.c_int, _P, _SZ, _P],
    ),
    "dt_tree_field_device": (
        C.c_int,
        [_P, _P, _I64, _P, _I64, _P, _P, _P, _I64, _D, _D, _I64, C.c_int, _D, _I64, _P, _P,
         _I64, _P, _P, _I64, _I64, _P, _SZ, _P],
    ),
    "dt_fp64_probe": (C.c_int, [_P, _I64, C.c_int, _P]),
    "dt_choose_p_batch": (
        C.c_int, [_P, _P, _I64, _D, _D, _I64, _P, _P, _I64, C.c_int, _P, _P, _P],
    ),
    "dt_phi_sum_direct": (
        C.c_int, [_P, _P, _I64, _P, _D, _P, _I64, _I64, C.c_int, C.c_int, _P],
    ),
    "dt_phi_sum_symmetric_workspace": (_SZ, [_I64]),
    "dt_phi_sum_symmetric": (C.c_int, [_P, _P, _I64, _D, _P, C.c_int, _P, _SZ, _P]),
}

_lib = None


def load():
    """dlopen the library (no GPU needed) and declare every signature."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or make -C paper_1710_05781_b200/csrc); there is no CPU fallback"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != DT_OK:
        msg = load().dt_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


_device_ok: dict[int, bool] = {}


def require_device():
    """Fail loudly unless a B200 (sm_100) is the current CUDA device."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1710_05781_b200 needs a CUDA device (B200, sm_100a); none is visible and "
            "there is no CPU fallback"
        )
    dev = torch.cuda.current_device()
    if dev not in _device_ok:
        check(load().dt_device_check(), "device check")
        _device_ok[dev] = True
    return torch.device("cuda", dev)


def stream_handle():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def zeros_i64(n: int, device):
    """int64 device words zeroed by dt_zero (flag counters; no torch fill kernel)."""
    import torch

    t = torch.empty(n, dtype=torch.int64, device=device)
    check(load().dt_zero(C.c_void_p(t.data_ptr()), 8 * n, stream_handle()), "dt_zero")
    return t


def ptr(t) -> C.c_void_p:
    """Device address of a torch tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())
