"""World-size-2 gloo tests of the multi-GPU orchestration on CPU.

Each rank evaluates its contiguous target slice; the CPU oracle stands in for
the per-rank device computation (there is no GPU here), so these tests cover
the host-side logic: slice bounds, the all-gather, and the world-size
invariance of the gathered field.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_case
from paper_1710_05781_b200.parallel import evaluate_sharded, gather_slices, shard_bounds


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds_match_run_chunked():
    for n in (0, 1, 7, 100, 16384):
        for world in (1, 2, 3, 8):
            bounds = np.linspace(0, n, world + 1).astype(np.int64)
            got = [shard_bounds(n, world, r) for r in range(world)]
            assert got == [(int(bounds[r]), int(bounds[r + 1])) for r in range(world)]
            assert sum(b - a for a, b in got) == n
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _oracle_field(g, i0, i1):
    from oracle import oracle as O

    t = g["targets"][i0:i1]
    E, _ = O.evaluate_tree(g["xs"], g["qs"], float(g["r_d"]), int(g["p"]), float(g["theta"]),
                           int(g["leaf_capacity"]), bool(g["adaptive"]),
                           float(g["tolerance"]), t)
    return torch.from_numpy(E)


def _worker(rank, world, port, case, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_case(case)
        ys = torch.from_numpy(g["targets"])
        full = evaluate_sharded(ys, lambda i0, i1: _oracle_field(g, i0, i1))
        # ragged gather of arbitrary slices
        n = 11
        a, b = shard_bounds(n, world, rank)
        ragged = gather_slices(torch.arange(a, b, dtype=torch.float64), n, world)
        assert torch.equal(ragged, torch.arange(n, dtype=torch.float64))
        if rank == 0:
            np.save(out_path, full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cfg1s", "rand_adaptive"])
def test_gloo_world2_matches_single_rank(tmp_path, case):
    out = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(2, _free_port(), case, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    g = load_case(case)
    want = _oracle_field(g, 0, len(g["targets"])).numpy()
    np.testing.assert_array_equal(got, want)  # bit-identical for any world size
    scale = np.abs(g["qs"]).sum()
    assert np.max(np.abs(got - g["E_tree"])) <= 1e-13 * scale
