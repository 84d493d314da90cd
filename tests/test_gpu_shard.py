"""GPU parity of the sharded upward pass.

All ranks of a world of G are run one after the other on the one GPU (each
with its own NaN-filled moment buffers); the all-gather is the concatenation
of their slots in rank order, exactly what ncclAllGather delivers.  Checks:
the device plan equals the numpy restatement (tests/shard_ref.py); every row
a rank holds is bit-identical to the single-GPU row and exactly the expected
rows are held; each rank's traversal of its target slice reads no missing
row and is bit-identical to the single-GPU field.
"""

import dataclasses

import numpy as np
import pytest

from conftest import load_case

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1710_05781_b200 as pkg

    return pkg


def _simulate(dt, system, kernel, cfg, ys, world, cut_level=None, sorted_targets=True):
    import shard_ref as S
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.parallel import ShardedMoments, default_cut_level, shard_bounds
    from paper_1710_05781_b200.tree import (TreeBuffers, eval_stride, moment_order_for,
                                            tree_phi_sum)

    full = dt.build(system, kernel, cfg)
    n_nodes = len(full)
    bufs = TreeBuffers(len(system), n_nodes + 64, system.xs.device)
    bufs.launch(system.xs, cfg.leaf_capacity)
    order = moment_order_for(cfg)
    es = eval_stride(order)
    cut = default_cut_level(world) if cut_level is None else cut_level
    host = full.numpy()
    full_m = full.moments.cpu().numpy()
    full_me = full.meval.cpu().numpy()
    want = torch.zeros_like(ys)
    tree_phi_sum(full, kernel, cfg, ys, want, accumulate=False)
    shards, sends = [], []
    for r in range(world):
        i0, i1 = shard_bounds(ys.numel(), world, r)
        m = torch.full((bufs.capacity, order + 1), float("nan"), dtype=torch.float64,
                       device=ys.device)
        me = torch.full((bufs.capacity, es), float("nan"), dtype=torch.float64, device=ys.device)
        sh = ShardedMoments(bufs, order, m, me, es, cfg.theta, world, r, cut_level=cut)
        sends.append(sh.local(system.xs, system.qs, ys[i0:i1].contiguous(), sorted_targets)
                     .clone())
        shards.append((sh, m, me, i0, i1))
    recv = torch.cat(sends)
    held = []
    for r, (sh, m, me, i0, i1) in enumerate(shards):
        sh.finish(recv)
        plan = sh.plan_host()
        ref = S.shard_plan(host, len(system), ys[i0:i1].cpu().numpy(), cfg.theta, cut, world, r)
        assert plan["cut"] == ref["cut"] and plan["level"] == ref["level"]
        assert plan["owners"] == ref["owners"] and plan["need"] == ref["need"]
        assert plan["src"] == ref["src"]
        mh = m[:n_nodes].cpu().numpy()
        meh = me[:n_nodes].cpu().numpy()
        formed = ~np.isnan(mh).any(axis=1)
        np.testing.assert_array_equal(formed, S.formed_rows(host, ref))
        np.testing.assert_array_equal(mh[formed], full_m[formed])
        np.testing.assert_array_equal(meh[formed], full_me[formed])
        held.append(formed.mean())
        if i1 == i0:
            continue
        tree_r = dataclasses.replace(full, moments_ref=m[:n_nodes], meval=me[:n_nodes])
        got = torch.zeros(i1 - i0, dtype=torch.float64, device=ys.device)
        tree_phi_sum(tree_r, kernel, cfg, ys[i0:i1].contiguous(), got, accumulate=False)
        g = got.cpu().numpy()
        assert np.isfinite(g).all(), f"rank {r} read a moment row it does not hold"
        np.testing.assert_array_equal(g, want[i0:i1].cpu().numpy())
    return held


@pytest.mark.parametrize("case", ["cfg0", "cfg1s", "cfg2s", "rand_adaptive", "rand_p20",
                                  "duplicates", "coincident", "leafcap1"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_moments_golden_cases(dt, case, world):
    g = load_case(case)
    system = dt.from_particles(np.column_stack([g["xs"], g["qs"]]))
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = dt.EvalConfig(p=int(g["p"]), theta=float(g["theta"]),
                        leaf_capacity=int(g["leaf_capacity"]), adaptive=bool(g["adaptive"]),
                        tolerance=float(g["tolerance"]))
    ys = torch.from_numpy(np.sort(g["targets"])).cuda()
    _simulate(dt, system, kernel, cfg, ys, world)


@pytest.mark.parametrize("cut", [0, 1, 3, 9, 20])
def test_sharded_moments_cut_levels(dt, cut):
    g = load_case("cfg2s")
    system = dt.from_particles(np.column_stack([g["xs"], g["qs"]]))
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = dt.EvalConfig(p=8, leaf_capacity=64, adaptive=True, tolerance=1e-10)
    ys = torch.from_numpy(np.sort(g["targets"])).cuda()
    _simulate(dt, system, kernel, cfg, ys, 4, cut_level=cut)


def test_sharded_moments_unsorted_and_empty_slices(dt):
    g = load_case("rand_adaptive")
    system = dt.from_particles(np.column_stack([g["xs"], g["qs"]]))
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = dt.EvalConfig(p=int(g["p"]), leaf_capacity=int(g["leaf_capacity"]), adaptive=True,
                        tolerance=float(g["tolerance"]))
    ys = torch.from_numpy(np.random.default_rng(3).permutation(g["targets"])).cuda()
    _simulate(dt, system, kernel, cfg, ys, 3, sorted_targets=False)
    few = torch.from_numpy(np.sort(g["targets"])[:5]).cuda()  # world 8: empty slices
    _simulate(dt, system, kernel, cfg, few, 8)


def test_sharded_moments_graded_2e20(dt):
    """Graded mesh at 2^20 sources, world 8: each rank holds a small share."""
    from paper_1710_05781_b200 import workloads as W

    w = W.cfg2(cells=1 << 18)
    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, theta=w.theta, leaf_capacity=w.leaf_capacity,
                        adaptive=w.adaptive, tolerance=w.tolerance)
    ys = torch.from_numpy(w.targets).cuda()
    held = _simulate(dt, system, kernel, cfg, ys, 8)
    assert max(held) < 0.3


def test_build_sharded_public_api_single_rank(dt):
    """build_sharded at world 1 (no collective) gives the full moments."""
    from paper_1710_05781_b200.parallel import build_sharded

    g = load_case("cfg1s")
    system = dt.from_particles(np.column_stack([g["xs"], g["qs"]]))
    kernel = dt.DiscKernel(float(g["r_d"]))
    cfg = dt.EvalConfig(p=int(g["p"]), leaf_capacity=64, adaptive=True, tolerance=1e-10)
    ys = torch.from_numpy(g["targets"])
    t1 = build_sharded(system, kernel, cfg, ys, 1, 0)
    t0 = dt.build(system, kernel, cfg)
    assert torch.equal(t1.moments, t0.moments) and torch.equal(t1.meval, t0.meval)
    e1 = dt.evaluate_all(t1, kernel, cfg, system, g["targets"]).values
    e0 = dt.evaluate_all(t0, kernel, cfg, system, g["targets"]).values
    np.testing.assert_array_equal(e1, e0)


def _pipeline_worker(rank, world, port, out_path):
    import os

    import torch.distributed as dist

    import paper_1710_05781_b200 as dtp
    from paper_1710_05781_b200 import workloads as W
    from paper_1710_05781_b200.parallel import shard_bounds
    from paper_1710_05781_b200.pipeline import TreePipeline

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = W.cfg2(cells=1 << 16)
        kernel = dtp.DiscKernel(w.r_d)
        cfg = dtp.EvalConfig(p=w.p, theta=w.theta, leaf_capacity=w.leaf_capacity,
                             adaptive=w.adaptive, tolerance=w.tolerance)
        xs = torch.from_numpy(w.xs).cuda()
        qs = torch.from_numpy(w.qs).cuda()
        ys = torch.from_numpy(w.targets).cuda()
        T = ys.numel()
        i0, i1 = shard_bounds(T, world, rank)
        pipe = TreePipeline.planned(xs, T, kernel, cfg, world=world, rank=rank)
        out = torch.full_like(ys, float("nan"))
        for _ in range(2):
            pipe.step(xs, qs, ys, out, i0, i1)
        torch.cuda.synchronize()
        pipe.check()
        part = out[i0:i1].cpu()
        parts = [torch.empty(shard_bounds(T, world, r)[1] - shard_bounds(T, world, r)[0],
                             dtype=torch.float64) for r in range(world)]
        dist.all_gather(parts, part)  # T is even: equal slices
        if rank == 0:
            np.save(out_path, torch.cat(parts).numpy())
    finally:
        dist.destroy_process_group()


def test_pipeline_world2_gloo_on_one_gpu(dt, tmp_path):
    """The pipelined step with world 2 (two processes, gloo all-gather of the
    cut-level rows staged through the host) equals the world-1 step."""
    import socket

    import torch.multiprocessing as mp

    from paper_1710_05781_b200 import workloads as W
    from paper_1710_05781_b200.pipeline import TreePipeline

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    path = str(tmp_path / "e.npy")
    mp.start_processes(_pipeline_worker, args=(2, port, path), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(path)
    w = W.cfg2(cells=1 << 16)
    kernel = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, theta=w.theta, leaf_capacity=w.leaf_capacity,
                        adaptive=w.adaptive, tolerance=w.tolerance)
    xs = torch.from_numpy(w.xs).cuda()
    qs = torch.from_numpy(w.qs).cuda()
    ys = torch.from_numpy(w.targets).cuda()
    pipe = TreePipeline.planned(xs, ys.numel(), kernel, cfg)
    out = torch.empty_like(ys)
    pipe.step(xs, qs, ys, out)
    np.testing.assert_array_equal(got, out.cpu().numpy())
