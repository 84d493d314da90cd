"""Multi-GPU orchestration: contiguous target shards, one process per GPU.

The reference parallelises evaluate_all over CPU threads by splitting the
targets into contiguous chunks (_kernels.run_chunked, _kernels.py:269-289,
bounds from np.linspace) and every target's result is independent of the
chunking.  Here each rank of a torch.distributed job (NCCL over NVLink on a
B200 box; gloo in the CPU tests) owns one contiguous slice of the sorted
targets, with the sources replicated on every rank.  A target's traversal
does not depend on which rank runs it, so the gathered field is
bit-identical for any world size.

Per rank the hot path runs on the device without host round trips
(pipeline.TreePipeline).  The tree build is replicated (deterministic, so
every rank holds the same tree).  The upward pass is sharded
(ShardedMoments): each rank forms only the subtrees below a
cut level that it owns or that its targets can open, one all-gather
exchanges the owners' cut-level rows (KB), and every rank forms the few
levels above the cut.  The only other collective is the optional all-gather
of the per-rank field slices (8 bytes per target).
"""

from __future__ import annotations

from typing import Callable

import torch


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [i0, i1) of n items for `rank` (the same
    integer bounds as np.linspace(0, n, world + 1).astype(int64))."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return (rank * n) // world, ((rank + 1) * n) // world


def gather_slices(local: torch.Tensor, n: int, world: int, group=None) -> torch.Tensor:
    """All-gather equal-or-ragged contiguous slices into the full [n] array."""
    import torch.distributed as dist

    if world == 1:
        return local
    width = (n + world - 1) // world + 1
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.empty(n, dtype=local.dtype, device=local.device)
    for r in range(world):
        i0, i1 = shard_bounds(n, world, r)
        out[i0:i1] = parts[r][: i1 - i0]
    return out


def evaluate_sharded(ys: torch.Tensor, compute_slice: Callable[[int, int], torch.Tensor],
                     world: int | None = None, rank: int | None = None, gather: bool = True,
                     group=None) -> torch.Tensor:
    """Evaluate targets ys on this rank's slice with `compute_slice(i0, i1)`
    (returns the field for ys[i0:i1]) and optionally all-gather the result."""
    import torch.distributed as dist

    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = ys.numel()
    i0, i1 = shard_bounds(n, world, rank)
    local = compute_slice(i0, i1)
    if local.numel() != i1 - i0:
        raise RuntimeError("compute_slice returned a slice of the wrong length")
    return gather_slices(local, n, world, group) if gather else local


def gpu_slice_evaluator(tree, kernel, config, system, ys: torch.Tensor):
    """compute_slice for the GPU path: sign term + traversal on ys[i0:i1]."""
    from .charges import _sign_terms
    from .tree import tree_phi_sum

    def run(i0: int, i1: int) -> torch.Tensor:
        part = ys[i0:i1].contiguous()
        vals = _sign_terms(system, part)
        tree_phi_sum(tree, kernel, config, part, vals)
        return vals

    return run


def default_cut_level(world: int) -> int:
    """Cut level of the sharded upward pass: about 16 cut-level nodes per
    rank (2^(ceil(log2 world) + 4) nodes at most), identical on every rank."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    return (world - 1).bit_length() + 4


def gather_rows(send: torch.Tensor, recv: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather equal-size per-rank slots (rank order) into recv."""
    import torch.distributed as dist

    if recv.numel() != world * send.numel():
        raise ValueError("recv must hold world * send.numel() elements")
    if world == 1:
        recv.copy_(send)
    elif send.is_cuda and dist.get_backend(group) == "gloo":
        # gloo (CPU tests, several ranks sharing one GPU) gathers host tensors
        host = torch.empty(recv.numel(), dtype=recv.dtype)
        dist.all_gather_into_tensor(host, send.cpu(), group=group)
        recv.copy_(host)
    else:  # NCCL over NVLink: stream-ordered, no host round trip
        dist.all_gather_into_tensor(recv, send, group=group)
    return recv


class ShardedMoments:
    """Sharded upward pass (c) for one rank of a target-sharded job.

    The tree (bufs, from dt_build_tree) is the same on every rank.  For the
    rank's targets ys (its contiguous slice, sorted or not) ``launch`` runs:
      dt_shard_plan       cut level, owners, this rank's source range   (1 block)
      dt_moments_partial  P2M + M2M of this rank's subtrees below the cut
      dt_shard_pack       owned cut-level rows -> gather slot
      all-gather          one collective of dt_shard_rows_bytes per rank
      dt_shard_finish     scatter the owners' rows, M2M above the cut (1 block)
    all stream-ordered on the current stream, no host round trip.  Every row
    the rank's traversal can read is then bit-identical to dt_moments' row.
    Rows of subtrees no target of this rank can open are left untouched.
    """

    LAUNCHES = 5  # plan, prep, upward, row pack, finish (the all-gather is NCCL's)

    def __init__(self, bufs, order: int, moments: torch.Tensor | None, meval: torch.Tensor,
                 estride: int, theta: float, world: int, rank: int, group=None,
                 cut_level: int | None = None):
        from . import _lib

        if not 0 <= rank < world <= _lib.DT_MAX_WORLD:
            raise ValueError(f"bad rank {rank} / world size {world}")
        if order + 1 > 32:
            raise ValueError("sharded moments need moment order <= 31")
        self.bufs, self.order = bufs, int(order)
        # moments (reference layout) may be None: the gathered and formed rows
        # are traversal rows (meval); finish() derives moments when given
        self.moments, self.meval = moments, meval
        self.estride = int(estride)
        self.theta = float(theta)
        self.world, self.rank, self.group = int(world), int(rank), group
        self.cut = default_cut_level(world) if cut_level is None else int(cut_level)
        dev = meval.device
        nbytes = int(_lib.load().dt_shard_rows_bytes(self.cut, self.order, self.estride))
        if nbytes == 0:
            raise ValueError(f"bad cut level {self.cut}")
        self.plan = torch.zeros(_lib.DT_PLAN_WORDS, dtype=torch.int64, device=dev)
        self.send = torch.zeros(nbytes // 8, dtype=torch.float64, device=dev)
        self.recv = torch.zeros(self.world * (nbytes // 8), dtype=torch.float64, device=dev)

    def local(self, xs: torch.Tensor, qs: torch.Tensor, ys: torch.Tensor,
              targets_sorted: bool = True) -> torch.Tensor:
        """Plan + this rank's subtrees + pack; returns the gather slot."""
        from . import _lib

        L, p, s, b = _lib.load(), _lib.ptr, _lib.stream_handle(), self.bufs
        _lib.check(L.dt_shard_plan(p(b.center), p(b.half), p(b.start), p(b.end), p(b.meta),
                                   xs.numel(), p(ys), ys.numel(), int(bool(targets_sorted)),
                                   self.theta, self.cut, self.world, self.rank, p(self.plan), s),
                   "dt_shard_plan")
        _lib.check(L.dt_moments_partial(p(xs), p(qs), p(b.center), p(b.start), p(b.end),
                                        p(b.left), p(b.right), p(b.meta), p(self.plan),
                                        self.order, p(self.moments), p(self.meval),
                                        self.estride, b.capacity, p(b.mws), b.mws_bytes, s),
                   "dt_moments_partial")
        _lib.check(L.dt_shard_pack(p(self.plan), self.rank, self.cut, self.order,
                                   p(self.moments), p(self.meval), self.estride, p(self.send), s),
                   "dt_shard_pack")
        return self.send

    def finish(self, recv: torch.Tensor | None = None) -> None:
        """Scatter the gathered cut-level rows and form the levels above."""
        from . import _lib

        recv = self.recv if recv is None else recv
        L, p, b = _lib.load(), _lib.ptr, self.bufs
        _lib.check(L.dt_shard_finish(p(self.plan), self.world, self.cut, p(recv), p(b.center),
                                     p(b.left), p(b.right), p(b.meta), self.order,
                                     p(self.moments), p(self.meval), self.estride,
                                     _lib.stream_handle()), "dt_shard_finish")

    def launch(self, xs: torch.Tensor, qs: torch.Tensor, ys: torch.Tensor,
               targets_sorted: bool = True) -> None:
        self.local(xs, qs, ys, targets_sorted)
        gather_rows(self.send, self.recv, self.world, self.group)
        self.finish()

    def plan_host(self) -> dict:
        """The plan block as a dict (synchronises; tests and diagnostics)."""
        from . import _lib

        v = self.plan.cpu().tolist()
        return {"cut": v[_lib.DT_PLAN_CUT],
                "level": (v[_lib.DT_PLAN_LEVEL_BEGIN], v[_lib.DT_PLAN_LEVEL_END]),
                "src": (v[_lib.DT_PLAN_SRC_LO], v[_lib.DT_PLAN_SRC_HI]),
                "need": (v[_lib.DT_PLAN_NEED_LO], v[_lib.DT_PLAN_NEED_HI]),
                "owners": v[_lib.DT_PLAN_OWNER0:_lib.DT_PLAN_OWNER0 + self.world + 1]}


def build_sharded(system, kernel, config, ys_local: torch.Tensor, world: int, rank: int,
                  group=None, cut_level: int | None = None, targets_sorted: bool = False):
    """tree.build for one rank of a target-sharded job: the same tree on every
    rank, moments formed with ShardedMoments for this rank's targets
    ys_local.  Moment rows no target of this rank can open are NaN."""
    from .tree import _build

    if not ys_local.is_cuda:
        ys_local = ys_local.to(system.xs.device, non_blocking=True)

    def upward(bufs, order, moments, meval):
        if order + 1 > 32:  # the sharded pass covers orders <= 31: form every row
            from .tree import launch_moments

            launch_moments(bufs, system.xs, system.qs, order, moments, meval)
            return
        meval.fill_(float("nan"))
        ShardedMoments(bufs, order, moments, meval, meval.shape[1], config.theta, world, rank,
                       group, cut_level).launch(system.xs, system.qs, ys_local, targets_sorted)

    return _build(system, config, upward)
