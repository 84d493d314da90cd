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
(pipeline.TreePipeline); the only collective is the optional all-gather of
the per-rank field slices (8 bytes per target).  The tree build and the
moments are replicated per rank in this round (they cost ~1.8 ms at 2^24 on
one B200); DESIGN.md describes the sharded-moment variant with an all-gather
of the upper-level moment rows.
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
