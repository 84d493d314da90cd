"""Test-side restatement of the sharded upward pass (dt_shard_plan).

numpy over the node arrays of a built tree (oracle or GPU, both bit-exact
with the reference's tree.py:156-222).  Used by the gloo CPU tests (with the
oracle's moments) and by the GPU tests (against the device plan).
"""

from __future__ import annotations

import numpy as np


def default_cut_level(world: int) -> int:
    return (world - 1).bit_length() + 4


def shard_plan(tree: dict, n_src: int, ys: np.ndarray, theta: float, cut_req: int, world: int,
               rank: int) -> dict:
    """Plan of `rank`: cut level, level range, owners, opened set, source range."""
    level = np.asarray(tree["level"])
    start, end = np.asarray(tree["start"]), np.asarray(tree["end"])
    center, half = np.asarray(tree["center"]), np.asarray(tree["half"])
    depth = int(level.max())
    cut = min(cut_req, depth)
    idx = np.nonzero(level == cut)[0]
    b, e = int(idx[0]), int(idx[-1]) + 1
    assert np.array_equal(idx, np.arange(b, e)), "BFS levels are contiguous"
    owners = [b]
    for r in range(1, world):
        owners.append(b + int(np.searchsorted(start[b:e], (r * n_src) // world, side="left")))
    owners.append(e)
    need_lo, need_hi = b, b
    if len(ys):
        ylo, yhi = float(np.min(ys)), float(np.max(ys))
        c, h = center[b:e], half[b:e]
        dist = np.where(c < ylo, ylo - c, np.where(c > yhi, c - yhi, 0.0))
        need = np.nonzero(h * (1.0 + 2.0**-40) > theta * dist)[0]
        if len(need):
            need_lo, need_hi = b + int(need[0]), b + int(need[-1]) + 1
    ulo, uhi = owners[rank], owners[rank + 1]
    if need_lo < need_hi:
        if ulo >= uhi:
            ulo, uhi = need_lo, need_hi
        else:
            ulo, uhi = min(ulo, need_lo), max(uhi, need_hi)
    src = (int(start[ulo]), int(end[uhi - 1])) if ulo < uhi else (0, 0)
    return {"cut": cut, "level": (b, e), "src": src, "need": (need_lo, need_hi),
            "owners": owners}


def formed_rows(tree: dict, plan: dict) -> np.ndarray:
    """Rows a rank holds after the sharded pass: every node at levels <= cut,
    plus the nodes below the cut whose sources lie in plan['src']."""
    start, end = np.asarray(tree["start"]), np.asarray(tree["end"])
    n = len(start)
    b, e = plan["level"]
    lo, hi = plan["src"]
    idx = np.arange(n)
    return (idx < e) | ((idx >= b) & (start >= lo) & (end <= hi))


def local_rows(tree: dict, plan: dict) -> np.ndarray:
    """Rows a rank forms itself before the all-gather (dt_moments_partial)."""
    start, end = np.asarray(tree["start"]), np.asarray(tree["end"])
    left, right = np.asarray(tree["left"]), np.asarray(tree["right"])
    n = len(start)
    b, _ = plan["level"]
    lo, hi = plan["src"]
    idx = np.arange(n)
    leaf = (left < 0) & (right < 0)
    return (leaf & (idx < b)) | ((idx >= b) & (start >= lo) & (end <= hi))
