"""Charge systems on the GPU: sorted sources, prefix sums, the sign term e(y).

Mirror of disctree.charges (charges.py:16-54, 114-132, 183-202): same names,
argument meaning and errors.  Arrays live on the current CUDA device as
float64 torch tensors; the prefix sum and the sign term run in
csrc/dt_scan.cu (stage (a) of the hot path).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class Charge:
    x: float
    q: float


def _to_device(a, dtype=torch.float64) -> torch.Tensor:
    dev = _lib.require_device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype, non_blocking=a.is_pinned()).contiguous()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(dev).to(dtype).contiguous()


def _to_host(v: torch.Tensor) -> torch.Tensor:
    """Device -> page-locked host copy (a pageable destination runs the DMA
    at a few GB/s; numpy views of the pinned buffer keep it alive)."""
    out = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
    out.copy_(v, non_blocking=True)
    torch.cuda.current_stream(v.device).synchronize()
    return out


def prefix_sum(qs: torch.Tensor) -> torch.Tensor:
    """Inclusive scan of q on the device (replaces np.cumsum, charges.py:130)."""
    n = qs.numel()
    out = torch.empty_like(qs)
    if n == 0:
        return out
    L = _lib.load()
    ws_bytes = L.dt_prefix_scan_workspace(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=qs.device)
    _lib.check(
        L.dt_prefix_scan(_lib.ptr(qs), _lib.ptr(out), n, _lib.ptr(ws), ws_bytes,
                         _lib.stream_handle()),
        "dt_prefix_scan",
    )
    return out


@dataclass(frozen=True, eq=False)
class ChargeSystem:
    """Charges sorted ascending by position (charges.py:28-54).

    ``xs``, ``qs``, ``prefix`` are float64 CUDA tensors; ``prefix[m]`` is the
    sum of the first m + 1 strengths and ``total == prefix[-1]``.
    """

    xs: torch.Tensor
    qs: torch.Tensor
    prefix: torch.Tensor
    total: float | None = None  # None: prefix[-1], read on first access

    def __getattribute__(self, name):
        # the total is read back from the device only when asked for, so
        # building a system does not wait for its prefix scan
        if name == "total":
            v = object.__getattribute__(self, "total")
            if v is None:
                pre = object.__getattribute__(self, "prefix")
                v = float(pre[-1]) if pre.numel() else 0.0
                object.__setattr__(self, "total", v)
            return v
        return object.__getattribute__(self, name)

    def __post_init__(self) -> None:
        for name in ("xs", "qs", "prefix"):
            v = getattr(self, name)
            if not (isinstance(v, torch.Tensor) and v.is_cuda and v.dtype == torch.float64):
                object.__setattr__(self, name, _to_device(v))

    def __len__(self) -> int:
        return int(self.xs.shape[0])

    def __getitem__(self, m: int) -> Charge:
        return Charge(float(self.xs[m]), float(self.qs[m]))

    def __iter__(self) -> Iterator[Charge]:
        for x, q in zip(self.xs.cpu().tolist(), self.qs.cpu().tolist()):
            yield Charge(float(x), float(q))

    def numpy(self) -> tuple[np.ndarray, np.ndarray]:
        return self.xs.cpu().numpy(), self.qs.cpu().numpy()


def from_sorted(xs, qs) -> ChargeSystem:
    """ChargeSystem from positions already sorted ascending (no sort, no copy
    if they are float64 CUDA tensors)."""
    x = _to_device(xs)
    q = _to_device(qs)
    return ChargeSystem(xs=x, qs=q, prefix=prefix_sum(q))


def check_values(v: torch.Tensor, flags: torch.Tensor | None = None) -> torch.Tensor:
    """Enqueue dt_check_values on a contiguous float64 CUDA tensor: returns
    the device flags (non-finite count, descent count), accumulated into
    ``flags`` when given."""
    if flags is None:
        flags = _lib.zeros_i64(2, v.device)
    if v.numel():
        _lib.check(_lib.load().dt_check_values(_lib.ptr(v), v.numel(), _lib.ptr(flags),
                                               _lib.stream_handle()), "dt_check_values")
    return flags


def sort_stable(v: torch.Tensor, payload: torch.Tensor | None = None):
    """(sorted v, permutation int64, payload[perm] or None) on the device:
    the stable radix sort dt_sort_stable (np.argsort(kind="stable"))."""
    n = v.numel()
    out = torch.empty_like(v)
    perm = torch.empty(n, dtype=torch.int64, device=v.device)
    pay = torch.empty_like(payload) if payload is not None else None
    if n:
        L = _lib.load()
        wsb = int(L.dt_sort_workspace(n))
        ws = torch.empty(wsb, dtype=torch.uint8, device=v.device)
        _lib.check(L.dt_sort_stable(_lib.ptr(v), n, _lib.ptr(out), _lib.ptr(perm),
                                    _lib.ptr(payload), _lib.ptr(pay), _lib.ptr(ws), wsb,
                                    _lib.stream_handle()), "dt_sort_stable")
    return out, perm, pay


def permute(src: torch.Tensor, perm: torch.Tensor, scatter: bool = False,
            out: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = src[perm[i]], or out[perm[i]] = src[i] with scatter (dt_permute)."""
    if out is None:
        out = torch.empty_like(src)
    if src.numel():
        _lib.check(_lib.load().dt_permute(_lib.ptr(src), _lib.ptr(perm), src.numel(),
                                          _lib.ptr(out), int(bool(scatter)),
                                          _lib.stream_handle()), "dt_permute")
    return out


def from_particles(raw) -> ChargeSystem:
    """Sorted ChargeSystem from (x, q) pairs (charges.py:114-132).

    Duplicates are kept in input order (stable sort); NaN/inf rejected.  One
    device pass splits the pairs and counts non-finite values and descents.
    """
    if not isinstance(raw, torch.Tensor):
        raw = np.asarray(raw, dtype=np.float64)
    if raw.size == 0 if isinstance(raw, np.ndarray) else raw.numel() == 0:
        raw = raw.reshape(0, 2)
    if raw.ndim != 2 or raw.shape[1] != 2:
        raise ValueError(f"expected (x, q) pairs, got array of shape {tuple(raw.shape)}")
    arr = _to_device(raw)
    if arr.data_ptr() % 16:
        arr = arr.clone()
    n = arr.shape[0]
    x = torch.empty(n, dtype=torch.float64, device=arr.device)
    q = torch.empty(n, dtype=torch.float64, device=arr.device)
    flags = _lib.zeros_i64(2, arr.device)
    if n:
        _lib.check(_lib.load().dt_unpack_pairs(_lib.ptr(arr), n, _lib.ptr(x), _lib.ptr(q),
                                               _lib.ptr(flags), _lib.stream_handle()),
                   "dt_unpack_pairs")
    # the prefix of the (usually already sorted) input is enqueued before the
    # host reads the flags, so the scan runs while the host waits
    pre = prefix_sum(q)
    bad, desc = flags.tolist()
    if bad:
        raise ValueError("positions and strengths must all be finite")
    if desc:  # stable sort by position (charges.py:127), q carried along
        x, _, q = sort_stable(x, q)
        pre = prefix_sum(q)
    return ChargeSystem(xs=x, qs=q, prefix=pre)


def _sign_terms(system: ChargeSystem, targets: torch.Tensor) -> torch.Tensor:
    """e(y) for targets in any order (charges.py:183-187), on the device."""
    out = torch.empty_like(targets)
    T = targets.numel()
    if T == 0:
        return out
    L = _lib.load()
    ws_bytes = int(L.dt_sign_terms_workspace(T))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=targets.device)
    _lib.check(
        L.dt_sign_terms(_lib.ptr(system.xs), _lib.ptr(system.prefix), len(system),
                        _lib.ptr(targets), _lib.ptr(out), T, _lib.ptr(ws), ws_bytes,
                        _lib.stream_handle()),
        "dt_sign_terms",
    )
    return out


def sign_term_all(system: ChargeSystem, targets):
    """e(y) = sum(q_j, x_j < y) - sum(q_j, x_j >= y) for ascending targets
    (charges.py:190-202).  Returns the same kind of array as ``targets``."""
    t, kind = as_targets(targets, check_finite=False)
    if t.numel() > 1 and check_values(t).tolist()[1]:
        raise ValueError("targets must be sorted ascending")
    return kind(_sign_terms(system, t))


def as_targets(targets, check_finite: bool = True):
    """Validate targets (direct.py:43-49) -> (float64 CUDA tensor, converter back).

    The shape check runs on the host before any device work; finiteness is
    checked on the device."""
    if isinstance(targets, torch.Tensor):
        if targets.ndim != 1:
            raise ValueError(f"targets must be one-dimensional, got shape {tuple(targets.shape)}")
        back = (lambda v: v) if targets.is_cuda else _to_host  # noqa: E731
        t = _to_device(targets)
    else:
        arr = np.asarray(targets, dtype=np.float64)
        if arr.ndim != 1:
            raise ValueError(f"targets must be one-dimensional, got shape {arr.shape}")
        back = lambda v: _to_host(v).numpy()  # noqa: E731
        t = _to_device(arr)
    if check_finite and t.numel() and check_values(t).tolist()[0]:
        raise ValueError("targets must all be finite")
    return t, back


def host_targets(targets) -> torch.Tensor | None:
    """The targets as a 1-D float64 CPU tensor when they live on the host
    (numpy / sequence / CPU tensor), else None."""
    if isinstance(targets, torch.Tensor):
        if targets.is_cuda or targets.ndim != 1:
            return None
        return targets.to(torch.float64).contiguous()
    arr = np.asarray(targets, dtype=np.float64)
    if arr.ndim != 1:
        return None
    return torch.from_numpy(np.ascontiguousarray(arr))


# ---------------------------------------------------------------- assembly
# Charge assembly on the device (SURVEY.md §8(f) "next" #2): the step before
# the hot path, so a time-stepping loop never leaves the GPU.

MAX_QUADRATURE_ORDER = 16  # charges.py:111


@dataclass(frozen=True)
class DensitySpec:
    """Line charge density discretised by Gauss-Legendre quadrature
    (charges.py:58-88): ``values`` holds one constant per cell (length
    ``cells``) or endpoint values (length ``cells + 1``, linear in between)."""

    domain: tuple
    cells: int
    values: object
    quadrature_order: int
    eps0: float = 8.8541878128e-12

    def __post_init__(self) -> None:
        a, b = self.domain
        if not (np.isfinite(a) and np.isfinite(b) and a < b):
            raise ValueError(f"domain must be a finite interval, got {self.domain!r}")
        if self.cells < 1:
            raise ValueError(f"cells must be >= 1, got {self.cells!r}")
        if self.quadrature_order < 1:
            raise ValueError(f"quadrature_order must be >= 1, got {self.quadrature_order!r}")
        if self.eps0 <= 0:
            raise ValueError(f"eps0 must be positive, got {self.eps0!r}")
        n_values = len(self.values)
        if n_values not in (self.cells, self.cells + 1):
            raise ValueError(
                f"values must have length cells ({self.cells}) for per-cell constants "
                f"or cells + 1 ({self.cells + 1}) for endpoint tabulation, got {n_values}"
            )


@dataclass(frozen=True)
class ImageSpec:
    """Mirror charges across one or two electrode planes (charges.py:91-108)."""

    gap_length: float
    lower_electrode: float = 0.0
    reflect_lower: bool = True
    reflect_upper: bool = True

    def __post_init__(self) -> None:
        if not (np.isfinite(self.gap_length) and self.gap_length > 0):
            raise ValueError(f"gap_length must be positive, got {self.gap_length!r}")
        if not np.isfinite(self.lower_electrode):
            raise ValueError(f"lower_electrode must be finite, got {self.lower_electrode!r}")


def from_density(spec: DensitySpec) -> ChargeSystem:
    """One charge per Gauss-Legendre node (charges.py:135-161), generated on
    the device (dt_density_nodes, numpy's arithmetic) and passed through
    from_particles; positions and strengths are bit-identical to the
    reference's."""
    if not 1 <= spec.quadrature_order <= MAX_QUADRATURE_ORDER:
        raise ValueError(
            f"quadrature_order must be in 1..{MAX_QUADRATURE_ORDER}, got {spec.quadrature_order}"
        )
    dev = _lib.require_device()
    a, b = spec.domain
    nodes, weights = np.polynomial.legendre.leggauss(spec.quadrature_order)
    values = _to_device(spec.values if isinstance(spec.values, torch.Tensor)
                        else np.asarray(spec.values, dtype=np.float64))
    nd = torch.from_numpy(nodes).to(dev)
    wt = torch.from_numpy(weights).to(dev)
    n = spec.cells * spec.quadrature_order
    pairs = torch.empty((n, 2), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().dt_density_nodes(
        float(a), float(b), int(spec.cells), _lib.ptr(values), values.numel(),
        int(spec.quadrature_order), _lib.ptr(nd), _lib.ptr(wt), float(spec.eps0),
        _lib.ptr(pairs), _lib.stream_handle()), "dt_density_nodes")
    return from_particles(pairs)


def with_images(system: ChargeSystem, spec: ImageSpec) -> ChargeSystem:
    """Add sign-flipped mirror charges across the enabled electrode planes
    (charges.py:164-180): originals, then the kept lower images, then the
    kept upper images, stably sorted (from_particles)."""
    planes = []
    if spec.reflect_lower:
        planes.append(spec.lower_electrode)
    if spec.reflect_upper:
        planes.append(spec.lower_electrode + spec.gap_length)
    n = len(system)
    dev = system.xs.device
    L = _lib.load()
    pairs = torch.empty((n * (1 + len(planes)), 2), dtype=torch.float64, device=dev)
    if n:  # the originals, then each plane's kept images, in index order
        _lib.check(L.dt_pack_sources(_lib.ptr(system.xs), _lib.ptr(system.qs), n,
                                     _lib.ptr(pairs), _lib.stream_handle()), "dt_pack_sources")
    total = n
    if planes and n:
        xm = torch.empty_like(system.xs)
        qm = torch.empty_like(system.qs)
        keep = torch.empty(n, dtype=torch.uint8, device=dev)
        count = torch.empty(1, dtype=torch.int64, device=dev)
        wsb = int(L.dt_compact_workspace(n))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        for plane in planes:
            _lib.check(L.dt_mirror_charges(
                _lib.ptr(system.xs), _lib.ptr(system.qs), n, float(plane),
                float(spec.gap_length), _lib.ptr(xm), _lib.ptr(qm), _lib.ptr(keep),
                _lib.stream_handle()), "dt_mirror_charges")
            _lib.check(L.dt_compact_pairs(_lib.ptr(xm), _lib.ptr(qm), _lib.ptr(keep), n,
                                          _lib.ptr(pairs), total, _lib.ptr(count), _lib.ptr(ws),
                                          wsb, _lib.stream_handle()), "dt_compact_pairs")
            total += int(count.item())
    return from_particles(pairs[:total])
