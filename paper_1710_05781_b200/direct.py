"""O(N*T) direct evaluator: sign term + full pair sum (stage (f)).

Mirror of disctree.direct (direct.py:23-88).  The pair sum runs in
csrc/dt_direct.cu: fp64 (phi_sum_plain), Kahan (phi_sum_kahan, bit-identical)
or the fp32-evaluation / fp64-accumulation bench variant.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from . import _lib


@dataclass(frozen=True)
class FieldResult:
    """Field values plus timings (direct.py:23-40)."""

    values: object
    build_time: float
    eval_time: float
    method: str

    def __post_init__(self) -> None:
        if self.method not in ("tree", "direct"):
            raise ValueError(f"method must be 'tree' or 'direct', got {self.method!r}")
        if self.build_time < 0 or self.eval_time < 0:
            raise ValueError("timings must be nonnegative")


def phi_sum_direct(xs: torch.Tensor, qs: torch.Tensor, ys: torch.Tensor, rd2: float,
                   out: torch.Tensor, mode: int = _lib.DT_DIRECT_FP64, accumulate: bool = True,
                   i0: int = 0, i1: int | None = None) -> None:
    """out[i] (+)= sum_j q_j (x_j - y_i)/sqrt((x_j - y_i)^2 + rd2), i in [i0, i1)."""
    if i1 is None:
        i1 = ys.numel()
    if i1 <= i0:
        return
    p = _lib.ptr
    _lib.check(
        _lib.load().dt_phi_sum_direct(p(xs), p(qs), xs.numel(), p(ys), float(rd2), p(out),
                                      int(i0), int(i1), int(mode), int(bool(accumulate)),
                                      _lib.stream_handle()),
        "dt_phi_sum_direct",
    )


# Upper bound on the symmetric path's partial-sum workspace (bytes); above it
# evaluate_direct takes the plain kernel (same values to round-off).
SYM_MAX_WORKSPACE = 8 << 30


def phi_sum_symmetric(xs: torch.Tensor, qs: torch.Tensor, rd2: float, out: torch.Tensor,
                      accumulate: bool = True) -> bool:
    """out[i] (+)= sum_j q_j (x_j - x_i)/sqrt((x_j - x_i)^2 + rd2) for targets ==
    sources, each pair evaluated once (_kernels.phi_sum_symmetric,
    _kernels.py:107-142).  Returns False (nothing done) when the partial
    sums (~4 n^2 / 2048 bytes: 2 GB at n = 2^20, 8 GB at 2^21) would exceed
    SYM_MAX_WORKSPACE or a quarter of the free device memory; the caller
    then uses the plain kernel."""
    n = xs.numel()
    if n == 0:
        return True
    L = _lib.load()
    need = int(L.dt_phi_sum_symmetric_workspace(n))
    free, _ = torch.cuda.mem_get_info(xs.device)
    if need > min(free // 4, SYM_MAX_WORKSPACE):
        return False
    ws = torch.empty(need, dtype=torch.uint8, device=xs.device)
    p = _lib.ptr
    _lib.check(
        L.dt_phi_sum_symmetric(p(xs), p(qs), n, float(rd2), p(out), int(bool(accumulate)),
                               p(ws), need, _lib.stream_handle()),
        "dt_phi_sum_symmetric",
    )
    return True


def evaluate_direct(system, kernel, targets, threads: int | None = 1,
                    compensated: bool = False, *, precision: str = "fp64"):
    """Field at every target by direct summation (direct.py:52-88).

    ``compensated=True`` selects the Kahan kernel (bit-identical to the
    reference's).  ``precision="fp32"`` selects fp32 pair evaluation with
    fp64 accumulation (bench variant; not in the reference).  ``threads`` is
    accepted for API compatibility; results do not depend on it.
    """
    from .charges import _sign_terms, as_targets

    t, back = as_targets(targets)
    if precision not in ("fp64", "fp32"):
        raise ValueError(f"precision must be 'fp64' or 'fp32', got {precision!r}")
    dev = t.device
    torch.cuda.synchronize(dev)
    start = time.perf_counter()
    values = _sign_terms(system, t)
    mode = _lib.DT_DIRECT_KAHAN if compensated else (
        _lib.DT_DIRECT_FP32 if precision == "fp32" else _lib.DT_DIRECT_FP64)
    rd2 = kernel.r_d * kernel.r_d
    # targets == sources: each pair once (direct.py:80 -> phi_sum_symmetric)
    done = (mode == _lib.DT_DIRECT_FP64 and t.numel() == system.xs.numel()
            and bool(torch.equal(t, system.xs))
            and phi_sum_symmetric(system.xs, system.qs, rd2, values))
    if not done:
        phi_sum_direct(system.xs, system.qs, t, rd2, values, mode)
    torch.cuda.synchronize(dev)
    elapsed = time.perf_counter() - start
    return FieldResult(values=back(values), build_time=0.0, eval_time=elapsed, method="direct")
