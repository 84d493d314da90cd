"""Benchmark: tree field evaluations per second at N = 2^24, tolerance 1e-10.

BASELINE.json metric "tree field evals (targets/s) at N=2^24, tol 1e-10";
workload configs[2] (graded streamer mesh, 2^24 sources = targets, r_d =
0.005, adaptive order from the 1e-10 bound, leaf 64).  One step = the whole
hot path on one batch: prefix scan + sign term, tree build, P2M/M2M moments,
traversal (far + near field).  Inputs are resident in HBM for `value`; `e2e`
runs the public API (from_particles -> build -> evaluate_all) from pinned
host buffers with the copies inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (targets sharded by rank)

`--impl reference` times the reference algorithm on the host cores (the C
restatement in oracle/, all threads) on the same config and prints the same
JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "tree field evals (targets/s) at N=2^24, tol 1e-10"
UNIT = "targets/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cells", type=int, default=1 << 22, help="GL cells (N = 4 * cells)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU-baseline eval sample budget (seconds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload(cells):
    from paper_1710_05781_b200 import workloads as W

    return W.cfg2(cells=cells)


def config_dict(w, n_gpus):
    return {
        "workload": "configs[2]: graded streamer mesh (ratio 1.0005 toward x=0.3, max/min "
                    "width 1e4), sigma = 1e-3 exp(-((x-0.3)/1e-3)^2) + seeded exp tail",
        "n_sources": int(w.n), "n_targets": int(len(w.targets)), "r_d": w.r_d,
        "tolerance": w.tolerance, "adaptive": True, "leaf_capacity": w.leaf_capacity,
        "theta": w.theta, "moment_order": 30, "seed": w.meta.get("seed"),
        "sharding": f"contiguous target slices over {n_gpus} rank(s), sources replicated",
        "l2": "inputs (3 x 8 x 2^24 B = 403 MB) exceed the 126 MB L2; no flush needed",
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.lines: list[str] = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-i", str(self.gpu), "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
            self.lines.clear()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in list(self.lines):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ peaks
def measure_fp64_peak(torch, L, ptr, stream):
    """DFMA probe: 148 x 8 CTAs x 256 threads x 8 chains (TFLOP/s, best of 3)."""
    blocks, iters = 148 * 8, 20000
    out = torch.empty(blocks * 256, dtype=torch.float64, device="cuda")
    best = 0.0
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.dt_fp64_probe(ptr(out), iters, blocks, stream())
        b.record()
        torch.cuda.synchronize()
        best = max(best, 16.0 * iters * blocks * 256 / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best


def ncu_traffic():
    """dram bytes per launch of the traversal kernel from a committed ncu
    --set full capture summary (profiles/), else None."""
    path = os.path.join(REPO, "profiles", "ncu_eval_cfg2.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


# ------------------------------------------------------------------ CPU oracle
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_rate(w, seconds: float, threads: int | None = None):
    """Reference algorithm (oracle/ C restatement) on the host cores: full
    build + a strided target sample sized to ~`seconds`, extrapolated to all
    targets.  Returns (targets/s, info)."""
    from oracle import oracle as O

    if threads:
        O.set_threads(threads)
    cores = O.num_threads()
    t0 = time.perf_counter()
    tree = O.build(w.xs, w.qs, w.p, w.leaf_capacity, w.adaptive)
    t_build = time.perf_counter() - t0
    pre = O.prefix(w.qs)
    T = len(w.targets)
    tol = O.tol_share(w.tolerance, tree.depth)
    pilot = w.targets[:: max(1, T // 512)]
    t0 = time.perf_counter()
    O.tree_phi_sum(tree, w.xs, w.qs, w.r_d**2, w.theta, w.p, w.adaptive, tol, pilot)
    per = (time.perf_counter() - t0) / len(pilot)
    S = int(min(T, max(len(pilot), seconds / max(per, 1e-9))))
    stride = max(1, T // S)
    sample = w.targets[::stride]
    t0 = time.perf_counter()
    e = O.sign_terms(w.xs, pre, float(pre[-1]), sample)
    O.tree_phi_sum(tree, w.xs, w.qs, w.r_d**2, w.theta, w.p, w.adaptive, tol, sample)
    t_eval = time.perf_counter() - t0
    t_full = t_build + t_eval * T / len(sample)
    info = {
        "cores": cores, "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
        "sample": f"full build ({len(tree)} nodes, {t_build:.2f} s) + every {stride}-th target "
                  f"({len(sample)} of {T}, {t_eval:.2f} s), eval extrapolated to all targets",
        "build_s": t_build, "eval_sample_s": t_eval, "n_sample": len(sample),
    }
    del e
    return T / t_full, info


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(args.cells)
    # each timed step: full build + an eval sample; the whole run stays
    # within a few minutes.  Warm-up steps run a small pilot only.
    budget = max(1.0, 120.0 / max(1, args.steps))
    from paper_1710_05781_b200 import workloads as W

    small = W.cfg2(cells=4096)
    for _ in range(args.warmup):
        cpu_reference_rate(small, seconds=0.05)
    rates = []
    info = None
    for _ in range(args.steps):
        r, info = cpu_reference_rate(w, seconds=budget * 0.5)
        rates.append(r)
    value = float(np.mean(rates))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": len(w.targets) / value * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(w, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "port",
                         "sample": info["sample"], "cpu_model": info["cpu_model"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1710_05781_b200 as dtp
    from paper_1710_05781_b200 import _lib
    from paper_1710_05781_b200.parallel import build_sharded
    from paper_1710_05781_b200.pipeline import TreePipeline
    from paper_1710_05781_b200.tree import tree_phi_sum

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % torch.cuda.device_count()  # several ranks per GPU only in gloo test mode
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink; DISCTREE_BENCH_BACKEND=gloo only to exercise the
        # multi-rank code path with several ranks on one GPU (no timing value)
        backend = os.environ.get("DISCTREE_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # communicator init lines (nranks, NVLS/NVLink transport) on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        nccl_info = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                     "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
        if rank == 0:
            print(f"[bench] process group {nccl_info}", file=sys.stderr, flush=True)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    w = workload(args.cells)
    T = len(w.targets)
    i0, i1 = rank * T // world, (rank + 1) * T // world
    kernel = dtp.DiscKernel(w.r_d)
    cfg = dtp.EvalConfig(p=w.p, theta=w.theta, leaf_capacity=w.leaf_capacity,
                         adaptive=w.adaptive, tolerance=w.tolerance)
    xs = torch.from_numpy(w.xs).cuda()
    qs = torch.from_numpy(w.qs).cuda()
    ys = torch.from_numpy(w.targets).cuda()
    out = torch.empty_like(ys)
    pipe = TreePipeline.planned(xs, T, kernel, cfg, world=world, rank=rank)

    # algorithmic work of this rank's slice (stats pass, outside the timed region)
    system = dtp.from_sorted(xs, qs)
    tree = dtp.build(system, kernel, cfg)
    names = ("hash", "near_pairs", "n_far", "sum_p", "n_p0", "n_exact")
    sb = {k: torch.zeros(T, dtype=torch.int64, device="cuda") for k in names}
    st = _lib.EvalStats(*[sb[k].data_ptr() for k in names])
    tree_phi_sum(tree, kernel, cfg, ys, torch.zeros_like(ys), i0=i0, i1=i1, accumulate=False,
                 stats=st)
    sl = slice(i0, i1)
    near = int(sb["near_pairs"][sl].sum())
    nfar = int(sb["n_far"][sl].sum())
    sump = int(sb["sum_p"][sl].sum())
    np0 = int(sb["n_p0"][sl].sum())
    nexact = int(sb["n_exact"][sl].sum())
    flops = 14 * near + 20 * (nfar - np0) + 11 * sump + 14 * np0
    tree_info = {"nodes": len(tree), "depth": tree.depth, "leaves": tree.leaf_count}
    del sb, tree, system

    L = _lib.load()
    peak = measure_fp64_peak(torch, L, _lib.ptr, _lib.stream_handle)

    for _ in range(args.warmup):
        pipe.step(xs, qs, ys, out, i0, i1)
    torch.cuda.synchronize()
    pipe.check()

    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    t_start.record()
    for k in range(args.steps):
        pipe.step(xs, qs, ys, out, i0, i1, eval_events=ev[k])
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end) / args.steps
    eval_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    pipe.check()
    ms_max = allmax(ms)
    value = T / (ms_max * 1e-3)

    # spot-check the pipelined result against the public API on a sample
    res = dtp.evaluate_all(dtp.build(dtp.from_sorted(xs, qs), kernel, cfg), kernel, cfg,
                           dtp.from_sorted(xs, qs), ys[i0:i1][::997])
    diff = float((out[i0:i1][::997] - res.values).abs().max())
    scale = float(np.abs(w.qs).sum())

    # end to end through the public API, pinned host buffers, copies timed
    pairs = torch.from_numpy(np.column_stack([w.xs, w.qs])).pin_memory()
    tgt = torch.from_numpy(w.targets[i0:i1].copy()).pin_memory()
    vout = torch.empty(tgt.numel(), dtype=torch.float64).pin_memory()
    e2e_times = []
    for k in range(2 + args.e2e_steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sysm = dtp.from_particles(pairs)
        if world == 1:
            tr = dtp.build(sysm, kernel, cfg)
            vals = dtp.evaluate_all(tr, kernel, cfg, sysm, tgt).values
        else:  # same tree on every rank, sharded upward pass for this rank's targets
            tdev = tgt.cuda(non_blocking=True)
            tr = build_sharded(sysm, kernel, cfg, tdev, world, rank, targets_sorted=True)
            vals = vout.copy_(dtp.evaluate_all(tr, kernel, cfg, sysm, tdev).values,
                              non_blocking=True)
        torch.cuda.synchronize()
        dt_s = time.perf_counter() - t0
        barrier()
        if k > 1:
            e2e_times.append(dt_s)
        del sysm, tr, vals
    e2e_s = allmax(float(np.mean(e2e_times)))
    e2e = {"value": T / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(pairs.numel() * 8 +
                                                                      tgt.numel() * 8),
           "d2h_bytes_per_step": int(tgt.numel() * 8), "ms_per_step": e2e_s * 1e3,
           "ms_per_call": [round(t * 1e3, 3) for t in e2e_times],
           "api": "from_particles(pinned (N,2)) -> build -> evaluate_all(pinned targets)"}

    flops_all = allsum(flops)
    achieved = flops / (eval_ms * 1e-3) / 1e12
    roofline = {
        "bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak, "traffic": ncu_traffic(),
        "kernel": "tree_eval_kernel<adaptive> (dt_tree_eval_device)",
        "algorithmic_flops_per_launch": flops,
        "work_units": "W = 14*near_pairs + sum_far F_far(p), F_far = 20 + 11p (14 at p=0); "
                      "SURVEY 8(d)",
        "eval_ms": eval_ms, "share_of_step": eval_ms / ms,
        "peak_source": "measured DFMA probe (dt_fp64_probe) in this run; MEASURED_PEAKS.json "
                       "has no fp64 entry",
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config_dict(w, world), **tree_info),
        "e2e": e2e, "roofline": roofline, "clocks": clk,
        "gpu_launches": pipe.launches_per_step * args.steps,
        "interactions": {"near_pairs_per_target": near / max(1, i1 - i0),
                         "far_per_target": nfar / max(1, i1 - i0),
                         "mean_p": sump / max(1, nfar), "exact_tier_frac": nexact / max(1, nfar),
                         "flops_all_ranks": flops_all},
        "check": {"max_abs_diff_vs_api_over_sum_abs_q": diff / scale},
    }
    if world > 1:
        line["process_group"] = nccl_info
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, info = cpu_reference_rate(w, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": info["cores"],
                                "kind": "port", "sample": info["sample"],
                                "cpu_model": info["cpu_model"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
