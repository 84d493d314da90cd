"""Copy a bench line + ncu artefacts from gpurun_out/ into profiles/ summaries.

    python tools/summarize_profiles.py <tag> <bench.json> <launches.csv> <eval.ncu-rep>
"""
import csv, io, json, os, shutil, subprocess, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, bench, launches, rep = sys.argv[1:5]
prof = os.path.join(REPO, "profiles")
shutil.copy(bench, os.path.join(prof, f"{tag}_bench_cfg2.json"))
shutil.copy(launches, os.path.join(prof, f"{tag}_launches_cfg2.csv"))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
g = lambda n: float(v[h.index(n)])
unit = lambda n: u[h.index(n)]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
dram = g("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")] + \
    g("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
b = json.load(open(bench))
d = {
    "tag": tag,
    "kernel": "tree_eval_kernel<adaptive=1,stats=0,wide=0> (dt_tree_eval_device)",
    "workload": "configs[2] 2^24 sources = targets, tol 1e-10",
    "capture": "ncu --set full --clock-control none --import-source on -k regex:tree_eval -s 1 -c 1 python tools/prof_eval.py",
    "duration_ms": g("gpu__time_duration.sum") * (1 if unit("gpu__time_duration.sum") == "ms" else 1e-3),
    "dram_bytes_per_launch": dram,
    "instructions": g("smsp__inst_executed.sum"),
    "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers": g("launch__registers_per_thread"),
    "threads_per_inst": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "algorithmic_bytes_per_launch": 16 * 2**24 + 8 * 2**24 + 16 * 2**24 + (32 + 8 * 32) * b["config"]["nodes"],
    "algorithmic_flops_per_launch": b["roofline"]["algorithmic_flops_per_launch"],
    "bench_eval_ms": b["roofline"]["eval_ms"],
    "bench_achieved_tflops": b["roofline"]["achieved"],
    "bench_fp64_peak_tflops": b["roofline"]["peak"],
}
json.dump(d, open(os.path.join(prof, "ncu_eval_cfg2.json"), "w"), indent=1)
lines = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_lines.py"), rep, "40"],
                       capture_output=True, text=True).stdout
open(os.path.join(prof, f"{tag}_ncu_eval_cfg2_lines.txt"), "w").write(lines)
print(json.dumps(d, indent=1))

# optional 5th argument: ncu report of the build / moments kernels
if len(sys.argv) > 5:
    raw = subprocess.run(["ncu", "-i", sys.argv[5], "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    nodes, leaves = b["config"]["nodes"], b["config"]["leaves"]
    N, P1 = 2**24, 31
    # B_build = 8N + 72 nodes; B_P2M + B_M2M = 16N + 8(P+1) leaves
    # + 24(P+1) internal nodes (the fused upward kernel does both); B_scan = 16N
    # over the two scan passes (reported per pass: q read + prefix write).
    alg = {"build_kernel": 8 * N + 72 * nodes,
           "upward_kernel": 16 * N + 8 * P1 * leaves + 24 * P1 * (nodes - leaves),
           "moments_prep_kernel": 0,
           "tile_sums_kernel": 8 * N,
           "tile_apply_kernel": 8 * N + 8 * N}
    aux = {"capture": "ncu --set full --clock-control none --import-source on -k "
                      "regex:'build_kernel|upward|moments_prep|tile_' -s 6 -c 5 python "
                      "tools/prof_eval.py (configs[2]; the second pipeline step)",
           "note": "ncu flushes caches between kernels: tile_apply's L2 reuse of q is not "
                   "seen here; moments_prep (parent / arrival bookkeeping) has no 8(d) bytes",
           "kernels": []}
    for v in r[2:]:
        gv = lambda k: float(v[h.index(k)]) * scale.get(u[h.index(k)], 1)
        name = v[h.index("Kernel Name")]
        key = next(k for k in alg if k in name)
        t = float(v[h.index("gpu__time_duration.sum")]) * (
            1e-3 if u[h.index("gpu__time_duration.sum")] == "us" else 1)
        aux["kernels"].append({
            "kernel": name.split("(")[0], "duration_ms": t,
            "dram_bytes": gv("dram__bytes_read.sum") + gv("dram__bytes_write.sum"),
            "algorithmic_bytes": alg[key], "algorithmic_GBps": alg[key] / (t * 1e-3) / 1e9,
            "frac_of_hbm_6553GBps": alg[key] / (t * 1e-3) / 1e9 / 6553.0,
            "fp64_pipe_active_pct": float(v[h.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")]),
            "issue_active_pct": float(v[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]),
            "warps_active_pct": float(v[h.index("sm__warps_active.avg.pct_of_peak_sustained_active")]),
        })
    json.dump(aux, open(os.path.join(prof, f"{tag}_ncu_aux_cfg2.json"), "w"), indent=1)
    for kk in aux["kernels"]:
        print(kk["kernel"], "%.3f ms" % kk["duration_ms"], "%.0f GB/s" % kk["algorithmic_GBps"])
