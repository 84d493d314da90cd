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
