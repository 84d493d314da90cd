"""ncu summaries of the direct kernels at configs[4] -> profiles/<tag>_ncu_direct_cfg4.json

    python tools/summarize_direct.py <tag> <report.ncu-rep> [<report2.ncu-rep> ...]
"""
import csv, io, json, math, os, subprocess, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, reps = sys.argv[1], sys.argv[2:]
out = {"capture": "ncu --set full --clock-control none -k regex:<kernel> python tools/direct_time.py "
                  "(configs[4]: 2^20 sources = targets, r_d = 0.01)",
       "note": "ncu durations are serialised replays; the symmetric path is three launches "
               "(sym_band_kernel carries all but ~0.2% of the pairs)",
       "kernels": []}
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u = r[0], r[1]
    for v in r[2:]:
        g = lambda k: float(v[h.index(k)])
        if math.isnan(g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")):
            continue
        unit = u[h.index("gpu__time_duration.sum")]
        out["kernels"].append({
            "kernel": v[h.index("Kernel Name")].split("(")[0],
            "duration_ms": g("gpu__time_duration.sum") * {"ms": 1, "us": 1e-3, "s": 1e3}[unit],
            "fp64_pipe_active_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "registers": g("launch__registers_per_thread"),
        })
json.dump(out, open(os.path.join(REPO, "profiles", f"{tag}_ncu_direct_cfg4.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
