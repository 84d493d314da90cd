"""Summarise an ncu --set full capture of the step's non-traversal kernels.

    python tools/summarize_aux.py <tag> <bench.json> <aux.ncu-rep>

Writes profiles/<tag>_ncu_aux_cfg2.json.  Algorithmic bytes per SURVEY.md
§8(d): B_scan = 16N over the two scan passes, B_build = 8N + 72 nodes,
B_P2M = 16N + 8(P+1) leaves, B_M2M = 24(P+1) internal nodes, sign = 16T.
The build kernel also forms the leaves of the levels its block 0 has
finished (dt_build_tree_p2m), so build and upward are also reported together
against B_build + B_P2M + B_M2M.
"""
import csv, io, json, os, subprocess, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, bench, rep = sys.argv[1:4]
b = json.load(open(bench))
nodes, leaves = b["config"]["nodes"], b["config"]["leaves"]
N = T = 2**24
P1 = 31
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
B_build = 8 * N + 72 * nodes
B_up = 16 * N + 8 * P1 * leaves + 24 * P1 * (nodes - leaves)
alg = {"build_kernel": B_build, "upward_kernel": 24 * P1 * (nodes - leaves),
       "moments_prep_kernel": 0, "tile_sums_kernel": 8 * N, "tile_apply_kernel": 16 * N,
       "sign_bracket_kernel": 0, "sign_terms_kernel": 16 * T}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u = r[0], r[1]
out = {"capture": "ncu --set full --clock-control none --import-source on -k "
                  "regex:'build_kernel|upward|moments_prep|tile_|sign_' python tools/prof_eval.py "
                  "(configs[2]; the second pipeline step)",
       "note": "ncu flushes caches and serialises kernels: tile_apply's L2 reuse of q is not "
               "seen, and the sign kernels (a side stream in the bench) run alone here; "
               "build_kernel's algorithmic bytes are B_build only, it also runs most of P2M",
       "kernels": []}
seen = set()
tot = {}
for v in r[2:]:
    name = v[h.index("Kernel Name")]
    key = next((k for k in alg if k in name), None)
    if key is None or key in seen:
        continue
    seen.add(key)
    gv = lambda k: float(v[h.index(k)]) * scale.get(u[h.index(k)], 1)
    t = float(v[h.index("gpu__time_duration.sum")]) * {"ns": 1e-6, "us": 1e-3, "ms": 1}[
        u[h.index("gpu__time_duration.sum")]]
    tot[key] = t
    out["kernels"].append({
        "kernel": name.split("(")[0], "duration_ms": t,
        "dram_bytes": gv("dram__bytes_read.sum") + gv("dram__bytes_write.sum"),
        "algorithmic_bytes": alg[key],
        "algorithmic_GBps": alg[key] / (t * 1e-3) / 1e9,
        "frac_of_hbm_6553GBps": alg[key] / (t * 1e-3) / 1e9 / 6553.0,
        "fp64_pipe_active_pct": float(v[h.index("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")]),
        "issue_active_pct": float(v[h.index("smsp__issue_active.avg.pct_of_peak_sustained_active")]),
        "warps_active_pct": float(v[h.index("sm__warps_active.avg.pct_of_peak_sustained_active")]),
    })
if "build_kernel" in tot and "upward_kernel" in tot:
    t = tot["build_kernel"] + tot["upward_kernel"] + tot.get("moments_prep_kernel", 0)
    out["build_plus_moments"] = {
        "duration_ms": t, "algorithmic_bytes": B_build + B_up,
        "algorithmic_GBps": (B_build + B_up) / (t * 1e-3) / 1e9,
        "frac_of_hbm_6553GBps": (B_build + B_up) / (t * 1e-3) / 1e9 / 6553.0}
json.dump(out, open(os.path.join(REPO, "profiles", f"{tag}_ncu_aux_cfg2.json"), "w"), indent=1)
for k in out["kernels"]:
    print("%-40s %.3f ms %6.0f GB/s" % (k["kernel"], k["duration_ms"], k["algorithmic_GBps"]))
print(out.get("build_plus_moments"))
