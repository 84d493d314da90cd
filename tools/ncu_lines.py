"""Aggregate an ncu source page (cuda,sass) by CUDA source line."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; agg = collections.Counter(); stall = collections.Counter(); src = {}; line = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        line = (cur, int(r[0])); src[line] = r[1]
    try: k = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError: k = 0
    try: s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError: s = 0
    if line: agg[line] += k; stall[line] += s
tot = sum(agg.values()) or 1; stot = sum(stall.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{k[0]}:{k[1]:4d} {v/tot*100:5.1f}% stall {stall[k]/stot*100:5.1f}%  {src[k].strip()[:90]}")
