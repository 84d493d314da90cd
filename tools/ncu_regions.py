"""Traversal-kernel instruction and stall-sample shares by code region (dev aid).

    python tools/ncu_regions.py <eval.ncu-rep> [source-file]

Regions are the functions of csrc/dt_eval.cu (line ranges found from the
source), everything else is the walk.  Reports instructions per 32-target
task (2^24 targets) and the share of warp-stall samples.
"""
import collections, csv, re, subprocess, sys

rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_1710_05781_b200/csrc/dt_eval.cu"
lines = open(src).read().split("\n")
def span(pat):
    i = next(k for k, l in enumerate(lines) if re.search(pat, l))
    depth, j, seen = 0, i, False
    while True:
        depth += lines[j].count("{") - lines[j].count("}")
        seen = seen or "{" in lines[j]
        if seen and depth == 0:
            return i + 1, j + 1
        j += 1
regions = {
    "far_field": span(r"double far_field\("),
    "near_field": span(r"double near_field\("),
    "near_term": span(r"double near_term\("),
    "psel_table": span(r"int psel_table\("),
    "psel_fast": span(r"int psel_fast\("),
    "pt_level": span(r"int pt_level\("),
}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; hdr = None; line = None
ins = collections.Counter(); st = collections.Counter()
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        line = (cur, int(r[0]))
    try: k = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError: k = 0
    try: s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError: s = 0
    if line is None:
        continue
    name = "other-file:" + line[0]
    if line[0] == "dt_eval.cu":
        name = next((n for n, (a, b) in regions.items() if a <= line[1] <= b), "walk/kernel")
    elif line[0] == "dt_common.cuh":
        name = "dt_common (rsqrt, loads)"
    ins[name] += k; st[name] += s
T = 2**24 / 32
tot_s = sum(st.values()) or 1
for n in sorted(ins, key=lambda n: -st[n]):
    print(f"{n:28s} {ins[n]/T:8.0f} instr/task  {100*st[n]/tot_s:5.1f}% of stall samples")
print(f"{'total':28s} {sum(ins.values())/T:8.0f}")
