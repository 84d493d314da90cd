"""dt_tree_field_packed with targets/results in HBM vs in pinned host memory
(same kernel; dev aid for the cost of reading targets over the host link)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, _lib
from paper_1710_05781_b200.tree import _tol_share, contour_tables
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
system = dt.from_sorted(w.xs, w.qs)
tree = dt.build(system, k, cfg)
L, p = _lib.load(), _lib.ptr
cos_t, sin_t = contour_tables(system.xs.device)
T = len(w.targets)
ws = torch.empty(int(L.dt_tree_field_workspace(T)), dtype=torch.uint8, device="cuda")
for where in ("cuda", "pinned", "cuda", "pinned"):
    ys = torch.from_numpy(w.targets.copy())
    ys = ys.cuda() if where == "cuda" else ys.pin_memory()
    out = torch.empty_like(ys)
    if where == "pinned":
        out = out.pin_memory()
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = L.dt_tree_field_packed(
            p(tree.packed), len(tree), p(tree.meval), tree.meval.shape[1], p(tree.xq),
            p(system.xs), p(system.prefix), len(system), k.r_d ** 2, float(cfg.theta),
            int(cfg.p), 1, _tol_share(tree, cfg), int(tree.moment_order), p(cos_t), p(sin_t),
            cos_t.numel(), ys.data_ptr(), out.data_ptr(), 0, T, None, p(ws), ws.numel(),
            torch.cuda.current_stream().cuda_stream)
        b.record()
        torch.cuda.synchronize()
        assert rc == 0
        ts.append(a.elapsed_time(b))
    print(where, "field ms", ["%.3f" % t for t in ts])
