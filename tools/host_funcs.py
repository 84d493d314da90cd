"""Per-function host time (inclusive, microseconds) of the public API calls,
GPU idle before each call (dev aid: the host work that precedes launches)."""
import functools, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, tree as TR, charges as CH, _lib
w = W.cfg2()
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
pairs = torch.from_numpy(np.column_stack([w.xs, w.qs])).pin_memory()
tgt = torch.from_numpy(w.targets.copy()).pin_memory()
acc = {}
def wrap(mod, name):
    f = getattr(mod, name)
    @functools.wraps(f)
    def g(*a, **kw):
        t = time.perf_counter_ns()
        try:
            return f(*a, **kw)
        finally:
            acc[f"{mod.__name__.split('.')[-1]}.{name}"] = acc.get(f"{mod.__name__.split('.')[-1]}.{name}", 0) + time.perf_counter_ns() - t
    setattr(mod, name, g)
for n in ["_looks_sorted", "contour_tables", "_workspace", "_timing_events", "_elapsed", "as_targets",
          "_evaluate_host_mapped", "_build", "launch_moments", "initial_node_capacity", "_tol_share"]:
    if hasattr(TR, n): wrap(TR, n)
for n in ["prefix_sum", "_to_device"]:
    if hasattr(CH, n): wrap(CH, n)
wrap(_lib, "zeros_i64"); wrap(_lib, "check")
_tb_init = TR.TreeBuffers.__init__
def _tb(self, *a, **kw):
    t = time.perf_counter_ns()
    _tb_init(self, *a, **kw)
    acc["TreeBuffers.__init__"] = acc.get("TreeBuffers.__init__", 0) + time.perf_counter_ns() - t
TR.TreeBuffers.__init__ = _tb
for _ in range(3):
    s = dt.from_particles(pairs); tr = dt.build(s, k, cfg); v = dt.evaluate_all(tr, k, cfg, s, tgt).values
acc.clear()
R = 5
for _ in range(R):
    s = dt.from_particles(pairs); torch.cuda.synchronize()
    tr = dt.build(s, k, cfg); torch.cuda.synchronize()
    v = dt.evaluate_all(tr, k, cfg, s, tgt).values
for kname, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{kname:32s} {v / R / 1e3:9.1f} us")
