"""Small end-to-end run of every device path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run):

  compute-sanitizer --tool memcheck python tools/sanitize_run.py

Graded configs[2] mesh at 2^14 sources (deep tree: the build's block-0 level
runs and flag wait, the upward pass's arrival protocol), the device-resident
step, the public API on device / pinned / pageable targets, the sharded
upward pass for 2 ranks run one after the other (plan, partial pass, pack,
finish), the direct sums (plain, Kahan, fp32, pair-symmetric), the adaptive
order tables and charge assembly."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W
from paper_1710_05781_b200.parallel import ShardedMoments, shard_bounds
from paper_1710_05781_b200.pipeline import TreePipeline
from paper_1710_05781_b200.tree import TreeBuffers, eval_stride, moment_order_for, tree_phi_sum

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 12
w = W.cfg2(cells=cells)
k = dt.DiscKernel(w.r_d)
cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=True, tolerance=w.tolerance)
pairs = torch.from_numpy(np.column_stack([w.xs, w.qs])).cuda()
system = dt.from_particles(pairs)
tree = dt.build(system, k, cfg)
ys = torch.from_numpy(w.targets).cuda()
e_dev = dt.evaluate_all(tree, k, cfg, system, ys).values
e_host = dt.evaluate_all(tree, k, cfg, system, w.targets).values
e_pin = dt.evaluate_all(tree, k, cfg, system, torch.from_numpy(w.targets).pin_memory()).values
perm = np.random.default_rng(0).permutation(len(w.targets))
e_perm = dt.evaluate_all(tree, k, cfg, system, w.targets[perm]).values
_ = tree.moments  # reference layout derived from the traversal rows
# device-resident step, world 1
xs, qs = system.xs, system.qs
pipe = TreePipeline.planned(xs, ys.numel(), k, cfg)
out = torch.empty_like(ys)
for _ in range(2):
    pipe.step(xs, qs, ys, out)
pipe.check()
# sharded upward pass, 2 ranks one after the other on this GPU
G = 2
bufs = TreeBuffers(len(system), len(tree) + 64, xs.device)
bufs.launch(xs, cfg.leaf_capacity)
order = moment_order_for(cfg)
es = eval_stride(order)
sends, shards = [], []
for r in range(G):
    i0, i1 = shard_bounds(ys.numel(), G, r)
    me = torch.full((bufs.capacity, es), float("nan"), dtype=torch.float64, device="cuda")
    sh = ShardedMoments(bufs, order, None, me, es, cfg.theta, G, r)
    sends.append(sh.local(xs, qs, ys[i0:i1].contiguous(), True).clone())
    shards.append((sh, me, i0, i1))
recv = torch.cat(sends)
for sh, me, i0, i1 in shards:
    sh.finish(recv)
# direct sums
t = ys[::7].contiguous()
d64 = dt.evaluate_direct(system, k, t).values
d32 = dt.evaluate_direct(system, k, t, precision="fp32").values
dk = dt.evaluate_direct(system, k, t[:256], compensated=True).values
dsym = dt.evaluate_direct(system, k, xs).values
# assembly
spec = dt.DensitySpec(domain=(0.0, 1.0), cells=512, values=list(np.linspace(1, 2, 513)),
                      quadrature_order=4)
sys2 = dt.with_images(dt.from_density(spec), dt.ImageSpec(gap_length=1.0))
torch.cuda.synchronize()
assert np.array_equal(e_host, e_dev.cpu().numpy()) and np.array_equal(e_pin.numpy(), e_host)
assert np.array_equal(e_perm, e_host[perm])
assert torch.equal(out, e_dev)
print(f"sanitize run ok: N={len(system)} nodes={len(tree)} depth={tree.depth} "
      f"direct={float(d64.abs().sum()):.6e} sym={float(dsym.abs().sum()):.6e} images={len(sys2)}")
