"""Ad-hoc stage timing on one GPU (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1710_05781_b200 as dt
from paper_1710_05781_b200 import workloads as W, _lib
from paper_1710_05781_b200.tree import TreeBuffers, launch_moments, tree_phi_sum, moment_order_for, initial_node_capacity, pack_sources

def ev():
    return torch.cuda.Event(enable_timing=True)

def run(w, reps=3):
    dev = torch.device("cuda")
    t0 = time.time()
    system = dt.from_sorted(w.xs, w.qs)
    kernel = dt.DiscKernel(w.r_d)
    cfg = dt.EvalConfig(p=w.p, leaf_capacity=w.leaf_capacity, adaptive=w.adaptive, tolerance=w.tolerance)
    tree = dt.build(system, kernel, cfg)
    ys = torch.from_numpy(w.targets).to(dev)
    out = torch.zeros_like(ys)
    print(f"{w.name}: N={w.n} T={len(w.targets)} nodes={len(tree)} depth={tree.depth} leaves={tree.leaf_count} setup={time.time()-t0:.2f}s", flush=True)
    n = w.n
    bufs = TreeBuffers(n, initial_node_capacity(n, w.leaf_capacity), dev)
    order = moment_order_for(cfg)
    mom = torch.empty((bufs.capacity, order + 1), dtype=torch.float64, device=dev)
    for r in range(reps):
        e = [ev() for _ in range(6)]
        e[0].record()
        pre = dt.charges.prefix_sum(system.qs)
        e[1].record()
        bufs.launch(system.xs, w.leaf_capacity)
        e[2].record()
        launch_moments(bufs, system.xs, system.qs, order, mom)
        e[3].record()
        sg = dt.charges._sign_terms(system, ys)
        e[4].record()
        tree_phi_sum(tree, kernel, cfg, ys, out, accumulate=False)
        e[5].record()
        torch.cuda.synchronize()
        ts = [e[i].elapsed_time(e[i+1]) for i in range(5)]
        print(f"  rep{r}: scan {ts[0]:.3f} build {ts[1]:.3f} moments {ts[2]:.3f} sign {ts[3]:.3f} eval {ts[4]:.3f} ms  -> {len(w.targets)/sum(ts)*1e3:.3e} targets/s", flush=True)
    # check build from bufs equals tree
    nn = int(bufs.meta[0])
    assert nn == len(tree)
    assert torch.equal(bufs.left[:nn], tree.left)
    # direct timing (subset of targets)
    # interaction statistics -> algorithmic flops
    T = len(w.targets)
    bs = {k: torch.zeros(T, dtype=torch.int64, device=dev) for k in ("hash","near_pairs","n_far","sum_p","n_p0","n_exact")}
    st = _lib.EvalStats(*[bs[k].data_ptr() for k in ("hash","near_pairs","n_far","sum_p","n_p0","n_exact")])
    tree_phi_sum(tree, kernel, cfg, ys, out, accumulate=False, stats=st)
    torch.cuda.synchronize()
    near = bs["near_pairs"].sum().item(); nfar = bs["n_far"].sum().item(); sump = bs["sum_p"].sum().item(); np0 = bs["n_p0"].sum().item(); nex = bs["n_exact"].sum().item()
    W = 14*near + 20*(nfar-np0) + 11*sump + 14*np0
    print(f"  stats: near/t {near/T:.1f} far/t {nfar/T:.2f} mean p {sump/max(nfar,1):.2f} exact-tier frac {nex/max(nfar,1):.2e} W/t {W/T:.0f} flop; eval {W/ts[4]*1e-9:.2f} TFLOP/s(alg)", flush=True)
    if w.name in ("cfg1",):
        T = 1 << 20
        o2 = torch.zeros(T, dtype=torch.float64, device=dev)
        for mode in (0, 1):
            a, b = ev(), ev()
            a.record()
            dt.direct.phi_sum_direct(system.xs, system.qs, ys[:T], w.r_d**2, o2, mode, False)
            b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            print(f"  direct mode{mode}: {T}x{n} pairs in {ms:.3f} ms = {T*n/ms*1e3:.3e} pairs/s = {T*n*14/ms*1e-9:.2f} TFLOP/s(alg)", flush=True)

which = sys.argv[1:] or ["cfg0", "cfg1", "cfg2"]
for name in which:
    run(getattr(W, name)())
