// (b) Tree construction: level-synchronous, breadth-first, bit-exact.
//
// Reference: tree.py:156-222 (build, structure part).  The reference walks
// the frontier in Python, one np.searchsorted per node.  Here one cooperative
// persistent kernel processes a level per step:
//   phase A  every frontier node decides leaf/split (count <= leaf_capacity or
//            level >= max_depth), finds split = lower_bound(xs[start:end], mid)
//            and counts its non-empty children; block-local exclusive scan.
//   phase B  block offsets (fixed-order sum of the block totals) give every
//            child its breadth-first index f1 + offset; children are written
//            and the parent's left/right slots are set with the reference's
//            rule "left iff child_hi == mid" (tree.py:205-208).
// BFS numbering equals level offset + spatial rank within the level, because
// the reference appends left-then-right children of an in-order frontier.
// Levels with few nodes run inside block 0 alone (no grid barrier).
// mid/center/half use explicit round-to-nearest intrinsics so that nvcc can
// never contract them: 0.5*(lo+hi) and 0.5*(hi-lo) exactly as numpy does.
#include <cooperative_groups.h>

#include "dt_common.cuh"
#include "dt_p2m.cuh"

namespace cg = cooperative_groups;

namespace {

#ifndef DT_BUILD_THREADS
#define DT_BUILD_THREADS 512
#endif
constexpr int BUILD_THREADS = DT_BUILD_THREADS;
#ifndef DT_BUILD_SMALL
#define DT_BUILD_SMALL (2 * BUILD_THREADS)
#endif
constexpr int SMALL_LEVEL = DT_BUILD_SMALL;
#ifndef DT_BUILD_STAGE
#define DT_BUILD_STAGE 1  // block-0 runs write staged 32-byte records (expand_stage)
#endif
#ifndef DT_BUILD_FLAGWAIT
#define DT_BUILD_FLAGWAIT 1
#endif  // nodes handled by block 0 alone

struct BuildArgs {
    const double *xs;
    int64_t n;
    int64_t leaf_capacity;
    int64_t max_depth;
    int64_t capacity;
    double *lo, *hi, *center, *half;
    int64_t *level, *start, *end, *left, *right;
    dt_node *packed;
    int64_t *meta;
    int32_t *scratch_off;    // [capacity] local exclusive offset within the block chunk
    int32_t *scratch_split;  // [capacity] split index found in phase A
    int64_t *block_total;    // [gridDim]
    // [2^DYADIC_LEVELS + 1] the dyadic points of the root interval in
    // position order, point j = (value, lower_bound in xs): the bounds of node
    // (L, k) are points k 2^(DYADIC_LEVELS - L) and (k + 1) 2^(DYADIC_LEVELS - L),
    // its midpoint (2k + 1) 2^(DYADIC_LEVELS - L - 1)
    double2 *dy_point;
    int k_top;               // levels 0..k_top built in one pass (0: level by level)
    unsigned *irregular;     // set if some top dyadic interval has mid not strictly inside
    // optional (dt_build_tree_p2m): while block 0 runs a sparse level run,
    // the other blocks form the leaves of the finished levels (P2M)
    int p2m_kmax;                    // 0: off, else 8/16/24/32 (order + 1 rounded up)
    P2mArgs p2m;
    unsigned long long *p2m_ctr;     // next 32-node chunk to form (zeroed per launch)
    // the nodes of level k_top that split, in BFS order, written by the
    // one-pass top (count, or -1 when the top was not built in one pass)
    int64_t *deep_count;
    struct Front *deep_list;
    double *dy_samples;      // every stride-th source (dyadic_splits)
};

// A frontier node of a block-0 run: kept in shared memory from one level to
// the next, so a level reads no node fields back from global memory.
struct Front {
    double lo, hi;
    int64_t node;
    int32_t s, e;
};

// A node created by a block-0 run, staged in the workspace (32 bytes instead
// of the 104 bytes of node arrays and packed record): one SM's store
// bandwidth bounds a run level, so block 0 writes only these, and after the
// run every block expands them into the node arrays (expand_stage).
struct StageRec {
    double lo, hi;
    int32_t s, e, l, r;  // source range, child links (-1: none)
};
struct Stage {
    StageRec *rec;
    int64_t base, cap;  // rec[i] is node base + i, for i < cap
};


// One warp forms leaves of 32-node chunks below `upto` (final nodes: the
// levels before block 0's current run), claimed with one atomicAdd each,
// until the chunks run out or block 0 publishes `phase` on `flag`.  Claims
// are contiguous from 0, so every chunk below min(counter, limit) was handed
// out and is formed before the kernel ends.  (A CAS-bounded claim loop,
// tried first, let 2352 warps hammer one L2 line and slowed block 0's own
// traffic by ~1 ms.)
template <int KMAX>
__device__ void build_p2m_until(const BuildArgs &a, unsigned long long limit,
                                unsigned long long phase, const unsigned long long *flag)
{
    constexpr int G = DT_P2M_G;
    const int lane = dt_lane(), sub = lane & (G - 1), grp = lane / G;
    while (true) {
        long long c = -1;
        if (lane == 0) {
            unsigned long long v;
            asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
            if (v < phase) {
                const unsigned long long got = atomicAdd(a.p2m_ctr, 1ull);
                c = got < limit ? (long long)got : -1;
            }
        }
        c = __shfl_sync(DT_FULL, c, 0);
        if (c < 0)
            return;
        const int64_t c0 = (int64_t)c * 32, mine = c0 + lane;
        // the build's own leaf rule (final once the node is written; its
        // child links may still be in flight for the first level of the run)
        const bool leaf = __ldcg(a.end + mine) - __ldcg(a.start + mine) <= a.leaf_capacity ||
                          __ldcg(a.level + mine) >= a.max_depth;
        unsigned leaves = __ballot_sync(DT_FULL, leaf);
        while (leaves) {
            unsigned m = leaves;
            for (int i = 0; i < grp && m; ++i)
                m &= m - 1;
            const bool active = m != 0;
            const int64_t node = c0 + (active ? __ffs(m) - 1 : 0);
            for (int i = 0; i < 32 / G && leaves; ++i)
                leaves &= leaves - 1;
            p2m_split_leaf<G, KMAX, true>(a.p2m, node, active, sub);
        }
    }
}

// Splits of the top dyadic levels, all at once.  The bisection intervals do
// not depend on the data (only which of them become nodes does), and for a
// node with source range [s, e) and midpoint mid,
//     lower_bound(xs[s:e], mid) = clamp(lower_bound(xs[0:n], mid), s, e)
// because xs is sorted.  So the lower_bounds of the 2^(K+1) - 1 midpoints of
// levels 0..K are found by independent searches in one parallel phase
// instead of K + 1 dependent rounds of DRAM-latency binary searches.
#ifndef DT_DYADIC_LEVELS
#define DT_DYADIC_LEVELS 18  // with the one-pass top: 16: 0.254 ms, 18: 0.248, 20: 0.384 (configs[2])
#endif
constexpr int DYADIC_LEVELS = DT_DYADIC_LEVELS;  // levels 0..DYADIC_LEVELS-1
constexpr int DYADIC = (1 << DYADIC_LEVELS) - 1;

// point j of the dyadic table: value and lower bound
__device__ __forceinline__ double2 dy_load(const BuildArgs &a, int64_t j)
{
    return __ldcg(a.dy_point + j);
}
__device__ __forceinline__ int64_t dy_lb(double2 p) { return __double_as_longlong(p.y); }

__device__ __forceinline__ double mid_of(double lo, double hi)
{
    return __dmul_rn(0.5, __dadd_rn(lo, hi));
}

__device__ void write_node(const BuildArgs &a, int64_t c, double lo, double hi, int64_t lev,
                           int64_t s, int64_t e, int64_t l_slot = -1, int64_t r_slot = -1)
{
    double ctr = __dmul_rn(0.5, __dadd_rn(lo, hi));
    double hw = __dmul_rn(0.5, __dsub_rn(hi, lo));
    a.lo[c] = lo;
    a.hi[c] = hi;
    a.center[c] = ctr;
    a.half[c] = hw;
    a.level[c] = lev;
    a.start[c] = s;
    a.end[c] = e;
    a.left[c] = l_slot;
    a.right[c] = r_slot;
    if (a.packed) {
        dt_node nd;
        nd.center = ctr;
        nd.half = hw;
        dt_node_children(nd, l_slot, r_slot);
        nd.start = (int32_t)s;
        nd.end = (int32_t)e;
        a.packed[c] = nd;
    }
}

// Node fields written earlier in this launch by other blocks are read with
// ld.global.cg (L2, never a stale L1 line).
__device__ __forceinline__ int64_t ld_cg(const int64_t *p) { return __ldcg(p); }
__device__ __forceinline__ double ld_cg(const double *p) { return __ldcg(p); }

// Root interval (tree.py:173-175): [x0 - pad, x_last + pad].
__device__ __forceinline__ void root_interval(const BuildArgs &a, double *lo, double *hi)
{
    const double x0 = a.xs[0], xl = a.xs[a.n - 1];
    const double m = fmax(1.0, fmax(fabs(x0), fabs(xl)));
    const double pad = __dmul_rn(1e-12, m);
    *lo = __dsub_rn(x0, pad);
    *hi = __dadd_rn(xl, pad);
}

// Phase 0: the dyadic point table (dy_point) for the midpoint of every
// dyadic interval idx of levels < DYADIC_LEVELS (level L = floor(log2(idx + 1)),
// position k = idx + 1 - 2^L), following the same midpoint arithmetic as the build.
// The lower_bounds are found in two steps: every stride-th source is copied
// to a sample array (<= 2^18 values, L2-resident), a grid barrier, then each
// midpoint is bisected over the samples and finished inside one stride of xs
// (the same index as one search over xs[0:n]: lower_bound is unique).  The
// searches then touch one or two DRAM lines each instead of ~12.
constexpr int64_t DY_SAMPLES = (int64_t)1 << 18;

#ifdef DT_BUILD_TRACE
#define DY_STAMP(slot)                                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                               \
        unsigned long long t_;                                                               \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
        a.block_total[2048 + (slot)] = (int64_t)t_;                                          \
    }
#else
#define DY_STAMP(slot)
#endif

__device__ __forceinline__ void dyadic_samples(const BuildArgs &a, int tid, int nth)
{
    const int64_t stride = (a.n + DY_SAMPLES - 1) / DY_SAMPLES;
    const int64_t ns = (a.n + stride - 1) / stride;
    for (int64_t i = tid; i < ns; i += nth)
        a.dy_samples[i] = __ldcs(a.xs + i * stride);
}

__device__ __forceinline__ void dyadic_search(const BuildArgs &a, int tid, int nth)
{
    const int64_t stride = (a.n + DY_SAMPLES - 1) / DY_SAMPLES;
    const int64_t ns = (a.n + stride - 1) / stride;
    double lo0, hi0;
    root_interval(a, &lo0, &hi0);
    const double *smp = a.dy_samples;
    for (int idx = tid; idx < DYADIC; idx += nth) {
        const int L = 31 - __clz(idx + 1);
        const int k = idx + 1 - (1 << L);
        double lo = lo0, hi = hi0;
        for (int b = L - 1; b >= 0; --b) {
            const double m = mid_of(lo, hi);
            if ((k >> b) & 1)
                lo = m;
            else
                hi = m;
        }
        const double mid = mid_of(lo, hi);
        const int64_t j = (int64_t)(2 * k + 1) << (DYADIC_LEVELS - L - 1);
        if (!(lo < mid && mid < hi))  // degenerate interval: no one-pass top
            atomicOr(a.irregular, 1u);
        // first sample >= mid
        int64_t l = 0, h = ns;
        while (l < h) {
            const int64_t m = (l + h) >> 1;
            if (smp[m] < mid)
                l = m + 1;
            else
                h = m;
        }
        // the answer lies in [s0, s1]: xs[s0 - 1] < mid <= xs[s1] (or s1 = n)
        int64_t s0 = l == 0 ? 0 : (l - 1) * stride + 1;
        int64_t s1 = l == ns ? a.n : l * stride;
        if (l > 0 && l < ns && s1 - s0 > 1) {
            // probe where the two bracketing samples put mid (on a locally
            // smooth mesh usually next to the answer), then its neighbour;
            // every outcome keeps the exact bracket
            const double xa = smp[l - 1], xb = smp[l];
            const double f = (mid - xa) / (xb - xa);
            int64_t g = s0 + (int64_t)(f * (double)(s1 - s0));
            g = g < s0 ? s0 : g > s1 - 1 ? s1 - 1 : g;
            if (__ldg(a.xs + g) < mid)
                s0 = g + 1;
            else
                s1 = g;
            if (s0 < s1) {
                const int64_t g2 = s0 == g + 1 ? s0 : s1 - 1;
                if (__ldg(a.xs + g2) < mid)
                    s0 = g2 + 1;
                else
                    s1 = g2;
            }
        }
        a.dy_point[j] = make_double2(mid, __longlong_as_double(dt_lower_bound(a.xs, s0, s1, mid)));
    }
    if (tid == 0) {
        a.dy_point[0] = make_double2(lo0, __longlong_as_double(0));
        a.dy_point[(int64_t)1 << DYADIC_LEVELS] = make_double2(hi0, __longlong_as_double(a.n));
    }
}

// In the cooperative build (16 warps per SM there) or, by default, as two
// small kernels ahead of it at full occupancy: the searches are latency
// chains (~20 dependent L2 probes each), so they want all the warps an SM
// can hold rather than the build's 128-register blocks.
#ifndef DT_BUILD_DYADIC_KERNELS
#define DT_BUILD_DYADIC_KERNELS 1
#endif
__device__ void dyadic_splits(const BuildArgs &a, cg::grid_group &grid)
{
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nth = gridDim.x * blockDim.x;
    dyadic_samples(a, tid, nth);
    DY_STAMP(73)
    grid.sync();
    DY_STAMP(74)
    dyadic_search(a, tid, nth);
    DY_STAMP(75)
}

constexpr int DY_THREADS = 256;
__global__ void __launch_bounds__(DY_THREADS) dyadic_samples_kernel(BuildArgs a)
{
    dyadic_samples(a, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}
__global__ void __launch_bounds__(DY_THREADS) dyadic_search_kernel(BuildArgs a)
{
    dyadic_search(a, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// Number of children of frontier node `node` (0 if it is a leaf) and split.
// Shared-memory samples of xs[r0, r1) (every stride-th source) for the
// block-0 runs of small levels: a split search bisects the samples first and
// then only a window of `stride` sources in global memory, so a deep level
// costs one or two dependent global accesses per node instead of
// log2(e - s).  The result is the plain lower_bound's: samples[j - 1] < v <=
// samples[j] bound the global lower bound to the window, and the split is
// its clamp to [s, e) (xs is sorted).
#ifndef DT_BUILD_WINCOUNT
#define DT_BUILD_WINCOUNT 0
#endif
#ifndef DT_BUILD_SAMPLES
#define DT_BUILD_SAMPLES 12288
#endif
constexpr int BUILD_SAMPLES = DT_BUILD_SAMPLES;  // dynamic shared memory, 8 bytes each
struct SplitSamples {
    const double *v;  // shared memory, count entries
    int64_t r0, r1, stride;
    int count;
};

__device__ __forceinline__ int64_t sampled_lower_bound(const BuildArgs &a, const SplitSamples &sm,
                                                       int64_t s, int64_t e, double v)
{
    int lo = 0, hi = sm.count;  // first sample >= v
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (sm.v[m] < v)
            lo = m + 1;
        else
            hi = m;
    }
    const int64_t wlo = lo == 0 ? sm.r0 : sm.r0 + (int64_t)(lo - 1) * sm.stride + 1;
    const int64_t whi = lo == sm.count ? sm.r1 : sm.r0 + (int64_t)lo * sm.stride;
#if DT_BUILD_WINCOUNT
    int64_t g;
    if (whi - wlo <= 32) {
        // short window: independent loads and a count (one memory round
        // trip instead of a chain of dependent probes); xs is sorted, so the
        // number of values below v is the lower bound's offset
        g = wlo;
#pragma unroll 4
        for (int64_t j = wlo; j < whi; ++j)
            g += __ldg(a.xs + j) < v ? 1 : 0;
    } else {
        g = dt_lower_bound(a.xs, wlo, whi, v);
    }
#else
    int64_t w0 = wlo, w1 = whi;
    if (lo > 0 && lo < sm.count && w1 - w0 > 1) {
        // probe where the bracketing samples put v (a locally smooth mesh
        // puts the answer next to it), then the neighbour; every outcome
        // keeps the exact bracket [w0, w1]
        const double xa = sm.v[lo - 1], xb = sm.v[lo];
        const double f = (v - xa) / (xb - xa);
        int64_t g = w0 + (int64_t)(f * (double)(w1 - w0));
        g = g < w0 ? w0 : g > w1 - 1 ? w1 - 1 : g;
        if (__ldg(a.xs + g) < v)
            w0 = g + 1;
        else
            w1 = g;
        if (w0 < w1) {
            const int64_t g2 = w0 == g + 1 ? w0 : w1 - 1;
            if (__ldg(a.xs + g2) < v)
                w0 = g2 + 1;
            else
                w1 = g2;
        }
    }
    const int64_t g = dt_lower_bound(a.xs, w0, w1, v);
#endif
    return g < s ? s : (g > e ? e : g);
}

// split = lower_bound(xs[s:e], mid) of a splitting node [lo, hi) of level lev
__device__ __forceinline__ int64_t split_of(const BuildArgs &a, int64_t lev, double lo, double hi,
                                            int64_t s, int64_t e, const SplitSamples *sm)
{
    const double mid = mid_of(lo, hi);
    int64_t split = -1;
    if (lev < DYADIC_LEVELS) {
        // dyadic position of the node from its lower bound; used only if the
        // recorded midpoint is exactly this node's midpoint
        double lo0 = ld_cg(a.lo + 0), hi0 = ld_cg(a.hi + 0);
        const double pos = (lo - lo0) / (hi0 - lo0) * (double)(1 << lev);
        const int k = (int)rint(pos);
        if (k >= 0 && k < (1 << lev)) {
            const double2 pt = dy_load(a, (int64_t)(2 * k + 1) << (DYADIC_LEVELS - lev - 1));
            if (pt.x == mid) {
                const int64_t g = dy_lb(pt);
                split = g < s ? s : (g > e ? e : g);
            }
        }
    }
    if (split < 0)
        split = sm && s >= sm->r0 && e <= sm->r1 ? sampled_lower_bound(a, *sm, s, e, mid)
                                                  : dt_lower_bound(a.xs, s, e, mid);
    return split;
}

__device__ __forceinline__ int node_children(const BuildArgs &a, int64_t node, int64_t lev,
                                             int64_t *split_out,
                                             const SplitSamples *sm = nullptr)
{
    int64_t s = ld_cg(a.start + node), e = ld_cg(a.end + node);
    if (e - s <= a.leaf_capacity || lev >= a.max_depth)
        return 0;
    const double lo = ld_cg(a.lo + node), hi = ld_cg(a.hi + node);
    const int64_t split = split_of(a, lev, lo, hi, s, e, sm);
    *split_out = split;
    return (split > s) + (e > split);
}

__device__ void emit_children(const BuildArgs &a, int64_t node, int64_t lev, int64_t first_child,
                              int64_t split)
{
    int64_t s = ld_cg(a.start + node), e = ld_cg(a.end + node);
    double lo = ld_cg(a.lo + node), hi = ld_cg(a.hi + node);
    double mid = mid_of(lo, hi);
    int64_t c = first_child;
    int64_t l_slot = -1, r_slot = -1;
    if (split > s) {  // (lo, mid): child_hi == mid -> left
        write_node(a, c, lo, mid, lev + 1, s, split);
        l_slot = c;
        ++c;
    }
    if (e > split) {  // (mid, hi): left iff hi == mid (tree.py:205-208)
        write_node(a, c, mid, hi, lev + 1, split, e);
        if (hi == mid)
            l_slot = c;
        else
            r_slot = c;
    }
    a.left[node] = l_slot;
    a.right[node] = r_slot;
    if (a.packed) {
        dt_node_children(a.packed[node], l_slot, r_slot);
    }
}

// Block-wide exclusive scan of ints; returns the block total.
__device__ int block_excl_scan(int v, int *excl, int *warp_sums)
{
    const int lane = dt_lane(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(DT_FULL, x, o);
        if (lane >= o)
            x += t;
    }
    if (lane == 31)
        warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(DT_FULL, w, o);
            if (lane >= o)
                w += t;
        }
        if (lane < nw)
            warp_sums[lane] = w;
    }
    __syncthreads();
    int base = warp > 0 ? warp_sums[warp - 1] : 0;
    int total = warp_sums[nw - 1];
    __syncthreads();
    *excl = base + x - v;
    return total;
}

__device__ __forceinline__ void stage_node(const Stage &st, int64_t c, double lo, double hi,
                                           int64_t s, int64_t e)
{
    StageRec *r = st.rec + (c - st.base);
    *reinterpret_cast<double2 *>(r) = make_double2(lo, hi);
    *reinterpret_cast<int4 *>(&r->s) = make_int4((int)s, (int)e, -1, -1);
}

// All blocks: the staged nodes [st.base, min(n_nodes, st.base + st.cap))
// into the node arrays; node levels from the level offsets in meta (levels
// lev0 + 1 .. of the run).
__device__ void expand_stage(const BuildArgs &a, const Stage &st, int64_t n_nodes, int64_t lev0)
{
    const int64_t n = min(n_nodes - st.base, st.cap);
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth) {
        const int64_t node = st.base + i;
        int64_t l = lev0 + 1;
        while (node >= ((volatile int64_t *)a.meta)[DT_META_LEVEL0 + l + 1])
            ++l;
        const double2 lh = __ldcg(reinterpret_cast<const double2 *>(st.rec + i));
        const int4 se = __ldcg(reinterpret_cast<const int4 *>(&st.rec[i].s));
        write_node(a, node, lh.x, lh.y, l, se.x, se.y, se.z, se.w);
    }
}

// One level of a block-0 run: the frontier `cur` (F nodes of level lev) is
// in shared memory; the children are written to the node arrays at BFS
// index g1 + rank and, while they fit, to the next frontier `nxt`.
// Returns the number of children written (or -1 on capacity overflow).
__device__ int64_t level_in_block(const BuildArgs &a, const Front *cur, int F, int64_t g1,
                                  int64_t lev, int *warp_sums, int64_t *leaves,
                                  const SplitSamples *sm, Front *nxt, const Stage &st)
{
    int64_t next = g1;
    int64_t leaf_acc = 0;
#ifdef DT_BUILD_TRACE
#define FINE(k) if (lev == 20 && threadIdx.x == 0) { a.block_total[2048 + 100 + (k)] = (int64_t)clock64(); }
#else
#define FINE(k)
#endif
    FINE(0)
    for (int t0 = 0; t0 < F; t0 += blockDim.x) {
        const int i = t0 + threadIdx.x;
        int nc = 0;
        int64_t split = 0;
        Front f{};
        if (i < F) {
            f = cur[i];
            if (f.e - f.s > a.leaf_capacity && lev < a.max_depth) {
                split = split_of(a, lev, f.lo, f.hi, f.s, f.e, sm);
                nc = (split > f.s) + (f.e > split);
            } else {
                ++leaf_acc;
            }
        }
        __syncthreads();
        FINE(1)
        int excl;
        const int tot = block_excl_scan(nc, &excl, warp_sums);
        FINE(2)
        if (next + tot > a.capacity)
            return -1;
        if (nc) {
            const double mid = mid_of(f.lo, f.hi);
            int64_t c = next + excl;
            int64_t l_slot = -1, r_slot = -1;
            if (split > f.s) {  // (lo, mid): child_hi == mid -> left
                if (c - st.base < st.cap)
                    stage_node(st, c, f.lo, mid, f.s, split);
                else
                    write_node(a, c, f.lo, mid, lev + 1, f.s, split);
                if (c - g1 < SMALL_LEVEL)
                    nxt[c - g1] = Front{f.lo, mid, c, f.s, (int32_t)split};
                l_slot = c;
                ++c;
            }
            if (f.e > split) {  // (mid, hi): left iff hi == mid (tree.py:205-208)
                if (c - st.base < st.cap)
                    stage_node(st, c, mid, f.hi, split, f.e);
                else
                    write_node(a, c, mid, f.hi, lev + 1, split, f.e);
                if (c - g1 < SMALL_LEVEL)
                    nxt[c - g1] = Front{mid, f.hi, c, (int32_t)split, f.e};
                if (f.hi == mid)
                    l_slot = c;
                else
                    r_slot = c;
            }
            if (f.node >= st.base && f.node - st.base < st.cap) {
                *reinterpret_cast<int2 *>(&st.rec[f.node - st.base].l) =
                    make_int2((int)l_slot, (int)r_slot);
            } else {
                a.left[f.node] = l_slot;
                a.right[f.node] = r_slot;
                if (a.packed)
                    dt_node_children(a.packed[f.node], l_slot, r_slot);
            }
        }
        next += tot;
    }
    __syncthreads();
    FINE(3)
    *leaves += leaf_acc;
    return next - g1;
}

#ifdef DT_BUILD_TRACE
#define BUILD_STAMP(slot)                                                                    \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                               \
        unsigned long long t_;                                                               \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
        a.block_total[2048 + (slot)] = (int64_t)t_;                                          \
    }
#else
#define BUILD_STAMP(slot)
#endif

// ---- the top levels in one pass
//
// Every node of level L <= k_top is a dyadic interval [k/2^L, (k+1)/2^L) of
// the root (its bounds are midpoints of its ancestors, recorded by
// dyadic_splits), and its source range is [lower_bound(lo), lower_bound(hi))
// of the whole array (the clamp in node_children never binds, since the
// ranges nest).  So which slots become nodes is known in closed form:
//     slot (L, k) is a node  iff  count(L, k) > 0 and (L = 0 or the parent
//     slot splits: count(L-1, k/2) > leaf_capacity and L-1 < max_depth),
// (counts shrink down the path, so the parent's test covers every ancestor)
// and its breadth-first index is the number of node slots before it in
// level-major order.  One exclusive scan over the 2^(k_top+1) - 1 slots
// replaces 2 (k_top + 1) grid barriers of the level-by-level build.
// Requires every top interval to be regular (lo < mid < hi, else the
// reference's one-child cases apply and the build goes level by level).

#ifndef DT_TOP_R1
#define DT_TOP_R1 4
#endif
#ifndef DT_TOP_R2
#define DT_TOP_R2 2
#endif
constexpr int TOP_R1 = DT_TOP_R1, TOP_R2 = DT_TOP_R2;  // rows per group in the top's passes

struct TopSlot {
    int L;
    int64_t k;
    double lo, hi;
    int64_t s, e;
    bool node, splits;
};

// Slot f of the top (level L, position k): bounds, source range, and whether
// it is a node / splits.  Three point loads: its two bounds and the parent's
// other bound (the parent shares one bound with the slot).
__device__ __forceinline__ TopSlot top_slot(const BuildArgs &a, int64_t f)
{
    TopSlot t;
    t.L = 63 - __clzll(f + 1);
    t.k = f + 1 - ((int64_t)1 << t.L);
    const int sh = DYADIC_LEVELS - t.L;
    const double2 p0 = dy_load(a, t.k << sh), p1 = dy_load(a, (t.k + 1) << sh);
    const int64_t kx = (t.k & 1) ? t.k - 1 : t.k + 2;  // the parent's other bound
    const int64_t px = t.L > 0 ? dy_lb(dy_load(a, kx << sh)) : 0;
    t.lo = p0.x;
    t.hi = p1.x;
    t.s = dy_lb(p0);
    t.e = dy_lb(p1);
    bool parent_splits = true;
    if (t.L > 0) {
        const int64_t ps = (t.k & 1) ? px : t.s, pe = (t.k & 1) ? t.e : px;
        parent_splits = pe - ps > a.leaf_capacity && t.L - 1 < a.max_depth;
    }
    t.node = t.e > t.s && parent_splits;
    t.splits = t.node && t.e - t.s > a.leaf_capacity && t.L < a.max_depth;
    return t;
}

// Returns the first level for the level-by-level loop (k_top, or 0 if the
// top cannot be built in one pass).  Grid-uniform.
__device__ int64_t build_top(const BuildArgs &a, cg::grid_group &grid, int *warp_sums,
                             int64_t *bases_s, int64_t *bases2_s)
{
    const int K = a.k_top;
    if (K <= 0 || *(volatile unsigned *)a.irregular)
        return 0;
    const int G = gridDim.x;
    const int64_t S = ((int64_t)2 << K) - 1;  // slots of levels 0..K
    const int64_t chunk = (S + G - 1) / G;
    const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = min(S, b0 + chunk);
    // the level-K nodes that split are also listed (in slot order, which is
    // BFS order) with their intervals, so the level-by-level build continues
    // from them alone instead of testing every level-K node; the two counts
    // share one scan (16 bits each: a block chunk has < 2^15 slots)
    const bool listing = chunk < (1 << 15) && G <= 1024;
    // pass 1: node flags, block-local exclusive offsets, leaves above level K
    // (TOP_R1 rows of blockDim.x slots at a time: their point loads are all
    // in flight together, then one block scan per row)
    int64_t run = 0, run2 = 0, leaves = 0;
    for (int64_t g0 = b0; g0 < b1; g0 += (int64_t)TOP_R1 * blockDim.x) {
        int flag[TOP_R1];
#pragma unroll
        for (int r = 0; r < TOP_R1; ++r) {
            const int64_t f = g0 + (int64_t)r * blockDim.x + threadIdx.x;
            flag[r] = 0;
            if (f < b1) {
                const TopSlot t = top_slot(a, f);
                flag[r] = t.node | ((listing && t.splits && t.L == K) ? 1 << 16 : 0);
                leaves += t.node && !t.splits && t.L < K;
            }
        }
#pragma unroll
        for (int r = 0; r < TOP_R1; ++r) {
            const int64_t t0 = g0 + (int64_t)r * blockDim.x;
            if (t0 >= b1)
                break;  // block-uniform
            const int64_t f = t0 + threadIdx.x;
            int excl;
            const int tot = block_excl_scan(flag[r], &excl, warp_sums);
            if (f < b1) {
                a.scratch_off[f] = (int32_t)(run + (excl & 0xffff));
                a.scratch_split[f] = (int32_t)(run2 + (excl >> 16));
            }
            run += tot & 0xffff;
            run2 += tot >> 16;
        }
    }
    if (threadIdx.x == 0) {
        a.block_total[blockIdx.x] = run;
        if (listing)
            a.block_total[1024 + blockIdx.x] = run2;
    }
    {
        int64_t lv = leaves;
        for (int o = 16; o > 0; o >>= 1)
            lv += __shfl_xor_sync(DT_FULL, lv, o);
        if (dt_lane() == 0 && lv)
            atomicAdd((unsigned long long *)&a.meta[DT_META_LEAVES], (unsigned long long)lv);
    }
    BUILD_STAMP(76)
    grid.sync();
    BUILD_STAMP(77)
    // every block's base: exclusive scans over the block totals (integer
    // sums, so any order gives the same bases)
    if (G <= (int)blockDim.x) {
        const int b = threadIdx.x;
        const int v1 = b < G ? (int)__ldcg(a.block_total + b) : 0;
        const int v2 = listing && b < G ? (int)__ldcg(a.block_total + 1024 + b) : 0;
        int e1, e2;
        const int t1 = block_excl_scan(v1, &e1, warp_sums);
        const int t2 = block_excl_scan(v2, &e2, warp_sums);
        if (b < G) {
            bases_s[b] = e1;
            bases2_s[b] = e2;
        }
        if (b == 0) {
            bases_s[G] = t1;
            bases2_s[G] = t2;
        }
    } else if (threadIdx.x == 0) {
        int64_t acc = 0, acc2 = 0;
        for (int b = 0; b < G; ++b) {
            bases_s[b] = acc;
            bases2_s[b] = acc2;
            acc += __ldcg(a.block_total + b);
            acc2 += listing ? __ldcg(a.block_total + 1024 + b) : 0;
        }
        bases_s[G] = acc;
        bases2_s[G] = acc2;
    }
    __syncthreads();
    BUILD_STAMP(78)
    const int64_t total = bases_s[G];
    if (total > a.capacity) {  // every block sees the same total
        if (blockIdx.x == 0 && threadIdx.x == 0)
            a.meta[DT_META_OVERFLOW] = 1;
        return -1;
    }
    const unsigned uchunk = (unsigned)chunk;  // S < 2^31: 32-bit divisions
    auto index_of = [&](int64_t f) -> int64_t {  // exclusive node count before slot f
        return f >= S ? total : bases_s[(unsigned)f / uchunk] + __ldcg(a.scratch_off + f);
    };
    // pass 2: write the nodes with their child links.  Every global load of
    // a slot is issued before any of them is used: one L2 round trip per slot
    // instead of a chain of three
    for (int64_t g0 = b0 + threadIdx.x; g0 < b1; g0 += (int64_t)TOP_R2 * blockDim.x) {
#pragma unroll
        for (int r = 0; r < TOP_R2; ++r) {
            const int64_t f = g0 + (int64_t)r * blockDim.x;
            if (f >= b1)
                break;
            const int64_t fl = 2 * f + 1;  // slot (L + 1, 2k)
            const int32_t off = __ldcg(a.scratch_off + f);
            const int32_t offl = fl < S ? __ldcg(a.scratch_off + fl) : 0;
            const int32_t offr = fl + 1 < S ? __ldcg(a.scratch_off + fl + 1) : 0;
            const int32_t off2 = listing ? __ldcg(a.scratch_split + f) : 0;
            const TopSlot t = top_slot(a, f);
            // this slot's own midpoint (levels < K only)
            const int64_t split =
                t.L < K ? dy_lb(dy_load(a, (2 * t.k + 1) << (DYADIC_LEVELS - t.L - 1))) : 0;
            if (!t.node)
                continue;
            const int64_t c = bases_s[blockIdx.x] + off;
            int64_t l_slot = -1, r_slot = -1;
            if (t.splits && t.L < K) {
                if (split > t.s)
                    l_slot = fl >= S ? total : bases_s[(unsigned)fl / uchunk] + offl;
                if (t.e > split)
                    r_slot = fl + 1 >= S ? total : bases_s[(unsigned)(fl + 1) / uchunk] + offr;
            }
#ifdef DT_TOP_NOWRITE
            if (c == -12345)
#endif
            write_node(a, c, t.lo, t.hi, t.L, t.s, t.e, l_slot, r_slot);
            if (listing && t.splits && t.L == K)
                a.deep_list[bases2_s[blockIdx.x] + off2] =
                    Front{t.lo, t.hi, c, (int32_t)t.s, (int32_t)t.e};
        }
    }
    if (blockIdx.x == 0 && threadIdx.x <= K + 1) {
        const int L = threadIdx.x;  // level offsets 0 .. K + 1
        a.meta[DT_META_LEVEL0 + L] = index_of(((int64_t)1 << L) - 1);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.deep_count = listing ? bases2_s[G] : -1;
        a.meta[DT_META_NODES] = total;
        int depth = 0;
        for (int L = 0; L <= K; ++L)
            if (index_of(((int64_t)2 << L) - 1) > index_of(((int64_t)1 << L) - 1))
                depth = L;
        a.meta[DT_META_DEPTH] = depth;
    }
    BUILD_STAMP(79)
    grid.sync();
    return K;
}

__global__ void __launch_bounds__(BUILD_THREADS) build_kernel(BuildArgs a)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ int warp_sums[BUILD_THREADS / 32];
    __shared__ int64_t sh_i64[4];
    __shared__ int64_t top_bases_s[BUILD_THREADS + 1];
    __shared__ int64_t top_bases2_s[BUILD_THREADS + 1];
    // BUILD_SAMPLES split samples, then two frontier buffers of SMALL_LEVEL
    extern __shared__ double samples_s[];
    Front *const front_s = reinterpret_cast<Front *>(samples_s + BUILD_SAMPLES);
    volatile int64_t *meta = a.meta;
    const int G = gridDim.x;

    if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int i = 0; i < DT_META_WORDS; ++i)
            a.meta[i] = 0;
        a.meta[DT_META_LEVEL0 + 0] = 0;
        a.meta[DT_META_LEVEL0 + 1] = 1;
        a.meta[DT_META_NODES] = 1;
        *a.deep_count = -1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // tree.py:173-175: pad = 1e-12 * max(1.0, |x0|, |x_last|)
        double lo0, hi0;
        root_interval(a, &lo0, &hi0);
        write_node(a, 0, lo0, hi0, 0, 0, a.n);
    }
#if DT_BUILD_FLAGWAIT
    // phase counter of the small-level runs (see below)
    unsigned long long *const small_flag =
        reinterpret_cast<unsigned long long *>(a.block_total + 4095);
    unsigned long long small_phase = 0;
    unsigned long long p2m_limit = 0;  // chunks of the first sparse run (0: none yet)
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *small_flag = 0;
#endif
    BUILD_STAMP(70)
    if (!DT_BUILD_DYADIC_KERNELS) {
        dyadic_splits(a, grid);
        grid.sync();
    }
    BUILD_STAMP(71)
    int64_t lev = build_top(a, grid, warp_sums, top_bases_s, top_bases2_s);
    const int64_t k_listed = lev;  // the level whose splitting nodes are listed
    BUILD_STAMP(72)
    if (lev < 0)
        return;  // capacity overflow (flagged in meta)
    while (lev <= a.max_depth) {
#ifdef DT_BUILD_TRACE
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.block_total[2048 + lev] = (int64_t)t;
        }
#endif
        int64_t f0 = meta[DT_META_LEVEL0 + lev];
        int64_t f1 = meta[DT_META_LEVEL0 + lev + 1];
        int64_t F = f1 - f0;
        if (F == 0 || meta[DT_META_OVERFLOW])
            break;
        // level k_top continues from the listed nodes that split
        const int64_t n_listed = lev == k_listed && k_listed > 0 ? *(volatile int64_t *)a.deep_count : -1;
        const bool listed = n_listed >= 0 && n_listed <= SMALL_LEVEL;
        if (F <= SMALL_LEVEL || listed) {
            // block 0 runs consecutive small levels with the frontier in
            // shared memory; the others wait (and form leaves, below).  The
            // run's nodes are staged in the scratch slots (free until the
            // next big level) and expanded by every block after the run.
            const int64_t lev0_of_run = lev;
            Stage st;
            st.rec = reinterpret_cast<StageRec *>(a.scratch_off);
            st.base = f1;
            st.cap = DT_BUILD_STAGE ? a.capacity * 2 * (int64_t)sizeof(int32_t) / (int64_t)sizeof(StageRec) : 0;
            if (blockIdx.x == 0) {
                int64_t leaves = 0;
                int64_t l = lev, g1 = f1;
                Front *cur = front_s, *nxt = front_s + SMALL_LEVEL;
                int Fl;
                if (listed) {
                    Fl = (int)n_listed;
                    for (int i = threadIdx.x; i < Fl; i += blockDim.x) {
                        const double2 lh = __ldcg(reinterpret_cast<const double2 *>(a.deep_list + i));
                        const double2 ns = __ldcg(reinterpret_cast<const double2 *>(a.deep_list + i) + 1);
                        cur[i] = Front{lh.x, lh.y, (int64_t)__double_as_longlong(ns.x),
                                       __double2loint(ns.y), __double2hiint(ns.y)};
                    }
                    if (threadIdx.x == 0)
                        leaves += F - Fl;  // the level's other nodes are leaves
                } else {
                    Fl = (int)F;
                    for (int i = threadIdx.x; i < Fl; i += blockDim.x) {
                        const int64_t node = f0 + i;
                        cur[i] = Front{ld_cg(a.lo + node), ld_cg(a.hi + node), node,
                                       (int32_t)ld_cg(a.start + node), (int32_t)ld_cg(a.end + node)};
                    }
                }
                __syncthreads();
                // the run's nodes all lie inside the first frontier's source
                // range: sample it once (below the dyadic levels only)
                SplitSamples sm{samples_s, 0, 0, 1, 0};
                if (lev >= DYADIC_LEVELS && Fl > 0) {
                    sm.r0 = cur[0].s;
                    sm.r1 = cur[Fl - 1].e;
                    const int64_t len = sm.r1 - sm.r0;
                    sm.stride = len > BUILD_SAMPLES ? (len + BUILD_SAMPLES - 1) / BUILD_SAMPLES : 1;
                    sm.count = (int)((len + sm.stride - 1) / sm.stride);
                    for (int j = threadIdx.x; j < sm.count; j += blockDim.x)
                        samples_s[j] = __ldg(a.xs + sm.r0 + (int64_t)j * sm.stride);
                    __syncthreads();
                }
                while (true) {
#ifdef DT_BUILD_TRACE
                    if (threadIdx.x == 0) {
                        unsigned long long t;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                        a.block_total[2048 + l] = (int64_t)t;
                    }
#endif
                    const int64_t made = level_in_block(a, cur, Fl, g1, l, warp_sums, &leaves,
                                                        lev >= DYADIC_LEVELS ? &sm : nullptr, nxt, st);
                    __syncthreads();
                    if (made < 0) {
                        if (threadIdx.x == 0)
                            a.meta[DT_META_OVERFLOW] = 1;
                        break;
                    }
                    // (the next level reads its nodes from the frontier in
                    // shared memory: no fence or second barrier per level)
                    if (threadIdx.x == 0) {
                        a.meta[DT_META_LEVEL0 + l + 2] = g1 + made;
                        a.meta[DT_META_NODES] = g1 + made;
                        if (made > 0)
                            a.meta[DT_META_DEPTH] = l + 1;
                    }
                    if (l == 20 && threadIdx.x == 0) { a.block_total[2048 + 104] = (int64_t)clock64(); }
                    ++l;
                    if (made == 0 || made > SMALL_LEVEL || l > a.max_depth)
                        break;
                    Fl = (int)made;
                    g1 += made;
                    Front *t = cur;
                    cur = nxt;
                    nxt = t;
                }
                // leaves counted per thread: reduce
                int64_t lv = leaves;
                for (int o = 16; o > 0; o >>= 1)
                    lv += __shfl_xor_sync(DT_FULL, lv, o);
                if (dt_lane() == 0 && lv)
                    atomicAdd((unsigned long long *)&a.meta[DT_META_LEAVES],
                              (unsigned long long)lv);
                if (threadIdx.x == 0)
                    a.meta[DT_META_CURLEVEL] = l;
                __threadfence();
            }
            // nodes below p2m_upto are final (the listed level's nodes too:
            // the P2M leaf test reads only their ranges and levels)
            const int64_t p2m_upto = listed ? f1 : f0;
            if (blockIdx.x == 0 && a.p2m_kmax && p2m_limit == 0 && p2m_upto >= 32)
                p2m_limit = (unsigned long long)(p2m_upto / 32);  // as the other blocks
#if DT_BUILD_FLAGWAIT
            // block 0 announces the end of its run with a release store; the
            // other blocks wait on it with back-off instead of polling a grid
            // barrier (which slows block 0's own L2 traffic)
            ++small_phase;
            if (blockIdx.x == 0) {
                __syncthreads();
                if (threadIdx.x == 0)
                    asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(small_flag), "l"(small_phase)
                                 : "memory");
            } else {
                if (a.p2m_kmax && p2m_limit == 0 && p2m_upto >= 32) {
                    // meanwhile (the first run with whole chunks before it
                    // only): form the leaves of the levels before this run
                    p2m_limit = (unsigned long long)(p2m_upto / 32);
                    switch (a.p2m_kmax) {
                    case 8: build_p2m_until<8>(a, p2m_limit, small_phase, small_flag); break;
                    case 16: build_p2m_until<16>(a, p2m_limit, small_phase, small_flag); break;
                    case 24: build_p2m_until<24>(a, p2m_limit, small_phase, small_flag); break;
                    default: build_p2m_until<32>(a, p2m_limit, small_phase, small_flag); break;
                    }
                }
                if (threadIdx.x == 0) {
                    unsigned long long v;
                    while (true) {
                        asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(small_flag)
                                     : "memory");
                        if (v >= small_phase)
                            break;
                        __nanosleep(256);
                    }
                }
                __syncthreads();
            }
#else
            grid.sync();
#endif
            lev = meta[DT_META_CURLEVEL];
            if (st.cap > 0) {
                expand_stage(a, st, meta[DT_META_NODES], lev0_of_run);
                // a following level reads the run's last nodes from the arrays
                if (lev <= a.max_depth && !meta[DT_META_OVERFLOW] &&
                    meta[DT_META_LEVEL0 + lev + 1] > meta[DT_META_LEVEL0 + lev])
                    grid.sync();
            }
            continue;
        }
        // ---- big level: all blocks, contiguous chunk per block
        const int64_t chunk = (F + G - 1) / G;
        const int64_t b0 = f0 + (int64_t)blockIdx.x * chunk;
        const int64_t b1 = min(f1, b0 + chunk);
        int64_t run = 0, leaves = 0;
        for (int64_t t0 = b0; t0 < b1; t0 += blockDim.x) {
            int64_t node = t0 + threadIdx.x;
            int64_t split = 0;
            int nc = node < b1 ? node_children(a, node, lev, &split) : 0;
            if (node < b1 && nc == 0)
                ++leaves;
            int excl;
            int tot = block_excl_scan(nc, &excl, warp_sums);
            if (node < b1) {
                a.scratch_off[node - f0] = (int32_t)(run + excl);
                a.scratch_split[node - f0] = (int32_t)split;
            }
            run += tot;
        }
        if (threadIdx.x == 0)
            a.block_total[blockIdx.x] = run;
        {
            int64_t lv = leaves;
            for (int o = 16; o > 0; o >>= 1)
                lv += __shfl_xor_sync(DT_FULL, lv, o);
            if (dt_lane() == 0 && lv)
                atomicAdd((unsigned long long *)&a.meta[DT_META_LEAVES], (unsigned long long)lv);
        }
        grid.sync();
        // block base and level total, fixed-order sums
        if (threadIdx.x < 32) {
            int64_t base = 0, total = 0;
            for (int b = threadIdx.x; b < G; b += 32) {
                int64_t v = ((volatile int64_t *)a.block_total)[b];
                total += v;
                if (b < (int)blockIdx.x)
                    base += v;
            }
            for (int o = 16; o > 0; o >>= 1) {
                base += __shfl_xor_sync(DT_FULL, base, o);
                total += __shfl_xor_sync(DT_FULL, total, o);
            }
            if (threadIdx.x == 0) {
                sh_i64[0] = base;
                sh_i64[1] = total;
            }
        }
        __syncthreads();
        const int64_t base = sh_i64[0], total = sh_i64[1];
        if (f1 + total > a.capacity) {
            if (blockIdx.x == 0 && threadIdx.x == 0)
                a.meta[DT_META_OVERFLOW] = 1;
            break;  // every block sees the same total
        }
        for (int64_t node = b0 + threadIdx.x; node < b1; node += blockDim.x) {
            int64_t s = ld_cg(a.start + node), e = ld_cg(a.end + node);
            if (e - s <= a.leaf_capacity || lev >= a.max_depth)
                continue;
            emit_children(a, node, lev, f1 + base + __ldcg(a.scratch_off + (node - f0)),
                          __ldcg(a.scratch_split + (node - f0)));
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.meta[DT_META_LEVEL0 + lev + 2] = f1 + total;
            a.meta[DT_META_NODES] = f1 + total;
            if (total > 0)
                a.meta[DT_META_DEPTH] = lev + 1;
        }
        grid.sync();
        ++lev;
    }
    // every chunk below min(claims, limit) is formed before the kernel ends
    if (a.p2m_kmax && blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long got = *(volatile unsigned long long *)a.p2m_ctr;
        a.meta[DT_META_P2M_UPTO] = (int64_t)(32 * (got < p2m_limit ? got : p2m_limit));
    }
}

}  // namespace

extern "C" size_t dt_build_workspace(int64_t n, int64_t node_capacity)
{
    (void)n;
    return (size_t)node_capacity * 2 * sizeof(int32_t) + 4096 * sizeof(int64_t) + 16 +
           (((size_t)1 << DYADIC_LEVELS) + 2) * sizeof(double2) + 32 + 64 +
           ((size_t)1 << DYADIC_LEVELS) * sizeof(Front) + (size_t)DY_SAMPLES * sizeof(double);
}

static int build_launch(const double *xs, int64_t n, int64_t leaf_capacity, int64_t max_depth,
                        int64_t node_capacity, double *lo, double *hi, double *center,
                        double *half, int64_t *level, int64_t *start, int64_t *end,
                        int64_t *left, int64_t *right, void *packed, int64_t *meta,
                        void *workspace, size_t workspace_bytes, void *stream,
                        const P2mArgs *p2m)
{
    DT_CHECK_ARG(n > 0, "cannot build a tree over an empty charge system");
    DT_CHECK_ARG(n < (int64_t)1 << 31, "n must be < 2^31");
    DT_CHECK_ARG(leaf_capacity >= 1, "leaf_capacity must be >= 1");
    DT_CHECK_ARG(max_depth >= 0 && max_depth <= DT_MAX_DEPTH, "max_depth must be in [0, 60]");
    DT_CHECK_ARG(node_capacity >= 1 && node_capacity < (int64_t)1 << 31,
                 "node_capacity must be in [1, 2^31)");
    DT_CHECK_ARG(xs && lo && hi && center && half && level && start && end && left && right &&
                     meta,
                 "null pointer");
    if (!workspace || workspace_bytes < dt_build_workspace(n, node_capacity))
        return dt_set_error(DT_ERR_WORKSPACE, "build workspace too small");

    BuildArgs a;
    a.xs = xs;
    a.n = n;
    a.leaf_capacity = leaf_capacity;
    a.max_depth = max_depth;
    a.capacity = node_capacity;
    a.lo = lo;
    a.hi = hi;
    a.center = center;
    a.half = half;
    a.level = level;
    a.start = start;
    a.end = end;
    a.left = left;
    a.right = right;
    a.packed = (dt_node *)packed;
    a.meta = meta;
    a.scratch_off = (int32_t *)workspace;
    a.scratch_split = a.scratch_off + node_capacity;
    a.block_total = (int64_t *)((char *)workspace + (size_t)node_capacity * 2 * sizeof(int32_t));
    // 8-byte align block_total
    a.block_total = (int64_t *)(((uintptr_t)a.block_total + 7) & ~(uintptr_t)7);
    a.dy_point = (double2 *)(((uintptr_t)(a.block_total + 4096) + 15) & ~(uintptr_t)15);
    a.irregular = (unsigned *)(a.dy_point + ((size_t)1 << DYADIC_LEVELS) + 1);
    // one-pass top: levels 0..k_top need 2^(k_top+1) - 1 scratch slots and
    // the dyadic midpoints of levels < k_top
    a.k_top = 0;
#ifndef DT_BUILD_TOP
#define DT_BUILD_TOP 1
#endif
    if (DT_BUILD_TOP)
        for (int K = DYADIC_LEVELS; K >= 1; --K)
            if (((int64_t)2 << K) - 1 <= node_capacity) {
                a.k_top = K;
                break;
            }
    a.p2m_ctr = (unsigned long long *)(a.irregular + 2);
    a.deep_count = (int64_t *)(a.p2m_ctr + 1);
    a.deep_list = (Front *)(((uintptr_t)(a.deep_count + 1) + 31) & ~(uintptr_t)31);
    a.dy_samples = (double *)(a.deep_list + ((size_t)1 << DYADIC_LEVELS));
    a.p2m_kmax = 0;
    if (p2m) {
        a.p2m = *p2m;
        const int64_t o1 = p2m->order + 1;
        a.p2m_kmax = o1 <= 8 ? 8 : o1 <= 16 ? 16 : o1 <= 24 ? 24 : 32;
    }
    // the irregular flag and the chunk counter
    DT_CUDA_TRY(cudaMemsetAsync(a.irregular, 0, 16, (cudaStream_t)stream));

    // the attribute and the occupancy are per device and fixed: queried once
    // (they sit in front of every launch otherwise)
    static int cached_dev = -1, per_sm = 0;
    int dev = 0;
    DT_CUDA_TRY(cudaGetDevice(&dev));
    const size_t smem = (size_t)BUILD_SAMPLES * sizeof(double) + 2 * SMALL_LEVEL * sizeof(Front);
    if (dev != cached_dev) {
        DT_CUDA_TRY(cudaFuncSetAttribute((const void *)build_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, build_kernel,
                                                                  BUILD_THREADS, smem));
        cached_dev = dev;
    }
    if (per_sm < 1)
        return dt_set_error(DT_ERR_CUDA, "build kernel cannot be resident");
#ifndef DT_BUILD_PER_SM
#define DT_BUILD_PER_SM 1  // one block per SM: cheaper grid barriers (0.34 -> 0.31 ms)
#endif
    int grid = dt_num_sms() * (per_sm > DT_BUILD_PER_SM ? DT_BUILD_PER_SM : per_sm);
    if (grid > 3000)
        grid = 3000;
    if (DT_BUILD_DYADIC_KERNELS) {
        const int dy_blocks = (int)((DY_SAMPLES + DY_THREADS - 1) / DY_THREADS);
        dyadic_samples_kernel<<<dy_blocks, DY_THREADS, 0, (cudaStream_t)stream>>>(a);
        dyadic_search_kernel<<<dy_blocks, DY_THREADS, 0, (cudaStream_t)stream>>>(a);
        DT_CUDA_TRY(cudaGetLastError());
    }
    void *args[] = {&a};
    DT_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)build_kernel, grid, BUILD_THREADS, args,
                                            smem, (cudaStream_t)stream));
    return DT_OK;
}

extern "C" int dt_build_tree(const double *xs, int64_t n, int64_t leaf_capacity, int64_t max_depth,
                             int64_t node_capacity, double *lo, double *hi, double *center,
                             double *half, int64_t *level, int64_t *start, int64_t *end,
                             int64_t *left, int64_t *right, void *packed, int64_t *meta,
                             void *workspace, size_t workspace_bytes, void *stream)
{
    return build_launch(xs, n, leaf_capacity, max_depth, node_capacity, lo, hi, center, half,
                        level, start, end, left, right, packed, meta, workspace, workspace_bytes,
                        stream, nullptr);
}

extern "C" int dt_build_tree_p2m(const double *xs, const double *qs, int64_t n,
                                 int64_t leaf_capacity, int64_t max_depth, int64_t node_capacity,
                                 double *lo, double *hi, double *center, double *half,
                                 int64_t *level, int64_t *start, int64_t *end, int64_t *left,
                                 int64_t *right, void *packed, int64_t *meta, int64_t order,
                                 double *moments_eval, int64_t eval_stride, double *xq,
                                 void *workspace, size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(order >= 0 && order + 1 <= 32, "dt_build_tree_p2m needs moment order <= 31");
    DT_CHECK_ARG(qs && moments_eval && xq, "null pointer");
    DT_CHECK_ARG(eval_stride >= order + 1 && eval_stride % 2 == 0,
                 "eval_stride must be even and >= order + 1");
    DT_CHECK_ARG(((uintptr_t)moments_eval & 15) == 0 && ((uintptr_t)xq & 15) == 0,
                 "moments_eval and xq must be 16-byte aligned");
    const P2mArgs p2m{xs, qs, center, start, end, order, moments_eval, eval_stride,
                      (double2 *)xq};
    return build_launch(xs, n, leaf_capacity, max_depth, node_capacity, lo, hi, center, half,
                        level, start, end, left, right, packed, meta, workspace, workspace_bytes,
                        stream, &p2m);
}
