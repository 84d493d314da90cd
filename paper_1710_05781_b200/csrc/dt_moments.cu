// (c) Upward pass: P2M at the leaves, M2M (binomial shift) bottom-up.
//
// Reference: tree.py:224-238 computes every node's moments
//     m_k = sum_j q_j (x_j - c)^k / k!,   k = 0..order,
// directly from its own sources, level by level (O(depth * N * order)).
// Here each leaf is formed from its sources and each internal node is the
// sum of its children shifted to its center,
//     m_k(parent) = sum_{j<=k} m_j(child) * delta^(k-j) / (k-j)!,
//     delta = c_child - c_parent,
// the binomial transform of the raw power sums S_k = k! m_k, applied in
// place as 31 passes of Pascal's rule S_k += delta S_(k-1).
//   order + 1 <= 32 (upward_kernel): one fused kernel on the traversal-layout
//     rows M_k = c_k S_k only (the reference layout is derived on request):
//     warps take 32 node slots at a time, deepest first, form the leaves
//     among them (P2M with split powers, 2 lanes per leaf), and every formed
//     leaf climbs: sibling pairs formed by the same warp complete their
//     parent directly, others bump the parent's arrival counter and the
//     lane whose arrival completes a parent keeps it; the warp forms the
//     kept parents two lanes per parent (one child each, raw sums in
//     registers) before those lanes climb on.  The M2M chains thus run while other
//     warps are still in P2M.  The shard plan (multi-GPU) restricts it to
//     one rank's subtrees; shard_finish_kernel forms the levels above the
//     cut with the same arithmetic, thread per node.
//   higher orders: warp per leaf + the same dataflow with a Toeplitz shift,
//     both layouts written.
// The shift is exact algebra; round-off differs from the reference's direct
// sums at the 1e-16 level of sum|q| r^k / k!.
// Algorithmic HBM bytes: P2M 16 N + 8 (order+1) leaves; M2M 24 (order+1)
// per internal node (two child rows read, one row written).

#include <algorithm>

#include "dt_common.cuh"
#include "dt_farcoef.cuh"
#include "dt_p2m.cuh"


namespace {

constexpr int MOM_THREADS = 128;
constexpr int MOM_WARPS = MOM_THREADS / 32;
constexpr int REG_ORDER = 32;      // order + 1 <= 32: register path
constexpr int MAX_ORDER1 = 128;    // order + 1 <= 128 supported

struct MomArgs {
    const double *xs, *qs, *center;
    const int64_t *start, *end, *left, *right, *meta;
    int64_t order;
    double *moments;
    double *meval;     // optional traversal copy: M_0 = m_0, M_k = (k-1)! gamma_(k-1) m_k
    int64_t estride;   // its row stride (even, >= order + 1; pad entries are 0)
    int32_t *parent;   // workspace: parent index per node (-1 at the root)
    int32_t *arrived;  // workspace: finished children per node
    const int64_t *plan;  // optional shard plan (DT_PLAN_*): restrict to this rank's subtrees
    unsigned *chunk_ctr;  // workspace: upward_kernel's chunk counter (zeroed by the prep kernel)
    double2 *xq;          // optional: the traversal's (x, q) pairs, written by P2M
};

__constant__ double c_inv_k[MAX_ORDER1] = {  // 1/k rounded to nearest (k >= 1)
    0.0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-2,
    0x1.0000000000000p-2, 0x1.999999999999ap-3, 0x1.5555555555555p-3, 0x1.2492492492492p-3,
    0x1.0000000000000p-3, 0x1.c71c71c71c71cp-4, 0x1.999999999999ap-4, 0x1.745d1745d1746p-4,
    0x1.5555555555555p-4, 0x1.3b13b13b13b14p-4, 0x1.2492492492492p-4, 0x1.1111111111111p-4,
    0x1.0000000000000p-4, 0x1.e1e1e1e1e1e1ep-5, 0x1.c71c71c71c71cp-5, 0x1.af286bca1af28p-5,
    0x1.999999999999ap-5, 0x1.8618618618618p-5, 0x1.745d1745d1746p-5, 0x1.642c8590b2164p-5,
    0x1.5555555555555p-5, 0x1.47ae147ae147bp-5, 0x1.3b13b13b13b14p-5, 0x1.2f684bda12f68p-5,
    0x1.2492492492492p-5, 0x1.1a7b9611a7b96p-5, 0x1.1111111111111p-5, 0x1.0842108421084p-5,
    0x1.0000000000000p-5, 0x1.f07c1f07c1f08p-6, 0x1.e1e1e1e1e1e1ep-6, 0x1.d41d41d41d41dp-6,
    0x1.c71c71c71c71cp-6, 0x1.bacf914c1bad0p-6, 0x1.af286bca1af28p-6, 0x1.a41a41a41a41ap-6,
    0x1.999999999999ap-6, 0x1.8f9c18f9c18fap-6, 0x1.8618618618618p-6, 0x1.7d05f417d05f4p-6,
    0x1.745d1745d1746p-6, 0x1.6c16c16c16c17p-6, 0x1.642c8590b2164p-6, 0x1.5c9882b931057p-6,
    0x1.5555555555555p-6, 0x1.4e5e0a72f0539p-6, 0x1.47ae147ae147bp-6, 0x1.4141414141414p-6,
    0x1.3b13b13b13b14p-6, 0x1.3521cfb2b78c1p-6, 0x1.2f684bda12f68p-6, 0x1.29e4129e4129ep-6,
    0x1.2492492492492p-6, 0x1.1f7047dc11f70p-6, 0x1.1a7b9611a7b96p-6, 0x1.15b1e5f75270dp-6,
    0x1.1111111111111p-6, 0x1.0c9714fbcda3bp-6, 0x1.0842108421084p-6, 0x1.0410410410410p-6,
    0x1.0000000000000p-6, 0x1.f81f81f81f820p-7, 0x1.f07c1f07c1f08p-7, 0x1.e9131abf0b767p-7,
    0x1.e1e1e1e1e1e1ep-7, 0x1.dae6076b981dbp-7, 0x1.d41d41d41d41dp-7, 0x1.cd85689039b0bp-7,
    0x1.c71c71c71c71cp-7, 0x1.c0e070381c0e0p-7, 0x1.bacf914c1bad0p-7, 0x1.b4e81b4e81b4fp-7,
    0x1.af286bca1af28p-7, 0x1.a98ef606a63bep-7, 0x1.a41a41a41a41ap-7, 0x1.9ec8e951033d9p-7,
    0x1.999999999999ap-7, 0x1.948b0fcd6e9e0p-7, 0x1.8f9c18f9c18fap-7, 0x1.8acb90f6bf3aap-7,
    0x1.8618618618618p-7, 0x1.8181818181818p-7, 0x1.7d05f417d05f4p-7, 0x1.78a4c8178a4c8p-7,
    0x1.745d1745d1746p-7, 0x1.702e05c0b8170p-7, 0x1.6c16c16c16c17p-7, 0x1.6816816816817p-7,
    0x1.642c8590b2164p-7, 0x1.6058160581606p-7, 0x1.5c9882b931057p-7, 0x1.58ed2308158edp-7,
    0x1.5555555555555p-7, 0x1.51d07eae2f815p-7, 0x1.4e5e0a72f0539p-7, 0x1.4afd6a052bf5bp-7,
    0x1.47ae147ae147bp-7, 0x1.446f86562d9fbp-7, 0x1.4141414141414p-7, 0x1.3e22cbce4a902p-7,
    0x1.3b13b13b13b14p-7, 0x1.3813813813814p-7, 0x1.3521cfb2b78c1p-7, 0x1.323e34a2b10bfp-7,
    0x1.2f684bda12f68p-7, 0x1.2c9fb4d812ca0p-7, 0x1.29e4129e4129ep-7, 0x1.27350b8812735p-7,
    0x1.2492492492492p-7, 0x1.21fb78121fb78p-7, 0x1.1f7047dc11f70p-7, 0x1.1cf06ada2811dp-7,
    0x1.1a7b9611a7b96p-7, 0x1.1811811811812p-7, 0x1.15b1e5f75270dp-7, 0x1.135c81135c811p-7,
    0x1.1111111111111p-7, 0x1.0ecf56be69c90p-7, 0x1.0c9714fbcda3bp-7, 0x1.0a6810a6810a7p-7,
    0x1.0842108421084p-7, 0x1.0624dd2f1a9fcp-7, 0x1.0410410410410p-7, 0x1.0204081020408p-7,
};


__device__ __forceinline__ double inv_k(int k) { return c_inv_k[k]; }

// Store m_k of `node` (and its scaled traversal copy).
__device__ __forceinline__ void put_moment(const MomArgs &a, int64_t node, int k, double m)
{
    a.moments[node * (a.order + 1) + k] = m;
    if (a.meval) {
        a.meval[node * a.estride + k] = k == 0 ? m : __dmul_rn(m, c_mev_m[k]);
        if (k == a.order && a.estride > a.order + 1)
            a.meval[node * a.estride + k + 1] = 0.0;
    }
}

// P2M for one leaf, any order <= 127 (per-order warp reductions).
__device__ void p2m_leaf_generic(const MomArgs &a, int64_t node, int64_t s, int64_t e, double c,
                                 double *row_smem)
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    for (int k = lane; k < o1; k += 32)
        row_smem[k] = 0.0;
    __syncwarp();
    for (int64_t j0 = s; j0 < e; j0 += 32) {
        int64_t j = j0 + lane;
        double t = 0.0, term = 0.0;
        if (j < e) {
            t = __ldg(a.xs + j) - c;
            term = __ldg(a.qs + j);
        }
        for (int k = 0; k < o1; ++k) {
            if (k > 0)
                term *= t * inv_k(k);
            double v = dt_warp_sum(term);
            if (lane == 0)
                row_smem[k] += v;
        }
    }
    __syncwarp();
    for (int k = lane; k < o1; k += 32)
        put_moment(a, node, k, row_smem[k]);
    __syncwarp();
}

// M2M for one internal node (one warp): sum of shifted child rows.
__device__ void m2m_node(const MomArgs &a, int64_t node, int64_t left, int64_t right, double c,
                         double *pw, double *mrow)
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    double out[MAX_ORDER1 / 32];
#pragma unroll
    for (int i = 0; i < MAX_ORDER1 / 32; ++i)
        out[i] = 0.0;
    const int64_t kids[2] = {left, right};
    for (int ci = 0; ci < 2; ++ci) {
        const int64_t ch = kids[ci];
        if (ch < 0)
            continue;
        const double delta = __ldg(a.center + ch) - c;
        // pw[i] = delta^i / i!  (multiplicative scan across lanes, chunks of 32)
        double carry = 1.0;
        for (int b = 0; b < o1; b += 32) {
            int i = b + lane;
            double v = (i == 0) ? 1.0 : delta * inv_k(i < MAX_ORDER1 ? i : 1);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                double t = __shfl_up_sync(DT_FULL, v, o);
                if (lane >= o)
                    v *= t;
            }
            v *= carry;
            if (i < o1)
                pw[i] = v;
            carry = __shfl_sync(DT_FULL, v, 31);
        }
        for (int k = lane; k < o1; k += 32)
            mrow[k] = __ldcg(a.moments + ch * o1 + k);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < MAX_ORDER1 / 32; ++i) {
            int k = lane + 32 * i;
            if (k < o1) {
                double s = 0.0;
                for (int j = 0; j <= k; ++j)
                    s = __fma_rn(mrow[j], pw[k - j], s);
                out[i] += s;
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < MAX_ORDER1 / 32; ++i) {
        int k = lane + 32 * i;
        if (k < o1)
            put_moment(a, node, k, out[i]);
    }
}

__global__ void moments_prep_kernel(MomArgs a)
{
    if (__ldg(a.meta + DT_META_OVERFLOW))
        return;  // the build ran out of node capacity: the caller rebuilds
    const int64_t n = __ldg(a.meta + DT_META_NODES);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        a.arrived[i] = 0;
        if (i == 0 && a.chunk_ctr)
            *a.chunk_ctr = 0u;
        const int64_t l = __ldg(a.left + i), r = __ldg(a.right + i);
        if (l >= 0)
            a.parent[l] = (int32_t)i;
        if (r >= 0)
            a.parent[r] = (int32_t)i;
        if (i == 0)
            a.parent[0] = -1;
    }
}

__global__ void __launch_bounds__(MOM_THREADS) moments_kernel(MomArgs a)
{
    __shared__ double pw_s[MOM_WARPS][MAX_ORDER1];
    __shared__ double row_s[MOM_WARPS][MAX_ORDER1];
    const int warp = threadIdx.x >> 5, lane = dt_lane();
    const int64_t gwarp = (int64_t)blockIdx.x * MOM_WARPS + warp;
    const int64_t nwarps = (int64_t)gridDim.x * MOM_WARPS;
    const int64_t n_nodes = __ldg(a.meta + DT_META_NODES);

    // each warp scans 32 consecutive nodes at a time for leaves
    for (int64_t c0 = gwarp * 32; c0 < n_nodes; c0 += nwarps * 32) {
        const int64_t mine = c0 + lane;
        bool leaf = false;
        int64_t s = 0, e = 0;
        double ctr = 0.0;
        if (mine < n_nodes) {
            leaf = __ldg(a.left + mine) < 0 && __ldg(a.right + mine) < 0;
            s = __ldg(a.start + mine);
            e = __ldg(a.end + mine);
            ctr = __ldg(a.center + mine);
        }
        unsigned leaves = __ballot_sync(DT_FULL, leaf);
        while (leaves) {
            const int i = __ffs(leaves) - 1;
            leaves &= leaves - 1;
            int64_t node = c0 + i;
            const int64_t ns = __shfl_sync(DT_FULL, s, i);
            const int64_t ne = __shfl_sync(DT_FULL, e, i);
            const double nc = __shfl_sync(DT_FULL, ctr, i);
            p2m_leaf_generic(a, node, ns, ne, nc, row_s[warp]);
            // climb while this warp completes the parent's last child
            while (true) {
                __threadfence();
                __syncwarp();
                int64_t par = -1;
                if (lane == 0) {
                    const int32_t pp = __ldcg(a.parent + node);
                    if (pp >= 0) {
                        const int64_t pl = __ldg(a.left + pp), pr = __ldg(a.right + pp);
                        const int need = (pl >= 0) + (pr >= 0);
                        const int got = atomicAdd(a.arrived + pp, 1) + 1;
                        if (got == need)
                            par = pp;
                    }
                }
                par = __shfl_sync(DT_FULL, par, 0);
                if (par < 0)
                    break;
                __threadfence();
                m2m_node(a, par, __ldg(a.left + par), __ldg(a.right + par),
                         __ldg(a.center + par), pw_s[warp], row_s[warp]);
                node = par;
            }
        }
    }
}

// ---- order + 1 <= 32: one fused upward pass on traversal-layout rows ----
//
// Rows are stored once, in the traversal layout M_k = c_k S_k (c_0 = 1,
// c_k = gamma_(k-1) / k = c_mev_s[k], dt_farcoef.cuh; S_k = k! m_k the raw
// power sums), which is all the traversal reads; the reference layout m_k is
// derived from them only on request (dt_moments_from_eval).  A parent is
// formed by shift_child on each child row (to raw sums, binomial shift, back)
// and one addition; the two-lane form (form_node_pair) and the thread form
// (up_level_threads, shard_finish) do exactly that, so the rows are
// bit-identical whichever form (and whichever rank) produced them.

// ---- M2M: two lanes per node (or one thread), raw sums in registers ----
//
// Child shift: a child row (M basis) is
// converted to raw sums S_k = M_k / c_k, shifted to the parent's centre by
// 31 in-place Pascal passes S_k += delta S_(k-1) (descending k, so every
// update reads the previous pass), and converted back, T_k = S_k c_k; the
// parent row is T(left) + T(right) (an only child's T as it is).  One
// thread holds the whole row in registers: no shuffles or selects, and the
// 496 FMAs of a pass sequence are independent within a pass.
__device__ __forceinline__ void shift_child(const double *__restrict__ row, int o1, double delta,
                                            double (&T)[REG_ORDER])
{
    const double2 *r2 = reinterpret_cast<const double2 *>(row);
#pragma unroll
    for (int k = 0; k < REG_ORDER; k += 2) {
        double2 v = k < o1 ? __ldcg(r2 + (k >> 1)) : make_double2(0.0, 0.0);
        T[k] = k == 0 ? v.x : __dmul_rn(v.x, c_inv_mevs[k]);
        T[k + 1] = k + 1 < o1 ? __dmul_rn(v.y, c_inv_mevs[k + 1]) : 0.0;
    }
#pragma unroll
    for (int i = 1; i < REG_ORDER; ++i) {
#pragma unroll
        for (int k = REG_ORDER - 1; k >= i; --k)
            T[k] = __fma_rn(delta, T[k - 1], T[k]);
    }
#pragma unroll
    for (int k = 1; k < REG_ORDER; ++k)
        T[k] = __dmul_rn(T[k], c_mev_s[k]);
}

// Node `node` (internal) formed by the lane pair (sub 0: left child, sub 1:
// right child); each lane then stores half of the row.  Both lanes of the
// pair must call it (inactive pairs with node < 0).
#ifdef DT_UP_TRACE
// development (tools/upward_levels.py): [0] kernel start (min over blocks),
// [1 + L] the last formation of level L
__device__ unsigned long long g_uptrace[72];
#endif
__device__ __forceinline__ void form_node_pair(const MomArgs &a, int64_t node, int sub)
{
    const int o1 = (int)a.order + 1;
    const int64_t es = a.estride;
    int64_t ch = -1, other = -1;
    double delta = 0.0;
    if (node >= 0) {
        const int64_t l = __ldg(a.left + node), r = __ldg(a.right + node);
        ch = sub ? r : l;
        other = sub ? l : r;
        if (ch >= 0)
            delta = __ldg(a.center + ch) - __ldg(a.center + node);
    }
    double T[REG_ORDER];
    if (ch >= 0) {
        shift_child(a.meval + ch * es, o1, delta, T);
    } else {
#pragma unroll
        for (int k = 0; k < REG_ORDER; ++k)
            T[k] = 0.0;
    }
    // lane sub keeps orders [16 sub, 16 sub + 16): its own T plus the partner's
    double out[REG_ORDER / 2];
#pragma unroll
    for (int k = 0; k < REG_ORDER / 2; ++k) {
        const double give = sub ? T[k] : T[k + REG_ORDER / 2];
        const double mine = sub ? T[k + REG_ORDER / 2] : T[k];
        const double got = __shfl_xor_sync(DT_FULL, give, 1);
        // left + right in that order; an only child's T as it is
        const double tl = sub ? got : mine, tr = sub ? mine : got;
        const bool has_l = sub ? other >= 0 : ch >= 0, has_r = sub ? ch >= 0 : other >= 0;
        out[k] = has_l && has_r ? tl + tr : (has_l ? tl : tr);
    }
    if (node < 0)
        return;
#ifdef DT_UP_TRACE
    if (sub == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        int L = 0;
        while (L < 60 && __ldg(a.meta + DT_META_LEVEL0 + L + 1) <= node)
            ++L;
        atomicMax(g_uptrace + 1 + L, t_);
    }
#endif
    double2 *dst = reinterpret_cast<double2 *>(a.meval + node * es);
#pragma unroll
    for (int k = 0; k < REG_ORDER / 2; k += 2) {
        const int kk = 16 * sub + k;
        if (kk < es)
            dst[kk >> 1] = make_double2(kk < o1 ? out[k] : 0.0, kk + 1 < o1 ? out[k + 1] : 0.0);
    }
}

// The fused upward pass (after moments_prep_kernel wrote parent[] and zeroed
// arrived[]): warps take 32 consecutive node slots at a time, deepest
// first (their chains are the critical path); every leaf among them is
// formed by P2M (32 / G leaves per round), then each formed leaf arrives at
// its parent, and a lane whose arrival completes a parent keeps it: the warp
// forms the kept parents (16 per call, two lanes each: 0.287 ms at
// configs[2] against 0.300 ms for the earlier 4-parents-per-warp Pascal
// passes on 8 lanes) and those lanes climb on.  Chains start while other warps are still in P2M,
// so the M2M latency overlaps the P2M throughput.  With a shard plan, leaves
// below the cut outside the rank's source range are skipped and climbs stop
// below the cut level.
#ifndef DT_UP_MINB
#define DT_UP_MINB 2
#endif
template <int G, int KMAX>
__global__ void __launch_bounds__(256, DT_UP_MINB) upward_kernel(MomArgs a)
{
    __shared__ int64_t frontier_s[8][32];
    const int warp = threadIdx.x >> 5;
    const int lane = dt_lane();
    const int sub = lane & (G - 1), grp = lane / G;
    const P2mArgs p2m{a.xs, a.qs, a.center, a.start, a.end, a.order, a.meval, a.estride, a.xq};
    // leaves below this node index were formed by the build's idle blocks
    // (dt_build_tree_p2m); they only climb here
    const int64_t preformed = a.plan ? 0 : __ldg(a.meta + DT_META_P2M_UPTO);
#ifdef DT_UP_TRACE
    if (threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        atomicMin(g_uptrace, t_);
    }
#endif
    if (__ldg(a.meta + DT_META_OVERFLOW))
        return;  // the build ran out of node capacity: the caller rebuilds
    const int64_t n = __ldg(a.meta + DT_META_NODES);
    int64_t cut_begin = 0, lo = 0, hi = 0;
    if (a.plan) {
        cut_begin = __ldg(a.plan + DT_PLAN_LEVEL_BEGIN);
        lo = __ldg(a.plan + DT_PLAN_SRC_LO);
        hi = __ldg(a.plan + DT_PLAN_SRC_HI);
    }
    // chunks are taken from a counter: a warp busy climbing does not hold
    // back the leaves of the chunks after it
    while (true) {
        unsigned chunk = 0;
        if (lane == 0)
            chunk = atomicAdd(a.chunk_ctr, 1u);
        const int64_t r0 = (int64_t)__shfl_sync(DT_FULL, chunk, 0) * 32;
        if (r0 >= n)
            break;
        const int64_t c0 = n - 32 - r0;  // may be negative for the last chunk
        const int64_t mine = c0 + lane;
        bool form = false, climb = false;
        int64_t par = -1;
        if (mine >= 0 && mine < n && __ldg(a.left + mine) < 0 && __ldg(a.right + mine) < 0) {
            const bool in = !a.plan ||
                            (__ldg(a.start + mine) >= lo && __ldg(a.end + mine) <= hi);
            // leaves above the cut are formed by every rank; they never climb
            form = (in || mine < cut_begin) && mine >= preformed;
            par = __ldcg(a.parent + mine);
            climb = in && par >= cut_begin && par >= 0;
#if DT_UP_NOCLIMB
            climb = false;
#endif
        }
        unsigned leaves = __ballot_sync(DT_FULL, form);
        while (leaves) {
            // group grp takes the grp-th remaining leaf
            unsigned m = leaves;
            for (int i = 0; i < grp && m; ++i)
                m &= m - 1;
            const bool active = m != 0;
            const int64_t node = c0 + (active ? __ffs(m) - 1 : 0);
            for (int i = 0; i < 32 / G && leaves; ++i)
                leaves &= leaves - 1;
            p2m_split_leaf<G, KMAX, false>(p2m, node, active, sub);
        }
        // Climb in rounds over a frontier of formed nodes, kept sorted and
        // compacted in the lanes, so siblings sit in adjacent lanes: a pair of
        // siblings (or an only child) completes its parent locally, with no
        // atomic; a node whose sibling is outside the frontier arrives at the
        // parent's counter (release) and keeps the parent if it is last.
        // Then the kept parents are formed, four per call (eight lanes each)
        // or one on the whole warp, and become the next frontier.
        int64_t v = climb ? mine : -1;
#ifdef DT_UP_MAXROUNDS
        for (int round_ = 0; round_ < DT_UP_MAXROUNDS; ++round_) {
#else
        while (true) {
#endif
            __syncwarp();  // this warp's rows precede the loads and releasing arrivals
            const unsigned fr = __ballot_sync(DT_FULL, v >= 0);
            if (!fr)
                break;
            const int rank = __popc(fr & ((1u << lane) - 1u));
            if (v >= 0)
                frontier_s[warp][rank] = v;
            __syncwarp();
            const int cnt = __popc(fr);
            v = lane < cnt ? frontier_s[warp][lane] : -1;
            int64_t p = -1;
            if (v >= 0) {
                p = __ldg(a.parent + v);
                if (p < cut_begin)
                    p = -1;
            }
            const int64_t p_up = __shfl_up_sync(DT_FULL, p, 1);
            const int64_t p_dn = __shfl_down_sync(DT_FULL, p, 1);
            const bool pair_hi = p >= 0 && lane > 0 && p_up == p;  // the lane below takes p
            const bool pair_lo = p >= 0 && lane < 31 && p_dn == p;
            bool take = false;
            if (p >= 0 && !pair_hi) {
                const int need = (__ldg(a.left + p) >= 0) + (__ldg(a.right + p) >= 0);
                take = pair_lo || need == 1 || arrive_acq_rel(a.arrived + p) == need - 1;
            }
            const unsigned tk = __ballot_sync(DT_FULL, take);
            if (!tk)
                break;
            if (take)
                frontier_s[warp][__popc(tk & ((1u << lane) - 1u))] = p;
            __syncwarp();  // the acquires and the parent list precede the loads
            const int np = __popc(tk);
            // two lanes per parent (left child, right child), 16 parents per call
            for (int c = 0; c < np; c += 16) {
                const int gi = c + (lane >> 1);
                form_node_pair(a, gi < np ? frontier_s[warp][gi] : -1, lane & 1);
            }
            v = lane < np ? frontier_s[warp][lane] : -1;
        }
    }
}

// M2M of one level with one thread per internal node (shard_finish): the
// child shift of form_node_pair, so the rows match bit for bit.
__device__ __forceinline__ void up_level_threads(const MomArgs &a, int64_t f0, int64_t f1,
                                                 int64_t tid, int64_t nthreads)
{
    const int o1 = (int)a.order + 1;
    const int64_t es = a.estride;
    for (int64_t node = f0 + tid; node < f1; node += nthreads) {
        const int64_t l = __ldg(a.left + node), r = __ldg(a.right + node);
        if (l < 0 && r < 0)
            continue;
        const double c = __ldg(a.center + node);
        double tl[REG_ORDER], tr[REG_ORDER];
        if (l >= 0)
            shift_child(a.meval + l * es, o1, __ldg(a.center + l) - c, tl);
        if (r >= 0)
            shift_child(a.meval + r * es, o1, __ldg(a.center + r) - c, tr);
#pragma unroll
        for (int k = 0; k < REG_ORDER; ++k) {
            const double v = l >= 0 && r >= 0 ? tl[k] + tr[k] : (l >= 0 ? tl[k] : tr[k]);
            if (k < es)
                a.meval[node * es + k] = k < o1 ? v : 0.0;
        }
    }
}


// Reference-layout moments from traversal rows: m_k = M_k / ((k-1)! gamma_(k-1))
// (tree.py:224-238 semantics, for the API's Tree.moments).
__global__ void moments_from_eval_kernel(const double *__restrict__ meval, int64_t es,
                                         const int64_t *meta, int64_t n, int64_t o1,
                                         double *__restrict__ moments)
{
    if (meta)
        n = __ldg(meta + DT_META_NODES);
    const int64_t total = n * o1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = i / o1;
        const int k = (int)(i - node * o1);
        const double v = __ldg(meval + node * es + k);
        moments[i] = k == 0 ? v : __ddiv_rn(v, c_mev_m[k]);
    }
}

// ---- multi-GPU sharding (include/disctree_b200.h "(c) sharded") ----

constexpr int PLAN_THREADS = 256;

__global__ void __launch_bounds__(PLAN_THREADS)
    shard_plan_kernel(const double *center, const double *half, const int64_t *start,
                      const int64_t *end, const int64_t *meta, int64_t n_src, const double *ys,
                      int64_t n_targets, int sorted, double theta, int64_t cut_req, int world,
                      int rank, int64_t *plan)
{
    __shared__ double s_lo[PLAN_THREADS / 32], s_hi[PLAN_THREADS / 32];
    __shared__ unsigned long long s_need_lo, s_need_hi;
    const int tid = threadIdx.x, lane = dt_lane(), warp = tid >> 5;
    const int64_t depth = __ldg(meta + DT_META_DEPTH);
    const int64_t cut = cut_req < depth ? cut_req : depth;
    const int64_t b = __ldg(meta + DT_META_LEVEL0 + cut), e = __ldg(meta + DT_META_LEVEL0 + cut + 1);
    // target extremes
    double ylo = INFINITY, yhi = -INFINITY;
    if (n_targets > 0) {
        if (sorted) {
            ylo = __ldg(ys);
            yhi = __ldg(ys + n_targets - 1);
        } else {
            for (int64_t i = tid; i < n_targets; i += PLAN_THREADS) {
                const double y = __ldg(ys + i);
                ylo = fmin(ylo, y);
                yhi = fmax(yhi, y);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ylo = fmin(ylo, __shfl_xor_sync(DT_FULL, ylo, o));
                yhi = fmax(yhi, __shfl_xor_sync(DT_FULL, yhi, o));
            }
            if (lane == 0) {
                s_lo[warp] = ylo;
                s_hi[warp] = yhi;
            }
            __syncthreads();
            ylo = s_lo[0];
            yhi = s_hi[0];
            for (int w = 1; w < PLAN_THREADS / 32; ++w) {
                ylo = fmin(ylo, s_lo[w]);
                yhi = fmax(yhi, s_hi[w]);
            }
        }
    }
    if (tid == 0) {
        s_need_lo = (unsigned long long)e;
        s_need_hi = (unsigned long long)b;
    }
    __syncthreads();
    // level-l nodes some target may open: not (h <= theta R) for some y
    if (n_targets > 0) {
        for (int64_t i = b + tid; i < e; i += PLAN_THREADS) {
            const double c = __ldg(center + i), h = __ldg(half + i);
            const double dist = c < ylo ? ylo - c : (c > yhi ? c - yhi : 0.0);
            if (h * (1.0 + 0x1p-40) > theta * dist) {
                atomicMin(&s_need_lo, (unsigned long long)i);
                atomicMax(&s_need_hi, (unsigned long long)(i + 1));
            }
        }
    }
    // owners: rank r starts at the first level-l node with start >= floor(r n / world)
    for (int r = tid; r <= world; r += PLAN_THREADS) {
        int64_t at;
        if (r == 0) {
            at = b;
        } else if (r == world) {
            at = e;
        } else {
            const int64_t want = (int64_t)(((__int128)r * n_src) / world);
            int64_t lo = b, hi = e;
            while (lo < hi) {
                const int64_t mid = lo + ((hi - lo) >> 1);
                if (__ldg(start + mid) < want)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            at = lo;
        }
        plan[DT_PLAN_OWNER0 + r] = at;
    }
    __syncthreads();
    if (tid == 0) {
        const int64_t nlo = (int64_t)s_need_lo, nhi = (int64_t)s_need_hi;
        int64_t ulo = plan[DT_PLAN_OWNER0 + rank], uhi = plan[DT_PLAN_OWNER0 + rank + 1];
        if (nlo < nhi) {
            if (ulo >= uhi) {
                ulo = nlo;
                uhi = nhi;
            } else {
                ulo = nlo < ulo ? nlo : ulo;
                uhi = nhi > uhi ? nhi : uhi;
            }
        }
        plan[DT_PLAN_CUT] = cut;
        plan[DT_PLAN_LEVEL_BEGIN] = b;
        plan[DT_PLAN_LEVEL_END] = e;
        plan[DT_PLAN_SRC_LO] = ulo < uhi ? __ldg(start + ulo) : 0;
        plan[DT_PLAN_SRC_HI] = ulo < uhi ? __ldg(end + uhi - 1) : 0;
        plan[DT_PLAN_NEED_LO] = nlo < nhi ? nlo : b;
        plan[DT_PLAN_NEED_HI] = nlo < nhi ? nhi : b;
        for (int r = world + 1; r <= DT_MAX_WORLD; ++r)
            plan[DT_PLAN_OWNER0 + r] = e;
    }
}

__global__ void shard_pack_kernel(const int64_t *plan, int rank, const double *meval, int64_t es,
                                  double *send)
{
    const int64_t a0 = __ldg(plan + DT_PLAN_OWNER0 + rank);
    const int64_t rows = __ldg(plan + DT_PLAN_OWNER0 + rank + 1) - a0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * es;
         i += (int64_t)gridDim.x * blockDim.x)
        send[i] = __ldg(meval + a0 * es + i);
}

// One block: scatter every owner's level-l rows, then M2M levels cut-1 .. 0
// (thread per node; the arithmetic of form_node_pair, so the rows match the
// single-GPU pass bit for bit).
__global__ void __launch_bounds__(256) shard_finish_kernel(MomArgs a, int world, int64_t slot_rows,
                                                           const double *recv)
{
    const int64_t es = a.estride;
    for (int r = 0; r < world; ++r) {
        const int64_t a0 = __ldg(a.plan + DT_PLAN_OWNER0 + r);
        const int64_t rows = __ldg(a.plan + DT_PLAN_OWNER0 + r + 1) - a0;
        const double *slot = recv + (int64_t)r * slot_rows * es;
        for (int64_t i = threadIdx.x; i < rows * es; i += blockDim.x)
            a.meval[a0 * es + i] = slot[i];
    }
    __syncthreads();
    const int64_t cut = __ldg(a.plan + DT_PLAN_CUT);
    for (int64_t lev = cut - 1; lev >= 0; --lev) {
        up_level_threads(a, __ldg(a.meta + DT_META_LEVEL0 + lev),
                         __ldg(a.meta + DT_META_LEVEL0 + lev + 1), threadIdx.x, blockDim.x);
        __syncthreads();
    }
}

// Upward pass for order + 1 <= 32 (honouring a.plan): the parent/arrival
// bookkeeping (which also zeroes the chunk counter), then the fused P2M +
// M2M dataflow kernel.  A level-synchronous cooperative variant (P2M, grid
// barrier, levels bottom-up two lanes per node, sparse levels in one block)
// measured 0.43-0.55 ms at configs[2] against 0.30 ms for this one: a level
// costs >= 2.6 us of formation latency plus ~5 us per grid barrier, and the
// tree is 32 levels deep.
int launch_level_moments(MomArgs &a, cudaStream_t s)
{
    const int sms = dt_num_sms();
    if (!a.parent || !a.chunk_ctr)
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace missing");
    if (!a.meval)
        return dt_set_error(DT_ERR_INVALID, "order <= 31 needs the traversal rows (moments_eval)");
    moments_prep_kernel<<<sms * 8, 256, 0, s>>>(a);
    DT_CUDA_TRY(cudaGetLastError());
    const int64_t o1 = a.order + 1;
    const int grid = sms * DT_UP_MINB;
    if (o1 <= 8)
        upward_kernel<DT_P2M_G, 8><<<grid, 256, 0, s>>>(a);
    else if (o1 <= 16)
        upward_kernel<DT_P2M_G, 16><<<grid, 256, 0, s>>>(a);
    else if (o1 <= 24)
        upward_kernel<DT_P2M_G, 24><<<grid, 256, 0, s>>>(a);
    else
        upward_kernel<DT_P2M_G, 32><<<grid, 256, 0, s>>>(a);
    DT_CUDA_TRY(cudaGetLastError());
    if (a.moments) {  // the reference layout as well (API builds ask for it lazily instead)
        moments_from_eval_kernel<<<sms * 8, 256, 0, s>>>(a.meval, a.estride, a.meta, 0, o1,
                                                         a.moments);
        DT_CUDA_TRY(cudaGetLastError());
    }
    return DT_OK;
}

}  // namespace

extern "C" size_t dt_moments_workspace(int64_t node_capacity)
{
    return (size_t)node_capacity * 2 * sizeof(int32_t) + 1024;
}

extern "C" int dt_moments(const double *xs, const double *qs, const double *center,
                          const int64_t *start, const int64_t *end, const int64_t *left,
                          const int64_t *right, const int64_t *meta, int64_t order,
                          double *moments, double *moments_eval, int64_t eval_stride,
                          int64_t node_capacity, void *workspace, size_t workspace_bytes,
                          void *stream)
{
    DT_CHECK_ARG(!moments_eval || (eval_stride >= order + 1 && eval_stride % 2 == 0),
                 "eval_stride must be even and >= order + 1");
    DT_CHECK_ARG(order >= 0 && order < MAX_ORDER1, "moment order must be in [0, 127]");
    DT_CHECK_ARG(node_capacity >= 1 && node_capacity < (int64_t)1 << 31, "bad node capacity");
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta, "null pointer");
    DT_CHECK_ARG(order + 1 <= REG_ORDER ? moments_eval != nullptr : moments != nullptr,
                 "order <= 31 needs moments_eval, higher orders need moments");
    DT_CHECK_ARG(((uintptr_t)moments_eval & 15) == 0, "moments_eval must be 16-byte aligned");
    if (!workspace || workspace_bytes < dt_moments_workspace(node_capacity))
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace too small");
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, moments, moments_eval,
              eval_stride, (int32_t *)workspace, (int32_t *)workspace + node_capacity, nullptr,
              (unsigned *)((int32_t *)workspace + 2 * node_capacity)};
    cudaStream_t s = (cudaStream_t)stream;
    const int sms = dt_num_sms();
    if (order + 1 <= REG_ORDER)
        return launch_level_moments(a, s);
    moments_prep_kernel<<<sms * 8, 256, 0, s>>>(a);
    DT_CUDA_TRY(cudaGetLastError());
    moments_kernel<<<sms * 8, MOM_THREADS, 0, s>>>(a);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_shard_plan(const double *center, const double *half, const int64_t *start,
                             const int64_t *end, const int64_t *meta, int64_t n_src,
                             const double *ys, int64_t n_targets, int targets_sorted,
                             double theta, int64_t cut_level, int world, int rank, int64_t *plan,
                             void *stream)
{
    DT_CHECK_ARG(center && half && start && end && meta && plan, "null pointer");
    DT_CHECK_ARG(n_targets == 0 || ys, "null targets");
    DT_CHECK_ARG(world >= 1 && world <= DT_MAX_WORLD && rank >= 0 && rank < world,
                 "bad world size / rank");
    DT_CHECK_ARG(cut_level >= 0 && cut_level <= 20, "cut_level must be in [0, 20]");
    DT_CHECK_ARG(theta > 0.0, "theta must be > 0");
    shard_plan_kernel<<<1, PLAN_THREADS, 0, (cudaStream_t)stream>>>(
        center, half, start, end, meta, n_src, ys, n_targets, targets_sorted, theta, cut_level,
        world, rank, plan);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

// dt_moments that also writes the traversal's interleaved sources xq[2n]
// (what dt_pack_sources does) from the loads P2M makes anyway: every source
// lies in exactly one leaf.  Orders > 31 pack with the separate kernel.
extern "C" int dt_pack_sources(const double *xs, const double *qs, int64_t n, double *xq,
                               void *stream);
extern "C" int dt_moments_pack(const double *xs, const double *qs, int64_t n_src,
                               const double *center, const int64_t *start, const int64_t *end,
                               const int64_t *left, const int64_t *right, const int64_t *meta,
                               int64_t order, double *moments, double *moments_eval,
                               int64_t eval_stride, int64_t node_capacity, double *xq,
                               void *workspace, size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(n_src >= 0 && (n_src == 0 || xq), "null xq");
    DT_CHECK_ARG(((uintptr_t)xq & 15) == 0, "xq must be 16-byte aligned");
    DT_CHECK_ARG(eval_stride >= order + 1 && eval_stride % 2 == 0,
                 "eval_stride must be even and >= order + 1");
    DT_CHECK_ARG(order >= 0 && order < MAX_ORDER1, "moment order must be in [0, 127]");
    DT_CHECK_ARG(node_capacity >= 1 && node_capacity < (int64_t)1 << 31, "bad node capacity");
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta, "null pointer");
    if (order + 1 > REG_ORDER) {
        const int rc = dt_moments(xs, qs, center, start, end, left, right, meta, order, moments,
                                  moments_eval, eval_stride, node_capacity, workspace,
                                  workspace_bytes, stream);
        return rc != DT_OK ? rc : dt_pack_sources(xs, qs, n_src, xq, stream);
    }
    DT_CHECK_ARG(moments_eval && ((uintptr_t)moments_eval & 15) == 0,
                 "moments_eval must be given and 16-byte aligned");
    if (!workspace || workspace_bytes < dt_moments_workspace(node_capacity))
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace too small");
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, moments, moments_eval,
              eval_stride, (int32_t *)workspace, (int32_t *)workspace + node_capacity, nullptr,
              (unsigned *)((int32_t *)workspace + 2 * node_capacity), (double2 *)xq};
    return launch_level_moments(a, (cudaStream_t)stream);
}

extern "C" int dt_moments_from_eval(const double *moments_eval, int64_t eval_stride,
                                    int64_t n_nodes, int64_t order, double *moments,
                                    void *stream)
{
    DT_CHECK_ARG(n_nodes >= 0 && order >= 0 && order < MAX_ORDER1, "bad node count / order");
    DT_CHECK_ARG(eval_stride >= order + 1, "eval_stride must be >= order + 1");
    if (n_nodes == 0)
        return DT_OK;
    DT_CHECK_ARG(moments_eval && moments, "null pointer");
    const int64_t total = n_nodes * (order + 1);
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)dt_num_sms() * 8);
    moments_from_eval_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        moments_eval, eval_stride, nullptr, n_nodes, order + 1, moments);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" size_t dt_shard_rows_bytes(int64_t cut_level, int64_t order, int64_t eval_stride)
{
    if (cut_level < 0 || cut_level > 20 || order < 0 || eval_stride < order + 1)
        return 0;
    return ((size_t)1 << cut_level) * (size_t)eval_stride * sizeof(double);
}

extern "C" int dt_moments_partial(const double *xs, const double *qs, const double *center,
                                  const int64_t *start, const int64_t *end, const int64_t *left,
                                  const int64_t *right, const int64_t *meta, const int64_t *plan,
                                  int64_t order, double *moments, double *moments_eval,
                                  int64_t eval_stride, int64_t node_capacity, void *workspace,
                                  size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(order >= 0 && order + 1 <= REG_ORDER, "sharded moments need order <= 31");
    DT_CHECK_ARG(!moments_eval || (eval_stride >= order + 1 && eval_stride % 2 == 0),
                 "eval_stride must be even and >= order + 1");
    DT_CHECK_ARG(node_capacity >= 1 && node_capacity < (int64_t)1 << 31, "bad node capacity");
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta && plan &&
                     moments_eval,
                 "null pointer");
    if (!workspace || workspace_bytes < dt_moments_workspace(node_capacity))
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace too small");
    // the reference layout (moments) is derived by dt_shard_finish, once every row exists
    (void)moments;
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, nullptr, moments_eval,
              eval_stride, (int32_t *)workspace, (int32_t *)workspace + node_capacity, plan,
              (unsigned *)((int32_t *)workspace + 2 * node_capacity)};
    return launch_level_moments(a, (cudaStream_t)stream);
}

extern "C" int dt_shard_pack(const int64_t *plan, int rank, int64_t cut_level, int64_t order,
                             const double *moments, const double *moments_eval,
                             int64_t eval_stride, double *send, void *stream)
{
    (void)moments;  // the traversal rows carry everything (reference layout derived later)
    DT_CHECK_ARG(plan && moments_eval && send, "null pointer");
    DT_CHECK_ARG(rank >= 0 && rank < DT_MAX_WORLD, "bad rank");
    DT_CHECK_ARG(cut_level >= 0 && cut_level <= 20 && order >= 0, "bad cut level / order");
    DT_CHECK_ARG(eval_stride >= order + 1 && eval_stride % 2 == 0,
                 "eval_stride must be even and >= order + 1");
    const int64_t cells = ((int64_t)1 << cut_level) * eval_stride;
    int blocks = (int)((cells + 255) / 256);
    blocks = blocks < 1 ? 1 : (blocks > 4 * dt_num_sms() ? 4 * dt_num_sms() : blocks);
    shard_pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(plan, rank, moments_eval,
                                                               eval_stride, send);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_shard_finish(const int64_t *plan, int world, int64_t cut_level,
                               const double *recv, const double *center, const int64_t *left,
                               const int64_t *right, const int64_t *meta, int64_t order,
                               double *moments, double *moments_eval, int64_t eval_stride,
                               void *stream)
{
    DT_CHECK_ARG(plan && recv && center && left && right && meta && moments_eval, "null pointer");
    DT_CHECK_ARG(world >= 1 && world <= DT_MAX_WORLD, "bad world size");
    DT_CHECK_ARG(cut_level >= 0 && cut_level <= 20, "bad cut level");
    DT_CHECK_ARG(order >= 0 && order + 1 <= REG_ORDER, "sharded moments need order <= 31");
    DT_CHECK_ARG(eval_stride >= order + 1 && eval_stride % 2 == 0,
                 "eval_stride must be even and >= order + 1");
    // start/end are only read by the range filter, which is open here
    MomArgs a{nullptr, nullptr, center, nullptr, nullptr, left, right, meta, order, nullptr,
              moments_eval, eval_stride, nullptr, nullptr, plan};
    cudaStream_t s = (cudaStream_t)stream;
    shard_finish_kernel<<<1, 256, 0, s>>>(a, world, (int64_t)1 << cut_level, recv);
    DT_CUDA_TRY(cudaGetLastError());
    if (moments) {
        moments_from_eval_kernel<<<dt_num_sms() * 8, 256, 0, s>>>(moments_eval, eval_stride, meta,
                                                                  0, order + 1, moments);
        DT_CUDA_TRY(cudaGetLastError());
    }
    return DT_OK;
}

#ifdef DT_UP_TRACE
extern "C" int dt_debug_uptrace(unsigned long long *host, int reset)
{
    cudaMemcpyFromSymbol(host, g_uptrace, sizeof(g_uptrace));
    if (reset) {
        unsigned long long z[72];
        for (int i = 0; i < 72; ++i)
            z[i] = 0;
        z[0] = ~0ull;
        cudaMemcpyToSymbol(g_uptrace, z, sizeof(z));
    }
    return 0;
}
#endif
