// (c) Upward pass: P2M at the leaves, M2M (binomial shift) per level.
//
// Reference: tree.py:224-238 computes every node's moments
//     m_k = sum_j q_j (x_j - c)^k / k!,   k = 0..order,
// directly from its own sources, level by level (O(depth * N * order)).
// Here each leaf is formed from its sources (one warp per leaf, coalesced
// loads, per-lane register accumulators, smem transpose-reduce), then each
// internal node is the sum of its children shifted to its center:
//     m_k(parent) = sum_{j<=k} m_j(child) * delta^(k-j) / (k-j)!,
//     delta = c_child - c_parent,
// bottom-up, one grid barrier per level (cooperative persistent kernel).
// The shift is exact algebra; round-off differs from the reference's direct
// sums at the 1e-16 level of sum|q| r^k / k!.
// Algorithmic HBM bytes: P2M 16 N + 8 (order+1) leaves; M2M 24 (order+1)
// per internal node (two child rows read, one row written).
#include <cooperative_groups.h>

#include "dt_common.cuh"

namespace cg = cooperative_groups;

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

// P2M for one leaf, order + 1 <= 32, one warp.
__device__ void p2m_leaf_reg(const MomArgs &a, int64_t node, double (*tr)[33])
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    const int64_t s = a.start[node], e = a.end[node];
    const double c = a.center[node];
    double acc[REG_ORDER];
#pragma unroll
    for (int k = 0; k < REG_ORDER; ++k)
        acc[k] = 0.0;
    for (int64_t j = s + lane; j < e; j += 32) {
        double t = __ldg(a.xs + j) - c;
        double term = __ldg(a.qs + j);
        acc[0] += term;
#pragma unroll
        for (int k = 1; k < REG_ORDER; ++k) {
            if (k < o1) {
                term *= t * inv_k(k);
                acc[k] += term;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < REG_ORDER; ++k)
        tr[k][lane] = acc[k];
    __syncwarp();
    if (lane < o1) {
        double sum = 0.0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l)
            sum += tr[lane][l];
        a.moments[node * o1 + lane] = sum;
    }
    __syncwarp();
}

// P2M for one leaf, any order <= 127 (per-order warp reductions).
__device__ void p2m_leaf_generic(const MomArgs &a, int64_t node, double *row_smem)
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    const int64_t s = a.start[node], e = a.end[node];
    const double c = a.center[node];
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
        a.moments[node * o1 + k] = row_smem[k];
    __syncwarp();
}

// M2M for one internal node (one warp): sum of shifted child rows.
__device__ void m2m_node(const MomArgs &a, int64_t node, double *pw, double *mrow)
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    const double c = a.center[node];
    double out[MAX_ORDER1 / 32];
#pragma unroll
    for (int i = 0; i < MAX_ORDER1 / 32; ++i)
        out[i] = 0.0;
    const int64_t kids[2] = {__ldcg(a.left + node), __ldcg(a.right + node)};
    for (int ci = 0; ci < 2; ++ci) {
        const int64_t ch = kids[ci];
        if (ch < 0)
            continue;
        const double delta = a.center[ch] - c;
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
            a.moments[node * o1 + k] = out[i];
    }
}

__global__ void __launch_bounds__(MOM_THREADS) moments_kernel(MomArgs a)
{
    cg::grid_group grid = cg::this_grid();
    __shared__ double tr[MOM_WARPS][32][33];
    __shared__ double pw_s[MOM_WARPS][MAX_ORDER1];
    __shared__ double row_s[MOM_WARPS][MAX_ORDER1];
    const volatile int64_t *meta = a.meta;
    const int warp = threadIdx.x >> 5;
    const int64_t gwarp = (int64_t)blockIdx.x * MOM_WARPS + warp;
    const int64_t nwarps = (int64_t)gridDim.x * MOM_WARPS;
    const int64_t n_nodes = meta[DT_META_NODES];
    const int64_t depth = meta[DT_META_DEPTH];
    const bool reg_path = a.order + 1 <= REG_ORDER;

    // P2M: every leaf, any level
    for (int64_t node = gwarp; node < n_nodes; node += nwarps) {
        if (__ldg(a.left + node) >= 0 || __ldg(a.right + node) >= 0)
            continue;
        if (reg_path)
            p2m_leaf_reg(a, node, tr[warp]);
        else
            p2m_leaf_generic(a, node, row_s[warp]);
    }
    grid.sync();
    // M2M bottom-up
    for (int64_t lev = depth - 1; lev >= 0; --lev) {
        const int64_t f0 = meta[DT_META_LEVEL0 + lev];
        const int64_t f1 = meta[DT_META_LEVEL0 + lev + 1];
        for (int64_t node = f0 + gwarp; node < f1; node += nwarps) {
            if (__ldg(a.left + node) < 0 && __ldg(a.right + node) < 0)
                continue;
            m2m_node(a, node, pw_s[warp], row_s[warp]);
        }
        grid.sync();
    }
}

}  // namespace

extern "C" int dt_moments(const double *xs, const double *qs, const double *center,
                          const int64_t *start, const int64_t *end, const int64_t *left,
                          const int64_t *right, const int64_t *meta, int64_t order,
                          double *moments, void *stream)
{
    DT_CHECK_ARG(order >= 0 && order < MAX_ORDER1, "moment order must be in [0, 127]");
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta && moments,
                 "null pointer");
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, moments};
    int per_sm = 0;
    DT_CUDA_TRY(
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, moments_kernel, MOM_THREADS, 0));
    if (per_sm < 1)
        return dt_set_error(DT_ERR_CUDA, "moments kernel cannot be resident");
    int grid = dt_num_sms() * (per_sm > 4 ? 4 : per_sm);
    void *args[] = {&a};
    DT_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)moments_kernel, grid, MOM_THREADS, args,
                                            0, (cudaStream_t)stream));
    return DT_OK;
}
