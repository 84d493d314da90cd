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
    double *meval;     // optional traversal copy: M'_0 = m_0, M'_k = (k-1)! m_k
    int64_t estride;   // its row stride (even, >= order + 1; pad entries are 0)
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

__constant__ double c_fact_km1[MAX_ORDER1] = {  // (k-1)! rounded (k >= 1)
    0.0, 0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p+1,
    0x1.8000000000000p+2, 0x1.8000000000000p+4, 0x1.e000000000000p+6, 0x1.6800000000000p+9,
    0x1.3b00000000000p+12, 0x1.3b00000000000p+15, 0x1.6260000000000p+18, 0x1.baf8000000000p+21,
    0x1.308a800000000p+25, 0x1.c8cfc00000000p+28, 0x1.7328cc0000000p+32, 0x1.44c3b28000000p+36,
    0x1.3077775800000p+40, 0x1.3077775800000p+44, 0x1.437eeecd80000p+48, 0x1.6beecca730000p+52,
    0x1.b02b930689000p+56, 0x1.0e1b3be415a00p+61, 0x1.6283be9b5c620p+65, 0x1.e77526159f06cp+69,
    0x1.5e5c335f8a4cep+74, 0x1.06c52687a7b9ap+79, 0x1.9a940c33f6121p+83, 0x1.4d9849ea37eebp+88,
    0x1.19787e5d9f316p+93, 0x1.ec92dd23d6967p+97, 0x1.be6518687a785p+102, 0x1.a27ec6e1f2d0dp+107,
    0x1.956ad0aae33a4p+112, 0x1.956ad0aae33a4p+117, 0x1.a21627303a541p+122, 0x1.bc3789a33df96p+127,
    0x1.e5dcbe8a8bc8cp+132, 0x1.114c2b2deea0fp+138, 0x1.3c0011ed1bea1p+143, 0x1.774015499125fp+148,
    0x1.c95619f1a8e64p+153, 0x1.1dd5d037098fep+159, 0x1.6e39f2c684406p+164, 0x1.e0ac0ea48d948p+169,
    0x1.42f399d68f1fcp+175, 0x1.bc0ef38704cbbp+180, 0x1.383a833aef5f3p+186, 0x1.c0d41ca4b818ep+191,
    0x1.499bc508f7324p+197, 0x1.ee69a78d72cb6p+202, 0x1.7a88e4484be3bp+208, 0x1.27baf2587b49ep+214,
    0x1.d751f23d047dcp+219, 0x1.7ef294d193a63p+225, 0x1.3d20e33d8e45ap+231, 0x1.0b93bfbbf00acp+237,
    0x1.cbe5f18b04928p+242, 0x1.92693359a4003p+248, 0x1.6665b1bbd6102p+254, 0x1.44cc291239feap+260,
    0x1.2b6c35dccd76cp+266, 0x1.18b5727f009f5p+272, 0x1.0b8cf1210c97ep+278, 0x1.0330899804332p+284,
    0x1.fe478ee34844ap+289, 0x1.fe478ee34844ap+295, 0x1.0320568f6ab2ep+302, 0x1.0b395943e6087p+308,
    0x1.17c0097314d0dp+314, 0x1.293c0a0a461dep+320, 0x1.4074bad313983p+326, 0x1.5e7fac56dd6e8p+332,
    0x1.84d5a3305da69p+338, 0x1.b5705796695b6p+344, 0x1.f2f423e7902c4p+350, 0x1.207524c1df599p+357,
    0x1.5209471331bd0p+363, 0x1.916b0466cb107p+369, 0x1.e2f4c14bac4fcp+375, 0x1.264d25ca1d009p+382,
    0x1.6b473aa57bcccp+388, 0x1.c619094edabffp+394, 0x1.1f5bd7e3e66d7p+401, 0x1.702dac9bff3c4p+407,
    0x1.dd7b3bda4f022p+413, 0x1.3958df4743d96p+420, 0x1.a02a088aa61cbp+426, 0x1.179c3dbd279b5p+433,
    0x1.7c1863ed21d72p+439, 0x1.0550c4b30743ep+446, 0x1.6b645188f61a6p+452, 0x1.ff0512a89a152p+458,
    0x1.6b4d9b43dd8b0p+465, 0x1.051fc798c73bfp+472, 0x1.7b722e0a01831p+478, 0x1.16a7d9cf591c4p+485,
    0x1.9da1274fc845fp+491, 0x1.3638dd7bd6347p+498, 0x1.d62e2fafb0a78p+504, 0x1.67fb5c8283404p+511,
    0x1.166c698cf183bp+518, 0x1.b30964ec395dcp+524, 0x1.574569a265440p+531, 0x1.118b502d68b23p+538,
    0x1.b83c3509147ecp+544, 0x1.65b0eb1760a70p+551, 0x1.256b20d92d490p+558, 0x1.e5f96e67b300ep+564,
    0x1.963e824aafa2cp+571, 0x1.56c4bdef04315p+578, 0x1.23e389bd89920p+585, 0x1.f5af14bdc472fp+591,
    0x1.b30dd3fc905bap+598, 0x1.7cac197cfe503p+605, 0x1.500fee805882dp+612, 0x1.2b4e306a4ed48p+619,
    0x1.0ce83f7f82d2fp+626, 0x1.e764f3171d1e4p+632, 0x1.bd824633209dbp+639, 0x1.9ab418b722116p+646,
    0x1.7dd36efa41ac2p+653, 0x1.65f6380a9d916p+660, 0x1.5262c0fa08f37p+667, 0x1.42861fee50880p+674,
    0x1.35ece2af0162bp+681, 0x1.2c3d7b998957ap+688, 0x1.25340ab3f01f9p+695, 0x1.209f3a89205f1p+702,
};

__device__ __forceinline__ double inv_k(int k) { return c_inv_k[k]; }

// Store m_k of `node` (and its scaled traversal copy).
__device__ __forceinline__ void put_moment(const MomArgs &a, int64_t node, int k, double m)
{
    a.moments[node * (a.order + 1) + k] = m;
    if (a.meval) {
        a.meval[node * a.estride + k] = k == 0 ? m : __dmul_rn(m, c_fact_km1[k]);
        if (k == a.order && a.estride > a.order + 1)
            a.meval[node * a.estride + k + 1] = 0.0;
    }
}

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
        put_moment(a, node, lane, sum);
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
        put_moment(a, node, k, row_smem[k]);
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
            put_moment(a, node, k, out[i]);
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
                          double *moments, double *moments_eval, int64_t eval_stride,
                          void *stream)
{
    DT_CHECK_ARG(!moments_eval || (eval_stride >= order + 1 && eval_stride % 2 == 0),
                 "eval_stride must be even and >= order + 1");
    DT_CHECK_ARG(order >= 0 && order < MAX_ORDER1, "moment order must be in [0, 127]");
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta && moments,
                 "null pointer");
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, moments, moments_eval,
              eval_stride};
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
