// (c) Upward pass: P2M at the leaves, M2M (binomial shift) bottom-up.
//
// Reference: tree.py:224-238 computes every node's moments
//     m_k = sum_j q_j (x_j - c)^k / k!,   k = 0..order,
// directly from its own sources, level by level (O(depth * N * order)).
// Here each leaf is formed from its sources and each internal node is the
// sum of its children shifted to its center,
//     m_k(parent) = sum_{j<=k} m_j(child) * delta^(k-j) / (k-j)!,
//     delta = c_child - c_parent,
// computed on raw power sums S_k = k! m_k, where the shift is the binomial
// transform S'_k = sum_j C(k,j) delta^(k-j) S_j, applied in place as 31
// passes of Pascal's rule S_k += delta S_(k-1).
//   order + 1 <= 32: P2M with 2 lanes per leaf (p2m_group_kernel), then a
//     barrier-free dataflow (m2m_flow_kernel): every leaf bumps its parent's
//     arrival counter; the lane whose arrival completes a parent keeps it,
//     and the warp forms four kept parents at a time (8 lanes each, 4 orders
//     per lane) before those lanes climb on.  The shard plan (multi-GPU) restricts
//     both to one rank's subtrees; shard_finish_kernel forms the levels above
//     the cut with the same arithmetic, thread per node.
//   higher orders: warp per leaf + the same dataflow with a Toeplitz shift.
// The shift is exact algebra; round-off differs from the reference's direct
// sums at the 1e-16 level of sum|q| r^k / k!.
// Algorithmic HBM bytes: P2M 16 N + 8 (order+1) leaves; M2M 24 (order+1)
// per internal node (two child rows read, one row written).

#include "dt_common.cuh"
#include "dt_farcoef.cuh"

#ifndef DT_P2M_G
#define DT_P2M_G 2
#endif

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

__constant__ double c_inv_fact[MAX_ORDER1] = {  // 1/k! rounded
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26,
    0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41,
    0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53, 0x1.2f49b46814157p-57,
    0x1.e542ba4020225p-62, 0x1.71b8ef6dcf572p-66, 0x1.0ce396db7f853p-70, 0x1.761b413163819p-75,
    0x1.f2cf01972f578p-80, 0x1.3f3ccdd165fa9p-84, 0x1.88e85fc6a4e59p-89, 0x1.d1ab1c2dccea3p-94,
    0x1.0a18a2635085dp-98, 0x1.259f98b4358aep-103, 0x1.3932c5047d60ep-108, 0x1.434d2e783f5bdp-113,
    0x1.434d2e783f5bdp-118, 0x1.3981254dd0d52p-123, 0x1.2710231c0fd7ap-128, 0x1.0dc59c716d91fp-133,
    0x1.df983290c2ca8p-139, 0x1.9ec8d1c94e85bp-144, 0x1.5d4acb9c0c3abp-149, 0x1.1e99449a4bacep-154,
    0x1.ca8ed42a12ae4p-160, 0x1.65e61c39d0241p-165, 0x1.10af527530de8p-170, 0x1.95db45257e512p-176,
    0x1.272b1b03fec6ap-181, 0x1.a3cb872220648p-187, 0x1.240804f659510p-192, 0x1.8da8e0a127ebap-198,
    0x1.091b406b6ff27p-203, 0x1.5a42f0dfeb086p-209, 0x1.bb36f6e12cd79p-215, 0x1.161872bf7b824p-220,
    0x1.56457989358c9p-226, 0x1.9d4f1058674dfp-232, 0x1.e9d8f6ed83eaap-238, 0x1.1d008faac5c50p-243,
    0x1.45b77f9e98e12p-249, 0x1.6db793c887b97p-255, 0x1.938cc661b03f6p-261, 0x1.b5bfc17fa97d2p-267,
    0x1.d2eeac43e7fd0p-273, 0x1.e9e56d649f768p-279, 0x1.f9b3059128bc6p-285, 0x1.00dcf6a320e1cp-290,
    0x1.00dcf6a320e1cp-296, 0x1.f9d2a2bb5471ap-303, 0x1.ea7ead50ce01ap-309, 0x1.d48849da8f4a3p-315,
    0x1.b8f8bdfae136cp-321, 0x1.99046602abcafp-327, 0x1.75f56494ba531p-333, 0x1.5116e3adb9fb9p-339,
    0x1.2ba2917dfaa6cp-345, 0x1.06b1981a48762p-351, 0x1.c6639f500ea2dp-358, 0x1.83bed30a49edep-364,
    0x1.4685bf3115d5dp-370, 0x1.0f653132c5ae6p-376, 0x1.bd5dda94f5a18p-383, 0x1.68cda75b82f10p-389,
    0x1.20a485e2cf273p-395, 0x1.c8206e6fe560cp-402, 0x1.64005631debbep-408, 0x1.1281cd42368abp-414,
    0x1.a24be3711628bp-421, 0x1.3af3de7343e27p-427, 0x1.d4c44522a0927p-434, 0x1.58d700d5cb749p-440,
    0x1.f595d2ab567b0p-447, 0x1.68b0c583d6a34p-453, 0x1.007db446ff080p-459, 0x1.68c751f8f632ap-466,
    0x1.f5f3ec7bc5d71p-473, 0x1.596e0e189e2b7p-479, 0x1.d65f64e59b771p-486, 0x1.3ce1f3216b6dep-492,
    0x1.a6829981e4928p-499, 0x1.16c503a23d142p-505, 0x1.6c1b7275dcd65p-512, 0x1.d6c3cf76c59b9p-519,
    0x1.2d4a1e607e781p-525, 0x1.7dd50faf84657p-532, 0x1.df297d187dfcdp-539, 0x1.29bb552f8772dp-545,
    0x1.6e7068d8092aep-552, 0x1.beb4eb15fc8c0p-559, 0x1.0db5afbffdea5p-565, 0x1.42a4b5885d34fp-572,
    0x1.7e64655f3f0f6p-579, 0x1.c10c3547ec1b7p-586, 0x1.05439cac2c47dp-592, 0x1.2d470c4e9d270p-599,
    0x1.585132a2fcbeep-606, 0x1.8605e345153bep-613, 0x1.b5eba9d8cb7dap-620, 0x1.e76cb424808bcp-627,
    0x1.0cec86b309210p-633, 0x1.263516a53c4fep-640, 0x1.3f23e47f2bba7p-647, 0x1.5746e043f2ccep-654,
    0x1.6e2977bff1eb9p-661, 0x1.83584be68daaep-668, 0x1.9665084a05f25p-675, 0x1.a6ea2e16eb21ap-682,
    0x1.b48ea3306e964p-689, 0x1.bf08d841fa750p-696, 0x1.c6215db8ddeccp-703, 0x1.c9b4c7476cc65p-710,
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

// Store from the raw power sum S_k = sum_j q_j (x_j - c)^k:
// m_k = S_k / k!, traversal copy M_k = gamma_(k-1) S_k / k (dt_farcoef.cuh).
__device__ __forceinline__ void put_raw_sum(const MomArgs &a, int64_t node, int k, double S)
{
    a.moments[node * (a.order + 1) + k] = __dmul_rn(S, c_inv_fact[k]);
    if (a.meval) {
        a.meval[node * a.estride + k] = k == 0 ? S : __dmul_rn(S, c_mev_s[k]);
        if (k == a.order && a.estride > a.order + 1)
            a.meval[node * a.estride + k + 1] = 0.0;
    }
}

// P2M for one leaf, order + 1 <= 32, one warp: raw power sums in two
// halves of 16 orders (2 FP64 ops per source and order), smem transpose-
// reduce over the 32 lanes.
__device__ void p2m_leaf_reg(const MomArgs &a, int64_t node, int64_t s, int64_t e, double c,
                             double (*tr)[33])
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    for (int base = 0; base < o1; base += 16) {
        double acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
            acc[k] = 0.0;
        for (int64_t j = s + lane; j < e; j += 32) {
            const double t = __ldg(a.xs + j) - c;
            double w = __ldg(a.qs + j);
            if (base) {
                const double t2 = t * t, t4 = t2 * t2, t8 = t4 * t4;
                w *= t8 * t8;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                acc[k] += w;
                w *= t;
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            tr[k][lane] = acc[k];
        __syncwarp();
        if (lane < 16 && base + lane < o1) {
            double sum = 0.0;
#pragma unroll 8
            for (int l = 0; l < 32; ++l)
                sum += tr[lane][l];
            put_raw_sum(a, node, base + lane, sum);
        }
        __syncwarp();
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
    const int64_t n = __ldg(a.meta + DT_META_NODES);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        a.arrived[i] = 0;
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
    __shared__ double tr[MOM_WARPS][16][33];
    __shared__ double pw_s[MOM_WARPS][MAX_ORDER1];
    __shared__ double row_s[MOM_WARPS][MAX_ORDER1];
    const int warp = threadIdx.x >> 5, lane = dt_lane();
    const int64_t gwarp = (int64_t)blockIdx.x * MOM_WARPS + warp;
    const int64_t nwarps = (int64_t)gridDim.x * MOM_WARPS;
    const int64_t n_nodes = __ldg(a.meta + DT_META_NODES);
    const bool reg_path = a.order + 1 <= REG_ORDER;

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
            if (reg_path)
                p2m_leaf_reg(a, node, ns, ne, nc, tr[warp]);
            else
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

// ---- order + 1 <= 32: G lanes per leaf (P2M), dataflow M2M (in-place Pascal) ----

// P2M with G consecutive lanes per leaf: each lane sums every G-th source of
// the leaf (the group's loads cover contiguous sectors), four sources in
// flight, then a butterfly over the G lanes.  Leaves are gathered per warp
// from 32 consecutive node slots (ballot) so no group idles on internal
// nodes.  Raw power sums S_k = sum q (x - c)^k in registers.
// KMAX: orders computed, a multiple of 8 >= order + 1, fixed at compile time
// so the order loop has no per-step guard (a uniform branch per order step
// costs 25% of the instructions and splits the scheduling window).
template <int G, int KMAX>
__global__ void __launch_bounds__(256) p2m_group_kernel(MomArgs a)
{
    const int lane = dt_lane();
    const int sub = lane & (G - 1), grp = lane / G;
    const int64_t n = __ldg(a.meta + DT_META_NODES);
    const int o1 = (int)a.order + 1;
    int64_t cut_begin = INT64_MAX, lo = 0, hi = 0;
    if (a.plan) {
        cut_begin = __ldg(a.plan + DT_PLAN_LEVEL_BEGIN);
        lo = __ldg(a.plan + DT_PLAN_SRC_LO);
        hi = __ldg(a.plan + DT_PLAN_SRC_HI);
    }
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t c0 = gwarp * 32; c0 < n; c0 += nwarps * 32) {
        const int64_t mine = c0 + lane;
        bool leaf = false;
        if (mine < n) {
            const int64_t l = __ldg(a.left + mine), r = __ldg(a.right + mine);
            if (a.parent) {  // dataflow M2M bookkeeping (m2m_flow_kernel)
                a.arrived[mine] = 0;
                if (l >= 0)
                    a.parent[l] = (int32_t)mine;
                if (r >= 0)
                    a.parent[r] = (int32_t)mine;
                if (mine == 0)
                    a.parent[0] = -1;
            }
            leaf = l < 0 && r < 0;
            if (leaf && mine >= cut_begin)
                leaf = __ldg(a.start + mine) >= lo && __ldg(a.end + mine) <= hi;
        }
        unsigned leaves = __ballot_sync(DT_FULL, leaf);
        while (leaves) {
            // group grp takes the grp-th remaining leaf
            unsigned m = leaves;
            for (int i = 0; i < grp && m; ++i)
                m &= m - 1;
            const bool active = m != 0;
            const int64_t node = c0 + (active ? __ffs(m) - 1 : 0);
            for (int i = 0; i < 32 / G && leaves; ++i)
                leaves &= leaves - 1;
            int64_t s = 0, e = 0;
            double c = 0.0;
            if (active) {
                s = __ldg(a.start + node);
                e = __ldg(a.end + node);
                c = __ldg(a.center + node);
            }
            double acc[KMAX];
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
                acc[k] = 0.0;
            int64_t j = s + sub;
            for (; j + 3 * G < e; j += 4 * G) {
                const double t0 = __ldg(a.xs + j) - c, t1 = __ldg(a.xs + j + G) - c;
                const double t2 = __ldg(a.xs + j + 2 * G) - c, t3 = __ldg(a.xs + j + 3 * G) - c;
                double w0 = __ldg(a.qs + j), w1 = __ldg(a.qs + j + G);
                double w2 = __ldg(a.qs + j + 2 * G), w3 = __ldg(a.qs + j + 3 * G);
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    acc[k] += (w0 + w1) + (w2 + w3);
                    w0 *= t0;
                    w1 *= t1;
                    w2 *= t2;
                    w3 *= t3;
                }
            }
            for (; j < e; j += G) {
                const double t0 = __ldg(a.xs + j) - c;
                double w0 = __ldg(a.qs + j);
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    acc[k] += w0;
                    w0 *= t0;
                }
            }
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1)
                    acc[k] += __shfl_xor_sync(DT_FULL, acc[k], o);
            }
            if (active) {
#pragma unroll
                for (int k = 0; k < KMAX; ++k)
                    if ((k & (G - 1)) == sub && k < o1)
                        put_raw_sum(a, node, k, acc[k]);
            }
        }
    }
}

// Form internal node P from its children, one warp, lane k = order k, on
// raw power sums S_k = k! m_k: the binomial shift S'_k = sum_j C(k, j)
// delta^(k-j) S_j is applied in place as 31 passes of S_k += delta S_(k-1)
// (Pascal's rule; the previous pass's S_(k-1) comes from lane k-1).  Both
// children run in the same passes.  Same arithmetic, term for term, as the
// thread-per-node form m2m_level_threads (skipped orders take a zero shift).
__device__ __forceinline__ void m2m_form_warp(const MomArgs &a, int64_t P)
{
    const int lane = dt_lane();
    const int o1 = (int)a.order + 1;
    const int64_t l = __ldg(a.left + P), r = __ldg(a.right + P);
    const double c = __ldg(a.center + P);
    const double dl = l >= 0 ? __ldg(a.center + l) - c : 0.0;
    const double dr = r >= 0 ? __ldg(a.center + r) - c : 0.0;
    const double fk = c_fact_km1[lane + 1];
    double Sl = (l >= 0 && lane < o1) ? __dmul_rn(__ldcg(a.moments + l * o1 + lane), fk) : 0.0;
    double Sr = (r >= 0 && lane < o1) ? __dmul_rn(__ldcg(a.moments + r * o1 + lane), fk) : 0.0;
#pragma unroll
    for (int i = 1; i < REG_ORDER; ++i) {
        const double tl = __shfl_up_sync(DT_FULL, Sl, 1);
        const double tr = __shfl_up_sync(DT_FULL, Sr, 1);
        // orders below i take a zero shift (in place, as m2m_form_group8)
        const bool on = lane >= i;
        Sl = __fma_rn(on ? dl : 0.0, tl, Sl);
        Sr = __fma_rn(on ? dr : 0.0, tr, Sr);
    }
    double out = 0.0;
    if (l >= 0)
        out += Sl;
    if (r >= 0)
        out += Sr;
    if (lane < o1)
        put_raw_sum(a, P, lane, out);
}

// Four parents per warp at once: lanes [8g, 8g + 8) form parent P (of group
// g), lane l of a group holding orders 4l .. 4l + 3 of both children.  A
// Pascal pass then needs one neighbour value per lane (the last order of
// lane l - 1), so a parent costs 8x fewer shuffles than with one order per
// lane.  Same arithmetic, term for term, as m2m_form_warp / the thread form
// (orders a pass skips take a zero shift, fma(0, x, S) = S: equal values, a
// zero's sign aside).
__device__ __forceinline__ void m2m_form_group8(const MomArgs &a, int64_t P)
{
    const int gl = dt_lane() & 7;  // lane within the group
    const int o1 = (int)a.order + 1;
    int64_t l = -1, r = -1;
    double dl = 0.0, dr = 0.0;
    double Sl[4], Sr[4];
    if (P >= 0) {
        l = __ldg(a.left + P);
        r = __ldg(a.right + P);
        const double c = __ldg(a.center + P);
        if (l >= 0)
            dl = __ldg(a.center + l) - c;
        if (r >= 0)
            dr = __ldg(a.center + r) - c;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int k = 4 * gl + u;
        const double fk = c_fact_km1[k + 1];
        Sl[u] = (l >= 0 && k < o1) ? __dmul_rn(__ldcg(a.moments + l * o1 + k), fk) : 0.0;
        Sr[u] = (r >= 0 && k < o1) ? __dmul_rn(__ldcg(a.moments + r * o1 + k), fk) : 0.0;
    }
    const unsigned mask = DT_FULL;
#pragma unroll
    for (int i = 1; i < REG_ORDER; ++i) {
        const double nl = __shfl_up_sync(mask, Sl[3], 1, 8);
        const double nr = __shfl_up_sync(mask, Sr[3], 1, 8);
        // descending within the lane: every update reads the previous pass
#pragma unroll
        for (int u = 3; u >= 0; --u) {
            // orders k = 4 gl + u < i sit this pass out: their shift is 0,
            // and fma(0, x, S) = S (up to the sign of a zero S), which keeps
            // every update in place; gl >= ceil((i - u) / 4) takes at most
            // two values per pass
            const bool on = gl >= ((i - u + 3) >> 2);
            const double el = on ? dl : 0.0, er = on ? dr : 0.0;
            Sl[u] = __fma_rn(el, u ? Sl[u - 1] : nl, Sl[u]);
            Sr[u] = __fma_rn(er, u ? Sr[u - 1] : nr, Sr[u]);
        }
    }
    if (P < 0)
        return;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int k = 4 * gl + u;
        double out = 0.0;
        if (l >= 0)
            out += Sl[u];
        if (r >= 0)
            out += Sr[u];
        if (k < o1)
            put_raw_sum(a, P, k, out);
    }
}

// Arrival on a node's counter with acquire-release semantics at GPU scope:
// the release publishes the rows this warp formed (ordered before it by a
// __syncwarp), the acquire makes the rows behind earlier arrivals visible to
// the lane that completes the node (and, after a __syncwarp, to its group).
// One MEMBAR.ALL.GPU per round instead of two MEMBAR.SC.GPU fences.
__device__ __forceinline__ int arrive_acq_rel(int32_t *p)
{
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}

// A leaf's arrival: its row comes from the P2M launch (ordered by the kernel
// boundary), so only the acquire is needed.
__device__ __forceinline__ int arrive_acquire(int32_t *p)
{
    int old;
    asm volatile("atom.add.acquire.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}

// Upward pass without grid barriers (after the P2M kernel, which also wrote
// parent[] and zeroed arrived[]): every leaf bumps its parent's arrival
// counter; the warp whose arrival completes a parent forms it and keeps
// climbing while it completes the next ancestor.  With a shard plan the
// climb stops below the cut level and covers the plan's subtrees only.
#ifndef DT_M2M_MINB
#define DT_M2M_MINB 4  // 64 registers: 4 blocks per SM (3: 0.43 ms, 5: 0.42 ms, 4: 0.39 ms)
#endif
__global__ void __launch_bounds__(256, DT_M2M_MINB) m2m_flow_kernel(MomArgs a)
{
    const int lane = dt_lane();
    const int64_t n = __ldg(a.meta + DT_META_NODES);
    int64_t cut_begin = 0, lo = 0, hi = 0;
    if (a.plan) {
        cut_begin = __ldg(a.plan + DT_PLAN_LEVEL_BEGIN);
        lo = __ldg(a.plan + DT_PLAN_SRC_LO);
        hi = __ldg(a.plan + DT_PLAN_SRC_HI);
    }
    const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int CH = 32;  // nodes scanned per warp step
    for (int64_t r0 = gwarp * CH; r0 < n; r0 += nwarps * CH) {
        // deepest levels first: their chains are the critical path
        const int64_t c0 = n - CH - r0;  // may be negative for the last chunk
        const int64_t mine = c0 + lane;
        bool done = false;
        int64_t par = -1;
        if (lane < CH && mine >= 0 && mine < n && __ldg(a.left + mine) < 0 &&
            __ldg(a.right + mine) < 0) {
            par = __ldcg(a.parent + mine);
            bool in = par >= cut_begin;
            if (in && a.plan)
                in = __ldg(a.start + mine) >= lo && __ldg(a.end + mine) <= hi;
            if (in) {
                const int need = (__ldg(a.left + par) >= 0) + (__ldg(a.right + par) >= 0);
                done = arrive_acquire(a.arrived + par) == need - 1;
            }
        }
        // lanes hold the parents they completed; four of them are formed at a
        // time (one per 8-lane group), then each of those lanes arrives at its
        // own grandparent and keeps it if the arrival completes it
        if (!done)
            par = -1;
        while (true) {
            const unsigned todo = __ballot_sync(DT_FULL, par >= 0);
            if (!todo)
                break;
            if (__popc(todo) == 1) {
                // a lone parent (the usual case high in a chain): all 32
                // lanes, one order each, a third of the group form's work
                const int src = __ffs(todo) - 1;
                __syncwarp();
                m2m_form_warp(a, __shfl_sync(DT_FULL, par, src));
                __syncwarp();
                if (lane == src) {
                    const int64_t q = __ldcg(a.parent + par);
                    int64_t nxt = -1;
                    if (q >= cut_begin && q >= 0) {
                        const int need = (__ldg(a.left + q) >= 0) + (__ldg(a.right + q) >= 0);
                        if (arrive_acq_rel(a.arrived + q) == need - 1)
                            nxt = q;
                    }
                    par = nxt;
                }
                continue;
            }
            unsigned sel = 0, t = todo;
            int64_t mine_p = -1;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                int64_t pg = -1;
                if (t) {
                    const int src = __ffs(t) - 1;
                    t &= t - 1;
                    sel |= 1u << src;
                    pg = __shfl_sync(DT_FULL, par, src);
                }
                if ((lane >> 3) == g)
                    mine_p = pg;
            }
            __syncwarp();  // the completing lanes' acquires precede the group's loads
            m2m_form_group8(a, mine_p);
            __syncwarp();  // the group's stores precede the releasing arrivals
            if ((sel >> lane) & 1u) {
                const int64_t q = __ldcg(a.parent + par);
                int64_t nxt = -1;
                if (q >= cut_begin && q >= 0) {
                    const int need = (__ldg(a.left + q) >= 0) + (__ldg(a.right + q) >= 0);
                    if (arrive_acq_rel(a.arrived + q) == need - 1)
                        nxt = q;
                }
                par = nxt;
            }
        }
    }
}

// M2M of one level with one thread per internal node, on raw power sums:
// S'_k = sum_j C(k, j) delta^(k-j) S_j (the binomial transform) computed in
// place by k passes of S_k += delta S_(k-1) over descending k (Pascal's
// rule), so a child row needs only its own 32 registers.
__device__ __forceinline__ void m2m_level_threads(const MomArgs &a, int64_t f0, int64_t f1,
                                                  int64_t tid, int64_t nthreads, bool filter,
                                                  int64_t src_lo, int64_t src_hi)
{
    const int o1 = (int)a.order + 1;
    for (int64_t node = f0 + tid; node < f1; node += nthreads) {
        const int64_t l = __ldg(a.left + node), r = __ldg(a.right + node);
        if (l < 0 && r < 0)
            continue;
        if (filter && (__ldg(a.start + node) < src_lo || __ldg(a.end + node) > src_hi))
            continue;
        const double c = __ldg(a.center + node);
        double out[REG_ORDER];
#pragma unroll
        for (int k = 0; k < REG_ORDER; ++k)
            out[k] = 0.0;
#pragma unroll 1
        for (int ci = 0; ci < 2; ++ci) {
            const int64_t ch = ci == 0 ? l : r;
            if (ch < 0)
                continue;
            const double delta = __ldg(a.center + ch) - c;
            const double *row = a.moments + ch * o1;
            // L2-coherent loads (the row was formed earlier in this kernel),
            // all issued before the first use
            double S[REG_ORDER];
#pragma unroll
            for (int k = 0; k < REG_ORDER; ++k)
                S[k] = k < o1 ? __ldcg(row + k) : 0.0;
#pragma unroll
            for (int k = 0; k < REG_ORDER; ++k)
                S[k] = __dmul_rn(S[k], c_fact_km1[k + 1]);
#pragma unroll
            for (int i = 1; i < REG_ORDER; ++i) {
#pragma unroll
                for (int k = REG_ORDER - 1; k >= i; --k)
                    S[k] = __fma_rn(delta, S[k - 1], S[k]);
            }
#pragma unroll
            for (int k = 0; k < REG_ORDER; ++k)
                out[k] += S[k];
        }
#pragma unroll
        for (int k = 0; k < REG_ORDER; ++k)
            if (k < o1)
                put_raw_sum(a, node, k, out[k]);
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

__global__ void shard_pack_kernel(const int64_t *plan, int rank, int64_t o1, const double *moments,
                                  const double *meval, int64_t es, double *send)
{
    const int64_t a0 = __ldg(plan + DT_PLAN_OWNER0 + rank);
    const int64_t rows = __ldg(plan + DT_PLAN_OWNER0 + rank + 1) - a0;
    const int64_t w = o1 + es;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * w;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / w, k = i - row * w;
        send[i] = k < o1 ? __ldg(moments + (a0 + row) * o1 + k)
                         : __ldg(meval + (a0 + row) * es + (k - o1));
    }
}

// One block: scatter every owner's level-l rows, then M2M levels cut-1 .. 0
// (thread per node; the same arithmetic as m2m_form_warp, so the rows match
// the single-GPU pass bit for bit).
__global__ void __launch_bounds__(256) shard_finish_kernel(MomArgs a, int world, int64_t slot_rows,
                                                           const double *recv)
{
    const int64_t o1 = a.order + 1, es = a.meval ? a.estride : 0, w = o1 + es;
    for (int r = 0; r < world; ++r) {
        const int64_t a0 = __ldg(a.plan + DT_PLAN_OWNER0 + r);
        const int64_t rows = __ldg(a.plan + DT_PLAN_OWNER0 + r + 1) - a0;
        const double *slot = recv + (int64_t)r * slot_rows * w;
        for (int64_t i = threadIdx.x; i < rows * w; i += blockDim.x) {
            const int64_t row = i / w, k = i - row * w;
            if (k < o1)
                a.moments[(a0 + row) * o1 + k] = slot[i];
            else
                a.meval[(a0 + row) * es + (k - o1)] = slot[i];
        }
    }
    __syncthreads();
    const int64_t cut = __ldg(a.plan + DT_PLAN_CUT);
    for (int64_t lev = cut - 1; lev >= 0; --lev) {
        m2m_level_threads(a, __ldg(a.meta + DT_META_LEVEL0 + lev),
                          __ldg(a.meta + DT_META_LEVEL0 + lev + 1), threadIdx.x, blockDim.x,
                          false, 0, 0);
        __syncthreads();
    }
}

// Upward pass for order + 1 <= 32 (honouring a.plan): P2M, then the
// barrier-free M2M dataflow.  Level-synchronous M2M variants (grid barrier
// per level, one launch per level, narrow/wide phases) all measured slower
// on configs[2] (0.47-0.95 ms against 0.36 ms): a grid barrier costs ~5 us
// and the tree is 32 levels deep.
int launch_level_moments(MomArgs &a, cudaStream_t s)
{
    const int sms = dt_num_sms();
    if (!a.parent)
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace missing");
    const int64_t o1 = a.order + 1;
    if (o1 <= 8)
        p2m_group_kernel<DT_P2M_G, 8><<<sms * 8, 256, 0, s>>>(a);
    else if (o1 <= 16)
        p2m_group_kernel<DT_P2M_G, 16><<<sms * 8, 256, 0, s>>>(a);
    else if (o1 <= 24)
        p2m_group_kernel<DT_P2M_G, 24><<<sms * 8, 256, 0, s>>>(a);
    else
        p2m_group_kernel<DT_P2M_G, 32><<<sms * 8, 256, 0, s>>>(a);
    DT_CUDA_TRY(cudaGetLastError());
    m2m_flow_kernel<<<sms * 8, 256, 0, s>>>(a);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

}  // namespace

extern "C" size_t dt_moments_workspace(int64_t node_capacity)
{
    return (size_t)node_capacity * 2 * sizeof(int32_t) + 256;
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
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta && moments,
                 "null pointer");
    if (!workspace || workspace_bytes < dt_moments_workspace(node_capacity))
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace too small");
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, moments, moments_eval,
              eval_stride, (int32_t *)workspace, (int32_t *)workspace + node_capacity, nullptr};
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

extern "C" size_t dt_shard_rows_bytes(int64_t cut_level, int64_t order, int64_t eval_stride)
{
    if (cut_level < 0 || cut_level > 20 || order < 0 || eval_stride < 0)
        return 0;
    return ((size_t)1 << cut_level) * (size_t)(order + 1 + eval_stride) * sizeof(double);
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
    DT_CHECK_ARG(xs && qs && center && start && end && left && right && meta && plan && moments,
                 "null pointer");
    if (!workspace || workspace_bytes < dt_moments_workspace(node_capacity))
        return dt_set_error(DT_ERR_WORKSPACE, "moments workspace too small");
    MomArgs a{xs, qs, center, start, end, left, right, meta, order, moments, moments_eval,
              eval_stride, (int32_t *)workspace, (int32_t *)workspace + node_capacity, plan};
    return launch_level_moments(a, (cudaStream_t)stream);
}

extern "C" int dt_shard_pack(const int64_t *plan, int rank, int64_t cut_level, int64_t order,
                             const double *moments, const double *moments_eval,
                             int64_t eval_stride, double *send, void *stream)
{
    DT_CHECK_ARG(plan && moments && send, "null pointer");
    DT_CHECK_ARG(rank >= 0 && rank < DT_MAX_WORLD, "bad rank");
    DT_CHECK_ARG(cut_level >= 0 && cut_level <= 20 && order >= 0, "bad cut level / order");
    const int64_t es = moments_eval ? eval_stride : 0;
    DT_CHECK_ARG(!moments_eval || (eval_stride >= order + 1 && eval_stride % 2 == 0),
                 "eval_stride must be even and >= order + 1");
    const int64_t cells = ((int64_t)1 << cut_level) * (order + 1 + es);
    int blocks = (int)((cells + 255) / 256);
    blocks = blocks < 1 ? 1 : (blocks > 4 * dt_num_sms() ? 4 * dt_num_sms() : blocks);
    shard_pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(plan, rank, order + 1, moments,
                                                               moments_eval, es, send);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_shard_finish(const int64_t *plan, int world, int64_t cut_level,
                               const double *recv, const double *center, const int64_t *left,
                               const int64_t *right, const int64_t *meta, int64_t order,
                               double *moments, double *moments_eval, int64_t eval_stride,
                               void *stream)
{
    DT_CHECK_ARG(plan && recv && center && left && right && meta && moments, "null pointer");
    DT_CHECK_ARG(world >= 1 && world <= DT_MAX_WORLD, "bad world size");
    DT_CHECK_ARG(cut_level >= 0 && cut_level <= 20, "bad cut level");
    DT_CHECK_ARG(order >= 0 && order + 1 <= REG_ORDER, "sharded moments need order <= 31");
    DT_CHECK_ARG(!moments_eval || (eval_stride >= order + 1 && eval_stride % 2 == 0),
                 "eval_stride must be even and >= order + 1");
    // start/end are only read by the range filter, which is open here
    MomArgs a{nullptr, nullptr, center, nullptr, nullptr, left, right, meta, order, moments,
              moments_eval, eval_stride, nullptr, nullptr, plan};
    shard_finish_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(a, world, (int64_t)1 << cut_level,
                                                             recv);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}
