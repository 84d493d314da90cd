// P2M of one leaf (tree.py:224-238 for the leaves):
// shared by the upward pass (dt_moments.cu) and the build, whose idle blocks
// form leaves of finished levels while block 0 runs the sparse deep levels
// (dt_build.cu).
#pragma once

#include "dt_common.cuh"
#include "dt_farcoef.cuh"

#ifndef DT_P2M_PREFETCH
#define DT_P2M_PREFETCH 1
#endif
#ifndef DT_P2M_G
#define DT_P2M_G 2
#endif

namespace {

struct P2mArgs {
    const double *xs, *qs, *center;
    const int64_t *start, *end;
    int64_t order;
    double *meval;   // traversal-layout rows M_k = c_k S_k, stride estride
    int64_t estride;
    double2 *xq;     // optional: the traversal's (x, q) pairs
};

// P2M of one leaf over G lanes: raw power sums S_k = sum q (x - c)^k for
// k < KMAX, with the powers split as t^(8m + r) = t^r (t^8)^m: per source 7
// products q t^r, t^8 and its powers, 8 additions and KMAX - 8 FMAs (44 FP64
// operations at KMAX = 32 instead of 64 for the running-product form).  Two
// sources per trip; then a butterfly over the G lanes.  Lane `sub` stores
// orders [sub KMAX/G, (sub + 1) KMAX/G) of the row (16-byte stores; orders
// >= order + 1 are the row's zero padding).
template <int G, int KMAX, bool COHERENT>
__device__ __forceinline__ void p2m_split_leaf(const P2mArgs &a, int64_t node, bool active,
                                               int sub)
{
    static_assert(KMAX % 8 == 0 && KMAX >= 8, "KMAX must be a multiple of 8");
    constexpr int NM = KMAX / 8;
    int64_t s = 0, e = 0;
    double c = 0.0;
    if (active) {
        // nodes written earlier in the same kernel (the build) are read
        // through L2 (ld.global.cg), never a stale L1 line
        s = COHERENT ? __ldcg(a.start + node) : __ldg(a.start + node);
        e = COHERENT ? __ldcg(a.end + node) : __ldg(a.end + node);
        c = COHERENT ? __ldcg(a.center + node) : __ldg(a.center + node);
    }
    double acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
        acc[k] = 0.0;
    int64_t j = s + sub;
#if DT_P2M_PREFETCH
    // the next pair's loads are issued before this pair's arithmetic
    bool have = j + G < e;
    double cx0 = 0.0, cx1 = 0.0, cq0 = 0.0, cq1 = 0.0;
    if (have) {
        cx0 = __ldg(a.xs + j);
        cx1 = __ldg(a.xs + j + G);
        cq0 = __ldg(a.qs + j);
        cq1 = __ldg(a.qs + j + G);
    }
    while (have) {
        const int64_t jn = j + 2 * G;
        const bool hn = jn + G < e;
        double nx0 = 0.0, nx1 = 0.0, nq0 = 0.0, nq1 = 0.0;
        if (hn) {
            nx0 = __ldg(a.xs + jn);
            nx1 = __ldg(a.xs + jn + G);
            nq0 = __ldg(a.qs + jn);
            nq1 = __ldg(a.qs + jn + G);
        }
        if (a.xq) {  // the traversal's interleaved (x, q), every source written once
            a.xq[j] = make_double2(cx0, cq0);
            a.xq[j + G] = make_double2(cx1, cq1);
        }
        const double t0 = cx0 - c, t1 = cx1 - c;
        double p0[8], p1[8];
        p0[0] = cq0;
        p1[0] = cq1;
        cx0 = nx0;
        cx1 = nx1;
        cq0 = nq0;
        cq1 = nq1;
        j = jn;
        have = hn;
#else
    for (; j + G < e; j += 2 * G) {
        const double x0 = __ldg(a.xs + j), x1 = __ldg(a.xs + j + G);
        const double t0 = x0 - c, t1 = x1 - c;
        double p0[8], p1[8];
        p0[0] = __ldg(a.qs + j);
        p1[0] = __ldg(a.qs + j + G);
        if (a.xq) {
            a.xq[j] = make_double2(x0, p0[0]);
            a.xq[j + G] = make_double2(x1, p1[0]);
        }
#endif
#pragma unroll
        for (int r = 1; r < 8; ++r) {
            p0[r] = p0[r - 1] * t0;
            p1[r] = p1[r - 1] * t1;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
            acc[r] += p0[r] + p1[r];
        if (NM > 1) {
            const double u0 = t0 * t0, u1 = t1 * t1;
            const double v0 = u0 * u0, v1 = u1 * u1;
            const double w0 = v0 * v0, w1 = v1 * v1;  // t^8
            double b0 = w0, b1 = w1;
#pragma unroll
            for (int m = 1; m < NM; ++m) {
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    acc[8 * m + r] = __fma_rn(p1[r], b1, __fma_rn(p0[r], b0, acc[8 * m + r]));
                if (m + 1 < NM) {
                    b0 *= w0;
                    b1 *= w1;
                }
            }
        }
    }
    if (j < e) {
        const double x0 = __ldg(a.xs + j);
        const double t0 = x0 - c;
        double p0[8];
        p0[0] = __ldg(a.qs + j);
        if (a.xq)
            a.xq[j] = make_double2(x0, p0[0]);
#pragma unroll
        for (int r = 1; r < 8; ++r)
            p0[r] = p0[r - 1] * t0;
#pragma unroll
        for (int r = 0; r < 8; ++r)
            acc[r] += p0[r];
        if (NM > 1) {
            const double u0 = t0 * t0, v0 = u0 * u0, w0 = v0 * v0;
            double b0 = w0;
#pragma unroll
            for (int m = 1; m < NM; ++m) {
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    acc[8 * m + r] = __fma_rn(p0[r], b0, acc[8 * m + r]);
                if (m + 1 < NM)
                    b0 *= w0;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1)
            acc[k] += __shfl_xor_sync(DT_FULL, acc[k], o);
    }
    if (!active)
        return;
    const int o1 = (int)a.order + 1;
    double2 *row = reinterpret_cast<double2 *>(a.meval + node * a.estride);
    constexpr int PER = KMAX / G;
#pragma unroll
    for (int k = 0; k < KMAX; k += 2) {
        if (k / PER == sub && k < a.estride) {
            const double v0 = k < o1 ? (k == 0 ? acc[0] : __dmul_rn(acc[k], c_mev_s[k])) : 0.0;
            const double v1 = k + 1 < o1 ? __dmul_rn(acc[k + 1], c_mev_s[k + 1]) : 0.0;
            row[k >> 1] = make_double2(v0, v1);
        }
    }
}

// Arrival on a node's counter with acquire-release semantics at GPU scope:
// the release publishes the rows this warp wrote (ordered before it by a
// __syncwarp), the acquire makes the rows behind earlier arrivals visible to
// the lane that completes the node (and, after a __syncwarp, to its warp).
__device__ __forceinline__ int arrive_acq_rel(int32_t *p)
{
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}


}  // namespace
