// Shared device helpers for the disctree B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/disctree_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "disctree_b200 is built for sm_100a only"
#endif

#define DT_WARP 32
#define DT_FULL 0xffffffffu

// Host-side status plumbing -------------------------------------------------
int dt_set_error(int code, const char *msg);
#define DT_CUDA_TRY(expr)                                        \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess)                                   \
            return dt_set_error(DT_ERR_CUDA, cudaGetErrorString(_e)); \
    } while (0)
#define DT_CHECK_ARG(cond, msg)                                  \
    do {                                                         \
        if (!(cond))                                             \
            return dt_set_error(DT_ERR_INVALID, msg);            \
    } while (0)

// Tree metadata block written by the build kernel (int64, device memory).
// Layout mirrors include/disctree_b200.h DT_META_*.
static_assert(DT_META_LEVEL0 + DT_MAX_LEVELS + 1 <= DT_META_WORDS, "meta layout");

// Packed node record consumed by the traversal kernel: one 32-byte sector.
// The children are stored in visit order: `first` is the left child if there
// is one, else the right one (-1: leaf); `second` is the right child when
// both exist (the one the walk defers), else -1.
struct __align__(16) dt_node {
    double center;
    double half;
    int32_t first;
    int32_t second;
    int32_t start;
    int32_t end;
};
static_assert(sizeof(dt_node) == 32, "dt_node must be one sector");

__device__ __forceinline__ void dt_node_children(dt_node &nd, int64_t left, int64_t right)
{
    nd.first = (int32_t)(left >= 0 ? left : right);
    nd.second = (int32_t)(left >= 0 && right >= 0 ? right : -1);
}

// Fast fp64 reciprocal square root: MUFU seed + one cubic Newton step.
// Inputs are finite and > 0 on every call site (s = d^2 + r_d^2, r_d > 0).
__device__ __forceinline__ double dt_rsqrt(double s)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
    double t = s * y;
    double e = __fma_rn(-t, y, 1.0);
    double p = __fma_rn(0.375, e, 0.5);
    double ye = y * e;
    return __fma_rn(ye, p, y);
}

// Fast fp64 reciprocal: MUFU seed + two Newton steps (finite, nonzero input).
__device__ __forceinline__ double dt_rcp(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = __fma_rn(-x, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-x, r, 1.0);
    return __fma_rn(r, e, r);
}

// one 256-bit read-only load (LDG.E.ENL2.256); p must be 32-byte aligned
__device__ __forceinline__ double4 dt_ldg256(const void *p)
{
    double4 r;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ int dt_lane() { return threadIdx.x & (DT_WARP - 1); }

__device__ __forceinline__ unsigned dt_smid()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ double dt_shfl(double v, int src)
{
    return __shfl_sync(DT_FULL, v, src);
}

__device__ __forceinline__ double dt_warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(DT_FULL, v, o);
    return v;
}

// first index i in [lo, hi) with xs[i] >= v (np.searchsorted side='left')
__device__ __forceinline__ int64_t dt_lower_bound(const double *__restrict__ xs, int64_t lo,
                                                  int64_t hi, double v)
{
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(xs + mid) < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

static inline int dt_num_sms()
{
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0)
            sms = 148;
    }
    return sms;
}
