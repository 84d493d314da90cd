// (f) Brute-force O(N*T) direct sum: accuracy oracle and FP64 roofline bench.
//
// Reference: _kernels.py:49-59 (phi_sum_plain), 145-160 (phi_sum_kahan),
// dispatched by evaluate_direct (direct.py:52-88).  The reference's
// pair-symmetric path (_kernels.py:62-142) exists to halve CPU work; on the
// GPU every target is independent, so targets == sources uses the plain
// kernel.
//   FP64   4 targets per thread in registers, sources staged through shared
//          memory in 512-pair tiles and read as broadcast 16-byte loads; per
//          pair 10 FP64-pipe instructions (d, s = fma(d,d,rd2), MUFU rsqrt
//          seed + cubic Newton (5), (q*d)*r, add).  The pair term is rounded
//          before it is accumulated, like the reference's q*d/sqrt(s), so
//          the term is odd in d and mirrored pairs cancel exactly.
//   FP32   bench variant: d formed from (hi, lo) float splits of x and y so
//          near pairs keep their precision, fp32 pair evaluation (MUFU
//          rsqrt), 32-pair fp32 partials promoted into an fp64 accumulator.
//   KAHAN  one target per thread, strictly ascending j, IEEE _rn operations
//          only: bit-identical to the numba kernel (no fastmath there).
#include "dt_common.cuh"

namespace {

constexpr int DIR_THREADS = 256;
constexpr int DIR_TPT = 4;  // targets per thread
constexpr int DIR_TILE = 512;

__global__ void __launch_bounds__(DIR_THREADS) direct_fp64_kernel(
    const double *__restrict__ xs, const double *__restrict__ qs, int64_t n,
    const double *__restrict__ ys, double rd2, double *__restrict__ out, int64_t i0, int64_t i1,
    int accumulate)
{
    __shared__ double2 tile[DIR_TILE];
    const int64_t base = i0 + (int64_t)blockIdx.x * (DIR_THREADS * DIR_TPT) + threadIdx.x;
    double y[DIR_TPT], acc[DIR_TPT];
#pragma unroll
    for (int t = 0; t < DIR_TPT; ++t) {
        int64_t i = base + t * DIR_THREADS;
        y[t] = i < i1 ? __ldg(ys + i) : 0.0;
        acc[t] = 0.0;
    }
    for (int64_t j0 = 0; j0 < n; j0 += DIR_TILE) {
        const int m = (int)min((int64_t)DIR_TILE, n - j0);
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += DIR_THREADS)
            tile[j] = make_double2(__ldg(xs + j0 + j), __ldg(qs + j0 + j));
        __syncthreads();
#pragma unroll 2
        for (int j = 0; j < m; ++j) {
            const double2 v = tile[j];
#pragma unroll
            for (int t = 0; t < DIR_TPT; ++t) {
                const double d = v.x - y[t];
                const double r = dt_rsqrt(__fma_rn(d, d, rd2));
                // term rounded before accumulation (as the reference's
                // q*d/sqrt(s)): mirrored pairs cancel exactly
                acc[t] = __dadd_rn(acc[t], __dmul_rn(__dmul_rn(v.y, d), r));
            }
        }
    }
#pragma unroll
    for (int t = 0; t < DIR_TPT; ++t) {
        int64_t i = base + t * DIR_THREADS;
        if (i < i1)
            out[i] = accumulate ? out[i] + acc[t] : acc[t];
    }
}

__global__ void __launch_bounds__(DIR_THREADS) direct_fp32_kernel(
    const double *__restrict__ xs, const double *__restrict__ qs, int64_t n,
    const double *__restrict__ ys, double rd2, double *__restrict__ out, int64_t i0, int64_t i1,
    int accumulate)
{
    __shared__ float4 tile[DIR_TILE];  // (x_hi, x_lo, q, 0)
    const int64_t base = i0 + (int64_t)blockIdx.x * (DIR_THREADS * DIR_TPT) + threadIdx.x;
    const float rd2f = (float)rd2;
    float yh[DIR_TPT], yl[DIR_TPT];
    double acc[DIR_TPT];
#pragma unroll
    for (int t = 0; t < DIR_TPT; ++t) {
        int64_t i = base + t * DIR_THREADS;
        double yv = i < i1 ? __ldg(ys + i) : 0.0;
        yh[t] = (float)yv;
        yl[t] = (float)(yv - (double)yh[t]);
        acc[t] = 0.0;
    }
    for (int64_t j0 = 0; j0 < n; j0 += DIR_TILE) {
        const int m = (int)min((int64_t)DIR_TILE, n - j0);
        __syncthreads();
        for (int j = threadIdx.x; j < DIR_TILE; j += DIR_THREADS) {
            if (j < m) {
                double xv = __ldg(xs + j0 + j);
                float xh = (float)xv;
                tile[j] = make_float4(xh, (float)(xv - (double)xh), (float)__ldg(qs + j0 + j), 0.f);
            } else {
                tile[j] = make_float4(0.f, 0.f, 0.f, 0.f);  // q = 0 pads the last tile
            }
        }
        __syncthreads();
        for (int jb = 0; jb < m; jb += 32) {
            float part[DIR_TPT];
#pragma unroll
            for (int t = 0; t < DIR_TPT; ++t)
                part[t] = 0.f;
#pragma unroll 8
            for (int j = jb; j < jb + 32; ++j) {
                const float4 v = tile[j];
#pragma unroll
                for (int t = 0; t < DIR_TPT; ++t) {
                    const float d = (v.x - yh[t]) + (v.y - yl[t]);
                    const float r = rsqrtf(fmaf(d, d, rd2f));
                    part[t] = fmaf(v.z * d, r, part[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < DIR_TPT; ++t)
                acc[t] += (double)part[t];
        }
    }
#pragma unroll
    for (int t = 0; t < DIR_TPT; ++t) {
        int64_t i = base + t * DIR_THREADS;
        if (i < i1)
            out[i] = accumulate ? out[i] + acc[t] : acc[t];
    }
}

__global__ void __launch_bounds__(DIR_THREADS) direct_kahan_kernel(
    const double *__restrict__ xs, const double *__restrict__ qs, int64_t n,
    const double *__restrict__ ys, double rd2, double *__restrict__ out, int64_t i0, int64_t i1,
    int accumulate)
{
    __shared__ double2 tile[DIR_TILE];
    const int64_t i = i0 + (int64_t)blockIdx.x * DIR_THREADS + threadIdx.x;
    const double y = i < i1 ? __ldg(ys + i) : 0.0;
    double acc = 0.0, comp = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += DIR_TILE) {
        const int m = (int)min((int64_t)DIR_TILE, n - j0);
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += DIR_THREADS)
            tile[j] = make_double2(__ldg(xs + j0 + j), __ldg(qs + j0 + j));
        __syncthreads();
        for (int j = 0; j < m; ++j) {
            const double2 v = tile[j];
            const double d = __dsub_rn(v.x, y);
            const double term =
                __ddiv_rn(__dmul_rn(v.y, d), __dsqrt_rn(__dadd_rn(__dmul_rn(d, d), rd2)));
            const double t = __dsub_rn(term, comp);
            const double s = __dadd_rn(acc, t);
            comp = __dsub_rn(__dsub_rn(s, acc), t);
            acc = s;
        }
    }
    if (i < i1)
        out[i] = accumulate ? __dadd_rn(out[i], acc) : acc;
}

}  // namespace

extern "C" int dt_phi_sum_direct(const double *xs, const double *qs, int64_t n, const double *ys,
                                 double rd2, double *out, int64_t i0, int64_t i1, int mode,
                                 int accumulate, void *stream)
{
    DT_CHECK_ARG(n >= 0 && i0 >= 0 && i1 >= i0, "bad size or range");
    DT_CHECK_ARG(rd2 > 0.0, "rd2 must be > 0");
    DT_CHECK_ARG(mode == DT_DIRECT_FP64 || mode == DT_DIRECT_FP32 || mode == DT_DIRECT_KAHAN,
                 "unknown direct mode");
    if (i1 == i0)
        return DT_OK;
    DT_CHECK_ARG(ys && out && (n == 0 || (xs && qs)), "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t T = i1 - i0;
    if (mode == DT_DIRECT_KAHAN) {
        direct_kahan_kernel<<<(unsigned)((T + DIR_THREADS - 1) / DIR_THREADS), DIR_THREADS, 0, s>>>(
            xs, qs, n, ys, rd2, out, i0, i1, accumulate);
    } else {
        const int64_t per_block = DIR_THREADS * DIR_TPT;
        const unsigned grid = (unsigned)((T + per_block - 1) / per_block);
        if (mode == DT_DIRECT_FP64)
            direct_fp64_kernel<<<grid, DIR_THREADS, 0, s>>>(xs, qs, n, ys, rd2, out, i0, i1,
                                                            accumulate);
        else
            direct_fp32_kernel<<<grid, DIR_THREADS, 0, s>>>(xs, qs, n, ys, rd2, out, i0, i1,
                                                            accumulate);
    }
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}
