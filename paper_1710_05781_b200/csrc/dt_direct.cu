// (f) Brute-force O(N*T) direct sum: accuracy oracle and FP64 roofline bench.
//
// Reference: _kernels.py:49-59 (phi_sum_plain), 145-160 (phi_sum_kahan),
// dispatched by evaluate_direct (direct.py:52-88).  targets == sources:
// dt_phi_sum_symmetric (below), each pair evaluated once as in the
// reference's phi_sum_symmetric (_kernels.py:62-142).
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

// ---- targets == sources: each pair once (_kernels.py:62-142, phi_sum_symmetric)
//
// The reference splits the pair matrix into row blocks, evaluates each pair
// once and applies it with both signs, accumulating into a partial matrix
// that is summed in a fixed order.  Here: bands of SYM_BAND rows (one block
// each, 8 rows per thread in registers); block b evaluates the pairs of its
// rows with every later column j (j >= the band's end), staged through
// shared memory, one block per (band, chunk of SYM_CHUNK columns) so no
// block carries a whole band (load balance).  s = d * rsqrt(d^2 + r_d^2),
// d = x_j - x_i, adds q_j s to row i (registers; one row partial per chunk)
// and -q_i s to column j: the column terms are summed over the thread's 8
// rows, over the warp (butterfly) and over the 8 warps in a fixed order, then
// stored once per (band, column) in a packed partial array.  The pairs inside
// a band are summed plainly (sym_diag_kernel), and sym_combine_kernel adds,
// per target, diagonal + its row partials in ascending chunk order + the
// column partials of the earlier bands in ascending band order:
// deterministic, ~10 FP64 instructions per pair, i.e. ~5 per (target,
// source) interaction against 10 for the plain kernel.
constexpr int SYM_THREADS = 256;
constexpr int SYM_TPT = 8;
constexpr int64_t SYM_BAND = SYM_THREADS * SYM_TPT;
constexpr int SYM_TILE = 256;
constexpr int64_t SYM_CHUNK = 32768;  // columns per block (a multiple of SYM_BAND)
static_assert(SYM_CHUNK % SYM_BAND == 0, "chunks hold whole bands");

// first chunk holding columns of band b (columns j >= (b + 1) SYM_BAND)
__host__ __device__ inline int64_t sym_first_chunk(int64_t b)
{
    return (b + 1) * SYM_BAND / SYM_CHUNK;
}

// first column-partial word of band b (columns j >= (b + 1) SYM_BAND)
__host__ __device__ inline int64_t sym_col_offset(int64_t b, int64_t n)
{
    return b * n - SYM_BAND * (b * (b + 1) / 2);
}

__global__ void __launch_bounds__(SYM_THREADS) sym_band_kernel(const double *__restrict__ xs,
                                                               const double *__restrict__ qs,
                                                               int64_t n, double rd2,
                                                               double *__restrict__ rows,
                                                               double *__restrict__ cols)
{
    __shared__ double2 tile[SYM_TILE];
    __shared__ double csum[SYM_THREADS / 32][SYM_TILE];
    const int64_t b = blockIdx.y, chunk = blockIdx.x, r0 = b * SYM_BAND, c0 = r0 + SYM_BAND;
    if (chunk < sym_first_chunk(b))
        return;
    const int64_t cbeg = max(c0, chunk * SYM_CHUNK), cend = min(n, (chunk + 1) * SYM_CHUNK);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double y[SYM_TPT], q[SYM_TPT], acc[SYM_TPT];
#pragma unroll
    for (int k = 0; k < SYM_TPT; ++k) {
        const int64_t i = r0 + threadIdx.x + (int64_t)k * SYM_THREADS;
        y[k] = i < n ? __ldg(xs + i) : 0.0;
        q[k] = i < n ? __ldg(qs + i) : 0.0;  // a missing row adds nothing to any column
        acc[k] = 0.0;
    }
    double *const out_cols = cols + sym_col_offset(b, n);
    for (int64_t j0 = cbeg; j0 < cend; j0 += SYM_TILE) {
        const int m = (int)min((int64_t)SYM_TILE, cend - j0);
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += SYM_THREADS)
            tile[j] = make_double2(__ldg(xs + j0 + j), __ldg(qs + j0 + j));
        __syncthreads();
#pragma unroll 2
        for (int j = 0; j < m; ++j) {
            const double2 v = tile[j];
            double c = 0.0;
#pragma unroll
            for (int k = 0; k < SYM_TPT; ++k) {
                const double d = v.x - y[k];
                const double sv = d * dt_rsqrt(__fma_rn(d, d, rd2));
                acc[k] = __fma_rn(v.y, sv, acc[k]);
                c = __fma_rn(-q[k], sv, c);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                c += __shfl_xor_sync(DT_FULL, c, o);
            if (lane == 0)
                csum[warp][j] = c;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += SYM_THREADS) {
            double t = csum[0][j];
#pragma unroll
            for (int w = 1; w < SYM_THREADS / 32; ++w)
                t += csum[w][j];
            out_cols[j0 - c0 + j] = t;
        }
    }
#pragma unroll
    for (int k = 0; k < SYM_TPT; ++k) {
        const int64_t i = r0 + threadIdx.x + (int64_t)k * SYM_THREADS;
        if (i < n)
            rows[chunk * n + i] = acc[k];
    }
}

// pairs inside band b, plainly: diag[i] = sum_{j in band} q_j s(x_j - x_i)
__global__ void __launch_bounds__(SYM_THREADS) sym_diag_kernel(const double *__restrict__ xs,
                                                               const double *__restrict__ qs,
                                                               int64_t n, double rd2,
                                                               double *__restrict__ diag)
{
    __shared__ double2 tile[SYM_TILE];
    const int64_t r0 = (int64_t)blockIdx.x * SYM_BAND, r1 = min(n, r0 + SYM_BAND);
    double y[SYM_TPT], acc[SYM_TPT];
#pragma unroll
    for (int k = 0; k < SYM_TPT; ++k) {
        const int64_t i = r0 + threadIdx.x + (int64_t)k * SYM_THREADS;
        y[k] = i < n ? __ldg(xs + i) : 0.0;
        acc[k] = 0.0;
    }
    for (int64_t j0 = r0; j0 < r1; j0 += SYM_TILE) {
        const int m = (int)min((int64_t)SYM_TILE, r1 - j0);
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += SYM_THREADS)
            tile[j] = make_double2(__ldg(xs + j0 + j), __ldg(qs + j0 + j));
        __syncthreads();
        for (int j = 0; j < m; ++j) {
            const double2 v = tile[j];
#pragma unroll
            for (int k = 0; k < SYM_TPT; ++k) {
                const double d = v.x - y[k];
                acc[k] = __fma_rn(v.y, d * dt_rsqrt(__fma_rn(d, d, rd2)), acc[k]);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < SYM_TPT; ++k) {
        const int64_t i = r0 + threadIdx.x + (int64_t)k * SYM_THREADS;
        if (i < n)
            diag[i] = acc[k];
    }
}

// out[i] (+)= diag[i] + rows[i] + sum over earlier bands b' (ascending) of
// the column partial of (b', i)
__global__ void sym_combine_kernel(const double *__restrict__ diag, const double *__restrict__ rows,
                                   const double *__restrict__ cols, int64_t n,
                                   double *__restrict__ out, int accumulate)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int64_t band = i / SYM_BAND, nch = (n + SYM_CHUNK - 1) / SYM_CHUNK;
    double t = diag[i];
    for (int64_t c = sym_first_chunk(band); c < nch; ++c)
        t += rows[c * n + i];
    for (int64_t bb = 0; bb < band; ++bb)
        t += __ldg(cols + sym_col_offset(bb, n) + (i - (bb + 1) * SYM_BAND));
    out[i] = accumulate ? out[i] + t : t;
}

}  // namespace

extern "C" size_t dt_phi_sum_symmetric_workspace(int64_t n)
{
    if (n <= 0)
        return 0;
    const int64_t nb = (n + SYM_BAND - 1) / SYM_BAND, nch = (n + SYM_CHUNK - 1) / SYM_CHUNK;
    return (size_t)((1 + nch) * n + sym_col_offset(nb, n) + SYM_BAND * nb) * sizeof(double);
}

extern "C" int dt_phi_sum_symmetric(const double *xs, const double *qs, int64_t n, double rd2,
                                    double *out, int accumulate, void *workspace,
                                    size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(xs && qs && out, "null pointer");
    DT_CHECK_ARG(rd2 > 0.0, "rd2 must be > 0");
    if (!workspace || workspace_bytes < dt_phi_sum_symmetric_workspace(n))
        return dt_set_error(DT_ERR_WORKSPACE, "symmetric direct workspace too small");
    DT_CHECK_ARG(((uintptr_t)workspace & 7) == 0, "workspace must be 8-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nb = (n + SYM_BAND - 1) / SYM_BAND, nch = (n + SYM_CHUNK - 1) / SYM_CHUNK;
    DT_CHECK_ARG(nb < 65536, "too many sources for the symmetric path");
    double *diag = (double *)workspace, *rows = diag + n, *cols = rows + nch * n;
    sym_band_kernel<<<dim3((unsigned)nch, (unsigned)nb), SYM_THREADS, 0, s>>>(xs, qs, n, rd2, rows,
                                                                             cols);
    sym_diag_kernel<<<(unsigned)nb, SYM_THREADS, 0, s>>>(xs, qs, n, rd2, diag);
    sym_combine_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(diag, rows, cols, n, out,
                                                                    accumulate);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

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
