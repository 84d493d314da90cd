// (a) e_m term: deterministic prefix scan of q and the sign term.
//
// Reference: charges.py:130 (prefix = np.cumsum(qs), sequential) and
// charges.py:183-187 (_sign_terms).  The scan is a fixed-shape reduction
// tree (tile sums -> one-block scan of tile sums -> tile scans), so repeated
// calls are bit-identical; it differs from the sequential cumsum by
// round-off (<= ~1e-15 * sum|q| at 2^24).  HBM traffic: 8N (tile sums) +
// 16N (scan pass) + 16T (sign terms).
#include "dt_common.cuh"

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096 elements
constexpr int PARTIAL_THREADS = 1024;

// Block-wide inclusive scan of one double per thread; returns the block total.
__device__ double block_inclusive_scan(double v, double *warp_tot)
{
    const int lane = dt_lane(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_up_sync(DT_FULL, v, o);
        if (lane >= o)
            v += t;
    }
    if (lane == 31)
        warp_tot[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double w = lane < nw ? warp_tot[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            double t = __shfl_up_sync(DT_FULL, w, o);
            if (lane >= o)
                w += t;
        }
        if (lane < nw)
            warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    if (warp > 0)
        v += warp_tot[warp - 1];
    __syncthreads();
    return v;
}

// Pass 1: per-tile sums (each thread sums SCAN_ITEMS consecutive values).
__global__ void __launch_bounds__(SCAN_THREADS) tile_sums_kernel(const double *__restrict__ q,
                                                                 int64_t n,
                                                                 double *__restrict__ tile_sum)
{
    __shared__ double wt[SCAN_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        int64_t j = base + i;
        if (j < n)
            s += __ldg(q + j);
    }
    // fixed-order block reduction (warp tree, then warp totals in order)
    s = dt_warp_sum(s);
    if (dt_lane() == 0)
        wt[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w)
            t += wt[w];
        tile_sum[blockIdx.x] = t;
    }
}

// Pass 2: exclusive scan of the tile sums in one block (sequential chunks per
// thread, then a block scan of the chunk totals).
__global__ void __launch_bounds__(PARTIAL_THREADS) tile_scan_kernel(double *__restrict__ tile_sum,
                                                                    int64_t n_tiles)
{
    __shared__ double wt[PARTIAL_THREADS / 32];
    const int64_t per = (n_tiles + PARTIAL_THREADS - 1) / PARTIAL_THREADS;
    const int64_t b0 = (int64_t)threadIdx.x * per;
    double s = 0.0;
    for (int64_t i = 0; i < per; ++i)
        if (b0 + i < n_tiles)
            s += tile_sum[b0 + i];
    double incl = block_inclusive_scan(s, wt);
    double run = incl - s;  // exclusive offset of this thread's chunk
    // recompute exclusive prefix sequentially within the chunk
    for (int64_t i = 0; i < per; ++i) {
        int64_t b = b0 + i;
        if (b < n_tiles) {
            double v = tile_sum[b];
            tile_sum[b] = run;
            run += v;
        }
    }
}

// Pass 3: scan each tile with its exclusive offset.
__global__ void __launch_bounds__(SCAN_THREADS) tile_apply_kernel(const double *__restrict__ q,
                                                                  int64_t n,
                                                                  const double *__restrict__ tile_off,
                                                                  double *__restrict__ prefix)
{
    __shared__ double wt[SCAN_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    double v[SCAN_ITEMS];
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        int64_t j = base + i;
        v[i] = j < n ? __ldg(q + j) : 0.0;
        s += v[i];
    }
    double incl = block_inclusive_scan(s, wt);
    double run = tile_off[blockIdx.x] + (incl - s);
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        run += v[i];
        int64_t j = base + i;
        if (j < n)
            prefix[j] = run;
    }
}

// e(y) for arbitrary targets; total = prefix[n-1].
__global__ void sign_terms_kernel(const double *__restrict__ xs,
                                  const double *__restrict__ prefix, int64_t n,
                                  const double *__restrict__ ys, double *__restrict__ e,
                                  int64_t t)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t)
        return;
    if (n == 0) {
        e[i] = 0.0;
        return;
    }
    double y = __ldg(ys + i);
    int64_t idx = dt_lower_bound(xs, 0, n, y);
    double total = __ldg(prefix + n - 1);
    double below = idx == 0 ? 0.0 : __ldg(prefix + idx - 1);
    e[i] = __dsub_rn(__dmul_rn(2.0, below), total);
}

}  // namespace

extern "C" size_t dt_prefix_scan_workspace(int64_t n)
{
    int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    return (size_t)(tiles > 0 ? tiles : 1) * sizeof(double);
}

extern "C" int dt_prefix_scan(const double *qs, double *prefix, int64_t n, void *workspace,
                              size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(n >= 0, "n must be >= 0");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(qs && prefix, "null pointer");
    if (workspace_bytes < dt_prefix_scan_workspace(n) || !workspace)
        return dt_set_error(DT_ERR_WORKSPACE, "prefix scan workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    double *tsum = (double *)workspace;
    tile_sums_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(qs, n, tsum);
    tile_scan_kernel<<<1, PARTIAL_THREADS, 0, s>>>(tsum, tiles);
    tile_apply_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(qs, n, tsum, prefix);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_sign_terms(const double *xs, const double *prefix, int64_t n, const double *ys,
                             double *e_out, int64_t n_targets, void *stream)
{
    DT_CHECK_ARG(n >= 0 && n_targets >= 0, "negative size");
    if (n_targets == 0)
        return DT_OK;
    DT_CHECK_ARG(ys && e_out && (n == 0 || (xs && prefix)), "null pointer");
    const int th = 256;
    sign_terms_kernel<<<(unsigned)((n_targets + th - 1) / th), th, 0, (cudaStream_t)stream>>>(
        xs, prefix, n, ys, e_out, n_targets);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}
