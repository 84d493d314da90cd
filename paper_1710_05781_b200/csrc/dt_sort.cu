// Stable sort of fp64 keys on the device (charges.py:127: np.argsort(x,
// kind="stable") in from_particles; evaluate_all sorts unsorted targets).
//
// LSD radix sort, 8-bit digits, on order-preserving 64-bit codes of the keys
// (sign bit flipped for positives, all bits for negatives; -0.0 is mapped to
// +0.0 first, so equal values keep their input order as in numpy's stable
// argsort).  One pass over the keys builds all eight digit histograms; a pass
// whose digit is the same for every key is skipped (the exponent bytes of a
// narrow range).  Each remaining pass:
//   rank    per 4096-key tile: counts per digit (smem atomics), written digit-
//           major so one exclusive scan of the counts gives every (digit,
//           tile) its output offset;
//   scan    exclusive scan of the 256 x tiles counts (one block per digit
//           row, then the rows' totals in order: deterministic);
//   scatter every key goes to offset(digit, tile) + the number of earlier keys
//           of its tile with the same digit (warp match + per-warp counters in
//           tile order: stable).
// The payload is the original index (int32), so the permutation comes out
// too; the sorted values are gathered through it at the end.
#include <algorithm>

#include "dt_common.cuh"

namespace {

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 16;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 4096 keys
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int RADIX = 256;

__device__ __forceinline__ unsigned long long encode_key(double v)
{
    if (v == 0.0)
        v = 0.0;  // -0.0 and +0.0 compare equal: one code
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void sort_encode_kernel(const double *__restrict__ v, int64_t n,
                                   unsigned long long *__restrict__ keys, int32_t *__restrict__ idx,
                                   unsigned *__restrict__ hist)  // [8][256]
{
    __shared__ unsigned h[8][RADIX];
    for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x)
        (&h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long c = encode_key(__ldg(v + i));
        keys[i] = c;
        idx[i] = (int32_t)i;
#pragma unroll
        for (int d = 0; d < 8; ++d)
            atomicAdd(&h[d][(c >> (8 * d)) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * RADIX; i += blockDim.x)
        if ((&h[0][0])[i])
            atomicAdd(hist + i, (&h[0][0])[i]);
}

// counts[d * tiles + t] = keys of tile t with digit d
__global__ void __launch_bounds__(SORT_THREADS) sort_count_kernel(
    const unsigned long long *__restrict__ keys, int64_t n, int shift, unsigned *__restrict__ counts,
    int64_t tiles)
{
    __shared__ unsigned h[RADIX];
    for (int i = threadIdx.x; i < RADIX; i += blockDim.x)
        h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SORT_TILE;
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = base + (int64_t)r * SORT_THREADS + threadIdx.x;
        if (i < n)
            atomicAdd(&h[(__ldg(keys + i) >> shift) & 0xff], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += blockDim.x)
        counts[(int64_t)d * tiles + blockIdx.x] = h[d];
}

// Exclusive scan of counts[256 * tiles] in digit-major order: block d scans
// row d in place and writes its total; sort_rows_excl_kernel then turns the
// totals into the offsets of the rows (fixed order).
__global__ void __launch_bounds__(1024) sort_scan_row_kernel(unsigned *counts, int64_t tiles,
                                                             unsigned *row_total)
{
    __shared__ unsigned ws[32];
    unsigned *row = counts + (int64_t)blockIdx.x * tiles;
    const int lane = dt_lane(), warp = threadIdx.x >> 5;
    unsigned carry = 0;
    for (int64_t t0 = 0; t0 < tiles; t0 += blockDim.x) {
        const int64_t t = t0 + threadIdx.x;
        const unsigned v = t < tiles ? row[t] : 0u;
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(DT_FULL, x, o);
            if (lane >= o)
                x += y;
        }
        if (lane == 31)
            ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(DT_FULL, w, o);
                if (lane >= o)
                    w += y;
            }
            ws[lane] = w;
        }
        __syncthreads();
        const unsigned before = (warp ? ws[warp - 1] : 0u) + carry;
        if (t < tiles)
            row[t] = before + x - v;
        const unsigned tot = ws[(blockDim.x >> 5) - 1];
        __syncthreads();
        carry += tot;
    }
    if (threadIdx.x == 0)
        row_total[blockIdx.x] = carry;
}

// row_total[d] -> sum of the totals of the rows below d (one block, fixed order)
__global__ void sort_rows_excl_kernel(unsigned *row_total)
{
    if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int d = 0; d < RADIX; ++d) {
            const unsigned t = row_total[d];
            row_total[d] = acc;
            acc += t;
        }
    }
}

// Stable scatter: warp w of the tile handles keys [w * 512, w * 512 + 512) in
// 16 rounds of 32 (tile order = (warp, round, lane)).
__global__ void __launch_bounds__(SORT_THREADS) sort_scatter_kernel(
    const unsigned long long *__restrict__ keys_in, const int32_t *__restrict__ idx_in, int64_t n,
    int shift, const unsigned *__restrict__ counts, const unsigned *__restrict__ row_total,
    int64_t tiles, unsigned long long *__restrict__ keys_out, int32_t *__restrict__ idx_out)
{
    __shared__ unsigned wcnt[SORT_WARPS][RADIX];  // per warp: running count per digit
    __shared__ unsigned base_s[RADIX];
    const int lane = dt_lane(), warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < SORT_WARPS * RADIX; i += blockDim.x)
        (&wcnt[0][0])[i] = 0;
    // output offset of (digit, this tile): the rows below d, then the row scan
    for (int d = threadIdx.x; d < RADIX; d += blockDim.x)
        base_s[d] = __ldg(row_total + d) + __ldg(counts + (int64_t)d * tiles + blockIdx.x);
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SORT_TILE + (int64_t)warp * (32 * SORT_ITEMS);
    unsigned long long k[SORT_ITEMS];
    int32_t p[SORT_ITEMS];
    unsigned local[SORT_ITEMS];
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = base + 32 * r + lane;
        const bool ok = i < n;
        k[r] = ok ? __ldg(keys_in + i) : 0ull;
        p[r] = ok ? __ldg(idx_in + i) : 0;
        const unsigned d = (unsigned)(k[r] >> shift) & 0xff;
        const unsigned act = __ballot_sync(DT_FULL, ok);
        const unsigned peers = __match_any_sync(DT_FULL, ok ? d : 0x100u) & act;
        const unsigned before = __popc(peers & ((1u << lane) - 1u));
        local[r] = 0;
        if (ok) {
            local[r] = wcnt[warp][d] + before;  // keys of this warp's earlier rounds, then lanes
            __syncwarp(peers);
            if (before == 0)  // the first lane of each digit group advances the count
                wcnt[warp][d] += __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();
    // earlier warps' keys of the same digit come first
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = base + 32 * r + lane;
        if (i < n) {
            const unsigned d = (unsigned)(k[r] >> shift) & 0xff;
            unsigned off = base_s[d] + local[r];
            for (int w = 0; w < warp; ++w)
                off += wcnt[w][d];
            keys_out[off] = k[r];
            idx_out[off] = p[r];
        }
    }
}

// Outputs gathered through the permutation (sorted values keep their exact
// bits, -0.0 included).
__global__ void sort_gather_kernel(const double *__restrict__ v, const int32_t *__restrict__ idx,
                                   int64_t n, double *__restrict__ sorted,
                                   int64_t *__restrict__ perm, const double *__restrict__ payload,
                                   double *__restrict__ payload_out)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = __ldg(idx + i);
        if (sorted)
            sorted[i] = __ldg(v + j);
        if (perm)
            perm[i] = j;
        if (payload_out)
            payload_out[i] = __ldg(payload + j);
    }
}

__global__ void permute_kernel(const double *__restrict__ src, const int64_t *__restrict__ perm,
                               int64_t n, double *__restrict__ dst, int scatter)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = __ldg(perm + i);
        if (scatter)
            dst[j] = __ldg(src + i);
        else
            dst[i] = __ldg(src + j);
    }
}

int64_t sort_tiles(int64_t n) { return (n + SORT_TILE - 1) / SORT_TILE; }

}  // namespace

extern "C" size_t dt_sort_workspace(int64_t n)
{
    if (n <= 0)
        return 0;
    const int64_t tiles = sort_tiles(n);
    // keys and indices twice (ping-pong), counts, row totals, histograms
    return (size_t)n * 2 * (sizeof(unsigned long long) + sizeof(int32_t)) +
           (size_t)RADIX * tiles * sizeof(unsigned) + RADIX * sizeof(unsigned) +
           8 * RADIX * sizeof(unsigned) + 64;
}

extern "C" int dt_sort_stable(const double *v, int64_t n, double *sorted, int64_t *perm,
                              const double *payload, double *payload_out, void *workspace,
                              size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(n >= 0 && n < ((int64_t)1 << 31), "n must be in [0, 2^31)");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(v, "null pointer");
    DT_CHECK_ARG(!payload_out || payload, "payload_out needs payload");
    if (!workspace || workspace_bytes < dt_sort_workspace(n))
        return dt_set_error(DT_ERR_WORKSPACE, "sort workspace too small");
    DT_CHECK_ARG(((uintptr_t)workspace & 7) == 0, "sort workspace must be 8-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tiles = sort_tiles(n);
    unsigned long long *k0 = (unsigned long long *)workspace, *k1 = k0 + n;
    int32_t *i0 = (int32_t *)(k1 + n), *i1 = i0 + n;
    unsigned *counts = (unsigned *)(i1 + n);
    unsigned *rows = counts + (size_t)RADIX * tiles;
    unsigned *hist = rows + RADIX;
    DT_CUDA_TRY(cudaMemsetAsync(hist, 0, 8 * RADIX * sizeof(unsigned), s));
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dt_num_sms() * 8);
    sort_encode_kernel<<<(unsigned)blocks, 256, 0, s>>>(v, n, k0, i0, hist);
    DT_CUDA_TRY(cudaGetLastError());
    // which passes move anything (a digit shared by every key is a no-op pass)
    unsigned h[8 * RADIX];
    DT_CUDA_TRY(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s));
    DT_CUDA_TRY(cudaStreamSynchronize(s));
    for (int d = 0; d < 8; ++d) {
        bool trivial = false;
        for (int b = 0; b < RADIX; ++b)
            if (h[d * RADIX + b] == (unsigned)n)
                trivial = true;
        if (trivial)
            continue;
        const int shift = 8 * d;
        sort_count_kernel<<<(unsigned)tiles, SORT_THREADS, 0, s>>>(k0, n, shift, counts, tiles);
        sort_scan_row_kernel<<<RADIX, 1024, 0, s>>>(counts, tiles, rows);
        sort_rows_excl_kernel<<<1, 32, 0, s>>>(rows);
        sort_scatter_kernel<<<(unsigned)tiles, SORT_THREADS, 0, s>>>(k0, i0, n, shift, counts, rows,
                                                                   tiles, k1, i1);
        DT_CUDA_TRY(cudaGetLastError());
        std::swap(k0, k1);
        std::swap(i0, i1);
    }
    sort_gather_kernel<<<(unsigned)blocks, 256, 0, s>>>(v, i0, n, sorted, perm, payload,
                                                        payload_out);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_permute(const double *src, const int64_t *perm, int64_t n, double *dst,
                          int scatter, void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(src && perm && dst, "null pointer");
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dt_num_sms() * 8);
    permute_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(src, perm, n, dst,
                                                                       scatter != 0);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

// ---- order-preserving compaction (with_images, charges.py:164-180) ----
//
// out[2 (offset + r)] = (xs[i], qs[i]) for the r-th i with keep[i] != 0, in
// index order.  Two passes over 4096-element tiles: kept counts per tile,
// then each tile's rank base = the counts of the tiles before it (summed in
// a fixed order by the tile's first warp) plus a block scan.  *count (device)
// receives the number kept.
namespace {

__global__ void __launch_bounds__(SORT_THREADS) compact_count_kernel(const uint8_t *__restrict__ keep,
                                                                     int64_t n,
                                                                     unsigned *__restrict__ tile_cnt)
{
    __shared__ unsigned c_s;
    if (threadIdx.x == 0)
        c_s = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SORT_TILE;
    unsigned c = 0;
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = base + (int64_t)r * SORT_THREADS + threadIdx.x;
        c += i < n && __ldg(keep + i);
    }
    for (int o = 16; o > 0; o >>= 1)
        c += __shfl_xor_sync(DT_FULL, c, o);
    if (dt_lane() == 0)
        atomicAdd(&c_s, c);
    __syncthreads();
    if (threadIdx.x == 0)
        tile_cnt[blockIdx.x] = c_s;
}

__global__ void __launch_bounds__(SORT_THREADS) compact_write_kernel(
    const double *__restrict__ xs, const double *__restrict__ qs, const uint8_t *__restrict__ keep,
    int64_t n, const unsigned *__restrict__ tile_cnt, int64_t tiles, double2 *__restrict__ out,
    int64_t offset, int64_t *count)
{
    __shared__ unsigned long long base_s;
    __shared__ unsigned wsum[SORT_WARPS];
    const int lane = dt_lane(), warp = threadIdx.x >> 5;
    if (warp == 0) {
        unsigned long long b = 0;
        for (int64_t t = lane; t < blockIdx.x; t += 32)
            b += __ldg(tile_cnt + t);
        for (int o = 16; o > 0; o >>= 1)
            b += __shfl_xor_sync(DT_FULL, b, o);
        if (lane == 0) {
            base_s = b;
            if (blockIdx.x == tiles - 1)
                *count = (int64_t)(b + __ldg(tile_cnt + blockIdx.x));
        }
    }
    // keys of this tile in index order: warp w owns 512 consecutive elements
    const int64_t t0 = (int64_t)blockIdx.x * SORT_TILE + (int64_t)warp * (32 * SORT_ITEMS);
    unsigned mine = 0;
    unsigned masks[SORT_ITEMS];
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = t0 + 32 * r + lane;
        masks[r] = __ballot_sync(DT_FULL, i < n && __ldg(keep + i));
        mine += __popc(masks[r]);
    }
    if (lane == 0)
        wsum[warp] = mine;
    __syncthreads();
    unsigned long long off = base_s;
    for (int w = 0; w < warp; ++w)
        off += wsum[w];
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; ++r) {
        const int64_t i = t0 + 32 * r + lane;
        if ((masks[r] >> lane) & 1u)
            out[offset + (int64_t)off + __popc(masks[r] & ((1u << lane) - 1u))] =
                make_double2(__ldg(xs + i), __ldg(qs + i));
        off += __popc(masks[r]);
    }
}

}  // namespace

extern "C" size_t dt_compact_workspace(int64_t n)
{
    return (size_t)(n > 0 ? (n + SORT_TILE - 1) / SORT_TILE : 1) * sizeof(unsigned);
}

extern "C" int dt_compact_pairs(const double *xs, const double *qs, const uint8_t *keep, int64_t n,
                                double *out_pairs, int64_t offset, int64_t *count,
                                void *workspace, size_t workspace_bytes, void *stream)
{
    DT_CHECK_ARG(n >= 0 && offset >= 0, "negative size");
    DT_CHECK_ARG(count, "null count");
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        DT_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int64_t), s));
        return DT_OK;
    }
    DT_CHECK_ARG(xs && qs && keep && out_pairs, "null pointer");
    DT_CHECK_ARG(((uintptr_t)out_pairs & 15) == 0, "out_pairs must be 16-byte aligned");
    if (!workspace || workspace_bytes < dt_compact_workspace(n))
        return dt_set_error(DT_ERR_WORKSPACE, "compaction workspace too small");
    const int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
    unsigned *cnt = (unsigned *)workspace;
    compact_count_kernel<<<(unsigned)tiles, SORT_THREADS, 0, s>>>(keep, n, cnt);
    compact_write_kernel<<<(unsigned)tiles, SORT_THREADS, 0, s>>>(xs, qs, keep, n, cnt, tiles,
                                                                (double2 *)out_pairs, offset, count);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_zero(void *p, size_t bytes, void *stream)
{
    if (bytes == 0)
        return DT_OK;
    DT_CHECK_ARG(p, "null pointer");
    DT_CUDA_TRY(cudaMemsetAsync(p, 0, bytes, (cudaStream_t)stream));
    return DT_OK;
}
