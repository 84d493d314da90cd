// (a) e_m term: deterministic prefix scan of q and the sign term.
//
// Reference: charges.py:130 (prefix = np.cumsum(qs), sequential) and
// charges.py:183-187 (_sign_terms).  The scan is a fixed-shape reduction
// tree (tile sums and group sums of 64 tiles -> tile scans offset by the
// group and tile sums below them, the second pass in reverse tile order so
// most of its reads of q hit L2), so repeated calls
// are bit-identical; it differs from the sequential cumsum by round-off
// (<= ~1e-15 * sum|q| at 2^24).  Algorithmic HBM traffic 16N (read q, write
// prefix) + 16T (sign terms).  A single-pass variant (tile sums published
// and summed in a fixed order by every later tile, no look-back) measured
// 97 us against 79 us for the earlier three passes: its tiles wait on their
// predecessors while holding their SM slots; a decoupled look-back would
// make the last bits depend on timing.
#include <algorithm>

#include "dt_common.cuh"

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096 elements

constexpr int SCAN_GROUP = 64;  // tiles per group sum

// Pass 1: per-tile sums A_t, coalesced (thread t sums elements t, t+256,
// ...), fixed-order block reduction.  The last tile of a group of 64 to
// finish (arrival counter) also forms the group sum B_g = A_(64g) + ... in
// index order, so pass 2 needs no separate scan of the tile sums.
__global__ void __launch_bounds__(SCAN_THREADS) tile_sums_kernel(const double *__restrict__ q,
                                                                 int64_t n, int64_t n_tiles,
                                                                 double *tile_sum,
                                                                 double *group_sum,
                                                                 unsigned *group_ctr)
{
    __shared__ double wt[SCAN_THREADS / 32];
    __shared__ bool last_s;
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const int64_t j = base + (int64_t)i * SCAN_THREADS;
        if (j < n)
            s += __ldg(q + j);
    }
    // fixed-order block reduction (warp tree, then warp totals in order)
    s = dt_warp_sum(s);
    if (dt_lane() == 0)
        wt[threadIdx.x >> 5] = s;
    __syncthreads();
    const int64_t g = blockIdx.x / SCAN_GROUP, g0 = g * SCAN_GROUP;
    const int64_t g1 = min(n_tiles, g0 + SCAN_GROUP);
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w)
            t += wt[w];
        tile_sum[blockIdx.x] = t;
        __threadfence();  // the sum precedes the arrival
        last_s = atomicAdd(group_ctr + g, 1u) == (unsigned)(g1 - g0 - 1);
    }
    __syncthreads();
    if (last_s && threadIdx.x < 32) {
        __threadfence();  // every arrival's sum is visible after ours
        double b = 0.0;
        for (int64_t i = g0 + threadIdx.x; i < g1; i += 32)
            b += __ldcg(tile_sum + i);
        b = dt_warp_sum(b);
        if (threadIdx.x == 0)
            group_sum[g] = b;
    }
}

// Pass 2: scan each tile with its exclusive offset.  Warp w owns 512
// consecutive elements, read/written coalesced in 16 rows of 32; each row is
// a warp shuffle scan carried across rows, then warps are offset in order.
// Tiles run in reverse order: pass 1 left the last ~100 MB of q in L2 (126 MB),
// so most of this pass's reads hit L2 instead of HBM; q is read with an
// evict-first hint and prefix written with streaming stores so they do not
// push the rest of q out.
#ifndef DT_SCAN_MINB
#define DT_SCAN_MINB 4  // 64 registers: 78 us against 91 us at 82 registers (configs[2])
#endif
__global__ void __launch_bounds__(SCAN_THREADS, DT_SCAN_MINB) tile_apply_kernel(const double *__restrict__ q,
                                                                  int64_t n,
                                                                  const double *__restrict__ tile_sum,
                                                                  const double *__restrict__ group_sum,
                                                                  double *__restrict__ prefix)
{
    __shared__ double wt[SCAN_THREADS / 32];
    __shared__ double part_s[2];
    const int lane = dt_lane(), warp = threadIdx.x >> 5;
    const int64_t tile = (int64_t)gridDim.x - 1 - blockIdx.x;
    const int64_t base = tile * SCAN_TILE + (int64_t)warp * (32 * SCAN_ITEMS) + lane;
    double v[SCAN_ITEMS];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const int64_t j = base + 32 * i;
        v[i] = j < n ? __ldcs(q + j) : 0.0;
    }
    double carry = 0.0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        double x = v[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(DT_FULL, x, o);
            if (lane >= o)
                x += t;
        }
        x += carry;
        carry = __shfl_sync(DT_FULL, x, 31);
        v[i] = x;
    }
    if (lane == 31)
        wt[warp] = carry;
    // exclusive offset (B_0 + .. + B_(G-1)) + (A_(64G) + .. + A_(t-1)), each
    // a fixed-order warp reduction (identical on every call)
    const int64_t g = tile / SCAN_GROUP;
    if (warp < 2) {
        double a = 0.0;
        if (warp == 0) {
            for (int64_t i = lane; i < g; i += 32)
                a += __ldg(group_sum + i);
        } else {
            for (int64_t i = g * SCAN_GROUP + lane; i < tile; i += 32)
                a += __ldg(tile_sum + i);
        }
        a = dt_warp_sum(a);
        if (lane == 0)
            part_s[warp] = a;
    }
    __syncthreads();
    double off = part_s[0] + part_s[1];
    for (int w = 0; w < warp; ++w)
        off += wt[w];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const int64_t j = base + 32 * i;
        if (j < n)
            __stcs(prefix + j, off + v[i]);
    }
}

// One pass (default): every tile scans its 4096 values in registers and
// publishes its total; tile totals are combined up a binary tree of aligned
// groups (the second of two siblings to arrive forms their parent, left +
// right), and a tile's exclusive offset is the sum of the aligned groups
// that tile the range before it, taken from the largest to the smallest
// (the binary digits of its index).  Every addition has a fixed position in
// a fixed tree, so the result does not depend on timing (a decoupled
// look-back adds whatever predecessor prefixes happen to be ready), and q is
// read once.  Tiles take their index from a ticket, so every group a tile
// waits for belongs to tiles that are already running; it waits only after
// publishing its own total.  Measured at 2^24 values: 0.193 ms with a binary
// group tree, 0.115 ms with groups of 16 (three levels above 4096 tiles),
// against 0.078 ms for the two passes below (whose second pass reads most of
// q from L2): a tile holds its SM slot while the groups before it form
// (a fence, an acq_rel arrival and a 16-value reduction per level), so the
// two passes stay the default.  Both are deterministic.
#ifndef DT_SCAN_ONEPASS
#define DT_SCAN_ONEPASS 0  // 0.115 ms against 0.078 ms for the two passes (configs[2], see below)
#endif
constexpr int SCAN_MAX_LEVELS = 32;
struct ScanTree {
    unsigned *ticket;
    double *sum;          // level b groups at sum[off[b] ..]
    unsigned *ready;      // 1 once sum[] of that group is written
    unsigned *arrived;    // children arrived at the group (level >= 1)
    int64_t off[SCAN_MAX_LEVELS + 1];
    int64_t count[SCAN_MAX_LEVELS + 1];
    int levels;
};

constexpr int SCAN_RADIX = 16;  // groups of 16 groups: 3 levels above 4096 tiles

__global__ void __launch_bounds__(SCAN_THREADS, DT_SCAN_MINB) scan_onepass_kernel(
    const double *__restrict__ q, int64_t n, double *__restrict__ prefix, ScanTree t)
{
    __shared__ double wt[SCAN_THREADS / 32];
    __shared__ double off_s;
    __shared__ unsigned tile_s;
    const int lane = dt_lane(), warp = threadIdx.x >> 5;
    if (threadIdx.x == 0)
        tile_s = atomicAdd(t.ticket, 1u);
    __syncthreads();
    const int64_t tile = tile_s;
    const int64_t base = tile * SCAN_TILE + (int64_t)warp * (32 * SCAN_ITEMS) + lane;
    double v[SCAN_ITEMS];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const int64_t j = base + 32 * i;
        v[i] = j < n ? __ldcs(q + j) : 0.0;
    }
    double carry = 0.0;
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        double x = v[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double u = __shfl_up_sync(DT_FULL, x, o);
            if (lane >= o)
                x += u;
        }
        x += carry;
        carry = __shfl_sync(DT_FULL, x, 31);
        v[i] = x;
    }
    if (lane == 31)
        wt[warp] = carry;
    __syncthreads();
    if (warp == 0) {
        // publish the tile total; the last of 16 siblings to arrive forms
        // their parent (a fixed-order reduction of the 16) and climbs on
        double val = 0.0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w)
            val += wt[w];
        int64_t idx = tile;
        for (int b = 0;; ++b) {
            if (lane == 0) {
                t.sum[t.off[b] + idx] = val;
                __threadfence();
                asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(t.ready + t.off[b] + idx), "r"(1u)
                             : "memory");
            }
            const int64_t g = idx / SCAN_RADIX;
            if (b + 1 > t.levels || (g + 1) * SCAN_RADIX > t.count[b])
                break;  // the parent group is not whole: never used
            unsigned old = 0;
            if (lane == 0)
                asm volatile("atom.acq_rel.gpu.add.u32 %0, [%1], 1;"
                             : "=r"(old)
                             : "l"(t.arrived + t.off[b + 1] + g)
                             : "memory");
            old = __shfl_sync(DT_FULL, old, 0);
            if (old != SCAN_RADIX - 1)
                break;  // a sibling forms the parent
            double x = lane < SCAN_RADIX ? __ldcg(t.sum + t.off[b] + g * SCAN_RADIX + lane) : 0.0;
            val = dt_warp_sum(x);
            idx = g;
        }
        // exclusive offset: per level (top first) the whole sibling groups
        // before the tile's own, each level a fixed-order warp reduction
        double off = 0.0;
        for (int b = t.levels; b >= 0; --b) {
            const int64_t own = tile >> (4 * b);  // the tile's group at level b
            const int d = (int)(own % SCAN_RADIX);
            if (d == 0)
                continue;
            const int64_t first = t.off[b] + (own - d);
            double x = 0.0;
            if (lane < d) {
                unsigned r;
                while (true) {
                    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(r) : "l"(t.ready + first + lane)
                                 : "memory");
                    if (r)
                        break;
                    __nanosleep(32);
                }
                x = __ldcg(t.sum + first + lane);
            }
            off += dt_warp_sum(x);
        }
        if (lane == 0)
            off_s = off;
    }
    __syncthreads();
    double off = off_s;
    for (int w = 0; w < warp; ++w)
        off += wt[w];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        const int64_t j = base + 32 * i;
        if (j < n)
            __stcs(prefix + j, off + v[i]);
    }
}

// e(y) for arbitrary targets; total = prefix[n-1].  A block owns 2048
// consecutive targets.  When they ascend (the usual case: evaluate_all sorts
// them) two threads bracket the block's source range with global searches,
// the range is staged in shared memory and every target is located there;
// otherwise each target is searched in global memory.
#ifndef DT_SIGN_PER_THREAD
#define DT_SIGN_PER_THREAD 2  // 512-target tiles: 0.154 ms at configs[2] (4: 0.166, 1: 0.193)
#endif
#ifndef DT_SIGN_SMEM
#define DT_SIGN_SMEM 1024
#endif
constexpr int SIGN_THREADS = 256;
constexpr int SIGN_PER_THREAD = DT_SIGN_PER_THREAD;
constexpr int SIGN_TILE = SIGN_THREADS * SIGN_PER_THREAD;
constexpr int SIGN_SMEM = DT_SIGN_SMEM;

// bracket[b] = lower_bound(xs, ys[b * SIGN_TILE]) for every tile boundary
// (and the last target), all searched in parallel.
__global__ void sign_bracket_kernel(const double *__restrict__ xs, int64_t n,
                                    const double *__restrict__ ys, int64_t t,
                                    int64_t *__restrict__ bracket, int64_t nb)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb)
        return;
    const int64_t i = b < nb ? b * SIGN_TILE : t - 1;
    bracket[b] = dt_lower_bound(xs, 0, n, __ldg(ys + i));
}

__global__ void __launch_bounds__(SIGN_THREADS) sign_terms_kernel(
    const double *__restrict__ xs, const double *__restrict__ prefix, int64_t n,
    const double *__restrict__ ys, double *__restrict__ e, int64_t t,
    const int64_t *__restrict__ bracket, int64_t nb)
{
    __shared__ double xsm[SIGN_SMEM];
    const int64_t t0 = (int64_t)blockIdx.x * SIGN_TILE;
    const int64_t t1 = min(t, t0 + SIGN_TILE);
    if (n == 0) {
#pragma unroll
        for (int k = 0; k < SIGN_PER_THREAD; ++k) {
            const int64_t i = t0 + (int64_t)k * SIGN_THREADS + threadIdx.x;
            if (i < t1)
                e[i] = 0.0;
        }
        return;
    }
    // the bracket is read with the targets, and the source range staged
    // before the sortedness of the tile is known (discarded if it is not):
    // two dependent rounds of global loads before the searches instead of four
    int64_t blo = 0, bhi = n;
    if (bracket) {
        // the next tile's first target bounds this tile's last one from above
        blo = __ldg(bracket + blockIdx.x);
        bhi = min(n, __ldg(bracket + blockIdx.x + 1) + 1);
    }
    double y[SIGN_PER_THREAD];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < SIGN_PER_THREAD; ++k) {
        const int64_t i = t0 + (int64_t)k * SIGN_THREADS + threadIdx.x;
        y[k] = i < t1 ? __ldg(ys + i) : 0.0;
        // across the tile boundary too: the next tile's first target bounds
        // this tile's search range from above only if it is not below ours
        if (i < t1 && i + 1 < t && !(y[k] <= __ldg(ys + i + 1)))
            ok = false;
    }
    const bool fits = bracket && blo <= bhi && bhi - blo <= SIGN_SMEM;
    if (fits)
        for (int64_t j = blo + threadIdx.x; j < bhi; j += SIGN_THREADS)
            xsm[j - blo] = __ldg(xs + j);
    const bool sorted = __syncthreads_and(ok);  // also orders the staging
    int64_t lo = 0, hi = n;
    if (sorted && bracket) {
        lo = blo;
        hi = bhi;
    }
    const bool staged = sorted && fits;
    const double total = __ldg(prefix + n - 1);
#pragma unroll
    for (int k = 0; k < SIGN_PER_THREAD; ++k) {
        const int64_t i = t0 + (int64_t)k * SIGN_THREADS + threadIdx.x;
        if (i >= t1)
            continue;
        int64_t idx;
        if (staged) {
            int a = 0, b = (int)(hi - lo);
            while (a < b) {
                const int m = (a + b) >> 1;
                if (xsm[m] < y[k])
                    a = m + 1;
                else
                    b = m;
            }
            idx = lo + a;
        } else {
            idx = dt_lower_bound(xs, lo, hi, y[k]);
        }
        const double below = idx == 0 ? 0.0 : __ldg(prefix + idx - 1);
        e[i] = __dsub_rn(__dmul_rn(2.0, below), total);
    }
}

}  // namespace

// Workspace: two-pass: tile sums, group sums (8 bytes each), group arrival
// counters; one pass: the group tree (a sum, a ready flag and an arrival
// counter per group of every level, about 2 x tiles groups) and a ticket.
static int64_t scan_tree_nodes(int64_t tiles, int64_t *off, int64_t *count, int *levels)
{
    int64_t total = 0, c = tiles;
    int b = 0;
    for (;; ++b) {
        if (off) {
            off[b] = total;
            count[b] = c;
        }
        total += c;
        if (c <= 1 || b == SCAN_MAX_LEVELS)
            break;
        c = (c + SCAN_RADIX - 1) / SCAN_RADIX;
    }
    if (levels)
        *levels = b;
    return total;
}

extern "C" size_t dt_prefix_scan_workspace(int64_t n)
{
    const int64_t tiles = n > 0 ? (n + SCAN_TILE - 1) / SCAN_TILE : 1;
    const int64_t groups = (tiles + SCAN_GROUP - 1) / SCAN_GROUP;
    const size_t two_pass = (size_t)(tiles + groups) * sizeof(double) + (size_t)groups * sizeof(unsigned);
    const int64_t nodes = scan_tree_nodes(tiles, nullptr, nullptr, nullptr);
    const size_t one_pass = (size_t)nodes * (sizeof(double) + 2 * sizeof(unsigned)) + 16;
    return std::max(two_pass, one_pass);
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
    DT_CHECK_ARG(((uintptr_t)workspace & 7) == 0, "scan workspace must be 8-byte aligned");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    DT_CHECK_ARG(tiles < ((int64_t)1 << 31), "too many values");
#if DT_SCAN_ONEPASS
    ScanTree t;
    const int64_t nodes = scan_tree_nodes(tiles, t.off, t.count, &t.levels);
    t.sum = (double *)workspace;
    t.ready = (unsigned *)(t.sum + nodes);
    t.arrived = t.ready + nodes;
    t.ticket = t.arrived + nodes;
    DT_CUDA_TRY(cudaMemsetAsync(t.ready, 0, (size_t)(2 * nodes + 1) * sizeof(unsigned), s));
    scan_onepass_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(qs, n, prefix, t);
#else
    const int64_t groups = (tiles + SCAN_GROUP - 1) / SCAN_GROUP;
    double *tsum = (double *)workspace, *gsum = tsum + tiles;
    unsigned *gctr = (unsigned *)(gsum + groups);
    DT_CUDA_TRY(cudaMemsetAsync(gctr, 0, (size_t)groups * sizeof(unsigned), s));
    tile_sums_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(qs, n, tiles, tsum, gsum, gctr);
    tile_apply_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(qs, n, tsum, gsum, prefix);
#endif
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" size_t dt_sign_terms_workspace(int64_t n_targets)
{
    return (size_t)((n_targets + SIGN_TILE - 1) / SIGN_TILE + 2) * sizeof(int64_t);
}

static int sign_terms(const double *xs, const double *prefix, int64_t n, const double *ys,
                      double *e_out, int64_t n_targets, void *workspace, size_t workspace_bytes,
                      void *stream, int mode)
{
    DT_CHECK_ARG(n >= 0 && n_targets >= 0, "negative size");
    if (n_targets == 0)
        return DT_OK;
    DT_CHECK_ARG(ys && (mode == 1 || e_out) && (n == 0 || xs) && (mode == 1 || n == 0 || prefix),
                 "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nb = (n_targets + SIGN_TILE - 1) / SIGN_TILE;
    int64_t *bracket = nullptr;
    if (workspace && workspace_bytes >= dt_sign_terms_workspace(n_targets) && n > 0) {
        bracket = (int64_t *)workspace;
        if (mode != 2)
            sign_bracket_kernel<<<(unsigned)((nb + 1 + 127) / 128), 128, 0, s>>>(xs, n, ys,
                                                                             n_targets, bracket, nb);
    } else if (mode != 0 && n > 0) {
        return dt_set_error(DT_ERR_WORKSPACE, "sign-term workspace too small");
    }
    if (mode != 1)
        sign_terms_kernel<<<(unsigned)nb, SIGN_THREADS, 0, s>>>(xs, prefix, n, ys, e_out,
                                                                n_targets, bracket, nb);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_sign_terms(const double *xs, const double *prefix, int64_t n, const double *ys,
                             double *e_out, int64_t n_targets, void *workspace,
                             size_t workspace_bytes, void *stream)
{
    return sign_terms(xs, prefix, n, ys, e_out, n_targets, workspace, workspace_bytes, stream, 0);
}

extern "C" int dt_sign_bracket(const double *xs, int64_t n, const double *ys, int64_t n_targets,
                               void *workspace, size_t workspace_bytes, void *stream)
{
    return sign_terms(xs, nullptr, n, ys, nullptr, n_targets, workspace, workspace_bytes, stream,
                      1);
}

extern "C" int dt_sign_terms_bracketed(const double *xs, const double *prefix, int64_t n,
                                       const double *ys, double *e_out, int64_t n_targets,
                                       void *workspace, size_t workspace_bytes, void *stream)
{
    return sign_terms(xs, prefix, n, ys, e_out, n_targets, workspace, workspace_bytes, stream, 2);
}

// ---- input validation (charges.py:114-132 from_particles, direct.py:43-49
// _as_targets): one pass counting non-finite values and descents, so the
// host reads back two integers instead of running several torch reductions.

namespace {

__device__ __forceinline__ void add_flags(unsigned long long bad, unsigned long long desc,
                                          int64_t *flags)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad += __shfl_xor_sync(DT_FULL, bad, o);
        desc += __shfl_xor_sync(DT_FULL, desc, o);
    }
    if (dt_lane() == 0 && (bad | desc)) {
        if (bad)
            atomicAdd(reinterpret_cast<unsigned long long *>(flags), bad);
        if (desc)
            atomicAdd(reinterpret_cast<unsigned long long *>(flags + 1), desc);
    }
}

__global__ void check_values_kernel(const double *__restrict__ v, int64_t n, int64_t *flags)
{
    unsigned long long bad = 0, desc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double a = __ldg(v + i);
        bad += !isfinite(a);
        if (i + 1 < n)
            desc += __ldg(v + i + 1) < a;
    }
    add_flags(bad, desc, flags);
}

__global__ void unpack_pairs_kernel(const double2 *__restrict__ xq, int64_t n,
                                    double *__restrict__ xs, double *__restrict__ qs,
                                    int64_t *flags)
{
    unsigned long long bad = 0, desc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = __ldg(xq + i);
        xs[i] = p.x;
        qs[i] = p.y;
        bad += !isfinite(p.x) + !isfinite(p.y);
        if (i + 1 < n)
            desc += __ldg(reinterpret_cast<const double *>(xq) + 2 * (i + 1)) < p.x;
    }
    add_flags(bad, desc, flags);
}

}  // namespace

extern "C" int dt_check_values(const double *v, int64_t n, int64_t *flags, void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    DT_CHECK_ARG(flags, "null flags");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(v, "null pointer");
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dt_num_sms() * 8);
    check_values_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(v, n, flags);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_unpack_pairs(const double *pairs, int64_t n, double *xs, double *qs,
                               int64_t *flags, void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    DT_CHECK_ARG(flags, "null flags");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(pairs && xs && qs, "null pointer");
    DT_CHECK_ARG(((uintptr_t)pairs & 15) == 0, "pairs must be 16-byte aligned");
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dt_num_sms() * 8);
    unpack_pairs_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        (const double2 *)pairs, n, xs, qs, flags);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

// ---- charge assembly on the device (SURVEY.md §8(f) "next" #2) ----
//
// from_density (charges.py:135-161): one charge per Gauss-Legendre node,
// x = mid_c + (dx/2) node_j, q = ((0.5 w_j) sigma(x)) dx / (2 eps0), with
// numpy's operation order (edges = a + dx*i, mids = 0.5 (e_c + e_c+1),
// np.interp for endpoint tabulation: slope (x - e_j) + v_j).  The pairs come
// out interleaved, in ascending cell/node order, ready for dt_unpack_pairs.
// with_images (charges.py:164-180): mirrored = 2 plane - x, kept iff
// |mirrored - plane| < gap.

namespace {

__global__ void density_nodes_kernel(double a, double dx, int64_t cells,
                                     const double *__restrict__ values, int per_cell, int order,
                                     const double *__restrict__ nodes,
                                     const double *__restrict__ weights, double two_eps0,
                                     double2 *__restrict__ pairs)
{
    const int64_t n = cells * order;
    const double hdx = __dmul_rn(0.5, dx);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / order;
        const int j = (int)(i - c * order);
        const double e0 = __dadd_rn(a, __dmul_rn(dx, (double)c));
        const double e1 = __dadd_rn(a, __dmul_rn(dx, (double)(c + 1)));
        const double x = __dadd_rn(__dmul_rn(0.5, __dadd_rn(e0, e1)), __dmul_rn(hdx, nodes[j]));
        double sigma;
        if (per_cell) {
            sigma = values[c];
        } else {
            // np.interp(x, edges, values): k = last edge <= x (edges ascending)
            int64_t lo = 0, hi = cells + 1;  // search in [0, cells]
            while (hi - lo > 1) {
                const int64_t mid = (lo + hi) >> 1;
                const double em = __dadd_rn(a, __dmul_rn(dx, (double)mid));
                if (em <= x)
                    lo = mid;
                else
                    hi = mid;
            }
            const int64_t k = lo;
            const double ek = __dadd_rn(a, __dmul_rn(dx, (double)k));
            if (x < __dadd_rn(a, 0.0) || k >= cells) {
                sigma = x < a ? values[0] : values[cells];
            } else if (ek == x) {
                sigma = values[k];
            } else {
                const double ek1 = __dadd_rn(a, __dmul_rn(dx, (double)(k + 1)));
                const double slope = __ddiv_rn(__dsub_rn(values[k + 1], values[k]),
                                               __dsub_rn(ek1, ek));
                sigma = __dadd_rn(__dmul_rn(slope, __dsub_rn(x, ek)), values[k]);
                if (isnan(sigma)) {
                    sigma = __dadd_rn(__dmul_rn(slope, __dsub_rn(x, ek1)), values[k + 1]);
                    if (isnan(sigma) && values[k] == values[k + 1])
                        sigma = values[k];
                }
            }
        }
        const double q = __ddiv_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(0.5, weights[j]), sigma), dx), two_eps0);
        pairs[i] = make_double2(x, q);
    }
}

__global__ void mirror_kernel(const double *__restrict__ xs, const double *__restrict__ qs,
                              int64_t n, double plane, double gap, double *__restrict__ xm,
                              double *__restrict__ qm, uint8_t *__restrict__ keep)
{
    const double two_plane = __dmul_rn(2.0, plane);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double m = __dsub_rn(two_plane, xs[i]);
        xm[i] = m;
        qm[i] = -qs[i];
        keep[i] = fabs(__dsub_rn(m, plane)) < gap;
    }
}

}  // namespace

extern "C" int dt_density_nodes(double a, double b, int64_t cells, const double *values,
                                int64_t n_values, int64_t order, const double *nodes,
                                const double *weights, double eps0, double *pairs, void *stream)
{
    DT_CHECK_ARG(cells >= 1 && order >= 1 && order <= 16, "bad cells / quadrature order");
    DT_CHECK_ARG(n_values == cells || n_values == cells + 1, "values must have cells or cells+1 entries");
    DT_CHECK_ARG(eps0 > 0.0 && a < b, "bad eps0 / domain");
    DT_CHECK_ARG(values && nodes && weights && pairs, "null pointer");
    DT_CHECK_ARG(((uintptr_t)pairs & 15) == 0, "pairs must be 16-byte aligned");
    const double dx = (b - a) / (double)cells;  // host IEEE division, as numpy
    const int64_t n = cells * order;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dt_num_sms() * 8);
    density_nodes_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        a, dx, cells, values, n_values == cells ? 1 : 0, (int)order, nodes, weights, 2.0 * eps0,
        (double2 *)pairs);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_mirror_charges(const double *xs, const double *qs, int64_t n, double plane,
                                 double gap, double *xm, double *qm, uint8_t *keep, void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(xs && qs && xm && qm && keep, "null pointer");
    DT_CHECK_ARG(gap > 0.0, "gap_length must be positive");
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)dt_num_sms() * 8);
    mirror_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(xs, qs, n, plane, gap, xm,
                                                                      qm, keep);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}
