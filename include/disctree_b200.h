/*
 * disctree_b200.h -- C ABI of the B200 (sm_100a) disc-field treecode.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/disctree).  The reference is a Python package
 * whose native layer is a set of numba-jitted kernels called from
 * tree.py / direct.py / charges.py; every entry point below names the
 * reference routine it replaces.  INTEGRATION.md shows the ctypes binding a
 * maintainer would add to the reference.
 *
 * Conventions (all entry points):
 *   - Array arguments are DEVICE pointers (CUDA global memory on the current
 *     device) unless the parameter name ends in _host.  Scalars by value.
 *   - Work is enqueued on `stream` (a cudaStream_t, NULL = legacy default
 *     stream) and is asynchronous: results are valid once the stream is
 *     synchronised.  No entry point synchronises the device.
 *   - The caller owns every buffer, including outputs and workspaces; the
 *     library never allocates device memory.  `*_workspace()` functions give
 *     the required workspace size in bytes.
 *   - Return value: DT_OK (0) or a negative DT_ERR_* code; dt_last_error()
 *     returns a thread-local message for the last failure.  The reference's
 *     numba kernels have no error returns; its Python wrappers validate first
 *     (SURVEY.md §8(b)).  Validation here is limited to what is checkable
 *     without reading device memory.
 *   - Reentrant; no global mutable state besides the thread-local error text.
 *   - Indices inside the library are 32-bit: n_src, n_nodes < 2^31.
 */
#ifndef DISCTREE_B200_H
#define DISCTREE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DT_OK 0
#define DT_ERR_INVALID (-1)   /* bad argument */
#define DT_ERR_CUDA (-2)      /* CUDA runtime error (message in dt_last_error) */
#define DT_ERR_WORKSPACE (-3) /* workspace too small */
#define DT_ERR_DEVICE (-4)    /* current device is not sm_100 */

/* tree.py:32 MAX_DEPTH; levels are 0..DT_MAX_DEPTH */
#define DT_MAX_DEPTH 60
#define DT_MAX_LEVELS (DT_MAX_DEPTH + 1)

/* Tree metadata block (int64, device memory, DT_META_WORDS words) written by
 * dt_build_tree and read by dt_moments.  Level l occupies node indices
 * [meta[DT_META_LEVEL0 + l], meta[DT_META_LEVEL0 + l + 1]) (BFS order). */
#define DT_META_NODES 0    /* number of nodes                          */
#define DT_META_DEPTH 1    /* deepest level (Tree.depth)               */
#define DT_META_LEAVES 2   /* Tree.leaf_count                          */
#define DT_META_OVERFLOW 3 /* nonzero: node_capacity was too small     */
#define DT_META_CURLEVEL 4 /* internal                                 */
#define DT_META_P2M_UPTO 5 /* leaves below this index already formed (dt_build_tree_p2m) */
#define DT_META_LEVEL0 8
#define DT_META_WORDS 72

/* Direct-sum arithmetic (direct.py:52-88) */
#define DT_DIRECT_FP64 0  /* fp64 pairs, fp64 accumulation (phi_sum_plain)        */
#define DT_DIRECT_FP32 1  /* fp32 pair evaluation, fp64 accumulation (bench only)  */
#define DT_DIRECT_KAHAN 2 /* IEEE pairs, Kahan in ascending order (phi_sum_kahan)  */

/* Adaptive truncation-order selection mode (dt_choose_p_batch, eval) */
#define DT_PSEL_FAST 0  /* fp32 bound estimate, exact replica inside the margin */
#define DT_PSEL_EXACT 1 /* always the exact replica of the compiled reference   */

const char *dt_version(void);
const char *dt_last_error(void);
/* DT_OK iff the current CUDA device is compute capability 10.0 (B200). */
int dt_device_check(void);

/* ---------------------------------------------------------------- (a) */

/* Inclusive prefix sum prefix[i] = sum_{j<=i} qs[j] (replaces the sequential
 * np.cumsum of charges.py:130).  Deterministic (fixed reduction tree); it
 * differs from the sequential sum by round-off only. */
size_t dt_prefix_scan_workspace(int64_t n);
int dt_prefix_scan(const double *qs, double *prefix, int64_t n, void *workspace,
                   size_t workspace_bytes, void *stream);

/* e(y) = 2 * prefix_excl[lower_bound(xs, y)] - total, total = prefix[n-1]
 * (charges.py:183-187 _sign_terms; a source exactly at y counts on the minus
 * side).  Targets in any order (ascending runs are located through shared
 * memory when a workspace of dt_sign_terms_workspace() bytes is given; NULL
 * workspace searches every target in global memory).  n == 0 gives e = 0. */
size_t dt_sign_terms_workspace(int64_t n_targets);
int dt_sign_terms(const double *xs, const double *prefix, int64_t n, const double *ys,
                  double *e_out, int64_t n_targets, void *workspace, size_t workspace_bytes,
                  void *stream);
/* dt_sign_terms in two launches (the first needs no prefix, so a caller can
 * run it beside other work): dt_sign_bracket writes the tile brackets into
 * the workspace (dt_sign_terms_workspace(n_targets) bytes, required), and
 * dt_sign_terms_bracketed, after it in stream order, computes e from them.
 * The result equals dt_sign_terms'. */
int dt_sign_bracket(const double *xs, int64_t n, const double *ys, int64_t n_targets,
                    void *workspace, size_t workspace_bytes, void *stream);
int dt_sign_terms_bracketed(const double *xs, const double *prefix, int64_t n, const double *ys,
                            double *e_out, int64_t n_targets, void *workspace,
                            size_t workspace_bytes, void *stream);

/* Input validation in one pass (charges.py:114-132 rejects non-finite
 * positions/strengths; direct.py:43-49 non-finite targets; charges.py:200
 * and tree.py use ascending order).  flags[0] += number of non-finite
 * values, flags[1] += number of descents v[i+1] < v[i]; the caller zeroes
 * flags (2 int64 in device memory).  dt_unpack_pairs also splits
 * interleaved (x, q) pairs (16-byte aligned) into xs and qs, counting the
 * descents of x. */
int dt_check_values(const double *v, int64_t n, int64_t *flags, void *stream);
int dt_unpack_pairs(const double *pairs, int64_t n, double *xs, double *qs, int64_t *flags,
                    void *stream);

/* Charge assembly on the device (SURVEY.md §8(f) "next" #2).
 * dt_density_nodes: charges.py:135-161 from_density -- one (x, q) pair per
 * Gauss-Legendre node of each of `cells` cells on [a, b], interleaved into
 * pairs[2 cells order] in ascending order; values has cells (per-cell
 * constants) or cells + 1 entries (endpoint tabulation, np.interp); nodes and
 * weights are leggauss(order) on [-1, 1] (device arrays).  Bit-identical to
 * the reference's numpy arithmetic.
 * dt_mirror_charges: charges.py:164-180 with_images for one plane --
 * xm = 2 plane - xs, qm = -qs, keep = |xm - plane| < gap. */
int dt_density_nodes(double a, double b, int64_t cells, const double *values, int64_t n_values,
                     int64_t order, const double *nodes, const double *weights, double eps0,
                     double *pairs, void *stream);
int dt_mirror_charges(const double *xs, const double *qs, int64_t n, double plane, double gap,
                      double *xm, double *qm, uint8_t *keep, void *stream);

/* ---------------------------------------------------------------- (b) */

/* Level-synchronous breadth-first bisection tree over sorted xs[0..n)
 * (tree.py:156-222): bit-identical node arrays (BFS order, -1 = no child),
 * depth and leaf_count.  The padded root interval is computed on the device
 * exactly as tree.py:173-175 (pad = 1e-12 * max(1, |x_0|, |x_{n-1}|)).
 * `packed` (optional, may be NULL) receives node_capacity 32-byte records
 * for the traversal.
 * If the tree needs more than node_capacity nodes, meta[DT_META_OVERFLOW]
 * is set and the arrays are incomplete: enlarge and call again. */
size_t dt_build_workspace(int64_t n, int64_t node_capacity);
int dt_build_tree(const double *xs, int64_t n, int64_t leaf_capacity, int64_t max_depth,
                  int64_t node_capacity, double *lo, double *hi, double *center, double *half,
                  int64_t *level, int64_t *start, int64_t *end, int64_t *left, int64_t *right,
                  void *packed, int64_t *meta, void *workspace, size_t workspace_bytes,
                  void *stream);

/* dt_build_tree, and while block 0 runs the sparse deep levels the other
 * blocks form the leaves of the finished levels (P2M into moments_eval, the
 * traversal layout of dt_moments, and the (x, q) pairs into xq); meta[
 * DT_META_P2M_UPTO] records how far (leaves below that node index are
 * formed), and dt_moments / dt_moments_pack with the same moments_eval and
 * order skip those leaves.  order <= 31. */
int dt_build_tree_p2m(const double *xs, const double *qs, int64_t n, int64_t leaf_capacity,
                      int64_t max_depth, int64_t node_capacity, double *lo, double *hi,
                      double *center, double *half, int64_t *level, int64_t *start, int64_t *end,
                      int64_t *left, int64_t *right, void *packed, int64_t *meta, int64_t order,
                      double *moments_eval, int64_t eval_stride, double *xq, void *workspace,
                      size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- (c) */

/* Node moments m_k = sum_j q_j (x_j - c)^k / k!, k = 0..order (tree.py:224-238):
 * P2M at every leaf from its sources, then M2M (binomial shift) bottom-up
 * as a dataflow without grid barriers (the warp completing a node's last
 * child forms the node), fused into one kernel for order <= 31.  Reads the
 * tree produced by dt_build_tree (meta gives n_nodes); node_capacity bounds
 * the node arrays.  Two layouts:
 *   moments_eval: the traversal layout read by the *_packed and *_device
 *     evaluators, M_0 = m_0, M_k = (k-1)! gamma_(k-1) m_k with gamma_0 =
 *     gamma_1 = 1, gamma_n = (n+1)/n gamma_(n-2) (the scaling of the
 *     three-term far-field recurrence, csrc/dt_farcoef.cuh), row stride
 *     eval_stride (even, >= order + 1; padding zeroed; 16-byte aligned).
 *     Required for order <= 31, where the pass works on these rows only.
 *   moments: the reference layout, row-major [n_nodes][order + 1]; optional
 *     for order <= 31 (then derived from moments_eval at the end, as
 *     dt_moments_from_eval does), required above. */size_t dt_moments_workspace(int64_t node_capacity);
int dt_moments(const double *xs, const double *qs, const double *center, const int64_t *start,
               const int64_t *end, const int64_t *left, const int64_t *right,
               const int64_t *meta, int64_t order, double *moments, double *moments_eval,
               int64_t eval_stride, int64_t node_capacity, void *workspace,
               size_t workspace_bytes, void *stream);
/* dt_moments that also writes xq[2 n_src], the interleaved (x, q) pairs of
 * dt_pack_sources, from the loads P2M makes anyway (every source lies in one
 * leaf), so a step needs no separate pack pass (orders > 31: the pack kernel
 * runs after).  moments_eval is required. */
int dt_moments_pack(const double *xs, const double *qs, int64_t n_src, const double *center,
                    const int64_t *start, const int64_t *end, const int64_t *left,
                    const int64_t *right, const int64_t *meta, int64_t order, double *moments,
                    double *moments_eval, int64_t eval_stride, int64_t node_capacity, double *xq,
                    void *workspace, size_t workspace_bytes, void *stream);
/* Reference-layout moments[n_nodes][order + 1] from traversal rows:
 * m_k = M_k / ((k-1)! gamma_(k-1)) (one rounding per entry). */
int dt_moments_from_eval(const double *moments_eval, int64_t eval_stride, int64_t n_nodes,
                         int64_t order, double *moments, void *stream);

/* ---------------------------------------------------------------- (c) sharded */

/* Multi-GPU upward pass (the reference's run_chunked,
 * _kernels.py:269-289, shards targets only).  Every rank holds the full tree
 * and sources; rank r evaluates a contiguous slice of the sorted targets.
 * The moments are split at a cut level l: rank r forms (P2M + M2M) only the
 * subtrees under the level-l nodes it owns or its targets can open, the
 * level-l rows of the owners are all-gathered (one NCCL all-gather of
 * dt_shard_rows_bytes() per rank), and every rank forms levels < l
 * redundantly.  Each row is produced by the same arithmetic as dt_moments,
 * so every row a rank's traversal reads is bit-identical to the
 * single-GPU row and the field is bit-identical for any world size.
 *
 * Plan block: int64[DT_PLAN_WORDS] in device memory, written by
 * dt_shard_plan without host round trips. */
#define DT_MAX_WORLD 64
#define DT_PLAN_CUT 0         /* cut level l = min(requested, depth)               */
#define DT_PLAN_LEVEL_BEGIN 1 /* level-l nodes are [begin, end)                     */
#define DT_PLAN_LEVEL_END 2
#define DT_PLAN_SRC_LO 3      /* this rank forms the subtrees under level l whose   */
#define DT_PLAN_SRC_HI 4      /* source ranges lie in [src_lo, src_hi)              */
#define DT_PLAN_NEED_LO 5     /* level-l nodes its targets may open: [lo, hi)       */
#define DT_PLAN_NEED_HI 6
#define DT_PLAN_OWNER0 8      /* rank r owns level-l nodes [plan[8 + r], plan[9 + r]) */
#define DT_PLAN_WORDS (DT_PLAN_OWNER0 + DT_MAX_WORLD + 1)

/* Plan for `rank` of `world`: owners split the level-l nodes into contiguous
 * runs of ~n_src / world sources; the opened set holds every level-l node
 * with half * (1 + 2^-40) > theta * dist(center, [min ys, max ys]) -- a
 * superset of the nodes the MAC (R > 0 && h <= theta R, _kernels.py:211)
 * can reject for any of this rank's targets ys[0..n_targets).
 * targets_sorted != 0 reads the extremes from the ends of ys. */
int dt_shard_plan(const double *center, const double *half, const int64_t *start,
                  const int64_t *end, const int64_t *meta, int64_t n_src, const double *ys,
                  int64_t n_targets, int targets_sorted, double theta, int64_t cut_level,
                  int world, int rank, int64_t *plan, void *stream);
/* Per-rank slot of the gather buffer: 2^cut_level traversal rows of
 * eval_stride doubles (cut_level <= 20; 0 on bad arguments). */
size_t dt_shard_rows_bytes(int64_t cut_level, int64_t order, int64_t eval_stride);
/* dt_moments restricted to the plan: leaves above level l, and every node at
 * levels >= l whose sources lie in [src_lo, src_hi).  order <= 31; writes
 * moments_eval only (moments is ignored: dt_shard_finish derives it); the
 * workspace is dt_moments_workspace(node_capacity) bytes. */
int dt_moments_partial(const double *xs, const double *qs, const double *center,
                       const int64_t *start, const int64_t *end, const int64_t *left,
                       const int64_t *right, const int64_t *meta, const int64_t *plan,
                       int64_t order, double *moments, double *moments_eval,
                       int64_t eval_stride, int64_t node_capacity, void *workspace,
                       size_t workspace_bytes, void *stream);
/* Copy this rank's owned level-l rows into its gather slot `send`. */
int dt_shard_pack(const int64_t *plan, int rank, int64_t cut_level, int64_t order,
                  const double *moments, const double *moments_eval, int64_t eval_stride,
                  double *send, void *stream);
/* After the all-gather (recv = world slots, rank order): write every owner's
 * level-l rows, then form levels < l (M2M), in one kernel; if moments is not
 * NULL the reference layout of every node is derived as well. */
int dt_shard_finish(const int64_t *plan, int world, int64_t cut_level, const double *recv,
                    const double *center, const int64_t *left, const int64_t *right,
                    const int64_t *meta, int64_t order, double *moments, double *moments_eval,
                    int64_t eval_stride, void *stream);

/* ---------------------------------------------------------------- (d)+(e) */

typedef struct dt_eval_stats {
    uint64_t *hash;      /* ordered hash of the interaction events: h <- splitmix64(h ^ code)
                          * in the target's depth-first visit order (oracle.c) */
    int64_t *near_pairs; /* near-field (source, target) pairs                    */
    int64_t *n_far;      /* accepted far nodes                                   */
    int64_t *sum_p;      /* sum of truncation orders over accepted far nodes     */
    int64_t *n_p0;       /* accepted far nodes with p_use == 0                   */
    int64_t *n_exact;    /* far nodes whose order came from the exact replica    */
    /* a-posteriori bound audit (SURVEY.md §8(f) "next" #4): per target the sum
     * over accepted far nodes of bound_value(M, R, h, p_use) * sum_node |q|
     * (kernel.py:130-182, test_tree.py:216-250) with M the exact contour
     * supremum (rigorous); needs abs_prefix = inclusive prefix sums of |q_j|
     * over the sorted sources. */
    double *bound;
    const double *abs_prefix;
} dt_eval_stats;

/* Interleave (x_j, q_j) into xq[2n] for the traversal kernel.  The packed
 * evaluators read the node records with 32-byte loads and xq and the moment
 * rows with 16-byte loads: packed must be 32-byte aligned, xq and moments
 * 16-byte aligned and the moment stride even (DT_ERR_INVALID otherwise). */
int dt_pack_sources(const double *xs, const double *qs, int64_t n, double *xq, void *stream);
/* Pack the SoA node arrays into 32-byte records (`packed`, n_nodes). */
int dt_pack_tree(const double *centers, const double *halves, const int64_t *starts,
                 const int64_t *ends, const int64_t *lefts, const int64_t *rights,
                 int64_t n_nodes, void *packed, void *stream);

/* Traversal workspace slot (the workspace of the *_packed and *_device
 * evaluators must hold at least this many bytes and be 16-byte aligned):
 * the task counters (zeroed by the call, stream-ordered; warps take
 * 32-target tasks from per-SM segments of the target range, so
 * neighbouring targets run on the same SM), then the adaptive-order tables
 * each call builds for its tree (breakpoints of the bound scan per level). */
#define DT_EVAL_COUNTER_BYTES 65536

/* Workspace of dt_tree_phi_sum (packed copies + the counter slot). */
size_t dt_tree_eval_workspace(int64_t n_nodes, int64_t n_src, int64_t moment_stride);

/* Mirror of the numba seam _kernels.tree_phi_sum (_kernels.py:163-266):
 * far-field/near-field traversal for targets ys[i0:i1]; writes out[i0:i1]
 * (out[i] += phi if accumulate != 0).  The MAC and the adaptive truncation
 * order are bit-identical to the compiled reference; cos_tab/sin_tab are the
 * n_samples contour tables (tree.py:342, from host numpy).  Targets may be
 * in any order; sorted targets traverse coherently (fast).  Orders are
 * limited to 127 as in dt_moments: p, p_cap <= 127 and moment_stride <= 128
 * (DT_ERR_ARG otherwise; the recurrence tables end there). */
int dt_tree_phi_sum(const double *centers, const double *halves, const int64_t *starts,
                    const int64_t *ends, const int64_t *lefts, const int64_t *rights,
                    const double *moments, int64_t moment_stride, int64_t n_nodes,
                    const double *xs, const double *qs, int64_t n_src, double rd2, double theta,
                    int64_t p, int adaptive, double tol_share, int64_t p_cap,
                    const double *cos_tab, const double *sin_tab, int64_t n_samples,
                    const double *ys, double *out, int64_t i0, int64_t i1, int accumulate,
                    void *workspace, size_t workspace_bytes, void *stream);

/* Same, on pre-packed nodes/sources and traversal-layout moments (dt_moments
 * moments_eval, even stride); what the Python layer uses.
 * `stats`
 * (host struct of device pointers, indexed by target) may be NULL; psel_mode
 * is DT_PSEL_FAST or DT_PSEL_EXACT. */
int dt_tree_phi_sum_packed(const void *packed_nodes, int64_t n_nodes, const double *moments,
                           int64_t moment_stride, const double *xq, int64_t n_src, double rd2,
                           double theta, int64_t p, int adaptive, double tol_share,
                           int64_t p_cap, const double *cos_tab, const double *sin_tab,
                           int64_t n_samples, const double *ys, double *out, int64_t i0,
                           int64_t i1, int accumulate, int psel_mode,
                           const dt_eval_stats *stats, void *workspace,
                           size_t workspace_bytes, void *stream);

/* dt_tree_eval_device with the sign term fused (the field E = e + phi, as
 * dt_tree_field_packed): out[i] = E(ys[i]) for i in [i0, i1); xs / prefix
 * are the sorted sources and their inclusive prefix sums; a workspace of
 * dt_tree_field_workspace(i1 - i0) bytes adds the per-tile search brackets. */
int dt_tree_field_device(const void *packed_nodes, const int64_t *meta, int64_t node_capacity,
                         const double *moments, int64_t moment_stride, const double *xq,
                         const double *xs, const double *prefix, int64_t n_src, double rd2,
                         double theta, int64_t p, int adaptive, double tolerance, int64_t p_cap,
                         const double *cos_tab, const double *sin_tab, int64_t n_samples,
                         const double *ys, double *out, int64_t i0, int64_t i1, void *workspace,
                         size_t workspace_bytes, void *stream);

/* Whole field E(y) = e(y) + phi(y) (tree.py:340-373) in one kernel: the
 * sign term is computed per target from the sorted sources xs[0..n_src) and
 * their inclusive prefix sums exactly as dt_sign_terms does, then added to
 * the traversal sum as evaluate_all does.  ys and out may live in pinned
 * host memory (UVA): each target is read once and each value written once
 * over the host link while the traversal runs.  flags (device int64[2], may
 * be NULL): flags[0] += number of non-finite targets (those are not
 * traversed; the caller rejects the call).  The workspace holds the task
 * counters; with dt_tree_field_workspace(i1 - i0) bytes it also holds the
 * lower_bound of every 1024th target, which brackets the sign-term searches
 * of sorted targets (checked per target, so any order stays correct). */
size_t dt_tree_field_workspace(int64_t n_targets);
int dt_tree_field_packed(const void *packed_nodes, int64_t n_nodes, const double *moments,
                         int64_t moment_stride, const double *xq, const double *xs,
                         const double *prefix, int64_t n_src, double rd2, double theta,
                         int64_t p, int adaptive, double tol_share, int64_t p_cap,
                         const double *cos_tab, const double *sin_tab, int64_t n_samples,
                         const double *ys, double *out, int64_t i0, int64_t i1,
                         int64_t *flags, void *workspace, size_t workspace_bytes, void *stream);

/* Same traversal on a tree fresh from dt_build_tree without any host
 * round trip: the tree depth (and so tol_share = tolerance / (3 max(depth,1)),
 * tree.py:268-270) is read from `meta` on the device.  node_capacity bounds
 * the node arrays.  Used by the pipelined (CUDA-graph capturable) step. */
int dt_tree_eval_device(const void *packed_nodes, const int64_t *meta, int64_t node_capacity,
                        const double *moments, int64_t moment_stride, const double *xq,
                        int64_t n_src, double rd2, double theta, int64_t p, int adaptive,
                        double tolerance, int64_t p_cap, const double *cos_tab,
                        const double *sin_tab, int64_t n_samples, const double *ys, double *out,
                        int64_t i0, int64_t i1, int accumulate, void *workspace,
                        size_t workspace_bytes, void *stream);

/* dt_tree_eval_device in two launches, so the order tables can be built on
 * another stream while the moments are formed: dt_eval_prepare zeroes the
 * workspace slot's task counters and builds the tables (same arguments;
 * ys/out are not read); dt_tree_eval_device_prepared then runs only the
 * traversal on that slot, after the prepare call in stream order (an event
 * when the streams differ).  The result equals dt_tree_eval_device's. */
int dt_eval_prepare(const void *packed_nodes, const int64_t *meta, int64_t node_capacity,
                    const double *moments, int64_t moment_stride, const double *xq,
                    int64_t n_src, double rd2, double theta, int64_t p, int adaptive,
                    double tolerance, int64_t p_cap, const double *cos_tab,
                    const double *sin_tab, int64_t n_samples, const double *ys, double *out,
                    int64_t i0, int64_t i1, int accumulate, void *workspace,
                    size_t workspace_bytes, void *stream);
int dt_tree_eval_device_prepared(const void *packed_nodes, const int64_t *meta,
                                 int64_t node_capacity, const double *moments,
                                 int64_t moment_stride, const double *xq, int64_t n_src,
                                 double rd2, double theta, int64_t p, int adaptive,
                                 double tolerance, int64_t p_cap, const double *cos_tab,
                                 const double *sin_tab, int64_t n_samples, const double *ys,
                                 double *out, int64_t i0, int64_t i1, int accumulate,
                                 void *workspace, size_t workspace_bytes, void *stream);

/* Adaptive order for n (R, h) pairs (test hook for _kernels.py:212-231):
 * p_out[i] = order chosen; tier_out[i] (may be NULL) = 0 fast path, 1 exact. */
int dt_choose_p_batch(const double *big_r, const double *h, int64_t n, double rd2,
                      double tol_share, int64_t p_cap, const double *cos_tab,
                      const double *sin_tab, int64_t n_samples, int psel_mode, int64_t *p_out,
                      int32_t *tier_out, void *stream);

/* ---------------------------------------------------------------- (f) */

/* out[i] (+)= sum_j qs[j] (xs[j] - ys[i]) / sqrt((xs[j] - ys[i])^2 + rd2),
 * i in [i0, i1): _kernels.phi_sum_plain (mode DT_DIRECT_FP64),
 * _kernels.phi_sum_kahan (DT_DIRECT_KAHAN, bit-identical), or the
 * fp32-evaluation / fp64-accumulation bench variant (DT_DIRECT_FP32). */
int dt_phi_sum_direct(const double *xs, const double *qs, int64_t n, const double *ys,
                      double rd2, double *out, int64_t i0, int64_t i1, int mode, int accumulate,
                      void *stream);

/* Replaces _kernels.phi_sum_symmetric (_kernels.py:107-142), the path
 * evaluate_direct takes when targets == sources (direct.py:80): out[i] (+)=
 * sum_j q_j (x_j - x_i) / sqrt((x_j - x_i)^2 + rd2) for i < n, every pair
 * evaluated once and applied to both of its targets; a fixed summation order
 * (deterministic).  workspace: dt_phi_sum_symmetric_workspace(n) bytes
 * (~4 n^2 / 2048 bytes: the packed column partials; 2 GB at n = 2^20,
 * 8 GB at 2^21, quadratic beyond).  The Python layer caps it
 * (direct.SYM_MAX_WORKSPACE = 8 GiB) and uses dt_phi_sum_direct above. */
size_t dt_phi_sum_symmetric_workspace(int64_t n);
int dt_phi_sum_symmetric(const double *xs, const double *qs, int64_t n, double rd2, double *out,
                         int accumulate, void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------- sorting */

/* Stable sort of v[0..n) (charges.py:127: np.argsort(x, kind="stable") in
 * from_particles; unsorted targets in evaluate_all): LSD radix sort on
 * order-preserving 64-bit codes (-0.0 taken as +0.0: equal keys keep their
 * input order, as numpy's).  Outputs (each may be NULL): sorted[i] =
 * v[perm[i]], perm[i], payload_out[i] = payload[perm[i]].  n < 2^31.  Reads
 * the eight digit histograms back to the host once to skip passes whose digit
 * is the same for every key (synchronises the stream).  NaN keys sort by
 * their bits (callers reject them first). */
size_t dt_sort_workspace(int64_t n);
int dt_sort_stable(const double *v, int64_t n, double *sorted, int64_t *perm,
                   const double *payload, double *payload_out, void *workspace,
                   size_t workspace_bytes, void *stream);
/* Order-preserving compaction (with_images, charges.py:164-180): the r-th
 * kept (xs[i], qs[i]) (keep[i] != 0, index order) goes to out_pairs[2 (offset
 * + r)]; *count (device int64) receives the number kept.  Workspace
 * dt_compact_workspace(n) bytes. */
size_t dt_compact_workspace(int64_t n);
int dt_compact_pairs(const double *xs, const double *qs, const uint8_t *keep, int64_t n,
                     double *out_pairs, int64_t offset, int64_t *count, void *workspace,
                     size_t workspace_bytes, void *stream);
/* Stream-ordered zero fill of device memory (flag words of the checks). */
int dt_zero(void *p, size_t bytes, void *stream);
/* dst[i] = src[perm[i]] (scatter == 0) or dst[perm[i]] = src[i] (scatter != 0). */
int dt_permute(const double *src, const int64_t *perm, int64_t n, double *dst, int scatter,
               void *stream);

/* ---------------------------------------------------------------- diagnostics */

/* FP64 FMA throughput probe for the roofline denominator: `blocks` x 256
 * threads, each running 8 independent DFMA chains for `iters` steps; writes
 * one value per thread to out (keeps the work live).  Flops = 16 * iters *
 * blocks * 256. */
int dt_fp64_probe(double *out, int64_t iters, int blocks, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DISCTREE_B200_H */
