/*
 * oracle.c -- CPU restatement of the disctree hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_1710_05781_b200/) links, loads or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it, and only as the checker or the timed CPU baseline.
 *
 * Each routine restates one piece of the reference (`disctree`, a Python +
 * numba package) in plain C so that the GPU path can be checked against it
 * without the reference being present (it does not exist on the GPU box).
 * The oracle is pinned against fixtures produced by the live reference in
 * tests/golden/ (make_golden.py); see tests/test_oracle_golden.py.
 *
 * Fidelity levels:
 *   - tree structure (or_build): bit-exact restatement of tree.py:156-222.
 *   - MAC and adaptive truncation order (or_tree_phi_sum): bit-exact
 *     restatement of the compiled numba kernel _kernels.py:199-231.  The
 *     contour sample loop reproduces the exact operation sequence LLVM emits
 *     for it under fastmath={"reassoc","contract"} (numba 0.65 / llvmlite
 *     0.47 on x86-64 with FMA): wr = fma(R, cos, -R); Re(z^2) =
 *     fma(wr, wr, -(wi*wi)); the numpy/CACM-312 csqrt of numba's cmathimpl
 *     (libm hypot + sqrt); CPython's _Py_c_quot with its products fused;
 *     |.| = libm hypot; and the bound value reassociated to
 *     ((R*(1.1*M))*(h/R)) / (R-h).  Compile with -ffp-contract=off so that
 *     only the explicit fma() calls below are fused.
 *   - field values: same formulas as the reference, sequential sums.  The
 *     reference accumulates with interleaved partial sums (reassoc), so
 *     agreement is at round-off level (tests use 1e-13 * sum|q|).
 *
 * Build: oracle/Makefile  ->  oracle/liboracle.so
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- (a) */

/* charges.py:130  prefix = np.cumsum(qs)  (sequential running sum) */
void or_prefix(const double *qs, int64_t n, double *prefix)
{
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        acc += qs[i];
        prefix[i] = acc;
    }
}

/* first index i in [lo, hi) with xs[i] >= v  (np.searchsorted side='left') */
static int64_t lower_bound(const double *xs, int64_t lo, int64_t hi, double v)
{
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (xs[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* charges.py:183-187  e(y) = 2 * prefix_excl[searchsorted(xs, y, 'left')] - total */
void or_sign_terms(const double *xs, const double *prefix, double total, int64_t n,
                   const double *ys, int64_t t, double *out)
{
    for (int64_t i = 0; i < t; ++i) {
        int64_t idx = lower_bound(xs, 0, n, ys[i]);
        double below = idx == 0 ? 0.0 : prefix[idx - 1];
        out[i] = 2.0 * below - total;
    }
}

/* ---------------------------------------------------------------- (b) */

typedef struct {
    int64_t n_nodes;
    int64_t capacity;
    double *lo, *hi, *center, *half;
    int64_t *level, *start, *end, *left, *right;
    int64_t depth;
    int64_t leaf_count;
} or_tree;

static int tree_reserve(or_tree *t, int64_t want)
{
    if (want <= t->capacity)
        return 0;
    int64_t cap = t->capacity ? t->capacity : 64;
    while (cap < want)
        cap *= 2;
#define GROW(f, T)                                               \
    do {                                                         \
        void *p = realloc(t->f, (size_t)cap * sizeof(T));        \
        if (!p)                                                  \
            return -1;                                           \
        t->f = (T *)p;                                           \
    } while (0)
    GROW(lo, double);
    GROW(hi, double);
    GROW(center, double);
    GROW(half, double);
    GROW(level, int64_t);
    GROW(start, int64_t);
    GROW(end, int64_t);
    GROW(left, int64_t);
    GROW(right, int64_t);
#undef GROW
    t->capacity = cap;
    return 0;
}

void or_tree_free(or_tree *t)
{
    free(t->lo);
    free(t->hi);
    free(t->center);
    free(t->half);
    free(t->level);
    free(t->start);
    free(t->end);
    free(t->left);
    free(t->right);
    memset(t, 0, sizeof(*t));
}

/*
 * tree.py:156-222 (structure part of build).  Breadth-first bisection at
 * mid = 0.5*(lo+hi); a side that would receive no sources is skipped; a node
 * is a leaf iff count <= leaf_capacity or level >= max_depth.  The child
 * slot rule "left iff child_hi == mid" (tree.py:205-208) is kept verbatim.
 * Returns 0 on success, -1 on allocation failure, -2 on empty input.
 */
int or_build(const double *xs, int64_t n, int64_t leaf_capacity, int64_t max_depth,
             or_tree *t)
{
    memset(t, 0, sizeof(*t));
    if (n <= 0)
        return -2;
    double x0 = xs[0], xl = xs[n - 1];
    double m = 1.0;
    if (fabs(x0) > m)
        m = fabs(x0);
    if (fabs(xl) > m)
        m = fabs(xl);
    double pad = 1e-12 * m;
    if (tree_reserve(t, 1))
        return -1;
    t->lo[0] = x0 - pad;
    t->hi[0] = xl + pad;
    t->level[0] = 0;
    t->start[0] = 0;
    t->end[0] = n;
    t->left[0] = -1;
    t->right[0] = -1;
    t->n_nodes = 1;
    int64_t depth = 0;
    int64_t f0 = 0, f1 = 1; /* BFS levels are contiguous index ranges */
    while (f0 < f1) {
        for (int64_t node = f0; node < f1; ++node) {
            int64_t s = t->start[node], e = t->end[node];
            if (e - s <= leaf_capacity || t->level[node] >= max_depth)
                continue;
            double lo = t->lo[node], hi = t->hi[node];
            double mid = 0.5 * (lo + hi);
            int64_t split = lower_bound(xs, s, e, mid);
            for (int side = 0; side < 2; ++side) {
                double clo = side ? mid : lo;
                double chi = side ? hi : mid;
                int64_t cs = side ? split : s;
                int64_t ce = side ? e : split;
                if (ce == cs)
                    continue;
                if (tree_reserve(t, t->n_nodes + 1))
                    return -1;
                int64_t c = t->n_nodes++;
                t->lo[c] = clo;
                t->hi[c] = chi;
                t->level[c] = t->level[node] + 1;
                t->start[c] = cs;
                t->end[c] = ce;
                t->left[c] = -1;
                t->right[c] = -1;
                if (chi == mid)
                    t->left[node] = c;
                else
                    t->right[node] = c;
                if (t->level[c] > depth)
                    depth = t->level[c];
            }
        }
        f0 = f1;
        f1 = t->n_nodes;
    }
    int64_t leaves = 0;
    for (int64_t i = 0; i < t->n_nodes; ++i) {
        t->center[i] = 0.5 * (t->lo[i] + t->hi[i]);
        t->half[i] = 0.5 * (t->hi[i] - t->lo[i]);
        if (t->left[i] < 0 && t->right[i] < 0)
            ++leaves;
    }
    t->depth = depth;
    t->leaf_count = leaves;
    return 0;
}

/* ---------------------------------------------------------------- (c) */

/*
 * tree.py:224-238: every node's moments m_k = sum_j q_j (x_j - c)^k / k!
 * computed directly from its own sources with the recursive term
 * term *= t / k.  Row-major [n_nodes][order + 1].
 */
void or_moments(const double *xs, const double *qs, int64_t n_nodes, const double *center,
                const int64_t *start, const int64_t *end, int64_t order, double *moments)
{
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t node = 0; node < n_nodes; ++node) {
        double *row = moments + node * (order + 1);
        for (int64_t k = 0; k <= order; ++k)
            row[k] = 0.0;
        double c = center[node];
        for (int64_t j = start[node]; j < end[node]; ++j) {
            double t = xs[j] - c;
            double term = qs[j];
            row[0] += term;
            for (int64_t k = 1; k <= order; ++k) {
                term *= t / (double)k;
                row[k] += term;
            }
        }
    }
}

/*
 * The same per-source terms as or_moments (term *= t / k, tree.py:235-237),
 * summed with cascade (pairwise) summation instead of the reference's
 * sequential np.add.reduceat: blocks of 64 terms are summed in order and the
 * block sums merged like a binary counter, so the summation error is
 * ~(64 + log2 n) eps instead of ~sqrt(n) eps (random walk) for a node of n
 * sources.  A more accurate yardstick than the reference's own sums for the
 * GPU's moments of large nodes (the root of configs[3] has 2^27 sources).
 */
#define OR_CASCADE_BLOCK 64
#define OR_CASCADE_LEVELS 48
void or_moments_cascade(const double *xs, const double *qs, int64_t n_nodes,
                        const double *center, const int64_t *start, const int64_t *end,
                        int64_t order, double *moments)
{
    const int64_t o1 = order + 1;
#pragma omp parallel
    {
        double *stack = (double *)calloc((size_t)(OR_CASCADE_LEVELS * o1), sizeof(double));
        double *blk = (double *)malloc(sizeof(double) * (size_t)o1);
#pragma omp for schedule(dynamic, 16)
        for (int64_t node = 0; node < n_nodes; ++node) {
            double *row = moments + node * o1;
            const double c = center[node];
            uint64_t count = 0; /* full blocks pushed so far: bit l set <=> stack[l] holds a sum */
            for (int64_t j0 = start[node]; j0 < end[node]; j0 += OR_CASCADE_BLOCK) {
                int64_t j1 = j0 + OR_CASCADE_BLOCK < end[node] ? j0 + OR_CASCADE_BLOCK : end[node];
                for (int64_t k = 0; k < o1; ++k)
                    blk[k] = 0.0;
                for (int64_t j = j0; j < j1; ++j) {
                    double t = xs[j] - c;
                    double term = qs[j];
                    blk[0] += term;
                    for (int64_t k = 1; k < o1; ++k) {
                        term *= t / (double)k;
                        blk[k] += term;
                    }
                }
                /* binary-counter merge: carry while the level is occupied */
                int lev = 0;
                while (count & ((uint64_t)1 << lev)) {
                    double *s = stack + (size_t)lev * o1;
                    for (int64_t k = 0; k < o1; ++k)
                        blk[k] = s[k] + blk[k];
                    ++lev;
                }
                memcpy(stack + (size_t)lev * o1, blk, sizeof(double) * (size_t)o1);
                ++count;
            }
            for (int64_t k = 0; k < o1; ++k)
                row[k] = 0.0;
            for (int lev = 0; lev < OR_CASCADE_LEVELS; ++lev)
                if (count & ((uint64_t)1 << lev)) {
                    const double *s = stack + (size_t)lev * o1;
                    for (int64_t k = 0; k < o1; ++k)
                        row[k] += s[k];
                }
        }
        free(blk);
        free(stack);
    }
}

/* ---------------------------------------------------------------- (d) */

/* numba cmathimpl.sqrt_impl (numpy npy_csqrt, CACM algorithm 312) for the
 * finite, not-both-zero arguments the contour loop produces. */
static void np_csqrt(double a, double b, double *re, double *im)
{
    const double thres = 0x1.a827999fcef32p+1021; /* DBL_MAX / (1 + sqrt 2) */
    int scale = 0;
    if (fabs(a) >= thres || fabs(b) >= thres) {
        a *= 0.25;
        b *= 0.25;
        scale = 1;
    }
    double r, i;
    if (a >= 0.0) {
        double t = sqrt((a + hypot(a, b)) * 0.5);
        r = t;
        i = b / (t + t);
    } else {
        double t = sqrt((hypot(a, b) - a) * 0.5);
        r = fabs(b) / (t + t);
        i = copysign(t, b);
    }
    if (scale)
        r = r + r;
    *re = r;
    *im = i;
}

/*
 * Sampled contour maximum and the p=0 bound value of the adaptive scan,
 * _kernels.py:216-225 as compiled (see file header for the fused forms).
 * Returns value = ((R * (1.1 * M)) * (h / R)) / (R - h).
 */
double or_adaptive_value(double big_r, double h, double rd2, const double *cos_tab,
                         const double *sin_tab, int64_t n_samples, double *m_out)
{
    double m_max = 0.0;
    for (int64_t t = 0; t < n_samples; ++t) {
        double wr = fma(big_r, cos_tab[t], -big_r);
        double wi = big_r * sin_tab[t];
        double wi2 = wi * wi;
        double zr = fma(wr, wr, -wi2);
        double pr = wr * wi;
        double zi = pr + pr;
        double a = zr + rd2;
        double b = zi + 0.0;
        double sr, si;
        np_csqrt(a, b, &sr, &si);
        /* CPython _Py_c_quot(z, s) */
        double re, im;
        if (fabs(sr) >= fabs(si)) {
            double ratio = si / sr;
            double denom = fma(ratio, si, sr);
            re = fma(wi, ratio, wr) / denom;
            im = fma(-wr, ratio, wi) / denom;
        } else {
            double ratio = sr / si;
            double denom = fma(ratio, sr, si);
            re = fma(wr, ratio, wi) / denom;
            im = fma(wi, ratio, -wr) / denom;
        }
        double fv = hypot(re, im);
        if (fv > m_max)
            m_max = fv;
    }
    if (m_out)
        *m_out = m_max;
    double ratio = h / big_r;
    double m1 = m_max * 1.1;
    return ((big_r * m1) * ratio) / (big_r - h);
}

/* _kernels.py:224-231: linear scan for the smallest adequate order */
int64_t or_choose_p(double big_r, double h, double rd2, double tol_share, int64_t p_cap,
                    const double *cos_tab, const double *sin_tab, int64_t n_samples)
{
    double value = or_adaptive_value(big_r, h, rd2, cos_tab, sin_tab, n_samples, 0);
    double ratio = h / big_r;
    for (int64_t cand = 0; cand < p_cap; ++cand) {
        if (value <= tol_share)
            return cand;
        value *= ratio;
    }
    return p_cap;
}

/* kernel.py:92-127 / _kernels.py:232-251: Phi^(k)(c, y), k = 0..p */
void or_phi_derivatives(double d, double rd2, int64_t p, double *deriv)
{
    double s2 = d * d + rd2;
    double sq = sqrt(s2);
    deriv[0] = d / sq;
    if (p < 1)
        return;
    deriv[1] = rd2 / (s2 * sq);
    double denom = d * s2;
    for (int64_t k = 2; k <= p; ++k) {
        double km1 = (double)(k - 1);
        double tk = (rd2 - km1 * (3.0 * d * d + rd2)) * deriv[k - 1];
        if (k >= 3)
            tk -= 3.0 * (double)((k - 1) * (k - 2)) * d * deriv[k - 2];
        if (k >= 4)
            tk -= (double)((k - 1) * (k - 2) * (k - 3)) * deriv[k - 3];
        deriv[k] = tk / denom;
    }
}

/* Interaction-list hash, ordered: h <- splitmix64(h ^ code) for every event
 * in the target's depth-first visit order (_kernels.py:204-264: pop, accept
 * -> far, else leaf -> near, else push right then left), code = node*256 +
 * p_use (far) or node*256 + 255 (near).  Two lists hash equal only if they
 * hold the same events in the same order (up to 64-bit collisions). */
static inline uint64_t mix64(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/*
 * _kernels.py:163-266 (tree_phi_sum) for targets [i0, i1).  Optional
 * instrumentation (any pointer may be NULL):
 *   hash[i]      ordered hash of the target's interaction events (visit
 *                order): far node -> node*256 + p_use, near leaf -> node*256 + 255
 *   near[i]      number of near-field (source, target) pairs
 *   nfar[i]      number of accepted far nodes
 *   sump[i]      sum of p_use over accepted far nodes
 *   np0[i]       number of accepted far nodes with p_use == 0
 */
void or_tree_phi_sum(const double *centers, const double *halves, const int64_t *starts,
                     const int64_t *ends, const int64_t *lefts, const int64_t *rights,
                     const double *moments, int64_t moment_stride, const double *xs,
                     const double *qs, double rd2, double theta, int64_t p, int adaptive,
                     double tol_share, int64_t p_cap, const double *cos_tab,
                     const double *sin_tab, int64_t n_samples, const double *ys, double *out,
                     int64_t i0, int64_t i1, uint64_t *hash, int64_t *near, int64_t *nfar,
                     int64_t *sump, int64_t *np0)
{
#pragma omp parallel
    {
        double *deriv = (double *)malloc(sizeof(double) * (size_t)(p_cap + 1 > p + 1 ? p_cap + 1 : p + 1));
        int64_t stack[160];
#pragma omp for schedule(static)
        for (int64_t i = i0; i < i1; ++i) {
            double y = ys[i];
            double acc = 0.0;
            uint64_t hh = 0;
            int64_t c_near = 0, c_far = 0, c_sump = 0, c_p0 = 0;
            int top = 0;
            stack[0] = 0;
            while (top >= 0) {
                int64_t node = stack[top--];
                double c = centers[node];
                double h = halves[node];
                double d = c - y;
                double big_r = fabs(d);
                if (big_r > 0.0 && h <= theta * big_r) {
                    int64_t p_use = p;
                    if (adaptive)
                        p_use = or_choose_p(big_r, h, rd2, tol_share, p_cap, cos_tab, sin_tab,
                                            n_samples);
                    or_phi_derivatives(d, rd2, p_use, deriv);
                    const double *mrow = moments + node * moment_stride;
                    for (int64_t k = 0; k <= p_use; ++k)
                        acc += deriv[k] * mrow[k];
                    hh = mix64(hh ^ ((uint64_t)node * 256u + (uint64_t)p_use));
                    ++c_far;
                    c_sump += p_use;
                    if (p_use == 0)
                        ++c_p0;
                } else if (lefts[node] < 0 && rights[node] < 0) {
                    for (int64_t j = starts[node]; j < ends[node]; ++j) {
                        double dd = xs[j] - y;
                        acc += qs[j] * dd / sqrt(dd * dd + rd2);
                    }
                    hh = mix64(hh ^ ((uint64_t)node * 256u + 255u));
                    c_near += ends[node] - starts[node];
                } else {
                    if (rights[node] >= 0)
                        stack[++top] = rights[node];
                    if (lefts[node] >= 0)
                        stack[++top] = lefts[node];
                }
            }
            out[i] = acc;
            if (hash)
                hash[i] = hh;
            if (near)
                near[i] = c_near;
            if (nfar)
                nfar[i] = c_far;
            if (sump)
                sump[i] = c_sump;
            if (np0)
                np0[i] = c_p0;
        }
        free(deriv);
    }
}

/* ---------------------------------------------------------------- (f) */

/* _kernels.py:49-59 phi_sum_plain (ascending j, plain accumulation) */
void or_phi_sum_plain(const double *xs, const double *qs, int64_t n, const double *ys,
                      double rd2, double *out, int64_t i0, int64_t i1)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = i0; i < i1; ++i) {
        double y = ys[i];
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double d = xs[j] - y;
            acc += qs[j] * d / sqrt(d * d + rd2);
        }
        out[i] = acc;
    }
}

/* _kernels.py:145-160 phi_sum_kahan (strict ascending order, compensated) */
void or_phi_sum_kahan(const double *xs, const double *qs, int64_t n, const double *ys,
                      double rd2, double *out, int64_t i0, int64_t i1)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = i0; i < i1; ++i) {
        double y = ys[i];
        double acc = 0.0, comp = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double d = xs[j] - y;
            double term = qs[j] * d / sqrt(d * d + rd2);
            double tt = term - comp;
            double s = acc + tt;
            comp = (s - acc) - tt;
            acc = s;
        }
        out[i] = acc;
    }
}

int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0)
        omp_set_num_threads(n);
#else
    (void)n;
#endif
}
