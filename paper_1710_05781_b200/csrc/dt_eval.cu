// (d)+(e) Tree field evaluation: warp-coherent traversal, far field with
// adaptive truncation order, near field by direct summation.
//
// Reference: _kernels.py:163-266 (tree_phi_sum), the numba kernel behind
// evaluate_all (tree.py:318-373).  Per target the reference walks the tree
// depth-first (left subtree first): a node with R = |c - y| > 0 and
// h <= theta*R contributes sum_k Phi^(k)(c, y) m_k, k <= p_use (Eq. 10
// recurrence); an unaccepted leaf contributes its direct pair sum; anything
// else descends.
//
// B200 mapping: one warp owns 32 consecutive (sorted) targets and walks the
// UNION of their traversals with a per-entry lane mask (an opened node
// continues into its first child; pending right siblings sit on a per-warp
// stack in shared memory).  Each lane applies the reference's MAC to its own
// target, so the per-target interaction lists -- and their DFS order -- are
// exactly the reference's.  Warps pull 32-target tasks from per-SM segments
// of the target range (persistent grid, 148 x 4 CTAs), so the warps of an SM
// share node records and moment rows in L1.
//   far   accepting lanes evaluate the recurrence together up to the warp's
//         largest order; the moment row is a broadcast load.
//   near  lanes that reach an unaccepted leaf sum its (x, q) pairs, read as
//         one broadcast 16-byte load per source; rsqrt = MUFU seed + one
//         cubic Newton step.
// Adaptive order (reference lines 212-231): the reference samples
// |f| = |w / sqrt(w^2 + r_d^2)| at 64 contour points per accepted pair with
// complex arithmetic.  On the contour |f|^4 = 1 / ((1 - s*/s_t)^2 + s*) with
// s_t = |e^{i theta_t} - 1|^2 and s* = r_d^2 / R^2, unimodal in t, so the
// sampled maximum sits at the samples bracketing s_t = s*.  Tier 1 evaluates
// that closed form in fp32 and solves the bound scan for p directly in
// log2 space; when log2(value_p / tol) lies within PSEL_MARGIN_LOG2 of 0 at
// the candidate order, tier 2 re-runs the reference's exact double-precision
// operation sequence (numpy csqrt, CPython complex quotient, glibc's
// hypot, the fused forms LLVM emitted) on the bracketing samples and their
// mirrors, and tier 3 (tiny s*, out-of-range inputs or DT_PSEL_EXACT) on all
// samples.  The chosen orders are bit-identical to the reference's.
#include <stdlib.h>

#include <algorithm>

#include "dt_common.cuh"
#include "dt_farcoef.cuh"

namespace {

#ifndef DT_EVAL_MINB
#define DT_EVAL_MINB 2
#endif
#ifndef DT_EVAL_THREADS
#define DT_EVAL_THREADS 512  // 2 x 512 per SM: one order-table copy per 16 warps (10.35 against 10.38 ms at 4 x 256)
#endif
#ifndef DT_EVAL_SEGMENTS
#define DT_EVAL_SEGMENTS 148  // per-SM task segments (0: one global counter)
#endif
static_assert(DT_EVAL_SEGMENTS * 4 <= DT_EVAL_COUNTER_BYTES, "counter slot too small");
#ifndef DT_EVAL_UTIL
#define DT_EVAL_UTIL 0  // development: lane-utilisation counters (variant builds only)
#endif
#if DT_EVAL_UTIL
__device__ unsigned long long g_util[16];
#define UTIL_ADD(k, v) u_[k] += (unsigned long long)(v)
#else
#define UTIL_ADD(k, v) ((void)0)
#endif
constexpr int EVAL_THREADS = DT_EVAL_THREADS;
constexpr int64_t FIELD_TILE = 1024;  // targets per sign-term bracket (dt_tree_field_packed)
constexpr int EVAL_WARPS = EVAL_THREADS / 32;
constexpr int MAX_SAMPLES = 256;
constexpr float PSEL_MARGIN_LOG2 = 2e-4f;  // ambiguity band of log2(value_n / tol)
constexpr double CONTOUR_SAFETY = 1.1;  // kernel.py:27

struct EvalArgs {
    const dt_node *nodes;
    int64_t n_nodes;
    const double *moments;
    int64_t stride;
    const double2 *xq;
    double rd2, theta;
    int p;
    int p_cap;
    double tol_share;
    const double *cos_tab, *sin_tab;
    int n_samples;
    const double *ys;
    double *out;
    int64_t i0, i1;
    int accumulate;
    int psel_mode;
    dt_eval_stats stats;
    unsigned long long *counter;
    // fused field E = e + phi (dt_tree_field_packed): sign term from the
    // sorted sources and their prefix sums; vflags[0] counts non-finite targets
    const double *sign_xs, *sign_prefix;
    int64_t sign_n;
    int64_t *vflags;
    // optional: lower_bound of every FIELD_TILE-th target (and of the last),
    // bracketing the search of the targets in between when they are sorted
    const int64_t *sign_bracket;
    const int64_t *meta;  // if set: tol_share = tolerance / (3 max(depth, 1)) on device
    double tolerance;
    // order-selection tables in the workspace slot (built per call), or null
    const double *pt_bp;
    const unsigned char *pt_bins;
};

// tree.py:268-270 _tol_share, evaluated from the device-side tree depth.
__device__ __forceinline__ double tol_share_of(const EvalArgs &a)
{
    if (!a.meta)
        return a.tol_share;
    const int64_t depth = __ldg(a.meta + DT_META_DEPTH);
    return __ddiv_rn(a.tolerance, __dmul_rn(3.0, (double)(depth > 1 ? depth : 1)));
}

// ------------------------------------------------------------------ exact tier

// hypot(a, b): the corrected algorithm of C. F. Borges, "An improved
// algorithm for hypot(a, b)" (2019), non-FMA variant -- what glibc 2.35+
// libm computes on x86-64 (checked bit-for-bit against glibc 2.39 on 2e7
// random pairs, including near-equal arguments).  The reference reaches it
// through numba's abs(complex) and cmath.sqrt.  Arguments in this kernel
// are far from the overflow/underflow ranges where libm rescales.
__device__ double dt_hypot(double a, double b)
{
    double ax = fabs(a), ay = fabs(b);
    if (ax < ay) {
        double t = ax;
        ax = ay;
        ay = t;
    }
    if (ay <= __dmul_rn(ax, 0x1p-54))
        return __dadd_rn(ax, ay);
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay),
                       __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

// numpy npy_csqrt / numba cmathimpl.sqrt_impl (CACM 312), finite inputs.
__device__ void np_csqrt(double a, double b, double *re, double *im)
{
    const double thres = 0x1.a827999fcef32p+1021;
    bool scale = false;
    if (fabs(a) >= thres || fabs(b) >= thres) {
        a = __dmul_rn(a, 0.25);
        b = __dmul_rn(b, 0.25);
        scale = true;
    }
    double r, i;
    double hyp = dt_hypot(a, b);
    if (a >= 0.0) {
        double t = __dsqrt_rn(__dmul_rn(__dadd_rn(a, hyp), 0.5));
        r = t;
        i = __ddiv_rn(b, __dadd_rn(t, t));
    } else {
        double t = __dsqrt_rn(__dmul_rn(__dsub_rn(hyp, a), 0.5));
        r = __ddiv_rn(fabs(b), __dadd_rn(t, t));
        i = copysign(t, b);
    }
    if (scale)
        r = __dadd_rn(r, r);
    *re = r;
    *im = i;
}

// |f| at one contour sample, exactly as the compiled reference computes it.
__device__ double contour_sample(double big_r, double c, double s, double rd2)
{
    double wr = __fma_rn(big_r, c, -big_r);
    double wi = __dmul_rn(big_r, s);
    double wi2 = __dmul_rn(wi, wi);
    double zr = __fma_rn(wr, wr, -wi2);
    double pr = __dmul_rn(wr, wi);
    double zi = __dadd_rn(pr, pr);
    double a = __dadd_rn(zr, rd2);
    double b = __dadd_rn(zi, 0.0);
    double sr, si;
    np_csqrt(a, b, &sr, &si);
    double re, im;
    if (fabs(sr) >= fabs(si)) {
        double ratio = __ddiv_rn(si, sr);
        double denom = __fma_rn(ratio, si, sr);
        re = __ddiv_rn(__fma_rn(wi, ratio, wr), denom);
        im = __ddiv_rn(__fma_rn(-wr, ratio, wi), denom);
    } else {
        double ratio = __ddiv_rn(sr, si);
        double denom = __fma_rn(ratio, sr, si);
        re = __ddiv_rn(__fma_rn(wr, ratio, wi), denom);
        im = __ddiv_rn(__fma_rn(wi, ratio, -wr), denom);
    }
    return dt_hypot(re, im);
}

// value -> order scan (reference lines 224-231, value reassociated as compiled)
__device__ int exact_scan(double m_max, double big_r, double h, double tol, int p_cap)
{
    double ratio = __ddiv_rn(h, big_r);
    double m1 = __dmul_rn(m_max, CONTOUR_SAFETY);
    double value = __ddiv_rn(__dmul_rn(__dmul_rn(big_r, m1), ratio), __dsub_rn(big_r, h));
    for (int cand = 0; cand < p_cap; ++cand) {
        if (value <= tol)
            return cand;
        value = __dmul_rn(value, ratio);
    }
    return p_cap;
}

__device__ int psel_exact_all(double big_r, double h, const EvalArgs &a, const double *cs,
                              const double *sn)
{
    double m = 0.0;
    for (int t = 0; t < a.n_samples; ++t) {
        double fv = contour_sample(big_r, cs[t], sn[t], a.rd2);
        if (fv > m)
            m = fv;
    }
    return exact_scan(m, big_r, h, a.tol_share, a.p_cap);
}

__device__ int psel_exact_bracket(double big_r, double h, int t0, const EvalArgs &a,
                                  const double *cs, const double *sn)
{
    double m = 0.0;
#pragma unroll 1
    for (int c = -1; c <= 2; ++c) {
        int t = min(max(t0 + c, 1), 32);
        double fv = contour_sample(big_r, cs[t], sn[t], a.rd2);
        if (fv > m)
            m = fv;
        int tm = 64 - t;
        if (tm != t) {
            fv = contour_sample(big_r, cs[tm], sn[tm], a.rd2);
            if (fv > m)
                m = fv;
        }
    }
    return exact_scan(m, big_r, h, a.tol_share, a.p_cap);
}

// ------------------------------------------------------------------ fast tier

// MUFU reciprocal (rcp.approx.ftz.f32, ~1 ulp): the order estimate's error
// budget absorbs it; IEEE division would cost a Newton step and a fixup.
// double -> float, round to nearest (one F2F; a subnormal result is kept and
// the ftz arithmetic that follows reads it as 0, which the range guards catch)
__device__ __forceinline__ float f32_of(double x)
{
    float r;
    asm("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(x));
    return r;
}

__device__ __forceinline__ float fast_rcp(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// log2(x) = e + f for normal x > 0, f = log2(mantissa) in [0, 1) (MUFU.LG2,
// absolute error ~2^-22 on [1, 2)).
__device__ __forceinline__ void split_log2(float x, int *e, float *f)
{
    int bits = __float_as_int(x);
    *e = ((bits >> 23) & 0xff) - 127;
    *f = __log2f(__int_as_float((bits & 0x007fffff) | 0x3f800000));
}

// Returns p >= 0 on a confident decision, or -(t0 + 2) (<= -2) when the
// decision is within the margin (tier 2 with bracket t0), or -1 for tier 3.
// The decision is the sign of resid = log2(value_n / tol) at the candidate
// n; its absolute error (log2 units) is below 5e-5: MUFU.LG2 (2 ulp of a
// result below 128, /4 for the contour term; 2^-22 for the mantissa of
// ratio), fp32 rounding of the few sums of magnitude < 128, (n + 1) <= 32
// times the log2 error of the fp32 ratio (~3e-7).  PSEL_MARGIN_LOG2 = 2e-4
// is 4x that; inside it the exact replica decides.
// s* = r_d^2/R^2 >= 4 puts every sample below the peak of |f| (maximum at
// t = 32, the far side of the contour) and s* <= s_1 puts every sample above
// it (maximum at t = 1); only in between is the bracket located (asin).
__device__ int psel_fast(double big_r, double h, const EvalArgs &a, const float *isig,
                         float rd2f, float log_c)
{
    // h == 0 (a node of coincident sources) gives ratio 0, which the range
    // guard sends to the exact replica (value 0 there, p = 0)
    const float Rf = f32_of(big_r);
    const float hf = f32_of(h);
    const float iR = fast_rcp(Rf);
    const float ratio = hf * iR;
    const float sstar = rd2f * iR * iR;
    // one combined range guard (out of range -> exact tier 3)
    if (!(Rf > 1e-15f && Rf < 1e15f && ratio > 1e-30f && sstar > 1e-12f && sstar < 1e30f))
        return -1;
    int t0;
    float emin;
    if (sstar >= 4.0f) {
        t0 = 32;
        const float u = sstar * 0.25f;
        emin = (1.0f - u) * (1.0f - u);
    } else if (sstar <= isig[34]) {
        t0 = 0;
        const float u = sstar * isig[1];
        emin = (1.0f - u) * (1.0f - u);
    } else {
        // bracket: s_t = 4 sin^2(pi t / 64) = s*  ->  t* = (64/pi) asin(sqrt(s*)/2);
        // asin via Abramowitz-Stegun 4.4.45 (|err| < 7e-5 rad).  The sampled
        // maximum is at t0 or t0 + 1 (a t* error of ~1e-3 samples can only
        // swap in the sample sitting on the peak, which then wins).
        const float z = 0.5f * sstar * rsqrtf(sstar);
        const float om = 1.0f - z;
        const float poly = fmaf(fmaf(fmaf(-0.0187293f, z, 0.0742610f), z, -0.2121144f), z,
                                1.5707288f);
        const float asz = 1.57079633f - om * rsqrtf(fmaxf(om, 1e-30f)) * poly;
        t0 = (int)(asz * 20.371832715762604f);
        const int ta = max(t0, 1), tb = min(t0 + 1, 32);
        const float ua = sstar * isig[ta], ub = sstar * isig[tb];
        emin = fminf((1.0f - ua) * (1.0f - ua), (1.0f - ub) * (1.0f - ub));
    }
    // log2(value_0 / tol) = log2(1.1 / tol) + log2 M + log2 ratio - log2(1 - ratio),
    // log2 M = -log2(emin + s*) / 4 (the sampled contour maximum of |f|).
    // log2 ratio = er + fr keeps its integer part exact: it is multiplied by
    // the candidate order below.
    int er;
    float fr;
    split_log2(ratio, &er, &fr);
    const float lx = (fmaf(-0.25f, __log2f(emin + sstar), log_c) - __log2f(1.0f - ratio)) + fr;
    const float L = -((float)er + fr);         // -log2(ratio) > 0
    const float iL = fast_rcp(L);
    // candidate order, clamped to [-1, p_cap]: outside, the decision below
    // gives 0 resp. p_cap and never reports an ambiguity
    const float pstar_approx =
        fminf(fmaxf((lx + (float)er) * iL, -1.0f), (float)a.p_cap);
    const int n = __float2int_rn(pstar_approx);
    // residual log2(value_n / tol) = lx + (n + 1) er + n fr, integer part exact
    const float resid = fmaf((float)n, fr, lx) + (float)((n + 1) * er);
    if (fabsf(resid) < PSEL_MARGIN_LOG2 && n >= 0 && n <= a.p_cap - 1)
        return -(t0 + 2);
    const int p = max(resid > 0.0f ? n + 1 : n, 0);  // value_n > tol: one more order
    return min(p, a.p_cap);
}

// ------------------------------------------------------------ order table
//
// For n >= PT_MIN_N the bound value V_n(R) = 1.1 M(R) R (h/R)^(n+1) / (R - h)
// of a node of half-width h decreases strictly in R: on the reference's
// 64-point contour d ln M / d ln R <= 5.6 (dense scan of s* = r_d^2/R^2),
// while the rest falls at least as fast as R^-(n+1), so the slope of ln V_n
// in ln R is <= -1.4.  "V_n <= tol" is then "R >= b_n", one breakpoint per
// (level, n): the nodes of level L have the half-width h_L = h0 2^-L up to
// a relative PT_DH (interval rounding).  The bins partition R per level by
// the bits of R itself: bin j holds the R whose high word lies in
// [hi(h_L) + (j + jbase) 2^13, hi(h_L) + (j + jbase + 1) 2^13) -- 128 bins
// per binade, a monotone, integer-only function of R (no logarithms in the
// traversal).  With x = log2(R/h_L), the breakpoints x_n = log2(b_n / h_L)
// make each bin
//   clean (no x_n within PT_ETA of the bin's x-range): the bin's constant p;
//   one-breakpoint: p = m or m + 1 by comparing R with b_m in double;
//   anything else (two breakpoints, p <= PT_MIN_N possible): psel_fast.
// A node's level comes from the bits of its h as well,
// L = (hi(h0) - hi(h) + 2^19) >> 20, and a level whose nodes do not all have
// |h - h_L| <= PT_DH h_L (scanned when the tables are built) gets no table.
// PT_ETA covers the level's spread of h (which moves a breakpoint in x by
// < 1e-5); the double comparison keeps a relative margin PT_EPS >=
// (31 + 2) PT_DH / 1.4 (the spread's effect in R) plus the bisection
// tolerance, else psel_fast decides.
constexpr int PT_LEVELS = 61;  // levels 0..max_depth
constexpr int PT_N = 32;       // n = 0..31 (p_cap <= 31)
constexpr int PT_MIN_N = 6;
constexpr int PT_BINS = 512;   // per level: four binades of R from just below h_L / theta
constexpr double PT_DH = 1e-6;
constexpr double PT_EPS = 3e-5;
constexpr double PT_ETA = 5e-5;
constexpr unsigned char PT_FALLBACK = 0xff, PT_SPLIT = 0x80;

// log V_n(R) in double, the contour maximum over the reference's 64
// samples (one warp: lane l holds samples l and l + 32, then a max
// reduction); lh = log h
struct LaneSamples {
    double c0, s0, c1, s1;
};

__device__ double log_bound_value(double R, double h, double lh, int n, double rd2,
                                  const LaneSamples &q)
{
    double m2;  // max |f|^2
    {
        const double wr = R * (q.c0 - 1.0), wi = R * q.s0;
        const double zr = wr * wr - wi * wi + rd2, zi = 2.0 * wr * wi;
        m2 = (wr * wr + wi * wi) / sqrt(zr * zr + zi * zi);
    }
    {
        const double wr = R * (q.c1 - 1.0), wi = R * q.s1;
        const double zr = wr * wr - wi * wi + rd2, zi = 2.0 * wr * wi;
        m2 = fmax(m2, (wr * wr + wi * wi) / sqrt(zr * zr + zi * zi));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        m2 = fmax(m2, __shfl_xor_sync(DT_FULL, m2, o));
    const double lr = log(R);
    return log(1.1) + 0.5 * log(m2) + lr + (double)(n + 1) * (lh - lr) - log(R - h);
}

// jbase: bin 0 starts below every far R of a level.  With blog(v) = e + m - 1
// for v = 2^e m (1 <= m < 2), log2(v) - 0.0861 <= blog(v) <= log2(v), so
// (hi(R) - hi(h_L)) / 2^20 = blog(R) - blog(h_L) >= log2(R / h_L) - 0.0861 and
// R >= h / theta >= h_L (1 - PT_DH) / theta.
__host__ __device__ inline int pt_jbase(double theta)
{
    return (int)floor(128.0 * (log2(1.0 / theta) - 0.0862)) - 1;
}

// the level of a node of half-width h from the bits of h (h0: the root's)
__device__ __forceinline__ int pt_level(int hi0, double h)
{
    return (hi0 - __double2hiint(h) + 0x80000) >> 20;
}

// The breakpoints depend only on the inputs below; they are kept in the
// workspace slot with this key and rebuilt only when it changes (the
// regula falsi is ~45 us; a device-resident step repeats the same tree
// depth, root half-width, r_d, tolerance and tables).
struct PtKey {
    unsigned long long magic, h0, rd2, tol, theta, tables;
    long long p_cap, used_depth, n_samples;
    unsigned long long bp_hash;  // the breakpoint table's content (the slot may be reused)
};
constexpr int PT_BP_WORDS = 2 * PT_LEVELS * PT_N + PT_LEVELS;

// Order-independent 64-bit hash of the breakpoint table, by the whole block.
__device__ unsigned long long pt_bp_hash(const double *bp)
{
    __shared__ unsigned long long part_s[32];
    unsigned long long h = 0;
    for (int i = threadIdx.x; i < PT_BP_WORDS; i += blockDim.x) {
        unsigned long long z = (unsigned long long)__double_as_longlong(__ldcg(bp + i)) +
                               0x9e3779b97f4a7c15ull * (unsigned long long)(i + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        h += z ^ (z >> 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        h += __shfl_xor_sync(DT_FULL, h, o);
    if (dt_lane() == 0)
        part_s[threadIdx.x >> 5] = h;
    __syncthreads();
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        t += part_s[w];
    __syncthreads();
    return t;
}
constexpr unsigned long long PT_KEY_MAGIC = 0x6474707472656531ull;

__device__ PtKey pt_key_of(const EvalArgs &a)
{
    PtKey k;
    k.magic = PT_KEY_MAGIC;
    k.h0 = (unsigned long long)__double_as_longlong(__ldg(&a.nodes[0].half));
    k.rd2 = (unsigned long long)__double_as_longlong(a.rd2);
    k.tol = (unsigned long long)__double_as_longlong(a.meta ? tol_share_of(a) : a.tol_share);
    k.theta = (unsigned long long)__double_as_longlong(a.theta);
    unsigned long long f = 0x9e3779b97f4a7c15ull;  // fingerprint of the contour tables
    for (int t = 0; t < a.n_samples; ++t) {
        f = (f ^ (unsigned long long)__double_as_longlong(__ldg(a.cos_tab + t))) * 0x100000001b3ull;
        f = (f ^ (unsigned long long)__double_as_longlong(__ldg(a.sin_tab + t))) * 0x100000001b3ull;
    }
    k.tables = f;
    k.p_cap = a.p_cap;
    k.used_depth = a.meta ? __ldg(a.meta + DT_META_DEPTH) : -1;
    k.n_samples = a.n_samples;
    return k;
}

__device__ __forceinline__ bool pt_key_equal(const PtKey &x, const PtKey &y)
{
    return x.magic == y.magic && x.h0 == y.h0 && x.rd2 == y.rd2 && x.tol == y.tol &&
           x.theta == y.theta && x.tables == y.tables && x.p_cap == y.p_cap &&
           x.used_depth == y.used_depth && x.n_samples == y.n_samples && x.bp_hash == y.bp_hash;
}

// bp[L][n] = b_n for h_L: the R with V_n(R) = tol_share (h_L / theta if V_n
// <= tol there already, +inf if never); 0 for n >= p_cap (the reference's
// loop stops there).  One warp per entry.  First, a grid-stride scan of the
// nodes sets bad[L] for every level L = pt_level(h) holding a node with
// |h - h_L| > PT_DH h_L (or lying below the tree's depth, where no
// breakpoints are computed); bad[] is zeroed by the caller.
__global__ void psel_breakpoints_kernel(EvalArgs a, double *bp, unsigned *bad, const PtKey *key)
{
    {
        const double h0 = __ldg(&a.nodes[0].half);
        const int hi0 = __double2hiint(h0);
        const int64_t nn = a.meta ? __ldg(a.meta + DT_META_NODES) : a.n_nodes;
        const int64_t dep = a.meta ? __ldg(a.meta + DT_META_DEPTH) : PT_LEVELS - 1;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn;
             i += (int64_t)gridDim.x * blockDim.x) {
            const double h = __ldg(&a.nodes[i].half);
            const int L = pt_level(hi0, h);
            if ((unsigned)L < (unsigned)PT_LEVELS &&
                (L > dep || !(fabs(h - ldexp(h0, -L)) <= PT_DH * ldexp(h0, -L))))
                atomicOr(bad + L, 1u);
        }
    }
    {
        // tables from an earlier call with the same key are still valid
        __shared__ int same_s;
        const unsigned long long hbp = pt_bp_hash(bp);
        if (threadIdx.x == 0) {
            PtKey cur = pt_key_of(a);
            cur.bp_hash = hbp;
            same_s = pt_key_equal(cur, *key);
        }
        __syncthreads();
        if (same_s)
            return;
    }
    const int id = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (id >= PT_LEVELS * PT_N)
        return;
    const int L = id / PT_N, n = id % PT_N;
    const double tol = a.meta ? tol_share_of(a) : a.tol_share;
    const double h = ldexp(__ldg(&a.nodes[0].half), -L);
    // levels below the tree's depth (when known) hold no nodes
    const bool used = !a.meta || L <= __ldg(a.meta + DT_META_DEPTH);
    double b = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    if (n >= a.p_cap) {
        b = 0.0;
    } else if (used && n >= PT_MIN_N && h > 0.0) {
        // F(u) = ln V_n(e^u) - ln tol falls with slope in [-38, -1.4]:
        // F(u0) / 1.4 past u0 = ln(h/theta) brackets the root; then
        // regula falsi with the Illinois modification
        const double lt = log(tol), lh = log(h);
        const int l = dt_lane();
        const LaneSamples q{__ldg(a.cos_tab + l), __ldg(a.sin_tab + l), __ldg(a.cos_tab + l + 32),
                            __ldg(a.sin_tab + l + 32)};
        const double rmin = h / a.theta;
        double ulo = log(rmin);
        double flo = log_bound_value(rmin, h, lh, n, a.rd2, q) - lt;
        if (!(flo > 0.0)) {
            b = rmin;
        } else if (flo < 1e4) {
            double uhi = ulo + flo / 1.4;
            double fhi = log_bound_value(exp(uhi), h, lh, n, a.rd2, q) - lt;
            int side = 0;
            for (int it = 0; it < 100 && uhi - ulo > 1e-10; ++it) {
                double um = (ulo * fhi - uhi * flo) / (fhi - flo);
                if (!(um > ulo && um < uhi))
                    um = 0.5 * (ulo + uhi);
                const double fm =
                    log_bound_value(exp(um), h, lh, n, a.rd2, q) - lt;
                if (fm > 0.0) {
                    ulo = um;
                    flo = fm;
                    if (side == 1)
                        fhi *= 0.5;
                    side = 1;
                } else {
                    uhi = um;
                    fhi = fm;
                    if (side == -1)
                        flo *= 0.5;
                    side = -1;
                }
            }
            b = exp(uhi) * (1.0 + 1e-12);  // on the V_n <= tol side
        }
    }
    if (dt_lane() == 0) {
        bp[id] = b;
        // x_n = log2(b_n / h_L) for the bins (-huge for b_n = 0)
        bp[PT_LEVELS * PT_N + PT_LEVELS + id] = b > 0.0 ? log2(b / h) : -1e300;
        if (n == 0)
            bp[PT_LEVELS * PT_N + L] = h;  // h_L
    }
}

// A bin's order without any monotonicity in R (used where p <= PT_MIN_N is
// possible): the reference's p is the smallest n < p_cap with V_n(R) <= tol
// (else p_cap), and V_n(R) = V_0(R) (h/R)^n falls with n, so p is constant
// on [rlo, rhi] if V_p <= tol and V_(p-1) > tol hold on the whole bin.  Bounds
// of ln V_n = ln 1.1 + ln M(R) + (n+1) ln h - n ln R - ln(R - h) over the bin
// (h within PT_DH of h_L): ln M at the bin's centre +- PT_LIPM times the
// half-width in ln R (|d ln M / d ln R| <= 5.61 on the 64-point contour over
// 14 decades of R / r_d), the other terms at the bin's ends.  A margin of 1e-9
// covers round-off in the reference's value.  PT_FALLBACK if undecided.
constexpr double PT_LIPM = 7.0;
__device__ unsigned char psel_bin_interval(const EvalArgs &a, double rlo, double rhi, double hL)
{
    const double hmin = hL * (1.0 - PT_DH), hmax = hL * (1.0 + PT_DH);
    if (!(rlo > 2.0 * hmax))
        return PT_FALLBACK;
    const double rc = sqrt(rlo * rhi);
    double m2 = 0.0;
    for (int t = 0; t < 64; ++t) {
        const double wr = rc * (__ldg(a.cos_tab + t) - 1.0), wi = rc * __ldg(a.sin_tab + t);
        const double zr = wr * wr - wi * wi + a.rd2, zi = 2.0 * wr * wi;
        m2 = fmax(m2, (wr * wr + wi * wi) / sqrt(zr * zr + zi * zi));
    }
    const double lrlo = log(rlo), lrhi = log(rhi);
    const double slack = PT_LIPM * 0.5 * (lrhi - lrlo) + 1e-12;
    const double lm = 0.5 * log(m2);
    const double lt = log(a.meta ? tol_share_of(a) : a.tol_share), c = log(1.1), mg = 1e-9;
    // upper / lower bounds of ln V_n - ln tol, n = 0, 1, ...
    const double up0 = c + lm + slack + log(hmax) - log(rlo - hmax) - lt;
    const double lo0 = c + lm - slack + log(hmin) - log(rhi - hmin) - lt;
    const double dup = log(hmax) - lrlo, dlo = log(hmin) - lrhi;  // d/dn, both < 0
    for (int n = 0; n < a.p_cap; ++n) {
        if (up0 + n * dup < -mg)  // V_n <= tol on the whole bin
            return (n == 0 || lo0 + (n - 1) * dlo > mg) ? (unsigned char)n : PT_FALLBACK;
        if (!(lo0 + n * dlo > mg))  // V_n may fall to tol inside the bin
            return PT_FALLBACK;
    }
    return (unsigned char)a.p_cap;  // V_n > tol for every n < p_cap
}

// bins[L][j]: the order of bin j, PT_SPLIT | m for a bin holding b_m only,
// PT_FALLBACK otherwise
__global__ void psel_bins_kernel(EvalArgs a, const double *bp, const unsigned *bad,
                                 unsigned char *bins, PtKey *key)
{
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.x == 0) {  // the breakpoints now match this key (stream order)
        const unsigned long long hbp = pt_bp_hash(bp);
        if (threadIdx.x == 0) {
            PtKey k = pt_key_of(a);
            k.bp_hash = hbp;
            *key = k;
        }
    }
    if (id >= PT_LEVELS * PT_BINS)
        return;
    const int L = id / PT_BINS, j = id % PT_BINS;
    const double hL = bp[PT_LEVELS * PT_N + L];
    const double *xs = bp + PT_LEVELS * PT_N + PT_LEVELS + L * PT_N;
    // the bin's R-range: high words hiL + (j + jbase) 2^13 .. + 2^13 (exact
    // doubles); the traversal's hiL = hi(h0) - (L << 20) must be hL's high
    // word (no subnormals) and hL must share h0's low word
    const double h0 = __ldg(&a.nodes[0].half);
    const int hiL = __double2hiint(h0) - (L << 20);
    const int jb = pt_jbase(a.theta) + j;
    const bool exact_level = hL > 0.0 && __double2hiint(hL) == hiL &&
                             __double2loint(hL) == __double2loint(h0) && bad[L] == 0;
    const double rlo = __hiloint2double(hiL + (jb << 13), 0);
    const double rhi = __hiloint2double(hiL + ((jb + 1) << 13), 0);
    const double xlo = log2(rlo / hL) - PT_ETA, xhi = log2(rhi / hL) + PT_ETA;
    unsigned char e = PT_FALLBACK;
    // x_n = log2(b_n / h_L), decreasing in n; p <= PT_MIN_N is possible once
    // x reaches x_(PT_MIN_N)
    const double x6 = xs[PT_MIN_N];
    if (exact_level && xhi < x6) {
        int inside = 0, m = -1, p = a.p_cap;
        for (int n = PT_MIN_N + 1; n < a.p_cap; ++n) {
            const double xn = xs[n];
            if (xn >= xlo && xn <= xhi) {
                ++inside;
                m = n;
            } else if (xn < xlo && p == a.p_cap) {
                p = n;  // first n whose breakpoint lies below the bin
            }
        }
        if (inside == 0)
            e = (unsigned char)p;
        else if (inside == 1)
            e = (unsigned char)(PT_SPLIT | m);
    }
    if (e == PT_FALLBACK && exact_level && a.n_samples == 64)
        e = psel_bin_interval(a, rlo, rhi, hL);
    bins[id] = e;
}

// the workspace slot: task counters and the bad-level flags (zeroed per
// call), then the tables
constexpr size_t PT_BAD_OFFSET = 768, PT_BP_OFFSET = 1024, PT_BINS_OFFSET = 32768;
static_assert(DT_EVAL_SEGMENTS * 4 <= PT_BAD_OFFSET && PT_BAD_OFFSET + 4 * PT_LEVELS <= PT_BP_OFFSET,
              "counter slot layout");
static_assert(PT_BP_OFFSET + sizeof(double) * (2 * PT_LEVELS * PT_N + PT_LEVELS) <= PT_BINS_OFFSET,
              "breakpoint table overlaps the bins");
constexpr size_t PT_KEY_OFFSET = PT_BINS_OFFSET + PT_LEVELS * PT_BINS;
static_assert(PT_KEY_OFFSET % 8 == 0 && PT_KEY_OFFSET + sizeof(PtKey) <= DT_EVAL_COUNTER_BYTES,
              "key slot");
static_assert(PT_BINS_OFFSET + PT_LEVELS * PT_BINS <= DT_EVAL_COUNTER_BYTES,
              "order tables exceed the workspace slot");

// p from the bins, or -1 (use psel_fast): integer arithmetic on the high
// words of R and h (hi0 = hi(h0), jbase = pt_jbase(theta)), one shared-memory
// byte, at most one double comparison
__device__ __forceinline__ int psel_table(double R, int hiR, double h, unsigned bins,
                                          const double *bp, int hi0, int jbase)
{
    const int L = pt_level(hi0, h);
    const int j = ((hiR - (hi0 - (L << 20))) >> 13) - jbase;
    if (!((unsigned)L < (unsigned)PT_LEVELS && (unsigned)j < (unsigned)PT_BINS))
        return -1;
    unsigned e;
    asm("ld.shared.u8 %0, [%1];" : "=r"(e) : "r"(bins + (unsigned)(L * PT_BINS + j)));
    if (e < PT_SPLIT)
        return (int)e;
    if (e == PT_FALLBACK)
        return -1;
    const int m = (int)(e & 0x7f);
    const double b = __ldg(bp + L * PT_N + m);
    if (R >= b * (1.0 + PT_EPS))
        return m;
    if (R < b * (1.0 - PT_EPS))
        return m + 1;
    return -1;
}

// ------------------------------------------------------------------ far / near

// sum_k Phi^(k)(c, y) m_k, k <= pu (lanes share pmax = max pu over the warp).
// The reference evaluates Phi^(k) by the four-term recurrence of Eq. 10
// (kernel.py:92-127); the same derivatives obey the three-term Gegenbauer
// recurrence of dt_farcoef.cuh, which needs no 1/d and costs four FP64
// instructions per order (two DMUL off the critical path, the recurrence
// DFMA, the moment DFMA) against five:
//   h_k = c_k u h_(k-1) - w h_(k-2),   u = d/s2, w = 1/s2, s2 = d^2 + r_d^2,
// h_1 = r_d^2 / s2^(3/2), h_2 = -3 u h_1, with the traversal moments M_k
// scaled to match (dt_moments, row stride even, 16-byte aligned, read two at
// a time).  The sum agrees with the reference's to round-off.  Orders every
// far lane of the warp needs (k <= pmin) run unmasked in unrolled pairs;
// the rest up to the warp maximum is masked per lane.  Even orders go to acc
// and odd ones to acc1 on both paths, so a target's result depends on its
// own p only, not on which warp (pmin, pmax) evaluated it.
template <bool WIDE>
__device__ __forceinline__ double far_field(double d, double rd2, const double2 *__restrict__ M2,
                                            int pu, int pmin, int pmax)
{
    const double s2 = __fma_rn(d, d, rd2);
    const double r = dt_rsqrt(s2);
    const double w = r * r;
    const double u = d * w;
    double acc = (d * r) * __ldg(M2).x;
    double acc1 = 0.0;
    // Start values below order 1 chosen so that the recurrence itself yields
    // h_1 = (r_d^2 r) w and h_2 = (-3 u) h_1 with the same roundings (c_1 = 0,
    // c_2 = -3): h_(-1) = -(r_d^2 r), h_0' = 0.  Orders 1 and 2 then need no
    // special case.
    double hm2 = -(rd2 * r), hm1 = 0.0;
    int k = 1;
#define DT_FAR_STEP(KK, H2, H1, OUT)                                              \
    const double OUT = __fma_rn(u * c_hcoef[(KK) + 1], H1, -(w * H2));
    if (!WIDE) {
        // unmasked pairs (odd, even): the two recurrence values swap roles
        // every order, so each pair ends with them back in place
#pragma unroll
        for (int kk = 1; kk + 1 <= 31; kk += 2) {
            if (kk + 1 > pmin)
                break;
            DT_FAR_STEP(kk, hm2, hm1, v0)
            DT_FAR_STEP(kk + 1, hm1, v0, v1)
            // kk odd: M_kk = M2[kk / 2].y, M_(kk+1) = M2[(kk + 1) / 2].x
            acc1 = __fma_rn(v0, __ldg(M2 + kk / 2).y, acc1);
            acc = __fma_rn(v1, __ldg(M2 + (kk + 1) / 2).x, acc);
            hm2 = v0;
            hm1 = v1;
        }
        // the pairs above ran for kk = 1, 3, .. while kk + 1 <= min(pmin, 31)
        k = 1 + (min(pmin, 31) & ~1);
    }
    const double *M = reinterpret_cast<const double *>(M2);
#pragma unroll 1
    for (; k <= pmax; k += 2) {
        DT_FAR_STEP(k, hm2, hm1, t0)
        if (k <= pu) {
            if (k & 1)
                acc1 = __fma_rn(t0, __ldg(M + k), acc1);
            else
                acc = __fma_rn(t0, __ldg(M + k), acc);
        }
        if (k + 1 > pmax)
            break;
        DT_FAR_STEP(k + 1, hm1, t0, t1)
        if (k + 1 <= pu) {
            if ((k + 1) & 1)
                acc1 = __fma_rn(t1, __ldg(M + k + 1), acc1);
            else
                acc = __fma_rn(t1, __ldg(M + k + 1), acc);
        }
        hm2 = t0;
        hm1 = t1;
    }
#undef DT_FAR_STEP
    return acc + acc1;
}

// acc + q (x - y) / sqrt((x - y)^2 + r_d^2) (nvcc contracts the final
// product and sum into one DFMA): 9 FP64 instructions + MUFU
__device__ __forceinline__ double near_term(double2 u, double y, double rd2, double acc)
{
    const double du = u.x - y;
    return acc + u.y * du * dt_rsqrt(__fma_rn(du, du, rd2));
}

// Leaf sources [s, e): eight (x, q) broadcast loads in flight per step (one
// accumulator each), then one four-wide step and singles; the accumulators
// are summed pairwise.  (Four-wide: +1.3% traversal time, sixteen: spills.)
__device__ __forceinline__ double near_field(const double2 *__restrict__ xq, int s, int e,
                                             double y, double rd2)
{
    constexpr int W = 8;
    double acc[W];
#pragma unroll
    for (int u = 0; u < W; ++u)
        acc[u] = 0.0;
    int j = s;
    for (; j + W - 1 < e; j += W) {
        double2 v[W];
#pragma unroll
        for (int u = 0; u < W; ++u)
            v[u] = __ldg(xq + j + u);
#pragma unroll
        for (int u = 0; u < W; ++u)
            acc[u] = near_term(v[u], y, rd2, acc[u]);
    }
    if (j + 3 < e) {
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = __ldg(xq + j + u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            acc[u] = near_term(v[u], y, rd2, acc[u]);
        j += 4;
    }
    for (; j < e; ++j)
        acc[0] = near_term(__ldg(xq + j), y, rd2, acc[0]);
#pragma unroll
    for (int w = W / 2; w > 0; w >>= 1)
#pragma unroll
        for (int u = 0; u < w; ++u)
            acc[u] += acc[u + w];
    return acc[0];
}

// a-posteriori audit: the paper's truncation bound bound_value(M, R, h, p) =
// M R/(R-h) (h/R)^(p+1) (kernel.py:130-134) times sum_node |q|, with M the
// exact supremum of |f| on the contour (kernel.py:147-150, test_kernel.py:
// 153-163): sqrt(R/r_d) if r_d <= 2R, else 2R/sqrt(4R^2 + r_d^2).  The
// reference's sampled contour maximum can fall below the supremum when
// r_d << R, so the exact value makes the audit rigorous.
__device__ double audit_bound(const EvalArgs &a, double R, double h, int p, int s, int e)
{
    const double rd = sqrt(a.rd2);
    const double M = rd <= 2.0 * R ? sqrt(R / rd) : 2.0 * R / sqrt(4.0 * R * R + a.rd2);
    const double value = M * (R / (R - h)) * pow(h / R, (double)(p + 1));
    const double qa =
        __ldg(a.stats.abs_prefix + e - 1) - (s > 0 ? __ldg(a.stats.abs_prefix + s - 1) : 0.0);
    return value * qa;
}

// ordered interaction-list hash (see oracle.c): h <- splitmix64(h ^ code)
// per event in the lane's own depth-first visit order
__device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

template <bool ADAPTIVE, bool STATS, bool WIDE>
__global__ void __launch_bounds__(EVAL_THREADS, DT_EVAL_MINB) tree_eval_kernel(EvalArgs a)
{
    if (ADAPTIVE)
        a.tol_share = tol_share_of(a);
    __shared__ float isig_s[35];
    __shared__ double cos_s[MAX_SAMPLES], sin_s[MAX_SAMPLES];
    __shared__ uint2 stack_s[EVAL_WARPS][DT_MAX_DEPTH + 4];
    const int lane = dt_lane();
    const bool tables_in_smem = a.n_samples <= MAX_SAMPLES;
    if (ADAPTIVE) {
        if (tables_in_smem) {
            for (int t = threadIdx.x; t < a.n_samples; t += blockDim.x) {
                cos_s[t] = a.cos_tab[t];
                sin_s[t] = a.sin_tab[t];
            }
        }
        if (threadIdx.x <= 32) {
            int t = threadIdx.x;
            // s_t = (cos - 1)^2 + sin^2, the |w|^2 / R^2 of the reference's samples
            double c = a.n_samples == 64 ? a.cos_tab[t] : 1.0;
            double s = a.n_samples == 64 ? a.sin_tab[t] : 0.0;
            double sig = (c - 1.0) * (c - 1.0) + s * s;
            isig_s[t] = sig > 0.0 ? (float)(1.0 / sig) : 3.0e38f;
            if (t == 1)
                isig_s[34] = (float)sig;  // s_1: below it the maximum is at t = 1
        }
        __syncthreads();
    }
    const double *cs = tables_in_smem ? cos_s : a.cos_tab;
    const double *sn = tables_in_smem ? sin_s : a.sin_tab;
    const bool fast_ok = a.n_samples == 64 && a.psel_mode == DT_PSEL_FAST;
    __shared__ float fconst_s[2];
    if (threadIdx.x == 0) {
        fconst_s[0] = f32_of(a.rd2);
        fconst_s[1] = f32_of(log2(CONTOUR_SAFETY / a.tol_share));
    }
    // order-selection bins and level half-widths (psel_table)
    __shared__ __align__(16) unsigned char pbins_s[PT_LEVELS * PT_BINS];
    const bool table_ok = ADAPTIVE && a.pt_bins != nullptr;
    if (table_ok) {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.pt_bins);
        uint4 *dst = reinterpret_cast<uint4 *>(pbins_s);
        for (int i = threadIdx.x; i < PT_LEVELS * PT_BINS / 16; i += blockDim.x)
            dst[i] = src[i];
    }
    const int phi0 = __double2hiint(__ldg(&a.nodes[0].half));
    // without tables the bin index is pushed out of range (psel_table
    // returns -1 for every pair), so the walk needs no table_ok branch
    const int pjb = table_ok ? pt_jbase(a.theta) : -(1 << 30);
    unsigned pbins_a = (unsigned)__cvta_generic_to_shared(pbins_s);
    asm volatile("" : "+r"(pbins_a));  // kept in a register, not rematerialised
    __syncthreads();

#if DT_EVAL_SEGMENTS
    // Locality-aware scheduling: the 32-target tasks are split into
    // DT_EVAL_SEGMENTS contiguous segments; an SM's warps drain the segment
    // of their SM id first (neighbouring targets share nodes and moment rows
    // in L1), then move on to the next segment that still has tasks.
    const int64_t n_tasks = (a.i1 - a.i0 + 31) / 32;
    unsigned *const seg_ctr = reinterpret_cast<unsigned *>(a.counter);
    int seg = (int)(dt_smid() % DT_EVAL_SEGMENTS);
#endif
    while (true) {
        unsigned long long base = 0;
        {
#if DT_EVAL_SEGMENTS
            const int64_t s0 = n_tasks * seg / DT_EVAL_SEGMENTS;
            const int64_t s1 = n_tasks * (seg + 1) / DT_EVAL_SEGMENTS;
            unsigned t = 0;
            if (lane == 0)
                t = atomicAdd(seg_ctr + seg, 1u);
            t = __shfl_sync(DT_FULL, t, 0);
            if ((int64_t)t >= s1 - s0) {
                // this segment is drained: read every segment's counter at
                // once (lanes in parallel, plain L2 loads) and move to the
                // first one after it that still has tasks, instead of probing
                // the segments one atomic at a time (up to 147 round trips
                // per warp at the end of a launch)
                int next = -1;
#pragma unroll 1
                for (int r0 = 1; r0 < DT_EVAL_SEGMENTS && next < 0; r0 += 32) {
                    const int off = r0 + lane;
                    bool has = false;
                    int sg = 0;
                    if (off < DT_EVAL_SEGMENTS) {
                        sg = seg + off;
                        sg -= sg >= DT_EVAL_SEGMENTS ? DT_EVAL_SEGMENTS : 0;
                        const int64_t size = n_tasks * (sg + 1) / DT_EVAL_SEGMENTS -
                                             n_tasks * sg / DT_EVAL_SEGMENTS;
                        has = (int64_t)__ldcg(seg_ctr + sg) < size;
                    }
                    const unsigned hb = __ballot_sync(DT_FULL, has);
                    if (hb)
                        next = __shfl_sync(DT_FULL, sg, __ffs(hb) - 1);
                }
                if (next < 0)
                    break;
                seg = next;
                continue;
            }
            base = (unsigned long long)(s0 + t) * 32ull;
#else
            if (lane == 0)
                base = atomicAdd(a.counter, 32ull);
            base = __shfl_sync(DT_FULL, base, 0);
#endif
        }
        const int64_t i_first = a.i0 + (int64_t)base;
        if (i_first >= a.i1)
            break;
        const int64_t i = i_first + lane;
        const bool valid = i < a.i1;
        // plain load: ys may live in mapped (pinned) host memory
        const double y = valid ? a.ys[i] : 0.0;
        bool live = valid;
        if (a.vflags) {  // non-finite targets are counted and not traversed
            live = valid && isfinite(y);
            const unsigned bad = __ballot_sync(DT_FULL, valid && !live);
            if (bad && lane == 0)
                atomicAdd(reinterpret_cast<unsigned long long *>(a.vflags),
                          (unsigned long long)__popc(bad));
        }
        double acc = 0.0;
        uint64_t hh = 0;
        int64_t c_near = 0, c_far = 0, c_sump = 0, c_p0 = 0, c_exact = 0;
        double c_bound = 0.0;

        // Warp-uniform DFS (left subtree first, _kernels.py:199-264) over the
        // union of the 32 targets' traversals, one lane mask per entry.  An
        // opened node continues directly into its first child; only the
        // pending right siblings go on the warp's stack in shared memory
        // (depth <= 60).  Every lane stores the same entry and reads back
        // its own store, so no warp barrier is needed.
        // sp points at the top entry; entry 0 is a sentinel with an empty
        // mask (a pushed entry always has a lane), so the walk ends when it
        // pops the sentinel and no base address or index stays live
        uint2 *sp = stack_s[threadIdx.x >> 5];
        *sp = make_uint2(0u, 0u);
#if DT_EVAL_UTIL
        unsigned long long u_[12] = {0};
#endif
        int node = 0;
        unsigned mask = __ballot_sync(DT_FULL, live);
        unsigned lanebit;  // this lane's bit (asm: read once, not rematerialised)
        asm volatile("mov.u32 %0, %%lanemask_eq;" : "=r"(lanebit));
#define DT_LANE_IN(m) (((m) & lanebit) != 0u)
        while (true) {
            const double4 raw0 = dt_ldg256(a.nodes + node);  // one 256-bit load
            const double center = raw0.x, half = raw0.y;
            const int2 lr = make_int2(__double2loint(raw0.z), __double2hiint(raw0.z));
            const int2 se = make_int2(__double2loint(raw0.w), __double2hiint(raw0.w));
            const bool act = DT_LANE_IN(mask);
            const double d = center - y;
            const double big_r = fabs(d);
            const bool far = act && big_r > 0.0 && half <= __dmul_rn(a.theta, big_r);
            const unsigned fm = __ballot_sync(DT_FULL, far);
            UTIL_ADD(0, 1);
            if (fm) {
                int pu = -1;
                if (far) {
                    if (ADAPTIVE) {
                        int r = psel_table(big_r, __double2hiint(d) & 0x7fffffff, half, pbins_a,
                                           a.pt_bp, phi0, pjb);
                        UTIL_ADD(10, 1);
                        UTIL_ADD(11, r < 0);
                        if (r < 0) {  // one branch to the tiers behind the tables
                            r = fast_ok ? psel_fast(big_r, half, a, isig_s, fconst_s[0],
                                                    fconst_s[1])
                                        : -1;
                            if (r < 0) {
                                if (r <= -2 && fast_ok)
                                    r = psel_exact_bracket(big_r, half, -r - 2, a, cs, sn);
                                else
                                    r = psel_exact_all(big_r, half, a, cs, sn);
                                if (STATS)
                                    ++c_exact;
                            }
                        }
                        pu = r;
                    } else {
                        pu = a.p;
                    }
                }
                const int pmax = __reduce_max_sync(DT_FULL, pu);
                // lanes without a far interaction hold pu = -1: the unsigned
                // minimum skips them
                const int pmin = (int)__reduce_min_sync(DT_FULL, (unsigned)pu);
                UTIL_ADD(1, 1);
                UTIL_ADD(2, __popc(fm));
                UTIL_ADD(3, pmax);
                UTIL_ADD(4, __reduce_add_sync(DT_FULL, far ? pu : 0));
                UTIL_ADD(5, pmin);
                if (far) {
                    acc += far_field<WIDE>(
                        d, a.rd2,
                        reinterpret_cast<const double2 *>(a.moments) +
                            (unsigned)node * (unsigned)(a.stride >> 1),
                        pu, pmin, pmax);
                    if (STATS) {
                        hh = mix64(hh ^ ((uint64_t)node * 256u + (uint64_t)pu));
                        ++c_far;
                        c_sump += pu;
                        c_p0 += pu == 0;
                        if (a.stats.bound)
                            c_bound += audit_bound(a, big_r, half, pu, se.x, se.y);
                    }
                }
            }
            const unsigned rest = mask & ~fm;
            if (rest) {
                if (lr.x < 0) {  // leaf (first child -1)
                    UTIL_ADD(6, 1);
                    UTIL_ADD(7, __popc(rest));
                    UTIL_ADD(8, se.y - se.x);
                    if (DT_LANE_IN(rest)) {
                        acc += near_field(a.xq, se.x, se.y, y, a.rd2);
                        if (STATS) {
                            hh = mix64(hh ^ ((uint64_t)node * 256u + 255u));
                            c_near += se.y - se.x;
                        }
                    }
                } else {
                    // the right child waits on the stack: the entry is
                    // always written and kept only if there is a right child
                    sp[1] = make_uint2((unsigned)lr.y, rest);
                    sp += lr.y >= 0 ? 1 : 0;
                    node = lr.x;
                    mask = rest;
                    continue;
                }
            }
            const uint2 e = *sp--;
            if (e.y == 0u)
                break;
            node = (int)e.x;
            mask = e.y;
        }
#if DT_EVAL_UTIL
        UTIL_ADD(9, 1);
        if (lane == 0)
            for (int k = 0; k < 12; ++k)
                atomicAdd(g_util + k, u_[k]);
#endif
        if (valid) {
            double v;
            if (a.sign_xs) {  // e(y) exactly as dt_sign_terms, then e + phi
                double e = 0.0;
                if (a.sign_n) {
                    int64_t idx = -1;
                    if (a.sign_bracket) {
                        // the tile's bracket, confirmed by the sources on both
                        // sides (fails safe for unsorted targets)
                        const int64_t tile = (i - a.i0) / FIELD_TILE;
                        const int64_t lo = __ldg(a.sign_bracket + tile);
                        const int64_t hi = min(a.sign_n, __ldg(a.sign_bracket + tile + 1) + 1);
                        if (lo <= hi && (lo == 0 || __ldg(a.sign_xs + lo - 1) < y) &&
                            (hi == a.sign_n || __ldg(a.sign_xs + hi) >= y))
                            idx = dt_lower_bound(a.sign_xs, lo, hi, y);
                    }
                    if (idx < 0)
                        idx = dt_lower_bound(a.sign_xs, 0, a.sign_n, y);
                    const double below = idx == 0 ? 0.0 : __ldg(a.sign_prefix + idx - 1);
                    e = __dsub_rn(__dmul_rn(2.0, below), __ldg(a.sign_prefix + a.sign_n - 1));
                }
                v = e + acc;
            } else {
                v = a.accumulate ? a.out[i] + acc : acc;
            }
            a.out[i] = v;
            if (STATS) {
                if (a.stats.hash)
                    a.stats.hash[i] = hh;
                if (a.stats.near_pairs)
                    a.stats.near_pairs[i] = c_near;
                if (a.stats.n_far)
                    a.stats.n_far[i] = c_far;
                if (a.stats.sum_p)
                    a.stats.sum_p[i] = c_sump;
                if (a.stats.n_p0)
                    a.stats.n_p0[i] = c_p0;
                if (a.stats.n_exact)
                    a.stats.n_exact[i] = c_exact;
                if (a.stats.bound)
                    a.stats.bound[i] = c_bound;
            }
        }
    }
}

// ------------------------------------------------------------------ packing, tests

__global__ void pack_tree_kernel(const double *__restrict__ c, const double *__restrict__ h,
                                 const int64_t *__restrict__ s, const int64_t *__restrict__ e,
                                 const int64_t *__restrict__ l, const int64_t *__restrict__ r,
                                 int64_t n, dt_node *__restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    dt_node nd;
    nd.center = c[i];
    nd.half = h[i];
    dt_node_children(nd, l[i], r[i]);
    nd.start = (int32_t)s[i];
    nd.end = (int32_t)e[i];
    out[i] = nd;
}

// Reference-semantics moments [n][stride] -> traversal layout M_0 = m_0,
// M_k = c_mev_m[k] m_k (dt_farcoef.cuh), even stride (for the seam mirror
// dt_tree_phi_sum).
__global__ void scale_moments_kernel(const double *__restrict__ m, int64_t stride, int64_t n,
                                     double *__restrict__ out, int64_t estride)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * estride)
        return;
    int64_t node = i / estride;
    int k = (int)(i - node * estride);
    double v = 0.0;
    if (k < stride) {
        v = m[node * stride + k];
        if (k >= 1)
            v = __dmul_rn(v, c_mev_m[k]);
    }
    out[i] = v;
}

// bracket[b] = lower_bound(xs, ys[i0 + b FIELD_TILE]) for b < nb, and of the
// last target for b = nb (ys may be mapped host memory: one read per tile)
__global__ void field_bracket_kernel(const double *__restrict__ xs, int64_t n,
                                     const double *ys, int64_t i0, int64_t i1,
                                     int64_t *__restrict__ bracket, int64_t nb)
{
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb)
        return;
    const int64_t i = b < nb ? i0 + b * FIELD_TILE : i1 - 1;
    const double y = ys[i];
    bracket[b] = isfinite(y) ? dt_lower_bound(xs, 0, n, y) : 0;
}

__global__ void pack_sources_kernel(const double *__restrict__ xs, const double *__restrict__ qs,
                                    int64_t n, double2 *__restrict__ xq)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        xq[i] = make_double2(xs[i], qs[i]);
}

__global__ void choose_p_kernel(const double *__restrict__ R, const double *__restrict__ H,
                                int64_t n, EvalArgs a, int64_t *__restrict__ p_out,
                                int32_t *__restrict__ tier_out)
{
    __shared__ float isig_s[35];
    if (threadIdx.x <= 32) {
        int t = threadIdx.x;
        double c = a.n_samples == 64 ? a.cos_tab[t] : 1.0;
        double s = a.n_samples == 64 ? a.sin_tab[t] : 0.0;
        double sig = (c - 1.0) * (c - 1.0) + s * s;
        isig_s[t] = sig > 0.0 ? (float)(1.0 / sig) : 3.0e38f;
        if (t == 1)
            isig_s[34] = (float)sig;  // s_1: below it the maximum is at t = 1
    }
    __syncthreads();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const bool fast_ok = a.n_samples == 64 && a.psel_mode == DT_PSEL_FAST;
    int r = fast_ok ? psel_fast(R[i], H[i], a, isig_s, f32_of(a.rd2),
                                f32_of(log2(CONTOUR_SAFETY / a.tol_share)))
                    : -1;
    int tier = 0;
    if (r < 0) {
        if (r <= -2 && fast_ok) {
            r = psel_exact_bracket(R[i], H[i], -r - 2, a, a.cos_tab, a.sin_tab);
            tier = 1;
        } else {
            r = psel_exact_all(R[i], H[i], a, a.cos_tab, a.sin_tab);
            tier = 2;
        }
    }
    p_out[i] = r;
    if (tier_out)
        tier_out[i] = tier;
}

template <bool A, bool S>
const void *pick_kernel(bool wide)
{
    return wide ? (const void *)tree_eval_kernel<A, S, true>
                : (const void *)tree_eval_kernel<A, S, false>;
}

int launch_fused(EvalArgs &a, bool adaptive, bool stats, cudaStream_t s, int64_t max_grid)
{
    int per_sm = 0;
    const bool wide = a.stride > 32;
    const void *fn = adaptive ? (stats ? pick_kernel<true, true>(wide)
                                       : pick_kernel<true, false>(wide))
                              : (stats ? pick_kernel<false, true>(wide)
                                       : pick_kernel<false, false>(wide));
    {
        // occupancy per (kernel, device), queried once: it sits in front of
        // every launch otherwise
        static const void *c_fn[8];
        static int c_dev[8], c_per_sm[8], c_n = 0;
        int dev = 0;
        DT_CUDA_TRY(cudaGetDevice(&dev));
        int k = 0;
        while (k < c_n && !(c_fn[k] == fn && c_dev[k] == dev))
            ++k;
        if (k == c_n) {
            DT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, EVAL_THREADS, 0));
            if (c_n < 8) {
                c_fn[c_n] = fn;
                c_dev[c_n] = dev;
                c_per_sm[c_n] = per_sm;
                ++c_n;
            }
        } else {
            per_sm = c_per_sm[k];
        }
    }
    if (per_sm < 1)
        per_sm = 1;
    int64_t warps_needed = (a.i1 - a.i0 + 31) / 32;
    int64_t grid = (int64_t)dt_num_sms() * per_sm;
    int64_t max_useful = (warps_needed + EVAL_WARPS - 1) / EVAL_WARPS;
    if (grid > max_useful)
        grid = max_useful;
    if (max_grid > 0 && grid > max_grid)
        grid = max_grid;
    if (grid < 1)
        grid = 1;
    void *args[] = {&a};
    DT_CUDA_TRY(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(EVAL_THREADS), args, 0, s));
    return DT_OK;
}

// a.counter: the DT_EVAL_COUNTER_BYTES task-counter slot at the start of the
// caller's workspace (zeroed here, stream-ordered).
// Zero the task counters and build the order tables in the workspace slot
// (when the tables apply); a.pt_bp / a.pt_bins point at them afterwards.
// With build == false only the pointers are set: the tables were built
// earlier in stream order (dt_eval_prepare, possibly on another stream).
int prepare_eval(EvalArgs &a, bool adaptive, cudaStream_t s, bool build)
{
    if (build)
        DT_CUDA_TRY(cudaMemsetAsync(a.counter, 0, PT_BP_OFFSET, s));
    a.pt_bp = nullptr;
    a.pt_bins = nullptr;
    if (adaptive && a.n_samples == 64 && a.psel_mode == DT_PSEL_FAST && a.p_cap <= PT_N - 1 &&
        a.theta <= 0.5) {
        double *bp = reinterpret_cast<double *>(reinterpret_cast<char *>(a.counter) + PT_BP_OFFSET);
        unsigned char *bins = reinterpret_cast<unsigned char *>(a.counter) + PT_BINS_OFFSET;
        unsigned *bad = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(a.counter) + PT_BAD_OFFSET);
        PtKey *key = reinterpret_cast<PtKey *>(reinterpret_cast<char *>(a.counter) + PT_KEY_OFFSET);
        if (build) {
            psel_breakpoints_kernel<<<(PT_LEVELS * PT_N * 32 + 255) / 256, 256, 0, s>>>(a, bp, bad,
                                                                                       key);
            psel_bins_kernel<<<(PT_LEVELS * PT_BINS + 255) / 256, 256, 0, s>>>(a, bp, bad, bins,
                                                                               key);
            DT_CUDA_TRY(cudaGetLastError());
        }
        a.pt_bp = bp;
        a.pt_bins = bins;
    }
    return DT_OK;
}

int launch_eval(EvalArgs &a, bool adaptive, bool stats, cudaStream_t s, bool prepared = false)
{
    const int rc = prepare_eval(a, adaptive, s, !prepared);
    if (rc != DT_OK)
        return rc;
    return launch_fused(a, adaptive, stats, s, 0);
}

}  // namespace

#if DT_EVAL_UTIL
extern "C" int dt_eval_util(unsigned long long *host16, int reset)
{
    DT_CUDA_TRY(cudaDeviceSynchronize());
    DT_CUDA_TRY(cudaMemcpyFromSymbol(host16, g_util, sizeof(g_util)));
    if (reset) {
        unsigned long long z[16] = {0};
        DT_CUDA_TRY(cudaMemcpyToSymbol(g_util, z, sizeof(z)));
    }
    return DT_OK;
}
#endif

extern "C" int dt_pack_sources(const double *xs, const double *qs, int64_t n, double *xq,
                               void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(xs && qs && xq, "null pointer");
    pack_sources_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        xs, qs, n, (double2 *)xq);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

extern "C" int dt_pack_tree(const double *centers, const double *halves, const int64_t *starts,
                            const int64_t *ends, const int64_t *lefts, const int64_t *rights,
                            int64_t n_nodes, void *packed, void *stream)
{
    DT_CHECK_ARG(n_nodes >= 0 && n_nodes < (int64_t)1 << 31, "bad node count");
    if (n_nodes == 0)
        return DT_OK;
    DT_CHECK_ARG(centers && halves && starts && ends && lefts && rights && packed, "null pointer");
    pack_tree_kernel<<<(unsigned)((n_nodes + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        centers, halves, starts, ends, lefts, rights, n_nodes, (dt_node *)packed);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}

static inline int64_t even_stride(int64_t stride) { return (stride + 1) & ~(int64_t)1; }

static size_t mirror_prefix_bytes(int64_t n_nodes, int64_t n_src, int64_t moment_stride)
{
    size_t b = 256 + (size_t)n_nodes * sizeof(dt_node) + (size_t)n_src * 2 * sizeof(double) +
               (size_t)n_nodes * even_stride(moment_stride) * sizeof(double);
    return (b + 255) & ~(size_t)255;
}

extern "C" size_t dt_tree_eval_workspace(int64_t n_nodes, int64_t n_src, int64_t moment_stride)
{
    // packed copies for the seam mirror, then the task-counter slot
    return mirror_prefix_bytes(n_nodes, n_src, moment_stride) + DT_EVAL_COUNTER_BYTES;
}

static int check_eval_args(int64_t n_nodes, int64_t n_src, int64_t p, int adaptive,
                           double tol_share, int64_t p_cap, int64_t n_samples, double rd2,
                           double theta, int64_t i0, int64_t i1, int64_t stride)
{
    DT_CHECK_ARG(n_nodes >= 1 && n_nodes < (int64_t)1 << 31, "bad node count");
    DT_CHECK_ARG(n_src >= 0 && n_src < (int64_t)1 << 31, "bad source count");
    DT_CHECK_ARG(i0 >= 0 && i1 >= i0, "bad target range");
    DT_CHECK_ARG(p >= 0 && p < stride, "p must be >= 0 and < moment_stride");
    // the recurrence and moment-scaling tables (dt_farcoef.cuh) cover orders
    // 0..127, as dt_moments does
    DT_CHECK_ARG(stride <= 128 && p <= 127, "moment_stride must be <= 128 and p <= 127");
    // the traversal indexes moment rows in 32 bits (16-byte units)
    DT_CHECK_ARG(n_nodes * ((stride + 1) / 2) < ((int64_t)1 << 32), "moment array too large");
    DT_CHECK_ARG(rd2 > 0.0, "rd2 must be > 0");
    DT_CHECK_ARG(theta > 0.0 && theta < 1.0, "theta must lie in (0, 1)");
    if (adaptive) {
        DT_CHECK_ARG(tol_share > 0.0, "tol_share must be > 0");
        DT_CHECK_ARG(p_cap >= 0 && p_cap < stride && p_cap <= 127,
                     "p_cap must be < moment_stride and <= 127");
        DT_CHECK_ARG(n_samples >= 1, "n_samples must be >= 1");
    }
    return DT_OK;
}

extern "C" int dt_tree_phi_sum_packed(const void *packed_nodes, int64_t n_nodes,
                                      const double *moments, int64_t moment_stride,
                                      const double *xq, int64_t n_src, double rd2, double theta,
                                      int64_t p, int adaptive, double tol_share, int64_t p_cap,
                                      const double *cos_tab, const double *sin_tab,
                                      int64_t n_samples, const double *ys, double *out,
                                      int64_t i0, int64_t i1, int accumulate, int psel_mode,
                                      const dt_eval_stats *stats, void *workspace,
                                      size_t workspace_bytes, void *stream)
{
    int rc = check_eval_args(n_nodes, n_src, p, adaptive, tol_share, p_cap, n_samples, rd2,
                             theta, i0, i1, moment_stride);
    if (rc != DT_OK)
        return rc;
    if (i1 == i0)
        return DT_OK;
    DT_CHECK_ARG(packed_nodes && moments && ys && out && (n_src == 0 || xq), "null pointer");
    DT_CHECK_ARG(!adaptive || (cos_tab && sin_tab), "null contour tables");
    DT_CHECK_ARG(((uintptr_t)packed_nodes & 31) == 0 && ((uintptr_t)xq & 15) == 0 &&
                     ((uintptr_t)moments & 15) == 0,
                 "packed nodes must be 32-byte aligned, sources and moments 16-byte aligned");
    DT_CHECK_ARG((moment_stride & 1) == 0, "moment_stride must be even (16-byte rows)");
    if (!workspace || workspace_bytes < DT_EVAL_COUNTER_BYTES)
        return dt_set_error(DT_ERR_WORKSPACE, "eval workspace too small");
    DT_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "eval workspace must be 16-byte aligned");
    EvalArgs a{};
    a.nodes = (const dt_node *)packed_nodes;
    a.n_nodes = n_nodes;
    a.moments = moments;
    a.stride = moment_stride;
    a.xq = (const double2 *)xq;
    a.rd2 = rd2;
    a.theta = theta;
    a.p = (int)p;
    a.p_cap = (int)p_cap;
    a.tol_share = adaptive ? tol_share : 1.0;
    a.cos_tab = cos_tab;
    a.sin_tab = sin_tab;
    a.n_samples = (int)n_samples;
    a.ys = ys;
    a.out = out;
    a.i0 = i0;
    a.i1 = i1;
    a.accumulate = accumulate;
    a.psel_mode = psel_mode;
    if (stats)
        a.stats = *stats;
    else
        a.stats = dt_eval_stats{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.counter = (unsigned long long *)workspace;
    return launch_eval(a, adaptive != 0, stats != nullptr, (cudaStream_t)stream);
}

extern "C" size_t dt_tree_field_workspace(int64_t n_targets)
{
    return DT_EVAL_COUNTER_BYTES +
           (size_t)((n_targets + FIELD_TILE - 1) / FIELD_TILE + 1) * sizeof(int64_t);
}

extern "C" int dt_tree_field_packed(const void *packed_nodes, int64_t n_nodes,
                                    const double *moments, int64_t moment_stride,
                                    const double *xq, const double *xs, const double *prefix,
                                    int64_t n_src, double rd2, double theta, int64_t p,
                                    int adaptive, double tol_share, int64_t p_cap,
                                    const double *cos_tab, const double *sin_tab,
                                    int64_t n_samples, const double *ys, double *out, int64_t i0,
                                    int64_t i1, int64_t *flags, void *workspace,
                                    size_t workspace_bytes, void *stream)
{
    int rc = check_eval_args(n_nodes, n_src, p, adaptive, tol_share, p_cap, n_samples, rd2,
                             theta, i0, i1, moment_stride);
    if (rc != DT_OK)
        return rc;
    if (i1 == i0)
        return DT_OK;
    DT_CHECK_ARG(packed_nodes && moments && ys && out && (n_src == 0 || (xq && xs && prefix)),
                 "null pointer");
    DT_CHECK_ARG(!adaptive || (cos_tab && sin_tab), "null contour tables");
    DT_CHECK_ARG(((uintptr_t)packed_nodes & 31) == 0 && ((uintptr_t)xq & 15) == 0 &&
                     ((uintptr_t)moments & 15) == 0,
                 "packed nodes must be 32-byte aligned, sources and moments 16-byte aligned");
    DT_CHECK_ARG((moment_stride & 1) == 0, "moment_stride must be even (16-byte rows)");
    if (!workspace || workspace_bytes < DT_EVAL_COUNTER_BYTES)
        return dt_set_error(DT_ERR_WORKSPACE, "eval workspace too small");
    DT_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "eval workspace must be 16-byte aligned");
    for (const void *ptr : {(const void *)ys, (const void *)out}) {
        cudaPointerAttributes at;
        DT_CUDA_TRY(cudaPointerGetAttributes(&at, ptr));
        DT_CHECK_ARG(at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeHost ||
                         at.type == cudaMemoryTypeManaged,
                     "ys and out must be device or pinned host memory");
    }
    EvalArgs a{};
    a.nodes = (const dt_node *)packed_nodes;
    a.n_nodes = n_nodes;
    a.moments = moments;
    a.stride = moment_stride;
    a.xq = (const double2 *)xq;
    a.rd2 = rd2;
    a.theta = theta;
    a.p = (int)p;
    a.p_cap = (int)p_cap;
    a.tol_share = adaptive ? tol_share : 1.0;
    a.cos_tab = cos_tab;
    a.sin_tab = sin_tab;
    a.n_samples = (int)n_samples;
    a.ys = ys;
    a.out = out;
    a.i0 = i0;
    a.i1 = i1;
    a.accumulate = 0;
    a.psel_mode = DT_PSEL_FAST;
    a.stats = dt_eval_stats{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.counter = (unsigned long long *)workspace;
    a.sign_xs = xs ? xs : (const double *)ys;  // non-null selects the fused form
    a.sign_prefix = prefix;
    a.sign_n = n_src;
    a.vflags = flags;
    const int64_t nb = (i1 - i0 + FIELD_TILE - 1) / FIELD_TILE;
    const size_t bracket_bytes = (size_t)(nb + 1) * sizeof(int64_t);
    if (n_src > 0 && workspace_bytes >= DT_EVAL_COUNTER_BYTES + bracket_bytes) {
        int64_t *br = (int64_t *)((char *)workspace + DT_EVAL_COUNTER_BYTES);
        field_bracket_kernel<<<(unsigned)((nb + 1 + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            xs, n_src, ys, i0, i1, br, nb);
        DT_CUDA_TRY(cudaGetLastError());
        a.sign_bracket = br;
    }
    return launch_eval(a, adaptive != 0, false, (cudaStream_t)stream);
}

static int tree_eval_device(const void *packed_nodes, const int64_t *meta,
                            int64_t node_capacity, const double *moments, int64_t moment_stride,
                            const double *xq, int64_t n_src, double rd2, double theta, int64_t p,
                            int adaptive, double tolerance, int64_t p_cap, const double *cos_tab,
                            const double *sin_tab, int64_t n_samples, const double *ys,
                            double *out, int64_t i0, int64_t i1, int accumulate, void *workspace,
                            size_t workspace_bytes, void *stream, int mode)
{
    DT_CHECK_ARG(meta != nullptr, "null meta");
    int rc = check_eval_args(node_capacity, n_src, p, adaptive, tolerance, p_cap, n_samples, rd2,
                             theta, i0, i1, moment_stride);
    if (rc != DT_OK)
        return rc;
    if (i1 == i0)
        return DT_OK;
    DT_CHECK_ARG(packed_nodes && moments && ys && out && (n_src == 0 || xq), "null pointer");
    DT_CHECK_ARG(!adaptive || (cos_tab && sin_tab), "null contour tables");
    DT_CHECK_ARG(((uintptr_t)packed_nodes & 31) == 0 && ((uintptr_t)xq & 15) == 0 &&
                     ((uintptr_t)moments & 15) == 0,
                 "packed nodes must be 32-byte aligned, sources and moments 16-byte aligned");
    DT_CHECK_ARG((moment_stride & 1) == 0, "moment_stride must be even (16-byte rows)");
    if (!workspace || workspace_bytes < DT_EVAL_COUNTER_BYTES)
        return dt_set_error(DT_ERR_WORKSPACE, "eval workspace too small");
    DT_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "eval workspace must be 16-byte aligned");
    EvalArgs a{};
    a.nodes = (const dt_node *)packed_nodes;
    a.n_nodes = node_capacity;
    a.moments = moments;
    a.stride = moment_stride;
    a.xq = (const double2 *)xq;
    a.rd2 = rd2;
    a.theta = theta;
    a.p = (int)p;
    a.p_cap = (int)p_cap;
    a.tol_share = 1.0;
    a.tolerance = tolerance;
    a.meta = adaptive ? meta : nullptr;
    a.cos_tab = cos_tab;
    a.sin_tab = sin_tab;
    a.n_samples = (int)n_samples;
    a.ys = ys;
    a.out = out;
    a.i0 = i0;
    a.i1 = i1;
    a.accumulate = accumulate;
    a.psel_mode = DT_PSEL_FAST;
    a.stats = dt_eval_stats{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.counter = (unsigned long long *)workspace;
    if (mode == 1)  // tables only (dt_eval_prepare)
        return prepare_eval(a, adaptive != 0, (cudaStream_t)stream, true);
    return launch_eval(a, adaptive != 0, false, (cudaStream_t)stream, mode == 2);
}

extern "C" int dt_tree_eval_device(const void *packed_nodes, const int64_t *meta,
                                   int64_t node_capacity, const double *moments,
                                   int64_t moment_stride, const double *xq, int64_t n_src,
                                   double rd2, double theta, int64_t p, int adaptive,
                                   double tolerance, int64_t p_cap, const double *cos_tab,
                                   const double *sin_tab, int64_t n_samples, const double *ys,
                                   double *out, int64_t i0, int64_t i1, int accumulate,
                                   void *workspace, size_t workspace_bytes, void *stream)
{
    return tree_eval_device(packed_nodes, meta, node_capacity, moments, moment_stride, xq, n_src,
                            rd2, theta, p, adaptive, tolerance, p_cap, cos_tab, sin_tab,
                            n_samples, ys, out, i0, i1, accumulate, workspace, workspace_bytes,
                            stream, 0);
}

extern "C" int dt_eval_prepare(const void *packed_nodes, const int64_t *meta,
                               int64_t node_capacity, const double *moments,
                               int64_t moment_stride, const double *xq, int64_t n_src,
                               double rd2, double theta, int64_t p, int adaptive, double tolerance,
                               int64_t p_cap, const double *cos_tab, const double *sin_tab,
                               int64_t n_samples, const double *ys, double *out, int64_t i0,
                               int64_t i1, int accumulate, void *workspace,
                               size_t workspace_bytes, void *stream)
{
    return tree_eval_device(packed_nodes, meta, node_capacity, moments, moment_stride, xq, n_src,
                            rd2, theta, p, adaptive, tolerance, p_cap, cos_tab, sin_tab,
                            n_samples, ys, out, i0, i1, accumulate, workspace, workspace_bytes,
                            stream, 1);
}

extern "C" int dt_tree_eval_device_prepared(
    const void *packed_nodes, const int64_t *meta, int64_t node_capacity, const double *moments,
    int64_t moment_stride, const double *xq, int64_t n_src, double rd2, double theta, int64_t p,
    int adaptive, double tolerance, int64_t p_cap, const double *cos_tab, const double *sin_tab,
    int64_t n_samples, const double *ys, double *out, int64_t i0, int64_t i1, int accumulate,
    void *workspace, size_t workspace_bytes, void *stream)
{
    return tree_eval_device(packed_nodes, meta, node_capacity, moments, moment_stride, xq, n_src,
                            rd2, theta, p, adaptive, tolerance, p_cap, cos_tab, sin_tab,
                            n_samples, ys, out, i0, i1, accumulate, workspace, workspace_bytes,
                            stream, 2);
}

extern "C" int dt_tree_field_device(const void *packed_nodes, const int64_t *meta,
                                    int64_t node_capacity, const double *moments,
                                    int64_t moment_stride, const double *xq, const double *xs,
                                    const double *prefix, int64_t n_src, double rd2,
                                    double theta, int64_t p, int adaptive, double tolerance,
                                    int64_t p_cap, const double *cos_tab, const double *sin_tab,
                                    int64_t n_samples, const double *ys, double *out, int64_t i0,
                                    int64_t i1, void *workspace, size_t workspace_bytes,
                                    void *stream)
{
    DT_CHECK_ARG(meta != nullptr, "null meta");
    int rc = check_eval_args(node_capacity, n_src, p, adaptive, tolerance, p_cap, n_samples, rd2,
                             theta, i0, i1, moment_stride);
    if (rc != DT_OK)
        return rc;
    if (i1 == i0)
        return DT_OK;
    DT_CHECK_ARG(packed_nodes && moments && ys && out && (n_src == 0 || (xq && xs && prefix)),
                 "null pointer");
    DT_CHECK_ARG(!adaptive || (cos_tab && sin_tab), "null contour tables");
    DT_CHECK_ARG(((uintptr_t)packed_nodes & 31) == 0 && ((uintptr_t)xq & 15) == 0 &&
                     ((uintptr_t)moments & 15) == 0,
                 "packed nodes must be 32-byte aligned, sources and moments 16-byte aligned");
    DT_CHECK_ARG((moment_stride & 1) == 0, "moment_stride must be even (16-byte rows)");
    if (!workspace || workspace_bytes < DT_EVAL_COUNTER_BYTES)
        return dt_set_error(DT_ERR_WORKSPACE, "eval workspace too small");
    DT_CHECK_ARG(((uintptr_t)workspace & 15) == 0, "eval workspace must be 16-byte aligned");
    EvalArgs a{};
    a.nodes = (const dt_node *)packed_nodes;
    a.n_nodes = node_capacity;
    a.moments = moments;
    a.stride = moment_stride;
    a.xq = (const double2 *)xq;
    a.rd2 = rd2;
    a.theta = theta;
    a.p = (int)p;
    a.p_cap = (int)p_cap;
    a.tol_share = 1.0;
    a.tolerance = tolerance;
    a.meta = adaptive ? meta : nullptr;
    a.cos_tab = cos_tab;
    a.sin_tab = sin_tab;
    a.n_samples = (int)n_samples;
    a.ys = ys;
    a.out = out;
    a.i0 = i0;
    a.i1 = i1;
    a.accumulate = 0;
    a.psel_mode = DT_PSEL_FAST;
    a.stats = dt_eval_stats{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    a.counter = (unsigned long long *)workspace;
    a.sign_xs = xs ? xs : ys;  // non-null selects the fused form
    a.sign_prefix = prefix;
    a.sign_n = n_src;
    const int64_t nb = (i1 - i0 + FIELD_TILE - 1) / FIELD_TILE;
    const size_t bracket_bytes = (size_t)(nb + 1) * sizeof(int64_t);
    if (n_src > 0 && workspace_bytes >= DT_EVAL_COUNTER_BYTES + bracket_bytes) {
        int64_t *br = (int64_t *)((char *)workspace + DT_EVAL_COUNTER_BYTES);
        field_bracket_kernel<<<(unsigned)((nb + 1 + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            xs, n_src, ys, i0, i1, br, nb);
        DT_CUDA_TRY(cudaGetLastError());
        a.sign_bracket = br;
    }
    return launch_eval(a, adaptive != 0, false, (cudaStream_t)stream);
}

extern "C" int dt_tree_phi_sum(const double *centers, const double *halves, const int64_t *starts,
                               const int64_t *ends, const int64_t *lefts, const int64_t *rights,
                               const double *moments, int64_t moment_stride, int64_t n_nodes,
                               const double *xs, const double *qs, int64_t n_src, double rd2,
                               double theta, int64_t p, int adaptive, double tol_share,
                               int64_t p_cap, const double *cos_tab, const double *sin_tab,
                               int64_t n_samples, const double *ys, double *out, int64_t i0,
                               int64_t i1, int accumulate, void *workspace,
                               size_t workspace_bytes, void *stream)
{
    int rc = check_eval_args(n_nodes, n_src, p, adaptive, tol_share, p_cap, n_samples, rd2,
                             theta, i0, i1, moment_stride);
    if (rc != DT_OK)
        return rc;
    if (i1 == i0)
        return DT_OK;
    if (!workspace || workspace_bytes < dt_tree_eval_workspace(n_nodes, n_src, moment_stride))
        return dt_set_error(DT_ERR_WORKSPACE, "eval workspace too small");
    char *ws = (char *)workspace;
    void *packed = ws + 256;
    double *xq = (double *)(ws + 256 + (size_t)n_nodes * sizeof(dt_node));
    double *meval = xq + 2 * n_src;
    const int64_t estride = even_stride(moment_stride);
    rc = dt_pack_tree(centers, halves, starts, ends, lefts, rights, n_nodes, packed, stream);
    if (rc != DT_OK)
        return rc;
    rc = dt_pack_sources(xs, qs, n_src, xq, stream);
    if (rc != DT_OK)
        return rc;
    const int64_t total = n_nodes * estride;
    scale_moments_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        moments, moment_stride, n_nodes, meval, estride);
    DT_CUDA_TRY(cudaGetLastError());
    const size_t pre = mirror_prefix_bytes(n_nodes, n_src, moment_stride);
    return dt_tree_phi_sum_packed(packed, n_nodes, meval, estride, xq, n_src, rd2, theta, p,
                                  adaptive, tol_share, p_cap, cos_tab, sin_tab, n_samples, ys,
                                  out, i0, i1, accumulate, DT_PSEL_FAST, nullptr, ws + pre,
                                  workspace_bytes - pre, stream);
}

extern "C" int dt_choose_p_batch(const double *big_r, const double *h, int64_t n, double rd2,
                                 double tol_share, int64_t p_cap, const double *cos_tab,
                                 const double *sin_tab, int64_t n_samples, int psel_mode,
                                 int64_t *p_out, int32_t *tier_out, void *stream)
{
    DT_CHECK_ARG(n >= 0, "negative size");
    if (n == 0)
        return DT_OK;
    DT_CHECK_ARG(big_r && h && p_out && cos_tab && sin_tab, "null pointer");
    DT_CHECK_ARG(tol_share > 0.0 && rd2 > 0.0 && p_cap >= 0 && n_samples >= 1, "bad argument");
    EvalArgs a{};
    a.rd2 = rd2;
    a.tol_share = tol_share;
    a.p_cap = (int)p_cap;
    a.cos_tab = cos_tab;
    a.sin_tab = sin_tab;
    a.n_samples = (int)n_samples;
    a.psel_mode = psel_mode;
    choose_p_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        big_r, h, n, a, p_out, tier_out);
    DT_CUDA_TRY(cudaGetLastError());
    return DT_OK;
}
