/*
 * duhl_oracle.c -- plain, slow, single-threaded CPU oracle for the DuHL hot path
 * (arXiv 1708.05357, "Efficient Use of Limited-Memory Accelerators for Linear
 * Learning on Heterogeneous Systems").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1708_05357_b200/csrc); neither side includes the other.
 *
 * Conventions (citations: P:n = PAPER.md line n, with section/equation):
 *   A is d x n, column-major float32: column a_i starts at A + i*ld (Eq. 1).
 *   Every accumulation is in double; a float32 value converts to double exactly.
 *   model 0 = Lasso  (App. C eq. lassoobj):  (1/2d)||A a - b||^2 + lambda ||a||_1
 *   model 1 = SVM dual (App. C eq. dualsvm): (1/n) sum(-y_i a_i) + (1/(2 lambda n^2)) ||A a||^2,
 *             y_i a_i in [0,1].
 *   Primal-dual map (App. E): Lasso w = A a - b; SVM w = A a / (lambda n).
 *   Lasso Lipschitzing bound B = ||b||^2 / (2 lambda d)  (reading R1).
 *
 * Every function below is the plain definition or the paper's algorithm written
 * out step by step: no blocking, fusion or reordering.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
typedef uint64_t u64;

#define OR_LASSO 0
#define OR_SVM 1
#define OR_RIDGE 2   /* ridge regression: f as Lasso, g_i = (lambda/2) alpha_i^2 */
#define OR_ELASTIC 3 /* elastic net: g_i = lambda (eta/2 alpha_i^2 + (1-eta)|alpha_i|), 0 < eta < 1 */

/* eta of the elastic-net model (or_set_eta; test infrastructure, one value at a time). */
static double or_eta = 0.5;
void or_set_eta(double eta) { or_eta = eta; }
#define OR_HAS_B(model) ((model) != OR_SVM)   /* regression models: labels b, v~ = A alpha - b */

#define OR_OK 0
#define OR_E_INVALID 2
#define OR_E_NUMERIC 4
#define OR_E_NOT_CONVERGED 9

/* ------------------------------------------------------------------------- */
/* Counter-based generator for permutations and uniform blocks (DESIGN.md
 * "Randomness").  splitmix64 finaliser; key(seed, round, pass, j).  The CUDA
 * side implements the same documented generator independently. */
u64 or_mix64(u64 x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

u64 or_perm_key(u64 seed, i64 round, i64 pass, i64 j) {
    u64 h = or_mix64(seed);
    h = or_mix64(h ^ (u64)round);
    h = or_mix64(h ^ (u64)pass);
    return or_mix64(h ^ (u64)j);
}

/* ------------------------------------------------------------------------- */
/* Precompute: ||a_i||^2 for every column. */
void or_col_norms(const float* A, i64 d, i64 n, i64 ld, double* norms) {
    for (i64 i = 0; i < n; ++i) {
        const float* a = A + i * ld;
        double acc = 0.0;
        for (i64 k = 0; k < d; ++k) acc += (double)a[k] * (double)a[k];
        norms[i] = acc;
    }
}

/* B = ||b||^2 / (2 lambda d)   (App. E "Lasso"). */
double or_lasso_B(const double* b, i64 d, double lambda) {
    double bb = 0.0;
    for (i64 k = 0; k < d; ++k) bb += b[k] * b[k];
    return bb / (2.0 * lambda * (double)d);
}

/* v = A alpha  ("current shared state v := A alpha"). */
void or_matvec(const float* A, i64 d, i64 n, i64 ld, const double* alpha, double* v) {
    for (i64 k = 0; k < d; ++k) v[k] = 0.0;
    for (i64 i = 0; i < n; ++i) {
        if (alpha[i] == 0.0) continue;
        const float* a = A + i * ld;
        for (i64 k = 0; k < d; ++k) v[k] += (double)a[k] * alpha[i];
    }
}

/* Primal-dual map w(alpha) from v = A alpha  (App. E: P:855 Lasso, P:870 SVM). */
void or_primal_dual_w(int model, const double* v, const double* b, i64 d, i64 n, double lambda,
                      double* w) {
    for (i64 k = 0; k < d; ++k)
        w[k] = OR_HAS_B(model) ? (v[k] - b[k]) : (v[k] / (lambda * (double)n));
}

/* Per-coordinate duality gap, Eq. 4 in the closed forms of App. E:
 *   Lasso: gap_i = (1/d) [ a_i s_i + B [|s_i| - lambda d]_+ + lambda d |a_i| ]
 *   Ridge: gap_i = (1/d) [ a_i s_i + s_i^2/(2 lambda d) + (lambda d/2) a_i^2 ]
 *   SVM: gap_i = (1/n) [ a_i s_i + max(0, 1 - y_i s_i) - y_i a_i ]
 * with s_i = a_i^T w.  gap_out[i] = max(gap_i, +0.0) (reading R17: gap_i >= 0 in exact
 * arithmetic, so a rounding-negative value clamps to +0.0, which also maps -0.0 to
 * +0.0); returns OR_E_NUMERIC if a gap is below -1e-12 * (scale of its terms) or not finite.
 * idx == NULL means all columns (k must equal n).  s_out may be NULL. */
int or_coord_gaps(int model, const float* A, i64 d, i64 n, i64 ld, const double* alpha,
                  const double* y, const double* w, double lambda, double B, const i64* idx,
                  i64 k, double* s_out, double* gap_out) {
    int status = OR_OK;
    for (i64 t = 0; t < k; ++t) {
        i64 i = idx ? idx[t] : t;
        const float* a = A + i * ld;
        double s = 0.0;
        for (i64 r = 0; r < d; ++r) s += (double)a[r] * w[r];
        double g, scale;
        if (model == OR_LASSO) {
            double lam_d = lambda * (double)d;
            double thr = fabs(s) - lam_d;
            double t1 = alpha[i] * s, t2 = B * (thr > 0.0 ? thr : 0.0), t3 = lam_d * fabs(alpha[i]);
            g = (t1 + t2 + t3) / (double)d;
            scale = (fabs(t1) + t2 + t3) / (double)d;
        } else if (model == OR_ELASTIC) {
            /* Eq. 4 with g_i(a) = lambda (eta/2 a^2 + (1-eta)|a|) and its conjugate
             * g*(x) = [|x| - lambda (1-eta)]_+^2 / (2 lambda eta):
             * gap_i = g_i(a_i) + g*(-s_i/d) + a_i s_i/d  (reading R20; eta = 1 gives P:841) */
            double e = or_eta, x = fabs(s) / (double)d - lambda * (1.0 - e);
            double t1 = alpha[i] * s / (double)d;
            double t2 = lambda * (0.5 * e * alpha[i] * alpha[i] + (1.0 - e) * fabs(alpha[i]));
            double t3 = x > 0.0 ? x * x / (2.0 * lambda * e) : 0.0;
            g = t1 + t2 + t3;
            scale = fabs(t1) + t2 + t3;
        } else if (model == OR_RIDGE) {
            /* gap_i = (1/d) [ a_i s_i + s_i^2/(2 lambda d) + (lambda d/2) a_i^2 ] */
            double lam_d = lambda * (double)d;
            double t1 = alpha[i] * s, t2 = s * s / (2.0 * lam_d), t3 = 0.5 * lam_d * alpha[i] * alpha[i];
            g = (t1 + t2 + t3) / (double)d;
            scale = (fabs(t1) + t2 + t3) / (double)d;
        } else {
            double h = 1.0 - y[i] * s;
            double t1 = alpha[i] * s, t2 = (h > 0.0 ? h : 0.0), t3 = y[i] * alpha[i];
            g = (t1 + t2 - t3) / (double)n;
            scale = (fabs(t1) + t2 + fabs(t3)) / (double)n;
        }
        if (!isfinite(g) || g < -1e-12 * (scale > 1.0 ? scale : 1.0)) status = OR_E_NUMERIC;
        if (s_out) s_out[t] = s;
        /* reading R17: gap_i >= 0 in exact arithmetic; clamp at +0.0 */
        gap_out[t] = (g > 0.0) ? g : 0.0;
    }
    return status;
}

/* Top-m selection, Eq. 9 / Eq. 11:
 * P := argmax_{|P|=m} sum_{j in P} z_j  == the m largest z, ties to the lowest
 * index (reading R7).  Output: the m indices in (-z, i) order.
 * Plain stable insertion into a sorted list is O(n m); a library sort would do,
 * this is written out so the order rule is visible. */
static int or_before(const double* z, i64 a, i64 b) { /* a ranks before b */
    if (z[a] != z[b]) return z[a] > z[b];
    return a < b;
}
static void or_sort_idx(const double* z, i64* idx, i64 len) { /* merge sort by (-z, i) */
    if (len < 2) return;
    i64 h = len / 2;
    or_sort_idx(z, idx, h);
    or_sort_idx(z, idx + h, len - h);
    i64* tmp = (i64*)malloc(sizeof(i64) * (size_t)len);
    i64 p = 0, q = h, o = 0;
    while (p < h && q < len) tmp[o++] = or_before(z, idx[q], idx[p]) ? idx[q++] : idx[p++];
    while (p < h) tmp[o++] = idx[p++];
    while (q < len) tmp[o++] = idx[q++];
    memcpy(idx, tmp, sizeof(i64) * (size_t)len);
    free(tmp);
}
void or_select_topm(const double* z, i64 n, i64 m, i64* P_out) {
    i64* idx = (i64*)malloc(sizeof(i64) * (size_t)n);
    for (i64 i = 0; i < n; ++i) idx[i] = i;
    or_sort_idx(z, idx, n);
    for (i64 t = 0; t < m; ++t) P_out[t] = idx[t];
    free(idx);
}

/* rho_{t,P} of Eq. 6 (Sec. 3.2): (1/m sum_{j in P} gap_j) / (1/n sum_j gap_j),
 * written out on the gap vector z it is given (DuHL's gap memory, reading R21).
 * Returns 1 when sum_j z_j = 0 (every block is equally (un)important). */
double or_rho(const double* z, i64 n, const i64* P, i64 m) {
    double sp = 0.0, sa = 0.0;
    for (i64 t = 0; t < m; ++t) sp += z[P[t]];
    for (i64 j = 0; j < n; ++j) sa += z[j];
    if (!(sa > 0.0) || m <= 0) return 1.0;
    return (sp / (double)m) / (sa / (double)n);
}

/* Baseline selection policies (P:401 sequential blocks [Yu 2012]; P:434 uniform;
 * P:403-404 importance sampling [Zhao 2015]):
 *   sequential: block k = round mod ceil(n/m), indices [k m, min((k+1) m, n))
 *   uniform   : the m indices with the smallest (key(seed, round, -1, j), j)
 *   importance: m draws without replacement, each next draw with probability
 *               proportional to ||a_j||^2 among the remaining columns (static
 *               probabilities): the m smallest (e_j, j) with
 *               e_j = -ln(u_j) / ||a_j||^2, u_j = (key(seed, round, -2, j) >> 11 + 1/2) 2^-53
 *               (exponential clocks; zero columns never ahead of a nonzero one).
 *               z holds ||a_j||^2 for this policy.
 * Returns the number of indices written (sequential's last block may be short). */
static double or_is_clock(u64 seed, i64 round, i64 j, double w) {
    double u = ((double)(or_perm_key(seed, round, -2, j) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    return w > 0.0 ? -log(u) / w : INFINITY;
}
static void or_sort_by_dkey(double* key, i64* idx, i64 len) { /* merge sort on (key, idx) */
    if (len < 2) return;
    i64 h = len / 2;
    or_sort_by_dkey(key, idx, h);
    or_sort_by_dkey(key + h, idx + h, len - h);
    double* tk = (double*)malloc(sizeof(double) * (size_t)len);
    i64* ti = (i64*)malloc(sizeof(i64) * (size_t)len);
    i64 p = 0, q = h, o = 0;
    while (p < h && q < len) {
        int take_q = (key[q] < key[p]) || (key[q] == key[p] && idx[q] < idx[p]);
        if (take_q) { tk[o] = key[q]; ti[o++] = idx[q++]; }
        else { tk[o] = key[p]; ti[o++] = idx[p++]; }
    }
    while (p < h) { tk[o] = key[p]; ti[o++] = idx[p++]; }
    while (q < len) { tk[o] = key[q]; ti[o++] = idx[q++]; }
    memcpy(key, tk, sizeof(double) * (size_t)len);
    memcpy(idx, ti, sizeof(i64) * (size_t)len);
    free(tk);
    free(ti);
}
static void or_sort_by_key(u64* key, i64* idx, i64 len) { /* insertion-free merge sort */
    if (len < 2) return;
    i64 h = len / 2;
    or_sort_by_key(key, idx, h);
    or_sort_by_key(key + h, idx + h, len - h);
    u64* tk = (u64*)malloc(sizeof(u64) * (size_t)len);
    i64* ti = (i64*)malloc(sizeof(i64) * (size_t)len);
    i64 p = 0, q = h, o = 0;
    while (p < h && q < len) {
        int take_q = (key[q] < key[p]) || (key[q] == key[p] && idx[q] < idx[p]);
        if (take_q) { tk[o] = key[q]; ti[o++] = idx[q++]; }
        else { tk[o] = key[p]; ti[o++] = idx[p++]; }
    }
    while (p < h) { tk[o] = key[p]; ti[o++] = idx[p++]; }
    while (q < len) { tk[o] = key[q]; ti[o++] = idx[q++]; }
    memcpy(key, tk, sizeof(u64) * (size_t)len);
    memcpy(idx, ti, sizeof(i64) * (size_t)len);
    free(tk);
    free(ti);
}
i64 or_select_policy(int policy, i64 n, i64 m, i64 round, u64 seed, const double* z, i64* P_out) {
    if (policy == 0) { or_select_topm(z, n, m, P_out); return m; }
    if (policy == 1) {
        i64 nblk = (n + m - 1) / m, k = round % nblk, lo = k * m, hi = lo + m < n ? lo + m : n;
        for (i64 i = lo; i < hi; ++i) P_out[i - lo] = i;
        return hi - lo;
    }
    if (policy == 3) {
        double* e = (double*)malloc(sizeof(double) * (size_t)n);
        i64* ix = (i64*)malloc(sizeof(i64) * (size_t)n);
        for (i64 j = 0; j < n; ++j) { e[j] = or_is_clock(seed, round, j, z[j]); ix[j] = j; }
        or_sort_by_dkey(e, ix, n);
        for (i64 t = 0; t < m; ++t) P_out[t] = ix[t];
        free(e);
        free(ix);
        return m;
    }
    u64* key = (u64*)malloc(sizeof(u64) * (size_t)n);
    i64* idx = (i64*)malloc(sizeof(i64) * (size_t)n);
    for (i64 j = 0; j < n; ++j) { key[j] = or_perm_key(seed, round, -1, j); idx[j] = j; }
    or_sort_by_key(key, idx, n);
    for (i64 t = 0; t < m; ++t) P_out[t] = idx[t];
    free(key);
    free(idx);
    return m;
}

/* Permutation of the working set for one randomized pass ("randomized
 * passes"; reading R10): position t of the pass takes
 * P[pi(t)], where pi is a keyed 8-round Feistel bijection on [0, 4^h),
 * 4^h >= m, restricted to [0, m) by cycle walking; round function
 * F_r(x) = mix64(key ^ (r << 56) ^ x) mod 2^h, key = mix64(mix64(mix64(seed) ^ round) ^ pass). */
i64 or_perm_index(u64 seed, i64 round, i64 pass, i64 m, i64 t) {
    int h = 1;
    while (((i64)1 << (2 * h)) < m) ++h;
    u64 mask = ((u64)1 << h) - 1;
    u64 key = or_mix64(or_mix64(or_mix64(seed) ^ (u64)round) ^ (u64)pass);
    u64 x = (u64)t;
    do {
        u64 L = x >> h, R = x & mask;
        for (int r = 0; r < 8; ++r) {
            u64 F = or_mix64(key ^ ((u64)r << 56) ^ R) & mask;
            u64 nl = R;
            R = L ^ F;
            L = nl;
        }
        x = (L << h) | R;
    } while (x >= (u64)m);
    return (i64)x;
}
void or_make_perm(const i64* P, i64 m, u64 seed, i64 round, i64 pass, i64* out) {
    for (i64 t = 0; t < m; ++t) out[t] = P[or_perm_index(seed, round, pass, m, t)];
}

/* One exact coordinate step (App. D, eta = 0 for Lasso, eta = 1 for ridge):
 *   Lasso: gamma = (alpha_j ||a_j||^2 - a_j^T v~) / ||a_j||^2,
 *                      tau = lambda d / ||a_j||^2,  alpha' = sign(gamma) [|gamma| - tau]_+
 *   Ridge (eta = 1): alpha' = (alpha_j ||a_j||^2 - a_j^T v~) / (||a_j||^2 + lambda d)
 *   SVM: Delta = (y_j - a_j^T v^ /(lambda n)) / (||a_j||^2 /(lambda n)),
 *                      alpha' = y_j max(0, min(1, y_j (alpha_j + Delta)))
 * s = a_j^T v~ (Lasso, v~ = A alpha - b) or a_j^T v^ (SVM, v^ = A alpha).
 * Zero column (reading R5): the exact 1-D minimiser, Lasso 0, SVM y_j. */
double or_coord_update(int model, double alpha_j, double s, double norm, double y_j,
                       double lambda, i64 d, i64 n) {
    if (model == OR_RIDGE) {  /* P:808-813 with eta = 1: tau = 0, denominator ||a||^2 + lambda d */
        return (alpha_j * norm - s) / (norm + lambda * (double)d);
    }
    if (model == OR_ELASTIC) {  /* gamma, tau over ||a||^2 + lambda eta d; soft threshold */
        double den = norm + lambda * or_eta * (double)d;
        double gamma = (alpha_j * norm - s) / den;
        double tau = lambda * (double)d * (1.0 - or_eta) / den;
        double mag = fabs(gamma) - tau;
        if (mag <= 0.0) return 0.0;
        return gamma > 0.0 ? mag : -mag;
    }
    if (model == OR_LASSO) {
        if (norm == 0.0) return 0.0;
        double gamma = (alpha_j * norm - s) / norm;
        double tau = lambda * (double)d / norm;
        double mag = fabs(gamma) - tau;
        if (mag <= 0.0) return 0.0;
        return gamma > 0.0 ? mag : -mag;
    } else {
        if (norm == 0.0) return y_j;
        double ln = lambda * (double)n;
        double delta = (y_j - s / ln) / (norm / ln);
        double u = y_j * (alpha_j + delta);
        if (u < 0.0) u = 0.0;
        if (u > 1.0) u = 1.0;
        return y_j * u;
    }
}

/* Sequential SCD over `order` (one randomized pass; App. D, TPA-SCD run with
 * one coordinate at a time): s = a_j^T vt; alpha' by the closed form;
 * vt += (alpha' - alpha_j) a_j; alpha_j = alpha'.   vt is v~ (Lasso) or v^ (SVM). */
void or_scd_pass(int model, const float* A, i64 d, i64 n, i64 ld, const double* norms,
                 const double* y, double lambda, double* alpha, double* vt, const i64* order,
                 i64 len) {
    for (i64 t = 0; t < len; ++t) {
        i64 j = order[t];
        const float* a = A + j * ld;
        double s = 0.0;
        for (i64 r = 0; r < d; ++r) s += (double)a[r] * vt[r];
        double yj = (model == OR_SVM) ? y[j] : 0.0;
        double an = or_coord_update(model, alpha[j], s, norms[j], yj, lambda, d, n);
        double delta = an - alpha[j];
        if (delta != 0.0)
            for (i64 r = 0; r < d; ++r) vt[r] += delta * (double)a[r];
        alpha[j] = an;
    }
}

/* Certificate (Eq. 2 / Eq. 4, App. E) plus the independent O - D cross-check.
 * Recomputes v = A alpha from scratch.  Returns gap = sum_i gap_i and
 *   Lasso: primal O = (1/2d)||w||^2 + lambda ||alpha||_1 (w = v - b),
 *          dual  D = -(u^T b + (d/2)||u||^2) - sum_i B [|a_i^T u| - lambda]_+,  u = w/d
 *   Ridge: primal O = (1/2d)||w||^2 + (lambda/2)||alpha||^2,
 *          dual  D = -(u^T b + (d/2)||u||^2) - sum_i (a_i^T u)^2 / (2 lambda)
 *   SVM:   primal O = -(1/n) sum y_i alpha_i + ||v||^2/(2 lambda n^2)
 *          dual  D = -P(w) = -[(1/n) sum_i max(0, 1 - y_i a_i^T w) + (lambda/2)||w||^2]
 * so that gap == O - D in exact arithmetic.  b_or_y = b (Lasso) / y (SVM). */
int or_duality_gap(int model, const float* A, i64 d, i64 n, i64 ld, const double* alpha,
                   const double* b_or_y, double lambda, double B, double* gap, double* primal,
                   double* dual) {
    double* v = (double*)malloc(sizeof(double) * (size_t)d);
    double* w = (double*)malloc(sizeof(double) * (size_t)d);
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    double* g = (double*)malloc(sizeof(double) * (size_t)n);
    or_matvec(A, d, n, ld, alpha, v);
    const double* b = OR_HAS_B(model) ? b_or_y : NULL;
    const double* y = (model == OR_SVM) ? b_or_y : NULL;
    or_primal_dual_w(model, v, b, d, n, lambda, w);
    int st = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, NULL, n, s, g);
    double G = 0.0;
    for (i64 i = 0; i < n; ++i) G += g[i];
    double O = 0.0, D = 0.0;
    if (model == OR_LASSO) {
        double ww = 0.0, l1 = 0.0, ub = 0.0, uu = 0.0, conj = 0.0;
        for (i64 k = 0; k < d; ++k) ww += w[k] * w[k];
        for (i64 i = 0; i < n; ++i) l1 += fabs(alpha[i]);
        O = ww / (2.0 * (double)d) + lambda * l1;
        for (i64 k = 0; k < d; ++k) {
            double u = w[k] / (double)d;
            ub += u * b[k];
            uu += u * u;
        }
        for (i64 i = 0; i < n; ++i) {
            double x = fabs(s[i] / (double)d) - lambda;
            conj += B * (x > 0.0 ? x : 0.0);
        }
        D = -(ub + 0.5 * (double)d * uu) - conj;
    } else if (model == OR_ELASTIC) {
        /* O = (1/2d)||w||^2 + lambda sum (eta/2 a^2 + (1-eta)|a|);
         * D = -(u^T b + (d/2)||u||^2) - sum_i g*(a_i^T u),  u = w/d */
        double ww = 0.0, pen = 0.0, ub = 0.0, uu = 0.0, conj = 0.0, e = or_eta;
        for (i64 k = 0; k < d; ++k) ww += w[k] * w[k];
        for (i64 i = 0; i < n; ++i) pen += 0.5 * e * alpha[i] * alpha[i] + (1.0 - e) * fabs(alpha[i]);
        O = ww / (2.0 * (double)d) + lambda * pen;
        for (i64 k = 0; k < d; ++k) {
            double u = w[k] / (double)d;
            ub += u * b[k];
            uu += u * u;
        }
        for (i64 i = 0; i < n; ++i) {
            double x = fabs(s[i]) / (double)d - lambda * (1.0 - e);
            if (x > 0.0) conj += x * x / (2.0 * lambda * e);
        }
        D = -(ub + 0.5 * (double)d * uu) - conj;
    } else if (model == OR_RIDGE) {
        /* O = (1/2d)||w||^2 + (lambda/2)||alpha||^2;  g* of (lambda/2) x^2 is x^2/(2 lambda), so
         * D = -(u^T b + (d/2)||u||^2) - sum_i (a_i^T u)^2/(2 lambda),  u = w/d */
        double ww = 0.0, aa = 0.0, ub = 0.0, uu = 0.0, conj = 0.0;
        for (i64 k = 0; k < d; ++k) ww += w[k] * w[k];
        for (i64 i = 0; i < n; ++i) aa += alpha[i] * alpha[i];
        O = ww / (2.0 * (double)d) + 0.5 * lambda * aa;
        for (i64 k = 0; k < d; ++k) {
            double u = w[k] / (double)d;
            ub += u * b[k];
            uu += u * u;
        }
        for (i64 i = 0; i < n; ++i) {
            double x = s[i] / (double)d;
            conj += x * x / (2.0 * lambda);
        }
        D = -(ub + 0.5 * (double)d * uu) - conj;
    } else {
        double vv = 0.0, ya = 0.0, hinge = 0.0, ww = 0.0;
        for (i64 k = 0; k < d; ++k) vv += v[k] * v[k];
        for (i64 i = 0; i < n; ++i) ya += y[i] * alpha[i];
        O = -ya / (double)n + vv / (2.0 * lambda * (double)n * (double)n);
        for (i64 i = 0; i < n; ++i) {
            double h = 1.0 - y[i] * s[i];
            hinge += (h > 0.0 ? h : 0.0);
        }
        for (i64 k = 0; k < d; ++k) ww += w[k] * w[k];
        D = -(hinge / (double)n + 0.5 * lambda * ww);
    }
    *gap = G;
    if (primal) *primal = O;
    if (dual) *dual = D;
    free(v);
    free(w);
    free(s);
    free(g);
    return st;
}

/* Plain SCD over all n coordinates: the paper's single-threaded CPU baseline
 * (P:406).  One permutation of [n] per epoch (key(seed, epoch, 0, j)),
 * certificate after every epoch; stop at gap <= eps.  alpha (in/out) starts as
 * given.  Returns OR_OK, or OR_E_NOT_CONVERGED after max_epochs. */
int or_solve_scd(int model, const float* A, i64 d, i64 n, i64 ld, const double* b_or_y,
                 double lambda, double eps, i64 max_epochs, u64 seed, double* alpha,
                 double* gap_out, i64* epochs_out) {
    double* norms = (double*)malloc(sizeof(double) * (size_t)n);
    double* vt = (double*)malloc(sizeof(double) * (size_t)d);
    i64* all = (i64*)malloc(sizeof(i64) * (size_t)n);
    i64* perm = (i64*)malloc(sizeof(i64) * (size_t)n);
    or_col_norms(A, d, n, ld, norms);
    double B = (model == OR_LASSO) ? or_lasso_B(b_or_y, d, lambda) : 0.0;
    const double* y = (model == OR_SVM) ? b_or_y : NULL;
    or_matvec(A, d, n, ld, alpha, vt);
    if (OR_HAS_B(model))
        for (i64 k = 0; k < d; ++k) vt[k] -= b_or_y[k];
    for (i64 i = 0; i < n; ++i) all[i] = i;
    int st = OR_E_NOT_CONVERGED;
    double gap = INFINITY;
    i64 e = 0;
    for (e = 0; e < max_epochs; ++e) {
        or_make_perm(all, n, seed, e, 0, perm);
        or_scd_pass(model, A, d, n, ld, norms, y, lambda, alpha, vt, perm, n);
        int s2 = or_duality_gap(model, A, d, n, ld, alpha, b_or_y, lambda, B, &gap, NULL, NULL);
        if (s2 != OR_OK) { st = s2; ++e; break; }
        if (gap <= eps) { st = OR_OK; ++e; break; }
    }
    *gap_out = gap;
    if (epochs_out) *epochs_out = e;
    free(norms);
    free(vt);
    free(all);
    free(perm);
    return st;
}

/* DuHL, Algorithm 2, deterministic semantics (DESIGN.md readings
 * R6, R8, R9, R10):
 *   init  alpha = 0 (given alpha is used as is), z_i = gap_i(alpha) for all i      (R6)
 *   round t:
 *     1. P = select(z)   -- Eq. 11 top-m for policy 0; baselines 1/2;
 *        P is then an ascending index set                                       (l.3)
 *     2. swaps = |P \ P_prev|                                                   (l.4)
 *     3. unit A: z_j := gap_j(alpha^(t)) for the k = refresh_count columns of
 *        the rotating cursor (refresh_count = n: o-DuHL)  at the round-start
 *        state                                                            (l.7-10, R8)
 *     4. unit B: `passes` randomized SCD passes over P, permutation
 *        key(seed, t, pass, j); alpha and v~ updated in place (gamma = 1)    (l.6, l.11)
 *     5. z_P := gap_P(alpha^(t+1))                                              (R9)
 *     6. every cert_every rounds: certificate; its per-coordinate gaps refresh all of z (R25);
 *        stop at gap <= eps
 * Trace arrays (length >= max_rounds, may be NULL): swaps, certified gap (-1 if
 * not computed that round). */
/* w from the shared vector: Lasso w = v~ (P:855 with v~ = A alpha - b),
 * SVM w = v^/(lambda n). */
static void or_shadow_w(int model, const double* vt, i64 d, i64 n, double lambda, double* w) {
    for (i64 k = 0; k < d; ++k) w[k] = OR_HAS_B(model) ? vt[k] : vt[k] / (lambda * (double)n);
}

static int or_cmp_i64(const void* a, const void* b) {
    i64 x = *(const i64*)a, y = *(const i64*)b;
    return (x > y) - (x < y);
}

typedef struct {
    int model;
    int policy;           /* 0 gap top-m, 1 sequential, 2 uniform, 3 importance (norm-proportional) */
    i64 m;
    int passes;
    i64 refresh_count;    /* unit-A refreshes per round (rotating cursor) */
    double eps;
    i64 max_rounds;
    i64 cert_every;
    u64 seed;
} or_duhl_cfg;

int or_duhl_solve(const or_duhl_cfg* cfg, const float* A, i64 d, i64 n, i64 ld,
                  const double* b_or_y, double lambda, double* alpha, double* z,
                  i64* rounds_out, double* gap_out, i64* trace_swaps, double* trace_gap) {
    int model = cfg->model;
    i64 m = cfg->m;
    if (m < 1 || m > n) return OR_E_INVALID;
    double* norms = (double*)malloc(sizeof(double) * (size_t)n);
    double* v = (double*)malloc(sizeof(double) * (size_t)d);
    double* vt = (double*)malloc(sizeof(double) * (size_t)d);
    double* w = (double*)malloc(sizeof(double) * (size_t)d);
    i64* P = (i64*)malloc(sizeof(i64) * (size_t)m);
    i64* perm = (i64*)malloc(sizeof(i64) * (size_t)m);
    i64* idx = (i64*)malloc(sizeof(i64) * (size_t)n);
    double* gtmp = (double*)malloc(sizeof(double) * (size_t)n);
    char* in_prev = (char*)calloc((size_t)n, 1);
    char* in_cur = (char*)calloc((size_t)n, 1);
    const double* y = (model == OR_SVM) ? b_or_y : NULL;
    const double* b = OR_HAS_B(model) ? b_or_y : NULL;
    or_col_norms(A, d, n, ld, norms);
    double B = (model == OR_LASSO) ? or_lasso_B(b, d, lambda) : 0.0;
    int st = OR_E_NOT_CONVERGED;
    double gap = INFINITY;

    /* state: the shared vector of App. D, v~ = A alpha - b (Lasso) or
     * v^ = A alpha (SVM); w follows from it (App. E). */
    or_matvec(A, d, n, ld, alpha, v);
    for (i64 r = 0; r < d; ++r) vt[r] = OR_HAS_B(model) ? v[r] - b[r] : v[r];
    or_shadow_w(model, vt, d, n, lambda, w);
    int s0 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, NULL, n, NULL, z);
    if (s0 != OR_OK) st = s0;
    i64 cursor = 0, t = 0;
    for (t = 0; t < cfg->max_rounds && s0 == OR_OK; ++t) {
        /* 1. selection */
        i64 mt = or_select_policy(cfg->policy, n, m, t, cfg->seed, cfg->policy == 3 ? norms : z, P);
        qsort(P, (size_t)mt, sizeof(i64), or_cmp_i64); /* P as an ascending index set */
        /* 2. swap accounting */
        i64 swaps = 0;
        memset(in_cur, 0, (size_t)n);
        for (i64 q = 0; q < mt; ++q) { in_cur[P[q]] = 1; if (!in_prev[P[q]]) ++swaps; }
        memcpy(in_prev, in_cur, (size_t)n);
        if (trace_swaps) trace_swaps[t] = swaps;
        /* 3. unit A refresh at the round-start state (w from alpha^(t)) */
        or_shadow_w(model, vt, d, n, lambda, w);
        i64 k = cfg->refresh_count < n ? cfg->refresh_count : n;
        for (i64 q = 0; q < k; ++q) idx[q] = (cursor + q) % n;
        cursor = (cursor + k) % n;
        if (k > 0) {
            int s1 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, idx, k, NULL, gtmp);
            if (s1 != OR_OK) { st = s1; break; }
            for (i64 q = 0; q < k; ++q) z[idx[q]] = gtmp[q];
        }
        /* 4. unit B: randomized SCD passes on P, updating alpha and the shared vector */
        for (int p = 0; p < cfg->passes; ++p) {
            or_make_perm(P, mt, cfg->seed, t, p, perm);
            or_scd_pass(model, A, d, n, ld, norms, y, lambda, alpha, vt, perm, mt);
        }
        /* 5. refresh z on P at the new state */
        or_shadow_w(model, vt, d, n, lambda, w);
        int s5 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, P, mt, NULL, gtmp);
        if (s5 != OR_OK) { st = s5; break; }
        for (i64 q = 0; q < mt; ++q) z[P[q]] = gtmp[q];
        /* 6. certificate */
        if (trace_gap) trace_gap[t] = -1.0;
        if (cfg->cert_every > 0 && ((t + 1) % cfg->cert_every == 0)) {
            int s6 = or_duality_gap(model, A, d, n, ld, alpha, b_or_y, lambda, B, &gap, NULL, NULL);
            if (trace_gap) trace_gap[t] = gap;
            if (s6 != OR_OK) { st = s6; break; }
            /* reading R25: a certificate is a full unit-A pass (Alg. 2 l.7-10 over every j): its
             * gaps at the current state enter the gap memory */
            or_shadow_w(model, vt, d, n, lambda, w);
            int s7 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, NULL, n, NULL, z);
            if (s7 != OR_OK) { st = s7; break; }
            if (gap <= cfg->eps) { st = OR_OK; ++t; break; }
        }
    }
    *rounds_out = t;
    *gap_out = gap;
    free(norms); free(v); free(vt); free(w); free(P); free(perm); free(idx); free(gtmp);
    free(in_prev); free(in_cur);
    return st;
}

/* ------------------------------------------------------------------------- */
/* Multi-GPU aggregation (CoCoA-style; reading R16).
 *
 * Exact line search on the aggregation weight gamma in [0,1]: minimise the
 * global objective along alpha_old + gamma dalpha (v = v0 + gamma dv):
 *   SVM: O(g) = -(S + g sum_i y_i da_i)/n + ||v0 + g dv||^2/(2 lambda n^2)
 *                 -> g* = clip((sum y da / n - v0^T dv/(lambda n^2)) / (||dv||^2/(lambda n^2)), 0, 1)
 *   Ridge: O(g) = ||vt0 + g dv||^2/(2d) + (lambda/2) sum_i (a_i + g da_i)^2: quadratic,
 *                 g* = clip(-(vt0^T dv/d + lambda a.da) / (||dv||^2/d + lambda da.da), 0, 1)
 *   Lasso: O(g) = ||vt0 + g dv||^2/(2d) + lambda sum_i |a_i + g da_i|  (vt0 = A a - b)
 *                 convex piecewise quadratic: its right derivative
 *                 D(g) = (vt0^T dv + g ||dv||^2)/d + lambda sum_i da_i sgn+(a_i + g da_i)
 *                 is increasing; g* = the smallest g in [0,1] with D(g) >= 0, found by
 *                 walking the sorted breakpoints g_i = -a_i/da_i.
 * sgn+(x) = sign(x) for x != 0 and sign(da_i) at x = 0 (the right-limit).
 * (a_old, da, y) hold the k changed coordinates; v0/vt0, dv are length d. */
static int or_cmp_d(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}
static double or_sgnp(double x, double da) {
    if (x > 0.0) return 1.0;
    if (x < 0.0) return -1.0;
    return da > 0.0 ? 1.0 : (da < 0.0 ? -1.0 : 0.0);
}
/* right derivative along gamma; l1 = weight of the |.| part (1 Lasso, 1-eta elastic net), l2 = weight
 * of the quadratic part (0 Lasso, eta elastic net) with ada = a.da, dada = da.da */
static double or_lasso_rderiv(double g, const double* a_old, const double* da, i64 k, double vdv,
                              double dvdv, double lambda, i64 d, double l1, double l2, double ada, double dada) {
    double s = 0.0;
    for (i64 i = 0; i < k; ++i) s += da[i] * or_sgnp(a_old[i] + g * da[i], da[i]);
    return (vdv + g * dvdv) / (double)d + lambda * (l1 * s + l2 * (ada + g * dada));
}
double or_linesearch(int model, const double* v0, const double* dv, i64 d, const double* a_old,
                     const double* da, const double* y, i64 k, double lambda, i64 n) {
    double vdv = 0.0, dvdv = 0.0;
    for (i64 r = 0; r < d; ++r) { vdv += v0[r] * dv[r]; dvdv += dv[r] * dv[r]; }
    if (model == OR_SVM) {
        double ln2 = lambda * (double)n * (double)n, yda = 0.0;
        for (i64 i = 0; i < k; ++i) yda += y[i] * da[i];
        if (!(dvdv > 0.0)) return 1.0;
        double g = (yda / (double)n - vdv / ln2) / (dvdv / ln2);
        return g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g);
    }
    if (model == OR_RIDGE) {  /* quadratic in g: O'(g) = (vdv + g dvdv)/d + lambda (a.da + g da.da) */
        double ada = 0.0, dada = 0.0;
        for (i64 i = 0; i < k; ++i) { ada += a_old[i] * da[i]; dada += da[i] * da[i]; }
        double den = dvdv / (double)d + lambda * dada;
        if (!(den > 0.0)) return 1.0;
        double g = -(vdv / (double)d + lambda * ada) / den;
        return g < 0.0 ? 0.0 : (g > 1.0 ? 1.0 : g);
    }
    double l1 = 1.0, l2 = 0.0, ada = 0.0, dada = 0.0;
    if (model == OR_ELASTIC) {  /* elastic net: the Lasso walk plus the eta-weighted quadratic */
        l1 = 1.0 - or_eta;
        l2 = or_eta;
        for (i64 i = 0; i < k; ++i) { ada += a_old[i] * da[i]; dada += da[i] * da[i]; }
    }
    if (or_lasso_rderiv(0.0, a_old, da, k, vdv, dvdv, lambda, d, l1, l2, ada, dada) >= 0.0) return 0.0;
    if (or_lasso_rderiv(1.0, a_old, da, k, vdv, dvdv, lambda, d, l1, l2, ada, dada) < 0.0) return 1.0;
    /* breakpoints strictly inside (0, 1) */
    double* bp = (double*)malloc(sizeof(double) * (size_t)(k + 2));
    i64 nb = 0;
    bp[nb++] = 0.0;
    for (i64 i = 0; i < k; ++i)
        if (da[i] != 0.0) {
            double g = -a_old[i] / da[i];
            if (g > 0.0 && g < 1.0) bp[nb++] = g;
        }
    bp[nb++] = 1.0;
    qsort(bp, (size_t)nb, sizeof(double), or_cmp_d);
    double g = 1.0;
    for (i64 q = 0; q + 1 < nb; ++q) {
        double lo = bp[q], hi = bp[q + 1];
        if (!(hi > lo)) continue;
        double mid = 0.5 * (lo + hi);
        /* on (lo, hi) the sign pattern is constant:
         * D(x) = (vdv + x dvdv)/d + lambda (l1 S + l2 (ada + x dada)) */
        double S = 0.0;
        for (i64 i = 0; i < k; ++i) S += da[i] * or_sgnp(a_old[i] + mid * da[i], da[i]);
        if (or_lasso_rderiv(lo, a_old, da, k, vdv, dvdv, lambda, d, l1, l2, ada, dada) >= 0.0) { g = lo; break; }
        double den = dvdv / (double)d + lambda * l2 * dada;
        double x = den > 0.0 ? -(vdv / (double)d + lambda * (l1 * S + l2 * ada)) / den : hi;
        if (x < hi) { g = x > lo ? x : lo; break; }
    }
    free(bp);
    return g;
}

/* DuHL on K column shards (CoCoA-style aggregation): shard k
 * owns columns [k n/K, (k+1) n/K) and keeps its own gap memory, rotating
 * cursor and working set of m columns.  Round t:
 *   1. every shard: P_k = its top-m (policy) on its z, ascending
 *   2. every shard: unit-A refresh of refresh_count of its columns at alpha^(t)
 *   3. every shard: `passes` SCD passes on P_k from the common v0 (local
 *      shadow; pass permutation key (seed, t, pass) over P_k's positions),
 *      giving dv_k = v_k - v0 and dalpha on P_k
 *   4. dv = sum_k dv_k (shard order); gamma = linesearch (or 1);
 *      v = v0 + gamma dv, alpha_P = alpha_old + gamma dalpha
 *      (K = 1 without line search: v = v_1 exactly, == or_duhl_solve)
 *   5. every shard: z_P refresh at the new state; certificate every cert_every. */
int or_duhl_solve_cocoa(const or_duhl_cfg* cfg, int K, int linesearch, const float* A, i64 d, i64 n,
                        i64 ld, const double* b_or_y, double lambda, double* alpha, double* z,
                        i64* rounds_out, double* gap_out, double* trace_gap, double* trace_gamma) {
    int model = cfg->model;
    i64 m = cfg->m;
    if (K < 1 || m < 1 || m * K > n) return OR_E_INVALID;
    const double* y = (model == OR_SVM) ? b_or_y : NULL;
    const double* b = OR_HAS_B(model) ? b_or_y : NULL;
    double* norms = (double*)malloc(sizeof(double) * (size_t)n);
    double* v = (double*)malloc(sizeof(double) * (size_t)d);
    double* vt = (double*)malloc(sizeof(double) * (size_t)d);
    double* v0 = (double*)malloc(sizeof(double) * (size_t)d);
    double* vk = (double*)malloc(sizeof(double) * (size_t)d);
    double* dv = (double*)malloc(sizeof(double) * (size_t)d);
    double* w = (double*)malloc(sizeof(double) * (size_t)d);
    i64* P = (i64*)malloc(sizeof(i64) * (size_t)(m * K));
    i64* perm = (i64*)malloc(sizeof(i64) * (size_t)m);
    double* aold = (double*)malloc(sizeof(double) * (size_t)(m * K));
    double* da = (double*)malloc(sizeof(double) * (size_t)(m * K));
    double* yP = (double*)malloc(sizeof(double) * (size_t)(m * K));
    double* gtmp = (double*)malloc(sizeof(double) * (size_t)n);
    i64* idx = (i64*)malloc(sizeof(i64) * (size_t)n);
    i64* cursor = (i64*)calloc((size_t)K, sizeof(i64));
    double* zloc = (double*)malloc(sizeof(double) * (size_t)n);
    or_col_norms(A, d, n, ld, norms);
    double B = (model == OR_LASSO) ? or_lasso_B(b, d, lambda) : 0.0;
    int st = OR_E_NOT_CONVERGED;
    double gap = INFINITY;
    or_matvec(A, d, n, ld, alpha, v);
    for (i64 r = 0; r < d; ++r) vt[r] = OR_HAS_B(model) ? v[r] - b[r] : v[r];
    or_shadow_w(model, vt, d, n, lambda, w);
    int s0 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, NULL, n, NULL, z);
    if (s0 != OR_OK) st = s0;
    i64 t = 0;
    for (t = 0; t < cfg->max_rounds && s0 == OR_OK; ++t) {
        /* 1. per-shard selection */
        i64 nP = 0;
        for (int k = 0; k < K; ++k) {
            i64 lo = (i64)k * n / K, hi = (i64)(k + 1) * n / K, nk = hi - lo;
            for (i64 i = 0; i < nk; ++i) zloc[i] = cfg->policy == 3 ? norms[lo + i] : z[lo + i];
            i64 mt = or_select_policy(cfg->policy, nk, m, t, cfg->seed, zloc, P + nP);
            qsort(P + nP, (size_t)mt, sizeof(i64), or_cmp_i64);
            for (i64 q = 0; q < mt; ++q) P[nP + q] += lo;
            nP += mt;
        }
        /* 2. per-shard unit-A refresh at the round-start state */
        or_shadow_w(model, vt, d, n, lambda, w);
        for (int k = 0; k < K; ++k) {
            i64 lo = (i64)k * n / K, hi = (i64)(k + 1) * n / K, nk = hi - lo;
            i64 kr = cfg->refresh_count < nk ? cfg->refresh_count : nk;
            for (i64 q = 0; q < kr; ++q) idx[q] = lo + (cursor[k] + q) % nk;
            cursor[k] = (cursor[k] + kr) % nk;
            if (kr > 0) {
                int s1 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, idx, kr, NULL, gtmp);
                if (s1 != OR_OK) { st = s1; goto done; }
                for (i64 q = 0; q < kr; ++q) z[idx[q]] = gtmp[q];
            }
        }
        /* 3. per-shard SCD from the common v0 */
        memcpy(v0, vt, sizeof(double) * (size_t)d);
        for (i64 r = 0; r < d; ++r) dv[r] = 0.0;
        for (i64 q = 0; q < nP; ++q) aold[q] = alpha[P[q]];
        {
            i64 off = 0;
            for (int k = 0; k < K; ++k) {
                i64 lo = (i64)k * n / K, hi = (i64)(k + 1) * n / K, nk = hi - lo;
                i64 mk = m < nk ? m : nk;
                if (cfg->policy == 1) { /* sequential: the block may be short */
                    mk = 0;
                    while (off + mk < nP && P[off + mk] < hi) ++mk;
                }
                memcpy(vk, v0, sizeof(double) * (size_t)d);
                for (int p = 0; p < cfg->passes; ++p) {
                    or_make_perm(P + off, mk, cfg->seed, t, p, perm);
                    or_scd_pass(model, A, d, n, ld, norms, y, lambda, alpha, vk, perm, mk);
                }
                if (K == 1 && !linesearch) memcpy(dv, vk, sizeof(double) * (size_t)d);
                else for (i64 r = 0; r < d; ++r) dv[r] += vk[r] - v0[r];
                off += mk;
                (void)lo;
            }
        }
        /* 4. aggregation */
        double gamma = 1.0;
        if (K == 1 && !linesearch) {
            memcpy(vt, dv, sizeof(double) * (size_t)d);
        } else {
            for (i64 q = 0; q < nP; ++q) {
                da[q] = alpha[P[q]] - aold[q];
                yP[q] = y ? y[P[q]] : 0.0;
            }
            if (linesearch) gamma = or_linesearch(model, v0, dv, d, aold, da, yP, nP, lambda, n);
            for (i64 r = 0; r < d; ++r) vt[r] = v0[r] + gamma * dv[r];
            for (i64 q = 0; q < nP; ++q) alpha[P[q]] = aold[q] + gamma * da[q];
        }
        if (trace_gamma) trace_gamma[t] = gamma;
        /* 5. z_P refresh at the new state, certificate */
        or_shadow_w(model, vt, d, n, lambda, w);
        int s5 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, P, nP, NULL, gtmp);
        if (s5 != OR_OK) { st = s5; break; }
        for (i64 q = 0; q < nP; ++q) z[P[q]] = gtmp[q];
        if (trace_gap) trace_gap[t] = -1.0;
        if (cfg->cert_every > 0 && ((t + 1) % cfg->cert_every == 0)) {
            int s6 = or_duality_gap(model, A, d, n, ld, alpha, b_or_y, lambda, B, &gap, NULL, NULL);
            if (trace_gap) trace_gap[t] = gap;
            if (s6 != OR_OK) { st = s6; break; }
            /* reading R25: a certificate is a full unit-A pass (Alg. 2 l.7-10 over every j): its
             * gaps at the current state enter the gap memory */
            or_shadow_w(model, vt, d, n, lambda, w);
            int s7 = or_coord_gaps(model, A, d, n, ld, alpha, y, w, lambda, B, NULL, n, NULL, z);
            if (s7 != OR_OK) { st = s7; break; }
            if (gap <= cfg->eps) { st = OR_OK; ++t; break; }
        }
    }
done:
    *rounds_out = t;
    *gap_out = gap;
    free(norms); free(v); free(vt); free(v0); free(vk); free(dv); free(w); free(P); free(perm);
    free(aold); free(da); free(yP); free(gtmp); free(idx); free(cursor); free(zloc);
    return st;
}
