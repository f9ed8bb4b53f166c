/*
 * fg_oracle.c -- CPU restatement of the reference `fastgauss` algorithms.
 *
 * TEST INFRASTRUCTURE ONLY (see fg_oracle.h): the parity checker and the
 * CPU baseline, never the product.  Paths below are relative to
 * /root/reference/pkg/src/fastgauss/.
 *
 * The restatement follows the reference's operation order where it is cheap
 * to do so (per-coordinate squared distances without FMA, sequential
 * reductions), so that its outputs agree with the reference to ~1e-15
 * relative; it is pinned against golden vectors produced by the reference.
 */
#include "fg_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SQRT2 1.4142135623730951

/* ======================================================================
 * kernel_math.py: factorials (:20-29), graded-lex enumeration (:111-136),
 * MultiIndexSet (:139-203)
 * ====================================================================== */
static double fact_d(int n) {
    double f = 1.0;
    for (int i = 2; i <= n; i++) f *= (double)i;
    return f;
}

static int64_t binom_i(int n, int k) {
    if (k < 0 || k > n) return 0;
    int64_t r = 1;
    for (int i = 1; i <= k; i++) r = r * (n - k + i) / i;
    return r;
}

int fgo_iset_count(int dim, int order) { return (int)binom_i(dim + order - 1, dim); }

/* _compositions (kernel_math.py:111-119): digit tuples with the given sum,
 * leading digit descending. */
static void compositions(int total, int dims, int *prefix, int depth, int *out, int *k,
                         int dim) {
    if (dims == 1) {
        prefix[depth] = total;
        memcpy(out + (size_t)(*k) * dim, prefix, sizeof(int) * dim);
        (*k)++;
        return;
    }
    for (int head = total; head >= 0; head--) {
        prefix[depth] = head;
        compositions(total - head, dims - 1, prefix, depth + 1, out, k, dim);
    }
}

fgo_iset *fgo_iset_new(int dim, int order) {
    fgo_iset *s = (fgo_iset *)calloc(1, sizeof(fgo_iset));
    s->dim = dim;
    s->order = order;
    s->count = fgo_iset_count(dim, order);
    s->digits = (int *)malloc(sizeof(int) * s->count * dim);
    s->degrees = (int *)malloc(sizeof(int) * s->count);
    s->fact = (double *)malloc(sizeof(double) * s->count);
    s->inv_fact = (double *)malloc(sizeof(double) * s->count);
    s->prefix = (int *)malloc(sizeof(int) * (order + 1));
    int k = 0;
    int prefix[64];
    for (int deg = 0; deg < order; deg++) compositions(deg, dim, prefix, 0, s->digits, &k, dim);
    for (int i = 0; i < s->count; i++) {
        int deg = 0;
        double f = 1.0;
        for (int d = 0; d < dim; d++) {
            deg += s->digits[i * dim + d];
            f *= fact_d(s->digits[i * dim + d]);
        }
        s->degrees[i] = deg;
        s->fact[i] = f;
        s->inv_fact[i] = 1.0 / f;
    }
    for (int p = 0; p <= order; p++) {
        int c = 0;
        while (c < s->count && s->degrees[c] < p) c++;
        s->prefix[p] = c;
    }
    /* shift_pairs (kernel_math.py:178-203) */
    int cap = s->count * s->count;
    s->pa = (int *)malloc(sizeof(int) * cap);
    s->pb = (int *)malloc(sizeof(int) * cap);
    s->ps = (int *)malloc(sizeof(int) * cap);
    int np = 0;
    int tmp[64];
    for (int a = 0; a < s->count; a++) {
        for (int b = 0; b < s->count; b++) {
            if (s->degrees[a] + s->degrees[b] >= order) continue;
            for (int d = 0; d < dim; d++) tmp[d] = s->digits[a * dim + d] + s->digits[b * dim + d];
            int pos = -1;
            for (int c = 0; c < s->count; c++) {
                if (!memcmp(tmp, s->digits + (size_t)c * dim, sizeof(int) * dim)) {
                    pos = c;
                    break;
                }
            }
            s->pa[np] = a;
            s->pb[np] = b;
            s->ps[np] = pos;
            np++;
        }
    }
    s->npairs = np;
    return s;
}

void fgo_iset_free(fgo_iset *s) {
    if (!s) return;
    free(s->digits); free(s->degrees); free(s->fact); free(s->inv_fact);
    free(s->prefix); free(s->pa); free(s->pb); free(s->ps);
    free(s);
}

void fgo_iset_export(int dim, int order, int *digits, int *degrees, double *fact,
                     int *npairs, int *pairs) {
    fgo_iset *s = fgo_iset_new(dim, order);
    if (digits) memcpy(digits, s->digits, sizeof(int) * s->count * dim);
    if (degrees) memcpy(degrees, s->degrees, sizeof(int) * s->count);
    if (fact) memcpy(fact, s->fact, sizeof(double) * s->count);
    if (npairs) *npairs = s->npairs;
    if (pairs) {
        for (int i = 0; i < s->npairs; i++) {
            pairs[3 * i] = s->pa[i];
            pairs[3 * i + 1] = s->pb[i];
            pairs[3 * i + 2] = s->ps[i];
        }
    }
    fgo_iset_free(s);
}

/* small per-(dim, order) cache so hot loops do not rebuild tables */
#define ISET_CACHE 64
static fgo_iset *g_iset_cache[ISET_CACHE];
static fgo_iset *iset_get(int dim, int order) {
    fgo_iset *r = NULL;
#pragma omp critical(fgo_iset_cache)
    {
        for (int i = 0; i < ISET_CACHE && g_iset_cache[i]; i++) {
            if (g_iset_cache[i]->dim == dim && g_iset_cache[i]->order == order) {
                r = g_iset_cache[i];
                break;
            }
        }
        if (!r) {
            int i = 0;
            while (i < ISET_CACHE && g_iset_cache[i]) i++;
            r = fgo_iset_new(dim, order);
            if (i < ISET_CACHE) g_iset_cache[i] = r; /* else leak-free: cache full, caller frees? keep */
        }
    }
    return r;
}

/* hermite_ladder (kernel_math.py:42-65) */
static void ladder1(double t, int max_order, double *out) {
    double g = exp(-t * t);
    out[0] = g;
    if (max_order >= 1) out[1] = 2.0 * t * g;
    for (int n = 1; n < max_order; n++)
        out[n + 1] = 2.0 * t * out[n] - 2.0 * n * out[n - 1];
}

void fgo_hermite_ladder(const double *t, int64_t n, int max_order, double *out) {
    for (int64_t i = 0; i < n; i++) ladder1(t[i], max_order, out + i * (max_order + 1));
}

/* power_table (kernel_math.py:97-108) */
static void powers1(double u, int max_power, double *out) {
    out[0] = 1.0;
    for (int k = 1; k <= max_power; k++) out[k] = out[k - 1] * u;
}

void fgo_power_table(const double *u, int64_t n, int max_power, double *out) {
    for (int64_t i = 0; i < n; i++) powers1(u[i], max_power, out + i * (max_power + 1));
}

/* MultiIndexSet.products (kernel_math.py:169-176): prod_d table[d][digit] */
static inline double product(const fgo_iset *s, int k, const double *table, int L) {
    const int *dg = s->digits + (size_t)k * s->dim;
    double v = table[dg[0]];
    for (int d = 1; d < s->dim; d++) v *= table[d * L + dg[d]];
    return v;
}

/* ======================================================================
 * series_expansion.py
 * ====================================================================== */
/* accumulate_far_field (:76-92) */
void fgo_accumulate_far_field(const double *pts, const double *w, int64_t n, int dim,
                              const double *center, int order, double h, double *coeffs) {
    fgo_iset *s = iset_get(dim, order);
    int K = s->count;
    double table[64 * 64];
    for (int k = 0; k < K; k++) coeffs[k] = 0.0;
    double sc = SQRT2 * h;
    for (int64_t i = 0; i < n; i++) {
        for (int d = 0; d < dim; d++) powers1((pts[i * dim + d] - center[d]) / sc, order - 1, table + d * order);
        for (int k = 0; k < K; k++) coeffs[k] += w[i] * product(s, k, table, order);
    }
    for (int k = 0; k < K; k++) coeffs[k] *= s->inv_fact[k];
}

/* eval_far_field (:95-107), order = prefix order p */
void fgo_eval_far_field(const double *coeffs, const double *center, int dim, int order,
                        double h, const double *x, int64_t nx, double *out) {
    fgo_iset *s = iset_get(dim, order);
    double table[64 * 64];
    double sc = SQRT2 * h;
    for (int64_t i = 0; i < nx; i++) {
        for (int d = 0; d < dim; d++) ladder1((x[i * dim + d] - center[d]) / sc, order - 1, table + d * order);
        double acc = 0.0;
        for (int k = 0; k < s->count; k++) acc += product(s, k, table, order) * coeffs[k];
        out[i] = acc;
    }
}

/* accumulate_local_direct (:110-126) */
void fgo_accumulate_local_direct(const double *pts, const double *w, int64_t n, int dim,
                                 const double *center, int order, double h, double *coeffs) {
    fgo_iset *s = iset_get(dim, order);
    int K = s->count;
    double table[64 * 64];
    double sc = SQRT2 * h;
    for (int k = 0; k < K; k++) coeffs[k] = 0.0;
    for (int64_t i = 0; i < n; i++) {
        for (int d = 0; d < dim; d++) ladder1((pts[i * dim + d] - center[d]) / sc, order - 1, table + d * order);
        for (int k = 0; k < K; k++) coeffs[k] += w[i] * product(s, k, table, order);
    }
    for (int k = 0; k < K; k++) coeffs[k] *= s->inv_fact[k];
}

/* eval_local (:129-136) */
void fgo_eval_local(const double *coeffs, const double *center, int dim, int order,
                    double h, const double *x, int64_t nx, double *out) {
    fgo_iset *s = iset_get(dim, order);
    double table[64 * 64];
    double sc = SQRT2 * h;
    for (int64_t i = 0; i < nx; i++) {
        for (int d = 0; d < dim; d++) powers1((x[i * dim + d] - center[d]) / sc, order - 1, table + d * order);
        double acc = 0.0;
        for (int k = 0; k < s->count; k++) acc += product(s, k, table, order) * coeffs[k];
        out[i] = acc;
    }
}

/* translate_h2h (:139-157) */
void fgo_translate_h2h(const double *coeffs, const double *old_c, const double *new_c,
                       int dim, int order, double h, double *out) {
    fgo_iset *s = iset_get(dim, order);
    double table[64 * 64];
    double shift[4096];
    double sc = SQRT2 * h;
    for (int d = 0; d < dim; d++) powers1((old_c[d] - new_c[d]) / sc, order - 1, table + d * order);
    for (int k = 0; k < s->count; k++) shift[k] = product(s, k, table, order) * s->inv_fact[k];
    for (int k = 0; k < s->count; k++) out[k] = 0.0;
    for (int i = 0; i < s->npairs; i++) out[s->ps[i]] += coeffs[s->pa[i]] * shift[s->pb[i]];
}

/* translate_h2l (:167-194) */
void fgo_translate_h2l(const double *coeffs, const double *src_c, const double *dst_c,
                       int dim, int src_order, int dst_order, double h, double *out) {
    fgo_iset *sd = iset_get(dim, dst_order);
    fgo_iset *ss = iset_get(dim, src_order);
    int L = (dst_order - 1) + (src_order - 1) + 1;
    double lad[64 * 64];
    double sc = SQRT2 * h;
    for (int d = 0; d < dim; d++) ladder1((dst_c[d] - src_c[d]) / sc, L - 1, lad + d * L);
    for (int b = 0; b < sd->count; b++) {
        double acc = 0.0;
        for (int a = 0; a < ss->count; a++) {
            double v = 1.0;
            for (int d = 0; d < dim; d++) {
                double x = lad[d * L + sd->digits[b * dim + d] + ss->digits[a * dim + d]];
                v = (d == 0) ? x : v * x;
            }
            acc += v * coeffs[a];
        }
        double sign = (sd->degrees[b] % 2 == 0) ? 1.0 : -1.0;
        out[b] = sign * sd->inv_fact[b] * acc;
    }
}

/* translate_l2l (:197-217) */
void fgo_translate_l2l(const double *coeffs, const double *old_c, const double *new_c,
                       int dim, int order, double h, double *out) {
    fgo_iset *s = iset_get(dim, order);
    double table[64 * 64];
    double mono[4096];
    double sc = SQRT2 * h;
    for (int d = 0; d < dim; d++) powers1((new_c[d] - old_c[d]) / sc, order - 1, table + d * order);
    for (int k = 0; k < s->count; k++) mono[k] = product(s, k, table, order);
    for (int k = 0; k < s->count; k++) out[k] = 0.0;
    for (int i = 0; i < s->npairs; i++) {
        int a = s->pa[i], b = s->pb[i], c = s->ps[i];
        double binom = s->fact[c] * s->inv_fact[a] * s->inv_fact[b];
        out[a] += binom * coeffs[c] * mono[b];
    }
}

/* ======================================================================
 * error_bounds.py
 * ====================================================================== */
/* _tail_tables (:73-92) */
void fgo_tail_tables(int dim, int plimit, double *count, double *denom, double *cross) {
    for (int p = 0; p <= plimit; p++) {
        count[p] = 0.0;
        denom[p] = 1.0;
        cross[p] = 0.0;
    }
    for (int p = 1; p <= plimit; p++) {
        count[p] = (double)binom_i(dim + p - 1, dim - 1);
        int q = p / dim, r = p % dim;
        /* floor(p/D)!^(D-r) * (floor(p/D)+1)!^r as an exact integer product */
        long double prod = 1.0L;
        long double fq = (long double)fact_d(q), fq1 = (long double)fact_d(q + 1);
        for (int i = 0; i < dim - r; i++) prod *= fq;
        for (int i = 0; i < r; i++) prod *= fq1;
        denom[p] = sqrt((double)prod);
        cross[p] = (double)binom_i(dim + p - 1, dim);
    }
}

/* series_floor_constant (:148-159) */
double fgo_series_floor_constant(int dim, int plimit) {
    double count[65], denom[65], cross[65];
    fgo_tail_tables(dim, plimit, count, denom, cross);
    double m = INFINITY;
    for (int p = 1; p <= plimit; p++) {
        double v = count[p] / denom[p];
        if (v < m) m = v;
    }
    return m;
}

/* best_method (:168-230) */
void fgo_best_method(double min_sq, double max_sq, double r_ref, double r_query,
                     double w_ref, int64_t n_query, int64_t n_ref, int dim, double h,
                     double maxerr, int plimit,
                     int *method, int *order, double *bound, double *cost) {
    (void)max_sq;
    double count[65], denom[65], cross[65], ct[65];
    fgo_tail_tables(dim, plimit, count, denom, cross);
    for (int p = 0; p <= plimit; p++) ct[p] = count[p] / denom[p];
    double base = w_ref * exp(-0.25 * min_sq / (h * h));
    double rr = r_ref, rq = r_query, sq = SQRT2 * rq, sr = SQRT2 * rr;
    int p_h = 0, p_l = 0, p_t = 0;
    double e_h = INFINITY, e_l = INFINITY, e_t = INFINITY;
    if (base == 0.0) {
        p_h = p_l = p_t = 1;
        e_h = e_l = e_t = 0.0;
    } else {
        double x_r = rr, x_q = rq, x_sr = sr, x_sq = 1.0;
        for (int p = 1; p <= plimit; p++) {
            if (!p_h) {
                double err = base * ct[p] * x_r;
                if (err <= maxerr) { p_h = p; e_h = err; }
            }
            if (!p_l) {
                double err = base * ct[p] * x_q;
                if (err <= maxerr) { p_l = p; e_l = err; }
            }
            if (!p_t) {
                double step = sq > 1.0 ? x_sq : 1.0;
                double err = base * ct[p] * (x_q + x_sr * cross[p] * step);
                if (err <= maxerr) { p_t = p; e_t = err; }
            }
            if (p_h && p_l && p_t) break;
            x_r *= rr;
            x_q *= rq;
            x_sr *= sr;
            x_sq *= sq;
        }
    }
    double d = (double)dim;
    double c_h = p_h ? (double)n_query * pow(d, p_h + 1) : INFINITY;
    double c_l = p_l ? (double)n_ref * pow(d, p_l + 1) : INFINITY;
    double c_t = p_t ? pow(d, 2 * p_t + 1) : INFINITY;
    double c_x = d * (double)n_query * (double)n_ref;
    double c = c_h;
    if (c_l < c) c = c_l;
    if (c_t < c) c = c_t;
    if (c_x < c) c = c_x;
    if (c == c_h) { *method = 2; *order = p_h; *bound = e_h; *cost = c_h; return; }
    if (c == c_l) { *method = 3; *order = p_l; *bound = e_l; *cost = c_l; return; }
    if (c == c_t) { *method = 4; *order = p_t; *bound = e_t; *cost = c_t; return; }
    *method = 0; *order = 0; *bound = 0.0; *cost = c_x;
}

/* ======================================================================
 * summation_engine.py: naive_sum (:122-154)
 * ====================================================================== */
void fgo_naive_sum(const double *q, int64_t m, const double *r, const double *w,
                   int64_t n, int dim, double h, double *out) {
    double neg = -0.5 / (h * h);
    for (int64_t i = 0; i < m; i++) {
        const double *x = q + i * dim;
        double acc = 0.0;
        for (int64_t j = 0; j < n; j++) {
            const double *y = r + j * dim;
            double d2 = 0.0;
            for (int d = 0; d < dim; d++) {
                double diff = x[d] - y[d];
                double sqd = diff * diff;
                d2 += sqd;
            }
            d2 *= neg;
            acc += exp(d2) * w[j];
        }
        out[i] = acc;
    }
}

/* naive_sum with Neumaier-compensated accumulation: the same terms, summed to
 * within a few ulp of their exact sum whatever n -- the fixture for the
 * exhaustive kernel at full BASELINE sizes (a plain sequential sum of 4e6
 * terms carries ~1e-12 of its own rounding). */
void fgo_naive_sum_comp_mt(const double *q, int64_t m, const double *r, const double *w,
                           int64_t n, int dim, double h, double *out, int nthreads) {
    const double neg = -0.5 / (h * h);
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < m; i++) {
        const double *x = q + i * dim;
        double s = 0.0, c = 0.0;
        for (int64_t j = 0; j < n; j++) {
            const double *y = r + j * dim;
            double d2 = 0.0;
            for (int d = 0; d < dim; d++) {
                const double diff = x[d] - y[d];
                d2 += diff * diff;
            }
            const double v = exp(d2 * neg) * w[j];
            const double t = s + v;
            c += fabs(s) >= fabs(v) ? (s - t) + v : (v - t) + s;
            s = t;
        }
        out[i] = s + c;
    }
}

void fgo_naive_sum_mt(const double *q, int64_t m, const double *r, const double *w,
                      int64_t n, int dim, double h, double *out, int nthreads) {
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < m; i++) fgo_naive_sum(q + i * dim, 1, r, w, n, dim, h, out + i);
}

/* ======================================================================
 * spatial_index.py: KdTree, build_tree (:231-276), refresh_moments (:171-197)
 * ====================================================================== */
struct fgo_tree {
    int64_t n;
    int dim, leaf;
    double *pts, *w;
    int64_t *perm;
    int64_t nnodes, cap;
    int64_t *start, *end, *left, *right;
    double *lo, *hi, *center, *weight, *rad;
    double total_w;
    /* moments */
    int mom_order, K;
    double mom_h;
    int mom_valid;
    double *moments;
};

static int64_t tree_new_node(fgo_tree *t) {
    if (t->nnodes == t->cap) {
        int64_t c = t->cap ? 2 * t->cap : 64;
        int D = t->dim;
        t->start = (int64_t *)realloc(t->start, sizeof(int64_t) * c);
        t->end = (int64_t *)realloc(t->end, sizeof(int64_t) * c);
        t->left = (int64_t *)realloc(t->left, sizeof(int64_t) * c);
        t->right = (int64_t *)realloc(t->right, sizeof(int64_t) * c);
        t->lo = (double *)realloc(t->lo, sizeof(double) * c * D);
        t->hi = (double *)realloc(t->hi, sizeof(double) * c * D);
        t->center = (double *)realloc(t->center, sizeof(double) * c * D);
        t->weight = (double *)realloc(t->weight, sizeof(double) * c);
        t->rad = (double *)realloc(t->rad, sizeof(double) * c);
        t->cap = c;
    }
    return t->nnodes++;
}

/* construct (spatial_index.py:246-273), operating on `order` in place */
static int64_t construct(fgo_tree *t, const double *P, const double *W, int64_t *order,
                         int64_t *scratch, int64_t s, int64_t e) {
    int D = t->dim;
    int64_t id = tree_new_node(t);
    double lo[64], hi[64], sum[64];
    for (int d = 0; d < D; d++) {
        lo[d] = INFINITY;
        hi[d] = -INFINITY;
        sum[d] = 0.0;
    }
    double wsum = 0.0;
    for (int64_t i = s; i < e; i++) {
        const double *x = P + order[i] * D;
        for (int d = 0; d < D; d++) {
            if (x[d] < lo[d]) lo[d] = x[d];
            if (x[d] > hi[d]) hi[d] = x[d];
            sum[d] += x[d];
        }
        wsum += W[order[i]];
    }
    double cnt = (double)(e - s);
    double rad = 0.0;
    for (int d = 0; d < D; d++) t->center[id * D + d] = sum[d] / cnt;
    for (int64_t i = s; i < e; i++) {
        const double *x = P + order[i] * D;
        for (int d = 0; d < D; d++) {
            double a = fabs(x[d] - t->center[id * D + d]);
            if (a > rad) rad = a;
        }
    }
    for (int d = 0; d < D; d++) {
        t->lo[id * D + d] = lo[d];
        t->hi[id * D + d] = hi[d];
    }
    t->start[id] = s;
    t->end[id] = e;
    t->weight[id] = wsum;
    t->rad[id] = rad;
    t->left[id] = -1;
    t->right[id] = -1;
    int sd = 0;
    double best = hi[0] - lo[0];
    for (int d = 1; d < D; d++) {
        double wd = hi[d] - lo[d];
        if (wd > best) { best = wd; sd = d; }
    }
    if (e - s <= t->leaf || best == 0.0) return id;
    double mid = 0.5 * (lo[sd] + hi[sd]);
    int64_t nl = 0, nr = 0;
    for (int64_t i = s; i < e; i++) {
        if (P[order[i] * D + sd] < mid) order[s + nl++] = order[i];
        else scratch[nr++] = order[i];
    }
    if (nl == 0 || nl == e - s) {
        /* restore (all went one way; order unchanged when nl==e-s; when nl==0 scratch holds all) */
        if (nl == 0) memcpy(order + s, scratch, sizeof(int64_t) * nr);
        return id;
    }
    memcpy(order + s + nl, scratch, sizeof(int64_t) * nr);
    int64_t l = construct(t, P, W, order, scratch, s, s + nl);
    int64_t r = construct(t, P, W, order, scratch, s + nl, e);
    t->left[id] = l;
    t->right[id] = r;
    return id;
}

fgo_tree *fgo_build_tree(const double *pts, const double *w, int64_t n, int dim,
                         int leaf_threshold) {
    if (n < 1 || dim < 1 || dim > 64 || leaf_threshold < 1) return NULL;
    fgo_tree *t = (fgo_tree *)calloc(1, sizeof(fgo_tree));
    t->n = n;
    t->dim = dim;
    t->leaf = leaf_threshold;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *scratch = (int64_t *)malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; i++) order[i] = i;
    construct(t, pts, w, order, scratch, 0, n);
    free(scratch);
    t->perm = order;
    t->pts = (double *)malloc(sizeof(double) * n * dim);
    t->w = (double *)malloc(sizeof(double) * n);
    double tw = 0.0;
    for (int64_t i = 0; i < n; i++) {
        memcpy(t->pts + i * dim, pts + order[i] * dim, sizeof(double) * dim);
        t->w[i] = w[order[i]];
        tw += t->w[i];
    }
    t->total_w = tw;
    return t;
}

void fgo_tree_free(fgo_tree *t) {
    if (!t) return;
    free(t->pts); free(t->w); free(t->perm);
    free(t->start); free(t->end); free(t->left); free(t->right);
    free(t->lo); free(t->hi); free(t->center); free(t->weight); free(t->rad);
    free(t->moments);
    free(t);
}

int64_t fgo_tree_nnodes(const fgo_tree *t) { return t->nnodes; }

void fgo_tree_export(const fgo_tree *t, int64_t *perm, int64_t *start, int64_t *end,
                     double *lo, double *hi, double *center, double *weight,
                     double *inf_radius, int64_t *left, int64_t *right) {
    int64_t nn = t->nnodes;
    int D = t->dim;
    if (perm) memcpy(perm, t->perm, sizeof(int64_t) * t->n);
    if (start) memcpy(start, t->start, sizeof(int64_t) * nn);
    if (end) memcpy(end, t->end, sizeof(int64_t) * nn);
    if (lo) memcpy(lo, t->lo, sizeof(double) * nn * D);
    if (hi) memcpy(hi, t->hi, sizeof(double) * nn * D);
    if (center) memcpy(center, t->center, sizeof(double) * nn * D);
    if (weight) memcpy(weight, t->weight, sizeof(double) * nn);
    if (inf_radius) memcpy(inf_radius, t->rad, sizeof(double) * nn);
    if (left) memcpy(left, t->left, sizeof(int64_t) * nn);
    if (right) memcpy(right, t->right, sizeof(int64_t) * nn);
}

/* refresh_moments (spatial_index.py:171-197): direct at leaves, H2H up */
static void moments_build(fgo_tree *t, int64_t id, double h, int order) {
    int D = t->dim, K = t->K;
    double *A = t->moments + id * K;
    if (t->left[id] < 0) {
        fgo_accumulate_far_field(t->pts + t->start[id] * D, t->w + t->start[id],
                                 t->end[id] - t->start[id], D, t->center + id * D, order, h, A);
        return;
    }
    int64_t l = t->left[id], r = t->right[id];
    moments_build(t, l, h, order);
    moments_build(t, r, h, order);
    double tmp[4096];
    fgo_translate_h2h(t->moments + l * K, t->center + l * D, t->center + id * D, D, order, h, A);
    fgo_translate_h2h(t->moments + r * K, t->center + r * D, t->center + id * D, D, order, h, tmp);
    for (int k = 0; k < K; k++) A[k] += tmp[k];
}

void fgo_refresh_moments(fgo_tree *t, double h, int plimit) {
    int K = fgo_iset_count(t->dim, plimit);
    if (K != t->K || !t->moments) {
        free(t->moments);
        t->moments = (double *)malloc(sizeof(double) * t->nnodes * K);
        t->K = K;
    }
    moments_build(t, 0, h, plimit);
    t->mom_h = h;
    t->mom_order = plimit;
    t->mom_valid = 1;
}

int fgo_moments_count(const fgo_tree *t) { return t->K; }
void fgo_tree_export_moments(const fgo_tree *t, double *out) {
    memcpy(out, t->moments, sizeof(double) * t->nnodes * t->K);
}

/* ======================================================================
 * summation_engine.py: the dual-tree traversal (:157-455)
 * ====================================================================== */
typedef struct {
    double *tokens, *mass_lo, *mass_hi, *pend_lo, *pend_hi, *est;
    double *local; /* nnodes*K */
    char *local_used;
    double *q_mass_lo, *q_mass_hi, *q_est;
} qstate;

typedef struct {
    fgo_tree *q, *r;
    qstate st;
    double eps, h, neg_inv, inv_h, total_w, floor_c;
    int use_tokens, use_series, plimit, K;
    int64_t cnt[6];
    double ct[65], cross[65];
} trav;

/* _required_tokens (:157-173) */
static inline double required_tokens(double wr, double err, double eps, double mass_lo,
                                     double tw) {
    if (err <= 0.0) return -wr;
    double denom = eps * mass_lo;
    if (denom <= 0.0) return INFINITY;
    return tw * err / denom - wr;
}

/* dito_base (:221-250) incl. _leaf_kernel_block (:206-218) */
static void dito_base(trav *T, int64_t q, int64_t r) {
    fgo_tree *Q = T->q, *R = T->r;
    qstate *S = &T->st;
    int D = Q->dim;
    int64_t s = Q->start[q], e = Q->end[q];
    if (S->pend_lo[q] != 0.0 || S->pend_hi[q] != 0.0) {
        for (int64_t i = s; i < e; i++) {
            S->q_mass_lo[i] += S->pend_lo[q];
            S->q_mass_hi[i] += S->pend_hi[q];
        }
        S->pend_lo[q] = 0.0;
        S->pend_hi[q] = 0.0;
    }
    int64_t rs = R->start[r], re = R->end[r];
    double wr = R->weight[r];
    double mlo = INFINITY, mhi = -INFINITY;
    for (int64_t i = s; i < e; i++) {
        const double *x = Q->pts + i * D;
        double acc = 0.0;
        for (int64_t j = rs; j < re; j++) {
            const double *y = R->pts + j * D;
            double diff = x[0] - y[0];
            double d2 = diff * diff;
            for (int d = 1; d < D; d++) {
                double df = x[d] - y[d];
                df *= df;
                d2 += df;
            }
            d2 *= T->neg_inv;
            acc += exp(d2) * R->w[j];
        }
        S->q_mass_lo[i] += acc;
        S->q_mass_hi[i] += acc - wr;
        S->q_est[i] += acc;
        if (S->q_mass_lo[i] < mlo) mlo = S->q_mass_lo[i];
        if (S->q_mass_hi[i] > mhi) mhi = S->q_mass_hi[i];
    }
    if (T->use_tokens) S->tokens[q] += wr;
    S->mass_lo[q] = mlo;
    S->mass_hi[q] = mhi;
    T->cnt[1]++;
}

static void push_pending(trav *T, int64_t q) {
    qstate *S = &T->st;
    double pl = S->pend_lo[q], ph = S->pend_hi[q];
    if (pl != 0.0 || ph != 0.0) {
        int64_t ch[2] = {T->q->left[q], T->q->right[q]};
        for (int i = 0; i < 2; i++) {
            S->mass_lo[ch[i]] += pl;
            S->mass_hi[ch[i]] += ph;
            S->pend_lo[ch[i]] += pl;
            S->pend_hi[ch[i]] += ph;
        }
        S->pend_lo[q] = 0.0;
        S->pend_hi[q] = 0.0;
    }
}

static void visit(trav *T, int64_t q, int64_t r) {
    fgo_tree *Q = T->q, *R = T->r;
    qstate *S = &T->st;
    int D = Q->dim;
    T->cnt[0]++;
    const double *qlo = Q->lo + q * D, *qhi = Q->hi + q * D;
    const double *rlo = R->lo + r * D, *rhi = R->hi + r * D;
    double min_sq = 0.0, max_sq = 0.0;
    for (int d = 0; d < D; d++) {
        double a = qlo[d] - rhi[d], b = rlo[d] - qhi[d];
        double g = a > b ? a : b;
        if (g > 0.0) min_sq += g * g;
        double s1 = qhi[d] - rlo[d], s2 = rhi[d] - qlo[d];
        double sm = s1 > s2 ? s1 : s2;
        max_sq += sm * sm;
    }
    double k_hi = exp(min_sq * T->neg_inv);
    double k_lo = exp(max_sq * T->neg_inv);
    double w_r = R->weight[r];
    double mass_lo = S->mass_lo[q];
    double fd_err = 0.5 * w_r * (k_hi - k_lo);
    double req;
    if (fd_err <= 0.0) req = -w_r;
    else {
        double denom = T->eps * mass_lo;
        req = denom > 0.0 ? T->total_w * fd_err / denom - w_r : INFINITY;
    }
    if (req <= 0.0 || (T->use_tokens && S->tokens[q] >= req)) {
        if (T->use_tokens) S->tokens[q] -= req;
        double dl = w_r * k_lo, du = w_r * k_hi - w_r;
        S->mass_lo[q] = mass_lo + dl;
        S->mass_hi[q] += du;
        S->pend_lo[q] += dl;
        S->pend_hi[q] += du;
        S->est[q] += 0.5 * (dl + du + w_r);
        T->cnt[2]++;
        return;
    }
    if (T->use_series) {
        double maxerr = T->eps * (w_r + S->tokens[q]) * mass_lo / T->total_w;
        double r_ref = R->rad[r] * T->inv_h;
        double r_qu = Q->rad[q] * T->inv_h;
        double rmin = r_ref < r_qu ? r_ref : r_qu;
        double possible = sqrt(k_hi) * w_r * T->floor_c;
        if (rmin < 1.0) possible *= pow(rmin, T->plimit);
        if (possible <= maxerr) {
            int method, p;
            double bound, cost;
            fgo_best_method(min_sq, max_sq, r_ref, r_qu, w_r, Q->end[q] - Q->start[q],
                            R->end[r] - R->start[r], D, T->h, maxerr, T->plimit, &method, &p,
                            &bound, &cost);
            if (method != 0) {
                double rq = required_tokens(w_r, bound, T->eps, mass_lo, T->total_w);
                if (rq <= 0.0 || S->tokens[q] >= rq) {
                    S->tokens[q] -= rq;
                    int K = T->K;
                    if (method == 2) {
                        int64_t s = Q->start[q], e = Q->end[q];
                        double *tmp = (double *)malloc(sizeof(double) * (e - s));
                        fgo_eval_far_field(R->moments + r * R->K, R->center + r * D, D, p,
                                           T->h, Q->pts + s * D, e - s, tmp);
                        for (int64_t i = s; i < e; i++) S->q_est[i] += tmp[i - s];
                        free(tmp);
                        T->cnt[3]++;
                    } else if (method == 3) {
                        double c[4096];
                        fgo_accumulate_local_direct(R->pts + R->start[r] * D, R->w + R->start[r],
                                                    R->end[r] - R->start[r], D, Q->center + q * D,
                                                    p, T->h, c);
                        int kp = fgo_iset_count(D, p);
                        for (int k = 0; k < kp; k++) S->local[q * K + k] += c[k];
                        S->local_used[q] = 1;
                        T->cnt[4]++;
                    } else {
                        double c[4096];
                        fgo_translate_h2l(R->moments + r * R->K, R->center + r * D,
                                          Q->center + q * D, D, p, p, T->h, c);
                        int kp = fgo_iset_count(D, p);
                        for (int k = 0; k < kp; k++) S->local[q * K + k] += c[k];
                        S->local_used[q] = 1;
                        T->cnt[5]++;
                    }
                    double dl = w_r * k_lo, du = w_r * k_hi - w_r;
                    S->mass_lo[q] += dl;
                    S->mass_hi[q] += du;
                    S->pend_lo[q] += dl;
                    S->pend_hi[q] += du;
                    return;
                }
            }
        }
    }
    int q_leaf = Q->left[q] < 0, r_leaf = R->left[r] < 0;
    if (q_leaf && r_leaf) {
        dito_base(T, q, r);
        return;
    }
    if (q_leaf) {
        visit(T, q, R->left[r]);
        visit(T, q, R->right[r]);
        return;
    }
    push_pending(T, q);
    int64_t ql = Q->left[q], qr = Q->right[q];
    if (r_leaf) {
        visit(T, ql, r);
        visit(T, qr, r);
    } else {
        visit(T, ql, R->left[r]);
        visit(T, ql, R->right[r]);
        visit(T, qr, R->left[r]);
        visit(T, qr, R->right[r]);
    }
    S->mass_lo[q] = S->mass_lo[ql] < S->mass_lo[qr] ? S->mass_lo[ql] : S->mass_lo[qr];
    S->mass_hi[q] = S->mass_hi[ql] > S->mass_hi[qr] ? S->mass_hi[ql] : S->mass_hi[qr];
}

/* dito_post (:253-281) */
static void post(trav *T, int64_t node) {
    fgo_tree *Q = T->q;
    qstate *S = &T->st;
    int D = Q->dim, K = T->K;
    if (Q->left[node] < 0) {
        int64_t s = Q->start[node], e = Q->end[node];
        if (S->est[node] != 0.0)
            for (int64_t i = s; i < e; i++) S->q_est[i] += S->est[node];
        if (S->local_used && S->local_used[node]) {
            double *tmp = (double *)malloc(sizeof(double) * (e - s));
            fgo_eval_local(S->local + node * K, Q->center + node * D, D, T->plimit, T->h,
                           Q->pts + s * D, e - s, tmp);
            for (int64_t i = s; i < e; i++) S->q_est[i] += tmp[i - s];
            free(tmp);
        }
        return;
    }
    int64_t ch[2] = {Q->left[node], Q->right[node]};
    for (int i = 0; i < 2; i++) {
        S->est[ch[i]] += S->est[node];
        if (S->local_used && S->local_used[node]) {
            double tmp[4096];
            fgo_translate_l2l(S->local + node * K, Q->center + node * D, Q->center + ch[i] * D,
                              D, T->plimit, T->h, tmp);
            for (int k = 0; k < K; k++) S->local[ch[i] * K + k] += tmp[k];
            S->local_used[ch[i]] = 1;
        }
    }
    S->est[node] = 0.0;
    post(T, ch[0]);
    post(T, ch[1]);
}

static const int PLIMIT_SCHEDULE[7] = {1, 8, 8, 6, 4, 4, 2};
static int default_plimit(int dim) { return dim <= 6 ? PLIMIT_SCHEDULE[dim] : 1; }

/* _run_tree_algorithm (:431-455) */
int fgo_run(fgo_tree *q, fgo_tree *r, double h, double eps, int mode, int plimit,
            double *values, int64_t *counters) {
    trav T;
    memset(&T, 0, sizeof(T));
    T.q = q;
    T.r = r;
    T.h = h;
    T.eps = eps;
    T.neg_inv = -0.5 / (h * h);
    T.inv_h = 1.0 / h;
    T.total_w = r->total_w;
    T.use_tokens = mode >= 2;
    T.use_series = mode == 3;
    T.plimit = plimit > 0 ? plimit : default_plimit(q->dim);
    if (T.use_series) {
        if (!r->mom_valid || r->mom_h != h || r->mom_order < T.plimit) return 2;
        T.floor_c = fgo_series_floor_constant(q->dim, T.plimit);
        T.K = fgo_iset_count(q->dim, T.plimit);
    }
    int64_t nn = q->nnodes, n = q->n;
    qstate *S = &T.st;
    S->tokens = (double *)calloc(nn, sizeof(double));
    S->mass_lo = (double *)calloc(nn, sizeof(double));
    S->mass_hi = (double *)malloc(sizeof(double) * nn);
    S->pend_lo = (double *)calloc(nn, sizeof(double));
    S->pend_hi = (double *)calloc(nn, sizeof(double));
    S->est = (double *)calloc(nn, sizeof(double));
    for (int64_t i = 0; i < nn; i++) S->mass_hi[i] = r->total_w;
    if (T.use_series) {
        S->local = (double *)calloc((size_t)nn * T.K, sizeof(double));
        S->local_used = (char *)calloc(nn, 1);
    }
    S->q_mass_lo = (double *)calloc(n, sizeof(double));
    S->q_mass_hi = (double *)malloc(sizeof(double) * n);
    S->q_est = (double *)calloc(n, sizeof(double));
    for (int64_t i = 0; i < n; i++) S->q_mass_hi[i] = r->total_w;
    visit(&T, 0, 0);
    post(&T, 0);
    for (int64_t i = 0; i < n; i++) values[q->perm[i]] = S->q_est[i];
    if (counters) memcpy(counters, T.cnt, sizeof(T.cnt));
    free(S->tokens); free(S->mass_lo); free(S->mass_hi); free(S->pend_lo); free(S->pend_hi);
    free(S->est); free(S->local); free(S->local_used);
    free(S->q_mass_lo); free(S->q_mass_hi); free(S->q_est);
    return 0;
}

int fgo_run_sharded(const double *qpts, int64_t m, fgo_tree *r, int leaf_threshold,
                    double h, double eps, int mode, int plimit, int nthreads,
                    double *values, int64_t *counters) {
    int D = r->dim;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    if ((int64_t)nthreads > m) nthreads = (int)m;
    int64_t tot[6] = {0, 0, 0, 0, 0, 0};
    int status = 0;
    double *ones = (double *)malloc(sizeof(double) * m);
    for (int64_t i = 0; i < m; i++) ones[i] = 1.0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static, 1) num_threads(nthreads)
#endif
    for (int s = 0; s < nthreads; s++) {
        int64_t a = m * s / nthreads, b = m * (s + 1) / nthreads;
        if (b <= a) continue;
        fgo_tree *qt = fgo_build_tree(qpts + a * D, ones + a, b - a, D, leaf_threshold);
        int64_t c[6];
        int st = fgo_run(qt, r, h, eps, mode, plimit, values + a, c);
        fgo_tree_free(qt);
#ifdef _OPENMP
#pragma omp critical(fgo_shard_sum)
#endif
        {
            for (int k = 0; k < 6; k++) tot[k] += c[k];
            if (st) status = st;
        }
    }
    free(ones);
    if (counters) memcpy(counters, tot, sizeof(tot));
    return status;
}
