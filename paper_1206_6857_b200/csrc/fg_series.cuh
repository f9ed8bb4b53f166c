// fg_series.cuh -- device restatements of the series algebra
// (series_expansion.py) and the approximation selector (error_bounds.py).
//
// Coefficient vectors are dense over the graded-lex index set of their order
// (kernel_math.py:122-209); the digit table is uint8 K x kMaxDim (padded).
// The routines come in two flavours: per-lane (each lane evaluates at its own
// point: EVALM / EVALL) and lanes-over-coefficients (a warp builds one
// expansion: accumulate / translate), which keeps every lane busy without
// shuffles.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fg_device.cuh"
#include "fg_internal.cuh"

namespace fg {

struct TailArgs {
    double ct[kMaxOrder + 1], cross[kMaxOrder + 1];
};

// h_0 .. h_L of t (kernel_math.py:42-65)
__device__ __forceinline__ void hermite_ladder(double t, int L, double *out) {
    double g = exp(-t * t);
    out[0] = g;
    if (L >= 1) out[1] = 2.0 * t * g;
    for (int n = 1; n < L; n++) out[n + 1] = 2.0 * t * out[n] - 2.0 * n * out[n - 1];
}

// u^0 .. u^L (kernel_math.py:97-108)
__device__ __forceinline__ void power_ladder(double u, int L, double *out) {
    out[0] = 1.0;
    for (int k = 1; k <= L; k++) out[k] = out[k - 1] * u;
}

__device__ __forceinline__ uint64_t digits_of(const uint8_t *__restrict__ digits, int k) {
    return __ldg(reinterpret_cast<const unsigned long long *>(digits) + k);
}

// digit d of a packed row (rows hold 8 digits; beyond that only order-1
// index sets exist, whose digits are all zero)
__device__ __forceinline__ int digit(uint64_t dg, int d) {
    return d < 8 ? (int)((dg >> (8 * d)) & 0xff) : 0;
}

// prod_d table[d][digit_d] (MultiIndexSet.products, kernel_math.py:169-176)
template <int D, class Table>
__device__ __forceinline__ double product(uint64_t dg, const Table &table) {
    double v = table[0][digit(dg, 0)];
#pragma unroll
    for (int d = 1; d < D; d++) v *= table[d][digit(dg, d)];
    return v;
}

// EVALM: sum_{k<Kp} A_k prod_d h_{a_d}((x_d - c_d)/sc) (series_expansion.py:95-107)
template <int D>
__device__ double eval_far_lane(const double (&x)[D], const double *__restrict__ c,
                                const double *__restrict__ A, int p, int Kp, double sc,
                                const uint8_t *__restrict__ digits) {
    double lad[D][2 * kMaxOrder];
#pragma unroll
    for (int d = 0; d < D; d++) hermite_ladder((x[d] - __ldg(c + d)) / sc, p - 1, lad[d]);
    double acc = 0.0;
    for (int k = 0; k < Kp; k++) acc += product<D>(digits_of(digits, k), lad) * __ldg(A + k);
    return acc;
}

// ---- compile-time graded-lex tables (kernel_math.py:111-136) ----------------
__host__ __device__ constexpr int glex_count(int D, int P) {
    // C(D+P-1, D)
    long long r = 1;
    for (int i = 1; i <= D; i++) r = r * (P - 1 + i) / i;
    return (int)r;
}

__host__ __device__ constexpr int default_plimit_c(int D) {
    return D == 1 ? 8 : D == 2 ? 8 : D == 3 ? 6 : D == 4 ? 4 : D == 5 ? 4 : D == 6 ? 2 : 1;
}

template <int D, int P>
struct GLex {
    static constexpr int K = glex_count(D, P);
    int dig[K][D];
    int prefix[P + 1];
    constexpr GLex() : dig{}, prefix{} {
        int k = 0;
        for (int g = 0; g < P; g++) {
            prefix[g] = k;
            int a[D] = {};
            a[0] = g;
            for (;;) {
                for (int d = 0; d < D; d++) dig[k][d] = a[d];
                k++;
                // previous composition in lexicographically descending order
                int j = D - 2;
                while (j >= 0 && a[j] == 0) j--;
                if (j < 0) break;
                int rest = 1;
                for (int t = j + 1; t < D; t++) rest += a[t];
                a[j] -= 1;
                a[j + 1] = rest;
                for (int t = j + 2; t < D; t++) a[t] = 0;
            }
        }
        prefix[P] = k;
    }
};

// EVALM with a compile-time index set: the ladders live in registers and every
// product indexes them with constants.  Evaluates the order-p prefix (p <= P).
// The Hermite functions factor as h_n(t) = H_n(t) e^{-t^2} (kernel_math.py:42-65
// builds them by the same recurrence from h_0 = e^{-t^2}), so the ladders carry
// the Hermite polynomials and the product over dimensions takes ONE
// exponential, e^{-|t|^2}, applied to the sum (instead of one per dimension).
template <int D, int P, class ExpF>
__device__ __forceinline__ double eval_far_fixed(const double (&x)[D],
                                                 const double *__restrict__ c,
                                                 const double *__restrict__ A, int p,
                                                 double inv_sc, ExpF expf) {
    constexpr GLex<D, P> G;
    double lad[D][P], tt = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double t = (x[d] - c[d]) * inv_sc;
        tt = fma(t, t, tt);
        lad[d][0] = 1.0;
        if (P > 1) lad[d][1] = 2.0 * t;
#pragma unroll
        for (int n = 1; n + 1 < P; n++) lad[d][n + 1] = 2.0 * t * lad[d][n] - 2.0 * n * lad[d][n - 1];
    }
    int kmax = G.K;  // coefficients of the order-p prefix
#pragma unroll
    for (int q = 1; q < P; q++)
        if (q == p) kmax = G.prefix[q];
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < G.K; k++) {
        if (k < kmax) {
            double v = lad[0][G.dig[k][0]];
#pragma unroll
            for (int d = 1; d < D; d++) v *= lad[d][G.dig[k][d]];
            acc = fma(v, A[k], acc);
        }
    }
    const double g = expf(-tt);
    return g == 0.0 ? 0.0 : acc * g;  // (no inf * 0 for absurdly distant centres)
}

// Graded-lex position of a 3-digit index (for the factorised D = 3 EVALM).
template <int P>
struct GLexIndex3 {
    int idx[P][P][P];
    constexpr GLexIndex3() : idx{} {
        constexpr GLex<3, P> G{};
        for (int a = 0; a < P; a++)
            for (int b = 0; b < P; b++)
                for (int c = 0; c < P; c++) idx[a][b][c] = -1;
        for (int k = 0; k < G.K; k++) idx[G.dig[k][0]][G.dig[k][1]][G.dig[k][2]] = k;
    }
};

// EVALM for D = 3, factorised: sum_a L0[a] sum_b L1[b] sum_c A_abc L2[c], which
// takes K + C(P+1,2) + P FMAs instead of 3K multiplies (56 + 21 + 6 vs 168 at
// P = 6).  Terms of degree >= p are masked (coefficient 0).
template <int P, class ExpF>
__device__ __forceinline__ double eval_far_fixed3(const double (&x)[3],
                                                  const double *__restrict__ c,
                                                  const double *__restrict__ A, int p,
                                                  double inv_sc, ExpF expf) {
    constexpr GLexIndex3<P> I{};
    double lad[3][P], tt = 0.0;  // Hermite polynomials; e^{-|t|^2} applied once
#pragma unroll
    for (int d = 0; d < 3; d++) {
        const double t = (x[d] - c[d]) * inv_sc;
        tt = fma(t, t, tt);
        lad[d][0] = 1.0;
        if (P > 1) lad[d][1] = 2.0 * t;
#pragma unroll
        for (int n = 1; n + 1 < P; n++) lad[d][n + 1] = 2.0 * t * lad[d][n] - 2.0 * n * lad[d][n - 1];
    }
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < P; a++) {
        double t1 = 0.0;
#pragma unroll
        for (int b = 0; a + b < P; b++) {
            double t2 = 0.0;
#pragma unroll
            for (int cc = 0; a + b + cc < P; cc++) {
                const double coef = (a + b + cc < p) ? A[I.idx[a][b][cc]] : 0.0;
                t2 = fma(coef, lad[2][cc], t2);
            }
            t1 = fma(t2, lad[1][b], t1);
        }
        acc = fma(t1, lad[0][a], acc);
    }
    const double g = expf(-tt);
    return g == 0.0 ? 0.0 : acc * g;  // (no inf * 0 for absurdly distant centres)
}

// EVALL: sum_{k<K} B_k prod_d ((x_d - c_d)/sc)^{b_d} (series_expansion.py:129-136)
template <int D>
__device__ double eval_local_lane(const double (&x)[D], const double (&c)[D],
                                  const double *B, int p, int K, double sc,
                                  const uint8_t *__restrict__ digits) {
    double pw[D][2 * kMaxOrder];
#pragma unroll
    for (int d = 0; d < D; d++) power_ladder((x[d] - c[d]) / sc, p - 1, pw[d]);
    double acc = 0.0;
    for (int k = 0; k < K; k++) acc += product<D>(digits_of(digits, k), pw) * B[k];
    return acc;
}

// Warp-cooperative accumulation over a point range (lanes own coefficients):
// kind 0 = far-field moments A_a = sum_r w_r/a! ((x_r-c)/sc)^a (:76-92),
// kind 1 = direct local B_b = sum_r w_r/b! h_b((x_r-c)/sc)       (:110-126).
// Adds inv_fact-scaled sums into out[k] for k < Kp (out may alias shared mem).
template <int D>
__device__ void accumulate_warp(int kind, const double *__restrict__ pw_pts, int64_t r0,
                                int64_t r1, const double (&c)[D], int p, int Kp, double sc,
                                const uint8_t *__restrict__ digits,
                                const double *__restrict__ inv_fact, double *out,
                                bool overwrite) {
    constexpr int S = packed_stride(D);
    const int lane = threadIdx.x & 31;
    double acc[kMaxK / 32];
    uint64_t dg[kMaxK / 32];
#pragma unroll
    for (int j = 0; j < kMaxK / 32; j++) {
        acc[j] = 0.0;
        int k = lane + 32 * j;
        dg[j] = k < Kp ? digits_of(digits, k) : 0;
    }
    double tab[D][2 * kMaxOrder];
    for (int64_t r = r0; r < r1; r++) {
        double y[D], w;
        load_point_w<D>(pw_pts + r * S, y, w);
#pragma unroll
        for (int d = 0; d < D; d++) {
            double u = (y[d] - c[d]) / sc;
            if (kind == 0) power_ladder(u, p - 1, tab[d]);
            else hermite_ladder(u, p - 1, tab[d]);
        }
#pragma unroll
        for (int j = 0; j < kMaxK / 32; j++) {
            if (32 * j < Kp) acc[j] += w * product<D>(dg[j], tab);
        }
    }
#pragma unroll
    for (int j = 0; j < kMaxK / 32; j++) {
        int k = lane + 32 * j;
        if (k < Kp) {
            double v = acc[j] * __ldg(inv_fact + k);
            if (overwrite) out[k] = v;
            else out[k] += v;
        }
    }
}

// H2L (series_expansion.py:167-194): source order ps (Ks coefficients),
// destination order pd (Kd coefficients); lanes own destination coefficients
// and add into out[b] for b < Kd.
template <int D>
__device__ void h2l_warp_add(const double *__restrict__ A, const double *__restrict__ src_c,
                             const double (&dst_c)[D], int ps, int Ks, int pd, int Kd,
                             double sc, const uint8_t *__restrict__ digits,
                             const double *__restrict__ inv_fact, const int *__restrict__ degrees,
                             double *out) {
    const int lane = threadIdx.x & 31;
    double lad[D][2 * kMaxOrder];
#pragma unroll
    for (int d = 0; d < D; d++)
        hermite_ladder((dst_c[d] - __ldg(src_c + d)) / sc, (pd - 1) + (ps - 1), lad[d]);
    for (int b = lane; b < Kd; b += 32) {
        const uint64_t db = digits_of(digits, b);
        double acc = 0.0;
        for (int a = 0; a < Ks; a++) {
            const uint64_t s = db + digits_of(digits, a);  // per-byte digit sums (< 2*8)
            acc += product<D>(s, lad) * __ldg(A + a);
        }
        const double sign = (__ldg(degrees + b) % 2 == 0) ? 1.0 : -1.0;
        out[b] += sign * __ldg(inv_fact + b) * acc;
    }
}

// C(n, k) for the small digits of the index sets (n <= 2 kMaxOrder)
__device__ __forceinline__ double binom_small(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; i++) r = r * (double)(n - k + i) / (double)i;
    return r;
}

// L2L (series_expansion.py:197-217): B'_a = sum_{s >= a} C(s, a) B_s u^{s-a},
// u = (c_dst - c_src)/sc, multi-index binomials and powers per dimension;
// lanes own destination coefficients and add into out[a] for a < K.
template <int D>
__device__ void l2l_warp_add(const double *__restrict__ B, const double *__restrict__ src_c,
                             const double *dst_c, int p, int K, double sc,
                             const uint8_t *__restrict__ digits, double *out) {
    const int lane = threadIdx.x & 31;
    double pw[D][kMaxOrder];
#pragma unroll
    for (int d = 0; d < D; d++) power_ladder((dst_c[d] - __ldg(src_c + d)) / sc, p - 1, pw[d]);
    for (int a = lane; a < K; a += 32) {
        const uint64_t da = digits_of(digits, a);
        double acc = 0.0;
        for (int s = 0; s < K; s++) {
            const uint64_t ds = digits_of(digits, s);
            double v = __ldg(B + s);
            bool ok = true;
#pragma unroll
            for (int d = 0; d < D; d++) {
                const int sd = digit(ds, d), ad = digit(da, d);
                if (sd < ad) ok = false;
                else v *= binom_small(sd, ad) * pw[d][sd - ad];
            }
            if (ok) acc += v;
        }
        out[a] += acc;
    }
}

// Smallest feasible order of each series method (the order scan of
// error_bounds.py:196-225).  p == 0 marks an infeasible method.
// base = an upper bound on W_R exp(-min_sq / 4h^2) (error_bounds.py:196).
__device__ __forceinline__ void feasible_orders(double base, double r_ref, double r_query,
                                                double maxerr, int plimit, const double *ct,
                                                const double *cross, int &p_h, int &p_l,
                                                int &p_t, double &e_h, double &e_l,
                                                double &e_t) {
    const double rr = r_ref, rq = r_query, sq = kSqrt2 * rq, sr = kSqrt2 * rr;
    p_h = p_l = p_t = 0;
    e_h = e_l = e_t = CUDART_INF;
    if (base == 0.0) {
        p_h = p_l = p_t = 1;
        e_h = e_l = e_t = 0.0;
        return;
    }
    double x_r = rr, x_q = rq, x_sr = sr, x_sq = 1.0;
    for (int p = 1; p <= plimit; p++) {
        const double c = ct[p];
        if (!p_h) {
            double err = base * c * x_r;
            if (err <= maxerr) { p_h = p; e_h = err; }
        }
        if (!p_l) {
            double err = base * c * x_q;
            if (err <= maxerr) { p_l = p; e_l = err; }
        }
        if (!p_t) {
            double step = sq > 1.0 ? x_sq : 1.0;
            double err = base * c * (x_q + x_sr * cross[p] * step);
            if (err <= maxerr) { p_t = p; e_t = err; }
        }
        if (p_h && p_l && p_t) break;
        x_r *= rr;
        x_q *= rq;
        x_sr *= sr;
        x_sq *= sq;
    }
}

// Method selection for the traversal kernel: the same feasibility rule as
// best_method, with costs in warp-instruction units of THIS engine instead of
// the reference's sequential-CPU costs (error_bounds.py:217-221).  A warp owns
// a block of <= 32 nq queries, nq per lane, so
//   exhaustive ~ nq N_R c_pair            (lanes evaluate 32 pairs per step;
//                c_pair = 2D + 20 in FP64, (3D + 8) / 6 with FP32 leaves: tuned)
//   Hermite    ~ nq (32 D + K_p (D + 1)) (per-query ladders + one K_p product sum)
//   local      ~ N_R (32 D + ceil(K_p/32)(D + 1))
//   H2L        ~ 32 D + ceil(K_p/32) K_p (D + 1)
// Any feasible method keeps the error guarantee; only speed depends on this.
// base: an upper bound on W_R exp(-min_sq / 4h^2); the traversal passes
// W_R sqrt(K_hi) from its own K_hi = exp(-min_sq / 2h^2) (see there).
__device__ __forceinline__ void select_method_gpu(double base, double r_ref, double r_query,
                                                  double n_ref, int dim, double maxerr,
                                                  int plimit, const double *ct,
                                                  const double *cross, const int *kp, double nq,
                                                  double pair_cost, int &method, int &order,
                                                  double &bound) {
    int p_h, p_l, p_t;
    double e_h, e_l, e_t;
    feasible_orders(base, r_ref, r_query, maxerr, plimit, ct, cross, p_h, p_l, p_t, e_h, e_l,
                    e_t);
    const double d = (double)dim;
    double c_h = CUDART_INF, c_l = CUDART_INF, c_t = CUDART_INF;
    if (p_h) c_h = nq * (32.0 * d + kp[p_h] * (d + 1.0));
    if (p_l) c_l = n_ref * (32.0 * d + ((kp[p_l] + 31) / 32) * (d + 1.0));
    if (p_t) c_t = 32.0 * d + ((kp[p_t] + 31) / 32) * (double)kp[p_t] * (d + 1.0);
    const double c_x = nq * n_ref * pair_cost;
    const double c = fmin(fmin(c_h, c_l), fmin(c_t, c_x));
    if (c == c_h) { method = 2; order = p_h; bound = e_h; return; }
    if (c == c_l) { method = 3; order = p_l; bound = e_l; return; }
    if (c == c_t) { method = 4; order = p_t; bound = e_t; return; }
    method = 0; order = 0; bound = 0.0;
}

// best_method (error_bounds.py:168-230).  ct/cross indexed by p (1..plimit).
// method: 0 exhaustive, 2 hermite, 3 local, 4 h2l.
__device__ __forceinline__ void best_method_dev(double min_sq, double r_ref, double r_query,
                                                double w_ref, double n_query, double n_ref,
                                                int dim, double h, double maxerr, int plimit,
                                                const double *ct, const double *cross,
                                                int &method, int &order, double &bound,
                                                double &cost) {
    const double base = w_ref * exp(-0.25 * min_sq / (h * h));
    const double rr = r_ref, rq = r_query, sq = kSqrt2 * rq, sr = kSqrt2 * rr;
    int p_h = 0, p_l = 0, p_t = 0;
    double e_h = CUDART_INF, e_l = CUDART_INF, e_t = CUDART_INF;
    if (base == 0.0) {
        p_h = p_l = p_t = 1;
        e_h = e_l = e_t = 0.0;
    } else {
        double x_r = rr, x_q = rq, x_sr = sr, x_sq = 1.0;
        for (int p = 1; p <= plimit; p++) {
            const double c = ct[p];
            if (!p_h) {
                double err = base * c * x_r;
                if (err <= maxerr) { p_h = p; e_h = err; }
            }
            if (!p_l) {
                double err = base * c * x_q;
                if (err <= maxerr) { p_l = p; e_l = err; }
            }
            if (!p_t) {
                double step = sq > 1.0 ? x_sq : 1.0;
                double err = base * c * (x_q + x_sr * cross[p] * step);
                if (err <= maxerr) { p_t = p; e_t = err; }
            }
            if (p_h && p_l && p_t) break;
            x_r *= rr;
            x_q *= rq;
            x_sr *= sr;
            x_sq *= sq;
        }
    }
    const double d = (double)dim;
    double c_h = CUDART_INF, c_l = CUDART_INF, c_t = CUDART_INF;
    if (p_h) c_h = n_query * pow(d, (double)(p_h + 1));
    if (p_l) c_l = n_ref * pow(d, (double)(p_l + 1));
    if (p_t) c_t = pow(d, (double)(2 * p_t + 1));
    const double c_x = d * n_query * n_ref;
    double c = fmin(fmin(c_h, c_l), fmin(c_t, c_x));
    if (c == c_h) { method = 2; order = p_h; bound = e_h; cost = c_h; return; }
    if (c == c_l) { method = 3; order = p_l; bound = e_l; cost = c_l; return; }
    if (c == c_t) { method = 4; order = p_t; bound = e_t; cost = c_t; return; }
    method = 0; order = 0; bound = 0.0; cost = c_x;
}

}  // namespace fg
