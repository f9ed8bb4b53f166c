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
#include "fg_exp.cuh"
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

__host__ __device__ constexpr int nest3_group(int m) {  // G(m): doubles of rows 1..m
    int g = 0;
    for (int n = 1; n <= m; n++) g += (n + 1) & ~1;
    return g;
}

// Staging permutation: position of graded-lex coefficient q (< K_p) in the
// order-p nested layout of the row machine below, all orders 1..PMAX
// concatenated (off[p] = first entry of order p).  The traversal kernel copies
// it to shared memory once per CTA.
template <int PMAX>
struct Nest3Perm {
    static constexpr int kTotal = (PMAX * (PMAX + 1) * (PMAX + 2) * (PMAX + 3)) / 24;  // sum of K_p
    unsigned short pos[kTotal];
    int off[PMAX + 2];
    constexpr Nest3Perm() : pos{}, off{} {
        constexpr GLex<3, PMAX> G{};
        int o = 0;
        off[0] = 0;
        for (int p = 1; p <= PMAX; p++) {
            off[p] = o;
            for (int q = 0; q < G.prefix[p]; q++) {
                const int a = G.dig[q][0], b = G.dig[q][1], c = G.dig[q][2];
                // groups in order of a; inside a group rows by ascending length
                int st = nest3_group(p - a - b - 1);
                for (int aa = 0; aa < a; aa++) st += nest3_group(p - aa);
                pos[o + q] = (unsigned short)(st + c);
            }
            o += G.prefix[p];
        }
        off[PMAX + 1] = o;
    }
};
// doubles per staged item (nested coefficients, then the centre in the last
// four): the order-10 layout takes 250, the order-12 layout 406
__host__ __device__ constexpr int nest3_slot(int plimit) { return plimit <= 10 ? 256 : 512; }

// ---- EVALM at D = 3: the row machine ---------------------------------------
// sum_{a+b+c<p} A_abc H_a(t0) H_b(t1) H_c(t2) e^{-|t|^2} for both query slots of
// a lane at the item's own order p (exactly K_p coefficient FMAs per slot) from
// ONE compact code region (~300 instructions for every order).  Straight-line
// code per order (K_p FMAs unrolled, ~60 KB for orders 1..10) reaches 0.4-0.5
// of the DFMA peak alone, but inside the traversal kernel, with the 16 warps of
// an SM at different items and orders, it is bound by instruction fetch (ncu:
// 66 % of stall samples "no instruction", 22 % issue utilisation; L0 ~6 KB,
// L1.5 32 KB): profiles/r02_hermite_evaluators.txt.
// Layout (Nest3Perm): groups a = 0 .. p-1; group a (m = p - a rows) stores its
// rows in ASCENDING length n = 1 .. m (b = m - n), every row padded to an even
// length so that it is read with 16-byte loads.  The chain block_1, block_2,
// ... is specialised on the row length (straight-line inner sums over c, the
// inner ladder H_c(t2) in registers), entered at block_1 and left after
// block_m.  Sum_b S_b H_b(t1) is folded by Clenshaw's recurrence
// y_b = S_b + 2 t1 y_{b+1} - 2 (b + 1) y_{b+2} (result y_0): two FMAs per row
// and slot and no middle ladder; H_a(t0) is advanced once per group.
#ifndef FG_ROWS123
#define FG_ROWS123 1
#endif
constexpr int kRowPairs = (kMaxOrder + 1) / 2;  // 16-byte pairs of the longest row
// 16-byte shared-memory load that stays where it is written (the compiler sinks
// an ordinary load down to its first use, which undoes the row prefetch)
__device__ __forceinline__ double2 lds_pair(unsigned addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
template <int N, int PMAX>
__device__ __forceinline__ void far3_row_cl(unsigned gs, const double (&l2a)[kMaxOrder],
                                            const double (&l2b)[kMaxOrder], double t1a,
                                            double t1b, double &twob, double &y1a, double &y2a,
                                            double &y1b, double &y2b,
                                            const double2 (&v)[kRowPairs],
                                            double2 (&pre)[kRowPairs]) {
    // this row's coefficients were loaded one block ahead (`v`); load the next
    // row's now into the other register set (inside the staged slot even when
    // this is the group's last row)
    constexpr int NPN = N < PMAX ? (N + 2) / 2 : 0;
#pragma unroll
    for (int k = 0; k < NPN; k++) pre[k] = lds_pair(gs + 8 * nest3_group(N) + 16 * k);
    double ea = 0.0, oa = 0.0, eb = 0.0, ob = 0.0;
#pragma unroll
    for (int cc = 0; cc < N; cc += 2) {
        const double2 w = v[cc >> 1];
        if (cc == 0) {
            ea = w.x;
            eb = w.x;
        } else {
            ea = fma(w.x, l2a[cc], ea);
            eb = fma(w.x, l2b[cc], eb);
        }
        if (cc + 1 < N) {
            if (N >= 6) {  // two partial sums per slot on long rows
                oa = cc == 0 ? w.y * l2a[1] : fma(w.y, l2a[cc + 1], oa);
                ob = cc == 0 ? w.y * l2b[1] : fma(w.y, l2b[cc + 1], ob);
            } else {
                ea = fma(w.y, l2a[cc + 1], ea);
                eb = fma(w.y, l2b[cc + 1], eb);
            }
        }
    }
    if (N >= 6) {
        ea += oa;
        eb += ob;
    }
    if (N == 1) {
        y1a = ea;
        y1b = eb;
    } else {
        const double na = fma(t1a, y1a, N == 2 ? ea : fma(-twob, y2a, ea));
        const double nb = fma(t1b, y1b, N == 2 ? eb : fma(-twob, y2b, eb));
        y2a = y1a;
        y1a = na;
        y2b = y1b;
        y1b = nb;
    }
    twob -= 2.0;
}

template <int PMAX>
__device__ __forceinline__ void far3_rows_cl(int p, const double (&ta)[3], const double (&tb)[3],
                                             const double *A, double &va, double &vb) {
    static_assert(PMAX <= kMaxOrder && PMAX <= 12, "row chain covers orders up to 12");
    double l2a[kMaxOrder], l2b[kMaxOrder];  // registers
    l2a[0] = l2b[0] = 1.0;
    l2a[1] = 2.0 * ta[2];
    l2b[1] = 2.0 * tb[2];
#pragma unroll
    for (int n = 1; n + 1 < PMAX; n++) {
        if (n + 1 < p) {  // (uniform)
            l2a[n + 1] = 2.0 * ta[2] * l2a[n] - 2.0 * n * l2a[n - 1];
            l2b[n + 1] = 2.0 * tb[2] * l2b[n] - 2.0 * n * l2b[n - 1];
        }
    }
    const double t1a = 2.0 * ta[1], t1b = 2.0 * tb[1];
    double acca = 0.0, ha = 1.0, ham = 0.0, accb = 0.0, hb = 1.0, hbm = 0.0, twoa = 0.0;
    unsigned gs = (unsigned)__cvta_generic_to_shared(A);  // group start (byte address)
#pragma unroll 1
    for (int m = p; m >= 1; m--) {
        double y1a = 0.0, y2a = 0.0, y1b = 0.0, y2b = 0.0;
        double twob = 2.0 * m;  // 2 (b + 1) of the row being folded
        double2 pre0[kRowPairs], pre1[kRowPairs];  // rows of odd / even length
#if FG_ROWS123
        if (m >= 3 && PMAX >= 4) {
            // rows 1, 2, 3 of the group (6 coefficients in 4 pairs) in one block:
            // one branch instead of three, their sums independent
            const double2 r1 = lds_pair(gs), r2 = lds_pair(gs + 16), r3 = lds_pair(gs + 32),
                          r3b = lds_pair(gs + 48);
            pre1[0] = lds_pair(gs + 64);  // row 4, should the group have one
            pre1[1] = lds_pair(gs + 80);
            const double s2a = fma(r2.y, l2a[1], r2.x), s2b = fma(r2.y, l2b[1], r2.x);
            const double s3a = fma(r3b.x, l2a[2], fma(r3.y, l2a[1], r3.x));
            const double s3b = fma(r3b.x, l2b[2], fma(r3.y, l2b[1], r3.x));
            // Clenshaw: y(row 1) = S1; y(row 2) = S2 + t1 S1; y(row 3) = S3 + t1 y(row 2) - (2m - 4) S1
            const double ya = fma(t1a, r1.x, s2a), yb = fma(t1b, r1.x, s2b);
            const double c3 = 4.0 - twob;
            y1a = fma(t1a, ya, fma(c3, r1.x, s3a));
            y1b = fma(t1b, yb, fma(c3, r1.x, s3b));
            y2a = ya;
            y2b = yb;
            twob -= 6.0;
            if (m > 3) {
                do {
#define FG_ROWC(N)                                                                  \
    if constexpr (N <= PMAX) {                                                      \
        far3_row_cl<N, PMAX>(gs, l2a, l2b, t1a, t1b, twob, y1a, y2a, y1b, y2b,       \
                             (N & 1) ? pre0 : pre1, (N & 1) ? pre1 : pre0);          \
        if (m == N) break;                                                          \
    }
                    FG_ROWC(4) FG_ROWC(5) FG_ROWC(6) FG_ROWC(7) FG_ROWC(8) FG_ROWC(9)
                    FG_ROWC(10) FG_ROWC(11) FG_ROWC(12)
#undef FG_ROWC
                } while (0);
            }
        } else
#endif
        {
        pre0[0] = lds_pair(gs);
        do {
#define FG_ROWC(N)                                                                  \
    if constexpr (N <= PMAX) {                                                      \
        far3_row_cl<N, PMAX>(gs, l2a, l2b, t1a, t1b, twob, y1a, y2a, y1b, y2b,       \
                             (N & 1) ? pre0 : pre1, (N & 1) ? pre1 : pre0);          \
        if (m == N) break;                                                          \
    }
#if FG_ROWS123
            FG_ROWC(1) FG_ROWC(2)
#else
            FG_ROWC(1) FG_ROWC(2) FG_ROWC(3) FG_ROWC(4) FG_ROWC(5) FG_ROWC(6) FG_ROWC(7)
            FG_ROWC(8) FG_ROWC(9) FG_ROWC(10) FG_ROWC(11) FG_ROWC(12)
#endif
#undef FG_ROWC
        } while (0);
        }
        gs += ((m + 1) >> 1) * (((m + 1) >> 1) + ((m & 1) ? 0 : 1)) * 16;  // G(m) doubles
        acca = fma(y1a, ha, acca);
        accb = fma(y1b, hb, accb);
        const double hna = 2.0 * ta[0] * ha - twoa * ham;
        const double hnb = 2.0 * tb[0] * hb - twoa * hbm;
        ham = ha;
        ha = hna;
        hbm = hb;
        hb = hnb;
        twoa += 2.0;
    }
    va = acca;
    vb = accb;
}

// out-of-line instance (the ladders then do not weigh on the caller's registers);
// the item is addressed through the dynamic shared-memory window so that its
// loads stay shared-memory loads across the call
template <int PMAX>
__device__ __noinline__ double2 far3_rows_cl_call(int p, double a0, double a1, double a2,
                                                  double b0, double b1, double b2, int off) {
    extern __shared__ double fg_dyn_smem[];
    const double ta[3] = {a0, a1, a2}, tb[3] = {b0, b1, b2};
    double2 r;
    far3_rows_cl<PMAX>(p, ta, tb, fg_dyn_smem + off, r.x, r.y);
    return r;
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
template <int D, int KSLOTS = kMaxK / 32>
__device__ void accumulate_warp(int kind, const double *__restrict__ pw_pts, int64_t r0,
                                int64_t r1, const double (&c)[D], int p, int Kp, double sc,
                                const uint8_t *__restrict__ digits,
                                const double *__restrict__ inv_fact, double *out,
                                bool overwrite) {
    constexpr int S = packed_stride(D);
    const int lane = threadIdx.x & 31;
    double acc[KSLOTS];
    uint64_t dg[KSLOTS];
#pragma unroll
    for (int j = 0; j < KSLOTS; j++) {
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
        for (int j = 0; j < KSLOTS; j++) {
            if (32 * j < Kp) acc[j] += w * product<D>(dg[j], tab);
        }
    }
#pragma unroll
    for (int j = 0; j < KSLOTS; j++) {
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
                                                double maxerr, int plimit, int plimit_loc,
                                                const double *ct,
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
        if (!p_l && p <= plimit_loc) {
            double err = base * c * x_q;
            if (err <= maxerr) { p_l = p; e_l = err; }
        }
        if (!p_t && p <= plimit_loc) {
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
                                                  int plimit, int plimit_loc, const double *ct,
                                                  const double *cross, const int *kp, double nq,
                                                  double pair_cost, double herm_c0,
                                                  double herm_c1, int &method, int &order,
                                                  double &bound) {
    int p_h, p_l, p_t;
    double e_h, e_l, e_t;
    feasible_orders(base, r_ref, r_query, maxerr, plimit, plimit_loc, ct, cross, p_h, p_l, p_t,
                    e_h, e_l, e_t);
    const double d = (double)dim;
    double c_h = CUDART_INF, c_l = CUDART_INF, c_t = CUDART_INF;
    if (p_h) c_h = nq * (herm_c0 + kp[p_h] * herm_c1);
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
