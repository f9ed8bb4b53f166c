// fg_exp.cuh -- FP64 exp used by the pair kernels.
//
// The exhaustive and base-case kernels are FP64-pipe bound and exp is most of
// the per-pair DP work.  libdevice's exp costs 16 DP-pipe ops (degree-11
// polynomial) plus a slow-path test.  fg_exp_fast uses a 64-entry table of
// 2^(j/64) in shared memory, so the reduced argument |r| <= ln2/128 needs only
// a degree-5 polynomial: 10 DP-pipe ops.  Accuracy: <= 1 ulp against glibc's
// exp over [-708.3, 0] (20M-point sweep, tools/exp_accuracy.c); arguments below
// -708.3 (subnormal or zero results) take the libdevice path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fg {

static __constant__ double c_exp_tab[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};

// 64-bit FP immediates with a non-zero low word cannot be encoded in DFMA; nvcc
// then re-materialises them through two UMOVs at every use.  Reading them from
// the constant bank lets DFMA take them as c[][] operands for free.
static __constant__ double c_exp_coef[6] = {
    0x1.71547652b82fep+6,     // 64 / ln 2
    0x1.62e42fee00000p-7,     // ln 2 / 64, high part (32 significant bits)
    0x1.a39ef35793c76p-39,    // ln 2 / 64, low part
    1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0};

// copy the table to shared memory; call with all threads of the CTA, then sync
__device__ __forceinline__ void exp_table_init(double *s_tab) {
    for (int i = threadIdx.x; i < 64; i += blockDim.x) s_tab[i] = c_exp_tab[i];
}

// Fast path only: valid for x >= -708.3 (normal results).  Callers that can
// bound their arguments (a pair of boxes with K_lo >= DBL_MIN) use this
// directly and skip the range test.
__device__ __forceinline__ double fg_exp_normal(double x, const double *s_tab) {
    const double magic = 6755399441055744.0;  // 1.5 * 2^52: round to nearest integer
    double kd = fma(x, c_exp_coef[0], magic);
    const int k = __double2loint(kd);
    kd -= magic;
    double r = fma(kd, -c_exp_coef[1], x);
    r = fma(kd, -c_exp_coef[2], r);
    double q = fma(r, c_exp_coef[3], c_exp_coef[4]);
    q = fma(q, r, c_exp_coef[5]);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    const double t = s_tab[k & 63];
    const double y = fma(t, r * q, t);
    return __hiloint2double(__double2hiint(y) + ((k >> 6) << 20), __double2loint(y));
}

// Register-resident constants for hot loops.  The values pass through an
// opaque `mov` so the compiler cannot re-materialise them (LDC / UMOV pairs)
// inside the loop, and the table is addressed with a 32-bit shared-window
// address, avoiding a per-use generic-to-shared conversion.
struct ExpK {
    double l2e, ln2hi, ln2lo, c5, c4, c3;
    unsigned tab;  // shared-memory address of the 2^(j/64) table
};

__device__ __forceinline__ double opaque(double v) {
    double r;
    asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
    return r;
}

__device__ __forceinline__ ExpK exp_consts(const double *s_tab) {
    ExpK k;
    k.l2e = opaque(c_exp_coef[0]);
    k.ln2hi = opaque(-c_exp_coef[1]);
    k.ln2lo = opaque(-c_exp_coef[2]);
    k.c5 = opaque(c_exp_coef[3]);
    k.c4 = opaque(c_exp_coef[4]);
    k.c3 = opaque(c_exp_coef[5]);
    unsigned a = (unsigned)__cvta_generic_to_shared(s_tab);
    asm volatile("mov.b32 %0, %1;" : "=r"(k.tab) : "r"(a));
    return k;
}

// fg_exp_normal with register constants (x >= -708.3)
__device__ __forceinline__ double fg_exp_k(double x, const ExpK &K) {
    const double magic = 6755399441055744.0;
    double kd = fma(x, K.l2e, magic);
    const int k = __double2loint(kd);
    kd -= magic;
    double r = fma(kd, K.ln2hi, x);
    r = fma(kd, K.ln2lo, r);
    double q = fma(r, K.c5, K.c4);
    q = fma(q, r, K.c3);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    double t;
    asm("ld.shared.f64 %0, [%1];" : "=d"(t) : "r"(K.tab + ((unsigned)(k & 63) << 3)));
    const double y = fma(t, r * q, t);
    return __hiloint2double(__double2hiint(y) + ((k >> 6) << 20), __double2loint(y));
}

// full range with register constants: zero below -745.2, libdevice in the
// subnormal band (rare)
__device__ __forceinline__ double fg_exp_kc(double x, const ExpK &K) {
    if (x < -708.3) return x < -745.2 ? 0.0 : exp(x);
    return fg_exp_k(x, K);
}

__device__ __forceinline__ double fg_exp_fast(double x, const double *s_tab) {
    if (x < -708.3) return x < -745.2 ? 0.0 : exp(x);
    return fg_exp_normal(x, s_tab);
}

__device__ __forceinline__ double fg_exp(double x) { return exp(x); }

}  // namespace fg
