// fg_naive.cu -- K1: exhaustive FP64 Gaussian sums (replaces naive_sum,
// summation_engine.py:122-154).
//
// Layout: queries and references are packed into 16-byte-aligned AoS records
// (coords, weight, pad).  A CTA owns 256*QPT queries held in registers and
// streams a slice of the references through shared memory in tiles; every
// thread reads the same reference record (broadcast LDS), so the inner loop
// is pure FP64 pipe work: D DADD + D DFMA + 1 DMUL + exp + 1 DFMA per pair.
// The reference range is split across blockIdx.y so that small M still fills
// 148 SMs; partial sums are combined in a fixed order (deterministic).
#include <vector>

#include "fg_device.cuh"
#include "fg_exp.cuh"
#include "fg_internal.cuh"

namespace fg {

constexpr int kNaiveThreads = 256;
constexpr int kNaiveTile = 256;

// Pack row-major (n x dim) coordinates (+ optional weights) into records.
// records of the kernel dimension kd >= dim: coordinates, zero padding, weight
__global__ void pack_points_kernel(const double *__restrict__ pts, const double *__restrict__ w,
                                   int64_t n, int dim, int kd, int stride, double *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double *o = out + i * stride;
    for (int d = 0; d < kd; d++) o[d] = d < dim ? pts[i * dim + d] : 0.0;
    o[kd] = w ? w[i] : 1.0;
    for (int d = kd + 1; d < stride; d++) o[d] = 0.0;
}

// CTA-wide min of lo[] and max of hi[]; every thread gets the result
template <int D>
__device__ __forceinline__ void block_minmax(double (&lo)[D], double (&hi)[D], double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = kNaiveThreads / 32;
#pragma unroll
    for (int d = 0; d < D; d++) {
        lo[d] = warp_min(lo[d]);
        hi[d] = warp_max(hi[d]);
    }
    __syncthreads();  // previous users of sh are done
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; d++) {
            sh[wid * 2 * D + d] = lo[d];
            sh[wid * 2 * D + D + d] = hi[d];
        }
    }
    __syncthreads();
#pragma unroll
    for (int d = 0; d < D; d++) {
        lo[d] = sh[d];
        hi[d] = sh[D + d];
        for (int k = 1; k < NW; k++) {
            lo[d] = fmin(lo[d], sh[k * 2 * D + d]);
            hi[d] = fmax(hi[d], sh[k * 2 * D + D + d]);
        }
    }
}

// one reference record against this thread's QPT queries
template <int D, int QPT, bool CHECKED>
__device__ __forceinline__ void naive_pair_step(const double (&x)[QPT][D], const double *rec,
                                                double neg_inv, const ExpK &K, double (&acc)[QPT]) {
    constexpr int S = packed_stride(D);
    double y[D], w;
    const double2 *t2 = reinterpret_cast<const double2 *>(rec);
#pragma unroll
    for (int k = 0; k < S / 2; k++) {
        const double2 v = t2[k];
        if (2 * k < D) y[2 * k] = v.x;
        else if (2 * k == D) w = v.x;
        if (2 * k + 1 < D) y[2 * k + 1] = v.y;
        else if (2 * k + 1 == D) w = v.y;
    }
#pragma unroll
    for (int i = 0; i < QPT; i++) {
        const double diff = x[i][0] - y[0];
        double d2 = diff * diff;
#pragma unroll
        for (int d = 1; d < D; d++) {
            const double df = x[i][d] - y[d];
            d2 = fma(df, df, d2);
        }
        const double e = CHECKED ? fg_exp_kc(d2 * neg_inv, K) : fg_exp_k(d2 * neg_inv, K);
        acc[i] = fma(e, w, acc[i]);
    }
}

template <int D, int QPT>
__global__ void __launch_bounds__(kNaiveThreads)
naive_kernel(const double *__restrict__ q, int64_t m, const double *__restrict__ r, int64_t n,
             int64_t rchunk, double neg_inv, double *__restrict__ part) {
    constexpr int S = packed_stride(D);
    __shared__ __align__(16) double tile[kNaiveTile * S];
    __shared__ double s_tab[kExpTab];
    __shared__ double s_red[2 * D * (kNaiveThreads / 32)];
    exp_table_init(s_tab);
    const ExpK K = exp_consts(s_tab);
    const int64_t q0 = (int64_t)blockIdx.x * kNaiveThreads * QPT;
    const int64_t r0 = (int64_t)blockIdx.y * rchunk;
    const int64_t r1 = min(n, r0 + rchunk);
    double x[QPT][D], acc[QPT];
#pragma unroll
    for (int i = 0; i < QPT; i++) {
        int64_t qi = q0 + threadIdx.x + (int64_t)i * kNaiveThreads;
        acc[i] = 0.0;
        if (qi < m) {
            load_point<D>(q + qi * S, x[i]);
        } else {
#pragma unroll
            for (int d = 0; d < D; d++) x[i][d] = 0.0;
        }
    }
    // bounding box of this CTA's queries (uniform across the CTA)
    double qlo[D], qhi[D];
#pragma unroll
    for (int d = 0; d < D; d++) {
        qlo[d] = CUDART_INF;
        qhi[d] = -CUDART_INF;
#pragma unroll
        for (int i = 0; i < QPT; i++) {
            if (q0 + threadIdx.x + (int64_t)i * kNaiveThreads < m) {
                qlo[d] = fmin(qlo[d], x[i][d]);
                qhi[d] = fmax(qhi[d], x[i][d]);
            }
        }
    }
    block_minmax<D>(qlo, qhi, s_red);
    for (int64_t t0 = r0; t0 < r1; t0 += kNaiveTile) {
        const int cnt = (int)min((int64_t)kNaiveTile, r1 - t0);
        __syncthreads();
        {
            const double2 *src = reinterpret_cast<const double2 *>(r + t0 * S);
            double2 *dst = reinterpret_cast<double2 *>(tile);
            for (int k = threadIdx.x; k < cnt * S / 2; k += kNaiveThreads) dst[k] = __ldg(src + k);
        }
        __syncthreads();  // the tile is complete before anyone reads a record
        // tile box -> skip the tile (every exp underflows to exactly 0), run the
        // range-test-free exp (every argument >= -708), or the checked exp
        double tlo[D], thi[D];
        {
            const bool v = threadIdx.x < cnt;
#pragma unroll
            for (int d = 0; d < D; d++) {
                tlo[d] = v ? tile[threadIdx.x * S + d] : CUDART_INF;
                thi[d] = v ? tile[threadIdx.x * S + d] : -CUDART_INF;
            }
            block_minmax<D>(tlo, thi, s_red);
        }
        double min_sq = 0.0, max_sq = 0.0;
#pragma unroll
        for (int d = 0; d < D; d++) {
            const double g = fmax(fmax(qlo[d] - thi[d], tlo[d] - qhi[d]), 0.0);
            min_sq += g * g;
            const double s = fmax(qhi[d] - tlo[d], thi[d] - qlo[d]);
            max_sq += s * s;
        }
        if (min_sq * neg_inv < -746.0) continue;
        if (max_sq * neg_inv > -708.0) {
#pragma unroll 2
            for (int j = 0; j < cnt; j++) naive_pair_step<D, QPT, false>(x, tile + j * S, neg_inv, K, acc);
        } else {
#pragma unroll 2
            for (int j = 0; j < cnt; j++) naive_pair_step<D, QPT, true>(x, tile + j * S, neg_inv, K, acc);
        }
    }
#pragma unroll
    for (int i = 0; i < QPT; i++) {
        int64_t qi = q0 + threadIdx.x + (int64_t)i * kNaiveThreads;
        if (qi < m) part[(int64_t)blockIdx.y * m + qi] = acc[i];
    }
}

__global__ void reduce_parts_kernel(const double *__restrict__ part, int64_t m, int nsplit,
                                    double *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    double s = 0.0;
    for (int k = 0; k < nsplit; k++) s += part[(int64_t)k * m + i];
    out[i] = s;
}

template <int D>
static int launch_naive(const double *dq, int64_t m, const double *dr, int64_t n, double h,
                        double *dpart, int nsplit, int64_t rchunk, int64_t qtiles) {
    constexpr int QPT = (D <= 4) ? 2 : 1;
    dim3 grid((unsigned)qtiles, (unsigned)nsplit);
    count_launch();
    naive_kernel<D, QPT><<<grid, kNaiveThreads, 0, stream()>>>(dq, m, dr, n, rchunk,
                                                               -0.5 / (h * h), dpart);
    FG_CUDA_TRY(cudaGetLastError());
    return FG_OK;
}

struct NaiveScr {
    DBuf q, r, part;
};

int naive_sum(const double *d_q, int64_t m, const double *d_r, const double *d_w, int64_t n,
              int dim_user, const double *hs, int nh, double *d_out) {
    const int dim = kernel_dim(dim_user);
    FG_REQUIRE(dim > 0, FG_EUNSUPPORTED, "naive_sum: dimension > 16 is not supported by this build");
    const int S = packed_stride(dim);
    NaiveScr &ns = scratch<NaiveScr, NaiveScr>();
    DBuf &g_naive_q = ns.q, &g_naive_r = ns.r, &g_naive_part = ns.part;
    FG_TRY(g_naive_q.reserve(sizeof(double) * m * S));
    FG_TRY(g_naive_r.reserve(sizeof(double) * n * S));
    count_launch();
    pack_points_kernel<<<(unsigned)((m + 255) / 256), 256, 0, stream()>>>(
        d_q, nullptr, m, dim_user, dim, S, g_naive_q.as<double>());
    count_launch();
    pack_points_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream()>>>(
        d_r, d_w, n, dim_user, dim, S, g_naive_r.as<double>());
    FG_CUDA_TRY(cudaGetLastError());
    const int qpt = dim <= 4 ? 2 : 1;
    const int64_t qtiles = (m + kNaiveThreads * qpt - 1) / (kNaiveThreads * qpt);
    // aim for >= 6 CTAs per SM worth of work; split the reference range
    int64_t target = 148 * 6;
    int64_t nsplit = (target + qtiles - 1) / qtiles;
    int64_t max_split = (n + kNaiveTile - 1) / kNaiveTile;
    if (nsplit > max_split) nsplit = max_split;
    if (nsplit < 1) nsplit = 1;
    if (nsplit > 65535) nsplit = 65535;
    int64_t rchunk = (n + nsplit - 1) / nsplit;
    rchunk = (rchunk + kNaiveTile - 1) / kNaiveTile * kNaiveTile;
    nsplit = (n + rchunk - 1) / rchunk;
    FG_TRY(g_naive_part.reserve(sizeof(double) * m * nsplit));
    for (int k = 0; k < nh; k++) {
        const double h = hs[k];
        int st = FG_OK;
        switch (dim) {
#define FG_NAIVE_CASE(DD)                                                                   \
    case DD:                                                                                \
        st = launch_naive<DD>(g_naive_q.as<double>(), m, g_naive_r.as<double>(), n, h,      \
                              g_naive_part.as<double>(), (int)nsplit, rchunk, qtiles);      \
        break;
            FG_NAIVE_CASE(1)
            FG_NAIVE_CASE(2)
            FG_NAIVE_CASE(3)
            FG_NAIVE_CASE(4)
            FG_NAIVE_CASE(5)
            FG_NAIVE_CASE(6)
            FG_NAIVE_CASE(7)
            FG_NAIVE_CASE(8)
            FG_NAIVE_CASE(12)
            FG_NAIVE_CASE(16)
#undef FG_NAIVE_CASE
            default:
                set_error("naive_sum: dimension > 16 is not supported by this build");
                return FG_EUNSUPPORTED;
        }
        FG_TRY(st);
        count_launch();
        reduce_parts_kernel<<<(unsigned)((m + 255) / 256), 256, 0, stream()>>>(
            g_naive_part.as<double>(), m, (int)nsplit, d_out + (int64_t)k * m);
        FG_CUDA_TRY(cudaGetLastError());
    }
    return FG_OK;
}

}  // namespace fg
