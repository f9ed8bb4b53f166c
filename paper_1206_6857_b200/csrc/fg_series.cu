// fg_series.cu -- batched device entry points for the series algebra and
// the selector (series_expansion.py, error_bounds.py:168-230).  The engine
// uses the same device routines inside the traversal; these entry points
// expose them for the Python mirror of the reference API and for parity.
#include <cuda_runtime.h>

#include <vector>

#include "fg_device.cuh"
#include "fg_internal.cuh"
#include "fg_series.cuh"

namespace fg {

__global__ void pack_rows_kernel(const double *__restrict__ pts, const double *__restrict__ w,
                                 int64_t n, int dim, int stride, double *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double *o = out + i * stride;
    for (int d = 0; d < dim; d++) o[d] = pts[i * dim + d];
    o[dim] = w ? w[i] : 1.0;
    for (int d = dim + 1; d < stride; d++) o[d] = 0.0;
}

template <int D>
__global__ void accumulate_batch_kernel(int kind, const double *__restrict__ pw,
                                        const int64_t *__restrict__ off, int batch,
                                        const double *__restrict__ centers, int p, int K,
                                        double sc, const uint8_t *__restrict__ digits,
                                        const double *__restrict__ inv_fact,
                                        double *__restrict__ out) {
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= batch) return;
    double c[D];
#pragma unroll
    for (int d = 0; d < D; d++) c[d] = centers[(int64_t)b * D + d];
    accumulate_warp<D>(kind, pw, off[b], off[b + 1], c, p, K, sc, digits, inv_fact,
                       out + (int64_t)b * K, true);
}

template <int D>
__global__ void eval_batch_kernel(int kind, const double *__restrict__ coeffs, int kstored,
                                  const double *__restrict__ centers, int batch, int p, int Kp,
                                  double sc, const double *__restrict__ x,
                                  const int64_t *__restrict__ off,
                                  const uint8_t *__restrict__ digits, double *__restrict__ out) {
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= batch) return;
    double c[D];
#pragma unroll
    for (int d = 0; d < D; d++) c[d] = centers[(int64_t)b * D + d];
    const double *A = coeffs + (int64_t)b * kstored;
    for (int64_t i = off[b] + lane; i < off[b + 1]; i += 32) {
        double xi[D];
#pragma unroll
        for (int d = 0; d < D; d++) xi[d] = x[i * D + d];
        out[i] = kind == 0 ? eval_far_lane<D>(xi, centers + (int64_t)b * D, A, p, Kp, sc, digits)
                           : eval_local_lane<D>(xi, c, A, p, Kp, sc, digits);
    }
}

template <int D>
__global__ void translate_batch_kernel(int kind, const double *__restrict__ coeffs, int kstored,
                                       const double *__restrict__ src_c,
                                       const double *__restrict__ dst_c, int batch, int ps,
                                       int Ks, int pd, int Kd, double sc,
                                       const uint8_t *__restrict__ digits,
                                       const double *__restrict__ inv_fact,
                                       const double *__restrict__ fact,
                                       const int *__restrict__ degrees,
                                       const int *__restrict__ off, const int2 *__restrict__ pr,
                                       double *__restrict__ out) {
    extern __shared__ double sh[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const bool live = b < batch;
    double *tab = sh + wib * (Kd > Ks ? Kd : Ks);
    const double *A = coeffs + (int64_t)(live ? b : 0) * kstored;
    double *o = out + (int64_t)(live ? b : 0) * Kd;
    double sc_[D], dc[D];
#pragma unroll
    for (int d = 0; d < D; d++) {
        sc_[d] = live ? src_c[(int64_t)b * D + d] : 0.0;
        dc[d] = live ? dst_c[(int64_t)b * D + d] : 0.0;
    }
    if (kind == 2) {
        if (!live) return;
        for (int k = lane; k < Kd; k += 32) o[k] = 0.0;
        __syncwarp();
        h2l_warp_add<D>(A, src_c + (int64_t)b * D, dc, ps, Ks, pd, Kd, sc, digits, inv_fact,
                        degrees, o);
        return;
    }
    // kind 0 (H2H): u = (old - new)/sc, shift[k] = u^k / k!, out[s] = sum A[a] shift[b]
    // kind 1 (L2L): u = (new - old)/sc, mono[k] = u^k,
    //               out[a] = sum C(s,a) B[s] mono[b] over pairs (a, b, s)
    double pwt[D][2 * kMaxOrder];
#pragma unroll
    for (int d = 0; d < D; d++) {
        const double u = kind == 0 ? (sc_[d] - dc[d]) / sc : (dc[d] - sc_[d]) / sc;
        power_ladder(u, ps - 1, pwt[d]);
    }
    for (int k = lane; k < Ks; k += 32) {
        double v = product<D>(digits_of(digits, k), pwt);
        tab[k] = kind == 0 ? v * inv_fact[k] : v;
    }
    __syncwarp();
    if (!live) return;
    for (int t = lane; t < Ks; t += 32) {
        double acc = 0.0;
        for (int q = off[t]; q < off[t + 1]; q++) {
            const int2 e = pr[q];
            if (kind == 0) {
                acc += A[e.x] * tab[e.y];  // (a, b) for this s
            } else {
                const int bb = e.x, s = e.y;  // (b, s) for this a
                const double binom = fact[s] * inv_fact[t] * inv_fact[bb];
                acc += binom * A[s] * tab[bb];
            }
        }
        o[t] = acc;
    }
}

__global__ void best_method_kernel(const double *__restrict__ geom, int batch, int dim,
                                   int plimit, TailArgs T, double *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch) return;
    const double *g = geom + (int64_t)i * 9;
    int method, order;
    double bound, cost;
    best_method_dev(g[0], g[2], g[3], g[4], g[5], g[6], dim, g[7], g[8], plimit, T.ct, T.cross,
                    method, order, bound, cost);
    double *o = out + (int64_t)i * 4;
    o[0] = method;
    o[1] = order;
    o[2] = bound;
    o[3] = cost;
}

}  // namespace fg

using namespace fg;

struct SeriesScr {
    DBuf a, b, c, d, out, pw;
};
#define FG_SERIES_SCRATCH                                                          \
    SeriesScr &ss_ = scratch<SeriesScr, SeriesScr>();                              \
    DBuf &g_s_a = ss_.a, &g_s_b = ss_.b, &g_s_c = ss_.c, &g_s_d = ss_.d,          \
         &g_s_out = ss_.out, &g_s_pw = ss_.pw;                                     \
    (void)g_s_a; (void)g_s_b; (void)g_s_c; (void)g_s_d; (void)g_s_out; (void)g_s_pw

#define FG_DISPATCH_D(DIM, CALL)                                             \
    switch (DIM) {                                                           \
        case 1: { constexpr int DD = 1; CALL; } break;                       \
        case 2: { constexpr int DD = 2; CALL; } break;                       \
        case 3: { constexpr int DD = 3; CALL; } break;                       \
        case 4: { constexpr int DD = 4; CALL; } break;                       \
        case 5: { constexpr int DD = 5; CALL; } break;                       \
        case 6: { constexpr int DD = 6; CALL; } break;                       \
        case 7: { constexpr int DD = 7; CALL; } break;                       \
        case 8: { constexpr int DD = 8; CALL; } break;                       \
        default: set_error("dimension > 8 unsupported"); return FG_EUNSUPPORTED; \
    }

extern "C" {

int fg_series_accumulate(int32_t kind, const double *pts, const double *w,
                         const int64_t *offsets, int32_t batch, int32_t dim,
                         const double *centers, int32_t order, double h, double *coeffs) {
    FG_SERIES_SCRATCH;
    FG_REQUIRE(batch >= 1 && dim >= 1 && offsets && centers && coeffs, FG_EINVAL, "bad args");
    FG_REQUIRE(order >= 1, FG_EINVAL, "truncation order must be at least 1");
    FG_REQUIRE(h > 0.0, FG_EINVAL, "bandwidth must be positive");
    int st = FG_OK;
    const SeriesTables *T = series_tables(dim, order, &st);
    FG_TRY(st);
    std::vector<int64_t> hoff(batch + 1);
    if (is_device_ptr(offsets)) {
        FG_CUDA_TRY(cudaMemcpy(hoff.data(), offsets, sizeof(int64_t) * (batch + 1),
                               cudaMemcpyDeviceToHost));
    } else {
        std::copy(offsets, offsets + batch + 1, hoff.begin());
    }
    const int64_t npts = hoff[batch];
    const void *dp = nullptr, *dw = nullptr, *doff, *dc;
    DBuf sp, sw, so, scn;
    if (npts > 0) {
        FG_TRY(to_device(pts, sizeof(double) * npts * dim, sp, &dp));
        FG_TRY(to_device(w, sizeof(double) * npts, sw, &dw));
    }
    FG_TRY(to_device(offsets, sizeof(int64_t) * (batch + 1), so, &doff));
    FG_TRY(to_device(centers, sizeof(double) * batch * dim, scn, &dc));
    const int S = packed_stride(dim);
    FG_TRY(g_s_pw.reserve(sizeof(double) * (npts > 0 ? npts : 1) * S));
    if (npts > 0) {
        count_launch();
        pack_rows_kernel<<<(unsigned)((npts + 255) / 256), 256, 0, stream()>>>(
            (const double *)dp, (const double *)dw, npts, dim, S, g_s_pw.as<double>());
    }
    FG_TRY(g_s_out.reserve(sizeof(double) * batch * T->K));
    const unsigned blocks = (unsigned)((batch * 32 + 127) / 128);
    count_launch();
    FG_DISPATCH_D(dim, (accumulate_batch_kernel<DD><<<blocks, 128, 0, stream()>>>(
                           kind, g_s_pw.as<double>(), (const int64_t *)doff, batch,
                           (const double *)dc, order, T->K, kSqrt2 * h,
                           T->digits.as<uint8_t>(), T->inv_fact.as<double>(),
                           g_s_out.as<double>())));
    FG_CUDA_TRY(cudaGetLastError());
    return from_device(coeffs, g_s_out.p, sizeof(double) * batch * T->K);
}

int fg_series_eval(int32_t kind, const double *coeffs, int32_t k_stored, const double *centers,
                   int32_t batch, int32_t dim, int32_t order, double h, const double *x,
                   const int64_t *offsets, double *out) {
    FG_SERIES_SCRATCH;
    FG_REQUIRE(batch >= 1 && dim >= 1 && coeffs && centers && x && offsets && out, FG_EINVAL,
               "bad args");
    FG_REQUIRE(order >= 1 && h > 0.0, FG_EINVAL, "bad order or bandwidth");
    int st = FG_OK;
    const SeriesTables *T = series_tables(dim, order, &st);
    FG_TRY(st);
    FG_REQUIRE(k_stored >= T->K, FG_EINVAL, "fewer stored coefficients than the order needs");
    std::vector<int64_t> hoff(batch + 1);
    if (is_device_ptr(offsets)) {
        FG_CUDA_TRY(cudaMemcpy(hoff.data(), offsets, sizeof(int64_t) * (batch + 1),
                               cudaMemcpyDeviceToHost));
    } else {
        std::copy(offsets, offsets + batch + 1, hoff.begin());
    }
    const int64_t npts = hoff[batch];
    const void *dco, *dc, *dx, *doff;
    DBuf s1, s2, s3, s4;
    FG_TRY(to_device(coeffs, sizeof(double) * batch * k_stored, s1, &dco));
    FG_TRY(to_device(centers, sizeof(double) * batch * dim, s2, &dc));
    FG_TRY(to_device(x, sizeof(double) * (npts > 0 ? npts : 1) * dim, s3, &dx));
    FG_TRY(to_device(offsets, sizeof(int64_t) * (batch + 1), s4, &doff));
    FG_TRY(g_s_out.reserve(sizeof(double) * (npts > 0 ? npts : 1)));
    const unsigned blocks = (unsigned)((batch * 32 + 127) / 128);
    count_launch();
    FG_DISPATCH_D(dim, (eval_batch_kernel<DD><<<blocks, 128, 0, stream()>>>(
                           kind, (const double *)dco, k_stored, (const double *)dc, batch,
                           order, T->K, kSqrt2 * h, (const double *)dx, (const int64_t *)doff,
                           T->digits.as<uint8_t>(), g_s_out.as<double>())));
    FG_CUDA_TRY(cudaGetLastError());
    return from_device(out, g_s_out.p, sizeof(double) * npts);
}

int fg_series_translate(int32_t kind, const double *coeffs, int32_t k_stored,
                        const double *src_centers, const double *dst_centers, int32_t batch,
                        int32_t dim, int32_t order_src, int32_t order, double h, double *out) {
    FG_SERIES_SCRATCH;
    FG_REQUIRE(batch >= 1 && dim >= 1 && coeffs && src_centers && dst_centers && out,
               FG_EINVAL, "bad args");
    FG_REQUIRE(order >= 1 && order_src >= 1 && h > 0.0, FG_EINVAL, "bad order or bandwidth");
    FG_REQUIRE(kind >= 0 && kind <= 2, FG_EINVAL, "bad translate kind");
    if (kind != 2) order_src = order;
    int st = FG_OK;
    const SeriesTables *Td = series_tables(dim, order, &st);
    FG_TRY(st);
    const SeriesTables *Ts = series_tables(dim, order_src, &st);
    FG_TRY(st);
    // H2L needs the digit table of the larger order (nested prefixes)
    const SeriesTables *Tbig = order >= order_src ? Td : Ts;
    FG_REQUIRE(k_stored >= Ts->K, FG_EINVAL, "fewer stored coefficients than the order needs");
    const void *dco, *dsc, *ddc;
    DBuf s1, s2, s3;
    FG_TRY(to_device(coeffs, sizeof(double) * batch * k_stored, s1, &dco));
    FG_TRY(to_device(src_centers, sizeof(double) * batch * dim, s2, &dsc));
    FG_TRY(to_device(dst_centers, sizeof(double) * batch * dim, s3, &ddc));
    FG_TRY(g_s_out.reserve(sizeof(double) * batch * Td->K));
    const int warps = 4;
    const unsigned blocks = (unsigned)((batch + warps - 1) / warps);
    const size_t smem = sizeof(double) * warps * (Td->K > Ts->K ? Td->K : Ts->K);
    const int *off = kind == 0 ? Td->h2h_off.as<int>() : Td->l2l_off.as<int>();
    const int2 *pr = kind == 0 ? Td->h2h_ab.as<int2>() : Td->l2l_bs.as<int2>();
    count_launch();
    FG_DISPATCH_D(dim, (translate_batch_kernel<DD><<<blocks, 32 * warps, smem, stream()>>>(
                           kind, (const double *)dco, k_stored, (const double *)dsc,
                           (const double *)ddc, batch, order_src, Ts->K, order, Td->K,
                           kSqrt2 * h, Tbig->digits.as<uint8_t>(),
                           Tbig->inv_fact.as<double>(), Tbig->fact.as<double>(),
                           Tbig->degrees.as<int>(), off, pr, g_s_out.as<double>())));
    FG_CUDA_TRY(cudaGetLastError());
    return from_device(out, g_s_out.p, sizeof(double) * batch * Td->K);
}

int fg_best_method(const double *geom, int32_t batch, int32_t dim, int32_t plimit, double *out) {
    FG_SERIES_SCRATCH;
    FG_REQUIRE(geom && out && batch >= 1 && dim >= 1 && plimit >= 1, FG_EINVAL, "bad args");
    FG_REQUIRE(plimit <= kMaxOrder, FG_EUNSUPPORTED, "plimit above the device order cap (12) is not supported");
    TailArgs T;
    double floor_c;
    tail_tables(dim, plimit, T.ct, T.cross, &floor_c);
    const void *dg;
    DBuf s1;
    FG_TRY(to_device(geom, sizeof(double) * batch * 9, s1, &dg));
    FG_TRY(g_s_out.reserve(sizeof(double) * batch * 4));
    count_launch();
    best_method_kernel<<<(batch + 127) / 128, 128, 0, stream()>>>(
        (const double *)dg, batch, dim, plimit, T, g_s_out.as<double>());
    FG_CUDA_TRY(cudaGetLastError());
    return from_device(out, g_s_out.p, sizeof(double) * batch * 4);
}

}  // extern "C"
