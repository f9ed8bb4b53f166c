// fg_device.cuh -- device helpers shared by the engine's kernels.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace fg {

constexpr unsigned kFull = 0xffffffffu;

// Packed stride (in doubles) of one point record: coordinates, weight, pad to
// an even count so records are 16-byte aligned (double2 loads).
__host__ __device__ constexpr int packed_stride(int dim) { return (dim + 2) & ~1; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

// Load the D coordinates (and weight) of a packed record.
template <int D>
__device__ __forceinline__ void load_point(const double *__restrict__ rec, double (&x)[D]) {
    constexpr int S = packed_stride(D);
    const double2 *r2 = reinterpret_cast<const double2 *>(rec);
#pragma unroll
    for (int k = 0; k < S / 2; k++) {
        double2 v = __ldg(r2 + k);
        if (2 * k < D) x[2 * k] = v.x;
        if (2 * k + 1 < D) x[2 * k + 1] = v.y;
    }
}

template <int D>
__device__ __forceinline__ void load_point_w(const double *__restrict__ rec, double (&x)[D],
                                             double &w) {
    constexpr int S = packed_stride(D);
    const double2 *r2 = reinterpret_cast<const double2 *>(rec);
#pragma unroll
    for (int k = 0; k < S / 2; k++) {
        double2 v = __ldg(r2 + k);
        if (2 * k < D) x[2 * k] = v.x;
        else if (2 * k == D) w = v.x;
        if (2 * k + 1 < D) x[2 * k + 1] = v.y;
        else if (2 * k + 1 == D) w = v.y;
    }
}

// Box-to-box squared distance bounds, inlined exactly as the reference's
// traversal computes them (summation_engine.py:315-326).
template <int D>
__device__ __forceinline__ void box_bounds(const double (&qlo)[D], const double (&qhi)[D],
                                           const double *__restrict__ rbox, double &min_sq,
                                           double &max_sq) {
    min_sq = 0.0;
    max_sq = 0.0;
#pragma unroll
    for (int d = 0; d < D; d++) {
        double rlo = __ldg(rbox + d), rhi = __ldg(rbox + D + d);
        double a = qlo[d] - rhi, b = rlo - qhi[d];
        double g = a > b ? a : b;
        if (g > 0.0) min_sq += g * g;
        double s1 = qhi[d] - rlo, s2 = rhi - qlo[d];
        double s = s1 > s2 ? s1 : s2;
        max_sq += s * s;
    }
}

}  // namespace fg
