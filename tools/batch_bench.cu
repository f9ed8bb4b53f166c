// Microbenchmark of the FP32 batch loop alone (no traversal): every warp
// streams a staged batch of anchored FP32 records with batch_f32, as the
// traversal kernel does, at the traversal's launch shape.  Reports pairs/s
// against the ex2 (SFU) bound.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1206_6857_b200/csrc tools/batch_bench.cu -o tools/batch_bench
#include <cstdio>
#include "fg_traverse_kernel.cuh"

using namespace fg;

template <int D, int MB>
__global__ void __launch_bounds__(128, MB) bench_kernel(int reps, int items, int per_item, float *out) {
    constexpr int F = fstride<D>(), FD = f32_fd<D>();
    __shared__ float fst[4][256 * F];
    __shared__ int itab[4][64];
    __shared__ float idl[4][32 * FD];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < 256 * F; i += 32) fst[w][i] = (i % F == D) ? 1e-5f : 0.01f * ((i * 7) % 13);
    for (int t = lane; t < items; t += 32) {
        itab[w][t] = t * per_item;
        itab[w][32 + t] = per_item;
        for (int d = 0; d < D; d++) idl[w][t * FD + d] = 0.001f * d;
    }
    __syncwarp();
    unsigned long long xf2[D];
    for (int d = 0; d < D; d++) xf2[d] = f2_pack(0.01f * lane, 0.02f * lane);
    double s = 0.0;
    for (int r = 0; r < reps; r++) {
        double s0, s1;
        batch_f32<D>(xf2, fst[w], itab[w], itab[w] + 32, idl[w], items, -0.5f, s0, s1);
        s += s0 + s1;
    }
    out[blockIdx.x * 128 + threadIdx.x] = (float)s;
}

// dot-form candidate: records {y_0..y_{D-1}, |y|^2, w} (8 floats at D <= 6);
// per item the lane forms q2s_d = 2 s xq_d and aq = -s |xq|^2 (packed)
template <int D>
__device__ __forceinline__ void batch_dot(const unsigned long long (&xf2)[D], const float *fst,
                                          const int *ioff, const int *icnt, int nitems, float s,
                                          double &sum0, double &sum1) {
    constexpr int F = (D + 2 + 3) & ~3;
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
    const unsigned long long ms2 = f2_pack(-s, -s), ts2 = f2_pack(2.f * s, 2.f * s);
#pragma unroll 1
    for (int it = 0; it < nitems; it++) {
        const int off = ioff[it], cnt = icnt[it];
        unsigned long long q2[D], aq = 0ull;
#pragma unroll
        for (int d = 0; d < D; d++) {
            q2[d] = f2_mul(xf2[d], ts2);
            aq = d == 0 ? f2_mul(xf2[d], xf2[d]) : f2_fma(xf2[d], xf2[d], aq);
        }
        aq = f2_mul(aq, ms2);
        const float *rec = fst + off * F;
        for (int j = 0; j + 4 <= cnt; j += 4) {
            float y[4][F];
#pragma unroll
            for (int u = 0; u < 4; u++)
#pragma unroll
                for (int k = 0; k < F; k += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(rec + (j + u) * F + k);
                    y[u][k] = v.x; y[u][k + 1] = v.y; y[u][k + 2] = v.z; y[u][k + 3] = v.w;
                }
            unsigned long long t[4];
#pragma unroll
            for (int u = 0; u < 4; u++) t[u] = f2_fma(f2_pack(y[u][D], y[u][D]), ms2, aq);
#pragma unroll
            for (int d = 0; d < D; d++)
#pragma unroll
                for (int u = 0; u < 4; u++) f2_fma_acc(t[u], q2[d], f2_pack(y[u][d], y[u][d]));
#pragma unroll
            for (int u = 0; u < 4; u++) f2_fma_acc(acc[u], f2_ex2(t[u]), f2_pack(y[u][D + 1], y[u][D + 1]));
        }
    }
    sum0 = ((double)f2_lo(acc[0]) + (double)f2_lo(acc[1])) + ((double)f2_lo(acc[2]) + (double)f2_lo(acc[3]));
    sum1 = ((double)f2_hi(acc[0]) + (double)f2_hi(acc[1])) + ((double)f2_hi(acc[2]) + (double)f2_hi(acc[3]));
}

template <int D, int U>
__device__ __forceinline__ void batch_diff_u(const unsigned long long (&xf2)[D], const float *fst,
                                            const int *ioff, const int *icnt, const float *idl,
                                            int nitems, float ex2s, double &sum0, double &sum1) {
    constexpr int F = fstride<D>(), FD = f32_fd<D>();
    const unsigned long long s2 = f2_pack(ex2s, ex2s);
    unsigned long long acc[U];
#pragma unroll
    for (int u = 0; u < U; u++) acc[u] = 0ull;
#pragma unroll 1
    for (int it = 0; it < nitems; it++) {
        const int off = ioff[it], cnt = icnt[it];
        unsigned long long q2[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            const float dv = idl[it * FD + d];
            q2[d] = f2_sub(xf2[d], f2_pack(dv, dv));
        }
        const float *rec = fst + off * F;
        for (int j = 0; j + U <= cnt; j += U) {
            float y[U][F];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int k = 0; k < F; k += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(rec + (j + u) * F + k);
                    y[u][k] = v.x; y[u][k + 1] = v.y; y[u][k + 2] = v.z; y[u][k + 3] = v.w;
                }
            unsigned long long dd[U];
#pragma unroll
            for (int d = 0; d < D; d++)
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const unsigned long long f = f2_sub(q2[d], f2_pack(y[u][d], y[u][d]));
                    dd[u] = d == 0 ? f2_mul(f, f) : f2_fma(f, f, dd[u]);
                }
#pragma unroll
            for (int u = 0; u < U; u++) dd[u] = f2_ex2(f2_mul(dd[u], s2));
#pragma unroll
            for (int u = 0; u < U; u++) f2_fma_acc(acc[u], dd[u], f2_pack(y[u][D], y[u][D]));
        }
    }
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int u = 0; u < U; u++) {
        a0 += (double)f2_lo(acc[u]);
        a1 += (double)f2_hi(acc[u]);
    }
    sum0 = a0;
    sum1 = a1;
}

template <int D, int MB, int U>
__global__ void __launch_bounds__(128, MB) bench_u(int reps, int items, int per_item, float *out) {
    constexpr int F = fstride<D>(), FD = f32_fd<D>();
    __shared__ float fst[4][256 * F];
    __shared__ int itab[4][64];
    __shared__ float idl[4][32 * FD];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < 256 * F; i += 32) fst[w][i] = (i % F == D) ? 1e-5f : 0.01f * ((i * 7) % 13);
    for (int t = lane; t < items; t += 32) {
        itab[w][t] = t * per_item;
        itab[w][32 + t] = per_item;
        for (int d = 0; d < D; d++) idl[w][t * FD + d] = 0.001f * d;
    }
    __syncwarp();
    unsigned long long xf2[D];
    for (int d = 0; d < D; d++) xf2[d] = f2_pack(0.01f * lane, 0.02f * lane);
    double s = 0.0;
    for (int r = 0; r < reps; r++) {
        double s0, s1;
        batch_diff_u<D, U>(xf2, fst[w], itab[w], itab[w] + 32, idl[w], items, -0.5f, s0, s1);
        s += s0 + s1;
    }
    out[blockIdx.x * 128 + threadIdx.x] = (float)s;
}

template <int D, int MB, int U>
void run_u(int items, int per_item) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * MB, reps = 2000;
    float *out;
    cudaMalloc(&out, sizeof(float) * grid * 128);
    bench_u<D, MB, U><<<grid, 128>>>(10, items, per_item, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench_u<D, MB, U><<<grid, 128>>>(reps, items, per_item, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * 4 * reps * items * per_item * 64;
    printf("DIFF U=%d D=%d MINB=%d items=%d x %d records: %.3e pairs/s (%.1f%% of 4.63e12 ex2 bound)\n", U, D, MB,
           items, per_item, pairs / (ms * 1e-3), 100.0 * pairs / (ms * 1e-3) / 4.63e12);
    cudaFree(out);
}

template <int D, int MB>
__global__ void __launch_bounds__(128, MB) bench_dot(int reps, int items, int per_item, float *out) {
    constexpr int F = (D + 2 + 3) & ~3;
    __shared__ float fst[4][256 * F];
    __shared__ int itab[4][64];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < 256 * F; i += 32) fst[w][i] = (i % F == D + 1) ? 1e-5f : 0.01f * ((i * 7) % 13);
    for (int t = lane; t < items; t += 32) {
        itab[w][t] = t * per_item;
        itab[w][32 + t] = per_item;
    }
    __syncwarp();
    unsigned long long xf2[D];
    for (int d = 0; d < D; d++) xf2[d] = f2_pack(0.01f * lane, 0.02f * lane);
    double s = 0.0;
    for (int r = 0; r < reps; r++) {
        double s0, s1;
        batch_dot<D>(xf2, fst[w], itab[w], itab[w] + 32, items, 0.5f, s0, s1);
        s += s0 + s1;
    }
    out[blockIdx.x * 128 + threadIdx.x] = (float)s;
}

template <int D, int MB>
void run_dot(int items, int per_item) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * MB, reps = 2000;
    float *out;
    cudaMalloc(&out, sizeof(float) * grid * 128);
    bench_dot<D, MB><<<grid, 128>>>(10, items, per_item, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench_dot<D, MB><<<grid, 128>>>(reps, items, per_item, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * 4 * reps * items * per_item * 64;
    printf("DOT D=%d MINB=%d items=%d x %d records: %.3f ms, %.3e pairs/s (%.1f%% of 4.63e12 ex2 bound)\n", D, MB,
           items, per_item, ms, pairs / (ms * 1e-3), 100.0 * pairs / (ms * 1e-3) / 4.63e12);
    cudaFree(out);
}

template <int D, int MB>
void run(int items, int per_item) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * MB, reps = 2000;
    float *out;
    cudaMalloc(&out, sizeof(float) * grid * 128);
    bench_kernel<D, MB><<<grid, 128>>>(10, items, per_item, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench_kernel<D, MB><<<grid, 128>>>(reps, items, per_item, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = (double)grid * 4 * reps * items * per_item * 64;
    printf("D=%d MINB=%d items=%d x %d records: %.3f ms, %.3e pairs/s (%.1f%% of 4.63e12 ex2 bound)\n", D, MB,
           items, per_item, ms, pairs / (ms * 1e-3), 100.0 * pairs / (ms * 1e-3) / 4.63e12);
    cudaFree(out);
}

int main() {
    run<3, 4>(8, 32);
    run<3, 4>(16, 16);
    run<3, 4>(4, 64);
    run<3, 4>(32, 8);
    run<3, 3>(8, 32);
    run<2, 4>(8, 32);
    run_u<3, 4, 4>(8, 32);
    run_u<3, 4, 8>(8, 32);
    run_u<3, 4, 2>(8, 32);
    run_u<3, 3, 8>(8, 32);
    run_dot<3, 4>(8, 32);
    run_dot<3, 4>(16, 16);
    run_dot<3, 4>(4, 64);
    run_dot<2, 4>(8, 32);
    return 0;
}
