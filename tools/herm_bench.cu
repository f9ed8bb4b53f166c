// Microbenchmark of the D = 3 Hermite far-field evaluators alone (no
// traversal): every warp evaluates `items` staged expansions for its two query
// slots at the traversal kernel's launch shape (4 CTAs x 4 warps per SM).
// Reports evaluations/s and the share of the DFMA peak the counted FMAs reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -lineinfo -I paper_1206_6857_b200/csrc tools/herm_bench.cu -o tools/herm_bench
#include <cstdio>
#include <cstdlib>
#include <cuda_pipeline.h>
#include "fg_series.cuh"

using namespace fg;

constexpr int kSlot = 256;  // doubles per ring slot
constexpr int kRingN = 4;

// V: 0 = masked fixed-order (old), 1 = exact order graded-lex LDS.64,
//    2 = exact order nested layout (16-byte loads), 3 = nested, both slots fused
template <int V, int PP, int PMAX>
__global__ void __launch_bounds__(128, 4) herm_kernel(int items, const double *__restrict__ mom,
                                                      int nnodes, int stage, double *out) {
    extern __shared__ double smem[];
    __shared__ double s_tab[kExpTab];
    exp_table_init(s_tab);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *ring = smem + w * kRingN * kSlot;
    constexpr int KP = glex_count(3, PP);
    for (int i = lane; i < kRingN * kSlot; i += 32) ring[i] = 1e-3 * ((i * 7) % 13 - 6);
    __syncwarp();
    double x[2][3];
    for (int d = 0; d < 3; d++) {
        x[0][d] = 0.01 * lane + 0.1 * d;
        x[1][d] = 0.013 * lane - 0.1 * d;
    }
    const double c[3] = {0.3, 0.2, 0.1};
    double e0 = 0.0, e1 = 0.0;
    unsigned node = (blockIdx.x * 4 + w) * 977u;
    auto stage_item = [&](int k) {
        node = node * 1664525u + 1013904223u;
        const double *src = mom + (size_t)(node % (unsigned)nnodes) * kSlot;
        double *dst = ring + (k % kRingN) * kSlot;
        for (int q = lane; q < KP; q += 32) __pipeline_memcpy_async(dst + q, src + q, 8);
    };
    if (stage)
        for (int k = 0; k < kRingN - 1; k++) {
            stage_item(k);
            __pipeline_commit();
        }
#pragma unroll 1
    for (int it = 0; it < items; it++) {
        if (stage) {
            if (it + kRingN - 1 < items) stage_item(it + kRingN - 1);
            __pipeline_commit();
            __pipeline_wait_prior(kRingN - 1);
            __syncwarp();
        }
        const double *A0 = ring + (it % kRingN) * kSlot;
        const double inv_sc = 1.0 + 1e-9 * it;
        if constexpr (V == 0) {
#pragma unroll 1
            for (int q = 0; q < 2; q++) {
                const double *A = A0;
                asm volatile("" : "+l"(A));  // no hoisting / sharing of the coefficient loads
                double xq[3] = {q ? x[1][0] : x[0][0], q ? x[1][1] : x[0][1], q ? x[1][2] : x[0][2]};
                const double v = eval_far_fixed3<PMAX>(xq, c, A, PP, inv_sc,
                                                       [&](double t) { return fg_exp_fast(t, s_tab); });
                if (q) e1 += v; else e0 += v;
            }
        } else if constexpr (V == 1) {
#pragma unroll 1
            for (int q = 0; q < 2; q++) {
                const double *A = A0;
                asm volatile("" : "+l"(A));  // no hoisting / sharing of the coefficient loads
                const double t0 = ((q ? x[1][0] : x[0][0]) - c[0]) * inv_sc;
                const double t1 = ((q ? x[1][1] : x[0][1]) - c[1]) * inv_sc;
                const double t2 = ((q ? x[1][2] : x[0][2]) - c[2]) * inv_sc;
                const double g = fg_exp_fast(-(t0 * t0 + t1 * t1 + t2 * t2), s_tab);
                const double v = far3_poly<PP, PMAX>(t0, t1, t2, A) * g;
                if (q) e1 += v; else e0 += v;
            }
        } else if constexpr (V == 2) {
#pragma unroll 1
            for (int q = 0; q < 2; q++) {
                const double *A = A0;
                asm volatile("" : "+l"(A));  // no hoisting / sharing of the coefficient loads
                const double t0 = ((q ? x[1][0] : x[0][0]) - c[0]) * inv_sc;
                const double t1 = ((q ? x[1][1] : x[0][1]) - c[1]) * inv_sc;
                const double t2 = ((q ? x[1][2] : x[0][2]) - c[2]) * inv_sc;
                const double g = fg_exp_fast(-(t0 * t0 + t1 * t1 + t2 * t2), s_tab);
                const double v = far3_nested<PP>(t0, t1, t2, A) * g;
                if (q) e1 += v; else e0 += v;
            }
        } else {
            double ta[3], tb[3];
            for (int d = 0; d < 3; d++) {
                ta[d] = (x[0][d] - c[d]) * inv_sc;
                tb[d] = (x[1][d] - c[d]) * inv_sc;
            }
            const double ga = fg_exp_fast(-(ta[0] * ta[0] + ta[1] * ta[1] + ta[2] * ta[2]), s_tab);
            const double gb = fg_exp_fast(-(tb[0] * tb[0] + tb[1] * tb[1] + tb[2] * tb[2]), s_tab);
            double va, vb;
            far3_nested2<PP>(ta, tb, A0, va, vb);
            e0 += va * ga;
            e1 += vb * gb;
        }
        if (stage) __syncwarp();
    }
    out[blockIdx.x * 128 + threadIdx.x] = e0 + e1;
}

template <int V, int PP, int PMAX>
void run(int items, const double *mom, int nnodes, int stage, double *out, double peak_tflops) {
    auto kern = herm_kernel<V, PP, PMAX>;
    const size_t smem = sizeof(double) * 4 * kRingN * kSlot + 16 * 1024;  // ~48 KB: 4 CTAs per SM
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 4;
    kern<<<grid, 128, smem>>>(items / 8, mom, nnodes, stage, out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    kern<<<grid, 128, smem>>>(items, mom, nnodes, stage, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    const double evals = (double)grid * 128 * 2 * items;
    const int K = glex_count(3, PP);
    const double fma = K + (PP + 1) * PP / 2 + PP;  // counted FMAs per evaluation
    const double tf = evals * fma * 2 / (ms * 1e-3) / 1e12;
    printf("V%d p=%2d stage=%d: %8.3f ms  %.3e evals/s  %6.1f cycles/warp-eval  counted %.2f TF (%.2f of DFMA peak) %s\n",
           V, PP, stage, ms, evals / (ms * 1e-3), ms * 1e-3 * 1.965e9 * 148 * 16 / (evals / 32), tf,
           tf / peak_tflops, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char **argv) {
    const int items = argc > 1 ? atoi(argv[1]) : 2000;
    const int nnodes = 200000;
    double *mom, *out;
    cudaMalloc(&mom, sizeof(double) * (size_t)nnodes * kSlot);
    cudaMemset(mom, 0, sizeof(double) * (size_t)nnodes * kSlot);
    cudaMalloc(&out, sizeof(double) * 148 * 4 * 128);
    const double peak = 33.7;
    for (int stage = 0; stage < 2; stage++) {
        run<0, 6, 6>(items, mom, nnodes, stage, out, peak);
        run<0, 10, 10>(items, mom, nnodes, stage, out, peak);
        run<1, 4, 10>(items, mom, nnodes, stage, out, peak);
        run<1, 6, 10>(items, mom, nnodes, stage, out, peak);
        run<1, 8, 10>(items, mom, nnodes, stage, out, peak);
        run<1, 10, 10>(items, mom, nnodes, stage, out, peak);
        run<2, 4, 10>(items, mom, nnodes, stage, out, peak);
        run<2, 6, 10>(items, mom, nnodes, stage, out, peak);
        run<2, 8, 10>(items, mom, nnodes, stage, out, peak);
        run<2, 10, 10>(items, mom, nnodes, stage, out, peak);
        run<3, 4, 10>(items, mom, nnodes, stage, out, peak);
        run<3, 6, 10>(items, mom, nnodes, stage, out, peak);
        run<3, 8, 10>(items, mom, nnodes, stage, out, peak);
        run<3, 10, 10>(items, mom, nnodes, stage, out, peak);
    }
    return 0;
}
