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

// Every warp draws its own order sequence in [plo, phi] (warps desynchronised,
// as in the traversal kernel) and evaluates with the row machine far3_rows_cl.
template <int V, int PP, int PMAX>
__global__ void __launch_bounds__(128, 4) herm_kernel(int items, const double *__restrict__ mom,
                                                      int nnodes, int plo, int phi, double *out,
                                                      unsigned long long *terms) {
    extern __shared__ double smem[];
    __shared__ double s_tab[kExpTab];
    exp_table_init(s_tab);
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *ring = smem + w * kRingN * kSlot;
    for (int i = lane; i < kRingN * kSlot; i += 32) ring[i] = 1e-3 * ((i * 7) % 13 - 6);
    __syncwarp();
    double x[2][3];
    for (int d = 0; d < 3; d++) {
        x[0][d] = 0.01 * lane + 0.1 * d;
        x[1][d] = 0.013 * lane - 0.1 * d;
    }
    const double c[3] = {0.3, 0.2, 0.1};
    double e0 = 0.0, e1 = 0.0;
    unsigned node = (blockIdx.x * 4 + w) * 977u + 12345u, prng = (blockIdx.x * 4 + w) * 7919u + 1u;
    unsigned long long nterms = 0;
    auto order_of = [&](int k) {
        unsigned v = (prng + 2654435761u * (unsigned)k);
        v ^= v >> 15; v *= 2246822519u; v ^= v >> 13;
        return plo + (int)(v % (unsigned)(phi - plo + 1));
    };
    auto stage_item = [&](int k) {
        node = node * 1664525u + 1013904223u;
        const int kc = glex_count(3, order_of(k));
        const double *src = mom + (size_t)(node % (unsigned)nnodes) * kSlot;
        double *dst = ring + (k % kRingN) * kSlot;
        for (int q = lane; q < kc; q += 32) __pipeline_memcpy_async(dst + q, src + q, 8);
    };
    for (int k = 0; k < kRingN - 1; k++) {
        stage_item(k);
        __pipeline_commit();
    }
#pragma unroll 1
    for (int it = 0; it < items; it++) {
        if (it + kRingN - 1 < items) stage_item(it + kRingN - 1);
        __pipeline_commit();
        __pipeline_wait_prior(kRingN - 1);
        __syncwarp();
        const double *A0 = ring + (it % kRingN) * kSlot;
        const double inv_sc = 1.0 + 1e-9 * it;
        const int p = order_of(it);
        nterms += glex_count(3, p);
        double ta[3], tb[3];
        for (int d = 0; d < 3; d++) {
            ta[d] = (x[0][d] - c[d]) * inv_sc;
            tb[d] = (x[1][d] - c[d]) * inv_sc;
        }
        const double ga = fg_exp_fast(-(ta[0] * ta[0] + ta[1] * ta[1] + ta[2] * ta[2]), s_tab);
        const double gb = fg_exp_fast(-(tb[0] * tb[0] + tb[1] * tb[1] + tb[2] * tb[2]), s_tab);
        double va, vb;
        far3_rows_cl<PMAX>(p, ta, tb, A0, va, vb);
        e0 += va * ga;
        e1 += vb * gb;
        __syncwarp();
    }
    out[blockIdx.x * 128 + threadIdx.x] = e0 + e1;
    if (lane == 0) atomicAdd(terms, nterms);
}

template <int V, int PP, int PMAX>
void run(int items, const double *mom, int nnodes, int plo, int phi, double *out,
         unsigned long long *terms, double peak_tflops) {
    auto kern = herm_kernel<V, PP, PMAX>;
    const size_t smem = sizeof(double) * 4 * kRingN * kSlot + 16 * 1024;  // ~48 KB: 4 CTAs per SM
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 4;
    kern<<<grid, 128, smem>>>(items / 8, mom, nnodes, plo, phi, out, terms);
    cudaDeviceSynchronize();
    cudaMemset(terms, 0, 8);
    cudaEventRecord(a);
    kern<<<grid, 128, smem>>>(items, mom, nnodes, plo, phi, out, terms);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    unsigned long long ht = 0;
    cudaMemcpy(&ht, terms, 8, cudaMemcpyDeviceToHost);
    const double evals = (double)grid * 128 * 2 * items;
    // bench.py's Hermite leg: 2 K_p + 31 + 4 D flops per evaluation
    const double flops = (double)ht * 64 * 2 + evals * 43;
    const double tf = flops / (ms * 1e-3) / 1e12;
    printf("p=%d..%d: %8.3f ms  %.3e evals/s  mean K_p %.1f  counted %.2f TF (%.2f of DFMA peak) %s\n",
           plo, phi, ms, evals / (ms * 1e-3),
           (double)ht / ((double)grid * 4 * items), tf, tf / peak_tflops,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char **argv) {
    const int items = argc > 1 ? atoi(argv[1]) : 2000;
    const int nnodes = 200000;
    double *mom, *out;
    unsigned long long *terms;
    cudaMalloc(&mom, sizeof(double) * (size_t)nnodes * kSlot);
    cudaMemset(mom, 0, sizeof(double) * (size_t)nnodes * kSlot);
    cudaMalloc(&out, sizeof(double) * 148 * 4 * 128);
    cudaMalloc(&terms, 8);
    const double peak = 33.7;
    const int ranges[][2] = {{10, 10}, {8, 8}, {6, 6}, {4, 4}, {2, 10}, {6, 10}, {2, 6}};
    for (auto &r : ranges) run<9, 0, 10>(items, mom, nnodes, r[0], r[1], out, terms, peak);
    return 0;
}
