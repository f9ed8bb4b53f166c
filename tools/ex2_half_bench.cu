// Throughput of ex2.approx: f32 against f16x2 / bf16x2 (two results per instruction?)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ex2_half_bench.cu -o tools/ex2_half_bench
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k_f32(int n, float *out) {
    float a = threadIdx.x * 1e-3f, b = a + 0.1f, c = a + 0.2f, d = a + 0.3f;
    for (int i = 0; i < n; i++) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
        a -= 1.f; b -= 1.f; c -= 1.f; d -= 1.f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_f16x2(int n, unsigned *out) {
    unsigned a = 0x3c003800u + threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    const unsigned one = 0x3c003c00u;
    for (int i = 0; i < n; i++) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a));
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b));
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(c));
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(d));
        asm volatile("sub.f16x2 %0, %0, %1;" : "+r"(a) : "r"(one));
        asm volatile("sub.f16x2 %0, %0, %1;" : "+r"(b) : "r"(one));
        asm volatile("sub.f16x2 %0, %0, %1;" : "+r"(c) : "r"(one));
        asm volatile("sub.f16x2 %0, %0, %1;" : "+r"(d) : "r"(one));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_bf16x2(int n, unsigned *out) {
    unsigned a = 0x3f803f00u + threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    const unsigned one = 0x3f803f80u;
    for (int i = 0; i < n; i++) {
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(c));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(d));
        asm volatile("sub.bf16x2 %0, %0, %1;" : "+r"(a) : "r"(one));
        asm volatile("sub.bf16x2 %0, %0, %1;" : "+r"(b) : "r"(one));
        asm volatile("sub.bf16x2 %0, %0, %1;" : "+r"(c) : "r"(one));
        asm volatile("sub.bf16x2 %0, %0, %1;" : "+r"(d) : "r"(one));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
template <class F> void timeit(const char *name, F f, double per_thread_iter) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    f(1000); cudaDeviceSynchronize();
    const int n = 20000;
    cudaEventRecord(e0); f(n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)148 * 8 * 256 * n * per_thread_iter;
    printf("%s: %.3f ms, %.3e results/s (%.2f per clk per SM at 1.965 GHz) %s\n", name, ms, ops / (ms * 1e-3),
           ops / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    float *o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    timeit("ex2 f32   ", [&](int n) { k_f32<<<148 * 8, 256>>>(n, o); }, 4);
    timeit("ex2 f16x2 ", [&](int n) { k_f16x2<<<148 * 8, 256>>>(n, (unsigned *)o); }, 8);
    timeit("ex2 bf16x2", [&](int n) { k_bf16x2<<<148 * 8, 256>>>(n, (unsigned *)o); }, 8);
    return 0;
}
