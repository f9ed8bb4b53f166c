// ex2_accuracy.cu -- measures the relative error of ex2.approx.ftz.f32 against
// exp2 in FP64 over the argument range the FP32 base case uses ([-116, 0]),
// sweeping every FP32 value in the range.  The bound fp32_item_bound assumes
// <= 2^-21.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// /tmp/ex2acc tools/ex2_accuracy.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__global__ void sweep(uint32_t lo_bits, uint32_t count, unsigned long long *worst) {
    const uint32_t stride = gridDim.x * blockDim.x;
    double m = 0.0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float v = __uint_as_float(lo_bits + i);  // negative floats: bits grow with |v|
        float r;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
        const double e = exp2((double)v);
        const double rel = fabs((double)r - e) / e;
        m = fmax(m, rel);
    }
    atomicMax(worst, (unsigned long long)__double_as_longlong(m));
}

int main() {
    const float lo = -0.0f, hi = -116.0f;
    uint32_t b0, b1;
    memcpy(&b0, &lo, 4);
    memcpy(&b1, &hi, 4);
    unsigned long long *w;
    cudaMallocManaged(&w, 8);
    *w = 0;
    sweep<<<148 * 8, 256>>>(b0, b1 - b0 + 1, w);
    cudaDeviceSynchronize();
    double m;
    memcpy(&m, w, 8);
    printf("ex2.approx.ftz.f32 max rel error on [-116, 0]: %.3e (2^%.2f)\n", m, log2(m));
    return 0;
}
