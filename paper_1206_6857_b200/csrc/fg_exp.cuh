// fg_exp.cuh -- FP64 exp used by the pair kernels.
//
// The exhaustive and base-case kernels are FP64-pipe bound and exp is ~70% of
// the per-pair DP work.  fg_exp is the single switch point for the exp
// implementation used by those kernels ("exp").
#pragma once
#include <cuda_runtime.h>

namespace fg {

__device__ __forceinline__ double fg_exp(double x) { return exp(x); }

}  // namespace fg
