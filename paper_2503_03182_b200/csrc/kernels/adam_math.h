// AdamW element arithmetic shared by the device kernel (K9) and the host
// optimizer of T-Offload (K10). Every operation is an explicitly
// rounded fp32 op (no FMA contraction: device uses __f*_rn intrinsics, host
// code is compiled with -ffp-contract=off), so host and device results are
// bit-identical ("offload on/off bit-exact").
#pragma once
#include <cmath>
#include "kernels.h"

// __host__/__device__/__forceinline__ come from cuda_runtime.h (via kernels.h)
// in both nvcc and plain g++ compilation.

namespace tpipe {

struct AdamOut {
    float w, m, v;
};

__host__ __device__ __forceinline__ float f_mul(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fmul_rn(a, b);
#else
    return a * b;
#endif
}
__host__ __device__ __forceinline__ float f_add(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}
__host__ __device__ __forceinline__ float f_sub(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fsub_rn(a, b);
#else
    return a - b;
#endif
}
__host__ __device__ __forceinline__ float f_div(float a, float b) {
#ifdef __CUDA_ARCH__
    return __fdiv_rn(a, b);
#else
    return a / b;
#endif
}
__host__ __device__ __forceinline__ float f_sqrt(float a) {
#ifdef __CUDA_ARCH__
    return __fsqrt_rn(a);
#else
    return sqrtf(a);
#endif
}

__host__ __device__ __forceinline__ AdamOut adam_elem(float w, float m, float v, float g, int decay,
                                                      const AdamHyper& hp) {
    if (decay) w = f_mul(w, f_sub(1.0f, f_mul(hp.lr, hp.wd)));
    m = f_add(f_mul(hp.b1, m), f_mul(f_sub(1.0f, hp.b1), g));
    v = f_add(f_mul(hp.b2, v), f_mul(f_mul(f_sub(1.0f, hp.b2), g), g));
    const float mhat = f_div(m, hp.bc1);
    const float vhat = f_div(v, hp.bc2);
    const float den = f_add(f_sqrt(vhat), hp.eps);
    w = f_sub(w, f_mul(hp.lr, f_div(mhat, den)));
    return {w, m, v};
}

}  // namespace tpipe
