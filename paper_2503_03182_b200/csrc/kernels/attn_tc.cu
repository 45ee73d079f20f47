// Tensor-core causal attention for bf16 (placeholder dispatch to the SIMT path
// until the mma kernels land).
#include "kernels.h"

namespace tpipe {
int attn_fwd_simt(int dtype, const void* qkv, void* o, float* lse, int b, int s, int a, int d,
                  cudaStream_t st);
int attn_bwd_simt(int dtype, const void* qkv, const void* o, const void* dout, const float* lse,
                  void* dqkv, float* ws, int b, int s, int a, int d, cudaStream_t st);

int attn_fwd_tc(const void* qkv, void* o, float* lse, int b, int s, int a, int d, cudaStream_t st) {
    return attn_fwd_simt(DT_BF16, qkv, o, lse, b, s, a, d, st);
}
int attn_bwd_tc(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                float* ws, int b, int s, int a, int d, cudaStream_t st) {
    return attn_bwd_simt(DT_BF16, qkv, o, dout, lse, dqkv, ws, b, s, a, d, st);
}
}  // namespace tpipe
