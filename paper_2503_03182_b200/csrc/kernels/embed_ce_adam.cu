// Embedding (K7), cross-entropy (K8 softmax part), AdamW (K9) and small
// helpers. All deterministic: no floating-point atomics anywhere.
#include <cstring>

#include "adam_math.h"
#include "common.cuh"
#include "kernels.h"

namespace tpipe {

// ============================================================== embedding
template <typename T>
__global__ void embed_fwd_kernel(const int* __restrict__ tok, const T* __restrict__ wte,
                                 const T* __restrict__ wpe, T* __restrict__ x, int rows, int s,
                                 int h) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)rows * h) return;
    const int r = (int)(i / h), c = (int)(i % h);
    const float v = to_f<T>(wte[(long)tok[r] * h + c]) + to_f<T>(wpe[(long)(r % s) * h + c]);
    x[i] = from_f<T>(v);
}

int embed_fwd(int dtype, const int* tok, const void* wte, const void* wpe, void* x, int rows,
              int s, int h, cudaStream_t st) {
    if (rows <= 0) return 0;
    const long n = (long)rows * h;
    const int blocks = (int)((n + 255) / 256);
    if (dtype == DT_BF16)
        embed_fwd_kernel<bf16><<<blocks, 256, 0, st>>>(tok, (const bf16*)wte, (const bf16*)wpe,
                                                       (bf16*)x, rows, s, h);
    else
        embed_fwd_kernel<float><<<blocks, 256, 0, st>>>(tok, (const float*)wte, (const float*)wpe,
                                                        (float*)x, rows, s, h);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// Single-CTA bitonic sort of keys (tok << 15 | row) in shared memory.
__global__ void embed_sort_kernel(const int* __restrict__ tok, int* __restrict__ keys_out, int rows,
                                  int n_pow2) {
    extern __shared__ unsigned int sk[];
    for (int i = threadIdx.x; i < n_pow2; i += blockDim.x)
        sk[i] = i < rows ? ((unsigned)tok[i] << 15) | (unsigned)i : 0xFFFFFFFFu;
    __syncthreads();
    for (int k = 2; k <= n_pow2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    unsigned a = sk[i], b = sk[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        sk[i] = b;
                        sk[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < rows; i += blockDim.x) keys_out[i] = (int)sk[i];
}

// One CTA per sorted position; run-start CTAs sum their run in row order.
template <typename T>
__global__ void embed_wte_bwd_kernel(const int* __restrict__ keys, const T* __restrict__ dx,
                                     float* __restrict__ dwte, int rows, int h) {
    const int i = blockIdx.x;
    const unsigned k = (unsigned)keys[i];
    const unsigned t = k >> 15;
    if (i > 0 && ((unsigned)keys[i - 1] >> 15) == t) return;
    int end = i + 1;
    while (end < rows && ((unsigned)keys[end] >> 15) == t) ++end;
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
        float s = 0.f;
        for (int j = i; j < end; ++j) {
            const int r = (int)((unsigned)keys[j] & 0x7FFFu);
            s += to_f<T>(dx[(long)r * h + c]);
        }
        dwte[(long)t * h + c] += s;
    }
}

template <typename T>
__global__ void embed_wpe_bwd_kernel(const T* __restrict__ dx, float* __restrict__ dwpe, int rows,
                                     int s, int h) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)s * h) return;
    const int t = (int)(i / h), c = (int)(i % h);
    float acc = 0.f;
    for (int r = t; r < rows; r += s) acc += to_f<T>(dx[(long)r * h + c]);
    dwpe[i] += acc;
}

int embed_bwd(int dtype, const int* tok, const void* dx, float* dwte, float* dwpe, int* ws,
              int rows, int s, int h, cudaStream_t st) {
    if (rows <= 0) return 0;
    if (rows > 32768) return -1;
    int n2 = 1;
    while (n2 < rows) n2 <<= 1;
    const size_t smem = (size_t)n2 * 4;
    static PerDeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(embed_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             32768 * 4);
    }
    embed_sort_kernel<<<1, 1024, smem, st>>>(tok, ws, rows, n2);
    const int wpe_blocks = (int)(((long)s * h + 255) / 256);
    if (dtype == DT_BF16) {
        embed_wte_bwd_kernel<bf16><<<rows, 256, 0, st>>>(ws, (const bf16*)dx, dwte, rows, h);
        embed_wpe_bwd_kernel<bf16><<<wpe_blocks, 256, 0, st>>>((const bf16*)dx, dwpe, rows, s, h);
    } else {
        embed_wte_bwd_kernel<float><<<rows, 256, 0, st>>>(ws, (const float*)dx, dwte, rows, h);
        embed_wpe_bwd_kernel<float><<<wpe_blocks, 256, 0, st>>>((const float*)dx, dwpe, rows, s, h);
    }
    note_launches(3);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ============================================================== cross entropy
__global__ void ce_lse_kernel(const float* __restrict__ logits, float* __restrict__ lse, int V) {
    const int r = blockIdx.x;
    const float* l = logits + (long)r * V;
    __shared__ float red[32];
    float mx = -INFINITY;
    for (int c = threadIdx.x; c < V; c += blockDim.x) mx = fmaxf(mx, l[c]);
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
        v = warp_max(v);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    mx = red[0];
    __syncthreads();
    float s = 0.f;
    for (int c = threadIdx.x; c < V; c += blockDim.x) s += expf(l[c] - mx);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) lse[r] = mx + logf(v);
    }
}

// one block: loss_out[0] += scale * sum_r (lse_r - logit[r, tgt_r]); fixed tree order
__global__ void ce_loss_kernel(const float* __restrict__ logits, const int* __restrict__ tgt,
                               const float* __restrict__ lse, float* __restrict__ loss_out,
                               float scale, int rows, int V) {
    __shared__ float red[32];
    float s = 0.f;
    for (int r = threadIdx.x; r < rows; r += blockDim.x)
        s += lse[r] - logits[(long)r * V + tgt[r]];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) loss_out[0] += v * scale;
    }
}

// single pass: per-thread online (max, sum), float4 loads, block combine in a
// fixed order (V % 4 == 0)
__device__ __forceinline__ void lse_push(float& m, float& s, float x) {
    if (x > m) {
        s = s * expf(m - x) + 1.0f;
        m = x;
    } else {
        s += expf(x - m);
    }
}

__global__ void ce_lse1_kernel(const float* __restrict__ logits, float* __restrict__ lse, int V) {
    const int r = blockIdx.x;
    const float4* l4 = reinterpret_cast<const float4*>(logits + (long)r * V);
    __shared__ float rm[32], rsum[32];
    float m = -INFINITY, s = 0.f;
    for (int c = threadIdx.x; c < V / 4; c += blockDim.x) {
        const float4 v = l4[c];
        lse_push(m, s, v.x);
        lse_push(m, s, v.y);
        lse_push(m, s, v.z);
        lse_push(m, s, v.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {   // combine (m, s) pairs within the warp
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float mm = fmaxf(m, m2);
        s = (m == -INFINITY ? 0.f : s * expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mm));
        m = mm;
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        rm[w] = m;
        rsum[w] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY;
        for (int i = 0; i < nw; ++i) M = fmaxf(M, rm[i]);
        float S = 0.f;
        for (int i = 0; i < nw; ++i) S += rm[i] == -INFINITY ? 0.f : rsum[i] * expf(rm[i] - M);
        lse[r] = M + logf(S);
    }
}

__global__ void ce_bwd4_kernel(const float* __restrict__ logits, const int* __restrict__ tgt,
                               const float* __restrict__ lse, bf16* __restrict__ d, float scale,
                               int rows, int V) {
    const long i4 = (long)blockIdx.x * blockDim.x + threadIdx.x;   // float4 index
    if (i4 >= (long)rows * V / 4) return;
    const long i = i4 * 4;
    const int r = (int)(i / V), c = (int)(i % V);
    const float4 v = reinterpret_cast<const float4*>(logits)[i4];
    const float L = lse[r];
    const int t = tgt[r];
    float p0 = expf(v.x - L), p1 = expf(v.y - L), p2 = expf(v.z - L), p3 = expf(v.w - L);
    if (t == c) p0 -= 1.f;
    if (t == c + 1) p1 -= 1.f;
    if (t == c + 2) p2 -= 1.f;
    if (t == c + 3) p3 -= 1.f;
    __nv_bfloat162 a = __floats2bfloat162_rn(p0 * scale, p1 * scale);
    __nv_bfloat162 b = __floats2bfloat162_rn(p2 * scale, p3 * scale);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    reinterpret_cast<uint2*>(d)[i4] = u;
}

// one warp per row: lane l folds groups l, l+32, ... in order, then a fixed
// xor-tree combines the lanes (deterministic)
__global__ void ce_combine_kernel(const float2* __restrict__ part, int ngrp, const float* __restrict__ zt,
                                  float* __restrict__ lse, float* __restrict__ lrow, int rows) {
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float2* p = part + (size_t)r * ngrp;
    float m = -INFINITY, s = 0.f;
    for (int j = lane; j < ngrp; j += 32) {
        const float2 q = p[j];
        const float mm = fmaxf(m, q.x);
        s = (m == -INFINITY ? 0.f : s * expf(m - mm)) + (q.x == -INFINITY ? 0.f : q.y * expf(q.x - mm));
        m = mm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
        const float mm = fmaxf(m, m2);
        s = (m == -INFINITY ? 0.f : s * expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mm));
        m = mm;
    }
    if (lane == 0) {
        const float L = m + logf(s);
        lse[r] = L;
        lrow[r] = L - zt[r];
    }
}

// one block: loss_out[0] += scale * sum_r x[r]; fixed tree order
__global__ void ordered_sum_kernel(const float* __restrict__ x, float* __restrict__ loss_out, float scale,
                                   int rows) {
    __shared__ float red[32];
    float s = 0.f;
    for (int r = threadIdx.x; r < rows; r += blockDim.x) s += x[r];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        v = warp_sum(v);
        if (threadIdx.x == 0) loss_out[0] += v * scale;
    }
}

int ce_combine(const float* part, int ngrp, const float* zt, float* lse, float* lrow, float* loss_out,
               float scale, int rows, cudaStream_t st) {
    if (rows <= 0) return 0;
    ce_combine_kernel<<<(rows + 7) / 8, 256, 0, st>>>(reinterpret_cast<const float2*>(part), ngrp, zt, lse,
                                                       lrow, rows);
    int n = 1;
    if (loss_out) {
        ordered_sum_kernel<<<1, 1024, 0, st>>>(lrow, loss_out, scale, rows);
        ++n;
    }
    note_launches(n);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int ce_fwd(const float* logits, const int* tgt, float* lse, float* loss_out, float scale, int rows,
           int V, cudaStream_t st) {
    if (rows <= 0) return 0;
    if (V % 4 == 0) {
        ce_lse1_kernel<<<rows, 512, 0, st>>>(logits, lse, V);
        ce_loss_kernel<<<1, 1024, 0, st>>>(logits, tgt, lse, loss_out, scale, rows, V);
        note_launches(2);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
    ce_lse_kernel<<<rows, 512, 0, st>>>(logits, lse, V);
    ce_loss_kernel<<<1, 1024, 0, st>>>(logits, tgt, lse, loss_out, scale, rows, V);
    note_launches(2);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <typename T>
__global__ void ce_bwd_kernel(const float* __restrict__ logits, const int* __restrict__ tgt,
                              const float* __restrict__ lse, T* __restrict__ d, float scale,
                              int rows, int V) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)rows * V) return;
    const int r = (int)(i / V), c = (int)(i % V);
    float p = expf(logits[i] - lse[r]);
    if (c == tgt[r]) p -= 1.0f;
    d[i] = from_f<T>(p * scale);
}

int ce_bwd(int dtype, const float* logits, const int* tgt, const float* lse, void* dlogits,
           float scale, int rows, int V, cudaStream_t st) {
    if (rows <= 0) return 0;
    const long n = (long)rows * V;
    if (dtype == DT_BF16 && V % 4 == 0) {
        ce_bwd4_kernel<<<(int)((n / 4 + 255) / 256), 256, 0, st>>>(logits, tgt, lse, (bf16*)dlogits,
                                                                   scale, rows, V);
        note_launches(1);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
    const int blocks = (int)((n + 255) / 256);
    if (dtype == DT_BF16)
        ce_bwd_kernel<bf16><<<blocks, 256, 0, st>>>(logits, tgt, lse, (bf16*)dlogits, scale, rows, V);
    else
        ce_bwd_kernel<float><<<blocks, 256, 0, st>>>(logits, tgt, lse, (float*)dlogits, scale, rows, V);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ============================================================== AdamW
// The arithmetic below is written with explicit round-to-nearest intrinsics
// (no FMA contraction) so that adamw_host (compiled with -ffp-contract=off)
// produces bit-identical results (T-Offload on/off bit-exactness).
template <typename T>
__global__ void adamw_kernel(float* __restrict__ master, float* __restrict__ m,
                             float* __restrict__ v, float* __restrict__ grad, T* __restrict__ w,
                             long n, int decay, AdamHyper hp, const AdamHyper* __restrict__ hp_dev) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (hp_dev) hp = *hp_dev;
    AdamOut o = adam_elem(master[i], m[i], v[i], grad[i], decay, hp);
    master[i] = o.w;
    m[i] = o.m;
    v[i] = o.v;
    grad[i] = 0.f;
    if (w) w[i] = from_f<T>(o.w);
}

// Four consecutive parameters per thread with 16-byte loads / stores (the
// fp32 states are ~29 of the 30 bytes per parameter; scalar loads left the
// kernel at ~0.79 of the HBM peak). Same adam_elem arithmetic per element.
template <typename T>
__global__ void adamw4_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                              float* __restrict__ grad, T* __restrict__ w, long n, int decay, AdamHyper hp,
                              const AdamHyper* __restrict__ hp_dev) {
    const long i = ((long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= n) return;
    if (hp_dev) hp = *hp_dev;
    if (i + 4 <= n) {
        const float4 w4 = *reinterpret_cast<const float4*>(master + i);
        const float4 m4 = *reinterpret_cast<const float4*>(m + i);
        const float4 v4 = *reinterpret_cast<const float4*>(v + i);
        const float4 g4 = *reinterpret_cast<const float4*>(grad + i);
        const AdamOut a = adam_elem(w4.x, m4.x, v4.x, g4.x, decay, hp);
        const AdamOut b = adam_elem(w4.y, m4.y, v4.y, g4.y, decay, hp);
        const AdamOut c = adam_elem(w4.z, m4.z, v4.z, g4.z, decay, hp);
        const AdamOut d = adam_elem(w4.w, m4.w, v4.w, g4.w, decay, hp);
        *reinterpret_cast<float4*>(master + i) = make_float4(a.w, b.w, c.w, d.w);
        *reinterpret_cast<float4*>(m + i) = make_float4(a.m, b.m, c.m, d.m);
        *reinterpret_cast<float4*>(v + i) = make_float4(a.v, b.v, c.v, d.v);
        *reinterpret_cast<float4*>(grad + i) = make_float4(0.f, 0.f, 0.f, 0.f);
        if (w) {
            w[i] = from_f<T>(a.w);
            w[i + 1] = from_f<T>(b.w);
            w[i + 2] = from_f<T>(c.w);
            w[i + 3] = from_f<T>(d.w);
        }
        return;
    }
    for (long j = i; j < n; ++j) {   // ragged tail (< 4 elements)
        const AdamOut o = adam_elem(master[j], m[j], v[j], grad[j], decay, hp);
        master[j] = o.w;
        m[j] = o.m;
        v[j] = o.v;
        grad[j] = 0.f;
        if (w) w[j] = from_f<T>(o.w);
    }
}

int adamw(int dtype, float* master, float* m, float* v, float* grad, void* w, long n, int decay,
          const AdamHyper& hp, cudaStream_t st, const AdamHyper* hp_dev) {
    if (n <= 0) return 0;
    if (((reinterpret_cast<uintptr_t>(master) | reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v) |
          reinterpret_cast<uintptr_t>(grad)) & 15) == 0) {
        const int blocks4 = (int)((n + 1023) / 1024);
        if (dtype == DT_BF16)
            adamw4_kernel<bf16><<<blocks4, 256, 0, st>>>(master, m, v, grad, (bf16*)w, n, decay, hp, hp_dev);
        else
            adamw4_kernel<float><<<blocks4, 256, 0, st>>>(master, m, v, grad, (float*)(w == master ? nullptr : w),
                                                         n, decay, hp, hp_dev);
        note_launches(1);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
    const int blocks = (int)((n + 255) / 256);
    if (dtype == DT_BF16)
        adamw_kernel<bf16><<<blocks, 256, 0, st>>>(master, m, v, grad, (bf16*)w, n, decay, hp, hp_dev);
    else  // fp32: the weight IS the master
        adamw_kernel<float><<<blocks, 256, 0, st>>>(master, m, v, grad,
                                                    (float*)(w == master ? nullptr : w), n, decay, hp, hp_dev);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ZeRO-1 step (R31): one thread per parameter of this replica's shard; the
// reduction over replicas is in replica order, so every run and every
// replica sees the same bits.
template <typename T>
__global__ void dp_adamw_kernel(const DpPtrs p, int dp, float* __restrict__ master, float* __restrict__ m,
                                float* __restrict__ v, long lo, long n, int decay, AdamHyper hp) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long gi = lo + i;
    float g = 0.f;
    for (int j = 0; j < dp; ++j) g = f_add(g, p.grad[j][gi]);
    for (int j = 0; j < dp; ++j) p.grad[j][gi] = 0.f;
    AdamOut o = adam_elem(master[i], m[i], v[i], g, decay, hp);
    master[i] = o.w;
    m[i] = o.m;
    v[i] = o.v;
    const T wv = from_f<T>(o.w);
    for (int j = 0; j < dp; ++j) reinterpret_cast<T*>(p.w[j])[gi] = wv;
}

int dp_adamw(int dtype, const DpPtrs& p, int dp, float* master, float* m, float* v, long lo, long n,
             int decay, const AdamHyper& hp, cudaStream_t st) {
    if (n <= 0) return 0;
    if (dp < 1 || dp > 64) return -4;
    const int blocks = (int)((n + 255) / 256);
    if (dtype == DT_BF16)
        dp_adamw_kernel<bf16><<<blocks, 256, 0, st>>>(p, dp, master, m, v, lo, n, decay, hp);
    else
        dp_adamw_kernel<float><<<blocks, 256, 0, st>>>(p, dp, master, m, v, lo, n, decay, hp);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ============================================================== misc
int fill_zero(void* p, size_t bytes, cudaStream_t st) {
    return cudaMemsetAsync(p, 0, bytes, st) == cudaSuccess ? 0 : -3;
}

template <typename T>
__global__ void cast_kernel(const float* __restrict__ s, T* __restrict__ d, long n) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = from_f<T>(s[i]);
}

int cast_f32_to(int dtype, const float* src, void* dst, long n, cudaStream_t st) {
    if (n <= 0) return 0;
    const int blocks = (int)((n + 255) / 256);
    if (dtype == DT_BF16)
        cast_kernel<bf16><<<blocks, 256, 0, st>>>(src, (bf16*)dst, n);
    else
        cast_kernel<float><<<blocks, 256, 0, st>>>(src, (float*)dst, n);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace tpipe
