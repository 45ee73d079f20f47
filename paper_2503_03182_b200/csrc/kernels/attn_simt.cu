// Causal attention, exact-fp32 SIMT path.
//
// Used for fp32 mode (parity at 1e-4) and as the reference-structure path for
// bf16 until the tensor-core kernel takes over for head_dim 64/128. One warp
// per query (forward, dQ) or key (dK, dV) row, online softmax (FlashAttention
// recurrence), P recomputed from the saved LSE in the backward (operator-level
// recompute). Deterministic: fixed loop order, no atomics.
#include "common.cuh"
#include "kernels.h"

namespace tpipe {

constexpr int MAXE = 4;  // head_dim <= 128

template <typename T>
__device__ __forceinline__ void load_row(const T* p, int d, int lane, float (&r)[MAXE]) {
#pragma unroll
    for (int i = 0; i < MAXE; ++i) {
        int e = lane + 32 * i;
        r[i] = e < d ? to_f<T>(p[e]) : 0.f;
    }
}

template <typename T>
__global__ void attn_fwd_simt_kernel(const T* __restrict__ qkv, T* __restrict__ o,
                                     float* __restrict__ lse, int s, int a, int d) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int head = blockIdx.y, b = blockIdx.z;
    if (i >= s) return;
    const int h = a * d;
    const long ld = 3L * h;
    const T* base = qkv + (long)b * s * ld;
    const float scale = rsqrtf((float)d);
    float q[MAXE], acc[MAXE] = {};
    load_row(base + (long)i * ld + head * d, d, lane, q);
    float mx = -INFINITY, l = 0.f;
    for (int j = 0; j <= i; ++j) {
        float kv[MAXE];
        load_row(base + (long)j * ld + h + head * d, d, lane, kv);
        float part = 0.f;
#pragma unroll
        for (int e = 0; e < MAXE; ++e) part += q[e] * kv[e];
        const float sc = warp_sum(part) * scale;
        const float mn = fmaxf(mx, sc);
        const float corr = expf(mx - mn);
        const float p = expf(sc - mn);
        l = l * corr + p;
        load_row(base + (long)j * ld + 2 * h + head * d, d, lane, kv);
#pragma unroll
        for (int e = 0; e < MAXE; ++e) acc[e] = acc[e] * corr + p * kv[e];
        mx = mn;
    }
    T* orow = o + ((long)b * s + i) * h + head * d;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
        int c = lane + 32 * e;
        if (c < d) orow[c] = from_f<T>(acc[e] / l);
    }
    if (lane == 0) lse[((long)b * a + head) * s + i] = mx + logf(l);
}

// D[b,head,i] = sum_e dO[i,e] * O[i,e]
template <typename T>
__global__ void attn_bwd_d_kernel(const T* __restrict__ o, const T* __restrict__ dout,
                                  float* __restrict__ D, int s, int a, int d) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int head = blockIdx.y, b = blockIdx.z;
    if (i >= s) return;
    const int h = a * d;
    float x[MAXE], y[MAXE];
    load_row(o + ((long)b * s + i) * h + head * d, d, lane, x);
    load_row(dout + ((long)b * s + i) * h + head * d, d, lane, y);
    float part = 0.f;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) part += x[e] * y[e];
    part = warp_sum(part);
    if (lane == 0) D[((long)b * a + head) * s + i] = part;
}

// dQ_i = scale * sum_{j<=i} P_ij (dP_ij - D_i) K_j
template <typename T>
__global__ void attn_bwd_dq_kernel(const T* __restrict__ qkv, const T* __restrict__ dout,
                                   const float* __restrict__ lse, const float* __restrict__ D,
                                   T* __restrict__ dqkv, int s, int a, int d) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int head = blockIdx.y, b = blockIdx.z;
    if (i >= s) return;
    const int h = a * d;
    const long ld = 3L * h;
    const T* base = qkv + (long)b * s * ld;
    const float scale = rsqrtf((float)d);
    const long ri = ((long)b * a + head) * s + i;
    const float L = lse[ri], Di = D[ri];
    float q[MAXE], g[MAXE], acc[MAXE] = {};
    load_row(base + (long)i * ld + head * d, d, lane, q);
    load_row(dout + ((long)b * s + i) * h + head * d, d, lane, g);
    for (int j = 0; j <= i; ++j) {
        float k[MAXE], v[MAXE];
        load_row(base + (long)j * ld + h + head * d, d, lane, k);
        load_row(base + (long)j * ld + 2 * h + head * d, d, lane, v);
        float ps = 0.f, pd = 0.f;
#pragma unroll
        for (int e = 0; e < MAXE; ++e) {
            ps += q[e] * k[e];
            pd += g[e] * v[e];
        }
        const float p = expf(warp_sum(ps) * scale - L);
        const float ds = p * (warp_sum(pd) - Di);
#pragma unroll
        for (int e = 0; e < MAXE; ++e) acc[e] += ds * k[e];
    }
    T* dq = dqkv + ((long)b * s + i) * ld + head * d;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
        int c = lane + 32 * e;
        if (c < d) dq[c] = from_f<T>(acc[e] * scale);
    }
}

// dK_j = scale * sum_{i>=j} dS_ij Q_i ; dV_j = sum_{i>=j} P_ij dO_i
template <typename T>
__global__ void attn_bwd_dkv_kernel(const T* __restrict__ qkv, const T* __restrict__ dout,
                                    const float* __restrict__ lse, const float* __restrict__ D,
                                    T* __restrict__ dqkv, int s, int a, int d) {
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int head = blockIdx.y, b = blockIdx.z;
    if (j >= s) return;
    const int h = a * d;
    const long ld = 3L * h;
    const T* base = qkv + (long)b * s * ld;
    const float scale = rsqrtf((float)d);
    float k[MAXE], v[MAXE], dk[MAXE] = {}, dv[MAXE] = {};
    load_row(base + (long)j * ld + h + head * d, d, lane, k);
    load_row(base + (long)j * ld + 2 * h + head * d, d, lane, v);
    for (int i = j; i < s; ++i) {
        float q[MAXE], g[MAXE];
        load_row(base + (long)i * ld + head * d, d, lane, q);
        load_row(dout + ((long)b * s + i) * h + head * d, d, lane, g);
        const long ri = ((long)b * a + head) * s + i;
        float ps = 0.f, pd = 0.f;
#pragma unroll
        for (int e = 0; e < MAXE; ++e) {
            ps += q[e] * k[e];
            pd += g[e] * v[e];
        }
        const float p = expf(warp_sum(ps) * scale - lse[ri]);
        const float ds = p * (warp_sum(pd) - D[ri]);
#pragma unroll
        for (int e = 0; e < MAXE; ++e) {
            dv[e] += p * g[e];
            dk[e] += ds * q[e];
        }
    }
    T* dkr = dqkv + ((long)b * s + j) * ld + h + head * d;
    T* dvr = dkr + h;
#pragma unroll
    for (int e = 0; e < MAXE; ++e) {
        int c = lane + 32 * e;
        if (c < d) {
            dkr[c] = from_f<T>(dk[e] * scale);
            dvr[c] = from_f<T>(dv[e]);
        }
    }
}

int attn_fwd_simt(int dtype, const void* qkv, void* o, float* lse, int b, int s, int a, int d,
                  cudaStream_t st) {
    dim3 grid((s + 3) / 4, a, b);
    if (dtype == DT_BF16)
        attn_fwd_simt_kernel<bf16><<<grid, 128, 0, st>>>((const bf16*)qkv, (bf16*)o, lse, s, a, d);
    else
        attn_fwd_simt_kernel<float><<<grid, 128, 0, st>>>((const float*)qkv, (float*)o, lse, s, a, d);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int attn_bwd_simt(int dtype, const void* qkv, const void* o, const void* dout, const float* lse,
                  void* dqkv, float* ws, int b, int s, int a, int d, cudaStream_t st) {
    dim3 grid((s + 3) / 4, a, b);
    if (dtype == DT_BF16) {
        attn_bwd_d_kernel<bf16><<<grid, 128, 0, st>>>((const bf16*)o, (const bf16*)dout, ws, s, a, d);
        attn_bwd_dq_kernel<bf16><<<grid, 128, 0, st>>>((const bf16*)qkv, (const bf16*)dout, lse, ws,
                                                       (bf16*)dqkv, s, a, d);
        attn_bwd_dkv_kernel<bf16><<<grid, 128, 0, st>>>((const bf16*)qkv, (const bf16*)dout, lse, ws,
                                                        (bf16*)dqkv, s, a, d);
    } else {
        attn_bwd_d_kernel<float><<<grid, 128, 0, st>>>((const float*)o, (const float*)dout, ws, s, a, d);
        attn_bwd_dq_kernel<float><<<grid, 128, 0, st>>>((const float*)qkv, (const float*)dout, lse, ws,
                                                        (float*)dqkv, s, a, d);
        attn_bwd_dkv_kernel<float><<<grid, 128, 0, st>>>((const float*)qkv, (const float*)dout, lse,
                                                         ws, (float*)dqkv, s, a, d);
    }
    note_launches(3);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// Dispatch: tcgen05 kernels (attn_tc5.cu) for bf16 with head_dim 64/128,
// SIMT otherwise.
int attn_fwd_tc5(const void* qkv, void* o, float* lse, int b, int s, int a, int d, cudaStream_t st);
int attn_bwd_tc5(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                 float* ws, int b, int s, int a, int d, cudaStream_t st, bool have_d);

// bf16 with head_dim 64/128: tcgen05 kernels (attn_tc5.cu); fp32 (parity
// mode) and other head dims: SIMT.
int attn_fwd(int dtype, const void* qkv, void* o, float* lse, int b, int s, int a, int d,
             cudaStream_t st) {
    if (d > 32 * MAXE) return -1;
    if (dtype == DT_BF16 && (d == 64 || d == 128))
        return attn_fwd_tc5(qkv, o, lse, b, s, a, d, st);
    return attn_fwd_simt(dtype, qkv, o, lse, b, s, a, d, st);
}

int attn_bwd(int dtype, const void* qkv, const void* o, const void* dout, const float* lse,
             void* dqkv, float* ws, int b, int s, int a, int d, cudaStream_t st, bool have_d) {
    if (d > 32 * MAXE) return -1;
    if (dtype == DT_BF16 && (d == 64 || d == 128))
        return attn_bwd_tc5(qkv, o, dout, lse, dqkv, ws, b, s, a, d, st, have_d);
    return attn_bwd_simt(dtype, qkv, o, dout, lse, dqkv, ws, b, s, a, d, st);
}

}  // namespace tpipe
