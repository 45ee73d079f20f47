// LayerNorm forward / recompute / backward (DESIGN.md §2 N-1:
// eps 1e-5, biased variance) and deterministic column reductions.
//
// HBM-bound: one warp per row, 16-byte vector loads, warp-shuffle reductions.
// dgamma/dbeta and bias gradients use fixed 64-row block partials followed by
// an in-order reduction, so results are bit-reproducible (no float atomics).
#include "common.cuh"
#include "kernels.h"

namespace tpipe {

constexpr float LN_EPS = 1e-5f;
constexpr int ROWBLK = 64;

template <typename T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<bf16> {
    static constexpr int N = 8;
    __device__ static void load(const bf16* p, float (&o)[8]) {
        uint4 u = *reinterpret_cast<const uint4*>(p);
        const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = __bfloat162float(h[j]);
    }
    __device__ static void store(bf16* p, const float (&v)[8]) {
        uint4 u;
        bf16* h = reinterpret_cast<bf16*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = __float2bfloat16_rn(v[j]);
        *reinterpret_cast<uint4*>(p) = u;
    }
};
template <>
struct Vec<float> {
    static constexpr int N = 4;
    __device__ static void load(const float* p, float (&o)[4]) {
        float4 u = *reinterpret_cast<const float4*>(p);
        o[0] = u.x; o[1] = u.y; o[2] = u.z; o[3] = u.w;
    }
    __device__ static void store(float* p, const float (&v)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};

// y element from saved statistics: shared by ln_fwd and ln_apply so the
// operator-level recompute is bit-identical to the forward.
__device__ __forceinline__ float ln_y(float x, float mean, float rstd, float g, float b) {
    return __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(x, mean), rstd), g), b);
}

template <typename T>
__global__ void ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ gamma,
                              const T* __restrict__ beta, T* __restrict__ y, float* __restrict__ mean,
                              float* __restrict__ rstd, int rows, int h, int apply_only) {
    constexpr int V = Vec<T>::N;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const T* xr = x + (long)warp * h;
    float mu, rs;
    if (!apply_only) {
        float s = 0.f;
        for (int c = lane * V; c < h; c += 32 * V) {
            float v[V];
            Vec<T>::load(xr + c, v);
#pragma unroll
            for (int j = 0; j < V; ++j) s += v[j];
        }
        mu = warp_sum(s) / (float)h;
        float q = 0.f;
        for (int c = lane * V; c < h; c += 32 * V) {
            float v[V];
            Vec<T>::load(xr + c, v);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                float dlt = v[j] - mu;
                q += dlt * dlt;
            }
        }
        float var = warp_sum(q) / (float)h;
        rs = 1.0f / sqrtf(var + LN_EPS);
        if (lane == 0) {
            mean[warp] = mu;
            rstd[warp] = rs;
        }
    } else {
        mu = mean[warp];
        rs = rstd[warp];
    }
    T* yr = y + (long)warp * h;
    for (int c = lane * V; c < h; c += 32 * V) {
        float v[V], g[V], b[V], o[V];
        Vec<T>::load(xr + c, v);
        Vec<T>::load(gamma + c, g);
        Vec<T>::load(beta + c, b);
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = ln_y(v[j], mu, rs, g[j], b[j]);
        Vec<T>::store(yr + c, o);
    }
}

int ln_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y, float* mean,
           float* rstd, int rows, int h, cudaStream_t st) {
    if (rows <= 0) return 0;
    if (h % 8) return -1;
    const int threads = 256, blocks = (rows * 32 + threads - 1) / threads;
    if (dtype == DT_BF16)
        ln_fwd_kernel<bf16><<<blocks, threads, 0, st>>>((const bf16*)x, (const bf16*)gamma,
                                                        (const bf16*)beta, (bf16*)y, mean, rstd, rows, h, 0);
    else
        ln_fwd_kernel<float><<<blocks, threads, 0, st>>>((const float*)x, (const float*)gamma,
                                                         (const float*)beta, (float*)y, mean, rstd, rows, h, 0);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int ln_apply(int dtype, const void* x, const void* gamma, const void* beta, const float* mean,
             const float* rstd, void* y, int rows, int h, cudaStream_t st) {
    if (rows <= 0) return 0;
    const int threads = 256, blocks = (rows * 32 + threads - 1) / threads;
    if (dtype == DT_BF16)
        ln_fwd_kernel<bf16><<<blocks, threads, 0, st>>>((const bf16*)x, (const bf16*)gamma,
                                                        (const bf16*)beta, (bf16*)y,
                                                        const_cast<float*>(mean),
                                                        const_cast<float*>(rstd), rows, h, 1);
    else
        ln_fwd_kernel<float><<<blocks, threads, 0, st>>>((const float*)x, (const float*)gamma,
                                                         (const float*)beta, (float*)y,
                                                         const_cast<float*>(mean),
                                                         const_cast<float*>(rstd), rows, h, 1);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// dx = resid + rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)), dxhat = dy * gamma
template <typename T>
__global__ void ln_bwd_dx_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                 const T* __restrict__ gamma, const float* __restrict__ mean,
                                 const float* __restrict__ rstd, const T* __restrict__ resid,
                                 T* __restrict__ dx, int rows, int h) {
    constexpr int V = Vec<T>::N;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rows) return;
    const long off = (long)warp * h;
    const float mu = mean[warp], rs = rstd[warp];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane * V; c < h; c += 32 * V) {
        float d[V], v[V], g[V];
        Vec<T>::load(dy + off + c, d);
        Vec<T>::load(x + off + c, v);
        Vec<T>::load(gamma + c, g);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            float xh = (v[j] - mu) * rs;
            float dxh = d[j] * g[j];
            s1 += dxh;
            s2 += dxh * xh;
        }
    }
    const float c1 = warp_sum(s1) / (float)h, c2 = warp_sum(s2) / (float)h;
    for (int c = lane * V; c < h; c += 32 * V) {
        float d[V], v[V], g[V], r[V], o[V];
        Vec<T>::load(dy + off + c, d);
        Vec<T>::load(x + off + c, v);
        Vec<T>::load(gamma + c, g);
        if (resid) Vec<T>::load(resid + off + c, r);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            float xh = (v[j] - mu) * rs;
            float dxh = d[j] * g[j];
            o[j] = rs * (dxh - c1 - xh * c2) + (resid ? r[j] : 0.f);
        }
        Vec<T>::store(dx + off + c, o);
    }
}

// partial[blk][col] for dgamma (sum dy*xhat) and dbeta (sum dy) over a 64-row block
template <typename T>
__global__ void ln_bwd_partial_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                      const float* __restrict__ mean, const float* __restrict__ rstd,
                                      float* __restrict__ ws, int rows, int h, int nblk) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    const int blk = blockIdx.y;
    if (col >= h) return;
    const int r0 = blk * ROWBLK, r1 = min(rows, r0 + ROWBLK);
    float sg = 0.f, sb = 0.f;
    for (int r = r0; r < r1; ++r) {
        float d = to_f<T>(dy[(long)r * h + col]);
        float xh = (to_f<T>(x[(long)r * h + col]) - mean[r]) * rstd[r];
        sg += d * xh;
        sb += d;
    }
    ws[(long)blk * h + col] = sg;
    ws[(long)(nblk + blk) * h + col] = sb;
}

// out[col] += sum over blocks in order
__global__ void reduce_blocks_kernel(const float* __restrict__ ws, float* __restrict__ out, int n,
                                     int nblk) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= n) return;
    float s = 0.f;
    for (int b = 0; b < nblk; ++b) s += ws[(long)b * n + col];
    out[col] += s;
}

int ln_bwd(int dtype, const void* dy, const void* x, const void* gamma, const float* mean,
           const float* rstd, const void* resid, void* dx, float* dgamma, float* dbeta, float* ws,
           int rows, int h, cudaStream_t st) {
    if (rows <= 0) return 0;
    if (h % 8) return -1;
    const int threads = 256, blocks = (rows * 32 + threads - 1) / threads;
    const int nblk = (rows + ROWBLK - 1) / ROWBLK;
    dim3 pg((h + 255) / 256, nblk);
    if (dtype == DT_BF16) {
        ln_bwd_dx_kernel<bf16><<<blocks, threads, 0, st>>>((const bf16*)dy, (const bf16*)x,
                                                           (const bf16*)gamma, mean, rstd,
                                                           (const bf16*)resid, (bf16*)dx, rows, h);
        ln_bwd_partial_kernel<bf16><<<pg, 256, 0, st>>>((const bf16*)dy, (const bf16*)x, mean, rstd,
                                                        ws, rows, h, nblk);
    } else {
        ln_bwd_dx_kernel<float><<<blocks, threads, 0, st>>>((const float*)dy, (const float*)x,
                                                            (const float*)gamma, mean, rstd,
                                                            (const float*)resid, (float*)dx, rows, h);
        ln_bwd_partial_kernel<float><<<pg, 256, 0, st>>>((const float*)dy, (const float*)x, mean,
                                                         rstd, ws, rows, h, nblk);
    }
    reduce_blocks_kernel<<<(h + 255) / 256, 256, 0, st>>>(ws, dgamma, h, nblk);
    reduce_blocks_kernel<<<(h + 255) / 256, 256, 0, st>>>(ws + (long)nblk * h, dbeta, h, nblk);
    note_launches(4);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <typename T>
__global__ void colsum_partial_kernel(const T* __restrict__ X, float* __restrict__ ws, int rows,
                                      int n) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    const int blk = blockIdx.y;
    if (col >= n) return;
    const int r0 = blk * ROWBLK, r1 = min(rows, r0 + ROWBLK);
    float s = 0.f;
    for (int r = r0; r < r1; ++r) s += to_f<T>(X[(long)r * n + col]);
    ws[(long)blk * n + col] = s;
}

int colsum_acc(int dtype, const void* X, float* out, float* ws, int rows, int n, cudaStream_t st) {
    if (rows <= 0 || n <= 0) return 0;
    const int nblk = (rows + ROWBLK - 1) / ROWBLK;
    dim3 pg((n + 255) / 256, nblk);
    if (dtype == DT_BF16)
        colsum_partial_kernel<bf16><<<pg, 256, 0, st>>>((const bf16*)X, ws, rows, n);
    else
        colsum_partial_kernel<float><<<pg, 256, 0, st>>>((const float*)X, ws, rows, n);
    reduce_blocks_kernel<<<(n + 255) / 256, 256, 0, st>>>(ws, out, n, nblk);
    note_launches(2);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace tpipe
