// LayerNorm forward / recompute / backward (DESIGN.md §2 N-1:
// eps 1e-5, biased variance) and deterministic column reductions.
//
// HBM-bound. bf16 rows with h % 256 == 0 take the wide path (a group of h/8
// threads per row, several row groups per CTA, next row prefetched); others a
// warp per row. dgamma/dbeta and bias gradients use fixed row-block partials
// (16 rows on the wide path, 64 otherwise) followed by a fixed-order
// reduction, so results are bit-reproducible (no float atomics).
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

// ---------------------------------------------------------------- wide-row path
// bf16, h % 256 == 0, h <= 4096: one thread per 16-byte vector of a row
// (tpr = h/8 threads form a "row group"; a CTA holds G row groups working on
// different rows at once, each prefetching its next row), reductions in a
// fixed order (deterministic). Partial-block layout: RB rows per CTA.
constexpr int RB = 16;        // rows per CTA in the backward / column-sum kernels
constexpr int FWD_RPC = 8;    // rows per CTA in the forward kernel
constexpr int WIDE_THREADS = 512;

// Sum of (a, b) over the tpr threads of row group `grp` (named barrier 1+grp).
// In-warp butterfly, then the per-warp values in warp order: same order for
// every call, so results are reproducible.
__device__ __forceinline__ void group_sum2(float& a, float& b, float (*red)[2], int grp, int tpr) {
    const int w = (threadIdx.x % tpr) >> 5, nw = tpr >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    named_bar_sync(1 + grp, tpr);          // previous readers of red[] are done
    if ((threadIdx.x & 31) == 0) {
        red[w][0] = a;
        red[w][1] = b;
    }
    named_bar_sync(1 + grp, tpr);
    a = 0.f;
    b = 0.f;
    for (int i = 0; i < nw; ++i) {
        a += red[i][0];
        b += red[i][1];
    }
}

__device__ __forceinline__ void ld8(const bf16* p, uint4& u) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ void unpack8(const uint4& u, float (&o)[8]) {
    const bf16* hp = reinterpret_cast<const bf16*>(&u);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = __bfloat162float(hp[j]);
}

// y = LN(x): FWD_RPC rows per CTA, row group grp takes rows r0+grp, r0+grp+G, ...
__global__ void __launch_bounds__(WIDE_THREADS)
ln_fwd_wide_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gamma,
                   const bf16* __restrict__ beta, bf16* __restrict__ y, float* __restrict__ mean,
                   float* __restrict__ rstd, int rows, int h, int apply_only) {
    __shared__ float red[4][32][2];
    const int tpr = h >> 3, G = blockDim.x / tpr, grp = threadIdx.x / tpr;
    const int c = (threadIdx.x % tpr) * 8;
    const int r0 = blockIdx.x * FWD_RPC, r1 = min(rows, r0 + FWD_RPC);
    float g[8], b[8];
    Vec<bf16>::load(gamma + c, g);
    Vec<bf16>::load(beta + c, b);
    int r = r0 + grp;
    uint4 cur = make_uint4(0, 0, 0, 0);
    if (r < r1) ld8(x + (long)r * h + c, cur);
    for (; r < r1; r += G) {
        uint4 nxt = make_uint4(0, 0, 0, 0);
        if (r + G < r1) ld8(x + (long)(r + G) * h + c, nxt);
        float v[8], o[8];
        unpack8(cur, v);
        float mu, rs;
        if (!apply_only) {
            float s = 0.f, dummy = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) s += v[j];
            group_sum2(s, dummy, red[grp], grp, tpr);
            mu = s / (float)h;
            float q = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float d = v[j] - mu;
                q += d * d;
            }
            group_sum2(q, dummy, red[grp], grp, tpr);
            rs = 1.0f / sqrtf(q / (float)h + LN_EPS);
            if (threadIdx.x % tpr == 0) {
                mean[r] = mu;
                rstd[r] = rs;
            }
        } else {
            mu = mean[r];
            rs = rstd[r];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = ln_y(v[j], mu, rs, g[j], b[j]);
        Vec<bf16>::store(y + (long)r * h + c, o);
        cur = nxt;
    }
}

// dx = resid + rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat)); per CTA (RB
// rows) partials into ws[k][nblk][h]: k=0 dgamma, k=1 dbeta, k=2 (if
// with_rsum) the column sum of resid — the bias gradient of the linear layer
// whose output gradient resid is, fused here to save one pass over it.
// Row groups combine their partials in group order through shared memory.
__global__ void __launch_bounds__(WIDE_THREADS)
ln_bwd_wide_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                   const bf16* __restrict__ gamma, const float* __restrict__ mean,
                   const float* __restrict__ rstd, const bf16* __restrict__ resid,
                   bf16* __restrict__ dx, float* __restrict__ ws, int rows, int h, int nblk,
                   int with_rsum) {
    __shared__ float red[4][32][2];
    extern __shared__ float buf[];          // [3][h] when G > 1
    const int tpr = h >> 3, G = blockDim.x / tpr, grp = threadIdx.x / tpr;
    const int c = (threadIdx.x % tpr) * 8;
    float g[8], pg[8] = {}, pb[8] = {}, pr[8] = {};
    Vec<bf16>::load(gamma + c, g);
    const int r0 = blockIdx.x * RB, r1 = min(rows, r0 + RB);
    int r = r0 + grp;
    uint4 cd = make_uint4(0, 0, 0, 0), cx = cd, cr = cd;
    if (r < r1) {
        ld8(dy + (long)r * h + c, cd);
        ld8(x + (long)r * h + c, cx);
        if (resid) ld8(resid + (long)r * h + c, cr);
    }
    for (; r < r1; r += G) {
        uint4 nd = make_uint4(0, 0, 0, 0), nx = nd, nr = nd;
        if (r + G < r1) {
            const long o2 = (long)(r + G) * h + c;
            ld8(dy + o2, nd);
            ld8(x + o2, nx);
            if (resid) ld8(resid + o2, nr);
        }
        float d[8], v[8], rr[8];
        unpack8(cd, d);
        unpack8(cx, v);
        unpack8(cr, rr);
        const float mu = mean[r], rs = rstd[r];
        float xh[8], dxh[8], s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            xh[j] = (v[j] - mu) * rs;
            dxh[j] = d[j] * g[j];
            s1 += dxh[j];
            s2 += dxh[j] * xh[j];
            pg[j] += d[j] * xh[j];
            pb[j] += d[j];
            pr[j] += rr[j];
        }
        group_sum2(s1, s2, red[grp], grp, tpr);
        const float c1 = s1 / (float)h, c2 = s2 / (float)h;
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (dxh[j] - c1 - xh[j] * c2) + (resid ? rr[j] : 0.f);
        Vec<bf16>::store(dx + (long)r * h + c, o);
        cd = nd;
        cx = nx;
        cr = nr;
    }
    // combine row groups in fixed order: p_0 + (p_1 + (... + p_{G-1}))
    for (int k = G - 1; k >= 1; --k) {
        if (grp == k) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const bool first = (k == G - 1);
                buf[c + j] = first ? pg[j] : pg[j] + buf[c + j];
                buf[h + c + j] = first ? pb[j] : pb[j] + buf[h + c + j];
                buf[2 * h + c + j] = first ? pr[j] : pr[j] + buf[2 * h + c + j];
            }
        }
        __syncthreads();
    }
    if (grp != 0) return;
    if (G > 1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            pg[j] += buf[c + j];
            pb[j] += buf[h + c + j];
            pr[j] += buf[2 * h + c + j];
        }
    }
    float* wg = ws + (long)blockIdx.x * h + c;
    float* wb = ws + (long)(nblk + blockIdx.x) * h + c;
    *reinterpret_cast<float4*>(wg) = make_float4(pg[0], pg[1], pg[2], pg[3]);
    *reinterpret_cast<float4*>(wg + 4) = make_float4(pg[4], pg[5], pg[6], pg[7]);
    *reinterpret_cast<float4*>(wb) = make_float4(pb[0], pb[1], pb[2], pb[3]);
    *reinterpret_cast<float4*>(wb + 4) = make_float4(pb[4], pb[5], pb[6], pb[7]);
    if (with_rsum) {
        float* wr = ws + (long)(2 * nblk + blockIdx.x) * h + c;
        *reinterpret_cast<float4*>(wr) = make_float4(pr[0], pr[1], pr[2], pr[3]);
        *reinterpret_cast<float4*>(wr + 4) = make_float4(pr[4], pr[5], pr[6], pr[7]);
    }
}

// per-CTA (RB rows) column partial sums of X[rows, n] into ws[nblk][n]; a CTA
// covers 2048 columns of its row block, all RB row loads issued up front.
constexpr int CS_COLS = 2048;
__global__ void __launch_bounds__(256)
colsum_wide_kernel(const bf16* __restrict__ X, float* __restrict__ ws, int rows, int n) {
    const int c = blockIdx.x * CS_COLS + threadIdx.x * 8;
    if (c >= n) return;
    const int r0 = blockIdx.y * RB, r1 = min(rows, r0 + RB);
    float p[8] = {};
    if (r1 - r0 == RB) {
        uint4 u[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) ld8(X + (long)(r0 + i) * n + c, u[i]);
#pragma unroll
        for (int i = 0; i < RB; ++i) {
            float v[8];
            unpack8(u[i], v);
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] += v[j];
        }
    } else {
        for (int r = r0; r < r1; ++r) {
            float v[8];
            Vec<bf16>::load(X + (long)r * n + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] += v[j];
        }
    }
    float* w = ws + (long)blockIdx.y * n + c;
    *reinterpret_cast<float4*>(w) = make_float4(p[0], p[1], p[2], p[3]);
    *reinterpret_cast<float4*>(w + 4) = make_float4(p[4], p[5], p[6], p[7]);
}

// out_t[col] += sum_{b < nblk} ws[t][b][col], t = blockIdx.y (up to 3 vectors per
// launch). n % 4 == 0. A CTA covers 32 columns: 8 float4 lanes x 32 row
// groups; row group g sums blocks g, g+32, ...; the 32 group sums are then
// added in a fixed binary tree (deterministic).
__global__ void __launch_bounds__(256)
reduce_parts_kernel(const float* __restrict__ ws, float* __restrict__ out0, float* __restrict__ out1,
                    float* __restrict__ out2, int n, int nblk) {
    __shared__ float4 red[32][8];
    const int t = blockIdx.y;
    float* out = t == 0 ? out0 : (t == 1 ? out1 : out2);
    const float* src = ws + (long)t * nblk * n;
    const int cg = threadIdx.x & 7, g = threadIdx.x >> 3;
    const int col = blockIdx.x * 32 + cg * 4;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col < n) {
#pragma unroll 4
        for (int b = g; b < nblk; b += 32) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(src + (long)b * n + col));
            s.x += v.x;
            s.y += v.y;
            s.z += v.z;
            s.w += v.w;
        }
    }
    red[g][cg] = s;
    __syncthreads();
    for (int stride = 16; stride > 0; stride >>= 1) {
        if (g < stride) {
            const float4 o = red[g + stride][cg];
            red[g][cg].x += o.x;
            red[g][cg].y += o.y;
            red[g][cg].z += o.z;
            red[g][cg].w += o.w;
        }
        __syncthreads();
    }
    if (g == 0 && col < n) {
        float4* po = reinterpret_cast<float4*>(out + col);
        float4 a = *po;
        const float4 r = red[0][cg];
        a.x += r.x;
        a.y += r.y;
        a.z += r.z;
        a.w += r.w;
        *po = a;
    }
}

static int wide_groups(int h) {
    const int tpr = h / 8;
    int G = WIDE_THREADS / tpr;
    return G < 1 ? 1 : (G > 4 ? 4 : G);
}

static bool wide_ok(int dtype, int h) { return dtype == DT_BF16 && h % 256 == 0 && h <= 8 * WIDE_THREADS; }

int ln_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y, float* mean,
           float* rstd, int rows, int h, cudaStream_t st) {
    if (rows <= 0) return 0;
    if (h % 8) return -1;
    if (wide_ok(dtype, h)) {
        const int G = wide_groups(h);
        ln_fwd_wide_kernel<<<(rows + FWD_RPC - 1) / FWD_RPC, G * (h / 8), 0, st>>>(
            (const bf16*)x, (const bf16*)gamma, (const bf16*)beta, (bf16*)y, mean, rstd, rows, h, 0);
        note_launches(1);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
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
    if (wide_ok(dtype, h)) {
        const int G = wide_groups(h);
        ln_fwd_wide_kernel<<<(rows + FWD_RPC - 1) / FWD_RPC, G * (h / 8), 0, st>>>(
            (const bf16*)x, (const bf16*)gamma, (const bf16*)beta, (bf16*)y, const_cast<float*>(mean),
            const_cast<float*>(rstd), rows, h, 1);
        note_launches(1);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
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
           int rows, int h, cudaStream_t st, float* dresid_sum) {
    if (rows <= 0) return 0;
    if (h % 8) return -1;
    if (dresid_sum && !resid) return -1;
    if (wide_ok(dtype, h)) {
        const int nb = (rows + RB - 1) / RB;
        const int G = wide_groups(h);
        const int rs = dresid_sum ? 1 : 0;
        ln_bwd_wide_kernel<<<nb, G * (h / 8), G > 1 ? 3 * h * sizeof(float) : 0, st>>>(
            (const bf16*)dy, (const bf16*)x, (const bf16*)gamma, mean, rstd, (const bf16*)resid,
            (bf16*)dx, ws, rows, h, nb, rs);
        reduce_parts_kernel<<<dim3((h + 31) / 32, 2 + rs), 256, 0, st>>>(ws, dgamma, dbeta, dresid_sum,
                                                                         h, nb);
        note_launches(2);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
    if (dresid_sum) {
        const int rc = colsum_acc(dtype, resid, dresid_sum, ws, rows, h, st);
        if (rc) return rc;
    }
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
    if (dtype == DT_BF16 && n % 8 == 0) {   // any width: CTAs tile 2048 columns
        const int nb = (rows + RB - 1) / RB;
        colsum_wide_kernel<<<dim3((n + CS_COLS - 1) / CS_COLS, nb), 256, 0, st>>>((const bf16*)X, ws,
                                                                                 rows, n);
        reduce_parts_kernel<<<dim3((n + 31) / 32, 1), 256, 0, st>>>(ws, out, nullptr, nullptr, n, nb);
        note_launches(2);
        return cudaGetLastError() == cudaSuccess ? 0 : -3;
    }
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
