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
// bf16, h % 256 == 0, h <= 4096. Forward: a warp per register-resident row.
// Backward: a CTA per RB-row block, rows staged in shared memory by bulk
// copies; a "row group" of tpr = h/8 threads (one 16-byte vector each) works
// on one row, G row groups per CTA; reductions in a fixed order
// (deterministic). Partial-block layout: RB rows per CTA.
constexpr int RB = 16;        // rows per CTA in the backward / column-sum kernels
constexpr int WIDE_THREADS = 512;
// row-parallel LN backward (ln_bwd_rows_kernel) for h <= 2048 (on by default;
// off = the staged kernel, for A/B runs)
static bool g_ln_rows = true;
void ln_set_rows_bwd(int on) { g_ln_rows = on != 0; }

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

// per-CTA (RB rows) column partial sums of X[rows, n] into ws[nblk][n]; a CTA
// covers 2048 columns of its row block, all RB row loads issued up front.
constexpr int CS_COLS = 2048;
__global__ void __launch_bounds__(256)
colsum_wide_kernel(const bf16* __restrict__ X, float* __restrict__ ws, int rows, int n) {
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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

// Segmented variant: up to 4 (partials, output, width) segments in one launch
// (blockIdx.y = segment); same per-column order as reduce_parts_kernel. Lets a
// layer backward reduce its bias / LayerNorm-affine partials in 2 launches
// instead of 4.
struct ReduceSegs {
    const float* src[4];
    float* out[4];
    int n[4];
    int cb[5];   // first 32-column block of each segment in the flat grid (cb[nseg] = grid size)
};
__global__ void __launch_bounds__(256) reduce_segs_kernel(const ReduceSegs segs, int nblk) {
    pdl_wait();
    pdl_trigger();
    __shared__ float4 red[32][8];
    // flat grid over every segment's 32-column blocks (no idle CTAs for the
    // narrower segments)
    int t = 0;
#pragma unroll
    for (int i = 1; i < 4; ++i)
        if ((int)blockIdx.x >= segs.cb[i] && segs.cb[i] < segs.cb[4]) t = i;
    const int bx = blockIdx.x - segs.cb[t];
    const int n = segs.n[t];
    const float* src = segs.src[t];
    float* out = segs.out[t];
    const int cg = threadIdx.x & 7, g = threadIdx.x >> 3;
    const int col = bx * 32 + cg * 4;
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    if (col < n) {
#pragma unroll 4
        for (int b = g; b < nblk; b += 32) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(src + (long)b * n + col));
            sum.x += v.x;
            sum.y += v.y;
            sum.z += v.z;
            sum.w += v.w;
        }
    }
    red[g][cg] = sum;
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

// ---------------------------------------------------------------- warp-per-row forward
// bf16, h = 256*NV: one warp per row, the whole row register-resident (NV
// 16-byte vectors per lane, all loads issued before any use), warp-shuffle
// reductions only (no block barriers), so every row of the launch is in
// flight at once. mean first, then the centred second moment from registers.
template <int NV>
__global__ void __launch_bounds__(256)
ln_fwd_warp_kernel(const bf16* __restrict__ x, const bf16* __restrict__ gamma,
                   const bf16* __restrict__ beta, bf16* __restrict__ y, float* __restrict__ mean,
                   float* __restrict__ rstd, int rows, int apply_only) {
    pdl_wait();
    pdl_trigger();
    constexpr int h = NV * 256;
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    // gamma / beta staged once per CTA in shared memory, loaded with the rows
    // (their latency off the tail; no registers held)
    __shared__ __align__(16) bf16 sg[h], sbt[h];
    for (int c = threadIdx.x * 8; c < h; c += 256 * 8) {
        *reinterpret_cast<uint4*>(sg + c) = __ldg(reinterpret_cast<const uint4*>(gamma + c));
        *reinterpret_cast<uint4*>(sbt + c) = __ldg(reinterpret_cast<const uint4*>(beta + c));
    }
    const bf16* xr = x + (long)row * h;
    uint4 u[NV];
    if (row < rows) {
#pragma unroll
        for (int i = 0; i < NV; ++i) ld8(xr + (i * 32 + lane) * 8, u[i]);
    }
    __syncthreads();
    if (row >= rows) return;
    float mu, rs;
    if (!apply_only) {
        // eight independent partial sums per lane (short dependency chains),
        // added in a fixed order
        float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            float v[8];
            unpack8(u[i], v);
#pragma unroll
            for (int j = 0; j < 8; ++j) s8[j] += v[j];
        }
        mu = warp_sum(((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]))) / (float)h;
        float q8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            float v[8];
            unpack8(u[i], v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float d = v[j] - mu;
                q8[j] += d * d;
            }
        }
        const float q = ((q8[0] + q8[1]) + (q8[2] + q8[3])) + ((q8[4] + q8[5]) + (q8[6] + q8[7]));
        rs = 1.0f / sqrtf(warp_sum(q) / (float)h + LN_EPS);
        if (lane == 0) {
            mean[row] = mu;
            rstd[row] = rs;
        }
    } else {
        mu = mean[row];
        rs = rstd[row];
    }
    bf16* yr = y + (long)row * h;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int c = (i * 32 + lane) * 8;
        float v[8], g[8], b[8], o[8];
        unpack8(u[i], v);
        unpack8(*reinterpret_cast<const uint4*>(sg + c), g);
        unpack8(*reinterpret_cast<const uint4*>(sbt + c), b);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = ln_y(v[j], mu, rs, g[j], b[j]);
        Vec<bf16>::store(yr + c, o);
    }
}

template <int NV>
static void launch_ln_fwd_warp(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean, float* rstd,
                               int rows, int apply_only, cudaStream_t st) {
    launch_k(ln_fwd_warp_kernel<NV>, dim3((rows + 7) / 8), dim3(256), 0, st, 1, x, g, b, y, mean, rstd, rows,
             apply_only);
}

static int ln_fwd_warp(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean, float* rstd, int rows,
                       int h, int apply_only, cudaStream_t st) {
    switch (h / 256) {
#define TP_LNW(NV) \
    case NV: launch_ln_fwd_warp<NV>(x, g, b, y, mean, rstd, rows, apply_only, st); return 0;
        TP_LNW(1) TP_LNW(2) TP_LNW(3) TP_LNW(4) TP_LNW(5) TP_LNW(6) TP_LNW(7) TP_LNW(8)
        TP_LNW(9) TP_LNW(10) TP_LNW(11) TP_LNW(12) TP_LNW(13) TP_LNW(14) TP_LNW(15) TP_LNW(16)
#undef TP_LNW
        default: return -1;
    }
}

// ---------------------------------------------------------------- staged backward
// One CTA per RB-row block; the block's dy / x / resid rows are fetched with
// 16-byte cp.async into shared memory in chunks of RC rows, so all of a
// chunk's bytes are in flight at once; the row groups then work from shared
// memory.
constexpr int LNB_SMEM_ROWS_BYTES = 192 * 1024;

// packed fp32x2 helpers (sm_100 FFMA2 / FADD2 / FMUL2)
__device__ __forceinline__ uint64_t fpair(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void funpair(uint64_t r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
// bf16x2 word (lo = element 0) -> (float lo, float hi)
__device__ __forceinline__ uint64_t bfpair(uint32_t w) {
    return fpair(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ uint64_t ffma2x(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2x(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fmul2x(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__global__ void __launch_bounds__(WIDE_THREADS, 1)
ln_bwd_stage_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                    const bf16* __restrict__ gamma, const float* __restrict__ mean,
                    const float* __restrict__ rstd, const bf16* __restrict__ resid,
                    bf16* __restrict__ dx, float* __restrict__ ws, int rows, int h, int nblk,
                    int with_rsum, int RC) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[4][32][2];
    __shared__ float smu[RB], srs[RB];
    extern __shared__ __align__(128) uint8_t smraw[];
    bf16* sdy = reinterpret_cast<bf16*>(smraw);          // [RC][h]
    bf16* sx = sdy + (size_t)RC * h;                     // [RC][h]
    bf16* sr = sx + (size_t)RC * h;                      // [RC][h]
    float* buf = reinterpret_cast<float*>(smraw);        // [3][h] group combine (after the rows)
    const int tpr = h >> 3, G = blockDim.x / tpr, grp = threadIdx.x / tpr;
    const int c = (threadIdx.x % tpr) * 8;
    const int r0 = blockIdx.x * RB, r1 = min(rows, r0 + RB);
    if (threadIdx.x < RB && r0 + threadIdx.x < r1) {   // row statistics off the per-row critical path
        smu[threadIdx.x] = mean[r0 + threadIdx.x];
        srs[threadIdx.x] = rstd[r0 + threadIdx.x];
    }
    __syncthreads();
    // packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2): the kernel is issue-bound
    // (profiles/r1_hbm_kernels_ncu.txt), bf16 pairs unpack with one shift / mask each
    uint64_t g2[4], pg2[4], pb2[4], pr2[4];
    {
        const uint4 gu = *reinterpret_cast<const uint4*>(gamma + c);
        const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            g2[j] = bfpair(gw[j]);
            pg2[j] = pb2[j] = pr2[j] = 0ull;
        }
    }
    for (int q0 = r0; q0 < r1; q0 += RC) {
        const int nr = min(RC, r1 - q0);
        // each thread fetches only the 16-byte slices it will read itself
        // (cp.async, no registers held), so no CTA barrier is needed before use;
        // two commit groups (rows [0, half), [half, nr)): the first half's rows
        // are processed and stored while the second half is still landing
        const int half = (nr + 1) / 2;
        for (int i = grp; i < nr; i += G) {
            const long off = (long)(q0 + i) * h + c;
            cp_async16(sdy + (size_t)i * h + c, dy + off);
            cp_async16(sx + (size_t)i * h + c, x + off);
            if (resid) cp_async16(sr + (size_t)i * h + c, resid + off);
            if (i < half && i + G >= half) asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        for (int i = grp; i < nr; i += G) {
            if (i < half) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            const int r = q0 + i;
            const uint4 du = *reinterpret_cast<const uint4*>(sdy + (size_t)i * h + c);
            const uint4 xu = *reinterpret_cast<const uint4*>(sx + (size_t)i * h + c);
            const uint32_t dw[4] = {du.x, du.y, du.z, du.w}, xw[4] = {xu.x, xu.y, xu.z, xu.w};
            uint64_t r2[4] = {0ull, 0ull, 0ull, 0ull};
            if (resid) {
                const uint4 ru = *reinterpret_cast<const uint4*>(sr + (size_t)i * h + c);
                r2[0] = bfpair(ru.x);
                r2[1] = bfpair(ru.y);
                r2[2] = bfpair(ru.z);
                r2[3] = bfpair(ru.w);
            }
            const float mu = smu[r - r0], rs = srs[r - r0];
            const uint64_t rs2 = fpair(rs, rs), nm2 = fpair(-mu, -mu);
            uint64_t xh2[4], dxh2[4], s1_2 = 0ull, s2_2 = 0ull;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t d2 = bfpair(dw[j]);
                xh2[j] = fmul2x(fadd2x(bfpair(xw[j]), nm2), rs2);   // (x - mu) * rstd
                dxh2[j] = fmul2x(d2, g2[j]);
                s1_2 = fadd2x(s1_2, dxh2[j]);
                s2_2 = ffma2x(dxh2[j], xh2[j], s2_2);
                pg2[j] = ffma2x(d2, xh2[j], pg2[j]);
                pb2[j] = fadd2x(pb2[j], d2);
                if (resid) pr2[j] = fadd2x(pr2[j], r2[j]);
            }
            float s1a, s1b, s2a, s2b;
            funpair(s1_2, s1a, s1b);
            funpair(s2_2, s2a, s2b);
            float s1 = s1a + s1b, s2 = s2a + s2b;
            group_sum2(s1, s2, red[grp], grp, tpr);
            const float c1 = s1 / (float)h, c2 = s2 / (float)h;
            const uint64_t nc1 = fpair(-c1, -c1), nc2 = fpair(-c2, -c2);
            uint32_t ow[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // rstd * (dxh - c1 - xh * c2) + resid
                const uint64_t t = ffma2x(xh2[j], nc2, fadd2x(dxh2[j], nc1));
                float o0, o1;
                funpair(ffma2x(t, rs2, r2[j]), o0, o1);
                __nv_bfloat162 hv = __floats2bfloat162_rn(o0, o1);
                ow[j] = *reinterpret_cast<uint32_t*>(&hv);
            }
            *reinterpret_cast<uint4*>(dx + (long)r * h + c) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
        __syncthreads();   // chunk buffer free for the next chunk / the combine below
    }
    float pg[8], pb[8], pr[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        funpair(pg2[j], pg[2 * j], pg[2 * j + 1]);
        funpair(pb2[j], pb[2 * j], pb[2 * j + 1]);
        funpair(pr2[j], pr[2 * j], pr[2 * j + 1]);
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

// ---------------------------------------------------------------- row-parallel backward
// LN backward for h = 256 * NSEG <= 2048 (the C2 width), one CTA of 8 warps per
// 16-row block. All of the block's dy / x / resid rows are fetched at once
// with 16-byte cp.async into shared memory (warp w fetches, lane-sliced, the
// two rows w and w + 8 it computes, one commit group per row), then:
//  1. dx: a warp per row, the two row means (of dxhat and dxhat * xhat) by
//     warp shuffles only -- no CTA barrier per row (the staged kernel above
//     serialised the rows behind a 256-thread named barrier each and ran at
//     0.36 of the HBM peak, bench hbm_kernels);
//  2. after one __syncthreads, the dgamma / dbeta / dresid column partials: a
//     thread owns 8 columns and accumulates them over the 16 rows in row order,
//     from shared memory.
// Deterministic: fixed shuffle trees, fixed row order. Same partial layout as
// ln_bwd_stage_kernel ([3][nblk][h]).
template <int NSEG>
__global__ void __launch_bounds__(256, 1)
ln_bwd_rows_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x, const bf16* __restrict__ gamma,
                   const float* __restrict__ mean, const float* __restrict__ rstd,
                   const bf16* __restrict__ resid, bf16* __restrict__ dx, float* __restrict__ ws, int rows,
                   int nblk, int with_rsum) {
    constexpr int h = NSEG * 256;
    pdl_wait();
    pdl_trigger();
    __shared__ float smu[RB], srs[RB];
    extern __shared__ __align__(128) uint8_t smraw[];
    bf16* sdy = reinterpret_cast<bf16*>(smraw);   // [RB][h]
    bf16* sx = sdy + RB * h;                      // [RB][h]
    bf16* sr = sx + RB * h;                       // [RB][h]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = blockIdx.x * RB, nr = min(RB, rows - r0);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int k = warp + 8 * q;
        if (k < nr) {
            const long base = (long)(r0 + k) * h;
#pragma unroll
            for (int i = 0; i < NSEG; ++i) {
                const int c = (i * 32 + lane) * 8;
                cp_async16(sdy + k * h + c, dy + base + c);
                cp_async16(sx + k * h + c, x + base + c);
                if (resid) cp_async16(sr + k * h + c, resid + base + c);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (threadIdx.x < nr) {
        smu[threadIdx.x] = mean[r0 + threadIdx.x];
        srs[threadIdx.x] = rstd[r0 + threadIdx.x];
    }
    uint4 gu[NSEG];
#pragma unroll
    for (int i = 0; i < NSEG; ++i) gu[i] = __ldg(reinterpret_cast<const uint4*>(gamma + (i * 32 + lane) * 8));
    __syncthreads();   // smu / srs
    // ---- phase 1: dx, rows warp and warp + 8
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int k = warp + 8 * q;
        if (q == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        if (k >= nr) continue;
        const float mu = smu[k], rs = srs[k];
        const uint64_t rs2 = fpair(rs, rs), nm2 = fpair(-mu, -mu);
        uint64_t s1_2 = 0ull, s2_2 = 0ull;
#pragma unroll
        for (int i = 0; i < NSEG; ++i) {
            const int c = (i * 32 + lane) * 8;
            const uint4 du = *reinterpret_cast<const uint4*>(sdy + k * h + c);
            const uint4 xu = *reinterpret_cast<const uint4*>(sx + k * h + c);
            const uint32_t dw[4] = {du.x, du.y, du.z, du.w}, xw[4] = {xu.x, xu.y, xu.z, xu.w},
                           gw[4] = {gu[i].x, gu[i].y, gu[i].z, gu[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t xh2 = fmul2x(fadd2x(bfpair(xw[j]), nm2), rs2);   // (x - mu) * rstd
                const uint64_t dxh2 = fmul2x(bfpair(dw[j]), bfpair(gw[j]));
                s1_2 = fadd2x(s1_2, dxh2);
                s2_2 = ffma2x(dxh2, xh2, s2_2);
            }
        }
        float s1a, s1b, s2a, s2b;
        funpair(s1_2, s1a, s1b);
        funpair(s2_2, s2a, s2b);
        const float s1 = warp_sum(s1a + s1b), s2 = warp_sum(s2a + s2b);
        const float c1 = s1 / (float)h, c2 = s2 / (float)h;
        const uint64_t nc1 = fpair(-c1, -c1), nc2 = fpair(-c2, -c2);
        const long base = (long)(r0 + k) * h;
#pragma unroll
        for (int i = 0; i < NSEG; ++i) {
            const int c = (i * 32 + lane) * 8;
            const uint4 du = *reinterpret_cast<const uint4*>(sdy + k * h + c);
            const uint4 xu = *reinterpret_cast<const uint4*>(sx + k * h + c);
            uint4 ru = make_uint4(0, 0, 0, 0);
            if (resid) ru = *reinterpret_cast<const uint4*>(sr + k * h + c);
            const uint32_t dw[4] = {du.x, du.y, du.z, du.w}, xw[4] = {xu.x, xu.y, xu.z, xu.w},
                           gw[4] = {gu[i].x, gu[i].y, gu[i].z, gu[i].w}, rw[4] = {ru.x, ru.y, ru.z, ru.w};
            uint32_t ow[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint64_t xh2 = fmul2x(fadd2x(bfpair(xw[j]), nm2), rs2);
                const uint64_t dxh2 = fmul2x(bfpair(dw[j]), bfpair(gw[j]));
                // rstd * (dxh - c1 - xh * c2) + resid
                const uint64_t t = ffma2x(xh2, nc2, fadd2x(dxh2, nc1));
                float o0, o1;
                funpair(ffma2x(t, rs2, bfpair(rw[j])), o0, o1);
                __nv_bfloat162 hv = __floats2bfloat162_rn(o0, o1);
                ow[j] = *reinterpret_cast<uint32_t*>(&hv);
            }
            *reinterpret_cast<uint4*>(dx + base + c) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
        }
    }
    __syncthreads();   // every row of the block is in shared memory
    // ---- phase 2: column partials over the block's rows (row order)
    const int c = threadIdx.x * 8;
    if (c >= h) return;
    uint64_t pg2[4] = {0ull, 0ull, 0ull, 0ull}, pb2[4] = {0ull, 0ull, 0ull, 0ull},
             pr2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll 4
    for (int k = 0; k < nr; ++k) {
        const uint4 du = *reinterpret_cast<const uint4*>(sdy + k * h + c);
        const uint4 xu = *reinterpret_cast<const uint4*>(sx + k * h + c);
        const uint64_t rs2 = fpair(srs[k], srs[k]), nm2 = fpair(-smu[k], -smu[k]);
        const uint32_t dw[4] = {du.x, du.y, du.z, du.w}, xw[4] = {xu.x, xu.y, xu.z, xu.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t d2 = bfpair(dw[j]);
            const uint64_t xh2 = fmul2x(fadd2x(bfpair(xw[j]), nm2), rs2);
            pg2[j] = ffma2x(d2, xh2, pg2[j]);
            pb2[j] = fadd2x(pb2[j], d2);
        }
        if (with_rsum) {
            const uint4 ru = *reinterpret_cast<const uint4*>(sr + k * h + c);
            const uint32_t rw[4] = {ru.x, ru.y, ru.z, ru.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) pr2[j] = fadd2x(pr2[j], bfpair(rw[j]));
        }
    }
    float pg[8], pb[8], pr[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        funpair(pg2[j], pg[2 * j], pg[2 * j + 1]);
        funpair(pb2[j], pb[2 * j], pb[2 * j + 1]);
        funpair(pr2[j], pr[2 * j], pr[2 * j + 1]);
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

// row-parallel backward for h in {256, 512, ..., 2048}; false = not handled
static bool launch_ln_bwd_rows(const void* dy, const void* x, const void* gamma, const float* mean,
                               const float* rstd, const void* resid, void* dx, float* ws, int rows, int h,
                               int nb, int with_rsum, cudaStream_t st) {
    if (!g_ln_rows || h % 256 || h > 2048) return false;
    switch (h / 256) {
#define TP_LNR(S)                                                                                         \
    case S: {                                                                                             \
        static PerDeviceOnce attr;                                                                        \
        if (attr.first())                                                                                 \
            cudaFuncSetAttribute(ln_bwd_rows_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                 3 * RB * 256 * S * 2);                                                   \
        launch_k(ln_bwd_rows_kernel<S>, dim3(nb), dim3(256), (size_t)3 * RB * h * 2, st, 1,               \
                 (const bf16*)dy, (const bf16*)x, (const bf16*)gamma, mean, rstd, (const bf16*)resid,     \
                 (bf16*)dx, ws, rows, nb, with_rsum);                                                     \
        return true;                                                                                      \
    }
        TP_LNR(1) TP_LNR(2) TP_LNR(3) TP_LNR(4) TP_LNR(5) TP_LNR(6) TP_LNR(7) TP_LNR(8)
#undef TP_LNR
        default: return false;
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
        if (ln_fwd_warp((const bf16*)x, (const bf16*)gamma, (const bf16*)beta, (bf16*)y, mean, rstd, rows, h, 0,
                        st))
            return -1;
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
        if (ln_fwd_warp((const bf16*)x, (const bf16*)gamma, (const bf16*)beta, (bf16*)y, const_cast<float*>(mean),
                        const_cast<float*>(rstd), rows, h, 1, st))
            return -1;
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
        // rows staged per chunk: all RB rows of the three inputs when they fit
        int RC = LNB_SMEM_ROWS_BYTES / (3 * h * 2);
        if (RC > RB) RC = RB;
        const size_t smem = (size_t)RC * 3 * h * 2;
        if (!launch_ln_bwd_rows(dy, x, gamma, mean, rstd, resid, dx, ws, rows, h, nb, rs, st)) {
            static PerDeviceOnce attr;
            if (attr.first()) {
                cudaFuncSetAttribute(ln_bwd_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     LNB_SMEM_ROWS_BYTES);
            }
            launch_k(ln_bwd_stage_kernel, dim3(nb), dim3(G * (h / 8)), smem, st, 1, (const bf16*)dy,
                     (const bf16*)x, (const bf16*)gamma, (const float*)mean, (const float*)rstd,
                     (const bf16*)resid, (bf16*)dx, ws, rows, h, nb, rs, RC);
        }
        launch_k(reduce_parts_kernel, dim3((h + 31) / 32, 2 + rs), dim3(256), 0, st, 1, (const float*)ws, dgamma,
                 dbeta, dresid_sum, h, nb);
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
        launch_k(colsum_wide_kernel, dim3((n + CS_COLS - 1) / CS_COLS, nb), dim3(256), 0, st, 1, (const bf16*)X, ws,
                 rows, n);
        launch_k(reduce_parts_kernel, dim3((n + 31) / 32, 1), dim3(256), 0, st, 1, (const float*)ws, out,
                 (float*)nullptr, (float*)nullptr, n, nb);
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

// ---------------------------------------------------------------- deferred reductions
// bf16 wide path only (return -1 otherwise: the caller uses ln_bwd / colsum_acc):
// write the RB-row-block partials, leave the reduce to reduce_segments.
int colsum_partials(int dtype, const void* X, float* ws, int rows, int n, cudaStream_t st) {
    if (rows <= 0 || n <= 0) return 0;
    if (!(dtype == DT_BF16 && n % 8 == 0)) return -1;
    const int nb = (rows + RB - 1) / RB;
    launch_k(colsum_wide_kernel, dim3((n + CS_COLS - 1) / CS_COLS, nb), dim3(256), 0, st, 1, (const bf16*)X, ws,
             rows, n);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int ln_bwd_partials(int dtype, const void* dy, const void* x, const void* gamma, const float* mean,
                    const float* rstd, const void* resid, void* dx, float* ws, int rows, int h, int with_rsum,
                    cudaStream_t st) {
    if (rows <= 0) return 0;
    if (!wide_ok(dtype, h) || (with_rsum && !resid)) return -1;
    const int nb = (rows + RB - 1) / RB;
    const int G = wide_groups(h);
    int RC = LNB_SMEM_ROWS_BYTES / (3 * h * 2);
    if (RC > RB) RC = RB;
    const size_t smem = (size_t)RC * 3 * h * 2;
    if (!launch_ln_bwd_rows(dy, x, gamma, mean, rstd, resid, dx, ws, rows, h, nb, with_rsum ? 1 : 0, st)) {
        static PerDeviceOnce attr;
        if (attr.first()) {
            cudaFuncSetAttribute(ln_bwd_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 LNB_SMEM_ROWS_BYTES);
        }
        launch_k(ln_bwd_stage_kernel, dim3(nb), dim3(G * (h / 8)), smem, st, 1, (const bf16*)dy, (const bf16*)x,
                 (const bf16*)gamma, (const float*)mean, (const float*)rstd, (const bf16*)resid, (bf16*)dx, ws,
                 rows, h, nb, with_rsum ? 1 : 0, RC);
    }
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int reduce_segments(const float* const* src, float* const* out, const int* n, int nseg, int rows,
                    cudaStream_t st) {
    if (nseg <= 0 || nseg > 4 || rows <= 0) return nseg == 0 ? 0 : -1;
    ReduceSegs sg{};
    for (int i = 0; i < nseg; ++i) {
        if (n[i] % 4) return -1;
        sg.src[i] = src[i];
        sg.out[i] = out[i];
        sg.n[i] = n[i];
    }
    const int nb = (rows + RB - 1) / RB;
    sg.cb[0] = 0;
    for (int i = 0; i < 4; ++i) sg.cb[i + 1] = sg.cb[i] + (i < nseg ? (sg.n[i] + 31) / 32 : 0);
    launch_k(reduce_segs_kernel, dim3(sg.cb[4]), dim3(256), 0, st, 1, sg, nb);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace tpipe
