// Causal flash attention on 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// bf16, head_dim 64 / 128 (FlashAttention is the paper's
// default). One CTA = 128 query rows (fwd, dQ) or 128 keys (dK/dV) of
// one (sequence, head).
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one
// thread), warp 2 = TMEM allocator, warps 4..7 = 128 "row" threads (thread r
// owns TMEM lane r = one query / key row) doing softmax / dS and epilogues.
//
// Shared-memory tiles are [64-element atom][rows][128 B] with the 128-byte
// swizzle, so one tile serves as a K-major operand (rows = M/N, K = head dim)
// and as an MN-major operand (rows = K, N = head dim) — Q, K, V, dO are each
// loaded once per block and used both ways. P / dS are written by the row
// threads into the same layout (rows = M, K = keys / queries) and consumed by
// tcgen05.mma from shared memory after fence.proxy.async.
//
//   fwd : S = Q K^T (TMEM), P = exp2(S*c - m), O_j = P V (TMEM) accumulated
//         into registers with the online-softmax correction; saves O, LSE.
//   dKdV: S^T = K Q^T, dP^T = V dO^T (TMEM); P^T, dS^T -> smem;
//         dV += P^T dO, dK += dS^T Q (TMEM accumulators).
//   dQ  : S = Q K^T, dP = dO V^T; dS -> smem; dQ += dS K.
// Deterministic: no atomics; every output row is owned by one CTA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace tpipe {
namespace fa5 {

constexpr int BR = 128;          // rows per tile (queries or keys)
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// kind::f16 instruction descriptor, M = 128, bf16 x bf16 -> f32
__device__ __forceinline__ uint32_t idesc(int N, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
           ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// tile of `rows` rows x D (bf16), [D/64 atoms][rows][128 B]
template <int D>
struct Tile {
    static constexpr int ATOM = BR * 128;        // bytes per atom (128 rows)
    static constexpr int BYTES = (D / 64) * ATOM;
};

// K-major descriptor for K-step k (16 elements) of a [atoms][128 rows][64] tile
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int k) {
    return umma_desc_sw128(base + (k >> 2) * (BR * 128) + (k & 3) * 32, 0, 1024);
}
// MN-major descriptor for K-step k (16 rows) of a tile whose rows are K and
// whose 64-element atoms run along N
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int k) {
    return umma_desc_sw128(base + k * 2048, BR * 128, 1024);
}

// swizzled byte offset of 16-byte chunk c (0..7) of row r within one atom
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

// write 32 consecutive bf16 values (columns col0..col0+31) of row r
__device__ __forceinline__ void st_row32(uint8_t* tile, int r, int col0, const float (&v)[32]) {
    uint8_t* atom = tile + (col0 >> 6) * (BR * 128);
    const int c0 = (col0 & 63) >> 3;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint4 u;
        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) hh[j] = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
        *reinterpret_cast<uint4*>(atom + swz(r, c0 + q)) = u;
    }
}

__device__ __forceinline__ void tmem_ld32f(uint32_t addr, float (&v)[32]) {
    uint32_t r[32];
    tmem_ld32(addr, r);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// TMA loads of a 128-row x D tile starting at (col, row) of a 2-D bf16 map
template <int D>
__device__ __forceinline__ void tma_tile(uint8_t* sm, const CUtensorMap* map, uint64_t* bar, int col,
                                         int row) {
#pragma unroll
    for (int a = 0; a < D / 64; ++a) tma_load_2d(sm + a * (BR * 128), map, bar, col + a * 64, row);
}

// ============================================================== forward
template <int D>
__global__ void __launch_bounds__(256, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, bf16* __restrict__ o,
               float* __restrict__ lse, int s, int a) {
    constexpr int TB = Tile<D>::BYTES;
    constexpr int STAGES = 2;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sK = sQ + TB;                   // STAGES
    uint8_t* sV = sK + STAGES * TB;          // STAGES
    uint8_t* sP = sV + STAGES * TB;          // 128 x 128 bf16 (2 atoms)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 2 * BR * 128);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;             // [STAGES]
    uint64_t* kv_empty = kv_full + STAGES;   // [STAGES]
    uint64_t* s_full = kv_empty + STAGES;
    uint64_t* p_full = s_full + 1;
    uint64_t* o_full = p_full + 1;           // PV done (also frees P and S)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int qb = nqb - 1 - blockIdx.x;  // heaviest first
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const int q0 = qb * BR;
    const int row0 = b * s;               // first row of this sequence in [b*s, 3h]
    const int nkb = qb + 1;               // key blocks 0..qb (BR == BN)

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        mbar_init(q_full, 1);
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(p_full, 128);
        mbar_init(o_full, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tO = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, TB);
            tma_tile<D>(sQ, &tm_qkv, q_full, head * D, row0 + q0);
            for (int j = 0; j < nkb; ++j) {
                const int st = j % STAGES;
                mbar_wait(&kv_empty[st], ((j / STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[st], 2 * TB);
                tma_tile<D>(sK + st * TB, &tm_qkv, &kv_full[st], h + head * D, row0 + j * BR);
                tma_tile<D>(sV + st * TB, &tm_qkv, &kv_full[st], 2 * h + head * D, row0 + j * BR);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t iS = idesc(BR, false, false);
            const uint32_t iO = idesc(D, false, true);
            const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
            mbar_wait(q_full, 0);
            for (int j = 0; j < nkb; ++j) {
                const int st = j % STAGES;
                mbar_wait(&kv_full[st], (j / STAGES) & 1);
                if (j > 0) mbar_wait(o_full, (j - 1) & 1);   // S/P of block j-1 consumed
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + st * TB), aV = smem_u32(sV + st * TB);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) umma_bf16(tS, desc_k(aQ, k), desc_k(aK, k), iS, k > 0);
                umma_commit(s_full);
                mbar_wait(p_full, j & 1);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < BR / 16; ++k) umma_bf16(tO, desc_k(aP, k), desc_mn(aV, k), iO, k > 0);
                umma_commit(o_full);
                umma_commit(&kv_empty[st]);
            }
        }
    } else if (warp >= 4) {
        const int r = threadIdx.x - 128;           // query row within the tile == TMEM lane
        const int q = q0 + r;
        const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        float m = -INFINITY, l = 0.f;
        float oacc[D];
#pragma unroll
        for (int i = 0; i < D; ++i) oacc[i] = 0.f;
        for (int j = 0; j < nkb; ++j) {
            mbar_wait(s_full, j & 1);
            tc_fence_after();
            const bool diag = (j == nkb - 1);
            // pass 1: row max of the scaled, masked scores
            float mx = m;
#pragma unroll
            for (int c = 0; c < BR / 32; ++c) {
                float v[32];
                tmem_ld32f(tS + lane_off + c * 32, v);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int key = j * BR + c * 32 + e;
                    const float x = (diag && key > q) ? -INFINITY : v[e] * sc;
                    mx = fmaxf(mx, x);
                }
            }
            const float corr = exp2f(m - mx);
            float rs = 0.f;
            // pass 2: P = exp2(x - mx) -> smem (bf16), row sum
#pragma unroll
            for (int c = 0; c < BR / 32; ++c) {
                float v[32];
                tmem_ld32f(tS + lane_off + c * 32, v);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int key = j * BR + c * 32 + e;
                    const float p = (diag && key > q) ? 0.f : exp2f(v[e] * sc - mx);
                    v[e] = p;
                    rs += p;
                }
                st_row32(sP, r, c * 32, v);
            }
            l = l * corr + rs;
            m = mx;
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(p_full);
            // O = O * corr + P V
            mbar_wait(o_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                float v[32];
                tmem_ld32f(tO + lane_off + c * 32, v);
#pragma unroll
                for (int e = 0; e < 32; ++e) oacc[c * 32 + e] = oacc[c * 32 + e] * corr + v[e];
            }
            tc_fence_before();
        }
        if (q < s) {
            const float inv = 1.0f / l;
            bf16* orow = o + ((long)b * s + q) * h + head * D;
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                uint4 u;
                __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    hh[jj] = __floats2bfloat162_rn(oacc[c * 8 + 2 * jj] * inv, oacc[c * 8 + 2 * jj + 1] * inv);
                *reinterpret_cast<uint4*>(orow + c * 8) = u;
            }
            lse[((long)b * a + head) * s + q] = (m + log2f(l)) / LOG2E;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ============================================================== forward v2
// S double-buffered in TMEM (columns [0,128) and [128,256)); P_j is written
// back over S_j as packed bf16 (64 columns) and consumed as the TMEM
// A-operand of O += P_j V_j; O (D columns at 256) accumulates in TMEM and is
// rescaled in place by the row threads when the running max moves.
//   MMA  : S_0 | for j: [S_{j+1} once PV_{j-1} freed its buffer] [PV_j once P_j ready]
//   rows : S_j -> P_j (one pass, 128 scores in registers) -> wait PV_{j-1}
//          -> O *= corr_j (skipped per warp when corr == 1) -> P_j ready
template <int D>
__global__ void __launch_bounds__(384, 1)
    fwd2_kernel(const __grid_constant__ CUtensorMap tm_qkv, bf16* __restrict__ o,
                float* __restrict__ lse, int s, int a) {
    constexpr int TB = Tile<D>::BYTES;
    constexpr int STAGES = 2;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sK = sQ + TB;                   // STAGES
    uint8_t* sV = sK + STAGES * TB;          // STAGES
    float* sMax = reinterpret_cast<float*>(sV + STAGES * TB);   // [2 iters][2 groups][128]
    float* sSum = sMax + 4 * BR;                                  // [2 groups][128]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sSum + 2 * BR);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;             // [STAGES]
    uint64_t* kv_empty = kv_full + STAGES;   // [STAGES]
    uint64_t* s_full = kv_empty + STAGES;    // [2] S buffer ready
    uint64_t* p_full = s_full + 2;           // P_j in TMEM + O corrected (128 arrivals)
    uint64_t* pv_done = p_full + 1;          // PV_j complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int qb = nqb - 1 - blockIdx.x;  // heaviest first
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const int q0 = qb * BR;
    const int row0 = b * s;
    const int nkb = qb + 1;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        mbar_init(q_full, 1);
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        mbar_init(p_full, 256);
        mbar_init(pv_done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tO = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, TB);
            tma_tile<D>(sQ, &tm_qkv, q_full, head * D, row0 + q0);
            for (int j = 0; j < nkb; ++j) {
                const int st = j % STAGES;
                mbar_wait(&kv_empty[st], ((j / STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[st], 2 * TB);
                tma_tile<D>(sK + st * TB, &tm_qkv, &kv_full[st], h + head * D, row0 + j * BR);
                tma_tile<D>(sV + st * TB, &tm_qkv, &kv_full[st], 2 * h + head * D, row0 + j * BR);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t iS = idesc(BR, false, false);
            const uint32_t iO = idesc(D, false, true);
            const uint32_t aQ = smem_u32(sQ);
            mbar_wait(q_full, 0);
            auto issue_s = [&](int j) {
                const int st = j % STAGES;
                mbar_wait(&kv_full[st], (j / STAGES) & 1);
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + st * TB);
                const uint32_t tS = tmem + (j & 1) * 128;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) umma_bf16(tS, desc_k(aQ, k), desc_k(aK, k), iS, k > 0);
                umma_commit(&s_full[j & 1]);
            };
            issue_s(0);
            for (int j = 0; j < nkb; ++j) {
                if (j + 1 < nkb) {
                    if (j >= 1) mbar_wait(pv_done, (j - 1) & 1);  // buffer (j+1)&1 held P_{j-1}
                    issue_s(j + 1);
                }
                mbar_wait(p_full, j & 1);
                tc_fence_after();
                const int st = j % STAGES;
                const uint32_t aV = smem_u32(sV + st * TB);
                const uint32_t tP = tmem + (j & 1) * 128;
#pragma unroll
                for (int k = 0; k < BR / 16; ++k)
                    umma_bf16_ts(tO, tP + k * 8, desc_mn(aV, k), iO, (j | k) > 0);
                umma_commit(pv_done);
                umma_commit(&kv_empty[st]);
            }
        }
    } else if (warp >= 4) {
        // 8 softmax warps: row r = TMEM lane (warp % 4 = lane quarter); column
        // group cg owns scores [64cg, 64cg+64) and O columns [cg D/2, (cg+1) D/2)
        const int et = threadIdx.x - 128;
        const int r = et & 127, cg = et >> 7;
        const int q = q0 + r;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nkb; ++j) {
            const uint32_t tS = tmem + (j & 1) * 128 + lane_off;
            mbar_wait(&s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            float sv[64];
            {
                uint32_t rr[32];
                tmem_ld32(tS + cg * 64, rr);
#pragma unroll
                for (int e = 0; e < 32; ++e) sv[e] = __uint_as_float(rr[e]);
                tmem_ld32(tS + cg * 64 + 32, rr);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) sv[32 + e] = __uint_as_float(rr[e]);
            }
            const bool diag = (j == nkb - 1);
            float lmx = -INFINITY;
#pragma unroll
            for (int e = 0; e < 64; ++e) {
                const float x = (diag && j * BR + cg * 64 + e > q) ? -INFINITY : sv[e] * sc;
                sv[e] = x;
                lmx = fmaxf(lmx, x);
            }
            float* mb = sMax + (j & 1) * 2 * BR;
            mb[cg * BR + r] = lmx;
            named_bar_sync(1, 256);
            const float mx = fmaxf(m, fmaxf(lmx, mb[(cg ^ 1) * BR + r]));
            float rs = 0.f;
            uint32_t pk[32];
#pragma unroll
            for (int e = 0; e < 64; e += 2) {
                const float p0 = exp2f(sv[e] - mx), p1 = exp2f(sv[e + 1] - mx);
                rs += p0 + p1;
                __nv_bfloat162 v2 = __floats2bfloat162_rn(p0, p1);
                pk[e / 2] = *reinterpret_cast<uint32_t*>(&v2);
            }
            const float corr = exp2f(m - mx);
            l = l * corr + rs;        // partial (this group's columns), same m history
            m = mx;
            tmem_st32(tS + cg * 32, pk);   // P_j over S_j: packed cols [32cg, 32cg+32)
            if (j > 0) {
                mbar_wait(pv_done, (j - 1) & 1);
                tc_fence_after();
                if (__any_sync(0xffffffffu, corr != 1.0f)) {
#pragma unroll
                    for (int c = cg * (D / 64); c < (cg + 1) * (D / 64); ++c) {
                        uint32_t ov[32];
                        tmem_ld32(tO + lane_off + c * 32, ov);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * corr);
                        tmem_st32(tO + lane_off + c * 32, ov);
                    }
                }
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        sSum[cg * BR + r] = l;
        named_bar_sync(1, 256);
        l += sSum[(cg ^ 1) * BR + r];
        mbar_wait(pv_done, (nkb - 1) & 1);
        tc_fence_after();
        // tcgen05.ld is .sync.aligned: every lane loads; only valid rows store
        const float inv = 1.0f / l;
        bf16* orow = o + ((long)b * s + q) * h + head * D;
#pragma unroll
        for (int c = cg * (D / 64); c < (cg + 1) * (D / 64); ++c) {
            float v[32];
            tmem_ld32f(tO + lane_off + c * 32, v);
            if (q < s) {
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8) {
                    uint4 u;
                    __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        hh[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj] * inv, v[q8 * 8 + 2 * jj + 1] * inv);
                    *reinterpret_cast<uint4*>(orow + c * 32 + q8 * 8) = u;
                }
            }
        }
        if (q < s && cg == 0) lse[((long)b * a + head) * s + q] = (m + log2f(l)) / LOG2E;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ============================================================== backward dK, dV
template <int D>
__global__ void __launch_bounds__(256, 1)
    dkdv_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                const float* __restrict__ lse, const float* __restrict__ Dv,
                bf16* __restrict__ dqkv, int s, int a) {
    constexpr int TB = Tile<D>::BYTES;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = sm;
    uint8_t* sV = sK + TB;
    uint8_t* sQ = sV + TB;            // per query block
    uint8_t* sO = sQ + TB;            // dO
    uint8_t* sP = sO + TB;            // P^T  [keys][queries] (2 atoms)
    uint8_t* sS = sP + 2 * BR * 128;  // dS^T
    float* sL = reinterpret_cast<float*>(sS + 2 * BR * 128);   // LSE*log2e of the q block
    float* sD = sL + BR;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sD + BR);
    uint64_t* kv_full = bar;
    uint64_t* q_full = bar + 1;
    uint64_t* s_full = bar + 2;       // S^T, dP^T ready
    uint64_t* p_full = bar + 3;       // P^T, dS^T written (128 arrivals)
    uint64_t* g_done = bar + 4;       // dV/dK MMAs of this block done (frees Q, dO, P, dS, S)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int kb = blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const int k0 = kb * BR;
    const int row0 = b * s;
    const float* lseb = lse + ((long)b * a + head) * s;
    const float* Db = Dv + ((long)b * a + head) * s;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        tma_prefetch_desc(&tm_do);
        mbar_init(kv_full, 1);
        mbar_init(q_full, 1);
        mbar_init(s_full, 1);
        mbar_init(p_full, 128);
        mbar_init(g_done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tP = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + D;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * TB);
            tma_tile<D>(sK, &tm_qkv, kv_full, h + head * D, row0 + k0);
            tma_tile<D>(sV, &tm_qkv, kv_full, 2 * h + head * D, row0 + k0);
            for (int qb = kb, it = 0; qb < nqb; ++qb, ++it) {
                if (it > 0) mbar_wait(g_done, (it - 1) & 1);
                mbar_arrive_expect_tx(q_full, 2 * TB);
                tma_tile<D>(sQ, &tm_qkv, q_full, head * D, row0 + qb * BR);
                tma_tile<D>(sO, &tm_do, q_full, head * D, row0 + qb * BR);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t iS = idesc(BR, false, false);
            const uint32_t iG = idesc(D, false, true);
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ),
                           aO = smem_u32(sO), aP = smem_u32(sP), aS = smem_u32(sS);
            mbar_wait(kv_full, 0);
            for (int qb = kb, it = 0; qb < nqb; ++qb, ++it) {
                mbar_wait(q_full, it & 1);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    umma_bf16(tS, desc_k(aK, k), desc_k(aQ, k), iS, k > 0);   // S^T = K Q^T
                    umma_bf16(tP, desc_k(aV, k), desc_k(aO, k), iS, k > 0);   // dP^T = V dO^T
                }
                umma_commit(s_full);
                mbar_wait(p_full, it & 1);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < BR / 16; ++k) {
                    umma_bf16(tdV, desc_k(aP, k), desc_mn(aO, k), iG, (it | k) > 0);  // dV += P^T dO
                    umma_bf16(tdK, desc_k(aS, k), desc_mn(aQ, k), iG, (it | k) > 0);  // dK += dS^T Q
                }
                umma_commit(g_done);
            }
        }
    } else if (warp >= 4) {
        const int r = threadIdx.x - 128;          // key row == TMEM lane
        const int key = k0 + r;
        const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        for (int qb = kb, it = 0; qb < nqb; ++qb, ++it) {
            const int q0 = qb * BR;
            // L, D of the query block -> smem (previous block's readers are done:
            // they arrived on p_full, and the MMA reading sP/sS has completed
            // before s_full of this block was committed)
            if (it > 0) mbar_wait(g_done, (it - 1) & 1);
            {
                const int qq = q0 + r;
                sL[r] = qq < s ? lseb[qq] * LOG2E : 0.f;
                sD[r] = qq < s ? Db[qq] : 0.f;
            }
            named_bar_sync(1, 128);
            mbar_wait(s_full, it & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BR / 32; ++c) {
                float sv[32], pv[32];
                tmem_ld32f(tS + lane_off + c * 32, sv);
                tmem_ld32f(tP + lane_off + c * 32, pv);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int ql = c * 32 + e, qq = q0 + ql;
                    const float p = (qq >= key && qq < s) ? exp2f(sv[e] * sc - sL[ql]) : 0.f;
                    sv[e] = p;
                    pv[e] = p * (pv[e] - sD[ql]);
                }
                st_row32(sP, r, c * 32, sv);
                st_row32(sS, r, c * 32, pv);
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        // epilogue: dK (scaled), dV
        mbar_wait(g_done, (nqb - kb - 1) & 1);
        tc_fence_after();
        {   // every lane loads (tcgen05.ld is .sync.aligned); only valid keys store
            const float scale = rsqrtf((float)D);
            bf16* dkr = dqkv + ((long)b * s + key) * (3L * h) + h + head * D;
            bf16* dvr = dkr + h;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                float v[32];
                tmem_ld32f(tdK + lane_off + c * 32, v);
                if (key < s) {
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        uint4 u;
                        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            hh[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj] * scale, v[q8 * 8 + 2 * jj + 1] * scale);
                        *reinterpret_cast<uint4*>(dkr + c * 32 + q8 * 8) = u;
                    }
                }
                tmem_ld32f(tdV + lane_off + c * 32, v);
                if (key < s) {
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        uint4 u;
                        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            hh[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj], v[q8 * 8 + 2 * jj + 1]);
                        *reinterpret_cast<uint4*>(dvr + c * 32 + q8 * 8) = u;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ============================================================== backward dQ
template <int D>
__global__ void __launch_bounds__(256, 1)
    dq_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
              const float* __restrict__ lse, const float* __restrict__ Dv, bf16* __restrict__ dqkv,
              int s, int a) {
    constexpr int TB = Tile<D>::BYTES;
    constexpr int STAGES = 2;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sO = sQ + TB;                  // dO
    uint8_t* sK = sO + TB;                  // STAGES
    uint8_t* sV = sK + STAGES * TB;         // STAGES
    uint8_t* sS = sV + STAGES * TB;         // dS [queries][keys] (2 atoms)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sS + 2 * BR * 128);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;            // [STAGES]
    uint64_t* kv_empty = kv_full + STAGES;  // [STAGES]
    uint64_t* s_full = kv_empty + STAGES;
    uint64_t* p_full = s_full + 1;
    uint64_t* g_done = p_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(g_done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int qb = nqb - 1 - blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const int q0 = qb * BR;
    const int row0 = b * s;
    const int nkb = qb + 1;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        tma_prefetch_desc(&tm_do);
        mbar_init(q_full, 1);
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(p_full, 128);
        mbar_init(g_done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tP = tmem + 128, tdQ = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, 2 * TB);
            tma_tile<D>(sQ, &tm_qkv, q_full, head * D, row0 + q0);
            tma_tile<D>(sO, &tm_do, q_full, head * D, row0 + q0);
            for (int j = 0; j < nkb; ++j) {
                const int st = j % STAGES;
                mbar_wait(&kv_empty[st], ((j / STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[st], 2 * TB);
                tma_tile<D>(sK + st * TB, &tm_qkv, &kv_full[st], h + head * D, row0 + j * BR);
                tma_tile<D>(sV + st * TB, &tm_qkv, &kv_full[st], 2 * h + head * D, row0 + j * BR);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t iS = idesc(BR, false, false);
            const uint32_t iG = idesc(D, false, true);
            const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO), aS = smem_u32(sS);
            mbar_wait(q_full, 0);
            for (int j = 0; j < nkb; ++j) {
                const int st = j % STAGES;
                mbar_wait(&kv_full[st], (j / STAGES) & 1);
                if (j > 0) mbar_wait(g_done, (j - 1) & 1);
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + st * TB), aV = smem_u32(sV + st * TB);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    umma_bf16(tS, desc_k(aQ, k), desc_k(aK, k), iS, k > 0);   // S = Q K^T
                    umma_bf16(tP, desc_k(aO, k), desc_k(aV, k), iS, k > 0);   // dP = dO V^T
                }
                umma_commit(s_full);
                mbar_wait(p_full, j & 1);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < BR / 16; ++k)
                    umma_bf16(tdQ, desc_k(aS, k), desc_mn(aK, k), iG, (j | k) > 0);   // dQ += dS K
                umma_commit(g_done);
                umma_commit(&kv_empty[st]);
            }
        }
    } else if (warp >= 4) {
        const int r = threadIdx.x - 128;
        const int q = q0 + r;
        const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        const float* lseb = lse + ((long)b * a + head) * s;
        const float* Db = Dv + ((long)b * a + head) * s;
        const float L = q < s ? lseb[q] * LOG2E : 0.f;
        const float Dq = q < s ? Db[q] : 0.f;
        for (int j = 0; j < nkb; ++j) {
            mbar_wait(s_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int c = 0; c < BR / 32; ++c) {
                float sv[32], pv[32];
                tmem_ld32f(tS + lane_off + c * 32, sv);
                tmem_ld32f(tP + lane_off + c * 32, pv);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int key = j * BR + c * 32 + e;
                    const float p = (key <= q) ? exp2f(sv[e] * sc - L) : 0.f;
                    pv[e] = p * (pv[e] - Dq);
                }
                st_row32(sS, r, c * 32, pv);
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(p_full);
            // dS smem is re-written next iteration only after g_done (the MMA that
            // reads it) — wait for it before touching sS again
            mbar_wait(g_done, j & 1);
        }
        tc_fence_after();
        {   // every lane loads (tcgen05.ld is .sync.aligned); only valid rows store
            const float scale = rsqrtf((float)D);
            bf16* dqr = dqkv + ((long)b * s + q) * (3L * h) + head * D;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                float v[32];
                tmem_ld32f(tdQ + lane_off + c * 32, v);
                if (q < s) {
#pragma unroll
                    for (int q8 = 0; q8 < 4; ++q8) {
                        uint4 u;
                        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            hh[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj] * scale, v[q8 * 8 + 2 * jj + 1] * scale);
                        *reinterpret_cast<uint4*>(dqr + c * 32 + q8 * 8) = u;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ============================================================== backward v2
// 64-row halves so the MMA of half h+1 overlaps the elementwise work of half h.
// Half tiles are [D/64 atoms][64 rows][128 B] (atom stride 8 KB).
constexpr int HR = 64;
__device__ __forceinline__ uint64_t desc_k_h(uint32_t base, int k) {   // 64-row tile, K-major
    return umma_desc_sw128(base + (k >> 2) * (HR * 128) + (k & 3) * 32, 0, 1024);
}
__device__ __forceinline__ uint64_t desc_mn_h(uint32_t base, int k) {  // 64-row tile, MN-major
    return umma_desc_sw128(base + k * 2048, HR * 128, 1024);
}
template <int D>
__device__ __forceinline__ void tma_half(uint8_t* sm, const CUtensorMap* map, uint64_t* bar, int col,
                                         int row) {
#pragma unroll
    for (int a = 0; a < D / 64; ++a) tma_load_2d(sm + a * (HR * 128), map, bar, col + a * 64, row);
}
// write 32 bf16 (cols col0..col0+31, col0 < 64) of row r of a one-atom [rows][64] tile
__device__ __forceinline__ void st_row32_h(uint8_t* tile, int r, int col0, const float (&v)[32]) {
    const int c0 = col0 >> 3;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint4 u;
        __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) hh[j] = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
        *reinterpret_cast<uint4*>(tile + swz(r, c0 + q)) = u;
    }
}

// dK/dV: CTA owns 128 keys; loops over 64-query halves from the diagonal.
template <int D>
__global__ void __launch_bounds__(384, 1)
    dkdv2_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_qkv64,
                 const __grid_constant__ CUtensorMap tm_do64, const float* __restrict__ lse,
                 const float* __restrict__ Dv, bf16* __restrict__ dqkv, int s, int a) {
    constexpr int TB = Tile<D>::BYTES;          // 128-row tile
    constexpr int HB = (D / 64) * HR * 128;      // 64-row tile
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = sm;
    uint8_t* sV = sK + TB;
    uint8_t* sQ = sV + TB;                 // [2] half tiles
    uint8_t* sO = sQ + 2 * HB;             // [2] dO half tiles
    uint8_t* sP = sO + 2 * HB;             // [2] P^T  [128 keys][64 q] (one atom, 16 KB)
    uint8_t* sS = sP + 2 * BR * 128;       // [2] dS^T
    float* sL = reinterpret_cast<float*>(sS + 2 * BR * 128);   // [2][64]
    float* sD = sL + 2 * HR;                                   // [2][64]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sD + 2 * HR);
    uint64_t* kv_full = bar;
    uint64_t* q_full = bar + 1;     // [2]
    uint64_t* q_empty = bar + 3;    // [2]
    uint64_t* s_full = bar + 5;     // [2]
    uint64_t* p_full = bar + 7;     // 128 arrivals per half
    uint64_t* g_done = bar + 8;     // [2] dV/dK MMAs of a half complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kb = blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const int k0 = kb * BR;
    const int row0 = b * s;
    const int hq0 = k0 / HR;                   // first 64-query half at the diagonal
    const int nh = (s + HR - 1) / HR - hq0;    // halves to process
    const float* lseb = lse + ((long)b * a + head) * s;
    const float* Db = Dv + ((long)b * a + head) * s;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        tma_prefetch_desc(&tm_qkv64);
        tma_prefetch_desc(&tm_do64);
        mbar_init(kv_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&g_done[i], 1);
        }
        mbar_init(p_full, 256);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tdV = tmem + 256, tdK = tmem + 256 + D;   // D <= 128

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(kv_full, 2 * TB);
            tma_tile<D>(sK, &tm_qkv, kv_full, h + head * D, row0 + k0);
            tma_tile<D>(sV, &tm_qkv, kv_full, 2 * h + head * D, row0 + k0);
            for (int hh = 0; hh < nh; ++hh) {
                const int sl = hh & 1;
                mbar_wait(&q_empty[sl], ((hh >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&q_full[sl], 2 * HB);
                const int qrow = row0 + (hq0 + hh) * HR;
                tma_half<D>(sQ + sl * HB, &tm_qkv64, &q_full[sl], head * D, qrow);
                tma_half<D>(sO + sl * HB, &tm_do64, &q_full[sl], head * D, qrow);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t iS = idesc(HR, false, false);   // M=128 keys, N=64 queries
            const uint32_t iG = idesc(D, false, true);
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
            mbar_wait(kv_full, 0);
            auto issue_s = [&](int hh) {
                const int sl = hh & 1;
                mbar_wait(&q_full[sl], (hh >> 1) & 1);
                tc_fence_after();
                const uint32_t aQ = smem_u32(sQ + sl * HB), aO = smem_u32(sO + sl * HB);
                const uint32_t tS = tmem + sl * 128, tP = tS + 64;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    umma_bf16(tS, desc_k(aK, k), desc_k_h(aQ, k), iS, k > 0);   // S^T = K Q^T
                    umma_bf16(tP, desc_k(aV, k), desc_k_h(aO, k), iS, k > 0);   // dP^T = V dO^T
                }
                umma_commit(&s_full[sl]);
            };
            issue_s(0);
            for (int hh = 0; hh < nh; ++hh) {
                const int sl = hh & 1;
                if (hh + 1 < nh) issue_s(hh + 1);   // TMEM buffer (hh+1)&1 freed by p_full(hh-1)
                mbar_wait(p_full, hh & 1);
                tc_fence_after();
                const uint32_t aQ = smem_u32(sQ + sl * HB), aO = smem_u32(sO + sl * HB);
                const uint32_t aP = smem_u32(sP + sl * BR * 128), aS = smem_u32(sS + sl * BR * 128);
#pragma unroll
                for (int k = 0; k < HR / 16; ++k) {
                    umma_bf16(tdV, desc_k(aP, k), desc_mn_h(aO, k), iG, (hh | k) > 0);  // dV += P^T dO
                    umma_bf16(tdK, desc_k(aS, k), desc_mn_h(aQ, k), iG, (hh | k) > 0);  // dK += dS^T Q
                }
                umma_commit(&g_done[sl]);
                umma_commit(&q_empty[sl]);
            }
        }
    } else if (warp >= 4) {
        // 8 elementwise warps: row r = TMEM lane (warp % 4 selects the lane quarter),
        // column group cg = which 32 of the 64 half-columns this thread owns
        const int et = threadIdx.x - 128;
        const int r = et & 127, cg = et >> 7;
        const int key = k0 + r;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        for (int hh = 0; hh < nh; ++hh) {
            const int sl = hh & 1;
            const int q0 = (hq0 + hh) * HR;
            // P/dS buffer and L/D slot `sl` were last read by the MMA of half hh-2
            if (hh >= 2) mbar_wait(&g_done[sl], ((hh - 2) >> 1) & 1);
            if (et < HR) {
                const int qq = q0 + et;
                sL[sl * HR + et] = qq < s ? lseb[qq] * LOG2E : 0.f;
                sD[sl * HR + et] = qq < s ? Db[qq] : 0.f;
            }
            named_bar_sync(1, 256);
            mbar_wait(&s_full[sl], (hh >> 1) & 1);
            tc_fence_after();
            const uint32_t tS = tmem + sl * 128 + lane_off, tP = tS + 64;
            uint8_t* P = sP + sl * BR * 128;
            uint8_t* Sd = sS + sl * BR * 128;
            const float* L = sL + sl * HR;
            const float* Dq = sD + sl * HR;
            {
                const int c = cg;
                float sv[32], pv[32];
                tmem_ld32f(tS + c * 32, sv);
                tmem_ld32f(tP + c * 32, pv);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int ql = c * 32 + e, qq = q0 + ql;
                    const float p = (qq >= key && qq < s) ? exp2f(sv[e] * sc - L[ql]) : 0.f;
                    sv[e] = p;
                    pv[e] = p * (pv[e] - Dq[ql]);
                }
                st_row32_h(P, r, c * 32, sv);
                st_row32_h(Sd, r, c * 32, pv);
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        mbar_wait(&g_done[(nh - 1) & 1], ((nh - 1) >> 1) & 1);
        tc_fence_after();
        const float scale = rsqrtf((float)D);
        bf16* dkr = dqkv + ((long)b * s + key) * (3L * h) + h + head * D;
        bf16* dvr = dkr + h;
#pragma unroll
        for (int c = cg * (D / 64); c < (cg + 1) * (D / 64); ++c) {
            float v[32];
            tmem_ld32f(tdK + lane_off + c * 32, v);
            if (key < s) {
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8) {
                    uint4 u;
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        h2[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj] * scale, v[q8 * 8 + 2 * jj + 1] * scale);
                    *reinterpret_cast<uint4*>(dkr + c * 32 + q8 * 8) = u;
                }
            }
            tmem_ld32f(tdV + lane_off + c * 32, v);
            if (key < s) {
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8) {
                    uint4 u;
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        h2[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj], v[q8 * 8 + 2 * jj + 1]);
                    *reinterpret_cast<uint4*>(dvr + c * 32 + q8 * 8) = u;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// dQ: CTA owns 128 queries; loops over 64-key halves up to the diagonal.
template <int D>
__global__ void __launch_bounds__(384, 1)
    dq2_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_qkv64, const float* __restrict__ lse,
               const float* __restrict__ Dv, bf16* __restrict__ dqkv, int s, int a) {
    constexpr int TB = Tile<D>::BYTES;
    constexpr int HB = (D / 64) * HR * 128;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;
    uint8_t* sO = sQ + TB;
    uint8_t* sK = sO + TB;              // [2] half tiles
    uint8_t* sV = sK + 2 * HB;          // [2]
    uint8_t* sS = sV + 2 * HB;          // [2] dS [128 q][64 keys] (one atom)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sS + 2 * BR * 128);
    uint64_t* q_full = bar;
    uint64_t* kv_full = bar + 1;        // [2]
    uint64_t* kv_empty = bar + 3;       // [2]
    uint64_t* s_full = bar + 5;         // [2]
    uint64_t* p_full = bar + 7;
    uint64_t* g_done = bar + 8;         // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int qb = nqb - 1 - blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const int q0 = qb * BR;
    const int row0 = b * s;
    const int last_q = min(q0 + BR, s) - 1;
    const int nh = last_q / HR + 1;     // key halves 0 .. containing the last query

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        tma_prefetch_desc(&tm_do);
        tma_prefetch_desc(&tm_qkv64);
        mbar_init(q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&g_done[i], 1);
        }
        mbar_init(p_full, 256);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tdQ = tmem + 256;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(q_full, 2 * TB);
            tma_tile<D>(sQ, &tm_qkv, q_full, head * D, row0 + q0);
            tma_tile<D>(sO, &tm_do, q_full, head * D, row0 + q0);
            for (int hh = 0; hh < nh; ++hh) {
                const int sl = hh & 1;
                mbar_wait(&kv_empty[sl], ((hh >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&kv_full[sl], 2 * HB);
                tma_half<D>(sK + sl * HB, &tm_qkv64, &kv_full[sl], h + head * D, row0 + hh * HR);
                tma_half<D>(sV + sl * HB, &tm_qkv64, &kv_full[sl], 2 * h + head * D, row0 + hh * HR);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t iS = idesc(HR, false, false);   // M=128 q, N=64 keys
            const uint32_t iG = idesc(D, false, true);
            const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO);
            mbar_wait(q_full, 0);
            auto issue_s = [&](int hh) {
                const int sl = hh & 1;
                mbar_wait(&kv_full[sl], (hh >> 1) & 1);
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + sl * HB), aV = smem_u32(sV + sl * HB);
                const uint32_t tS = tmem + sl * 128, tP = tS + 64;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    umma_bf16(tS, desc_k(aQ, k), desc_k_h(aK, k), iS, k > 0);   // S = Q K^T
                    umma_bf16(tP, desc_k(aO, k), desc_k_h(aV, k), iS, k > 0);   // dP = dO V^T
                }
                umma_commit(&s_full[sl]);
            };
            issue_s(0);
            for (int hh = 0; hh < nh; ++hh) {
                const int sl = hh & 1;
                if (hh + 1 < nh) issue_s(hh + 1);
                mbar_wait(p_full, hh & 1);
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + sl * HB), aS = smem_u32(sS + sl * BR * 128);
#pragma unroll
                for (int k = 0; k < HR / 16; ++k)
                    umma_bf16(tdQ, desc_k(aS, k), desc_mn_h(aK, k), iG, (hh | k) > 0);   // dQ += dS K
                umma_commit(&g_done[sl]);
                umma_commit(&kv_empty[sl]);
            }
        }
    } else if (warp >= 4) {
        const int et = threadIdx.x - 128;
        const int r = et & 127, cg = et >> 7;
        const int q = q0 + r;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        const float* lseb = lse + ((long)b * a + head) * s;
        const float* Db = Dv + ((long)b * a + head) * s;
        const float L = q < s ? lseb[q] * LOG2E : 0.f;
        const float Dq = q < s ? Db[q] : 0.f;
        for (int hh = 0; hh < nh; ++hh) {
            const int sl = hh & 1;
            if (hh >= 2) mbar_wait(&g_done[sl], ((hh - 2) >> 1) & 1);   // dS buffer reuse
            mbar_wait(&s_full[sl], (hh >> 1) & 1);
            tc_fence_after();
            const uint32_t tS = tmem + sl * 128 + lane_off, tP = tS + 64;
            uint8_t* Sd = sS + sl * BR * 128;
            {
                const int c = cg;
                float sv[32], pv[32];
                tmem_ld32f(tS + c * 32, sv);
                tmem_ld32f(tP + c * 32, pv);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const int key = hh * HR + c * 32 + e;
                    const float p = (key <= q) ? exp2f(sv[e] * sc - L) : 0.f;
                    pv[e] = p * (pv[e] - Dq);
                }
                st_row32_h(Sd, r, c * 32, pv);
            }
            fence_async_smem();
            tc_fence_before();
            mbar_arrive(p_full);
        }
        mbar_wait(&g_done[(nh - 1) & 1], ((nh - 1) >> 1) & 1);
        tc_fence_after();
        const float scale = rsqrtf((float)D);
        bf16* dqr = dqkv + ((long)b * s + q) * (3L * h) + head * D;
#pragma unroll
        for (int c = cg * (D / 64); c < (cg + 1) * (D / 64); ++c) {
            float v[32];
            tmem_ld32f(tdQ + lane_off + c * 32, v);
            if (q < s) {
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8) {
                    uint4 u;
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        h2[jj] = __floats2bfloat162_rn(v[q8 * 8 + 2 * jj] * scale, v[q8 * 8 + 2 * jj + 1] * scale);
                    *reinterpret_cast<uint4*>(dqr + c * 32 + q8 * 8) = u;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// D[b,head,i] = sum_e dO O (fp32), one warp per row
__global__ void d_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout,
                         float* __restrict__ Dv, int s, int a, int d) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int head = blockIdx.y, b = blockIdx.z;
    if (i >= s) return;
    const long off = ((long)b * s + i) * a * d + head * d;
    float part = 0.f;
    for (int e = lane * 2; e < d; e += 64) {
        const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(o + off + e);
        const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(dout + off + e);
        part += __bfloat162float(x.x) * __bfloat162float(y.x) + __bfloat162float(x.y) * __bfloat162float(y.y);
    }
    part = warp_sum(part);
    if (lane == 0) Dv[((long)b * a + head) * s + i] = part;
}

}  // namespace fa5

// ---------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D bf16 map over [rows, cols] row-major (row stride ld elements), box {64, box_rows}
static int map2d(CUtensorMap* m, const void* base, long cols, long rows, long ld, int box_rows = 128) {
    auto enc = encode_fn();
    if (!enc) return -1;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? 0
               : -2;
}

template <int D>
static int fwd5(const void* qkv, void* o, float* lse, int b, int s, int a, cudaStream_t st) {
    constexpr int TB = fa5::Tile<D>::BYTES;
    constexpr int smem = 1024 + TB * 5 + 6 * 128 * 4 + 256;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(fa5::fwd2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    CUtensorMap m;
    if (map2d(&m, qkv, 3L * a * D, (long)b * s, 3L * a * D)) return -2;
    dim3 grid((s + 127) / 128, a, b);
    fa5::fwd2_kernel<D><<<grid, 384, smem, st>>>(m, (bf16*)o, lse, s, a);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <int D>
static int bwd5(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                float* ws, int b, int s, int a, cudaStream_t st) {
    constexpr int TB = fa5::Tile<D>::BYTES;
    constexpr int HB = (D / 64) * 64 * 128;
    constexpr int smem_kv = 1024 + 2 * TB + 4 * HB + 4 * 128 * 128 + 4 * 64 * 4 + 256;
    constexpr int smem_q = 1024 + 2 * TB + 4 * HB + 2 * 128 * 128 + 256;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(fa5::dkdv2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
        cudaFuncSetAttribute(fa5::dq2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
        attr = true;
    }
    CUtensorMap mq, mq64, md, md64;
    if (map2d(&mq, qkv, 3L * a * D, (long)b * s, 3L * a * D)) return -2;
    if (map2d(&mq64, qkv, 3L * a * D, (long)b * s, 3L * a * D, 64)) return -2;
    if (map2d(&md, dout, (long)a * D, (long)b * s, (long)a * D)) return -2;
    if (map2d(&md64, dout, (long)a * D, (long)b * s, (long)a * D, 64)) return -2;
    dim3 gd((s + 3) / 4, a, b);
    fa5::d_kernel<<<gd, 128, 0, st>>>((const bf16*)o, (const bf16*)dout, ws, s, a, D);
    dim3 grid((s + 127) / 128, a, b);
    fa5::dkdv2_kernel<D><<<grid, 384, smem_kv, st>>>(mq, mq64, md64, lse, ws, (bf16*)dqkv, s, a);
    fa5::dq2_kernel<D><<<grid, 384, smem_q, st>>>(mq, md, mq64, lse, ws, (bf16*)dqkv, s, a);
    note_launches(3);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int attn_fwd_tc5(const void* qkv, void* o, float* lse, int b, int s, int a, int d, cudaStream_t st) {
    return d == 64 ? fwd5<64>(qkv, o, lse, b, s, a, st) : fwd5<128>(qkv, o, lse, b, s, a, st);
}

int attn_bwd_tc5(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                 float* ws, int b, int s, int a, int d, cudaStream_t st) {
    return d == 64 ? bwd5<64>(qkv, o, dout, lse, dqkv, ws, b, s, a, st)
                   : bwd5<128>(qkv, o, dout, lse, dqkv, ws, b, s, a, st);
}

}  // namespace tpipe
