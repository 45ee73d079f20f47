// Causal flash attention on 5th-generation tensor cores (tcgen05 + TMEM + TMA),
// bf16, head_dim 64 / 128 (FlashAttention is the paper's
// default). Persistent kernels: one CTA per SM loops over work items of
// 128 query rows (fwd, dQ) or 128 keys (dK/dV) of one (sequence, head), dealt
// heaviest first (causal work) in zigzag rounds.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one
// thread), warp 2 = TMEM allocator, warps 4..11 = 256 elementwise threads
// (two column groups; thread r of a group owns TMEM lane r = one query / key
// row) doing softmax / dS and the epilogues.
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
#include "tmap_cache.h"

namespace tpipe {
namespace fa5 {

constexpr int BR = 128;          // rows per tile (queries or keys)

// Timeline tracing for the probe build only (scripts/attn_trace.py compiles a
// separate library with -DTPIPE_ATTN_TRACE): SM clock stamps of CTA 0's role
// events, [event][index] with TR_N indices per event.
#ifdef TPIPE_ATTN_TRACE
constexpr int TR_N = 512;
__device__ unsigned long long* g_trace;
#define TR(ev, idx)                                                               \
    do {                                                                          \
        if (blockIdx.x == 0 && (idx) < TR_N) g_trace[(ev) * TR_N + (idx)] = clock64(); \
    } while (0)
#else
#define TR(ev, idx) \
    do {            \
    } while (0)
#endif
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


// ---- the single-instruction ex2 (MUFU.EX2; the .ftz flush only touches
// results below 2^-126); packed fp32x2 helpers (pk2, ffma2, ...) are in
// common.cuh. The elementwise warps of the backward kernels were issue-bound
// (~21 instructions per score); these cut it to ~4.
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x for a pair of x <= 8 on the FMA pipe (the forward softmax is bound by
// the MUFU pipe: 16 ex2 / clk / SM for 128 x 128 scores per tile; part of the
// exponentials go here instead). x = j + f, j = round(x) via the 1.5*2^23
// trick, f in [-0.5, 0.5]; 2^f by a degree-3 polynomial (relative-error fit,
// max 7.5e-5 — below bf16's 2^-9 rounding of P); 2^j added to the exponent
// bits (the magic's low 9 bits are zero, so bits(t) << 23 == j << 23).
// x is clamped at -125 (result ~2^-125 instead of 0: negligible against the
// row sum >= 1; only off-diagonal tiles, where no score is masked, use it).
__device__ __forceinline__ void ex2_poly2(uint64_t x2, float& p0, float& p1) {
    float a, b;
    upk2(x2, a, b);
    const uint64_t xc = pk2(fmaxf(a, -125.f), fmaxf(b, -125.f));
    const uint64_t t = fadd2(xc, pk2(12582912.f, 12582912.f));
    const uint64_t jf = fadd2(t, pk2(-12582912.f, -12582912.f));
    const uint64_t f = ffma2(jf, pk2(-1.f, -1.f), xc);
    uint64_t q = ffma2(f, pk2(0.0551716611f, 0.0551716611f), pk2(0.242611155f, 0.242611155f));
    q = ffma2(q, f, pk2(0.693260968f, 0.693260968f));
    q = ffma2(q, f, pk2(0.999928057f, 0.999928057f));
    float t0, t1, q0, q1;
    upk2(t, t0, t1);
    upk2(q, q0, q1);
    p0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
    p1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
}
// pairs (of the 32 per thread per tile) whose exponentials use ex2_poly2
#ifndef FWD_POLY_OF_16
#define FWD_POLY_OF_16 4
#endif
__device__ __forceinline__ uint32_t bf2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
// write 16 packed bf16x2 words (cols col0..col0+31, col0 < 64) of row r of a one-atom tile
__device__ __forceinline__ void st_row32_pk(uint8_t* tile, int r, int col0, const uint32_t (&w)[16]) {
    const int c0 = col0 >> 3;
    const uint32_t base = smem_u32(tile);
#pragma unroll
    for (int q = 0; q < 4; ++q) sts128(base + swz(r, c0 + q), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

// 32 lanes x 16 columns store (thread t writes lane base+t)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
// smem -> TMEM copy of one K-step (16 bf16 = 256 bits per row) of a 128-row
// operand tile, described by its MMA shared-memory descriptor: row i lands in
// lane i, 8 columns — the A-operand layout of a TS tcgen05.mma. Issued by the
// MMA thread: tcgen05.cp and tcgen05.mma execute in issue order.
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// ---------------------------------------------------------------- persistent schedule
// grid = min(items, SMs); items are numbered heaviest first (causal work falls
// with the item index) and dealt to CTAs in zigzag rounds: round r gives item
// r*G + c (r even) or r*G + G-1-c (r odd) to CTA c — a static LPT-style
// assignment, so every output row still has exactly one owner.
__device__ __forceinline__ int sched_item(int k, int T) {
    const int G = gridDim.x, c = blockIdx.x;
    const int t = k * G + ((k & 1) ? (G - 1 - c) : c);
    return t < T ? t : -1;
}

// ============================================================== forward (persistent)
// S double-buffered in TMEM (columns [0,128) and [128,256)); P_j is written
// back over S_j as packed bf16 (64 columns) and consumed as the TMEM
// A-operand of O += P_j V_j; O (D columns at 256) accumulates in TMEM and is
// rescaled in place by the row threads when the running max moves. The
// item's Q is copied into TMEM (columns [384, 384 + D/2), tcgen05.cp) and is
// the TMEM A operand of S = Q K^T: both MMAs read only K or V from shared
// memory (an SS MMA is bound by the tensor core's ~64 B/clk shared-memory
// operand path: profiles/r2_mma_rate.jsonl).
// All rings (K/V stages, S buffers, P/PV handshakes) run on a global tile
// counter g that continues across this CTA's items, so the S MMA of an item's
// first tile overlaps the previous item's last softmax and epilogue; Q is
// double-buffered per item in shared memory.
//   MMA  : S_0 | for g: [S_{g+1}] [PV_g once P_g ready] — S_{g+1} overwrites
//          P_{g-1}, read by PV_{g-1} issued before it (tcgen05.mma runs in
//          issue order), so no wait for PV_{g-1} to finish
//   rows : S_g -> P_g (one pass, 64 scores per thread in registers) -> wait PV_{g-1}
//          -> O *= corr_g (skipped per warp when corr == 1) -> P_g ready
// Item t (heaviest first): qb = nqb-1 - t/(a*nb), head = t%a, batch = (t/a)%nb.
// NG column groups of 4 softmax warps each (row r = TMEM lane; fwd5 uses 2).
template <int D, int NG>
__global__ void __launch_bounds__(128 + 128 * NG, 1)
    fwd2_kernel(const __grid_constant__ CUtensorMap tm_qkv, bf16* __restrict__ o,
                float* __restrict__ lse, int s, int a, int nb) {
    constexpr int SC = BR / NG;          // scores per softmax thread per tile
    constexpr int OC = D / NG / 32;      // 32-column O chunks per group
    constexpr int TB = Tile<D>::BYTES;
    constexpr int STAGES = 2;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm;                        // [2]
    uint8_t* sK = sQ + 2 * TB;               // [STAGES]
    uint8_t* sV = sK + STAGES * TB;          // [STAGES]
    float* sMax = reinterpret_cast<float*>(sV + STAGES * TB);   // [2 iters][NG groups][128]
    float* sSum = sMax + 2 * NG * BR;                             // [NG groups][128]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sSum + NG * BR);
    uint64_t* q_full = bar;                  // [2]
    uint64_t* q_empty = bar + 2;             // [2]
    // K and V stages have their own barriers: K_{g+2} is fetched once S_g has
    // read K_g, a whole softmax earlier than PV_g releases V_g
    uint64_t* k_full = bar + 4;              // [STAGES]
    uint64_t* k_empty = k_full + STAGES;     // [STAGES]
    uint64_t* v_full = k_empty + STAGES;     // [STAGES]
    uint64_t* v_empty = v_full + STAGES;     // [STAGES]
    uint64_t* s_full = v_empty + STAGES;     // [2] S buffer ready
    uint64_t* p_full = s_full + 2;           // P_g in TMEM + O corrected (256 arrivals)
    uint64_t* pv_done = p_full + 1;          // PV_g complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int T = nqb * a * nb;
    const int h = a * D;
    auto decode = [&](int t, int& qb, int& head, int& b) {
        qb = nqb - 1 - t / (a * nb);
        const int rem = t % (a * nb);
        head = rem % a;
        b = rem / a;
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&s_full[i], 1);
        }
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
        }
        mbar_init(p_full, 128 * NG);
        mbar_init(pv_done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();
    const uint32_t tO = tmem + 256, tQ = tmem + 384;

    if (warp == 0) {
        {   // whole warp waits; the elected lane issues the TMA loads
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = sched_item(k, T);
                if (t < 0) break;
                int qb, head, b;
                decode(t, qb, head, b);
                const int sl = k & 1;
                mbar_wait(&q_empty[sl], ((k >> 1) & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&q_full[sl], TB);
                    tma_tile<D>(sQ + sl * TB, &tm_qkv, &q_full[sl], head * D, b * s + qb * BR);
                }
                __syncwarp();
                for (int j = 0; j <= qb; ++j, ++g) {
                    const int st = g % STAGES;
                    const uint32_t ph = ((g / STAGES) & 1) ^ 1;
                    mbar_wait(&k_empty[st], ph);
                    if (lane == 0) TR(0, g);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&k_full[st], TB);
                        tma_tile<D>(sK + st * TB, &tm_qkv, &k_full[st], h + head * D, b * s + j * BR);
                    }
                    __syncwarp();
                    mbar_wait(&v_empty[st], ph);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&v_full[st], TB);
                        tma_tile<D>(sV + st * TB, &tm_qkv, &v_full[st], 2 * h + head * D, b * s + j * BR);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: loop state stays warp-uniform, the elected lane issues
            const uint32_t iS = idesc(BR, false, false);
            const uint32_t iO = idesc(D, false, true);
            // S-issue cursor: item k_s (tiles 0..qb_s), tile j_s, global index gs
            int k_s = 0, j_s = 0, nkb_s = 0, gs = 0;
            bool have_s;
            {
                const int t = sched_item(0, T);
                have_s = t >= 0;
                if (have_s) nkb_s = nqb - t / (a * nb);
            }
            auto issue_s = [&]() {
                const int sl = k_s & 1;
                if (j_s == 0) {
                    // the item's Q -> TMEM, after the previous item's S MMAs (issue order)
                    mbar_wait(&q_full[sl], (k_s >> 1) & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t aQ = smem_u32(sQ + sl * TB);
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) tmem_cp_128x256b(tQ + kk * 8, desc_k(aQ, kk));
                        umma_commit(&q_empty[sl]);   // smem Q free once copied
                    }
                    __syncwarp();
                }
                const int st = gs % STAGES;
                mbar_wait(&k_full[st], (gs / STAGES) & 1);
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + st * TB);
                const uint32_t tS = tmem + (gs & 1) * 128;
                if (lane == 0) TR(1, gs);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) umma_bf16_ts(tS, tQ + kk * 8, desc_k(aK, kk), iS, kk > 0);
                    umma_commit(&s_full[gs & 1]);
                    umma_commit(&k_empty[st]);
                }
                __syncwarp();
                ++gs;
                if (++j_s == nkb_s) {
                    j_s = 0;
                    const int t = sched_item(++k_s, T);
                    have_s = t >= 0;
                    if (have_s) nkb_s = nqb - t / (a * nb);
                }
            };
            if (have_s) issue_s();
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = sched_item(k, T);
                if (t < 0) break;
                const int nkb = nqb - t / (a * nb);
                for (int j = 0; j < nkb; ++j, ++g) {
                    if (have_s) issue_s();   // S buffer (g+1)&1 held P_{g-1}: PV_{g-1} was issued first
                    mbar_wait(p_full, g & 1);
                    const int st = g % STAGES;
                    mbar_wait(&v_full[st], (g / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t aV = smem_u32(sV + st * TB);
                    const uint32_t tP = tmem + (g & 1) * 128;
                    if (lane == 0) TR(2, g);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < BR / 16; ++kk)
                            umma_bf16_ts(tO, tP + kk * 8, desc_mn(aV, kk), iO, (j | kk) > 0);
                        umma_commit(pv_done);
                        umma_commit(&v_empty[st]);
                    }
                    __syncwarp();
                }
            }
        }
#ifdef TPIPE_ATTN_TRACE
    } else if (warp == 3 || warp == 2) {
        // trace build only: observers stamping when S_g (warp 3) / PV_g (warp 2)
        // complete on the tensor pipe, independent of the softmax warps
        int g = 0;
        for (int k = 0;; ++k) {
            const int t = sched_item(k, T);
            if (t < 0) break;
            const int nkb = nqb - t / (a * nb);
            for (int j = 0; j < nkb; ++j, ++g) {
                if (warp == 3) {
                    mbar_wait(&s_full[g & 1], (g >> 1) & 1);
                    if (lane == 0) TR(24, g);
                } else {
                    mbar_wait(pv_done, g & 1);
                    if (lane == 0) TR(25, g);
                }
            }
        }
#endif
    } else if (warp >= 4) {
        // 4 NG softmax warps: row r = TMEM lane (warp % 4 = lane quarter); column
        // group cg owns scores [SC cg, SC (cg+1)) and O columns [cg D/NG, (cg+1) D/NG)
        const int et = threadIdx.x - 128;
        const int r = et & 127, cg = et >> 7;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        int g = 0;
        for (int k = 0;; ++k) {
            const int t = sched_item(k, T);
            if (t < 0) break;
            int qb, head, b;
            decode(t, qb, head, b);
            const int nkb = qb + 1;
            const int q = qb * BR + r;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < nkb; ++j, ++g) {
                const uint32_t tS = tmem + (g & 1) * 128 + lane_off;
                mbar_wait(&s_full[g & 1], (g >> 1) & 1);
                if (threadIdx.x == 128) TR(3, g);
                tc_fence_after();
                float sv[SC];
#pragma unroll
                for (int hh = 0; hh < SC / 32; ++hh) {
                    uint32_t ra[32];
                    tmem_ld32(tS + cg * SC + hh * 32, ra);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) sv[hh * 32 + e] = __uint_as_float(ra[e]);
                }
                if (j == nkb - 1) {   // diagonal tile: keys after the query are masked
                    const int k0 = j * BR + cg * SC;
#pragma unroll
                    for (int e = 0; e < SC; ++e)
                        if (k0 + e > q) sv[e] = -INFINITY;
                }
                // running max in scaled units: max(s) * sc == max(s * sc) (sc > 0)
                float lmx = -INFINITY;
#pragma unroll
                for (int e = 0; e < SC; e += 2) lmx = fmax3(lmx, sv[e], sv[e + 1]);
                lmx *= sc;
                float* mb = sMax + (g & 1) * NG * BR;
                mb[cg * BR + r] = lmx;
                if (threadIdx.x == 128) TR(4, g);
                named_bar_sync(1, 128 * NG);
                // lazy rescaling: the reference max moves only when a score exceeds
                // it by more than 2^8 (P <= 256 is exact enough in bf16 and the sums
                // are fp32), so O is rarely rescaled; every column group sees the
                // same values and takes the same decision
                float mnew = m;
#pragma unroll
                for (int c2 = 0; c2 < NG; ++c2) mnew = fmaxf(mnew, mb[c2 * BR + r]);
                const float mx = mnew - m > 8.0f ? mnew : m;
                const uint64_t sc2 = pk2(sc, sc), nm2 = pk2(-mx, -mx);
                uint64_t rs2 = pk2(0.f, 0.f);
                uint32_t pk[SC / 2];
                if (j < nkb - 1) {   // no masked score: part of the exponentials on the FMA pipe
#pragma unroll
                    for (int e = 0; e < SC; e += 2) {
                        const uint64_t x2 = ffma2(pk2(sv[e], sv[e + 1]), sc2, nm2);
                        float p0, p1;
                        if (((e >> 1) & 15) < FWD_POLY_OF_16) {
                            ex2_poly2(x2, p0, p1);
                        } else {
                            float x0, x1;
                            upk2(x2, x0, x1);
                            p0 = ex2(x0);
                            p1 = ex2(x1);
                        }
                        rs2 = fadd2(rs2, pk2(p0, p1));
                        pk[e / 2] = bf2(p0, p1);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < SC; e += 2) {
                        float x0, x1;
                        upk2(ffma2(pk2(sv[e], sv[e + 1]), sc2, nm2), x0, x1);
                        const float p0 = ex2(x0), p1 = ex2(x1);
                        rs2 = fadd2(rs2, pk2(p0, p1));
                        pk[e / 2] = bf2(p0, p1);
                    }
                }
                float rs0, rs1;
                upk2(rs2, rs0, rs1);
                const float rs = rs0 + rs1;
                const float corr = ex2(m - mx);
                l = l * corr + rs;        // partial (this group's columns), same m history
                m = mx;
                // P_g over S_g: packed cols [SC/2 cg, SC/2 (cg+1)) (every group's S
                // was loaded before the barrier above)
                if constexpr (SC == 64) tmem_st32(tS + cg * 32, pk);
                else tmem_st16(tS + cg * 16, pk);
                if (threadIdx.x == 128) TR(5, g);
                if (j > 0) {
                    mbar_wait(pv_done, (g - 1) & 1);
                    tc_fence_after();
                    if (__any_sync(0xffffffffu, corr != 1.0f)) {
#pragma unroll
                        for (int c = cg * OC; c < (cg + 1) * OC; ++c) {
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
                if (threadIdx.x == 128) TR(6, g);
                if (threadIdx.x == 127 + 128 * NG) TR(7, g);
                mbar_arrive(p_full);
            }
            sSum[cg * BR + r] = l;
            named_bar_sync(1, 128 * NG);
            l = 0.f;   // every group adds the NG partial sums in the same order
#pragma unroll
            for (int c2 = 0; c2 < NG; ++c2) l += sSum[c2 * BR + r];
            mbar_wait(pv_done, (g - 1) & 1);
            tc_fence_after();
            // tcgen05.ld is .sync.aligned: every lane loads; only valid rows store
            const float inv = 1.0f / l;
            bf16* orow = o + ((long)b * s + q) * h + head * D;
#pragma unroll
            for (int c = cg * OC; c < (cg + 1) * OC; ++c) {
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
            // the next item's sSum write is ordered after the other groups' reads
            // above by the named barrier of its first tile
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

// operand ring depths of the backward kernels: the Q/dO (dK/dV kernel) or
// K/V (dQ kernel) half tile of step g+2 is loaded while step g's dV/dK (dQ)
// MMAs still read their slot, so the TMA latency is off the MMA issue chain
// (with 2 slots every half paid one L2 round trip). Sized to the 227 KB limit.
template <int D>
struct BwdCfg {
    static constexpr int NQ = D == 128 ? 5 : 6;
    static constexpr int NK = D == 128 ? 5 : 6;
};

// dK/dV (persistent): an item is 128 keys of one (sequence, head); it loops
// over 64-query halves from the diagonal. Item t (heaviest first):
// kb = t/(a*nb), head = t%a, batch = (t/a)%nb. Half rings (Q/dO halves, S/dP
// TMEM buffers) run on a global half counter across items; K/V are
// single-buffered per item and released after the item's last S MMA. P^T and
// dS^T are written back over S^T / dP^T in TMEM (bf16, each column group
// inside its own columns) and feed dV += P^T dO, dK += dS^T Q as TMEM A
// operands: no shared-memory round trip (the kernel was shared-memory
// bandwidth bound, profiles/r2_attn_trace.txt).
template <int D>
__global__ void __launch_bounds__(384, 1)
    dkdv2_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_qkv64,
                 const __grid_constant__ CUtensorMap tm_do64, const float* __restrict__ lse,
                 const float* __restrict__ Dv, bf16* __restrict__ dqkv, int s, int a, int nb) {
    constexpr int TB = Tile<D>::BYTES;          // 128-row tile
    constexpr int HB = (D / 64) * HR * 128;      // 64-row tile
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    constexpr int NQ = BwdCfg<D>::NQ;            // Q/dO half-tile ring depth
    uint8_t* sK = sm;
    uint8_t* sV = sK + TB;
    uint8_t* sQ = sV + TB;                 // [NQ] half tiles
    uint8_t* sO = sQ + NQ * HB;            // [NQ] dO half tiles
    float* sL = reinterpret_cast<float*>(sO + NQ * HB);        // [2][64]
    float* sD = sL + 2 * HR;                                   // [2][64]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sD + 2 * HR);
    uint64_t* kv_full = bar;
    uint64_t* kv_empty = bar + 1;
    uint64_t* q_full = bar + 2;          // [NQ]
    uint64_t* q_empty = q_full + NQ;     // [NQ]
    uint64_t* s_full = q_empty + NQ;     // [2]
    uint64_t* p_full = s_full + 2;       // [2] 256 arrivals per half (by g & 1: a fast warp may be one half ahead)
    uint64_t* g_done = p_full + 2;       // [2] dV/dK MMAs of a half complete
    uint64_t* ld_full = g_done + 2;      // [2] sL/sD of a half staged (warp 3)
    uint64_t* ld_empty = ld_full + 2;    // [2] sL/sD of a half consumed (256 arrivals)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ld_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = (s + BR - 1) / BR;
    const int nq64 = (s + HR - 1) / HR;
    const int T = nkb * a * nb;
    const int h = a * D;
    auto decode = [&](int t, int& kb, int& head, int& b) {
        kb = t / (a * nb);
        const int rem = t % (a * nb);
        head = rem % a;
        b = rem / a;
    };
    auto halves = [&](int t) { return nq64 - 2 * (t / (a * nb)); };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        tma_prefetch_desc(&tm_qkv64);
        tma_prefetch_desc(&tm_do64);
        mbar_init(kv_full, 1);
        mbar_init(kv_empty, 1);
        for (int i = 0; i < NQ; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&g_done[i], 1);
            mbar_init(&ld_full[i], 32);
            mbar_init(&ld_empty[i], 256);
        }
        mbar_init(&p_full[0], 256);
        mbar_init(&p_full[1], 256);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();
    const uint32_t tdV = tmem + 256, tdK = tmem + 256 + D;   // D <= 128

    if (warp == 0) {
        {   // whole warp waits; the elected lane issues the TMA loads
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = sched_item(k, T);
                if (t < 0) break;
                int kb, head, b;
                decode(t, kb, head, b);
                const int row0 = b * s;
                mbar_wait(kv_empty, (k & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(kv_full, 2 * TB);
                    tma_tile<D>(sK, &tm_qkv, kv_full, h + head * D, row0 + kb * BR);
                    tma_tile<D>(sV, &tm_qkv, kv_full, 2 * h + head * D, row0 + kb * BR);
                }
                __syncwarp();
                const int nh = halves(t);
                for (int hh = 0; hh < nh; ++hh, ++g) {
                    const int sl = g % NQ;
                    mbar_wait(&q_empty[sl], ((g / NQ) & 1) ^ 1);
                    if (lane == 0) TR(8, g);
                    const int qrow = row0 + (2 * kb + hh) * HR;
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&q_full[sl], 2 * HB);
                        tma_half<D>(sQ + sl * HB, &tm_qkv64, &q_full[sl], head * D, qrow);
                        tma_half<D>(sO + sl * HB, &tm_do64, &q_full[sl], head * D, qrow);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp; the elected lane issues
            const uint32_t iS = idesc(HR, false, false);   // M=128 keys, N=64 queries
            const uint32_t iG = idesc(D, false, true);
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
            int k_s = 0, h_s = 0, nh_s = 0, gs = 0;
            bool have_s;
            {
                const int t = sched_item(0, T);
                have_s = t >= 0;
                if (have_s) nh_s = halves(t);
            }
            auto issue_s = [&]() {
                const int sl = gs % NQ;
                if (h_s == 0) mbar_wait(kv_full, k_s & 1);
                mbar_wait(&q_full[sl], (gs / NQ) & 1);
                tc_fence_after();
                const uint32_t aQ = smem_u32(sQ + sl * HB), aO = smem_u32(sO + sl * HB);
                const uint32_t tS = tmem + (gs & 1) * 128, tP = tS + 64;
                if (lane == 0) TR(9, gs);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        umma_bf16(tS, desc_k(aK, kk), desc_k_h(aQ, kk), iS, kk > 0);   // S^T = K Q^T
                        umma_bf16(tP, desc_k(aV, kk), desc_k_h(aO, kk), iS, kk > 0);   // dP^T = V dO^T
                    }
                    umma_commit(&s_full[gs & 1]);
                    if (h_s == nh_s - 1) umma_commit(kv_empty);   // K, V of this item consumed
                }
                __syncwarp();
                ++gs;
                if (++h_s == nh_s) {
                    h_s = 0;
                    const int t = sched_item(++k_s, T);
                    have_s = t >= 0;
                    if (have_s) nh_s = halves(t);
                }
            };
            if (have_s) issue_s();
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = sched_item(k, T);
                if (t < 0) break;
                const int nh = halves(t);
                for (int hh = 0; hh < nh; ++hh, ++g) {
                    const int sl = g & 1;
                    if (have_s) issue_s();   // TMEM buffer (g+1)&1 freed by p_full(g-1)
                    mbar_wait(&p_full[g & 1], (g >> 1) & 1);
                    tc_fence_after();
                    const int qs = g % NQ;
                    const uint32_t aQ = smem_u32(sQ + qs * HB), aO = smem_u32(sO + qs * HB);
                    const uint32_t tPt = tmem + sl * 128, tSt = tPt + 64;   // P^T, dS^T (packed)
                    if (lane == 0) TR(10, g);
                    if (elect_one()) {
                        // queries [32c, 32c+32) of a half sit packed in columns [32c, 32c+16)
#pragma unroll
                        for (int kk = 0; kk < HR / 16; ++kk) {
                            const uint32_t ca = (kk >> 1) * 32 + (kk & 1) * 8;
                            umma_bf16_ts(tdV, tPt + ca, desc_mn_h(aO, kk), iG, (hh | kk) > 0);  // dV += P^T dO
                            umma_bf16_ts(tdK, tSt + ca, desc_mn_h(aQ, kk), iG, (hh | kk) > 0);  // dK += dS^T Q
                        }
                        umma_commit(&g_done[sl]);
                        umma_commit(&q_empty[qs]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 3) {
        // lse / D of each 64-query half, negated and pre-scaled, staged one half
        // ahead so the elementwise warps never wait on a global load
        int g = 0;
        for (int k = 0;; ++k) {
            const int t = sched_item(k, T);
            if (t < 0) break;
            int kb, head, b;
            decode(t, kb, head, b);
            const int nh = halves(t);
            const float* lseb = lse + ((long)b * a + head) * s;
            const float* Db = Dv + ((long)b * a + head) * s;
            for (int hh = 0; hh < nh; ++hh, ++g) {
                const int sl = g & 1;
                const int q0 = (2 * kb + hh) * HR;
                mbar_wait(&ld_empty[sl], ((g >> 1) & 1) ^ 1);
#pragma unroll
                for (int i = lane; i < HR; i += 32) {
                    const int qq = q0 + i;
                    sL[sl * HR + i] = qq < s ? -lseb[qq] * LOG2E : 0.f;
                    sD[sl * HR + i] = qq < s ? -Db[qq] : 0.f;
                }
                mbar_arrive(&ld_full[sl]);
            }
        }
    } else if (warp >= 4) {
        // 8 elementwise warps: row r = TMEM lane (warp % 4 selects the lane quarter),
        // column group cg = which 32 of the 64 half-columns this thread owns
        const int et = threadIdx.x - 128;
        const int r = et & 127, cg = et >> 7;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        const float scale = rsqrtf((float)D);
        int g = 0;
        for (int k = 0;; ++k) {
            const int t = sched_item(k, T);
            if (t < 0) break;
            int kb, head, b;
            decode(t, kb, head, b);
            const int nh = halves(t);
            const int key = kb * BR + r;
            for (int hh = 0; hh < nh; ++hh, ++g) {
                const int sl = g & 1;
                const int q0 = (2 * kb + hh) * HR;
                // (TMEM buffer `sl`'s P^T / dS^T of half g-2 were read by dV / dK
                // MMAs issued before S_g: tcgen05.mma executes in issue order)
                mbar_wait(&ld_full[sl], (g >> 1) & 1);
                if (threadIdx.x == 128) TR(11, g);
                mbar_wait(&s_full[sl], (g >> 1) & 1);
                if (threadIdx.x == 128) TR(12, g);
                tc_fence_after();
                const uint32_t tS = tmem + sl * 128 + lane_off, tP = tS + 64;
                const float* L = sL + sl * HR;
                const float* Dq = sD + sl * HR;
                {
                    const int c = cg;
                    uint32_t sr[32], pr[32];
                    tmem_ld32(tS + c * 32, sr);
                    tmem_ld32(tP + c * 32, pr);
                    tmem_wait_ld();
                    // P^T = exp2(S^T sc - L_q); every key of the block precedes every
                    // query of this column group except on the diagonal halves
                    if (threadIdx.x == 128) TR(13, g);
                    const int qc = q0 + c * 32;
                    const bool full = qc >= kb * BR + BR - 1 && qc + 32 <= s;
                    const uint64_t sc2 = pk2(sc, sc);
                    const uint32_t nL = smem_u32(L + c * 32);
                    const uint32_t nD = smem_u32(Dq + c * 32);
                    float p[32];
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const uint64_t x2 = ffma2(pk2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sc2,
                                                  lds64(nL + 4 * e));
                        float x0, x1;
                        upk2(x2, x0, x1);
                        p[e] = ex2(x0);
                        p[e + 1] = ex2(x1);
                    }
                    if (!full) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const int qq = qc + e;
                            if (!(qq >= key && qq < s)) p[e] = 0.f;
                        }
                    }
                    uint32_t wp[16], wd[16];
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const uint64_t p2 = pk2(p[e], p[e + 1]);
                        const uint64_t d2 = fmul2(p2, fadd2(pk2(__uint_as_float(pr[e]), __uint_as_float(pr[e + 1])),
                                                            lds64(nD + 4 * e)));
                        float d0, d1;
                        upk2(d2, d0, d1);
                        wp[e / 2] = bf2(p[e], p[e + 1]);
                        wd[e / 2] = bf2(d0, d1);
                    }
                    tmem_st16(tS + c * 32, wp);   // P^T over this group's own S^T columns
                    tmem_st16(tP + c * 32, wd);   // dS^T over its own dP^T columns
                }
                mbar_arrive(&ld_empty[sl]);
                tmem_wait_st();
                tc_fence_before();
                if (threadIdx.x == 128) TR(14, g);
                if (threadIdx.x == 383) TR(15, g);
                mbar_arrive(&p_full[sl]);
            }
            mbar_wait(&g_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
            tc_fence_after();
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
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// dQ (persistent): an item is 128 queries of one (sequence, head); it loops
// over 64-key halves up to the diagonal. Item t (heaviest first):
// qb = nqb-1 - t/(a*nb). Shared memory holds only the streamed operands: the
// item's Q / dO tiles are copied once into TMEM (tcgen05.cp, the A operands
// of the S and dP MMAs) and dS is written back over S in TMEM (the A operand
// of dQ += dS K), so per 64-key half the tensor core reads just the K and V
// halves from shared memory (profiles/r2_attn_trace.txt: the smem-operand
// version was shared-memory-bandwidth bound). TMEM: S/dP [2 buffers x 128],
// dQ [128], Q [64], dO [64] columns.
template <int D>
__global__ void __launch_bounds__(384, 1)
    dq2_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_qkv64, const float* __restrict__ lse,
               const float* __restrict__ Dv, bf16* __restrict__ dqkv, int s, int a, int nb) {
    constexpr int TB = Tile<D>::BYTES;
    constexpr int HB = (D / 64) * HR * 128;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    constexpr int NK = BwdCfg<D>::NK;   // K/V half-tile ring depth
    uint8_t* sQ = sm;
    uint8_t* sO = sQ + TB;
    uint8_t* sK = sO + TB;              // [NK] half tiles
    uint8_t* sV = sK + NK * HB;         // [NK]
    uint64_t* bar = reinterpret_cast<uint64_t*>(sV + NK * HB);
    uint64_t* q_full = bar;
    uint64_t* q_empty = bar + 1;
    uint64_t* kv_full = bar + 2;          // [NK]
    uint64_t* kv_empty = kv_full + NK;    // [NK]
    uint64_t* s_full = kv_empty + NK;     // [2]
    uint64_t* p_full = s_full + 2;        // [2] by g & 1 (a fast warp may be one half ahead)
    uint64_t* g_done = p_full + 2;        // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(g_done + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nqb = (s + BR - 1) / BR;
    const int T = nqb * a * nb;
    const int h = a * D;
    auto decode = [&](int t, int& qb, int& head, int& b) {
        qb = nqb - 1 - t / (a * nb);
        const int rem = t % (a * nb);
        head = rem % a;
        b = rem / a;
    };
    auto halves = [&](int t) {   // key halves 0 .. the one holding the item's last query
        const int qb = nqb - 1 - t / (a * nb);
        return (min(qb * BR + BR, s) - 1) / HR + 1;
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tm_qkv);
        tma_prefetch_desc(&tm_do);
        tma_prefetch_desc(&tm_qkv64);
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < NK; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&g_done[i], 1);
        }
        mbar_init(&p_full[0], 256);
        mbar_init(&p_full[1], 256);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();
    const uint32_t tdQ = tmem + 256, tQ = tmem + 384, tdO = tmem + 448;

    if (warp == 0) {
        {   // whole warp waits; the elected lane issues the TMA loads
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = sched_item(k, T);
                if (t < 0) break;
                int qb, head, b;
                decode(t, qb, head, b);
                const int row0 = b * s;
                mbar_wait(q_empty, (k & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full, 2 * TB);
                    tma_tile<D>(sQ, &tm_qkv, q_full, head * D, row0 + qb * BR);
                    tma_tile<D>(sO, &tm_do, q_full, head * D, row0 + qb * BR);
                }
                __syncwarp();
                const int nh = halves(t);
                for (int hh = 0; hh < nh; ++hh, ++g) {
                    const int sl = g % NK;
                    mbar_wait(&kv_empty[sl], ((g / NK) & 1) ^ 1);
                    if (lane == 0) TR(16, g);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&kv_full[sl], 2 * HB);
                        tma_half<D>(sK + sl * HB, &tm_qkv64, &kv_full[sl], h + head * D, row0 + hh * HR);
                        tma_half<D>(sV + sl * HB, &tm_qkv64, &kv_full[sl], 2 * h + head * D, row0 + hh * HR);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp; the elected lane issues
            const uint32_t iS = idesc(HR, false, false);   // M=128 q, N=64 keys
            const uint32_t iG = idesc(D, false, true);
            const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO);
            int k_s = 0, h_s = 0, nh_s = 0, gs = 0;
            bool have_s;
            {
                const int t = sched_item(0, T);
                have_s = t >= 0;
                if (have_s) nh_s = halves(t);
            }
            auto issue_s = [&]() {
                const int sl = gs % NK;
                if (h_s == 0) {
                    // the item's Q, dO -> TMEM (after the previous item's last S / dP
                    // MMAs read the old copies: tcgen05.cp and .mma run in issue order)
                    mbar_wait(q_full, k_s & 1);
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            tmem_cp_128x256b(tQ + kk * 8, desc_k(aQ, kk));
                            tmem_cp_128x256b(tdO + kk * 8, desc_k(aO, kk));
                        }
                        umma_commit(q_empty);   // smem Q, dO free once copied
                    }
                    __syncwarp();
                }
                mbar_wait(&kv_full[sl], (gs / NK) & 1);
                tc_fence_after();
                const uint32_t aK = smem_u32(sK + sl * HB), aV = smem_u32(sV + sl * HB);
                const uint32_t tS = tmem + (gs & 1) * 128, tP = tS + 64;
                if (lane == 0) TR(17, gs);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        umma_bf16_ts(tS, tQ + kk * 8, desc_k_h(aK, kk), iS, kk > 0);    // S = Q K^T
                        umma_bf16_ts(tP, tdO + kk * 8, desc_k_h(aV, kk), iS, kk > 0);   // dP = dO V^T
                    }
                    umma_commit(&s_full[gs & 1]);
                }
                __syncwarp();
                ++gs;
                if (++h_s == nh_s) {
                    h_s = 0;
                    const int t = sched_item(++k_s, T);
                    have_s = t >= 0;
                    if (have_s) nh_s = halves(t);
                }
            };
            if (have_s) issue_s();
            int g = 0;
            for (int k = 0;; ++k) {
                const int t = sched_item(k, T);
                if (t < 0) break;
                const int nh = halves(t);
                for (int hh = 0; hh < nh; ++hh, ++g) {
                    const int sl = g & 1;
                    if (have_s) issue_s();
                    mbar_wait(&p_full[g & 1], (g >> 1) & 1);
                    tc_fence_after();
                    const int ks = g % NK;
                    const uint32_t aK = smem_u32(sK + ks * HB), tdS = tmem + sl * 128;
                    if (lane == 0) TR(18, g);
                    if (elect_one()) {
                        // dS of keys [32c, 32c+32) sits packed in columns [32c, 32c+16)
#pragma unroll
                        for (int kk = 0; kk < HR / 16; ++kk)
                            umma_bf16_ts(tdQ, tdS + (kk >> 1) * 32 + (kk & 1) * 8, desc_mn_h(aK, kk), iG,
                                         (hh | kk) > 0);   // dQ += dS K
                        umma_commit(&g_done[sl]);
                        umma_commit(&kv_empty[ks]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp >= 4) {
        const int et = threadIdx.x - 128;
        const int r = et & 127, cg = et >> 7;
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const float sc = rsqrtf((float)D) * LOG2E;
        const float scale = rsqrtf((float)D);
        int g = 0;
        for (int k = 0;; ++k) {
            const int t = sched_item(k, T);
            if (t < 0) break;
            int qb, head, b;
            decode(t, qb, head, b);
            const int nh = halves(t);
            const int q = qb * BR + r;
            const float* lseb = lse + ((long)b * a + head) * s;
            const float* Db = Dv + ((long)b * a + head) * s;
            const float L = q < s ? lseb[q] * LOG2E : 0.f;
            const float Dq = q < s ? Db[q] : 0.f;
            for (int hh = 0; hh < nh; ++hh, ++g) {
                const int sl = g & 1;
                // (the S buffer's dS of half g-2 was read by dQ MMAs issued before S_g)
                if (threadIdx.x == 128) TR(19, g);
                mbar_wait(&s_full[sl], (g >> 1) & 1);
                if (threadIdx.x == 128) TR(20, g);
                tc_fence_after();
                const uint32_t tS = tmem + sl * 128 + lane_off, tP = tS + 64;
                {
                    const int c = cg;
                    uint32_t sr[32], pr[32];
                    tmem_ld32(tS + c * 32, sr);
                    tmem_ld32(tP + c * 32, pr);
                    tmem_wait_ld();
                    if (threadIdx.x == 128) TR(21, g);
                    const int kc = hh * HR + c * 32;
                    const bool full = kc + 31 <= qb * BR;   // below the diagonal for every row
                    const uint64_t sc2 = pk2(sc, sc), nl2 = pk2(-L, -L), nd2 = pk2(-Dq, -Dq);
                    float p[32];
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const uint64_t x2 =
                            ffma2(pk2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sc2, nl2);
                        float x0, x1;
                        upk2(x2, x0, x1);
                        p[e] = ex2(x0);
                        p[e + 1] = ex2(x1);
                    }
                    if (!full) {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (kc + e > q) p[e] = 0.f;
                    }
                    uint32_t wd[16];
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const uint64_t d2 = fmul2(pk2(p[e], p[e + 1]),
                                                  fadd2(pk2(__uint_as_float(pr[e]), __uint_as_float(pr[e + 1])), nd2));
                        float d0, d1;
                        upk2(d2, d0, d1);
                        wd[e / 2] = bf2(d0, d1);
                    }
                    tmem_st16(tS + c * 32, wd);   // dS over this group's own S columns
                }
                tmem_wait_st();
                tc_fence_before();
                if (threadIdx.x == 128) TR(22, g);
                if (threadIdx.x == 383) TR(23, g);
                mbar_arrive(&p_full[sl]);
            }
            mbar_wait(&g_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
            tc_fence_after();
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
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// D[b,head,i] = sum_e dO O (fp32), one warp per row
// D[b,head,q] = sum_e dO O (fp32). One 16-byte chunk of O and of dO per
// thread (TPR = d/8 threads per (token, head) row, rows ordered token-major so
// a warp reads contiguous memory), reduced over the row's lanes by shuffles.
template <int TPR>
__global__ void __launch_bounds__(256) d_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout,
                                                float* __restrict__ Dv, int s, int a, long rows) {
    const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long row = gt / TPR;   // = (b*s + q)*a + head
    pdl_wait();
    pdl_trigger();
    float part = 0.f;
    if (row < rows) {
        const long off = gt * 8;   // row * (TPR*8) + chunk*8
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(o + off));
        const uint4 y = __ldg(reinterpret_cast<const uint4*>(dout + off));
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&x);
        const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 xf = __bfloat1622float2(xh[j]), yf = __bfloat1622float2(yh[j]);
            part = fmaf(xf.x, yf.x, part);
            part = fmaf(xf.y, yf.y, part);
        }
    }
#pragma unroll
    for (int w = TPR / 2; w > 0; w >>= 1) part += __shfl_xor_sync(0xffffffffu, part, w);
    if (row < rows && (threadIdx.x % TPR) == 0) {
        const long tok = row / a;
        const int head = (int)(row % a);
        const long b = tok / s, q = tok % s;
        Dv[(b * a + head) * s + q] = part;
    }
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
    return tmap_encode_2d_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, (uint64_t)cols, (uint64_t)rows,
                                 (uint64_t)(ld * 2), 64u, (uint32_t)box_rows, CU_TENSOR_MAP_SWIZZLE_128B) ==
                   CUDA_SUCCESS
               ? 0
               : -2;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static int persistent_grid(int items) { return items < num_sms() ? items : num_sms(); }

template <int D>
static int fwd5(const void* qkv, void* o, float* lse, int b, int s, int a, cudaStream_t st) {
    // softmax column groups: 4 (16 softmax warps, 32 scores per thread) measured
    // 3% slower than 2 at D = 128 (profiles/r2_attn_fwd_ng.jsonl)
    constexpr int NG = 2;
    constexpr int TB = fa5::Tile<D>::BYTES;
    constexpr int smem = 1024 + TB * 6 + 3 * NG * 128 * 4 + 256;
    static_assert(smem <= 232448, "forward smem over the 227 KB limit");
    static PerDeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(fa5::fwd2_kernel<D, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    CUtensorMap m;
    if (map2d(&m, qkv, 3L * a * D, (long)b * s, 3L * a * D)) return -2;
    const int grid = persistent_grid(((s + 127) / 128) * a * b);
    if (launch_k(fa5::fwd2_kernel<D, NG>, dim3(grid), dim3(128 + 128 * NG), smem, st, 1, m, (bf16*)o, lse, s, a,
                 b) != cudaSuccess)
        return -3;
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <int D>
static int bwd5(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                float* ws, int b, int s, int a, cudaStream_t st, bool have_d) {
    constexpr int TB = fa5::Tile<D>::BYTES;
    constexpr int HB = (D / 64) * 64 * 128;
    constexpr int smem_kv = 1024 + 2 * TB + 2 * fa5::BwdCfg<D>::NQ * HB + 4 * 64 * 4 + 256;
    constexpr int smem_q = 1024 + 2 * TB + 2 * fa5::BwdCfg<D>::NK * HB + 256;
    static_assert(smem_kv <= 232448 && smem_q <= 232448, "backward smem over the 227 KB limit");
    static PerDeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(fa5::dkdv2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
        cudaFuncSetAttribute(fa5::dq2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
    }
    CUtensorMap mq, mq64, md, md64;
    if (map2d(&mq, qkv, 3L * a * D, (long)b * s, 3L * a * D)) return -2;
    if (map2d(&mq64, qkv, 3L * a * D, (long)b * s, 3L * a * D, 64)) return -2;
    if (map2d(&md, dout, (long)a * D, (long)b * s, (long)a * D)) return -2;
    if (map2d(&md64, dout, (long)a * D, (long)b * s, (long)a * D, 64)) return -2;
    const long drows = (long)b * s * a;
    const unsigned dblocks = (unsigned)((drows * (D / 8) + 255) / 256);
    if (!have_d && launch_k(fa5::d_kernel<D / 8>, dim3(dblocks), dim3(256), 0, st, 1, (const bf16*)o,
                            (const bf16*)dout, ws, s, a, drows) != cudaSuccess)
        return -3;
    const int grid = persistent_grid(((s + 127) / 128) * a * b);
    if (launch_k(fa5::dkdv2_kernel<D>, dim3(grid), dim3(384), smem_kv, st, 1, mq, mq64, md64, lse,
                 (const float*)ws, (bf16*)dqkv, s, a, b) != cudaSuccess)
        return -3;
    if (launch_k(fa5::dq2_kernel<D>, dim3(grid), dim3(384), smem_q, st, 1, mq, md, mq64, lse, (const float*)ws,
                 (bf16*)dqkv, s, a, b) != cudaSuccess)
        return -3;
    note_launches(have_d ? 2 : 3);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

#ifdef TPIPE_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) int tpipe_attn_trace_set(void* buf) {
    return cudaMemcpyToSymbol(fa5::g_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -1;
}
#endif

int attn_fwd_tc5(const void* qkv, void* o, float* lse, int b, int s, int a, int d, cudaStream_t st) {
    return d == 64 ? fwd5<64>(qkv, o, lse, b, s, a, st) : fwd5<128>(qkv, o, lse, b, s, a, st);
}

int attn_bwd_tc5(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                 float* ws, int b, int s, int a, int d, cudaStream_t st, bool have_d) {
    return d == 64 ? bwd5<64>(qkv, o, dout, lse, dqkv, ws, b, s, a, st, have_d)
                   : bwd5<128>(qkv, o, dout, lse, dqkv, ws, b, s, a, st, have_d);
}

}  // namespace tpipe
