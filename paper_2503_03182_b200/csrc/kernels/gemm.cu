// Dense GEMMs for the stage executor.
//
//   C = A * B^T   A logical [M,K], B logical [N,K], fp32 accumulation,
//   fused epilogues (bias, residual, GELU, dGELU, fp32 main-grad accumulate).
//
// bf16: tcgen05.mma (kind::f16, M=128, N=BN, K=16) issued by one thread, A/B
// staged by TMA (128B swizzle) into a 4-6 stage mbarrier ring, fp32
// accumulators double-buffered in TMEM, 4 epilogue warps read TMEM with
// tcgen05.ld and apply the epilogue in registers. Persistent grid (<= #SMs).
// Both operands may be K-major or MN-major (fprop: K/K, dgrad: K/MN,
// wgrad: MN/MN), so no transposes are materialised.
//
// Two schedules were built, measured and removed (round 2): stream-K
// (K iterations split over CTAs with an ordered fp32 fix-up; 20-50% slower on
// the model shapes) and 256 x 512 pair tiles (one TMEM accumulator, exposed
// epilogue; profiles/r1_gemm_wide_ab.jsonl). DESIGN §9b has the numbers.
//
// fp32: exact-fp32 SIMT tiled kernel (parity mode).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tmap_cache.h"

namespace tpipe {

static int g_pdl = -1;   // -1: from TPIPE_PDL (default on)
bool pdl_enabled() {
    if (g_pdl < 0) {
        const char* e = getenv("TPIPE_PDL");
        g_pdl = (e && e[0] == '0') ? 0 : 1;
    }
    return g_pdl != 0;
}
void set_pdl(int on) { g_pdl = on != 0; }

// ============================================================== epilogue
template <typename T>
__device__ __forceinline__ void load32(const T* p, float (&o)[32]);
template <>
__device__ __forceinline__ void load32<bf16>(const bf16* p, float (&o)[32]) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint4 u = q[i];
        const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[i * 8 + j] = __bfloat162float(h[j]);
    }
}
template <>
__device__ __forceinline__ void load32<float>(const float* p, float (&o)[32]) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float4 u = q[i];
        o[4 * i] = u.x; o[4 * i + 1] = u.y; o[4 * i + 2] = u.z; o[4 * i + 3] = u.w;
    }
}

template <typename T>
__device__ __forceinline__ void store32(T* p, const float (&v)[32]);
template <>
__device__ __forceinline__ void store32<bf16>(bf16* p, const float (&v)[32]) {
    uint4* q = reinterpret_cast<uint4*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint4 u;
        bf16* h = reinterpret_cast<bf16*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = __float2bfloat16_rn(v[i * 8 + j]);
        q[i] = u;
    }
}
template <>
__device__ __forceinline__ void store32<float>(float* p, const float (&v)[32]) {
    float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}

// Apply the epilogue to 32 consecutive columns n0..n0+31 of row m (all in range).
template <typename T>
__device__ __forceinline__ void epi_chunk32(const GemmDesc& g, long m, long n0, float (&v)[32]) {
    const int epi = g.epi;
    if (epi == EPI_ACC_F32 || epi == EPI_STORE_F32) {
        float* C = reinterpret_cast<float*>(g.C) + m * g.ldc + n0;
        if (epi == EPI_ACC_F32) {
            float c[32];
            load32<float>(C, c);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = c[j] + v[j];
        }
        store32<float>(C, v);
        return;
    }
    if (epi == EPI_BIAS || epi == EPI_BIAS_RES || epi == EPI_BIAS_GELU) {
        float b[32];
        load32<T>(reinterpret_cast<const T*>(g.bias) + n0, b);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = v[j] + b[j];
    }
    if (epi == EPI_BIAS_RES) {
        float r[32];
        load32<T>(reinterpret_cast<const T*>(g.res) + m * g.ldr + n0, r);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = v[j] + r[j];
    }
    if (epi == EPI_BIAS_GELU) {
        float gg[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) gg[j] = gelu_tanh(rnd<T>(v[j]));
        store32<T>(reinterpret_cast<T*>(g.C2) + m * g.ldc2 + n0, gg);
    }
    if (epi == EPI_DGELU) {
        float u[32], gg[32];
        load32<T>(reinterpret_cast<const T*>(g.aux) + m * g.ldaux + n0, u);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            gg[j] = gelu_tanh(u[j]);
            v[j] = v[j] * gelu_tanh_grad(u[j]);
        }
        store32<T>(reinterpret_cast<T*>(g.C2) + m * g.ldc2 + n0, gg);
    }
    store32<T>(reinterpret_cast<T*>(g.C) + m * g.ldc + n0, v);
}

// ============================================================== SIMT (fp32 parity mode)
constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename T>
__device__ __forceinline__ float ldA(const GemmDesc& g, long m, long k) {
    const T* A = reinterpret_cast<const T*>(g.A);
    return to_f<T>(g.a_kmajor ? A[m * g.lda + k] : A[k * g.lda + m]);
}
template <typename T>
__device__ __forceinline__ float ldB(const GemmDesc& g, long n, long k) {
    const T* B = reinterpret_cast<const T*>(g.B);
    return to_f<T>(g.b_kmajor ? B[n * g.ldb + k] : B[k * g.ldb + n]);
}

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmDesc g) {
    __shared__ float As[SB_K][SB_M + 4];
    __shared__ float Bs[SB_K][SB_N + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const long m0 = (long)blockIdx.y * SB_M, n0 = (long)blockIdx.x * SB_N;
    float acc[4][4] = {};
    for (long k0 = 0; k0 < g.K; k0 += SB_K) {
        for (int e = threadIdx.x; e < SB_M * SB_K; e += 256) {
            // coalesce along the contiguous dimension of each operand
            int mm, kk;
            if (g.a_kmajor) { kk = e % SB_K; mm = e / SB_K; } else { mm = e % SB_M; kk = e / SB_M; }
            long gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < g.M && gk < g.K) ? ldA<T>(g, gm, gk) : 0.f;
            int nn, kb;
            if (g.b_kmajor) { kb = e % SB_K; nn = e / SB_K; } else { nn = e % SB_N; kb = e / SB_N; }
            long gn = n0 + nn, gk2 = k0 + kb;
            Bs[kb][nn] = (gn < g.N && gk2 < g.K) ? ldB<T>(g, gn, gk2) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < SB_K; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    // scalar epilogue
    for (int i = 0; i < 4; ++i) {
        long m = m0 + ty * 4 + i;
        if (m >= g.M) continue;
        for (int j = 0; j < 4; ++j) {
            long n = n0 + tx * 4 + j;
            if (n >= g.N) continue;
            float v = acc[i][j];
            switch (g.epi) {
                case EPI_ACC_F32: {
                    float* C = reinterpret_cast<float*>(g.C) + m * g.ldc + n;
                    *C = *C + v;
                    continue;
                }
                case EPI_STORE_F32:
                    reinterpret_cast<float*>(g.C)[m * g.ldc + n] = v;
                    continue;
                case EPI_BIAS:
                case EPI_BIAS_RES:
                case EPI_BIAS_GELU:
                    v = v + to_f<T>(reinterpret_cast<const T*>(g.bias)[n]);
                    if (g.epi == EPI_BIAS_RES)
                        v = v + to_f<T>(reinterpret_cast<const T*>(g.res)[m * g.ldr + n]);
                    if (g.epi == EPI_BIAS_GELU)
                        reinterpret_cast<T*>(g.C2)[m * g.ldc2 + n] = from_f<T>(gelu_tanh(rnd<T>(v)));
                    break;
                case EPI_DGELU: {
                    float u = to_f<T>(reinterpret_cast<const T*>(g.aux)[m * g.ldaux + n]);
                    reinterpret_cast<T*>(g.C2)[m * g.ldc2 + n] = from_f<T>(gelu_tanh(u));
                    v = v * gelu_tanh_grad(u);
                    break;
                }
                default:
                    break;
            }
            reinterpret_cast<T*>(g.C)[m * g.ldc + n] = from_f<T>(v);
        }
    }
}

int gemm_simt(int dtype, const GemmDesc& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return 0;
    dim3 grid((g.N + SB_N - 1) / SB_N, (g.M + SB_M - 1) / SB_M);
    if (dtype == DT_BF16)
        gemm_simt_kernel<bf16><<<grid, 256, 0, st>>>(g);
    else
        gemm_simt_kernel<float><<<grid, 256, 0, st>>>(g);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ============================================================== tcgen05 (bf16)
constexpr int TC_BM = 128, TC_BK = 64;

// Probe build only (libtpipe_gprobe.so, `make gprobe`, scripts/gemm_probe.py;
// never loaded by the product path): TPIPE_GEMM_PROBE bit 1 = the producer
// skips the TMA loads (operands are whatever the smem ring holds), bit 2 = the
// epilogue skips its math and stores -- which part of the pipeline bounds a shape.
#ifdef TPIPE_GEMM_PROBE
__constant__ int c_gemm_probe;
#define GEMM_PROBE c_gemm_probe
// SM-clock stamps of CTA 0's roles, [event][index] (scripts/gemm_probe.py --trace):
// 0 MMA: first MMA of k-block i issued, 1 MMA: full[] wait of k-block i done,
// 2 epilogue warp 4: tile i accumulator ready, 3 epilogue warp 4: tile i done,
// 4 producer: empty[] wait of k-block i done
constexpr int GTR_N = 1024;
__device__ unsigned long long* g_gtrace;
#define GTR(ev, idx)                                                                          \
    do {                                                                                      \
        if (g_gtrace && blockIdx.x == 0 && (idx) < GTR_N) g_gtrace[(ev) * GTR_N + (idx)] = clock64(); \
    } while (0)
// per-CTA stamps (index = blockIdx.x): 5 entry / 6 exit globaltimer (ns),
// 7 entry / 8 exit clock64, 9 first MMA issued (ns), 10 last tile epilogue done (ns)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define GTRB(ev, val)                                                      \
    do {                                                                   \
        if (g_gtrace && blockIdx.x < GTR_N) g_gtrace[(ev) * GTR_N + blockIdx.x] = (val); \
    } while (0)
#else
#define GTRB(ev, val) \
    do {              \
    } while (0)
#define GEMM_PROBE 0
#define GTR(ev, idx) \
    do {             \
    } while (0)
#endif
// EW = 8 epilogue warps (two warpgroups, warps 4..11) for the math-heavy
// epilogues (GELU, dGELU, residual): warp w reads TMEM lane quarter w % 4 and
// column half (w - 4) / 4 of every tile, so the fused math runs on 2 warps per
// scheduler and stays under the next tile's main loop (with 4 warps it was the
// critical path of the dGELU GEMM: 775 -> 1029 TFLOP/s). The light epilogues
// (store, bias, fp32 reduce-add) keep EW = 4.
__host__ __device__ constexpr int tc_threads(int ew) { return 128 + 32 * ew; }
static bool g_pair_enabled = true;
void gemm_set_pair(int on) { g_pair_enabled = on != 0; }
// CTA-pair tiles from this many 256 x 256 tiles on (measured crossover, see gemm_tc)
static int g_pair_min_tiles = 96;
void gemm_set_pair_min_tiles(int n) { g_pair_min_tiles = n > 0 ? n : 96; }
// 240 / 224-wide tiles where they fill the waves better (on by default; off =
// 256 only, for A/B runs)
static bool g_wide_choice = true;
void gemm_set_wide_choice(int on) { g_wide_choice = on != 0; }

// CG = 1: one CTA computes a 128 x BN tile. CG = 2: a CTA pair (cluster of 2
// on one TPC) computes a 256 x BN tile with tcgen05.mma.cta_group::2; each CTA
// stages 128 rows of A and BN/2 rows of B, so per-SM operand traffic (L2->smem
// and smem->tensor core) is 2/3 of the CG = 1, BN = 256 tile's.
// BN = 256, 240, 224 (or 128): 240 / 224-wide tiles make the tile count of
// the model's 2048 / 6144 / 8192-wide outputs fill the 74 CTA pairs (148 SMs)
// where 256-wide tiles leave 14% of every wave idle (gemm_tc's choice); their
// last 16 columns (BN = 240) are a half chunk stored without TMA.
template <int BN, int CG = 1, int EPI_WARPS = 4>
struct TcCfg {
    static_assert(BN <= 256 && BN % 16 == 0, "one tcgen05.mma covers N <= 256");
    static constexpr int BNC = BN / CG;                      // B rows (N) staged per CTA
    static constexpr int BNC64 = (BNC + 63) / 64 * 64;       // MN-major B: whole 64-column boxes
    // 2-deep staging ring per epilogue warp; pair tiles keep 6 operand stages
    // (a 4-deep ring for the two-output epilogues at the cost of a 6th stage
    // measured 1-2% slower on FC1 / FC2-dgrad, profiles/r2_gemm_ab_ring4.jsonl)
    static constexpr int NSTG = 2;
    static constexpr int STAGES = CG == 2 ? 6 : (BN > 128 ? 4 : 6);
    static_assert(1024 + STAGES * (TC_BM * TC_BK * 2 + ((BN / CG + 63) / 64 * 64) * TC_BK * 2) +
                          EPI_WARPS * NSTG * (EPI_WARPS == 8 ? 2048 : 4096) + 256 <= 232448,
                  "shared memory over the 227 KB per-CTA limit");
    static constexpr int A_BYTES = TC_BM * TC_BK * 2;
    static constexpr int B_BYTES = BNC64 * TC_BK * 2;         // smem per stage
    static constexpr int B_LOAD_K = BNC * TC_BK * 2;          // bytes one stage's TMA loads (K-major B)
    static constexpr int B_LOAD_MN = BNC64 * TC_BK * 2;       // (MN-major B)
    static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;   // double-buffered accumulators (pow2)
    static constexpr int NCHUNK = (BN + 31) / 32;             // 32-column epilogue chunks (last may be 16)
    // epilogue staging: EPI_WARPS warps x 2 buffers x one 32 x 32 chunk; the
    // 8-warp epilogues (GELU, dGELU, residual) only store bf16 (2 KB chunks),
    // so both variants fit the same operand ring depth
    static constexpr int STG_BUF = EPI_WARPS == 8 ? 2048 : 4096;
    static constexpr int STAGING = EPI_WARPS * NSTG * STG_BUF;
    static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + STAGING + 256;
};

// Global operands of one 32-column epilogue chunk (bias, residual / dGELU's
// u), loaded one chunk ahead so their latency hides under the previous
// chunk's math and stores (and, for the first chunk, under the wait for the
// accumulator): a chunk's loads issued on demand cost ~1-2K cycles
// (profiles/r2_gemm_trace_*.jsonl).
struct EpiPre {
    uint4 b[4];   // bias[n0 .. n0+31], bf16
    uint4 x[4];   // residual / aux row m, columns n0 .. n0+31, bf16
};

template <int EPI>
__device__ __forceinline__ void epi_prefetch(const GemmDesc& g, long m, long n0, bool row_ok, EpiPre& p,
                                             bool half) {
    constexpr int epi = EPI;
    if (epi == EPI_BIAS || epi == EPI_BIAS_RES || epi == EPI_BIAS_GELU) {
        const uint4* q = reinterpret_cast<const uint4*>(reinterpret_cast<const bf16*>(g.bias) + n0);
#pragma unroll
        for (int i = 0; i < 4; ++i) p.b[i] = (i < 2 || !half) ? __ldg(q + i) : make_uint4(0, 0, 0, 0);
    }
    if (epi == EPI_BIAS_RES || epi == EPI_DGELU || epi == EPI_STORE_DOT) {
        const bf16* src = epi == EPI_BIAS_RES ? reinterpret_cast<const bf16*>(g.res) + m * g.ldr
                                              : reinterpret_cast<const bf16*>(g.aux) + m * g.ldaux;
        const uint4* q = reinterpret_cast<const uint4*>(src + n0);
#pragma unroll
        for (int i = 0; i < 4; ++i) p.x[i] = (row_ok && (i < 2 || !half)) ? q[i] : make_uint4(0, 0, 0, 0);
    }
}

// Direct stores of NC columns n0 .. n0+NC-1 of row m by the thread that owns
// the row (no shared-memory staging): the 16-column half chunk of a BN = 240
// tile (in range: N and n0 are multiples of 16), and every chunk when the
// staging path is off. REDUCE: fp32 C += v with red.global.add (one add per
// element per launch, by its only owner: deterministic).
template <int NC, bool F32, bool REDUCE>
__device__ __forceinline__ void row_store(void* C, long ldc, long m, long n0, const float (&v)[32]) {
    if (F32) {
        float* q = reinterpret_cast<float*>(C) + m * ldc + n0;
#pragma unroll
        for (int i = 0; i < NC / 4; ++i) {
            if (REDUCE)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(q + 4 * i), "f"(v[4 * i]),
                             "f"(v[4 * i + 1]), "f"(v[4 * i + 2]), "f"(v[4 * i + 3])
                             : "memory");
            else
                reinterpret_cast<float4*>(q)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
    } else {
        uint4* q = reinterpret_cast<uint4*>(reinterpret_cast<bf16*>(C) + m * ldc + n0);
#pragma unroll
        for (int i = 0; i < NC / 8; ++i) {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
                w[j] = *reinterpret_cast<uint32_t*>(&h2);
            }
            q[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

// a bf16x2 word as an fp32 pair (exact)
__device__ __forceinline__ uint64_t bf2_to_f2(uint32_t w) {
    return pk2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// epilogue math on 32 columns (no stores); out2 for GELU/dGELU. Rows m >= M
// (TMA clips their stores) prefetched zeros. Packed fp32x2 ops throughout
// (the epilogue's FP issue was the larger part of its per-chunk time,
// profiles/r2_gemm_trace_*.jsonl; see gelu_fast2 on contraction).
template <int EPI>
__device__ __forceinline__ void epi_math(const EpiPre& p, float (&v)[32], float (&v2)[32]) {
    constexpr int epi = EPI;
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(p.b);
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(p.x);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        uint64_t x = pk2(v[2 * q], v[2 * q + 1]);
        if (epi == EPI_BIAS || epi == EPI_BIAS_RES || epi == EPI_BIAS_GELU) x = fadd2(x, bf2_to_f2(bw[q]));
        if (epi == EPI_BIAS_RES) x = fadd2(x, bf2_to_f2(xw[q]));
        if (epi == EPI_BIAS_GELU) {
            // GELU of the stored (bf16-rounded) pre-activation u
            float x0, x1;
            upk2(x, x0, x1);
            const __nv_bfloat162 u = __floats2bfloat162_rn(x0, x1);
            const uint64_t gg = gelu_fast2(bf2_to_f2(*reinterpret_cast<const uint32_t*>(&u)));
            upk2(gg, v2[2 * q], v2[2 * q + 1]);
        }
        if (epi == EPI_DGELU) {
            uint64_t gg, gd;
            gelu_fast_and_grad2(bf2_to_f2(xw[q]), gg, gd);
            upk2(gg, v2[2 * q], v2[2 * q + 1]);
            x = fmul2(x, gd);
        }
        upk2(x, v[2 * q], v[2 * q + 1]);
    }
}

__device__ __forceinline__ void tma_store_2d(const void* map, const void* smem, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(smem)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const void* map, const void* smem, int x, int y) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     map),
                 "r"(smem_u32(smem)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Stage one warp's 32 x 32 chunk (row = lane) in swizzled smem and issue one
// TMA store (or fp32 reduce-add) of the box at (n0, m0). NSTG: the warp's
// staging ring depth (the store that last used `buf` was NSTG stores ago).
template <int NSTG>
__device__ __forceinline__ void stage_store(uint8_t* buf, const float (&v)[32], bool f32, bool reduce,
                                            const CUtensorMap* map, int n0, int m0, int lane) {
    if (lane == 0) bulk_wait_read<NSTG - 1>();   // the store that last used `buf` has read it
    __syncwarp();
    const uint32_t sb = smem_u32(buf);
    if (f32) {   // 128 B rows, 128B swizzle: chunk q of row r at (q ^ (r & 7))
#pragma unroll
        for (int q = 0; q < 8; ++q)
            sts128(sb + lane * 128 + ((q ^ (lane & 7)) << 4), __float_as_uint(v[4 * q]),
                   __float_as_uint(v[4 * q + 1]), __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
    } else {     // 64 B rows, 64B swizzle: chunk q of row r at (q ^ ((r >> 1) & 3))
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
                w[j] = *reinterpret_cast<uint32_t*>(&h2);
            }
            sts128(sb + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4), w[0], w[1], w[2], w[3]);
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        if (reduce) tma_reduce_add_2d(map, buf, n0, m0);
        else tma_store_2d(map, buf, n0, m0);
        bulk_commit();
    }
}

// instruction descriptor: bf16 x bf16 -> f32, M=128*CG, N=BN, majors
template <int BN, bool A_MN, bool B_MN, int CG>
__device__ __forceinline__ uint32_t tc_idesc() {
    return (1u << 4)                     // D format f32
           | (1u << 7)                   // A bf16
           | (1u << 10)                  // B bf16
           | ((A_MN ? 1u : 0u) << 15)    // A major
           | ((B_MN ? 1u : 0u) << 16)    // B major
           | ((uint32_t)(BN >> 3) << 17) // N
           | ((uint32_t)((TC_BM * CG) >> 4) << 24);  // M
}

// Persistent data-parallel schedule: unit u (a CTA, or a CTA pair for CG = 2,
// whose CTAs walk the same tiles) takes tiles u, u + G, u + 2G, ...
struct TcSched {
    int num_tiles, tile, stride;
    __device__ void init(int nt, int cg = 1) {
        num_tiles = nt;
        tile = blockIdx.x / cg;
        stride = gridDim.x / cg;
    }
    __device__ bool next(int& t) {
        if (tile >= num_tiles) return false;
        t = tile;
        tile += stride;
        return true;
    }
};

// One kernel per epilogue kind (EPI): a kernel that carried every epilogue
// variant was 39-48 KB of SASS, over the 32 KB instruction cache, with the
// producer, MMA and epilogue loops far apart in it.
template <int BN, bool A_MN, bool B_MN, int CG, int EPI_WARPS, int EPI>
__global__ void __launch_bounds__(tc_threads(EPI_WARPS), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                   const GemmDesc g, int num_m, int num_n, int num_kb) {
    using Cfg = TcCfg<BN, CG, EPI_WARPS>;
    constexpr int STAGES = Cfg::STAGES;
    constexpr int TM = TC_BM * CG;        // tile rows
    constexpr int BNC = BN / CG;          // B rows staged per CTA
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
    uint8_t* stg = sB + STAGES * Cfg::B_BYTES;          // epilogue staging (1 KB aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::STAGING);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_tiles = num_m * num_n;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;   // 0 = pair leader (issues the MMAs)
    if (threadIdx.x == 0) {
        GTRB(5, gtimer());
        GTRB(7, clock64());
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmC);
        tma_prefetch_desc(&tmC2);
    }
    if (warp == 1 && lane == 0) {
        // CG = 2: the leader's full[] gets both CTAs' arrivals and TMA bytes;
        // empty[] / tfull[] of each CTA are signalled by the leader's multicast
        // commits; the leader's tempty[] gets one arrival per epilogue warp of
        // both CTAs.
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], CG);
            mbar_init(&empty[s], 1);
        }
        for (int e = 0; e < 2; ++e) {
            mbar_init(&tfull[e], 1);
            mbar_init(&tempty[e], CG == 2 ? 2 * EPI_WARPS : 32 * EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        if (CG == 2) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
        else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    }
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_trigger();

    if (warp == 0) {
        {   // ---------------- TMA producer (whole warp waits, the elected lane issues)
            int stage = 0;
            uint32_t phase = 0;
            TcSched sch;
            sch.init(num_tiles, CG);
            int tile;
            int gkb = 0;
            (void)gkb;
            while (sch.next(tile)) {
                const int mb = tile % num_m, nb = tile / num_m;
                const int am = mb * TM + rank * TC_BM;     // this CTA's A rows
                const int bn = nb * BN + rank * BNC;       // this CTA's B rows: [bn, bn + BNC)
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    GTR(4, gkb++);
                    uint8_t* a = sA + stage * Cfg::A_BYTES;
                    uint8_t* b = sB + stage * Cfg::B_BYTES;
                    if (!elect_one()) {
                    } else if (GEMM_PROBE & 1) {
                        if (CG == 1) mbar_arrive(&full[stage]);
                        else if (rank == 0) mbar_arrive(&full[stage]);
                        else mbar_arrive_cluster(mapa_shared(&full[stage], 0));
                    } else if (CG == 1) {
                        if (!A_MN) {
                            tma_load_2d(a, &tmA, &full[stage], kb * TC_BK, am);
                        } else {
#pragma unroll
                            for (int i = 0; i < TC_BM / 64; ++i)
                                tma_load_2d(a + i * 64 * TC_BK * 2, &tmA, &full[stage], am + i * 64, kb * TC_BK);
                        }
                        if (!B_MN) {
                            tma_load_2d(b, &tmB, &full[stage], kb * TC_BK, bn);
                        } else {
#pragma unroll
                            for (int i = 0; i < Cfg::BNC64 / 64; ++i)
                                tma_load_2d(b + i * 64 * TC_BK * 2, &tmB, &full[stage], bn + i * 64, kb * TC_BK);
                        }
                        mbar_arrive_expect_tx(&full[stage], Cfg::A_BYTES + (B_MN ? Cfg::B_LOAD_MN : Cfg::B_LOAD_K));
                    } else {
                        const uint32_t fb = mapa_shared(&full[stage], 0);   // leader's barrier
                        if (rank == 0)
                            mbar_arrive_expect_tx(&full[stage],
                                                  2 * (Cfg::A_BYTES + (B_MN ? Cfg::B_LOAD_MN : Cfg::B_LOAD_K)));
                        if (!A_MN) {
                            tma_load_2d_pair(a, &tmA, fb, kb * TC_BK, am);
                        } else {
#pragma unroll
                            for (int i = 0; i < TC_BM / 64; ++i)
                                tma_load_2d_pair(a + i * 64 * TC_BK * 2, &tmA, fb, am + i * 64, kb * TC_BK);
                        }
                        if (!B_MN) {
                            tma_load_2d_pair(b, &tmB, fb, kb * TC_BK, bn);
                        } else {
#pragma unroll
                            for (int i = 0; i < Cfg::BNC64 / 64; ++i)
                                tma_load_2d_pair(b + i * 64 * TC_BK * 2, &tmB, fb, bn + i * 64, kb * TC_BK);
                        }
                        if (rank != 0) mbar_arrive_cluster(fb);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ---------------- MMA issuer (whole warp of the pair leader; the elected lane issues)
            const uint32_t idesc = tc_idesc<BN, A_MN, B_MN, CG>();
            // descriptors of stage 0, k = 0; stage s / K-slice k are 64-bit adds
            // on the start-address field (addr >> 4; smem < 256 KB, no carry),
            // so the issuing loop between MMAs stays a few instructions long
            const uint64_t da0 = A_MN ? umma_desc_sw128(smem_u32(sA), TC_BK * 128, 1024)
                                      : umma_desc_sw128(smem_u32(sA), 0, 1024);
            const uint64_t db0 = B_MN ? umma_desc_sw128(smem_u32(sB), TC_BK * 128, 1024)
                                      : umma_desc_sw128(smem_u32(sB), 0, 1024);
            constexpr uint64_t DK_A = A_MN ? (2048 >> 4) : (32 >> 4), DK_B = B_MN ? (2048 >> 4) : (32 >> 4);
            // The elected lane runs the whole issue loop alone, and waits for
            // the next stage's operands between the last two MMAs of a k-block
            // (under the in-flight MMAs): UTCHMMA issue stalls while the tensor
            // pipe's short queue is full, so any instruction latency between
            // the last MMA of one k-block and the first of the next is a bubble
            // (scripts/microbench/mma_loop.cu, profiles/r2_gemm_probe_*.jsonl).
            if (elect_one()) {
                int stage = 0;
                uint32_t phase = 0;
                int it = 0;
                int gkb = 0;
                (void)gkb;
                TcSched sch;
                sch.init(num_tiles, CG);
                int tile;
                for (; sch.next(tile); ++it) {
                    const int acc = it & 1;
                    const uint32_t aph = (it >> 1) & 1;
                    mbar_wait(&tempty[acc], aph ^ 1);
                    mbar_wait(&full[stage], phase);
                    GTR(1, gkb);
                    tc_fence_after();
                    const uint32_t d = tmem_base + acc * BN;
                    for (int kb = 0; kb < num_kb; ++kb) {
                        const uint64_t das = da0 + (uint64_t)(stage * (Cfg::A_BYTES >> 4));
                        const uint64_t dbs = db0 + (uint64_t)(stage * (Cfg::B_BYTES >> 4));
                        const int nstage = stage + 1 == STAGES ? 0 : stage + 1;
                        const uint32_t nphase = stage + 1 == STAGES ? phase ^ 1 : phase;
#pragma unroll
                        for (int k = 0; k < TC_BK / 16; ++k) {
                            // K-major: 16 elements = 32 bytes inside the 128B swizzle atom row;
                            // MN-major: 16 K-rows of 128 B = 2048 bytes; MN atoms 8192 B apart.
                            if (k == TC_BK / 16 - 1 && kb + 1 < num_kb) {
                                mbar_wait(&full[nstage], nphase);
                                GTR(1, gkb + 1);
                                tc_fence_after();
                            }
                            const uint64_t da = das + k * DK_A;
                            const uint64_t db = dbs + k * DK_B;
                            const uint32_t accum = (kb != 0 || k != 0) ? 1u : 0u;
                            if (CG == 2) umma_bf16_pair(d, da, db, idesc, accum);
                            else umma_bf16(d, da, db, idesc, accum);
                            if (k == 0) GTR(0, gkb);
                            if (k == 0 && gkb == 0) GTRB(9, gtimer());
                        }
                        if (CG == 2) umma_commit_pair(&empty[stage], 3);
                        else umma_commit(&empty[stage]);
                        stage = nstage;
                        phase = nphase;
                        ++gkb;
                    }
                    if (CG == 2) umma_commit_pair(&tfull[acc], 3);
                    else umma_commit(&tfull[acc]);
                }
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> fused math -> swizzled smem -> TMA
        const int ew = warp & 3;             // TMEM lane quarter = tile rows [32ew, 32ew+32)
        const int chalf = (warp - 4) >> 2;   // column half of the tile
        uint8_t* mystg = stg + (warp - 4) * Cfg::NSTG * Cfg::STG_BUF;
        constexpr bool f32out = (EPI == EPI_ACC_F32 || EPI == EPI_STORE_F32);
        constexpr bool reduce = (EPI == EPI_ACC_F32);
        constexpr bool two = (EPI == EPI_BIAS_GELU || EPI == EPI_DGELU);
        int sb = 0;
        int it = 0;
        TcSched sch;
        sch.init(num_tiles, CG);
        const uint32_t tempty_leader = CG == 2 ? mapa_shared(&tempty[0], 0) : 0;
        // 32-column chunks per column group (two groups with 8 warps; BN = 224 / 240
        // split 4 + 3 / 4 + 3.5)
        constexpr int NCH0 = EPI_WARPS == 8 ? (Cfg::NCHUNK + 1) / 2 : Cfg::NCHUNK;
        const int c_lo = chalf * NCH0, c_hi = chalf ? Cfg::NCHUNK : NCH0;
        constexpr bool HAS_HALF = BN % 32 != 0;   // chunk NCHUNK - 1 is 16 columns wide
        int tile;
        for (; sch.next(tile); ++it) {
            const int mb = tile % num_m, nb = tile / num_m;
            const int acc = it & 1;
            const uint32_t aph = (it >> 1) & 1;
            const int m0 = mb * TM + rank * TC_BM + ew * 32;
            const long m = m0 + lane;
            const bool row_ok = m < g.M;
            // fused LM head + CE (K8): this thread owns row m of the tile
            constexpr bool lse_mode = EPI == EPI_LSE_PART, ce_mode = EPI == EPI_CE_GRAD;
            const bool pre = !lse_mode && !ce_mode && EPI != EPI_STORE && EPI != EPI_STORE_F32 &&
                             EPI != EPI_ACC_F32 && !(GEMM_PROBE & 8);
            EpiPre cur;
            if (GEMM_PROBE & 8) {
#pragma unroll
                for (int i = 0; i < 4; ++i) cur.b[i] = cur.x[i] = make_uint4(0, 0, 0, 0);
            }
            if (pre && nb * BN + c_lo * 32 < g.N)
                epi_prefetch<EPI>(g, m, nb * BN + c_lo * 32, row_ok, cur, HAS_HALF && c_lo == Cfg::NCHUNK - 1);
            int tgt = -1;
            float lse_m = 0.f, gmax = -INFINITY, gsum = 0.f;
            float dacc = 0.f;   // EPI_STORE_DOT
            if ((lse_mode || ce_mode) && row_ok) {
                tgt = g.targets[m];
                if (ce_mode) lse_m = g.lse[m];
            }
            mbar_wait(&tfull[acc], aph);
            if (warp == 4) GTR(2, it);
            tc_fence_after();
#pragma unroll 1
            for (int c = c_lo; c < c_hi; ++c) {
                uint32_t r[32];
                tmem_ld32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, r);
                const int n0 = nb * BN + c * 32;
                tmem_wait_ld();
                if (c + 1 == c_hi) {
                    // the tile's accumulator is in registers: release it to the MMA
                    // warp now, before the last chunk's math and stores
                    tc_fence_before();
                    if (CG == 2) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
                    } else {
                        mbar_arrive(&tempty[acc]);
                    }
                }
                if (warp == 4) GTR(11, it * 8 + (c - c_lo));
                if (n0 >= g.N || (GEMM_PROBE & 2)) continue;      // warp-uniform; TMA clips partial rows
                float v[32], v2[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                if (lse_mode) {
                    // online (max, sum exp) over the 64-column group, fp32 from
                    // the accumulators; the target logit captured in passing
                    float cm = v[0];
#pragma unroll
                    for (int j = 1; j < 32; ++j) cm = fmaxf(cm, v[j]);
                    if (cm > gmax) {
                        gsum *= exp2f((gmax - cm) * 1.4426950408889634f);
                        gmax = cm;
                    }
                    float zt = 0.f;
                    bool hit = false;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        gsum += exp2f((v[j] - gmax) * 1.4426950408889634f);
                        if (n0 + j == tgt) {
                            zt = v[j];
                            hit = true;
                        }
                    }
                    if (hit) g.zt[m] = zt;
                    if ((((n0 + 32) & 63) == 0 || n0 + 32 >= g.N)) {
                        if (row_ok)
                            reinterpret_cast<float2*>(g.part)[(size_t)m * ((g.N + 63) >> 6) + (n0 >> 6)] =
                                make_float2(gmax, gsum);
                        gmax = -INFINITY;
                        gsum = 0.f;
                    }
                    continue;
                }
                if (ce_mode) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        float pj = exp2f((v[j] - lse_m) * 1.4426950408889634f);
                        if (n0 + j == tgt) pj -= 1.f;
                        v[j] = pj * g.scale;
                    }
                } else {
                    epi_math<EPI>(cur, v, v2);
                    if (EPI == EPI_STORE_DOT) {
                        // D of (row m, head): the stored (bf16-rounded) dO times O, in
                        // column order; written when the head's last chunk is done
                        const uint32_t* xw = reinterpret_cast<const uint32_t*>(cur.x);
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const __nv_bfloat162 d2 = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
                            const float2 df = __bfloat1622float2(d2);
                            dacc = fmaf(df.x, __uint_as_float(xw[q] << 16), dacc);
                            dacc = fmaf(df.y, __uint_as_float(xw[q] & 0xffff0000u), dacc);
                        }
                        if ((n0 + 32) % g.dot_hd == 0) {
                            if (row_ok) {
                                const long bb = m / g.dot_s, qq = m % g.dot_s;
                                const int heads = g.N / g.dot_hd, head = (n0 + 32) / g.dot_hd - 1;
                                g.part[(bb * heads + head) * g.dot_s + qq] = dacc;
                            }
                            dacc = 0.f;
                        }
                    }
                    // next chunk's operands: in flight during this chunk's stores
                    // and the next TMEM load
                    if (pre && c + 1 < c_hi && n0 + 32 < g.N)
                        epi_prefetch<EPI>(g, m, n0 + 32, row_ok, cur, HAS_HALF && c + 1 == Cfg::NCHUNK - 1);
                }
                if (GEMM_PROBE & 4) {   // probe: math only, keep the result live
                    float x = 0.f;
#pragma unroll
                    for (int j = 0; j < 32; ++j) x += v[j] + v2[j];
                    if (x == 12345.f) g.zt[0] = x;
                    continue;
                }
                if (HAS_HALF && c == Cfg::NCHUNK - 1) {
                    // 16-column half chunk: direct stores of this thread's row
                    if (row_ok) {
                        row_store<16, f32out, reduce>(g.C, g.ldc, m, n0, v);
                        if (two) row_store<16, false, false>(g.C2, g.ldc2, m, n0, v2);
                    }
                    continue;
                }
                if (GEMM_PROBE & 16) {   // probe: direct row stores instead of smem staging + TMA
                    if (row_ok) {
                        row_store<32, f32out, reduce>(g.C, g.ldc, m, n0, v);
                        if (two) row_store<32, false, false>(g.C2, g.ldc2, m, n0, v2);
                    }
                    continue;
                }
                stage_store<Cfg::NSTG>(mystg + sb * Cfg::STG_BUF, v, f32out, reduce, &tmC, n0, m0, lane);
                sb = (sb + 1) & (Cfg::NSTG - 1);
                if (warp == 4) GTR(12, it * 8 + (c - c_lo));
                if (two) {
                    stage_store<Cfg::NSTG>(mystg + sb * Cfg::STG_BUF, v2, false, false, &tmC2, n0, m0, lane);
                    sb = (sb + 1) & (Cfg::NSTG - 1);
                }
                if (warp == 4) GTR(13, it * 8 + (c - c_lo));
            }
            if (warp == 4) GTR(3, it);
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
    if (warp == 4 && lane == 0) GTRB(10, gtimer());
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (threadIdx.x == 0) {
        GTRB(6, gtimer());
        GTRB(8, clock64());
    }
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
        else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                             &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D tensor map over a row-major [rows, cols] array with row stride ld
// (elements); box = {box_inner (cols), box_outer (rows)}.
static int make_map(CUtensorMap* map, const void* base, long cols, long rows, long ld, int box_inner,
                    int box_outer, bool f32 = false,
                    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto enc = get_encode();
    if (!enc) return -1;
    CUresult r = tmap_encode_2d_cached(enc, map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                       base, (uint64_t)cols, (uint64_t)rows, (uint64_t)(ld * (f32 ? 4 : 2)),
                                       (uint32_t)box_inner, (uint32_t)box_outer, sw);
    return r == CUDA_SUCCESS ? 0 : -2;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

template <int BN, bool A_MN, bool B_MN, int CG, int EPI_WARPS, int EPI>
static int launch_tc(const GemmDesc& g, cudaStream_t st) {
    using Cfg = TcCfg<BN, CG, EPI_WARPS>;
    constexpr int TC_THREADS = tc_threads(EPI_WARPS);
    constexpr int BNC = BN / CG;
    CUtensorMap ta, tb;
    int rc;
    if (!A_MN)
        rc = make_map(&ta, g.A, g.K, g.M, g.lda, TC_BK, TC_BM);
    else
        rc = make_map(&ta, g.A, g.M, g.K, g.lda, 64, TC_BK);
    if (rc) return rc;
    if (!B_MN)
        rc = make_map(&tb, g.B, g.K, g.N, g.ldb, TC_BK, BNC);
    else
        rc = make_map(&tb, g.B, g.N, g.K, g.ldb, 64, TC_BK);
    if (rc) return rc;
    // output maps: 32 x 32 boxes (fp32: 128 B rows, 128B swizzle; bf16: 64 B rows, 64B swizzle)
    CUtensorMap tc, tc2;
    const bool f32out = (g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32);
    if (g.epi == EPI_LSE_PART) {
        tc = ta;   // no C store: the map is never used
    } else {
        rc = make_map(&tc, g.C, g.N, g.M, g.ldc, 32, 32, f32out,
                      f32out ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
        if (rc) return rc;
    }
    if (g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU) {
        rc = make_map(&tc2, g.C2, g.N, g.M, g.ldc2, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
        if (rc) return rc;
    } else {
        tc2 = tc;
    }
    const int num_m = (g.M + TC_BM * CG - 1) / (TC_BM * CG);
    const int num_n = (g.N + BN - 1) / BN;
    const int num_kb = (g.K + TC_BK - 1) / TC_BK;
    const int tiles = num_m * num_n;
    const int units = num_sms() / CG;
    const int grid = CG * (tiles < units ? tiles : units);
    auto kern = gemm_tc_kernel<BN, A_MN, B_MN, CG, EPI_WARPS, EPI>;
    static PerDeviceOnce attr_set;
    if (attr_set.first()) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    }
#ifdef TPIPE_GEMM_PROBE
    static int probe_set = 0;   // once per process (one switch setting per run)
    if (!probe_set) {
        const char* e = getenv("TPIPE_GEMM_PROBE");
        const int v = e ? atoi(e) : 0;
        cudaMemcpyToSymbol(c_gemm_probe, &v, sizeof(int));
        probe_set = 1;
    }
#endif
    if (launch_k(kern, dim3(grid), dim3(TC_THREADS), Cfg::SMEM, st, CG, ta, tb, tc, tc2, g, num_m, num_n,
                 num_kb) != cudaSuccess)
        return -3;
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// 8 epilogue warps for the math-heavy epilogues (all store bf16 only: the
// 8-warp variant stages 2 KB chunks), 4 for the light ones
__host__ __device__ constexpr int epi_warps(int epi) {
    return (epi == EPI_BIAS_GELU || epi == EPI_DGELU || epi == EPI_BIAS_RES || epi == EPI_LSE_PART ||
            epi == EPI_CE_GRAD) ? 8 : 4;
}
template <int BN, int CG, int EPI>
static int launch_majors_epi(const GemmDesc& g, cudaStream_t st) {
    constexpr int EW = epi_warps(EPI);
    const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
    if (!amn && !bmn) return launch_tc<BN, false, false, CG, EW, EPI>(g, st);
    if (!amn && bmn) return launch_tc<BN, false, true, CG, EW, EPI>(g, st);
    if (amn && bmn) return launch_tc<BN, true, true, CG, EW, EPI>(g, st);
    return launch_tc<BN, true, false, CG, EW, EPI>(g, st);
}
template <int BN, int CG>
static int launch_majors(const GemmDesc& g, cudaStream_t st) {
    switch (g.epi) {
        case EPI_STORE: return launch_majors_epi<BN, CG, EPI_STORE>(g, st);
        case EPI_BIAS: return launch_majors_epi<BN, CG, EPI_BIAS>(g, st);
        case EPI_BIAS_RES: return launch_majors_epi<BN, CG, EPI_BIAS_RES>(g, st);
        case EPI_BIAS_GELU: return launch_majors_epi<BN, CG, EPI_BIAS_GELU>(g, st);
        case EPI_DGELU: return launch_majors_epi<BN, CG, EPI_DGELU>(g, st);
        case EPI_ACC_F32: return launch_majors_epi<BN, CG, EPI_ACC_F32>(g, st);
        case EPI_STORE_F32: return launch_majors_epi<BN, CG, EPI_STORE_F32>(g, st);
        // the fused head's 64-column LSE groups need each column group to be a
        // multiple of 64 wide (BN = 128 or 256; gemm_tc never picks 224 / 240)
        case EPI_LSE_PART:
            return BN % 128 == 0 ? launch_majors_epi<(BN % 128 == 0 ? BN : 256), CG, EPI_LSE_PART>(g, st) : -4;
        case EPI_CE_GRAD:
            return BN % 128 == 0 ? launch_majors_epi<(BN % 128 == 0 ? BN : 256), CG, EPI_CE_GRAD>(g, st) : -4;
        // a column group must hold whole heads (dot_hd <= 128)
        case EPI_STORE_DOT:
            return BN % 128 == 0 ? launch_majors_epi<(BN % 128 == 0 ? BN : 256), CG, EPI_STORE_DOT>(g, st) : -4;
        default: return -4;
    }
}

#ifdef TPIPE_GEMM_PROBE
extern "C" __attribute__((visibility("default"))) int tpipe_gemm_trace_set(void* buf) {
    return cudaMemcpyToSymbol(g_gtrace, &buf, sizeof(buf)) == cudaSuccess ? 0 : -1;
}
#endif

int gemm_tc(const GemmDesc& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return 0;
    if (g.K <= 0) return -4;
    // TMA: 16-byte aligned bases and row strides; 32-column epilogue chunks
    if ((g.epi == EPI_LSE_PART || g.epi == EPI_CE_GRAD) && (!g.targets || (g.epi == EPI_LSE_PART ? !g.part || !g.zt : !g.lse)))
        return -4;
    if (g.epi == EPI_STORE_DOT && (!g.aux || !g.part || g.dot_s <= 0 || (g.dot_hd != 64 && g.dot_hd != 128) ||
                                   g.N % g.dot_hd || g.M % g.dot_s || (g.ldaux % 8)))
        return -4;
    if ((g.N % 32) || (g.lda % 8) || (g.ldb % 8) || (g.epi != EPI_LSE_PART && (g.ldc % 8)) ||
        ((g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU) && (g.ldc2 % 8)))
        return -5;
    // CTA-pair 256 x 256 tiles: per SM they move 32 KB of operands per 64-deep
    // K block instead of 48 KB. Measured on the model shapes (profiles/
    // r1_gemm_modes.jsonl) they win once there are >= 96 pair tiles or the K
    // loop is long (>= 4096); a 2048 x 2048 x 2048 GEMM (64 pair tiles on 74
    // pairs) is faster as 128 single-CTA tiles.
    const long pair_tiles = (long)((g.M + 255) / 256) * ((g.N + 255) / 256);
    // tile width: the MMA time of a wave is ~ BN (tcgen05.mma runs at its N/2
    // cycles per K=16 step when fed, profiles/r2_mma_loop.jsonl), so pick the
    // width with the fewest waves x BN: e.g. N = 8192 on 74 pairs: 256-wide =
    // 4 waves of 256 (3.46 full), 224-wide = 296 tiles = 4 full waves of 224
    const bool head = g.epi == EPI_LSE_PART || g.epi == EPI_CE_GRAD || g.epi == EPI_STORE_DOT;
    auto width = [&](int rows, int units, int allow224) {
        const long mt = (g.M + rows - 1) / rows;
        int best = 256;
        long bestc = (mt * ((g.N + 255) / 256) + units - 1) / units * 256;
        // K-major B only (the forward GEMMs): an MN-major B tile of 112 / 120
        // columns per CTA starts off the 128-byte swizzle atoms and is loaded as
        // two 64-column boxes; measured 13-15% slower than 256-wide
        // (profiles/r2_gemm_ab_wide.jsonl), while the K-major widths gain 2-4%
        if (head || !g_wide_choice || !g.b_kmajor) return best;
        for (int bn : {240, 224}) {
            if (bn == 224 && !allow224) continue;
            const long c = (mt * ((g.N + bn - 1) / bn) + units - 1) / units * bn;
            if (c < bestc) {
                bestc = c;
                best = bn;
            }
        }
        return best;
    };
    if (g_pair_enabled && (pair_tiles >= g_pair_min_tiles || (pair_tiles >= 32 && g.K >= 4096))) {
        const int bn = width(256, num_sms() / 2, 1);
        if (bn == 224) return launch_majors<224, 2>(g, st);
        if (bn == 240) return launch_majors<240, 2>(g, st);
        return launch_majors<256, 2>(g, st);
    }
    const int num_m = (g.M + TC_BM - 1) / TC_BM;
    // N=128 tiles read 8 KB of operands per 64-cycle MMA (128 B/cycle, the
    // shared-memory limit); N=256 tiles need 96 B/cycle. Prefer 256 whenever
    // it still occupies >= ~65% of the SMs.
    // (a ragged last N tile is fine: TMA zero-fills, the epilogue masks n >= N)
    const bool wide = (long)num_m * ((g.N + 255) / 256) * 3 >= 2L * num_sms();
    if (wide) return width(128, num_sms(), 0) == 240 ? launch_majors<240, 1>(g, st) : launch_majors<256, 1>(g, st);
    return launch_majors<128, 1>(g, st);
}

int gemm(int dtype, const GemmDesc& g, cudaStream_t st) {
    if (dtype == DT_BF16) return gemm_tc(g, st);
    if (g.epi == EPI_STORE_DOT) return -4;   // tcgen05 path only
    return gemm_simt(DT_FP32, g, st);
}

}  // namespace tpipe
