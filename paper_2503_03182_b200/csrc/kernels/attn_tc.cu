// Causal flash attention, bf16 tensor-core path (
// FlashAttention is the paper's default).
//
// mma.sync m16n8k16 (bf16 -> fp32) with ldmatrix from XOR-swizzled shared
// memory and cp.async double buffering; online softmax in the exp2 domain.
//   forward : CTA = 128 query rows (8 warps x 16), loops over 64-key blocks up
//             to the diagonal; saves O and the row LSE only.
//   backward: deterministic, no atomics —
//             dK/dV kernel: CTA owns 64 keys, loops over 64-query blocks,
//               S^T = K Q^T, P^T from LSE, dV += P^T dO, dP^T = V dO^T,
//               dS^T = P^T (dP^T - D), dK += dS^T Q;
//             dQ kernel: CTA owns 64 queries, loops over key blocks,
//               dQ += dS K.
// head_dim 64 or 128. (The tcgen05/TMEM attention is the next step; this is
// the first tensor-core path.)
#include "common.cuh"
#include "kernels.h"

namespace tpipe {

namespace fa {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const int bytes = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Tile of R rows x D bf16 in smem, rows of D*2 bytes, 16-byte chunks XOR-swizzled
// by (row % 8). Element (r, k) with k a multiple of 8 -> chunk address.
template <int D>
__device__ __forceinline__ bf16* tile_ptr(bf16* base, int r, int k) {
    const int chunk = (k >> 3) ^ (r & 7);
    return base + r * D + chunk * 8;
}

// async copy of `rows` rows (row stride ld elements) into a swizzled tile;
// rows beyond `valid` are zero-filled.
template <int D, int ROWS, int NT>
__device__ __forceinline__ void load_tile(bf16* sm, const bf16* g, long ld, int valid) {
    constexpr int CH = D / 8;  // 16-byte chunks per row
    for (int e = threadIdx.x; e < ROWS * CH; e += NT) {
        const int r = e / CH, c = e % CH;
        const bool ok = r < valid;
        const bf16* src = g + (long)(ok ? r : 0) * ld + c * 8;
        cp_async16(tile_ptr<D>(sm, r, c * 8), src, ok);
    }
}

constexpr float LOG2E = 1.4426950408889634f;

// ----------------------------------------------------------------------- forward
template <int D>
__global__ void __launch_bounds__(256) fwd_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ o,
                                                  float* __restrict__ lse, int s, int a) {
    constexpr int BM = 128, BN = 64, NT = 256;
    extern __shared__ __align__(128) uint8_t smraw[];
    bf16* sQ = reinterpret_cast<bf16*>(smraw);
    bf16* sK = sQ + BM * D;          // 2 stages
    bf16* sV = sK + 2 * BN * D;      // 2 stages
    const int nqb = (s + BM - 1) / BM;
    const int qb = nqb - 1 - blockIdx.x;   // heaviest first
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const long ld = 3L * h;
    const bf16* base = qkv + (long)b * s * ld;
    const int q0 = qb * BM;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const float sc = rsqrtf((float)D) * LOG2E;

    load_tile<D, BM, NT>(sQ, base + (long)q0 * ld + head * D, ld, s - q0);
    const int nkb = (q0 + BM + BN - 1) / BN < (s + BN - 1) / BN ? (q0 + BM + BN - 1) / BN : (s + BN - 1) / BN;
    load_tile<D, BN, NT>(sK, base + h + head * D, ld, s);
    load_tile<D, BN, NT>(sV, base + 2 * h + head * D, ld, s);
    cp_async_commit();

    float oacc[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const int wr0 = q0 + warp * 16;  // first query row of this warp

    for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb & 1;
        if (kb + 1 < nkb) {
            const int k0n = (kb + 1) * BN;
            load_tile<D, BN, NT>(sK + (st ^ 1) * BN * D, base + (long)k0n * ld + h + head * D, ld, s - k0n);
            load_tile<D, BN, NT>(sV + (st ^ 1) * BN * D, base + (long)k0n * ld + 2 * h + head * D, ld, s - k0n);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int k0 = kb * BN;
        if (k0 <= wr0 + 15) {  // warp has unmasked keys in this block
            bf16* K = sK + st * BN * D;
            bf16* V = sV + st * BN * D;
            float sacc[BN / 8][4];
#pragma unroll
            for (int j = 0; j < BN / 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint32_t af[4];
                ldsm_x4(af, tile_ptr<D>(sQ, warp * 16 + (lane & 15), kk * 16 + (lane >> 4) * 8));
#pragma unroll
                for (int jp = 0; jp < BN / 16; ++jp) {
                    uint32_t bfr[4];
                    ldsm_x4(bfr, tile_ptr<D>(K, jp * 16 + (lane & 7) + (lane >> 4) * 8,
                                             kk * 16 + ((lane >> 3) & 1) * 8));
                    mma16816(sacc[2 * jp], af, bfr[0], bfr[1]);
                    mma16816(sacc[2 * jp + 1], af, bfr[2], bfr[3]);
                }
            }
            // scale, causal mask, online softmax (rows g and g+8 of the warp tile)
            float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
            for (int j = 0; j < BN / 8; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int qrow = wr0 + g + (e >> 1) * 8;
                    const int key = k0 + j * 8 + 2 * t + (e & 1);
                    float v = sacc[j][e] * sc;
                    if (key > qrow) v = -INFINITY;
                    sacc[j][e] = v;
                    mx[e >> 1] = fmaxf(mx[e >> 1], v);
                }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
                mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
            }
            float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
            for (int r = 0; r < 2; ++r) corr[r] = exp2f(mrow[r] - mx[r]);
#pragma unroll
            for (int j = 0; j < BN / 8; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float p = exp2f(sacc[j][e] - mx[e >> 1]);
                    sacc[j][e] = p;
                    rs[e >> 1] += p;
                }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                lrow[r] = lrow[r] * corr[r] + rs[r];
                mrow[r] = mx[r];
            }
#pragma unroll
            for (int i = 0; i < D / 8; ++i) {
                oacc[i][0] *= corr[0]; oacc[i][1] *= corr[0];
                oacc[i][2] *= corr[1]; oacc[i][3] *= corr[1];
            }
            // O += P V
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
                uint32_t pa[4];
                pa[0] = pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]);
                pa[1] = pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]);
                pa[2] = pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
                pa[3] = pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
                for (int np = 0; np < D / 16; ++np) {
                    uint32_t bfr[4];
                    ldsm_x4_t(bfr, tile_ptr<D>(V, kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8,
                                               np * 16 + (lane >> 4) * 8));
                    mma16816(oacc[2 * np], pa, bfr[0], bfr[1]);
                    mma16816(oacc[2 * np + 1], pa, bfr[2], bfr[3]);
                }
            }
        }
        __syncthreads();
    }
    // row sums across the quad, normalise, write
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
        lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int qrow = wr0 + g + r * 8;
        if (qrow >= s) continue;
        const float inv = 1.0f / lrow[r];
        bf16* orow = o + ((long)b * s + qrow) * h + head * D;
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
            *reinterpret_cast<uint32_t*>(orow + i * 8 + 2 * t) =
                pack_bf16(oacc[i][2 * r] * inv, oacc[i][2 * r + 1] * inv);
        if (t == 0) lse[((long)b * a + head) * s + qrow] = (mrow[r] + log2f(lrow[r])) / LOG2E;
    }
}

// ----------------------------------------------------------------------- backward dK dV
template <int D>
__global__ void __launch_bounds__(128) bwd_dkdv_kernel(const bf16* __restrict__ qkv,
                                                       const bf16* __restrict__ dout,
                                                       const float* __restrict__ lse,
                                                       const float* __restrict__ Dv,
                                                       bf16* __restrict__ dqkv, int s, int a) {
    constexpr int BN = 64, BM = 64, NT = 128;
    extern __shared__ __align__(128) uint8_t smraw[];
    bf16* sK = reinterpret_cast<bf16*>(smraw);
    bf16* sV = sK + BN * D;
    bf16* sQ = sV + BN * D;          // 2 stages
    bf16* sO = sQ + 2 * BM * D;      // dO, 2 stages
    float* sL = reinterpret_cast<float*>(sO + 2 * BM * D);   // 2 x BM lse
    float* sD = sL + 2 * BM;                                 // 2 x BM D
    const int nkb = (s + BN - 1) / BN;
    const int kbi = blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const long ld = 3L * h;
    const bf16* base = qkv + (long)b * s * ld;
    const bf16* dob = dout + (long)b * s * h + head * D;
    const float* lseb = lse + ((long)b * a + head) * s;
    const float* Db = Dv + ((long)b * a + head) * s;
    const int k0 = kbi * BN;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const float sc = rsqrtf((float)D) * LOG2E;
    (void)nkb;

    load_tile<D, BN, NT>(sK, base + (long)k0 * ld + h + head * D, ld, s - k0);
    load_tile<D, BN, NT>(sV, base + (long)k0 * ld + 2 * h + head * D, ld, s - k0);
    const int qb0 = k0 / BM;                      // first query block touching these keys
    const int nqb = (s + BM - 1) / BM;
    auto load_q = [&](int qb, int st) {
        const int q0 = qb * BM;
        load_tile<D, BM, NT>(sQ + st * BM * D, base + (long)q0 * ld + head * D, ld, s - q0);
        load_tile<D, BM, NT>(sO + st * BM * D, dob + (long)q0 * h, h, s - q0);
        for (int e = threadIdx.x; e < BM; e += NT) {
            const int q = q0 + e;
            sL[st * BM + e] = q < s ? lseb[q] * LOG2E : 0.f;
            sD[st * BM + e] = q < s ? Db[q] : 0.f;
        }
    };
    load_q(qb0, 0);
    cp_async_commit();

    float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
    const int wk0 = k0 + warp * 16;   // first key row of this warp

    for (int qb = qb0; qb < nqb; ++qb) {
        const int st = (qb - qb0) & 1;
        if (qb + 1 < nqb) load_q(qb + 1, st ^ 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int q0 = qb * BM;
        bf16* Q = sQ + st * BM * D;
        bf16* dO = sO + st * BM * D;
        const float* L = sL + st * BM;
        const float* Dq = sD + st * BM;
        if (q0 + BM - 1 >= wk0) {
            // S^T = K Q^T  [16 keys x BM queries]; dP^T = V dO^T
            float sacc[BM / 8][4], pacc[BM / 8][4];
#pragma unroll
            for (int j = 0; j < BM / 8; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) sacc[j][e] = pacc[j][e] = 0.f;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint32_t ka[4], va[4];
                ldsm_x4(ka, tile_ptr<D>(sK, warp * 16 + (lane & 15), kk * 16 + (lane >> 4) * 8));
                ldsm_x4(va, tile_ptr<D>(sV, warp * 16 + (lane & 15), kk * 16 + (lane >> 4) * 8));
#pragma unroll
                for (int jp = 0; jp < BM / 16; ++jp) {
                    uint32_t qb4[4], ob4[4];
                    const int rr = jp * 16 + (lane & 7) + (lane >> 4) * 8;
                    const int cc = kk * 16 + ((lane >> 3) & 1) * 8;
                    ldsm_x4(qb4, tile_ptr<D>(Q, rr, cc));
                    ldsm_x4(ob4, tile_ptr<D>(dO, rr, cc));
                    mma16816(sacc[2 * jp], ka, qb4[0], qb4[1]);
                    mma16816(sacc[2 * jp + 1], ka, qb4[2], qb4[3]);
                    mma16816(pacc[2 * jp], va, ob4[0], ob4[1]);
                    mma16816(pacc[2 * jp + 1], va, ob4[2], ob4[3]);
                }
            }
            // P^T = exp2(S^T sc - L[q]); dS^T = P^T (dP^T - D[q])
#pragma unroll
            for (int j = 0; j < BM / 8; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int key = wk0 + g + (e >> 1) * 8;
                    const int ql = j * 8 + 2 * t + (e & 1);
                    const int q = q0 + ql;
                    float p = (q >= key && q < s) ? exp2f(sacc[j][e] * sc - L[ql]) : 0.f;
                    sacc[j][e] = p;
                    pacc[j][e] = p * (pacc[j][e] - Dq[ql]);
                }
            // dV += P^T dO ; dK += dS^T Q   (B operands [query][d] -> ldmatrix.trans)
#pragma unroll
            for (int kk = 0; kk < BM / 16; ++kk) {
                uint32_t pa[4], sa[4];
                pa[0] = pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]);
                pa[1] = pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]);
                pa[2] = pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
                pa[3] = pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
                sa[0] = pack_bf16(pacc[2 * kk][0], pacc[2 * kk][1]);
                sa[1] = pack_bf16(pacc[2 * kk][2], pacc[2 * kk][3]);
                sa[2] = pack_bf16(pacc[2 * kk + 1][0], pacc[2 * kk + 1][1]);
                sa[3] = pack_bf16(pacc[2 * kk + 1][2], pacc[2 * kk + 1][3]);
#pragma unroll
                for (int np = 0; np < D / 16; ++np) {
                    uint32_t ob4[4], qb4[4];
                    const int rr = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    const int cc = np * 16 + (lane >> 4) * 8;
                    ldsm_x4_t(ob4, tile_ptr<D>(dO, rr, cc));
                    ldsm_x4_t(qb4, tile_ptr<D>(Q, rr, cc));
                    mma16816(dv[2 * np], pa, ob4[0], ob4[1]);
                    mma16816(dv[2 * np + 1], pa, ob4[2], ob4[3]);
                    mma16816(dk[2 * np], sa, qb4[0], qb4[1]);
                    mma16816(dk[2 * np + 1], sa, qb4[2], qb4[3]);
                }
            }
        }
        __syncthreads();
    }
    const float scale = rsqrtf((float)D);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int key = wk0 + g + r * 8;
        if (key >= s) continue;
        bf16* dkr = dqkv + ((long)b * s + key) * ld + h + head * D;
        bf16* dvr = dkr + h;
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            *reinterpret_cast<uint32_t*>(dkr + i * 8 + 2 * t) =
                pack_bf16(dk[i][2 * r] * scale, dk[i][2 * r + 1] * scale);
            *reinterpret_cast<uint32_t*>(dvr + i * 8 + 2 * t) = pack_bf16(dv[i][2 * r], dv[i][2 * r + 1]);
        }
    }
}

// ----------------------------------------------------------------------- backward dQ
template <int D>
__global__ void __launch_bounds__(128) bwd_dq_kernel(const bf16* __restrict__ qkv,
                                                     const bf16* __restrict__ dout,
                                                     const float* __restrict__ lse,
                                                     const float* __restrict__ Dv,
                                                     bf16* __restrict__ dqkv, int s, int a) {
    constexpr int BM = 64, BN = 64, NT = 128;
    extern __shared__ __align__(128) uint8_t smraw[];
    bf16* sQ = reinterpret_cast<bf16*>(smraw);
    bf16* sO = sQ + BM * D;
    bf16* sK = sO + BM * D;          // 2 stages
    bf16* sV = sK + 2 * BN * D;      // 2 stages
    const int nqb = (s + BM - 1) / BM;
    const int qb = nqb - 1 - blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int h = a * D;
    const long ld = 3L * h;
    const bf16* base = qkv + (long)b * s * ld;
    const int q0 = qb * BM;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const float sc = rsqrtf((float)D) * LOG2E;
    const int wr0 = q0 + warp * 16;
    const float* lseb = lse + ((long)b * a + head) * s;
    const float* Db = Dv + ((long)b * a + head) * s;
    float Lr[2], Dr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = wr0 + g + r * 8;
        Lr[r] = q < s ? lseb[q] * LOG2E : 0.f;
        Dr[r] = q < s ? Db[q] : 0.f;
    }
    load_tile<D, BM, NT>(sQ, base + (long)q0 * ld + head * D, ld, s - q0);
    load_tile<D, BM, NT>(sO, dout + ((long)b * s + q0) * h + head * D, h, s - q0);
    const int nkb = (q0 + BM + BN - 1) / BN;
    load_tile<D, BN, NT>(sK, base + h + head * D, ld, s);
    load_tile<D, BN, NT>(sV, base + 2 * h + head * D, ld, s);
    cp_async_commit();

    float dq[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

    for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb & 1;
        if (kb + 1 < nkb) {
            const int k0n = (kb + 1) * BN;
            load_tile<D, BN, NT>(sK + (st ^ 1) * BN * D, base + (long)k0n * ld + h + head * D, ld, s - k0n);
            load_tile<D, BN, NT>(sV + (st ^ 1) * BN * D, base + (long)k0n * ld + 2 * h + head * D, ld, s - k0n);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int k0 = kb * BN;
        if (k0 <= wr0 + 15) {
            bf16* K = sK + st * BN * D;
            bf16* V = sV + st * BN * D;
            float sacc[BN / 8][4], pacc[BN / 8][4];
#pragma unroll
            for (int j = 0; j < BN / 8; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) sacc[j][e] = pacc[j][e] = 0.f;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint32_t qa[4], oa[4];
                ldsm_x4(qa, tile_ptr<D>(sQ, warp * 16 + (lane & 15), kk * 16 + (lane >> 4) * 8));
                ldsm_x4(oa, tile_ptr<D>(sO, warp * 16 + (lane & 15), kk * 16 + (lane >> 4) * 8));
#pragma unroll
                for (int jp = 0; jp < BN / 16; ++jp) {
                    uint32_t kb4[4], vb4[4];
                    const int rr = jp * 16 + (lane & 7) + (lane >> 4) * 8;
                    const int cc = kk * 16 + ((lane >> 3) & 1) * 8;
                    ldsm_x4(kb4, tile_ptr<D>(K, rr, cc));
                    ldsm_x4(vb4, tile_ptr<D>(V, rr, cc));
                    mma16816(sacc[2 * jp], qa, kb4[0], kb4[1]);
                    mma16816(sacc[2 * jp + 1], qa, kb4[2], kb4[3]);
                    mma16816(pacc[2 * jp], oa, vb4[0], vb4[1]);
                    mma16816(pacc[2 * jp + 1], oa, vb4[2], vb4[3]);
                }
            }
#pragma unroll
            for (int j = 0; j < BN / 8; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int q = wr0 + g + (e >> 1) * 8;
                    const int key = k0 + j * 8 + 2 * t + (e & 1);
                    float p = (key <= q) ? exp2f(sacc[j][e] * sc - Lr[e >> 1]) : 0.f;
                    pacc[j][e] = p * (pacc[j][e] - Dr[e >> 1]);
                }
            // dQ += dS K   (B = K[key][d] -> ldmatrix.trans)
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
                uint32_t sa[4];
                sa[0] = pack_bf16(pacc[2 * kk][0], pacc[2 * kk][1]);
                sa[1] = pack_bf16(pacc[2 * kk][2], pacc[2 * kk][3]);
                sa[2] = pack_bf16(pacc[2 * kk + 1][0], pacc[2 * kk + 1][1]);
                sa[3] = pack_bf16(pacc[2 * kk + 1][2], pacc[2 * kk + 1][3]);
#pragma unroll
                for (int np = 0; np < D / 16; ++np) {
                    uint32_t kb4[4];
                    ldsm_x4_t(kb4, tile_ptr<D>(K, kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8,
                                               np * 16 + (lane >> 4) * 8));
                    mma16816(dq[2 * np], sa, kb4[0], kb4[1]);
                    mma16816(dq[2 * np + 1], sa, kb4[2], kb4[3]);
                }
            }
        }
        __syncthreads();
    }
    const float scale = rsqrtf((float)D);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int q = wr0 + g + r * 8;
        if (q >= s) continue;
        bf16* dqr = dqkv + ((long)b * s + q) * ld + head * D;
#pragma unroll
        for (int i = 0; i < D / 8; ++i)
            *reinterpret_cast<uint32_t*>(dqr + i * 8 + 2 * t) =
                pack_bf16(dq[i][2 * r] * scale, dq[i][2 * r + 1] * scale);
    }
}

}  // namespace fa

// D[b,head,i] = sum_e dO[i,e] O[i,e] (fp32), one warp per row
__global__ void fa_bwd_d_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout,
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

template <int D>
static int launch_fwd(const void* qkv, void* o, float* lse, int b, int s, int a, cudaStream_t st) {
    constexpr int smem = (128 * D + 4 * 64 * D) * 2;
    static PerDeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(fa::fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    dim3 grid((s + 127) / 128, a, b);
    fa::fwd_kernel<D><<<grid, 256, smem, st>>>((const bf16*)qkv, (bf16*)o, lse, s, a);
    note_launches(1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

template <int D>
static int launch_bwd(const void* qkv, const void* o, const void* dout, const float* lse,
                      void* dqkv, float* ws, int b, int s, int a, cudaStream_t st) {
    constexpr int smem_kv = (2 * 64 * D + 4 * 64 * D) * 2 + 4 * 64 * 4;
    constexpr int smem_q = (2 * 64 * D + 4 * 64 * D) * 2;
    static PerDeviceOnce attr;
    if (attr.first()) {
        cudaFuncSetAttribute(fa::bwd_dkdv_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
        cudaFuncSetAttribute(fa::bwd_dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
    }
    dim3 gd((s + 3) / 4, a, b);
    fa_bwd_d_kernel<<<gd, 128, 0, st>>>((const bf16*)o, (const bf16*)dout, ws, s, a, D);
    dim3 grid((s + 63) / 64, a, b);
    fa::bwd_dkdv_kernel<D><<<grid, 128, smem_kv, st>>>((const bf16*)qkv, (const bf16*)dout, lse, ws,
                                                       (bf16*)dqkv, s, a);
    fa::bwd_dq_kernel<D><<<grid, 128, smem_q, st>>>((const bf16*)qkv, (const bf16*)dout, lse, ws,
                                                    (bf16*)dqkv, s, a);
    note_launches(3);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int attn_fwd_tc(const void* qkv, void* o, float* lse, int b, int s, int a, int d, cudaStream_t st) {
    return d == 64 ? launch_fwd<64>(qkv, o, lse, b, s, a, st) : launch_fwd<128>(qkv, o, lse, b, s, a, st);
}

int attn_bwd_tc(const void* qkv, const void* o, const void* dout, const float* lse, void* dqkv,
                float* ws, int b, int s, int a, int d, cudaStream_t st) {
    return d == 64 ? launch_bwd<64>(qkv, o, dout, lse, dqkv, ws, b, s, a, st)
                   : launch_bwd<128>(qkv, o, dout, lse, dqkv, ws, b, s, a, st);
}

}  // namespace tpipe
