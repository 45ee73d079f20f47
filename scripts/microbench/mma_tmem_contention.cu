// Does tcgen05.ld / tcgen05.st traffic from other warps slow the tensor pipe?
// One CTA per SM, 4 + 8 warps: warp 0's elected lane issues ITER TS MMAs
// (kind::f16, M = 128, N = 64 or 128, A in TMEM columns [384, 448), B K-major
// in shared memory, accumulator columns [0, N)) back to back; warps 4..11
// meanwhile loop tcgen05.ld (32 lanes x 32 columns) [+ tcgen05.st back] over
// TMEM columns [128, 384) (the attention backward's elementwise pattern) until
// the MMAs are done. Reports MMA cycles per instruction with and without it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_03182_b200/csrc \
//        scripts/microbench/mma_tmem_contention.cu -o /tmp/mtc && /tmp/mtc
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels/common.cuh"

using namespace tpipe;

constexpr int ITER = 65536;   // long enough (~2 ms per CTA) for the power state to settle

__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,"
        "%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(384, 1) contention(int N, int mode, long long* out, const uint8_t* gsrc) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, bar2, bar3;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        mbar_init(&bar3, 1);
        fence_mbar_init();
        done = 0;
    }
    if (warp == 1) tmem_alloc(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (warp == 0) {
        long long t0 = clock64();
        if (elect_one()) {
            const uint64_t db0 = umma_desc_sw128(smem_u32(sm), 0, 1024);
            if (mode == 7 || mode == 8 || mode == 9 || mode == 10) {
                // the forward kernel's pattern (D = 128): per tile, S = Q K^T (8 TS
                // MMAs, A = Q in TMEM [384, 448), B = K K-major in 2 swizzle atoms of
                // 64 d x 128 keys) into S buffer (tile & 1) * 128, then O += P V (8
                // TS MMAs, A = P packed in the other S buffer, B = V MN-major), a
                // commit after each group (mode 8: + a second commit, as the kernel)
                const uint32_t idS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
                const uint32_t idO = idS | (1u << 16);   // B MN-major
                const uint32_t aK = smem_u32(sm), aV = smem_u32(sm + 32768);
                for (int tile = 0; tile < ITER / 16; ++tile) {
                    const uint32_t tS = tmem + (tile & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_bf16_ts(tS, tmem + 384 + kk * 8,
                                     umma_desc_sw128(aK + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 0, 1024), idS,
                                     kk > 0);
                    umma_commit(&bar2);
                    if (mode == 8) umma_commit(&bar3);
                    const uint32_t tP = tmem + ((tile + 1) & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_bf16_ts(tmem + 256, tP + kk * 8, umma_desc_sw128(aV + kk * 2048, 128 * 128, 1024), idO,
                                     (tile | kk) > 0);
                    umma_commit(&bar2);
                    if (mode == 8) umma_commit(&bar3);
                }
            } else if (mode < 3 || mode >= 5) {
                for (int i = 0; i < ITER; ++i) {
                    const int k = i & 3;
                    umma_bf16_ts(tmem, tmem + 384 + 8 * k, db0 + 2 * k, id, i > 0);
                }
            } else {
                // the dQ kernel's pattern: S = Q K^T and dP = dO V^T interleaved per
                // K = 16 step (D = 128: 8 steps), A operands Q / dO in TMEM columns
                // [384, 448) / [448, 512), B = two 64-row half tiles (2 swizzle atoms
                // of 64 x 128 B each), accumulators [0, N) and [N, 2N)
                const uint32_t aK = smem_u32(sm), aV = smem_u32(sm + 16384);
                for (int i = 0; i < ITER / 2; ++i) {
                    const int kk = i & 7;
                    const uint64_t dk = umma_desc_sw128(aK + (kk >> 2) * (64 * 128) + (kk & 3) * 32, 0, 1024);
                    const uint64_t dv = umma_desc_sw128(aV + (kk >> 2) * (64 * 128) + (kk & 3) * 32, 0, 1024);
                    umma_bf16_ts(tmem, tmem + 384 + 8 * kk, dk, id, kk > 0);
                    umma_bf16_ts(tmem + N, tmem + 448 + 8 * kk, dv, id, kk > 0);
                }
            }
            umma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) {
            out[blockIdx.x] = t1 - t0;
            done = 1;
        }
    } else if (warp == 3 && (mode == 9 || mode == 10)) {
        // a TMA-like producer: 32 KB bulk copies global -> shared (the
        // forward's K / V tile loads, ~64 KB per 2000 cycles), back to back
        __shared__ uint64_t cbar;
        if (threadIdx.x == 96) {
            mbar_init(&cbar, 1);
            fence_mbar_init();
        }
        __syncwarp();
        uint32_t ph = 0;
        long off = (long)blockIdx.x * 65536;
        while (!done) {
            if (threadIdx.x == 96) {
                mbar_arrive_expect_tx(&cbar, 32768);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];" ::"r"(
                        smem_u32(sm + 65536)),
                    "l"(gsrc + off), "r"(smem_u32(&cbar))
                    : "memory");
            }
            __syncwarp();
            mbar_wait(&cbar, ph);
            ph ^= 1;
            off = (off + 32768) % (64L << 20);
        }
    } else if (warp >= 4 && (mode == 5 || mode == 10 || (mode == 6 && (warp & 3) != 0))) {
        // ALU-heavy warps (softmax-like: packed FMAs + MUFU.EX2), mode 6 only on
        // the three sub-partitions the MMA-issuing warp 0 does not use
        float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.5f, acc = 0.f;
        while (!done) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(x1) : "f"(x0));
                x0 = fmaf(x1, 0.999f, -0.25f);
                acc += x1;
            }
        }
        if (acc == 1234.5f) out[gridDim.x] = 1;
    } else if (warp >= 4 && (mode == 1 || mode == 2 || mode == 4)) {
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const int cg = (warp - 4) >> 2;   // two column groups
        uint32_t acc = 0;
        int it = 0;
        while (!done) {
            uint32_t r[32];
            const uint32_t col = 128 + cg * 128 + (it & 3) * 32;
            tld32(tmem + lane_off + col, r);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += r[j];
            if (mode == 2 || mode == 4) {
                tmem_st32(tmem + lane_off + col, r);
                tmem_wait_st();
            }
            ++it;
        }
        if (acc == 0x12345678u) out[gridDim.x] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, (sms + 1) * sizeof(long long));
    uint8_t* gsrc;
    cudaMalloc(&gsrc, (64L << 20) + 65536L * 160);
    cudaFuncSetAttribute(contention, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    if (argc > 1) {   // soak: mode argv[1] (N = 128) back to back for argv[2] seconds, report each launch
        const int mode = atoi(argv[1]);
        const double secs = argc > 2 ? atof(argv[2]) : 5.0;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        double el = 0;
        int it = 0;
        while (el < secs * 1e3) {
            cudaEventRecord(e0);
            contention<<<sms, 384, 100 * 1024>>>(128, mode, d, gsrc);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            el += ms;
            long long h[160];
            cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms; ++i) avg += h[i];
            avg /= sms;
            if (it % 50 == 0)
                printf("{\"mode\": %d, \"t_ms\": %.0f, \"cycles_per_mma\": %.1f, \"launch_ms\": %.3f}\n", mode, el,
                       avg / ITER, ms);
            ++it;
        }
        return 0;
    }
    static const char* names[] = {"mma_alone", "with_tmem_ld", "with_tmem_ld_st", "dq_pattern_alone",
                                  "dq_pattern_with_tmem_ld_st", "with_alu_warps_all_sps",
                                  "with_alu_warps_other_sps", "fwd_pattern", "fwd_pattern_2commits",
                                  "fwd_pattern_with_bulk_copies", "fwd_pattern_bulk_copies_alu_warps"};
    for (int N : {64, 128})
        for (int mode = 0; mode < 11; ++mode) {
            if ((mode == 3 || mode == 4) && N != 64) continue;
            if (mode >= 7 && N != 128) continue;
            contention<<<sms, 384, 100 * 1024>>>(N, mode, d, gsrc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            long long h[160];
            cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms; ++i) avg += h[i];
            avg /= sms;
            printf("{\"N\": %d, \"mode\": \"%s\", \"cycles_per_mma\": %.1f, \"floor\": %d}\n", N, names[mode],
                   avg / ITER, N / 2);
        }
    return 0;
}
