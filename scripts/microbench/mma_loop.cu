// What does the MMA-issuing thread's loop cost?  tcgen05.mma rate (kind::f16,
// M = 128, SS) when the issue loop looks like the GEMM's k-block loop:
//   per k-block: wait on the stage's full barrier (pre-completed here, so the
//   wait succeeds at once), tcgen05 fence, 4 MMAs (K = 64), commit to the
//   stage's empty barrier, advance stage / phase.
// Variants remove one piece of per-k-block work at a time:
//   0 gemm-like   1 no barrier wait   2 no commit   3 descriptors precomputed
//   (64-bit adds on a base descriptor)   4 = 3 + 2 k-blocks per iteration
//   5 tight (no wait / commit, precomputed descriptors; the floor reference)
//   6 tight TS (A from TMEM), B K-major   7 tight TS, B MN-major   8 tight SS, B MN-major
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_03182_b200/csrc \
//        scripts/microbench/mma_loop.cu -o /tmp/mma_loop && /tmp/mma_loop
#include <cstdio>
#include <cuda_runtime.h>

#include "kernels/common.cuh"

using namespace tpipe;

constexpr int KB = 512;   // k-blocks per measurement (4 MMAs each)

template <int V, int N>
__global__ void __launch_bounds__(128, 1) loop_rate(long long* out) {
    constexpr int STAGES = N > 128 ? 4 : 6;
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t ready, empty[STAGES], done;
    __shared__ uint32_t slot;
    constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = N * 64 * 2;
    for (int i = threadIdx.x; i < STAGES * (A_BYTES + B_BYTES) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&ready, 1);
        for (int s = 0; s < STAGES; ++s) mbar_init(&empty[s], 1);
        mbar_init(&done, 1);
        fence_mbar_init();
        mbar_arrive(&ready);   // phase 0 complete: every parity-0 wait succeeds
    }
    if (warp == 1) tmem_alloc(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    uint8_t* sA = sm;
    uint8_t* sB = sm + STAGES * A_BYTES;
    long long t0 = 0, t1 = 0;
    for (int rep = 0; rep < 2; ++rep) {
        if (warp == 0) {
            __syncwarp();
            t0 = clock64();
            if (V >= 5) {
                if (elect_one()) {
                    const uint64_t da0 = umma_desc_sw128(smem_u32(sA), 0, 1024);
                    const uint64_t db0 = (V == 7 || V == 8) ? umma_desc_sw128(smem_u32(sB), 64 * 128, 1024)
                                                            : umma_desc_sw128(smem_u32(sB), 0, 1024);
                    const uint64_t dbk = (V == 7 || V == 8) ? 128 : 2;   // per K=16 step
                    const uint32_t idb = idesc | ((V == 7 || V == 8) ? (1u << 16) : 0u);
                    for (int i = 0; i < KB * 4; ++i) {
                        const int k = i & 3;
                        if (V == 6 || V == 7) umma_bf16_ts(tmem, tmem + 256 + 8 * k, db0 + dbk * k, idb, i > 0);
                        else umma_bf16(tmem, da0 + 2 * k, db0 + dbk * k, idb, i > 0);
                    }
                }
            } else {
                int stage = 0;
                const uint64_t da0 = umma_desc_sw128(smem_u32(sA), 0, 1024);
                const uint64_t db0 = umma_desc_sw128(smem_u32(sB), 0, 1024);
                constexpr int STEP = V == 4 ? 2 : 1;
                for (int kb = 0; kb < KB; kb += STEP) {
#pragma unroll
                    for (int u = 0; u < STEP; ++u) {
                        if (V != 1) {
                            mbar_wait(&ready, 0);
                            tc_fence_after();
                        }
                        if (elect_one()) {
                            if (V >= 3) {
                                const uint64_t da = da0 + (uint64_t)(stage * (A_BYTES >> 4));
                                const uint64_t db = db0 + (uint64_t)(stage * (B_BYTES >> 4));
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb + u) != 0 || k != 0);
                            } else {
                                const uint32_t a_addr = smem_u32(sA + stage * A_BYTES);
                                const uint32_t b_addr = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    umma_bf16(tmem, umma_desc_sw128(a_addr + k * 32, 0, 1024),
                                              umma_desc_sw128(b_addr + k * 32, 0, 1024), idesc,
                                              (kb + u) != 0 || k != 0);
                            }
                            if (V != 2) umma_commit(&empty[stage]);
                        }
                        __syncwarp();
                        if (++stage == STAGES) stage = 0;
                    }
                }
            }
            if (elect_one()) umma_commit(&done);
            __syncwarp();
            mbar_wait(&done, rep & 1);
            t1 = clock64();
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int V, int N>
static void run(int grid, long long* d) {
    static const char* names[] = {"gemm_like", "no_wait", "no_commit", "precomputed_desc", "precomputed_x2",
                                  "tight",     "tight_ts_bK", "tight_ts_bMN", "tight_ss_bMN"};
    auto k = loop_rate<V, N>;
    constexpr int STAGES = N > 128 ? 4 : 6;
    const int smem = 1024 + STAGES * (128 * 64 * 2 + N * 64 * 2);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, 128, smem>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return;
    }
    long long h[160];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += h[i];
    avg /= grid;
    const double cyc = avg / (KB * 4), fl = N / 2.0;
    printf("{\"grid\": %d, \"N\": %d, \"variant\": \"%s\", \"cycles_per_mma\": %.1f, \"floor\": %.0f, "
           "\"efficiency\": %.3f}\n", grid, N, names[V], cyc, fl, fl / cyc);
    fflush(stdout);
}

template <int N>
static void all(int grid, long long* d) {
    run<0, N>(grid, d);
    run<5, N>(grid, d);
    run<8, N>(grid, d);
    if (N <= 256 - 32) {   // A in TMEM columns [256, 288): accumulator N <= 224 (N = 256: SS only)
        run<6, N>(grid, d);
        run<7, N>(grid, d);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, 160 * sizeof(long long));
    for (int grid : {1, sms}) {
        all<256>(grid, d);
        all<128>(grid, d);
        all<64>(grid, d);
        all<32>(grid, d);
    }
    return 0;
}
