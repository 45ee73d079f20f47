// tcgen05.mma issue-rate microbenchmark (kind::f16, bf16 x bf16 -> f32, M = 128,
// cta_group::1): cycles per instruction for N = 64 / 128 / 256, one or several
// independent accumulators, A from shared memory (SS) or tensor memory (TS).
// One CTA per SM (grid = 1 or #SMs); the elected thread of warp 0 issues ITER
// MMAs back to back, commits, waits; clock64 around the loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_03182_b200/csrc \
//        scripts/microbench/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "kernels/common.cuh"

using namespace tpipe;

__device__ __forceinline__ uint32_t idesc_f16(int N, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}

constexpr int ITER = 512;

__global__ void __launch_bounds__(128, 1) mma_rate(int N, int nacc, int ts, int b_mn, long long* out) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint32_t aA = smem_u32(sm), aB = smem_u32(sm + 32 * 1024);
        const uint32_t id = idesc_f16(N, b_mn);
        for (int rep = 0; rep < 2; ++rep) {
            __syncwarp();
            t0 = clock64();
            if (elect_one()) {
                for (int i = 0; i < ITER; ++i) {
                    const int kk = i & 3, acc = i % nacc;
                    const uint64_t db = b_mn ? umma_desc_sw128(aB + kk * 2048, 64 * 128, 1024)
                                             : umma_desc_sw128(aB + kk * 32, 0, 1024);
                    const uint32_t d = tmem + acc * N;
                    if (ts) umma_bf16_ts(d, tmem + 448 + kk * 8, db, id, i >= nacc);
                    else umma_bf16(d, umma_desc_sw128(aA + kk * 32, 0, 1024), db, id, i >= nacc);
                }
                umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, rep & 1);
            t1 = clock64();
        }
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// cta_group::2: a cluster of 2 (one CTA pair), M = 256, each CTA supplies 128
// rows of A and N/2 rows of B; the leader issues. cycles per instruction.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_rate_pair(int N, int ts, long long* out) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc_pair(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = 0, t1 = 0;
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    for (int rep = 0; rep < 2; ++rep) {
        if (warp == 0) {
            __syncwarp();
            t0 = clock64();
            if (rank == 0 && elect_one()) {
                const uint32_t aA = smem_u32(sm), aB = smem_u32(sm + 32 * 1024);
                for (int i = 0; i < ITER; ++i) {
                    const int kk = i & 3;
                    if (ts)
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (i & 1) * N),
                            "r"(tmem + 448 + kk * 8), "l"(umma_desc_sw128(aB + kk * 32, 0, 1024)), "r"(id),
                            "r"((uint32_t)(i >= 2))
                            : "memory");
                    else
                        umma_bf16_pair(tmem + (i & 1) * N, umma_desc_sw128(aA + kk * 32, 0, 1024),
                                       umma_desc_sw128(aB + kk * 32, 0, 1024), id, i >= 2);
                }
                umma_commit_pair(&bar, 3);
            }
            __syncwarp();
            mbar_wait(&bar, rep & 1);
            t1 = clock64();
        }
        tc_fence_before();
        cluster_sync_all();
        tc_fence_after();
    }
    if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / 2] = t1 - t0;
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem, 512);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    struct Cfg { int N, nacc, ts, bmn; };
    const Cfg cfgs[] = {{256, 1, 0, 0}, {256, 2, 0, 0}, {256, 1, 0, 1}, {128, 1, 0, 0}, {128, 2, 0, 0},
                        {128, 4, 0, 0}, {64, 1, 0, 0},  {64, 2, 0, 0},  {64, 4, 0, 0},  {128, 1, 1, 1},
                        {128, 2, 1, 1}, {64, 2, 1, 0},  {256, 1, 1, 0}, {128, 2, 0, 1}};
    for (int grid : {1, sms}) {
        for (const Cfg& c : cfgs) {
            if (c.ts && c.N * c.nacc > 448) continue;
            mma_rate<<<grid, 128, 100 * 1024>>>(c.N, c.nacc, c.ts, c.bmn, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[256];
            cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += h[i];
            avg /= grid;
            const double cyc = avg / ITER, floor_ = 128.0 * c.N / 256.0;
            printf("{\"grid\": %d, \"N\": %d, \"nacc\": %d, \"A\": \"%s\", \"B\": \"%s\", \"cycles_per_mma\": %.1f, "
                   "\"floor\": %.0f, \"efficiency\": %.3f}\n", grid, c.N, c.nacc, c.ts ? "tmem" : "smem",
                   c.bmn ? "MN" : "K", cyc, floor_, floor_ / cyc);
        }
    }
    cudaFuncSetAttribute(mma_rate_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int grid : {2, 2 * (sms / 2)}) {
        for (int cfg = 0; cfg < 5; ++cfg) {
            const int N = cfg == 0 ? 64 : (cfg == 1 || cfg == 3) ? 128 : 256, ts = cfg >= 3;
            if (ts && N * 2 > 448) continue;
            mma_rate_pair<<<grid, 128, 100 * 1024>>>(N, ts, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("pair error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[128];
            cudaMemcpy(h, d, (grid / 2) * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid / 2; ++i) avg += h[i];
            avg /= grid / 2;
            const double cyc = avg / ITER, floor_ = 256.0 * N / 512.0;
            printf("{\"grid\": %d, \"cta_group\": 2, \"M\": 256, \"N\": %d, \"A\": \"%s\", \"B\": \"K\", "
                   "\"cycles_per_mma\": %.1f, \"floor\": %.0f, \"efficiency\": %.3f}\n", grid, N, ts ? "tmem" : "smem",
                   cyc, floor_,
                   floor_ / cyc);
        }
    }
    return 0;
}
