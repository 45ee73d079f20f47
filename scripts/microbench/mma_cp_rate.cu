// tcgen05.cp + TS-MMA rate microbenchmark: can a GEMM keep its A operand in
// TMEM by copying every K16 slice smem -> TMEM (tcgen05.cp.128x256b) right
// before the MMA that reads it, and still run at the TS-MMA rate
// (profiles/r2_mma_rate.jsonl: TS ~10 + N/2 cycles per instruction vs SS
// ~45 + N/2)?  Modes, per iteration i (slot = i % R of an R-slot TMEM ring):
//   0 "ss":        SS MMA (baseline)
//   1 "cp+ts":     cp(slot i) ; ts-mma(slot i)
//   2 "cp_ahead":  cp(slot i + R/2) ; ts-mma(slot i)   (copy issued R/2 slices ahead)
//   3 "cp_only":   cp(slot i)                          (copy throughput alone)
// cta_group::1 (grid 148) and cta_group::2 pairs (grid 148, M = 256).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_03182_b200/csrc \
//        scripts/microbench/mma_cp_rate.cu -o /tmp/mma_cp_rate && /tmp/mma_cp_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "kernels/common.cuh"

using namespace tpipe;

constexpr int ITER = 1024;

__device__ __forceinline__ void cp1(uint32_t taddr, uint64_t d) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}
__device__ __forceinline__ void cp2(uint32_t taddr, uint64_t d) {
    asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(taddr), "l"(d) : "memory");
}
__device__ __forceinline__ void ts2(uint32_t d, uint32_t a, uint64_t db, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(db), "r"(id), "r"(acc)
        : "memory");
}

template <int CG>
__global__ void __launch_bounds__(128, 1) cp_rate(int N, int R, int mode, long long* out) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 1) {
        if (CG == 2) tmem_alloc_pair(&slot, 512);
        else tmem_alloc(&slot, 512);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t tA = tmem + 512 - R * 8;
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                        ((uint32_t)((128 * CG) >> 4) << 24);
    long long t0 = 0, t1 = 0;
    for (int rep = 0; rep < 2; ++rep) {
        if (warp == 0) {
            __syncwarp();
            t0 = clock64();
            if (rank == 0 && elect_one()) {
                const uint32_t aA = smem_u32(sm), aB = smem_u32(sm + 32 * 1024);
                if (mode == 2)
                    for (int j = 0; j < R / 2; ++j) {
                        const uint64_t da = umma_desc_sw128(aA + (j & 3) * 32, 0, 1024);
                        if (CG == 2) cp2(tA + j * 8, da);
                        else cp1(tA + j * 8, da);
                    }
                for (int i = 0; i < ITER; ++i) {
                    const int kk = i & 3;
                    const uint64_t db = umma_desc_sw128(aB + kk * 32, 0, 1024);
                    const uint32_t acc = i >= 1;
                    if (mode == 0) {
                        if (CG == 2) umma_bf16_pair(tmem, umma_desc_sw128(aA + kk * 32, 0, 1024), db, id, acc);
                        else umma_bf16(tmem, umma_desc_sw128(aA + kk * 32, 0, 1024), db, id, acc);
                        continue;
                    }
                    const int cs = mode == 2 ? (i + R / 2) % R : i % R;
                    const uint64_t da = umma_desc_sw128(aA + ((mode == 2 ? i + R / 2 : i) & 3) * 32, 0, 1024);
                    if (CG == 2) cp2(tA + cs * 8, da);
                    else cp1(tA + cs * 8, da);
                    if (mode == 3) continue;
                    if (CG == 2) ts2(tmem, tA + (i % R) * 8, db, id, acc);
                    else umma_bf16_ts(tmem, tA + (i % R) * 8, db, id, acc);
                }
                if (CG == 2) umma_commit_pair(&bar, 3);
                else umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, rep & 1);
            t1 = clock64();
        }
        tc_fence_before();
        if (CG == 2) cluster_sync_all();
        else __syncthreads();
        tc_fence_after();
    }
    if (threadIdx.x == 0 && rank == 0) out[blockIdx.x / CG] = t1 - t0;
    tc_fence_before();
    if (CG == 2) cluster_sync_all();
    else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2) tmem_dealloc_pair(tmem, 512);
        else tmem_dealloc(tmem, 512);
    }
}

template <int CG>
static int run(int sms, long long* d) {
    static const char* names[] = {"ss", "cp+ts", "cp_ahead", "cp_only"};
    auto k = cp_rate<CG>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int grid = CG * (sms / CG);
    for (int N : {128, 192, 224, 240, 256})
        for (int R : {4, 8, 16, 32})
            for (int mode = 0; mode < 4; ++mode) {
                if (N + R * 8 > 512) continue;
                if (mode == 0 && R != 4) continue;
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(128);
                cfg.dynamicSmemBytes = 100 * 1024;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = CG;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                if (cudaLaunchKernelEx(&cfg, k, N, R, mode, d) != cudaSuccess) {
                    printf("launch error\n");
                    return 1;
                }
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s (N %d R %d mode %d cg %d)\n", cudaGetErrorString(e), N, R, mode, CG);
                    return 1;
                }
                long long h[160];
                const int units = grid / CG;
                cudaMemcpy(h, d, units * sizeof(long long), cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < units; ++i) avg += h[i];
                avg /= units;
                const double cyc = avg / ITER, floor_ = N / 2.0;
                printf("{\"cta_group\": %d, \"N\": %d, \"ring\": %d, \"mode\": \"%s\", \"cycles_per_k16\": %.1f, "
                       "\"floor\": %.0f, \"efficiency\": %.3f}\n",
                       CG, N, R, names[mode], cyc, floor_, mode == 3 ? 0.0 : floor_ / cyc);
                fflush(stdout);
            }
    return 0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    if (run<1>(sms, d)) return 1;
    if (run<2>(sms, d)) return 1;
    return 0;
}
