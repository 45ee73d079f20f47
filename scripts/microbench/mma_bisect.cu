#include <cstdio>
#include <cuda_runtime.h>
#include "kernels/common.cuh"
using namespace tpipe;
constexpr int ITER = 1024;
// variant bits: 1 = d = tmem + (i % nacc) * N ; 2 = accumulate i >= nacc ; 4 = runtime b_mn select ; 8 = ts/ss predicated select; 16 = grid launched without cluster attr (n/a here)
__global__ void __launch_bounds__(128, 1) v(int N, int var, int nacc, int bmn, int ts, long long* out) {
    extern __shared__ uint8_t smraw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 1) tmem_alloc(&slot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint32_t aA = smem_u32(sm), aB = smem_u32(sm + 32 * 1024);
        const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bmn ? 1 : 0) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int rep = 0; rep < 2; ++rep) {
            __syncwarp();
            t0 = clock64();
            if (elect_one()) {
                for (int i = 0; i < ITER; ++i) {
                    const int kk = i & 3;
                    const int acc = (var & 1) ? i % nacc : 0;
                    const uint64_t db = ((var & 4) && bmn) ? umma_desc_sw128(aB + kk * 2048, 64 * 128, 1024)
                                                          : umma_desc_sw128(aB + kk * 32, 0, 1024);
                    const uint32_t d = tmem + acc * N;
                    const uint32_t accum = (var & 2) ? (i >= nacc) : (i >= 1);
                    if ((var & 8) && ts) umma_bf16_ts(d, tmem + 448 + kk * 8, db, id, accum);
                    else umma_bf16(d, umma_desc_sw128(aA + kk * 32, 0, 1024), db, id, accum);
                }
                umma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, rep & 1);
            t1 = clock64();
        }
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
int main() {
    long long* d; cudaMalloc(&d, 256 * sizeof(long long));
    cudaFuncSetAttribute(v, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int N : {128, 256})
    for (int var : {0, 1, 2, 4, 8, 15}) {
        v<<<1, 128, 100 * 1024>>>(N, var, 1, 0, 0, d);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"N\": %d, \"var\": %d, \"cycles_per_mma\": %.1f}\n", N, var, (double)h / ITER);
    }
    return 0;
}
