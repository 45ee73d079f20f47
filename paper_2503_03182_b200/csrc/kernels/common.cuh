// Common device helpers for the TPipe sm_100a kernels.
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace tpipe {

// True once per (call site, CUDA device): per-device one-time setup such as
// cudaFuncSetAttribute (function attributes are per device, so a process-wide
// flag would leave a second device at the default shared-memory limit).
struct PerDeviceOnce {
    unsigned long long mask = 0;
    bool first() {
        int d = 0;
        cudaGetDevice(&d);
        const unsigned long long bit = 1ull << (d & 63);
        return !(__atomic_fetch_or(&mask, bit, __ATOMIC_ACQ_REL) & bit);
    }
};


using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------- conversions
template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// round a float through the storage type T (identity for float)
template <typename T> __device__ __forceinline__ float rnd(float x) { return to_f<T>(from_f<T>(x)); }

// ---------------------------------------------------------------- programmatic dependent launch
// The hot-path kernels (tcgen05 GEMMs, tcgen05 attention, LayerNorm, column
// sums) are launched with programmatic stream serialisation: a kernel may be
// scheduled while its predecessor on the stream drains its last CTAs, runs its
// prologue (barrier init, TMEM alloc, descriptor prefetch) and then blocks in
// pdl_wait() until the predecessor has completed and its writes are visible.
// Every such kernel calls pdl_wait() before its first global-memory access
// (read or write), so stream order semantics are unchanged; pdl_trigger()
// lets the successor be scheduled early. Without the launch attribute both are
// no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();
void set_pdl(int on);

// cudaLaunchKernelEx with the PDL attribute (when enabled) and an optional
// cluster dimension.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            int cluster, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    unsigned n = 0;
    if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- math
// GELU, tanh approximation (DESIGN.md §2 reading N-1). Written with explicit
// _rn intrinsics so that the forward epilogue and the backward recompute give
// identical bits (operator-level recompute).
__device__ __forceinline__ float gelu_tanh(float u) {
    const float c = 0.7978845608028654f;   // sqrt(2/pi)
    float u3 = __fmul_rn(__fmul_rn(u, u), u);
    float inner = __fmul_rn(c, __fadd_rn(u, __fmul_rn(0.044715f, u3)));
    float t = tanhf(inner);
    return __fmul_rn(__fmul_rn(0.5f, u), __fadd_rn(1.0f, t));
}

__device__ __forceinline__ float gelu_tanh_grad(float u) {
    const float c = 0.7978845608028654f;
    float u2 = __fmul_rn(u, u);
    float inner = __fmul_rn(c, __fadd_rn(u, __fmul_rn(0.044715f, __fmul_rn(u2, u))));
    float t = tanhf(inner);
    float dt = __fmul_rn(__fmul_rn(__fsub_rn(1.0f, __fmul_rn(t, t)), c),
                         __fadd_rn(1.0f, __fmul_rn(0.134145f, u2)));
    return __fadd_rn(__fmul_rn(0.5f, __fadd_rn(1.0f, t)), __fmul_rn(__fmul_rn(0.5f, u), dt));
}

// bf16 tensor-core epilogues: GELU / GELU' with the hardware tanh
// (tanh.approx.f32, rel. error ~2^-11, far below bf16's 2^-9 rounding), one
// tanh shared by the value and the derivative. Forward (EPI_BIAS_GELU) and
// backward recompute (EPI_DGELU) both call gelu_fast on the same bf16 u, so
// the recomputed activation is bit-identical to the stored one.
__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float gelu_fast(float u) {
    const float c = 0.7978845608028654f;
    const float t = tanh_fast(__fmul_rn(c, __fadd_rn(u, __fmul_rn(0.044715f, __fmul_rn(__fmul_rn(u, u), u)))));
    return __fmul_rn(__fmul_rn(0.5f, u), __fadd_rn(1.0f, t));
}
__device__ __forceinline__ void gelu_fast_and_grad(float u, float& g, float& dg) {
    const float c = 0.7978845608028654f;
    const float u2 = __fmul_rn(u, u);
    const float t = tanh_fast(__fmul_rn(c, __fadd_rn(u, __fmul_rn(0.044715f, __fmul_rn(u2, u)))));
    g = __fmul_rn(__fmul_rn(0.5f, u), __fadd_rn(1.0f, t));
    const float dt = __fmul_rn(__fmul_rn(__fsub_rn(1.0f, __fmul_rn(t, t)), c),
                               __fadd_rn(1.0f, __fmul_rn(0.134145f, u2)));
    dg = __fadd_rn(__fmul_rn(0.5f, __fadd_rn(1.0f, t)), __fmul_rn(__fmul_rn(0.5f, u), dt));
}

// ---- packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100): one
// instruction per pair, each lane rounded exactly as the scalar .rn op
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// gelu_fast / gelu_fast_and_grad on a pair: the same op sequence per lane,
// half the FP instructions. ptxas contracts the packed u + 0.044715 u^3 into
// an FFMA2 (so these are not bit-identical to the scalar versions), the same
// way in both: the forward's stored GELU and the backward's recomputed one
// stay bit-identical (tests/test_gpu_kernels.py::test_gelu_recompute_bitexact)
__device__ __forceinline__ uint64_t gelu_fast2(uint64_t u) {
    const uint64_t C = pk2(0.7978845608028654f, 0.7978845608028654f), A = pk2(0.044715f, 0.044715f);
    const uint64_t inner = fmul2(C, fadd2(u, fmul2(A, fmul2(fmul2(u, u), u))));
    float i0, i1;
    upk2(inner, i0, i1);
    const uint64_t t = pk2(tanh_fast(i0), tanh_fast(i1));
    return fmul2(fmul2(pk2(0.5f, 0.5f), u), fadd2(pk2(1.f, 1.f), t));
}
__device__ __forceinline__ void gelu_fast_and_grad2(uint64_t u, uint64_t& g, uint64_t& dg) {
    const uint64_t C = pk2(0.7978845608028654f, 0.7978845608028654f), A = pk2(0.044715f, 0.044715f);
    const uint64_t H = pk2(0.5f, 0.5f), ONE = pk2(1.f, 1.f);
    const uint64_t u2 = fmul2(u, u);
    const uint64_t inner = fmul2(C, fadd2(u, fmul2(A, fmul2(u2, u))));
    float i0, i1;
    upk2(inner, i0, i1);
    const uint64_t t = pk2(tanh_fast(i0), tanh_fast(i1));
    const uint64_t hu = fmul2(H, u), opt = fadd2(ONE, t);
    g = fmul2(hu, opt);
    const uint64_t tt = fmul2(t, t ^ 0x8000000080000000ull);   // -(t*t), exactly
    const uint64_t dt = fmul2(fmul2(fadd2(ONE, tt), C), fadd2(ONE, fmul2(pk2(0.134145f, 0.134145f), u2)));
    dg = fadd2(fmul2(H, opt), fmul2(hu, dt));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------- PTX: smem, mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}

// named barrier over `n` threads (id 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------- PTX: TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* map, uint64_t* bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------- PTX: tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 inputs, fp32 accumulate)
// explicit shared-space accesses: tile pointers derived from the aligned
// dynamic-smem base (via uintptr_t) lose their address space, and the compiler
// then emits generic ST.E / LD.E (slower, and fence.proxy.async waits on them)
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    return v;
}

// elect.sync: true in exactly one lane (the lowest active one) of a converged
// warp. MMA issue roles run on the whole warp (so descriptors and loop state
// are warp-uniform and live in uniform registers) and issue tcgen05.mma /
// tcgen05.commit from the elected lane; a `lane == 0` region instead makes the
// compiler wrap every UTCHMMA in a uniformity waterfall loop.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T (A in tensor memory: 128 lanes = M rows,
// K packed two bf16 per 32-bit column), kind::f16
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t desc_b,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(desc_b), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0)
        : "memory");
}

// 32 lanes x 32 columns store (thread t writes lane base+t)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// arrive on an mbarrier when all previously issued tcgen05.mma have completed
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp receives lane (base+t),
// columns col..col+31.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

// ---------------------------------------------------------------- PTX: CTA pair (cta_group::2)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// all threads of both CTAs of the cluster
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cluster address of the same shared variable in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// TMA 2-D load into this CTA's smem; completion bytes counted on the mbarrier
// at shared::cluster address `bar_cluster` (the pair leader's barrier)
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* map, uint32_t bar_cluster,
                                                 int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(map), "r"(x), "r"(y), "r"(bar_cluster)
        : "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem of both CTAs] (+)= A[smem of both] * B[smem of both]^T, M = 256
// (each CTA supplies 128 rows of A and N/2 rows of B at the same offsets)
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate)
        : "memory");
}

// arrive on the mbarrier at this offset in every CTA of `mask` when all
// previously issued tcgen05.mma of the pair have completed
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// UMMA shared-memory matrix descriptor (sm_100, "version 1"), 128B swizzle.
// lbo/sbo in bytes. Tile bases must be 1024-byte aligned (base_offset = 0).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;          // version = 1 (sm_100)
    d |= (uint64_t)2 << 61;          // SWIZZLE_128B
    return d;
}

}  // namespace tpipe
