// Host AdamW for T-Offload ("performing its optimizer
// updates" on the CPU in the cooldown bubble). Same element arithmetic as the
// device kernel (adam_math.h), compiled with -ffp-contract=off, so the result
// is bit-identical to tpipe::adamw on the GPU. Multithreaded over contiguous
// slices (order of elements is irrelevant: the update is elementwise).
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "kernels/adam_math.h"

namespace tpipe {

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // quiet NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// branch-free RNE (vectorisable); NaN -> quiet NaN as above
static inline uint16_t f32_to_bf16_rne_v(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t r = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
    const uint32_t q = (u >> 16) | 0x40u;
    return (uint16_t)(((u & 0x7fffffffu) > 0x7f800000u) ? q : r);
}

// The loop is compiled -O3 -fno-math-errno (sqrt inline) with FMA contraction
// off, in AVX-512 / AVX2 / baseline clones picked at load time: vector
// mul/add/div/sqrt are correctly rounded IEEE ops, so every clone is
// bit-identical to the scalar arithmetic and to the device kernel.
__attribute__((target_clones("avx512f", "avx2", "default")))
static void adamw_host_range(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                             const float* __restrict__ grad, uint16_t* __restrict__ w_bf16, long lo, long hi,
                             int decay, const AdamHyper& hp) {
    const AdamHyper h = hp;
    if (w_bf16) {
        for (long i = lo; i < hi; ++i) {
            AdamOut o = adam_elem(master[i], m[i], v[i], grad[i], decay, h);
            master[i] = o.w;
            m[i] = o.m;
            v[i] = o.v;
            w_bf16[i] = f32_to_bf16_rne_v(o.w);
        }
    } else {
        for (long i = lo; i < hi; ++i) {
            AdamOut o = adam_elem(master[i], m[i], v[i], grad[i], decay, h);
            master[i] = o.w;
            m[i] = o.m;
            v[i] = o.v;
        }
    }
}

static std::atomic<long> g_launches{0};
void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long launch_count() { return g_launches.load(std::memory_order_relaxed); }

void host_cast_bf16(const float* src, uint16_t* dst, long n) {
    for (long i = 0; i < n; ++i) dst[i] = f32_to_bf16_rne(src[i]);
}

void adamw_host(float* master, float* m, float* v, const float* grad, uint16_t* w_bf16, long n,
                int decay, const AdamHyper& hp) {
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    if (nt > 32) nt = 32;
    if (n < (1L << 16)) nt = 1;
    if (nt == 1) {
        adamw_host_range(master, m, v, grad, w_bf16, 0, n, decay, hp);
        return;
    }
    std::vector<std::thread> th;
    const long chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const long lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        th.emplace_back(adamw_host_range, master, m, v, grad, w_bf16, lo, hi, decay, std::cref(hp));
    }
    for (auto& x : th) x.join();
}

}  // namespace tpipe
