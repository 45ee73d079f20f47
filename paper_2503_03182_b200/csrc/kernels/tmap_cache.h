// Host-side cache of 2-D TMA tensor maps. The runtime's buffers have fixed
// addresses (planned pool arena, runtime/pool.h), so every step encodes the
// same maps again; cuTensorMapEncodeTiled is a driver call on the launch
// path of every GEMM / attention kernel (3-4 maps per GEMM launch, ~9,300
// GEMM launches per C2 step). The cache returns the encoded 128-byte map for
// an identical request. Bounded: cleared when it exceeds MAX_ENTRIES.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <unordered_map>

namespace tpipe {

struct TmapKey {
    const void* base;
    uint64_t cols, rows, ld_bytes;
    uint32_t box0, box1;
    int dtype, swizzle;
    bool operator==(const TmapKey& o) const { return std::memcmp(this, &o, sizeof(TmapKey)) == 0; }
};
struct TmapKeyHash {
    size_t operator()(const TmapKey& k) const {
        const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
        uint64_t h = 1469598103934665603ull;
        for (size_t i = 0; i < sizeof(TmapKey) / 8; ++i) h = (h ^ w[i]) * 1099511628211ull;
        return (size_t)h;
    }
};

template <typename EncodeFn>
inline CUresult tmap_encode_2d_cached(EncodeFn enc, CUtensorMap* out, CUtensorMapDataType dt, const void* base,
                                      uint64_t cols, uint64_t rows, uint64_t ld_bytes, uint32_t box0,
                                      uint32_t box1, CUtensorMapSwizzle sw) {
    static std::mutex mu;
    static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
    constexpr size_t MAX_ENTRIES = 1 << 18;
    TmapKey k;
    std::memset(&k, 0, sizeof(k));
    k.base = base;
    k.cols = cols;
    k.rows = rows;
    k.ld_bytes = ld_bytes;
    k.box0 = box0;
    k.box1 = box1;
    k.dtype = (int)dt;
    k.swizzle = (int)sw;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(k);
        if (it != cache.end()) {
            *out = it->second;
            return CUDA_SUCCESS;
        }
    }
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld_bytes};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(out, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS) {
        std::lock_guard<std::mutex> lk(mu);
        if (cache.size() >= MAX_ENTRIES) cache.clear();
        cache.emplace(k, *out);
    }
    return r;
}

}  // namespace tpipe
