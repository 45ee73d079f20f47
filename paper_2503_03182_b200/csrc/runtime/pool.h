// HBM pool with exact live-byte accounting.
//
// One cudaMalloc arena carved best-fit at 256-byte granularity. The ledger
// counts the REQUESTED bytes of every live allocation per stage, at the
// instruction boundaries the plan prescribes, so its high-water equals the
// plan's (and the oracle's) per-stage peak exactly; alignment padding and
// fragmentation show up only in the physical `reserved` figure.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <unordered_map>
#include <vector>

namespace tpipe {

class Pool {
public:
    ~Pool() { release(); }
    int init(size_t bytes, int n_stages);
    void release();
    // returns nullptr on failure; `cap` (0 = none) bounds the stage's ledger
    void* alloc(int stage, uint64_t bytes);
    void free(int stage, void* p);
    uint64_t live(int stage) const { return cur_[stage]; }
    uint64_t high_water(int stage) const { return hw_[stage]; }
    void reset_high_water() {
        for (size_t s = 0; s < hw_.size(); ++s) hw_[s] = cur_[s];
    }
    size_t reserved() const { return cap_ + overflow_bytes_; }
    void set_cap(int stage, uint64_t cap) { limit_[stage] = cap; }
    bool over_cap() const { return over_cap_; }

private:
    char* base_ = nullptr;
    size_t cap_ = 0;
    std::map<size_t, size_t> free_;                       // offset -> size
    std::unordered_map<void*, std::pair<size_t, size_t>> used_;  // ptr -> (offset, size)
    std::unordered_map<void*, uint64_t> req_;             // ptr -> requested bytes
    std::vector<void*> overflow_;
    size_t overflow_bytes_ = 0;
    std::vector<uint64_t> cur_, hw_, limit_;
    bool over_cap_ = false;
};

}  // namespace tpipe
