// HBM pool with exact live-byte accounting.
//
// One cudaMalloc arena per stage. Planned mode (what the runtime uses): the
// plan fixes every buffer's lifetime (allocating and releasing instruction),
// so the arena layout is computed once at runtime creation — greedy by size,
// each buffer at the lowest 256-byte-aligned offset not overlapping any
// placed buffer whose lifetime intersects its own — and the arena is exactly
// as large as that layout: no fragmentation at run time, deterministic
// addresses. (Dynamic best-fit mode remains for standalone use.) The ledger
// counts the REQUESTED bytes of every live allocation per stage, at the
// instruction boundaries the plan prescribes, so its high-water equals the
// plan's (and the oracle's) per-stage peak exactly; alignment padding and
// packing slack show up only in the physical `reserved` figure.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <unordered_map>
#include <vector>

namespace tpipe {

struct PoolItem {
    uint64_t bytes;   // requested
    int first, last;  // live from instruction `first` (start) to `last` (end), inclusive
};

class Pool {
public:
    ~Pool() { release(); }
    int init(size_t bytes, int n_stages);
    // planned mode: lay out `items` (indexed by buffer id) and allocate the arena
    int init_planned(const std::vector<PoolItem>& items, int n_stages, bool canary);
    // planned mode: the buffer `id`'s fixed address (ledger updated)
    void* alloc_id(int stage, int id, uint64_t bytes);
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
    size_t overflow_bytes() const { return overflow_bytes_; }
    void set_cap(int stage, uint64_t cap) { limit_[stage] = cap; }
    bool over_cap() const { return over_cap_; }
    // the arena (exported to peer ranks by the IPC transport)
    void* arena() const { return base_; }
    size_t arena_bytes() const { return cap_; }
    // physical bound: a fragmentation overflow block may be cudaMalloc'ed
    // only while arena + overflow stays within `bytes` (0 = unbounded); beyond
    // it alloc() fails (the runtime reports TPIPE_E_OOM) instead of silently
    // exceeding the HBM budget the plan was made for
    void set_phys_limit(size_t bytes) { phys_limit_ = bytes; }
    bool last_fail_physical() const { return last_fail_phys_; }
    // debug canaries (TPIPE_DEBUG_POOL_CANARY): CANARY guard bytes of a fixed
    // pattern right after each allocation's requested bytes, written on
    // `st` at alloc; check_canaries() returns the first live allocation whose
    // guard changed (nullptr if none), after synchronising `st`
    static constexpr size_t CANARY = 512;
    void set_canary(bool on, cudaStream_t st) { canary_ = on; canary_st_ = st; }
    void* check_canaries(cudaStream_t st, uint64_t* req_bytes);

private:
    char* base_ = nullptr;
    size_t cap_ = 0;
    std::map<size_t, size_t> free_;                       // offset -> size
    std::unordered_map<void*, std::pair<size_t, size_t>> used_;  // ptr -> (offset, size)
    std::unordered_map<void*, uint64_t> req_;             // ptr -> requested bytes
    std::vector<void*> overflow_;
    size_t overflow_bytes_ = 0;
    std::vector<uint64_t> cur_, hw_, limit_;
    std::vector<size_t> planned_off_;
    bool over_cap_ = false;
    size_t phys_limit_ = 0;
    bool last_fail_phys_ = false;
    bool canary_ = false;
    cudaStream_t canary_st_ = nullptr;
};

}  // namespace tpipe
