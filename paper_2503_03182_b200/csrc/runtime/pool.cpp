#include "runtime/pool.h"

#include <algorithm>

namespace tpipe {

static constexpr size_t ALIGN = 256;
static constexpr unsigned char CANARY_BYTE = 0xA7;

int Pool::init(size_t bytes, int n_stages) {
    release();
    cur_.assign(n_stages, 0);
    hw_.assign(n_stages, 0);
    limit_.assign(n_stages, 0);
    bytes = (bytes + ALIGN - 1) / ALIGN * ALIGN;
    if (bytes) {
        if (cudaMalloc(&base_, bytes) != cudaSuccess) {
            base_ = nullptr;
            return -1;
        }
        cap_ = bytes;
        free_[0] = bytes;
    }
    return 0;
}

int Pool::init_planned(const std::vector<PoolItem>& items, int n_stages, bool canary) {
    release();
    cur_.assign(n_stages, 0);
    hw_.assign(n_stages, 0);
    limit_.assign(n_stages, 0);
    canary_ = canary;
    const size_t n = items.size();
    std::vector<size_t> size(n), order(n);
    for (size_t i = 0; i < n; ++i) {
        const uint64_t phys = items[i].bytes + (canary ? CANARY : 0);
        size[i] = std::max<size_t>(ALIGN, (phys + ALIGN - 1) / ALIGN * ALIGN);
        order[i] = i;
    }
    std::sort(order.begin(), order.end(), [&](size_t x, size_t y) {
        if (size[x] != size[y]) return size[x] > size[y];
        if (items[x].first != items[y].first) return items[x].first < items[y].first;
        return x < y;
    });
    planned_off_.assign(n, 0);
    std::vector<size_t> placed;
    size_t top = 0;
    for (size_t id : order) {
        std::vector<std::pair<size_t, size_t>> busy;   // (offset, size) of lifetime-overlapping buffers
        for (size_t q : placed)
            if (!(items[q].last < items[id].first || items[id].last < items[q].first))
                busy.push_back({planned_off_[q], size[q]});
        std::sort(busy.begin(), busy.end());
        size_t cand = 0;
        for (auto& b : busy) {
            if (cand + size[id] <= b.first) break;
            cand = std::max(cand, b.first + b.second);
        }
        planned_off_[id] = cand;
        top = std::max(top, cand + size[id]);
        placed.push_back(id);
    }
    if (top) {
        if (cudaMalloc(&base_, top) != cudaSuccess) {
            base_ = nullptr;
            return -1;
        }
        cap_ = top;
    }
    return 0;
}

void* Pool::alloc_id(int stage, int id, uint64_t bytes) {
    if (id < 0 || (size_t)id >= planned_off_.size() || !base_) return nullptr;
    void* p = base_ + planned_off_[id];
    req_[p] = bytes;
    used_[p] = {planned_off_[id], 0};
    if (canary_) cudaMemsetAsync((char*)p + bytes, CANARY_BYTE, CANARY, canary_st_);
    cur_[stage] += bytes;
    hw_[stage] = std::max(hw_[stage], cur_[stage]);
    if (limit_[stage] && cur_[stage] > limit_[stage]) over_cap_ = true;
    return p;
}

void Pool::release() {
    if (base_) cudaFree(base_);
    for (void* p : overflow_) cudaFree(p);
    base_ = nullptr;
    cap_ = 0;
    overflow_.clear();
    overflow_bytes_ = 0;
    planned_off_.clear();
    free_.clear();
    used_.clear();
    req_.clear();
}


void* Pool::alloc(int stage, uint64_t bytes) {
    last_fail_phys_ = false;
    const uint64_t phys = bytes + (canary_ ? CANARY : 0);
    const size_t need = std::max<size_t>(ALIGN, (phys + ALIGN - 1) / ALIGN * ALIGN);
    // best fit
    auto best = free_.end();
    for (auto it = free_.begin(); it != free_.end(); ++it)
        if (it->second >= need && (best == free_.end() || it->second < best->second)) best = it;
    void* p = nullptr;
    if (best != free_.end()) {
        const size_t off = best->first, sz = best->second;
        free_.erase(best);
        if (sz > need) free_[off + need] = sz - need;
        p = base_ + off;
        used_[p] = {off, need};
    } else {
        // arena exhausted by fragmentation: dedicated block (physical only; the
        // ledger below is unaffected), bounded by the physical limit
        if (phys_limit_ && std::max(cap_, phys_limit_) < cap_ + overflow_bytes_ + need) {
            last_fail_phys_ = true;
            return nullptr;
        }
        if (cudaMalloc(&p, need) != cudaSuccess) return nullptr;
        overflow_.push_back(p);
        overflow_bytes_ += need;
        used_[p] = {SIZE_MAX, need};
    }
    req_[p] = bytes;
    if (canary_) cudaMemsetAsync((char*)p + bytes, CANARY_BYTE, CANARY, canary_st_);
    cur_[stage] += bytes;
    hw_[stage] = std::max(hw_[stage], cur_[stage]);
    if (limit_[stage] && cur_[stage] > limit_[stage]) over_cap_ = true;
    return p;
}

void Pool::free(int stage, void* p) {
    auto it = used_.find(p);
    if (it == used_.end()) return;
    const size_t off = it->second.first, sz = it->second.second;
    used_.erase(it);
    cur_[stage] -= req_[p];
    req_.erase(p);
    if (!planned_off_.empty()) return;   // planned mode: addresses are fixed, nothing to merge
    if (off == SIZE_MAX) {
        cudaFree(p);
        overflow_.erase(std::find(overflow_.begin(), overflow_.end(), p));
        overflow_bytes_ -= sz;
        return;
    }
    size_t o = off, s = sz;
    auto nxt = free_.lower_bound(o);
    if (nxt != free_.end() && nxt->first == o + s) {
        s += nxt->second;
        nxt = free_.erase(nxt);
    }
    if (nxt != free_.begin()) {
        auto prv = std::prev(nxt);
        if (prv->first + prv->second == o) {
            o = prv->first;
            s += prv->second;
            free_.erase(prv);
        }
    }
    free_[o] = s;
}

void* Pool::check_canaries(cudaStream_t st, uint64_t* req_bytes) {
    if (!canary_) return nullptr;
    cudaStreamSynchronize(st);
    std::vector<unsigned char> g(CANARY);
    for (auto& kv : req_) {
        if (cudaMemcpy(g.data(), (char*)kv.first + kv.second, CANARY, cudaMemcpyDeviceToHost) != cudaSuccess)
            return kv.first;
        for (unsigned char x : g)
            if (x != CANARY_BYTE) {
                if (req_bytes) *req_bytes = kv.second;
                return kv.first;
            }
    }
    return nullptr;
}

}  // namespace tpipe
