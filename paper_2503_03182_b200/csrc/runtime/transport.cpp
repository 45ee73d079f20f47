// Stage transport implementations (see transport.h).
#include "runtime/transport.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <deque>
#include <map>
#include <thread>

#include "runtime/errors.h"
#include "runtime/nccl_dl.h"
#include "tpipe.h"

namespace tpipe {

using Clock = std::chrono::steady_clock;

static double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// poll-wait: spin briefly, then sleep in short steps (the waits are on other
// processes' host progress, normally microseconds to milliseconds)
template <typename Pred, typename Abort>
static int poll_until(Pred pred, Abort aborted, int timeout_ms, const char* what) {
    const auto t0 = Clock::now();
    for (int it = 0;; ++it) {
        if (pred()) return 0;
        if (aborted()) return set_error(TPIPE_E_STATE, "%s: a peer rank aborted", what);
        if (it > 256) {
            if (ms_since(t0) > timeout_ms)
                return set_error(TPIPE_E_TIMEOUT, "%s: timed out after %d ms", what, timeout_ms);
            std::this_thread::sleep_for(std::chrono::microseconds(it < 4096 ? 2 : 50));
        }
    }
}

int Transport::sync(cudaStream_t cs, int timeout_ms) {
    const auto t0 = Clock::now();
    for (;;) {
        cudaError_t e = cudaStreamQuery(cs);
        if (e == cudaSuccess) return 0;
        if (e != cudaErrorNotReady)
            return set_error(TPIPE_E_CUDA, "step stream: %s", cudaGetErrorString(e));
        if (ms_since(t0) > timeout_ms)
            return set_error(TPIPE_E_TIMEOUT, "step did not complete within %d ms", timeout_ms);
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// ================================================================ virtual
namespace {

class VirtualTransport final : public Transport {
public:
    // each stage may run on its own stream: a message carries the sender's
    // "ready" event, the receiver copies after it and records "done", which
    // the sender's SEND_WAIT waits for before the buffer is reused
    struct Msg {
        const void* src;
        cudaEvent_t ready;
    };
    explicit VirtualTransport(size_t n) : q_(n), popped_(n, 0), done_(n) {}
    ~VirtualTransport() override {
        for (auto e : ev_) cudaEventDestroy(e);
        if (comm_) {
            if (aborted_ && nccl()->CommAbort) nccl()->CommAbort(comm_);
            else nccl()->CommDestroy(comm_);
        }
    }
    const char* name() const override { return comm_ ? "virtual-nccl" : "virtual"; }
    void begin_step() override {
        for (auto& q : q_) q.clear();
        for (auto& n : popped_) n = 0;
        for (auto& d : done_) d.clear();
        evnext_ = 0;
    }
    cudaEvent_t ev() {
        if (evnext_ == ev_.size()) {
            cudaEvent_t e;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            ev_.push_back(e);
        }
        return ev_[evnext_++];
    }
    int send(int ch, int, const void* src, size_t, cudaStream_t cs) override {
        cudaEvent_t e = ev();
        if (cudaEventRecord(e, cs)) return set_error(TPIPE_E_CUDA, "virtual send: event");
        q_[ch].push_back({src, e});
        return 0;
    }
    int recv(int ch, void* dst, size_t bytes, cudaStream_t cs) override {
        if (q_[ch].empty()) return set_error(TPIPE_E_STATE, "virtual recv on an empty channel %d", ch);
        const Msg mg = q_[ch].front();
        q_[ch].pop_front();
        cudaEvent_t d = ev();
        cudaError_t e = cudaStreamWaitEvent(cs, mg.ready, 0);
        if (!e && comm_) {
            // loopback: the message travels as an ncclSend / ncclRecv pair on
            // the one-rank communicator (rank 0 to itself), on the receiver's stream
            const NcclApi* N = nccl();
            ncclResult_t r = N->GroupStart();
            if (r == ncclSuccess) r = N->Send(mg.src, bytes, ncclUint8, 0, comm_, cs);
            if (r == ncclSuccess) r = N->Recv(dst, bytes, ncclUint8, 0, comm_, cs);
            const ncclResult_t r2 = N->GroupEnd();
            if (r == ncclSuccess) r = r2;
            if (r != ncclSuccess) return set_error(TPIPE_E_NCCL, "loopback ncclSend/ncclRecv: %s", N->GetErrorString(r));
        } else if (!e) {
            e = cudaMemcpyAsync(dst, mg.src, bytes, cudaMemcpyDeviceToDevice, cs);
        }
        if (!e) e = cudaEventRecord(d, cs);
        if (e) return set_error(TPIPE_E_CUDA, "virtual recv copy: %s", cudaGetErrorString(e));
        done_[ch].push_back(d);
        popped_[ch]++;
        return 0;
    }
    int send_wait(int ch, int msg, cudaStream_t cs) override {
        if (msg >= (int)done_[ch].size()) return set_error(TPIPE_E_STATE, "virtual SEND_WAIT before RECV");
        return cudaStreamWaitEvent(cs, done_[ch][msg], 0) ? set_error(TPIPE_E_CUDA, "send_wait") : 0;
    }
    bool recv_ready(int ch) const override { return !q_[ch].empty(); }
    bool send_wait_ready(int ch, int msg) const override { return popped_[ch] > msg; }
    int sync(cudaStream_t cs, int timeout_ms) override {
        if (!comm_) return Transport::sync(cs, timeout_ms);
        const NcclApi* N = nccl();
        const auto t0 = Clock::now();
        for (;;) {
            cudaError_t e = cudaStreamQuery(cs);
            if (e == cudaSuccess) return 0;
            if (e != cudaErrorNotReady) return set_error(TPIPE_E_CUDA, "step stream: %s", cudaGetErrorString(e));
            ncclResult_t ae = ncclSuccess;
            if (N->CommGetAsyncError && N->CommGetAsyncError(comm_, &ae) == ncclSuccess && ae != ncclSuccess &&
                ae != ncclInProgress) {
                abort();
                return set_error(TPIPE_E_NCCL, "NCCL asynchronous error: %s", N->GetErrorString(ae));
            }
            if (ms_since(t0) > timeout_ms) {
                abort();
                return set_error(TPIPE_E_TIMEOUT, "step did not complete within %d ms", timeout_ms);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    void abort() override { aborted_ = true; }

    ncclComm_t comm_ = nullptr;   // NCCL loopback (TPIPE_TRANSPORT_NCCL_LOOPBACK)
    bool aborted_ = false;

private:
    std::vector<std::deque<Msg>> q_;
    std::vector<int> popped_;
    std::vector<std::vector<cudaEvent_t>> done_;
    std::vector<cudaEvent_t> ev_;
    size_t evnext_ = 0;
};

// ================================================================ nccl
class NcclTransport final : public Transport {
public:
    struct Ch {
        ncclComm_t comm = nullptr;
        cudaStream_t st = nullptr;
        std::vector<cudaEvent_t> done;   // per message of the step
    };
    ~NcclTransport() override {
        const NcclApi* N = nccl();
        for (auto& c : ch_) {
            if (c.comm && N) {
                if (aborted_ && N->CommAbort) N->CommAbort(c.comm);
                else N->CommDestroy(c.comm);
            }
            if (c.st) cudaStreamDestroy(c.st);
        }
        for (auto e : ev_) cudaEventDestroy(e);
    }
    const char* name() const override { return "nccl"; }
    void begin_step() override {
        evnext_ = 0;
        for (auto& c : ch_) c.done.clear();
    }
    cudaEvent_t ev() {
        if (evnext_ == ev_.size()) {
            cudaEvent_t e;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            ev_.push_back(e);
        }
        return ev_[evnext_++];
    }
    int send(int ch, int msg, const void* src, size_t bytes, cudaStream_t cs) override {
        Ch& c = ch_[ch];
        const NcclApi* N = nccl();
        cudaEvent_t e0 = ev();
        if (cudaEventRecord(e0, cs) || cudaStreamWaitEvent(c.st, e0, 0))
            return set_error(TPIPE_E_CUDA, "nccl send: event");
        ncclResult_t r = N->Send(src, bytes, ncclUint8, 1, c.comm, c.st);
        if (r != ncclSuccess) return set_error(TPIPE_E_NCCL, "ncclSend: %s", N->GetErrorString(r));
        if ((int)c.done.size() <= msg) c.done.resize(msg + 1, nullptr);
        c.done[msg] = ev();
        if (cudaEventRecord(c.done[msg], c.st)) return set_error(TPIPE_E_CUDA, "nccl send: event");
        return 0;
    }
    int recv(int ch, void* dst, size_t bytes, cudaStream_t cs) override {
        Ch& c = ch_[ch];
        const NcclApi* N = nccl();
        cudaEvent_t e0 = ev(), e1 = ev();
        if (cudaEventRecord(e0, cs) || cudaStreamWaitEvent(c.st, e0, 0))
            return set_error(TPIPE_E_CUDA, "nccl recv: event");
        ncclResult_t r = N->Recv(dst, bytes, ncclUint8, 0, c.comm, c.st);
        if (r != ncclSuccess) return set_error(TPIPE_E_NCCL, "ncclRecv: %s", N->GetErrorString(r));
        if (cudaEventRecord(e1, c.st) || cudaStreamWaitEvent(cs, e1, 0))
            return set_error(TPIPE_E_CUDA, "nccl recv: event");
        return 0;
    }
    int send_wait(int ch, int msg, cudaStream_t cs) override {
        Ch& c = ch_[ch];
        if (msg >= (int)c.done.size() || !c.done[msg])
            return set_error(TPIPE_E_STATE, "SEND_WAIT(%d) on channel %d before its SEND", msg, ch);
        return cudaStreamWaitEvent(cs, c.done[msg], 0) ? set_error(TPIPE_E_CUDA, "send_wait") : 0;
    }
    // step completion with asynchronous-error polling (a failed or hung peer
    // surfaces as an error instead of a silent hang)
    int sync(cudaStream_t cs, int timeout_ms) override {
        const NcclApi* N = nccl();
        const auto t0 = Clock::now();
        for (;;) {
            cudaError_t e = cudaStreamQuery(cs);
            if (e == cudaSuccess) return 0;
            if (e != cudaErrorNotReady) return set_error(TPIPE_E_CUDA, "step stream: %s", cudaGetErrorString(e));
            for (auto& c : ch_) {
                if (!c.comm) continue;
                ncclResult_t ae = ncclSuccess;
                if (N->CommGetAsyncError && N->CommGetAsyncError(c.comm, &ae) == ncclSuccess &&
                    ae != ncclSuccess && ae != ncclInProgress) {
                    abort();
                    return set_error(TPIPE_E_NCCL, "NCCL asynchronous error: %s", N->GetErrorString(ae));
                }
            }
            if (ms_since(t0) > timeout_ms) {
                abort();
                return set_error(TPIPE_E_TIMEOUT, "step did not complete within %d ms (NCCL peers hung?)",
                                 timeout_ms);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    void abort() override { aborted_ = true; }

    std::vector<Ch> ch_;
    std::vector<cudaEvent_t> ev_;
    size_t evnext_ = 0;
    bool aborted_ = false;
};

// ================================================================ ipc
constexpr int RING = 4;
constexpr uint64_t SHM_MAGIC = 0x7470697065495043ull;   // "tpipeIPC"

struct alignas(64) ShmSlot {
    std::atomic<uint64_t> posted;     // sender: 1 + global message index
    uint64_t offset, bytes;           // message location in the sender's arena
};
struct alignas(64) ShmCons {
    std::atomic<uint64_t> consumed;   // receiver: 1 + global index whose copy is issued
};
struct ShmChan {
    cudaIpcEventHandle_t ready[RING];     // sender-owned
    cudaIpcEventHandle_t used[RING];      // receiver-owned
    ShmSlot slot[RING];
    ShmCons cons[RING];
};
struct alignas(64) ShmRank {
    cudaIpcMemHandle_t arena;
    uint64_t arena_bytes;
    int32_t device, pid;
};
struct alignas(64) ShmHeader {
    std::atomic<uint64_t> magic;
    std::atomic<int32_t> p, n_ch;
    std::atomic<int32_t> arrived;
    std::atomic<int32_t> abort;
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "shared-memory atomics");

static size_t shm_size(int p, int n_ch) {
    return sizeof(ShmHeader) + (size_t)p * sizeof(ShmRank) + (size_t)n_ch * sizeof(ShmChan);
}

class IpcTransport final : public Transport {
public:
    struct Ch {
        int src = 0, dst = 0;
        bool out = false, in = false;
        cudaStream_t st = nullptr;
        cudaEvent_t own[RING] = {};       // sender: ready; receiver: used
        cudaEvent_t peer[RING] = {};      // sender: peer's used; receiver: peer's ready
        uint64_t sent = 0, base = 0, recvd = 0;
        uint8_t* peer_arena = nullptr;
    };
    ~IpcTransport() override {
        for (auto& c : ch_) {
            for (int r = 0; r < RING; ++r) {
                if (c.own[r]) cudaEventDestroy(c.own[r]);
                if (c.peer[r]) cudaEventDestroy(c.peer[r]);
            }
            if (c.st) cudaStreamDestroy(c.st);
        }
        for (auto& kv : peer_arena_) cudaIpcCloseMemHandle(kv.second);
        for (auto e : ev_) cudaEventDestroy(e);
        if (shm_) munmap(shm_, shm_bytes_);
    }
    const char* name() const override { return "ipc"; }
    void begin_step() override {
        evnext_ = 0;
        for (auto& c : ch_) c.base = c.sent;
    }
    cudaEvent_t ev() {
        if (evnext_ == ev_.size()) {
            cudaEvent_t e;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            ev_.push_back(e);
        }
        return ev_[evnext_++];
    }
    bool aborted() const { return hdr()->abort.load(std::memory_order_acquire) != 0; }
    int send(int ch, int msg, const void* src, size_t bytes, cudaStream_t cs) override {
        Ch& c = ch_[ch];
        const uint64_t n = c.base + (uint64_t)msg;
        if (!c.out || n != c.sent)
            return set_error(TPIPE_E_STATE, "ipc send: channel %d message %d out of order", ch, msg);
        const uint8_t* p = (const uint8_t*)src;
        if (p < arena_ || p + bytes > arena_ + arena_bytes_)
            return set_error(TPIPE_E_STATE, "ipc send: message buffer outside the exported pool arena");
        const int r = (int)(n % RING);
        ShmChan& S = chan(ch);
        // the slot's previous message (n - RING) must have been picked up; the
        // plan's send window W <= RING already guarantees it (defensive)
        if (n >= RING)
            if (int rc = poll_until([&] { return S.cons[r].consumed.load(std::memory_order_acquire) >= n - RING + 1; },
                                    [&] { return aborted(); }, timeout_ms_, "ipc send slot"))
                return rc;
        if (cudaEventRecord(c.own[r], cs)) return set_error(TPIPE_E_CUDA, "ipc send: event record");
        S.slot[r].offset = (uint64_t)(p - arena_);
        S.slot[r].bytes = bytes;
        S.slot[r].posted.store(n + 1, std::memory_order_release);
        c.sent++;
        return 0;
    }
    int recv(int ch, void* dst, size_t bytes, cudaStream_t cs) override {
        Ch& c = ch_[ch];
        if (!c.in) return set_error(TPIPE_E_STATE, "ipc recv: channel %d not inbound", ch);
        const uint64_t n = c.recvd;
        const int r = (int)(n % RING);
        ShmChan& S = chan(ch);
        if (int rc = poll_until([&] { return S.slot[r].posted.load(std::memory_order_acquire) == n + 1; },
                                [&] { return aborted(); }, timeout_ms_, "ipc recv"))
            return rc;
        if (S.slot[r].bytes != bytes)
            return set_error(TPIPE_E_STATE, "ipc recv: %llu-byte message, expected %zu",
                             (unsigned long long)S.slot[r].bytes, bytes);
        const uint8_t* src = c.peer_arena + S.slot[r].offset;
        cudaEvent_t e0 = ev();
        cudaError_t e = cudaEventRecord(e0, cs);                      // dst is free for writing
        if (!e) e = cudaStreamWaitEvent(c.st, e0, 0);
        if (!e) e = cudaStreamWaitEvent(c.st, c.peer[r], 0);          // the sender's message is complete
        if (!e) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c.st);   // copy-engine pull
        if (!e) e = cudaEventRecord(c.own[r], c.st);
        if (!e) e = cudaStreamWaitEvent(cs, c.own[r], 0);
        if (e) return set_error(TPIPE_E_CUDA, "ipc recv: %s", cudaGetErrorString(e));
        S.cons[r].consumed.store(n + 1, std::memory_order_release);
        c.recvd++;
        return 0;
    }
    int send_wait(int ch, int msg, cudaStream_t cs) override {
        Ch& c = ch_[ch];
        const uint64_t n = c.base + (uint64_t)msg;
        if (!c.out || n >= c.sent) return set_error(TPIPE_E_STATE, "ipc SEND_WAIT(%d) before its SEND", msg);
        const int r = (int)(n % RING);
        ShmChan& S = chan(ch);
        if (int rc = poll_until([&] { return S.cons[r].consumed.load(std::memory_order_acquire) >= n + 1; },
                                [&] { return aborted(); }, timeout_ms_, "ipc send_wait"))
            return rc;
        return cudaStreamWaitEvent(cs, c.peer[r], 0) ? set_error(TPIPE_E_CUDA, "ipc send_wait") : 0;
    }
    int sync(cudaStream_t cs, int timeout_ms) override {
        const auto t0 = Clock::now();
        for (;;) {
            cudaError_t e = cudaStreamQuery(cs);
            if (e == cudaSuccess) return 0;
            if (e != cudaErrorNotReady) return set_error(TPIPE_E_CUDA, "step stream: %s", cudaGetErrorString(e));
            if (aborted()) return set_error(TPIPE_E_STATE, "a peer rank aborted the step");
            if (ms_since(t0) > timeout_ms) {
                abort();
                return set_error(TPIPE_E_TIMEOUT, "step did not complete within %d ms", timeout_ms);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    void abort() override {
        if (shm_) hdr()->abort.store(1, std::memory_order_release);
    }

    ShmHeader* hdr() const { return (ShmHeader*)shm_; }
    ShmRank& rank(int s) const { return ((ShmRank*)(shm_ + sizeof(ShmHeader)))[s]; }
    ShmChan& chan(int c) const {
        return ((ShmChan*)(shm_ + sizeof(ShmHeader) + (size_t)p_ * sizeof(ShmRank)))[c];
    }

    int init(const ChannelList& chl, int p, int stage, int device, const char* name, void* arena,
             size_t arena_bytes, int window, int timeout_ms) {
        p_ = p;
        timeout_ms_ = timeout_ms;
        arena_ = (uint8_t*)arena;
        arena_bytes_ = arena_bytes;
        if (!name || !name[0] || name[0] != '/')
            return set_error(TPIPE_E_INVALID, "ipc_name must be a POSIX shm name starting with '/'");
        if (window > RING) return set_error(TPIPE_E_INVALID, "send window %d > ipc mailbox ring %d", window, RING);
        shm_bytes_ = shm_size(p, (int)chl.size());
        int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
        if (fd < 0) return set_error(TPIPE_E_INVALID, "shm_open(%s): %s", name, strerror(errno));
        if (ftruncate(fd, (off_t)shm_bytes_) != 0) {
            close(fd);
            return set_error(TPIPE_E_INVALID, "ftruncate(%s): %s", name, strerror(errno));
        }
        void* m = mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) return set_error(TPIPE_E_INVALID, "mmap(%s): %s", name, strerror(errno));
        shm_ = (uint8_t*)m;
        ShmHeader* H = hdr();
        uint64_t zero = 0;
        if (H->magic.compare_exchange_strong(zero, SHM_MAGIC)) {
            H->p.store(p);
            H->n_ch.store((int)chl.size());
        } else if (zero != SHM_MAGIC) {
            return set_error(TPIPE_E_INVALID, "shm %s holds foreign data", name);
        }
        // publish this rank's arena and events
        ShmRank& me = rank(stage);
        if (cudaIpcGetMemHandle(&me.arena, arena) != cudaSuccess)
            return set_error(TPIPE_E_CUDA, "cudaIpcGetMemHandle of the pool arena failed");
        me.arena_bytes = arena_bytes;
        me.device = device;
        me.pid = (int32_t)getpid();
        ch_.resize(chl.size());
        for (size_t k = 0; k < chl.size(); ++k) {
            Ch& c = ch_[k];
            c.src = chl[k][1];
            c.dst = chl[k][2];
            c.out = c.src == stage;
            c.in = c.dst == stage;
            if (!c.out && !c.in) continue;
            for (int r = 0; r < RING; ++r) {
                if (cudaEventCreateWithFlags(&c.own[r], cudaEventDisableTiming | cudaEventInterprocess))
                    return set_error(TPIPE_E_CUDA, "interprocess event");
                cudaIpcEventHandle_t* h = c.out ? &chan((int)k).ready[r] : &chan((int)k).used[r];
                if (cudaIpcGetEventHandle(h, c.own[r])) return set_error(TPIPE_E_CUDA, "cudaIpcGetEventHandle");
            }
            if (c.in && cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking))
                return set_error(TPIPE_E_CUDA, "ipc channel stream");
        }
        std::atomic_thread_fence(std::memory_order_seq_cst);
        H->arrived.fetch_add(1, std::memory_order_acq_rel);
        if (int rc = poll_until([&] { return H->arrived.load(std::memory_order_acquire) >= p; },
                                [&] { return aborted(); }, timeout_ms, "ipc rendezvous"))
            return rc;
        if (H->p.load() != p || H->n_ch.load() != (int)chl.size())
            return set_error(TPIPE_E_INVALID, "ipc rendezvous: ranks disagree on the plan (p, channels)");
        if (stage == 0) shm_unlink(name);   // every rank has it mapped; the name is no longer needed
        // open the peers' arenas and events
        for (size_t k = 0; k < chl.size(); ++k) {
            Ch& c = ch_[k];
            if (!c.out && !c.in) continue;
            const int peer = c.out ? c.dst : c.src;
            for (int r = 0; r < RING; ++r) {
                cudaIpcEventHandle_t h = c.out ? chan((int)k).used[r] : chan((int)k).ready[r];
                if (cudaIpcOpenEventHandle(&c.peer[r], h))
                    return set_error(TPIPE_E_CUDA, "cudaIpcOpenEventHandle (peer %d)", peer);
            }
            if (c.in) {
                auto it = peer_arena_.find(peer);
                if (it == peer_arena_.end()) {
                    void* pa = nullptr;
                    cudaError_t e = cudaIpcOpenMemHandle(&pa, rank(peer).arena, cudaIpcMemLazyEnablePeerAccess);
                    if (e) return set_error(TPIPE_E_CUDA, "cudaIpcOpenMemHandle (peer %d): %s", peer,
                                            cudaGetErrorString(e));
                    it = peer_arena_.emplace(peer, pa).first;
                }
                c.peer_arena = (uint8_t*)it->second;
            }
        }
        return 0;
    }

    std::vector<Ch> ch_;
    std::map<int, void*> peer_arena_;
    std::vector<cudaEvent_t> ev_;
    size_t evnext_ = 0;
    uint8_t* shm_ = nullptr;
    size_t shm_bytes_ = 0;
    uint8_t* arena_ = nullptr;
    size_t arena_bytes_ = 0;
    int p_ = 0, timeout_ms_ = 0;
};

}  // namespace

std::unique_ptr<Transport> make_virtual_transport(const ChannelList& ch) {
    return std::unique_ptr<Transport>(new VirtualTransport(ch.size()));
}

int make_virtual_nccl_transport(const ChannelList& ch, std::unique_ptr<Transport>* out) {
    const NcclApi* N = nccl();
    if (!N) return set_error(TPIPE_E_NCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    ncclResult_t r = N->GetUniqueId(&id);
    if (r != ncclSuccess) return set_error(TPIPE_E_NCCL, "ncclGetUniqueId: %s", N->GetErrorString(r));
    std::unique_ptr<VirtualTransport> T(new VirtualTransport(ch.size()));
    r = N->CommInitRank(&T->comm_, 1, id, 0);
    if (r != ncclSuccess) {
        T->comm_ = nullptr;
        return set_error(TPIPE_E_NCCL, "ncclCommInitRank (1 rank): %s", N->GetErrorString(r));
    }
    *out = std::move(T);
    return 0;
}

int make_nccl_transport(const ChannelList& chl, int stage, const void* ids_, int timeout_ms,
                        std::unique_ptr<Transport>* out) {
    (void)timeout_ms;
    const NcclApi* N = nccl();
    if (!N) return set_error(TPIPE_E_NCCL, "libnccl.so.2 not loadable");
    if (!ids_) return set_error(TPIPE_E_INVALID, "nccl_ids required for the NCCL transport");
    const ncclUniqueId* ids = (const ncclUniqueId*)ids_;
    std::unique_ptr<NcclTransport> T(new NcclTransport);
    T->ch_.resize(chl.size());
    N->GroupStart();
    for (size_t c = 0; c < chl.size(); ++c) {
        const int src = chl[c][1], dst = chl[c][2];
        if (src != stage && dst != stage) continue;
        auto& C = T->ch_[c];
        if (cudaStreamCreateWithFlags(&C.st, cudaStreamNonBlocking)) {
            N->GroupEnd();
            return set_error(TPIPE_E_CUDA, "nccl channel stream");
        }
        ncclResult_t r = N->CommInitRank(&C.comm, 2, ids[c], src == stage ? 0 : 1);
        if (r != ncclSuccess && r != ncclInProgress) {
            N->GroupEnd();
            return set_error(TPIPE_E_NCCL, "ncclCommInitRank: %s", N->GetErrorString(r));
        }
    }
    ncclResult_t r = N->GroupEnd();
    if (r != ncclSuccess) return set_error(TPIPE_E_NCCL, "ncclGroupEnd: %s", N->GetErrorString(r));
    *out = std::move(T);
    return 0;
}

int make_ipc_transport(const ChannelList& ch, int p, int stage, int device, const char* shm_name,
                       void* arena, size_t arena_bytes, int window, int timeout_ms,
                       std::unique_ptr<Transport>* out) {
    std::unique_ptr<IpcTransport> T(new IpcTransport);
    int rc = T->init(ch, p, stage, device, shm_name, arena, arena_bytes, window, timeout_ms);
    if (rc) {
        T->abort();
        return rc;
    }
    *out = std::move(T);
    return 0;
}

// ================================================================ dp group
namespace {

constexpr int DP_MAX = 64;
struct alignas(64) DpMember {
    cudaIpcMemHandle_t arena;
    uint64_t arena_bytes;
    uint64_t w_off[5], g_off[5];
    cudaIpcEventHandle_t ready[5], done[5];
    std::atomic<uint64_t> ready_seq[5], done_seq[5];
};
struct alignas(64) DpHeader {
    std::atomic<uint64_t> magic;
    std::atomic<int32_t> dp, v;
    std::atomic<int32_t> arrived;
    std::atomic<int32_t> abort;
};
constexpr uint64_t DP_MAGIC = 0x7470697065445030ull;

class IpcDpGroup final : public DpGroup {
public:
    ~IpcDpGroup() override {
        for (int j = 0; j < dp_; ++j)
            for (int c = 0; c < 5; ++c) {
                if (ev_ready_[j][c]) cudaEventDestroy(ev_ready_[j][c]);
                if (ev_done_[j][c]) cudaEventDestroy(ev_done_[j][c]);
            }
        for (int j = 0; j < dp_; ++j)
            if (j != rank_ && peer_arena_[j]) cudaIpcCloseMemHandle(peer_arena_[j]);
        if (shm_) munmap(shm_, shm_bytes_);
    }
    int dp() const override { return dp_; }
    int rank() const override { return rank_; }
    DpHeader* hdr() const { return (DpHeader*)shm_; }
    DpMember& mem(int j) const { return ((DpMember*)(shm_ + sizeof(DpHeader)))[j]; }
    bool aborted() const { return hdr()->abort.load(std::memory_order_acquire) != 0; }
    void abort() override {
        if (shm_) hdr()->abort.store(1, std::memory_order_release);
    }
    int post(cudaEvent_t e, std::atomic<uint64_t>& slot, uint64_t seq, cudaStream_t cs) {
        if (cudaEventRecord(e, cs)) return set_error(TPIPE_E_CUDA, "dp: event record");
        slot.store(seq, std::memory_order_release);
        return 0;
    }
    int wait_all(bool ready, int c, uint64_t seq, cudaStream_t cs) {
        for (int j = 0; j < dp_; ++j) {
            if (j == rank_) continue;
            std::atomic<uint64_t>& s = ready ? mem(j).ready_seq[c] : mem(j).done_seq[c];
            if (int rc = poll_until([&] { return s.load(std::memory_order_acquire) >= seq; },
                                    [&] { return aborted(); }, timeout_ms_, ready ? "dp ready" : "dp done"))
                return rc;
            if (cudaStreamWaitEvent(cs, ready ? ev_ready_[j][c] : ev_done_[j][c], 0))
                return set_error(TPIPE_E_CUDA, "dp: stream wait");
        }
        return 0;
    }
    int post_ready(int c, uint64_t seq, cudaStream_t cs) override {
        return post(ev_ready_[rank_][c], mem(rank_).ready_seq[c], seq, cs);
    }
    int wait_ready(int c, uint64_t seq, cudaStream_t cs) override { return wait_all(true, c, seq, cs); }
    int post_done(int c, uint64_t seq, cudaStream_t cs) override {
        return post(ev_done_[rank_][c], mem(rank_).done_seq[c], seq, cs);
    }
    int wait_done(int c, uint64_t seq, cudaStream_t cs) override { return wait_all(false, c, seq, cs); }
    void* peer_w(int j, int c) override { return (uint8_t*)arena_of(j) + mem(j).w_off[c]; }
    float* peer_grad(int j, int c) override { return (float*)((uint8_t*)arena_of(j) + mem(j).g_off[c]); }
    void* arena_of(int j) const { return j == rank_ ? own_arena_ : peer_arena_[j]; }

    int init(int dp, int rank, int v, const char* name, void* arena, size_t arena_bytes, const uint64_t* w_off,
             const uint64_t* g_off, int timeout_ms) {
        dp_ = dp;
        rank_ = rank;
        timeout_ms_ = timeout_ms;
        own_arena_ = arena;
        if (dp < 2 || dp > DP_MAX || rank < 0 || rank >= dp || v < 1 || v > 4)
            return set_error(TPIPE_E_INVALID, "dp group: dp %d rank %d", dp, rank);
        if (!name || name[0] != '/') return set_error(TPIPE_E_INVALID, "dp group needs an ipc_name ('/...')");
        shm_bytes_ = sizeof(DpHeader) + (size_t)dp * sizeof(DpMember);
        int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
        if (fd < 0) return set_error(TPIPE_E_INVALID, "shm_open(%s): %s", name, strerror(errno));
        if (ftruncate(fd, (off_t)shm_bytes_) != 0) {
            close(fd);
            return set_error(TPIPE_E_INVALID, "ftruncate(%s): %s", name, strerror(errno));
        }
        void* m = mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) return set_error(TPIPE_E_INVALID, "mmap(%s): %s", name, strerror(errno));
        shm_ = (uint8_t*)m;
        uint64_t zero = 0;
        if (hdr()->magic.compare_exchange_strong(zero, DP_MAGIC)) {
            hdr()->dp.store(dp);
            hdr()->v.store(v);
        } else if (zero != DP_MAGIC) {
            return set_error(TPIPE_E_INVALID, "shm %s holds foreign data", name);
        }
        DpMember& me = mem(rank);
        if (cudaIpcGetMemHandle(&me.arena, arena)) return set_error(TPIPE_E_CUDA, "dp: cudaIpcGetMemHandle");
        me.arena_bytes = arena_bytes;
        for (int c = 1; c <= v; ++c) {
            me.w_off[c] = w_off[c];
            me.g_off[c] = g_off[c];
            if (cudaEventCreateWithFlags(&ev_ready_[rank][c], cudaEventDisableTiming | cudaEventInterprocess) ||
                cudaEventCreateWithFlags(&ev_done_[rank][c], cudaEventDisableTiming | cudaEventInterprocess) ||
                cudaIpcGetEventHandle(&me.ready[c], ev_ready_[rank][c]) ||
                cudaIpcGetEventHandle(&me.done[c], ev_done_[rank][c]))
                return set_error(TPIPE_E_CUDA, "dp: interprocess events");
        }
        std::atomic_thread_fence(std::memory_order_seq_cst);
        hdr()->arrived.fetch_add(1, std::memory_order_acq_rel);
        if (int rc = poll_until([&] { return hdr()->arrived.load(std::memory_order_acquire) >= dp; },
                                [&] { return aborted(); }, timeout_ms, "dp rendezvous"))
            return rc;
        if (hdr()->dp.load() != dp || hdr()->v.load() != v)
            return set_error(TPIPE_E_INVALID, "dp rendezvous: members disagree (dp, chunks)");
        if (rank == 0) shm_unlink(name);
        for (int j = 0; j < dp; ++j) {
            if (j == rank) continue;
            cudaError_t e = cudaIpcOpenMemHandle(&peer_arena_[j], mem(j).arena, cudaIpcMemLazyEnablePeerAccess);
            if (e) return set_error(TPIPE_E_CUDA, "dp: cudaIpcOpenMemHandle (replica %d): %s", j, cudaGetErrorString(e));
            for (int c = 1; c <= v; ++c)
                if (cudaIpcOpenEventHandle(&ev_ready_[j][c], mem(j).ready[c]) ||
                    cudaIpcOpenEventHandle(&ev_done_[j][c], mem(j).done[c]))
                    return set_error(TPIPE_E_CUDA, "dp: cudaIpcOpenEventHandle (replica %d)", j);
        }
        return 0;
    }

    int dp_ = 0, rank_ = 0, timeout_ms_ = 0;
    uint8_t* shm_ = nullptr;
    size_t shm_bytes_ = 0;
    void* own_arena_ = nullptr;
    void* peer_arena_[DP_MAX] = {};
    cudaEvent_t ev_ready_[DP_MAX][5] = {}, ev_done_[DP_MAX][5] = {};
};

}  // namespace

int make_dp_group(int dp, int dp_rank, int stage, int v, const char* shm_name, void* arena,
                  size_t arena_bytes, const uint64_t* w_off, const uint64_t* g_off, int timeout_ms,
                  std::unique_ptr<DpGroup>* out) {
    (void)stage;
    std::unique_ptr<IpcDpGroup> G(new IpcDpGroup);
    int rc = G->init(dp, dp_rank, v, shm_name, arena, arena_bytes, w_off, g_off, timeout_ms);
    if (rc) {
        G->abort();
        return rc;
    }
    *out = std::move(G);
    return 0;
}

}  // namespace tpipe
