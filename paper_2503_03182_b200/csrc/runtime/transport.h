// Stage transport: the FIFO channels of a plan carry one
// [b·s, h] activation (forward) or activation-gradient (backward) message per
// (chunk boundary, micro-batch) — the pipeline-parallel P2P of P:195 / P:210.
//
// One interface, three implementations (plus an NCCL loopback of the first); the runtime's SEND / RECV /
// SEND_WAIT instructions are the same code for all of them:
//   * virtual — every stage in one process on one GPU (stage == -1); a
//     message is a device-to-device copy from the sender's MSG buffer, the
//     scheduler runs an op only when its message exists (recv_ready).
//   * nccl    — one process per GPU, one 2-rank communicator + stream per
//     channel (ncclSend / ncclRecv), completion by events.
//   * ipc     — one process per GPU (or several processes on one GPU):
//     CUDA IPC. Every rank exports its HBM pool arena and interprocess events
//     through a POSIX shared-memory rendezvous; the receiver PULLS message n
//     from the sender's MSG buffer with a copy-engine cudaMemcpyAsync over
//     NVLink (no SMs, unlike NCCL's P2P kernels — the contention P:396 warns
//     about) once the sender's "ready" event fires, and signals "consumed"
//     with its own event. Host-side, a ring of R mailbox slots per channel
//     carries (sequence, arena offset); RECV(n) waits until the sender's host
//     has posted n, SEND_WAIT(n) until the receiver's host has issued the
//     copy of n. These host waits are exactly the edges of the plan's static
//     deadlock check (program order ∪ SEND→RECV ∪ RECV→SEND_WAIT, DESIGN
//     R12), so a plan that passes it cannot deadlock here; every wait has a
//     timeout and a shared abort flag.
//
// Message semantics common to all three (the send window W of R12):
//   send(ch, j, src)      message j of this step is complete in `src` once
//                         the work issued on `cs` so far is done;
//   recv(ch, dst)         the next message of `ch` is in `dst` for the work
//                         issued on `cs` after this call;
//   send_wait(ch, j)      `src` of message j may be overwritten by the work
//                         issued on `cs` after this call.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstddef>
#include <memory>
#include <vector>

namespace tpipe {

class Transport {
public:
    virtual ~Transport() = default;
    virtual const char* name() const = 0;
    virtual void begin_step() {}
    virtual int send(int ch, int msg, const void* src, size_t bytes, cudaStream_t cs) = 0;
    virtual int recv(int ch, void* dst, size_t bytes, cudaStream_t cs) = 0;
    virtual int send_wait(int ch, int msg, cudaStream_t cs) = 0;
    // in-process virtual pipeline: may the instruction run now (its input exists)
    virtual bool recv_ready(int) const { return true; }
    virtual bool send_wait_ready(int, int) const { return true; }
    // wait for everything issued on cs, polling transport errors; TPIPE_E_TIMEOUT
    // after timeout_ms
    virtual int sync(cudaStream_t cs, int timeout_ms);
    // a local failure: release peers blocked on this rank
    virtual void abort() {}
};

using ChannelList = std::vector<std::array<int, 3>>;   // {kind, src, dst}

std::unique_ptr<Transport> make_virtual_transport(const ChannelList& ch);
// the virtual transport with every message moved by an ncclSend / ncclRecv
// pair on a one-rank communicator (rank 0 to itself): runs the NCCL library
// path — dlopen'd entry points, group calls, stream ordering, asynchronous
// error polling — on one GPU, where NCCL refuses two ranks per device
int make_virtual_nccl_transport(const ChannelList& ch, std::unique_ptr<Transport>* out);

int make_nccl_transport(const ChannelList& ch, int stage, const void* ids, int timeout_ms,
                        std::unique_ptr<Transport>* out);

// arena/arena_bytes: the HBM pool arena every MSG buffer lives in (exported
// to the peers); window: the plan's send window W (<= the mailbox ring)
int make_ipc_transport(const ChannelList& ch, int p, int stage, int device, const char* shm_name,
                       void* arena, size_t arena_bytes, int window, int timeout_ms,
                       std::unique_ptr<Transport>* out);

// Data-parallel group (DESIGN R31): the dp replicas of one
// pipeline stage (one process each). Every member exports its pool arena, the
// arena offsets of each chunk's weights and gradients, and two interprocess
// events per chunk ("gradients final", "update done") through a POSIX-shm
// rendezvous; host-side sequence numbers say which step an event belongs to.
class DpGroup {
public:
    virtual ~DpGroup() = default;
    virtual int dp() const = 0;
    virtual int rank() const = 0;
    // this member's chunk-c gradients are final up to the work issued on cs
    virtual int post_ready(int c, uint64_t seq, cudaStream_t cs) = 0;
    // cs waits until every member posted ready(c, seq)
    virtual int wait_ready(int c, uint64_t seq, cudaStream_t cs) = 0;
    virtual int post_done(int c, uint64_t seq, cudaStream_t cs) = 0;
    virtual int wait_done(int c, uint64_t seq, cudaStream_t cs) = 0;
    // member j's chunk-c weights / gradients in this process's address space
    virtual void* peer_w(int j, int c) = 0;
    virtual float* peer_grad(int j, int c) = 0;
    virtual void abort() = 0;
};

// w_off / g_off[c]: arena offsets of chunk c's weights and gradients (c = 1..v)
int make_dp_group(int dp, int dp_rank, int stage, int v, const char* shm_name, void* arena,
                  size_t arena_bytes, const uint64_t* w_off, const uint64_t* g_off, int timeout_ms,
                  std::unique_ptr<DpGroup>* out);

}  // namespace tpipe
