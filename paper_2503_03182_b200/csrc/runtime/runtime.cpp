// tpipe_runtime / tpipe_step: executes a plan's per-stage instruction streams
// (SURVEY CS2, §8(a) a2-a9).
//
// * Every buffer is allocated from the HBM pool at the instruction the plan
//   names and released at the instruction the plan names, so the pool's
//   ledger high-water equals the plan's byte-exact peak (tpipe_plan_stage_peak).
// * Transport (runtime/transport.h): stage >= 0 -> one process per stage
//   (one GPU each, or several on one GPU for tests), FIFO channels over NCCL
//   send/recv or CUDA IPC copy-engine pulls, send window by SEND_WAIT;
//   stage == -1 -> all stages in this process on one GPU with
//   device-to-device copies (a virtual pipeline used for parity tests).
// * T-Offload: GRAD_D2H on a copy-engine stream, HOST_OPT on a host
//   thread (bit-identical AdamW), W_H2D on a second copy stream in the next
//   step's warm-up, W_WAIT before the first deep-chunk forward.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "kernels/kernels.h"
#include "plan/plan.h"
#include "runtime/errors.h"
#include "runtime/nccl_dl.h"
#include "runtime/pool.h"
#include "runtime/stage.h"
#include "runtime/transport.h"
#include "tpipe.h"



using namespace tpipe;

#define TP_API extern "C" __attribute__((visibility("default")))

#define CU(x)                                                                          \
    do {                                                                               \
        cudaError_t _e = (x);                                                          \
        if (_e != cudaSuccess)                                                         \
            return set_error(TPIPE_E_CUDA, "%s: %s", #x, cudaGetErrorString(_e));      \
    } while (0)

#define TRY(x)               \
    do {                     \
        int _rc = (x);       \
        if (_rc) return _rc; \
    } while (0)

namespace {

struct ChunkState {
    long P = 0;
    bool offloaded = false;
    ParamLayout lay;
    StashLayout sl;
    void* w = nullptr;
    float *grad = nullptr, *master = nullptr, *m = nullptr, *v = nullptr;
    // T-Offload host side (pinned)
    float *h_master = nullptr, *h_m = nullptr, *h_v = nullptr, *h_grad = nullptr;
    void* h_w = nullptr;
    cudaEvent_t ev_d2h = nullptr, ev_h2d = nullptr;
    bool d2h_pending = false, h2d_pending = false;
    std::thread host_thr;
    double host_ms = 0;
    // streamed device AdamW (TPIPE_OFFLOAD_DEVICE_OPT, DESIGN R24): two
    // staging slots of [master | m | v] x slice fp32 in the static block
    bool sopt = false;
    long slice = 0;
    float* stg[2] = {nullptr, nullptr};
    // ZeRO-1 data parallelism (R31): this replica's optimizer shard [lo, hi)
    // of the chunk's parameters, the replicas' grad / weight pointers, and the
    // sequence number of the last DP_OPT (0 = none yet)
    long lo = 0, hi = 0;
    DpPtrs dptr{};
    uint64_t dp_seq = 0;
    cudaEvent_t ev_sopt_done = nullptr;   // last slice's AdamW done (w, grad final)
    cudaEvent_t ev_sopt_out = nullptr;    // last slice's master/m/v back on the host
    bool sopt_done_pending = false, sopt_out_pending = false;
};

struct StageState {
    int s = 0;
    // compute stream of this stage: the runtime stream, or (virtual pipeline,
    // opt-in) its own stream so that a stage waiting on a message or an offload
    // copy does not hold back the other stages' work; the step stream
    // rt->stream forks into it at step start and joins it at the end
    cudaStream_t own = nullptr, cs = nullptr;
    std::unique_ptr<Pool> pool;   // this stage's HBM pool (reuse stays on one stream)
    ChunkState ch[5];   // chunks 1..v (v <= 4)
    int* tokens = nullptr;
    int* targets = nullptr;
    float* loss_slots = nullptr;
    std::vector<void*> bufptr;
    std::map<std::tuple<int, int, int>, void*> live;
    size_t pc = 0;
    // activation offload (R23): pinned host slots per micro-batch, free list
    std::map<int, void*> act_host;
    std::vector<void*> act_free;
    std::map<int, cudaEvent_t> act_ev_d2h, act_ev_h2d;
};

}  // namespace

struct tpipe_runtime {
    tpipe_plan plan;                 // deep copy (immutable)
    int stage_sel = -1, device = 0;
    Dims D;
    std::vector<int> owned;
    std::vector<std::unique_ptr<StageState>> st;   // indexed by stage (null if not owned)
    std::unique_ptr<Transport> tr;
    std::unique_ptr<DpGroup> dpg;      // dp > 1: this stage's replica group
    int dp_rank = 0;
    int transport_kind = -1;           // -1 virtual, else TPIPE_TRANSPORT_*
    double host_issue_ms = 0;
    int timeout_ms = 300000;
    uint32_t debug = 0;
    bool selftest_done = false;
    cudaStream_t stream = nullptr, d2h = nullptr, h2d = nullptr, opt = nullptr;
    cudaEvent_t ev_tmp = nullptr;
    AdamHyper hp{};
    float lr = 3e-4f, b1 = 0.9f, b2 = 0.95f, eps = 1e-8f, wd = 0.1f;
    long t = 0;
    long launches_last = 0;
    // TPIPE_STEP_GRAPH: the captured step (one per NO_OPT setting), its launch
    // count, and the device copy of the AdamW hyper-parameters it reads
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    long glaunches[2] = {0, 0};
    AdamHyper* hp_dev = nullptr;
    bool capturing = false;
    double d2h_bytes = 0, h2d_bytes = 0;
    // timing-enabled event pairs bracketing each offload copy of the last step
    std::vector<cudaEvent_t> tevpool;
    size_t tevnext = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> d2h_ev, h2d_ev;
    int* h_tok_stage = nullptr;   // pinned staging for tpipe_step host inputs
    size_t h_tok_bytes = 0;
    std::vector<cudaEvent_t> evpool;
    size_t evnext = 0;
    double kms[4] = {0, 0, 0, 0}, kflops[4] = {0, 0, 0, 0};
    int64_t kcount[4] = {0, 0, 0, 0};
    // TPIPE_STEP_OP_TIMES: per stage, (start, end) events of each compute op
    // (F / B / R, plan order) of the last step, and their durations (ms)
    std::vector<std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> op_ev;
    std::vector<std::vector<float>> op_ms;

    explicit tpipe_runtime(const tpipe_plan& p) : plan(p), D(p.model) {}
};

namespace {

cudaEvent_t next_timed_event(tpipe_runtime* rt) {
    if (rt->tevnext == rt->tevpool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        rt->tevpool.push_back(e);
    }
    return rt->tevpool[rt->tevnext++];
}

// offload copy on a copy-engine stream, bracketed by timing events
cudaError_t timed_copy(tpipe_runtime* rt, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                       cudaStream_t st, bool down) {
    cudaEvent_t a = next_timed_event(rt), b = next_timed_event(rt);
    cudaError_t e = cudaEventRecord(a, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, kind, st);
    if (e == cudaSuccess) e = cudaEventRecord(b, st);
    (down ? rt->d2h_ev : rt->h2d_ev).push_back({a, b});
    return e;
}

cudaEvent_t next_event(tpipe_runtime* rt) {
    if (rt->evnext == rt->evpool.size()) {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        rt->evpool.push_back(e);
    }
    return rt->evpool[rt->evnext++];
}

AdamHyper hyper(const tpipe_runtime* rt, long step) {
    AdamHyper h;
    h.lr = rt->lr;
    h.b1 = rt->b1;
    h.b2 = rt->b2;
    h.eps = rt->eps;
    h.wd = rt->wd;
    h.bc1 = (float)(1.0 - std::pow((double)rt->b1, (double)step));
    h.bc2 = (float)(1.0 - std::pow((double)rt->b2, (double)step));
    return h;
}

std::tuple<int, int, int> key_of(const tpipe_buf& b) { return {b.role, b.chunk, b.mb}; }

void* live_get(StageState& S, int role, int chunk, int mb) {
    auto it = S.live.find({role, chunk, mb});
    return it == S.live.end() ? nullptr : it->second;
}

int op_alloc_ptr(tpipe_runtime* rt, StageState& S, const tpipe_op& op, int role, int chunk_or_any,
                 void** out) {
    const auto& ev = rt->plan.events[S.s];
    const auto& bufs = rt->plan.bufs[S.s];
    for (int e = 0; e < op.n_alloc; ++e) {
        const int id = ev[op.alloc_first + e];
        if (bufs[id].role == role && (chunk_or_any < 0 || bufs[id].chunk == chunk_or_any)) {
            *out = S.bufptr[id];
            return 1;
        }
    }
    *out = nullptr;
    return 0;
}

int adam_chunk(tpipe_runtime* rt, ChunkState& C, const AdamHyper& hp, cudaStream_t st) {
    const int dt = rt->D.dtype;
    for (auto& sg : C.lay.segments) {
        const long off = sg[0], n = sg[1];
        void* w = dt == DT_BF16 ? (void*)((uint16_t*)C.w + off) : (void*)(C.master + off);
        if (adamw(dt, C.master + off, C.m + off, C.v + off, C.grad + off, w, n, (int)sg[2], hp, st,
                  rt->capturing ? rt->hp_dev : nullptr))
            return set_error(TPIPE_E_CUDA, "adamw launch failed");
    }
    return 0;
}

void host_opt_run(tpipe_runtime* rt, ChunkState* C, AdamHyper hp) {
    auto t0 = std::chrono::steady_clock::now();
    cudaEventSynchronize(C->ev_d2h);
    uint16_t* wb = rt->D.dtype == DT_BF16 ? (uint16_t*)C->h_w : nullptr;
    for (auto& sg : C->lay.segments) {
        const long off = sg[0], n = sg[1];
        adamw_host(C->h_master + off, C->h_m + off, C->h_v + off, C->h_grad + off,
                   wb ? wb + off : nullptr, n, (int)sg[2], hp);
    }
    C->host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void join_host(ChunkState& C) {
    if (C.host_thr.joinable()) C.host_thr.join();
    if (C.sopt_out_pending) {
        cudaEventSynchronize(C.ev_sopt_out);
        C.sopt_out_pending = false;
    }
}

// Streamed device AdamW of an offloaded chunk (R24): slice k's fp32
// master/m/v go H2D into staging slot k&1 (h2d stream), the AdamW kernel
// updates them with the chunk's device grads and writes the bf16 weights in
// place (opt stream), and the slice returns D2H (d2h stream); slot reuse waits
// for the D2H of slice k-2. Same kernel and per-segment decay as OPT, so the
// parameters are bit-identical to the device and host optimizers.
int stream_opt(tpipe_runtime* rt, ChunkState& C, const AdamHyper& hp, cudaStream_t cs) {
    const int dt = rt->D.dtype;
    cudaEvent_t ready = next_event(rt);
    CU(cudaEventRecord(ready, cs));                      // the chunk's grads are final
    CU(cudaStreamWaitEvent(rt->h2d, ready, 0));
    CU(cudaStreamWaitEvent(rt->opt, ready, 0));
    if (C.sopt_out_pending) CU(cudaStreamWaitEvent(rt->h2d, C.ev_sopt_out, 0));   // last step's D2H
    const long SL = C.slice;
    std::vector<cudaEvent_t> out_ev;
    int k = 0;
    for (long lo = 0; lo < C.P; lo += SL, ++k) {
        const long n = std::min(SL, C.P - lo);
        float* st = C.stg[k & 1];
        if (k >= 2) CU(cudaStreamWaitEvent(rt->h2d, out_ev[k - 2], 0));
        CU(timed_copy(rt, st, C.h_master + lo, (size_t)n * 4, cudaMemcpyHostToDevice, rt->h2d, false));
        CU(timed_copy(rt, st + SL, C.h_m + lo, (size_t)n * 4, cudaMemcpyHostToDevice, rt->h2d, false));
        CU(timed_copy(rt, st + 2 * SL, C.h_v + lo, (size_t)n * 4, cudaMemcpyHostToDevice, rt->h2d, false));
        rt->h2d_bytes += (double)n * 12;
        cudaEvent_t in = next_event(rt);
        CU(cudaEventRecord(in, rt->h2d));
        CU(cudaStreamWaitEvent(rt->opt, in, 0));
        for (auto& sg : C.lay.segments) {
            const long a = std::max(lo, (long)sg[0]), b = std::min(lo + n, (long)(sg[0] + sg[1]));
            if (a >= b) continue;
            const long r = a - lo;
            void* w = dt == DT_BF16 ? (void*)((uint16_t*)C.w + a) : (void*)((float*)C.w + a);
            if (adamw(dt, st + r, st + SL + r, st + 2 * SL + r, C.grad + a, w, b - a, (int)sg[2], hp, rt->opt))
                return set_error(TPIPE_E_CUDA, "adamw launch failed");
        }
        cudaEvent_t done = next_event(rt);
        CU(cudaEventRecord(done, rt->opt));
        CU(cudaStreamWaitEvent(rt->d2h, done, 0));
        CU(timed_copy(rt, C.h_master + lo, st, (size_t)n * 4, cudaMemcpyDeviceToHost, rt->d2h, true));
        CU(timed_copy(rt, C.h_m + lo, st + SL, (size_t)n * 4, cudaMemcpyDeviceToHost, rt->d2h, true));
        CU(timed_copy(rt, C.h_v + lo, st + 2 * SL, (size_t)n * 4, cudaMemcpyDeviceToHost, rt->d2h, true));
        rt->d2h_bytes += (double)n * 12;
        cudaEvent_t out = next_event(rt);
        CU(cudaEventRecord(out, rt->d2h));
        out_ev.push_back(out);
    }
    CU(cudaEventRecord(C.ev_sopt_done, rt->opt));
    CU(cudaEventRecord(C.ev_sopt_out, rt->d2h));
    C.sopt_done_pending = C.sopt_out_pending = true;
    return 0;
}

// ------------------------------------------------------------------ one instruction
int exec_op(tpipe_runtime* rt, StageState& S, const tpipe_op& op, uint32_t flags) {
    const int s = S.s;
    const auto& P = rt->plan;
    const auto& bufs = P.bufs[s];
    const auto& ev = P.events[s];
    const Dims& D = rt->D;
    cudaStream_t cs = S.cs;
    Pool& pool = *S.pool;
    const int p = P.p, v = P.v;
    const bool trecomp = P.strategy == TPIPE_S_TPIPE_TRECOMP || P.strategy == TPIPE_S_INTERLEAVE_TRECOMP;
    const bool no_opt = flags & TPIPE_STEP_NO_OPT;

    // allocations at instruction start
    for (int e = 0; e < op.n_alloc; ++e) {
        const int id = ev[op.alloc_first + e];
        void* ptr = pool.alloc_id(s, id, bufs[id].bytes);
        if (!ptr && pool.last_fail_physical())
            return set_error(TPIPE_E_OOM, "stage %d: pool fragmentation would place %llu bytes beyond the "
                             "HBM budget (arena %zu + overflow %zu)", s, (unsigned long long)bufs[id].bytes,
                             pool.arena_bytes(), pool.overflow_bytes());
        if (!ptr) return set_error(TPIPE_E_CUDA, "pool allocation of %llu bytes failed",
                                   (unsigned long long)bufs[id].bytes);
        S.bufptr[id] = ptr;
        S.live[key_of(bufs[id])] = ptr;
    }
    if (pool.over_cap())
        return set_error(TPIPE_E_OOM, "stage %d ledger exceeds the plan peak (ledger bug)", s);
    if ((rt->debug & TPIPE_DEBUG_POOL_CANARY_SELFTEST) && !rt->selftest_done && op.n_alloc > 0) {
        const int id = ev[op.alloc_first];
        CU(cudaMemsetAsync((uint8_t*)S.bufptr[id] + bufs[id].bytes, 0x5A, 1, cs));
        rt->selftest_done = true;
    }

    const int c = op.chunk, i = op.mb;
    switch (op.kind) {
        case TPIPE_OP_F:
        case TPIPE_OP_R: {
            ChunkState& C = S.ch[c];
            const bool emb = (s == 0 && c == 1);
            FwdArgs a{};
            a.in = emb ? nullptr : live_get(S, TPIPE_BUF_IN, c, i);
            a.tokens = S.tokens ? S.tokens + (long)(i - 1) * D.M : nullptr;
            a.targets = (S.targets && s == p - 1 && c == v) ? S.targets + (long)(i - 1) * D.M : nullptr;
            a.loss_slot = S.loss_slots ? S.loss_slots + (i - 1) : nullptr;
            a.loss_scale = 1.0f / ((float)(P.dp * P.m) * (float)D.M);
            void* ws = nullptr;
            op_alloc_ptr(rt, S, op, TPIPE_BUF_WS, -1, &ws);
            a.ws = (uint8_t*)ws;
            const bool partial = trecomp && c == 1 && P.rl_of(s) < P.sl[s][0];
            if (op.kind == TPIPE_OP_R) {
                void* rb;
                op_alloc_ptr(rt, S, op, TPIPE_BUF_RBUF, -1, &rb);
                a.stash = (uint8_t*)rb;
                a.out = nullptr;
                a.targets = nullptr;
                if (partial) a.split = a.n_run = P.rl_of(s);   // regenerate layers 1..r only
            } else {
                void *tst = nullptr, *kst = nullptr;
                op_alloc_ptr(rt, S, op, TPIPE_BUF_TSTASH, -1, &tst);
                op_alloc_ptr(rt, S, op, TPIPE_BUF_STASH, -1, &kst);
                a.stash = (uint8_t*)(tst ? tst : kst);
                if (tst && partial) {
                    if (!kst) return set_error(TPIPE_E_STATE, "stage %d F(1,%d): kept stash missing", s, i);
                    a.stash2 = (uint8_t*)kst;
                    a.split = P.rl_of(s);
                }
                void* out = nullptr;
                if (!op_alloc_ptr(rt, S, op, TPIPE_BUF_MSG, -1, &out))
                    op_alloc_ptr(rt, S, op, TPIPE_BUF_IN, c + 1, &out);
                a.out = out;
            }
            if (!a.stash || !a.ws || (!emb && !a.in))
                return set_error(TPIPE_E_STATE, "stage %d op %d: missing buffer", s, op.kind);
            ChunkParamsDev cp{&C.lay, C.w, C.grad};
            if (chunk_forward(D, C.sl, cp, a, cs))
                return set_error(TPIPE_E_CUDA, "chunk_forward failed: %s",
                                 cudaGetErrorString(cudaGetLastError()));
            break;
        }
        case TPIPE_OP_B: {
            ChunkState& C = S.ch[c];
            const bool emb = (s == 0 && c == 1), head = (s == p - 1 && c == v);
            BwdArgs a{};
            a.in = emb ? nullptr : live_get(S, TPIPE_BUF_IN, c, i);
            a.tokens = S.tokens ? S.tokens + (long)(i - 1) * D.M : nullptr;
            a.targets = head ? S.targets + (long)(i - 1) * D.M : nullptr;
            a.loss_slot = (head && S.loss_slots) ? S.loss_slots + (i - 1) : nullptr;
            a.loss_scale = 1.0f / ((float)(P.dp * P.m) * (float)D.M);
            void* stp = (trecomp && c == 1) ? live_get(S, TPIPE_BUF_RBUF, c, i)
                                            : live_get(S, TPIPE_BUF_STASH, c, i);
            a.stash = (uint8_t*)stp;
            if (trecomp && c == 1 && P.rl_of(s) < P.sl[s][0]) {   // partial T-Recomp (R25)
                a.stash2 = (uint8_t*)live_get(S, TPIPE_BUF_STASH, c, i);
                a.split = P.rl_of(s);
                if (!a.stash2) return set_error(TPIPE_E_STATE, "stage %d B(1,%d): kept stash missing", s, i);
            }
            void* ws = nullptr;
            op_alloc_ptr(rt, S, op, TPIPE_BUF_WS, -1, &ws);
            a.ws = (uint8_t*)ws;
            a.gin = head ? nullptr : live_get(S, TPIPE_BUF_GIN, c, i);
            void* gout = nullptr;
            if (!op_alloc_ptr(rt, S, op, TPIPE_BUF_MSG, -1, &gout))
                op_alloc_ptr(rt, S, op, TPIPE_BUF_GIN, c - 1, &gout);
            a.gout = gout;
            if (!a.stash || !a.ws || (!emb && !a.in) || (!head && !a.gin) || (!emb && !a.gout))
                return set_error(TPIPE_E_STATE, "stage %d B(%d,%d): missing buffer", s, c, i);
            ChunkParamsDev cp{&C.lay, C.w, C.grad};
            if (chunk_backward(D, C.sl, cp, a, cs))
                return set_error(TPIPE_E_CUDA, "chunk_backward failed: %s",
                                 cudaGetErrorString(cudaGetLastError()));
            break;
        }
        case TPIPE_OP_RECV_ACT:
        case TPIPE_OP_RECV_GRAD: {
            void* dst = nullptr;
            op_alloc_ptr(rt, S, op, op.kind == TPIPE_OP_RECV_ACT ? TPIPE_BUF_IN : TPIPE_BUF_GIN, -1, &dst);
            if (!dst) return set_error(TPIPE_E_STATE, "stage %d RECV: receive buffer missing", s);
            TRY(rt->tr->recv(op.channel, dst, (size_t)D.M * D.h * D.es, cs));
            break;
        }
        case TPIPE_OP_SEND_ACT:
        case TPIPE_OP_SEND_GRAD: {
            void* src = live_get(S, TPIPE_BUF_MSG, op.channel, op.msg);
            if (!src) return set_error(TPIPE_E_STATE, "send buffer missing");
            TRY(rt->tr->send(op.channel, op.msg, src, (size_t)D.M * D.h * D.es, cs));
            break;
        }
        case TPIPE_OP_SEND_WAIT:
            TRY(rt->tr->send_wait(op.channel, op.msg, cs));
            break;
        case TPIPE_OP_OPT:
            if (!no_opt) TRY(adam_chunk(rt, S.ch[c], hyper(rt, rt->t + 1), cs));
            break;
        case TPIPE_OP_DP_OPT: {
            // ZeRO-1 (R31): every replica's chunk-c gradients are final -> this
            // replica reduces its shard over the replicas, updates it, and writes
            // the new weights into every replica (one fused kernel per segment)
            if (no_opt) break;
            ChunkState& C = S.ch[c];
            const uint64_t seq = (uint64_t)rt->t + 1;
            TRY(rt->dpg->post_ready(c, seq, cs));
            TRY(rt->dpg->wait_ready(c, seq, cs));
            const AdamHyper hp = hyper(rt, rt->t + 1);
            for (auto& sg : C.lay.segments) {
                const long a = std::max(C.lo, (long)sg[0]), b = std::min(C.hi, (long)(sg[0] + sg[1]));
                if (a >= b) continue;
                if (dp_adamw(D.dtype, C.dptr, P.dp, C.master + (a - C.lo), C.m + (a - C.lo), C.v + (a - C.lo), a,
                             b - a, (int)sg[2], hp, cs))
                    return set_error(TPIPE_E_CUDA, "dp_adamw launch failed");
            }
            TRY(rt->dpg->post_done(c, seq, cs));
            C.dp_seq = seq;
            break;
        }
        case TPIPE_OP_DP_WAIT: {
            ChunkState& C = S.ch[c];
            if (C.dp_seq) TRY(rt->dpg->wait_done(c, C.dp_seq, cs));
            break;
        }
        case TPIPE_OP_GRAD_D2H: {
            if (no_opt) break;
            ChunkState& C = S.ch[c];
            cudaEvent_t e0 = next_event(rt);
            CU(cudaEventRecord(e0, cs));
            CU(cudaStreamWaitEvent(rt->d2h, e0, 0));
            CU(timed_copy(rt, C.h_grad, C.grad, (size_t)C.P * 4, cudaMemcpyDeviceToHost, rt->d2h, true));
            CU(cudaMemsetAsync(C.grad, 0, (size_t)C.P * 4, rt->d2h));
            CU(cudaEventRecord(C.ev_d2h, rt->d2h));
            C.d2h_pending = true;
            rt->d2h_bytes += (double)C.P * 4;
            break;
        }
        case TPIPE_OP_HOST_OPT: {
            if (no_opt) break;
            ChunkState& C = S.ch[c];
            join_host(C);
            C.host_thr = std::thread(host_opt_run, rt, &C, hyper(rt, rt->t + 1));
            break;
        }
        case TPIPE_OP_W_H2D: {
            ChunkState& C = S.ch[c];
            join_host(C);
            CU(timed_copy(rt, C.w, C.h_w, (size_t)C.P * D.es, cudaMemcpyHostToDevice, rt->h2d, false));
            CU(cudaEventRecord(C.ev_h2d, rt->h2d));
            C.h2d_pending = true;
            rt->h2d_bytes += (double)C.P * D.es;
            break;
        }
        case TPIPE_OP_STREAM_OPT: {
            if (no_opt) break;
            TRY(stream_opt(rt, S.ch[c], hyper(rt, rt->t + 1), cs));
            break;
        }
        case TPIPE_OP_W_WAIT: {
            ChunkState& C = S.ch[c];
            if (C.sopt_done_pending) CU(cudaStreamWaitEvent(cs, C.ev_sopt_done, 0));
            C.sopt_done_pending = false;
            if (C.h2d_pending) CU(cudaStreamWaitEvent(cs, C.ev_h2d, 0));
            if (C.d2h_pending) CU(cudaStreamWaitEvent(cs, C.ev_d2h, 0));
            C.h2d_pending = C.d2h_pending = false;
            break;
        }
        case TPIPE_OP_ACT_D2H: {
            ChunkState& C = S.ch[1];
            void* dev = live_get(S, TPIPE_BUF_STASH, 1, i);
            if (!dev) return set_error(TPIPE_E_STATE, "ACT_D2H: stash (1,%d) not live", i);
            const size_t bytes = (size_t)C.sl.total;
            void* host;
            if (!S.act_free.empty()) {
                host = S.act_free.back();
                S.act_free.pop_back();
            } else {
                CU(cudaHostAlloc(&host, bytes, cudaHostAllocDefault));
            }
            S.act_host[i] = host;
            cudaEvent_t e0 = next_event(rt), e1 = next_event(rt);
            CU(cudaEventRecord(e0, cs));
            CU(cudaStreamWaitEvent(rt->d2h, e0, 0));
            CU(timed_copy(rt, host, dev, bytes, cudaMemcpyDeviceToHost, rt->d2h, true));
            CU(cudaEventRecord(e1, rt->d2h));
            S.act_ev_d2h[i] = e1;
            rt->d2h_bytes += (double)bytes;
            break;
        }
        case TPIPE_OP_ACT_D2H_WAIT:
            // device copy may be released only once the copy engine has read it
            CU(cudaStreamWaitEvent(cs, S.act_ev_d2h.at(i), 0));
            break;
        case TPIPE_OP_ACT_H2D: {
            ChunkState& C = S.ch[1];
            void* dev = live_get(S, TPIPE_BUF_STASH, 1, i);
            void* host = S.act_host.at(i);
            cudaEvent_t e0 = next_event(rt), e1 = next_event(rt);
            CU(cudaEventRecord(e0, cs));   // previous users of `dev` are done
            CU(cudaStreamWaitEvent(rt->h2d, e0, 0));
            CU(timed_copy(rt, dev, host, (size_t)C.sl.total, cudaMemcpyHostToDevice, rt->h2d, false));
            CU(cudaEventRecord(e1, rt->h2d));
            S.act_ev_h2d[i] = e1;
            rt->h2d_bytes += (double)C.sl.total;
            break;
        }
        case TPIPE_OP_ACT_H2D_WAIT:
            CU(cudaStreamWaitEvent(cs, S.act_ev_h2d.at(i), 0));
            S.act_free.push_back(S.act_host.at(i));
            S.act_host.erase(i);
            break;
        default:
            return set_error(TPIPE_E_STATE, "unknown op kind %d", op.kind);
    }

    // debug: a kernel of this instruction wrote past a buffer's planned bytes
    if (rt->debug & TPIPE_DEBUG_POOL_CANARY) {
        uint64_t rb = 0;
        if (void* bad = pool.check_canaries(cs, &rb)) {
            int role = -1, chunk = -1, mb = -1;
            for (int s2 : rt->owned)
                for (size_t id = 0; id < rt->st[s2]->bufptr.size(); ++id)
                    if (rt->st[s2]->bufptr[id] == bad) {
                        role = P.bufs[s2][id].role;
                        chunk = P.bufs[s2][id].chunk;
                        mb = P.bufs[s2][id].mb;
                    }
            return set_error(TPIPE_E_STATE, "pool canary: stage %d op kind %d (chunk %d, mb %d) overran a "
                             "%llu-byte buffer (role %d, chunk %d, mb %d)", s, op.kind, op.chunk, op.mb,
                             (unsigned long long)rb, role, chunk, mb);
        }
    }
    // releases at instruction end
    for (int e = 0; e < op.n_free; ++e) {
        const int id = ev[op.free_first + e];
        pool.free(s, S.bufptr[id]);
        S.live.erase(key_of(bufs[id]));
        S.bufptr[id] = nullptr;
    }
    return 0;
}

bool op_ready(tpipe_runtime* rt, const tpipe_op& op) {
    if (op.kind == TPIPE_OP_RECV_ACT || op.kind == TPIPE_OP_RECV_GRAD) return rt->tr->recv_ready(op.channel);
    if (op.kind == TPIPE_OP_SEND_WAIT) return rt->tr->send_wait_ready(op.channel, op.msg);
    return true;
}

int run_step_impl(tpipe_runtime* rt, const int32_t* tok_dev, const int32_t* tgt_dev, uint32_t flags,
                  float* loss_out);

// a failed step releases peers blocked on this rank (IPC abort flag)
int run_step(tpipe_runtime* rt, const int32_t* tok_dev, const int32_t* tgt_dev, uint32_t flags,
             float* loss_out) {
    const int rc = run_step_impl(rt, tok_dev, tgt_dev, flags, loss_out);
    if (rc && rt->tr) rt->tr->abort();
    return rc;
}

// The instruction streams of one step: every op of every owned stage, issued
// on the stage streams in plan order (the host only orders the issue; all
// waiting is on the device), joined back into rt->stream.
static int issue_ops(tpipe_runtime* rt, uint32_t flags, bool op_times) {
    const auto& P = rt->plan;
    cudaStream_t cs = rt->stream;
    // (after the token / target copies, so every stage sees them)
    cudaEvent_t fork = next_event(rt);
    CU(cudaEventRecord(fork, cs));
    for (int s : rt->owned) {
        StageState& S = *rt->st[s];
        S.cs = (S.own && !op_times && !(flags & TPIPE_STEP_PROFILE)) ? S.own : cs;
        if (S.cs != cs) CU(cudaStreamWaitEvent(S.cs, fork, 0));
        S.pool->set_canary((rt->debug & TPIPE_DEBUG_POOL_CANARY) != 0, S.cs);
    }
    rt->tr->begin_step();
    size_t remaining = 0;
    for (int s : rt->owned) remaining += P.ops[s].size();
    rt->op_ev.assign(P.p, {});
    rt->op_ms.assign(P.p, {});
    while (remaining) {
        bool prog = false;
        for (int s : rt->owned) {
            StageState& S = *rt->st[s];
            const auto& ops = P.ops[s];
            while (S.pc < ops.size() && op_ready(rt, ops[S.pc])) {
                const int k = ops[S.pc].kind;
                const bool timed = op_times && (k == TPIPE_OP_F || k == TPIPE_OP_B || k == TPIPE_OP_R);
                cudaEvent_t ea = nullptr, eb = nullptr;
                if (timed) {
                    ea = next_timed_event(rt);
                    eb = next_timed_event(rt);
                    CU(cudaEventRecord(ea, S.cs));
                }
                TRY(exec_op(rt, S, ops[S.pc], flags));
                if (timed) {
                    CU(cudaEventRecord(eb, S.cs));   // the layer side stream joins cs inside the op
                    rt->op_ev[s].push_back({ea, eb});
                }
                S.pc++;
                remaining--;
                prog = true;
            }
        }
        if (!prog) return set_error(TPIPE_E_DEADLOCK, "virtual transport made no progress");
    }
    if (rt->dpg && !(flags & TPIPE_STEP_NO_OPT)) {
        // synchronous data parallelism: the step is complete when every replica
        // has written this step's weights into this replica
        for (int s : rt->owned)
            for (int c = 1; c <= P.v; ++c)
                if (rt->st[s]->ch[c].dp_seq == (uint64_t)rt->t + 1)
                    TRY(rt->dpg->wait_done(c, rt->st[s]->ch[c].dp_seq, rt->st[s]->cs));
    }
    for (int s : rt->owned) {   // join: the step stream waits for every stage
        StageState& S = *rt->st[s];
        if (S.cs == cs) continue;
        cudaEvent_t j = next_event(rt);
        CU(cudaEventRecord(j, S.cs));
        CU(cudaStreamWaitEvent(cs, j, 0));
    }
    return 0;
}

int run_step_impl(tpipe_runtime* rt, const int32_t* tok_dev, const int32_t* tgt_dev, uint32_t flags,
             float* loss_out) {
    const auto& P = rt->plan;
    const Dims& D = rt->D;
    cudaStream_t cs = rt->stream;
    const size_t io_bytes = (size_t)P.m * D.M * 4;
    rt->evnext = 0;
    rt->tevnext = 0;
    rt->d2h_ev.clear();
    rt->h2d_ev.clear();
    rt->d2h_bytes = rt->h2d_bytes = 0;
    const auto t_issue0 = std::chrono::steady_clock::now();
    const long l0 = launch_count();
    profiler().begin_step((flags & TPIPE_STEP_PROFILE) != 0);
    const bool op_times = (flags & TPIPE_STEP_OP_TIMES) != 0;
    const bool graph = (flags & TPIPE_STEP_GRAPH) && !op_times && !(flags & TPIPE_STEP_PROFILE);
    if (graph && (rt->transport_kind != -1 || std::strcmp(rt->tr->name(), "virtual") != 0 || rt->dpg ||
                  P.offload != 0 || rt->debug != 0))
        return set_error(TPIPE_E_INVALID,
                         "TPIPE_STEP_GRAPH needs an in-process transport, no T-Offload, no DP, no debug canaries");
    // stage streams: separate per stage in the virtual pipeline, except while
    // timing ops or kernel classes (OP_TIMES / PROFILE: serial, each op's or
    // kernel's own GPU time)
    for (int s : rt->owned) {
        StageState& S = *rt->st[s];
        S.pc = 0;
        if (s == 0 && tok_dev) CU(cudaMemcpyAsync(S.tokens, tok_dev, io_bytes, cudaMemcpyDeviceToDevice, cs));
        if (s == P.p - 1) {
            if (tgt_dev) CU(cudaMemcpyAsync(S.targets, tgt_dev, io_bytes, cudaMemcpyDeviceToDevice, cs));
            CU(cudaMemsetAsync(S.loss_slots, 0, (size_t)P.m * 4, cs));
        }
    }
    const int gi = (flags & TPIPE_STEP_NO_OPT) ? 1 : 0;
    bool replayed = false;
    if (graph) {
        // this step's AdamW hyper-parameters, read by the graph's AdamW launches
        if (!rt->hp_dev) CU(cudaMalloc(&rt->hp_dev, sizeof(AdamHyper)));
        const AdamHyper hp = hyper(rt, rt->t + 1);
        CU(cudaMemcpyAsync(rt->hp_dev, &hp, sizeof(hp), cudaMemcpyHostToDevice, cs));
        if (rt->gexec[gi]) {
            CU(cudaGraphLaunch(rt->gexec[gi], cs));
            replayed = true;
        } else {
            CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
            rt->capturing = true;
        }
    }
    if (!replayed) {
        const int rc = issue_ops(rt, flags, op_times);
        if (rt->capturing) {
            rt->capturing = false;
            cudaGraph_t gr = nullptr;
            const cudaError_t e = cudaStreamEndCapture(cs, &gr);
            if (rc) {
                if (gr) cudaGraphDestroy(gr);
                return rc;
            }
            if (e != cudaSuccess || !gr) return set_error(TPIPE_E_CUDA, "step graph capture failed");
            const cudaError_t ei = cudaGraphInstantiate(&rt->gexec[gi], gr, 0);
            cudaGraphDestroy(gr);
            if (ei != cudaSuccess) {
                rt->gexec[gi] = nullptr;
                return set_error(TPIPE_E_CUDA, "step graph instantiate failed");
            }
            rt->glaunches[gi] = launch_count() - l0;
            CU(cudaGraphLaunch(rt->gexec[gi], cs));
        } else if (rc) {
            return rc;
        }
    }
    rt->host_issue_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_issue0).count();
    float loss = 0.f;
    if (std::find(rt->owned.begin(), rt->owned.end(), P.p - 1) != rt->owned.end()) {
        std::vector<float> slots(P.m);
        CU(cudaMemcpyAsync(slots.data(), rt->st[P.p - 1]->loss_slots, (size_t)P.m * 4,
                           cudaMemcpyDeviceToHost, cs));
        TRY(rt->tr->sync(cs, rt->timeout_ms));
        for (float x : slots) loss += x;   // micro-batch index order
    } else {
        TRY(rt->tr->sync(cs, rt->timeout_ms));
    }
    if (loss_out) *loss_out = loss;
    if (flags & TPIPE_STEP_PROFILE) {
        profiler().collect(rt->kms, rt->kflops, rt->kcount);
        profiler().on = false;
    }
    if (op_times) {
        for (int s : rt->owned)
            for (auto& pr : rt->op_ev[s]) {
                float ms = 0.f;
                CU(cudaEventElapsedTime(&ms, pr.first, pr.second));
                rt->op_ms[s].push_back(ms);
            }
    }
    if (!(flags & TPIPE_STEP_NO_OPT)) rt->t += 1;
    rt->launches_last = replayed ? rt->glaunches[gi] : launch_count() - l0;
    return 0;
}

// Every buffer the plan sizes must equal what the kernels carve out of it
// (StashLayout for STASH / TSTASH / RBUF, chunk_forward / chunk_backward for
// the workspaces): the byte model and the layouts are written separately,
// and a drift would silently overrun a neighbouring pool block.
int check_layouts(const tpipe_plan& P, const std::vector<int>& owned) {
    const Dims D(P.model);
    const bool full = P.strategy == TPIPE_S_1F1B_FULL_RECOMP;
    const bool trecomp = P.strategy == TPIPE_S_TPIPE_TRECOMP || P.strategy == TPIPE_S_INTERLEAVE_TRECOMP;
    for (int s : owned) {
        for (const tpipe_op& op : P.ops[s]) {
            for (int e = 0; e < op.n_alloc; ++e) {
                const tpipe_buf& b = P.bufs[s][P.events[s][op.alloc_first + e]];
                if (b.role == TPIPE_BUF_STATIC || b.role == TPIPE_BUF_IN || b.role == TPIPE_BUF_GIN ||
                    b.role == TPIPE_BUF_MSG)
                    continue;
                const int c = b.chunk;
                const bool emb = (s == 0 && c == 1), head = (s == P.p - 1 && c == P.v);
                const StashLayout SL = make_stash_layout(P.model, P.sl[s][c - 1], emb, head, full, P.rl_of(s));
                const int split = (trecomp && c == 1 && P.rl_of(s) < P.sl[s][0]) ? P.rl_of(s) : 0;
                const uint64_t front = split ? (uint64_t)SL.layer[split].x_in : (uint64_t)SL.total;
                uint64_t want = 0;
                const char* what = "";
                switch (b.role) {
                    case TPIPE_BUF_STASH:   // kept part [split, n) under partial T-Recomp
                        want = split ? (uint64_t)SL.total - front : (uint64_t)SL.total;
                        what = "stash";
                        break;
                    case TPIPE_BUF_TSTASH:
                    case TPIPE_BUF_RBUF:
                        want = front;
                        what = b.role == TPIPE_BUF_RBUF ? "recompute buffer" : "transient stash";
                        break;
                    case TPIPE_BUF_WS:
                        want = op.kind == TPIPE_OP_B ? bwd_ws_bytes(D, SL, head, emb) : fwd_ws_bytes(D, SL, head);
                        what = op.kind == TPIPE_OP_B ? "backward workspace" : "forward workspace";
                        break;
                    default:
                        continue;
                }
                if (b.bytes != want)
                    return set_error(TPIPE_E_STATE, "stage %d chunk %d: plan %s %llu bytes != kernel layout %llu",
                                     s, c, what, (unsigned long long)b.bytes, (unsigned long long)want);
            }
        }
    }
    return 0;
}

}  // namespace

// ================================================================== C-ABI
TP_API int tpipe_runtime_create(const tpipe_plan* plan, const tpipe_runtime_opts* opts,
                                tpipe_runtime** out) {
    if (!plan || !out) return set_error(TPIPE_E_INVALID, "NULL argument");
    *out = nullptr;
    tpipe_runtime_opts o{};
    o.stage = -1;
    if (opts) o = *opts;
    if (o.stage < -1 || o.stage >= plan->p) return set_error(TPIPE_E_INVALID, "stage");
    if (plan->dp > 1 && (o.stage < 0 || !o.ipc_name || o.dp_rank < 0 || o.dp_rank >= plan->dp))
        return set_error(TPIPE_E_INVALID, "dp > 1 needs stage >= 0, an ipc_name and 0 <= dp_rank < dp");
    if (plan->dp == 1 && o.dp_rank != 0) return set_error(TPIPE_E_INVALID, "dp_rank with dp = 1");
    if ((long)plan->model.micro_batch * plan->model.seq_len % 8)
        return set_error(TPIPE_E_INVALID, "micro_batch*seq_len must be a multiple of 8");
    std::unique_ptr<tpipe_runtime> rt(new (std::nothrow) tpipe_runtime(*plan));
    if (!rt) return set_error(TPIPE_E_INVALID, "out of host memory");
    rt->stage_sel = o.stage;
    rt->device = o.device;
    if (o.lr > 0) rt->lr = o.lr;
    if (o.beta1 > 0) rt->b1 = o.beta1;
    if (o.beta2 > 0) rt->b2 = o.beta2;
    if (o.eps > 0) rt->eps = o.eps;
    if (o.weight_decay > 0) rt->wd = o.weight_decay;
    CU(cudaSetDevice(o.device));
    CU(cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&rt->d2h, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&rt->h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&rt->opt, cudaStreamNonBlocking));
    const tpipe_plan& P = rt->plan;
    const Dims& D = rt->D;
    if (o.stage < 0) {
        for (int s = 0; s < P.p; ++s) rt->owned.push_back(s);
    } else {
        rt->owned.push_back(o.stage);
    }
    rt->debug = o.debug_flags;
    rt->timeout_ms = o.timeout_ms > 0 ? o.timeout_ms : 300000;
    // the kernels' buffer carve-ups must equal the plan's byte model (a drift
    // would overrun a neighbouring pool block): checked once per stage / chunk
    TRY(check_layouts(P, rt->owned));
    rt->st.resize(P.p);
    const bool off = (P.offload & TPIPE_OFFLOAD_MODEL_STATE) != 0;
    const bool sopt = off && (P.offload & TPIPE_OFFLOAD_DEVICE_OPT) != 0;
    for (int s : rt->owned) {
        auto S = std::make_unique<StageState>();
        S->s = s;
        // one pool (arena) per stage: a block freed by one stage is never handed
        // to another stage's stream
        // planned arena: every buffer's lifetime is fixed by the plan, so the
        // layout is computed once (pool.h) and nothing fragments at run time
        std::vector<PoolItem> items(P.bufs[s].size());
        for (size_t id = 0; id < items.size(); ++id)
            items[id] = {P.bufs[s][id].bytes, -1, std::numeric_limits<int>::max()};
        for (size_t j = 0; j < P.ops[s].size(); ++j) {
            const tpipe_op& op = P.ops[s][j];
            for (int e = 0; e < op.n_alloc; ++e) items[P.events[s][op.alloc_first + e]].first = (int)j;
            for (int e = 0; e < op.n_free; ++e) items[P.events[s][op.free_first + e]].last = (int)j;
        }
        S->pool.reset(new Pool);
        if (S->pool->init_planned(items, P.p, (o.debug_flags & TPIPE_DEBUG_POOL_CANARY) != 0))
            return set_error(TPIPE_E_CUDA, "pool: cudaMalloc of the planned arena failed (plan peak %llu bytes)",
                             (unsigned long long)P.peak[s].total_peak);
        if (P.hbm_budget) S->pool->set_phys_limit((size_t)P.hbm_budget);
        S->pool->set_cap(s, o.pool_cap ? o.pool_cap : P.peak[s].total_peak);
        S->pool->set_canary((o.debug_flags & TPIPE_DEBUG_POOL_CANARY) != 0, rt->stream);
        S->cs = rt->stream;
        // (opt-in, env TPIPE_VIRTUAL_STAGE_STREAMS=1: measured slower on one GPU —
        // the stages' persistent GEMM grids contend — profiles/r2_capacity_v2.json)
        if (o.stage < 0 && P.p > 1 && getenv("TPIPE_VIRTUAL_STAGE_STREAMS") &&
            getenv("TPIPE_VIRTUAL_STAGE_STREAMS")[0] == '1')
            CU(cudaStreamCreateWithFlags(&S->own, cudaStreamNonBlocking));
        S->bufptr.assign(P.bufs[s].size(), nullptr);
        for (size_t id = 0; id < P.bufs[s].size(); ++id) {
            const tpipe_buf& b = P.bufs[s][id];
            if (b.role != TPIPE_BUF_STATIC) continue;
            void* ptr = S->pool->alloc_id(s, (int)id, b.bytes);
            if (!ptr) return set_error(TPIPE_E_CUDA, "pool: static allocation failed");
            S->bufptr[id] = ptr;
            CU(cudaMemset(ptr, 0, b.bytes));
            if (b.category == TPIPE_CAT_MODEL_STATE) {
                const int c = b.chunk;
                ChunkState& C = S->ch[c];
                const bool emb = (s == 0 && c == 1), head = (s == P.p - 1 && c == P.v);
                C.lay = make_param_layout(P.model, P.sl[s][c - 1], emb, head);
                C.sl = make_stash_layout(P.model, P.sl[s][c - 1], emb, head,
                                         P.strategy == TPIPE_S_1F1B_FULL_RECOMP, P.rl_of(s));
                C.P = C.lay.total;
                if ((uint64_t)C.P != P.chunk_params[s][c - 1])
                    return set_error(TPIPE_E_STATE, "param layout mismatch");
                C.offloaded = off && c >= 2;   // T-Offload of chunks 2..v (R32)
                uint8_t* q = (uint8_t*)ptr;
                C.w = q;
                q += (size_t)C.P * D.es;
                C.grad = (float*)q;
                q += (size_t)C.P * 4;
                if (!C.offloaded) {
                    // optimizer shard (ZeRO-1, R31; the whole chunk when dp = 1)
                    const long S1 = P.dp > 1 ? (long)zero1_shard((uint64_t)C.P, P.dp) : C.P;
                    C.lo = std::min(C.P, (long)o.dp_rank * S1);
                    C.hi = std::min(C.P, C.lo + S1);
                    if (D.dtype == DT_BF16) {
                        C.master = (float*)q;
                        q += (size_t)S1 * 4;
                    } else {
                        C.master = (float*)C.w + C.lo;   // fp32: the weights are the master
                    }
                    C.m = (float*)q;
                    q += (size_t)S1 * 4;
                    C.v = (float*)q;
                } else {
                    CU(cudaHostAlloc(&C.h_master, (size_t)C.P * 4, cudaHostAllocDefault));
                    CU(cudaHostAlloc(&C.h_m, (size_t)C.P * 4, cudaHostAllocDefault));
                    CU(cudaHostAlloc(&C.h_v, (size_t)C.P * 4, cudaHostAllocDefault));
                    CU(cudaHostAlloc(&C.h_grad, (size_t)C.P * 4, cudaHostAllocDefault));
                    std::memset(C.h_m, 0, (size_t)C.P * 4);
                    std::memset(C.h_v, 0, (size_t)C.P * 4);
                    if (D.dtype == DT_BF16) CU(cudaHostAlloc(&C.h_w, (size_t)C.P * 2, cudaHostAllocDefault));
                    else C.h_w = C.h_master;
                    CU(cudaEventCreateWithFlags(&C.ev_d2h, cudaEventDisableTiming));
                    CU(cudaEventCreateWithFlags(&C.ev_h2d, cudaEventDisableTiming));
                    if (sopt) {   // staging slots follow w | grad in the static block
                        C.sopt = true;
                        C.slice = std::min<long>(C.P, TPIPE_SOPT_SLICE_PARAMS);
                        C.stg[0] = (float*)q;
                        C.stg[1] = C.stg[0] + 3 * C.slice;
                        CU(cudaEventCreateWithFlags(&C.ev_sopt_done, cudaEventDisableTiming));
                        CU(cudaEventCreateWithFlags(&C.ev_sopt_out, cudaEventDisableTiming));
                    }
                }
            } else if (b.category == TPIPE_CAT_IO) {
                if (b.mb == 0) S->tokens = (int*)ptr;
                else {
                    S->targets = (int*)ptr;
                    S->loss_slots = (float*)((uint8_t*)ptr + (size_t)P.m * D.M * 4);
                }
            }
        }
        rt->st[s] = std::move(S);
    }
    // stage transport (runtime/transport.h)
    CU(cudaDeviceSynchronize());   // static buffers initialised before peers map the arena
    rt->dp_rank = o.dp_rank;
    std::string ipc_pipe = o.ipc_name ? o.ipc_name : "";
    if (P.dp > 1) {
        StageState& S0 = *rt->st[o.stage];
        uint8_t* arena = (uint8_t*)S0.pool->arena();
        uint64_t w_off[5] = {0, 0, 0, 0, 0}, g_off[5] = {0, 0, 0, 0, 0};
        for (int c = 1; c <= P.v; ++c) {
            ChunkState& C = S0.ch[c];
            const uint8_t *w = (const uint8_t*)C.w, *g = (const uint8_t*)C.grad;
            if (w < arena || g < arena || w >= arena + S0.pool->arena_bytes())
                return set_error(TPIPE_E_STATE, "dp: model state outside the pool arena");
            w_off[c] = (uint64_t)(w - arena);
            g_off[c] = (uint64_t)(g - arena);
        }
        const std::string dp_name = std::string(o.ipc_name) + "_s" + std::to_string(o.stage);
        TRY(make_dp_group(P.dp, o.dp_rank, o.stage, P.v, dp_name.c_str(), arena, S0.pool->arena_bytes(), w_off,
                          g_off, rt->timeout_ms, &rt->dpg));
        for (int c = 1; c <= P.v; ++c) {
            ChunkState& C = S0.ch[c];
            for (int j = 0; j < P.dp; ++j) {
                C.dptr.grad[j] = rt->dpg->peer_grad(j, c);
                C.dptr.w[j] = rt->dpg->peer_w(j, c);
            }
        }
        ipc_pipe += "_r" + std::to_string(o.dp_rank);   // each replica's own pipeline rendezvous
    }
    if ((o.stage < 0 || P.p == 1) && o.transport == TPIPE_TRANSPORT_NCCL_LOOPBACK) {
        TRY(make_virtual_nccl_transport(P.channels, &rt->tr));
        rt->transport_kind = TPIPE_TRANSPORT_NCCL_LOOPBACK;
    } else if (o.stage < 0 || P.p == 1) {
        rt->tr = make_virtual_transport(P.channels);
        rt->transport_kind = -1;
    } else if (o.transport == TPIPE_TRANSPORT_IPC) {
        Pool& pl = *rt->st[o.stage]->pool;
        TRY(make_ipc_transport(P.channels, P.p, o.stage, o.device, ipc_pipe.c_str(), pl.arena(),
                               pl.arena_bytes(), P.W, rt->timeout_ms, &rt->tr));
        rt->transport_kind = TPIPE_TRANSPORT_IPC;
    } else if (o.transport == TPIPE_TRANSPORT_NCCL) {
        TRY(make_nccl_transport(P.channels, o.stage, o.nccl_ids, rt->timeout_ms, &rt->tr));
        rt->transport_kind = TPIPE_TRANSPORT_NCCL;
    } else {
        return set_error(TPIPE_E_INVALID, "transport %d", o.transport);
    }
    CU(cudaDeviceSynchronize());
    *out = rt.release();
    return 0;
}

TP_API void tpipe_runtime_destroy(tpipe_runtime* rt) {
    if (!rt) return;
    cudaSetDevice(rt->device);
    cudaDeviceSynchronize();
    for (int s : rt->owned) {
        for (void* hp : rt->st[s]->act_free) cudaFreeHost(hp);
        for (auto& kv : rt->st[s]->act_host) cudaFreeHost(kv.second);
        for (auto& C : rt->st[s]->ch) {
            join_host(C);
            if (C.h_master) cudaFreeHost(C.h_master);
            if (C.h_m) cudaFreeHost(C.h_m);
            if (C.h_v) cudaFreeHost(C.h_v);
            if (C.h_grad) cudaFreeHost(C.h_grad);
            if (C.h_w && C.h_w != C.h_master) cudaFreeHost(C.h_w);
            if (C.ev_d2h) cudaEventDestroy(C.ev_d2h);
            if (C.ev_h2d) cudaEventDestroy(C.ev_h2d);
            if (C.ev_sopt_done) cudaEventDestroy(C.ev_sopt_done);
            if (C.ev_sopt_out) cudaEventDestroy(C.ev_sopt_out);
        }
    }
    rt->tr.reset();
    rt->dpg.reset();
    for (auto& g : rt->gexec)
        if (g) cudaGraphExecDestroy(g);
    if (rt->hp_dev) cudaFree(rt->hp_dev);
    for (auto e : rt->evpool) cudaEventDestroy(e);
    for (auto e : rt->tevpool) cudaEventDestroy(e);
    if (rt->h_tok_stage) cudaFreeHost(rt->h_tok_stage);
    for (int s : rt->owned) {
        rt->st[s]->pool.reset();
        if (rt->st[s]->own) {
            stage_release_side_streams(rt->st[s]->own);
            cudaStreamDestroy(rt->st[s]->own);
        }
    }
    stage_release_side_streams(rt->stream);
    cudaStreamDestroy(rt->stream);
    cudaStreamDestroy(rt->d2h);
    cudaStreamDestroy(rt->h2d);
    cudaStreamDestroy(rt->opt);
    delete rt;
}

static int chunk_of(tpipe_runtime* rt, int32_t s, int32_t c, uint64_t n, ChunkState** out) {
    if (!rt || s < 0 || s >= rt->plan.p || !rt->st[s]) return set_error(TPIPE_E_INVALID, "stage not owned");
    if (c < 1 || c > rt->plan.v) return set_error(TPIPE_E_INVALID, "chunk");
    ChunkState& C = rt->st[s]->ch[c];
    if ((uint64_t)C.P != n) return set_error(TPIPE_E_INVALID, "n (%llu) != chunk params (%ld)",
                                             (unsigned long long)n, C.P);
    *out = &C;
    return 0;
}

TP_API int tpipe_runtime_set_params(tpipe_runtime* rt, int32_t s, int32_t c, const float* src,
                                    uint64_t n) {
    ChunkState* C;
    TRY(chunk_of(rt, s, c, n, &C));
    join_host(*C);
    CU(cudaSetDevice(rt->device));
    CU(cudaStreamSynchronize(rt->stream));
    // stream-ordered copies: a pageable cudaMemcpy may return before its DMA
    // lands, so the cast kernel below must be ordered on the same stream
    if (!C->offloaded) {
        // the full fp32 values go through the grad buffer (zeroed below): the
        // weights take all of them, the master only this replica's shard
        const long sh = C->hi - C->lo;
        if (rt->D.dtype == DT_BF16) {
            CU(cudaMemcpyAsync(C->grad, src, n * 4, cudaMemcpyHostToDevice, rt->stream));
            if (cast_f32_to(DT_BF16, C->grad, C->w, (long)n, rt->stream)) return set_error(TPIPE_E_CUDA, "cast");
            CU(cudaMemcpyAsync(C->master, C->grad + C->lo, (size_t)sh * 4, cudaMemcpyDeviceToDevice, rt->stream));
        } else {
            CU(cudaMemcpyAsync(C->w, src, n * 4, cudaMemcpyHostToDevice, rt->stream));
        }
        CU(cudaMemsetAsync(C->m, 0, (size_t)sh * 4, rt->stream));
        CU(cudaMemsetAsync(C->v, 0, (size_t)sh * 4, rt->stream));
    } else {
        std::memcpy(C->h_master, src, n * 4);
        std::memset(C->h_m, 0, n * 4);
        std::memset(C->h_v, 0, n * 4);
        if (rt->D.dtype == DT_BF16) host_cast_bf16(C->h_master, (uint16_t*)C->h_w, (long)n);
        CU(cudaMemcpyAsync(C->w, C->h_w, n * rt->D.es, cudaMemcpyHostToDevice, rt->stream));
    }
    CU(cudaMemsetAsync(C->grad, 0, n * 4, rt->stream));
    CU(cudaStreamSynchronize(rt->stream));
    rt->t = 0;
    return 0;
}

TP_API int tpipe_runtime_get_params(tpipe_runtime* rt, int32_t s, int32_t c, float* dst, uint64_t n) {
    ChunkState* C;
    TRY(chunk_of(rt, s, c, n, &C));
    join_host(*C);
    CU(cudaStreamSynchronize(rt->stream));
    if (C->offloaded) {
        std::memcpy(dst, C->h_master, n * 4);
    } else if (rt->D.dtype == DT_FP32) {
        CU(cudaMemcpyAsync(dst, C->w, n * 4, cudaMemcpyDeviceToHost, rt->stream));   // w is the master
    } else if (C->lo == 0 && C->hi == C->P) {
        CU(cudaMemcpyAsync(dst, C->master, n * 4, cudaMemcpyDeviceToHost, rt->stream));
    } else {
        // ZeRO-1 (R31): the master of this replica's shard; elsewhere the bf16
        // weights (= RNE of the owning replica's master) widened to fp32
        std::vector<uint16_t> wb(n);
        CU(cudaMemcpyAsync(wb.data(), C->w, n * 2, cudaMemcpyDeviceToHost, rt->stream));
        CU(cudaStreamSynchronize(rt->stream));
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t u = (uint32_t)wb[i] << 16;
            std::memcpy(&dst[i], &u, 4);
        }
        CU(cudaMemcpyAsync(dst + C->lo, C->master, (size_t)(C->hi - C->lo) * 4, cudaMemcpyDeviceToHost,
                           rt->stream));
    }
    CU(cudaStreamSynchronize(rt->stream));
    return 0;
}

TP_API int tpipe_runtime_get_grads(tpipe_runtime* rt, int32_t s, int32_t c, float* dst, uint64_t n) {
    ChunkState* C;
    TRY(chunk_of(rt, s, c, n, &C));
    CU(cudaStreamSynchronize(rt->stream));
    CU(cudaStreamSynchronize(rt->d2h));
    CU(cudaStreamSynchronize(rt->opt));
    CU(cudaMemcpyAsync(dst, C->grad, n * 4, cudaMemcpyDeviceToHost, rt->stream));
    CU(cudaStreamSynchronize(rt->stream));
    return 0;
}

TP_API int tpipe_step_device(tpipe_runtime* rt, const int32_t* tok, const int32_t* tgt, uint32_t flags,
                             float* loss_out) {
    if (!rt) return set_error(TPIPE_E_INVALID, "runtime is NULL");
    CU(cudaSetDevice(rt->device));
    return run_step(rt, tok, tgt, flags, loss_out);
}

TP_API int tpipe_step(tpipe_runtime* rt, const int32_t* tokens, const int32_t* targets, uint32_t flags,
                      float* loss_out) {
    if (!rt) return set_error(TPIPE_E_INVALID, "runtime is NULL");
    CU(cudaSetDevice(rt->device));
    const auto& P = rt->plan;
    const size_t io = (size_t)P.m * rt->D.M * 4;
    if (rt->h_tok_bytes < 2 * io) {
        if (rt->h_tok_stage) cudaFreeHost(rt->h_tok_stage);
        CU(cudaHostAlloc(&rt->h_tok_stage, 2 * io, cudaHostAllocDefault));
        rt->h_tok_bytes = 2 * io;
    }
    // host -> pinned staging -> HBM (the H2D is part of the step)
    for (int s : rt->owned) {
        StageState& S = *rt->st[s];
        if (s == 0 && tokens) {
            std::memcpy(rt->h_tok_stage, tokens, io);
            CU(cudaMemcpyAsync(S.tokens, rt->h_tok_stage, io, cudaMemcpyHostToDevice, rt->stream));
        }
        if (s == P.p - 1 && targets) {
            std::memcpy((uint8_t*)rt->h_tok_stage + io, targets, io);
            CU(cudaMemcpyAsync(S.targets, (uint8_t*)rt->h_tok_stage + io, io, cudaMemcpyHostToDevice,
                               rt->stream));
        }
    }
    return run_step(rt, nullptr, nullptr, flags, loss_out);
}

TP_API int tpipe_runtime_get_stats(const tpipe_runtime* rt, tpipe_runtime_stats* out) {
    if (!rt || !out) return set_error(TPIPE_E_INVALID, "NULL argument");
    std::memset(out, 0, sizeof(*out));
    for (int s : rt->owned) {
        if (s < 64) out->pool_high_water[s] = rt->st[s]->pool->high_water(s);
        out->pool_reserved += rt->st[s]->pool->reserved();
        out->pool_overflow_bytes += rt->st[s]->pool->overflow_bytes();
    }
    out->kernel_launches = rt->launches_last;
    out->step = rt->t;
    out->offload_d2h_bytes = rt->d2h_bytes;
    out->offload_h2d_bytes = rt->h2d_bytes;
    for (int s : rt->owned)
        for (auto& C : rt->st[s]->ch) out->host_opt_ms += C.host_ms;
    auto span_ms = [](const std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
        double ms = 0;
        for (auto& pr : v) {
            float x = 0;
            if (cudaEventSynchronize(pr.second) == cudaSuccess && cudaEventElapsedTime(&x, pr.first, pr.second) == cudaSuccess)
                ms += x;
        }
        return ms;
    };
    out->offload_d2h_ms = span_ms(rt->d2h_ev);
    out->offload_h2d_ms = span_ms(rt->h2d_ev);
    out->transport = rt->transport_kind;
    out->host_issue_ms = rt->host_issue_ms;
    for (int c = 0; c < 4; ++c) {
        out->kernel_ms[c] = rt->kms[c];
        out->kernel_flops[c] = rt->kflops[c];
        out->kernel_count[c] = rt->kcount[c];
    }
    return 0;
}

TP_API void* tpipe_runtime_stream(const tpipe_runtime* rt) { return rt ? (void*)rt->stream : nullptr; }

TP_API int tpipe_runtime_op_times(const tpipe_runtime* rt, int32_t stage, float* ms, size_t cap, size_t* n) {
    if (!rt || !n || stage < 0 || stage >= rt->plan.p) return set_error(TPIPE_E_INVALID, "stage");
    const auto& v = rt->op_ms.size() > (size_t)stage ? rt->op_ms[stage] : std::vector<float>();
    *n = v.size();
    if (ms)
        for (size_t i = 0; i < v.size() && i < cap; ++i) ms[i] = v[i];
    return 0;
}

TP_API void tpipe_set_side_stream(int on) { stage_set_side_stream(on); }
TP_API void tpipe_set_pdl(int on) { tpipe::set_pdl(on); }

TP_API int tpipe_nccl_unique_id(void* out128) {
    const NcclApi* N = nccl();
    if (!N) return set_error(TPIPE_E_NCCL, "libnccl.so.2 not loadable");
    if (!out128) return set_error(TPIPE_E_INVALID, "NULL argument");
    ncclResult_t r = N->GetUniqueId((ncclUniqueId*)out128);
    if (r != ncclSuccess) return set_error(TPIPE_E_NCCL, "ncclGetUniqueId: %s", N->GetErrorString(r));
    return 0;
}
