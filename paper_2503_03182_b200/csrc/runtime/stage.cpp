// Per-chunk forward / block-wise recompute / backward of the pre-LN GPT block
// stack (model reading DESIGN.md §2 = SURVEY N-1).
//
// Per layer, forward:
//   LN1 -> QKV GEMM(+bias) -> causal attention -> out-proj GEMM(+bias+residual)
//   -> LN2 -> FC1 GEMM(+bias, GELU fused: u stashed, g transient)
//   -> FC2 GEMM(+bias+residual).
// Saved per layer (20h+16+4a bytes/token in bf16, N-2 with op-level recompute):
//   x_in, LN1 stats, qkv, attn out, LSE, x_mid, LN2 stats, u.
// Backward recomputes LN outputs from saved stats and GELU(u) inside the FC2
// dgrad epilogue (operator-level recompute), and P from the LSE in
// the attention backward. Weight gradients accumulate (fp32, beta = 1) per
// micro-batch in index order; no atomics anywhere, so recompute on/off and
// offload on/off give bit-identical gradients.
#include "runtime/stage.h"

#include <mutex>
#include <vector>

#include <array>

namespace tpipe {

Dims::Dims(const tpipe_model_desc& d)
    : dtype(d.dtype == TPIPE_BF16 ? DT_BF16 : DT_FP32),
      M(d.micro_batch * d.seq_len),
      h(d.hidden),
      a(d.n_heads),
      hd(d.hidden / d.n_heads),
      f(d.ffn_hidden),
      V(d.vocab),
      s(d.seq_len),
      b(d.micro_batch),
      es(d.dtype == TPIPE_BF16 ? 2 : 4) {}

ParamLayout make_param_layout(const tpipe_model_desc& d, int n_layers, bool emb, bool head) {
    ParamLayout P;
    P.emb = emb;
    P.head = head;
    const long h = d.hidden, f = d.ffn_hidden, V = d.vocab, s = d.seq_len;
    long off = 0;
    auto seg = [&](long n, int decay) {
        P.segments.push_back({off, n, decay});
        long o = off;
        off += n;
        return o;
    };
    if (emb) {
        P.wte = seg(V * h, 1);
        P.wpe = seg(s * h, 1);
    }
    const long sizes[N_LAYER_TENSORS] = {h, h, 3 * h * h, 3 * h, h * h, h, h, h, f * h, f, h * f, h};
    const int decay[N_LAYER_TENSORS] = {0, 0, 1, 0, 1, 0, 0, 0, 1, 0, 1, 0};
    for (int l = 0; l < n_layers; ++l) {
        std::array<long, N_LAYER_TENSORS> o{};
        for (int t = 0; t < N_LAYER_TENSORS; ++t) o[t] = seg(sizes[t], decay[t]);
        P.layer.push_back(o);
    }
    if (head) {
        P.lnf_g = seg(h, 0);
        P.lnf_b = seg(h, 0);
        P.w_head = seg(V * h, 1);
    }
    P.total = off;
    return P;
}

StashLayout make_stash_layout(const tpipe_model_desc& d, int n_layers, bool emb, bool head,
                              bool ckpt_only, int ckpt_layers) {
    // layer-grouped recompute (1F1B + recompute): layers [0, ck) keep only
    // their input (checkpoint), the deeper ones their full stash (DESIGN R33)
    const int ck = !ckpt_only ? 0 : (ckpt_layers > 0 && ckpt_layers < n_layers ? ckpt_layers : n_layers);
    StashLayout S;
    S.ckpt_only = ck > 0;
    S.ckpt_layers = ck;
    const long M = (long)d.micro_batch * d.seq_len, h = d.hidden, a = d.n_heads, f = d.ffn_hidden;
    const long es = d.dtype == TPIPE_BF16 ? 2 : 4;
    long off = 0;
    auto take = [&](long bytes) {
        long o = off;
        off += bytes;
        return o;
    };
    auto internals = [&](StashLayout::L& L) {
        L.ln1_mean = take(4 * M);
        L.ln1_rstd = take(4 * M);
        L.qkv = take(3 * M * h * es);
        L.o = take(M * h * es);
        L.lse = take(4 * a * M);
        L.x_mid = take(M * h * es);
        L.ln2_mean = take(4 * M);
        L.ln2_rstd = take(4 * M);
        L.u = take(M * f * es);
    };
    for (int l = 0; l < n_layers; ++l) {
        StashLayout::L L{};
        L.x_in = (l == 0 && !emb) ? -1 : take(M * h * es);
        if (l >= ck) internals(L);
        S.layer.push_back(L);
    }
    if (head) {
        S.x_f = take(M * h * es);
        S.lnf_mean = take(4 * M);
        S.lnf_rstd = take(4 * M);
        S.ce_lse = take(4 * M);
    }
    S.total = off;
    if (ck > 0) {
        off = 0;
        S.scratch.x_in = -1;
        internals(S.scratch);
        S.scratch_bytes = off;
    }
    return S;
}

// ---------------------------------------------------------------- helpers
#define TRY(x)                        \
    do {                              \
        int _rc = (x);                \
        if (_rc) return _rc;          \
    } while (0)

template <typename T>
static inline T* at(void* base, long byte_off) {
    return reinterpret_cast<T*>(reinterpret_cast<uint8_t*>(base) + byte_off);
}

KernelProfiler& profiler() {
    static KernelProfiler P;
    return P;
}
cudaEvent_t KernelProfiler::ev() {
    if (next == pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        pool.push_back(e);
    }
    return pool[next++];
}
void KernelProfiler::collect(double ms[4], double flops[4], int64_t count[4]) {
    for (int c = 0; c < 4; ++c) ms[c] = flops[c] = 0, count[c] = 0;
    for (auto& r : recs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        ms[r.cls] += t;
        flops[r.cls] += r.flops;
        count[r.cls] += 1;
    }
}
KernelProfiler::~KernelProfiler() {
    for (auto e : pool) cudaEventDestroy(e);
}

// bracket one launch with events when profiling
struct ProfScope {
    KernelProfiler& P;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    int cls;
    double flops;
    ProfScope(int c, double f, cudaStream_t s) : P(profiler()), st(s), cls(c), flops(f) {
        if (P.on) {
            a = P.ev();
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (P.on) {
            cudaEvent_t b = P.ev();
            cudaEventRecord(b, st);
            P.recs.push_back({a, b, cls, flops});
        }
    }
};

static int mm(const Dims& D, int M, int N, int K, const void* A, long lda, int ak, const void* B,
              long ldb, int bk, int epi, void* C, long ldc, const void* bias = nullptr,
              const void* R = nullptr, long ldr = 0, void* C2 = nullptr, long ldc2 = 0,
              const void* aux = nullptr, long ldaux = 0, cudaStream_t st = nullptr) {
    GemmDesc g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_kmajor = ak;
    g.B = B; g.ldb = ldb; g.b_kmajor = bk;
    g.epi = epi; g.C = C; g.ldc = ldc; g.bias = bias; g.res = R; g.ldr = ldr;
    g.C2 = C2; g.ldc2 = ldc2; g.aux = aux; g.ldaux = ldaux;
    ProfScope ps(0, 2.0 * M * N * K, st);
    return gemm(D.dtype, g, st) ? -7 : 0;
}

struct LayerPtrs {  // one layer's saved tensors
    const void* x_in;
    float *ln1_mean, *ln1_rstd;
    void *qkv, *o;
    float* lse;
    void* x_mid;
    float *ln2_mean, *ln2_rstd;
    void* u;
};

static LayerPtrs layer_ptrs(const StashLayout::L& L, uint8_t* stash, const void* x_in) {
    LayerPtrs p;
    p.x_in = L.x_in >= 0 ? (const void*)(stash + L.x_in) : x_in;
    p.ln1_mean = at<float>(stash, L.ln1_mean);
    p.ln1_rstd = at<float>(stash, L.ln1_rstd);
    p.qkv = stash + L.qkv;
    p.o = stash + L.o;
    p.lse = at<float>(stash, L.lse);
    p.x_mid = stash + L.x_mid;
    p.ln2_mean = at<float>(stash, L.ln2_mean);
    p.ln2_rstd = at<float>(stash, L.ln2_rstd);
    p.u = stash + L.u;
    return p;
}

// partial T-Recomp (R25): base pointer for layer l's StashLayout offsets; the
// kept part [split, n) of the chunk stash starts at layer split's x_in
static uint8_t* stash_base(const StashLayout& SL, uint8_t* stash, uint8_t* stash2, int split, int l) {
    if (split <= 0 || l < split) return stash;
    return stash2 - SL.layer[split].x_in;
}

// full recompute: layer input from the checkpoint stash, internals in `scratch`
static LayerPtrs scratch_ptrs(const StashLayout& SL, int l, uint8_t* stash, const void* x_in,
                              uint8_t* scratch) {
    LayerPtrs p = layer_ptrs(SL.scratch, scratch, nullptr);
    p.x_in = SL.layer[l].x_in >= 0 ? (const void*)(stash + SL.layer[l].x_in) : x_in;
    return p;
}

struct LW {  // one layer's weights (es) and fp32 grads
    const void* w[N_LAYER_TENSORS];
    float* g[N_LAYER_TENSORS];
};

static LW layer_w(const Dims& D, const ChunkParamsDev& P, int l) {
    LW r;
    for (int t = 0; t < N_LAYER_TENSORS; ++t) {
        r.w[t] = reinterpret_cast<const uint8_t*>(P.w) + P.lay->layer[l][t] * D.es;
        r.g[t] = P.grad + P.lay->layer[l][t];
    }
    return r;
}

// forward of one layer: x_in -> out, saving into lp; ws_ln [M,h], ws_g [M,f]
static int layer_forward(const Dims& D, const LW& W, const LayerPtrs& lp, void* ws_ln, void* ws_g,
                         void* out, cudaStream_t st) {
    const int M = D.M, h = D.h, f = D.f;
    {
        ProfScope _ps(3, 0.0, st);
        TRY(ln_fwd(D.dtype, lp.x_in, W.w[LN1_G], W.w[LN1_B], ws_ln, lp.ln1_mean, lp.ln1_rstd, M, h, st));
    }
    TRY(mm(D, M, 3 * h, h, ws_ln, h, 1, W.w[W_QKV], h, 1, EPI_BIAS, lp.qkv, 3 * h, W.w[B_QKV],
           nullptr, 0, nullptr, 0, nullptr, 0, st));
    {
        ProfScope ps(1, 4.0 * D.b * D.a * (0.5 * D.s * (D.s + 1)) * D.hd, st);
        TRY(attn_fwd(D.dtype, lp.qkv, lp.o, lp.lse, D.b, D.s, D.a, D.hd, st));
    }
    TRY(mm(D, M, h, h, lp.o, h, 1, W.w[W_O], h, 1, EPI_BIAS_RES, lp.x_mid, h, W.w[B_O], lp.x_in, h,
           nullptr, 0, nullptr, 0, st));
    {
        ProfScope _ps(3, 0.0, st);
        TRY(ln_fwd(D.dtype, lp.x_mid, W.w[LN2_G], W.w[LN2_B], ws_ln, lp.ln2_mean, lp.ln2_rstd, M, h, st));
    }
    TRY(mm(D, M, f, h, ws_ln, h, 1, W.w[W_1], h, 1, EPI_BIAS_GELU, lp.u, f, W.w[B_1], nullptr, 0,
           ws_g, f, nullptr, 0, st));
    TRY(mm(D, M, h, f, ws_g, f, 1, W.w[W_2], f, 1, EPI_BIAS_RES, out, h, W.w[B_2], lp.x_mid, h,
           nullptr, 0, nullptr, 0, st));
    return 0;
}

// backward workspace carve-up (ws_b)
struct BwdWs {
    void *G0, *G1, *du, *g, *ln, *dln, *dout;
    void* dqkv;
    float* Dv;
    float* part;
    uint8_t* rbuf;  // one-layer recompute buffer (full-recompute strategy)
    void *lnf, *dlnf;
    float* logits;     // fp32 mode only
    void* dlogits;
    float *ce_part, *ce_zt, *ce_lrow;   // bf16 fused head (K8)
    int* emb_ws;
    long total;     // bytes carved (== the plan's ws_b; checked at runtime creation)
};

static BwdWs carve_bwd(const Dims& D, uint8_t* ws, bool head, bool emb, long part_elems,
                       long rbuf_bytes) {
    const long M = D.M, h = D.h, f = D.f, es = D.es;
    BwdWs w;
    long off = 0;
    auto take = [&](long bytes) {
        uint8_t* p = ws + off;
        off += bytes;
        return p;
    };
    w.G0 = take(M * h * es);
    w.G1 = take(M * h * es);
    w.du = take(M * f * es);
    w.g = take(M * f * es);
    w.ln = take(M * h * es);
    w.dln = take(M * h * es);
    w.dout = take(M * h * es);
    w.dqkv = take(3 * M * h * es);
    w.Dv = reinterpret_cast<float*>(take(4L * D.a * M));
    w.part = reinterpret_cast<float*>(take(4 * part_elems));
    w.rbuf = rbuf_bytes ? take(rbuf_bytes) : nullptr;
    w.lnf = w.dlnf = w.dlogits = nullptr;
    w.logits = nullptr;
    w.ce_part = w.ce_zt = w.ce_lrow = nullptr;
    if (head) {
        w.lnf = take(M * h * es);
        w.dlnf = take(M * h * es);
        if (D.dtype == DT_BF16) {   // fused LM head + CE (K8, DESIGN R30): no [M, V] logits
            w.dlogits = take(M * D.V * es);
            w.ce_part = reinterpret_cast<float*>(take(8 * M * (long)ce_groups(D.V)));
            w.ce_zt = reinterpret_cast<float*>(take(4 * M));
            w.ce_lrow = reinterpret_cast<float*>(take(4 * M));
        } else {
            w.logits = reinterpret_cast<float*>(take(4 * M * D.V));
            w.dlogits = take(M * D.V * es);
        }
    }
    w.emb_ws = emb ? reinterpret_cast<int*>(take(8 * M)) : nullptr;
    w.total = off;
    return w;
}

static long part_elems(const Dims& D) {
    // column-partial workspace: b1 [nb][f] + LN2 [3][nb][h], or bqkv [nb][3h] + LN1 [3][nb][h]
    const long nb = (D.M + 15) / 16;
    return nb * (D.f + 3L * D.h > 6L * D.h ? D.f + 3L * D.h : 6L * D.h);
}

uint64_t bwd_ws_bytes(const Dims& D, const StashLayout& SL, bool head, bool emb) {
    return (uint64_t)carve_bwd(D, nullptr, head, emb, part_elems(D), SL.ckpt_only ? SL.scratch_bytes : 0).total;
}

// chunk_forward's workspace: [ln out M·h | gelu out M·f | full recompute: one
// layer's internals | head: LN_f out M·h]
uint64_t fwd_ws_bytes(const Dims& D, const StashLayout& SL, bool head) {
    return (uint64_t)D.M * (D.h + D.f) * D.es + (SL.ckpt_only ? SL.scratch_bytes : 0) +
           (head ? (uint64_t)D.M * D.h * D.es : 0);
}

// Side stream for the backward of a layer: weight-gradient GEMMs (and the LN
// recomputes that feed them) are independent of the data-gradient chain, so
// they run concurrently on a second stream and fill the SMs the other
// chain's last GEMM wave leaves idle (each tcgen05 GEMM is a persistent grid
// of <= #SMs CTAs; a 2048-multiple shape occupies ~86% of the SM-waves).
// One side stream + events per compute stream, created on first use.
struct SideStream {
    int dev = 0;
    cudaStream_t main = nullptr, aux = nullptr;
    // ev[0..4]: within a layer; ev[5..7]: the aux stream's FC1 wgrad, out-proj
    // wgrad and QKV wgrad of a layer, waited on by the next layer's main-stream
    // writers of the buffers they read (deferred join, layer_backward); ev[8]:
    // dlogits ready for the LM-head weight gradient on aux (chunk_backward)
    cudaEvent_t ev[9] = {};
};
static std::mutex g_side_mu;
static std::vector<SideStream*> g_side;
static SideStream* side_stream(cudaStream_t main) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_side_mu);
    for (auto* s : g_side)
        if (s->main == main && s->dev == dev) return s;
    auto* s = new SideStream;
    s->dev = dev;
    s->main = main;
    if (cudaStreamCreateWithFlags(&s->aux, cudaStreamNonBlocking) != cudaSuccess) {
        delete s;
        return nullptr;
    }
    for (auto& e : s->ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            delete s;
            return nullptr;
        }
    g_side.push_back(s);
    return s;
}
void stage_release_side_streams(cudaStream_t main) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_side_mu);
    for (size_t i = 0; i < g_side.size();) {
        SideStream* s = g_side[i];
        if (s->main == main && s->dev == dev) {
            cudaStreamSynchronize(s->aux);
            cudaStreamDestroy(s->aux);
            for (auto e : s->ev) cudaEventDestroy(e);
            delete s;
            g_side.erase(g_side.begin() + i);
        } else {
            ++i;
        }
    }
}
static bool g_side_stream_enabled = true;
void stage_set_side_stream(int on) { g_side_stream_enabled = on != 0; }

// `b` waits for everything issued so far on `a`
static int stream_dep(cudaStream_t a, cudaStream_t b, cudaEvent_t e) {
    if (a == b) return 0;
    if (cudaEventRecord(e, a) != cudaSuccess) return -3;
    return cudaStreamWaitEvent(b, e, 0) == cudaSuccess ? 0 : -3;
}

// backward of one layer: dy -> dx (dx may alias G0 == dy buffer: dy is fully
// consumed before the LN1 backward writes dx)
//   main: fc2 dgrad | colsum b1, fc1 dgrad, LN2 bwd (+b2) | out dgrad, attn bwd
//         | colsum bqkv, qkv dgrad, LN1 bwd (+bo) | join
//   aux : (after fc2 dgrad) fc2 wgrad, LN2 apply, fc1 wgrad, LN1 apply
//         | (after LN2 bwd) out wgrad | (after attn bwd) qkv wgrad
// Every buffer is written and read on one stream or ordered by an event
// (the partial-sum workspace is used on main only; dy is read by fc2 wgrad on
// aux before LN1 bwd overwrites it on main: ev[2]).
// wait_prev: the previous layer's backward deferred its join (its aux-stream
// weight gradients may still run): wait for the ones that read a buffer this
// layer's main stream is about to overwrite (w.du / w.g, w.G1, w.dqkv).
// defer_join: leave this layer's aux work running into the next layer's
// backward (the next layer must be called with wait_prev) instead of joining.
static int layer_backward(const Dims& D, const LW& W, const LayerPtrs& lp, const void* dy, void* dx,
                          const BwdWs& w, cudaStream_t st, bool wait_prev = false, bool defer_join = false) {
    const int M = D.M, h = D.h, f = D.f, dt = D.dtype;
    SideStream* ss = (g_side_stream_enabled && !profiler().on) ? side_stream(st) : nullptr;
    const cudaStream_t ax = ss ? ss->aux : st;
    cudaEvent_t* ev = ss ? ss->ev : nullptr;
    if (!ss) wait_prev = defer_join = false;
    // (previous layer's FC2 / FC1 wgrads read w.g / w.du, written next)
    if (wait_prev && cudaStreamWaitEvent(st, ev[5], 0) != cudaSuccess) return -3;
    // FC2: dg = dy W2 (dGELU fused: du = dg * gelu'(u), g = gelu(u) recomputed)
    TRY(mm(D, M, f, h, dy, h, 1, W.w[W_2], f, 0, EPI_DGELU, w.du, f, nullptr, nullptr, 0, w.g, f,
           lp.u, f, st));
    if (ss) TRY(stream_dep(st, ax, ev[0]));
    // ---- aux: weight gradients of FC2 / FC1 and the LN recomputes
    TRY(mm(D, h, f, M, dy, h, 0, w.g, f, 0, EPI_ACC_F32, W.g[W_2], f, nullptr, nullptr, 0, nullptr,
           0, nullptr, 0, ax));
    if (ss && cudaEventRecord(ev[1], ax) != cudaSuccess) return -3;   // dy consumed on aux
    {
        ProfScope _ps(3, 0.0, ax);
        TRY(ln_apply(dt, lp.x_mid, W.w[LN2_G], W.w[LN2_B], lp.ln2_mean, lp.ln2_rstd, w.ln, M, h, ax));
    }
    TRY(mm(D, f, h, M, w.du, f, 0, w.ln, h, 0, EPI_ACC_F32, W.g[W_1], h, nullptr, nullptr, 0,
           nullptr, 0, nullptr, 0, ax));
    if (defer_join && cudaEventRecord(ev[5], ax) != cudaSuccess) return -3;
    // ---- main: data-gradient chain. bf16: the b1 column partials and LN2's
    // (gamma, beta, b2) partials sit side by side in w.part and are reduced by
    // one launch after the LN2 backward (same per-column order)
    const long nb16 = (M + 15) / 16;
    float* part_b = w.part + nb16 * f;
    bool deferred = false;
    {
        ProfScope _ps(3, 0.0, st);
        const int rc = colsum_partials(dt, w.du, w.part, M, f, st);
        if (rc > 0 || rc < -1) return rc;
        deferred = rc == 0;
        if (!deferred) TRY(colsum_acc(dt, w.du, W.g[B_1], w.part, M, f, st));
    }
    TRY(mm(D, M, h, f, w.du, f, 1, W.w[W_1], h, 0, EPI_STORE, w.dln, h, nullptr, nullptr, 0,
           nullptr, 0, nullptr, 0, st));
    // (previous layer's out-proj wgrad reads w.G1, written next)
    if (wait_prev && cudaStreamWaitEvent(st, ev[6], 0) != cudaSuccess) return -3;
    {
        ProfScope _ps(3, 0.0, st);
        // + dB2 = colsum(dy), fused (dy is LN2's residual-branch gradient)
        if (deferred && ln_bwd_partials(dt, w.dln, lp.x_mid, W.w[LN2_G], lp.ln2_mean, lp.ln2_rstd, dy, w.G1,
                                        part_b, M, h, 1, st) == 0) {
            const float* src[4] = {w.part, part_b, part_b + nb16 * h, part_b + 2 * nb16 * h};
            float* out[4] = {W.g[B_1], W.g[LN2_G], W.g[LN2_B], W.g[B_2]};
            const int n[4] = {f, h, h, h};
            TRY(reduce_segments(src, out, n, 4, M, st));
        } else {
            if (deferred) TRY(reduce_segments((const float* const*)&w.part, &W.g[B_1], &f, 1, M, st));
            TRY(ln_bwd(dt, w.dln, lp.x_mid, W.w[LN2_G], lp.ln2_mean, lp.ln2_rstd, dy, w.G1, W.g[LN2_G],
                       W.g[LN2_B], w.part, M, h, st, W.g[B_2]));
        }
    }
    // aux (in order after FC1 wgrad, so w.ln is free): LN1 recompute; then,
    // once G1 exists, the out-proj weight gradient
    {
        ProfScope _ps(3, 0.0, ax);
        TRY(ln_apply(dt, lp.x_in, W.w[LN1_G], W.w[LN1_B], lp.ln1_mean, lp.ln1_rstd, w.ln, M, h, ax));
    }
    if (ss) TRY(stream_dep(st, ax, ev[2]));
    TRY(mm(D, h, h, M, w.G1, h, 0, lp.o, h, 0, EPI_ACC_F32, W.g[W_O], h, nullptr, nullptr, 0,
           nullptr, 0, nullptr, 0, ax));
    if (defer_join && cudaEventRecord(ev[6], ax) != cudaSuccess) return -3;
    // main: out-proj dgrad, attention backward (P recomputed from LSE). On the
    // tcgen05 path the dgrad GEMM's epilogue also produces the backward's
    // D = rowsum(dO o O) per (token, head) (EPI_STORE_DOT): no separate pass
    const bool fuse_d = dt == DT_BF16 && (D.hd == 64 || D.hd == 128);
    if (fuse_d) {
        GemmDesc g;
        g.M = M; g.N = h; g.K = h;
        g.A = w.G1; g.lda = h; g.a_kmajor = 1;
        g.B = W.w[W_O]; g.ldb = h; g.b_kmajor = 0;
        g.epi = EPI_STORE_DOT; g.C = w.dout; g.ldc = h;
        g.aux = lp.o; g.ldaux = h; g.part = w.Dv; g.dot_s = D.s; g.dot_hd = D.hd;
        ProfScope ps(0, 2.0 * M * h * h, st);
        if (gemm(dt, g, st)) return -7;
    } else {
        TRY(mm(D, M, h, h, w.G1, h, 1, W.w[W_O], h, 0, EPI_STORE, w.dout, h, nullptr, nullptr, 0,
               nullptr, 0, nullptr, 0, st));
    }
    // (previous layer's QKV wgrad reads w.dqkv, written next)
    if (wait_prev && cudaStreamWaitEvent(st, ev[7], 0) != cudaSuccess) return -3;
    {
        // algorithmic: P recompute + dV, dP, dQ, dK = 5 GEMMs over the causal triangle
        ProfScope ps(2, 10.0 * D.b * D.a * (0.5 * D.s * (D.s + 1)) * D.hd, st);
        TRY(attn_bwd(dt, lp.qkv, lp.o, w.dout, lp.lse, w.dqkv, w.Dv, D.b, D.s, D.a, D.hd, st, fuse_d));
    }
    if (ss) TRY(stream_dep(st, ax, ev[3]));
    // aux: QKV weight gradient
    TRY(mm(D, 3 * h, h, M, w.dqkv, 3 * h, 0, w.ln, h, 0, EPI_ACC_F32, W.g[W_QKV], h, nullptr,
           nullptr, 0, nullptr, 0, nullptr, 0, ax));
    if (defer_join && cudaEventRecord(ev[7], ax) != cudaSuccess) return -3;
    // main: QKV bias / dgrad, LN1 backward (bqkv and LN1's (gamma, beta, bo)
    // partials reduced together, as above)
    float* part_q = w.part + nb16 * 3 * h;
    {
        ProfScope _ps(3, 0.0, st);
        const int rc = colsum_partials(dt, w.dqkv, w.part, M, 3 * h, st);
        if (rc > 0 || rc < -1) return rc;
        deferred = rc == 0;
        if (!deferred) TRY(colsum_acc(dt, w.dqkv, W.g[B_QKV], w.part, M, 3 * h, st));
    }
    TRY(mm(D, M, h, 3 * h, w.dqkv, 3 * h, 1, W.w[W_QKV], h, 0, EPI_STORE, w.dln, h, nullptr,
           nullptr, 0, nullptr, 0, nullptr, 0, st));
    if (ss && cudaStreamWaitEvent(st, ev[1], 0) != cudaSuccess) return -3;   // dx may alias dy
    {
        ProfScope _ps(3, 0.0, st);
        // + dBo = colsum(G1), fused (G1 is LN1's residual-branch gradient)
        if (deferred && ln_bwd_partials(dt, w.dln, lp.x_in, W.w[LN1_G], lp.ln1_mean, lp.ln1_rstd, w.G1, dx,
                                        part_q, M, h, 1, st) == 0) {
            const float* src[4] = {w.part, part_q, part_q + nb16 * h, part_q + 2 * nb16 * h};
            float* out[4] = {W.g[B_QKV], W.g[LN1_G], W.g[LN1_B], W.g[B_O]};
            const int n[4] = {3 * h, h, h, h};
            TRY(reduce_segments(src, out, n, 4, M, st));
        } else {
            if (deferred) {
                const int n3 = 3 * h;
                TRY(reduce_segments((const float* const*)&w.part, &W.g[B_QKV], &n3, 1, M, st));
            }
            TRY(ln_bwd(dt, w.dln, lp.x_in, W.w[LN1_G], lp.ln1_mean, lp.ln1_rstd, w.G1, dx, W.g[LN1_G],
                       W.g[LN1_B], w.part, M, h, st, W.g[B_O]));
        }
    }
    // join: the layer's gradients are complete and w.* free for the next layer
    // (deferred: the next layer waits on ev[5..7] where it needs to)
    if (ss && !defer_join) TRY(stream_dep(ax, st, ev[4]));
    return 0;
}

int chunk_forward(const Dims& D, const StashLayout& SL, const ChunkParamsDev& P, const FwdArgs& a,
                  cudaStream_t st) {
    const ParamLayout& lay = *P.lay;
    const int n = (int)lay.layer.size();
    const long M = D.M, h = D.h;
    uint8_t* ws = a.ws;
    void* ws_ln = ws;
    void* ws_g = ws + M * h * D.es;
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(P.w);
    uint8_t* scratch = ws + M * (h + D.f) * D.es;   // full-recompute: one layer's internals
    if (lay.emb)
        {
            ProfScope _ps(3, 0.0, st);
            TRY(embed_fwd(D.dtype, a.tokens, wb + lay.wte * D.es, wb + lay.wpe * D.es,
                      a.stash + SL.layer[0].x_in, D.M, D.s, D.h, st));
        }
    const int n_run = a.n_run > 0 ? a.n_run : n;
    for (int l = 0; l < n_run; ++l) {
        LayerPtrs lp = l < SL.ckpt_layers ? scratch_ptrs(SL, l, a.stash, a.in, scratch)
                                    : layer_ptrs(SL.layer[l], stash_base(SL, a.stash, a.stash2, a.split, l), a.in);
        void* out;
        if (l + 1 < n_run) out = stash_base(SL, a.stash, a.stash2, a.split, l + 1) + SL.layer[l + 1].x_in;
        else if (l + 1 < n) out = ws_ln;    // partial recompute: layer n_run's input is kept
        else if (lay.head) out = a.stash + SL.x_f;
        else out = a.out ? a.out : ws_ln;   // recompute: discard into free scratch
        TRY(layer_forward(D, layer_w(D, P, l), lp, ws_ln, ws_g, out, st));
    }
    if (lay.head && a.targets) {
        // LN_f forward only: its statistics are stashed for the backward. The
        // logits, LSE, loss and dlogits are all produced in the head chunk's
        // backward (the loss is read after the step), so the [M, V] LM-head
        // GEMM runs once per micro-batch instead of once in F and again in B.
        // (On the last stage B(p-1,c,i) directly follows F(p-1,c,i) in T-Pipe,
        // B = F+1, and in 1F1B, so nothing is held longer.)
        uint8_t* lnf = scratch + SL.scratch_bytes;
        ProfScope _ps(3, 0.0, st);
        TRY(ln_fwd(D.dtype, a.stash + SL.x_f, wb + lay.lnf_g * D.es, wb + lay.lnf_b * D.es, lnf,
                   at<float>(a.stash, SL.lnf_mean), at<float>(a.stash, SL.lnf_rstd), M, h, st));
    }
    return 0;
}

int chunk_backward(const Dims& D, const StashLayout& SL, const ChunkParamsDev& P, const BwdArgs& a,
                   cudaStream_t st) {
    const ParamLayout& lay = *P.lay;
    const int n = (int)lay.layer.size();
    const long M = D.M, h = D.h;
    BwdWs w = carve_bwd(D, a.ws, lay.head, lay.emb, part_elems(D), SL.ckpt_only ? SL.scratch_bytes : 0);
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(P.w);
    const void* dy = a.gin;
    bool head_on_aux = false;
    if (lay.head) {
        const void* ln_g = wb + lay.lnf_g * D.es;
        {
            ProfScope _ps(3, 0.0, st);
            TRY(ln_apply(D.dtype, a.stash + SL.x_f, ln_g, wb + lay.lnf_b * D.es,
                     at<float>(a.stash, SL.lnf_mean), at<float>(a.stash, SL.lnf_rstd), w.lnf, M, h,
                     st));
        }
        const void* wh = wb + lay.w_head * D.es;
        float* lse = at<float>(a.stash, SL.ce_lse);
        if (D.dtype == DT_BF16) {
            // fused LM head + softmax CE (K8, DESIGN R30): the head GEMM runs twice
            // and the logits live only in TMEM / registers. Pass 1: per-row
            // (max, sum exp) over 128-column groups + the target logit; a small
            // combine gives LSE and the loss; pass 2 recomputes the logits and
            // writes dlogits = (softmax - onehot) * scale in bf16.
            GemmDesc g;
            g.M = M; g.N = D.V; g.K = h;
            g.A = w.lnf; g.lda = h; g.a_kmajor = 1;
            g.B = wh; g.ldb = h; g.b_kmajor = 1;
            g.epi = EPI_LSE_PART;
            g.targets = a.targets;
            g.part = w.ce_part;
            g.zt = w.ce_zt;
            {
                ProfScope ps(0, 2.0 * M * D.V * h, st);
                if (gemm(D.dtype, g, st)) return -7;
            }
            {
                ProfScope _ps(3, 0.0, st);
                TRY(ce_combine(w.ce_part, ce_groups(D.V), w.ce_zt, lse, w.ce_lrow, a.loss_slot, a.loss_scale,
                               M, st));
            }
            g.epi = EPI_CE_GRAD;
            g.lse = lse;
            g.C = w.dlogits;
            g.ldc = D.V;
            g.scale = a.loss_scale;
            {
                ProfScope ps(0, 2.0 * M * D.V * h, st);
                if (gemm(D.dtype, g, st)) return -7;
            }
        } else {
            TRY(mm(D, M, D.V, h, w.lnf, h, 1, wh, h, 1, EPI_STORE_F32, w.logits, D.V, nullptr, nullptr,
                   0, nullptr, 0, nullptr, 0, st));
            ProfScope _ps(3, 0.0, st);
            // LSE and loss (the forward deferred them: see chunk_forward), then dlogits
            TRY(ce_fwd(w.logits, a.targets, lse, a.loss_slot, a.loss_scale, M, D.V, st));
            TRY(ce_bwd(D.dtype, w.logits, a.targets, lse, w.dlogits, a.loss_scale, M, D.V, st));
        }
        // LM-head weight gradient on the side stream, concurrent with the head's
        // data gradient (a single wave of 64 CTA-pair tiles with a 50K-deep K
        // loop leaves 10 of 74 pairs idle); dlogits / lnf are head-only
        // workspace, untouched until the chunk's final join
        SideStream* hs = (g_side_stream_enabled && !profiler().on) ? side_stream(st) : nullptr;
        const cudaStream_t hax = hs ? hs->aux : st;
        if (hs) TRY(stream_dep(st, hax, hs->ev[8]));
        TRY(mm(D, D.V, h, M, w.dlogits, D.V, 0, w.lnf, h, 0, EPI_ACC_F32, P.grad + lay.w_head, h,
               nullptr, nullptr, 0, nullptr, 0, nullptr, 0, hax));
        head_on_aux = hs != nullptr;
        TRY(mm(D, M, h, D.V, w.dlogits, D.V, 1, wh, h, 0, EPI_STORE, w.dlnf, h, nullptr, nullptr, 0,
               nullptr, 0, nullptr, 0, st));
        {
            ProfScope _ps(3, 0.0, st);
            TRY(ln_bwd(D.dtype, w.dlnf, a.stash + SL.x_f, ln_g, at<float>(a.stash, SL.lnf_mean),
                   at<float>(a.stash, SL.lnf_rstd), nullptr, w.G0, P.grad + lay.lnf_g,
                   P.grad + lay.lnf_b, w.part, M, h, st));
        }
        dy = w.G0;
    }
    bool prev_deferred = false;
    for (int l = n - 1; l >= 0; --l) {
        LayerPtrs lp;
        if (l < SL.ckpt_layers) {
            // layer-grouped just-in-time recompute (1F1B + full recompute):
            // regenerate this layer's internals from its checkpoint, output discarded
            lp = scratch_ptrs(SL, l, a.stash, a.in, w.rbuf);
            TRY(layer_forward(D, layer_w(D, P, l), lp, w.ln, w.g, w.dout, st));
        } else {
            lp = layer_ptrs(SL.layer[l], stash_base(SL, a.stash, a.stash2, a.split, l), a.in);
        }
        void* dx = (l > 0 || lay.emb) ? w.G0 : a.gout;
        // the join of a layer's aux-stream weight gradients is deferred into the
        // next layer's backward unless that layer recomputes its internals first
        // (the recompute forward writes w.ln / w.g, which they read) or this is
        // the chunk's last layer
        const bool defer = l > 0 && l - 1 >= SL.ckpt_layers;
        TRY(layer_backward(D, layer_w(D, P, l), lp, dy, dx, w, st, prev_deferred, defer));
        prev_deferred = defer;
        dy = w.G0;
    }
    if (head_on_aux && n == 0) {   // no layer backward joined the side stream
        SideStream* hs = side_stream(st);
        if (!hs) return -3;
        TRY(stream_dep(hs->aux, st, hs->ev[4]));
    }
    if (lay.emb)
        {
            ProfScope _ps(3, 0.0, st);
            TRY(embed_bwd(D.dtype, a.tokens, w.G0, P.grad + lay.wte, P.grad + lay.wpe, w.emb_ws, M, D.s,
                      h, st));
        }
    return 0;
}

}  // namespace tpipe
