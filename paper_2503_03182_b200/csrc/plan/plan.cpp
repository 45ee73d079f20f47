// tpipe_plan: schedule generator (SURVEY §8(a) a1, §8(b) boundary).
//
// Turns (model, p, m, HBM budget) into per-stage instruction streams:
//   1. compute order per stage —
//        T-Pipe  (App. A): closed-form slot table
//                 (R1) sorted per stage, executed ASAP;
//        T-Recomp (App. B/C P:641-670): R(s,1,i) immediately before
//                 B(s,1,i), chunk-1 forwards advanced k rounds with k
//                 from the App. B constraint as printed (R3);
//        1F1B and 1F1B + full layer-grouped recompute;
//   2. SEND/RECV on FIFO channels per (kind, src, dst) with a send window W
//      (SEND_WAIT placement);
//   3. T-Offload: GRAD_D2H + HOST_OPT after the deep chunk's last
//      backward, W_H2D after the first forward, W_WAIT before the first deep
//      forward (windows Eq. 5 P:680 / Eq. 7);
//   4. byte-exact live-set replay at instruction granularity.
//
// Written independently of oracle/stream.py; tests/test_plan_parity.py
// checks the two element by element.
#include "plan/plan.h"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <map>
#include <new>
#include <set>
#include <string>
#include <tuple>

#include "runtime/errors.h"

namespace tpipe {

static int cdiv(int n, int d) {  // ceiling division, n may be negative
    return n >= 0 ? (n + d - 1) / d : -((-n) / d);
}

int delay_rounds_appB(int p) {
    if (p < 3) return 0;
    const int a = cdiv(p - 3, 6);
    const int fwd_interval = 3 + 6 * a - p;
    const int delta = cdiv(p - 1, 2) - a - 1;
    int k = 0;
    while (fwd_interval - delta + 7 * k < 0) ++k;
    return k;
}

uint64_t layer_params(const tpipe_model_desc& d) {
    const uint64_t h = d.hidden, f = d.ffn_hidden;
    return 2 * h + (3 * h * h + 3 * h) + (h * h + h) + 2 * h + (f * h + f) + (h * f + h);
}

uint64_t chunk_params(const tpipe_model_desc& d, int p, int v, const int* layers, int s, int c) {
    uint64_t P = (uint64_t)layers[c - 1] * layer_params(d);
    if (s == 0 && c == 1) P += (uint64_t)d.vocab * d.hidden + (uint64_t)d.seq_len * d.hidden;
    if (s == p - 1 && c == v) P += 2ull * d.hidden + (uint64_t)d.vocab * d.hidden;
    return P;
}

uint64_t zero1_shard(uint64_t P, int dp) {
    const uint64_t s = (P + dp - 1) / dp;
    return (s + 63) / 64 * 64;
}

// per-layer stash: x_in, ln1 stats, qkv, attn out, lse, x_mid, ln2 stats, u (fc1 pre-act)
static uint64_t layer_stash_bytes(const tpipe_model_desc& d) {
    const uint64_t M = (uint64_t)d.micro_batch * d.seq_len, h = d.hidden, a = d.n_heads,
                   f = d.ffn_hidden, es = d.dtype == TPIPE_BF16 ? 2 : 4;
    return M * h * es + 8 * M + 3 * M * h * es + M * h * es + 4 * a * M + M * h * es + 8 * M + M * f * es;
}

// full_recomp: 1F1B + layer-grouped recompute of the ckpt (<= n, 0 = all)
// shallowest layers of the chunk (DESIGN R33)
static ChunkSizes chunk_sizes(const tpipe_model_desc& d, int p, int v, const int* layers, int s,
                              int c, bool full_recomp, int ckpt = 0) {
    const uint64_t M = (uint64_t)d.micro_batch * d.seq_len, h = d.hidden, a = d.n_heads,
                   f = d.ffn_hidden, V = d.vocab, es = d.dtype == TPIPE_BF16 ? 2 : 4;
    const uint64_t n = layers[c - 1];
    const bool emb = (s == 0 && c == 1), head = (s == p - 1 && c == v);
    ChunkSizes z;
    z.act = M * h * es;
    z.input_is_act = !emb;
    z.has_output = !head;
    const uint64_t LS = layer_stash_bytes(d);
    const uint64_t head_stash = M * h * es + 8 * M + 4 * M;   // x_f, ln_f stats, CE lse
    const uint64_t ck = full_recomp ? (ckpt > 0 && (uint64_t)ckpt < n ? (uint64_t)ckpt : n) : 0;
    uint64_t stash = ck * M * h * es + (n - ck) * LS;
    if (!emb) stash -= z.act;
    if (head) stash += head_stash;
    z.stash = stash;
    const uint64_t nb = (M + 15) / 16;   // 16-row reduction blocks
    uint64_t ws_f = M * (h + f) * es;
    if (full_recomp) ws_f += LS - M * h * es;  // one layer's transient internals
    if (head) ws_f += M * h * es;   // LN_f output only: logits / CE run in the head backward
    uint64_t ws_b = M * (2 * f + 8 * h) * es + 4 * a * M + 4 * nb * std::max(f + 3 * h, 6 * h);
    if (full_recomp) ws_b += LS - M * h * es;
    // head: LN_f out / grad; bf16: dlogits + the fused head's LSE partials
    // (8 B per 64-column group), target logit and row loss (K8, R30); fp32:
    // fp32 logits + dlogits
    if (head) ws_b += 2 * M * h * es + M * V * es +
                      (d.dtype == TPIPE_BF16 ? 8 * M * ((V + 63) / 64) + 8 * M : 4 * M * V);
    if (emb) ws_b += 8 * M;
    z.ws_f = ws_f;
    z.ws_b = ws_b;
    return z;
}

// ---------------------------------------------------------------- compute orders
using COp = std::array<int, 3>;  // {kind, chunk, mb}; kind: 0 F, 1 B, 2 R
enum { KF = 0, KB = 1, KR = 2 };

// T-Pipe slot order (D-1; v > 2: D-11's generalisation with period 3v,
// DESIGN R32): F(s,1,i) = 3v(i-1) + s; F(0,c+1,i) = first t >= F(0,c,i) + p
// with t = 3c mod 3v; B(0,v,i) = F(0,v,i) + 3p - 2; B(0,c-1,i) = first
// t >= B(0,c,i) + 2p with t = B(0,c,i) + 3 mod 3v; F(s,c,i) = F(0,c,i) + s,
// B(s,c,i) = B(0,c,i) - 2s. At v = 2 this is the App. A table
// (a = ceil((p-3)/6), b = ceil((2p-3)/6)).
static std::vector<std::vector<COp>> tpipe_order(int p, int m, bool recomp, int k, int v = 2) {
    const long per = 3L * v;
    auto first_at_least = [&](long lo, long residue) { return lo + (((residue - lo) % per) + per) % per; };
    std::vector<std::vector<COp>> out(p);
    for (int s = 0; s < p; ++s) {
        std::vector<std::pair<long, COp>> slots;
        for (int i = 1; i <= m; ++i) {
            long f0[5], b0[5];
            f0[1] = per * (i - 1);
            for (int c = 1; c < v; ++c) f0[c + 1] = first_at_least(f0[c] + p, 3L * c);
            b0[v] = f0[v] + 3L * p - 2;
            for (int c = v; c > 1; --c) b0[c - 1] = first_at_least(b0[c] + 2L * p, b0[c] + 3);
            for (int c = 1; c <= v; ++c) {
                slots.push_back({f0[c] + s, {KF, c, i}});
                slots.push_back({b0[c] - 2L * s, {KB, c, i}});
            }
        }
        std::sort(slots.begin(), slots.end(),
                  [](const auto& x, const auto& y) { return x.first < y.first; });
        std::vector<COp> lst;
        for (auto& x : slots) lst.push_back(x.second);
        if (recomp && k > 0) {
            std::vector<COp> rel;
            for (int i = 1; i <= std::min(k, m); ++i) rel.push_back({KF, 1, i});
            int n = 0;
            for (auto& op : lst) {
                if (op[0] == KF && op[1] == 1) {
                    ++n;
                    if (n + k <= m) rel.push_back({KF, 1, n + k});
                } else {
                    rel.push_back(op);
                }
            }
            lst.swap(rel);
        }
        if (recomp) {
            std::vector<COp> withr;
            for (auto& op : lst) {
                if (op[0] == KB && op[1] == 1) withr.push_back({KR, 1, op[2]});
                withr.push_back(op);
            }
            lst.swap(withr);
        }
        out[s] = lst;
    }
    return out;
}

// Interleave-1F1B (Megatron virtual pipeline) for v = 2, m % p == 0:
// virtual forward q (0 .. 2m-1) runs chunk (q mod 2p)/p + 1 of micro-batch
// (q / 2p) p + q mod p + 1; virtual backward q runs the mirrored chunk
// 2 - (q mod 2p)/p of the same micro-batch. Stage s warms up with
// min(2(p-s-1) + p, 2m) forwards, then alternates one forward / one backward,
// then drains. recomp: R(s,1,i) right before each B(s,1,i) (R26).
static std::vector<std::vector<COp>> interleave_order(int p, int m, bool recomp, int v = 2) {
    const int total = v * m;
    auto fwd = [&](int q) -> COp { return {KF, (q % (v * p)) / p + 1, (q / (v * p)) * p + q % p + 1}; };
    auto bwd = [&](int q) -> COp { return {KB, v - (q % (v * p)) / p, (q / (v * p)) * p + q % p + 1}; };
    std::vector<std::vector<COp>> out(p);
    for (int s = 0; s < p; ++s) {
        const int w = std::min(2 * (p - s - 1) + (v - 1) * p, total);
        std::vector<COp> lst;
        auto push_b = [&](int q) {
            const COp b = bwd(q);
            if (recomp && b[1] == 1) lst.push_back({KR, 1, b[2]});
            lst.push_back(b);
        };
        for (int q = 0; q < w; ++q) lst.push_back(fwd(q));
        for (int q = 0; q < total - w; ++q) {
            lst.push_back(fwd(w + q));
            push_b(q);
        }
        for (int q = total - w; q < total; ++q) push_b(q);
        out[s] = lst;
    }
    return out;
}

static std::vector<std::vector<COp>> onef1b_order(int p, int m) {
    std::vector<std::vector<COp>> out(p);
    for (int s = 0; s < p; ++s) {
        const int w = std::min(p - s - 1, m);
        auto& lst = out[s];
        for (int i = 1; i <= w; ++i) lst.push_back({KF, 1, i});
        for (int i = 1; i <= m - w; ++i) {
            lst.push_back({KF, 1, w + i});
            lst.push_back({KB, 1, i});
        }
        for (int i = m - w + 1; i <= m; ++i) lst.push_back({KB, 1, i});
    }
    return out;
}

// destination of a compute op's output message; returns false if none / local
struct Msg {
    int kind, src, dst;  // kind 0 = act, 1 = grad
};
static bool message_of(int s, const COp& op, int p, int v, Msg* out) {
    const int kind = op[0], c = op[1];
    int dst;
    if (kind == KF) {
        if (s < p - 1) dst = s + 1;
        else if (c < v) dst = 0;
        else return false;
        *out = {0, s, dst};
    } else if (kind == KB) {
        if (s > 0) dst = s - 1;
        else if (c > 1) dst = p - 1;
        else return false;
        *out = {1, s, dst};
    } else {
        return false;
    }
    return dst != s;
}

// stage producing the input (F) / output grad (B) of (s, c); -1 if none
static int src_stage(int s, int c, int p, int v, int kind) {
    if (kind == KF) {
        if (s > 0) return s - 1;
        if (c > 1) return p - 1;
        return -1;
    }
    if (s < p - 1) return s + 1;
    if (c < v) return 0;
    return -1;
}

// ---------------------------------------------------------------- plan builder
struct Builder {
    tpipe_plan* P;
    int s;
    std::vector<tpipe_op>& ops;
    std::vector<tpipe_buf>& bufs;
    std::vector<int32_t>& ev;
    std::map<std::tuple<int, int, int, int>, int> live;  // (role, chunk, mb, extra) -> buf id

    Builder(tpipe_plan* P_, int s_)
        : P(P_), s(s_), ops(P_->ops[s_]), bufs(P_->bufs[s_]), ev(P_->events[s_]) {}

    int newbuf(int role, int cat, int chunk, int mb, uint64_t bytes, int extra = 0) {
        bufs.push_back({role, cat, chunk, mb, bytes});
        const int id = (int)bufs.size() - 1;
        live[{role, chunk, mb, extra}] = id;
        return id;
    }
    int take(int role, int chunk, int mb, int extra = 0) {
        auto it = live.find({role, chunk, mb, extra});
        if (it == live.end()) return -1;
        int id = it->second;
        live.erase(it);
        return id;
    }
    struct Pending {
        std::vector<int> allocs, frees;
    };
    void emit(int kind, int chunk, int mb, int peer, int channel, int msg, const Pending& pe) {
        tpipe_op op{};
        op.kind = kind;
        op.chunk = chunk;
        op.mb = mb;
        op.peer = peer;
        op.channel = channel;
        op.msg = msg;
        op.alloc_first = (int)ev.size();
        op.n_alloc = (int)pe.allocs.size();
        for (int id : pe.allocs) ev.push_back(id);
        op.free_first = (int)ev.size();
        op.n_free = (int)pe.frees.size();
        for (int id : pe.frees) ev.push_back(id);
        ops.push_back(op);
    }
};

static int build(tpipe_plan* P, bool trecomp, bool full_recomp) {
    const tpipe_model_desc& d = P->model;
    const int p = P->p, m = P->m, v = P->v;
    P->ops.assign(p, {});
    P->bufs.assign(p, {});
    P->events.assign(p, {});
    P->peak.assign(p, {});
    P->chunk_params.assign(p, std::array<uint64_t, 4>{});

    // channel table sorted by (kind, src, dst)
    std::map<std::tuple<int, int, int>, int> chan_id;
    for (int s = 0; s < p; ++s)
        for (auto& op : P->order[s]) {
            Msg mg;
            if (message_of(s, op, p, v, &mg)) chan_id[{mg.kind, mg.src, mg.dst}] = 0;
        }
    P->channels.clear();
    for (auto& kv : chan_id) {
        kv.second = (int)P->channels.size();
        P->channels.push_back({std::get<0>(kv.first), std::get<1>(kv.first), std::get<2>(kv.first)});
    }

    const bool off = (P->offload & TPIPE_OFFLOAD_MODEL_STATE) != 0;
    const bool sopt = off && (P->offload & TPIPE_OFFLOAD_DEVICE_OPT) != 0;
    const bool aoff_on = (P->offload & TPIPE_OFFLOAD_ACTIVATIONS) != 0 && v == 2 && !trecomp;
    const uint64_t es = d.dtype == TPIPE_BF16 ? 2 : 4;
    const uint64_t M = (uint64_t)d.micro_batch * d.seq_len;
    P->params_total = 0;

    for (int s = 0; s < p; ++s) {
        Builder B(P, s);
        // static buffers: model state per chunk, io
        for (int c = 1; c <= v; ++c) {
            const uint64_t np = chunk_params(d, p, v, P->sl[s].data(), s, c);
            P->chunk_params[s][c - 1] = np;
            P->params_total += np;
            const bool o = off && c >= 2;   // T-Offload of chunks 2..v (R32)
            const uint64_t opt_b = (d.dtype == TPIPE_BF16 ? 4 : 0) + 8;   // master (bf16 mode) + m, v
            // ZeRO-1 (R31): master / m / v cover one shard of the chunk
            const uint64_t ms = o ? np * (es + 4)
                                  : np * (es + 4) + (P->dp > 1 ? zero1_shard(np, P->dp) : np) * opt_b;
            // streamed device AdamW (R24): + double-buffered master/m/v slice staging
            const uint64_t stg = (o && sopt) ? 2ull * 12ull * std::min<uint64_t>(np, TPIPE_SOPT_SLICE_PARAMS) : 0;
            B.bufs.push_back({TPIPE_BUF_STATIC, TPIPE_CAT_MODEL_STATE, c, 0, ms + stg});
        }
        if (s == 0) B.bufs.push_back({TPIPE_BUF_STATIC, TPIPE_CAT_IO, 0, 0, 4ull * m * M});
        if (s == p - 1) B.bufs.push_back({TPIPE_BUF_STATIC, TPIPE_CAT_IO, 0, 1, 4ull * m * M + 4ull * m});

        ChunkSizes z[5];
        for (int c = 1; c <= v; ++c) z[c] = chunk_sizes(d, p, v, P->sl[s].data(), s, c, full_recomp, P->rl_of(s));
        // partial T-Recomp (R25): layers 1..r of chunk 1 are regenerated by R (TSTASH during
        // F, RBUF from R to B); the stash of layers r+1..n1 is kept from F to B (STASH).
        // The two parts add up to the full chunk-1 stash.
        uint64_t keep1 = 0, rec1 = z[1].stash;
        if (trecomp && P->rl_of(s) < P->sl[s][0]) {
            keep1 = (uint64_t)(P->sl[s][0] - P->rl_of(s)) * layer_stash_bytes(d);
            rec1 = z[1].stash - keep1;
        }

        const auto& order = P->order[s];
        std::map<int, int> sent, waited;  // channel -> count
        int last_b[5] = {0, 0, 0, 0, 0}, first_f[5] = {1 << 30, 1 << 30, 1 << 30, 1 << 30, 1 << 30};
        for (auto& op : order) {
            if (op[0] == KB) last_b[op[1]] = std::max(last_b[op[1]], op[2]);
            if (op[0] == KF) first_f[op[1]] = std::min(first_f[op[1]], op[2]);
        }
        bool first_f_done = false;
        // activation offload of chunk-1 stash blocks (R23): blocks whose
        // F(1,i) -> B(1,i) distance exceeds 2d compute ops go to pinned host
        std::set<int> aoff;
        std::map<int, std::vector<int>> arel, afet;
        const int dd = P->act_distance;
        if (aoff_on) {
            for (size_t n = 0; n < order.size(); ++n) {
                if (order[n][0] != KF || order[n][1] != 1) continue;
                const int mb = order[n][2];
                size_t nb = n;
                while (nb < order.size() && !(order[nb][0] == KB && order[nb][1] == 1 && order[nb][2] == mb)) ++nb;
                if ((long)nb - (long)n > 2L * dd) {
                    aoff.insert(mb);
                    arel[(int)n + dd].push_back(mb);
                    afet[(int)nb - dd].push_back(mb);
                }
            }
            for (auto& kv : arel) std::sort(kv.second.begin(), kv.second.end());
            for (auto& kv : afet) std::sort(kv.second.begin(), kv.second.end());
        }
        for (size_t n_op = 0; n_op < order.size(); ++n_op) {
            const auto& op = order[n_op];
            const int kind = op[0], c = op[1], i = op[2];
            const ChunkSizes& zz = z[c];
            Msg mg;
            const bool has_msg = message_of(s, op, p, v, &mg);
            const int ch = has_msg ? chan_id[{mg.kind, mg.src, mg.dst}] : -1;
            // 0. activation offload: release copied blocks, start prefetches
            if (arel.count((int)n_op))
                for (int mb : arel[(int)n_op]) {
                    Builder::Pending pe;
                    pe.frees.push_back(B.take(TPIPE_BUF_STASH, 1, mb));
                    B.emit(TPIPE_OP_ACT_D2H_WAIT, 1, mb, -1, -1, -1, pe);
                }
            if (afet.count((int)n_op))
                for (int mb : afet[(int)n_op]) {
                    Builder::Pending pe;
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_STASH, TPIPE_CAT_ACT, 1, mb, z[1].stash));
                    B.emit(TPIPE_OP_ACT_H2D, 1, mb, -1, -1, -1, pe);
                }
            // 1. send-window waits
            if (has_msg) {
                const int j = sent[ch];
                while (waited[ch] <= j - P->W) {
                    const int jj = waited[ch];
                    Builder::Pending pe;
                    pe.frees.push_back(B.take(TPIPE_BUF_MSG, ch, jj));
                    B.emit(TPIPE_OP_SEND_WAIT, 0, 0, mg.dst, ch, jj, pe);
                    waited[ch] += 1;
                }
            }
            // 2. weight-upload wait and receives
            if (off && kind == KF && c >= 2 && i == first_f[c]) B.emit(TPIPE_OP_W_WAIT, c, 0, -1, -1, -1, {});
            if (P->dp > 1 && kind == KF && i == first_f[c]) B.emit(TPIPE_OP_DP_WAIT, c, 0, -1, -1, -1, {});
            if (kind == KF && zz.input_is_act) {
                const int src = src_stage(s, c, p, v, KF);
                if (src >= 0 && src != s) {
                    Builder::Pending pe;
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_IN, TPIPE_CAT_ACT, c, i, zz.act));
                    B.emit(TPIPE_OP_RECV_ACT, c, i, src, chan_id[{0, src, s}], -1, pe);
                }
            }
            if (kind == KB && zz.has_output) {
                const int src = src_stage(s, c, p, v, KB);
                if (src >= 0 && src != s) {
                    Builder::Pending pe;
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_GIN, TPIPE_CAT_COMM, c, i, zz.act));
                    B.emit(TPIPE_OP_RECV_GRAD, c, i, src, chan_id[{1, src, s}], -1, pe);
                }
            }
            if (kind == KB && c == 1 && aoff.count(i)) B.emit(TPIPE_OP_ACT_H2D_WAIT, 1, i, -1, -1, -1, {});
            // 3. the compute op
            Builder::Pending pe;
            if (kind == KF) {
                if (trecomp && c == 1) {
                    int id = B.newbuf(TPIPE_BUF_TSTASH, TPIPE_CAT_ACT, c, i, rec1);
                    pe.allocs.push_back(id);
                    pe.frees.push_back(B.take(TPIPE_BUF_TSTASH, c, i));
                    if (keep1) pe.allocs.push_back(B.newbuf(TPIPE_BUF_STASH, TPIPE_CAT_ACT, c, i, keep1));
                } else {
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_STASH, TPIPE_CAT_ACT, c, i, zz.stash));
                }
                if (has_msg) {
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_MSG, TPIPE_CAT_COMM, ch, sent[ch], zz.act));
                } else if (zz.has_output) {
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_IN, TPIPE_CAT_ACT, c + 1, i, zz.act));
                }
                int ws = B.newbuf(TPIPE_BUF_WS, TPIPE_CAT_WORKSPACE, c, i, zz.ws_f, 1);
                pe.allocs.push_back(ws);
                pe.frees.push_back(B.take(TPIPE_BUF_WS, c, i, 1));
            } else if (kind == KR) {
                pe.allocs.push_back(B.newbuf(TPIPE_BUF_RBUF, TPIPE_CAT_RECOMP_BUF, c, i, rec1));
                pe.allocs.push_back(B.newbuf(TPIPE_BUF_WS, TPIPE_CAT_WORKSPACE, c, i, zz.ws_f, 2));
                pe.frees.push_back(B.take(TPIPE_BUF_WS, c, i, 2));
            } else {
                if (has_msg) {
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_MSG, TPIPE_CAT_COMM, ch, sent[ch], zz.act));
                } else if (!(s == 0 && c == 1)) {
                    pe.allocs.push_back(B.newbuf(TPIPE_BUF_GIN, TPIPE_CAT_COMM, c - 1, i, zz.act));
                }
                pe.allocs.push_back(B.newbuf(TPIPE_BUF_WS, TPIPE_CAT_WORKSPACE, c, i, zz.ws_b, 3));
                pe.frees.push_back(B.take(TPIPE_BUF_WS, c, i, 3));
                if (trecomp && c == 1) {
                    pe.frees.push_back(B.take(TPIPE_BUF_RBUF, c, i));
                    if (keep1) pe.frees.push_back(B.take(TPIPE_BUF_STASH, c, i));
                } else {
                    pe.frees.push_back(B.take(TPIPE_BUF_STASH, c, i));
                }
                if (zz.input_is_act) pe.frees.push_back(B.take(TPIPE_BUF_IN, c, i));
                if (zz.has_output) pe.frees.push_back(B.take(TPIPE_BUF_GIN, c, i));
            }
            for (int id : pe.frees)
                if (id < 0) return set_error(TPIPE_E_CONFLICT, "stage %d: free of a buffer never allocated", s);
            B.emit(kind == KF ? TPIPE_OP_F : kind == KB ? TPIPE_OP_B : TPIPE_OP_R, c, i, -1, -1, -1, pe);
            // 4. send
            if (has_msg) {
                B.emit(kind == KF ? TPIPE_OP_SEND_ACT : TPIPE_OP_SEND_GRAD, c, i, mg.dst, ch, sent[ch], {});
                sent[ch] += 1;
            }
            if (kind == KF && c == 1 && aoff.count(i)) B.emit(TPIPE_OP_ACT_D2H, 1, i, -1, -1, -1, {});
            // 5. optimizer after the chunk's last backward
            if (kind == KB && i == last_b[c]) {
                if (off && c >= 2 && sopt) {
                    B.emit(TPIPE_OP_STREAM_OPT, c, 0, -1, -1, -1, {});
                } else if (off && c >= 2) {
                    B.emit(TPIPE_OP_GRAD_D2H, c, 0, -1, -1, -1, {});
                    B.emit(TPIPE_OP_HOST_OPT, c, 0, -1, -1, -1, {});
                } else {
                    B.emit(P->dp > 1 ? TPIPE_OP_DP_OPT : TPIPE_OP_OPT, c, 0, -1, -1, -1, {});
                }
            }
            // 6. weight upload after the first forward
            if (off && !sopt && !first_f_done && kind == KF)
                for (int cc = 2; cc <= v; ++cc) B.emit(TPIPE_OP_W_H2D, cc, 0, -1, -1, -1, {});
            first_f_done = first_f_done || kind == KF;
        }
        // flush outstanding sends, channels in id order (= sorted (kind, src, dst))
        for (auto& kv : sent) {
            const int ch = kv.first;
            while (waited[ch] < kv.second) {
                const int jj = waited[ch];
                Builder::Pending pe;
                pe.frees.push_back(B.take(TPIPE_BUF_MSG, ch, jj));
                B.emit(TPIPE_OP_SEND_WAIT, 0, 0, P->channels[ch][2], ch, jj, pe);
                waited[ch] += 1;
            }
        }
        if (!B.live.empty()) return set_error(TPIPE_E_CONFLICT, "stage %d: %zu buffers leak", s, B.live.size());

        // live-byte replay
        tpipe_mem_report r{};
        uint64_t cur = 0, cat_live[TPIPE_CAT_COUNT] = {};
        for (auto& b : B.bufs)
            if (b.role == TPIPE_BUF_STATIC) {
                cur += b.bytes;
                cat_live[b.category] += b.bytes;
                r.peak[b.category] = std::max(r.peak[b.category], cat_live[b.category]);
            }
        r.static_bytes = cur;
        uint64_t peak = cur;
        for (auto& op : B.ops) {
            for (int e = 0; e < op.n_alloc; ++e) {
                const tpipe_buf& b = B.bufs[B.ev[op.alloc_first + e]];
                cur += b.bytes;
                cat_live[b.category] += b.bytes;
                r.peak[b.category] = std::max(r.peak[b.category], cat_live[b.category]);
            }
            peak = std::max(peak, cur);
            for (int e = 0; e < op.n_free; ++e) {
                const tpipe_buf& b = B.bufs[B.ev[op.free_first + e]];
                cur -= b.bytes;
                cat_live[b.category] -= b.bytes;
            }
        }
        r.total_peak = peak;
        P->peak[s] = r;
    }
    (void)M;
    return 0;
}

// static deadlock check: program order + SEND(j)->RECV(j) + RECV(j)->SEND_WAIT(j)
static bool deadlock_free(const tpipe_plan* P) {
    const int p = P->p;
    std::vector<int> base(p + 1, 0);
    for (int s = 0; s < p; ++s) base[s + 1] = base[s] + (int)P->ops[s].size();
    const int N = base[p];
    std::vector<std::vector<int>> succ(N);
    std::vector<int> indeg(N, 0);
    auto edge = [&](int a, int b) {
        succ[a].push_back(b);
        indeg[b]++;
    };
    std::map<std::pair<int, int>, int> sends, recvs, waits;
    std::map<int, int> rcount;
    for (int s = 0; s < p; ++s)
        for (int n = 0; n < (int)P->ops[s].size(); ++n) {
            const tpipe_op& op = P->ops[s][n];
            const int id = base[s] + n;
            if (n) edge(id - 1, id);
            if (op.kind == TPIPE_OP_SEND_ACT || op.kind == TPIPE_OP_SEND_GRAD) sends[{op.channel, op.msg}] = id;
            if (op.kind == TPIPE_OP_RECV_ACT || op.kind == TPIPE_OP_RECV_GRAD) recvs[{op.channel, rcount[op.channel]++}] = id;
            if (op.kind == TPIPE_OP_SEND_WAIT) waits[{op.channel, op.msg}] = id;
        }
    for (auto& kv : sends) {
        auto it = recvs.find(kv.first);
        if (it == recvs.end()) return false;
        edge(kv.second, it->second);
    }
    for (auto& kv : waits) {
        auto it = recvs.find(kv.first);
        if (it == recvs.end()) return false;
        edge(it->second, kv.second);
    }
    std::vector<int> q;
    for (int i = 0; i < N; ++i)
        if (!indeg[i]) q.push_back(i);
    int seen = 0;
    while (!q.empty()) {
        int x = q.back();
        q.pop_back();
        ++seen;
        for (int y : succ[x])
            if (--indeg[y] == 0) q.push_back(y);
    }
    return seen == N;
}

static int validate(const tpipe_model_desc* d, int p, int m) {
    if (!d) return set_error(TPIPE_E_INVALID, "model is NULL");
    if (p < 1 || p > 64) return set_error(TPIPE_E_INVALID, "n_stages must be in [1, 64]");
    if (m < 1) return set_error(TPIPE_E_INVALID, "n_microbatches must be >= 1");
    if (d->dtype != TPIPE_FP32 && d->dtype != TPIPE_BF16) return set_error(TPIPE_E_INVALID, "dtype");
    if (d->n_layers < 1) return set_error(TPIPE_E_INVALID, "n_layers must be a positive multiple of n_stages");
    if (d->hidden < 64 || d->hidden % 64) return set_error(TPIPE_E_INVALID, "hidden must be a multiple of 64");
    if (d->ffn_hidden < 64 || d->ffn_hidden % 64) return set_error(TPIPE_E_INVALID, "ffn_hidden must be a multiple of 64");
    if (d->vocab < 64 || d->vocab % 64 || d->vocab >= (1 << 17)) return set_error(TPIPE_E_INVALID, "vocab must be a multiple of 64 below 131072");
    if (d->n_heads < 1 || d->hidden % d->n_heads) return set_error(TPIPE_E_INVALID, "n_heads must divide hidden");
    const int hd = d->hidden / d->n_heads;
    if (hd > 128 || hd % 8) return set_error(TPIPE_E_INVALID, "head_dim must be a multiple of 8, <= 128");
    if (d->seq_len < 1 || d->micro_batch < 1) return set_error(TPIPE_E_INVALID, "seq_len / micro_batch");
    if ((long)d->seq_len * d->micro_batch > 32768) return set_error(TPIPE_E_INVALID, "micro_batch*seq_len must be <= 32768");
    return 0;
}

}  // namespace tpipe

using namespace tpipe;

#define TP_API extern "C" __attribute__((visibility("default")))

// ASAP replay of the compute order with per-op durations dur(s, j) (j = index
// of the op in stage s's compute order); returns makespan and busy per stage
template <typename T, typename DurFn>
static int replay_order(const tpipe_plan* P, DurFn dur, T* makespan, T* busy_out,
                        std::vector<std::vector<std::array<T, 2>>>* times = nullptr) {
    const int p = P->p, v = P->v;
    const bool rec = P->strategy == TPIPE_S_TPIPE_TRECOMP || P->strategy == TPIPE_S_INTERLEAVE_TRECOMP;
    std::map<std::tuple<int, int, int, int>, T> endt;  // (stage, kind, chunk, mb)
    std::vector<size_t> pos(p, 0);
    std::vector<T> freet(p, 0), busy(p, 0);
    size_t total = 0, done = 0;
    for (auto& o : P->order) total += o.size();
    if (times) {
        times->assign(p, {});
        for (int s = 0; s < p; ++s) (*times)[s].resize(P->order[s].size());
    }
    while (done < total) {
        bool prog = false;
        for (int s = 0; s < p; ++s) {
            while (pos[s] < P->order[s].size()) {
                const COp& op = P->order[s][pos[s]];
                const int kind = op[0], c = op[1], i = op[2];
                std::vector<std::tuple<int, int, int, int>> deps;
                if (kind == KF) {
                    if (s > 0) deps.push_back({s - 1, KF, c, i});
                    else if (c > 1) deps.push_back({p - 1, KF, c - 1, i});
                } else if (kind == KR) {
                    deps.push_back({s, KF, c, i});
                } else {
                    deps.push_back({s, KF, c, i});
                    if (rec && c == 1) deps.push_back({s, KR, c, i});
                    if (s < p - 1) deps.push_back({s + 1, KB, c, i});
                    else if (c < v) deps.push_back({0, KB, c + 1, i});
                }
                T t0 = freet[s];
                bool ready = true;
                for (auto& dd : deps) {
                    auto it = endt.find(dd);
                    if (it == endt.end()) { ready = false; break; }
                    t0 = std::max(t0, it->second);
                }
                if (!ready) break;
                const T t1 = t0 + dur(s, (int)pos[s], kind);
                endt[{s, kind, c, i}] = t1;
                if (times) (*times)[s][pos[s]] = {t0, t1};
                freet[s] = t1;
                busy[s] += t1 - t0;
                ++pos[s];
                ++done;
                prog = true;
            }
        }
        if (!prog) return set_error(TPIPE_E_DEADLOCK, "compute order deadlocks");
    }
    *makespan = 0;
    for (int s = 0; s < p; ++s) *makespan = std::max(*makespan, freet[s]);
    for (int s = 0; s < 64; ++s) busy_out[s] = s < p ? busy[s] : 0;
    return 0;
}

// ---------------------------------------------------------------- cost model (DESIGN R28)
struct CostModel {
    double bw = 50e9, host = 3e9, flops = 1e15;
};

static double layer_fwd_s(const tpipe_model_desc& d, const CostModel& cm) {
    const double M = (double)d.micro_batch * d.seq_len, h = d.hidden, f = d.ffn_hidden;
    const double hd = (double)d.hidden / d.n_heads, s = d.seq_len;
    const double fl = 2.0 * M * (4.0 * h * h + 2.0 * h * f) +
                      4.0 * d.micro_batch * d.n_heads * (s * (s + 1) / 2.0) * hd;
    return fl / cm.flops;
}

static double head_fwd_s(const tpipe_model_desc& d, const CostModel& cm) {
    return 2.0 * d.micro_batch * d.seq_len * (double)d.vocab * d.hidden / cm.flops;
}

// F = the chunk's layers (+ the LM head on the last stage's last chunk),
// B = 2F (+ the layers' forward again under 1F1B + full recompute), R = the
// recomputed layers (P:611 unit model with T_bwd = 2 T_fwd, scaled by FLOPs)
static double op_seconds(const tpipe_plan* P, int s, int kind, int c, double tl, double th) {
    if (kind == KR) return P->rl_of(s) * tl;
    const double f = P->sl[s][c - 1] * tl + ((s == P->p - 1 && c == P->v) ? th : 0.0);
    if (kind == KB) return 2.0 * f + (P->strategy == TPIPE_S_1F1B_FULL_RECOMP ? P->rl_of(s) * tl : 0.0);
    return f;
}

// Modeled step time: ASAP replay of the order with op_seconds, plus per stage
// the offload transfer time that does not fit its window:
//  * model-state T-Offload of chunk v: the window runs from the stage's last
//    B(s, v, .) to the end of the step and on to the next step's first
//    F(s, v, .) (P:680 / P:694: the cool-down and warm-up bubbles); host AdamW
//    needs grads down (4 B/param) + the host update + bf16 weights up, the
//    streamed device AdamW 12 B/param each way (both directions in parallel);
//  * activation offload: n_off blocks each way against the stage's busy time.
static double estimate(const tpipe_plan* P, const CostModel& cm, double* exposed_out) {
    const tpipe_model_desc& d = P->model;
    const double tl = layer_fwd_s(d, cm), th = head_fwd_s(d, cm);
    std::vector<std::vector<std::array<double, 2>>> times;
    double mk = 0, busy[64];
    auto dur = [&](int s, int j, int kind) { return op_seconds(P, s, kind, P->order[s][j][1], tl, th); };
    if (replay_order<double>(P, dur, &mk, busy, &times)) return 1e30;
    double worst = 0;
    const double es = d.dtype == TPIPE_BF16 ? 2.0 : 4.0;
    for (int s = 0; s < P->p; ++s) {
        double exposed = 0;
        // offloaded chunks 2..v (R32): each chunk's transfer against its own
        // window; the chunks share one link, so the exposures add up
        for (int ch = 2; (P->offload & TPIPE_OFFLOAD_MODEL_STATE) && ch <= P->v; ++ch) {
            const double np = (double)P->chunk_params[s][ch - 1];
            double end_b = 0, start_f = mk;
            for (size_t j = 0; j < P->order[s].size(); ++j) {
                const COp& op = P->order[s][j];
                if (op[1] != ch) continue;
                if (op[0] == KB) end_b = std::max(end_b, times[s][j][1]);
                if (op[0] == KF) start_f = std::min(start_f, times[s][j][0]);
            }
            const double window = (mk - end_b) + start_f;
            const double need = (P->offload & TPIPE_OFFLOAD_DEVICE_OPT)
                                    ? 12.0 * np / cm.bw
                                    : np * 4.0 / cm.bw + np / cm.host + np * es / cm.bw;
            exposed += std::max(0.0, need - window);
        }
        if (P->offload & TPIPE_OFFLOAD_ACTIVATIONS) {
            int n_off = 0;
            uint64_t bytes = 0;
            for (const tpipe_op& op : P->ops[s])
                if (op.kind == TPIPE_OP_ACT_H2D) {
                    ++n_off;
                    bytes = P->bufs[s][P->events[s][op.alloc_first]].bytes;
                }
            exposed += std::max(0.0, n_off * (double)bytes / cm.bw - busy[s]);
        }
        worst = std::max(worst, exposed);
    }
    if (exposed_out) *exposed_out = worst;
    return mk + worst;
}

static int make_plan(const tpipe_model_desc* model, int p, int m, int strategy, int k, int W,
                     int offload, int act_distance, int recomp_layers, const int32_t* stage_layers,
                     const int32_t* stage_chunk1, const CostModel& cm, tpipe_plan** out, int dp = 1,
                     int chunks = 2) {
    if ((offload & TPIPE_OFFLOAD_DEVICE_OPT) && !(offload & TPIPE_OFFLOAD_MODEL_STATE))
        return set_error(TPIPE_E_INVALID, "offload: DEVICE_OPT needs MODEL_STATE");
    if ((offload & TPIPE_OFFLOAD_ACTIVATIONS) && strategy != TPIPE_S_TPIPE)
        return set_error(TPIPE_E_INCOMPAT, "activation offload applies to T-Pipe without T-Recomp");
    tpipe_plan* P = new (std::nothrow) tpipe_plan();
    if (!P) return set_error(TPIPE_E_INVALID, "out of host memory");
    P->model = *model;
    P->p = p;
    P->m = m;
    P->strategy = strategy;
    P->W = W;
    P->offload = offload;
    P->act_distance = act_distance > 0 ? act_distance : 1;   // derived below when 0 (Q12)
    P->dp = dp;
    if (dp > 1 && (offload & TPIPE_OFFLOAD_MODEL_STATE)) {
        delete P;
        return set_error(TPIPE_E_INCOMPAT, "dp > 1 shards the device optimizer (ZeRO-1): no model-state offload");
    }
    const bool is_il = strategy == TPIPE_S_INTERLEAVE || strategy == TPIPE_S_INTERLEAVE_TRECOMP;
    const bool is_tp = strategy == TPIPE_S_TPIPE || strategy == TPIPE_S_TPIPE_TRECOMP || is_il;
    if (is_il && m % p) {
        delete P;
        return set_error(TPIPE_E_INCOMPAT, "interleave-1F1B needs n_microbatches %% n_stages == 0");
    }
    P->v = is_tp ? chunks : 1;
    if (!is_tp && chunks != 2) {
        delete P;
        return set_error(TPIPE_E_INCOMPAT, "chunks applies to the T-Pipe and Interleave strategies");
    }
    if (P->v > 2 && ((stage_chunk1 && stage_chunk1[0]) || model->layers_chunk[0] || model->layers_chunk[1])) {
        delete P;
        return set_error(TPIPE_E_INVALID, "layers_chunk / stage_chunk1 are two-chunk options (chunks = 2)");
    }
    // v chunks: n / v layers each, the extra ones to the shallowest chunks (R14, R32)
    auto split = [&](int ns) {
        std::array<int, 4> x{};
        for (int c = 0; c < P->v; ++c) x[c] = ns / P->v + (c < ns % P->v ? 1 : 0);
        return x;
    };
    const int n = model->n_layers / p;
    const bool part = stage_layers && stage_layers[0] != 0;
    if (part) {   // cost-balanced partition (R27)
        long sum = 0;
        for (int s = 0; s < p; ++s) {
            const int ns = stage_layers[s];
            if (ns < P->v || (model->layers_chunk[0] || model->layers_chunk[1])) {
                const int vv = P->v;
                delete P;
                return set_error(TPIPE_E_INVALID, "stage_layers[%d] = %d: need >= %d layers per stage "
                                 "(and layers_chunk {0,0})", s, ns, vv);
            }
            sum += ns;
            const int c1 = (stage_chunk1 && stage_chunk1[s] > 0) ? stage_chunk1[s] : (ns + 1) / 2;
            if (P->v == 2 && (c1 < 1 || c1 > ns - 1)) {
                delete P;
                return set_error(TPIPE_E_INVALID, "stage_chunk1[%d] = %d: need 1 .. %d", s, c1, ns - 1);
            }
            P->sl.push_back(P->v == 2 ? std::array<int, 4>{c1, ns - c1}
                            : P->v == 1 ? std::array<int, 4>{ns, 0} : split(ns));
        }
        if (sum != model->n_layers) {
            delete P;
            return set_error(TPIPE_E_INVALID, "stage_layers sum %ld != n_layers %d", sum, model->n_layers);
        }
        if (offload & TPIPE_OFFLOAD_MODEL_STATE && P->v < 2) {
            delete P;
            return set_error(TPIPE_E_INCOMPAT, "model-state offload requires T-Pipe (v >= 2)");
        }
        for (int c = 0; c < 4; ++c) P->layers[c] = P->sl[0][c];
    } else if (P->v > 2) {
        if (n < P->v) {
            delete P;
            return set_error(TPIPE_E_INCOMPAT, "%d chunks need >= %d layers per stage", P->v, P->v);
        }
        const auto x = split(n);
        for (int c = 0; c < 4; ++c) P->layers[c] = x[c];
    } else if (P->v == 2) {
        if (model->layers_chunk[0] || model->layers_chunk[1]) {
            if (model->layers_chunk[0] < 1 || model->layers_chunk[1] < 1 ||
                model->layers_chunk[0] + model->layers_chunk[1] != n) {
                delete P;
                return set_error(TPIPE_E_INVALID, "layers_chunk must be >= 1 and sum to n_layers/n_stages");
            }
            P->layers[0] = model->layers_chunk[0];
            P->layers[1] = model->layers_chunk[1];
        } else {
            if (n < 2) {
                delete P;
                return set_error(TPIPE_E_INCOMPAT, "T-Pipe needs >= 2 layers per stage (2 chunks)");
            }
            P->layers[0] = (n + 1) / 2;  // extra layer to the shallow chunk (DESIGN R14)
            P->layers[1] = n / 2;
        }
    } else {
        if (offload) {
            delete P;
            return set_error(TPIPE_E_INCOMPAT, "model-state offload requires T-Pipe (v >= 2)");
        }
        P->layers[0] = n;
    }
    if (!part) P->sl.assign(p, std::array<int, 4>{P->layers[0], P->layers[1], P->layers[2], P->layers[3]});
    int n1max = 0;
    for (auto& x : P->sl) n1max = std::max(n1max, x[0]);
    const bool trecomp = strategy == TPIPE_S_TPIPE_TRECOMP || strategy == TPIPE_S_INTERLEAVE_TRECOMP;
    if (trecomp && recomp_layers > n1max) {
        delete P;
        return set_error(TPIPE_E_INVALID, "recomp_layers %d exceeds the %d chunk-1 layers per stage",
                         recomp_layers, n1max);
    }
    const bool full_rc = strategy == TPIPE_S_1F1B_FULL_RECOMP;
    if (full_rc && recomp_layers > n1max) {
        delete P;
        return set_error(TPIPE_E_INVALID, "recomp_layers %d exceeds the %d layers per stage", recomp_layers, n1max);
    }
    // T-Recomp: chunk-1 layers R regenerates; 1F1B + recompute: layers per stage
    // recomputed layer-wise in B, shallowest first (R33; 0 = all)
    P->rl = (trecomp || full_rc) ? (recomp_layers > 0 ? recomp_layers : n1max) : 0;
    // App. B's delay rounds are derived for two chunks; v > 2 runs undelayed (R32)
    P->k = (trecomp && !is_il) ? (k < 0 ? (P->v == 2 ? delay_rounds_appB(p) : 0) : k) : 0;
    if (is_il) {
        auto ord = interleave_order(p, m, trecomp, P->v);
        P->order.assign(p, {});
        for (int s = 0; s < p; ++s) P->order[s] = ord[s];
    } else if (is_tp) {
        auto ord = tpipe_order(p, m, trecomp, P->k, P->v);
        P->order.assign(p, {});
        for (int s = 0; s < p; ++s) P->order[s] = ord[s];
    } else {
        auto ord = onef1b_order(p, m);
        P->order.assign(p, {});
        for (int s = 0; s < p; ++s) P->order[s] = ord[s];
    }
    if ((offload & TPIPE_OFFLOAD_ACTIVATIONS) && act_distance <= 0) {
        // release / prefetch a block d compute ops after F / before
        // B, with d the smallest count of chunk-1 forward times (the shortest
        // op, cost model) that covers the block's copy at host_link_bps
        double worst = 1.0;
        const double tl = layer_fwd_s(*model, cm);
        for (int s = 0; s < p; ++s) {
            const ChunkSizes z = chunk_sizes(*model, p, P->v, P->sl[s].data(), s, 1, false);
            const double copy = (double)z.stash / cm.bw, t1 = P->sl[s][0] * tl;
            worst = std::max(worst, std::ceil(copy / t1 - 1e-9));
        }
        P->act_distance = (int)std::min(16.0, worst);
    }
    int rc = build(P, trecomp, strategy == TPIPE_S_1F1B_FULL_RECOMP);
    if (rc) {
        delete P;
        return rc;
    }
    P->est_step_s = estimate(P, cm, &P->est_exposed_s);
    if (!deadlock_free(P)) {
        delete P;
        return set_error(TPIPE_E_DEADLOCK, "instruction streams can deadlock (send window %d)", W);
    }
    *out = P;
    return 0;
}

static uint64_t max_peak(const tpipe_plan* P) {
    uint64_t x = 0;
    for (auto& r : P->peak) x = std::max(x, r.total_peak);
    return x;
}

// Cost-balanced partition (DESIGN R27, SURVEY D-12): the last stage also runs
// the LM head, worth `head_layers` layers of forward work; choose its layer
// count n_last >= v minimising the largest stage cost and spread the other
// L - n_last layers evenly (extra layers on the earliest stages).
static std::vector<int> balanced_partition(int L, int p, int v, double head_layers) {
    if (p < 2) return {};
    double best = 1e30;
    int best_last = -1;
    for (int n_last = v; n_last <= L / p; ++n_last) {
        const int rest = L - n_last;
        if (rest < v * (p - 1)) break;
        const int hi = (rest + p - 2) / (p - 1);
        const double cost = std::max((double)hi, n_last + head_layers);
        if (cost < best - 1e-9) {
            best = cost;
            best_last = n_last;
        }
    }
    if (best_last < 0) return {};
    std::vector<int> out;
    const int rest = L - best_last, base = rest / (p - 1), extra = rest % (p - 1);
    for (int s = 0; s < p - 1; ++s) out.push_back(base + (s < extra ? 1 : 0));
    out.push_back(best_last);
    return out;
}

// Modeled makespan of a plan's compute order with per-stage (chunk-1, chunk-2)
// layer counts `sl` (no offload terms): the cost model's ASAP replay.
static double order_makespan(tpipe_plan* S, const std::vector<std::array<int, 4>>& sl, const CostModel& cm) {
    S->sl = sl;
    const double tl = layer_fwd_s(S->model, cm), th = head_fwd_s(S->model, cm);
    double mk = 0, busy[64];
    auto dur = [&](int s, int j, int kind) { return op_seconds(S, s, kind, S->order[s][j][1], tl, th); };
    if (replay_order<double>(S, dur, &mk, busy)) return 1e30;
    return mk;
}

// Duration-aware partition (DESIGN R29): steepest descent over
// per-stage layer counts n(s) and (v = 2) chunk splits n1(s), minimising the
// modeled makespan of the plan's own order (T-Pipe's slot order stays the
// paper's; what adapts to the unequal durations — the LM head on the last
// stage's deep chunk — is how many layers each stage and chunk holds).
// Moves, in this fixed order: one layer from stage i to stage j (both chunks
// re-split ceil/floor), then n1(s) +- 1; the best strictly improving move is
// taken until none improves. Started from the uniform split and from the R27
// closed form; the better end point wins (ties: uniform start).
static double search_partition(const tpipe_plan* U, const CostModel& cm, std::vector<int>* n_out,
                               std::vector<int>* c1_out) {
    tpipe_plan S = *U;   // order, p, v, strategy, model, rl
    const int p = S.p, v = S.v, L = S.model.n_layers;
    auto split = [&](int n) { return v == 2 ? std::array<int, 4>{(n + 1) / 2, n / 2} : std::array<int, 4>{n, 0}; };
    auto descend = [&](std::vector<std::array<int, 4>> sl) {
        double cur = order_makespan(&S, sl, cm);
        for (int it = 0; it < 256; ++it) {
            double best = cur;
            std::vector<std::array<int, 4>> best_sl;
            for (int i = 0; i < p; ++i)
                for (int j = 0; j < p; ++j) {
                    if (i == j) continue;
                    const int ni = sl[i][0] + sl[i][1], nj = sl[j][0] + sl[j][1];
                    if (ni - 1 < v) continue;
                    auto t = sl;
                    t[i] = split(ni - 1);
                    t[j] = split(nj + 1);
                    const double c = order_makespan(&S, t, cm);
                    if (c < best * (1.0 - 1e-12)) {
                        best = c;
                        best_sl = t;
                    }
                }
            if (v == 2)
                for (int s = 0; s < p; ++s)
                    for (int dlt : {1, -1}) {
                        auto t = sl;
                        t[s][0] += dlt;
                        t[s][1] -= dlt;
                        if (t[s][0] < 1 || t[s][1] < 1) continue;
                        const double c = order_makespan(&S, t, cm);
                        if (c < best * (1.0 - 1e-12)) {
                            best = c;
                            best_sl = t;
                        }
                    }
            if (best_sl.empty()) break;
            sl = best_sl;
            cur = best;
        }
        return std::make_pair(cur, sl);
    };
    std::vector<std::array<int, 4>> starts[2];
    starts[0] = U->sl;
    const auto r27 = balanced_partition(L, p, v, head_fwd_s(S.model, cm) / layer_fwd_s(S.model, cm));
    double best = 1e30;
    std::vector<std::array<int, 4>> best_sl;
    for (int k = 0; k < 2; ++k) {
        if (k == 1) {
            if (r27.empty()) break;
            for (int x : r27) starts[1].push_back(split(x));
        }
        auto r = descend(starts[k]);
        if (r.first < best * (1.0 - 1e-12)) {
            best = r.first;
            best_sl = r.second;
        }
    }
    n_out->clear();
    c1_out->clear();
    for (auto& x : best_sl) {
        n_out->push_back(x[0] + x[1]);
        c1_out->push_back(x[0]);
    }
    return best;
}

TP_API int tpipe_plan_create(const tpipe_model_desc* model, int32_t n_stages, int32_t n_microbatches,
                             uint64_t hbm_budget_bytes, const tpipe_plan_opts* opts,
                             tpipe_plan** out) {
    if (!out) return set_error(TPIPE_E_INVALID, "out is NULL");
    *out = nullptr;
    if (int rc = validate(model, n_stages, n_microbatches)) return rc;
    tpipe_plan_opts o{};
    o.strategy = -1;
    o.delay_rounds = -1;
    o.offload = -1;
    if (opts) o = *opts;
    if (o.stage_layers[0] == 0 && model && n_stages > 0 && model->n_layers % n_stages)
        return set_error(TPIPE_E_INVALID, "n_layers must be a positive multiple of n_stages");
    // send window (R12): 2; W = v chunks (the v - 1 chunk turnarounds share the
    // wrap channel; W = 2 deadlocks at v = 4, R32)
    const int W = o.send_window > 0 ? o.send_window : std::max(2, o.chunks > 0 ? o.chunks : 2);
    if (o.strategy < -1 || o.strategy > TPIPE_S_INTERLEAVE_TRECOMP) return set_error(TPIPE_E_INVALID, "strategy");
    if (o.delay_rounds < -1) return set_error(TPIPE_E_INVALID, "delay_rounds");
    if (o.recomp_layers < 0) return set_error(TPIPE_E_INVALID, "recomp_layers");
    if (o.host_link_bps < 0 || o.host_adam_params_per_s < 0 || o.device_flops < 0)
        return set_error(TPIPE_E_INVALID, "cost model rates must be >= 0");
    if (o.dp < 0 || o.dp > 64) return set_error(TPIPE_E_INVALID, "dp must be in [1, 64]");
    const int dp = o.dp > 0 ? o.dp : 1;
    if (o.chunks < 0 || o.chunks == 1 || o.chunks > 4) return set_error(TPIPE_E_INVALID, "chunks must be 2, 3 or 4");
    const int chunks = o.chunks > 0 ? o.chunks : 2;
    if (chunks > 2 && o.balance) return set_error(TPIPE_E_INVALID, "balance is a two-chunk option");
    CostModel cm;
    if (o.host_link_bps > 0) cm.bw = o.host_link_bps;
    if (o.host_adam_params_per_s > 0) cm.host = o.host_adam_params_per_s;
    if (o.device_flops > 0) cm.flops = o.device_flops;
    // cost-balanced, duration-aware partition chosen by the planner (R27 / R29),
    // decided once on the strategy's plain schedule (T-Pipe for auto) and used
    // by every rung
    int32_t part[64] = {0}, chunk1[64] = {0};
    bool balanced = false;
    if (o.stage_layers[0]) {
        std::copy(o.stage_layers, o.stage_layers + 64, part);
        std::copy(o.stage_chunk1, o.stage_chunk1 + 64, chunk1);
    } else if (o.balance && n_stages > 1 && !model->layers_chunk[0] && !model->layers_chunk[1]) {
        const int base = o.strategy >= 0 ? o.strategy : TPIPE_S_TPIPE;
        tpipe_plan* U = nullptr;
        if (!make_plan(model, n_stages, n_microbatches, base, o.delay_rounds, W, 0, o.act_distance,
                       o.recomp_layers, part, chunk1, cm, &U)) {
            std::vector<int> bn, bc;
            const double best = search_partition(U, cm, &bn, &bc);
            if (best < 0.97 * U->est_step_s) {
                for (int s = 0; s < n_stages; ++s) {
                    part[s] = bn[s];
                    chunk1[s] = U->v == 2 ? bc[s] : 0;
                }
                balanced = true;
            }
            delete U;
        }
    }
    auto finish = [&](tpipe_plan* P) {
        P->hbm_budget = hbm_budget_bytes;
        P->balanced = balanced;
        *out = P;
        return 0;
    };
    if (o.strategy >= 0) {
        const int off = o.offload < 0 ? 0 : o.offload;
        tpipe_plan* P = nullptr;
        int rc = make_plan(model, n_stages, n_microbatches, o.strategy, o.delay_rounds, W, off,
                           o.act_distance, o.recomp_layers, part, chunk1, cm, &P, dp, chunks);
        if (rc) return rc;
        if (hbm_budget_bytes && max_peak(P) > hbm_budget_bytes) {
            const uint64_t pk = max_peak(P);
            delete P;
            return set_error(TPIPE_E_BUDGET, "peak %llu bytes exceeds budget %llu",
                             (unsigned long long)pk, (unsigned long long)hbm_budget_bytes);
        }
        return finish(P);
    }
    // auto (fit the budget with the least throughput loss): every rung
    // that fits is costed by the model (R28) and the cheapest wins; ties go to
    // the earlier (simpler) rung
    int n1 = model->layers_chunk[0] ? model->layers_chunk[0] : (model->n_layers / n_stages + 1) / 2;
    if (part[0])
        for (int s = 0; s < n_stages && s < 64; ++s) n1 = std::max(n1, (part[s] + 1) / 2);
    const int rmin = o.recomp_layers > 0 ? o.recomp_layers : 1;
    const int rmax = o.recomp_layers > 0 ? o.recomp_layers : n1;
    const bool ms_ok = o.offload < 0 || (o.offload & TPIPE_OFFLOAD_MODEL_STATE);
    const bool act_ok = o.offload < 0 || (o.offload & TPIPE_OFFLOAD_ACTIVATIONS);
    const int off_ms = TPIPE_OFFLOAD_MODEL_STATE | (o.offload > 0 ? (o.offload & TPIPE_OFFLOAD_DEVICE_OPT) : 0);
    std::vector<std::array<int, 4>> ladder;   // {strategy, offload, r, chunks}
    // chunk counts: the requested one, or (chunks = 0) 2, 3 and 4 (R32: finer
    // chunks recompute a smaller chunk 1 and offload (v - 1)/v of the states)
    std::vector<int> vs;
    if (o.chunks > 0) vs.push_back(o.chunks);
    else vs = {2, 3, 4};
    for (int vv : vs) {
        const int rmx = o.recomp_layers > 0 ? o.recomp_layers
                        : (vv == 2 ? rmax : (model->n_layers / n_stages + vv - 1) / vv);
        ladder.push_back({TPIPE_S_TPIPE, 0, 0, vv});
        if (ms_ok) ladder.push_back({TPIPE_S_TPIPE, off_ms, 0, vv});
        if (act_ok && vv == 2) ladder.push_back({TPIPE_S_TPIPE, TPIPE_OFFLOAD_ACTIVATIONS, 0, vv});
        if (act_ok && ms_ok && vv == 2)
            ladder.push_back({TPIPE_S_TPIPE, TPIPE_OFFLOAD_ACTIVATIONS | off_ms, 0, vv});
        for (int r = rmin; r <= rmx; ++r) ladder.push_back({TPIPE_S_TPIPE_TRECOMP, 0, r, vv});
        if (ms_ok)
            for (int r = rmin; r <= rmx; ++r) ladder.push_back({TPIPE_S_TPIPE_TRECOMP, off_ms, r, vv});
    }
    uint64_t best_peak = ~0ull;
    tpipe_plan* best = nullptr;
    for (auto& rung : ladder) {
        tpipe_plan* P = nullptr;
        const int Wr = o.send_window > 0 ? o.send_window : std::max(2, rung[3]);
        int rc = make_plan(model, n_stages, n_microbatches, rung[0], o.delay_rounds, Wr, rung[1],
                           o.act_distance, rung[2], part, chunk1, cm, &P, dp, rung[3]);
        if (rc) {
            if (rc == TPIPE_E_INCOMPAT || rc == TPIPE_E_INVALID) continue;   // rung not applicable
            delete best;
            return rc;
        }
        best_peak = std::min(best_peak, max_peak(P));
        if ((!hbm_budget_bytes || max_peak(P) <= hbm_budget_bytes) &&
            (!best || P->est_step_s < best->est_step_s * (1.0 - 1e-9))) {
            delete best;
            best = P;
        } else {
            delete P;
        }
    }
    if (best) return finish(best);
    return set_error(TPIPE_E_BUDGET, "no escalation fits: best peak %llu > budget %llu",
                     (unsigned long long)best_peak, (unsigned long long)hbm_budget_bytes);
}

TP_API void tpipe_plan_destroy(tpipe_plan* plan) { delete plan; }

TP_API int tpipe_plan_get_info(const tpipe_plan* P, tpipe_plan_info* out) {
    if (!P || !out) return set_error(TPIPE_E_INVALID, "NULL argument");
    out->n_stages = P->p;
    out->n_microbatches = P->m;
    out->v = P->v;
    out->strategy = P->strategy;
    out->delay_rounds = P->k;
    out->send_window = P->W;
    out->offload = P->offload;
    out->act_distance = P->act_distance;
    out->layers_chunk[0] = P->layers[0];
    out->layers_chunk[1] = P->layers[1];
    out->n_channels = (int32_t)P->channels.size();
    out->params_total = P->params_total;
    out->recomp_layers = P->rl;
    out->est_step_s = P->est_step_s;
    out->est_exposed_offload_s = P->est_exposed_s;
    out->balanced = P->balanced ? 1 : 0;
    out->dp = P->dp;
    return 0;
}

TP_API int tpipe_plan_stage_ops(const tpipe_plan* P, int32_t s, const tpipe_op** ops, size_t* n) {
    if (!P || !ops || !n || s < 0 || s >= P->p) return set_error(TPIPE_E_INVALID, "stage");
    *ops = P->ops[s].data();
    *n = P->ops[s].size();
    return 0;
}

TP_API int tpipe_plan_stage_bufs(const tpipe_plan* P, int32_t s, const tpipe_buf** b, size_t* n) {
    if (!P || !b || !n || s < 0 || s >= P->p) return set_error(TPIPE_E_INVALID, "stage");
    *b = P->bufs[s].data();
    *n = P->bufs[s].size();
    return 0;
}

TP_API int tpipe_plan_stage_events(const tpipe_plan* P, int32_t s, const int32_t** ids, size_t* n) {
    if (!P || !ids || !n || s < 0 || s >= P->p) return set_error(TPIPE_E_INVALID, "stage");
    *ids = P->events[s].data();
    *n = P->events[s].size();
    return 0;
}

TP_API int tpipe_plan_stage_peak(const tpipe_plan* P, int32_t s, tpipe_mem_report* out) {
    if (!P || !out || s < 0 || s >= P->p) return set_error(TPIPE_E_INVALID, "stage");
    *out = P->peak[s];
    return 0;
}

TP_API int tpipe_plan_channel(const tpipe_plan* P, int32_t c, int32_t* kind, int32_t* src,
                              int32_t* dst) {
    if (!P || c < 0 || c >= (int)P->channels.size()) return set_error(TPIPE_E_INVALID, "channel");
    if (kind) *kind = P->channels[c][0];
    if (src) *src = P->channels[c][1];
    if (dst) *dst = P->channels[c][2];
    return 0;
}

TP_API int tpipe_plan_stage_layers(const tpipe_plan* P, int32_t s, int32_t out[2]) {
    if (!P || !out || s < 0 || s >= P->p) return set_error(TPIPE_E_INVALID, "stage");
    out[0] = P->sl[s][0];
    out[1] = P->sl[s][1];
    return 0;
}

TP_API int tpipe_plan_chunk_layers(const tpipe_plan* P, int32_t s, int32_t c, int32_t* n) {
    if (!P || !n || s < 0 || s >= P->p || c < 1 || c > P->v) return set_error(TPIPE_E_INVALID, "stage/chunk");
    *n = P->sl[s][c - 1];
    return 0;
}

TP_API int tpipe_plan_chunk_params(const tpipe_plan* P, int32_t s, int32_t c, uint64_t* n) {
    if (!P || !n || s < 0 || s >= P->p || c < 1 || c > P->v) return set_error(TPIPE_E_INVALID, "stage/chunk");
    *n = P->chunk_params[s][c - 1];
    return 0;
}

// unit-time ASAP replay of the compute order (F=1,B=2,R=1 at v=2; F=2,B=4(+2) at v=1)
TP_API int tpipe_plan_simulate(const tpipe_plan* P, tpipe_sim_report* out) {
    if (!P || !out) return set_error(TPIPE_E_INVALID, "NULL argument");
    const int v = P->v;
    auto dur = [&](int s, int, int kind) -> int64_t {
        if (v >= 2) return kind == KB ? 2 : 1;
        if (kind == KF) return 2;
        if (P->strategy != TPIPE_S_1F1B_FULL_RECOMP) return 4;
        const int n = P->sl[s][0];   // + 2 units per recomputed fraction of the stage's layers (R50: 5)
        return 4 + (2 * P->rl_of(s) + n / 2) / n;
    };
    int64_t mk = 0;
    int rc = replay_order<int64_t>(P, dur, &mk, out->busy);
    out->makespan = mk;
    return rc;
}

TP_API int tpipe_plan_simulate_durations(const tpipe_plan* P, const float* const* op_ms,
                                         tpipe_sim_report_ms* out) {
    if (!P || !out || !op_ms) return set_error(TPIPE_E_INVALID, "NULL argument");
    for (int s = 0; s < P->p; ++s)
        if (!op_ms[s]) return set_error(TPIPE_E_INVALID, "op_ms[%d] is NULL", s);
    auto dur = [&](int s, int j, int) -> double { return (double)op_ms[s][j]; };
    return replay_order<double>(P, dur, &out->makespan_ms, out->busy_ms);
}

TP_API int tpipe_version(void) { return 1; }
