"""Oracle Part 1 (bytes) — per-stage instruction streams and byte-exact replay.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Expands the compute orders of ``oracle.schedule`` into the instruction streams
that ``tpipe_plan`` must emit (DESIGN.md §3 "instruction stream"), attaching
to every instruction the buffers it allocates (at its start) and frees (at its
end). Replaying a stage's stream in order gives the live bytes after every
instruction boundary; its maximum is the stage's peak HBM bytes, which is
order-determined (independent of durations, SURVEY D-16). The byte model
 is the reading of N-2 for this build's kernels.

Everything here is integer arithmetic, written out long-hand.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from collections import defaultdict

from . import schedule as S

FP32, BF16 = 0, 1


@dataclass(frozen=True)
class ModelDesc:
    n_layers: int
    hidden: int
    n_heads: int
    ffn_hidden: int
    vocab: int
    seq_len: int
    micro_batch: int
    dtype: int = BF16
    layers_chunk: tuple = (0, 0)  # per-stage (chunk1, chunk2) layers; 0 = auto
    stage_layers: tuple = ()      # cost-balanced partition: layers of each stage (DESIGN R27)
    stage_chunk1: tuple = ()      # with stage_layers, v=2: chunk-1 layers of each stage (R29)

    @property
    def es(self) -> int:
        return 2 if self.dtype == BF16 else 4

    @property
    def tokens(self) -> int:
        return self.seq_len * self.micro_batch


def layers_per_chunk(d: ModelDesc, p: int, v: int, s: int = 0):
    """n = L/p layers per stage (p | L required). v=2: the extra layer of an odd
    n goes to chunk 1. Override via d.layers_chunk. With
    d.stage_layers (DESIGN R27) stage s holds n(s) layers, split the same way."""
    def split(n):
        # v chunks: n // v each, the extra layers to the shallowest chunks
        # (SURVEY Q14's "extra layer to chunk 1", generalised; DESIGN R32)
        return tuple(n // v + (1 if c < n % v else 0) for c in range(v))

    if d.stage_layers:
        if len(d.stage_layers) != p or sum(d.stage_layers) != d.n_layers:
            raise ValueError("stage_layers")
        n = d.stage_layers[s]
        if n < v:
            raise ValueError("stage_layers")
        if v == 1:
            return (n,)
        if v > 2:
            return split(n)
        n1 = d.stage_chunk1[s] if d.stage_chunk1 and d.stage_chunk1[s] else (n + 1) // 2
        if not 1 <= n1 <= n - 1:
            raise ValueError("stage_chunk1")
        return (n1, n - n1)
    if d.n_layers % p:
        raise ValueError("n_layers")
    n = d.n_layers // p
    if v == 1:
        return (n,)
    if v == 2 and (d.layers_chunk[0] or d.layers_chunk[1]):
        if sum(d.layers_chunk) != n or min(d.layers_chunk) < 1:
            raise ValueError("layers_chunk")
        return tuple(d.layers_chunk)
    if n < v:
        raise ValueError("n_layers")
    return split(n)


def layer_params(d: ModelDesc) -> int:
    h, f = d.hidden, d.ffn_hidden
    ln = 2 * h
    qkv = 3 * h * h + 3 * h
    proj = h * h + h
    fc1 = f * h + f
    fc2 = h * f + h
    return ln + qkv + proj + ln + fc1 + fc2


def chunk_params(d: ModelDesc, p: int, v: int, s: int, c: int) -> int:
    n = layers_per_chunk(d, p, v, s)[c - 1]
    P = n * layer_params(d)
    if s == 0 and c == 1:
        P += d.vocab * d.hidden + d.seq_len * d.hidden          # wte, wpe
    if s == p - 1 and c == v:
        P += 2 * d.hidden + d.vocab * d.hidden                  # ln_f, lm head
    return P


def zero1_shard(P: int, dp: int) -> int:
    """ZeRO-1 optimizer shard of a chunk with P params over dp replicas
    (NEXT-3, DESIGN R31): ceil(P/dp) rounded up to 64 elements; replica r owns
    [r*S, min(P, (r+1)*S))."""
    return -(-(-(-P // dp)) // 64) * 64


def model_state_bytes(d: ModelDesc, P: int, offloaded: bool, dp: int = 1) -> int:
    """bf16: weight 2 + fp32 grad 4 + fp32 master 4 + Adam m,v 8 = 18 B/param;
    fp32: weight(=master) 4 + grad 4 + m,v 8 = 16 B/param.
    T-Offload keeps only weight + grad on the device. With dp > 1
    data-parallel replicas (ZeRO-1) the weight and grad stay whole and
    the master / m / v cover one shard."""
    if offloaded:
        return P * (d.es + 4)
    master = 4 if d.dtype == BF16 else 0
    if dp == 1:
        return P * (d.es + 4 + master + 8)
    return P * (d.es + 4) + zero1_shard(P, dp) * (master + 8)


SOPT_SLICE = 8388608   # parameters per streamed-optimizer slice (include/tpipe.h)


def sopt_staging_bytes(P: int) -> int:
    """Streamed device AdamW (R24; SURVEY §8(d) B200-native option
    for Q11): fp32 master, m, v (12 B/param) of one slice, double-buffered."""
    return 2 * 12 * min(P, SOPT_SLICE)


def n_partials(M: int) -> int:
    """Row blocks of 16 for deterministic column reductions."""
    return -(-M // 16)


def sizes(d: ModelDesc, p: int, v: int, s: int, c: int, full_recomp: bool = False,
          ckpt_layers: int = 0):
    """Byte model per (stage, chunk), DESIGN.md §4. full_recomp: 1F1B +
    layer-grouped recompute of the `ckpt_layers` shallowest layers (0 = all;
    n/2 = 1F1B + R50; DESIGN R33): those keep only their input."""
    M, h, a, f, V, es = d.tokens, d.hidden, d.n_heads, d.ffn_hidden, d.vocab, d.es
    n = layers_per_chunk(d, p, v, s)[c - 1]
    act = M * h * es
    emb = (s == 0 and c == 1)
    head = (s == p - 1 and c == v)
    # per-layer stash: x_in, ln1 mean/rstd, qkv, attn out, lse, x_mid, ln2 stats, u
    LS = M * h * es + 8 * M + 3 * M * h * es + M * h * es + 4 * a * M \
        + M * h * es + 8 * M + M * f * es
    head_stash = M * h * es + 8 * M + 4 * M       # x_f, ln_f stats, CE lse
    ck = (min(ckpt_layers, n) if ckpt_layers else n) if full_recomp else 0
    stash = ck * M * h * es + (n - ck) * LS      # checkpointed layers: their input only
    if not emb:
        stash -= act                             # layer-0 input is the IN buffer
    if head:
        stash += head_stash
    nb = n_partials(M)
    ws_f = M * (h + f) * es
    if full_recomp:
        ws_f += LS - M * h * es                  # one layer's transient internals
    if head:
        ws_f += M * h * es                       # LN_f output (logits and CE run in B)
    ws_b = M * (2 * f + 8 * h) * es + 4 * a * M + 4 * nb * max(f + 3 * h, 6 * h)
    if full_recomp:
        ws_b += LS - M * h * es                  # one-layer recompute buffer
    if head:
        # LN_f output and its gradient, dlogits (es); bf16 runs the fused LM head
        # + CE (DESIGN R30): per-row (max, sum-exp) partials per 64-column group
        # (8 B), target logit and row loss (4 B each) instead of fp32 logits
        ws_b += 2 * M * h * es + M * V * es
        ws_b += 8 * M * (-(-V // 64)) + 8 * M if d.dtype == BF16 else 4 * M * V
    if emb:
        ws_b += 8 * M
    return {
        "act": act, "stash": stash, "ws_f": ws_f, "ws_b": ws_b, "layer_stash": LS,
        "input_is_act": not emb, "has_output": not head,
    }


def partial_trecomp_split(z: dict, n1: int, r: int):
    """Partial T-Recomp (NEXT-1; the recompute ratio r/n1 of P:551, Fig. E56;
    DESIGN.md R25): R regenerates chunk-1 layers 1..r (shallowest first) from
    the checkpoint, so only their stash is transient (TSTASH during F, RBUF
    from R to B); layers r+1..n1 keep theirs from F to B like plain T-Pipe.
    Returns (kept bytes, recomputed bytes) of the chunk-1 stash ``z``."""
    if not 1 <= r <= n1:
        raise ValueError("recomp_layers")
    keep = (n1 - r) * z["layer_stash"]
    return keep, z["stash"] - keep


# --------------------------------------------------------------------------
# instruction streams
# --------------------------------------------------------------------------

@dataclass
class Instr:
    kind: str                      # F B R RECV_ACT RECV_GRAD SEND_ACT SEND_GRAD SEND_WAIT
                                   # OPT GRAD_D2H HOST_OPT W_H2D W_WAIT
                                   # ACT_D2H ACT_D2H_WAIT ACT_H2D ACT_H2D_WAIT STREAM_OPT
    chunk: int = 0
    mb: int = 0
    peer: int = -1
    channel: tuple = ()
    msg: int = -1                  # message index on channel
    allocs: list = field(default_factory=list)   # (name, category, bytes)
    frees: list = field(default_factory=list)    # names

    def key(self):
        return (self.kind, self.chunk, self.mb, self.peer, self.msg)


STRATS = {
    # name: (order strategy, v, recompute chunk-1 block-wise, layer-grouped full)
    "tpipe": ("tpipe", 2, False, False),
    "tpipe_trecomp": ("tpipe_trecomp", 2, True, False),
    "1f1b": ("1f1b", 1, False, False),
    "1f1b_full_recomp": ("1f1b_full_recomp", 1, False, True),
    "interleave": ("interleave", 2, False, False),
    "interleave_trecomp": ("interleave_trecomp", 2, True, False),
}


def act_offload_sets(order, d_release: int, d_prefetch: int):
    """Activation offload (R23; north-star extension of
    P:416): chunk-1 stash blocks whose compute-op distance F(1,i) -> B(1,i)
    exceeds d_release + d_prefetch are copied to host after F, released
    d_release compute ops after F, and prefetched d_prefetch ops before B.
    Returns (offloaded mbs, release_at[op index], fetch_at[op index])."""
    pos = {op: n for n, op in enumerate(order)}
    off, rel, fet = [], defaultdict(list), defaultdict(list)
    for op, n in pos.items():
        if op[0] == "F" and op[1] == 1:
            nb = pos[("B", 1, op[2])]
            if nb - n > d_release + d_prefetch:
                off.append(op[2])
                rel[n + d_release].append(op[2])
                fet[nb - d_prefetch].append(op[2])
    return set(off), rel, fet


def build_streams(d: ModelDesc, p: int, m: int, strategy: str, k=None,
                  window: int | None = None, offload_model_state: bool = False,
                  offload_activations: bool = False, act_distance: int = 2,
                  offload_device_opt: bool = False, recomp_layers: int = 0, dp: int = 1,
                  chunks: int = 2):
    """Per-stage instruction streams. Returns (streams, static)
    where static[s] = list of (name, category, bytes) live for the whole step.
    ``recomp_layers`` = r of partial T-Recomp (0 = all chunk-1 layers)."""
    ostrat, v, trecomp, full = STRATS[strategy]
    if v == 2:
        v = chunks          # T-Pipe / Interleave with v chunks per stage (NEXT-4, R32)
    elif chunks != 2:
        raise ValueError("chunks applies to the T-Pipe and Interleave strategies")
    if window is None:
        # send window (R12, D-14): 2; v chunks put v - 1 chunk turnarounds on the
        # wrap channel, and W = v is the smallest deadlock-free window at v = 4
        # (R32, tests/test_multichunk.py)
        window = max(2, v)
    if offload_model_state and v < 2:
        raise ValueError("offload requires T-Pipe chunks (v >= 2)")
    if offload_device_opt and not offload_model_state:
        raise ValueError("device optimizer streaming applies to model-state offload")
    if dp > 1 and offload_model_state:
        raise ValueError("ZeRO-1 data parallelism shards the device optimizer (no model-state offload)")
    if offload_activations and (v != 2 or trecomp):
        raise ValueError("activation offload applies to T-Pipe chunk 1 (no T-Recomp)")
    orders = S.strategy_orders(ostrat, p, m, k=k, v=v)[0]
    if full and recomp_layers > max(layers_per_chunk(d, p, v, s)[0] for s in range(p)):
        raise ValueError("recomp_layers")
    # 1F1B + recompute: stage s recomputes min(r, n(s)) layers (0 = all)
    sz = {(s, c): sizes(d, p, v, s, c, full_recomp=full,
                        ckpt_layers=min(recomp_layers, layers_per_chunk(d, p, v, s)[0]) if full else 0)
          for s in range(p) for c in range(1, v + 1)}
    keep1, rec1 = {}, {}
    if trecomp:
        n1max = max(layers_per_chunk(d, p, v, s)[0] for s in range(p))
        r = recomp_layers if recomp_layers else n1max
        if r > n1max:
            raise ValueError("recomp_layers")
        for s in range(p):
            n1 = layers_per_chunk(d, p, v, s)[0]
            keep1[s], rec1[s] = partial_trecomp_split(sz[(s, 1)], n1, min(r, n1))

    static = []
    for s in range(p):
        st = []
        for c in range(1, v + 1):
            P = chunk_params(d, p, v, s, c)
            off = offload_model_state and c >= 2        # chunks 2..v (R32)
            extra = sopt_staging_bytes(P) if (off and offload_device_opt) else 0
            st.append((f"MS{c}", "model_state", model_state_bytes(d, P, off, dp) + extra))
        if s == 0:
            st.append(("TOKENS", "io", 4 * m * d.tokens))
        if s == p - 1:
            st.append(("TARGETS", "io", 4 * m * d.tokens + 4 * m))
        static.append(st)

    # message indices per channel on the sender side
    streams = []
    for s in range(p):
        out = []
        sent = defaultdict(int)          # channel -> messages produced so far
        waited = defaultdict(int)        # channel -> messages waited
        last_b = {c: max(op[2] for op in orders[s] if op[0] == "B" and op[1] == c)
                  for c in range(1, v + 1)}
        first_f = {c: min(op[2] for op in orders[s] if op[0] == "F" and op[1] == c)
                   for c in range(1, v + 1)}
        first_op_done = False
        if offload_activations:
            aoff, arel, afet = act_offload_sets(orders[s], act_distance, act_distance)
        else:
            aoff, arel, afet = set(), {}, {}
        for n_op, op in enumerate(orders[s]):
            kind, c, i = op
            z = sz[(s, c)]
            msg = S.message_of(s, op, p, v)
            # 0. activation offload: release copied blocks, start prefetches
            for mb in sorted(arel.get(n_op, [])):
                out.append(Instr("ACT_D2H_WAIT", 1, mb, frees=[("STASH", 1, mb)]))
            for mb in sorted(afet.get(n_op, [])):
                out.append(Instr("ACT_H2D", 1, mb,
                                 allocs=[(("STASH", 1, mb), "act", sz[(s, 1)]["stash"])]))
            # 1. send-window wait before the op producing message j+W
            if msg is not None:
                ch = msg[0]
                j = sent[ch]
                while waited[ch] <= j - window:
                    jj = waited[ch]
                    out.append(Instr("SEND_WAIT", channel=ch, peer=ch[2], msg=jj,
                                     frees=[_msgbuf(ch, jj)]))
                    waited[ch] += 1
            # 2. receive before the consuming op
            if offload_model_state and kind == "F" and c >= 2 and i == first_f[c]:
                out.append(Instr("W_WAIT", chunk=c))
            if dp > 1 and kind == "F" and i == first_f[c]:
                # the replicas' previous-step ZeRO-1 update of this chunk is complete
                out.append(Instr("DP_WAIT", chunk=c))
            if kind == "F" and z["input_is_act"]:
                src = _src_stage(s, c, p, "F")
                if src is not None and src != s:
                    ch = ("A", src, s)
                    out.append(Instr("RECV_ACT", c, i, peer=src, channel=ch,
                                     allocs=[(("IN", c, i), "act", z["act"])]))
            if kind == "B" and z["has_output"]:
                src = _src_stage(s, c, p, "B", v)
                if src is not None and src != s:
                    ch = ("G", src, s)
                    out.append(Instr("RECV_GRAD", c, i, peer=src, channel=ch,
                                     allocs=[(("GIN", c, i), "comm", z["act"])]))
            if kind == "B" and c == 1 and i in aoff:
                out.append(Instr("ACT_H2D_WAIT", 1, i))
            # 3. the compute op
            ins = Instr(kind, c, i)
            if kind == "F":
                if trecomp and c == 1:
                    ins.allocs.append((("TSTASH", c, i), "act", rec1[s]))
                    ins.frees.append(("TSTASH", c, i))
                    if keep1[s]:
                        ins.allocs.append((("STASH", c, i), "act", keep1[s]))
                else:
                    ins.allocs.append((("STASH", c, i), "act", z["stash"]))
                if msg is not None:
                    ins.allocs.append((_msgbuf(msg[0], sent[msg[0]]), "comm", z["act"]))
                elif z["has_output"]:
                    # p == 1 local hand-off: output is the next chunk's input
                    ins.allocs.append((("IN", c + 1, i), "act", z["act"]))
                ins.allocs.append((("WSF", c, i), "workspace", z["ws_f"]))
                ins.frees.append(("WSF", c, i))
            elif kind == "R":
                ins.allocs.append((("RBUF", c, i), "recomp_buf", rec1[s]))
                ins.allocs.append((("WSR", c, i), "workspace", z["ws_f"]))
                ins.frees.append(("WSR", c, i))
            else:  # B
                if msg is not None:
                    ins.allocs.append((_msgbuf(msg[0], sent[msg[0]]), "comm", z["act"]))
                elif not (s == 0 and c == 1):
                    ins.allocs.append((("GIN", c - 1, i), "comm", z["act"]))
                ins.allocs.append((("WSB", c, i), "workspace", z["ws_b"]))
                ins.frees.append(("WSB", c, i))
                if trecomp and c == 1:
                    ins.frees.append(("RBUF", c, i))
                    if keep1[s]:
                        ins.frees.append(("STASH", c, i))
                else:
                    ins.frees.append(("STASH", c, i))
                if z["input_is_act"]:
                    ins.frees.append(("IN", c, i))
                if z["has_output"]:
                    ins.frees.append(("GIN", c, i))
            out.append(ins)
            # 4. send after the producing op
            if msg is not None:
                ch = msg[0]
                out.append(Instr("SEND_ACT" if kind == "F" else "SEND_GRAD", c, i,
                                 peer=ch[2], channel=ch, msg=sent[ch]))
                sent[ch] += 1
            if kind == "F" and c == 1 and i in aoff:
                out.append(Instr("ACT_D2H", 1, i))
            # 5. optimizer / offload after the chunk's last backward
            if kind == "B" and i == last_b[c]:
                if offload_model_state and c >= 2 and offload_device_opt:
                    out.append(Instr("STREAM_OPT", chunk=c))
                elif offload_model_state and c >= 2:
                    out.append(Instr("GRAD_D2H", chunk=c))
                    out.append(Instr("HOST_OPT", chunk=c))
                elif dp > 1:
                    out.append(Instr("DP_OPT", chunk=c))
                else:
                    out.append(Instr("OPT", chunk=c))
            # weight upload right after the stage's first forward
            if offload_model_state and not offload_device_opt and not first_op_done and kind == "F":
                for cc in range(2, v + 1):
                    out.append(Instr("W_H2D", chunk=cc))
            first_op_done = first_op_done or kind == "F"
        # 6. flush outstanding sends (channels sorted, then message order)
        for ch in sorted(sent):
            while waited[ch] < sent[ch]:
                jj = waited[ch]
                out.append(Instr("SEND_WAIT", channel=ch, peer=ch[2], msg=jj,
                                 frees=[_msgbuf(ch, jj)]))
                waited[ch] += 1
        streams.append(out)
    return streams, static


def _msgbuf(ch, j):
    return ("MSG", ch, j)


def _src_stage(s, c, p, kind, v=2):
    """Stage producing the input (F) or output-grad (B) of chunk op (s, c)."""
    if kind == "F":
        if s > 0:
            return s - 1
        if c > 1:
            return p - 1
        return None
    if s < p - 1:
        return s + 1
    if c < v:
        return 0
    return None


def replay(stream, static):
    """Live-byte replay: allocs at instruction start, frees at its end.
    Returns {'total_peak', per-category peaks, 'final'}; 'final' must equal the
    static bytes (everything transient released at step end)."""
    live = {}
    cat_live = defaultdict(int)
    cat_peak = defaultdict(int)
    base = sum(b for _n, _c, b in static)
    for _n, cat, b in static:
        cat_live[cat] += b
        cat_peak[cat] = max(cat_peak[cat], cat_live[cat])
    cur = base
    peak = cur
    for ins in stream:
        for name, cat, b in ins.allocs:
            assert name not in live, f"double alloc {name}"
            live[name] = (cat, b)
            cur += b
            cat_live[cat] += b
            cat_peak[cat] = max(cat_peak[cat], cat_live[cat])
        peak = max(peak, cur)
        for name in ins.frees:
            cat, b = live.pop(name)
            cur -= b
            cat_live[cat] -= b
    assert not live, f"leaked {list(live)[:4]}"
    out = dict(cat_peak)
    out["total_peak"] = peak
    out["final"] = cur
    return out


def deadlock_free(streams) -> bool:
    """Static deadlock test: nodes are instructions;
    edges are program order, SEND(j) -> RECV(j) and RECV(j) -> SEND_WAIT(j)
    (a send completes only once its receive is posted). Acyclic <=> no
    deadlock for any durations. Kahn's algorithm."""
    nodes = []
    idx = {}
    for s, st in enumerate(streams):
        for n, ins in enumerate(st):
            idx[(s, n)] = len(nodes)
            nodes.append((s, n, ins))
    succ = defaultdict(list)
    indeg = [0] * len(nodes)

    def edge(a, b):
        succ[a].append(b)
        indeg[b] += 1

    sends, recvs, waits = {}, {}, {}
    recv_count = defaultdict(int)
    for s, st in enumerate(streams):
        for n, ins in enumerate(st):
            if n:
                edge(idx[(s, n - 1)], idx[(s, n)])
            if ins.kind in ("SEND_ACT", "SEND_GRAD"):
                sends[(ins.channel, ins.msg)] = idx[(s, n)]
            elif ins.kind in ("RECV_ACT", "RECV_GRAD"):
                j = recv_count[ins.channel]
                recv_count[ins.channel] += 1
                recvs[(ins.channel, j)] = idx[(s, n)]
            elif ins.kind == "SEND_WAIT":
                waits[(ins.channel, ins.msg)] = idx[(s, n)]
    for key, a in sends.items():
        edge(a, recvs[key])
    for key, w in waits.items():
        edge(recvs[key], w)
    q = [x for x in range(len(nodes)) if indeg[x] == 0]
    seen = 0
    while q:
        x = q.pop()
        seen += 1
        for y in succ[x]:
            indeg[y] -= 1
            if indeg[y] == 0:
                q.append(y)
    return seen == len(nodes)


def fifo_consistent(streams) -> bool:
    """Receiver consume order equals sender production order on every channel
    (SURVEY D-14): the j-th RECV on a channel must receive the (chunk, mb) the
    j-th SEND produced for it."""
    sent = defaultdict(list)
    got = defaultdict(list)
    p = len(streams)
    for s, st in enumerate(streams):
        for ins in st:
            if ins.kind == "SEND_ACT":
                # consumer (chunk, mb): wrap edge p-1 -> 0 advances the chunk
                c = ins.chunk + 1 if (s == p - 1 and ins.channel[2] == 0 and p > 1
                                      and s != 0) else ins.chunk
                sent[ins.channel].append((c, ins.mb))
            elif ins.kind == "SEND_GRAD":
                c = ins.chunk - 1 if (s == 0 and ins.channel[2] == p - 1 and p > 1) else ins.chunk
                sent[ins.channel].append((c, ins.mb))
            elif ins.kind in ("RECV_ACT", "RECV_GRAD"):
                got[ins.channel].append((ins.chunk, ins.mb))
    return all(sent[ch] == got[ch] for ch in set(sent) | set(got))
