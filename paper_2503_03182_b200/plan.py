"""Thin Python binding of tpipe_plan_* (include/tpipe.h): marshals a model
description into the C struct and reads the immutable plan back."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _decl_plan as D
from ._lib import check, lib

FP32, BF16 = 0, 1
S_1F1B, S_1F1B_FULL_RECOMP, S_TPIPE, S_TPIPE_TRECOMP, S_INTERLEAVE, S_INTERLEAVE_TRECOMP = range(6)
STRATEGY = {"1f1b": S_1F1B, "1f1b_full_recomp": S_1F1B_FULL_RECOMP, "tpipe": S_TPIPE,
            "tpipe_trecomp": S_TPIPE_TRECOMP, "interleave": S_INTERLEAVE,
            "interleave_trecomp": S_INTERLEAVE_TRECOMP}
OFFLOAD_MODEL_STATE = 1
OFFLOAD_ACTIVATIONS = 2
OFFLOAD_DEVICE_OPT = 4   # with OFFLOAD_MODEL_STATE: streamed device AdamW (DESIGN R24)
OP_NAMES = ["F", "B", "R", "RECV_ACT", "RECV_GRAD", "SEND_ACT", "SEND_GRAD", "SEND_WAIT", "OPT",
            "GRAD_D2H", "HOST_OPT", "W_H2D", "W_WAIT", "ACT_D2H", "ACT_D2H_WAIT", "ACT_H2D",
            "ACT_H2D_WAIT", "STREAM_OPT", "DP_OPT", "DP_WAIT"]
CATS = ["model_state", "io", "act", "recomp_buf", "comm", "workspace"]


@dataclass
class Model:
    n_layers: int
    hidden: int
    n_heads: int
    ffn_hidden: int
    vocab: int
    seq_len: int
    micro_batch: int
    dtype: int = BF16
    layers_chunk: tuple = (0, 0)

    def c(self):
        d = D.ModelDesc(self.n_layers, self.hidden, self.n_heads, self.ffn_hidden, self.vocab,
                        self.seq_len, self.micro_batch, self.dtype)
        d.layers_chunk[0], d.layers_chunk[1] = self.layers_chunk
        return d


class Plan:
    """tpipe_plan_create(model, n_stages, n_microbatches, hbm_budget, opts)."""

    def __init__(self, model: Model, n_stages: int, n_microbatches: int, hbm_budget: int = 0,
                 strategy="tpipe", delay_rounds: int = -1, send_window: int = 0, offload: int = 0,
                 act_distance: int = 0, recomp_layers: int = 0, stage_layers=None,
                 host_link_bps: float = 0.0, host_adam_params_per_s: float = 0.0,
                 device_flops: float = 0.0, balance: bool = False, stage_chunk1=None, dp: int = 1,
                 chunks: int = 2):
        L = lib()
        st = -1 if strategy in (None, "auto") else STRATEGY.get(strategy, strategy)
        if st < 0 and offload == 0:
            offload = -1
        sl = (C.c_int32 * 64)(*(list(stage_layers or [])[:64]))
        opts = D.PlanOpts(st, delay_rounds, send_window, offload, act_distance, recomp_layers, sl,
                          host_link_bps, host_adam_params_per_s, device_flops, 1 if balance else 0,
                          (C.c_int32 * 64)(*(list(stage_chunk1 or [])[:64])), dp, chunks)
        self._h = C.c_void_p()
        self.model = model
        check(L.tpipe_plan_create(C.byref(model.c()), n_stages, n_microbatches, hbm_budget,
                                  C.byref(opts), C.byref(self._h)), "tpipe_plan_create")
        info = D.PlanInfo()
        check(L.tpipe_plan_get_info(self._h, C.byref(info)))
        self.p, self.m, self.v = info.n_stages, info.n_microbatches, info.v
        self.strategy, self.k, self.W, self.offload = (info.strategy, info.delay_rounds,
                                                       info.send_window, info.offload)
        self.act_distance = info.act_distance
        self.recomp_layers = info.recomp_layers
        self.est_step_s = info.est_step_s
        self.est_exposed_offload_s = info.est_exposed_offload_s
        self.balanced = bool(info.balanced)
        self.dp = info.dp
        # per-stage (chunk-1, chunk-2) layers (DESIGN R27); == [layers_chunk] * p when uniform
        self.partition = []
        for s in range(self.p):
            row = []
            for ch in range(1, self.v + 1):
                n = C.c_int32()
                check(L.tpipe_plan_chunk_layers(self._h, s, ch, C.byref(n)))
                row.append(n.value)
            self.partition.append(tuple(row))
        self.layers_chunk = (info.layers_chunk[0], info.layers_chunk[1])
        self.params_total = info.params_total
        self.channels = []
        for c in range(info.n_channels):
            k, s, d = C.c_int32(), C.c_int32(), C.c_int32()
            check(L.tpipe_plan_channel(self._h, c, C.byref(k), C.byref(s), C.byref(d)))
            self.channels.append(("A" if k.value == 0 else "G", s.value, d.value))

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().tpipe_plan_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def ops(self, stage):
        L = lib()
        p_ops, n = C.POINTER(D.Op)(), C.c_size_t()
        check(L.tpipe_plan_stage_ops(self._h, stage, C.byref(p_ops), C.byref(n)))
        p_b, nb = C.POINTER(D.Buf)(), C.c_size_t()
        check(L.tpipe_plan_stage_bufs(self._h, stage, C.byref(p_b), C.byref(nb)))
        p_e, ne = C.POINTER(C.c_int32)(), C.c_size_t()
        check(L.tpipe_plan_stage_events(self._h, stage, C.byref(p_e), C.byref(ne)))
        bufs = [(p_b[i].role, CATS[p_b[i].category], p_b[i].chunk, p_b[i].mb, p_b[i].bytes)
                for i in range(nb.value)]
        out = []
        for i in range(n.value):
            o = p_ops[i]
            allocs = [p_e[o.alloc_first + j] for j in range(o.n_alloc)]
            frees = [p_e[o.free_first + j] for j in range(o.n_free)]
            out.append(dict(kind=OP_NAMES[o.kind], chunk=o.chunk, mb=o.mb, peer=o.peer,
                            channel=self.channels[o.channel] if o.channel >= 0 else (),
                            msg=o.msg, allocs=allocs, frees=frees))
        return out, bufs

    def peak(self, stage):
        r = D.MemReport()
        check(lib().tpipe_plan_stage_peak(self._h, stage, C.byref(r)))
        d = {CATS[i]: r.peak[i] for i in range(D.CAT_COUNT)}
        d["total_peak"] = r.total_peak
        d["static"] = r.static_bytes
        return d

    def simulate(self):
        r = D.SimReport()
        check(lib().tpipe_plan_simulate(self._h, C.byref(r)))
        return r.makespan, [r.busy[i] for i in range(min(self.p, 64))]

    def n_compute_ops(self, stage):
        return sum(o["kind"] in ("F", "B", "R") for o in self.ops(stage)[0])

    def simulate_durations(self, op_ms):
        """ASAP replay with per-op durations: op_ms[s] = durations (ms) of stage
        s's compute ops (F/B/R, plan order). Returns (makespan_ms, busy_ms)."""
        arrs = []
        for s in range(self.p):
            a = (C.c_float * len(op_ms[s]))(*[float(x) for x in op_ms[s]])
            if len(op_ms[s]) != self.n_compute_ops(s):
                raise ValueError(f"stage {s}: {len(op_ms[s])} durations for {self.n_compute_ops(s)} ops")
            arrs.append(a)
        ptrs = (C.POINTER(C.c_float) * self.p)(*[C.cast(a, C.POINTER(C.c_float)) for a in arrs])
        r = D.SimReportMs()
        check(lib().tpipe_plan_simulate_durations(self._h, ptrs, C.byref(r)))
        return r.makespan_ms, [r.busy_ms[i] for i in range(min(self.p, 64))]

    def chunk_params(self, stage, chunk):
        n = C.c_uint64()
        check(lib().tpipe_plan_chunk_params(self._h, stage, chunk, C.byref(n)))
        return n.value
