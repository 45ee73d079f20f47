"""Thin Python binding of tpipe_runtime_* / tpipe_step (include/tpipe.h).
Marshals host arrays / device pointers; all work runs in libtpipe.so."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _decl_plan as D
from ._lib import check, lib

STEP_NO_OPT = 1
STEP_PROFILE = 2
STEP_OP_TIMES = 4
STEP_GRAPH = 8

TRANSPORT_NCCL = 0
TRANSPORT_IPC = 1
TRANSPORT_NCCL_LOOPBACK = 2   # stage = -1: virtual pipeline, messages as ncclSend/ncclRecv to self
DEBUG_POOL_CANARY = 1
DEBUG_POOL_CANARY_SELFTEST = 2


class Runtime:
    def __init__(self, plan, stage: int = -1, device: int = 0, nccl_ids: bytes | None = None,
                 lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, pool_cap: int = 0,
                 transport: int = TRANSPORT_NCCL, timeout_ms: int = 0, ipc_name: str | None = None,
                 debug_flags: int = 0, dp_rank: int = 0):
        """stage -1: every stage in this process (virtual pipeline); stage >= 0:
        this process runs one stage and talks to its peers over `transport`
        (NCCL with `nccl_ids`, or CUDA IPC with the job-unique shm `ipc_name`)."""
        self.plan = plan                     # keep the plan alive
        self._ids = C.create_string_buffer(nccl_ids) if nccl_ids else None
        self._ipc = ipc_name.encode() if ipc_name else None
        o = D.RuntimeOpts(stage, device, C.cast(self._ids, C.c_void_p) if self._ids else None,
                          pool_cap, lr, beta1, beta2, eps, weight_decay, transport, timeout_ms,
                          self._ipc, debug_flags, dp_rank)
        self._h = C.c_void_p()
        check(lib().tpipe_runtime_create(plan.handle, C.byref(o), C.byref(self._h)),
              "tpipe_runtime_create")
        self.stage = stage

    def close(self):
        if getattr(self, "_h", None):
            try:
                lib().tpipe_runtime_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    __del__ = close

    def set_params(self, stage, chunk, flat):
        a = np.ascontiguousarray(flat, np.float32)
        check(lib().tpipe_runtime_set_params(self._h, stage, chunk, a.ctypes.data, a.size),
              "set_params")

    def _get(self, fn, stage, chunk):
        n = self.plan.chunk_params(stage, chunk)
        a = np.empty(n, np.float32)
        check(fn(self._h, stage, chunk, a.ctypes.data, n), fn.__name__)
        return a

    def get_params(self, stage, chunk):
        return self._get(lib().tpipe_runtime_get_params, stage, chunk)

    def get_grads(self, stage, chunk):
        return self._get(lib().tpipe_runtime_get_grads, stage, chunk)

    def step(self, tokens, targets, flags: int = 0) -> float:
        """tokens/targets: host int32 [m, b, s] (copied H2D inside the step)."""
        t = np.ascontiguousarray(tokens, np.int32)
        g = np.ascontiguousarray(targets, np.int32)
        loss = C.c_float()
        check(lib().tpipe_step(self._h, t.ctypes.data, g.ctypes.data, flags, C.byref(loss)),
              "tpipe_step")
        return loss.value

    def step_device(self, tok_ptr: int, tgt_ptr: int, flags: int = 0) -> float:
        loss = C.c_float()
        check(lib().tpipe_step_device(self._h, tok_ptr, tgt_ptr, flags, C.byref(loss)),
              "tpipe_step_device")
        return loss.value

    def stats(self):
        s = D.RuntimeStats()
        check(lib().tpipe_runtime_get_stats(self._h, C.byref(s)))
        p = self.plan.p
        return dict(pool_high_water=[s.pool_high_water[i] for i in range(min(p, 64))],
                    pool_reserved=s.pool_reserved, kernel_launches=s.kernel_launches,
                    step=s.step, offload_d2h_bytes=s.offload_d2h_bytes,
                    offload_h2d_bytes=s.offload_h2d_bytes, host_opt_ms=s.host_opt_ms,
                    kernel_ms=list(s.kernel_ms), kernel_flops=list(s.kernel_flops),
                    kernel_count=list(s.kernel_count), offload_d2h_ms=s.offload_d2h_ms,
                    offload_h2d_ms=s.offload_h2d_ms, pool_overflow_bytes=s.pool_overflow_bytes,
                    transport=s.transport, host_issue_ms=s.host_issue_ms)

    def op_times(self, stage):
        """Per compute op (F/B/R, plan order) GPU ms of the last STEP_OP_TIMES step."""
        n = C.c_size_t()
        check(lib().tpipe_runtime_op_times(self._h, stage, None, 0, C.byref(n)))
        a = (C.c_float * max(1, n.value))()
        check(lib().tpipe_runtime_op_times(self._h, stage, a, n.value, C.byref(n)))
        return [a[i] for i in range(n.value)]

    def stream(self) -> int:
        return lib().tpipe_runtime_stream(self._h) or 0


def set_pdl(on: bool) -> None:
    """Programmatic dependent launch of the hot-path kernels (tpipe_set_pdl)."""
    lib().tpipe_set_pdl(1 if on else 0)


def set_side_stream(on: bool) -> None:
    """Weight-gradient GEMMs of each layer backward on a side stream (default on)."""
    lib().tpipe_set_side_stream(1 if on else 0)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().tpipe_nccl_unique_id(buf), "tpipe_nccl_unique_id")
    return buf.raw
