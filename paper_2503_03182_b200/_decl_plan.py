"""ctypes prototypes for the plan / runtime part of include/tpipe.h."""

import ctypes as C

i32, u32, u64, i64, f32, vp = C.c_int32, C.c_uint32, C.c_uint64, C.c_int64, C.c_float, C.c_void_p


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", i32), ("hidden", i32), ("n_heads", i32), ("ffn_hidden", i32),
                ("vocab", i32), ("seq_len", i32), ("micro_batch", i32), ("dtype", i32),
                ("layers_chunk", i32 * 2)]


class PlanOpts(C.Structure):
    _fields_ = [("strategy", i32), ("delay_rounds", i32), ("send_window", i32), ("offload", i32),
                ("act_distance", i32), ("recomp_layers", i32), ("stage_layers", i32 * 64),
                ("host_link_bps", C.c_double), ("host_adam_params_per_s", C.c_double),
                ("device_flops", C.c_double), ("balance", i32), ("stage_chunk1", i32 * 64),
                ("dp", i32), ("chunks", i32)]


class Op(C.Structure):
    _fields_ = [("kind", i32), ("chunk", i32), ("mb", i32), ("peer", i32), ("channel", i32),
                ("msg", i32), ("alloc_first", i32), ("n_alloc", i32), ("free_first", i32),
                ("n_free", i32)]


class Buf(C.Structure):
    _fields_ = [("role", i32), ("category", i32), ("chunk", i32), ("mb", i32), ("bytes", u64)]


CAT_COUNT = 6


class MemReport(C.Structure):
    _fields_ = [("peak", u64 * CAT_COUNT), ("total_peak", u64), ("static_bytes", u64)]


class PlanInfo(C.Structure):
    _fields_ = [("n_stages", i32), ("n_microbatches", i32), ("v", i32), ("strategy", i32),
                ("delay_rounds", i32), ("send_window", i32), ("offload", i32), ("act_distance", i32),
                ("layers_chunk", i32 * 2), ("n_channels", i32), ("params_total", u64),
                ("recomp_layers", i32), ("est_step_s", C.c_double),
                ("est_exposed_offload_s", C.c_double), ("balanced", i32), ("dp", i32)]


class SimReport(C.Structure):
    _fields_ = [("makespan", i64), ("busy", i64 * 64)]


class SimReportMs(C.Structure):
    _fields_ = [("makespan_ms", C.c_double), ("busy_ms", C.c_double * 64)]


class RuntimeOpts(C.Structure):
    _fields_ = [("stage", i32), ("device", i32), ("nccl_ids", vp), ("pool_cap", u64),
                ("lr", f32), ("beta1", f32), ("beta2", f32), ("eps", f32), ("weight_decay", f32),
                ("transport", i32), ("timeout_ms", i32), ("ipc_name", C.c_char_p),
                ("debug_flags", u32), ("dp_rank", i32)]


class RuntimeStats(C.Structure):
    _fields_ = [("pool_high_water", u64 * 64), ("pool_reserved", u64), ("kernel_launches", i64),
                ("step", i64), ("offload_d2h_bytes", C.c_double),
                ("offload_h2d_bytes", C.c_double), ("host_opt_ms", C.c_double),
                ("kernel_ms", C.c_double * 4), ("kernel_flops", C.c_double * 4),
                ("kernel_count", i64 * 4), ("offload_d2h_ms", C.c_double),
                ("offload_h2d_ms", C.c_double), ("pool_overflow_bytes", u64), ("transport", i32),
                ("host_issue_ms", C.c_double)]


def declare(L):
    P = C.POINTER
    L.tpipe_plan_create.argtypes = [P(ModelDesc), i32, i32, u64, P(PlanOpts), P(vp)]
    L.tpipe_plan_destroy.argtypes = [vp]
    L.tpipe_plan_destroy.restype = None
    L.tpipe_plan_get_info.argtypes = [vp, P(PlanInfo)]
    L.tpipe_plan_stage_ops.argtypes = [vp, i32, P(P(Op)), P(C.c_size_t)]
    L.tpipe_plan_stage_bufs.argtypes = [vp, i32, P(P(Buf)), P(C.c_size_t)]
    L.tpipe_plan_stage_events.argtypes = [vp, i32, P(P(i32)), P(C.c_size_t)]
    L.tpipe_plan_stage_peak.argtypes = [vp, i32, P(MemReport)]
    L.tpipe_plan_channel.argtypes = [vp, i32, P(i32), P(i32), P(i32)]
    L.tpipe_plan_simulate.argtypes = [vp, P(SimReport)]
    L.tpipe_plan_simulate_durations.argtypes = [vp, P(P(f32)), P(SimReportMs)]
    L.tpipe_plan_chunk_params.argtypes = [vp, i32, i32, P(u64)]
    L.tpipe_plan_stage_layers.argtypes = [vp, i32, P(i32)]
    L.tpipe_plan_chunk_layers.argtypes = [vp, i32, i32, P(i32)]
    L.tpipe_version.argtypes = []
    if hasattr(L, "tpipe_runtime_create"):
        L.tpipe_runtime_create.argtypes = [vp, P(RuntimeOpts), P(vp)]
        L.tpipe_runtime_destroy.argtypes = [vp]
        L.tpipe_runtime_destroy.restype = None
        for n in ("tpipe_runtime_set_params", "tpipe_runtime_get_params", "tpipe_runtime_get_grads"):
            getattr(L, n).argtypes = [vp, i32, i32, vp, u64]
        L.tpipe_step.argtypes = [vp, vp, vp, u32, P(f32)]
        L.tpipe_step_device.argtypes = [vp, vp, vp, u32, P(f32)]
        L.tpipe_runtime_get_stats.argtypes = [vp, P(RuntimeStats)]
        L.tpipe_runtime_op_times.argtypes = [vp, i32, P(f32), C.c_size_t, P(C.c_size_t)]
        L.tpipe_runtime_stream.argtypes = [vp]
        L.tpipe_runtime_stream.restype = vp
        L.tpipe_nccl_unique_id.argtypes = [vp]
        L.tpipe_set_side_stream.argtypes = [i32]
        L.tpipe_set_side_stream.restype = None
        L.tpipe_set_pdl.argtypes = [i32]
        L.tpipe_set_pdl.restype = None
