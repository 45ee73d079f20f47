/*
 * tpipe.h — C-ABI of libtpipe.so: the B200-native TPipe training hot path.
 *
 * Problem statement: given a model,
 * P pipeline stages, m micro-batches and a fixed HBM capacity, choose a
 * pipeline schedule plus recompute / offload decisions that fit HBM with
 * minimal throughput loss. Two calls follow it:
 *
 *   tpipe_plan_create(model, n_stages, n_microbatches, hbm_budget, opts)
 *       -> per-stage instruction streams (T-Pipe order P:303-310 / App. A
 *          P:611-636; T-Recomp P:324-367 / App. B-C; T-Offload
 *          P:376-420 / App. D), byte-exact per-stage peak HBM.
 *   tpipe_step(runtime, tokens, targets, ...)
 *       -> one training step executed from those streams with sm_100a
 *          kernels, an exact-accounting HBM pool, copy-engine offload and
 *          stage-to-stage transport.
 *
 * Conventions
 *   - All functions return 0 on success or a negative TPIPE_E_* code; the
 *     thread-local message of the last failure is tpipe_last_error().
 *   - Pointers are HOST pointers unless documented as device pointers.
 *   - Structs passed in are copied; nothing caller-owned is retained.
 *   - Objects returned through `**out` are owned by the library and released
 *     by the matching *_destroy. Pointers borrowed from a plan
 *     (tpipe_plan_stage_ops/bufs/events) stay valid until tpipe_plan_destroy.
 *   - A plan is immutable and may be read concurrently; a runtime is not
 *     thread-safe (one per process / rank).
 *
 * Readings of the paper used here are listed in DESIGN.md (R1..R22); the
 * instruction-stream and byte model are DESIGN.md §3-§4.
 */
#ifndef TPIPE_H
#define TPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ codes */
#define TPIPE_OK            0
#define TPIPE_E_INVALID    -1   /* invalid argument / config field (message names it) */
#define TPIPE_E_INCOMPAT   -2   /* strategy incompatible with config (e.g. v) */
#define TPIPE_E_DOMAIN     -3   /* outside a formula's domain */
#define TPIPE_E_CONFLICT   -4   /* schedule dependency conflict */
#define TPIPE_E_DEADLOCK   -5   /* instruction streams can deadlock */
#define TPIPE_E_BUDGET     -6   /* no escalation fits the HBM budget */
#define TPIPE_E_CUDA       -7
#define TPIPE_E_NCCL       -8
#define TPIPE_E_OOM        -9   /* runtime pool cap hit (a ledger bug) */
#define TPIPE_E_STATE     -10   /* call not valid in the current state */
#define TPIPE_E_TIMEOUT   -11   /* a transport wait or the step exceeded timeout_ms (peer hung) */

#define TPIPE_FP32 0
#define TPIPE_BF16 1

/* ------------------------------------------------------------------ plan */
typedef struct {
    int32_t n_layers;        /* L, transformer blocks; must be divisible by n_stages */
    int32_t hidden;          /* h, multiple of 64 */
    int32_t n_heads;         /* a, h % a == 0, head_dim <= 128 */
    int32_t ffn_hidden;      /* multiple of 64 */
    int32_t vocab;           /* V, multiple of 64 */
    int32_t seq_len;         /* s */
    int32_t micro_batch;     /* b; tokens per micro-batch M = b*s */
    int32_t dtype;           /* TPIPE_FP32 | TPIPE_BF16 */
    int32_t layers_chunk[2]; /* per-stage layers of chunk 1 / chunk 2; {0,0} = auto (R14) */
} tpipe_model_desc;

enum {
    TPIPE_S_1F1B = 0,             /* DAPPLE 1F1B, P:202 (baseline) */
    TPIPE_S_1F1B_FULL_RECOMP = 1, /* 1F1B + full layer-grouped recompute */
    TPIPE_S_TPIPE = 2,            /* T-Pipe, v = 2 */
    TPIPE_S_TPIPE_TRECOMP = 3,    /* T-Pipe + block-wise T-Recomp of chunk 1 */
    TPIPE_S_INTERLEAVE = 4,       /* Interleave-1F1B, v = 2 (Megatron virtual pipeline);
                                     needs n_microbatches % n_stages == 0 */
    TPIPE_S_INTERLEAVE_TRECOMP = 5 /* Interleave-1F1B + block-wise T-Recomp of chunk 1 (P:367,
                                     Fig. 6(e); DESIGN R26) */
};

#define TPIPE_OFFLOAD_MODEL_STATE 1   /* T-Offload of chunk-2 grads/optimizer/weights */
#define TPIPE_OFFLOAD_ACTIVATIONS 2   /* chunk-1 stash to pinned host and back (R23) */
/* With TPIPE_OFFLOAD_MODEL_STATE: run the offloaded chunk's AdamW on the
 * device instead of the host (SURVEY §8(d), B200-native option for Q11;
 * DESIGN R24). fp32 master / m / v stay in pinned host memory and are streamed
 * through a double-buffered device staging area in slices of
 * TPIPE_SOPT_SLICE_PARAMS parameters (H2D -> device AdamW -> D2H); the fp32
 * grads never leave HBM and the bf16 weights are written in place. The
 * staging area, 2 x min(P, slice) x 12 bytes, is static model-state memory. */
#define TPIPE_OFFLOAD_DEVICE_OPT 4
#define TPIPE_SOPT_SLICE_PARAMS 8388608

typedef struct {
    int32_t strategy;      /* TPIPE_S_*, or -1 = auto (fit hbm_budget with the least
                              throughput loss): among T-Pipe, T-Pipe + model-state T-Offload,
                              T-Pipe + activation offload (+ model-state T-Offload), T-Recomp
                              with r = 1..n1 recomputed layers (+ model-state T-Offload), the
                              plan with the smallest cost-model step time that fits (offload
                              kinds limited by `offload` when it is not -1; DEVICE_OPT if
                              requested there) */
    int32_t delay_rounds;  /* T-Recomp k; -1 = App. B constraint as printed */
    int32_t send_window;   /* W, max in-flight sends per channel; 0 = default max(2, chunks)
                              (DESIGN R12, R32); the IPC transport supports W <= 4 */
    int32_t offload;       /* TPIPE_OFFLOAD_* bitmask (explicit strategies); -1 = auto */
    int32_t act_distance;  /* activation offload: release / prefetch distance in compute
                              ops; 0 = derived: the smallest d whose d chunk-1 forward
                              times (cost model) cover one block's copy at host_link_bps
                              (SURVEY Q12), >= 1; blocks with F->B distance <= 2d are kept */
    int32_t recomp_layers; /* partial T-Recomp (the recompute ratio of
                              P:551, Fig. E56): chunk-1 layers per stage that R regenerates,
                              shallowest first; the deeper n1 - r layers keep their stash
                              from F to B. 0 = all n1 layers (block-wise T-Recomp).
                              Must be <= n1. With strategy -1 (auto) and 0 here, the
                              escalation tries r = 1..n1 at each rung (DESIGN R25);
                              with stage_layers, stage s recomputes min(r, n1(s)) layers.
                              With TPIPE_S_1F1B_FULL_RECOMP: the shallowest r layers of each
                              stage are recomputed layer-wise in B (r = n/2 is the paper's
                              1F1B + R50 baseline; DESIGN R33); 0 = all (full) */
    int32_t stage_layers[64]; /* cost-balanced partition (SURVEY D-12, DESIGN R27): transformer
                              layers held by stage s (chunk split ceil/floor of n(s)/2 at
                              v = 2); all zero = uniform n_layers / n_stages. When set: the
                              first n_stages entries sum to n_layers, each >= 2 at v = 2 (>= 1
                              at v = 1), model.layers_chunk must be {0, 0} */
    /* Planner cost model (DESIGN R28; SURVEY §8(b) host_link_bps /
     * host_adam_params_per_s): per-op durations from FLOPs (F = the chunk's
     * layers (+ the LM head), B = 2F, R = recomputed layers) replayed ASAP over
     * the plan's order, plus the offload transfer time that does not fit the
     * window the schedule leaves it (model states: from the last deep-chunk
     * backward to the next step's first deep-chunk forward, P:680/P:694;
     * activations: the stage's busy time). Used to (1) order the auto ladder by
     * estimated step time, (2) derive the activation release / prefetch
     * distance from bytes / bandwidth when act_distance = 0, and
     * (3) choose a cost-balanced partition when `balance` is set.
     * 0 = defaults (50e9 B/s, 3e9 params/s, 1e15 FLOP/s: this build's measured
     * pinned-link, host AdamW and in-step GEMM rates on B200). */
    double host_link_bps;
    double host_adam_params_per_s;
    double device_flops;
    int32_t balance;       /* 1: use the cost-balanced stage_layers partition (the last stage
                              also runs the LM head, SURVEY D-12) when the modeled step is >= 3%
                              shorter than the uniform split; ignored if stage_layers is set.
                              The partition is found by steepest descent over per-stage layer
                              counts and chunk splits on the cost model's ASAP replay of the
                              strategy's own order (duration-aware T-Pipe, SURVEY NEXT-5,
                              DESIGN R29), started from the uniform split and the R27 closed form */
    int32_t stage_chunk1[64]; /* with stage_layers at v = 2: chunk-1 layers of stage s
                              (1 .. n(s)-1); 0 = ceil(n(s)/2) */
    int32_t dp;            /* data-parallel replicas of the pipeline (SURVEY NEXT-3, P:484;
                              DESIGN R31); 0 = 1. Each replica runs n_microbatches per step,
                              the loss is the mean over all dp * n_microbatches micro-batches,
                              optimizer states are sharded ZeRO-1 (master / m / v of
                              ceil64(P / dp) parameters per replica) and updated by
                              TPIPE_OP_DP_OPT. Incompatible with model-state offload */
    int32_t chunks;        /* v, chunks per stage of the T-Pipe and Interleave strategies
                              (DESIGN R32): 0 = 2, or 3, 4.
                              Per stage n / v layers per chunk, the extra ones to the
                              shallowest chunks; T-Pipe uses the period-3v slot table (D-11);
                              T-Recomp regenerates chunk 1; model-state T-Offload moves chunks
                              2..v. layers_chunk, stage_chunk1 and balance need v = 2.
                              With strategy -1 (auto), 0 lets the ladder try v = 2, 3, 4 */
} tpipe_plan_opts;

enum {
    TPIPE_OP_F = 0, TPIPE_OP_B = 1, TPIPE_OP_R = 2,
    TPIPE_OP_RECV_ACT = 3, TPIPE_OP_RECV_GRAD = 4,
    TPIPE_OP_SEND_ACT = 5, TPIPE_OP_SEND_GRAD = 6, TPIPE_OP_SEND_WAIT = 7,
    TPIPE_OP_OPT = 8, TPIPE_OP_GRAD_D2H = 9, TPIPE_OP_HOST_OPT = 10,
    TPIPE_OP_W_H2D = 11, TPIPE_OP_W_WAIT = 12,
    TPIPE_OP_ACT_D2H = 13,       /* copy STASH(1,i) to pinned host (after F) */
    TPIPE_OP_ACT_D2H_WAIT = 14,  /* copy done -> release STASH(1,i) on the device */
    TPIPE_OP_ACT_H2D = 15,       /* re-allocate STASH(1,i), start the prefetch */
    TPIPE_OP_ACT_H2D_WAIT = 16,  /* prefetch landed (before B(1,i)) */
    TPIPE_OP_STREAM_OPT = 17,    /* TPIPE_OFFLOAD_DEVICE_OPT: streamed device AdamW of the
                                    offloaded chunk (replaces GRAD_D2H, HOST_OPT, W_H2D) */
    TPIPE_OP_DP_OPT = 18,        /* dp > 1 (ZeRO-1, DESIGN R31): replaces OPT. One kernel per
                                    replica reads its parameter shard's gradients from every
                                    replica of the stage over peer memory (NVLink), sums them
                                    in replica order, zeroes them, runs AdamW on its shard of
                                    master / m / v and writes the bf16 weights into every
                                    replica (reduce-scatter + optimizer + all-gather fused) */
    TPIPE_OP_DP_WAIT = 19        /* dp > 1: before a chunk's first forward, wait until every
                                    replica's previous-step DP_OPT of that chunk finished */
};

/* One instruction of a stage's stream. Buffers listed in
 * events[alloc_first .. +n_alloc) are allocated when the instruction starts,
 * events[free_first .. +n_free) are released when it ends. */
typedef struct {
    int32_t kind;        /* TPIPE_OP_* */
    int32_t chunk;       /* 1 or 2 (0 if not applicable) */
    int32_t mb;          /* micro-batch 1..m (0 if not applicable) */
    int32_t peer;        /* peer stage for SEND/RECV/SEND_WAIT, else -1 */
    int32_t channel;     /* channel id (tpipe_plan_channel), else -1 */
    int32_t msg;         /* message index on the channel (sender side), else -1 */
    int32_t alloc_first, n_alloc, free_first, n_free;
} tpipe_op;

enum {
    TPIPE_CAT_MODEL_STATE = 0, TPIPE_CAT_IO = 1, TPIPE_CAT_ACT = 2, TPIPE_CAT_RECOMP_BUF = 3,
    TPIPE_CAT_COMM = 4, TPIPE_CAT_WORKSPACE = 5, TPIPE_CAT_COUNT = 6
};

enum {  /* buffer roles */
    TPIPE_BUF_STASH = 0, TPIPE_BUF_TSTASH = 1, TPIPE_BUF_IN = 2, TPIPE_BUF_MSG = 3,
    TPIPE_BUF_GIN = 4, TPIPE_BUF_RBUF = 5, TPIPE_BUF_WS = 6, TPIPE_BUF_STATIC = 7
};

typedef struct {
    int32_t role;        /* TPIPE_BUF_* */
    int32_t category;    /* TPIPE_CAT_* */
    int32_t chunk, mb;   /* owner (chunk, micro-batch); for MSG: channel, msg index */
    uint64_t bytes;      /* requested bytes (the ledger counts exactly these) */
} tpipe_buf;

typedef struct {
    uint64_t peak[TPIPE_CAT_COUNT];  /* per-category maxima */
    uint64_t total_peak;             /* maximum simultaneous live bytes */
    uint64_t static_bytes;           /* model state + io, live the whole step */
} tpipe_mem_report;

typedef struct {
    int32_t n_stages, n_microbatches, v, strategy, delay_rounds, send_window, offload;
    int32_t act_distance;
    int32_t layers_chunk[2];
    int32_t n_channels;
    uint64_t params_total;
    int32_t recomp_layers;   /* effective r of partial T-Recomp (0 unless T-Recomp) */
    double est_step_s;       /* cost-model step time (seconds, see tpipe_plan_opts) */
    double est_exposed_offload_s;   /* of which: offload transfer time left exposed */
    int32_t balanced;        /* 1 if the planner chose a cost-balanced partition */
    int32_t dp;              /* data-parallel replicas */
} tpipe_plan_info;

typedef struct {
    int64_t makespan;      /* unit-time model: F=1, B=2, R=1 (v=2); F=2, B=4(+recompute) (v=1) */
    int64_t busy[64];      /* per-stage busy units (first 64 stages) */
} tpipe_sim_report;

typedef struct tpipe_plan tpipe_plan;

int tpipe_plan_create(const tpipe_model_desc* model, int32_t n_stages, int32_t n_microbatches,
                      uint64_t hbm_budget_bytes, const tpipe_plan_opts* opts, tpipe_plan** out);
void tpipe_plan_destroy(tpipe_plan* plan);
int tpipe_plan_get_info(const tpipe_plan* plan, tpipe_plan_info* out);
int tpipe_plan_stage_ops(const tpipe_plan* plan, int32_t stage, const tpipe_op** ops, size_t* n);
int tpipe_plan_stage_bufs(const tpipe_plan* plan, int32_t stage, const tpipe_buf** bufs, size_t* n);
int tpipe_plan_stage_events(const tpipe_plan* plan, int32_t stage, const int32_t** ids, size_t* n);
int tpipe_plan_stage_peak(const tpipe_plan* plan, int32_t stage, tpipe_mem_report* out);
/* channel c: kind (0 = activations, 1 = activation grads), src stage, dst stage */
int tpipe_plan_channel(const tpipe_plan* plan, int32_t c, int32_t* kind, int32_t* src, int32_t* dst);
/* unit-time ASAP replay of the compute order (mirror of the oracle simulator) */
int tpipe_plan_simulate(const tpipe_plan* plan, tpipe_sim_report* out);
/* The same ASAP replay with given durations: op_ms[s][j] = duration of the
 * j-th compute op (F / B / R, plan order) of stage s, e.g. measured with
 * TPIPE_STEP_OP_TIMES (caller-owned arrays of the stage's compute-op count).
 * Transport time is not modelled. makespan_ms, busy_ms[s] out. */
typedef struct {
    double makespan_ms;
    double busy_ms[64];
} tpipe_sim_report_ms;
int tpipe_plan_simulate_durations(const tpipe_plan* plan, const float* const* op_ms,
                                  tpipe_sim_report_ms* out);
/* layers of (stage, chunk 1) and (stage, chunk 2) (chunk 2 = 0 at v = 1) */
int tpipe_plan_stage_layers(const tpipe_plan* plan, int32_t stage, int32_t out[2]);
/* transformer layers of (stage, chunk), chunk 1..v */
int tpipe_plan_chunk_layers(const tpipe_plan* plan, int32_t stage, int32_t chunk, int32_t* n);
/* parameters of (stage, chunk) in the packed order of DESIGN.md §2.3 */
int tpipe_plan_chunk_params(const tpipe_plan* plan, int32_t stage, int32_t chunk, uint64_t* n);

/* ------------------------------------------------------------------ runtime */
/* Stage transport of a one-stage-per-process runtime (stage >= 0, P:195/P:210
 * pipeline P2P). Both carry the same FIFO channel messages with the
 * plan's send window; see paper_2503_03182_b200/csrc/runtime/transport.h. */
#define TPIPE_TRANSPORT_NCCL 0   /* ncclSend / ncclRecv, one 2-rank communicator per channel */
#define TPIPE_TRANSPORT_IPC  1   /* CUDA IPC: copy-engine pull from the sender's pool arena,
                                    interprocess events, POSIX-shm mailbox (`ipc_name`); works
                                    across GPUs (NVLink peer access) and for several ranks on
                                    one GPU (tests) */
#define TPIPE_TRANSPORT_NCCL_LOOPBACK 2   /* stage = -1 only: the in-process virtual pipeline
                                    with every message moved by an ncclSend / ncclRecv pair on a
                                    one-rank communicator (rank 0 to itself) — runs the NCCL
                                    library path on one GPU, where NCCL refuses two ranks per
                                    device (profiles/r2_nccl_samegpu_refused.txt); tests */

/* debug_flags */
#define TPIPE_DEBUG_POOL_CANARY 1u  /* guard bytes after every pool allocation, checked after
                                       each instruction: a kernel writing past a buffer's
                                       planned bytes fails the step with TPIPE_E_STATE (slow) */
#define TPIPE_DEBUG_POOL_CANARY_SELFTEST 2u  /* with POOL_CANARY: the first instruction that
                                       allocates writes one byte past its first buffer (proves
                                       the check fires; tests only) */

typedef struct {
    int32_t stage;          /* stage executed by this process; -1 = all stages in-process
                               (virtual pipeline on one GPU, device-local transport) */
    int32_t device;         /* CUDA device ordinal */
    const void* nccl_ids;   /* n_channels x 128-byte ncclUniqueId (NCCL transport, stage >= 0,
                               n_stages > 1) */
    uint64_t pool_cap;      /* hard cap of the HBM pool in bytes; 0 = plan peak of owned stages */
    float lr, beta1, beta2, eps, weight_decay;   /* AdamW (DESIGN R16); 0 -> defaults */
    int32_t transport;      /* TPIPE_TRANSPORT_* (stage >= 0, n_stages > 1) */
    int32_t timeout_ms;     /* bound on every transport wait and on the step's completion
                               (TPIPE_E_TIMEOUT; NCCL asynchronous errors are polled meanwhile);
                               0 = 300000 */
    const char* ipc_name;   /* IPC transport: POSIX shm name ("/..."), the same string on the
                               n_stages ranks of one job and unique per job; unlinked once
                               every rank has attached */
    uint32_t debug_flags;   /* TPIPE_DEBUG_* */
    int32_t dp_rank;        /* plan dp > 1: this process's replica (0 .. dp-1); requires
                               stage >= 0 and ipc_name (the replicas of a stage map each
                               other's gradients and weights through CUDA IPC; the pipeline
                               transport of replica k uses ipc_name + "_r<k>") */
} tpipe_runtime_opts;

typedef struct {
    uint64_t pool_high_water[64];   /* ledger high-water per stage (bytes, exact) */
    uint64_t pool_reserved;         /* physical bytes reserved by the pool */
    int64_t  kernel_launches;       /* kernels launched by the last step */
    int64_t  step;                  /* completed steps */
    double   offload_d2h_bytes, offload_h2d_bytes;   /* last step */
    double   host_opt_ms;           /* last host optimizer duration */
    /* TPIPE_STEP_PROFILE only: per kernel class (0 GEMM, 1 attention fwd,
     * 2 attention bwd, 3 other), summed CUDA-event durations of the launches in the
     * last step (ms), launch counts and algorithmic FLOPs (2MNK for GEMMs,
     * causal-triangle counts for attention); class 3 = all other stage
     * kernels (LayerNorm, bias-grad sums, embedding, cross-entropy). */
    double   kernel_ms[4];
    double   kernel_flops[4];
    int64_t  kernel_count[4];
    /* copy-engine time of the last step's offload copies (sum of CUDA-event
     * spans on the D2H / H2D side streams, ms); bytes / ms = host-link GB/s */
    double   offload_d2h_ms, offload_h2d_ms;
    /* physical bytes the pool had to place outside its arena (fragmentation
     * overflow; 0 in a healthy run, TPIPE_E_OOM if it would exceed pool_cap) */
    uint64_t pool_overflow_bytes;
    int32_t  transport;             /* -1 virtual, else TPIPE_TRANSPORT_* in use */
    double   host_issue_ms;         /* last step: host time to issue all its work (before the
                                       final wait); near the step time = submission-bound */
} tpipe_runtime_stats;

typedef struct tpipe_runtime tpipe_runtime;

#define TPIPE_STEP_NO_OPT 1u        /* skip optimizer ops: gradients stay accumulated */
#define TPIPE_STEP_PROFILE 2u       /* bracket GEMM / attention launches with CUDA events */
#define TPIPE_STEP_OP_TIMES 4u      /* record each compute op's (F / B / R) duration with CUDA
                                       events on the stage stream (tpipe_runtime_op_times) */
#define TPIPE_STEP_GRAPH 8u         /* run the step's device work as one CUDA graph: the first
                                       step with this flag (and a given NO_OPT setting) captures
                                       the instruction stream's launches, events and copies,
                                       later steps replay it; AdamW reads its per-step
                                       hyper-parameters from device memory. Same kernels, same
                                       order, same results. Needs an in-process (virtual)
                                       transport, no T-Offload, no DP, no debug pool canaries
                                       (else TPIPE_E_INVALID); ignored with PROFILE / OP_TIMES */

int tpipe_runtime_create(const tpipe_plan* plan, const tpipe_runtime_opts* opts,
                         tpipe_runtime** out);
void tpipe_runtime_destroy(tpipe_runtime* rt);
/* fp32 parameters of (stage, chunk), packed order, n values */
int tpipe_runtime_set_params(tpipe_runtime* rt, int32_t stage, int32_t chunk, const float* src,
                             uint64_t n);
int tpipe_runtime_get_params(tpipe_runtime* rt, int32_t stage, int32_t chunk, float* dst,
                             uint64_t n);
int tpipe_runtime_get_grads(tpipe_runtime* rt, int32_t stage, int32_t chunk, float* dst,
                            uint64_t n);
/* One training step. tokens/targets: int32 [m, b, s]; HOST pointers for
 * tpipe_step (copied in by the runtime), DEVICE pointers for tpipe_step_device.
 * loss_out (host) receives the mean token cross-entropy of the step (read on
 * the last stage; 0 elsewhere). Synchronous. */
int tpipe_step(tpipe_runtime* rt, const int32_t* tokens, const int32_t* targets, uint32_t flags,
               float* loss_out);
int tpipe_step_device(tpipe_runtime* rt, const int32_t* tokens_dev, const int32_t* targets_dev,
                      uint32_t flags, float* loss_out);
int tpipe_runtime_get_stats(const tpipe_runtime* rt, tpipe_runtime_stats* out);

/* Durations (ms) of stage `stage`'s compute ops (F, B, R only, in the plan's
 * order) from the last tpipe_step run with TPIPE_STEP_OP_TIMES; *n = count
 * (0 if the last step did not record), at most `cap` written to `ms`
 * (caller-owned, may be NULL to query n). In the virtual pipeline (stage -1)
 * the ops of all stages run one after another on one GPU, so each duration is
 * the op's own GPU time. */
int tpipe_runtime_op_times(const tpipe_runtime* rt, int32_t stage, float* ms, size_t cap, size_t* n);
/* CUDA stream the runtime launches compute on (cudaStream_t), for event timing */
void* tpipe_runtime_stream(const tpipe_runtime* rt);

/* Run each layer backward's weight-gradient GEMMs (and the LayerNorm
 * recomputes feeding them) on a side stream concurrent with the data-gradient
 * chain (1, default) or everything on the compute stream (0). Process-wide;
 * results are bit-identical either way (every output has one writer and the
 * fp32 accumulations keep their order); forced off while TPIPE_STEP_PROFILE
 * times kernel classes. */
void tpipe_set_side_stream(int on);

/* Launch the bf16 hot-path kernels (tcgen05 GEMMs and attention, LayerNorm,
 * column sums) with programmatic dependent launch (1, default; env TPIPE_PDL=0
 * starts with 0): a kernel's prologue overlaps its predecessor's drain and it
 * waits (griddepcontrol.wait) before touching global memory, so results are
 * bit-identical either way. Process-wide. */
void tpipe_set_pdl(int on);

/* 128-byte ncclUniqueId (for stage >= 0 runtimes); TPIPE_E_NCCL if NCCL absent */
int tpipe_nccl_unique_id(void* out128);

const char* tpipe_last_error(void);
int tpipe_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TPIPE_H */
