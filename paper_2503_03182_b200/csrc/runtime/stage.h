// Per-chunk forward / recompute / backward of the pre-LN GPT block stack
// over the sm_100a kernels.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "kernels/kernels.h"
#include "tpipe.h"

namespace tpipe {

// Packed parameter order of one chunk, offsets in elements.
enum LayerTensor {
    LN1_G = 0, LN1_B, W_QKV, B_QKV, W_O, B_O, LN2_G, LN2_B, W_1, B_1, W_2, B_2, N_LAYER_TENSORS
};

struct ParamLayout {
    bool emb = false, head = false;
    long wte = -1, wpe = -1, lnf_g = -1, lnf_b = -1, w_head = -1;
    std::vector<std::array<long, N_LAYER_TENSORS>> layer;
    long total = 0;
    // (offset, size, decay) segments for AdamW (decay on 2-D tensors)
    std::vector<std::array<long, 3>> segments;
};

ParamLayout make_param_layout(const tpipe_model_desc& d, int n_layers, bool emb, bool head);

// Byte offsets of the saved tensors inside one chunk's stash.
struct StashLayout {
    struct L {
        long x_in, ln1_mean, ln1_rstd, qkv, o, lse, x_mid, ln2_mean, ln2_rstd, u;
    };
    std::vector<L> layer;   // x_in == -1 for layer 0 when the chunk input is the IN buffer
    long x_f = -1, lnf_mean = -1, lnf_rstd = -1, ce_lse = -1;
    long total = 0;
    // 1F1B + full recompute: the stash keeps only layer inputs (checkpoints);
    // one layer's internals live in a scratch (offsets relative to its base)
    bool ckpt_only = false;
    int ckpt_layers = 0;    // layers [0, ckpt_layers) are checkpoint-only (recomputed in B)
    L scratch{};
    long scratch_bytes = 0;
};

// ckpt_only: 1F1B + layer-grouped recompute; ckpt_layers = how many of the
// shallowest layers are checkpoint-only (0 = all of them)
StashLayout make_stash_layout(const tpipe_model_desc& d, int n_layers, bool emb, bool head,
                              bool ckpt_only = false, int ckpt_layers = 0);

struct Dims {
    int dtype, M, h, a, hd, f, V, s, b, es;
    Dims(const tpipe_model_desc& d);
};

// Device views of one chunk's parameters (es) and fp32 gradients.
struct ChunkParamsDev {
    const ParamLayout* lay;
    void* w;       // es
    float* grad;   // fp32
};

struct FwdArgs {
    const void* in;          // chunk input (IN buffer) or nullptr for the embedding chunk
    const int* tokens;       // [M] (embedding chunk)
    const int* targets;      // [M] (head chunk)
    float* loss_slot;        // unused: the head chunk's loss is computed in its backward
    float loss_scale;
    uint8_t* stash;          // STASH / TSTASH / RBUF
    uint8_t* ws;             // forward workspace (ws_f bytes)
    void* out;               // chunk output [M,h] (nullptr: head chunk, or recompute -> scratch)
    // partial T-Recomp (DESIGN R25): layers [0, split) live in `stash`
    // (TSTASH / RBUF), layers [split, n) in `stash2` (the kept STASH); split 0 =
    // every layer in `stash`. n_run > 0: run only layers [0, n_run) (R op).
    uint8_t* stash2;
    int split, n_run;
};

struct BwdArgs {
    const void* in;          // chunk input (layer-0 x_in) or nullptr (embedding chunk)
    const int* tokens;
    const int* targets;
    float* loss_slot;        // head chunk: += scale * sum CE (computed with the logits in B)
    float loss_scale;
    uint8_t* stash;
    uint8_t* stash2;         // partial T-Recomp: kept stash of layers [split, n)
    int split;               // 0 = every layer in `stash`
    uint8_t* ws;             // backward workspace (ws_b bytes)
    const void* gin;         // d(chunk output) [M,h]; nullptr for the head chunk
    void* gout;              // d(chunk input) [M,h]; nullptr for the embedding chunk
};

// Per-kernel-class CUDA-event profiler (TPIPE_STEP_PROFILE): classes
// 0 GEMM, 1 attention fwd, 2 attention bwd.
struct KernelProfiler {
    bool on = false;
    struct Rec {
        cudaEvent_t a, b;
        int cls;
        double flops;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t next = 0;
    cudaEvent_t ev();
    void begin_step(bool enable) { on = enable; recs.clear(); next = 0; }
    // after the stream is synchronised
    void collect(double ms[4], double flops[4], int64_t count[4]);
    ~KernelProfiler();
};
KernelProfiler& profiler();

// workspace bytes chunk_forward / chunk_backward carve (must equal the plan's
// ws_f / ws_b: tpipe_runtime_create checks every (stage, chunk))
uint64_t fwd_ws_bytes(const Dims& D, const StashLayout& SL, bool head);
uint64_t bwd_ws_bytes(const Dims& D, const StashLayout& SL, bool head, bool emb);

int chunk_forward(const Dims& D, const StashLayout& SL, const ChunkParamsDev& P, const FwdArgs& a,
                  cudaStream_t st);
// layer backward: run weight-gradient GEMMs on a side stream (default on;
// always off while TPIPE_STEP_PROFILE is timing kernel classes)
void stage_set_side_stream(int on);
// release the side stream + events cached for `main` on the current device
void stage_release_side_streams(cudaStream_t main);
int chunk_backward(const Dims& D, const StashLayout& SL, const ChunkParamsDev& P, const BwdArgs& a,
                   cudaStream_t st);

}  // namespace tpipe
