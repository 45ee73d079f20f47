// Internal representation of an immutable TPipe plan (see include/tpipe.h).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "tpipe.h"

struct tpipe_plan {
    tpipe_model_desc model{};
    int p = 0, m = 0, v = 0;
    int strategy = 0, k = 0, W = 2, offload = 0, act_distance = 2;
    int layers[4] = {0, 0, 0, 0};   // per-stage chunk layers (uniform partition)
    int rl = 0;   // partial T-Recomp: chunk-1 layers recomputed (R25); 0 unless T-Recomp
    // per-stage (chunk-1, chunk-2) layers (R27; all equal to `layers` unless a
    // stage_layers partition was requested)
    std::vector<std::array<int, 4>> sl;
    int rl_of(int s) const { return rl < sl[s][0] ? rl : sl[s][0]; }
    uint64_t params_total = 0;
    uint64_t hbm_budget = 0;   // per-stage budget the plan was fitted to (0 = none)
    double est_step_s = 0, est_exposed_s = 0;   // cost model (DESIGN R28)
    bool balanced = false;     // cost-balanced partition chosen by the planner
    int dp = 1;                // data-parallel replicas (ZeRO-1, R31)
    // per stage
    std::vector<std::vector<tpipe_op>> ops;
    std::vector<std::vector<tpipe_buf>> bufs;
    std::vector<std::vector<int32_t>> events;
    std::vector<tpipe_mem_report> peak;
    std::vector<std::array<uint64_t, 4>> chunk_params;
    // compute order (F/B/R only) per stage: {kind, chunk, mb}
    std::vector<std::vector<std::array<int, 3>>> order;
    // channels: {kind (0 act, 1 grad), src, dst}
    std::vector<std::array<int, 3>> channels;
};

namespace tpipe {

// byte model of one (stage, chunk)
struct ChunkSizes {
    uint64_t act = 0, stash = 0, ws_f = 0, ws_b = 0;
    bool input_is_act = true, has_output = true;
};

int delay_rounds_appB(int p);
uint64_t layer_params(const tpipe_model_desc& d);
// ZeRO-1 shard (R31): ceil(P / dp) rounded up to 64 parameters
uint64_t zero1_shard(uint64_t P, int dp);
uint64_t chunk_params(const tpipe_model_desc& d, int p, int v, const int* layers, int s, int c);

}  // namespace tpipe
