"""One pipeline stage in its own process (tpipe_runtime_create(stage=s)),
driven by tests/test_gpu_multirank.py: every stage of a p-stage job is a
separate process, all on cuda:0, talking over the CUDA-IPC transport
(TPIPE_TRANSPORT_IPC) — the same SEND / RECV / SEND_WAIT code, pool
lifetimes and events as a one-GPU-per-stage job.

Writes the stage's loss, gradients (after step 1, no optimizer) and
parameters (after `steps` optimizer steps) to an .npz file.

    python tests/mp_stage_worker.py OUT.npz STAGE P M STRATEGY DTYPE IPC_NAME
        L H A F V S B [STEPS] [OFFLOAD] [TIMEOUT_MS] [SEED] [DP] [DP_RANK] [CHUNKS]

With DP > 1 (ZeRO-1 data parallelism, DESIGN R31) replica k runs
micro-batches [k*M, (k+1)*M) of a DP*M-micro-batch step.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(argv):
    out, stage, p, m, strategy, dtype, ipc = argv[:7]
    stage, p, m, dtype = int(stage), int(p), int(m), int(dtype)
    L, h, a, f, V, s, b = (int(x) for x in argv[7:14])
    steps = int(argv[14]) if len(argv) > 14 else 1
    offload = int(argv[15]) if len(argv) > 15 else 0
    timeout_ms = int(argv[16]) if len(argv) > 16 else 120000
    seed = int(argv[17]) if len(argv) > 17 else 11
    dp = int(argv[18]) if len(argv) > 18 else 1
    dp_rank = int(argv[19]) if len(argv) > 19 else 0
    chunks = int(argv[20]) if len(argv) > 20 else 2
    import synth
    from paper_2503_03182_b200 import params as PR, plan as P, runtime as RT

    plan = P.Plan(P.Model(L, h, a, f, V, s, b, dtype), p, m, strategy=strategy, offload=offload, dp=dp,
                  chunks=chunks)
    rt = RT.Runtime(plan, stage=stage, device=0, lr=1e-3, transport=RT.TRANSPORT_IPC,
                    ipc_name=ipc, timeout_ms=timeout_ms, dp_rank=dp_rank)

    def batch(step):
        tok, tgt = synth.tokens(V, dp * m, b, s, step=step)
        return tok[dp_rank * m:(dp_rank + 1) * m], tgt[dp_rank * m:(dp_rank + 1) * m]
    W = synth.weights(L, h, f, V, s, seed=seed, std=0.05, bias_std=0.02, ln_jitter=0.05)
    for c in range(1, plan.v + 1):
        rt.set_params(stage, c, PR.pack(W, p, plan.v, plan.partition, stage, c))
    res = {}
    tok, tgt = batch(0)
    res["loss0"] = np.float64(rt.step(tok, tgt, RT.STEP_NO_OPT))
    for c in range(1, plan.v + 1):
        res[f"grad{c}"] = rt.get_grads(stage, c)
    st = rt.stats()
    res["high_water"] = np.uint64(st["pool_high_water"][stage])
    res["plan_peak"] = np.uint64(plan.peak(stage)["total_peak"])
    res["transport"] = np.int32(st["transport"])
    res["launches"] = np.int64(st["kernel_launches"])
    # optimizer steps (fresh gradients: re-load the parameters first)
    for c in range(1, plan.v + 1):
        rt.set_params(stage, c, PR.pack(W, p, plan.v, plan.partition, stage, c))
    losses = []
    for k in range(steps):
        tok, tgt = batch(k)
        losses.append(rt.step(tok, tgt, 0))
    res["losses"] = np.array(losses, np.float64)
    for c in range(1, plan.v + 1):
        res[f"param{c}"] = rt.get_params(stage, c)
    rt.close()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1:])
