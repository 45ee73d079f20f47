"""Multi-process pipeline: one process per stage (tpipe_runtime_create with
stage = s), all on cuda:0, stages connected by the CUDA-IPC transport
(TPIPE_TRANSPORT_IPC: copy-engine pulls from the peer's pool arena,
interprocess events, a POSIX-shm mailbox). This runs the runtime's
one-stage-per-rank path — SEND / RECV / SEND_WAIT through a real
inter-process transport, per-rank pools and ledgers, the host optimizer
thread with p > 1 Eq. 5/7 windows — and checks it against the
fp64 oracle (fp32: max-rel <= 1e-4) and bit for bit against the in-process
virtual pipeline (same kernels; R21).

Stage-to-stage P2P of the pipeline: P:195. p = 8 with L = 16 gives
T-Recomp delay rounds k = 1 (App. B; SURVEY D-3).
"""

import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import model as R  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mp_stage_worker.py")
C1 = dict(L=8, h=64, a=4, f=256, V=256, s=32, b=2)
C1_16 = dict(C1, L=16)     # C1 width, 16 layers: p = 8 with two chunks of one layer


def run_job(tmp_path, cfg, p, m, strategy, dtype, steps=1, offload=0, timeout_ms=120000,
            stages=None, wall=600, dp=1, tag="", chunks=2):
    """Launch one process per (replica, stage); results keyed by stage (dp = 1)
    or by (replica, stage)."""
    name = f"/tpipe_t_{os.getpid()}_{uuid.uuid4().hex[:12]}"
    procs = []
    for k in range(dp):
        for s in (range(p) if stages is None else stages):
            key = s if dp == 1 else (k, s)
            out = str(tmp_path / f"{tag}r{k}_stage{s}.npz")
            args = [sys.executable, WORKER, out, str(s), str(p), str(m), strategy, str(dtype), name,
                    *(str(cfg[kk]) for kk in ("L", "h", "a", "f", "V", "s", "b")), str(steps),
                    str(offload), str(timeout_ms), "11", str(dp), str(k), str(chunks)]
            procs.append((key, out, subprocess.Popen(args, stdout=subprocess.PIPE,
                                                     stderr=subprocess.STDOUT, cwd=ROOT)))
    res, logs = {}, {}
    for s, out, pr in procs:
        try:
            o, _ = pr.communicate(timeout=wall)
        except subprocess.TimeoutExpired:
            for _, _, q in procs:
                q.kill()
            raise
        logs[s] = (pr.returncode, o.decode(errors="replace"))
        if pr.returncode == 0:
            res[s] = dict(np.load(out))
    return res, logs


def assert_ok(res, logs):
    bad = {s: l for s, l in logs.items() if l[0] != 0}
    assert not bad, "\n".join(f"stage {s} rc={rc}:\n{o[-3000:]}" for s, (rc, o) in bad.items())


def max_rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / (np.abs(b).max() + 1e-30))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


def _plan(cfg, p, m, strategy, dtype, offload=0, chunks=2):
    from paper_2503_03182_b200 import plan as P
    return P.Plan(P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], dtype),
                  p, m, strategy=strategy, offload=offload, chunks=chunks)


def check_vs_oracle(cfg, p, m, strategy, dtype, res, tol, metric):
    from paper_2503_03182_b200 import params as PR
    plan = _plan(cfg, p, m, strategy, dtype)
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    assert abs(float(res[p - 1]["loss0"]) - lref) / abs(lref) < tol
    worst = 0.0
    for s in range(p):
        assert int(res[s]["transport"]) == 1          # ran over the IPC transport
        assert int(res[s]["launches"]) > 0
        assert int(res[s]["high_water"]) == int(res[s]["plan_peak"])   # per-rank ledger
        for c in range(1, plan.v + 1):
            got = PR.unpack(res[s][f"grad{c}"], W, p, plan.v, plan.partition, s, c)
            for (k, l), g in got.items():
                ref = G["layers"][l][k] if l is not None else G[k]
                err = metric(g, ref)
                worst = max(worst, err)
                assert err <= tol, (s, c, k, l, err)
    return worst


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "interleave_trecomp"])
@pytest.mark.parametrize("p", [2, 4])
def test_multiprocess_fp32_parity(tmp_path, p, strategy):
    res, logs = run_job(tmp_path, C1, p, 8, strategy, 0)
    assert_ok(res, logs)
    check_vs_oracle(C1, p, 8, strategy, 0, res, 1e-4, max_rel)


@pytest.mark.parametrize("strategy,offload", [("tpipe_trecomp", 0), ("tpipe", 1), ("interleave", 0)])
def test_multiprocess_p8_fp32_parity(tmp_path, strategy, offload):
    """p = 8 (k = 1 delay round for T-Recomp), 8 processes."""
    if strategy == "tpipe_trecomp":
        assert _plan(C1_16, 8, 16, strategy, 0).k == 1
    res, logs = run_job(tmp_path, C1_16, 8, 16, strategy, 0, offload=offload)
    assert_ok(res, logs)
    check_vs_oracle(C1_16, 8, 16, strategy, 0, res, 1e-4, max_rel)


def _virtual(cfg, p, m, strategy, dtype, steps, offload=0, transport=None):
    from paper_2503_03182_b200 import params as PR, runtime as RT
    plan = _plan(cfg, p, m, strategy, dtype, offload)
    rt = RT.Runtime(plan, stage=-1, lr=1e-3, **({} if transport is None else {"transport": transport}))
    if transport is not None:
        assert rt.stats()["transport"] == transport
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    for s in range(p):
        for c in range(1, plan.v + 1):
            rt.set_params(s, c, PR.pack(W, p, plan.v, plan.partition, s, c))
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
    loss0 = rt.step(tok, tgt, RT.STEP_NO_OPT)
    grads = {(s, c): rt.get_grads(s, c) for s in range(p) for c in range(1, plan.v + 1)}
    for s in range(p):
        for c in range(1, plan.v + 1):
            rt.set_params(s, c, PR.pack(W, p, plan.v, plan.partition, s, c))
    losses = []
    for k in range(steps):
        tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=k)
        losses.append(rt.step(tok, tgt, 0))
    params = {(s, c): rt.get_params(s, c) for s in range(p) for c in range(1, plan.v + 1)}
    rt.close()
    return loss0, grads, losses, params


@pytest.mark.parametrize("p,strategy,offload,cfg,m", [
    (4, "tpipe_trecomp", 0, C1, 8),
    (4, "tpipe_trecomp", 1, C1, 8),       # host AdamW of chunk 2 with p > 1 windows
    (8, "tpipe_trecomp", 5, C1_16, 16),   # streamed device AdamW, k = 1
])
def test_multiprocess_bf16_bitexact_vs_virtual(tmp_path, p, strategy, offload, cfg, m):
    """bf16, 2 optimizer steps: the multi-process run reproduces the virtual
    pipeline bit for bit (loss, gradients, updated parameters)."""
    res, logs = run_job(tmp_path, cfg, p, m, strategy, 1, steps=2, offload=offload)
    assert_ok(res, logs)
    loss0, grads, losses, params = _virtual(cfg, p, m, strategy, 1, 2, offload)
    assert float(res[p - 1]["loss0"]) == loss0
    assert list(res[p - 1]["losses"]) == losses
    for (s, c), g in grads.items():
        assert np.array_equal(res[s][f"grad{c}"].view(np.uint32), g.view(np.uint32)), (s, c)
    for (s, c), w in params.items():
        assert np.array_equal(res[s][f"param{c}"].view(np.uint32), w.view(np.uint32)), (s, c)


def test_multiprocess_missing_peer_times_out(tmp_path):
    """A rank whose peer never arrives fails with TPIPE_E_TIMEOUT instead of hanging."""
    res, logs = run_job(tmp_path, C1, 2, 8, "tpipe", 0, timeout_ms=3000, stages=[0], wall=120)
    rc, out = logs[0]
    assert rc != 0
    assert "timed out" in out and "rc=-11" in out


def _assemble(res, p, dp, plan, key):
    """Per stage and chunk, the replicas' arrays in replica order."""
    return {(s, c): [res[(k, s)][f"{key}{c}"] for k in range(dp)]
            for s in range(p) for c in range(1, plan.v + 1)}


@pytest.mark.parametrize("p,dp,strategy", [(1, 2, "tpipe"), (2, 2, "tpipe_trecomp"), (2, 4, "tpipe"),
                                           (4, 2, "1f1b")])
def test_dp_pp_zero1_fp32(tmp_path, p, dp, strategy):
    """DP x PP with ZeRO-1 (NEXT-3; DESIGN R31), dp*p processes on one GPU:
    * the replicas' summed gradients equal the oracle's full-batch gradients over
      all dp*m micro-batches (max-rel <= 1e-4), the summed loss its loss;
    * after two optimizer steps every replica holds the same weights, and they
      match the single-replica virtual pipeline run on the dp*m micro-batches
      (same AdamW; only the fp32 gradient summation order differs);
    * each rank's pool high-water equals its plan peak (optimizer states of one
      shard)."""
    from paper_2503_03182_b200 import params as PR
    cfg, m = C1, 4
    res, logs = run_job(tmp_path, cfg, p, m, strategy, 0, steps=2, dp=dp)
    assert_ok(res, logs)
    plan = _plan(cfg, p, m, strategy, 0)
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    tok, tgt = synth.tokens(cfg["V"], dp * m, cfg["b"], cfg["s"], step=0)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    loss = sum(float(res[(k, p - 1)]["loss0"]) for k in range(dp))
    assert abs(loss - lref) / abs(lref) < 1e-5
    grads = _assemble(res, p, dp, plan, "grad")
    for (s, c), gs in grads.items():
        got = PR.unpack(np.sum(gs, axis=0), W, p, plan.v, plan.partition, s, c)
        for (k, l), g in got.items():
            ref = G["layers"][l][k] if l is not None else G[k]
            assert max_rel(g, ref) <= 1e-4, (s, c, k, l)
    for k in range(dp):
        for s in range(p):
            assert int(res[(k, s)]["high_water"]) == int(res[(k, s)]["plan_peak"])
    # reference: one replica over all dp*m micro-batches (virtual pipeline)
    _l0, _g, _losses, vparams = _virtual(cfg, p, dp * m, strategy, 0, 2)
    params = _assemble(res, p, dp, plan, "param")
    for (s, c), ps in params.items():
        for k in range(1, dp):
            assert np.array_equal(ps[0], ps[k]), (s, c, k)       # all-gather: identical replicas
        ref = vparams[(s, c)]
        bad = np.abs(ps[0] - ref) > 1e-6 + 1e-5 * np.abs(ref)
        assert bad.mean() < 1e-3, (s, c, int(bad.sum()))


def test_dp_pp_zero1_bf16_deterministic(tmp_path):
    """bf16, p = 2 x dp = 2: two identical jobs give bit-identical losses and
    parameters, replicas agree bit for bit, and the bf16 weights are the RNE
    of the owning replica's fp32 master."""
    cfg, p, dp, m = C1, 2, 2, 4
    runs = []
    for t in ("a", "b"):
        res, logs = run_job(tmp_path, cfg, p, m, "tpipe", 1, steps=2, dp=dp, tag=t)
        assert_ok(res, logs)
        runs.append(res)
    plan = _plan(cfg, p, m, "tpipe", 1)
    for key in ("param", "grad"):
        A = _assemble(runs[0], p, dp, plan, key)
        B = _assemble(runs[1], p, dp, plan, key)
        for sc in A:
            for x, y in zip(A[sc], B[sc]):
                assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), (key, sc)
    for k in range(dp):
        assert list(runs[0][(k, p - 1)]["losses"]) == list(runs[1][(k, p - 1)]["losses"])
    # replicas agree on the bf16 weights (upper 16 bits) everywhere
    P_ = _assemble(runs[0], p, dp, plan, "param")
    for sc, ps in P_.items():
        hi = [(x.view(np.uint32) + 0x7FFF + ((x.view(np.uint32) >> 16) & 1)) >> 16 for x in ps]
        for k in range(1, dp):
            assert np.array_equal(hi[0], hi[k]), sc


def test_multiprocess_v3_dp2_fp32(tmp_path):
    """Three chunks per stage (R32) with two ZeRO-1 replicas (R31), p = 2:
    4 processes; the replicas' summed gradients equal the oracle's full-batch
    gradients, replicas hold identical parameters after two steps."""
    from paper_2503_03182_b200 import params as PR
    cfg, p, dp, m, v = dict(C1, L=12), 2, 2, 4, 3
    res, logs = run_job(tmp_path, cfg, p, m, "tpipe_trecomp", 0, steps=2, dp=dp, chunks=v)
    assert_ok(res, logs)
    plan = _plan(cfg, p, m, "tpipe_trecomp", 0, chunks=v)
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    tok, tgt = synth.tokens(cfg["V"], dp * m, cfg["b"], cfg["s"], step=0)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    for s in range(p):
        for c in range(1, v + 1):
            g = np.sum([res[(k, s)][f"grad{c}"] for k in range(dp)], axis=0)
            for (kk, l), gg in PR.unpack(g, W, p, v, plan.partition, s, c).items():
                ref = G["layers"][l][kk] if l is not None else G[kk]
                assert max_rel(gg, ref) <= 1e-4, (s, c, kk, l)
            assert np.array_equal(res[(0, s)][f"param{c}"], res[(1, s)][f"param{c}"])


@pytest.mark.parametrize("p,strategy,offload,cfg,m", [
    (4, "interleave_trecomp", 0, C1, 8),
    (8, "tpipe_trecomp", 5, C1_16, 16),
])
def test_nccl_loopback_bitexact_vs_virtual(p, strategy, offload, cfg, m):
    """NCCL refuses two ranks on one GPU (profiles/r2_nccl_samegpu_refused.txt),
    so the NCCL library path runs here as a loopback: every stage-to-stage
    message of the virtual pipeline is an ncclSend / ncclRecv pair on a
    one-rank communicator (TPIPE_TRANSPORT_NCCL_LOOPBACK), with the step's
    completion polling ncclCommGetAsyncError. bf16, 2 optimizer steps:
    bit-identical to the device-copy virtual pipeline."""
    from paper_2503_03182_b200 import runtime as RT
    ref = _virtual(cfg, p, m, strategy, 1, 2, offload)
    got = _virtual(cfg, p, m, strategy, 1, 2, offload, transport=RT.TRANSPORT_NCCL_LOOPBACK)
    assert got[0] == ref[0] and got[2] == ref[2]
    for part in (1, 3):
        for k, v in ref[part].items():
            assert np.array_equal(got[part][k].view(np.uint32), v.view(np.uint32)), k
