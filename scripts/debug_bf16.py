"""Diagnostics for the bf16 step: per-tensor gradient error vs the oracle and
placement sensitivity (offload on/off changes the pool layout)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from oracle import model as R
from paper_2503_03182_b200 import plan as P, runtime as RT, params as PR, kernels as K

C1 = dict(n_layers=8, hidden=64, n_heads=4, ffn_hidden=256, vocab=256, seq_len=32, micro_batch=2)


def build(p, m, strategy, dtype, offload=0):
    md = P.Model(8, 64, 4, 256, 256, 32, 2, dtype)
    pl = P.Plan(md, p, m, strategy=strategy, offload=offload)
    rt = RT.Runtime(pl, stage=-1, lr=1e-3)
    W = synth.weights(8, 64, 256, 256, 32, seed=11, std=0.05, bias_std=0.02, ln_jitter=0.05)
    for s in range(p):
        for c in range(1, pl.v + 1):
            rt.set_params(s, c, PR.pack(W, p, pl.v, pl.layers_chunk, s, c))
    return pl, rt, W


tok, tgt = synth.tokens(256, 8, 2, 32, step=0)
for trial in range(3):
    pl, rt, W = build(4, 8, "tpipe", 1, offload=(trial == 2) * 0)
    print("bf16 loss trial", trial, rt.step(tok, tgt, RT.STEP_NO_OPT))
for off in (0, 1):
    pl, rt, W = build(4, 8, "tpipe_trecomp", 1, offload=off)
    print("offload", off, "loss", rt.step(tok, tgt, RT.STEP_NO_OPT))
pl, rt, W = build(1, 8, "tpipe", 1)
print("p1 bf16 loss", rt.step(tok, tgt, RT.STEP_NO_OPT))
lref, G = R.step_grads(R.to64(W), tok, tgt, 4)
print("oracle loss", lref)
pl, rt, W = build(4, 8, "tpipe", 1)
loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
print("p4 bf16 loss", loss)
for s in range(4):
    for c in (1, 2):
        got = PR.unpack(rt.get_grads(s, c), W, 4, 2, pl.layers_chunk, s, c)
        for (k, l), g in got.items():
            ref = G["layers"][l][k] if l is not None else G[k]
            e = np.linalg.norm(g - ref) / (np.linalg.norm(ref) + 1e-30)
            if e > 5e-3:
                print(f"  s{s} c{c} {k} L{l}: relL2 {e:.3e} |ref| {np.linalg.norm(ref):.3e}")

# GEMM shapes of the C1 model with NaN guard bands around every operand
dev = "cuda"
def guarded(shape, dtype, fill):
    n = int(np.prod(shape))
    buf = torch.full((n + 4096,), float("nan"), device=dev, dtype=dtype)
    v = buf[2048:2048 + n].view(*shape)
    v.copy_(fill)
    return buf, v
M, h, f, V = 64, 64, 256, 256
cases = [("qkv", M, 3*h, h, 1, 1), ("o", M, h, h, 1, 1), ("fc1", M, f, h, 1, 1), ("fc2", M, h, f, 1, 1),
         ("head", M, V, h, 1, 1), ("fc2_dgrad", M, f, h, 1, 0), ("fc1_dgrad", M, h, f, 1, 0),
         ("qkv_dgrad", M, h, 3*h, 1, 0), ("head_dgrad", M, h, V, 1, 0),
         ("fc2_wgrad", h, f, M, 0, 0), ("fc1_wgrad", f, h, M, 0, 0), ("qkv_wgrad", 3*h, h, M, 0, 0),
         ("head_wgrad", V, h, M, 0, 0), ("o_wgrad", h, h, M, 0, 0)]
for name, Mm, N, Kk, ak, bk in cases:
    A0 = torch.randn((Mm, Kk) if ak else (Kk, Mm), device=dev)
    B0 = torch.randn((N, Kk) if bk else (Kk, N), device=dev)
    _, A = guarded(A0.shape, torch.bfloat16, A0)
    _, B = guarded(B0.shape, torch.bfloat16, B0)
    _, C = guarded((Mm, N), torch.float32, torch.zeros(Mm, N, device=dev))
    K.tpipe_k_gemm(1, Mm, N, Kk, A, Kk if ak else Mm, ak, B, Kk if bk else N, bk, K.EPI_STORE_F32, C, N)
    torch.cuda.synchronize()
    Af = A.float() if ak else A.float().T
    Bf = B.float() if bk else B.float().T
    ref = Af @ Bf.T
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    print(f"gemm {name:10s} M={Mm} N={N} K={Kk} majors={ak}{bk} err={err:.2e} nan={torch.isnan(C).any().item()}")
