"""Kernel-level parity: each sm_100a kernel (called through the C-ABI of
include/tpipe_kernels.h) vs the fp64 oracle / definition, element by element.

Tolerances: fp32 mode <= 1e-4 max-relative (per tensor, vs the
tensor's max magnitude); bf16 outputs <= 2e-2 relative L2; fp32-accumulator
outputs of bf16 GEMMs <= 1e-4 (inputs are exact bf16 values).
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import model as R  # noqa: E402

dev = "cuda"


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2503_03182_b200 import lib
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    lib()


def K():
    from paper_2503_03182_b200 import kernels
    return kernels


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


def max_rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-30))


def t(x, dtype):
    tt = torch.tensor(np.asarray(x, np.float32), device=dev)
    return tt.to(torch.bfloat16) if dtype == "bf16" else tt


def h(x):
    return x.float().cpu().numpy().astype(np.float64)


# ------------------------------------------------------------------ GEMM
GEMM_SHAPES = [(256, 512, 256), (296, 192, 320), (64, 64, 64), (2048, 6144, 2048), (136, 96, 200)]


@pytest.mark.parametrize("M,N,Kd", GEMM_SHAPES)
@pytest.mark.parametrize("majors", [(1, 1), (1, 0), (0, 0)])
def test_gemm_bf16_tcgen05(M, N, Kd, majors):
    """tcgen05 GEMM, all operand majors (fprop K/K, dgrad K/MN, wgrad MN/MN),
    fp32-output epilogue: near-exact vs fp64 of the same bf16 inputs."""
    ak, bk = majors
    rng = np.random.default_rng(M + N + Kd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    At = t(A if ak else A.T.copy(), "bf16")
    Bt = t(B if bk else B.T.copy(), "bf16")
    ref = h(At if ak else At.T) @ h(Bt if bk else Bt.T).T
    C = torch.zeros((M, N), device=dev, dtype=torch.float32)
    K().tpipe_k_gemm(1, M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk,
                     K().EPI_STORE_F32, C, N)
    torch.cuda.synchronize()
    assert max_rel(h(C), ref) < 1e-4
    # accumulate epilogue: C += A B^T
    K().tpipe_k_gemm(1, M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk,
                     K().EPI_ACC_F32, C, N)
    torch.cuda.synchronize()
    assert max_rel(h(C), 2 * ref) < 1e-4


@pytest.mark.parametrize("M,N,Kd", [(512, 512, 4160), (296, 320, 4200), (2048, 2048, 2048)])
@pytest.mark.parametrize("majors", [(1, 1), (1, 0), (0, 0)])
def test_gemm_underfilled(M, N, Kd, majors):
    """Shapes whose whole tiles under-fill the SMs (a partial last wave, long
    K): matches fp64 and is bit-identical run to run (fp32 store, fp32
    accumulate, bias and dGELU epilogues)."""
    ak, bk = majors
    k = K()
    rng = np.random.default_rng(M * 7 + Kd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    At = t(A if ak else A.T.copy(), "bf16")
    Bt = t(B if bk else B.T.copy(), "bf16")
    ref = h(At if ak else At.T) @ h(Bt if bk else Bt.T).T
    bias = t(rng.standard_normal(N), "bf16")
    U = t(rng.standard_normal((M, N)), "bf16")
    args = (M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk)

    def run():
        C = torch.zeros((M, N), device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_STORE_F32, C, N)
        Acc = torch.ones((M, N), device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_ACC_F32, Acc, N)
        Cb = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_BIAS, Cb, N, bias=bias)
        Cd = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Cg = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_DGELU, Cd, N, C2=Cg, ldc2=N, aux=U, ldaux=N)
        torch.cuda.synchronize()
        return C, Acc, Cb, Cd
    r1 = run()
    r2 = run()
    for u, v in zip(r1, r2):
        assert torch.equal(u, v)
    C, Acc, Cb, Cd = r1
    assert max_rel(h(C), ref) < 1e-4
    assert max_rel(h(Acc), 1 + ref) < 1e-4
    assert rel_l2(h(Cb), ref + h(bias)) < 1e-2
    assert rel_l2(h(Cd), ref * R.gelu_grad(h(U))) < 1e-2


@pytest.mark.parametrize("M,N,Kd", [(2048, 6144, 2048), (2000, 2080, 4200), (4096, 2816, 520)])
@pytest.mark.parametrize("majors", [(1, 1), (1, 0), (0, 0)])
def test_gemm_cta_pair(M, N, Kd, majors):
    """CTA-pair (cta_group::2, 256 x 256) tiles incl. ragged M/N edges: matches
    fp64 and the single-CTA kernel (pair off) for fp32 store,
    fp32 accumulate and the bf16 dGELU epilogue."""
    ak, bk = majors
    k = K()
    rng = np.random.default_rng(M + 3 * N + Kd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    At = t(A if ak else A.T.copy(), "bf16")
    Bt = t(B if bk else B.T.copy(), "bf16")
    ref = h(At if ak else At.T) @ h(Bt if bk else Bt.T).T
    U = t(rng.standard_normal((M, N)), "bf16")
    args = (M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk)

    def run():
        C = torch.zeros((M, N), device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_STORE_F32, C, N)
        Acc = torch.full((M, N), 2.0, device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_ACC_F32, Acc, N)
        Cd = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Cg = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_DGELU, Cd, N, C2=Cg, ldc2=N, aux=U, ldaux=N)
        torch.cuda.synchronize()
        return C, Acc, Cd, Cg
    pair = run()
    try:
        k.tpipe_k_gemm_set_pair(0)
        single = run()
    finally:
        k.tpipe_k_gemm_set_pair(1)
    C, Acc, Cd, Cg = pair
    assert max_rel(h(C), ref) < 1e-4
    assert max_rel(h(Acc), 2 + ref) < 1e-4
    assert rel_l2(h(Cd), ref * R.gelu_grad(h(U))) < 1e-2
    assert rel_l2(h(Cg), R.gelu(h(U))) < 1e-2
    assert max_rel(h(C), h(single[0])) < 1e-5
    assert max_rel(h(Acc), h(single[1])) < 1e-5


@pytest.mark.parametrize("M,N,Kd", [(2048, 8192, 2048), (8192, 2048, 1024), (2000, 8992, 320),
                                    (2048, 50304, 256)])
@pytest.mark.parametrize("majors", [(1, 1), (1, 0), (0, 0)])
def test_gemm_pair_ragged(M, N, Kd, majors):
    """CTA-pair shapes incl. ragged M / N / K edges and the vocabulary-wide
    N: matches fp64 and is bit-identical run to run for fp32 store, fp32
    accumulate, bias+GELU and dGELU epilogues."""
    ak, bk = majors
    k = K()
    rng = np.random.default_rng(M + 5 * N + Kd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    At = t(A if ak else A.T.copy(), "bf16")
    Bt = t(B if bk else B.T.copy(), "bf16")
    ref = h(At if ak else At.T) @ h(Bt if bk else Bt.T).T
    U = t(rng.standard_normal((M, N)), "bf16")
    bias = t(rng.standard_normal(N), "bf16")
    args = (M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk)

    def run():
        C = torch.zeros((M, N), device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_STORE_F32, C, N)
        Acc = torch.full((M, N), 2.0, device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_ACC_F32, Acc, N)
        Cd = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Cg = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_DGELU, Cd, N, C2=Cg, ldc2=N, aux=U, ldaux=N)
        Cu = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Cgl = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_BIAS_GELU, Cu, N, bias=bias, C2=Cgl, ldc2=N)
        torch.cuda.synchronize()
        return C, Acc, Cd, Cg, Cu, Cgl
    first = run()
    again = run()
    C, Acc, Cd, Cg, Cu, Cgl = first
    assert max_rel(h(C), ref) < 1e-4
    assert max_rel(h(Acc), 2 + ref) < 1e-4
    assert rel_l2(h(Cd), ref * R.gelu_grad(h(U))) < 1e-2
    assert rel_l2(h(Cu), ref + h(bias)) < 1e-2
    for u, v in zip(first, again):
        assert torch.equal(u, v)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_gemm_epilogues(dtype):
    """bias / residual / GELU / dGELU epilogues vs fp64 definitions."""
    dt = 1 if dtype == "bf16" else 0
    M, N, Kd = 192, 320, 128
    rng = np.random.default_rng(7)
    A = t(rng.standard_normal((M, Kd)), dtype)
    B = t(rng.standard_normal((N, Kd)) * 0.1, dtype)
    bias = t(rng.standard_normal(N), dtype)
    Rm = t(rng.standard_normal((M, N)), dtype)
    U = t(rng.standard_normal((M, N)), dtype)
    acc = h(A) @ h(B).T
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tol = 2e-2 if dtype == "bf16" else 1e-4
    metric = rel_l2 if dtype == "bf16" else max_rel
    C = torch.empty((M, N), device=dev, dtype=tdt)
    C2 = torch.empty((M, N), device=dev, dtype=tdt)
    k = K()
    k.tpipe_k_gemm(dt, M, N, Kd, A, Kd, 1, B, Kd, 1, k.EPI_STORE, C, N)
    torch.cuda.synchronize()
    assert metric(h(C), acc) < tol
    k.tpipe_k_gemm(dt, M, N, Kd, A, Kd, 1, B, Kd, 1, k.EPI_BIAS, C, N, bias=bias)
    torch.cuda.synchronize()
    assert metric(h(C), acc + h(bias)) < tol
    k.tpipe_k_gemm(dt, M, N, Kd, A, Kd, 1, B, Kd, 1, k.EPI_BIAS_RES, C, N, bias=bias, R=Rm, ldr=N)
    torch.cuda.synchronize()
    assert metric(h(C), acc + h(bias) + h(Rm)) < tol
    k.tpipe_k_gemm(dt, M, N, Kd, A, Kd, 1, B, Kd, 1, k.EPI_BIAS_GELU, C, N, bias=bias, C2=C2, ldc2=N)
    torch.cuda.synchronize()
    u = acc + h(bias)
    assert metric(h(C), u) < tol
    assert metric(h(C2), R.gelu(h(C))) < tol
    k.tpipe_k_gemm(dt, M, N, Kd, A, Kd, 1, B, Kd, 1, k.EPI_DGELU, C, N, C2=C2, ldc2=N, aux=U,
                   ldaux=N)
    torch.cuda.synchronize()
    assert metric(h(C), acc * R.gelu_grad(h(U))) < tol
    assert metric(h(C2), R.gelu(h(U))) < tol


@pytest.mark.parametrize("majors", [(1, 1), (1, 0), (0, 0)])
def test_gemm_fp32_simt(majors):
    ak, bk = majors
    M, N, Kd = 130, 96, 200
    rng = np.random.default_rng(3)
    A = rng.standard_normal((M, Kd))
    B = rng.standard_normal((N, Kd))
    At = t(A if ak else A.T.copy(), "fp32")
    Bt = t(B if bk else B.T.copy(), "fp32")
    C = torch.zeros((M, N), device=dev)
    K().tpipe_k_gemm(0, M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk,
                     K().EPI_STORE_F32, C, N)
    torch.cuda.synchronize()
    assert max_rel(h(C), A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).T) < 1e-5


# ------------------------------------------------------------------ LayerNorm
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("rows,hd", [(64, 64), (130, 2048), (5, 5120), (45, 1024), (3, 4096),
                                     (9, 256)])
def test_layernorm(dtype, rows, hd):
    dt = 1 if dtype == "bf16" else 0
    rng = np.random.default_rng(rows)
    x = t(rng.standard_normal((rows, hd)) * 2 + 0.5, dtype)
    g = t(1 + 0.1 * rng.standard_normal(hd), dtype)
    b = t(0.1 * rng.standard_normal(hd), dtype)
    dy = t(rng.standard_normal((rows, hd)), dtype)
    res = t(rng.standard_normal((rows, hd)), dtype)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    k = K()
    k.tpipe_k_ln_fwd(dt, x, g, b, y, mean, rstd, rows, hd)
    yr, cache = R.ln_fwd(h(x), h(g), h(b))
    dx = torch.empty_like(x)
    dg = torch.zeros(hd, device=dev)
    db = torch.zeros(hd, device=dev)
    ws = torch.empty(2 * ((rows + 15) // 16) * hd, device=dev)
    k.tpipe_k_ln_bwd(dt, dy, x, g, mean, rstd, res, dx, dg, db, ws, rows, hd)
    torch.cuda.synchronize()
    dxr, dgr, dbr = R.ln_bwd(h(dy), cache)
    tol, metric = (2e-2, rel_l2) if dtype == "bf16" else (1e-4, max_rel)
    assert metric(h(y), yr) < tol
    assert max_rel(h(mean), h(x).mean(-1)) < 1e-5
    assert metric(h(dx), dxr + h(res)) < tol
    assert max_rel(h(dg), dgr) < (1e-2 if dtype == "bf16" else 1e-4)
    assert max_rel(h(db), dbr) < 1e-4


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("rows,hd", [(64, 64), (130, 2048), (45, 1024), (33, 4096)])
def test_layernorm_bwd_rsum(dtype, rows, hd):
    """ln_bwd with the fused residual-gradient column sum (bias grad of the
    preceding linear): equals ln_bwd + colsum(resid), accumulates (+=), and is
    bit-reproducible run to run."""
    dt = 1 if dtype == "bf16" else 0
    rng = np.random.default_rng(rows + hd)
    x = t(rng.standard_normal((rows, hd)) * 2 + 0.5, dtype)
    g = t(1 + 0.1 * rng.standard_normal(hd), dtype)
    b = t(0.1 * rng.standard_normal(hd), dtype)
    dy = t(rng.standard_normal((rows, hd)), dtype)
    res = t(rng.standard_normal((rows, hd)), dtype)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    k = K()
    k.tpipe_k_ln_fwd(dt, x, g, b, y, mean, rstd, rows, hd)
    _, cache = R.ln_fwd(h(x), h(g), h(b))
    dxr, dgr, dbr = R.ln_bwd(h(dy), cache)
    ws = torch.empty(3 * ((rows + 15) // 16) * hd, device=dev)
    outs = []
    for _ in range(2):
        dx = torch.empty_like(x)
        dg = torch.zeros(hd, device=dev)
        db = torch.zeros(hd, device=dev)
        drs = torch.full((hd,), 0.25, device=dev)
        k.tpipe_k_ln_bwd_rsum(dt, dy, x, g, mean, rstd, res, dx, dg, db, drs, ws, rows, hd)
        torch.cuda.synchronize()
        outs.append((dx.clone(), dg.clone(), db.clone(), drs.clone()))
    dx, dg, db, drs = outs[0]
    for u, v in zip(outs[0], outs[1]):
        assert torch.equal(u, v)
    tol, metric = (2e-2, rel_l2) if dtype == "bf16" else (1e-4, max_rel)
    assert metric(h(dx), dxr + h(res)) < tol
    assert max_rel(h(dg), dgr) < (1e-2 if dtype == "bf16" else 1e-4)
    assert max_rel(h(db), dbr) < 1e-4
    assert max_rel(h(drs), 0.25 + h(res).sum(0)) < 1e-4


# ------------------------------------------------------------------ attention
@pytest.mark.parametrize("dtype,impl", [("fp32", "default"), ("bf16", "default")])
@pytest.mark.parametrize("b,s,a,d", [(2, 32, 4, 16), (1, 100, 2, 64), (1, 257, 2, 128),
                                     (2, 384, 2, 128), (3, 200, 4, 64)])
def test_attention(dtype, impl, b, s, a, d):
    """bf16 d=64/128 = tcgen05/TMEM kernels; other d and fp32 = the SIMT kernels."""
    dt = 1 if dtype == "bf16" else 0
    hdim = a * d
    rng = np.random.default_rng(s + d)
    qkv = t(rng.standard_normal((b * s, 3 * hdim)), dtype)
    dout = t(rng.standard_normal((b * s, hdim)), dtype)
    o = torch.empty((b * s, hdim), device=dev, dtype=qkv.dtype)
    lse = torch.empty((b, a, s), device=dev)
    k = K()
    k.tpipe_k_attn_fwd(dt, qkv, o, lse, b, s, a, d)
    Q = h(qkv).reshape(b, s, 3 * hdim)
    q = R.split_heads(Q[..., :hdim], a)
    kk = R.split_heads(Q[..., hdim:2 * hdim], a)
    v = R.split_heads(Q[..., 2 * hdim:], a)
    Oref, cache, lref = R.attn_fwd(q, kk, v)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty((b, a, s), device=dev)
    k.tpipe_k_attn_bwd(dt, qkv, o, dout, lse, dqkv, ws, b, s, a, d)
    torch.cuda.synchronize()
    dQ, dK, dV = R.attn_bwd(R.split_heads(h(dout).reshape(b, s, hdim), a), cache)
    tol, metric = (2e-2, rel_l2) if dtype == "bf16" else (1e-4, max_rel)
    assert metric(h(o).reshape(b, s, hdim), R.merge_heads(Oref)) < tol
    assert max_rel(h(lse), lref) < 1e-4
    got = h(dqkv).reshape(b, s, 3 * hdim)
    assert metric(got[..., :hdim], R.merge_heads(dQ)) < tol
    assert metric(got[..., hdim:2 * hdim], R.merge_heads(dK)) < tol
    assert metric(got[..., 2 * hdim:], R.merge_heads(dV)) < tol


# ------------------------------------------------------------------ embedding / CE / colsum
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_embedding(dtype):
    dt = 1 if dtype == "bf16" else 0
    V, s, bsz, hd = 97, 32, 3, 64
    rows = s * bsz
    rng = np.random.default_rng(11)
    tok = torch.tensor(rng.integers(0, V, rows), dtype=torch.int32, device=dev)
    wte = t(rng.standard_normal((V, hd)), dtype)
    wpe = t(rng.standard_normal((s, hd)), dtype)
    x = torch.empty((rows, hd), device=dev, dtype=wte.dtype)
    k = K()
    k.tpipe_k_embed_fwd(dt, tok, wte, wpe, x, rows, s, hd)
    dx = t(rng.standard_normal((rows, hd)), dtype)
    dwte = torch.zeros((V, hd), device=dev)
    dwpe = torch.zeros((s, hd), device=dev)
    ws = torch.empty(2 * rows, dtype=torch.int32, device=dev)
    k.tpipe_k_embed_bwd(dt, tok, dx, dwte, dwpe, ws, rows, s, hd)
    torch.cuda.synchronize()
    tk = tok.cpu().numpy()
    ref = h(wte)[tk] + h(wpe)[np.arange(rows) % s]
    assert max_rel(h(x), ref) < (1e-2 if dtype == "bf16" else 1e-6)
    dref = np.zeros((V, hd))
    for r in range(rows):
        dref[tk[r]] += h(dx)[r]
    assert max_rel(h(dwte), dref) < 1e-5
    assert max_rel(h(dwpe), h(dx).reshape(bsz, s, hd).sum(0)) < 1e-5
    # determinism: a second run gives identical bits
    dwte2 = torch.zeros_like(dwte)
    k.tpipe_k_embed_bwd(dt, tok, dx, dwte2, dwpe, ws, rows, s, hd)
    torch.cuda.synchronize()
    assert torch.equal(dwte, dwte2)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_cross_entropy(dtype):
    dt = 1 if dtype == "bf16" else 0
    rows, V = 70, 50304
    rng = np.random.default_rng(5)
    logits = torch.tensor(rng.standard_normal((rows, V)).astype(np.float32) * 3, device=dev)
    tgt = torch.tensor(rng.integers(0, V, rows), dtype=torch.int32, device=dev)
    lse = torch.empty(rows, device=dev)
    loss = torch.zeros(1, device=dev)
    k = K()
    k.tpipe_k_ce_fwd(logits, tgt, lse, loss, 1.0 / rows, rows, V)
    d = torch.empty((rows, V), device=dev, dtype=torch.bfloat16 if dt else torch.float32)
    k.tpipe_k_ce_bwd(dt, logits, tgt, lse, d, 1.0 / rows, rows, V)
    torch.cuda.synchronize()
    L = h(logits)
    mx = L.max(-1, keepdims=True)
    lref = (mx + np.log(np.exp(L - mx).sum(-1, keepdims=True)))[:, 0]
    tk = tgt.cpu().numpy()
    assert max_rel(h(lse), lref) < 1e-6
    assert abs(h(loss)[0] - (lref - L[np.arange(rows), tk]).mean()) < 1e-5
    P = np.exp(L - lref[:, None])
    P[np.arange(rows), tk] -= 1
    tol = 2e-2 if dt else 1e-4
    assert (rel_l2 if dt else max_rel)(h(d), P / rows) < tol


@pytest.mark.parametrize("rows,n", [(300, 192), (2048, 2048), (130, 8192), (37, 6144), (16, 2056)])
def test_colsum(rows, n):
    rng = np.random.default_rng(2)
    for dtype in ("fp32", "bf16"):
        X = t(rng.standard_normal((rows, n)), dtype)
        out = torch.ones(n, device=dev)
        ws = torch.empty(((rows + 15) // 16) * n, device=dev)
        K().tpipe_k_colsum(1 if dtype == "bf16" else 0, X, out, ws, rows, n)
        torch.cuda.synchronize()
        assert max_rel(h(out), 1 + h(X).sum(0)) < 1e-5


# ------------------------------------------------------------------ AdamW
@pytest.mark.parametrize("off", [0, 1])
@pytest.mark.parametrize("decay", [0, 1])
def test_adamw_device_host_bitexact(decay, off):
    """Device AdamW == host AdamW bit for bit (T-Offload on/off),
    and both match the fp64 oracle step. off = 1: fp32 states one element past
    a 16-byte boundary (the scalar kernel; off = 0 the 4-wide one with a
    ragged tail)."""
    n = 100_003
    rng = np.random.default_rng(9)
    w0 = rng.standard_normal(n).astype(np.float32)
    m0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v0 = (rng.random(n) * 1e-6).astype(np.float32)
    g0 = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    hp = dict(lr=3e-3, b1=0.9, b2=0.95, eps=1e-8, wd=0.1)
    step = 3
    bc1, bc2 = 1 - 0.9 ** step, 1 - 0.95 ** step
    Wm, Mm, Vm, Gm = (torch.tensor(np.concatenate([np.zeros(off, np.float32), x]), device=dev)[off:]
                      for x in (w0, m0, v0, g0))
    wb = torch.empty(n, dtype=torch.bfloat16, device=dev)
    K().tpipe_k_adamw(1, Wm, Mm, Vm, Gm, wb, n, decay, hp["lr"], hp["b1"], hp["b2"], hp["eps"],
                      hp["wd"], bc1, bc2)
    torch.cuda.synchronize()
    hw, hm, hv = w0.copy(), m0.copy(), v0.copy()
    hb = np.empty(n, np.uint16)
    K().tpipe_host_adamw(hw, hm, hv, g0, hb, n, decay, hp["lr"], hp["b1"], hp["b2"], hp["eps"],
                         hp["wd"], bc1, bc2)
    assert np.array_equal(Wm.cpu().numpy().view(np.uint32), hw.view(np.uint32))
    assert np.array_equal(Mm.cpu().numpy().view(np.uint32), hm.view(np.uint32))
    assert np.array_equal(Vm.cpu().numpy().view(np.uint32), hv.view(np.uint32))
    assert np.array_equal(wb.cpu().view(torch.int16).numpy().view(np.uint16), hb)
    assert float(Gm.abs().max()) == 0.0            # grad zeroed
    rw, rm, rv = R.adamw(w0, g0.astype(np.float64), m0.astype(np.float64),
                         v0.astype(np.float64), step, hp["lr"], bool(decay))
    assert max_rel(hw, rw) < 1e-6


@pytest.mark.parametrize("rows,V,h", [(2048, 50304, 2048), (256, 512, 256), (200, 320, 128)])
def test_head_ce_fused_vs_fp64(rows, V, h):
    """Fused LM head + softmax CE (K8, DESIGN R30): the logits never reach HBM.
    LSE / loss / dlogits against an fp64 reference of the same bf16 operands
    (ragged rows and a partial 128-column group covered)."""
    from paper_2503_03182_b200 import kernels as K
    g = torch.Generator(device="cpu").manual_seed(rows + V)
    x = torch.randn(rows, h, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(V, h, generator=g) * 0.05).to(torch.bfloat16).cuda()
    tgt = torch.randint(0, V, (rows,), generator=g, dtype=torch.int32).cuda()
    lse = torch.empty(rows, device="cuda")
    dl = torch.empty(rows, V, device="cuda", dtype=torch.bfloat16)
    loss = torch.zeros(1, device="cuda")
    ng = (V + 63) // 64
    ws = torch.empty(2 * rows * ng + 2 * rows, device="cuda")
    scale = 1.0 / rows
    K.tpipe_k_head_ce(x, w, tgt, lse, dl, loss, scale, rows, V, h, ws)
    torch.cuda.synchronize()
    z = x.double() @ w.double().T
    lref = torch.logsumexp(z, dim=1)
    loss_ref = float((lref - z.gather(1, tgt.long()[:, None])[:, 0]).sum() * scale)
    p = torch.softmax(z, dim=1)
    p[torch.arange(rows), tgt.long()] -= 1.0
    dref = p * scale
    assert float((lse.double() - lref).abs().max()) < 2e-5 * max(1.0, float(lref.abs().max()))
    assert abs(float(loss) - loss_ref) / abs(loss_ref) < 1e-5
    err = float(torch.linalg.norm(dl.double() - dref) / torch.linalg.norm(dref))
    assert err < 1e-2, err


@pytest.mark.parametrize("M,N,Kd,width", [(2048, 8192, 512, 224), (2048, 6144, 320, 240),
                                          (2048, 2048, 4160, 240), (2048, 2048, 512, 240),
                                          (1904, 2080, 200, 240), (6144, 2048, 256, 240)])
@pytest.mark.parametrize("majors", [(1, 1), (1, 0), (0, 0)])
def test_gemm_wide_choice(M, N, Kd, width, majors):
    """240 / 224-column tiles (chosen where they fill the 148 SMs better;
    `width` is the cost model's pick for the shape: CTA pairs for all but
    (2048, 2048, 512) and (1904, 2080, 200)) incl. the 16-column half chunk
    stored without TMA and ragged M / N / K: every epilogue matches fp64 and
    the 256-wide kernel (wide choice off) to fp32 accumulation-order tolerance.
    The widths apply to K-major B (majors (1, 1)); the others stay 256 wide."""
    ak, bk = majors
    k = K()
    rng = np.random.default_rng(M + 7 * N + Kd + width)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    At = t(A if ak else A.T.copy(), "bf16")
    Bt = t(B if bk else B.T.copy(), "bf16")
    ref = h(At if ak else At.T) @ h(Bt if bk else Bt.T).T
    U = t(rng.standard_normal((M, N)), "bf16")
    Rr = t(rng.standard_normal((M, N)), "bf16")
    bias = t(rng.standard_normal(N), "bf16")
    args = (M, N, Kd, At, Kd if ak else M, ak, Bt, Kd if bk else N, bk)

    def run():
        C = torch.zeros((M, N), device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_STORE_F32, C, N)
        Acc = torch.full((M, N), 2.0, device=dev, dtype=torch.float32)
        k.tpipe_k_gemm(1, *args, k.EPI_ACC_F32, Acc, N)
        Cs = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_STORE, Cs, N)
        Cr = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_BIAS_RES, Cr, N, bias=bias, R=Rr, ldr=N)
        Cd = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Cg = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_DGELU, Cd, N, C2=Cg, ldc2=N, aux=U, ldaux=N)
        Cu = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Cgl = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        k.tpipe_k_gemm(1, *args, k.EPI_BIAS_GELU, Cu, N, bias=bias, C2=Cgl, ldc2=N)
        torch.cuda.synchronize()
        return C, Acc, Cs, Cr, Cd, Cg, Cu, Cgl
    wide = run()
    try:
        k.tpipe_k_gemm_set_wide_choice(0)
        narrow = run()
    finally:
        k.tpipe_k_gemm_set_wide_choice(1)
    C, Acc, Cs, Cr, Cd, Cg, Cu, Cgl = wide
    assert max_rel(h(C), ref) < 1e-4
    assert max_rel(h(Acc), 2 + ref) < 1e-4
    assert rel_l2(h(Cs), ref) < 1e-2
    assert rel_l2(h(Cr), ref + h(bias) + h(Rr)) < 1e-2
    assert rel_l2(h(Cd), ref * R.gelu_grad(h(U))) < 1e-2
    assert rel_l2(h(Cg), R.gelu(h(U))) < 1e-2
    assert rel_l2(h(Cu), ref + h(bias)) < 1e-2
    assert rel_l2(h(Cgl), R.gelu(h(Cu))) < 1e-2
    # same math, different tile grouping: fp32 results agree to accumulation order
    assert max_rel(h(C), h(narrow[0])) < 1e-5
    assert max_rel(h(Acc), h(narrow[1])) < 1e-5
    for a, b in zip(wide[2:], narrow[2:]):
        assert rel_l2(h(a), h(b)) < 1e-2


@pytest.mark.parametrize("rows,hd", [(2048, 2048), (37, 256), (130, 1792)])
def test_layernorm_bwd_rows_vs_staged(rows, hd):
    """The row-parallel LN backward (bf16, h <= 2048) against the staged
    kernel it replaces and against fp64: dx, dgamma, dbeta and the fused
    residual column sum; bit-reproducible run to run."""
    rng = np.random.default_rng(rows * 3 + hd)
    x = t(rng.standard_normal((rows, hd)) * 2 + 0.5, "bf16")
    g = t(1 + 0.1 * rng.standard_normal(hd), "bf16")
    b = t(0.1 * rng.standard_normal(hd), "bf16")
    dy = t(rng.standard_normal((rows, hd)), "bf16")
    res = t(rng.standard_normal((rows, hd)), "bf16")
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    k = K()
    k.tpipe_k_ln_fwd(1, x, g, b, y, mean, rstd, rows, hd)
    _, cache = R.ln_fwd(h(x), h(g), h(b))
    dxr, dgr, dbr = R.ln_bwd(h(dy), cache)
    ws = torch.empty(3 * ((rows + 15) // 16) * hd, device=dev)

    def run():
        dx = torch.empty_like(x)
        dg = torch.zeros(hd, device=dev)
        db = torch.zeros(hd, device=dev)
        drs = torch.zeros(hd, device=dev)
        k.tpipe_k_ln_bwd_rsum(1, dy, x, g, mean, rstd, res, dx, dg, db, drs, ws, rows, hd)
        torch.cuda.synchronize()
        return dx, dg, db, drs
    new, again = run(), run()
    for u, v in zip(new, again):
        assert torch.equal(u, v)
    try:
        k.tpipe_k_ln_set_rows_bwd(0)
        old = run()
    finally:
        k.tpipe_k_ln_set_rows_bwd(1)
    dx, dg, db, drs = new
    assert rel_l2(h(dx), dxr + h(res)) < 2e-2
    assert max_rel(h(dg), dgr) < 1e-2
    assert max_rel(h(db), dbr) < 1e-4
    assert max_rel(h(drs), h(res).sum(0)) < 1e-4
    assert rel_l2(h(dx), h(old[0])) < 1e-2
    for u, v in zip(new[1:], old[1:]):
        assert max_rel(h(u), h(v)) < 1e-5


@pytest.mark.parametrize("M,N,Kd,s,hd,bk", [(2048, 2048, 2048, 2048, 128, 0), (512, 256, 320, 256, 64, 0),
                                             (4096, 4096, 512, 1024, 128, 0), (1024, 2048, 256, 512, 128, 1)])
def test_gemm_dot_epilogue(M, N, Kd, s, hd, bk):
    """EPI_STORE_DOT (the out-projection data gradient with the attention
    backward's D = rowsum(dO o O) fused into its epilogue): C matches fp64 and
    D equals the fp64 dot of the stored bf16 C with O per (token, head) in the
    [b, a, s] layout the attention backward reads; bit-reproducible."""
    k = K()
    rng = np.random.default_rng(M + N + Kd + hd)
    A = rng.standard_normal((M, Kd)).astype(np.float32)
    B = rng.standard_normal((N, Kd)).astype(np.float32)
    At = t(A, "bf16")
    Bt = t(B if bk else B.T.copy(), "bf16")
    O = t(rng.standard_normal((M, N)), "bf16")
    ref = h(At) @ h(Bt if bk else Bt.T).T

    def run():
        C = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        Dv = torch.full((M // s, N // hd, s), 7.0, device=dev)
        k.tpipe_k_gemm_dot(M, N, Kd, At, Kd, 1, Bt, Kd if bk else N, bk, C, N, O, N, Dv, s, hd)
        torch.cuda.synchronize()
        return C, Dv
    (C, Dv), (C2, Dv2) = run(), run()
    assert torch.equal(C, C2) and torch.equal(Dv, Dv2)
    assert rel_l2(h(C), ref) < 1e-2
    a = N // hd
    prod = (h(C) * h(O)).reshape(M // s, s, a, hd).sum(-1)          # [b, s, a]
    Dref = prod.transpose(0, 2, 1)                                    # [b, a, s]
    assert max_rel(h(Dv), Dref) < 1e-4


@pytest.mark.parametrize("M,N,Kd,majors", [(2048, 8192, 256, (1, 1)), (512, 1024, 128, (1, 0))])
def test_gelu_recompute_bitexact(M, N, Kd, majors):
    """The GELU the backward recomputes (EPI_DGELU's C2 = gelu(U)) is
    bit-identical to the activation the forward stored (EPI_BIAS_GELU's C2 =
    gelu(u)) for the same stored pre-activation u: the FC2 weight gradient sees
    exactly the forward's operand."""
    ak, bk = majors
    k = K()
    rng = np.random.default_rng(M + N)
    A = t(rng.standard_normal((M, Kd)), "bf16")
    B = t(rng.standard_normal((N, Kd)) if bk else rng.standard_normal((Kd, N)), "bf16")
    bias = t(0.5 * rng.standard_normal(N), "bf16")
    U = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    Gf = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    k.tpipe_k_gemm(1, M, N, Kd, A, Kd, ak, B, Kd if bk else N, bk, k.EPI_BIAS_GELU, U, N, bias=bias, C2=Gf, ldc2=N)
    Dd = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    Gb = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    k.tpipe_k_gemm(1, M, N, Kd, A, Kd, ak, B, Kd if bk else N, bk, k.EPI_DGELU, Dd, N, C2=Gb, ldc2=N, aux=U, ldaux=N)
    torch.cuda.synchronize()
    assert torch.equal(Gf, Gb)


def test_ln_bwd_partials_capi():
    """tpipe_k_ln_bwd_partials (the layer backward's LN backward): dx equals
    the reduced form's and the column partials sum to its dgamma / dbeta /
    residual column sum in block order."""
    rows, hd = 300, 2048
    rng = np.random.default_rng(5)
    x = t(rng.standard_normal((rows, hd)), "bf16")
    g = t(1 + 0.1 * rng.standard_normal(hd), "bf16")
    b = t(0.1 * rng.standard_normal(hd), "bf16")
    dy = t(rng.standard_normal((rows, hd)), "bf16")
    res = t(rng.standard_normal((rows, hd)), "bf16")
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=dev)
    rstd = torch.empty(rows, device=dev)
    k = K()
    k.tpipe_k_ln_fwd(1, x, g, b, y, mean, rstd, rows, hd)
    nb = (rows + 15) // 16
    ws = torch.empty(3 * nb * hd, device=dev)
    dx = torch.empty_like(x)
    k.tpipe_k_ln_bwd_partials(dy, x, g, mean, rstd, res, dx, ws, rows, hd, 1)
    dx2 = torch.empty_like(x)
    dg, db, drs = torch.zeros(hd, device=dev), torch.zeros(hd, device=dev), torch.zeros(hd, device=dev)
    ws2 = torch.empty(3 * nb * hd, device=dev)
    k.tpipe_k_ln_bwd_rsum(1, dy, x, g, mean, rstd, res, dx2, dg, db, drs, ws2, rows, hd)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2)
    parts = h(ws).reshape(3, nb, hd).sum(1)
    for got, ref in zip(parts, (h(dg), h(db), h(drs))):
        assert max_rel(got, ref) < 1e-5
