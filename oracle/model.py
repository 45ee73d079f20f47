"""Oracle Part 2 — fp64 NumPy forward/backward of the transformer + AdamW.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

The paper specifies no model equations (it trains "LLAMA2-70B / GPT3-175B"
shapes, with FlashAttention and operator-level recompute enabled by
default). The readings below are SURVEY §8(c) N-1..N-4 / DESIGN.md §2:

* pre-LN GPT block (N-1):
    x2 = x  + Attn(LN1(x)) W_o^T + b_o
    x3 = x2 + GELU_tanh(LN2(x2) W_1^T + b_1) W_2^T + b_2
  LN eps 1e-5, biased variance; causal softmax attention, scale 1/sqrt(d);
  qkv = LN1(x) W_qkv^T + b_qkv with columns [q | k | v], head j = columns
  j*d:(j+1)*d of each; learned absolute position embedding; final LN_f;
  untied LM head without bias; no dropout.
* loss = mean token cross-entropy over all m*b*s tokens of the step (N-1).
* AdamW (N-3), PyTorch semantics: decoupled decay on 2-D tensors only,
  bias-corrected moments, constant lr, no clipping.

Schedule-free: the step's gradient is the sum over microbatches in index
order. Plain loops over heads/sequences; every backward formula
is the textbook derivative of the line it mirrors.
"""

from __future__ import annotations

import math

import numpy as np

LN_EPS = 1e-5
GELU_C = math.sqrt(2.0 / math.pi)


# ---------------------------------------------------------------- layernorm
def ln_fwd(x, g, b):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (x - mu) * rstd
    return xhat * g + b, (xhat, rstd, g)


def ln_bwd(dy, cache):
    xhat, rstd, g = cache
    dg = (dy * xhat).reshape(-1, xhat.shape[-1]).sum(axis=0)
    db = dy.reshape(-1, dy.shape[-1]).sum(axis=0)
    dxhat = dy * g
    dx = rstd * (dxhat - dxhat.mean(axis=-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True))
    return dx, dg, db


# ---------------------------------------------------------------- gelu
def gelu(u):
    return 0.5 * u * (1.0 + np.tanh(GELU_C * (u + 0.044715 * u ** 3)))


def gelu_grad(u):
    t = np.tanh(GELU_C * (u + 0.044715 * u ** 3))
    dt = (1.0 - t * t) * GELU_C * (1.0 + 3 * 0.044715 * u * u)
    return 0.5 * (1.0 + t) + 0.5 * u * dt


# ---------------------------------------------------------------- attention
def attn_fwd(q, k, v):
    """q,k,v: [b, a, s, d]. Causal softmax(q k^T / sqrt(d)) v."""
    d = q.shape[-1]
    s = q.shape[-2]
    scale = 1.0 / math.sqrt(d)
    S = (q @ k.swapaxes(-1, -2)) * scale                  # [b, a, s, s]
    mask = np.triu(np.ones((s, s), dtype=bool), k=1)       # j > i masked
    S = np.where(mask, -np.inf, S)
    Smax = S.max(axis=-1, keepdims=True)
    E = np.exp(S - Smax)
    P = E / E.sum(axis=-1, keepdims=True)
    O = P @ v
    lse = (Smax + np.log(E.sum(axis=-1, keepdims=True)))[..., 0]
    return O, (q, k, v, P, scale), lse


def attn_bwd(dO, cache):
    q, k, v, P, scale = cache
    dV = P.swapaxes(-1, -2) @ dO
    dP = dO @ v.swapaxes(-1, -2)
    dS = P * (dP - (dP * P).sum(axis=-1, keepdims=True))
    dQ = (dS @ k) * scale
    dK = (dS.swapaxes(-1, -2) @ q) * scale
    return dQ, dK, dV


def split_heads(x, a):
    b, s, h = x.shape
    return x.reshape(b, s, a, h // a).transpose(0, 2, 1, 3)


def merge_heads(x):
    b, a, s, d = x.shape
    return x.transpose(0, 2, 1, 3).reshape(b, s, a * d)


# ---------------------------------------------------------------- block
def layer_fwd(x, L, a):
    """x: [b, s, h] -> (y, cache). L: dict of fp64 tensors (synth names)."""
    h = x.shape[-1]
    ln1, c_ln1 = ln_fwd(x, L["ln1_g"], L["ln1_b"])
    qkv = ln1 @ L["w_qkv"].T + L["b_qkv"]
    q = split_heads(qkv[..., 0:h], a)
    k = split_heads(qkv[..., h:2 * h], a)
    v = split_heads(qkv[..., 2 * h:3 * h], a)
    O, c_att, lse = attn_fwd(q, k, v)
    o = merge_heads(O)
    x2 = x + o @ L["w_o"].T + L["b_o"]
    ln2, c_ln2 = ln_fwd(x2, L["ln2_g"], L["ln2_b"])
    u = ln2 @ L["w_1"].T + L["b_1"]
    g = gelu(u)
    y = x2 + g @ L["w_2"].T + L["b_2"]
    cache = dict(x=x, ln1=ln1, c_ln1=c_ln1, c_att=c_att, o=o, x2=x2, ln2=ln2,
                 c_ln2=c_ln2, u=u, g=g, lse=lse, qkv=qkv)
    return y, cache


def layer_bwd(dy, C, L, a):
    """Returns (dx, grads dict with synth names)."""
    G = {}
    h = dy.shape[-1]
    flat = lambda t: t.reshape(-1, t.shape[-1])
    # FC2: y = x2 + g W2^T + b2
    G["w_2"] = flat(dy).T @ flat(C["g"])
    G["b_2"] = flat(dy).sum(axis=0)
    dg = dy @ L["w_2"]
    du = dg * gelu_grad(C["u"])
    # FC1: u = ln2 W1^T + b1
    G["w_1"] = flat(du).T @ flat(C["ln2"])
    G["b_1"] = flat(du).sum(axis=0)
    dln2 = du @ L["w_1"]
    dx2_ln, G["ln2_g"], G["ln2_b"] = ln_bwd(dln2, C["c_ln2"])
    dx2 = dy + dx2_ln
    # out-proj: x2 = x + o Wo^T + bo
    G["w_o"] = flat(dx2).T @ flat(C["o"])
    G["b_o"] = flat(dx2).sum(axis=0)
    do = dx2 @ L["w_o"]
    dQ, dK, dV = attn_bwd(split_heads(do, a), C["c_att"])
    dqkv = np.concatenate([merge_heads(dQ), merge_heads(dK), merge_heads(dV)], axis=-1)
    G["w_qkv"] = flat(dqkv).T @ flat(C["ln1"])
    G["b_qkv"] = flat(dqkv).sum(axis=0)
    dln1 = dqkv @ L["w_qkv"]
    dx_ln, G["ln1_g"], G["ln1_b"] = ln_bwd(dln1, C["c_ln1"])
    dx = dx2 + dx_ln
    assert dx.shape[-1] == h
    return dx, G


# ---------------------------------------------------------------- model
def to64(W):
    out = {k: np.asarray(v, np.float64) for k, v in W.items() if k != "layers"}
    out["layers"] = [{k: np.asarray(v, np.float64) for k, v in L.items()} for L in W["layers"]]
    return out


def microbatch_fwd_bwd(W, tok, tgt, n_heads, n_total_tokens):
    """One microbatch. tok, tgt: int [b, s]. Returns (loss contribution, grads).
    loss contribution = sum_tokens CE / n_total_tokens."""
    b, s = tok.shape
    x = W["wte"][tok] + W["wpe"][np.arange(s)][None, :, :]
    caches = []
    for L in W["layers"]:
        x, C = layer_fwd(x, L, n_heads)
        caches.append(C)
    xf, c_lnf = ln_fwd(x, W["lnf_g"], W["lnf_b"])
    logits = xf @ W["w_head"].T                            # [b, s, V]
    mx = logits.max(axis=-1, keepdims=True)
    lse = (mx + np.log(np.exp(logits - mx).sum(axis=-1, keepdims=True)))[..., 0]
    picked = np.take_along_axis(logits, tgt[..., None], axis=-1)[..., 0]
    loss = float((lse - picked).sum()) / n_total_tokens
    # backward: dCE/dlogits = softmax - onehot, scaled by 1/N
    P = np.exp(logits - lse[..., None])
    onehot = np.zeros_like(P)
    np.put_along_axis(onehot, tgt[..., None], 1.0, axis=-1)
    dlogits = (P - onehot) / n_total_tokens
    G = {"w_head": dlogits.reshape(-1, dlogits.shape[-1]).T @ xf.reshape(-1, xf.shape[-1])}
    dxf = dlogits @ W["w_head"]
    dx, G["lnf_g"], G["lnf_b"] = ln_bwd(dxf, c_lnf)
    G["layers"] = [None] * len(W["layers"])
    for li in reversed(range(len(W["layers"]))):
        dx, G["layers"][li] = layer_bwd(dx, caches[li], W["layers"][li], n_heads)
    # embedding: x0 = wte[tok] + wpe[pos]
    dwte = np.zeros_like(W["wte"])
    flat_tok = tok.reshape(-1)
    flat_dx = dx.reshape(-1, dx.shape[-1])
    for r in range(flat_tok.shape[0]):                     # index order
        dwte[flat_tok[r]] += flat_dx[r]
    G["wte"] = dwte
    G["wpe"] = dx.sum(axis=0)
    return loss, G


def zeros_like_tree(W):
    out = {k: np.zeros_like(v) for k, v in W.items() if k != "layers"}
    out["layers"] = [{k: np.zeros_like(v) for k, v in L.items()} for L in W["layers"]]
    return out


def add_tree(A, B):
    for k in A:
        if k == "layers":
            for La, Lb in zip(A["layers"], B["layers"]):
                for kk in La:
                    La[kk] += Lb[kk]
        else:
            A[k] += B[k]


def step_grads(W, tokens, targets, n_heads):
    """Full step: loss (mean CE over m*b*s tokens) and grads summed over the m
    microbatches in index order. tokens, targets: int [m, b, s]."""
    W = W if isinstance(W["wte"], np.ndarray) and W["wte"].dtype == np.float64 else to64(W)
    m = tokens.shape[0]
    N = tokens.size
    G = zeros_like_tree(W)
    loss = 0.0
    for i in range(m):
        li, Gi = microbatch_fwd_bwd(W, tokens[i], targets[i], n_heads, N)
        loss += li
        add_tree(G, Gi)
    return loss, G


def loss_only(W, tokens, targets, n_heads):
    """Forward-only loss (used by the finite-difference pin)."""
    m = tokens.shape[0]
    N = tokens.size
    total = 0.0
    for i in range(m):
        tok, tgt = tokens[i], targets[i]
        b, s = tok.shape
        x = W["wte"][tok] + W["wpe"][np.arange(s)][None]
        for L in W["layers"]:
            x, _ = layer_fwd(x, L, n_heads)
        xf, _ = ln_fwd(x, W["lnf_g"], W["lnf_b"])
        logits = xf @ W["w_head"].T
        mx = logits.max(axis=-1, keepdims=True)
        lse = (mx + np.log(np.exp(logits - mx).sum(axis=-1, keepdims=True)))[..., 0]
        picked = np.take_along_axis(logits, tgt[..., None], axis=-1)[..., 0]
        total += float((lse - picked).sum())
    return total / N


# ---------------------------------------------------------------- AdamW
ADAM_B1, ADAM_B2, ADAM_EPS, WEIGHT_DECAY = 0.9, 0.95, 1e-8, 0.1


def adamw(w, g, m, v, t, lr, decay: bool, b1=ADAM_B1, b2=ADAM_B2, eps=ADAM_EPS,
          wd=WEIGHT_DECAY):
    """One AdamW step at (1-based) step t, PyTorch torch.optim.AdamW semantics:
    w <- w (1 - lr wd)   [decayed tensors only]
    m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2
    w <- w - lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)
    Returns new (w, m, v)."""
    w = np.array(w, np.float64)
    if decay:
        w = w * (1.0 - lr * wd)
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    w = w - lr * mhat / (np.sqrt(vhat) + eps)
    return w, m, v
