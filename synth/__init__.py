"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds NONE of the method's arithmetic: only random-number generation with the
recipe of SURVEY §8(d) / DESIGN.md §6 (tokens uniform in [0, V_eff) from
PCG64(seed_data + step), weights from PCG64(seed_w) with GPT-2/3 init N-1).

Weights are returned per global layer as float32 arrays with the shapes of
DESIGN.md §2 (out-features first, like ``y = x @ W.T``).
"""

from __future__ import annotations

import math

import numpy as np

SEED_W = 1234
SEED_DATA = 5678


def tokens(vocab: int, m: int, micro_batch: int, seq_len: int, step: int = 0,
           seed: int = SEED_DATA, vocab_eff: int | None = None):
    """Returns (inputs, targets), each int32 [m, micro_batch, seq_len]."""
    rng = np.random.Generator(np.random.PCG64(seed + step))
    hi = vocab if vocab_eff is None else vocab_eff
    t = rng.integers(0, hi, size=(m, micro_batch, seq_len + 1), dtype=np.int64)
    return t[..., :-1].astype(np.int32), t[..., 1:].astype(np.int32)


LAYER_TENSORS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                 "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")


def layer_shapes(h: int, f: int):
    return {
        "ln1_g": (h,), "ln1_b": (h,),
        "w_qkv": (3 * h, h), "b_qkv": (3 * h,),
        "w_o": (h, h), "b_o": (h,),
        "ln2_g": (h,), "ln2_b": (h,),
        "w_1": (f, h), "b_1": (f,),
        "w_2": (h, f), "b_2": (h,),
    }


def weights(n_layers: int, hidden: int, ffn: int, vocab: int, seq_len: int,
            seed: int = SEED_W, std: float = 0.02, bias_std: float = 0.0,
            ln_jitter: float = 0.0):
    """Full-model float32 weights. Init (SURVEY N-1): matrices N(0, std);
    w_o and w_2 N(0, std/sqrt(2L)); biases 0; LN gamma 1, beta 0. Tests may
    set bias_std / ln_jitter > 0 so that bias and LN-affine terms are exercised
    (a zero bias would hide a dropped bias term)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    h, f = hidden, ffn
    proj_std = std / math.sqrt(2 * n_layers)

    def normal(shape, sd):
        return (rng.standard_normal(size=shape, dtype=np.float32) * np.float32(sd))

    W = {"wte": normal((vocab, h), std), "wpe": normal((seq_len, h), std)}
    layers = []
    for _ in range(n_layers):
        L = {}
        for name, shape in layer_shapes(h, f).items():
            if name in ("w_o", "w_2"):
                L[name] = normal(shape, proj_std)
            elif name.startswith("w_"):
                L[name] = normal(shape, std)
            elif name.endswith("_g"):
                L[name] = (np.ones(shape, np.float32)
                           + normal(shape, ln_jitter) if ln_jitter else np.ones(shape, np.float32))
            else:
                L[name] = normal(shape, bias_std) if bias_std else np.zeros(shape, np.float32)
        layers.append(L)
    W["layers"] = layers
    W["lnf_g"] = (np.ones((h,), np.float32) + normal((h,), ln_jitter)
                  if ln_jitter else np.ones((h,), np.float32))
    W["lnf_b"] = normal((h,), bias_std) if bias_std else np.zeros((h,), np.float32)
    W["w_head"] = normal((vocab, h), std)
    return W
