"""Packed parameter layout of one chunk, for marshalling
weights in and gradients out of the runtime:

  [stage 0, chunk 1]  wte [V,h], wpe [s,h]
  per layer           ln1_g, ln1_b, w_qkv [3h,h], b_qkv, w_o [h,h], b_o,
                      ln2_g, ln2_b, w_1 [f,h], b_1, w_2 [h,f], b_2
  [last stage, chunk v] lnf_g, lnf_b, w_head [V,h]

Chunk c of stage s holds global layer block (c-1)p + s (P:210 layout)."""

from __future__ import annotations

import numpy as np

LAYER_TENSORS = ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
                 "ln2_g", "ln2_b", "w_1", "b_1", "w_2", "b_2")


def global_layers(p: int, v: int, layers_chunk, s: int, c: int):
    """Global layer indices held by (stage s, chunk c). `layers_chunk` is the
    uniform per-stage (n1, .., nv) (or (n,) at v = 1), or a per-stage list of
    such tuples (plan.partition, DESIGN R27): chunk-1 layers are numbered
    through the stages first, then chunk-2 layers, ... (P:210 layout)."""
    if layers_chunk and isinstance(layers_chunk[0], (tuple, list)):
        part = [tuple(x) for x in layers_chunk]
    else:
        part = [tuple(layers_chunk)] * p
    # chunk c's layers come after every stage's chunks 1..c-1 (v chunks, R32)
    off = sum(x[cc] for x in part for cc in range(c - 1)) + sum(part[t][c - 1] for t in range(s))
    return list(range(off, off + part[s][c - 1]))


def chunk_entries(p, v, layers_chunk, s, c):
    """[(key, layer or None)] in packed order; key names follow synth.weights."""
    out = []
    if s == 0 and c == 1:
        out += [("wte", None), ("wpe", None)]
    for g in global_layers(p, v, layers_chunk, s, c):
        out += [(t, g) for t in LAYER_TENSORS]
    if s == p - 1 and c == v:
        out += [("lnf_g", None), ("lnf_b", None), ("w_head", None)]
    return out


def _get(W, key, layer):
    return W["layers"][layer][key] if layer is not None else W[key]


def pack(W, p, v, layers_chunk, s, c, dtype=np.float32):
    parts = [np.asarray(_get(W, k, l), dtype).reshape(-1)
             for k, l in chunk_entries(p, v, layers_chunk, s, c)]
    return np.ascontiguousarray(np.concatenate(parts))


def unpack(flat, W_like, p, v, layers_chunk, s, c):
    """Split a flat chunk vector into {(key, layer): array shaped like W_like}."""
    out, off = {}, 0
    for k, l in chunk_entries(p, v, layers_chunk, s, c):
        shape = np.shape(_get(W_like, k, l))
        n = int(np.prod(shape))
        out[(k, l)] = np.asarray(flat[off:off + n]).reshape(shape)
        off += n
    assert off == len(flat), (off, len(flat))
    return out
