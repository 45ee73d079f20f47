"""Independent pins of the oracle's stash byte model (oracle/stream.sizes).

The pins are the per-token stash accounting of SURVEY §8(c) N-2 — the
reading of what a pre-LN GPT layer must keep for its backward when
operator-level recompute regenerates the LN outputs, GELU(u) and the
attention probabilities — written as closed forms in (h, a, b, s), not as the
oracle's per-tensor sum:

  bf16, f = 4h:  LS = b·s·(20h + 16 + 4a)   [x_in 2h, qkv 6h, attn-out 2h,
                                             x_mid 2h, u 8h; LN1/LN2
                                             mean+rstd 16; LSE 4 per head]
  fp32, f = 4h:  LS = b·s·(40h + 16 + 4a)

and the chunk-level composition of SURVEY §8(c) "Part 1 bytes":
  * a chunk's stash is n·LS, minus its input activation when that input is
    the received IN buffer (the checkpoint, b·s·h·es, counted once);
  * the head chunk adds x_f (b·s·h·es), LN_f mean/rstd (8 B/token) and the
    CE log-sum-exp (4 B/token);
  * 1F1B + full recompute keeps only the layer inputs (b·s·h·es per layer);
  * model state 18 B/param in bf16 (bf16 w 2, fp32 grad 4, master 4, Adam
    m, v 8); 12 of them leave HBM under T-Offload (D-8).

The planner's byte model equals the oracle's element by element
(tests/test_plan_parity.py), and at runtime creation the kernels' own
carve-ups are checked against the planner's buffer bytes
(runtime.cpp check_layouts; GPU canary test in test_gpu_realkernels.py).
The per-op workspace bytes are the implementation's declared maxima (SURVEY
§8(c): "per-op workspace = the declared maximum for that op kind"); they are
pinned here only by lower bounds on what each op must hold at once.
"""

import pytest

from oracle import stream as T

SHAPES = [  # (h, a, s, b): C1, C2 (1.3B), C3-like (7B), C4-like (13B)
    (64, 4, 32, 2), (2048, 16, 2048, 1), (4096, 32, 4096, 1), (5120, 40, 8192, 1)]


def desc(h, a, s, b, L=8, dtype=T.BF16):
    return T.ModelDesc(L, h, a, 4 * h, 256 if h == 64 else 32000, s, b, dtype)


@pytest.mark.parametrize("h,a,s,b", SHAPES)
@pytest.mark.parametrize("dtype,per_h", [(T.BF16, 20), (T.FP32, 40)])
def test_layer_stash_closed_form(h, a, s, b, dtype, per_h):
    d = desc(h, a, s, b, dtype=dtype)
    z = T.sizes(d, 4, 2, 1, 1)
    assert z["layer_stash"] == b * s * (per_h * h + 16 + 4 * a)


@pytest.mark.parametrize("h,a,s,b", SHAPES)
@pytest.mark.parametrize("p", [2, 4])
def test_chunk_stash_composition(h, a, s, b, p):
    L = 4 * p                                    # two layers per chunk
    d = desc(h, a, s, b, L=L)
    LS = b * s * (20 * h + 16 + 4 * a)
    act = b * s * h * 2
    n = 2
    mid = T.sizes(d, p, 2, 1, 1)                 # stage 1 chunk 1: input received
    assert mid["stash"] == n * LS - act
    emb = T.sizes(d, p, 2, 0, 1)                 # stage 0 chunk 1: input is the embedding
    assert emb["stash"] == n * LS
    head = T.sizes(d, p, 2, p - 1, 2)            # last stage chunk 2: LM head
    assert head["stash"] == n * LS - act + act + b * s * (8 + 4)
    full = T.sizes(d, p, 1, 1, 1, full_recomp=True)   # 1F1B + full recompute, v = 1
    if p > 2:                                          # stage 1 is a middle stage
        assert full["stash"] == (L // p) * act - act
    else:                                              # stage 1 holds the head
        assert full["stash"] == (L // p) * act - act + act + b * s * 12
    assert mid["act"] == act


def test_model_state_bytes_per_param():
    d = desc(64, 4, 32, 2)
    assert T.model_state_bytes(d, 1000, offloaded=False) == 18 * 1000
    assert T.model_state_bytes(d, 1000, offloaded=True) == 6 * 1000
    d32 = desc(64, 4, 32, 2, dtype=T.FP32)
    assert T.model_state_bytes(d32, 1000, offloaded=False) == 16 * 1000   # fp32 w is the master


@pytest.mark.parametrize("h,a,s,b", SHAPES)
def test_workspace_lower_bounds(h, a, s, b):
    """A layer backward must hold at once: dy and dx (2·M·h), the FC1
    pre-activation gradient and GELU(u) (2·M·f), one recomputed LN output
    and its gradient (2·M·h), the attention-output gradient (M·h) and dqkv
    (3·M·h) plus D = rowsum(dO∘O) (4·a·M); the forward a LN output (M·h) and
    GELU output (M·f). The head chunk's backward additionally holds the
    logits' gradient (es·M·V; the bf16 fused head never stores the logits,
    DESIGN R30) plus, in fp32 mode, the fp32 logits (4·M·V)."""
    d = desc(h, a, s, b, L=8)
    M, f, V = b * s, 4 * h, d.vocab
    z = T.sizes(d, 4, 2, 1, 1)
    assert z["ws_b"] >= 2 * (2 * M * h + 2 * M * f + 2 * M * h + M * h + 3 * M * h) + 4 * a * M
    assert z["ws_f"] >= 2 * (M * h + M * f)
    zh = T.sizes(d, 4, 2, 3, 2)
    assert zh["ws_b"] - z["ws_b"] >= 2 * M * V
    # no fp32 [M, V] logits in bf16 (R30): below the unfused 4·M·V + 2·M·V
    assert zh["ws_b"] - z["ws_b"] < 6 * M * V
    d32 = desc(h, a, s, b, L=8, dtype=T.FP32)
    assert T.sizes(d32, 4, 2, 3, 2)["ws_b"] - T.sizes(d32, 4, 2, 1, 1)["ws_b"] >= 8 * M * V
