"""TPipe CPU oracle — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA
path is checked against. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2503_03182_b200``) never imports it, and it never
imports the product path. The only module both sides share is ``synth``
(seeded input generation, no method arithmetic).

Parts
-----
``oracle.schedule``  Part 1: exact integer unit-time schedule simulator
                     (T-Pipe, T-Recomp, 1F1B, 1F1B+recompute, Interleave-1F1B),
                     channel FIFO / send-window model, block-level memory replay.
``oracle.stream``    Part 1 bytes: per-stage instruction streams with SEND/RECV
                     and offload instructions, byte-exact live-set replay.
``oracle.model``     Part 2: fp64 NumPy forward/backward of the pre-LN GPT block
                     stack + AdamW, schedule-free (sums microbatches in index order).

Citations: ``P:n`` = PAPER.md line n (arxiv 2503.03182 LaTeX source);
``S:n`` = SPEC.md line n; ``D-x`` = SURVEY.md derived results.
"""
