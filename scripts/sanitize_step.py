"""One training step through the C-ABI for compute-sanitizer runs
(memcheck / racecheck / synccheck). No torch import: only libtpipe.so's
kernels run under the tool.

    compute-sanitizer --tool memcheck python scripts/sanitize_step.py CFG STRATEGY OFFLOAD DTYPE P M [CHUNKS] [R]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2503_03182_b200 import params as PR, plan as P, runtime as RT  # noqa: E402

CFGS = {"c1": dict(L=8, h=64, a=4, f=256, V=256, s=32, b=2),
        "cmid": dict(L=4, h=256, a=2, f=1024, V=512, s=256, b=1),
        "cmid12": dict(L=12, h=256, a=2, f=1024, V=512, s=256, b=1)}


def main(cfg="c1", strategy="tpipe_trecomp", offload="0", dtype="1", p="2", m="4", chunks="2", r="0"):
    c = CFGS[cfg]
    p, m, offload, dtype, chunks, r = int(p), int(m), int(offload), int(dtype), int(chunks), int(r)
    plan = P.Plan(P.Model(c["L"], c["h"], c["a"], c["f"], c["V"], c["s"], c["b"], dtype), p, m,
                  strategy=strategy, offload=offload, chunks=chunks, recomp_layers=r)
    rt = RT.Runtime(plan, stage=-1, lr=1e-3)
    W = synth.weights(c["L"], c["h"], c["f"], c["V"], c["s"], seed=5, std=0.05, bias_std=0.02,
                      ln_jitter=0.05)
    for s in range(p):
        for ch in range(1, plan.v + 1):
            rt.set_params(s, ch, PR.pack(W, p, plan.v, plan.partition, s, ch))
    tok, tgt = synth.tokens(c["V"], m, c["b"], c["s"], step=0)
    loss = rt.step(tok, tgt, 0)
    print(f"sanitize_step {cfg} {strategy} offload={offload} dtype={dtype} p={p} m={m} loss={loss:.6f} "
          f"launches={rt.stats()['kernel_launches']}")
    rt.close()


if __name__ == "__main__":
    main(*sys.argv[1:])
