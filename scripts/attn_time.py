"""Time the tcgen05 attention kernels over several shapes (CUDA events, warm):
python scripts/attn_time.py [--lib libtpipe_variant.so] [b,s,a,d ...]   e.g. 1,2048,16,128 4,4096,16,128"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import _lib
if len(sys.argv) > 2 and sys.argv[1] == "--lib":   # time a variant build of the library
    _lib.LIB_PATH = os.path.abspath(sys.argv[2])
    del sys.argv[1:3]
from paper_2503_03182_b200 import kernels as K

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or \
    [(1, 2048, 16, 128), (4, 2048, 16, 128), (1, 8192, 16, 128), (1, 4096, 32, 128), (2, 2048, 32, 64)]


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for b, s, a, d in shapes:
    h = a * d
    qkv = (torch.randn((b * s, 3 * h), device="cuda") * 0.5).to(torch.bfloat16)
    o = torch.empty((b * s, h), device="cuda", dtype=torch.bfloat16)
    lse = torch.empty((b, a, s), device="cuda")
    dout = torch.randn((b * s, h), device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty((b, a, s), device="cuda")
    ffl = 4.0 * b * a * (s * (s + 1) / 2) * d
    mf = timeit(lambda: K.tpipe_k_attn_fwd(1, qkv, o, lse, b, s, a, d))
    mb = timeit(lambda: K.tpipe_k_attn_bwd(1, qkv, o, dout, lse, dqkv, ws, b, s, a, d))
    print(json.dumps(dict(b=b, s=s, heads=a, d=d, fwd_ms=round(mf, 4), fwd_tflops=round(ffl / mf / 1e9, 1),
                          bwd_ms=round(mb, 4), bwd_tflops=round(2.5 * ffl / mb / 1e9, 1))), flush=True)
