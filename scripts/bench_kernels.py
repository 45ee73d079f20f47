"""Micro-benchmark of the stage-executor kernels at the C2/C3 shapes
(CUDA events on torch's current stream, after warm-up). Prints one line per
kernel: shape, ms, TFLOP/s or GB/s."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import kernels as K

dev = "cuda"
out = []


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


def gemm_case(name, M, N, Kd, ak, bk, epi):
    A = torch.randn((M, Kd) if ak else (Kd, M), device=dev).to(torch.bfloat16)
    B = torch.randn((N, Kd) if bk else (Kd, N), device=dev).to(torch.bfloat16)
    f32 = epi in (K.EPI_ACC_F32, K.EPI_STORE_F32)
    C = torch.zeros((M, N), device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
    bias = torch.zeros(N, device=dev, dtype=torch.bfloat16)
    fn = lambda: K.tpipe_k_gemm(1, M, N, Kd, A, Kd if ak else M, ak, B, Kd if bk else N, bk, epi, C, N, bias=bias)
    ms = timeit(fn)
    tf = 2 * M * N * Kd / ms / 1e9
    out.append(dict(kernel="gemm_" + name, M=M, N=N, K=Kd, ms=round(ms, 4), tflops=round(tf, 1)))


h, s, f = 2048, 2048, 8192
if len(sys.argv) > 1 and sys.argv[1] == "c3":
    h, s, f = 4096, 4096, 16384
M = s
gemm_case("qkv_fprop", M, 3 * h, h, 1, 1, K.EPI_BIAS)
gemm_case("fc1_fprop", M, f, h, 1, 1, K.EPI_BIAS)
gemm_case("fc2_fprop", M, h, f, 1, 1, K.EPI_BIAS)
gemm_case("fc1_dgrad", M, h, f, 1, 0, K.EPI_STORE)
gemm_case("fc2_dgrad", M, f, h, 1, 0, K.EPI_STORE)
gemm_case("fc1_wgrad", f, h, M, 0, 0, K.EPI_ACC_F32)
gemm_case("qkv_wgrad", 3 * h, h, M, 0, 0, K.EPI_ACC_F32)
gemm_case("o_fprop", M, h, h, 1, 1, K.EPI_BIAS)
gemm_case("o_wgrad", h, h, M, 0, 0, K.EPI_ACC_F32)
V = 50304 if h == 2048 else 32000
gemm_case("head_fprop", M, V, h, 1, 1, K.EPI_STORE_F32)
gemm_case("head_dgrad", M, h, V, 1, 0, K.EPI_STORE)
gemm_case("head_wgrad", V, h, M, 0, 0, K.EPI_ACC_F32)
gemm_case("sq8192", 8192, 8192, 8192, 1, 1, K.EPI_STORE)
for ak, bk in ((1, 1), (1, 0), (0, 0), (0, 1)):
    gemm_case(f"sq4096_maj{ak}{bk}_f32", 4096, 4096, 4096, ak, bk, K.EPI_STORE_F32)
    gemm_case(f"sq4096_maj{ak}{bk}_acc", 4096, 4096, 4096, ak, bk, K.EPI_ACC_F32)
    gemm_case(f"sq4096_maj{ak}{bk}_bf16", 4096, 4096, 4096, ak, bk, K.EPI_STORE)
for o in out:
    print(json.dumps(o))

# attention at the C2 / C3 shape (tcgen05)
b, a, d = 1, h // 128, 128
qkv = (torch.randn((b * s, 3 * h), device=dev) * 0.5).to(torch.bfloat16)
o = torch.empty((b * s, h), device=dev, dtype=torch.bfloat16)
lse = torch.empty((b, a, s), device=dev)
dout = torch.randn((b * s, h), device=dev).to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
ws = torch.empty((b, a, s), device=dev)
ffl = 4.0 * b * a * (s * (s + 1) / 2) * d
for name, f_fwd, f_bwd in (("tcgen05", lambda: K.tpipe_k_attn_fwd(1, qkv, o, lse, b, s, a, d),
                            lambda: K.tpipe_k_attn_bwd(1, qkv, o, dout, lse, dqkv, ws, b, s, a, d)),):
    ms = timeit(f_fwd)
    print(json.dumps(dict(kernel=f"attn_fwd_{name}", s=s, heads=a, d=d, ms=round(ms, 4),
                          tflops=round(ffl / ms / 1e9, 1))))
    ms = timeit(f_bwd)
    print(json.dumps(dict(kernel=f"attn_bwd_{name}", s=s, heads=a, d=d, ms=round(ms, 4),
                          tflops=round(2.5 * ffl / ms / 1e9, 1))))
