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
gemm_case("sq8192", 8192, 8192, 8192, 1, 1, K.EPI_STORE)
for o in out:
    print(json.dumps(o))
