"""Our tcgen05 GEMM vs cuBLAS (torch.matmul, bf16 in / bf16 out, fp32 accumulate)
on the GEMM shapes of one GPT-3 1.3B layer + LM head, same operand majors;
20 launches captured in one CUDA graph each, CUDA-event-timed replay.
Our kernel runs its production epilogue (bias / GELU / dGELU / residual /
fp32 reduce-add), cuBLAS a plain store, so cuBLAS does strictly less work.
python scripts/gemm_vs_cublas.py > gpurun_out/gemm_vs_cublas.jsonl"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import kernels as K

h, s, f, V = 2048, 2048, 8192, 50304
M = s
E = K
shapes = [("qkv_fprop", M, 3 * h, h, 1, 1, E.EPI_BIAS), ("o_fprop", M, h, h, 1, 1, E.EPI_BIAS_RES),
          ("fc1_fprop", M, f, h, 1, 1, E.EPI_BIAS_GELU), ("fc2_fprop", M, h, f, 1, 1, E.EPI_BIAS_RES),
          ("fc2_dgrad", M, f, h, 1, 0, E.EPI_DGELU), ("fc2_wgrad", h, f, M, 0, 0, E.EPI_ACC_F32),
          ("fc1_wgrad", f, h, M, 0, 0, E.EPI_ACC_F32), ("fc1_dgrad", M, h, f, 1, 0, E.EPI_STORE),
          ("o_wgrad", h, h, M, 0, 0, E.EPI_ACC_F32), ("o_dgrad", M, h, h, 1, 0, E.EPI_STORE),
          ("qkv_wgrad", 3 * h, h, M, 0, 0, E.EPI_ACC_F32), ("qkv_dgrad", M, h, 3 * h, 1, 0, E.EPI_STORE),
          ("head_fprop", M, V, h, 1, 1, E.EPI_STORE_F32), ("head_dgrad", M, h, V, 1, 0, E.EPI_STORE),
          ("head_wgrad", V, h, M, 0, 0, E.EPI_ACC_F32), ("sq8192", 8192, 8192, 8192, 1, 1, E.EPI_STORE)]


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(iters):
                fn()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    tot = [0.0, 0.0]
    for name, m, n, k, ak, bk, epi in shapes:
        A = torch.randn((m, k) if ak else (k, m), device="cuda").to(torch.bfloat16)
        B = torch.randn((n, k) if bk else (k, n), device="cuda").to(torch.bfloat16)
        f32 = epi in (E.EPI_ACC_F32, E.EPI_STORE_F32)
        C = torch.zeros((m, n), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
        C2 = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
        Rr = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
        bias = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
        ours = lambda: K.tpipe_k_gemm(1, m, n, k, A, k if ak else m, ak, B, k if bk else n, bk, epi, C, n,
                                      bias=bias, R=Rr, ldr=n, C2=C2, ldc2=n, aux=Rr, ldaux=n)
        Am = A if ak else A.t()          # logical [m, k]
        Bm = B.t() if bk else B          # logical [k, n]
        Cb = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
        cub = lambda: torch.matmul(Am, Bm, out=Cb)
        t0, t1 = timed(ours), timed(cub)
        if name != "sq8192":
            tot[0] += t0
            tot[1] += t1
        fl = 2 * m * n * k
        print(json.dumps({"kernel": name, "M": m, "N": n, "K": k, "ours_us": round(t0 * 1e3, 2),
                          "ours_tflops": round(fl / t0 / 1e9, 1), "cublas_us": round(t1 * 1e3, 2),
                          "cublas_tflops": round(fl / t1 / 1e9, 1), "ours_over_cublas": round(t1 / t0, 3)}),
              flush=True)
        del A, B, C, C2, Rr, Cb
    print(json.dumps({"layer_plus_head_total_ms": {"ours": round(tot[0], 4), "cublas": round(tot[1], 4),
                                                   "ours_speed_vs_cublas": round(tot[1] / tot[0], 3)}}))


if __name__ == "__main__":
    main()
