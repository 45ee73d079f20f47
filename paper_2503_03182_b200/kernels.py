"""Thin wrappers over the kernel-level C-ABI (include/tpipe_kernels.h).
Arguments are torch CUDA tensors (device memory) or plain ints; each call
forwards pointers/sizes to libtpipe.so on torch's current stream."""

from __future__ import annotations

from ._lib import check, lib

FP32, BF16 = 0, 1

EPI_STORE, EPI_BIAS, EPI_BIAS_RES, EPI_BIAS_GELU, EPI_DGELU, EPI_ACC_F32, EPI_STORE_F32 = range(7)


def _p(t):
    if t is None:
        return None
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def tpipe_k_gemm(dtype, M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, epi, C, ldc, bias=None,
                 R=None, ldr=0, C2=None, ldc2=0, aux=None, ldaux=0, simt=False):
    fn = lib().tpipe_k_gemm_simt if simt else lib().tpipe_k_gemm
    check(fn(dtype, M, N, K, _p(A), lda, a_kmajor, _p(B), ldb, b_kmajor, epi, _p(C), ldc, _p(bias),
             _p(R), ldr, _p(C2), ldc2, _p(aux), ldaux, _stream()), "tpipe_k_gemm")


def tpipe_k_gemm_dot(M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, C, ldc, O, ldo, Dout, s, hd):
    check(lib().tpipe_k_gemm_dot(M, N, K, _p(A), lda, a_kmajor, _p(B), ldb, b_kmajor, _p(C), ldc, _p(O), ldo,
                                 _p(Dout), s, hd, _stream()), "tpipe_k_gemm_dot")


def tpipe_k_ln_fwd(dtype, x, g, b, y, mean, rstd, rows, h):
    check(lib().tpipe_k_ln_fwd(dtype, _p(x), _p(g), _p(b), _p(y), _p(mean), _p(rstd), rows, h,
                               _stream()), "ln_fwd")


def tpipe_k_ln_bwd(dtype, dy, x, g, mean, rstd, resid, dx, dg, db, ws, rows, h):
    check(lib().tpipe_k_ln_bwd(dtype, _p(dy), _p(x), _p(g), _p(mean), _p(rstd), _p(resid), _p(dx),
                               _p(dg), _p(db), _p(ws), rows, h, _stream()), "ln_bwd")


def tpipe_k_ln_bwd_partials(dy, x, g, mean, rstd, resid, dx, ws, rows, h, with_rsum=1):
    check(lib().tpipe_k_ln_bwd_partials(_p(dy), _p(x), _p(g), _p(mean), _p(rstd), _p(resid), _p(dx), _p(ws),
                                        rows, h, 1 if with_rsum else 0, _stream()), "ln_bwd_partials")


def tpipe_k_ln_bwd_rsum(dtype, dy, x, g, mean, rstd, resid, dx, dg, db, drs, ws, rows, h):
    check(lib().tpipe_k_ln_bwd_rsum(dtype, _p(dy), _p(x), _p(g), _p(mean), _p(rstd), _p(resid),
                                    _p(dx), _p(dg), _p(db), _p(drs), _p(ws), rows, h, _stream()),
          "ln_bwd_rsum")


def tpipe_k_attn_fwd(dtype, qkv, o, lse, b, s, a, d):
    check(lib().tpipe_k_attn_fwd(dtype, _p(qkv), _p(o), _p(lse), b, s, a, d, _stream()), "attn_fwd")


def tpipe_k_attn_bwd(dtype, qkv, o, dout, lse, dqkv, ws, b, s, a, d):
    check(lib().tpipe_k_attn_bwd(dtype, _p(qkv), _p(o), _p(dout), _p(lse), _p(dqkv), _p(ws), b, s,
                                 a, d, _stream()), "attn_bwd")


def tpipe_k_embed_fwd(dtype, tok, wte, wpe, x, rows, s, h):
    check(lib().tpipe_k_embed_fwd(dtype, _p(tok), _p(wte), _p(wpe), _p(x), rows, s, h, _stream()),
          "embed_fwd")


def tpipe_k_embed_bwd(dtype, tok, dx, dwte, dwpe, ws, rows, s, h):
    check(lib().tpipe_k_embed_bwd(dtype, _p(tok), _p(dx), _p(dwte), _p(dwpe), _p(ws), rows, s, h,
                                  _stream()), "embed_bwd")


def tpipe_k_ce_fwd(logits, tgt, lse, loss, scale, rows, V):
    check(lib().tpipe_k_ce_fwd(_p(logits), _p(tgt), _p(lse), _p(loss), scale, rows, V, _stream()),
          "ce_fwd")


def tpipe_k_head_ce(x, w, tgt, lse, dlogits, loss, scale, rows, V, h, ws):
    check(lib().tpipe_k_head_ce(_p(x), _p(w), _p(tgt), _p(lse), _p(dlogits), _p(loss), scale, rows, V,
                                h, _p(ws), _stream()), "tpipe_k_head_ce")


def tpipe_k_ce_bwd(dtype, logits, tgt, lse, dlogits, scale, rows, V):
    check(lib().tpipe_k_ce_bwd(dtype, _p(logits), _p(tgt), _p(lse), _p(dlogits), scale, rows, V,
                               _stream()), "ce_bwd")


def tpipe_k_colsum(dtype, X, out, ws, rows, n):
    check(lib().tpipe_k_colsum(dtype, _p(X), _p(out), _p(ws), rows, n, _stream()), "colsum")


def tpipe_k_adamw(dtype, master, m, v, grad, w, n, decay, lr, b1, b2, eps, wd, bc1, bc2):
    check(lib().tpipe_k_adamw(dtype, _p(master), _p(m), _p(v), _p(grad), _p(w), n, decay, lr, b1,
                              b2, eps, wd, bc1, bc2, _stream()), "adamw")


def tpipe_host_adamw(master, m, v, grad, w_bf16, n, decay, lr, b1, b2, eps, wd, bc1, bc2):
    """numpy arrays (host)."""
    ptr = (lambda a: None if a is None else a.ctypes.data)
    lib().tpipe_host_adamw(ptr(master), ptr(m), ptr(v), ptr(grad), ptr(w_bf16), n, decay, lr, b1,
                           b2, eps, wd, bc1, bc2)


def tpipe_k_gemm_set_pair(on):
    lib().tpipe_k_gemm_set_pair(1 if on else 0)


def tpipe_k_gemm_set_wide_choice(on):
    lib().tpipe_k_gemm_set_wide_choice(1 if on else 0)


def tpipe_k_ln_set_rows_bwd(on):
    lib().tpipe_k_ln_set_rows_bwd(1 if on else 0)
