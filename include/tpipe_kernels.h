/*
 * tpipe_kernels.h — kernel-level entry points of libtpipe.so (C-ABI).
 *
 * These expose the individual sm_100a kernels of the stage executor so that
 * each can be checked element by element against the fp64 oracle
 * (tests/test_gpu_kernels.py). The training step itself is driven through
 * include/tpipe.h (tpipe_plan_* / tpipe_runtime_* / tpipe_step).
 *
 * Conventions (all functions):
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *     the caller owns all memory; nothing is retained after return;
 *   - `dtype` is TPIPE_FP32 (0) or TPIPE_BF16 (1) and gives the element type
 *     of the activation/weight tensors ("es" below); statistics, LSE, losses
 *     and gradient accumulators are always fp32;
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default);
 *     calls are asynchronous;
 *   - return 0 on success, a negative TPIPE_E_* code on invalid arguments or
 *     launch failure (tpipe_last_error() gives the message).
 *
 * Citations: P:n = PAPER.md line n (arxiv 2503.03182). The paper gives no
 * model equations; the operations follow the readings in DESIGN.md §2
 * (SURVEY §8(c) N-1..N-4): pre-LN GPT block, FlashAttention,
 * operator-level recompute.
 */
#ifndef TPIPE_KERNELS_H
#define TPIPE_KERNELS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM  C = A * B^T (+ epilogue), A logical [M,K], B logical [N,K].
 * A[m,k] = a_kmajor ? A[m*lda + k] : A[k*lda + m]; likewise B with b_kmajor.
 * epi: 0 C=acc | 1 C=acc+bias | 2 C=acc+bias+R | 3 C=u=acc+bias, C2=gelu(u)
 *      | 4 C=acc*gelu'(U), C2=gelu(U) (U = aux) | 5 Cf32 += acc | 6 Cf32 = acc.
 * bf16 runs on tcgen05 tensor cores (requires N % 32 == 0, lda, ldb % 8 == 0);
 * fp32 runs an exact fp32 SIMT kernel. Row strides in elements. */
int tpipe_k_gemm(int dtype, int M, int N, int K,
                 const void* A, long lda, int a_kmajor,
                 const void* B, long ldb, int b_kmajor,
                 int epi, void* C, long ldc, const void* bias,
                 const void* R, long ldr, void* C2, long ldc2,
                 const void* aux, long ldaux, void* stream);

/* bf16 GEMM with the attention-backward row statistic fused into its
 * epilogue (the out-projection data gradient): C = dO = A * B^T (bf16, ldc);
 * Dout[(b*a + head)*s + q] = sum_{e < hd} C[m, head*hd + e] * O[m, head*hd + e]
 * (fp32, the stored bf16 C times O, in column order) for m = b*s + q,
 * a = N / hd heads. hd in {64, 128}, N % hd == 0, M % s == 0, ldo % 8 == 0.
 * Dout is the D = rowsum(dO o O) of the attention backward (P:461,
 * FlashAttention), so tpipe_k_attn_bwd's D pass can be skipped. */
int tpipe_k_gemm_dot(int M, int N, int K, const void* A, long lda, int a_kmajor,
                     const void* B, long ldb, int b_kmajor, void* C, long ldc,
                     const void* O, long ldo, float* Dout, int s, int hd, void* stream);

/* Same contract, always the SIMT kernel (used as the fp32-mode path). */
int tpipe_k_gemm_simt(int dtype, int M, int N, int K,
                      const void* A, long lda, int a_kmajor,
                      const void* B, long ldb, int b_kmajor,
                      int epi, void* C, long ldc, const void* bias,
                      const void* R, long ldr, void* C2, long ldc2,
                      const void* aux, long ldaux, void* stream);

/* Enable (1, default) or disable (0) CTA-pair tiles in the tcgen05 GEMM
 * (process-wide; for A/B measurement): a cluster of two CTAs on one TPC
 * computes a 256 x 256 tile with tcgen05.mma.cta_group::2, each CTA staging
 * half of the A and B operands. Used when the shape yields >= 32 such tiles. */
void tpipe_k_gemm_set_pair(int on);
/* CTA-pair 256 x 256 tiles once a GEMM has >= n of them (default 96; A/B knob) */
void tpipe_k_gemm_set_pair_min_tiles(int n);
/* Enable (1, default) or disable (0) the 240 / 224-column tile widths: for a
 * K-major B operand the GEMM picks, per shape, the width in {256, 240, 224}
 * with the fewest waves x width over the 148 SMs (74 CTA pairs); 0 = always
 * 256 (A/B knob). */
void tpipe_k_gemm_set_wide_choice(int on);
/* Enable (1, default) or disable (0) the row-parallel LayerNorm backward
 * kernel for bf16 h <= 2048 (0 = the staged kernel; process-wide A/B knob). */
void tpipe_k_ln_set_rows_bwd(int on);

/* LayerNorm forward over rows of length h (eps 1e-5, biased variance):
 * y = (x-mean)*rstd*gamma + beta; mean/rstd fp32 [rows]. */
int tpipe_k_ln_fwd(int dtype, const void* x, const void* gamma, const void* beta,
                   void* y, float* mean, float* rstd, int rows, int h, void* stream);

/* LayerNorm backward: dx = resid + dLN(dy) (resid may be NULL);
 * dgamma/dbeta (fp32 [h]) are ACCUMULATED (+=) deterministically.
 * ws: fp32 scratch of 2*ceil(rows/16)*h elements. */
int tpipe_k_ln_bwd(int dtype, const void* dy, const void* x, const void* gamma,
                   const float* mean, const float* rstd, const void* resid, void* dx,
                   float* dgamma, float* dbeta, float* ws, int rows, int h, void* stream);

/* tpipe_k_ln_bwd plus dresid_sum[h] += column sums of resid (required, with
 * resid): in a pre-LN block the gradient entering LN's residual branch is also
 * the output gradient of the preceding linear, so its bias gradient is fused
 * here (one pass over resid instead of two). ws: fp32 scratch of
 * 3*ceil(rows/16)*h elements. */
int tpipe_k_ln_bwd_rsum(int dtype, const void* dy, const void* x, const void* gamma,
                        const float* mean, const float* rstd, const void* resid, void* dx,
                        float* dgamma, float* dbeta, float* dresid_sum, float* ws, int rows,
                        int h, void* stream);

/* The layer backward's form of the LN backward (bf16, h % 256 == 0): dx as
 * in tpipe_k_ln_bwd (+ resid) and, instead of reduced dgamma / dbeta /
 * dresid_sum, the per-16-row-block column partials ws[3][ceil(rows/16)][h]
 * (fp32; the layer backward reduces them together with its bias-gradient
 * partials in one launch). with_rsum: the third partial. */
int tpipe_k_ln_bwd_partials(const void* dy, const void* x, const void* gamma, const float* mean,
                            const float* rstd, const void* resid, void* dx, float* ws, int rows, int h,
                            int with_rsum, void* stream);

/* Causal attention forward. qkv [b*s, 3h] (q|k|v, head j at columns j*d),
 * o [b*s, h], lse fp32 [b, a, s]; h = a*d, scale 1/sqrt(d). */
int tpipe_k_attn_fwd(int dtype, const void* qkv, void* o, float* lse,
                     int b, int s, int a, int d, void* stream);

/* Causal attention backward (recomputes P from lse; deterministic, no atomics).
 * dout [b*s, h]; dqkv [b*s, 3h]; ws fp32 [b*a*s]. */
int tpipe_k_attn_bwd(int dtype, const void* qkv, const void* o, const void* dout,
                     const float* lse, void* dqkv, float* ws,
                     int b, int s, int a, int d, void* stream);


/* Embedding: x[r] = wte[tok[r]] + wpe[r mod s]; tok int32 [rows]. */
int tpipe_k_embed_fwd(int dtype, const int* tok, const void* wte, const void* wpe,
                      void* x, int rows, int s, int h, void* stream);

/* Embedding backward, deterministic (rows sorted by (token, row)):
 * dwte[tok[r]] += dx[r], dwpe[r mod s] += dx[r] (fp32 accumulators).
 * ws: int32 scratch of 2*rows elements. rows <= 32768, vocab < 131072. */
int tpipe_k_embed_bwd(int dtype, const int* tok, const void* dx, float* dwte, float* dwpe,
                      int* ws, int rows, int s, int h, void* stream);

/* Cross-entropy forward on fp32 logits [rows, V]: lse[r] = logsumexp(logits[r]);
 * loss_out[0] += scale * sum_r (lse[r] - logits[r, tgt[r]]) in row order. */
int tpipe_k_ce_fwd(const float* logits, const int* tgt, float* lse, float* loss_out,
                   float scale, int rows, int V, void* stream);

/* dlogits (es) [rows, V] = scale * (exp(logits - lse) - onehot(tgt)). */
int tpipe_k_ce_bwd(int dtype, const float* logits, const int* tgt, const float* lse,
                   void* dlogits, float scale, int rows, int V, void* stream);

/* Fused LM head + softmax cross-entropy (K8, DESIGN R30), bf16, tcgen05:
 * logits z = x · W^T (x [rows, h] bf16 row-major, W [V, h] bf16 row-major)
 * are never written to HBM. Pass 1 (head GEMM, epilogue) -> per row and
 * 64-column group (max, sum exp(z - max)) + z[r, tgt[r]]; combine ->
 * lse[r] (fp32) and loss_out[0] += scale * sum_r (lse[r] - z[r, tgt[r]]) in
 * row order; pass 2 (head GEMM again) -> dlogits [rows, V] bf16 =
 * scale * (exp(z - lse) - onehot(tgt)). ws: fp32 scratch of
 * 2*rows*ceil(V/64) + 2*rows floats. V % 64 == 0, h % 64 == 0. */
int tpipe_k_head_ce(const void* x, const void* w, const int* tgt, float* lse, void* dlogits,
                    float* loss_out, float scale, int rows, int V, int h, float* ws, void* stream);

/* out[n] += sum_r X[r, n] (fp32, deterministic). ws fp32 [ceil(rows/16)*n]. */
int tpipe_k_colsum(int dtype, const void* X, float* out, float* ws, int rows, int n,
                   void* stream);

/* AdamW (torch.optim.AdamW semantics, DESIGN.md §2 N-3) on fp32 master/m/v with
 * fp32 grad; writes the es weight copy w (bf16: RNE of master; fp32: w may
 * alias master) and ZEROES grad. bc1 = 1-b1^t, bc2 = 1-b2^t (caller, host). */
int tpipe_k_adamw(int dtype, float* master, float* m, float* v, float* grad, void* w,
                  long n, int decay, float lr, float b1, float b2, float eps, float wd,
                  float bc1, float bc2, void* stream);

/* HOST implementation of the same AdamW arithmetic, bit-identical to
 * tpipe_k_adamw (T-Offload host optimizer). All pointers are HOST
 * pointers; w_bf16 may be NULL. Does not touch grad. */
void tpipe_host_adamw(float* master, float* m, float* v, const float* grad,
                      uint16_t* w_bf16, long n, int decay, float lr, float b1,
                      float b2, float eps, float wd, float bc1, float bc2);

#ifdef __cplusplus
}
#endif
#endif /* TPIPE_KERNELS_H */
