// Internal kernel launchers (not part of the C-ABI; see include/tpipe.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tpipe {

enum DType : int { DT_FP32 = 0, DT_BF16 = 1 };

// GEMM epilogues. C = A * B^T with A logical [M,K], B logical [N,K], fp32 accumulate.
enum Epi : int {
    EPI_STORE = 0,      // C(es)  = acc
    EPI_BIAS = 1,       // C(es)  = acc + bias[n]
    EPI_BIAS_RES = 2,   // C(es)  = acc + bias[n] + R[m,n]
    EPI_BIAS_GELU = 3,  // C(es)  = u = acc + bias[n];  C2(es) = gelu(rnd(u))
    EPI_DGELU = 4,      // C(es)  = acc * gelu'(U[m,n]); C2(es) = gelu(U[m,n])
    EPI_ACC_F32 = 5,    // Cf32  += acc
    EPI_STORE_F32 = 6,  // Cf32   = acc
    // fused LM head + softmax cross-entropy (K8, DESIGN R30; tcgen05 path only).
    // The logits z = acc never reach HBM:
    EPI_LSE_PART = 7,   // part[m][n/64] = (max, sum exp(z - max)) over each 64-column
                        // group; zt[m] = z[m, targets[m]]; no C store
    EPI_CE_GRAD = 8,    // C(bf16) = (exp(z - lse[m]) - [n == targets[m]]) * scale
    // attention-output gradient with the backward's row statistic (tcgen05 path
    // only): C(bf16) = dO = acc; part[(b*a + head)*s + q] = sum over the head's
    // dot_hd columns of dO[m, .] * aux[m, .] (= O), fp32, column order, for
    // m = b*s + q (the attention backward's D = rowsum(dO o O))
    EPI_STORE_DOT = 9,
};

struct GemmDesc {
    int M = 0, N = 0, K = 0;
    const void* A = nullptr; long lda = 0; int a_kmajor = 1;  // A[m,k] = kmajor ? A[m*lda+k] : A[k*lda+m]
    const void* B = nullptr; long ldb = 0; int b_kmajor = 1;  // B[n,k] = kmajor ? B[n*ldb+k] : B[k*ldb+n]
    int epi = EPI_STORE;
    void* C = nullptr; long ldc = 0;
    const void* bias = nullptr;
    const void* res = nullptr; long ldr = 0;
    void* C2 = nullptr; long ldc2 = 0;
    const void* aux = nullptr; long ldaux = 0;
    // EPI_LSE_PART / EPI_CE_GRAD
    const int* targets = nullptr;
    const float* lse = nullptr;
    float* part = nullptr;     // [M][ceil(N/64)][2]
    float* zt = nullptr;       // [M]
    float scale = 0.f;
    // EPI_STORE_DOT: sequence length and head dim (N = heads * dot_hd)
    int dot_s = 0, dot_hd = 0;
};

// 64-column groups of the fused head's LSE partials (the narrowest column span
// one epilogue thread owns: BN = 128 split over two 4-warp groups)
inline int ce_groups(int V) { return (V + 63) / 64; }

// dtype DT_BF16 -> tcgen05/TMA tensor-core kernel; DT_FP32 -> exact fp32 SIMT kernel.
int gemm(int dtype, const GemmDesc& g, cudaStream_t st);
// Plain SIMT kernel for either dtype (fp32 arithmetic); used for fp32 mode.
int gemm_simt(int dtype, const GemmDesc& g, cudaStream_t st);
// tcgen05 kernel (bf16 only).
int gemm_tc(const GemmDesc& g, cudaStream_t st);
// CTA-pair (cta_group::2) 256-row tiles on/off (default on)
void gemm_set_pair(int on);
// pair tiles from n 256 x 256 tiles on (default 96)
void gemm_set_pair_min_tiles(int n);
void gemm_set_wide_choice(int on);
void ln_set_rows_bwd(int on);

// ---------------------------------------------------------------- layernorm
// y = (x - mean) * rstd * gamma + beta over rows of length h; saves mean/rstd (fp32).
int ln_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y, float* mean,
           float* rstd, int rows, int h, cudaStream_t st);
// y from saved stats (operator-level recompute); bit-identical to ln_fwd's y.
int ln_apply(int dtype, const void* x, const void* gamma, const void* beta, const float* mean,
             const float* rstd, void* y, int rows, int h, cudaStream_t st);
// dx = resid + LN_bwd(dy); dgamma/dbeta partials per 16-row block into ws (fp32
// [2][nblk][h], [3][nblk][h] with dresid_sum), then reduced in a fixed order and
// ADDED to dgamma/dbeta (fp32). dresid_sum (optional, needs resid): += column
// sums of resid (the bias gradient of the linear whose output gradient resid is).
int ln_bwd(int dtype, const void* dy, const void* x, const void* gamma, const float* mean,
           const float* rstd, const void* resid, void* dx, float* dgamma, float* dbeta, float* ws,
           int rows, int h, cudaStream_t st, float* dresid_sum = nullptr);

// ---------------------------------------------------------------- attention
// qkv: [b*s, 3h] (q | k | v, head j = cols j*d..), o: [b*s, h], lse: [b, a, s] fp32.
int attn_fwd(int dtype, const void* qkv, void* o, float* lse, int b, int s, int a, int d,
             cudaStream_t st);
// dqkv: [b*s, 3h]; ws: fp32 [b, a, s] for D = rowsum(dO * O).
// have_d: ws already holds D (written by the out-projection dgrad GEMM's
// EPI_STORE_DOT epilogue); the tcgen05 path then skips its D kernel.
int attn_bwd(int dtype, const void* qkv, const void* o, const void* dout, const float* lse,
             void* dqkv, float* ws, int b, int s, int a, int d, cudaStream_t st, bool have_d = false);


// ---------------------------------------------------------------- embedding
// x[r] = wte[tok[r]] + wpe[r % s]
int embed_fwd(int dtype, const int* tok, const void* wte, const void* wpe, void* x, int rows,
              int s, int h, cudaStream_t st);
// dwte[tok] += dx rows (deterministic: sort by (token, row)); dwpe[t] += sum_b dx[b*s+t].
// ws: int32 [2*rows].
int embed_bwd(int dtype, const int* tok, const void* dx, float* dwte, float* dwpe, int* ws,
              int rows, int s, int h, cudaStream_t st);

// ---------------------------------------------------------------- cross entropy
// logits fp32 [rows, V]; loss_out[0] += sum_r (lse_r - logit[r, tgt_r]) * scale (fixed order);
// lse fp32 [rows].
int ce_fwd(const float* logits, const int* tgt, float* lse, float* loss_out, float scale, int rows,
           int V, cudaStream_t st);
// dlogits(es) [rows, V] = (exp(logit - lse) - onehot) * scale
int ce_bwd(int dtype, const float* logits, const int* tgt, const float* lse, void* dlogits,
           float scale, int rows, int V, cudaStream_t st);
// fused LM head + CE (K8, DESIGN R30): combine the head GEMM's per-128-column
// (max, sum exp) partials [rows][ngrp] in a fixed order into lse[r]; lrow[r] =
// lse[r] - zt[r] (row CE); loss_out[0] += scale * sum_r lrow[r] in a fixed order.
int ce_combine(const float* part, int ngrp, const float* zt, float* lse, float* lrow, float* loss_out,
               float scale, int rows, cudaStream_t st);

// ---------------------------------------------------------------- reductions
// out[n] += sum_r X[r, n] (deterministic; 16-row partials into ws fp32 [ceil(rows/16), n]).
int colsum_acc(int dtype, const void* X, float* out, float* ws, int rows, int n, cudaStream_t st);
// Deferred-reduce variants (bf16, wide rows; return -1 when the shape is not
// supported and the caller should use ln_bwd / colsum_acc): write RB-row-block
// partials only ([nb][n]; LN: [2 or 3][nb][h]); reduce_segments then adds up to
// 4 partial sets (src[i] [nb][n[i]], n[i] % 4 == 0) into out[i] in one launch,
// in the same fixed order as the immediate variants.
int colsum_partials(int dtype, const void* X, float* ws, int rows, int n, cudaStream_t st);
int ln_bwd_partials(int dtype, const void* dy, const void* x, const void* gamma, const float* mean,
                    const float* rstd, const void* resid, void* dx, float* ws, int rows, int h, int with_rsum,
                    cudaStream_t st);
int reduce_segments(const float* const* src, float* const* out, const int* n, int nseg, int rows,
                    cudaStream_t st);

// ---------------------------------------------------------------- optimizer
struct AdamHyper {
    float lr, b1, b2, eps, wd;
    float bc1, bc2;  // 1 - b1^t, 1 - b2^t (computed on the host in double, rounded once)
};
// master/m/v/grad fp32 [n]; w (es) [n] = master rounded (bf16) or master itself (fp32: w==master).
// decay_mask: per-element? No: ranges [dec_lo, dec_hi) list handled by caller -> one call per range.
// ZeRO-1 data parallelism (DESIGN R31): the replicas' gradient and weight
// buffers of one chunk, as seen from this process (peer memory over NVLink).
struct DpPtrs {
    float* grad[64];
    void* w[64];
};
// Fused reduce-scatter + AdamW + all-gather over peer memory for the global
// parameter range [lo, lo + n) of the chunk (this replica's shard segment):
// g = sum_j grad_j (replica order), grad_j = 0, AdamW on master/m/v (shard-local
// arrays, element i <-> lo + i), the new weight written into every replica's w.
int dp_adamw(int dtype, const DpPtrs& p, int dp, float* master, float* m, float* v, long lo, long n,
             int decay, const AdamHyper& hp, cudaStream_t st);
// hp_dev (optional): read the hyper-parameters from device memory instead of
// the by-value hp (a CUDA-graph step replays the launch with its captured
// arguments; the runtime updates *hp_dev before each replay)
int adamw(int dtype, float* master, float* m, float* v, float* grad, void* w, long n, int decay,
          const AdamHyper& hp, cudaStream_t st, const AdamHyper* hp_dev = nullptr);
// host reference of the same arithmetic, bit-identical (T-Offload host optimizer)
void adamw_host(float* master, float* m, float* v, const float* grad, uint16_t* w_bf16, long n,
                int decay, const AdamHyper& hp);

// ---------------------------------------------------------------- misc
// programmatic dependent launch of the hot-path kernels (common.cuh)
bool pdl_enabled();
void set_pdl(int on);
// count of kernels launched by this library (gpu_launches evidence)
void note_launches(int n);
long launch_count();
void host_cast_bf16(const float* src, uint16_t* dst, long n);
int fill_zero(void* p, size_t bytes, cudaStream_t st);
int cast_f32_to(int dtype, const float* src, void* dst, long n, cudaStream_t st);

}  // namespace tpipe
