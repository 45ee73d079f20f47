// C-ABI wrappers for the kernel-level entry points (include/tpipe_kernels.h).
#include "tpipe.h"
#include "tpipe_kernels.h"

#include "kernels/kernels.h"
#include "runtime/errors.h"

using namespace tpipe;

#define TP_API extern "C" __attribute__((visibility("default")))

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int chk_dtype(int dtype) {
    if (dtype != TPIPE_FP32 && dtype != TPIPE_BF16) return set_error(TPIPE_E_INVALID, "dtype");
    return 0;
}

static int launch_rc(int rc, const char* what) {
    if (rc == 0) return 0;
    cudaError_t e = cudaGetLastError();
    return set_error(TPIPE_E_CUDA, "%s failed (rc=%d, cuda: %s)", what, rc, cudaGetErrorString(e));
}

static GemmDesc mk(int M, int N, int K, const void* A, long lda, int ak, const void* B, long ldb,
                   int bk, int epi, void* C, long ldc, const void* bias, const void* R, long ldr,
                   void* C2, long ldc2, const void* aux, long ldaux) {
    GemmDesc g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_kmajor = ak;
    g.B = B; g.ldb = ldb; g.b_kmajor = bk;
    g.epi = epi; g.C = C; g.ldc = ldc; g.bias = bias; g.res = R; g.ldr = ldr;
    g.C2 = C2; g.ldc2 = ldc2; g.aux = aux; g.ldaux = ldaux;
    return g;
}

TP_API int tpipe_k_gemm(int dtype, int M, int N, int K, const void* A, long lda, int a_kmajor,
                        const void* B, long ldb, int b_kmajor, int epi, void* C, long ldc,
                        const void* bias, const void* R, long ldr, void* C2, long ldc2,
                        const void* aux, long ldaux, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    if (epi < 0 || epi > 6) return set_error(TPIPE_E_INVALID, "epi");
    GemmDesc g = mk(M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, epi, C, ldc, bias, R, ldr, C2,
                    ldc2, aux, ldaux);
    return launch_rc(gemm(dtype, g, S(stream)), "gemm");
}

TP_API int tpipe_k_gemm_dot(int M, int N, int K, const void* A, long lda, int a_kmajor, const void* B,
                            long ldb, int b_kmajor, void* C, long ldc, const void* O, long ldo, float* Dout,
                            int s, int hd, void* stream) {
    GemmDesc g = mk(M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, EPI_STORE_DOT, C, ldc, nullptr, nullptr, 0,
                    nullptr, 0, O, ldo);
    g.part = Dout;
    g.dot_s = s;
    g.dot_hd = hd;
    return launch_rc(gemm(DT_BF16, g, S(stream)), "gemm_dot");
}

TP_API int tpipe_k_gemm_simt(int dtype, int M, int N, int K, const void* A, long lda,
                             int a_kmajor, const void* B, long ldb, int b_kmajor, int epi, void* C,
                             long ldc, const void* bias, const void* R, long ldr, void* C2,
                             long ldc2, const void* aux, long ldaux, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    GemmDesc g = mk(M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, epi, C, ldc, bias, R, ldr, C2,
                    ldc2, aux, ldaux);
    return launch_rc(gemm_simt(dtype, g, S(stream)), "gemm_simt");
}

TP_API void tpipe_k_gemm_set_pair(int on) { gemm_set_pair(on); }
TP_API void tpipe_k_gemm_set_pair_min_tiles(int n) { gemm_set_pair_min_tiles(n); }
TP_API void tpipe_k_gemm_set_wide_choice(int on) { gemm_set_wide_choice(on); }
TP_API void tpipe_k_ln_set_rows_bwd(int on) { ln_set_rows_bwd(on); }

TP_API int tpipe_k_ln_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y,
                          float* mean, float* rstd, int rows, int h, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(ln_fwd(dtype, x, gamma, beta, y, mean, rstd, rows, h, S(stream)), "ln_fwd");
}

TP_API int tpipe_k_ln_bwd(int dtype, const void* dy, const void* x, const void* gamma,
                          const float* mean, const float* rstd, const void* resid, void* dx,
                          float* dgamma, float* dbeta, float* ws, int rows, int h, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(ln_bwd(dtype, dy, x, gamma, mean, rstd, resid, dx, dgamma, dbeta, ws, rows, h,
                            S(stream)),
                     "ln_bwd");
}

TP_API int tpipe_k_ln_bwd_partials(const void* dy, const void* x, const void* gamma, const float* mean,
                                   const float* rstd, const void* resid, void* dx, float* ws, int rows, int h,
                                   int with_rsum, void* stream) {
    return launch_rc(ln_bwd_partials(DT_BF16, dy, x, gamma, mean, rstd, resid, dx, ws, rows, h, with_rsum,
                                     S(stream)),
                     "ln_bwd_partials");
}

TP_API int tpipe_k_ln_bwd_rsum(int dtype, const void* dy, const void* x, const void* gamma,
                               const float* mean, const float* rstd, const void* resid, void* dx,
                               float* dgamma, float* dbeta, float* dresid_sum, float* ws, int rows,
                               int h, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    if (!resid || !dresid_sum) return set_error(TPIPE_E_INVALID, "ln_bwd_rsum: resid and dresid_sum are required");
    return launch_rc(ln_bwd(dtype, dy, x, gamma, mean, rstd, resid, dx, dgamma, dbeta, ws, rows, h,
                            S(stream), dresid_sum),
                     "ln_bwd_rsum");
}

TP_API int tpipe_k_attn_fwd(int dtype, const void* qkv, void* o, float* lse, int b, int s, int a,
                            int d, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(attn_fwd(dtype, qkv, o, lse, b, s, a, d, S(stream)), "attn_fwd");
}

TP_API int tpipe_k_attn_bwd(int dtype, const void* qkv, const void* o, const void* dout,
                            const float* lse, void* dqkv, float* ws, int b, int s, int a, int d,
                            void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(attn_bwd(dtype, qkv, o, dout, lse, dqkv, ws, b, s, a, d, S(stream)),
                     "attn_bwd");
}

TP_API int tpipe_k_embed_fwd(int dtype, const int* tok, const void* wte, const void* wpe, void* x,
                             int rows, int s, int h, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(embed_fwd(dtype, tok, wte, wpe, x, rows, s, h, S(stream)), "embed_fwd");
}

TP_API int tpipe_k_embed_bwd(int dtype, const int* tok, const void* dx, float* dwte, float* dwpe,
                             int* ws, int rows, int s, int h, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(embed_bwd(dtype, tok, dx, dwte, dwpe, ws, rows, s, h, S(stream)), "embed_bwd");
}

TP_API int tpipe_k_ce_fwd(const float* logits, const int* tgt, float* lse, float* loss_out,
                          float scale, int rows, int V, void* stream) {
    return launch_rc(ce_fwd(logits, tgt, lse, loss_out, scale, rows, V, S(stream)), "ce_fwd");
}

TP_API int tpipe_k_ce_bwd(int dtype, const float* logits, const int* tgt, const float* lse,
                          void* dlogits, float scale, int rows, int V, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(ce_bwd(dtype, logits, tgt, lse, dlogits, scale, rows, V, S(stream)), "ce_bwd");
}

TP_API int tpipe_k_head_ce(const void* x, const void* w, const int* tgt, float* lse, void* dlogits,
                           float* loss_out, float scale, int rows, int V, int h, float* ws, void* stream) {
    if (!x || !w || !tgt || !lse || !dlogits || !ws) return set_error(TPIPE_E_INVALID, "NULL argument");
    if (V % 64 || h % 64 || rows <= 0) return set_error(TPIPE_E_INVALID, "V, h multiples of 64; rows > 0");
    const int ng = ce_groups(V);
    float* part = ws;
    float* zt = ws + 2L * rows * ng;
    float* lrow = zt + rows;
    GemmDesc g;
    g.M = rows; g.N = V; g.K = h;
    g.A = x; g.lda = h; g.a_kmajor = 1;
    g.B = w; g.ldb = h; g.b_kmajor = 1;
    g.epi = EPI_LSE_PART;
    g.targets = tgt;
    g.part = part;
    g.zt = zt;
    if (int rc = launch_rc(gemm(DT_BF16, g, S(stream)), "head gemm (lse)")) return rc;
    if (int rc = launch_rc(ce_combine(part, ng, zt, lse, lrow, loss_out, scale, rows, S(stream)), "ce_combine"))
        return rc;
    g.epi = EPI_CE_GRAD;
    g.lse = lse;
    g.C = dlogits;
    g.ldc = V;
    g.scale = scale;
    return launch_rc(gemm(DT_BF16, g, S(stream)), "head gemm (dlogits)");
}

TP_API int tpipe_k_colsum(int dtype, const void* X, float* out, float* ws, int rows, int n,
                          void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    return launch_rc(colsum_acc(dtype, X, out, ws, rows, n, S(stream)), "colsum");
}

TP_API int tpipe_k_adamw(int dtype, float* master, float* m, float* v, float* grad, void* w, long n,
                         int decay, float lr, float b1, float b2, float eps, float wd, float bc1,
                         float bc2, void* stream) {
    if (int e = chk_dtype(dtype)) return e;
    AdamHyper hp{lr, b1, b2, eps, wd, bc1, bc2};
    return launch_rc(adamw(dtype, master, m, v, grad, w, n, decay, hp, S(stream)), "adamw");
}

TP_API void tpipe_host_adamw(float* master, float* m, float* v, const float* grad,
                             uint16_t* w_bf16, long n, int decay, float lr, float b1, float b2,
                             float eps, float wd, float bc1, float bc2) {
    AdamHyper hp{lr, b1, b2, eps, wd, bc1, bc2};
    adamw_host(master, m, v, grad, w_bf16, n, decay, hp);
}
