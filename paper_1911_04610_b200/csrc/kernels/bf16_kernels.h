// bf16_kernels.h -- launchers of kernels/bf16.cu (conv-path elementwise and reductions).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace xp {
int bn_chunks(int M, int C);
size_t bn_ws_floats(int M, int C);
// stats [4][C]: mean, rstd, gamma_f, beta_f (the forward's affine parameters)
// counter: one zero-initialised int owned by the calling stream (last-block merge)
cudaError_t launch_bn_stats(const __nv_bfloat16* x, int M, int C, float eps, const __nv_bfloat16* gamma,
                            const __nv_bfloat16* beta, float* ws, int* counter, float* stats, cudaStream_t st);
// Opt-in (XPIPE_BN_FOLD=1, measured slower): small layers (chunks x C <= 8192, M x C <= 2^20) fold
// the final merges into the elementwise kernels (sequential merge order: equal to the separate
// merge launches to fp32 rounding, not bit for bit): launch_bn_bwd_reduce then
// launches only the reduction and launch_bn_bwd_apply merges the totals (and accumulates dgamma /
// dbeta into g_gamma / g_beta); launch_bn_apply_stats merges the forward partials and applies.
// The partials of the stored conv output alone (chunks = bn_chunks, rows bn_chunk_rows):
cudaError_t launch_bn_stats_partial(const __nv_bfloat16* x, int M, int C, float* ws, cudaStream_t st);
int bn_chunk_rows(int M, int C);
// merge of the partials [chunks][2][C] of RC-row chunks + BN-apply (folded or as two launches)
cudaError_t launch_bn_apply_stats(const float* part, int chunks, int RC, float eps, const __nv_bfloat16* gamma,
                                  const __nv_bfloat16* beta, float* stats, const __nv_bfloat16* x, __nv_bfloat16* y,
                                  uint8_t* pidx, int n, int H, int W, int C, int P, int Q, int kh, int kw, int sh,
                                  int sw, int ph, int pw, bool pool, bool relu, cudaStream_t st,
                                  const __nv_bfloat16* res, int ldy);
// the final merge alone, over partials [chunks][2][C] (mean, M2) of RC-row chunks (the last
// one ragged) produced elsewhere -- the fprop GEMM epilogue (RC = 128)
cudaError_t launch_bn_stats_final(const float* part, int chunks, int M, int RC, int C, float eps,
                                  const __nv_bfloat16* gamma, const __nv_bfloat16* beta, float* stats, cudaStream_t st);
// pool: pidx receives the winner's position in every window (uint8 per pooled element);
// res (unpooled only): a folded residual Add, y = relu?(Q(Q(BN(x)) + res)); ldy: row pitch of y
// (0 = C; larger for a concat view), x / res / pidx dense
cudaError_t launch_bn_apply(const __nv_bfloat16* x, const float* stats, __nv_bfloat16* y, uint8_t* pidx, int n, int H,
                            int W, int C, int P, int Q, int kh, int kw, int sh, int sw, int ph, int pw, bool pool,
                            bool relu, cudaStream_t st, const __nv_bfloat16* res = nullptr, int ldy = 0);
// backward through [pool] + ReLU + BN: dgamma/dbeta into g_gamma/g_beta, dx = BN input grad
// routes dout through the stored forward output y (ReLU mask) and pool winners pidx
// backward through [pool] + ReLU + BN, in two launches: the reductions (sum dy, sum dy*xhat per
// channel; dgamma/dbeta into g_gamma/g_beta, totals kept in ws) and the BN input gradient dx.
// Both route dout through the stored forward output y (ReLU mask) and pool winners pidx.
// dres (unpooled, folded residual Add): the residual input's gradient dy' (= or Q(old + dy')).
// ldy: row pitch of dout and y (0 = C; larger for a concat view).
cudaError_t launch_bn_bwd_reduce(const __nv_bfloat16* x, const __nv_bfloat16* dout, const __nv_bfloat16* y,
                                 const uint8_t* pidx, const float* stats, int n, int H, int W, int C, int P, int Q,
                                 int kh, int kw, int sh, int sw, int ph, int pw, bool pool, bool relu, float* ws,
                                 float* g_gamma, float* g_beta, bool accumulate, cudaStream_t st,
                                 __nv_bfloat16* dres = nullptr, bool acc_res = false, int ldy = 0);
cudaError_t launch_bn_bwd_apply(const __nv_bfloat16* x, const __nv_bfloat16* dout, const __nv_bfloat16* y,
                                const uint8_t* pidx, const float* stats, const __nv_bfloat16* gamma_b, int n, int H,
                                int W, int C, int P, int Q, int kh, int kw, int sh, int sw, int ph, int pw, bool pool,
                                bool relu, const float* ws, __nv_bfloat16* dx, cudaStream_t st, int ldy,
                                float* g_gamma, float* g_beta, bool accumulate);
// explicit im2col of an NHWC conv input (C % 8 == 0): cols [n*P*Q][R*S*C], (r, s, c) c fastest
cudaError_t launch_im2col_bf16(const __nv_bfloat16* x, __nv_bfloat16* cols, int n, int H, int W, int C, int P, int Q,
                               int R, int S, int sh, int sw, int ph, int pw, cudaStream_t st);
// the tensor-core Linear backward's output-gradient operand dyp [n][ldp] bf16 and the bias
// gradient gb (may be null); see tc_linear_dgrad / tc_linear_wgrad
cudaError_t launch_linear_dy_prep(const void* dy, bool dy_f32, const __nv_bfloat16* mask, __nv_bfloat16* dyp, int ldp,
                                  float* gb, int n, int out, bool accumulate, cudaStream_t st);
cudaError_t launch_linear_fwd_bf16(const __nv_bfloat16* x, const __nv_bfloat16* W, const __nv_bfloat16* b, void* y,
                                   int n, int in, int out, bool relu, bool f32out, cudaStream_t st);
cudaError_t launch_linear_dgrad_bf16(const void* dy, bool dy_f32, const __nv_bfloat16* mask, const __nv_bfloat16* W,
                                     __nv_bfloat16* dx, int n, int in, int out, cudaStream_t st);
cudaError_t launch_linear_wgrad_bf16(const void* dy, bool dy_f32, const __nv_bfloat16* mask, const __nv_bfloat16* x,
                                     float* gW, float* gb, int n, int in, int out, bool accumulate, cudaStream_t st);
}  // namespace xp

namespace xp {
cudaError_t launch_add_fwd(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* y, int64_t n, bool relu,
                           cudaStream_t st);
cudaError_t launch_add_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* y, __nv_bfloat16* da, __nv_bfloat16* db,
                           int64_t n, bool relu, bool acc_a, bool acc_b, cudaStream_t st);
cudaError_t launch_concat_fwd(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* y, int64_t rows, int Ca,
                              int Cb, cudaStream_t st);
cudaError_t launch_concat_bwd(const __nv_bfloat16* dy, __nv_bfloat16* da, __nv_bfloat16* db, int64_t rows, int Ca,
                              int Cb, bool acc_a, bool acc_b, cudaStream_t st);
cudaError_t launch_pool_fwd(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int H, int W, int C, int P, int Q, int kh,
                            int kw, int sh, int sw, int ph, int pw, bool avg, cudaStream_t st, int ldy = 0);
cudaError_t launch_pool_bwd(const __nv_bfloat16* x, const __nv_bfloat16* dy, __nv_bfloat16* dx, int n, int H, int W,
                            int C, int P, int Q, int kh, int kw, int sh, int sw, int ph, int pw, bool avg,
                            bool accumulate, cudaStream_t st, int ldy = 0);
cudaError_t launch_gap_fwd(const __nv_bfloat16* x, __nv_bfloat16* y, int n, int HW, int C, cudaStream_t st);
cudaError_t launch_gap_bwd(const __nv_bfloat16* dy, __nv_bfloat16* dx, int n, int HW, int C, bool accumulate,
                           cudaStream_t st);
}  // namespace xp
