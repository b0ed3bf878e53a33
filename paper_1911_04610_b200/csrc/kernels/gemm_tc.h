// gemm_tc.h -- tcgen05 implicit-GEMM entry points (kernels/gemm_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace xp {

enum { GEMM_PLAIN = 0, GEMM_FPROP = 1, GEMM_DGRAD = 2, GEMM_WGRAD = 3 };
// EPI_LINEAR_T: swap-AB Linear, D[m = feature][c = sample] -> out[c][m] (ldo = features) with
// the bias of feature m, optional ReLU, bf16 or (f32out) fp32
enum { EPI_BF16 = 0, EPI_F32 = 1, EPI_WGRAD_T = 2, EPI_LINEAR_T = 3 };
constexpr int kTileCounters = 1 << 14;  // per-stream split-K arrival counters (zero-initialised)

struct ConvGeo {
  int Nimg, H, W, C;      // input NHWC, C = channel stride (Cin padded to a multiple of 8)
  int Co, R, S, P, Q;     // output channels, filter, output spatial
  int sh, sw, ph, pw;
};

struct GemmArgs {
  int M, N, K;
  const __nv_bfloat16* A;
  const __nv_bfloat16* B;
  int64_t lda, ldb;
  ConvGeo g;
  int epi;
  void* out;
  int64_t ldo;
  int accumulate;
  int64_t split_stride;   // unused (kept 0)
  int kb_per_split;
  // split-K: grid.z = splits = cs x nc CTAs per tile; clusters of cs CTAs along z reduce over
  // DSMEM (CTA rank z owns rows [z*128/cs, (z+1)*128/cs) of the tile); with nc > 1 clusters
  // every row slice goes to the workspace `ws` and the last of the nc CTAs owning that slice
  // (per-slice arrival counter, self-resetting) sums the nc slices in order c = 0..nc-1
  int splits, cs, nc;
  float* ws;              // caller workspace (ws_elems floats)
  int64_t ws_elems;
  int l2red;              // 1: partial tiles go through ws (L2) [tile][split], else through DSMEM
  float* ws_x;            // cross-cluster partial slices [tile][cluster] (nc > 1)
  int* tile_counters;
  // B operand by TMA (cp.async.bulk.tensor into the 128B-swizzled UMMA layout):
  // 0 = cp.async gather, 1 = 2D K-major box {64, BN}, 2 = 2D MN-major boxes {64, 64},
  // 3 = 3D dgrad weights view {C, R*S, Co} boxes {64, 1, 64}
  int b_tma;
  // A operand by TMA (stride-1 convs with C % 64 == 0 whose tile rows form a box of the pixel
  // grid): 4D tiled map over the NHWC activation {C, W, H, N}, box {64, bq, bp, bn}; the tile's
  // pixel origin comes from the m (fprop/dgrad) or k (wgrad) index on the grid {gq, gp}
  int a_tma;
  int gq, gp;
  int stages;  // smem ring depth (set by the launcher)
  // FPROP without split-K: the epilogue also writes the BatchNorm partial statistics of every
  // 128-row tile of the stored (bf16-rounded) output, bn_part[mtile][0][co] = tile mean and
  // bn_part[mtile][1][co] = sum of squared deviations (rows < M only), or null
  float* bn_part;
  int force_tma;            // PLAIN: stream both operands by TMA (the im2col'd first layer)
  unsigned long long* dbg;  // development timing probe (XPIPE_GEMM_DBG), else null
  int dev_flags;            // development experiments (XPIPE_GEMM_DEV), 0 in production
  const __nv_bfloat16* bias;  // EPI_LINEAR_T: per-row bias (or null)
  int relu, f32out;           // EPI_LINEAR_T: ReLU on the bf16 output / fp32 output (logits);
                              // bnf: ReLU after the BatchNorm (and residual)
  // bnf (FPROP, no split-K): the CTAs of one N tile form a cluster along M (grid (mt, nt),
  // cluster (mt, 1, 1), one tile each); after the tile partials of the BatchNorm statistics
  // (as bn_part) are exchanged over DSMEM, every CTA merges them (the fixed tree of
  // bn_stats_final_kernel) and applies BN [+ residual] [+ ReLU] to its accumulator tile:
  // y[row][col] (row pitch ldy) = Q(relu?(gamma (x - mean) rstd + beta)) of x = Q(acc), or with
  // res: relu?(Q(Q(gamma (x - mean) rstd + beta) + res[row][col])); CTA rank 0 stores the
  // statistics [4][N] (mean, rstd, gamma, beta) for the backward
  // DGRAD from an explicit operand (a_tma = 4): A = cols [M][K] dense (tc_dgrad_cols), k = tap *
  // kco + co with kco = Co rounded up to 64 (every k-block inside one tap); 0 = implicit gather
  int kco;
  // EPI_BF16 row map (strided 1x1 dgrad): GEMM row m = (n, p, q) of a [rm_P][rm_Q] grid stores to
  // row (n * rm_H + p * rm_sh) * rm_W + q * rm_sw; rm_Q = 0: identity
  int rm_P, rm_Q, rm_H, rm_W, rm_sh, rm_sw;
  int bnf;
  const __nv_bfloat16* gamma;
  const __nv_bfloat16* beta;
  float bn_eps;
  float* stats;
  __nv_bfloat16* y;
  int64_t ldy;
  const __nv_bfloat16* res;
};

// the fused BatchNorm of a conv's forward (see GemmArgs::bnf); res may be null
struct BnFuse {
  const __nv_bfloat16* gamma;
  const __nv_bfloat16* beta;
  float eps;
  float* stats;
  __nv_bfloat16* y;
  int ldy;
  const __nv_bfloat16* res;
  bool relu;
};

// plain GEMM for unit parity: D[M][N] fp32 (ldd) = A(m,k) B(n,k)
cudaError_t tc_gemm_plain(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int M, int N, int K, bool a_kmajor,
                          bool b_kmajor, int64_t ldd, cudaStream_t st);

// Y [Nimg*P*Q][Co] bf16 = conv(X [Nimg][H][W][C] bf16, W [Co][R][S][C] bf16)
// ws: fp32 split-K workspace of ws_elems; counters: kTileCounters zeroed ints owned by the
// calling stream (NULL = no split-K)
// bn_part (optional): if the launch runs without split-K, the per-128-row-tile BatchNorm
// partials of Y go there ([ceil(M/128)][2][Co], see GemmArgs::bn_part) and *bn_tiles is set to
// ceil(M/128); otherwise *bn_tiles = 0 and the caller computes the statistics itself
// bnf (optional): fuse the BatchNorm statistics and apply into the GEMM when the launch runs
// without split-K and the M tiles fit one thread-block cluster; *bnf_done tells the caller
cudaError_t tc_conv_fprop(const ConvGeo& g, const __nv_bfloat16* X, const __nv_bfloat16* Wt, __nv_bfloat16* Y,
                          float* ws, int64_t ws_elems, int* counters, cudaStream_t st, float* bn_part = nullptr,
                          int* bn_tiles = nullptr, const BnFuse* bnf = nullptr, bool* bnf_done = nullptr);
// dX [Nimg*H*W][Cx] bf16 (Cx = real input channels, multiple of 8) from dY [Nimg*P*Q][Co].
// Paths: 1x1 stride-1 convs as a dense GEMM (dY x W); strided 1x1 convs as a dense GEMM over dY
// whose rows scatter to the strided input pixels (the others zero, or untouched when
// accumulating); geometries the TMA pixel boxes cannot serve (stride > 1, Co % 64, tile rows
// that are not a box of the input grid) through an explicit transposed-conv operand built in
// dcols (tc_dgrad_cols_elems(g) bf16, caller scratch; NULL keeps the implicit cp.async gather)
cudaError_t tc_conv_dgrad(const ConvGeo& g, int Cx, const __nv_bfloat16* dY, const __nv_bfloat16* Wt,
                          __nv_bfloat16* dX, float* ws, int64_t ws_elems, int* counters, cudaStream_t st,
                          bool accumulate = false, __nv_bfloat16* dcols = nullptr, int64_t dcols_elems = 0);
// elements of the explicit dgrad operand a geometry needs (0: the conv runs without one)
int64_t tc_dgrad_cols_elems(const ConvGeo& g);
// the forward / weight-gradient A operand cannot come from TMA pixel boxes of the activation
// (and the conv is not a 1x1 stride-1 one, which runs dense): use the explicit im2col path
bool tc_conv_needs_cols(const ConvGeo& g);
// gW [Co][R][S][C] fp32 (=|+=) sum over pixels of dY x im2col(X)
cudaError_t tc_conv_wgrad(const ConvGeo& g, const __nv_bfloat16* X, const __nv_bfloat16* dY, float* gW, bool accumulate,
                          float* ws, int64_t ws_elems, int* counters, cudaStream_t st);
// A conv whose input channels are too few for the TMA pixel-box path (C % 64 != 0, the
// network's first layer) runs on an explicit im2col matrix cols [Nimg*P*Q][R*S*C] (bf16,
// (r, s, c) with c fastest -- the weight layout): fprop = cols . W^T (+ the fused BN partials),
// wgrad: g (=|+=) (cols^T . dY)^T, both dense GEMMs with TMA-fed operands.
cudaError_t tc_im2col_fprop(const ConvGeo& g, const __nv_bfloat16* cols, const __nv_bfloat16* Wt, __nv_bfloat16* Y,
                            float* ws, int64_t ws_elems, int* counters, cudaStream_t st, float* bn_part,
                            int* bn_tiles);
cudaError_t tc_im2col_wgrad(const ConvGeo& g, const __nv_bfloat16* cols, const __nv_bfloat16* dY, float* gW,
                            bool accumulate, float* ws, int64_t ws_elems, int* counters, cudaStream_t st);
// bf16 Linear layers on the tensor cores, swap-AB (the micro-batch is the narrow N side of the
// UMMA, features the 128-row M side), both operands by TMA:
//   fwd  : y[r][o] = epi(sum_i W[o][i] x[r][i] + b[o])      (M = out, N = n, K = in; y fp32 if
//          f32out, else Q(relu?(.)) bf16)
//   dgrad: dx[r][i] = Q(sum_o dyp[r][o] W[o][i])              (M = in, N = n, K = out)
//   wgrad: gW[o][i] (=|+=) sum_r dyp[r][o] x[r][i]           (M = in, N = out, K = n)
// dyp [n][ldp] bf16 (ldp % 8 == 0, columns >= out zero) is the masked, bf16-rounded output
// gradient (launch_linear_dy_prep); x rows and W rows need in % 8 == 0.
cudaError_t tc_linear_fwd(const __nv_bfloat16* x, const __nv_bfloat16* W, const __nv_bfloat16* b, void* y, int n,
                          int in, int out, bool relu, bool f32out, float* ws, int64_t ws_elems, int* counters,
                          cudaStream_t st);
cudaError_t tc_linear_dgrad(const __nv_bfloat16* dyp, int ldp, const __nv_bfloat16* W, __nv_bfloat16* dx, int n,
                            int in, int out, float* ws, int64_t ws_elems, int* counters, cudaStream_t st);
cudaError_t tc_linear_wgrad(const __nv_bfloat16* x, const __nv_bfloat16* dyp, int ldp, float* gW, int n, int in,
                            int out, bool accumulate, float* ws, int64_t ws_elems, int* counters, cudaStream_t st);
// number of pipeline stages whose streams share this process's busiest device (sets the
// split-K threshold; 1 = one stage per device)
void tc_set_coresident_stages(int n);
// workspace (floats) the launchers above can use profitably for split-K
int64_t tc_conv_ws_elems(const ConvGeo& g);

}  // namespace xp
