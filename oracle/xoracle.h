/*
 * xoracle.h -- the plain CPU oracle of the XPipe hot path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load liboracle.so.  It shares no code, header or constant with the CUDA
 * product (include/xpipe.h, paper_1911_04610_b200/); the struct layouts below are this
 * file's own.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n):
 *   - the XPipe asynchronous micro-batch pipeline (Sec. III-A) replayed step by
 *     step: K stages, T micro-batches per mini-batch, gradient accumulation, update after
 *     the T-th micro-batch's backward;
 *   - the bellwether weight prediction (Sec. III-B): version differences
 *     Eq. (1) P:104-109 and Eq. (2), prediction Eq. (3) P:117-121 with
 *     dW from Adam's own moments (BASELINE.json north_star; Eq. (4) P:122-133 as the
 *     opt-in XO_DELTA_PAPER form), cached and reused by the other T-1 micro-batches
 *     (P:141-147);
 *   - plain layer maths (Linear, Conv2d, BatchNorm2d, ReLU, MaxPool2d, global AvgPool,
 *     Flatten, Add, Concat, softmax cross-entropy), NCHW, PyTorch parameter layouts.
 *
 * Modes: XO_FP64 (all double), XO_FP32 (every op in float, fmaf dot products in index
 * order -- the canonical order of DESIGN.md "fp32 contract"), XO_BF16 (bf16 rounding at
 * the documented points, double accumulation, fp32 master/moments/gradients).
 */
#ifndef XORACLE_H
#define XORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { XO_LINEAR = 1, XO_CONV2D, XO_BATCHNORM2D, XO_RELU, XO_MAXPOOL2D, XO_AVGPOOL_GLOBAL,
       XO_FLATTEN, XO_ADD, XO_CONCAT, XO_SOFTMAX_XENT, XO_AVGPOOL2D };
enum { XO_FP64 = 0, XO_FP32 = 1, XO_BF16 = 2 };
enum { XO_SCHED_XPIPE = 0, XO_SCHED_GPIPE = 1 };
enum { XO_PRED_PAPER = 0, XO_PRED_OFF = 1, XO_PRED_FIXED = 2 };
enum { XO_DELTA_ADAM = 0, XO_DELTA_PAPER = 1 };
enum { XO_PARAM = 0, XO_M = 1, XO_V = 2, XO_PRED_FWD = 3, XO_PRED_BWD = 4, XO_GRAD = 5, XO_BUF = 6 };
/* training optimizer: Adam (north star) or the paper's main-experiment Momentum SGD
   (momentum 0.9, weight decay 5e-4) with the prediction's moments tracked
   alongside by Eq. (4) */
enum { XO_OPT_ADAM = 0, XO_OPT_SGD = 1 };

typedef struct {
  int32_t kind, in_c, out_c, kh, kw, sh, sw, ph, pw, bias;
  float bn_eps;
  int32_t src0, src1;   /* producer layer indices, -1 = previous layer */
  int32_t concat_off;   /* unused by the oracle (concat is by source order) */
  int32_t stage;        /* -1 = layer-count rule; else explicit contiguous stage id */
} xo_layer;

typedef struct {
  int32_t in_c, in_h, in_w, classes;
  int32_t mode, schedule, predict, s_fwd, s_bwd, delta_form, snapshots;
  /* init_params[2*layer + tensor]: tensor 0 = weight (BN: gamma), 1 = bias (BN: beta);
     PyTorch layout; NULL entries are not allowed for layers that own the tensor. */
  const double* const* init_params;
  /* optional paper moment init for both moments, flattened per stage in layer
     order; NULL = zeros */
  const double* const* init_m;
  const double* const* init_v;
  /* XO_OPT_SGD (requires delta_form = XO_DELTA_PAPER): W <- W - lr*buf, buf <- mu*buf + (g + wd*W) */
  int32_t optimizer;
  double momentum, weight_decay;
  /* f3: the backward re-runs the stage forward under W_hat_b from the stashed stage
     input (the last stage also recomputes its loss gradient) and differentiates that */
  int32_t recompute;
} xo_config;

typedef struct { int32_t stage, op /*0=F 1=B 2=U*/, t, j, version, s, bellwether; } xo_trace_rec;

typedef struct xo_ctx xo_ctx;

int  xo_init(const xo_layer* layers, int32_t n_layers, int32_t stages, int32_t micro_batches,
             int32_t mini_batch, double lr, double beta1, double beta2, double eps,
             const xo_config* cfg, xo_ctx** out);
/* feed M mini-batches: x [M*N, C, H, W] fp32 NCHW, y [M*N]; flush != 0 drains */
int  xo_step(xo_ctx* h, const float* x, const int32_t* y, int32_t M, int32_t flush,
             float* losses /* nullable, M*T entries in micro-batch order */);
int  xo_get_param(xo_ctx* h, int32_t layer, int32_t tensor, int32_t state, int64_t version,
                  double* dst, size_t count);
int  xo_get_trace(xo_ctx* h, int32_t stage, xo_trace_rec* dst, size_t cap, size_t* n_out);
int  xo_stage_of_layer(xo_ctx* h, int32_t layer);
int  xo_stage_version(xo_ctx* h, int32_t stage);
int64_t xo_param_count(xo_ctx* h, int32_t layer, int32_t tensor);
/* loss (mean over n) and gradient of all parameters (layer order, weight then bias) at the
   current master weights, one forward+backward of the whole network (no prediction) */
int  xo_eval_loss_grad(xo_ctx* h, const float* x, const int32_t* y, int32_t n,
                       double* loss, double* grad, size_t count);
/* Eq. (1) (pass 0) / Eq. (2) (pass 1), half-up rounding */
int  xo_version_difference(int32_t K, int32_t T, int32_t rank, int32_t pass);
/* the elementwise Adam update + prediction, version k = new version */
/* one Momentum-SGD step with the paper-literal prediction (Eq. (3)-(4)), elementwise:
   outputs W', buf', m' (Eq. (4) v_t, first moment), v' (Eq. (4) m_t, second moment), W_hat_f/b */
int  xo_sgd_predict(int32_t mode, size_t n, const float* W, const float* g, const float* buf, const float* m,
                    const float* v, float lr, float beta1, float beta2, float eps, float momentum,
                    float weight_decay, int32_t s_f, int32_t s_b, float* W_out, float* buf_out, float* m_out,
                    float* v_out, float* pf_out, float* pb_out);
int  xo_adam_predict(int32_t mode, int32_t delta_form, size_t n, const float* W, const float* g,
                     const float* m, const float* v, int64_t k, float lr, float beta1, float beta2,
                     float eps, int32_t s_f, int32_t s_b, float* W_out, float* m_out, float* v_out,
                     float* pf_out, float* pb_out);
void xo_finalize(xo_ctx* h);
const char* xo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
