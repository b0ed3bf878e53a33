/*
 * xpipe.h -- C ABI of the B200-native XPipe hot path (libxpipe.so).
 *
 * XPipe (Guan, Yin, Li, Lu; arXiv 1911.04610; P:n = /root/reference/PAPER.md line n):
 * an asynchronous micro-batch pipeline across K GPU stages (Sec. III-A) in which
 * every stage runs its forward and backward passes under weights predicted by the
 * mini-batch's bellwether (Sec. III-B):
 *     W_hat = W - s * lr * m_hat / (sqrt(v_hat) + eps)            (Eq. (3), BJ north star)
 * with the version difference s of Eq. (1) (forward) or Eq. (2) (backward,
 * P:111-115), and Adam's own moments.  Gradients of the T micro-batches of a mini-batch are
 * accumulated and applied when the T-th micro-batch finishes its backward by one
 * fused Adam-update + prediction sweep that also materialises the next W_hat buffers.
 *
 * Conventions for every function:
 *   - returns int: XP_OK (0) or a negative XP_E* code; no C++ exception crosses the ABI;
 *   - pointers are host pointers unless the argument says "device";
 *   - the library copies what it needs from its inputs before returning (nothing borrowed
 *     is retained); outputs go to caller-owned buffers;
 *   - a device or communication fault poisons the context: every later call except
 *     xpipe_last_error and xpipe_finalize returns XP_ESTATE.
 * Thread safety: one context must not be used from two threads at once.
 */
#ifndef XPIPE_H
#define XPIPE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------------------- */
enum {
  XP_OK = 0,
  XP_EINVAL = -1,        /* invalid argument; detected before any device work */
  XP_ENOMEM = -2,        /* device or host allocation failed */
  XP_ECUDA = -3,         /* CUDA runtime/driver error (context poisoned) */
  XP_ECOMM = -4,         /* stage-to-stage transport error (context poisoned) */
  XP_ESCHED = -5,        /* schedule/cache violation or pipeline watchdog timeout (internal) */
  XP_ENONFINITE = -6,    /* non-finite loss seen by the loss kernel (device flag, read at the end of a
                            synchronous xpipe_step; the context stays usable) */
  XP_ESTATE = -7,        /* context is poisoned */
  XP_EUNSUPPORTED = -8   /* valid request this build does not implement */
};

/* ---- layer kinds (the DNN is partitioned layer-wise into stages) ----------- */
enum { XP_LINEAR = 1, XP_CONV2D, XP_BATCHNORM2D, XP_RELU, XP_MAXPOOL2D, XP_AVGPOOL_GLOBAL,
       XP_FLATTEN, XP_ADD, XP_CONCAT, XP_SOFTMAX_XENT,
       XP_AVGPOOL2D /* kh x kw window, zero padding counted in the divisor (Inception branch pool) */ };

/* ---- configuration enums -------------------------------------------------------------- */
enum { XP_FP32 = 0,   /* fp32 SIMT path, bit-exact with the oracle's fp32 contract */
       XP_BF16 = 1 }; /* bf16 operands on tcgen05 tensor cores, fp32 master/moments/grads */
enum { XP_SCHED_XPIPE = 0, XP_SCHED_GPIPE = 1 };
enum { XP_PRED_PAPER = 0,  /* s from Eq. (1)/(2) */
       XP_PRED_OFF = 1,    /* s = 0 (plain asynchronous pipeline / GPipe semantics) */
       XP_PRED_FIXED = 2 };/* s = cfg.s_fwd / cfg.s_bwd */
enum { XP_DELTA_ADAM = 0,  /* dW = lr * m_hat / (sqrt(v_hat) + eps)   (north star) */
       XP_DELTA_PAPER = 1 };/* dW = lr * (m/(1-b1)) / sqrt(v/(1-b2) + eps)  (Eq. (3)-(4) literal) */
enum { XP_MOM_ZERO = 0, XP_MOM_GIVEN = 1 /* cfg.init_m / cfg.init_v (e.g. 1e-4*U[0,1)) */ };
/* training optimizer.  XP_OPT_MOMENTUM_SGD is the paper's main-experiment optimizer
   (SURVEY 8f row f2): buf = momentum*buf + (g + weight_decay*W), W -= lr*buf, while
   the prediction keeps its own Eq. (4) moments of the raw gradient and uses the
   literal Eq. (3)/(4) dW, so it requires delta_form = XP_DELTA_PAPER. */
enum { XP_OPT_ADAM = 0, XP_OPT_MOMENTUM_SGD = 1 };
/* where the backward's predicted weights W_hat_b come from (the bellwether makes the
   prediction and caches it for the other T-1 micro-batches of its pass):
   XP_WBWD_MATERIALIZE -- the update sweep writes W_hat_b of the new version (32 B/param sweep);
   XP_WBWD_BELLWETHER  -- the update sweep writes W_hat_f only (30 B/param) and the backward
   bellwether B(t,1) computes W_hat_b from the stage's current W, m, v (one 14 B/param pass:
   read W, m, v, write bf16 W_hat_b), bit-identical to the materialised values. */
enum { XP_WBWD_MATERIALIZE = 0, XP_WBWD_BELLWETHER = 1 };
enum { XP_TRANSPORT_P2P = 0 };  /* the producer stream copies its boundary tensor into the consumer's
                                   ring slot with the copy engine (cudaMemcpyAsync, same device or
                                   NVLink peer, or a CUDA-IPC-mapped slot in multi-process mode),
                                   then writes the slot's ready flag with a stream memory operation
                                   (cuStreamWriteValue32); the consumer stream waits on the flag
                                   (cuStreamWaitValue32) -- no SM spins, no host involvement */

/* xpipe_step flags */
enum { XP_FLUSH = 1,        /* drain the pipeline at the end of the call */
       XP_DEVICE_PTRS = 2,  /* x and y are device pointers on stage 0's / stage K-1's device */
       XP_ASYNC = 4 };      /* return after enqueue; the next call (or xpipe_sync) waits -- except
                                 that consecutive replays of captured graphs (single process, one
                                 device) chain on the device without a host wait; a call stamped by
                                 cfg.timing always completes (its statistics are read back) */

/* xpipe_get_weights selectors */
enum { XP_T_WEIGHT = 0, XP_T_BIAS = 1 };       /* BatchNorm: WEIGHT = gamma, BIAS = beta */
enum { XP_S_PARAM = 0, XP_S_M = 1, XP_S_V = 2, XP_S_PRED_FWD = 3, XP_S_PRED_BWD = 4, XP_S_GRAD = 5,
       XP_S_BUF = 6 /* Momentum-SGD velocity (XP_OPT_MOMENTUM_SGD) */ };

/* One layer.  src0/src1: producer layer indices (-1 = the previous layer); a DAG edge may
   not cross a stage cut except into the next stage's first layer.  stage: -1 = automatic
   (layer-count rule of P:154-156: partition units begin at every Linear/Conv2d layer, the
   remainder goes to the last stages); otherwise an explicit, contiguous stage id. */
typedef struct {
  int32_t kind, in_c, out_c, kh, kw, sh, sw, ph, pw, bias;
  float bn_eps;
  int32_t src0, src1;
  int32_t concat_off;
  int32_t stage;
} xpipe_layer;

/* optional device-memory hooks (the Python binding routes them to PyTorch's allocator) */
typedef void* (*xpipe_alloc_fn)(size_t bytes, int32_t device, void* user);
typedef void (*xpipe_free_fn)(void* ptr, size_t bytes, int32_t device, void* user);

/* Zero-initialised = defaults. */
typedef struct {
  int32_t in_c, in_h, in_w, classes;  /* network input [C,H,W] and number of classes (required) */
  uint64_t seed;                      /* weight init when init_params is NULL (default 1) */
  int32_t precision;                  /* XP_FP32 | XP_BF16 */
  int32_t schedule;                   /* XP_SCHED_XPIPE | XP_SCHED_GPIPE */
  int32_t predict;                    /* XP_PRED_* */
  int32_t s_fwd, s_bwd;               /* with XP_PRED_FIXED */
  int32_t delta_form;                 /* XP_DELTA_ADAM | XP_DELTA_PAPER */
  int32_t moment_init;                /* XP_MOM_ZERO | XP_MOM_GIVEN (requires XP_DELTA_PAPER) */
  int32_t n_devices;                  /* stage k runs on devices[k % n_devices]; 0 = current device */
  int32_t devices[8];
  int32_t transport;                  /* XP_TRANSPORT_P2P */
  int32_t snapshots;                  /* keep W after every version for get_weights(version=v) */
  int32_t trace;                      /* record per-op device trace (K12); disables graphs */
  int32_t graphs;                     /* capture repeated step calls as CUDA graphs */
  int32_t profile;                    /* record CUDA events around every sweep launch */
  int32_t watchdog_ms;                /* xpipe_step timeout (0 = 120000) */
  int32_t multi_process;              /* 1 = one process per stage: this process owns stage my_stage
                                         only; neighbours are attached with xpipe_ipc_import */
  int32_t my_stage;
  /* optional initial tensors, float32, PyTorch layout, [2*layer + XP_T_*]; NULL = seeded init */
  const float* const* init_params;
  const float* const* init_m;         /* with XP_MOM_GIVEN, same indexing */
  const float* const* init_v;
  xpipe_alloc_fn alloc;               /* NULL = cudaMalloc / cudaFree */
  xpipe_free_fn free;
  void* alloc_user;
  int32_t optimizer;                  /* XP_OPT_ADAM (default) | XP_OPT_MOMENTUM_SGD */
  float momentum, weight_decay;       /* XP_OPT_MOMENTUM_SGD: in [0,1) and >= 0 (paper: 0.9, 5e-4) */
  int32_t recompute;                  /* 1 = activation recomputation: every
                                         backward B(u) first re-runs the stage forward under W_hat_b
                                         from the stashed stage input (the last stage also its loss
                                         gradient) and differentiates that forward */
  int32_t serialize;                  /* profiling aid (single process, one device): all stages and
                                         their weight-gradient work on one stream in the dataflow
                                         enqueue order, so every kernel runs alone */
  int32_t fb_overlap;                 /* 1 = each stage runs its forwards on a second stream, so
                                         F(u+S) overlaps B(u) (one more ring/stash slot per stage;
                                         ordering by events: F(u) -> B(u), B(u) -> F(u+S+1),
                                         update -> next bellwether forward); same results */
  int32_t timing;                     /* p > 0: every p-th xpipe_step call (the first, p+1-th, ...) stamps
                                         each forward/backward op with %globaltimer on the stream it
                                         runs on (1-thread kernels at its start and end, and around the
                                         hand-off of bellwether micro-batches; also inside replayed
                                         graphs, which exist per variant) and fills the span / busy /
                                         bubble / steady-rate / hand-off fields of xpipe_stats
                                         (ops_timed = 0 on the other calls); 0 = off */
  int32_t wbwd;                       /* XP_WBWD_MATERIALIZE (default) | XP_WBWD_BELLWETHER */
} xpipe_config;

/* one device-trace record (K12): op 0 = forward, 1 = backward, 2 = update.  version is the
   weight version the op ran under (update: the version it produced), s the version
   difference used, wbuf the W_hat buffer (forward: version & 1).  t0/t1: %globaltimer ns. */
typedef struct {
  int32_t stage, op, t, j, version, s, bellwether, wbuf;
  uint64_t t0_ns, t1_ns;
} xpipe_trace_rec;

/* kernel classes timed with CUDA events on the launching stream when cfg.profile != 0 */
enum { XP_PROF_SWEEP = 0,       /* K1: work = algorithmic bytes */
       XP_PROF_CONV_FPROP = 1,  /* tcgen05 implicit-GEMM conv forward: work = 2*M*N*K flops */
       XP_PROF_CONV_DGRAD = 2,
       XP_PROF_CONV_WGRAD = 3,
       XP_PROF_BN_STATS = 4,    /* BN statistics (partial chunks + fixed-order merge): work = algorithmic bytes */
       XP_PROF_BN_APPLY = 5,    /* BN apply [+ ReLU + max-pool]: work = algorithmic bytes */
       XP_PROF_BN_BWD_REDUCE = 6, /* BN backward reductions (sum dy, sum dy*xhat) + merge: bytes */
       XP_PROF_BN_BWD_APPLY = 7,  /* BN input gradient: bytes */
       XP_PROF_N = 8 };

#define XP_STATS_STAGES 16
typedef struct {
  double span_ms;                    /* cfg.timing: device time from the first op start to the last
                                        op end of this call over the process's stages (%globaltimer);
                                        else 0 */
  double prof_ms[XP_PROF_N];         /* summed device time per kernel class (cfg.profile) */
  int64_t prof_launches[XP_PROF_N];
  double prof_work[XP_PROF_N];       /* algorithmic bytes (sweep, BN) or flops (GEMM classes) */
  int64_t kernel_launches;           /* kernels enqueued by this call (directly or in a graph) */
  int64_t graph_replays;             /* 1 if this call replayed a captured CUDA graph */
  float* losses;                     /* optional caller buffer of M*T per-micro-batch mean losses */
  /* ---- cfg.timing (zero otherwise) ---- */
  double busy_ms[XP_STATS_STAGES];   /* per stage: length of the union of its op intervals (an op
                                        runs from its input's arrival to the end of its hand-off, a
                                        backward B(t,T) to the end of the update sweep) */
  double bubble_fraction;            /* 1 - sum_k busy_ms[k] / (stages owned * span_ms) */
  double steady_samples_per_s;       /* mini-batches / time between the bellwether forwards
                                        on stage 0 (0 if stage 0 is not owned or too few); the first
                                        K mini-batches after an empty pipeline and the last K of a
                                        flushing call are excluded (warm-up / drain) */
  /* hand-off times, sampled on the bellwether micro-batches (1 in T; the other messages are
     the same size): stage k's activation messages k->k+1 and gradient messages k->k-1, summed
     time and bytes over the sampled messages (GB/s = bytes / time) */
  double p2p_fwd_ms[XP_STATS_STAGES];
  double p2p_bwd_ms[XP_STATS_STAGES];
  double p2p_fwd_bytes[XP_STATS_STAGES];
  double p2p_bwd_bytes[XP_STATS_STAGES];
  int64_t ops_timed;                 /* forward + backward ops timed in this call */
} xpipe_stats;

/* Build the pipeline.  layers/n_layers: the network, last layer XP_SOFTMAX_XENT;
   stages = K; micro_batches = T; mini_batch = N (N % T == 0); lr > 0; betas in [0,1);
   eps > 0 (defaults of P:168: 0.9, 0.999, 1e-8).  cfg may be NULL only if the input
   shape can be inferred (it cannot: pass cfg).  Allocates every device buffer, writes the
   initial weights and version-0 predictions (W_hat = W).  All-or-nothing: on failure
   *out = NULL and nothing stays allocated.  Errors: XP_EINVAL (shapes, partition,
   hyperparameters, unsupported DAG), XP_EUNSUPPORTED, XP_ENOMEM, XP_ECUDA. */
int xpipe_init(const xpipe_layer* layers, int32_t n_layers, int32_t stages, int32_t micro_batches,
               int32_t mini_batch, float lr, const float betas[2], float eps,
               const xpipe_config* cfg, struct xpipe_ctx** out);

/* Feed n_minibatches mini-batches into the running pipeline and execute every op whose
   inputs exist.  x: [M*N, C, H, W] fp32 NCHW (stage 0 reads it);
   y: [M*N] int32 labels in [0, classes) (the last stage reads them).  Host pointers
   unless XP_DEVICE_PTRS.  With XP_FLUSH the pipeline drains: afterwards every stage's
   version equals the number of mini-batches fed.  Splitting a sequence of mini-batches
   across calls (flush only at the end) gives bit-identical weights and traces.
   Errors: XP_EINVAL (labels out of range: checked on the host before any device work for host
   pointers, by the loss kernel for device pointers -- then reported at the end of the call, the
   affected rows got no one-hot term), XP_ECUDA, XP_ESCHED (watchdog), XP_ENONFINITE (a non-finite
   loss; the call's work completed).  With XP_ASYNC these device-side checks are reported by the
   next synchronous call; st->losses (when set) is then filled by an asynchronous copy, valid
   after the next synchronous call or xpipe_sync. */
int xpipe_step(struct xpipe_ctx* h, const float* x, const int32_t* y, int32_t n_minibatches,
               uint32_t flags, xpipe_stats* st);

/* Wait for all enqueued work (after XP_ASYNC). */
int xpipe_sync(struct xpipe_ctx* h);

/* Copy one parameter tensor (or its moment / prediction / gradient state) to dst as fp32
   in PyTorch layout.  count must equal the tensor size (else XP_EINVAL).  version: -1 =
   latest; otherwise a snapshot (cfg.snapshots, XP_S_PARAM only).  PRED_FWD returns the
   W_hat_f buffer of the latest version, PRED_BWD the W_hat_b buffer (bf16 values widened
   exactly in XP_BF16). */
int xpipe_get_weights(struct xpipe_ctx* h, int32_t layer, int32_t tensor, int32_t state,
                      int64_t version, float* dst, size_t count);

/* Overwrite one parameter tensor's state (XP_S_PARAM, XP_S_M, XP_S_V or XP_S_BUF) with src,
   fp32 in PyTorch layout, count = the tensor size (else XP_EINVAL).  Waits for the pipeline
   first; the W_hat buffers are NOT updated -- call xpipe_refresh_predictions after the last
   set.  Used for teacher-forced parity diagnostics: the oracle's state is
   loaded before each step.  XP_EINVAL for a stage of another process. */
int xpipe_set_weights(struct xpipe_ctx* h, int32_t layer, int32_t tensor, int32_t state, const float* src,
                      size_t count);

/* Recompute every owned stage's W_hat_f (buffer of the current version) and W_hat_b from its
   current W, m, v and version, as the update sweep would have (Eq. (3) with the stage's
   s_f / s_b).  Only between calls of a flushed pipeline (XP_ESTATE otherwise is not checked:
   the caller flushes). */
int xpipe_refresh_predictions(struct xpipe_ctx* h);

/* Number of trace records of a stage (*n_out) and up to cap of them (dst may be NULL). */
int xpipe_get_trace(struct xpipe_ctx* h, int32_t stage, xpipe_trace_rec* dst, size_t cap,
                    size_t* n_out);

/* Introspection: stage of a layer; current version of a stage (host mirror of the device
   counter); parameters of a stage (arena elements incl. alignment padding). */
int xpipe_stage_of_layer(struct xpipe_ctx* h, int32_t layer);
int xpipe_stage_version(struct xpipe_ctx* h, int32_t stage);
int64_t xpipe_stage_params(struct xpipe_ctx* h, int32_t stage);

/* Device timing across every stage stream: which = 0 records a start event on each stage's
   stream, which = 1 a stop event; after a stop, *ms_out (nullable) = max over stages of the
   device time between the two events (CUDA events on the streams the kernels run on). */
int xpipe_timer(struct xpipe_ctx* h, int32_t which, double* ms_out);

/* One-process-per-GPU mode (cfg.multi_process = 1).  Each process owns one stage; its
   input ring, gradient ring and flags are exported as CUDA IPC handles (xpipe_ipc_export
   writes an opaque blob of *len <= cap bytes, cap >= 4096) and every process imports the
   blobs of its neighbours (xpipe_ipc_import, any order, before the first xpipe_step).  The
   host logic never waits on another process: the device flags carry all ordering.
   Errors: XP_EINVAL (not in multi-process mode, foreign or malformed blob), XP_ECUDA. */
int xpipe_ipc_export(struct xpipe_ctx* h, void* blob, size_t cap, size_t* len);
int xpipe_ipc_import(struct xpipe_ctx* h, const void* blob, size_t len);

/* NULL-safe, idempotent; frees everything the context owns. */
int xpipe_finalize(struct xpipe_ctx* h);

/* Last error message of h (h == NULL: this thread's last init error). Never NULL. */
const char* xpipe_last_error(const struct xpipe_ctx* h);

/* The first n ops of stage `stage`'s program (reading R7) as the
   runtime executes them: ops[p] = 0 (forward) or 1 (backward) of micro-batch us[p] (1-based,
   an unbounded stream; the update follows B(u) exactly when u % micro_batches == 0).  Generated
   by the runtime's dependency-driven simulation (schedule.h); host-only, needs no GPU.
   schedule = XP_SCHED_XPIPE | XP_SCHED_GPIPE.  Errors: XP_EINVAL. */
int xpipe_schedule_program(int32_t stages, int32_t micro_batches, int32_t schedule, int32_t stage, int64_t n,
                           int32_t* ops, int64_t* us);

/* ---- kernel-level entry points (config 5 and unit parity) ----------------------------- */

/* K1, the fused Adam-update + weight-prediction sweep over n fp32 parameters (device
   pointers, 16-byte aligned).  Reads W, g, m, v once; writes W, m, v (in place) and
   W_hat_f = W' - s_f*d, W_hat_b = W' - s_b*d (either may be NULL) as fp32
   (pred_bf16 = 0) or bf16 (pred_bf16 = 1, round-to-nearest-even), where
   d = (c1*m')/(sqrt(v')*r2 + eps), c1 = lr/(1-b1^k), r2 = 1/sqrt(1-b2^k), k = version >= 1,
   beta^k by k repeated double multiplications.  stream: cudaStream_t
   (NULL = legacy default).  Asynchronous; errors: XP_EINVAL, XP_ECUDA (launch). */
int xpipe_adam_predict(float* W, const float* g, float* m, float* v, void* pred_f, void* pred_b,
                       int64_t n, int64_t version, float lr, float beta1, float beta2, float eps,
                       int32_t s_f, int32_t s_b, int32_t pred_bf16, int32_t delta_form, void* stream);

/* Kernel-level entry point of the f2 sweep (XP_OPT_MOMENTUM_SGD): one Momentum-SGD step with
   the Eq. (4) moments tracked alongside and the paper-literal prediction, over n device
   floats in place (W, buf, m, v; 16-byte aligned), predictions into pred_f / pred_b (bf16 if
   pred_bf16, else fp32; either may be NULL).  Op order: DESIGN.md "f2".  Errors: XP_EINVAL for
   NULL / misaligned pointers or n < 0; XP_ECUDA for a launch failure. */
int xpipe_sgd_predict(float* W, const float* g, float* buf, float* m, float* v, void* pred_f, void* pred_b,
                      int64_t n, float lr, float beta1, float beta2, float eps, float momentum, float weight_decay,
                      int32_t s_f, int32_t s_b, int32_t pred_bf16, void* stream /* cudaStream_t, NULL = default */);

/* bf16 tensor-core GEMM used by the conv/linear path, exposed for unit parity:
   D[M][N] (fp32, row-major, ldd) = sum_k A(m,k) * B(n,k) with A given row-major [M][K]
   (a_kmajor = 1) or [K][M] (0), B row-major [N][K] (b_kmajor = 1) or [K][N] (0); device
   pointers, bf16 inputs.  Asynchronous on stream. */
int xpipe_gemm_bf16(const void* A, const void* B, float* D, int32_t M, int32_t N, int32_t K,
                    int32_t a_kmajor, int32_t b_kmajor, int64_t ldd, void* stream);

/* Implicit-GEMM convolution on the same tensor-core path, exposed for unit parity.
   geo = {Nimg, H, W, C, Co, R, S, P, Q, sh, sw, ph, pw}: input NHWC [Nimg][H][W][C] bf16 (C a
   multiple of 8), weights KRSC [Co][R][S][C] bf16, output NHWC [Nimg][P][Q][Co].  mode:
   1 = fprop (in0 = X, in1 = W, out = Y bf16), 4 = the same through an explicit im2col operand
   (built in the upper half of ws, which must hold Nimg*P*Q*R*S*C bf16 there; the pipeline's path
   for geometries the TMA pixel boxes cannot serve), 5 = wgrad likewise (as 3),
   2 = dgrad (in0 = dY, in1 = W, out = dX bf16
   [Nimg][H][W][C]), 3 = wgrad (in0 = X, in1 = dY, out = dW fp32 [Co][R][S][C], accumulate
   adds into out).  ws: optional fp32 device workspace of ws_elems for split-K across
   several clusters (NULL = split-K within one thread-block cluster only); its last 16384
   elements hold the split-K arrival counters: they must be zero before the first call and
   every call leaves them zero (so zero the workspace once).  Dgrad of a geometry the TMA pixel
   boxes cannot serve (stride > 1, Co % 64 != 0, tile rows that are not a box of the input grid)
   builds its explicit operand in the upper half of ws when it fits there (else the implicit
   cp.async gather runs); 1x1 convs run as dense GEMMs.  Calls sharing one ws must be
   stream-ordered.  Device pointers; asynchronous on stream.  Errors: XP_EINVAL (bad
   geometry: C or Co not a multiple of 8, P/Q inconsistent), XP_ECUDA (launch). */
int xpipe_conv2d_bf16(int32_t mode, const int32_t geo[13], const void* in0, const void* in1, void* out,
                      int32_t accumulate, float* ws, int64_t ws_elems, void* stream);

/* bf16 Linear layer on the tensor cores (swap-AB: the features are the 128-row UMMA side, the
   micro-batch the narrow side; both operands by TMA), exposed for unit parity -- the ops the
   bf16 pipeline runs for every Linear with in % 8 == 0 (north star (b)).
   x [n][in] bf16, W [out][in] bf16 (PyTorch layout), in a multiple of 8.  mode:
   1 = forward: y[r][o] = sum_i W[o][i] x[r][i] + b[o] (fp32 accumulation; b may be NULL);
       y fp32 [n][out] if f32out, else bf16 [n][out] = Q(relu ? max(v, 0) : v).
   2 = dgrad: dx [n][in] bf16 = Q(sum_o dy[r][o] W[o][i]); dy [n][ldp] bf16, ldp a multiple of
       8, columns >= out zero.
   3 = wgrad: gW [out][in] fp32 (=, or += when accumulate) sum_r dy[r][o] x[r][i].
   ws: optional fp32 split-K workspace (as xpipe_conv2d_bf16, counters in its last 16384
   elements).  Device pointers; asynchronous on stream.  Errors: XP_EINVAL (in or ldp not a
   multiple of 8, ldp < out, n/in/out < 1), XP_ECUDA (launch). */
int xpipe_linear_bf16(int32_t mode, const void* x, const void* W, const void* b, const void* dy, int32_t ldp,
                      void* out, int32_t n, int32_t in, int32_t out_features, int32_t relu, int32_t f32out,
                      int32_t accumulate, float* ws, int64_t ws_elems, void* stream);

/* Development probe of the GEMM kernels (not part of the training path).  When the process
   runs with XPIPE_GEMM_DBG=1 every tensor-core GEMM launch records, per CTA c, 16 uint64 at
   host[16c ..]: globaltimer ns at start (after the PDL wait), first operand stage ready, all
   MMAs issued, accumulator ready, end; the SM id; the number of tiles the CTA processed; then
   (split-K only) partial parked in smem, first cluster barrier passed, cluster reduction done,
   cross-cluster reduction done.  Each launch overwrites the buffer.  Copies n values (synchronous).  Errors: XP_EINVAL (probe
   disabled or bad n), XP_ECUDA. */
int xpipe_dev_gemm_probe(unsigned long long* host, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* XPIPE_H */
