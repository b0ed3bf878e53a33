// internal.h -- declarations shared by the host runtime (xpipe.cu) and the kernels.
// Product code only; nothing here is shared with oracle/.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace xp {

// Per-stage device state (K12 bookkeeping + the sweep's scalars).  The version counter
// lives on the device so a captured CUDA graph replays correctly; the host keeps a mirror.
struct DevState {
  int32_t ver;      // current weight version of the stage (number of updates applied)
  int32_t fver;     // version the current forward bellwether predicted from
  int32_t bver;     // version the current backward bellwether predicted from
  int32_t pad;
  double b1p, b2p;  // beta1^ver, beta2^ver by repeated multiplication
  float c1, r2;     // lr/(1-b1^ver), 1/sqrt(1-b2^ver) rounded to fp32
  float omb1, omb2; // 1-b1, 1-b2 (fp32)
  float inv1, inv2; // 1/(1-b1), 1/(1-b2) (paper delta form)
  float lr, b1, b2, eps;
  float mu, wd;     // Momentum-SGD momentum and weight decay (XP_OPT_MOMENTUM_SGD, f2)
};

// Scalars of one sweep launch (host-computed for the standalone entry point).
struct SweepScalars {
  float c1, r2, omb1, omb2, inv1, inv2, lr, b1, b2, eps, mu, wd;
};

struct TraceRec {  // identical layout to xpipe_trace_rec
  int32_t stage, op, t, j, version, s, bellwether, wbuf;
  uint64_t t0_ns, t1_ns;
};

// ---- K1: fused Adam + prediction sweep (kernels/sweep.cu) --------------------------------
// Scalars come from ds (device) when ds != nullptr, else from *hs.
cudaError_t launch_sweep(float* W, const float* g, float* m, float* v, void* pf, void* pb, int64_t n,
                         const DevState* ds, const SweepScalars* hs, float s_f, float s_b, bool bf16,
                         int delta_form, bool update, cudaStream_t st);
// f2: Momentum-SGD step (buf = mu*buf + (g + wd*W), W -= lr*buf) with the Eq. (4) moments
// tracked alongside and the paper-literal prediction dW (Eq. (3)/(4)), one pass
cudaError_t launch_sweep_sgd(float* W, const float* g, float* buf, float* m, float* v, void* pf, void* pb, int64_t n,
                             const DevState* ds, const SweepScalars* hs, float s_f, float s_b, bool bf16,
                             cudaStream_t st);
// W_hat = W converted (version 0 with zero moments: no delta)
cudaError_t launch_predict_copy(const float* W, void* pf, void* pb, int64_t n, bool bf16, cudaStream_t st);
// version bump before an update: ver += 1, beta powers, c1, r2 (1 thread)
cudaError_t launch_bump(DevState* ds, TraceRec* rec, int stage, int t, int T, cudaStream_t st);
cudaError_t launch_state_init(DevState* ds, float lr, float b1, float b2, float eps, float mu, float wd,
                              cudaStream_t st);
void host_scalars(int64_t k, float lr, float b1, float b2, float eps, SweepScalars* out);

// ---- misc kernels (kernels/f32.cu) -----------------------------------------------------
cudaError_t launch_trace_begin(DevState* ds, TraceRec* rec, int stage, int op, int t, int j, int s, int bw,
                               cudaStream_t st);
cudaError_t launch_trace_end(TraceRec* rec, cudaStream_t st);
cudaError_t launch_stamp(uint64_t* dst, cudaStream_t st);
// ring flags inside graphs of the one-process-per-GPU mode: wait until / write *base + rel
cudaError_t launch_flag_wait(const uint32_t* flag, const int64_t* base, int32_t rel, cudaStream_t st);
cudaError_t launch_flag_write(uint32_t* flag, const int64_t* base, int32_t rel, cudaStream_t st);
cudaError_t launch_set_i64(int64_t* dst, int64_t v, cudaStream_t st);  // *dst = %globaltimer after the stream's prior work
cudaError_t launch_rebase_flags(uint32_t* flags, int n, uint32_t delta, cudaStream_t st);
cudaError_t launch_fill_uniform(float* dst, int64_t n, float bound, uint64_t seed, uint64_t stream_id,
                                cudaStream_t st);
cudaError_t launch_fill_const(float* dst, int64_t n, float value, cudaStream_t st);

// fp32 contract kernels (C1): see DESIGN.md section 4 for the frozen op order.
cudaError_t launch_linear_fwd_f32(const float* x, const float* W, const float* b, float* y, int n, int in,
                                  int out, bool relu, cudaStream_t st);
// dx[r][i] = sum_o fmaf(dy'[r][o], W[o][i]) with dy' = (ymask[r][o] > 0 ? dy : 0) if ymask
cudaError_t launch_linear_dgrad_f32(const float* dy, const float* ymask, const float* W, float* dx, int n,
                                    int in, int out, cudaStream_t st);
// g[o][i] (=|+=) sum_r fmaf(dy'[r][o], x[r][i]); gb[o] (=|+=) sum_r dy'[r][o]
cudaError_t launch_linear_wgrad_f32(const float* dy, const float* ymask, const float* x, float* gW, float* gb,
                                    int n, int in, int out, bool accumulate, cudaStream_t st);
// softmax cross-entropy: dz[r][c] = (p - onehot) * invN; loss[0] = mean_r -log p_y; one CTA,
// one thread per row (n <= kXentMaxRows); status bits below are OR-ed into *status (nullable)
constexpr int kXentMaxRows = 256;
enum { XP_STATUS_NONFINITE = 1, XP_STATUS_LABEL = 2 };
cudaError_t launch_xent_f32(const float* z, const int32_t* y, float* dz, float* loss, int n, int classes,
                            float invN, uint32_t* status, cudaStream_t st);

// ---- bf16 path (kernels/bf16.cu, kernels/gemm_tc.cu) -----------------------------------
// NCHW fp32 -> NHWC bf16 with the channel count padded to Cp (zeros)
cudaError_t launch_stage_input_bf16(const float* x, __nv_bfloat16* y, int n, int C, int H, int W, int Cp,
                                    cudaStream_t st);

}  // namespace xp
