// runtime.h -- host-side context of the XPipe runtime (shared by xpipe.cu, blocks.cu, plan.cu).
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../include/xpipe.h"
#include "internal.h"
#include "plan.h"
#include "schedule.h"

#define XP_CUDA(c, call)                                                                           \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return set_err(c, XP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +     \
                                      std::to_string(__LINE__));                                   \
  } while (0)

#define XP_TRY(x)            \
  do {                       \
    int r_ = (x);            \
    if (r_ != XP_OK) return r_; \
  } while (0)


namespace xp {
// ----------------------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------------------
struct Alloc { void* p; size_t bytes; int dev; };

struct Snapshot { int ver; std::vector<float> W; float* pinned; };

// cfg.timing: one forward/backward op of a call and the indices (into StageRT::tstamp) of the
// stamps taken at its input arrival, compute end, hand-off end and op end (-1 = none)
struct TimedOp {
  int op = 0;
  int64_t u_rel = 0;   // micro-batch relative to the call's first fed micro-batch
  int e[4] = {-1, -1, -1, -1};
};

struct StageRT {
  int k = 0, dev = 0;
  cudaStream_t stream = nullptr;
  int l0 = 0, l1 = 0;
  StagePlan plan;                       // blocks, arena layout (plan.h)
  float *W = nullptr, *g = nullptr, *m = nullptr, *v = nullptr;
  float* buf = nullptr;                 // Momentum-SGD velocity (XP_OPT_MOMENTUM_SGD only)
  void* pf[2] = {nullptr, nullptr};
  void* pb = nullptr;
  DevState* ds = nullptr;
  int64_t* dbase = nullptr;             // multi-process graphs: the call's micro-batch base (device)
  uint32_t* flags = nullptr;            // [0] act_ready [1] grad_ready [2] act_ack [3] grad_ack
  int S = 1;                            // stash slots (max micro-batches in flight)
  // batched weight gradients (bf16 conv stages): a conv op's wgrad runs once per mini-batch, at
  // B(t,T), as one GEMM over the T micro-batches' stashed inputs (T consecutive, contiguous ring
  // slots: S is a multiple of T) and their conv-output gradients (dmid_all[op], [T][n*P*Q*Co])
  bool wbatch = false;
  std::vector<void*> dmid_all;          // [op] conv-output gradients of the mini-batch's T micro-batches
  int cur_j = 1, cur_slot0 = 0;         // the backward being enqueued: its j and its mini-batch's first slot
  void* in_ring = nullptr;              // contiguous ring allocations (IPC-exportable)
  void* gin_ring = nullptr;
  size_t in_stride = 0, gin_stride = 0;
  std::vector<void*> in_slot;           // input ring (R = S); = act[0]
  std::vector<void*> gin_slot;          // gradient ring (R = S), k < K-1
  std::vector<std::vector<void*>> act;  // [tensor][slot] stashed activations (tensor 0 = in_slot)
  std::vector<std::vector<void*>> mid;  // [op][slot] conv outputs before BN (bf16 path)
  std::vector<std::vector<float*>> stats;  // [op][slot] BN mean, rstd, gamma_f, beta_f
  std::vector<std::vector<uint8_t*>> pidx; // [op][slot] max-pool winner positions (conv op with pool)
  std::vector<float*> dz;               // [slot] logits gradient (last stage)
  std::vector<void*> grad;              // [tensor] activation-gradient buffers (per op pass)
  void* gmid = nullptr;                 // conv op: gradient of the conv output (bf16), buffer 0
  void* dcols = nullptr;                // explicit dgrad operand scratch (tc_dgrad_cols_elems), bf16
  int64_t dcols_elems = 0;
  void* lin_dy = nullptr;               // tensor-core Linear backward operand dyp [n][lin_ldp] bf16
  int lin_ldp = 0;
  void* gmid1 = nullptr;                //   buffer 1 (consecutive conv ops alternate; see side)
  // weight gradients run on a side stream, off the critical path of the backward chain
  // (bn-backward -> dgrad -> next op): forked after the op's BN backward, joined at the end of
  // the micro-batch's backward; conv op i waits for the wgrad of op i-2 before reusing its
  // gradient buffer.  The side stream has its own split-K workspace and counters.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_gdone[2] = {nullptr, nullptr};
  bool gdone_valid[2] = {false, false};
  int gsel = 0;
  bool side_used = false;
  float* ws_side = nullptr;
  int* ctr_side = nullptr;
  int64_t gbuf_elems = 0;
  // fb_overlap: forwards on their own stream with their own scratch (swapped in by FwdScope)
  cudaStream_t fstream = nullptr;
  float* ws_f = nullptr;
  int* ctr_f = nullptr;
  float* bnws_f = nullptr;
  std::vector<cudaEvent_t> ev_fdone, ev_bdone;  // per slot: F(u) done, B(u) done
  std::vector<int64_t> fdone_epoch, bdone_epoch;
  cudaEvent_t ev_upd = nullptr, ev_fmark = nullptr, ev_fjoin = nullptr;
  cudaEvent_t ev_in = nullptr;          // the call's input / label copies (main stream) are done
  // cfg.timing: per-op %globaltimer stamps (device buffer reused every call and by replayed
  // graphs, pinned host mirror) and the ops they belong to
  uint64_t* tstamp = nullptr;
  uint64_t* tstamp_host = nullptr;
  size_t tstamp_cap = 0, tev_used = 0;
  std::vector<TimedOp> tops;
  int64_t upd_epoch = -1;
  float* ws = nullptr;                  // split-K workspace (fp32)
  int64_t ws_elems = 0;
  float* bnws = nullptr;                // BatchNorm partial-reduction workspace
  std::vector<std::vector<void*>> cols; // per op, per slot: im2col of a few-channel conv input
  int* ctr = nullptr;                   // split-K arrival counters of this stage's stream
  // host program state
  int64_t pos = 0;
  bool done = false;
  int64_t fwd_enq = 0, bwd_enq = 0;     // last micro-batch whose F / B has been enqueued
  int host_ver = 0, host_fver = 0, host_bver = 0;
  // trace
  TraceRec* trace_dev = nullptr;
  int64_t trace_cap = 0, trace_n = 0;
  std::vector<Snapshot> snaps;
  std::vector<float*> snap_pool;         // pinned buffers reserved before enqueue
  void* diag = nullptr;                  // pinned scratch for watchdog diagnostics
  // profiling (cfg.profile): event pool and the (class, work) of each recorded pair
  std::vector<cudaEvent_t> ev_pool;
  std::vector<cudaEvent_t> ev_flag[4];  // per-slot events standing in for the flags inside graphs
  cudaEvent_t tmark[2] = {nullptr, nullptr};
  size_t ev_used = 0;
  std::vector<int> prof_cls;
  std::vector<double> prof_work;
};

}  // namespace xp

struct xpipe_ctx {
  using StageRT = xp::StageRT;
  using Alloc = xp::Alloc;
  using NetPlan = xp::NetPlan;
  std::string err;
  bool poisoned = false;
  NetPlan net;
  int K = 1, T = 1, N = 1, n = 1;
  float lr = 0, b1 = 0, b2 = 0, eps = 0;
  xpipe_config cfg{};
  std::vector<StageRT> S;
  xp::ScheduleSim sched;              // stage programs (a1), generated by simulation
  std::vector<Alloc> allocs;
  std::vector<void*> ipc_allocs;     // cudaMalloc'ed (exportable) rings/flags, multi-process mode
  std::vector<void*> ipc_opened;     // neighbour memory mapped with cudaIpcOpenMemHandle
  bool mp() const { return cfg.multi_process != 0; }
  // per-call buffers
  float* x_dev = nullptr; int64_t x_cap = 0;
  int32_t* y_dev = nullptr; int64_t y_cap = 0;
  float* loss_dev = nullptr; int64_t loss_cap = 0;
  // staging of host inputs for chained calls (one process): the next call's H2D copies run on
  // cstream while the previous call's graph executes; a device-to-device copy on the launch
  // stream then moves them into x_dev / y_dev at the call boundary
  float* x_stage = nullptr; int32_t* y_stage = nullptr; int64_t x_stage_cap = 0, y_stage_cap = 0;
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_stage_free = nullptr;
  int64_t fed = 0;           // micro-batches fed (absolute, 1-based count)
  int64_t base = 0;          // micro-batch offset of the current epoch
  int64_t call_first = 0;    // first micro-batch (absolute) of the current call's input buffer
  int64_t kernels = 0;
  int64_t flag_base = 0;     // flag values are micro-batch indices minus flag_base
  // CUDA graphs of steady-state steps (cfg.graphs): signature -> executable + host-state deltas
  struct GraphRec {
    cudaGraphExec_t exec = nullptr;
    int seen = 0;
    int64_t kernels = 0;
    std::vector<int64_t> dpos, dfwd, dbwd;
    std::vector<int> dver, dfver, dbver;
    std::vector<std::vector<xp::TimedOp>> tops;
    std::vector<size_t> tev_used;
    std::vector<std::vector<int>> prof_cls;
    std::vector<std::vector<double>> prof_work;
  };
  std::map<std::string, GraphRec> graphs;
  int64_t graph_replays = 0;
  bool capturing = false;
  bool recompute_pass = false;          // f3: op_forward is re-running a stage forward inside B(u)
  int64_t call_epoch = 0;               // bumped per call: events recorded in earlier calls are complete
  float* loss_scratch = nullptr;        // the recomputed forward's loss (the reported loss is F(u)'s)
  uint32_t* status_dev = nullptr;       // last stage: XP_STATUS_* bits set by the loss kernel
  uint32_t* status_host = nullptr;      // pinned mirror read after a synchronous call
  std::vector<int64_t> cap_fwd0, cap_bwd0;  // enqueue counters when the capture started
  int64_t cap_base = 0;                 // multi-process capture: fed_before of the captured call
  int64_t calls = 0;                    // xpipe_step calls so far (cfg.timing sampling)
  bool timed = false;                   // this call is stamped (cfg.timing)
  bool chain_ok = false;                // the last call was an asynchronous graph replay (XP_ASYNC)
  bool graph_launched = false;          // this call's work went out as one graph launch
  std::vector<std::pair<int64_t, int64_t>> loss_map;  // (u, index into loss_dev)
};


namespace xp {
// blocks.cu
void* dmalloc(xpipe_ctx* c, size_t bytes, int dev);
void* dmalloc_shared(xpipe_ctx* c, size_t bytes, int dev);  // IPC-exportable in multi-process mode
inline bool owned(const StageRT& s) { return s.stream != nullptr; }
int set_err(xpipe_ctx* c, int code, const std::string& m);
int check_launch(xpipe_ctx* c, cudaError_t e, const char* what);
int allocate_stage(xpipe_ctx* c, StageRT& s);
int init_stage_params(xpipe_ctx* c, StageRT& s, const xpipe_layer* layers);
int stage_input(xpipe_ctx* c, StageRT& s, const float* x_nchw, void* dst);
// forward of op o on micro-batch slot under Wf (writes act[o.out][slot])
int op_forward(xpipe_ctx* c, StageRT& s, int o, const void* Wf, int slot, int64_t u);
// backward of op o: dy = gradient of its output; writes/accumulates the input gradients
// (dx0/dx1 may be NULL when not needed; acc0/acc1 = add into an existing contribution)
int op_backward(xpipe_ctx* c, StageRT& s, int o, const void* dy, void* dx0, bool acc0, void* dx1, bool acc1,
                const void* Wb, int slot, bool accumulate_g);
// bf16_blocks.cu
int bf16_op_forward(xpipe_ctx* c, StageRT& s, int o, const void* Wf, int slot);
int bf16_op_backward(xpipe_ctx* c, StageRT& s, int o, const void* dy, void* dx0, bool acc0, void* dx1, bool acc1,
                     const void* Wb, int slot, bool accumulate_g);
// xpipe.cu
int version_difference(const xpipe_ctx* c, int k, int pass);
int version_difference_public(const xpipe_ctx* c, int k, int pass);
// profiling: bracket one kernel launch on s.stream (no-ops unless cfg.profile)
int prof_begin(xpipe_ctx* c, StageRT& s, cudaStream_t st = nullptr);  // st: default the stage stream
int prof_end(xpipe_ctx* c, StageRT& s, int cls, double work, cudaStream_t st = nullptr);
}  // namespace xp
