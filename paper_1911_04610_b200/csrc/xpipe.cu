// xpipe.cu -- host runtime of the B200-native XPipe hot path and its C ABI (include/xpipe.h).
//
// One CUDA stream per pipeline stage (stage k on devices[k % n_devices]).  The host turns
// every stage's program (reading R7: K-k warm-up forwards, then B(i),
// F(i+K-k) pairs, then drain; or GPipe) into stream work in program order; ordering
// between stages is carried entirely by device-side 32-bit flags written and waited with
// CUDA stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32):
//   act_ready[k]  = last micro-batch u whose activation message reached stage k's ring
//   grad_ready[k] = last micro-batch u whose gradient message reached stage k's ring
//   act_ack[k]    = last u whose activation message stage k+1 released (ring credit)
//   grad_ack[k]   = last u whose gradient message stage k-1 released (ring credit)
// so the host never blocks on another stage, a stage never spins on an SM, and the same
// code drives K stages on one GPU, on K GPUs (peer copies over NVLink), or -- with the
// rings/flags mapped through CUDA IPC -- one process per GPU.
//
// Messages (a5, a8) are copied by the copy engine (cudaMemcpyAsync, same-device or peer)
// from the producer's local stash into the consumer's ring slot, then the flag is written
// (the write value op orders after the copy).  Ring slots double as the consumer's stash of
// its first layer's input.  The fused Adam+prediction sweep (K1) runs after B(t,T) and
// materialises W_hat_f[(v+1) & 1] and W_hat_b of the new version.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/xpipe.h"
#include "kernels/gemm_tc.h"
#include "runtime.h"

using namespace xp;

// ----------------------------------------------------------------------------------------
// driver entry points (no link-time dependency on libcuda: the .so loads without a GPU)
// ----------------------------------------------------------------------------------------
namespace {
typedef int (*PFN_waitValue32)(cudaStream_t, unsigned long long, uint32_t, unsigned int);
typedef int (*PFN_writeValue32)(cudaStream_t, unsigned long long, uint32_t, unsigned int);
PFN_waitValue32 p_wait32 = nullptr;
PFN_writeValue32 p_write32 = nullptr;

bool load_driver_entry_points() {
  if (p_wait32 && p_write32) return true;
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return false;
  p_wait32 = (PFN_waitValue32)f;
  f = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return false;
  p_write32 = (PFN_writeValue32)f;
  return true;
}

thread_local std::string g_init_error;
}  // namespace

namespace xp {

int set_err(xpipe_ctx* c, int code, const std::string& m) {
  if (c) {
    c->err = m;
    if (code == XP_ECUDA || code == XP_ECOMM || code == XP_ESCHED) c->poisoned = true;
  } else {
    g_init_error = m;
  }
  return code;
}

void* dmalloc(xpipe_ctx* c, size_t bytes, int dev) {
  if (bytes == 0) bytes = 256;
  bytes = (bytes + 255) & ~size_t(255);
  void* p = nullptr;
  if (c->cfg.alloc) {
    p = c->cfg.alloc(bytes, dev, c->cfg.alloc_user);
  } else {
    cudaSetDevice(dev);
    if (cudaMalloc(&p, bytes) != cudaSuccess) p = nullptr;
  }
  if (p) c->allocs.push_back({p, bytes, dev});
  return p;
}

void* dmalloc_shared(xpipe_ctx* c, size_t bytes, int dev) {
  if (!c->mp()) return dmalloc(c, bytes, dev);
  bytes = (bytes + 255) & ~size_t(255);
  void* p = nullptr;
  cudaSetDevice(dev);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  c->ipc_allocs.push_back(p);
  return p;
}

void free_all(xpipe_ctx* c) {
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  c->graphs.clear();
  for (auto& s : c->S) {
    for (auto& sn : s.snaps) if (sn.pinned) cudaFreeHost(sn.pinned);
    s.snaps.clear();
    for (auto p : s.snap_pool) cudaFreeHost(p);
    s.snap_pool.clear();
    if (s.diag) { cudaFreeHost(s.diag); s.diag = nullptr; }
    for (auto e : s.ev_pool) cudaEventDestroy(e);
    s.ev_pool.clear();
    if (s.tstamp_host) { cudaFreeHost(s.tstamp_host); s.tstamp_host = nullptr; }
    for (auto& v : s.ev_flag) { for (auto e : v) cudaEventDestroy(e); v.clear(); }
    for (auto& e : s.tmark) if (e) { cudaEventDestroy(e); e = nullptr; }
    // a serialised context shares stage 0's stream: destroy each stream once
    const bool shared = c->cfg.serialize && !c->mp() && s.k > 0 && s.dev == c->S[0].dev;
    const bool own_fstream = s.fstream && s.fstream != s.stream;
    if (s.side && s.side != s.stream && !shared) {
      cudaSetDevice(s.dev); cudaStreamSynchronize(s.side); cudaStreamDestroy(s.side);
    }
    s.side = nullptr;
    if (shared) s.stream = nullptr;
    for (cudaEvent_t* e : {&s.ev_fork, &s.ev_join, &s.ev_gdone[0], &s.ev_gdone[1], &s.ev_upd, &s.ev_fmark, &s.ev_fjoin,
                           &s.ev_in})
      if (*e) { cudaEventDestroy(*e); *e = nullptr; }
    for (auto* v : {&s.ev_fdone, &s.ev_bdone}) { for (auto e : *v) if (e) cudaEventDestroy(e); v->clear(); }
    if (own_fstream) {
      cudaSetDevice(s.dev); cudaStreamSynchronize(s.fstream); cudaStreamDestroy(s.fstream);
    }
    s.fstream = nullptr;
    if (s.stream) { cudaSetDevice(s.dev); cudaStreamSynchronize(s.stream); cudaStreamDestroy(s.stream); s.stream = nullptr; }
  }
  if (c->cstream) {
    cudaStreamSynchronize(c->cstream);
    cudaStreamDestroy(c->cstream);
    c->cstream = nullptr;
  }
  for (cudaEvent_t* e : {&c->ev_staged, &c->ev_stage_free})
    if (*e) { cudaEventDestroy(*e); *e = nullptr; }
  if (c->status_host) { cudaFreeHost(c->status_host); c->status_host = nullptr; }
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  c->ipc_opened.clear();
  for (void* p : c->ipc_allocs) cudaFree(p);
  c->ipc_allocs.clear();
  for (auto it = c->allocs.rbegin(); it != c->allocs.rend(); ++it) {
    if (c->cfg.free) c->cfg.free(it->p, it->bytes, it->dev, c->cfg.alloc_user);
    else { cudaSetDevice(it->dev); cudaFree(it->p); }
  }
  c->allocs.clear();
}

int check_launch(xpipe_ctx* c, cudaError_t e, const char* what) {
  c->kernels++;
  if (e != cudaSuccess) return set_err(c, XP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return XP_OK;
}

}  // namespace xp

namespace xp {
// Eq. (1) P:104-109 / Eq. (2) P:111-115 with half-up rounding (R3), integer form:
//   s_f = floor((2K + 3T - 4 - k) / (2T)),  s_b = floor((3T + 2*floor(k/2) - 2) / (2T))
int version_difference(const xpipe_ctx* c, int k, int pass) {
  if (c->cfg.predict == XP_PRED_OFF) return 0;
  if (c->cfg.predict == XP_PRED_FIXED) return pass == 0 ? c->cfg.s_fwd : c->cfg.s_bwd;
  const int K = c->K, T = c->T;
  int s = pass == 0 ? (2 * K + 3 * T - 4 - k) / (2 * T) : (3 * T + 2 * (k / 2) - 2) / (2 * T);
  return s < 0 ? 0 : s;
}

int version_difference_public(const xpipe_ctx* c, int k, int pass) { return version_difference(c, k, pass); }

int prof_begin(xpipe_ctx* c, StageRT& s, cudaStream_t st) {
  if (!c->cfg.profile) return XP_OK;
  if (!st) st = s.stream;
  while (s.ev_pool.size() < s.ev_used + 2) {
    cudaEvent_t e;
    XP_CUDA(c, cudaEventCreate(&e));
    s.ev_pool.push_back(e);
  }
  // external record: inside a stream capture this becomes an event-record node of the graph
  if (c->capturing) XP_CUDA(c, cudaEventRecordWithFlags(s.ev_pool[s.ev_used], st, cudaEventRecordExternal));
  else XP_CUDA(c, cudaEventRecord(s.ev_pool[s.ev_used], st));
  return XP_OK;
}

int prof_end(xpipe_ctx* c, StageRT& s, int cls, double work, cudaStream_t st) {
  if (!c->cfg.profile) return XP_OK;
  if (!st) st = s.stream;
  if (c->capturing) XP_CUDA(c, cudaEventRecordWithFlags(s.ev_pool[s.ev_used + 1], st, cudaEventRecordExternal));
  else XP_CUDA(c, cudaEventRecord(s.ev_pool[s.ev_used + 1], st));
  s.ev_used += 2;
  s.prof_cls.push_back(cls);
  s.prof_work.push_back(work);
  return XP_OK;
}
// cfg.timing: take the next %globaltimer stamp of stage s on stream st (a 1-thread kernel after
// the stream's prior work; inside a captured graph it is replayed with the same slot);
// *idx = its slot (or -1 when timing is off or `want` is false)
int tmark(xpipe_ctx* c, StageRT& s, cudaStream_t st, int* idx, bool want = true) {
  *idx = -1;
  if (!c->timed || !want) return XP_OK;
  if (s.tev_used >= s.tstamp_cap) return set_err(c, XP_ESCHED, "timing stamp buffer (internal)");
  XP_TRY(check_launch(c, launch_stamp(s.tstamp + s.tev_used, st), "stamp"));
  *idx = (int)s.tev_used++;
  return XP_OK;
}
}  // namespace xp

namespace {

// development switch: XPIPE_NO_WGRAD_BATCH=1 runs the conv weight gradients per micro-batch
bool no_wgrad_batch() {
  static const bool v = [] { const char* e = getenv("XPIPE_NO_WGRAD_BATCH"); return e && *e && *e != '0'; }();
  return v;
}

// the activation-ring credit a producer waits for before writing message u into stage q's ring:
// q released message u - S_q; with batched weight gradients q releases a mini-batch's slots
// together, at its B(t,T) (flag value t*T)
int64_t ring_credit(const xpipe_ctx* c, const StageRT& q, int64_t u) {
  int64_t v = u - q.S;
  if (q.wbatch && v > 0) v = (v + c->T - 1) / c->T * c->T;  // acks are written at multiples of T
  return v;
}

// Flag values are micro-batch indices relative to c->flag_base (rebased between calls when
// CUDA graphs are on); GEQ compares the wraparound-safe signed difference, so rebased values
// may go negative.
bool verbose() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("XPIPE_VERBOSE"); v = (e && *e && *e != '0') ? 1 : 0; }
  return v == 1;
}

// Cross-stage dependency on ring flag `which` of stage s (0 act_ready, 1 grad_ready,
// 2 act_ack, 3 grad_ack) reaching micro-batch `value`.  Normally a device-side memop wait.
// While a CUDA graph is being captured it becomes a graph edge (wait on the per-slot event the
// producer recorded), and waits on producers enqueued before this call are dropped (every
// earlier op completed before the call started).
int flag_wait(xpipe_ctx* c, StageRT& s, int which, int64_t value) {
  uint32_t* flag = &s.flags[which];
  if (verbose()) fprintf(stderr, "[xpipe] stage %d wait %d(%p) >= %lld%s\n", s.k, which, (void*)flag, (long long)value,
                         value <= 0 ? " (skip)" : "");
  if (value <= 0) return XP_OK;  // absolute: that message never existed
  if (c->capturing && c->mp()) {  // another process writes the flag: device-side wait on base + rel
    XP_TRY(check_launch(c, launch_flag_wait(flag, s.dbase, (int32_t)(value - c->cap_base), s.stream), "flag_wait"));
    return XP_OK;
  }
  if (c->capturing) {
    // producer's enqueue counter at capture start: waits on earlier messages are satisfied
    const int prod = (which == 0 || which == 3) ? s.k - 1 : s.k + 1;
    const int64_t before = (which == 0) ? c->cap_fwd0[prod] : c->cap_bwd0[prod];
    if (value <= before) return XP_OK;
    auto& evs = s.ev_flag[which];
    XP_CUDA(c, cudaStreamWaitEvent(s.stream, evs[(value - 1) % evs.size()], 0));
    return XP_OK;
  }
  int r = p_wait32(s.stream, (unsigned long long)(uintptr_t)flag, (uint32_t)(value - c->flag_base), 0 /*GEQ*/);
  if (r != 0) return set_err(c, XP_ECOMM, "cuStreamWaitValue32 failed: " + std::to_string(r));
  return XP_OK;
}

// producer side: set ring flag `which` of stage `tgt` to `value` from stream s (memop write,
// ordered after the preceding work); while capturing also record the per-slot event
int flag_write(xpipe_ctx* c, StageRT& s, StageRT& tgt, int which, int64_t value) {
  uint32_t* flag = &tgt.flags[which];
  if (verbose()) fprintf(stderr, "[xpipe] stage %d write stage %d flag %d(%p) = %lld\n", s.k, tgt.k, which, (void*)flag,
                         (long long)value);
  if (c->capturing && c->mp()) {
    return check_launch(c, launch_flag_write(flag, s.dbase, (int32_t)(value - c->cap_base), s.stream), "flag_write");
  }
  if (c->capturing) {
    auto& evs = tgt.ev_flag[which];
    XP_CUDA(c, cudaEventRecord(evs[(value - 1) % evs.size()], s.stream));
  }
  int r = p_write32(s.stream, (unsigned long long)(uintptr_t)flag, (uint32_t)(value - c->flag_base),
                    0 /*DEFAULT: with barrier*/);
  if (r != 0) return set_err(c, XP_ECOMM, "cuStreamWriteValue32 failed: " + std::to_string(r));
  return XP_OK;
}

// ---- stage program (a1; R7) ------------------------------------------------------------------
// op (0 = F, 1 = B) and micro-batch u (absolute, 1-based) at program position p of stage k, from
// the dependency-driven schedule simulation (schedule.h)
void program_op(xpipe_ctx* c, int k, int64_t p, int* op, int64_t* u) {
  c->sched.op_at(k, p, op, u);
  *u += c->base;
}

void reset_schedule(xpipe_ctx* c) {
  std::vector<bool> rec;
  for (const auto& s : c->S) rec.push_back(owned(s));
  c->sched.reset(c->K, c->T, c->cfg.schedule == XP_SCHED_GPIPE, rec);
}

int trace_slot(xpipe_ctx* c, StageRT& s, TraceRec** rec) {
  *rec = nullptr;
  if (!c->cfg.trace) return XP_OK;
  if (s.trace_n >= s.trace_cap) return set_err(c, XP_ESCHED, "trace capacity (internal)");
  *rec = s.trace_dev + s.trace_n++;
  return XP_OK;
}

// Everything that can allocate (and so implicitly synchronise the device) happens here,
// before any op of the call is enqueued: once stream work waits on a flag that only later
// work writes, a device-wide synchronisation would deadlock the pipeline.
int reserve_for_call(xpipe_ctx* c, int64_t M) {
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    if (c->cfg.trace) {
      const int64_t need = 3 * (c->fed + c->T) + 64;  // <= 2 ops per micro-batch + 1 update per mini-batch
      if (need > s.trace_cap) {
        const int64_t cap = std::max<int64_t>(need, 2 * s.trace_cap);
        TraceRec* nt = (TraceRec*)dmalloc(c, cap * sizeof(TraceRec), s.dev);
        if (!nt) return set_err(c, XP_ENOMEM, "trace buffer");
        cudaSetDevice(s.dev);
        if (s.trace_n) XP_CUDA(c, cudaMemcpy(nt, s.trace_dev, s.trace_n * sizeof(TraceRec), cudaMemcpyDeviceToDevice));
        s.trace_dev = nt;
        s.trace_cap = cap;
      }
    }
    if (c->cfg.profile) {
      int nconv = 0;
      for (const Op& O : s.plan.ops) nconv += O.kind == OP_CONV;
      const size_t want = (size_t)2 * (3 * nconv + 1) * (size_t)(M * c->T + c->K + 1);
      while (s.ev_pool.size() < want) {
        cudaEvent_t e;
        XP_CUDA(c, cudaEventCreate(&e));
        s.ev_pool.push_back(e);
      }
    }
    if (c->cfg.timing) {
      const size_t want = (size_t)4 * (2 * (M * c->T + 2 * c->K + c->T) + 8);
      if (s.tstamp_cap < want) {
        // captured graphs hold the old buffer's addresses: drop them (re-captured on demand)
        for (auto& kv : c->graphs)
          if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        c->graphs.clear();
        const size_t cap = std::max(want, 2 * s.tstamp_cap);
        s.tstamp = (uint64_t*)dmalloc(c, cap * 8, s.dev);
        if (s.tstamp_host) cudaFreeHost(s.tstamp_host);
        s.tstamp_host = nullptr;
        if (!s.tstamp || cudaMallocHost(&s.tstamp_host, cap * 8) != cudaSuccess)
          return set_err(c, XP_ENOMEM, "timing stamps");
        s.tstamp_cap = cap;
      }
    }
    if (c->cfg.snapshots) {
      const size_t want = (size_t)(M + c->K + 1);
      while (s.snap_pool.size() < want) {
        float* p = nullptr;
        XP_CUDA(c, cudaMallocHost(&p, s.plan.P * sizeof(float)));
        s.snap_pool.push_back(p);
      }
    }
  }
  return XP_OK;
}

// ---- fb_overlap plumbing -------------------------------------------------------------------
// A forward runs on the stage's forward stream with the forward scratch (split-K workspace,
// counters, BN partials) swapped in, so every launcher below uses them unchanged.
struct FwdScope {
  StageRT& s;
  bool on;
  explicit FwdScope(StageRT& st) : s(st), on(st.fstream && st.fstream != st.stream) { if (on) swap(); }
  ~FwdScope() { if (on) swap(); }
  void swap() {
    std::swap(s.stream, s.fstream);
    std::swap(s.ws, s.ws_f);
    std::swap(s.ctr, s.ctr_f);
    std::swap(s.bnws, s.bnws_f);
  }
};
// events between a stage's two streams; an event recorded in an earlier call is complete (every
// call starts from a drained pipeline), so waiting on it is skipped -- which also keeps graph
// captures free of edges to work outside the capture
int ev_record(xpipe_ctx* c, cudaStream_t st, cudaEvent_t e, int64_t* epoch) {
  XP_CUDA(c, cudaEventRecord(e, st));
  *epoch = c->call_epoch;
  return XP_OK;
}
int ev_wait(xpipe_ctx* c, cudaStream_t st, cudaEvent_t e, int64_t epoch) {
  if (epoch != c->call_epoch) return XP_OK;
  XP_CUDA(c, cudaStreamWaitEvent(st, e, 0));
  return XP_OK;
}
// make the stage stream's completion imply the forward stream's (end of a drive)
int join_fstreams(xpipe_ctx* c) {
  for (auto& s : c->S) {
    if (!owned(s) || !s.fstream || s.fstream == s.stream) continue;
    cudaSetDevice(s.dev);
    XP_CUDA(c, cudaEventRecord(s.ev_fjoin, s.fstream));
    XP_CUDA(c, cudaStreamWaitEvent(s.stream, s.ev_fjoin, 0));
  }
  return XP_OK;
}

// ---- forward / backward of one stage on one micro-batch -----------------------------------
int enqueue_forward(xpipe_ctx* c, int k, int64_t u) {
  StageRT& s = c->S[k];
  cudaSetDevice(s.dev);
  FwdScope fwd(s);  // fb_overlap: from here s.stream is the forward stream
  if (fwd.on) {
    const int slot0 = (int)((u - 1) % s.S);
    XP_TRY(ev_wait(c, s.stream, s.ev_bdone[slot0], s.bdone_epoch[slot0]));  // B(u - S) freed the slot
    const int64_t t0 = (u - 1) / c->T + 1;
    if (u - (t0 - 1) * c->T == 1) XP_TRY(ev_wait(c, s.stream, s.ev_upd, s.upd_epoch));  // W_hat_f of the version
  }
  const int64_t t = (u - 1) / c->T + 1, j = u - (t - 1) * c->T;
  const int slot = (int)((u - 1) % s.S);
  const int sf = version_difference(c, k, 0);
  const bool bw = (j == 1);
  cudaSetDevice(s.dev);
  // input: stage 0 stages the call's input into its stash slot; others wait for the message
  TimedOp top;
  top.op = 0;
  top.u_rel = u - c->call_first;
  if (k == 0) {
    XP_TRY(tmark(c, s, s.stream, &top.e[0]));
    const int64_t per = (int64_t)c->cfg.in_c * c->cfg.in_h * c->cfg.in_w;
    const float* src = c->x_dev + (u - c->call_first) * c->n * per;
    XP_TRY(stage_input(c, s, src, s.in_slot[slot]));
  } else {
    XP_TRY(flag_wait(c, s, 0, u));
    XP_TRY(tmark(c, s, s.stream, &top.e[0]));
  }
  TraceRec* rec = nullptr;
  XP_TRY(trace_slot(c, s, &rec));
  if (rec) XP_TRY(check_launch(c, launch_trace_begin(s.ds, rec, k, 0, (int)t, (int)j, sf, bw, s.stream), "trace"));
  if (bw) s.host_fver = s.host_ver;
  const void* Wf = s.pf[s.host_fver & 1];
  for (size_t o = 0; o < s.plan.ops.size(); ++o) XP_TRY(op_forward(c, s, (int)o, Wf, slot, u));
  // hand-off timing is sampled on the bellwether micro-batches (1 in T) to keep stamps few
  XP_TRY(tmark(c, s, s.stream, &top.e[1], bw && k + 1 < c->K));
  if (k + 1 < c->K) {
    StageRT& nx = c->S[k + 1];
    XP_TRY(flag_wait(c, s, 2, ring_credit(c, nx, u)));  // ring credit: consumer released u - R
    XP_CUDA(c, cudaMemcpyAsync(nx.in_slot[(u - 1) % nx.S], s.act[s.plan.out_tensor][slot], s.plan.out_bytes,
                               cudaMemcpyDefault, s.stream));
    XP_TRY(flag_write(c, s, nx, 0, u));
  }
  XP_TRY(tmark(c, s, s.stream, &top.e[3]));  // the op's end
  if (c->timed) s.tops.push_back(top);
  if (rec) XP_TRY(check_launch(c, launch_trace_end(rec, s.stream), "trace"));
  if (fwd.on) XP_TRY(ev_record(c, s.stream, s.ev_fdone[slot], &s.fdone_epoch[slot]));
  return XP_OK;
}

int enqueue_backward(xpipe_ctx* c, int k, int64_t u) {
  StageRT& s = c->S[k];
  const int64_t t = (u - 1) / c->T + 1, j = u - (t - 1) * c->T;
  const int slot = (int)((u - 1) % s.S);
  const int sb = version_difference(c, k, 1);
  const bool bw = (j == 1);
  cudaSetDevice(s.dev);
  const bool ov = s.fstream && s.fstream != s.stream;
  if (ov) XP_TRY(ev_wait(c, s.stream, s.ev_fdone[slot], s.fdone_epoch[slot]));  // F(u) on the forward stream
  if (k + 1 < c->K) XP_TRY(flag_wait(c, s, 1, u));
  TimedOp top;
  top.op = 1;
  top.u_rel = u - c->call_first;
  XP_TRY(tmark(c, s, s.stream, &top.e[0]));
  TraceRec* rec = nullptr;
  XP_TRY(trace_slot(c, s, &rec));
  if (rec) XP_TRY(check_launch(c, launch_trace_begin(s.ds, rec, k, 1, (int)t, (int)j, sb, bw, s.stream), "trace"));
  if (bw) s.host_bver = s.host_ver;
  if (bw && c->cfg.wbwd == XP_WBWD_BELLWETHER) {
    // the backward bellwether predicts W_hat_b from the stage's current state (version
    // t-1: no update falls between B(t,1) and B(t,T)); the other T-1 backwards reuse it
    const bool bf = c->cfg.precision == XP_BF16;
    XP_TRY(prof_begin(c, s));
    if (c->cfg.delta_form == XP_DELTA_ADAM && s.host_ver == 0)
      XP_TRY(check_launch(c, launch_predict_copy(s.W, nullptr, s.pb, s.plan.P, bf, s.stream), "predict_b"));
    else
      XP_TRY(check_launch(c, launch_sweep(s.W, s.g, s.m, s.v, nullptr, s.pb, s.plan.P, s.ds, nullptr, 0.f, (float)sb, bf,
                                          c->cfg.delta_form, false, s.stream), "predict_b"));
    XP_TRY(prof_end(c, s, XP_PROF_SWEEP, (double)s.plan.P * (12.0 + (bf ? 2.0 : 4.0))));
  }
  if (c->cfg.recompute) {
    // f3: re-run the stage forward for this micro-batch under W_hat_b from its stashed
    // input (ring slot), overwriting the slot's activations, statistics and pool winners (and
    // on the last stage dz) -- the backward below then differentiates this forward exactly
    c->recompute_pass = true;
    int r = XP_OK;
    for (size_t o = 0; o < s.plan.ops.size() && r == XP_OK; ++o) r = op_forward(c, s, (int)o, s.pb, slot, u);
    c->recompute_pass = false;
    XP_TRY(r);
  }
  const bool accumulate = (j != 1);
  s.cur_j = (int)j;
  s.cur_slot0 = (int)(((t - 1) * c->T) % s.S);  // slot of B(t,1) (contiguous T slots when wbatch)
  s.gsel = 0;
  s.gdone_valid[0] = s.gdone_valid[1] = false;
  // gradient bookkeeping over the stage's tensors: the output gradient is the gradient ring
  // slot (or dz on the last stage); every other tensor's gradient is written by its first
  // consumer (reverse op order) and accumulated by the others
  const StagePlan& P = s.plan;
  std::vector<char> has(P.tensors.size(), 0);
  std::vector<void*> gp(s.grad);
  gp[P.out_tensor] = (k + 1 < c->K) ? s.gin_slot[slot] : (void*)s.dz[slot];
  has[P.out_tensor] = 1;
  // concat views: the gradient of a view is the slice of its concat's gradient (complete once
  // every consumer of the concat has run, i.e. before the view's producer in reverse order)
  for (size_t t = 0; t < P.tensors.size(); ++t)
    if (P.tensors[t].alias >= 0) gp[t] = (uint8_t*)gp[P.tensors[t].alias] + (size_t)P.tensors[t].coff * P.tensors[t].es;
  auto have = [&](int t) { return has[t] || (P.tensors[t].alias >= 0 && has[P.tensors[t].alias]); };
  for (int o = (int)P.ops.size() - 1; o >= 0; --o) {
    const Op& O = P.ops[o];
    if (O.kind == OP_XENT || !have(O.out)) continue;
    const bool need0 = !(O.in0 == 0 && k == 0);  // the first stage needs no input gradient
    const bool need1 = O.in1 >= 0 && !(O.in1 == 0 && k == 0);
    XP_TRY(op_backward(c, s, o, gp[O.out], need0 ? gp[O.in0] : nullptr, need0 && has[O.in0],
                       need1 ? gp[O.in1] : nullptr, need1 && has[O.in1], s.pb, slot, accumulate));
    if (need0) has[O.in0] = 1;
    if (need1) has[O.in1] = 1;
  }
  XP_TRY(tmark(c, s, s.stream, &top.e[1], bw && k > 0));
  if (k + 1 < c->K) XP_TRY(flag_write(c, s, c->S[k + 1], 3, u));  // released gin slot u
  if (k > 0) {
    if (!has[0]) return set_err(c, XP_ESCHED, "no gradient reaches the stage input (internal)");
    StageRT& pv = c->S[k - 1];
    XP_TRY(flag_wait(c, s, 3, u - pv.S));
    XP_CUDA(c, cudaMemcpyAsync(pv.gin_slot[(u - 1) % pv.S], gp[0], P.in_bytes, cudaMemcpyDefault, s.stream));
    XP_TRY(tmark(c, s, s.stream, &top.e[2], bw));
    XP_TRY(flag_write(c, s, pv, 1, u));
    if (!s.wbatch) XP_TRY(flag_write(c, s, pv, 2, u));  // released our input slot u
  }
  if (s.side_used) {  // join the weight-gradient side stream (the update reads g)
    XP_CUDA(c, cudaEventRecord(s.ev_join, s.side));
    XP_CUDA(c, cudaStreamWaitEvent(s.stream, s.ev_join, 0));
    s.side_used = false;
  }
  // batched weight gradients read every input slot of the mini-batch: release them together
  if (s.wbatch && j == c->T && k > 0) XP_TRY(flag_write(c, s, c->S[k - 1], 2, u));
  if (rec) XP_TRY(check_launch(c, launch_trace_end(rec, s.stream), "trace"));
  if (ov && !s.wbatch) XP_TRY(ev_record(c, s.stream, s.ev_bdone[slot], &s.bdone_epoch[slot]));  // slot free for F(u + S)
  if (ov && s.wbatch && j == c->T)  // the mini-batch's T slots are free once its batched wgrads ran
    for (int q = 0; q < c->T; ++q) {
      const int sl = (s.cur_slot0 + q) % s.S;
      XP_TRY(ev_record(c, s.stream, s.ev_bdone[sl], &s.bdone_epoch[sl]));
    }
  if (j == c->T) {
    // the T-th micro-batch's backward ends the mini-batch: update + prediction (K1)
    if (ov) {  // forwards enqueued so far (still reading W_hat_f buffers) finish before the sweep
      int64_t e = 0;
      XP_TRY(ev_record(c, s.fstream, s.ev_fmark, &e));
      XP_TRY(ev_wait(c, s.stream, s.ev_fmark, e));
    }
    TraceRec* urec = nullptr;
    XP_TRY(trace_slot(c, s, &urec));
    XP_TRY(check_launch(c, launch_bump(s.ds, urec, k, (int)t, c->T, s.stream), "bump"));
    const int nv = s.host_ver + 1;
    const float sf = (float)version_difference(c, k, 0), sbf = (float)sb;
    const bool bf16 = c->cfg.precision == XP_BF16;
    XP_TRY(prof_begin(c, s));
    void* pbw = c->cfg.wbwd == XP_WBWD_BELLWETHER ? nullptr : s.pb;  // bellwether mode: W_hat_b later
    if (c->cfg.optimizer == XP_OPT_MOMENTUM_SGD)
      XP_TRY(check_launch(c, launch_sweep_sgd(s.W, s.g, s.buf, s.m, s.v, s.pf[nv & 1], pbw, s.plan.P, s.ds, nullptr, sf,
                                              sbf, bf16, s.stream), "sweep_sgd"));
    else
      XP_TRY(check_launch(c, launch_sweep(s.W, s.g, s.m, s.v, s.pf[nv & 1], pbw, s.plan.P, s.ds, nullptr, sf, sbf,
                                          bf16, c->cfg.delta_form, true, s.stream), "sweep"));
    // algorithmic bytes per parameter: Adam 16 B read + 12 B written + the predictions written
    // (2, or 1 in bellwether mode); the f2 Momentum-SGD sweep also reads and writes the velocity
    const double sgd_extra = c->cfg.optimizer == XP_OPT_MOMENTUM_SGD ? 8.0 : 0.0;
    const double pred_b = (bf16 ? 2.0 : 4.0) * (pbw ? 2.0 : 1.0);
    XP_TRY(prof_end(c, s, XP_PROF_SWEEP, (double)s.plan.P * (28.0 + pred_b + sgd_extra)));
    s.host_ver = nv;
    if (ov) XP_TRY(ev_record(c, s.stream, s.ev_upd, &s.upd_epoch));  // the next bellwether forward waits
    if (c->cfg.snapshots) {
      if (s.snap_pool.empty()) return set_err(c, XP_ESCHED, "snapshot pool (internal)");
      Snapshot sn{nv, {}, s.snap_pool.back()};
      s.snap_pool.pop_back();
      XP_CUDA(c, cudaMemcpyAsync(sn.pinned, s.W, s.plan.P * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      s.snaps.push_back(std::move(sn));
    }
  }
  XP_TRY(tmark(c, s, s.stream, &top.e[3]));  // the op's end: side-stream joined (+ update)
  if (c->timed) s.tops.push_back(top);
  return XP_OK;
}

// Host enqueue loop in dataflow order (the oracle's O2 driver, on enqueue counters): a stage's
// next op is enqueued only once every op its device waits depend on has been enqueued, so a
// full hardware queue can never block the host while the work it waits for is unenqueued.
// In multi-process mode the other stages' progress is unknown: only program order applies.
bool op_ready(const xpipe_ctx* c, int k, int op, int64_t u) {
  if (c->mp()) return true;
  const auto& S = c->S;
  if (op == 0) {
    if (k > 0 && S[k - 1].fwd_enq < u) return false;                          // activation message
    if (k + 1 < c->K && S[k + 1].bwd_enq < ring_credit(c, S[k + 1], u)) return false;  // ring credit
  } else {
    if (k + 1 < c->K ? S[k + 1].bwd_enq < u : S[k].fwd_enq < u) return false; // gradient / logits
    if (k > 0 && S[k - 1].bwd_enq < u - S[k - 1].S) return false;             // gradient ring credit
  }
  return true;
}

int drive(xpipe_ctx* c, int64_t total) {
  for (bool progress = true; progress;) {
    progress = false;
    for (int k = 0; k < c->K; ++k) {
      StageRT& s = c->S[k];
      if (!owned(s)) continue;
      while (!s.done) {
        int op;
        int64_t u;
        program_op(c, k, s.pos, &op, &u);
        if (total >= 0 && u > total) {
          if (op == 1 || c->cfg.schedule == XP_SCHED_GPIPE) { s.done = true; break; }
          ++s.pos;  // flushing: forwards beyond the last fed micro-batch are dropped
          continue;
        }
        if (u > c->fed || !op_ready(c, k, op, u)) break;
        if (verbose()) fprintf(stderr, "[xpipe] stage %d pos %lld: %c(%lld) slot %lld\n", k, (long long)s.pos,
                               op == 0 ? 'F' : 'B', (long long)u, (long long)((u - 1) % s.S));
        XP_TRY(op == 0 ? enqueue_forward(c, k, u) : enqueue_backward(c, k, u));
        if (op == 0) s.fwd_enq = u; else s.bwd_enq = u;
        ++s.pos;
        progress = true;
      }
    }
  }
  return join_fstreams(c);
}

// on a watchdog timeout: read the ring flags and the trace tail through a side stream
// (never blocking on a hung device) into the error message
std::string pipeline_state(xpipe_ctx* c) {
  std::string out;
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    cudaSetDevice(s.dev);
    cudaStream_t side;
    if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) return out + " (no side stream)";
    uint32_t* f = (uint32_t*)s.diag;  // pinned, allocated at init: the copy never blocks the host
    TraceRec& last = *(TraceRec*)((char*)s.diag + 64);
    if (!f) return out + " (no diag buffer)";
    f[0] = f[1] = f[2] = f[3] = 0xFFFFFFFFu;
    last = TraceRec{};
    cudaMemcpyAsync(f, s.flags, 16, cudaMemcpyDeviceToHost, side);
    if (c->cfg.trace && s.trace_n) cudaMemcpyAsync(&last, s.trace_dev + s.trace_n - 1, sizeof(TraceRec), cudaMemcpyDeviceToHost, side);
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, side);
    auto t0 = std::chrono::steady_clock::now();
    bool ok = false;
    while (std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count() < 2000) {
      if (cudaEventQuery(e) == cudaSuccess) { ok = true; break; }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    char buf[512];
    snprintf(buf, sizeof buf, " | stage %d: pos=%lld host_ver=%d flags(act_ready,grad_ready,act_ack,grad_ack)=%s%u,%u,%u,%u"
             " trace_n=%lld last={op=%d t=%d j=%d t1=%llu}", s.k, (long long)s.pos, s.host_ver, ok ? "" : "(unread)",
             f[0], f[1], f[2], f[3], (long long)s.trace_n, last.op, last.t, last.j, (unsigned long long)last.t1_ns);
    out += buf;
    out += " base=" + std::to_string(c->flag_base);
  }
  return out;
}

int sync_all(xpipe_ctx* c) {
  const int ms = c->cfg.watchdog_ms > 0 ? c->cfg.watchdog_ms : 120000;
  auto t0 = std::chrono::steady_clock::now();
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    cudaSetDevice(s.dev);
    for (;;) {
      cudaError_t e = cudaStreamQuery(s.stream);
      if (e == cudaSuccess && s.fstream && s.fstream != s.stream) e = cudaStreamQuery(s.fstream);
      if (e == cudaSuccess) break;
      if (e != cudaErrorNotReady) return set_err(c, XP_ECUDA, std::string("stream: ") + cudaGetErrorString(e));
      if (std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count() > ms)
        return set_err(c, XP_ESCHED, "pipeline watchdog: stage " + std::to_string(s.k) + " did not drain" +
                                         pipeline_state(c));
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  return XP_OK;
}

// ---- streams --------------------------------------------------------------------------------
// CUDA_DEVICE_MAX_CONNECTIONS (hardware work queues per context, default 8) is read when the
// CUDA context is created: a pipeline of K stages enqueues on 2-3 streams per stage, and with 8
// queues independent streams serialise behind each other (VGG-16 K=4 on one B200: 99.5k ->
// 117k samples/s with 32).  Set the default when the library is loaded (no effect if the
// process created its context before, or the caller chose a value).
__attribute__((constructor)) void xp_default_connections() { setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0); }

// role 0 = a stage's main (backward / update) stream, 1 = its forward stream (fb_overlap), 2 = its
// weight-gradient side stream.  Development knob XPIPE_STREAM_PRIO (default 0: all equal):
// 1 = main streams high, side streams low; 2 = main high, forward and side low;
// 3 = later stages higher (the pipeline drains from the last stage)
cudaError_t make_stream(cudaStream_t* st, int role, int k, int K) {
  static const int mode = [] { const char* e = getenv("XPIPE_STREAM_PRIO"); return (e && *e) ? atoi(e) : 0; }();
  int lo = 0, hi = 0;  // numerically: greatest (lowest priority), least (highest priority)
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  int prio = lo;
  if (mode == 1) prio = role == 0 ? hi : (role == 2 ? lo : (lo + hi) / 2);
  else if (mode == 2) prio = role == 0 ? hi : lo;
  else if (mode == 3) prio = lo + (int)((long)(hi - lo) * k / std::max(1, K - 1));
  return cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, prio);
}

// ---- CUDA graphs of steady-state steps -------------------------------------------------------
// In steady state (no flush, every in-flight wait already past the warm-up) a call's enqueue is
// a pure function of: M, the call buffers, and per stage (pos - 2*(fed - base)), (fed - base)
// mod S (ring-slot phase), and the parities of the version counters (W_hat_f buffer choice);
// the ring flags are rebased to fed so their values repeat too.
bool graph_eligible(const xpipe_ctx* c, uint32_t flags, int64_t M, int64_t fed_before) {
  if (!c->cfg.graphs || c->cfg.trace || c->cfg.snapshots) return false;
  if ((flags & XP_FLUSH) || M <= 0 || fed_before - c->base < 2 * c->K) return false;
  if (c->mp()) {
    // one process per GPU: the other processes' previous calls may still be running, so every
    // flag wait of the call must be a real (positive) micro-batch index at capture already
    int smax = 0;
    for (const auto& s : c->S) smax = std::max(smax, s.S);
    return fed_before - c->base >= smax + 2 * c->K + c->T;
  }
  for (const auto& s : c->S)
    if (s.dev != c->S[0].dev) return false;  // single-process capture: one device
  return true;
}

std::string graph_signature(const xpipe_ctx* c, int64_t M, int64_t fed_before) {
  std::string sig = std::to_string(M) + (c->timed ? "t:" : ":") + std::to_string((uintptr_t)c->x_dev) + ":" +
                    std::to_string((uintptr_t)c->y_dev) + ":" + std::to_string((uintptr_t)c->loss_dev);
  const int64_t f = fed_before - c->base;
  for (const auto& s : c->S) {
    if (!owned(s)) continue;  // one process per GPU: other ranks' stages are not enqueued here
    sig += "|" + std::to_string(s.pos - 2 * f) + "," + std::to_string(s.fwd_enq - fed_before) + "," +
           std::to_string(s.bwd_enq - fed_before) + "," + std::to_string(f % s.S) + "," + std::to_string(s.host_ver & 1) +
           "," + std::to_string(s.host_fver & 1) + "," + std::to_string((int)s.done);
  }
  return sig;
}

int rebase_flags(xpipe_ctx* c, int64_t new_base) {
  const int64_t delta = new_base - c->flag_base;
  if (delta == 0) return XP_OK;
  for (auto& s : c->S) {
    cudaSetDevice(s.dev);
    XP_TRY(check_launch(c, launch_rebase_flags(s.flags, 4, (uint32_t)delta, s.stream), "rebase"));
  }
  for (auto& s : c->S) { cudaSetDevice(s.dev); XP_CUDA(c, cudaStreamSynchronize(s.stream)); }
  c->flag_base = new_base;
  return XP_OK;
}

int drive_graph(xpipe_ctx* c, int64_t M, int64_t fed_before, bool chain = false) {
  // single process: flags rebased to the call's base (every stage drained); multi-process: the
  // flags stay absolute (neighbours may still be running) and the graph's flag kernels read the
  // call's base from the device.  Chained replay (the previous call's graph still running): the
  // rebase kernels go on the launch stream, ordered after that graph and before this one
  const std::string sig = graph_signature(c, M, fed_before);
  xpipe_ctx::GraphRec& g = c->graphs[sig];
  StageRT& o = c->mp() ? c->S[c->cfg.my_stage] : c->S[0];
  if (!c->mp()) {
    if (chain) {
      const int64_t delta = fed_before - c->flag_base;
      cudaSetDevice(o.dev);
      for (auto& s : c->S)
        if (delta) XP_TRY(check_launch(c, launch_rebase_flags(s.flags, 4, (uint32_t)delta, o.stream), "rebase"));
      c->flag_base = fed_before;
    } else {
      XP_TRY(rebase_flags(c, fed_before));
    }
  }
  cudaSetDevice(o.dev);
  if (c->mp()) XP_TRY(check_launch(c, launch_set_i64(o.dbase, fed_before, o.stream), "base"));
  if (g.exec) {
    XP_CUDA(c, cudaGraphLaunch(g.exec, o.stream));
    c->graph_launched = true;
    for (size_t k = 0; k < c->S.size(); ++k) {
      StageRT& s = c->S[k];
      const int v0 = s.host_ver;
      s.pos += g.dpos[k];
      s.fwd_enq += g.dfwd[k];
      s.bwd_enq += g.dbwd[k];
      s.host_ver += g.dver[k];
      s.host_fver = v0 + g.dfver[k];
      s.host_bver = v0 + g.dbver[k];
    }
    c->kernels += g.kernels;
    c->graph_replays++;
    for (size_t k = 0; k < c->S.size(); ++k) {  // the graph re-records the same profiling events
      c->S[k].prof_cls = g.prof_cls[k];
      c->S[k].prof_work = g.prof_work[k];
      c->S[k].ev_used = 2 * g.prof_cls[k].size();
      c->S[k].tops = g.tops[k];                   // ... and the same timing stamps
      c->S[k].tev_used = g.tev_used[k];
    }
    return XP_OK;
  }
  if (g.seen++ == 0) return drive(c, -1);  // first sighting: plain enqueue
  // second sighting: capture this call's enqueue, then launch it
  std::vector<int64_t> pos0, fwd0, bwd0;
  std::vector<int> ver0;
  for (auto& s : c->S) { pos0.push_back(s.pos); ver0.push_back(s.host_ver); fwd0.push_back(s.fwd_enq); bwd0.push_back(s.bwd_enq); }
  const int64_t k0 = c->kernels;
  static thread_local std::vector<cudaEvent_t> evs;
  while (evs.size() < c->S.size() + 2) {
    cudaEvent_t e;
    XP_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evs.push_back(e);
  }
  XP_CUDA(c, cudaStreamBeginCapture(o.stream, cudaStreamCaptureModeThreadLocal));
  XP_CUDA(c, cudaEventRecord(evs[0], o.stream));
  for (auto& s : c->S)
    if (owned(s) && &s != &o) XP_CUDA(c, cudaStreamWaitEvent(s.stream, evs[0], 0));
  for (auto& s : c->S)
    if (owned(s) && s.fstream && s.fstream != s.stream) XP_CUDA(c, cudaStreamWaitEvent(s.fstream, evs[0], 0));
  c->cap_base = fed_before;
  c->cap_fwd0.clear(); c->cap_bwd0.clear();
  for (auto& s : c->S) {
    c->cap_fwd0.push_back(s.fwd_enq);
    c->cap_bwd0.push_back(s.bwd_enq);
    for (int w = 0; w < 4; ++w) {
      const int k = s.k;
      const size_t n = (w == 0 || w == 1) ? s.S : (w == 2 ? (k + 1 < c->K ? c->S[k + 1].S : 1) : (k > 0 ? c->S[k - 1].S : 1));
      while (s.ev_flag[w].size() < n) {
        cudaEvent_t e;
        XP_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        s.ev_flag[w].push_back(e);
      }
    }
  }
  c->capturing = true;
  int r = drive(c, -1);
  c->capturing = false;
  for (size_t k = 0; k < c->S.size() && r == XP_OK; ++k) {
    if (!owned(c->S[k]) || &c->S[k] == &o) continue;
    if (cudaEventRecord(evs[k + 1], c->S[k].stream) != cudaSuccess ||
        cudaStreamWaitEvent(o.stream, evs[k + 1], 0) != cudaSuccess)
      r = set_err(c, XP_ECUDA, "graph join");
  }
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(o.stream, &graph);
  if (r != XP_OK) return r;
  if (e != cudaSuccess) return set_err(c, XP_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_err(c, XP_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  g.kernels = c->kernels - k0;
  g.dpos.clear(); g.dver.clear(); g.dfver.clear(); g.dbver.clear(); g.dfwd.clear(); g.dbwd.clear();
  g.prof_cls.clear(); g.prof_work.clear(); g.tops.clear(); g.tev_used.clear();
  for (auto& s : c->S) {
    g.prof_cls.push_back(s.prof_cls); g.prof_work.push_back(s.prof_work);
    g.tops.push_back(s.tops); g.tev_used.push_back(s.tev_used);
  }
  for (size_t k = 0; k < c->S.size(); ++k) {
    StageRT& s = c->S[k];
    g.dpos.push_back(s.pos - pos0[k]);
    g.dfwd.push_back(s.fwd_enq - fwd0[k]);
    g.dbwd.push_back(s.bwd_enq - bwd0[k]);
    g.dver.push_back(s.host_ver - ver0[k]);
    g.dfver.push_back(s.host_fver - ver0[k]);
    g.dbver.push_back(s.host_bver - ver0[k]);
  }
  XP_CUDA(c, cudaGraphLaunch(g.exec, o.stream));
  c->graph_launched = true;
  return XP_OK;
}

// cfg.timing: the call's span, per-stage busy time (union of op intervals), bubble fraction,
// steady-phase rate and hand-off times, from the per-op events
int timing_stats(xpipe_ctx* c, int64_t M, bool empty_before, bool flush, xpipe_stats* st) {
  double t_lo = 1e300, t_hi = -1e300, busy_sum = 0;
  int owned_n = 0, ops = 0;
  // one copy of every owned stage's stamps; times in ms relative to the first stamp seen
  uint64_t t_ref = 0;
  for (auto& s : c->S) {
    if (!owned(s) || !s.tev_used) continue;
    cudaSetDevice(s.dev);
    XP_CUDA(c, cudaMemcpy(s.tstamp_host, s.tstamp, s.tev_used * 8, cudaMemcpyDeviceToHost));
    if (!t_ref || s.tstamp_host[0] < t_ref) t_ref = s.tstamp_host[0];
  }
  auto at = [&](StageRT& s, int e, double* ms) -> int {
    *ms = ((double)(int64_t)(s.tstamp_host[e] - t_ref)) * 1e-6;
    return XP_OK;
  };
  std::vector<double> bell;  // stage 0's bellwether forward starts, in order
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    ++owned_n;
    cudaSetDevice(s.dev);
    std::vector<std::pair<double, double>> iv;
    double pf = 0, pb = 0, bf = 0, bb = 0;
    for (const TimedOp& o : s.tops) {
      if (o.e[0] < 0 || o.e[3] < 0) continue;
      double t0, t1 = 0, t2 = 0, tend = 0;
      XP_TRY(at(s, o.e[0], &t0));
      XP_TRY(at(s, o.e[3], &tend));
      if (o.e[1] >= 0) {  // a sampled hand-off: compute end -> copy end (forward: op end)
        XP_TRY(at(s, o.e[1], &t1));
        if (o.op == 0) { pf += tend - t1; bf += (double)s.plan.out_bytes; }
        else if (o.e[2] >= 0) { XP_TRY(at(s, o.e[2], &t2)); pb += t2 - t1; bb += (double)s.plan.in_bytes; }
      }
      iv.push_back({t0, tend});
      t_lo = std::min(t_lo, t0);
      t_hi = std::max(t_hi, tend);
      ++ops;
      if (s.k == 0 && o.op == 0) {
        const int64_t u = o.u_rel + c->call_first;
        if ((u - 1) % c->T == 0 && o.u_rel >= 0) bell.push_back(t0);
      }
    }
    std::sort(iv.begin(), iv.end());
    double busy = 0, a = -1e300, b = -1e300;
    for (auto& p : iv) {
      if (p.first > b) { if (b > a) busy += b - a; a = p.first; b = p.second; }
      else b = std::max(b, p.second);
    }
    if (b > a) busy += b - a;
    busy_sum += busy;
    if (s.k < XP_STATS_STAGES) {
      st->busy_ms[s.k] = busy;
      st->p2p_fwd_ms[s.k] = pf; st->p2p_bwd_ms[s.k] = pb;
      st->p2p_fwd_bytes[s.k] = bf; st->p2p_bwd_bytes[s.k] = bb;
    }
  }
  st->ops_timed = ops;
  st->span_ms = t_hi > t_lo ? t_hi - t_lo : 0;
  st->bubble_fraction = st->span_ms > 0 ? 1.0 - busy_sum / (owned_n * st->span_ms) : 0;
  // steady phase: drop the warm-up (first K mini-batches after an empty pipeline) and the drain
  // (last K mini-batches of a flushing call)
  const size_t lo = empty_before ? (size_t)c->K : 0;
  const size_t hi = bell.size() >= (flush ? (size_t)c->K : 0) ? bell.size() - (flush ? (size_t)c->K : 0) : 0;
  st->steady_samples_per_s = 0;
  if (hi > lo + 1 && bell[hi - 1] > bell[lo])
    st->steady_samples_per_s = (double)(hi - 1 - lo) * c->N / ((bell[hi - 1] - bell[lo]) * 1e-3);
  (void)M;
  return XP_OK;
}

int ensure_call_buffers(xpipe_ctx* c, int64_t M) {
  if (c->cfg.recompute && !c->loss_scratch && owned(c->S[c->K - 1])) {
    c->loss_scratch = (float*)dmalloc(c, 256, c->S[c->K - 1].dev);
    if (!c->loss_scratch) return set_err(c, XP_ENOMEM, "loss scratch");
  }
  const int64_t per = (int64_t)c->cfg.in_c * c->cfg.in_h * c->cfg.in_w;
  const int64_t xs = M * c->N * per, ys = M * c->N, ls = M * c->T;
  if (xs > c->x_cap || ys > c->y_cap || ls > c->loss_cap) {
    XP_TRY(sync_all(c));
    const bool first = owned(c->S[0]), last = owned(c->S[c->K - 1]);
    if (first && xs > c->x_cap) { c->x_dev = (float*)dmalloc(c, xs * 4, c->S[0].dev); c->x_cap = xs; }
    if (last && ys > c->y_cap) { c->y_dev = (int32_t*)dmalloc(c, ys * 4, c->S[c->K - 1].dev); c->y_cap = ys; }
    if (last && ls > c->loss_cap) { c->loss_dev = (float*)dmalloc(c, ls * 4, c->S[c->K - 1].dev); c->loss_cap = ls; }
    if ((first && !c->x_dev) || (last && (!c->y_dev || !c->loss_dev))) return set_err(c, XP_ENOMEM, "call buffers");
  }
  if (!c->mp() && !c->cfg.serialize && (c->x_stage_cap < c->x_cap || c->y_stage_cap < c->y_cap)) {
    const int dev = c->S[0].dev;
    cudaSetDevice(dev);
    if (!c->cstream) {
      if (cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev_staged, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&c->ev_stage_free, cudaEventDisableTiming) != cudaSuccess)
        return set_err(c, XP_ECUDA, "staging stream");
    }
    XP_CUDA(c, cudaStreamSynchronize(c->cstream));
    c->x_stage = (float*)dmalloc(c, c->x_cap * 4, dev);
    c->y_stage = (int32_t*)dmalloc(c, c->y_cap * 4, dev);
    if (!c->x_stage || !c->y_stage) return set_err(c, XP_ENOMEM, "staging buffers");
    c->x_stage_cap = c->x_cap;
    c->y_stage_cap = c->y_cap;
  }
  return XP_OK;
}

// a chained replay (see xpipe_step) needs: the single-process graph path, the same call
// buffers (no reallocation), no stamping / profiling / tracing / snapshots, and an already
// captured graph for this call's signature
__host__ bool no_chain() { static const bool v = [] { const char* e = getenv("XPIPE_NO_CHAIN"); return e && *e && *e != '0'; }(); return v; }
bool can_chain(xpipe_ctx* c, uint32_t flags, int64_t M) {
  if (no_chain() || c->mp() || M <= 0 || (flags & XP_FLUSH) || c->timed || c->cfg.profile || c->cfg.trace ||
      c->cfg.snapshots || c->cfg.recompute)
    return false;
  const int64_t per = (int64_t)c->cfg.in_c * c->cfg.in_h * c->cfg.in_w;
  if (M * c->N * per > c->x_cap || M * c->N > c->y_cap || M * c->T > c->loss_cap) return false;
  if (!graph_eligible(c, flags, M, c->fed)) return false;
  auto it = c->graphs.find(graph_signature(c, M, c->fed));
  return it != c->graphs.end() && it->second.exec != nullptr;
}

}  // namespace

// ----------------------------------------------------------------------------------------
// C ABI
// ----------------------------------------------------------------------------------------
extern "C" {

const char* xpipe_last_error(const xpipe_ctx* h) { return h ? h->err.c_str() : g_init_error.c_str(); }

int xpipe_finalize(xpipe_ctx* h) {
  if (!h) return XP_OK;
  free_all(h);
  delete h;
  return XP_OK;
}

int xpipe_init(const xpipe_layer* layers, int32_t n_layers, int32_t stages, int32_t T, int32_t N, float lr,
               const float betas[2], float eps, const xpipe_config* cfg, xpipe_ctx** out) {
  if (!out) return set_err(nullptr, XP_EINVAL, "out is NULL");
  *out = nullptr;
  if (!layers || n_layers < 2 || !cfg || !betas) return set_err(nullptr, XP_EINVAL, "layers/cfg/betas required");
  if (stages < 1 || stages > 64 || T < 1 || N < 1 || N % T) return set_err(nullptr, XP_EINVAL, "mini_batch % micro_batches != 0");
  if (!(lr > 0) || !(betas[0] >= 0 && betas[0] < 1) || !(betas[1] >= 0 && betas[1] < 1) || !(eps > 0))
    return set_err(nullptr, XP_EINVAL, "hyperparameters: lr > 0, betas in [0,1), eps > 0");
  if (cfg->moment_init == XP_MOM_GIVEN && (cfg->delta_form != XP_DELTA_PAPER || !cfg->init_m || !cfg->init_v))
    return set_err(nullptr, XP_EINVAL, "XP_MOM_GIVEN requires XP_DELTA_PAPER and init_m/init_v (R2)");
  if (cfg->optimizer != XP_OPT_ADAM && cfg->optimizer != XP_OPT_MOMENTUM_SGD)
    return set_err(nullptr, XP_EINVAL, "optimizer");
  if (cfg->optimizer == XP_OPT_MOMENTUM_SGD &&
      (cfg->delta_form != XP_DELTA_PAPER || !(cfg->momentum >= 0 && cfg->momentum < 1) || !(cfg->weight_decay >= 0)))
    return set_err(nullptr, XP_EINVAL, "XP_OPT_MOMENTUM_SGD requires XP_DELTA_PAPER, momentum in [0,1), weight_decay >= 0");
  if (cfg->precision != XP_FP32 && cfg->precision != XP_BF16) return set_err(nullptr, XP_EINVAL, "precision");
  if (cfg->wbwd != XP_WBWD_MATERIALIZE && cfg->wbwd != XP_WBWD_BELLWETHER) return set_err(nullptr, XP_EINVAL, "wbwd");
  if (cfg->schedule != XP_SCHED_XPIPE && cfg->schedule != XP_SCHED_GPIPE) return set_err(nullptr, XP_EINVAL, "schedule");
  if (cfg->predict < 0 || cfg->predict > 2 || (cfg->predict == XP_PRED_FIXED && (cfg->s_fwd < 0 || cfg->s_bwd < 0)))
    return set_err(nullptr, XP_EINVAL, "predict");
  if (cfg->schedule == XP_SCHED_GPIPE && cfg->predict == XP_PRED_PAPER)
    return set_err(nullptr, XP_EINVAL, "GPipe runs under the current weights: use XP_PRED_OFF (or XP_PRED_FIXED for diagnostics)");
  if (N / T > kXentMaxRows)
    return set_err(nullptr, XP_EUNSUPPORTED, "micro-batch N/T > " + std::to_string(kXentMaxRows) + " (loss kernel limit)");
  if (cfg->multi_process && (cfg->my_stage < 0 || cfg->my_stage >= stages))
    return set_err(nullptr, XP_EINVAL, "my_stage out of range");
  std::unique_ptr<xpipe_ctx> c(new xpipe_ctx());
  c->cfg = *cfg;
  if (!c->cfg.seed) c->cfg.seed = 1;
  c->K = stages; c->T = T; c->N = N; c->n = N / T;
  c->lr = lr; c->b1 = betas[0]; c->b2 = betas[1]; c->eps = eps;
  std::string perr;
  int r = build_net_plan(layers, n_layers, stages, c->cfg, c->n, &c->net, &perr);
  if (r != XP_OK) return set_err(nullptr, r, perr);
  for (const auto& sp : c->net.stages)
    for (const Op& O : sp.ops)
      if (O.kind == OP_CONV && (O.smid.c % 8 || O.smid.c > 2048))
        return set_err(nullptr, XP_EUNSUPPORTED, "BatchNorm kernels need C % 8 == 0 and C <= 2048 (conv output channels " +
                                                     std::to_string(O.smid.c) + ")");
  if (!load_driver_entry_points()) return set_err(nullptr, XP_ECUDA, "CUDA driver stream memory operations unavailable");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return set_err(nullptr, XP_ECUDA, "no CUDA device");
  int cur = 0;
  cudaGetDevice(&cur);
  c->S.resize(stages);
  for (int k = 0; k < stages; ++k) {
    StageRT& s = c->S[k];
    s.k = k;
    s.dev = c->mp() ? cur : (c->cfg.n_devices > 0 ? c->cfg.devices[k % c->cfg.n_devices] : cur);
    if (s.dev < 0 || s.dev >= ndev) return set_err(nullptr, XP_EINVAL, "device id out of range");
    s.plan = c->net.stages[k];
    s.S = c->cfg.schedule == XP_SCHED_GPIPE ? T : (stages - k);
    bool has_conv = false;
    for (const Op& O : s.plan.ops) has_conv |= O.kind == OP_CONV;
    s.wbatch = c->cfg.precision == XP_BF16 && has_conv && !no_wgrad_batch();
    if (s.wbatch && c->cfg.schedule != XP_SCHED_GPIPE) {
      // a slot is reused by F(u+S) only after the mini-batch of u finished (its batched wgrad
      // reads all T slots at B(t,T)): F(u') follows B(u'-W) in program order (W = K-k), so
      // S >= W + T - 1 (+1 when F(u') may overlap B(u'-W) on its own stream), a multiple of T
      // so that a mini-batch's T slots are contiguous
      const int want = stages - k + T - 1 + (c->cfg.fb_overlap ? 1 : 0);
      s.S = (want + T - 1) / T * T;
    } else if (c->cfg.fb_overlap) {
      // one more slot, so F(u+S) can overlap B(u); rounded to a divisor or a multiple of T so
      // the slot phase of every stage repeats each call (a call feeds whole mini-batches) and
      // steady-state calls keep replaying one CUDA graph
      int want = s.S + 1;
      if (want <= T) { while (T % want) ++want; }
      else want = (want + T - 1) / T * T;
      s.S = want;
    }
  }
  {
    int most = 1;
    for (int k = 0; k < stages; ++k) {
      int same = 0;
      for (int q = 0; q < stages; ++q) same += c->S[q].dev == c->S[k].dev;
      most = std::max(most, same);
    }
    // multi-process mode: this process runs only its own stage
    tc_set_coresident_stages(c->cfg.serialize || c->mp() ? 1 : most);
  }
  // peer access between the devices of neighbouring stages (multi-process mode: lazily, by
  // cudaIpcOpenMemHandle)
  for (int k = 0; k + 1 < stages && !c->mp(); ++k) {
    int a = c->S[k].dev, b = c->S[k + 1].dev;
    if (a == b) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, a, b);
    if (!ok) return set_err(nullptr, XP_EUNSUPPORTED, "no peer access between stage devices");
    cudaSetDevice(a); cudaDeviceEnablePeerAccess(b, 0); cudaGetLastError();
    cudaSetDevice(b); cudaDeviceEnablePeerAccess(a, 0); cudaGetLastError();
  }
  xpipe_ctx* cp = c.get();
  auto fail_init = [&](int code, const std::string& m) {
    std::string msg = m + (cp->err.empty() ? "" : (": " + cp->err));
    free_all(cp);
    return set_err(nullptr, code, msg);
  };
  for (int k = 0; k < stages; ++k) {
    StageRT& s = c->S[k];
    if (c->mp() && k != c->cfg.my_stage) continue;
    cudaSetDevice(s.dev);
    if (c->cfg.serialize && !c->mp() && k > 0 && s.dev == c->S[0].dev) {
      // profiling aid: every stage (and its weight-gradient work) on stage 0's stream, in the
      // host's dataflow enqueue order -- each kernel then runs alone, as in ncu's launch list
      s.stream = c->S[0].stream;
      s.side = c->S[0].stream;
    } else {
      if (make_stream(&s.stream, 0, k, c->K) != cudaSuccess) return fail_init(XP_ECUDA, "stream");
      if (c->cfg.serialize && !c->mp()) s.side = s.stream;
      else if (make_stream(&s.side, 2, k, c->K) != cudaSuccess)
        return fail_init(XP_ECUDA, "stream");
    }
    s.fstream = s.stream;
    if (c->cfg.fb_overlap && !c->cfg.serialize && make_stream(&s.fstream, 1, k, c->K) != cudaSuccess)
      return fail_init(XP_ECUDA, "stream");
    s.ev_fdone.assign(s.S, nullptr); s.ev_bdone.assign(s.S, nullptr);
    s.fdone_epoch.assign(s.S, -1); s.bdone_epoch.assign(s.S, -1);
    for (auto* v : {&s.ev_fdone, &s.ev_bdone})
      for (auto& e : *v)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return fail_init(XP_ECUDA, "event");
    for (cudaEvent_t* e : {&s.ev_upd, &s.ev_fmark, &s.ev_fjoin, &s.ev_in})
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return fail_init(XP_ECUDA, "event");
    for (cudaEvent_t* e : {&s.ev_fork, &s.ev_join, &s.ev_gdone[0], &s.ev_gdone[1]})
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return fail_init(XP_ECUDA, "event");
    if (cudaMallocHost(&s.diag, 256) != cudaSuccess) return fail_init(XP_ENOMEM, "diag buffer");
    int rr = allocate_stage(cp, s);
    if (rr != XP_OK) return fail_init(rr, "stage allocation");
    rr = init_stage_params(cp, s, layers);
    if (rr != XP_OK) return fail_init(rr, "parameter init");
  }
  if (owned(c->S[stages - 1])) {
    StageRT& sl = c->S[stages - 1];
    cudaSetDevice(sl.dev);
    c->status_dev = (uint32_t*)dmalloc(cp, 256, sl.dev);
    if (!c->status_dev || cudaMallocHost(&c->status_host, 256) != cudaSuccess) return fail_init(XP_ENOMEM, "status word");
    if (cudaMemsetAsync(c->status_dev, 0, 4, sl.stream) != cudaSuccess) return fail_init(XP_ECUDA, "status word");
  }
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    cudaSetDevice(s.dev);
    if (cudaStreamSynchronize(s.stream) != cudaSuccess) return fail_init(XP_ECUDA, "init sync");
  }
  reset_schedule(cp);
  cudaSetDevice(cur);
  *out = c.release();
  return XP_OK;
}

int xpipe_step(xpipe_ctx* c, const float* x, const int32_t* y, int32_t M, uint32_t flags, xpipe_stats* st) {
  if (!c) return set_err(nullptr, XP_EINVAL, "ctx is NULL");
  if (c->poisoned) return XP_ESTATE;
  if (M < 0 || (M > 0 && (!x || !y))) return set_err(c, XP_EINVAL, "x/y");
  const bool dev_ptrs = flags & XP_DEVICE_PTRS;
  if (c->mp()) {
    const int me = c->cfg.my_stage;
    if ((me + 1 < c->K && c->S[me + 1].in_slot.empty()) || (me > 0 && c->S[me - 1].gin_slot.empty()))
      return set_err(c, XP_EINVAL, "multi-process: neighbour stages not attached (xpipe_ipc_import)");
  }
  if (!dev_ptrs && M > 0)
    for (int64_t i = 0; i < (int64_t)M * c->N; ++i)
      if (y[i] < 0 || y[i] >= c->cfg.classes) return set_err(c, XP_EINVAL, "label out of range");
  int cur = 0;
  cudaGetDevice(&cur);
  const int64_t k0 = c->kernels, g0 = c->graph_replays;
  // cfg.timing = p: this call is stamped when it is the p-th since the last stamped one
  c->timed = c->cfg.timing > 0 && (c->calls++ % c->cfg.timing) == 0;
  // Chained replay: the previous call was an asynchronous replay of a captured graph and this
  // one replays one too.  Both graphs, the rebase and the input copies are then ordered on the
  // launch stream (a graph launch is one stream operation there), so the previous call's work
  // need not be waited for on the host; otherwise it must be done before its call buffers are
  // overwritten
  const bool chain = c->chain_ok && can_chain(c, flags, M);
  c->chain_ok = false;
  c->graph_launched = false;
  if (!chain) XP_TRY(sync_all(c));
  ++c->call_epoch;  // every event recorded before this point is complete (chain: no event logic runs)
  if (M > 0 && chain) {
    const int64_t per = (int64_t)c->cfg.in_c * c->cfg.in_h * c->cfg.in_w;
    StageRT& s0 = c->S[0];
    cudaSetDevice(s0.dev);
    const size_t xb = (size_t)M * c->N * per * 4, yb = (size_t)M * c->N * 4;
    if (!dev_ptrs && c->cstream && (int64_t)M * c->N * per <= c->x_stage_cap && (int64_t)M * c->N <= c->y_stage_cap) {
      // host inputs: H2D into the staging buffers now, concurrently with the previous call's
      // graph (cstream waits only for the previous call's staging copy-out), then a device copy
      // into the call buffers at the boundary
      XP_CUDA(c, cudaStreamWaitEvent(c->cstream, c->ev_stage_free, 0));
      XP_CUDA(c, cudaMemcpyAsync(c->x_stage, x, xb, cudaMemcpyHostToDevice, c->cstream));
      XP_CUDA(c, cudaMemcpyAsync(c->y_stage, y, yb, cudaMemcpyHostToDevice, c->cstream));
      XP_CUDA(c, cudaEventRecord(c->ev_staged, c->cstream));
      XP_CUDA(c, cudaStreamWaitEvent(s0.stream, c->ev_staged, 0));
      XP_CUDA(c, cudaMemcpyAsync(c->x_dev, c->x_stage, xb, cudaMemcpyDeviceToDevice, s0.stream));
      XP_CUDA(c, cudaMemcpyAsync(c->y_dev, c->y_stage, yb, cudaMemcpyDeviceToDevice, s0.stream));
      XP_CUDA(c, cudaEventRecord(c->ev_stage_free, s0.stream));
    } else {
      XP_CUDA(c, cudaMemcpyAsync(c->x_dev, x, xb, dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 s0.stream));
      XP_CUDA(c, cudaMemcpyAsync(c->y_dev, y, yb, dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 s0.stream));
    }
    XP_CUDA(c, cudaMemsetAsync(c->loss_dev, 0xff, (size_t)M * c->T * 4, s0.stream));  // NaN = not computed
    c->call_first = c->fed + 1;
    c->fed += (int64_t)M * c->T;
  } else if (M > 0) {
    XP_TRY(ensure_call_buffers(c, M));
    const int64_t per = (int64_t)c->cfg.in_c * c->cfg.in_h * c->cfg.in_w;
    StageRT& s0 = c->S[0];
    StageRT& sl = c->S[c->K - 1];
    // the copies run on the stages' main streams; the forward streams (fb_overlap) and, for a
    // graph replay, the launch stream wait for them (ev_in) before any op reads x / y / losses
    if (owned(s0)) {
      cudaSetDevice(s0.dev);
      XP_CUDA(c, cudaMemcpyAsync(c->x_dev, x, (size_t)M * c->N * per * 4,
                                 dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s0.stream));
    }
    if (owned(sl)) {
      cudaSetDevice(sl.dev);
      XP_CUDA(c, cudaMemcpyAsync(c->y_dev, y, (size_t)M * c->N * 4,
                                 dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, sl.stream));
      XP_CUDA(c, cudaMemsetAsync(c->loss_dev, 0xff, (size_t)M * c->T * 4, sl.stream));  // NaN = not computed
    }
    for (StageRT* q : {&s0, &sl}) {
      if (!owned(*q)) continue;
      cudaSetDevice(q->dev);
      XP_CUDA(c, cudaEventRecord(q->ev_in, q->stream));
      if (q->fstream && q->fstream != q->stream) XP_CUDA(c, cudaStreamWaitEvent(q->fstream, q->ev_in, 0));
    }
    if (owned(s0) && owned(sl) && sl.dev == s0.dev && &sl != &s0) {
      cudaSetDevice(s0.dev);
      XP_CUDA(c, cudaStreamWaitEvent(s0.stream, sl.ev_in, 0));  // graph launch stream sees the label copy
    }
    c->call_first = c->fed + 1;
    c->fed += (int64_t)M * c->T;
  }
  for (auto& s : c->S) { s.ev_used = 0; s.prof_cls.clear(); s.prof_work.clear(); s.tev_used = 0; s.tops.clear(); }
  if (!chain) XP_TRY(reserve_for_call(c, M));  // chain: the same M as a replayed call, nothing to reserve
  const bool empty_before = c->fed - (int64_t)M * c->T == c->base;  // pipeline empty at the call's start

  const int64_t fed_before = c->fed - (int64_t)M * c->T;
  if (graph_eligible(c, flags, M, fed_before)) XP_TRY(drive_graph(c, M, fed_before, chain));
  else XP_TRY(drive(c, -1));
  if (flags & XP_FLUSH) {
    XP_TRY(drive(c, c->fed));
    for (auto& s : c->S) {
      if (!owned(s)) continue;
      if (!s.done) return set_err(c, XP_ESCHED, "flush did not drain stage " + std::to_string(s.k));
      s.done = false;
      s.pos = 0;
    }
    c->base = c->fed;
    reset_schedule(c);
  }
  int rr = XP_OK;
  // XP_ASYNC: return after enqueue -- except a stamped call (its statistics are read back); an
  // asynchronous single-process graph replay lets the next replay chain behind it
  const bool replayed = c->graph_launched;  // a replay, or the launch right after the capture
  if ((flags & XP_ASYNC) && c->timed) flags &= ~(uint32_t)XP_ASYNC;
  if (!(flags & XP_ASYNC)) rr = sync_all(c);
  if (rr != XP_OK) return rr;
  c->chain_ok = (flags & XP_ASYNC) && replayed && !c->mp() && !(flags & XP_FLUSH) && !c->cfg.profile;
  if ((flags & XP_ASYNC) && st && st->losses && M > 0 && owned(c->S[c->K - 1])) {
    // the losses follow the call's work on its stream (a replay: the launch stream; else the last
    // stage's, where the loss kernel ran); the caller's buffer is read after a sync
    StageRT& q = (replayed && !c->mp()) ? c->S[0] : c->S[c->K - 1];
    cudaSetDevice(q.dev);
    XP_CUDA(c, cudaMemcpyAsync(st->losses, c->loss_dev, (size_t)M * c->T * 4, cudaMemcpyDeviceToHost, q.stream));
  }
  uint32_t status = 0;
  if (!(flags & XP_ASYNC) && c->status_dev) {
    // loss-kernel status word (device-side label range and non-finite loss checks)
    StageRT& sl = c->S[c->K - 1];
    cudaSetDevice(sl.dev);
    XP_CUDA(c, cudaMemcpy(c->status_host, c->status_dev, 4, cudaMemcpyDeviceToHost));
    status = *c->status_host;
    if (status) XP_CUDA(c, cudaMemset(c->status_dev, 0, 4));
  }
  if (st) {
    st->kernel_launches = c->kernels - k0;
    st->graph_replays = c->graph_replays - g0;
    st->span_ms = 0;
    st->bubble_fraction = st->steady_samples_per_s = 0;
    st->ops_timed = 0;
    for (int q = 0; q < XP_STATS_STAGES; ++q)
      st->busy_ms[q] = st->p2p_fwd_ms[q] = st->p2p_bwd_ms[q] = st->p2p_fwd_bytes[q] = st->p2p_bwd_bytes[q] = 0;
    for (int q = 0; q < XP_PROF_N; ++q) { st->prof_ms[q] = 0; st->prof_launches[q] = 0; st->prof_work[q] = 0; }
    if (c->cfg.profile && !(flags & XP_ASYNC)) {
      for (auto& s : c->S) {
        for (size_t i = 0; i < s.prof_cls.size(); ++i) {
          float ms = 0;
          cudaEventElapsedTime(&ms, s.ev_pool[2 * i], s.ev_pool[2 * i + 1]);
          const int q = s.prof_cls[i];
          st->prof_ms[q] += ms;
          st->prof_launches[q]++;
          st->prof_work[q] += s.prof_work[i];
        }
      }
    }
    if (c->timed && !(flags & XP_ASYNC)) XP_TRY(timing_stats(c, M, empty_before, (flags & XP_FLUSH) != 0, st));
    if (st->losses && M > 0 && !(flags & XP_ASYNC) && owned(c->S[c->K - 1])) {
      cudaSetDevice(c->S[c->K - 1].dev);
      XP_CUDA(c, cudaMemcpy(st->losses, c->loss_dev, (size_t)M * c->T * 4, cudaMemcpyDeviceToHost));
    }
  }
  cudaSetDevice(cur);
  if (status & XP_STATUS_LABEL) return set_err(c, XP_EINVAL, "label out of range (device check)");
  if (status & XP_STATUS_NONFINITE) return set_err(c, XP_ENONFINITE, "non-finite loss");
  return XP_OK;
}

int xpipe_timer(xpipe_ctx* c, int32_t which, double* ms_out) {
  if (!c || (which != 0 && which != 1)) return set_err(c, XP_EINVAL, "timer args");
  if (c->poisoned) return XP_ESTATE;
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    cudaSetDevice(s.dev);
    if (!s.tmark[which]) XP_CUDA(c, cudaEventCreate(&s.tmark[which]));
    XP_CUDA(c, cudaEventRecord(s.tmark[which], s.stream));
  }
  if (which == 1) {
    XP_TRY(sync_all(c));
    double mx = 0;
    for (auto& s : c->S) {
      if (!owned(s)) continue;
      float ms = 0;
      XP_CUDA(c, cudaEventElapsedTime(&ms, s.tmark[0], s.tmark[1]));
      mx = std::max(mx, (double)ms);
    }
    if (ms_out) *ms_out = mx;
  }
  return XP_OK;
}

namespace {
struct IpcBlob {
  uint32_t magic;
  int32_t stage, K, S, n;
  uint64_t in_stride, gin_stride, in_bytes, out_bytes;
  int32_t has_gin;
  cudaIpcMemHandle_t in_ring, gin_ring, flags;
};
const uint32_t kIpcMagic = 0x58504950u;  // "XPIP"
}  // namespace

int xpipe_ipc_export(xpipe_ctx* c, void* blob, size_t cap, size_t* len) {
  if (!c || !blob || !len || !c->mp()) return set_err(c, XP_EINVAL, "ipc_export: not in multi-process mode");
  if (cap < sizeof(IpcBlob)) return set_err(c, XP_EINVAL, "ipc_export: buffer too small");
  StageRT& s = c->S[c->cfg.my_stage];
  IpcBlob b{};
  b.magic = kIpcMagic; b.stage = s.k; b.K = c->K; b.S = s.S; b.n = c->n;
  b.in_stride = s.in_stride; b.gin_stride = s.gin_stride;
  b.in_bytes = s.plan.in_slot_bytes; b.out_bytes = s.plan.out_bytes;
  cudaSetDevice(s.dev);
  XP_CUDA(c, cudaIpcGetMemHandle(&b.in_ring, s.in_ring));
  XP_CUDA(c, cudaIpcGetMemHandle(&b.flags, s.flags));
  b.has_gin = s.gin_ring != nullptr;
  if (b.has_gin) XP_CUDA(c, cudaIpcGetMemHandle(&b.gin_ring, s.gin_ring));
  std::memcpy(blob, &b, sizeof b);
  *len = sizeof b;
  return XP_OK;
}

int xpipe_ipc_import(xpipe_ctx* c, const void* blob, size_t len) {
  if (!c || !blob || !c->mp() || len != sizeof(IpcBlob)) return set_err(c, XP_EINVAL, "ipc_import: bad blob");
  IpcBlob b;
  std::memcpy(&b, blob, sizeof b);
  const int me = c->cfg.my_stage;
  if (b.magic != kIpcMagic || b.K != c->K || b.n != c->n || b.stage < 0 || b.stage >= c->K)
    return set_err(c, XP_EINVAL, "ipc_import: blob of another pipeline");
  if (b.stage != me - 1 && b.stage != me + 1) return XP_OK;  // not a neighbour: nothing to map
  StageRT& nb = c->S[b.stage];
  if (b.S != nb.S) return set_err(c, XP_EINVAL, "ipc_import: ring size mismatch");
  cudaSetDevice(c->S[me].dev);
  void* p = nullptr;
  XP_CUDA(c, cudaIpcOpenMemHandle(&p, b.flags, cudaIpcMemLazyEnablePeerAccess));
  c->ipc_opened.push_back(p);
  nb.flags = (uint32_t*)p;
  if (b.stage == me + 1) {  // we write activations into its input ring
    XP_CUDA(c, cudaIpcOpenMemHandle(&p, b.in_ring, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    nb.in_slot.resize(nb.S);
    for (int i = 0; i < nb.S; ++i) nb.in_slot[i] = (uint8_t*)p + i * b.in_stride;
  } else {                  // we write input gradients into its gradient ring
    if (!b.has_gin) return set_err(c, XP_EINVAL, "ipc_import: upstream stage without a gradient ring");
    XP_CUDA(c, cudaIpcOpenMemHandle(&p, b.gin_ring, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_opened.push_back(p);
    nb.gin_slot.resize(nb.S);
    for (int i = 0; i < nb.S; ++i) nb.gin_slot[i] = (uint8_t*)p + i * b.gin_stride;
  }
  return XP_OK;
}

int xpipe_sync(xpipe_ctx* c) {
  if (!c) return set_err(nullptr, XP_EINVAL, "ctx is NULL");
  if (c->poisoned) return XP_ESTATE;
  return sync_all(c);
}

int xpipe_stage_of_layer(xpipe_ctx* c, int32_t layer) {
  if (!c || layer < 0 || layer >= (int)c->net.layers.size()) return set_err(c, XP_EINVAL, "layer");
  return c->net.layers[layer].stage;
}

int xpipe_stage_version(xpipe_ctx* c, int32_t stage) {
  if (!c || stage < 0 || stage >= c->K) return set_err(c, XP_EINVAL, "stage");
  return c->S[stage].host_ver;
}

int64_t xpipe_stage_params(xpipe_ctx* c, int32_t stage) {
  if (!c || stage < 0 || stage >= c->K) return set_err(c, XP_EINVAL, "stage");
  return c->S[stage].plan.P;
}

int xpipe_get_weights(xpipe_ctx* c, int32_t layer, int32_t tensor, int32_t state, int64_t version, float* dst,
                      size_t count) {
  if (!c || !dst) return set_err(c, XP_EINVAL, "args");
  if (c->poisoned) return XP_ESTATE;
  if (layer < 0 || layer >= (int)c->net.layers.size()) return set_err(c, XP_EINVAL, "layer");
  const LayerInfo& L = c->net.layers[layer];
  if (tensor != XP_T_WEIGHT && tensor != XP_T_BIAS) return set_err(c, XP_EINVAL, "tensor");
  const int64_t n = tensor == XP_T_WEIGHT ? L.nw_torch : L.nb;
  if ((int64_t)count != n) return set_err(c, XP_EINVAL, "count is not the tensor size");
  if (n == 0) return XP_OK;
  XP_TRY(sync_all(c));
  StageRT& s = c->S[L.stage];
  if (!owned(s)) return set_err(c, XP_EINVAL, "layer belongs to a stage of another process");
  const int64_t off = tensor == XP_T_WEIGHT ? L.woff : L.boff;
  const int64_t ng = tensor == XP_T_WEIGHT ? L.nw_gpu : L.nb;
  std::vector<float> buf(ng);
  cudaSetDevice(s.dev);
  const bool bf16 = c->cfg.precision == XP_BF16;
  if (state == XP_S_PRED_FWD || state == XP_S_PRED_BWD) {
    const void* src = state == XP_S_PRED_FWD ? s.pf[s.host_ver & 1] : s.pb;
    if (bf16) {
      std::vector<uint16_t> hb(ng);
      XP_CUDA(c, cudaMemcpy(hb.data(), (const __nv_bfloat16*)src + off, ng * 2, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < ng; ++i) { uint32_t u = (uint32_t)hb[i] << 16; std::memcpy(&buf[i], &u, 4); }
    } else {
      XP_CUDA(c, cudaMemcpy(buf.data(), (const float*)src + off, ng * 4, cudaMemcpyDeviceToHost));
    }
  } else {
    const float* src = nullptr;
    if (state == XP_S_PARAM && version >= 0 && version != s.host_ver) {
      if (version == 0 || !c->cfg.snapshots) {
        if (!c->cfg.snapshots) return set_err(c, XP_EINVAL, "snapshots disabled");
      }
      const Snapshot* sn = nullptr;
      for (auto& q : s.snaps) if (q.ver == version) sn = &q;
      if (!sn) return set_err(c, XP_EINVAL, "no snapshot of that version");
      std::memcpy(buf.data(), sn->pinned + off, ng * 4);
    } else {
      switch (state) {
        case XP_S_PARAM: src = s.W; break;
        case XP_S_M: src = s.m; break;
        case XP_S_V: src = s.v; break;
        case XP_S_GRAD: src = s.g; break;
        case XP_S_BUF:
          if (!s.buf) return set_err(c, XP_EINVAL, "XP_S_BUF needs XP_OPT_MOMENTUM_SGD");
          src = s.buf;
          break;
        default: return set_err(c, XP_EINVAL, "state");
      }
      XP_CUDA(c, cudaMemcpy(buf.data(), src + off, ng * 4, cudaMemcpyDeviceToHost));
    }
  }
  gpu_to_torch_layout(L, tensor, buf.data(), dst);
  return XP_OK;
}

int xpipe_set_weights(xpipe_ctx* c, int32_t layer, int32_t tensor, int32_t state, const float* src, size_t count) {
  if (!c || !src) return set_err(c, XP_EINVAL, "args");
  if (c->poisoned) return XP_ESTATE;
  if (layer < 0 || layer >= (int)c->net.layers.size()) return set_err(c, XP_EINVAL, "layer");
  const LayerInfo& L = c->net.layers[layer];
  if (tensor != XP_T_WEIGHT && tensor != XP_T_BIAS) return set_err(c, XP_EINVAL, "tensor");
  const int64_t n = tensor == XP_T_WEIGHT ? L.nw_torch : L.nb;
  if ((int64_t)count != n) return set_err(c, XP_EINVAL, "count is not the tensor size");
  if (n == 0) return XP_OK;
  XP_TRY(sync_all(c));
  StageRT& s = c->S[L.stage];
  if (!owned(s)) return set_err(c, XP_EINVAL, "layer belongs to a stage of another process");
  float* dst = nullptr;
  switch (state) {
    case XP_S_PARAM: dst = s.W; break;
    case XP_S_M: dst = s.m; break;
    case XP_S_V: dst = s.v; break;
    case XP_S_BUF: dst = s.buf; break;
    default: return set_err(c, XP_EINVAL, "state");
  }
  if (!dst) return set_err(c, XP_EINVAL, "XP_S_BUF needs XP_OPT_MOMENTUM_SGD");
  const int64_t off = tensor == XP_T_WEIGHT ? L.woff : L.boff;
  const int64_t ng = tensor == XP_T_WEIGHT ? L.nw_gpu : L.nb;
  std::vector<float> buf(ng, 0.f);  // channel padding stays zero
  torch_to_gpu_layout(L, tensor, src, buf.data());
  cudaSetDevice(s.dev);
  XP_CUDA(c, cudaMemcpy(dst + off, buf.data(), ng * 4, cudaMemcpyHostToDevice));
  return XP_OK;
}

int xpipe_refresh_predictions(xpipe_ctx* c) {
  if (!c) return set_err(c, XP_EINVAL, "args");
  if (c->poisoned) return XP_ESTATE;
  XP_TRY(sync_all(c));
  const bool bf = c->cfg.precision == XP_BF16;
  for (auto& s : c->S) {
    if (!owned(s)) continue;
    cudaSetDevice(s.dev);
    const float sf = (float)version_difference(c, s.k, 0), sb = (float)version_difference(c, s.k, 1);
    void* pf = s.pf[s.host_ver & 1];
    if (c->cfg.delta_form == XP_DELTA_ADAM && s.host_ver == 0)
      XP_TRY(check_launch(c, launch_predict_copy(s.W, pf, s.pb, s.plan.P, bf, s.stream), "refresh"));
    else
      XP_TRY(check_launch(c, launch_sweep(s.W, s.g, s.m, s.v, pf, s.pb, s.plan.P, s.ds, nullptr, sf, sb, bf,
                                          c->cfg.delta_form, false, s.stream), "refresh"));
    XP_CUDA(c, cudaStreamSynchronize(s.stream));
  }
  return XP_OK;
}

int xpipe_get_trace(xpipe_ctx* c, int32_t stage, xpipe_trace_rec* dst, size_t cap, size_t* n_out) {
  if (!c || !n_out || stage < 0 || stage >= c->K) return set_err(c, XP_EINVAL, "args");
  if (c->poisoned) return XP_ESTATE;
  XP_TRY(sync_all(c));
  StageRT& s = c->S[stage];
  if (!owned(s)) return set_err(c, XP_EINVAL, "stage of another process");
  *n_out = (size_t)s.trace_n;
  if (dst && s.trace_n) {
    cudaSetDevice(s.dev);
    const size_t n = std::min(cap, (size_t)s.trace_n);
    static_assert(sizeof(TraceRec) == sizeof(xpipe_trace_rec), "trace layout");
    XP_CUDA(c, cudaMemcpy(dst, s.trace_dev, n * sizeof(TraceRec), cudaMemcpyDeviceToHost));
  }
  return XP_OK;
}

int xpipe_schedule_program(int32_t stages, int32_t micro_batches, int32_t schedule, int32_t stage, int64_t n,
                           int32_t* ops, int64_t* us) {
  if (stages < 1 || micro_batches < 1 || stage < 0 || stage >= stages || n < 0 || (n > 0 && (!ops || !us)) ||
      (schedule != XP_SCHED_XPIPE && schedule != XP_SCHED_GPIPE))
    return set_err(nullptr, XP_EINVAL, "schedule_program args");
  ScheduleSim sim;
  std::vector<bool> rec(stages, false);
  rec[stage] = true;
  sim.reset(stages, micro_batches, schedule == XP_SCHED_GPIPE, rec);
  for (int64_t p = 0; p < n; ++p) {
    int op;
    int64_t u;
    sim.op_at(stage, p, &op, &u);
    ops[p] = op;
    us[p] = u;
  }
  return XP_OK;
}

int xpipe_adam_predict(float* W, const float* g, float* m, float* v, void* pred_f, void* pred_b, int64_t n,
                       int64_t version, float lr, float beta1, float beta2, float eps, int32_t s_f, int32_t s_b,
                       int32_t pred_bf16, int32_t delta_form, void* stream) {
  if (!W || !g || !m || !v || n < 0 || version < 1) return set_err(nullptr, XP_EINVAL, "adam_predict args");
  if (((uintptr_t)W | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v | (uintptr_t)pred_f | (uintptr_t)pred_b) & 15)
    return set_err(nullptr, XP_EINVAL, "alignment (all six arrays 16-byte aligned)");
  SweepScalars hs;
  host_scalars(version, lr, beta1, beta2, eps, &hs);
  cudaError_t e = launch_sweep(W, g, m, v, pred_f, pred_b, n, nullptr, &hs, (float)s_f, (float)s_b, pred_bf16 != 0,
                               delta_form, true, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_err(nullptr, XP_ECUDA, cudaGetErrorString(e));
  return XP_OK;
}

int xpipe_sgd_predict(float* W, const float* g, float* buf, float* m, float* v, void* pred_f, void* pred_b, int64_t n,
                      float lr, float beta1, float beta2, float eps, float momentum, float weight_decay, int32_t s_f,
                      int32_t s_b, int32_t pred_bf16, void* stream) {
  if (!W || !g || !buf || !m || !v || n < 0) return set_err(nullptr, XP_EINVAL, "sgd_predict args");
  if (((uintptr_t)W | (uintptr_t)g | (uintptr_t)buf | (uintptr_t)m | (uintptr_t)v | (uintptr_t)pred_f | (uintptr_t)pred_b) & 15)
    return set_err(nullptr, XP_EINVAL, "alignment (all seven arrays 16-byte aligned)");
  SweepScalars hs;
  host_scalars(1, lr, beta1, beta2, eps, &hs);  // the paper form uses only the constant corrections
  hs.mu = momentum;
  hs.wd = weight_decay;
  cudaError_t e = launch_sweep_sgd(W, g, buf, m, v, pred_f, pred_b, n, nullptr, &hs, (float)s_f, (float)s_b,
                                   pred_bf16 != 0, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_err(nullptr, XP_ECUDA, cudaGetErrorString(e));
  return XP_OK;
}

}  // extern "C"
