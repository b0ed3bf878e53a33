// f32.cu -- the fp32 SIMT path (C1, the MLP) and small bookkeeping kernels.
//
// The fp32 kernels implement the frozen op order of DESIGN.md section 4 ("fp32
// contract"): every dot product is a sequential fmaf chain in index order starting from 0,
// every batch sum is sequential in row order, the bias is added once at the end; all
// arithmetic is explicit round-to-nearest intrinsics (never contracted).  With that order
// the results are bit-identical to the oracle's fp32 mode, which is what lets the 1e-4
// max-relative bar of the north star hold for Adam's sign-like steps.
// Tiles are staged through shared memory only to coalesce global loads; the per-output
// reduction order is untouched.
#include "../internal.h"
#include "launch.h"

namespace xp {

namespace {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// K12: trace record at op start.  The version comes from the device counter (the sweep's
// bump kernel increments it), the bellwether latches it for the other T-1 micro-batches.
__global__ void trace_begin_kernel(DevState* ds, TraceRec* rec, int stage, int op, int t, int j, int s, int bw) {
  pdl_wait();
  int ver;
  if (op == 0) { if (bw) ds->fver = ds->ver; ver = ds->fver; }
  else { if (bw) ds->bver = ds->ver; ver = ds->bver; }
  rec->stage = stage; rec->op = op; rec->t = t; rec->j = j; rec->version = ver; rec->s = s;
  rec->bellwether = bw; rec->wbuf = op == 0 ? (ver & 1) : 0;
  rec->t0_ns = globaltimer();
  rec->t1_ns = 0;
}

// Ring flags inside CUDA graphs of the one-process-per-GPU mode.  The flags hold absolute
// micro-batch indices written by other processes, so a captured graph cannot bake the values
// in: the graph stores them relative to *base (the call's first micro-batch minus 1, set by a
// kernel launched before every replay) and these 1-thread kernels wait / write base + rel.
// flag_wait spins (acquire, system scope, wraparound-safe >=) with a nanosleep backoff.
__global__ void flag_wait_kernel(const uint32_t* flag, const int64_t* base, int32_t rel) {
  pdl_wait();
  const uint32_t want = (uint32_t)(*base + rel);
  unsigned ns = 32;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int32_t)(v - want) >= 0) break;
    __nanosleep(ns);
    if (ns < 1024) ns *= 2;
  }
}
__global__ void flag_write_kernel(uint32_t* flag, const int64_t* base, int32_t rel) {
  pdl_wait();
  __threadfence_system();
  const uint32_t v = (uint32_t)(*base + rel);
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(flag), "r"(v) : "memory");
}
__global__ void set_i64_kernel(int64_t* dst, int64_t v) {
  pdl_wait();
  *dst = v;
}

// cfg.timing: one %globaltimer stamp after the preceding work of the stream (1 thread)
__global__ void stamp_kernel(uint64_t* dst) {
  pdl_wait();
  *dst = globaltimer();
}

__global__ void trace_end_kernel(TraceRec* rec) {
  pdl_wait(); rec->t1_ns = globaltimer(); }

// ring flags hold micro-batch indices relative to a base; rebasing subtracts delta (mod 2^32)
__global__ void rebase_flags_kernel(uint32_t* f, int n, uint32_t delta) {
  pdl_wait();
  if (threadIdx.x < n) f[threadIdx.x] -= delta;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// counter-based U(-bound, bound): value i of stream (seed, id) -- no state, any launch shape
__global__ void fill_uniform_kernel(float* d, int64_t n, float bound, uint64_t seed, uint64_t id) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t r = splitmix64(seed * 0x632be59bd9b4e019ull ^ splitmix64(id * 0x100000001b3ull + (uint64_t)i));
    double u = (double)(r >> 11) * (1.0 / 9007199254740992.0);  // [0,1)
    d[i] = (float)((2.0 * u - 1.0) * (double)bound);
  }
}

__global__ void fill_const_kernel(float* d, int64_t n, float v) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = v;
}

// y[r][o] = (sum_i fmaf(x[r][i], W[o][i], acc), i ascending from acc = 0) + b[o]; relu optional.
// Block: 32 outputs (tx) x 8 rows (ty); i in chunks of 32 staged through smem (coalesced).
__global__ void __launch_bounds__(256) linear_fwd_f32_kernel(const float* __restrict__ x, const float* __restrict__ W,
                                                             const float* __restrict__ b, float* __restrict__ y, int n,
                                                             int in, int out, int relu) {
  pdl_wait();
  __shared__ float Ws[32][33];
  __shared__ float xs[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + tx, r = blockIdx.y * 8 + ty;
  float acc = 0.f;
  for (int i0 = 0; i0 < in; i0 += 32) {
    for (int q = ty; q < 32; q += 8) {  // W tile rows o0+q, cols i0+tx
      const int oo = blockIdx.x * 32 + q, ii = i0 + tx;
      Ws[q][tx] = (oo < out && ii < in) ? W[(int64_t)oo * in + ii] : 0.f;
    }
    {
      const int ii = i0 + tx;
      xs[ty][tx] = (r < n && ii < in) ? x[(int64_t)r * in + ii] : 0.f;
    }
    __syncthreads();
    const int lim = min(32, in - i0);
    for (int q = 0; q < lim; ++q) acc = __fmaf_rn(xs[ty][q], Ws[tx][q], acc);
    __syncthreads();
  }
  if (o < out && r < n) {
    float v = b ? __fadd_rn(acc, b[o]) : acc;
    if (relu) v = v > 0.f ? v : 0.f;
    y[(int64_t)r * out + o] = v;
  }
}

// dx[r][i] = sum_o fmaf(dy'[r][o], W[o][i], acc), o ascending; dy' = ymask > 0 ? dy : 0
__global__ void __launch_bounds__(256) linear_dgrad_f32_kernel(const float* __restrict__ dy,
                                                               const float* __restrict__ ymask,
                                                               const float* __restrict__ W, float* __restrict__ dx,
                                                               int n, int in, int out) {
  pdl_wait();
  __shared__ float Ws[32][33];
  __shared__ float ds[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + tx, r = blockIdx.y * 8 + ty;
  float acc = 0.f;
  for (int o0 = 0; o0 < out; o0 += 32) {
    for (int q = ty; q < 32; q += 8) {  // W rows o0+q, cols i (coalesced along i)
      const int oo = o0 + q;
      Ws[q][tx] = (oo < out && i < in) ? W[(int64_t)oo * in + i] : 0.f;
    }
    {
      const int oo = o0 + tx;
      float d = 0.f;
      if (r < n && oo < out) {
        d = dy[(int64_t)r * out + oo];
        if (ymask && !(ymask[(int64_t)r * out + oo] > 0.f)) d = 0.f;
      }
      ds[ty][tx] = d;
    }
    __syncthreads();
    const int lim = min(32, out - o0);
    for (int q = 0; q < lim; ++q) acc = __fmaf_rn(ds[ty][q], Ws[q][tx], acc);
    __syncthreads();
  }
  if (i < in && r < n) dx[(int64_t)r * in + i] = acc;
}

// gW[o][i] (=|+=) sum_r fmaf(dy'[r][o], x[r][i], acc), r ascending; column i == in is the bias
__global__ void __launch_bounds__(256) linear_wgrad_f32_kernel(const float* __restrict__ dy,
                                                               const float* __restrict__ ymask,
                                                               const float* __restrict__ x, float* __restrict__ gW,
                                                               float* __restrict__ gb, int n, int in, int out,
                                                               int accumulate) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // i in [0, in] (in = bias column)
  const int o = blockIdx.y;
  if (i > in || (i == in && !gb)) return;
  float acc = 0.f;
  for (int r = 0; r < n; ++r) {
    float d = dy[(int64_t)r * out + o];
    if (ymask && !(ymask[(int64_t)r * out + o] > 0.f)) d = 0.f;
    if (i < in) acc = __fmaf_rn(d, x[(int64_t)r * in + i], acc);
    else acc = __fadd_rn(acc, d);
  }
  float* dst = i < in ? &gW[(int64_t)o * in + i] : &gb[o];
  *dst = accumulate ? __fadd_rn(*dst, acc) : acc;
}

// softmax cross-entropy, one thread per row (classes sequential):
// e_c = (float)exp((double)(z_c - max)); s = sum_c e_c (class order); p = e/s;
// dz = (p - onehot) * invN; loss row = -log(e_y/s) (reporting only).
// status (nullable): bit XP_STATUS_LABEL if a label lies outside [0, C) (its row then gets no
// onehot term), bit XP_STATUS_NONFINITE if the mean loss is not finite; read by xpipe_step.
__global__ void xent_f32_kernel(const float* __restrict__ z, const int32_t* __restrict__ y, float* __restrict__ dz,
                                float* __restrict__ loss, int n, int C, float invN, uint32_t* __restrict__ status) {
  pdl_wait();
  __shared__ double lsum[256];
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  double l = 0.0;
  if (r < n) {
    const float* zr = z + (int64_t)r * C;
    float mx = zr[0];
    for (int c = 1; c < C; ++c) mx = fmaxf(mx, zr[c]);
    float s = 0.f;
    for (int c = 0; c < C; ++c) s = __fadd_rn(s, (float)exp((double)__fsub_rn(zr[c], mx)));
    const int lab = y[r];
    if ((lab < 0 || lab >= C) && status) atomicOr(status, (uint32_t)XP_STATUS_LABEL);
    for (int c = 0; c < C; ++c) {
      const float e = (float)exp((double)__fsub_rn(zr[c], mx));
      const float p = __fdiv_rn(e, s);
      dz[(int64_t)r * C + c] = __fmul_rn(__fsub_rn(p, c == lab ? 1.f : 0.f), invN);
      if (c == lab) l = -log((double)p);
    }
  }
  lsum[threadIdx.x] = l;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < n && q < 256; ++q) t += lsum[q];
    const float lv = (float)(t / n);
    *loss = lv;
    if (status && !isfinite(lv)) atomicOr(status, (uint32_t)XP_STATUS_NONFINITE);
  }
}

// The same arithmetic with one warp per row (rows w, w + 8, ... of the 8 warps): the lanes
// evaluate the class exponentials in parallel into shared memory, lane 0 adds them in class order
// (the sum above, bit for bit), the lanes write dz; the max is order-independent.  The serial
// kernel ran 75 us per micro-batch for the 200-class heads (fp64 exp, 2 x C per thread in turn),
// on the last stage's critical path.  C <= kXentWarpC.
constexpr int kXentWarpC = 1024;
__global__ void __launch_bounds__(256) xent_warp_kernel(const float* __restrict__ z, const int32_t* __restrict__ y,
                                                        float* __restrict__ dz, float* __restrict__ loss, int n, int C,
                                                        float invN, uint32_t* __restrict__ status) {
  extern __shared__ float xe[];  // [8][C] exponentials of each warp's current row
  __shared__ double lsum[256];
  __shared__ float ssum[8];
  pdl_wait();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* e = xe + wid * C;
  for (int r = wid; r < n; r += 8) {
    const float* zr = z + (int64_t)r * C;
    float mx = zr[0];
    for (int c = lane; c < C; c += 32) mx = fmaxf(mx, zr[c]);
#pragma unroll
    for (int off = 16; off; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    for (int c = lane; c < C; c += 32) e[c] = (float)exp((double)__fsub_rn(zr[c], mx));
    __syncwarp();
    if (lane == 0) {
      float sacc = 0.f;
      for (int c = 0; c < C; ++c) sacc = __fadd_rn(sacc, e[c]);
      ssum[wid] = sacc;
    }
    __syncwarp();
    const float sv = ssum[wid];
    const int lab = y[r];
    if (lane == 0 && (lab < 0 || lab >= C) && status) atomicOr(status, (uint32_t)XP_STATUS_LABEL);
    for (int c = lane; c < C; c += 32) {
      const float pc = __fdiv_rn(e[c], sv);
      dz[(int64_t)r * C + c] = __fmul_rn(__fsub_rn(pc, c == lab ? 1.f : 0.f), invN);
      if (c == lab) lsum[r] = -log((double)pc);
    }
    if (lane == 0 && (lab < 0 || lab >= C)) lsum[r] = 0.0;
    __syncwarp();  // e[] is rewritten by the warp's next row
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < n; ++q) t += lsum[q];
    const float lv = (float)(t / n);
    *loss = lv;
    if (status && !isfinite(lv)) atomicOr(status, (uint32_t)XP_STATUS_NONFINITE);
  }
}

int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

cudaError_t launch_trace_begin(DevState* ds, TraceRec* rec, int stage, int op, int t, int j, int s, int bw,
                               cudaStream_t st) {
  launch_pdl(trace_begin_kernel, dim3(1), dim3(1), 0, st, ds, rec, stage, op, t, j, s, bw);
  return cudaGetLastError();
}

cudaError_t launch_rebase_flags(uint32_t* flags, int n, uint32_t delta, cudaStream_t st) {
  launch_pdl(rebase_flags_kernel, dim3(1), dim3(32), 0, st, flags, n, delta);
  return cudaGetLastError();
}

cudaError_t launch_flag_wait(const uint32_t* flag, const int64_t* base, int32_t rel, cudaStream_t st) {
  launch_pdl(flag_wait_kernel, dim3(1), dim3(1), 0, st, flag, base, rel);
  return cudaGetLastError();
}
cudaError_t launch_flag_write(uint32_t* flag, const int64_t* base, int32_t rel, cudaStream_t st) {
  launch_pdl(flag_write_kernel, dim3(1), dim3(1), 0, st, flag, base, rel);
  return cudaGetLastError();
}
cudaError_t launch_set_i64(int64_t* dst, int64_t v, cudaStream_t st) {
  launch_pdl(set_i64_kernel, dim3(1), dim3(1), 0, st, dst, v);
  return cudaGetLastError();
}

cudaError_t launch_stamp(uint64_t* dst, cudaStream_t st) {
  launch_pdl(stamp_kernel, dim3(1), dim3(1), 0, st, dst);
  return cudaGetLastError();
}

cudaError_t launch_trace_end(TraceRec* rec, cudaStream_t st) {
  launch_pdl(trace_end_kernel, dim3(1), dim3(1), 0, st, rec);
  return cudaGetLastError();
}

cudaError_t launch_fill_uniform(float* dst, int64_t n, float bound, uint64_t seed, uint64_t id, cudaStream_t st) {
  launch_pdl(fill_uniform_kernel, dim3(grid_for(n)), dim3(256), 0, st, dst, n, bound, seed, id);
  return cudaGetLastError();
}

cudaError_t launch_fill_const(float* dst, int64_t n, float value, cudaStream_t st) {
  launch_pdl(fill_const_kernel, dim3(grid_for(n)), dim3(256), 0, st, dst, n, value);
  return cudaGetLastError();
}

cudaError_t launch_linear_fwd_f32(const float* x, const float* W, const float* b, float* y, int n, int in, int out,
                                  bool relu, cudaStream_t st) {
  dim3 grid((out + 31) / 32, (n + 7) / 8);
  launch_pdl(linear_fwd_f32_kernel, dim3(grid), dim3(256), 0, st, x, W, b, y, n, in, out, relu ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_linear_dgrad_f32(const float* dy, const float* ymask, const float* W, float* dx, int n, int in,
                                    int out, cudaStream_t st) {
  dim3 grid((in + 31) / 32, (n + 7) / 8);
  launch_pdl(linear_dgrad_f32_kernel, dim3(grid), dim3(256), 0, st, dy, ymask, W, dx, n, in, out);
  return cudaGetLastError();
}

cudaError_t launch_linear_wgrad_f32(const float* dy, const float* ymask, const float* x, float* gW, float* gb, int n,
                                    int in, int out, bool accumulate, cudaStream_t st) {
  dim3 grid((in + 1 + 127) / 128, out);
  launch_pdl(linear_wgrad_f32_kernel, dim3(grid), dim3(128), 0, st, dy, ymask, x, gW, gb, n, in, out, accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_xent_f32(const float* z, const int32_t* y, float* dz, float* loss, int n, int classes, float invN,
                            uint32_t* status, cudaStream_t st) {
  if (n > kXentMaxRows) return cudaErrorInvalidValue;
  // few classes (VGG-16's 10): the per-row serial loop is shorter than the warp kernel's
  // cross-lane steps (ncu: 8.1 vs 9.3 us); the warp kernel from 64 classes on
  if (classes > 64 && classes <= kXentWarpC) {
    const size_t shm = (size_t)8 * classes * sizeof(float);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(xent_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kXentWarpC * 4);
      attr = true;
    }
    launch_pdl(xent_warp_kernel, dim3(1), dim3(256), shm, st, z, y, dz, loss, n, classes, invN, status);
  } else {
    launch_pdl(xent_f32_kernel, dim3(1), dim3(256), 0, st, z, y, dz, loss, n, classes, invN, status);
  }
  return cudaGetLastError();
}

}  // namespace xp
