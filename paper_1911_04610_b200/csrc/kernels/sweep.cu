// sweep.cu -- K1, the fused Adam-update + weight-prediction sweep.
//
// Runs once per stage per mini-batch, after the T-th micro-batch's backward: one
// pass over the stage's flat parameter arena that reads W, g, m, v exactly once and writes
// W, m, v and the two predicted-weight buffers of the new version:
//   W_hat_f = W' - s_f * d  (Eq. (1) staleness, forward)   W_hat_b = W' - s_b * d  (Eq. (2))
// with d = lr * m_hat / (sqrt(v_hat) + eps) from the moments just updated (Eq. (3) with
// Adam's moments, BASELINE.json north star).  The op order is the fp32 contract of
// every operation an explicit IEEE round-to-nearest intrinsic, so the
// result is bit-identical to the oracle's sweep:
//   m' = fmaf(b1, m, omb1*g); v' = fmaf(b2, v, omb2*(g*g)); den = sqrt(v')*r2 + eps;
//   d = (c1*m')/den; W' = W - d; W_hat = fmaf(-s, d, W')   [bf16: round-to-nearest-even]
//
// HBM roofline: 16 B read + 12 B write fp32 state + 2x(2 or 4) B predictions = 32/36 B per
// parameter; 8 parameters per thread (two 128-bit loads per fp32 stream, one 128-bit store per
// bf16 prediction stream), one group per thread over a grid as large as the arena needs;
// streaming loads/stores (evict-first) for the optimizer state, default policy for W_hat which
// the next forward/backward reads from L2.
#include <cstdlib>

#include "../internal.h"
#include "launch.h"

namespace xp {

namespace {

struct Sc {
  float c1, r2, omb1, omb2, inv1, inv2, lr, b1, b2, eps, mu, wd;
};

__device__ __forceinline__ Sc load_sc(const DevState* ds, const SweepScalars& hs) {
  Sc s;
  if (ds) {
    s.c1 = ds->c1; s.r2 = ds->r2; s.omb1 = ds->omb1; s.omb2 = ds->omb2; s.inv1 = ds->inv1; s.inv2 = ds->inv2;
    s.lr = ds->lr; s.b1 = ds->b1; s.b2 = ds->b2; s.eps = ds->eps; s.mu = ds->mu; s.wd = ds->wd;
  } else {
    s.c1 = hs.c1; s.r2 = hs.r2; s.omb1 = hs.omb1; s.omb2 = hs.omb2; s.inv1 = hs.inv1; s.inv2 = hs.inv2;
    s.lr = hs.lr; s.b1 = hs.b1; s.b2 = hs.b2; s.eps = hs.eps; s.mu = hs.mu; s.wd = hs.wd;
  }
  return s;
}

// one parameter, f2: Momentum-SGD update in place (PyTorch semantics: buf = mu*buf + (g + wd*W),
// W -= lr*buf) with the Eq. (4) moments tracked from the raw gradient, returning the paper-form
// prediction delta -- the op order of the oracle's sgd_elem
__device__ __forceinline__ float elem_sgd(const Sc& s, float& W, float g, float& buf, float& m, float& v) {
  m = __fmaf_rn(s.b1, m, __fmul_rn(s.omb1, g));
  v = __fmaf_rn(s.b2, v, __fmul_rn(s.omb2, __fmul_rn(g, g)));
  const float gw = __fmaf_rn(s.wd, W, g);
  buf = __fmaf_rn(s.mu, buf, gw);
  W = __fsub_rn(W, __fmul_rn(s.lr, buf));
  return __fdiv_rn(__fmul_rn(s.lr, __fmul_rn(m, s.inv1)), __fsqrt_rn(__fadd_rn(__fmul_rn(v, s.inv2), s.eps)));
}

// one parameter: Adam update in place + prediction delta (Adam or paper form)
template <bool UPDATE, int DELTA>
__device__ __forceinline__ float elem(const Sc& s, float& W, float g, float& m, float& v) {
  if (UPDATE) {
    m = __fmaf_rn(s.b1, m, __fmul_rn(s.omb1, g));
    v = __fmaf_rn(s.b2, v, __fmul_rn(s.omb2, __fmul_rn(g, g)));
  }
  const float den = __fadd_rn(__fmul_rn(__fsqrt_rn(v), s.r2), s.eps);
  const float d = __fdiv_rn(__fmul_rn(s.c1, m), den);
  if (UPDATE) W = __fsub_rn(W, d);
  if (DELTA == 1)  // paper form: lr * (m/(1-b1)) / sqrt(v/(1-b2) + eps)
    return __fdiv_rn(__fmul_rn(s.lr, __fmul_rn(m, s.inv1)), __fsqrt_rn(__fadd_rn(__fmul_rn(v, s.inv2), s.eps)));
  return d;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // round-to-nearest-even
  return *reinterpret_cast<uint32_t*>(&h);
}

template <bool BF16, bool UPDATE, int DELTA>
__global__ void __launch_bounds__(256) sweep_kernel(float* __restrict__ W, const float* __restrict__ g,
                                                    float* __restrict__ m, float* __restrict__ v,
                                                    void* __restrict__ pf, void* __restrict__ pb, int64_t n,
                                                    const DevState* __restrict__ ds, SweepScalars hs, float sf,
                                                    float sb) {
  pdl_wait();
  const Sc s = load_sc(ds, hs);
  const float nsf = -sf, nsb = -sb;
  const int64_t n8 = n >> 3;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    const int64_t e = i << 3;
    float4 w0 = __ldcs(reinterpret_cast<const float4*>(W + e));
    float4 w1 = __ldcs(reinterpret_cast<const float4*>(W + e + 4));
    float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), g1 = g0;
    if (UPDATE) {
      g0 = __ldcs(reinterpret_cast<const float4*>(g + e));
      g1 = __ldcs(reinterpret_cast<const float4*>(g + e + 4));
    }
    float4 m0 = __ldcs(reinterpret_cast<const float4*>(m + e));
    float4 m1 = __ldcs(reinterpret_cast<const float4*>(m + e + 4));
    float4 v0 = __ldcs(reinterpret_cast<const float4*>(v + e));
    float4 v1 = __ldcs(reinterpret_cast<const float4*>(v + e + 4));
    float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    float mv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    float fv[8], bv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float d = elem<UPDATE, DELTA>(s, wv[q], gv[q], mv[q], vv[q]);
      fv[q] = __fmaf_rn(nsf, d, wv[q]);
      bv[q] = __fmaf_rn(nsb, d, wv[q]);
    }
    if (UPDATE) {
      __stcs(reinterpret_cast<float4*>(W + e), make_float4(wv[0], wv[1], wv[2], wv[3]));
      __stcs(reinterpret_cast<float4*>(W + e + 4), make_float4(wv[4], wv[5], wv[6], wv[7]));
      __stcs(reinterpret_cast<float4*>(m + e), make_float4(mv[0], mv[1], mv[2], mv[3]));
      __stcs(reinterpret_cast<float4*>(m + e + 4), make_float4(mv[4], mv[5], mv[6], mv[7]));
      __stcs(reinterpret_cast<float4*>(v + e), make_float4(vv[0], vv[1], vv[2], vv[3]));
      __stcs(reinterpret_cast<float4*>(v + e + 4), make_float4(vv[4], vv[5], vv[6], vv[7]));
    }
    if (BF16) {
      if (pf) *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(pf) + e) =
          make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
      if (pb) *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(pb) + e) =
          make_uint4(pack_bf16(bv[0], bv[1]), pack_bf16(bv[2], bv[3]), pack_bf16(bv[4], bv[5]), pack_bf16(bv[6], bv[7]));
    } else {
      if (pf) {
        float* p = static_cast<float*>(pf) + e;
        *reinterpret_cast<float4*>(p) = make_float4(fv[0], fv[1], fv[2], fv[3]);
        *reinterpret_cast<float4*>(p + 4) = make_float4(fv[4], fv[5], fv[6], fv[7]);
      }
      if (pb) {
        float* p = static_cast<float*>(pb) + e;
        *reinterpret_cast<float4*>(p) = make_float4(bv[0], bv[1], bv[2], bv[3]);
        *reinterpret_cast<float4*>(p + 4) = make_float4(bv[4], bv[5], bv[6], bv[7]);
      }
    }
  }
  // tail (n % 8 elements), scalar
  const int64_t tail0 = n8 << 3;
  for (int64_t e = tail0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    float w = W[e], gg = UPDATE ? g[e] : 0.f, mm = m[e], vv = v[e];
    const float d = elem<UPDATE, DELTA>(s, w, gg, mm, vv);
    if (UPDATE) { W[e] = w; m[e] = mm; v[e] = vv; }
    const float f = __fmaf_rn(nsf, d, w), b = __fmaf_rn(nsb, d, w);
    if (BF16) {
      if (pf) static_cast<__nv_bfloat16*>(pf)[e] = __float2bfloat16_rn(f);
      if (pb) static_cast<__nv_bfloat16*>(pb)[e] = __float2bfloat16_rn(b);
    } else {
      if (pf) static_cast<float*>(pf)[e] = f;
      if (pb) static_cast<float*>(pb)[e] = b;
    }
  }
}

// f2 sweep: reads W, g, buf, m, v (20 B) and writes W, buf, m, v (16 B) + two predictions per
// parameter; 8 parameters per thread-iteration as in the Adam sweep
template <bool BF16>
__global__ void __launch_bounds__(256) sweep_sgd_kernel(float* __restrict__ W, const float* __restrict__ g,
                                                        float* __restrict__ buf, float* __restrict__ m,
                                                        float* __restrict__ v, void* __restrict__ pf,
                                                        void* __restrict__ pb, int64_t n,
                                                        const DevState* __restrict__ ds, SweepScalars hs, float sf,
                                                        float sb) {
  pdl_wait();
  const Sc s = load_sc(ds, hs);
  const float nsf = -sf, nsb = -sb;
  const int64_t n8 = n >> 3;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
    const int64_t e = i << 3;
    float wv[8], gv[8], bv[8], mv[8], vv[8], fv[8], pv[8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 w4 = __ldcs(reinterpret_cast<const float4*>(W + e) + h);
      const float4 g4 = __ldcs(reinterpret_cast<const float4*>(g + e) + h);
      const float4 b4 = __ldcs(reinterpret_cast<const float4*>(buf + e) + h);
      const float4 m4 = __ldcs(reinterpret_cast<const float4*>(m + e) + h);
      const float4 v4 = __ldcs(reinterpret_cast<const float4*>(v + e) + h);
      wv[4 * h] = w4.x; wv[4 * h + 1] = w4.y; wv[4 * h + 2] = w4.z; wv[4 * h + 3] = w4.w;
      gv[4 * h] = g4.x; gv[4 * h + 1] = g4.y; gv[4 * h + 2] = g4.z; gv[4 * h + 3] = g4.w;
      bv[4 * h] = b4.x; bv[4 * h + 1] = b4.y; bv[4 * h + 2] = b4.z; bv[4 * h + 3] = b4.w;
      mv[4 * h] = m4.x; mv[4 * h + 1] = m4.y; mv[4 * h + 2] = m4.z; mv[4 * h + 3] = m4.w;
      vv[4 * h] = v4.x; vv[4 * h + 1] = v4.y; vv[4 * h + 2] = v4.z; vv[4 * h + 3] = v4.w;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float d = elem_sgd(s, wv[q], gv[q], bv[q], mv[q], vv[q]);
      fv[q] = __fmaf_rn(nsf, d, wv[q]);
      pv[q] = __fmaf_rn(nsb, d, wv[q]);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      __stcs(reinterpret_cast<float4*>(W + e) + h, make_float4(wv[4 * h], wv[4 * h + 1], wv[4 * h + 2], wv[4 * h + 3]));
      __stcs(reinterpret_cast<float4*>(buf + e) + h, make_float4(bv[4 * h], bv[4 * h + 1], bv[4 * h + 2], bv[4 * h + 3]));
      __stcs(reinterpret_cast<float4*>(m + e) + h, make_float4(mv[4 * h], mv[4 * h + 1], mv[4 * h + 2], mv[4 * h + 3]));
      __stcs(reinterpret_cast<float4*>(v + e) + h, make_float4(vv[4 * h], vv[4 * h + 1], vv[4 * h + 2], vv[4 * h + 3]));
    }
    if (BF16) {
      if (pf) *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(pf) + e) =
          make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
      if (pb) *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(pb) + e) =
          make_uint4(pack_bf16(pv[0], pv[1]), pack_bf16(pv[2], pv[3]), pack_bf16(pv[4], pv[5]), pack_bf16(pv[6], pv[7]));
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (pf) reinterpret_cast<float4*>(static_cast<float*>(pf) + e)[h] =
            make_float4(fv[4 * h], fv[4 * h + 1], fv[4 * h + 2], fv[4 * h + 3]);
        if (pb) reinterpret_cast<float4*>(static_cast<float*>(pb) + e)[h] =
            make_float4(pv[4 * h], pv[4 * h + 1], pv[4 * h + 2], pv[4 * h + 3]);
      }
    }
  }
  const int64_t tail0 = n8 << 3;
  for (int64_t e = tail0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
    float w = W[e], bb = buf[e], mm = m[e], vv = v[e];
    const float d = elem_sgd(s, w, g[e], bb, mm, vv);
    W[e] = w; buf[e] = bb; m[e] = mm; v[e] = vv;
    const float f = __fmaf_rn(nsf, d, w), b = __fmaf_rn(nsb, d, w);
    if (BF16) {
      if (pf) static_cast<__nv_bfloat16*>(pf)[e] = __float2bfloat16_rn(f);
      if (pb) static_cast<__nv_bfloat16*>(pb)[e] = __float2bfloat16_rn(b);
    } else {
      if (pf) static_cast<float*>(pf)[e] = f;
      if (pb) static_cast<float*>(pb)[e] = b;
    }
  }
}

template <bool BF16>
__global__ void predict_copy_kernel(const float* __restrict__ W, void* __restrict__ pf, void* __restrict__ pb,
                                    int64_t n) {
  pdl_wait();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const float w = W[e];
    if (BF16) {
      if (pf) static_cast<__nv_bfloat16*>(pf)[e] = __float2bfloat16_rn(w);
      if (pb) static_cast<__nv_bfloat16*>(pb)[e] = __float2bfloat16_rn(w);
    } else {
      if (pf) static_cast<float*>(pf)[e] = w;
      if (pb) static_cast<float*>(pb)[e] = w;
    }
  }
}

// beta^k by repeated multiplication, c1/r2 in double then rounded
__global__ void bump_kernel(DevState* ds, TraceRec* rec, int stage, int t, int T) {
  pdl_wait();
  ds->ver += 1;
  ds->b1p = ds->b1p * (double)ds->b1;
  ds->b2p = ds->b2p * (double)ds->b2;
  ds->c1 = (float)((double)ds->lr / (1.0 - ds->b1p));
  ds->r2 = (float)(1.0 / sqrt(1.0 - ds->b2p));
  if (rec) {
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    rec->stage = stage; rec->op = 2; rec->t = t; rec->j = T; rec->version = ds->ver; rec->s = 0;
    rec->bellwether = 0; rec->wbuf = ds->ver & 1; rec->t0_ns = now; rec->t1_ns = now;
  }
}

__global__ void state_init_kernel(DevState* ds, float lr, float b1, float b2, float eps, float mu, float wd) {
  pdl_wait();
  ds->ver = 0; ds->fver = 0; ds->bver = 0; ds->pad = 0;
  ds->b1p = 1.0; ds->b2p = 1.0;
  ds->c1 = 0.f; ds->r2 = 0.f;
  ds->omb1 = (float)(1.0 - (double)b1);
  ds->omb2 = (float)(1.0 - (double)b2);
  ds->inv1 = (float)(1.0 / (1.0 - (double)b1));
  ds->inv2 = (float)(1.0 / (1.0 - (double)b2));
  ds->lr = lr; ds->b1 = b1; ds->b2 = b2; ds->eps = eps;
  ds->mu = mu; ds->wd = wd;
}

}  // namespace

void host_scalars(int64_t k, float lr, float b1, float b2, float eps, SweepScalars* o) {
  double b1p = 1.0, b2p = 1.0;
  for (int64_t i = 0; i < k; ++i) { b1p *= (double)b1; b2p *= (double)b2; }
  o->c1 = (float)((double)lr / (1.0 - b1p));
  o->r2 = (float)(1.0 / sqrt(1.0 - b2p));
  o->omb1 = (float)(1.0 - (double)b1);
  o->omb2 = (float)(1.0 - (double)b2);
  o->inv1 = (float)(1.0 / (1.0 - (double)b1));
  o->inv2 = (float)(1.0 / (1.0 - (double)b2));
  o->lr = lr; o->b1 = b1; o->b2 = b2; o->eps = eps; o->mu = 0.f; o->wd = 0.f;
}

static int sweep_grid(int64_t n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  // one 8-parameter group per thread, as many CTAs as that takes (the block scheduler streams
  // them): measured 6.55 TB/s at 2^28 parameters (101 % of the measured copy peak) against
  // 5.4-5.5 TB/s for a grid-stride loop over 4-8 resident CTAs per SM.  XPIPE_SWEEP_CTAS caps
  // the grid at that many CTAs per SM (development knob; 0 = no cap).
  static const int per_sm = [] {
    const char* e = getenv("XPIPE_SWEEP_CTAS");
    return (e && *e) ? atoi(e) : 0;
  }();
  int64_t want = ((n >> 3) + 255) / 256;
  const int64_t cap = per_sm > 0 ? (int64_t)sms * per_sm : ((int64_t)1 << 30);
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

cudaError_t launch_sweep(float* W, const float* g, float* m, float* v, void* pf, void* pb, int64_t n,
                         const DevState* ds, const SweepScalars* hs, float s_f, float s_b, bool bf16, int delta_form,
                         bool update, cudaStream_t st) {
  SweepScalars h{};
  if (hs) h = *hs;
  const int grid = sweep_grid(n);
#define XP_SWEEP(B, U, D) launch_pdl(sweep_kernel<B, U, D>, dim3(grid), dim3(256), 0, st, W, g, m, v, pf, pb, n, ds, h, s_f, s_b)
  if (bf16) {
    if (update) { if (delta_form) XP_SWEEP(true, true, 1); else XP_SWEEP(true, true, 0); }
    else { if (delta_form) XP_SWEEP(true, false, 1); else XP_SWEEP(true, false, 0); }
  } else {
    if (update) { if (delta_form) XP_SWEEP(false, true, 1); else XP_SWEEP(false, true, 0); }
    else { if (delta_form) XP_SWEEP(false, false, 1); else XP_SWEEP(false, false, 0); }
  }
#undef XP_SWEEP
  return cudaGetLastError();
}

cudaError_t launch_sweep_sgd(float* W, const float* g, float* buf, float* m, float* v, void* pf, void* pb, int64_t n,
                             const DevState* ds, const SweepScalars* hs, float s_f, float s_b, bool bf16,
                             cudaStream_t st) {
  SweepScalars h{};
  if (hs) h = *hs;
  const int grid = sweep_grid(n);
  if (bf16) launch_pdl(sweep_sgd_kernel<true>, dim3(grid), dim3(256), 0, st, W, g, buf, m, v, pf, pb, n, ds, h, s_f, s_b);
  else launch_pdl(sweep_sgd_kernel<false>, dim3(grid), dim3(256), 0, st, W, g, buf, m, v, pf, pb, n, ds, h, s_f, s_b);
  return cudaGetLastError();
}

cudaError_t launch_predict_copy(const float* W, void* pf, void* pb, int64_t n, bool bf16, cudaStream_t st) {
  int grid = (int)((n + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  if (bf16) launch_pdl(predict_copy_kernel<true>, dim3(grid), dim3(256), 0, st, W, pf, pb, n);
  else launch_pdl(predict_copy_kernel<false>, dim3(grid), dim3(256), 0, st, W, pf, pb, n);
  return cudaGetLastError();
}

cudaError_t launch_bump(DevState* ds, TraceRec* rec, int stage, int t, int T, cudaStream_t st) {
  launch_pdl(bump_kernel, dim3(1), dim3(1), 0, st, ds, rec, stage, t, T);
  return cudaGetLastError();
}

cudaError_t launch_state_init(DevState* ds, float lr, float b1, float b2, float eps, float mu, float wd,
                              cudaStream_t st) {
  launch_pdl(state_init_kernel, dim3(1), dim3(1), 0, st, ds, lr, b1, b2, eps, mu, wd);
  return cudaGetLastError();
}

}  // namespace xp
