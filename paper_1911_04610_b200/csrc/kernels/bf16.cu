// bf16.cu -- the non-GEMM kernels of the bf16 conv path:
//   input staging (NCHW fp32 -> NHWC bf16, channels padded to 8);
//   BatchNorm statistics of the stored conv output (per-chunk Welford, fixed-order Chan merge);
//   BN-apply + ReLU (+ MaxPool, first-max rule) fused, bf16 out;
//   backward: max-pool routing + ReLU mask + BN reductions fused, then BN input gradient;
//   the small bf16-operand Linear layers (fp32 accumulation, fp32 logits).
// Rounding points follow DESIGN.md section 5: every stored activation / activation gradient
// is bf16 (round-to-nearest-even); statistics, logits and parameter gradients are fp32.
// All reductions are deterministic (fixed order, no atomics).
#include <cstdlib>

#include "../internal.h"
#include "launch.h"
#include "bf16_kernels.h"

namespace xp {

namespace {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float q16(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// 8 consecutive per-channel constants (c0 % 8 == 0): two 16-byte loads where aligned
__device__ __forceinline__ void ld8f(const float* __restrict__ p, float (&v)[8]) {
  if (((uintptr_t)p & 15) == 0) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = p[e];
  }
}
__device__ __forceinline__ void ld8bf(const __nv_bfloat16* __restrict__ p, float (&v)[8]) {
  if (((uintptr_t)p & 15) == 0) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __bfloat162float(b[e]);
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __bfloat162float(p[e]);
  }
}

// The BN-apply + ReLU of one element, bit-identical wherever it is (re)computed:
// a = Q(relu(gamma * ((x - mean) * rstd) + beta))
__device__ __forceinline__ float bn_act(float x, float mean, float rstd, float gamma, float beta, int relu) {
  const float t = __fmul_rn(__fsub_rn(x, mean), rstd);
  const float v = __fadd_rn(__fmul_rn(gamma, t), beta);
  return q16((relu && !(v > 0.f)) ? 0.f : v);
}

// ---- K11 ---------------------------------------------------------------------------------
__global__ void stage_input_bf16_kernel(const float* __restrict__ x, bf16* __restrict__ y, int n, int C, int H, int W,
                                        int Cp) {
  pdl_wait();
  const int total = n * H * W * Cp;  // < 2^30 (checked at launch): 32-bit index arithmetic
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c = i % Cp;
    int r = i / Cp;
    const int w = r % W;
    r /= W;
    const int h = r % H;
    const int s = r / H;
    const float v = c < C ? x[(((int64_t)s * C + c) * H + h) * W + w] : 0.f;
    y[i] = __float2bfloat16_rn(v);
  }
}

// Chan's pairwise merge with explicit roundings (no contraction), so the GEMM epilogue's fused
// BatchNorm (kernels/gemm_tc.cu chan_merge_rn) reproduces it bit for bit
__device__ __forceinline__ void chan_merge(float& na, float& mean, float& m2, float nb, float mb, float m2b) {
  if (nb == 0.f) return;
  if (na == 0.f) { na = nb; mean = mb; m2 = m2b; return; }
  const float nab = __fadd_rn(na, nb);
  const float d = __fsub_rn(mb, mean);
  mean = __fadd_rn(mean, __fmul_rn(d, __fdiv_rn(nb, nab)));
  m2 = __fadd_rn(m2, __fadd_rn(m2b, __fmul_rn(__fmul_rn(d, d), __fdiv_rn(__fmul_rn(na, nb), nab))));
  na = nab;
}

// ---- BN statistics: x [M][C] bf16 -> partial (mean, M2) per row chunk ----------------------
// block: G = C/8 channel groups x RL = T/G row lanes; chunk = RC <= kBnRows*RL rows, so every
// lane keeps its rows in registers.  Two passes over the registers: chunk sum -> chunk mean,
// then sum of squared deviations from that mean; lanes are combined by a fixed pairwise tree
// (deterministic, no divisions on the critical path).
#ifndef XP_BN_ROWS
#define XP_BN_ROWS 4  // 8 measured 0.2-0.7 % slower once the reductions were templated (A/B, r02v)
#endif
constexpr int kBnRows = XP_BN_ROWS;
constexpr int kFinalU = 2;  // partial loads in flight per lane in the final merges

// fixed-order tree over the RL row lanes of slot [rl][G][W] (W floats per (lane, group));
// the result lands in lane 0.  Every thread of the block must call it.
__device__ __forceinline__ void lane_tree(float* sh, int RL, int G, int W, int rl, int g) {
  int p2 = 1;
  while (p2 < RL) p2 <<= 1;
  for (int stride = p2 >> 1; stride > 0; stride >>= 1) {
    __syncthreads();
    if (rl < stride && rl + stride < RL) {
      float* d = sh + ((size_t)rl * G + g) * W;
      const float* o = sh + ((size_t)(rl + stride) * G + g) * W;
      for (int e = 0; e < W; ++e) d[e] = __fadd_rn(d[e], o[e]);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void stats_partial_body(const bf16* __restrict__ x, int M, int C, int RC,
                                                   float* __restrict__ part, int blk) {
  extern __shared__ float sh[];  // [RL][G][8]
  const int G = C / 8, RL = blockDim.x / G;
  const int g = threadIdx.x % G, rl = threadIdx.x / G;
  const bool act = rl < RL;
  const int r0 = blk * RC, r1 = min(M, r0 + RC);
  uint4 keep[kBnRows];
  float sum[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) sum[e] = 0.f;
#pragma unroll
  for (int k = 0; k < kBnRows; ++k) {
    const int r = r0 + rl + k * RL;
    keep[k] = make_uint4(0u, 0u, 0u, 0u);
    if (act && r < r1) {
      keep[k] = *reinterpret_cast<const uint4*>(x + (int64_t)r * C + g * 8);
      const bf16* v = reinterpret_cast<const bf16*>(&keep[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) sum[e] = __fadd_rn(sum[e], __bfloat162float(v[e]));
    }
  }
  float* slot = sh + ((size_t)rl * G + g) * 8;
  if (act)
#pragma unroll
    for (int e = 0; e < 8; ++e) slot[e] = sum[e];
  lane_tree(sh, RL, G, 8, rl, g);
  const float n = (float)(r1 - r0);
  float mean[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) mean[e] = act ? sh[(size_t)g * 8 + e] / n : 0.f;
  __syncthreads();  // everyone has read the sums before the slots are reused
  float m2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) m2[e] = 0.f;
#pragma unroll
  for (int k = 0; k < kBnRows; ++k) {
    const int r = r0 + rl + k * RL;
    if (act && r < r1) {
      const bf16* v = reinterpret_cast<const bf16*>(&keep[k]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = __fsub_rn(__bfloat162float(v[e]), mean[e]);
        m2[e] = __fadd_rn(m2[e], __fmul_rn(d, d));
      }
    }
  }
  if (act)
#pragma unroll
    for (int e = 0; e < 8; ++e) slot[e] = m2[e];
  lane_tree(sh, RL, G, 8, rl, g);
  if (rl == 0) {
    float* p = part + (size_t)blk * 2 * C;
#pragma unroll
    for (int e = 0; e < 8; ++e) { p[g * 8 + e] = mean[e]; p[C + g * 8 + e] = sh[(size_t)g * 8 + e]; }
  }
}
__global__ void bn_stats_partial_kernel(const bf16* __restrict__ x, int M, int C, int RC, float* __restrict__ part) {
  pdl_wait();
  stats_partial_body(x, M, C, RC, part, blockIdx.x);
  pdl_trigger();
}

// Final merge (its own launch, ceil(C/8) blocks of 256 threads): thread (j, cc) = (tid / 8,
// tid % 8) takes channel c = 8*blockIdx.x + cc and merges chunks j, j+32, j+64, ... in order
// (Chan's pairwise formula; loads batched 8 deep), then the 32 lanes of a channel are combined by
// a fixed pairwise tree in shared memory (deterministic).
__device__ __forceinline__ void stats_final_body(const float* __restrict__ part, int chunks, int M, int RC, int C,
                                                 float eps, const bf16* __restrict__ gamma,
                                                 const bf16* __restrict__ beta, float* __restrict__ stats, int unit,
                                                 float* __restrict__ sout = nullptr) {
  // threads >= 256 of a wider block (the fused final + apply kernel) only pass the barriers;
  // sout (shared memory, [4][C], nullable): the 8 channels' results for the block itself
  __shared__ float sh[32][8][3];
  const bool act = threadIdx.x < 256;
  const int cc = threadIdx.x & 7, j = (threadIdx.x >> 3) & 31, c = unit * 8 + cc;
  float na = 0.f, mean = 0.f, m2 = 0.f;
  if (act && c < C) {
    // loads batched kFinalU deep (the ~64 partials of a layer are two per lane; a deeper batch
    // only adds predicated code to fetch), merged in chunk order j, j+32, ...
    for (int k = j; k < chunks; k += kFinalU * 32) {
      float mb[kFinalU], qb[kFinalU];
#pragma unroll
      for (int u = 0; u < kFinalU; ++u) {
        const int kk = k + 32 * u;
        mb[u] = kk < chunks ? __ldcg(part + (size_t)kk * 2 * C + c) : 0.f;
        qb[u] = kk < chunks ? __ldcg(part + (size_t)kk * 2 * C + C + c) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kFinalU; ++u) {
        const int kk = k + 32 * u;
        if (kk < chunks) chan_merge(na, mean, m2, (float)min(RC, M - kk * RC), mb[u], qb[u]);
      }
    }
  }
  if (act) { sh[j][cc][0] = na; sh[j][cc][1] = mean; sh[j][cc][2] = m2; }
  for (int stride = 16; stride > 0; stride >>= 1) {
    __syncthreads();
    if (act && j < stride) {
      float a = sh[j][cc][0], b = sh[j][cc][1], q = sh[j][cc][2];
      chan_merge(a, b, q, sh[j + stride][cc][0], sh[j + stride][cc][1], sh[j + stride][cc][2]);
      sh[j][cc][0] = a; sh[j][cc][1] = b; sh[j][cc][2] = q;
    }
  }
  __syncthreads();
  if (act && j == 0 && c < C) {
    const float mu = sh[0][cc][1];
    const float rs = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(sh[0][cc][2], sh[0][cc][0]), eps)));
    const float ga = __bfloat162float(gamma[c]), be = __bfloat162float(beta[c]);
    stats[c] = mu; stats[C + c] = rs; stats[2 * C + c] = ga; stats[3 * C + c] = be;
    if (sout) { sout[c] = mu; sout[C + c] = rs; sout[2 * C + c] = ga; sout[3 * C + c] = be; }
  }
}
__global__ void bn_stats_final_kernel(const float* __restrict__ part, int chunks, int M, int RC, int C, float eps,
                                      const bf16* __restrict__ gamma, const bf16* __restrict__ beta,
                                      float* __restrict__ stats) {
  pdl_wait();
  stats_final_body(part, chunks, M, RC, C, eps, gamma, beta, stats, blockIdx.x);
  pdl_trigger();
}

// ---- BN-apply [+ ReLU] [+ pool] ----------------------------------------------------------
// y[n][p][q][c] = first max over the pool window (row-major scan) of bn_act(x[n][h][w][c]);
// pidx[n][p][q][c] = the winner's position in the window (the backward routes through it)
// PK = 2: pools whose 2x2 windows tile the map exactly (compile-time window, no bounds checks,
// the four loads issued together); PK = 0: any window, runtime loop
template <int PK>
__device__ __forceinline__ void bn_apply_body(const bf16* __restrict__ x, const float* __restrict__ st,
                                              bf16* __restrict__ y, uint8_t* __restrict__ pidx, int n, int H, int W,
                                              int C, int P, int Q, int kh, int kw, int sh, int sw, int ph, int pw,
                                              int pool, int relu, int i0, int istride,
                                              const bf16* __restrict__ res, int ldy) {
  const int G = C / 8;
  const int total = n * P * Q * G;  // < 2^30 (checked at launch): 32-bit index arithmetic
  for (int i = i0; i < total; i += istride) {
    const int g = i % G;
    int r = i / G;
    const int q = r % Q;
    r /= Q;
    const int p = r % P;
    const int s = r / P;
    const int c0 = g * 8;
    float mean[8], rstd[8], ga[8], be[8], best[8];
    int arg[8];
    ld8f(st + c0, mean); ld8f(st + C + c0, rstd); ld8f(st + 2 * C + c0, ga); ld8f(st + 3 * C + c0, be);
#pragma unroll
    for (int e = 0; e < 8; ++e) { best[e] = 0.f; arg[e] = 0; }
    if (!pool && res) {  // folded residual Add: relu?(Q(Q(BN(x)) + res))
      const int64_t o = (((int64_t)s * H + p) * W + q) * C + c0;
      const uint4 u = *reinterpret_cast<const uint4*>(x + o);
      const uint4 ur = *reinterpret_cast<const uint4*>(res + o);
      const bf16* v = reinterpret_cast<const bf16*>(&u);
      const bf16* rv = reinterpret_cast<const bf16*>(&ur);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float t = q16(__fadd_rn(bn_act(__bfloat162float(v[e]), mean[e], rstd[e], ga[e], be[e], 0),
                                      __bfloat162float(rv[e])));
        best[e] = (relu && !(t > 0.f)) ? 0.f : t;
      }
    } else if (!pool) {
      const uint4 u = *reinterpret_cast<const uint4*>(x + (((int64_t)s * H + p) * W + q) * C + c0);
      const bf16* v = reinterpret_cast<const bf16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) best[e] = bn_act(__bfloat162float(v[e]), mean[e], rstd[e], ga[e], be[e], relu);
    } else {
      bool first = true;
      const int KH = PK ? PK : kh, KW = PK ? PK : kw;
#pragma unroll
      for (int a = 0; a < KH; ++a)
#pragma unroll
        for (int b = 0; b < KW; ++b) {
          const int hh = p * sh - ph + a, ww = q * sw - pw + b;
          if (!PK && (hh < 0 || hh >= H || ww < 0 || ww >= W)) continue;
          const uint4 u = *reinterpret_cast<const uint4*>(x + (((int64_t)s * H + hh) * W + ww) * C + c0);
          const bf16* v = reinterpret_cast<const bf16*>(&u);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float t = bn_act(__bfloat162float(v[e]), mean[e], rstd[e], ga[e], be[e], relu);
            if (first || t > best[e]) { best[e] = t; arg[e] = a * KW + b; }
          }
          first = false;
        }
      uint32_t w2[2] = {0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e) w2[e >> 2] |= (uint32_t)arg[e] << (8 * (e & 3));
      *reinterpret_cast<uint2*>(pidx + (((int64_t)s * P + p) * Q + q) * C + c0) = make_uint2(w2[0], w2[1]);
    }
    uint32_t w4[4];
#pragma unroll
    for (int h2 = 0; h2 < 4; ++h2) {
      __nv_bfloat162 t = __floats2bfloat162_rn(best[2 * h2], best[2 * h2 + 1]);
      w4[h2] = *reinterpret_cast<uint32_t*>(&t);
    }
    *reinterpret_cast<uint4*>(y + (((int64_t)s * P + p) * Q + q) * ldy + c0) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}
template <int PK>
__global__ void bn_apply_kernel(const bf16* __restrict__ x, const float* __restrict__ st, bf16* __restrict__ y,
                                uint8_t* __restrict__ pidx, int n, int H, int W, int C, int P, int Q, int kh, int kw,
                                int sh, int sw, int ph, int pw, int pool, int relu, const bf16* __restrict__ res,
                                int ldy) {
  pdl_wait();
  bn_apply_body<PK>(x, st, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool, relu,
                    blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, res, ldy);
}

// The gradient reaching 8 channels of BN-output element (s,h,w,c0..c0+7), from the stash of
// the forward only (no recomputation): max-pool routing through the stored winner index of
// every window containing (h,w), masked by ReLU on the stored output (the window max is the
// winner's activation, so `y > 0` is exactly the ReLU mask of the winner).
struct BwdGeo {
  int H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool, relu;
  int ldy;  // row pitch of dout / y (the op output; > C for a concat view), pidx stays dense
};

// PM: the pool mode as a compile-time constant (0 none, 2 exact tiling, 1 general windows; G.pool
// holds the same value), or -1 to dispatch on G.pool at run time.  The unrolled reduction loop
// instantiates one mode only: with all three inlined in each of its kBnRows iterations the kernel
// was 7k instructions and stalled mostly on instruction fetch (ncu: "no instruction" 11.6 vs
// long scoreboard 5.2 cycles per issue)
template <int PM = -1>
__device__ __forceinline__ void routed_dy8(const bf16* __restrict__ dout, const bf16* __restrict__ y,
                                           const uint8_t* __restrict__ pidx, const BwdGeo& G, int row, int c0,
                                           float (&dy)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) dy[e] = 0.f;
  if (PM == 0 || (PM < 0 && !G.pool)) {  // row = (s*H + h)*W + w indexes dout/y directly
    const int64_t o = (int64_t)row * G.ldy + c0;
    const uint4 ud = *reinterpret_cast<const uint4*>(dout + o);
    const uint4 uy = *reinterpret_cast<const uint4*>(y + o);
    const bf16* d = reinterpret_cast<const bf16*>(&ud);
    const bf16* yy = reinterpret_cast<const bf16*>(&uy);
#pragma unroll
    for (int e = 0; e < 8; ++e) dy[e] = (G.relu && !(__bfloat162float(yy[e]) > 0.f)) ? 0.f : __bfloat162float(d[e]);
    return;
  }
  const int w = row % G.W, t = row / G.W, h = t % G.H, s = t / G.H;
  if (PM == 2 || (PM < 0 && G.pool == 2)) {  // windows tile the map exactly: the one window holding (h, w)
    const int p = h / G.kh, q = w / G.kw;
    const int pos = (h - p * G.kh) * G.kw + (w - q * G.kw);
    const int64_t ro = ((int64_t)s * G.P + p) * G.Q + q;
    const uint2 ui = *reinterpret_cast<const uint2*>(pidx + ro * G.C + c0);
    const uint4 ud = *reinterpret_cast<const uint4*>(dout + ro * G.ldy + c0);
    const uint4 uy = *reinterpret_cast<const uint4*>(y + ro * G.ldy + c0);
    const bf16* d = reinterpret_cast<const bf16*>(&ud);
    const bf16* yy = reinterpret_cast<const bf16*>(&uy);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int win = (int)(((e < 4 ? ui.x : ui.y) >> (8 * (e & 3))) & 0xFF);
      if (win == pos && !(G.relu && !(__bfloat162float(yy[e]) > 0.f))) dy[e] = __bfloat162float(d[e]);
    }
    return;
  }
  const int plo = max(0, (h + G.ph - G.kh + G.sh) / G.sh), phi = min(G.P - 1, (h + G.ph) / G.sh);
  const int qlo = max(0, (w + G.pw - G.kw + G.sw) / G.sw), qhi = min(G.Q - 1, (w + G.pw) / G.sw);
  int hits[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = plo; p <= phi; ++p)
    for (int q = qlo; q <= qhi; ++q) {
      const int a = h - (p * G.sh - G.ph), b = w - (q * G.sw - G.pw);
      if (a < 0 || a >= G.kh || b < 0 || b >= G.kw) continue;
      const int pos = a * G.kw + b;
      const int64_t ro = ((int64_t)s * G.P + p) * G.Q + q;
      const uint2 ui = *reinterpret_cast<const uint2*>(pidx + ro * G.C + c0);
      const uint4 ud = *reinterpret_cast<const uint4*>(dout + ro * G.ldy + c0);
      const uint4 uy = *reinterpret_cast<const uint4*>(y + ro * G.ldy + c0);
      const bf16* d = reinterpret_cast<const bf16*>(&ud);
      const bf16* yy = reinterpret_cast<const bf16*>(&uy);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int win = (int)(((e < 4 ? ui.x : ui.y) >> (8 * (e & 3))) & 0xFF);
        if (win != pos) continue;
        if (G.relu && !(__bfloat162float(yy[e]) > 0.f)) continue;
        const float g = __bfloat162float(d[e]);
        dy[e] = hits[e] ? __fadd_rn(dy[e], g) : g;
        ++hits[e];
      }
    }
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (hits[e] > 1) dy[e] = q16(dy[e]);
}

// per chunk of RC rows: sum dy and sum dy*xhat per channel (8 channels per thread, row lanes
// combined by a fixed tree) -> part[chunk][2][C]

template <int PM, bool DRES>
__device__ __forceinline__ void bwd_reduce_body(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                                const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                                const float* __restrict__ st, const BwdGeo& G, int M, int RC,
                                                float* __restrict__ part, int blk, bf16* __restrict__ dres,
                                                int acc_res) {
  extern __shared__ float sh[];
  const int C = G.C, NG = C / 8, RL = blockDim.x / NG;
  const int g = threadIdx.x % NG, rl = threadIdx.x / NG;
  const int c0 = g * 8;
  const int r0 = blk * RC, r1 = min(M, r0 + RC);
  float s1[8], s2[8], mean[8], rstd[8];
  ld8f(st + c0, mean); ld8f(st + C + c0, rstd);
#pragma unroll
  for (int e = 0; e < 8; ++e) { s1[e] = 0.f; s2[e] = 0.f; }
#pragma unroll
  for (int k = 0; k < kBnRows; ++k) {  // RC <= kBnRows*RL: every row of the lane, loads in flight together
    const int r = r0 + rl + k * RL;
    if (rl < RL && r < r1) {
      float dy[8];
      routed_dy8<PM>(dout, y, pidx, G, r, c0, dy);
      if (DRES) {  // folded residual Add (unpooled): the residual input's gradient is dy' too
        bf16* dp = dres + (int64_t)r * C + c0;
        float o8[8];
        if (acc_res) ld8bf(dp, o8);
        uint32_t w4[4];
#pragma unroll
        for (int h2 = 0; h2 < 4; ++h2) {
          float v2[2];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int e = 2 * h2 + t;
            v2[t] = acc_res ? __fadd_rn(o8[e], q16(dy[e])) : dy[e];
          }
          __nv_bfloat162 t2 = __floats2bfloat162_rn(v2[0], v2[1]);
          w4[h2] = *reinterpret_cast<uint32_t*>(&t2);
        }
        *reinterpret_cast<uint4*>(dp) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
      const uint4 ux = *reinterpret_cast<const uint4*>(x + (int64_t)r * C + c0);
      const bf16* xv = reinterpret_cast<const bf16*>(&ux);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = __fmul_rn(__fsub_rn(__bfloat162float(xv[e]), mean[e]), rstd[e]);
        s1[e] = __fadd_rn(s1[e], dy[e]);
        s2[e] = __fadd_rn(s2[e], __fmul_rn(dy[e], xh));
      }
    }
  }
  float* slot = sh + ((size_t)rl * NG + g) * 16;
  if (rl < RL)
#pragma unroll
    for (int e = 0; e < 8; ++e) { slot[e] = s1[e]; slot[8 + e] = s2[e]; }
  lane_tree(sh, RL, NG, 16, rl, g);
  if (rl == 0) {
    float* p = part + (size_t)blk * 2 * C;
#pragma unroll
    for (int e = 0; e < 8; ++e) { p[c0 + e] = slot[e]; p[C + c0 + e] = slot[8 + e]; }
  }
}
template <int PM, bool DRES>
__global__ void bn_bwd_reduce_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                     const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                     const float* __restrict__ st, BwdGeo G, int M, int RC, float* __restrict__ part,
                                     bf16* __restrict__ dres, int acc_res) {
  pdl_wait();
  bwd_reduce_body<PM, DRES>(x, dout, y, pidx, st, G, M, RC, part, blockIdx.x, dres, acc_res);
  pdl_trigger();
}

// totals over chunks (layout as bn_stats_final_kernel: 32 lanes per channel over chunks in
// order, then a fixed tree); dgamma/dbeta into the accumulator
__device__ __forceinline__ void bwd_final_body(const float* __restrict__ part, int chunks, int C,
                                               float* __restrict__ tot, float* __restrict__ g_gamma,
                                               float* __restrict__ g_beta, int accumulate, int unit,
                                               float* __restrict__ sout = nullptr) {
  // wider blocks / sout ([2][C], shared): as stats_final_body
  __shared__ float sh[32][8][2];
  const bool act = threadIdx.x < 256;
  const int cc = threadIdx.x & 7, j = (threadIdx.x >> 3) & 31, c = unit * 8 + cc;
  float s1 = 0.f, s2 = 0.f;
  if (act && c < C) {
    for (int k = j; k < chunks; k += kFinalU * 32) {
      float a[kFinalU], b[kFinalU];
#pragma unroll
      for (int u = 0; u < kFinalU; ++u) {
        const int kk = k + 32 * u;
        a[u] = kk < chunks ? __ldcg(part + (size_t)kk * 2 * C + c) : 0.f;
        b[u] = kk < chunks ? __ldcg(part + (size_t)kk * 2 * C + C + c) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kFinalU; ++u)
        if (k + 32 * u < chunks) { s1 = __fadd_rn(s1, a[u]); s2 = __fadd_rn(s2, b[u]); }
    }
  }
  if (act) { sh[j][cc][0] = s1; sh[j][cc][1] = s2; }
  for (int stride = 16; stride > 0; stride >>= 1) {
    __syncthreads();
    if (act && j < stride) {
      sh[j][cc][0] = __fadd_rn(sh[j][cc][0], sh[j + stride][cc][0]);
      sh[j][cc][1] = __fadd_rn(sh[j][cc][1], sh[j + stride][cc][1]);
    }
  }
  __syncthreads();
  if (act && j == 0 && c < C) {
    s1 = sh[0][cc][0]; s2 = sh[0][cc][1];
    tot[c] = s1;
    tot[C + c] = s2;
    if (sout) { sout[c] = s1; sout[C + c] = s2; }
    g_beta[c] = accumulate ? __fadd_rn(g_beta[c], s1) : s1;
    g_gamma[c] = accumulate ? __fadd_rn(g_gamma[c], s2) : s2;
  }
}
__global__ void bn_bwd_final_kernel(const float* __restrict__ part, int chunks, int C, float* __restrict__ tot,
                                    float* __restrict__ g_gamma, float* __restrict__ g_beta, int accumulate) {
  pdl_wait();
  bwd_final_body(part, chunks, C, tot, g_gamma, g_beta, accumulate, blockIdx.x);
  pdl_trigger();
}

// dx = Q(gamma_b * rstd * (dy - sum(dy)/cnt - xhat * sum(dy xhat)/cnt)), 8 channels per thread
template <int PM = -1>
__device__ __forceinline__ void bwd_apply_body(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                               const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                               const float* __restrict__ st, const float* __restrict__ tot,
                                               const bf16* __restrict__ gamma_b, const BwdGeo& G, int M,
                                               bf16* __restrict__ dx, int i0, int istride) {
  const int C = G.C, NG = C / 8;
  const float inv_cnt = 1.f / (float)M;
  const int total = M * NG;  // < 2^30 (checked at launch): 32-bit index arithmetic
  for (int i = i0; i < total; i += istride) {
    const int g = i % NG;
    const int r = i / NG;
    const int c0 = g * 8;
    float dy[8];
    routed_dy8<PM>(dout, y, pidx, G, r, c0, dy);
    const uint4 ux = *reinterpret_cast<const uint4*>(x + (int64_t)r * C + c0);
    const bf16* xv = reinterpret_cast<const bf16*>(&ux);
    float mean[8], rstd[8], gb[8], t1[8], t2[8];
    ld8f(st + c0, mean); ld8f(st + C + c0, rstd); ld8bf(gamma_b + c0, gb); ld8f(tot + c0, t1); ld8f(tot + C + c0, t2);
    uint32_t o4[4];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      float v2[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int e = 2 * e2 + q;
        const float xh = __fmul_rn(__fsub_rn(__bfloat162float(xv[e]), mean[e]), rstd[e]);
        v2[q] = __fmul_rn(__fmul_rn(gb[e], rstd[e]), __fsub_rn(__fsub_rn(dy[e], __fmul_rn(t1[e], inv_cnt)),
                                                              __fmul_rn(xh, __fmul_rn(t2[e], inv_cnt))));
      }
      __nv_bfloat162 t2 = __floats2bfloat162_rn(v2[0], v2[1]);
      o4[e2] = *reinterpret_cast<uint32_t*>(&t2);
    }
    *reinterpret_cast<uint4*>(dx + (int64_t)r * C + c0) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
  }
}
template <int PM>
__global__ void bn_bwd_apply_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                    const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                    const float* __restrict__ st, const float* __restrict__ tot,
                                    const bf16* __restrict__ gamma_b, BwdGeo G, int M, bf16* __restrict__ dx) {
  pdl_wait();
  bwd_apply_body<PM>(x, dout, y, pidx, st, tot, gamma_b, G, M, dx, blockIdx.x * blockDim.x + threadIdx.x,
                 gridDim.x * blockDim.x);
}

// Pooled layers whose windows tile the map exactly (kh == sh, kw == sw, no padding, H = P*kh,
// W = Q*kw): one thread per (pooled output, 8 channels) -- the routed gradient, winner index and
// ReLU mask are loaded once for the kh*kw inputs of the window; per element the arithmetic is
// bn_bwd_apply_kernel's (every input lies in exactly one window, so no Q() of a fan-in sum).
template <int PK>  // 2: 2x2 windows (compile-time, unrolled), 0: runtime kh x kw
__device__ __forceinline__ void bwd_apply_tiled_body(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                                     const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                                     const float* __restrict__ st, const float* __restrict__ tot,
                                                     const bf16* __restrict__ gamma_b, const BwdGeo& G, int M, int Mo,
                                                     bf16* __restrict__ dx, int i0, int istride) {
  const int C = G.C, NG = C / 8;
  const float inv_cnt = 1.f / (float)M;
  const int total = Mo * NG;  // < 2^30 (checked at launch)
  for (int i = i0; i < total; i += istride) {
    const int g = i % NG, ro = i / NG;
    const int q = ro % G.Q, t = ro / G.Q, p = t % G.P, s = t / G.P;
    const int c0 = g * 8;
    const uint2 ui = *reinterpret_cast<const uint2*>(pidx + (int64_t)ro * C + c0);
    const uint4 ud = *reinterpret_cast<const uint4*>(dout + (int64_t)ro * G.ldy + c0);
    const uint4 uy = *reinterpret_cast<const uint4*>(y + (int64_t)ro * G.ldy + c0);
    const bf16* d = reinterpret_cast<const bf16*>(&ud);
    const bf16* yy = reinterpret_cast<const bf16*>(&uy);
    float gv[8];
    int win[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      win[e] = (int)(((e < 4 ? ui.x : ui.y) >> (8 * (e & 3))) & 0xFF);
      gv[e] = (G.relu && !(__bfloat162float(yy[e]) > 0.f)) ? 0.f : __bfloat162float(d[e]);
    }
    float mean[8], rstd[8], gb[8], t1[8], t2[8];
    ld8f(st + c0, mean); ld8f(st + C + c0, rstd); ld8bf(gamma_b + c0, gb); ld8f(tot + c0, t1); ld8f(tot + C + c0, t2);
    const int KH = PK ? PK : G.kh, KW = PK ? PK : G.kw;
#pragma unroll
    for (int a = 0; a < KH; ++a)
#pragma unroll
      for (int b = 0; b < KW; ++b) {
        const int pos = a * KW + b;
        const int64_t r = ((int64_t)s * G.H + p * KH + a) * G.W + q * KW + b;
        const uint4 ux = *reinterpret_cast<const uint4*>(x + r * C + c0);
        const bf16* xv = reinterpret_cast<const bf16*>(&ux);
        uint32_t o4[4];
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          float v2[2];
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int e = 2 * e2 + h2;
            const float dy = win[e] == pos ? gv[e] : 0.f;
            const float xh = __fmul_rn(__fsub_rn(__bfloat162float(xv[e]), mean[e]), rstd[e]);
            v2[h2] = __fmul_rn(__fmul_rn(gb[e], rstd[e]), __fsub_rn(__fsub_rn(dy, __fmul_rn(t1[e], inv_cnt)),
                                                                    __fmul_rn(xh, __fmul_rn(t2[e], inv_cnt))));
          }
          __nv_bfloat162 t2v = __floats2bfloat162_rn(v2[0], v2[1]);
          o4[e2] = *reinterpret_cast<uint32_t*>(&t2v);
        }
        *reinterpret_cast<uint4*>(dx + r * C + c0) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
      }
  }
}
template <int PK>
__global__ void bn_bwd_apply_tiled_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                          const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                          const float* __restrict__ st, const float* __restrict__ tot,
                                          const bf16* __restrict__ gamma_b, BwdGeo G, int M, int Mo,
                                          bf16* __restrict__ dx) {
  pdl_wait();
  bwd_apply_tiled_body<PK>(x, dout, y, pidx, st, tot, gamma_b, G, M, Mo, dx, blockIdx.x * blockDim.x + threadIdx.x,
                           gridDim.x * blockDim.x);
}

// ---- final merge + elementwise pass in one launch, one block per 8 channels ------------------
// Layers with few rows (M <= kFaRows): block u merges the partials of channels 8u..8u+7 exactly as
// the separate final kernel does (same body, same bits) and then runs the elementwise pass for
// those channels over every row (i = u + G*tid, stride G*blockDim: the separate kernels' item
// index restricted to group u).  No block repeats another's merge, so one launch per BatchNorm
// and direction disappears at no extra work.
constexpr int kFaThreads = 512;
template <int PK>
__global__ void __launch_bounds__(kFaThreads) bn_final_apply_kernel(
    const float* __restrict__ part, int chunks, int M, int RC, float eps, const bf16* __restrict__ gamma,
    const bf16* __restrict__ beta, float* __restrict__ stats, const bf16* __restrict__ x, bf16* __restrict__ y,
    uint8_t* __restrict__ pidx, int n, int H, int W, int C, int P, int Q, int kh, int kw, int sh, int sw, int ph,
    int pw, int pool, int relu, const bf16* __restrict__ res, int ldy) {
  extern __shared__ float fst[];  // [4][C]: this block's 8 channels filled
  pdl_wait();
  stats_final_body(part, chunks, M, RC, C, eps, gamma, beta, stats, blockIdx.x, fst);
  __syncthreads();
  const int G = C / 8;
  bn_apply_body<PK>(x, fst, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool, relu,
                    (int)blockIdx.x + G * (int)threadIdx.x, G * (int)blockDim.x, res, ldy);
}
// TL: 2 / 1 the exact-tiling pooled body (2x2 / runtime window), 0 the row body (PM = G.pool)
template <int TL>
__global__ void __launch_bounds__(kFaThreads) bn_bwd_final_apply_kernel(
    const float* __restrict__ part, int chunks, float* __restrict__ tot, float* __restrict__ g_gamma,
    float* __restrict__ g_beta, int accumulate, const bf16* __restrict__ x, const bf16* __restrict__ dout,
    const bf16* __restrict__ y, const uint8_t* __restrict__ pidx, const float* __restrict__ st,
    const bf16* __restrict__ gamma_b, BwdGeo G, int M, int Mo, bf16* __restrict__ dx) {
  extern __shared__ float ftot[];  // [2][C]
  pdl_wait();
  const int C = G.C, NG = C / 8;
  bwd_final_body(part, chunks, C, tot, g_gamma, g_beta, accumulate, blockIdx.x, ftot);
  __syncthreads();
  const int i0 = (int)blockIdx.x + NG * (int)threadIdx.x, is = NG * (int)blockDim.x;
  if (TL == 2) bwd_apply_tiled_body<2>(x, dout, y, pidx, st, ftot, gamma_b, G, M, Mo, dx, i0, is);
  else if (TL == 1) bwd_apply_tiled_body<0>(x, dout, y, pidx, st, ftot, gamma_b, G, M, Mo, dx, i0, is);
  else if (G.pool) bwd_apply_body<1>(x, dout, y, pidx, st, ftot, gamma_b, G, M, dx, i0, is);
  else bwd_apply_body<0>(x, dout, y, pidx, st, ftot, gamma_b, G, M, dx, i0, is);
}

// ---- folded BatchNorm merges (small layers) -------------------------------------------------
// The per-channel merge of the partials (bn_stats_final_kernel / bn_bwd_final_kernel) done by
// every CTA of the elementwise kernel that needs its result, into shared memory, so one launch
// per BatchNorm and direction disappears.  Used where the partials are few (chunks x C <= kFoldFloats) and the layer small
// (M x C <= kFoldElems): every CTA then re-reads at most 64 KB of partials from L2.
constexpr int kFoldFloats = 8192;
constexpr int64_t kFoldElems = int64_t(1) << 20;

// Each CTA merges the (few) partials of every channel sequentially in chunk order, all of a
// channel's loads in flight together (the separate final kernels use 32 lanes per channel and a
// pairwise tree, one CTA per 8 channels -- a different summation order: this path matches them
// to fp32 rounding, not bit for bit)
__device__ __forceinline__ void stats_merge_seq(const float* __restrict__ part, int chunks, int M, int RC, int C, int c,
                                                float& mean, float& m2, float& n) {
  n = 0.f; mean = 0.f; m2 = 0.f;
  for (int k0 = 0; k0 < chunks; k0 += 8) {
    float mb[8], qb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u;
      mb[u] = k < chunks ? __ldcg(part + (size_t)k * 2 * C + c) : 0.f;
      qb[u] = k < chunks ? __ldcg(part + (size_t)k * 2 * C + C + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < chunks) chan_merge(n, mean, m2, (float)min(RC, M - (k0 + u) * RC), mb[u], qb[u]);
  }
}
__device__ __forceinline__ void sums_merge_seq(const float* __restrict__ part, int chunks, int C, int c, float& s1,
                                               float& s2) {
  s1 = 0.f; s2 = 0.f;
  for (int k0 = 0; k0 < chunks; k0 += 8) {
    float a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u;
      a[u] = k < chunks ? __ldcg(part + (size_t)k * 2 * C + c) : 0.f;
      b[u] = k < chunks ? __ldcg(part + (size_t)k * 2 * C + C + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < chunks) { s1 = __fadd_rn(s1, a[u]); s2 = __fadd_rn(s2, b[u]); }
  }
}

// forward: statistics merge (+ the stashed stats, by CTA 0) then BN-apply [+ ReLU] [+ pool]
template <int PK>
__global__ void __launch_bounds__(256, 2) bn_apply_fold_kernel(const bf16* __restrict__ x, const float* __restrict__ part, int chunks, int M, int RC,
                                     float eps, const bf16* __restrict__ gamma, const bf16* __restrict__ beta,
                                     float* __restrict__ stats, bf16* __restrict__ y, uint8_t* __restrict__ pidx, int n,
                                     int H, int W, int C, int P, int Q, int kh, int kw, int sh, int sw, int ph, int pw,
                                     int pool, int relu, const bf16* __restrict__ res, int ldy) {
  extern __shared__ float sst[];  // [4][C]: mean, rstd, gamma, beta
  pdl_wait();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float mean, m2, cnt;
    stats_merge_seq(part, chunks, M, RC, C, c, mean, m2, cnt);
    const float rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(m2, cnt), eps)));
    const float ga = __bfloat162float(gamma[c]), be = __bfloat162float(beta[c]);
    sst[c] = mean; sst[C + c] = rstd; sst[2 * C + c] = ga; sst[3 * C + c] = be;
    if (blockIdx.x == 0) { stats[c] = mean; stats[C + c] = rstd; stats[2 * C + c] = ga; stats[3 * C + c] = be; }
  }
  __syncthreads();
  bn_apply_body<PK>(x, sst, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool, relu,
                    blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, res, ldy);
}

// backward: totals merge (+ dgamma, dbeta into the accumulator, by CTA 0) then the input gradient
template <int AP>
__global__ void __launch_bounds__(256, 2) bn_bwd_apply_fold_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dout,
                                         const bf16* __restrict__ y, const uint8_t* __restrict__ pidx,
                                         const float* __restrict__ st, const float* __restrict__ part, int chunks,
                                         float* __restrict__ g_gamma, float* __restrict__ g_beta, int accumulate,
                                         const bf16* __restrict__ gamma_b, BwdGeo G, int M, int Mo,
                                         bf16* __restrict__ dx) {
  extern __shared__ float stot[];  // [2][C]
  pdl_wait();
  const int C = G.C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float s1, s2;
    sums_merge_seq(part, chunks, C, c, s1, s2);
    stot[c] = s1; stot[C + c] = s2;
    if (blockIdx.x == 0) {
      g_beta[c] = accumulate ? __fadd_rn(g_beta[c], s1) : s1;
      g_gamma[c] = accumulate ? __fadd_rn(g_gamma[c], s2) : s2;
    }
  }
  __syncthreads();
  const int i0 = blockIdx.x * blockDim.x + threadIdx.x, is = gridDim.x * blockDim.x;
  if (AP == 0) bwd_apply_body(x, dout, y, pidx, st, stot, gamma_b, G, M, dx, i0, is);
  else bwd_apply_tiled_body<AP == 2 ? 2 : 0>(x, dout, y, pidx, st, stot, gamma_b, G, M, Mo, dx, i0, is);
}

// ---- bf16-operand Linear (small: micro-batch rows) ------------------------------------------
// y[r][o] = sum_i x[r][i] W[o][i] (fp32) + b[o]; logits: fp32 out, else Q(relu?) bf16.
// One warp per (r, o); lanes stride over i, shuffle reduction.
__global__ void linear_fwd_bf16_kernel(const bf16* __restrict__ x, const bf16* __restrict__ W,
                                       const bf16* __restrict__ b, void* __restrict__ y, int n, int in, int out,
                                       int relu, int f32out) {
  pdl_wait();
  const int wid = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wid >= n * out) return;
  const int r = wid / out, o = wid % out;
  float acc = 0.f;
  for (int i = lane; i < in; i += 32) acc += __bfloat162float(x[(int64_t)r * in + i]) * __bfloat162float(W[(int64_t)o * in + i]);
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    float v = b ? __fadd_rn(acc, __bfloat162float(b[o])) : acc;
    if (f32out) static_cast<float*>(y)[(int64_t)r * out + o] = v;
    else {
      if (relu) v = v > 0.f ? v : 0.f;
      static_cast<bf16*>(y)[(int64_t)r * out + o] = __float2bfloat16_rn(v);
    }
  }
}

template <bool DY_F32>
__device__ __forceinline__ float load_dy(const void* dy, int64_t idx, const bf16* mask) {
  float d = DY_F32 ? q16(static_cast<const float*>(dy)[idx]) : __bfloat162float(static_cast<const bf16*>(dy)[idx]);
  if (mask && !(__bfloat162float(mask[idx]) > 0.f)) d = 0.f;
  return d;
}

// tensor-core Linear backward operand: dyp[r][o] = dy'[r][o] (bf16; the masked, bf16-rounded
// output gradient load_dy gives), zero for out <= o < ldp; gb[o] (=|+=) sum_r dy'[r][o] in r order
// (the bias gradient of linear_wgrad_bf16_kernel, same bits)
template <bool DY_F32>
__global__ void linear_dy_prep_kernel(const void* __restrict__ dy, const bf16* __restrict__ mask, bf16* __restrict__ dyp,
                                      int ldp, float* __restrict__ gb, int n, int out, int accumulate) {
  pdl_wait();
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= ldp) return;
  float acc = 0.f;
  for (int r0 = 0; r0 < n; r0 += 8) {  // eight rows' loads in flight, then the in-order sum
    float d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      d[u] = (o < out && r0 + u < n) ? load_dy<DY_F32>(dy, (int64_t)(r0 + u) * out + o, mask) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (r0 + u < n) {
        dyp[(int64_t)(r0 + u) * ldp + o] = __float2bfloat16_rn(d[u]);
        acc += d[u];
      }
  }
  if (gb && o < out) gb[o] = accumulate ? __fadd_rn(gb[o], acc) : acc;
}

// dx[r][i] = Q(sum_o dy'[r][o] W[o][i]); thread per (r, i)
template <bool DY_F32>
__global__ void linear_dgrad_bf16_kernel(const void* __restrict__ dy, const bf16* __restrict__ mask,
                                         const bf16* __restrict__ W, bf16* __restrict__ dx, int n, int in, int out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  if (i >= in || r >= n) return;
  float acc = 0.f;
  for (int o = 0; o < out; ++o) acc += load_dy<DY_F32>(dy, (int64_t)r * out + o, mask) * __bfloat162float(W[(int64_t)o * in + i]);
  dx[(int64_t)r * in + i] = __float2bfloat16_rn(acc);
}

// gW[o][i] (=|+=) sum_r dy'[r][o] x[r][i]; gb[o] (=|+=) sum_r dy'[r][o]
template <bool DY_F32>
__global__ void linear_wgrad_bf16_kernel(const void* __restrict__ dy, const bf16* __restrict__ mask,
                                         const bf16* __restrict__ x, float* __restrict__ gW, float* __restrict__ gb,
                                         int n, int in, int out, int accumulate) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int o = blockIdx.y;
  if (i > in || (i == in && !gb)) return;
  float acc = 0.f;
  for (int r = 0; r < n; ++r) {
    const float d = load_dy<DY_F32>(dy, (int64_t)r * out + o, mask);
    acc += i < in ? d * __bfloat162float(x[(int64_t)r * in + i]) : d;
  }
  float* dst = i < in ? &gW[(int64_t)o * in + i] : &gb[o];
  *dst = accumulate ? __fadd_rn(*dst, acc) : acc;
}

// development switch: XPIPE_NO_BN_TILED=1 keeps the per-input-element pooled BN backward
bool bn_tiled_off() {
  static const bool v = [] { const char* e = getenv("XPIPE_NO_BN_TILED"); return e && *e && *e != '0'; }();
  return v;
}

// element-count bound of the 32-bit-indexed elementwise kernels (index + grid stride < 2^31)
constexpr int64_t kMaxElems = int64_t(1) << 30;

int grid1d(int64_t n, int threads = 256) {
  static const int cap = [] {  // development knob: CTA cap of the elementwise kernels
    const char* e = getenv("XPIPE_EW_CTAS");
    return (e && *e) ? std::max(1, atoi(e)) : 148 * 16;
  }();
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap));
}

}  // namespace

// explicit im2col of a conv input with few channels (C % 8 == 0, C < 64): cols[m][(r*S+s)*C + c]
// = x[n][p*sh-ph+r][q*sw-pw+s][c] (zero outside), m = (n*P + p)*Q + q; 8 channels per thread
__global__ void im2col_bf16_kernel(const bf16* __restrict__ x, bf16* __restrict__ cols, int n, int H, int W, int C,
                                   int P, int Q, int R, int S, int sh, int sw, int ph, int pw) {
  pdl_wait();
  const int G = C / 8, taps = R * S;
  const int total = n * P * Q * taps * G;  // < 2^30 (checked at launch): 32-bit index arithmetic
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % G;
    const int r0 = i / G;
    const int tap = r0 % taps;
    const int m = r0 / taps;
    const int q = m % Q, t = m / Q, p = t % P, s_img = t / P;
    const int r = tap / S, s = tap - r * S;
    const int ih = p * sh - ph + r, iw = q * sw - pw + s;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (ih >= 0 && ih < H && iw >= 0 && iw < W)
      v = *reinterpret_cast<const uint4*>(x + (((int64_t)s_img * H + ih) * W + iw) * C + g * 8);
    *reinterpret_cast<uint4*>(cols + (int64_t)m * taps * C + tap * C + g * 8) = v;
  }
}

cudaError_t launch_im2col_bf16(const bf16* x, bf16* cols, int n, int H, int W, int C, int P, int Q, int R, int S,
                               int sh, int sw, int ph, int pw, cudaStream_t st) {
  if (C % 8 || (int64_t)n * P * Q * R * S * (C / 8) >= kMaxElems) return cudaErrorInvalidValue;
  launch_pdl(im2col_bf16_kernel, dim3(grid1d((int64_t)n * P * Q * R * S * (C / 8))), dim3(256), 0, st, x, cols, n, H, W,
             C, P, Q, R, S, sh, sw, ph, pw);
  return cudaGetLastError();
}

cudaError_t launch_stage_input_bf16(const float* x, bf16* y, int n, int C, int H, int W, int Cp, cudaStream_t st) {
  if ((int64_t)n * H * W * Cp >= kMaxElems) return cudaErrorInvalidValue;
  launch_pdl(stage_input_bf16_kernel, dim3(grid1d((int64_t)n * H * W * Cp)), dim3(256), 0, st, x, y, n, C, H, W, Cp);
  return cudaGetLastError();
}

// block shape of the BN reductions: G = C/8 channel groups x RL row lanes (256 threads, or G)
int bn_threads(int C) { const int G = C / 8; return G >= 256 ? G : (256 / G) * G; }
// rows per partial chunk: ~64 chunks (a few rows per lane, every load in flight at once; fewer
// partials make the final merge a single round of loads -- 512 chunks measured 9 % slower in the
// 4-stage pipeline), at most kBnRows rows per lane (register-resident two passes)
// folded merges are opt-in (XPIPE_BN_FOLD=1): measured slower in the pipeline (VGG-16 K=4 102.7k
// vs 113.1k samples/s, ResNet-101 K=8 23.8k vs 27.9k, Inception-V3 K=4 24.2k vs 25.3k) -- every
// CTA's merge is a chain of dependent L2 round trips ahead of its elementwise work
bool bn_fold_off() {
  static const bool v = [] { const char* e = getenv("XPIPE_BN_FOLD"); return !(e && *e == '1'); }();
  return v;
}
int bn_chunk_rows(int M, int C) {
  const int RL = bn_threads(C) / (C / 8);
  static const int target = [] {  // development knob: target chunk count
    const char* e = getenv("XPIPE_BN_CHUNKS");
    return (e && *e) ? std::max(1, atoi(e)) : 64;  // measured: 512 -> 64 chunks +9 % (VGG-16 K=4)
  }();
  const int rc = std::max(1, std::min(std::max(RL, (M + target - 1) / target), kBnRows * RL));
  // a small layer whose partials could be folded into the elementwise pass with the longest
  // chunks: take those (fewer partials)
  const int rmax = std::max(1, kBnRows * RL);
  if (!bn_fold_off() && (int64_t)M * C <= kFoldElems && (int64_t)((M + rc - 1) / rc) * C > kFoldFloats &&
      (int64_t)((M + rmax - 1) / rmax) * C <= kFoldFloats)
    return rmax;
  return rc;
}
// fold the final merge of `chunks` partials into the elementwise kernel (see bn_apply_fold_kernel)
bool bn_fold(int M, int C, int chunks) {
  return !bn_fold_off() && (int64_t)M * C <= kFoldElems && (int64_t)chunks * C <= kFoldFloats;
}
// final merge and elementwise pass as one launch (bn_final_apply_kernel / bn_bwd_final_apply_kernel)
// for layers of at most XPIPE_BN_FA_ROWS rows (default 2048: at most 4 rows per thread of the
// 512-thread blocks).  Opt-in (XPIPE_BN_FA=1): bit-identical, one launch per BatchNorm and
// direction fewer, but measured slower in the pipeline (A/B on one B200: VGG-16 K=4 111.0k vs
// 120.7k, ResNet-101 K=8 23.9k vs 28.8k, Inception-V3 K=4 25.8k vs 27.0k samples/s) -- C/8
// blocks walking every row with 16-byte row-strided accesses replace a wide, coalesced grid
bool bn_fa(int M) {
  static const int rows = [] {
    const char* e = getenv("XPIPE_BN_FA");
    if (!(e && *e == '1')) return 0;
    const char* r = getenv("XPIPE_BN_FA_ROWS");
    return (r && *r) ? atoi(r) : 2048;
  }();
  return M <= rows;
}
inline float* ws_mut(const float* p) { return const_cast<float*>(p); }
int fold_grid(int64_t items) { return std::min(grid1d(items), 2 * 148); }
int bn_chunks(int M, int C) { return (M + bn_chunk_rows(M, C) - 1) / bn_chunk_rows(M, C); }
size_t bn_ws_floats(int M, int C) { return (size_t)bn_chunks(M, C) * 2 * C + 2 * (size_t)C; }

cudaError_t launch_bn_stats(const bf16* x, int M, int C, float eps, const bf16* gamma, const bf16* beta, float* ws,
                            int* counter, float* stats, cudaStream_t st) {
  if (C % 8 || C > 2048) return cudaErrorInvalidValue;
  const int RC = bn_chunk_rows(M, C), chunks = bn_chunks(M, C);
  const int threads = bn_threads(C);
  const size_t shm = (size_t)threads * 8 * 4;
  (void)counter;
  launch_pdl(bn_stats_partial_kernel, dim3(chunks), dim3(threads), shm, st, x, M, C, RC, ws);
  launch_pdl(bn_stats_final_kernel, dim3((C + 7) / 8), dim3(256), 0, st, (const float*)ws, chunks, M, RC, C, eps, gamma,
             beta, stats);
  return cudaGetLastError();
}

cudaError_t launch_bn_stats_partial(const bf16* x, int M, int C, float* ws, cudaStream_t st) {
  if (C % 8 || C > 2048) return cudaErrorInvalidValue;
  const int RC = bn_chunk_rows(M, C), chunks = bn_chunks(M, C);
  const int threads = bn_threads(C);
  launch_pdl(bn_stats_partial_kernel, dim3(chunks), dim3(threads), (size_t)threads * 8 * 4, st, x, M, C, RC, ws);
  return cudaGetLastError();
}

cudaError_t launch_bn_apply_stats(const float* part, int chunks, int RC, float eps, const bf16* gamma, const bf16* beta,
                                  float* stats, const bf16* x, bf16* y, uint8_t* pidx, int n, int H, int W, int C,
                                  int P, int Q, int kh, int kw, int sh, int sw, int ph, int pw, bool pool, bool relu,
                                  cudaStream_t st, const bf16* res, int ldy) {
  const int M = n * H * W;
  if (!bn_fold(M, C, chunks) && bn_fa(M)) {
    if (!ldy) ldy = C;
    const int64_t total = (int64_t)n * P * Q * (C / 8);
    if (C % 8 || C > 2048 || total >= kMaxElems || (res && pool)) return cudaErrorInvalidValue;
    const size_t shm = (size_t)4 * C * 4;
    if (pool && kh == 2 && kw == 2 && sh == 2 && sw == 2 && ph == 0 && pw == 0 && H == 2 * P && W == 2 * Q &&
        !bn_tiled_off())
      launch_pdl(bn_final_apply_kernel<2>, dim3(C / 8), dim3(kFaThreads), shm, st, part, chunks, M, RC, eps, gamma,
                 beta, stats, x, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, 1, relu ? 1 : 0,
                 (const bf16*)nullptr, ldy);
    else
      launch_pdl(bn_final_apply_kernel<0>, dim3(C / 8), dim3(kFaThreads), shm, st, part, chunks, M, RC, eps, gamma,
                 beta, stats, x, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool ? 1 : 0, relu ? 1 : 0, res,
                 ldy);
    return cudaGetLastError();
  }
  if (!bn_fold(M, C, chunks)) {
    cudaError_t e = launch_bn_stats_final(part, chunks, M, RC, C, eps, gamma, beta, stats, st);
    if (e != cudaSuccess) return e;
    return launch_bn_apply(x, stats, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool, relu, st, res, ldy);
  }
  if (!ldy) ldy = C;
  const int64_t total = (int64_t)n * P * Q * (C / 8);
  if (C % 8 || C > 2048 || total >= kMaxElems || (res && pool)) return cudaErrorInvalidValue;
  const size_t shm = (size_t)4 * C * 4;
  if (pool && kh == 2 && kw == 2 && sh == 2 && sw == 2 && ph == 0 && pw == 0 && H == 2 * P && W == 2 * Q &&
      !bn_tiled_off())
    launch_pdl(bn_apply_fold_kernel<2>, dim3(fold_grid(total)), dim3(256), shm, st, x, part, chunks, M, RC, eps, gamma,
               beta, stats, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, 1, relu ? 1 : 0, (const bf16*)nullptr,
               ldy);
  else
    launch_pdl(bn_apply_fold_kernel<0>, dim3(fold_grid(total)), dim3(256), shm, st, x, part, chunks, M, RC, eps, gamma,
               beta, stats, y, pidx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw, pool ? 1 : 0, relu ? 1 : 0, res, ldy);
  return cudaGetLastError();
}

cudaError_t launch_bn_stats_final(const float* part, int chunks, int M, int RC, int C, float eps, const bf16* gamma,
                                  const bf16* beta, float* stats, cudaStream_t st) {
  if (C % 8 || C > 2048) return cudaErrorInvalidValue;
  launch_pdl(bn_stats_final_kernel, dim3((C + 7) / 8), dim3(256), 0, st, part, chunks, M, RC, C, eps, gamma, beta, stats);
  return cudaGetLastError();
}

cudaError_t launch_bn_apply(const bf16* x, const float* stats, bf16* y, uint8_t* pidx, int n, int H, int W, int C, int P,
                            int Q, int kh, int kw, int sh, int sw, int ph, int pw, bool pool, bool relu, cudaStream_t st,
                            const bf16* res, int ldy) {
  if (!ldy) ldy = C;
  const int64_t total = (int64_t)n * P * Q * (C / 8);
  if (C % 8 || total >= kMaxElems || (res && pool)) return cudaErrorInvalidValue;
  if (pool && kh == 2 && kw == 2 && sh == 2 && sw == 2 && ph == 0 && pw == 0 && H == 2 * P && W == 2 * Q &&
      !bn_tiled_off())
    launch_pdl(bn_apply_kernel<2>, dim3(grid1d(total)), dim3(256), 0, st, x, stats, y, pidx, n, H, W, C, P, Q, kh, kw, sh,
               sw, ph, pw, 1, relu ? 1 : 0, (const bf16*)nullptr, ldy);
  else
    launch_pdl(bn_apply_kernel<0>, dim3(grid1d(total)), dim3(256), 0, st, x, stats, y, pidx, n, H, W, C, P, Q, kh, kw, sh,
               sw, ph, pw, pool ? 1 : 0, relu ? 1 : 0, res, ldy);
  return cudaGetLastError();
}

cudaError_t launch_bn_bwd_reduce(const bf16* x, const bf16* dout, const bf16* y, const uint8_t* pidx,
                                 const float* stats, int n, int H, int W, int C, int P, int Q, int kh, int kw, int sh,
                                 int sw, int ph, int pw, bool pool, bool relu, float* ws, float* g_gamma, float* g_beta,
                                 bool accumulate, cudaStream_t st, bf16* dres, bool acc_res, int ldy) {
  if (C % 8 || C > 2048 || (dres && pool) || (ldy && ldy % 8)) return cudaErrorInvalidValue;
  BwdGeo G{H, W, C, pool ? P : H, pool ? Q : W, kh, kw, sh, sw, ph, pw, pool ? 1 : 0, relu ? 1 : 0, ldy ? ldy : C};
  if (pool && kh == sh && kw == sw && ph == 0 && pw == 0 && H == P * kh && W == Q * kw && !bn_tiled_off()) G.pool = 2;
  const int M = n * H * W;
  const int RC = bn_chunk_rows(M, C), chunks = bn_chunks(M, C);
  const int threads = bn_threads(C);
  const size_t shm = (size_t)threads * 16 * 4;
  float* tot = ws + (size_t)chunks * 2 * C;
  const int ar = acc_res ? 1 : 0;
  if (G.pool == 2)
    launch_pdl(bn_bwd_reduce_kernel<2, false>, dim3(chunks), dim3(threads), shm, st, x, dout, y, pidx, stats, G, M, RC,
               ws, (bf16*)nullptr, ar);
  else if (G.pool)
    launch_pdl(bn_bwd_reduce_kernel<1, false>, dim3(chunks), dim3(threads), shm, st, x, dout, y, pidx, stats, G, M, RC,
               ws, (bf16*)nullptr, ar);
  else if (dres)
    launch_pdl(bn_bwd_reduce_kernel<0, true>, dim3(chunks), dim3(threads), shm, st, x, dout, y, pidx, stats, G, M, RC,
               ws, dres, ar);
  else
    launch_pdl(bn_bwd_reduce_kernel<0, false>, dim3(chunks), dim3(threads), shm, st, x, dout, y, pidx, stats, G, M, RC,
               ws, (bf16*)nullptr, ar);
  if (bn_fold(M, C, chunks) || bn_fa(M)) return cudaGetLastError();  // the merge runs in launch_bn_bwd_apply
  launch_pdl(bn_bwd_final_kernel, dim3((C + 7) / 8), dim3(256), 0, st, (const float*)ws, chunks, C, tot, g_gamma, g_beta,
             accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_bn_bwd_apply(const bf16* x, const bf16* dout, const bf16* y, const uint8_t* pidx, const float* stats,
                                const bf16* gamma_b, int n, int H, int W, int C, int P, int Q, int kh, int kw, int sh,
                                int sw, int ph, int pw, bool pool, bool relu, const float* ws, bf16* dx,
                                cudaStream_t st, int ldy, float* g_gamma, float* g_beta, bool accumulate) {
  if (C % 8 || C > 2048 || (ldy && ldy % 8)) return cudaErrorInvalidValue;
  BwdGeo G{H, W, C, pool ? P : H, pool ? Q : W, kh, kw, sh, sw, ph, pw, pool ? 1 : 0, relu ? 1 : 0, ldy ? ldy : C};
  const int M = n * H * W;
  const int chunks = bn_chunks(M, C);
  const float* tot = ws + (size_t)chunks * 2 * C;
  if ((int64_t)M * (C / 8) >= kMaxElems) return cudaErrorInvalidValue;
  const bool tiled = pool && kh == sh && kw == sw && ph == 0 && pw == 0 && H == P * kh && W == Q * kw &&
                     kh * kw <= 255 && !bn_tiled_off();
  if (bn_fold(M, C, chunks)) {  // the totals merge (and dgamma / dbeta) in this kernel
    if (!g_gamma || !g_beta) return cudaErrorInvalidValue;
    const size_t shm = (size_t)2 * C * 4;
    const int acc = accumulate ? 1 : 0;
    const int Mo = n * P * Q;
    if (!tiled)
      launch_pdl(bn_bwd_apply_fold_kernel<0>, dim3(fold_grid((int64_t)M * (C / 8))), dim3(256), shm, st, x, dout, y,
                 pidx, stats, (const float*)ws, chunks, g_gamma, g_beta, acc, gamma_b, G, M, Mo, dx);
    else if (kh == 2 && kw == 2)
      launch_pdl(bn_bwd_apply_fold_kernel<2>, dim3(fold_grid((int64_t)Mo * (C / 8))), dim3(256), shm, st, x, dout, y,
                 pidx, stats, (const float*)ws, chunks, g_gamma, g_beta, acc, gamma_b, G, M, Mo, dx);
    else
      launch_pdl(bn_bwd_apply_fold_kernel<1>, dim3(fold_grid((int64_t)Mo * (C / 8))), dim3(256), shm, st, x, dout, y,
                 pidx, stats, (const float*)ws, chunks, g_gamma, g_beta, acc, gamma_b, G, M, Mo, dx);
    return cudaGetLastError();
  }
  if (bn_fa(M)) {  // the totals merge (and dgamma / dbeta) and the input gradient, one block per 8 channels
    if (!g_gamma || !g_beta) return cudaErrorInvalidValue;
    const size_t shm = (size_t)2 * C * 4;
    const int acc = accumulate ? 1 : 0;
    const int Mo = n * P * Q;
    float* totw = ws_mut(ws) + (size_t)chunks * 2 * C;
    if (tiled && kh == 2 && kw == 2)
      launch_pdl(bn_bwd_final_apply_kernel<2>, dim3(C / 8), dim3(kFaThreads), shm, st, ws, chunks, totw, g_gamma,
                 g_beta, acc, x, dout, y, pidx, stats, gamma_b, G, M, Mo, dx);
    else if (tiled)
      launch_pdl(bn_bwd_final_apply_kernel<1>, dim3(C / 8), dim3(kFaThreads), shm, st, ws, chunks, totw, g_gamma,
                 g_beta, acc, x, dout, y, pidx, stats, gamma_b, G, M, Mo, dx);
    else
      launch_pdl(bn_bwd_final_apply_kernel<0>, dim3(C / 8), dim3(kFaThreads), shm, st, ws, chunks, totw, g_gamma,
                 g_beta, acc, x, dout, y, pidx, stats, gamma_b, G, M, Mo, dx);
    return cudaGetLastError();
  }
  if (pool && kh == sh && kw == sw && ph == 0 && pw == 0 && H == P * kh && W == Q * kw && kh * kw <= 255 &&
      !bn_tiled_off()) {
    const int Mo = n * P * Q;
    if (kh == 2 && kw == 2)
      launch_pdl(bn_bwd_apply_tiled_kernel<2>, dim3(grid1d((int64_t)Mo * (C / 8))), dim3(256), 0, st, x, dout, y, pidx,
                 stats, tot, gamma_b, G, M, Mo, dx);
    else
      launch_pdl(bn_bwd_apply_tiled_kernel<0>, dim3(grid1d((int64_t)Mo * (C / 8))), dim3(256), 0, st, x, dout, y, pidx,
                 stats, tot, gamma_b, G, M, Mo, dx);
    return cudaGetLastError();
  }
  if (G.pool)
    launch_pdl(bn_bwd_apply_kernel<1>, dim3(grid1d((int64_t)M * (C / 8))), dim3(256), 0, st, x, dout, y, pidx, stats,
               tot, gamma_b, G, M, dx);
  else
    launch_pdl(bn_bwd_apply_kernel<0>, dim3(grid1d((int64_t)M * (C / 8))), dim3(256), 0, st, x, dout, y, pidx, stats,
               tot, gamma_b, G, M, dx);
  return cudaGetLastError();
}

cudaError_t launch_linear_dy_prep(const void* dy, bool dy_f32, const bf16* mask, bf16* dyp, int ldp, float* gb, int n,
                                  int out, bool accumulate, cudaStream_t st) {
  if (ldp % 8 || ldp < out) return cudaErrorInvalidValue;
  if (dy_f32)
    launch_pdl(linear_dy_prep_kernel<true>, dim3((ldp + 127) / 128), dim3(128), 0, st, dy, mask, dyp, ldp, gb, n, out,
               accumulate ? 1 : 0);
  else
    launch_pdl(linear_dy_prep_kernel<false>, dim3((ldp + 127) / 128), dim3(128), 0, st, dy, mask, dyp, ldp, gb, n, out,
               accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_linear_fwd_bf16(const bf16* x, const bf16* W, const bf16* b, void* y, int n, int in, int out,
                                   bool relu, bool f32out, cudaStream_t st) {
  launch_pdl(linear_fwd_bf16_kernel, dim3((n * out + 7) / 8), dim3(256), 0, st, x, W, b, y, n, in, out, relu ? 1 : 0, f32out ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_linear_dgrad_bf16(const void* dy, bool dy_f32, const bf16* mask, const bf16* W, bf16* dx, int n,
                                     int in, int out, cudaStream_t st) {
  dim3 grid((in + 127) / 128, n);
  if (dy_f32) launch_pdl(linear_dgrad_bf16_kernel<true>, dim3(grid), dim3(128), 0, st, dy, mask, W, dx, n, in, out);
  else launch_pdl(linear_dgrad_bf16_kernel<false>, dim3(grid), dim3(128), 0, st, dy, mask, W, dx, n, in, out);
  return cudaGetLastError();
}

cudaError_t launch_linear_wgrad_bf16(const void* dy, bool dy_f32, const bf16* mask, const bf16* x, float* gW, float* gb,
                                     int n, int in, int out, bool accumulate, cudaStream_t st) {
  dim3 grid((in + 1 + 127) / 128, out);
  if (dy_f32) launch_pdl(linear_wgrad_bf16_kernel<true>, dim3(grid), dim3(128), 0, st, dy, mask, x, gW, gb, n, in, out, accumulate ? 1 : 0);
  else launch_pdl(linear_wgrad_bf16_kernel<false>, dim3(grid), dim3(128), 0, st, dy, mask, x, gW, gb, n, in, out, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace xp

// =========================================================================================
// DAG-model kernels (ResNet-101 / Inception-V3): residual add (+ReLU), channel concat,
// standalone max / average pooling and global average pooling, and the gradient side of
// each.  Activation gradients accumulate with the oracle's rounding point:
// out = Q(old + Q(g)) when a tensor already holds a contribution (fan-out), else out = Q(g).
// =========================================================================================
namespace xp {

namespace {
typedef __nv_bfloat16 bf16;
__device__ __forceinline__ float q16b(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
__device__ __forceinline__ void put_grad(bf16* p, float g, int accumulate) {
  const float gq = q16b(g);
  *p = __float2bfloat16_rn(accumulate ? __fadd_rn(__bfloat162float(*p), gq) : gq);
}
int g1(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// y = Q(relu?(a + b)) elementwise over n elements
__global__ void add_fwd_kernel(const bf16* a, const bf16* b, bf16* y, int64_t n, int relu) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float v = q16b(__fadd_rn(__bfloat162float(a[i]), __bfloat162float(b[i])));
    if (relu) v = v > 0.f ? v : 0.f;
    y[i] = __float2bfloat16_rn(v);
  }
}
// da (=|+=) dy', db (=|+=) dy' with dy' = (relu && !(y > 0)) ? 0 : dy
__global__ void add_bwd_kernel(const bf16* dy, const bf16* y, bf16* da, bf16* db, int64_t n, int relu, int acc_a,
                               int acc_b) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float g = __bfloat162float(dy[i]);
    if (relu && !(__bfloat162float(y[i]) > 0.f)) g = 0.f;
    if (da) put_grad(da + i, g, acc_a);
    if (db) put_grad(db + i, g, acc_b);
  }
}
// y[r][0:Ca] = a[r], y[r][Ca:Ca+Cb] = b[r]   (r = pixel)
__global__ void concat_fwd_kernel(const bf16* a, const bf16* b, bf16* y, int64_t rows, int Ca, int Cb) {
  pdl_wait();
  const int C = Ca + Cb;
  const int64_t n = rows * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = (int)(i - r * C);
    y[i] = c < Ca ? a[r * Ca + c] : b[r * Cb + (c - Ca)];
  }
}
__global__ void concat_bwd_kernel(const bf16* dy, bf16* da, bf16* db, int64_t rows, int Ca, int Cb, int acc_a,
                                  int acc_b) {
  pdl_wait();
  const int C = Ca + Cb;
  const int64_t n = rows * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C;
    const int c = (int)(i - r * C);
    const float g = __bfloat162float(dy[i]);
    if (c < Ca) { if (da) put_grad(da + r * Ca + c, g, acc_a); }
    else if (db) put_grad(db + r * Cb + (c - Ca), g, acc_b);
  }
}
// pooling forward: mode 0 max (first max, padded positions skipped), 1 avg (count_include_pad)
__global__ void pool_fwd_kernel(const bf16* x, bf16* y, int n, int H, int W, int C, int P, int Q, int kh, int kw,
                                int sh, int sw, int ph, int pw, int mode, int ldy) {
  pdl_wait();
  const int64_t total = (int64_t)n * P * Q * C;
  const float inv = 1.f / (float)(kh * kw);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t r = i / C;
    const int q = (int)(r % Q); r /= Q;
    const int p = (int)(r % P);
    const int s = (int)(r / P);
    float best = 0.f, acc = 0.f;
    bool first = true;
    for (int a = 0; a < kh; ++a)
      for (int b = 0; b < kw; ++b) {
        const int hh = p * sh - ph + a, ww = q * sw - pw + b;
        if (hh < 0 || hh >= H || ww < 0 || ww >= W) continue;
        const float v = __bfloat162float(x[(((int64_t)s * H + hh) * W + ww) * C + c]);
        if (mode == 0) { if (first || v > best) best = v; first = false; }
        else acc = __fadd_rn(acc, v);
      }
    y[(((int64_t)s * P + p) * Q + q) * ldy + c] = __float2bfloat16_rn(mode == 0 ? best : __fmul_rn(acc, inv));
  }
}
// pooling backward, gather form over the input: for each input element sum the gradients of
// the windows that route to it (max: it is the window's first max; avg: every window
// covering it contributes g*inv), then store/accumulate
__global__ void pool_bwd_kernel(const bf16* x, const bf16* dy, bf16* dx, int n, int H, int W, int C, int P, int Q,
                                int kh, int kw, int sh, int sw, int ph, int pw, int mode, int accumulate, int ldy) {
  pdl_wait();
  const int64_t total = (int64_t)n * H * W * C;
  const float inv = 1.f / (float)(kh * kw);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t r = i / C;
    const int w = (int)(r % W); r /= W;
    const int h = (int)(r % H);
    const int s = (int)(r / H);
    const int plo = max(0, (h + ph - kh + sh) / sh), phi = min(P - 1, (h + ph) / sh);
    const int qlo = max(0, (w + pw - kw + sw) / sw), qhi = min(Q - 1, (w + pw) / sw);
    float acc = 0.f;
    int hits = 0;
    for (int p = plo; p <= phi; ++p)
      for (int q = qlo; q <= qhi; ++q) {
        if (h < p * sh - ph || h >= p * sh - ph + kh || w < q * sw - pw || w >= q * sw - pw + kw) continue;
        const float g = __bfloat162float(dy[(((int64_t)s * P + p) * Q + q) * ldy + c]);
        if (mode == 0) {
          float best = 0.f;
          int bh = -1, bw = -1;
          for (int a = 0; a < kh; ++a)
            for (int b = 0; b < kw; ++b) {
              const int hh = p * sh - ph + a, ww = q * sw - pw + b;
              if (hh < 0 || hh >= H || ww < 0 || ww >= W) continue;
              const float v = __bfloat162float(x[(((int64_t)s * H + hh) * W + ww) * C + c]);
              if (bh < 0 || v > best) { best = v; bh = hh; bw = ww; }
            }
          if (bh != h || bw != w) continue;
          acc = hits ? __fadd_rn(acc, g) : g;
        } else {
          const float gi = __fmul_rn(g, inv);
          acc = hits ? __fadd_rn(acc, gi) : gi;
        }
        ++hits;
      }
    put_grad(dx + i, acc, accumulate);
  }
}
// The two pooling kernels above, 8 channels per thread (16-byte loads / stores, 32-bit index
// arithmetic; C % 8 == 0, row pitches % 8 == 0): per element the same window scan, the same
// first-max rule and the same sums in the same order, so the results are bit-identical
__device__ __forceinline__ void unpack8(const uint4& u, float (&v)[8]) {
  const bf16* b = reinterpret_cast<const bf16*>(&u);
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = __bfloat162float(b[e]);
}
__device__ __forceinline__ uint4 pack8(const float (&v)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    __nv_bfloat162 t = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
    w[h] = *reinterpret_cast<uint32_t*>(&t);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__global__ void pool_fwd8_kernel(const bf16* __restrict__ x, bf16* __restrict__ y, int n, int H, int W, int C, int P,
                                 int Q, int kh, int kw, int sh, int sw, int ph, int pw, int mode, int ldy) {
  pdl_wait();
  const int G = C / 8, total = n * P * Q * G;
  const float inv = 1.f / (float)(kh * kw);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % G;
    int r = i / G;
    const int q = r % Q; r /= Q;
    const int p = r % P;
    const int s = r / P;
    float best[8], acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { best[e] = 0.f; acc[e] = 0.f; }
    bool first = true;
    for (int a = 0; a < kh; ++a)
      for (int b = 0; b < kw; ++b) {
        const int hh = p * sh - ph + a, ww = q * sw - pw + b;
        if (hh < 0 || hh >= H || ww < 0 || ww >= W) continue;
        float v[8];
        unpack8(*reinterpret_cast<const uint4*>(x + ((s * H + hh) * W + ww) * C + g * 8), v);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (mode == 0) { if (first || v[e] > best[e]) best[e] = v[e]; }
          else acc[e] = __fadd_rn(acc[e], v[e]);
        }
        first = false;
      }
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = mode == 0 ? best[e] : __fmul_rn(acc[e], inv);
    *reinterpret_cast<uint4*>(y + ((s * P + p) * Q + q) * ldy + g * 8) = pack8(o);
  }
}
__global__ void pool_bwd8_kernel(const bf16* __restrict__ x, const bf16* __restrict__ dy, bf16* __restrict__ dx,
                                 int n, int H, int W, int C, int P, int Q, int kh, int kw, int sh, int sw, int ph,
                                 int pw, int mode, int accumulate, int ldy) {
  pdl_wait();
  const int G = C / 8, total = n * H * W * G;
  const float inv = 1.f / (float)(kh * kw);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i % G;
    int r = i / G;
    const int w = r % W; r /= W;
    const int h = r % H;
    const int s = r / H;
    const int plo = max(0, (h + ph - kh + sh) / sh), phi = min(P - 1, (h + ph) / sh);
    const int qlo = max(0, (w + pw - kw + sw) / sw), qhi = min(Q - 1, (w + pw) / sw);
    float acc[8];
    int hits[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { acc[e] = 0.f; hits[e] = 0; }
    for (int p = plo; p <= phi; ++p)
      for (int q = qlo; q <= qhi; ++q) {
        if (h < p * sh - ph || h >= p * sh - ph + kh || w < q * sw - pw || w >= q * sw - pw + kw) continue;
        float gv[8];
        unpack8(*reinterpret_cast<const uint4*>(dy + ((s * P + p) * Q + q) * ldy + g * 8), gv);
        if (mode == 0) {
          float best[8];
          int bpos[8];  // the window's first max, as h * W + w (-1: none yet)
#pragma unroll
          for (int e = 0; e < 8; ++e) { best[e] = 0.f; bpos[e] = -1; }
          for (int a = 0; a < kh; ++a)
            for (int b = 0; b < kw; ++b) {
              const int hh = p * sh - ph + a, ww = q * sw - pw + b;
              if (hh < 0 || hh >= H || ww < 0 || ww >= W) continue;
              float v[8];
              unpack8(*reinterpret_cast<const uint4*>(x + ((s * H + hh) * W + ww) * C + g * 8), v);
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (bpos[e] < 0 || v[e] > best[e]) { best[e] = v[e]; bpos[e] = hh * W + ww; }
            }
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (bpos[e] == h * W + w) { acc[e] = hits[e] ? __fadd_rn(acc[e], gv[e]) : gv[e]; ++hits[e]; }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float gi = __fmul_rn(gv[e], inv);
            acc[e] = hits[e] ? __fadd_rn(acc[e], gi) : gi;
            ++hits[e];
          }
        }
      }
    bf16* d = dx + (int64_t)i * 8;
    float o[8];
    if (accumulate) {
      float old[8];
      unpack8(*reinterpret_cast<const uint4*>(d), old);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(old[e], q16b(acc[e]));
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = q16b(acc[e]);
    }
    *reinterpret_cast<uint4*>(d) = pack8(o);
  }
}
// global average pool: y[s][c] = (sum over H*W in raster order) * (1/(H*W))
__global__ void gap_fwd_kernel(const bf16* x, bf16* y, int n, int HW, int C) {
  pdl_wait();
  const int64_t total = (int64_t)n * C;
  const float inv = 1.f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t s = i / C;
    float acc = 0.f;
    for (int k = 0; k < HW; ++k) acc = __fadd_rn(acc, __bfloat162float(x[(s * HW + k) * C + c]));
    y[i] = __float2bfloat16_rn(__fmul_rn(acc, inv));
  }
}
__global__ void gap_bwd_kernel(const bf16* dy, bf16* dx, int n, int HW, int C, int accumulate) {
  pdl_wait();
  const int64_t total = (int64_t)n * HW * C;
  const float inv = 1.f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t s = i / ((int64_t)HW * C);
    put_grad(dx + i, __fmul_rn(__bfloat162float(dy[s * C + c]), inv), accumulate);
  }
}
}  // namespace

cudaError_t launch_add_fwd(const bf16* a, const bf16* b, bf16* y, int64_t n, bool relu, cudaStream_t st) {
  launch_pdl(add_fwd_kernel, dim3(g1(n)), dim3(256), 0, st, a, b, y, n, relu ? 1 : 0);
  return cudaGetLastError();
}
cudaError_t launch_add_bwd(const bf16* dy, const bf16* y, bf16* da, bf16* db, int64_t n, bool relu, bool acc_a,
                           bool acc_b, cudaStream_t st) {
  launch_pdl(add_bwd_kernel, dim3(g1(n)), dim3(256), 0, st, dy, y, da, db, n, relu ? 1 : 0, acc_a ? 1 : 0, acc_b ? 1 : 0);
  return cudaGetLastError();
}
cudaError_t launch_concat_fwd(const bf16* a, const bf16* b, bf16* y, int64_t rows, int Ca, int Cb, cudaStream_t st) {
  launch_pdl(concat_fwd_kernel, dim3(g1(rows * (Ca + Cb))), dim3(256), 0, st, a, b, y, rows, Ca, Cb);
  return cudaGetLastError();
}
cudaError_t launch_concat_bwd(const bf16* dy, bf16* da, bf16* db, int64_t rows, int Ca, int Cb, bool acc_a, bool acc_b,
                              cudaStream_t st) {
  launch_pdl(concat_bwd_kernel, dim3(g1(rows * (Ca + Cb))), dim3(256), 0, st, dy, da, db, rows, Ca, Cb, acc_a ? 1 : 0, acc_b ? 1 : 0);
  return cudaGetLastError();
}
bool pool_vec_off() { static const bool v = getenv("XPIPE_NO_POOL_VEC") != nullptr; return v; }
cudaError_t launch_pool_fwd(const bf16* x, bf16* y, int n, int H, int W, int C, int P, int Q, int kh, int kw, int sh,
                            int sw, int ph, int pw, bool avg, cudaStream_t st, int ldy) {
  if (!ldy) ldy = C;
  if (C % 8 == 0 && ldy % 8 == 0 && (int64_t)n * std::max(H * W, P * Q) * C < kMaxElems && !pool_vec_off()) {
    launch_pdl(pool_fwd8_kernel, dim3(g1((int64_t)n * P * Q * C / 8)), dim3(256), 0, st, x, y, n, H, W, C, P, Q, kh,
               kw, sh, sw, ph, pw, avg ? 1 : 0, ldy);
    return cudaGetLastError();
  }
  launch_pdl(pool_fwd_kernel, dim3(g1((int64_t)n * P * Q * C)), dim3(256), 0, st, x, y, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw,
             avg ? 1 : 0, ldy ? ldy : C);
  return cudaGetLastError();
}
cudaError_t launch_pool_bwd(const bf16* x, const bf16* dy, bf16* dx, int n, int H, int W, int C, int P, int Q, int kh,
                            int kw, int sh, int sw, int ph, int pw, bool avg, bool accumulate, cudaStream_t st, int ldy) {
  if (!ldy) ldy = C;
  if (C % 8 == 0 && ldy % 8 == 0 && (int64_t)n * std::max(H * W, P * Q) * C < kMaxElems && !pool_vec_off()) {
    launch_pdl(pool_bwd8_kernel, dim3(g1((int64_t)n * H * W * C / 8)), dim3(256), 0, st, x, dy, dx, n, H, W, C, P, Q,
               kh, kw, sh, sw, ph, pw, avg ? 1 : 0, accumulate ? 1 : 0, ldy);
    return cudaGetLastError();
  }
  launch_pdl(pool_bwd_kernel, dim3(g1((int64_t)n * H * W * C)), dim3(256), 0, st, x, dy, dx, n, H, W, C, P, Q, kh, kw, sh, sw, ph, pw,
                                                              avg ? 1 : 0, accumulate ? 1 : 0, ldy ? ldy : C);
  return cudaGetLastError();
}
cudaError_t launch_gap_fwd(const bf16* x, bf16* y, int n, int HW, int C, cudaStream_t st) {
  launch_pdl(gap_fwd_kernel, dim3(g1((int64_t)n * C)), dim3(256), 0, st, x, y, n, HW, C);
  return cudaGetLastError();
}
cudaError_t launch_gap_bwd(const bf16* dy, bf16* dx, int n, int HW, int C, bool accumulate, cudaStream_t st) {
  launch_pdl(gap_bwd_kernel, dim3(g1((int64_t)n * HW * C)), dim3(256), 0, st, dy, dx, n, HW, C, accumulate ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace xp
