/*
 * xoracle.cpp -- plain, slow, obviously-correct CPU oracle of the XPipe hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs; never by the product path.  Shares no code with
 * the CUDA product.  Built with -O3 -march=native -fopenmp -ffp-contract=off (no -ffast-math;
 * oracle/__init__.py) so every float operation written here is one IEEE operation: vector code
 * only evaluates the written operations lane by lane, and no multiply-add is contracted except
 * the explicit std::fmaf calls of the fp32 contract.
 *
 * Every function cites the passage it follows (P:n = /root/reference/PAPER.md line n;
 * "R<n>" = DESIGN.md reading n; "fp32 contract" = DESIGN.md section 4).
 *
 * Layout: NCHW activations, PyTorch parameter layouts ([out][in] Linear, [out][in][kh][kw]
 * Conv2d), parameters of a stage flattened in layer order (weight, then bias).
 *
 * Parity pins: tests/test_oracle_*.py.  Parity unpinned: the multi-stage trajectory with
 * s > 0 at K > 1 has no external reference.
 */
#include "xoracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;
int fail(int code, const std::string& m) { g_err = m; return code; }
enum { E_OK = 0, E_INVAL = -1, E_SCHED = -5, E_UNSUP = -8 };

typedef std::vector<double> Vec;

/* bf16 round-to-nearest-even of a float */
double q_bf16(double xd) {
  float x = (float)xd;
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) {          /* inf / nan: truncate, keep nan quiet */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
  }
  std::memcpy(&x, &u, 4);
  return (double)x;
}

struct Shape {
  int c = 0, h = 0, w = 0;
  size_t size() const { return (size_t)c * h * w; }
};

struct Layer {
  xo_layer d;
  int src0 = -1, src1 = -1;    /* resolved producer indices; -1 = network input */
  Shape in0, in1, out;
  int stage = 0;
  size_t nw = 0, nb = 0;       /* parameter counts (weight, bias) */
  size_t woff = 0, boff = 0;   /* offsets inside the stage's flat parameter vector */
};

struct Model {
  int mode = XO_FP64;
  std::vector<Layer> L;
  Shape input;
  int classes = 0;
  bool is_logits(int i) const {   /* output of layer i feeds the softmax-xent: stays fp32 */
    return i + 1 < (int)L.size() && L[i + 1].d.kind == XO_SOFTMAX_XENT;
  }
  double qa(double v, int i) const {  /* rounding point of a stored activation */
    if (mode == XO_BF16 && !is_logits(i)) return q_bf16(v);
    if (mode != XO_FP64) return (double)(float)v;
    return v;
  }
  double qg(double v) const {         /* rounding point of an activation gradient */
    if (mode == XO_BF16) return q_bf16(v);
    if (mode != XO_FP64) return (double)(float)v;
    return v;
  }
  double add(double a, double b) const {   /* one addition in the mode's arithmetic */
    if (mode == XO_FP64) return a + b;
    return (double)((float)a + (float)b);
  }
};

/* ------------------------------------------------------------------------------------ */
/* Layer maths (plain definitions).  n = samples in this micro-batch.      */
/* ------------------------------------------------------------------------------------ */

/* y = x W^T + b.  fp32 contract: y[r][o] = (sum_i fmaf(x,W,acc) from 0, i ascending) + b[o] */
void linear_fwd(const Model& M, int li, int n, const Vec& x, const double* W, const double* b, Vec& y) {
  const Layer& l = M.L[li];
  int in = l.d.in_c, out = l.d.out_c;
  y.assign((size_t)n * out, 0.0);
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < n; ++r)
    for (int o = 0; o < out; ++o) {
      double v;
      if (M.mode == XO_FP32) {
        float acc = 0.f;
        for (int i = 0; i < in; ++i) acc = std::fmaf((float)x[(size_t)r * in + i], (float)W[(size_t)o * in + i], acc);
        v = l.d.bias ? (double)(acc + (float)b[o]) : (double)acc;
      } else if (M.mode == XO_BF16) {
        double acc = 0.0;
        for (int i = 0; i < in; ++i) acc += x[(size_t)r * in + i] * W[(size_t)o * in + i];
        v = l.d.bias ? (double)((float)acc + (float)b[o]) : (double)(float)acc;
      } else {
        double acc = 0.0;
        for (int i = 0; i < in; ++i) acc += x[(size_t)r * in + i] * W[(size_t)o * in + i];
        v = l.d.bias ? acc + b[o] : acc;
      }
      y[(size_t)r * out + o] = M.qa(v, li);
    }
}

/* dx = dy W (o ascending), dW = dy^T x (r ascending), db = sum_r dy (r ascending) */
void linear_bwd(const Model& M, int li, int n, const Vec& x, const Vec& dy, const double* W,
                Vec& dx, double* dW, double* db, bool need_dx) {
  const Layer& l = M.L[li];
  int in = l.d.in_c, out = l.d.out_c;
  if (need_dx) {
    dx.assign((size_t)n * in, 0.0);
#pragma omp parallel for collapse(2) schedule(static)
    for (int r = 0; r < n; ++r)
      for (int i = 0; i < in; ++i) {
        double v;
        if (M.mode == XO_FP32) {
          float acc = 0.f;
          for (int o = 0; o < out; ++o) acc = std::fmaf((float)dy[(size_t)r * out + o], (float)W[(size_t)o * in + i], acc);
          v = acc;
        } else {
          double acc = 0.0;
          for (int o = 0; o < out; ++o) acc += dy[(size_t)r * out + o] * W[(size_t)o * in + i];
          v = (M.mode == XO_BF16) ? (double)(float)acc : acc;
        }
        dx[(size_t)r * in + i] = M.qg(v);
      }
  }
#pragma omp parallel for collapse(2) schedule(static)
  for (int o = 0; o < out; ++o)
    for (int i = 0; i < in; ++i) {
      if (M.mode == XO_FP32) {
        float acc = 0.f;
        for (int r = 0; r < n; ++r) acc = std::fmaf((float)dy[(size_t)r * out + o], (float)x[(size_t)r * in + i], acc);
        dW[(size_t)o * in + i] = acc;
      } else {
        double acc = 0.0;
        for (int r = 0; r < n; ++r) acc += dy[(size_t)r * out + o] * x[(size_t)r * in + i];
        dW[(size_t)o * in + i] = (M.mode == XO_BF16) ? (double)(float)acc : acc;
      }
    }
  if (l.d.bias)
    for (int o = 0; o < out; ++o) {
      if (M.mode == XO_FP32) {
        float acc = 0.f;
        for (int r = 0; r < n; ++r) acc = acc + (float)dy[(size_t)r * out + o];
        db[o] = acc;
      } else {
        double acc = 0.0;
        for (int r = 0; r < n; ++r) acc += dy[(size_t)r * out + o];
        db[o] = (M.mode == XO_BF16) ? (double)(float)acc : acc;
      }
    }
}

/* output columns q whose input column q*sw - pw + s lies inside [0, W) */
void valid_range(int sw, int pw, int s, int W, int Q, int& qlo, int& qhi) {
  qlo = 0;
  while (qlo < Q && qlo * sw - pw + s < 0) ++qlo;
  qhi = Q;
  while (qhi > qlo && (qhi - 1) * sw - pw + s >= W) --qhi;
}

/* Loop blocking of the conv sums below: a task owns a block of kPix output (or input) pixels x
   kChan channels and keeps their independent sums in a small array; each sum still runs over
   its terms one at a time in the order its comment states.  Blocking only decides which sums
   advance together (weights and inputs are reused from cache); no sum is split or reordered. */
constexpr int kPix = 32, kChan = 64, kOut = 8;

/* Conv2d: cross-correlation with zero padding (PyTorch semantics), NCHW.
   y[n][co][p][q] = sum_{ci,r,s} x[n][ci][p*sh-ph+r][q*sw-pw+s] * W[co][ci][r][s] (+ b)
   Every output is one sequential sum in (ci, r, s) order over its in-range taps (taps that
   fall into the zero padding are skipped); weights are read from a copy laid out
   [ci][r][s][co]. */
void conv_fwd(const Model& M, int li, int n, const Vec& x, const double* W, const double* b, Vec& y) {
  const Layer& l = M.L[li];
  const int C = l.in0.c, H = l.in0.h, Wd = l.in0.w, K = l.d.out_c, R = l.d.kh, S = l.d.kw;
  const int P = l.out.h, Q = l.out.w;
  const bool f32 = M.mode == XO_FP32;
  Vec Wt((size_t)C * R * S * K);
  std::vector<float> Wtf(f32 ? Wt.size() : 0);
  for (int co = 0; co < K; ++co)
    for (int ci = 0; ci < C; ++ci)
      for (int rs = 0; rs < R * S; ++rs) {
        const double w = W[((size_t)co * C + ci) * R * S + rs];
        Wt[((size_t)ci * R * S + rs) * K + co] = w;
        if (f32) Wtf[((size_t)ci * R * S + rs) * K + co] = (float)w;
      }
  y.assign((size_t)n * K * P * Q, 0.0);
  const int64_t npix = (int64_t)n * P * Q;
  const int64_t pblocks = (npix + kPix - 1) / kPix, cblocks = (K + kChan - 1) / kChan;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t task = 0; task < pblocks * cblocks; ++task) {
    const int64_t px0 = (task / cblocks) * kPix;
    const int c0 = (int)(task % cblocks) * kChan;
    const int np = (int)std::min<int64_t>(kPix, npix - px0), nc = std::min(kChan, K - c0);
    double acc[kPix][kChan] = {};
    float accf[kPix][kChan] = {};
    int s0v[kPix], pv[kPix], qv[kPix];
    for (int i = 0; i < np; ++i) {
      const int64_t px = px0 + i;
      s0v[i] = (int)(px / ((int64_t)P * Q));
      pv[i] = (int)(px / Q % P);
      qv[i] = (int)(px % Q);
    }
    for (int ci = 0; ci < C; ++ci)
      for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
          const size_t wo = (((size_t)ci * R + r) * S + s) * K + c0;
          for (int i = 0; i < np; ++i) {
            const int ih = pv[i] * l.d.sh - l.d.ph + r, iw = qv[i] * l.d.sw - l.d.pw + s;
            if (ih < 0 || ih >= H || iw < 0 || iw >= Wd) continue;
            const double xv = x[(((size_t)s0v[i] * C + ci) * H + ih) * Wd + iw];
            if (f32) {
              const float xf = (float)xv;
              const float* w = &Wtf[wo];
              float* a = accf[i];
              for (int co = 0; co < nc; ++co) a[co] = std::fmaf(xf, w[co], a[co]);
            } else {
              const double* w = &Wt[wo];
              double* a = acc[i];
              for (int co = 0; co < nc; ++co) a[co] += xv * w[co];
            }
          }
        }
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < nc; ++j) {
        const int co = c0 + j;
        double v = f32 ? (double)accf[i][j] : acc[i][j];
        if (M.mode == XO_BF16) v = (double)(float)v;
        if (l.d.bias) v = (M.mode == XO_FP64) ? v + b[co] : (double)((float)v + (float)b[co]);
        y[(((size_t)s0v[i] * K + co) * P + pv[i]) * Q + qv[i]] = M.qa(v, li);
      }
  }
}

void conv_bwd(const Model& M, int li, int n, const Vec& x, const Vec& dy, const double* W,
              Vec& dx, double* dW, double* db, bool need_dx) {
  const Layer& l = M.L[li];
  const int C = l.in0.c, H = l.in0.h, Wd = l.in0.w, K = l.d.out_c, R = l.d.kh, S = l.d.kw;
  const int P = l.out.h, Q = l.out.w;
  const bool f32 = M.mode == XO_FP32;
  if (need_dx) {
    /* dx[n][ci][ih][iw] = sum_{co,r,s : ih = p*sh-ph+r, iw = q*sw-pw+s} dy[n][co][p][q] W[co][ci][r][s]:
       one sequential sum per input element in (co, r, s) order over the taps that map it to an
       output pixel; weights read from a copy laid out [co][r][s][ci] */
    Vec Wk((size_t)K * R * S * C);
    std::vector<float> Wkf(f32 ? Wk.size() : 0);
    for (int co = 0; co < K; ++co)
      for (int ci = 0; ci < C; ++ci)
        for (int rs = 0; rs < R * S; ++rs) {
          const double w = W[((size_t)co * C + ci) * R * S + rs];
          Wk[((size_t)co * R * S + rs) * C + ci] = w;
          if (f32) Wkf[((size_t)co * R * S + rs) * C + ci] = (float)w;
        }
    dx.assign((size_t)n * C * H * Wd, 0.0);
    const int64_t npix = (int64_t)n * H * Wd;
    const int64_t pblocks = (npix + kPix - 1) / kPix, cblocks = (C + kChan - 1) / kChan;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t task = 0; task < pblocks * cblocks; ++task) {
      const int64_t px0 = (task / cblocks) * kPix;
      const int c0 = (int)(task % cblocks) * kChan;
      const int np = (int)std::min<int64_t>(kPix, npix - px0), nc = std::min(kChan, C - c0);
      double acc[kPix][kChan] = {};
      float accf[kPix][kChan] = {};
      int s0v[kPix], hv[kPix], wv[kPix];
      for (int i = 0; i < np; ++i) {
        const int64_t px = px0 + i;
        s0v[i] = (int)(px / ((int64_t)H * Wd));
        hv[i] = (int)(px / Wd % H);
        wv[i] = (int)(px % Wd);
      }
      for (int co = 0; co < K; ++co)
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s) {
            const size_t wo = (((size_t)co * R + r) * S + s) * C + c0;
            for (int i = 0; i < np; ++i) {
              const int ph_ = hv[i] + l.d.ph - r, qw_ = wv[i] + l.d.pw - s;   /* = p * sh, q * sw */
              if (ph_ < 0 || qw_ < 0 || ph_ % l.d.sh || qw_ % l.d.sw) continue;
              const int p = ph_ / l.d.sh, q = qw_ / l.d.sw;
              if (p >= P || q >= Q) continue;
              const double d = dy[(((size_t)s0v[i] * K + co) * P + p) * Q + q];
              if (f32) {
                const float df = (float)d;
                const float* w = &Wkf[wo];
                float* a = accf[i];
                for (int j = 0; j < nc; ++j) a[j] = std::fmaf(df, w[j], a[j]);
              } else {
                const double* w = &Wk[wo];
                double* a = acc[i];
                for (int j = 0; j < nc; ++j) a[j] += d * w[j];
              }
            }
          }
      for (int i = 0; i < np; ++i)
        for (int j = 0; j < nc; ++j) {
          double v = f32 ? (double)accf[i][j] : acc[i][j];
          if (M.mode == XO_BF16) v = (double)(float)v;
          dx[(((size_t)s0v[i] * C + c0 + j) * H + hv[i]) * Wd + wv[i]] = M.qg(v);
        }
    }
  }
  /* dW[co][ci][r][s] = sum_{n,p,q} dy[n][co][p][q] x[n][ci][p*sh-ph+r][q*sw-pw+s]; every dW
     element is one sequential sum in (n, p, q) order over its in-range taps; the input is read
     from a copy laid out [n][h][w][ci] */
  Vec xt((size_t)n * H * Wd * C);
  for (int s0 = 0; s0 < n; ++s0)
    for (int ci = 0; ci < C; ++ci)
      for (int hw = 0; hw < H * Wd; ++hw)
        xt[((size_t)s0 * H * Wd + hw) * C + ci] = x[((size_t)s0 * C + ci) * H * Wd + hw];
  const int oblocks = (K + kOut - 1) / kOut, cblocks = (C + kChan - 1) / kChan;
#pragma omp parallel for schedule(dynamic, 1)
  for (int task = 0; task < oblocks * cblocks; ++task) {
    const int o0 = (task / cblocks) * kOut, c0 = (task % cblocks) * kChan;
    const int no = std::min(kOut, K - o0), nc = std::min(kChan, C - c0);
    Vec acc((size_t)kOut * R * S * kChan, 0.0);
    std::vector<float> accf((size_t)kOut * R * S * kChan, 0.f);
    for (int s0 = 0; s0 < n; ++s0)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q)
          for (int r = 0; r < R; ++r) {
            const int ih = p * l.d.sh - l.d.ph + r;
            if (ih < 0 || ih >= H) continue;
            for (int s = 0; s < S; ++s) {
              const int iw = q * l.d.sw - l.d.pw + s;
              if (iw < 0 || iw >= Wd) continue;
              const double* xr = &xt[(((size_t)s0 * H + ih) * Wd + iw) * C + c0];
              for (int oi = 0; oi < no; ++oi) {
                const double a = dy[(((size_t)s0 * K + o0 + oi) * P + p) * Q + q];
                const size_t ao = (((size_t)oi * R + r) * S + s) * kChan;
                if (f32) {
                  const float af = (float)a;
                  float* ac = &accf[ao];
                  for (int j = 0; j < nc; ++j) ac[j] = std::fmaf(af, (float)xr[j], ac[j]);
                } else {
                  double* ac = &acc[ao];
                  for (int j = 0; j < nc; ++j) ac[j] += a * xr[j];
                }
              }
            }
          }
    for (int oi = 0; oi < no; ++oi)
      for (int j = 0; j < nc; ++j)
        for (int rs = 0; rs < R * S; ++rs) {
          const size_t ai = ((size_t)oi * R * S + rs) * kChan + j;
          double v = f32 ? (double)accf[ai] : acc[ai];
          if (M.mode == XO_BF16) v = (double)(float)v;
          dW[((size_t)(o0 + oi) * C + c0 + j) * R * S + rs] = v;
        }
  }
  if (l.d.bias)
    for (int co = 0; co < K; ++co) {
      double acc = 0.0;
      float accf = 0.f;
      for (int s0 = 0; s0 < n; ++s0)
        for (int pq = 0; pq < P * Q; ++pq) {
          double a = dy[((size_t)s0 * K + co) * P * Q + pq];
          if (M.mode == XO_FP32) accf = accf + (float)a; else acc += a;
        }
      double v = (M.mode == XO_FP32) ? (double)accf : acc;
      if (M.mode == XO_BF16) v = (double)(float)v;
      db[co] = v;
    }
}

/* BatchNorm2d, training mode (R11): per-channel statistics over the micro-batch's n*H*W
   values; biased two-pass variance; y = gamma (x-mean) rstd + beta, rstd = 1/sqrt(var+eps) */
void bn_stats(const Model& M, const Layer& l, int n, const Vec& x, int c, double& mean, double& rstd) {
  const int C = l.in0.c;
  const size_t HW = (size_t)l.in0.h * l.in0.w;
  const double cnt = (double)n * HW;
  if (M.mode == XO_FP32) {
    float s = 0.f;
    for (int s0 = 0; s0 < n; ++s0) for (size_t i = 0; i < HW; ++i) s = s + (float)x[((size_t)s0 * C + c) * HW + i];
    float mu = s / (float)cnt;
    float v = 0.f;
    for (int s0 = 0; s0 < n; ++s0) for (size_t i = 0; i < HW; ++i) {
      float d = (float)x[((size_t)s0 * C + c) * HW + i] - mu;
      v = v + d * d;
    }
    float var = v / (float)cnt;
    mean = mu;
    rstd = 1.0f / std::sqrt(var + l.d.bn_eps);
  } else {
    double s = 0.0;
    for (int s0 = 0; s0 < n; ++s0) for (size_t i = 0; i < HW; ++i) s += x[((size_t)s0 * C + c) * HW + i];
    double mu = s / cnt, v = 0.0;
    for (int s0 = 0; s0 < n; ++s0) for (size_t i = 0; i < HW; ++i) {
      double d = x[((size_t)s0 * C + c) * HW + i] - mu;
      v += d * d;
    }
    mean = mu;
    rstd = 1.0 / std::sqrt(v / cnt + (double)l.d.bn_eps);
  }
}

void bn_fwd(const Model& M, int li, int n, const Vec& x, const double* gamma, const double* beta, Vec& y) {
  const Layer& l = M.L[li];
  const int C = l.in0.c;
  const size_t HW = (size_t)l.in0.h * l.in0.w;
  y.assign(x.size(), 0.0);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    double mean, rstd;
    bn_stats(M, l, n, x, c, mean, rstd);
    for (int s0 = 0; s0 < n; ++s0)
      for (size_t i = 0; i < HW; ++i) {
        size_t idx = ((size_t)s0 * C + c) * HW + i;
        double v;
        if (M.mode == XO_FP32) v = (float)gamma[c] * (((float)x[idx] - (float)mean) * (float)rstd) + (float)beta[c];
        else v = gamma[c] * ((x[idx] - mean) * rstd) + beta[c];
        y[idx] = M.qa(v, li);
      }
  }
}

/* dx = gamma rstd (dy - sum(dy)/cnt - xhat sum(dy xhat)/cnt); dgamma = sum dy xhat; dbeta = sum dy */
void bn_bwd(const Model& M, int li, int n, const Vec& x, const Vec& dy, const double* gamma,
            Vec& dx, double* dgamma, double* dbeta) {
  const Layer& l = M.L[li];
  const int C = l.in0.c;
  const size_t HW = (size_t)l.in0.h * l.in0.w;
  const double cnt = (double)n * HW;
  dx.assign(x.size(), 0.0);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    double mean, rstd;
    bn_stats(M, l, n, x, c, mean, rstd);
    double sdy = 0.0, sdyx = 0.0;
    float sdyf = 0.f, sdyxf = 0.f;
    for (int s0 = 0; s0 < n; ++s0)
      for (size_t i = 0; i < HW; ++i) {
        size_t idx = ((size_t)s0 * C + c) * HW + i;
        if (M.mode == XO_FP32) {
          float xh = ((float)x[idx] - (float)mean) * (float)rstd;
          sdyf = sdyf + (float)dy[idx];
          sdyxf = sdyxf + (float)dy[idx] * xh;
        } else {
          double xh = (x[idx] - mean) * rstd;
          sdy += dy[idx];
          sdyx += dy[idx] * xh;
        }
      }
    if (M.mode == XO_FP32) { sdy = sdyf; sdyx = sdyxf; }
    dbeta[c] = (M.mode == XO_FP64) ? sdy : (double)(float)sdy;
    dgamma[c] = (M.mode == XO_FP64) ? sdyx : (double)(float)sdyx;
    for (int s0 = 0; s0 < n; ++s0)
      for (size_t i = 0; i < HW; ++i) {
        size_t idx = ((size_t)s0 * C + c) * HW + i;
        double v;
        if (M.mode == XO_FP32) {
          float xh = ((float)x[idx] - (float)mean) * (float)rstd;
          v = ((float)gamma[c] * (float)rstd) * (((float)dy[idx] - (float)sdy / (float)cnt) - xh * ((float)sdyx / (float)cnt));
        } else {
          double xh = (x[idx] - mean) * rstd;
          v = gamma[c] * rstd * (dy[idx] - sdy / cnt - xh * sdyx / cnt);
        }
        dx[idx] = M.qg(v);
      }
  }
}

/* MaxPool2d: the first maximum in the row-major window scan wins ties (R: DESIGN 4);
   padded positions never win. */
void maxpool_fwd(const Model& M, int li, int n, const Vec& x, Vec& y, std::vector<int64_t>* arg) {
  const Layer& l = M.L[li];
  const int C = l.in0.c, H = l.in0.h, Wd = l.in0.w, P = l.out.h, Q = l.out.w;
  y.assign((size_t)n * C * P * Q, 0.0);
  if (arg) arg->assign(y.size(), -1);
  for (int s0 = 0; s0 < n; ++s0)
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          double best = -INFINITY;
          int64_t bi = -1;
          for (int r = 0; r < l.d.kh; ++r)
            for (int s = 0; s < l.d.kw; ++s) {
              int ih = p * l.d.sh - l.d.ph + r, iw = q * l.d.sw - l.d.pw + s;
              if (ih < 0 || ih >= H || iw < 0 || iw >= Wd) continue;
              int64_t idx = (((int64_t)s0 * C + c) * H + ih) * Wd + iw;
              if (bi < 0 || x[idx] > best) { best = x[idx]; bi = idx; }
            }
          size_t o = (((size_t)s0 * C + c) * P + p) * Q + q;
          y[o] = best;
          if (arg) (*arg)[o] = bi;
        }
}

void maxpool_bwd(const Model& M, int li, int n, const Vec& x, const Vec& dy, Vec& dx) {
  Vec y;
  std::vector<int64_t> arg;
  maxpool_fwd(M, li, n, x, y, &arg);
  dx.assign(x.size(), 0.0);
  for (size_t o = 0; o < dy.size(); ++o) dx[arg[o]] = M.add(dx[arg[o]], dy[o]);
  for (auto& v : dx) v = M.qg(v);
}

/* global average pool: y = (sum over H*W in raster order) * (1/(H*W)) */
void avgpool_fwd(const Model& M, int li, int n, const Vec& x, Vec& y) {
  const Layer& l = M.L[li];
  const int C = l.in0.c;
  const size_t HW = (size_t)l.in0.h * l.in0.w;
  y.assign((size_t)n * C, 0.0);
  for (int s0 = 0; s0 < n; ++s0)
    for (int c = 0; c < C; ++c) {
      double v;
      if (M.mode == XO_FP32) {
        float acc = 0.f;
        for (size_t i = 0; i < HW; ++i) acc = acc + (float)x[((size_t)s0 * C + c) * HW + i];
        v = acc * (float)(1.0 / (double)HW);
      } else {
        double acc = 0.0;
        for (size_t i = 0; i < HW; ++i) acc += x[((size_t)s0 * C + c) * HW + i];
        v = acc / (double)HW;
      }
      y[(size_t)s0 * C + c] = M.qa(v, li);
    }
}

void avgpool_bwd(const Model& M, int li, int n, const Vec& dy, Vec& dx) {
  const Layer& l = M.L[li];
  const int C = l.in0.c;
  const size_t HW = (size_t)l.in0.h * l.in0.w;
  dx.assign((size_t)n * C * HW, 0.0);
  for (int s0 = 0; s0 < n; ++s0)
    for (int c = 0; c < C; ++c)
      for (size_t i = 0; i < HW; ++i) {
        double v = (M.mode == XO_FP32) ? (double)((float)dy[(size_t)s0 * C + c] * (float)(1.0 / (double)HW))
                                       : dy[(size_t)s0 * C + c] / (double)HW;
        dx[((size_t)s0 * C + c) * HW + i] = M.qg(v);
      }
}

/* AvgPool2d with zero padding counted in the divisor (PyTorch count_include_pad=True, the
   torchvision Inception-V3 branch pool): y = (sum over the kh*kw window) * (1/(kh*kw)) */
void avgpool2d_fwd(const Model& M, int li, int n, const Vec& x, Vec& y) {
  const Layer& l = M.L[li];
  const int C = l.in0.c, H = l.in0.h, Wd = l.in0.w, P = l.out.h, Q = l.out.w;
  const double inv = 1.0 / (double)(l.d.kh * l.d.kw);
  y.assign((size_t)n * C * P * Q, 0.0);
  for (int s0 = 0; s0 < n; ++s0)
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          double acc = 0.0;
          float accf = 0.f;
          for (int r = 0; r < l.d.kh; ++r)
            for (int s = 0; s < l.d.kw; ++s) {
              int ih = p * l.d.sh - l.d.ph + r, iw = q * l.d.sw - l.d.pw + s;
              if (ih < 0 || ih >= H || iw < 0 || iw >= Wd) continue;
              double v = x[(((size_t)s0 * C + c) * H + ih) * Wd + iw];
              if (M.mode == XO_FP32) accf = accf + (float)v; else acc += v;
            }
          double v = (M.mode == XO_FP32) ? (double)(accf * (float)inv) : acc * inv;
          y[(((size_t)s0 * C + c) * P + p) * Q + q] = M.qa(v, li);
        }
}

void avgpool2d_bwd(const Model& M, int li, int n, const Vec& dy, Vec& dx) {
  const Layer& l = M.L[li];
  const int C = l.in0.c, H = l.in0.h, Wd = l.in0.w, P = l.out.h, Q = l.out.w;
  const double inv = 1.0 / (double)(l.d.kh * l.d.kw);
  dx.assign((size_t)n * C * H * Wd, 0.0);
  for (int s0 = 0; s0 < n; ++s0)
    for (int c = 0; c < C; ++c)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          const double g = dy[(((size_t)s0 * C + c) * P + p) * Q + q];
          const double gi = (M.mode == XO_FP64) ? g * inv : (double)((float)g * (float)inv);
          for (int r = 0; r < l.d.kh; ++r)
            for (int s = 0; s < l.d.kw; ++s) {
              int ih = p * l.d.sh - l.d.ph + r, iw = q * l.d.sw - l.d.pw + s;
              if (ih < 0 || ih >= H || iw < 0 || iw >= Wd) continue;
              size_t idx = (((size_t)s0 * C + c) * H + ih) * Wd + iw;
              dx[idx] = M.add(dx[idx], gi);
            }
        }
  for (auto& v : dx) v = M.qg(v);
}

/* softmax cross-entropy (a6, R8): row max; e_i = exp(z_i - max) (fp32 modes: the exp is
   taken in double and rounded to fp32); sum in class order; p = e/sum;
   dz = (p - onehot) * (1/N) with N the mini-batch size; loss = -log p_y (reporting). */
void xent(const Model& M, int n, int classes, int N, const Vec& z, const int32_t* y, Vec& dz, double* loss_sum) {
  dz.assign((size_t)n * classes, 0.0);
  double ls = 0.0;
  const float invN = (float)(1.0 / (double)N);
  for (int r = 0; r < n; ++r) {
    const double* zr = &z[(size_t)r * classes];
    if (M.mode == XO_FP64) {
      double mx = zr[0];
      for (int c = 1; c < classes; ++c) mx = std::max(mx, zr[c]);
      double s = 0.0;
      Vec e(classes);
      for (int c = 0; c < classes; ++c) { e[c] = std::exp(zr[c] - mx); s += e[c]; }
      for (int c = 0; c < classes; ++c) dz[(size_t)r * classes + c] = (e[c] / s - (c == y[r] ? 1.0 : 0.0)) / (double)N;
      ls += -std::log(e[y[r]] / s);
    } else {
      float mx = (float)zr[0];
      for (int c = 1; c < classes; ++c) mx = std::max(mx, (float)zr[c]);
      std::vector<float> e(classes);
      float s = 0.f;
      for (int c = 0; c < classes; ++c) { e[c] = (float)std::exp((double)((float)zr[c] - mx)); s = s + e[c]; }
      for (int c = 0; c < classes; ++c) {
        float p = e[c] / s;
        float d = (p - (c == y[r] ? 1.f : 0.f)) * invN;
        dz[(size_t)r * classes + c] = M.qg(d);
      }
      ls += -std::log((double)(e[y[r]] / s));
    }
  }
  *loss_sum = ls;
}

/* ------------------------------------------------------------------------------------ */
/* Adam update and prediction (north star; Eq. (3); R1; DESIGN "sweep")        */
/* ------------------------------------------------------------------------------------ */

struct Hyper {
  double lr, b1, b2, eps;   /* as given (already float-representable) */
  int delta_form = XO_DELTA_ADAM;
  int opt = XO_OPT_ADAM;
  double mu = 0.0, wd = 0.0;  /* Momentum SGD, float-representable */
};

/* beta^k by k repeated multiplications in double, starting from 1 (DESIGN "scalars") */
double beta_pow(double beta, int64_t k) {
  double p = 1.0;
  for (int64_t i = 0; i < k; ++i) p *= beta;
  return p;
}

struct Scalars { float c1, r2, omb1, omb2, inv1, inv2; double c1d, r2d; };
Scalars scalars(const Hyper& h, int64_t k) {
  Scalars s{};
  double b1p = beta_pow(h.b1, k), b2p = beta_pow(h.b2, k);
  s.c1d = h.lr / (1.0 - b1p);
  s.r2d = 1.0 / std::sqrt(1.0 - b2p);
  s.c1 = (float)s.c1d;
  s.r2 = (float)s.r2d;
  s.omb1 = (float)(1.0 - h.b1);
  s.omb2 = (float)(1.0 - h.b2);
  s.inv1 = (float)(1.0 / (1.0 - h.b1));
  s.inv2 = (float)(1.0 / (1.0 - h.b2));
  return s;
}

/* dW of the prediction from the current moments at version k:
   Adam form  d = lr * mhat / (sqrt(vhat) + eps)  (BJ north star);
   paper form d = lr * (m/(1-b1)) / sqrt(v/(1-b2) + eps)  (Eq. (3)-(4) literal). */
double delta(int mode, const Hyper& h, const Scalars& s, double m, double v) {
  if (h.delta_form == XO_DELTA_PAPER) {
    if (mode == XO_FP64) return h.lr * (m / (1.0 - h.b1)) / std::sqrt(v / (1.0 - h.b2) + h.eps);
    return (double)(((float)h.lr * ((float)m * s.inv1)) / std::sqrt((float)v * s.inv2 + (float)h.eps));
  }
  if (mode == XO_FP64) return (s.c1d * m) / (std::sqrt(v) * s.r2d + h.eps);
  float den = std::sqrt((float)v) * s.r2 + (float)h.eps;
  return (double)((s.c1 * (float)m) / den);
}

double predict_elem(int mode, double W, double d, int s) {
  if (mode == XO_FP64) return W - (double)s * d;
  double v = (double)std::fmaf(-(float)s, (float)d, (float)W);
  return mode == XO_BF16 ? q_bf16(v) : v;
}

/* one Adam step at new version k (k >= 1), in place; returns d per element via dout */
void adam_elem(int mode, const Hyper& h, const Scalars& s, double& W, double& m, double& v, double g, double* dout) {
  if (mode == XO_FP64) {
    m = h.b1 * m + (1.0 - h.b1) * g;
    v = h.b2 * v + (1.0 - h.b2) * g * g;
    double d = (s.c1d * m) / (std::sqrt(v) * s.r2d + h.eps);
    W = W - d;
    if (dout) *dout = delta(mode, h, s, m, v);
    return;
  }
  float mf = std::fmaf((float)h.b1, (float)m, s.omb1 * (float)g);
  float vf = std::fmaf((float)h.b2, (float)v, s.omb2 * ((float)g * (float)g));
  float den = std::sqrt(vf) * s.r2 + (float)h.eps;
  float d = (s.c1 * mf) / den;
  W = (double)((float)W - d);
  m = mf;
  v = vf;
  if (dout) *dout = delta(mode, h, s, m, v);
}

/* one Momentum-SGD step (the paper's training optimizer: momentum 0.9, weight
   decay 5e-4; PyTorch SGD semantics, dampening 0, no Nesterov) with the prediction's moments
   tracked by Eq. (4) (g_t = the raw stochastic gradient; R26), in place; returns the
   paper-literal dW of Eq. (3)/(4) via dout.  fp32 order (DESIGN "f2 sweep"):
     m' = fmaf(b1, m, omb1*g)     v' = fmaf(b2, v, omb2*(g*g))
     gw = fmaf(wd, W, g)          buf' = fmaf(mu, buf, gw)         W' = W - lr*buf'           */
void sgd_elem(int mode, const Hyper& h, const Scalars& s, double& W, double& buf, double& m, double& v, double g,
              double* dout) {
  if (mode == XO_FP64) {
    m = h.b1 * m + (1.0 - h.b1) * g;
    v = h.b2 * v + (1.0 - h.b2) * g * g;
    const double gw = g + h.wd * W;
    buf = h.mu * buf + gw;
    W = W - h.lr * buf;
    if (dout) *dout = delta(mode, h, s, m, v);
    return;
  }
  const float mf = std::fmaf((float)h.b1, (float)m, s.omb1 * (float)g);
  const float vf = std::fmaf((float)h.b2, (float)v, s.omb2 * ((float)g * (float)g));
  const float gw = std::fmaf((float)h.wd, (float)W, (float)g);
  const float bf = std::fmaf((float)h.mu, (float)buf, gw);
  W = (double)((float)W - (float)h.lr * bf);
  buf = bf;
  m = mf;
  v = vf;
  if (dout) *dout = delta(mode, h, s, m, v);
}

/* ------------------------------------------------------------------------------------ */
/* Pipeline state                                                      */
/* ------------------------------------------------------------------------------------ */

struct Cache { int64_t t = -1; int ver = 0; Vec Wp; };

struct Stage {
  int k = 0, l0 = 0, l1 = 0;
  Vec W, m, v, g, buf;   /* buf: Momentum-SGD velocity (XO_OPT_SGD) */
  int ver = 0;
  Cache cf, cb;
  std::map<int64_t, std::vector<Vec>> stash;          /* u -> [stage input, outputs of l0..l1-1] */
  std::map<int64_t, Vec> inbox_act, inbox_grad, dlogits;
  int64_t pos = 0;                                    /* position in this epoch's program */
  bool done = false;
  std::vector<xo_trace_rec> trace;
  std::map<int, Vec> snaps;
};

}  // namespace

struct xo_ctx {
  Model M;
  Hyper H;
  int K = 1, T = 1, N = 1, n = 1;
  int schedule = XO_SCHED_XPIPE, predict = XO_PRED_PAPER, s_fwd = 0, s_bwd = 0;
  bool snapshots = false;
  bool recompute = false;                /* f3: backward re-runs the stage forward under W_hat_b */
  std::vector<Stage> S;
  std::map<int64_t, Vec> inputs;         /* micro-batch u -> input [n, C, H, W] */
  std::map<int64_t, std::vector<int32_t>> labels;
  std::map<int64_t, double> losses;
  int64_t fed = 0;                       /* micro-batches fed (absolute) */
  int64_t base = 0;                      /* first micro-batch of the current epoch minus 1 */
  int64_t total = -1;                    /* >= 0 while flushing: last micro-batch of the epoch */
};

namespace {

/* Eq. (1) P:104-109 and Eq. (2), round() read as half-up (R3), rank/2 real in
   Eq. (1) and floored in Eq. (2) as printed (R4). */
int version_difference(int K, int T, int rank, int pass) {
  double x = pass == 0 ? ((double)K + T - rank / 2.0 - 2.0) / T
                       : ((double)T + std::floor(rank / 2.0) - 1.0) / T;
  double s = std::floor(x + 0.5);
  return s < 0 ? 0 : (int)s;
}

int s_of(const xo_ctx& c, int k, int pass) {
  if (c.predict == XO_PRED_OFF) return 0;
  if (c.predict == XO_PRED_FIXED) return pass == 0 ? c.s_fwd : c.s_bwd;
  return version_difference(c.K, c.T, k, pass);
}

/* bellwether prediction: W_hat = W - s*lr*dW from the stage's current moments;
   at version 0 with zero moments dW is undefined and W_hat = W. */
Vec predict_stage(const xo_ctx& c, const Stage& st, int s) {
  Vec out(st.W.size());
  bool trivial = (c.H.delta_form == XO_DELTA_ADAM && st.ver == 0);
  Scalars sc = scalars(c.H, st.ver);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < st.W.size(); ++i) {
    if (trivial) { out[i] = c.M.mode == XO_BF16 ? q_bf16(st.W[i]) : st.W[i]; continue; }
    double d = delta(c.M.mode, c.H, sc, st.m[i], st.v[i]);
    out[i] = predict_elem(c.M.mode, st.W[i], d, s);
  }
  return out;
}

/* forward of layers l0..l1-1 on n samples under weights Wp; acts[0] = stage input,
   acts[1 + (i - l0)] = output of layer i (the XENT layer stores its input, unused) */
void stage_forward(const xo_ctx& c, const Stage& st, const Vec& Wp, int n, Vec in, std::vector<Vec>& acts) {
  const Model& M = c.M;
  acts.assign(st.l1 - st.l0 + 1, Vec());
  acts[0] = std::move(in);
  auto src = [&](int li, int which) -> const Vec& {
    int s = which == 0 ? M.L[li].src0 : M.L[li].src1;
    return acts[s - st.l0 + 1];   /* s == l0 - 1 maps to acts[0] */
  };
  for (int li = st.l0; li < st.l1; ++li) {
    const Layer& l = M.L[li];
    Vec& y = acts[li - st.l0 + 1];
    const double* Wl = Wp.data() + l.woff;
    const double* bl = Wp.data() + l.boff;
    switch (l.d.kind) {
      case XO_LINEAR: linear_fwd(M, li, n, src(li, 0), Wl, bl, y); break;
      case XO_CONV2D: conv_fwd(M, li, n, src(li, 0), Wl, bl, y); break;
      case XO_BATCHNORM2D: bn_fwd(M, li, n, src(li, 0), Wl, bl, y); break;
      case XO_RELU: {
        const Vec& x = src(li, 0);
        y.resize(x.size());
        for (size_t i = 0; i < x.size(); ++i) y[i] = x[i] > 0 ? x[i] : 0.0;
        break;
      }
      case XO_MAXPOOL2D: maxpool_fwd(M, li, n, src(li, 0), y, nullptr); break;
      case XO_AVGPOOL_GLOBAL: avgpool_fwd(M, li, n, src(li, 0), y); break;
      case XO_AVGPOOL2D: avgpool2d_fwd(M, li, n, src(li, 0), y); break;
      case XO_FLATTEN: y = src(li, 0); break;
      case XO_ADD: {
        const Vec &a = src(li, 0), &b = src(li, 1);
        y.resize(a.size());
        for (size_t i = 0; i < a.size(); ++i) y[i] = M.qa(M.add(a[i], b[i]), li);
        break;
      }
      case XO_CONCAT: {
        const Vec &a = src(li, 0), &b = src(li, 1);
        const size_t ca = l.in0.size(), cb = l.in1.size();
        y.resize((size_t)n * (ca + cb));
        for (int s0 = 0; s0 < n; ++s0) {
          std::copy(a.begin() + s0 * ca, a.begin() + (s0 + 1) * ca, y.begin() + s0 * (ca + cb));
          std::copy(b.begin() + s0 * cb, b.begin() + (s0 + 1) * cb, y.begin() + s0 * (ca + cb) + ca);
        }
        break;
      }
      case XO_SOFTMAX_XENT: y = src(li, 0); break;
    }
  }
}

/* backward of the stage (stash mode, R10): activations from the forward under Wf, dgrad
   under Wb; returns d(stage input) and the parameter gradient (stage-flat) */
void stage_backward(const xo_ctx& c, const Stage& st, const Vec& Wb, int n, const std::vector<Vec>& acts,
                    const Vec& dout, Vec& din, Vec& gW) {
  const Model& M = c.M;
  const int nl = st.l1 - st.l0;
  std::vector<Vec> d(nl + 1);
  std::vector<bool> has(nl + 1, false);
  gW.assign(st.W.size(), 0.0);
  auto acc = [&](int s, Vec&& g) {    /* gradient w.r.t. output of layer s (l0-1 = input) */
    int idx = s - st.l0 + 1;
    if (!has[idx]) { d[idx] = std::move(g); has[idx] = true; }
    else { for (size_t i = 0; i < g.size(); ++i) d[idx][i] = M.qg(M.add(d[idx][i], g[i])); }
  };
  /* seed: gradient of the stage output (last layer's output, or the XENT input) */
  int last = st.l1 - 1;
  if (M.L[last].d.kind == XO_SOFTMAX_XENT) acc(M.L[last].src0, Vec(dout));
  else acc(last, Vec(dout));
  for (int li = st.l1 - 1; li >= st.l0; --li) {
    const Layer& l = M.L[li];
    if (l.d.kind == XO_SOFTMAX_XENT) continue;
    int idx = li - st.l0 + 1;
    if (!has[idx]) continue;
    const Vec& dy = d[idx];
    const Vec& x0 = acts[l.src0 - st.l0 + 1];
    bool need_dx = !(l.src0 == st.l0 - 1 && st.k == 0);   /* first layer's dgrad is skipped */
    Vec dx;
    const double* Wl = Wb.data() + l.woff;
    switch (l.d.kind) {
      case XO_LINEAR:
        linear_bwd(M, li, n, x0, dy, Wl, dx, gW.data() + l.woff, gW.data() + l.boff, need_dx);
        if (need_dx) acc(l.src0, std::move(dx));
        break;
      case XO_CONV2D:
        conv_bwd(M, li, n, x0, dy, Wl, dx, gW.data() + l.woff, gW.data() + l.boff, need_dx);
        if (need_dx) acc(l.src0, std::move(dx));
        break;
      case XO_BATCHNORM2D:
        bn_bwd(M, li, n, x0, dy, Wl, dx, gW.data() + l.woff, gW.data() + l.boff);
        acc(l.src0, std::move(dx));
        break;
      case XO_RELU: {
        const Vec& y = acts[idx];
        dx.resize(dy.size());
        for (size_t i = 0; i < dy.size(); ++i) dx[i] = y[i] > 0 ? dy[i] : 0.0;
        acc(l.src0, std::move(dx));
        break;
      }
      case XO_MAXPOOL2D: maxpool_bwd(M, li, n, x0, dy, dx); acc(l.src0, std::move(dx)); break;
      case XO_AVGPOOL_GLOBAL: avgpool_bwd(M, li, n, dy, dx); acc(l.src0, std::move(dx)); break;
      case XO_AVGPOOL2D: avgpool2d_bwd(M, li, n, dy, dx); acc(l.src0, std::move(dx)); break;
      case XO_FLATTEN: acc(l.src0, Vec(dy)); break;
      case XO_ADD: acc(l.src0, Vec(dy)); acc(l.src1, Vec(dy)); break;
      case XO_CONCAT: {
        const size_t ca = l.in0.size(), cb = l.in1.size();
        Vec da((size_t)n * ca), db((size_t)n * cb);
        for (int s0 = 0; s0 < n; ++s0) {
          std::copy(dy.begin() + s0 * (ca + cb), dy.begin() + s0 * (ca + cb) + ca, da.begin() + s0 * ca);
          std::copy(dy.begin() + s0 * (ca + cb) + ca, dy.begin() + (s0 + 1) * (ca + cb), db.begin() + s0 * cb);
        }
        acc(l.src0, std::move(da));
        acc(l.src1, std::move(db));
        break;
      }
    }
  }
  if (has[0]) din = d[0]; else din.clear();
}

/* the stage program (a1; R7): XPipe = K-k warm-up forwards, then B(i), F(i+K-k) pairs,
   then drain; GPipe = per mini-batch all T forwards then all T backwards. op: 0=F 1=B */
void program_op(const xo_ctx& c, const Stage& st, int64_t p, int& op, int64_t& u) {
  if (c.schedule == XO_SCHED_GPIPE) {
    int64_t t = p / (2 * c.T), r = p % (2 * c.T);
    op = r < c.T ? 0 : 1;
    u = t * c.T + (r < c.T ? r : r - c.T) + 1;
  } else {
    int64_t W = c.K - st.k;
    if (p < W) { op = 0; u = p + 1; }
    else {
      int64_t q = p - W, i = q / 2 + 1;
      if (q % 2 == 0) { op = 1; u = i; } else { op = 0; u = i + W; }
    }
  }
  u += c.base;
}

void trace_push(Stage& st, int op, int64_t t, int64_t j, int ver, int s, int bw) {
  xo_trace_rec r{st.k, op, (int32_t)t, (int32_t)j, ver, s, bw};
  st.trace.push_back(r);
}

/* try to run stage k's next op (O2-O4); returns 1 if an op ran, 0 if blocked/done, <0 err */
int try_step(xo_ctx& c, int k) {
  Stage& st = c.S[k];
  if (st.done) return 0;
  for (;;) {
    int op;
    int64_t u;
    program_op(c, st, st.pos, op, u);
    if (c.total >= 0 && u > c.total) {
      if (op == 1 || c.schedule == XO_SCHED_GPIPE) { st.done = true; return 0; }
      ++st.pos;      /* flushing: forwards beyond the last fed micro-batch are dropped */
      continue;
    }
    const int64_t t = (u - 1) / c.T + 1, j = u - (t - 1) * c.T;
    if (op == 0) {
      if (u > c.fed) return 0;
      if (k > 0 && !st.inbox_act.count(u)) return 0;
      /* O3 */
      const int s = s_of(c, k, 0);
      if (j == 1) { st.cf.t = t; st.cf.ver = st.ver; st.cf.Wp = predict_stage(c, st, s); }
      else if (st.cf.t != t) return fail(E_SCHED, "forward cache miss");
      Vec in;
      if (k == 0) in = c.inputs.at(u);
      else { in = std::move(st.inbox_act[u]); st.inbox_act.erase(u); }
      std::vector<Vec> acts;
      stage_forward(c, st, st.cf.Wp, c.n, std::move(in), acts);
      st.stash[u] = std::move(acts);
      trace_push(st, 0, t, j, st.cf.ver, s, j == 1);
      if (k + 1 < c.K) {
        c.S[k + 1].inbox_act[u] = st.stash[u].back();
      } else {
        const std::vector<Vec>& a = st.stash[u];
        Vec dz;
        double ls;
        xent(c.M, c.n, c.M.classes, c.N, a.back(), c.labels.at(u).data(), dz, &ls);
        c.losses[u] = ls / c.n;
        st.dlogits[u] = std::move(dz);
      }
      ++st.pos;
      return 1;
    } else {
      if (k + 1 < c.K) { if (!st.inbox_grad.count(u)) return 0; }
      else if (!st.dlogits.count(u)) return 0;
      if (!st.stash.count(u)) return fail(E_SCHED, "backward without stash");
      /* O4 */
      const int s = s_of(c, k, 1);
      if (j == 1) { st.cb.t = t; st.cb.ver = st.ver; st.cb.Wp = predict_stage(c, st, s); }
      else if (st.cb.t != t) return fail(E_SCHED, "backward cache miss");
      Vec dout;
      if (k + 1 < c.K) { dout = std::move(st.inbox_grad[u]); st.inbox_grad.erase(u); }
      else { dout = std::move(st.dlogits[u]); st.dlogits.erase(u); }
      Vec din, gW;
      if (c.recompute) {
        /* f3: activation recomputation -- the stage forward again, now under W_hat_b,
           from the stashed stage input; the backward differentiates this forward (an exact
           VJP of the stage at W_hat_b), the last stage from its recomputed loss gradient */
        std::vector<Vec> acts;
        stage_forward(c, st, st.cb.Wp, c.n, st.stash[u][0], acts);
        if (k + 1 == c.K) {
          double ls;
          xent(c.M, c.n, c.M.classes, c.N, acts.back(), c.labels.at(u).data(), dout, &ls);
        }
        stage_backward(c, st, st.cb.Wp, c.n, acts, dout, din, gW);
      } else {
        stage_backward(c, st, st.cb.Wp, c.n, st.stash[u], dout, din, gW);
      }
      st.stash.erase(u);
      if (j == 1) st.g = gW;
      else {
        const int64_t ng = (int64_t)gW.size();
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < ng; ++i) st.g[i] = c.M.add(st.g[i], gW[i]);
      }
      if (k > 0) c.S[k - 1].inbox_grad[u] = std::move(din);
      trace_push(st, 1, t, j, st.cb.ver, s, j == 1);
      if (j == c.T) {
        /* the T-th micro-batch's backward ends the mini-batch: update */
        const int64_t kv = st.ver + 1;
        Scalars sc = scalars(c.H, kv);
        const int64_t np = (int64_t)st.W.size();  /* elementwise: each element's step is independent */
        if (c.H.opt == XO_OPT_SGD) {
#pragma omp parallel for schedule(static)
          for (int64_t i = 0; i < np; ++i)
            sgd_elem(c.M.mode, c.H, sc, st.W[i], st.buf[i], st.m[i], st.v[i], st.g[i], nullptr);
        } else {
#pragma omp parallel for schedule(static)
          for (int64_t i = 0; i < np; ++i) adam_elem(c.M.mode, c.H, sc, st.W[i], st.m[i], st.v[i], st.g[i], nullptr);
        }
        st.ver = (int)kv;
        trace_push(st, 2, t, j, st.ver, 0, 0);
        if (c.snapshots) st.snaps[st.ver] = st.W;
      }
      ++st.pos;
      return 1;
    }
  }
}

int drive(xo_ctx& c) {
  for (;;) {
    bool progress = false;
    for (int k = 0; k < c.K; ++k) {
      for (;;) {
        int r = try_step(c, k);
        if (r < 0) return r;
        if (r == 0) break;
        progress = true;
      }
    }
    if (!progress) return 0;
  }
}

}  // namespace

/* ====================================================================================== */
/* C ABI                                                                                  */
/* ====================================================================================== */

extern "C" {

const char* xo_last_error(void) { return g_err.c_str(); }

int xo_version_difference(int32_t K, int32_t T, int32_t rank, int32_t pass) {
  return version_difference(K, T, rank, pass);
}

int xo_init(const xo_layer* layers, int32_t n_layers, int32_t stages, int32_t T, int32_t N, double lr,
            double beta1, double beta2, double eps, const xo_config* cfg, xo_ctx** out) {
  if (!out) return fail(E_INVAL, "out is NULL");
  *out = nullptr;
  if (!layers || n_layers < 2 || !cfg) return fail(E_INVAL, "layers/cfg");
  if (stages < 1 || T < 1 || N < 1 || N % T) return fail(E_INVAL, "mini_batch % micro_batches != 0");
  if (!(lr > 0) || !(beta1 >= 0 && beta1 < 1) || !(beta2 >= 0 && beta2 < 1) || !(eps > 0))
    return fail(E_INVAL, "hyperparameters");
  std::unique_ptr<xo_ctx> c(new xo_ctx());
  c->K = stages; c->T = T; c->N = N; c->n = N / T;
  c->H.lr = lr; c->H.b1 = beta1; c->H.b2 = beta2; c->H.eps = eps; c->H.delta_form = cfg->delta_form;
  c->H.opt = cfg->optimizer; c->H.mu = cfg->momentum; c->H.wd = cfg->weight_decay;
  if (c->H.opt != XO_OPT_ADAM && c->H.opt != XO_OPT_SGD) return fail(E_INVAL, "optimizer");
  if (c->H.opt == XO_OPT_SGD && (cfg->delta_form != XO_DELTA_PAPER || !(c->H.mu >= 0 && c->H.mu < 1) || !(c->H.wd >= 0)))
    return fail(E_INVAL, "Momentum SGD needs the paper prediction form, momentum in [0,1), weight decay >= 0");
  c->schedule = cfg->schedule; c->predict = cfg->predict; c->s_fwd = cfg->s_fwd; c->s_bwd = cfg->s_bwd;
  c->snapshots = cfg->snapshots != 0;
  c->recompute = cfg->recompute != 0;
  Model& M = c->M;
  M.mode = cfg->mode;
  M.input = Shape{cfg->in_c, cfg->in_h, cfg->in_w};
  M.classes = cfg->classes;
  if (M.input.size() == 0 || M.classes < 1) return fail(E_INVAL, "input shape / classes");
  if (layers[n_layers - 1].kind != XO_SOFTMAX_XENT) return fail(E_INVAL, "last layer must be softmax-xent");
  M.L.resize(n_layers);
  /* shapes */
  for (int i = 0; i < n_layers; ++i) {
    Layer& l = M.L[i];
    l.d = layers[i];
    l.src0 = l.d.src0 < 0 ? i - 1 : l.d.src0;
    l.src1 = l.d.src1 < 0 ? -1 : l.d.src1;
    if (l.src0 >= i || l.src1 >= i) return fail(E_INVAL, "sources must precede the layer");
    l.in0 = l.src0 < 0 ? M.input : M.L[l.src0].out;
    if (l.src1 >= 0) l.in1 = M.L[l.src1].out;
    const Shape& x = l.in0;
    switch (l.d.kind) {
      case XO_LINEAR:
        if ((size_t)l.d.in_c != x.size()) return fail(E_INVAL, "linear in_features");
        l.out = Shape{l.d.out_c, 1, 1};
        l.nw = (size_t)l.d.out_c * l.d.in_c; l.nb = l.d.bias ? l.d.out_c : 0;
        break;
      case XO_CONV2D: {
        if (l.d.in_c != x.c || l.d.kh < 1 || l.d.kw < 1 || l.d.sh < 1 || l.d.sw < 1) return fail(E_INVAL, "conv shape");
        int P = (x.h + 2 * l.d.ph - l.d.kh) / l.d.sh + 1, Q = (x.w + 2 * l.d.pw - l.d.kw) / l.d.sw + 1;
        if (P < 1 || Q < 1) return fail(E_INVAL, "conv output empty");
        l.out = Shape{l.d.out_c, P, Q};
        l.nw = (size_t)l.d.out_c * x.c * l.d.kh * l.d.kw; l.nb = l.d.bias ? l.d.out_c : 0;
        break;
      }
      case XO_BATCHNORM2D:
        if (l.d.in_c != x.c) return fail(E_INVAL, "bn channels");
        l.out = x; l.nw = x.c; l.nb = x.c;
        break;
      case XO_RELU: case XO_FLATTEN: case XO_SOFTMAX_XENT:
        l.out = l.d.kind == XO_FLATTEN ? Shape{(int)x.size(), 1, 1} : x;
        if (l.d.kind == XO_SOFTMAX_XENT && (i != n_layers - 1 || x.size() != (size_t)M.classes))
          return fail(E_INVAL, "softmax-xent must be last and see [classes] logits");
        break;
      case XO_MAXPOOL2D: case XO_AVGPOOL2D: {
        int P = (x.h + 2 * l.d.ph - l.d.kh) / l.d.sh + 1, Q = (x.w + 2 * l.d.pw - l.d.kw) / l.d.sw + 1;
        if (P < 1 || Q < 1 || l.d.sh < 1 || l.d.sw < 1) return fail(E_INVAL, "pool shape");
        l.out = Shape{x.c, P, Q};
        break;
      }
      case XO_AVGPOOL_GLOBAL: l.out = Shape{x.c, 1, 1}; break;
      case XO_ADD:
        if (l.src1 < 0 || l.in1.c != x.c || l.in1.h != x.h || l.in1.w != x.w) return fail(E_INVAL, "add shapes");
        l.out = x;
        break;
      case XO_CONCAT:
        if (l.src1 < 0 || l.in1.h != x.h || l.in1.w != x.w) return fail(E_INVAL, "concat shapes");
        l.out = Shape{x.c + l.in1.c, x.h, x.w};
        break;
      default: return fail(E_INVAL, "unknown layer kind");
    }
  }
  /* partition (A20, R17): units begin at every Linear/Conv2d layer (and at layer 0);
     layer-count rule with the remainder to the last r stages. */
  bool explicit_stage = layers[0].stage >= 0;
  if (explicit_stage) {
    for (int i = 0; i < n_layers; ++i) {
      int s = layers[i].stage;
      if (s < 0 || s >= stages) return fail(E_INVAL, "explicit stage out of range");
      if (i > 0 && s != layers[i - 1].stage && s != layers[i - 1].stage + 1) return fail(E_INVAL, "stages must be contiguous");
      M.L[i].stage = s;
    }
    if (M.L[n_layers - 1].stage != stages - 1 || M.L[0].stage != 0) return fail(E_INVAL, "every stage must own layers");
  } else {
    std::vector<int> unit_of(n_layers);
    int units = 0;
    for (int i = 0; i < n_layers; ++i) {
      bool starts = (i == 0) || ((M.L[i].d.kind == XO_LINEAR || M.L[i].d.kind == XO_CONV2D) &&
                                  [&] { for (int j = 0; j < i; ++j) if (M.L[j].d.kind == XO_LINEAR || M.L[j].d.kind == XO_CONV2D) return true; return false; }());
      if (starts && i > 0) ++units;
      unit_of[i] = units;
    }
    ++units;
    if (stages > units) return fail(E_INVAL, "more stages than partition units");
    int base = units / stages, r = units % stages;
    std::vector<int> stage_of_unit(units);
    int u = 0;
    for (int k = 0; k < stages; ++k) {
      int cnt = base + (k >= stages - r ? 1 : 0);
      for (int q = 0; q < cnt; ++q) stage_of_unit[u++] = k;
    }
    for (int i = 0; i < n_layers; ++i) M.L[i].stage = stage_of_unit[unit_of[i]];
  }
  /* stages, parameter offsets, DAG-edge check */
  c->S.resize(stages);
  for (int k = 0; k < stages; ++k) { c->S[k].k = k; c->S[k].l0 = -1; }
  for (int i = 0; i < n_layers; ++i) {
    Stage& st = c->S[M.L[i].stage];
    if (st.l0 < 0) st.l0 = i;
    st.l1 = i + 1;
  }
  for (int i = 0; i < n_layers; ++i) {
    const Layer& l = M.L[i];
    const Stage& st = c->S[l.stage];
    for (int s : {l.src0, l.src1}) {
      if (s == -1 && l.src1 == s && s != l.src0) continue;
      if (s < st.l0 - 1 && !(s == -1 && st.l0 == 0)) return fail(E_INVAL, "DAG edge crosses a stage cut");
    }
  }
  for (int k = 0; k < stages; ++k) {
    Stage& st = c->S[k];
    size_t off = 0;
    for (int i = st.l0; i < st.l1; ++i) {
      Layer& l = M.L[i];
      l.woff = off; off += l.nw;
      l.boff = off; off += l.nb;
    }
    st.W.assign(off, 0.0); st.m.assign(off, 0.0); st.v.assign(off, 0.0); st.g.assign(off, 0.0);
    st.buf.assign(off, 0.0);
    for (int i = st.l0; i < st.l1; ++i) {
      const Layer& l = M.L[i];
      if (l.nw) {
        const double* p = cfg->init_params ? cfg->init_params[2 * i] : nullptr;
        if (!p) return fail(E_INVAL, "init_params missing a weight tensor");
        for (size_t q = 0; q < l.nw; ++q) st.W[l.woff + q] = M.mode == XO_FP64 ? p[q] : (double)(float)p[q];
      }
      if (l.nb) {
        const double* p = cfg->init_params ? cfg->init_params[2 * i + 1] : nullptr;
        if (!p) return fail(E_INVAL, "init_params missing a bias tensor");
        for (size_t q = 0; q < l.nb; ++q) st.W[l.boff + q] = M.mode == XO_FP64 ? p[q] : (double)(float)p[q];
      }
    }
    if (cfg->init_m && cfg->init_m[k]) for (size_t q = 0; q < off; ++q) st.m[q] = cfg->init_m[k][q];
    if (cfg->init_v && cfg->init_v[k]) for (size_t q = 0; q < off; ++q) st.v[q] = cfg->init_v[k][q];
    if (c->snapshots) st.snaps[0] = st.W;
  }
  if (c->M.mode != XO_FP64 && c->M.mode != XO_FP32 && c->M.mode != XO_BF16) return fail(E_INVAL, "mode");
  *out = c.release();
  return E_OK;
}

int xo_step(xo_ctx* c, const float* x, const int32_t* y, int32_t Mb, int32_t flush, float* losses) {
  if (!c) return fail(E_INVAL, "ctx");
  if (Mb < 0 || (Mb > 0 && (!x || !y))) return fail(E_INVAL, "inputs");
  const size_t per = c->M.input.size();
  const int64_t first = c->fed + 1;
  for (int64_t b = 0; b < (int64_t)Mb * c->T; ++b) {
    const int64_t u = c->fed + 1;
    Vec in((size_t)c->n * per);
    std::vector<int32_t> lab(c->n);
    for (size_t i = 0; i < in.size(); ++i) {
      double v = x[(size_t)b * c->n * per + i];
      in[i] = c->M.mode == XO_BF16 ? q_bf16(v) : v;  /* the network input is a rounding point */
    }
    for (int r = 0; r < c->n; ++r) {
      lab[r] = y[(size_t)b * c->n + r];
      if (lab[r] < 0 || lab[r] >= c->M.classes) return fail(E_INVAL, "label out of range");
    }
    c->inputs[u] = std::move(in);
    c->labels[u] = std::move(lab);
    c->fed = u;
  }
  int r = drive(*c);
  if (r < 0) return r;
  if (flush) {
    c->total = c->fed;
    r = drive(*c);
    if (r < 0) return r;
    for (auto& st : c->S) {
      if (!st.done || !st.stash.empty()) return fail(E_SCHED, "flush did not drain");
      st.done = false;
      st.pos = 0;
    }
    c->base = c->fed;
    c->total = -1;
  }
  /* inputs/labels of micro-batches whose forward ran on stage 0 / last stage can go */
  if (losses)
    for (int64_t u = first; u <= c->fed; ++u) {
      auto it = c->losses.find(u);
      losses[u - first] = it == c->losses.end() ? NAN : (float)it->second;
    }
  return E_OK;
}

int xo_stage_of_layer(xo_ctx* c, int32_t layer) {
  if (!c || layer < 0 || layer >= (int)c->M.L.size()) return fail(E_INVAL, "layer");
  return c->M.L[layer].stage;
}

int xo_stage_version(xo_ctx* c, int32_t stage) {
  if (!c || stage < 0 || stage >= c->K) return fail(E_INVAL, "stage");
  return c->S[stage].ver;
}

int64_t xo_param_count(xo_ctx* c, int32_t layer, int32_t tensor) {
  if (!c || layer < 0 || layer >= (int)c->M.L.size()) return fail(E_INVAL, "layer");
  return tensor == 0 ? (int64_t)c->M.L[layer].nw : (int64_t)c->M.L[layer].nb;
}

int xo_get_param(xo_ctx* c, int32_t layer, int32_t tensor, int32_t state, int64_t version, double* dst, size_t count) {
  if (!c || layer < 0 || layer >= (int)c->M.L.size() || !dst) return fail(E_INVAL, "args");
  const Layer& l = c->M.L[layer];
  const size_t n = tensor == 0 ? l.nw : l.nb;
  if (count != n) return fail(E_INVAL, "count is not the tensor size");
  const Stage& st = c->S[l.stage];
  const size_t off = tensor == 0 ? l.woff : l.boff;
  const Vec* src = nullptr;
  Vec tmp;
  switch (state) {
    case XO_PARAM:
      if (version < 0 || version == st.ver) src = &st.W;
      else {
        auto it = st.snaps.find((int)version);
        if (it == st.snaps.end()) return fail(E_INVAL, "no snapshot of that version");
        src = &it->second;
      }
      break;
    case XO_M: src = &st.m; break;
    case XO_BUF: src = &st.buf; break;
    case XO_V: src = &st.v; break;
    case XO_GRAD: src = &st.g; break;
    case XO_PRED_FWD: case XO_PRED_BWD:
      tmp = predict_stage(*c, st, s_of(*c, st.k, state == XO_PRED_FWD ? 0 : 1));
      src = &tmp;
      break;
    default: return fail(E_INVAL, "state");
  }
  for (size_t i = 0; i < n; ++i) dst[i] = (*src)[off + i];
  return E_OK;
}

int xo_get_trace(xo_ctx* c, int32_t stage, xo_trace_rec* dst, size_t cap, size_t* n_out) {
  if (!c || stage < 0 || stage >= c->K || !n_out) return fail(E_INVAL, "args");
  const auto& tr = c->S[stage].trace;
  *n_out = tr.size();
  if (dst) std::memcpy(dst, tr.data(), std::min(cap, tr.size()) * sizeof(xo_trace_rec));
  return E_OK;
}

int xo_eval_loss_grad(xo_ctx* c, const float* x, const int32_t* y, int32_t n, double* loss, double* grad, size_t count) {
  if (!c || !x || !y || n < 1 || !loss) return fail(E_INVAL, "args");
  const size_t per = c->M.input.size();
  Vec in((size_t)n * per);
  for (size_t i = 0; i < in.size(); ++i) in[i] = c->M.mode == XO_BF16 ? q_bf16(x[i]) : x[i];
  /* forward through every stage under the master weights (Q'd in bf16 mode) */
  std::vector<std::vector<Vec>> acts(c->K);
  std::vector<Vec> Wq(c->K);
  Vec cur = std::move(in);
  for (int k = 0; k < c->K; ++k) {
    const Stage& st = c->S[k];
    Wq[k] = st.W;
    if (c->M.mode == XO_BF16) for (auto& w : Wq[k]) w = q_bf16(w);
    stage_forward(*c, st, Wq[k], n, std::move(cur), acts[k]);
    cur = acts[k].back();
  }
  Vec dz;
  double ls;
  xent(c->M, n, c->M.classes, n, cur, y, dz, &ls);
  *loss = ls / n;
  /* backward through every stage; the gradient of layer i's tensors goes to its slot */
  size_t total = 0;
  for (const auto& l : c->M.L) total += l.nw + l.nb;
  if (grad && count != total) return fail(E_INVAL, "count is not the parameter total");
  std::vector<Vec> gk(c->K);
  Vec dcur = std::move(dz);
  for (int k = c->K - 1; k >= 0; --k) {
    Vec din;
    stage_backward(*c, c->S[k], Wq[k], n, acts[k], dcur, din, gk[k]);
    dcur = std::move(din);
  }
  if (grad) {
    size_t o = 0;
    for (const auto& l : c->M.L) {
      const Vec& g = gk[l.stage];
      for (size_t q = 0; q < l.nw; ++q) grad[o++] = g[l.woff + q];
      for (size_t q = 0; q < l.nb; ++q) grad[o++] = g[l.boff + q];
    }
  }
  return E_OK;
}

int xo_sgd_predict(int32_t mode, size_t n, const float* W, const float* g, const float* buf, const float* m,
                   const float* v, float lr, float beta1, float beta2, float eps, float momentum, float weight_decay,
                   int32_t s_f, int32_t s_b, float* W_out, float* buf_out, float* m_out, float* v_out, float* pf_out,
                   float* pb_out) {
  Hyper h;
  h.lr = lr; h.b1 = beta1; h.b2 = beta2; h.eps = eps; h.delta_form = XO_DELTA_PAPER;
  h.opt = XO_OPT_SGD; h.mu = momentum; h.wd = weight_decay;
  Scalars sc = scalars(h, 1);  /* the paper form uses only the constant corrections */
  for (size_t i = 0; i < n; ++i) {
    double Wd = W[i], bd = buf[i], md = m[i], vd = v[i], d;
    sgd_elem(mode, h, sc, Wd, bd, md, vd, g[i], &d);
    W_out[i] = (float)Wd; buf_out[i] = (float)bd; m_out[i] = (float)md; v_out[i] = (float)vd;
    if (pf_out) pf_out[i] = (float)predict_elem(mode, Wd, d, s_f);
    if (pb_out) pb_out[i] = (float)predict_elem(mode, Wd, d, s_b);
  }
  return E_OK;
}

int xo_adam_predict(int32_t mode, int32_t delta_form, size_t n, const float* W, const float* g, const float* m,
                    const float* v, int64_t k, float lr, float beta1, float beta2, float eps, int32_t s_f, int32_t s_b,
                    float* W_out, float* m_out, float* v_out, float* pf_out, float* pb_out) {
  if (k < 1) return fail(E_INVAL, "version must be >= 1");
  Hyper h;
  h.lr = lr; h.b1 = beta1; h.b2 = beta2; h.eps = eps; h.delta_form = delta_form;
  Scalars sc = scalars(h, k);
  for (size_t i = 0; i < n; ++i) {
    double Wd = W[i], md = m[i], vd = v[i], d;
    adam_elem(mode, h, sc, Wd, md, vd, g[i], &d);
    W_out[i] = (float)Wd; m_out[i] = (float)md; v_out[i] = (float)vd;
    if (pf_out) pf_out[i] = (float)predict_elem(mode, Wd, d, s_f);
    if (pb_out) pb_out[i] = (float)predict_elem(mode, Wd, d, s_b);
  }
  return E_OK;
}

void xo_finalize(xo_ctx* c) { delete c; }

}  // extern "C"
