// plan.cu -- shape inference, layer-wise partition, fused blocks, parameter arena.
#include <algorithm>

#include "plan.h"

namespace xp {

namespace {
int64_t align64(int64_t x) { return (x + 63) & ~int64_t(63); }
int round8(int c) { return (c + 7) & ~7; }
}  // namespace

int build_net_plan(const xpipe_layer* layers, int n, int K, const xpipe_config& cfg, int nm, NetPlan* out,
                   std::string* err) {
  auto bad = [&](int code, const std::string& m) { *err = m; return code; };
  const bool bf16 = cfg.precision == XP_BF16;
  NetPlan P;
  P.layers.resize(n);
  Shape input{cfg.in_c, cfg.in_h, cfg.in_w};
  if (input.size() <= 0 || cfg.classes < 1) return bad(XP_EINVAL, "input shape / classes");
  if (layers[n - 1].kind != XP_SOFTMAX_XENT) return bad(XP_EINVAL, "last layer must be XP_SOFTMAX_XENT");
  // ---- shapes (PyTorch semantics) ----
  for (int i = 0; i < n; ++i) {
    LayerInfo& L = P.layers[i];
    L.d = layers[i];
    L.src0 = L.d.src0 < 0 ? i - 1 : L.d.src0;
    L.src1 = L.d.src1 < 0 ? -1 : L.d.src1;
    if (L.src0 >= i || L.src1 >= i) return bad(XP_EINVAL, "layer sources must precede the layer");
    L.in0 = L.src0 < 0 ? input : P.layers[L.src0].out;
    if (L.src1 >= 0) L.in1 = P.layers[L.src1].out;
    const Shape& x = L.in0;
    switch (L.d.kind) {
      case XP_LINEAR:
        if (L.d.in_c != x.size() || L.d.out_c < 1) return bad(XP_EINVAL, "linear in_features");
        L.out = {L.d.out_c, 1, 1};
        L.nw_torch = L.nw_gpu = (int64_t)L.d.out_c * L.d.in_c;
        L.nb = L.d.bias ? L.d.out_c : 0;
        break;
      case XP_CONV2D: {
        if (L.d.in_c != x.c || L.d.kh < 1 || L.d.kw < 1 || L.d.sh < 1 || L.d.sw < 1 || L.d.ph < 0 || L.d.pw < 0)
          return bad(XP_EINVAL, "conv geometry");
        const int Pp = (x.h + 2 * L.d.ph - L.d.kh) / L.d.sh + 1, Q = (x.w + 2 * L.d.pw - L.d.kw) / L.d.sw + 1;
        if (Pp < 1 || Q < 1) return bad(XP_EINVAL, "conv output is empty");
        L.out = {L.d.out_c, Pp, Q};
        L.cin_pad = bf16 ? round8(x.c) : x.c;
        L.nw_torch = (int64_t)L.d.out_c * x.c * L.d.kh * L.d.kw;
        L.nw_gpu = (int64_t)L.d.out_c * L.d.kh * L.d.kw * L.cin_pad;
        L.nb = L.d.bias ? L.d.out_c : 0;
        break;
      }
      case XP_BATCHNORM2D:
        if (L.d.in_c != x.c) return bad(XP_EINVAL, "batchnorm channels");
        L.out = x;
        L.nw_torch = L.nw_gpu = x.c;
        L.nb = x.c;
        break;
      case XP_RELU: L.out = x; break;
      case XP_MAXPOOL2D: {
        if (L.d.kh < 1 || L.d.kw < 1 || L.d.sh < 1 || L.d.sw < 1) return bad(XP_EINVAL, "pool geometry");
        const int Pp = (x.h + 2 * L.d.ph - L.d.kh) / L.d.sh + 1, Q = (x.w + 2 * L.d.pw - L.d.kw) / L.d.sw + 1;
        if (Pp < 1 || Q < 1) return bad(XP_EINVAL, "pool output is empty");
        L.out = {x.c, Pp, Q};
        break;
      }
      case XP_AVGPOOL_GLOBAL: L.out = {x.c, 1, 1}; break;
      case XP_FLATTEN: L.out = {(int)x.size(), 1, 1}; break;
      case XP_ADD:
        if (L.src1 < 0 || L.in1.c != x.c || L.in1.h != x.h || L.in1.w != x.w) return bad(XP_EINVAL, "add shapes");
        L.out = x;
        break;
      case XP_CONCAT:
        if (L.src1 < 0 || L.in1.h != x.h || L.in1.w != x.w) return bad(XP_EINVAL, "concat shapes");
        L.out = {x.c + L.in1.c, x.h, x.w};
        break;
      case XP_SOFTMAX_XENT:
        if (i != n - 1 || x.size() != cfg.classes) return bad(XP_EINVAL, "softmax-xent must be last, on [classes] logits");
        L.out = x;
        break;
      default: return bad(XP_EINVAL, "unknown layer kind");
    }
  }
  // ---- partition: units begin at each Linear/Conv2d after the first (layer 0 opens unit 0);
  //      layer-count rule, remainder to the last r stages ("latter GPUs ... slightly
  //      greater number of layers") ----
  if (layers[0].stage >= 0) {
    for (int i = 0; i < n; ++i) {
      const int s = layers[i].stage;
      if (s < 0 || s >= K) return bad(XP_EINVAL, "explicit stage out of range");
      if (i > 0 && s != layers[i - 1].stage && s != layers[i - 1].stage + 1) return bad(XP_EINVAL, "stages must be contiguous");
      P.layers[i].stage = s;
    }
    if (P.layers[0].stage != 0 || P.layers[n - 1].stage != K - 1) return bad(XP_EINVAL, "every stage must own layers");
  } else {
    std::vector<int> unit(n);
    int u = 0;
    bool seen_weight = false;
    for (int i = 0; i < n; ++i) {
      const bool w = P.layers[i].d.kind == XP_LINEAR || P.layers[i].d.kind == XP_CONV2D;
      if (w && seen_weight) ++u;
      if (w) seen_weight = true;
      unit[i] = u;
    }
    const int units = u + 1;
    if (K > units) return bad(XP_EINVAL, "more stages than partition units");
    std::vector<int> st(units);
    const int base = units / K, r = units % K;
    int q = 0;
    for (int k = 0; k < K; ++k)
      for (int c = 0; c < base + (k >= K - r ? 1 : 0); ++c) st[q++] = k;
    for (int i = 0; i < n; ++i) P.layers[i].stage = st[unit[i]];
  }
  // ---- stages, blocks, arena ----
  P.stages.resize(K);
  for (int k = 0; k < K; ++k) P.stages[k].l0 = -1;
  for (int i = 0; i < n; ++i) {
    StagePlan& s = P.stages[P.layers[i].stage];
    if (s.l0 < 0) s.l0 = i;
    s.l1 = i + 1;
  }
  const int es = bf16 ? 2 : 4;
  for (int k = 0; k < K; ++k) {
    StagePlan& s = P.stages[k];
    // sequential chains only in this build (DAG models: ResNet/Inception are the next rows)
    for (int i = s.l0; i < s.l1; ++i) {
      const LayerInfo& L = P.layers[i];
      if (L.src1 >= 0 || L.src0 != i - 1) return bad(XP_EUNSUPPORTED, "DAG layers (add/concat/skip) are not supported yet");
    }
    int64_t off = 0;
    for (int i = s.l0; i < s.l1; ++i) {
      LayerInfo& L = P.layers[i];
      if (L.nw_gpu) { L.woff = off; off = align64(off + L.nw_gpu); }
      if (L.nb) { L.boff = off; off = align64(off + L.nb); }
    }
    s.P = std::max<int64_t>(64, off);
    s.in = P.layers[s.l0].in0;
    s.max_act = s.in.size();
    for (int i = s.l0; i < s.l1;) {
      const LayerInfo& L = P.layers[i];
      Block B;
      B.in = L.in0;
      switch (L.d.kind) {
        case XP_LINEAR:
          B.kind = BK_LINEAR; B.lmain = i; B.out = L.out;
          if (i + 1 < s.l1 && P.layers[i + 1].d.kind == XP_RELU) B.lrelu = ++i;
          ++i;
          break;
        case XP_CONV2D:
          if (!bf16) return bad(XP_EUNSUPPORTED, "Conv2d needs precision XP_BF16");
          B.kind = BK_CONV; B.lmain = i; B.mid = L.out; B.out = L.out;
          ++i;
          if (i < s.l1 && P.layers[i].d.kind == XP_BATCHNORM2D) B.lbn = i++;
          if (i < s.l1 && P.layers[i].d.kind == XP_RELU) B.lrelu = i++;
          if (i < s.l1 && P.layers[i].d.kind == XP_MAXPOOL2D) { B.lpool = i; B.out = P.layers[i].out; ++i; }
          if (B.lbn < 0 || B.lrelu < 0) return bad(XP_EUNSUPPORTED, "Conv2d must be followed by BatchNorm2d and ReLU");
          if (L.d.bias) return bad(XP_EUNSUPPORTED, "Conv2d bias before BatchNorm (R16: bias-free)");
          if (L.d.out_c % 8) return bad(XP_EUNSUPPORTED, "Conv2d out_channels must be a multiple of 8");
          if (B.lmain != 0 && L.in0.c % 8) return bad(XP_EUNSUPPORTED, "Conv2d in_channels must be a multiple of 8");
          break;
        case XP_FLATTEN:
          if (L.in0.h != 1 || L.in0.w != 1) return bad(XP_EUNSUPPORTED, "Flatten of a spatial map (needs 1x1)");
          ++i;
          continue;
        case XP_SOFTMAX_XENT:
          B.kind = BK_XENT; B.out = L.in0;
          ++i;
          break;
        default:
          return bad(XP_EUNSUPPORTED, "layer kind not supported standalone in this build (kind " +
                                          std::to_string(L.d.kind) + ")");
      }
      s.max_act = std::max({s.max_act, B.in.size(), B.mid.size(), B.out.size()});
      s.blocks.push_back(B);
    }
    for (size_t b = 0; b + 1 < s.blocks.size(); ++b)
      if (s.blocks[b + 1].kind == BK_XENT) s.blocks[b].logits = true;
    for (const Block& B : s.blocks)
      if (B.kind == BK_LINEAR && !bf16 && (B.lmain < 0)) return bad(XP_EINVAL, "internal");
    // stage output = output of the last non-xent block
    s.out = s.blocks.back().kind == BK_XENT ? s.blocks.back().out : s.blocks.back().out;
    s.in_bytes = (size_t)nm * s.in.size() * es;
    s.in_slot_bytes = s.in_bytes;
    if (k == 0 && bf16) s.in_slot_bytes = (size_t)nm * s.in.h * s.in.w * round8(s.in.c) * 2;
    s.out_bytes = (size_t)nm * s.out.size() * es;
  }
  if (!bf16)
    for (const auto& L : P.layers)
      if (L.d.kind != XP_LINEAR && L.d.kind != XP_RELU && L.d.kind != XP_FLATTEN && L.d.kind != XP_SOFTMAX_XENT)
        return bad(XP_EUNSUPPORTED, "XP_FP32 supports Linear/ReLU/Flatten/softmax-xent (the C1 MLP)");
  *out = std::move(P);
  return XP_OK;
}

void gpu_to_torch_layout(const LayerInfo& L, int tensor, const float* gpu, float* torch) {
  if (L.d.kind == XP_CONV2D && tensor == XP_T_WEIGHT) {
    const int Co = L.d.out_c, Ci = L.in0.c, R = L.d.kh, S = L.d.kw, Cp = L.cin_pad;
    for (int co = 0; co < Co; ++co)
      for (int ci = 0; ci < Ci; ++ci)
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s)
            torch[(((int64_t)co * Ci + ci) * R + r) * S + s] = gpu[(((int64_t)co * R + r) * S + s) * Cp + ci];
    return;
  }
  const int64_t n = tensor == XP_T_WEIGHT ? L.nw_torch : L.nb;
  std::copy(gpu, gpu + n, torch);
}

void torch_to_gpu_layout(const LayerInfo& L, int tensor, const float* torch, float* gpu) {
  if (L.d.kind == XP_CONV2D && tensor == XP_T_WEIGHT) {
    const int Co = L.d.out_c, Ci = L.in0.c, R = L.d.kh, S = L.d.kw, Cp = L.cin_pad;
    std::fill(gpu, gpu + L.nw_gpu, 0.f);
    for (int co = 0; co < Co; ++co)
      for (int ci = 0; ci < Ci; ++ci)
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s)
            gpu[(((int64_t)co * R + r) * S + s) * Cp + ci] = torch[(((int64_t)co * Ci + ci) * R + r) * S + s];
    return;
  }
  const int64_t n = tensor == XP_T_WEIGHT ? L.nw_torch : L.nb;
  std::copy(torch, torch + n, gpu);
}

}  // namespace xp
