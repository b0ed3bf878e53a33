// plan.cu -- shape inference, layer-wise partition, fused ops, tensors, parameter arena.
#include <algorithm>

#include "plan.h"

#include <cstdlib>

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
      case XP_MAXPOOL2D: case XP_AVGPOOL2D: {
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
  // ---- stages, ops, tensors, arena ----
  P.stages.resize(K);
  for (int k = 0; k < K; ++k) P.stages[k].l0 = -1;
  for (int i = 0; i < n; ++i) {
    StagePlan& s = P.stages[P.layers[i].stage];
    if (s.l0 < 0) s.l0 = i;
    s.l1 = i + 1;
  }
  const int es = bf16 ? 2 : 4;
  // consumers of every layer output (fusion is legal only along single-consumer chains)
  std::vector<int> nuse(n, 0);
  for (int i = 0; i < n; ++i) {
    if (P.layers[i].src0 >= 0) nuse[P.layers[i].src0]++;
    if (P.layers[i].src1 >= 0) nuse[P.layers[i].src1]++;
  }
  auto next_is = [&](int i, int kind, int l1) {
    return i + 1 < l1 && P.layers[i + 1].d.kind == kind && P.layers[i + 1].src0 == i && P.layers[i + 1].src1 < 0 &&
           nuse[i] == 1;
  };
  for (int k = 0; k < K; ++k) {
    StagePlan& s = P.stages[k];
    // DAG edges may reach back only to the stage input (layer l0-1) -- R17
    for (int i = s.l0; i < s.l1; ++i) {
      const LayerInfo& L = P.layers[i];
      for (int q : {L.src0, L.src1})
        if (q >= 0 && q < s.l0 - 1) return bad(XP_EINVAL, "a DAG edge crosses a stage cut");
      if (L.src1 >= 0 && L.src1 == s.l0 - 1 && L.src0 == s.l0 - 1 && L.d.kind == XP_ADD)
        return bad(XP_EUNSUPPORTED, "add of the stage input with itself");
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
    // tensor ids: 0 = stage input; every op output gets a new id; flatten aliases its input
    std::vector<int> tid(n, -1);
    if (s.l0 > 0) tid[s.l0 - 1] = 0;
    TensorInfo tin;
    tin.shape = s.in; tin.es = es; tin.producer = -1;
    s.tensors.push_back(tin);
    auto tensor_of = [&](int layer) -> int { return layer < 0 ? 0 : tid[layer]; };
    for (int i = s.l0; i < s.l1;) {
      const LayerInfo& L = P.layers[i];
      Op o;
      o.in0 = tensor_of(L.src0);
      o.in1 = L.src1 >= 0 ? tensor_of(L.src1) : -1;
      if (o.in0 < 0 || (L.src1 >= 0 && o.in1 < 0)) return bad(XP_EINVAL, "source is not a tensor of this stage");
      o.sin0 = L.in0; o.sin1 = L.in1;
      int last = i;
      switch (L.d.kind) {
        case XP_LINEAR:
          o.kind = OP_LINEAR; o.lmain = i; o.sout = L.out;
          if (next_is(i, XP_RELU, s.l1)) { o.lrelu = ++last; o.relu = true; }
          break;
        case XP_CONV2D:
          if (!bf16) return bad(XP_EUNSUPPORTED, "Conv2d needs precision XP_BF16");
          o.kind = OP_CONV; o.lmain = i; o.smid = L.out; o.sout = L.out;
          if (!next_is(last, XP_BATCHNORM2D, s.l1)) return bad(XP_EUNSUPPORTED, "Conv2d must be followed by BatchNorm2d");
          o.lbn = ++last;
          if (next_is(last, XP_RELU, s.l1)) { o.lrelu = ++last; o.relu = true; }
          if (o.relu && next_is(last, XP_MAXPOOL2D, s.l1)) { o.lpool = ++last; o.sout = P.layers[last].out; }
          if (L.d.bias) return bad(XP_EUNSUPPORTED, "Conv2d bias before BatchNorm (R16: bias-free)");
          if (L.d.out_c % 8) return bad(XP_EUNSUPPORTED, "Conv2d out_channels must be a multiple of 8");
          if (!(k == 0 && L.src0 < 0) && L.in0.c % 8) return bad(XP_EUNSUPPORTED, "Conv2d in_channels must be a multiple of 8");
          break;
        case XP_ADD:
          if (!bf16) return bad(XP_EUNSUPPORTED, "Add needs precision XP_BF16");
          o.kind = OP_ADD; o.lmain = i; o.sout = L.out;
          if (next_is(i, XP_RELU, s.l1)) { o.lrelu = ++last; o.relu = true; }
          break;
        case XP_CONCAT:
          if (!bf16) return bad(XP_EUNSUPPORTED, "Concat needs precision XP_BF16");
          o.kind = OP_CONCAT; o.lmain = i; o.sout = L.out;
          break;
        case XP_MAXPOOL2D: case XP_AVGPOOL2D: case XP_AVGPOOL_GLOBAL:
          if (!bf16) return bad(XP_EUNSUPPORTED, "pooling needs precision XP_BF16");
          o.kind = L.d.kind == XP_MAXPOOL2D ? OP_MAXPOOL : (L.d.kind == XP_AVGPOOL2D ? OP_AVGPOOL : OP_GAP);
          o.lmain = i; o.sout = L.out;
          if (o.sin0.c % 8) return bad(XP_EUNSUPPORTED, "pooling needs channels % 8 == 0");
          break;
        case XP_FLATTEN:
          if (L.in0.h != 1 || L.in0.w != 1) return bad(XP_EUNSUPPORTED, "Flatten of a spatial map (needs 1x1)");
          tid[i] = o.in0;   // alias
          ++i;
          continue;
        case XP_SOFTMAX_XENT:
          o.kind = OP_XENT; o.lmain = i; o.sout = L.in0;
          break;
        default:
          return bad(XP_EUNSUPPORTED, "layer kind not supported standalone in this build (kind " +
                                          std::to_string(L.d.kind) + ")");
      }
      if (o.kind != OP_XENT) {
        TensorInfo t;
        t.shape = o.sout; t.es = es; t.producer = (int)s.ops.size();
        o.out = (int)s.tensors.size();
        s.tensors.push_back(t);
        for (int q = i; q <= last; ++q) tid[q] = o.out;
      }
      s.tensors[o.in0].consumers++;
      if (o.in1 >= 0) s.tensors[o.in1].consumers++;
      s.max_act = std::max({s.max_act, o.sin0.size(), o.sin1.size(), o.smid.size(), o.sout.size()});
      s.ops.push_back(o);
      i = last + 1;
    }
    // fold a residual Add into the conv block right before it: Add(a, b) [+ ReLU] where the
    // previous op is a conv block without ReLU / pool producing a or b for this Add alone; the
    // fused op computes relu?(Q(Q(BN(conv)) + other)) -- the rounding points of the separate ops
    // (XPIPE_NO_ADD_FUSE=1 keeps the separate Add, development)
    static const bool no_fuse = [] { const char* e = getenv("XPIPE_NO_ADD_FUSE"); return e && *e && *e != '0'; }();
    for (int o = 1; o < (int)s.ops.size() && !no_fuse; ++o) {
      Op& A = s.ops[o];
      Op& C = s.ops[o - 1];
      if (A.kind != OP_ADD || C.kind != OP_CONV || C.relu || C.lpool >= 0 || C.in1 >= 0) continue;
      if (C.out != A.in0 && C.out != A.in1) continue;
      if (A.in0 == A.in1 || s.tensors[C.out].consumers != 1 || C.out == s.out_tensor) continue;
      const int other = C.out == A.in0 ? A.in1 : A.in0;
      const Shape so = C.out == A.in0 ? A.sin1 : A.sin0;
      if (so.c != C.sout.c || so.h != C.sout.h || so.w != C.sout.w) continue;
      const int dead = C.out;
      C.in1 = other; C.sin1 = so; C.ladd = A.lmain; C.relu = A.relu; C.lrelu = A.lrelu;
      C.out = A.out;
      s.tensors[dead].consumers = 0;
      s.tensors[dead].producer = -2;  // unused: no buffers
      s.ops.erase(s.ops.begin() + o);
      for (auto& t : s.tensors)
        if (t.producer >= o) --t.producer;
      s.tensors[C.out].producer = o - 1;
    }
    // concat elimination: a Concat whose two inputs are each produced in this stage by a conv
    // block, a pooling op or another eliminated Concat, and consumed by this Concat alone,
    // becomes channel-offset views of its output (outermost Concat first, so nested and chained
    // concats resolve to one buffer); the producers store in place (XPIPE_NO_CONCAT_VIEWS=1 keeps
    // the copies, development)
    static const bool no_views = [] { const char* e = getenv("XPIPE_NO_CONCAT_VIEWS"); return e && *e && *e != '0'; }();
    if (!no_views) {
      const int no = (int)s.ops.size();
      std::vector<char> cand(no, 0);
      auto leaf_ok = [&](int t) {
        if (t <= 0 || s.tensors[t].consumers != 1) return false;
        const int pr = s.tensors[t].producer;
        if (pr < 0) return false;
        const int kd = s.ops[pr].kind;
        return kd == OP_CONV || kd == OP_MAXPOOL || kd == OP_AVGPOOL || (kd == OP_CONCAT && cand[pr]);
      };
      for (int o = 0; o < no; ++o)
        if (s.ops[o].kind == OP_CONCAT && s.ops[o].in0 != s.ops[o].in1)
          cand[o] = leaf_ok(s.ops[o].in0) && leaf_ok(s.ops[o].in1);
      for (int o = no - 1; o >= 0; --o) {
        if (!cand[o]) continue;
        const Op& O = s.ops[o];
        const TensorInfo& Y = s.tensors[O.out];
        const int base = Y.alias >= 0 ? Y.alias : O.out;
        const int off = Y.alias >= 0 ? Y.coff : 0;
        const int bc = s.tensors[base].shape.c;
        TensorInfo& A = s.tensors[O.in0];
        TensorInfo& B = s.tensors[O.in1];
        A.alias = base; A.coff = off; A.base_c = bc;
        B.alias = base; B.coff = off + O.sin0.c; B.base_c = bc;
      }
      std::vector<int> remap(no, -1);
      std::vector<Op> kept;
      for (int o = 0; o < no; ++o)
        if (!cand[o]) { remap[o] = (int)kept.size(); kept.push_back(s.ops[o]); }
      for (auto& t : s.tensors)
        if (t.producer >= 0) t.producer = cand[t.producer] ? -3 : remap[t.producer];  // -3: view of an eliminated concat
      s.ops.swap(kept);
    }
    // the op producing the logits keeps fp32
    if (s.ops.back().kind == OP_XENT) {
      const int lt = s.ops.back().in0;
      const int pr = s.tensors[lt].producer;
      if (pr < 0 || s.ops[pr].kind != OP_LINEAR) return bad(XP_EUNSUPPORTED, "logits must come from a Linear on the last stage");
      s.ops[pr].logits = true;
      s.tensors[lt].es = 4;
      s.out_tensor = lt;
    } else {
      s.out_tensor = tid[s.l1 - 1];
    }
    s.out = s.tensors[s.out_tensor].shape;
    s.in_bytes = (size_t)nm * s.in.size() * es;
    s.in_slot_bytes = s.in_bytes;
    if (k == 0 && bf16) s.in_slot_bytes = (size_t)nm * s.in.h * s.in.w * round8(s.in.c) * 2;
    s.out_bytes = (size_t)nm * s.out.size() * es;
    // stage-0 channel padding only feeds convolutions
    if (k == 0 && bf16 && s.in.c % 8)
      for (const Op& o : s.ops)
        if ((o.in0 == 0 || o.in1 == 0) && o.kind != OP_CONV) return bad(XP_EUNSUPPORTED, "network input must feed a Conv2d");
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
