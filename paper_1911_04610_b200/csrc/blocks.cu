// blocks.cu -- per-stage device memory; op dispatch (fp32 contract path here, bf16 in bf16_blocks.cu).
#include <algorithm>
#include <cstring>
#include <vector>

#include "kernels/bf16_kernels.h"
#include "kernels/gemm_tc.h"
#include "runtime.h"

namespace xp {

namespace {
bool is_bf16(const xpipe_ctx* c) { return c->cfg.precision == XP_BF16; }
}  // namespace

// Device memory of one stage: the flat parameter arena (W, g, m, v fp32 + W_hat_f[2] and
// W_hat_b), the version/scalar state, the four ring flags, the input and gradient rings and
// one stash set per in-flight micro-batch.
// development switch: XPIPE_NO_IM2COL=1 runs few-channel convs through the cp.async gather
static bool no_im2col() {
  static const bool v = [] { const char* e = getenv("XPIPE_NO_IM2COL"); return e && *e && *e != '0'; }();
  return v;
}

int allocate_stage(xpipe_ctx* c, StageRT& s) {
  const StagePlan& p = s.plan;
  const bool bf = is_bf16(c);
  const size_t pes = bf ? 2 : 4;
  const size_t P = (size_t)p.P;
  auto A = [&](size_t bytes) { return dmalloc(c, bytes, s.dev); };
  s.W = (float*)A(P * 4); s.g = (float*)A(P * 4); s.m = (float*)A(P * 4); s.v = (float*)A(P * 4);
  s.pf[0] = A(P * pes); s.pf[1] = A(P * pes); s.pb = A(P * pes);
  s.ds = (DevState*)A(sizeof(DevState));
  s.dbase = (int64_t*)A(64);
  if (!s.dbase) return set_err(c, XP_ENOMEM, "arena");
  s.flags = (uint32_t*)dmalloc_shared(c, 64, s.dev);
  if (!s.W || !s.g || !s.m || !s.v || !s.pf[0] || !s.pf[1] || !s.pb || !s.ds || !s.flags)
    return set_err(c, XP_ENOMEM, "arena");
  if (c->cfg.optimizer == XP_OPT_MOMENTUM_SGD && !(s.buf = (float*)A(P * 4))) return set_err(c, XP_ENOMEM, "arena");
  XP_CUDA(c, cudaMemsetAsync(s.flags, 0, 64, s.stream));
  const int n = c->n;
  // rings: one contiguous allocation each (one IPC handle per ring in multi-process mode)
  // batched weight gradients read T consecutive slots as one [T*n][H][W][C] tensor: slots are
  // packed at exactly the slot size (a multiple of 16 bytes for bf16 NHWC with C % 8 == 0)
  s.in_stride = s.wbatch ? ((p.in_slot_bytes + 15) & ~size_t(15)) : ((p.in_slot_bytes + 255) & ~size_t(255));
  s.gin_stride = (p.out_bytes + 255) & ~size_t(255);
  uint8_t* ring = (uint8_t*)dmalloc_shared(c, s.in_stride * s.S, s.dev);
  if (!ring) return set_err(c, XP_ENOMEM, "input ring");
  s.in_ring = ring;
  s.in_slot.resize(s.S);
  for (int i = 0; i < s.S; ++i) s.in_slot[i] = ring + i * s.in_stride;
  if (s.k + 1 < c->K) {
    uint8_t* gr = (uint8_t*)dmalloc_shared(c, s.gin_stride * s.S, s.dev);
    if (!gr) return set_err(c, XP_ENOMEM, "gradient ring");
    s.gin_ring = gr;
    s.gin_slot.resize(s.S);
    for (int i = 0; i < s.S; ++i) s.gin_slot[i] = gr + i * s.gin_stride;
  }
  // per-micro-batch stash of every op output (tensor 0 is the input ring itself)
  s.act.assign(p.tensors.size(), {});
  s.act[0] = s.in_slot;
  s.grad.assign(p.tensors.size(), nullptr);
  for (size_t t = 1; t < p.tensors.size(); ++t) {
    const TensorInfo& T = p.tensors[t];
    if (T.producer == -2 || T.alias >= 0) continue;  // folded into a conv block / a concat view
    const size_t bytes = ((size_t)n * T.shape.size() * T.es + 15) & ~size_t(15);
    uint8_t* base = (uint8_t*)A(bytes * s.S);  // the S slots of one tensor, packed
    if (!base) return set_err(c, XP_ENOMEM, "stash");
    s.act[t].resize(s.S);
    for (int i = 0; i < s.S; ++i) s.act[t][i] = base + i * bytes;
  }
  // channel-offset views into their concat's buffers (slots of the same layout)
  for (size_t t = 1; t < p.tensors.size(); ++t) {
    const TensorInfo& T = p.tensors[t];
    if (T.alias < 0) continue;
    s.act[t].resize(s.S);
    for (int i = 0; i < s.S; ++i) s.act[t][i] = (uint8_t*)s.act[T.alias][i] + (size_t)T.coff * T.es;
  }
  // activation-gradient buffers, one per tensor (reused by every backward pass, stream-ordered)
  for (size_t t = 0; t < p.tensors.size(); ++t) {
    if (t == (size_t)p.out_tensor || p.tensors[t].producer == -2 || p.tensors[t].alias >= 0)
      continue;  // seeded by the ring / dz; unused; a slice of its concat's gradient
    if (!(s.grad[t] = A((size_t)n * p.tensors[t].shape.size() * 4))) return set_err(c, XP_ENOMEM, "gradient buffers");
  }
  s.mid.assign(p.ops.size(), {});
  s.stats.assign(p.ops.size(), {});
  s.pidx.assign(p.ops.size(), {});
  for (size_t o = 0; o < p.ops.size(); ++o) {
    const Op& O = p.ops[o];
    if (O.kind != OP_CONV) continue;
    s.mid[o].resize(s.S);
    s.stats[o].resize(s.S);
    for (auto& q : s.mid[o]) if (!(q = A((size_t)n * O.smid.size() * 2))) return set_err(c, XP_ENOMEM, "stash");
    for (auto& q : s.stats[o]) if (!(q = (float*)A((size_t)O.smid.c * 4 * 4))) return set_err(c, XP_ENOMEM, "stash");
    const LayerInfo& LC = c->net.layers[O.lmain];
    const ConvGeo cg{n, O.sin0.h, O.sin0.w, LC.cin_pad, LC.d.out_c, LC.d.kh, LC.d.kw, O.smid.h, O.smid.w,
                     LC.d.sh, LC.d.sw, LC.d.ph, LC.d.pw};
    // explicit dgrad operand scratch (geometries the TMA pixel boxes cannot serve)
    if (!(O.in0 == 0 && s.k == 0)) s.dcols_elems = std::max(s.dcols_elems, tc_dgrad_cols_elems(cg));
    // too few channels, or a geometry the TMA pixel boxes cannot serve: explicit im2col
    if ((LC.cin_pad < 64 || tc_conv_needs_cols(cg)) && !no_im2col()) {
      if (s.cols.size() < p.ops.size()) s.cols.assign(p.ops.size(), {});
      s.cols[o].resize(s.S);
      const size_t cb = (size_t)n * O.smid.h * O.smid.w * LC.d.kh * LC.d.kw * LC.cin_pad * 2;
      uint8_t* base = (uint8_t*)A(cb * s.S);  // packed slots (batched wgrad reads T of them)
      if (!base) return set_err(c, XP_ENOMEM, "im2col");
      for (int i = 0; i < s.S; ++i) s.cols[o][i] = base + i * cb;
    }
    if (s.wbatch) {
      if (s.dmid_all.size() < p.ops.size()) s.dmid_all.assign(p.ops.size(), nullptr);
      if (!(s.dmid_all[o] = A((size_t)c->T * n * O.smid.size() * 2))) return set_err(c, XP_ENOMEM, "wgrad operands");
    }
    if (O.lpool >= 0) {
      s.pidx[o].resize(s.S);
      for (auto& q : s.pidx[o]) if (!(q = (uint8_t*)A((size_t)n * O.sout.size()))) return set_err(c, XP_ENOMEM, "stash");
    }
  }
  if (s.k == c->K - 1) {
    s.dz.resize(s.S);
    for (auto& q : s.dz) if (!(q = (float*)A((size_t)n * c->cfg.classes * 4))) return set_err(c, XP_ENOMEM, "dz");
  }
  if (s.dcols_elems && !(s.dcols = A((size_t)s.dcols_elems * 2))) return set_err(c, XP_ENOMEM, "dgrad operand");
  s.gbuf_elems = (int64_t)n * p.max_act;
  s.gmid = A((size_t)s.gbuf_elems * 4);
  s.gmid1 = A((size_t)s.gbuf_elems * 4);
  if (!s.gmid || !s.gmid1) return set_err(c, XP_ENOMEM, "gradient scratch");
  if (bf) {
    int64_t ws = 0;
    size_t bnws = 64;
    for (const Op& O : p.ops) {
      if (O.kind != OP_CONV) continue;
      const LayerInfo& L = c->net.layers[O.lmain];
      ConvGeo g{n, O.sin0.h, O.sin0.w, L.cin_pad, L.d.out_c, L.d.kh, L.d.kw, O.smid.h, O.smid.w, L.d.sh, L.d.sw, L.d.ph, L.d.pw};
      ws = std::max(ws, tc_conv_ws_elems(g));
      if (s.wbatch) {  // the batched weight gradient: one GEMM over T micro-batches
        ConvGeo gb = g;
        gb.Nimg = n * c->T;
        ws = std::max(ws, tc_conv_ws_elems(gb));
      }
      const int Mmid = n * O.smid.h * O.smid.w;
      bnws = std::max(bnws, bn_ws_floats(Mmid, O.smid.c));
      bnws = std::max(bnws, (size_t)((Mmid + 127) / 128) * 2 * O.smid.c);  // fprop-epilogue partials
    }
    for (const Op& O : p.ops)
      if (O.kind == OP_LINEAR) s.lin_ldp = std::max(s.lin_ldp, (c->net.layers[O.lmain].d.out_c + 7) / 8 * 8);
    if (s.lin_ldp && !(s.lin_dy = A((size_t)n * s.lin_ldp * 2))) return set_err(c, XP_ENOMEM, "linear operand");
    s.ws_elems = ws;
    s.ws = (float*)A((size_t)std::max<int64_t>(ws, 64) * 4);
    s.bnws = (float*)A(bnws * 4);
    s.ctr = (int*)A((size_t)kTileCounters * sizeof(int));
    s.ws_side = (float*)A((size_t)std::max<int64_t>(ws, 64) * 4);
    s.ctr_side = (int*)A((size_t)kTileCounters * sizeof(int));
    if (!s.ws || !s.bnws || !s.ctr || !s.ws_side || !s.ctr_side) return set_err(c, XP_ENOMEM, "workspace");
    if (s.fstream != s.stream) {  // fb_overlap: the forward stream's own scratch
      s.ws_f = (float*)A((size_t)std::max<int64_t>(ws, 64) * 4);
      s.bnws_f = (float*)A(bnws * 4);
      s.ctr_f = (int*)A((size_t)kTileCounters * sizeof(int));
      if (!s.ws_f || !s.bnws_f || !s.ctr_f) return set_err(c, XP_ENOMEM, "workspace");
      XP_CUDA(c, cudaMemsetAsync(s.ctr_f, 0, (size_t)kTileCounters * sizeof(int), s.stream));
    }
    XP_CUDA(c, cudaMemsetAsync(s.ctr, 0, (size_t)kTileCounters * sizeof(int), s.stream));
    XP_CUDA(c, cudaMemsetAsync(s.ctr_side, 0, (size_t)kTileCounters * sizeof(int), s.stream));
  }
  return XP_OK;
}

// Initial weights (init_params in PyTorch layout, or the seeded U(-1/sqrt(fan_in), ..)
// recipe on the device), zero (or given) moments, version-0 state and predictions.
int init_stage_params(xpipe_ctx* c, StageRT& s, const xpipe_layer* layers) {
  (void)layers;
  const StagePlan& p = s.plan;
  XP_CUDA(c, cudaMemsetAsync(s.W, 0, p.P * 4, s.stream));
  XP_CUDA(c, cudaMemsetAsync(s.g, 0, p.P * 4, s.stream));
  XP_CUDA(c, cudaMemsetAsync(s.m, 0, p.P * 4, s.stream));
  XP_CUDA(c, cudaMemsetAsync(s.v, 0, p.P * 4, s.stream));
  if (s.buf) XP_CUDA(c, cudaMemsetAsync(s.buf, 0, p.P * 4, s.stream));
  std::vector<float> host_w, host_m, host_v;
  const bool given = c->cfg.init_params != nullptr;
  const bool mom = c->cfg.moment_init == XP_MOM_GIVEN;
  if (given || mom) {
    host_w.assign(p.P, 0.f);
    if (mom) { host_m.assign(p.P, 0.f); host_v.assign(p.P, 0.f); }
  }
  for (int i = p.l0; i < p.l1; ++i) {
    const LayerInfo& L = c->net.layers[i];
    for (int t = 0; t < 2; ++t) {
      const int64_t off = t == 0 ? L.woff : L.boff;
      const int64_t cnt = t == 0 ? L.nw_torch : L.nb;
      if (off < 0 || cnt == 0) continue;
      if (given) {
        const float* src = c->cfg.init_params[2 * i + t];
        if (!src) return set_err(c, XP_EINVAL, "init_params missing tensor of layer " + std::to_string(i));
        torch_to_gpu_layout(L, t, src, host_w.data() + off);
      } else {
        const int64_t ng = t == 0 ? L.nw_gpu : L.nb;
        if (L.d.kind == XP_BATCHNORM2D) {
          XP_TRY(check_launch(c, launch_fill_const(s.W + off, ng, t == 0 ? 1.f : 0.f, s.stream), "init"));
        } else {
          const int64_t fan_in = L.d.kind == XP_LINEAR ? L.d.in_c : (int64_t)L.in0.c * L.d.kh * L.d.kw;
          const float bound = (float)(1.0 / std::sqrt((double)fan_in));
          if (L.d.kind == XP_CONV2D && t == 0 && L.cin_pad != L.in0.c) {
            // generate in PyTorch layout on the host side of the recipe, then scatter
            std::vector<float> tmp(L.nw_torch), gw(L.nw_gpu);
            float* dtmp = (float*)dmalloc(c, L.nw_torch * 4, s.dev);
            if (!dtmp) return set_err(c, XP_ENOMEM, "init scratch");
            XP_TRY(check_launch(c, launch_fill_uniform(dtmp, L.nw_torch, bound, c->cfg.seed, 2 * i + t, s.stream), "init"));
            XP_CUDA(c, cudaMemcpyAsync(tmp.data(), dtmp, L.nw_torch * 4, cudaMemcpyDeviceToHost, s.stream));
            XP_CUDA(c, cudaStreamSynchronize(s.stream));
            torch_to_gpu_layout(L, t, tmp.data(), gw.data());
            XP_CUDA(c, cudaMemcpyAsync(s.W + off, gw.data(), L.nw_gpu * 4, cudaMemcpyHostToDevice, s.stream));
            XP_CUDA(c, cudaStreamSynchronize(s.stream));
          } else {
            XP_TRY(check_launch(c, launch_fill_uniform(s.W + off, ng, bound, c->cfg.seed, 2 * i + t, s.stream), "init"));
          }
        }
      }
      if (mom) {
        const float* sm = c->cfg.init_m[2 * i + t];
        const float* sv = c->cfg.init_v[2 * i + t];
        if (!sm || !sv) return set_err(c, XP_EINVAL, "init_m/init_v missing a tensor");
        torch_to_gpu_layout(L, t, sm, host_m.data() + off);
        torch_to_gpu_layout(L, t, sv, host_v.data() + off);
      }
    }
  }
  if (given) XP_CUDA(c, cudaMemcpyAsync(s.W, host_w.data(), p.P * 4, cudaMemcpyHostToDevice, s.stream));
  if (mom) {
    XP_CUDA(c, cudaMemcpyAsync(s.m, host_m.data(), p.P * 4, cudaMemcpyHostToDevice, s.stream));
    XP_CUDA(c, cudaMemcpyAsync(s.v, host_v.data(), p.P * 4, cudaMemcpyHostToDevice, s.stream));
  }
  XP_TRY(check_launch(c, launch_state_init(s.ds, c->lr, c->b1, c->b2, c->eps, c->cfg.momentum, c->cfg.weight_decay,
                                           s.stream), "state"));
  const bool bf = is_bf16(c);
  if (c->cfg.delta_form == XP_DELTA_PAPER) {
    // version 0 under the paper form: W_hat = W - s * dW_paper(m0, v0) (moments may be non-zero)
    const float sf = (float)version_difference_public(c, s.k, 0), sb = (float)version_difference_public(c, s.k, 1);
    XP_TRY(check_launch(c, launch_sweep(s.W, s.g, s.m, s.v, s.pf[0], s.pb, p.P, s.ds, nullptr, sf, sb, bf, 1, false,
                                        s.stream), "predict0"));
  } else {
    XP_TRY(check_launch(c, launch_predict_copy(s.W, s.pf[0], s.pb, p.P, bf, s.stream), "predict0"));
  }
  XP_CUDA(c, cudaMemsetAsync(s.pf[1], 0, p.P * (bf ? 2 : 4), s.stream));
  if (c->cfg.snapshots) {
    Snapshot sn{0, {}, nullptr};
    XP_CUDA(c, cudaMallocHost(&sn.pinned, p.P * 4));
    XP_CUDA(c, cudaMemcpyAsync(sn.pinned, s.W, p.P * 4, cudaMemcpyDeviceToHost, s.stream));
    s.snaps.push_back(std::move(sn));
  }
  XP_CUDA(c, cudaStreamSynchronize(s.stream));
  return XP_OK;
}

// K11: stage 0 copies (fp32) or converts (NCHW fp32 -> NHWC bf16, channels padded to 8)
// its micro-batch into its input stash slot.
int stage_input(xpipe_ctx* c, StageRT& s, const float* x, void* dst) {
  const Shape& in = s.plan.in;
  if (!is_bf16(c)) {
    XP_CUDA(c, cudaMemcpyAsync(dst, x, (size_t)c->n * in.size() * 4, cudaMemcpyDeviceToDevice, s.stream));
    return XP_OK;
  }
  return check_launch(c, launch_stage_input_bf16(x, (__nv_bfloat16*)dst, c->n, in.c, in.h, in.w, (in.c + 7) & ~7,
                                                 s.stream), "stage_input");
}

int op_forward(xpipe_ctx* c, StageRT& s, int o, const void* Wf, int slot, int64_t u) {
  const Op& O = s.plan.ops[o];
  if (O.kind == OP_XENT) {
    const int32_t* y = c->y_dev + (u - c->call_first) * c->n;
    float* loss = c->recompute_pass ? c->loss_scratch : c->loss_dev + (u - c->call_first);
    return check_launch(c, launch_xent_f32((const float*)s.act[O.in0][slot], y, s.dz[slot], loss, c->n, O.sin0.c,
                                           (float)(1.0 / (double)c->N), c->status_dev, s.stream), "xent");
  }
  if (!is_bf16(c)) {
    if (O.kind != OP_LINEAR) return set_err(c, XP_EUNSUPPORTED, "fp32 op");
    const LayerInfo& L = c->net.layers[O.lmain];
    const float* W = (const float*)Wf;
    return check_launch(c, launch_linear_fwd_f32((const float*)s.act[O.in0][slot], W + L.woff,
                                                 L.nb ? W + L.boff : nullptr, (float*)s.act[O.out][slot], c->n,
                                                 L.d.in_c, L.d.out_c, O.relu, s.stream), "linear_fwd_f32");
  }
  return bf16_op_forward(c, s, o, Wf, slot);
}

int op_backward(xpipe_ctx* c, StageRT& s, int o, const void* dy, void* dx0, bool acc0, void* dx1, bool acc1,
                const void* Wb, int slot, bool accumulate_g) {
  const Op& O = s.plan.ops[o];
  if (!is_bf16(c)) {
    const LayerInfo& L = c->net.layers[O.lmain];
    if (acc0) return set_err(c, XP_EUNSUPPORTED, "fan-out into a Linear input");
    const float* W = (const float*)Wb;
    const float* mask = O.relu ? (const float*)s.act[O.out][slot] : nullptr;
    if (dx0)
      XP_TRY(check_launch(c, launch_linear_dgrad_f32((const float*)dy, mask, W + L.woff, (float*)dx0, c->n, L.d.in_c,
                                                     L.d.out_c, s.stream), "linear_dgrad_f32"));
    return check_launch(c, launch_linear_wgrad_f32((const float*)dy, mask, (const float*)s.act[O.in0][slot],
                                                   s.g + L.woff, L.nb ? s.g + L.boff : nullptr, c->n, L.d.in_c,
                                                   L.d.out_c, accumulate_g, s.stream), "linear_wgrad_f32");
  }
  return bf16_op_backward(c, s, o, dy, dx0, acc0, dx1, acc1, Wb, slot, accumulate_g);
}

}  // namespace xp
