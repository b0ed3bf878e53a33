// blocks.cu -- per-stage device memory and the forward/backward of one fused block.
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
int allocate_stage(xpipe_ctx* c, StageRT& s) {
  const StagePlan& p = s.plan;
  const bool bf = is_bf16(c);
  const size_t pes = bf ? 2 : 4;
  const size_t P = (size_t)p.P;
  auto A = [&](size_t bytes) { return dmalloc(c, bytes, s.dev); };
  s.W = (float*)A(P * 4); s.g = (float*)A(P * 4); s.m = (float*)A(P * 4); s.v = (float*)A(P * 4);
  s.pf[0] = A(P * pes); s.pf[1] = A(P * pes); s.pb = A(P * pes);
  s.ds = (DevState*)A(sizeof(DevState));
  s.flags = (uint32_t*)A(64);
  if (!s.W || !s.g || !s.m || !s.v || !s.pf[0] || !s.pf[1] || !s.pb || !s.ds || !s.flags)
    return set_err(c, XP_ENOMEM, "arena");
  XP_CUDA(c, cudaMemsetAsync(s.flags, 0, 64, s.stream));
  const int n = c->n;
  s.in_slot.resize(s.S);
  for (auto& q : s.in_slot) if (!(q = A(p.in_slot_bytes))) return set_err(c, XP_ENOMEM, "input ring");
  if (s.k + 1 < c->K) {
    s.gin_slot.resize(s.S);
    for (auto& q : s.gin_slot) if (!(q = A(p.out_bytes))) return set_err(c, XP_ENOMEM, "gradient ring");
  }
  const size_t aes = bf ? 2 : 4;
  s.out.assign(p.blocks.size(), {});
  s.mid.assign(p.blocks.size(), {});
  s.stats.assign(p.blocks.size(), {});
  for (size_t b = 0; b < p.blocks.size(); ++b) {
    const Block& B = p.blocks[b];
    if (B.kind == BK_XENT) continue;
    const size_t oes = B.logits ? 4 : aes;
    s.out[b].resize(s.S);
    for (auto& q : s.out[b]) if (!(q = A((size_t)n * B.out.size() * oes))) return set_err(c, XP_ENOMEM, "stash");
    if (B.kind == BK_CONV) {
      s.mid[b].resize(s.S);
      s.stats[b].resize(s.S);
      for (auto& q : s.mid[b]) if (!(q = A((size_t)n * B.mid.size() * 2))) return set_err(c, XP_ENOMEM, "stash");
      for (auto& q : s.stats[b]) if (!(q = (float*)A((size_t)B.mid.c * 4 * 4))) return set_err(c, XP_ENOMEM, "stash");
    }
  }
  if (s.k == c->K - 1) {
    s.dz.resize(s.S);
    for (auto& q : s.dz) if (!(q = (float*)A((size_t)n * c->cfg.classes * 4))) return set_err(c, XP_ENOMEM, "dz");
  }
  s.gbuf_elems = (int64_t)n * p.max_act;
  s.gbuf[0] = A((size_t)s.gbuf_elems * 4);
  s.gbuf[1] = A((size_t)s.gbuf_elems * 4);
  s.gmid = A((size_t)s.gbuf_elems * 4);
  if (!s.gbuf[0] || !s.gbuf[1] || !s.gmid) return set_err(c, XP_ENOMEM, "gradient scratch");
  if (bf) {
    int64_t ws = 0;
    size_t bnws = 64;
    for (const Block& B : p.blocks) {
      if (B.kind != BK_CONV) continue;
      const LayerInfo& L = c->net.layers[B.lmain];
      ConvGeo g{n, B.in.h, B.in.w, L.cin_pad, L.d.out_c, L.d.kh, L.d.kw, B.mid.h, B.mid.w, L.d.sh, L.d.sw, L.d.ph, L.d.pw};
      ws = std::max(ws, tc_conv_ws_elems(g));
      bnws = std::max(bnws, bn_ws_floats(n * B.mid.h * B.mid.w, B.mid.c));
    }
    s.ws_elems = ws;
    s.ws = (float*)A((size_t)std::max<int64_t>(ws, 64) * 4);
    s.bnws = (float*)A(bnws * 4);
    if (!s.ws || !s.bnws) return set_err(c, XP_ENOMEM, "workspace");
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
  XP_TRY(check_launch(c, launch_state_init(s.ds, c->lr, c->b1, c->b2, c->eps, s.stream), "state"));
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

int block_forward(xpipe_ctx* c, StageRT& s, size_t b, const void* x, const void* Wf, int slot) {
  const Block& B = s.plan.blocks[b];
  const LayerInfo& L = c->net.layers[B.lmain];
  if (!is_bf16(c)) {
    if (B.kind != BK_LINEAR) return set_err(c, XP_EUNSUPPORTED, "fp32 block");
    const float* W = (const float*)Wf;
    return check_launch(c, launch_linear_fwd_f32((const float*)x, W + L.woff, L.nb ? W + L.boff : nullptr,
                                                 (float*)s.out[b][slot], c->n, L.d.in_c, L.d.out_c, B.lrelu >= 0,
                                                 s.stream), "linear_fwd_f32");
  }
  return bf16_block_forward(c, s, b, x, Wf, slot);
}

int block_backward(xpipe_ctx* c, StageRT& s, int b, const void* x, const void* dy, void* dx, const void* Wb, int slot,
                   bool accumulate) {
  const Block& B = s.plan.blocks[b];
  const LayerInfo& L = c->net.layers[B.lmain];
  if (!is_bf16(c)) {
    const float* W = (const float*)Wb;
    const float* mask = B.lrelu >= 0 ? (const float*)s.out[b][slot] : nullptr;
    if (dx)
      XP_TRY(check_launch(c, launch_linear_dgrad_f32((const float*)dy, mask, W + L.woff, (float*)dx, c->n, L.d.in_c,
                                                     L.d.out_c, s.stream), "linear_dgrad_f32"));
    return check_launch(c, launch_linear_wgrad_f32((const float*)dy, mask, (const float*)x, s.g + L.woff,
                                                   L.nb ? s.g + L.boff : nullptr, c->n, L.d.in_c, L.d.out_c,
                                                   accumulate, s.stream), "linear_wgrad_f32");
  }
  return bf16_block_backward(c, s, b, x, dy, dx, Wb, slot, accumulate);
}

}  // namespace xp
