// bf16_blocks.cu -- forward/backward of the bf16 fused blocks:
//   BK_CONV   : tcgen05 implicit-GEMM conv -> BN statistics -> BN-apply + ReLU (+ MaxPool)
//               backward: pool routing + ReLU mask + BN reductions -> BN input gradient ->
//               wgrad (into the fp32 accumulator g) and dgrad (under W_hat_b)
//   BK_LINEAR : bf16-operand Linear (+ ReLU), fp32 logits when it feeds the softmax-xent
// Forward runs under W_hat_f, backward under W_hat_b (stash mode, R10); BN's forward affine
// parameters and statistics are stashed per micro-batch so the backward recompute of the
// activation is bit-identical to the forward.
#include "kernels/bf16_kernels.h"
#include "kernels/gemm_tc.h"
#include "runtime.h"

namespace xp {

namespace {
typedef __nv_bfloat16 bf16;

ConvGeo conv_geo(const xpipe_ctx* c, const Block& B, const LayerInfo& L) {
  ConvGeo g;
  g.Nimg = c->n; g.H = B.in.h; g.W = B.in.w; g.C = L.cin_pad;
  g.Co = L.d.out_c; g.R = L.d.kh; g.S = L.d.kw; g.P = B.mid.h; g.Q = B.mid.w;
  g.sh = L.d.sh; g.sw = L.d.sw; g.ph = L.d.ph; g.pw = L.d.pw;
  return g;
}
// algorithmic flops of one conv GEMM (real channels; padding of C to 8 not counted as work)
double conv_flops(const ConvGeo& g) { return 2.0 * g.Nimg * g.P * g.Q * (double)g.Co * g.R * g.S * g.C; }
}  // namespace

int bf16_block_forward(xpipe_ctx* c, StageRT& s, size_t b, const void* x, const void* Wf, int slot) {
  const Block& B = s.plan.blocks[b];
  const LayerInfo& L = c->net.layers[B.lmain];
  const bf16* W = static_cast<const bf16*>(Wf);
  if (B.kind == BK_LINEAR) {
    return check_launch(c, launch_linear_fwd_bf16((const bf16*)x, W + L.woff, L.nb ? W + L.boff : nullptr,
                                                  s.out[b][slot], c->n, L.d.in_c, L.d.out_c, B.lrelu >= 0, B.logits,
                                                  s.stream), "linear_fwd_bf16");
  }
  const ConvGeo g = conv_geo(c, B, L);
  bf16* mid = (bf16*)s.mid[b][slot];
  XP_TRY(prof_begin(c, s));
  XP_TRY(check_launch(c, tc_conv_fprop(g, (const bf16*)x, W + L.woff, mid, s.ws, s.ws_elems, s.stream), "conv_fprop"));
  XP_TRY(prof_end(c, s, XP_PROF_CONV_FPROP, conv_flops(g)));
  const LayerInfo& N = c->net.layers[B.lbn];
  const int M = c->n * B.mid.h * B.mid.w;
  XP_TRY(check_launch(c, launch_bn_stats(mid, M, B.mid.c, N.d.bn_eps, W + N.woff, W + N.boff, s.bnws, s.stats[b][slot],
                                         s.stream), "bn_stats"));
  int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
  const bool pool = B.lpool >= 0;
  if (pool) {
    const LayerInfo& Pl = c->net.layers[B.lpool];
    kh = Pl.d.kh; kw = Pl.d.kw; sh = Pl.d.sh; sw = Pl.d.sw; ph = Pl.d.ph; pw = Pl.d.pw;
  }
  return check_launch(c, launch_bn_apply(mid, s.stats[b][slot], (bf16*)s.out[b][slot], c->n, B.mid.h, B.mid.w, B.mid.c,
                                         B.out.h, B.out.w, kh, kw, sh, sw, ph, pw, pool, s.stream), "bn_apply");
}

int bf16_block_backward(xpipe_ctx* c, StageRT& s, int b, const void* x, const void* dy, void* dx, const void* Wb,
                        int slot, bool accumulate) {
  const Block& B = s.plan.blocks[b];
  const LayerInfo& L = c->net.layers[B.lmain];
  const bf16* W = static_cast<const bf16*>(Wb);
  if (B.kind == BK_LINEAR) {
    const bf16* mask = B.lrelu >= 0 ? (const bf16*)s.out[b][slot] : nullptr;
    if (dx)
      XP_TRY(check_launch(c, launch_linear_dgrad_bf16(dy, B.logits, mask, W + L.woff, (bf16*)dx, c->n, L.d.in_c,
                                                      L.d.out_c, s.stream), "linear_dgrad_bf16"));
    return check_launch(c, launch_linear_wgrad_bf16(dy, B.logits, mask, (const bf16*)x, s.g + L.woff,
                                                    L.nb ? s.g + L.boff : nullptr, c->n, L.d.in_c, L.d.out_c,
                                                    accumulate, s.stream), "linear_wgrad_bf16");
  }
  const ConvGeo g = conv_geo(c, B, L);
  const LayerInfo& N = c->net.layers[B.lbn];
  int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
  const bool pool = B.lpool >= 0;
  if (pool) {
    const LayerInfo& Pl = c->net.layers[B.lpool];
    kh = Pl.d.kh; kw = Pl.d.kw; sh = Pl.d.sh; sw = Pl.d.sw; ph = Pl.d.ph; pw = Pl.d.pw;
  }
  bf16* dmid = (bf16*)s.gmid;
  XP_TRY(check_launch(c, launch_bn_backward((const bf16*)s.mid[b][slot], (const bf16*)dy, s.stats[b][slot],
                                            W + N.woff, c->n, B.mid.h, B.mid.w, B.mid.c, B.out.h, B.out.w, kh, kw, sh,
                                            sw, ph, pw, pool, s.bnws, s.g + N.woff, s.g + N.boff, accumulate, dmid,
                                            s.stream), "bn_backward"));
  XP_TRY(prof_begin(c, s));
  XP_TRY(check_launch(c, tc_conv_wgrad(g, (const bf16*)x, dmid, s.g + L.woff, accumulate, s.ws, s.ws_elems, s.stream),
                      "conv_wgrad"));
  XP_TRY(prof_end(c, s, XP_PROF_CONV_WGRAD, conv_flops(g)));
  if (dx) {
    XP_TRY(prof_begin(c, s));
    XP_TRY(check_launch(c, tc_conv_dgrad(g, B.in.c, dmid, W + L.woff, (bf16*)dx, s.ws, s.ws_elems, s.stream),
                        "conv_dgrad"));
    XP_TRY(prof_end(c, s, XP_PROF_CONV_DGRAD, conv_flops(g)));
  }
  return XP_OK;
}

}  // namespace xp
