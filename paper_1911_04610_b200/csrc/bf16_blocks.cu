// bf16_blocks.cu -- forward/backward of the bf16 fused ops:
//   OP_CONV    : tcgen05 implicit-GEMM conv -> BN statistics -> BN-apply [+ ReLU] [+ MaxPool]
//                backward: pool routing + ReLU mask + BN reductions -> BN input gradient ->
//                wgrad (into the fp32 accumulator g) and dgrad (under W_hat_b)
//   OP_LINEAR  : bf16-operand Linear [+ ReLU], fp32 logits when it feeds the softmax-xent
//   OP_ADD / OP_CONCAT / OP_MAXPOOL / OP_AVGPOOL / OP_GAP : the DAG glue of ResNet / Inception
// Forward runs under W_hat_f, backward under W_hat_b (stash mode, R10); BN's forward affine
// parameters and statistics are stashed per micro-batch so the backward recompute of the
// activation is bit-identical to the forward (R24).  Activation gradients that fan in from
// several consumers accumulate with the oracle's rounding point, Q(old + Q(g)).
#include <cstdlib>

#include "kernels/bf16_kernels.h"
#include "kernels/gemm_tc.h"
#include "runtime.h"

namespace xp {

namespace {
typedef __nv_bfloat16 bf16;

// bf16 Linear layers run on the tensor cores when they are a GEMM the UMMA tile can use (at
// least 32 output features: the 2048 -> 200 heads of ResNet-101 / Inception-V3, the MLP's
// hidden layers) and their rows are TMA-legal (in % 8 == 0).  The 512 -> 10 VGG-16 head (0.3
// MFLOP per micro-batch, a GEMV) stays on the SIMT kernels: on the tensor cores it costs an
// operand-preparation launch and two GEMM prologues (VGG-16 K=4: 99.6k vs 101.5k samples/s).
// XPIPE_LINEAR_SIMT=1 / =0 (development) forces either path.
bool linear_on_tc(const LayerInfo& L) {
  static const int force = [] {
    const char* e = getenv("XPIPE_LINEAR_SIMT");
    return (e && *e) ? (*e != '0' ? 1 : 0) : -1;
  }();
  if (force == 1 || L.d.in_c % 8) return false;
  return force == 0 || L.d.out_c >= 32;
}

ConvGeo conv_geo(const xpipe_ctx* c, const Op& O, const LayerInfo& L) {
  ConvGeo g;
  g.Nimg = c->n; g.H = O.sin0.h; g.W = O.sin0.w; g.C = L.cin_pad;
  g.Co = L.d.out_c; g.R = L.d.kh; g.S = L.d.kw; g.P = O.smid.h; g.Q = O.smid.w;
  g.sh = L.d.sh; g.sw = L.d.sw; g.ph = L.d.ph; g.pw = L.d.pw;
  return g;
}
// algorithmic flops of one conv GEMM (channel padding to 8 is not counted as work)
double conv_flops(const ConvGeo& g, int cin) { return 2.0 * g.Nimg * g.P * g.Q * (double)g.Co * g.R * g.S * cin; }

struct PoolGeo { int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0; };
PoolGeo pool_geo(const xpipe_ctx* c, int l) {
  PoolGeo p;
  if (l < 0) return p;
  const LayerInfo& P = c->net.layers[l];
  p.kh = P.d.kh; p.kw = P.d.kw; p.sh = P.d.sh; p.sw = P.d.sw; p.ph = P.d.ph; p.pw = P.d.pw;
  return p;
}
}  // namespace

int bf16_op_forward(xpipe_ctx* c, StageRT& s, int o, const void* Wf, int slot) {
  const Op& O = s.plan.ops[o];
  const LayerInfo& L = c->net.layers[O.lmain];
  const bf16* W = static_cast<const bf16*>(Wf);
  const bf16* x = (const bf16*)s.act[O.in0][slot];
  void* y = s.act[O.out][slot];
  const int n = c->n;
  switch (O.kind) {
    case OP_LINEAR:
      if (linear_on_tc(L))  // swap-AB tcgen05 GEMM, bias / ReLU / fp32 logits in the epilogue
        return check_launch(c, tc_linear_fwd(x, W + L.woff, L.nb ? W + L.boff : nullptr, y, n, L.d.in_c, L.d.out_c,
                                             O.relu, O.logits, s.ws, s.ws_elems, s.ctr, s.stream), "linear_fwd");
      return check_launch(c, launch_linear_fwd_bf16(x, W + L.woff, L.nb ? W + L.boff : nullptr, y, n, L.d.in_c,
                                                    L.d.out_c, O.relu, O.logits, s.stream), "linear_fwd_bf16");
    case OP_CONV: {
      const ConvGeo g = conv_geo(c, O, L);
      bf16* mid = (bf16*)s.mid[o][slot];
      // without split-K the GEMM epilogue also emits the BN partials of its 128-row tiles
      int bn_tiles = 0;
      XP_TRY(prof_begin(c, s));
      if (o < (int)s.cols.size() && !s.cols[o].empty()) {  // few input channels: explicit im2col + dense GEMM
        bf16* cols = (bf16*)s.cols[o][slot];
        XP_TRY(check_launch(c, launch_im2col_bf16(x, cols, n, g.H, g.W, g.C, g.P, g.Q, g.R, g.S, g.sh, g.sw, g.ph,
                                                  g.pw, s.stream), "im2col"));
        XP_TRY(check_launch(c, tc_im2col_fprop(g, cols, W + L.woff, mid, s.ws, s.ws_elems, s.ctr, s.stream, s.bnws,
                                               &bn_tiles), "conv_fprop"));
      } else {
        // unpooled blocks whose M tiles fit one thread-block cluster: the BN statistics and the
        // BN-apply [+ residual] [+ ReLU] run in the GEMM's epilogue (GemmArgs::bnf)
        const LayerInfo& NB = c->net.layers[O.lbn];
        BnFuse f{W + NB.woff, W + NB.boff, NB.d.bn_eps, s.stats[o][slot], (bf16*)y, s.plan.tensors[O.out].pitch(),
                 O.in1 >= 0 ? (const bf16*)s.act[O.in1][slot] : nullptr, O.relu};
        bool fused = false;
        XP_TRY(check_launch(c, tc_conv_fprop(g, x, W + L.woff, mid, s.ws, s.ws_elems, s.ctr, s.stream, s.bnws,
                                             &bn_tiles, O.lpool < 0 ? &f : nullptr, &fused), "conv_fprop"));
        if (fused) {
          // algorithmic work: the GEMM's flops (the BN pass re-reads nothing from memory)
          return prof_end(c, s, XP_PROF_CONV_FPROP, conv_flops(g, L.in0.c));
        }
      }
      XP_TRY(prof_end(c, s, XP_PROF_CONV_FPROP, conv_flops(g, L.in0.c)));
      const LayerInfo& N = c->net.layers[O.lbn];
      const int M = n * O.smid.h * O.smid.w;
      const PoolGeo p = pool_geo(c, O.lpool);
      uint8_t* pidx = O.lpool >= 0 ? s.pidx[o][slot] : nullptr;
      const double out_elems = (double)n * O.sout.h * O.sout.w * O.sout.c;
      // statistics partials: from the fprop epilogue (128-row tiles), else one reduction launch
      int chunks = bn_tiles, rc = 128;
      if (!bn_tiles) {
        XP_TRY(prof_begin(c, s));
        XP_TRY(check_launch(c, launch_bn_stats_partial(mid, M, O.smid.c, s.bnws, s.stream), "bn_stats"));
        // algorithmic bytes: the conv output read once (register-resident two passes)
        XP_TRY(prof_end(c, s, XP_PROF_BN_STATS, 2.0 * M * O.smid.c));
        rc = bn_chunk_rows(M, O.smid.c);
        chunks = (M + rc - 1) / rc;
      }
      // merge + BN-apply [+ residual] [+ ReLU] [+ pool] (one launch for small layers)
      XP_TRY(prof_begin(c, s));
      XP_TRY(check_launch(c, launch_bn_apply_stats(s.bnws, chunks, rc, N.d.bn_eps, W + N.woff, W + N.boff,
                                                   s.stats[o][slot], mid, (bf16*)y, pidx, n, O.smid.h, O.smid.w,
                                                   O.smid.c, O.sout.h, O.sout.w, p.kh, p.kw, p.sh, p.sw, p.ph, p.pw,
                                                   O.lpool >= 0, O.relu, s.stream,
                                                   O.in1 >= 0 ? (const bf16*)s.act[O.in1][slot] : nullptr,
                                                   s.plan.tensors[O.out].pitch()),
                          "bn_apply"));
      // algorithmic bytes: conv output read, output written (+ 1 B pool winner per output)
      return prof_end(c, s, XP_PROF_BN_APPLY, 2.0 * M * O.smid.c + out_elems * (O.lpool >= 0 ? 3.0 : 2.0));
    }
    case OP_ADD:
      return check_launch(c, launch_add_fwd(x, (const bf16*)s.act[O.in1][slot], (bf16*)y, (int64_t)n * O.sout.size(),
                                            O.relu, s.stream), "add_fwd");
    case OP_CONCAT:
      return check_launch(c, launch_concat_fwd(x, (const bf16*)s.act[O.in1][slot], (bf16*)y,
                                               (int64_t)n * O.sout.h * O.sout.w, O.sin0.c, O.sin1.c, s.stream),
                          "concat_fwd");
    case OP_MAXPOOL: case OP_AVGPOOL: {
      const PoolGeo p = pool_geo(c, O.lmain);
      return check_launch(c, launch_pool_fwd(x, (bf16*)y, n, O.sin0.h, O.sin0.w, O.sin0.c, O.sout.h, O.sout.w, p.kh,
                                             p.kw, p.sh, p.sw, p.ph, p.pw, O.kind == OP_AVGPOOL, s.stream,
                                             s.plan.tensors[O.out].pitch()), "pool_fwd");
    }
    case OP_GAP:
      return check_launch(c, launch_gap_fwd(x, (bf16*)y, n, O.sin0.h * O.sin0.w, O.sin0.c, s.stream), "gap_fwd");
  }
  return set_err(c, XP_EUNSUPPORTED, "op kind");
}

int bf16_op_backward(xpipe_ctx* c, StageRT& s, int o, const void* dy, void* dx0, bool acc0, void* dx1, bool acc1,
                     const void* Wb, int slot, bool accumulate_g) {
  const Op& O = s.plan.ops[o];
  const LayerInfo& L = c->net.layers[O.lmain];
  const bf16* W = static_cast<const bf16*>(Wb);
  const int n = c->n;
  switch (O.kind) {
    case OP_LINEAR: {
      if (acc0) return set_err(c, XP_EUNSUPPORTED, "fan-out into a Linear input");
      const bf16* mask = O.relu ? (const bf16*)s.act[O.out][slot] : nullptr;
      if (linear_on_tc(L) && s.lin_dy) {
        // masked bf16 output gradient (+ bias gradient), then wgrad and dgrad as tcgen05 GEMMs
        bf16* dyp = (bf16*)s.lin_dy;
        XP_TRY(check_launch(c, launch_linear_dy_prep(dy, O.logits, mask, dyp, s.lin_ldp, L.nb ? s.g + L.boff : nullptr, n,
                                                     L.d.out_c, accumulate_g, s.stream), "linear_dy_prep"));
        XP_TRY(check_launch(c, tc_linear_wgrad((const bf16*)s.act[O.in0][slot], dyp, s.lin_ldp, s.g + L.woff, n,
                                               L.d.in_c, L.d.out_c, accumulate_g, s.ws, s.ws_elems, s.ctr, s.stream),
                            "linear_wgrad"));
        if (dx0)
          XP_TRY(check_launch(c, tc_linear_dgrad(dyp, s.lin_ldp, W + L.woff, (bf16*)dx0, n, L.d.in_c, L.d.out_c, s.ws,
                                                 s.ws_elems, s.ctr, s.stream), "linear_dgrad"));
        return XP_OK;
      }
      if (dx0)
        XP_TRY(check_launch(c, launch_linear_dgrad_bf16(dy, O.logits, mask, W + L.woff, (bf16*)dx0, n, L.d.in_c,
                                                        L.d.out_c, s.stream), "linear_dgrad_bf16"));
      return check_launch(c, launch_linear_wgrad_bf16(dy, O.logits, mask, (const bf16*)s.act[O.in0][slot],
                                                      s.g + L.woff, L.nb ? s.g + L.boff : nullptr, n, L.d.in_c,
                                                      L.d.out_c, accumulate_g, s.stream), "linear_wgrad_bf16");
    }
    case OP_CONV: {
      const ConvGeo g = conv_geo(c, O, L);
      const LayerInfo& N = c->net.layers[O.lbn];
      const PoolGeo p = pool_geo(c, O.lpool);
      // gradient of the conv output.  Batched weight gradients: this micro-batch's slot of the
      // op's per-mini-batch buffer [T][n*P*Q*Co].  Otherwise alternate between two scratch
      // buffers so the side-stream wgrad of this op can overlap the next op's BN backward;
      // before reuse, wait for the wgrad two ops back
      const int b = s.gsel;
      bf16* dmid;
      const int64_t mid_elems = (int64_t)n * O.smid.size();
      if (s.wbatch) {
        dmid = (bf16*)s.dmid_all[o] + (int64_t)(s.cur_j - 1) * mid_elems;
      } else {
        s.gsel ^= 1;
        dmid = (bf16*)(b ? s.gmid1 : s.gmid);
        if (s.gdone_valid[b]) XP_CUDA(c, cudaStreamWaitEvent(s.stream, s.ev_gdone[b], 0));
      }
      const bf16* xmid = (const bf16*)s.mid[o][slot];
      const int ldy = s.plan.tensors[O.out].pitch();  // dout / y rows (a concat view: its concat's)
      const bf16* yout = (const bf16*)s.act[O.out][slot];
      const uint8_t* pw8 = O.lpool >= 0 ? s.pidx[o][slot] : nullptr;
      // algorithmic bytes per pass: the conv output, plus dout and y (+ pool winners) at the
      // output resolution; the apply pass also writes dmid
      const double mid_e = (double)n * O.smid.h * O.smid.w * O.smid.c;
      const double out_e = (double)n * O.sout.h * O.sout.w * O.sout.c;
      const double pass_bytes = 2.0 * mid_e + out_e * (O.lpool >= 0 ? 5.0 : 4.0);
      XP_TRY(prof_begin(c, s));
      XP_TRY(check_launch(c, launch_bn_bwd_reduce(xmid, (const bf16*)dy, yout, pw8, s.stats[o][slot], n, O.smid.h,
                                                  O.smid.w, O.smid.c, O.sout.h, O.sout.w, p.kh, p.kw, p.sh, p.sw, p.ph,
                                                  p.pw, O.lpool >= 0, O.relu, s.bnws, s.g + N.woff, s.g + N.boff,
                                                  accumulate_g, s.stream, O.in1 >= 0 ? (bf16*)dx1 : nullptr, acc1,
                                                  ldy), "bn_bwd_reduce"));
      XP_TRY(prof_end(c, s, XP_PROF_BN_BWD_REDUCE, pass_bytes));
      XP_TRY(prof_begin(c, s));
      XP_TRY(check_launch(c, launch_bn_bwd_apply(xmid, (const bf16*)dy, yout, pw8, s.stats[o][slot], W + N.woff, n,
                                                 O.smid.h, O.smid.w, O.smid.c, O.sout.h, O.sout.w, p.kh, p.kw, p.sh,
                                                 p.sw, p.ph, p.pw, O.lpool >= 0, O.relu, s.bnws, dmid, s.stream, ldy,
                                                 s.g + N.woff, s.g + N.boff, accumulate_g),
                          "bn_bwd_apply"));
      XP_TRY(prof_end(c, s, XP_PROF_BN_BWD_APPLY, pass_bytes + 2.0 * mid_e));
      // fork: the weight gradient (into g, read only by the update) on the side stream.
      // Batched: once per mini-batch, after the T-th micro-batch's conv-output gradient, as one
      // GEMM over the T micro-batches (K = T*n*P*Q; g stored, "accumulate, then apply")
      if (!s.wbatch || s.cur_j == c->T) {
        XP_CUDA(c, cudaEventRecord(s.ev_fork, s.stream));
        XP_CUDA(c, cudaStreamWaitEvent(s.side, s.ev_fork, 0));
        ConvGeo gw = g;
        int wslot = slot;
        const bf16* wdy = dmid;
        bool wacc = accumulate_g;
        if (s.wbatch) {
          gw.Nimg = n * c->T;
          wslot = s.cur_slot0;
          wdy = (const bf16*)s.dmid_all[o];
          wacc = false;
        }
        XP_TRY(prof_begin(c, s, s.side));
        if (o < (int)s.cols.size() && !s.cols[o].empty())
          XP_TRY(check_launch(c, tc_im2col_wgrad(gw, (const bf16*)s.cols[o][wslot], wdy, s.g + L.woff, wacc,
                                                 s.ws_side, s.ws_elems, s.ctr_side, s.side), "conv_wgrad"));
        else
          XP_TRY(check_launch(c, tc_conv_wgrad(gw, (const bf16*)s.act[O.in0][wslot], wdy, s.g + L.woff, wacc,
                                               s.ws_side, s.ws_elems, s.ctr_side, s.side), "conv_wgrad"));
        XP_TRY(prof_end(c, s, XP_PROF_CONV_WGRAD, conv_flops(gw, L.in0.c), s.side));
        if (!s.wbatch) {
          XP_CUDA(c, cudaEventRecord(s.ev_gdone[b], s.side));
          s.gdone_valid[b] = true;
        }
        s.side_used = true;
      }
      if (dx0) {
        XP_TRY(prof_begin(c, s));
        XP_TRY(check_launch(c, tc_conv_dgrad(g, O.sin0.c, dmid, W + L.woff, (bf16*)dx0, s.ws, s.ws_elems, s.ctr,
                                             s.stream, acc0, (bf16*)s.dcols, s.dcols_elems), "conv_dgrad"));
        XP_TRY(prof_end(c, s, XP_PROF_CONV_DGRAD, conv_flops(g, L.in0.c)));
      }
      return XP_OK;
    }
    case OP_ADD:
      return check_launch(c, launch_add_bwd((const bf16*)dy, (const bf16*)s.act[O.out][slot], (bf16*)dx0, (bf16*)dx1,
                                            (int64_t)n * O.sout.size(), O.relu, acc0, acc1, s.stream), "add_bwd");
    case OP_CONCAT:
      return check_launch(c, launch_concat_bwd((const bf16*)dy, (bf16*)dx0, (bf16*)dx1,
                                               (int64_t)n * O.sout.h * O.sout.w, O.sin0.c, O.sin1.c, acc0, acc1,
                                               s.stream), "concat_bwd");
    case OP_MAXPOOL: case OP_AVGPOOL: {
      if (!dx0) return XP_OK;
      const PoolGeo p = pool_geo(c, O.lmain);
      return check_launch(c, launch_pool_bwd((const bf16*)s.act[O.in0][slot], (const bf16*)dy, (bf16*)dx0, n,
                                             O.sin0.h, O.sin0.w, O.sin0.c, O.sout.h, O.sout.w, p.kh, p.kw, p.sh, p.sw,
                                             p.ph, p.pw, O.kind == OP_AVGPOOL, acc0, s.stream,
                                             s.plan.tensors[O.out].pitch()), "pool_bwd");
    }
    case OP_GAP:
      if (!dx0) return XP_OK;
      return check_launch(c, launch_gap_bwd((const bf16*)dy, (bf16*)dx0, n, O.sin0.h * O.sin0.w, O.sin0.c, acc0,
                                            s.stream), "gap_bwd");
  }
  return set_err(c, XP_EUNSUPPORTED, "op kind");
}

}  // namespace xp
