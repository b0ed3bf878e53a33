#!/usr/bin/env python
"""Per-geometry timing of the tcgen05 conv GEMMs of a BASELINE model (development tool): every
unique conv geometry of ResNet-101 / Inception-V3 (64x64, micro-batch 32) or VGG-16, timed as
fprop / dgrad at one micro-batch and the batched wgrad at T micro-batches, through the C ABI
(graph replay of `iters` launches).  Prints a table sorted by each geometry's share of the
model's GEMM time per mini-batch (count x (T x (fprop + dgrad) + wgrad)).

  python scripts/model_conv_bench.py --model inception [--iters 30] [--md out.md]
"""
import argparse
import collections
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic as S  # noqa: E402
from synthetic.models import infer_shapes, resnet101, inception_v3, CONV2D  # noqa: E402
from paper_1911_04610_b200 import xpipe  # noqa: E402


def geometries(model, image):
    if model == "resnet101":
        L, _ = resnet101(classes=200)
        shape, T = (3, image, image), 8
    elif model == "inception":
        L, _ = inception_v3(classes=200, stem_pad=image < 75)
        shape, T = (3, image, image), 4
    else:
        L, shape, T = S.vgg16_cifar(), (3, 32, 32), 4
    outs = infer_shapes(L, shape)
    geo = collections.Counter()
    first = True
    for i, l in enumerate(L):
        if l.kind != CONV2D:
            continue
        s0 = i - 1 if l.src0 < 0 else l.src0
        c, h, w = shape if s0 < 0 else outs[s0]
        cp = (c + 7) // 8 * 8
        geo[(h, w, cp, l.out_c, l.kh, l.kw, l.sh, l.sw, l.ph, l.pw, first)] += 1
        first = False
    return geo, T


def pixel_box(T, Q, P):
    if Q % T == 0:
        return True
    if T % Q:
        return False
    rp = T // Q
    return P % rp == 0 or rp % P == 0


def needs_cols(geo):
    """the pipeline's rule (kernels/gemm_tc.cu tc_conv_needs_cols, blocks.cu): explicit im2col for
    few channels or a geometry the TMA pixel boxes cannot serve (not a 1x1 stride-1 conv)"""
    n, H, W, C, Co, R, S_, P, Q, sh, sw, ph, pw = geo
    if R == 1 and S_ == 1 and ph == 0 and pw == 0 and sh == 1 and sw == 1:
        return False
    return C < 64 or C % 64 != 0 or sh != 1 or sw != 1 or not pixel_box(128, Q, P) or not pixel_box(64, Q, P)


def time_launch(fn, iters):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn(st.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = torch.cuda.current_stream().cuda_stream
        for _ in range(iters):
            fn(cs)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="inception", choices=["inception", "resnet101", "vgg16"])
    ap.add_argument("--image", type=int, default=64)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--md", default="")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    geo, T = geometries(args.model, args.image)
    ws = torch.zeros((160 << 20) + (1 << 14), dtype=torch.float32, device=dev)  # upper half: im2col / dgrad operands
    n = args.batch
    rows = []
    for (H, W, C, Co, kh, kw, sh, sw, ph, pw, first), cnt in geo.items():
        P, Q = (H + 2 * ph - kh) // sh + 1, (W + 2 * pw - kw) // sw + 1
        x = torch.randn(T * n, H, W, C, device=dev).to(torch.bfloat16)
        w = (torch.randn(Co, kh, kw, C, device=dev) * 0.05).to(torch.bfloat16)
        dy = torch.randn(T * n, P, Q, Co, device=dev).to(torch.bfloat16)
        y = torch.empty(n, P, Q, Co, device=dev, dtype=torch.bfloat16)
        dx = torch.empty(n, H, W, C, device=dev, dtype=torch.bfloat16)
        gw = torch.empty(Co, kh, kw, C, device=dev, dtype=torch.float32)
        g1 = (n, H, W, C, Co, kh, kw, P, Q, sh, sw, ph, pw)
        gT = (T * n, H, W, C, Co, kh, kw, P, Q, sh, sw, ph, pw)
        flops = 2.0 * n * P * Q * Co * kh * kw * C
        # the pipeline's path: explicit im2col where the TMA pixel boxes cannot serve the geometry
        cols = needs_cols(g1)
        mf, mw = (4, 5) if cols else (1, 3)
        tf = time_launch(lambda s: xpipe.conv2d_bf16(mf, g1, x, w, y, ws=ws, stream=s), args.iters)
        td = float("nan") if first else time_launch(lambda s: xpipe.conv2d_bf16(2, g1, dy, w, dx, ws=ws, stream=s),
                                                    args.iters)
        tw = time_launch(lambda s: xpipe.conv2d_bf16(mw, gT, x, dy, gw, ws=ws, stream=s), args.iters)
        per_mb = cnt * (T * (tf + (0 if first else td)) + tw)
        rows.append(((H, W, C, Co, kh, kw, sh, ph, pw), cnt, tf, td, tw, flops, per_mb))
    rows.sort(key=lambda r: -r[6])
    total = sum(r[6] for r in rows)
    hdr = "| HxW | C->Co | kernel s/p | count | fprop us | dgrad us | wgrad(T) us | TF/s f | TF/s d | TF/s w | share |"
    out = ["# %s conv GEMMs per geometry (micro-batch %d, T=%d, one B200, graph replay)" % (args.model, n, T), "",
           "GEMM time per mini-batch: %.0f us (sum over geometries of count x (T x (fprop + dgrad) + batched wgrad))"
           % total, "", hdr, "|" + "---|" * 11]
    for (H, W, C, Co, kh, kw, sh, ph, pw), cnt, tf, td, tw, fl, pm in rows:
        out.append("| %dx%d | %d->%d | %dx%d s%d p%d,%d | %d | %.1f | %s | %.1f | %.0f | %s | %.0f | %.1f%% |" % (
            H, W, C, Co, kh, kw, sh, ph, pw, cnt, tf, "-" if td != td else "%.1f" % td, tw, fl / tf / 1e6,
            "-" if td != td else "%.0f" % (fl / td / 1e6), T * fl / tw / 1e6, 100 * pm / total))
    txt = "\n".join(out) + "\n"
    print(txt)
    if args.md:
        open(args.md, "w").write(txt)


if __name__ == "__main__":
    main()
