#!/usr/bin/env python
"""Per-layer timing of the tcgen05 conv GEMMs (fprop / dgrad / wgrad) through the C ABI on
the VGG-16 CIFAR layer shapes at one micro-batch (default 32 images).  Development tool: it
prints us and TFLOP/s per layer and GEMM, and the totals per micro-batch.

  python scripts/conv_bench.py [--batch 32] [--iters 50] [--check]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_04610_b200 import xpipe  # noqa: E402

VGG = [(32, 8, 64, 3), (32, 64, 64, 3), (16, 64, 128, 3), (16, 128, 128, 3), (8, 128, 256, 3), (8, 256, 256, 3),
       (8, 256, 256, 3), (4, 256, 512, 3), (4, 512, 512, 3), (4, 512, 512, 3), (2, 512, 512, 3), (2, 512, 512, 3),
       (2, 512, 512, 3)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--check", action="store_true", help="compare each GEMM with torch (fp32 math)")
    ap.add_argument("--only", type=int, default=-1, help="run only this layer index")
    ap.add_argument("--modes", default="123", help="subset of 1 fprop / 2 dgrad / 3 wgrad")
    ap.add_argument("--acc", action="store_true", help="wgrad accumulates into g (micro-batches j > 1)")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    ws = torch.zeros((16 << 20) + (1 << 14), dtype=torch.float32, device=dev)
    st = torch.cuda.Stream()
    tot = {1: 0.0, 2: 0.0, 3: 0.0}
    flops_tot = 0.0
    print("%-22s %10s %10s %10s %8s %8s %8s" % ("layer", "fprop us", "dgrad us", "wgrad us", "TF/s f", "TF/s d",
                                                 "TF/s w"))
    for li, (H, C, Co, R) in enumerate(VGG):
        if args.only >= 0 and li != args.only:
            continue
        n = args.batch
        x = torch.randn(n, H, H, C, device=dev).to(torch.bfloat16)
        w = (torch.randn(Co, R, R, C, device=dev) * 0.05).to(torch.bfloat16)
        dy = torch.randn(n, H, H, Co, device=dev).to(torch.bfloat16)
        y = torch.empty(n, H, H, Co, device=dev, dtype=torch.bfloat16)
        dx = torch.empty(n, H, H, C, device=dev, dtype=torch.bfloat16)
        gw = torch.empty(Co, R, R, C, device=dev, dtype=torch.float32)
        geo = (n, H, H, C, Co, R, R, H, H, 1, 1, R // 2, R // 2)
        flops = 2.0 * n * H * H * Co * R * R * C
        res = []
        for mode, a, b, o in ((1, x, w, y), (2, dy, w, dx), (3, x, dy, gw)):
            if str(mode) not in args.modes:
                res.append(float("nan"))
                continue
            with torch.cuda.stream(st):
                for _ in range(3):
                    xpipe.conv2d_bf16(mode, geo, a, b, o, accumulate=args.acc and mode == 3, ws=ws, stream=st.cuda_stream)
            st.synchronize()
            # GPU time: replay a CUDA graph of `iters` launches (host launch cost excluded)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cs = torch.cuda.current_stream().cuda_stream
                for _ in range(args.iters):
                    xpipe.conv2d_bf16(mode, geo, a, b, o, accumulate=args.acc and mode == 3, ws=ws, stream=cs)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.iters
            res.append(us)
            tot[mode] += us
            if args.check:
                xf, wf, dyf = x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), dy.float().permute(0, 3, 1, 2)
                if mode == 1:
                    ref = torch.nn.functional.conv2d(xf, wf, padding=R // 2).permute(0, 2, 3, 1)
                    got = o.float()
                elif mode == 2:
                    ref = torch.nn.grad.conv2d_input(xf.shape, wf, dyf, padding=R // 2).permute(0, 2, 3, 1)
                    got = o.float()
                else:
                    ref = torch.nn.grad.conv2d_weight(xf, wf.shape, dyf, padding=R // 2).permute(0, 2, 3, 1)
                    got = o
                err = ((got - ref).norm() / ref.norm().clamp_min(1e-30)).item()
                if err > 1e-2:
                    print("  MISMATCH mode %d relFrob %.3e" % (mode, err))
        flops_tot += flops
        print("%-22s %10.2f %10.2f %10.2f %8.1f %8.1f %8.1f" % (
            "%dx%d %d->%d" % (H, H, C, Co), res[0], res[1], res[2], flops / res[0] / 1e6, flops / res[1] / 1e6,
            flops / res[2] / 1e6))
    s = sum(tot.values())
    print("total us: fprop %.1f dgrad %.1f wgrad %.1f = %.1f us per micro-batch; %.1f TFLOP/s overall" % (
        tot[1], tot[2], tot[3], s, 3 * flops_tot / s / 1e6))


if __name__ == "__main__":
    main()
