#!/usr/bin/env python
"""Per-CTA phase timing of one conv GEMM launch (development tool; needs XPIPE_GEMM_DBG=1).

  XPIPE_GEMM_DBG=1 python scripts/gemm_probe.py --layer 1 --mode 1
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_04610_b200 import xpipe  # noqa: E402
from conv_bench import VGG  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", type=int, default=1)
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--batch", type=int, default=32)
    args = ap.parse_args()
    assert os.environ.get("XPIPE_GEMM_DBG") == "1"
    dev = torch.device("cuda:0")
    H, Cc, Co, R = VGG[args.layer]
    n = args.batch
    x = torch.randn(n, H, H, Cc, device=dev).to(torch.bfloat16)
    w = (torch.randn(Co, R, R, Cc, device=dev) * 0.05).to(torch.bfloat16)
    dy = torch.randn(n, H, H, Co, device=dev).to(torch.bfloat16)
    out = {1: torch.empty(n, H, H, Co, device=dev, dtype=torch.bfloat16),
           2: torch.empty(n, H, H, Cc, device=dev, dtype=torch.bfloat16),
           3: torch.empty(Co, R, R, Cc, device=dev, dtype=torch.float32)}[args.mode]
    ins = {1: (x, w), 2: (dy, w), 3: (x, dy)}[args.mode]
    ws = torch.zeros((16 << 20) + (1 << 14), device=dev)
    geo = (n, H, H, Cc, Co, R, R, H, H, 1, 1, R // 2, R // 2)
    lib = xpipe.lib()
    for it in range(3):
        xpipe.conv2d_bf16(args.mode, geo, ins[0], ins[1], out, ws=ws)
        torch.cuda.synchronize()
    buf = (C.c_ulonglong * (16 * 65536))()
    assert lib.xpipe_dev_gemm_probe(buf, 16 * 65536) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 16).astype(np.int64)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    st, ff, mm, acc, end = (a[:, i] - t0 for i in range(5))
    print("layer %d mode %d: %d CTAs, span %.2f us" % (args.layer, args.mode, len(a), (end.max()) / 1e3))
    for name, v in (("start", st), ("first stage", ff), ("mma issued", mm), ("acc ready", acc), ("end", end),
                    ("first-start", ff - st), ("mma-first", mm - ff), ("acc-mma", acc - mm), ("end-acc", end - acc)):
        print("  %-12s min %7.2f med %7.2f max %7.2f us" % (name, v.min() / 1e3, np.median(v) / 1e3, v.max() / 1e3))
    if a[:, 8].max() > 0:
        park, cs1, red, xcl = (a[:, i] - t0 for i in (7, 8, 9, 10))
        for name, v in (("park-acc", park - acc), ("csync-park", cs1 - park), ("reduce", red - cs1),
                        ("xcluster", xcl - red), ("end-xcl", end - xcl)):
            print("  %-12s min %7.2f med %7.2f max %7.2f us" % (name, v.min() / 1e3, np.median(v) / 1e3, v.max() / 1e3))
    if a[:, 8].max() > 0:
        park, cs1, red, xcl = (a[:, i] - t0 for i in (7, 8, 9, 10))
        for name, v in (("park-acc", park - acc), ("csync-park", cs1 - park), ("reduce", red - cs1),
                        ("xcluster", xcl - red), ("end-xcl", end - xcl)):
            print("  %-12s min %7.2f med %7.2f max %7.2f us" % (name, v.min() / 1e3, np.median(v) / 1e3, v.max() / 1e3))
    print("  units/CTA:", np.bincount(a[:, 6])[1:] if a[:, 6].max() > 0 else "-", " distinct SMs:", len(set(a[:, 5])))


if __name__ == "__main__":
    main()
