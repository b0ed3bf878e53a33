#!/usr/bin/env python
"""Summarise a gpu_f1.sh run (gpurun_out/<run>/*.json) into profiles/<run>_f1.md: XPipe vs
GPipe-flush samples/s per (model, K, T), the ratio, the timed run's bubble fraction from
xpipe_stats, and the uniform-cost ideals (XPipe (K-1)/(MT+K-1), GPipe (K-1)/(T+K-1)).
usage: python scripts/f1_summary.py gpurun_out/r02f profiles/r02f_f1.md"""
import glob
import json
import os
import re
import sys

PAPER = {"inception": "+20.0 % avg (up to +31.9 %) on 2 GPUs, +88.1 % avg (up to +150.8 %) on 4 GPUs",
         "resnet101": "+10.8 % avg (up to +21.2 %) on 2 GPUs, +84.6 % avg (up to +142.7 %) on 4 GPUs"}


def main(src, dst):
    rows = {}
    for f in sorted(glob.glob(os.path.join(src, "*_K*_T*_*.json"))):
        m = re.match(r"(\w+?)_K(\d+)_T(\d+)_(xpipe|gpipe)\.json", os.path.basename(f))
        if not m:
            continue
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
        except Exception:
            continue
        model, K, T, sch = m.group(1), int(m.group(2)), int(m.group(3)), m.group(4)
        b = d.get("bubble") or {}
        rows[(model, K, T, sch)] = (d["value"], b.get("bubble_fraction"), d["config"]["minibatches_per_step"],
                                    d["config"]["global_batch"])
    out = ["# f1: XPipe vs GPipe-flush on the paper's throughput grid (P:338, P:394)", "",
           "Inception-V3 and ResNet-101 on synthetic Tiny-ImageNet upscaled to 224x224 (P:161), K in {2, 4},",
           "T in {1, 2, 4}, mini-batch 50T (K=2) / 100T (K=4), Adam; GPipe = the same kernels with the",
           "flush schedule and prediction off.  One B200: all K stages share the GPU (the paper used one GPU",
           "per stage), so an idle stage's SMs are used by the others and the GPipe bubble costs less",
           "throughput than on K GPUs; the bubble column is the per-stage idle fraction of the timed run",
           "(xpipe_stats: 1 - sum busy_k / (K span)), which is the schedule property the paper argues about.", "",
           "| model | K | T | N | XPipe samples/s | GPipe samples/s | XPipe/GPipe | bubble XPipe | bubble GPipe | ideal XPipe | ideal GPipe |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    ratios = {}
    for (model, K, T) in sorted({k[:3] for k in rows}):
        x = rows.get((model, K, T, "xpipe"))
        g = rows.get((model, K, T, "gpipe"))
        if not x or not g:
            continue
        M = x[2]
        ix = (K - 1) / (M * T + K - 1)
        ig = (K - 1) / (T + K - 1)
        r = x[0] / g[0]
        ratios.setdefault((model, K), []).append(r)
        fb = lambda v: "-" if v is None else "%.3f" % v
        out.append("| %s | %d | %d | %d | %.0f | %.0f | %.3f | %s | %s | %.3f | %.3f |" %
                   (model, K, T, x[3], x[0], g[0], r, fb(x[1]), fb(g[1]), ix, ig))
    out += ["", "| model | K | mean XPipe/GPipe over T | max | paper (V100s, one stage per GPU) |", "|---|---|---|---|---|"]
    for (model, K), rs in sorted(ratios.items()):
        out.append("| %s | %d | %.3f | %.3f | %s |" % (model, K, sum(rs) / len(rs), max(rs), PAPER.get(model, "")))
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
