"""Dump the parameters after a short seeded bf16 pipeline run (VGG-16 CIFAR blocks, K=2, T=2,
N=32, 4 mini-batches) -- used to check that a kernel change is bit-identical across two builds
(scripts/gpu_ab_so.sh swaps the library between runs)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic as S  # noqa: E402
from paper_1911_04610_b200 import XPipe  # noqa: E402

L, shape, K, T, N, M = S.vgg16_cifar(), (3, 32, 32), 2, 2, 32, 4
P = S.make_params(L, 1)
x, y = S.make_inputs(M * N, shape, 10, 1, kind="cifar")
g = XPipe(L, K, T, N, 1e-3, (0.9, 0.999), 1e-8, shape, 10, params=P, precision="bf16", watchdog_ms=120000)
g.step(x, y, M, flush=True)
np.save(sys.argv[1], g.params_flat())
g.close()
