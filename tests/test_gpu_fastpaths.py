"""Fast paths that must be bit-identical to the general path they replace (which the oracle
parity tests cover).  Each switch is read once per process, so both runs go through
subprocesses on the same seeded inputs:
  * XPIPE_NO_ADD_FUSE=1 -- the residual Add folded into the preceding conv block's BN-apply
    (forward: relu?(Q(Q(BN(conv)) + residual)); backward: the residual gradient emitted by the
    BN-backward reduction) vs the separate Add op: ResNet blocks (identity and downsample
    shortcuts, stage cuts inside the network), K=3, with CUDA graphs and fb_overlap;
  * XPIPE_NO_CONCAT_VIEWS=1 -- Inception's channel concats eliminated (conv blocks and pooling
    ops store in place at their channel offset, their backward reads the gradient slice) vs
    the copy ops: the full Inception-V3 at 64x64 (four-way chains, the nested 1x3 / 3x1 concats
    of Mixed_7, max-pool branches of the reductions), K=3;
  * XPIPE_BN_FUSE=1 (opt-in) -- the BatchNorm statistics and BN-apply [+ residual] [+ ReLU] in the
    fprop GEMM's epilogue (the M tiles of an N tile as one thread-block cluster, partials over
    DSMEM) vs the separate statistics-merge and apply launches: VGG-16 at CIFAR size K=2 (its
    unpooled 8x8 / 4x4 layers), the ResNet blocks (residual blocks at 4x4 / 2x2) and Inception;
  * XPIPE_BN_FA=1 (opt-in) -- for layers of at most 2048 rows, the BatchNorm final merge and the elementwise
    pass as one launch with one block per 8 channels (forward: statistics merge + BN-apply
    [+ residual] [+ ReLU] [+ pool]; backward: totals merge + dgamma/dbeta + input gradient,
    pooled tiled / general / unpooled) vs the two launches: VGG-16, ResNet blocks, Inception;
  * XPIPE_NO_POOL_VEC=1 -- the standalone max / average pools (Inception's branch and reduction
    pools) 8 channels per thread vs one element per thread: Inception."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

RUN = r"""
import sys, numpy as np
sys.path[:0] = [{root!r}, {here!r}]
import synthetic as S
from synthetic.models import resnet101, inception_v3, assign_stages
from paper_1911_04610_b200 import XPipe
which = {which!r}
if which == "vgg16":
    L, shape, K, T, N, calls, kind = S.vgg16_cifar(), (3, 32, 32), 2, 2, 64, (3, 3, 3), "cifar"
elif which == "resnet":
    L, units = resnet101(classes=10, layers=(2, 2, 2, 1))
    L, shape, K, T, N, calls, kind = assign_stages(L, units, 3), (3, 32, 32), 3, 2, 16, (3, 3, 3), "imagenet"
else:
    L, units = inception_v3(classes=10)
    L, shape, K, T, N, calls, kind = assign_stages(L, units, 3), (3, 64, 64), 3, 2, 16, (2, 2), "imagenet"
P = S.make_params(L, 1)
M = sum(calls)
x, y = S.make_inputs(M * N, shape, 10, 1, kind=kind)
g = XPipe(L, K, T, N, 1e-3, (0.9, 0.999), 1e-8, shape, 10, params=P, precision="bf16", watchdog_ms=120000,
          graphs=True, fb_overlap=True)
b = 0
for i, m in enumerate(calls):
    g.step(x[b * N:(b + m) * N], y[b * N:(b + m) * N], m, flush=(i == len(calls) - 1))
    b += m
np.save({out!r}, g.params_flat())
g.close()
"""


def run(which, env_set, out):
    env = dict(os.environ)
    for k in ("XPIPE_NO_ADD_FUSE", "XPIPE_NO_CONCAT_VIEWS", "XPIPE_BN_FUSE", "XPIPE_BN_FOLD", "XPIPE_BN_FA",
              "XPIPE_NO_POOL_VEC"):
        env.pop(k, None)
    if env_set:
        k, v = env_set.split("=")
        env[k] = v
    code = RUN.format(root=ROOT, here=HERE, which=which, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


# (environment of the fast path, of the general path, model)
CASES = [("", "XPIPE_NO_ADD_FUSE=1", "resnet"), ("", "XPIPE_NO_CONCAT_VIEWS=1", "inception"),
         ("XPIPE_BN_FUSE=1", "", "vgg16"), ("XPIPE_BN_FUSE=1", "", "resnet"), ("XPIPE_BN_FUSE=1", "", "inception"),
         ("XPIPE_BN_FA=1", "", "vgg16"), ("XPIPE_BN_FA=1", "", "resnet"), ("XPIPE_BN_FA=1", "", "inception"),
         ("", "XPIPE_NO_POOL_VEC=1", "inception")]


@pytest.mark.parametrize("fast_env,general_env,which", CASES)
def test_fast_path_bit_identical(tmp_path, fast_env, general_env, which):
    fast = run(which, fast_env, str(tmp_path / "fast.npy"))
    general = run(which, general_env, str(tmp_path / "general.npy"))
    assert fast.shape == general.shape
    assert np.isfinite(fast).all()
    assert np.array_equal(fast, general)
