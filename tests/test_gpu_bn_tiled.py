"""The exact-tiling max-pool fast path of the BN backward (bn_bwd_apply_tiled_kernel: one thread
per pooled output, kh == sh, kw == sw, no padding) must be bit-identical to the general routing
path (bn_bwd_apply_kernel), which the oracle parity tests cover.  The switch XPIPE_NO_BN_TILED is
read once per process, so both runs go through subprocesses on the same seeded inputs: the
VGG-16 blocks at CIFAR size (pools 32->16->8->4->2->1) and a small VGG at 8x8."""
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
from paper_1911_04610_b200 import XPipe
which = {which!r}
if which == "vgg16":
    L, shape, K, T, N, M = S.vgg16_cifar(), (3, 32, 32), 2, 2, 32, 4
else:
    from test_gpu_bf16 import vgg_small
    L, shape, K, T, N, M = vgg_small(), (3, 8, 8), 2, 2, 16, 6
P = S.make_params(L, 1)
x, y = S.make_inputs(M * N, shape, 10, 1, kind="cifar")
g = XPipe(L, K, T, N, 1e-3, (0.9, 0.999), 1e-8, shape, 10, params=P, precision="bf16", watchdog_ms=120000)
g.step(x, y, M, flush=True)
np.save({out!r}, g.params_flat())
g.close()
"""


def run(which, env_off, out):
    env = dict(os.environ)
    env.pop("XPIPE_NO_BN_TILED", None)
    if env_off:
        env["XPIPE_NO_BN_TILED"] = "1"
    code = RUN.format(root=ROOT, here=HERE, which=which, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("which", ["small", "vgg16"])
def test_tiled_pool_backward_bit_identical(tmp_path, which):
    fast = run(which, False, str(tmp_path / "fast.npy"))
    general = run(which, True, str(tmp_path / "general.npy"))
    assert fast.shape == general.shape
    assert np.array_equal(fast, general)
