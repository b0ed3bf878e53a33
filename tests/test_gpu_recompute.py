"""GPU parity of SURVEY 8f row f3 (cfg.recompute): every backward first re-runs the stage
forward under W_hat_b from the stashed stage input.  fp32 MLP pipeline bit-exact with
the oracle's recompute replay (weights after every version, trace); bf16 conv pipeline within
the north-star tolerance."""
import numpy as np
import pytest

import synthetic as S
from helpers import rel_frob

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,T", [(2, 4), (3, 1)])
def test_recompute_mlp_bit_exact(oracle_mod, K, T):
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    N, M, lr = 32, 6, 1e-3
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 2, kind="mnist")
    g = XPipe(L, K, T, N, lr, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", recompute=True,
              trace=True, snapshots=True, watchdog_ms=60000)
    o = oracle_mod.Oracle(L, K, T, N, lr, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32", recompute=True,
                          snapshots=True)
    lg = g.step(x, y, M, flush=True)
    lo = o.step(x, y, M, flush=True)
    for k in range(K):
        assert g.trace(k) == o.trace(k), k
    for v in range(M + 1):
        assert np.array_equal(g.params_flat("param", v), o.params_flat("param", v).astype(np.float32)), v
    assert np.array_equal(lg, lo)  # the reported loss is the forward's, not the recompute's
    g.close()


def test_recompute_bf16_conv(oracle_mod):
    from paper_1911_04610_b200 import XPipe
    from test_gpu_bf16 import vgg_small
    L = vgg_small()
    P = S.make_params(L, 1)
    K, T, N, M, lr = 2, 2, 16, 8, 1e-4
    x, y = S.make_inputs(M * N, (3, 8, 8), 10, 1, kind="cifar")
    g = XPipe(L, K, T, N, lr, (0.9, 0.999), 1e-8, (3, 8, 8), 10, params=P, precision="bf16", recompute=True,
              trace=True, watchdog_ms=60000)
    o = oracle_mod.Oracle(L, K, T, N, lr, (0.9, 0.999), 1e-8, (3, 8, 8), 10, P, mode="bf16", recompute=True)
    g.step(x, y, M, flush=True)
    o.step(x, y, M, flush=True)
    for k in range(K):
        assert g.trace(k) == o.trace(k), k
    assert rel_frob(g.params_flat(), o.params_flat()) <= 2e-2
    g.close()
