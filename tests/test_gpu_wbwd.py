"""The bellwether-computed backward prediction (cfg.wbwd = XP_WBWD_BELLWETHER: the
backward bellwether B(t,1) predicts W_hat_b from the stage's current W, m, v and the other T-1
backwards reuse it) against the materialised one (the update sweep writes W_hat_b): the same
values, so the fp32 pipeline stays bit-exact with the oracle and the bf16 pipeline bit-identical
to the materialised run."""
import numpy as np
import pytest

import synthetic as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_fp32_bellwether_wbwd_bit_exact(oracle_mod):
    """Adam, fp32 contract: trace and weights bit-exact with the oracle's replay."""
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    K, T, N, M = 2, 4, 32, 6
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 1, kind="mnist")
    g = XPipe(L, K, T, N, 1e-3, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", trace=True,
              wbwd="bellwether", watchdog_ms=20000)
    o = oracle_mod.Oracle(L, K, T, N, 1e-3, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32")
    g.step(x, y, M, flush=True)
    o.step(x, y, M, flush=True)
    for k in range(K):
        assert g.trace(k) == o.trace(k)
    assert np.array_equal(g.params_flat(), o.params_flat().astype(np.float32))
    g.close()


def test_fp32_sgd_bellwether_wbwd_equals_materialized(oracle_mod):
    """f2 (Momentum SGD + paper-literal prediction, moments from 1e-4*U[0,1)): both modes give
    bit-identical parameters, velocities and moments."""
    from paper_1911_04610_b200 import XPipe
    from test_gpu_sgd import moment_tables
    L = S.mlp()
    P = S.make_params(L, 1)
    K, T, N, M, lr = 2, 4, 32, 6, 1e-2
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 1, kind="mnist")
    o0 = oracle_mod.Oracle(L, K, T, N, lr, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32", delta="paper",
                           optimizer="sgd")
    tm, tv = moment_tables(L, o0.count, 3)
    out = {}
    for mode in ("materialize", "bellwether"):
        g = XPipe(L, K, T, N, lr, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", delta="paper",
                  optimizer="sgd", momentum=0.9, weight_decay=5e-4, init_m=tm, init_v=tv, wbwd=mode,
                  watchdog_ms=20000)
        g.step(x, y, M, flush=True)
        out[mode] = [g.params_flat(st) for st in ("param", "buf", "m", "v")]
        g.close()
    for a, b in zip(out["materialize"], out["bellwether"]):
        assert np.array_equal(a, b)


def test_bf16_bellwether_wbwd_equals_materialized():
    from paper_1911_04610_b200 import XPipe
    from test_gpu_bf16 import vgg_small
    L = vgg_small()
    P = S.make_params(L, 1)
    K, T, N, M = 2, 2, 16, 6
    x, y = S.make_inputs(M * N, (3, 8, 8), 10, 1, kind="cifar")
    out = {}
    for mode in ("materialize", "bellwether"):
        g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (3, 8, 8), 10, params=P, precision="bf16", wbwd=mode,
                  fb_overlap=True, watchdog_ms=60000)
        g.step(x, y, M, flush=True)
        out[mode] = g.params_flat()
        g.close()
    assert np.array_equal(out["materialize"], out["bellwether"])
