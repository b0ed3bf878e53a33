"""BASELINE configs at their full sizes in the bench's launch configuration (all stages on one
GPU): ResNet-101 (configs[2]: K=8, N=256, T=8, 64x64) and Inception-V3 (configs[3]: K=4 and 8,
N=128, T=4).  The oracle cannot replay these trajectories in test time, so what the oracle fixes
at any size is checked: the schedule/version trace field by field (it depends on K, T and M
only -- replayed by the oracle on a K-layer MLP), W_hat_f / W_hat_b bit-exact against the
prediction evaluated from the GPU's own (W, m, v, version), finite losses that track the
oracle-free expectation ln(classes) at initialisation."""
import numpy as np
import pytest

import synthetic as S
from helpers import predict_from_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def schedule_oracle(oracle_mod, K, T, N, M):
    L = S.mlp(tuple([16] * K + [10]))
    P = S.make_params(L, 1)
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (16, 1, 1), 10, P, mode="fp32")
    x, y = S.make_inputs(M * N, (16, 1, 1), 10, 1, kind="gauss")
    o.step(x, y, M, flush=True)
    return o


@pytest.mark.parametrize("name,K,T,N,M", [("resnet101", 8, 8, 256, 2), ("inception", 4, 4, 128, 3),
                                          ("inception", 8, 4, 128, 3)])
def test_full_size_config(oracle_mod, name, K, T, N, M):
    from paper_1911_04610_b200 import XPipe
    from synthetic.models import resnet101, inception_v3, assign_stages
    L, units = resnet101(classes=200) if name == "resnet101" else inception_v3(classes=200)
    L = assign_stages(L, units, K)
    P = S.make_params(L, 1)
    x, y = S.make_inputs(M * N, (3, 64, 64), 200, 1, kind="imagenet")
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (3, 64, 64), 200, params=P, precision="bf16", trace=True,
              watchdog_ms=300000)
    losses = g.step(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), M, flush=True)
    assert np.all(np.isfinite(losses))
    assert abs(float(np.mean(losses[:T])) - np.log(200)) < 1.0  # first mini-batch near ln(classes)
    o = schedule_oracle(oracle_mod, K, T, N, M)
    for k in range(K):
        assert g.trace(k) == o.trace(k), k
        assert g.version(k) == M
    # W_hat self-consistency on the first weighted layer of every stage
    for k in range(K):
        sf = o.trace(k)[0][5]
        sb = next(r for r in o.trace(k) if r[1] == 1)[5]
        i = next(i for i in range(len(L)) if g.stage_of(i) == k and g._count(i, 0))
        W, m, v = (g.get(i, 0, st) for st in ("param", "m", "v"))
        for st, s in (("pred_fwd", sf), ("pred_bwd", sb)):
            ref = predict_from_state(W, m, v, g.version(k), s, 1e-4, 0.9, 0.999, 1e-8)
            assert np.array_equal(g.get(i, 0, st), ref), (k, i, st)
    g.close()
