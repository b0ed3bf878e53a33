"""GPU parity of SURVEY 8f row f2 (XP_OPT_MOMENTUM_SGD): the paper's Momentum-SGD training
 with the Eq. (4) moments tracked alongside and the literal Eq. (3)/(4) prediction,
moments initialised to 1e-4*U[0,1).  fp32 MLP pipeline bit-exact with the oracle
(weights, velocity, moments, trace); the f2 sweep bit-exact element by element; a bf16 conv
pipeline within the north-star tolerance with its W_hat buffers bit-exact against the paper
prediction evaluated from the GPU's own state."""
import numpy as np
import pytest

import synthetic as S
from helpers import bf16_round, rel_frob

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

B32 = (float(np.float32(0.9)), float(np.float32(0.999)))
E32 = float(np.float32(1e-8))
MU, WD = float(np.float32(0.9)), float(np.float32(5e-4))


def moment_tables(L, count, seed):
    """per-(layer, tensor) 1e-4*U[0,1) arrays (GPU binding layout) and the oracle's per-stage
    flattened copy (layer order, weight then bias)."""
    rng = np.random.default_rng(seed)
    tm, tv = [], []
    for i in range(len(L)):
        pair_m, pair_v = [], []
        for t in (0, 1):
            n = count(i, t)
            pair_m.append((1e-4 * rng.random(n)).astype(np.float32) if n else None)
            pair_v.append((1e-4 * rng.random(n)).astype(np.float32) if n else None)
        tm.append(pair_m)
        tv.append(pair_v)
    return tm, tv


def stage_flat(tab, L, stage_of, K):
    out = [[] for _ in range(K)]
    for i in range(len(L)):
        for t in (0, 1):
            if tab[i][t] is not None:
                out[stage_of(i)].append(tab[i][t].astype(np.float64))
    return [np.concatenate(o) for o in out]


@pytest.mark.parametrize("n,bf", [(4099, True), (4099, False), (1 << 20, True)])
def test_sgd_sweep_bit_exact(oracle_mod, n, bf):
    from paper_1911_04610_b200 import sgd_predict
    rng = np.random.default_rng(7)
    W = rng.uniform(-0.05, 0.05, n).astype(np.float32)
    g = rng.uniform(-1e-2, 1e-2, n).astype(np.float32)
    buf = (0.1 * rng.uniform(-1e-2, 1e-2, n)).astype(np.float32)
    m = (0.1 * rng.uniform(-1e-2, 1e-2, n)).astype(np.float32)
    v = rng.uniform(1e-6, 1e-4, n).astype(np.float32)
    lr = float(np.float32(1e-2))
    ref = oracle_mod.sgd_predict(W, g, buf, m, v, lr, B32, E32, MU, WD, 3, 1, mode="fp32")
    t = [torch.from_numpy(a.copy()).cuda() for a in (W, g, buf, m, v)]
    dt = torch.bfloat16 if bf else torch.float32
    pf = torch.empty(n, dtype=dt, device="cuda")
    pb = torch.empty(n, dtype=dt, device="cuda")
    sgd_predict(t[0], t[1], t[2], t[3], t[4], pf, pb, lr, B32, E32, MU, WD, 3, 1, bf)
    torch.cuda.synchronize()
    got = [t[0], t[2], t[3], t[4], pf.float(), pb.float()]
    want = list(ref[:4]) + [bf16_round(ref[4]) if bf else ref[4], bf16_round(ref[5]) if bf else ref[5]]
    for name, a, b in zip(("W", "buf", "m", "v", "pf", "pb"), got, want):
        assert np.array_equal(a.cpu().numpy(), b), name


def test_sgd_mlp_pipeline_bit_exact(oracle_mod):
    """Config-1 MLP, 2 stages, T=4, Momentum SGD (lr 1e-2) with the paper moment init: the
    trace and every stage's W, velocity and moments equal the oracle's fp32 replay bit for bit."""
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    K, T, N, M, lr = 2, 4, 32, 6, 1e-2
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 1, kind="mnist")
    o0 = oracle_mod.Oracle(L, K, T, N, lr, B32, E32, (784, 1, 1), 10, P, mode="fp32", delta="paper",
                           optimizer="sgd", momentum=MU, weight_decay=WD)
    tm, tv = moment_tables(L, o0.count, 3)
    stage_of = o0.stage_of
    g = XPipe(L, K, T, N, lr, B32, E32, (784, 1, 1), 10, params=P, precision="fp32", delta="paper",
              optimizer="sgd", momentum=MU, weight_decay=WD, trace=True, snapshots=True, watchdog_ms=60000,
              init_m=tm, init_v=tv)
    o = oracle_mod.Oracle(L, K, T, N, lr, B32, E32, (784, 1, 1), 10, P, mode="fp32", delta="paper",
                          optimizer="sgd", momentum=MU, weight_decay=WD, snapshots=True,
                          init_m=stage_flat(tm, L, stage_of, K), init_v=stage_flat(tv, L, stage_of, K))
    g.step(x, y, M, flush=True)
    o.step(x, y, M, flush=True)
    for k in range(K):
        assert g.trace(k) == o.trace(k), k
    for state in ("param", "buf", "m", "v"):
        a, b = g.params_flat(state), o.params_flat(state).astype(np.float32)
        assert np.array_equal(a, b), state
    for v in range(M + 1):
        assert np.array_equal(g.params_flat("param", v), o.params_flat("param", v).astype(np.float32)), v
    g.close()


def test_sgd_bf16_conv_pipeline(oracle_mod):
    """bf16 conv blocks on tcgen05 under Momentum SGD (lr 1e-3): weights within the north-star
    relative-Frobenius bar of the oracle's bf16 emulation, trace bit-exact, and both W_hat
    buffers bit-exact against Eq. (3)/(4) evaluated from the GPU's own W, m, v."""
    from paper_1911_04610_b200 import XPipe
    from test_gpu_bf16 import vgg_small
    L = vgg_small()
    P = S.make_params(L, 1)
    K, T, N, M, lr = 2, 2, 16, 6, 1e-3
    x, y = S.make_inputs(M * N, (3, 8, 8), 10, 1, kind="cifar")
    g = XPipe(L, K, T, N, lr, B32, E32, (3, 8, 8), 10, params=P, precision="bf16", delta="paper", optimizer="sgd",
              momentum=MU, weight_decay=WD, trace=True, watchdog_ms=60000)
    o = oracle_mod.Oracle(L, K, T, N, lr, B32, E32, (3, 8, 8), 10, P, mode="bf16", delta="paper", optimizer="sgd",
                          momentum=MU, weight_decay=WD)
    g.step(x, y, M, flush=True)
    o.step(x, y, M, flush=True)
    for k in range(K):
        assert g.trace(k) == o.trace(k), k
    assert rel_frob(g.params_flat(), o.params_flat()) <= 2e-2
    lr32 = np.float32(lr)
    for k in range(K):
        sf = o.trace(k)[0][5]
        sb = next(r for r in o.trace(k) if r[1] == 1)[5]
        for i in range(len(L)):
            if g.stage_of(i) != k:
                continue
            for t in (0, 1):
                n = g._count(i, t)
                if not n:
                    continue
                W, m, v = (g.get(i, t, st) for st in ("param", "m", "v"))
                # Eq. (3)/(4), fp32 op order of the sweep: d = lr*(m*inv1)/sqrt(v*inv2 + eps)
                inv1 = np.float32(1.0 / (1.0 - B32[0]))
                inv2 = np.float32(1.0 / (1.0 - B32[1]))
                d = (lr32 * (m * inv1)) / np.sqrt(v * inv2 + np.float32(E32))
                for st, s in (("pred_fwd", sf), ("pred_bwd", sb)):
                    ref = bf16_round((-(float(s)) * d.astype(np.float64) + W.astype(np.float64)).astype(np.float32))
                    assert np.array_equal(g.get(i, t, st), ref), (k, i, t, st)
    g.close()
