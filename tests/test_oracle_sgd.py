"""Oracle pins for SURVEY 8f row f2: the paper's main-experiment optimizer (Momentum SGD,
momentum 0.9, weight decay 5e-4) with the prediction's moments tracked by Eq. (4)
and the literal Eq. (3)/(4) dW (constant bias corrections, eps inside the root),
moments optionally initialised to 1e-4*U[0,1).

Pinned against library routines (torch.optim.SGD for the training step, torch.optim.Adam's
exp_avg / exp_avg_sq for the Eq. (4) moment recurrences), the first-step closed form and
invariants of the prediction -- not against a retyped copy of the oracle's formulas.
"""
import numpy as np
import pytest
import torch

import synthetic as S
from test_oracle_numerics import TorchNet, NETS, BETAS32, EPS32

MU, WD = 0.9, 5e-4
MU32, WD32 = float(np.float32(MU)), float(np.float32(WD))


@pytest.fixture(autouse=True)
def _float64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def make(name, K=1, T=1, N=8, mode="fp64", predict="off", lr=1e-2, seed=3, **kw):
    import oracle
    build, shape, classes = NETS[name]
    L = build()
    P = S.make_params(L, seed)
    o = oracle.Oracle(L, K, T, N, lr, BETAS32, EPS32, shape, classes, P, mode=mode, predict=predict, delta="paper",
                      optimizer="sgd", momentum=MU, weight_decay=WD, **kw)
    return o, L, P, shape, classes


def stage_moment_init(o, L, seed):
    """1e-4 * U[0,1) per parameter, flattened per stage in layer order."""
    rng = np.random.default_rng(seed)
    per_stage = {}
    for i in range(len(L)):
        for t in (0, 1):
            n = o.count(i, t)
            if n:
                per_stage.setdefault(o.stage_of(i), []).append(n)
    init_m = [1e-4 * rng.random(sum(per_stage[k])) for k in sorted(per_stage)]
    init_v = [1e-4 * rng.random(sum(per_stage[k])) for k in sorted(per_stage)]
    return init_m, init_v


@pytest.mark.parametrize("name,T", [("mlp", 1), ("mlp", 4), ("cnn", 2), ("res", 2)])
def test_single_stage_s0_equals_torch_sgd(oracle_mod, name, T):
    """1 stage, s = 0: the training trajectory equals torch.optim.SGD(momentum=0.9,
    weight_decay=5e-4) in fp64 on the mini-batch-mean gradient accumulated over T micro-batches."""
    N, M, lr = 8, 5, 1e-2
    o, L, P, shape, classes = make(name, K=1, T=T, N=N, lr=lr)
    x, y = S.make_inputs(M * N, shape, classes, 9, kind="gauss")
    o.step(x, y, M, flush=True)
    net = TorchNet(L, P)
    opt = torch.optim.SGD(net.parameters(), lr=float(np.float32(lr)), momentum=MU32, weight_decay=WD32)
    n = N // T
    for t in range(M):
        opt.zero_grad()
        for j in range(T):
            sl = slice(t * N + j * n, t * N + (j + 1) * n)
            z = net(torch.tensor(x[sl], dtype=torch.float64))
            l = torch.nn.functional.cross_entropy(z, torch.tensor(y[sl], dtype=torch.long), reduction="sum") / N
            l.backward()
        opt.step()
    np.testing.assert_allclose(o.params_flat(), net.flat(), rtol=0, atol=1e-12)
    # the velocity buffer is torch's momentum_buffer
    buf = np.concatenate([opt.state[p]["momentum_buffer"].detach().numpy().ravel() for p in net.w])
    np.testing.assert_allclose(o.params_flat("buf"), buf, rtol=0, atol=1e-12)


def test_prediction_moments_are_exponential_averages(oracle_mod):
    """Eq. (4): v_t (first moment, gamma) and m_t (second raw moment, lambda) are the
    exponential moving averages torch.optim.Adam keeps as exp_avg / exp_avg_sq, from the given
    initial values 1e-4*U[0,1), over the SGD trajectory's gradients."""
    N, M, T, lr = 8, 4, 2, 1e-2
    o0, L, P, shape, classes = make("mlp", K=1, T=T, N=N, lr=lr)
    init_m, init_v = stage_moment_init(o0, L, 5)
    o, *_ = make("mlp", K=1, T=T, N=N, lr=lr, init_m=init_m, init_v=init_v)
    x, y = S.make_inputs(M * N, shape, classes, 11, kind="gauss")
    o.step(x, y, M, flush=True)
    net = TorchNet(L, P)
    sgd = torch.optim.SGD(net.parameters(), lr=float(np.float32(lr)), momentum=MU32, weight_decay=WD32)
    # a shadow parameter per tensor, stepped by Adam on the same raw gradients (R26: Eq. (4)'s
    # g_t is the stochastic gradient, without the weight-decay term)
    shadow = [torch.nn.Parameter(p.detach().clone()) for p in net.w]
    adam = torch.optim.Adam(shadow, lr=1.0, betas=BETAS32, eps=EPS32)
    off = 0
    for p, q in zip(net.w, shadow):
        k = p.numel()
        adam.state[q] = {"step": torch.tensor(0.0), "exp_avg": torch.tensor(init_m[0][off:off + k]).reshape(p.shape),
                         "exp_avg_sq": torch.tensor(init_v[0][off:off + k]).reshape(p.shape)}
        off += k
    n = N // T
    for t in range(M):
        sgd.zero_grad()
        for j in range(T):
            sl = slice(t * N + j * n, t * N + (j + 1) * n)
            z = net(torch.tensor(x[sl], dtype=torch.float64))
            l = torch.nn.functional.cross_entropy(z, torch.tensor(y[sl], dtype=torch.long), reduction="sum") / N
            l.backward()
        for p, q in zip(net.w, shadow):
            q.grad = p.grad.detach().clone()
        adam.step()
        sgd.step()
    ea = np.concatenate([adam.state[q]["exp_avg"].detach().numpy().ravel() for q in shadow])
    eq = np.concatenate([adam.state[q]["exp_avg_sq"].detach().numpy().ravel() for q in shadow])
    np.testing.assert_allclose(o.params_flat("m"), ea, rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(o.params_flat("v"), eq, rtol=1e-12, atol=1e-18)


def test_sgd_sweep_first_step_closed_form(oracle_mod):
    """From zero moments the first tracked moments are (1-gamma) g and (1-lambda) g^2, so the
    bias-corrected dW of Eq. (3)/(4) is exactly lr * g / sqrt(g^2 + eps); the training step is
    torch.optim.SGD's first step (velocity = g + wd*W)."""
    rng = np.random.default_rng(1)
    n = 4096
    W = rng.uniform(-0.05, 0.05, n).astype(np.float32)
    g = rng.uniform(-1e-2, 1e-2, n).astype(np.float32)
    z = np.zeros(n, np.float32)
    lr = float(np.float32(1e-2))
    W1, buf1, m1, v1, pf, pb = oracle_mod.sgd_predict(W, g, z, z, z, lr, BETAS32, EPS32, MU32, WD32, 2, 1,
                                                      mode="fp64")
    p = torch.nn.Parameter(torch.tensor(W.astype(np.float64)))
    opt = torch.optim.SGD([p], lr=lr, momentum=MU32, weight_decay=WD32)
    p.grad = torch.tensor(g.astype(np.float64))
    opt.step()
    np.testing.assert_allclose(W1, p.detach().numpy().astype(np.float32), rtol=0, atol=0)
    np.testing.assert_allclose(buf1, opt.state[p]["momentum_buffer"].numpy().astype(np.float32), rtol=0, atol=0)
    g64 = g.astype(np.float64)
    d = lr * g64 / np.sqrt(g64 * g64 + EPS32)
    np.testing.assert_allclose(pb.astype(np.float64), (W1.astype(np.float64) - d).astype(np.float32), rtol=0,
                               atol=8e-9)  # two float32 ulps at |W| <= 0.06 (rounding of W' first)
    np.testing.assert_allclose(pf.astype(np.float64), (W1.astype(np.float64) - 2 * d).astype(np.float32), rtol=0,
                               atol=8e-9)  # two float32 ulps at |W| <= 0.06 (rounding of W' first)


def test_sgd_sweep_prediction_invariants(oracle_mod):
    """W_hat - W' = -s*dW: linear in s, W_hat = W' at s = 0, and it moves W against the tracked
    first moment (sign); fp32 mode agrees with fp64 to rounding."""
    rng = np.random.default_rng(2)
    n = 8192
    W = rng.uniform(-0.05, 0.05, n).astype(np.float32)
    g = rng.uniform(-1e-2, 1e-2, n).astype(np.float32)
    buf = (0.1 * rng.uniform(-1e-2, 1e-2, n)).astype(np.float32)
    m = (0.1 * rng.uniform(-1e-2, 1e-2, n)).astype(np.float32)
    v = rng.uniform(1e-6, 1e-4, n).astype(np.float32)
    lr = float(np.float32(1e-2))
    r64 = oracle_mod.sgd_predict(W, g, buf, m, v, lr, BETAS32, EPS32, MU32, WD32, 4, 0, mode="fp64")
    W1, buf1, m1, v1, p4, p0 = (a.astype(np.float64) for a in r64)
    np.testing.assert_array_equal(p0, W1)
    r2 = oracle_mod.sgd_predict(W, g, buf, m, v, lr, BETAS32, EPS32, MU32, WD32, 2, 0, mode="fp64")
    p2 = r2[4].astype(np.float64)
    np.testing.assert_allclose(p4 - W1, 2 * (p2 - W1), rtol=1e-5, atol=8e-9)  # outputs rounded to float32
    nz = np.abs(m1) > 1e-6
    assert np.all(np.sign(W1 - p4)[nz] == np.sign(m1)[nz])
    r32 = oracle_mod.sgd_predict(W, g, buf, m, v, lr, BETAS32, EPS32, MU32, WD32, 4, 0, mode="fp32")
    for a, b in zip(r32, r64):
        np.testing.assert_allclose(a.astype(np.float64), b.astype(np.float64), rtol=2e-6, atol=1e-9)


@pytest.mark.parametrize("K", [2, 3])
def test_sgd_gpipe_no_prediction_equals_single_stage(oracle_mod, K):
    """P6 for the SGD optimizer: the GPipe schedule with s = 0 equals K = 1 bit-exactly in the
    fp32 mode (stage placement changes no per-layer op order)."""
    N, M, T = 8, 3, 2
    res = []
    for k in (1, K):
        o, L, P, shape, classes = make("mlp", K=k, T=T, N=N, mode="fp32", schedule="gpipe")
        x, y = S.make_inputs(M * N, shape, classes, 6, kind="gauss")
        o.step(x, y, M, flush=True)
        res.append((o.params_flat(), o.params_flat("buf"), o.params_flat("m"), o.params_flat("v")))
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)


def test_sgd_requires_paper_delta(oracle_mod):
    import oracle
    build, shape, classes = NETS["mlp"]
    L = build()
    with pytest.raises(oracle.OracleError):
        oracle.Oracle(L, 1, 1, 8, 1e-2, BETAS32, EPS32, shape, classes, S.make_params(L, 1), optimizer="sgd")
