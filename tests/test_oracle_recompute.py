"""Oracle pins for SURVEY 8f row f3: activation recomputation -- the backward re-runs
the stage forward under W_hat_b from the stashed stage input and differentiates it.  Pinned by
torch autograd at W_hat_b (the exact VJP), by the special case W_hat_f = W_hat_b (identical to
stash mode, bit for bit) and by GPipe(s=0) = K=1."""
import numpy as np
import pytest
import torch

import synthetic as S
from test_oracle_numerics import TorchNet, NETS, BETAS32, EPS32


@pytest.fixture(autouse=True)
def _float64_default():
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


def make(name, K=1, T=1, N=8, mode="fp64", lr=1e-3, seed=3, **kw):
    import oracle
    build, shape, classes = NETS[name]
    L = build()
    P = S.make_params(L, seed)
    o = oracle.Oracle(L, K, T, N, lr, BETAS32, EPS32, shape, classes, P, mode=mode, **kw)
    return o, L, P, shape, classes


@pytest.mark.parametrize("name", ["mlp", "cnn", "res"])
def test_recompute_gradient_is_autograd_at_w_hat_b(oracle_mod, name):
    """K=1, s_f = 2 != s_b = 1: the mini-batch gradient of the second mini-batch equals torch
    autograd of the loss at the backward's predicted weights W_hat_b (read from the oracle
    between the two calls); stash mode differs (activations from W_hat_f)."""
    N = 8
    kw = dict(K=1, T=1, N=N, predict="fixed", s_fwd=2, s_bwd=1)
    o, L, P, shape, classes = make(name, recompute=True, **kw)
    x, y = S.make_inputs(2 * N, shape, classes, 5, kind="gauss")
    o.step(x[:N], y[:N], 1, flush=True)
    wb = [(o.get(i, 0, "pred_bwd") if o.count(i, 0) else None, o.get(i, 1, "pred_bwd") if o.count(i, 1) else None)
          for i in range(len(L))]
    wf = o.params_flat("pred_fwd")
    o.step(x[N:], y[N:], 1, flush=True)
    g = o.params_flat("grad")
    P_b = []
    for i, l in enumerate(L):
        w = wb[i][0].reshape(np.shape(P[i][0])) if wb[i][0] is not None else None
        b = wb[i][1].reshape(np.shape(P[i][1])) if wb[i][1] is not None else None
        P_b.append((w, b))
    net = TorchNet(L, P_b)
    z = net(torch.tensor(x[N:], dtype=torch.float64))
    torch.nn.functional.cross_entropy(z, torch.tensor(y[N:], dtype=torch.long)).backward()
    np.testing.assert_allclose(g, net.flat_grad(), rtol=1e-9, atol=1e-14)
    assert not np.allclose(wf, np.concatenate([a.ravel() for pair in wb for a in pair if a is not None]))
    # stash mode on the same inputs differs (forward activations under W_hat_f)
    o2, *_ = make(name, recompute=False, **kw)
    o2.step(x[:N], y[:N], 1, flush=True)
    o2.step(x[N:], y[N:], 1, flush=True)
    assert not np.allclose(o2.params_flat("grad"), g, rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
def test_recompute_equals_stash_when_predictions_coincide(oracle_mod, mode):
    """One stage (forward and backward of a mini-batch at the same version) with s_f = s_b:
    W_hat_f = W_hat_b, so recomputing the forward reproduces the stash and the trajectory is
    bit-identical to stash mode."""
    res = []
    for rc in (False, True):
        o, L, P, shape, classes = make("res", K=1, T=2, N=8, mode=mode, predict="fixed", s_fwd=1, s_bwd=1,
                                       recompute=rc)
        x, y = S.make_inputs(4 * 8, shape, classes, 6, kind="gauss")
        o.step(x, y, 4, flush=True)
        res.append((o.params_flat(), o.trace(0)))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    assert res[0][1:] == res[1][1:]


@pytest.mark.parametrize("K", [2, 3])
def test_recompute_gpipe_no_prediction_equals_single_stage(oracle_mod, K):
    """P6 with recomputation: GPipe, s = 0, K stages = K = 1 bit-exactly (fp32)."""
    out = []
    for k in (1, K):
        o, *_, shape, classes = make("mlp", K=k, T=2, N=8, mode="fp32", schedule="gpipe", predict="off",
                                     recompute=True)
        x, y = S.make_inputs(3 * 8, shape, classes, 7, kind="gauss")
        o.step(x, y, 3, flush=True)
        out.append(o.params_flat())
    np.testing.assert_array_equal(out[0], out[1])
