"""Oracle pins for the arithmetic: layer maths, Adam, the prediction sweep, bf16 rounding.

Pinned against library routines (torch autograd, torch.optim.Adam, torch bf16 casts),
central finite differences, closed forms and a hand-worked example -- never against a
retyped copy of the oracle's own formulas.
"""
import os

import numpy as np
import pytest
import torch

import synthetic as S
from synthetic.models import conv, bn, relu, maxpool, linear, xent, Layer, FLATTEN, AVGPOOL_GLOBAL, ADD, CONCAT

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BETAS32 = (float(np.float32(0.9)), float(np.float32(0.999)))
EPS32 = float(np.float32(1e-8))


@pytest.fixture(autouse=True)
def _float64_default():
    """fp64 torch twins for this module only (a module-level set_default_dtype would leak into
    every test module collected after this one, e.g. the GPU tests' fp32 buffers)."""
    old = torch.get_default_dtype()
    torch.set_default_dtype(torch.float64)
    yield
    torch.set_default_dtype(old)


# ----------------------------------------------------------------------------- torch twin
class TorchNet(torch.nn.Module):
    """The same layer list as a torch module (library reference for the layer maths)."""

    def __init__(self, layers, params):
        super().__init__()
        self.layers = layers
        self.w = torch.nn.ParameterList()
        self.idx = {}
        for i, (l, (w, b)) in enumerate(zip(layers, params)):
            for t, a in enumerate((w, b)):
                if a is not None:
                    self.idx[(i, t)] = len(self.w)
                    self.w.append(torch.nn.Parameter(torch.tensor(a)))

    def p(self, i, t):
        return self.w[self.idx[(i, t)]] if (i, t) in self.idx else None

    def forward(self, x):
        outs = []
        F = torch.nn.functional
        for i, l in enumerate(self.layers):
            s0 = i - 1 if l.src0 < 0 else l.src0
            a = x if s0 < 0 else outs[s0]
            if l.kind == S.LINEAR:
                y = F.linear(a.reshape(a.shape[0], -1), self.p(i, 0), self.p(i, 1))
            elif l.kind == S.CONV2D:
                y = F.conv2d(a, self.p(i, 0), self.p(i, 1), (l.sh, l.sw), (l.ph, l.pw))
            elif l.kind == S.BATCHNORM2D:
                y = F.batch_norm(a, None, None, self.p(i, 0), self.p(i, 1), training=True, eps=float(np.float32(l.bn_eps)))
            elif l.kind == S.RELU:
                y = F.relu(a)
            elif l.kind == S.MAXPOOL2D:
                y = F.max_pool2d(a, (l.kh, l.kw), (l.sh, l.sw), (l.ph, l.pw))
            elif l.kind == S.AVGPOOL2D:
                y = F.avg_pool2d(a, (l.kh, l.kw), (l.sh, l.sw), (l.ph, l.pw), count_include_pad=True)
            elif l.kind == S.AVGPOOL_GLOBAL:
                y = a.mean(dim=(2, 3), keepdim=True)
            elif l.kind == S.FLATTEN:
                y = a.reshape(a.shape[0], -1)
            elif l.kind == S.ADD:
                y = a + outs[l.src1]
            elif l.kind == S.CONCAT:
                y = torch.cat([a, outs[l.src1]], dim=1)
            else:
                y = a
            outs.append(y)
        return outs[-1].reshape(x.shape[0], -1)

    def flat_grad(self):
        g = []
        for i in range(len(self.layers)):
            for t in (0, 1):
                p = self.p(i, t)
                if p is not None:
                    g.append(p.grad.detach().numpy().ravel())
        return np.concatenate(g)

    def flat(self):
        return np.concatenate([p.detach().numpy().ravel() for p in self.w])


def small_mlp():
    return S.mlp((20, 16, 12, 5))


def residual_net():
    """conv -> BN -> ReLU -> [conv -> BN] + skip -> ReLU -> concat(branch) -> avgpool -> FC"""
    L = [conv(3, 8, 3, 1, 1), bn(8), relu(),                               # 0,1,2
         conv(8, 8, 3, 1, 1), bn(8), Layer(ADD, src0=4, src1=2), relu(),   # 3,4,5,6
         conv(8, 4, 1, 2, 0), Layer(S.MAXPOOL2D, kh=3, kw=3, sh=2, sw=2, ph=1, pw=1, src0=6),  # 7, 8
         Layer(CONCAT, src0=7, src1=8),                                    # 9 (4+8 ch)
         Layer(AVGPOOL_GLOBAL), Layer(FLATTEN), linear(12, 5), xent()]
    return L


NETS = {
    "mlp": (small_mlp, (20, 1, 1), 5),
    "cnn": (lambda: S.tiny_cnn(3, 5, 4), (3, 8, 8), 5),
    "res": (residual_net, (3, 8, 8), 5),
    "inception_branch": (lambda: [conv(3, 8, 3, 1, 1), bn(8), relu(),
                                  Layer(S.AVGPOOL2D, kh=3, kw=3, sh=1, sw=1, ph=1, pw=1), conv(8, 4, 1, 1, 0),
                                  bn(4), relu(), Layer(CONCAT, src0=6, src1=2), Layer(AVGPOOL_GLOBAL),
                                  Layer(FLATTEN), linear(12, 5), xent()], (3, 7, 7), 5),
    "conv_s2": (lambda: [conv(2, 4, (3, 1), (2, 1), (1, 0), bias=1), relu(), conv(4, 3, (1, 3), 1, (0, 1)),
                         maxpool(2, 2), Layer(FLATTEN), linear(3 * 2 * 4, 5), xent()], (2, 7, 8), 5),
}


def make(name, K=1, T=1, N=8, mode="fp64", predict="off", lr=1e-3, seed=3, **kw):
    import oracle
    build, shape, classes = NETS[name]
    L = build()
    P = S.make_params(L, seed)
    o = oracle.Oracle(L, K, T, N, lr, BETAS32, EPS32, shape, classes, P, mode=mode, predict=predict, **kw)
    return o, L, P, shape, classes


# ----------------------------------------------------------------------------- tests
@pytest.mark.parametrize("name", list(NETS))
def test_loss_grad_matches_torch_autograd(oracle_mod, name):
    """P8/O6: every layer kind's forward+backward equals torch autograd (fp64)."""
    o, L, P, shape, classes = make(name)
    x, y = S.make_inputs(8, shape, classes, 5, kind="gauss")
    loss, g = o.eval_loss_grad(x, y)
    net = TorchNet(L, P)
    z = net(torch.tensor(x, dtype=torch.float64))
    ref = torch.nn.functional.cross_entropy(z, torch.tensor(y, dtype=torch.long))
    ref.backward()
    assert abs(loss - ref.item()) <= 1e-12 * max(1, abs(ref.item()))
    np.testing.assert_allclose(g, net.flat_grad(), rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("name", ["mlp", "cnn", "res", "conv_s2", "inception_branch"])
def test_loss_grad_matches_finite_differences(oracle_mod, name):
    """P8: central differences, h=1e-5, relative error < 1e-4, fp64."""
    import oracle
    o, L, P, shape, classes = make(name)
    x, y = S.make_inputs(8, shape, classes, 11, kind="gauss")
    _, g = o.eval_loss_grad(x, y)
    rng = np.random.default_rng(0)
    flat_index = []
    for i, (w, b) in enumerate(P):
        for t, a in enumerate((w, b)):
            if a is not None:
                for q in rng.choice(a.size, size=min(6, a.size), replace=False):
                    flat_index.append((i, t, int(q)))
    offs, off = {}, 0
    for i, (w, b) in enumerate(P):
        for t, a in enumerate((w, b)):
            if a is not None:
                offs[(i, t)] = off
                off += a.size
    h = 1e-5
    for (i, t, q) in flat_index:
        vals = []
        for sgn in (+1, -1):
            P2 = [[None if a is None else a.copy() for a in p] for p in P]
            P2[i][t].ravel()[q] += sgn * h
            o2 = oracle.Oracle(L, 1, 1, 8, 1e-3, BETAS32, EPS32, shape, classes, P2, mode="fp64", predict="off")
            vals.append(o2.eval_loss_grad(x, y)[0])
            o2.close()
        fd = (vals[0] - vals[1]) / (2 * h)
        an = g[offs[(i, t)] + q]
        assert abs(fd - an) <= 1e-4 * max(abs(fd), abs(an)) + 1e-7, (i, t, q, fd, an)


def test_softmax_uniform_logits(oracle_mod):
    """uniform logits give loss ln C; gradient rows sum to 0.  A single Linear with
    zero weights makes the logits uniform."""
    import oracle
    L = [linear(4, 7), xent()]
    P = [[np.zeros((7, 4)), np.zeros(7)], [None, None]]
    o = oracle.Oracle(L, 1, 1, 3, 1e-3, BETAS32, EPS32, (4, 1, 1), 7, P, mode="fp64", predict="off")
    x, y = S.make_inputs(3, (4, 1, 1), 7, 2, kind="gauss")
    loss, g = o.eval_loss_grad(x, y)
    assert abs(loss - np.log(7)) < 1e-14
    db = g[28:]
    assert abs(db.sum()) < 1e-15


@pytest.mark.parametrize("name,T", [("mlp", 1), ("mlp", 4), ("cnn", 1), ("cnn", 2), ("res", 2)])
def test_single_stage_s0_equals_torch_adam(oracle_mod, name, T):
    """P4 / BJ: 1 stage with s=0 equals plain Adam (torch.optim.Adam, fp64) on the same
    model and data; the mini-batch gradient is accumulated over T micro-batches with
    per-micro-batch BatchNorm statistics (R8, R11)."""
    N, M, lr = 8, 4, 1e-3
    o, L, P, shape, classes = make(name, K=1, T=T, N=N, lr=lr)
    x, y = S.make_inputs(M * N, shape, classes, 9, kind="gauss")
    o.step(x, y, M, flush=True)
    net = TorchNet(L, P)
    opt = torch.optim.Adam(net.parameters(), lr=float(np.float32(lr)), betas=BETAS32, eps=EPS32)
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


def test_first_update_closed_form(oracle_mod):
    """P5: from zero moments the first Adam step is W1 = W0 - lr * g / (|g| + eps) exactly
    (bias corrections cancel), g the mini-batch-mean gradient at W0 (torch autograd)."""
    N, lr = 8, 1e-3
    o, L, P, shape, classes = make("cnn", K=1, T=1, N=N, lr=lr)
    x, y = S.make_inputs(N, shape, classes, 4, kind="gauss")
    net = TorchNet(L, P)
    z = net(torch.tensor(x, dtype=torch.float64))
    torch.nn.functional.cross_entropy(z, torch.tensor(y, dtype=torch.long)).backward()
    g = net.flat_grad()
    W0 = net.flat()
    o.step(x, y, 1, flush=True)
    lr32 = float(np.float32(lr))
    np.testing.assert_allclose(o.params_flat(), W0 - lr32 * g / (np.abs(g) + EPS32), rtol=0, atol=1e-15)


@pytest.mark.parametrize("T", [1, 2, 4])
def test_accumulation_equals_full_batch_gradient(oracle_mod, T):
    """P7: summing the T micro-batch gradients (dlogits scaled by 1/N, R8)
    gives the full mini-batch gradient (no BatchNorm), fp64, within 1e-12."""
    N = 8
    o, L, P, shape, classes = make("mlp", K=1, T=T, N=N)
    x, y = S.make_inputs(N, shape, classes, 6, kind="gauss")
    o.step(x, y, 1, flush=True)
    g = np.concatenate([o.get(i, t, "grad") for i in range(len(L)) for t in (0, 1)])
    net = TorchNet(L, P)
    torch.nn.functional.cross_entropy(net(torch.tensor(x, dtype=torch.float64)), torch.tensor(y, dtype=torch.long)).backward()
    np.testing.assert_allclose(g, net.flat_grad(), rtol=0, atol=1e-12)


def test_fp32_mode_tracks_fp64(oracle_mod):
    """The fp32-contract path is the same computation at fp32 precision: close to fp64 (catches
    a dropped term in the fp32 code path, which the bit-exact GPU parity would inherit)."""
    for name in ("mlp", "res"):
        a, L, P, shape, classes = make(name, mode="fp64")
        b, *_ = make(name, mode="fp32")
        x, y = S.make_inputs(8, shape, classes, 8, kind="gauss")
        la, ga = a.eval_loss_grad(x, y)
        lb, gb = b.eval_loss_grad(x, y)
        assert abs(la - lb) < 1e-5
        assert np.linalg.norm(ga - gb) <= 1e-5 * np.linalg.norm(ga)


def test_bf16_mode_tracks_fp64(oracle_mod):
    a, L, P, shape, classes = make("cnn", mode="fp64")
    b, *_ = make("cnn", mode="bf16")
    x, y = S.make_inputs(8, shape, classes, 8, kind="gauss")
    la, ga = a.eval_loss_grad(x, y)
    lb, gb = b.eval_loss_grad(x, y)
    assert abs(la - lb) < 2e-2
    assert np.linalg.norm(ga - gb) <= 0.1 * np.linalg.norm(ga)


# ----------------------------------------------------------------------------- the sweep
def _rand_state(n, seed):
    rng = np.random.default_rng(seed)
    W = rng.uniform(-0.05, 0.05, n)
    g = rng.uniform(-1e-2, 1e-2, n)
    m = 0.1 * rng.uniform(-1e-2, 1e-2, n)
    v = rng.uniform(1e-6, 1e-4, n)
    return [a.astype(np.float32) for a in (W, g, m, v)]


@pytest.mark.parametrize("k", [1, 2, 7, 1000])
def test_sweep_fp64_equals_torch_adam(oracle_mod, k):
    """P3: the sweep's W', m', v' equal torch.optim.Adam's step k (fp64) and its predictions
    are W' - s*d with d = W - W' the Adam step just taken ("computed from Adam's own
    moments", north star)."""
    W, g, m, v = _rand_state(1000, k)
    lr = float(np.float32(1e-4))
    Wn, mn, vn, pf, pb = oracle_mod.adam_predict(W, g, m, v, k, lr, BETAS32, EPS32, 3, 1, mode="fp64")
    p = torch.nn.Parameter(torch.tensor(W.astype(np.float64)))
    opt = torch.optim.Adam([p], lr=lr, betas=BETAS32, eps=EPS32)
    p.grad = torch.tensor(g.astype(np.float64))
    opt.step()   # initialises the state at step 1; overwrite and redo for step k
    st = opt.state[p]
    with torch.no_grad():
        p.copy_(torch.tensor(W.astype(np.float64)))
    st["exp_avg"] = torch.tensor(m.astype(np.float64))
    st["exp_avg_sq"] = torch.tensor(v.astype(np.float64))
    st["step"] = torch.tensor(float(k - 1))
    opt.step()
    Wt = p.detach().numpy()
    # outputs are returned as float32: compare at that resolution, plus the exact relations
    np.testing.assert_allclose(Wn, Wt, rtol=0, atol=2e-9)
    np.testing.assert_allclose(mn, st["exp_avg"].numpy(), rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(vn, st["exp_avg_sq"].numpy(), rtol=1e-6, atol=1e-14)
    d = W.astype(np.float64) - Wt
    np.testing.assert_allclose(pf, Wt - 3 * d, rtol=0, atol=4e-9)
    np.testing.assert_allclose(pb, Wt - 1 * d, rtol=0, atol=4e-9)


def test_sweep_prediction_properties(oracle_mod):
    """s=0 gives W_hat = W' exactly; W_hat - W' is linear in s (fp64)."""
    W, g, m, v = _rand_state(500, 3)
    r0 = oracle_mod.adam_predict(W, g, m, v, 5, 1e-3, BETAS32, EPS32, 0, 1, mode="fp32")
    assert np.array_equal(r0[3], r0[0])
    a = oracle_mod.adam_predict(W, g, m, v, 5, 1e-3, BETAS32, EPS32, 1, 2, mode="fp64")
    b = oracle_mod.adam_predict(W, g, m, v, 5, 1e-3, BETAS32, EPS32, 4, 7, mode="fp64")
    d1 = a[0].astype(np.float64) - a[3]
    # outputs are fp32-rounded: W' and W_hat each carry half an ulp (|W| < 0.06 -> ulp 3.7e-9)
    np.testing.assert_allclose(b[0].astype(np.float64) - b[3], 4 * d1, rtol=0, atol=3e-8)
    np.testing.assert_allclose(a[0].astype(np.float64) - a[4], 2 * d1, rtol=0, atol=2e-8)


def test_sweep_worked_example(oracle_mod):
    """SURVEY A.5 hand-worked two-step example (fp32 canonical order), 8 significant digits."""
    rows = [list(map(float, l.split())) for l in open(os.path.join(GOLD, "adam_worked_example.txt"))
            if l.strip() and not l.startswith("#")]
    W = np.array([0.5, -0.25, 0.125, 0], np.float32)
    m = np.zeros(4, np.float32)
    v = np.zeros(4, np.float32)
    for k, g in ((1, [0.2, -0.1, 1e-9, 0]), (2, [-0.1, -0.1, 0.3, 0])):
        W, m, v, pf, pb = oracle_mod.adam_predict(W, np.array(g, np.float32), m, v, k, 1e-3, (0.9, 0.999), 1e-8, 3, 1)
        row = rows[k - 1]
        assert row[0] == k
        np.testing.assert_allclose(W, row[1:5], rtol=2e-7, atol=1e-9)
        np.testing.assert_allclose(pf, row[5:9], rtol=2e-7, atol=1e-9)
        np.testing.assert_allclose(pb, row[9:13], rtol=2e-7, atol=1e-9)


def test_bf16_rounding_matches_torch(oracle_mod):
    """The bf16 rounding point (round-to-nearest-even) equals torch's float32->bfloat16 cast,
    including exact ties."""
    W, g, m, v = _rand_state(4096, 8)
    a = oracle_mod.adam_predict(W, g, m, v, 3, 1e-3, BETAS32, EPS32, 2, 1, mode="fp32")
    b = oracle_mod.adam_predict(W, g, m, v, 3, 1e-3, BETAS32, EPS32, 2, 1, mode="bf16")
    ref = torch.tensor(a[3], dtype=torch.float32).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(b[3], ref)
    assert np.array_equal(b[0], a[0])     # masters stay fp32
    ties = np.array([1.00390625, 1.01171875, -1.00390625, 3.0e38, 1e-40], np.float32)  # exact halfway cases
    z = np.zeros_like(ties)
    r = oracle_mod.adam_predict(ties, z, z, z + 1.0, 1, 1e-30, BETAS32, EPS32, 0, 0, mode="bf16")
    ref = torch.tensor(r[0]).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(r[3], ref)


def test_paper_delta_form(oracle_mod):
    """Eq. (3)-(4) literal form (opt-in XO_DELTA_PAPER): with g=0 and moments set so
    that v_bar = m/(1-gamma) = 0.5 and m_bar = v/(1-lambda) = 0.25, dW = 0.5/sqrt(0.25+eps)
    ~= 1 and W - W_hat = s*lr*dW (s=2, lr=0.1 -> 0.2)."""
    b1, b2 = BETAS32
    m = np.array([0.05 / b1 * (1 - b1) / 0.1], np.float32)  # m' = b1*m -> m'/(1-b1) ~ 0.5
    v = np.array([0.025 * (1 - b2) / b2 / 0.1], np.float32)
    z = np.zeros(1, np.float32)
    W = np.ones(1, np.float32)
    Wn, mn, vn, pf, pb = oracle_mod.adam_predict(W, z, m, v, 1, 0.1, BETAS32, EPS32, 2, 1, mode="fp64", delta="paper")
    dW = (mn[0] / (1 - b1)) / np.sqrt(vn[0] / (1 - b2) + EPS32)
    assert abs(dW - 1.0) < 1e-5
    assert abs((Wn[0] - pf[0]) - 0.2) < 1e-5


def test_dag_models_match_torch_autograd(oracle_mod):
    """ResNet bottlenecks (residual add, strided 1x1 downsample, 7x7 s2 stem, 3x3 s2 maxpool)
    and Inception modules (asymmetric kernels, avgpool branch, multi-way concat) against torch
    autograd in fp64: reduced depth, the real block structure."""
    import oracle
    from synthetic.models import resnet101, inception_v3
    for L, shape, classes in ((resnet101(classes=7, layers=(1, 1, 1, 1))[0], (3, 32, 32), 7),
                              (inception_v3(classes=7)[0], (3, 64, 64), 7)):
        P = S.make_params(L, 2)
        o = oracle.Oracle(L, 1, 1, 4, 1e-3, BETAS32, EPS32, shape, classes, P, mode="fp64", predict="off")
        x, y = S.make_inputs(4, shape, classes, 3, kind="imagenet")
        loss, g = o.eval_loss_grad(x, y)
        net = TorchNet(L, P)
        ref = torch.nn.functional.cross_entropy(net(torch.tensor(x, dtype=torch.float64)), torch.tensor(y, dtype=torch.long))
        ref.backward()
        assert abs(loss - ref.item()) <= 1e-10
        ref_g = net.flat_grad()
        # fp64 accumulation-order noise only: bound relative to the gradient's scale
        np.testing.assert_allclose(g, ref_g, rtol=1e-8, atol=1e-11 * np.abs(ref_g).max())


@pytest.mark.parametrize("K", [2, 3])
def test_dag_gpipe_no_prediction_equals_single_stage(oracle_mod, K):
    """P6 on a DAG model with explicit unit-based stage assignment (R17)."""
    import oracle
    from synthetic.models import resnet101, assign_stages
    L, units = resnet101(classes=5, layers=(1, 1, 1, 1))
    P = S.make_params(L, 4)
    x, y = S.make_inputs(3 * 4, (3, 16, 16), 5, 4, kind="imagenet")
    res = []
    for k in (1, K):
        Lk = assign_stages(L, units, k)
        o = oracle.Oracle(Lk, k, 2, 4, 1e-3, BETAS32, EPS32, (3, 16, 16), 5, P, mode="fp32", schedule="gpipe",
                          predict="off")
        o.step(x, y, 3, flush=True)
        res.append(o.params_flat())
    assert np.array_equal(res[0], res[1])
