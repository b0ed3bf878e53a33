"""Pipeline parity on the bf16 tensor-core path (conv blocks on tcgen05): weights within
relative Frobenius error 2e-2 of the oracle's bf16-emulation replay after 10 mini-batches
(north star), the schedule/version trace bit-exact, and the materialised W_hat buffers
bit-exact against the prediction evaluated on the GPU's own state (the bf16 tolerance cannot
see prediction bugs)."""
import numpy as np
import pytest

import synthetic as S
from synthetic.models import conv, bn, relu, maxpool, linear, xent, Layer, FLATTEN
from helpers import rel_frob, predict_from_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def vgg_small(width=16):
    """VGG-shaped: 3 x [conv3x3, BN, ReLU, maxpool2], flatten, Linear (8x8 input)."""
    return [conv(3, width, 3, 1, 1), bn(width), relu(), maxpool(2, 2),
            conv(width, 2 * width, 3, 1, 1), bn(2 * width), relu(), maxpool(2, 2),
            conv(2 * width, 2 * width, 3, 1, 1), bn(2 * width), relu(), maxpool(2, 2),
            Layer(FLATTEN), linear(2 * width, 10), xent()]


def stage_params(model, L, k, get):
    parts = []
    for i in range(len(L)):
        if model.stage_of(i) != k:
            continue
        for t in (0, 1):
            n = model_count(L, i, t)
            if n:
                parts.append(np.asarray(get(i, t), np.float64))
    return np.concatenate(parts)


def model_count(L, i, t):
    l = L[i]
    if l.kind == S.LINEAR:
        return l.out_c * l.in_c if t == 0 else (l.out_c if l.bias else 0)
    if l.kind == S.CONV2D:
        return l.out_c * l.in_c * l.kh * l.kw if t == 0 else (l.out_c if l.bias else 0)
    if l.kind == S.BATCHNORM2D:
        return l.in_c
    return 0


def run_bf16(oracle_mod, L, in_shape, K, T, N, M, lr=1e-4, kind="cifar", classes=10, seed=1, schedule="xpipe",
             predict="paper"):
    from paper_1911_04610_b200 import XPipe
    P = S.make_params(L, seed)
    x, y = S.make_inputs(M * N, in_shape, classes, seed, kind=kind)
    g = XPipe(L, K, T, N, lr, (0.9, 0.999), 1e-8, in_shape, classes, params=P, precision="bf16",
              schedule=schedule, predict=predict, trace=True, snapshots=True, watchdog_ms=120000)
    o = oracle_mod.Oracle(L, K, T, N, lr, (0.9, 0.999), 1e-8, in_shape, classes, P, mode="bf16",
                          schedule=schedule, predict=predict, snapshots=True)
    lg = g.step(x, y, M, flush=True)
    lo = o.step(x, y, M, flush=True)
    return g, o, P, lg, lo


def check(g, o, L, K, M, bar=2e-2, lr=1e-4):
    for k in range(K):
        assert g.trace(k) == o.trace(k), k
    curves = []
    for k in range(K):
        curve = []
        for v in range(M + 1):
            a = stage_params(g, L, k, lambda i, t: g.get(i, t, "param", v))
            b = stage_params(o, L, k, lambda i, t: o.get(i, t, "param", v))
            curve.append(rel_frob(a, b))
        curves.append(curve)
        # prediction self-consistency: W_hat buffers == prediction from the GPU's own state
        sf = o.trace(k)[0][5]
        sb = next(r for r in o.trace(k) if r[1] == 1)[5]
        for i in range(len(L)):
            if g.stage_of(i) != k:
                continue
            for t in (0, 1):
                if not model_count(L, i, t):
                    continue
                W, m, vv = (g.get(i, t, st) for st in ("param", "m", "v"))
                for st, s in (("pred_fwd", sf), ("pred_bwd", sb)):
                    ref = predict_from_state(W, m, vv, g.version(k), s, lr, 0.9, 0.999, 1e-8)
                    assert np.array_equal(g.get(i, t, st), ref), (k, i, t, st)
    print("relFrob per stage per version:", [[round(c, 5) for c in cu] for cu in curves])
    for k in range(K):
        assert curves[k][M] <= bar, (k, curves[k])
    return curves


@pytest.mark.parametrize("K,T", [(1, 2), (2, 2), (4, 1)])
def test_vgg_small_bf16(oracle_mod, K, T):
    L = vgg_small()
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 8, 8), K, T, 16, 10, kind="cifar")
    check(g, o, L, K, 10)
    assert np.all(np.isfinite(lg)) and np.abs(lg - lo).max() < 0.05


def test_vgg_small_gpipe_bf16(oracle_mod):
    L = vgg_small()
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 8, 8), 2, 4, 16, 6, schedule="gpipe", predict="off")
    check(g, o, L, 2, 6)


def test_config2_vgg16_cifar(oracle_mod):
    """BASELINE.json configs[1]: VGG-16 on synthetic CIFAR-10 32x32, 4 stages, mini-batch 128,
    4 micro-batches, bf16; 10 mini-batches at lr 1e-4; bar relFrob <= 2e-2."""
    L = S.vgg16_cifar()
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 32, 32), 4, 4, 128, 10, kind="cifar")
    check(g, o, L, 4, 10)


def model_count_dag(L, i, t):
    return model_count(L, i, t)


@pytest.mark.parametrize("K", [1, 3])
def test_resnet_blocks_bf16(oracle_mod, K):
    """ResNet-101 block structure (7x7 s2 stem + 3x3 s2 maxpool, bottlenecks with strided 1x1
    downsample, residual add + ReLU, global average pool), one bottleneck per stage group,
    explicit unit-based stages (R17)."""
    from synthetic.models import resnet101, assign_stages
    L, units = resnet101(classes=10, layers=(1, 1, 1, 1))
    L = assign_stages(L, units, K)
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 32, 32), K, 2, 16, 6, kind="imagenet")
    check(g, o, L, K, 6)


def test_inception_v3_bf16(oracle_mod):
    """The full Inception-V3 topology at 64x64 (R14): asymmetric 1x7/7x1/1x3/3x1 kernels,
    average-pool branches, stride-2 reductions, four-way concats; 2 stages."""
    from synthetic.models import inception_v3, assign_stages
    L, units = inception_v3(classes=10)
    L = assign_stages(L, units, 2)
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 64, 64), 2, 2, 16, 3, kind="imagenet")
    check(g, o, L, 2, 3)


def test_paper_224_shapes_bf16(oracle_mod):
    """f4: the paper's Tiny-ImageNet upscaled to 224x224 -- the ResNet stem (7x7 s2
    conv, 3x3 s2 max-pool) and one bottleneck per stage group at 224^2 (112^2 stem output, 4 MB
    bf16 per image), 2 stages; and the full Inception-V3 with its unmodified torchvision stem."""
    from synthetic.models import resnet101, inception_v3, assign_stages
    L, units = resnet101(classes=10, layers=(1, 1, 1, 1))
    L = assign_stages(L, units, 2)
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 224, 224), 2, 2, 4, 3, kind="imagenet")
    check(g, o, L, 2, 3)
    L, units = inception_v3(classes=10, stem_pad=False)
    L = assign_stages(L, units, 2)
    g, o, P, lg, lo = run_bf16(oracle_mod, L, (3, 224, 224), 2, 1, 2, 2, kind="imagenet")
    check(g, o, L, 2, 2)


@pytest.mark.parametrize("K,T", [(2, 2), (4, 1)])
def test_vgg_small_bf16_fb_overlap(oracle_mod, K, T):
    """The bf16 conv pipeline with forwards on their own stream per stage (cfg.fb_overlap):
    same tolerance, traces and W_hat self-consistency as without."""
    from paper_1911_04610_b200 import XPipe
    L = vgg_small()
    P = S.make_params(L, 1)
    N, M = 16, 8
    x, y = S.make_inputs(M * N, (3, 8, 8), 10, 1, kind="cifar")
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (3, 8, 8), 10, params=P, precision="bf16", trace=True,
              snapshots=True, fb_overlap=True, watchdog_ms=120000)
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (3, 8, 8), 10, P, mode="bf16", snapshots=True)
    g.step(x, y, M, flush=True)
    o.step(x, y, M, flush=True)
    check(g, o, L, K, M)
