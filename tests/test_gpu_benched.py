"""Parity of the configurations bench.py actually times (BASELINE configs at full size, all
stages on one B200): CUDA graphs captured and replayed, forwards on their own stream per stage
(fb_overlap), per-op timing events, several mini-batches per xpipe_step call, the mini-batch
sequence split across calls, and a flush at the end -- compared with the oracle's bf16
replay of the same 10 mini-batches (north star: relative Frobenius error <= 2e-2 per stage
after 10 mini-batches at lr 1e-4), plus the W_hat buffers bit-exact against the
prediction evaluated from the GPU's own state.

Inputs are pinned host buffers that differ from call to call, so a replayed graph that read a
stale or in-flight input copy would train on the wrong data.  Graph mode
excludes trace and snapshots; traces at these sizes are checked in test_gpu_fullsize.py."""
import numpy as np
import pytest

import synthetic as S
from helpers import rel_frob, predict_from_state, log_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LR = 1e-4


def stage_vec(model, L, k, get):
    parts = []
    for i in range(len(L)):
        if model.stage_of(i) != k:
            continue
        for t in (0, 1):
            n = model._count(i, t) if hasattr(model, "_count") else None
            if n is None:
                n = _count(L, i, t)
            if n:
                parts.append(np.asarray(get(i, t), np.float64))
    return np.concatenate(parts)


def _count(L, i, t):
    l = L[i]
    if l.kind == S.LINEAR:
        return l.out_c * l.in_c if t == 0 else (l.out_c if l.bias else 0)
    if l.kind == S.CONV2D:
        return l.out_c * l.in_c * l.kh * l.kw if t == 0 else (l.out_c if l.bias else 0)
    if l.kind == S.BATCHNORM2D:
        return l.in_c
    return 0


def run_benched(L, shape, classes, kind, K, T, N, calls):
    """The bench's launch configuration through the public API; returns (model, losses, replays)."""
    from paper_1911_04610_b200 import XPipe
    P = S.make_params(L, 1)
    M = sum(calls)
    x, y = S.make_inputs(M * N, shape, classes, 1, kind=kind)
    g = XPipe(L, K, T, N, LR, (0.9, 0.999), 1e-8, shape, classes, params=P, precision="bf16", graphs=True,
              fb_overlap=True, timing=True, watchdog_ms=300000)
    # pinned host staging buffers, refilled with each call's mini-batches
    per = int(np.prod(shape))
    big = max(calls)
    xh = torch.empty((big * N, per), dtype=torch.float32).pin_memory()
    yh = torch.empty(big * N, dtype=torch.int32).pin_memory()
    losses, replays, off = [], 0, 0
    for c in calls:
        xs, ys = x[off * N:(off + c) * N].reshape(c * N, per), y[off * N:(off + c) * N]
        xh[:c * N].copy_(torch.from_numpy(xs))
        yh[:c * N].copy_(torch.from_numpy(ys))
        lo = g.step(xh[:c * N].numpy(), yh[:c * N].numpy(), c)
        st = g.last_stats
        replays += st.graph_replays
        tm = st.timing(K)
        assert tm["span_ms"] > 0 and 0 <= tm["bubble_fraction"] < 1, tm
        assert all(0 < b <= tm["span_ms"] * 1.0001 for b in tm["busy_ms"]), tm
        # poison the staging buffers: a graph reading them after the call returned would see NaN
        xh.fill_(float("nan"))
        yh.fill_(-1)
        losses.append(lo)
        off += c
    g.step(x[:0], y[:0], 0, flush=True)
    return g, P, x, y, np.concatenate(losses), replays


def oracle_run(oracle_mod, L, shape, classes, kind, K, T, N, M, P, x, y):
    o = oracle_mod.Oracle(L, K, T, N, LR, (0.9, 0.999), 1e-8, shape, classes, P, mode="bf16")
    lo = o.step(x, y, M, flush=True)
    return o, np.asarray(lo)


def compare(name, g, o, L, K, M, lg, lo, bar=2e-2):
    rel = []
    for k in range(K):
        assert g.version(k) == M, (k, g.version(k))
        a = stage_vec(g, L, k, lambda i, t: g.get(i, t, "param"))
        b = stage_vec(o, L, k, lambda i, t: o.get(i, t, "param"))
        rel.append(rel_frob(a, b))
    # W_hat self-consistency on every weighted tensor (bit-exact)
    for k in range(K):
        sf = o.trace(k)[0][5]
        sb = next(r for r in o.trace(k) if r[1] == 1)[5]
        for i in range(len(L)):
            if g.stage_of(i) != k:
                continue
            for t in (0, 1):
                if not _count(L, i, t):
                    continue
                W, m, v = (g.get(i, t, st) for st in ("param", "m", "v"))
                for st, s in (("pred_fwd", sf), ("pred_bwd", sb)):
                    ref = predict_from_state(W, m, v, M, s, LR, 0.9, 0.999, 1e-8)
                    assert np.array_equal(g.get(i, t, st), ref), (k, i, t, st)
    dl = float(np.nanmax(np.abs(lg - lo)))
    log_parity(name, relfrob_final_per_stage=rel, bar=bar, margin=bar / max(rel), loss_maxabs_diff=dl,
               minibatches=M)
    print(name, "relFrob per stage after", M, "mini-batches:", [round(r, 5) for r in rel], "loss diff", dl)
    assert np.all(np.isfinite(lg))
    assert max(rel) <= bar, rel
    return rel


def test_config2_as_benched(oracle_mod):
    """configs[1]: VGG-16 / synthetic CIFAR-10, K=4, N=128, T=4, bf16; 10 mini-batches fed as
    2+2+2+2+2 calls (graphs captured at the 3rd call, replayed after), then a flush."""
    L = S.vgg16_cifar()
    K, T, N, calls = 4, 4, 128, [2, 2, 2, 2, 2]
    g, P, x, y, lg, replays = run_benched(L, (3, 32, 32), 10, "cifar", K, T, N, calls)
    assert replays >= 2, replays
    o, lo = oracle_run(oracle_mod, L, (3, 32, 32), 10, "cifar", K, T, N, sum(calls), P, x, y)
    compare("config2_as_benched", g, o, L, K, sum(calls), lg, lo)
    g.close()


@pytest.mark.parametrize("name,K,T,N,calls", [("resnet101", 8, 8, 256, [2, 2, 2, 2, 2]),
                                              ("inception", 4, 4, 128, [2, 2, 2, 2, 2]),
                                              ("inception", 8, 4, 128, [2, 2, 2, 2, 2])])
def test_full_size_weights_as_benched(oracle_mod, name, K, T, N, calls):
    """configs[2] (ResNet-101, K=8, N=256, T=8) and configs[3] (Inception-V3, K=4 and 8, N=128,
    T=4) on synthetic Tiny-ImageNet 64x64, 10 mini-batches in the bench's launch configuration,
    against the oracle's bf16 replay at the same size."""
    from synthetic.models import resnet101, inception_v3, assign_stages
    L, units = resnet101(classes=200) if name == "resnet101" else inception_v3(classes=200)
    L = assign_stages(L, units, K)
    g, P, x, y, lg, replays = run_benched(L, (3, 64, 64), 200, "imagenet", K, T, N, calls)
    # Inception K=8, T=4: the ring-slot phase of its 12-slot stages repeats every 3 calls of 2
    # mini-batches, so 10 mini-batches end before a signature is seen twice (no replay); the
    # capture/replay path is the same code the other configurations replay
    if not (name == "inception" and K == 8):
        assert replays >= 1, replays
    o, lo = oracle_run(oracle_mod, L, (3, 64, 64), 200, "imagenet", K, T, N, sum(calls), P, x, y)
    compare("%s_K%d_as_benched" % (name, K), g, o, L, K, sum(calls), lg, lo)
    g.close()


def test_fp32_graphs_overlap_changing_pinned_inputs(oracle_mod):
    """The fp32 contract path (bit-exact with the oracle) in the bench's launch configuration:
    graphs + fb_overlap + timing, 16 mini-batches per call from pinned host buffers refilled
    every call (6.4 MB H2D each, so a graph replay racing the input copy would read the previous
    call's data) -- weights bit-exact after the flush."""
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    K, T, N, C, calls = 2, 4, 32, 16, 6
    M = C * calls
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 5, kind="mnist")
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", graphs=True,
              fb_overlap=True, timing=True, watchdog_ms=60000)
    xh = torch.empty((C * N, 784), dtype=torch.float32).pin_memory()
    yh = torch.empty(C * N, dtype=torch.int32).pin_memory()
    replays = 0
    for i in range(calls):
        xh.copy_(torch.from_numpy(x[i * C * N:(i + 1) * C * N].reshape(C * N, 784)))
        yh.copy_(torch.from_numpy(y[i * C * N:(i + 1) * C * N]))
        g.step(xh.numpy(), yh.numpy(), C)
        replays += g.last_stats.graph_replays
        xh.fill_(float("nan"))
    g.step(x[:0], y[:0], 0, flush=True)
    assert replays >= 2, replays
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32")
    o.step(x, y, M, flush=True)
    assert np.array_equal(g.params_flat(), o.params_flat().astype(np.float32))
    g.close()


@pytest.mark.parametrize("timing,host", [(0, False), (3, False), (0, True), (3, True)])
def test_fp32_async_chained_replays(oracle_mod, timing, host):
    """Asynchronous calls (XP_ASYNC) whose graph replays chain on the device without a host wait
    (the bench's timed loop): every call's inputs are distinct device tensors (host=True: distinct
    pinned host buffers -- the e2e loop -- whose H2D copies are staged on the copy stream while the
    previous call's graph runs) and its losses go to a pinned buffer by an asynchronous copy;
    weights bit-exact with the oracle after the flush and the losses equal the oracle's.
    timing=3: every third call is stamped and completes synchronously in between."""
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    K, T, N, C, calls = 2, 4, 32, 8, 12
    M = C * calls
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 7, kind="mnist")
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", graphs=True,
              fb_overlap=True, timing=timing, watchdog_ms=60000)
    xs = [torch.from_numpy(x[i * C * N:(i + 1) * C * N].copy()) for i in range(calls)]
    ys = [torch.from_numpy(y[i * C * N:(i + 1) * C * N].copy()) for i in range(calls)]
    if host:  # pinned host buffers (kept alive until the sync below), passed as numpy views
        xs = [t.pin_memory() for t in xs]
        ys = [t.pin_memory() for t in ys]
        xs_arg, ys_arg = [t.numpy() for t in xs], [t.numpy() for t in ys]
    else:
        xs_arg, ys_arg = [t.cuda() for t in xs], [t.cuda() for t in ys]
    outs = [torch.full((C * T,), float("nan")).pin_memory() for _ in range(calls)]
    replays = 0
    for i in range(calls):
        g.step(xs_arg[i], ys_arg[i], C, async_=True, loss_out=outs[i])
        replays += g.last_stats.graph_replays
    g.sync()
    g.step(x[:0], y[:0], 0, flush=True)
    assert replays >= 4, replays
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32")
    lo = o.step(x, y, M, flush=True)
    assert np.array_equal(g.params_flat(), o.params_flat().astype(np.float32))
    got = torch.cat(outs).numpy()
    assert np.isfinite(got).all()
    if lo is not None:
        assert np.allclose(got, np.asarray(lo, dtype=np.float32).ravel()[:got.size], rtol=0, atol=0)
    g.close()


def test_device_label_range_and_nonfinite(oracle_mod):
    """Device-pointer labels are range-checked by the loss kernel (XP_EINVAL after the call) and
    a non-finite loss is reported as XP_ENONFINITE."""
    from paper_1911_04610_b200 import XPipe, XPipeError
    L = S.mlp((16, 8, 10))
    P = S.make_params(L, 1)
    x, y = S.make_inputs(2 * 8, (16, 1, 1), 10, 1, kind="gauss")
    g = XPipe(L, 1, 2, 8, 1e-4, (0.9, 0.999), 1e-8, (16, 1, 1), 10, params=P, precision="fp32")
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    g.step(xd, yd, 2)
    bad = yd.clone()
    bad[3] = 10
    with pytest.raises(XPipeError) as e:
        g.step(xd, bad, 2)
    assert e.value.code == -1
    with pytest.raises(TypeError):
        g.step(xd, yd.long(), 2)
    xn = xd.clone()
    xn[0, 0] = float("inf")
    with pytest.raises(XPipeError) as e:
        g.step(xn, yd, 2)
    assert e.value.code == -6
    g.close()
