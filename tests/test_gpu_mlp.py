"""Pipeline parity on the fp32 path (config 1, the MLP): the GPU pipeline equals the
oracle's replay bit for bit -- weights after every version (bar: max relative error 1e-4,
expected 0) and the schedule/version trace field by field."""
import numpy as np
import pytest

import synthetic as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def max_rel(a, b):
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    den = np.abs(b)
    num = np.abs(a - b)
    r = np.where(den > 0, num / np.where(den > 0, den, 1), np.where(num > 0, np.inf, 0))
    return float(r.max()) if r.size else 0.0


def run_pair(oracle_mod, K, T, N, M, lr=1e-4, calls=None, schedule="xpipe", predict="paper", s_fwd=0, s_bwd=0,
             layers=None, in_shape=(784, 1, 1), seed=1, graphs=False):
    from paper_1911_04610_b200 import XPipe
    L = layers or S.mlp()
    P = S.make_params(L, seed)
    x, y = S.make_inputs(M * N, in_shape, 10, seed, kind="mnist")
    o = oracle_mod.Oracle(L, K, T, N, lr, (0.9, 0.999), 1e-8, in_shape, 10, P, mode="fp32", schedule=schedule,
                          predict=predict, s_fwd=s_fwd, s_bwd=s_bwd, snapshots=True)
    g = XPipe(L, K, T, N, lr, (0.9, 0.999), 1e-8, in_shape, 10, params=P, precision="fp32", schedule=schedule,
              predict=predict, s_fwd=s_fwd, s_bwd=s_bwd, snapshots=not graphs, trace=not graphs,
              watchdog_ms=20000, graphs=graphs)
    calls = calls or [M]
    off = 0
    lo, lg = [], []
    g.replays = 0
    for i, m in enumerate(calls):
        sl = slice(off * N, (off + m) * N)
        fl = i == len(calls) - 1
        lo.append(o.step(x[sl], y[sl], m, flush=fl))
        lg.append(g.step(x[sl], y[sl], m, flush=fl))
        g.replays += g.last_stats.graph_replays
        off += m
    return o, g, L, np.concatenate(lo), np.concatenate(lg)


def assert_pipeline_equal(o, g, L, K, M):
    for k in range(K):
        assert g.version(k) == o.version(k) == M
        to = o.trace(k)
        tg = g.trace(k)
        assert len(to) == len(tg) and to == tg, k
    for i in range(len(L)):
        assert g.stage_of(i) == o.stage_of(i)
    for v in range(M + 1):
        for i in range(len(L)):
            for t in (0, 1):
                n = o.count(i, t)
                if not n:
                    continue
                a = g.get(i, t, "param", v, n)
                b = o.get(i, t, "param", v).astype(np.float32)
                assert max_rel(a, b) <= 1e-4, (v, i, t)
                assert np.array_equal(a, b), ("not bit-exact", v, i, t, max_rel(a, b))
    for i in range(len(L)):
        for t in (0, 1):
            n = o.count(i, t)
            if n:
                for st in ("m", "v", "pred_fwd", "pred_bwd"):
                    assert np.array_equal(g.get(i, t, st, -1, n), o.get(i, t, st).astype(np.float32)), (st, i, t)


@pytest.mark.parametrize("lr", [1e-4, 1e-3])
def test_config1_mlp_two_stages(oracle_mod, lr):  # noqa: runs after the single-stage case below
    """BASELINE.json configs[0]: MLP 784-256-256-256-10, 2 stages, N=32, T=4, Adam, M=10."""
    o, g, L, lo, lg = run_pair(oracle_mod, 2, 4, 32, 10, lr=lr)
    assert_pipeline_equal(o, g, L, 2, 10)
    np.testing.assert_allclose(lg, lo, rtol=1e-5)


@pytest.mark.parametrize("K,T", [(1, 4), (4, 2), (4, 4), (2, 1), (3, 2)])
def test_mlp_stage_counts(oracle_mod, K, T):
    o, g, L, lo, lg = run_pair(oracle_mod, K, T, 16, 5)
    assert_pipeline_equal(o, g, L, K, 5)


def test_gpipe_schedule(oracle_mod):
    o, g, L, _, _ = run_pair(oracle_mod, 2, 4, 32, 4, schedule="gpipe", predict="off")
    assert_pipeline_equal(o, g, L, 2, 4)


def test_fixed_staleness(oracle_mod):
    o, g, L, _, _ = run_pair(oracle_mod, 2, 2, 16, 4, predict="fixed", s_fwd=5, s_bwd=3)
    assert_pipeline_equal(o, g, L, 2, 4)


def test_call_splitting(oracle_mod):
    """3+4+3 mini-batches with a flush only at the end (both sides) equal the oracle."""
    o, g, L, _, _ = run_pair(oracle_mod, 2, 4, 32, 10, calls=[3, 4, 3])
    assert_pipeline_equal(o, g, L, 2, 10)


def test_determinism_two_runs(oracle_mod):
    _, g1, L, _, _ = run_pair(oracle_mod, 2, 4, 32, 3)
    _, g2, _, _, _ = run_pair(oracle_mod, 2, 4, 32, 3)
    assert np.array_equal(g1.params_flat(), g2.params_flat())


@pytest.mark.parametrize("K,T", [(2, 4), (4, 2), (1, 4)])
def test_cuda_graph_replay_bit_exact(oracle_mod, K, T):
    """Steady-state steps captured as CUDA graphs and replayed (flags rebased per call) give
    the same weights, bit for bit, as the oracle's replay of the same calls.  (The ring-slot
    phase repeats with period lcm(S_k)/gcd(.., micro-batches per call) calls: 16 calls cover it.)"""
    calls = [2] * 16 + [2]
    o, g, L, lo, lg = run_pair(oracle_mod, K, T, 16, sum(calls), calls=calls, graphs=True)
    assert g.replays >= 4, g.replays
    for k in range(K):
        assert g.version(k) == o.version(k) == sum(calls)
    assert np.array_equal(g.params_flat(), o.params_flat().astype(np.float32))
    np.testing.assert_allclose(lg[np.isfinite(lg)], lo[np.isfinite(lg)], rtol=1e-5)


@pytest.mark.parametrize("K,T", [(2, 4), (3, 2)])
def test_serialized_streams_bit_exact(oracle_mod, K, T):
    """cfg.serialize (the bench's profiling mode: every stage on one stream in the dataflow
    enqueue order) runs the same pipeline: weights and trace bit-exact with the oracle."""
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    N, M = 32, 5
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 1, kind="mnist")
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32")
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", trace=True,
              serialize=True, watchdog_ms=20000)
    o.step(x, y, M, flush=True)
    g.step(x, y, M, flush=True)
    for k in range(K):
        assert g.trace(k) == o.trace(k)
    assert np.array_equal(g.params_flat(), o.params_flat().astype(np.float32))
    g.close()


@pytest.mark.parametrize("K,T,schedule", [(2, 4, "xpipe"), (3, 2, "xpipe"), (1, 4, "xpipe"), (2, 2, "gpipe")])
def test_fb_overlap_bit_exact(oracle_mod, K, T, schedule):
    """cfg.fb_overlap (forwards on a second stream per stage, one more ring slot, event
    ordering F(u) -> B(u) -> F(u+S+1) and update -> bellwether forward): weights after every
    version, trace and losses bit-exact with the oracle; split calls and CUDA graphs too."""
    from paper_1911_04610_b200 import XPipe
    L = S.mlp()
    P = S.make_params(L, 1)
    N, M = 32, 8
    pred = "off" if schedule == "gpipe" else "paper"  # GPipe runs under the current weights
    x, y = S.make_inputs(M * N, (784, 1, 1), 10, 1, kind="mnist")
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32", schedule=schedule,
                          predict=pred, snapshots=True)
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", trace=True,
              snapshots=True, schedule=schedule, fb_overlap=True, watchdog_ms=20000)
    lo = o.step(x, y, M, flush=True)
    lg = np.concatenate([g.step(x[:3 * N], y[:3 * N], 3), g.step(x[3 * N:], y[3 * N:], M - 3, flush=True)])
    assert np.array_equal(lg, lo)
    for k in range(K):
        assert g.trace(k) == o.trace(k)
    for v in range(M + 1):
        assert np.array_equal(g.params_flat("param", v), o.params_flat("param", v).astype(np.float32)), v
    g.close()
    # CUDA-graph replay of steady-state calls with the overlap
    g = XPipe(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32", graphs=True,
              schedule=schedule, fb_overlap=True, watchdog_ms=20000)
    o = oracle_mod.Oracle(L, K, T, N, 1e-4, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32", schedule=schedule,
                          predict=pred)
    xs, ys = S.make_inputs(12 * N, (784, 1, 1), 10, 3, kind="mnist")
    reps = 0
    for i in range(12):
        g.step(xs[i * N:(i + 1) * N], ys[i * N:(i + 1) * N], 1, flush=(i == 11))
        reps += g.last_stats.graph_replays
    o.step(xs, ys, 12, flush=True)
    assert np.array_equal(g.params_flat(), o.params_flat().astype(np.float32))
    g.close()
