"""Oracle pins: version differences (Eq. 1/2), the schedule and version bookkeeping.

Pinned against: the paper's worked example, SPEC's hand-evaluated values, the paper's
own definition of s evaluated on a unit-cost timeline, and the golden traces of
reading R7 (tests/golden/).  Nothing here retypes the oracle's formulas.
"""
import os

import numpy as np
import pytest

import synthetic as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fmt(tr):
    out = []
    for (_st, op, t, j, ver, _s, bw) in tr:
        out.append("U->v%d" % ver if op == 2 else "%s%d.%d@v%d%s" % ("FB"[op], t, j, ver, "*" if bw else ""))
    return " ".join(out)


def read_golden_trace(name):
    rows = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            k, rest = line.split(" ", 1)
            rows[int(k)] = rest.strip()
    return rows


def test_version_difference_golden(oracle_mod):
    """P:76 and SPEC S:231-233, S:264 hand values."""
    with open(os.path.join(GOLD, "version_difference.txt")) as f:
        rows = [list(map(int, l.split())) for l in f if l.strip() and not l.startswith("#")]
    assert len(rows) >= 10
    for K, T, rank, p, s in rows:
        assert oracle_mod.version_difference(K, T, rank, p) == s, (K, T, rank, p)


def _program(K, T, k, U):
    """Stage k's op order under reading R7 (K-k warm-up forwards, then B(i), F(i+K-k), drain);
    written from the prose of R7, independently of the oracle's implementation."""
    W = K - k
    ops = [("F", u) for u in range(1, min(W, U) + 1)]
    for i in range(1, U + 1):
        ops.append(("B", i))
        if i + W <= U:
            ops.append(("F", i + W))
    return ops


def _timeline(K, T, U, cf=1, cb=1):
    """Unit-cost earliest-start timeline: op (stage k) starts when the stage is free and its
    input exists (F(u) needs F(u) on k-1; B(u) needs B(u) on k+1 and F(u) on k)."""
    progs = [_program(K, T, k, U) for k in range(K)]
    end = {}
    pos = [0] * K
    free = [0] * K
    while any(pos[k] < len(progs[k]) for k in range(K)):
        moved = False
        for k in range(K):
            while pos[k] < len(progs[k]):
                op, u = progs[k][pos[k]]
                if op == "F":
                    dep = [("F", k - 1, u)] if k > 0 else []
                else:
                    dep = [("F", k, u)] + ([("B", k + 1, u)] if k < K - 1 else [])
                if not all(d in end for d in dep):
                    break
                start = max([free[k]] + [end[d] for d in dep])
                e = start + (cf if op == "F" else cb)
                end[(op, k, u)] = e
                free[k] = e
                pos[k] += 1
                moved = True
        assert moved
    return end


@pytest.mark.parametrize("K", [2, 4, 8])
@pytest.mark.parametrize("T", [1, 2])
def test_eq1_equals_paper_definition_of_s(oracle_mod, K, T):
    """P:102 defines s as the number of weight updates between the bellwether's pipeline unit
    and the unit at which the mini-batch's T-th micro-batch completes its round trip on
    GPU 0.  Counted on a unit-cost timeline of the R7 schedule, it equals half-up Eq. (1)
    for T in {1, 2}."""
    M = 6 * K
    U = M * T
    end = _timeline(K, T, U)
    t = M // 2                              # a steady-phase mini-batch
    for k in range(K):
        f_start = end[("F", k, (t - 1) * T + 1)] - 1
        rt_end = end[("B", 0, t * T)]
        upd = [end[("B", k, tt * T)] for tt in range(1, M + 1)]
        count = sum(1 for e in upd if f_start < e < rt_end)
        assert oracle_mod.version_difference(K, T, k, 0) == count, (K, T, k, count)


@pytest.mark.parametrize("K", [2, 4, 8])
def test_eq2_equals_backward_count_T1(oracle_mod, K):
    """Backward analogue at T=1: updates on stage k from the bellwether's backward to the end
    of the round trip on GPU 0, excluding the mini-batch's own update."""
    T, M = 1, 6 * K
    end = _timeline(K, T, M)
    t = M // 2
    for k in range(K):
        b_start = end[("B", k, t)] - 1
        rt_end = end[("B", 0, t)]
        upd = [(tt, end[("B", k, tt)]) for tt in range(1, M + 1)]
        count = sum(1 for tt, e in upd if tt != t and b_start <= e <= rt_end)
        assert oracle_mod.version_difference(K, T, k, 1) == count


def _run(oracle_mod, K, T, M, calls=None, mode="fp32", schedule="xpipe", predict="paper", layers=None, seed=1,
         N=32, lr=1e-3):
    L = layers or S.mlp()
    P = S.make_params(L, seed)
    shape = (784, 1, 1) if layers is None else (3, 8, 8)
    o = oracle_mod.Oracle(L, K, T, N, lr, (0.9, 0.999), 1e-8, shape, 10, P, mode=mode, schedule=schedule,
                          predict=predict, snapshots=True)
    x, y = S.make_inputs(M * N, shape, 10, seed, kind="mnist" if layers is None else "gauss")
    calls = calls or [M]
    off = 0
    for i, m in enumerate(calls):
        o.step(x[off * N:(off + m) * N], y[off * N:(off + m) * N], m, flush=(i == len(calls) - 1))
        off += m
    return o


@pytest.mark.parametrize("name,K,T,M", [("trace_K2_T4_M3.txt", 2, 4, 3), ("trace_K4_T2_M4.txt", 4, 2, 4),
                                        ("trace_K1_T4_M2.txt", 1, 4, 2)])
def test_golden_traces(oracle_mod, name, K, T, M):
    gold = read_golden_trace(name)
    layers = None if K <= 4 else None
    o = _run(oracle_mod, K, T, M)
    for k in range(K):
        assert fmt(o.trace(k)) == gold[k], k


def test_paper_worked_example_P76(oracle_mod):
    """K=4, T=2; GPU 0 runs micro-batch 5's forward with the initial weights, and its
    weights are updated twice (after micro-batches 2 and 4) before micro-batch 5's backward."""
    o = _run(oracle_mod, 4, 2, 4)
    tr = o.trace(0)
    iF = next(i for i, r in enumerate(tr) if r[1] == 0 and (r[2], r[3]) == (3, 1))
    iB = next(i for i, r in enumerate(tr) if r[1] == 1 and (r[2], r[3]) == (3, 1))
    assert tr[iF][4] == 0                                  # forward at version 0
    upd = [r for r in tr[iF:iB] if r[1] == 2]
    assert [r[4] for r in upd] == [1, 2]                   # two updates in between ...
    ends = [r for r in tr[:iB] if r[1] == 1 and r[3] == 2] # ... after micro-batches 2 and 4
    assert [(r[2] - 1) * 2 + r[3] for r in ends] == [2, 4]


@pytest.mark.parametrize("K,T", [(1, 1), (2, 4), (4, 2), (4, 4), (2, 1)])
def test_schedule_invariants(oracle_mod, K, T):
    """P2: one F and one B per (u, k); F before B; every F(t,.) uses F(t,1)'s version; every
    B(t,.) uses version t-1; exactly M updates per stage."""
    M = 5
    layers = None
    o = _run(oracle_mod, K, T, M)
    for k in range(K):
        tr = o.trace(k)
        seen_f, seen_b = {}, {}
        fver, nupd = {}, 0
        for i, (st, op, t, j, ver, s, bw) in enumerate(tr):
            u = (t - 1) * T + j
            if op == 0:
                assert u not in seen_f
                seen_f[u] = i
                fver.setdefault(t, ver)
                assert fver[t] == ver and bw == (j == 1)
            elif op == 1:
                assert u in seen_f and u not in seen_b
                seen_b[u] = i
                assert ver == t - 1
            else:
                nupd += 1
                assert ver == nupd
        assert len(seen_f) == len(seen_b) == M * T and nupd == M
        assert o.version(k) == M


def test_staleness_direction_prediction_off(oracle_mod):
    """with prediction off, updates between F(u) and B(u) on rank 0 are >=
    those on rank K-1 ("GPUs with smaller index tend to use staler weights")."""
    K, T, M = 4, 2, 6
    o = _run(oracle_mod, K, T, M, predict="off")

    def inflight(k):
        tr = o.trace(k)
        res = {}
        for i, r in enumerate(tr):
            if r[1] == 0:
                u = (r[2] - 1) * T + r[3]
                jb = next(q for q in range(i, len(tr)) if tr[q][1] == 1 and (tr[q][2], tr[q][3]) == (r[2], r[3]))
                res[u] = sum(1 for q in range(i, jb) if tr[q][1] == 2)
        return res
    a, b = inflight(0), inflight(K - 1)
    assert all(a[u] >= b[u] for u in a) and sum(a.values()) > sum(b.values())


def test_call_splitting_invariance(oracle_mod):
    """Feeding 3+4+3 mini-batches then a flush equals feeding 10 then a flush (8b)."""
    a = _run(oracle_mod, 2, 4, 10, calls=[3, 4, 3])
    b = _run(oracle_mod, 2, 4, 10, calls=[10])
    for k in range(2):
        assert a.trace(k) == b.trace(k)
    assert np.array_equal(a.params_flat(), b.params_flat())


@pytest.mark.parametrize("mode", ["fp32", "fp64"])
@pytest.mark.parametrize("K", [2, 4])
def test_gpipe_no_prediction_equals_single_stage(oracle_mod, mode, K):
    """P6: the GPipe schedule with s=0 equals K=1 bit-exactly: stage placement
    does not change any per-layer op order."""
    ref = _run(oracle_mod, 1, 4, 4, mode=mode, schedule="gpipe", predict="off")
    got = _run(oracle_mod, K, 4, 4, mode=mode, schedule="gpipe", predict="off")
    assert np.array_equal(ref.params_flat(), got.params_flat())
    # and XPipe at K=1 with s=0 is GPipe at K=1
    xp = _run(oracle_mod, 1, 4, 4, mode=mode, schedule="xpipe", predict="off")
    assert np.array_equal(ref.params_flat(), xp.params_flat())


def test_prediction_changes_the_trajectory(oracle_mod):
    """Sanity: with K>1 the predicted run differs from the prediction-off run."""
    a = _run(oracle_mod, 2, 4, 4, predict="paper")
    b = _run(oracle_mod, 2, 4, 4, predict="off")
    assert not np.array_equal(a.params_flat(), b.params_flat())
