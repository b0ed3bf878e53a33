"""The runtime's stage programs against the oracle's, on the host.

The product generates each stage's op order with a dependency-driven unit-time simulation
(paper_1911_04610_b200/csrc/schedule.h: B-first 1F1B with K-k stash slots, or GPipe's flush);
the oracle writes the same table as a closed form (reading R7).  Agreement of the two
formulations over many (K, T) is what the GPU trace-parity tests then rely on.  Host only:
xpipe_schedule_program needs no GPU."""
import os

import pytest

import synthetic as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def executed(prog, T, U):
    """Ops a flushed run of U micro-batches executes from an unbounded program: forwards of
    micro-batches beyond U are dropped, the first backward beyond U ends the stage; an update
    follows B(u) when u % T == 0."""
    out = []
    for op, u in prog:
        if u > U:
            if op == 1:
                break
            continue
        t, j = (u - 1) // T + 1, (u - 1) % T + 1
        out.append((op, t, j))
        if op == 1 and j == T:
            out.append((2, t, T))
    return out


def oracle_ops(oracle_mod, K, T, M, schedule):
    L = S.mlp(tuple([4] * K + [3]))
    P = S.make_params(L, 1)
    pred = "off" if schedule == "gpipe" else "paper"
    o = oracle_mod.Oracle(L, K, T, 4 * T, 1e-3, (0.9, 0.999), 1e-8, (4, 1, 1), 3, P, mode="fp64",
                          schedule=schedule, predict=pred)
    x, y = S.make_inputs(M * 4 * T, (4, 1, 1), 3, 1, kind="gauss")
    o.step(x, y, M, flush=True)
    return [[(r[1], r[2], r[3]) for r in o.trace(k)] for k in range(K)]


@pytest.mark.parametrize("schedule", ["xpipe", "gpipe"])
@pytest.mark.parametrize("K,T", [(1, 1), (1, 3), (2, 1), (2, 4), (3, 2), (4, 1), (4, 2), (4, 4), (5, 3), (8, 1),
                                 (8, 4), (8, 8)])
def test_runtime_program_equals_oracle(oracle_mod, K, T, schedule):
    from paper_1911_04610_b200.xpipe import schedule_program
    M = 5
    U = M * T
    ref = oracle_ops(oracle_mod, K, T, M, schedule)
    for k in range(K):
        prog = schedule_program(K, T, k, 2 * U + 2 * K + 4, schedule)
        assert executed(prog, T, U) == ref[k], (K, T, k)


def test_runtime_program_paper_worked_example():
    """P:76 (K=4, T=2): GPU 0 runs micro-batch 5's forward before its backward of micro-batch 2
    finishes the first update, i.e. F1 F2 F3 F4 B1 F5 B2 ..., with the updates after B2 and B4
    preceding B5."""
    from paper_1911_04610_b200.xpipe import schedule_program
    prog = schedule_program(4, 2, 0, 13)
    s = " ".join("%s%d" % ("FB"[op], u) for op, u in prog)
    assert s == "F1 F2 F3 F4 B1 F5 B2 F6 B3 F7 B4 F8 B5"


def test_runtime_program_golden_traces():
    """The golden traces of reading R7 (tests/golden/): the product's op order per
    stage matches the F/B sequence recorded there."""
    from paper_1911_04610_b200.xpipe import schedule_program
    names = [f for f in os.listdir(GOLD) if f.startswith("trace_")]
    assert names
    for name in names:
        head = name[len("trace_"):-4]  # e.g. K4_T2_M3
        parts = dict((p[0], int(p[1:])) for p in head.split("_"))
        K, T, M = parts["K"], parts["T"], parts["M"]
        rows = {}
        with open(os.path.join(GOLD, name)) as f:
            for line in f:
                if line.startswith("#") or not line.strip():
                    continue
                k, rest = line.split(" ", 1)
                rows[int(k)] = [tok for tok in rest.split() if not tok.startswith("U")]
        for k, toks in rows.items():
            prog = executed(schedule_program(K, T, k, 2 * M * T + 2 * K + 4), T, M * T)
            got = ["%s%d.%d" % ("FB"[op], t, j) for op, t, j in prog if op != 2]
            want = [tok.split("@")[0] for tok in toks]
            assert got == want, (name, k)
