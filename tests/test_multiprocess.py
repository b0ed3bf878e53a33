"""The one-process-per-GPU mode: host plumbing with gloo world size 2 on CPU, and
(on a GPU box) two processes sharing one B200 through CUDA IPC-mapped rings and flags running
the C1 MLP pipeline, each stage bit-exact with the oracle."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_1911_04610_b200.xpipe import exchange_blobs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blobs = exchange_blobs(b"stage-%d" % rank + bytes(range(rank, rank + 40)))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, blobs))


def test_blob_exchange_gloo_world2():
    """Every rank receives every rank's IPC blob, in rank order (the plumbing connect_pipeline
    uses before the first xpipe_step)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [b"stage-%d" % r + bytes(range(r, r + 40)) for r in range(2)]
    assert res[0] == expect and res[1] == expect


def test_multiprocess_validation_without_gpu():
    """my_stage out of range is rejected before any device work."""
    import synthetic as S
    from paper_1911_04610_b200 import XPipe, XPipeError
    with pytest.raises(XPipeError) as e:
        XPipe(S.mlp(), 2, 4, 32, 1e-3, (0.9, 0.999), 1e-8, (784, 1, 1), 10, my_stage=2, torch_allocator=False)
    assert e.value.code == -1


def _ipc_worker(rank, world, port, q, overlap=False, graphs=False):
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist
        import synthetic as S
        from paper_1911_04610_b200 import XPipe, connect_pipeline
        torch.cuda.set_device(0)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        L = S.mlp()
        P = S.make_params(L, 1)
        M = 24 if graphs else 10
        x, y = S.make_inputs(M * 32, (784, 1, 1), 10, 1, kind="mnist")
        g = XPipe(L, world, 4, 32, 1e-3, (0.9, 0.999), 1e-8, (784, 1, 1), 10, params=P, precision="fp32",
                  trace=not graphs, my_stage=rank, watchdog_ms=60000, fb_overlap=overlap, graphs=graphs)
        connect_pipeline(g)
        dist.barrier()
        replays = 0
        if graphs:
            # 2 mini-batches per call: steady-state calls are captured per process (device-side
            # flag kernels on the call's base) and replayed, the processes never synchronising
            for i in range(12):
                sl = slice(i * 64, (i + 1) * 64)
                g.step(x[sl], y[sl], 2)
                replays += g.last_stats.graph_replays
            g.step(x[:0], y[:0], 0, flush=True)
        else:
            g.step(x[:96], y[:96], 3)             # call splitting across processes too
            g.step(x[96:], y[96:], 7, flush=True)
        out = {(i, t): g.get(i, t) for i in range(len(L)) for t in (0, 1) if g.stage_of(i) == rank and g._count(i, t)}
        q.put((rank, out, None if graphs else g.trace(rank), replays))
        dist.barrier()
        g.close()
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        q.put((rank, repr(e), None, 0))


@pytest.mark.gpu
@pytest.mark.parametrize("overlap,graphs", [(False, False), (True, False), (False, True), (True, True)])
def test_two_process_pipeline_one_gpu(oracle_mod, overlap, graphs):
    """Two processes, one stage each, rings and flags shared through CUDA IPC on one B200:
    weights (and, without graphs, traces) bit-exact with the oracle's K=2 replay; with graphs
    each process captures and replays its own stage's steady-state calls."""
    import torch.multiprocessing as mp
    import synthetic as S
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, overlap, graphs)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, w, tr, reps = q.get(timeout=600)
        assert not isinstance(w, str), w
        res[r] = (w, tr, reps)
    for p in procs:
        p.join(timeout=120)
    L = S.mlp()
    P = S.make_params(L, 1)
    M = 24 if graphs else 10
    x, y = S.make_inputs(M * 32, (784, 1, 1), 10, 1, kind="mnist")
    o = oracle_mod.Oracle(L, 2, 4, 32, 1e-3, (0.9, 0.999), 1e-8, (784, 1, 1), 10, P, mode="fp32")
    o.step(x, y, M, flush=True)
    for r in range(2):
        w, tr, reps = res[r]
        if graphs:
            assert reps >= 4, (r, reps)
        else:
            assert tr == o.trace(r)
        for (i, t), a in w.items():
            assert np.array_equal(a, o.get(i, t).astype(np.float32)), (r, i, t)
