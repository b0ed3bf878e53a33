"""Thin ctypes binding of libxpipe.so (include/xpipe.h).  Argument marshalling only: every
step of the hot path runs in the library's CUDA kernels.  PyTorch is used for device memory
(the allocator hooks route to torch's caching allocator) and nothing else.

Fails loudly when the extension is missing -- there is no CPU fallback.
"""
import ctypes as C
import os

# A pipeline stage enqueues on two or three streams (backward/update, forward, weight gradient);
# with K stages on one device the CUDA default of 8 hardware work queues makes independent
# streams wait on each other (VGG-16 K=4 on one B200: 99.5k -> 117k samples/s, timed-run bubble
# 0.27 -> 0.09 with 32).  Read when the CUDA context is created, so it is set at import, before
# the first CUDA call; libxpipe.so sets the same default for C callers (xpipe.cu).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libxpipe.so")

XP_OK, XP_EINVAL, XP_ENOMEM, XP_ECUDA, XP_ECOMM, XP_ESCHED, XP_ENONFINITE, XP_ESTATE, XP_EUNSUPPORTED = \
    0, -1, -2, -3, -4, -5, -6, -7, -8
PRECISION = {"fp32": 0, "bf16": 1}
SCHEDULE = {"xpipe": 0, "gpipe": 1}
PREDICT = {"paper": 0, "off": 1, "fixed": 2}
DELTA = {"adam": 0, "paper": 1}
STATE = {"param": 0, "m": 1, "v": 2, "pred_fwd": 3, "pred_bwd": 4, "grad": 5, "buf": 6}
OPTIMIZER = {"adam": 0, "sgd": 1}
WBWD = {"materialize": 0, "bellwether": 1}
XP_FLUSH, XP_DEVICE_PTRS, XP_ASYNC = 1, 2, 4


class Layer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "in_c", "out_c", "kh", "kw", "sh", "sw", "ph", "pw", "bias")] + \
               [("bn_eps", C.c_float)] + [(n, C.c_int32) for n in ("src0", "src1", "concat_off", "stage")]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p)


class Config(C.Structure):
    _fields_ = [("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32), ("classes", C.c_int32),
                ("seed", C.c_uint64)] + \
               [(n, C.c_int32) for n in ("precision", "schedule", "predict", "s_fwd", "s_bwd", "delta_form",
                                         "moment_init", "n_devices")] + \
               [("devices", C.c_int32 * 8)] + \
               [(n, C.c_int32) for n in ("transport", "snapshots", "trace", "graphs", "profile", "watchdog_ms",
                                         "multi_process", "my_stage")] + \
               [("init_params", C.POINTER(C.POINTER(C.c_float))),
                ("init_m", C.POINTER(C.POINTER(C.c_float))),
                ("init_v", C.POINTER(C.POINTER(C.c_float))),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_user", C.c_void_p),
                ("optimizer", C.c_int32), ("momentum", C.c_float), ("weight_decay", C.c_float),
                ("recompute", C.c_int32), ("serialize", C.c_int32), ("fb_overlap", C.c_int32),
                ("timing", C.c_int32), ("wbwd", C.c_int32)]


class TraceRec(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("stage", "op", "t", "j", "version", "s", "bellwether", "wbuf")] + \
               [("t0_ns", C.c_uint64), ("t1_ns", C.c_uint64)]


PROF_CLASSES = ("sweep", "conv_fprop", "conv_dgrad", "conv_wgrad", "bn_stats", "bn_apply", "bn_bwd_reduce",
                "bn_bwd_apply")
BYTE_CLASSES = ("sweep", "bn_stats", "bn_apply", "bn_bwd_reduce", "bn_bwd_apply")  # work in bytes (else flops)


STATS_STAGES = 16


class Stats(C.Structure):
    _fields_ = [("span_ms", C.c_double), ("prof_ms", C.c_double * 8), ("prof_launches", C.c_int64 * 8),
                ("prof_work", C.c_double * 8), ("kernel_launches", C.c_int64), ("graph_replays", C.c_int64),
                ("losses", C.POINTER(C.c_float)),
                ("busy_ms", C.c_double * STATS_STAGES), ("bubble_fraction", C.c_double),
                ("steady_samples_per_s", C.c_double),
                ("p2p_fwd_ms", C.c_double * STATS_STAGES), ("p2p_bwd_ms", C.c_double * STATS_STAGES),
                ("p2p_fwd_bytes", C.c_double * STATS_STAGES), ("p2p_bwd_bytes", C.c_double * STATS_STAGES),
                ("ops_timed", C.c_int64)]

    def timing(self, K):
        """cfg.timing fields as a dict (stages 0..K-1)."""
        k = min(K, STATS_STAGES)
        return dict(span_ms=self.span_ms, busy_ms=list(self.busy_ms[:k]), bubble_fraction=self.bubble_fraction,
                    steady_samples_per_s=self.steady_samples_per_s, p2p_fwd_ms=list(self.p2p_fwd_ms[:k]),
                    p2p_bwd_ms=list(self.p2p_bwd_ms[:k]), p2p_fwd_bytes=list(self.p2p_fwd_bytes[:k]),
                    p2p_bwd_bytes=list(self.p2p_bwd_bytes[:k]), ops_timed=self.ops_timed)

    def profile(self):
        return {n: dict(ms=self.prof_ms[i], launches=self.prof_launches[i], work=self.prof_work[i])
                for i, n in enumerate(PROF_CLASSES)}


_lib = None


def lib():
    """Load libxpipe.so; raise if it was not built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError("libxpipe.so not built: run paper_1911_04610_b200/build.py (no CPU fallback)")
        L = C.CDLL(SO_PATH)
        vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        L.xpipe_init.argtypes = [C.POINTER(Layer), i32, i32, i32, i32, f32, C.POINTER(f32), f32, C.POINTER(Config),
                                 C.POINTER(vp)]
        L.xpipe_step.argtypes = [vp, vp, vp, i32, C.c_uint32, C.POINTER(Stats)]
        L.xpipe_sync.argtypes = [vp]
        L.xpipe_timer.argtypes = [vp, i32, C.POINTER(C.c_double)]
        L.xpipe_ipc_export.argtypes = [vp, vp, C.c_size_t, C.POINTER(C.c_size_t)]
        L.xpipe_ipc_import.argtypes = [vp, vp, C.c_size_t]
        L.xpipe_get_weights.argtypes = [vp, i32, i32, i32, i64, vp, C.c_size_t]
        L.xpipe_get_trace.argtypes = [vp, i32, vp, C.c_size_t, C.POINTER(C.c_size_t)]
        L.xpipe_stage_of_layer.argtypes = [vp, i32]
        L.xpipe_stage_version.argtypes = [vp, i32]
        L.xpipe_stage_params.argtypes = [vp, i32]
        L.xpipe_stage_params.restype = i64
        L.xpipe_finalize.argtypes = [vp]
        L.xpipe_last_error.argtypes = [vp]
        L.xpipe_last_error.restype = C.c_char_p
        L.xpipe_adam_predict.argtypes = [vp, vp, vp, vp, vp, vp, i64, i64, f32, f32, f32, f32, i32, i32, i32, i32, vp]
        L.xpipe_sgd_predict.argtypes = [vp, vp, vp, vp, vp, vp, vp, i64, f32, f32, f32, f32, f32, f32, i32, i32, i32,
                                        vp]
        L.xpipe_set_weights.argtypes = [vp, i32, i32, i32, vp, C.c_size_t]
        L.xpipe_refresh_predictions.argtypes = [vp]
        L.xpipe_gemm_bf16.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, i64, vp]
        L.xpipe_conv2d_bf16.argtypes = [i32, C.POINTER(i32), vp, vp, vp, i32, vp, i64, vp]
        L.xpipe_linear_bf16.argtypes = [i32, vp, vp, vp, vp, i32, vp, i32, i32, i32, i32, i32, i32, vp, i64, vp]
        L.xpipe_schedule_program.argtypes = [i32, i32, i32, i32, i64, vp, vp]
        _lib = L
    return _lib


class XPipeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("xpipe error %d: %s" % (code, msg))
        self.code = code


def _check(r, h=None):
    if r < 0:
        raise XPipeError(r, lib().xpipe_last_error(h).decode())
    return r


def _torch_allocator():
    import torch

    def alloc(nbytes, device, user):
        return torch.cuda.caching_allocator_alloc(int(nbytes), device=int(device))

    def free(ptr, nbytes, device, user):
        torch.cuda.caching_allocator_delete(ptr)
    return ALLOC_FN(alloc), FREE_FN(free)


def _ptr(a):
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


class XPipe:
    """One pipeline context: xpipe_init / xpipe_step / xpipe_get_weights / xpipe_get_trace /
    xpipe_finalize."""

    def __init__(self, layers, stages, micro_batches, mini_batch, lr, betas, eps, in_shape, classes, params=None,
                 precision="fp32", schedule="xpipe", predict=None, s_fwd=0, s_bwd=0, delta="adam",
                 init_m=None, init_v=None, devices=None, snapshots=False, trace=False, graphs=False, profile=False,
                 seed=1, watchdog_ms=0, torch_allocator=True, my_stage=None, optimizer="adam", momentum=0.9,
                 weight_decay=5e-4, recompute=False, serialize=False, fb_overlap=False, timing=False,
                 wbwd="materialize"):
        self.h = None
        L = lib()
        if predict is None:  # GPipe runs under the current weights (no prediction)
            predict = "off" if schedule == "gpipe" else "paper"
        self.layers = list(layers)
        arr = (Layer * len(self.layers))()
        for i, l in enumerate(self.layers):
            for f, _ in Layer._fields_:
                setattr(arr[i], f, getattr(l, f))
        self._keep = []
        cfg = Config(in_c=in_shape[0], in_h=in_shape[1], in_w=in_shape[2], classes=classes, seed=seed,
                     precision=PRECISION[precision], schedule=SCHEDULE[schedule], predict=PREDICT[predict],
                     s_fwd=s_fwd, s_bwd=s_bwd, delta_form=DELTA[delta], snapshots=int(snapshots), trace=int(trace),
                     graphs=int(graphs), profile=int(profile), watchdog_ms=watchdog_ms,
                     multi_process=int(my_stage is not None), my_stage=my_stage or 0,
                     optimizer=OPTIMIZER[optimizer], momentum=momentum if optimizer == "sgd" else 0.0,
                     weight_decay=weight_decay if optimizer == "sgd" else 0.0, recompute=int(recompute),
                     serialize=int(serialize), fb_overlap=int(fb_overlap), timing=int(timing),  # bool -> every call
                     wbwd=WBWD[wbwd])
        if devices:
            cfg.n_devices = len(devices)
            for i, d in enumerate(devices):
                cfg.devices[i] = d

        def table(src):
            tab = (C.POINTER(C.c_float) * (2 * len(self.layers)))()
            for i, pair in enumerate(src):
                for t, a in enumerate(pair):
                    if a is not None:
                        a = np.ascontiguousarray(a, dtype=np.float32).ravel()
                        self._keep.append(a)
                        tab[2 * i + t] = a.ctypes.data_as(C.POINTER(C.c_float))
            self._keep.append(tab)
            return tab
        if params is not None:
            cfg.init_params = table(params)
        if init_m is not None:
            cfg.moment_init = 1
            cfg.init_m = table(init_m)
            cfg.init_v = table(init_v)
        if torch_allocator:
            self._alloc = _torch_allocator()
            cfg.alloc, cfg.free = self._alloc
        b = (C.c_float * 2)(*betas)
        h = C.c_void_p()
        r = L.xpipe_init(arr, len(self.layers), stages, micro_batches, mini_batch, lr, b, eps, C.byref(cfg),
                         C.byref(h))
        _check(r, None)
        self.h = h
        self.K, self.T, self.N = stages, micro_batches, mini_batch
        self.in_shape, self.classes = tuple(in_shape), classes

    def close(self):
        if self.h:
            lib().xpipe_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, x, y, M, flush=False, async_=False, losses=True, loss_out=None):
        """x: [M*N, C, H, W] float32, y: [M*N] int32 -- numpy (host) or torch CUDA tensors (device).
        async_: return after enqueue (XP_ASYNC; replays of captured graphs then chain on the device);
        loss_out: a caller buffer of M*T float32 (pinned host memory for an asynchronous copy)
        receiving the losses, valid after the next synchronous call or sync()."""
        flags = (XP_FLUSH if flush else 0) | (XP_ASYNC if async_ else 0)
        per = self.in_shape[0] * self.in_shape[1] * self.in_shape[2]
        if hasattr(x, "is_cuda") and x.is_cuda:
            if not (hasattr(y, "is_cuda") and y.is_cuda):
                raise TypeError("x and y must both be CUDA tensors or both host arrays")
            _want("x", x, ("float32",), M * self.N * per)
            _want("y", y, ("int32",), M * self.N)
            flags |= XP_DEVICE_PTRS
        else:
            x = np.ascontiguousarray(x, dtype=np.float32)
            y = np.ascontiguousarray(y, dtype=np.int32)
        st = Stats()
        out = None
        if loss_out is not None:
            _want("loss_out", loss_out, ("float32",), M * self.T)
            st.losses = C.cast(_ptr(loss_out), C.POINTER(C.c_float))
            out = loss_out
        elif losses and not async_:
            out = np.empty(M * self.T, dtype=np.float32)
            st.losses = out.ctypes.data_as(C.POINTER(C.c_float))
        _check(lib().xpipe_step(self.h, _ptr(x), _ptr(y), M, flags, C.byref(st)), self.h)
        self.last_stats = st
        return out

    def ipc_export(self):
        buf = C.create_string_buffer(4096)
        n = C.c_size_t()
        _check(lib().xpipe_ipc_export(self.h, buf, 4096, C.byref(n)), self.h)
        return buf.raw[:n.value]

    def ipc_import(self, blob):
        b = C.create_string_buffer(blob, len(blob))
        _check(lib().xpipe_ipc_import(self.h, b, len(blob)), self.h)

    def timer_start(self):
        _check(lib().xpipe_timer(self.h, 0, None), self.h)

    def timer_stop(self):
        ms = C.c_double()
        _check(lib().xpipe_timer(self.h, 1, C.byref(ms)), self.h)
        return ms.value

    def sync(self):
        _check(lib().xpipe_sync(self.h), self.h)

    def get(self, layer, tensor=0, state="param", version=-1, count=None):
        if count is None:
            count = self._count(layer, tensor)
        out = np.empty(count, dtype=np.float32)
        _check(lib().xpipe_get_weights(self.h, layer, tensor, STATE[state], version, _ptr(out), count), self.h)
        return out

    def set(self, layer, tensor, state, values):
        """xpipe_set_weights: overwrite one tensor's W / m / v / buf (PyTorch layout)."""
        a = np.ascontiguousarray(values, dtype=np.float32).ravel()
        _check(lib().xpipe_set_weights(self.h, layer, tensor, STATE[state], _ptr(a), a.size), self.h)

    def refresh_predictions(self):
        """xpipe_refresh_predictions: rematerialise W_hat_f / W_hat_b from the current state."""
        _check(lib().xpipe_refresh_predictions(self.h), self.h)

    def _count(self, layer, tensor):
        l = self.layers[layer]
        kinds_w = {1: lambda: l.out_c * l.in_c, 2: lambda: l.out_c * l.in_c * l.kh * l.kw, 3: lambda: l.in_c}
        if tensor == 0:
            return kinds_w[l.kind]() if l.kind in kinds_w else 0
        if l.kind == 3:
            return l.in_c
        return l.out_c if (l.kind in (1, 2) and l.bias) else 0

    def params_flat(self, state="param", version=-1):
        parts = []
        for i in range(len(self.layers)):
            for t in (0, 1):
                n = self._count(i, t)
                if n:
                    parts.append(self.get(i, t, state, version, n))
        return np.concatenate(parts)

    def stage_of(self, layer):
        return _check(lib().xpipe_stage_of_layer(self.h, layer), self.h)

    def version(self, stage):
        return _check(lib().xpipe_stage_version(self.h, stage), self.h)

    def stage_params(self, stage):
        return lib().xpipe_stage_params(self.h, stage)

    def trace(self, stage, timestamps=False):
        n = C.c_size_t()
        _check(lib().xpipe_get_trace(self.h, stage, None, 0, C.byref(n)), self.h)
        buf = (TraceRec * max(1, n.value))()
        _check(lib().xpipe_get_trace(self.h, stage, buf, n.value, C.byref(n)), self.h)
        f = [x for x, _ in TraceRec._fields_][:7 + (3 if timestamps else 0)]
        return [tuple(getattr(buf[i], q) for q in f) for i in range(n.value)]


def _want(name, t, dtypes, n=None):
    """Marshalling check (the C ABI sees only pointers): element type, contiguity, size."""
    if t is None:
        return
    dt = str(getattr(t, "dtype", ""))
    if not any(dt.endswith(d) for d in dtypes):
        raise TypeError("%s: dtype %s, expected %s" % (name, dt, "/".join(dtypes)))
    if hasattr(t, "is_contiguous") and not t.is_contiguous():
        raise ValueError("%s must be contiguous" % name)
    if n is not None and t.numel() < n:
        raise ValueError("%s has %d elements, needs %d" % (name, t.numel(), n))
    if hasattr(t, "data_ptr") and t.data_ptr() % 16:
        raise ValueError("%s must be 16-byte aligned" % name)


def adam_predict(W, g, m, v, pf, pb, version, lr, betas, eps, s_f, s_b, pred_bf16, delta="adam", stream=None):
    """K1 on torch CUDA tensors (in place on W, m, v)."""
    n = W.numel()
    for nm, t in (("W", W), ("g", g), ("m", m), ("v", v)):
        _want(nm, t, ("float32",), n)
    for nm, t in (("pf", pf), ("pb", pb)):
        _want(nm, t, ("bfloat16",) if pred_bf16 else ("float32",), n)
    _check(lib().xpipe_adam_predict(_ptr(W), _ptr(g), _ptr(m), _ptr(v), _ptr(pf) if pf is not None else None,
                                    _ptr(pb) if pb is not None else None, n, version, lr, betas[0], betas[1], eps,
                                    s_f, s_b, int(pred_bf16), DELTA[delta],
                                    C.c_void_p(stream) if stream else None))


def sgd_predict(W, g, buf, m, v, pf, pb, lr, betas, eps, momentum, weight_decay, s_f, s_b, pred_bf16, stream=None):
    """The f2 sweep (Momentum SGD + paper-literal prediction) on torch CUDA tensors, in place."""
    n = W.numel()
    for nm, t in (("W", W), ("g", g), ("buf", buf), ("m", m), ("v", v)):
        _want(nm, t, ("float32",), n)
    for nm, t in (("pf", pf), ("pb", pb)):
        _want(nm, t, ("bfloat16",) if pred_bf16 else ("float32",), n)
    _check(lib().xpipe_sgd_predict(_ptr(W), _ptr(g), _ptr(buf), _ptr(m), _ptr(v), _ptr(pf) if pf is not None else None,
                                   _ptr(pb) if pb is not None else None, n, lr, betas[0], betas[1], eps, momentum,
                                   weight_decay, s_f, s_b, int(pred_bf16), C.c_void_p(stream) if stream else None))


def gemm_bf16(A, B, D, M, N, K, a_kmajor=True, b_kmajor=True, ldd=None, stream=None):
    _want("A", A, ("bfloat16",), M * K)
    _want("B", B, ("bfloat16",), N * K)
    _want("D", D, ("float32",))
    _check(lib().xpipe_gemm_bf16(_ptr(A), _ptr(B), _ptr(D), M, N, K, int(a_kmajor), int(b_kmajor),
                                 ldd if ldd is not None else N, C.c_void_p(stream) if stream else None))


def conv2d_bf16(mode, geo, in0, in1, out, accumulate=False, ws=None, stream=None):
    """mode 1 fprop / 2 dgrad / 3 wgrad / 4, 5 fprop, wgrad via explicit im2col;
    geo = (Nimg, H, W, C, Co, R, S, P, Q, sh, sw, ph, pw)."""
    _want("in0", in0, ("bfloat16",))
    _want("in1", in1, ("bfloat16",))
    _want("out", out, ("float32",) if mode in (3, 5) else ("bfloat16",))
    _want("ws", ws, ("float32",))
    g = (C.c_int32 * 13)(*geo)
    _check(lib().xpipe_conv2d_bf16(mode, g, _ptr(in0), _ptr(in1), _ptr(out), int(accumulate),
                                   _ptr(ws) if ws is not None else None, ws.numel() if ws is not None else 0,
                                   C.c_void_p(stream) if stream else None))


def linear_bf16(mode, out, n, in_f, out_f, x=None, W=None, b=None, dy=None, ldp=0, relu=False, f32out=False,
                accumulate=False, ws=None, stream=None):
    """mode 1 forward (x, W, b -> out [n][out_f]) / 2 dgrad (dy [n][ldp], W -> out [n][in_f]) /
    3 wgrad (x, dy -> out [out_f][in_f] fp32); see xpipe_linear_bf16 in include/xpipe.h."""
    for nm, t in (("x", x), ("W", W), ("b", b), ("dy", dy)):
        if t is not None:
            _want(nm, t, ("bfloat16",))
    _want("out", out, ("float32",) if (mode == 3 or (mode == 1 and f32out)) else ("bfloat16",))
    _want("ws", ws, ("float32",))
    p = lambda t: _ptr(t) if t is not None else None
    _check(lib().xpipe_linear_bf16(mode, p(x), p(W), p(b), p(dy), ldp, _ptr(out), n, in_f, out_f, int(relu),
                                   int(f32out), int(accumulate), p(ws), ws.numel() if ws is not None else 0,
                                   C.c_void_p(stream) if stream else None))


def exchange_blobs(blob, group=None):
    """All-gather one opaque bytes blob per rank over torch.distributed (any backend);
    returns the list ordered by rank.  Host-side plumbing of the multi-process mode."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def connect_pipeline(model, group=None):
    """One-process-per-GPU mode: exchange the CUDA IPC handles of every stage's rings and
    flags, then attach this process's neighbours (xpipe_ipc_import)."""
    blobs = exchange_blobs(model.ipc_export(), group)
    for b in blobs:
        model.ipc_import(b)
    return blobs


def schedule_program(stages, micro_batches, stage, n, schedule="xpipe"):
    """xpipe_schedule_program: the first n (op, u) of a stage's program (host-only)."""
    ops = np.empty(n, np.int32)
    us = np.empty(n, np.int64)
    _check(lib().xpipe_schedule_program(stages, micro_batches, SCHEDULE[schedule], stage, n, _ptr(ops), _ptr(us)))
    return list(zip(ops.tolist(), us.tolist()))
