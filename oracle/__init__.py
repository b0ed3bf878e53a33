"""ctypes loader of the CPU oracle (liboracle.so) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_1911_04610_b200) never does; the two
share no code (the struct definitions below are this package's own).
"""
import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "xoracle.cpp")
_HDR = os.path.join(_HERE, "xoracle.h")

MODES = {"fp64": 0, "fp32": 1, "bf16": 2}
SCHEDULES = {"xpipe": 0, "gpipe": 1}
PREDICT = {"paper": 0, "off": 1, "fixed": 2}
DELTA = {"adam": 0, "paper": 1}
STATES = {"param": 0, "m": 1, "v": 2, "pred_fwd": 3, "pred_bwd": 4, "grad": 5, "buf": 6}
OPTIMIZERS = {"adam": 0, "sgd": 1}


def build(force=False):
    """Compile liboracle.so (plain C++17 + OpenMP, -ffp-contract=off, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["g++", "-std=c++17", "-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


class _Layer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "in_c", "out_c", "kh", "kw", "sh", "sw", "ph", "pw", "bias")] + \
               [("bn_eps", C.c_float)] + [(n, C.c_int32) for n in ("src0", "src1", "concat_off", "stage")]


class _Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("in_c", "in_h", "in_w", "classes", "mode", "schedule", "predict",
                                         "s_fwd", "s_bwd", "delta_form", "snapshots")] + \
               [("init_params", C.POINTER(C.POINTER(C.c_double))),
                ("init_m", C.POINTER(C.POINTER(C.c_double))),
                ("init_v", C.POINTER(C.POINTER(C.c_double))),
                ("optimizer", C.c_int32), ("momentum", C.c_double), ("weight_decay", C.c_double),
                ("recompute", C.c_int32)]


class _Trace(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("stage", "op", "t", "j", "version", "s", "bellwether")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.xo_init.restype = C.c_int
        _lib.xo_init.argtypes = [C.POINTER(_Layer), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.POINTER(_Config), C.POINTER(C.c_void_p)]
        _lib.xo_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        _lib.xo_get_param.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_size_t]
        _lib.xo_get_trace.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        _lib.xo_stage_of_layer.argtypes = [C.c_void_p, C.c_int32]
        _lib.xo_stage_version.argtypes = [C.c_void_p, C.c_int32]
        _lib.xo_param_count.restype = C.c_int64
        _lib.xo_param_count.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        _lib.xo_eval_loss_grad.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_double),
                                           C.c_void_p, C.c_size_t]
        _lib.xo_version_difference.argtypes = [C.c_int32] * 4
        _lib.xo_adam_predict.argtypes = [C.c_int32, C.c_int32, C.c_size_t] + [C.c_void_p] * 4 + \
            [C.c_int64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int32, C.c_int32] + [C.c_void_p] * 5
        _lib.xo_sgd_predict.argtypes = [C.c_int32, C.c_size_t] + [C.c_void_p] * 5 + [C.c_float] * 6 + \
            [C.c_int32, C.c_int32] + [C.c_void_p] * 6
        _lib.xo_finalize.argtypes = [C.c_void_p]
        _lib.xo_last_error.restype = C.c_char_p
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("oracle error %d: %s" % (code, msg))
        self.code = code


def _check(r):
    if r < 0:
        raise OracleError(r, lib().xo_last_error().decode())
    return r


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def version_difference(K, T, rank, pass_):
    """Eq. (1) (pass_=0) / Eq. (2) (pass_=1) as the oracle evaluates them."""
    return lib().xo_version_difference(K, T, rank, pass_)


def adam_predict(W, g, m, v, k, lr, betas, eps, s_f, s_b, mode="fp32", delta="adam"):
    W, g, m, v = (np.ascontiguousarray(a, dtype=np.float32) for a in (W, g, m, v))
    outs = [np.empty_like(W) for _ in range(5)]
    _check(lib().xo_adam_predict(MODES[mode], DELTA[delta], W.size, _ptr(W), _ptr(g), _ptr(m), _ptr(v), k,
                                 lr, betas[0], betas[1], eps, s_f, s_b, *[_ptr(o) for o in outs]))
    return outs  # W', m', v', W_hat_f, W_hat_b


def sgd_predict(W, g, buf, m, v, lr, betas, eps, momentum, weight_decay, s_f, s_b, mode="fp32"):
    """One Momentum-SGD step with the paper-literal prediction (f2), elementwise."""
    W, g, buf, m, v = (np.ascontiguousarray(a, dtype=np.float32) for a in (W, g, buf, m, v))
    outs = [np.empty_like(W) for _ in range(6)]
    _check(lib().xo_sgd_predict(MODES[mode], W.size, _ptr(W), _ptr(g), _ptr(buf), _ptr(m), _ptr(v), lr, betas[0],
                                betas[1], eps, momentum, weight_decay, s_f, s_b, *[_ptr(o) for o in outs]))
    return outs  # W', buf', m', v', W_hat_f, W_hat_b


class Oracle:
    """Stateful oracle context (mirrors the product's xpipe_init/step/get_weights/trace)."""

    def __init__(self, layers, stages, micro_batches, mini_batch, lr, betas, eps, in_shape, classes, params,
                 mode="fp64", schedule="xpipe", predict="paper", s_fwd=0, s_bwd=0, delta="adam",
                 snapshots=False, init_m=None, init_v=None, optimizer="adam", momentum=0.9, weight_decay=5e-4,
                 recompute=False):
        self.layers = list(layers)
        arr = (_Layer * len(self.layers))()
        for i, l in enumerate(self.layers):
            for f, _ in _Layer._fields_:
                setattr(arr[i], f, getattr(l, f))
        self._keep = []
        pp = (C.POINTER(C.c_double) * (2 * len(self.layers)))()
        for i, (w, b) in enumerate(params):
            for t, a in enumerate((w, b)):
                if a is not None:
                    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
                    self._keep.append(a)
                    pp[2 * i + t] = a.ctypes.data_as(C.POINTER(C.c_double))
        cfg = _Config(in_c=in_shape[0], in_h=in_shape[1], in_w=in_shape[2], classes=classes, mode=MODES[mode],
                      schedule=SCHEDULES[schedule], predict=PREDICT[predict], s_fwd=s_fwd, s_bwd=s_bwd,
                      delta_form=DELTA[delta], snapshots=int(snapshots), init_params=pp,
                      optimizer=OPTIMIZERS[optimizer], momentum=float(np.float32(momentum)),
                      weight_decay=float(np.float32(weight_decay)), recompute=int(recompute))
        for name, src in (("init_m", init_m), ("init_v", init_v)):
            if src is not None:
                tab = (C.POINTER(C.c_double) * stages)()
                for k, a in enumerate(src):
                    a = np.ascontiguousarray(a, dtype=np.float64)
                    self._keep.append(a)
                    tab[k] = a.ctypes.data_as(C.POINTER(C.c_double))
                self._keep.append(tab)
                setattr(cfg, name, tab)
        h = C.c_void_p()
        f32 = lambda a: float(np.float32(a))   # the C ABI of the product takes fp32 hyperparameters
        lr, betas, eps = f32(lr), (f32(betas[0]), f32(betas[1])), f32(eps)
        _check(lib().xo_init(arr, len(self.layers), stages, micro_batches, mini_batch, lr, betas[0], betas[1], eps,
                             C.byref(cfg), C.byref(h)))
        self.h = h
        self.K, self.T, self.N = stages, micro_batches, mini_batch
        self.in_shape, self.classes = tuple(in_shape), classes

    def close(self):
        if getattr(self, "h", None):
            lib().xo_finalize(self.h)
            self.h = None

    __del__ = close

    def step(self, x, y, M, flush=False):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.int32)
        assert x.shape[0] == M * self.N and y.shape[0] == M * self.N
        losses = np.empty(M * self.T, dtype=np.float32)
        _check(lib().xo_step(self.h, _ptr(x), _ptr(y), M, int(flush), _ptr(losses)))
        return losses

    def count(self, layer, tensor):
        return lib().xo_param_count(self.h, layer, tensor)

    def get(self, layer, tensor=0, state="param", version=-1, shape=True):
        n = self.count(layer, tensor)
        out = np.empty(n, dtype=np.float64)
        _check(lib().xo_get_param(self.h, layer, tensor, STATES[state], version, _ptr(out), n))
        return out

    def stage_of(self, layer):
        return _check(lib().xo_stage_of_layer(self.h, layer))

    def version(self, stage):
        return _check(lib().xo_stage_version(self.h, stage))

    def trace(self, stage):
        n = C.c_size_t()
        _check(lib().xo_get_trace(self.h, stage, None, 0, C.byref(n)))
        buf = (_Trace * max(1, n.value))()
        _check(lib().xo_get_trace(self.h, stage, buf, n.value, C.byref(n)))
        return [tuple(getattr(buf[i], f) for f, _ in _Trace._fields_) for i in range(n.value)]

    def eval_loss_grad(self, x, y):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.int32)
        total = sum(self.count(i, t) for i in range(len(self.layers)) for t in (0, 1))
        g = np.empty(total, dtype=np.float64)
        loss = C.c_double()
        _check(lib().xo_eval_loss_grad(self.h, _ptr(x), _ptr(y), x.shape[0], C.byref(loss), _ptr(g), total))
        return loss.value, g

    def params_flat(self, state="param", version=-1):
        return np.concatenate([self.get(i, t, state, version) for i in range(len(self.layers)) for t in (0, 1)])
