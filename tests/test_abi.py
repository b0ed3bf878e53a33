"""CPU tests of the C-ABI boundary: the library builds for sm_100a, loads without a GPU and
exports every function include/xpipe.h declares; the product package never imports oracle/."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "xpipe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(xpipe_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def so():
    from paper_1911_04610_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("xpipe_init", "xpipe_step", "xpipe_get_weights", "xpipe_finalize", "xpipe_get_trace",
              "xpipe_adam_predict", "xpipe_gemm_bf16", "xpipe_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol(so):
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_loads_without_gpu(so):
    import ctypes
    L = ctypes.CDLL(so)
    L.xpipe_last_error.restype = ctypes.c_char_p
    L.xpipe_last_error.argtypes = [ctypes.c_void_p]
    assert L.xpipe_last_error(None) is not None
    assert L.xpipe_finalize(None) == 0


def test_init_validates_before_device_work(so):
    """XP_EINVAL for N % T != 0, lr <= 0, bad betas -- returned before any CUDA call."""
    import numpy as np
    import synthetic as S
    from paper_1911_04610_b200 import XPipe, XPipeError
    L = S.mlp()
    for kw in (dict(mini_batch=30, micro_batches=4), dict(lr=0.0), dict(betas=(1.0, 0.999))):
        args = dict(stages=2, micro_batches=4, mini_batch=32, lr=1e-3, betas=(0.9, 0.999))
        args.update(kw)
        with pytest.raises(XPipeError) as e:
            XPipe(L, args["stages"], args["micro_batches"], args["mini_batch"], args["lr"], args["betas"], 1e-8,
                  (784, 1, 1), 10, torch_allocator=False)
        assert e.value.code == -1


def test_product_package_does_not_import_oracle():
    code = "import sys, paper_1911_04610_b200; assert 'oracle' not in sys.modules; print('ok')"
    out = subprocess.check_output([sys.executable, "-c", code], cwd=ROOT, text=True)
    assert "ok" in out


def test_no_oracle_reference_in_product_sources():
    pkg = os.path.join(ROOT, "paper_1911_04610_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "xoracle" not in txt and "liboracle" not in txt, f


def test_sgd_optimizer_validation(so):
    """XP_OPT_MOMENTUM_SGD (f2) needs the paper prediction form and a momentum in [0, 1):
    XP_EINVAL before any device work otherwise."""
    import synthetic as S
    from paper_1911_04610_b200 import XPipe, XPipeError
    L = S.mlp()
    for kw in (dict(delta="adam"), dict(delta="paper", momentum=1.0), dict(delta="paper", weight_decay=-1.0)):
        with pytest.raises(XPipeError) as e:
            XPipe(L, 2, 4, 32, 1e-2, (0.9, 0.999), 1e-8, (784, 1, 1), 10, torch_allocator=False, optimizer="sgd",
                  **kw)
        assert e.value.code == -1
