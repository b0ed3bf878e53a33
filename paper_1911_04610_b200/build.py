"""Build libxpipe.so in-tree (sm_100a only): nvcc -gencode arch=compute_100a,code=sm_100a.

The fp32-contract translation units (sweep.cu, f32.cu) are compiled with --fmad=false on
top of their explicit round-to-nearest intrinsics, so no multiply-add is ever contracted.
"""
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
SO = os.path.join(HERE, "libxpipe.so")
ROOT = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
                 "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
STRICT = {"sweep.cu", "f32.cu"}


def sources():
    out = []
    for d in (CSRC, os.path.join(CSRC, "kernels")):
        for f in sorted(os.listdir(d)):
            if f.endswith(".cu"):
                out.append(os.path.join(d, f))
    return out


def headers():
    out = [os.path.join(ROOT, "include", "xpipe.h")]
    for d in (CSRC, os.path.join(CSRC, "kernels")):
        for f in os.listdir(d):
            if f.endswith(".h") or f.endswith(".cuh"):
                out.append(os.path.join(d, f))
    return out


def _compile(src, extra):
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    hdr_t = max(os.path.getmtime(h) for h in headers())
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
        return obj
    flags = list(COMMON) + list(extra) + os.environ.get("XPIPE_NVCC_EXTRA", "").split()
    if os.path.basename(src) in STRICT:
        flags.append("--fmad=false")
    cmd = [NVCC] + flags + ["-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, " ".join(cmd), r.stderr[-6000:]))
    os.replace(obj + ".tmp", obj)
    return obj


def build(force=False, verbose=False, extra=()):
    if not os.path.exists(NVCC) and not shutil.which("nvcc"):
        raise RuntimeError("nvcc not found: the CUDA extension cannot be built")
    os.makedirs(BUILD, exist_ok=True)
    if force:
        for f in os.listdir(BUILD):
            os.remove(os.path.join(BUILD, f))
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < newest:
        tmp = SO + ".tmp%d" % os.getpid()
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-Xlinker", "-z", "-Xlinker", "defs", "-o", tmp] + objs + ["-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s" % r.stderr[-4000:])
        os.replace(tmp, SO)
        if verbose:
            print("built", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
