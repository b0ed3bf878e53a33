"""Layer lists of the paper's workloads (inputs to both the oracle and the CUDA path).

A model is a list of `Layer` records with the same fields as the C structs of both
libraries (kind, in_c, out_c, kh, kw, sh, sw, ph, pw, bias, bn_eps, src0, src1,
concat_off, stage).  src0/src1 = -1 means "previous layer".  stage = -1 selects the
layer-count partition rule.
"""
from dataclasses import dataclass, replace

LINEAR, CONV2D, BATCHNORM2D, RELU, MAXPOOL2D, AVGPOOL_GLOBAL, FLATTEN, ADD, CONCAT, SOFTMAX_XENT = range(1, 11)


@dataclass(frozen=True)
class Layer:
    kind: int
    in_c: int = 0
    out_c: int = 0
    kh: int = 0
    kw: int = 0
    sh: int = 1
    sw: int = 1
    ph: int = 0
    pw: int = 0
    bias: int = 0
    bn_eps: float = 1e-5
    src0: int = -1
    src1: int = -1
    concat_off: int = 0
    stage: int = -1

    def with_stage(self, s):
        return replace(self, stage=s)


def linear(i, o, bias=1):
    return Layer(LINEAR, in_c=i, out_c=o, bias=bias)


def conv(i, o, k, s=1, p=0, bias=0):
    kh, kw = (k, k) if isinstance(k, int) else k
    sh, sw = (s, s) if isinstance(s, int) else s
    ph, pw = (p, p) if isinstance(p, int) else p
    return Layer(CONV2D, in_c=i, out_c=o, kh=kh, kw=kw, sh=sh, sw=sw, ph=ph, pw=pw, bias=bias)


def bn(c, eps=1e-5):
    return Layer(BATCHNORM2D, in_c=c, out_c=c, bn_eps=eps)


def relu():
    return Layer(RELU)


def maxpool(k, s, p=0):
    return Layer(MAXPOOL2D, kh=k, kw=k, sh=s, sw=s, ph=p, pw=p)


def xent():
    return Layer(SOFTMAX_XENT)


def mlp(dims=(784, 256, 256, 256, 10)):
    """C1: the 4-layer MLP 784-256-256-256-10 (BASELINE.json configs[0])."""
    L = []
    for a, b in zip(dims[:-2], dims[1:-1]):
        L += [linear(a, b), relu()]
    L += [linear(dims[-2], dims[-1]), xent()]
    return L


VGG16_CFG = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def vgg16_cifar(classes=10, in_c=3):
    """C2: VGG-16 for CIFAR (R15): 13 x [conv3x3 p1 (no bias, R16), BN, ReLU], maxpool 2x2
    after convs 2, 4, 7, 10, 13; flatten; Linear 512 -> classes."""
    L, c = [], in_c
    for v in VGG16_CFG:
        if v == "M":
            L.append(maxpool(2, 2))
        else:
            L += [conv(c, v, 3, 1, 1), bn(v), relu()]
            c = v
    L += [Layer(FLATTEN), linear(512, classes), xent()]
    return L


def tiny_cnn(in_c=3, classes=10, width=16, pool=True):
    """A small conv/BN/ReLU/pool network for unit tests (not a BASELINE config)."""
    L = [conv(in_c, width, 3, 1, 1), bn(width), relu()]
    if pool:
        L.append(maxpool(2, 2))
    L += [conv(width, 2 * width, 3, 1, 1), bn(2 * width), relu(), Layer(AVGPOOL_GLOBAL),
          Layer(FLATTEN), linear(2 * width, classes), xent()]
    return L


def infer_shapes(layers, in_shape):
    """(C, H, W) of every layer's output; plain shape propagation (no arithmetic of the method)."""
    outs = []
    for i, l in enumerate(layers):
        s0 = i - 1 if l.src0 < 0 else l.src0
        x = in_shape if s0 < 0 else outs[s0]
        c, h, w = x
        if l.kind == LINEAR:
            o = (l.out_c, 1, 1)
        elif l.kind == CONV2D:
            o = (l.out_c, (h + 2 * l.ph - l.kh) // l.sh + 1, (w + 2 * l.pw - l.kw) // l.sw + 1)
        elif l.kind == MAXPOOL2D:
            o = (c, (h + 2 * l.ph - l.kh) // l.sh + 1, (w + 2 * l.pw - l.kw) // l.sw + 1)
        elif l.kind == AVGPOOL_GLOBAL:
            o = (c, 1, 1)
        elif l.kind == FLATTEN:
            o = (c * h * w, 1, 1)
        elif l.kind == CONCAT:
            y = outs[l.src1]
            o = (c + y[0], h, w)
        else:
            o = x
        outs.append(o)
    return outs
