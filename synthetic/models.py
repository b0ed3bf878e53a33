"""Layer lists of the paper's workloads (inputs to both the oracle and the CUDA path).

A model is a list of `Layer` records with the same fields as the C structs of both
libraries (kind, in_c, out_c, kh, kw, sh, sw, ph, pw, bias, bn_eps, src0, src1,
concat_off, stage).  src0/src1 = -1 means "previous layer".  stage = -1 selects the
layer-count partition rule.
"""
from dataclasses import dataclass, replace

LINEAR, CONV2D, BATCHNORM2D, RELU, MAXPOOL2D, AVGPOOL_GLOBAL, FLATTEN, ADD, CONCAT, SOFTMAX_XENT, AVGPOOL2D = range(1, 12)


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


def avgpool(k, s, p=0):
    return Layer(AVGPOOL2D, kh=k, kw=k, sh=s, sw=s, ph=p, pw=p)


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
        elif l.kind in (MAXPOOL2D, AVGPOOL2D):
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


# ---------------------------------------------------------------------------------------
# DAG models (configs C3, C4).  Built as layer lists with explicit producer indices; each
# layer carries the partition unit it belongs to (R17) so `assign_stages` can apply the
# layer-count rule over units and write explicit stage ids (skip/branch edges never cross).
# ---------------------------------------------------------------------------------------
class Builder:
    def __init__(self):
        self.L, self.units, self.unit = [], [], 0

    def add(self, layer, src0=None, src1=None):
        kw = {}
        if src0 is not None:
            kw["src0"] = src0
        if src1 is not None:
            kw["src1"] = src1
        self.L.append(replace(layer, **kw))
        self.units.append(self.unit)
        return len(self.L) - 1

    def next_unit(self):
        self.unit += 1

    def conv_bn(self, src, i, o, k, s=1, p=0, relu_=True, eps=1e-5):
        a = self.add(conv(i, o, k, s, p), src0=src)
        b = self.add(bn(o, eps), src0=a)
        return self.add(relu(), src0=b) if relu_ else b

    def concat(self, srcs):
        cur = srcs[0]
        for s in srcs[1:]:
            cur = self.add(Layer(CONCAT), src0=cur, src1=s)
        return cur


def _bottleneck(B, x, inplanes, planes, stride):
    a = B.conv_bn(x, inplanes, planes, 1)
    a = B.conv_bn(a, planes, planes, 3, stride, 1)
    a = B.conv_bn(a, planes, 4 * planes, 1, relu_=False)
    sc = x
    if stride != 1 or inplanes != 4 * planes:
        sc = B.conv_bn(x, inplanes, 4 * planes, 1, stride, 0, relu_=False)
    s = B.add(Layer(ADD), src0=a, src1=sc)
    return B.add(relu(), src0=s)


def resnet101(classes=200, in_c=3, layers=(3, 4, 23, 3)):
    """C3: torchvision ResNet-101 (v1.5: stride on the 3x3 conv), 64x64 input, no change
    other than the input size (R19).  Units: stem / each bottleneck / head (35 units)."""
    B = Builder()
    x = B.conv_bn(-1, in_c, 64, 7, 2, 3)
    x = B.add(maxpool(3, 2, 1), src0=x)
    inplanes = 64
    for li, (planes, n) in enumerate(zip((64, 128, 256, 512), layers)):
        for b in range(n):
            B.next_unit()
            stride = 2 if (b == 0 and li > 0) else 1
            x = _bottleneck(B, x, inplanes, planes, stride)
            inplanes = 4 * planes
    B.next_unit()
    x = B.add(Layer(AVGPOOL_GLOBAL), src0=x)
    x = B.add(Layer(FLATTEN), src0=x)
    x = B.add(linear(2048, classes), src0=x)
    B.add(xent(), src0=x)
    return B.L, B.units


def inception_v3(classes=200, in_c=3, stem_pad=True):
    """C4: torchvision Inception-V3 with aux_logits off and no dropout, padding 1 on the
    unpadded stem convs Conv2d_1a, 2a, 4a so 64x64 inputs survive to Mixed_7 (R14).
    stem_pad=False: the unmodified torchvision stem, for the paper's 224x224 inputs (f4).
    BasicConv2d = conv (no bias) + BN(eps=1e-3) + ReLU.  Units: stem conv / module / head."""
    B = Builder()
    e = 1e-3
    sp = 1 if stem_pad else 0
    cb = lambda src, i, o, k, s=1, p=0: B.conv_bn(src, i, o, k, s, p, True, e)
    x = cb(-1, in_c, 32, 3, 2, sp)                      # Conv2d_1a (padded at 64x64, R14)
    B.next_unit(); x = cb(x, 32, 32, 3, 1, sp)          # Conv2d_2a
    B.next_unit(); x = cb(x, 32, 64, 3, 1, 1)           # Conv2d_2b
    x = B.add(maxpool(3, 2), src0=x)
    B.next_unit(); x = cb(x, 64, 80, 1)                 # Conv2d_3b
    B.next_unit(); x = cb(x, 80, 192, 3, 1, sp)         # Conv2d_4a
    x = B.add(maxpool(3, 2), src0=x)

    def incA(x, cin, pf):
        b1 = cb(x, cin, 64, 1)
        b5 = cb(cb(x, cin, 48, 1), 48, 64, 5, 1, 2)
        b3 = cb(cb(cb(x, cin, 64, 1), 64, 96, 3, 1, 1), 96, 96, 3, 1, 1)
        bp = cb(B.add(avgpool(3, 1, 1), src0=x), cin, pf, 1)
        return B.concat([b1, b5, b3, bp])

    def incB(x, cin):
        b3 = cb(x, cin, 384, 3, 2)
        bd = cb(cb(cb(x, cin, 64, 1), 64, 96, 3, 1, 1), 96, 96, 3, 2)
        bp = B.add(maxpool(3, 2), src0=x)
        return B.concat([b3, bd, bp])

    def incC(x, c7):
        b1 = cb(x, 768, 192, 1)
        b7 = cb(cb(cb(x, 768, c7, 1), c7, c7, (1, 7), 1, (0, 3)), c7, 192, (7, 1), 1, (3, 0))
        d = cb(x, 768, c7, 1)
        d = cb(d, c7, c7, (7, 1), 1, (3, 0))
        d = cb(d, c7, c7, (1, 7), 1, (0, 3))
        d = cb(d, c7, c7, (7, 1), 1, (3, 0))
        d = cb(d, c7, 192, (1, 7), 1, (0, 3))
        bp = cb(B.add(avgpool(3, 1, 1), src0=x), 768, 192, 1)
        return B.concat([b1, b7, d, bp])

    def incD(x):
        b3 = cb(cb(x, 768, 192, 1), 192, 320, 3, 2)
        b7 = cb(x, 768, 192, 1)
        b7 = cb(b7, 192, 192, (1, 7), 1, (0, 3))
        b7 = cb(b7, 192, 192, (7, 1), 1, (3, 0))
        b7 = cb(b7, 192, 192, 3, 2)
        bp = B.add(maxpool(3, 2), src0=x)
        return B.concat([b3, b7, bp])

    def incE(x, cin):
        b1 = cb(x, cin, 320, 1)
        t = cb(x, cin, 384, 1)
        b3 = B.concat([cb(t, 384, 384, (1, 3), 1, (0, 1)), cb(t, 384, 384, (3, 1), 1, (1, 0))])
        d = cb(cb(x, cin, 448, 1), 448, 384, 3, 1, 1)
        bd = B.concat([cb(d, 384, 384, (1, 3), 1, (0, 1)), cb(d, 384, 384, (3, 1), 1, (1, 0))])
        bp = cb(B.add(avgpool(3, 1, 1), src0=x), cin, 192, 1)
        return B.concat([b1, b3, bd, bp])

    for cin, pf in ((192, 32), (256, 64), (288, 64)):
        B.next_unit(); x = incA(x, cin, pf)
    B.next_unit(); x = incB(x, 288)
    for c7 in (128, 160, 160, 192):
        B.next_unit(); x = incC(x, c7)
    B.next_unit(); x = incD(x)
    for cin in (1280, 2048):
        B.next_unit(); x = incE(x, cin)
    B.next_unit()
    x = B.add(Layer(AVGPOOL_GLOBAL), src0=x)
    x = B.add(Layer(FLATTEN), src0=x)
    x = B.add(linear(2048, classes), src0=x)
    B.add(xent(), src0=x)
    return B.L, B.units


def assign_stages(layers, units, K):
    """Layer-count rule over partition units (remainder to the last r stages,
    S:107), written as explicit stage ids on the layers."""
    n_units = max(units) + 1
    if K > n_units:
        raise ValueError("more stages than units")
    base, r = divmod(n_units, K)
    st, u = [], 0
    for k in range(K):
        st += [k] * (base + (1 if k >= K - r else 0))
    return [l.with_stage(st[units[i]]) for i, l in enumerate(layers)]


def chain_units(layers):
    """Partition units of a chain model (R17): a unit begins at every Linear / Conv2d."""
    units, u = [], -1
    for l in layers:
        if l.kind in (LINEAR, CONV2D) or u < 0:
            u += 1
        units.append(u)
    return units


def unit_macs(layers, units, in_shape):
    """Forward multiply-accumulates per sample of every unit (a cost model for partitioning;
    no arithmetic of the method)."""
    shapes = infer_shapes(layers, in_shape)
    cost = [0.0] * (max(units) + 1)
    for i, l in enumerate(layers):
        if l.kind == LINEAR:
            cost[units[i]] += l.in_c * l.out_c
        elif l.kind == CONV2D:
            c, h, w = shapes[i]
            cost[units[i]] += c * h * w * l.in_c * l.kh * l.kw
    return cost


def balanced_stages(layers, units, cost, K):
    """Contiguous partition of the units into K stages minimising the largest stage cost
    (SURVEY 8e "cost-balanced split"; exact search over cut positions by dynamic programming),
    written as explicit stage ids."""
    n = len(cost)
    pre = [0.0]
    for c in cost:
        pre.append(pre[-1] + c)
    INF = float("inf")
    best = [[INF] * (n + 1) for _ in range(K + 1)]
    cut = [[0] * (n + 1) for _ in range(K + 1)]
    best[0][0] = 0.0
    for k in range(1, K + 1):
        for j in range(k, n + 1):
            for i in range(k - 1, j):
                v = max(best[k - 1][i], pre[j] - pre[i])
                if v < best[k][j]:
                    best[k][j], cut[k][j] = v, i
    bounds, j = [], n
    for k in range(K, 0, -1):
        bounds.append((cut[k][j], j))
        j = cut[k][j]
    bounds.reverse()
    stage_of_unit = [0] * n
    for k, (a, b) in enumerate(bounds):
        for u in range(a, b):
            stage_of_unit[u] = k
    return [l.with_stage(stage_of_unit[units[i]]) for i, l in enumerate(layers)]


def param_count(layers, in_shape):
    shapes = infer_shapes(layers, in_shape)
    n = 0
    for i, l in enumerate(layers):
        if l.kind == LINEAR:
            n += l.out_c * l.in_c + (l.out_c if l.bias else 0)
        elif l.kind == CONV2D:
            n += l.out_c * l.in_c * l.kh * l.kw + (l.out_c if l.bias else 0)
        elif l.kind == BATCHNORM2D:
            n += 2 * l.in_c
    return n
