"""Tensor-core (tcgen05) GEMM and implicit-GEMM convolution parity against fp64 references of
the same bf16 operands (torch, a library routine).  Bound: fp32 accumulation of exact bf16
products, |err| <= K * 2^-23 * sum|a||b| per output (generous: 2^-16 relative to sum|a||b|)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def bf(t):
    return t.to(torch.bfloat16)


@pytest.mark.parametrize("a_k,b_k", [(True, True), (True, False), (False, True), (False, False)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (300, 200, 136), (129, 256, 1000), (64, 72, 8), (1000, 512, 64)])
def test_plain_gemm_all_majorness(a_k, b_k, M, N, K):
    from paper_1911_04610_b200 import gemm_bf16, XPipeError
    g = torch.Generator().manual_seed(M * 7 + N)
    A = torch.randn(M, K, generator=g)
    B = torch.randn(N, K, generator=g)
    Ab, Bb = bf(A), bf(B)
    A_dev = (Ab if a_k else Ab.t().contiguous()).to(DEV)
    B_dev = (Bb if b_k else Bb.t().contiguous()).to(DEV)
    D = torch.full((M, N), float("nan"), device=DEV)
    if (K if a_k else M) % 8 or (K if b_k else N) % 8:
        with pytest.raises(XPipeError):   # rows of 16 bytes are required (documented EINVAL)
            gemm_bf16(A_dev, B_dev, D, M, N, K, a_k, b_k)
        return
    gemm_bf16(A_dev, B_dev, D, M, N, K, a_k, b_k)
    torch.cuda.synchronize()
    ref = Ab.double() @ Bb.double().t()
    bound = (Ab.double().abs() @ Bb.double().abs().t()) * 2.0 ** -16 + 1e-30
    err = (D.cpu().double() - ref).abs()
    assert torch.isfinite(D).all()
    assert (err <= bound).all(), float((err / bound).max())


CONVS = [
    # (Nimg, C, H, W, Co, R, S, sh, sw, ph, pw)
    (2, 8, 8, 8, 16, 3, 3, 1, 1, 1, 1),
    (3, 64, 9, 7, 64, 3, 3, 1, 1, 1, 1),
    (2, 16, 16, 16, 32, 3, 3, 2, 2, 1, 1),
    (2, 32, 7, 7, 48, 1, 1, 1, 1, 0, 0),
    (1, 16, 9, 9, 24, 1, 7, 1, 1, 0, 3),
    (2, 24, 8, 8, 40, 7, 1, 1, 1, 3, 0),
    (2, 8, 15, 15, 16, 7, 7, 2, 2, 3, 3),
    (1, 128, 4, 4, 256, 3, 3, 1, 1, 1, 1),
    (32, 512, 2, 2, 512, 3, 3, 1, 1, 1, 1),     # VGG late layer (M=128, K=4608)
    (32, 64, 32, 32, 64, 3, 3, 1, 1, 1, 1),     # VGG layer 2 (M=32768)
    # full-TMA operand paths (stride 1, C % 64 == 0, tile rows form a pixel box)
    (4, 64, 8, 8, 64, 3, 3, 1, 1, 1, 1),        # box {8, 8, 2}
    (3, 64, 16, 16, 128, 3, 3, 1, 1, 1, 1),     # box {16, 8, 1}
    (3, 128, 4, 4, 192, 3, 3, 1, 1, 1, 1),      # ragged images past the last one (zero fill)
    (5, 64, 8, 8, 64, 1, 1, 1, 1, 0, 0),        # wgrad M = 64 (half an MN tile)
    (2, 64, 8, 8, 64, 1, 7, 1, 1, 0, 3),        # asymmetric filter / padding
    (6, 192, 2, 2, 320, 3, 3, 1, 1, 1, 1),      # box {2, 2, 32}, ragged N tiles
    # Inception-V3 / ResNet-101 geometries at 64x64: dense 1x1 GEMMs (stride 1 at any spatial size,
    # strided 1x1 dgrad scattering rows), and the explicit dgrad operand where the TMA pixel boxes
    # cannot serve (7x7 / 3x3 maps, Co % 64 != 0, stride 2)
    (4, 96, 7, 7, 96, 3, 3, 1, 1, 1, 1),
    (3, 192, 3, 3, 160, 1, 7, 1, 1, 0, 3),
    (3, 160, 3, 3, 192, 7, 1, 1, 1, 3, 0),
    (2, 288, 7, 7, 384, 3, 3, 2, 2, 0, 0),
    (2, 48, 7, 7, 64, 5, 5, 1, 1, 2, 2),
    (2, 768, 3, 3, 192, 1, 1, 1, 1, 0, 0),
    (2, 256, 16, 16, 512, 1, 1, 2, 2, 0, 0),
    (3, 1024, 4, 4, 2048, 1, 1, 2, 2, 0, 0),
    (2, 256, 8, 8, 256, 3, 3, 2, 2, 1, 1),
]


def geo_of(cfg):
    n, c, h, w, co, r, s, sh, sw, ph, pw = cfg
    P = (h + 2 * ph - r) // sh + 1
    Q = (w + 2 * pw - s) // sw + 1
    return (n, h, w, c, co, r, s, P, Q, sh, sw, ph, pw)


def rel_ok(got, ref, absref):
    err = (got.double() - ref).abs()
    bound = absref * 2.0 ** -15 + 1e-30
    return bool((err <= bound).all()), float((err / bound).max())


@pytest.mark.parametrize("cfg", CONVS)
def test_conv_fprop_dgrad_wgrad(cfg):
    from paper_1911_04610_b200 import conv2d_bf16
    F = torch.nn.functional
    n, c, h, w, co, r, s, sh, sw, ph, pw = cfg
    geo = geo_of(cfg)
    P, Q = geo[7], geo[8]
    g = torch.Generator().manual_seed(sum(cfg))
    X = bf(torch.randn(n, c, h, w, generator=g))
    Wt = bf(torch.randn(co, c, r, s, generator=g) * 0.1)
    dY = bf(torch.randn(n, co, P, Q, generator=g))
    Xd = X.permute(0, 2, 3, 1).contiguous().to(DEV)        # NHWC
    Wd = Wt.permute(0, 2, 3, 1).contiguous().to(DEV)       # KRSC
    dYd = dY.permute(0, 2, 3, 1).contiguous().to(DEV)
    ws = torch.zeros(16 << 20, device=DEV)  # zero once: the split-K counters live in its tail
    for use_ws in (None, ws):
        Y = torch.empty(n, P, Q, co, dtype=torch.bfloat16, device=DEV)
        conv2d_bf16(1, geo, Xd, Wd, Y, ws=use_ws)
        dX = torch.empty(n, h, w, c, dtype=torch.bfloat16, device=DEV)
        conv2d_bf16(2, geo, dYd, Wd, dX, ws=use_ws)
        dW = torch.full((co, r, s, c), 1.0, device=DEV)
        conv2d_bf16(3, geo, Xd, dYd, dW, accumulate=True, ws=use_ws)
        torch.cuda.synchronize()
        Xr, Wr, dYr = X.double(), Wt.double(), dY.double()
        ref = F.conv2d(Xr, Wr, None, (sh, sw), (ph, pw))
        absr = F.conv2d(Xr.abs(), Wr.abs(), None, (sh, sw), (ph, pw))
        ok, worst = rel_ok(Y.permute(0, 3, 1, 2).cpu().float(), ref, absr + ref.abs() * 2 ** -8 * 2 ** 15)
        assert ok, ("fprop", worst)
        refx = torch.nn.grad.conv2d_input(Xr.shape, Wr, dYr, (sh, sw), (ph, pw))
        absx = torch.nn.grad.conv2d_input(Xr.shape, Wr.abs(), dYr.abs(), (sh, sw), (ph, pw))
        ok, worst = rel_ok(dX.permute(0, 3, 1, 2).cpu().float(), refx, absx + refx.abs() * 2 ** -8 * 2 ** 15)
        assert ok, ("dgrad", worst)
        refw = torch.nn.grad.conv2d_weight(Xr, Wr.shape, dYr, (sh, sw), (ph, pw)) + 1.0
        absw = torch.nn.grad.conv2d_weight(Xr.abs(), Wr.shape, dYr.abs(), (sh, sw), (ph, pw)) + 1.0
        ok, worst = rel_ok(dW.permute(0, 3, 1, 2).cpu(), refw, absw)
        assert ok, ("wgrad", worst)


LINEARS = [
    # (n, in, out): VGG-16 head, ResNet-101 / Inception-V3 heads (2048 -> 200, split-K), the MLP
    # hidden layers in bf16 mode, ragged feature counts, a micro-batch wider than one N tile
    (32, 512, 10), (32, 2048, 200), (8, 784, 256), (50, 64, 33), (100, 136, 130),
]


@pytest.mark.parametrize("n,inf,outf", LINEARS)
def test_linear_tensor_core(n, inf, outf):
    """xpipe_linear_bf16 (swap-AB tcgen05 GEMMs of the bf16 Linear layers) against fp64 torch on
    the same bf16 operands: forward with bias (fp32 logits; bf16 with and without ReLU: every
    output within one bf16 rounding of the fp64 value evaluated in fp32), dgrad (bf16), wgrad
    stored then accumulated (fp32)."""
    from paper_1911_04610_b200 import linear_bf16
    g = torch.Generator().manual_seed(n * 31 + outf)
    x = bf(torch.randn(n, inf, generator=g))
    W = bf(torch.randn(outf, inf, generator=g) / inf ** 0.5)
    b = bf(torch.randn(outf, generator=g))
    ldp = (outf + 7) // 8 * 8
    dy = torch.zeros(n, ldp, dtype=torch.bfloat16)
    dy[:, :outf] = bf(torch.randn(n, outf, generator=g))
    xd, Wd, bd, dyd = (t.to(DEV) for t in (x, W, b, dy))
    ws = torch.zeros(1 << 22, device=DEV)
    ref = x.double() @ W.double().t() + b.double()
    mag = x.double().abs() @ W.double().abs().t() + b.double().abs()
    # fp32 logits
    y = torch.full((n, outf), float("nan"), device=DEV)
    linear_bf16(1, y, n, inf, outf, x=xd, W=Wd, b=bd, f32out=True, ws=ws)
    torch.cuda.synchronize()
    assert ((y.cpu().double() - ref).abs() <= mag * 2.0 ** -16 + 1e-30).all()
    # bf16 out, with / without ReLU: within one bf16 ulp of the exact value
    for relu in (False, True):
        yb = torch.full((n, outf), float("nan"), device=DEV, dtype=torch.bfloat16)
        linear_bf16(1, yb, n, inf, outf, x=xd, W=Wd, b=bd, relu=relu, ws=ws)
        torch.cuda.synchronize()
        r = ref.clamp(min=0) if relu else ref
        err = (yb.cpu().double() - r).abs()
        assert (err <= r.abs() * 2.0 ** -8 + mag * 2.0 ** -16 + 1e-30).all()
        if relu:
            assert (yb.cpu() >= 0).all()
    # dgrad
    dx = torch.full((n, inf), float("nan"), device=DEV, dtype=torch.bfloat16)
    linear_bf16(2, dx, n, inf, outf, W=Wd, dy=dyd, ldp=ldp, ws=ws)
    torch.cuda.synchronize()
    rdx = dy[:, :outf].double() @ W.double()
    mdx = dy[:, :outf].double().abs() @ W.double().abs()
    assert ((dx.cpu().double() - rdx).abs() <= rdx.abs() * 2.0 ** -8 + mdx * 2.0 ** -16 + 1e-30).all()
    # wgrad: store, then accumulate
    gW = torch.full((outf, inf), float("nan"), device=DEV)
    linear_bf16(3, gW, n, inf, outf, x=xd, dy=dyd, ldp=ldp, ws=ws)
    torch.cuda.synchronize()
    rgw = dy[:, :outf].double().t() @ x.double()
    mgw = dy[:, :outf].double().abs().t() @ x.double().abs()
    assert ((gW.cpu().double() - rgw).abs() <= mgw * 2.0 ** -16 + 1e-30).all()
    linear_bf16(3, gW, n, inf, outf, x=xd, dy=dyd, ldp=ldp, accumulate=True, ws=ws)
    torch.cuda.synchronize()
    assert ((gW.cpu().double() - 2 * rgw).abs() <= 2 * mgw * 2.0 ** -16 + 1e-30).all()
