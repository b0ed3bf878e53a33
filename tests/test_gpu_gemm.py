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
