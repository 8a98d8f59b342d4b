"""GPU unit parity of the tcgen05 implicit-GEMM conv kernel (pk_convgemm.cuh)
against torch's fp32 convolution of the same bf16-rounded operands.

FPROP / DGRAD / WGRAD over the conv shapes the pack nets use (1x1, 3x3, 5x5,
7x7; stride 1 and 2; channel counts that are and are not multiples of 64;
ragged M tails).  The kernel accumulates in fp32 in TMEM, so the only
difference from torch's fp32 result is summation order: the check is
|Δ| <= 2^-8·|ref| (bf16 output rounding) + 1e-4·max|ref| elementwise; the
fp32 WGRAD partials at 1e-5·max|ref|.
"""
import ctypes as C

import pytest

from _helpers import has_gpu

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2002_02885_b200 import _lib, cnn  # noqa: E402

SHAPES = [
    # n, h, w, c, k, r, s, stride, pad
    (2, 8, 8, 64, 64, 3, 3, 1, 1),
    (3, 7, 9, 16, 48, 3, 3, 1, 1),
    (2, 11, 11, 8, 32, 5, 5, 1, 0),
    (2, 16, 16, 8, 64, 7, 7, 2, 3),
    (4, 14, 14, 96, 24, 1, 1, 1, 0),
    (2, 15, 15, 128, 256, 3, 3, 2, 1),
    (2, 9, 9, 64, 128, 1, 1, 2, 0),
    (5, 6, 6, 160, 320, 1, 1, 1, 0),
]


def _rup(a, b):
    return (a + b - 1) // b * b


def _geom(n, h, w, c, k, r, s, st, pad):
    p = (h + 2 * pad - r) // st + 1
    q = (w + 2 * pad - s) // st + 1
    return _lib.ConvGeom(n, h, w, c, k, r, s, st, pad, p, q), p, q


def _data(n, h, w, c, k, r, s, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(n, c, h, w, generator=g).bfloat16().double().cuda()
    wt = (torch.randn(k, c, r, s, generator=g) / (r * s * c) ** 0.5).bfloat16().double().cuda()
    return x, wt


def _nhwc(t):
    return t.permute(0, 2, 3, 1).contiguous()


def _w_dev(wt):  # [k][(r*S+s)*C+ci] padded to 64
    k, c, r, s = wt.shape
    m = wt.permute(0, 2, 3, 1).reshape(k, r * s * c)
    out = torch.zeros(k, _rup(r * s * c, 64), device="cuda", dtype=torch.float64)
    out[:, :r * s * c] = m
    return out.bfloat16().contiguous()


def _wt_dev(wt):  # [ci][(r*S+s)*K+co] padded to 64
    k, c, r, s = wt.shape
    m = wt.permute(1, 2, 3, 0).reshape(c, r * s * k)
    out = torch.zeros(c, _rup(r * s * k, 64), device="cuda", dtype=torch.float64)
    out[:, :r * s * k] = m
    return out.bfloat16().contiguous()


def _run(mode, g, x, w, dy, out, ntile, splits=1, stages=4):
    L = _lib.lib()
    rc = L.pk_conv_gemm_test(mode, C.byref(g), x.data_ptr() if x is not None else None,
                             w.data_ptr() if w is not None else None,
                             dy.data_ptr() if dy is not None else None, out.data_ptr(), ntile,
                             splits, stages, None)
    assert rc == 0
    torch.cuda.synchronize()


def _close(got, want, tol, bf16_out=True):
    """|got - want| <= (bf16 output rounding, 2^-8 relative) + tol·max|want|"""
    err = (got.double() - want).abs()
    bound = tol * want.abs().max().item() + 1e-6
    if bf16_out:
        bound = bound + 2.0 ** -8 * want.abs()
    assert bool((err <= bound).all()), (err.max().item(), want.abs().max().item())


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("ntile", [64, 128])
def test_fprop(shape, ntile):
    n, h, w, c, k, r, s, st, pad = shape
    g, p, q = _geom(*shape)
    x, wt = _data(n, h, w, c, k, r, s)
    ref = _nhwc(F.conv2d(x, wt, stride=st, padding=pad)).reshape(n * p * q, k)
    out = torch.empty(n * p * q, k, dtype=torch.bfloat16, device="cuda")
    _run(0, g, _nhwc(x).bfloat16(), _w_dev(wt), None, out, ntile)
    _close(out, ref, 1e-4)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("ntile", [16, 64, 256])
def test_dgrad(shape, ntile):
    n, h, w, c, k, r, s, st, pad = shape
    g, p, q = _geom(*shape)
    x, wt = _data(n, h, w, c, k, r, s)
    dy = torch.randn(n, k, p, q, generator=torch.Generator().manual_seed(1)).bfloat16().double().cuda()
    ref = torch.nn.grad.conv2d_input(x.shape, wt, dy, stride=st, padding=pad)
    ref = _nhwc(ref).reshape(n * h * w, c)
    out = torch.empty(n * h * w, c, dtype=torch.bfloat16, device="cuda")
    _run(1, g, None, _wt_dev(wt), _nhwc(dy).bfloat16(), out, ntile)
    _close(out, ref, 1e-4)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("ntile,splits", [(64, 1), (128, 3), (256, 2)])
def test_wgrad(shape, ntile, splits):
    n, h, w, c, k, r, s, st, pad = shape
    g, p, q = _geom(*shape)
    x, wt = _data(n, h, w, c, k, r, s)
    dy = torch.randn(n, k, p, q, generator=torch.Generator().manual_seed(1)).bfloat16().double().cuda()
    ref = torch.nn.grad.conv2d_weight(x, wt.shape, dy, stride=st, padding=pad)
    ref = ref.permute(0, 2, 3, 1).reshape(k, r * s * c)
    kpad = _rup(r * s * c, 64)
    pix = n * p * q
    kper = _rup(-(-pix // splits), 64)
    ns = -(-pix // kper)
    out = torch.zeros(ns, k, kpad, device="cuda")
    _run(2, g, _nhwc(x).bfloat16(), None, _nhwc(dy).bfloat16(), out, ntile, splits)
    got = out.double().sum(0)[:, :r * s * c]
    _close(got, ref, 1e-5, bf16_out=False)


# ---- the same GEMMs through the program path (pk_cnn_prog), which feeds the
# activation operands by TMA: 2-D tiles for 1x1 stride-1 layers, im2col boxes
# for C % 64 == 0 (FPROP, WGRAD; DGRAD at stride 1), cp.async otherwise --------
PROG_SHAPES = [
    # n, h, w, c, k, r, s, stride, pad           modes (fprop a, dgrad a, wgrad b)
    (3, 10, 10, 96, 24, 1, 1, 1, 0),            # 1, 1, 1 (c % 64 != 0)
    (2, 9, 11, 64, 64, 3, 3, 1, 1),             # 2, 2, 2
    (2, 15, 15, 128, 256, 3, 3, 2, 1),          # 2, 0, 2 (stride-2 dgrad gathers)
    (3, 14, 14, 64, 128, 1, 1, 2, 0),           # 2, 0, 2
    (2, 16, 16, 64, 64, 7, 7, 2, 3),            # 2, 0, 2
    (2, 7, 7, 512, 512, 3, 3, 1, 1),            # 2, 2, 2 (deep K)
    (2, 12, 12, 8, 64, 7, 7, 2, 3),             # 0, 0, 0 (first-layer shape)
    (3, 10, 10, 40, 48, 1, 1, 1, 0),            # 1, 1, 1 + swapped WGRAD (co 48)
]


def _prog_conv(kind, g, x, w, dy, out, ntile, splits=1, stages=4):
    from paper_2002_02885_b200 import cnn
    cs = _lib.CnnConv()
    cs.n, cs.h, cs.w, cs.c, cs.k = g.n, g.h, g.w, g.c, g.k
    cs.r, cs.s, cs.stride, cs.pad, cs.p, cs.q = g.r, g.s, g.stride, g.pad, g.p, g.q
    cs.ldx, cs.ldy = g.c, g.k
    if kind == "CONV_FPROP":
        cs.src, cs.wt, cs.dst, cs.ldo = x.data_ptr(), w.data_ptr(), out.data_ptr(), g.k
    elif kind == "CONV_DGRAD":
        cs.src, cs.wt, cs.dst, cs.ldo = dy.data_ptr(), w.data_ptr(), out.data_ptr(), g.c
    else:
        cs.src, cs.dy, cs.dst, cs.splits = x.data_ptr(), dy.data_ptr(), out.data_ptr(), splits
    prog = cnn.CnnProgram([(_lib.CNN[kind], (ntile, stages), [cs])], 0)
    prog.run(torch.cuda.current_stream().cuda_stream, graph=False)
    torch.cuda.synchronize()


@pytest.mark.parametrize("shape", PROG_SHAPES)
def test_prog_fprop_dgrad_wgrad(shape):
    n, h, w, c, k, r, s, st, pad = shape
    g, p, q = _geom(*shape)
    x, wt = _data(n, h, w, c, k, r, s)
    dy = torch.randn(n, k, p, q, generator=torch.Generator().manual_seed(1)).bfloat16() \
        .double().cuda()
    # FPROP
    ref = _nhwc(F.conv2d(x, wt, stride=st, padding=pad)).reshape(n * p * q, k)
    out = torch.empty(n * p * q, k, dtype=torch.bfloat16, device="cuda")
    _prog_conv("CONV_FPROP", g, _nhwc(x).bfloat16(), _w_dev(wt), None, out,
               min(256, -(-k // 16) * 16))
    _close(out, ref, 1e-4)
    # DGRAD
    ref = _nhwc(torch.nn.grad.conv2d_input(x.shape, wt, dy, stride=st, padding=pad))
    ref = ref.reshape(n * h * w, c)
    out = torch.empty(n * h * w, c, dtype=torch.bfloat16, device="cuda")
    _prog_conv("CONV_DGRAD", g, None, _wt_dev(wt), _nhwc(dy).bfloat16(), out,
               min(256, -(-c // 16) * 16))
    _close(out, ref, 1e-4)
    # WGRAD (split over pixels: splits chosen so every split is non-empty)
    ref = torch.nn.grad.conv2d_weight(x, wt.shape, dy, stride=st, padding=pad)
    ref = ref.permute(0, 2, 3, 1).reshape(k, r * s * c)
    kpad = _rup(r * s * c, 64)
    pix = n * p * q
    for splits in (1, 2):
        kper = _rup(-(-pix // splits), 64)
        if -(-pix // kper) != splits:
            continue
        outw = torch.zeros(splits, k, kpad, device="cuda")
        # k <= 64 with a 64-wide N tile takes the swapped orientation (M = r·s·c)
        _prog_conv("CONV_WGRAD", g, _nhwc(x).bfloat16(), None, _nhwc(dy).bfloat16(), outw,
                   64 if k <= 64 else 128, splits)
        got = outw.double().sum(0)[:, :r * s * c]
        _close(got, ref, 1e-5, bf16_out=False)
