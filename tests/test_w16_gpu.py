"""Pre-split weights (monet_conv_fwd_w16 / monet_conv_dgrad_w16, monet_split_bf16*).

The bf16x3 GEMM splits every fp32 operand element into hi = bf16(x), lo = bf16(x - hi);
loading the weights' split from bf16 planes instead of splitting them per tile must give
BIT-identical results to the fp32 entry points (same products, same accumulation order),
on every shape class: pointwise / im2col forward, stride-1 and sub-pixel-phase dgrad,
64-wide N tiles, K_out not a multiple of 64, split-K, conv bias, accumulate mode, and the
shapes that fall back to the fp32 path (weights not 16-B aligned in the planes, K_out % 32).
"""
import ctypes
import math

import pytest
import torch

from paper_2010_14501_b200 import _native as N

pytestmark = pytest.mark.gpu

CASES = [
    # n, h, w, c, k, r, s, stride, pad
    (2, 8, 8, 64, 64, 1, 1, 1, 0),        # pointwise, 64-wide N tile
    (4, 14, 14, 256, 512, 1, 1, 1, 0),    # pointwise, K-major A
    (2, 9, 7, 32, 64, 3, 3, 1, 1),        # im2col fprop, C = 32
    (3, 14, 14, 64, 128, 3, 3, 2, 1),     # strided: phase dgrad
    (2, 15, 15, 128, 256, 1, 1, 2, 0),    # strided pointwise
    (4, 7, 7, 256, 96, 3, 3, 1, 1),       # K_out = 96 (32-deep dgrad boxes straddle taps)
    (2, 12, 12, 64, 32, 3, 3, 2, 1),      # K_out = 32
    (1, 6, 6, 192, 64, 3, 3, 1, 1),       # C = 192: three 64-channel chunks, the last partial
    (2, 10, 10, 96, 200, 3, 3, 1, 1),     # N = 200: partial n-tile; K_out % 32 != 0 -> dgrad falls back
    (1, 5, 6, 8, 12, 3, 3, 1, 1),         # tiny channels: falls back to fp32 B
    (8, 56, 56, 64, 64, 3, 3, 1, 1),      # ResNet-50 layer-1 shape class (several waves)
    (4, 8, 8, 128, 192, 3, 3, 1, 1),      # N = 192: the second n-tile's last two 32-col chunks are empty
    (4, 16, 16, 64, 192, 3, 3, 1, 1),     # ... with split-K partials
    (64, 14, 14, 64, 192, 1, 1, 1, 0),    # ... and several tiles per CTA (store-buffer pairing)
    (64, 14, 14, 64, 200, 1, 1, 1, 0),    # N = 200: a partial trailing chunk, several tiles per CTA
]


def _s():
    return torch.cuda.current_stream().cuda_stream


def _split(w):
    hi = w.bfloat16()
    lo = (w - hi.float()).bfloat16()
    return hi, lo


def _planes(w, cuda, offset=0):
    """bf16 hi / lo planes of w as monet_split_bf16 writes them (lo plane after hi)."""
    n = w.numel()
    n8 = (n + offset + 7) // 8 * 8
    buf = torch.zeros(2 * n8, dtype=torch.int16, device=cuda)
    lib = N.lib().dll
    hi = buf.data_ptr() + 2 * offset
    lo = buf.data_ptr() + 2 * (n8 + offset)
    assert lib.monet_split_bf16(w.data_ptr(), hi, lo, n, None) == 0
    return buf, hi, lo


def test_split_kernel_rounding(cuda):
    g = torch.Generator().manual_seed(0)
    w = torch.randn(1 << 16, generator=g) * torch.logspace(-20, 20, 1 << 16)
    w[:4] = torch.tensor([0.0, -0.0, 1.0 + 2 ** -8, 3.0 + 2 ** -7])  # ties round to even
    wd = w.to(cuda)
    buf, hi, lo = _planes(wd, cuda)
    torch.cuda.synchronize()
    n8 = buf.numel() // 2
    got_hi = buf[:w.numel()].view(torch.bfloat16).cpu()
    got_lo = buf[n8:n8 + w.numel()].view(torch.bfloat16).cpu()
    want_hi, want_lo = _split(w)
    assert torch.equal(got_hi.view(torch.int16), want_hi.view(torch.int16))
    assert torch.equal(got_lo.view(torch.int16), want_lo.view(torch.int16))


def test_split_segments(cuda):
    g = torch.Generator().manual_seed(1)
    src = torch.randn(1000, generator=g).to(cuda)
    segs = [(3, 0, 10), (100, 16, 257), (500, 280, 1)]
    table = torch.tensor(segs, dtype=torch.int64, device=cuda).reshape(-1)
    hi = torch.zeros(512, dtype=torch.int16, device=cuda)
    lo = torch.zeros(512, dtype=torch.int16, device=cuda)
    rc = N.lib().dll.monet_split_bf16_segments(src.data_ptr(), hi.data_ptr(), lo.data_ptr(), table.data_ptr(),
                                                len(segs), 257, None)
    assert rc == 0
    want_hi, want_lo = torch.zeros(512, dtype=torch.int16), torch.zeros(512, dtype=torch.int16)
    for s0, d0, n in segs:
        h, l = _split(src[s0:s0 + n].cpu())
        want_hi[d0:d0 + n] = h.view(torch.int16)
        want_lo[d0:d0 + n] = l.view(torch.int16)
    assert torch.equal(hi.cpu(), want_hi) and torch.equal(lo.cpu(), want_lo)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("variant", ["implicit", "splitk"])
def test_w16_bit_identical(cuda, case, variant):
    n, h, w, c, k, r, s, stride, pad = case
    g = torch.Generator().manual_seed(2)
    x = torch.randn(n, h, w, c, generator=g).to(cuda)
    wt = (torch.randn(k, r, s, c, generator=g) / math.sqrt(r * s * c)).to(cuda)
    bias = torch.randn(k, generator=g).to(cuda)
    dy = torch.randn(n, (h + 2 * pad - r) // stride + 1, (w + 2 * pad - s) // stride + 1, k, generator=g).to(cuda)
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    lib = N.lib()
    dll = lib.dll
    v = N.CONV_VARIANTS[variant]
    _, hi, lo = _planes(wt, cuda)
    wsb = max(lib.conv_ws_bytes(v, 0, d), lib.conv_ws_bytes(v, 3, d))
    ws = torch.empty(max(wsb, 16) // 4 + 1, device=cuda)
    y0 = torch.empty(n, d.p, d.q, k, device=cuda)
    y1 = torch.full_like(y0, 5.0)
    assert lib.conv_fwd(v, d, x.data_ptr(), wt.data_ptr(), y0.data_ptr(), ws.data_ptr(), wsb, _s()) == 0
    assert dll.monet_conv_fwd_w16(v, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y1.data_ptr(),
                                  ws.data_ptr(), wsb, None) == 0
    assert torch.equal(y0, y1)
    y2 = torch.full_like(y0, -5.0)  # run to run: the smem-staged TMA stores are race-free
    assert dll.monet_conv_fwd_w16(v, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y2.data_ptr(),
                                  ws.data_ptr(), wsb, None) == 0
    assert torch.equal(y1, y2)
    # with the conv bias (VGG / UNet convs)
    assert dll.monet_conv_fwd_bias(v, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), bias.data_ptr(), y0.data_ptr(),
                                   ws.data_ptr(), wsb, None) == 0
    assert dll.monet_conv_fwd_w16(v, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, bias.data_ptr(),
                                  y1.data_ptr(), ws.data_ptr(), wsb, None) == 0
    assert torch.equal(y0, y1)
    for acc in (0, 1):
        dx0 = torch.full((n, h, w, c), 0.5, device=cuda)
        dx1 = dx0.clone()
        assert lib.conv_dgrad(v, d, dy.data_ptr(), wt.data_ptr(), dx0.data_ptr(), acc, ws.data_ptr(), wsb, _s()) == 0
        assert dll.monet_conv_dgrad_w16(v, ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), hi, lo, dx1.data_ptr(),
                                        acc, ws.data_ptr(), wsb, None) == 0
        assert torch.equal(dx0, dx1)


def test_w16_misaligned_planes_fall_back(cuda):
    """Planes at an odd element offset are not 16-B aligned: the fp32 path runs instead."""
    n, h, w, c, k, r, s, stride, pad = CASES[1]
    g = torch.Generator().manual_seed(3)
    x = torch.randn(n, h, w, c, generator=g).to(cuda)
    wt = torch.randn(k, r, s, c, generator=g).to(cuda)
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    _, hi, lo = _planes(wt, cuda, offset=3)
    y0 = torch.empty(n, d.p, d.q, k, device=cuda)
    y1 = torch.empty_like(y0)
    lib = N.lib()
    assert lib.conv_fwd(0, d, x.data_ptr(), wt.data_ptr(), y0.data_ptr(), None, 0, _s()) == 0
    assert lib.dll.monet_conv_fwd_w16(0, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y1.data_ptr(),
                                      None, 0, None) == 0
    assert torch.equal(y0, y1)
