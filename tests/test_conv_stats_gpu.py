"""Conv -> BN statistics handed over (monet_conv_fwd_w16_stats + monet_bn_stats_finalize).

The BN training forward after a conv takes the batch mean / variance from per-128-row-tile
(mean, M2) statistics the conv leaves behind -- from the GEMM epilogue when every tile is
final in one accumulation chain (K <= 1024, no split-K), else from one pass over y -- merged
with Chan's formula in fp64.  Checked against float64 torch statistics of the conv output
(including |mean| >> std, where E[x^2] - mean^2 would cancel), the running-stat update, and
run-to-run determinism; the conv output itself is bit-identical to monet_conv_fwd_w16.
"""
import ctypes
import math

import pytest
import torch

from paper_2010_14501_b200 import _native as N

pytestmark = pytest.mark.gpu

CASES = [
    # n, h, w, c, k, r, s, stride, pad, bias offset
    (8, 28, 28, 64, 256, 1, 1, 1, 0, 0.0),      # single chain, epilogue statistics
    (4, 14, 14, 64, 64, 3, 3, 1, 1, 0.0),       # K = 576, 64-wide N tile
    (3, 9, 11, 96, 200, 1, 1, 1, 0, 0.0),       # partial m- and n-tiles
    (4, 14, 14, 256, 128, 3, 3, 1, 1, 0.0),     # K = 2304: chunked chains -> pass over y
    (8, 28, 28, 64, 256, 1, 1, 1, 0, 1000.0),   # |mean| / std ~ 1000
    (184, 56, 56, 64, 64, 3, 3, 1, 1, 0.0),     # ResNet-50 layer 1 at b184: 577k rows, 4508 tiles
    (184, 56, 56, 64, 256, 1, 1, 1, 0, 0.0),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("variant", ["implicit", "splitk"])
def test_conv_stats_match_float64(cuda, case, variant):
    n, h, w, c, k, r, s, stride, pad, off = case
    g = torch.Generator().manual_seed(4)
    x = torch.randn(n, h, w, c, generator=g).to(cuda)
    wt = (torch.randn(k, r, s, c, generator=g) / math.sqrt(r * s * c)).to(cuda)
    bias = (torch.randn(k, generator=g) + off).to(cuda)
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    lib = N.lib()
    dll = lib.dll
    v = N.CONV_VARIANTS[variant]
    n8 = (wt.numel() + 7) // 8 * 8
    planes = torch.zeros(2 * n8, dtype=torch.int16, device=cuda)
    hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
    lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
    wsb = lib.conv_ws_bytes(v, 0, d)
    ws = torch.empty(max(wsb, 16) // 4 + 1, device=cuda)
    stats = torch.empty(dll.monet_conv_stats_bytes(ctypes.byref(d)) // 4 + 1, device=cuda)
    y0 = torch.empty(n, d.p, d.q, k, device=cuda)
    y1 = torch.empty_like(y0)
    assert dll.monet_conv_fwd_w16(v, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, bias.data_ptr(),
                                  y0.data_ptr(), ws.data_ptr(), wsb, None) == 0
    outs = []
    for _ in range(2):
        assert dll.monet_conv_fwd_w16_stats(v, ctypes.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo,
                                            bias.data_ptr(), y1.data_ptr(), stats.data_ptr(), ws.data_ptr(), wsb,
                                            None) == 0
        assert torch.equal(y0, y1)
        mean, inv = torch.empty(k, device=cuda), torch.empty(k, device=cuda)
        rm, rv = torch.zeros(k, device=cuda), torch.ones(k, device=cuda)
        rows = n * d.p * d.q
        assert dll.monet_bn_stats_finalize(stats.data_ptr(), rows, k, ctypes.c_float(1e-5), ctypes.c_float(0.1), 1,
                                           mean.data_ptr(), inv.data_ptr(), rm.data_ptr(), rv.data_ptr(), None) == 0
        outs.append((mean.clone(), inv.clone(), rm.clone(), rv.clone()))
    for a, b in zip(*outs):  # deterministic
        assert torch.equal(a, b)
    mean, inv, rm, rv = outs[0]
    yd = y1.double().reshape(-1, k)
    want_mean = yd.mean(0)
    want_var = yd.var(0, unbiased=False)
    assert ((mean.double() - want_mean).abs() / want_var.sqrt()).max() < 1e-4
    assert ((inv.double() - 1 / (want_var + 1e-5).sqrt()).abs() / inv.double()).max() < 1e-4
    assert ((rm.double() - 0.1 * want_mean).abs() / (want_var.sqrt() + 0.1 * want_mean.abs())).max() < 1e-4
    unb = yd.var(0, unbiased=True)
    assert ((rv.double() - (0.9 + 0.1 * unb)).abs() / (0.9 + 0.1 * unb)).max() < 1e-4
