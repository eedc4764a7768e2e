"""Numerics of every sm_100a kernel against a plain PyTorch reference of the same op.

Floating-point ops are compared with a float64 CPU torch computation of the
same formula; the tolerance is max|gpu - ref| / max|ref| <= 5e-5 for the
bf16x3 / 3xTF32 tensor-core paths (products carry ~2^-17 relative error, so
the sums land near 1e-5; the engine-level parity bar is 1e-4) and 1e-5 for
fp32 CUDA-core ops.  Bit-level outputs (ReLU sign masks, maxpool indices) are exact.
"""
import ctypes
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2010_14501_b200 import _native as N

pytestmark = pytest.mark.gpu

REL_TC = 5e-5     # bf16x3 / 3xTF32 tensor-core conv / gemm
REL_TF32 = 3e-3   # single-pass tf32 variant
REL_EW = 1e-5     # CUDA-core fp32 kernels


def rel_err(out, ref):
    out = out.detach().double().cpu()
    ref = ref.detach().double().cpu()
    return (out - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)


def stream():
    return torch.cuda.current_stream().cuda_stream


def conv_ref(x, w, stride, pad):
    # x NHWC, w KRSC -> y NHWC (float64 CPU)
    y = F.conv2d(x.double().cpu().permute(0, 3, 1, 2), w.double().cpu().permute(0, 3, 1, 2),
                 stride=stride, padding=pad)
    return y.permute(0, 2, 3, 1)


CONV_CASES = [
    # n, h, w, c, k, r, s, stride, pad
    (2, 8, 8, 64, 64, 1, 1, 1, 0),
    (2, 9, 7, 32, 64, 3, 3, 1, 1),
    (3, 14, 14, 64, 128, 3, 3, 2, 1),
    (2, 15, 15, 128, 256, 1, 1, 2, 0),
    (2, 32, 32, 4, 64, 7, 7, 2, 3),
    (4, 7, 7, 256, 96, 3, 3, 1, 1),
    (1, 5, 6, 8, 12, 3, 3, 1, 1),
    (2, 10, 10, 64, 64, 3, 3, 1, 1),     # wgrad row tile spans two taps (bulk segments)
    (1, 6, 6, 192, 64, 3, 3, 1, 1),      # C % 128 != 0: wgrad falls back to 16B groups
    (2, 12, 12, 64, 32, 3, 3, 2, 1),     # stride-2 dgrad gather, K = 32
    (21, 40, 40, 4, 160, 3, 3, 1, 1),    # wgrad tap view (>= 32K pixels): two m-tiles, q padded 40 -> 64
    (2, 350, 202, 8, 64, 5, 5, 2, 2),    # wgrad tap view: 3 filter rows (120 columns) per n-tile, Q = 101
    (8, 129, 127, 4, 64, 7, 7, 2, 3),    # splitk fprop tap view (C*S <= 32, Q <= 128, >= 32K pixels)
]


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("variant", ["implicit", "splitk", "tf32x3"])
def test_conv_passes(cuda, case, variant):
    n, h, w, c, k, r, s, stride, pad = case
    g = torch.Generator().manual_seed(0)
    x = torch.randn(n, h, w, c, generator=g)
    wt = torch.randn(k, r, s, c, generator=g) / math.sqrt(r * s * c)
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    lib = N.lib()
    v = N.CONV_VARIANTS[variant]
    xd, wd = x.to(cuda), wt.to(cuda)
    y = torch.empty(n, d.p, d.q, k, device=cuda)
    ws_f = lib.conv_ws_bytes(v, 0, d)
    ws = torch.empty(max(ws_f, 4) // 4 + 1, device=cuda)
    lib.conv_fwd(v, d, xd.data_ptr(), wd.data_ptr(), y.data_ptr(), ws.data_ptr(), ws_f, stream())
    ref = conv_ref(x, wt, stride, pad)
    assert rel_err(y, ref) < REL_TC

    dy = torch.randn(n, d.p, d.q, k, generator=g)
    dyd = dy.to(cuda)
    ws_b = lib.conv_ws_bytes(v, 3, d)
    ws = torch.empty(max(ws_b, 4) // 4 + 1, device=cuda)
    dx = torch.full((n, h, w, c), 7.0, device=cuda)
    lib.conv_dgrad(v, d, dyd.data_ptr(), wd.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), ws_b, stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    yr = F.conv2d(xr, wt.double().permute(0, 3, 1, 2), stride=stride, padding=pad)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    assert rel_err(dx, xr.grad.permute(0, 2, 3, 1)) < REL_TC
    # accumulate mode adds onto the existing gradient
    lib.conv_dgrad(v, d, dyd.data_ptr(), wd.data_ptr(), dx.data_ptr(), 1, ws.data_ptr(), ws_b, stream())
    assert rel_err(dx, 2 * xr.grad.permute(0, 2, 3, 1)) < REL_TC

    dw = torch.empty(k, r, s, c, device=cuda)
    lib.conv_wgrad(v, d, xd.data_ptr(), dyd.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), ws_b, stream())
    wr = wt.double().permute(0, 3, 1, 2).requires_grad_()
    yr = F.conv2d(x.double().permute(0, 3, 1, 2), wr, stride=stride, padding=pad)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    assert rel_err(dw, wr.grad.permute(0, 2, 3, 1)) < REL_TC


def test_conv_tf32_variant(cuda):
    n, h, w, c, k, r, s, stride, pad = CONV_CASES[1]
    g = torch.Generator().manual_seed(1)
    x = torch.randn(n, h, w, c, generator=g)
    wt = torch.randn(k, r, s, c, generator=g) / math.sqrt(r * s * c)
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    y = torch.empty(n, d.p, d.q, k, device=cuda)
    xd, wd = x.to(cuda), wt.to(cuda)  # keep the device copies alive while the kernel reads them
    N.lib().conv_fwd(2, d, xd.data_ptr(), wd.data_ptr(), y.data_ptr(), None, 0, stream())
    e = rel_err(y, conv_ref(x, wt, stride, pad))
    assert 1e-7 < e < REL_TF32  # visibly less accurate than 3xTF32, still tf32-accurate


@pytest.mark.parametrize("mnk", [(200, 1000, 2048), (128, 128, 32), (77, 36, 20), (300, 260, 1000)])
@pytest.mark.parametrize("amn,bmn", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_gemm_layouts(cuda, mnk, amn, bmn):
    m, n, k = mnk
    if (amn and m % 4) or (bmn and n % 4) or (not amn and k % 4) or (not bmn and k % 4):
        pytest.skip("16B operand groups need the contiguous extent % 4 == 0")
    g = torch.Generator().manual_seed(2)
    A = torch.randn(m, k, generator=g)
    B = torch.randn(n, k, generator=g)
    a_store = A.t().contiguous() if amn else A
    b_store = B.t().contiguous() if bmn else B
    lda = m if amn else k
    ldb = n if bmn else k
    C = torch.zeros(m, n, device=cuda)
    ad, bd = a_store.to(cuda), b_store.to(cuda)
    for variant in (0, 1, 3):  # 4 ("pair") is retired
        wsb = N.lib().gemm_ws_bytes(variant, m, n, k)
        ws = torch.empty(wsb // 4 + 1, device=cuda)
        N.lib().gemm(variant, ad.data_ptr(), amn, lda, bd.data_ptr(), bmn, ldb,
                     C.data_ptr(), n, m, n, k, 0, ws.data_ptr(), wsb, stream())
        assert rel_err(C, A.double() @ B.double().t()) < REL_TC


def test_linear(cuda):
    n, fi, fo = 24, 512, 1000
    g = torch.Generator().manual_seed(3)
    x, W, b = torch.randn(n, fi, generator=g), torch.randn(fo, fi, generator=g) * 0.05, torch.randn(fo, generator=g)
    dy = torch.randn(n, fo, generator=g)
    lib = N.lib()
    xd, Wd, bd, dyd = (t.to(cuda) for t in (x, W, b, dy))
    y = torch.empty(n, fo, device=cuda)
    for variant in (0, 1):
        wsb = max(lib.linear_ws_bytes(variant, 0, n, fi, fo), lib.linear_ws_bytes(variant, 3, n, fi, fo))
        ws = torch.empty(wsb // 4 + 1, device=cuda)
        lib.linear_fwd(variant, xd.data_ptr(), Wd.data_ptr(), bd.data_ptr(), y.data_ptr(), n, fi, fo,
                       ws.data_ptr(), wsb, stream())
        xr, Wr, br = (t.double().requires_grad_() for t in (x, W, b))
        yr = F.linear(xr, Wr, br)
        assert rel_err(y, yr) < REL_TC
        yr.backward(dy.double())
        dx, dW, db = torch.empty_like(xd), torch.empty_like(Wd), torch.empty_like(bd)
        lib.linear_bwd(variant, xd.data_ptr(), Wd.data_ptr(), dyd.data_ptr(), dx.data_ptr(), 0, dW.data_ptr(),
                       db.data_ptr(), n, fi, fo, ws.data_ptr(), wsb, stream())
        assert rel_err(dx, xr.grad) < REL_TC
        assert rel_err(dW, Wr.grad) < REL_TC
        assert rel_err(db, br.grad) < REL_EW


def pack_mask_np(x):
    bits = (x.reshape(-1).numpy() > 0).astype(np.uint8)
    pad = (-len(bits)) % 32
    bits = np.concatenate([bits, np.zeros(pad, np.uint8)])
    return np.packbits(bits.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").reshape(-1).astype(np.uint32)


@pytest.mark.parametrize("n", [1, 31, 32, 1000, 4099, 1 << 20])
def test_relu_mask_exact(cuda, n):
    g = torch.Generator().manual_seed(n)
    x = torch.randn(n, generator=g)
    x[::7] = 0.0
    x[::11] = -0.0
    if n > 20:
        x[13] = float("nan")
    lib = N.lib()
    xd = x.to(cuda)
    y = torch.empty_like(xd)
    mask = torch.zeros((n + 31) // 32, dtype=torch.int32, device=cuda)
    lib.relu_fwd(xd.data_ptr(), y.data_ptr(), mask.data_ptr(), n, stream())
    ref_y = torch.where(x > 0, x, torch.zeros_like(x))
    assert torch.equal(y.cpu(), ref_y)
    assert np.array_equal(mask.cpu().numpy().view(np.uint32), pack_mask_np(x))
    dy = torch.randn(n, generator=g)
    dyd = dy.to(cuda)
    ref_dx = torch.where(x > 0, dy, torch.zeros_like(dy))
    for fn, src in (("relu_bwd_mask", mask), ("relu_bwd_out", y), ("relu_bwd_in", xd)):
        dx = torch.empty_like(dyd)
        getattr(lib, fn)(src.data_ptr(), dyd.data_ptr(), dx.data_ptr(), n, 0, stream())
        assert torch.equal(dx.cpu(), ref_dx), fn
        getattr(lib, fn)(src.data_ptr(), dyd.data_ptr(), dx.data_ptr(), n, 1, stream())
        assert torch.equal(dx.cpu(), ref_dx + ref_dx), fn


@pytest.mark.parametrize("shape", [(8, 16, 16, 64), (4, 7, 7, 2048), (3, 5, 5, 96), (2, 3, 3, 1024)])
def test_batchnorm(cuda, shape):
    n, h, w, c = shape
    rows = n * h * w
    g = torch.Generator().manual_seed(4)
    x = torch.randn(n, h, w, c, generator=g) * 3 + 1.5
    gamma = torch.rand(c, generator=g) + 0.5
    beta = torch.randn(c, generator=g)
    dy = torch.randn(n, h, w, c, generator=g)
    lib = N.lib()
    xd, gd, bd, dyd = (t.to(cuda) for t in (x, gamma, beta, dy))
    y = torch.empty_like(xd)
    mean, invstd = torch.empty(c, device=cuda), torch.empty(c, device=cuda)
    rm, rv = torch.zeros(c, device=cuda), torch.ones(c, device=cuda)
    scratch = torch.empty(lib.bn_scratch_bytes(rows, c) // 4 + 1, device=cuda)
    lib.bn_fwd_train(xd.data_ptr(), y.data_ptr(), gd.data_ptr(), bd.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                     rm.data_ptr(), rv.data_ptr(), rows, c, 1e-5, 0.1, 1, scratch.data_ptr(), stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    gr, br = gamma.double().requires_grad_(), beta.double().requires_grad_()
    rmr, rvr = torch.zeros(c, dtype=torch.float64), torch.ones(c, dtype=torch.float64)
    yr = F.batch_norm(xr, rmr, rvr, gr, br, training=True, momentum=0.1, eps=1e-5)
    assert rel_err(y, yr.permute(0, 2, 3, 1)) < REL_EW
    assert rel_err(rm, rmr) < REL_EW and rel_err(rv, rvr) < REL_EW
    # replay with saved statistics is bit-identical and leaves running stats alone
    y2 = torch.empty_like(y)
    rm_before = rm.clone()
    lib.bn_fwd_replay(xd.data_ptr(), y2.data_ptr(), gd.data_ptr(), bd.data_ptr(), mean.data_ptr(),
                      invstd.data_ptr(), rows, c, stream())
    assert torch.equal(y, y2) and torch.equal(rm, rm_before)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    ref_dx = xr.grad.permute(0, 2, 3, 1)
    for fn in ("bn_bwd_in", "bn_bwd_out"):
        dx = torch.empty_like(xd)
        dg, db = torch.empty(c, device=cuda), torch.empty(c, device=cuda)
        if fn == "bn_bwd_in":
            lib.bn_bwd_in(xd.data_ptr(), dyd.data_ptr(), dx.data_ptr(), 0, gd.data_ptr(), mean.data_ptr(),
                          invstd.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c, scratch.data_ptr(), stream())
            tol = REL_EW
        else:
            lib.bn_bwd_out(y.data_ptr(), dyd.data_ptr(), dx.data_ptr(), 0, gd.data_ptr(), bd.data_ptr(),
                           invstd.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c, scratch.data_ptr(), stream())
            tol = 2e-5  # xhat reconstructed from the output costs one extra rounding
        assert rel_err(dx, ref_dx) < tol, fn
        assert rel_err(dg, gr.grad) < tol, fn
        assert rel_err(db, br.grad) < REL_EW, fn


@pytest.mark.parametrize("shape", [(4, 7, 7, 64), (2, 9, 5, 256)])
def test_fused_bn_relu(cuda, shape):
    n, h, w, c = shape
    rows = n * h * w
    g = torch.Generator().manual_seed(5)
    x = torch.randn(n, h, w, c, generator=g) * 2 + 0.3
    gamma = torch.rand(c, generator=g) + 0.5
    beta = torch.randn(c, generator=g) * 0.5
    dz = torch.randn(n, h, w, c, generator=g)
    lib = N.lib()
    xd, gd, bd, dzd = (t.to(cuda) for t in (x, gamma, beta, dz))
    z = torch.empty_like(xd)
    mean, invstd = torch.empty(c, device=cuda), torch.empty(c, device=cuda)
    rm, rv = torch.zeros(c, device=cuda), torch.ones(c, device=cuda)
    scratch = torch.empty(lib.bn_scratch_bytes(rows, c) // 4 + 1, device=cuda)
    lib.bnrelu_fwd_train(xd.data_ptr(), z.data_ptr(), gd.data_ptr(), bd.data_ptr(), mean.data_ptr(),
                         invstd.data_ptr(), rm.data_ptr(), rv.data_ptr(), rows, c, 1e-5, 0.1, 1, scratch.data_ptr(),
                         stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    gr, br = gamma.double().requires_grad_(), beta.double().requires_grad_()
    rmr, rvr = torch.zeros(c, dtype=torch.float64), torch.ones(c, dtype=torch.float64)
    zr = F.relu(F.batch_norm(xr, rmr, rvr, gr, br, training=True, momentum=0.1, eps=1e-5))
    assert rel_err(z, zr.permute(0, 2, 3, 1)) < REL_EW
    assert rel_err(rm, rmr) < REL_EW and rel_err(rv, rvr) < REL_EW
    # the separate BN + ReLU kernels give the identical output (fusion changes no bits)
    y = torch.empty_like(xd)
    lib.bn_fwd_replay(xd.data_ptr(), y.data_ptr(), gd.data_ptr(), bd.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                      rows, c, stream())
    z2 = torch.empty_like(xd)
    lib.relu_fwd(y.data_ptr(), z2.data_ptr(), None, y.numel(), stream())
    assert torch.equal(z, z2)
    z3 = torch.empty_like(xd)
    lib.bnrelu_fwd_replay(xd.data_ptr(), z3.data_ptr(), gd.data_ptr(), bd.data_ptr(), mean.data_ptr(),
                          invstd.data_ptr(), rows, c, stream())
    assert torch.equal(z, z3)
    zr.backward(dz.double().permute(0, 3, 1, 2))
    dx = torch.full_like(xd, 2.0)
    dg, db = torch.empty(c, device=cuda), torch.empty(c, device=cuda)
    lib.bnrelu_bwd(xd.data_ptr(), dzd.data_ptr(), dx.data_ptr(), 1, gd.data_ptr(), bd.data_ptr(), mean.data_ptr(),
                   invstd.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c, scratch.data_ptr(), stream())
    assert rel_err(dx - 2.0, xr.grad.permute(0, 2, 3, 1)) < 2e-5  # accumulate mode
    assert rel_err(dg, gr.grad) < 2e-5 and rel_err(db, br.grad) < REL_EW


def test_maxpool_and_avgpool(cuda):
    n, h, w, c = 3, 13, 12, 64
    g = torch.Generator().manual_seed(5)
    x = torch.randn(n, h, w, c, generator=g)
    d = N.conv_desc(n, h, w, c, c, 3, 3, 2, 1)
    lib = N.lib()
    xd = x.to(cuda)
    y = torch.empty(n, d.p, d.q, c, device=cuda)
    idx = torch.empty(n, d.p, d.q, c, dtype=torch.uint8, device=cuda)
    lib.maxpool_fwd(d, xd.data_ptr(), y.data_ptr(), idx.data_ptr(), stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    yr, ir = F.max_pool2d(xr, 3, 2, 1, return_indices=True)
    assert torch.equal(y.cpu().double(), yr.permute(0, 2, 3, 1))
    # 8-bit window index -> torch's flat input index
    ii = idx.cpu().long().permute(0, 3, 1, 2)
    pp = torch.arange(d.p).view(1, 1, -1, 1) * 2 - 1 + ii // 3
    qq = torch.arange(d.q).view(1, 1, 1, -1) * 2 - 1 + ii % 3
    assert torch.equal(pp * w + qq, ir)
    dy = torch.randn(n, d.p, d.q, c, generator=g)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    for use_idx in (True, False):
        dx = torch.empty_like(xd)
        lib.maxpool_bwd(d, idx.data_ptr() if use_idx else None, xd.data_ptr(), dy.to(cuda).data_ptr(),
                        dx.data_ptr(), 0, stream())
        assert rel_err(dx, xr.grad.permute(0, 2, 3, 1)) < REL_EW
    ya = torch.empty(n, c, device=cuda)
    lib.avgpool_fwd(xd.data_ptr(), ya.data_ptr(), n, h * w, c, stream())
    assert rel_err(ya, x.double().mean(dim=(1, 2))) < REL_EW


def test_xent_and_sgd(cuda):
    n, k = 16, 1000
    g = torch.Generator().manual_seed(6)
    z = torch.randn(n, k, generator=g) * 3
    lab = torch.randint(0, k, (n,), generator=g)
    lib = N.lib()
    zd, ld = z.to(cuda), lab.to(torch.int32).to(cuda)
    loss = torch.empty(1, device=cuda)
    scratch = torch.empty(n, device=cuda)
    lib.xent_fwd(zd.data_ptr(), ld.data_ptr(), loss.data_ptr(), n, k, scratch.data_ptr(), stream())
    zr = z.double().requires_grad_()
    lr = F.cross_entropy(zr, lab)
    assert abs(loss.item() - lr.item()) / abs(lr.item()) < REL_EW
    lr.backward()
    one = torch.ones(1, device=cuda)
    dz = torch.empty_like(zd)
    lib.xent_bwd(zd.data_ptr(), ld.data_ptr(), one.data_ptr(), dz.data_ptr(), n, k, 0, stream())
    assert rel_err(dz, zr.grad) < REL_EW
    w = torch.randn(1000, generator=g)
    gr = torch.randn(1000, generator=g)
    wd, gd, buf = w.to(cuda), gr.to(cuda), torch.zeros(1000, device=cuda)
    ref = w.clone().requires_grad_()
    opt = torch.optim.SGD([ref], lr=0.1, momentum=0.9, weight_decay=1e-4)
    for step in range(3):
        ref.grad = gr.clone()
        opt.step()
        lib.sgd_step(wd.data_ptr(), gd.data_ptr(), buf.data_ptr(), 1000, 0.1, 0.9, 1e-4, 1.0, int(step == 0),
                     stream())
    assert rel_err(wd, ref) < REL_EW


@pytest.mark.parametrize("variant", ["implicit", "splitk", "tf32x3"])
def test_conv_bias_and_bias_grad(cuda, variant):
    n, h, w, c, k, r, s, stride, pad = (2, 12, 12, 32, 48, 3, 3, 1, 1)
    g = torch.Generator().manual_seed(5)
    x = torch.randn(n, h, w, c, generator=g)
    wt = torch.randn(k, r, s, c, generator=g) / math.sqrt(r * s * c)
    b = torch.randn(k, generator=g)
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    lib = N.lib()
    v = N.CONV_VARIANTS[variant]
    xd, wd, bd = x.to(cuda), wt.to(cuda), b.to(cuda)
    y = torch.empty(n, d.p, d.q, k, device=cuda)
    wsb = lib.conv_ws_bytes(v, 0, d)
    ws = torch.empty(max(wsb, 4) // 4 + 1, device=cuda)
    lib.conv_fwd_bias(v, d, xd.data_ptr(), wd.data_ptr(), bd.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, stream())
    ref = conv_ref(x, wt, stride, pad) + b
    assert rel_err(y, ref) < REL_TC
    dy = torch.randn(n * d.p * d.q, k, generator=g).to(cuda)
    db = torch.full((k,), 3.0, device=cuda)
    scratch = torch.empty(lib.bn_scratch_bytes(dy.shape[0], k) // 4 + 1, device=cuda)
    lib.bias_grad(dy.data_ptr(), db.data_ptr(), dy.shape[0], k, 0, scratch.data_ptr(), stream())
    assert rel_err(db, dy.double().sum(0)) < 1e-6
    lib.bias_grad(dy.data_ptr(), db.data_ptr(), dy.shape[0], k, 1, scratch.data_ptr(), stream())
    assert rel_err(db, 2 * dy.double().sum(0)) < 1e-6


def test_dropout_mask_matches_oracle(cuda):
    """The keep-mask is bit-identical to the oracle's restatement; backward
    regenerates it; the seed is read from device memory at run time."""
    from oracle.dropout import keep_mask

    n, p, salt = 1 << 20, 0.4, 13
    lib = N.lib()
    x = torch.randn(n, device=cuda).abs_().add_(0.1)  # nonzero: y == 0 <=> dropped
    y = torch.empty_like(x)
    seed = torch.tensor([7], dtype=torch.int64, device=cuda)
    lib.dropout_fwd(x.data_ptr(), y.data_ptr(), n, ctypes.c_float(p), seed.data_ptr(), salt, stream())
    keep = torch.from_numpy(keep_mask(n, p, 7, salt)).to(cuda)
    assert torch.equal(y != 0, keep)
    scale = float(np.float32(1.0 / (1.0 - float(np.float32(p)))))
    assert torch.equal(y[keep], x[keep] * scale)
    assert abs(keep.float().mean().item() - (1 - p)) < 3e-3
    dy = torch.randn(n, device=cuda)
    dx = torch.ones(n, device=cuda)
    lib.dropout_bwd(dy.data_ptr(), dx.data_ptr(), n, ctypes.c_float(p), seed.data_ptr(), salt, 1, stream())
    assert torch.equal(dx, 1 + torch.where(keep, dy * scale, torch.zeros_like(dy)))
    lib.seed_advance(seed.data_ptr(), stream())
    lib.dropout_fwd(x.data_ptr(), y.data_ptr(), n, ctypes.c_float(p), seed.data_ptr(), salt, stream())
    assert int(seed.item()) == 8
    assert torch.equal(y != 0, torch.from_numpy(keep_mask(n, p, 8, salt)).to(cuda))


@pytest.mark.parametrize("case", [(2, 14, 14, 32, 3, 1, 1), (3, 15, 13, 96, 3, 2, 1), (2, 8, 8, 8, 3, 2, 1),
                                  (1, 33, 30, 144, 3, 1, 1), (4, 4, 4, 96, 3, 1, 1), (4, 2, 2, 160, 3, 1, 1),
                                  (2, 7, 5, 48, 3, 2, 1), (2, 56, 56, 32, 3, 1, 1), (2, 112, 112, 16, 3, 2, 1),
                                  (3, 28, 28, 48, 3, 1, 1), (2, 61, 58, 32, 3, 1, 1), (1, 120, 114, 16, 3, 2, 1)])
def test_dwconv_passes(cuda, case):
    n, h, w, c, r, stride, pad = case
    g = torch.Generator().manual_seed(7)
    x = torch.randn(n, h, w, c, generator=g)
    wt = torch.randn(c, 1, r, r, generator=g) / r
    d = N.conv_desc(n, h, w, c, c, r, r, stride, pad)
    lib = N.lib()
    xd = x.to(cuda)
    wd = wt.view(c, r, r).permute(1, 2, 0).contiguous().to(cuda)  # [R][S][C]
    y = torch.empty(n, d.p, d.q, c, device=cuda)
    lib.dwconv_fwd(d, xd.data_ptr(), wd.data_ptr(), y.data_ptr(), stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    wr = wt.double().requires_grad_()
    yr = F.conv2d(xr, wr, stride=stride, padding=pad, groups=c)
    assert rel_err(y, yr.detach().permute(0, 2, 3, 1)) < 1e-6
    dy = torch.randn(n, d.p, d.q, c, generator=g)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    dyd = dy.to(cuda)
    dx = torch.full((n, h, w, c), 2.0, device=cuda)
    lib.dwconv_dgrad(d, dyd.data_ptr(), wd.data_ptr(), dx.data_ptr(), 1, stream())
    assert rel_err(dx, 2.0 + xr.grad.permute(0, 2, 3, 1)) < 1e-6
    wsb = lib.dwconv_ws_bytes(d)
    ws = torch.empty(wsb // 4 + 1, device=cuda)
    dw = torch.empty(r, r, c, device=cuda)
    lib.dwconv_wgrad(d, xd.data_ptr(), dyd.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, stream())
    assert rel_err(dw, wr.grad.view(c, r, r).permute(1, 2, 0)) < 1e-5
    dw2 = torch.empty_like(dw)
    lib.dwconv_wgrad(d, xd.data_ptr(), dyd.data_ptr(), dw2.data_ptr(), ws.data_ptr(), wsb, stream())
    assert torch.equal(dw, dw2)  # fixed-order two-level reduction: deterministic


def test_relu6_mask_and_backward(cuda):
    from oracle.bitmask import pack_sign_mask

    n = 100003
    g = torch.Generator().manual_seed(8)
    x = (torch.randn(n, generator=g) * 5).to(cuda)
    x[:64] = torch.tensor([0.0, 6.0, -0.0, 5.999, 6.001, 1e-30] * 10 + [3.0] * 4, device=cuda)
    lib = N.lib()
    y = torch.empty_like(x)
    mask = torch.zeros((n + 31) // 32, dtype=torch.int32, device=cuda)
    lib.relu6_fwd(x.data_ptr(), y.data_ptr(), mask.data_ptr(), n, stream())
    assert torch.equal(y, torch.clamp(x, 0, 6))
    gate = ((x > 0) & (x < 6)).cpu()
    want = pack_sign_mask(torch.where(gate, 1.0, -1.0).numpy())
    assert np.array_equal(mask.cpu().numpy().view(np.uint32), want)
    dy = torch.randn(n, device=cuda)
    ref = torch.where(gate.to(cuda), dy, torch.zeros_like(dy))
    for fn, src in ((lib.relu_bwd_mask, mask), (lib.relu6_bwd_out, y), (lib.relu6_bwd_in, x)):
        dx = torch.empty_like(x)
        fn(src.data_ptr(), dy.data_ptr(), dx.data_ptr(), n, 0, stream())
        assert torch.equal(dx, ref)


@pytest.mark.parametrize("variant", ["implicit", "splitk"])
def test_conv_transpose(cuda, variant):
    """ConvTranspose2d(2x2, stride 2) through the conv kernels: forward = dgrad (+ bias),
    input gradient = forward conv (accumulating), weight gradient = wgrad."""
    n, h, w, cin, cout = 2, 9, 13, 64, 32
    g = torch.Generator().manual_seed(9)
    x = torch.randn(n, h, w, cin, generator=g)
    wt = torch.randn(cin, cout, 2, 2, generator=g) / 8
    b = torch.randn(cout, generator=g)
    d = N.conv_desc(n, 2 * h, 2 * w, cout, cin, 2, 2, 2, 0)  # the adjoint conv: y -> x
    assert (d.p, d.q) == (h, w)
    lib = N.lib()
    v = N.CONV_VARIANTS[variant]
    xd, wd, bd = x.to(cuda), wt.permute(0, 2, 3, 1).contiguous().to(cuda), b.to(cuda)
    y = torch.empty(n, 2 * h, 2 * w, cout, device=cuda)
    wsb = max(lib.convT_ws_bytes(v, 0, d), lib.convT_ws_bytes(v, 3, d))
    ws = torch.empty(wsb // 4 + 1, device=cuda)
    lib.convT_fwd(v, d, xd.data_ptr(), wd.data_ptr(), bd.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    wr = wt.double().requires_grad_()
    yr = F.conv_transpose2d(xr, wr, b.double(), stride=2)
    assert rel_err(y, yr.detach().permute(0, 2, 3, 1)) < REL_TC
    dy = torch.randn(n, 2 * h, 2 * w, cout, generator=g)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    dx = torch.ones(n, h, w, cin, device=cuda)
    dw = torch.empty(cin, 2, 2, cout, device=cuda)
    lib.convT_bwd(v, d, xd.data_ptr(), wd.data_ptr(), dy.to(cuda).data_ptr(), dx.data_ptr(), 1, dw.data_ptr(),
                  ws.data_ptr(), wsb, stream())
    assert rel_err(dx, 1 + xr.grad.permute(0, 2, 3, 1)) < REL_TC
    assert rel_err(dw, wr.grad.permute(0, 2, 3, 1)) < REL_TC


def test_pixel_xent(cuda):
    """Per-pixel softmax cross-entropy (K <= 32 path): loss = mean over N*H*W rows."""
    rows, k = 3 * 40 * 56, 4
    g = torch.Generator().manual_seed(10)
    z = torch.randn(rows, k, generator=g)
    lab = torch.randint(0, k, (rows,), generator=g, dtype=torch.int32)
    lib = N.lib()
    zd, ld = z.to(cuda), lab.to(cuda)
    loss = torch.zeros(1, device=cuda)
    scratch = torch.empty(lib.xent_scratch_bytes(rows) // 4 + 1, device=cuda)
    lib.xent_fwd(zd.data_ptr(), ld.data_ptr(), loss.data_ptr(), rows, k, scratch.data_ptr(), stream())
    zr = z.double().requires_grad_()
    ref = F.cross_entropy(zr, lab.long())
    ref.backward()
    assert abs(loss.item() - ref.item()) < 1e-5 * abs(ref.item())
    one = torch.ones(1, device=cuda)
    dz = torch.empty(rows, k, device=cuda)
    lib.xent_bwd(zd.data_ptr(), ld.data_ptr(), one.data_ptr(), dz.data_ptr(), rows, k, 0, stream())
    assert rel_err(dz, zr.grad) < 1e-5


@pytest.mark.parametrize("from_out", [1, 0])
def test_fused_bn_add_relu(cuda, from_out):
    """z = relu(BN(x) + skip) forward (train) and backward (gate from z or from x, skip):
    dx, dskip (accumulated), dgamma, dbeta against float64 autograd."""
    rows, c = 4 * 9 * 11, 64
    g = torch.Generator().manual_seed(11)
    x = torch.randn(rows, c, generator=g)
    k = torch.randn(rows, c, generator=g)
    gam, bet = torch.rand(c, generator=g) + 0.5, torch.randn(c, generator=g) * 0.1
    lib = N.lib()
    xd, kd, gd, bd = x.to(cuda), k.to(cuda), gam.to(cuda), bet.to(cuda)
    z = torch.empty(rows, c, device=cuda)
    sm, si, rm, rv, dg, db = (torch.zeros(c, device=cuda) for _ in range(6))
    rv += 1
    scratch = torch.empty(lib.bn_scratch_bytes(rows, c) // 4 + 1, device=cuda)
    lib.bnaddrelu_fwd_train(xd.data_ptr(), kd.data_ptr(), z.data_ptr(), gd.data_ptr(), bd.data_ptr(), sm.data_ptr(),
                            si.data_ptr(), rm.data_ptr(), rv.data_ptr(), rows, c, 1e-5, 0.1, 1, scratch.data_ptr(),
                            stream())
    xr, kr = x.double().requires_grad_(), k.double().requires_grad_()
    gr, br = gam.double().requires_grad_(), bet.double().requires_grad_()
    zr = torch.relu(F.batch_norm(xr, None, None, gr, br, training=True, eps=1e-5) + kr)
    assert rel_err(z, zr.detach()) < 1e-5
    dz = torch.randn(rows, c, generator=g)
    zr.backward(dz.double())
    dx = torch.ones(rows, c, device=cuda)
    dk = torch.full((rows, c), 2.0, device=cuda)
    gate = z if from_out else kd
    lib.bnaddrelu_bwd(xd.data_ptr(), gate.data_ptr(), from_out, dz.to(cuda).data_ptr(), dx.data_ptr(), 1, dk.data_ptr(),
                      1, gd.data_ptr(), bd.data_ptr(), sm.data_ptr(), si.data_ptr(), dg.data_ptr(), db.data_ptr(), rows,
                      c, scratch.data_ptr(), stream())
    assert rel_err(dx, 1 + xr.grad) < 1e-4
    assert rel_err(dk, 2 + kr.grad) < 1e-5
    assert rel_err(dg, gr.grad) < 1e-4 and rel_err(db, br.grad) < 1e-5


@pytest.mark.parametrize("k,st,pad", [(2, 2, 0), (3, 2, 1), (3, 2, 0), (3, 1, 1), (2, 1, 0)])
def test_maxpool_bwd_index_paths(cuda, k, st, pad):
    """Backward from the 8-bit index: the specialised 2x2/2 and 3x3/2 kernels and the generic one
    (stride 1), with accumulation, against float64 autograd."""
    n, h, w, c = 2, 11, 14, 32
    g = torch.Generator().manual_seed(12)
    x = torch.randn(n, h, w, c, generator=g)
    d = N.conv_desc(n, h, w, c, c, k, k, st, pad)
    lib = N.lib()
    xd = x.to(cuda)
    y = torch.empty(n, d.p, d.q, c, device=cuda)
    idx = torch.empty(n, d.p, d.q, c, dtype=torch.uint8, device=cuda)
    lib.maxpool_fwd(d, xd.data_ptr(), y.data_ptr(), idx.data_ptr(), stream())
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    yr = F.max_pool2d(xr, k, st, pad)
    dy = torch.randn(n, d.p, d.q, c, generator=g)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    dx = torch.ones(n, h, w, c, device=cuda)
    lib.maxpool_bwd(d, idx.data_ptr(), None, dy.to(cuda).data_ptr(), dx.data_ptr(), 1, stream())
    assert rel_err(dx, 1 + xr.grad.permute(0, 2, 3, 1)) < REL_EW
