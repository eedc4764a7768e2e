"""Accuracy of the bf16x3 GEMM vs the TMEM accumulation-chain length (MONET_CHUNK).
    MONET_CHUNK=8 python tools/chunk_accuracy.py"""
import os
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

dev = torch.device("cuda:0")
lib = N.lib()
st = torch.cuda.current_stream().cuda_stream
out = []
for (n, h, w, c, k, r, s, stride, pad) in [(64, 7, 7, 512, 512, 3, 3, 1, 1), (184, 28, 28, 128, 128, 3, 3, 1, 1)]:
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(n, h, w, c, device=dev, generator=g)
    wt = torch.randn(k, r, s, c, device=dev, generator=g) / (r * s * c) ** 0.5
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    dy = torch.randn(n, d.p, d.q, k, device=dev, generator=g)
    xr = x.double().permute(0, 3, 1, 2).requires_grad_()
    wr = wt.double().permute(0, 3, 1, 2).requires_grad_()
    yr = F.conv2d(xr, wr, stride=stride, padding=pad)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    for vname in ("implicit", "splitk"):
        v = N.CONV_VARIANTS[vname]
        y = torch.empty(n, d.p, d.q, k, device=dev)
        dw = torch.empty_like(wt)
        wsb = lib.conv_ws_bytes(v, 3, d)
        ws = torch.empty(max(wsb, 16) // 4, device=dev)
        lib.conv_fwd(v, d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, st)
        lib.conv_wgrad(v, d, x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), wsb, st)
        torch.cuda.synchronize()
        ey = ((y.double() - yr.permute(0, 2, 3, 1)).abs().max() / yr.abs().max()).item()
        ew = ((dw.double() - wr.grad.permute(0, 2, 3, 1)).abs().max() / wr.grad.abs().max()).item()
        out.append(f"K_fwd={r*s*c} K_wgrad={n*d.p*d.q} {vname:8s} fwd {ey:.2e} wgrad {ew:.2e}")
print(f"chunk={os.environ.get('MONET_CHUNK', '8')}: " + " | ".join(out))
