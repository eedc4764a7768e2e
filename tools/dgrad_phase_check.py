"""Strided (sub-pixel phase) dgrad: fp32-weight vs pre-split-weight path, run to run."""
import ctypes as C
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

import os
lib = N.debug_lib() if os.environ.get("DBG") else N.lib()
dev = torch.device("cuda:0")
for (n, h, w, c, k, r, s, st, pd) in [(32, 56, 56, 256, 512, 1, 1, 2, 0), (32, 56, 56, 128, 128, 3, 3, 2, 1),
                                       (4, 56, 56, 256, 512, 1, 1, 2, 0), (3, 14, 14, 64, 128, 3, 3, 2, 1)]:
    d = N.conv_desc(n, h, w, c, k, r, s, st, pd)
    g = torch.Generator().manual_seed(0)
    wt = (torch.randn(k, r, s, c, generator=g) / (r * s * c) ** 0.5).to(dev)
    dy = torch.randn(n, d.p, d.q, k, generator=g).to(dev)
    n8 = (wt.numel() + 7) // 8 * 8
    planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
    hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
    lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
    xr = torch.zeros(n, c, h, w, dtype=torch.float64, requires_grad=True)
    F.conv2d(xr, wt.double().cpu().permute(0, 3, 1, 2), stride=st, padding=pd).backward(dy.double().cpu().permute(0, 3, 1, 2))
    ref = xr.grad.permute(0, 2, 3, 1)
    out = []
    for path in ("fp32", "fp32", "w16", "w16", "w16"):
        dx = torch.full((n, h, w, c), 3.0, device=dev)
        if path == "fp32":
            lib.conv_dgrad(0, d, dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, None, 0, None)
        else:
            lib.conv_dgrad_w16(0, C.byref(d), dy.data_ptr(), wt.data_ptr(), hi, lo, dx.data_ptr(), 0, None, 0, None)
        torch.cuda.synchronize()
        e = ((dx.double().cpu() - ref).abs().max() / ref.abs().max()).item()
        bad = ((dx.double().cpu() - ref).abs() > 1e-3 * ref.abs().max()).nonzero()
        out.append(f"{path} {e:.1e} nbad={len(bad)}" + (f" first={bad[0].tolist()}" if len(bad) else ""))
    print(f"n{n} {h}x{w} c{c} k{k} {r}x{s}/{st}: " + " | ".join(out), flush=True)
