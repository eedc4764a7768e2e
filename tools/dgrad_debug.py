"""Per-phase error of the strided dgrad (debug tool).
    python tools/dgrad_debug.py n h w c k r s stride pad [variant] [accumulate]"""
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

a = [int(v) for v in sys.argv[1:10]]
variant = sys.argv[10] if len(sys.argv) > 10 else "implicit"
n, h, w, c, k, r, s, stride, pad = a
dev = torch.device("cuda:0")
g = torch.Generator().manual_seed(0)
wt = torch.randn(k, r, s, c, generator=g)
d = N.conv_desc(*a)
dy = torch.randn(n, d.p, d.q, k, generator=g)
v = N.CONV_VARIANTS[variant]
wsb = N.lib().conv_ws_bytes(v, 1, d)
ws = torch.empty(max(wsb, 16) // 4, device=dev)
dx = torch.full((n, h, w, c), 7.0, device=dev)
dyd, wd = dy.to(dev), wt.to(dev)
N.lib().conv_dgrad(v, d, dyd.data_ptr(), wd.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), wsb,
                   torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
xr = torch.zeros(n, c, h, w, dtype=torch.float64, requires_grad=True)
F.conv2d(xr, wt.double().permute(0, 3, 1, 2), stride=stride, padding=pad).backward(dy.double().permute(0, 3, 1, 2))
ref = xr.grad.permute(0, 2, 3, 1)
err = (dx.double().cpu() - ref).abs() / ref.abs().max()
print("max rel", err.max().item())
for pa in range(stride):
    for pb in range(stride):
        e = err[:, pa::stride, pb::stride, :]
        bad = (e > 1e-4).any(dim=3)
        print(f"phase ({pa},{pb}): max {e.max().item():.2e} bad pixels {bad.sum().item()} of {bad.numel()}")
        if bad.any():
            print("   first bad (n,i,j):", bad.nonzero()[:6].tolist(), " value", dx.cpu()[tuple(bad.nonzero()[0].tolist()[:1]) + (pa + stride * bad.nonzero()[0, 1].item(), pb + stride * bad.nonzero()[0, 2].item())][:4].tolist(), "ref", ref[tuple(bad.nonzero()[0].tolist()[:1]) + (pa + stride * bad.nonzero()[0, 1].item(), pb + stride * bad.nonzero()[0, 2].item())][:4].tolist())
