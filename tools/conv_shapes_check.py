"""Bit-compare the pre-split-weight conv path with the fp32 path on every conv shape of a
traced network, check run-to-run determinism, and the error against float64 torch.
    python tools/conv_shapes_check.py googlenet 4 64 [--fuse]"""
import ctypes as C
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402
from paper_2010_14501_b200.tracer import build_network  # noqa: E402

arch, batch, image = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
net = build_network(arch, batch, image, num_classes=10, fuse="--fuse" in sys.argv)
lib = N.lib()
dev = torch.device("cuda:0")
seen = set()
bad = 0
for op in net.ops:
    if op.kind not in ("conv", "convrelu"):
        continue
    d = net.conv_desc(op)
    key = tuple(getattr(d, f) for f, _ in N.ConvDesc._fields_) + (net.op(op.deps[0]).kind == "input",)
    if key in seen:
        continue
    seen.add(key)
    g = torch.Generator().manual_seed(len(seen))
    x = torch.randn(d.n, d.h, d.w, d.c, generator=g).to(dev)
    wt = (torch.randn(d.k, d.r, d.s, d.c, generator=g) / (d.r * d.s * d.c) ** 0.5).to(dev)
    dy = torch.randn(d.n, d.p, d.q, d.k, generator=g).to(dev)
    n8 = (wt.numel() + 7) // 8 * 8
    planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
    hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
    lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
    msgs = []
    for v in (0, 1):
        wsb = max(lib.conv_ws_bytes(v, 0, d), lib.conv_ws_bytes(v, 3, d))
        ws = torch.empty(max(wsb, 16) // 4 + 1, device=dev)
        ys = []
        for fn in ("fp32", "w16", "w16"):
            y = torch.full((d.n, d.p, d.q, d.k), 3.0, device=dev)
            if fn == "fp32":
                lib.conv_fwd(v, d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, None)
            else:
                lib.conv_fwd_w16(v, C.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y.data_ptr(),
                                 ws.data_ptr(), wsb, None)
            ys.append(y)
        ref = F.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(0, 3, 1, 2), stride=d.stride_h,
                       padding=d.pad_h).permute(0, 2, 3, 1)
        e = ((ys[1].double() - ref).abs().max() / ref.abs().max()).item()
        if not torch.equal(ys[0], ys[1]) or not torch.equal(ys[1], ys[2]) or e > 5e-5:
            msgs.append(f"fwd v{v}: eq_fp32={torch.equal(ys[0], ys[1])} det={torch.equal(ys[1], ys[2])} rel={e:.2e}")
        if net.op(op.deps[0]).kind != "input":
            dxs = []
            for fn in ("fp32", "w16", "w16"):
                dx = torch.full_like(x, 3.0)
                if fn == "fp32":
                    lib.conv_dgrad(v, d, dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), wsb, None)
                else:
                    lib.conv_dgrad_w16(v, C.byref(d), dy.data_ptr(), wt.data_ptr(), hi, lo, dx.data_ptr(), 0,
                                       ws.data_ptr(), wsb, None)
                dxs.append(dx)
            xr = x.double().permute(0, 3, 1, 2).requires_grad_()
            F.conv2d(xr, wt.double().permute(0, 3, 1, 2), stride=d.stride_h, padding=d.pad_h).backward(
                dy.double().permute(0, 3, 1, 2))
            ref = xr.grad.permute(0, 2, 3, 1)
            e = ((dxs[1].double() - ref).abs().max() / ref.abs().max()).item()
            if not torch.equal(dxs[0], dxs[1]) or not torch.equal(dxs[1], dxs[2]) or e > 5e-5:
                msgs.append(f"dgrad v{v}: eq_fp32={torch.equal(dxs[0], dxs[1])} det={torch.equal(dxs[1], dxs[2])} "
                            f"rel={e:.2e}")
    torch.cuda.synchronize()
    line = f"{op.name:40s} n{d.n} {d.h}x{d.w} c{d.c} k{d.k} {d.r}x{d.s}/{d.stride_h}"
    print(line, "OK" if not msgs else "BAD " + "; ".join(msgs), flush=True)
    bad += bool(msgs)
print("bad shapes:", bad)
