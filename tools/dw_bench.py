"""Depthwise conv passes of MobileNet-V2 b272 224^2 (every distinct shape, weighted by count):
time per pass and achieved HBM GB/s over the algorithmic bytes (x + y, dy + dx, x + dy).
    python tools/dw_bench.py [H [stride]] [--iters N] [--warmup N]   (H / stride: only those shapes)"""
import argparse
import sys
from collections import Counter
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402
from paper_2010_14501_b200.tracer import build_network  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("h", type=int, nargs="?")
ap.add_argument("stride", type=int, nargs="?")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
net = build_network("mobilenet_v2", 272, 224, fuse=True)
lib = N.lib()
dev = torch.device("cuda:0")
shapes = Counter()
for op in net.ops:
    if op.kind == "dwconv":
        d = net.conv_desc(op)
        if (a.h is None or d.h == a.h) and (a.stride is None or d.stride_h == a.stride):
            shapes[(d.n, d.h, d.w, d.c, d.r, d.s, d.stride_h, d.pad_h)] += 1
tot = {"fwd": 0.0, "dgrad": 0.0, "wgrad": 0.0}
for (n, h, w, c, r, s, st, pd), cnt in sorted(shapes.items()):
    d = N.conv_desc(n, h, w, c, c, r, s, st, pd)
    x = torch.randn(n, h, w, c, device=dev)
    wt = torch.randn(r, s, c, device=dev)
    y = torch.empty(n, d.p, d.q, c, device=dev)
    dx, dw = torch.empty_like(x), torch.empty_like(wt)
    wsb = lib.dwconv_ws_bytes(d)
    ws = torch.empty(wsb // 4 + 1, device=dev)
    line = f"{cnt}x {h}x{w} c{c} s{st}:"
    for pss, fn, nbytes in (
            ("fwd", lambda: lib.dwconv_fwd(d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), None), x.numel() + y.numel()),
            ("dgrad", lambda: lib.dwconv_dgrad(d, y.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, None),
             x.numel() + y.numel()),
            ("wgrad", lambda: lib.dwconv_wgrad(d, x.data_ptr(), y.data_ptr(), dw.data_ptr(), ws.data_ptr(), wsb, None),
             x.numel() + y.numel())):
        for _ in range(a.warmup):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        tot[pss] += ms * cnt
        line += f" {pss} {ms * 1e3:7.1f} us ({4 * nbytes / ms / 1e6:5.0f} GB/s)"
    print(line, flush=True)
print("TOTAL " + "  ".join(f"{k} {v:.2f} ms" for k, v in tot.items()))
