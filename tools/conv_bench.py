"""Micro-benchmark of the tcgen05 conv passes on representative ResNet-50 b184 layers.

    python tools/conv_bench.py [--iters 5] [--only NAME]
Prints achieved algorithmic TFLOP/s per (layer, pass, variant).
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

LAYERS = {  # name: n, h, w, c, k, r, s, stride, pad
    "stem7x7": (184, 224, 224, 4, 64, 7, 7, 2, 3),
    "l1_1x1_64_256": (184, 56, 56, 64, 256, 1, 1, 1, 0),
    "l1_3x3_64": (184, 56, 56, 64, 64, 3, 3, 1, 1),
    "l2_3x3_128": (184, 28, 28, 128, 128, 3, 3, 1, 1),
    "l3_1x1_1024_256": (184, 14, 14, 1024, 256, 1, 1, 1, 0),
    "l4_3x3_512": (184, 7, 7, 512, 512, 3, 3, 1, 1),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--only", default=None)
    ap.add_argument("--passes", default="fwd,dgrad,wgrad")
    ap.add_argument("--variants", default="splitk")
    ap.add_argument("--fp32-weights", action="store_true", help="fwd / dgrad split the fp32 weights per tile")
    ap.add_argument("--resnet50", action="store_true",
                    help="every unique conv shape of ResNet-50 b184 224^2, weighted by its count")
    a = ap.parse_args()
    if a.resnet50:
        return resnet50_table(a)
    lib = N.lib()
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    for name, (n, h, w, c, k, r, s, stride, pad) in LAYERS.items():
        if a.only and a.only not in name:
            continue
        d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
        x = torch.randn(n, h, w, c, device=dev)
        wt = torch.randn(k, r, s, c, device=dev)
        y = torch.randn(n, d.p, d.q, k, device=dev)
        dw = torch.empty_like(wt)
        dx = torch.empty_like(x)
        n8 = (wt.numel() + 7) // 8 * 8  # the weights' bf16 split (monet_conv_*_w16)
        planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
        hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
        lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
        flops = 2.0 * n * d.p * d.q * k * c * r * s
        for vname in a.variants.split(","):
            v = N.CONV_VARIANTS[vname]
            for pss in a.passes.split(","):
                pid = N.PASS[pss]
                wsb = lib.conv_ws_bytes(v, pid, d)
                ws = torch.empty(max(wsb, 16) // 4, device=dev)
                if pss == "fwd" and a.fp32_weights:
                    fn = lambda: lib.conv_fwd(v, d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, st)
                elif pss == "fwd":
                    fn = lambda: lib.conv_fwd_w16(v, C.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None,
                                                  y.data_ptr(), ws.data_ptr(), wsb, st)
                elif pss == "dgrad" and a.fp32_weights:
                    fn = lambda: lib.conv_dgrad(v, d, y.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), wsb, st)
                elif pss == "dgrad":
                    fn = lambda: lib.conv_dgrad_w16(v, C.byref(d), y.data_ptr(), wt.data_ptr(), hi, lo, dx.data_ptr(),
                                                    0, ws.data_ptr(), wsb, st)
                else:
                    fn = lambda: lib.conv_wgrad(v, d, x.data_ptr(), y.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), wsb, st)
                fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                print(f"{name:18s} {pss:6s} {vname:8s} {ms:8.3f} ms  {flops / ms / 1e9:8.1f} TFLOP/s  ws {wsb/2**20:.1f} MiB")


def resnet50_table(a):
    """Per-shape and total conv time of one ResNet-50 training step (fwd + dgrad + wgrad)."""
    from collections import Counter

    from paper_2010_14501_b200.tracer import build_network
    net = build_network("resnet50", 184, 224)
    shapes = Counter()
    for op in net.ops:
        if op.kind == "conv":
            d = net.conv_desc(op)
            first = net.op(op.deps[0]).kind == "input"
            shapes[(d.n, d.h, d.w, d.c, d.k, d.r, d.s, d.stride_h, d.pad_h, first)] += 1
    lib = N.lib()
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    totals = {}
    for (n, h, w, c, k, r, s, stride, pad, first), cnt in sorted(shapes.items()):
        d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
        x = torch.randn(n, h, w, c, device=dev)
        wt = torch.randn(k, r, s, c, device=dev)
        y = torch.randn(n, d.p, d.q, k, device=dev)
        dw, dx = torch.empty_like(wt), torch.empty_like(x)
        # the weights' bf16 split as the executor keeps it (monet_conv_*_w16)
        n8 = (wt.numel() + 7) // 8 * 8
        planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
        hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
        lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
        flops = 2.0 * n * d.p * d.q * k * c * r * s
        line = f"{cnt:2d}x n{n} {h}x{w} c{c:4d} k{k:4d} {r}x{s}/{stride}"
        for vname in a.variants.split(","):
            v = N.CONV_VARIANTS[vname]
            tot = 0.0
            for pss in ("fwd", "dgrad", "wgrad"):
                if pss == "dgrad" and first:
                    continue
                pid = N.PASS[pss]
                wsb = lib.conv_ws_bytes(v, pid, d)
                ws = torch.empty(max(wsb, 16) // 4, device=dev)
                if pss == "fwd" and a.fp32_weights:
                    fn = lambda: lib.conv_fwd(v, d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, st)
                elif pss == "fwd":
                    fn = lambda: lib.conv_fwd_w16(v, C.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None,
                                                  y.data_ptr(), ws.data_ptr(), wsb, st)
                elif pss == "dgrad" and a.fp32_weights:
                    fn = lambda: lib.conv_dgrad(v, d, y.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), wsb, st)
                elif pss == "dgrad":
                    fn = lambda: lib.conv_dgrad_w16(v, C.byref(d), y.data_ptr(), wt.data_ptr(), hi, lo, dx.data_ptr(),
                                                    0, ws.data_ptr(), wsb, st)
                else:
                    fn = lambda: lib.conv_wgrad(v, d, x.data_ptr(), y.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), wsb, st)
                fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.iters
                tot += ms * cnt
                totals[(vname, pss)] = totals.get((vname, pss), 0.0) + ms * cnt
                line += f" | {vname[:6]} {pss[:2]} {ms:6.3f} ({flops / ms / 1e9:5.0f})"
        print(line, flush=True)
    for vname in a.variants.split(","):
        t = {p: totals.get((vname, p), 0.0) for p in ("fwd", "dgrad", "wgrad")}
        print(f"TOTAL {vname}: fwd {t['fwd']:.2f} ms  dgrad {t['dgrad']:.2f} ms  wgrad {t['wgrad']:.2f} ms  "
              f"sum {sum(t.values()):.2f} ms")


if __name__ == "__main__":
    main()
