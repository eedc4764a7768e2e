"""Run-to-run stress of the pre-split-weight conv passes on every conv shape of a traced network
at a batch large enough for several tiles per CTA: each forward / input-gradient launch must be
bit-identical to the first (the epilogue order is fixed, so any difference is a race).

    python tools/w16_race_stress.py resnet50 64 224 [--reps 8]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402
from paper_2010_14501_b200.tracer import build_network  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("arch")
    ap.add_argument("batch", type=int)
    ap.add_argument("image", type=int)
    ap.add_argument("--reps", type=int, default=8)
    a = ap.parse_args()
    net = build_network(a.arch, a.batch, a.image, num_classes=10, fuse=True)
    lib = N.lib()
    dev = torch.device("cuda:0")
    seen, bad = set(), 0
    for op in net.ops:
        if op.kind not in ("conv", "convrelu"):
            continue
        d = net.conv_desc(op)
        key = tuple(getattr(d, f) for f, _ in N.ConvDesc._fields_)
        if key in seen:
            continue
        seen.add(key)
        g = torch.Generator(device=dev).manual_seed(len(seen))
        x = torch.randn(d.n, d.h, d.w, d.c, device=dev, generator=g)
        wt = torch.randn(d.k, d.r, d.s, d.c, device=dev, generator=g)
        dy = torch.randn(d.n, d.p, d.q, d.k, device=dev, generator=g)
        n8 = (wt.numel() + 7) // 8 * 8
        planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
        hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
        lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
        msgs = []
        for v in (0, 1):
            wsb = max(lib.conv_ws_bytes(v, 0, d), lib.conv_ws_bytes(v, 3, d))
            ws = torch.empty(max(wsb, 16) // 4 + 1, device=dev)
            y0, dx0 = None, None
            for rep in range(a.reps):
                y = torch.full((d.n, d.p, d.q, d.k), float(rep), device=dev)
                lib.conv_fwd_w16(v, C.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y.data_ptr(),
                                 ws.data_ptr(), wsb, None)
                if y0 is None:
                    y0 = y
                elif not torch.equal(y0, y):
                    msgs.append(f"fwd v{v} rep {rep}")
                    break
            if net.op(op.deps[0]).kind == "input":
                continue
            for rep in range(a.reps):
                dx = torch.full_like(x, float(rep))
                lib.conv_dgrad_w16(v, C.byref(d), dy.data_ptr(), wt.data_ptr(), hi, lo, dx.data_ptr(), 0,
                                   ws.data_ptr(), wsb, None)
                if dx0 is None:
                    dx0 = dx
                elif not torch.equal(dx0, dx):
                    msgs.append(f"dgrad v{v} rep {rep}")
                    break
        torch.cuda.synchronize()
        print(f"{op.name:40s} n{d.n} {d.h}x{d.w} c{d.c} k{d.k} {d.r}x{d.s}/{d.stride_h}",
              "OK" if not msgs else "RACE " + ", ".join(msgs), flush=True)
        bad += bool(msgs)
    print("racy shapes:", bad)


if __name__ == "__main__":
    main()
