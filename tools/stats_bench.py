"""Conv forward with / without the BN statistics hand-over (monet_conv_fwd_w16[_stats]).
    python tools/stats_bench.py"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

lib = N.lib()
dev = torch.device("cuda:0")
for (n, h, w, c, k, r, s, st, pd) in [(184, 56, 56, 64, 64, 1, 1, 1, 0), (184, 56, 56, 64, 256, 1, 1, 1, 0),
                                       (184, 56, 56, 256, 64, 1, 1, 1, 0), (184, 56, 56, 64, 64, 3, 3, 1, 1),
                                       (184, 28, 28, 128, 128, 3, 3, 1, 1), (184, 14, 14, 256, 256, 3, 3, 1, 1)]:
    d = N.conv_desc(n, h, w, c, k, r, s, st, pd)
    x = torch.randn(n, h, w, c, device=dev)
    wt = torch.randn(k, r, s, c, device=dev)
    y = torch.empty(n, d.p, d.q, k, device=dev)
    n8 = (wt.numel() + 7) // 8 * 8
    planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
    hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
    lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
    stats = torch.empty(lib.conv_stats_bytes(d) // 4 + 1, device=dev)
    res = []
    for v in (0, 1):
        wsb = lib.conv_ws_bytes(v, 0, d)
        ws = torch.empty(max(wsb, 16) // 4, device=dev)
        for withs in (False, True):
            fn = (lambda: lib.conv_fwd_w16_stats(v, C.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y.data_ptr(),
                                                 stats.data_ptr(), ws.data_ptr(), wsb, None)) if withs else \
                 (lambda: lib.conv_fwd_w16(v, C.byref(d), x.data_ptr(), wt.data_ptr(), hi, lo, None, y.data_ptr(),
                                           ws.data_ptr(), wsb, None))
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res.append(f"v{v}{'+stats' if withs else '      '} {e0.elapsed_time(e1) / 10 * 1e3:7.1f} us")
    print(f"n{n} {h}x{w} c{c} k{k} {r}x{s}: " + " | ".join(res), flush=True)
