"""Which stage of the bf16x3 GEMM pipeline limits a conv pass (debug build only).

    MONET_DBG_MODE=<bits> python tools/gemm_limiter.py LAYER PASS [LAYER PASS ...]

Bits of MONET_DBG_MODE skip work while keeping every barrier hand-off: 1 the A split
(LDS + split + tcgen05.st), 2 the B split (LDS + STS), 4 the MMAs, 8 the epilogue
stores.  Mode 15 leaves only the TMA operand delivery; the drop in time per skipped
stage says what the full kernel waits on.  Results are garbage in the skip modes.
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402
from tools.conv_bench import LAYERS  # noqa: E402

lib = N.debug_lib()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
mode = int(os.environ.get("MONET_DBG_MODE", "0"))
args = sys.argv[1:]
for name, pss in zip(args[::2], args[1::2]):
    n, h, w, c, k, r, s, stride, pad = LAYERS[name]
    d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
    x = torch.randn(n, h, w, c, device=dev)
    wt = torch.randn(k, r, s, c, device=dev)
    y = torch.randn(n, d.p, d.q, k, device=dev)
    v = N.CONV_VARIANTS["splitk"]
    wsb = lib.conv_ws_bytes(v, N.PASS[pss], d)
    ws = torch.empty(max(wsb, 16) // 4, device=dev)
    n8 = (wt.numel() + 7) // 8 * 8  # the weights' bf16 split, as the executor keeps it
    planes = torch.zeros(2 * n8, dtype=torch.int16, device=dev)
    hi, lo = planes.data_ptr(), planes.data_ptr() + 2 * n8
    lib.split_bf16(wt.data_ptr(), hi, lo, wt.numel(), None)
    if pss == "fwd":
        fn = lambda: lib.conv_fwd_w16(v, d, x.data_ptr(), wt.data_ptr(), hi, lo, None, y.data_ptr(), ws.data_ptr(),
                                      wsb, st)
    elif pss == "dgrad":
        dx = torch.empty_like(x)
        fn = lambda: lib.conv_dgrad_w16(v, d, y.data_ptr(), wt.data_ptr(), hi, lo, dx.data_ptr(), 0, ws.data_ptr(),
                                        wsb, st)
    else:
        dw = torch.empty_like(wt)
        fn = lambda: lib.conv_wgrad(v, d, x.data_ptr(), y.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), wsb, st)
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flops = 2.0 * n * d.p * d.q * k * c * r * s
    print(f"mode {mode:2d} {name:16s} {pss:5s} {ms * 1e3:8.1f} us  {flops / ms / 1e9:6.1f} TF/s")
