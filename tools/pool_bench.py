"""Event-timed maxpool backward (index path) at the VGG-16 and ResNet-50 shapes (debug tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

dev = torch.device("cuda:0")
lib = N.lib()
st = torch.cuda.current_stream().cuda_stream
for (n, h, w, c, k, s, pad) in ((176, 224, 224, 64, 2, 2, 0), (184, 112, 112, 64, 3, 2, 1)):
    d = N.conv_desc(n, h, w, c, c, k, k, s, pad)
    x = torch.randn(n, h, w, c, device=dev)
    y = torch.empty(n, d.p, d.q, c, device=dev)
    idx = torch.empty(n, d.p, d.q, c, dtype=torch.uint8, device=dev)
    lib.maxpool_fwd(d, x.data_ptr(), y.data_ptr(), idx.data_ptr(), st)
    dx = torch.empty_like(x)
    fn = lambda: lib.maxpool_bwd(d, idx.data_ptr(), None, y.data_ptr(), dx.data_ptr(), 0, st)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nb = x.numel() * 4 + y.numel() * 5
    print(f"maxpool_bwd {k}x{k}/{s} [{n},{h},{w},{c}]: {ms * 1e3:.1f} us, {nb / (ms * 1e-3) / 1e9:.0f} GB/s")
