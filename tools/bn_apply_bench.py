"""Event-timed BN backward-apply kernels at a ResNet-50 layer1 tensor (debug tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

dev = torch.device("cuda:0")
lib = N.lib()
st = torch.cuda.current_stream().cuda_stream
n, h, w, c = 184, 56, 56, 256
rows = n * h * w
x, dz, z, k = (torch.randn(rows * c, device=dev) for _ in range(4))
dx, dk = torch.empty_like(x), torch.empty_like(x)
g, b = torch.rand(c, device=dev) + 0.5, torch.randn(c, device=dev)
m, s, rm, rv, dg, db = (torch.zeros(c, device=dev) for _ in range(6))
s += 1
scratch = torch.empty(lib.bn_scratch_bytes(rows, c) // 4 + 1, device=dev)
E = x.numel()


def timed(name, fn, nbytes):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:22s} {ms * 1e3:8.1f} us {nbytes / (ms * 1e-3) / 1e9:8.0f} GB/s")


timed("bnrelu_bwd", lambda: lib.bnrelu_bwd(x.data_ptr(), dz.data_ptr(), dx.data_ptr(), 0, g.data_ptr(), b.data_ptr(),
                                           m.data_ptr(), s.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c,
                                           scratch.data_ptr(), st), 20 * E)
timed("bnaddrelu_bwd", lambda: lib.bnaddrelu_bwd(x.data_ptr(), z.data_ptr(), 1, dz.data_ptr(), dx.data_ptr(), 0,
                                                 dk.data_ptr(), 0, g.data_ptr(), b.data_ptr(), m.data_ptr(),
                                                 s.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c,
                                                 scratch.data_ptr(), st), 32 * E)
timed("bnaddrelu_fwd", lambda: lib.bnaddrelu_fwd_train(x.data_ptr(), k.data_ptr(), z.data_ptr(), g.data_ptr(),
                                                       b.data_ptr(), m.data_ptr(), s.data_ptr(), rm.data_ptr(),
                                                       rv.data_ptr(), rows, c, 1e-5, 0.1, 1, scratch.data_ptr(), st),
      16 * E)
timed("bn_bwd_in", lambda: lib.bn_bwd_in(x.data_ptr(), dz.data_ptr(), dx.data_ptr(), 0, g.data_ptr(), m.data_ptr(),
                                         s.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c, scratch.data_ptr(), st),
      20 * E)
print("ok")
