"""One launch each of the C3/C4 kernels at their largest config shapes (profiling target):
MobileNet-V2 b272 depthwise 3x3 on [272,112,112,96] (stride 2) and [272,56,56,144] (stride 1),
fused BN+ReLU6 on [272,112,112,96], dropout on VGG-16's fc input [176,25088], concat of GoogLeNet
inception3a ([320,28,28,64+128+32+32]).  Prints event-timed GB/s for each as a cross-check."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

dev = torch.device("cuda:0")
lib = N.lib()
st = torch.cuda.current_stream().cuda_stream


def timed(name, fn, nbytes, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"{name:34s} {ms * 1e3:9.1f} us  {nbytes / (ms * 1e-3) / 1e9:8.1f} GB/s (algorithmic {nbytes / 1e6:.0f} MB)")


# depthwise 3x3 stride 2 on the 112^2 expand output (block 2) and stride 1 at 56^2 (block 3)
for (n, h, w, c, s) in ((272, 112, 112, 96, 2), (272, 56, 56, 144, 1)):
    d = N.conv_desc(n, h, w, c, c, 3, 3, s, 1)
    x = torch.randn(n, h, w, c, device=dev)
    wt = torch.randn(3, 3, c, device=dev)
    y = torch.empty(n, d.p, d.q, c, device=dev)
    dy = torch.randn_like(y)
    dx = torch.empty_like(x)
    dw = torch.empty_like(wt)
    wsb = lib.dwconv_ws_bytes(d)
    ws = torch.empty(wsb // 4 + 1, device=dev)
    xb, yb = x.numel() * 4, y.numel() * 4
    timed(f"dwconv_fwd s{s} c{c}", lambda: lib.dwconv_fwd(d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), st), xb + yb)
    timed(f"dwconv_dgrad s{s} c{c}", lambda: lib.dwconv_dgrad(d, dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, st),
          xb + yb)
    timed(f"dwconv_wgrad s{s} c{c}", lambda: lib.dwconv_wgrad(d, x.data_ptr(), dy.data_ptr(), dw.data_ptr(),
                                                              ws.data_ptr(), wsb, st), xb + yb)
    del x, y, dy, dx

# fused BN+ReLU6 forward (stats + apply) and backward
n, h, w, c = 272, 112, 112, 96
rows = n * h * w
x = torch.randn(rows * c, device=dev)
z, dz, dxx = torch.empty_like(x), torch.randn_like(x), torch.empty_like(x)
g, b = torch.rand(c, device=dev) + 0.5, torch.randn(c, device=dev)
m, s_, rm, rv, dg, db = (torch.zeros(c, device=dev) for _ in range(6))
scratch = torch.empty(lib.bn_scratch_bytes(rows, c) // 4 + 1, device=dev)
E = x.numel()
timed("bnrelu6_fwd_train", lambda: lib.bnrelu6_fwd_train(x.data_ptr(), z.data_ptr(), g.data_ptr(), b.data_ptr(),
                                                         m.data_ptr(), s_.data_ptr(), rm.data_ptr(), rv.data_ptr(),
                                                         rows, c, 1e-5, 0.1, 1, scratch.data_ptr(), st), 12 * E)
timed("bnrelu6_bwd", lambda: lib.bnrelu6_bwd(x.data_ptr(), dz.data_ptr(), dxx.data_ptr(), 0, g.data_ptr(),
                                             b.data_ptr(), m.data_ptr(), s_.data_ptr(), dg.data_ptr(), db.data_ptr(),
                                             rows, c, scratch.data_ptr(), st), 20 * E)
del x, z, dz, dxx

# dropout on the VGG-16 classifier input and a large activation-sized tensor
seed = torch.zeros(1, dtype=torch.int64, device=dev)
for numel in (176 * 25088, 184 * 56 * 56 * 256):
    a, o = torch.randn(numel, device=dev), torch.empty(numel, device=dev)
    timed(f"dropout_fwd n={numel}", lambda: lib.dropout_fwd(a.data_ptr(), o.data_ptr(), numel, 0.5, seed.data_ptr(), 3,
                                                            st), 8 * numel)

# GoogLeNet inception3a concat: 4 branches into 256 channels at 28^2, batch 320
n, h, w = 320, 28, 28
chans = (64, 128, 32, 32)
ins = [torch.randn(n * h * w * cj, device=dev) for cj in chans]
out = torch.empty(n * h * w * sum(chans), device=dev)


def cat():
    off = 0
    for t, cj in zip(ins, chans):
        lib.channel_copy(t.data_ptr(), cj, 0, out.data_ptr(), sum(chans), off, cj, n * h * w, 0, st)
        off += cj


timed("concat (4 channel_copy)", cat, 8 * out.numel())
print("ok")
