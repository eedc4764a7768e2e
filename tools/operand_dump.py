"""Compare the raw operands the bf16x3 GEMM consumed with CPU im2col (debug tool).
    python tools/operand_dump.py n h w c k r s stride pad"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

n, h, w, c, k, r, s, stride, pad = [int(v) for v in sys.argv[1:10]]
dev = torch.device("cuda:0")
g = torch.Generator().manual_seed(0)
x = torch.randn(n, h, w, c, generator=g)
wt = torch.randn(k, r, s, c, generator=g)
d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
M, Kd = n * d.p * d.q, r * s * c
kpad = (Kd + 63) // 64 * 64
da = torch.full((M, kpad), 777.0, device=dev)
db = torch.full((k, kpad), 777.0, device=dev)
lib = N.debug_lib()  # the debug build carries the GEMM hooks
lib.dll.monet_debug_dump(da.data_ptr(), db.data_ptr())
xd, wd = x.to(dev), wt.to(dev)
y = torch.empty(n, d.p, d.q, k, device=dev)
lib.conv_fwd(0, d, xd.data_ptr(), wd.data_ptr(), y.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
lib.dll.monet_debug_dump(None, None)
xp = torch.nn.functional.pad(x, (0, 0, pad, pad, pad, pad))
cols = [xp[:, rr:rr + stride * d.p:stride, ss:ss + stride * d.q:stride, :] for rr in range(r) for ss in range(s)]
im = torch.cat(cols, dim=3).reshape(M, Kd)
A = da.cpu()[:, :Kd]
B = db.cpu()[:, :Kd]
badA = (A != im)
print("A mismatches", badA.sum().item(), "of", A.numel(), " unwritten", (A == 777).sum().item())
if badA.any():
    rows = badA.any(1).nonzero().flatten()
    print("  bad rows", rows[:10].tolist(), "count", rows.numel())
    m = rows[0].item()
    kb = badA[m].nonzero().flatten()
    print("  row", m, "bad k", kb[:40].tolist())
    for kk in kb[:6].tolist():
        v = A[m, kk].item()
        hits = (im[:, kk] == v).nonzero().flatten().tolist()[:4]
        hitk = (im[m] == v).nonzero().flatten().tolist()[:4]
        print(f"    A[{m},{kk}]={v:.4f} want {im[m, kk].item():.4f}; same value at rows {hits} / same row cols {hitk}")
Wm = wt.reshape(k, Kd)
badB = (B != Wm)
print("B mismatches", badB.sum().item(), "of", B.numel())
if badB.any():
    nz = badB.nonzero()
    print("  bad B rows", sorted(set(nz[:, 0].tolist()))[:20], "bad kblocks", sorted(set((nz[:, 1] // 32).tolist()))[:40])
    for (nn, kk) in nz[:8].tolist():
        v = B[nn, kk].item()
        hit = (Wm == v).nonzero().tolist()[:3]
        print(f"    B[{nn},{kk}]={v:.4f} want {Wm[nn, kk].item():.4f}; value found at {hit}")
