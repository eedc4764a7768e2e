"""Locate mismatching output rows of one conv pass (debug tool).
    python tools/conv_debug.py n h w c k r s stride pad [variant]"""
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402

a = [int(v) for v in sys.argv[1:10]]
variant = sys.argv[10] if len(sys.argv) > 10 else "implicit"
n, h, w, c, k, r, s, stride, pad = a
dev = torch.device("cuda:0")
g = torch.Generator().manual_seed(0)
x = torch.randn(n, h, w, c, generator=g)
wt = torch.randn(k, r, s, c, generator=g)
d = N.conv_desc(*a)
v = N.CONV_VARIANTS[variant]
xd, wd = x.to(dev), wt.to(dev)
y = torch.full((n, d.p, d.q, k), 12345.0, device=dev)
N.lib().conv_fwd(v, d, xd.data_ptr(), wd.data_ptr(), y.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ref = F.conv2d(x.double().permute(0, 3, 1, 2), wt.double().permute(0, 3, 1, 2), stride=stride, padding=pad)
ref = ref.permute(0, 2, 3, 1)
err = (y.double().cpu() - ref).abs() / ref.abs().max()
bad = (err > 1e-4).any(dim=3)
print("rows bad:", bad.sum().item(), "of", bad.numel())
idx = bad.nonzero().tolist()
for (i, j, kk) in idx[:40]:
    m = (i * d.p + j) * d.q + kk
    cols = (err[i, j, kk] > 1e-4).nonzero().flatten().tolist()
    print(f"  n{i} p{j} q{kk} (m={m}, tile {m // 128} row {m % 128}) bad cols {len(cols)}: {cols[:8]}")

# attribute the error of each bad row to k-blocks (32 channels of one tap):
# err[m, :] ~= sum_kb alpha_kb * P_kb[m, :]  (alpha = -1: block missing, +1: doubled)
if bad.any() and len(sys.argv) > 11:
    xp = torch.nn.functional.pad(x.double(), (0, 0, pad, pad, pad, pad))  # NHWC pad W,H
    blocks = []
    names = []
    for rr in range(r):
        for ss in range(s):
            for c0 in range(0, c, 32):
                patch = xp[:, rr:rr + stride * d.p:stride, ss:ss + stride * d.q:stride, c0:c0 + 32]
                contrib = torch.einsum("nhwc,kc->nhwk", patch, wt.double()[:, rr, ss, c0:c0 + 32])
                blocks.append(contrib.reshape(-1, k))
                names.append(f"t{rr}{ss}c{c0}")
    Pm = torch.stack(blocks, 0)  # B, M, K
    E = (y.double().cpu() - ref).reshape(-1, k)
    for m in bad.reshape(-1).nonzero().flatten().tolist()[:12]:
        A = Pm[:, m, :].t()  # K x B
        sol = torch.linalg.lstsq(A, E[m].unsqueeze(1)).solution.flatten()
        big = [(names[i], round(sol[i].item(), 2)) for i in range(len(names)) if abs(sol[i]) > 0.05]
        print(f"  m={m}: {big[:10]}")

# chunk-level attribution: contributions of k ranges [512 j, 512 (j+1)) (8 MMA stages)
if bad.any() and len(sys.argv) > 11:
    xp = torch.nn.functional.pad(x.double(), (0, 0, pad, pad, pad, pad))
    cols = []
    for rr in range(r):
        for ss in range(s):
            patch = xp[:, rr:rr + stride * d.p:stride, ss:ss + stride * d.q:stride, :]
            cols.append(patch)
    im = torch.cat(cols, dim=3).reshape(-1, r * s * c)   # M x Kd (k = tap*C + c)
    wk = wt.double().reshape(k, -1)                       # K x Kd
    E = (y.double().cpu() - ref).reshape(-1, k)
    CH = 512
    parts = [im[:, j:j + CH] @ wk[:, j:j + CH].t() for j in range(0, r * s * c, CH)]
    P = torch.stack(parts, 0)
    for m in bad.reshape(-1).nonzero().flatten().tolist()[:6]:
        sol = torch.linalg.lstsq(P[:, m, :].t(), E[m].unsqueeze(1)).solution.flatten()
        print(f"  chunk attribution m={m}: {[round(v, 3) for v in sol.tolist()]}  resid "
              f"{(P[:, m, :].t() @ sol - E[m]).abs().max().item():.3e} |E| {E[m].abs().max().item():.3e}")
