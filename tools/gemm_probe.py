"""GPU probe of the tcgen05 GEMM layouts (debug tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N

lib = N.lib()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream


def run(A, B, amn, bmn, variant=0):
    m, k = A.shape
    n = B.shape[0]
    a = (A.t().contiguous() if amn else A).to(dev)
    b = (B.t().contiguous() if bmn else B).to(dev)
    C = torch.full((m, n), -7.0, device=dev)
    lib.gemm(variant, a.data_ptr(), amn, m if amn else k, b.data_ptr(), bmn, n if bmn else k, C.data_ptr(), n, m, n,
             k, 0, None, 0, st)
    torch.cuda.synchronize()
    return C.cpu()


torch.manual_seed(0)
for (m, n, k) in [(128, 128, 32), (128, 128, 64), (200, 1000, 2048), (256, 128, 32), (128, 256, 32), (77, 36, 20)]:
    A, B = torch.randn(m, k), torch.randn(n, k)
    ref = A.double() @ B.double().t()
    for amn, bmn in [(0, 0), (0, 1), (1, 0), (1, 1)]:
        if (amn and m % 4) or (bmn and n % 4):
            continue
        for v in (0, 3, 2):
            C = run(A, B, amn, bmn, v)
            err = (C.double() - ref).abs().max().item() / ref.abs().max().item()
            print(f"m{m} n{n} k{k} amn{amn} bmn{bmn} v{v}: rel {err:.3e} untouched {(C == -7).sum().item()} zeros {(C == 0).sum().item()}")

# pattern probe: which k does each (m, n) pick up
m, n, k = 128, 128, 32
A = torch.zeros(m, k)
for i in range(m):
    A[i, i % k] = 1.0
B = torch.arange(n * k, dtype=torch.float32).view(n, k)  # B[n,k] = n*k + k
for amn, bmn in [(0, 0), (0, 1), (1, 0), (1, 1)]:
    C = run(A, B, amn, bmn, 0)
    ref = (A @ B.t())
    bad = (C != ref).nonzero()
    print("pattern", amn, bmn, "mismatches", bad.shape[0])
    for (i, j) in bad[:12].tolist():
        print(f"   C[{i},{j}]={C[i,j].item()} want {ref[i,j].item()}")
