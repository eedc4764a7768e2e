"""One launch each of the HBM-bound local-op kernels on a ResNet-50 layer1 tensor (profiling target)."""
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
x = torch.randn(rows * c, device=dev)
z = torch.empty_like(x)
dz = torch.randn_like(x)
dx = torch.empty_like(x)
mask = torch.empty((x.numel() + 31) // 32, dtype=torch.int32, device=dev)
g, b = torch.rand(c, device=dev) + 0.5, torch.randn(c, device=dev)
m, s, rm, rv, dg, db = (torch.zeros(c, device=dev) for _ in range(6))
scratch = torch.empty(lib.bn_scratch_bytes(rows, c) // 4 + 1, device=dev)
lib.relu_fwd(x.data_ptr(), z.data_ptr(), mask.data_ptr(), x.numel(), st)
lib.bnrelu_fwd_train(x.data_ptr(), z.data_ptr(), g.data_ptr(), b.data_ptr(), m.data_ptr(), s.data_ptr(),
                     rm.data_ptr(), rv.data_ptr(), rows, c, 1e-5, 0.1, 1, scratch.data_ptr(), st)
lib.bnrelu_bwd(x.data_ptr(), dz.data_ptr(), dx.data_ptr(), 0, g.data_ptr(), b.data_ptr(), m.data_ptr(),
               s.data_ptr(), dg.data_ptr(), db.data_ptr(), rows, c, scratch.data_ptr(), st)
torch.cuda.synchronize()
print("ok")
