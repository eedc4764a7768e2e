"""Per-role barrier wait cycles of the bf16x3 GEMM for one conv pass (debug tool).
    python tools/gemm_waits.py LAYER PASS   (layers of tools/conv_bench.py)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_14501_b200 import _native as N  # noqa: E402
from tools.conv_bench import LAYERS  # noqa: E402

name, pss = sys.argv[1], sys.argv[2]
n, h, w, c, k, r, s, stride, pad = LAYERS[name]
dev = torch.device("cuda:0")
d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
x = torch.randn(n, h, w, c, device=dev)
wt = torch.randn(k, r, s, c, device=dev)
y = torch.randn(n, d.p, d.q, k, device=dev)
lib = N.debug_lib()  # the debug build carries the GEMM hooks
v = N.CONV_VARIANTS["splitk"]
pid = N.PASS[pss]
wsb = lib.conv_ws_bytes(v, pid, d)
ws = torch.empty(max(wsb, 16) // 4, device=dev)
st = torch.cuda.current_stream().cuda_stream
cnt = torch.zeros(16, dtype=torch.int64, device=dev)
if pss == "fwd":
    fn = lambda: lib.conv_fwd(v, d, x.data_ptr(), wt.data_ptr(), y.data_ptr(), ws.data_ptr(), wsb, st)
elif pss == "dgrad":
    dx = torch.empty_like(x)
    fn = lambda: lib.conv_dgrad(v, d, y.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), wsb, st)
else:
    dw = torch.empty_like(wt)
    fn = lambda: lib.conv_wgrad(v, d, x.data_ptr(), y.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), wsb, st)
fn()
torch.cuda.synchronize()
lib.dll.monet_debug_timers(cnt.data_ptr())
fn()
torch.cuda.synchronize()
lib.dll.monet_debug_timers(None)
c_ = cnt.cpu().tolist()
tot = c_[15]
names = {0: "loader raw_empty", 3: "MMA a_full", 4: "MMA b_full", 5: "MMA tempty", 6: "epi tfull",
         7: "Asplit st_empty", 8: "Asplit raw_full", 9: "Bsplit st_empty", 10: "Bsplit raw_full",
         11: "MMA issue loop"}
print(f"{name} {pss}: kernel cycles (sum over CTAs) {tot:.3e}")
for i, nm in names.items():
    print(f"  {nm:18s} {100.0 * c_[i] / max(tot, 1):6.1f}%")
