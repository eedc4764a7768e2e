"""Repeat every conv pass of tests/test_kernels_gpu.py's shapes many times and
check that each launch is bit-identical to the first (the GEMM epilogue order is
fixed, so any difference is a race) and within tolerance of float64 torch.

    python tools/race_stress.py [--reps 50] [--variants implicit,splitk]
"""
import argparse
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2010_14501_b200 import _native as N  # noqa: E402
from test_kernels_gpu import CONV_CASES, conv_ref, rel_err  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--variants", default="implicit,splitk")
    a = ap.parse_args()
    cuda = torch.device("cuda:0")
    lib = N.lib()
    st = torch.cuda.current_stream().cuda_stream
    bad = 0
    for variant in a.variants.split(","):
        v = N.CONV_VARIANTS[variant]
        for ci, (n, h, w, c, k, r, s, stride, pad) in enumerate(CONV_CASES):
            g = torch.Generator().manual_seed(0)
            x = torch.randn(n, h, w, c, generator=g)
            wt = torch.randn(k, r, s, c, generator=g) / math.sqrt(r * s * c)
            d = N.conv_desc(n, h, w, c, k, r, s, stride, pad)
            xd, wd = x.to(cuda), wt.to(cuda)
            y = torch.empty(n, d.p, d.q, k, device=cuda)
            ws_b = max(lib.conv_ws_bytes(v, p, d) for p in (0, 1, 2))
            ws = torch.empty(max(ws_b, 4) // 4 + 1, device=cuda)
            dy = torch.randn(n, d.p, d.q, k, generator=g).to(cuda)
            dx = torch.empty_like(xd)
            dw = torch.empty_like(wd)
            ref = conv_ref(x, wt, stride, pad)
            first = {}
            diffs = {"fwd": 0, "dgrad": 0, "wgrad": 0}
            worst = {"fwd": 0.0}
            for _ in range(a.reps):
                lib.conv_fwd(v, d, xd.data_ptr(), wd.data_ptr(), y.data_ptr(), ws.data_ptr(), ws_b, st)
                lib.conv_dgrad(v, d, dy.data_ptr(), wd.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), ws_b, st)
                lib.conv_wgrad(v, d, xd.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, ws.data_ptr(), ws_b, st)
                torch.cuda.synchronize()
                for name, t in (("fwd", y), ("dgrad", dx), ("wgrad", dw)):
                    if name not in first:
                        first[name] = t.clone()
                    elif not torch.equal(first[name], t):
                        diffs[name] += 1
                worst["fwd"] = max(worst["fwd"], rel_err(y, ref))
            flag = any(diffs.values()) or worst["fwd"] > 5e-5
            bad += flag
            print(f"{variant:8s} case{ci:2d} {(n, h, w, c, k, r, s, stride, pad)}: nondeterministic "
                  f"{diffs} worst fwd rel {worst['fwd']:.2e}{'  <-- FAIL' if flag else ''}", flush=True)
    print(f"race_stress: {bad} failing (variant, case) pairs")


if __name__ == "__main__":
    main()
