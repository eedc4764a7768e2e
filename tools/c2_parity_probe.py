"""Where does the headline step's gradient error come from?  One ResNet-50 b184 step of the
committed 8 GiB schedule on the GPU, then the CPU oracle fed the GPU's activations and BN
statistics twice -- in fp32 and in fp64 -- and the per-tensor errors of the GPU and of the
fp32 CPU oracle, both against the fp64 oracle (max|a - ref| / max|ref|).

    python tools/c2_parity_probe.py [--batch 184] [--top 12]
"""
import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2010_14501_b200 as M  # noqa: E402
from oracle.cpu_executor import CpuState, run_step  # noqa: E402
from oracle.parity import capture, gpu_stats, grads_nhwc  # noqa: E402
from paper_2010_14501_b200.engine import Runtime  # noqa: E402
from paper_2010_14501_b200.tracer import build_network  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    net = build_network("resnet50", 184, 224, fuse=True)
    doc = json.loads((ROOT / "schedules" / "resnet50_fused_b184_224_8gib.json").read_text())
    cdoc = json.loads((ROOT / "profiles" / "catalog_resnet50_fused_b184_224.json").read_text())
    dg = hashlib.sha256(json.dumps(net.graph_doc(), sort_keys=True).encode()).hexdigest()[:16]
    assert doc["graph_digest"] == dg
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(cdoc["catalog"], g)
    sched = M.schedule_from_doc(doc["schedule"])
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(184, 3, 224, 224, generator=gen)
    y = torch.randint(0, 1000, (184,), generator=gen)
    rt = Runtime(net, device=dev, budget_bytes=doc["budget_bytes"])
    rt.set_batch(x.to(dev), y.to(dev))
    plan = rt.plan(sched, g, cat)
    acts, mism = capture(rt, plan)
    assert not mism
    stats = gpu_stats(rt)
    gpu = {k: rt.gview[k].detach().double().cpu() for k in rt.gview}
    res = {}
    for dt in (torch.float32, torch.float64):
        t = time.perf_counter()
        st = CpuState(net, dtype=dt)
        run_step(st, doc["schedule"], x, y, forced=acts, forced_stats=stats)
        res[dt] = {k: v.double() for k, v in grads_nhwc(st).items()}
        print(f"oracle {dt}: {time.perf_counter() - t:.1f} s", flush=True)
    ref = res[torch.float64]
    rows = []
    for k, r in ref.items():
        den = max(r.abs().max().item(), 1e-30)
        eg = (gpu[k].view(r.shape) - r).abs().max().item() / den
        ec = (res[torch.float32][k] - r).abs().max().item() / den
        rows.append((eg, ec, f"{net.op(k[0]).name}.{k[1]}"))
    rows.sort(reverse=True)
    print(f"{'tensor':40s} {'gpu vs f64':>12s} {'cpu f32 vs f64':>15s}")
    for eg, ec, n in rows[:a.top]:
        print(f"{n:40s} {eg:12.2e} {ec:15.2e}")
    print(f"worst gpu {max(r[0] for r in rows):.2e}   worst cpu-f32 {max(r[1] for r in rows):.2e}   "
          f"tensors {len(rows)}; gpu > 1e-4: {sum(r[0] > 1e-4 for r in rows)}; cpu-f32 > 1e-4: "
          f"{sum(r[1] > 1e-4 for r in rows)}")


if __name__ == "__main__":
    main()
