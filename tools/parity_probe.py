"""GPU-vs-CPU(fp32)-vs-CPU(fp64) gradient parity probe for ResNet-18 (debug tool)."""
import json, sys
import torch
import paper_2010_14501_b200 as M
from oracle.cpu_executor import CpuState, run_step
from paper_2010_14501_b200.engine import Runtime, execute
from paper_2010_14501_b200.tracer import build_network

doc = json.load(open("tests/golden/r18_b8_64.json"))
net = build_network("resnet18", 8, 64)
g = M.load_graph(doc["graph"]); cat = M.load_catalog(doc["catalog"], g)
gen = torch.Generator().manual_seed(0)
x = torch.randn(8, 3, 64, 64, generator=gen); y = torch.randint(0, 1000, (8,), generator=gen)
dev = torch.device("cuda:0")
for name, case in [("store_all", doc["store_everything"])] + [(c["status"], c) for c in doc["cases"] if "trace_csv" in c][:1]:
    sched = M.schedule_from_doc(case["schedule"])
    rt = Runtime(net)
    res = execute(sched, g, cat, runtime=rt, images=x.to(dev), labels=y.to(dev))
    s32 = CpuState(net); l32 = run_step(s32, case["schedule"], x, y)
    s64 = CpuState(net, dtype=torch.float64); l64 = run_step(s64, case["schedule"], x.double(), y)
    print(name, "loss gpu %.9f cpu32 %.9f cpu64 %.9f" % (res.loss, l32, l64))
    worst = []
    for (nid, pname), g64 in s64.grads.items():
        op = net.op(nid)
        shape = g64.shape
        gg = rt.gview[(nid, pname)].double().cpu()
        t64 = g64.double()
        t32 = s32.grads[(nid, pname)].double()
        if op.kind == "conv" and pname == "weight":
            t64 = t64.permute(0, 2, 3, 1).reshape(-1); t32 = t32.permute(0, 2, 3, 1).reshape(-1)
        t64 = t64.reshape(-1); t32 = t32.reshape(-1)
        den = t64.abs().max().item() + 1e-30
        e_g64 = (gg - t64).abs().max().item() / den
        e_32 = (t32 - t64).abs().max().item() / den
        e_g32 = (gg - t32).abs().max().item() / den
        worst.append((nid, e_g64, op.name, pname, e_g32, e_32))
    worst.sort(reverse=True)
    for w in worst:
        print("  %3d %-28s %-6s gpu-f64 %.2e  gpu-f32 %.2e  f32-f64 %.2e" % (w[0], w[2], w[3], w[1], w[4], w[5]))
    break
