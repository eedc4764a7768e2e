"""Compare every backward step's input gradients, GPU engine vs CPU oracle (debug tool)."""
import json
import torch
import paper_2010_14501_b200 as M
from oracle.cpu_executor import CpuState, run_step
from paper_2010_14501_b200.engine import Runtime
from paper_2010_14501_b200.tracer import build_network

doc = json.load(open("tests/golden/r18_b8_64.json"))
net = build_network("resnet18", 8, 64)
g = M.load_graph(doc["graph"]); cat = M.load_catalog(doc["catalog"], g)
gen = torch.Generator().manual_seed(0)
x = torch.randn(8, 3, 64, 64, generator=gen); y = torch.randint(0, 1000, (8,), generator=gen)
dev = torch.device("cuda:0")
case = doc["store_everything"]
sched = M.schedule_from_doc(case["schedule"])
rec = {}
st = CpuState(net, dtype=torch.float64)
run_step(st, case["schedule"], x.double(), y, record=rec)
rt = Runtime(net)
rt.set_batch(x.to(dev), y.to(dev))
plan = rt.plan(sched, g, cat)
base = rt.arena.data_ptr()
printed = [0]


def view(ptr, shape):
    off = ptr - base
    n = 1
    for d in shape:
        n *= d
    return rt.arena[off:off + 4 * n].view(torch.float32).view(shape)


def after(i):
    s = plan.steps[i]
    if s.kind != "backward" or printed[0] > 25:
        return
    torch.cuda.synchronize()
    op = net.op(s.node)
    for j in op.deps:
        key = ("g", j)
        if key not in plan.step_ptrs[i] or net.grad_bytes(net.op(j)) == 0:
            continue
        shp = net.op(j).shape
        got = view(plan.step_ptrs[i][key], shp).double().cpu()
        want = rec[s.stage][j]
        if want.dim() == 4:
            want = want.permute(0, 2, 3, 1)
        e = (got - want).abs().max().item() / (want.abs().max().item() + 1e-30)
        flag = "  <<<" if e > 1e-4 else ""
        if e > 1e-4 or s.node > 40:
            print(f"stage {s.stage:3d} node {s.node:3d} {op.kind:7s} {op.name:24s} [{s.impl}] -> grad {j:3d} rel {e:.2e} new={j in s.new_grads}{flag}")
            if e > 1e-4:
                printed[0] += 1


rt.run(plan, after_step=after)
torch.cuda.synchronize()
