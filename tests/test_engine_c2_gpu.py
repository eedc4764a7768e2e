"""Parity at the headline configuration: ResNet-50, batch 184, 224x224, fused BN+ReLU graph,
the committed 8 GiB MONeT schedule (schedules/resnet50_fused_b184_224_8gib.json) and the
measured catalog it was planned on -- exactly what bench.py times.

One training step on the B200 against the torch-CPU oracle (oracle/cpu_executor.py):

  * the executed ledger equals simulate() and the planned footprint stays within the
    ILP bound and the 8 GiB budget;
  * every recompute is bit-identical to the first forward (BN replays saved statistics);
  * loss: the free-running oracle (its own forward) within rel 1e-4;
  * with the GPU's activations fed to the oracle (ReLU gates and maxpool argmax are
    discontinuous): every parameter gradient, every SGD-updated weight,
    and (from the free-running oracle) every BN running statistic within rel 1e-4 --
    max|gpu - cpu| / max|cpu| per tensor (oracle/parity.py:step_parity).
"""
import json
from pathlib import Path

import pytest
import torch

import paper_2010_14501_b200 as M
from oracle.cpu_executor import CpuState, run_step
from oracle.parity import capture, gpu_stats, step_parity, worst
from paper_2010_14501_b200.engine import Runtime
from paper_2010_14501_b200.tracer import build_network

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
REL = 1e-4
BATCH = 184


def rel(a, b, scale=None):
    """max|a - b| / max|b| (or / max|scale| for means, whose size is the spread's)."""
    a, b = a.double(), b.double()
    den = (b if scale is None else 1.0 / scale.double()).abs().max().item()
    return (a - b).abs().max().item() / max(den, 1e-30)


@pytest.fixture(scope="module")
def c2():
    import hashlib

    net = build_network("resnet50", BATCH, 224, fuse=True)
    doc = json.loads((ROOT / "schedules" / "resnet50_fused_b184_224_8gib.json").read_text())
    digest = hashlib.sha256(json.dumps(net.graph_doc(), sort_keys=True).encode()).hexdigest()[:16]
    assert doc["graph_digest"] == digest, "committed schedule was planned for another graph"
    cat_doc = json.loads((ROOT / "profiles" / "catalog_resnet50_fused_b184_224.json").read_text())
    assert cat_doc["graph_digest"] == digest
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(cat_doc["catalog"], g)
    return net, g, cat, doc


def test_resnet50_b184_8gib_step_matches_oracle(cuda, c2):
    net, g, cat, doc = c2
    sched = M.schedule_from_doc(doc["schedule"])
    assert sum(1 for s in sched.stages for u, impl in s.recompute if impl is not None) > 0
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(BATCH, 3, 224, 224, generator=gen)
    y = torch.randint(0, 1000, (BATCH,), generator=gen)

    rt = Runtime(net, device=cuda, budget_bytes=doc["budget_bytes"])
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    assert M.trace_report(plan.trace) == M.trace_report(M.simulate(sched, g, cat))
    assert plan.ledger_peak <= plan.bound_peak <= doc["budget_bytes"]
    assert plan.within_bound
    acts, mismatched = capture(rt, plan)
    assert not mismatched, f"recomputes not bit-identical: {mismatched}"
    gpu_loss = rt.loss_value()

    torch.set_num_threads(max(1, torch.get_num_threads()))
    free = CpuState(net)
    loss = run_step(free, doc["schedule"], x, y)
    assert abs(gpu_loss - loss) <= REL * abs(loss), (gpu_loss, loss)

    # the GPU's saved batch statistics against float64 statistics of the GPU's own BN inputs
    stats = gpu_stats(rt)
    for i, (m, s) in stats.items():
        op = net.op(i)
        xin = acts[op.attrs["x"] if op.kind == "bnaddrelu" else op.deps[0]].double()
        m64 = xin.mean(dim=(0, 2, 3))
        s64 = 1.0 / torch.sqrt(xin.var(dim=(0, 2, 3), unbiased=False) + op.attrs["eps"])
        assert rel(m, m64, s64) <= 1e-5 and rel(s, s64) <= 1e-5, (op.name, rel(m, m64, s64), rel(s, s64))

    st = CpuState(net)
    run_step(st, doc["schedule"], x, y, forced=acts, forced_stats=stats)
    del acts
    rep = step_parity(rt, st, free)
    kind, err, name = worst(rep)
    counts = {k: len(v) for k, v in rep.items()}
    print(f"C2 parity: loss gpu {gpu_loss:.6f} cpu {loss:.6f}; tensors {counts}; worst {kind} {name} {err:.2e}")
    assert counts["grad"] == counts["param"] == sum(len(op.params) for op in net.ops)
    assert counts["running"] == 2 * len(rt.bn)
    for k, v in rep.items():
        bad = [(e, n) for e, n in v if not e <= REL]
        assert not bad, (k, sorted(bad, reverse=True)[:5])
