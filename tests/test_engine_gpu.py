"""End-to-end parity of the GPU executor (config 1: ResNet-18, batch 8, 64x64).

For the store-everything schedule and the reference-planned recompute
schedule at a tight budget (tests/golden/r18_b8_64.json):
  * the executed ledger equals the reference simulate() trace byte for byte;
  * the planned physical footprint (params_bytes + arena high-water mark)
    stays within the budget, and the ledger peak within the ILP bound;
  * every recompute reproduces its forward activation bit for bit (BN replays
    saved statistics);
  * forward activations and the loss match the CPU oracle within
    rel 1e-4 (max|gpu-cpu| / max|cpu| per tensor);
  * with the GPU's activations fed to the oracle (ReLU/maxpool derivatives are
    discontinuous: a 1-ulp difference in x near 0 flips a mask bit), every
    parameter gradient, updated weight and BN running statistic matches within
    rel 1e-4 (fp32 storage, 3xTF32 tensor-core convolutions).
"""
import json
from pathlib import Path

import pytest
import torch

import paper_2010_14501_b200 as M
from oracle.cpu_executor import CpuState, params_nhwc, run_step
from paper_2010_14501_b200.engine import Runtime
from paper_2010_14501_b200.tracer import build_network
from oracle.parity import capture, gpu_stats, rel, step_parity

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
REL = 1e-4


def _assert_step_parity(rt, st):
    """Every parameter gradient, SGD-updated weight and BN running statistic within REL,
    per tensor (oracle/parity.py:step_parity:
    tensors whose exact value is ~0 -- e.g. the bias gradient of a BN feeding a 1x1
    conv and another BN in MobileNet-V2's linear bottlenecks -- are judged against
    1 % of the largest tensor of their kind instead of their own rounding noise)."""
    rep = step_parity(rt, st)
    assert rep["grad"] and rep["param"]
    for kind, v in rep.items():
        bad = sorted(((e, n) for e, n in v if not e <= REL), reverse=True)
        assert not bad, (kind, bad[:5])


@pytest.fixture(scope="module")
def r18():
    doc = json.loads((GOLD / "r18_b8_64.json").read_text())
    net = build_network("resnet18", 8, 64)
    assert net.graph_doc() == doc["graph"], "tracer output drifted from the frozen graph"
    g = M.load_graph(doc["graph"])
    cat = M.load_catalog(doc["catalog"], g)
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(8, 3, 64, 64, generator=gen)
    y = torch.randint(0, 1000, (8,), generator=gen)
    cases = [("store_everything", doc["store_everything"], None)]
    cases += [(f"{c['status']}-{c['budget']}", c, c["budget"]) for c in doc["cases"] if "trace_csv" in c]
    return net, g, cat, x, y, cases


@pytest.mark.parametrize("which", [0, 1])
def test_engine_matches_reference_ledger_and_oracle(cuda, r18, which):
    net, g, cat, x, y, cases = r18
    name, case, budget = cases[which]
    sched = M.schedule_from_doc(case["schedule"])
    rt = Runtime(net, budget_bytes=budget)
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    acts, mismatched = capture(rt, plan)
    assert not mismatched, f"recompute not bit-identical for nodes {mismatched}"
    assert M.trace_report(plan.trace) == case["trace_csv"]
    assert plan.ledger_peak == case["peak"]
    if budget is not None:
        assert g.params_bytes + plan.arena_bytes <= budget
        assert plan.ledger_peak <= plan.bound_peak <= budget
    # free-running oracle: forward and loss
    free = CpuState(net)
    loss = run_step(free, case["schedule"], x, y)
    assert abs(rt.loss_value() - loss) <= REL * abs(loss)
    # oracle fed with the GPU activations: backward, weights, statistics
    st = CpuState(net)
    run_step(st, case["schedule"], x, y, forced=acts, forced_stats=gpu_stats(rt))
    for (nid, pname), v in params_nhwc(st).items():
        got = rt.pview[(nid, pname)].view(v.shape)
        assert rel(got, v) <= REL, (name, net.op(nid).name, pname, rel(got, v))
        gg = st.grads[(nid, pname)]
        if net.op(nid).kind in ("conv", "convrelu") and pname == "weight":
            gg = gg.permute(0, 2, 3, 1)
        assert rel(rt.gview[(nid, pname)].view(gg.shape), gg) <= REL, (name, net.op(nid).name, pname, "grad")
    for op in net.ops:
        if op.kind == "bn":
            rm, rv = free.running[op.id]
            assert rel(rt.bn[op.id][2], rm) <= REL and rel(rt.bn[op.id][3], rv) <= REL


@pytest.mark.parametrize("split", [False, True])
def test_fused_bn_relu_engine(cuda, split):
    """ResNet-18 with fused BN+ReLU ops under a recompute schedule: ledger = simulate(),
    loss / weights / gradients = CPU oracle (fed the GPU activations).  ``split``: conv
    backward split into dgrad / wgrad nodes (tracer.split_conv_backward), with in-place
    recomputes where the planner finds them."""
    net = build_network("resnet18", 4, 32, num_classes=10, fuse=True, split=split)
    assert net.split == split
    assert any(op.kind == "bnrelu" for op in net.ops)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    se = M.store_everything_schedule(g, cat)
    act = M.simulate(se, g, cat).peak_memory - g.params_bytes
    from paper_2010_14501_b200.planner import plan_schedule
    sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.5 * act), kinds=net.storable_kinds())
    assert sched is not None and any(s.recompute for s in sched.stages)
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(4, 3, 32, 32, generator=gen)
    y = torch.randint(0, 10, (4,), generator=gen)
    rt = Runtime(net)
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    assert M.trace_report(plan.trace) == M.trace_report(M.simulate(sched, g, cat))
    acts, mismatched = capture(rt, plan)
    assert not mismatched
    doc = M.schedule_to_doc(sched)
    free = CpuState(net)
    loss = run_step(free, doc, x, y)
    assert abs(rt.loss_value() - loss) <= REL * abs(loss)
    st = CpuState(net)
    run_step(st, doc, x, y, forced=acts, forced_stats=gpu_stats(rt))
    _assert_step_parity(rt, st)


def test_forward_ops_match_oracle(cuda, r18):
    """Each forward op, evaluated by the oracle on the GPU's own inputs, matches the GPU output."""
    net, g, cat, x, y, cases = r18
    sched = M.schedule_from_doc(cases[0][1]["schedule"])
    rt = Runtime(net)
    rt.set_batch(x.to(cuda), y.to(cuda))
    acts, _ = capture(rt, rt.plan(sched, g, cat))
    mine = {}
    run_step(CpuState(net), cases[0][1]["schedule"], x, y, forced=acts, fwd_record=mine)
    worst = max((rel(acts[i], mine[i]), net.op(i).name) for i in acts if i in mine)
    assert worst[0] <= REL, worst


def test_budget_exceeded_raises(cuda, r18):
    net, g, cat, x, y, cases = r18
    se = M.schedule_from_doc(cases[0][1]["schedule"])
    rt = Runtime(net, budget_bytes=g.params_bytes + 1024)
    with pytest.raises(M.BudgetExceeded):
        rt.plan(se, g, cat)


def test_invalid_schedule_raises(cuda, r18):
    net, g, cat, x, y, cases = r18
    doc = json.loads(json.dumps(cases[0][1]["schedule"]))
    doc["stages"][3]["store"] = []  # drop a dependency the backward still needs
    rt = Runtime(net)
    with pytest.raises(M.SimulationError):
        rt.plan(M.schedule_from_doc(doc), g, cat)


@pytest.mark.parametrize("fuse,split", [(False, False), (True, False), (True, True)])
def test_vgg_style_engine(cuda, fuse, split):
    """VGG-family ops (biased convs, identity adaptive pool, flatten -> fc, dropout)
    under a recompute schedule: ledger = simulate(), every recompute bit-identical
    (dropout regenerates its mask), loss / weights / gradients = CPU oracle; also with
    conv+ReLU fused (convrelu: in-place ReLU + mask, dy gated in place) and split."""
    from nets import SmallVGG

    torch.manual_seed(0)
    net = M.trace_graph(SmallVGG(), torch.empty(4, 3, 32, 32, device="meta"), 10, fuse, split)
    assert any(op.kind == "dropout" for op in net.ops)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    se = M.store_everything_schedule(g, cat)
    act = M.simulate(se, g, cat).peak_memory - g.params_bytes
    from paper_2010_14501_b200.planner import plan_schedule
    sched = None
    for frac in (0.6, 0.7, 0.8):  # the tightest fraction with a recompute schedule
        sched, _ = plan_schedule(g, cat, g.params_bytes + int(frac * act), kinds=net.storable_kinds())
        if sched is not None and any(s.recompute for s in sched.stages):
            break
    assert sched is not None and any(s.recompute for s in sched.stages)
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(4, 3, 32, 32, generator=gen)
    y = torch.randint(0, 10, (4,), generator=gen)
    rt = Runtime(net)
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    assert M.trace_report(plan.trace) == M.trace_report(M.simulate(sched, g, cat))
    acts, mismatched = capture(rt, plan)  # one step at dropout seed 0
    assert not mismatched
    doc = M.schedule_to_doc(sched)
    free = CpuState(net)
    loss = run_step(free, doc, x, y)
    assert abs(rt.loss_value() - loss) <= REL * abs(loss)
    st = CpuState(net)
    run_step(st, doc, x, y, forced=acts, forced_stats=gpu_stats(rt))
    for (nid, pname), v in params_nhwc(st).items():
        assert rel(rt.pview[(nid, pname)].view(v.shape), v) <= REL, (net.op(nid).name, pname)
        gg = st.grads[(nid, pname)]
        if net.op(nid).kind in ("conv", "convrelu") and pname == "weight":
            gg = gg.permute(0, 2, 3, 1)
        assert rel(rt.gview[(nid, pname)].view(gg.shape), gg) <= REL, (net.op(nid).name, pname, "grad")
    assert int(rt.seed.item()) == 1  # advanced once by the optimizer group


@pytest.mark.parametrize("fuse", [False, True])
def test_mobilenet_v2_engine(cuda, fuse):
    """torchvision MobileNet-V2 (width 0.25, 64 x 64): depthwise convs, ReLU6 masks,
    residual adds, dropout under a recompute schedule -- ledger = simulate(), recomputes
    bit-identical, loss / weights / gradients = CPU oracle (fed the GPU activations)."""
    import torchvision

    torch.manual_seed(0)
    model = torchvision.models.mobilenet_v2(num_classes=10, width_mult=0.25)
    net = M.trace_graph(model, torch.empty(4, 3, 64, 64, device="meta"), 10, fuse=fuse)
    assert any(op.kind == "bnrelu6" for op in net.ops) == fuse
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    se = M.store_everything_schedule(g, cat)
    act = M.simulate(se, g, cat).peak_memory - g.params_bytes
    from paper_2010_14501_b200.planner import plan_schedule
    sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.6 * act), kinds=net.storable_kinds())
    assert sched is not None and any(s.recompute for s in sched.stages)
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(4, 3, 64, 64, generator=gen)
    y = torch.randint(0, 10, (4,), generator=gen)
    rt = Runtime(net)
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    assert M.trace_report(plan.trace) == M.trace_report(M.simulate(sched, g, cat))
    acts, mismatched = capture(rt, plan)
    assert not mismatched
    doc = M.schedule_to_doc(sched)
    free = CpuState(net)
    loss = run_step(free, doc, x, y)
    assert abs(rt.loss_value() - loss) <= REL * abs(loss)
    st = CpuState(net)
    run_step(st, doc, x, y, forced=acts, forced_stats=gpu_stats(rt))
    _assert_step_parity(rt, st)


@pytest.mark.parametrize("fuse", [False, True])
def test_googlenet_engine(cuda, fuse):
    """torchvision GoogLeNet (64 x 64): concat forward / slice backward, ceil-mode pools with
    8-bit indices, under a recompute schedule -- ledger = simulate(), recomputes
    bit-identical, loss and updated weights = CPU oracle (fed the GPU activations)."""
    import torchvision

    torch.manual_seed(0)
    model = torchvision.models.googlenet(num_classes=10, aux_logits=False, init_weights=True)
    net = M.trace_graph(model, torch.empty(4, 3, 64, 64, device="meta"), 10, fuse=fuse)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    se = M.store_everything_schedule(g, cat)
    act = M.simulate(se, g, cat).peak_memory - g.params_bytes
    from paper_2010_14501_b200.planner import plan_schedule
    sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.6 * act), kinds=net.storable_kinds())
    assert sched is not None and any(s.recompute for s in sched.stages)
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(4, 3, 64, 64, generator=gen)
    y = torch.randint(0, 10, (4,), generator=gen)
    rt = Runtime(net)
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    assert M.trace_report(plan.trace) == M.trace_report(M.simulate(sched, g, cat))
    acts, mismatched = capture(rt, plan)
    assert not mismatched
    doc = M.schedule_to_doc(sched)
    free = CpuState(net)
    loss = run_step(free, doc, x, y)
    assert abs(rt.loss_value() - loss) <= REL * abs(loss)
    st = CpuState(net)
    run_step(st, doc, x, y, forced=acts, forced_stats=gpu_stats(rt))
    _assert_step_parity(rt, st)


def test_unet_engine(cuda):
    """UNet (width 8, 32 x 48): transposed convs with bias, decoder concats, per-pixel loss, under a
    recompute schedule -- ledger = simulate(), recomputes bit-identical, loss / weights = oracle."""
    from paper_2010_14501_b200.tracer import UNet

    torch.manual_seed(0)
    net = M.trace_graph(UNet(num_classes=4, width=8), torch.empty(2, 3, 32, 48, device="meta"), 4, fuse=True)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    se = M.store_everything_schedule(g, cat)
    act = M.simulate(se, g, cat).peak_memory - g.params_bytes
    from paper_2010_14501_b200.planner import plan_schedule
    sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.6 * act), kinds=net.storable_kinds())
    assert sched is not None and any(s.recompute for s in sched.stages)
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(2, 3, 32, 48, generator=gen)
    y = torch.randint(0, 4, (2, 32, 48), generator=gen)
    rt = Runtime(net)
    rt.set_batch(x.to(cuda), y.to(cuda))
    plan = rt.plan(sched, g, cat)
    assert M.trace_report(plan.trace) == M.trace_report(M.simulate(sched, g, cat))
    acts, mismatched = capture(rt, plan)
    assert not mismatched
    doc = M.schedule_to_doc(sched)
    free = CpuState(net)
    loss = run_step(free, doc, x, y)
    assert abs(rt.loss_value() - loss) <= REL * abs(loss)
    st = CpuState(net)
    run_step(st, doc, x, y, forced=acts, forced_stats=gpu_stats(rt))
    _assert_step_parity(rt, st)


def test_cli_train_execute_exit_codes(cuda, tmp_path):
    """`train` / `execute` on the GPU with the reference's exit codes: 0 ok, 5 invalid schedule,
    6 planned footprint over the budget."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    common = ["--arch", "resnet18", "--batch", "4", "--image", "32", "--classes", "10", "--fuse"]

    def run(*args):
        return subprocess.run([sys.executable, "-m", "paper_2010_14501_b200", *args], cwd=root, capture_output=True,
                              text=True, timeout=900)

    r = run("train", *common, "--budget-gib", "1", "--steps", "2", "-o", str(tmp_path / "t.json"))
    assert r.returncode == 0, r.stderr
    out = json.loads((tmp_path / "t.json").read_text())
    assert len(out["losses"]) == 2 and out["physical_peak_bytes"] <= out["ilp_bound_bytes"] <= 1 << 30
    assert run("plan", *common, "--budget-gib", "1", "-o", str(tmp_path / "s.json")).returncode == 0
    assert run("execute", *common, "--schedule", str(tmp_path / "s.json"), "--budget-gib", "1").returncode == 0
    doc = json.loads((tmp_path / "s.json").read_text())
    doc["schedule"]["stages"][2]["store"] = []  # drop what the remaining backward stages read
    (tmp_path / "bad.json").write_text(json.dumps(doc))
    assert run("execute", *common, "--schedule", str(tmp_path / "bad.json")).returncode == 5
    assert run("execute", *common, "--schedule", str(tmp_path / "s.json"), "--budget-gib", "0.01").returncode == 6


def test_prefetch_pipeline_matches_direct_staging(cuda):
    """Runtime.prefetch (the next batch copied while the step runs, after the step's last
    read of the staging buffer) gives the same losses and weights, bit for bit, as staging
    each batch synchronously -- on a schedule that recomputes the input copy as well."""
    net = build_network("resnet18", 4, 32, num_classes=10)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    sets = M.compute_dependency_sets(g)
    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    sched = M.checkpoint_heuristic(g, sets, cat, g.params_bytes + int(0.6 * act))
    assert sched is not None
    gen = torch.Generator().manual_seed(5)
    xs = [torch.randn(4, 32, 32, 4, generator=gen).pin_memory() for _ in range(3)]
    ys = [torch.randint(0, 10, (4,), generator=gen, dtype=torch.int32).pin_memory() for _ in range(3)]
    out = []
    for mode in ("direct", "prefetch"):
        rt = Runtime(net, device=cuda)
        plan = rt.plan(sched, g, cat)
        rt.capture(plan)
        losses = []
        if mode == "prefetch":
            rt.prefetch(xs[0], ys[0])
        for i in range(3):
            if mode == "direct":
                lt = rt.train_step(plan, xs[i], ys[i])
            else:
                lt = rt.train_step(plan)
                if i + 1 < 3:
                    rt.prefetch(xs[i + 1], ys[i + 1])
            losses.append(float(lt.item()))
        out.append((losses, rt.params.clone()))
    assert out[0][0] == out[1][0]
    assert torch.equal(out[0][1], out[1][1])
