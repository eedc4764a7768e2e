"""Conv-backward split.

split_conv_backward turns every conv whose input has a gradient into two graph nodes: the
conv (forward; backward = dgrad, reading only dy and the weights) and a zero-byte "wgrad"
anchor right after it (backward = the weight gradient, reading x and the conv's dy).  The
graph stays a reference graph document: it loads in the reference's remsched, which
simulates it to the same ledger as the product, and the CPU oracle gives the same loss and
gradients as the unsplit graph.  The memory point: the conv input can die right after
its weight gradient, so VGG-16 b176 plans at 8.5 GiB with the split and not without.
"""
import os
import sys

import pytest
import torch

import paper_2010_14501_b200 as M
from oracle.cpu_executor import CpuState, run_step
from oracle.parity import grads_nhwc
from paper_2010_14501_b200.planner import plan_schedule
from paper_2010_14501_b200.tracer import build_network


def _net(split, fuse=True):
    net = build_network("resnet18", 2, 32, num_classes=10, fuse=fuse, split=split)
    g = M.load_graph(net.graph_doc())
    return net, g, M.load_catalog(net.catalog_doc(), g)


def test_split_graph_structure():
    net, g, cat = _net(True)
    convs = [op for op in net.ops if op.kind == "conv"]
    anchors = [op for op in net.ops if op.kind == "wgrad"]
    assert len(anchors) == len(convs) - 1                 # the stem reads the network input: not split
    loss = net.ops[-1]
    assert loss.kind == "xent" and set(loss.deps[1:]) == {a.id for a in anchors}
    for w in anchors:
        conv = net.op(w.attrs["conv"])
        assert w.deps == (conv.id,) and w.id == conv.id + 1 and conv.attrs["split"]
        assert g.output_bytes(w.id) == 0 and g.grad_bytes(w.id) == 0
        assert [list(v.deps) for v in cat.bwd(w.id)] == [[conv.deps[0]]] * 2    # wgrad reads x
        assert [list(v.deps) for v in cat.bwd(conv.id)] == [[], []]             # dgrad reads nothing


@pytest.mark.parametrize("fuse", [False, True])
def test_split_oracle_equals_unsplit(fuse):
    gen = torch.Generator().manual_seed(0)
    x = torch.randn(2, 3, 32, 32, generator=gen)
    y = torch.tensor([1, 7])
    res = []
    for split in (False, True):
        net, g, cat = _net(split, fuse)
        act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
        sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.5 * act), kinds=net.storable_kinds())
        assert sched is not None and any(s.recompute for s in sched.stages)
        st = CpuState(net)
        loss = run_step(st, M.schedule_to_doc(sched), x, y)
        by_name = {(net.op(n).name, p): v for (n, p), v in grads_nhwc(st).items()}
        res.append((loss, by_name))
    (l0, g0), (l1, g1) = res
    assert l0 == l1 and g0.keys() == g1.keys()
    for k in g0:
        assert torch.equal(g0[k], g1[k]), k


def test_vgg16_plans_lower_with_split():
    """VGG-16 b176 224^2: without the split the conv1_2 backward holds x, dy and dx (2.1 GiB
    each) at once; with it no 8.5 GiB schedule is needed to hold them together."""
    budget = int(8.5 * (1 << 30))
    found = {}
    for split in (False, True):
        net = build_network("vgg16", 176, 224, split=split)
        g = M.load_graph(net.graph_doc())
        cat = M.load_catalog(net.catalog_doc(), g)
        sched, info = plan_schedule(g, cat, budget, kinds=net.storable_kinds())
        found[split] = sched
        if sched is not None:
            ok, bound, _ = M.check_schedule(g, M.compute_dependency_sets(g), cat, sched, budget)
            assert ok and M.simulate(sched, g, cat).peak_memory <= bound <= budget
    assert found[False] is None and found[True] is not None


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_split_graph_in_reference():
    sys.path.insert(0, "/root/reference/pkg/src")
    import remsched as R

    net, g, cat = _net(True)
    rg = R.load_graph(net.graph_doc())
    rc = R.load_catalog(net.catalog_doc(), rg)
    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.5 * act), kinds=net.storable_kinds())
    rs = R.schedule_from_doc(M.schedule_to_doc(sched))
    assert R.validate(rs, rg, R.compute_dependency_sets(rg), rc) == []
    assert R.trace_report(R.simulate(rs, rg, rc)) == M.trace_report(M.simulate(sched, g, cat))
    budget = g.params_bytes + int(0.5 * act)
    assert R.check_schedule(rg, R.compute_dependency_sets(rg), rc, rs, budget)[:2] == \
        M.check_schedule(g, M.compute_dependency_sets(g), cat, sched, budget)[:2]


def test_vgg16_fused_split_plans_at_7gib():
    """VGG-16 b176 224^2 with conv+ReLU fused (convrelu: dy gated in place by the 1-bit mask)
    and the conv backward split: the conv1_2 backward holds only x and dy (2.1 GiB each) next
    to the 1.7 GiB fixed region, so the reference ILP (solved by HiGHS) is feasible at 7 GiB,
    where the unfused split graph -- which also holds the ReLU's separate input gradient --
    is not; the planned schedule passes the exact bound and the simulator."""
    budget = 7 << 30
    for fuse in (False, True):
        net = build_network("vgg16", 176, 224, fuse=fuse, split=True)
        g = M.load_graph(net.graph_doc())
        cat = M.load_catalog(net.catalog_doc(), g)
        sched, info = plan_schedule(g, cat, budget, kinds=net.storable_kinds(), lp=True, mip_time_s=60)
        if not fuse:
            assert sched is None
            continue
        assert sched is not None, info
        ok, bound, _ = M.check_schedule(g, M.compute_dependency_sets(g), cat, sched, budget)
        assert ok and M.simulate(sched, g, cat).peak_memory <= bound <= budget


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_fused_split_vgg_graph_in_reference():
    """The convrelu graph (mask intermediate, split anchors reading the mask) is a valid
    reference graph document: a planned schedule validates and simulates identically."""
    sys.path.insert(0, "/root/reference/pkg/src")
    import remsched as R
    from nets import SmallVGG
    from paper_2010_14501_b200.tracer import trace_graph

    torch.manual_seed(0)
    net = trace_graph(SmallVGG(), torch.empty(4, 3, 32, 32, device="meta"), 10, True, True)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    rg = R.load_graph(net.graph_doc())
    rc = R.load_catalog(net.catalog_doc(), rg)
    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    budget = g.params_bytes + int(0.6 * act)
    sched, _ = plan_schedule(g, cat, budget, kinds=net.storable_kinds())
    assert sched is not None and any(st.recompute for st in sched.stages)
    rs = R.schedule_from_doc(M.schedule_to_doc(sched))
    assert R.validate(rs, rg, R.compute_dependency_sets(rg), rc) == []
    assert R.trace_report(R.simulate(rs, rg, rc)) == M.trace_report(M.simulate(sched, g, cat))
    assert R.check_schedule(rg, R.compute_dependency_sets(rg), rc, rs, budget)[:2] == \
        M.check_schedule(g, M.compute_dependency_sets(g), cat, sched, budget)[:2]
