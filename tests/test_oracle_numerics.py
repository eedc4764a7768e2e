"""Pin the CPU oracle executor's numerics against plain torch autograd.

The reference package has no numeric implementation ("parity unpinned",
SURVEY.md §8c), so the oracle is pinned here instead: replaying ANY valid
schedule (store-everything or with recomputation and memory-efficient
backward variants) must give the same loss, updated weights and BN running
statistics as one ordinary autograd + SGD step of the same torchvision model.
"""
import numpy as np
import pytest
import torch
import torchvision

import paper_2010_14501_b200 as M
from oracle.bitmask import pack_sign_mask, unpack_sign_mask
from oracle.cpu_executor import CpuState, params_nhwc, run_step
from paper_2010_14501_b200.tracer import trace_graph

TOL = 1e-9  # both sides in float64: pins the algorithm, not fp32 rounding (small-batch BN is ill-conditioned)


def _rel(a, b):
    return (a.double() - b.double()).abs().max().item() / max(b.double().abs().max().item(), 1e-30)


def _setup(batch=2, hw=32, arch="resnet18", fuse=False):
    torch.manual_seed(0)
    model = getattr(torchvision.models, arch)(num_classes=10)
    net = trace_graph(model, torch.empty(batch, 3, hw, hw, device="meta"), 10, fuse=fuse)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    gen = torch.Generator().manual_seed(1)
    x = torch.randn(batch, 3, hw, hw, generator=gen)
    y = torch.randint(0, 10, (batch,), generator=gen)
    return model, net, g, cat, x, y


def _autograd_step(model, x, y):
    model.double().train()
    x = x.double()
    opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)
    _OPT[id(model)] = opt
    loss = torch.nn.functional.cross_entropy(model(x), y)
    opt.zero_grad()
    loss.backward()
    opt.step()
    return loss.item()


def _schedules(g, cat):
    se = M.store_everything_schedule(g, cat)
    sets = M.compute_dependency_sets(g)
    peak = M.simulate(se, g, cat).peak_memory
    act = peak - g.params_bytes
    out = [("store_everything", se)]
    for f in (0.6, 0.45):
        h = M.checkpoint_heuristic(g, sets, cat, g.params_bytes + int(f * act))
        if h is None:
            continue
        try:
            M.simulate(h, g, cat)
        except M.SimulationError:
            continue
        out.append((f"heuristic-{f}", h))
    return out


@pytest.mark.parametrize("arch,fuse", [("resnet18", False), ("resnet18", True)])
def test_oracle_replay_equals_autograd(arch, fuse):
    model, net, g, cat, x, y = _setup(arch=arch, fuse=fuse)
    assert fuse == any(op.kind == "bnrelu" for op in net.ops)
    ref_loss = _autograd_step(model, x, y)
    ref = {n: p.detach() for n, p in model.named_parameters()}
    ref_bn = {n: b for n, b in model.named_buffers() if "running" in n}
    scheds = _schedules(g, cat)
    assert any(n != "store_everything" for n, _ in scheds), "no recompute schedule to test"
    for name, sched in scheds:
        st = CpuState(net, dtype=torch.float64)
        loss = run_step(st, M.schedule_to_doc(sched), x.double(), y)
        assert abs(loss - ref_loss) <= TOL * abs(ref_loss), name
        got = params_nhwc(st)
        for op in net.ops:
            for pname in op.params:
                want = ref[f"{op.name.split('+')[0]}.{pname}"]
                have = got[(op.id, pname)]
                if op.kind == "conv":
                    have = have[..., : want.shape[1]].permute(0, 3, 1, 2)
                assert _rel(have, want) < TOL, (name, op.name, pname)
            if op.kind in ("bn", "bnrelu", "bnaddrelu"):
                rm, rv = st.running[op.id]
                base = op.name.split('+')[0]
                assert _rel(rm, ref_bn[f"{base}.running_mean"]) < TOL
                assert _rel(rv, ref_bn[f"{base}.running_var"]) < TOL


def test_fusion_pass():
    _, net, g, cat, _, _ = _setup(fuse=True)
    _, plain, _, _, _, _ = _setup(fuse=False)

    def fusable(op):  # a BN / add whose only reader is a ReLU of it
        readers = [o for o in plain.ops if op.id in o.deps]
        return op.kind in ("bn", "add") and len(readers) == 1 and readers[0].kind == "relu"
    n_bn = sum(1 for op in plain.ops if op.kind == "bn" and fusable(op))
    n_add = sum(1 for op in plain.ops if op.kind == "add" and fusable(op))
    # every add+ReLU join then absorbs one BN input whose only reader it is (the block's last BN)
    n_join_bn = sum(op.kind == "bnaddrelu" for op in net.ops)
    assert sum(op.kind == "bnrelu" for op in net.ops) == n_bn > 0
    assert sum(op.kind in ("addrelu", "bnaddrelu") for op in net.ops) == n_add > 0
    assert n_join_bn == n_add  # ResNet: every join has such a BN
    assert net.n == plain.n - n_bn - n_add - n_join_bn
    for op in net.ops:
        if op.kind == "bnrelu":  # backward reads the BN input only
            (v,) = cat.bwd(op.id)
            assert v.name == "bwd-in" and set(v.deps) == set(op.deps)
        elif op.kind == "addrelu":  # gate from the output or from both inputs
            assert {v.name: set(v.deps) for v in cat.bwd(op.id)} == {"bwd-out": {op.id}, "bwd-in": set(op.deps)}
        elif op.kind == "bnaddrelu":  # BN backward from x; gate from z, or from x and the skip
            assert {v.name: set(v.deps) for v in cat.bwd(op.id)} == {"bwd-out": {op.attrs["x"], op.id},
                                                                      "bwd-in": set(op.deps)}
            assert net.op(op.attrs["skip"]).kind in ("bnrelu", "addrelu", "bnaddrelu", "bn", "maxpool")
    assert g.params_bytes == plain.params_bytes()


def test_bitmask_roundtrip():
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 1000):
        x = rng.standard_normal(n).astype(np.float32)
        x[::5] = 0
        w = pack_sign_mask(x)
        assert w.dtype == np.uint32 and len(w) == (n + 31) // 32
        assert np.array_equal(unpack_sign_mask(w, n), x > 0)
        # bit b of word k <-> element 32k+b
        for e in range(n):
            assert ((w[e // 32] >> (e % 32)) & 1) == (x[e] > 0)


def _torch_layout(net, op, pname, have, want):
    """Engine-layout parameter -> torch layout (conv KRSC, fc over an NHWC-flattened input)."""
    if op.kind in ("conv", "convrelu") and pname == "weight":
        return have[..., : want.shape[1]].permute(0, 3, 1, 2)
    if op.kind == "fc" and pname == "weight" and len(net.op(op.deps[0]).shape) == 4:
        _, h, w, c = net.op(op.deps[0]).shape
        return have.view(-1, h, w, c).permute(0, 3, 1, 2).reshape(have.shape[0], -1)
    return have


@pytest.mark.parametrize("fuse,split", [(False, False), (True, False), (True, True)])
def test_oracle_vgg_style_equals_autograd(fuse, split):
    """Conv bias, identity adaptive pool, flatten-to-fc and dropout (hash keep-mask):
    two consecutive oracle steps under recompute schedules equal autograd + SGD --
    also with conv+ReLU fused ("convrelu": in-place ReLU and 1-bit mask, dy gated in
    place) and with the conv backward split into dgrad / wgrad nodes."""
    from nets import SmallVGG, use_hash_dropout

    torch.manual_seed(0)
    model = SmallVGG()
    net = trace_graph(model, torch.empty(2, 3, 32, 32, device="meta"), 10, fuse, split)
    kinds = {op.kind for op in net.ops}
    conv = "convrelu" if fuse else "conv"
    assert {conv, "dropout", "fc", "maxpool"} <= kinds and "avgpool" not in kinds
    assert ("wgrad" in kinds) == split
    assert fuse == all(net.op(op.deps[0]).kind != "conv" for op in net.ops if op.kind == "relu")
    assert all("bias" in op.params for op in net.ops if op.kind == conv)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    gen = torch.Generator().manual_seed(1)
    x = torch.randn(2, 3, 32, 32, generator=gen)
    y = torch.randint(0, 10, (2,), generator=gen)
    scheds = _schedules(g, cat) + _planned(net, g, cat)
    assert any(n != "store_everything" for n, _ in scheds), "no recompute schedule to test"
    for name, sched in scheds:
        ref_model = SmallVGG()
        ref_model.load_state_dict(model.state_dict())
        st = CpuState(net, dtype=torch.float64)
        for step in range(2):  # the second step draws a new mask (seed advanced)
            use_hash_dropout(ref_model, net, seed=step)
            ref_loss = _autograd_step(ref_model, x, y) if step == 0 else _autograd_step_keep(ref_model, x, y)
            loss = run_step(st, M.schedule_to_doc(sched), x.double(), y)
            assert abs(loss - ref_loss) <= TOL * abs(ref_loss), (name, step)
        ref = {n: p.detach() for n, p in ref_model.named_parameters()}
        got = params_nhwc(st)
        for op in net.ops:
            for pname in op.params:
                want = ref[f"{op.name.split('+')[0]}.{pname}"]
                have = _torch_layout(net, op, pname, got[(op.id, pname)], want)
                assert _rel(have, want) < TOL, (name, op.name, pname)


_OPT = {}


def _planned(net, g, cat, fracs=(0.7, 0.6)):
    """Host-planner recompute schedules at fractions of the store-everything activations."""
    from paper_2010_14501_b200.planner import plan_schedule

    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    out = []
    for f in fracs:
        s, _ = plan_schedule(g, cat, g.params_bytes + int(f * act), kinds=net.storable_kinds())
        if s is not None and any(st.recompute for st in s.stages):
            out.append((f"planned-{f}", s))
    return out


def _autograd_step_keep(model, x, y):
    """Second SGD step with the optimizer (momentum buffers) of the first."""
    opt = _OPT[id(model)]
    loss = torch.nn.functional.cross_entropy(model(x.double()), y)
    opt.zero_grad()
    loss.backward()
    opt.step()
    return loss.item()


@pytest.mark.parametrize("fuse", [False, True])
def test_oracle_mobilenet_v2_equals_autograd(fuse):
    """Depthwise convs, ReLU6 (mask / output / input backward), residual adds without
    ReLU, functional adaptive pool and dropout: torchvision MobileNet-V2 (width 0.25) at 64 x 64 (the last BNs then see 8 values per channel, not 2)."""
    from nets import use_hash_dropout

    torch.manual_seed(0)
    model = torchvision.models.mobilenet_v2(num_classes=10, width_mult=0.25)
    net = trace_graph(model, torch.empty(2, 3, 64, 64, device="meta"), 10, fuse=fuse)
    kinds = {op.kind for op in net.ops}
    assert {"dwconv", "add", "avgpool", "dropout"} <= kinds
    assert ("bnrelu6" in kinds) == fuse and ("relu6" in kinds) != fuse
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    gen = torch.Generator().manual_seed(1)
    x = torch.randn(2, 3, 64, 64, generator=gen)
    y = torch.randint(0, 10, (2,), generator=gen)
    scheds = [("store_everything", M.store_everything_schedule(g, cat))] + _planned(net, g, cat, fracs=(0.6,))
    assert len(scheds) > 1, "no recompute schedule to test"
    for name, sched in scheds:
        ref_model = torchvision.models.mobilenet_v2(num_classes=10, width_mult=0.25)
        ref_model.load_state_dict(model.state_dict())
        use_hash_dropout(ref_model, net, seed=0)
        ref_loss = _autograd_step(ref_model, x, y)
        st = CpuState(net, dtype=torch.float64)
        loss = run_step(st, M.schedule_to_doc(sched), x.double(), y)
        assert abs(loss - ref_loss) <= TOL * abs(ref_loss), name
        ref = {n: p.detach() for n, p in ref_model.named_parameters()}
        ref_bn = {n: b for n, b in ref_model.named_buffers() if "running" in n}
        got = params_nhwc(st)
        for op in net.ops:
            for pname in op.params:
                want = ref[f"{op.name.removesuffix('+relu6')}.{pname}"]
                have = got[(op.id, pname)]
                if op.kind == "dwconv":
                    have = have.permute(2, 0, 1).unsqueeze(1)
                else:
                    have = _torch_layout(net, op, pname, have, want)
                # floor: BN biases feeding another BN (through a 1x1 conv) have a zero gradient;
                # both sides then hold ~1e-16 rounding noise
                err = (have.double() - want.double()).abs().max().item()
                assert err <= TOL * max(want.double().abs().max().item(), 1e-3), (name, op.name, pname)
            if op.kind in ("bn", "bnrelu6"):
                rm, rv = st.running[op.id]
                base = op.name.removesuffix("+relu6")
                for have, want in ((rm, ref_bn[f"{base}.running_mean"]), (rv, ref_bn[f"{base}.running_var"])):
                    err = (have.double() - want.double()).abs().max().item()
                    assert err <= TOL * max(want.double().abs().max().item(), 1e-3), (name, op.name)


@pytest.mark.parametrize("fuse", [False, True])
def test_oracle_googlenet_equals_autograd(fuse):
    """Inception concats (backward = channel slices), ceil-mode max pools (stride 1 and 2),
    functional ReLU, BN eps 1e-3 and dropout: torchvision GoogLeNet at 64 x 64."""
    from nets import use_hash_dropout

    torch.manual_seed(0)
    mk = lambda: torchvision.models.googlenet(num_classes=10, aux_logits=False, init_weights=True)  # noqa: E731
    model = mk()
    net = trace_graph(model, torch.empty(2, 3, 64, 64, device="meta"), 10, fuse=fuse)
    kinds = {op.kind for op in net.ops}
    assert {"concat", "maxpool", "dropout"} <= kinds
    assert any(op.attrs.get("ceil") for op in net.ops if op.kind == "maxpool")
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    gen = torch.Generator().manual_seed(1)
    x = torch.randn(2, 3, 64, 64, generator=gen)
    y = torch.randint(0, 10, (2,), generator=gen)
    scheds = [("store_everything", M.store_everything_schedule(g, cat))] + _planned(net, g, cat, fracs=(0.6,))
    assert len(scheds) > 1, "no recompute schedule to test"
    for name, sched in scheds:
        ref_model = mk()
        ref_model.load_state_dict(model.state_dict())
        use_hash_dropout(ref_model, net, seed=0)
        ref_loss = _autograd_step(ref_model, x, y)
        st = CpuState(net, dtype=torch.float64)
        loss = run_step(st, M.schedule_to_doc(sched), x.double(), y)
        assert abs(loss - ref_loss) <= TOL * abs(ref_loss), name
        ref = {n: p.detach() for n, p in ref_model.named_parameters()}
        got = params_nhwc(st)
        for op in net.ops:
            for pname in op.params:
                want = ref[f"{op.name.split('+')[0]}.{pname}"]
                have = _torch_layout(net, op, pname, got[(op.id, pname)], want)
                err = (have.double() - want.double()).abs().max().item()
                assert err <= TOL * max(want.double().abs().max().item(), 1e-3), (name, op.name, pname)


def test_oracle_unet_equals_autograd():
    """UNet: transposed convs (with bias), decoder concats and the per-pixel cross-entropy."""
    from paper_2010_14501_b200.tracer import UNet

    torch.manual_seed(0)
    model = UNet(num_classes=4, width=8)
    net = trace_graph(model, torch.empty(2, 3, 32, 48, device="meta"), 4)
    assert {"convT", "concat", "xent"} <= {op.kind for op in net.ops}
    assert net.label_count() == 2 * 32 * 48
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    gen = torch.Generator().manual_seed(1)
    x = torch.randn(2, 3, 32, 48, generator=gen)
    y = torch.randint(0, 4, (2, 32, 48), generator=gen)
    scheds = [("store_everything", M.store_everything_schedule(g, cat))] + _planned(net, g, cat)
    assert len(scheds) > 1, "no recompute schedule to test"
    for name, sched in scheds:
        ref_model = UNet(num_classes=4, width=8)
        ref_model.load_state_dict(model.state_dict())
        ref_loss = _autograd_step(ref_model, x, y)
        st = CpuState(net, dtype=torch.float64)
        loss = run_step(st, M.schedule_to_doc(sched), x.double(), y)
        assert abs(loss - ref_loss) <= TOL * abs(ref_loss), name
        ref = {n: p.detach() for n, p in ref_model.named_parameters()}
        got = params_nhwc(st)
        for op in net.ops:
            for pname in op.params:
                want = ref[f"{op.name.split('+')[0]}.{pname}"]
                have = got[(op.id, pname)]
                if op.kind == "conv" and pname == "weight":
                    have = have[..., : want.shape[1]].permute(0, 3, 1, 2)
                elif op.kind == "convT" and pname == "weight":
                    have = have.permute(0, 3, 1, 2)
                err = (have.double() - want.double()).abs().max().item()
                assert err <= TOL * max(want.double().abs().max().item(), 1e-3), (name, op.name, pname)
