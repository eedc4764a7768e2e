"""The on-device profiler (R3) through the C-ABI entry point monet_profile_variant.

profile() on a small traced network emits a catalog document that the planner loads
(load_catalog, costmodel.py:85-181) and that round-trips (catalog_to_doc); every cost is
a positive integer (units.py:61-62); every conv variant's workspace_bytes equals the
library's own query monet_conv_ws_bytes, which is also what monet_profile_variant reports.
"""
import ctypes as C

import pytest
import torch

import paper_2010_14501_b200 as M
from paper_2010_14501_b200 import _native
from paper_2010_14501_b200.profiler import profile, profile_variant
from paper_2010_14501_b200.tracer import build_network

pytestmark = pytest.mark.gpu


def test_profile_catalog(cuda):
    net = build_network("resnet18", 4, 32, num_classes=10, fuse=True)
    doc = profile(net, device=cuda, iters=2, reps=2)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(doc, g)
    assert M.catalog_to_doc(M.load_catalog(M.catalog_to_doc(cat), g)) == M.catalog_to_doc(cat)
    lib = _native.lib().dll
    n_conv = 0
    for op in net.ops:
        fv, bv = cat.forward[op.id], cat.backward.get(op.id, ())
        for v in list(fv) + list(bv):
            assert isinstance(v.cost.numerator, int) and v.cost.denominator == 1 and v.cost > 0, (op.name, v)
        if op.kind != "conv":
            continue
        n_conv += 1
        d = net.conv_desc(op)
        for v in fv:
            assert v.workspace_bytes == lib.monet_conv_ws_bytes(_native.CONV_VARIANTS[v.name], 0, C.byref(d))
        for v in bv:
            assert v.workspace_bytes == lib.monet_conv_ws_bytes(_native.CONV_VARIANTS[v.name], 3, C.byref(d))
    assert n_conv > 10


def test_profile_variant_entry_point(cuda):
    net = build_network("resnet18", 4, 32, num_classes=10)
    conv = next(op for op in net.ops if op.kind == "conv" and net.op(op.deps[0]).kind != "input")
    d = net.conv_desc(conv)
    lib = _native.lib().dll
    for name, v in (("implicit", 0), ("splitk", 1)):
        for pss, code in (("fwd", 0), ("bwd", 3)):
            ns, ws = profile_variant(net, conv, pss, name)
            assert ns > 0 and ws == lib.monet_conv_ws_bytes(v, code, C.byref(d))
    bn = next(op for op in net.ops if op.kind == "bn")
    for pss, name in (("fwd", "bn"), ("bwd", "bwd-in"), ("bwd", "bwd-out")):
        ns, ws = profile_variant(net, bn, pss, name)
        assert ns > 0 and ws == 0
    # invalid descriptors are rejected with an error code, not a crash
    bad = _native.ProfDesc()
    bad.op, bad.pass_ = 99, 0
    ns, wsb = C.c_int64(0), C.c_size_t(0)
    assert lib.monet_profile_variant(C.byref(bad), 0, 1, C.byref(ns), C.byref(wsb),
                                     C.c_void_p(torch.cuda.current_stream().cuda_stream)) < 0
