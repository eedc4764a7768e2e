"""Analytic roofline costs (ns) for catalog variants before the profiler has run.

The on-device profiler (profiler.py) replaces these with measured integer
nanoseconds; the analytic numbers keep the ILP well-posed on a CPU-only host
and are the "expected" side of the estimate-vs-measurement check
(B200_PROFILING.md: write the expected numbers down before measuring).
Units: integer nanoseconds, exact ints as units.py requires.
"""

from __future__ import annotations

import dataclasses

TC_FLOPS = 250e12      # sustained 3xTF32 conv throughput assumed before profiling
HBM_BPS = 6.0e12       # sustained HBM bandwidth for local ops
LAUNCH_NS = 4000       # per-kernel fixed cost


def _ns(flops=0.0, nbytes=0.0, launches=1) -> int:
    return max(1, int(max(flops / TC_FLOPS, nbytes / HBM_BPS) * 1e9 + launches * LAUNCH_NS))


def analytic_cost(net, op, pass_, name) -> int:
    n = op.numel
    if op.kind == "convT":  # same GEMM work as the conv it is the adjoint of
        x = net.op(op.deps[0])
        flops = 2.0 * x.numel * op.shape[3] * op.attrs["r"] * op.attrs["s"]
        return _ns(flops if pass_ == "fwd" else 2 * flops, 4.0 * (x.numel + n) * (1 if pass_ == "fwd" else 2),
                   launches=1 if pass_ == "fwd" else 3)
    if op.kind == "wgrad":  # split conv: the weight gradient (r x, r dy)
        if pass_ == "fwd":
            return 1
        conv = net.op(op.attrs["conv"])
        x = net.op(conv.deps[0])
        gate = 8.125 * conv.numel if conv.kind == "convrelu" else 0.0  # a split convrelu's dy mask gate
        return gate / HBM_BPS * 1e9 // 1 + _ns(2.0 * conv.numel * x.shape[3] * conv.attrs["r"] * conv.attrs["s"], 4.0 * (x.numel + conv.numel))
    if op.kind == "convrelu":  # the conv plus its in-place ReLU (fwd: r4 w4 + mask; bwd: mask gate of dy)
        relu = _ns(nbytes=8.125 * n)
        return analytic_cost(net, dataclasses.replace(op, kind="conv"), pass_, name) + (
            relu if pass_ == "fwd" or not op.attrs.get("split") else 0)
    if op.kind == "conv":
        x = net.op(op.deps[0])
        flops = 2.0 * n * x.shape[3] * op.attrs["r"] * op.attrs["s"]
        if pass_ == "fwd":
            return _ns(flops, 4.0 * (x.numel + n))
        if op.attrs.get("split"):  # dgrad only (+ bias gradient)
            bias = 4.0 * n if "bias" in op.params else 0.0
            return _ns(flops, 4.0 * (x.numel + n) + bias, launches=2)
        passes = 1 if net.op(op.deps[0]).kind == "input" else 2
        bias = 4.0 * n if "bias" in op.params else 0.0  # bias gradient: one more read of dy
        return _ns(passes * flops, 8.0 * (x.numel + n) + bias, launches=3)
    if op.kind == "concat":  # each input read once, output written once (bwd: slices of dy)
        return _ns(nbytes=8.0 * n, launches=len(op.attrs["inputs"]))
    if op.kind == "dropout":  # r4 w4, mask regenerated (never stored)
        return _ns(nbytes=8.0 * n)
    if op.kind == "fc":
        fi = net.fc_dims(op)[1]
        flops = 2.0 * n * fi
        return _ns(flops if pass_ == "fwd" else 2 * flops, launches=2 if pass_ == "fwd" else 4)
    if op.kind == "dwconv":  # direct, HBM-bound: fwd r x w y; bwd r dy (x2) r x w dx
        x = net.op(op.deps[0])
        return _ns(nbytes=4.0 * (x.numel + n) if pass_ == "fwd" else 4.0 * (2 * n + 2 * x.numel),
                   launches=1 if pass_ == "fwd" else 3)
    if op.kind in ("relu", "relu6"):
        if pass_ == "fwd":
            return _ns(nbytes=8.125 * n)
        return _ns(nbytes=(8.125 if name == "bwd-mask" else 12.0) * n)
    if op.kind == "bn":
        return _ns(nbytes=(12.0 if pass_ == "fwd" else 20.0) * n, launches=3)
    if op.kind == "bnaddrelu":  # stats r4 + apply r4 r4 w4; bwd reduce r4 r4 r4 + apply r4 r4 r4 w4 w4
        return _ns(nbytes=(16.0 if pass_ == "fwd" else 32.0) * n, launches=3)
    if op.kind in ("bnrelu", "bnrelu6"):  # stats r4 + apply r4 w4; bwd reduce r4 r4 + apply r4 r4 w4
        return _ns(nbytes=(12.0 if pass_ == "fwd" else 20.0) * n, launches=3)
    if op.kind == "addrelu":  # fwd r4 r4 w4; bwd r4 (gate) r4 (dz) w4 w4
        return _ns(nbytes=(12.0 if pass_ == "fwd" else (16.0 if name == "bwd-out" else 20.0)) * n)
    if op.kind == "add":
        return _ns(nbytes=(12.0 if pass_ == "fwd" else 16.0) * n, launches=1 if pass_ == "fwd" else 2)
    if op.kind == "maxpool":
        x = net.op(op.deps[0])
        return _ns(nbytes=4.0 * x.numel * (2.25 if pass_ == "fwd" else 2.0) + 5.0 * n)
    if op.kind == "avgpool":
        return _ns(nbytes=4.0 * net.op(op.deps[0]).numel)
    if op.kind == "input":
        return _ns(nbytes=8.0 * n) if pass_ == "fwd" else 1
    if op.kind == "xent":
        return _ns(nbytes=8.0 * net.op(op.deps[0]).numel, launches=2)
    raise ValueError(op.kind)
