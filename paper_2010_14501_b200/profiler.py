"""On-device profiler: measured catalog for the planner.

``profile(model, batch, device)`` times every (operator, variant) of a traced
network on the B200 with CUDA events -- the same sm_100a kernels and the same
argument shapes the executor launches -- and emits the catalog document the
reference planner consumes (costmodel.py:85-181): per node, ordered forward /
backward variants with integer ``workspace_bytes`` (the bytes the variant
takes from the arena, from the library's own workspace queries) and an
integer ``cost`` in nanoseconds (units.py:46-67 forbids floats).

Timing: after `warmup` launches, the median of `reps` event-timed groups of
`iters` launches; identical shapes are measured once.  Catalogs are frozen to
JSON for planning (costs vary run to run).
"""

from __future__ import annotations

import ctypes as C
import statistics

import torch

from . import _native

__all__ = ["profile", "profile_network", "profile_variant"]


class _Bench:
    def __init__(self, device, warmup=2, iters=5, reps=3):
        self.dev = torch.device(device)
        self.warmup, self.iters, self.reps = warmup, iters, reps
        self.lib = _native.lib().dll
        self.stream = torch.cuda.current_stream(self.dev)
        self.sp = C.c_void_p(self.stream.cuda_stream)

    def time_ns(self, fn) -> int:
        for _ in range(self.warmup):
            fn()
        samples = []
        for _ in range(self.reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
            for _ in range(self.iters):
                fn()
            b.record(self.stream)
            b.synchronize()
            samples.append(a.elapsed_time(b) * 1e6 / self.iters)
        return max(1, int(round(statistics.median(samples))))

    def buf(self, nbytes: int) -> torch.Tensor:
        t = torch.empty(max(int(nbytes), 16) // 4 + 1, dtype=torch.float32, device=self.dev)
        return t.normal_()

    def check(self, rc):
        if rc != 0:
            raise _native.NativeError(f"profiled kernel failed with code {rc}")


def _convT_calls(bx: _Bench, net, op, variant: str):
    """(fwd closure, bwd closure) of a transposed-conv variant (the conv kernels, roles swapped)."""
    lib, sp = bx.lib, bx.sp
    d = net.conv_desc(op)
    v = _native.CONV_VARIANTS[variant]
    xin = net.op(op.deps[0])
    x, y, dy, dx = bx.buf(xin.nbytes), bx.buf(op.nbytes), bx.buf(op.nbytes), bx.buf(xin.nbytes)
    w = bx.buf(4 * op.attrs["r"] * op.attrs["s"] * xin.shape[3] * op.shape[3])
    dw = bx.buf(w.numel() * 4)
    b = bx.buf(4 * op.shape[3]) if "bias" in op.params else None
    ws_f = lib.monet_convT_ws_bytes(v, 0, C.byref(d))
    ws_b = lib.monet_convT_ws_bytes(v, 3, C.byref(d))
    ws = bx.buf(max(ws_f, ws_b))
    if b is not None:
        db = bx.buf(4 * op.shape[3])
        rows = op.numel // op.shape[3]
        scratch = bx.buf(lib.monet_bn_scratch_bytes(rows, op.shape[3]))

    def fwd():
        bx.check(lib.monet_convT_fwd(v, C.byref(d), x.data_ptr(), w.data_ptr(), None if b is None else b.data_ptr(),
                                     y.data_ptr(), ws.data_ptr(), ws_f, sp))

    def bwd():
        bx.check(lib.monet_convT_bwd(v, C.byref(d), x.data_ptr(), w.data_ptr(), dy.data_ptr(),
                                     dx.data_ptr() if xin.kind != "input" else None, 0, dw.data_ptr(),
                                     ws.data_ptr(), ws_b, sp))
        if b is not None:
            bx.check(lib.monet_bias_grad(dy.data_ptr(), db.data_ptr(), rows, op.shape[3], 0, scratch.data_ptr(), sp))
    return fwd, bwd


def _local_calls(bx: _Bench, net, op):
    """{(pass, variant): closure} for the non-conv operators (engine.Runtime._bind)."""
    lib, sp = bx.lib, bx.sp
    out = {}
    n = op.numel
    kind = op.kind
    if kind == "input":
        y, src = bx.buf(op.nbytes), bx.buf(op.nbytes)
        out[("fwd", "load")] = lambda: bx.check(lib.monet_copy_async(y.data_ptr(), src.data_ptr(), op.nbytes, sp))
        return out
    xin = net.op(op.deps[0])
    x, y, dy, dx = bx.buf(xin.nbytes), bx.buf(op.nbytes), bx.buf(op.nbytes), bx.buf(xin.nbytes)
    if kind in ("relu", "bn", "conv"):
        raise ValueError(f"{kind} is profiled through monet_profile_variant")
    elif kind in ("bnrelu", "bnrelu6"):
        c = op.shape[-1]
        rows = n // c
        ch = [bx.buf(4 * c) for _ in range(8)]
        for t in ch[:4]:
            t.abs_().add_(0.5)
        scratch = bx.buf(lib.monet_bn_scratch_bytes(rows, c))
        g_, b_, m_, s_, rm, rv, dg, db = (t.data_ptr() for t in ch)
        six = kind == "bnrelu6"
        fwd_fn = lib.monet_bnrelu6_fwd_train if six else lib.monet_bnrelu_fwd_train
        bwd_fn = lib.monet_bnrelu6_bwd if six else lib.monet_bnrelu_bwd
        if op.id in net.stats_convs().values():  # statistics handed over by the conv
            st = _stats_buf(bx, rows, c)
            rep_fn = lib.monet_bnrelu6_fwd_replay if six else lib.monet_bnrelu_fwd_replay

            def fwd_stats():
                bx.check(lib.monet_bn_stats_finalize(st.data_ptr(), rows, c, C.c_float(1e-5), C.c_float(0.1), 1,
                                                      m_, s_, rm, rv, sp))
                bx.check(rep_fn(x.data_ptr(), y.data_ptr(), g_, b_, m_, s_, rows, c, sp))
            out[("fwd", kind)] = fwd_stats
        else:
            out[("fwd", kind)] = lambda: bx.check(fwd_fn(
                x.data_ptr(), y.data_ptr(), g_, b_, m_, s_, rm, rv, rows, c, C.c_float(1e-5), C.c_float(0.1), 1,
                scratch.data_ptr(), sp))
        out[("bwd", "bwd-in")] = lambda: bx.check(bwd_fn(
            x.data_ptr(), dy.data_ptr(), dx.data_ptr(), 0, g_, b_, m_, s_, dg, db, rows, c, scratch.data_ptr(), sp))
    elif kind == "bnaddrelu":
        c = op.shape[-1]
        rows = n // c
        ch = [bx.buf(4 * c) for _ in range(8)]
        for t in ch[:4]:
            t.abs_().add_(0.5)
        scratch = bx.buf(lib.monet_bn_scratch_bytes(rows, c))
        g_, b_, m_, s_, rm, rv, dg, db = (t.data_ptr() for t in ch)
        xx, kk, dk = bx.buf(op.nbytes), bx.buf(op.nbytes), bx.buf(op.nbytes)
        if op.id in net.stats_convs().values():  # statistics handed over by the conv
            st = _stats_buf(bx, rows, c)

            def fwd_stats():
                bx.check(lib.monet_bn_stats_finalize(st.data_ptr(), rows, c, C.c_float(1e-5), C.c_float(0.1), 1,
                                                      m_, s_, rm, rv, sp))
                bx.check(lib.monet_bnaddrelu_fwd_replay(xx.data_ptr(), kk.data_ptr(), y.data_ptr(), g_, b_, m_, s_,
                                                         rows, c, sp))
            out[("fwd", "bnaddrelu")] = fwd_stats
        else:
            out[("fwd", "bnaddrelu")] = lambda: bx.check(lib.monet_bnaddrelu_fwd_train(
                xx.data_ptr(), kk.data_ptr(), y.data_ptr(), g_, b_, m_, s_, rm, rv, rows, c, C.c_float(1e-5),
                C.c_float(0.1), 1, scratch.data_ptr(), sp))
        for name, src, from_out in (("bwd-out", y, 1), ("bwd-in", kk, 0)):
            out[("bwd", name)] = (lambda src=src, from_out=from_out: bx.check(lib.monet_bnaddrelu_bwd(
                xx.data_ptr(), src.data_ptr(), from_out, dy.data_ptr(), dx.data_ptr(), 0, dk.data_ptr(), 0, g_, b_,
                m_, s_, dg, db, rows, c, scratch.data_ptr(), sp)))
    elif kind == "add":
        x2 = bx.buf(op.nbytes)
        out[("fwd", "add")] = lambda: bx.check(lib.monet_add_fwd(x.data_ptr(), x2.data_ptr(), y.data_ptr(), n, sp))

        def add_bwd():
            for _ in range(2):
                bx.check(lib.monet_grad_pass(dy.data_ptr(), dx.data_ptr(), n, C.c_float(1.0), 0, sp))
        out[("bwd", "bwd")] = add_bwd
    elif kind == "addrelu":
        x2, dx2 = bx.buf(op.nbytes), bx.buf(op.nbytes)
        out[("fwd", "addrelu")] = lambda: bx.check(lib.monet_addrelu_fwd(x.data_ptr(), x2.data_ptr(), y.data_ptr(),
                                                                          n, sp))
        out[("bwd", "bwd-out")] = lambda: bx.check(lib.monet_addrelu_bwd_out(
            y.data_ptr(), dy.data_ptr(), dx.data_ptr(), 0, dx2.data_ptr(), 0, n, sp))
        out[("bwd", "bwd-in")] = lambda: bx.check(lib.monet_addrelu_bwd_in(
            x.data_ptr(), x2.data_ptr(), dy.data_ptr(), dx.data_ptr(), 0, dx2.data_ptr(), 0, n, sp))
    elif kind == "maxpool":
        d = net.pool_desc(op)
        idx = bx.buf(op.numel)
        out[("fwd", "maxpool")] = lambda: bx.check(lib.monet_maxpool_fwd(C.byref(d), x.data_ptr(), y.data_ptr(),
                                                                          idx.data_ptr(), sp))
        out[("bwd", "bwd-in")] = lambda: bx.check(lib.monet_maxpool_bwd(C.byref(d), None, x.data_ptr(),
                                                                         dy.data_ptr(), dx.data_ptr(), 0, sp))

        def bwd_idx():  # a valid index tensor first (window positions 0..R*S-1)
            bx.check(lib.monet_maxpool_bwd(C.byref(d), idx.data_ptr(), None, dy.data_ptr(), dx.data_ptr(), 0, sp))
        lib.monet_maxpool_fwd(C.byref(d), x.data_ptr(), y.data_ptr(), idx.data_ptr(), sp)
        out[("bwd", "bwd-idx")] = bwd_idx
    elif kind == "avgpool":
        nb, h, w, c = xin.shape
        out[("fwd", "avgpool")] = lambda: bx.check(lib.monet_avgpool_fwd(x.data_ptr(), y.data_ptr(), nb, h * w, c, sp))
        out[("bwd", "bwd")] = lambda: bx.check(lib.monet_avgpool_bwd(dy.data_ptr(), dx.data_ptr(), nb, h * w, c, 0,
                                                                       sp))
    elif kind == "concat":
        ins = [(bx.buf(net.op(j).nbytes), net.op(j).shape[3]) for j in op.attrs["inputs"]]
        pix, ct = n // op.shape[3], op.shape[3]

        def cat(backward):
            off = 0
            for t, cj in ins:
                if backward:
                    bx.check(lib.monet_channel_copy(dy.data_ptr(), ct, off, t.data_ptr(), cj, 0, cj, pix, 0, sp))
                else:
                    bx.check(lib.monet_channel_copy(t.data_ptr(), cj, 0, y.data_ptr(), ct, off, cj, pix, 0, sp))
                off += cj
        out[("fwd", "concat")] = lambda: cat(False)
        out[("bwd", "bwd")] = lambda: cat(True)
    elif kind == "relu6":
        mask = bx.buf((n + 31) // 32 * 4)
        out[("fwd", "relu6")] = lambda: bx.check(lib.monet_relu6_fwd(x.data_ptr(), y.data_ptr(), mask.data_ptr(), n,
                                                                      sp))
        out[("bwd", "bwd-in")] = lambda: bx.check(lib.monet_relu6_bwd_in(x.data_ptr(), dy.data_ptr(), dx.data_ptr(),
                                                                          n, 0, sp))
        out[("bwd", "bwd-out")] = lambda: bx.check(lib.monet_relu6_bwd_out(y.data_ptr(), dy.data_ptr(),
                                                                            dx.data_ptr(), n, 0, sp))
        out[("bwd", "bwd-mask")] = lambda: bx.check(lib.monet_relu_bwd_mask(mask.data_ptr(), dy.data_ptr(),
                                                                             dx.data_ptr(), n, 0, sp))
    elif kind == "dwconv":
        d = net.conv_desc(op)
        wgt, dw = bx.buf(4 * op.attrs["r"] * op.attrs["s"] * op.shape[3]), bx.buf(4 * op.attrs["r"] * op.attrs["s"] *
                                                                                   op.shape[3])
        wsb = lib.monet_dwconv_ws_bytes(C.byref(d))
        ws = bx.buf(wsb)
        need_dx = xin.kind != "input"
        out[("fwd", "direct")] = lambda: bx.check(lib.monet_dwconv_fwd(C.byref(d), x.data_ptr(), wgt.data_ptr(),
                                                                        y.data_ptr(), sp))

        def dw_bwd():
            if need_dx:
                bx.check(lib.monet_dwconv_dgrad(C.byref(d), dy.data_ptr(), wgt.data_ptr(), dx.data_ptr(), 0, sp))
            bx.check(lib.monet_dwconv_wgrad(C.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), ws.data_ptr(),
                                            wsb, sp))
        out[("bwd", "direct")] = dw_bwd
    elif kind == "dropout":
        seed = torch.zeros(1, dtype=torch.int64, device=bx.dev)
        pf = C.c_float(op.attrs["p"])
        out[("fwd", "dropout")] = lambda: bx.check(lib.monet_dropout_fwd(x.data_ptr(), y.data_ptr(), n, pf,
                                                                          seed.data_ptr(), op.id, sp))
        out[("bwd", "bwd-rng")] = lambda: bx.check(lib.monet_dropout_bwd(dy.data_ptr(), dx.data_ptr(), n, pf,
                                                                          seed.data_ptr(), op.id, 0, sp))
    elif kind == "fc":
        nb, fi = net.fc_dims(op)
        fo = op.shape[1]
        wgt, bias, dw, dbias = bx.buf(4 * fi * fo), bx.buf(4 * fo), bx.buf(4 * fi * fo), bx.buf(4 * fo)
        for name, v in (("gemm", 0), ("gemm-splitk", 1)):
            wf = lib.monet_linear_ws_bytes(v, 0, nb, fi, fo)
            wb = lib.monet_linear_ws_bytes(v, 3, nb, fi, fo)
            ws = bx.buf(max(wf, wb))
            out[("fwd", name)] = (lambda v=v, wf=wf, ws=ws: bx.check(lib.monet_linear_fwd(
                v, x.data_ptr(), wgt.data_ptr(), bias.data_ptr(), y.data_ptr(), nb, fi, fo, ws.data_ptr(), wf, sp)))
            out[("bwd", name)] = (lambda v=v, wb=wb, ws=ws: bx.check(lib.monet_linear_bwd(
                v, x.data_ptr(), wgt.data_ptr(), dy.data_ptr(), dx.data_ptr(), 0, dw.data_ptr(), dbias.data_ptr(),
                nb, fi, fo, ws.data_ptr(), wb, sp)))
    elif kind == "xent":  # (N, K) or per-pixel NHWC logits
        classes = xin.shape[-1]
        nb = xin.numel // classes
        labels = torch.randint(0, classes, (nb,), dtype=torch.int32, device=bx.dev)
        loss = bx.buf(4)
        scratch = bx.buf(lib.monet_xent_scratch_bytes(nb))
        one = torch.ones(1, device=bx.dev)
        out[("fwd", "xent")] = lambda: bx.check(lib.monet_xent_fwd(x.data_ptr(), labels.data_ptr(), loss.data_ptr(),
                                                                    nb, classes, scratch.data_ptr(), sp))
        out[("bwd", "bwd")] = lambda: bx.check(lib.monet_xent_bwd(x.data_ptr(), labels.data_ptr(), one.data_ptr(),
                                                                   dx.data_ptr(), nb, classes, 0, sp))
    else:
        raise ValueError(f"profiler: unsupported op kind {kind!r}")
    return out


def _stats_buf(bx, rows, c):
    """A conv -> BN statistics buffer (tile means / M2, the merge scratch after them) with
    positive values, as monet_conv_fwd_w16_stats would leave it."""
    t = (rows + 127) // 128
    nb = (t * 2 * c * 4 + 255) // 256 * 256 + ((t + 31) // 32 * 3 * c * 8 + 255) // 256 * 256
    buf = bx.buf(nb)
    buf.abs_().add_(0.5)
    return buf


def profile_variant(net, op, pss: str, variant: str, iters: int = 5, stream=None) -> tuple[int, int]:
    """(ns per launch, workspace bytes) of one variant through the C-ABI profiler entry
    point monet_profile_variant (csrc/profile.cu): conv fwd / bwd, ReLU, BN, fused BN+ReLU."""
    d = _native.ProfDesc()
    d.op = _native.PROF_OP["conv" if op.kind in ("wgrad", "convrelu") else op.kind]
    d.pass_ = _native.PASS["fwd"] if pss == "fwd" else _native.PASS["bwd"]
    if op.kind in ("conv", "convrelu", "wgrad"):
        conv = net.op(op.attrs["conv"]) if op.kind == "wgrad" else op
        d.conv = net.conv_desc(conv)
        d.conv_needs_dx = int(net.op(conv.deps[0]).kind != "input")
        if pss == "bwd" and op.kind == "wgrad":  # a split conv's weight-gradient node
            d.pass_ = _native.PASS["wgrad"]
        elif pss == "bwd" and op.attrs.get("split"):  # ... and its input-gradient node
            d.pass_ = _native.PASS["dgrad"]
        v = _native.CONV_VARIANTS[variant]
    else:
        d.c = op.shape[-1]
        d.rows = op.numel // d.c
        v = 0 if pss == "fwd" else _native.PROF_BWD[variant]
    # conv -> BN statistics handed over in the forward pass (Network.stats_convs): the BN's
    # training forward is the merge + apply.  The conv is timed without them -- its catalog cost
    # is what a recompute pays (recomputes never produce statistics); the statistics the first
    # forward produces are the same for every schedule, so they do not move the ILP's decisions
    sc = net.stats_convs()
    d.fused_stats = int(pss == "fwd" and op.id in sc.values())
    ns, ws = C.c_int64(0), C.c_size_t(0)
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    rc = _native.lib().dll.monet_profile_variant(C.byref(d), v, iters, C.byref(ns), C.byref(ws), C.c_void_p(stream))
    if rc != 0:
        raise _native.NativeError(f"monet_profile_variant({op.kind} {pss} {variant}) failed with code {rc}")
    conv = net.op(op.attrs["conv"]) if op.kind == "wgrad" else op
    if conv.kind == "convrelu" and (op.kind == "convrelu" or pss == "bwd") and not (
            op.kind == "convrelu" and pss == "bwd" and op.attrs.get("split")):
        # the fused ReLU: in-place forward (+ mask), or the in-place mask gate of dy that the
        # backward (unsplit) / the weight-gradient stage (split) runs first
        r = _native.ProfDesc()
        r.op, r.c = _native.PROF_OP["relu"], conv.shape[-1]
        r.rows = conv.numel // r.c
        r.pass_ = _native.PASS["fwd"] if pss == "fwd" else _native.PASS["bwd"]
        rns = C.c_int64(0)
        rc = _native.lib().dll.monet_profile_variant(C.byref(r), 0 if pss == "fwd" else _native.PROF_BWD["bwd-mask"],
                                                     iters, C.byref(rns), None, C.c_void_p(stream))
        if rc != 0:
            raise _native.NativeError(f"monet_profile_variant(relu of {op.kind}) failed with code {rc}")
        return int(ns.value) + int(rns.value), int(ws.value)
    return int(ns.value), int(ws.value)


_NATIVE_PROFILED = ("conv", "convrelu", "wgrad", "relu", "bn", "bnrelu")


def _signature(net, op):
    if op.kind == "wgrad":  # identical to its conv's shape
        return ("wgrad",) + _signature(net, net.op(op.attrs["conv"]))
    ins = tuple((net.op(j).kind == "input", net.op(j).shape) for j in op.deps)
    attrs = tuple(sorted((k, v) for k, v in op.attrs.items()
                         if isinstance(v, (int, float, str)) and k not in ("conv", "wgrad_node")))
    sc = net.stats_convs()
    return op.kind, ins, op.shape, attrs, op.id in sc or op.id in sc.values()


def profile_network(net, device="cuda:0", warmup=2, iters=5, reps=3, log=None) -> dict:
    """{(node, "fwd"|"bwd", variant name): ns} for every variant of every node."""
    bx = _Bench(device, warmup, iters, reps)
    cache: dict[tuple, dict] = {}
    costs: dict[tuple, int] = {}
    for op in net.ops:
        fv, bv = net.variants(op)
        sig = _signature(net, op)
        if sig not in cache:
            res = {}
            if op.kind == "wgrad":  # no forward work
                res[("fwd", "none")] = 1
                for name, ws, _ in bv:
                    ns, ws_k = profile_variant(net, op, "bwd", name, iters, bx.stream.cuda_stream)
                    assert ws_k == ws, (op.name, name, ws_k, ws)
                    res[("bwd", name)] = ns
            elif op.kind in _NATIVE_PROFILED:  # through the C-ABI profiler entry point
                for name, ws in fv:
                    ns, ws_k = profile_variant(net, op, "fwd", name, iters, bx.stream.cuda_stream)
                    assert ws_k == ws, (op.name, name, ws_k, ws)
                    res[("fwd", name)] = ns
                for name, ws, _ in bv:
                    ns, ws_k = profile_variant(net, op, "bwd", name, iters, bx.stream.cuda_stream)
                    assert op.kind not in ("conv", "convrelu") or ws_k == ws, (op.name, name, ws_k, ws)
                    res[("bwd", name)] = ns
            elif op.kind == "convT":
                for name, _ in fv:
                    f, _b = _convT_calls(bx, net, op, name)
                    res[("fwd", name)] = bx.time_ns(f)
                for name, _, _ in bv:
                    _f, b = _convT_calls(bx, net, op, name)
                    res[("bwd", name)] = bx.time_ns(b)
            else:
                calls = _local_calls(bx, net, op)
                for name, _ in fv:
                    res[("fwd", name)] = bx.time_ns(calls[("fwd", name)])
                for name, _, _ in bv:
                    key = ("bwd", name)
                    res[key] = bx.time_ns(calls[key]) if key in calls else 1  # e.g. the input's "none"
            cache[sig] = res
            torch.cuda.empty_cache()
            if log:
                log(f"{op.name or op.kind:28s} {op.kind:8s} {res}")
        for (pss, name), ns in cache[sig].items():
            costs[(op.id, pss, name)] = ns
    return costs


def profile(model, batch: int | None = None, device="cuda:0", image: int = 224, num_classes: int = 1000,
            **kw) -> dict:
    """Measured catalog document of `model` (a traced Network, a torchvision
    architecture name, or a torch module traced at [batch, 3, image, image])."""
    from .tracer import Network, build_network, trace_graph

    if isinstance(model, Network):
        net = model
    elif isinstance(model, str):
        net = build_network(model, batch, image, num_classes)
    else:
        net = trace_graph(model, torch.empty(batch, 3, image, image, device="meta"), num_classes)
    return net.catalog_doc(profile_network(net, device, **kw))
