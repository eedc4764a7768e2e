"""GPU-vs-oracle parity helpers (test infrastructure; imported by GPU tests and smoke()).

capture(): run one scheduled step on the GPU, copying every forward output
(NCHW, fp32, CPU) as it is produced, and verifying that every recompute
reproduces the forward value bit for bit.
"""
import torch


def _view(rt, ptr, shape):
    base = rt.arena.data_ptr()
    n = 1
    for d in shape:
        n *= d
    return rt.arena[ptr - base: ptr - base + 4 * n].view(torch.float32).view(shape)


def capture(rt, plan):
    net = rt.net
    acts, mismatched = {}, []

    def after(i):
        s = plan.steps[i]
        if s.kind == "backward":
            return
        op = net.op(s.node)
        if op.kind in ("xent", "wgrad"):  # the loss scalar; split-conv anchors hold no tensor
            return
        v = _view(rt, plan.step_ptrs[i][("a", s.node)], op.shape).clone()
        if s.kind == "forward":
            acts[s.node] = v
        elif not torch.equal(acts[s.node], v):
            mismatched.append(s.node)

    rt.run(plan, after_step=after)
    torch.cuda.synchronize()
    nchw = {k: (v.permute(0, 3, 1, 2).contiguous() if v.dim() == 4 else v).cpu() for k, v in acts.items()}
    return nchw, mismatched


def gpu_stats(rt):
    """BN node id -> (saved mean, saved invstd) of the GPU's last forward (CPU fp32 copies),
    for run_step(..., forced_stats=...)."""
    return {i: (v[0].detach().cpu().clone(), v[1].detach().cpu().clone()) for i, v in rt.bn.items()}


def rel(a, b):
    a, b = a.detach().double().cpu(), b.detach().double().cpu()
    return (a - b).abs().max().item() / max(b.abs().max().item(), 1e-30)


def grads_nhwc(state):
    """Parameter gradients of the oracle in the engine layout (conv weights KRSC)."""
    out = {}
    for (nid, name), g in state.grads.items():
        kind = state.net.op(nid).kind
        if kind in ("conv", "convrelu", "convT") and name == "weight":
            g = g.permute(0, 2, 3, 1).contiguous()
        elif kind == "dwconv" and name == "weight":
            g = g.squeeze(1).permute(1, 2, 0).contiguous()
        out[(nid, name)] = g
    return out


def step_parity(rt, st, floor=1e-2):
    """Per-tensor errors of one GPU training step against the oracle.

    ``st``: the oracle state after ``run_step(..., forced=acts, forced_stats=...)``
    (the GPU's activations and batch statistics fed in; its BN running statistics
    are updated from the GPU's own BN inputs, so they are the exact reference for
    the GPU's).  Each error is
    max|gpu - cpu| / max(max|cpu|, floor * G), G = the largest magnitude of that
    kind of tensor over the whole model: tensors whose exact value is ~0 (e.g.
    the bias gradient of a BN whose output reaches another BN through a conv:
    the second BN's input gradient sums to zero per channel, so the first bias
    gradient is exactly 0) are judged against 1 % of the model's scale instead
    of their own rounding noise.

    Returns {"grad": [(err, name)], "param": [...], "running": [...]}.
    """
    from .cpu_executor import params_nhwc

    net = rt.net
    out = {"grad": [], "param": [], "running": []}

    def errs(pairs, kind):
        pairs = list(pairs)
        scale = max((ref.abs().max().item() for _, _, ref in pairs), default=0.0)
        for name, got, ref in pairs:
            ref64 = ref.detach().double().cpu()
            got64 = got.detach().double().cpu().view(ref64.shape)
            den = max(ref64.abs().max().item(), floor * scale, 1e-30)
            out[kind].append(((got64 - ref64).abs().max().item() / den, name))

    g = grads_nhwc(st)
    errs(((f"{net.op(n).name}.{p}", rt.gview[(n, p)], g[(n, p)]) for (n, p) in g), "grad")
    pv = params_nhwc(st)
    errs(((f"{net.op(n).name}.{p}", rt.pview[(n, p)], v) for (n, p), v in pv.items()), "param")
    pairs = []
    for op in net.ops:
        if op.id in rt.bn:
            rm, rv = st.running[op.id]
            pairs += [(f"{op.name}.running_mean", rt.bn[op.id][2], rm),
                      (f"{op.name}.running_var", rt.bn[op.id][3], rv)]
    errs(pairs, "running")
    return out


def worst(report):
    """(kind, err, name) of the largest error in a step_parity report."""
    return max(((k, e, n) for k, v in report.items() for e, n in v), key=lambda t: t[1], default=("", 0.0, ""))
