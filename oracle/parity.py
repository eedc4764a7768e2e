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
        if op.kind == "xent":
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


def rel(a, b):
    a, b = a.detach().double().cpu(), b.detach().double().cpu()
    return (a - b).abs().max().item() / max(b.abs().max().item(), 1e-30)
