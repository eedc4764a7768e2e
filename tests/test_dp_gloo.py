"""Data-parallel gradient exchange on CPU: world size 2 over gloo.

Each rank runs the CPU oracle's training step on its own shard (per-shard
BN statistics, as on the GPUs), copies the parameter gradients into a flat
buffer laid out like the engine's fixed region, and drives the product's
dp.DataParallel exactly as the executor does: `bucket_ready(node)` in
backward-stage order (descending node ids), then `finish()`.  The reduced
buffer must equal the sum of both shards' gradients (the "DP oracle":
per-shard restatement + sum; SGD then scales by 1/world).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.cpu_executor import CpuState, run_step
import paper_2010_14501_b200 as M
from paper_2010_14501_b200.dp import DataParallel, plan_buckets
from paper_2010_14501_b200.tracer import build_network

WORLD = 2
SHARD = 2


class _StubRuntime:
    """The slice of engine.Runtime that DataParallel uses: net, flat grads, grad_scale."""

    def __init__(self, net, grads):
        self.net, self.grads, self.grad_scale, self.comm = net, grads, 1.0, None


def _shard_grads(net, sched_doc, rank):
    gen = torch.Generator().manual_seed(100 + rank)
    x = torch.randn(SHARD, 3, 32, 32, generator=gen)
    y = torch.randint(0, 10, (SHARD,), generator=gen)
    st = CpuState(net, lr=0.0)  # lr 0: the step leaves the parameters, we want the gradients
    run_step(st, sched_doc, x, y)
    flat = []
    for nid, name, _ in net.param_items():
        flat.append(st.grads[(nid, name)].reshape(-1))
    return torch.cat(flat).float()


def _worker(rank, port, sched_doc, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        net = build_network("resnet18", SHARD, 32, num_classes=10, fuse=True)
        rt = _StubRuntime(net, _shard_grads(net, sched_doc, rank).clone())
        dp = DataParallel(rt, bucket_bytes=4 << 20)
        assert rt.grad_scale == 1.0 / WORLD and rt.comm is dp
        launched = []
        for node in range(net.n, 0, -1):  # the executor's backward stage order
            before = len(dp.works)
            dp.bucket_ready(node)
            launched += [node] * (len(dp.works) - before)
        dp.finish()
        out[rank] = (rt.grads.clone(), launched)
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
def test_bucketed_allreduce_matches_dp_oracle():
    net = build_network("resnet18", SHARD, 32, num_classes=10, fuse=True)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    sched = M.checkpoint_heuristic(g, M.compute_dependency_sets(g), cat, g.params_bytes + int(0.7 * act))
    if sched is None:
        sched = M.store_everything_schedule(g, cat)
    doc = M.schedule_to_doc(sched)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(_port(), doc, out), nprocs=WORLD, join=True)
        results = dict(out)
    want = _shard_grads(net, doc, 0) + _shard_grads(net, doc, 1)
    for rank in range(WORLD):
        got, launched = results[rank]
        assert torch.allclose(got, want, rtol=1e-6, atol=1e-7), rank
    buckets = plan_buckets(net, 4 << 20)
    assert sorted(results[0][1]) == sorted(n for _, _, n in buckets)  # every bucket launched exactly once
    assert results[0][1] == sorted(results[0][1], reverse=True)        # in backward order


def test_bucket_plan_covers_buffer():
    net = build_network("resnet50", 2, 64)
    total = sum(t.numel() for _, _, t in net.param_items())
    b = plan_buckets(net)
    assert b[0][1] == total and b[-1][0] == 0
    for (a0, _, n0), (_, b1, n1) in zip(b, b[1:]):
        assert b1 == a0 and n1 < n0  # contiguous, highest nodes first
    assert all((e - s) * 4 >= 25 << 20 for s, e, _ in b[:-1])
