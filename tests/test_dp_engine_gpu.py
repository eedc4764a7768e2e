"""Batch-sharded data parallelism on the real engine, on one B200.

* Two processes share the GPU, each running engine.Runtime + dp.DataParallel on its
  half of the batch (per-shard BN statistics), gradients all-reduced over gloo (CUDA
  tensors; NCCL refuses two ranks on one device).  The reduced gradient buffer must equal
  the sum of the per-shard oracle gradients (the CPU oracle fed each shard's GPU
  activations and statistics -- the DP oracle: per-shard restatement + sum), and the
  SGD-updated weights must equal the oracle's update with the averaged gradient.
* The native communicator (csrc/comm.cu: NCCL all-reduce forked per bucket onto a comm
  stream, joined before SGD) at world size 1: the whole step, bucket all-reduces
  included, is captured into one CUDA graph and replays bit-identically to the
  single-GPU step without a communicator.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
WORLD = 2
SHARD = 4
REL = 1e-4


def _net_and_schedule():
    import paper_2010_14501_b200 as M
    from paper_2010_14501_b200.planner import plan_schedule
    from paper_2010_14501_b200.tracer import build_network

    net = build_network("resnet18", SHARD, 32, num_classes=10, fuse=True)
    g = M.load_graph(net.graph_doc())
    cat = M.load_catalog(net.catalog_doc(), g)
    act = M.simulate(M.store_everything_schedule(g, cat), g, cat).peak_memory - g.params_bytes
    sched, _ = plan_schedule(g, cat, g.params_bytes + int(0.5 * act), kinds=net.storable_kinds())
    return net, g, cat, sched


def _shard(rank):
    gen = torch.Generator().manual_seed(100 + rank)
    return torch.randn(SHARD, 3, 32, 32, generator=gen), torch.randint(0, 10, (SHARD,), generator=gen)


def _worker(rank, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2010_14501_b200 as M
        from oracle.cpu_executor import CpuState, run_step
        from oracle.parity import capture, grads_nhwc, gpu_stats
        from paper_2010_14501_b200.dp import DataParallel
        from paper_2010_14501_b200.engine import Runtime

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        net, g, cat, sched = _net_and_schedule()
        rt = Runtime(net, device=dev)
        dp = DataParallel(rt, bucket_bytes=2 << 20, backend="torch")
        assert len(dp.buckets) > 1 and rt.grad_scale == 1.0 / WORLD
        x, y = _shard(rank)
        rt.set_batch(x.to(dev), y.to(dev))
        p0 = rt.params.detach().cpu().clone()
        plan = rt.plan(sched, g, cat)
        acts, mism = capture(rt, plan)  # one DP step: backward, bucket all-reduces, SGD
        assert not mism
        st = CpuState(net, dtype=torch.float64, lr=0.0)  # the shard's exact gradients
        run_step(st, M.schedule_to_doc(sched), x, y, forced=acts, forced_stats=gpu_stats(rt))
        order = [(nid, name) for nid, name, _ in net.param_items()]
        og = grads_nhwc(st)
        out[rank] = {"grads": rt.grads.detach().cpu().clone(), "params": rt.params.detach().cpu().clone(),
                     "p0": p0, "oracle": torch.cat([og[k].reshape(-1) for k in order]), "loss": rt.loss_value()}
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(900)
def test_dp_world2_engine_matches_dp_oracle(cuda):
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(_port(), out), nprocs=WORLD, join=True)
        res = dict(out)
    want = res[0]["oracle"] + res[1]["oracle"]   # DP oracle: the sum of the shard gradients
    for rank in range(WORLD):
        got = res[rank]["grads"].double()
        err = (got - want).abs().max().item() / want.abs().max().item()
        assert err <= REL, (rank, err)
    assert torch.equal(res[0]["grads"], res[1]["grads"])           # every rank holds the same sum
    assert torch.equal(res[0]["params"], res[1]["params"])         # ... and takes the same SGD step
    assert res[0]["loss"] != res[1]["loss"]                        # on different shards
    # SGD (lr 0.1, momentum 0.9, fresh momentum): w1 = w0 - lr * (sum / world)
    upd = res[0]["p0"].double() - 0.1 * want / WORLD
    err = (res[0]["params"].double() - upd).abs().max().item() / upd.abs().max().item()
    assert err <= REL, err


@pytest.mark.timeout(600)
def test_native_comm_graph_captured_world1(cuda):
    from paper_2010_14501_b200.dp import DataParallel
    from paper_2010_14501_b200.engine import Runtime

    net, g, cat, sched = _net_and_schedule()
    x, y = _shard(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        results = []
        for with_comm in (False, True):
            rt = Runtime(net, device=cuda)
            dp = DataParallel(rt, bucket_bytes=2 << 20, backend="native") if with_comm else None
            if dp is not None:
                assert dp.capturable and len(dp.buckets) > 1
            rt.set_batch(x.to(cuda), y.to(cuda))
            plan = rt.plan(sched, g, cat)
            rt.capture(plan)                       # first run + capture (two steps)
            for _ in range(3):
                rt.train_step(plan)                # graph replays
            torch.cuda.synchronize()
            results.append((rt.params.detach().cpu().clone(), rt.grads.detach().cpu().clone(), rt.loss_value()))
            if dp is not None:
                kinds = [c[1].__name__ for grp in plan.calls for c in grp if c[0] == "k"]
                assert kinds.count("monet_allreduce_bucket") == len(dp.buckets)
                assert kinds.count("monet_comm_join") == 1
                dp.close()
        (p0, g0, l0), (p1, g1, l1) = results
        assert torch.equal(p0, p1) and torch.equal(g0, g1) and l0 == l1
    finally:
        dist.destroy_process_group()
