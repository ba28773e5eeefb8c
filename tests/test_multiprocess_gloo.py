"""Multi-process host logic on CPU with the gloo backend, world size 2:
* batch sharding: shards are disjoint, cover the batch, and are rank-seeded;
* max-over-ranks timing reduction used by bench.py;
* config-5 data-parallel step: after DDP's gradient all-reduce and the SGD update, every rank holds
  identical parameters, equal to a single-process step on the union batch.
The 3x3 layer is the fp32 stand-in (the sm_100a layer needs a GPU); the DDP plumbing is the same."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2004_11077_b200 import training as TR


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # sharding
        lo, hi = TR.shard_range(10, rank, world)
        got = [None] * world
        dist.all_gather_object(got, (lo, hi))
        # timing reduction
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # DDP training step on a small ResNet-18 with the fp32 stand-in convolution
        torch.manual_seed(0)
        model = TR.ResNet18(TR.plain_conv_factory)
        ddp = torch.nn.parallel.DistributedDataParallel(model)
        opt = TR.make_optimizer(ddp, lr=0.1)
        x, y = TR.synthetic_batch(4, rank, seed=7)
        TR.train_step(ddp, opt, x, y)
        flat = torch.cat([p.detach().flatten() for p in model.parameters()])
        gathered = [torch.zeros_like(flat) for _ in range(world)]
        dist.all_gather(gathered, flat)
        same = all(torch.equal(gathered[0], g) for g in gathered)
        if rank == 0:
            # numpy pickles by value (a torch tensor would be shared through a file descriptor that
            # disappears when this process exits before the parent reads it)
            q.put({"shards": got, "tmax": float(t), "same": same, "params": flat.numpy().copy()})
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_gloo_world2_sharding_timing_and_ddp_step():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=540)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["shards"] == [(0, 5), (5, 10)]
    assert res["tmax"] == 2.0
    assert res["same"]
    # single-process reference: same init, union batch, mean of per-rank losses == DDP average
    torch.manual_seed(0)
    ref = TR.ResNet18(TR.plain_conv_factory)
    opt = TR.make_optimizer(ref, lr=0.1)
    xs, ys = zip(*(TR.synthetic_batch(4, r, seed=7) for r in range(world)))
    # DDP averages gradients of per-rank mean losses == gradient of the mean over the union batch;
    # BatchNorm statistics are per rank in DDP, so compare against per-rank forwards
    opt.zero_grad()
    loss = sum(torch.nn.functional.cross_entropy(ref(x), y) for x, y in zip(xs, ys)) / world
    loss.backward()
    opt.step()
    flat = torch.cat([p.detach().flatten() for p in ref.parameters()])
    assert torch.allclose(flat, torch.from_numpy(res["params"]), atol=1e-5, rtol=1e-4)


def test_shard_range_properties():
    for total in (0, 1, 7, 1024):
        for world in (1, 2, 3, 8):
            spans = [TR.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_resnet18_layer_inventory():
    model = TR.ResNet18(TR.plain_conv_factory)
    n3 = sum(1 for m in model.modules() if isinstance(m, torch.nn.Conv2d) and m.kernel_size == (3, 3)
             and m.stride == (1, 1))
    assert n3 == 14  # stem + 13 stride-1 3x3 convs become Winograd layers
