"""World-size-2 run of the consumer training loop (train.DecodeTrainLoop,
BASELINE config 5's structure): both ranks on cuda:0 with the gloo backend
(gpurun provides one GPU; the ranks never spin on each other, the gradient
all-reduce goes through host memory).  Each rank opens its shard of ONE
archive through Store(..., shard_rank, shard_world), decodes its own
batches, and DDP's all-reduce keeps the ResNet-18 replicas bit-identical."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    try:
        import torch
        import torch.distributed as dist
        import torchvision

        from paper_2306_16699_b200 import train

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        st = train.open_sharded_store("c2", 512, rank, world, device="cuda:0", seed=11)
        glob = [st.record_meta(k)["global_index"] for k in range(len(st))]
        torch.manual_seed(0)  # identical initial weights on both ranks
        model = torchvision.models.resnet18(num_classes=10)
        loop = train.DecodeTrainLoop(st, 32, 32, 16, 10, precision="bf16", aug="offset", seed=100 + rank,
                                     ddp=True, device="cuda:0", model=model)
        losses = [float(loop.step().item()) for _ in range(2)]
        torch.cuda.synchronize()
        chk = train.param_checksum(loop.model)
        out = [None] * world
        dist.all_gather_object(out, (glob, chk.tolist(), losses))
        q.put((rank, out, None))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_ddp_two_ranks_sharded_store():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, out, err in res:
        assert err is None, err
    out = res[0][1]
    shards = [set(o[0]) for o in out]
    assert shards[0].isdisjoint(shards[1]) and shards[0] | shards[1] == set(range(512))
    assert all(g % world == r for r, s in enumerate(shards) for g in s)
    assert out[0][1] == out[1][1], "DDP replicas diverged"
    assert all(np.isfinite(o[2]).all() for o in out)
    assert out[0][2] != out[1][2], "ranks must train on different batches"
