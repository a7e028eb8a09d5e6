"""World-size-2 checks of the multi-GPU path on CPU (gloo): the store shard
rule (record k lives on rank k % world, csrc/store.cpp) partitions the archive
exactly, every rank validates the whole archive, and the bench's timing
reduction is the max over ranks.  Decode itself has no collective."""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, data, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    import bench
    from paper_2306_16699_b200 import _native

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = _native.archive_shard(data, rank, world).tolist()
        shards = [None] * world
        dist.all_gather_object(shards, mine)
        slowest = bench.reduce_max(0.5 + rank, dist)
        q.put((rank, shards, slowest, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shards_partition_and_max_timing(world):
    from paper_2306_16699_b200 import synth
    data = synth.archive_bytes(synth.config2(37, seed=5))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, shards, slowest, err in results:
        assert err is None, err
        allidx = sorted(i for s in shards for i in s)
        assert allidx == list(range(37))  # disjoint and complete
        for r, s in enumerate(shards):
            assert all(i % world == r for i in s)
        assert slowest == 0.5 + (world - 1)


def test_shard_rejects_bad_rank():
    from paper_2306_16699_b200 import _native, errors, synth
    data = synth.archive_bytes(synth.config2(4, seed=1))
    with pytest.raises(errors.InvalidInputError):
        _native.archive_shard(data, 2, 2)
    assert list(_native.archive_shard(data, 0, 1)) == [0, 1, 2, 3]
    assert np.array_equal(_native.archive_shard(data, 1, 3), [1])
