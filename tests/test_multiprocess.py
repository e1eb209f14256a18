"""N>1 host logic on CPU: world_size-2 gloo processes exercise bench.py's
data-parallel plumbing -- the batch-block round-robin sampler partition
(sample i -> GPU floor(i/B) mod G), the max-over-ranks timing
reduce and the single end-of-run counter all-reduce (the only collective the
north_star allows) -- plus the exactly-once audit over the union of shards."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, n_batches, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = bench.shard_ids(n_batches, B, rank, world)
    # every shard gets whole batches: no batch straddles two GPUs
    assert len(ids) == n_batches * B
    assert all((i // B) % world == rank for i in ids)
    elapsed = 10.0 + rank                                   # per-rank device time
    el_max = bench.allreduce_max(dist, elapsed, rank)
    counters = bench.allreduce_sum(dist, [len(ids), 1, 0], rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, ids)
    bench.barrier(dist)
    if rank == 0:
        out.put((el_max, counters, gathered))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_shard_partition_and_counter_reduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    B, n_batches = 4, 5
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, n_batches, q))
             for r in range(world)]
    for p in procs:
        p.start()
    el_max, counters, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert el_max == 10.0 + world - 1                       # max over ranks
    assert counters == [n_batches * B * world, world, 0]
    union = sorted(i for part in gathered for i in part)    # exactly-once over shards
    assert union == list(range(n_batches * B * world))
