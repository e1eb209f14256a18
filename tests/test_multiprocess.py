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


def _bench_line(env_extra, *argv):
    import json
    import subprocess
    import sys
    env = dict(os.environ, LFG_BENCH_BACKEND="gloo", **env_extra)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True,
                       text=True, env=env, timeout=600, cwd=ROOT)
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    return r.returncode, (json.loads(lines[-1]) if lines else None), r.stderr


def test_bench_main_spawns_one_rank_per_gpu():
    """`bench.py --gpus 2` with no launcher re-runs itself under torch.distributed.run
    (2 ranks, gloo here; NCCL on the GPU box) and main() goes through the whole
    multi-rank path: partition, max-over-ranks spans, the counter / id-digest reduce
    and the exactly-once audit over the union of the shards.  The shard itself is
    the CPU stand-in (LFG_BENCH_FAKE_SHARD, marked in the line)."""
    rc, line, err = _bench_line({"LFG_BENCH_FAKE_SHARD": "1"}, "--gpus", "2", "--steps", "4", "--warmup", "3")
    assert rc == 0, err
    assert line["n_gpus"] == 2 and line["fake_shard"] is True
    assert line["config"]["parallelism"] == "dp2 independent loader shards"
    assert line["exactly_once"] is True
    assert line["ms_per_step"] == 2.0 / 4                   # max over ranks (1.0, 2.0 ms)
    assert line["value"] == 2 * 4 * 256 / 2e-3               # samples of all ranks / max span


def test_bench_exactly_once_catches_a_lost_and_duplicated_id():
    rc, line, err = _bench_line({"LFG_BENCH_FAKE_SHARD": "dup"}, "--gpus", "2", "--steps", "3", "--warmup", "3")
    assert rc == 0, err
    assert line["exactly_once"] is False


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", LFG_BENCH_FAKE_SHARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                       text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr


def test_reference_arm_reports_the_same_config():
    """--impl reference prints the identical `config` object as the repo arm."""
    import sys
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    a = argparse.Namespace(workload="rrc", group=0, workers=16, pool=0, seed=1)
    c1 = bench.bench_config(a, 1)
    assert c1["batch"] == 256 and c1["launch_group"] == 256
    assert c1["raw_pool_bytes"] == 459821312            # the pool the repo arm allocates
