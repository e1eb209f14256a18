"""Streaming consumer API (lfg_shard_start / lfg_shard_next_batch / lfg_shard_finish):
the shard loop runs on a library thread and hands every sealed batch to the caller,
who is the trainer (the reference's BatchQueue between build_batches and
run_consumer, batcher.cpp:50-58, trainer.cpp:7-18).

The consumer here holds several batches at once (so the loop must wait for batch
buffers: back-pressure), interleaves its releases with sealing, reads every
delivered batch tensor back and compares each sample with the CPU oracle.
"""
import os
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import checks  # noqa: E402  (oracle/checks.py: the checker)

SEED = 7


def _images(lfgpu, ctx, n, rng):
    imgs, ptrs = [], []
    for _ in range(n):
        H, W = int(rng.integers(180, 420)), int(rng.integers(180, 420))
        im = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        p = ctx.device_alloc(im.nbytes)
        ctx.h2d(p, im)
        imgs.append(im)
        ptrs.append(p)
    return imgs, ptrs


def test_stream_delivers_every_batch_to_the_consumer(lfgpu, oracle):
    B, n_pool, n = 16, 24, 16 * 12 + 5          # a short tail batch
    ctx = lfgpu.Context(batch_size=B, n_workers=4, max_group=16, max_slot_buffers=6, seed=SEED)
    rng = np.random.default_rng(3)
    imgs, ptrs = _images(lfgpu, ctx, n_pool, rng)
    ch = ctx.chain(lfgpu.obj_det_ops())
    ocfg = oracle.cfg2d()
    ids = list(range(100, 100 + n))
    descs = [lfgpu.sample_desc(i, imgs[i % n_pool].shape, ptrs[i % n_pool]) for i in ids]
    plane = 3 * 224 * 224 * 4
    try:
        st = ctx.shard_stream(ch, descs, lfgpu.run_config(batch_size=B, n_workers=4))
        # while the stream owns the context, submitting and other runs are refused
        with pytest.raises(lfgpu.LfgError) as e:
            ctx.submit(ch, descs[0])
        assert e.value.code == lfgpu.ERR_STATE
        held, seen, sizes, worst = [], [], [], 0.0
        checked = 0
        while True:
            r = st.next_batch(timeout_us=5_000_000)
            if r is None:
                break
            b, nb = r
            info = ctx.batch_info(b)
            assert info["n"] == nb
            seen += info["ids"]
            sizes.append(nb)
            raw = ctx.batch_to_host(b, nb * plane)
            for k in range(0, nb, 5):                      # every 5th sample of each batch
                sid = info["ids"][k]
                worst = max(worst, checks.check_rrc(oracle, ocfg, SEED, sid, imgs[sid % n_pool],
                                                    raw[k * plane:(k + 1) * plane]))
                checked += 1
            held.append(b)
            if len(held) == 3:                             # the consumer holds 3 batches
                time.sleep(0.002)                          # ... while the loop keeps sealing
                ctx.batch_release(held.pop(0))
        for b in held:
            ctx.batch_release(b)
        rep, consumed, bsz, cls = st.finish()
    finally:
        for p in ptrs:
            ctx.device_free(p)
        ctx.close()
    assert worst <= 1.0, f"worst err/bound {worst:.3f}"
    assert checked >= n // 5
    assert sorted(seen) == ids and len(seen) == len(set(seen))
    assert consumed.tolist() == seen                        # delivery order == consumption order
    assert bsz.tolist() == sizes and sum(sizes) == n and sizes.count(B) == n // B
    assert rep.exactly_once == 1 and rep.samples == n
    assert 0.0 <= rep.consumer_idle_frac <= 1.0 and rep.consumer_span_ms > 0


def test_stream_finish_drains_untaken_batches(lfgpu):
    """finish() before the end of the stream releases what the consumer never took
    and still reports every sample exactly once."""
    B = 8
    ctx = lfgpu.Context(batch_size=B, n_workers=4, max_group=8, max_slot_buffers=3, seed=SEED)
    rng = np.random.default_rng(4)
    imgs, ptrs = _images(lfgpu, ctx, 8, rng)
    ch = ctx.chain(lfgpu.obj_det_ops())
    descs = [lfgpu.sample_desc(i, imgs[i % 8].shape, ptrs[i % 8]) for i in range(80)]
    try:
        st = ctx.shard_stream(ch, descs, lfgpu.run_config(batch_size=B))
        b, nb = st.next_batch(timeout_us=5_000_000)
        ctx.batch_release(b)
        rep, consumed, bsz, _ = st.finish()
        assert rep.exactly_once == 1 and sorted(consumed.tolist()) == list(range(80))
        # the context is usable again
        rep2, consumed2, _, _ = ctx.run_shard(ch, descs[:16], lfgpu.run_config(batch_size=B))
        assert rep2.exactly_once == 1
        with pytest.raises(lfgpu.LfgError):
            st.finish()
    finally:
        for p in ptrs:
            ctx.device_free(p)
        ctx.close()


def test_cpp_run_consumer_over_shard_feed():
    """The reference's own run_consumer (trainer.cpp:20-66) consuming the high-throughput
    path: gpu::feed_shard publishes each sealed device batch into a BatchQueue as it is
    sealed; exactly-once, batch accounting and one batch tensor against the oracle are
    checked inside the program (tests/cpp/shard_feed.cpp)."""
    import subprocess
    root = ROOT
    pkg = os.path.join(root, "paper_2509_10712_b200")
    ora = os.path.join(root, "oracle")
    src = os.path.join(root, "tests", "cpp", "shard_feed.cpp")
    exe = os.path.join(root, "tests", "cpp", "shard_feed")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"), src, "-o", exe,
                           "-L", pkg, "-lloadflow_b200", "-llfgpu", f"-Wl,-rpath,{pkg}",
                           "-L", ora, "-llf_oracle", f"-Wl,-rpath,{ora}", "-lpthread"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
