"""Parity of the BENCHMARKED path: bench.py's exact shard contexts (batch size,
launch group, workers, slot buffers, chains, synthetic pools) run through
lfg_run_shard -- fast-first eager seals, zero-copy and collated batches, the
pre-drawn parameters of the draw thread pool -- and every delivered sample is
copied out of its batch tensor (lfg_run_config capture) and compared with the CPU
oracle (oracle/checks.py bars: labels / windows / masks / padding bit-exact, values
within 1e-5 relative).

  C2  rrc     batch 256, launch groups of 256, 1,024-image 256..512 px pool, 640 ids
  C4  speech  batch 64, groups of 64, max_len 170,000, L in {30k, 100k, 170k} + random;
              int16 PCM (the bench default) and f32 samples
  C1  img3d   batch 2, groups of 16, D x 384 x 384 volumes with D in {128, 300, 512};
              also with RandomCrop's foreground oversampling (K2) on
Both input sources: HBM-resident (bench "value") and pinned host (bench "e2e").
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import checks  # noqa: E402  (oracle/checks.py)

SEED = 1


class _Args:
    pool = 0
    heavy_frac = 0.2
    time_scale = 10.0


def _run_and_check(lfgpu, oracle, ctx, wl, ids, check_one, workers=16):
    """Run `ids` through the shard with every position captured; check each delivered
    sample; return the captured batch indices and the worst err/bound."""
    B = wl.B
    rc = lfgpu.run_config(batch_size=B, n_workers=workers, d2h_probe=1)
    rep, consumed, bsz, _ = ctx.run_shard(wl.chain, wl.descs(ids), rc, capture=list(range(len(ids))))
    cap = ctx.last_capture
    assert rep.exactly_once == 1 and sorted(consumed.tolist()) == sorted(ids)
    assert len(cap) == len(ids), f"{len(ids) - len(cap)} delivered samples were not captured"
    # the captured batch index of each sample agrees with the consumed-id order
    order = np.repeat(np.arange(len(bsz)), bsz)
    where = {int(i): int(b) for i, b in zip(consumed, order)}
    for pos, (_, b) in cap.items():
        assert where[ids[pos]] == b
    with ThreadPoolExecutor(max(1, min(16, os.cpu_count() or 1))) as ex:
        ratios = list(ex.map(lambda kv: check_one(ids[kv[0]], kv[1][0]), cap.items()))
    worst = max(ratios)
    assert worst <= 1.0, f"worst err/bound {worst:.3f}"
    return rep, worst


@pytest.mark.parametrize("host", [False, True], ids=["hbm", "pinned"])
def test_c2_rrc_bench_config(lfgpu, oracle, host):
    ctx, B, group = bench.make_context(lfgpu, "rrc", seed=SEED)
    assert (B, group) == (256, 256)
    wl = bench.make_workload("rrc", lfgpu, ctx, host=host, seed=SEED, args=_Args())
    ocfg = oracle.cfg2d()
    try:
        ids = list(range(3000, 3000 + 640))          # 2.5 launch groups: a short tail batch
        rep, worst = _run_and_check(
            lfgpu, oracle, ctx, wl, ids,
            lambda sid, raw: checks.check_rrc(oracle, ocfg, SEED, sid, wl.source(sid)[0], raw))
        assert rep.batches == 3 and rep.inplace_batches >= 1
        print(f"C2 {'pinned' if host else 'hbm'}: 640 samples, worst err/bound {worst:.3f}")
    finally:
        wl.close()
        ctx.close()


@pytest.mark.parametrize("pcm16", [True, False], ids=["pcm16", "f32"])
@pytest.mark.parametrize("host", [False, True], ids=["hbm", "pinned"])
def test_c4_speech_bench_config(lfgpu, oracle, host, pcm16):
    ctx, B, group = bench.make_context(lfgpu, "speech", seed=SEED)
    assert (B, group) == (64, 64)
    lens = np.random.default_rng(5).integers(30000, 170001, size=64)
    lens[:6] = [30000, 100000, 170000, 170000, 30001, 99999]
    wl = bench.SpeechWorkload(lfgpu, ctx, pool=64, host=host, seed=SEED, lens=lens, pcm16=pcm16)
    ocfg = oracle.cfgsp()
    try:
        ids = list(range(0, 160))                    # 2.5 batches of 64
        rep, worst = _run_and_check(
            lfgpu, oracle, ctx, wl, ids,
            lambda sid, raw: checks.check_speech(oracle, ocfg, SEED, sid, wl.source(sid)[0], raw))
        print(f"C4 {'pinned' if host else 'hbm'} {'pcm16' if pcm16 else 'f32'}: 160 utterances, "
              f"worst err/bound {worst:.3f}")
    finally:
        wl.close()
        ctx.close()


@pytest.mark.parametrize("fg", [0.0, 0.4], ids=["crop", "fg_oversampling"])
@pytest.mark.parametrize("host", [False, True], ids=["hbm", "pinned"])
def test_c1_img3d_bench_config(lfgpu, oracle, host, fg):
    ctx, B, group = bench.make_context(lfgpu, "img3d_fg" if fg else "img3d", seed=SEED)
    assert (B, group) == (2, 16)
    wl = bench.Img3dWorkload(lfgpu, ctx, pool=3, host=host, seed=SEED, p_fg=fg, depths=[128, 300, 512])
    ocfg = oracle.cfg3d(has_fg=1 if fg else 0, p_fg=fg)
    vols = {k: wl.source(k) for k in range(3)}       # D2H once per volume
    try:
        ids = list(range(0, 40))                     # 2.5 launch groups of 16
        rep, worst = _run_and_check(
            lfgpu, oracle, ctx, wl, ids,
            lambda sid, raw: checks.check_img3d(oracle, ocfg, SEED, sid, *vols[sid % 3], raw, (128, 128, 128)))
        print(f"C1 {'pinned' if host else 'hbm'} fg={fg}: 40 samples, worst err/bound {worst:.3f}")
    finally:
        wl.close()
        ctx.close()
