#!/usr/bin/env python
"""C5: timeout / slow-ratio sweep of the heavy-tailed 3D-UNet loader,
B200 shard vs the reference CPU loader on the host cores.

For every slow fraction f in {0.1, 0.2, 0.3} and timeout policy t_out in {p50, p75, p90,
none} (nearest-rank percentile of the per-sample totals window, fixed -- no p75->p90
escalation -- after a warm-up; "none" = kNoTimeout):

  gpu : bench.py's img3d_heavy workload (KiTS19-shaped volumes, crop 128^3 chain, a
        fraction f of samples carries a synthetic cost of cost_ms x time_scale us on the
        device (K14 spin) and a 2 ms synthetic trainer step per batch of 2 on a
        high-priority stream).  Reports delivered samples/s, consumer idle % (CUDA
        events, trainer.hpp:41-46 formula), slow fraction and the final t_out.
  cpu : oracle/_ref/minato_cpu -- the reference libloadflow realtime Minato pipeline
        with the oracle transforms, a leading SampleCost transform sleeping heavy_ms for
        a fraction f of samples, run_consumer at 200 ms per batch (trainer.hpp:15) and
        the same percentile policy.  Bounded sample per point.

  python tools/sweep.py [--out profiles/r1_c5_sweep.md] [--no-cpu]
Multi-GPU: launch under torchrun like bench.py; rank 0 prints (max over ranks of the
device time, sum of samples; one all-reduce of counters at the end of each point).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

FRACS = (0.1, 0.2, 0.3)
# (name, percentile): 0 = no timeout; -1 = the synchronous head-of-line baseline
# (start_sync_loader, baselines.cpp:12-151; GPU: lfg_run_config.policy 3)
POLICIES = (("p50", 50), ("p75", 75), ("p90", 90), ("none", 0), ("sync", -1))


class _Args:
    pool = 0
    workers = 16
    time_scale = 10.0
    heavy_frac = 0.2


def gpu_point(L, wl, frac, pct, steps, warmup, rank, world, dist, local):
    ctx = wl.ctx
    wl.heavy_frac = frac
    B = wl.B
    a = _Args()
    ids = bench.shard_ids(warmup + steps, B, rank, world)
    warm, timed = ids[: warmup * B], ids[warmup * B:]
    rc = L.run_config(batch_size=B, policy=3 if pct < 0 else (2 if pct else 0), percentile=pct if pct > 0 else 75,
                      t_out_us=0,
                      trainer_us=2000, n_workers=a.workers, warmup_us=20000, update_interval_us=1000)
    ctx.run_shard(wl.chain, wl.descs(warm), rc, want_ids=False)
    ctx.synchronize()
    bench.barrier(dist)
    rep, _, _, _ = ctx.run_shard(wl.chain, wl.descs(timed), rc)
    ctx.synchronize()
    bench.barrier(dist)
    el = bench.allreduce_max(dist, rep.elapsed_ms, local)
    tot = bench.allreduce_sum(dist, [rep.timed_samples, rep.slow, rep.samples,
                                     rep.consumer_busy_ms, rep.consumer_span_ms], local)
    return {"samples_per_s": round(tot[0] / (el / 1e3), 1),
            "idle_pct": round(100 * (1 - tot[3] / tot[4]), 2) if tot[4] > 0 else None,
            "slow_frac": round(tot[1] / max(1, tot[2]), 3),
            "final_t_out_us": round(rep.final_t_out_us, 1) if pct > 0 else None}


def cpu_point(frac, pct, steps):
    h = bench.ref_harness()
    if h is None:
        return None
    cores = os.cpu_count() or 1
    extra = ["--loader", "sync", "--pct", "0"] if pct < 0 else ["--pct", str(pct)]
    out = subprocess.run([h, "--workload", "img3d", "--steps", str(steps if pct >= 0 else min(steps, 6)),
                          "--warmup", "2", "--workers", str(cores), "--heavy-frac", str(frac),
                          "--heavy-ms", "470", "--trainer-ms", "200", "--profiler-warmup-ms", "1500",
                          "--max-seconds", "40"] + extra,
                         capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
    b = json.loads(out)
    return {"samples_per_s": b["value"], "idle_pct": round(100 * b["idle_frac"], 2),
            "slow_frac": round(b["slow"] / max(1.0, b["samples"] + 4), 3),
            "final_t_out_ms": b["final_t_out_ms"] if pct > 0 else None, "cores": b["cores"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400, help="timed batches per GPU point")
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2509_10712_b200 import lfgpu as L
    rank, local, world, dist = bench.dist_setup(args.gpus)
    ctx = L.Context(device=local, batch_size=2, n_workers=16, max_group=1, max_slot_buffers=24, seed=1)
    wl = bench.make_workload("img3d_heavy", L, ctx, False, 1, _Args())
    rows = []
    for frac in FRACS:
        for name, pct in POLICIES:
            g = gpu_point(L, wl, frac, pct, args.steps, args.warmup, rank, world, dist, local)
            c = None if (args.no_cpu or rank != 0) else cpu_point(frac, pct, args.cpu_steps)
            rows.append({"slow_frac_target": frac, "t_out": name, "gpu": g, "cpu": c})
            if rank == 0:
                print(json.dumps(rows[-1]), flush=True)
    wl.close()
    ctx.close()
    if rank != 0:
        return
    lines = [f"# C5 timeout / slow-ratio sweep ({world} x B200 shard(s) vs reference CPU loader)",
             "",
             "GPU: img3d_heavy (crop 128^3 chain; heavy samples spin cost_ms x 10 us; 2 ms trainer "
             "step per batch of 2). CPU: reference libloadflow Minato pipeline + oracle transforms, "
             "heavy samples sleep 470 ms, 200 ms trainer step per batch of 2.",
             "t_out = fixed nearest-rank percentile of the per-sample totals window after warm-up "
             "(none = kNoTimeout); sync = the synchronous head-of-line loader (batch k = ids "
             "[kB, (k+1)B), sealed when complete, in order: start_sync_loader on the CPU, "
             "lfg_run_config.policy 3 on the GPU).",
             "",
             "| slow frac | t_out | GPU samples/s | GPU idle % | GPU slow | GPU t_out (us) | "
             "CPU samples/s | CPU idle % | CPU slow | CPU t_out (ms) |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        g, c = r["gpu"], r["cpu"] or {}
        lines.append(f"| {r['slow_frac_target']} | {r['t_out']} | {g['samples_per_s']} | {g['idle_pct']} | "
                     f"{g['slow_frac']} | {g['final_t_out_us']} | {c.get('samples_per_s')} | "
                     f"{c.get('idle_pct')} | {c.get('slow_frac')} | {c.get('final_t_out_ms')} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
