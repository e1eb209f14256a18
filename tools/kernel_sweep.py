#!/usr/bin/env python
"""Kernel-alone timing of one workload's dominant kernel under A/B environment
switches (each variant in its own process: the launchers read their switches once).

  python tools/kernel_sweep.py img3d "LFG_IMG3D_DEBUG=0" "LFG_IMG3D_DEBUG=4" ...
  python tools/kernel_sweep.py --one img3d 16      (internal: one variant, prints JSON)

Times back-to-back launches of `group` samples on one stream with CUDA events
(lfg_time_kernels, the bench's roofline pass), inputs HBM-resident (> L2)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(workload: str, group: int, n_launch: int = 8):
    import bench
    from paper_2509_10712_b200 import lfgpu as L

    class A:
        pool = 0
        heavy_frac = 0.0
        time_scale = 10.0
        fg = 0.4
        workers = 16
    A.workload = workload
    ctx, B, g = bench.make_context(L, workload, group=group)
    wl = bench.make_workload(workload, L, ctx, host=False, seed=1, args=A)
    ids = list(range(1000, 1000 + group * n_launch))
    hbm, tf32, _ = bench.peaks()
    r = min((bench.kernel_roofline(L, ctx, wl, ids, hbm, tf32) for _ in range(3)),
            key=lambda x: x["mean_launch_us"])                 # best of 3 passes (each after a warm-up)
    wl.close()
    ctx.close()
    return r


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        print(json.dumps(one(sys.argv[2], int(sys.argv[3]))))
        sys.exit(0)
    wl = sys.argv[1]
    group = int(os.environ.get("GROUP", "0")) or {"img3d": 16, "img3d_fg": 16, "img3d_zoom": 16, "rrc": 256, "speech": 64, "speech_f32": 64}[wl]
    for var in sys.argv[2:] or [""]:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, __file__, "--one", wl, str(group)], env=env,
                             capture_output=True, text=True, timeout=600)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
        print(f"{var or 'default':40s} {line}", flush=True)
