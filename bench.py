#!/usr/bin/env python
"""bench.py -- MinatoLoader preprocessing hot path on B200 (one process per GPU).

Metric (BASELINE.json): samples/sec/GPU delivered to the trainer; consumer GPU
idle %; transform HBM GB/s.  A "step" is one batch through the whole hot path:
submit -> fused transform kernels -> timeout classification -> eager seal ->
delivered (resident, stream-ordered) to the trainer stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload rrc|img3d|img3d_heavy]
  python bench.py --impl reference ...   # the reference CPU loader on host cores

Workloads:
  rrc          C2: ImageNet-shaped u8 3x(256..512)^2 -> RandomResizedCrop 224 + flip +
               normalize, batch 256 (BASELINE configs[1], the N=1 headline)
  img3d        C1/C3 shapes: KiTS19-shaped volumes (H=W=384, D from gen_empirical
               img_seg sizes) -> crop 128^3 + flip + brightness + noise, batch 2
  img3d_fg     C1 shapes with RandomCrop's MLPerf foreground oversampling (p 0.4): those
               samples scan their whole label volume (K2) -- a real heavy tail
  img3d_heavy  C3: img3d_fg's REAL heavy tail (40% of crops scan their label volume;
               from pinned memory that whole volume crosses PCIe) in launch groups of 16,
               4 in-flight groups, a synthetic trainer step calibrated to 90% of the
               loader's measured capacity; Minato (adaptive p75/p90 timeout) reports
               consumer idle %, and the synchronous head-of-line loader runs beside it

value      : whole-job samples/s with raw inputs resident in HBM (device events on
             each rank's trainer stream, max over ranks)
e2e        : same metric with raw inputs in pinned host memory (H2D of each sample's
             crop box / window inside the timed region) plus a 16-byte D2H read of every
             delivered batch, consumed through the public streaming API (lfg_shard_start /
             lfg_shard_next_batch / lfg_batch_release: this process is the trainer)
dropin     : (rrc) the drop-in C++ path -- the reference's own realtime Minato wiring over our
             headers, process_sample worker threads submitting through the C ABI
others     : (rrc at N=1) C1 / C1-fg / C3 / C4 each measured by this script in a sub-process
             after the headline run ("other_workloads"; --no-others skips them)
roofline   : the dominant kernel timed alone (serial mode) with CUDA events:
             algorithmic bytes per launch / mean launch time, against MEASURED_PEAKS.json
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# one hardware queue per launch-group stream (CUDA reads it at context creation;
# the library never sets it: engine.cpp Context())
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ROOT)

METRIC = "samples/sec/GPU delivered to trainer; consumer GPU idle %; transform HBM GB/s"

# workload -> (batch size, samples per launch group, default timed steps)
BATCH = {"rrc": (256, 256, 1000), "img3d": (2, 16, 4000), "img3d_fg": (2, 16, 2000),
         "img3d_heavy": (2, 16, 400),
         "img3d_zoom": (2, 16, 2000),
         "speech": (64, 64, 500),
         "speech_f32": (64, 64, 500)}


def peaks():
    """(HBM GB/s, dense TF32 TFLOP/s, source).  TF32 is half the dense bf16 rate on
    B200 (1.1 vs 2.25 PFLOP/s nominal), so the tensor denominator is the measured
    cuBLAS bf16 burst figure / 2."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return (float(p["hbm_gbs"]), float(p["bf16_tflops"]) / 2.0,
                "measured (MEASURED_PEAKS.json; tf32 = bf16_tflops / 2)")
    except Exception:
        return 6650.0, 1590.0 / 2.0, "fallback (B200_PROFILING.md; tf32 = bf16 / 2)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ distributed
def launch_ranks(args) -> int | None:
    """`--gpus N` (N > 1) without a launcher: re-run this very command under
    torch.distributed.run, one process per GPU (the driver's own launch line).
    Returns the launcher's exit code, or None when already inside a launcher."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup(n_gpus: int):
    """One process per GPU: RANK / LOCAL_RANK / WORLD_SIZE from the launcher; the
    world must be exactly --gpus.  NCCL (gloo with LFG_BENCH_BACKEND=gloo: the CPU
    test of this plumbing)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but WORLD_SIZE={world} (one rank per GPU)")
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("LFG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            torch.cuda.set_device(local)
            try:   # bind the process group to this rank's GPU up front (eager NCCL init)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            except TypeError:
                dist.init_process_group("nccl")
        else:
            dist.init_process_group(backend)
        return rank, local, world, dist
    return 0, 0, 1, None


def _coll_device(dist, local: int) -> str:
    return f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"


def allreduce_max(dist, x: float, local: int) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device(dist, local))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(dist, xs, local: int):
    """The run's only collective use: one reduce of a small counter vector (north_star)."""
    if dist is None:
        return list(xs)
    import torch
    t = torch.tensor(list(xs), dtype=torch.float64, device=_coll_device(dist, local))
    dist.all_reduce(t)
    return t.tolist()


def allreduce_sum_i64(dist, xs, local: int):
    if dist is None:
        return [int(x) for x in xs]
    import torch
    t = torch.tensor([int(x) for x in xs], dtype=torch.int64, device=_coll_device(dist, local))
    dist.all_reduce(t)
    return [int(v) for v in t.tolist()]


def barrier(dist):
    if dist is None:
        return
    if dist.get_backend() == "nccl":
        import torch
        dist.barrier(device_ids=[torch.cuda.current_device()])
    else:
        dist.barrier()


def id_digest(ids) -> list[int]:
    """Order-independent digest of a set of sample ids, summable across ranks without
    overflow (<= 2^23 ids): [count, sum id, sum h1, sum h2] with h1 / h2 the low 40
    bits of two splitmix64 hashes.  The union of the shards is exactly-once iff the
    summed digest equals the digest of the expected ids (and no shard saw a duplicate)."""
    a = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = a + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    m = np.uint64((1 << 40) - 1)
    return [int(a.size), int(a.sum(dtype=np.uint64)), int((z & m).sum(dtype=np.uint64)),
            int(((z >> np.uint64(24)) & m).sum(dtype=np.uint64))]


# ------------------------------------------------------------------ workloads
def shard_ids(n_total_batches: int, B: int, rank: int, world: int):
    """Batch-block round robin: global sample i goes to GPU floor(i/B) mod G."""
    ids = []
    for k in range(n_total_batches * world):
        if k % world == rank:
            ids.extend(range(k * B, (k + 1) * B))
    return ids


class RrcWorkload:
    name = "rrc"
    B = 256

    def __init__(self, L, ctx, pool: int, host: bool, seed: int):
        self.L, self.ctx, self.seed = L, ctx, seed
        rng = np.random.default_rng(seed)
        self.hw = rng.integers(256, 513, size=(pool, 2))
        sizes = [int(h * w * 3) for h, w in self.hw]
        self.offs = np.concatenate([[0], np.cumsum([(s + 255) // 256 * 256 for s in sizes])])
        total = int(self.offs[-1])
        self.host = host
        self.base = ctx.host_alloc(total) if host else ctx.device_alloc(total)
        for i, (h, w) in enumerate(self.hw):
            ctx.synth_image(seed, i, int(h), int(w), self.base + int(self.offs[i]),
                            on_device=not host)
        self.pool = pool
        self.pool_bytes = total
        self.chain = ctx.chain(L.obj_det_ops())

    def descs(self, ids):
        L = self.L
        out = []
        for i in ids:
            k = i % self.pool
            h, w = self.hw[k]
            out.append(L.sample_desc(i, (int(h), int(w), 3), self.base + int(self.offs[k]),
                                     src_kind=L.SRC_HOST_PINNED if self.host else L.SRC_DEVICE))
        return out

    def source(self, i):
        """HWC u8 source image of sample id i (for the oracle check)."""
        k = i % self.pool
        h, w = (int(x) for x in self.hw[k])
        return (_read(self.ctx, self.base + int(self.offs[k]), h * w * 3, np.uint8, self.host).reshape(h, w, 3),)

    @staticmethod
    def pool_bytes_of(pool: int, seed: int) -> int:
        hw = np.random.default_rng(seed).integers(256, 513, size=(pool, 2))
        return int(sum((int(h * w * 3) + 255) // 256 * 256 for h, w in hw))

    def close(self):
        (self.ctx.host_free if self.host else self.ctx.device_free)(self.base)


def _read(ctx, ptr: int, n: int, dtype, host: bool) -> np.ndarray:
    """n elements at ptr (pinned host: a copy of the view; device: D2H)."""
    nb = n * np.dtype(dtype).itemsize
    if host:
        import ctypes
        return np.frombuffer((ctypes.c_uint8 * nb).from_address(ptr), dtype=np.uint8).view(dtype).copy()
    out = np.empty(nb, dtype=np.uint8)
    ctx.d2h(out, ptr)
    return out.view(dtype)


def img_seg_dims(n: int, seed: int):
    """Volume depth from the reference's img_seg size model (workloads.cpp:180-185):
    bytes_in ~ 30..375 MB cost-correlated; D = clamp(round(bytes_in / (5*384^2)), 128, 512)."""
    mu = math.log(470.0)
    sigma = math.log(750.0 / 470.0) / 1.2815515655446004
    rng = np.random.default_rng(seed)
    z = rng.standard_normal(n)
    total = np.clip(np.exp(mu + sigma * z), 10, 2230)
    q = 0.5 * (1 + np.vectorize(math.erf)((np.log(total) - mu) / (sigma * math.sqrt(2))))
    pos = np.clip(0.85 * q + 0.15 * rng.random(n), 0, 1)
    mb = 30.0 + 345.0 * pos
    D = np.clip(np.rint(mb * 1e6 / (5 * 384 * 384)), 128, 512).astype(int)
    return D, np.rint(total).astype(int)


class Img3dWorkload:
    name = "img3d"
    B = 2

    def __init__(self, L, ctx, pool: int, host: bool, seed: int, heavy_frac: float = 0.0,
                 time_scale_us_per_ms: float = 0.0, p_fg: float = 0.0, depths=None, zoom=None):
        self.L, self.ctx, self.seed, self.host = L, ctx, seed, host
        self.D, self.cost_ms = img_seg_dims(pool, seed)
        if depths is not None:                    # explicit volume depths (parity tests)
            self.D = np.asarray(depths, dtype=int)[:pool]
        self.pool = pool
        self.bufs = []
        for i in range(pool):
            D = int(self.D[i])
            vox = D * 384 * 384
            pi = ctx.host_alloc(vox * 4) if host else ctx.device_alloc(vox * 4)
            pl = ctx.host_alloc(vox) if host else ctx.device_alloc(vox)
            ctx.synth_volume(seed, i, D, 384, 384, pi, pl, on_device=not host)
            self.bufs.append((pi, pl))
        self.pool_bytes = int(sum(int(d) * 384 * 384 * 5 for d in self.D))
        self.heavy_frac = heavy_frac
        self.scale = time_scale_us_per_ms
        self.p_fg = p_fg
        self.zoom = zoom
        self.chain = ctx.chain(L.img_seg_ops(spin_first=heavy_frac > 0, p_fg=p_fg, zoom=zoom))
        self.roof_chain = ctx.chain(L.img_seg_ops()) if heavy_frac > 0 else self.chain

    def descs(self, ids):
        L = self.L
        rng = np.random.default_rng(self.seed + 17)
        heavy = rng.random(max(ids) + 1 if ids else 1) < self.heavy_frac
        out = []
        for i in ids:
            k = i % self.pool
            spin = [int(self.cost_ms[k] * self.scale)] if heavy[i] else [0]
            pi, pl = self.bufs[k]
            out.append(L.sample_desc(i, (int(self.D[k]), 384, 384), pi, pl,
                                     src_kind=L.SRC_HOST_PINNED if self.host else L.SRC_DEVICE,
                                     spin_us=spin))
        return out

    def source(self, i):
        """(f32 image, u8 label) volumes of sample id i (for the oracle check)."""
        k = i % self.pool
        dims = (int(self.D[k]), 384, 384)
        vox = int(np.prod(dims))
        pi, pl = self.bufs[k]
        return (_read(self.ctx, pi, vox, np.float32, self.host).reshape(dims),
                _read(self.ctx, pl, vox, np.uint8, self.host).reshape(dims))

    @staticmethod
    def pool_bytes_of(pool: int, seed: int) -> int:
        return int(sum(int(d) * 384 * 384 * 5 for d in img_seg_dims(pool, seed)[0]))

    def close(self):
        f = self.ctx.host_free if self.host else self.ctx.device_free
        for pi, pl in self.bufs:
            f(pi)
            f(pl)


class SpeechWorkload:
    """C4: 16 kHz utterances, L ~ U{30000..170000}; three sines + N(0, 0.01) noise.
    pcm16 (the default C4 input): int16 PCM -- the reference's speech bytes_in of
    60k-340k B (2 B per sample, workloads.cpp:115) -- quantised from the f32 synth as
    round(20000 x) and read by the kernel as s / 32768; else f32 samples."""
    name = "speech"
    B = 64
    PCM_SCALE = 20000.0

    def __init__(self, L, ctx, pool: int, host: bool, seed: int, lens=None, pcm16: bool = True):
        self.L, self.ctx, self.host, self.pcm16 = L, ctx, host, pcm16
        rng = np.random.default_rng(seed)
        self.lens = rng.integers(30000, 170001, size=pool)
        if lens is not None:                      # explicit lengths (parity tests)
            self.lens = np.asarray(lens, dtype=int)[:pool]
        self.esize = 2 if pcm16 else 4
        offs = np.concatenate([[0], np.cumsum([(int(n) * self.esize + 255) // 256 * 256 for n in self.lens])])
        self.offs = offs
        total = int(offs[-1])
        self.base = ctx.host_alloc(total) if host else ctx.device_alloc(total)
        if pcm16:
            tmp = ctx.device_alloc(4 * int(max(self.lens)))
            try:
                for i, n in enumerate(self.lens):
                    ctx.synth_waveform(seed, i, int(n), tmp, on_device=True)
                    x = _read(ctx, tmp, int(n), np.float32, False)
                    pcm = np.clip(np.rint(x.astype(np.float64) * self.PCM_SCALE), -32768, 32767).astype(np.int16)
                    self._write(self.base + int(offs[i]), pcm)
            finally:
                ctx.device_free(tmp)
        else:
            for i, n in enumerate(self.lens):
                ctx.synth_waveform(seed, i, int(n), self.base + int(offs[i]), on_device=not host)
        self.pool = pool
        self.pool_bytes = total
        self.chain = ctx.chain(L.speech_ops(pcm16=pcm16))

    def _write(self, ptr: int, arr: np.ndarray):
        if self.host:
            import ctypes
            ctypes.memmove(ptr, arr.ctypes.data, arr.nbytes)
        else:
            self.ctx.h2d(ptr, arr)

    def descs(self, ids):
        L = self.L
        return [L.sample_desc(i, (int(self.lens[i % self.pool]),), self.base + int(self.offs[i % self.pool]),
                              src_kind=L.SRC_HOST_PINNED if self.host else L.SRC_DEVICE) for i in ids]

    def source(self, i):
        """f32 waveform of sample id i (for the oracle check; PCM as its exact f32 image s / 32768)."""
        k = i % self.pool
        if self.pcm16:
            pcm = _read(self.ctx, self.base + int(self.offs[k]), int(self.lens[k]), np.int16, self.host)
            return (pcm.astype(np.float32) / np.float32(32768.0),)
        return (_read(self.ctx, self.base + int(self.offs[k]), int(self.lens[k]), np.float32, self.host),)

    @staticmethod
    def pool_bytes_of(pool: int, seed: int, esize: int = 2) -> int:
        lens = np.random.default_rng(seed).integers(30000, 170001, size=pool)
        return int(sum((int(n) * esize + 255) // 256 * 256 for n in lens))

    def close(self):
        (self.ctx.host_free if self.host else self.ctx.device_free)(self.base)


def pool_size(workload: str, host: bool, pool_arg: int = 0) -> int:
    if pool_arg:
        return pool_arg
    if workload.startswith("speech"):
        return 512
    if workload == "rrc":
        return 1024
    # device pools: 48 volumes, so the touched crop windows (48 x 10.5 MB) exceed the
    # 126 MB L2; pinned-host pools stay at 12 (every window crosses PCIe anyway)
    return 12 if host else 48


def make_context(L, workload: str, device: int = 0, workers: int = 16, group: int = 0, seed: int = 1):
    """The shard context bench.py measures: batch size and launch group of the
    workload, `workers` in-flight launch groups, enough output slot buffers for every
    in-flight group plus the batches being consumed.  Returns (ctx, B, group)."""
    B = BATCH[workload][0]
    group = group or BATCH[workload][1]
    slots = max(8, -(-workers * group // B) + 4)
    ctx = L.Context(device=device, batch_size=B, n_workers=workers, max_group=group,
                    max_slot_buffers=slots, seed=seed)
    return ctx, B, group


def make_workload(name, L, ctx, host, seed, args):
    pool = pool_size(name, host, args.pool)
    if name == "speech":        # int16 PCM input, the reference's speech bytes_in
        return SpeechWorkload(L, ctx, pool=pool, host=host, seed=seed, pcm16=True)
    if name == "speech_f32":    # the same utterances as f32 samples
        return SpeechWorkload(L, ctx, pool=pool, host=host, seed=seed, pcm16=False)
    if name == "rrc":
        return RrcWorkload(L, ctx, pool=pool, host=host, seed=seed)
    if name == "img3d":
        return Img3dWorkload(L, ctx, pool=pool, host=host, seed=seed)
    if name == "img3d_fg":   # MLPerf RandBalancedCrop: 40% of crops scan the label volume (K2)
        return Img3dWorkload(L, ctx, pool=pool, host=host, seed=seed, p_fg=0.4)
    if name == "img3d_zoom":    # north_star "trilinear resize": RandomZoom3D on every crop (K4)
        return Img3dWorkload(L, ctx, pool=pool, host=host, seed=seed, zoom=(1.0, 0.8, 1.2))
    if name == "img3d_heavy":   # the real tail (foreground oversampling); optional spin tail on top
        return Img3dWorkload(L, ctx, pool=pool, host=host, seed=seed, p_fg=args.fg,
                             heavy_frac=args.heavy_frac, time_scale_us_per_ms=args.time_scale)
    raise SystemExit(f"unknown workload {name}")


WORKLOAD_NAMES = {
    "rrc": "C2 ImageNet-shaped u8 3x(256..512)^2 -> RRC224+hflip+normalize",
    "img3d": "C1 KiTS19-shaped 3D crop128^3+flip+brightness+noise+cast",
    "img3d_fg": "C1 shapes, RandomCrop with MLPerf foreground oversampling 0.4 (K2 label scan + K1)",
    "img3d_zoom": "C1 shapes with RandomZoom3D (p 1, f in [0.8, 1.2]: window round(128 f), trilinear back to 128^3)",
    "img3d_heavy": "C3 heavy-tailed 3D (MLPerf foreground oversampling 0.4 as the tail) + synthetic "
                   "trainer at 90% of loader capacity",
    "speech": "C4 speech 16 kHz int16 PCM L~U{30k..170k} -> STFT (warp-per-frame fp32 real FFT) + log-mel + SpecAugment + splice, batch 64",
    "speech_f32": "C4 speech 16 kHz f32 samples L~U{30k..170k} -> STFT (warp-per-frame fp32 real FFT) + log-mel + SpecAugment + splice, batch 64",
}


def workers_of(args) -> int:
    """In-flight launch groups: 16, or 4 for C3 (64 samples in flight, so head-of-line
    blocking is not hidden behind a deep window)."""
    return args.workers or (4 if args.workload == "img3d_heavy" else 16)


def bench_config(args, world: int) -> dict:
    """The `config` object of the JSON line -- identical for both arms (--impl)."""
    wl = args.workload
    cls = {"rrc": RrcWorkload, "speech": SpeechWorkload, "speech_f32": SpeechWorkload}.get(wl, Img3dWorkload)
    extra = {"esize": 4} if wl == "speech_f32" else {}
    return {"workload": WORKLOAD_NAMES[wl], "batch": BATCH[wl][0],
            "launch_group": args.group or BATCH[wl][1], "workers": workers_of(args),
            "raw_pool_bytes": cls.pool_bytes_of(pool_size(wl, False, args.pool), args.seed, **extra),
            "l2": "inputs > L2 (pool larger than 126 MB)",
            "parallelism": f"dp{world} independent loader shards",
            **({"trainer": "synthetic step per batch calibrated to 90% of the loader capacity measured "
                           "in a drain run (trainer.hpp:14-21 consumer model)",
                "fg": args.fg} if wl == "img3d_heavy" else {})}


# ------------------------------------------------------------------ runs
def run_timed(L, ctx, wl, ids_warm, ids_timed, args, dist, local, trainer_us=0, policy=0,
              t_out_us=0, d2h_probe=0, capture=None, stream=False):
    """Warm-up run, then the timed run (`ids_timed` through lfg_run_shard); the
    delivered outputs of the feed positions in `capture` are copied out of their
    batch tensors on the trainer stream (counted in d2h_bytes) for the oracle check."""
    B = wl.B
    rc_w = L.run_config(batch_size=B, t_out_us=t_out_us, policy=policy, trainer_us=trainer_us,
                        n_workers=workers_of(args), warmup_us=args.profiler_warmup_us,
                        update_interval_us=1000, d2h_probe=d2h_probe)
    if ids_warm:
        ctx.run_shard(wl.chain, wl.descs(ids_warm), rc_w, want_ids=False)
    ctx.synchronize()
    barrier(dist)
    c0 = ctx.counters()
    descs = wl.descs(ids_timed)
    t0 = time.perf_counter()
    if stream:
        # through the public streaming API: this loop is the trainer -- it receives
        # each sealed batch (lfg_shard_next_batch) and hands it back (lfg_batch_release)
        st = ctx.shard_stream(wl.chain, descs, rc_w, capture=capture)
        for b, _ in st:
            ctx.batch_release(b)
        rep, ids, bsz, cls = st.finish()
    else:
        rep, ids, bsz, cls = ctx.run_shard(wl.chain, descs, rc_w, capture=capture)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    barrier(dist)
    c1 = ctx.counters()
    cap = dict(getattr(ctx, "last_capture", {})) if capture else {}
    return rep, ids, wall, {k: c1[k] - c0[k] for k in c1}, cap


def calibrated_trainer_us(L, ctx, wl, ids, args, util: float = 0.9) -> int:
    """C3's consumer: the loader's capacity R (samples/s) from a drain run (no trainer
    step, no timeout) over `ids`; the synthetic step per batch of B is B / (util * R),
    so the loader runs at `util` of its capacity (trainer.hpp:14-21 consumer model),
    refined with the trainer running beside the loader (below)."""
    rc = L.run_config(batch_size=wl.B, n_workers=workers_of(args))
    rep, *_ = ctx.run_shard(wl.chain, wl.descs(ids), rc, want_ids=False)
    ctx.synchronize()
    t = max(1, int(round(wl.B / (util * rep.samples_per_s) * 1e6)))
    # The trainer's step is a kernel on the same GPU, so the loader's capacity while it
    # runs is lower than the drain run's: re-measure with the trainer in place and re-aim
    # at `util` of what the loader then delivers (two fixed-point steps; the trainer only
    # ever slows down, so the pipeline stays loader-bound at most at that utilisation).
    for _ in range(2):
        rc_t = L.run_config(batch_size=wl.B, n_workers=workers_of(args), trainer_us=t)
        rep, *_ = ctx.run_shard(wl.chain, wl.descs(ids), rc_t, want_ids=False)
        ctx.synchronize()
        if rep.consumer_idle_frac < 0.02:
            break
        t = max(t, int(round(wl.B / (util * rep.samples_per_s) * 1e6)))
    return t


def capture_positions(n_timed: int, k: int, seed: int) -> list[int]:
    """k feed positions among the first 60% of the timed run (their batches are
    delivered while the rest of the run is still in flight)."""
    rng = np.random.default_rng(seed + 99)
    hi = max(1, int(0.6 * n_timed))
    return sorted(int(x) for x in rng.choice(hi, size=min(k, hi), replace=False))


def oracle_check(wl, ids_timed, cap) -> dict:
    """Verification leg (after the timed region): the captured delivered samples
    against the CPU oracle (oracle/checks.py; the oracle is the checker only)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import checks
    import lf_oracle as O
    seed = wl.ctx.cfg.seed
    worst, n = 0.0, 0
    for pos, (raw, _) in sorted(cap.items()):
        sid = int(ids_timed[pos])
        src = wl.source(sid)
        if wl.name == "rrc":
            r = checks.check_rrc(O, O.cfg2d(), seed, sid, src[0], raw)
        elif wl.name == "speech":
            r = checks.check_speech(O, O.cfgsp(), seed, sid, src[0], raw)
        else:
            zk = {}
            if getattr(wl, "zoom", None) is not None:
                zk = dict(has_zoom=1, p_zoom=wl.zoom[0], zoom_lo=wl.zoom[1], zoom_hi=wl.zoom[2])
            ocfg = O.cfg3d(has_fg=1 if wl.p_fg > 0 else 0, p_fg=wl.p_fg, **zk)
            r = checks.check_img3d(O, ocfg, seed, sid, src[0], src[1], raw, (128, 128, 128))
        worst = max(worst, r)
        n += 1
    return {"samples": n, "worst_err_over_bound": round(worst, 4), "ok": n > 0 and worst <= 1.0}


def traffic_of(workload: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/r2_traffic.json), or None when there is no capture for this workload."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            t = json.load(f).get(workload)
        return int(t["dram_read"] + t["dram_write"]) if t else None
    except Exception:
        return None


def kernel_roofline(L, ctx, wl, ids, hbm_peak, tf32_peak):
    """Dominant kernel alone: serial stream, device-resident inputs, CUDA events around
    every launch (the group's stage events); achieved = algorithmic bytes (or tensor
    FLOPs) / summed launch time."""
    chain = getattr(wl, "roof_chain", None) or wl.chain     # no synthetic spin stages
    ctx.time_kernels(chain, wl.descs(ids[: max(1, len(ids) // 4)]))   # warm-up pass (untimed)
    t = ctx.time_kernels(chain, wl.descs(ids))              # launches back to back, CUDA events
    launches = t["launches"]
    ms = t["mean_ms"] * launches                            # total transform-kernel time
    kernel = {"rrc": "rrc2d_kernel", "img3d": "img3d_tma_kernel", "speech": "speech_kernel"}[
        wl.name.split("_")[0]]
    if getattr(wl, "p_fg", 0) > 0:
        kernel = "fg_scan_kernel + img3d_tma_kernel (one stage)"
    if getattr(wl, "zoom", None) is not None:
        kernel = "img3d_zoom_kernel"
    out = {"kernel": kernel, "launches": int(launches), "mean_launch_us": round(1e3 * t["mean_ms"], 2),
           "traffic": traffic_of("zoom" if getattr(wl, "zoom", None) is not None else wl.name),
           "algo_bytes_per_launch": int(t["bytes"] / max(launches, 1))}
    if wl.name == "speech" and os.environ.get("LFG_SPEECH_KERNEL") == "tc":
        # the tcgen05 3xTF32 DFT-GEMM kernel (A/B switch): tensor-bound
        tf = t["flops"] / (ms / 1e3) / 1e12 if ms > 0 else 0.0
        out.update({"bound": "tensor", "achieved": round(tf, 1), "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": round(tf / tf32_peak, 4),
                    "flops_per_launch": int(t["flops"] / max(launches, 1)),
                    "hbm_gbs": round(t["bytes"] / (ms / 1e3) / 1e9, 1) if ms > 0 else 0.0})
    elif wl.name == "speech":
        # the FFT kernel (default): waveform read + spliced log-mel written, against HBM;
        # it is issue-bound (~12 k CUDA-core FLOPs per frame), so the HBM fraction is low.
        # dft_equiv: the 3xTF32 DFT-GEMM FLOPs the same work costs on the tensor cores
        gbs = t["bytes"] / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        out.update({"kernel": "speech_fft_kernel", "bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(gbs / hbm_peak, 4),
                    "dft_equiv_tflops": round(t["flops"] / (ms / 1e3) / 1e12, 1) if ms > 0 else 0.0})
    else:
        gbs = t["bytes"] / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        out.update({"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(gbs / hbm_peak, 4)})
    return out


def ref_harness():
    p = os.path.join(ROOT, "oracle", "_ref", "minato_cpu")
    return p if os.path.exists(p) else None


def cpu_baseline(workload: str, seconds: float = 12.0, steps: int = 0, warmup: int = 2):
    """Reported CPU baseline on this host's cores: the reference CPU loader
    (oracle/_ref/minato_cpu: reference libloadflow + oracle transforms) when it
    was built, else the oracle port alone on a thread pool.  Bounded sample."""
    cores = os.cpu_count() or 1
    h = ref_harness()
    wl = {"rrc": "rrc", "speech": "speech", "speech_f32": "speech"}.get(workload, "img3d")
    if h and wl != "speech" and workload != "img3d_zoom":   # (the reference harness has no zoom op)
        k = steps or (8 if wl == "rrc" else 10)
        fg = ["--fg", "0.4"] if workload == "img3d_fg" else []
        out = subprocess.run([h, "--workload", wl, "--steps", str(k), "--warmup", str(warmup),
                              "--workers", str(cores), "--max-seconds", "150"] + fg,
                             capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
        b = json.loads(out)
        return {"value": b["value"], "unit": "samples/s", "cores": b["cores"], "kind": "reference",
                "sample": b["sample"] + f"; timed {b['samples']:.0f} samples over {b['span_ms']:.0f} ms"}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lf_oracle as O
    from concurrent.futures import ThreadPoolExecutor
    rng = np.random.default_rng(5)
    if wl == "rrc":
        cfg = O.cfg2d()
        imgs = [rng.integers(0, 256, (int(h_), int(w_), 3), dtype=np.uint8)
                for h_, w_ in rng.integers(256, 513, size=(32, 2))]

        def one(i):
            O.chain2d(cfg, 1, i, imgs[i % len(imgs)])
        sample = "RandomResizedCrop224+flip+normalize on 3x(256..512)^2 u8 images"
    else:
        cfg = O.cfg3d(**(dict(has_zoom=1, p_zoom=1.0, zoom_lo=0.8, zoom_hi=1.2) if workload == "img3d_zoom" else {}))
        vols = [(rng.standard_normal((128, 384, 384)).astype(np.float32),
                 rng.integers(0, 3, (128, 384, 384), dtype=np.uint8)) for _ in range(2)]

        def one(i):
            v = vols[i % len(vols)]
            O.chain3d(cfg, 1, i, v[0], v[1])
        sample = ("crop128^3+" + ("zoom(0.8..1.2, trilinear)+" if workload == "img3d_zoom" else "") +
                  "flip+brightness+noise+cast on 128x384x384 volumes")
    if wl == "speech":
        cfg = O.cfgsp()
        waves = [(0.3 * rng.standard_normal(int(n))).astype(np.float32)
                 for n in rng.integers(30000, 170001, size=8)]

        def one(i):
            O.chainsp(cfg, 1, i, waves[i % len(waves)])
        sample = "STFT(512/320/160)+80 slaney mels+log+SpecAugment on 30k..170k-sample utterances"
    done = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(cores) as ex:
        while time.perf_counter() - t0 < seconds:
            list(ex.map(one, range(done, done + cores)))
            done += cores
    el = time.perf_counter() - t0
    return {"value": round(done / el, 2), "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{done} samples of {sample} in {el:.1f} s (oracle, fp64, {cores} threads)"}


def reference_arm(args):
    """--impl reference: the reference's own CPU loader on all host cores (rank 0 only;
    the other ranks of a torchrun launch exit 0 without work)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = args.workload
    B = BATCH[wl][0]
    base = cpu_baseline(wl, seconds=max(5.0, min(60.0, 2.0 * args.steps)), steps=args.steps,
                        warmup=args.warmup)
    v = base["value"]
    line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * B / v, 3) if v else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(args, args.gpus),
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": base["cores"],
                             "kind": base["kind"], "sample": base["sample"]},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure(args, rank: int, local: int, world: int, dist) -> dict:
    """One rank's shard: the resident-input run (value), the roofline pass, the
    pinned-host run (e2e), and the oracle check of samples captured from both runs."""
    from paper_2509_10712_b200 import lfgpu as L
    hbm_peak, tf32_peak, peak_src = peaks()
    ctx, B, group = make_context(L, args.workload, device=local, workers=workers_of(args),
                                 group=args.group, seed=args.seed)
    ids_all = shard_ids(args.warmup + args.steps, B, rank, world)
    ids_warm, ids_timed = ids_all[: args.warmup * B], ids_all[args.warmup * B:]
    heavy = args.workload == "img3d_heavy"
    trainer_us = args.trainer_us
    cap_pos = capture_positions(len(ids_timed), args.check, args.seed + rank) if args.check else None
    out = {"group": group}
    if args.serial:
        ctx.set_serial(True)

    # ---- value: inputs resident in HBM
    wl = make_workload(args.workload, L, ctx, host=False, seed=args.seed, args=args)
    if heavy and not args.trainer_us:
        trainer_us = calibrated_trainer_us(L, ctx, wl, ids_all, args)
    out["trainer_us"] = {"value": trainer_us}
    # the dominant kernel alone first (untimed for the value; it also brings the GPU and
    # the host path up to speed before the timed runs)
    out["roof"] = dict(kernel_roofline(L, ctx, wl, ids_timed[: min(len(ids_timed), 64 * B if B > 2 else 64)],
                                       hbm_peak, tf32_peak), peak_source=peak_src)
    with ClockSampler(local) as clk:
        rep, ids, wall, dc, cap = run_timed(L, ctx, wl, ids_warm, ids_timed, args, dist, local,
                                            trainer_us=trainer_us, policy=1 if heavy else 0,
                                            capture=cap_pos)
    out["clocks"] = clk.summary()
    if os.environ.get("LFG_BENCH_DIAG"):
        print(json.dumps({"diag": {"elapsed_ms": rep.elapsed_ms, "wall_s": wall, "kernel_ms": rep.kernel_ms,
                                   "launches": rep.launches, "batches": rep.batches,
                                   "inplace": rep.inplace_batches}}), file=sys.stderr, flush=True)
    out["check_value"] = oracle_check(wl, ids_timed, cap) if cap_pos and rank == 0 else None
    if not heavy:
        # the same resident run with MinatoLoader's timeout machinery live: the Profiler's
        # adaptive p75 / p90 budget over device-timed per-sample totals (policy 1), stage
        # events timed -- what the fast / slow classification costs the headline path
        rep_t, *_ = run_timed(L, ctx, wl, ids_warm, ids_timed, args, dist, local, trainer_us=0, policy=1)
        out["value_timeouts"] = rep_t.timed_samples / (rep_t.elapsed_ms / 1e3) if rep_t.elapsed_ms > 0 else None
        out["timeouts_slow"] = rep_t.slow / max(1, rep_t.samples)
        out["timeouts_t_out_us"] = rep_t.final_t_out_us
    out["pool_bytes"] = int(wl.pool_bytes)
    wl.close()

    # ---- e2e: inputs in pinned host memory, H2D + a D2H read of every delivered batch
    wl_h = make_workload(args.workload, L, ctx, host=True, seed=args.seed, args=args)
    trainer_h = trainer_us
    if heavy and not args.trainer_us:
        trainer_h = calibrated_trainer_us(L, ctx, wl_h, ids_all, args)
    out["trainer_us"]["e2e"] = trainer_h
    rep_h, ids_h, wall_h, dc_h, cap_h = run_timed(L, ctx, wl_h, ids_warm, ids_timed, args, dist, local,
                                                  trainer_us=trainer_h, policy=1 if heavy else 0,
                                                  d2h_probe=1, capture=cap_pos, stream=trainer_h == 0)
    out["check_e2e"] = oracle_check(wl_h, ids_timed, cap_h) if cap_pos and rank == 0 else None
    out["e2e_idle"] = rep_h.consumer_idle_frac if trainer_h else None
    out["e2e_slow"] = rep_h.slow / max(1, rep_h.samples)
    if heavy:
        # the synchronous head-of-line loader on the same stream, trainer and workers
        # (start_sync_loader, baselines.cpp:12-151; lfg_run_config.policy 3)
        rep_s, *_ = run_timed(L, ctx, wl_h, ids_warm, ids_timed, args, dist, local,
                              trainer_us=trainer_h, policy=3, d2h_probe=1)
        out["sync_e2e_idle"] = rep_s.consumer_idle_frac
        out["sync_e2e_value"] = rep_s.timed_samples / (rep_s.elapsed_ms / 1e3)
    wl_h.close()
    ctx.close()
    consumed = ids.tolist()
    out.update(elapsed_ms=rep.elapsed_ms, timed_samples=rep.timed_samples, e2e_elapsed_ms=rep_h.elapsed_ms,
               e2e_samples=rep_h.timed_samples, h2d=rep_h.h2d_bytes, d2h=rep_h.d2h_bytes,
               launches=dc["launches"], idle=rep.consumer_idle_frac if trainer_us else None,
               samples=rep.samples, fast=rep.fast, slow=rep.slow,
               dups=int(len(consumed) - len(set(consumed))) + rep.duplicates,
               digest=id_digest(consumed), digest_e2e=id_digest(ids_h.tolist()), wall=wall)
    return out


def fake_measure(args, rank: int, local: int, world: int, dist) -> dict:
    """TEST HOOK (LFG_BENCH_FAKE_SHARD=1, CPU tests of the multi-rank plumbing only):
    stands in for measure() without a GPU -- each rank "delivers" exactly its
    partition's timed ids; the line it produces carries "fake_shard": true."""
    B = BATCH[args.workload][0]
    ids_all = shard_ids(args.warmup + args.steps, B, rank, world)
    ids_timed = ids_all[args.warmup * B:]
    if os.environ.get("LFG_BENCH_FAKE_SHARD") == "dup" and rank == world - 1:
        ids_timed = ids_timed[:-1] + ids_timed[:1]      # one id lost, one delivered twice
    return {"group": args.group or BATCH[args.workload][1], "clocks": {"sm_mhz": None, "reasons": ["fake"]},
            "check_value": None, "check_e2e": None, "roof": None, "pool_bytes": 0,
            "elapsed_ms": 1.0 + rank, "timed_samples": len(ids_timed), "e2e_elapsed_ms": 2.0 + rank,
            "e2e_samples": len(ids_timed), "h2d": 0, "d2h": 0, "launches": 0, "idle": None,
            "samples": len(ids_timed), "fast": len(ids_timed), "slow": 0,
            "dups": len(ids_timed) - len(set(ids_timed)),
            "digest": id_digest(ids_timed), "digest_e2e": id_digest(ids_timed), "wall": 0.0}


def other_workloads(args) -> dict:
    """The other SURVEY 8(d) configurations, each measured by this same script in its own
    process (default steps, oracle check of 8 delivered samples) after the headline run,
    so the driver's N=1 record carries C1, C1-fg, C3, C4 and C1 with RandomZoom3D next to C2."""
    out = {}
    for wl in ("img3d", "img3d_fg", "img3d_heavy", "speech", "speech_f32", "img3d_zoom"):
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--workload", wl, "--no-cpu-baseline",
                                "--no-dropin", "--no-others", "--seed", str(args.seed)],
                               capture_output=True, text=True, timeout=240)
            d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
            roof = d.get("roofline") or {}
            out[wl] = {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"],
                       "steps": d["steps"], "ms_per_step": d["ms_per_step"], "e2e": d["e2e"]["value"],
                       "roofline": {k: roof.get(k) for k in ("kernel", "bound", "mean_launch_us", "achieved", "unit", "frac")},
                       "checked": d.get("checked"), "exactly_once": d.get("exactly_once"),
                       "clocks": d.get("clocks")}
            for k in ("consumer_idle_pct", "e2e_consumer_idle_pct", "sync_e2e_consumer_idle_pct", "trainer_us_per_batch"):
                if d.get(k) is not None:
                    out[wl][k] = d[k]
        except Exception as e:   # reported, never fatal for the headline line
            out[wl] = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    return out


def dropin_arm():
    """Throughput of the DROP-IN C++ path on the same C2 workload: the reference's own
    realtime Minato wiring (process_sample worker threads, resume, build_batches,
    run_consumer) over our headers, every process_sample submitting through the C ABI,
    concurrent workers' samples coalesced into shared launch groups
    (`loadflow_b200 dropin`, host/lf_dropin.cpp).  Host clock over the whole run."""
    exe = os.path.join(ROOT, "paper_2509_10712_b200", "loadflow_b200")
    try:
        r = subprocess.run([exe, "dropin", "--workers", "32", "--coalesce-us", "150", "--samples", "20480",
                            "--batch", "256", "--group", "64", "--max-seconds", "60"],
                           capture_output=True, text=True, timeout=90)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:   # reported, never fatal for the headline line
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    return {k: d[k] for k in ("path", "value", "unit", "workers", "coalesce_us", "max_group", "samples",
                              "samples_per_launch", "exactly_once")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0, help="timed batches (0 = workload default)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="rrc", choices=list(BATCH))
    ap.add_argument("--pool", type=int, default=0)
    ap.add_argument("--workers", type=int, default=0, help="in-flight launch groups (0 = 16; C3: 4)")
    ap.add_argument("--fg", type=float, default=0.4, help="img3d_heavy: foreground oversampling probability")
    ap.add_argument("--group", type=int, default=0, help="samples per launch group (0 = auto)")
    ap.add_argument("--heavy-frac", type=float, default=0.0, help="img3d_heavy: extra synthetic spin tail")
    ap.add_argument("--time-scale", type=float, default=10.0, help="spin us per reference ms")
    ap.add_argument("--trainer-us", type=int, default=0)
    ap.add_argument("--profiler-warmup-us", type=int, default=20000)
    ap.add_argument("--check", type=int, default=8, help="delivered samples checked against the oracle")
    ap.add_argument("--serial", action="store_true", help="(experiment) all launch groups on one stream")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true", help="skip the drop-in C++ path measurement")
    ap.add_argument("--no-others", action="store_true", help="(rrc, N=1) skip the other workloads' sub-runs")
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.steps <= 0:
        args.steps = BATCH[args.workload][2]

    rc = launch_ranks(args)          # --gpus N without a launcher: one process per GPU
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        reference_arm(args)
        return

    rank, local, world, dist = dist_setup(args.gpus)
    fake = os.environ.get("LFG_BENCH_FAKE_SHARD") in ("1", "dup")
    r = (fake_measure if fake else measure)(args, rank, local, world, dist)
    B = BATCH[args.workload][0]

    # the run's only collectives: max of the device-timed spans, one counter reduce
    el_max = allreduce_max(dist, r["elapsed_ms"], local)
    el_h = allreduce_max(dist, r["e2e_elapsed_ms"], local)
    cnt = allreduce_sum(dist, [r["timed_samples"], r["e2e_samples"], r["samples"], r["fast"], r["slow"],
                               r["dups"], r["launches"], r["h2d"], r["d2h"]], local)
    dig = allreduce_sum_i64(dist, r["digest"] + r["digest_e2e"], local)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    # exactly-once over the union of the shards (experiment.cpp:396-413): the timed
    # ids of all ranks are batches warmup*world .. (warmup+steps)*world - 1
    want = id_digest(range(args.warmup * world * B, (args.warmup + args.steps) * world * B))
    exactly_once = dig[:4] == want and dig[4:] == want and cnt[5] == 0
    value = cnt[0] / (el_max / 1e3)
    e2e = cnt[1] / (el_h / 1e3)
    # the CPU baseline and the drop-in arm: rank 0 at N = 1 only (the scaling runs report GPU shards)
    cpu = None if (args.no_cpu_baseline or fake or world > 1) else cpu_baseline(args.workload)
    dropin = dropin_arm() if (args.workload == "rrc" and world == 1 and not fake and not args.no_dropin) else None
    steps = args.steps
    checks = [c for c in (r["check_value"], r["check_e2e"]) if c is not None]
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "samples/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": round(el_max / steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Philox(seed,id) images/volumes generated on device / pinned host)",
        "config": bench_config(args, world),
        "roofline": r["roof"],
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e, 1), "unit": "samples/s",
                "h2d_bytes_per_step": int(cnt[7] / max(1, steps)),     # whole job (all ranks)
                "d2h_bytes_per_step": int(cnt[8] / max(1, steps))},
        "clocks": r["clocks"],
        "gpu_launches": int(cnt[6]),
        "consumer_idle_pct": round(100 * r["idle"], 2) if r["idle"] is not None else None,
        **({"e2e_consumer_idle_pct": round(100 * r["e2e_idle"], 2),
            "sync_e2e_consumer_idle_pct": round(100 * r["sync_e2e_idle"], 2),
            "sync_e2e_value": round(r["sync_e2e_value"], 1),
            "e2e_slow_frac": round(r["e2e_slow"], 4),
            "trainer_us_per_batch": r["trainer_us"]} if r.get("sync_e2e_idle") is not None else {}),
        "slow_frac": round(cnt[4] / max(1, cnt[2]), 4),
        "exactly_once": bool(exactly_once),
        "checked": bool(checks) and all(c["ok"] for c in checks),
        "check": {"value_run": r["check_value"], "e2e_run": r["check_e2e"]},
        "wall_s": round(r["wall"], 3),
    }
    if r.get("value_timeouts") is not None:
        # rank-local figures of the extra run (rank 0's shard)
        line["value_with_timeouts"] = {"value": round(r["value_timeouts"] * world, 1), "unit": "samples/s",
                                       "policy": "profiler p75 -> p90 (adaptive)",
                                       "slow_frac": round(r["timeouts_slow"], 4),
                                       "final_t_out_us": round(r["timeouts_t_out_us"], 1)}
    if dropin is not None:
        line["dropin"] = dropin
    if args.workload == "rrc" and world == 1 and not fake and not args.no_others:
        if dist is not None:
            dist.destroy_process_group()
            dist = None
        line["other_workloads"] = other_workloads(args)
    if fake:
        line["fake_shard"] = True
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
