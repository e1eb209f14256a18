"""ctypes binding of liblfgpu.so (include/lfgpu.h).

The product path: every call goes to the in-tree CUDA library.  There is no
CPU fallback -- importing this module raises if liblfgpu.so is missing, and
opening a context raises if no GPU is visible.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Iterable, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# LFG_LIB: an alternative build of the same library (A/B experiments: tools/kernel_sweep.py)
LIB_PATH = os.environ.get("LFG_LIB") or os.path.join(_PKG, "liblfgpu.so")
HEADER_PATH = os.path.join(os.path.dirname(_PKG), "include", "lfgpu.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# ---- constants (mirror lfgpu.h) -------------------------------------------------
LFG_OK = 0
ERRORS = {-1: "LFG_ERR_INVALID", -2: "LFG_ERR_STATE", -3: "LFG_ERR_CLOSED", -4: "LFG_ERR_AGAIN",
          -5: "LFG_ERR_CUDA", -6: "LFG_ERR_NOMEM", -7: "LFG_ERR_UNSUPPORTED"}
ERR_INVALID, ERR_STATE, ERR_CLOSED, ERR_AGAIN, ERR_CUDA, ERR_NOMEM, ERR_UNSUPPORTED = (
    -1, -2, -3, -4, -5, -6, -7)

OP_RANDOM_CROP, OP_RANDOM_FLIP, OP_RANDOM_BRIGHTNESS, OP_GAUSSIAN_NOISE, OP_CAST = 1, 2, 3, 4, 5
OP_RANDOM_ZOOM3D, OP_RANDOM_CONTRAST = 6, 7      # optional img_seg ops (not in the reference chain)
OP_RESIZE, OP_RANDOM_HFLIP, OP_TO_TENSOR, OP_NORMALIZE = 10, 11, 12, 13
OP_PAD, OP_SPEC_AUGMENT, OP_FILTER_BANK, OP_FRAME_SPLICING, OP_PERMUTE_AUDIO = 20, 21, 22, 23, 24
OP_SPIN = 30
DT_U8, DT_I16, DT_F32 = 1, 2, 3
SRC_DEVICE, SRC_HOST_PINNED = 0, 1
FAM_IMG3D, FAM_RRC2D, FAM_SPEECH = 1, 2, 3


class LfgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("barrier", C.c_int32), ("size_factor", C.c_double),
                ("param", C.c_double * 8), ("name", C.c_char * 32)]


class SampleDesc(C.Structure):
    _fields_ = [("id", C.c_uint64), ("src_kind", C.c_int32), ("ndim", C.c_int32),
                ("dims", C.c_int64 * 4), ("data", C.c_void_p), ("aux", C.c_void_p),
                ("spin_us", C.c_int64 * 4)]


class Config(C.Structure):
    _fields_ = [("device", C.c_int32), ("n_workers", C.c_int32), ("max_group", C.c_int32),
                ("batch_size", C.c_int32), ("max_slot_buffers", C.c_int32),
                ("coalesce_us", C.c_int32), ("seed", C.c_uint64), ("max_raw_bytes", C.c_int64)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "submitted", "completed", "fast", "slow", "batches", "short_batches", "inplace_batches",
        "gathered_batches", "launches", "h2d_bytes", "d2h_bytes", "kernel_bytes")] + [
        ("reserved", C.c_int64 * 4)]


_P_i64 = C.POINTER(C.c_int64)
_P_i32 = C.POINTER(C.c_int32)


class RunConfig(C.Structure):
    _fields_ = [("batch_size", C.c_int32), ("policy", C.c_int32), ("t_out_us", C.c_int64),
                ("warmup_us", C.c_int64), ("update_interval_us", C.c_int64),
                ("window", C.c_int32), ("n_workers", C.c_int32), ("trainer_us", C.c_int64),
                ("trainer_priority", C.c_int32), ("warmup_batches", C.c_int32),
                ("record_trace", C.c_int32), ("d2h_probe", C.c_int32), ("percentile", C.c_int32),
                ("scheduler", C.c_int32), ("max_workers", C.c_int32), ("sched_tick_us", C.c_int64),
                ("prefetch_factor", C.c_int32), ("n_capture", C.c_int32), ("sample_stamps", C.c_int32),
                ("capture_pos", _P_i64), ("capture_buf", C.c_void_p), ("capture_stride", C.c_int64),
                ("capture_done", _P_i32)]


class RunReport(C.Structure):
    _fields_ = [("samples", C.c_int64), ("batches", C.c_int64), ("short_batches", C.c_int64),
                ("fast", C.c_int64), ("slow", C.c_int64), ("inplace_batches", C.c_int64),
                ("elapsed_ms", C.c_double), ("timed_samples", C.c_double),
                ("samples_per_s", C.c_double), ("consumer_busy_ms", C.c_double),
                ("consumer_span_ms", C.c_double), ("consumer_idle_frac", C.c_double),
                ("final_t_out_us", C.c_double), ("final_percentile", C.c_int32),
                ("exactly_once", C.c_int32), ("duplicates", C.c_int64), ("kernel_ms", C.c_double),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("launches", C.c_int64),
                ("final_workers", C.c_int32), ("sched_ticks", C.c_int32), ("mean_workers", C.c_double),
                ("pct_up", C.c_int32), ("pct_down", C.c_int32), ("profiled", C.c_int64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = C.POINTER
_vp = C.c_void_p
_sig = {
    "lfg_last_error": ([], C.c_char_p),
    "lfg_abi_version": ([], C.c_int),
    "lfg_device_count": ([_P(C.c_int)], C.c_int),
    "lfg_config_default": ([_P(Config)], None),
    "lfg_open": ([_P(Config), _P(_vp)], C.c_int),
    "lfg_close": ([_vp], C.c_int),
    "lfg_synchronize": ([_vp], C.c_int),
    "lfg_host_alloc": ([_vp, C.c_size_t, _P(_vp)], C.c_int),
    "lfg_host_free": ([_vp, _vp], C.c_int),
    "lfg_device_alloc": ([_vp, C.c_size_t, _P(_vp)], C.c_int),
    "lfg_device_free": ([_vp, _vp], C.c_int),
    "lfg_memcpy_h2d": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "lfg_memcpy_d2h": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "lfg_chain_create": ([_vp, _P(Op), C.c_int, _P(_vp)], C.c_int),
    "lfg_chain_destroy": ([_vp, _vp], C.c_int),
    "lfg_chain_info": ([_vp, _P(C.c_int), _P(C.c_int64), _P(C.c_int)], C.c_int),
    "lfg_chain_stage": ([_vp, C.c_int, _P(C.c_int), _P(C.c_int)], C.c_int),
    "lfg_draw_params": ([_vp, C.c_uint64, _P(SampleDesc), _P(C.c_double), C.c_int,
                         _P(C.c_int)], C.c_int),
    "lfg_rng_outputs": ([C.c_uint64, C.c_uint64, C.c_int, _P(C.c_uint64)], C.c_int),
    "lfg_submit": ([_vp, _vp, _P(SampleDesc), _P(C.c_int64)], C.c_int),
    "lfg_flush": ([_vp], C.c_int),
    "lfg_progress": ([_vp, C.c_int64, _P(C.c_int), _P(C.c_int), _P(C.c_int64)], C.c_int),
    "lfg_wait": ([_vp, C.c_int64], C.c_int),
    "lfg_wait_for": ([_vp, C.c_int64, C.c_int64, _P(C.c_int)], C.c_int),
    "lfg_exec_costs": ([_vp, C.c_int64, _P(C.c_double), C.c_int, _P(C.c_int)], C.c_int),
    "lfg_ticket_output": ([_vp, C.c_int64, _vp, C.c_size_t], C.c_int),
    "lfg_ticket_release": ([_vp, C.c_int64], C.c_int),
    "lfg_seal_batch": ([_vp, _P(C.c_int64), C.c_int, _P(C.c_int64)], C.c_int),
    "lfg_batch_info": ([_vp, C.c_int64, _P(_vp), _P(C.c_int64), _P(C.c_int), _P(C.c_uint64),
                        _P(C.c_int)], C.c_int),
    "lfg_batch_wait_stream": ([_vp, C.c_int64, _vp], C.c_int),
    "lfg_batch_copy_to_host": ([_vp, C.c_int64, _vp, C.c_size_t], C.c_int),
    "lfg_batch_lengths": ([_vp, C.c_int64, _P(C.c_int32), _P(C.c_int32)], C.c_int),
    "lfg_batch_release": ([_vp, C.c_int64, _vp], C.c_int),
    "lfg_trainer_step": ([_vp, C.c_int64, _vp, C.c_int64], C.c_int),
    "lfg_synth_volume": ([_vp, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _vp, _vp,
                          C.c_int], C.c_int),
    "lfg_synth_image": ([_vp, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, _vp, C.c_int], C.c_int),
    "lfg_synth_waveform": ([_vp, C.c_uint64, C.c_uint64, C.c_int64, _vp, C.c_int], C.c_int),
    "lfg_get_counters": ([_vp, _P(Counters)], C.c_int),
    "lfg_set_serial": ([_vp, C.c_int], C.c_int),
    "lfg_time_kernels": ([_vp, _vp, _P(SampleDesc), C.c_int, _P(C.c_double), _P(C.c_int64),
                          _P(C.c_int64), _P(C.c_int64)], C.c_int),
    "lfg_run_shard": ([_vp, _vp, _P(SampleDesc), C.c_int64, _P(RunConfig), _P(RunReport),
                       _P(C.c_uint64), _P(C.c_int32), _P(C.c_int32)], C.c_int),
    "lfg_run_shard_source": ([_vp, _vp, _vp, C.c_int64, _P(RunConfig), _P(RunReport),
                              _P(C.c_uint64), _P(C.c_int32), _P(C.c_int32)], C.c_int),
    "lfg_shard_start": ([_vp, _vp, _P(SampleDesc), C.c_int64, _P(RunConfig), _P(_vp)], C.c_int),
    "lfg_shard_next_batch": ([_vp, C.c_int64, _P(C.c_int64), _P(C.c_int)], C.c_int),
    "lfg_shard_finish": ([_vp, _P(RunReport), _P(C.c_uint64), _P(C.c_int32), _P(C.c_int32)], C.c_int),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_sig)


def _check(rc: int):
    if rc != LFG_OK:
        raise LfgError(rc, _lib.lfg_last_error().decode(errors="replace"))


def rng_outputs(seed: int, sid: int, n: int) -> np.ndarray:
    """First n outputs of sample `sid`'s generator (host only)."""
    out = (C.c_uint64 * max(n, 1))()
    _check(_lib.lfg_rng_outputs(seed, sid, n, out))
    return np.array(out[:n], dtype=np.uint64)


def device_count() -> int:
    n = C.c_int(0)
    _check(_lib.lfg_device_count(C.byref(n)))
    return n.value


# ---- ops: names and size factors from the reference chains ------------------------
def op(kind: int, name: str, size_factor: float = 1.0, params: Sequence[float] = (),
       barrier: bool = False) -> Op:
    o = Op()
    o.kind = kind
    o.barrier = int(barrier)
    o.size_factor = size_factor
    for i, p in enumerate(params):
        o.param[i] = float(p)
    o.name = name.encode()[:31]
    return o


def img_seg_ops(crop=(128, 128, 128), p_flip=1 / 3, p_bright=0.1, bright=(0.7, 1.3),
                p_noise=0.1, noise_std_max=0.1, spin_first: bool = False,
                zoom=None, contrast=None, p_fg: float = 0.0) -> list[Op]:
    """img_seg chain, proj/src/workloads.cpp:142-148 (size factors included).

    Optional ops (north_star "trilinear resize" / "brightness/contrast"; not in the
    reference chain, so off by default): ``p_fg`` > 0 makes RandomCrop oversample the
    foreground with that probability (MLPerf RandBalancedCrop, kernel K2; from pinned
    host memory such samples stage their whole volume); ``zoom=(p, lo, hi)`` adds RandomZoom3D after
    RandomCrop (window edge round(crop * f), trilinear back to the crop; labels
    nearest); ``contrast=(p, lo, hi)`` adds RandomContrast after RandomBrightness."""
    ops = [op(OP_SPIN, "SampleCost")] if spin_first else []
    ops.append(op(OP_RANDOM_CROP, "RandomCrop", 0.0735, list(crop) + [p_fg]))
    if zoom is not None:
        ops.append(op(OP_RANDOM_ZOOM3D, "RandomZoom3D", 1.0, list(zoom)))
    ops += [
        op(OP_RANDOM_FLIP, "RandomFlip", 1.0, [p_flip]),
        op(OP_RANDOM_BRIGHTNESS, "RandomBrightness", 1.0, [p_bright, bright[0], bright[1]]),
    ]
    if contrast is not None:
        ops.append(op(OP_RANDOM_CONTRAST, "RandomContrast", 1.0, list(contrast)))
    ops += [
        op(OP_GAUSSIAN_NOISE, "GaussianNoise", 1.0, [p_noise, noise_std_max]),
        op(OP_CAST, "Cast", 1.0),
    ]
    return ops


IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


def obj_det_ops(out=(224, 224), scale=(0.08, 1.0), ratio=(3 / 4, 4 / 3), p_hflip=0.5,
                mean=IMAGENET_MEAN, std=IMAGENET_STD) -> list[Op]:
    """obj_det chain, proj/src/workloads.cpp:151-156 (Resize = RandomResizedCrop)."""
    return [
        op(OP_RESIZE, "Resize", 1.2, [out[0], out[1], scale[0], scale[1], ratio[0], ratio[1]]),
        op(OP_RANDOM_HFLIP, "RandomHorizontalFlip", 1.0, [p_hflip]),
        op(OP_TO_TENSOR, "ToTensor", 8.0),
        op(OP_NORMALIZE, "Normalize", 1.0, list(mean) + list(std)),
    ]


def speech_ops(max_len=170_000, freq_masks=2, freq_mask_max=27, time_masks=10,
               time_mask_frac=0.05, stack=3, pcm16=False) -> list[Op]:
    """speech chain, proj/src/workloads.cpp:103-108: Pad, SpecAugment, FilterBank
    (STFT 512/320/160 -> 80 slaney mels -> log), FrameSplicing, PermuteAudio.
    pcm16: the waveforms are int16 PCM (the reference's speech bytes_in, 2 B per
    sample, workloads.cpp:115), read as s / 32768; else f32."""
    ops = [
        op(OP_PAD, "Pad", 1.12),
        op(OP_SPEC_AUGMENT, "SpecAugment", 1.0, [freq_masks, freq_mask_max, time_masks, time_mask_frac]),
        op(OP_FILTER_BANK, "FilterBank", 1.0, [512, 320, 160, 80, max_len, DT_I16 if pcm16 else DT_F32]),
    ]
    if stack > 1:
        ops.append(op(OP_FRAME_SPLICING, "FrameSplicing", 0.9, [stack]))
    ops.append(op(OP_PERMUTE_AUDIO, "PermuteAudio", 1.0))
    return ops


def _arr_ptr(a) -> int:
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return int(a)


def sample_desc(sid: int, dims: Sequence[int], data, aux=None, src_kind=SRC_DEVICE,
                spin_us: Iterable[int] = ()) -> SampleDesc:
    d = SampleDesc()
    d.id = sid
    d.src_kind = src_kind
    d.ndim = len(dims)
    for i, v in enumerate(dims):
        d.dims[i] = int(v)
    d.data = _arr_ptr(data) if data is not None else None
    d.aux = _arr_ptr(aux) if aux is not None else None
    for i, v in enumerate(spin_us):
        d.spin_us[i] = int(v)
    return d


class Chain:
    def __init__(self, ctx: "Context", handle: int):
        self.ctx = ctx
        self.handle = handle

    def info(self):
        ns, ob, fam = C.c_int(), C.c_int64(), C.c_int()
        _check(_lib.lfg_chain_info(self.handle, C.byref(ns), C.byref(ob), C.byref(fam)))
        return ns.value, ob.value, fam.value

    def stages(self):
        out = []
        for s in range(self.info()[0]):
            a, b = C.c_int(), C.c_int()
            _check(_lib.lfg_chain_stage(self.handle, s, C.byref(a), C.byref(b)))
            out.append((a.value, b.value))
        return out

    def draw_params(self, seed: int, desc: SampleDesc) -> np.ndarray:
        buf = (C.c_double * 64)()
        n = C.c_int()
        _check(_lib.lfg_draw_params(self.handle, seed, C.byref(desc), buf, 64, C.byref(n)))
        return np.array(buf[: n.value])


class Context:
    """One GPU shard (lfg_ctx)."""

    def __init__(self, device=0, batch_size=24, n_workers=12, max_group=1, max_slot_buffers=8,
                 seed=1, coalesce_us=0):
        cfg = Config()
        _lib.lfg_config_default(C.byref(cfg))
        cfg.device, cfg.batch_size, cfg.n_workers = device, batch_size, n_workers
        cfg.max_group, cfg.max_slot_buffers, cfg.seed = max_group, max_slot_buffers, seed
        cfg.coalesce_us = coalesce_us
        self.cfg = cfg
        h = _vp()
        _check(_lib.lfg_open(C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            _check(_lib.lfg_close(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # memory
    def host_alloc(self, nbytes: int) -> int:
        p = _vp()
        _check(_lib.lfg_host_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def host_free(self, p: int):
        _check(_lib.lfg_host_free(self.h, p))

    def device_alloc(self, nbytes: int) -> int:
        p = _vp()
        _check(_lib.lfg_device_alloc(self.h, nbytes, C.byref(p)))
        return p.value

    def device_free(self, p: int):
        _check(_lib.lfg_device_free(self.h, p))

    def h2d(self, dst: int, src: np.ndarray):
        _check(_lib.lfg_memcpy_h2d(self.h, dst, src.ctypes.data, src.nbytes))

    def d2h(self, dst: np.ndarray, src: int):
        _check(_lib.lfg_memcpy_d2h(self.h, dst.ctypes.data, src, dst.nbytes))

    def synchronize(self):
        _check(_lib.lfg_synchronize(self.h))

    # chains
    def chain(self, ops: Sequence[Op]) -> Chain:
        arr = (Op * len(ops))(*ops)
        h = _vp()
        _check(_lib.lfg_chain_create(self.h, arr, len(ops), C.byref(h)))
        return Chain(self, h.value)

    def destroy_chain(self, ch: Chain):
        _check(_lib.lfg_chain_destroy(self.h, ch.handle))

    # samples
    def submit(self, ch: Chain, desc: SampleDesc) -> int:
        t = C.c_int64()
        _check(_lib.lfg_submit(self.h, ch.handle, C.byref(desc), C.byref(t)))
        return t.value

    def flush(self):
        _check(_lib.lfg_flush(self.h))

    def progress(self, t: int):
        od, cp, el = C.c_int(), C.c_int(), C.c_int64()
        _check(_lib.lfg_progress(self.h, t, C.byref(od), C.byref(cp), C.byref(el)))
        return od.value, bool(cp.value), el.value

    def wait_for(self, t: int, timeout_us: int) -> bool:
        """lfg_wait_for: True once the sample finished, False at the timeout."""
        done = C.c_int(0)
        _check(_lib.lfg_wait_for(self.h, t, timeout_us, C.byref(done)))
        return bool(done.value)

    def wait(self, t: int):
        _check(_lib.lfg_wait(self.h, t))

    def exec_costs(self, t: int, n_ops: int) -> np.ndarray:
        buf = (C.c_double * n_ops)()
        n = C.c_int()
        _check(_lib.lfg_exec_costs(self.h, t, buf, n_ops, C.byref(n)))
        return np.array(buf[: n.value])

    def ticket_output(self, t: int, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        _check(_lib.lfg_ticket_output(self.h, t, out.ctypes.data, nbytes))
        return out

    def release(self, t: int):
        _check(_lib.lfg_ticket_release(self.h, t))

    def seal(self, tickets: Sequence[int]) -> int:
        arr = (C.c_int64 * len(tickets))(*tickets)
        b = C.c_int64()
        _check(_lib.lfg_seal_batch(self.h, arr, len(tickets), C.byref(b)))
        return b.value

    def batch_info(self, b: int):
        p, nb, n, ip = _vp(), C.c_int64(), C.c_int(), C.c_int()
        ids = (C.c_uint64 * self.cfg.batch_size)()
        _check(_lib.lfg_batch_info(self.h, b, C.byref(p), C.byref(nb), C.byref(n), ids,
                                   C.byref(ip)))
        return {"ptr": p.value, "bytes": nb.value, "n": n.value, "ids": list(ids[: n.value]),
                "in_place": bool(ip.value)}

    def batch_to_host(self, b: int, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        _check(_lib.lfg_batch_copy_to_host(self.h, b, out.ctypes.data, nbytes))
        return out

    def batch_lengths(self, b: int):
        n = self.batch_info(b)["n"]
        lens = (C.c_int32 * n)()
        tm = C.c_int32()
        _check(_lib.lfg_batch_lengths(self.h, b, lens, C.byref(tm)))
        return list(lens), tm.value

    def batch_release(self, b: int, stream: int = 0):
        _check(_lib.lfg_batch_release(self.h, b, stream))

    def trainer_step(self, b: int, stream: int = 0, us: int = 0):
        _check(_lib.lfg_trainer_step(self.h, b, stream, us))

    def counters(self) -> dict:
        c = Counters()
        _check(_lib.lfg_get_counters(self.h, C.byref(c)))
        out = {f: getattr(c, f) for f, _ in Counters._fields_ if f != "reserved"}
        out["gather_bytes"] = c.reserved[0]      # collation (seal) kernel bytes
        out["tensor_flops"] = c.reserved[1]      # speech DFT GEMM flops (3xTF32 counted x3)
        return out

    # synthetic inputs
    def synth_volume(self, seed, sid, D, H, W, img_ptr, lbl_ptr, on_device=True):
        _check(_lib.lfg_synth_volume(self.h, seed, sid, D, H, W, img_ptr, lbl_ptr, int(on_device)))

    def synth_image(self, seed, sid, H, W, ptr, on_device=True):
        _check(_lib.lfg_synth_image(self.h, seed, sid, H, W, ptr, int(on_device)))

    def synth_waveform(self, seed, sid, L, ptr, on_device=True):
        _check(_lib.lfg_synth_waveform(self.h, seed, sid, L, ptr, int(on_device)))

    def time_kernels(self, ch: Chain, descs):
        arr = (SampleDesc * len(descs))(*descs)
        ms, nl, by, fl = C.c_double(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.lfg_time_kernels(self.h, ch.handle, arr, len(descs), C.byref(ms), C.byref(nl),
                                     C.byref(by), C.byref(fl)))
        return {"mean_ms": ms.value, "launches": nl.value, "bytes": by.value, "flops": fl.value}

    def set_serial(self, serial: bool):
        _check(_lib.lfg_set_serial(self.h, int(serial)))

    # whole shard
    def run_shard(self, ch: Chain, descs: Sequence[SampleDesc], rc: RunConfig,
                  want_ids: bool = True, capture: Sequence[int] | None = None):
        """lfg_run_shard.  ``capture``: feed positions whose delivered outputs are copied
        out of their batch tensors (lfg_run_config capture); they are returned as
        ``self.last_capture = {position: (uint8 array, batch index)}``."""
        n = len(descs)
        arr = (SampleDesc * n)(*descs)
        rep = RunReport()
        ids = (C.c_uint64 * max(n, 1))()
        bs = (C.c_int32 * max(n, 1))()
        cls = (C.c_int32 * max(n, 1))()
        cap = self._capture_begin(ch, rc, capture)
        try:
            _check(_lib.lfg_run_shard(self.h, ch.handle, arr, n, C.byref(rc), C.byref(rep),
                                      ids if want_ids else None, bs if want_ids else None,
                                      cls if want_ids else None))
            self._capture_collect(cap)
        finally:
            self._capture_end(rc, cap)
        nb = rep.batches
        return rep, np.array(ids[:n], dtype=np.uint64), np.array(bs[:nb]), np.array(cls[:n])

    # output capture of delivered samples (lfg_run_config capture fields)
    def _capture_begin(self, ch: Chain, rc: RunConfig, capture):
        if not capture:
            return None
        _, stride, _ = ch.info()
        stride = (stride + 255) // 256 * 256
        pos = (C.c_int64 * len(capture))(*capture)
        done = (C.c_int32 * len(capture))()
        buf = self.host_alloc(stride * len(capture))
        rc.n_capture, rc.capture_pos, rc.capture_buf = len(capture), pos, buf
        rc.capture_stride, rc.capture_done = stride, done
        return (list(capture), stride, pos, done, buf)

    def _capture_collect(self, cap):
        if cap is None:
            return
        capture, stride, _, done, buf = cap
        raw = np.ctypeslib.as_array((C.c_uint8 * (stride * len(capture))).from_address(buf))
        self.last_capture = {int(p): (raw[k * stride:(k + 1) * stride].copy(), int(done[k]) - 1)
                             for k, p in enumerate(capture) if done[k] > 0}

    def _capture_end(self, rc: RunConfig, cap):
        if cap is None:
            return
        rc.n_capture, rc.capture_pos, rc.capture_buf, rc.capture_done = 0, None, None, None
        self.host_free(cap[4])

    def shard_stream(self, ch: Chain, descs: Sequence[SampleDesc], rc: RunConfig,
                     capture: Sequence[int] | None = None) -> "ShardStream":
        """lfg_shard_start: the shard loop on a library thread; iterate the returned
        stream for sealed batches (the caller is the trainer and releases each one).
        ``capture`` as in run_shard (collected into ``last_capture`` by finish())."""
        return ShardStream(self, ch, descs, rc, capture)

    def run_shard_source(self, ch: Chain, src: "FileSource", rc: RunConfig):
        """lfg_run_shard_source: the shard pulls samples from a streaming source."""
        n = src.n
        rep = RunReport()
        ids = (C.c_uint64 * n)()
        bs = (C.c_int32 * n)()
        cls = (C.c_int32 * n)()
        _check(_lib.lfg_run_shard_source(self.h, ch.handle, C.addressof(src.src), n, C.byref(rc), C.byref(rep),
                                         ids, bs, cls))
        return rep, np.array(ids[:n], dtype=np.uint64), np.array(bs[:rep.batches]), np.array(cls[:n])


class ShardStream:
    """A streaming shard run (lfg_shard_start / lfg_shard_next_batch / lfg_shard_finish):
    ``next_batch()`` returns ``(batch, n)``, ``None`` at the end of the stream; the batch
    is the caller's until ``ctx.batch_release(batch, stream)``.  ``finish()`` returns
    ``(report, consumed ids, batch sizes, sample classes)`` as ``Context.run_shard``;
    release every batch taken before calling it (held batches keep their buffers)."""

    def __init__(self, ctx: Context, ch: Chain, descs: Sequence[SampleDesc], rc: RunConfig, capture=None):
        self.ctx = ctx
        self.n = len(descs)
        arr = (SampleDesc * max(self.n, 1))(*descs)
        self.h = _vp()
        self.rc = rc
        self.cap = ctx._capture_begin(ch, rc, capture)   # kept alive until finish()
        try:
            _check(_lib.lfg_shard_start(ctx.h, ch.handle, arr, self.n, C.byref(rc), C.byref(self.h)))
        except Exception:
            ctx._capture_end(rc, self.cap)
            raise

    def next_batch(self, timeout_us: int = -1):
        b, n = C.c_int64(-1), C.c_int(0)
        rc = _lib.lfg_shard_next_batch(self.h, timeout_us, C.byref(b), C.byref(n))
        if rc == ERR_CLOSED:
            return None
        if rc == ERR_AGAIN:
            raise TimeoutError(_lib.lfg_last_error().decode(errors="replace"))
        _check(rc)
        return b.value, n.value

    def __iter__(self):
        while True:
            r = self.next_batch()
            if r is None:
                return
            yield r

    def finish(self):
        if not self.h:
            raise LfgError(ERR_STATE, "stream already finished")
        n = max(self.n, 1)
        rep = RunReport()
        ids = (C.c_uint64 * n)()
        bs = (C.c_int32 * n)()
        cls = (C.c_int32 * n)()
        h, self.h = self.h, _vp()
        try:
            _check(_lib.lfg_shard_finish(h, C.byref(rep), ids, bs, cls))
            self.ctx._capture_collect(self.cap)
        finally:
            self.ctx._capture_end(self.rc, self.cap)
        return rep, np.array(ids[:self.n], dtype=np.uint64), np.array(bs[:rep.batches]), np.array(cls[:self.n])


# ---- raw sample files + reader-thread source (include/lfgpu_files.h, host library) ----
FILE_VOLUME, FILE_IMAGE, FILE_WAVEFORM, FILE_PCM16 = 1, 2, 3, 4
HOST_LIB_PATH = os.path.join(_PKG, "libloadflow_b200.so")
_host = None


def _hostlib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB_PATH):
            raise ImportError(f"{HOST_LIB_PATH} is missing: build it with __graft_entry__.build()")
        h = C.CDLL(HOST_LIB_PATH)
        h.lfg_write_sample_file.argtypes = [C.c_char_p, C.c_int, C.c_int, _P(C.c_int64), _vp, _vp]
        h.lfg_file_source_open.argtypes = [_vp, _P(C.c_char_p), _P(C.c_uint64), C.c_int64, C.c_int, C.c_int,
                                           _P(_vp)]
        h.lfg_file_source_get.argtypes = [_vp, _vp]
        h.lfg_file_source_stats.argtypes = [_vp, _P(C.c_int64), _P(C.c_double)]
        h.lfg_file_source_close.argtypes = [_vp]
        h.lfg_files_last_error.restype = C.c_char_p
        _host = h
    return _host


def _hcheck(rc: int):
    if rc != LFG_OK:
        raise LfgError(rc, _hostlib().lfg_files_last_error().decode(errors="replace"))


def write_sample_file(path: str, kind: int, dims, data: np.ndarray, aux: np.ndarray | None = None):
    d = (C.c_int64 * 4)(*(list(dims) + [0] * (4 - len(dims))))
    data = np.ascontiguousarray(data)
    a = np.ascontiguousarray(aux) if aux is not None else None
    _hcheck(_hostlib().lfg_write_sample_file(path.encode(), kind, len(dims), d, data.ctypes.data,
                                             a.ctypes.data if a is not None else None))


class FileSource:
    """Reads sample files with `readers` threads into `slots` pinned buffers, in order,
    ahead of the shard (lfg_run_shard_source); buffers are refilled on release."""

    def __init__(self, ctx: "Context", paths: Sequence[str], ids: Sequence[int], readers: int = 4,
                 slots: int = 16):
        n = len(paths)
        self._paths = (C.c_char_p * n)(*[p.encode() for p in paths])
        self._ids = (C.c_uint64 * n)(*ids)
        self.h = _vp()
        self.n = n
        _hcheck(_hostlib().lfg_file_source_open(ctx.h, self._paths, self._ids, n, readers, slots,
                                                C.byref(self.h)))
        self.src = (C.c_byte * 32)()   # lfg_source {void*, fn*, fn*}
        _hcheck(_hostlib().lfg_file_source_get(self.h, self.src))

    def stats(self):
        b, t = C.c_int64(), C.c_double()
        _hcheck(_hostlib().lfg_file_source_stats(self.h, C.byref(b), C.byref(t)))
        return b.value, t.value

    def close(self):
        if self.h:
            _hostlib().lfg_file_source_close(self.h)
            self.h = _vp()


def run_config(batch_size: int, t_out_us: int = 0, policy: int = 0, trainer_us: int = 0,
               warmup_batches: int = 0, n_workers: int = 0, warmup_us: int = 0,
               update_interval_us: int = 1000, window: int = 1024,
               trainer_priority: int = 1, d2h_probe: int = 0, percentile: int = 75,
               scheduler: int = 0, max_workers: int = 0, sched_tick_us: int = 0,
               prefetch_factor: int = 0, sample_stamps: int = 0) -> RunConfig:
    rc = RunConfig()
    rc.batch_size = batch_size
    rc.policy = policy
    rc.t_out_us = t_out_us
    rc.warmup_us = warmup_us
    rc.update_interval_us = update_interval_us
    rc.window = window
    rc.n_workers = n_workers
    rc.trainer_us = trainer_us
    rc.trainer_priority = trainer_priority
    rc.warmup_batches = warmup_batches
    rc.d2h_probe = d2h_probe
    rc.percentile = percentile
    rc.scheduler = scheduler
    rc.max_workers = max_workers
    rc.sched_tick_us = sched_tick_us
    rc.prefetch_factor = prefetch_factor
    rc.sample_stamps = sample_stamps
    return rc
