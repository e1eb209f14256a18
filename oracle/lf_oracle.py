"""ctypes front-end for the C oracle (liblf_oracle.so).

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs -- never by the product package.
See lf_oracle.h for provenance (reference file:line citations) and parity status.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblf_oracle.so")


def _load():
    if not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liblf_oracle.so"])
    return C.CDLL(_LIB_PATH)


_lib = _load()


class MT64(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class Cfg3D(C.Structure):
    _fields_ = [("crop", C.c_int64 * 3), ("p_flip", C.c_double), ("p_bright", C.c_double),
                ("bright_lo", C.c_double), ("bright_hi", C.c_double),
                ("p_noise", C.c_double), ("noise_std_max", C.c_double),
                ("has_zoom", C.c_int32), ("p_zoom", C.c_double), ("zoom_lo", C.c_double),
                ("zoom_hi", C.c_double), ("has_contrast", C.c_int32), ("p_contrast", C.c_double),
                ("contrast_lo", C.c_double), ("contrast_hi", C.c_double), ("has_fg", C.c_int32),
                ("p_fg", C.c_double)]


class Params3D(C.Structure):
    _fields_ = [("off", C.c_int64 * 3), ("flip", C.c_int32 * 3), ("scale", C.c_double),
                ("sigma", C.c_double), ("key", C.c_uint32 * 2), ("win", C.c_int64 * 3),
                ("contrast", C.c_double), ("fg", C.c_int32), ("u_cls", C.c_double),
                ("u_adj", C.c_double * 3)]


class Cfg2D(C.Structure):
    _fields_ = [("out_h", C.c_int32), ("out_w", C.c_int32), ("scale_lo", C.c_double),
                ("scale_hi", C.c_double), ("ratio_lo", C.c_double), ("ratio_hi", C.c_double),
                ("p_hflip", C.c_double), ("mean", C.c_double * 3), ("std", C.c_double * 3)]


class Params2D(C.Structure):
    _fields_ = [("top", C.c_int64), ("left", C.c_int64), ("h", C.c_int64), ("w", C.c_int64),
                ("flip", C.c_int32)]


class CfgSp(C.Structure):
    _fields_ = [("n_fft", C.c_int32), ("win_length", C.c_int32), ("hop", C.c_int32),
                ("n_mels", C.c_int32), ("sample_rate", C.c_double), ("f_min", C.c_double),
                ("f_max", C.c_double), ("log_eps", C.c_double), ("freq_masks", C.c_int32),
                ("freq_mask_max", C.c_int32), ("time_masks", C.c_int32),
                ("time_mask_frac", C.c_double)]


class ParamsSp(C.Structure):
    _fields_ = [("n_frames", C.c_int32), ("f_lo", C.c_int32 * 8), ("f_w", C.c_int32 * 8),
                ("t_lo", C.c_int32 * 32), ("t_w", C.c_int32 * 32), ("n_fmask", C.c_int32),
                ("n_tmask", C.c_int32)]


_P = C.POINTER
_lib.lfo_mt64_seed.argtypes = [_P(MT64), C.c_uint64]
_lib.lfo_mt64_next.argtypes = [_P(MT64)]
_lib.lfo_mt64_next.restype = C.c_uint64
_lib.lfo_philox4x32_10.argtypes = [_P(C.c_uint32), _P(C.c_uint32), _P(C.c_uint32)]
_lib.lfo_normals4.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, _P(C.c_double)]
_lib.lfo_cfg3d_default.argtypes = [_P(Cfg3D)]
_lib.lfo_draw3d.argtypes = [_P(Cfg3D), C.c_uint64, C.c_uint64, _P(C.c_int64), _P(Params3D)]
_lib.lfo_apply3d.argtypes = [_P(Cfg3D), _P(Params3D), C.c_void_p, C.c_void_p, _P(C.c_int64),
                             C.c_void_p, C.c_void_p]
_lib.lfo_fg_offsets.argtypes = [_P(Params3D), C.c_void_p, _P(C.c_int64), _P(C.c_int64)]
_lib.lfo_cfg2d_default.argtypes = [_P(Cfg2D)]
_lib.lfo_draw2d.argtypes = [_P(Cfg2D), C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                            _P(Params2D)]
_lib.lfo_apply2d.argtypes = [_P(Cfg2D), _P(Params2D), C.c_void_p, C.c_int64, C.c_int64,
                             C.c_void_p]
_lib.lfo_bilinear_chw.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                  C.c_int64, C.c_void_p]
_lib.lfo_cfgsp_default.argtypes = [_P(CfgSp)]
_lib.lfo_sp_frames.argtypes = [_P(CfgSp), C.c_int64]
_lib.lfo_sp_frames.restype = C.c_int32
_lib.lfo_drawsp.argtypes = [_P(CfgSp), C.c_uint64, C.c_uint64, C.c_int64, _P(ParamsSp)]
_lib.lfo_mel_fbank.argtypes = [_P(CfgSp), C.c_void_p]
_lib.lfo_applysp.argtypes = [_P(CfgSp), _P(ParamsSp), C.c_void_p, C.c_int64, C.c_void_p,
                             C.c_void_p]


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def mt64(seed: int, n: int) -> np.ndarray:
    g = MT64()
    _lib.lfo_mt64_seed(C.byref(g), seed)
    return np.array([_lib.lfo_mt64_next(C.byref(g)) for _ in range(n)], dtype=np.uint64)


def philox(ctr, key) -> np.ndarray:
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    _lib.lfo_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def normals4(group: int, k0: int, k1: int) -> np.ndarray:
    z = (C.c_double * 4)()
    _lib.lfo_normals4(group, k0, k1, z)
    return np.array(list(z))


# ---------------------------------------------------------------- 3D
def cfg3d(**kw) -> Cfg3D:
    c = Cfg3D()
    _lib.lfo_cfg3d_default(C.byref(c))
    for k, v in kw.items():
        if k == "crop":
            c.crop = (C.c_int64 * 3)(*v)
        else:
            setattr(c, k, v)
    return c


def draw3d(cfg: Cfg3D, seed: int, sid: int, dims) -> Params3D:
    p = Params3D()
    d = (C.c_int64 * 3)(*dims)
    _lib.lfo_draw3d(C.byref(cfg), seed, sid, d, C.byref(p))
    return p


def apply3d(cfg: Cfg3D, p: Params3D, img: np.ndarray, lbl: np.ndarray):
    img = np.ascontiguousarray(img, dtype=np.float32)
    lbl = np.ascontiguousarray(lbl, dtype=np.uint8)
    dims = (C.c_int64 * 3)(*img.shape)
    shape = tuple(cfg.crop)
    out_img = np.empty(shape, dtype=np.float64)
    out_lbl = np.empty(shape, dtype=np.uint8)
    _lib.lfo_apply3d(C.byref(cfg), C.byref(p), _ptr(img), _ptr(lbl), dims, _ptr(out_img),
                     _ptr(out_lbl))
    return out_img, out_lbl


def fg_offsets(p: Params3D, lbl: np.ndarray):
    """Final window origin of a foreground-biased crop, or None (random offsets hold)."""
    lbl = np.ascontiguousarray(lbl, dtype=np.uint8)
    dims = (C.c_int64 * 3)(*lbl.shape)
    off = (C.c_int64 * 3)()
    r = _lib.lfo_fg_offsets(C.byref(p), _ptr(lbl), dims, off)
    return None if r != 0 else list(off)


def chain3d(cfg: Cfg3D, seed: int, sid: int, img: np.ndarray, lbl: np.ndarray):
    p = draw3d(cfg, seed, sid, img.shape)
    return apply3d(cfg, p, img, lbl), p


# ---------------------------------------------------------------- 2D
def cfg2d(**kw) -> Cfg2D:
    c = Cfg2D()
    _lib.lfo_cfg2d_default(C.byref(c))
    for k, v in kw.items():
        if k in ("mean", "std"):
            setattr(c, k, (C.c_double * 3)(*v))
        else:
            setattr(c, k, v)
    return c


def draw2d(cfg: Cfg2D, seed: int, sid: int, H: int, W: int) -> Params2D:
    p = Params2D()
    _lib.lfo_draw2d(C.byref(cfg), seed, sid, H, W, C.byref(p))
    return p


def apply2d(cfg: Cfg2D, p: Params2D, img_hwc: np.ndarray) -> np.ndarray:
    img = np.ascontiguousarray(img_hwc, dtype=np.uint8)
    H, W, _ = img.shape
    out = np.empty((3, cfg.out_h, cfg.out_w), dtype=np.float64)
    _lib.lfo_apply2d(C.byref(cfg), C.byref(p), _ptr(img), H, W, _ptr(out))
    return out


def chain2d(cfg: Cfg2D, seed: int, sid: int, img_hwc: np.ndarray):
    H, W, _ = img_hwc.shape
    p = draw2d(cfg, seed, sid, H, W)
    return apply2d(cfg, p, img_hwc), p


def bilinear_chw(src: np.ndarray, oh: int, ow: int) -> np.ndarray:
    src = np.ascontiguousarray(src, dtype=np.float32)
    Cc, H, W = src.shape
    out = np.empty((Cc, oh, ow), dtype=np.float64)
    _lib.lfo_bilinear_chw(_ptr(src), Cc, H, W, oh, ow, _ptr(out))
    return out


# ---------------------------------------------------------------- speech
def cfgsp(**kw) -> CfgSp:
    c = CfgSp()
    _lib.lfo_cfgsp_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def drawsp(cfg: CfgSp, seed: int, sid: int, L: int) -> ParamsSp:
    p = ParamsSp()
    _lib.lfo_drawsp(C.byref(cfg), seed, sid, L, C.byref(p))
    return p


def mel_fbank(cfg: CfgSp) -> np.ndarray:
    fb = np.empty((cfg.n_mels, cfg.n_fft // 2 + 1), dtype=np.float64)
    _lib.lfo_mel_fbank(C.byref(cfg), _ptr(fb))
    return fb


def applysp(cfg: CfgSp, p: ParamsSp, wav: np.ndarray, want_power: bool = False):
    wav = np.ascontiguousarray(wav, dtype=np.float32)
    T = p.n_frames
    logmel = np.empty((cfg.n_mels, T), dtype=np.float64)
    power = np.empty((cfg.n_fft // 2 + 1, T), dtype=np.float64) if want_power else None
    _lib.lfo_applysp(C.byref(cfg), C.byref(p), _ptr(wav), wav.shape[0], _ptr(logmel),
                     _ptr(power) if power is not None else None)
    return logmel, power


def chainsp(cfg: CfgSp, seed: int, sid: int, wav: np.ndarray, want_power: bool = False):
    p = drawsp(cfg, seed, sid, wav.shape[0])
    return applysp(cfg, p, wav, want_power), p
