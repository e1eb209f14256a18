"""Comparison of delivered GPU outputs with the CPU oracle.

TEST INFRASTRUCTURE ONLY (like lf_oracle.py): used by tests/ and by bench.py's
verification leg, which checks samples captured from the timed runs AFTER the
timed region.  Never imported by the product package.

Bars (north_star "bit-exact for crop, flip and indexing,
within <= 1e-5 relative in fp32 for interpolation, normalization and spectrogram"):
  * labels / crop windows / flips / masks / padding: bit-exact (== on integers);
  * image values: |gpu - oracle| <= 1e-5 * |oracle| + atol, atol 1e-6 (3D, unit
    variance voxels) or 1e-5 (normalised 2D, O(1) values) -- the absolute floor only
    matters where relative error is undefined (values near 0);
  * speech: see speech_error() -- relative error 1e-5 in the mel-energy domain, with
    an absolute floor of 1e-8 x the frame's peak mel energy for near-empty bands (log
    amplifies fp32 round-off there): measured, the FFT kernel needs 7.6e-10 and stays
    within 1.2e-6 relative for every bin within 20 dB of its frame's peak.
Each function returns the worst err / bound ratio (<= 1 passes) and raises
AssertionError on an integer mismatch.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-5
ATOL_3D = 1e-6
ATOL_2D = 1e-5
# Speech: relative error bound in the mel-energy domain, with an absolute floor
# proportional to the frame's peak mel energy (fp32 round-off of the 320-tap DFT
# sums is relative to the frame's scale, not to a quiet band's own energy).
SPEECH_REL = 1e-5
SPEECH_FLOOR = 1.0e-8     # x frame peak energy (measured need of the default FFT kernel: <= 7.6e-10)


def ratio_close(got: np.ndarray, want: np.ndarray, atol: float) -> float:
    err = np.abs(got.astype(np.float64) - want)
    bound = RTOL * np.abs(want) + atol
    return float((err / bound).max()) if err.size else 0.0


def check_img3d(O, ocfg, seed: int, sid: int, img: np.ndarray, lbl: np.ndarray, raw: np.ndarray,
                crop) -> float:
    """raw = captured slot bytes: f32 image [crop] then u8 label [crop]."""
    vox = int(np.prod(crop))
    (e_img, e_lbl), _ = O.chain3d(ocfg, seed, sid, img, lbl)
    g_img = raw[: vox * 4].view(np.float32).reshape(crop)
    g_lbl = raw[vox * 4: vox * 5].reshape(crop)
    assert np.array_equal(g_lbl, e_lbl), f"sample {sid}: label crop / flip not bit-exact"
    return ratio_close(g_img, e_img, ATOL_3D)


def check_rrc(O, ocfg, seed: int, sid: int, img_hwc: np.ndarray, raw: np.ndarray, oh=224, ow=224) -> float:
    e, _ = O.chain2d(ocfg, seed, sid, img_hwc)
    g = raw[: 3 * oh * ow * 4].view(np.float32).reshape(3, oh, ow)
    return ratio_close(g, e, ATOL_2D)


def splice(logmel: np.ndarray, stack: int = 3) -> np.ndarray:
    """FrameSplicing (stack, subsample) of the oracle's [80, T] log-mel -> [T', 80*stack]."""
    m, T = logmel.shape
    rows = (T + stack - 1) // stack
    out = np.zeros((rows, m * stack))
    for s in range(stack):
        idx = np.arange(rows) * stack + s
        ok = idx < T
        out[ok, s * m:(s + 1) * m] = logmel[:, idx[ok]].T
    return out


def speech_levels(got: np.ndarray, want: np.ndarray, n_mels: int = 80, stack: int = 3) -> dict:
    """Error statistics by band level below the frame peak (diagnostics): for each
    level range, the max relative error and the max error / frame peak energy."""
    nz = want != 0.0
    ge, oe = np.exp(got.astype(np.float64)), np.exp(want)
    peak = np.exp(want.reshape(want.shape[0], stack, n_mels).max(axis=2)).repeat(n_mels, axis=1)
    err, lvl = np.abs(ge - oe), oe / peak
    out = {}
    for lo, hi in ((1e-2, 1.01), (1e-4, 1e-2), (1e-6, 1e-4), (0.0, 1e-6)):
        m = nz & (lvl >= lo) & (lvl < hi)
        if m.any():
            out[f"{lo:g}"] = (float((err / oe)[m].max()), float((err / peak)[m].max()))
    return out


def speech_error(got: np.ndarray, want: np.ndarray, n_mels: int = 80, stack: int = 3) -> float:
    """got / want: spliced log-mel [T', stack * n_mels].  Zeros (SpecAugment masks,
    splice padding) must match exactly; other entries are compared as energies:
    |e^g - e^o| <= SPEECH_REL * e^o + SPEECH_FLOOR * (frame peak energy)."""
    zero = want == 0.0
    assert np.array_equal(got[zero], want[zero]), "SpecAugment / padding zeros differ"
    ge, oe = np.exp(got[~zero].astype(np.float64)), np.exp(want[~zero])
    peak = np.exp(want.reshape(want.shape[0], stack, n_mels).max(axis=2)).repeat(n_mels, axis=1)[~zero]
    err = np.abs(ge - oe)
    bound = SPEECH_REL * oe + SPEECH_FLOOR * peak
    return float((err / bound).max()) if err.size else 0.0


def check_speech(O, ocfg, seed: int, sid: int, wav: np.ndarray, raw: np.ndarray, stack: int = 3) -> float:
    (lm, _), _ = O.chainsp(ocfg, seed, sid, wav)
    e = splice(lm, stack)
    g = raw[: e.size * 4].view(np.float32).reshape(e.shape)
    return speech_error(g, e, stack=stack)
