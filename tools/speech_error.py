#!/usr/bin/env python
"""Speech error against the oracle by band level: the floor (x frame peak mel energy)
the GPU kernel needs on top of 1e-5 relative, and the max relative error per level
below the frame peak.  LFG_SPEECH_KERNEL=tc measures the tcgen05 kernel.  GPU only;
the oracle is the checker."""
import os, sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from paper_2509_10712_b200 import lfgpu
import lf_oracle as oracle
sys.path.insert(0, 'tests')
def splice(logmel, stack=3):
    m, T = logmel.shape
    rows = (T + stack - 1) // stack
    out = np.zeros((rows, m * stack))
    for s in range(stack):
        idx = np.arange(rows) * stack + s
        ok = idx < T
        out[ok, s * m:(s + 1) * m] = logmel[:, idx[ok]].T
    return out
SEED=1
ctx = lfgpu.Context(batch_size=8, n_workers=4, max_group=8, max_slot_buffers=8, seed=SEED)
ch = ctx.chain(lfgpu.speech_ops(max_len=170000))
ocfg = oracle.cfgsp()
rng = np.random.default_rng(21)
need_floor = 0.0; rel = {}
for k, L in enumerate([4000, 20000, 39999, 100000, 170000, 1000, 50000, 12345]):
    t = np.arange(L) / 16000.0
    if k % 2 == 0:
        wav = (0.5 * np.sin(2 * np.pi * (200 + 50 * k) * t) + 0.2 * np.sin(2 * np.pi * 3100 * t) + 0.01 * rng.standard_normal(L)).astype(np.float32)
    else:
        wav = (0.3 * rng.standard_normal(L)).astype(np.float32)
    p = ctx.device_alloc(wav.nbytes); ctx.h2d(p, wav)
    sid = 700 + k
    tk = ctx.submit(ch, lfgpu.sample_desc(sid, (L,), p)); ctx.flush(); ctx.wait(tk)
    (lm, _), _ = oracle.chainsp(ocfg, SEED, sid, wav)
    e = splice(lm)
    _, ob, _ = ch.info()
    got = ctx.ticket_output(tk, ob).view(np.float32).reshape(-1, 240)[: e.shape[0]]
    zero = e == 0.0
    ge, oe = np.exp(got[~zero].astype(np.float64)), np.exp(e[~zero])
    peak = np.exp(e.reshape(e.shape[0], 3, 80).max(axis=2)).repeat(80, axis=1)[~zero]
    err = np.abs(ge - oe)
    need_floor = max(need_floor, float(((err - 1e-5 * oe) / peak).max()))
    lvl = oe / peak
    for lo, hi in ((1e-2, 1.01), (1e-4, 1e-2), (1e-6, 1e-4), (0, 1e-6)):
        m = (lvl >= lo) & (lvl < hi)
        if m.any(): rel[lo] = max(rel.get(lo, 0), float((err / oe)[m].max()))
    ctx.release(tk); ctx.device_free(p)
print(os.environ.get("LFG_SPEECH_KERNEL", "fft"), "floor needed (x frame peak) with 1e-5 relative:", need_floor, "max rel err by level:", rel)
