"""Generates tests/golden/*.npz -- frozen oracle outputs for small cases.

Run from the repo root:  python tests/golden/make_golden.py
The reference has no transform arithmetic and no golden vectors for pixel /
voxel / audio values ("parity unpinned"), so these fixtures
freeze the oracle itself: tests/test_oracle.py checks the oracle reproduces
them bit-for-bit (regression pin) and cross-checks the formulas against
torch / torchvision / torchaudio; the GPU parity tests check the kernels
against the oracle.  The mt19937_64 known-answer vector comes from
libstdc++'s std::mt19937_64 (compiled here by this script).
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import lf_oracle as O  # noqa: E402

SEED = 1


def mt_kat():
    src = r'''
#include <random>
#include <cstdio>
int main() {
  const unsigned long long seeds[] = {5489ULL, 42ULL, 1ULL ^ (0x9e3779b97f4a7c15ULL * 8ULL)};
  for (auto s : seeds) { std::mt19937_64 g(s); for (int i = 0; i < 8; ++i) std::printf("%llu\n", (unsigned long long)g()); }
  std::mt19937_64 g(5489); unsigned long long x = 0; for (int i = 0; i < 10000; ++i) x = g();
  std::printf("%llu\n", x);
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "kat.cpp")
        open(c, "w").write(src)
        subprocess.check_call(["g++", "-O1", c, "-o", os.path.join(d, "kat")])
        out = subprocess.check_output([os.path.join(d, "kat")]).decode().split()
    return np.array([int(v) for v in out], dtype=np.uint64)


def main():
    rng = np.random.default_rng(2024)
    # ---- 3D: 8 ids, small volumes, all probabilities forced on + defaults
    cases3 = []
    for k in range(8):
        dims = (12 + k, 14, 20)
        img = rng.standard_normal(dims).astype(np.float32)
        lbl = rng.integers(0, 3, dims, dtype=np.uint8)
        kw = dict(crop=(8, 8, 16))
        if k % 2 == 0:
            kw.update(p_flip=0.5, p_bright=1.0, p_noise=1.0)
        cfg = O.cfg3d(**kw)
        sid = 1000 + 37 * k
        (o_img, o_lbl), p = O.chain3d(cfg, SEED, sid, img, lbl)
        cases3.append(dict(sid=sid, forced=int(k % 2 == 0), img=img, lbl=lbl, out_img=o_img,
                           out_lbl=o_lbl, off=np.array(p.off), flip=np.array(p.flip),
                           scale=p.scale, sigma=p.sigma, key=np.array(p.key, dtype=np.uint32)))
    np.savez_compressed(os.path.join(HERE, "img3d.npz"),
                        **{f"{i}_{k}": v for i, c in enumerate(cases3) for k, v in c.items()})
    # ---- 2D: 8 ids, small images, 32x32 output
    cases2 = []
    for k in range(8):
        H, W = (int(x) for x in rng.integers(24, 60, 2))
        img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        cfg = O.cfg2d(out_h=32, out_w=32)
        sid = 7 + 101 * k
        out, p = O.chain2d(cfg, SEED, sid, img)
        cases2.append(dict(sid=sid, img=img, out=out,
                           box=np.array([p.top, p.left, p.h, p.w, p.flip])))
    np.savez_compressed(os.path.join(HERE, "rrc2d.npz"),
                        **{f"{i}_{k}": v for i, c in enumerate(cases2) for k, v in c.items()})
    # ---- speech: 4 utterances, L = 4000..4300
    cases_s = []
    for k in range(4):
        L = 4000 + 100 * k
        wav = (0.3 * rng.standard_normal(L)).astype(np.float32)
        cfg = O.cfgsp()
        sid = 55 + k
        (lm, _), p = O.chainsp(cfg, SEED, sid, wav)
        masks = np.array([p.n_frames] + [p.f_lo[i] for i in range(2)] + [p.f_w[i] for i in range(2)]
                         + [p.t_lo[i] for i in range(10)] + [p.t_w[i] for i in range(10)])
        cases_s.append(dict(sid=sid, wav=wav, logmel=lm, masks=masks))
    np.savez_compressed(os.path.join(HERE, "speech.npz"),
                        **{f"{i}_{k}": v for i, c in enumerate(cases_s) for k, v in c.items()})
    # ---- generators
    np.save(os.path.join(HERE, "mt19937_64_kat.npy"), mt_kat())
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
