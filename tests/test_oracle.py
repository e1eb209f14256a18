"""CPU tests of the oracle (test infrastructure) -- pinning it before trusting it.

1. Generators: mt19937_64 against libstdc++'s std::mt19937_64 (the reference's
   Rng, sample.hpp:25) and Philox4x32-10 against the Random123 known-answer
   vectors.
2. Formulas: bilinear resize against torch F.interpolate(antialias=False);
   STFT power against torch.stft; the slaney mel filterbank against
   torchaudio.functional.melscale_fbanks; normalize against torchvision.
3. Regression: the committed golden fixtures (tests/golden, made by
   make_golden.py) are reproduced exactly.
4. Semantics: parameter draws stay in range; crop/flip/label movement is a
   pure permutation; noise statistics."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SEED = 1


def test_mt19937_64_matches_libstdcxx(oracle):
    kat = np.load(os.path.join(GOLD, "mt19937_64_kat.npy"))
    seeds = [5489, 42, 1 ^ ((0x9e3779b97f4a7c15 * 8) & (2**64 - 1))]
    got = np.concatenate([oracle.mt64(s, 8) for s in seeds])
    assert np.array_equal(got, kat[:24])
    assert oracle.mt64(5489, 10000)[-1] == kat[24] == 9981545732273789042  # C++ standard KAT


@pytest.mark.parametrize("ctr,key,want", [
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
])
def test_philox4x32_10_random123_kat(oracle, ctr, key, want):
    assert list(oracle.philox(ctr, key)) == want


def test_box_muller_normals_are_standard(oracle):
    z = np.concatenate([oracle.normals4(g, 12345, 678) for g in range(20000)])
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1.0) < 0.02
    assert abs(np.mean(z ** 3)) < 0.05 and abs(np.mean(z ** 4) - 3.0) < 0.15


# ------------------------------------------------------------ formulas vs torch
def test_bilinear_matches_torch_interpolate(oracle):
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F
    rng = np.random.default_rng(0)
    for (H, W), (oh, ow) in [((37, 53), (16, 16)), ((37, 53), (224, 224)), ((300, 420), (224, 224)),
                             ((512, 130), (224, 224))]:
        src = (rng.random((3, H, W)) * 255).astype(np.float32)
        a = oracle.bilinear_chw(src, oh, ow)
        b = F.interpolate(torch.from_numpy(src)[None].double(), size=(oh, ow), mode="bilinear",
                          align_corners=False, antialias=False)[0].numpy()
        assert np.abs(a - b).max() < 1e-9


def test_rrc_chain_matches_torchvision_ops(oracle):
    torch = pytest.importorskip("torch")
    tvf = pytest.importorskip("torchvision.transforms.v2.functional")
    import torch.nn.functional as F
    cfg = oracle.cfg2d()
    rng = np.random.default_rng(1)
    for sid in range(6):
        H, W = (int(x) for x in rng.integers(256, 513, 2))
        img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        out, p = oracle.chain2d(cfg, SEED, sid, img)
        crop = torch.from_numpy(img).permute(2, 0, 1)[:, p.top:p.top + p.h, p.left:p.left + p.w]
        r = F.interpolate(crop[None].double(), size=(224, 224), mode="bilinear",
                          align_corners=False, antialias=False)[0]
        if p.flip:
            r = torch.flip(r, dims=[2])
        r = tvf.normalize(r / 255.0, list(cfg.mean), list(cfg.std))
        assert np.abs(out - r.numpy()).max() < 1e-9


def test_rrc_params_follow_torchvision_rules(oracle):
    cfg = oracle.cfg2d()
    rng = np.random.default_rng(2)
    n_fallback = 0
    for sid in range(2000):
        H, W = (int(x) for x in rng.integers(16, 700, 2))
        p = oracle.draw2d(cfg, SEED, sid, H, W)
        assert 0 <= p.top <= H - p.h and 0 <= p.left <= W - p.w
        assert 0 < p.h <= H and 0 < p.w <= W
        area = p.h * p.w / (H * W)
        if not (0.08 * 0.9 <= area <= 1.0 + 1e-9):
            n_fallback += 1   # centre-crop fallback after 10 rejected tries
    assert n_fallback < 200


def test_stft_power_and_mel_match_torch(oracle):
    torch = pytest.importorskip("torch")
    ta = pytest.importorskip("torchaudio")
    cfg = oracle.cfgsp(freq_masks=0, time_masks=0)
    rng = np.random.default_rng(3)
    wav = rng.standard_normal(4000).astype(np.float32)
    (lm, pw), p = oracle.chainsp(cfg, SEED, 9, wav, want_power=True)
    X = torch.stft(torch.from_numpy(wav).double(), 512, hop_length=160, win_length=320,
                   window=torch.hann_window(320, dtype=torch.float64), center=True,
                   pad_mode="reflect", return_complex=True)
    P = (X.abs() ** 2).numpy()
    assert pw.shape == P.shape and np.abs(pw - P).max() / P.max() < 1e-12
    fb = ta.functional.melscale_fbanks(257, 0.0, 8000.0, 80, 16000, norm="slaney",
                                       mel_scale="slaney").T.double().numpy()
    ofb = oracle.mel_fbank(cfg)
    assert np.abs(ofb - fb).max() < 1e-6 * np.abs(fb).max() * 10   # torchaudio builds it in fp32
    lm2 = np.log(ofb @ P + 2.0 ** -24)
    assert np.abs(lm - lm2).max() < 1e-9


# ------------------------------------------------------------ golden fixtures
def _cases(path):
    z = np.load(path)
    n = 1 + max(int(k.split("_")[0]) for k in z.files)
    return [{k.split("_", 1)[1]: z[k] for k in z.files if k.startswith(f"{i}_")} for i in range(n)]


def test_golden_img3d(oracle):
    for c in _cases(os.path.join(GOLD, "img3d.npz")):
        kw = dict(crop=(8, 8, 16))
        if int(c["forced"]):
            kw.update(p_flip=0.5, p_bright=1.0, p_noise=1.0)
        cfg = oracle.cfg3d(**kw)
        (o_img, o_lbl), p = oracle.chain3d(cfg, SEED, int(c["sid"]), c["img"], c["lbl"])
        assert list(p.off) == list(c["off"]) and list(p.flip) == list(c["flip"])
        assert p.scale == float(c["scale"]) and p.sigma == float(c["sigma"])
        assert np.array_equal(o_lbl, c["out_lbl"]) and np.array_equal(o_img, c["out_img"])


def test_golden_rrc2d(oracle):
    cfg = oracle.cfg2d(out_h=32, out_w=32)
    for c in _cases(os.path.join(GOLD, "rrc2d.npz")):
        out, p = oracle.chain2d(cfg, SEED, int(c["sid"]), c["img"])
        assert [p.top, p.left, p.h, p.w, p.flip] == list(c["box"])
        assert np.array_equal(out, c["out"])


def test_golden_speech(oracle):
    cfg = oracle.cfgsp()
    for c in _cases(os.path.join(GOLD, "speech.npz")):
        (lm, _), p = oracle.chainsp(cfg, SEED, int(c["sid"]), c["wav"])
        assert p.n_frames == int(c["masks"][0])
        assert np.array_equal(lm, c["logmel"])


# ------------------------------------------------------------ semantics
def test_img3d_crop_flip_is_a_permutation(oracle):
    """With brightness/noise off, the image output is an exact re-indexing of the
    input (crop + flips), and labels move identically (bit-exact movement)."""
    cfg = oracle.cfg3d(crop=(8, 8, 16), p_flip=0.5, p_bright=0.0, p_noise=0.0)
    dims = (10, 12, 20)
    n = int(np.prod(dims))
    img = np.arange(n, dtype=np.float32).reshape(dims)
    lbl = (np.arange(n) % 251).astype(np.uint8).reshape(dims)
    for sid in range(50):
        (o_img, o_lbl), p = oracle.chain3d(cfg, SEED, sid, img, lbl)
        sl = tuple(slice(p.off[a], p.off[a] + (8, 8, 16)[a]) for a in range(3))
        want = img[sl]
        for a in range(3):
            if p.flip[a]:
                want = np.flip(want, axis=a)
        assert np.array_equal(o_img, want.astype(np.float64))
        assert np.array_equal(o_lbl, (want.astype(np.int64) % 251).astype(np.uint8))


def test_img3d_zero_pads_small_volumes(oracle):
    cfg = oracle.cfg3d(crop=(16, 16, 32), p_flip=0.0, p_bright=0.0, p_noise=0.0)
    img = np.ones((5, 6, 7), np.float32)
    lbl = np.ones((5, 6, 7), np.uint8)
    (o_img, o_lbl), p = oracle.chain3d(cfg, SEED, 3, img, lbl)
    assert list(p.off) == [0, 0, 0]
    assert o_img.sum() == 5 * 6 * 7 and o_img[5:].sum() == 0 and o_lbl[:, 6:].sum() == 0


def test_specaugment_masks_in_range(oracle):
    cfg = oracle.cfgsp()
    for sid in range(300):
        L = 30000 + 467 * sid
        p = oracle.drawsp(cfg, SEED, sid, L)
        T = p.n_frames
        assert T == 1 + L // 160
        for i in range(2):
            assert 0 <= p.f_w[i] <= 27 and 0 <= p.f_lo[i] and p.f_lo[i] + p.f_w[i] <= 80
        for i in range(10):
            assert 0 <= p.t_w[i] <= int(0.05 * T) and p.t_lo[i] + p.t_w[i] <= T


# ------------------------------------------------------------ optional ops (zoom, contrast)
def test_zoom_trilinear_matches_torch_interpolate(oracle):
    """RandomZoom3D: the zoomed window resampled to the crop equals torch's trilinear
    F.interpolate(align_corners=False) of the zero-padded window (fp64, exact); labels
    take the integer nearest index min(dst * win // crop, win - 1)."""
    import torch
    rng = np.random.default_rng(7)
    dims = (30, 34, 40)
    img = rng.standard_normal(dims).astype(np.float32)
    lbl = rng.integers(0, 5, dims, dtype=np.uint8)
    crop = (16, 16, 32)
    cfg = oracle.cfg3d(crop=crop, has_zoom=1, p_zoom=1.0, zoom_lo=0.7, zoom_hi=1.3,
                       p_flip=0.0, p_bright=0.0, p_noise=0.0)
    zoomed = 0
    for sid in range(12):
        (o_img, o_lbl), p = oracle.chain3d(cfg, SEED, sid, img, lbl)
        w, o = list(p.win), list(p.off)
        zoomed += w != list(crop)
        win = np.zeros(w)
        wl = np.zeros(w, np.uint8)
        src = img[o[0]:o[0] + w[0], o[1]:o[1] + w[1], o[2]:o[2] + w[2]]
        win[:src.shape[0], :src.shape[1], :src.shape[2]] = src
        wl[:src.shape[0], :src.shape[1], :src.shape[2]] = lbl[o[0]:o[0] + w[0], o[1]:o[1] + w[1],
                                                              o[2]:o[2] + w[2]]
        t = torch.nn.functional.interpolate(torch.from_numpy(win)[None, None], size=crop,
                                            mode="trilinear", align_corners=False)[0, 0].numpy()
        assert np.abs(t - o_img).max() < 1e-12
        idx = [np.minimum(np.arange(crop[a]) * w[a] // crop[a], w[a] - 1) for a in range(3)]
        assert np.array_equal(o_lbl, wl[np.ix_(*idx)])
    assert zoomed >= 8


def test_zoom_window_equal_to_crop_is_a_plain_crop(oracle):
    cfg = oracle.cfg3d(crop=(8, 8, 16), has_zoom=1, p_zoom=1.0, zoom_lo=1.0, zoom_hi=1.0,
                       p_flip=0.5, p_bright=0.0, p_noise=0.0)
    dims = (10, 12, 20)
    img = np.arange(int(np.prod(dims)), dtype=np.float32).reshape(dims)
    lbl = (img.astype(np.int64) % 251).astype(np.uint8)
    for sid in range(20):
        (o_img, o_lbl), p = oracle.chain3d(cfg, SEED, sid, img, lbl)
        assert list(p.win) == [8, 8, 16]
        want = img[tuple(slice(p.off[a], p.off[a] + (8, 8, 16)[a]) for a in range(3))]
        for a in range(3):
            if p.flip[a]:
                want = np.flip(want, axis=a)
        assert np.array_equal(o_img, want.astype(np.float64))


def test_contrast_scales_deviation_about_the_crop_mean(oracle):
    """RandomContrast: (v - m) * c + m with m the crop mean (after brightness)."""
    rng = np.random.default_rng(9)
    dims = (12, 20, 24)
    img = (rng.standard_normal(dims) + 0.3).astype(np.float32)
    lbl = np.zeros(dims, np.uint8)
    base = oracle.cfg3d(crop=(8, 8, 16), p_flip=0.0, p_bright=1.0, p_noise=0.0)
    cfg = oracle.cfg3d(crop=(8, 8, 16), p_flip=0.0, p_bright=1.0, p_noise=0.0,
                       has_contrast=1, p_contrast=1.0)
    for sid in range(10):
        p = oracle.draw3d(cfg, SEED, sid, dims)
        assert 0.75 <= p.contrast <= 1.25
        out, _ = oracle.apply3d(cfg, p, img, lbl)
        q = oracle.draw3d(base, SEED, sid, dims)   # same crop, no contrast
        for a in range(3):
            q.off[a] = p.off[a]
        q.scale = p.scale
        plain, _ = oracle.apply3d(base, q, img, lbl)
        m = plain.mean()
        assert abs(out.mean() - m) < 1e-12
        assert np.abs((out - m) - p.contrast * (plain - m)).max() < 1e-12


def _fg_offsets_numpy(p, lbl):
    """Independent restatement of RandBalancedCrop's window placement (MLPerf adjust()
    on the bounding box of every voxel of the chosen class)."""
    if not p.fg:
        return None
    present = [v for v in range(1, 8) if (lbl == v).any()]
    if not present:
        return None
    cl = present[min(int(np.floor(p.u_cls * len(present))), len(present) - 1)]
    idx = np.nonzero(lbl == cl)
    off = []
    for a in range(3):
        lo, hi = int(idx[a].min()), int(idx[a].max()) + 1
        patch, dim = int(p.win[a]), lbl.shape[a]
        diff = patch - (hi - lo)
        sign = -1 if diff < 0 else 1
        diff = abs(diff)
        ladj = min(int(np.floor(p.u_adj[a] * diff)), diff - 1) if diff > 0 else 0
        hadj = diff - ladj
        low, high = max(0, lo - sign * ladj), min(dim, hi + sign * hadj)
        d2 = patch - (high - low)
        if d2 > 0:
            if low == 0:
                high += d2
            else:
                low -= d2
        off.append(int(np.clip(low, 0, max(dim - patch, 0))))
    return off


def test_foreground_crop_matches_numpy_restatement(oracle):
    """RandomCrop with foreground oversampling: the oracle's window origin equals an
    independent numpy restatement, the window holds foreground of the chosen class
    when it fits, and non-oversampled draws keep the random offsets."""
    rng = np.random.default_rng(3)
    dims = (40, 48, 56)
    z, y, x = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    lbl = np.zeros(dims, np.uint8)
    lbl[((z - 25) / 6) ** 2 + ((y - 30) / 8) ** 2 + ((x - 15) / 9) ** 2 <= 1] = 1
    lbl[((z - 12) / 4) ** 2 + ((y - 10) / 5) ** 2 + ((x - 40) / 6) ** 2 <= 1] = 2
    img = rng.standard_normal(dims).astype(np.float32)
    cfg = oracle.cfg3d(crop=(16, 16, 32), has_fg=1, p_fg=0.5, p_flip=0.0, p_bright=0.0, p_noise=0.0)
    n_fg = 0
    for sid in range(60):
        p = oracle.draw3d(cfg, 1, sid, dims)
        got = oracle.fg_offsets(p, lbl)
        assert got == _fg_offsets_numpy(p, lbl)
        (out_img, out_lbl), _ = oracle.chain3d(cfg, 1, sid, img, lbl)
        off = got if got is not None else list(p.off)
        want = img[off[0]:off[0] + 16, off[1]:off[1] + 16, off[2]:off[2] + 32]
        assert np.array_equal(out_img, want.astype(np.float64))
        if got is not None:
            n_fg += 1
            assert (out_lbl > 0).any()
    assert 15 <= n_fg <= 45
    # no foreground at all: the random offsets hold
    p = oracle.draw3d(cfg, 1, 0, dims)
    assert oracle.fg_offsets(p, np.zeros(dims, np.uint8)) is None
