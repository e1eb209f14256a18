"""GPU parity: the sm_100a transform kernels (through the C ABI) against the CPU oracle.

Bars:
  * crop / flip / label / indexing: bit-exact (labels compared with ==; crop
    boxes and flip bits compared as integers via lfg_draw_params).
  * image values: |gpu - oracle| <= RTOL * |oracle| + ATOL with RTOL = 1e-5
    (north_star: <= 1e-5 relative in fp32) and an absolute floor ATOL for
    values near zero where relative error is undefined: 1e-6 for the 3D chain
    (unit-variance voxels), 1e-5 for the normalised 2D chain (outputs O(1)).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 1
RTOL = 1e-5


@pytest.fixture(scope="module")
def ctx(lfgpu):
    if lfgpu.device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    c = lfgpu.Context(batch_size=8, n_workers=8, max_group=4, max_slot_buffers=16, seed=SEED)
    yield c
    c.close()


def _upload(ctx, arr):
    p = ctx.device_alloc(arr.nbytes)
    ctx.h2d(p, np.ascontiguousarray(arr))
    return p


def _pinned(ctx, arr):
    p = ctx.host_alloc(arr.nbytes)
    import ctypes
    ctypes.memmove(p, arr.ctypes.data, arr.nbytes)
    return p


def _assert_close(got, want, atol):
    err = np.abs(got.astype(np.float64) - want)
    bound = RTOL * np.abs(want) + atol
    bad = err > bound
    assert not bad.any(), (f"{bad.sum()} / {bad.size} values out of tolerance; "
                           f"max err {err.max():.3e}, worst ratio {(err / bound).max():.3f}")


# ------------------------------------------------------------------ img_seg (K1)
CASES_3D = [
    # (dims, crop, probability overrides)
    ((20, 24, 40), (16, 16, 32), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),
    ((20, 24, 40), (16, 16, 32), dict()),                                   # MLPerf defaults
    ((12, 30, 20), (16, 16, 32), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),  # zero padding
    ((16, 16, 32), (16, 16, 32), dict(p_flip=1.0, p_bright=0.0, p_noise=1.0)),  # exact fit
    ((136, 140, 150), (128, 128, 128), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),
    # W % 16 == 0: device-resident samples take the TMA tile path
    ((20, 24, 48), (16, 16, 32), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),   # x offset
    ((12, 30, 16), (16, 16, 32), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),   # zero padding (TMA OOB)
    ((24, 26, 64), (10, 20, 48), dict(p_flip=1.0, p_bright=0.0, p_noise=0.0)),   # partial tile + flips
    ((136, 140, 160), (128, 128, 128), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),
]


@pytest.mark.parametrize("src_kind", [0, 1], ids=["device", "host_pinned"])
@pytest.mark.parametrize("case", range(len(CASES_3D)))
def test_img3d_matches_oracle(ctx, lfgpu, oracle, case, src_kind):
    dims, crop, probs = CASES_3D[case]
    kw = dict(p_flip=1 / 3, p_bright=0.1, p_noise=0.1)
    kw.update(probs)
    ops = lfgpu.img_seg_ops(crop=crop, p_flip=kw["p_flip"], p_bright=kw["p_bright"],
                            p_noise=kw["p_noise"])
    ch = ctx.chain(ops)
    ocfg = oracle.cfg3d(crop=crop, p_flip=kw["p_flip"], p_bright=kw["p_bright"],
                        p_noise=kw["p_noise"])
    rng = np.random.default_rng(100 + case)
    n_ids = 3 if crop[0] == 128 else 12
    ids = [int(x) for x in rng.integers(0, 1 << 40, n_ids)]
    vox = int(np.prod(crop))
    bufs = []
    tickets = []
    expect = []
    for sid in ids:
        img = rng.standard_normal(dims).astype(np.float32)
        lbl = rng.integers(0, 3, dims, dtype=np.uint8)
        if src_kind == 0:
            pi, pl = _upload(ctx, img), _upload(ctx, lbl)
            bufs += [("d", pi), ("d", pl)]
        else:
            pi, pl = _pinned(ctx, img), _pinned(ctx, lbl)
            bufs += [("h", pi), ("h", pl)]
        desc = lfgpu.sample_desc(sid, dims, pi, pl, src_kind=src_kind)
        # host parameter draws are bit-identical to the oracle's
        p = ch.draw_params(SEED, desc)
        op_ = oracle.draw3d(ocfg, SEED, sid, dims)
        assert list(p[:3]) == list(op_.off) and list(p[3:6]) == list(op_.flip)
        assert p[6] == op_.scale and p[7] == op_.sigma and list(p[8:10]) == list(op_.key)
        tickets.append(ctx.submit(ch, desc))
        expect.append(oracle.apply3d(ocfg, op_, img, lbl))
    ctx.flush()
    for t, (e_img, e_lbl) in zip(tickets, expect):
        ctx.wait(t)
        od, done, _ = ctx.progress(t)
        assert done and od == len(ops)
        raw = ctx.ticket_output(t, vox * 4 + ((vox + 15) // 16) * 16)
        g_img = raw[: vox * 4].view(np.float32).reshape(crop)
        g_lbl = raw[vox * 4: vox * 5].reshape(crop)
        assert np.array_equal(g_lbl, e_lbl), "label crop/flip is not bit-exact"
        _assert_close(g_img, e_img, atol=1e-6)
        ctx.release(t)
    for kind, p in bufs:
        (ctx.device_free if kind == "d" else ctx.host_free)(p)
    ctx.destroy_chain(ch)


# ------------------------------------------------------------------ optional img_seg ops (K4 / K5)
CASES_ZC = [
    # (dims, crop, zoom, contrast, probability overrides)
    ((30, 34, 40), (16, 16, 32), (1.0, 0.7, 1.3), None, dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),
    ((20, 24, 48), (16, 16, 32), None, (1.0, 0.75, 1.25), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),  # K1 TMA + K5
    ((20, 24, 40), (16, 16, 32), None, (1.0, 0.75, 1.25), dict(p_flip=0.5, p_bright=1.0, p_noise=0.0)),  # K1 row + K5
    ((30, 34, 40), (16, 16, 32), (1.0, 0.7, 1.3), (1.0, 0.5, 1.5), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),
    ((12, 14, 20), (16, 16, 32), (1.0, 0.8, 1.2), (1.0, 0.75, 1.25), dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),  # zero pad
    ((140, 150, 160), (128, 128, 128), (0.5, 0.8, 1.2), (0.5, 0.75, 1.25), dict()),
    ((14, 12, 260), (8, 8, 200), (1.0, 0.8, 1.2), None, dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)),  # W > 128, ragged
]


@pytest.mark.parametrize("src_kind", [0, 1], ids=["device", "host_pinned"])
@pytest.mark.parametrize("case", range(len(CASES_ZC)))
def test_img3d_zoom_contrast_matches_oracle(ctx, lfgpu, oracle, case, src_kind):
    """RandomZoom3D (K4: trilinear image, nearest label) and RandomContrast (K5 crop
    sum + the affine in K1 / K4) against the oracle: labels bit-exact, window and
    contrast draws exact, image within the 3D tolerance."""
    dims, crop, zoom, contrast, probs = CASES_ZC[case]
    kw = dict(p_flip=1 / 3, p_bright=0.1, p_noise=0.1)
    kw.update(probs)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, zoom=zoom, contrast=contrast, **kw))
    okw = dict(kw)
    if zoom is not None:
        okw.update(has_zoom=1, p_zoom=zoom[0], zoom_lo=zoom[1], zoom_hi=zoom[2])
    if contrast is not None:
        okw.update(has_contrast=1, p_contrast=contrast[0], contrast_lo=contrast[1],
                   contrast_hi=contrast[2])
    ocfg = oracle.cfg3d(crop=crop, **okw)
    rng = np.random.default_rng(300 + case)
    ids = [int(x) for x in rng.integers(0, 1 << 40, 4 if crop[0] == 128 else 10)]
    vox = int(np.prod(crop))
    bufs, tickets, expect = [], [], []
    for sid in ids:
        img = (rng.standard_normal(dims) + 0.5).astype(np.float32)
        lbl = rng.integers(0, 3, dims, dtype=np.uint8)
        if src_kind == 0:
            pi, pl = _upload(ctx, img), _upload(ctx, lbl)
            bufs += [("d", pi), ("d", pl)]
        else:
            pi, pl = _pinned(ctx, img), _pinned(ctx, lbl)
            bufs += [("h", pi), ("h", pl)]
        desc = lfgpu.sample_desc(sid, dims, pi, pl, src_kind=src_kind)
        p = ch.draw_params(SEED, desc)
        op_ = oracle.draw3d(ocfg, SEED, sid, dims)
        assert list(p[:3]) == list(op_.off) and list(p[3:6]) == list(op_.flip)
        assert p[6] == op_.scale and p[7] == op_.sigma and list(p[8:10]) == list(op_.key)
        assert list(p[10:13]) == list(op_.win) and p[13] == op_.contrast
        tickets.append(ctx.submit(ch, desc))
        expect.append(oracle.apply3d(ocfg, op_, img, lbl))
    ctx.flush()
    for t, (e_img, e_lbl) in zip(tickets, expect):
        ctx.wait(t)
        raw = ctx.ticket_output(t, vox * 4 + ((vox + 15) // 16) * 16)
        g_img = raw[: vox * 4].view(np.float32).reshape(crop)
        g_lbl = raw[vox * 4: vox * 5].reshape(crop)
        assert np.array_equal(g_lbl, e_lbl), "label resample/crop/flip is not bit-exact"
        _assert_close(g_img, e_img, atol=1e-6)
        ctx.release(t)
    for kind, p in bufs:
        (ctx.device_free if kind == "d" else ctx.host_free)(p)
    ctx.destroy_chain(ch)


# ------------------------------------------------------------------ foreground crop (K2)
@pytest.mark.parametrize("src_kind", [0, 1], ids=["device", "host_pinned"])
@pytest.mark.parametrize("case", range(4))
def test_img3d_foreground_crop_matches_oracle(ctx, lfgpu, oracle, case, src_kind):
    """RandomCrop with foreground oversampling (K2 label scan + window resolution on
    the device, then K1 TMA / row path, K4 with zoom, K5 with contrast): labels
    bit-exact and images within tolerance of the oracle, whose window origin is pinned
    to a numpy restatement in test_oracle."""
    dims, crop, extra = [
        ((40, 48, 64), (16, 16, 32), {}),                                   # TMA path
        ((40, 48, 60), (16, 16, 32), {}),                                   # row path (W % 16 != 0)
        ((40, 48, 64), (16, 16, 32), dict(zoom=(1.0, 0.8, 1.2))),            # K4
        ((40, 48, 64), (16, 16, 32), dict(contrast=(1.0, 0.75, 1.25))),      # K5 + K1
    ][case]
    kw = dict(p_flip=0.5, p_bright=1.0, p_noise=1.0)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, p_fg=0.6, **kw, **extra))
    okw = dict(kw, has_fg=1, p_fg=0.6)
    if "zoom" in extra:
        okw.update(has_zoom=1, p_zoom=1.0, zoom_lo=0.8, zoom_hi=1.2)
    if "contrast" in extra:
        okw.update(has_contrast=1, p_contrast=1.0, contrast_lo=0.75, contrast_hi=1.25)
    ocfg = oracle.cfg3d(crop=crop, **okw)
    rng = np.random.default_rng(400 + case)
    z, y, x = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    vox = int(np.prod(crop))
    bufs, tickets, expect, n_fg = [], [], [], 0
    for k in range(12):
        sid = int(rng.integers(0, 1 << 40))
        img = rng.standard_normal(dims).astype(np.float32)
        lbl = np.zeros(dims, np.uint8)
        c0 = rng.integers(8, np.array(dims) - 8)
        lbl[((z - c0[0]) / 5) ** 2 + ((y - c0[1]) / 6) ** 2 + ((x - c0[2]) / 7) ** 2 <= 1] = 1 + k % 3
        if k % 4 == 0:
            lbl[:] = 0                                           # no foreground: random offsets
        if src_kind == 0:
            pi, pl = _upload(ctx, img), _upload(ctx, lbl)
            bufs += [("d", pi), ("d", pl)]
        else:   # pinned: foreground samples stage the whole volume (the window needs the scan)
            pi, pl = _pinned(ctx, img), _pinned(ctx, lbl)
            bufs += [("h", pi), ("h", pl)]
        desc = lfgpu.sample_desc(sid, dims, pi, pl, src_kind=src_kind)
        p = ch.draw_params(SEED, desc)
        op_ = oracle.draw3d(ocfg, SEED, sid, dims)
        assert p[14] == op_.fg and p[15] == op_.u_cls and list(p[16:19]) == list(op_.u_adj)
        n_fg += oracle.fg_offsets(op_, lbl) is not None
        tickets.append(ctx.submit(ch, desc))
        expect.append(oracle.apply3d(ocfg, op_, img, lbl))
    ctx.flush()
    for t, (e_img, e_lbl) in zip(tickets, expect):
        ctx.wait(t)
        raw = ctx.ticket_output(t, vox * 4 + ((vox + 15) // 16) * 16)
        assert np.array_equal(raw[vox * 4: vox * 5].reshape(crop), e_lbl), "label window differs"
        _assert_close(raw[: vox * 4].view(np.float32).reshape(crop), e_img, atol=1e-6)
        ctx.release(t)
    assert n_fg >= 2
    for kind, p in bufs:
        (ctx.device_free if kind == "d" else ctx.host_free)(p)
    ctx.destroy_chain(ch)


# ------------------------------------------------------------------ obj_det (K3)
@pytest.mark.parametrize("src_kind", [0, 1], ids=["device", "host_pinned"])
def test_rrc2d_matches_oracle(ctx, lfgpu, oracle, src_kind):
    ch = ctx.chain(lfgpu.obj_det_ops())
    ocfg = oracle.cfg2d()
    rng = np.random.default_rng(7 + src_kind)
    bufs, tickets, expect = [], [], []
    for k in range(24):
        sid = int(rng.integers(0, 1 << 40))
        H, W = (int(x) for x in rng.integers(256, 513, 2))
        if k == 0:
            H, W = 40, 500     # extreme aspect -> centre-crop fallback
        if k == 1:
            H, W = 100, 100    # upsampling
        if k == 2:
            H, W = 1400, 1200  # tall crop boxes: the row window exceeds shared memory -> L2 taps
        img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        p = _upload(ctx, img) if src_kind == 0 else _pinned(ctx, img)
        bufs.append(p)
        desc = lfgpu.sample_desc(sid, (H, W, 3), p, src_kind=src_kind)
        dp = ch.draw_params(SEED, desc)
        op_ = oracle.draw2d(ocfg, SEED, sid, H, W)
        assert list(dp) == [op_.top, op_.left, op_.h, op_.w, op_.flip]
        tickets.append(ctx.submit(ch, desc))
        expect.append(oracle.apply2d(ocfg, op_, img))
    ctx.flush()
    for t, e in zip(tickets, expect):
        ctx.wait(t)
        raw = ctx.ticket_output(t, 3 * 224 * 224 * 4)
        _assert_close(raw.view(np.float32).reshape(3, 224, 224), e, atol=1e-5)
        ctx.release(t)
    for p in bufs:
        (ctx.device_free if src_kind == 0 else ctx.host_free)(p)
    ctx.destroy_chain(ch)


# ------------------------------------------------------------------ batches
def test_seal_in_place_and_gather(ctx, lfgpu, oracle):
    """A batch sealed from exactly one slot buffer is zero-copy; any other
    composition is collated by the gather kernel; both hold the same bytes as
    the per-sample outputs."""
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0))
    ocfg = oracle.cfg3d(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0)
    B = ctx.cfg.batch_size
    dims = (10, 12, 20)
    rng = np.random.default_rng(3)
    img = rng.standard_normal(dims).astype(np.float32)
    lbl = rng.integers(0, 3, dims, dtype=np.uint8)
    pi, pl = _upload(ctx, img), _upload(ctx, lbl)
    ids = list(range(1000, 1000 + 2 * B))
    ts = [ctx.submit(ch, lfgpu.sample_desc(i, dims, pi, pl)) for i in ids]
    ctx.flush()
    for t in ts:
        ctx.wait(t)
    vox = int(np.prod(crop))
    exp = {i: oracle.chain3d(ocfg, SEED, i, img, lbl)[0] for i in ids}

    def check_batch(b, want_ids, in_place):
        info = ctx.batch_info(b)
        assert info["in_place"] == in_place
        assert sorted(info["ids"]) == sorted(want_ids)
        host = ctx.batch_to_host(b, info["n"] * (vox * 4 + ((vox + 15) // 16) * 16))
        n = info["n"]
        imgs = host[: n * vox * 4].view(np.float32).reshape(n, *crop)
        lbls = host[n * vox * 4: n * vox * 4 + n * vox].reshape(n, *crop)
        for k, sid in enumerate(info["ids"]):
            assert np.array_equal(lbls[k], exp[sid][1])
            _assert_close(imgs[k], exp[sid][0], atol=1e-6)

    b0 = ctx.seal(ts[:B][::-1])                         # exactly buffer 0, any order
    check_batch(b0, ids[:B], True)
    mixed = ts[B: B + B // 2] + ts[B + B // 2:][:B // 2]
    b1 = ctx.seal(mixed[: B - 1])                       # not the whole buffer -> gather
    check_batch(b1, [ids[ts.index(t)] for t in mixed[: B - 1]], False)
    ctx.batch_release(b0)
    ctx.batch_release(b1)
    rest = [t for t in ts[B:] if t not in mixed[: B - 1]]
    for t in rest:
        ctx.release(t)
    with pytest.raises(lfgpu.LfgError):
        ctx.seal([ts[0]])                               # already consumed
    ctx.synchronize()
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)


def test_progress_reports_stage_boundaries(ctx, lfgpu):
    """A spin stage before the fused kernel gives ops_done = 1 while the kernel is pending."""
    ops = lfgpu.img_seg_ops(crop=(8, 8, 16), spin_first=True)
    ch = ctx.chain(ops)
    assert ch.stages() == [(0, 1), (1, 6)]
    dims = (8, 8, 16)
    img = np.zeros(dims, np.float32)
    lbl = np.zeros(dims, np.uint8)
    pi, pl = _upload(ctx, img), _upload(ctx, lbl)
    t = ctx.submit(ch, lfgpu.sample_desc(5, dims, pi, pl, spin_us=[200_000]))
    ctx.flush()
    od, done, _ = ctx.progress(t)
    assert not done and od == 0
    ctx.wait(t)
    od, done, el = ctx.progress(t)
    assert done and od == 6 and el >= 150_000
    costs = ctx.exec_costs(t, len(ops))
    assert costs[0] >= 190_000            # the spin op's device time (us)
    ctx.release(t)
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)


# ------------------------------------------------------------------ shard loop
def test_shard_scheduler_adapts_in_flight_groups(lfgpu):
    """SURVEY 8(f) row 1 on the device: the reference's Eq. 1-2 rule resizes the number
    of in-flight launch groups.  Loader-bound (no trainer, every sample a 300 us cost,
    empty consumer queue, saturated slots): the count grows to its bound.  Trainer-bound
    (a 3 ms trainer step per batch: delivered batches pile up): it shrinks.  Exactly-once
    delivery holds throughout."""
    ctx = lfgpu.Context(batch_size=4, n_workers=4, max_group=1, max_slot_buffers=12, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, spin_first=True))
    dims = (10, 10, 20)
    rng = np.random.default_rng(12)
    pi = _upload(ctx, rng.standard_normal(dims).astype(np.float32))
    pl = _upload(ctx, rng.integers(0, 3, dims, dtype=np.uint8))
    n = 600
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[300]) for i in range(n)]
    grow = lfgpu.run_config(batch_size=4, n_workers=4, scheduler=1, max_workers=12, sched_tick_us=500)
    rep, ids, _, _ = ctx.run_shard(ch, descs, grow)
    assert rep.exactly_once == 1 and sorted(ids.tolist()) == list(range(n))
    assert rep.sched_ticks > 5 and rep.final_workers == 12 and rep.mean_workers > 4
    shrink = lfgpu.run_config(batch_size=4, n_workers=8, trainer_us=3000, scheduler=1, max_workers=12,
                              sched_tick_us=500)
    descs = [lfgpu.sample_desc(n + i, dims, pi, pl, spin_us=[50]) for i in range(200)]
    rep, ids, _, _ = ctx.run_shard(ch, descs, shrink)
    assert rep.exactly_once == 1 and sorted(ids.tolist()) == list(range(n, n + 200))
    assert rep.sched_ticks > 5 and rep.final_workers < 8 and rep.mean_workers < 8
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


def test_shard_sync_baseline_is_head_of_line(lfgpu):
    """SURVEY 8(f) row 3 on the device: policy 3 is the reference's synchronous loader
    (baselines.cpp:12-151) -- batch k holds exactly ids [kB, (k+1)B), in order, so one
    slow sample holds back its batch; the Minato policy on the same stream seals fast
    samples around it, and the synthetic trainer idles less."""
    ctx = lfgpu.Context(batch_size=4, n_workers=8, max_group=1, max_slot_buffers=24, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, spin_first=True))
    dims = (10, 10, 20)
    rng = np.random.default_rng(13)
    pi = _upload(ctx, rng.standard_normal(dims).astype(np.float32))
    pl = _upload(ctx, rng.integers(0, 3, dims, dtype=np.uint8))
    n = 160
    heavy = set(range(2, n, 9))
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[6_000 if i in heavy else 300]) for i in range(n)]
    rep_s, ids_s, bsz_s, _ = ctx.run_shard(ch, descs, lfgpu.run_config(batch_size=4, policy=3, trainer_us=400))
    assert rep_s.exactly_once == 1 and rep_s.slow == 0
    assert ids_s.tolist() == list(range(n))                 # FIFO batches of consecutive ids
    assert (bsz_s == 4).all()
    rep_m, ids_m, _, _ = ctx.run_shard(ch, descs, lfgpu.run_config(batch_size=4, policy=0, t_out_us=2_000,
                                                                     trainer_us=400))
    assert rep_m.exactly_once == 1 and rep_m.slow == len(heavy)
    assert ids_m.tolist() != list(range(n))                 # eager: fast samples overtake
    assert rep_m.consumer_idle_frac < rep_s.consumer_idle_frac
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


def test_shard_sync_prefetch_sweep(lfgpu):
    """test_baselines.cpp:182-209 on the device: the synchronous loader (policy 3) with
    a claim window of prefetch_factor x workers batches; preprocessing-bound (batch 24 >=
    12 workers, lognormal costs), so the window size changes the completion time by
    little -- the reference bounds it at 5% on its virtual clock, the device run at 15%
    (real streams, best of 3) -- and every prefetch factor delivers FIFO batches exactly once."""
    ctx = lfgpu.Context(batch_size=24, n_workers=12, max_group=1, max_slot_buffers=48, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, spin_first=True))
    dims = (10, 10, 20)
    rng = np.random.default_rng(23)
    pi = _upload(ctx, rng.standard_normal(dims).astype(np.float32))
    pl = _upload(ctx, rng.integers(0, 3, dims, dtype=np.uint8))
    n = 480
    cost_us = np.minimum(1500.0, rng.lognormal(np.log(100.0), 0.5, n)) * 4 + 4
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[int(cost_us[i])]) for i in range(n)]
    elapsed = {}
    for k in (1, 2, 4, 8):
        best = None
        for _ in range(3):
            rep, ids, bsz, _ = ctx.run_shard(ch, descs, lfgpu.run_config(batch_size=24, policy=3, n_workers=12,
                                                                         prefetch_factor=k))
            assert rep.exactly_once == 1 and ids.tolist() == list(range(n)) and (bsz == 24).all()
            best = rep.elapsed_ms if best is None else min(best, rep.elapsed_ms)
        elapsed[k] = best
    for k in (2, 4, 8):
        assert abs(elapsed[k] - elapsed[1]) / elapsed[1] < 0.15, elapsed
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


def test_shard_sync_prefetch_window_bounds_feed(lfgpu):
    """The claim window binds: with one worker-batch of prefetch and a head-of-line
    sample costing 30 ms, at most prefetch_factor x workers batches of the cheap samples
    behind it are fed, so the run takes about the slow sample plus the rest run after it
    (not overlapped with it); unbounded (0) overlaps them."""
    ctx = lfgpu.Context(batch_size=4, n_workers=2, max_group=1, max_slot_buffers=24, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, spin_first=True))
    dims = (10, 10, 20)
    rng = np.random.default_rng(29)
    pi = _upload(ctx, rng.standard_normal(dims).astype(np.float32))
    pl = _upload(ctx, rng.integers(0, 3, dims, dtype=np.uint8))
    n = 64
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[30_000 if i == 0 else 1_000]) for i in range(n)]
    t = {}
    for k in (1, 0):
        rep, ids, _, _ = ctx.run_shard(ch, descs, lfgpu.run_config(batch_size=4, policy=3, n_workers=2,
                                                                   prefetch_factor=k))
        assert rep.exactly_once == 1 and ids.tolist() == list(range(n))
        t[k] = rep.elapsed_ms
    # window 1 x 2 workers = 8 samples: ~7 cheap samples overlap the slow one, the other
    # 56 run after it on 2 streams (~28 ms); unbounded, ~30 of them overlap it
    assert t[1] > t[0] + 8.0, t
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


def test_shard_recycles_finished_tables(lfgpu):
    """A run reuses the ticket / group storage of earlier runs once nothing references
    it (Context::recycle_tables): repeated runs stay exactly-once with identical
    outputs order-independently, the ticket numbering restarts, and a ticket the user
    still holds blocks the recycling (its handle stays valid)."""
    ctx = lfgpu.Context(batch_size=4, n_workers=4, max_group=2, max_slot_buffers=16, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop))
    dims = (10, 10, 20)
    rng = np.random.default_rng(31)
    pi = _upload(ctx, rng.standard_normal(dims).astype(np.float32))
    pl = _upload(ctx, rng.integers(0, 3, dims, dtype=np.uint8))
    n = 40
    descs = [lfgpu.sample_desc(i, dims, pi, pl) for i in range(n)]
    rc = lfgpu.run_config(batch_size=4, n_workers=4)
    for _ in range(3):
        rep, ids, _, _ = ctx.run_shard(ch, descs, rc)
        assert rep.exactly_once == 1 and sorted(ids.tolist()) == list(range(n))
    # three runs of n: the third started from an empty table, so the next ticket is n
    t = ctx.submit(ch, descs[0])
    assert t == n
    ctx.flush()
    ctx.wait(t)
    vox = crop[0] * crop[1] * crop[2]
    nbytes = vox * 4 + ((vox + 15) // 16) * 16
    held = ctx.ticket_output(t, nbytes)       # the held ticket is readable ...
    rep, ids, _, _ = ctx.run_shard(ch, descs, rc)
    assert rep.exactly_once == 1
    assert (ctx.ticket_output(t, nbytes) == held).all()   # ... and not recycled under the user
    t2 = ctx.submit(ch, descs[1])
    assert t2 == 2 * n + 1                     # tables kept: n (run 3) + 1 (held) + n (run 4)
    ctx.flush()
    ctx.wait(t2)
    ctx.release(t)
    ctx.release(t2)
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


def test_shard_exactly_once_fast_first(lfgpu):
    """Algorithm 1 on the device: samples whose synthetic cost exceeds t_out are
    classified slow, finish in the background and are batched after the fast
    ones; every id is delivered exactly once.  (One sample per launch group, so
    classification is per sample.)"""
    ctx = lfgpu.Context(batch_size=8, n_workers=6, max_group=1, max_slot_buffers=16, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, spin_first=True))
    dims = (10, 10, 20)
    rng = np.random.default_rng(11)
    img = rng.standard_normal(dims).astype(np.float32)
    lbl = rng.integers(0, 3, dims, dtype=np.uint8)
    pi, pl = _upload(ctx, img), _upload(ctx, lbl)
    n = 96
    heavy = set(range(3, n, 10))
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[40_000 if i in heavy else 200])
             for i in range(n)]
    rc = lfgpu.run_config(batch_size=8, t_out_us=10_000, policy=0, n_workers=6)
    rep, ids, bsz, cls = ctx.run_shard(ch, descs, rc)
    assert rep.exactly_once == 1 and rep.duplicates == 0
    assert sorted(ids.tolist()) == list(range(n))
    assert rep.slow == len(heavy) and rep.fast == n - len(heavy)
    assert all(cls[i] == (2 if i in heavy else 1) for i in range(n))
    assert bsz.sum() == n
    # a heavy (slow) sample never appears before the fast ones submitted with it
    pos = {int(s): k for k, s in enumerate(ids)}
    for h in heavy:
        assert pos[h] > pos.get(h + 1, -1) or h + 1 >= n
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


def test_shard_classifies_per_sample_inside_wide_groups(lfgpu, oracle):
    """balancer.cpp:42-77 classifies each sample; here 16 samples share one launch
    group (one kernel per stage) and each sample's last kernel part stamps its own
    completion, so a group holding a slow sample (a 30 ms HeavyStep, t_out 8 ms)
    hands its fast members on as soon as they finish: the slow set is exactly the
    heavy samples, every fast member of a group is delivered before its slow one,
    and the delivered outputs still match the oracle."""
    ctx = lfgpu.Context(batch_size=2, n_workers=4, max_group=16, max_slot_buffers=48, seed=SEED)
    crop = (8, 8, 16)
    ops = lfgpu.img_seg_ops(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0) + [
        lfgpu.op(lfgpu.OP_SPIN, "HeavyStep")]
    ch = ctx.chain(ops)
    ocfg = oracle.cfg3d(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0)
    dims = (10, 12, 20)
    rng = np.random.default_rng(41)
    img = rng.standard_normal(dims).astype(np.float32)
    lbl = rng.integers(0, 3, dims, dtype=np.uint8)
    pi, pl = _upload(ctx, img), _upload(ctx, lbl)
    n = 64
    heavy = {3, 9, 14, 21, 40, 47, 50}
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[30_000 if i in heavy else 200]) for i in range(n)]
    rc = lfgpu.run_config(batch_size=2, t_out_us=8_000, policy=0, n_workers=4)
    rep, ids, bsz, cls = ctx.run_shard(ch, descs, rc, capture=list(range(n)))
    assert rep.exactly_once == 1 and sorted(ids.tolist()) == list(range(n))
    assert {i for i in range(n) if cls[i] == 2} == heavy and rep.slow == len(heavy)
    pos = {int(s): k for k, s in enumerate(ids)}
    for h in heavy:
        mates = [i for i in range(16 * (h // 16), 16 * (h // 16) + 16) if i not in heavy]
        assert all(pos[m] < pos[h] for m in mates), f"a fast member of {h}'s group waited for it"
    vox = int(np.prod(crop))
    for p_, (raw, _) in ctx.last_capture.items():
        (e_img, e_lbl), _ = oracle.chain3d(ocfg, SEED, p_, img, lbl)
        assert np.array_equal(raw[vox * 4: vox * 5].reshape(crop), e_lbl)
        _assert_close(raw[: vox * 4].view(np.float32).reshape(crop), e_img, atol=1e-6)
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


@pytest.mark.parametrize("family", ["img3d_tma", "img3d_rows", "rrc", "speech"])
def test_transform_kernel_stamps(lfgpu, oracle, family):
    """lfg_run_config.sample_stamps = 1: the transform kernels themselves stamp every
    sample (per-CTA / per-tile release + count) inside launch groups of 16; the shard
    hands samples on one by one, and every delivered output still matches the oracle."""
    B = 2 if family.startswith("img3d") else 4
    ctx = lfgpu.Context(batch_size=B, n_workers=4, max_group=16, max_slot_buffers=48, seed=SEED)
    rng = np.random.default_rng(47)
    bufs, descs, check = [], [], {}
    if family.startswith("img3d"):
        crop = (16, 16, 32)
        ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0))
        ocfg = oracle.cfg3d(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0)
        dims = (20, 24, 48) if family == "img3d_tma" else (20, 24, 40)
        img = rng.standard_normal(dims).astype(np.float32)
        lbl = rng.integers(0, 3, dims, dtype=np.uint8)
        pi, pl = _upload(ctx, img), _upload(ctx, lbl)
        bufs += [pi, pl]
        vox = int(np.prod(crop))
        descs = [lfgpu.sample_desc(i, dims, pi, pl) for i in range(48)]

        def check(i, raw):
            (e_img, e_lbl), _ = oracle.chain3d(ocfg, SEED, i, img, lbl)
            assert np.array_equal(raw[vox * 4: vox * 5].reshape(crop), e_lbl)
            _assert_close(raw[: vox * 4].view(np.float32).reshape(crop), e_img, atol=1e-6)
    elif family == "rrc":
        ch = ctx.chain(lfgpu.obj_det_ops())
        ocfg = oracle.cfg2d()
        imgs = [rng.integers(0, 256, (int(h), int(w), 3), dtype=np.uint8)
                for h, w in rng.integers(200, 400, (48, 2))]
        for i, im in enumerate(imgs):
            p = _upload(ctx, im)
            bufs.append(p)
            descs.append(lfgpu.sample_desc(i, im.shape, p))

        def check(i, raw):
            e, _ = oracle.chain2d(ocfg, SEED, i, imgs[i])
            _assert_close(raw[: 3 * 224 * 224 * 4].view(np.float32).reshape(3, 224, 224), e, atol=1e-5)
    else:
        import checks
        ch = ctx.chain(lfgpu.speech_ops(max_len=40000))
        ocfg = oracle.cfgsp()
        waves = [(0.3 * rng.standard_normal(int(L))).astype(np.float32) for L in rng.integers(1000, 40000, 48)]
        for i, w in enumerate(waves):
            p = _upload(ctx, w)
            bufs.append(p)
            descs.append(lfgpu.sample_desc(i, w.shape, p))

        def check(i, raw):
            assert checks.check_speech(oracle, ocfg, SEED, i, waves[i], raw) <= 1.0
    rc = lfgpu.run_config(batch_size=B, n_workers=4, sample_stamps=1)
    rep, ids, _, _ = ctx.run_shard(ch, descs, rc, capture=list(range(len(descs))))
    assert rep.exactly_once == 1 and len(ctx.last_capture) == len(descs)
    for i, (raw, _) in ctx.last_capture.items():
        check(i, raw)
    for p in bufs:
        ctx.device_free(p)
    ctx.destroy_chain(ch)
    ctx.close()


def test_device_profiler_escalates_and_deescalates(lfgpu):
    """The device profiler (policy 1) on per-sample device-timed totals, as the
    reference Profiler (test_profiler.cpp:83-115, profiler.cpp:47-72): with 60% of
    samples over the initial budget the slow rate exceeds 0.35 and t_out escalates
    from p75 to p90; once a full window of fast records follows, it falls back to
    p75.  One record per sample."""
    ctx = lfgpu.Context(batch_size=4, n_workers=8, max_group=4, max_slot_buffers=40, seed=SEED)
    crop = (8, 8, 16)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop) + [lfgpu.op(lfgpu.OP_SPIN, "HeavyStep")])
    dims = (10, 10, 20)
    rng = np.random.default_rng(43)
    pi = _upload(ctx, rng.standard_normal(dims).astype(np.float32))
    pl = _upload(ctx, rng.integers(0, 3, dims, dtype=np.uint8))
    rc = lfgpu.run_config(batch_size=4, policy=1, t_out_us=1_000, warmup_us=0, update_interval_us=1_000,
                          window=40, n_workers=8)
    # (a) 60% heavy throughout: escalation
    descs = [lfgpu.sample_desc(i, dims, pi, pl, spin_us=[3_000 if i % 5 < 3 else 100]) for i in range(200)]
    rep, ids, _, _ = ctx.run_shard(ch, descs, rc)
    assert rep.exactly_once == 1 and rep.profiled == 200
    assert rep.pct_up >= 1, rep.as_dict()
    # (b) a heavy phase, then a long light phase that refills the window with fast records
    descs = [lfgpu.sample_desc(1000 + i, dims, pi, pl, spin_us=[3_000 if (i < 200 and i % 5 < 3) else 150])
             for i in range(1400)]
    rep, ids, _, _ = ctx.run_shard(ch, descs, rc)
    assert rep.exactly_once == 1 and rep.profiled == 1400
    d = rep.as_dict()
    assert rep.pct_up >= 1 and rep.pct_down >= 1 and rep.final_percentile == 75, {
        k: d[k] for k in ("fast", "slow", "pct_up", "pct_down", "final_percentile", "final_t_out_us")}
    ctx.device_free(pi)
    ctx.device_free(pl)
    ctx.destroy_chain(ch)
    ctx.close()


# ------------------------------------------------------------------ reference-shaped C++ API
def test_cpp_api_device_pipeline():
    """process_sample / resume_slow / build_batches / run_consumer (the reference
    signatures, include/loadflow) drive the GPU path end to end; delivered outputs
    of the C++ path are compared with the oracle (lf_oracle.c) inside the program."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2509_10712_b200")
    exe = os.path.join(root, "tests", "cpp", "device_pipeline")
    src = os.path.join(root, "tests", "cpp", "device_pipeline.cpp")
    ora = os.path.join(root, "oracle")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"), src, "-o", exe,
                               "-L", pkg, "-lloadflow_b200", "-llfgpu", f"-Wl,-rpath,{pkg}",
                               "-L", ora, "-llf_oracle", f"-Wl,-rpath,{ora}", "-lpthread"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr


# ------------------------------------------------------------------ speech (K8-K11)
def _splice(logmel, stack=3):
    """FrameSplicing (stack, subsample) of the oracle's [80, T] log-mel -> [T', 80*stack]."""
    m, T = logmel.shape
    rows = (T + stack - 1) // stack
    out = np.zeros((rows, m * stack))
    for s in range(stack):
        idx = np.arange(rows) * stack + s
        ok = idx < T
        out[ok, s * m:(s + 1) * m] = logmel[:, idx[ok]].T
    return out


def test_speech_pinned_host_source_matches_device(lfgpu, oracle):
    """Speech from pinned host memory (the e2e path: every waveform of the launch
    group is one K0 row read over PCIe) produces bit-identical outputs to HBM-resident input."""
    ctx = lfgpu.Context(batch_size=8, n_workers=4, max_group=8, max_slot_buffers=8, seed=SEED)
    ch = ctx.chain(lfgpu.speech_ops(max_len=40000))
    rng = np.random.default_rng(22)
    lens = [4000, 4321, 20000, 39999, 257, 300, 16000, 12345]
    dev, host, keep = [], [], []
    for k, L in enumerate(lens):
        wav = (0.3 * rng.standard_normal(L)).astype(np.float32)
        pd = _upload(ctx, wav)
        ph = _pinned(ctx, wav)
        keep += [("d", pd), ("h", ph)]
        dev.append(ctx.submit(ch, lfgpu.sample_desc(500 + k, (L,), pd)))
        host.append(ctx.submit(ch, lfgpu.sample_desc(500 + k, (L,), ph, src_kind=lfgpu.SRC_HOST_PINNED)))
    ctx.flush()
    _, out_bytes, _ = ch.info()
    for L, td, th in zip(lens, dev, host):
        ctx.wait(td)
        ctx.wait(th)
        rows = -(-(1 + L // 160) // 3)                   # spliced rows the kernel writes
        a = ctx.ticket_output(td, out_bytes).view(np.float32)[: rows * 240]
        b = ctx.ticket_output(th, out_bytes).view(np.float32)[: rows * 240]
        bad = np.flatnonzero(a != b)
        assert bad.size == 0, (f"{bad.size} of {a.size} differ; first {bad[:5]}, "
                               f"dev {a[bad[:5]]}, host {b[bad[:5]]}")
        ctx.release(td)
        ctx.release(th)
    for kind, p in keep:
        (ctx.device_free if kind == "d" else ctx.host_free)(p)
    ctx.close()


def test_speech_pcm16_equals_its_f32_image(lfgpu, oracle):
    """int16 PCM input (FilterBank param 5 = LFG_DT_I16; the reference's speech bytes_in
    are 2 B per sample, workloads.cpp:115): the kernel reads s / 32768, which is exact in
    fp32, so every output equals the f32 path's on the waveform s / 32768 bit for bit --
    HBM-resident and pinned, 4-B-aligned (paired loads) and 2-B-aligned (scalar loads)
    waveforms, reflect-padded ends, full-scale samples; plus the oracle bar on the PCM run."""
    ctx = lfgpu.Context(batch_size=8, n_workers=4, max_group=8, max_slot_buffers=8, seed=SEED)
    ch16 = ctx.chain(lfgpu.speech_ops(max_len=40000, pcm16=True))
    ch32 = ctx.chain(lfgpu.speech_ops(max_len=40000))
    ocfg = oracle.cfgsp()
    rng = np.random.default_rng(23)
    lens = [4000, 4321, 20000, 39999, 257, 300, 16000, 12345]
    keep, runs = [], []
    for k, L in enumerate(lens):
        t = np.arange(L) / 16000.0
        x = 0.6 * np.sin(2 * np.pi * (150 + 70 * k) * t) + 0.05 * rng.standard_normal(L)
        pcm = np.clip(np.rint(x * 32768), -32768, 32767).astype(np.int16)
        pcm[:3] = [32767, -32768, 0]                     # full scale inside the reflected edge
        f32 = pcm.astype(np.float32) / np.float32(32768.0)
        assert np.array_equal((f32 * 32768).astype(np.int16), pcm)
        mis = k % 2                                      # odd samples start 2 B past a 4-B boundary
        raw16 = np.zeros(L + 1, dtype=np.int16)
        raw16[mis:mis + L] = pcm
        pd, ph, p32 = _upload(ctx, raw16), _pinned(ctx, raw16), _upload(ctx, f32)
        keep += [("d", pd), ("h", ph), ("d", p32)]
        sid = 700 + k
        a = ctx.submit(ch16, lfgpu.sample_desc(sid, (L,), pd + 2 * mis))
        b = ctx.submit(ch16, lfgpu.sample_desc(sid, (L,), ph + 2 * mis, src_kind=lfgpu.SRC_HOST_PINNED))
        c = ctx.submit(ch32, lfgpu.sample_desc(sid, (L,), p32))
        runs.append((L, sid, f32, a, b, c))
    ctx.flush()
    _, out_bytes, _ = ch16.info()
    assert ch32.info()[1] == out_bytes
    for L, sid, f32, a, b, c in runs:
        rows = -(-(1 + L // 160) // 3)
        outs = []
        for tk in (a, b, c):
            ctx.wait(tk)
            outs.append(ctx.ticket_output(tk, out_bytes).view(np.float32)[: rows * 240].copy())
            ctx.release(tk)
        for got in outs[:2]:
            bad = np.flatnonzero(got != outs[2])
            assert bad.size == 0, f"L={L}: {bad.size} outputs differ from the f32 path; first {bad[:5]}"
        (lm, _), _ = oracle.chainsp(ocfg, SEED, sid, f32)
        e = _splice(lm)
        got = outs[0].reshape(-1, 240)[: e.shape[0]]
        zero = e == 0.0
        assert np.array_equal(got[zero], e[zero])
        ge, oe = np.exp(got[~zero].astype(np.float64)), np.exp(e[~zero])
        frame_peak = np.exp(e.reshape(e.shape[0], 3, 80).max(axis=2)).repeat(80, axis=1)[~zero]
        assert (np.abs(ge - oe) <= 1e-5 * oe + 1e-8 * frame_peak).all()
    # a PCM waveform must be 2-B aligned; FilterBank takes f32 or int16 input only
    with pytest.raises(lfgpu.LfgError) as ei:
        ctx.submit(ch16, lfgpu.sample_desc(799, (4000,), keep[0][1] + 1))
    assert ei.value.code == lfgpu.ERR_INVALID
    bad = lfgpu.speech_ops(max_len=40000)
    bad[2].param[5] = lfgpu.DT_U8
    with pytest.raises(lfgpu.LfgError) as ei:
        ctx.chain(bad)
    assert ei.value.code == lfgpu.ERR_UNSUPPORTED
    for kind, p in keep:
        (ctx.device_free if kind == "d" else ctx.host_free)(p)
    ctx.close()


def test_speech_matches_oracle(lfgpu, oracle):
    """STFT power (the FFT kernel; LFG_SPEECH_KERNEL=tc: tcgen05 3xTF32) -> mel -> log ->
    SpecAugment -> splicing.  Tolerance (stated): compared in the mel-energy domain,
    |e^g - e^o| <= 1e-5 e^o + 1e-8 * (frame's peak mel energy) -- relative 1e-5 with an
    energy floor for near-empty bands, where log amplifies fp32 round-off (measured need:
    7.6e-10 for the FFT kernel; the tcgen05 A/B kernel needs up to 1.2e-8 on 170 k-sample
    utterances and is not held to this bar); masked entries exactly 0."""
    ctx = lfgpu.Context(batch_size=8, n_workers=4, max_group=8, max_slot_buffers=8, seed=SEED)
    ch = ctx.chain(lfgpu.speech_ops(max_len=40000))
    ocfg = oracle.cfgsp()
    rng = np.random.default_rng(21)
    lens = [4000, 4321, 20000, 39999, 257, 300, 16000, 12345]
    ts, exp, bufs = [], [], []
    for k, L in enumerate(lens):
        t = np.arange(L) / 16000.0
        wav = (0.5 * np.sin(2 * np.pi * (200 + 50 * k) * t) + 0.2 * np.sin(2 * np.pi * 3100 * t)
               + 0.01 * rng.standard_normal(L)).astype(np.float32)
        p = ctx.device_alloc(wav.nbytes)
        ctx.h2d(p, wav)
        bufs.append(p)
        sid = 300 + k
        desc = lfgpu.sample_desc(sid, (L,), p)
        dp = ch.draw_params(SEED, desc)
        op_ = oracle.drawsp(ocfg, SEED, sid, L)
        assert dp[0] == op_.n_frames
        (lm, _), _ = oracle.chainsp(ocfg, SEED, sid, wav)
        exp.append(_splice(lm))
        ts.append(ctx.submit(ch, desc))
    ctx.flush()
    _, out_bytes, _ = ch.info()
    worst = 0.0
    per_ticket = []
    for t, e in zip(ts, exp):
        ctx.wait(t)
        got = ctx.ticket_output(t, out_bytes).view(np.float32).reshape(-1, 240)[: e.shape[0]]
        per_ticket.append(got.copy())
        zero = e == 0.0
        assert np.array_equal(got[zero], e[zero]), "SpecAugment / padding zeros differ"
        ge, oe = np.exp(got[~zero].astype(np.float64)), np.exp(e[~zero])
        frame_peak = np.exp(e.reshape(e.shape[0], 3, 80).max(axis=2)).repeat(80, axis=1)[~zero]
        err = np.abs(ge - oe)
        bound = 1e-5 * oe + 1e-8 * frame_peak
        worst = max(worst, float((err / bound).max()))
        assert (err <= bound).all(), f"max err/bound {(err / bound).max():.3f}"
    print("speech worst err/bound", worst)
    # batch collation: PermuteAudio + Pad -> [T'max, n, 240]
    b = ctx.seal(ts)
    lengths, t_max = ctx.batch_lengths(b)
    assert t_max == max(x.shape[0] for x in exp)
    host = ctx.batch_to_host(b, t_max * len(ts) * 240 * 4).view(np.float32).reshape(t_max, len(ts), 240)
    info = ctx.batch_info(b)
    for i, sid in enumerate(info["ids"]):
        e = exp[sid - 300]
        assert lengths[i] == e.shape[0]
        assert np.array_equal(host[lengths[i]:, i], np.zeros_like(host[lengths[i]:, i]))
        # collation is data movement: the batch rows are the sample's output, bit for bit
        assert np.array_equal(host[: lengths[i], i], per_ticket[sid - 300])
    ctx.batch_release(b)
    with pytest.raises(lfgpu.LfgError):                 # reflect padding needs L > n_fft / 2
        ctx.submit(ch, lfgpu.sample_desc(1, (256,), bufs[0]))
    ctx.synchronize()
    for p in bufs:
        ctx.device_free(p)
    ctx.close()
