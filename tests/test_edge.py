"""Edge cases of the device path (the reference's tests cover empty streams, short and
ragged batches and exactly-once at odd sizes: test_batcher.cpp:165-205,
test_core.cpp): empty shard runs and streams, batch size 1, a single sample, and
obj_det images at the size limits (1 x 1, extreme aspect ratios) against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 11


def _images(ctx, shapes, rng):
    out = []
    for H, W in shapes:
        im = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        p = ctx.device_alloc(im.nbytes)
        ctx.h2d(p, im)
        out.append((im, p))
    return out


def test_empty_shard_run_and_stream(lfgpu):
    ctx = lfgpu.Context(batch_size=4, n_workers=2, max_group=4, max_slot_buffers=4, seed=SEED)
    ch = ctx.chain(lfgpu.obj_det_ops())
    try:
        rep, ids, bsz, cls = ctx.run_shard(ch, [], lfgpu.run_config(batch_size=4))
        assert rep.samples == 0 and rep.batches == 0 and rep.exactly_once == 1
        assert len(ids) == 0 and len(bsz) == 0
        st = ctx.shard_stream(ch, [], lfgpu.run_config(batch_size=4))
        assert st.next_batch(timeout_us=1_000_000) is None          # end of stream at once
        rep2, ids2, _, _ = st.finish()
        assert rep2.samples == 0 and rep2.exactly_once == 1
    finally:
        ctx.close()


@pytest.mark.parametrize("B,n", [(1, 7), (3, 1), (5, 23)])
def test_odd_batch_sizes_exactly_once(lfgpu, oracle, B, n):
    """batch size 1, a single sample, and a ragged tail: every sample delivered once, in
    batches of B except the last, and the delivered tensors equal the oracle's."""
    rng = np.random.default_rng(B * 100 + n)
    ctx = lfgpu.Context(batch_size=B, n_workers=3, max_group=max(1, B), max_slot_buffers=8, seed=SEED)
    ch = ctx.chain(lfgpu.obj_det_ops())
    imgs = _images(ctx, [(int(rng.integers(200, 300)), int(rng.integers(200, 300))) for _ in range(4)], rng)
    descs = [lfgpu.sample_desc(900 + i, imgs[i % 4][0].shape, imgs[i % 4][1]) for i in range(n)]
    try:
        rep, ids, bsz, _ = ctx.run_shard(ch, descs, lfgpu.run_config(batch_size=B),
                                         capture=list(range(n)))
        assert rep.exactly_once == 1 and sorted(ids.tolist()) == [900 + i for i in range(n)]
        assert bsz.sum() == n and all(b == B for b in bsz[:-1]) and 1 <= bsz[-1] <= B
        ocfg = oracle.cfg2d()
        for pos, (raw, _) in ctx.last_capture.items():
            got = raw[: 3 * 224 * 224 * 4].view(np.float32).reshape(3, 224, 224)
            want = oracle.chain2d(ocfg, SEED, 900 + pos, imgs[pos % 4][0])[0]
            assert (np.abs(got - want) <= 1e-5 * np.abs(want) + 1e-5).all()
        assert len(ctx.last_capture) == n
    finally:
        for _, p in imgs:
            ctx.device_free(p)
        ctx.close()


@pytest.mark.parametrize("H,W", [(1, 1), (1, 700), (700, 1), (3, 5000), (2, 2)])
def test_rrc_size_limits_match_oracle(lfgpu, oracle, H, W):
    """RandomResizedCrop on degenerate images (one pixel, single rows / columns, extreme
    aspect ratios: the centre-crop fallback and the border taps), HBM and pinned."""
    ctx = lfgpu.Context(batch_size=4, n_workers=2, max_group=4, max_slot_buffers=4, seed=SEED)
    ch = ctx.chain(lfgpu.obj_det_ops())
    rng = np.random.default_rng(H * 7 + W)
    im = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    pd = ctx.device_alloc(im.nbytes)
    ctx.h2d(pd, im)
    ph = ctx.host_alloc(im.nbytes)
    import ctypes
    ctypes.memmove(ph, im.ctypes.data, im.nbytes)
    try:
        ocfg = oracle.cfg2d()
        for k, (p, kind) in enumerate([(pd, lfgpu.SRC_DEVICE), (ph, lfgpu.SRC_HOST_PINNED)]):
            sid = 4000 + k
            t = ctx.submit(ch, lfgpu.sample_desc(sid, (H, W, 3), p, src_kind=kind))
            ctx.flush()
            ctx.wait(t)
            got = ctx.ticket_output(t, 3 * 224 * 224 * 4).view(np.float32).reshape(3, 224, 224)
            want = oracle.chain2d(ocfg, SEED, sid, im)[0]
            assert (np.abs(got - want) <= 1e-5 * np.abs(want) + 1e-5).all(), (H, W, kind)
            ctx.release(t)
    finally:
        ctx.synchronize()
        ctx.device_free(pd)
        ctx.host_free(ph)
        ctx.close()


def test_img3d_thin_volumes_match_oracle(lfgpu, oracle):
    """Volumes thinner than the crop along one or two axes (zero padding on every side
    the source does not reach), W not a multiple of 16 (the row kernel), HBM source."""
    ctx = lfgpu.Context(batch_size=4, n_workers=2, max_group=4, max_slot_buffers=4, seed=SEED)
    crop = (16, 16, 32)
    ch = ctx.chain(lfgpu.img_seg_ops(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0))
    ocfg = oracle.cfg3d(crop=crop, p_flip=0.5, p_bright=1.0, p_noise=1.0)
    rng = np.random.default_rng(5)
    bufs = []
    try:
        for k, dims in enumerate([(1, 40, 40), (20, 1, 33), (3, 2, 1), (16, 16, 32)]):
            img = rng.standard_normal(dims).astype(np.float32)
            lbl = rng.integers(0, 3, dims, dtype=np.uint8)
            pi, pl = ctx.device_alloc(img.nbytes), ctx.device_alloc(lbl.nbytes)
            ctx.h2d(pi, img)
            ctx.h2d(pl, lbl)
            bufs += [pi, pl]
            sid = 6000 + k
            t = ctx.submit(ch, lfgpu.sample_desc(sid, dims, pi, pl))
            ctx.flush()
            ctx.wait(t)
            vox = int(np.prod(crop))
            raw = ctx.ticket_output(t, vox * 5)
            (e_img, e_lbl), _ = oracle.chain3d(ocfg, SEED, sid, img, lbl)
            assert np.array_equal(raw[vox * 4:].reshape(crop), e_lbl), dims
            g = raw[: vox * 4].view(np.float32).reshape(crop)
            assert (np.abs(g - e_img) <= 1e-5 * np.abs(e_img) + 1e-6).all(), dims
            ctx.release(t)
    finally:
        ctx.synchronize()
        for p in bufs:
            ctx.device_free(p)
        ctx.close()
