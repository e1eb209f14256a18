"""lfg_config.coalesce_us: per-sample submit + flush (the drop-in process_sample path)
shares launch groups; the coalesced launches produce the oracle's outputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 3


def test_coalesced_groups_match_oracle(lfgpu, oracle):
    ctx = lfgpu.Context(batch_size=16, n_workers=8, max_group=8, max_slot_buffers=8, seed=SEED,
                        coalesce_us=1_000_000)            # only full groups launch on flush
    rng = np.random.default_rng(9)
    ch = ctx.chain(lfgpu.obj_det_ops())
    ims, ptrs, ts = [], [], []
    try:
        c0 = ctx.counters()["launches"]
        for k in range(12):
            im = rng.integers(0, 256, (int(rng.integers(200, 400)), int(rng.integers(200, 400)), 3), dtype=np.uint8)
            p = ctx.device_alloc(im.nbytes)
            ctx.h2d(p, im)
            ims.append(im)
            ptrs.append(p)
            ts.append(ctx.submit(ch, lfgpu.sample_desc(40 + k, im.shape, p)))
            ctx.flush()                                    # per-sample flush: coalesced
        # the first 8 filled a group (launched when full); 4 remain open
        assert ctx.progress(ts[-1])[1] == 0
        launched = ctx.counters()["launches"] - c0
        assert launched == 1
        for k, t in enumerate(ts):
            ctx.wait(t)                                    # wait launches an open group at once
            got = ctx.ticket_output(t, 3 * 224 * 224 * 4).view(np.float32).reshape(3, 224, 224)
            want = oracle.chain2d(oracle.cfg2d(), SEED, 40 + k, ims[k])[0]
            assert (np.abs(got - want) <= 1e-5 * np.abs(want) + 1e-5).all()
            ctx.release(t)
        assert ctx.counters()["launches"] - c0 == 2
    finally:
        ctx.synchronize()
        for p in ptrs:
            ctx.device_free(p)
        ctx.close()
