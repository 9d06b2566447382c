"""The multi-GPU request batcher (include/lbx/batcher.h): every request completes exactly once,
with the same pixels as a direct lbx_reconstruct of the same blob; batches respect max_batch;
timestamps are ordered (submit <= start <= end)."""
import numpy as np
import pytest

import weights_ref

pytestmark = pytest.mark.gpu


def test_batcher_matches_direct_decode(lbx):
    z = weights_ref.make_latents("sd3", 10, 64, 64, seed=31)
    blobs = [lbx.pack(z[i], 1) for i in range(10)]
    ref = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=10).reconstruct(blobs)
    b = lbx.Batcher([0], [("sd3", 64, 64)], max_batch=4, max_wait_us=2000)
    outs = [np.zeros((512, 512, 3), dtype=np.uint8) for _ in range(10)]
    for i in range(10):
        b.submit(100 + i, 0, blobs[i], outs[i])
    done = []
    for _ in range(400):
        done += b.poll(wait_us=50000)
        if len(done) == 10:
            break
    assert sorted(c["id"] for c in done) == list(range(100, 110))
    for c in done:
        assert c["status"] == 0 and 1 <= c["batch"] <= 4
        assert c["t_submit"] <= c["t_start"] <= c["t_end"]
    for i in range(10):
        assert np.array_equal(outs[i], ref[i]), i
    assert b.pending() == 0
    b.close()


@pytest.mark.parametrize("policy", ["greedy", "cost"])
def test_batcher_two_shape_classes(lbx, policy):
    """Two shape classes (SD1.5 4-channel and SD3 16-channel) through one worker; with the cost
    policy each class has its own measured service curve."""
    za = weights_ref.make_latents("sd15", 3, 64, 64, seed=32)
    zb = weights_ref.make_latents("sd3", 3, 64, 64, seed=33)
    b = lbx.Batcher([0], [("sd15", 64, 64), ("sd3", 64, 64)], max_batch=8, max_wait_us=1000, policy=policy)
    outs = {}
    for i in range(3):
        for s, z in ((0, za), (1, zb)):
            rid = s * 10 + i
            outs[rid] = np.zeros((512, 512, 3), dtype=np.uint8)
            b.submit(rid, s, lbx.pack(z[i], 1), outs[rid])
    done = []
    for _ in range(400):
        done += b.poll(wait_us=50000)
        if len(done) == 6:
            break
    assert len(done) == 6 and all(c["status"] == 0 for c in done)
    ra = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=3).reconstruct_latents(za)
    rb = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=3).reconstruct_latents(zb)
    for i in range(3):
        assert np.array_equal(outs[i], ra[i]) and np.array_equal(outs[10 + i], rb[i])
    b.close()


def test_batcher_cost_policy(lbx):
    """policy "cost": each worker measures its service curve at creation and closes the batch size
    lbx_batch_pick chooses; on B200 (time per image flat in the batch size) that is 1."""
    z = weights_ref.make_latents("sd3", 6, 64, 64, seed=34)
    blobs = [lbx.pack(z[i], 1) for i in range(6)]
    ref = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=6).reconstruct(blobs)
    b = lbx.Batcher([0], [("sd3", 64, 64)], max_batch=8, max_wait_us=0, policy="cost")
    outs = [np.zeros((512, 512, 3), dtype=np.uint8) for _ in range(6)]
    for i in range(6):
        b.submit(i, 0, blobs[i], outs[i])
    done = []
    for _ in range(400):
        done += b.poll(wait_us=50000)
        if len(done) == 6:
            break
    assert sorted(c["id"] for c in done) == list(range(6))
    assert all(c["status"] == 0 and 1 <= c["batch"] <= 8 for c in done)
    for i in range(6):
        assert np.array_equal(outs[i], ref[i]), i
    b.close()
