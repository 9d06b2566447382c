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


def _drain(b, n, tries=600):
    done = []
    for _ in range(tries):
        done += b.poll(wait_us=50000)
        if len(done) >= n:
            break
    return done


def test_batcher_two_workers_one_gpu(lbx):
    """Two workers (devices=[0, 0]: two decoders, two pipelines on one GPU) share the queue: every
    request completes exactly once, pixels equal a direct decode, and both workers take work."""
    n = 24
    z = weights_ref.make_latents("sd3", n, 64, 64, seed=41)
    blobs = [lbx.pack(z[i], 1) for i in range(n)]
    ref = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=n).reconstruct(blobs)
    b = lbx.Batcher([0, 0], [("sd3", 64, 64)], max_batch=2, max_wait_us=0, policy="greedy")
    outs = [np.zeros((512, 512, 3), dtype=np.uint8) for _ in range(n)]
    for i in range(n):
        b.submit(1000 + i, 0, blobs[i], outs[i])
    done = _drain(b, n)
    assert sorted(c["id"] for c in done) == list(range(1000, 1000 + n))  # each exactly once
    assert all(c["status"] == 0 and c["device"] == 0 and 1 <= c["batch"] <= 2 for c in done)
    assert {c["worker"] for c in done} == {0, 1}, "both workers must take work"
    for i in range(n):
        assert np.array_equal(outs[i], ref[i]), i
    assert b.pending() == 0
    b.close()


def test_batcher_rejects_duplicate_inflight_id_and_bad_out(lbx):
    z = weights_ref.make_latents("sd3", 1, 64, 64, seed=42)
    blob = lbx.pack(z[0], 1)
    b = lbx.Batcher([0], [("sd3", 64, 64)], max_batch=2, max_wait_us=200000)
    out = np.zeros((512, 512, 3), dtype=np.uint8)
    b.submit(7, 0, blob, out)
    with pytest.raises(lbx.LbxError) as e:
        b.submit(7, 0, blob, np.zeros((512, 512, 3), dtype=np.uint8))
    assert e.value.status == lbx.E_CONFIG
    with pytest.raises(lbx.LbxError) as e:
        b.submit(8, 0, blob, np.zeros((512, 512, 2), dtype=np.uint8))  # too small
    assert e.value.status == lbx.E_CONFIG
    with pytest.raises(lbx.LbxError):
        b.submit(9, 0, blob, np.zeros((512, 512, 3, 2), dtype=np.uint8)[..., 0])  # strided
    done = _drain(b, 1)
    assert [c["id"] for c in done] == [7] and done[0]["status"] == 0
    assert np.array_equal(out, lbx.Decoder("sd3", (64, 64), seed=0).reconstruct([blob])[0])
    b.submit(7, 0, blob, out)  # the id is free again once its completion was polled
    assert [c["id"] for c in _drain(b, 1)] == [7]
    b.close()


def test_async_pipeline_submit_wait(lbx):
    """lbx_reconstruct_submit / _wait: batches of different sizes in flight two at a time decode
    exactly like lbx_reconstruct; a third submit before a wait is refused; a malformed blob surfaces
    as LBX_E_FORMAT at its wait and the decoder keeps working."""
    z = weights_ref.make_latents("sd15", 7, 64, 64, seed=43)
    blobs = [lbx.pack(z[i], 1) for i in range(7)]
    dec = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=3)
    ref = np.concatenate([dec.reconstruct(blobs[i:i + 3]) for i in range(0, 7, 3)])
    outs = [np.zeros((512, 512, 3), dtype=np.uint8) for _ in range(7)]
    t1 = dec.submit(blobs[0:3], outs[0:3])
    t2 = dec.submit(blobs[3:5], outs[3:5])
    with pytest.raises(lbx.LbxError) as e:
        dec.submit(blobs[5:7], outs[5:7])
    assert e.value.status == lbx.E_RUNTIME
    dec.wait(t1)
    t3 = dec.submit(blobs[5:7], outs[5:7])
    dec.wait(t2)
    dec.wait(t3)
    for i in range(7):
        assert np.array_equal(outs[i], ref[i]), i
    # a payload corruption that passes the host header check is caught by the device unpack
    bad = bytearray(blobs[0])
    bad[-1] ^= 0xFF
    bad[len(bad) // 2] ^= 0xFF
    o = [np.zeros((512, 512, 3), dtype=np.uint8)]
    try:
        t = dec.submit([bytes(bad)], o)
        try:
            dec.wait(t)
        except lbx.LbxError as err:
            assert err.status == lbx.E_FORMAT
    except lbx.LbxError as err:  # rejected by the host-side validation instead
        assert err.status == lbx.E_FORMAT
    t = dec.submit(blobs[:1], o)
    dec.wait(t)
    assert np.array_equal(o[0], ref[0])


def test_graph_cache_keyed_by_batch_size_only(lbx):
    """lbx_decode on 100 distinct caller buffer pairs reuses the one graph per batch size: no new
    captures (the cache used to be keyed by the caller's pointers)."""
    import torch
    z = weights_ref.make_latents("sd15", 2, 64, 64, seed=44)
    dec = lbx.Decoder("sd15", (64, 64), seed=0, max_batch=2)
    dec.prepare(2)
    base = dec.graph_captures()
    assert base == 2
    ref = dec.reconstruct_latents(z)
    lat_bytes, rgb_bytes = z.nbytes, ref.nbytes
    lat_big = torch.zeros(lat_bytes + 100 * 256, dtype=torch.uint8, device="cuda")
    rgb_big = torch.zeros(rgb_bytes + 100 * 256, dtype=torch.uint8, device="cuda")
    zb = torch.from_numpy(z.view(np.uint8).reshape(-1).copy())
    for k in range(100):  # 100 distinct (latents, rgb) pointer pairs, 256 B apart
        lat_big[256 * k:256 * k + lat_bytes].copy_(zb)
        torch.cuda.synchronize()  # the decoder's own stream does not order with torch's default stream
        dec.decode_ptr(lat_big.data_ptr() + 256 * k, 2, rgb_big.data_ptr() + 256 * k)
    torch.cuda.synchronize()
    assert dec.graph_captures() == base
    got = rgb_big[256 * 99:256 * 99 + rgb_bytes].cpu().numpy().reshape(ref.shape)
    assert np.array_equal(got, ref)


def _device_blobs(lbx, blobs, device):
    """LBLP blobs copied into one GPU buffer (an HBM latent tier): [(ptr, nbytes)], the tensor."""
    import torch
    offs, total = [], 0
    for b in blobs:
        offs.append(total)
        total += (len(b) + 255) // 256 * 256
    buf = torch.zeros(total, dtype=torch.uint8)
    for o, b in zip(offs, blobs):
        buf[o:o + len(b)] = torch.frombuffer(bytearray(b), dtype=torch.uint8)
    dbuf = buf.to(f"cuda:{device}")
    torch.cuda.synchronize()
    return [(dbuf.data_ptr() + o, len(b)) for o, b in zip(offs, blobs)], dbuf


def test_batcher_device_resident_blobs(lbx):
    """Blobs resident in HBM (lbx_batcher_submit_device), mixed with host blobs in the same queue:
    pixels equal a direct decode; no spill on one GPU (every worker is local to the blobs)."""
    n = 10
    z = weights_ref.make_latents("sd3", n, 64, 64, seed=45)
    blobs = [lbx.pack(z[i], 1) for i in range(n)]
    ref = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=n).reconstruct(blobs)
    dev_blobs, keep = _device_blobs(lbx, blobs, 0)
    b = lbx.Batcher([0, 0], [("sd3", 64, 64)], max_batch=3, max_wait_us=0)
    outs = [np.zeros((512, 512, 3), dtype=np.uint8) for _ in range(n)]
    for i in range(n):
        if i % 3 == 0:
            b.submit(i, 0, blobs[i], outs[i])
        else:
            b.submit_device(i, 0, dev_blobs[i][0], dev_blobs[i][1], 0, outs[i], keep=keep)
    done = _drain(b, n)
    assert sorted(c["id"] for c in done) == list(range(n)) and all(c["status"] == 0 for c in done)
    for i in range(n):
        assert np.array_equal(outs[i], ref[i]), i
    st = b.stats()
    assert st["spills"] == 0 and st["peer_copies"] == 0
    b.close()


def test_batcher_nvlink_spill_two_gpus(lbx):
    """Blobs resident on GPU 1 decoded by workers on GPUs 0 and 1: the GPU-0 worker fetches its
    blobs over NVLink (peer copy); pixels equal a direct decode.  Needs two GPUs."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    n = 16
    z = weights_ref.make_latents("sd3", n, 64, 64, seed=46)
    blobs = [lbx.pack(z[i], 1) for i in range(n)]
    ref = lbx.Decoder("sd3", (64, 64), seed=0, max_batch=n).reconstruct(blobs)
    dev_blobs, keep = _device_blobs(lbx, blobs, 1)
    b = lbx.Batcher([0, 1], [("sd3", 64, 64)], max_batch=1, max_wait_us=0)
    outs = [np.zeros((512, 512, 3), dtype=np.uint8) for _ in range(n)]
    for i in range(n):
        b.submit_device(i, 0, dev_blobs[i][0], dev_blobs[i][1], 1, outs[i], keep=keep)
    done = _drain(b, n)
    assert sorted(c["id"] for c in done) == list(range(n)) and all(c["status"] == 0 for c in done)
    for i in range(n):
        assert np.array_equal(outs[i], ref[i]), i
    st = b.stats()
    spilled = sum(1 for c in done if c["device"] == 0)
    assert st["spills"] == spilled == st["peer_copies"]
    b.close()


def test_reference_binding_with_measured_decode(lbx):
    """tools/ref_binding (reference simulator sources + liblbx.so): the decode the reference models
    as 40 ms is measured through lbx_reconstruct on this GPU and fed to the reference's lbx::run."""
    import json
    import os
    import subprocess
    p = os.path.join(os.path.dirname(lbx.LIB_PATH), "..", "oracle", "_ref", "ref_binding")
    if not os.path.exists(p):
        pytest.skip("oracle/_ref/ref_binding not built")
    out = subprocess.run([p, "--requests-per-day", "50000", "--days", "4"], capture_output=True, text=True,
                         timeout=600, check=True).stdout
    print(out)
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert lines[0]["decode_measured"] is True
    assert 2.0 < lines[2]["decode_ms"] < 40.0
