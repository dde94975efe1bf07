"""Multi-process (gloo, world size 2, CPU) checks of the sharding logic, and a
GPU check of the channel-sharded partials.  The per-rank partial on CPU comes
from the oracle (test-side stand-in for the GPU kernels); the product code
under test is the channel partition and the single all-reduce."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_covers_exactly():
    from paper_2510_15602_b200.sharding import shard_range
    for n in (1, 7, 64, 512, 513):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, x, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle import qfca_oracle as O
    from paper_2510_15602_b200.sharding import combine_partials, shard_range
    s, e = shard_range(x.shape[0], world, rank)
    _, _, _, st = O.detect(x[s:e], return_stages=True)
    acc = torch.from_numpy(st["agg"] * max(st["used"], 1) if st["used"] else st["agg"])
    total, used = combine_partials(acc, st["used"])
    if rank == 0:
        out.put((total.numpy(), used))
    dist.destroy_process_group()


def test_channel_sharded_combine_gloo():
    from oracle import qfca_oracle as O
    rng = np.random.default_rng(3)
    x = np.maximum(rng.standard_normal((10, 20, 24)), 0).astype(np.float32)
    x[4] = 0.0  # a degenerate channel on rank 0's slice
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, used = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, _, _, st = O.detect(x, return_stages=True)
    assert used == st["used"] == 9
    agg = total / used
    np.testing.assert_allclose(agg, st["agg"], rtol=1e-12, atol=1e-14)
    final = O.smooth_scores(agg, 1.0)
    ref, _, _ = O.detect(x)
    np.testing.assert_allclose(final, ref, rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_channel_partials_gpu():
    """Two channel slices scored separately and summed reproduce detect."""
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200.sharding import channel_partial, detect_channel_sharded
    from oracle import qfca_oracle as O
    rng = np.random.default_rng(5)
    x = np.maximum(rng.standard_normal((40, 64, 64)) + 0.1, 0).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    cfg = Q.PipelineConfig()
    a0, u0 = channel_partial(xt[:17], cfg)
    a1, u1 = channel_partial(xt[17:], cfg)
    _, _, _, st = O.detect(x, return_stages=True)
    assert u0 + u1 == st["used"]
    agg = ((a0 + a1) / (u0 + u1)).cpu().numpy()
    assert np.abs(agg - st["agg"]).max() <= 1e-4 * np.abs(st["agg"]).max()
    final, img, degen = detect_channel_sharded(xt, cfg)  # world size 1
    ref, img_ref, _ = O.detect(x)
    assert np.abs(final.cpu().numpy() - ref).max() <= 1e-4 * np.abs(ref).max()
    assert not degen


def test_strip_geometry():
    """sharding.strips: every column owned by exactly one segment, owned outputs
    at least 2R columns from a segment's inner edges (so the segment's own border
    padding never reaches them), true borders at segment borders."""
    from paper_2510_15602_b200.sharding import strips
    for w in (129, 200, 257, 300, 1000, 1024, 4096):
        for t in (1, 3, 5, 9, 15):
            for sw in (128, 256):
                if w <= sw:
                    st, own, loc = strips(w, t, sw)
                    assert st == [0] and (own == 0).all() and (loc == np.arange(w)).all()
                    continue
                st, own, loc = strips(w, t, sw)
                halo = 2 * (t // 2)
                assert st[0] == 0 and st[-1] + sw == w
                assert (np.diff(own) >= 0).all()
                for x in range(w):
                    a = st[own[x]]
                    assert 0 <= x - a < sw and loc[x] == x - a
                    if own[x] > 0:
                        assert x - a >= halo              # far from the left inner edge
                    if own[x] < len(st) - 1:
                        assert a + sw - 1 - x >= halo     # far from the right inner edge


def _pca_worker(rank, world, port, x, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_2510_15602_b200.sharding import _all_reduce, _world, local_pixels
    w, r = _world()
    xs = local_pixels(torch.from_numpy(x), w, r).double()  # (C, n_local)
    s = _all_reduce(xs.sum(1))
    mean = s / float(x[0].size)
    xc = xs - mean[:, None]
    g = _all_reduce(xc @ xc.T)
    if rank == 0:
        out.put((mean.numpy(), (g / float(x[0].size)).numpy()))
    dist.destroy_process_group()


def test_pixel_sharded_pca_reductions_gloo():
    """QFCA+ on one huge image: the pixel partition and the two all-reduces
    (channel sums, centred Gram) reproduce pca_fit's mean and covariance
    (features.py:169-172).  The per-rank partial is plain torch fp64 here."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((6, 13, 11)).astype(np.float32)  # 143 pixels: ragged split
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pca_worker, args=(r, 2, port, x, q)) for r in range(2)]
    for p in procs:
        p.start()
    mean, cov = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v = x.reshape(6, -1).T.astype(np.float64)
    np.testing.assert_allclose(mean, v.mean(0), rtol=1e-13, atol=1e-15)
    xc = v - v.mean(0)
    np.testing.assert_allclose(cov, xc.T @ xc / v.shape[0], rtol=1e-12, atol=1e-14)


@pytest.mark.gpu
def test_pca_sharded_gpu():
    """Pixel-sharded pca_fit partials (two simulated ranks summed) equal the
    whole-plane ones; detect_pca_sharded (world size 1) matches the oracle's
    QFCA+ detect.  150 x 140 = 21000 pixels: one exact 16384-pixel block plus
    a ragged tail per covariance."""
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200.sharding import (centred_gram, channel_sums, detect_pca_sharded,
                                                local_pixels, pca_fit_sharded)
    from oracle import qfca_oracle as O
    rng = np.random.default_rng(6)
    c = 256  # the block-Lanczos eigensolver's range; a decaying spectrum (5 strong directions)
    u = np.linalg.qr(rng.standard_normal((c, 5)))[0]
    z = rng.standard_normal((5, 150 * 140)) * np.array([6.0, 5.0, 4.0, 3.0, 2.5])[:, None]
    x = (u @ z + 0.5 * rng.standard_normal((c, 150 * 140))).reshape(c, 150, 140)
    x = np.maximum(x + 0.5, 0).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    hw = 150 * 140
    full = local_pixels(xt, 1, 0)
    mean = channel_sums(full) / hw
    halves = [local_pixels(xt, 2, r) for r in range(2)]
    mean2 = (channel_sums(halves[0]) + channel_sums(halves[1])) / hw
    torch.testing.assert_close(mean2, mean, rtol=1e-12, atol=1e-14)
    g = centred_gram(full, mean)
    g2 = centred_gram(halves[0], mean) + centred_gram(halves[1], mean)
    v = x.reshape(c, -1).astype(np.float64)
    vc = v - v.mean(1, keepdims=True)
    ref_cov = vc @ vc.T / hw
    scale = np.abs(ref_cov).max()
    assert np.abs(g.cpu().numpy() / hw - ref_cov).max() <= 1e-9 * scale
    assert np.abs(g2.cpu().numpy() / hw - ref_cov).max() <= 1e-9 * scale
    m, comps, ev = pca_fit_sharded(xt, 5)
    om, oc, oev = O.pca_fit(x, 5)
    np.testing.assert_allclose(ev.cpu().numpy(), oev, rtol=1e-8)
    proj = comps.T.cpu().numpy() @ comps.cpu().numpy()
    assert np.abs(proj - oc.T @ oc).max() <= 1e-7
    cfg = Q.PipelineConfig(pca_components=5)
    final, img, degen = detect_pca_sharded(xt, cfg)
    ref, img_ref, _ = O.detect(x, pca_components=5)
    assert np.abs(final.cpu().numpy() - ref).max() <= 1e-4 * np.abs(ref).max()
    assert abs(float(img) - img_ref) <= 1e-4 * np.abs(ref).max()
    assert not bool(degen)


@pytest.mark.gpu
def test_pca_residual_slice_matches_full():
    """A rank's channel-sliced residual (qfca_pca_residual_slice) is the same
    float32 values as the full residual's slice, for slices on and off the
    8-channel tiles."""
    import torch
    from paper_2510_15602_b200 import features as F
    rng = np.random.default_rng(5)
    x = torch.from_numpy(np.maximum(rng.standard_normal((2, 64, 24, 20)), 0).astype(np.float32)).cuda()
    mean, comps, _ = F.pca_fit_batch(x, 10)
    full = F.pca_residual_batch(x, mean, comps)
    for c0, c1 in ((0, 64), (0, 8), (8, 24), (5, 13), (21, 64), (63, 64)):
        part = F.pca_residual_slice(x, mean, comps, c0, c1)
        assert torch.equal(part, full[:, c0:c1]), (c0, c1)
