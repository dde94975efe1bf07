"""Parity on the benched configurations themselves (BASELINE.json configs[1],
[2], [4]), on the bench's own inputs (workloads.make_features: WRN50-2
random-init block-2 features of synthetic textures):

* configs[1]  QFCA+ (k=10), 4 x 512 ch x 64^2 (512^2 textures);
* configs[2]  QFCA, 2 x 512 ch x 128^2 (1024^2 textures);
* configs[4]  QFCA on a full 1024 x 1024 feature plane (8192^2 texture),
              8 channels, through the tiled wide-plane path.

Bar: lo / hi / bins / median-quan reference weights bit-exact
against the CPU oracle; maps max-abs <= 1e-4 x max|ref|.  For QFCA+ the
oracle scores the GPU's own residual (protocol (3)); the raw end-to-end
deviation (GPU PCA vs the oracle's NumPy PCA) is printed and
bounded separately.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel_err(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def O():
    from oracle import qfca_oracle as o
    o.set_threads(os.cpu_count() or 1)
    return o


def _stages_bit_exact(Q, O, x_dev, cfg):
    """fit_quantizer / bin_indices / select_reference of every image on the GPU
    (device tensors in, device tensors out) against the oracle."""
    for i in range(x_dev.shape[0]):
        v = x_dev[i]
        q = Q.fit_quantizer(v, cfg.n_bins)
        b = Q.bin_indices(v, q)
        ref = Q.select_reference(v, q, cfg.patch_size, sample_budget=cfg.sample_budget)
        vh = v.cpu().numpy()
        lo, hi, dg = O.fit_quantizer(vh, cfg.n_bins)
        np.testing.assert_array_equal(q.lo.cpu().numpy(), lo)
        np.testing.assert_array_equal(q.hi.cpu().numpy(), hi)
        ob = O.bin_indices(vh, lo, hi, dg, cfg.n_bins)
        np.testing.assert_array_equal(b.indices.cpu().numpy(), ob)
        orf = O.select_reference(vh, lo, hi, dg, cfg.n_bins, cfg.patch_size, "median-quan",
                                 cfg.sample_budget, cfg.pad)
        np.testing.assert_array_equal(ref.weights.cpu().numpy(), orf)


def test_configs1_qfca_plus_512(O):
    import torch
    import paper_2510_15602_b200 as Q
    import workloads
    with torch.no_grad():
        feats, _ = workloads.make_features(4, 512, seed=11)
    cfg = Q.PipelineConfig(pca_components=10)
    res = Q.detect_batch(feats, cfg)
    mean, comps, _ = Q.features.pca_fit_batch(feats, 10)
    resid = Q.features.pca_residual_batch(feats, mean, comps)
    cfg0 = Q.PipelineConfig()
    _stages_bit_exact(Q, O, resid, cfg0)
    got = res.scores.cpu().numpy()
    rh = resid.cpu().numpy()
    for i in range(feats.shape[0]):
        ref, img, _ = O.detect(rh[i])
        assert rel_err(got[i], ref) <= TOL
        assert abs(float(res.image_scores[i]) - img) <= TOL * np.abs(ref).max()
        raw, _, _ = O.detect(feats[i].cpu().numpy(), pca_components=10)
        e = rel_err(got[i], raw)
        print(f"configs[1] image {i}: raw end-to-end QFCA+ deviation {e:.2e} (SURVEY H5)")
        assert e <= 5e-3


def test_configs2_qfca_1024(O):
    import torch
    import paper_2510_15602_b200 as Q
    import workloads
    with torch.no_grad():
        feats, _ = workloads.make_features(2, 1024, seed=12)
    assert tuple(feats.shape) == (2, 512, 128, 128)
    cfg = Q.PipelineConfig()
    res = Q.detect_batch(feats, cfg)
    _stages_bit_exact(Q, O, feats, cfg)
    got = res.scores.cpu().numpy()
    for i in range(2):
        ref, img, _ = O.detect(feats[i].cpu().numpy())
        e = rel_err(got[i], ref)
        print(f"configs[2] image {i}: {e:.2e}")
        assert e <= TOL
        assert abs(float(res.image_scores[i]) - img) <= TOL * np.abs(ref).max()
    up = Q.upsample_batch(res.scores, 1024, 1024)
    ref_up = O.upsample_scores(O.detect(feats[0].cpu().numpy())[0], 1024, 1024)
    assert rel_err(up[0].cpu().numpy(), ref_up) <= TOL


def test_configs4_full_1024_plane_tiles(O):
    """8 channels of the 8192^2 texture's 512 x 1024^2 features: the tiled wide
    path (128 x 256 tiles, whole-plane K3 reference) vs the oracle's whole
    plane."""
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import sharding
    import workloads
    with torch.no_grad():
        imgs, _ = workloads.textures(1, 8192, seed=13)
        feats = workloads.features(imgs, chunk=1)
    sel = [0, 37, 101, 202, 255, 300, 411, 510]
    x = feats[0, sel].contiguous()
    del feats, imgs
    assert tuple(x.shape) == (8, 1024, 1024)
    cfg = Q.PipelineConfig()
    assert sharding.wide_supported(cfg, 1024, 1024, 8)
    res = Q.detect_batch(x[None], cfg)
    xh = x.cpu().numpy()
    ref, img, _ = O.detect(xh)
    e = rel_err(res.scores[0].cpu().numpy(), ref)
    print(f"configs[4] 8-channel 1024^2 plane: {e:.2e}")
    assert e <= TOL
    assert abs(float(res.image_scores[0]) - img) <= TOL * np.abs(ref).max()
    # channel-sharded form (one rank holding all 8 channels) gives the same map
    m, s, dg = sharding.detect_channel_sharded(x, cfg)
    assert rel_err(m.cpu().numpy(), ref) <= TOL
