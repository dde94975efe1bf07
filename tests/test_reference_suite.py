"""The reference's own unit tests for the path (pkg/tests/test_quantize.py,
test_scoring.py, test_transport.py, test_pooling.py), with the same inputs and assertions, run against
this package's drop-in API on the GPU.  Left out: `_lower_median` (a private
NumPy helper), the PGM writer (out of scope) and the continuous-FCA
convergence test (its oracle lives in the reference's tests/oracles.py; the
quantized path is pinned to the reference's own outputs by the goldens).
The transport tests follow pkg/tests/test_transport.py:39-127 (their sorted-
multiset oracle restated in a few lines).  The naive counting oracle of
test_patch_histograms_match_counting_oracle is
the C oracle's patch histograms (pinned to reference goldens)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fmap(arr):
    return np.asarray(arr, dtype=np.float32)


def _fm(values, scale=1):
    from paper_2510_15602_b200 import FeatureMap
    return FeatureMap(values=np.asarray(values, np.float32), scale=scale)


def smooth_random_map(rng, c, h, w, sigma=3.0):
    z = rng.standard_normal((c, h, w))
    f = np.fft.rfft2(z)
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.rfftfreq(w)[None, :]
    g = np.exp(-2 * (np.pi * sigma) ** 2 * (fy ** 2 + fx ** 2))
    out = np.fft.irfft2(f * g, s=(h, w))
    return (out / np.abs(out).max(axis=(1, 2), keepdims=True)).astype(np.float32)


# ------------------------------------------------------------ test_quantize.py

def test_fit_quantizer_centers():
    from paper_2510_15602_b200 import fit_quantizer
    q = fit_quantizer(fmap(np.arange(5).reshape(1, 1, 5)), 4)
    np.testing.assert_allclose(q.centers(0), [0.5, 1.5, 2.5, 3.5])


def test_fit_quantizer_degenerate_flag():
    from paper_2510_15602_b200 import fit_quantizer
    assert fit_quantizer(fmap(np.full((1, 3, 3), 2.0)), 8).degenerate[0]


def test_bin_indices_floor_rule_hi_and_clamp():
    from paper_2510_15602_b200 import bin_indices, fit_quantizer
    v = fmap(np.array([[[0.0, 2.0, 4.0]]]))
    assert bin_indices(v, fit_quantizer(v, 4)).indices[0, 0][1] == 2
    v = fmap(np.array([[[0.0, 4.0]]]))
    q = fit_quantizer(v, 4)
    assert bin_indices(v, q).indices[0, 0, 1] == 3
    assert bin_indices(fmap(np.array([[[-1e-6, 4.0]]])), q).indices[0, 0, 0] == 0


def test_patch_histograms_uniform_map():
    from paper_2510_15602_b200 import BinIndexMap, patch_histograms
    idx = np.full((1, 5, 5), 3, np.int32)
    hf = patch_histograms(BinIndexMap(indices=idx, n_bins=8), 3)
    np.testing.assert_array_equal(hf.counts[0, 3], 9.0)
    assert hf.counts[0].sum() == 25 * 9


def test_patch_histograms_t1_one_hot():
    from paper_2510_15602_b200 import bin_indices, fit_quantizer, patch_histograms
    rng = np.random.default_rng(0)
    v = fmap(rng.random((2, 4, 4)))
    hf = patch_histograms(bin_indices(v, fit_quantizer(v, 5)), 1)
    assert hf.counts.max() == 1.0
    np.testing.assert_array_equal(hf.counts.sum(axis=1), 1.0)


def test_patch_histograms_single_outlier():
    from paper_2510_15602_b200 import BinIndexMap, patch_histograms
    idx = np.ones((1, 3, 3), dtype=np.int32)
    idx[0, 1, 1] = 0
    hf = patch_histograms(BinIndexMap(indices=idx, n_bins=4), 3)
    np.testing.assert_array_equal(hf.counts[0, :, 1, 1], [1, 8, 0, 0])


@pytest.mark.parametrize("t", [1, 3, 5])
def test_patch_histograms_match_counting_oracle(t):
    from paper_2510_15602_b200 import BinIndexMap, patch_histograms
    from oracle import qfca_oracle as O
    rng = np.random.default_rng(t)
    idx = rng.integers(0, 6, (2, 13, 17)).astype(np.int32)
    hf = patch_histograms(BinIndexMap(indices=idx, n_bins=6), t)
    expected = O.patch_histograms(idx, 6, t)
    np.testing.assert_array_equal(np.asarray(hf.counts), expected)


def test_mass_conservation():
    from paper_2510_15602_b200 import BinIndexMap, patch_histograms
    rng = np.random.default_rng(5)
    idx = rng.integers(0, 16, (3, 20, 20)).astype(np.int32)
    hf = patch_histograms(BinIndexMap(indices=idx, n_bins=16), 9)
    assert np.max(np.abs(hf.counts.sum(axis=1) - 81.0)) <= 1e-3


def test_reference_constant_map_all_modes_agree():
    from paper_2510_15602_b200 import REFERENCE_MODES, fit_quantizer, select_reference
    v = fmap(np.full((1, 8, 8), 1.5))
    q = fit_quantizer(v, 4)
    for m in REFERENCE_MODES:
        ref = select_reference(v, q, 3, mode=m)
        assert ref.weights[0].sum() == pytest.approx(9.0, abs=1e-6)
        np.testing.assert_array_equal(ref.weights[0] > 0, [True, False, False, False])


def test_reference_identical_patches_exact():
    from paper_2510_15602_b200 import fit_quantizer, select_reference
    col = np.array([0.0, 1.0, 2.0])
    v = fmap(np.tile(col, (9, 3))[None])
    ref = select_reference(v, fit_quantizer(v, 3), 3, mode="median-quan", pad="wrap")
    np.testing.assert_allclose(ref.weights[0], [3.0, 3.0, 3.0], atol=1e-6)


def test_reference_invariance_under_affine_rescale():
    from paper_2510_15602_b200 import fit_quantizer, select_reference
    rng = np.random.default_rng(6)
    v = fmap(rng.random((2, 16, 16)))
    r1 = select_reference(v, fit_quantizer(v, 8), 5)
    v2 = fmap(3.0 * v + 1.0)
    r2 = select_reference(v2, fit_quantizer(v2, 8), 5)
    np.testing.assert_allclose(r1.weights, r2.weights, atol=1e-6)


def test_reference_mass_all_modes():
    from paper_2510_15602_b200 import REFERENCE_MODES, fit_quantizer, select_reference
    rng = np.random.default_rng(7)
    v = fmap(rng.random((2, 12, 12)))
    q = fit_quantizer(v, 6)
    for m in REFERENCE_MODES:
        ref = select_reference(v, q, 5, mode=m)
        np.testing.assert_allclose(np.asarray(ref.weights).sum(axis=1), 25.0, atol=1e-6)


def test_unknown_mode_and_even_patch_rejected():
    from paper_2510_15602_b200 import (BinIndexMap, fit_quantizer, patch_histograms,
                                       select_reference)
    v = fmap(np.zeros((1, 4, 4)))
    with pytest.raises(ValueError):
        select_reference(v, fit_quantizer(v, 2), 3, mode="bogus")
    with pytest.raises(ValueError):
        patch_histograms(BinIndexMap(indices=np.zeros((1, 4, 4), np.int32), n_bins=2), 4)


# ------------------------------------------------------------ test_scoring.py

def test_uniform_features_zero_errors():
    from paper_2510_15602_b200 import (bin_error_maps, bin_indices, fit_quantizer,
                                       patch_histograms, select_reference)
    v = np.full((2, 12, 12), 3.0, np.float32)
    q = fit_quantizer(v, 8)
    hf = patch_histograms(bin_indices(v, q), 3)
    err = bin_error_maps(hf, select_reference(v, q, 3), q)
    np.testing.assert_array_equal(err, 0.0)


def test_error_maps_localized_to_covering_windows():
    from paper_2510_15602_b200 import (ReferenceHistogram, bin_error_maps, bin_indices,
                                       fit_quantizer, patch_histograms)
    v = np.zeros((1, 5, 5), np.float32)
    v[0, 2, 2] = 1.0
    q = fit_quantizer(v, 2)
    hf = patch_histograms(bin_indices(v, q), 3)
    ref = np.zeros((1, 2))
    ref[0, 0] = 9.0
    err = bin_error_maps(hf, ReferenceHistogram(weights=ref, patch_size=3), q)
    total = np.asarray(err)[0].sum(axis=0)
    covered = np.zeros((5, 5), bool)
    covered[1:4, 1:4] = True
    assert np.all(total[covered] > 0)
    assert np.all(total[~covered] == 0)


def test_error_maps_channel_independence():
    from paper_2510_15602_b200 import (bin_error_maps, bin_indices, fit_quantizer,
                                       patch_histograms, select_reference)
    rng = np.random.default_rng(0)
    v = rng.random((3, 8, 8)).astype(np.float32)

    def maps(vv):
        q = fit_quantizer(vv, 4)
        return np.asarray(bin_error_maps(patch_histograms(bin_indices(vv, q), 3),
                                         select_reference(vv, q, 3), q))
    perm = [2, 0, 1]
    np.testing.assert_allclose(maps(v[perm]), maps(v)[perm], atol=1e-12)


def test_associate_zero_errors():
    from paper_2510_15602_b200 import PipelineConfig, associate_errors, bin_indices, fit_quantizer
    z = np.zeros((1, 6, 6), np.float32)
    out = associate_errors(np.zeros((1, 4, 6, 6)), bin_indices(z, fit_quantizer(z, 4)),
                           PipelineConfig(patch_size=3))
    np.testing.assert_array_equal(out, 0.0)


def test_uniform_equals_large_sigma_gaussian():
    from paper_2510_15602_b200 import PipelineConfig, associate_errors, bin_indices, fit_quantizer
    rng = np.random.default_rng(1)
    v = rng.random((1, 10, 10)).astype(np.float32)
    bins = bin_indices(v, fit_quantizer(v, 4))
    err = rng.random((1, 4, 10, 10))
    a = associate_errors(err, bins, PipelineConfig(patch_size=5, sigma_p=math.inf))
    b = associate_errors(err, bins, PipelineConfig(patch_size=5, sigma_p=1e6))
    assert np.max(np.abs(np.asarray(a) - np.asarray(b))) <= 1e-5


def test_associate_delta_error():
    from paper_2510_15602_b200 import BinIndexMap, PipelineConfig, associate_errors
    idx = np.zeros((1, 7, 7), np.int32)
    idx[0, ::2, ::2] = 1
    err = np.zeros((1, 2, 7, 7))
    err[0, 1, 3, 3] = 1.0
    out = np.asarray(associate_errors(err, BinIndexMap(indices=idx, n_bins=2),
                                      PipelineConfig(patch_size=3)))[0]
    expected = np.zeros((7, 7))
    for y in range(2, 5):
        for x in range(2, 5):
            if idx[0, y, x] == 1:
                expected[y, x] = 1 / 9
    np.testing.assert_allclose(out, expected, atol=1e-12)


def test_aggregate_channels_and_degenerate():
    from paper_2510_15602_b200 import aggregate_channels
    scores = np.stack([np.full((4, 4), 2.0), np.full((4, 4), 4.0)])
    agg, degen = aggregate_channels(scores)
    assert not degen
    np.testing.assert_array_equal(agg, 3.0)
    only, _ = aggregate_channels(scores[:1])
    np.testing.assert_array_equal(only, 2.0)
    s2 = np.stack([np.full((2, 2), 2.0), np.full((2, 2), 99.0)])
    agg, _ = aggregate_channels(s2, skip=np.array([False, True]))
    np.testing.assert_array_equal(agg, 2.0)
    with pytest.warns(UserWarning):
        agg, degen = aggregate_channels(np.zeros((2, 3, 3)), skip=np.array([True, True]))
    assert degen
    np.testing.assert_array_equal(agg, 0.0)


def test_smooth_scores_identity_and_constant():
    from paper_2510_15602_b200 import smooth_scores
    rng = np.random.default_rng(2)
    m = rng.random((6, 6))
    np.testing.assert_array_equal(smooth_scores(m, 0.0), m)
    c = np.full((8, 8), 1.25)
    np.testing.assert_allclose(smooth_scores(c, 1.0), c, atol=1e-12)


def test_default_config_matches_published_defaults():
    from paper_2510_15602_b200 import PipelineConfig
    cfg = PipelineConfig()
    assert (cfg.n_bins, cfg.patch_size, cfg.sigma_s, cfg.reference_mode, cfg.border) == \
        (16, 9, 1.0, "median-quan", 4)
    assert math.isinf(cfg.sigma_p)


def test_detect_periodic_texture_near_zero():
    from paper_2510_15602_b200 import FeatureMap, PipelineConfig, detect
    col = np.array([0.0, 1 / 3, 2 / 3], np.float32)
    plane = np.tile(col, (30, 10))
    v = np.stack([plane, plane.T])
    cfg = PipelineConfig(n_bins=16, patch_size=3, pad="wrap", sample_budget=30 * 30)
    assert detect(FeatureMap(values=v, scale=1), cfg).image_score <= 1e-5


def test_detect_planted_square_scores_higher():
    from paper_2510_15602_b200 import PipelineConfig, detect
    rng = np.random.default_rng(3)
    v = smooth_random_map(rng, 4, 48, 48)
    v[:, 20:28, 20:28] += 1.5
    amap = detect(_fm(v), PipelineConfig(patch_size=5))
    s = np.asarray(amap.scores)
    inside = s[20:28, 20:28].mean()
    outside = np.delete(s.ravel(), [y * 48 + x for y in range(16, 32)
                                    for x in range(16, 32)]).mean()
    assert inside > 3 * outside


def test_single_bin_gives_zero_map():
    from paper_2510_15602_b200 import PipelineConfig, detect
    rng = np.random.default_rng(4)
    v = rng.random((2, 16, 16)).astype(np.float32)
    amap = detect(_fm(v), PipelineConfig(n_bins=1, patch_size=3))
    np.testing.assert_allclose(amap.scores, 0.0, atol=1e-12)


def test_common_affine_rescale_scales_scores():
    from paper_2510_15602_b200 import PipelineConfig, detect
    rng = np.random.default_rng(6)
    v = smooth_random_map(rng, 3, 24, 24)
    cfg = PipelineConfig(patch_size=5, sample_budget=24 * 24)
    a = np.asarray(detect(_fm(v), cfg).scores)
    b = np.asarray(detect(_fm(v * 2.0 + 1.0), cfg).scores)
    np.testing.assert_allclose(b, 2.0 * a, rtol=1e-12, atol=1e-14)


def test_toroidal_shift_equivariance():
    from paper_2510_15602_b200 import PipelineConfig, detect
    rng = np.random.default_rng(7)
    v = smooth_random_map(rng, 2, 24, 24)
    cfg = PipelineConfig(patch_size=5, pad="wrap", sample_budget=24 * 24)
    a = np.asarray(detect(_fm(v), cfg).scores)
    b = np.asarray(detect(_fm(np.roll(v, (7, 11), axis=(1, 2))), cfg).scores)
    np.testing.assert_allclose(np.roll(a, (7, 11), axis=(0, 1)), b, atol=1e-9)


def test_image_score_excludes_border():
    from paper_2510_15602_b200 import image_score_of
    scores = np.zeros((10, 10))
    scores[0, 0] = 5.0
    scores[5, 5] = 1.0
    assert image_score_of(scores, 2) == 1.0
    assert image_score_of(scores, 0) == 5.0


def test_upsample_scores_shape():
    from paper_2510_15602_b200 import upsample_scores
    rng = np.random.default_rng(8)
    s = rng.random((16, 16))
    up = np.asarray(upsample_scores(s, 64, 64))
    assert up.shape == (64, 64)
    np.testing.assert_allclose(up.reshape(16, 4, 16, 4).mean(axis=(1, 3)).mean(), s.mean(),
                               atol=1e-2)


# ------------------------------------------------------------ test_transport.py

def _random_equal_mass_instance(rng, max_bins=32, max_weight=8):
    n = int(rng.integers(1, max_bins + 1))
    p = rng.integers(0, max_weight + 1, n).astype(np.float64)
    r = rng.integers(0, max_weight + 1, n).astype(np.float64)
    diff = p.sum() - r.sum()
    if diff > 0:
        r[rng.integers(0, n)] += diff
    elif diff < 0:
        p[rng.integers(0, n)] += -diff
    if p.sum() == 0:
        p[0] += 1
        r[0] += 1
    q = np.cumsum(rng.random(n) + 1e-3)
    return p, r, q


def _oracle_bin_errors(p, r, q):
    """Per-bin duplicate-averaged rank errors of the expanded sorted multisets
    (the reference tests' sorted_mismatch_oracle + expand_histogram)."""
    xs = np.repeat(q, p.astype(int))
    ys = np.repeat(q, r.astype(int))
    errs = np.abs(xs - ys)
    out = np.zeros(p.size)
    pos = 0
    for i in range(p.size):
        c = int(p[i])
        if c:
            out[i] = errs[pos:pos + c].mean()
            pos += c
    return out


def _w1(p, r, q):
    return float(np.sum(np.abs(np.cumsum(p) - np.cumsum(r))[:-1] * np.diff(q)))


def test_transport_hand_examples_and_errors():
    from paper_2510_15602_b200 import MassError, quantized_mismatch
    np.testing.assert_array_equal(
        quantized_mismatch(np.array([3.0, 2.0, 1.0]), np.array([3.0, 2.0, 1.0]),
                           np.array([0.0, 1.0, 2.0])), 0.0)
    np.testing.assert_allclose(quantized_mismatch([2, 1], [1, 2], [0, 1]), [0.5, 0.0])
    np.testing.assert_allclose(quantized_mismatch([3, 0], [0, 3], [0, 2]), [2.0, 0.0])
    e = quantized_mismatch([0, 2, 0, 2], [1, 1, 1, 1], [0.0, 1.0, 2.0, 3.0])
    assert e[0] == 0.0 and e[2] == 0.0
    with pytest.raises(MassError):
        quantized_mismatch([1, 1], [1, 2], [0, 1])
    with pytest.raises(ValueError):
        quantized_mismatch([1, 1], [1, 1], [1, 1])


def test_transport_equivalence_iteration_bound_and_cost_identity():
    from paper_2510_15602_b200 import quantized_mismatch
    rng = np.random.default_rng(7)
    for _ in range(200):
        p, r, q = _random_equal_mass_instance(rng)
        e, iters = quantized_mismatch(p, r, q, return_iterations=True)
        assert iters <= 2 * p.size - 1
        np.testing.assert_allclose(e, _oracle_bin_errors(p, r, q), rtol=1e-9, atol=1e-12)
        assert float(np.sum(e * p)) == pytest.approx(_w1(p, r, q), rel=1e-9, abs=1e-12)


def test_transport_scale_equivariance_and_mass_invariance():
    from paper_2510_15602_b200 import quantized_mismatch
    p, r, q = _random_equal_mass_instance(np.random.default_rng(9))
    e1 = quantized_mismatch(p, r, q)
    np.testing.assert_allclose(quantized_mismatch(p, r, 3.5 * q), 3.5 * e1, rtol=1e-12)
    p, r, q = _random_equal_mass_instance(np.random.default_rng(10))
    np.testing.assert_allclose(quantized_mismatch(7.0 * p, 7.0 * r, q),
                               quantized_mismatch(p, r, q), rtol=1e-12)


def test_transport_batch_kernel_matches_scalar():
    from paper_2510_15602_b200 import mismatch_batch, quantized_mismatch
    rng = np.random.default_rng(11)
    n = 16
    q = np.cumsum(rng.random(n) + 0.01)
    r = rng.integers(0, 9, n).astype(np.float64)
    r[0] += 1
    rows = []
    for _ in range(50):
        p = rng.integers(0, 9, n).astype(np.float64)
        if p.sum() == 0:
            p[0] = 1.0
        rows.append(p)
    pb = np.ascontiguousarray(np.array(rows))
    out = np.empty_like(pb)
    mismatch_batch(pb, r, q, out)
    for p, e in zip(rows, out):
        np.testing.assert_allclose(e, quantized_mismatch(p, r * (p.sum() / r.sum()), q),
                                   rtol=1e-9, atol=1e-12)


# ------------------------------------------------------------ test_pooling.py
# (the hand values and error cases are in tests/test_pooling.py)

def test_box_average_k1_identity_and_naive_identities():
    from paper_2510_15602_b200 import box_average, naive_box_average
    p = np.random.default_rng(0).random((7, 5))
    for pad in ("zero", "reflect"):
        np.testing.assert_allclose(box_average(p, 1, pad), p)
    for k in (1, 3, 5):
        np.testing.assert_allclose(naive_box_average(np.array([[3.5]]), k, "reflect"), [[3.5]])
    np.testing.assert_array_equal(naive_box_average(np.zeros((4, 4)), 3, "reflect"),
                                  np.zeros((4, 4)))


@pytest.mark.parametrize("k", [3, 9, 31])
@pytest.mark.parametrize("pad", ["zero", "reflect"])
def test_box_average_matches_naive_256(k, pad):
    from paper_2510_15602_b200 import box_average, naive_box_average
    p = np.random.default_rng(k).random((256, 256)).astype(np.float32)
    assert np.max(np.abs(box_average(p, k, pad) - naive_box_average(p, k, pad))) <= 1e-4


def test_box_average_linearity():
    from paper_2510_15602_b200 import box_average
    rng = np.random.default_rng(1)
    x, y = rng.random((16, 16)), rng.random((16, 16))
    lhs = box_average(2.5 * x - 1.25 * y, 5, "reflect")
    rhs = 2.5 * box_average(x, 5, "reflect") - 1.25 * box_average(y, 5, "reflect")
    np.testing.assert_allclose(lhs, rhs, atol=1e-10)


@pytest.mark.parametrize("pad", ["zero", "reflect", "wrap"])
def test_box_average_stack_matches_single(pad):
    from paper_2510_15602_b200 import box_average, box_average_stack
    planes = np.random.default_rng(2).random((4, 12, 10)).astype(np.float32)
    stacked = box_average_stack(planes, 5, pad)
    for i in range(4):
        np.testing.assert_allclose(stacked[i], box_average(planes[i], 5, pad), atol=1e-12)


def test_wrap_padding_is_toroidal():
    from paper_2510_15602_b200 import box_average
    p = np.random.default_rng(3).random((8, 8))
    a = box_average(p, 3, "wrap")
    b = box_average(np.roll(p, (3, 2), axis=(0, 1)), 3, "wrap")
    np.testing.assert_allclose(np.roll(a, (3, 2), axis=(0, 1)), b, atol=1e-12)
