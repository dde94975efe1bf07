"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from conftest import cfg_of, golden_names, load_golden
from oracle import qfca_oracle as O

CASES = [n for n in golden_names() if n not in ("transport_random", "wrn256_qfca_plus")]


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(name):
    d = load_golden(name)
    cfg = cfg_of(d)
    n = cfg.get("n_bins", 16)
    t = cfg.get("patch_size", 9)
    pad = cfg.get("pad", "reflect")
    v = d["values"]
    lo, hi, dg = O.fit_quantizer(v, n)
    np.testing.assert_array_equal(lo, d["lo"])
    np.testing.assert_array_equal(hi, d["hi"])
    np.testing.assert_array_equal(dg, d["degenerate"])
    bins = O.bin_indices(v, lo, hi, dg, n)
    np.testing.assert_array_equal(bins, d["bins"])
    refw = O.select_reference(v, lo, hi, dg, n, t, cfg.get("reference_mode", "median-quan"),
                              cfg.get("sample_budget", 4096), pad)
    if cfg.get("reference_mode", "median-quan") == "median-quan":
        np.testing.assert_array_equal(refw, d["ref_weights"])
    else:
        np.testing.assert_allclose(refw, d["ref_weights"], rtol=1e-12, atol=1e-12)
    if "counts" in d:
        np.testing.assert_array_equal(O.patch_histograms(bins, n, t, pad), d["counts"])
    kw = dict(cfg)
    scores, score, degen = O.detect(v, **kw)
    np.testing.assert_allclose(scores, d["scores"], rtol=1e-12, atol=1e-13)
    assert math.isclose(score, float(d["image_score"]), rel_tol=1e-12, abs_tol=1e-13)
    assert bool(degen) == bool(d["detect_degenerate"])


def test_oracle_upsample_matches_reference():
    d = load_golden("wrn256_qfca")
    up = O.upsample_scores(d["scores"], 256, 256)
    np.testing.assert_array_equal(up.astype(np.float32), d["upsampled"])


def test_oracle_pca_matches_reference():
    d = load_golden("wrn256_qfca")
    p = load_golden("wrn256_qfca_plus")
    mean, comps, ev = O.pca_fit(d["values"], 10)
    np.testing.assert_allclose(mean, p["pca_mean"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ev, p["pca_eigenvalues"], rtol=1e-9)
    # projector (sign-free) comparison
    a = comps.T @ comps
    b = p["pca_components"].T @ p["pca_components"]
    assert np.abs(a - b).max() < 1e-8
    res = O.pca_residual(d["values"], p["pca_mean"], p["pca_components"])
    np.testing.assert_allclose(res, p["residual"], rtol=0, atol=1e-6)
    scores, score, _ = O.detect(p["residual"])
    rel = np.abs(scores - p["scores"]).max() / np.abs(p["scores"]).max()
    assert rel < 1e-12


def test_oracle_transport_matches_reference():
    d = load_golden("transport_random")
    for p, r, q, e in zip(d["P"], d["R"], d["Q"], d["E"]):
        got = O.quantized_mismatch(p, r, q)
        np.testing.assert_allclose(got, e, rtol=1e-9, atol=1e-12)


def test_transport_kats():
    # test_transport.py:45-55 hand examples
    np.testing.assert_allclose(O.quantized_mismatch([2, 1], [1, 2], [0, 1]), [0.5, 0.0])
    np.testing.assert_allclose(O.quantized_mismatch([3, 0], [0, 3], [0, 2]), [2.0, 0.0])
