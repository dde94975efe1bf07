"""Evaluation metrics (reference pkg/src/qfca/metrics.py).

CPU: the oracle restatement against golden vectors produced by the reference
itself (tests/golden/make_metrics_golden.py).  GPU: the package's metrics.cu
path against the same goldens (bit-exact) and against the oracle on larger
random sets, connected components against scipy's labels.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import qfca_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SETS = ("f64", "f32_ties", "mixed")


def load_set(name):
    d = np.load(os.path.join(GOLDEN, f"metrics_{name}.npz"))
    n = int(d["n"])
    samples = [(d[f"scores_{i}"], d[f"mask_{i}"], bool(d["image_label"][i]), int(d["border"][i]))
               for i in range(n)]
    return d, samples


@pytest.mark.parametrize("name", SETS)
def test_oracle_metrics_match_reference_golden(name):
    d, s = load_set(name)
    sc, lb = O.metrics_pooled(s)
    assert O.rank_auroc(sc, lb) == pytest.approx(float(d["auroc_s"]), rel=0, abs=1e-15)
    assert O.f1_optimal(sc, lb) == float(d["f1"])
    assert O.auroc_image(s) == float(d["auroc_c"])
    fpr, pro = O.pro_curve(s, d["thresholds"])
    np.testing.assert_array_equal(fpr, d["fpr"])
    np.testing.assert_allclose(pro, d["pro_curve"], rtol=0, atol=1e-15)
    assert O.pro_at_fpr(s) == pytest.approx(float(d["pro"]), abs=1e-14)
    assert O.pro_at_fpr(s, 0.1) == pytest.approx(float(d["pro_limit_01"]), abs=1e-14)
    for i, (_, m, _, b) in enumerate(s):
        lab, _ = O.connected_components(m[b:-b, b:-b] if b else m)
        np.testing.assert_array_equal(lab, d[f"labels_cc_{i}"])


def _samples(M, s, torch_inputs=False):
    out = []
    for sc, m, lab, b in s:
        if torch_inputs:
            import torch
            sc, m = torch.from_numpy(sc).cuda(), torch.from_numpy(m).cuda()
        out.append(M.EvalSample(scores=sc, mask=m, image_label=lab, border=b))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", SETS)
@pytest.mark.parametrize("torch_inputs", [False, True])
def test_gpu_metrics_bit_exact_vs_reference_golden(name, torch_inputs):
    from paper_2510_15602_b200 import metrics as M
    d, s = load_set(name)
    ev = _samples(M, s, torch_inputs)
    assert M.auroc_pixel(ev) == float(d["auroc_s"])
    assert M.f1_optimal(ev) == float(d["f1"])
    assert M.auroc_image(ev) == float(d["auroc_c"])
    p = M._Pool(ev)
    np.testing.assert_array_equal(M._pro_thresholds(p), d["thresholds"])
    fpr, pro = M._pro_curve(p, d["thresholds"])
    np.testing.assert_array_equal(fpr, d["fpr"])
    np.testing.assert_array_equal(pro, d["pro_curve"])
    assert M.pro_at_fpr(ev) == float(d["pro"])
    assert M.pro_at_fpr(ev, 0.1) == float(d["pro_limit_01"])
    rep = M.MetricReport()
    row = rep.add_class("c", ev)
    assert row == {"n_images": len(ev), "pro": float(d["pro"]), "auroc_s": float(d["auroc_s"]),
                   "f1": float(d["f1"]), "auroc_c": float(d["auroc_c"])}
    assert rep.to_dict()["mean"]["n_images"] == len(ev)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,h,w,p", [(0, 1, 1, 0.5), (1, 1, 257, 0.5), (2, 300, 1, 0.6),
                                        (3, 64, 64, 0.45), (4, 517, 383, 0.55),
                                        (5, 1024, 1024, 0.5), (6, 50, 70, 0.0),
                                        (7, 50, 70, 1.0)])
def test_gpu_connected_components_match_scipy(seed, h, w, p):
    from paper_2510_15602_b200 import metrics as M
    rng = np.random.default_rng(seed)
    m = rng.random((h, w)) < p
    lab, n = M.connected_components(m)
    ref, rn = O.connected_components(m)
    assert n == rn
    np.testing.assert_array_equal(lab, ref)


def _random_set(rng, n_img, h, w, border, ties=None, dtype=np.float64):
    s = []
    for i in range(n_img):
        m = np.zeros((h, w), bool)
        if i % 3 != 2:
            for _ in range(rng.integers(1, 5)):
                y, x = rng.integers(0, h), rng.integers(0, w)
                m[max(0, y - 6):y + 6, max(0, x - 9):x + 4] = True
        sc = rng.standard_normal((h, w)) * 0.5 + m * rng.uniform(0.2, 1.0)
        if ties is not None:
            sc = np.round(sc, ties)
        s.append((sc.astype(dtype), m, bool(m.any()), border))
    return s


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n_img,h,w,border,ties,dtype", [
    (10, 8, 128, 96, 4, None, np.float64),
    (11, 5, 200, 200, 0, 1, np.float64),   # heavy ties
    (12, 6, 97, 131, 7, 2, np.float32),
    (13, 3, 256, 256, 2, 0, np.float64),   # very few distinct scores
])
@pytest.mark.parametrize("torch_inputs", [False, True])  # True: pointer-table pooling
def test_gpu_metrics_vs_oracle(seed, n_img, h, w, border, ties, dtype, torch_inputs):
    from paper_2510_15602_b200 import metrics as M
    rng = np.random.default_rng(seed)
    s = _random_set(rng, n_img, h, w, border, ties, dtype)
    ev = _samples(M, s, torch_inputs)
    sc, lb = O.metrics_pooled(s)
    assert M.auroc_pixel(ev) == pytest.approx(O.rank_auroc(sc, lb), abs=1e-15)
    assert M.f1_optimal(ev) == O.f1_optimal(sc, lb)
    assert M.auroc_image(ev) == O.auroc_image(s)
    assert M.pro_at_fpr(ev) == pytest.approx(O.pro_at_fpr(s), abs=1e-13)
    thr = np.array([3.0, 0.5, 0.5, -0.25, 1.0])  # caller thresholds, any order, repeats
    assert M.pro_at_fpr(ev, 0.3, thr) == pytest.approx(O.pro_at_fpr(s, 0.3, thr), abs=1e-13)


@pytest.mark.gpu
def test_gpu_metrics_undefined_and_errors():
    from paper_2510_15602_b200 import metrics as M
    z = np.zeros((8, 8))
    normal = [M.EvalSample(scores=np.arange(64.0).reshape(8, 8), mask=z > 1, image_label=False)]
    with pytest.raises(M.UndefinedMetricError):
        M.auroc_pixel(normal)
    with pytest.raises(M.UndefinedMetricError):
        M.f1_optimal(normal)
    with pytest.raises(M.UndefinedMetricError):
        M.pro_at_fpr(normal)
    with pytest.raises(M.UndefinedMetricError):
        M.auroc_image(normal)
    row = M.MetricReport().add_class("normal", normal)
    assert row == {"n_images": 1, "pro": None, "auroc_s": None, "f1": None, "auroc_c": None}
    with pytest.raises(ValueError):
        M.EvalSample(scores=z, mask=np.zeros((8, 7), bool), image_label=False)
    with pytest.raises(ValueError):
        M.EvalSample(scores=z, mask=z > 0, image_label=False, border=4)
    # all pixels anomalous: no normal pixels, FPR is zero everywhere
    allpos = [M.EvalSample(scores=np.arange(64.0).reshape(8, 8), mask=z == 0, image_label=True)]
    s = [(allpos[0].scores, allpos[0].mask, True, 0)]
    assert M.pro_at_fpr(allpos) == O.pro_at_fpr(s)


@pytest.mark.gpu
def test_gpu_pool_table_and_staged_paths_agree():
    """Device maps pooled in place (qfca_pool_interior_table) against the same
    maps staged (a non-contiguous view forces the staging copy)."""
    import torch
    from paper_2510_15602_b200 import metrics as M
    rng = np.random.default_rng(5)
    s = _random_set(rng, 4, 64, 80, 3, None, np.float32)
    ev_t = _samples(M, s, True)
    ev_s = [M.EvalSample(scores=torch.from_numpy(sc.T.copy()).cuda().t(),
                         mask=torch.from_numpy(m).cuda(), image_label=lab, border=b)
            for sc, m, lab, b in s]
    assert not ev_s[0].scores.is_contiguous()
    pt, ps = M._Pool(ev_t), M._Pool(ev_s)
    assert len(pt._tables) == 1 and len(ps._tables) == 0
    assert torch.equal(pt.scores, ps.scores) and torch.equal(pt.labels, ps.labels)
    assert torch.equal(pt.scores32, ps.scores32) and torch.equal(pt.image_max, ps.image_max)
