"""PRO / pixel AUROC / F1 / image AUROC parity on planted-defect textures
(north star: "identical PRO/AUROC on synthetic textures with
planted defects"; reference metrics.py:149-206, acceptance A6
pkg/tests/test_acceptance.py:176-192).

1. Against the reference itself: tests/golden/planted_filterbank.npz holds the
   reference's own end-to-end run (synth textures -> its filter-bank features
   -> detect -> upsample_scores -> metrics, 3 kinds x 10 images of 128^2;
   tests/golden/make_planted_golden.py).  The GPU path scores the same
   features (detect_batch, upsample_batch) and the GPU metrics (metrics.cu)
   must give the same four numbers to 4 decimals (|diff| <= 5e-5) and maps
   within 1e-4 of max|ref|.
2. On the reference's default backbone: WRN50-2 random-init block-2 features
   (512 ch) of 10 planted textures per kind at 256^2, computed on the GPU; the
   GPU path vs the CPU oracle (pinned to the reference by
   tests/test_oracle_golden.py) on those identical features, the GPU metrics
   vs the oracle's metrics restatement (pinned by tests/test_metrics.py).
"""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                    "planted_filterbank.npz")
KEYS = ("pro", "auroc_s", "f1", "auroc_c")


def test_planted_golden_present():
    d = np.load(GOLD)
    for kind in ("noise", "tiles", "stripes"):
        assert d[f"{kind}/features"].shape == (10, 39, 32, 32)
        assert d[f"{kind}/labels"].sum() == 7
        assert 0.5 < float(d[f"{kind}/auroc_s"]) <= 1.0


def _gpu_rows(Q, feats, masks, labels, border, size, cfg):
    import torch
    res = Q.detect_batch(torch.from_numpy(feats).cuda(), cfg)
    up = Q.upsample_batch(res.scores, size, size)
    mk = torch.from_numpy(np.ascontiguousarray(masks)).cuda()
    samples = [Q.metrics.EvalSample(scores=up[i], mask=mk[i], image_label=bool(labels[i]),
                                    border=border) for i in range(len(labels))]
    row = Q.metrics.MetricReport().add_class("c", samples)
    return res, up, row


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["noise", "tiles", "stripes"])
def test_planted_metrics_equal_reference(kind):
    import paper_2510_15602_b200 as Q
    d = np.load(GOLD)
    size = int(d["size"])
    feats = d[f"{kind}/features"]
    res, up, row = _gpu_rows(Q, feats, d[f"{kind}/masks"], d[f"{kind}/labels"],
                             int(d[f"{kind}/border"]), size, Q.PipelineConfig())
    ref_maps = d[f"{kind}/maps"]
    got = res.scores.cpu().numpy()
    assert np.abs(got - ref_maps).max() <= 1e-4 * np.abs(ref_maps).max()
    ref_up = d[f"{kind}/upsampled"].astype(np.float64)
    assert np.abs(up.cpu().numpy() - ref_up).max() <= 1e-4 * np.abs(ref_up).max()
    for k in KEYS:
        assert abs(row[k] - float(d[f"{kind}/{k}"])) <= 5e-5, (k, row[k], float(d[f"{kind}/{k}"]))


@pytest.fixture(scope="module")
def wrn_planted():
    import torch
    import workloads
    out = {}
    with torch.no_grad():
        for j, kind in enumerate(("noise", "tiles", "stripes")):
            imgs, masks = workloads.textures(10, 256, seed=77 + j, device="cuda", kinds=(kind,),
                                             n_good=3)
            out[kind] = (workloads.features(imgs), masks)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["noise", "tiles", "stripes"])
@pytest.mark.parametrize("pca", [0, 10])
def test_planted_wrn_metrics_equal_oracle(wrn_planted, kind, pca):
    import paper_2510_15602_b200 as Q
    from oracle import qfca_oracle as O
    feats, masks = wrn_planted[kind]
    cfg = Q.PipelineConfig(pca_components=pca)
    size = 256
    border = cfg.border * 8
    labels = np.array([i >= 3 for i in range(10)])
    x = feats
    if pca:
        # the oracle scores the GPU's own residual; the PCA stage
        # itself is checked against the reference in test_gpu_parity.py
        mean, comps, _ = Q.features.pca_fit_batch(feats, pca)
        x = Q.features.pca_residual_batch(feats, mean, comps)
        cfg0 = Q.PipelineConfig()
    else:
        cfg0 = cfg
    res, up, row = _gpu_rows(Q, x.cpu().numpy(), masks.cpu().numpy(), labels, border, size, cfg0)
    O.set_threads(os.cpu_count() or 1)
    xs = x.cpu().numpy()
    mk = masks.cpu().numpy()
    ref_maps = np.stack([O.detect(xs[i])[0] for i in range(10)])
    got = res.scores.cpu().numpy()
    assert np.abs(got - ref_maps).max() <= 1e-4 * np.abs(ref_maps).max()
    ref_up = [O.upsample_scores(ref_maps[i], size, size) for i in range(10)]
    samples = [(ref_up[i], mk[i], bool(labels[i]), border) for i in range(10)]
    sc, lb = O.metrics_pooled(samples)
    ref = {"pro": O.pro_at_fpr(samples), "auroc_s": O.rank_auroc(sc, lb),
           "f1": O.f1_optimal(sc, lb), "auroc_c": O.auroc_image(samples)}
    for k in KEYS:
        assert abs(row[k] - ref[k]) <= 5e-5, (k, row[k], ref[k])
