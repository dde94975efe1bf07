"""Generate golden input/output vectors by RUNNING THE REFERENCE ITSELF.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Writes small compressed .npz fixtures next to this script.  They pin the CPU
oracle (oracle/qfca_oracle.py) and are the parity targets of the GPU tests.
Nothing here is imported by the product or by tests at run time.
"""

from __future__ import annotations

import math
import os
import sys
import tempfile
import zlib

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_EXPORTER = "/root/reference/pkg/exporter/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_EXPORTER)

import qfca  # noqa: E402
from qfca import quantize, scoring, transport  # noqa: E402
from qfca.features import FeatureMap, pca_fit, pca_residual  # noqa: E402


def smooth_random_map(rng, c, h, w, sigma=3.0):
    z = rng.standard_normal((c, h, w))
    f = np.fft.rfft2(z)
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.rfftfreq(w)[None, :]
    g = np.exp(-2 * (np.pi * sigma) ** 2 * (fy ** 2 + fx ** 2))
    out = np.fft.irfft2(f * g, s=(h, w))
    return (out / np.abs(out).max(axis=(1, 2), keepdims=True)).astype(np.float32)


def run_case(values, cfg_kwargs, with_counts=True):
    cfg = scoring.PipelineConfig(**cfg_kwargs)
    v = np.ascontiguousarray(values, np.float32)
    q = quantize.fit_quantizer(v, cfg.n_bins)
    b = quantize.bin_indices(v, q)
    ref = quantize.select_reference(v, q, cfg.patch_size, mode=cfg.reference_mode,
                                    sample_budget=cfg.sample_budget, pad=cfg.pad)
    out = dict(values=v, lo=q.lo, hi=q.hi, degenerate=q.degenerate,
               bins=b.indices.astype(np.int32), ref_weights=ref.weights)
    if with_counts:
        out["counts"] = quantize.patch_histograms(b, cfg.patch_size, pad=cfg.pad).counts
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        am = scoring.detect(FeatureMap(values=v, scale=1), cfg)
    out.update(scores=am.scores, image_score=np.float64(am.image_score),
               detect_degenerate=np.bool_(am.degenerate))
    for k, val in cfg_kwargs.items():
        out["cfg_" + k] = np.asarray(val)
    return out


def save(name, d):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    print("wrote", name, {k: getattr(v, "shape", ()) for k, v in d.items()})


def small_cases():
    rng = np.random.default_rng(20261018)
    cases = [
        ("rand_n16_t9_reflect", (5, 13, 17), dict(n_bins=16, patch_size=9)),
        ("rand_n4_t3_reflect", (4, 11, 9), dict(n_bins=4, patch_size=3)),
        ("rand_n5_t5_wrap", (3, 12, 10), dict(n_bins=5, patch_size=5, pad="wrap")),
        ("rand_n16_t3_zero", (3, 10, 12), dict(n_bins=16, patch_size=3, pad="zero")),
        ("rand_n2_t1_reflect", (2, 6, 7), dict(n_bins=2, patch_size=1)),
        ("rand_n1_t3_reflect", (2, 8, 8), dict(n_bins=1, patch_size=3)),
        ("rand_n7_t5_budget", (3, 20, 18), dict(n_bins=7, patch_size=5, sample_budget=30)),
        ("rand_n16_t9_wrap", (3, 16, 16), dict(n_bins=16, patch_size=9, pad="wrap")),
        ("rand_n33_t7_reflect", (3, 15, 21), dict(n_bins=33, patch_size=7)),
        ("rand_n256_t9_reflect", (2, 24, 24), dict(n_bins=256, patch_size=9)),
        ("rand_n16_t17_reflect", (2, 20, 22), dict(n_bins=16, patch_size=17)),
        ("rand_n16_t9_border2", (3, 14, 14), dict(n_bins=16, patch_size=9,
                                                 border_exclusion=2, sigma_s=0.5)),
        ("rand_n16_t9_sigma0", (3, 14, 14), dict(n_bins=16, patch_size=9, sigma_s=0.0)),
    ]
    for name, shape, kw in cases:
        v = rng.random(shape).astype(np.float32)
        save("small_" + name, run_case(v, kw))
    # degenerate channels, ReLU-like zeros, tiny planes
    v = rng.random((4, 9, 11)).astype(np.float32)
    v[1] = 2.5
    v[2] = np.maximum(rng.standard_normal((9, 11)), 0).astype(np.float32)
    save("small_degenerate_mix", run_case(v, dict(n_bins=8, patch_size=3)))
    save("small_all_degenerate", run_case(np.full((2, 6, 6), 1.0, np.float32),
                                          dict(n_bins=8, patch_size=3)))
    save("small_tiny_2x2", run_case(rng.random((2, 2, 2)).astype(np.float32),
                                    dict(n_bins=4, patch_size=3)))
    save("small_tiny_1xw", run_case(rng.random((2, 1, 9)).astype(np.float32),
                                    dict(n_bins=4, patch_size=3)))
    save("small_tiny_hx1", run_case(rng.random((2, 7, 1)).astype(np.float32),
                                    dict(n_bins=4, patch_size=3)))
    save("small_margin_gt_plane", run_case(rng.random((2, 4, 5)).astype(np.float32),
                                           dict(n_bins=6, patch_size=9)))
    # smooth maps like the reference tests (test_scoring.py:166-175)
    v = smooth_random_map(np.random.default_rng(3), 4, 48, 48)
    v[:, 20:28, 20:28] += 1.5
    save("smooth_square_48", run_case(v, dict(patch_size=5)))
    v = smooth_random_map(np.random.default_rng(5), 4, 32, 32)
    save("smooth_n1024_32", run_case(v, dict(n_bins=1024, sample_budget=32 * 32),
                                     with_counts=False))
    # periodic stripes with wrap (test_scoring.py:154-163)
    col = np.array([0.0, 1 / 3, 2 / 3], np.float32)
    plane = np.tile(col, (30, 10))
    save("periodic_wrap", run_case(np.stack([plane, plane.T]),
                                   dict(n_bins=16, patch_size=3, pad="wrap",
                                        sample_budget=900), with_counts=False))
    # other reference modes and finite sigma_p (the "next" rows)
    v = smooth_random_map(np.random.default_rng(11), 3, 24, 26)
    for mode in ("mean-quan", "quan-median", "quan-mean"):
        save("mode_" + mode.replace("-", "_"),
             run_case(v, dict(n_bins=8, patch_size=5, reference_mode=mode),
                      with_counts=False))
    save("sigma_p_2", run_case(v, dict(n_bins=8, patch_size=5, sigma_p=2.0),
                               with_counts=False))
    extra_mode_cases()
    # T and N sweeps on one medium map
    v = smooth_random_map(np.random.default_rng(12), 4, 40, 40)
    for t in (3, 5, 9, 17, 33, 65):
        save(f"sweep_t{t}", run_case(v, dict(n_bins=16, patch_size=t),
                                     with_counts=False))
    for n in (8, 64, 256):
        save(f"sweep_n{n}", run_case(v, dict(n_bins=n, patch_size=9),
                                     with_counts=False))


def extra_mode_cases():
    """The other reference modes beyond the defaults: zero / wrap padding, sparse
    sample grids, N above 8 and 128 (NumPy's pairwise-sum branches in the quan-*
    rescale), patches of more than 128 values (mean-quan's segmented sort)."""
    rng = np.random.default_rng(21)
    v = np.maximum(smooth_random_map(rng, 3, 33, 37) + 0.2, 0).astype(np.float32)
    save("mode_mean_quan_zero", run_case(v, dict(n_bins=16, patch_size=9, pad="zero",
                                                 reference_mode="mean-quan", sample_budget=200),
                                         with_counts=False))
    save("mode_mean_quan_t17", run_case(v, dict(n_bins=16, patch_size=17,
                                                reference_mode="mean-quan", sample_budget=300),
                                        with_counts=False))
    save("mode_quan_mean_wrap_n32", run_case(v, dict(n_bins=32, patch_size=7, pad="wrap",
                                                     reference_mode="quan-mean"),
                                             with_counts=False))
    save("mode_quan_median_n200", run_case(v, dict(n_bins=200, patch_size=3,
                                                   reference_mode="quan-median"),
                                           with_counts=False))


def transport_cases():
    rng = np.random.default_rng(7)
    rows, refs, qs, outs = [], [], [], []
    for _ in range(200):
        n = int(rng.integers(1, 33))
        m = float(rng.integers(1, 100))
        p = rng.multinomial(int(m), np.ones(n) / n).astype(np.float64)
        r = rng.multinomial(int(m), rng.dirichlet(np.ones(n))).astype(np.float64)
        q = np.cumsum(rng.random(n) + 0.01)
        e = transport.quantized_mismatch(p, r, q)
        pad = 32 - n
        rows.append(np.r_[p, np.zeros(pad)])
        refs.append(np.r_[r, np.zeros(pad)])
        qs.append(np.r_[q, np.arange(1, pad + 1) + q[-1]])
        outs.append(np.r_[e, np.zeros(pad)])
    save("transport_random", dict(P=np.array(rows), R=np.array(refs),
                                  Q=np.array(qs), E=np.array(outs)))


def wrn_case():
    """Config 1: one 256x256 synthetic texture with a planted defect,
    reference default backbone with random init, default bins/patch size."""
    import torch
    from qfca.synth import SynthConfig, generate_class
    from qtf_exporter.export import _build_backbone, _load_image_tensor

    with tempfile.TemporaryDirectory() as d:
        generate_class(d, "noise", SynthConfig(kind="noise", size=256,
                                               n_images=4, n_good=3, seed=0))
        img = os.path.join(d, "noise", "test", "planted", "003.png")
        mask = os.path.join(d, "noise", "ground_truth", "planted", "003_mask.png")
        from qfca.tensor_io import load_mask
        m = load_mask(mask)
        trunk = _build_backbone("random")
        with torch.no_grad():
            feats = trunk(_load_image_tensor(img, 256))[0].numpy().astype(np.float32)
    d = run_case(feats, dict(), with_counts=False)
    up = scoring.upsample_scores(d["scores"], 256, 256)
    d.update(upsampled=up.astype(np.float32), mask=np.asarray(m, bool))
    save("wrn256_qfca", d)
    # QFCA+ (k = 10): the reference's own PCA model, residual and map
    fm = FeatureMap(values=feats, scale=8)
    model = pca_fit(fm, 10)
    res = pca_residual(fm, model).values
    cfg = scoring.PipelineConfig(pca_components=10)
    am = scoring.detect(fm, cfg)
    save("wrn256_qfca_plus", dict(
        pca_mean=model.mean, pca_components=model.components,
        pca_eigenvalues=model.eigenvalues, residual=res, scores=am.scores,
        image_score=np.float64(am.image_score)))


if __name__ == "__main__":
    small_cases()
    transport_cases()
    wrn_case()
