"""Golden vectors for the evaluation metrics, made by RUNNING THE REFERENCE's
qfca.metrics (build container only; the reference does not travel):

    python tests/golden/make_metrics_golden.py

Writes metrics_*.npz next to this script: the maps, masks, image labels and
borders of a few sample sets, and the reference's pro / auroc_s / f1 /
auroc_c, PRO thresholds and curve, and the component labels of each mask.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from qfca import metrics as M  # noqa: E402


def smooth(rng, h, w, sigma=2.5):
    z = rng.standard_normal((h, w))
    f = np.fft.rfft2(z)
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.rfftfreq(w)[None, :]
    return np.fft.irfft2(f * np.exp(-2 * (np.pi * sigma) ** 2 * (fy ** 2 + fx ** 2)), s=(h, w))


def blobs(rng, h, w, n):
    m = np.zeros((h, w), bool)
    yy, xx = np.mgrid[:h, :w]
    for _ in range(n):
        cy, cx = rng.integers(0, h), rng.integers(0, w)
        ry, rx = rng.integers(1, max(2, h // 6)), rng.integers(1, max(2, w // 6))
        m |= ((yy - cy) / ry) ** 2 + ((xx - cx) / rx) ** 2 <= 1.0
    # a few isolated pixels and diagonal chains (8-connectivity cases)
    for _ in range(3):
        y, x = rng.integers(0, h), rng.integers(0, w)
        m[y, x] = True
        for k in range(1, 4):
            if y + k < h and x + k < w:
                m[y + k, x + k] = True
    return m


def make_set(rng, shapes, n_per, dtype, border, round_to=None):
    samples = []
    for (h, w) in shapes:
        for i in range(n_per):
            label = bool(rng.integers(0, 2)) if i else True
            m = blobs(rng, h, w, int(rng.integers(1, 4))) if label else np.zeros((h, w), bool)
            s = smooth(rng, h, w) + m * rng.uniform(0.03, 0.15)
            if round_to is not None:
                s = np.round(s, round_to)
            samples.append(M.EvalSample(scores=s.astype(dtype), mask=m, image_label=label,
                                        border=border))
    return samples


def save(name, samples):
    d = {}
    for i, s in enumerate(samples):
        d[f"scores_{i}"] = s.scores
        d[f"mask_{i}"] = s.mask
        d[f"labels_cc_{i}"] = M.connected_components(s.interior()[1])[0].astype(np.int32)
    d["n"] = np.int64(len(samples))
    d["image_label"] = np.array([s.image_label for s in samples])
    d["border"] = np.array([s.border for s in samples])
    scores, _ = M._pooled(samples)
    thr = M._pro_thresholds(scores)
    fpr, pro = M._pro_curve(samples, thr)
    d["thresholds"], d["fpr"], d["pro_curve"] = thr, fpr, pro
    for key, fn in (("pro", M.pro_at_fpr), ("auroc_s", M.auroc_pixel), ("f1", M.f1_optimal),
                    ("auroc_c", M.auroc_image)):
        d[key] = np.float64(fn(samples))
    d["pro_limit_01"] = np.float64(M.pro_at_fpr(samples, 0.1))
    np.savez_compressed(os.path.join(OUT, f"metrics_{name}.npz"), **d)
    print(name, {k: float(d[k]) for k in ("pro", "auroc_s", "f1", "auroc_c")}, thr.size)


def main():
    rng = np.random.default_rng(2510)
    save("f64", make_set(rng, [(40, 48)], 6, np.float64, 2))
    save("f32_ties", make_set(rng, [(33, 37)], 5, np.float32, 1, round_to=2))
    save("mixed", make_set(rng, [(24, 24)], 3, np.float64, 0) +
         make_set(rng, [(30, 20)], 3, np.float64, 3))


if __name__ == "__main__":
    main()
