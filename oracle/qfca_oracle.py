"""CPU ORACLE for the QFCA scoring path -- TEST INFRASTRUCTURE, NOT PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / CPU baseline.  The product package never imports it.

This is a restatement of the reference implementation
(/root/reference/pkg/src/qfca) in plain C (``qfca_oracle.c``, loaded with
ctypes) plus NumPy for the small dense steps.  Each function names the
reference file:line it follows.  It is pinned against golden vectors that
were produced by running the reference itself (``tests/golden``), see
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import warnings

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
PAD_CODES = {"zero": 0, "reflect": 1, "wrap": 2}  # scoring.py:155
REFERENCE_MODES = ("median-quan", "mean-quan", "quan-median", "quan-mean")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (OpenMP) into oracle/_build/."""
    src = os.path.join(_HERE, "qfca_oracle.c")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src)):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                           "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.oracle_fit_quantizer.argtypes = [P, i64, i64, P, P, P]
        L.oracle_bin_indices.argtypes = [P, i64, i64, P, P, P, i32, P]
        L.oracle_sample_stride.argtypes = [i32, i32, i32]
        L.oracle_sample_stride.restype = i32
        L.oracle_select_reference_median.argtypes = [P, i64, i32, i32, P, P, P,
                                                     i32, i32, i32, i32, P]
        L.oracle_mismatch_row.argtypes = [P, P, P, i32, ctypes.c_double, P]
        L.oracle_mismatch_batch.argtypes = [P, i64, i32, P, P, P]
        L.oracle_channel_score.argtypes = [P, i32, i32, i32, i32, i32, P, P, P]
        L.oracle_channel_histograms.argtypes = [P, i32, i32, i32, i32, i32, P]
        L.oracle_score_channels.argtypes = [P, i64, i32, i32, i32, i32, i32, P,
                                            P, P, P, P]
        L.oracle_score_channels.restype = i32
        L.oracle_num_threads.restype = i32
        L.oracle_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------- quantizer
def fit_quantizer(values: np.ndarray, n_bins: int):
    """quantize.py:61-68 -> (lo f64, hi f64, degenerate bool)."""
    if n_bins < 1:
        raise ValueError(f"n_bins must be >= 1, got {n_bins}")
    v = np.ascontiguousarray(values, dtype=np.float32)
    c = v.shape[0]
    hw = int(np.prod(v.shape[1:]))
    lo = np.empty(c, np.float64)
    hi = np.empty(c, np.float64)
    dg = np.empty(c, np.uint8)
    lib().oracle_fit_quantizer(_p(v), c, hw, _p(lo), _p(hi), _p(dg))
    return lo, hi, dg.astype(bool)


def bin_indices(values, lo, hi, degen, n_bins: int) -> np.ndarray:
    """quantize.py:71-82 -> int32 (C, H, W)."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    c = v.shape[0]
    hw = int(np.prod(v.shape[1:]))
    out = np.empty(v.shape, np.int32)
    dg = np.ascontiguousarray(degen, dtype=np.uint8)
    lib().oracle_bin_indices(_p(v), c, hw, _p(np.ascontiguousarray(lo, np.float64)),
                             _p(np.ascontiguousarray(hi, np.float64)), _p(dg),
                             int(n_bins), _p(out))
    return out


def centers(lo: float, hi: float, n_bins: int) -> np.ndarray:
    """quantize.py:29-38."""
    lo, hi = float(lo), float(hi)
    width = (hi - lo) / n_bins if hi > lo else 1.0
    return lo + (np.arange(n_bins) + 0.5) * width


def sample_stride(h: int, w: int, budget: int) -> int:
    """quantize.py:109-116."""
    return int(lib().oracle_sample_stride(h, w, budget))


def _pad_plane(plane, margin, pad):
    """pooling.py:20-38."""
    if margin == 0:
        return plane
    if pad == "zero":
        return np.pad(plane, margin, mode="constant")
    if pad == "reflect":
        if plane.shape[0] > 1 and plane.shape[1] > 1:
            return np.pad(plane, margin, mode="reflect")
        return np.pad(plane, margin, mode="edge")
    if pad == "wrap":
        return np.pad(plane, margin, mode="wrap")
    raise ValueError(f"unknown pad mode {pad!r}")


def _sample_patches(plane, t, budget, pad):
    """quantize.py:119-132."""
    h, w = plane.shape
    r = t // 2
    padded = _pad_plane(plane, r, pad)
    s = sample_stride(h, w, budget)
    ys, xs = np.arange(0, h, s), np.arange(0, w, s)
    win = np.lib.stride_tricks.sliding_window_view(padded, (t, t))
    return win[np.ix_(ys, xs)].reshape(-1, t * t)


def _lower_median(a, axis=0):
    """quantize.py:135-140."""
    k = (a.shape[axis] - 1) // 2
    return np.take(np.partition(a, k, axis=axis), k, axis=axis)


def _quantize_values_to_hist(vals, lo, hi, n_bins):
    """quantize.py:143-147."""
    span = hi - lo if hi > lo else 1.0
    idx = np.clip(np.floor((vals - lo) * n_bins / span), 0, n_bins - 1)
    return np.bincount(idx.astype(np.int64), minlength=n_bins).astype(np.float64)


def select_reference(values, lo, hi, degen, n_bins, t, mode="median-quan",
                     sample_budget=4096, pad="reflect") -> np.ndarray:
    """quantize.py:150-200 -> weights (C, N) f64.  median-quan runs in C."""
    if mode not in REFERENCE_MODES:
        raise ValueError(f"unknown reference mode {mode!r}")
    if sample_budget < 1:
        raise ValueError("sample_budget must be >= 1")
    if t % 2 == 0 or t < 1:
        raise ValueError("patch size must be odd")
    v = np.ascontiguousarray(values, dtype=np.float32)
    c, h, w = v.shape
    t2 = t * t
    if mode == "median-quan":
        out = np.empty((c, n_bins), np.float64)
        lib().oracle_select_reference_median(
            _p(v), c, h, w, _p(np.ascontiguousarray(lo, np.float64)),
            _p(np.ascontiguousarray(hi, np.float64)),
            _p(np.ascontiguousarray(degen, np.uint8)), n_bins, t, sample_budget,
            PAD_CODES[pad], _p(out))
        return out
    weights = np.zeros((c, n_bins), np.float64)
    for ch in range(c):
        if degen[ch]:
            weights[ch, 0] = t2
            continue
        patches = _sample_patches(v[ch], t, sample_budget, pad)
        l, hh = float(lo[ch]), float(hi[ch])
        if mode == "mean-quan":
            ranked = np.sort(patches, axis=1)
            weights[ch] = _quantize_values_to_hist(
                ranked.mean(axis=0, dtype=np.float64), l, hh, n_bins)
        else:
            span = hh - l
            idx = np.clip(np.floor((patches.astype(np.float64) - l) * n_bins / span),
                          0, n_bins - 1).astype(np.int64)
            hists = np.zeros((patches.shape[0], n_bins), np.float64)
            np.add.at(hists, (np.repeat(np.arange(patches.shape[0]), t2),
                              idx.ravel()), 1.0)
            wv = _lower_median(hists, 0) if mode == "quan-median" else hists.mean(0)
            total = wv.sum()
            weights[ch] = wv * (t2 / total) if total > 0 else 0.0
            if total <= 0:
                weights[ch, 0] = t2
    return weights


def channel_histograms(idx_plane, n_bins, t, pad="reflect") -> np.ndarray:
    """(N, h, w) f64 window counts of one channel (quantize.py:85-89)."""
    idx = np.ascontiguousarray(idx_plane, dtype=np.int32)
    h, w = idx.shape
    out = np.empty((n_bins, h, w), np.float64)
    lib().oracle_channel_histograms(_p(idx), h, w, n_bins, t, PAD_CODES[pad], _p(out))
    return out


def patch_histograms(bins, n_bins, t, pad="reflect") -> np.ndarray:
    """quantize.py:92-106 -> (C, N, H, W) float32 counts."""
    if t % 2 == 0:
        raise ValueError(f"patch size must be odd, got {t}")
    return np.stack([channel_histograms(b, n_bins, t, pad) for b in bins]
                    ).astype(np.float32)


# ---------------------------------------------------------------- transport
def mismatch_batch(pb, r, q) -> np.ndarray:
    """transport.py:110-125."""
    pb = np.ascontiguousarray(pb, np.float64)
    out = np.empty_like(pb)
    lib().oracle_mismatch_batch(_p(pb), pb.shape[0], pb.shape[1],
                                _p(np.ascontiguousarray(r, np.float64)),
                                _p(np.ascontiguousarray(q, np.float64)), _p(out))
    return out


def quantized_mismatch(p, r, q) -> np.ndarray:
    """transport.py:38-70 without the validation (equal masses assumed)."""
    p = np.ascontiguousarray(p, np.float64)
    r = np.ascontiguousarray(r, np.float64)
    return mismatch_batch(p[None], r * (p.sum() / r.sum()) if r.sum() > 0 else r, q)[0]


# ---------------------------------------------------------------- smoothing
def _gauss_kernel(sigma):
    """features.py:49-53."""
    radius = int(np.ceil(3 * sigma))
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def _sep_convolve(plane, kernel, pad="reflect"):
    """features.py:56-69."""
    r = kernel.size // 2
    mode = {"reflect": "reflect", "wrap": "wrap", "zero": "constant"}[pad]
    p = np.pad(plane, ((r, r), (0, 0)), mode=mode)
    rows = np.zeros_like(plane, dtype=np.float64)
    for i, kv in enumerate(kernel):
        rows += kv * p[i:i + plane.shape[0]]
    p = np.pad(rows, ((0, 0), (r, r)), mode=mode)
    out = np.zeros_like(rows)
    for i, kv in enumerate(kernel):
        out += kv * p[:, i:i + plane.shape[1]]
    return out


def gaussian_blur(plane, sigma, pad="reflect"):
    """features.py:72-77."""
    if sigma <= 0:
        return np.asarray(plane, dtype=np.float64)
    return _sep_convolve(np.asarray(plane, np.float64), _gauss_kernel(sigma), pad)


def smooth_scores(m, sigma_s, pad="reflect"):
    """scoring.py:133-138."""
    if sigma_s == 0:
        return np.asarray(m, dtype=np.float64)
    return gaussian_blur(m, sigma_s, pad)


def image_score_of(scores, border):
    """scoring.py:141-146."""
    h, w = scores.shape
    b = min(border, (h - 1) // 2, (w - 1) // 2)
    interior = scores[b:h - b, b:w - b] if b > 0 else scores
    return float(interior.max())


def resize_plane(plane, out_h, out_w):
    """tensor_io.py:127-151 (bilinear, half-pixel centres, float32 result)."""
    h, w = plane.shape
    if (h, w) == (out_h, out_w):
        return plane.astype(np.float32, copy=False)
    ys = (np.arange(out_h) + 0.5) * h / out_h - 0.5
    xs = (np.arange(out_w) + 0.5) * w / out_w - 0.5
    y0 = np.clip(np.floor(ys), 0, h - 1).astype(int)
    x0 = np.clip(np.floor(xs), 0, w - 1).astype(int)
    y1 = np.clip(y0 + 1, 0, h - 1)
    x1 = np.clip(x0 + 1, 0, w - 1)
    fy = np.clip(ys - y0, 0.0, 1.0)[:, None]
    fx = np.clip(xs - x0, 0.0, 1.0)[None, :]
    p = plane.astype(np.float64)
    top = p[np.ix_(y0, x0)] * (1 - fx) + p[np.ix_(y0, x1)] * fx
    bot = p[np.ix_(y1, x0)] * (1 - fx) + p[np.ix_(y1, x1)] * fx
    return (top * (1 - fy) + bot * fy).astype(np.float32)


def upsample_scores(scores, out_h, out_w):
    """scoring.py:149-152."""
    return resize_plane(np.asarray(scores, np.float64), out_h, out_w).astype(np.float64)


# ---------------------------------------------------------------- PCA
def pca_fit(values, k):
    """features.py:157-180 -> (mean, components (k,C), eigenvalues)."""
    c = values.shape[0]
    if not (1 <= k <= c):
        raise ValueError(f"k must be in [1, {c}], got {k}")
    x = values.reshape(c, -1).astype(np.float64).T
    mean = x.mean(axis=0)
    xc = x - mean
    cov = xc.T @ xc / x.shape[0]
    evals, evecs = np.linalg.eigh(cov)
    order = np.argsort(evals, kind="stable")[::-1][:k]
    evals = np.clip(evals[order], 0.0, None)
    comps = evecs[:, order].T.copy()
    for row in comps:
        if row[np.argmax(np.abs(row))] < 0:
            row *= -1.0
    return mean, comps, evals


def pca_residual(values, mean, comps):
    """features.py:183-193 -> float32 residual."""
    c = values.shape[0]
    x = values.reshape(c, -1).astype(np.float64)
    xc = x - mean[:, None]
    proj = comps.T @ (comps @ xc)
    return (xc - proj).reshape(values.shape).astype(np.float32)


# ---------------------------------------------------------------- detect
def _smooth_error_planes(planes, t, sigma_p, pad):
    """scoring.py:88-98."""
    if math.isinf(sigma_p):
        r = t // 2
        if pad == "zero":
            h, w = planes.shape[1:]
            out = np.empty_like(planes, dtype=np.float64)
            for i, pl in enumerate(planes):
                cs = np.zeros((h + 1, w + 1))
                cs[1:, 1:] = np.cumsum(np.cumsum(pl, 0), 1)
                rr = np.arange(h)
                cc = np.arange(w)
                r0, r1 = np.maximum(rr - r, 0), np.minimum(rr + r + 1, h)
                c0, c1 = np.maximum(cc - r, 0), np.minimum(cc + r + 1, w)
                out[i] = (cs[np.ix_(r1, c1)] - cs[np.ix_(r0, c1)]
                          - cs[np.ix_(r1, c0)] + cs[np.ix_(r0, c0)]) / (t * t)
            return out
        padded = np.pad(planes, ((0, 0), (r, r), (r, r)),
                        mode={"reflect": "reflect", "wrap": "wrap"}[pad])
        b, h, w = planes.shape
        cs = np.zeros((b, padded.shape[1] + 1, padded.shape[2] + 1))
        cs[:, 1:, 1:] = padded
        cs = cs.cumsum(1).cumsum(2)
        out = cs[:, t:t + h, t:t + w] - cs[:, :h, t:t + w]
        out -= cs[:, t:t + h, :w]
        out += cs[:, :h, :w]
        return out / float(t * t)
    r = t // 2
    x = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma_p) ** 2)
    k /= k.sum()
    return np.stack([_sep_convolve(p, k, pad) for p in planes])


def detect(values, n_bins=16, patch_size=9, sigma_p=math.inf, sigma_s=1.0,
           pca_components=0, reference_mode="median-quan", sample_budget=4096,
           border_exclusion=None, pad="reflect", return_stages=False):
    """scoring.py:235-299 (detect) -> (scores f64 (h,w), image_score, degenerate).

    The uniform-sigma_p path runs the C restatement of _channel_score_kernel
    (parallel over channels, fixed-order fp64 sum).
    """
    values = np.ascontiguousarray(values, dtype=np.float32)
    stages = {}
    if pca_components > 0:
        mean, comps, ev = pca_fit(values, min(pca_components, values.shape[0]))
        values = pca_residual(values, mean, comps)
        stages.update(pca_mean=mean, pca_components=comps, pca_eigenvalues=ev,
                      residual=values)
    c, h, w = values.shape
    lo, hi, dg = fit_quantizer(values, n_bins)
    bins = bin_indices(values, lo, hi, dg, n_bins)
    refw = select_reference(values, lo, hi, dg, n_bins, patch_size,
                            reference_mode, sample_budget, pad)
    acc = np.zeros((h, w), np.float64)
    if math.isinf(sigma_p):
        used = int(lib().oracle_score_channels(
            _p(bins), c, h, w, n_bins, patch_size, PAD_CODES[pad], _p(lo), _p(hi),
            _p(dg.astype(np.uint8)), _p(np.ascontiguousarray(refw)), _p(acc)))
    else:
        used = 0
        for ch in range(c):
            if dg[ch]:
                continue
            counts = channel_histograms(bins[ch], n_bins, patch_size, pad)
            counts = counts.astype(np.float32).astype(np.float64)
            pb = counts.transpose(1, 2, 0).reshape(-1, n_bins)
            err = mismatch_batch(pb, refw[ch], centers(lo[ch], hi[ch], n_bins))
            err = err.reshape(h, w, n_bins).transpose(2, 0, 1)
            sm = _smooth_error_planes(err, patch_size, sigma_p, pad)
            acc += np.take_along_axis(sm, bins[ch][None].astype(np.int64), 0)[0]
            used += 1
    degenerate = used == 0
    if degenerate:
        warnings.warn("all channels degenerate; anomaly map is all zeros")
        agg = acc
    else:
        agg = acc / used
    final = smooth_scores(agg, sigma_s, pad)
    border = patch_size // 2 if border_exclusion is None else border_exclusion
    score = image_score_of(final, border)
    if return_stages:
        stages.update(lo=lo, hi=hi, degenerate=dg, bins=bins, ref_weights=refw,
                      agg=agg, used=used)
        return final, score, degenerate, stages
    return final, score, degenerate


# ---------------------------------------------------------------------------
# Evaluation metrics (reference pkg/src/qfca/metrics.py), restated with
# independent NumPy / SciPy formulations: the checker for metrics.cu.
# ---------------------------------------------------------------------------

def metrics_pooled(samples):
    """metrics.py:37-41, 61-68 -- interiors pooled in sample order.
    samples: list of (scores, mask, image_label, border)."""
    sc, lb = [], []
    for s, m, _, b in samples:
        if b:
            s, m = s[b:-b, b:-b], m[b:-b, b:-b]
        sc.append(np.asarray(s).ravel())
        lb.append(np.asarray(m, bool).ravel())
    return np.concatenate(sc), np.concatenate(lb)


def rank_auroc(scores, labels):
    """metrics.py:44-58 -- Mann-Whitney U with average ranks (scipy rankdata)."""
    from scipy.stats import rankdata
    pos = int(labels.sum())
    neg = labels.size - pos
    if pos == 0 or neg == 0:
        return None
    r = rankdata(np.asarray(scores, np.float64), method="average")
    return float((r[labels].sum() - pos * (pos + 1) / 2) / (pos * neg))


def f1_optimal(scores, labels):
    """metrics.py:157-172 -- best 2 tp / (predicted + positives) over the
    thresholds "score >= t" for every distinct score t."""
    n_pos = int(labels.sum())
    if n_pos == 0:
        return None
    u, inv = np.unique(scores, return_inverse=True)
    tot = np.bincount(inv, minlength=u.size)
    pos = np.bincount(inv, weights=labels.astype(np.float64), minlength=u.size).astype(np.int64)
    k = np.cumsum(tot[::-1])[::-1]
    tp = np.cumsum(pos[::-1])[::-1]
    return float((2.0 * tp / (k + n_pos)).max())


def connected_components(mask):
    """metrics.py:76-80 -- scipy.ndimage.label with the 3x3 structure."""
    from scipy import ndimage
    lab, n = ndimage.label(np.asarray(mask, bool), structure=np.ones((3, 3), int))
    return lab, int(n)


def pro_curve(samples, thresholds):
    """metrics.py:91-120 -- per-threshold mean component overlap and FPR,
    counting "score >= t" directly for every component."""
    comps, normal = [], []
    for s, m, _, b in samples:
        if b:
            s, m = s[b:-b, b:-b], m[b:-b, b:-b]
        m = np.asarray(m, bool)
        normal.append(s[~m])
        lab, n = connected_components(m)
        comps += [s[lab == k] for k in range(1, n + 1)]
    if not comps:
        return None
    normal = np.concatenate(normal)
    t = np.asarray(thresholds, np.float64)
    pro = np.zeros(t.size)
    for c in comps:
        pro += (c[None, :].astype(np.float64) >= t[:, None]).sum(1) / c.size
    pro /= len(comps)
    fpr = (np.zeros(t.size) if normal.size == 0 else
           (normal[None, :].astype(np.float64) >= t[:, None]).sum(1) / normal.size)
    return fpr, pro


def pro_at_fpr(samples, limit=0.3, thresholds=None):
    """metrics.py:83-88, 125-154 -- quantile thresholds, trapezoid to the limit."""
    if thresholds is None:
        scores, _ = metrics_pooled(samples)
        thresholds = np.unique(np.quantile(scores, np.linspace(0.0, 1.0, 500)))[::-1]
    r = pro_curve(samples, thresholds)
    if r is None:
        return None
    f = np.r_[0.0, r[0], 1.0]
    p = np.r_[0.0, r[1], 1.0]
    area = 0.0
    for i in range(1, f.size):
        if f[i] <= f[i - 1]:
            continue
        hi = min(f[i], limit)
        if hi <= f[i - 1]:
            break
        ph = p[i - 1] + (p[i] - p[i - 1]) * (hi - f[i - 1]) / (f[i] - f[i - 1])
        area += 0.5 * (p[i - 1] + ph) * (hi - f[i - 1])
        if f[i] >= limit:
            break
    return area / limit


def auroc_image(samples):
    """metrics.py:175-179 -- AUROC of per-image interior maxima."""
    mx, lab = [], []
    for s, m, l, b in samples:
        mx.append((s[b:-b, b:-b] if b else s).max())
        lab.append(bool(l))
    return rank_auroc(np.array(mx), np.array(lab))
