"""Evaluation metrics on the GPU -- drop-in for the reference's ``qfca.metrics``.

Same names, defaults, errors and results as reference pkg/src/qfca/metrics.py
(PRO up to an FPR limit, optimal-threshold F1, pixel and image AUROC with
average ranks for ties, 8-connected components).  The pixel work runs in
``csrc/metrics.cu`` through the C-ABI: the pooled interiors are gathered on
the device (``qfca_pool_interior``), sorted once (``qfca_rank_stats``, which
also yields the exact rank sum and the best F1), labelled
(``qfca_components``) and histogrammed over the PRO thresholds
(``qfca_pro_histograms`` / ``qfca_pro_accumulate``).  The host keeps the
O(thresholds) bookkeeping: NumPy's quantile interpolation over the <= 1000
order statistics it needs, and the trapezoid integration.

Scores and masks may be NumPy arrays or torch tensors (CUDA or not).  Every
result equals the reference's bit for bit: the rank sums and counts are exact
integers and the fp64 divisions / in-order sums are the reference's own.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._dev import empty, is_torch, zeros

PRO_FPR_LIMIT = 0.3  # metrics.py:13
PRO_MAX_THRESHOLDS = 500  # metrics.py:14
_MAX_KERNEL_THRESHOLDS = 2048  # csrc/metrics.cu MAX_THR
_HIST_CELLS = 1 << 26  # per-pass component histogram cells (256 MiB of int32)


class UndefinedMetricError(ValueError):
    """The metric is undefined for the given label distribution (metrics.py:19-20)."""


def _shape(a) -> tuple:
    return tuple(a.shape)


@dataclass(frozen=True)
class EvalSample:
    """metrics.py:23-42 -- one map, its ground-truth mask, image label, border."""

    scores: object  # (H, W) float, NumPy or torch
    mask: object  # (H, W) bool
    image_label: bool
    border: int = 0

    def __post_init__(self):
        if _shape(self.scores) != _shape(self.mask):
            raise ValueError("scores and mask shapes differ")
        h, w = _shape(self.scores)
        if self.border >= min(h, w) / 2:
            raise ValueError("border exclusion leaves no pixels")

    def interior(self):
        b = self.border
        if b == 0:
            return self.scores, self.mask
        return self.scores[b:-b, b:-b], self.mask[b:-b, b:-b]


def _np_dtype(a):
    if is_torch(a):
        return {torch.float64: np.float64, torch.float32: np.float32,
                torch.float16: np.float16}.get(a.dtype, np.float64)
    return np.asarray(a).dtype


def _device_tables(group, dev):
    """(score bytes, score pointer table, mask pointer table) on ``dev`` when
    every map of the group is already a contiguous device tensor (scores all
    float64 or all float32, masks bool / uint8), else None."""
    sd = None
    sp, mp = [], []
    for _, s in group:
        sc, m = s.scores, s.mask
        if not (is_torch(sc) and is_torch(m)) or sc.device != dev or m.device != dev:
            return None
        if sc.dtype not in (torch.float64, torch.float32) or (sd is not None and sc.dtype != sd):
            return None
        if m.dtype not in (torch.bool, torch.uint8) or tuple(m.shape) != tuple(sc.shape):
            return None
        if not (sc.is_contiguous() and m.is_contiguous()):
            return None
        sd = sc.dtype
        sp.append(sc.data_ptr())
        mp.append(m.data_ptr())
    tab = torch.tensor(sp + mp, dtype=torch.int64).pin_memory().to(dev, non_blocking=True)
    k = len(sp)
    return (8 if sd == torch.float64 else 4), tab[:k], tab[k:]


class _Pool:
    """Device copy of the pooled interiors (metrics.py:62-68 _pooled order).

    Consecutive samples of the same (H, W, border) form one group, gathered by
    one ``qfca_pool_interior`` call into a contiguous (images, h, w) slice.
    """

    def __init__(self, samples: list[EvalSample]):
        if not samples:
            raise ValueError("no samples")
        dev = N.require_cuda()
        stream = N.stream()
        self.groups = []  # (offset, images, h, w)
        self._tables = []
        groups, cur = [], []
        for s in samples:
            key = (_shape(s.scores), s.border)
            if cur and key != cur[0][0]:
                groups.append(cur)
                cur = []
            cur.append((key, s))
        groups.append(cur)
        sizes = []
        for g in groups:
            (H, W), b = g[0][0]
            sizes.append(len(g) * (H - 2 * b) * (W - 2 * b))
        self.n = int(sum(sizes))
        self.dtype = np.result_type(*[_np_dtype(s.scores) for s in samples])
        self.scores = empty((self.n,), torch.float64)
        self.scores32 = empty((self.n,), torch.float32)  # ranked instead when exact
        self.inexact = zeros((1,), torch.int32)
        self.labels = empty((self.n,), torch.uint8)
        enc = zeros((len(samples),), torch.int64)  # order-preserving max encoding
        off = img = 0
        for g, size in zip(groups, sizes):
            (H, W), b = g[0][0]
            k = len(g)
            h, w = H - 2 * b, W - 2 * b
            out = (self.scores[off:].data_ptr(), self.labels[off:].data_ptr(),
                   self.scores32[off:].data_ptr(), self.inexact.data_ptr(),
                   enc[img:].data_ptr(), stream)
            tbl = _device_tables(g, dev)
            if tbl is not None:
                # maps already resident: read each in place through a pointer table
                sb, stab, mtab = tbl
                self._tables.append(stab)  # alive until the pool is dropped
                N.call("qfca_pool_interior_table", stab.data_ptr(), sb, mtab.data_ptr(), k, H, W,
                       b, *out)
            else:
                sc = empty((k, H, W), torch.float64)
                mk = empty((k, H, W), torch.uint8)
                for i, (_, s) in enumerate(g):
                    sc[i].copy_(torch.as_tensor(np.asarray(s.scores, dtype=np.float64))
                                if not is_torch(s.scores) else s.scores.to(torch.float64))
                    m = s.mask if is_torch(s.mask) else torch.from_numpy(
                        np.ascontiguousarray(np.asarray(s.mask, dtype=bool)))
                    mk[i].copy_(m.to(device=dev, dtype=torch.uint8))
                N.call("qfca_pool_interior", sc.data_ptr(), 8, mk.data_ptr(), k, H, W, b, *out)
            self.groups.append((off, k, h, w))
            off += size
            img += k
        self.image_labels = np.array([bool(s.image_label) for s in samples], dtype=bool)
        # metrics.py:175-179 -- interior maxima, decoded from the pool kernel's encoding
        u = enc.cpu().numpy().view(np.uint64)
        top = (u >> np.uint64(63)).astype(bool)
        bits = np.where(top, u & np.uint64(0x7FFFFFFFFFFFFFFF), ~u)
        self.image_max = torch.from_numpy(bits.view(np.float64).copy()).to(dev)
        self._rank = None

    def rank(self):
        """(positives, 2 x positive rank sum, best F1, ascending scores).  When
        every pooled score is a float32 value (upsampled maps are) the sort
        runs on 32-bit keys: same order, same ties, half the radix passes."""
        if self._rank is None:
            keys = self.scores32 if int(self.inexact.item()) == 0 else self.scores
            self._rank = _rank_stats(keys, self.labels, want_sorted=True)
        return self._rank


def _rank_stats(scores: torch.Tensor, labels: torch.Tensor, want_sorted: bool):
    n = scores.numel()
    kb = scores.element_size()
    wsb = int(N.lib().qfca_rank_stats_workspace_bytes(n, kb))
    if wsb < 0:
        raise ValueError(f"{n} pooled pixels: the rank kernels take 1 .. 2^31 - 1")
    ws = empty((wsb,), torch.uint8)
    stats = zeros((3,), torch.int64)
    srt = empty((n,), scores.dtype) if want_sorted else None
    N.call("qfca_rank_stats", scores.data_ptr(), kb, labels.data_ptr(), n, ws.data_ptr(), wsb,
           N.ptr(srt), stats.data_ptr(), N.stream())
    pos, r2, f1bits = (int(v) & 0xFFFFFFFFFFFFFFFF for v in stats.cpu().tolist())
    f1 = struct.unpack("<d", struct.pack("<Q", f1bits))[0]
    return pos, r2, f1, srt


def _auroc(pos: int, n: int, r2: int) -> float:
    """metrics.py:44-58 -- Mann-Whitney from the exact rank sum."""
    neg = n - pos
    if pos == 0 or neg == 0:
        raise UndefinedMetricError("AUROC needs both classes")
    rank_sum = np.float64(r2) / 2.0  # exact: r2 < 2^53
    return float((rank_sum - pos * (pos + 1) / 2) / (pos * neg))


def auroc_pixel(samples: list[EvalSample]) -> float:
    """metrics.py:71-73 -- pixel AUROC over the pooled interiors."""
    return _pool_auroc(_Pool(samples))


def _pool_auroc(p: _Pool) -> float:
    pos, r2, _, _ = p.rank()
    return _auroc(pos, p.n, r2)


def f1_optimal(samples: list[EvalSample]) -> float:
    """metrics.py:157-172 -- best F1 over all thresholds of the pooled scores."""
    return _pool_f1(_Pool(samples))


def _pool_f1(p: _Pool) -> float:
    pos, _, f1, _ = p.rank()
    if pos == 0:
        raise UndefinedMetricError("F1 needs at least one positive pixel")
    return float(f1)


def auroc_image(samples: list[EvalSample]) -> float:
    """metrics.py:175-179 -- AUROC over per-image interior maxima."""
    return _pool_auroc_image(_Pool(samples))


def _pool_auroc_image(p: _Pool) -> float:
    lab = torch.from_numpy(p.image_labels.astype(np.uint8)).to(p.image_max.device)
    pos, r2, _, _ = _rank_stats(p.image_max, lab, want_sorted=False)
    return _auroc(pos, p.image_max.numel(), r2)


def connected_components(mask) -> tuple:
    """metrics.py:76-80 -- 8-connected labels in raster order starting at 1."""
    torch_in = is_torch(mask)
    m = mask if torch_in else torch.from_numpy(np.ascontiguousarray(np.asarray(mask, dtype=bool)))
    if m.dim() != 2:
        raise ValueError("connected_components takes a 2-D mask")
    m = m.to(device=N.require_cuda(), dtype=torch.uint8).contiguous()
    h, w = m.shape
    if h == 0 or w == 0:
        lab = torch.zeros((h, w), dtype=torch.int32, device=m.device)
        return (lab if torch_in else lab.cpu().numpy()), 0
    comp, count = _components(m.reshape(1, h, w), 1, h, w)
    lab = (comp + 1).reshape(h, w)
    return (lab if torch_in else lab.cpu().numpy()), count


def _components(mask_u8: torch.Tensor, images: int, h: int, w: int):
    n = images * h * w
    wsb = int(N.lib().qfca_components_workspace_bytes(n))
    if wsb < 0:
        raise ValueError(f"{n} mask pixels: the labelling kernels take 1 .. 2^31 - 1")
    ws = empty((wsb,), torch.uint8)
    comp = empty((n,), torch.int32)
    cnt = zeros((1,), torch.int32)
    N.call("qfca_components", mask_u8.data_ptr(), images, h, w, ws.data_ptr(), wsb, None,
           comp.data_ptr(), cnt.data_ptr(), N.stream())
    return comp, int(cnt.item())


def _lerp(a, b, t):
    """NumPy's quantile interpolation (numpy/lib/_function_base_impl.py _lerp)."""
    diff_b_a = np.subtract(b, a)
    lerp = np.asanyarray(np.add(a, diff_b_a * t))
    np.subtract(b, diff_b_a * (1 - t), out=lerp, where=t >= 0.5, casting="unsafe",
                dtype=type(lerp.dtype))
    return lerp


def _quantiles(sorted_dev: torch.Tensor, dtype, qs: np.ndarray) -> np.ndarray:
    """np.quantile(pooled, qs) (method "linear") from the device-sorted scores:
    only the order statistics the interpolation reads come back to the host."""
    n = sorted_dev.numel()
    vi = (n - 1) * qs  # linear: virtual index (n - 1) q
    prev = np.floor(vi)
    nxt = prev + 1
    above = vi >= n - 1
    prev[above] = -1
    nxt[above] = -1
    below = vi < 0
    prev[below] = 0
    nxt[below] = 0
    prev_i = prev.astype(np.intp) % n
    next_i = nxt.astype(np.intp) % n
    idx = torch.from_numpy(np.concatenate([prev_i, next_i]).astype(np.int64)).to(sorted_dev.device)
    vals = sorted_dev.index_select(0, idx).double().cpu().numpy().astype(dtype)
    a, b = vals[:qs.size], vals[qs.size:]
    gamma = np.asanyarray(vi - prev.astype(np.intp).astype(np.float64))
    return _lerp(a, b, gamma)


def _pro_thresholds(p: _Pool) -> np.ndarray:
    """metrics.py:83-88 -- distinct quantile scores, descending."""
    qs = np.linspace(0.0, 1.0, PRO_MAX_THRESHOLDS)
    thr = np.unique(_quantiles(p.rank()[3], p.dtype, qs))
    return thr[::-1]


def _pro_curve(p: _Pool, thresholds: np.ndarray):
    """metrics.py:91-120 -- (fpr, pro) at the given thresholds (score >= t)."""
    thresholds = np.asarray(thresholds, dtype=np.float64)
    uniq, inv = np.unique(thresholds, return_inverse=True)
    m = uniq.size
    if m == 0:
        raise ValueError("no thresholds")
    if m > _MAX_KERNEL_THRESHOLDS:
        raise NotImplementedError(f"{m} distinct thresholds (the kernel takes <= "
                                  f"{_MAX_KERNEL_THRESHOLDS})")
    stream = N.stream()
    comp = empty((p.n,), torch.int32)
    ncomp = 0
    for off, k, h, w in p.groups:
        c, cnt = _components(p.labels[off:off + k * h * w], k, h, w)
        if ncomp:
            c = torch.where(c >= 0, c + ncomp, c)
        comp[off:off + k * h * w].copy_(c)
        ncomp += cnt
    if ncomp == 0:
        raise UndefinedMetricError("PRO needs at least one ground-truth region")
    thr_dev = torch.from_numpy(uniq).to(comp.device)
    normal = zeros((m + 1,), torch.int64)
    pro = zeros((m,), torch.float64)
    chunk = max(1, _HIST_CELLS // (m + 1))
    for lo in range(0, ncomp, chunk):
        hi = min(ncomp, lo + chunk)
        hist = zeros((hi - lo, m + 1), torch.int32)
        N.call("qfca_pro_histograms", p.scores.data_ptr(), comp.data_ptr(), p.n,
               thr_dev.data_ptr(), m, lo, hi, hist.data_ptr(),
               normal.data_ptr() if lo == 0 else None, stream)
        N.call("qfca_pro_accumulate", hist.data_ptr(), hi - lo, m, pro.data_ptr(), stream)
    nh = normal.cpu().numpy()
    n_norm = int(nh.sum())
    # count of normal pixels >= uniq[j] = sum of slots > j
    ge_norm = np.cumsum(nh[::-1])[::-1][1:]
    pro_u = pro.cpu().numpy()
    pro_t = pro_u[inv]
    pro_t = pro_t / ncomp
    if n_norm == 0:
        fpr = np.zeros(thresholds.size)
    else:
        fpr = ge_norm[inv] / n_norm
    return fpr, pro_t


def _integrate_to_limit(fpr: np.ndarray, pro: np.ndarray, limit: float) -> float:
    """metrics.py:125-146 -- trapezoid area of PRO(FPR) on [0, limit], normalised."""
    f = np.r_[0.0, fpr, 1.0]
    p = np.r_[0.0, pro, 1.0]
    area = 0.0
    for i in range(1, f.size):
        f0, f1 = f[i - 1], f[i]
        p0, p1 = p[i - 1], p[i]
        if f1 <= f0:
            continue
        hi = min(f1, limit)
        if hi <= f0:
            break
        p_hi = p0 + (p1 - p0) * (hi - f0) / (f1 - f0)
        area += 0.5 * (p0 + p_hi) * (hi - f0)
        if f1 >= limit:
            break
    return area / limit


def pro_at_fpr(samples: list[EvalSample], fpr_limit: float = PRO_FPR_LIMIT,
               thresholds: np.ndarray | None = None) -> float:
    """metrics.py:149-154 -- area under the per-region-overlap curve up to fpr_limit."""
    return _pool_pro(_Pool(samples), fpr_limit, thresholds)


def _pool_pro(p: _Pool, fpr_limit: float = PRO_FPR_LIMIT, thresholds=None) -> float:
    if thresholds is None:
        thresholds = _pro_thresholds(p)
    fpr, pro = _pro_curve(p, thresholds)
    return _integrate_to_limit(fpr, pro, fpr_limit)


@dataclass
class MetricReport:
    """metrics.py:182-206 -- per-class rows and their mean.  One device pool
    (and one sort) per class serves all four metrics."""

    per_class: dict = field(default_factory=dict)

    def add_class(self, name: str, samples: list[EvalSample]) -> dict:
        row: dict = {"n_images": len(samples)}
        p = _Pool(samples)
        for key, fn in (("pro", _pool_pro), ("auroc_s", _pool_auroc),
                        ("f1", _pool_f1), ("auroc_c", _pool_auroc_image)):
            try:
                row[key] = fn(p)
            except UndefinedMetricError:
                row[key] = None
        self.per_class[name] = row
        return row

    def to_dict(self) -> dict:
        out = dict(self.per_class)
        keys = ("pro", "auroc_s", "f1", "auroc_c")
        mean_row: dict = {}
        for k in keys:
            vals = [r[k] for r in self.per_class.values() if r.get(k) is not None]
            mean_row[k] = float(np.mean(vals)) if vals else None
        mean_row["n_images"] = sum(r["n_images"] for r in self.per_class.values())
        out["mean"] = mean_row
        return out
