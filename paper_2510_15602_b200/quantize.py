"""Per-channel quantization, window histograms and reference selection (GPU).

Mirrors qfca.quantize (reference quantize.py:1-200): same names, dataclasses,
validation and error messages.  fit_quantizer / bin_indices run K1/K2
(csrc/quantize.cu), patch_histograms the window-count kernels
(csrc/generic.cu), select_reference the sort-free order-statistic kernel K3
(csrc/reference.cu) -- bit-exact against the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._dev import empty, is_torch, to_dev, to_host, zeros

REFERENCE_MODES = ("median-quan", "mean-quan", "quan-median", "quan-mean")

__all__ = ["Quantizer", "BinIndexMap", "HistogramField", "ReferenceHistogram",
           "REFERENCE_MODES", "fit_quantizer", "bin_indices", "patch_histograms",
           "select_reference", "sample_stride", "bins_dtype"]


@dataclass(frozen=True)
class Quantizer:
    """Equally-spaced bins per channel over [lo, hi] (quantize.py:16-38)."""

    lo: object  # (C,) fp64
    hi: object  # (C,) fp64
    n_bins: int
    degenerate: object  # (C,) bool

    @property
    def n_channels(self) -> int:
        return self.lo.shape[0]

    def centers(self, c: int) -> np.ndarray:
        lo, hi = float(self.lo[c]), float(self.hi[c])
        width = (hi - lo) / self.n_bins if hi > lo else 1.0
        return lo + (np.arange(self.n_bins) + 0.5) * width


@dataclass(frozen=True)
class BinIndexMap:
    indices: object  # (C, H, W) int32 in [0, N)
    n_bins: int


@dataclass(frozen=True)
class HistogramField:
    counts: object  # (C, N, H, W) float32
    patch_size: int


@dataclass(frozen=True)
class ReferenceHistogram:
    weights: object  # (C, N) fp64, mass T^2 per channel
    patch_size: int


def bins_dtype(n_bins: int):
    """Compact on-device bin storage: uint8 up to 256 bins, else int16 bits."""
    return (torch.uint8, 1) if n_bins <= 256 else (torch.int16, 2)


def sample_stride(h: int, w: int, budget: int) -> int:
    """quantize.py:109-116."""
    return int(N.lib().qfca_sample_stride(h, w, budget))


# ---------------------------------------------------------------- device ops
def minmax_dev(x: torch.Tensor, planes: int, plane_len: int):
    lo = empty((planes,), torch.float32)
    hi = empty((planes,), torch.float32)
    flag = zeros((1,), torch.int32)
    N.call("qfca_fit_quantizer", x.data_ptr(), planes, plane_len, lo.data_ptr(), hi.data_ptr(),
           flag.data_ptr(), N.stream())
    return lo, hi, flag


def bins_dev(x: torch.Tensor, lo: torch.Tensor, hi: torch.Tensor, planes: int, plane_len: int,
             n_bins: int, dtype=None) -> torch.Tensor:
    if dtype is None:
        dtype, nb = bins_dtype(n_bins)
    else:
        nb = {torch.uint8: 1, torch.int16: 2, torch.int32: 4}[dtype]
    out = empty((planes * plane_len,), dtype)
    N.call("qfca_bin_indices", x.data_ptr(), planes, plane_len, lo.data_ptr(), hi.data_ptr(),
           n_bins, out.data_ptr(), nb, N.stream())
    return out


def quantize_dev(x: torch.Tensor, planes: int, plane_len: int, n_bins: int):
    """minmax_dev + bins_dev in one C-ABI call (qfca_quantize: one pass over x
    when a plane fits in shared memory).  Returns (lo, hi, flag, bins)."""
    dtype, nb = bins_dtype(n_bins)
    lo = empty((planes,), torch.float32)
    hi = empty((planes,), torch.float32)
    flag = zeros((1,), torch.int32)
    out = empty((planes * plane_len,), dtype)
    N.call("qfca_quantize", x.data_ptr(), planes, plane_len, n_bins, lo.data_ptr(),
           hi.data_ptr(), flag.data_ptr(), out.data_ptr(), nb, N.stream())
    return lo, hi, flag, out


def reference_stats_dev(bins: torch.Tensor, lo: torch.Tensor, hi: torch.Tensor, planes: int,
                        h: int, w: int, n_bins: int, t: int, pad: str, budget: int,
                        mode: str) -> torch.Tensor:
    stats = empty((planes, n_bins), torch.int32)
    nb = bins.element_size()
    N.call("qfca_select_reference", bins.data_ptr(), nb, lo.data_ptr(), hi.data_ptr(), planes,
           h, w, n_bins, t, N.PAD_CODES[pad], budget, N.REF_MODE_CODES[mode],
           stats.data_ptr(), N.stream())
    return stats


def window_counts_dev(bins: torch.Tensor, planes: int, h: int, w: int, n_bins: int, t: int,
                      pad: str, kind=torch.float32) -> torch.Tensor:
    scratch = empty((planes * n_bins * h * w,), torch.int16)
    out = empty((planes, n_bins, h, w), kind)
    N.call("qfca_window_counts", bins.data_ptr(), bins.element_size(), planes, h, w, n_bins, t,
           N.PAD_CODES[pad], scratch.data_ptr(), out.data_ptr(),
           0 if kind == torch.float32 else 1, N.stream())
    return out


def _qtensors(q: Quantizer):
    lo = to_dev(q.lo, torch.float64).to(torch.float32)
    hi = to_dev(q.hi, torch.float64).to(torch.float32)
    return lo, hi


# ---------------------------------------------------------------- public API
def fit_quantizer(values, n_bins: int) -> Quantizer:
    """quantize.py:61-68 -- per-channel min/max range."""
    if n_bins < 1:
        raise ValueError(f"n_bins must be >= 1, got {n_bins}")
    x = to_dev(values)
    c = x.shape[0]
    lo, hi, _ = minmax_dev(x, c, x.numel() // c)
    lo64, hi64 = lo.to(torch.float64), hi.to(torch.float64)
    t = is_torch(values)
    return Quantizer(lo=to_host(lo64, t), hi=to_host(hi64, t), n_bins=n_bins,
                     degenerate=to_host(hi64 <= lo64, t))


def bin_indices(values, q: Quantizer) -> BinIndexMap:
    """quantize.py:71-82 -- clamp(floor((v - lo) * N / (hi - lo)), 0, N - 1)."""
    x = to_dev(values)
    if x.shape[0] != q.n_channels:
        raise ValueError("channel count mismatch with quantizer")
    # the kernel evaluates the rule from the float32 range; a Quantizer built
    # elsewhere must hold float32-representable bounds (fit_quantizer's do)
    lo, hi = _qtensors(q)
    c = x.shape[0]
    b = bins_dev(x, lo, hi, c, x.numel() // c, q.n_bins, torch.int32).reshape(x.shape)
    return BinIndexMap(indices=to_host(b, is_torch(values)), n_bins=q.n_bins)


def patch_histograms(b: BinIndexMap, patch_size: int, pad: str = "reflect") -> HistogramField:
    """quantize.py:92-106 -- window counts of every location (float32)."""
    if patch_size % 2 == 0:
        raise ValueError(f"patch size must be odd, got {patch_size}")
    if pad not in N.PAD_CODES:
        raise ValueError(f"unknown pad mode {pad!r}")
    idx = to_dev(b.indices, torch.int32)
    c, h, w = idx.shape
    counts = window_counts_dev(idx, c, h, w, b.n_bins, patch_size, pad)
    return HistogramField(counts=to_host(counts, is_torch(b.indices)), patch_size=patch_size)


def reference_weights_dev(x: torch.Tensor, bins: torch.Tensor | None, lo: torch.Tensor,
                          hi: torch.Tensor, planes: int, h: int, w: int, n_bins: int, t: int,
                          pad: str, budget: int, mode: str) -> torch.Tensor:
    """select_reference weights (planes, n_bins) fp64 of any mode on the device
    (quantize.py:150-200; csrc/refmodes.cu), bit-identical to the reference.
    mean-quan reads the float32 values x, the other modes the bins."""
    L = N.lib()
    code = N.REF_MODE_CODES[mode]
    nbytes = L.qfca_reference_weights_workspace_bytes(planes, h, w, n_bins, t, budget, code)
    if nbytes < 0:
        raise ValueError("unsupported reference configuration")
    ws = empty((max(int(nbytes), 1),), torch.uint8)
    out = empty((planes, n_bins), torch.float64)
    N.call("qfca_reference_weights", x.data_ptr() if x is not None else None,
           bins.data_ptr() if bins is not None else None,
           bins.element_size() if bins is not None else 1, lo.data_ptr(), hi.data_ptr(), planes,
           h, w, n_bins, t, N.PAD_CODES[pad], budget, code, ws.data_ptr(), nbytes,
           out.data_ptr(), N.stream())
    return out


def select_reference(values, q: Quantizer, patch_size: int, mode: str = "median-quan",
                     sample_budget: int = 4096, pad: str = "reflect") -> ReferenceHistogram:
    """quantize.py:150-200 -- global per-channel reference histogram."""
    if mode not in REFERENCE_MODES:
        raise ValueError(f"unknown reference mode {mode!r}")
    if sample_budget < 1:
        raise ValueError("sample_budget must be >= 1")
    if patch_size % 2 == 0 or patch_size < 1:
        raise ValueError(f"patch size must be odd, got {patch_size}")
    if pad not in N.PAD_CODES:
        raise ValueError(f"unknown pad mode {pad!r}")
    x = to_dev(values)
    c, h, w = x.shape
    lo, hi = _qtensors(q)
    b = None if mode == "mean-quan" else bins_dev(x, lo, hi, c, h * w, q.n_bins)
    weights = reference_weights_dev(x, b, lo, hi, c, h, w, q.n_bins, patch_size, pad,
                                    sample_budget, mode)
    weights = to_host(weights, is_torch(values))
    return ReferenceHistogram(weights=weights, patch_size=patch_size)
