"""End-to-end anomaly map on the GPU (drop-in for qfca.scoring).

Mirrors reference scoring.py:25-299: PipelineConfig / AnomalyMap dataclasses,
the step APIs (bin_error_maps, channel_error_maps, associate_errors,
aggregate_channels, smooth_scores, image_score_of, upsample_scores) and
detect(), plus the batched device entry point detect_batch().

Routing inside detect / detect_batch:
  * uniform sigma_p + median-quan + reflect / wrap (the default family):
    the fused path -- K1 min/max, K2 bins, K3 sort-free reference, K4 fused
    histogram / closed-form transport / association / channel sum, K5
    finalize (one C-ABI call, qfca_detect);
  * anything else (zero padding, non-integer references, finite sigma_p):
    the general path (csrc/generic.cu), the reference's unfused route.
Both run entirely on the GPU.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._dev import empty, is_torch, to_dev, to_host, zeros
from .features import (FeatureMap, _gauss_kernel, gaussian_blur, pca_fit_batch,
                       pca_residual_batch, sep_convolve_dev)
from .quantize import (BinIndexMap, HistogramField, Quantizer, ReferenceHistogram,
                       bins_dev, bins_dtype, minmax_dev, reference_weights_dev, sample_stride,
                       window_counts_dev)

__all__ = ["PipelineConfig", "AnomalyMap", "DetectResult", "detect", "detect_batch",
           "bin_error_maps", "channel_error_maps", "associate_errors", "aggregate_channels",
           "smooth_scores", "image_score_of", "upsample_scores", "fused_supported"]


@dataclass(frozen=True)
class PipelineConfig:
    """scoring.py:25-49 -- same fields, defaults and validation."""

    n_bins: int = 16
    patch_size: int = 9
    sigma_p: float = math.inf
    sigma_s: float = 1.0
    pca_components: int = 0
    reference_mode: str = "median-quan"
    sample_budget: int = 4096
    border_exclusion: int | None = None
    pad: str = "reflect"

    def __post_init__(self):
        if self.patch_size % 2 == 0 or self.patch_size < 1:
            raise ValueError("patch_size must be odd and >= 1")
        if self.n_bins < 1:
            raise ValueError("n_bins must be >= 1")
        if self.sigma_s < 0:
            raise ValueError("sigma_s must be >= 0")

    @property
    def border(self) -> int:
        if self.border_exclusion is None:
            return self.patch_size // 2
        return self.border_exclusion


@dataclass(frozen=True)
class AnomalyMap:
    scores: object  # (H, W) fp64
    image_score: float
    degenerate: bool = False


@dataclass(frozen=True)
class DetectResult:
    """Batched device result of detect_batch."""

    scores: torch.Tensor        # (B, h, w) fp64
    image_scores: torch.Tensor  # (B,) fp64
    used: torch.Tensor          # (B,) int32 non-degenerate channels
    nonfinite: torch.Tensor     # (1,) int32, != 0 if any input value was not finite

    @property
    def degenerate(self) -> torch.Tensor:
        return self.used == 0


def fused_supported(cfg: PipelineConfig) -> bool:
    return (math.isinf(cfg.sigma_p) and cfg.reference_mode == "median-quan"
            and cfg.pad in ("reflect", "wrap") and cfg.n_bins <= 65536
            and cfg.patch_size * cfg.patch_size <= 65535)


def _check_cfg(cfg: PipelineConfig):
    if cfg.pad not in N.PAD_CODES:
        raise ValueError(f"unknown pad mode {cfg.pad!r}")
    if cfg.reference_mode not in ("median-quan", "mean-quan", "quan-median", "quan-mean"):
        raise ValueError(f"unknown reference mode {cfg.reference_mode!r}")
    if cfg.sample_budget < 1:
        raise ValueError("sample_budget must be >= 1")


# ------------------------------------------------------------ fused path
_WS_CACHE: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    # one cached workspace per (device, stream): calls on different streams may overlap
    key = (device.index if device.index is not None else torch.cuda.current_device(),
           torch.cuda.current_stream(device).cuda_stream)
    ws = _WS_CACHE.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty((max(nbytes, 1),), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = ws
    return ws


def _qcfg(cfg: PipelineConfig, groups: int = 0) -> N.QfcaConfig:
    return N.QfcaConfig(cfg.n_bins, cfg.patch_size, N.PAD_CODES[cfg.pad], cfg.sample_budget,
                        cfg.border, groups, float(cfg.sigma_s))


def _fused_detect(x: torch.Tensor, cfg: PipelineConfig, groups: int = 0,
                  out: DetectResult | None = None, events=None) -> DetectResult:
    b, c, h, w = x.shape
    qc = _qcfg(cfg, groups)
    L = N.lib()
    nbytes = L.qfca_detect_workspace_bytes(b, c, h, w, ctypes.byref(qc))
    if nbytes < 0:
        raise NotImplementedError("configuration not supported by the fused kernel")
    ws = _workspace(nbytes, x.device)
    if out is None:
        out = DetectResult(scores=empty((b, h, w), torch.float64),
                           image_scores=empty((b,), torch.float64),
                           used=empty((b,), torch.int32), nonfinite=zeros((1,), torch.int32))
    ev = None
    if events is not None:
        for e in events:  # torch creates the cudaEvent handle lazily, on first record
            if not e.cuda_event:
                e.record()
        ev = (ctypes.c_void_p * 2)(events[0].cuda_event, events[1].cuda_event)
    N.check(L.qfca_detect_ex(x.data_ptr(), b, c, h, w, ctypes.byref(qc), ws.data_ptr(), nbytes,
                             out.scores.data_ptr(), out.image_scores.data_ptr(),
                             out.used.data_ptr(), out.nonfinite.data_ptr(), ev, N.stream()),
            "qfca_detect")
    return out


# ------------------------------------------------------------ general path
def _centers_dev(lo: torch.Tensor, hi: torch.Tensor, n_bins: int) -> torch.Tensor:
    """quantize.py:29-38 per plane, fp64, NumPy's operation order."""
    lo64, hi64 = lo.to(torch.float64), hi.to(torch.float64)
    width = torch.where(hi64 > lo64, (hi64 - lo64) / n_bins, torch.ones_like(lo64))
    ar = torch.arange(n_bins, dtype=torch.float64, device=lo.device) + 0.5
    return lo64[:, None] + ar[None, :] * width[:, None]


def _smooth_taps(cfg: PipelineConfig):
    t = cfg.patch_size
    if math.isinf(cfg.sigma_p):
        return np.ones(t, np.float64), 1.0 / float(t * t)
    r = t // 2
    xx = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-0.5 * (xx / cfg.sigma_p) ** 2)
    k /= k.sum()
    return k, 1.0


def _reference_weights_dev(x, bins, lo, hi, degen, cfg: PipelineConfig) -> torch.Tensor:
    """select_reference (quantize.py:150-200) weights (planes, N) fp64 on the device."""
    b, c, h, w = x.shape
    return reference_weights_dev(x.reshape(b * c, h, w), bins, lo, hi, b * c, h, w, cfg.n_bins,
                                 cfg.patch_size, cfg.pad, cfg.sample_budget, cfg.reference_mode)


def _general_partial(x: torch.Tensor, cfg: PipelineConfig, events=None):
    """The reference's unfused route up to the channel sum (scoring.py:251-281,
    the non-uniform branch 274-280 and bin_error_maps / associate_errors):
    returns (acc (B, h*w) fp64 channel sums, used (B,) int32, non-finite flag)."""
    b, c, h, w = x.shape
    hw = h * w
    planes = b * c
    n, t = cfg.n_bins, cfg.patch_size
    s = N.stream()
    lo, hi, flag = minmax_dev(x, planes, hw)
    degen = ~(hi > lo)
    bins = bins_dev(x, lo, hi, planes, hw, n)
    refw = _reference_weights_dev(x, bins, lo, hi, degen, cfg)
    centers = _centers_dev(lo, hi, n)
    if events is not None:
        events[0].record()
    taps, post = _smooth_taps(cfg)
    skip = degen.to(torch.uint8)
    acc = zeros((b, hw), torch.float64)
    used = zeros((b,), torch.int32)
    per_plane = n * hw * (2 + 2 + 8 + 8) + hw * 8
    chunk = max(1, min(c, (1 << 30) // max(per_plane, 1)))
    for i in range(b):
        for c0 in range(0, c, chunk):
            c1 = min(c, c0 + chunk)
            p0, p1 = i * c + c0, i * c + c1
            np_ = p1 - p0
            bsl = bins[p0 * hw:p1 * hw]
            counts = window_counts_dev(bsl, np_, h, w, n, t, cfg.pad, kind=torch.int16)
            err = empty((np_, n, hw), torch.float64)
            N.call("qfca_mismatch_pixels", counts.data_ptr(), np_, hw, n,
                   refw[p0:p1].contiguous().data_ptr(), centers[p0:p1].contiguous().data_ptr(),
                   skip[p0:p1].data_ptr(), err.data_ptr(), s)
            del counts
            tmp = empty((np_, n, hw), torch.float64)
            score = empty((np_, hw), torch.float64)
            N.call("qfca_smooth_gather", err.data_ptr(), bsl.data_ptr(), bsl.element_size(),
                   np_, h, w, n, t, N.PAD_CODES[cfg.pad], taps.ctypes.data_as(N._P),
                   float(post), tmp.data_ptr(), score.data_ptr(), s)
            del err, tmp
            N.call("qfca_channel_sum", score.data_ptr(), 1, np_, hw, skip[p0:p1].data_ptr(),
                   1, acc[i].data_ptr(), used[i:i + 1].data_ptr(), s)
    if events is not None:
        events[1].record()
    return acc, used, flag


def _finalize_dev(acc: torch.Tensor, used: torch.Tensor, cfg: PipelineConfig, h: int, w: int):
    """scoring.py:284-291: acc / used (zeros when all degenerate), smooth_scores,
    image_score_of, on (B, h*w) device sums -> (scores (B, h, w), image scores (B,))."""
    b = acc.shape[0]
    s = N.stream()
    agg = empty((b, h * w), torch.float64)
    N.call("qfca_divide_used", acc.data_ptr(), b, h * w, used.data_ptr(), agg.data_ptr(), s)
    agg = agg.reshape(b, h, w)
    final = sep_convolve_dev(agg, _gauss_kernel(cfg.sigma_s), cfg.pad) if cfg.sigma_s > 0 \
        else agg
    img = empty((b,), torch.float64)
    N.call("qfca_image_score", final.data_ptr(), b, h, w, cfg.border, img.data_ptr(), s)
    return final, img


def _general_detect(x: torch.Tensor, cfg: PipelineConfig, events=None) -> DetectResult:
    b, c, h, w = x.shape
    acc, used, flag = _general_partial(x, cfg, events)
    final, img = _finalize_dev(acc, used, cfg, h, w)
    return DetectResult(scores=final, image_scores=img, used=used, nonfinite=flag)


# ------------------------------------------------------------ public API
_MAX_ELEMS = (1 << 31) - 1  # features per detect_batch launch (32-bit offsets)


def detect_batch(values: torch.Tensor, cfg: PipelineConfig | None = None,
                 groups: int = 0, out: DetectResult | None = None,
                 score_events=None) -> DetectResult:
    """Batched detect on device features (B, C, h, w) float32 -> DetectResult.

    No host synchronisation: degenerate / non-finite flags stay on the device.
    ``score_events`` = (start, end) torch.cuda.Event pair recorded around the
    fused scoring kernel (fused path only).
    """
    cfg = cfg or PipelineConfig()
    _check_cfg(cfg)
    if values.dim() != 4:
        raise ValueError("values must be (B, C, H, W)")
    x = to_dev(values)
    if cfg.pca_components > 0:
        k = min(cfg.pca_components, x.shape[1])
        mean, comps, _ = pca_fit_batch(x, k)
        x = pca_residual_batch(x, mean, comps)
    b = x.shape[0]
    per_image = int(np.prod(x.shape[1:]))
    if b > 1 and b * per_image > _MAX_ELEMS and score_events is None:
        # keep every launch's element count inside 32-bit plane offsets
        step = max(1, _MAX_ELEMS // per_image)
        parts = [detect_batch(x[i:i + step], cfg, groups) for i in range(0, b, step)]
        return DetectResult(scores=torch.cat([p.scores for p in parts]),
                            image_scores=torch.cat([p.image_scores for p in parts]),
                            used=torch.cat([p.used for p in parts]),
                            nonfinite=torch.stack([p.nonfinite for p in parts]).amax(0))
    route = _route(x, cfg)
    if route == "fused":
        return _fused_detect(x, cfg, groups, out, score_events)
    if route == "wide":
        return _wide_detect(x, cfg, events=score_events)
    return _general_detect(x, cfg, events=score_events)


def _wide_detect(x: torch.Tensor, cfg: PipelineConfig, events=None) -> DetectResult:
    """Feature planes wider than the fused kernels' 128 columns (an 8192^2
    texture: 1024^2 per channel): each image through the tiled fused path of
    sharding.py (one rank holding every channel), then the channel mean,
    Gaussian and image score as in _fused_detect (scoring.py:258-299)."""
    from .sharding import _channel_partial
    b, c, h, w = x.shape
    out = DetectResult(scores=empty((b, h, w), torch.float64),
                       image_scores=empty((b,), torch.float64),
                       used=empty((b,), torch.int32), nonfinite=zeros((1,), torch.int32))
    taps = _gauss_kernel(cfg.sigma_s) if cfg.sigma_s > 0 else None
    if events is not None:
        events[0].record()
    for i in range(b):
        acc, used, flag = _channel_partial(x[i], cfg)
        out.nonfinite.bitwise_or_(flag)
        out.used[i:i + 1] = used
        agg = acc / used.clamp(min=1).to(torch.float64)  # all degenerate: zeros
        final = sep_convolve_dev(agg[None].contiguous(), taps, cfg.pad)[0] \
            if taps is not None else agg
        out.scores[i] = final
        N.call("qfca_image_score", out.scores[i].data_ptr(), 1, h, w, cfg.border,
               out.image_scores[i:i + 1].data_ptr(), N.stream())
    if events is not None:
        events[1].record()
    return out


def _route(x: torch.Tensor, cfg: PipelineConfig) -> str:
    """The path detect / detect_batch take for device features x (B, C, h, w)."""
    if not fused_supported(cfg):
        return "general"
    from .sharding import wide_supported
    if wide_supported(cfg, x.shape[2], x.shape[3], x.shape[1]):
        return "wide"
    L = N.lib()
    qc = _qcfg(cfg)
    if L.qfca_detect_workspace_bytes(x.shape[0], x.shape[1], x.shape[2], x.shape[3],
                                     ctypes.byref(qc)) < 0:
        return "general"  # shapes the fused kernels do not take (e.g. very wide planes)
    return "fused"


def detect(f: FeatureMap, cfg: PipelineConfig | None = None,
           timings: dict | None = None) -> AnomalyMap:
    """scoring.py:235-299: full anomaly-map pipeline on one feature map.

    ``timings`` receives the reference's four keys (scoring.py:294-298), timed
    on the device with CUDA events: ``pca_ms`` (pca_fit + pca_residual),
    ``quantize_ms`` (fit_quantizer + bin_indices + select_reference; on the fused
    path the median-quan selection may run inside the scoring kernel, then it
    is counted in transport_ms), ``transport_ms`` (histograms, transport,
    association, channel sum) and ``postprocess_ms`` (channel mean, smoothing,
    image score).
    """
    cfg = cfg or PipelineConfig()
    _check_cfg(cfg)
    like = is_torch(f.values)
    E = (lambda: torch.cuda.Event(enable_timing=True)) if timings is not None else None
    ev = [E() for _ in range(5)] if E else None
    x = to_dev(f.values)[None]
    if ev:
        ev[0].record()
    if cfg.pca_components > 0:
        k = min(cfg.pca_components, x.shape[1])
        mean, comps, _ = pca_fit_batch(x, k)
        x = pca_residual_batch(x, mean, comps)
    if ev:
        ev[1].record()
    route = _route(x, cfg)
    if route == "fused":
        res = _fused_detect(x, cfg, events=(ev[2], ev[3]) if ev else None)
    elif route == "wide":
        res = _wide_detect(x, cfg, events=(ev[2], ev[3]) if ev else None)
    else:
        res = _general_detect(x, cfg, events=(ev[2], ev[3]) if ev else None)
    if ev:
        ev[4].record()
        ev[4].synchronize()
        timings["pca_ms"] = ev[0].elapsed_time(ev[1])
        timings["quantize_ms"] = ev[1].elapsed_time(ev[2])
        timings["transport_ms"] = ev[2].elapsed_time(ev[3])
        timings["postprocess_ms"] = ev[3].elapsed_time(ev[4])
    used = int(res.used[0])
    degenerate = used == 0
    if degenerate:
        warnings.warn("all channels degenerate; anomaly map is all zeros")
    scores = to_host(res.scores[0], like)
    return AnomalyMap(scores=scores, image_score=float(res.image_scores[0]),
                      degenerate=degenerate)


def channel_error_maps(counts, ref_w, centers):
    """scoring.py:75-85: (N, H, W) errors of one channel's histogram field."""
    like = is_torch(counts)
    cnt = to_dev(counts, torch.float32)
    n, h, w = cnt.shape
    pb = cnt.permute(1, 2, 0).reshape(-1, n).to(torch.float64).contiguous()
    from .transport import mismatch_batch_dev
    e = mismatch_batch_dev(pb, to_dev(ref_w, torch.float64), to_dev(centers, torch.float64))
    return to_host(e.reshape(h, w, n).permute(2, 0, 1).contiguous(), like)


def bin_error_maps(hf: HistogramField, ref: ReferenceHistogram, q: Quantizer):
    """scoring.py:59-72: (C, N, H, W) per-bin mismatch scores."""
    like = is_torch(hf.counts)
    counts = to_dev(hf.counts, torch.float32)
    c, n, h, w = counts.shape
    cnt16 = counts.round().to(torch.int16).contiguous()
    lo = to_dev(q.lo, torch.float64)
    hi = to_dev(q.hi, torch.float64)
    centers = torch.stack([torch.from_numpy(q.centers(i)) for i in range(c)]).to(lo.device)
    skip = to_dev(np.asarray(q.degenerate.cpu() if is_torch(q.degenerate) else q.degenerate,
                             np.uint8), torch.uint8)
    err = empty((c, n, h * w), torch.float64)
    N.call("qfca_mismatch_pixels", cnt16.data_ptr(), c, h * w, n,
           to_dev(ref.weights, torch.float64).data_ptr(), centers.contiguous().data_ptr(),
           skip.data_ptr(), err.data_ptr(), N.stream())
    del lo, hi
    return to_host(err.reshape(c, n, h, w), like)


def associate_errors(err, bins: BinIndexMap, cfg: PipelineConfig):
    """scoring.py:101-112: smooth each channel's error planes, own-bin gather."""
    like = is_torch(err)
    e = to_dev(err, torch.float64)
    c, n, h, w = e.shape
    idx = to_dev(bins.indices, torch.int32)
    taps, post = _smooth_taps(cfg)
    tmp = empty((c, n, h * w), torch.float64)
    out = empty((c, h, w), torch.float64)
    N.call("qfca_smooth_gather", e.data_ptr(), idx.data_ptr(), 4, c, h, w, n, cfg.patch_size,
           N.PAD_CODES[cfg.pad], taps.ctypes.data_as(N._P), float(post), tmp.data_ptr(),
           out.data_ptr(), N.stream())
    return to_host(out, like)


def aggregate_channels(scores, skip=None):
    """scoring.py:115-130: mean over non-skipped channels (fixed order)."""
    like = is_torch(scores)
    s = to_dev(scores, torch.float64)
    if s.shape[0] < 1:
        raise ValueError("need at least one channel")
    c = s.shape[0]
    hw = int(np.prod(s.shape[1:]))
    if skip is None:
        sk = zeros((c,), torch.uint8)
    else:
        sk = to_dev(np.asarray(skip.cpu() if is_torch(skip) else skip, np.uint8), torch.uint8)
    acc = empty((1, hw), torch.float64)
    used = empty((1,), torch.int32)
    N.call("qfca_channel_sum", s.contiguous().data_ptr(), 1, c, hw, sk.data_ptr(), 0,
           acc.data_ptr(), used.data_ptr(), N.stream())
    if int(used[0]) == 0:
        warnings.warn("all channels degenerate; anomaly map is all zeros")
        return to_host(zeros(tuple(s.shape[1:]), torch.float64), like), True
    agg = empty((1, hw), torch.float64)
    N.call("qfca_divide_used", acc.data_ptr(), 1, hw, used.data_ptr(), agg.data_ptr(),
           N.stream())
    return to_host(agg.reshape(s.shape[1:]), like), False


def smooth_scores(score_map, sigma_s: float, pad: str = "reflect"):
    """scoring.py:133-138."""
    if sigma_s == 0:
        return score_map.to(torch.float64) if is_torch(score_map) else np.asarray(
            score_map, dtype=np.float64)
    return gaussian_blur(score_map, sigma_s, pad=pad)


def image_score_of(scores, border: int) -> float:
    """scoring.py:141-146: max over pixels at least ``border`` from the edge."""
    s = to_dev(scores, torch.float64)
    h, w = s.shape
    out = empty((1,), torch.float64)
    N.call("qfca_image_score", s.data_ptr(), 1, h, w, int(border), out.data_ptr(), N.stream())
    return float(out[0])


def upsample_scores(scores, out_h: int, out_w: int):
    """scoring.py:149-152: bilinear (half-pixel) resize, float32-rounded, fp64 out."""
    like = is_torch(scores)
    s = to_dev(scores, torch.float64)
    h, w = s.shape
    out = empty((out_h, out_w), torch.float32)
    N.call("qfca_upsample", s.data_ptr(), 1, h, w, out_h, out_w, out.data_ptr(), N.stream())
    return to_host(out.to(torch.float64), like)


def upsample_batch(scores: torch.Tensor, out_h: int, out_w: int,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """(B, h, w) fp64 device maps -> (B, out_h, out_w) float32 device maps
    (upsample_scores per map, scoring.py:149-152), into ``out`` when given."""
    b, h, w = scores.shape
    if out is None:
        out = empty((b, out_h, out_w), torch.float32)
    elif (tuple(out.shape) != (b, out_h, out_w) or out.dtype != torch.float32
          or not out.is_contiguous()):
        raise ValueError("out must be a contiguous (B, out_h, out_w) float32 tensor")
    N.call("qfca_upsample", scores.contiguous().data_ptr(), b, h, w, out_h, out_w,
           out.data_ptr(), N.stream())
    return out


def upsample_batch_into(scores: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    return upsample_batch(scores, out.shape[1], out.shape[2], out)
