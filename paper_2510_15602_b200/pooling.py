"""Box pooling with summed-area tables on the GPU (drop-in for qfca.pooling,
reference pooling.py:1-172).

The scoring path never materialises box filters (the fused kernel slides its
window counts on chip); this module is the reference's public pooling API with
the reference's exact arithmetic, every step a kernel of csrc/pooling.cu:

* ``pad_plane``          pooling.py:20-38 (np.pad modes; reflect falls back to
                         'edge' on both axes when either axis has length 1);
* ``build_sat``          pooling.py:56-64, fp64 cumsum down rows then columns,
                         sequential scans (bit-identical to NumPy);
* ``box_sum``            pooling.py:71-94 (same validation and errors);
* ``box_average``        pooling.py:120-122 via the SAT of build_sat;
* ``box_average_stack``  pooling.py:125-158 (np.pad per axis: a length-1 axis
                         reflects onto itself, the other axis still reflects);
* ``naive_box_average``  pooling.py:161-172 (direct shifted sums, the reference's check).

Inputs are NumPy arrays (results come back as NumPy) or CUDA tensors (results
stay on the device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._dev import empty, is_torch, require_cuda, to_dev, to_host

PAD_MODES = ("zero", "reflect", "wrap")
_ZERO, _REFLECT, _WRAP, _EDGE = 0, 1, 2, 3

__all__ = ["PAD_MODES", "SummedAreaTable", "pad_plane", "build_sat", "box_sum", "box_average",
           "box_average_stack", "naive_box_average"]

_DTYPE_CODES = {torch.float32: 0, torch.float64: 1, torch.uint8: 2, torch.int32: 3,
                torch.int64: 4, torch.int16: 5, torch.bool: 7}


def _check_kernel(k: int) -> int:
    """pooling.py:14-17."""
    if k < 1 or k % 2 == 0:
        raise ValueError(f"kernel size must be odd and >= 1, got {k}")
    return k // 2


def _as_dev(x) -> torch.Tensor:
    dev = require_cuda()
    if is_torch(x):
        return x.to(dev).contiguous()
    a = np.ascontiguousarray(np.asarray(x))
    if a.dtype == np.uint16:
        a = a.astype(np.int32)
    return torch.from_numpy(a).to(dev)


def _dtype_code(t: torch.Tensor) -> tuple[torch.Tensor, int]:
    if t.dtype in _DTYPE_CODES:
        return t, _DTYPE_CODES[t.dtype]
    return t.to(torch.float64), 1


def _pad_plane_modes(pad: str, h: int, w: int) -> tuple[int, int]:
    """Per-axis modes of pad_plane (pooling.py:29-38)."""
    if pad == "zero":
        return _ZERO, _ZERO
    if pad == "reflect":
        if h > 1 and w > 1:
            return _REFLECT, _REFLECT
        return _EDGE, _EDGE  # pooling.py:33-35
    if pad == "wrap":
        return _WRAP, _WRAP
    raise ValueError(f"unknown pad mode {pad!r}")


def _np_pad_modes(pad: str) -> tuple[int, int]:
    """Per-axis modes of np.pad(mode=pad) as box_average_stack uses it
    (pooling.py:143-144): a length-1 axis reflects onto its single element."""
    return {"reflect": (_REFLECT, _REFLECT), "wrap": (_WRAP, _WRAP)}[pad]


def pad_plane(plane, margin: int, pad: str):
    """pooling.py:20-38: pad a 2-D plane by ``margin`` on every side."""
    if margin == 0:
        return plane
    x = _as_dev(plane)
    if x.dim() != 2:
        raise ValueError("plane must be 2-D")
    h, w = x.shape
    mr, mc = _pad_plane_modes(pad, h, w)
    out = torch.empty((h + 2 * margin, w + 2 * margin), dtype=x.dtype, device=x.device)
    N.call("qfca_pad_planes", x.data_ptr(), 1, h, w, margin, mr, mc, x.element_size(),
           out.data_ptr(), N.stream())
    return to_host(out, is_torch(plane))


@dataclass(frozen=True)
class SummedAreaTable:
    """pooling.py:41-53: integral image with a zero first row / column."""

    height: int
    width: int
    margin: int
    cumsum: object  # (H + 2*margin + 1, W + 2*margin + 1) float64


def _sat_dev(x: torch.Tensor, margin: int, mr: int, mc: int) -> torch.Tensor:
    """(P, h, w) device planes -> (P, H + 1, W + 1) fp64 SATs."""
    x, code = _dtype_code(x)
    p, h, w = x.shape
    cs = empty((p, h + 2 * margin + 1, w + 2 * margin + 1), torch.float64)
    N.call("qfca_build_sat", x.data_ptr(), code, p, h, w, margin, mr, mc, cs.data_ptr(),
           N.stream())
    return cs


def build_sat(plane, margin: int = 0, pad: str = "zero") -> SummedAreaTable:
    """pooling.py:56-64: integral image of ``plane`` (optionally pre-padded)."""
    x = _as_dev(plane)
    if x.dim() != 2:
        raise ValueError("plane must be 2-D")
    h, w = x.shape
    if margin == 0:
        mr = mc = _ZERO  # no padding: the mode is never consulted
    else:
        mr, mc = _pad_plane_modes(pad, h, w)
    cs = _sat_dev(x[None], margin, mr, mc)[0]
    return SummedAreaTable(height=h, width=w, margin=margin,
                           cumsum=to_host(cs, is_torch(plane)))


def box_sum(sat: SummedAreaTable, cx: int, cy: int, k: int, pad: str = "zero") -> float:
    """pooling.py:71-94: sum over the k x k window centred at row cx, col cy."""
    r = _check_kernel(k)
    if not (0 <= cx < sat.height and 0 <= cy < sat.width):
        raise ValueError(f"center ({cx}, {cy}) out of bounds")
    m = sat.margin
    if pad == "zero":
        r0, r1 = max(cx - r, 0) + m, min(cx + r + 1, sat.height) + m
        c0, c1 = max(cy - r, 0) + m, min(cy + r + 1, sat.width) + m
    elif pad in ("reflect", "wrap"):
        if m < r:
            raise ValueError(f"SAT margin {m} too small for kernel {k}")
        r0, r1 = cx - r + m, cx + r + 1 + m
        c0, c1 = cy - r + m, cy + r + 1 + m
    else:
        raise ValueError(f"unknown pad mode {pad!r}")
    cs = to_dev(sat.cumsum, torch.float64)
    rect = torch.tensor([[r0, r1, c0, c1]], dtype=torch.int32, device=cs.device)
    out = empty((1,), torch.float64)
    N.call("qfca_sat_rects", cs.data_ptr(), cs.shape[-1], rect.data_ptr(), 1, out.data_ptr(),
           N.stream())
    return float(out[0])


def _box_from_sat(x: torch.Tensor, k: int, pad: str, modes) -> torch.Tensor:
    r = _check_kernel(k)
    p, h, w = x.shape
    if pad == "zero":
        cs = _sat_dev(x, 0, _ZERO, _ZERO)
        clamp = 1
    else:
        cs = _sat_dev(x, r, *modes)
        clamp = 0
    out = empty((p, h, w), torch.float64)
    N.call("qfca_sat_box", cs.data_ptr(), p, h, w, k, clamp, float(k * k), out.data_ptr(),
           N.stream())
    return out


def box_average(plane, k: int, pad: str = "reflect"):
    """pooling.py:120-122: k x k local average, O(H*W) regardless of k."""
    x = _as_dev(plane)
    if x.dim() != 2:
        raise ValueError("plane must be 2-D")
    h, w = x.shape
    # via build_sat -> pad_plane, which is not consulted for a zero margin
    modes = _pad_plane_modes(pad, h, w) if pad != "zero" and k > 1 else (_ZERO, _ZERO)
    out = _box_from_sat(x[None], k, "zero" if pad != "zero" and k == 1 else pad, modes)[0]
    return to_host(out, is_torch(plane))


def box_average_stack(planes, k: int, pad: str = "reflect"):
    """pooling.py:125-158: batched box_average over a (B, H, W) stack."""
    _check_kernel(k)
    if pad not in PAD_MODES:
        raise KeyError(pad)  # the reference's dict lookup (pooling.py:143)
    x = _as_dev(planes)
    if x.dim() != 3:
        raise ValueError("planes must be (B, H, W)")
    modes = _np_pad_modes(pad) if pad != "zero" else (_ZERO, _ZERO)
    return to_host(_box_from_sat(x, k, pad, modes), is_torch(planes))


def naive_box_average(plane, k: int, pad: str = "reflect"):
    """pooling.py:161-172: direct O(H*W*k^2) shifted summation."""
    _check_kernel(k)
    x = _as_dev(plane)
    if x.dim() != 2:
        raise ValueError("plane must be 2-D")
    h, w = x.shape
    mr, mc = _pad_plane_modes(pad, h, w)
    x, code = _dtype_code(x)
    out = empty((h, w), torch.float64)
    N.call("qfca_naive_box", x.data_ptr(), code, 1, h, w, k, mr, mc, out.data_ptr(), N.stream())
    return to_host(out, is_torch(plane))
