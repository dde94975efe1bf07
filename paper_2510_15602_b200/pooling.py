"""Box pooling on the GPU (reference pooling.py:97-158).

The scoring path never materialises box filters (the fused kernel slides),
but the reference exposes box_average / box_average_stack as API; here they
are two separable passes of csrc/finalize.cu's fp64 convolution with unit
taps, same pad semantics (zero = clamped window, reflect / wrap = np.pad).
"""

from __future__ import annotations

import numpy as np
import torch

from ._dev import is_torch, to_dev, to_host
from .features import sep_convolve_dev

PAD_MODES = ("zero", "reflect", "wrap")

__all__ = ["PAD_MODES", "box_average", "box_average_stack"]


def _check_kernel(k: int) -> int:
    if k < 1 or k % 2 == 0:
        raise ValueError(f"kernel size must be odd and >= 1, got {k}")
    return k // 2


def box_average_stack(planes, k: int, pad: str = "reflect"):
    """pooling.py:125-158: k x k local average of a (B, H, W) stack."""
    _check_kernel(k)
    if pad not in PAD_MODES:
        raise ValueError(f"unknown pad mode {pad!r}")
    x = to_dev(planes, torch.float64)
    out = sep_convolve_dev(x, np.ones(k, np.float64), pad) / float(k * k)
    return to_host(out, is_torch(planes))


def box_average(plane, k: int, pad: str = "reflect"):
    """pooling.py:120-122."""
    x = to_dev(plane, torch.float64)
    out = box_average_stack(x[None], k, pad)[0]
    return to_host(out, is_torch(plane))
