"""Host <-> device conversions for the drop-in API.

Public functions accept NumPy arrays (the reference's types) or torch CUDA
tensors.  NumPy inputs are copied to the GPU and results come back as NumPy
with the reference's dtypes; torch inputs stay on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from ._native import require_cuda


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_dev(x, dtype=torch.float32) -> torch.Tensor:
    dev = require_cuda()
    if is_torch(x):
        return x.to(device=dev, dtype=dtype).contiguous()
    np_dtype = {torch.float32: np.float32, torch.float64: np.float64,
                torch.int32: np.int32, torch.uint8: np.uint8,
                torch.int64: np.int64}[dtype]
    a = np.ascontiguousarray(np.asarray(x), dtype=np_dtype)
    return torch.from_numpy(a).to(dev, non_blocking=False)


def to_host(t: torch.Tensor, like_torch: bool):
    """Return t itself if the caller passed torch tensors, else a NumPy copy."""
    if like_torch:
        return t
    return t.detach().cpu().numpy()


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=require_cuda())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=require_cuda())
