"""QTF1 feature files (reference tensor_io.py:1-124) read straight into the GPU path.

The reference's on-disk / wire format for features:

    magic "QTF1" | dtype u8 (1 = float32, 2 = uint8) | ndim u8 |
    ndim x u64 little-endian dims | raw row-major little-endian data

Same byte layout, same validation and the same exception classes as
``qfca.tensor_io`` (write_tensor / read_tensor, tensor_io.py:79-124).  The
B200 addition is ``read_features``: the payload is read into page-locked host
memory and copied to the device asynchronously, so a batch of feature files
feeds ``detect_batch`` / ``DetectPipeline`` without a pageable staging copy.
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

MAGIC = b"QTF1"
_DTYPE_CODES = {np.dtype(np.float32): 1, np.dtype(np.uint8): 2}
_CODE_DTYPES = {1: np.dtype(np.float32), 2: np.dtype(np.uint8)}

__all__ = ["MAGIC", "TensorFormatError", "BadMagicError", "TruncatedError",
           "UnsupportedDtypeError", "write_tensor", "read_tensor", "read_features"]


class TensorFormatError(Exception):
    """Base class for QTF1 format violations (tensor_io.py:30)."""


class BadMagicError(TensorFormatError):
    pass


class TruncatedError(TensorFormatError):
    pass


class UnsupportedDtypeError(TensorFormatError):
    pass


def write_tensor(array, path: str | os.PathLike) -> None:
    """tensor_io.py:79-93: serialise a float32 / uint8 array (ndim 1..4)."""
    a = np.ascontiguousarray(array.detach().cpu().numpy() if isinstance(array, torch.Tensor)
                             else array)
    code = _DTYPE_CODES.get(a.dtype)
    if code is None:
        raise UnsupportedDtypeError(f"unsupported dtype {a.dtype}")
    if not 1 <= a.ndim <= 4:
        raise ValueError(f"ndim must be in [1, 4], got {a.ndim}")
    if any(d < 1 for d in a.shape):
        raise ValueError(f"shape entries must be >= 1, got {a.shape}")
    header = MAGIC + struct.pack("<BB", code, a.ndim) + struct.pack(f"<{a.ndim}Q", *a.shape)
    with open(path, "wb") as f:
        f.write(header)
        f.write(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())


def _parse_header(raw: bytes, path) -> tuple[np.dtype, tuple[int, ...], int]:
    """tensor_io.py:96-124: validate magic, dtype, ndim, dims, payload length."""
    if raw[:4] != MAGIC:
        raise BadMagicError(f"{path}: bad magic {raw[:4]!r}")
    if len(raw) < 6:
        raise TruncatedError(f"{path}: header truncated")
    code, ndim = struct.unpack_from("<BB", raw, 4)
    if code not in _CODE_DTYPES:
        raise UnsupportedDtypeError(f"{path}: unknown dtype code {code}")
    if not 1 <= ndim <= 4:
        raise TensorFormatError(f"{path}: ndim {ndim} outside [1, 4]")
    if len(raw) < 6 + 8 * ndim:
        raise TruncatedError(f"{path}: dims truncated")
    shape = tuple(int(s) for s in struct.unpack_from(f"<{ndim}Q", raw, 6))
    dtype = _CODE_DTYPES[code]
    off = 6 + 8 * ndim
    expected = off + int(np.prod(shape)) * dtype.itemsize
    if len(raw) < expected:
        raise TruncatedError(f"{path}: payload truncated ({len(raw)} bytes, expected {expected})")
    if len(raw) > expected:
        raise TensorFormatError(f"{path}: {len(raw) - expected} trailing bytes")
    return dtype, shape, off


def read_tensor(path: str | os.PathLike) -> np.ndarray:
    """Inverse of write_tensor: the array (reference Tensor.to_array())."""
    with open(path, "rb") as f:
        raw = f.read()
    dtype, shape, off = _parse_header(raw, path)
    n = int(np.prod(shape))
    return np.frombuffer(raw, dtype=dtype.newbyteorder("<"), count=n,
                         offset=off).astype(dtype, copy=False).reshape(shape)


def read_features(paths, device=None) -> torch.Tensor:
    """A batch of (C, h, w) float32 QTF1 feature files -> (B, C, h, w) device
    tensor: payloads land in one page-locked host buffer, then one
    non-blocking copy on the current stream.  All files must share a shape."""
    paths = [paths] if isinstance(paths, (str, os.PathLike)) else list(paths)
    if not paths:
        raise ValueError("no feature files")
    host = None
    for i, p in enumerate(paths):
        with open(p, "rb") as f:
            raw = f.read()
        dtype, shape, off = _parse_header(raw, p)
        if dtype != np.float32 or len(shape) != 3:
            raise TensorFormatError(f"{p}: features must be float32 (C, h, w), got "
                                    f"{dtype} {shape}")
        if host is None:
            host = torch.empty((len(paths),) + shape, dtype=torch.float32).pin_memory()
        elif tuple(host.shape[1:]) != shape:
            raise ValueError(f"{p}: shape {shape} differs from {tuple(host.shape[1:])}")
        host[i].numpy().reshape(-1)[:] = np.frombuffer(raw, dtype="<f4", offset=off,
                                                       count=int(np.prod(shape)))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    return host.to(dev, non_blocking=True)
