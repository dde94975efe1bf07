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
           "UnsupportedDtypeError", "write_tensor", "read_tensor", "read_features",
           "DecodeError", "DatasetIndexError", "DatasetSample", "load_dataset", "load_mask",
           "feature_scale"]


class TensorFormatError(Exception):
    """Base class for QTF1 format violations (tensor_io.py:27-28)."""


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


# ---- dataset tree, masks and external feature files (the CLI's inputs) ----

class DecodeError(Exception):
    """tensor_io.py:43-44 -- an image file could not be decoded."""


class DatasetIndexError(Exception):
    """tensor_io.py:47-48 -- the dataset tree is malformed."""


def _nearest_index(n_in: int, n_out: int) -> np.ndarray:
    """tensor_io.py:133-147 -- half-pixel centres, rounded, clamped."""
    c = (np.arange(n_out) + 0.5) * n_in / n_out - 0.5
    return np.clip(np.round(c), 0, n_in - 1).astype(int)


def load_mask(path, size=None) -> np.ndarray:
    """tensor_io.py:186-191 -- binary H x W mask (any value > 0), optionally
    resized with nearest sampling.  Pixel decode through Pillow like the
    reference's load_image (tensor_io.py:161-183)."""
    from PIL import Image
    try:
        with Image.open(path) as im:
            im = im.convert("RGB") if im.mode not in ("L", "RGB") else im
            arr = np.asarray(im)
    except Exception as e:  # noqa: BLE001 -- the reference wraps every decoder error
        raise DecodeError(f"cannot decode {path}: {e}") from e
    plane = arr if arr.ndim == 2 else arr[..., 0]
    m = plane > 0
    if size is not None:
        if isinstance(size, int):
            size = (size, size)
        if tuple(size) != m.shape:
            m = m[np.ix_(_nearest_index(m.shape[0], size[0]),
                         _nearest_index(m.shape[1], size[1]))]
    return m


class DatasetSample:
    """tensor_io.py:194-199."""

    __slots__ = ("image_path", "mask_path", "is_anomalous", "defect_type")

    def __init__(self, image_path, mask_path, is_anomalous, defect_type):
        self.image_path, self.mask_path = image_path, mask_path
        self.is_anomalous, self.defect_type = is_anomalous, defect_type


def load_dataset(root, class_name: str, layout: str = "mvtec") -> list:
    """tensor_io.py:207-239 -- index root/class/test/<defect>/*.png|ppm with
    masks at root/class/ground_truth/<defect>/<stem>_mask.png ("good" has
    none), lexicographic by defect then file name."""
    if layout != "mvtec":
        raise ValueError(f"unknown layout {layout!r}")
    test_dir = os.path.join(root, class_name, "test")
    gt_dir = os.path.join(root, class_name, "ground_truth")
    if not os.path.isdir(test_dir):
        raise DatasetIndexError(f"missing test directory {test_dir}")
    out = []
    for defect in sorted(os.listdir(test_dir)):
        ddir = os.path.join(test_dir, defect)
        if not os.path.isdir(ddir):
            continue
        bad = defect != "good"
        for fname in sorted(os.listdir(ddir)):
            if not fname.lower().endswith((".png", ".ppm")):
                continue
            mask = None
            if bad:
                mask = os.path.join(gt_dir, defect, os.path.splitext(fname)[0] + "_mask.png")
                if not os.path.isfile(mask):
                    raise DatasetIndexError(f"anomalous sample {os.path.join(ddir, fname)} "
                                            f"has no mask at {mask}")
            out.append(DatasetSample(os.path.join(ddir, fname), mask, bad, defect))
    return out


def feature_scale(path) -> int:
    """features.py:135-146 -- downsampling factor from the <path>.json sidecar
    ({"scale": s}), 8 when absent."""
    import json
    side = str(path) + ".json"
    if os.path.isfile(side):
        with open(side) as f:
            return int(json.load(f)["scale"])
    return 8
