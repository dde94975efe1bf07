"""ctypes binding of libqfca_b200.so (the C-ABI in include/qfca_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises.  Device buffers are torch CUDA tensors (PyTorch is only
the allocator / stream provider here); the kernels run on the current torch
stream.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# QFCA_B200_LIB: an alternative build of the same library (A/B timing of kernels)
LIB_PATH = os.environ.get("QFCA_B200_LIB") or os.path.join(_HERE, "libqfca_b200.so")

QFCA_OK, QFCA_ERR_ARG, QFCA_ERR_CUDA, QFCA_ERR_UNSUPPORTED = 0, 1, 2, 3
PAD_CODES = {"zero": 0, "reflect": 1, "wrap": 2}  # scoring.py:155
REF_MODE_CODES = {"median-quan": 0, "mean-quan": 1, "quan-median": 2, "quan-mean": 3}

_P, _I32, _I64, _F64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class QfcaConfig(ctypes.Structure):
    _fields_ = [("n_bins", _I32), ("patch_size", _I32), ("pad", _I32),
                ("sample_budget", _I32), ("border", _I32), ("groups", _I32),
                ("sigma_s", _F64)]


_SIGNATURES = {
    "qfca_abi_version": ([], _I32),
    "qfca_launch_count": ([], _I64),
    "qfca_status_str": ([_I32], ctypes.c_char_p),
    "qfca_fit_quantizer": ([_P, _I64, _I64, _P, _P, _P, _P], _I32),
    "qfca_bin_indices": ([_P, _I64, _I64, _P, _P, _I32, _P, _I32, _P], _I32),
    "qfca_quantize": ([_P, _I64, _I64, _I32, _P, _P, _P, _P, _I32, _P], _I32),
    "qfca_sample_stride": ([_I32, _I32, _I32], _I32),
    "qfca_select_reference": ([_P, _I32, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _I32,
                               _I32, _P, _P], _I32),
    "qfca_reference_weights_workspace_bytes": ([_I64, _I32, _I32, _I32, _I32, _I32, _I32],
                                               _I64),
    "qfca_reference_weights": ([_P, _P, _I32, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _I32,
                                _I32, _P, _I64, _P, _P], _I32),
    "qfca_window_counts": ([_P, _I32, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P, _I32, _P],
                           _I32),
    "qfca_mismatch_pixels": ([_P, _I64, _I64, _I32, _P, _P, _P, _P, _P], _I32),
    "qfca_mismatch_rows": ([_P, _I64, _I32, _P, _P, _P, _P], _I32),
    "qfca_smooth_gather": ([_P, _P, _I32, _I64, _I32, _I32, _I32, _I32, _I32, _P, _F64, _P,
                            _P, _P], _I32),
    "qfca_channel_sum": ([_P, _I64, _I32, _I64, _P, _I32, _P, _P, _P], _I32),
    "qfca_count_used": ([_P, _P, _I64, _I32, _P, _P], _I32),
    "qfca_score_version": ([_I32, _I32, _I32, _I32, _I32, _I64, _I32, _I32, _I32], _I32),
    "qfca_set_score_kernel": ([_I32], _I32),
    "qfca_score_groups": ([_I32, _I32, _I32, _I32, _I32, _I64, _I32, _I32, _I32, _I32], _I32),
    "qfca_score": ([_P, _I32, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                    _P, _P], _I32),
    "qfca_score_ex": ([_P, _I32, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                       _I32, _P, _I64, _P, _P], _I32),
    "qfca_score_tiles": ([_P, _I32, _P, _P, _P, _I32, _I32, _I32, _P, _I32, _P, _I32, _I32,
                          _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _I64, _P, _P], _I32),
    "qfca_score_scratch_bytes": ([_I32, _I32, _I32, _I32, _I32, _I64, _I32, _I32, _I32, _I32],
                                 _I64),
    "qfca_score_groups_ex": ([_I32, _I32, _I32, _I32, _I32, _I64, _I32, _I32, _I32, _I32, _I32],
                             _I32),
    "qfca_reduce_partials": ([_P, _I64, _I32, _I64, _P, _P, _P], _I32),
    "qfca_divide_used": ([_P, _I64, _I64, _P, _P, _P], _I32),
    "qfca_sep_conv": ([_P, _I64, _I32, _I32, _I32, _P, _I32, _I32, _P, _P], _I32),
    "qfca_image_score": ([_P, _I64, _I32, _I32, _I32, _P, _P], _I32),
    "qfca_upsample": ([_P, _I64, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "qfca_plane_mean": ([_P, _I64, _I64, _P, _P], _I32),
    "qfca_center": ([_P, _I64, _I64, _P, _P, _P], _I32),
    "qfca_cholqr": ([_P, _I64, _I32, _I32, _P], _I32),
    "qfca_chol_rinv": ([_P, _I64, _I32, _P, _P], _I32),
    "qfca_sym_eig": ([_P, _I64, _I32, _P, _P, _P], _I32),
    "qfca_lanczos": ([_P, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P], _I32),
    "qfca_ritz": ([_P, _I64, _I32, _P, _I32, _P, _P, _P], _I32),
    "qfca_gather_tiles": ([_P, _I32, _I32, _I32, _P, _I32, _P, _I32, _I32, _I32, _P, _P], _I32),
    "qfca_pad_planes": ([_P, _I64, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "qfca_build_sat": ([_P, _I32, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "qfca_sat_box": ([_P, _I64, _I32, _I32, _I32, _I32, _F64, _P, _P], _I32),
    "qfca_sat_rects": ([_P, _I32, _P, _I64, _P, _P], _I32),
    "qfca_naive_box": ([_P, _I32, _I64, _I32, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "qfca_covariance_workspace_bytes": ([_I64, _I32, _I32], _I64),
    "qfca_covariance": ([_P, _I64, _I32, _I32, _P, _P, _I64, _P, _P], _I32),
    "qfca_mean_covariance": ([_P, _I64, _I32, _I32, _P, _P, _I64, _P, _P], _I32),
    "qfca_pca_residual": ([_P, _I64, _I32, _I64, _P, _P, _I32, _I32, _P, _P], _I32),
    "qfca_pca_residual_slice": ([_P, _I64, _I32, _I64, _P, _P, _I32, _I32, _I32, _I32, _P, _P],
                                _I32),
    "qfca_detect_workspace_bytes": ([_I64, _I32, _I32, _I32, ctypes.POINTER(QfcaConfig)], _I64),
    "qfca_detect": ([_P, _I64, _I32, _I32, _I32, ctypes.POINTER(QfcaConfig), _P, _I64, _P, _P,
                     _P, _P, _P], _I32),
    "qfca_detect_ex": ([_P, _I64, _I32, _I32, _I32, ctypes.POINTER(QfcaConfig), _P, _I64, _P,
                        _P, _P, _P, _P, _P], _I32),
    "qfca_pool_interior": ([_P, _I32, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P], _I32),
    "qfca_pool_interior_table": ([_P, _I32, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P],
                                 _I32),
    "qfca_rank_stats_workspace_bytes": ([_I64, _I32], _I64),
    "qfca_rank_stats": ([_P, _I32, _P, _I64, _P, _I64, _P, _P, _P], _I32),
    "qfca_components_workspace_bytes": ([_I64], _I64),
    "qfca_components": ([_P, _I32, _I32, _I32, _P, _I64, _P, _P, _P, _P], _I32),
    "qfca_pro_histograms": ([_P, _P, _I64, _P, _I32, _I32, _I32, _P, _P, _P], _I32),
    "qfca_pro_accumulate": ([_P, _I32, _I32, _P, _P], _I32),
}

EXPORTED = tuple(_SIGNATURES)
_lib = None


class NativeUnavailable(ImportError):
    """libqfca_b200.so missing or unloadable -- build it; there is no fallback."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} not found: run `python -m paper_2510_15602_b200.build` "
                "(there is no CPU fallback)")
        try:
            L = ctypes.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_15602_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def check(status: int, what: str) -> None:
    if status == QFCA_OK:
        return
    msg = f"{what}: {lib().qfca_status_str(status).decode()}"
    if status == QFCA_ERR_ARG:
        raise ValueError(msg)
    if status == QFCA_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def launch_count() -> int:
    return int(lib().qfca_launch_count())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
