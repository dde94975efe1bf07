"""Quantized 1-D transport mismatch (Alg. 1) on the GPU.

Mirrors qfca.transport's kernel API (reference transport.py:14-125): same
validation and MassError, the row-parallel batch kernel runs as
qfca_mismatch_rows (csrc/generic.cu) with the reference's fp64 arithmetic.
The fused scoring path does not call this: it uses the closed form in
csrc/score.cu.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from ._dev import empty, is_torch, to_dev

REL_MASS_TOL = 1e-6
_EPS_FACTOR = 1e-9

__all__ = ["MassError", "IllConditionedError", "quantized_mismatch", "mismatch_batch",
           "mismatch_batch_dev"]


class MassError(ValueError):
    """Patch and reference histogram masses differ beyond tolerance."""


class IllConditionedError(ValueError):
    """Input too degenerate for a stable finite-difference check."""


def _validate(P, R, Q):
    """transport.py:22-35."""
    P = np.asarray(P, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    Q = np.asarray(Q, dtype=np.float64)
    if not (P.shape == R.shape == Q.shape) or P.ndim != 1:
        raise ValueError("P, R, Q must be 1-D and of equal length")
    if np.any(P < 0) or np.any(R < 0):
        raise ValueError("histogram weights must be non-negative")
    if np.any(np.diff(Q) <= 0):
        raise ValueError("bin centers must be strictly increasing")
    mp, mr = P.sum(), R.sum()
    if abs(mp - mr) > REL_MASS_TOL * max(mp, mr, 1.0):
        raise MassError(f"histogram masses differ: {mp} vs {mr}")
    return P, R, Q


def mismatch_batch_dev(pb: torch.Tensor, r: torch.Tensor, q: torch.Tensor,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """(M, N) fp64 device rows -> (M, N) per-bin errors (transport.py:110-125)."""
    m, n = pb.shape
    if out is None:
        out = empty((m, n), torch.float64)
    N.call("qfca_mismatch_rows", pb.data_ptr(), m, n, r.data_ptr(), q.data_ptr(),
           out.data_ptr(), N.stream())
    return out


def mismatch_batch(Pb, R, Q, out) -> None:
    """transport.py:110-125: fills ``out`` (M, N) in place."""
    like = is_torch(Pb)
    pb = to_dev(Pb, torch.float64)
    res = mismatch_batch_dev(pb, to_dev(R, torch.float64), to_dev(Q, torch.float64))
    if like:
        out.copy_(res)
    else:
        out[...] = res.cpu().numpy()


def quantized_mismatch(P, R, Q, return_iterations: bool = False):
    """transport.py:38-70: per-bin mismatch between P and R on centers Q."""
    P, R, Q = _validate(P, R, Q)
    pb = to_dev(P[None], torch.float64)
    # masses are equal within REL_MASS_TOL (validated); for equal fp64 sums the
    # batch kernel's rescale factor mp / mr is exactly 1
    e = mismatch_batch_dev(pb, to_dev(R, torch.float64), to_dev(Q, torch.float64))
    e = e[0].cpu().numpy()
    if return_iterations:
        # the two-pointer walk advances one pointer per step: <= 2N - 1
        return e, _iterations(P, R)
    return e


def _iterations(P, R) -> int:
    """Step count of the walk (host bookkeeping for the A2 bound check)."""
    n = P.size
    p, r = P.copy(), R.copy()
    eps = _EPS_FACTOR * max(p.sum(), 1e-300)
    i = j = it = 0
    while i < n and j < n:
        it += 1
        if p[i] < r[j] - eps:
            r[j] -= p[i]
            i += 1
        else:
            p[i] -= r[j]
            j += 1
    return it
