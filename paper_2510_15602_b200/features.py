"""Feature maps and PCA-residual preprocessing on the GPU.

Mirrors qfca.features (reference features.py:26-41, 49-77, 150-193): same
names, same dataclasses, same validation and error types.  pca_fit: plane
means and the exact covariance on the int8 tensor cores (csrc/cov_i8.cu),
top-k eigenpairs by block Lanczos on the fp64 tensor cores (csrc/lanczos.cu)
plus the Ritz step on the small projection (csrc/eig.cu); pca_residual: fp64
MMA kernel (csrc/residual.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._dev import empty, is_torch, to_dev, to_host, zeros

__all__ = ["FeatureMap", "PcaModel", "pca_fit", "pca_residual", "pca_fit_batch",
           "pca_residual_batch", "gaussian_blur", "FormatError"]


class FormatError(Exception):
    """External feature file does not match the expected layout."""


@dataclass(frozen=True)
class FeatureMap:
    """(C, H, W) float32 features + downsampling scale (features.py:26-41).

    ``values`` may be a NumPy array or a torch CUDA tensor.
    """

    values: object
    scale: int = 1

    def __post_init__(self):
        v = self.values
        if v.ndim != 3:
            raise ValueError("feature values must be (C, H, W)")
        if self.scale < 1:
            raise ValueError("scale must be >= 1")
        if is_torch(v):
            finite = bool(torch.isfinite(v).all())
        else:
            finite = bool(np.all(np.isfinite(v)))
        if not finite:
            raise ValueError("feature values must be finite")

    @property
    def n_channels(self) -> int:
        return self.values.shape[0]


@dataclass(frozen=True)
class PcaModel:
    mean: object        # (C,) fp64
    components: object  # (k, C) fp64, orthonormal rows
    eigenvalues: object  # (k,) fp64, non-increasing


def _gauss_kernel(sigma: float) -> np.ndarray:
    """features.py:49-53."""
    radius = int(np.ceil(3 * sigma))
    x = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def sep_convolve_dev(planes: torch.Tensor, kernel: np.ndarray, pad: str) -> torch.Tensor:
    """_sep_convolve (features.py:56-69) on a (B, H, W) fp64 device stack."""
    b, h, w = planes.shape
    k = np.ascontiguousarray(kernel, dtype=np.float64)
    tmp = empty((b, h, w), torch.float64)
    out = empty((b, h, w), torch.float64)
    s = N.stream()
    kp = k.ctypes.data_as(N._P)
    N.call("qfca_sep_conv", planes.data_ptr(), b, h, w, 0, kp, k.size, N.PAD_CODES[pad],
           tmp.data_ptr(), s)
    N.call("qfca_sep_conv", tmp.data_ptr(), b, h, w, 1, kp, k.size, N.PAD_CODES[pad],
           out.data_ptr(), s)
    return out


def gaussian_blur(plane, sigma: float, pad: str = "reflect"):
    """features.py:72-77 on the GPU; returns the input's kind (NumPy / torch)."""
    if sigma <= 0:
        return plane.to(torch.float64) if is_torch(plane) else np.asarray(plane, np.float64)
    x = to_dev(plane, torch.float64)
    out = sep_convolve_dev(x.reshape((1,) + tuple(x.shape)), _gauss_kernel(sigma), pad)[0]
    return to_host(out, is_torch(plane))


def _tf32_split(x: torch.Tensor):
    """x = hi + lo with hi exactly representable in TF32 (10-bit mantissa)."""
    hi_ = (x.view(torch.int32) & -8192).view(torch.float32)
    return hi_, x - hi_


def covariance_dev(xc: torch.Tensor, chunk: int = 1024, precise: str = "fp32"
                   ) -> torch.Tensor:
    """(B, C, HW) centred fp32 -> (B, C, C) fp64 population covariance.

    Tensor-core GEMMs over K-chunks summed in fp64, / HW.  "3xtf32" splits
    the operand into a TF32 head and an fp32 tail and keeps the three
    significant products (hi hi' + hi lo' + lo hi') at TF32 tensor-core
    speed; "fp32" (default) uses IEEE fp32 GEMMs.  Measured on the config-1
    golden: fp32 moves the QFCA+ map by 9e-9 (channel count aligned), 3xtf32
    by 1.7e-4 (the TF32 rounding of the tail is not negligible against the
    lambda_10 / lambda_11 gap), a single TF32 pass by ~4e-4.
    """
    b, c, hw = xc.shape
    nk = (hw + chunk - 1) // chunk
    if nk * chunk != hw:
        xc = torch.nn.functional.pad(xc, (0, nk * chunk - hw))
    blocks = xc.reshape(b, c, nk, chunk).permute(0, 2, 1, 3).reshape(b * nk, c, chunk)
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        if precise == "fp64":  # fp64 tensor-core GEMM (DMMA), the reference's precision
            part = torch.bmm(blocks.double(), blocks.double().transpose(1, 2))
        elif precise == "3xtf32":
            torch.backends.cuda.matmul.allow_tf32 = True
            hi_, lo_ = _tf32_split(blocks)
            part = torch.bmm(hi_, hi_.transpose(1, 2))
            cross = torch.bmm(hi_, lo_.transpose(1, 2))
            part += cross
            part += cross.transpose(1, 2)
        else:
            torch.backends.cuda.matmul.allow_tf32 = False
            part = torch.bmm(blocks, blocks.transpose(1, 2))
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    cov = part.reshape(b, nk, c, c).sum(dim=1, dtype=torch.float64)
    return cov / float(hw)


_COV_WS: dict = {}


def covariance_exact(x: torch.Tensor, mean: torch.Tensor | None) -> torch.Tensor:
    """(B, C, H, W) fp32 features, (B, C) fp64 means -> (B, C, C) fp64 covariance
    (features.py:167-171), fp64-accurate.

    The QFCA+ maps depend on the covariance at the 1e-8 level (an fp32 GEMM
    moves them by up to 3e-4 on the bench workload through residual bin
    flips), so the covariance is formed exactly: int8-digit fixed point on
    the int8 tensor cores (csrc/cov_i8.cu, ~1e-11 relative).  Planes larger
    than the kernel's exactness bound (hw > 16384) use an fp64 cuBLAS GEMM.
    """
    b, c = x.shape[:2]
    hw = x[0, 0].numel()
    L = N.lib()
    need = int(L.qfca_covariance_workspace_bytes(b, c, hw))
    cov = empty((b, c, c), torch.float64)
    # one cached workspace per (device, stream, size): calls on different streams may overlap
    key = (x.device.index, torch.cuda.current_stream(x.device).cuda_stream, need)
    ws = _COV_WS.get(key)
    if ws is None:
        if len(_COV_WS) > 8:
            _COV_WS.clear()
        ws = _COV_WS[key] = empty((max(need, 1),), torch.uint8)
    if mean is None:  # also form the plane means (features.py:170), returned
        mean_out = empty((b, c), torch.float64)
        st = L.qfca_mean_covariance(x.data_ptr(), b, c, hw, mean_out.data_ptr(), ws.data_ptr(),
                                    need, cov.data_ptr(), N.stream())
        if st == N.QFCA_ERR_UNSUPPORTED:
            N.call("qfca_plane_mean", x.data_ptr(), b * c, hw, mean_out.data_ptr(), N.stream())
            return covariance_exact(x, mean_out), mean_out
        N.check(st, "qfca_mean_covariance")
        return cov, mean_out
    st = L.qfca_covariance(x.data_ptr(), b, c, hw, mean.data_ptr(), ws.data_ptr(), need,
                           cov.data_ptr(), N.stream())
    if st == N.QFCA_ERR_UNSUPPORTED:
        xd = x.reshape(b, c, hw).double() - mean[:, :, None]
        return torch.bmm(xd, xd.mT) / float(hw)
    N.check(st, "qfca_covariance")
    return cov


def _cholqr_inplace(y: torch.Tensor) -> torch.Tensor:
    """Cholesky QR of a fresh contiguous (B, C, p) block, in place (csrc/eig.cu
    k_cqr_step: Gram, Cholesky, R^-1 and Y R^-1 in one launch per batch)."""
    b, c, p = y.shape
    N.call("qfca_cholqr", y.data_ptr(), b, c, p, N.stream())
    return y


def _cholqr(y: torch.Tensor) -> torch.Tensor:
    """Orthonormal basis of the columns of y (B, C, p) by Cholesky QR.

    One fused kernel per block (csrc/pca.cu k_cholqr: Gram, Cholesky and the
    triangular solve with the block resident in shared memory); torch's
    cuSOLVER / cuBLAS route for blocks that do not fit.
    """
    b, c, p = y.shape
    if y.is_cuda and (c * (p | 1) + p * p) * 8 <= 200 * 1024:
        out = y.contiguous().clone() if not y.is_contiguous() else y.clone()
        N.call("qfca_cholqr", out.data_ptr(), b, c, p, N.stream())
        return out
    g = y.mT @ y
    lo = torch.linalg.cholesky(g)
    return torch.linalg.solve_triangular(lo.mT, y, upper=True, left=False)


_X0: dict = {}


def _start_block(c: int, p: int, device) -> torch.Tensor:
    """Seeded orthonormal start block (c, p), cached per shape and device."""
    key = (c, p, str(device))
    if key not in _X0:
        gen = torch.Generator(device="cpu").manual_seed(20251018)
        x0 = torch.randn(c, p, generator=gen, dtype=torch.float64)
        _X0[key] = torch.linalg.qr(x0)[0].contiguous().to(device)
    return _X0[key]


def chol_rinv(g: torch.Tensor) -> torch.Tensor:
    """(B, p, p) Gram matrices -> R^-1 (Cholesky QR factor), p <= 32 (csrc/eig.cu)."""
    b, p, _ = g.shape
    out = empty((b, p, p), torch.float64)
    N.call("qfca_chol_rinv", g.contiguous().data_ptr(), b, p, out.data_ptr(), N.stream())
    return out


def sym_eig(h: torch.Tensor):
    """(B, p, p) symmetric -> (evals (B, p) descending, evecs (B, p, p) columns),
    p <= 32, parallel Jacobi (csrc/eig.cu); no host synchronisation."""
    b, p, _ = h.shape
    w = empty((b, p), torch.float64)
    v = empty((b, p, p), torch.float64)
    N.call("qfca_sym_eig", h.contiguous().data_ptr(), b, p, w.data_ptr(), v.data_ptr(),
           N.stream())
    return w, v


LANCZOS_BW, LANCZOS_PASSES = 8, 16  # csrc/lanczos.cu block width; passes over cov
LANCZOS_DIM = LANCZOS_BW * LANCZOS_PASSES
LANCZOS_SPLIT = True  # two-CTA clusters per covariance (csrc/lanczos.cu)


def _topk_eigh_lanczos(cov: torch.Tensor, k: int, block: int, iters: int):
    """Block Lanczos (csrc/lanczos.cu: 16 passes of an 8-column block over cov,
    full reorthogonalisation) -> the 128 x 128 projection H = B^T cov B, whose
    top-k Ritz pairs come from the small-matrix path of topk_eigh below and map
    back as V = B u (csrc/eig.cu k_ritz: the subspace iteration of this
    function on the small matrix, one launch).  Same answer as the subspace iteration on cov (the Krylov
    space holds the top-10 eigenvectors of the WRN50-2 covariances to ~1e-15,
    tools/lanczos_proto.py) for ~1/8 of its passes over cov and no C^3 product."""
    b, c, _ = cov.shape
    n = LANCZOS_DIM
    cov = cov.contiguous()
    q0 = _start_block(c, LANCZOS_BW, cov.device).contiguous()
    basis = empty((b, n, c), torch.float64)
    h = empty((b, n, n), torch.float64)
    if LANCZOS_SPLIT:  # two CTAs per matrix (cluster), partial S Q exchanged per pass
        twin = empty((b, n, c), torch.float64)
        xch = empty((b, 4, c, LANCZOS_BW), torch.float64)
        flags = zeros((b,), torch.int32)
        N.call("qfca_lanczos", cov.data_ptr(), b, c, LANCZOS_PASSES, q0.data_ptr(),
               basis.data_ptr(), h.data_ptr(), twin.data_ptr(), xch.data_ptr(),
               flags.data_ptr(), N.stream())
    else:
        N.call("qfca_lanczos", cov.data_ptr(), b, c, LANCZOS_PASSES, q0.data_ptr(),
               basis.data_ptr(), h.data_ptr(), None, None, None, N.stream())
    p = 32
    x0 = _start_block(n, p, cov.device).contiguous()
    x = empty((b, n, p), torch.float64)
    hm = empty((b, p, p), torch.float64)
    N.call("qfca_ritz", h.data_ptr(), b, n, x0.data_ptr(), (iters + 1) // 2, x.data_ptr(),
           hm.data_ptr(), N.stream())
    w, u = sym_eig(hm)
    return w[..., :k], basis.mT @ (x @ u[..., :k])


def topk_eigh(cov: torch.Tensor, k: int, block: int = 32, iters: int = 30,
              lanczos: bool = True):
    """Top-k eigenpairs of a batch of symmetric PSD matrices (B, C, C), fp64.

    Replaces the full ``np.linalg.eigh`` of features.py:173 (only the top-k
    pairs are used, features.py:174-176).  For 256 <= C <= 512 (C % 64 == 0)
    block Lanczos over cov (``_topk_eigh_lanczos``), whose 128 x 128
    projection goes through the path below.  Otherwise (and for that small
    matrix): block subspace iteration (block p = max(block, k) columns) on
    cov^2, re-orthonormalised by Cholesky QR, then a Rayleigh-Ritz step on cov
    with a parallel-Jacobi eigensolver.  The error of the k-th vector decays as
    (lambda_{p+1} / lambda_k)^iters; on random-init WRN50-2 block-2 features
    (lambda_33 / lambda_10 ~ 0.2-0.33) 30 iterations reach the fp64 eigh to
    ~1e-15.  C <= p degenerates to an exact eigen-decomposition of the whole
    matrix.  Returns (eigenvalues (B, k) descending, vectors (B, C, k)).
    """
    b, c, _ = cov.shape
    p = min(c, max(block, k))
    if p > 32:
        return _topk_eigh_torch(cov, k, p, iters)
    if lanczos and k <= 16 and c >= 2 * LANCZOS_DIM and c <= 512 and c % 64 == 0:
        return _topk_eigh_lanczos(cov, k, block, iters)
    if p == c:
        w, u = sym_eig(cov)
        return w[..., :k], u[..., :k]
    # iterate with cov^2 (one fp64 GEMM up front): same subspace, squared
    # rate, half the iterations; the squaring costs ~eps (lambda_1 /
    # lambda_k)^2 relative to lambda_k^2 (~1e-12 here)
    sq = cov @ cov
    x = _start_block(c, p, cov.device).expand(b, c, p)
    for _ in range((iters + 1) // 2):
        x = _cholqr_inplace(sq @ x)
    hm = x.mT @ (cov @ x)
    w, u = sym_eig(hm)
    return w[..., :k], x @ u[..., :k]


def _topk_eigh_torch(cov: torch.Tensor, k: int, p: int, iters: int):
    """Blocks wider than 32 columns: the same iteration on torch / cuSOLVER."""
    b, c, _ = cov.shape
    sq = cov @ cov
    x = _start_block(c, p, cov.device).expand(b, c, p)
    for _ in range((iters + 1) // 2):
        x = _cholqr(sq @ x)
    hm = x.mT @ (cov @ x)
    hm = 0.5 * (hm + hm.mT)
    w, u = torch.linalg.eigh(hm)  # ascending
    return w[..., -k:].flip(-1), x @ u[..., -k:].flip(-1)


def pca_fit_batch(x: torch.Tensor, k: int):
    """Batched pca_fit on (B, C, H, W) device features -> (mean, comps, evals)."""
    b, c, h, w = x.shape
    hw = h * w
    s = N.stream()
    cov, mean = covariance_exact(x, None)  # means and covariance in one pass over x
    # np.argsort(evals, kind="stable")[::-1][:k] of the ascending eigh output is
    # the top-k in descending order (ties keep the higher index first)
    evals, vecs = topk_eigh(cov, k)
    ev = evals.clamp(min=0.0)
    comps = vecs.transpose(1, 2).contiguous()  # (B, k, C)
    arg = comps.abs().argmax(dim=2, keepdim=True)
    sign = torch.where(torch.gather(comps, 2, arg) < 0, -1.0, 1.0).to(comps.dtype)
    comps = comps * sign
    return mean, comps, ev


def pca_residual_batch(x: torch.Tensor, mean: torch.Tensor, comps: torch.Tensor,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched pca_residual (per-image model) on (B, C, H, W) device features."""
    b, c, h, w = x.shape
    k = comps.shape[-2]
    if out is None:
        out = empty((b, c, h, w), torch.float32)
    per_image = 1 if mean.dim() == 2 else 0
    N.call("qfca_pca_residual", x.data_ptr(), b, c, h * w,
           mean.contiguous().data_ptr(), comps.contiguous().data_ptr(), k, per_image,
           out.data_ptr(), N.stream())
    return out


def pca_residual_slice(x: torch.Tensor, mean: torch.Tensor, comps: torch.Tensor, c0: int,
                       c1: int) -> torch.Tensor:
    """Residual of channels [c0, c1) only, (B, c1 - c0, H, W): a channel-sharded
    rank's slice (the projection still uses every channel)."""
    b, c, h, w = x.shape
    k = comps.shape[-2]
    out = empty((b, c1 - c0, h, w), torch.float32)
    per_image = 1 if mean.dim() == 2 else 0
    rc = N.lib().qfca_pca_residual_slice(x.data_ptr(), b, c, h * w, mean.contiguous().data_ptr(),
                                         comps.contiguous().data_ptr(), k, per_image, c0, c1,
                                         out.data_ptr(), N.stream())
    if rc == N.QFCA_ERR_UNSUPPORTED:  # shapes the tensor-core kernel does not take
        return pca_residual_batch(x, mean, comps)[:, c0:c1].contiguous()
    N.check(rc, "qfca_pca_residual_slice")
    return out


def pca_fit(f: FeatureMap, k: int) -> PcaModel:
    """features.py:157-180: top-k principal components of the pixel vectors."""
    c = f.n_channels
    if not (1 <= k <= c):
        raise ValueError(f"k must be in [1, {c}], got {k}")
    x = to_dev(f.values)
    mean, comps, ev = pca_fit_batch(x[None], k)
    t = is_torch(f.values)
    return PcaModel(mean=to_host(mean[0], t), components=to_host(comps[0], t),
                    eigenvalues=to_host(ev[0], t))


def pca_residual(f: FeatureMap, m: PcaModel) -> FeatureMap:
    """features.py:183-193: r = (x - mean) - V^T V (x - mean), float32."""
    c = f.n_channels
    if m.mean.shape[0] != c:
        raise ValueError(f"model has {m.mean.shape[0]} channels, features have {c}")
    x = to_dev(f.values)
    mean = to_dev(m.mean, torch.float64)
    comps = to_dev(m.components, torch.float64)
    r = pca_residual_batch(x[None], mean, comps)[0]
    return FeatureMap(values=to_host(r, is_torch(f.values)), scale=f.scale)
