"""Multi-GPU layouts of the scoring path.

* Batches of images: every image is independent -> shard the batch, one
  process per GPU, no collective (bench.py under torchrun, ``shard_batch``).
* One very large image (8192^2 -> 512 x 1024^2 features): every stage up to
  the channel sum is per channel (quantize.py:66-68, 168-199; scoring.py:
  264-281), so each rank scores a contiguous channel slice and ONE all-reduce
  (sum) of the (h*w + 1) fp64 partial -- channel-sum map plus the count of
  used channels -- combines them; every rank then finalises (channel mean,
  Gaussian, image score) identically.  NCCL over NVLink in production, gloo
  in the CPU tests.

Feature planes wider than the fused kernels' 128 columns (configs[4]: 1024 x
1024 per channel) are scored in full-height column strips of 128 (``strips``):
strip s covers columns [a_s, a_s + 128) and owns the outputs more than 2R
columns from its inner edges (an output needs E within R, E needs bins within
R), so the strips' own border padding never reaches an owned output; the true
image borders are strip borders and keep the reference's reflect padding.  The
median-quan reference of each channel comes from the whole plane (K3), so every
strip scores against the same reference; the strips run as one batched launch
of the plane-width-128 fused kernel.
"""

from __future__ import annotations

import torch

from . import _native as N
from ._dev import empty, zeros
from .features import _gauss_kernel, sep_convolve_dev
from .quantize import bins_dev, minmax_dev

__all__ = ["shard_range", "shard_batch", "combine_partials", "channel_partial",
           "detect_channel_sharded", "strips", "pca_fit_sharded", "detect_pca_sharded"]

STRIP_W = 128  # widest plane of the fused kernels
STRIP_H = 128  # tile height: 128 x 128 tiles keep the v6 count scratch L2-resident
USE_STRIPS = True  # route wide planes through strips (False: whole-plane generic kernel)


def strips(w: int, t: int, sw: int = STRIP_W):
    """Segments of length sw along an axis of length w (reflect pad, patch t):
    returns (starts, owner segment per index, local index per index).  A single
    segment when w <= sw."""
    import numpy as np
    halo = 2 * (t // 2)
    step = sw - 2 * halo
    if w <= sw:
        return [0], np.zeros(w, np.int64), np.arange(w)
    if step <= 0:
        raise ValueError("segments need length > 4 (T // 2)")
    starts = [0]
    while starts[-1] + sw < w:
        starts.append(min(starts[-1] + step, w - sw))
    owner = np.empty(w, np.int64)
    x = 0
    for s_, a in enumerate(starts):
        hi = w if s_ == len(starts) - 1 else a + sw - halo
        owner[x:hi] = s_
        x = max(x, hi)
    local = np.arange(w) - np.asarray(starts)[owner]
    return starts, owner, local


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of n items for rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_batch(batch: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    s, e = shard_range(batch.shape[0], world, rank)
    return batch[s:e]


def combine_partials(acc: torch.Tensor, used: int | torch.Tensor, group=None):
    """All-reduce(sum) of a rank's channel-sum map and used-channel count.

    One collective on an (h*w + 1) fp64 buffer.  Returns (sum map, total used):
    an int when ``used`` is an int, a 0-d device tensor (no host sync) when it
    is a tensor.
    """
    import torch.distributed as dist
    if isinstance(used, torch.Tensor):
        u = used.reshape(1).to(device=acc.device, dtype=torch.float64)
    else:
        u = torch.as_tensor([float(used)], dtype=torch.float64, device=acc.device)
    flat = torch.cat([acc.reshape(-1).to(torch.float64), u])
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    if isinstance(used, torch.Tensor):
        return flat[:-1].reshape(acc.shape), flat[-1]
    return flat[:-1].reshape(acc.shape), int(round(float(flat[-1])))


def channel_partial(values: torch.Tensor, cfg) -> tuple[torch.Tensor, int]:
    """Channel-sum map (h, w) fp64 and used-channel count for this rank's
    channel slice (C_local, h, w), fused path (scoring.py:258-281 without the
    division)."""
    acc, used, _ = _channel_partial(values, cfg)
    return acc, int(used[0])


def wide_supported(cfg, h: int, w: int, c: int) -> bool:
    """Planes wider than STRIP_W that the tiled fused path takes: the kernel
    scores a STRIP_H x STRIP_W tile, and strips() can cut the plane (a tile
    keeps the outputs more than 2 * (T // 2) from its inner edges, so that halo
    must leave a positive step along both axes)."""
    if not (USE_STRIPS and w > STRIP_W and cfg.pad == "reflect" and cfg.n_bins <= 256):
        return False
    halo = 2 * (cfg.patch_size // 2)
    if STRIP_W - 2 * halo <= 0 or (h > STRIP_H and STRIP_H - 2 * halo <= 0):
        return False
    L = N.lib()
    return L.qfca_score_groups_ex(min(h, STRIP_H), STRIP_W, cfg.n_bins, cfg.patch_size, c, 1, 0,
                                  N.PAD_CODES[cfg.pad], cfg.sample_budget, 1, 1) > 0


def _channel_partial(values: torch.Tensor, cfg):
    """channel_partial + the device non-finite flag of the slice."""
    from .scoring import _general_partial, fused_supported
    x = values.contiguous()
    c, h, w = x.shape
    hw = h * w
    L = N.lib()
    pad = N.PAD_CODES.get(cfg.pad, -1)

    def general():  # the reference's unfused route (any configuration), on the GPU
        acc, used, flag = _general_partial(x[None], cfg)
        return acc[0].reshape(h, w), used, flag

    if not fused_supported(cfg):
        return general()
    groups = L.qfca_score_groups_ex(h, w, cfg.n_bins, cfg.patch_size, c, 1, 0, pad,
                                    cfg.sample_budget, 0, 1)
    groups_k3 = L.qfca_score_groups_ex(h, w, cfg.n_bins, cfg.patch_size, c, 1, 0, pad,
                                       cfg.sample_budget, 1, 1)
    wide = wide_supported(cfg, h, w, c)
    if groups <= 0 and groups_k3 <= 0 and not wide:
        return general()
    s = N.stream()
    lo, hi, flag = minmax_dev(x, c, hw)
    bins = bins_dev(x, lo, hi, c, hw, cfg.n_bins)
    ref = None
    if bins.element_size() == 1 and wide:
        return _strip_partial(bins, lo, hi, cfg, c, h, w), _used(lo, hi, c), flag
    if groups <= 0:  # kernel without in-kernel reference selection: run K3 first
        groups = groups_k3
        ref = empty((c, cfg.n_bins), torch.int32)
        N.call("qfca_select_reference", bins.data_ptr(), bins.element_size(), lo.data_ptr(),
               hi.data_ptr(), c, h, w, cfg.n_bins, cfg.patch_size, pad, cfg.sample_budget, 0,
               ref.data_ptr(), s)
    partial = zeros((groups, hw), torch.float32)
    score_call(bins, lo, hi, ref, 1, c, h, w, cfg, groups, partial)
    used = empty((1,), torch.int32)
    N.call("qfca_count_used", lo.data_ptr(), hi.data_ptr(), 1, c, used.data_ptr(), s)
    ones = torch.ones((1,), dtype=torch.int32, device=x.device)
    acc = empty((1, hw), torch.float64)
    N.call("qfca_reduce_partials", partial.data_ptr(), 1, groups, hw, ones.data_ptr(),
           acc.data_ptr(), s)
    return acc.reshape(h, w), used, flag


_SCRATCH: dict = {}
TILES_IN_PLACE = True  # v6 reads the tiles of wide planes in place (False: gather first)


def _scratch(bins, h, w, cfg, c, images, groups, with_ref):
    """The cached per-stream scratch of the 128-column kernels (None: the chosen
    kernel needs none)."""
    L = N.lib()
    pad = N.PAD_CODES[cfg.pad]
    nbytes = L.qfca_score_scratch_bytes(h, w, cfg.n_bins, cfg.patch_size, c, images, groups, pad,
                                        cfg.sample_budget, 1 if with_ref else 0)
    if nbytes <= 0:
        return None
    key = (bins.device.index, torch.cuda.current_stream(bins.device).cuda_stream)
    scr = _SCRATCH.get(key)
    if scr is None or scr.numel() < nbytes:
        scr = torch.empty((nbytes,), dtype=torch.uint8, device=bins.device)
        _SCRATCH[key] = scr
    return scr


def score_call(bins, lo, hi, ref, images, c, h, w, cfg, groups, partial):
    """qfca_score_ex with a cached per-stream scratch (the 128-column kernel
    keeps each plane's window counts in it)."""
    pad = N.PAD_CODES[cfg.pad]
    scr = _scratch(bins, h, w, cfg, c, images, groups, ref is not None)
    nbytes = 0 if scr is None else scr.numel()
    N.call("qfca_score_ex", bins.data_ptr(), bins.element_size(), lo.data_ptr(), hi.data_ptr(),
           None if ref is None else ref.data_ptr(), images, c, h, w, cfg.n_bins, cfg.patch_size,
           pad, cfg.sample_budget, groups, None if scr is None else scr.data_ptr(),
           max(nbytes, 0), partial.data_ptr(), N.stream())


def _used(lo, hi, c) -> torch.Tensor:
    """(1,) int32 device count of non-degenerate channels (no host sync)."""
    used = empty((1,), torch.int32)
    N.call("qfca_count_used", lo.data_ptr(), hi.data_ptr(), 1, c, used.data_ptr(), N.stream())
    return used


def _strip_partial(bins, lo, hi, cfg, c, h, w) -> torch.Tensor:
    """Channel-sum map (h, w) fp64 of a wide plane from 128-column strips, cut
    into row bands of STRIP_H (same halo rule along rows), scored as one batch
    of tiles."""
    s = N.stream()
    pad = N.PAD_CODES[cfg.pad]
    cst, cown, cloc = strips(w, cfg.patch_size, STRIP_W)
    rst, rown, rloc = strips(h, cfg.patch_size, STRIP_H)
    th = min(h, STRIP_H)
    nt = len(rst) * len(cst)
    ref = empty((c, cfg.n_bins), torch.int32)  # whole-plane reference (K3)
    N.call("qfca_select_reference", bins.data_ptr(), bins.element_size(), lo.data_ptr(),
           hi.data_ptr(), c, h, w, cfg.n_bins, cfg.patch_size, pad, cfg.sample_budget, 0,
           ref.data_ptr(), s)
    ro, rl, co, cl, rst_d, cst_d = _tile_index(h, w, cfg.patch_size, bins.device, rst, rown,
                                               rloc, cst, cown, cloc)
    lo_r = lo.repeat(nt).contiguous()
    hi_r = hi.repeat(nt).contiguous()
    ref_r = ref.repeat(nt, 1).contiguous()
    L = N.lib()
    groups = L.qfca_score_groups_ex(th, STRIP_W, cfg.n_bins, cfg.patch_size, c, nt, 0, pad,
                                    cfg.sample_budget, 1, 1)
    if groups <= 0:
        raise NotImplementedError("no fused kernel for the tile shape")
    hw = th * STRIP_W
    partial = zeros((nt * groups, hw), torch.float32)
    # the 128-column kernel reads the tiles in place; else gather them first
    align = next((a for a in (16, 8, 4) if w % a == 0 and all(x % a == 0 for x in cst)), 0)
    st = N.QFCA_ERR_UNSUPPORTED
    if TILES_IN_PLACE and align and bins.element_size() == 1:
        scr = _scratch(bins, th, STRIP_W, cfg, c, nt, groups, True)
        nbytes = 0 if scr is None else scr.numel()
        st = L.qfca_score_tiles(bins.data_ptr(), 1, lo_r.data_ptr(), hi_r.data_ptr(),
                                ref_r.data_ptr(), c, h, w, rst_d.data_ptr(), len(rst),
                                cst_d.data_ptr(), len(cst), align, th, STRIP_W, cfg.n_bins,
                                cfg.patch_size, pad, cfg.sample_budget, groups,
                                None if scr is None else scr.data_ptr(), nbytes,
                                partial.data_ptr(), s)
    if st == N.QFCA_ERR_UNSUPPORTED:
        sb = empty((nt, c, th, STRIP_W), torch.uint8)
        if w % 4 == 0:
            N.call("qfca_gather_tiles", bins.data_ptr(), c, h, w, rst_d.data_ptr(), len(rst),
                   cst_d.data_ptr(), len(cst), th, STRIP_W, sb.data_ptr(), s)
        else:
            b3 = bins.view(c, h, w)
            sb.copy_(torch.stack([b3[:, r:r + th, a:a + STRIP_W] for r in rst for a in cst]))
        score_call(sb, lo_r, hi_r, ref_r, nt, c, th, STRIP_W, cfg, groups, partial)
    else:
        N.check(st, "qfca_score_tiles")
    ones = torch.ones((nt,), dtype=torch.int32, device=bins.device)
    acc = empty((nt, hw), torch.float64)
    N.call("qfca_reduce_partials", partial.data_ptr(), nt, groups, hw, ones.data_ptr(),
           acc.data_ptr(), s)
    a4 = acc.view(len(rst), len(cst), th, STRIP_W)
    return a4[ro, co, rl, cl].contiguous()  # (h, w)


_TILE_IDX: dict = {}


def _tile_index(h, w, t, dev, rst, rown, rloc, cst, cown, cloc):
    """Owner / local index tensors and tile starts of the decomposition, cached
    on the device."""
    key = (h, w, t, str(dev))
    if key not in _TILE_IDX:
        _TILE_IDX[key] = (torch.as_tensor(rown, device=dev)[:, None],
                          torch.as_tensor(rloc, device=dev)[:, None],
                          torch.as_tensor(cown, device=dev)[None, :],
                          torch.as_tensor(cloc, device=dev)[None, :],
                          torch.as_tensor(rst, dtype=torch.int32, device=dev),
                          torch.as_tensor(cst, dtype=torch.int32, device=dev))
    return _TILE_IDX[key]


def detect_channel_sharded(values_local: torch.Tensor, cfg=None, group=None):
    """Score one image whose channels are split across the ranks.

    ``values_local`` is this rank's (C_local, h, w) slice on its GPU.  Returns
    (scores (h, w) fp64, image_score, degenerate) on every rank; the last two
    are 0-d device tensors (float() / bool() them), so a step has no host sync.
    """
    from .scoring import PipelineConfig
    cfg = cfg or PipelineConfig()
    acc, used, _ = _channel_partial(values_local, cfg)
    total, used_all = combine_partials(acc, used, group)
    h, w = total.shape
    agg = total / used_all.clamp(min=1.0)  # all degenerate: the sum map is all zeros
    final = sep_convolve_dev(agg[None].contiguous(), _gauss_kernel(cfg.sigma_s), cfg.pad)[0] \
        if cfg.sigma_s > 0 else agg
    img = empty((1,), torch.float64)
    N.call("qfca_image_score", final.contiguous().data_ptr(), 1, h, w, cfg.border,
           img.data_ptr(), N.stream())
    return final, img[0], used_all == 0


# ---- QFCA+ on one huge image (option (a)) ----
#
# The covariance needs every channel of a pixel, so channel sharding alone
# cannot form it.  Features are replicated on every rank; the pixels are
# sharded for the two reductions of pca_fit (features.py:167-172): the channel
# sums (-> mean) and the centred Gram matrix, each combined with one
# all-reduce (C and C x C fp64).  The top-k eigenpairs are then formed
# identically on every rank, each rank takes the residual of its channel
# slice, and scoring continues as detect_channel_sharded (one more
# all-reduce of the channel-sum map).

COV_CHUNK = 16384  # pixels per exact int8-digit covariance block (cov_i8.cu bound)


def _world(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _all_reduce(t: torch.Tensor, group=None) -> torch.Tensor:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def local_pixels(values: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """This rank's contiguous pixel range of a (C, h, w) plane stack -> (C, n)."""
    c = values.shape[0]
    x = values.reshape(c, -1)
    p0, p1 = shard_range(x.shape[1], world, rank)
    return x[:, p0:p1].contiguous()


def channel_sums(xs: torch.Tensor) -> torch.Tensor:
    """(C, n) fp32 -> (C,) fp64 channel sums over the local pixels."""
    c, n = xs.shape
    m = empty((c,), torch.float64)
    N.call("qfca_plane_mean", xs.data_ptr(), c, n, m.data_ptr(), N.stream())
    return m * float(n)


def centred_gram(xs: torch.Tensor, mean: torch.Tensor) -> torch.Tensor:
    """sum over the local pixels of (x - mean)(x - mean)^T, (C, C) fp64.

    Blocks of COV_CHUNK pixels go through the exact int8-digit covariance
    (covariance_exact, batched over blocks, the global mean for every block);
    a ragged tail takes the same call on its own size."""
    from .features import covariance_exact
    c, n = xs.shape
    g = zeros((c, c), torch.float64)
    nf = n // COV_CHUNK
    if nf:
        blk = xs[:, :nf * COV_CHUNK].reshape(c, nf, COV_CHUNK).permute(1, 0, 2).contiguous()
        cov = covariance_exact(blk.view(nf, c, COV_CHUNK, 1),
                               mean.reshape(1, c).expand(nf, c).contiguous())
        g += cov.sum(0) * float(COV_CHUNK)
    r = n - nf * COV_CHUNK
    if r:
        tail = xs[:, nf * COV_CHUNK:].contiguous()
        g += covariance_exact(tail.view(1, c, r, 1), mean.reshape(1, c).contiguous())[0] * float(r)
    return g


def pca_fit_sharded(values: torch.Tensor, k: int, group=None):
    """pca_fit (features.py:157-180) of one (C, h, w) image replicated on every
    rank, pixel-sharded: -> (mean (C,), components (k, C), eigenvalues (k,))."""
    from .features import topk_eigh
    world, rank = _world(group)
    c = values.shape[0]
    hw = values[0].numel()
    if not 1 <= k <= c:
        raise ValueError(f"k must be in [1, {c}], got {k}")
    xs = local_pixels(values, world, rank)
    mean = _all_reduce(channel_sums(xs), group) / float(hw)
    cov = _all_reduce(centred_gram(xs, mean), group) / float(hw)
    evals, vecs = topk_eigh(cov[None], k)
    comps = vecs[0].transpose(0, 1).contiguous()  # (k, C)
    arg = comps.abs().argmax(dim=1, keepdim=True)
    sign = torch.where(torch.gather(comps, 1, arg) < 0, -1.0, 1.0).to(comps.dtype)
    return mean, comps * sign, evals[0].clamp(min=0.0)


def detect_pca_sharded(values: torch.Tensor, cfg=None, group=None):
    """QFCA+ (cfg.pca_components > 0) on one huge image: ``values`` is the full
    (C, h, w) stack on every rank.  Returns what detect_channel_sharded does."""
    import dataclasses

    from .features import pca_residual_slice
    from .scoring import PipelineConfig
    cfg = cfg or PipelineConfig()
    world, rank = _world(group)
    c = values.shape[0]
    if cfg.pca_components > 0:
        mean, comps, _ = pca_fit_sharded(values, min(cfg.pca_components, c), group)
        c0, c1 = shard_range(c, world, rank)
        local = pca_residual_slice(values[None].contiguous(), mean[None], comps[None], c0, c1)[0]
    else:
        c0, c1 = shard_range(c, world, rank)
        local = values[c0:c1].contiguous()
    return detect_channel_sharded(local, dataclasses.replace(cfg, pca_components=0), group)
