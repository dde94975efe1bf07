"""K4 v7 (csrc/score7.cu): large patches (T = 17 .. 65) on 128-wide planes and
tiles, exact fp64 2D-prefix association.  v7 is not bit-identical to the
ring kernels (different summation order), so it is checked against the CPU
oracle (max-abs <= 1e-4 x max|ref|, the SURVEY 8(c) bar) and against v5 (the
previous large-T kernel) on the same bins and reference."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _features(seed, images, C, h, w=128):
    rng = np.random.default_rng(seed)
    x = np.maximum(rng.standard_normal((images, C, h, w)) + 0.3, 0).astype(np.float32)
    # low-frequency structure so that large windows see varied histograms
    yy, xx = np.mgrid[0:h, 0:w]
    x[:, ::2] += (0.5 * np.sin(yy / 9.0) * np.cos(xx / 13.0)).astype(np.float32)
    x[0, 1] = 0.5  # a degenerate channel
    return x


@pytest.mark.parametrize("t,h,n,pad", [
    (17, 128, 16, "reflect"), (33, 128, 16, "reflect"), (65, 128, 16, "reflect"),
    (21, 128, 16, "wrap"), (65, 128, 16, "wrap"), (33, 100, 16, "reflect"),
    (65, 40, 8, "reflect"), (25, 128, 5, "reflect"), (19, 128, 2, "reflect"),
    (45, 77, 13, "wrap"),
    # bin passes (N > 16): 15 new bins per pass after the first
    (17, 128, 17, "reflect"), (33, 128, 32, "reflect"), (21, 100, 64, "wrap"),
    (65, 40, 48, "reflect"), (33, 128, 100, "reflect")])
def test_score7_vs_oracle(t, h, n, pad):
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native as N
    from oracle import qfca_oracle as O
    x = _features(t * 7 + h + n, 1, 6, h)
    cfg = Q.PipelineConfig(n_bins=n, patch_size=t, pad=pad)
    L = N.lib()
    ver = L.qfca_score_version(h, 128, n, t, 6, 1, N.PAD_CODES[pad], cfg.sample_budget, 1)
    assert ver == 7
    res = Q.detect_batch(torch.from_numpy(x).cuda(), cfg)
    ref, img, _ = O.detect(x[0], n_bins=n, patch_size=t, pad=pad)
    got = res.scores[0].cpu().numpy()
    assert np.abs(ref).max() > 0
    print(f"T={t} h={h} N={n} {pad}: max|err| / max|ref| = "
          f"{np.abs(got - ref).max() / np.abs(ref).max():.2e}")
    assert np.abs(got - ref).max() <= TOL * np.abs(ref).max()
    assert abs(float(res.image_scores[0]) - img) <= TOL * np.abs(ref).max()


@pytest.mark.parametrize("t", [17, 33, 65])
def test_score7_close_to_score5(t):
    """Same bins, same K3 reference: v7's partial maps agree with v5's (fp32
    ring sums) to fp32 rounding."""
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native as N
    from paper_2510_15602_b200 import quantize
    images, C, h, n = 2, 5, 128, 16
    x = _features(t, images, C, h)
    xd = torch.from_numpy(x).cuda().reshape(images * C, h * 128)
    lo, hi, _ = quantize.minmax_dev(xd, images * C, h * 128)
    bins = quantize.bins_dev(xd, lo, hi, images * C, h * 128, n)
    V = quantize.reference_stats_dev(bins, lo, hi, images * C, h, 128, n, t, "reflect", 4096,
                                     "median-quan").contiguous()
    L = N.lib()
    out = {}
    for ver in (5, 7):
        N.call("qfca_set_score_kernel", ver)
        try:
            groups = L.qfca_score_groups_ex(h, 128, n, t, C, images, 1, 1, 4096, 1, 1)
            assert groups == 1
            nbytes = L.qfca_score_scratch_bytes(h, 128, n, t, C, images, 1, 1, 4096, 1)
            scr = torch.empty((max(nbytes, 1),), dtype=torch.uint8, device="cuda")
            part = torch.zeros((images, 1, h * 128), dtype=torch.float32, device="cuda")
            N.call("qfca_score_ex", bins.data_ptr(), 1, lo.data_ptr(), hi.data_ptr(),
                   V.data_ptr(), images, C, h, 128, n, t, 1, 4096, 1,
                   scr.data_ptr() if nbytes > 0 else None, max(nbytes, 0), part.data_ptr(),
                   N.stream())
            out[ver] = part.cpu().numpy()
        finally:
            N.call("qfca_set_score_kernel", 0)
    assert np.abs(out[5]).max() > 0
    assert np.abs(out[7] - out[5]).max() <= 2e-5 * np.abs(out[5]).max()


def test_score7_batch_matches_single():
    """Several images per launch (one CTA per image x channel group) give the
    per-image maps, independent of batch position."""
    import torch
    import paper_2510_15602_b200 as Q
    x = _features(5, 3, 8, 128)
    cfg = Q.PipelineConfig(patch_size=33)
    xd = torch.from_numpy(x).cuda()
    both = Q.detect_batch(xd, cfg).scores.cpu().numpy()
    for i in range(3):
        one = Q.detect_batch(xd[i:i + 1].contiguous(), cfg).scores.cpu().numpy()
        np.testing.assert_array_equal(both[i], one[0])


@pytest.mark.parametrize("t,h,n,pad,budget", [
    (33, 128, 16, 1, 4096), (17, 128, 12, 2, 4096), (65, 100, 16, 1, 4096),
    (21, 128, 16, 1, 1000), (45, 60, 7, 2, 4096), (33, 128, 40, 1, 4096)])
def test_score7_inkernel_reference_equals_k3(t, h, n, pad, budget):
    """v7 selecting the reference itself (sample sweep over its own window
    counts + packed-compare order statistic) gives K3's reference exactly:
    the partial maps with and without the caller's K3 reference are
    bit-identical."""
    import torch
    from paper_2510_15602_b200 import _native as N
    from paper_2510_15602_b200 import quantize
    images, C = 2, 5
    x = _features(t + h + budget, images, C, h)
    xd = torch.from_numpy(x).cuda().reshape(images * C, h * 128)
    lo, hi, _ = quantize.minmax_dev(xd, images * C, h * 128)
    bins = quantize.bins_dev(xd, lo, hi, images * C, h * 128, n)
    padname = {1: "reflect", 2: "wrap"}[pad]
    V = quantize.reference_stats_dev(bins, lo, hi, images * C, h, 128, n, t, padname, budget,
                                     "median-quan").contiguous()
    L = N.lib()
    out = []
    for ref in (V, None):
        N.call("qfca_set_score_kernel", 7)
        try:
            groups = L.qfca_score_groups_ex(h, 128, n, t, C, images, 1, pad, budget,
                                            0 if ref is None else 1, 1)
            assert groups == 1
            nbytes = L.qfca_score_scratch_bytes(h, 128, n, t, C, images, 1, pad, budget,
                                                0 if ref is None else 1)
            assert nbytes > 0
            scr = torch.empty((nbytes,), dtype=torch.uint8, device="cuda")
            part = torch.zeros((images, 1, h * 128), dtype=torch.float32, device="cuda")
            N.call("qfca_score_ex", bins.data_ptr(), 1, lo.data_ptr(), hi.data_ptr(),
                   None if ref is None else ref.data_ptr(), images, C, h, 128, n, t, pad,
                   budget, 1, scr.data_ptr(), nbytes, part.data_ptr(), N.stream())
            out.append(part.cpu().numpy())
        finally:
            N.call("qfca_set_score_kernel", 0)
    assert np.abs(out[0]).max() > 0
    np.testing.assert_array_equal(out[1], out[0])
