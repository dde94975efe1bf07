"""K4 v6 (csrc/score6.cu) against K4 v3 (csrc/score3.cu): v6 restates v3's
fp32 arithmetic sequence (transport, register ring, own-bin box, channel
order), so their partial maps must be BIT-IDENTICAL on every shape v6 takes
(128-wide planes and tiles, T in {1, 3, 5, 9, 15}, reflect / wrap, N <= 16,
in-kernel reference or a caller-supplied one, degenerate channels); v6 vs
the oracle is covered by test_gpu_parity.test_fused_kernel_versions_vs_oracle
and tests/test_bench_scale.py."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _partials(ver, bins, lo, hi, V, images, C, h, n, t, pad, groups):
    import torch
    from paper_2510_15602_b200 import _native as N
    L = N.lib()
    part = torch.zeros((images, groups, h * 128), dtype=torch.float32, device="cuda")
    N.call("qfca_set_score_kernel", ver)
    try:
        nbytes = L.qfca_score_scratch_bytes(h, 128, n, t, C, images, groups, pad, 4096,
                                            0 if V is None else 1)
        if ver == 6:
            assert nbytes > 0
        scr = torch.empty((max(nbytes, 1),), dtype=torch.uint8, device="cuda")
        N.call("qfca_score_ex", bins.data_ptr(), 1, lo.data_ptr(), hi.data_ptr(),
               None if V is None else V.data_ptr(), images, C, h, 128, n, t, pad, 4096,
               groups, scr.data_ptr() if ver == 6 else None, nbytes if ver == 6 else 0,
               part.data_ptr(), N.stream())
    finally:
        N.call("qfca_set_score_kernel", 0)
    return part.cpu().numpy()


@pytest.mark.parametrize("images,C,h,n,t,pad,ext", [
    (2, 12, 128, 16, 9, 1, False), (1, 8, 128, 16, 9, 2, False), (2, 6, 128, 16, 3, 1, False),
    (1, 5, 128, 16, 5, 2, False), (1, 7, 128, 8, 1, 1, False), (1, 6, 256, 16, 9, 1, False),
    (1, 5, 128, 16, 5, 1, True), (2, 6, 128, 12, 9, 1, True), (1, 4, 40, 16, 9, 1, False),
    (1, 6, 19, 5, 3, 2, False), (1, 4, 130, 2, 9, 1, False), (1, 5, 128, 16, 7, 1, False),
    (1, 5, 128, 16, 11, 2, False), (1, 4, 64, 16, 13, 1, True), (1, 4, 128, 16, 1, 1, False)])
def test_score6_bit_identical_to_score3(images, C, h, n, t, pad, ext):
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import quantize
    rng = np.random.default_rng(images * 1000 + C * 10 + h + t)
    x = np.maximum(rng.standard_normal((images, C, h, 128)) + 0.3, 0).astype(np.float32)
    x[0, 1] = 0.5  # a degenerate channel
    xd = torch.from_numpy(x).cuda().reshape(images * C, h * 128)
    lo, hi, _ = quantize.minmax_dev(xd, images * C, h * 128)
    bins = quantize.bins_dev(xd, lo, hi, images * C, h * 128, n)
    V = None
    if ext:
        cfg = Q.PipelineConfig(n_bins=n, patch_size=t, pad={1: "reflect", 2: "wrap"}[pad])
        V = quantize.reference_stats_dev(bins, lo, hi, images * C, h, 128, n, t, cfg.pad, 4096,
                                         "median-quan").contiguous()
        assert V.dtype == torch.int32
    groups = 2
    p3 = _partials(3, bins, lo, hi, V, images, C, h, n, t, pad, groups)
    p6 = _partials(6, bins, lo, hi, V, images, C, h, n, t, pad, groups)
    assert np.abs(p3).max() > 0
    np.testing.assert_array_equal(p6, p3)


@pytest.mark.parametrize("t,pad", [(15, "reflect"), (13, "reflect"), (5, "wrap")])
def test_score6_vs_oracle_where_v3_cannot(t, pad):
    """T = 15 on 128-wide planes: v3's row buffers do not fit shared memory, v6
    runs it (the reference comes from K3); the map matches the oracle."""
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native as N
    from oracle import qfca_oracle as O
    rng = np.random.default_rng(t)
    x = np.maximum(rng.standard_normal((1, 6, 128, 128)) + 0.3, 0).astype(np.float32)
    cfg = Q.PipelineConfig(patch_size=t, pad=pad)
    N.call("qfca_set_score_kernel", 6)
    try:
        res = Q.detect_batch(torch.from_numpy(x).cuda(), cfg)
    finally:
        N.call("qfca_set_score_kernel", 0)
    ref, img, _ = O.detect(x[0], patch_size=t, pad=pad)
    got = res.scores[0].cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("n,t,pad", [(17, 9, "reflect"), (31, 9, "reflect"), (32, 9, "wrap"),
                                     (46, 5, "reflect"), (64, 9, "reflect"), (64, 3, "wrap"),
                                     (48, 11, "reflect"), (100, 9, "reflect"),
                                     (128, 9, "wrap"), (256, 9, "reflect"), (256, 15, "reflect")])
def test_score6_bin_passes_vs_oracle(n, t, pad):
    """N > 16 on v6: bins in passes of 16 thermometer lanes (15 new bins per
    pass after the first, the G table rebuilt per pass, up to N = 256); maps
    match the oracle, the detect path uses v6."""
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native as N
    from oracle import qfca_oracle as O
    rng = np.random.default_rng(n * 10 + t)
    x = np.maximum(rng.standard_normal((2, 5, 128, 128)) + 0.3, 0).astype(np.float32)
    x[1, 2] = 0.25  # degenerate
    cfg = Q.PipelineConfig(n_bins=n, patch_size=t, pad=pad)
    L = N.lib()
    assert L.qfca_score_version(128, 128, n, t, 5, 2, N.PAD_CODES[pad], 4096, 0) == 6
    res = Q.detect_batch(torch.from_numpy(x).cuda(), cfg)
    for i in range(2):
        ref, img, _ = O.detect(x[i], n_bins=n, patch_size=t, pad=pad)
        got = res.scores[i].cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max(), (n, t, pad, i)
