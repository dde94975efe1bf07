"""Pooling API (reference pooling.py:20-172) on the GPU against goldens made by
running the reference (tests/golden/make_pooling_golden.py), bit-exact, plus
the reference's own hand-computed cases (pkg/tests/test_pooling.py:8-106)."""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pooling.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def _split(key):
    return key.split("/")


def test_pooling_golden_is_self_consistent(gold):
    """CPU: the reference's SAT box average equals its naive oracle (<= 1e-12),
    so the fixture is what the reference computes (test_pooling.py:59-66)."""
    n = 0
    for key, v in gold.items():
        kind, *rest = _split(key)
        if kind != "avg":
            continue
        nv = gold["naive/" + "/".join(rest)]
        assert np.allclose(v, nv, rtol=0, atol=1e-9 * max(1.0, np.abs(nv).max())), key
        n += 1
    assert n > 100


@pytest.mark.gpu
def test_pad_plane_bit_exact(gold):
    from paper_2510_15602_b200 import pad_plane
    n = 0
    for key, ref in gold.items():
        kind, *rest = _split(key)
        if kind != "pad":
            continue
        name, pad, margin = rest
        got = pad_plane(gold[f"in/{name}"], int(margin), pad)
        assert got.dtype == ref.dtype and np.array_equal(got, ref), key
        n += 1
    assert n == 9 * 3 * 4


@pytest.mark.gpu
def test_build_sat_and_box_sum_bit_exact(gold):
    from paper_2510_15602_b200 import box_sum, build_sat
    for key, ref in gold.items():
        kind, *rest = _split(key)
        if kind != "sat":
            continue
        name, pad, margin = rest
        p = gold[f"in/{name}"]
        sat = build_sat(p, margin=int(margin), pad=pad)
        assert (sat.height, sat.width, sat.margin) == (p.shape[0], p.shape[1], int(margin))
        assert sat.cumsum.dtype == np.float64 and np.array_equal(sat.cumsum, ref), key
        for k in (1, 3, 5):
            bk = f"boxsum/{name}/{pad}/{margin}/{k}"
            if bk not in gold:
                continue
            got = [box_sum(sat, cx, cy, k, pad=pad)
                   for cx in range(p.shape[0]) for cy in range(p.shape[1])]
            assert np.array_equal(np.asarray(got), gold[bk]), bk


@pytest.mark.gpu
def test_box_average_and_naive_bit_exact(gold):
    from paper_2510_15602_b200 import box_average, naive_box_average
    n = 0
    for key, ref in gold.items():
        kind, *rest = _split(key)
        if kind not in ("avg", "naive"):
            continue
        name, pad, k = rest
        fn = box_average if kind == "avg" else naive_box_average
        got = fn(gold[f"in/{name}"], int(k), pad)
        assert got.dtype == np.float64 and np.array_equal(got, ref), key
        n += 1
    assert n == 2 * 9 * 3 * 5


@pytest.mark.gpu
def test_box_average_stack_bit_exact(gold):
    """Includes (B, 1, w) and (B, h, 1) stacks: np.pad reflects a length-1 axis
    onto itself while box_average's pad_plane switches both axes to 'edge'."""
    from paper_2510_15602_b200 import box_average_stack
    n = 0
    for key, ref in gold.items():
        kind, *rest = _split(key)
        if kind != "stack":
            continue
        name, pad, k = rest
        got = box_average_stack(gold[f"in/{name}"], int(k), pad)
        assert np.array_equal(got, ref), key
        n += 1
    assert n == 4 * 3 * 4


@pytest.mark.gpu
def test_pooling_hand_cases_and_errors():
    """pkg/tests/test_pooling.py:8-56 hand values; the same errors."""
    import torch
    from paper_2510_15602_b200 import box_average, box_average_stack, box_sum, build_sat
    assert np.array_equal(build_sat(np.array([[5.0]])).cumsum, [[0, 0], [0, 5]])
    assert np.array_equal(build_sat(np.array([[1.0, 2.0], [3.0, 4.0]])).cumsum,
                          [[0, 0, 0], [0, 1, 3], [0, 4, 10]])
    sat = build_sat(np.ones((3, 3)))
    assert box_sum(sat, 1, 1, 3, pad="zero") == 9.0
    assert box_sum(sat, 0, 0, 3, pad="zero") == 4.0
    assert box_sum(build_sat(np.ones((3, 3)), margin=1, pad="reflect"), 0, 0, 3,
                   pad="reflect") == 9.0
    with pytest.raises(ValueError):
        box_sum(sat, 1, 1, 2)
    with pytest.raises(ValueError):
        box_sum(sat, 3, 0, 3)
    with pytest.raises(ValueError):
        box_sum(sat, 1, 1, 3, pad="reflect")  # margin 0 < 1
    np.testing.assert_allclose(box_average(np.array([[1.0, 2.0], [3.0, 4.0]]), 3, "reflect"),
                               np.array([[27.0, 24.0], [21.0, 18.0]]) / 9.0)
    with pytest.raises(ValueError):
        box_average(np.ones((4, 4)), 4)
    with pytest.raises(KeyError):
        box_average_stack(np.ones((1, 4, 4)), 3, "mirror")
    # device tensors stay on the device; the stack equals per-plane box_average
    rng = np.random.default_rng(3)
    st = rng.standard_normal((5, 17, 19))
    dev = box_average_stack(torch.from_numpy(st).cuda(), 7, "wrap")
    assert dev.is_cuda
    for i in range(5):
        assert np.array_equal(dev[i].cpu().numpy(), box_average(st[i], 7, "wrap"))
