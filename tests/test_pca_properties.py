"""The reference's PCA property tests (pkg/tests/test_features.py:83-170 and
acceptance A9, pkg/tests/test_acceptance.py:300-321) run against the GPU
path: pca_fit (int8-digit covariance + Lanczos / Jacobi eigensolver) and
pca_residual (fp64 tensor-core contractions) through the package's drop-in
API, with the reference's inputs and bounds."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _fm(values, scale=1):
    from paper_2510_15602_b200 import FeatureMap
    return FeatureMap(values=np.asarray(values, dtype=np.float32), scale=scale)


def test_pca_constant_features_zero_eigenvalues():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    f = _fm(np.full((3, 8, 8), 2.0))
    m = pca_fit(f, 2)
    np.testing.assert_allclose(m.eigenvalues, 0.0, atol=1e-9)
    r = pca_residual(f, m)
    np.testing.assert_allclose(r.values, 0.0, atol=1e-6)


def test_pca_two_channel_line():
    from paper_2510_15602_b200 import pca_fit
    rng = np.random.default_rng(2)
    t = rng.standard_normal(256)
    f = _fm(np.stack([(t + 0.5).reshape(16, 16), (2 * t - 1.0).reshape(16, 16)]))
    m = pca_fit(f, 1)
    np.testing.assert_allclose(np.abs(m.components[0]), np.array([1.0, 2.0]) / np.sqrt(5),
                               atol=1e-4)
    full = pca_fit(f, 2)
    assert full.eigenvalues[1] == pytest.approx(0.0, abs=1e-6)


def test_full_rank_pca_lossless():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    rng = np.random.default_rng(3)
    f = _fm(rng.standard_normal((6, 12, 12)))
    r = pca_residual(f, pca_fit(f, 6))
    assert np.max(np.abs(r.values)) <= 1e-4


def test_residual_orthogonality():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    rng = np.random.default_rng(4)
    f = _fm(rng.standard_normal((10, 16, 16)))
    m = pca_fit(f, 4)
    r = pca_residual(f, m)
    x = f.values.reshape(10, -1).astype(np.float64)
    rr = r.values.reshape(10, -1).astype(np.float64)
    proj = m.components @ rr
    bound = 1e-4 * (1.0 + np.linalg.norm(x - m.mean[:, None], axis=0))
    assert np.all(np.linalg.norm(proj, axis=0) <= bound)


def test_residual_energy_monotone_in_k():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    rng = np.random.default_rng(5)
    f = _fm(rng.standard_normal((8, 16, 16)))
    energies = [float(np.sum(pca_residual(f, pca_fit(f, k)).values.astype(np.float64) ** 2))
                for k in range(1, 9)]
    assert all(a >= b - 1e-6 for a, b in zip(energies, energies[1:]))


def test_residual_idempotent_on_top_directions():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    rng = np.random.default_rng(6)
    f = _fm(rng.standard_normal((6, 20, 20)))
    m = pca_fit(f, 3)
    refit = pca_fit(pca_residual(f, m), 6)
    proj_var = (m.components @ refit.components.T) ** 2 @ refit.eigenvalues
    assert np.max(proj_var) <= 1e-8 * max(1.0, refit.eigenvalues[0])


def test_pca_k_out_of_range_and_channel_mismatch():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    f = _fm(np.zeros((3, 4, 4)))
    with pytest.raises(ValueError):
        pca_fit(f, 4)
    m = pca_fit(f, 2)
    with pytest.raises(ValueError):
        pca_residual(_fm(np.zeros((4, 4, 4))), m)


def test_component_sign_convention():
    from paper_2510_15602_b200 import pca_fit
    rng = np.random.default_rng(7)
    f = _fm(rng.standard_normal((5, 12, 12)))
    m = pca_fit(f, 5)
    for row in m.components:
        assert row[np.argmax(np.abs(row))] > 0
    np.testing.assert_allclose(m.components @ m.components.T, np.eye(5), atol=1e-5)
    assert np.all(np.diff(m.eigenvalues) <= 1e-12)


def test_a9_pca_properties():
    from paper_2510_15602_b200 import pca_fit, pca_residual
    rng = np.random.default_rng(9)
    f = _fm(rng.standard_normal((12, 24, 24)))
    x = f.values.reshape(12, -1).astype(np.float64)
    model = pca_fit(f, 5)
    res = pca_residual(f, model).values.reshape(12, -1).astype(np.float64)
    proj = np.linalg.norm(model.components @ res, axis=0)
    bound = 1e-4 * (1.0 + np.linalg.norm(x - model.mean[:, None], axis=0))
    assert np.all(proj <= bound)
    full = pca_residual(f, pca_fit(f, 12)).values
    assert float(np.max(np.abs(full))) <= 1e-4
    energies = [float(np.sum(pca_residual(f, pca_fit(f, k)).values.astype(np.float64) ** 2))
                for k in range(1, 13)]
    assert all(a >= b - 1e-6 for a, b in zip(energies, energies[1:]))


def test_pca_properties_at_bench_width():
    """The same properties on the bench's 512-channel WRN features (the
    Lanczos route, k = 10)."""
    import torch
    from paper_2510_15602_b200 import FeatureMap, pca_fit, pca_residual
    import workloads
    with torch.no_grad():
        feats, _ = workloads.make_features(1, 512, seed=21)
    f = FeatureMap(values=feats[0].cpu().numpy(), scale=8)
    m = pca_fit(f, 10)
    np.testing.assert_allclose(m.components @ m.components.T, np.eye(10), atol=1e-9)
    assert np.all(np.diff(m.eigenvalues) <= 1e-12)
    for row in m.components:
        assert row[np.argmax(np.abs(row))] > 0
    x = f.values.reshape(512, -1).astype(np.float64)
    r = pca_residual(f, m).values.reshape(512, -1).astype(np.float64)
    proj = np.linalg.norm(m.components @ r, axis=0)
    assert np.all(proj <= 1e-4 * (1.0 + np.linalg.norm(x - m.mean[:, None], axis=0)))
