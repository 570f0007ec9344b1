"""Host-side logic of the AO drop-in (no GPU): the per-axis filter matrices
and the keyframe / metric argument validation, against the oracle and the
reference's error behaviour (ao.py:27-45, :48-95)."""

import numpy as np
import pytest

from oracle import sim


@pytest.mark.parametrize("n,sigma,periodic", [(8, 1.0, True), (8, 1.0, False), (16, 4.0, False),
                                             (32, 8.0, True), (128, 32.0, False)])
def test_filter_matrix_matches_oracle(n, sigma, periodic):
    from paper_1608_01102_b200.ao import _filter_matrix
    m = _filter_matrix(n, sigma, periodic)
    assert np.array_equal(m, sim.axis_matrix(n, sigma, periodic))
    assert np.allclose(m.sum(axis=1), 1.0, rtol=0, atol=1e-14)


def test_keyframe_and_metric_validation():
    from paper_1608_01102_b200.ao import GaussianMetric, KeyframeSet
    from paper_1608_01102_b200.fields import GridSpec
    with pytest.raises(ValueError):
        KeyframeSet(3, {})
    with pytest.raises(ValueError):
        KeyframeSet(3, {0: np.zeros((8, 8))})
    with pytest.raises(ValueError):
        KeyframeSet(3, {1: -np.ones((8, 8))})
    kf = KeyframeSet(3, {1: np.zeros((8, 8)), 3: np.ones((8, 8))})
    assert list(kf.flags) == [False, True, False, True]
    spec = GridSpec(2, (16, 16), 1 / 16, "neumann")
    assert GaussianMetric(spec).levels == 3
    with pytest.raises(ValueError):
        GaussianMetric(spec, levels=0)
    with pytest.raises(ValueError):
        GaussianMetric(spec, levels=2, weights=(1.0,))


def test_fp32_ao_needs_a_reachable_projection_tolerance():
    """the reference's absolute projection_tol (1e-9) is below the
    fp32 floor; fp32 AO / ADMM is rejected up front instead of exhausting the
    Poisson budget on every frame."""
    import torch
    from paper_1608_01102_b200 import admm
    from paper_1608_01102_b200.ao import AoConfig, GaussianMetric, KeyframeSet, solve_ao
    from paper_1608_01102_b200.fields import GridSpec
    spec = GridSpec(2, (8, 8), 1 / 8)
    vg = tuple(torch.zeros((3,) + spec.face_shape(k), dtype=torch.float32) for k in range(2))
    rho0 = torch.zeros((8, 8), dtype=torch.float32)
    kf = KeyframeSet(3, {3: np.ones((8, 8))})
    with pytest.raises(ValueError, match="float32"):
        solve_ao(spec, vg, rho0, kf, None, AoConfig(K=1.0, dt=0.25))
    with pytest.raises(ValueError, match="float32"):
        admm.run(spec, rho0, kf, admm.AdmmConfig(dt=0.25), dtype=torch.float32)
