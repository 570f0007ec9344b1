"""GPU advection optimisation (ao.py drop-in) vs the reference's own outputs
and the oracle — B200.

Golden vectors come from the reference ``smokectrl.ao`` (tests/golden/
make_golden.py): the metric (2D both boundaries, 3D periodic with weights),
one ``ao_sweep`` (ao2p / ao2n) and ``solve_ao`` with and without the blending
safeguard (aos0 / aos1).  fp64, tolerances relative to the max.  The Taylor
orders must match exactly (adaptive truncation is part of the result).
"""

import numpy as np
import pytest
import torch

from conftest import GoldenCase, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_1608_01102_b200 import _lib, ao, fields
    _lib.load()
    return ao, fields


def test_axis_filter_all_axes(mods):
    """Each separable pass (plain, transposed, accumulated) against a
    host-side dense contraction, fp64 and fp32."""
    ao, F = mods
    from paper_1608_01102_b200 import _dev, _lib
    rng = np.random.default_rng(5)
    res = (6, 10, 12)
    x = rng.standard_normal(res)
    for k in range(3):
        n = res[k]
        m = rng.standard_normal((n, n))
        for tr in (0, 1):
            mm = m.T if tr else m
            want = np.moveaxis(np.tensordot(mm, x, axes=(1, k)), 0, k)
            y0 = rng.standard_normal(res)
            for dt, tol in ((torch.float64, 1e-14), (torch.float32, 1e-5)):
                xt = torch.from_numpy(x).to("cuda", dt)
                mt = torch.from_numpy(m).to("cuda", dt)
                yt = torch.from_numpy(y0).to("cuda", dt)
                outer, inner = int(np.prod(res[:k])), int(np.prod(res[k + 1:]))
                _lib.check(_lib.load().smk_axis_filter(_dev._DT[dt], outer, n, inner, mt.data_ptr(), tr, 0.5, 2.0,
                                                       xt.data_ptr(), yt.data_ptr(), _dev.stream()))
                assert rel_err(yt.double().cpu().numpy(), 0.5 * want + 2.0 * y0) < tol


def test_axis_filter_rejects_in_place(mods):
    from paper_1608_01102_b200 import _lib
    x = torch.zeros(8, device="cuda", dtype=torch.float64)
    m = torch.eye(8, device="cuda", dtype=torch.float64)
    rc = _lib.load().smk_axis_filter(_lib.SMK_F64, 1, 8, 1, m.data_ptr(), 0, 1.0, 0.0, x.data_ptr(), x.data_ptr(),
                                     None)
    assert rc == _lib.SMK_ERR_ARG


@pytest.mark.parametrize("tag", ["ao2p", "ao2n"])
def test_metric_and_sweep(golden, mods, tag):
    ao, F = mods
    c = GoldenCase(golden, tag)
    spec = F.GridSpec(2, (8, 8), 0.125, "periodic" if tag.endswith("p") else "neumann")
    metric = ao.GaussianMetric(spec)
    assert rel_err(metric.apply(c["rho0"] - c["target"]), c["metric_apply"]) < 1e-13
    guiding = c.comps("guiding")
    n = guiding[0].shape[0]
    state = ao.AoState(vstar=tuple(x.copy() for x in guiding), mu=np.zeros((n,) + spec.res),
                       rho=np.broadcast_to(c["rho0"], (n + 1,) + spec.res).copy())
    kf = ao.KeyframeSet(n, {n: c["target"]})
    res = ao.ao_sweep(spec, state, guiding, kf, metric, ao.AoConfig(K=10.0, dt=0.5))
    assert list(res.ks) == [int(k) for k in c["ks"]]
    assert rel_err(res.rho, c["rho"]) < 1e-12
    assert rel_err(res.mu, c["mu"]) < 1e-12
    assert rel_err(res.vstar, c.comps("vstar")) < 1e-10


def test_metric_3d_periodic_weights(golden, mods):
    ao, F = mods
    c = GoldenCase(golden, "met3")
    spec = F.GridSpec(3, (8, 8, 16), 0.125, "periodic")
    metric = ao.GaussianMetric(spec, levels=2, weights=(1.0, 0.5))
    assert rel_err(metric.apply(c["x"]), c["apply"]) < 1e-13
    assert abs(metric.quad(c["x"]) - float(c["quad"])) <= 1e-13 * float(c["quad"])
    # device tensors in, device tensors out
    xt = torch.from_numpy(c["x"]).cuda()
    out = metric.apply(xt)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert rel_err(out.cpu().numpy(), c["apply"]) < 1e-13


@pytest.mark.parametrize("tag,safeguard,iters", [("aos0", False, 2), ("aos1", True, 3)])
def test_solve_ao(golden, mods, tag, safeguard, iters):
    ao, F = mods
    c = GoldenCase(golden, tag)
    spec = F.GridSpec(2, (8, 8), 0.125, "neumann")
    guiding = c.comps("guiding")
    n = guiding[0].shape[0]
    kf = ao.KeyframeSet(n, {2: c["t2"], 4: c["t4"]})
    metric = ao.GaussianMetric(spec)
    cfg = ao.AoConfig(K=5.0, dt=0.5, iters=iters, safeguard=safeguard)
    obj0 = ao.ao_objective(spec, guiding, guiding, kf, metric, cfg, c["rho0"])
    assert abs(obj0 - float(c["obj0"])) <= 1e-12 * abs(float(c["obj0"]))
    res = ao.solve_ao(spec, guiding, c["rho0"], kf, metric, cfg)
    assert list(res.ks) == [int(k) for k in c["ks"]]
    assert rel_err(res.vstar, c.comps("vstar")) < 1e-10
    assert rel_err(res.mu, c["mu"]) < 1e-10
    assert rel_err(res.rho, c["rho"]) < 1e-11
    obj = ao.ao_objective(spec, res.vstar, guiding, kf, metric, cfg, c["rho0"])
    assert abs(obj - float(c["obj"])) <= 1e-10 * abs(float(c["obj"]))


def test_solve_ao_3d_vs_oracle(mods):
    """3D Neumann 8^3, two sweeps with the safeguard, against the oracle."""
    ao, F = mods
    from oracle import ops, sim
    from oracle.grid import Grid
    g = Grid(3, (8, 8, 8), 0.125, "neumann")
    spec = F.GridSpec(3, (8, 8, 8), 0.125, "neumann")
    rng = np.random.default_rng(41)
    n = 3
    frames = []
    for _ in range(n):
        comps = tuple(0.2 * rng.standard_normal(g.face_shape(k)) for k in range(3))
        frames.append(ops.project(g, ops.zero_walls(g, comps), 1e-11))
    guiding = tuple(np.stack([f[k] for f in frames]) for k in range(3))
    xs = np.meshgrid(*[(np.arange(8) + 0.5) / 8] * 3, indexing="ij")
    rho0 = np.exp(-((xs[0] - 0.4) ** 2 + (xs[1] - 0.5) ** 2 + (xs[2] - 0.5) ** 2) / 0.03)
    target = np.exp(-((xs[0] - 0.6) ** 2 + (xs[1] - 0.5) ** 2 + (xs[2] - 0.5) ** 2) / 0.03)
    om = sim.GaussianMetric(g)
    vs, mu, rho, ks = sim.solve_ao(g, guiding, rho0, {n: target}, om, 4.0, 0.25, 2, True)
    res = ao.solve_ao(spec, guiding, rho0, ao.KeyframeSet(n, {n: target}), ao.GaussianMetric(spec),
                      ao.AoConfig(K=4.0, dt=0.25, iters=2, safeguard=True))
    assert list(res.ks) == list(ks)
    assert rel_err(res.vstar, vs) < 1e-10
    assert rel_err(res.mu, mu) < 1e-10
    assert rel_err(res.rho, rho) < 1e-11


def test_keyframe_validation(mods):
    ao, F = mods
    with pytest.raises(ValueError):
        ao.KeyframeSet(3, {})
    with pytest.raises(ValueError):
        ao.KeyframeSet(3, {4: np.zeros((8, 8))})
    with pytest.raises(ValueError):
        ao.KeyframeSet(3, {2: -np.ones((8, 8))})
    with pytest.raises(ValueError):
        ao.GaussianMetric(F.GridSpec(2, (8, 8), 0.125, "neumann"), levels=2, weights=(1.0,))
