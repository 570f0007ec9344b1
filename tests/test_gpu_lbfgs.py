"""LBFGS adjoint baseline on the B200: the adjoint gradient
against central differences of the same forward map, the SPEC's trivial
cases, the generic L-BFGS on a convex quadratic, and a small control run."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_1608_01102_b200 import _lib, ao, fields, lbfgs
    _lib.load()
    return lbfgs, ao, fields


def setup(fields, ao, n=6, N=3, seed=0, r=1e-2):
    spec = fields.GridSpec(2, (n, n), 1.0 / n, "neumann")
    g = torch.Generator().manual_seed(seed)
    x = [(torch.arange(m, dtype=torch.float64) + 0.5) / m for m in spec.res]
    X, Y = torch.meshgrid(*x, indexing="ij")
    rho0 = torch.exp(-((X - 0.4) ** 2 + (Y - 0.5) ** 2) / 0.05).cuda()
    tgt = torch.exp(-((X - 0.6) ** 2 + (Y - 0.5) ** 2) / 0.05)
    kf = ao.KeyframeSet(N, {N: tgt})
    u = tuple((0.3 * torch.randn((N,) + spec.face_shape(k), generator=g, dtype=torch.float64)).cuda()
              for k in range(2))
    u = fields.zero_boundary_faces(spec, u)
    return spec, rho0, kf, u, g


def test_gradient_matches_central_differences(mods):
    """directional derivatives on 6^2 / N = 3 match to 1e-4."""
    lbfgs, ao, fields = mods
    spec, rho0, kf, u, g = setup(fields, ao)
    cfg = lbfgs.LbfgsConfig(dt=1.0 / 3, r=1e-2, sim_tol=1e-11)
    J, grad, _ = lbfgs.objective_and_gradient(spec, u, rho0, kf, cfg)
    for trial in range(3):
        d = fields.zero_boundary_faces(spec, tuple(torch.randn(c.shape, generator=g, dtype=torch.float64).cuda()
                                                   for c in u))
        eps = 1e-5
        up = tuple(a + eps * b for a, b in zip(u, d))
        um = tuple(a - eps * b for a, b in zip(u, d))
        Jp, _, _ = lbfgs.objective_and_gradient(spec, up, rho0, kf, cfg)
        Jm, _, _ = lbfgs.objective_and_gradient(spec, um, rho0, kf, cfg)
        fd = (Jp - Jm) / (2 * eps)
        an = fields.dot_fields(grad, d)
        print(f"[lbfgs] FD {fd:.10e} adjoint {an:.10e} rel {abs(fd - an) / abs(fd):.2e}")
        assert abs(fd - an) <= 1e-4 * abs(fd)


def test_regulariser_gradient_is_r_u(mods):
    """the force-regularisation term alone contributes r u."""
    lbfgs, ao, fields = mods
    spec, rho0, kf, u, _ = setup(fields, ao, seed=1)
    r = 0.37
    J1, g1, _ = lbfgs.objective_and_gradient(spec, u, rho0, kf, lbfgs.LbfgsConfig(dt=1.0 / 3, r=r))
    J0, g0, _ = lbfgs.objective_and_gradient(spec, u, rho0, kf, lbfgs.LbfgsConfig(dt=1.0 / 3, r=0.0))
    for a, b, c in zip(g1, g0, u):
        diff = (a - b - r * c).abs().max().item()
        assert diff <= 1e-12 * max(1.0, (r * c).abs().max().item())
    assert abs((J1 - J0) - 0.5 * r * fields.dot_fields(u, u)) <= 1e-12 * abs(J1)


def test_matched_unforced_rollout_is_stationary(mods):
    """u = 0 with the keyframe = the unforced rollout ->
    objective 0, gradient 0."""
    lbfgs, ao, fields = mods
    spec, rho0, _, u, _ = setup(fields, ao, seed=2)
    cfg = lbfgs.LbfgsConfig(dt=1.0 / 3, r=1.0)
    zero = tuple(torch.zeros_like(c) for c in u)
    rho = lbfgs.simulate(spec, zero, rho0, cfg)
    kf = ao.KeyframeSet(3, {3: rho[3].clone()})
    J, g, _ = lbfgs.objective_and_gradient(spec, zero, rho0, kf, cfg)
    assert J == 0.0
    assert all(float(c.abs().max()) == 0.0 for c in g)


def test_generic_lbfgs_on_convex_quadratic(mods):
    """convex quadratic in 100 variables -> gradient norm
    1e-10 within 50 iterations (A = Q Q^T / 400 + I, condition number ~2:
    with unit steps and history 8 the iteration count grows with the
    conditioning -- ~14 here, > 60 at condition 5)."""
    lbfgs, _, fields = mods
    gen = torch.Generator().manual_seed(3)
    Q = torch.randn(100, 100, generator=gen, dtype=torch.float64)
    A = (Q @ Q.T / 400 + torch.eye(100, dtype=torch.float64)).cuda()
    b = torch.randn(100, generator=gen, dtype=torch.float64).cuda()

    def fun(x):
        (v,) = x
        Av = A @ v
        return float(0.5 * v @ Av - b @ v), (Av - b,), None

    cfg = lbfgs.LbfgsConfig(dt=1.0, max_iter=50, grad_tol=1e-10)
    stop = lambda it, x, f, g, aux, prev, logs: logs[-1]["grad_inf"] <= 1e-10
    x, f, g, _, its, conv, logs = lbfgs.lbfgs(fun, (torch.zeros(100, dtype=torch.float64, device="cuda"),), cfg, stop)
    assert conv and its <= 50
    fs = [l["objective"] for l in logs]
    assert all(b <= a + 1e-12 * abs(a) for a, b in zip(fs, fs[1:]))


def test_minimize_reduces_the_objective(mods):
    """A small control problem (8^2 / N = 4): accepted iterates never
    increase the objective (Armijo) and the density moves
    toward the keyframe."""
    lbfgs, ao, fields = mods
    spec, rho0, kf, u, _ = setup(fields, ao, n=8, N=4, seed=4)
    cfg = lbfgs.LbfgsConfig(dt=0.25, r=1e-3, max_iter=15, eps_visual=1e-4)
    try:
        res = lbfgs.minimize(spec, rho0, kf, 1e-3, 0.25, cfg)
    except Exception as e:     # MaxIterations still carries the best iterate
        res = e.result
    J0, _, _ = lbfgs.objective_and_gradient(spec, tuple(torch.zeros_like(c) for c in u), rho0, kf, cfg)
    fs = [J0] + [l["objective"] for l in res.logs]
    assert all(b <= a for a, b in zip(fs, fs[1:]))
    assert res.objective < 0.5 * J0
