"""STFAS convergence on B200 (SPEC.md acceptance 1) and
converged-solution parity with the oracle (north_star: fp64 <= 1e-8 relative).
"""

import numpy as np
import pytest
import torch

from oracle import stfas
from problems import make_problem

pytestmark = pytest.mark.gpu


def run_gpu(pb, cycles, n_levels=99, dtype=torch.float64):
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=n_levels)
    s = nso.SpacetimeState.zeros(spec, pb.N, dtype)
    hier = nso.StfasHierarchy(spec, cfg, pb.N, dtype)
    hier.set_guide(pb.v0, pb.vstar)
    hist = [hier.residual_norms(s)[0]]
    for _ in range(cycles):
        hier.vcycle(s)
        hier.gauge_fix(s)
        hist.append(hier.residual_norms(s)[0])
    return s, hist


def test_resolution_independent_linear_rate():
    """Average reduction over cycles 2-6 <= 0.75 on 16^2/8, 32^2/8, 32^2/16
    with spread < 0.15 (SPEC acceptance 1)."""
    facs = []
    for n, N in [(16, 8), (32, 8), (32, 16)]:
        pb = make_problem(2, n=n, N=N, seed=100 + n + N)
        _, h = run_gpu(pb, 6)
        facs.append((h[6] / h[2]) ** 0.25)
    print("factors", facs)
    assert max(facs) <= 0.75
    assert max(facs) - min(facs) < 0.15


@pytest.mark.parametrize("bnd", ["neumann", "periodic"])
def test_converged_solution_matches_oracle(bnd):
    """Both solvers driven to ||f|| <= 1e-10: fields agree to 1e-8 relative."""
    pb = make_problem(2, n=16, N=6, boundary=bnd, seed=61)
    ref = stfas.solve_nso(pb, eps=1e-10, cycle_budget=60, n_levels=3)
    assert ref.converged
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    g = pb.g
    res = nso.solve_nso(GridSpec(g.dim, g.res, g.h, g.boundary),
                        nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=3), pb.v0, pb.vstar,
                        eps=1e-10, cycle_budget=60)
    V, PB, U, P = res.state.numpy()
    want = stfas.gauge_fix(ref.state)
    scale = max(np.max(np.abs(c)) for c in want.V + want.U)
    err = max(np.max(np.abs(a - b)) for a, b in zip(V + U, want.V + want.U))
    assert err <= 1e-8 * scale
    ax = tuple(range(1, P.ndim))
    f = lambda x: x - x.mean(axis=ax, keepdims=True)
    assert np.max(np.abs(f(P) - want.P)) <= 1e-8 * max(1.0, np.max(np.abs(want.P)))
    assert np.max(np.abs(f(PB) - want.PB)) <= 1e-8 * max(1.0, np.max(np.abs(want.PB)))


def test_colour_order_converges_to_same_solution():
    """north_star: colouring differences (red-black vs mod-2 vs mod-3)
    converge to the same solution within tolerance."""
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    pb = make_problem(2, n=24, N=4, seed=71, res=(24, 24))
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    out = []
    for rb, mod in ((True, 2), (False, 2), (False, 3)):
        r = nso.solve_nso(spec, nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, color_mod=mod, red_black=rb,
                                                n_levels=3),
                          pb.v0, pb.vstar, eps=1e-11, cycle_budget=80)
        out.append(r.state.numpy())
    a = out[0]
    scale = max(np.max(np.abs(c)) for c in a[0] + a[2])
    for b in out[1:]:
        err = max(np.max(np.abs(x - y)) for x, y in zip(a[0] + a[2], b[0] + b[2]))
        assert err <= 1e-8 * scale


def test_fp32_solution_bound():
    """fp32 mode: converged to a relative 1e-5 residual reduction, fields
    within 1e-4 relative of the fp64 solution (stated fp32 bound)."""
    pb = make_problem(2, n=16, N=6, seed=81)
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=3)
    r64 = nso.solve_nso(spec, cfg, pb.v0, pb.vstar, eps=1e-11, cycle_budget=80, dtype=torch.float64)
    r32 = nso.solve_nso(spec, cfg, pb.v0, pb.vstar, eps=1e-5, relative=True, cycle_budget=80,
                        dtype=torch.float32)
    a, b = r64.state.numpy(), r32.state.numpy()
    scale = max(np.max(np.abs(c)) for c in a[0] + a[2])
    err = max(np.max(np.abs(x - y)) for x, y in zip(a[0] + a[2], b[0] + b[2]))
    assert err <= 1e-4 * scale
