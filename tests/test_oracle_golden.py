"""Pin the oracle restatement to the reference's own outputs (CPU).

Golden vectors were produced by running the reference implementation
(``tests/golden/make_golden.py``); nothing here reads /root/reference.
"""

import numpy as np
import pytest

from conftest import GoldenCase, rel_err
from oracle import ops, sim

TAGS = ["n2p", "n2n", "r2n", "n3n", "n3p"]


@pytest.fixture(params=TAGS)
def case(request, golden):
    return GoldenCase(golden, request.param)


def test_div_grad(case):
    g = case.grid()
    assert rel_err(ops.div(g, case.comps("w")), case["div"]) < 1e-14
    assert rel_err(ops.grad(g, case["rho"]), case.comps("grad")) < 1e-14


def test_transport_and_taylor(case):
    g = case.grid()
    v, rho, mu = case.comps("v"), case["rho"], case["mu"]
    assert rel_err(ops.transport_scalar(g, v, rho), case["T"]) < 1e-14
    out, k, _ = ops.taylor(g, v, rho, 0.1)
    assert k == int(case["adv_k"])
    assert rel_err(out, case["adv"]) < 1e-13
    back, _, _ = ops.taylor(g, v, mu, 0.1, k_fixed=k, transpose=True)
    assert rel_err(back, case["advT"]) < 1e-13
    assert rel_err(ops.advect_v_T(g, v, rho, mu, 0.1, k), case.comps("advvT")) < 1e-13


def test_self_advection_family(case):
    g = case.grid()
    v, w, u = case.comps("v"), case.comps("w"), case.comps("u")
    assert rel_err(ops.transport_face(g, v, w), case.comps("S")) < 1e-14
    assert rel_err(ops.self_advection(g, v), case.comps("Sself")) < 1e-14
    assert rel_err(ops.jac_apply(g, v, w), case.comps("J")) < 1e-14
    assert rel_err(ops.jac_T_apply(g, v, u), case.comps("JT")) < 1e-13


def test_transfers_projection_poisson(case):
    g = case.grid()
    rho = case["rho"]
    assert rel_err(ops.restrict_cell(g, rho), case["rc"]) < 1e-15
    if case.has("pc"):
        gc = g.coarsen()
        assert rel_err(ops.prolong_cell(gc, ops.restrict_cell(g, rho)), case["pc"]) < 1e-15
    assert rel_err(ops.project(g, case.comps("w"), 1e-9), case.comps("proj")) < 1e-12
    p = ops.solve_poisson(g, case["mu"], 1e-9)
    want = case["pois"]
    assert rel_err(p - p.mean(), want - want.mean()) < 1e-10


def test_semi_lagrangian(case):
    g = case.grid()
    out = ops.semi_lagrangian(g, case.comps("v"), np.abs(case["rho"]), 0.3)
    assert rel_err(out, case["sl"]) < 1e-14


def test_sim_step(case):
    g = case.grid()
    v, p, rho, info = sim.step(g, case.comps("v"), np.abs(case["rho"]), case.comps("su"),
                               0.1, accept_stall=True)
    assert rel_err(v, case.comps("step_v")) < 1e-12
    assert rel_err(rho, case["step_rho"]) < 1e-13
    want = case["step_p"]
    assert rel_err(p - p.mean(), want - want.mean()) < 1e-9


@pytest.mark.parametrize("tag", ["ao2p", "ao2n"])
def test_ao_sweep(golden, tag):
    from oracle.grid import Grid
    c = GoldenCase(golden, tag)
    bnd = "periodic" if tag.endswith("p") else "neumann"
    g = Grid(2, (8, 8), 0.125, bnd)
    guiding = c.comps("guiding")
    target = c["target"]
    metric = sim.GaussianMetric(g)
    assert rel_err(metric.apply(c["rho0"] - target), c["metric_apply"]) < 1e-13
    vs, mu, rho, ks = sim.ao_sweep(g, guiding, guiding, c["rho0"], {3: target}, metric,
                                   10.0, 0.5)
    assert list(ks) == [int(k) for k in c["ks"]]
    assert rel_err(rho, c["rho"]) < 1e-12
    assert rel_err(mu, c["mu"]) < 1e-12
    assert rel_err(vs, c.comps("vstar")) < 1e-10


@pytest.mark.parametrize("tag,safeguard,iters", [("aos0", False, 2), ("aos1", True, 3)])
def test_solve_ao(golden, tag, safeguard, iters):
    from oracle.grid import Grid
    c = GoldenCase(golden, tag)
    g = Grid(2, (8, 8), 0.125, "neumann")
    guiding = c.comps("guiding")
    targets = {2: c["t2"], 4: c["t4"]}
    metric = sim.GaussianMetric(g)
    obj0 = sim.ao_objective(g, guiding, guiding, c["rho0"], targets, metric, 5.0, 0.5)
    assert abs(obj0 - float(c["obj0"])) <= 1e-13 * abs(float(c["obj0"]))
    vs, mu, rho, ks = sim.solve_ao(g, guiding, c["rho0"], targets, metric, 5.0, 0.5, iters, safeguard)
    assert list(ks) == [int(k) for k in c["ks"]]
    assert rel_err(vs, c.comps("vstar")) < 1e-10
    assert rel_err(mu, c["mu"]) < 1e-10
    assert rel_err(rho, c["rho"]) < 1e-11
    obj = sim.ao_objective(g, vs, guiding, c["rho0"], targets, metric, 5.0, 0.5)
    assert abs(obj - float(c["obj"])) <= 1e-10 * abs(float(c["obj"]))


def test_metric_3d_periodic(golden):
    from oracle.grid import Grid
    c = GoldenCase(golden, "met3")
    g = Grid(3, (8, 8, 16), 0.125, "periodic")
    metric = sim.GaussianMetric(g, levels=2, weights=(1.0, 0.5))
    assert rel_err(metric.apply(c["x"]), c["apply"]) < 1e-13
    assert abs(metric.quad(c["x"]) - float(c["quad"])) <= 1e-13 * float(c["quad"])


def test_scalar_stencil_v_adjoint_and_operator_masking(case):
    """``advection.py:105-130`` and the AdvectionOperator's wall masking
    (``advection.py:220-224``): the oracle on the masked velocity equals the
    reference operator built from the raw one."""
    g = case.grid()
    rho, mu = case["rho"], case["mu"]
    assert rel_err(ops.scalar_stencil_v_adjoint(g, rho, mu), case.comps("svadj")) < 1e-14
    vm = ops.zero_walls(g, case.comps("vraw"))
    assert rel_err(ops.transport_scalar(g, vm, rho), case["aop_st"]) < 1e-14
    out, k, _ = ops.taylor(g, vm, rho, 0.1)
    assert k == int(case["aop_k"])
    assert rel_err(out, case["aop_adv"]) < 1e-13
    assert rel_err(ops.taylor(g, vm, mu, 0.1, k_fixed=k, transpose=True)[0], case["aop_rT"]) < 1e-13
    assert rel_err(ops.advect_v_T(g, vm, rho, mu, 0.1, k), case.comps("aop_vT")) < 1e-13
