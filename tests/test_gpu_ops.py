"""GPU sub-operators vs the reference's own outputs (golden vectors) — B200.

Every call goes through libsmk.so (the C-ABI); tolerances are fp64
relative-to-max errors.
"""

import numpy as np
import pytest

from conftest import GoldenCase, rel_err

pytestmark = pytest.mark.gpu

TAGS = ["n2p", "n2n", "r2n", "n3n", "n3p"]


@pytest.fixture(scope="module")
def smk():
    import paper_1608_01102_b200 as pkg
    from paper_1608_01102_b200 import _lib, advection, fields, simulator
    _lib.load()
    return pkg, fields, advection, simulator


def spec_of(case, fields):
    g = case.grid()
    return fields.GridSpec(g.dim, g.res, g.h, g.boundary)


@pytest.fixture(params=TAGS)
def case(request, golden):
    return GoldenCase(golden, request.param)


def test_div_grad_lap(case, smk):
    _, F, _, _ = smk
    s = spec_of(case, F)
    assert rel_err(F.divergence_arrays(s, case.comps("w")), case["div"]) < 1e-14
    assert rel_err(F.gradient_arrays(s, case["rho"]), case.comps("grad")) < 1e-14


def test_transport_taylor_adjoints(case, smk):
    _, F, A, _ = smk
    s = spec_of(case, F)
    v, rho, mu = case.comps("v"), case["rho"], case["mu"]
    assert rel_err(A.transport_scalar(s, v, rho), case["T"]) < 1e-14
    out, rep = A.advect_scalar(s, v, rho, 0.1)
    assert rep.k_used == int(case["adv_k"])
    assert rel_err(out, case["adv"]) < 1e-13
    back, rep2 = A.advect_scalar_rho_T(s, v, mu, 0.1, k_fixed=rep.k_used)
    assert rel_err(back, case["advT"]) < 1e-13
    g, _ = A.advect_scalar_v_T(s, v, rho, mu, 0.1, k_fixed=rep.k_used)
    assert rel_err(g, case.comps("advvT")) < 1e-13


def test_self_advection_family(case, smk):
    _, F, A, _ = smk
    s = spec_of(case, F)
    v, w, u = case.comps("v"), case.comps("w"), case.comps("u")
    assert rel_err(A.transport_face(s, v, w), case.comps("S")) < 1e-14
    assert rel_err(A.self_advection(s, v), case.comps("Sself")) < 1e-14
    assert rel_err(A.self_adv_jacobian_apply(s, v, w), case.comps("J")) < 1e-14
    assert rel_err(A.self_adv_jacobian_T_apply(s, v, u), case.comps("JT")) < 1e-13


def test_cell_transfers(case, smk):
    _, F, _, _ = smk
    s = spec_of(case, F)
    rho = case["rho"]
    assert rel_err(F.restrict_cell(s, rho), case["rc"]) < 1e-15
    if case.has("pc"):
        sc = s.coarsen()
        assert rel_err(F.prolong_cell(sc, s, F.restrict_cell(s, rho)), case["pc"]) < 1e-15


def test_projection_poisson(case, smk):
    _, F, _, _ = smk
    s = spec_of(case, F)
    assert rel_err(F.project_arrays(s, case.comps("w"), 1e-9), case.comps("proj")) < 1e-11
    p = F.solve_poisson(s, case["mu"], 1e-9)
    want = case["pois"]
    assert rel_err(p - p.mean(), want - want.mean()) < 1e-9
    # post-condition of project_arrays (fields.py:350-358)
    out = F.project_arrays(s, case.comps("w"), 1e-9)
    assert F.inf_norm(F.divergence_arrays(s, out)) <= 1e-9


def test_semi_lagrangian(case, smk):
    _, F, A, _ = smk
    s = spec_of(case, F)
    out = A.semi_lagrangian(F.ScalarField(s, np.abs(case["rho"])), F.StaggeredVectorField(s, case.comps("v")), 0.3)
    assert rel_err(out.values.cpu().numpy(), case["sl"]) < 1e-14


def test_sim_step(case, smk):
    _, F, A, S = smk
    s = spec_of(case, F)
    st = S.SimState(F.StaggeredVectorField(s, case.comps("v")), F.ScalarField.zeros(s),
                    F.ScalarField(s, np.abs(case["rho"])))
    out = S.step(st, F.StaggeredVectorField(s, case.comps("su")), S.SimConfig(dt=0.1), accept_stall=True)
    v = tuple(c.cpu().numpy() for c in out.v.comps)
    assert rel_err(v, case.comps("step_v")) < 1e-11
    assert rel_err(out.rho.values.cpu().numpy(), case["step_rho"]) < 1e-13
    p = out.p.values.cpu().numpy()
    want = case["step_p"]
    assert rel_err(p - p.mean(), want - want.mean()) < 1e-8


def test_face_transfers_vs_oracle(smk):
    from oracle import ops
    from oracle.grid import Grid
    _, F, _, _ = smk
    rng = np.random.default_rng(5)
    for dim, bnd in [(2, "neumann"), (2, "periodic"), (3, "neumann"), (3, "periodic")]:
        g = Grid(dim, (8,) * dim, 1 / 8, bnd)
        s = F.GridSpec(dim, g.res, g.h, bnd)
        comps = tuple(rng.standard_normal((3,) + g.face_shape(k)) for k in range(dim))
        rc = F.restrict_face(s, comps)
        assert rel_err(rc, ops.restrict_face(g, comps)) < 1e-15
        gc = g.coarsen()
        pc = F.prolong_face(s.coarsen(), s, rc)
        assert rel_err(pc, ops.prolong_face(gc, ops.restrict_face(g, comps))) < 1e-15


def test_taylor_overflow_maps_to_exception(smk):
    from paper_1608_01102_b200.errors import TruncationOverflow
    _, F, A, _ = smk
    s = F.GridSpec(2, (8, 8), 1 / 8, "periodic")
    rng = np.random.default_rng(8)
    v = tuple(50 * rng.standard_normal(s.face_shape(k)) for k in range(2))
    with pytest.raises(TruncationOverflow):
        A.advect_scalar(s, v, rng.standard_normal(s.res), 10.0, cap=16)


def test_taylor_speculative_batches_keep_the_adaptive_stop(smk):
    """The adaptive Taylor stop (``advection.py:144-163``) is decided on the
    device: terms are launched in speculative batches gated on the previous
    term's norm.  A short line after a long one (over-launched, gated terms)
    and a long one after a short one (several batches) must give the oracle's
    order and the same bits as the fixed-order evaluation."""
    from oracle import ops
    from oracle.grid import Grid
    _, F, A, _ = smk
    s = F.GridSpec(2, (16, 16), 1 / 16, "neumann")
    g = Grid(2, (16, 16), 1 / 16, "neumann")
    rng = np.random.default_rng(10)
    v = F.zero_boundary_faces(s, tuple(rng.standard_normal(s.face_shape(k)) for k in range(2)))
    rho = rng.standard_normal(s.res)
    orders = []
    for dt in (0.002, 0.2, 0.0005, 0.1, 0.3, 0.001):
        out, rep = A.advect_scalar(s, v, rho, dt)
        want, k_ref, _ = ops.taylor(g, v, rho, dt, tol=A.DEFAULT_TRUNCATION_TOL, cap=A.DEFAULT_TERM_CAP)
        assert rep.k_used == k_ref
        assert rel_err(out, want) < 1e-11   # up to 37 alternating terms: 4e-13 measured at dt = 0.3
        fixed, _ = A.advect_scalar(s, v, rho, dt, k_fixed=rep.k_used)
        assert np.array_equal(out, fixed)
        back, repT = A.advect_scalar_rho_T(s, v, rho, dt)
        backf, _ = A.advect_scalar_rho_T(s, v, rho, dt, k_fixed=repT.k_used)
        assert np.array_equal(back, backf)
        orders.append(rep.k_used)
    assert max(orders) >= min(orders) + 8   # the sequence really alternates short and long lines


def test_determinism(smk):
    _, F, A, _ = smk
    s = F.GridSpec(2, (16, 16), 1 / 16, "neumann")
    rng = np.random.default_rng(9)
    v = F.zero_boundary_faces(s, tuple(rng.standard_normal(s.face_shape(k)) for k in range(2)))
    rho = rng.standard_normal(s.res)
    a, _ = A.advect_scalar(s, v, rho, 0.02)
    b, _ = A.advect_scalar(s, v, rho, 0.02)
    assert np.array_equal(a, b)


def test_scalar_stencil_v_adjoint(case, smk):
    """``advection.scalar_stencil_v_adjoint`` (``advection.py:105``) through
    ``smk_scalar_stencil_v_adjoint`` (k_stencil_v_adj) vs the reference."""
    _, F, A, _ = smk
    s = spec_of(case, F)
    got = A.scalar_stencil_v_adjoint(s, case["rho"], case["mu"])
    assert rel_err(got, case.comps("svadj")) < 1e-14


def test_advection_operator(case, smk):
    """``AdvectionOperator`` (``advection.py:213-248``) built from a velocity
    with nonzero wall faces (masked at construction) vs the reference's own
    operator on the same raw velocity."""
    _, F, A, _ = smk
    s = spec_of(case, F)
    op = A.AdvectionOperator(F.StaggeredVectorField(s, case.comps("vraw")))
    rho = F.ScalarField(s, case["rho"])
    mu = F.ScalarField(s, case["mu"])
    h = lambda t: t.detach().cpu().numpy()
    assert rel_err(h(op.apply_stencil(rho).values), case["aop_st"]) < 1e-14
    out, rep = op.advect(rho, 0.1)
    assert rep.k_used == int(case["aop_k"])
    assert rel_err(h(out.values), case["aop_adv"]) < 1e-13
    back, _ = op.jacobian_rho_T(mu, 0.1, k_fixed=rep.k_used)
    assert rel_err(h(back.values), case["aop_rT"]) < 1e-13
    gv = tuple(h(c) for c in op.jacobian_v_T(rho, mu, 0.1, k_fixed=rep.k_used).comps)
    assert rel_err(gv, case.comps("aop_vT")) < 1e-13
    with pytest.raises(ValueError):
        op.advect(rho, 0.0)
