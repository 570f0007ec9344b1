"""Known-answer tests pinning the STFAS oracle (CPU).

The reference has no STFAS code, so the oracle is pinned to the SPEC's own
acceptance recipes: dense-Newton KKT solution, exact
Eq. 9 blocks, exact block-Thomas solve, transfer-operator properties and the
V-cycle's linear convergence.
"""

import numpy as np
import pytest

from conftest import rel_err
from oracle import dense, ops, stfas
from oracle.grid import Grid
from problems import make_problem, random_residual, random_state


def test_zero_state_is_kkt_point_of_zero_guide():
    pb = make_problem(2, n=8, N=3, seed=0)
    pb.vstar = tuple(np.zeros_like(c) for c in pb.vstar)
    assert stfas.kkt_residual(pb, stfas.zero_state(pb.g, 3)).inf() == 0.0


@pytest.mark.parametrize("bnd", ["neumann", "periodic"])
def test_dense_newton_solution_zeroes_residual(bnd):
    # residual vanishes (<= 1e-8) at the dense Newton solution
    pb = make_problem(2, n=6, N=3, boundary=bnd, seed=1, res=(6, 6))
    st, hist = dense.newton(pb)
    assert hist[-1] <= 1e-10
    assert stfas.kkt_residual(pb, st).inf() <= 1e-8


def test_jacobian_rank_deficiency_is_gauge():
    # 2N nullspace = per-frame constants of p and pbar
    pb = make_problem(2, n=6, N=3, seed=2, res=(6, 6))
    pk = dense.Packer(pb)
    J = dense.jacobian(pb, pk, np.zeros(pk.n))
    sv = np.linalg.svd(J, compute_uv=False)
    assert int(np.sum(sv < 1e-9 * sv[0])) == 2 * pb.N


@pytest.mark.parametrize("bnd", ["neumann", "periodic"])
def test_local_blocks_match_fd_jacobian(bnd):
    """assemble_line's Eq. 9 blocks equal the finite-difference Jacobian of
    kkt_residual restricted to one cell's unknowns (u = 0 so the Gauss-Newton
    dropped term vanishes)."""
    pb = make_problem(2, n=8, N=3, boundary=bnd, seed=3)
    rng = np.random.default_rng(0)
    st = random_state(pb, rng, 0.3)
    st = stfas.State(st.V, st.PB, tuple(np.zeros_like(u) for u in st.U), st.P)
    pk = dense.Packer(pb)
    x = pk.pack_state(st)
    Jfd = dense.jacobian(pb, pk, x)
    cell = np.array([[3, 2]])
    slots = stfas.CellSlots(pb.g, cell)
    D, L, Up = stfas.assemble_line(pb, slots, stfas.local_jacobian(pb, st.V, slots))
    nb, b = D.shape[1], D.shape[2]
    full = np.zeros((nb * b, nb * b))
    for k in range(nb):
        full[k * b:(k + 1) * b, k * b:(k + 1) * b] = D[0, k]
        if k > 0:
            full[k * b:(k + 1) * b, (k - 1) * b:k * b] = L[0, k]
        if k + 1 < nb:
            full[k * b:(k + 1) * b, (k + 1) * b:(k + 2) * b] = Up[0, k]
    # map local (block, slot) -> packed index of the unknown / row
    g, N = pb.g, pb.N
    idx = np.full(nb * b, -1)
    fm = [m for m in pk.face_masks]
    offs = np.cumsum([0] + [int(m.sum()) for m in fm])
    flat = [np.full(m.shape, -1) for m in fm]
    for k, m in enumerate(fm):
        flat[k][m] = np.arange(int(m.sum())) + offs[k]
    nf, nc = pk.nf, pk.nc
    cflat = np.arange(nc).reshape((N,) + g.res)
    for i in range(N):
        for q, (k, fi) in enumerate(slots.face_idx):
            if slots.wall[0, q]:
                continue
            f = tuple(a[0] for a in fi)
            idx[(2 * i) * b + q] = nf + nc + flat[k][(i,) + f]          # u_i face
            idx[(2 * i + 1) * b + q] = flat[k][(i,) + f]                # v_{i+1} face
        c = tuple(cell[0])
        idx[(2 * i) * b + b - 1] = 2 * nf + nc + cflat[(i,) + c]        # p_{i+1}
        idx[(2 * i + 1) * b + b - 1] = nf + cflat[(i,) + c]             # pbar_{i+1}
    # rows: u-block rows are R3/R4 (packed after R1/R2), v-block rows R1/R2
    ridx = idx.copy()
    keep = idx >= 0
    sub = Jfd[np.ix_(ridx[keep], idx[keep])]
    assert np.max(np.abs(sub - full[np.ix_(keep, keep)])) <= 1e-9 * np.max(np.abs(sub))


def test_block_thomas_equals_dense_solve():
    rng = np.random.default_rng(4)
    pb = make_problem(2, n=8, N=4, seed=4)
    st = random_state(pb, rng, 0.2)
    cells = np.array([[2, 4], [5, 1]])
    slots = stfas.CellSlots(pb.g, cells)
    D, L, Up = stfas.assemble_line(pb, slots, stfas.local_jacobian(pb, st.V, slots))
    y = rng.standard_normal(D.shape[:3])
    x = stfas.block_thomas(D, L, Up, y)
    nb, b = D.shape[1], D.shape[2]
    for m in range(2):
        full = np.zeros((nb * b, nb * b))
        for k in range(nb):
            full[k * b:(k + 1) * b, k * b:(k + 1) * b] = D[m, k]
            if k > 0:
                full[k * b:(k + 1) * b, (k - 1) * b:k * b] = L[m, k]
            if k + 1 < nb:
                full[k * b:(k + 1) * b, (k + 1) * b:(k + 2) * b] = Up[m, k]
        want = np.linalg.solve(full, y[m].reshape(-1))
        assert rel_err(x[m].reshape(-1), want) < 1e-10


def test_smoother_fixes_exact_solution():
    pb = make_problem(2, n=8, N=4, seed=5)
    st = random_state(pb, np.random.default_rng(5))
    rhs = stfas.kkt_residual(pb, st)
    out = stfas.scgs_smooth(pb, st, rhs)
    assert max(rel_err(out.V, st.V), rel_err(out.U, st.U)) < 1e-12


def test_colouring_is_race_free_order_independent():
    """within a colour the result does not depend on traversal order."""
    pb = make_problem(2, n=8, N=3, seed=6)
    rng = np.random.default_rng(6)
    st = random_state(pb, rng, 0.1)
    cells = np.argwhere(stfas.color_of(pb.g) == 1)
    a = stfas.scgs_color(pb, st, None, 1, cells=cells)
    b = stfas.scgs_color(pb, st, None, 1, cells=cells[::-1].copy())
    assert max(rel_err(a.V, b.V), rel_err(a.U, b.U), rel_err(a.P, b.P), rel_err(a.PB, b.PB)) == 0.0


def test_transfers_preserve_constants_and_energy():
    for dim, bnd in [(2, "neumann"), (2, "periodic"), (3, "neumann")]:
        n = 16 if dim == 2 else 8
        g = Grid(dim, (n,) * dim, 1.0 / n, bnd)
        gc = g.coarsen()
        comps = tuple(np.full(g.face_shape(k), 2.5) for k in range(dim))
        for k, c in enumerate(ops.restrict_face(g, comps)):
            assert np.allclose(c, 2.5)
        for k, c in enumerate(ops.prolong_face(gc, tuple(np.full(gc.face_shape(k), -1.5) for k in range(dim)))):
            assert np.allclose(c, -1.5)
        assert np.allclose(ops.prolong_cell(gc, np.full(gc.res, 0.7)), 0.7)
    # >= 95% energy kept by P R on a low mode, 32^2
    g = Grid(2, (32, 32), 1 / 32, "periodic")
    x = (np.arange(32) + 0.5) / 32
    f = np.sin(2 * np.pi * x)[:, None] * np.cos(2 * np.pi * x)[None, :]
    pr = ops.prolong_cell(g.coarsen(), ops.restrict_cell(g, f))
    assert np.sum(pr * f) / np.sum(f * f) >= 0.95
    # checkerboard: the 2x2 box average annihilates it exactly (factor 0)
    cb = (-1.0) ** np.add.outer(np.arange(32), np.arange(32))
    assert np.max(np.abs(ops.restrict_cell(g, cb))) == 0.0


def test_vcycle_fixed_point():
    """An exact solution is a fixed point of the FAS V-cycle."""
    pb = make_problem(2, n=8, N=3, seed=7)
    st, hist = dense.newton(pb)
    levels = stfas.build_levels(pb, 2)
    out = stfas.vcycle(levels, 0, st)
    assert stfas.kkt_residual(pb, out).inf() <= 1e-9


def test_solve_nso_matches_dense_newton():
    """solve_nso reproduces the dense Newton solution (1e-6)."""
    pb = make_problem(2, n=8, N=3, seed=8)
    want, hist = dense.newton(pb)
    res = stfas.solve_nso(pb, eps=1e-11, cycle_budget=80, n_levels=2)
    assert res.converged
    got = stfas.gauge_fix(res.state)
    want = stfas.gauge_fix(want)
    for a, b in [(got.V, want.V), (got.U, want.U), ((got.P,), (want.P,)), ((got.PB,), (want.PB,))]:
        assert max(float(np.max(np.abs(x - y))) for x, y in zip(a, b)) <= 1e-6


def test_vcycle_linear_convergence_small():
    """Linear, mesh-independent reduction (SPEC.md:342 on CPU-sized cases)."""
    facs = []
    for n in (8, 16):
        pb = make_problem(2, n=n, N=4, seed=9)
        res = stfas.solve_nso(pb, eps=1e-14, cycle_budget=5, n_levels=2)
        r = [h[1] for h in res.history]
        facs.append((r[-1] / r[2]) ** (1.0 / (len(r) - 3)))
    # the 8^2 case coarsens to 4^2 (near-direct); mesh independence proper is
    # checked on the GPU at 16^2..32^2 (tests/test_gpu_convergence.py)
    assert max(facs) <= 0.75


def test_lm_shift_keeps_the_fixed_point():
    """oracle solve_nso_lm: with the shift forced on
    it still converges to the undamped solution; untriggered it is the plain
    solve."""
    from problems import make_problem
    pb = make_problem(2, n=8, N=4, seed=3)
    plain = stfas.solve_nso(pb, eps=1e-9, cycle_budget=30)
    lm = stfas.solve_nso_lm(pb, eps=1e-9, cycle_budget=30)
    assert [h[1] for h in lm.history] == [h[1] for h in plain.history]
    forced = stfas.solve_nso_lm(pb, eps=1e-9, cycle_budget=60, stall=0.3)
    assert forced.converged
    for a, b in zip(forced.state.V, plain.state.V):
        assert np.max(np.abs(a - b)) <= 1e-6 * max(1.0, np.max(np.abs(b)))
