"""Pin the C STFAS oracle (oracle/cstfas.c) to the numpy oracle (CPU).

oracle/stfas.py is pinned to the reference's golden vectors (sub-operators)
and to SPEC's known-answer tests (tests/test_oracle_stfas.py); the C
restatement must reproduce it on the same seeded inputs before it is used as
the checker at the BASELINE configs' real sizes (tests/test_gpu_configs.py)
and as the CPU baseline (bench.py).  Different summation / pivoting codes
(LAPACK gesv vs the C solve), so the bound is rounding-level, not bitwise.
"""

import ctypes

import numpy as np
import pytest

from conftest import rel_err
from oracle import cstfas, ops, stfas
from oracle.grid import Grid
from problems import make_problem, random_residual, random_state


def _st_err(a, b):
    return max(rel_err(a.V, b.V), rel_err(a.U, b.U), rel_err(a.P, b.P), rel_err(a.PB, b.PB))


def _res_err(a, b):
    return max(rel_err(a.R1, b.R1), rel_err(a.R3, b.R3), rel_err(a.R2, b.R2), rel_err(a.R4, b.R4))


CASES = [(2, 8, 3, "neumann"), (2, 8, 3, "periodic"), (3, 6, 2, "neumann"), (3, 4, 2, "periodic")]


@pytest.mark.parametrize("dim,n,N,bnd", CASES)
def test_kkt_residual_matches_numpy_oracle(dim, n, N, bnd):
    pb = make_problem(dim, n=n, N=N, boundary=bnd, seed=3)
    rng = np.random.default_rng(1)
    st = random_state(pb, rng, 0.3)
    rhs = random_residual(pb, rng, 0.1)
    assert _res_err(cstfas.kkt_residual(pb, st), stfas.kkt_residual(pb, st)) <= 1e-14
    assert _res_err(cstfas.kkt_residual(pb, st, rhs), stfas.kkt_residual(pb, st).sub(rhs)) <= 1e-14


@pytest.mark.parametrize("rb", [True, False])
@pytest.mark.parametrize("dim,n,N,bnd", CASES)
def test_colour_pass_matches_numpy_oracle(dim, n, N, bnd, rb):
    pb = make_problem(dim, n=n, N=N, boundary=bnd, seed=4)
    pb.red_black = rb
    rng = np.random.default_rng(2)
    st = random_state(pb, rng, 0.1)
    rhs = random_residual(pb, rng, 0.1)
    for colour in ((0, 1) if rb else (0, 3)):
        a, xa = stfas.scgs_color(pb, st, rhs, colour, return_delta=True)
        b, xb = cstfas.scgs_color(pb, st, rhs, colour, return_delta=True)
        assert rel_err(xb, xa) <= 1e-10
        assert _st_err(b, a) <= 1e-10


def test_colour_pass_cell_subset_and_order():
    pb = make_problem(2, n=8, N=3, seed=6)
    st = random_state(pb, np.random.default_rng(6), 0.1)
    cells = np.argwhere(stfas.color_of(pb.g, 2, pb.red_black) == 1)
    a, xa = cstfas.scgs_color(pb, st, None, 1, cells=cells, return_delta=True)
    b, xb = cstfas.scgs_color(pb, st, None, 1, cells=cells[::-1].copy(), return_delta=True)
    assert np.array_equal(xa, xb[::-1]) and _st_err(a, b) == 0.0
    w, xw = stfas.scgs_color(pb, st, None, 1, cells=cells[:5], return_delta=True)
    c, xc = cstfas.scgs_color(pb, st, None, 1, cells=cells[:5], return_delta=True)
    assert rel_err(xc, xw) <= 1e-10


def test_transfers_match_numpy_oracle_bitwise():
    P = cstfas._P
    L = cstfas.load()
    rng = np.random.default_rng(0)
    for dim, bnd in [(2, "neumann"), (2, "periodic"), (3, "neumann"), (3, "periodic")]:
        n = 8
        g = Grid(dim, (n,) * dim, 1 / n, bnd)
        gc = g.coarsen()
        x = rng.standard_normal((2,) + g.res)
        out = np.zeros((2,) + gc.res)
        L.cst_restrict_cell(ctypes.byref(cstfas._grid(g)), 2, cstfas._ptr(x), cstfas._ptr(out))
        assert np.array_equal(out, ops.restrict_cell(g, x))
        xc = rng.standard_normal((2,) + gc.res)
        o2 = np.zeros((2,) + g.res)
        L.cst_prolong_cell(ctypes.byref(cstfas._grid(gc)), 2, cstfas._ptr(xc), cstfas._ptr(o2), 0)
        assert np.array_equal(o2, ops.prolong_cell(gc, xc))
        f = tuple(rng.standard_normal((2,) + g.face_shape(k)) for k in range(dim))
        fo = tuple(np.zeros((2,) + gc.face_shape(k)) for k in range(dim))
        L.cst_restrict_face(ctypes.byref(cstfas._grid(g)), 2, (P * 3)(*[cstfas._ptr(a) for a in f]),
                            (P * 3)(*[cstfas._ptr(a) for a in fo]))
        assert all(np.array_equal(a, b) for a, b in zip(fo, ops.restrict_face(g, f)))
        fc = tuple(rng.standard_normal((2,) + gc.face_shape(k)) for k in range(dim))
        ff = tuple(np.zeros((2,) + g.face_shape(k)) for k in range(dim))
        L.cst_prolong_face(ctypes.byref(cstfas._grid(gc)), 2, (P * 3)(*[cstfas._ptr(a) for a in fc]),
                           (P * 3)(*[cstfas._ptr(a) for a in ff]), 0)
        assert all(np.array_equal(a, b) for a, b in zip(ff, ops.prolong_face(gc, fc)))


@pytest.mark.parametrize("dim,n,N,bnd,lv,rb", [(2, 16, 4, "neumann", 2, True), (2, 16, 4, "periodic", 3, True),
                                               (3, 8, 2, "neumann", 2, True), (2, 16, 4, "neumann", 3, False)])
def test_vcycle_matches_numpy_oracle(dim, n, N, bnd, lv, rb):
    pb = make_problem(dim, n=n, N=N, boundary=bnd, seed=3)
    pb.red_black = rb
    levels = stfas.build_levels(pb, lv)
    H = cstfas.Hierarchy(pb, lv)
    assert H.levels == len(levels)
    a = stfas.zero_state(pb.g, pb.N)
    b = a
    for _ in range(2):
        a = stfas.gauge_fix(stfas.vcycle(levels, 0, a))
        b = H.vcycle(b, gauge=True)
        assert _st_err(b, a) <= 1e-12
    ri, r2 = H.norms(b)
    r = stfas.kkt_residual(pb, a)
    assert abs(ri - r.inf()) <= 1e-12 * r.inf() and abs(r2 - r.l2()) <= 1e-12 * r.l2()


def test_solve_matches_numpy_oracle():
    pb = make_problem(2, n=8, N=3, seed=8)
    want = stfas.solve_nso(pb, eps=1e-10, cycle_budget=40, n_levels=2)
    st, hist, ok = cstfas.Hierarchy(pb, 2).solve(eps=1e-10, cycle_budget=40)
    assert ok and want.converged and len(hist) == len(want.history)
    for (c, a, b), (c2, a2, b2) in zip(hist, want.history):
        assert abs(a - a2) <= 1e-6 * max(a2, 1e-12)
    assert _st_err(st, stfas.gauge_fix(want.state)) <= 1e-9


def test_threads_do_not_change_results():
    pb = make_problem(2, n=16, N=4, seed=5)
    H = cstfas.Hierarchy(pb, 2)
    n0 = cstfas.set_threads(0)
    try:
        cstfas.set_threads(1)
        a = H.vcycle(stfas.zero_state(pb.g, pb.N))
        cstfas.set_threads(max(2, n0))
        b = H.vcycle(stfas.zero_state(pb.g, pb.N))
    finally:
        cstfas.set_threads(n0)
    assert _st_err(a, b) == 0.0
