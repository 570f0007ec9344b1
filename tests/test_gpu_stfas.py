"""STFAS kernels on B200 vs the CPU oracle (oracle/stfas.py) on seeded inputs.

fp64 bar: <= 1e-10 relative on single passes (residual, colour pass, sweep,
V-cycle) and <= 1e-8 relative on converged fields (v, u; p and pbar modulo
per-frame constants).  fp32 bar (stated): residual/sweep <= 1e-4 relative.
"""

import numpy as np
import pytest
import torch

from conftest import rel_err
from oracle import stfas
from problems import make_problem, random_residual, random_state

pytestmark = pytest.mark.gpu

CASES = [(2, "neumann"), (2, "periodic"), (3, "neumann"), (3, "periodic")]


@pytest.fixture(scope="module")
def nso():
    from paper_1608_01102_b200 import _lib, nso
    _lib.load()
    return nso


def spec_cfg(nso, pb, **kw):
    from paper_1608_01102_b200.fields import GridSpec
    g = pb.g
    s = GridSpec(g.dim, g.res, g.h, g.boundary)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, omega=pb.omega, color_mod=pb.colors,
                          red_black=pb.red_black, **kw)
    return s, cfg


def to_dev(nso, st, dtype=torch.float64):
    return nso.SpacetimeState.from_arrays(st.V, st.PB, st.U, st.P, dtype=dtype)


def to_dev_res(nso, r, dtype=torch.float64):
    from paper_1608_01102_b200._dev import as_dev
    return nso.SpacetimeResidual(tuple(as_dev(c, dtype) for c in r.R1), as_dev(r.R2, dtype),
                                 tuple(as_dev(c, dtype) for c in r.R3), as_dev(r.R4, dtype))


def state_err(dev, st, gauge=False):
    V, PB, U, P = dev.numpy()
    if gauge:
        ax = tuple(range(1, PB.ndim))
        f = lambda x: x - x.mean(axis=ax, keepdims=True)
        return max(rel_err(V, st.V), rel_err(U, st.U), rel_err(f(PB), f(st.PB)), rel_err(f(P), f(st.P)))
    return max(rel_err(V, st.V), rel_err(U, st.U), rel_err(PB, st.PB), rel_err(P, st.P))


def res_err(dev, r):
    R1, R2, R3, R4 = dev.numpy()
    return max(rel_err(R1, r.R1), rel_err(R2, r.R2), rel_err(R3, r.R3), rel_err(R4, r.R4))


@pytest.mark.parametrize("dim,bnd", CASES)
def test_kkt_residual(nso, dim, bnd):
    pb = make_problem(dim, n=8, N=3, boundary=bnd, seed=11)
    rng = np.random.default_rng(1)
    st = random_state(pb, rng)
    rhs = random_residual(pb, rng)
    s, cfg = spec_cfg(nso, pb)
    got = nso.kkt_residual(s, cfg, to_dev(nso, st), pb.v0, pb.vstar)
    assert res_err(got, stfas.kkt_residual(pb, st)) < 1e-12
    got = nso.kkt_residual(s, cfg, to_dev(nso, st), pb.v0, pb.vstar, rhs=to_dev_res(nso, rhs))
    assert res_err(got, stfas.kkt_residual(pb, st).sub(rhs)) < 1e-12


def test_kkt_zero_is_kkt_point_of_zero_guide(nso):
    pb = make_problem(2, n=8, N=3, seed=2)
    pb.vstar = tuple(np.zeros_like(c) for c in pb.vstar)
    s, cfg = spec_cfg(nso, pb)
    st = nso.SpacetimeState.zeros(s, 3)
    assert nso.kkt_residual(s, cfg, st, pb.v0, pb.vstar).inf() == 0.0


@pytest.mark.parametrize("dim,bnd", CASES)
def test_scgs_sweep(nso, dim, bnd):
    pb = make_problem(dim, n=8, N=3, boundary=bnd, seed=21)
    rng = np.random.default_rng(3)
    st = random_state(pb, rng, 0.05)
    rhs = random_residual(pb, rng, 0.05)
    s, cfg = spec_cfg(nso, pb)
    want = stfas.scgs_smooth(pb, st, rhs)
    dev = to_dev(nso, st)
    nso.scgs_smooth(s, cfg, dev, pb.v0, pb.vstar, rhs=to_dev_res(nso, rhs))
    assert state_err(dev, want) < 1e-10


def test_scgs_fixes_exact_solution(nso):
    # rhs = f(x) -> smoothing leaves x unchanged
    pb = make_problem(2, n=8, N=4, seed=5)
    rng = np.random.default_rng(4)
    st = random_state(pb, rng)
    rhs = stfas.kkt_residual(pb, st)
    s, cfg = spec_cfg(nso, pb)
    dev = to_dev(nso, st)
    nso.scgs_smooth(s, cfg, dev, pb.v0, pb.vstar, rhs=to_dev_res(nso, rhs))
    assert state_err(dev, st) < 1e-11


@pytest.mark.parametrize("dim,bnd", [(2, "neumann"), (2, "periodic"), (3, "neumann")])
def test_vcycle(nso, dim, bnd):
    n = 16 if dim == 2 else 8
    pb = make_problem(dim, n=n, N=4, boundary=bnd, seed=31)
    s, cfg = spec_cfg(nso, pb)
    levels = stfas.build_levels(pb, 2)
    want = stfas.vcycle(levels, 0, stfas.zero_state(pb.g, pb.N))
    cfg.n_levels = 2
    dev = nso.SpacetimeState.zeros(s, pb.N)
    hier = nso.StfasHierarchy(s, cfg, pb.N)
    hier.set_guide(pb.v0, pb.vstar)
    assert hier.levels == 2
    hier.vcycle(dev)
    assert state_err(dev, want) < 1e-9


def test_solve_nso_matches_oracle_cfg1_shape(nso):
    # 32^2 / N=16 shape of BASELINE cfg1 at small budget: same iterates
    pb = make_problem(2, n=16, N=8, seed=41)
    s, cfg = spec_cfg(nso, pb, n_levels=2)
    ref = stfas.solve_nso(pb, eps=1e-9, cycle_budget=6, n_levels=2)
    dev = nso.SpacetimeState.zeros(s, pb.N)
    hier = nso.StfasHierarchy(s, cfg, pb.N)
    hier.set_guide(pb.v0, pb.vstar)
    for c in range(6):
        hier.vcycle(dev)
        hier.gauge_fix(dev)
    assert state_err(dev, ref.state, gauge=True) < 1e-8
    ri, _ = hier.residual_norms(dev)
    assert abs(ri - ref.history[-1][1]) <= 1e-6 * ref.history[0][1]


def test_fp32_bound(nso):
    """fp32 mode bound (stated): residual rows <= 1e-6 relative on a random
    state; one sweep from a mid-solve state (after one fp64 V-cycle) <= 1e-4
    relative.  (A sweep from a random state is not used: the last frame's
    local systems carry no K anchor and amplify random residuals ~1e6x.)"""
    pb = make_problem(2, n=16, N=4, seed=51)
    rng = np.random.default_rng(6)
    st = random_state(pb, rng)
    s, cfg = spec_cfg(nso, pb)
    got = nso.kkt_residual(s, cfg, to_dev(nso, st, torch.float32), pb.v0, pb.vstar)
    assert res_err(got, stfas.kkt_residual(pb, st)) < 1e-6
    mid = stfas.vcycle(stfas.build_levels(pb, 2), 0, stfas.zero_state(pb.g, pb.N))
    want = stfas.scgs_smooth(pb, mid)
    dev = to_dev(nso, mid, torch.float32)
    nso.scgs_smooth(s, cfg, dev, pb.v0, pb.vstar)
    assert state_err(dev, want) < 1e-4


# Every launch shape of the colour-pass kernels is parity-checked: the bench
# sizes pick TM 64 / 1 producer group and the unpipelined backward on the fine
# levels, the tests' small grids would otherwise only reach TM 32 / 4 groups
# and the pipelined backward.  SMK_FWD_THRESH / SMK_BACK_FLAT are read when a
# hierarchy (or the one-shot sweep's temporary one) is created.
SHAPES = {"tm64p1": "0,0", "tm32p2": "1000000000,0", "tm32p4": "1000000000,1000000000"}


@pytest.fixture
def shape_env(monkeypatch):
    def set_shape(fwd, back_flat, deep=1):
        monkeypatch.setenv("SMK_FWD_THRESH", SHAPES[fwd])
        monkeypatch.setenv("SMK_BACK_FLAT", str(back_flat))
        monkeypatch.setenv("SMK_BACK_DEEP", str(deep))
    return set_shape


# backward variants: unpipelined (back_flat 0), load-pipelined (deep off),
# cp.async ring (deep on; the test colours are small)
BACKS = {"flat": (0, 1), "pipe": (1 << 40, 0), "deep": (1 << 40, 1)}


@pytest.mark.parametrize("rb", [True, False])
@pytest.mark.parametrize("fwd", list(SHAPES))
@pytest.mark.parametrize("back", list(BACKS))
@pytest.mark.parametrize("dim,bnd", [(2, "neumann"), (3, "neumann"), (3, "periodic")])
def test_scgs_sweep_every_kernel_shape(nso, shape_env, fwd, back, dim, bnd, rb):
    shape_env(fwd, *BACKS[back])
    pb = make_problem(dim, n=8, N=5, boundary=bnd, seed=23)
    pb.red_black = rb
    rng = np.random.default_rng(7)
    st = random_state(pb, rng, 0.05)
    rhs = random_residual(pb, rng, 0.05)
    s, cfg = spec_cfg(nso, pb)
    want = stfas.scgs_smooth(pb, st, rhs)
    dev = to_dev(nso, st)
    nso.scgs_smooth(s, cfg, dev, pb.v0, pb.vstar, rhs=to_dev_res(nso, rhs))
    assert state_err(dev, want) < 1e-10


@pytest.mark.parametrize("fwd", list(SHAPES) + ["tm64p1-one-group"])
def test_fp32_sweep_every_kernel_shape(nso, shape_env, monkeypatch, fwd):
    # fp32 TM 64 colours run two producer groups by default; SMK_FWD_P1=1
    # keeps the one-group shape (fp64's) reachable
    if fwd == "tm64p1-one-group":
        monkeypatch.setenv("SMK_FWD_P1", "1")
        fwd = "tm64p1"
    shape_env(fwd, 0)
    pb = make_problem(3, n=8, N=4, seed=52)
    s, cfg = spec_cfg(nso, pb)
    mid = stfas.vcycle(stfas.build_levels(pb, 2), 0, stfas.zero_state(pb.g, pb.N))
    want = stfas.scgs_smooth(pb, mid)
    dev = to_dev(nso, mid, torch.float32)
    nso.scgs_smooth(s, cfg, dev, pb.v0, pb.vstar)
    assert state_err(dev, want) < 1e-4


def test_shapes_agree_on_bench_sized_colours(nso, shape_env):
    """3D 64^3 x 6 fp64 (32^3 cells per colour -- the bench's fine-level
    regime): one sweep from a mid-solve state with every forward shape vs the
    C oracle (oracle/cstfas.c) on the same state, <= 1e-10 (the colour-pass
    bound).  The state is one oracle V-cycle from zero on a smooth projected
    guide: on white-noise states the coloured Vanka sweep is not contractive
    (updates grow ~1e3x per colour at 32^3), so two correct eliminations of
    the same systems (block Thomas vs LDL^T of the saddle) drift apart."""
    import numpy as np
    from oracle import cstfas
    from paper_1608_01102_b200.fields import GridSpec
    cstfas.load()
    pb = make_problem(3, n=64, N=6, seed=7)
    H = cstfas.Hierarchy(pb, 2)
    mid = H.vcycle(stfas.zero_state(pb.g, pb.N), gauge=True)
    H.close()
    want = cstfas.scgs_smooth(pb, mid)
    spec, cfg = spec_cfg(nso, pb)
    for fwd, bf in [("tm64p1", 0), ("tm32p2", 1 << 40), ("tm32p4", 1 << 40)]:
        shape_env(fwd, bf)
        dev = to_dev(nso, mid)
        nso.scgs_smooth(spec, cfg, dev, pb.v0, pb.vstar)
        e = state_err(dev, want)
        print(f"[parity] 64^3 sweep shape {fwd}: {e:.2e}", flush=True)
        assert e < 1e-10, (fwd, e)


@pytest.mark.parametrize("n", [64, 128])
def test_kkt_residual_compile_time_extents(nso, n):
    """The 64^3 / 128^3 Neumann levels run residual kernels with compile-time
    strides; check them against the oracle at those sizes (fp64, with rhs)."""
    pb = make_problem(3, n=n, N=2 if n == 64 else 1, seed=61)
    rng = np.random.default_rng(8)
    st = random_state(pb, rng)
    rhs = random_residual(pb, rng)
    s, cfg = spec_cfg(nso, pb)
    got = nso.kkt_residual(s, cfg, to_dev(nso, st), pb.v0, pb.vstar, rhs=to_dev_res(nso, rhs))
    assert res_err(got, stfas.kkt_residual(pb, st).sub(rhs)) < 1e-12


def test_vcycle_graph_replay_and_recapture(nso):
    """smk_nso_vcycle replays a captured CUDA graph and re-captures when the
    caller's buffers change: alternating two states on one hierarchy equals
    running each on its own hierarchy (bitwise), and equals direct launches."""
    import os
    pb = make_problem(3, n=8, N=4, seed=71)
    s, cfg = spec_cfg(nso, pb)
    cfg.n_levels = 2
    rng = np.random.default_rng(9)
    st_a, st_b = random_state(pb, rng, 0.05), random_state(pb, rng, 0.05)

    def run(states, order):
        hier = nso.StfasHierarchy(s, cfg, pb.N)
        hier.set_guide(pb.v0, pb.vstar)
        devs = [to_dev(nso, x) for x in states]
        for k in order:
            hier.vcycle(devs[k])
        torch.cuda.synchronize()
        out = [d.numpy() for d in devs]
        hier.close()
        return out

    shared = run([st_a, st_b], [0, 1, 0, 1, 0])
    own_a = run([st_a], [0, 0, 0])[0]
    own_b = run([st_b], [0, 0])[0]
    os.environ["SMK_NO_GRAPH"] = "1"
    try:
        direct_a = run([st_a], [0, 0, 0])[0]
    finally:
        del os.environ["SMK_NO_GRAPH"]
    flat = lambda t: np.concatenate([np.ravel(x) for grp in t for x in (grp if isinstance(grp, tuple) else (grp,))])
    assert np.array_equal(flat(shared[0]), flat(own_a))
    assert np.array_equal(flat(shared[1]), flat(own_b))
    assert np.array_equal(flat(own_a), flat(direct_a))


def test_solve_nso_lm_untriggered_equals_plain(nso):
    """lm=True on a problem that converges: the shift never engages, the
    iterates are the plain solve's (SPEC.md:351 'converge without LM')."""
    pb = make_problem(2, n=8, N=4, seed=3)
    s, cfg = spec_cfg(nso, pb)
    a = nso.solve_nso(s, cfg, pb.v0, pb.vstar, eps=1e-9, cycle_budget=30, lm=True)
    b = nso.solve_nso(s, cfg, pb.v0, pb.vstar, eps=1e-9, cycle_budget=30)
    assert [c for c, _, _ in a.history] == [c for c, _, _ in b.history]
    assert state_err(a.state, stfas.State(*b.state.numpy())) == 0.0


def test_solve_nso_lm_shifted_path_matches_oracle(nso):
    """Force the shifted (damped) cycles with a low stall threshold: every
    cycle from the third on runs with K + sigma, sigma doubling.  Same
    iterates and residual history as the oracle; the budget runs out on both
    sides (NonConvergence here, converged=False there)."""
    from paper_1608_01102_b200.errors import NonConvergence
    pb = make_problem(2, n=8, N=4, seed=3)
    s, cfg = spec_cfg(nso, pb)
    ref = stfas.solve_nso_lm(pb, eps=1e-12, cycle_budget=7, stall=0.05)
    assert not ref.converged
    dev = nso.SpacetimeState.zeros(s, pb.N)
    with pytest.raises(NonConvergence):
        nso.solve_nso(s, cfg, pb.v0, pb.vstar, s=dev, eps=1e-12, cycle_budget=7, lm=True, lm_stall=0.05)
    assert state_err(dev, ref.state, gauge=True) < 1e-8
    # the shifted cycles still reduce the undamped residual
    hist = [h[1] for h in ref.history]
    assert hist[-1] < hist[2]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("fwd", ["tm64p1", "tm32p2", "tm32p4"])
def test_singular_block_raised(nso, shape_env, fwd, dtype):
    """SingularBlock when a cell's block pivot falls below 1e-12
    (relative to the block's scale).  K = 0 at the zero state:
    every non-final pair's faces block D = (PM)^T PM + P/dt^2 is singular along
    g (M = I/dt at v = 0), so the unpivoted elimination breaks down on every
    launch shape; the Table-1 K passes on the same problem."""
    from paper_1608_01102_b200 import errors
    shape_env(fwd, 0 if fwd == "tm64p1" else 1 << 40)
    for dim in (2, 3):
        pb = make_problem(dim, n=8, N=3, seed=3, K=0.0)
        s, cfg = spec_cfg(nso, pb)
        dev = to_dev(nso, stfas.zero_state(pb.g, pb.N), dtype)
        with pytest.raises(errors.SingularBlock):
            nso.scgs_smooth(s, cfg, dev, pb.v0, pb.vstar)
        pb2 = make_problem(dim, n=8, N=3, seed=3)
        s2, cfg2 = spec_cfg(nso, pb2)
        dev2 = to_dev(nso, stfas.zero_state(pb2.g, pb2.N), dtype)
        nso.scgs_smooth(s2, cfg2, dev2, pb2.v0, pb2.vstar)
