"""Time-slab solver on B200 (libsmk engine): a single slab reproduces the
C++ hierarchy's V-cycle, two in-process slabs reproduce the oracle's slab
iterates and converge to the single-slab solution."""

import numpy as np
import pytest
import torch

from oracle import stfas
from problems import make_problem
from slab_oracle import build_oracle_solver

pytestmark = pytest.mark.gpu


def setup(pb, slab_ids, n_slabs, n_levels):
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    from paper_1608_01102_b200.slabs import build_lib_solver
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=n_levels)
    return spec, cfg, build_lib_solver(spec, cfg, pb.v0, pb.vstar, slab_ids, n_slabs, pb.N)


def flat_dev(st):
    V, PB, U, P = st.numpy()
    return np.concatenate([a.ravel() for a in V + (PB,) + U + (P,)])


def flat_np(st):
    return np.concatenate([a.ravel() for a in st.V + (st.PB,) + st.U + (st.P,)])


def test_single_slab_equals_hierarchy_vcycle():
    from paper_1608_01102_b200 import nso
    pb = make_problem(2, n=16, N=6, seed=201)
    spec, cfg, (solver, states) = setup(pb, [0], 1, 3)
    solver.vcycle(states)
    s = nso.SpacetimeState.zeros(spec, pb.N)
    hier = nso.StfasHierarchy(spec, cfg, pb.N)
    hier.set_guide(pb.v0, pb.vstar)
    hier.vcycle(s)
    a, b = flat_dev(states[0]), flat_dev(s)
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(b))


@pytest.mark.parametrize("dim", [2, 3])
def test_two_slabs_match_oracle_slabs(dim):
    n = 16 if dim == 2 else 8
    pb = make_problem(dim, n=n, N=6, seed=202)
    spec, cfg, (solver, states) = setup(pb, [0, 1], 2, 2)
    osolver, ostates = build_oracle_solver(pb, 2, [0, 1], 2)
    for _ in range(2):
        solver.vcycle(states)
        solver.gauge(states)
        osolver.vcycle(ostates)
        osolver.gauge(ostates)
    for d, o in zip(states, ostates):
        a, b = flat_dev(d), flat_np(o)
        assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))


def test_four_slabs_converge_to_single_slab_solution():
    pb = make_problem(2, n=16, N=8, seed=203)
    _, _, (one, s1) = setup(pb, [0], 1, 3)
    one.solve(s1, eps=1e-10, cycle_budget=80)
    _, _, (four, s4) = setup(pb, [0, 1, 2, 3], 4, 3)
    h4 = four.solve(s4, eps=1e-10, cycle_budget=120)
    assert h4[-1][1] <= 1e-10
    a = flat_dev(s1[0])
    V = [np.concatenate([st.numpy()[0][k] for st in s4]) for k in range(2)]
    U = [np.concatenate([st.numpy()[2][k] for st in s4]) for k in range(2)]
    V1, _, U1, _ = s1[0].numpy()
    scale = max(np.max(np.abs(x)) for x in V1 + U1)
    err = max(np.max(np.abs(x - y)) for x, y in zip(V + U, list(V1) + list(U1)))
    assert err <= 1e-8 * scale


# ---------------------------------------------------------------------------
# the C++ slab set (smk_slabs_*: the V-cycle graph-captured, no Python per
# colour pass) against the Python orchestrator, the hierarchy and the oracle
# ---------------------------------------------------------------------------


def c_setup(pb, slab_ids, n_slabs, n_levels, dtype=torch.float64):
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    from paper_1608_01102_b200.slabs import build_c_solver
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=n_levels)
    return spec, cfg, build_c_solver(spec, cfg, pb.v0, pb.vstar, slab_ids, n_slabs, pb.N, dtype)


@pytest.mark.parametrize("dim", [2, 3])
def test_c_single_slab_equals_hierarchy_bitwise(dim):
    """One C++ slab == the C++ hierarchy V-cycle (same kernels, halos = v0 and
    the guide's own frames): bitwise, over two V-cycles + gauge + norms."""
    from paper_1608_01102_b200 import nso
    pb = make_problem(dim, n=16 if dim == 2 else 8, N=6, seed=211)
    spec, cfg, (cs, st) = c_setup(pb, [0], 1, 3)
    s = nso.SpacetimeState.zeros(spec, pb.N)
    hier = nso.StfasHierarchy(spec, cfg, pb.N)
    hier.set_guide(pb.v0, pb.vstar)
    for _ in range(2):
        cs.vcycle(st)
        cs.gauge(st)
        hier.vcycle(s)
        hier.gauge_fix(s)
    assert np.array_equal(flat_dev(st[0]), flat_dev(s))
    assert cs.norms(st) == hier.residual_norms(s)
    cs.close()
    hier.close()


@pytest.mark.parametrize("n_slabs", [2, 3, 4])
def test_c_slabs_equal_python_orchestrator(n_slabs):
    """S C++ slabs == the Python SlabSolver with the same S slabs (fused vs
    unfused colour passes: same arithmetic), to rounding."""
    pb = make_problem(3, n=8, N=7, seed=212)
    _, _, (ps, pst) = setup(pb, list(range(n_slabs)), n_slabs, 2)
    _, _, (cs, cst) = c_setup(pb, list(range(n_slabs)), n_slabs, 2)
    for _ in range(2):
        ps.vcycle(pst)
        ps.gauge(pst)
        cs.vcycle(cst)
        cs.gauge(cst)
    for a, b in zip(cst, pst):
        x, y = flat_dev(a), flat_dev(b)
        assert np.max(np.abs(x - y)) <= 1e-13 * np.max(np.abs(y))
    ri_c, r2_c = cs.norms(cst)
    ri_p, r2_p = ps.norms(pst)
    assert abs(ri_c - ri_p) <= 1e-12 * ri_p and abs(r2_c - r2_p) <= 1e-12 * r2_p
    cs.close()
    ps.close()


@pytest.mark.parametrize("dim", [2, 3])
def test_c_two_slabs_match_oracle_slabs(dim):
    n = 16 if dim == 2 else 8
    pb = make_problem(dim, n=n, N=6, seed=202)
    _, _, (cs, cst) = c_setup(pb, [0, 1], 2, 2)
    osolver, ostates = build_oracle_solver(pb, 2, [0, 1], 2)
    for _ in range(2):
        cs.vcycle(cst)
        cs.gauge(cst)
        osolver.vcycle(ostates)
        osolver.gauge(ostates)
    for d, o in zip(cst, ostates):
        a, b = flat_dev(d), flat_np(o)
        assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))
    cs.close()


def test_c_four_slabs_converge_to_single_slab_solution():
    pb = make_problem(2, n=16, N=8, seed=203)
    _, _, (one, s1) = c_setup(pb, [0], 1, 3)
    one.solve(s1, eps=1e-10, cycle_budget=80)
    _, _, (four, s4) = c_setup(pb, [0, 1, 2, 3], 4, 3)
    h4 = four.solve(s4, eps=1e-10, cycle_budget=120)
    assert h4[-1][1] <= 1e-10
    V = [np.concatenate([st.numpy()[0][k] for st in s4]) for k in range(2)]
    U = [np.concatenate([st.numpy()[2][k] for st in s4]) for k in range(2)]
    V1, _, U1, _ = s1[0].numpy()
    scale = max(np.max(np.abs(x)) for x in V1 + U1)
    err = max(np.max(np.abs(x - y)) for x, y in zip(V + U, list(V1) + list(U1)))
    assert err <= 1e-8 * scale
    one.close()
    four.close()


def test_c_slabs_over_a_one_rank_nccl_world(monkeypatch):
    """The NCCL branch of the C++ slab set on the one GPU a test box has: a
    one-rank world (unique id from libsmk's dlopen'ed NCCL, broadcast by
    NcclSlabComm over a world_size-1 process group) creates a communicator
    with ncclCommInitRank on the device and reduces the stop-test norms
    through ncclAllReduce on the compute stream.  With SMK_SLABS_NCCL_LOCAL=1
    the halos between the local slabs travel by ncclSend / ncclRecv (to the
    rank itself) inside the captured V-cycle graph -- the remote-neighbour
    path, first V-cycle captured, the others replayed.  Both must equal the
    same slabs without NCCL bit for bit.  (A neighbour on another GPU needs a
    second GPU: the driver's scaling run.)"""
    import os
    import socket
    import torch.distributed as dist
    from paper_1608_01102_b200.slabs import NcclSlabComm, build_c_solver
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = NcclSlabComm()
        assert (comm.rank, comm.world) == (0, 1) and len(comm.uid) == 128 and any(comm.uid)
        pb = make_problem(3, n=8, N=7, seed=213)
        spec, cfg, (plain, pst) = c_setup(pb, [0, 1, 2], 3, 2)
        nc, nst = build_c_solver(spec, cfg, pb.v0, pb.vstar, [0, 1, 2], 3, pb.N, torch.float64, comm=comm)
        monkeypatch.setenv("SMK_SLABS_NCCL_LOCAL", "1")
        lb, lst = build_c_solver(spec, cfg, pb.v0, pb.vstar, [0, 1, 2], 3, pb.N, torch.float64, comm=NcclSlabComm())
        monkeypatch.delenv("SMK_SLABS_NCCL_LOCAL")
        for _ in range(3):
            for sv, st in ((plain, pst), (nc, nst), (lb, lst)):
                sv.vcycle(st)
                sv.gauge(st)
        for a, b, c in zip(nst, pst, lst):
            assert np.array_equal(flat_dev(a), flat_dev(b))
            assert np.array_equal(flat_dev(c), flat_dev(b))
        assert nc.norms(nst) == plain.norms(pst) == lb.norms(lst)
        for sv in (lb, nc, plain):
            sv.close()
    finally:
        dist.destroy_process_group()
