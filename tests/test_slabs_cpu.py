"""Time-slab (multi-GPU) orchestration on CPU: world_size-2 gloo ranks and
in-process slabs run the identical algorithm; the slab solver converges to
the single-slab solution."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import stfas
from problems import make_problem
from slab_oracle import build_oracle_solver

N_LEVELS = 2


def problem():
    return make_problem(2, n=8, N=6, seed=123)


def flat(st):
    return np.concatenate([a.ravel() for a in st.V + (st.PB,) + st.U + (st.P,)])


def concat_slabs(states):
    return stfas.State(tuple(np.concatenate([s.V[k] for s in states]) for k in range(len(states[0].V))),
                       np.concatenate([s.PB for s in states]),
                       tuple(np.concatenate([s.U[k] for s in states]) for k in range(len(states[0].U))),
                       np.concatenate([s.P for s in states]))


def test_split_frames():
    from paper_1608_01102_b200.slabs import split_frames
    assert split_frames(80, 8) == [(10 * i, 10 * i + 10) for i in range(8)]
    assert split_frames(7, 3) == [(0, 3), (3, 5), (5, 7)]


def test_single_slab_is_the_oracle_vcycle():
    pb = problem()
    solver, states = build_oracle_solver(pb, N_LEVELS, [0], 1)
    solver.vcycle(states)
    want = stfas.vcycle(stfas.build_levels(pb, N_LEVELS), 0, stfas.zero_state(pb.g, pb.N))
    assert np.max(np.abs(flat(states[0]) - flat(want))) <= 1e-13 * np.max(np.abs(flat(want)))


def test_slabs_converge_to_single_slab_solution():
    pb = problem()
    one, s1 = build_oracle_solver(pb, N_LEVELS, [0], 1)
    h1 = one.solve(s1, eps=1e-10, cycle_budget=60)
    two, s2 = build_oracle_solver(pb, N_LEVELS, [0, 1], 2)
    h2 = two.solve(s2, eps=1e-10, cycle_budget=80)
    assert h1[-1][1] <= 1e-10 and h2[-1][1] <= 1e-10
    a, b = flat(s1[0]), flat(concat_slabs(s2))
    assert np.max(np.abs(a - b)) <= 1e-7 * np.max(np.abs(a))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir, cycles):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1608_01102_b200.slabs import TorchComm
    pb = problem()
    solver, states = build_oracle_solver(pb, N_LEVELS, [rank], world, comm=TorchComm())
    hist = []
    for _ in range(cycles):
        solver.vcycle(states)
        solver.gauge(states)
        hist.append(solver.norms(states)[0])
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), flat(states[0]))
    np.save(os.path.join(out_dir, f"hist{rank}.npy"), np.array(hist))
    dist.destroy_process_group()


def test_gloo_two_ranks_equal_in_process_slabs(tmp_path):
    cycles = 3
    port = _free_port()
    mp.spawn(_rank_main, args=(2, port, str(tmp_path), cycles), nprocs=2, join=True)
    pb = problem()
    solver, states = build_oracle_solver(pb, N_LEVELS, [0, 1], 2)
    hist = []
    for _ in range(cycles):
        solver.vcycle(states)
        solver.gauge(states)
        hist.append(solver.norms(states)[0])
    for r in range(2):
        got = np.load(os.path.join(tmp_path, f"rank{r}.npy"))
        assert np.array_equal(got, flat(states[r]))
        assert np.allclose(np.load(os.path.join(tmp_path, f"hist{r}.npy")), hist, rtol=1e-14, atol=0)


def test_nccl_loader_and_unique_id():
    """libsmk loads NCCL with dlopen and resolves every entry point the C++
    slab set calls (smk_stfas.cu NcclApi); rank 0's unique id is 128 bytes,
    not all zero, and differs between calls."""
    import ctypes
    from paper_1608_01102_b200 import _lib
    L = _lib.load()
    ids = []
    for _ in range(2):
        raw = (ctypes.c_ubyte * 128)()
        _lib.check(L.smk_nccl_unique_id(ctypes.cast(raw, ctypes.c_void_p), 128), "nccl_unique_id")
        ids.append(bytes(raw))
    assert any(ids[0]) and ids[0] != ids[1]
    small = (ctypes.c_ubyte * 16)()
    assert L.smk_nccl_unique_id(ctypes.cast(small, ctypes.c_void_p), 16) == _lib.SMK_ERR_ARG


def _uid_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1608_01102_b200.slabs import NcclSlabComm
    comm = NcclSlabComm()
    assert (comm.rank, comm.world) == (rank, world)
    with open(os.path.join(out_dir, f"uid{rank}.bin"), "wb") as f:
        f.write(comm.uid)
    dist.destroy_process_group()


def test_nccl_unique_id_reaches_every_rank(tmp_path):
    """NcclSlabComm: rank 0's id broadcast over torch.distributed (gloo here,
    world_size 2) -- both ranks hand the same 128 bytes to smk_slabs_create."""
    port = _free_port()
    mp.spawn(_uid_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    a = open(os.path.join(tmp_path, "uid0.bin"), "rb").read()
    b = open(os.path.join(tmp_path, "uid1.bin"), "rb").read()
    assert len(a) == 128 and any(a) and a == b
