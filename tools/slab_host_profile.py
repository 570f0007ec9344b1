"""cProfile of the slab orchestrator's host side: cfg5 with 8 in-process
slabs on one GPU (the per-rank call pattern of an 8-GPU run)."""
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1608_01102_b200 import _lib, nso, slabs, workloads  # noqa: E402


def main():
    w = workloads.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    _lib.load()
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=w.levels)
    solver, states = slabs.build_lib_solver(w.spec, cfg, workloads.initial_velocity(w), workloads.guide_velocity(w),
                                            list(range(n)), n, w.N, w.dtype)
    solver.vcycle(states)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    solver.vcycle(states)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
