"""Per-rank view of an N-slab run on one GPU: build only slab `rank` of
`n` with a no-op halo exchange, and compare the host time to submit one
V-cycle with the device time of that V-cycle.  Host >= device means the
rank is host-bound (the orchestrator, not the GPU, sets the pace)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1608_01102_b200 import _lib, nso, slabs, workloads  # noqa: E402


class NullComm(slabs.SingleComm):
    host_sync = False

    def __init__(self, rank, world):
        self.rank, self.world = rank, world


def main():
    cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    rank = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    w = workloads.config(cfgno)
    _lib.load()
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=w.levels)
    solver, states = slabs.build_lib_solver(w.spec, cfg, workloads.initial_velocity(w), workloads.guide_velocity(w),
                                            [rank], n, w.N, w.dtype, comm=NullComm(rank, n))
    for _ in range(3):
        solver.vcycle(states)
    torch.cuda.synchronize()
    hs, ds = [], []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        t = time.perf_counter()
        solver.vcycle(states)
        hs.append((time.perf_counter() - t) * 1e3)
        b.record()
        torch.cuda.synchronize()
        ds.append(a.elapsed_time(b))
    print(f"cfg{cfgno} slab {rank}/{n}: host submit {min(hs):.2f} ms, device {min(ds):.2f} ms "
          f"(single-GPU whole problem /{n} for comparison)")


if __name__ == "__main__":
    main()
