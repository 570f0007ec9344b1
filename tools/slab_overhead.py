"""Host overhead of the Python slab orchestrator on one GPU: cfg5 V-cycle
through slabs.SlabSolver with 1 and 8 in-process slabs (SingleComm) vs the
C++ hierarchy V-cycle (CUDA graph).  Device-timed; prints one JSON line."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1608_01102_b200 import _lib, nso, slabs, workloads  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1000 / reps


def main():
    cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    w = workloads.config(cfg_i)
    _lib.load()
    vstar = workloads.guide_velocity(w)
    v0 = workloads.initial_velocity(w)
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=w.levels)
    out = {"workload": w.name}
    h = nso.StfasHierarchy(w.spec, cfg, w.N, w.dtype)
    h.set_guide(v0, vstar)
    st = nso.SpacetimeState.zeros(w.spec, w.N, w.dtype)
    out["hier_ms"], out["hier_wall_ms"] = timed(lambda: h.vcycle(st))
    h.close()
    del st
    torch.cuda.empty_cache()
    for n in (1, 8):
        solver, states = slabs.build_lib_solver(w.spec, cfg, v0, vstar, list(range(n)), n, w.N, w.dtype)
        out[f"slabs{n}_ms"], out[f"slabs{n}_wall_ms"] = timed(lambda: solver.vcycle(states))
        for e in solver.E:
            e.hier.close()
        del solver, states
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
