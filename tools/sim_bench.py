"""Time the GPU forward step (simulator.step, fp64 like the reference) per
BASELINE config from rest with a smooth control force, wall clock per step
(incl. its read-backs).  The reference's simulator.step on this container's
CPU is in BASELINE.md §2 (27 / 113 / - / 2670 ms at cfg1 / 2 / - / 4).

    python tools/sim_bench.py [cfg ...]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1608_01102_b200 import simulator as S, workloads  # noqa: E402
from paper_1608_01102_b200.fields import ScalarField, StaggeredVectorField  # noqa: E402


def main(cfgs):
    for c in cfgs:
        w = workloads.config(c, torch.float64)
        spec = w.spec
        u = StaggeredVectorField(spec, tuple(x[0] for x in workloads.guide_velocity(w, frames=1)))
        st = S.SimState.rest(spec, ScalarField(spec, workloads.initial_density(w).to(torch.float64)))
        cfg = S.SimConfig(dt=w.dt)
        st = S.step(st, u, cfg, accept_stall=True)   # warm-up, and a non-rest state
        torch.cuda.synchronize()
        reps = 5
        t = time.perf_counter()
        for _ in range(reps):
            out = S.step(st, u, cfg, accept_stall=True)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) / reps * 1e3
        print(json.dumps({"config": w.name.replace("fp32", "fp64"), "step_ms": ms,
                          "cells_per_s": w.n ** w.dim / (ms / 1e3), "dtype": "f64"}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 4])
