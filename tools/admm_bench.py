"""Time-to-solution of the GPU ADMM loop (admm.run) on a BASELINE config:
one Gaussian keyframe at t = N, K = r = 1e3, eps_STFAS = 1e-5, fp64.
Prints one JSON line with the outer iterations, their log and wall time.

    python tools/admm_bench.py [cfg] [max_outer] [K]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1608_01102_b200 import admm, ao, workloads  # noqa: E402
from paper_1608_01102_b200.errors import MaxIterations, SmokeCtrlError  # noqa: E402


def main(c, max_outer, K=None):
    w = workloads.config(c, torch.float64)
    spec = w.spec
    rho0 = workloads.initial_density(w).to(torch.float64)
    centre = (0.5, 0.7) + ((0.5,) if w.dim == 3 else ())
    target = workloads.gaussian(spec, centre, 0.1)
    kf = ao.KeyframeSet(w.N, {w.N: target})
    cfg = admm.AdmmConfig(dt=w.dt, K=K or w.K, r=w.r, max_outer=max_outer, n_levels=w.levels)
    torch.cuda.synchronize()
    t = time.perf_counter()
    status = "converged"
    try:
        res = admm.run(spec, rho0, kf, cfg)
    except MaxIterations as e:
        res, status = e.result, "max_outer"
    except SmokeCtrlError as e:
        print(json.dumps({"config": w.name, "error": str(e)}))
        return
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    obj = admm.objective(res.rho, kf, res.u, w.r)
    print(json.dumps({"config": w.name.replace("fp32", "fp64"), "K": cfg.K, "r": cfg.r, "status": status, "outer": len(res.logs),
                      "wall_s": wall, "s_per_outer": wall / len(res.logs), "objective": obj,
                      "logs": res.logs}), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2, int(sys.argv[2]) if len(sys.argv) > 2 else 10,
         float(sys.argv[3]) if len(sys.argv) > 3 else None)
