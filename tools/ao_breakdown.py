"""Per-operator wall-clock breakdown of one AO frame (fp64) at a BASELINE
config: forward Taylor advection, rho-adjoint, v-adjoint, projection and the
keyframe metric.  python tools/ao_breakdown.py [cfg]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1608_01102_b200 import advection as A, ao, fields as F, workloads  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3, out


def main(c):
    w = workloads.config(c, torch.float64)
    spec = w.spec
    vg = workloads.guide_velocity(w, frames=2)
    v = tuple(x[0] for x in vg)
    rho = workloads.initial_density(w).to(torch.float64)
    mu = rho.flip(0).contiguous()
    res = {}
    res["advect_scalar"], (_, rep) = timed(lambda: A.advect_scalar(spec, v, rho, w.dt))
    k = rep.k_used
    res["advect_rho_T"], _ = timed(lambda: A.advect_scalar_rho_T(spec, v, mu, w.dt, k_fixed=k))
    res["advect_v_T"], (f, _) = timed(lambda: A.advect_scalar_v_T(spec, v, rho, mu, w.dt, k_fixed=k))
    raw = tuple(a + b / w.K for a, b in zip(v, f))
    res["project_arrays_1e-9"], _ = timed(lambda: F.project_arrays(spec, raw, 1e-9))
    m = ao.GaussianMetric(spec)
    res["metric_apply"], _ = timed(lambda: m.apply(rho))
    print(json.dumps({"config": w.name, "k": k, "ms": {a: round(b, 3) for a, b in res.items()}}), flush=True)


if __name__ == "__main__":
    for c in [int(a) for a in sys.argv[1:]] or [2, 4]:
        main(c)
