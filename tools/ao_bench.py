"""Time one GPU AO sweep (ao.ao_sweep) per BASELINE config, fp64 like the
reference, and print one JSON line per config: ms per frame (wall clock of
the whole sweep incl. the per-frame Taylor-order read-backs, / N) and
cell-frames/s.  The reference's own ao_sweep per frame on this container's
CPU is in BASELINE.md §2 (9 / 34 / - / 750 ms at cfg1 / 2 / - / 4).

    python tools/ao_bench.py [cfg ...]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1608_01102_b200 import ao, workloads  # noqa: E402


def main(cfgs):
    for c in cfgs:
        w = workloads.config(c, torch.float64)
        spec = w.spec
        vg = workloads.guide_velocity(w)
        rho0 = workloads.initial_density(w).to(torch.float64)
        centre = (0.5, 0.7) + ((0.5,) if w.dim == 3 else ())
        target = workloads.gaussian(spec, centre, 0.1)
        kf = ao.KeyframeSet(w.N, {w.N: target})
        metric = ao.GaussianMetric(spec)
        cfg = ao.AoConfig(K=w.K, dt=w.dt)
        state = ao.AoState(vstar=tuple(x.clone() for x in vg), mu=torch.zeros((w.N,) + spec.res, dtype=torch.float64,
                                                                               device="cuda"),
                           rho=rho0.unsqueeze(0).expand((w.N + 1,) + spec.res).contiguous())
        ao.ao_sweep(spec, state, vg, kf, metric, cfg)   # warm-up
        torch.cuda.synchronize()
        reps = 3
        t = time.perf_counter()
        for _ in range(reps):
            res = ao.ao_sweep(spec, state, vg, kf, metric, cfg)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / reps
        print(json.dumps({"config": w.name.replace("fp32", "fp64"), "ao_sweep_ms": dt * 1e3,
                          "ms_per_frame": dt * 1e3 / w.N, "cell_frames_per_s": w.n ** w.dim * w.N / dt,
                          "ks": res.ks[:4], "dtype": "f64"}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 4])
