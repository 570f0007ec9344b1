"""Schwarz-in-time degradation of the slab STFAS on one GPU: the config's
problem split into S = 1, 2, 4, 8 contiguous time slabs (in-process, halos by
device copies -- the same orchestration the multi-GPU run uses),
solved to ||f||_inf <= eps (fp32: relative to ||f_0||, fp64: absolute), for
the config's hierarchy depth and the full-depth one.

    python tools/slab_convergence.py [--config 5] [--slabs 1 2 4 8] [--levels 0 99] [--budget 80]

One JSON line per (S, levels): V-cycles to eps, asymptotic factor, residual
history, device ms per V-cycle (all slabs serialised on one GPU: a convergence
study, not a timing of the multi-GPU run).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1608_01102_b200 import _lib, nso, slabs, workloads  # noqa: E402


def run(w, S, levels, budget, solver_kind):
    vstar = workloads.guide_velocity(w)
    v0 = workloads.initial_velocity(w)
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=levels or w.levels)
    if solver_kind == "c":
        solver, states = slabs.build_c_solver(w.spec, cfg, v0, vstar, list(range(S)), S, w.N, w.dtype)
    else:
        solver, states = slabs.build_lib_solver(w.spec, cfg, v0, vstar, list(range(S)), S, w.N, w.dtype)
    f0, _ = solver.norms(states)
    rel = w.dtype == torch.float32
    tol = 1e-5 * f0 if rel else 1e-5
    hist, ms, reached = [f0], 0.0, None
    for c in range(1, budget + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        solver.vcycle(states)
        solver.gauge(states)
        e1.record()
        ri, _ = solver.norms(states)
        ms += e0.elapsed_time(e1)
        hist.append(ri)
        if ri <= tol:
            reached = c
            break
    out = {"workload": w.name, "slabs": S, "levels": solver.L if hasattr(solver, "L") else solver.levels,
           "solver": solver_kind, "f0_inf": f0, "eps": 1e-5, "eps_kind": "relative" if rel else "absolute",
           "vcycles_to_eps": reached, "final": hist[-1],
           "asym_factor": (hist[-1] / hist[-4]) ** (1 / 3) if len(hist) >= 4 and hist[-4] > 0 else None,
           "ms_per_vcycle_serialised": ms / max(1, len(hist) - 1),
           "residual_history": [float(f"{x:.4e}") for x in hist]}
    solver.close()
    del solver, states
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--slabs", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--levels", type=int, nargs="+", default=[0, 99])
    ap.add_argument("--budget", type=int, default=80)
    ap.add_argument("--solver", default="c", choices=["c", "python"])
    args = ap.parse_args()
    _lib.load()
    w = workloads.config(args.config)
    for lv in args.levels:
        for S in args.slabs:
            print(json.dumps(run(w, S, lv, args.budget, args.solver)), flush=True)


if __name__ == "__main__":
    main()
