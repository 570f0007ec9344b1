"""STFAS convergence study on one GPU: residual history, V-cycles to eps and
time to solution per (config, dtype, levels, coarsest sweeps).

    python tools/conv_study.py --config 5 --levels 4 6 --n-coarse 10 --budget 60
Prints one JSON line per run.  Each V-cycle is timed with CUDA events
including the per-cycle stop test (k_kkt + norms) -- what solve_nso runs.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1608_01102_b200 import nso, workloads  # noqa: E402


def run(w, levels, n_coarse, budget, eps_rel, nu=(2, 2), color_mod=2, omega=0.8, red_black=True):
    spec = w.spec
    vstar = workloads.guide_velocity(w)
    v0 = workloads.initial_velocity(w)
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=levels, n_coarse=n_coarse, nu1=nu[0], nu2=nu[1],
                          color_mod=color_mod, omega=omega, red_black=red_black)
    hier = nso.StfasHierarchy(spec, cfg, w.N, w.dtype)
    hier.set_guide(v0, vstar)
    st = nso.SpacetimeState.zeros(spec, w.N, w.dtype)
    # warm (graph capture) on a scratch copy
    sc = st.copy()
    hier.vcycle(sc)
    torch.cuda.synchronize()
    del sc
    f0, l20 = hier.residual_norms(st)
    hist = [(0, f0, l20, 0.0)]
    t_tot = 0.0
    reached = None
    for c in range(1, budget + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        hier.vcycle(st)
        hier.gauge_fix(st)
        ri, r2 = hier.residual_norms(st)
        e1.record()
        e1.synchronize()
        t_tot += e0.elapsed_time(e1)
        hist.append((c, ri, r2, t_tot))
        if reached is None and ri <= eps_rel * f0:
            reached = (c, t_tot)
            break
        if not (ri == ri) or ri > 1e6 * f0:
            break
    facs = [hist[i + 1][1] / hist[i][1] for i in range(len(hist) - 1) if hist[i][1] > 0]
    tail = facs[-5:]
    asym = (hist[-1][1] / hist[-1 - len(tail)][1]) ** (1.0 / len(tail)) if tail else None
    out = {"config": w.index, "dtype": str(w.dtype).replace("torch.", ""), "levels": hier.levels,
           "n_coarse": n_coarse, "nu": list(nu), "color_mod": color_mod, "red_black": red_black, "omega": omega,
           "f0_inf": f0, "eps_rel": eps_rel, "vcycles_to_eps": reached[0] if reached else None,
           "s_to_solution": reached[1] / 1000.0 if reached else None,
           "ms_per_cycle_incl_stop": t_tot / max(1, len(hist) - 1), "asym_factor": asym,
           "res_inf": [h[1] for h in hist], "device_bytes": hier.device_bytes}
    hier.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, nargs="+", default=[5])
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--levels", type=int, nargs="+", default=[0])
    ap.add_argument("--n-coarse", type=int, nargs="+", default=[10])
    ap.add_argument("--budget", type=int, default=60)
    ap.add_argument("--eps", type=float, default=1e-5)
    ap.add_argument("--color-mod", type=int, default=2)
    ap.add_argument("--omega", type=float, default=0.8)
    ap.add_argument("--mod", action="store_true", help="mod-m colouring instead of red-black")
    a = ap.parse_args()
    dt = {"fp32": torch.float32, "fp64": torch.float64}.get(a.dtype)
    for ci in a.config:
        w = workloads.config(ci, dt)
        for lv in a.levels:
            for nc in a.n_coarse:
                t = time.time()
                o = run(w, lv if lv > 0 else w.levels, nc, a.budget, a.eps, color_mod=a.color_mod, omega=a.omega,
                        red_black=not a.mod)
                o["wall_s"] = time.time() - t
                print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
