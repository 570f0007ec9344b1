"""Command-line surface (SPEC.md:474-518 cli_io; ``smokectrl.cli:main``,
pkg/pyproject.toml:15-16).

    python -m paper_1608_01102_b200.cli optimize --config run.cfg --out out/ [--threads k] [--lm] [--fallback] [--safeguard]
    python -m paper_1608_01102_b200.cli simulate --config run.cfg --out out/ [--forces dir]
    python -m paper_1608_01102_b200.cli compare-baseline --config run.cfg --out out/
    python -m paper_1608_01102_b200.cli make-benchmark --name translated-blob --res 32 --frames 10 --out bench/
    python -m paper_1608_01102_b200.cli export-frames --in out/ --out frames/ [--field rho] [--axis 2] [--slice k]

Exit codes: 0 success; 2 usage (unknown subcommand / bad flags, usage text on
stderr); 3 MaxIterations (the best-so-far result is still written); 1 any
other error -- with a machine-readable JSON object on stderr
({"error": <class>, "message": ...}).  Every field file is SMKF
(fileio.py); output names are <field>_<frame:04d>.smkf.
"""

import argparse
import glob
import json
import os
import re
import sys
import time

import numpy as np

from . import fileio
from .errors import FormatError, MaxIterations, SmokeCtrlError

SUBCOMMANDS = ("optimize", "simulate", "compare-baseline", "make-benchmark", "export-frames")


def _parser():
    ap = argparse.ArgumentParser(prog="smokectrl", description="Keyframe smoke control (ADMM + STFAS on B200)")
    sub = ap.add_subparsers(dest="cmd", required=True, metavar="{" + ",".join(SUBCOMMANDS) + "}")
    o = sub.add_parser("optimize", help="run the ADMM controller (SPEC.md:376-426)")
    o.add_argument("--config", required=True)
    o.add_argument("--out", required=True)
    o.add_argument("--threads", type=int, default=None)
    o.add_argument("--lm", action="store_true")
    o.add_argument("--fallback", action="store_true")
    o.add_argument("--safeguard", action="store_true")
    s = sub.add_parser("simulate", help="forward rollout from a config (zero or given forces)")
    s.add_argument("--config", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("--forces", default=None, help="directory with u_XXXX.smkf (default: zero forces)")
    c = sub.add_parser("compare-baseline", help="ADMM vs the LBFGS adjoint baseline: timing table")
    c.add_argument("--config", required=True)
    c.add_argument("--out", required=True)
    m = sub.add_parser("make-benchmark", help="synthesise a desk-scale keyframe benchmark")
    m.add_argument("--name", required=True, choices=BENCHMARKS)
    m.add_argument("--res", type=int, default=32)
    m.add_argument("--frames", type=int, default=10)
    m.add_argument("--dim", type=int, default=2, choices=(2, 3))
    m.add_argument("--seed", type=int, default=0)
    m.add_argument("--out", required=True)
    e = sub.add_parser("export-frames", help="per-frame PGM slices of SMKF outputs")
    e.add_argument("--in", dest="inp", required=True)
    e.add_argument("--out", required=True)
    e.add_argument("--field", default="rho")
    e.add_argument("--axis", type=int, default=None, help="3D: slice axis (default: last)")
    e.add_argument("--slice", type=int, default=None, help="3D: slice index (default: middle)")
    return ap


# ---------------------------------------------------------------------------
# benchmarks (circle->letter, circle->two circles->silhouette,
# translated blob), deterministic in the seed
# ---------------------------------------------------------------------------

BENCHMARKS = ("translated-blob", "circle-letter", "circles")


def _centres(spec):
    ax = [(np.arange(n) + 0.5) * spec.h for n in spec.res]
    return np.meshgrid(*ax, indexing="ij")


def _disc(x, c, r, h):
    d = np.sqrt(sum((xi - ci) ** 2 for xi, ci in zip(x, c)))
    t = np.clip((d - (r - h)) / (2 * h), 0.0, 1.0)
    return 1.0 - t * t * (3.0 - 2.0 * t)


def _blob(x, c, sigma):
    return np.exp(-sum((xi - ci) ** 2 for xi, ci in zip(x, c)) / (2 * sigma * sigma))


def make_benchmark(name, res, frames, dim=2, seed=0):
    """(RunConfig, initial density, {timestep: keyframe}) of a benchmark."""
    spec = fileio.GridSpec(dim, (res,) * dim, 1.0 / res, "neumann")
    x = _centres(spec)
    rng = np.random.default_rng(seed)
    jit = lambda: rng.uniform(-0.02, 0.02, size=dim)
    mid = [0.5] * dim
    if name == "translated-blob":
        c0 = np.array([0.3] + mid[1:]) + jit()
        c1 = np.array([0.7] + mid[1:]) + jit()
        rho0 = _blob(x, c0, 0.08)
        kfs = {frames: _blob(x, c1, 0.08)}
    elif name == "circle-letter":
        rho0 = _disc(x, np.array([0.5, 0.3] + mid[2:]) + jit(), 0.15, spec.h)
        inside = lambda a0, a1, b0, b1: ((x[0] >= a0) & (x[0] <= a1) & (x[1] >= b0) & (x[1] <= b1))
        f = inside(0.35, 0.45, 0.3, 0.8) | inside(0.35, 0.7, 0.7, 0.8) | inside(0.35, 0.6, 0.5, 0.58)
        kfs = {frames: f.astype(np.float64)}
    elif name == "circles":
        rho0 = _disc(x, np.array([0.5, 0.3] + mid[2:]) + jit(), 0.15, spec.h)
        two = np.maximum(_disc(x, np.array([0.35, 0.55] + mid[2:]) + jit(), 0.1, spec.h),
                         _disc(x, np.array([0.65, 0.55] + mid[2:]) + jit(), 0.1, spec.h))
        # silhouette analogue: body ellipse + head disc + two ear ellipses
        e = lambda c, ax_: np.clip(1.0 - sum(((xi - ci) / ai) ** 2 for xi, ci, ai in zip(x, c, ax_)), 0.0, 1.0) > 0
        body = e([0.5, 0.45] + mid[2:], [0.2, 0.13] + [0.13] * (dim - 2))
        head = e([0.62, 0.62] + mid[2:], [0.09, 0.09] + [0.09] * (dim - 2))
        ears = e([0.6, 0.78] + mid[2:], [0.03, 0.1] + [0.03] * (dim - 2)) | \
            e([0.67, 0.77] + mid[2:], [0.03, 0.1] + [0.03] * (dim - 2))
        kfs = {max(1, frames // 2): two, frames: (body | head | ears).astype(np.float64)}
    else:
        raise SmokeCtrlError(f"unknown benchmark {name!r} (one of {', '.join(BENCHMARKS)})")
    cfg = fileio.RunConfig(dim=dim, res=(res,) * dim, frames=frames, seed=seed)
    return cfg, rho0, {int(t): np.asarray(v, dtype=np.float64) for t, v in kfs.items()}


# ---------------------------------------------------------------------------
# subcommands
# ---------------------------------------------------------------------------


def _dtype(cfg):
    import torch
    return torch.float32 if cfg.dtype == "float32" else torch.float64


def _inputs(cfg, base):
    from .ao import KeyframeSet
    spec = cfg.spec()
    rho0 = fileio.load_keyframe(os.path.join(base, cfg.initial_density), spec)
    kf = KeyframeSet(cfg.frames, {int(t): fileio.load_keyframe(os.path.join(base, p), spec)
                                  for t, p in cfg.keyframes.items()})
    return spec, rho0, kf


def _write_stack(out, name, spec, frames):
    for i, f in enumerate(frames):
        fileio.save_smkf(os.path.join(out, f"{name}_{i:04d}.smkf"), spec, f)


def _write_result(out, spec, res, extra):
    n = res.rho.shape[0] - 1
    _write_stack(out, "rho", spec, [res.rho[i] for i in range(n + 1)])
    _write_stack(out, "v", spec, [tuple(c[i] for c in res.v) for i in range(n)])
    _write_stack(out, "u", spec, [tuple(c[i] for c in res.u) for i in range(n)])
    _write_stack(out, "vstar", spec, [tuple(c[i] for c in res.vstar) for i in range(n)])
    res.write_log_csv(os.path.join(out, "admm_log.csv"))
    res.write_vcycle_csv(os.path.join(out, "vcycle_log.csv"))
    summary = {"converged": bool(res.converged), "outer_iterations": len(res.logs), **extra}
    with open(os.path.join(out, "result.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return summary


def cmd_optimize(args, cfg=None):
    from . import admm
    base = os.path.dirname(os.path.abspath(args.config))
    cfg = cfg or fileio.RunConfig.load(args.config)
    if args.lm:
        cfg.lm = True
    if args.fallback:
        cfg.fallback = True
    if args.safeguard:
        cfg.safeguard = True
    spec, rho0, kf = _inputs(cfg, base)
    os.makedirs(args.out, exist_ok=True)
    if cfg.solver == "lbfgs":
        return _run_lbfgs(cfg, spec, rho0, kf, args.out)
    acfg = admm.AdmmConfig(dt=cfg.timestep(), K=cfg.K, r=cfg.r, beta=cfg.beta, ao_iters=cfg.ao_iters,
                           eps_stfas=cfg.eps_stfas, eps_admm=cfg.eps_admm, max_outer=cfg.max_outer,
                           fallback=cfg.fallback, ao_safeguard=cfg.safeguard, lm=cfg.lm, n_levels=cfg.n_levels)
    t0 = time.perf_counter()
    try:
        res = admm.run(spec, rho0, kf, acfg, dtype=_dtype(cfg))
    except MaxIterations as e:
        if e.result is not None:
            _write_result(args.out, spec, e.result, {"wall_s": time.perf_counter() - t0, "max_iterations": True})
        raise
    obj = admm.objective(res.rho, kf, res.u, cfg.r)
    return _write_result(args.out, spec, res, {"wall_s": time.perf_counter() - t0, "objective": obj})


def _run_lbfgs(cfg, spec, rho0, kf, out):
    from . import lbfgs
    t0 = time.perf_counter()
    res = lbfgs.minimize(spec, rho0, kf, cfg.r, cfg.timestep(), dtype=_dtype(cfg))
    n = res.rho.shape[0] - 1
    _write_stack(out, "rho", spec, [res.rho[i] for i in range(n + 1)])
    _write_stack(out, "u", spec, [tuple(c[i] for c in res.u) for i in range(n)])
    summary = {"converged": bool(res.converged), "iterations": res.iterations, "objective": res.objective,
               "wall_s": time.perf_counter() - t0}
    with open(os.path.join(out, "result.json"), "w") as f:
        json.dump(summary, f, indent=1)
    return summary


def cmd_simulate(args):
    import torch
    from .fields import ScalarField, StaggeredVectorField
    from .simulator import SimConfig, SimState, simulate
    base = os.path.dirname(os.path.abspath(args.config))
    cfg = fileio.RunConfig.load(args.config)
    spec = cfg.spec()
    dt = _dtype(cfg)
    rho0 = fileio.load_keyframe(os.path.join(base, cfg.initial_density), spec)
    if args.forces:
        files = sorted(glob.glob(os.path.join(args.forces, "u_*.smkf")))
        if len(files) < cfg.frames:
            raise FormatError(f"{args.forces}: {len(files)} force files, need {cfg.frames}")
        forces = [StaggeredVectorField(spec, fileio.load_smkf(p, spec), dt) for p in files[:cfg.frames]]
    else:
        forces = [StaggeredVectorField.zeros(spec, dt) for _ in range(cfg.frames)]
    st0 = SimState.rest(spec, ScalarField(spec, torch.as_tensor(rho0), dt))
    states = simulate(st0, forces, SimConfig(dt=cfg.timestep()))
    os.makedirs(args.out, exist_ok=True)
    _write_stack(args.out, "rho", spec, [s.rho.values for s in states])
    _write_stack(args.out, "v", spec, [s.v.comps for s in states])
    return {"frames": len(states)}


def cmd_compare(args):
    cfg = fileio.RunConfig.load(args.config)
    os.makedirs(args.out, exist_ok=True)
    rows = []
    for solver in ("admm", "lbfgs"):
        cfg.solver = solver
        ns = argparse.Namespace(config=args.config, out=os.path.join(args.out, solver), lm=False, fallback=False,
                                safeguard=False, threads=None)
        summ = cmd_optimize(ns, cfg)
        rows.append({"solver": solver, "wall_s": summ["wall_s"], "objective": summ.get("objective"),
                     "converged": summ["converged"]})
    with open(os.path.join(args.out, "timing.csv"), "w") as f:
        f.write("solver,wall_s,objective,converged\n")
        for r in rows:
            f.write(f"{r['solver']},{r['wall_s']:.6g},{r['objective']},{r['converged']}\n")
    for r in rows:
        print(f"{r['solver']:6s} {r['wall_s']:10.3f} s  objective {r['objective']}  converged {r['converged']}")
    return {"rows": rows}


def cmd_make_benchmark(args):
    cfg, rho0, kfs = make_benchmark(args.name, args.res, args.frames, args.dim, args.seed)
    os.makedirs(args.out, exist_ok=True)
    spec = cfg.spec()
    fileio.save_smkf(os.path.join(args.out, "initial.smkf"), spec, rho0)
    for t, v in kfs.items():
        p = f"keyframe_{t:04d}.smkf"
        fileio.save_smkf(os.path.join(args.out, p), spec, v)
        cfg.keyframes[t] = p
    cfg.save(os.path.join(args.out, "run.cfg"))
    return {"config": os.path.join(args.out, "run.cfg"), "keyframes": sorted(kfs)}


def cmd_export(args):
    files = sorted(glob.glob(os.path.join(args.inp, f"{args.field}_*.smkf")))
    if not files:
        raise FormatError(f"{args.inp}: no {args.field}_*.smkf files")
    os.makedirs(args.out, exist_ok=True)
    for p in files:
        spec, kind, vals = fileio.read_smkf(p)
        if kind != fileio.KIND_CELL:
            raise FormatError(f"{p}: export-frames writes cell scalar fields")
        a = vals
        if spec.dim == 3:
            ax = 2 if args.axis is None else args.axis
            k = spec.res[ax] // 2 if args.slice is None else args.slice
            a = np.take(a, k, axis=ax)
        m = re.search(r"_(\d+)\.smkf$", p)
        fileio.write_pgm(os.path.join(args.out, f"{args.field}_{m.group(1)}.pgm"), a)
    return {"frames": len(files)}


COMMANDS = {"optimize": cmd_optimize, "simulate": cmd_simulate, "compare-baseline": cmd_compare,
            "make-benchmark": cmd_make_benchmark, "export-frames": cmd_export}


def main(argv=None):
    ap = _parser()
    args = ap.parse_args(argv)   # usage errors: argparse exits 2 with the usage text
    if getattr(args, "threads", None):
        import torch
        torch.set_num_threads(args.threads)
    try:
        out = COMMANDS[args.cmd](args)
    except MaxIterations as e:
        sys.stderr.write(json.dumps({"error": "MaxIterations", "message": str(e)}) + "\n")
        return 3
    except (SmokeCtrlError, OSError, ValueError) as e:
        sys.stderr.write(json.dumps({"error": type(e).__name__, "message": str(e)}) + "\n")
        return 1
    print(json.dumps(out, default=float))
    return 0


if __name__ == "__main__":
    sys.exit(main())
