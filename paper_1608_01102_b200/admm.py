"""ADMM outer loop on B200 (SPEC.md:376-426 admm_driver; Alg. 3).

The direct caller of the STFAS solve: alternate the AO step
(``ao.solve_ao``, guiding v + lambda/K) and the NSO step
(``nso.solve_nso`` to ||f||_inf <= eps_STFAS, warm-started from the previous
outer iteration's spacetime state), stop when the maximal visual
difference max_i ||rho_i^last - rho_i||_inf < eps_ADMM (rho from the rollout
under the AO's v*, the SPEC's design decision), else update
lambda += K beta (v - v*) (Alg. 3 order: only when the test fails).

Frozen choices shared with ``oracle/admm.py``: v_0 is pinned
(``v0``, zero by default) and v_i = V[i-1] of the NSO state for i >= 1; the
NSO guide is v* - lambda/K (the lambda^T (v - v*) term completed into the
K/2 square).  Everything is device-resident; the host only reads back the
scalars of the stop test and the logs.
"""

import csv
import time
from dataclasses import dataclass, field

import torch

from . import _dev
from .ao import AoConfig, GaussianMetric, KeyframeSet, _axpby, _objective_dev, _rollout_dev, solve_ao
from .errors import MaxIterations, SmokeCtrlError
from .fields import dot_fields, inf_norm
from .nso import SpacetimeState, StfasConfig, StfasHierarchy, _solve_lm


@dataclass
class AdmmConfig:
    """``SPEC.md:381-384`` (Table 1 defaults)."""

    dt: float
    K: float = 1e3
    r: float = 1e3
    beta: float = 1.0
    ao_iters: int = 2
    eps_stfas: float = 1e-5
    eps_admm: float = None          # None -> rho_max / 100 of the initial frame
    max_outer: int = 60
    fallback: bool = False          # suspend lambda updates while the augmented objective still drops
    fallback_tol: float = 1e-3      # ... by more than this relative amount per outer iteration
    ao_safeguard: bool = False
    nso_cycle_budget: int = 50
    relative_stfas: bool = False    # fp32: eps_STFAS relative to ||f_0||_inf
    n_levels: int = 99
    projection_tol: float = 1e-9
    lm: bool = False                # LM safeguard of the STFAS solves (nso._solve_lm)


@dataclass
class ControlResult:
    """``SPEC.md:385-388``: trajectory, forces, guides, multipliers, logs."""

    rho: torch.Tensor               # (N+1, *res), rollout under v*
    v: tuple                        # (N, face) stacks v_0 .. v_{N-1}
    u: tuple                        # (N, face) control forces u_0 .. u_{N-1}
    vstar: tuple
    lam: tuple
    state: SpacetimeState
    logs: list = field(default_factory=list)
    converged: bool = False
    vcycle_log: list = field(default_factory=list)   # (admm_iter, vcycle_index, residual_inf, residual_l2, wall_ms)
    best_outer_iter: int = None     # MaxIterations: the iteration these fields come from

    def write_log_csv(self, path):
        """Per-iteration CSV: outer_iter, ao_obj, nso_resid, visual_diff, wall_s."""
        with open(path, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=["outer_iter", "ao_obj", "nso_resid", "visual_diff", "wall_s"])
            w.writeheader()
            for row in self.logs:
                w.writerow(row)

    def write_vcycle_csv(self, path):
        """nso_solver convergence rows: admm_iter, vcycle_index,
        residual_inf, residual_l2, wall_ms (the solve's wall time averaged over
        its V-cycles: the cycles run back to back on the device)."""
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["admm_iter", "vcycle_index", "residual_inf", "residual_l2", "wall_ms"])
            w.writerows(self.vcycle_log)


def objective(rho, keyframes, u, r):
    """``SPEC.md:399-407``: 0.5 sum c_i |rho_i - rho*_i|^2 + (r/2) sum |u_i|^2 (unweighted)."""
    dt = rho.dtype
    mis = 0.0
    for i, t in keyframes.targets.items():
        d = _axpby(rho[i].clone(), _dev.as_dev(t, dt), -1.0, 1.0)
        mis += dot_fields((d,), (d,))
    return 0.5 * mis + 0.5 * r * dot_fields(tuple(u), tuple(u))


def _augmented(spec, cfg, rho, keyframes, s, v, vstar, lam):
    """Eq. 11 value: objective + lambda^T (v - v*) + K/2 |v - v*|^2 (for the fallback)."""
    d = tuple(_axpby(a.clone(), b, -1.0, 1.0) for a, b in zip(v, vstar))
    return objective(rho, keyframes, s.U, cfg.r) + dot_fields(lam, d) + 0.5 * cfg.K * dot_fields(d, d)


def run(spec, rho0, keyframes, cfg, metric=None, v0=None, dtype=torch.float64):
    """``SPEC.md:390-395`` run(rho0, keyframes, cfg) -> ControlResult.

    Raises MaxIterations (``.result`` = best-so-far ControlResult) when
    max_outer iterations pass without the stop test; inner failures propagate
    annotated with the outer iteration."""
    if dtype == torch.float32 and cfg.projection_tol < 1e-5:
        raise ValueError(f"ADMM in float32 needs projection_tol >= 1e-5 (got {cfg.projection_tol:g}): the AO "
                         "step's absolute projection tolerance is below the fp32 floor; run in float64")
    _dev.require_device()
    if not isinstance(keyframes, KeyframeSet):
        raise SmokeCtrlError("keyframes must be a KeyframeSet")
    n = keyframes.n_steps
    metric = metric or GaussianMetric(spec)
    r0 = _dev.as_dev(rho0, dtype)
    if tuple(r0.shape) != tuple(spec.res):
        raise ValueError(f"rho0 must have shape {spec.res}")
    faces = lambda: tuple(torch.zeros((n,) + spec.face_shape(k), dtype=dtype, device="cuda")
                          for k in range(spec.dim))
    v0 = tuple(_dev.as_dev(c, dtype) for c in v0) if v0 is not None else tuple(
        torch.zeros(spec.face_shape(k), dtype=dtype, device="cuda") for k in range(spec.dim))
    v = faces()
    for k in range(spec.dim):
        v[k][0] = v0[k]
    lam = faces()
    s = SpacetimeState.zeros(spec, n, dtype)
    rho_last = r0.unsqueeze(0).expand((n + 1,) + tuple(r0.shape)).contiguous()
    eps_admm = cfg.eps_admm if cfg.eps_admm is not None else inf_norm(r0) / 100.0
    aocfg = AoConfig(K=cfg.K, dt=cfg.dt, iters=cfg.ao_iters, safeguard=cfg.ao_safeguard,
                     projection_tol=cfg.projection_tol)
    ncfg = StfasConfig(dt=cfg.dt, K=cfg.K, r=cfg.r, n_levels=cfg.n_levels)
    hier = StfasHierarchy(spec, ncfg, n, dtype)
    logs = []
    vlog = []
    best = None
    prev_aug = None
    suspended = bool(cfg.fallback)   # fallback: lambda frozen until the augmented objective stalls
    t_start = time.perf_counter()
    try:
        for it in range(1, cfg.max_outer + 1):
            try:
                guiding = tuple(_axpby(vc.clone(), lc, 1.0 / cfg.K, 1.0) for vc, lc in zip(v, lam))
                ao = solve_ao(spec, guiding, r0, keyframes, metric, aocfg)
                vstar = tuple(ao.vstar)
                ao_obj = _objective_dev(spec, vstar, guiding, keyframes, metric, aocfg, r0)
                guide = tuple(_axpby(vc.clone(), lc, -1.0 / cfg.K, 1.0) for vc, lc in zip(vstar, lam))
                hier.set_guide(v0, guide)
                t_solve = time.perf_counter()
                if cfg.lm:
                    hist = _solve_lm(spec, ncfg, hier, v0, guide, s, cfg.eps_stfas, cfg.relative_stfas,
                                     cfg.nso_cycle_budget)
                else:
                    hist = hier.solve(s, eps=cfg.eps_stfas, relative=cfg.relative_stfas,
                                      cycle_budget=cfg.nso_cycle_budget)
            except SmokeCtrlError as e:
                e.args = (f"outer iteration {it}: {e.args[0] if e.args else ''}",) + e.args[1:]
                e.outer_iter = it
                raise
            per = (time.perf_counter() - t_solve) * 1e3 / max(1, len(hist) - 1)
            vlog.extend((it, c, ri, r2, per if c else 0.0) for c, ri, r2 in hist)
            for k in range(spec.dim):
                v[k][1:] = s.V[k][:n - 1]
            rho, _ = _rollout_dev(spec, vstar, r0, aocfg)
            diff = inf_norm(_axpby(rho_last.clone(), rho, 1.0, -1.0))
            logs.append({"outer_iter": it, "ao_obj": ao_obj, "nso_resid": hist[-1][1], "visual_diff": diff,
                         "wall_s": time.perf_counter() - t_start})
            if diff < eps_admm:
                return ControlResult(rho=rho, v=tuple(c.clone() for c in v), u=tuple(s.U), vstar=vstar,
                                     lam=tuple(c.clone() for c in lam), state=s, logs=logs, converged=True,
                                     vcycle_log=vlog)
            # best so far: the smallest visual difference; its
            # fields are copied (the live state keeps iterating)
            if best is None or diff < best.logs[-1]["visual_diff"]:
                sb = s.copy()
                best = ControlResult(rho=rho, v=tuple(c.clone() for c in v), u=tuple(sb.U), vstar=vstar,
                                     lam=tuple(c.clone() for c in lam), state=sb, logs=list(logs),
                                     vcycle_log=list(vlog))
            rho_last = rho
            if suspended:
                # the multiplier update is suspended once: from
                # the first iteration while the augmented objective still drops
                # by more than fallback_tol; the first iteration that does not
                # ends the suspension for good
                aug = _augmented(spec, cfg, rho, keyframes, s, v, vstar, lam)
                dropping = prev_aug is not None and aug < prev_aug * (1.0 - cfg.fallback_tol)
                first = prev_aug is None
                prev_aug = aug
                if first or dropping:
                    continue
                suspended = False
            for lc, vc, sc in zip(lam, v, vstar):
                d = _axpby(vc.clone(), sc, -1.0, 1.0)
                _axpby(lc, d, cfg.K * cfg.beta, 1.0)
        b_it, b_diff = best.logs[-1]["outer_iter"], best.logs[-1]["visual_diff"]
        best.best_outer_iter = b_it
        best.logs, best.vcycle_log = logs, vlog     # the full history rides along
        raise MaxIterations(f"ADMM did not reach eps_ADMM={eps_admm:g} in {cfg.max_outer} outer iterations "
                            f"(best visual difference {b_diff:.3e} at outer iteration {b_it})", result=best)
    finally:
        hier.close()
