"""LBFGS adjoint baseline on B200 (SPEC.md:428-472 lbfgs_baseline; PAPER §5).

The comparison optimizer of the paper: the constraints are eliminated by
forward simulation (the reference's ``simulator.step``, simulator.py:56-110:
Taylor density advection by the pre-step velocity, an implicit
self-advection solved by Picard sweeps w <- Q(v + dt (u - S(w, w))) with the
projection Q), the objective of Eq. 5

    J(u) = 1/2 sum_i c_i |rho_i - rho*_i|^2 + r/2 sum_i |u_i|^2

(unweighted sums, like ``admm.objective``) is differentiated with the
discrete adjoint of exactly that forward map, and minimised over the per-face
forces u_0..u_{N-1} by limited-memory BFGS (history 8, two-loop recursion)
with a backtracking Armijo line search (c = 1e-4).

Adjoint of one step (rho' = A(rho, v), v' = w^K), given the adjoints
lam_rho', lam_v' of its outputs:

    lam_rho = A(., v)^T lam_rho'                 (advect_scalar_rho_T, forward's k)
    lam_v   = (dA/dv)^T lam_rho'                  (advect_scalar_v_T)
    g = lam_v';  for k = K-1 .. 0:  mu = Q g;  lam_v += mu;  lam_u += dt mu;
                                    g = -dt J_Adv(w^k)^T mu   (self_adv_jacobian_T_apply)
    lam_v += g                                    (w^0 = v)

Q is the discrete Helmholtz projector, symmetric because grad = -div^T
exactly; the Picard sweeps actually executed by the forward
(its early exit included) are replayed.  Wall faces are not controls (the
step zero-masks v and u, simulator.py:82-83), so their gradient is zero.
Every operator is a libsmk kernel (advection.py / fields.py drop-ins);
vector algebra through ``smk_axpby`` / ``smk_dot``.
"""

import time
from dataclasses import dataclass, field

import torch

from . import _dev
from .advection import (DEFAULT_TERM_CAP, DEFAULT_TRUNCATION_TOL, advect_scalar, advect_scalar_rho_T,
                        advect_scalar_v_T, self_adv_jacobian_T_apply, self_advection)
from .ao import KeyframeSet, _axpby
from .errors import LineSearchFailure, MaxIterations, SmokeCtrlError
from .fields import dot_fields, inf_norm, project_arrays, zero_boundary_faces


@dataclass
class LbfgsConfig:
    """SPEC.md:457-460 (history 8, Armijo c = 1e-4) and the ADMM stop test
    ('same stopping criteria for both')."""

    dt: float
    r: float = 1e3
    history: int = 8
    armijo_c: float = 1e-4
    max_iter: int = 100
    max_backtracks: int = 30
    eps_visual: float = None        # None -> rho_max / 100 of the initial frame (as admm)
    grad_tol: float = 0.0           # optional: stop when |g|_inf <= grad_tol
    picard_iters: int = 3
    sim_tol: float = 1e-6
    truncation_tol: float = DEFAULT_TRUNCATION_TOL
    truncation_cap: int = DEFAULT_TERM_CAP


@dataclass
class LbfgsResult:
    rho: torch.Tensor               # (N+1, *res)
    u: tuple                        # (N, face) forces
    objective: float
    iterations: int
    converged: bool
    logs: list = field(default_factory=list)    # (iter, objective, |g|_inf, step, visual_diff, wall_s)


class AdjointWorkspace:
    """The stored forward trajectory: per step the masked
    pre-step velocity, the density, the Taylor order and the Picard iterates
    fed to S."""

    def __init__(self):
        self.v = []
        self.rho = []
        self.k = []
        self.w = []


def _faces_like(spec, dt):
    return tuple(torch.zeros(spec.face_shape(k), dtype=dt, device="cuda") for k in range(spec.dim))


def _vaxpby(y, x, a, b):
    for yy, xx in zip(y, x):
        _axpby(yy, xx, a, b)
    return y


def simulate(spec, u, rho0, cfg, ws=None):
    """Forward rollout under forces u ((N, face) stacks) from rest; returns
    rho (N+1, *res) and fills the workspace."""
    dt = rho0.dtype
    n = u[0].shape[0]
    rho = torch.empty((n + 1,) + tuple(spec.res), dtype=dt, device="cuda")
    rho[0].copy_(rho0)
    v = _faces_like(spec, dt)
    for i in range(n):
        vz = zero_boundary_faces(spec, v)
        uz = zero_boundary_faces(spec, tuple(c[i] for c in u))
        rn, rep = advect_scalar(spec, vz, rho[i], cfg.dt, cfg.truncation_tol, cfg.truncation_cap)
        rho[i + 1].copy_(rn)
        w, iters = vz, []
        for _ in range(cfg.picard_iters):
            adv = self_advection(spec, w)
            target = tuple(_axpby(_axpby(a.clone(), uu, cfg.dt, -cfg.dt), vv, 1.0, 1.0)
                           for a, uu, vv in zip(adv, uz, vz))     # v + dt (u - S(w, w))
            w_new = project_arrays(spec, target, cfg.sim_tol)
            iters.append(w)
            resid = inf_norm(tuple(_axpby(a.clone(), b, -1.0, 1.0) for a, b in zip(w_new, w)))
            w = w_new
            if resid <= cfg.sim_tol:
                break
        if ws is not None:
            ws.v.append(vz)
            ws.rho.append(rho[i])
            ws.k.append(rep.k_used)
            ws.w.append(iters)
        v = w
    return rho


def objective(rho, keyframes, u, r):
    """Eq. 5 (SPEC.md:399-407 form, as admm.objective)."""
    from .admm import objective as obj
    return obj(rho, keyframes, u, r)


def objective_and_gradient(spec, u, rho0, keyframes, cfg):
    """(J(u), dJ/du, rho trajectory)."""
    _dev.require_device()
    dt = rho0.dtype
    n = u[0].shape[0]
    ws = AdjointWorkspace()
    rho = simulate(spec, u, rho0, cfg, ws)
    J = objective(rho, keyframes, u, cfg.r)
    lam_rho = torch.zeros(tuple(spec.res), dtype=dt, device="cuda")
    lam_v = _faces_like(spec, dt)
    grad = tuple(torch.zeros_like(c) for c in u)
    targets = {i: _dev.as_dev(t, dt) for i, t in keyframes.targets.items()}
    if n in targets:
        _axpby(lam_rho, _axpby(rho[n].clone(), targets[n], -1.0, 1.0), 1.0, 1.0)
    for i in range(n - 1, -1, -1):
        vz, k = ws.v[i], ws.k[i]
        g_rho, _ = advect_scalar_rho_T(spec, vz, lam_rho, cfg.dt, k_fixed=k)
        lv, _ = advect_scalar_v_T(spec, vz, ws.rho[i], lam_rho, cfg.dt, k_fixed=k)
        lv = tuple(c.clone() for c in lv)
        lu = _faces_like(spec, dt)
        g = lam_v
        for w in reversed(ws.w[i]):
            mu = project_arrays(spec, zero_boundary_faces(spec, g), cfg.sim_tol)
            _vaxpby(lv, mu, 1.0, 1.0)
            _vaxpby(lu, mu, cfg.dt, 1.0)
            g = tuple(_axpby(c, c, 0.0, -cfg.dt) for c in self_adv_jacobian_T_apply(spec, w, mu))
        _vaxpby(lv, g, 1.0, 1.0)
        lu = zero_boundary_faces(spec, lu)
        for gc, lc, uc in zip(grad, lu, u):
            gc[i].copy_(lc)
            _axpby(gc[i], uc[i], cfg.r, 1.0)          # + r u_i (the regulariser)
        lam_v = zero_boundary_faces(spec, lv)
        lam_rho = g_rho.clone() if isinstance(g_rho, torch.Tensor) else _dev.as_dev(g_rho, dt)
        if i in targets and i >= 1:
            _axpby(lam_rho, _axpby(rho[i].clone(), targets[i], -1.0, 1.0), 1.0, 1.0)
    # wall faces are not controls (all N frames at once)
    return J, zero_boundary_faces(spec, grad), rho


def _two_loop(g, S, Y):
    """H g by the L-BFGS two-loop recursion (fixed-order device dots)."""
    q = tuple(c.clone() for c in g)
    alphas = []
    for s, y in reversed(list(zip(S, Y))):
        rho_ = 1.0 / dot_fields(y, s)
        a = rho_ * dot_fields(s, q)
        alphas.append((a, rho_, s, y))
        _vaxpby(q, y, -a, 1.0)
    if S:
        s, y = S[-1], Y[-1]
        _vaxpby(q, q, 0.0, dot_fields(s, y) / dot_fields(y, y))
    for a, rho_, s, y in reversed(alphas):
        b = rho_ * dot_fields(y, q)
        _vaxpby(q, s, a - b, 1.0)
    return q


def lbfgs(fun, x0, cfg, stop=None, t0=None):
    """Generic L-BFGS on tuples of device tensors (two-loop
    recursion, history cfg.history, backtracking Armijo c = cfg.armijo_c).

    fun(x) -> (f, g, aux); stop(it, x, f, g, aux, aux_prev, logs) -> bool.
    Returns (x, f, g, aux, iterations, converged, logs); raises
    LineSearchFailure / MaxIterations with ``.result`` = that tuple for the
    best (last accepted) iterate."""
    t0 = t0 if t0 is not None else time.perf_counter()
    x = tuple(c.clone() for c in x0)
    f, g, aux = fun(x)
    S, Y, logs = [], [], []
    for it in range(1, cfg.max_iter + 1):
        d = tuple(_axpby(c, c, 0.0, -1.0) for c in _two_loop(g, S, Y))   # d = -H g
        gd = dot_fields(g, d)
        if not gd < 0:                                                   # not a descent direction: restart
            S, Y = [], []
            d = tuple(_axpby(c.clone(), c, 0.0, -1.0) for c in g)
            gd = dot_fields(g, d)
        step = 1.0 if S else min(1.0, 1.0 / max(inf_norm(g), 1e-300))
        for _ in range(cfg.max_backtracks):
            xn = tuple(_axpby(xc.clone(), dc, step, 1.0) for xc, dc in zip(x, d))
            fn, gn, auxn = fun(xn)
            if fn <= f + cfg.armijo_c * step * gd:
                break
            step *= 0.5
        else:
            err = LineSearchFailure(f"Armijo backtracking failed at iteration {it} (f = {f:.6e})")
            err.result = (x, f, g, aux, it - 1, False, logs)
            raise err
        s = tuple(_axpby(a.clone(), b, -1.0, 1.0) for a, b in zip(xn, x))
        y = tuple(_axpby(a.clone(), b, -1.0, 1.0) for a, b in zip(gn, g))
        sy = dot_fields(s, y)
        if sy > 1e-12 * (dot_fields(y, y) * dot_fields(s, s)) ** 0.5:   # curvature pair kept only if positive
            S.append(s)
            Y.append(y)
            if len(S) > cfg.history:
                S.pop(0)
                Y.pop(0)
        aux_prev = aux
        x, f, g, aux = xn, fn, gn, auxn
        logs.append({"iter": it, "objective": f, "grad_inf": inf_norm(g), "step": step,
                     "wall_s": time.perf_counter() - t0})
        if stop is not None and stop(it, x, f, g, aux, aux_prev, logs):
            return x, f, g, aux, it, True, logs
    err = MaxIterations(f"LBFGS: {cfg.max_iter} iterations without meeting the stop test")
    err.result = (x, f, g, aux, cfg.max_iter, False, logs)
    raise err


def minimize(spec, rho0, keyframes, r, dt, cfg=None, u0=None, dtype=torch.float64):
    """L-BFGS over u from u0 (zero) until the density
    trajectory moves by less than eps_visual between accepted iterates (the
    ADMM stop test), or |g|_inf <= grad_tol.  LineSearchFailure /
    MaxIterations propagate with ``.result`` = the best LbfgsResult."""
    _dev.require_device()
    if not isinstance(keyframes, KeyframeSet):
        raise SmokeCtrlError("keyframes must be a KeyframeSet")
    cfg = cfg or LbfgsConfig(dt=dt, r=r)
    cfg.dt, cfg.r = dt, r
    n = keyframes.n_steps
    r0 = _dev.as_dev(rho0, dtype)
    u0 = tuple(c.clone() for c in u0) if u0 is not None else \
        tuple(torch.zeros((n,) + spec.face_shape(k), dtype=dtype, device="cuda") for k in range(spec.dim))
    eps = cfg.eps_visual if cfg.eps_visual is not None else inf_norm(r0) / 100.0

    def fun(u):
        return objective_and_gradient(spec, u, r0, keyframes, cfg)

    def stop(it, u, f, g, rho, rho_prev, logs):
        vis = inf_norm(_axpby(rho.clone(), rho_prev, -1.0, 1.0))
        logs[-1]["visual_diff"] = vis
        return vis < eps or (cfg.grad_tol > 0 and logs[-1]["grad_inf"] <= cfg.grad_tol)

    wrap = lambda t: LbfgsResult(t[3], t[0], t[1], t[4], t[5], t[6])
    try:
        return wrap(lbfgs(fun, u0, cfg, stop))
    except (LineSearchFailure, MaxIterations) as e:
        e.result = wrap(e.result)
        raise
