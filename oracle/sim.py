"""Forward step and AO sweep restated in numpy (TEST INFRASTRUCTURE ONLY).

``step`` follows ``pkg/src/smokectrl/simulator.py:56-110``; ``ao_sweep`` /
``rollout`` / ``GaussianMetric`` follow ``pkg/src/smokectrl/ao.py:48-213``.
"""

import numpy as np

from . import ops


class PicardStall(Exception):
    def __init__(self, residual, state):
        super().__init__("Picard update stalled")
        self.residual = residual
        self.state = state


def picard_velocity(g, v, u, dt, iters=3, sim_tol=1e-6):
    """``simulator.py:56-70``: w <- Q(v + dt (u - S(w, w)))."""
    w = v
    resid = np.inf
    used = 0
    for _ in range(iters):
        adv = ops.self_advection(g, w)
        tgt = tuple(a + dt * (b - c) for a, b, c in zip(v, u, adv))
        wn = ops.project(g, tgt, sim_tol)
        resid = max(ops.inf_norm(a - b) for a, b in zip(wn, w))
        w = wn
        used += 1
        if resid <= sim_tol:
            break
    return w, resid, used


def step(g, v, rho, u, dt, picard_iters=3, sim_tol=1e-6, tol=1e-5, cap=128,
         accept_stall=False):
    """One timestep (``simulator.py:73-110``).  Returns (v', p', rho', info)."""
    v = ops.zero_walls(g, v)
    u = ops.zero_walls(g, u)
    rho_new, k, _ = ops.taylor(g, v, rho, dt, tol, cap)
    w, resid, used = picard_velocity(g, v, u, dt, picard_iters, sim_tol)
    adv = ops.self_advection(g, w)
    src = tuple((a - b) / dt + c - e for a, b, c, e in zip(v, w, u, adv))
    ds = ops.div(g, src)
    ds = ds - ds.mean()
    if ops.inf_norm(ds) > sim_tol:
        p = ops.solve_poisson(g, ds, sim_tol)
    else:
        p = np.zeros(g.res)
    info = {"k": k, "picard_residual": resid, "picard_used": used}
    if resid > sim_tol and not accept_stall:
        raise PicardStall(resid, (w, p, rho_new, info))
    return w, p, rho_new, info


# ---------------------------------------------------------------------------
# AO (ao.py)
# ---------------------------------------------------------------------------


def gaussian_kernel(sigma):
    """``ao.py:48-52``."""
    r = max(1, int(np.ceil(3.0 * sigma)))
    o = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (o / sigma) ** 2)
    return w / w.sum()


def _fold(i, n, periodic):
    """``ao.py:55-60``: wrap, or mirror about the outer cell faces."""
    if periodic:
        return i % n
    m = np.mod(i, 2 * n)
    return np.where(m >= n, 2 * n - 1 - m, m)


def axis_matrix(n, sigma, periodic):
    """Dense per-axis filter matrix (``ao.py:63-71``)."""
    w = gaussian_kernel(sigma)
    r = (len(w) - 1) // 2
    m = np.zeros((n, n))
    rows = np.arange(n)
    for o in range(-r, r + 1):
        np.add.at(m, (rows, _fold(rows + o, n, periodic)), w[o + r])
    return m


class GaussianMetric:
    """C = sum_j w_j G_j^T G_j, sigma_j = sigma0 2^j (``ao.py:74-120``)."""

    def __init__(self, g, levels=None, sigma0=1.0, weights=None):
        if levels is None:
            levels = max(1, int(np.log2(min(g.res))) - 1)
        self.g = g
        self.levels = levels
        self.weights = tuple(weights) if weights is not None else (1.0,) * levels
        self.mats = [tuple(axis_matrix(g.res[k], sigma0 * 2.0 ** j, g.periodic)
                           for k in range(g.dim)) for j in range(levels)]

    @staticmethod
    def _filter(mats, x, transpose):
        for k, m in enumerate(mats):
            mm = m.T if transpose else m
            x = np.moveaxis(np.tensordot(mm, x, axes=(1, k)), 0, k)
        return x

    def apply(self, x):
        out = np.zeros_like(x)
        for w, mats in zip(self.weights, self.mats):
            out += w * self._filter(mats, self._filter(mats, x, False), True)
        return out

    def quad(self, x):
        val = 0.0
        for w, mats in zip(self.weights, self.mats):
            y = self._filter(mats, x, False)
            val += w * float(np.vdot(y, y))
        return val


def rollout(g, vstar, rho0, dt, tol=1e-5, cap=128):
    """``ao.py:159-170``."""
    n = vstar[0].shape[0]
    rho = np.empty((n + 1,) + g.res)
    rho[0] = rho0
    ks = []
    for i in range(n):
        out, k, _ = ops.taylor(g, tuple(c[i] for c in vstar), rho[i], dt, tol, cap)
        rho[i + 1] = out
        ks.append(k)
    return rho, ks


def ao_sweep(g, vstar, v_guiding, rho0, targets, metric, K, dt,
             projection_tol=1e-9, tol=1e-5, cap=128):
    """One forward/backward fixed-point sweep (``ao.py:186-213``).

    ``targets`` maps timestep -> keyframe density.  Returns (vstar, mu, rho, ks).
    Note the backward pass uses the already-updated v*_i (``ao.py:195``)."""
    n = vstar[0].shape[0]
    rho, ks = rollout(g, vstar, rho0, dt, tol, cap)
    vs = tuple(c.copy() for c in vstar)
    mu = np.zeros((n,) + g.res)
    mu_next = np.zeros(g.res)
    for i in range(n, 0, -1):
        if i < n:
            adj, _, _ = ops.taylor(g, tuple(c[i] for c in vs), mu_next, dt, tol,
                                   cap, k_fixed=ks[i], transpose=True)
        else:
            adj = np.zeros(g.res)
        if i in targets:
            adj = adj - metric.apply(rho[i] - targets[i])
        mu[i - 1] = adj
        mu_next = adj
        force = ops.advect_v_T(g, tuple(c[i - 1] for c in vs), rho[i - 1],
                               mu[i - 1], dt, ks[i - 1])
        raw = tuple(gd[i - 1] + f / K for gd, f in zip(v_guiding, force))
        proj = ops.project(g, raw, projection_tol)
        for k in range(g.dim):
            vs[k][i - 1] = proj[k]
    return vs, mu, rho, ks


def ao_objective(g, vstar, v_guiding, rho0, targets, metric, K, dt, tol=1e-5, cap=128):
    """``ao.py:173-183``: 0.5 sum |rho_i - rho*_i|_C^2 + (K/2) |v - v*|^2."""
    rho, _ = rollout(g, vstar, rho0, dt, tol, cap)
    mismatch = sum(metric.quad(rho[i] - t) for i, t in targets.items())
    vterm = sum(float(np.vdot(a - b, a - b)) for a, b in zip(v_guiding, vstar))
    return 0.5 * mismatch + 0.5 * K * vterm


def solve_ao(g, v_guiding, rho0, targets, metric, K, dt, iters=2, safeguard=False,
             projection_tol=1e-9, tol=1e-5, cap=128):
    """``ao.py:216-254``: fixed sweeps; with the safeguard each sweep's v* is
    blended with the previous one, halving alpha (> 1/64) until the objective
    does not increase.  Returns (vstar, mu, rho, ks)."""
    n = v_guiding[0].shape[0]
    vs = tuple(c.copy() for c in v_guiding)
    mu = np.zeros((n,) + g.res)
    rho = np.broadcast_to(rho0, (n + 1,) + g.res).copy()
    ks = []
    obj = ao_objective(g, vs, v_guiding, rho0, targets, metric, K, dt, tol, cap) if safeguard else None
    for _ in range(iters):
        nv, nmu, nrho, nks = ao_sweep(g, vs, v_guiding, rho0, targets, metric, K, dt,
                                      projection_tol, tol, cap)
        if not safeguard:
            vs, mu, rho, ks = nv, nmu, nrho, nks
            continue
        alpha, accepted = 1.0, None
        while alpha > 1.0 / 64.0:
            blend = tuple((1 - alpha) * a + alpha * b for a, b in zip(vs, nv))
            o = ao_objective(g, blend, v_guiding, rho0, targets, metric, K, dt, tol, cap)
            if o <= obj * (1 + 1e-12) + 1e-300:
                accepted = (blend, o)
                break
            alpha *= 0.5
        if accepted is None:
            break
        vs, obj = accepted
        mu = nmu
        rho, ks = rollout(g, vs, rho0, dt, tol, cap)
    return vs, mu, rho, ks
