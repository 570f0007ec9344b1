"""ADMM outer loop restated in numpy (TEST INFRASTRUCTURE ONLY — never on the
product path; only tests/ may import it).

The reference specifies but does not ship this module: it follows
``SPEC.md:376-426`` (admm_driver) and Alg. 3 (``PAPER.md:339-368``), composing
the pinned oracle AO (``oracle/sim.py``, ao.py:159-254) and STFAS
(``oracle/stfas.py``).  Parity unpinned beyond those components (no
reference golden vectors exist for the loop itself).  Frozen choices (DESIGN
§10): v_0 pinned and v_i = V[i-1] for i >= 1; the AO guide is v + lambda/K
(PAPER.md:160); the NSO guide is v* - lambda/K (the lambda^T (v - v*) term of
Eq. 11 completed into the K/2 square); rho for the stop test is the rollout
under the AO's final v* (SPEC.md:393 design decision); lambda += K beta (v - v*)
only when the stop test fails (Alg. 3 order).
"""

import numpy as np

from . import sim, stfas


def run(g, rho0, targets, n, dt, K=1e3, r=1e3, beta=1.0, ao_iters=2, eps_stfas=1e-5,
        eps_admm=None, max_outer=60, ao_safeguard=False, nso_cycle_budget=50, n_levels=None,
        tol=1e-5, cap=128):
    """Returns dict(v, vstar, lam, rho, state, logs, converged)."""
    v0 = tuple(np.zeros(g.face_shape(k)) for k in range(g.dim))
    v = tuple(np.zeros((n,) + g.face_shape(k)) for k in range(g.dim))
    lam = tuple(np.zeros_like(c) for c in v)
    st = stfas.zero_state(g, n)
    rho_last = np.broadcast_to(rho0, (n + 1,) + g.res).copy()
    if eps_admm is None:
        eps_admm = float(np.max(np.abs(rho0))) / 100.0
    metric = sim.GaussianMetric(g)
    logs = []
    out = None
    for it in range(1, max_outer + 1):
        guiding = tuple(a + b / K for a, b in zip(v, lam))
        vstar, _, _, _ = sim.solve_ao(g, guiding, rho0, targets, metric, K, dt, ao_iters,
                                      ao_safeguard, tol=tol, cap=cap)
        ao_obj = sim.ao_objective(g, vstar, guiding, rho0, targets, metric, K, dt, tol, cap)
        guide = tuple(a - b / K for a, b in zip(vstar, lam))
        pb = stfas.Problem(g, dt, K, r, v0, guide)
        res = stfas.solve_nso(pb, st, eps=eps_stfas, cycle_budget=nso_cycle_budget, n_levels=n_levels)
        st = res.state
        v = tuple(np.concatenate([v0c[None], Vc[:n - 1]], axis=0) for v0c, Vc in zip(v0, st.V))
        rho, _ = sim.rollout(g, vstar, rho0, dt, tol, cap)
        diff = float(np.max(np.abs(rho_last - rho)))
        logs.append({"outer_iter": it, "ao_obj": ao_obj, "nso_resid": res.history[-1][1],
                     "visual_diff": diff})
        out = dict(v=v, vstar=vstar, lam=lam, rho=rho, state=st, logs=logs, converged=False)
        if diff < eps_admm:
            out["converged"] = True
            return out
        rho_last = rho
        lam = tuple(l + K * beta * (a - b) for l, a, b in zip(lam, v, vstar))
        out["lam"] = lam
    return out


def objective(rho, targets, U, r):
    """``SPEC.md:399-407``: 0.5 sum_i |rho_i - rho*_i|^2 + (r/2) sum_i |u_i|^2 (unweighted)."""
    mis = sum(float(np.vdot(rho[i] - t, rho[i] - t)) for i, t in targets.items())
    force = sum(float(np.vdot(u, u)) for u in U)
    return 0.5 * mis + 0.5 * r * force
