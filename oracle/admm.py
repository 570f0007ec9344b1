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
        tol=1e-5, cap=128, fallback=False, fallback_tol=1e-3, nso="numpy"):
    """Returns dict(v, vstar, lam, rho, state, logs, converged, best).

    nso="c" runs the NSO step on the C restatement (oracle/cstfas.c, same
    algorithm) so the loop finishes at the BASELINE configs' sizes.  With
    fallback the multiplier update is suspended from the first iteration
    while the augmented objective (Eq. 11) drops by more than fallback_tol;
    the first iteration that does not ends the suspension.  ``best`` is the
    iteration with the smallest visual difference."""
    v0 = tuple(np.zeros(g.face_shape(k)) for k in range(g.dim))
    v = tuple(np.zeros((n,) + g.face_shape(k)) for k in range(g.dim))
    lam = tuple(np.zeros_like(c) for c in v)
    st = stfas.zero_state(g, n)
    rho_last = np.broadcast_to(rho0, (n + 1,) + g.res).copy()
    if eps_admm is None:
        eps_admm = float(np.max(np.abs(rho0))) / 100.0
    metric = sim.GaussianMetric(g)
    logs = []
    out = best = None
    suspended, prev_aug = fallback, None
    for it in range(1, max_outer + 1):
        guiding = tuple(a + b / K for a, b in zip(v, lam))
        vstar, _, _, _ = sim.solve_ao(g, guiding, rho0, targets, metric, K, dt, ao_iters,
                                      ao_safeguard, tol=tol, cap=cap)
        ao_obj = sim.ao_objective(g, vstar, guiding, rho0, targets, metric, K, dt, tol, cap)
        guide = tuple(a - b / K for a, b in zip(vstar, lam))
        pb = stfas.Problem(g, dt, K, r, v0, guide)
        if nso == "c":
            from . import cstfas
            st, hist, _ = cstfas.Hierarchy(pb, n_levels or 99).solve(st, eps=eps_stfas,
                                                                     cycle_budget=nso_cycle_budget)
            nso_resid = hist[-1][1]
        else:
            res = stfas.solve_nso(pb, st, eps=eps_stfas, cycle_budget=nso_cycle_budget, n_levels=n_levels)
            st, nso_resid = res.state, res.history[-1][1]
        v = tuple(np.concatenate([v0c[None], Vc[:n - 1]], axis=0) for v0c, Vc in zip(v0, st.V))
        rho, _ = sim.rollout(g, vstar, rho0, dt, tol, cap)
        diff = float(np.max(np.abs(rho_last - rho)))
        logs.append({"outer_iter": it, "ao_obj": ao_obj, "nso_resid": nso_resid,
                     "visual_diff": diff})
        out = dict(v=v, vstar=vstar, lam=lam, rho=rho, state=st, logs=list(logs), converged=False)
        if diff < eps_admm:
            out["converged"] = True
            out["best"] = out
            return out
        if best is None or diff < best["logs"][-1]["visual_diff"]:
            best = out
        rho_last = rho
        if suspended:
            d = tuple(a - b for a, b in zip(v, vstar))
            aug = objective(rho, targets, st.U, r) + sum(float(np.vdot(l, x)) for l, x in zip(lam, d)) \
                + 0.5 * K * sum(float(np.vdot(x, x)) for x in d)
            dropping = prev_aug is not None and aug < prev_aug * (1.0 - fallback_tol)
            first = prev_aug is None
            prev_aug = aug
            if first or dropping:
                continue
            suspended = False
        lam = tuple(l + K * beta * (a - b) for l, a, b in zip(lam, v, vstar))
    out["best"] = best
    return out


def objective(rho, targets, U, r):
    """``SPEC.md:399-407``: 0.5 sum_i |rho_i - rho*_i|^2 + (r/2) sum_i |u_i|^2 (unweighted)."""
    mis = sum(float(np.vdot(rho[i] - t, rho[i] - t)) for i, t in targets.items())
    force = sum(float(np.vdot(u, u)) for u in U)
    return 0.5 * mis + 0.5 * r * force
