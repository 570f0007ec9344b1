"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``smokectrl`` from ``/root/reference/pkg/src`` (read-only) and
writes ``tests/golden/ref_ops.npz``.  The fixtures pin the oracle
restatement (``oracle/ops.py``, ``oracle/sim.py``) to the reference's own
outputs; the GPU box never reads /root/reference — only these committed files.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_ops.npz")


def smooth(spec, rng, scale, modes=2):
    """Band-limited face field (same recipe as pkg/tests/oracles.py:46-66)."""
    from smokectrl.fields import zero_boundary_faces
    comps = []
    for k in range(spec.dim):
        shape = spec.face_shape(k)
        grids = np.meshgrid(*[np.arange(s) / spec.res[i]
                              for i, s in enumerate(shape)], indexing="ij")
        c = np.zeros(shape)
        for _ in range(modes):
            kv = rng.integers(1, 4, size=spec.dim)
            ph = rng.uniform(0, 2 * np.pi, size=spec.dim)
            wave = np.ones(shape)
            for i in range(spec.dim):
                wave = wave * np.sin(2 * np.pi * kv[i] * grids[i] + ph[i])
            c += rng.standard_normal() * wave
        comps.append(c)
    m = max(np.max(np.abs(c)) for c in comps)
    comps = tuple(scale * c / max(m, 1e-30) for c in comps)
    if not spec.periodic:
        comps = zero_boundary_faces(spec, comps)
    return comps


def main():
    sys.path.insert(0, REF)
    from smokectrl import fields as F
    from smokectrl import advection as A
    from smokectrl import simulator as S
    from smokectrl import ao as AO

    out = {}

    def put(prefix, name, val):
        if isinstance(val, tuple):
            for k, c in enumerate(val):
                out[f"{prefix}/{name}{k}"] = np.asarray(c)
        else:
            out[f"{prefix}/{name}"] = np.asarray(val)

    cases = [
        ("n2p", 2, (8, 8), "periodic", 0),
        ("n2n", 2, (8, 8), "neumann", 1),
        ("r2n", 2, (16, 8), "neumann", 2),
        ("n3n", 3, (8, 8, 8), "neumann", 3),
        ("n3p", 3, (8, 4, 8), "periodic", 4),
    ]
    for tag, dim, res, bnd, seed in cases:
        spec = F.GridSpec(dim, res, 1.0 / res[0], bnd)
        rng = np.random.default_rng(1000 + seed)
        v = smooth(spec, rng, 0.3 * spec.h / 0.1)
        w = tuple(rng.standard_normal(spec.face_shape(k)) for k in range(dim))
        w = F.zero_boundary_faces(spec, w)
        u = tuple(rng.standard_normal(spec.face_shape(k)) for k in range(dim))
        u = F.zero_boundary_faces(spec, u)
        rho = rng.standard_normal(res)
        mu = rng.standard_normal(res)
        put(tag, "meta", np.array([dim, *res, 0][:4] if dim == 2 else [dim, *res]))
        put(tag, "h", np.array(spec.h))
        put(tag, "bnd", np.array(bnd))
        put(tag, "v", v)
        put(tag, "w", w)
        put(tag, "u", u)
        put(tag, "rho", rho)
        put(tag, "mu", mu)
        put(tag, "div", F.divergence_arrays(spec, w))
        put(tag, "grad", F.gradient_arrays(spec, rho))
        put(tag, "T", A.transport_scalar(spec, v, rho))
        dt = 0.1
        a, rep = A.advect_scalar(spec, v, rho, dt)
        put(tag, "adv", a)
        put(tag, "adv_k", np.array(rep.k_used))
        b, rep2 = A.advect_scalar_rho_T(spec, v, mu, dt, k_fixed=rep.k_used)
        put(tag, "advT", b)
        c, _ = A.advect_scalar_v_T(spec, v, rho, mu, dt, k_fixed=rep.k_used)
        put(tag, "advvT", c)
        put(tag, "S", A.transport_face(spec, v, w))
        put(tag, "Sself", A.self_advection(spec, v))
        put(tag, "J", A.self_adv_jacobian_apply(spec, v, w))
        put(tag, "JT", A.self_adv_jacobian_T_apply(spec, v, u))
        put(tag, "rc", F.restrict_cell(spec, rho))
        cs = spec.coarsen()
        if cs is not None:
            put(tag, "pc", F.prolong_cell(cs, spec, F.restrict_cell(spec, rho)))
        put(tag, "proj", F.project_arrays(spec, w, 1e-9))
        put(tag, "pois", F.solve_poisson(spec, mu, 1e-9))
        put(tag, "sl", A.semi_lagrangian(F.ScalarField(spec, np.abs(rho)),
                                         F.StaggeredVectorField(spec, v), 0.3).values)
        # simulator step at moderate CFL (accept a stalled Picard)
        st = S.SimState(F.StaggeredVectorField(spec, v), F.ScalarField.zeros(spec),
                        F.ScalarField(spec, np.abs(rho)))
        uu = F.project_arrays(spec, smooth(spec, rng, 0.2), 1e-10)
        put(tag, "su", uu)
        s1 = S.step(st, F.StaggeredVectorField(spec, uu), S.SimConfig(dt=0.1),
                    accept_stall=True)
        put(tag, "step_v", s1.v.comps)
        put(tag, "step_p", s1.p.values)
        put(tag, "step_rho", s1.rho.values)
        # scalar_stencil_v_adjoint (advection.py:105) and the AdvectionOperator
        # methods (advection.py:213-248) on a velocity with nonzero wall faces
        # (the operator masks them at construction)
        put(tag, "svadj", A.scalar_stencil_v_adjoint(spec, rho, mu))
        vr = tuple(0.3 * rng.standard_normal(spec.face_shape(k)) for k in range(dim))
        put(tag, "vraw", vr)
        op = A.AdvectionOperator(F.StaggeredVectorField(spec, vr))
        put(tag, "aop_st", op.apply_stencil(F.ScalarField(spec, rho)).values)
        a2, r2 = op.advect(F.ScalarField(spec, rho), 0.1)
        put(tag, "aop_adv", a2.values)
        put(tag, "aop_k", np.array(r2.k_used))
        b2, _ = op.jacobian_rho_T(F.ScalarField(spec, mu), 0.1, k_fixed=r2.k_used)
        put(tag, "aop_rT", b2.values)
        put(tag, "aop_vT", op.jacobian_v_T(F.ScalarField(spec, rho), F.ScalarField(spec, mu), 0.1,
                                           k_fixed=r2.k_used).comps)

    # AO sweep (2D, both boundaries): one sweep from guiding = v*
    for tag, bnd, seed in [("ao2p", "periodic", 7), ("ao2n", "neumann", 8)]:
        spec = F.GridSpec(2, (8, 8), 0.125, bnd)
        rng = np.random.default_rng(2000 + seed)
        n = 3
        guiding = [F.project_arrays(spec, smooth(spec, rng, 0.2), 1e-11)
                   for _ in range(n)]
        guiding = tuple(np.stack([gd[k] for gd in guiding]) for k in range(2))
        g2 = np.meshgrid(*[(np.arange(m) + 0.5) * spec.h for m in spec.res],
                         indexing="ij")
        rho0 = np.exp(-((g2[0] - 0.4) ** 2 + (g2[1] - 0.5) ** 2) / 0.015)
        target = np.exp(-((g2[0] - 0.6) ** 2 + (g2[1] - 0.5) ** 2) / 0.015)
        kf = AO.KeyframeSet(n, {n: target})
        metric = AO.GaussianMetric(spec)
        cfg = AO.AoConfig(K=10.0, dt=0.5)
        state = AO.AoState(vstar=tuple(c.copy() for c in guiding),
                           mu=np.zeros((n,) + spec.res),
                           rho=np.broadcast_to(rho0, (n + 1,) + spec.res).copy())
        res = AO.ao_sweep(spec, state, guiding, kf, metric, cfg)
        put(tag, "guiding", guiding)
        put(tag, "rho0", rho0)
        put(tag, "target", target)
        put(tag, "vstar", res.vstar)
        put(tag, "mu", res.mu)
        put(tag, "rho", res.rho)
        put(tag, "ks", np.array(res.ks))
        put(tag, "metric_apply", metric.apply(rho0 - target))

    # solve_ao (2D Neumann, plain and safeguarded) + objective, and a 3D
    # periodic metric apply / quad
    for tag, safeguard, iters in [("aos0", False, 2), ("aos1", True, 3)]:
        spec = F.GridSpec(2, (8, 8), 0.125, "neumann")
        rng = np.random.default_rng(3100 + iters)
        n = 4
        guiding = [F.project_arrays(spec, smooth(spec, rng, 0.3), 1e-11)
                   for _ in range(n)]
        guiding = tuple(np.stack([gd[k] for gd in guiding]) for k in range(2))
        g2 = np.meshgrid(*[(np.arange(m) + 0.5) * spec.h for m in spec.res],
                         indexing="ij")
        rho0 = np.exp(-((g2[0] - 0.35) ** 2 + (g2[1] - 0.5) ** 2) / 0.02)
        t2 = np.exp(-((g2[0] - 0.5) ** 2 + (g2[1] - 0.55) ** 2) / 0.02)
        t4 = np.exp(-((g2[0] - 0.65) ** 2 + (g2[1] - 0.5) ** 2) / 0.02)
        kf = AO.KeyframeSet(n, {2: t2, 4: t4})
        metric = AO.GaussianMetric(spec)
        cfg = AO.AoConfig(K=5.0, dt=0.5, iters=iters, safeguard=safeguard)
        res = AO.solve_ao(spec, guiding, rho0, kf, metric, cfg)
        put(tag, "guiding", guiding)
        put(tag, "rho0", rho0)
        put(tag, "t2", t2)
        put(tag, "t4", t4)
        put(tag, "vstar", res.vstar)
        put(tag, "mu", res.mu)
        put(tag, "rho", res.rho)
        put(tag, "ks", np.array(res.ks))
        put(tag, "obj0", np.array(AO.ao_objective(spec, guiding, guiding, kf, metric, cfg, rho0)))
        put(tag, "obj", np.array(AO.ao_objective(spec, res.vstar, guiding, kf, metric, cfg, rho0)))
    spec = F.GridSpec(3, (8, 8, 16), 0.125, "periodic")
    rng = np.random.default_rng(3200)
    x = rng.standard_normal(spec.res)
    metric = AO.GaussianMetric(spec, levels=2, weights=(1.0, 0.5))
    put("met3", "x", x)
    put("met3", "apply", metric.apply(x))
    put("met3", "quad", np.array(metric.quad(x)))

    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
