"""Seeded synthetic STFAS problems for the parity tests (numpy, via the oracle)."""

import numpy as np

from oracle import ops, stfas
from oracle.grid import Grid


def smooth_vector(g, rng, scale, modes=2):
    """Band-limited face field (recipe of pkg/tests/oracles.py:46-66)."""
    comps = []
    for k in range(g.dim):
        shape = g.face_shape(k)
        grids = np.meshgrid(*[np.arange(s) / g.res[i] for i, s in enumerate(shape)], indexing="ij")
        c = np.zeros(shape)
        for _ in range(modes):
            kv = rng.integers(1, 4, size=g.dim)
            ph = rng.uniform(0, 2 * np.pi, size=g.dim)
            w = np.ones(shape)
            for i in range(g.dim):
                w = w * np.sin(2 * np.pi * kv[i] * grids[i] + ph[i])
            c += rng.standard_normal() * w
        comps.append(c)
    m = max(np.max(np.abs(c)) for c in comps)
    return ops.zero_walls(g, tuple(scale * c / max(m, 1e-30) for c in comps))


def make_problem(dim=2, n=16, N=4, boundary="neumann", K=1e3, r=1e3, cfl=1.0, seed=0, dt=None,
                 res=None):
    res = res or (n,) * dim
    g = Grid(dim, res, 1.0 / res[0], boundary)
    dt = dt or 1.0 / N
    rng = np.random.default_rng(seed)
    vs = [ops.project(g, smooth_vector(g, rng, cfl * g.h / dt), 1e-12) for _ in range(N)]
    vstar = tuple(np.stack([v[k] for v in vs]) for k in range(dim))
    v0 = tuple(np.zeros(g.face_shape(k)) for k in range(dim))
    return stfas.Problem(g, dt, K, r, v0, vstar)


def random_state(pb, rng, scale=0.1):
    g, N = pb.g, pb.N
    V = ops.zero_walls(g, tuple(scale * rng.standard_normal((N,) + g.face_shape(k)) for k in range(g.dim)))
    U = ops.zero_walls(g, tuple(scale * rng.standard_normal((N,) + g.face_shape(k)) for k in range(g.dim)))
    return stfas.State(V, scale * rng.standard_normal((N,) + g.res), U, scale * rng.standard_normal((N,) + g.res))


def random_residual(pb, rng, scale=0.1):
    g, N = pb.g, pb.N
    R1 = ops.zero_walls(g, tuple(scale * rng.standard_normal((N,) + g.face_shape(k)) for k in range(g.dim)))
    R3 = ops.zero_walls(g, tuple(scale * rng.standard_normal((N,) + g.face_shape(k)) for k in range(g.dim)))
    return stfas.Residual(R1, scale * rng.standard_normal((N,) + g.res), R3,
                          scale * rng.standard_normal((N,) + g.res))
