"""Seeded synthetic workloads of BASELINE.json (configs 1-5).

The paper's keyframe assets are not available; these seeded
stand-ins keep the configs' shapes, sizes and value distributions.  The STFAS
input v* is the throughput-mode guide of SURVEY.md §8d: a band-limited random
face field (recipe of pkg/tests/oracles.py:46-66) projected solenoidal on the
GPU and scaled so that dt*|v*|_inf/h = 1.  Generation runs on the device with
the library's own projection (no oracle involvement).
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from .fields import GridSpec, project_arrays

SEED_BASE = 160801102


@dataclass(frozen=True)
class Workload:
    index: int
    dim: int
    n: int
    N: int
    dtype: torch.dtype
    levels: int
    K: float
    r: float
    name: str

    @property
    def spec(self):
        return GridSpec(self.dim, (self.n,) * self.dim, 1.0 / self.n, "neumann")

    @property
    def dt(self):
        return 1.0 / self.N

    @property
    def cell_timesteps(self):
        return self.n ** self.dim * self.N


CONFIGS = {
    1: Workload(1, 2, 32, 16, torch.float64, 2, 1e3, 1e-3, "2D 32^2 x 16 fp64, 2-level"),
    2: Workload(2, 2, 128, 40, torch.float64, 3, 1e3, 1e3, "2D 128^2 x 40 fp64, 3-level"),
    3: Workload(3, 2, 256, 60, torch.float64, 4, 1e3, 1e3, "2D 256^2 x 60 fp64, 4-level"),
    4: Workload(4, 3, 64, 60, torch.float32, 3, 1e3, 1e3, "3D 64^3 x 60 fp32, 3-level"),
    5: Workload(5, 3, 128, 80, torch.float32, 4, 1e3, 1e3, "3D 128^3 x 80 fp32, 4-level"),
}


def config(index, dtype=None):
    w = CONFIGS[int(index)]
    if dtype is not None:
        w = Workload(w.index, w.dim, w.n, w.N, dtype, w.levels, w.K, w.r, w.name.replace(
            "fp32" if w.dtype == torch.float32 else "fp64", "fp64" if dtype == torch.float64 else "fp32"))
    return w


def smooth_faces(spec, gen, modes=2, device="cuda"):
    """Band-limited random face field, max-normalised to 1 (fp64)."""
    comps = []
    for k in range(spec.dim):
        shape = spec.face_shape(k)
        c = torch.zeros(shape, dtype=torch.float64, device=device)
        axes = [torch.arange(s, dtype=torch.float64, device=device) / spec.res[i] for i, s in enumerate(shape)]
        for _ in range(modes):
            kv = gen.integers(1, 4, size=spec.dim)
            ph = gen.uniform(0, 2 * np.pi, size=spec.dim)
            amp = gen.standard_normal()
            wave = None
            for i in range(spec.dim):
                f = torch.sin(2 * math.pi * float(kv[i]) * axes[i] + float(ph[i]))
                sh = [1] * spec.dim
                sh[i] = -1
                f = f.reshape(sh)
                wave = f if wave is None else wave * f
            c += amp * wave
        comps.append(c)
    m = max(float(c.abs().max()) for c in comps)
    comps = [c / max(m, 1e-30) for c in comps]
    if not spec.periodic:
        for k, c in enumerate(comps):
            idx = [slice(None)] * spec.dim
            idx[k] = 0
            c[tuple(idx)] = 0
            idx[k] = -1
            c[tuple(idx)] = 0
    return tuple(comps)


def guide_velocity(w, seed=None, frames=None):
    """v*_0..v*_{N-1} (device, w.dtype): solenoidal, dt*|v*|/h = 1."""
    gen = np.random.default_rng(SEED_BASE + w.index if seed is None else seed)
    spec = w.spec
    N = w.N if frames is None else frames
    scale = spec.h / w.dt
    out = [torch.empty((N,) + spec.face_shape(k), dtype=w.dtype, device="cuda") for k in range(spec.dim)]
    for i in range(N):
        comps = project_arrays(spec, smooth_faces(spec, gen), 1e-9)
        m = max(float(c.abs().max()) for c in comps)
        for k in range(spec.dim):
            out[k][i].copy_(comps[k] * (scale / max(m, 1e-30)))
    return tuple(out)


def initial_velocity(w):
    return tuple(torch.zeros(w.spec.face_shape(k), dtype=w.dtype, device="cuda") for k in range(w.dim))


def _cell_centres(spec, device="cuda"):
    ax = [(torch.arange(n, dtype=torch.float64, device=device) + 0.5) * spec.h for n in spec.res]
    return torch.meshgrid(*ax, indexing="ij")


def gaussian(spec, centre, sigma):
    x = _cell_centres(spec)
    r2 = sum((xi - ci) ** 2 for xi, ci in zip(x, centre))
    return torch.exp(-r2 / (2 * sigma * sigma))


def initial_density(w):
    """BASELINE.json initial densities (seeded where the config says so)."""
    gen = np.random.default_rng(SEED_BASE + w.index)
    s = w.spec
    if w.index == 1:
        return gaussian(s, (0.5, 0.25), 0.08)
    if w.index == 2:
        return gaussian(s, (0.5, 0.2), 0.06)
    if w.index == 4:
        return gaussian(s, (0.5, 0.2, 0.5), 0.08)
    n_g = 4
    lo, hi = (0.03, 0.08) if w.dim == 2 else (0.04, 0.1)
    cen = gen.uniform(0.2, 0.8, size=(n_g, w.dim))
    sig = gen.uniform(lo, hi, size=n_g)
    return sum(gaussian(s, tuple(c), float(sg)) for c, sg in zip(cen, sig))
