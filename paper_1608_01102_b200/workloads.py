"""Seeded synthetic workloads of BASELINE.json (configs 1-5).

The paper's keyframe assets are not available; these seeded
stand-ins keep the configs' shapes, sizes and value distributions: the
initial densities and keyframes are the ones BASELINE.json's configs describe
(``initial_density``, ``keyframes``; unspecified parameters per SURVEY.md
§8d: threshold 0.5 of the max-normalised sum, then a Gaussian blur of sigma
= 1 cell, clipped at 0 because KeyframeSet rejects negatives, ao.py:40-41).  The STFAS
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


def gaussian(spec, centre, sigma, device="cuda"):
    x = _cell_centres(spec, device)
    r2 = sum((xi - ci) ** 2 for xi, ci in zip(x, centre))
    return torch.exp(-r2 / (2 * sigma * sigma))


def initial_density(w, device="cuda"):
    """BASELINE.json initial densities (seeded where the config says so)."""
    gen = np.random.default_rng(SEED_BASE + w.index)
    s = w.spec
    if w.index == 1:
        return gaussian(s, (0.5, 0.25), 0.08, device)
    if w.index == 2:
        return gaussian(s, (0.5, 0.2), 0.06, device)
    if w.index == 4:
        return gaussian(s, (0.5, 0.2, 0.5), 0.08, device)
    n_g = 4
    lo, hi = (0.03, 0.08) if w.dim == 2 else (0.04, 0.1)
    cen = gen.uniform(0.2, 0.8, size=(n_g, w.dim))
    sig = gen.uniform(lo, hi, size=n_g)
    return sum(gaussian(s, tuple(c), float(sg), device) for c, sg in zip(cen, sig))


def _blur_axis(x, axis, sigma=1.0, truncate=4.0):
    """1-D Gaussian blur (sigma in cells, reflect at the domain walls, taps to
    truncate * sigma: scipy.ndimage.gaussian_filter's defaults)."""
    r = int(truncate * sigma + 0.5)
    t = torch.arange(-r, r + 1, dtype=torch.float64, device=x.device)
    wts = torch.exp(-0.5 * (t / sigma) ** 2)
    wts = wts / wts.sum()
    n = x.shape[axis]
    idx = torch.arange(-r, n + r, device=x.device)
    idx = torch.where(idx < 0, -idx - 1, idx)            # reflect (d c b a | a b c d)
    idx = torch.where(idx >= n, 2 * n - 1 - idx, idx)
    xp = torch.index_select(x, axis, idx)
    out = torch.zeros_like(x)
    for k in range(2 * r + 1):
        out += wts[k] * torch.narrow(xp, axis, k, n)
    return out


def blur(x, sigma=1.0):
    for a in range(x.dim()):
        x = _blur_axis(x, a, sigma)
    return x


def _threshold_smooth(field):
    """Threshold at 0.5 of the max, then blur sigma = 1 cell."""
    m = (field / field.max() >= 0.5).to(torch.float64)
    return blur(m, 1.0).clamp_min(0.0)


def _gauss_sum(spec, gen, count, lo, hi, device):
    cen = gen.uniform(0.2, 0.8, size=(count, spec.dim))
    sig = gen.uniform(lo, hi, size=count)
    return sum(gaussian(spec, tuple(c), float(sg), device) for c, sg in zip(cen, sig))


def keyframes(w, device="cuda"):
    """BASELINE.json keyframes {timestep: density (fp64)}.

    cfg1: disc r = 0.15 at (0.5, 0.7) with a smoothstep edge of +-1 cell at
    t = 16; cfg2: the letter-F mask (three rectangles) blurred by sigma = 1
    cell at t = 40; cfg3: t = 30, 60, each 6 seeded Gaussians (sigma
    U[0.03, 0.08]) thresholded and smoothed; cfg4: t = 60, 8 seeded 3D
    Gaussians (sigma U[0.04, 0.1]); cfg5: t = 20, 40, 60, 80, 8 seeded
    Gaussians each.  The seeded draws continue initial_density's stream
    (its centres and sigmas first, then each keyframe in time order)."""
    s = w.spec
    x = _cell_centres(s, device)
    if w.index == 1:
        d = torch.sqrt((x[0] - 0.5) ** 2 + (x[1] - 0.7) ** 2)
        a, b = 0.15 - s.h, 0.15 + s.h
        t = ((d - a) / (b - a)).clamp(0.0, 1.0)
        return {16: 1.0 - t * t * (3.0 - 2.0 * t)}
    if w.index == 2:
        inside = lambda x0, x1, y0, y1: (x[0] >= x0) & (x[0] <= x1) & (x[1] >= y0) & (x[1] <= y1)
        f = inside(0.35, 0.45, 0.3, 0.8) | inside(0.35, 0.7, 0.7, 0.8) | inside(0.35, 0.6, 0.5, 0.58)
        return {40: blur(f.to(torch.float64), 1.0).clamp_min(0.0)}
    gen = np.random.default_rng(SEED_BASE + w.index)
    lo, hi = (0.03, 0.08) if w.dim == 2 else (0.04, 0.1)
    if w.index != 4:                       # initial_density's draws come first
        gen.uniform(0.2, 0.8, size=(4, w.dim))
        gen.uniform(lo, hi, size=4)
    times = {3: (30, 60), 4: (60,), 5: (20, 40, 60, 80)}[w.index]
    count = {3: 6, 4: 8, 5: 8}[w.index]
    return {t: _threshold_smooth(_gauss_sum(s, gen, count, lo, hi, device)) for t in times}
