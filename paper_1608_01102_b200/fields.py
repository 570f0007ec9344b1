"""MAC field core on B200 — drop-in for ``pkg/src/smokectrl/fields.py``.

Same names, argument meaning and error behaviour as the reference raw
kernels (``fields.py:140-394``).  Inputs may be numpy arrays (results come
back as numpy, host<->device copies included) or CUDA torch tensors (results
stay on the device).  Arrays may carry a leading batch (frame) axis.
"""

from dataclasses import dataclass

import ctypes

import numpy as np
import torch

from . import _dev, _lib
from .errors import NonConvergence

NEUMANN = "neumann"
PERIODIC = "periodic"


@dataclass(frozen=True)
class GridSpec:
    """``fields.py:37-89``."""

    dim: int
    res: tuple
    h: float
    boundary: str = NEUMANN

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise ValueError(f"dim must be 2 or 3, got {self.dim}")
        res = tuple(int(r) for r in self.res)
        object.__setattr__(self, "res", res)
        if len(res) != self.dim:
            raise ValueError("res length must equal dim")
        if any(r < 4 for r in res):
            raise ValueError(f"every res component must be >= 4, got {res}")
        if not self.h > 0:
            raise ValueError("h must be positive")
        if self.boundary not in (NEUMANN, PERIODIC):
            raise ValueError(f"unknown boundary {self.boundary!r}")

    @property
    def periodic(self):
        return self.boundary == PERIODIC

    @property
    def n_cells(self):
        return int(np.prod(self.res))

    def face_shape(self, axis):
        s = list(self.res)
        if not self.periodic:
            s[axis] += 1
        return tuple(s)

    def n_face_values(self):
        return sum(int(np.prod(self.face_shape(k))) for k in range(self.dim))

    def coarsen(self):
        if any(r % 2 or r // 2 < 4 for r in self.res):
            return None
        return GridSpec(self.dim, tuple(r // 2 for r in self.res), 2.0 * self.h, self.boundary)


class ScalarField:
    """Cell-centred values (``fields.py:92-108``); payload is a CUDA tensor."""

    def __init__(self, spec, values, dtype=torch.float64):
        t = _dev.as_dev(values, _dev.infer_dtype(values) or dtype)
        if tuple(t.shape) != spec.res:
            raise ValueError(f"scalar payload {tuple(t.shape)} != res {spec.res}")
        self.spec = spec
        self.values = t

    @classmethod
    def zeros(cls, spec, dtype=torch.float64):
        return cls(spec, torch.zeros(spec.res, dtype=dtype, device="cuda"))

    def copy(self):
        return ScalarField(self.spec, self.values.clone())


class StaggeredVectorField:
    """Face-centred vector field (``fields.py:111-133``)."""

    def __init__(self, spec, comps, dtype=torch.float64):
        dt = _dev.infer_dtype(*comps) or dtype
        comps = tuple(_dev.as_dev(c, dt) for c in comps)
        if len(comps) != spec.dim:
            raise ValueError("component count must equal dim")
        for k, c in enumerate(comps):
            if tuple(c.shape) != spec.face_shape(k):
                raise ValueError(f"component {k} shape {tuple(c.shape)} != {spec.face_shape(k)}")
        self.spec = spec
        self.comps = comps

    @classmethod
    def zeros(cls, spec, dtype=torch.float64):
        return cls(spec, tuple(torch.zeros(spec.face_shape(k), dtype=dtype, device="cuda")
                               for k in range(spec.dim)))

    def copy(self):
        return StaggeredVectorField(self.spec, tuple(c.clone() for c in self.comps))


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def _frames(spec, t):
    """Number of leading batch frames of a field tensor."""
    lead = t.shape[:t.dim() - spec.dim]
    n = 1
    for s in lead:
        n *= int(s)
    return n, tuple(lead)


def _prep(spec, *args):
    """Common input handling: returns (numpy_out, dtype, device args)."""
    _dev.require_device()
    numpy = _dev.any_numpy(*args)
    dt = _dev.infer_dtype(*args) or torch.float64
    conv = []
    for a in args:
        if isinstance(a, (tuple, list)):
            conv.append(tuple(_dev.as_dev(c, dt) for c in a))
        else:
            conv.append(_dev.as_dev(a, dt))
    return numpy, dt, conv


class _Coarse:
    """Shape-only view of the half-resolution grid (no >= 4 validation, like
    the reference's restrict_cell which only needs even extents)."""

    def __init__(self, spec):
        if any(r % 2 for r in spec.res):
            raise ValueError("restriction needs even resolution")
        self.dim = spec.dim
        self.res = tuple(r // 2 for r in spec.res)
        self.periodic = spec.periodic

    def face_shape(self, axis):
        s = list(self.res)
        if not self.periodic:
            s[axis] += 1
        return tuple(s)


def _face_like(spec, lead, dt):
    return tuple(torch.empty(lead + spec.face_shape(k), dtype=dt, device="cuda") for k in range(spec.dim))


# ---------------------------------------------------------------------------
# raw kernels (fields.py:145-358)
# ---------------------------------------------------------------------------


def zero_boundary_faces(spec, comps):
    numpy, dt, (c,) = _prep(spec, comps)
    out = tuple(x.clone() for x in c)
    n, _ = _frames(spec, out[0])
    L = _lib.load()
    _lib.check(L.smk_zero_walls(_dev.grid(spec, dt), n, _lib.ptrs(out), _dev.stream()), "zero_walls")
    return _dev.out(out, numpy)


def divergence_arrays(spec, comps):
    numpy, dt, (c,) = _prep(spec, comps)
    n, lead = _frames(spec, c[0])
    out = torch.empty(lead + spec.res, dtype=dt, device="cuda")
    L = _lib.load()
    _lib.check(L.smk_div(_dev.grid(spec, dt), n, _lib.ptrs(c), out.data_ptr(), _dev.stream()), "div")
    return _dev.out(out, numpy)


def gradient_arrays(spec, p):
    numpy, dt, (pp,) = _prep(spec, p)
    n, lead = _frames(spec, pp)
    out = _face_like(spec, lead, dt)
    L = _lib.load()
    _lib.check(L.smk_grad(_dev.grid(spec, dt), n, pp.data_ptr(), _lib.ptrs(out), _dev.stream()), "grad")
    return _dev.out(out, numpy)


def _laplacian(spec, p):
    numpy, dt, (pp,) = _prep(spec, p)
    n, lead = _frames(spec, pp)
    out = torch.empty_like(pp)
    L = _lib.load()
    _lib.check(L.smk_laplacian(_dev.grid(spec, dt), n, pp.data_ptr(), out.data_ptr(), _dev.stream()), "lap")
    return _dev.out(out, numpy)


def inf_norm(arrs):
    """``fields.py:210-216`` (device reduction)."""
    if isinstance(arrs, (np.ndarray, torch.Tensor)):
        arrs = (arrs,)
    _dev.require_device()
    L = _lib.load()
    m = 0.0
    for a in arrs:
        t = _dev.as_dev(a, _dev.infer_dtype(a) or torch.float64)
        if t.numel() == 0:
            continue
        v = ctypes.c_double()
        _lib.check(L.smk_inf_norm(_dev._DT[t.dtype], t.data_ptr(), t.numel(), ctypes.byref(v), _dev.stream()))
        m = max(m, v.value)
    return m


def dot_fields(a, b):
    """Plain inner product (``fields.py:204-207``), fixed-order device sum."""
    _dev.require_device()
    L = _lib.load()
    s = 0.0
    for x, y in zip(a, b):
        dt = _dev.infer_dtype(x, y) or torch.float64
        tx, ty = _dev.as_dev(x, dt), _dev.as_dev(y, dt)
        v = ctypes.c_double()
        _lib.check(L.smk_dot(_dev._DT[dt], tx.data_ptr(), ty.data_ptr(), tx.numel(), ctypes.byref(v),
                             _dev.stream()))
        s += v.value
    return float(s)


def restrict_cell(spec_fine, x):
    numpy, dt, (xx,) = _prep(spec_fine, x)
    n, lead = _frames(spec_fine, xx)
    gc = _Coarse(spec_fine)
    out = torch.empty(lead + gc.res, dtype=dt, device="cuda")
    L = _lib.load()
    _lib.check(L.smk_restrict_cell(_dev.grid(spec_fine, dt), n, xx.data_ptr(), out.data_ptr(), _dev.stream()))
    return _dev.out(out, numpy)


def prolong_cell(spec_coarse, spec_fine, x):
    numpy, dt, (xx,) = _prep(spec_coarse, x)
    n, lead = _frames(spec_coarse, xx)
    out = torch.empty(lead + spec_fine.res, dtype=dt, device="cuda")
    L = _lib.load()
    _lib.check(L.smk_prolong_cell(_dev.grid(spec_coarse, dt), n, xx.data_ptr(), out.data_ptr(), 0,
                                  _dev.stream()))
    return _dev.out(out, numpy)


def restrict_face(spec_fine, comps):
    """STFAS face restriction."""
    numpy, dt, (c,) = _prep(spec_fine, comps)
    n, lead = _frames(spec_fine, c[0])
    gc = _Coarse(spec_fine)
    out = _face_like(gc, lead, dt)
    L = _lib.load()
    _lib.check(L.smk_restrict_face(_dev.grid(spec_fine, dt), n, _lib.ptrs(c), _lib.ptrs(out), _dev.stream()))
    return _dev.out(out, numpy)


def prolong_face(spec_coarse, spec_fine, comps):
    numpy, dt, (c,) = _prep(spec_coarse, comps)
    n, lead = _frames(spec_coarse, c[0])
    out = _face_like(spec_fine, lead, dt)
    L = _lib.load()
    _lib.check(L.smk_prolong_face(_dev.grid(spec_coarse, dt), n, _lib.ptrs(c), _lib.ptrs(out), 0,
                                  _dev.stream()))
    return _dev.out(out, numpy)


def solve_poisson(spec, rhs, tol, max_cycles=200):
    """``fields.py:330-347``: div(grad p) = rhs - mean to ||r||_inf <= tol."""
    numpy, dt, (r,) = _prep(spec, rhs)
    p = torch.empty_like(r)
    cyc, res = ctypes.c_int(), ctypes.c_double()
    L = _lib.load()
    rc = L.smk_poisson_solve(_dev.grid(spec, dt), r.data_ptr(), p.data_ptr(), float(tol), int(max_cycles),
                             ctypes.byref(cyc), ctypes.byref(res), _dev.stream())
    if rc == _lib.SMK_NONCONVERGENCE:
        raise NonConvergence("Poisson V-cycle budget exhausted", residual=res.value,
                             context=f"{spec.res} {spec.boundary}")
    _lib.check(rc, "poisson")
    return _dev.out(p, numpy)


def project_arrays(spec, comps, tol):
    """``fields.py:350-358``."""
    numpy, dt, (c,) = _prep(spec, comps)
    out = tuple(torch.empty_like(x) for x in c)
    cyc, res = ctypes.c_int(), ctypes.c_double()
    L = _lib.load()
    rc = L.smk_project(_dev.grid(spec, dt), _lib.ptrs(c), _lib.ptrs(out), float(tol), ctypes.byref(cyc),
                       ctypes.byref(res), _dev.stream())
    if rc == _lib.SMK_NONCONVERGENCE:
        raise NonConvergence("Poisson V-cycle budget exhausted", residual=res.value,
                             context=f"{spec.res} {spec.boundary}")
    _lib.check(rc, "project")
    return _dev.out(out, numpy)


# ---------------------------------------------------------------------------
# field-level API (fields.py:365-394)
# ---------------------------------------------------------------------------


def divergence(v):
    return ScalarField(v.spec, divergence_arrays(v.spec, v.comps))


def gradient(p):
    return StaggeredVectorField(p.spec, gradient_arrays(p.spec, p.values))


def project_solenoidal(v, tol=1e-9):
    if tol <= 0:
        raise ValueError("tol must be positive")
    if inf_norm(divergence_arrays(v.spec, v.comps)) <= tol:
        if v.spec.periodic:
            return v
        comps = zero_boundary_faces(v.spec, v.comps)
        if inf_norm(divergence_arrays(v.spec, comps)) <= tol:
            return StaggeredVectorField(v.spec, comps)
    return StaggeredVectorField(v.spec, project_arrays(v.spec, v.comps, tol))
