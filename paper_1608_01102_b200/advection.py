"""Transport on B200 — drop-in for ``pkg/src/smokectrl/advection.py``.

Skew scalar stencil T(v), truncated exp(T dt) with adaptive order, its rho-
and v-adjoints, self-advection S(a, w), its Jacobian and transpose, and the
semi-Lagrangian comparator; every call runs on libsmk.so kernels.
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _dev, _lib
from .errors import TruncationOverflow
from .fields import ScalarField, StaggeredVectorField, _face_like, _frames, _prep, zero_boundary_faces

DEFAULT_TRUNCATION_TOL = 1e-5
DEFAULT_TERM_CAP = 128


@dataclass(frozen=True)
class TruncationReport:
    """``advection.py:137-141``."""

    k_used: int
    last_term_norm: float


def transport_scalar(spec, vcomps, rho):
    """``advection.py:88-97`` (batch frames on rho and v)."""
    numpy, dt, (v, r) = _prep(spec, vcomps, rho)
    n, lead = _frames(spec, r)
    nv, _ = _frames(spec, v[0])
    if nv not in (1, n):
        raise ValueError("velocity batch must be 1 or match rho")
    if nv == 1 and n > 1:
        v = tuple(x.reshape((1,) + x.shape[x.dim() - spec.dim:]).expand((n,) + x.shape[x.dim() - spec.dim:])
                  .contiguous() for x in v)
    out = torch.empty_like(r)
    L = _lib.load()
    _lib.check(L.smk_transport_scalar(_dev.grid(spec, dt), n, _lib.ptrs(v), r.data_ptr(), out.data_ptr(),
                                      _dev.stream()), "transport_scalar")
    return _dev.out(out, numpy)


def transport_scalar_T(spec, vcomps, rho):
    """``advection.py:100-102``: T^T = -T."""
    out = transport_scalar(spec, vcomps, rho)
    return -out


def scalar_stencil_v_adjoint(spec, x, y):
    """``advection.py:105-130``."""
    numpy, dt, (xx, yy) = _prep(spec, x, y)
    n, lead = _frames(spec, xx)
    out = _face_like(spec, lead, dt)
    L = _lib.load()
    _lib.check(L.smk_scalar_stencil_v_adjoint(_dev.grid(spec, dt), n, xx.data_ptr(), yy.data_ptr(),
                                              _lib.ptrs(out), _dev.stream()))
    return _dev.out(out, numpy)


def _taylor(spec, vcomps, rho, dt_, tol, cap, k_fixed, transpose):
    numpy, dt, (v, r) = _prep(spec, vcomps, rho)
    if not dt_ > 0:
        raise ValueError("dt must be positive")
    out = torch.empty_like(r)
    k = ctypes.c_int()
    last = ctypes.c_double()
    L = _lib.load()
    rc = L.smk_advect(_dev.grid(spec, dt), _lib.ptrs(v), r.data_ptr(), out.data_ptr(), float(dt_), float(tol),
                      int(cap), int(k_fixed or 0), int(bool(transpose)), ctypes.byref(k), ctypes.byref(last),
                      _dev.stream())
    if rc == _lib.SMK_TRUNCATION_OVERFLOW:
        raise TruncationOverflow(f"Taylor term cap {cap} exceeded (dt*|v|/h too large)", k_cap=cap,
                                 last_term_norm=last.value)
    _lib.check(rc, "advect")
    return _dev.out(out, numpy), TruncationReport(k.value, last.value)


def advect_scalar(spec, vcomps, rho, dt, tol=DEFAULT_TRUNCATION_TOL, cap=DEFAULT_TERM_CAP, k_fixed=None):
    """``advection.py:165-168``."""
    return _taylor(spec, vcomps, rho, dt, tol, cap, k_fixed, False)


def advect_scalar_rho_T(spec, vcomps, mu, dt, tol=DEFAULT_TRUNCATION_TOL, cap=DEFAULT_TERM_CAP, k_fixed=None):
    """``advection.py:171-174``."""
    return _taylor(spec, vcomps, mu, dt, tol, cap, k_fixed, True)


def advect_scalar_v_T(spec, vcomps, rho, mu, dt, tol=DEFAULT_TRUNCATION_TOL, cap=DEFAULT_TERM_CAP, k_fixed=None):
    """``advection.py:177-210``; returns (face field, TruncationReport)."""
    k = k_fixed
    if k is None:
        _, rep = advect_scalar(spec, vcomps, rho, dt, tol, cap)
        k = rep.k_used
    numpy, dtp, (v, r, m) = _prep(spec, vcomps, rho, mu)
    out = _face_like(spec, (), dtp)
    L = _lib.load()
    _lib.check(L.smk_advect_v_T(_dev.grid(spec, dtp), _lib.ptrs(v), r.data_ptr(), m.data_ptr(), _lib.ptrs(out),
                                float(dt), int(k), _dev.stream()), "advect_v_T")
    return _dev.out(out, numpy), TruncationReport(int(k), float("nan"))


def _face_op(name, spec, a, w):
    numpy, dt, (aa, ww) = _prep(spec, a, w)
    n, lead = _frames(spec, aa[0])
    out = _face_like(spec, lead, dt)
    L = _lib.load()
    _lib.check(getattr(L, name)(_dev.grid(spec, dt), n, _lib.ptrs(aa), _lib.ptrs(ww), _lib.ptrs(out),
                                _dev.stream()), name)
    return _dev.out(out, numpy)


def transport_face(spec, acomps, wcomps):
    """S(a, w), ``advection.py:353-365``."""
    return _face_op("smk_transport_face", spec, acomps, wcomps)


def self_advection(spec, vcomps):
    """``advection.py:368-370``."""
    return transport_face(spec, vcomps, vcomps)


def self_adv_jacobian_apply(spec, vcomps, dcomps):
    """``advection.py:373-377``."""
    return _face_op("smk_self_adv_jac", spec, vcomps, dcomps)


def self_adv_jacobian_T_apply(spec, vcomps, ucomps):
    """``advection.py:437-441``."""
    return _face_op("smk_self_adv_jac_T", spec, vcomps, ucomps)


def semi_lagrangian(rho, v, dt):
    """``advection.py:264-272`` (field-level, like the reference)."""
    spec = rho.spec
    vc = zero_boundary_faces(spec, v.comps)
    numpy, dtp, (vv, r) = _prep(spec, vc, rho.values)
    out = torch.empty_like(r)
    L = _lib.load()
    _lib.check(L.smk_semi_lagrangian(_dev.grid(spec, dtp), _lib.ptrs(vv), r.data_ptr(), out.data_ptr(), float(dt),
                                     _dev.stream()))
    return ScalarField(spec, out)


class AdvectionOperator:
    """``advection.py:213-248``."""

    def __init__(self, v, truncation_tol=DEFAULT_TRUNCATION_TOL, cap=DEFAULT_TERM_CAP):
        self.spec = v.spec
        self.vcomps = zero_boundary_faces(v.spec, v.comps)
        self.truncation_tol = truncation_tol
        self.cap = cap

    def apply_stencil(self, rho):
        return ScalarField(self.spec, transport_scalar(self.spec, self.vcomps, rho.values))

    def advect(self, rho, dt):
        if dt <= 0:
            raise ValueError("dt must be positive")
        out, rep = advect_scalar(self.spec, self.vcomps, rho.values, dt, self.truncation_tol, self.cap)
        return ScalarField(self.spec, out), rep

    def jacobian_rho_T(self, mu, dt, k_fixed=None):
        out, rep = advect_scalar_rho_T(self.spec, self.vcomps, mu.values, dt, self.truncation_tol, self.cap,
                                       k_fixed)
        return ScalarField(self.spec, out), rep

    def jacobian_v_T(self, rho, mu, dt, k_fixed=None):
        out, _ = advect_scalar_v_T(self.spec, self.vcomps, rho.values, mu.values, dt, self.truncation_tol,
                                   self.cap, k_fixed)
        return StaggeredVectorField(self.spec, out)
