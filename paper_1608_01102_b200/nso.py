"""STFAS / Navier-Stokes Optimization on B200.

Host mirror of the reference's specified ``nso_solver`` module: the names
(``SpacetimeState``, ``SpacetimeResidual``, ``StfasHierarchy``,
``kkt_residual``, ``scgs_smooth``, ``restrict``, ``prolong``, ``vcycle``,
``solve_nso``), argument meaning and error behaviour follow SPEC.md; all
compute runs in libsmk.so (``smk_kkt_residual``, ``smk_scgs_sweep``,
``smk_nso_*``).  State layout (pair index i = 0..N-1):

    U[i] = u_i, P[i] = p_{i+1}, V[i] = v_{i+1}, PB[i] = pbar_{i+1};
    v0 = pinned initial velocity; vstar[i] = v*_i (AoState convention,
    ``ao.py:130-141``); the K-term acts on v_1..v_{N-1}.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib, memtrack
from .errors import NonConvergence
from .fields import GridSpec


@dataclass
class StfasConfig:
    """Solver parameters (PAPER Table 1 / Alg. 2 defaults)."""

    dt: float
    K: float = 1e3
    r: float = 1e3
    omega: float = 0.8          # smoother damping
    nu1: int = 2                # pre-smoothing (Alg. 2 line PRE)
    nu2: int = 2                # post-smoothing
    n_coarse: int = 10          # coarsest sweeps (Alg. 2 line FINAL)
    color_mod: int = 2          # mod-m colouring when not red-black: 4 colours (2D) / 8 colours (3D)
    red_black: bool = True      # 2 colours by (sum_k c_k) mod 2
    n_levels: int = 99          # clipped to the grid's coarsening chain

    def params(self, N, t0=0, n_total=0):
        p = _lib.smk_nso_params()
        p.t0 = int(t0)
        p.n_total = int(n_total)
        p.n_frames = int(N)
        p.n_levels = int(self.n_levels)
        p.dt = float(self.dt)
        p.K = float(self.K)
        p.r = float(self.r)
        p.omega = float(self.omega)
        p.nu1, p.nu2, p.n_coarse = int(self.nu1), int(self.nu2), int(self.n_coarse)
        p.color_mod = int(self.color_mod)
        p.red_black = 1 if self.red_black else 0
        return p


def _faces(spec, N, dtype):
    return tuple(torch.zeros((N,) + spec.face_shape(k), dtype=dtype, device="cuda") for k in range(spec.dim))


def _cells(spec, N, dtype):
    return torch.zeros((N,) + spec.res, dtype=dtype, device="cuda")


@dataclass
class SpacetimeState:
    """(v, pbar, u, p) over the whole time line, device-resident."""

    V: tuple
    PB: torch.Tensor
    U: tuple
    P: torch.Tensor

    def __post_init__(self):
        for t in (*self.V, self.PB, *self.U, self.P):
            memtrack.register(t)

    @classmethod
    def zeros(cls, spec, N, dtype=torch.float64):
        _dev.require_device()
        return cls(_faces(spec, N, dtype), _cells(spec, N, dtype), _faces(spec, N, dtype), _cells(spec, N, dtype))

    @classmethod
    def from_arrays(cls, V, PB, U, P, dtype=None):
        _dev.require_device()
        dt = dtype or _dev.infer_dtype(V, PB, U, P) or torch.float64
        return cls(tuple(_dev.as_dev(c, dt) for c in V), _dev.as_dev(PB, dt),
                   tuple(_dev.as_dev(c, dt) for c in U), _dev.as_dev(P, dt))

    @property
    def N(self):
        return int(self.PB.shape[0])

    @property
    def dtype(self):
        return self.PB.dtype

    def copy(self):
        return SpacetimeState(tuple(c.clone() for c in self.V), self.PB.clone(),
                              tuple(c.clone() for c in self.U), self.P.clone())

    def numpy(self):
        f = lambda t: t.detach().cpu().numpy()
        return (tuple(f(c) for c in self.V), f(self.PB), tuple(f(c) for c in self.U), f(self.P))

    def c_struct(self):
        s = _lib.smk_state()
        for k, c in enumerate(self.V):
            s.V[k] = c.data_ptr()
        for k, c in enumerate(self.U):
            s.U[k] = c.data_ptr()
        s.PB = self.PB.data_ptr()
        s.P = self.P.data_ptr()
        return s


@dataclass
class SpacetimeResidual:
    """The four Eq. 8 blocks."""

    R1: tuple
    R2: torch.Tensor
    R3: tuple
    R4: torch.Tensor

    def __post_init__(self):
        for t in (*self.R1, self.R2, *self.R3, self.R4):
            memtrack.register(t)

    @classmethod
    def zeros(cls, spec, N, dtype=torch.float64):
        return cls(_faces(spec, N, dtype), _cells(spec, N, dtype), _faces(spec, N, dtype), _cells(spec, N, dtype))

    @classmethod
    def empty(cls, spec, N, dtype=torch.float64):
        """Uninitialised buffers for a kernel that writes every row."""
        f = lambda: tuple(torch.empty((N,) + spec.face_shape(k), dtype=dtype, device="cuda") for k in range(spec.dim))
        c = lambda: torch.empty((N,) + tuple(spec.res), dtype=dtype, device="cuda")
        return cls(f(), c(), f(), c())

    def c_struct(self):
        s = _lib.smk_residual()
        for k, c in enumerate(self.R1):
            s.R1[k] = c.data_ptr()
        for k, c in enumerate(self.R3):
            s.R3[k] = c.data_ptr()
        s.R2 = self.R2.data_ptr()
        s.R4 = self.R4.data_ptr()
        return s

    def arrays(self):
        return tuple(self.R1) + (self.R2,) + tuple(self.R3) + (self.R4,)

    def inf(self):
        return max(float(a.abs().max()) if a.numel() else 0.0 for a in self.arrays())

    def numpy(self):
        f = lambda t: t.detach().cpu().numpy()
        return (tuple(f(c) for c in self.R1), f(self.R2), tuple(f(c) for c in self.R3), f(self.R4))


def _guide(spec, v0, vstar, dtype):
    v0 = tuple(_dev.as_dev(c, dtype) for c in v0)
    vs = tuple(_dev.as_dev(c, dtype) for c in vstar)
    return v0, vs


def kkt_residual(spec, cfg, s, v0, vstar, rhs=None):
    """Eq. 8 residual f(s) - rhs."""
    _dev.require_device()
    dt = s.dtype
    v0, vs = _guide(spec, v0, vstar, dt)
    out = SpacetimeResidual.zeros(spec, s.N, dt)
    L = _lib.load()
    st = s.c_struct()
    o = out.c_struct()
    r = rhs.c_struct() if rhs is not None else None
    rc = L.smk_kkt_residual(ctypes.byref(_dev.grid(spec, dt)), ctypes.byref(cfg.params(s.N)), ctypes.byref(st),
                            _lib.ptrs(v0), _lib.ptrs(vs), ctypes.byref(r) if r is not None else None,
                            ctypes.byref(o), _dev.stream())
    _lib.check(rc, "kkt_residual")
    return out


def scgs_smooth(spec, cfg, s, v0, vstar, rhs=None):
    """One coloured time-line SCGS sweep in place."""
    _dev.require_device()
    dt = s.dtype
    v0, vs = _guide(spec, v0, vstar, dt)
    L = _lib.load()
    st = s.c_struct()
    r = rhs.c_struct() if rhs is not None else None
    rc = L.smk_scgs_sweep(ctypes.byref(_dev.grid(spec, dt)), ctypes.byref(cfg.params(s.N)), ctypes.byref(st),
                          _lib.ptrs(v0), _lib.ptrs(vs), ctypes.byref(r) if r is not None else None, _dev.stream())
    _lib.check(rc, "scgs_smooth")
    return s


def restrict(spec_fine, x):
    """Per-frame spatial restriction of a state / residual."""
    from .fields import restrict_cell, restrict_face
    if isinstance(x, SpacetimeState):
        return SpacetimeState(restrict_face(spec_fine, x.V), restrict_cell(spec_fine, x.PB),
                              restrict_face(spec_fine, x.U), restrict_cell(spec_fine, x.P))
    if isinstance(x, SpacetimeResidual):
        return SpacetimeResidual(restrict_face(spec_fine, x.R1), restrict_cell(spec_fine, x.R2),
                                 restrict_face(spec_fine, x.R3), restrict_cell(spec_fine, x.R4))
    if isinstance(x, (tuple, list)):
        return restrict_face(spec_fine, x)
    return restrict_cell(spec_fine, x)


def prolong(spec_coarse, x):
    """Per-frame spatial prolongation."""
    from .fields import prolong_cell, prolong_face
    fine = GridSpec(spec_coarse.dim, tuple(2 * r for r in spec_coarse.res), spec_coarse.h / 2,
                    spec_coarse.boundary)
    if isinstance(x, SpacetimeState):
        return SpacetimeState(prolong_face(spec_coarse, fine, x.V), prolong_cell(spec_coarse, fine, x.PB),
                              prolong_face(spec_coarse, fine, x.U), prolong_cell(spec_coarse, fine, x.P))
    if isinstance(x, (tuple, list)):
        return prolong_face(spec_coarse, fine, x)
    return prolong_cell(spec_coarse, fine, x)


class StfasHierarchy:
    """Device-resident level hierarchy over libsmk's handle."""

    def __init__(self, spec, cfg, N, dtype=torch.float64, t0=0, n_total=0):
        _dev.require_device()
        self.spec, self.cfg, self.N, self.dtype = spec, cfg, int(N), dtype
        L = _lib.load()
        self._L = L
        self._g = _dev.grid(spec, dtype)
        self._p = cfg.params(N, t0, n_total)
        h = L.smk_nso_create(ctypes.byref(self._g), ctypes.byref(self._p))
        if not h:
            _lib.check(_lib.SMK_ERR_CUDA if "alloc" in _lib.last_error() else _lib.SMK_ERR_ARG, "nso_create")
        self._h = h
        self._guide = None
        self._payload = memtrack.OwnedPayload(L.smk_nso_payload_values(h))

    @property
    def levels(self):
        return self._L.smk_nso_levels(self._h)

    @property
    def device_bytes(self):
        return int(self._L.smk_nso_device_bytes(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._L.smk_nso_destroy(self._h)
            self._h = None
            self._payload = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def profile(self, enable=True):
        _lib.check(self._L.smk_nso_profile(self._h, int(bool(enable))), "profile")

    KERNELS = {0: "k_scgs_fwd", 1: "k_scgs_apply", 2: "k_kkt", 3: "k_scgs_back"}

    def profile_read(self, kind=0, level=None):
        """(summed kernel ms, launches, cell-timesteps) for kernel `kind`
        (KERNELS), over all levels or one hierarchy level."""
        ms, n, cells = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_longlong()
        if level is None:
            rc = self._L.smk_nso_profile_read(self._h, int(kind), ctypes.byref(ms), ctypes.byref(n), ctypes.byref(cells))
        else:
            rc = self._L.smk_nso_profile_read_level(self._h, int(kind), int(level), ctypes.byref(ms), ctypes.byref(n),
                                                    ctypes.byref(cells))
        _lib.check(rc, "profile_read")
        return ms.value, n.value, cells.value

    def set_guide(self, v0, vstar):
        v0, vs = _guide(self.spec, v0, vstar, self.dtype)
        self._guide = (v0, vs)   # keep alive: the handle stores the pointers
        _lib.check(self._L.smk_nso_set_guide(self._h, _lib.ptrs(v0), _lib.ptrs(vs), _dev.stream()), "set_guide")

    def set_K(self, K):
        """Update K on the handle in place (the LM shift)."""
        _lib.check(self._L.smk_nso_set_K(self._h, float(K)), "set_K")

    def vcycle(self, s):
        st = s.c_struct()
        _lib.check(self._L.smk_nso_vcycle(self._h, ctypes.byref(st), _dev.stream()), "vcycle")
        return s

    def gauge_fix(self, s):
        st = s.c_struct()
        _lib.check(self._L.smk_nso_gauge_fix(self._h, ctypes.byref(st), _dev.stream()), "gauge_fix")
        return s

    def residual_norms(self, s):
        st = s.c_struct()
        ri, r2 = ctypes.c_double(), ctypes.c_double()
        _lib.check(self._L.smk_nso_residual_norms(self._h, ctypes.byref(st), ctypes.byref(ri), ctypes.byref(r2),
                                                  _dev.stream()), "residual_norms")
        return ri.value, r2.value

    def solve(self, s, eps=1e-5, relative=False, cycle_budget=50):
        hist = (ctypes.c_double * (2 * (cycle_budget + 1)))()
        cyc = ctypes.c_int()
        st = s.c_struct()
        rc = self._L.smk_nso_solve(self._h, ctypes.byref(st), float(eps), int(bool(relative)), int(cycle_budget),
                                   ctypes.byref(cyc), hist, _dev.stream())
        h = [(c, hist[2 * c], hist[2 * c + 1]) for c in range(cyc.value + 1)]
        if rc == _lib.SMK_NONCONVERGENCE:
            raise NonConvergence(_lib.last_error(), residual=h[-1][1], context=f"{cyc.value} V-cycles")
        _lib.check(rc, "solve_nso")
        return h


def vcycle(hier, s):
    """One FAS V-cycle (PAPER Alg. 2)."""
    return hier.vcycle(s)


@dataclass
class NsoResult:
    state: SpacetimeState
    history: list = field(default_factory=list)   # (cycle, res_inf, res_l2)
    converged: bool = True
    hierarchy: object = None


def solve_nso(spec, cfg, v0, vstar, s=None, eps=1e-5, cycle_budget=50, relative=False, dtype=None,
              hierarchy=None, lm=False, lm_stall=None):
    """Repeat V-cycles until ||f||_inf <= eps.

    Raises NonConvergence when the cycle budget is exhausted.  With ``lm``
    the Levenberg-Marquardt safeguard of SPEC.md:347 runs (``_solve_lm``)."""
    _dev.require_device()
    N = int(vstar[0].shape[0])
    dt = dtype or (s.dtype if s is not None else (_dev.infer_dtype(vstar) or torch.float64))
    if s is None:
        s = SpacetimeState.zeros(spec, N, dt)
    hier = hierarchy or StfasHierarchy(spec, cfg, N, dt)
    hier.set_guide(v0, vstar)
    if lm:
        hist = _solve_lm(spec, cfg, hier, v0, vstar, s, eps, relative, cycle_budget,
                         LM_STALL if lm_stall is None else lm_stall)
    else:
        hist = hier.solve(s, eps=eps, relative=relative, cycle_budget=cycle_budget)
    return NsoResult(s, hist, True, hier)


LM_WINDOW = 3          # cycles over which the reduction factor is measured
LM_STALL = 0.95        # per-cycle factor above which the shift is raised
LM_MIN_SHIFT = 1e-3    # shift (relative to K) below which it is dropped
LM_MAX_SHIFT = 1e3     # cap on the shift (relative to K)


def _solve_lm(spec, cfg, hier, v0, vstar, s, eps, relative, budget, stall=LM_STALL):
    """SPEC.md:347 LM safeguard, frozen as a proximal shift.

    The per-cycle reduction factor of ||f||_inf over the last LM_WINDOW
    cycles is tested once LM_WINDOW cycles have run since the last change of
    the shift sigma: above LM_STALL sigma is raised (K, then doubled, capped
    at LM_MAX_SHIFT K), otherwise halved and dropped below LM_MIN_SHIFT K.  A
    shifted V-cycle solves the damped problem K' = K + sigma with guide
    (K v* + sigma v^k) / K' (v^k = the iterate entering the cycle): the K-term
    becomes K/r (v - v*) + sigma/r (v - v^k), so every fixed point of the
    damped cycles is the undamped solution.  One damped hierarchy serves every
    sigma (K updated in place, smk_nso_set_K) and its guide lives in
    persistent buffers updated in place, so the captured V-cycle graph is
    re-instantiated only when sigma changes.  The stop test always uses the
    undamped residual.  Raises NonConvergence when the budget is exhausted."""
    dt = s.dtype
    v0d, vs = _guide(spec, v0, vstar, dt)
    ri, r2 = hier.residual_norms(s)
    hist = [(0, ri, r2)]
    tol = eps * ri if relative else eps
    if ri <= tol:
        return hist
    sigma, changed = 0.0, 0
    damped, guide = None, None
    N = s.N
    try:
        for c in range(1, budget + 1):
            if sigma > 0:
                if damped is None:
                    damped = StfasHierarchy(spec, cfg, N, dt)
                    guide = tuple(g.clone() for g in vs)
                    damped.set_guide(v0d, guide)
                damped.set_K(cfg.K + sigma)
                a, b = cfg.K / (cfg.K + sigma), sigma / (cfg.K + sigma)
                for k in range(spec.dim):
                    if N > 1:
                        guide[k][1:].copy_(vs[k][1:])
                        _axpby_dev(guide[k][1:], s.V[k][:N - 1], b, a)
                damped.set_guide(v0d, guide)   # re-restricts the coarse guides
                damped.vcycle(s)
                damped.gauge_fix(s)
            else:
                hier.vcycle(s)
                hier.gauge_fix(s)
            ri, r2 = hier.residual_norms(s)
            hist.append((c, ri, r2))
            if ri <= tol:
                return hist
            if c - changed >= LM_WINDOW:
                prev = hist[c - LM_WINDOW][1]
                factor = (ri / prev) ** (1.0 / LM_WINDOW) if prev > 0 else 0.0
                new = sigma
                if factor > stall:
                    new = cfg.K if sigma == 0 else min(2.0 * sigma, LM_MAX_SHIFT * cfg.K)
                elif sigma > 0:
                    new = 0.5 * sigma
                    if new < LM_MIN_SHIFT * cfg.K:
                        new = 0.0
                if new != sigma:
                    sigma, changed = new, c
    finally:
        if damped is not None:
            damped.close()
    raise NonConvergence(f"STFAS (LM) cycle budget exhausted (residual {hist[-1][1]:.3e} > {tol:.3e})",
                         residual=hist[-1][1], context=f"{budget} V-cycles")


def _axpby_dev(y, x, a, b):
    """y <- a x + b y on a (possibly strided-frame) contiguous slice."""
    _lib.check(_lib.load().smk_axpby(_dev._DT[y.dtype], y.data_ptr(), x.data_ptr(), float(a), float(b), y.numel(),
                                     _dev.stream()), "axpby")
