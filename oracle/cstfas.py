"""ctypes binding of the C STFAS oracle (TEST INFRASTRUCTURE AND CPU BASELINE ONLY).

``oracle/cstfas.c`` restates ``oracle/stfas.py`` point by point (same
algorithm: probed local Jacobians, 2N-block partially pivoted block Thomas,
snapshot colour passes, FAS V-cycle) in multithreaded C so the oracle runs at
the BASELINE configs' real sizes.  The API mirrors ``oracle/stfas.py``:
``kkt_residual``, ``scgs_color``, ``scgs_smooth``, ``Hierarchy.vcycle`` /
``solve``; inputs are the same ``stfas.Problem`` / ``stfas.State`` numpy
objects.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
legs may use it.
"""

import ctypes
import os
import subprocess

import numpy as np

from . import stfas

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cstfas.c")
LIB = os.path.join(HERE, "_build", "libcstfas.so")
CFLAGS = ["-O3", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared"]

_P = ctypes.POINTER(ctypes.c_double)


class CGrid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n", ctypes.c_int * 3), ("h", ctypes.c_double), ("per", ctypes.c_int)]


class CState(ctypes.Structure):
    _fields_ = [("V", _P * 3), ("PB", _P), ("U", _P * 3), ("P", _P)]


class CRes(ctypes.Structure):
    _fields_ = [("R1", _P * 3), ("R2", _P), ("R3", _P * 3), ("R4", _P)]


class CProb(ctypes.Structure):
    _fields_ = [("g", CGrid), ("N", ctypes.c_int), ("dt", ctypes.c_double), ("K", ctypes.c_double),
                ("r", ctypes.c_double), ("omega", ctypes.c_double), ("colors", ctypes.c_int),
                ("t0", ctypes.c_int), ("Ng", ctypes.c_int), ("v0", _P * 3), ("vstar", _P * 3),
                ("vs_frames", ctypes.c_int), ("unext", _P * 3), ("red_black", ctypes.c_int)]


def build(force=False):
    """gcc the oracle into oracle/_build (no-op when up to date)."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + ".tmp"
    subprocess.check_call(["gcc"] + CFLAGS + ["-o", tmp, SRC])
    os.replace(tmp, LIB)
    return LIB


_lib = None


def load():
    global _lib
    if _lib is None:
        if os.path.exists(SRC):
            build()   # no-op when up to date (the GPU box has only the prebuilt .so)
        L = ctypes.CDLL(LIB)
        L.cst_hier_create.restype = ctypes.c_void_p
        L.cst_hier_create.argtypes = [ctypes.POINTER(CProb), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.cst_hier_destroy.argtypes = [ctypes.c_void_p]
        L.cst_hier_levels.argtypes = [ctypes.c_void_p]
        L.cst_hier_vcycle.argtypes = [ctypes.c_void_p, ctypes.POINTER(CState), ctypes.c_int]
        L.cst_hier_norms.argtypes = [ctypes.c_void_p, ctypes.POINTER(CState), _P, _P]
        L.cst_hier_solve.argtypes = [ctypes.c_void_p, ctypes.POINTER(CState), ctypes.c_double, ctypes.c_int,
                                     ctypes.c_int, ctypes.POINTER(ctypes.c_int), _P]
        L.cst_kkt_residual.argtypes = [ctypes.POINTER(CProb), ctypes.POINTER(CState), ctypes.POINTER(CRes),
                                       ctypes.POINTER(CRes)]
        L.cst_color_pass.argtypes = [ctypes.POINTER(CProb), ctypes.POINTER(CState), ctypes.POINTER(CRes), ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int), ctypes.c_int64, ctypes.c_int, _P]
        L.cst_sweep.argtypes = [ctypes.POINTER(CProb), ctypes.POINTER(CState), ctypes.POINTER(CRes)]
        L.cst_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def set_threads(n=0):
    """OpenMP threads (0 = query); returns the thread count in use."""
    return load().cst_set_threads(int(n))


def _ptr(a):
    return a.ctypes.data_as(_P)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _Keep:
    """Holds the numpy buffers behind a C struct alive."""

    def __init__(self):
        self.refs = []

    def p(self, a):
        a = _c(a)
        self.refs.append(a)
        return _ptr(a)


def _grid(g):
    cg = CGrid()
    cg.dim = g.dim
    for a in range(3):
        cg.n[a] = g.res[a] if a < g.dim else 1
    cg.h = g.h
    cg.per = 1 if g.periodic else 0
    return cg


def _prob(pb, keep):
    c = CProb()
    c.g = _grid(pb.g)
    c.N = pb.N
    c.dt, c.K, c.r, c.omega = pb.dt, pb.K, pb.r, pb.omega
    c.colors = pb.colors
    c.t0 = pb.t0
    c.Ng = pb.N_global
    for k in range(pb.g.dim):
        c.v0[k] = keep.p(pb.v0[k])
        c.vstar[k] = keep.p(pb.vstar[k])
        if pb.unext is not None:
            c.unext[k] = keep.p(pb.unext[k])
    c.vs_frames = pb.vstar[0].shape[0]
    c.red_black = 1 if pb.red_black else 0
    return c


def _state(st, keep, copy=True):
    """C view of a State; with copy the arrays are fresh (C writes in place)."""
    arrs = State_arrays(st, copy)
    c = CState()
    d = len(arrs[0])
    for k in range(d):
        c.V[k] = keep.p(arrs[0][k])
        c.U[k] = keep.p(arrs[2][k])
    c.PB = keep.p(arrs[1])
    c.P = keep.p(arrs[3])
    return c, arrs


def State_arrays(st, copy):
    f = (lambda a: np.array(a, dtype=np.float64, copy=True)) if copy else _c
    return (tuple(f(v) for v in st.V), f(st.PB), tuple(f(u) for u in st.U), f(st.P))


def _res(r, keep):
    c = CRes()
    for k in range(len(r.R1)):
        c.R1[k] = keep.p(r.R1[k])
        c.R3[k] = keep.p(r.R3[k])
    c.R2 = keep.p(r.R2)
    c.R4 = keep.p(r.R4)
    return c


def _zeros_res(g, N):
    f = lambda: tuple(np.zeros((N,) + g.face_shape(k)) for k in range(g.dim))
    return stfas.Residual(f(), np.zeros((N,) + g.res), f(), np.zeros((N,) + g.res))


def kkt_residual(pb, st, rhs=None):
    """f(st) - rhs (oracle/stfas.py kkt_residual)."""
    L = load()
    keep = _Keep()
    cp = _prob(pb, keep)
    cs, _ = _state(st, keep, copy=False)
    out = _zeros_res(pb.g, pb.N)
    co = _res(out, keep)
    cr = _res(rhs, keep) if rhs is not None else None
    L.cst_kkt_residual(ctypes.byref(cp), ctypes.byref(cs), ctypes.byref(cr) if cr is not None else None,
                       ctypes.byref(co))
    return out


def _as_state(arrs):
    return stfas.State(tuple(arrs[0]), arrs[1], tuple(arrs[2]), arrs[3])


def scgs_color(pb, st, rhs, color, cells=None, return_delta=False):
    """One colour pass (oracle/stfas.py scgs_color); cells = (M, dim) subset."""
    L = load()
    keep = _Keep()
    cp = _prob(pb, keep)
    cs, arrs = _state(st, keep, copy=True)
    cr = _res(rhs, keep) if rhs is not None else None
    cptr, M = None, 0
    if cells is not None:
        cells = np.asarray(cells, dtype=np.int32).reshape(-1, pb.g.dim)
        c3 = np.zeros((cells.shape[0], 3), dtype=np.int32)
        c3[:, :pb.g.dim] = cells
        keep.refs.append(c3)
        cptr, M = c3.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), c3.shape[0]
    else:
        col = stfas.color_of(pb.g, pb.colors, pb.red_black)
        M = int(np.sum(col == color))
    b = 2 * pb.g.dim + 1
    x = np.zeros((M, 2 * pb.N, b))
    rc = L.cst_color_pass(ctypes.byref(cp), ctypes.byref(cs), ctypes.byref(cr) if cr is not None else None,
                          int(color), cptr, M, 1, _ptr(x))
    if rc:
        raise RuntimeError(f"cstfas colour pass: singular block (rc {rc})")
    out = _as_state(arrs)
    return (out, x) if return_delta else out


def scgs_smooth(pb, st, rhs=None):
    L = load()
    keep = _Keep()
    cp = _prob(pb, keep)
    cs, arrs = _state(st, keep, copy=True)
    cr = _res(rhs, keep) if rhs is not None else None
    L.cst_sweep(ctypes.byref(cp), ctypes.byref(cs), ctypes.byref(cr) if cr is not None else None)
    return _as_state(arrs)


class Hierarchy:
    """StfasHierarchy of the C oracle (levels built like stfas.build_levels)."""

    def __init__(self, pb, n_levels=99, nu1=2, nu2=2, n_coarse=10):
        self.L = load()
        self.pb = pb
        self._keep = _Keep()
        self._cp = _prob(pb, self._keep)
        self.h = self.L.cst_hier_create(ctypes.byref(self._cp), int(n_levels), nu1, nu2, n_coarse)

    @property
    def levels(self):
        return self.L.cst_hier_levels(self.h)

    def close(self):
        if self.h:
            self.L.cst_hier_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def vcycle(self, st, gauge=False):
        """One FAS V-cycle (+ gauge fix); returns a new State."""
        keep = _Keep()
        cs, arrs = _state(st, keep, copy=True)
        self.L.cst_hier_vcycle(self.h, ctypes.byref(cs), int(bool(gauge)))
        return _as_state(arrs)

    def norms(self, st):
        keep = _Keep()
        cs, _ = _state(st, keep, copy=False)
        a, b = ctypes.c_double(), ctypes.c_double()
        self.L.cst_hier_norms(self.h, ctypes.byref(cs), ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def solve(self, st=None, eps=1e-5, relative=False, cycle_budget=50):
        """solve_nso: returns (State, history [(cycle, inf, l2)], converged)."""
        if st is None:
            st = stfas.zero_state(self.pb.g, self.pb.N)
        keep = _Keep()
        cs, arrs = _state(st, keep, copy=True)
        hist = np.zeros(2 * (cycle_budget + 1))
        cyc = ctypes.c_int()
        rc = self.L.cst_hier_solve(self.h, ctypes.byref(cs), float(eps), int(bool(relative)), int(cycle_budget),
                                   ctypes.byref(cyc), _ptr(hist))
        h = [(c, hist[2 * c], hist[2 * c + 1]) for c in range(cyc.value + 1)]
        return _as_state(arrs), h, rc == 0
