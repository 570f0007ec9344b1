"""STFAS / NSO solver in fp64 numpy (TEST INFRASTRUCTURE ONLY).

The reference ships no STFAS code; this restates the
specification: ``SPEC.md:285-374`` (nso_solver), PAPER Eq. 8
(``PAPER.md:226-233``), Eq. 9 (``PAPER.md:317-334``), Alg. 2
(``PAPER.md:261-300``) and Appendix A (``PAPER.md:549-564``), with the
semantic decisions frozen in DESIGN.md §3:

Unknowns (pair index i = 0..N-1)
    U[i] = u_i, P[i] = p_{i+1}, V[i] = v_{i+1}, PB[i] = pbar_{i+1};
    v_0 is pinned (initial condition), vstar holds v*_0..v*_{N-1}
    (``ao.py:130-141`` convention) and the K-term acts on v_1..v_{N-1}.
Rows (wall rows masked)
    R3[i] = (v_{i+1}-v_i)/dt + Adv(v_{i+1}) - u_i + grad p_{i+1}
    R4[i] = div u_i
    R1[i] = (K/r)(v_{i+1}-v*_{i+1})[i<N-1] - u_{i+1}/dt [i<N-1]
            + u_i/dt + J_Adv(v_{i+1})^T u_i + grad pbar_{i+1}
    R2[i] = div v_{i+1}
Smoother
    coloured (mod-2: 4 colours 2D / 8 colours 3D) time-line SCGS / Vanka:
    for each colour, with the state frozen (snapshot reads), every cell of
    the colour solves the Gauss-Newton Eq. 9 block-tridiagonal system of its
    2N blocks of (2d faces + 1 scalar) by block Thomas (partial pivoting
    inside each block), then all of the colour's unknowns take x += omega*dx.
"""

from dataclasses import dataclass, field

import numpy as np

from . import ops


# ---------------------------------------------------------------------------
# containers
# ---------------------------------------------------------------------------


@dataclass
class State:
    V: tuple
    PB: np.ndarray
    U: tuple
    P: np.ndarray

    def copy(self):
        return State(tuple(c.copy() for c in self.V), self.PB.copy(),
                     tuple(c.copy() for c in self.U), self.P.copy())

    def axpy(self, a, other):
        """self + a*other (new State)."""
        return State(tuple(x + a * y for x, y in zip(self.V, other.V)),
                     self.PB + a * other.PB,
                     tuple(x + a * y for x, y in zip(self.U, other.U)),
                     self.P + a * other.P)


@dataclass
class Residual:
    R1: tuple
    R2: np.ndarray
    R3: tuple
    R4: np.ndarray

    def inf(self):
        return ops.inf_norm(self.R1 + (self.R2,) + self.R3 + (self.R4,))

    def l2(self):
        return float(np.sqrt(sum(float(np.vdot(a, a)) for a in
                                 self.R1 + (self.R2,) + self.R3 + (self.R4,))))

    def sub(self, o):
        return Residual(tuple(a - b for a, b in zip(self.R1, o.R1)), self.R2 - o.R2,
                        tuple(a - b for a, b in zip(self.R3, o.R3)), self.R4 - o.R4)

    def add(self, o):
        return Residual(tuple(a + b for a, b in zip(self.R1, o.R1)), self.R2 + o.R2,
                        tuple(a + b for a, b in zip(self.R3, o.R3)), self.R4 + o.R4)


@dataclass
class Problem:
    g: object
    dt: float
    K: float
    r: float
    v0: tuple          # pinned initial velocity (face arrays)
    vstar: tuple       # (N, face) stacks: v*_0 .. v*_{N-1}
    omega: float = 0.8
    colors: int = 2    # colouring modulus per axis (2 -> 2^d colours), when not red-black
    red_black: bool = True   # 2 colours by (sum_k c_k) mod 2
    # time-slab mode: local pairs t0 .. t0+n_pairs-1 of Ng;
    # v0 is the left halo, unext the right halo u_{t0+n_pairs}, vstar holds
    # n_pairs + 1 frames (v*_{t0} .. v*_{t0+n_pairs})
    t0: int = 0
    Ng: int = 0
    n_pairs: int = 0
    unext: tuple = None

    @property
    def N(self):
        return self.n_pairs if self.n_pairs else self.vstar[0].shape[0]

    @property
    def N_global(self):
        return self.Ng if self.Ng else self.N

    @property
    def kr(self):
        return self.K / self.r


def zero_state(g, N):
    return State(tuple(np.zeros((N,) + g.face_shape(k)) for k in range(g.dim)),
                 np.zeros((N,) + g.res),
                 tuple(np.zeros((N,) + g.face_shape(k)) for k in range(g.dim)),
                 np.zeros((N,) + g.res))


def _mask(g, comps):
    return ops.zero_walls(g, comps)


# ---------------------------------------------------------------------------
# Eq. 8 residual
# ---------------------------------------------------------------------------


def kkt_residual(pb, st):
    g, N, dt = pb.g, pb.N, pb.dt
    V, U = st.V, st.U
    vprev = tuple(np.concatenate([v0[None], v[:-1]], axis=0)
                  for v0, v in zip(pb.v0, V))
    adv = ops.self_advection(g, V)
    gp = ops.grad(g, st.P)
    R3 = tuple((v - vp) / dt + a - u + q
               for v, vp, a, u, q in zip(V, vprev, adv, U, gp))
    R4 = ops.div(g, U)
    kmask = (pb.t0 + np.arange(N) < pb.N_global - 1).astype(np.float64)
    kmask = kmask.reshape((N,) + (1,) * g.dim)
    if pb.unext is not None:
        unext = tuple(np.concatenate([u[1:], h[None]], axis=0) for u, h in zip(U, pb.unext))
    else:
        unext = tuple(np.concatenate([u[1:], np.zeros_like(u[:1])], axis=0) for u in U)
    if pb.vstar[0].shape[0] == N + 1:
        vs_next = tuple(s[1:] for s in pb.vstar)
    else:
        vs_next = tuple(np.concatenate([s[1:], np.zeros_like(s[:1])], axis=0)
                        for s in pb.vstar)
    jt = ops.jac_T_apply(g, V, U)
    gpb = ops.grad(g, st.PB)
    R1 = tuple(kmask * (pb.kr * (v - s) - un / dt) + u / dt + j + q
               for v, s, un, u, j, q in zip(V, vs_next, unext, U, jt, gpb))
    R2 = ops.div(g, V)
    return Residual(_mask(g, R1), R2, _mask(g, R3), R4)


# ---------------------------------------------------------------------------
# local (per-cell) structure
# ---------------------------------------------------------------------------


def color_of(g, mod=2, red_black=False):
    """Colour id per cell: red-black (sum_k c_k) mod 2, else sum_k (c_k mod m) m^k."""
    idx = np.indices(g.res)
    if red_black:
        return np.sum(idx, axis=0) % 2
    col = np.zeros(g.res, dtype=np.int64)
    mul = 1
    for k in range(g.dim):
        col += (idx[k] % mod) * mul
        mul *= mod
    return col


def n_colors(g, mod=2, red_black=False):
    return 2 if red_black else mod ** g.dim


def colourable(g, mod=2, red_black=False):
    """Same-colour cells must not share a face: red-black needs
    an even last-axis extent (equal colour rows) and, periodic, even extents
    (the wrap neighbour has the other parity); mod-m colouring of a periodic
    grid needs every extent divisible by m."""
    if red_black:
        return g.res[-1] % 2 == 0 and (not g.periodic or all(r % 2 == 0 for r in g.res))
    return not g.periodic or all(r % mod == 0 for r in g.res)


class CellSlots:
    """Face slots of a set of cells: slot q = 2k + s (s=0 low, 1 high)."""

    def __init__(self, g, cells):
        self.g = g
        self.cells = cells                      # (M, dim) int
        M = cells.shape[0]
        d = g.dim
        self.M = M
        self.face_idx = []                      # per slot: tuple of index arrays
        self.wall = np.zeros((M, 2 * d), dtype=bool)
        self.gcol = np.zeros((M, 2 * d))         # d(grad p)_face / d p_cell
        for k in range(d):
            for s in (0, 1):
                q = 2 * k + s
                fi = cells.copy()
                fi[:, k] = cells[:, k] + s
                if g.periodic:
                    fi[:, k] %= g.res[k]
                    w = np.zeros(M, dtype=bool)
                else:
                    w = (cells[:, k] == 0) if s == 0 else (cells[:, k] == g.res[k] - 1)
                self.face_idx.append((k, tuple(fi[:, a] for a in range(d))))
                self.wall[:, q] = w
                self.gcol[:, q] = np.where(w, 0.0, (1.0 if s == 0 else -1.0) / g.h)
        self.cell_idx = tuple(cells[:, a] for a in range(d))

    def gather_faces(self, comps):
        """comps: tuple of (N, face) -> (M, N, 2d)."""
        out = []
        for k, fi in self.face_idx:
            a = comps[k]
            out.append(np.moveaxis(a[(slice(None),) + fi], 0, 1))
        return np.stack(out, axis=-1) * (~self.wall)[:, None, :]

    def gather_cells(self, arr):
        """(N, res) -> (M, N)."""
        return np.moveaxis(arr[(slice(None),) + self.cell_idx], 0, 1)

    def scatter_add_faces(self, comps, vals):
        """vals (M, N, 2d); adds into comps (in place); walls skipped."""
        for q, (k, fi) in enumerate(self.face_idx):
            keep = ~self.wall[:, q]
            sel = tuple(f[keep] for f in fi)
            comps[k][(slice(None),) + sel] += vals[keep, :, q].T

    def scatter_add_cells(self, arr, vals):
        arr[(slice(None),) + self.cell_idx] += vals.T


def local_jacobian(pb, V, slots, probe_mod=4):
    """J_loc[m, i, q_row, q_col] = d Adv(V[i])_{face q_row} / d V[i]_{face q_col}
    for every cell of ``slots``, by unit-vector probing of ``ops.jac_apply`` on
    classes of cells spaced >= 4 apart (no cross-talk: the Jacobian stencil has
    reach 1 face)."""
    g = pb.g
    d = g.dim
    cells = slots.cells
    M, N = slots.M, V[0].shape[0]
    J = np.zeros((M, N, 2 * d, 2 * d))
    cls = np.zeros(M, dtype=np.int64)
    mul = 1
    for k in range(d):
        cls += (cells[:, k] % probe_mod) * mul
        mul *= probe_mod
    for c in np.unique(cls):
        sel = np.nonzero(cls == c)[0]
        for qc, (kc, fi) in enumerate(slots.face_idx):
            E = [np.zeros(g.face_shape(k)) for k in range(d)]
            keep = sel[~slots.wall[sel, qc]]
            if keep.size == 0:
                continue
            E[kc][tuple(f[keep] for f in fi)] = 1.0
            col = ops.jac_apply(g, V, tuple(E))       # (N, face) per comp
            for qr, (kr, fr) in enumerate(slots.face_idx):
                J[keep, :, qr, qc] = col[kr][(slice(None),) + tuple(f[keep] for f in fr)].T
    # wall rows / cols are not unknowns
    wr = slots.wall[:, None, :, None] | slots.wall[:, None, None, :]
    J[np.broadcast_to(wr, J.shape)] = 0.0
    return J


def assemble_line(pb, slots, J):
    """Block-tridiagonal Eq. 9 (Gauss-Newton) system of every cell's time line.

    Returns (D, L, Up) of shapes (M, 2N, b, b): diagonal, lower (couples
    block b to b-1) and upper (couples b to b+1); b = 2d+1."""
    g = pb.g
    d = g.dim
    nf = 2 * d
    b = nf + 1
    M, N = slots.M, pb.N
    dt = pb.dt
    wall = slots.wall
    eye = np.broadcast_to(np.eye(nf), (M, nf, nf)) * (~wall)[:, None, :] * (~wall)[:, :, None]
    D = np.zeros((M, 2 * N, b, b))
    L = np.zeros((M, 2 * N, b, b))
    Up = np.zeros((M, 2 * N, b, b))
    gc = slots.gcol                       # (M, nf)
    for i in range(N):
        bu, bv = 2 * i, 2 * i + 1
        # u-block: rows R3[i] (faces) + R4[i] (cell); unknowns u_i, p_{i+1}
        D[:, bu, :nf, :nf] = -eye
        D[:, bu, :nf, nf] = gc
        D[:, bu, nf, :nf] = -gc           # div row = -grad^T
        # v-block: rows R1[i] + R2[i]; unknowns v_{i+1}, pbar_{i+1}
        alpha = pb.kr if pb.t0 + i < pb.N_global - 1 else 0.0
        D[:, bv, :nf, :nf] = alpha * eye
        D[:, bv, :nf, nf] = gc
        D[:, bv, nf, :nf] = -gc
        Ji = J[:, i]
        Up[:, bu, :nf, :nf] = eye / dt + Ji
        L[:, bv, :nf, :nf] = eye / dt + np.swapaxes(Ji, 1, 2)
        if i + 1 < N:
            Up[:, bv, :nf, :nf] = -eye / dt
            L[:, bv + 1, :nf, :nf] = -eye / dt
    # wall slots: decoupled identity rows so every block stays regular
    for q in range(nf):
        w = wall[:, q]
        if np.any(w):
            D[w, :, q, q] = 1.0
    return D, L, Up


def block_thomas(D, L, Up, y):
    """Solve the block-tridiagonal systems (batched over the leading axis)."""
    M, nb, b, _ = D.shape
    W = np.zeros((M, nb, b, b))
    z = np.zeros((M, nb, b))
    S = D[:, 0]
    rhs = y[:, 0]
    for k in range(nb):
        if k > 0:
            S = D[:, k] - L[:, k] @ W[:, k - 1]
            rhs = y[:, k] - np.einsum("mij,mj->mi", L[:, k], z[:, k - 1])
        sol = np.linalg.solve(S, np.concatenate([Up[:, k], rhs[:, :, None]], axis=2))
        W[:, k] = sol[:, :, :b]
        z[:, k] = sol[:, :, b]
    x = np.zeros((M, nb, b))
    x[:, nb - 1] = z[:, nb - 1]
    for k in range(nb - 2, -1, -1):
        x[:, k] = z[:, k] - np.einsum("mij,mj->mi", W[:, k], x[:, k + 1])
    return x


def _local_rhs(slots, res, rhs, N, nf):
    """-(f - rhs) gathered into (M, 2N, b)."""
    full = res if rhs is None else res.sub(rhs)
    M = slots.M
    y = np.zeros((M, 2 * N, nf + 1))
    y[:, 0::2, :nf] = -slots.gather_faces(full.R3)
    y[:, 0::2, nf] = -slots.gather_cells(full.R4)
    y[:, 1::2, :nf] = -slots.gather_faces(full.R1)
    y[:, 1::2, nf] = -slots.gather_cells(full.R2)
    return y


def scgs_color(pb, st, rhs, color, cells=None, return_delta=False):
    """One colour pass (snapshot reads, in-colour Jacobi); returns new State."""
    g = pb.g
    if cells is None:
        col = color_of(g, pb.colors, pb.red_black)
        cells = np.argwhere(col == color)
    slots = CellSlots(g, cells)
    N, nf = pb.N, 2 * g.dim
    res = kkt_residual(pb, st)
    y = _local_rhs(slots, res, rhs, N, nf)
    J = local_jacobian(pb, st.V, slots)
    D, L, Up = assemble_line(pb, slots, J)
    x = block_thomas(D, L, Up, y)
    out = st.copy()
    w = pb.omega
    slots.scatter_add_faces(out.U, w * x[:, 0::2, :nf])
    slots.scatter_add_cells(out.P, w * x[:, 0::2, nf])
    slots.scatter_add_faces(out.V, w * x[:, 1::2, :nf])
    slots.scatter_add_cells(out.PB, w * x[:, 1::2, nf])
    if return_delta:
        return out, x
    return out


def scgs_smooth(pb, st, rhs=None):
    """One full sweep over all colours."""
    for c in range(n_colors(pb.g, pb.colors, pb.red_black)):
        st = scgs_color(pb, st, rhs, c)
    return st


# ---------------------------------------------------------------------------
# transfers and FAS V-cycle (Alg. 2)
# ---------------------------------------------------------------------------


def restrict_state(g, st):
    return State(ops.restrict_face(g, st.V), ops.restrict_cell(g, st.PB),
                 ops.restrict_face(g, st.U), ops.restrict_cell(g, st.P))


def prolong_state(gc, st):
    return State(ops.prolong_face(gc, st.V), ops.prolong_cell(gc, st.PB),
                 ops.prolong_face(gc, st.U), ops.prolong_cell(gc, st.P))


def restrict_residual(g, r):
    return Residual(ops.restrict_face(g, r.R1), ops.restrict_cell(g, r.R2),
                    ops.restrict_face(g, r.R3), ops.restrict_cell(g, r.R4))


def build_levels(pb, n_levels):
    """Per-level problems: v* and v0 restricted by the face restriction."""
    levels = [pb]
    while len(levels) < n_levels:
        top = levels[-1]
        gc = top.g.coarsen()
        if gc is None or not colourable(gc, top.colors, top.red_black):
            break
        levels.append(Problem(gc, top.dt, top.K, top.r,
                              ops.restrict_face(top.g, top.v0),
                              ops.restrict_face(top.g, top.vstar),
                              top.omega, top.colors, top.red_black))
    return levels


def vcycle(levels, li, st, rhs=None, nu1=2, nu2=2, n_coarse=10):
    """FAS V(2,2) with 10 coarsest smoothings (PAPER Alg. 2)."""
    pb = levels[li]
    if li == len(levels) - 1:
        for _ in range(n_coarse):
            st = scgs_smooth(pb, st, rhs)
        return st
    for _ in range(nu1):
        st = scgs_smooth(pb, st, rhs)
    g = pb.g
    pc = levels[li + 1]
    sc0 = restrict_state(g, st)
    ff = kkt_residual(pb, st)
    rh = ff.sub(ff) if rhs is None else rhs
    rc = kkt_residual(pc, sc0).add(restrict_residual(g, rh.sub(ff)))
    sc = vcycle(levels, li + 1, sc0.copy(), rc, nu1, nu2, n_coarse)
    corr = prolong_state(pc.g, sc.axpy(-1.0, sc0))
    st = st.axpy(1.0, corr)
    for _ in range(nu2):
        st = scgs_smooth(pb, st, rhs)
    return st


def gauge_fix(st):
    """Subtract per-frame means of p and pbar."""
    ax = tuple(range(1, st.P.ndim))
    return State(st.V, st.PB - st.PB.mean(axis=ax, keepdims=True),
                 st.U, st.P - st.P.mean(axis=ax, keepdims=True))


@dataclass
class NsoResult:
    state: State
    history: list = field(default_factory=list)   # (cycle, res_inf, res_l2)
    converged: bool = False


def solve_nso(pb, st=None, eps=1e-5, cycle_budget=50, n_levels=None,
              relative=False):
    """Repeat V-cycles until ||f||_inf <= eps."""
    levels = build_levels(pb, n_levels if n_levels else 99)
    if st is None:
        st = zero_state(pb.g, pb.N)
    r0 = kkt_residual(pb, st)
    hist = [(0, r0.inf(), r0.l2())]
    tol = eps * r0.inf() if relative else eps
    if hist[0][1] <= tol:
        return NsoResult(st, hist, True)
    for c in range(1, cycle_budget + 1):
        st = gauge_fix(vcycle(levels, 0, st))
        r = kkt_residual(pb, st)
        hist.append((c, r.inf(), r.l2()))
        if r.inf() <= tol:
            return NsoResult(st, hist, True)
    return NsoResult(st, hist, False)


LM_WINDOW, LM_STALL, LM_MIN_SHIFT, LM_MAX_SHIFT = 3, 0.95, 1e-3, 1e3


def solve_nso_lm(pb, st=None, eps=1e-5, cycle_budget=50, n_levels=None, stall=LM_STALL):
    """SPEC.md:347 LM safeguard as frozen in DESIGN §11 (proximal shift):
    the per-cycle reduction factor over the last 3 cycles is tested only
    once 3 cycles have run since the last change of sigma; if it exceeds 0.95
    the K/r blocks get a shift sigma (K, then doubled, capped at 1e3 K), while
    progressing it is halved and dropped below 1e-3 K.  A shifted V-cycle
    solves the problem with K + sigma and guide (K v* + sigma v^k)/(K + sigma).
    The stop test uses the undamped residual."""
    import dataclasses
    levels = build_levels(pb, n_levels if n_levels else 99)
    if st is None:
        st = zero_state(pb.g, pb.N)
    N = pb.N
    r = kkt_residual(pb, st)
    hist = [(0, r.inf(), r.l2())]
    if hist[0][1] <= eps:
        return NsoResult(st, hist, True)
    sigma, changed = 0.0, 0
    for c in range(1, cycle_budget + 1):
        if sigma > 0:
            K2 = pb.K + sigma
            guide = []
            for k in range(pb.g.dim):
                gk = pb.vstar[k].copy()
                gk[1:] = (pb.K / K2) * pb.vstar[k][1:] + (sigma / K2) * st.V[k][:N - 1]
                guide.append(gk)
            pd = dataclasses.replace(pb, K=K2, vstar=tuple(guide))
            st = gauge_fix(vcycle(build_levels(pd, n_levels if n_levels else 99), 0, st))
        else:
            st = gauge_fix(vcycle(levels, 0, st))
        r = kkt_residual(pb, st)
        hist.append((c, r.inf(), r.l2()))
        if r.inf() <= eps:
            return NsoResult(st, hist, True)
        if c - changed >= LM_WINDOW:
            prev = hist[c - LM_WINDOW][1]
            factor = (r.inf() / prev) ** (1.0 / LM_WINDOW) if prev > 0 else 0.0
            new = sigma
            if factor > stall:
                new = pb.K if sigma == 0 else min(2.0 * sigma, LM_MAX_SHIFT * pb.K)
            elif sigma > 0:
                new = 0.5 * sigma
                if new < LM_MIN_SHIFT * pb.K:
                    new = 0.0
            if new != sigma:
                sigma, changed = new, c
    return NsoResult(st, hist, False)
