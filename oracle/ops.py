"""fp64 numpy restatement of the reference raw kernels (TEST INFRASTRUCTURE ONLY).

Every function takes arrays with an optional batch prefix; the trailing
``grid.dim`` axes are spatial (``fields.py:17-19``).  Face fields are tuples of
per-axis component arrays.  Functions cite the reference lines they restate.
"""

from functools import lru_cache

import numpy as np

# ---------------------------------------------------------------------------
# index helpers
# ---------------------------------------------------------------------------


def _axis(g, k):
    """Negative array axis of grid axis k (works with any batch prefix)."""
    return k - g.dim


def _take(a, ax, start, stop):
    idx = [slice(None)] * a.ndim
    idx[ax] = slice(start, stop)
    return a[tuple(idx)]


def _pad(a, ax, lo, hi):
    w = [(0, 0)] * a.ndim
    w[ax] = (lo, hi)
    return np.pad(a, w)


def nbr(g, a, k, s):
    """Value of ``a`` at index ``i + s`` along grid axis k (zero outside for
    Neumann, wrapped for periodic).  Same semantics as ``advection.py:43-59``
    ``_shift(spec, a, k, -s)``."""
    ax = _axis(g, k)
    if g.periodic:
        return np.roll(a, -s, axis=ax)
    n = a.shape[ax]
    if s > 0:
        return _pad(_take(a, ax, s, n), ax, 0, s)
    if s < 0:
        return _pad(_take(a, ax, 0, n + s), ax, -s, 0)
    return a.copy()


def wall_mask(g, a, k):
    """Zero the two wall layers of a k-face array (``advection.py:62-73``)."""
    a = np.array(a, dtype=np.float64, copy=True)
    if g.periodic:
        return a
    ax = _axis(g, k)
    idx = [slice(None)] * a.ndim
    idx[ax] = 0
    a[tuple(idx)] = 0.0
    idx[ax] = a.shape[ax] - 1
    a[tuple(idx)] = 0.0
    return a


def zero_walls(g, comps):
    """``fields.py:145-160``."""
    return tuple(wall_mask(g, c, k) for k, c in enumerate(comps))


def face_pair(g, vk, k):
    """(v at c+e_k/2, v at c-e_k/2) on the cell lattice (``advection.py:76-85``)."""
    ax = _axis(g, k)
    if g.periodic:
        return np.roll(vk, -1, axis=ax), vk
    n = vk.shape[ax]
    return _take(vk, ax, 1, n), _take(vk, ax, 0, n - 1)


# ---------------------------------------------------------------------------
# field core (fields.py)
# ---------------------------------------------------------------------------


def div(g, comps):
    """(1/h) sum_k (v_k[c+e_k] - v_k[c])  (``fields.py:163-178``)."""
    out = 0.0
    for k, c in enumerate(comps):
        hi, lo = face_pair(g, c, k)
        out = out + (hi - lo) / g.h
    return out


def grad(g, p):
    """(p[f] - p[f-e_k]) / h on faces; Neumann walls 0 (``fields.py:181-201``)."""
    comps = []
    for k in range(g.dim):
        ax = _axis(g, k)
        if g.periodic:
            comps.append((p - np.roll(p, 1, axis=ax)) / g.h)
        else:
            n = p.shape[ax]
            inner = (_take(p, ax, 1, n) - _take(p, ax, 0, n - 1)) / g.h
            comps.append(_pad(inner, ax, 1, 1))
    return tuple(comps)


def dot(a, b):
    """Plain (unweighted) inner product (``fields.py:204-207``)."""
    return float(sum(np.vdot(x, y) for x, y in zip(a, b)))


def inf_norm(arrs):
    """``fields.py:210-216``."""
    if isinstance(arrs, np.ndarray):
        arrs = (arrs,)
    m = 0.0
    for a in arrs:
        if a.size:
            m = max(m, float(np.max(np.abs(a))))
    return m


def laplacian(g, p):
    """div(grad p) (``fields.py:223-225``)."""
    return div(g, grad(g, p))


def lap_diag(g):
    """``fields.py:228-240``."""
    h2 = g.h * g.h
    d = np.full(g.res, -2.0 * g.dim / h2)
    if not g.periodic:
        for k in range(g.dim):
            idx = [slice(None)] * g.dim
            idx[k] = 0
            d[tuple(idx)] += 1.0 / h2
            idx[k] = g.res[k] - 1
            d[tuple(idx)] += 1.0 / h2
    return d


def restrict_cell(g_fine, x):
    """2^d box average (``fields.py:243-253``)."""
    for k in range(g_fine.dim):
        ax = _axis(g_fine, k)
        n = x.shape[ax]
        idx0 = [slice(None)] * x.ndim
        idx1 = [slice(None)] * x.ndim
        idx0[ax] = slice(0, n, 2)
        idx1[ax] = slice(1, n, 2)
        x = 0.5 * (x[tuple(idx0)] + x[tuple(idx1)])
    return x


def _prolong_cell_axis(g_coarse, x, k):
    """(3/4, 1/4) interpolation along one axis, wrap / clamp (``fields.py:256-284``)."""
    ax = _axis(g_coarse, k)
    n = x.shape[ax]
    if g_coarse.periodic:
        lo = np.roll(x, 1, axis=ax)
        hi = np.roll(x, -1, axis=ax)
    else:
        i = np.arange(n)
        lo = np.take(x, np.maximum(i - 1, 0), axis=ax)
        hi = np.take(x, np.minimum(i + 1, n - 1), axis=ax)
    even = 0.75 * x + 0.25 * lo
    odd = 0.75 * x + 0.25 * hi
    shape = list(x.shape)
    shape[ax] = 2 * n
    out = np.empty(shape)
    idx = [slice(None)] * x.ndim
    idx[ax] = slice(0, 2 * n, 2)
    out[tuple(idx)] = even
    idx[ax] = slice(1, 2 * n, 2)
    out[tuple(idx)] = odd
    return out


def prolong_cell(g_coarse, x):
    for k in range(g_coarse.dim):
        x = _prolong_cell_axis(g_coarse, x, k)
    return x


# ----- face transfers (STFAS R/P) -----


def restrict_face(g_fine, comps):
    """Coarse k-face = mean of the 2^(d-1) coincident fine k-faces."""
    out = []
    for k, c in enumerate(comps):
        for a in range(g_fine.dim):
            ax = _axis(g_fine, a)
            n = c.shape[ax]
            idx0 = [slice(None)] * c.ndim
            if a == k:
                idx0[ax] = slice(0, n, 2)
                c = c[tuple(idx0)]
            else:
                idx1 = [slice(None)] * c.ndim
                idx0[ax] = slice(0, n, 2)
                idx1[ax] = slice(1, n, 2)
                c = 0.5 * (c[tuple(idx0)] + c[tuple(idx1)])
        out.append(c)
    return tuple(out)


def prolong_face(g_coarse, comps):
    """Linear along the face normal, (3/4,1/4) across it; preserves constants."""
    out = []
    for k, c in enumerate(comps):
        for a in range(g_coarse.dim):
            if a != k:
                c = _prolong_cell_axis(g_coarse, c, a)
                continue
            ax = _axis(g_coarse, a)
            n = c.shape[ax]
            if g_coarse.periodic:
                nxt = np.roll(c, -1, axis=ax)
                m = n
            else:
                nxt = _take(c, ax, 1, n)
                m = n - 1
            mid = 0.5 * (_take(c, ax, 0, m) + nxt)
            shape = list(c.shape)
            shape[ax] = 2 * n if g_coarse.periodic else 2 * n - 1
            f = np.empty(shape)
            idx = [slice(None)] * c.ndim
            idx[ax] = slice(0, shape[ax], 2)
            f[tuple(idx)] = c
            idx[ax] = slice(1, shape[ax], 2)
            f[tuple(idx)] = mid
            c = f
        out.append(c)
    return tuple(out)


# ----- Poisson multigrid + projection (fields.py:287-358) -----


class PoissonLevels:
    """Hierarchy down to the coarsest size with a dense pinv (``fields.py:287-304``)."""

    def __init__(self, g):
        self.grids = [g]
        while self.grids[-1].coarsen() is not None:
            self.grids.append(self.grids[-1].coarsen())
        gc = self.grids[-1]
        n = gc.n_cells
        a = np.zeros((n, n))
        e = np.zeros(n)
        for j in range(n):
            e[j] = 1.0
            a[:, j] = laplacian(gc, e.reshape(gc.res)).reshape(-1)
            e[j] = 0.0
        self.coarse_pinv = np.linalg.pinv(a, rcond=1e-12)
        self.diags = [lap_diag(q) for q in self.grids]


@lru_cache(maxsize=32)
def poisson_levels(g):
    return PoissonLevels(g)


def poisson_vcycle(lv, li, p, rhs, nu=2, omega=0.8):
    """Correction-scheme V(2,2), damped Jacobi (``fields.py:312-327``)."""
    g = lv.grids[li]
    if li == len(lv.grids) - 1:
        return (lv.coarse_pinv @ rhs.reshape(-1)).reshape(g.res)
    d = lv.diags[li]
    for _ in range(nu):
        p = p + omega * (rhs - laplacian(g, p)) / d
    rc = restrict_cell(g, rhs - laplacian(g, p))
    pc = poisson_vcycle(lv, li + 1, np.zeros(lv.grids[li + 1].res), rc, nu, omega)
    p = p + prolong_cell(lv.grids[li + 1], pc)
    for _ in range(nu):
        p = p + omega * (rhs - laplacian(g, p)) / d
    return p


class PoissonNonConvergence(Exception):
    def __init__(self, residual):
        super().__init__("Poisson V-cycle budget exhausted")
        self.residual = residual


def solve_poisson(g, rhs, tol, max_cycles=200, return_cycles=False):
    """``fields.py:330-347``."""
    rhs = rhs - rhs.mean()
    if inf_norm(rhs) <= tol:
        z = np.zeros(g.res)
        return (z, 0) if return_cycles else z
    lv = poisson_levels(g)
    p = np.zeros(g.res)
    r = np.inf
    for it in range(max_cycles):
        p = poisson_vcycle(lv, 0, p, rhs)
        r = inf_norm(rhs - laplacian(g, p))
        if r <= tol:
            return (p, it + 1) if return_cycles else p
    raise PoissonNonConvergence(r)


def project(g, comps, tol):
    """Solenoidal projection Q (``fields.py:350-358``)."""
    comps = zero_walls(g, comps)
    dv = div(g, comps)
    if inf_norm(dv) <= tol:
        return comps
    phi = solve_poisson(g, dv, tol)
    gp = grad(g, phi)
    return tuple(c - q for c, q in zip(comps, gp))


# ---------------------------------------------------------------------------
# transport (advection.py)
# ---------------------------------------------------------------------------


def transport_scalar(g, v, rho):
    """(T(v) rho)_c = -(1/2h) sum_k [v_k+ rho(c+e_k) - v_k- rho(c-e_k)]
    (``advection.py:88-97``)."""
    c0 = 0.5 / g.h
    out = np.zeros(rho.shape)
    for k in range(g.dim):
        vp, vm = face_pair(g, v[k], k)
        out -= c0 * (vp * nbr(g, rho, k, 1) - vm * nbr(g, rho, k, -1))
    return out


def scalar_stencil_v_adjoint(g, x, y):
    """Face g = -(1/2h)(y_L x_R - y_R x_L) (``advection.py:105-130``)."""
    c0 = 0.5 / g.h
    out = []
    for k in range(g.dim):
        ax = _axis(g, k)
        if g.periodic:
            xl = np.roll(x, 1, axis=ax)
            yl = np.roll(y, 1, axis=ax)
            out.append(-c0 * (yl * x - y * xl))
        else:
            n = x.shape[ax]
            xl, xr = _take(x, ax, 0, n - 1), _take(x, ax, 1, n)
            yl, yr = _take(y, ax, 0, n - 1), _take(y, ax, 1, n)
            out.append(_pad(-c0 * (yl * xr - yr * xl), ax, 1, 1))
    return tuple(out)


class TaylorOverflow(Exception):
    def __init__(self, k_cap, last):
        super().__init__("Taylor term cap exceeded")
        self.k_cap = k_cap
        self.last_term_norm = last


def taylor(g, v, rho, dt, tol=1e-5, cap=128, k_fixed=None, transpose=False):
    """Truncated exp(T dt) rho, adaptive order (``advection.py:144-174``).

    Returns (out, k_used, last_term_norm)."""
    sgn = -1.0 if transpose else 1.0
    out = np.array(rho, dtype=np.float64, copy=True)
    term = out
    k = 0
    while True:
        k += 1
        if k > cap:
            raise TaylorOverflow(cap, inf_norm(term))
        term = (dt / k) * (sgn * transport_scalar(g, v, term))
        out = out + term
        nrm = inf_norm(term)
        if k_fixed is not None:
            if k == k_fixed:
                return out, k, nrm
        elif nrm < tol:
            return out, k, nrm


def advect_v_T(g, v, rho, mu, dt, k):
    """v-transpose Jacobian of the truncated series (``advection.py:177-210``)."""
    xs = [np.array(rho, dtype=np.float64)]
    ys = [np.array(mu, dtype=np.float64)]
    for _ in range(k - 1):
        xs.append(transport_scalar(g, v, xs[-1]))
        ys.append(-transport_scalar(g, v, ys[-1]))
    out = None
    coeff = 1.0
    for t in range(k):
        coeff = coeff * dt / (t + 1)
        acc = None
        for s in range(t + 1):
            q = scalar_stencil_v_adjoint(g, xs[s], ys[t - s])
            acc = q if acc is None else tuple(a + b for a, b in zip(acc, q))
        term = tuple(coeff * a for a in acc)
        out = term if out is None else tuple(a + b for a, b in zip(out, term))
    return out


# ----- velocity self-advection (advection.py:306-441) -----


def adv_samples(g, a, j, k):
    """Advecting component k sampled at the j-face lattice +/- e_k/2
    (``advection.py:306-350``).  Returns (plus, minus)."""
    if k == j:
        # centre averages of a_j, then the cell above / below each j-face
        hi, lo = face_pair(g, a[j], j)
        cc = 0.5 * (lo + hi)
        ax = _axis(g, j)
        if g.periodic:
            return cc, np.roll(cc, 1, axis=ax)
        return _pad(cc, ax, 0, 1), _pad(cc, ax, 1, 0)
    ak = a[k]
    axj, axk = _axis(g, j), _axis(g, k)
    if g.periodic:
        corner = 0.5 * (ak + np.roll(ak, 1, axis=axj))
        return np.roll(corner, -1, axis=axk), corner
    # corner[f_j] = 1/2 (a_k[f_j-1] + a_k[f_j]) with zero padding along j
    akp = _pad(ak, axj, 1, 1)
    nj = akp.shape[axj]
    corner = 0.5 * (_take(akp, axj, 0, nj - 1) + _take(akp, axj, 1, nj))
    nk = corner.shape[axk]
    return _take(corner, axk, 1, nk), _take(corner, axk, 0, nk - 1)


def transport_face(g, a, w):
    """S(a, w)_j = (1/2h) sum_k (A+ w_j[f+e_k] - A- w_j[f-e_k]), wall-masked
    (``advection.py:353-365``)."""
    c0 = 0.5 / g.h
    out = []
    for j in range(g.dim):
        acc = 0.0
        for k in range(g.dim):
            sp, sm = adv_samples(g, a, j, k)
            acc = acc + c0 * (sp * nbr(g, w[j], k, 1) - sm * nbr(g, w[j], k, -1))
        out.append(wall_mask(g, acc, j))
    return tuple(out)


def self_advection(g, v):
    return transport_face(g, v, v)


def jac_apply(g, v, d):
    """J_Adv(v) d = S(v, d) + S(d, v) (``advection.py:373-377``)."""
    return tuple(x + y for x, y in zip(transport_face(g, v, d),
                                       transport_face(g, d, v)))


def _samples_adjoint(g, v, u):
    """Adjoint of d -> S(d, v) tested against u (``advection.py:380-434``)."""
    c0 = 0.5 / g.h
    out = [np.zeros(vk.shape) for vk in v]
    for j in range(g.dim):
        vj, uj = v[j], u[j]
        for k in range(g.dim):
            axk = _axis(g, k)
            if k == j:
                if g.periodic:
                    gam = c0 * (uj * np.roll(vj, -1, axis=axk)
                                - np.roll(uj, -1, axis=axk) * vj)
                    out[j] += 0.5 * (gam + np.roll(gam, 1, axis=axk))
                else:
                    n = vj.shape[axk]
                    gam = c0 * (_take(uj, axk, 0, n - 1) * _take(vj, axk, 1, n)
                                - _take(uj, axk, 1, n) * _take(vj, axk, 0, n - 1))
                    out[j] += 0.5 * (_pad(gam, axk, 0, 1) + _pad(gam, axk, 1, 0))
                continue
            axj = _axis(g, j)
            if g.periodic:
                gam = c0 * (np.roll(uj, 1, axis=axk) * vj
                            - uj * np.roll(vj, 1, axis=axk))
                out[k] += 0.5 * (gam + np.roll(gam, -1, axis=axj))
            else:
                n = vj.shape[axk]
                inner = c0 * (_take(uj, axk, 0, n - 1) * _take(vj, axk, 1, n)
                              - _take(uj, axk, 1, n) * _take(vj, axk, 0, n - 1))
                gam = _pad(inner, axk, 1, 1)
                nj = gam.shape[axj]
                out[k] += 0.5 * (_take(gam, axj, 0, nj - 1) + _take(gam, axj, 1, nj))
    return tuple(wall_mask(g, o, k) for k, o in enumerate(out))


def jac_T_apply(g, v, u):
    """J_Adv(v)^T u = T(v, u) - S(v, u) (``advection.py:437-441``)."""
    a = transport_face(g, v, u)
    b = _samples_adjoint(g, v, u)
    return tuple(y - x for x, y in zip(a, b))


# ---------------------------------------------------------------------------
# semi-Lagrangian comparator (advection.py:255-299)
# ---------------------------------------------------------------------------


def semi_lagrangian(g, v, rho, dt):
    v = zero_walls(g, v)
    vel = []
    for k in range(g.dim):
        hi, lo = face_pair(g, v[k], k)
        vel.append(0.5 * (hi + lo))
    coords = np.meshgrid(*[np.arange(n) + 0.5 for n in g.res], indexing="ij")
    samples = [c - dt * u / g.h for c, u in zip(coords, vel)]
    i0, fr = [], []
    for s in samples:
        q = s - 0.5
        b = np.floor(q).astype(np.int64)
        i0.append(b)
        fr.append(q - b)
    out = np.zeros_like(rho)
    for corner in range(1 << g.dim):
        w = np.ones_like(rho)
        idx = []
        for k in range(g.dim):
            bit = (corner >> k) & 1
            ik = i0[k] + bit
            n = g.res[k]
            ik = np.mod(ik, n) if g.periodic else np.clip(ik, 0, n - 1)
            idx.append(ik)
            w = w * (fr[k] if bit else 1.0 - fr[k])
        out += w * rho[tuple(idx)]
    return out
