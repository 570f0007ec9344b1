"""Dense Newton solve of the Eq. 8 KKT system on tiny grids (TEST INFRASTRUCTURE ONLY).

Known-answer oracle of ``SPEC.md:315`` / ``:526``: assemble F(x) = Eq. 8
residual over all non-wall unknowns, build its Jacobian column by column
(F is at most quadratic, so a central difference with unit step is exact up
to rounding), and run Newton with minimum-norm steps (the Jacobian has the
2N-dimensional per-frame pressure-constant nullspace).
"""

import numpy as np

from . import stfas


class Packer:
    """Flatten / unflatten the non-wall unknowns of a State."""

    def __init__(self, pb):
        self.pb = pb
        g, N = pb.g, pb.N
        self.face_masks = []
        for k in range(g.dim):
            m = np.ones((N,) + g.face_shape(k), dtype=bool)
            if not g.periodic:
                idx = [slice(None)] * m.ndim
                idx[1 + k] = 0
                m[tuple(idx)] = False
                idx[1 + k] = -1
                m[tuple(idx)] = False
            self.face_masks.append(m)
        self.nf = sum(int(m.sum()) for m in self.face_masks)
        self.nc = N * g.n_cells
        self.n = 2 * self.nf + 2 * self.nc

    def _faces(self, comps):
        return np.concatenate([c[m] for c, m in zip(comps, self.face_masks)])

    def pack_state(self, st):
        return np.concatenate([self._faces(st.V), st.PB.reshape(-1), self._faces(st.U), st.P.reshape(-1)])

    def pack_res(self, r):
        return np.concatenate([self._faces(r.R1), r.R2.reshape(-1), self._faces(r.R3), r.R4.reshape(-1)])

    def _unfaces(self, x):
        out, o = [], 0
        for m in self.face_masks:
            a = np.zeros(m.shape)
            k = int(m.sum())
            a[m] = x[o:o + k]
            out.append(a)
            o += k
        return tuple(out)

    def unpack_state(self, x):
        g, N = self.pb.g, self.pb.N
        nf, nc = self.nf, self.nc
        V = self._unfaces(x[:nf])
        PB = x[nf:nf + nc].reshape((N,) + g.res)
        U = self._unfaces(x[nf + nc:2 * nf + nc])
        P = x[2 * nf + nc:].reshape((N,) + g.res)
        return stfas.State(V, PB.copy(), U, P.copy())


def residual_vec(pb, pk, x):
    return pk.pack_res(stfas.kkt_residual(pb, pk.unpack_state(x)))


def jacobian(pb, pk, x, step=1.0):
    n = pk.n
    J = np.zeros((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = step
        J[:, j] = (residual_vec(pb, pk, x + e) - residual_vec(pb, pk, x - e)) / (2 * step)
        e[j] = 0.0
    return J


def newton(pb, x0=None, tol=1e-13, iters=30):
    """Returns (State, ||F||_inf history)."""
    pk = Packer(pb)
    x = np.zeros(pk.n) if x0 is None else x0.copy()
    hist = []
    for _ in range(iters):
        F = residual_vec(pb, pk, x)
        hist.append(float(np.max(np.abs(F))))
        if hist[-1] <= tol:
            break
        J = jacobian(pb, pk, x)
        dx = np.linalg.lstsq(J, -F, rcond=1e-12)[0]
        x = x + dx
    return pk.unpack_state(x), hist
