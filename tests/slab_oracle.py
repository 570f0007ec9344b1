"""Oracle (numpy) engine for the time-slab orchestrator -- CPU tests only."""

import numpy as np

from oracle import ops, stfas


class OracleEngine:
    def __init__(self, g, dt, K, r, t0, t1, n_total, n_levels, omega=0.8, colors=2, red_black=True):
        self.grids = [gg for gg in g.hierarchy(n_levels)]
        keep = [self.grids[0]]
        for gg in self.grids[1:]:
            if not stfas.colourable(gg, colors, red_black):
                break
            keep.append(gg)
        self.grids = keep
        self.n_levels = len(self.grids)
        self.dt, self.K, self.r, self.omega, self.colors = dt, K, r, omega, colors
        self.red_black = red_black
        self.t0, self.t1, self.Nl, self.Ng = t0, t1, t1 - t0, n_total
        self.n_colors = stfas.n_colors(g, colors, red_black)

    def _pb(self, l, halo):
        g = self.grids[l]
        return stfas.Problem(g, self.dt, self.K, self.r, halo.vprev, halo.vs, self.omega, self.colors,
                             self.red_black, t0=self.t0, Ng=self.Ng, n_pairs=self.Nl, unext=halo.unext)

    def halo_buffers(self, l):
        g = self.grids[l]
        mk = lambda: tuple(np.zeros(g.face_shape(k)) for k in range(g.dim))
        return {"vprev": mk(), "unext": mk()}

    def last_v(self, st):
        return tuple(np.ascontiguousarray(c[-1]) for c in st.V)

    def first_u(self, st):
        return tuple(np.ascontiguousarray(c[0]) for c in st.U)

    def copy_frame(self, dst, src):
        for d, s in zip(dst, src):
            d[...] = s

    def sync(self):
        pass

    def zeros_state(self, l=0):
        return stfas.zero_state(self.grids[l], self.Nl)

    def copy_state(self, st):
        return st.copy()

    @staticmethod
    def _assign(dst, src):
        for a, b in zip(dst.V, src.V):
            a[...] = b
        for a, b in zip(dst.U, src.U):
            a[...] = b
        dst.PB[...] = src.PB
        dst.P[...] = src.P

    def residual(self, l, st, rhs, halo):
        r = stfas.kkt_residual(self._pb(l, halo), st)
        return r.sub(rhs) if rhs is not None else r

    def color_pass(self, l, colour, st, rhs, halo):
        self._assign(st, stfas.scgs_color(self._pb(l, halo), st, rhs, colour))

    def restrict_state(self, l, st):
        return stfas.restrict_state(self.grids[l], st)

    def restrict_res(self, l, r):
        return stfas.restrict_residual(self.grids[l], r)

    def restrict_faces(self, l, comps):
        return ops.restrict_face(self.grids[l], comps)

    def prolong_add(self, lc, delta, st):
        self._assign(st, st.axpy(1.0, stfas.prolong_state(self.grids[lc], delta)))

    def axpby_state(self, l, y, x, a, b):
        for yy, xx in zip(y.V + (y.PB,) + y.U + (y.P,), x.V + (x.PB,) + x.U + (x.P,)):
            yy[...] = a * xx + b * yy

    def gauge(self, st):
        self._assign(st, stfas.gauge_fix(st))

    def norms(self, r):
        return r.inf(), r.l2() ** 2


def build_oracle_solver(pb, n_levels, slab_ids, n_slabs, comm=None):
    from paper_1608_01102_b200.slabs import SlabSolver, split_frames
    N = pb.N
    ranges = split_frames(N, n_slabs)
    engines, guides = [], []
    for p in slab_ids:
        t0, t1 = ranges[p]
        e = OracleEngine(pb.g, pb.dt, pb.K, pb.r, t0, t1, N, n_levels, pb.omega, pb.colors, pb.red_black)
        vs = []
        for c in pb.vstar:
            pad = np.zeros((max(0, t1 + 1 - N),) + c.shape[1:])
            vs.append(np.ascontiguousarray(np.concatenate([c[t0:t1 + 1], pad], 0)))
        gl = [tuple(vs)]
        for l in range(e.n_levels - 1):
            gl.append(e.restrict_faces(l, gl[-1]))
        engines.append(e)
        guides.append(gl)
    v0l = [pb.v0]
    for l in range(engines[0].n_levels - 1):
        v0l.append(engines[0].restrict_faces(l, v0l[-1]))
    states = [e.zeros_state() for e in engines]
    return SlabSolver(engines, slab_ids, n_slabs, v0l, guides, comm), states
