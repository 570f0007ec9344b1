"""Time-slab STFAS across GPUs.

The spacetime volume is cut into contiguous time slabs; slab p owns the pairs
[t0_p, t1_p) at every spatial level.  Each V-cycle phase runs on all local
slabs in lockstep; between phases the slab halos are refreshed:

    vprev_p = last V frame of slab p-1   (pinned v0 on slab 0)
    unext_p = first U frame of slab p+1  (none on the last slab)

Local neighbours copy, remote neighbours go through ``Comm`` (NCCL over
NVLink via torch.distributed on GPUs; gloo on CPU in the tests).  Halos are
refreshed before every residual and before every smoother colour pass, so a
colour pass on any slab sees exactly the state a single-slab colour pass would
see; the only difference from the single-GPU solver is that each cell's
time-line solve is cut at slab boundaries (block-Jacobi / Schwarz in time with
frozen neighbour frames) -- the fixed point, hence the converged solution, is
unchanged.  ‖f‖∞ is an allreduce(max) per V-cycle.

The solver is engine-agnostic: ``LibEngine`` runs every per-slab operation on
libsmk (``smk_nso_level_*``, transfers, axpby); the tests drive the same
orchestration with an oracle engine on CPU.
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _dev, _lib
from .fields import GridSpec
from .nso import SpacetimeResidual, SpacetimeState, StfasConfig, StfasHierarchy


def split_frames(n_total, parts):
    """Contiguous, as-even-as-possible split: list of (t0, t1)."""
    base, extra = divmod(n_total, parts)
    out, t = [], 0
    for p in range(parts):
        n = base + (1 if p < extra else 0)
        out.append((t, t + n))
        t += n
    return out


@dataclass
class Halo:
    vprev: tuple
    unext: tuple      # None on the last slab
    vs: tuple         # level guide, n_local + 1 frames


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------


class SingleComm:
    """One process holds every slab."""

    rank, world = 0, 1
    host_sync = False

    def exchange(self, send_left, send_right, recv_left, recv_right):
        pass

    def allreduce_max(self, x):
        return x

    def allreduce_sum(self, x):
        return x


class TorchComm:
    """torch.distributed point-to-point halos (NCCL on GPU, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # NCCL P2P is ordered on the device (the NCCL stream waits for the
        # producing kernels, wait() makes the compute stream wait for the
        # transfer): no host round-trip per exchange.  Host backends (gloo)
        # read the buffers on the host, so the device work must be finished.
        self.host_sync = dist.get_backend(group) != "nccl"

    @staticmethod
    def _t(x):
        return x if isinstance(x, torch.Tensor) else torch.from_numpy(x)

    def exchange(self, send_left, send_right, recv_left, recv_right):
        d = self.dist
        ops = []
        if self.rank > 0:
            for t in send_left:
                ops.append(d.P2POp(d.isend, self._t(t), self.rank - 1, self.group))
            for t in recv_left:
                ops.append(d.P2POp(d.irecv, self._t(t), self.rank - 1, self.group))
        if self.rank < self.world - 1:
            for t in send_right:
                ops.append(d.P2POp(d.isend, self._t(t), self.rank + 1, self.group))
            for t in recv_right:
                ops.append(d.P2POp(d.irecv, self._t(t), self.rank + 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()

    def _reduce(self, x, op):
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=op, group=self.group)
        return float(t.item())

    def allreduce_max(self, x):
        return self._reduce(x, self.dist.ReduceOp.MAX)

    def allreduce_sum(self, x):
        return self._reduce(x, self.dist.ReduceOp.SUM)


# ---------------------------------------------------------------------------
# the orchestrator
# ---------------------------------------------------------------------------


class SlabSolver:
    """FAS V-cycle over time slabs (PAPER Alg. 2 with slab halos).

    engines   one per local slab (same level structure)
    slab_ids  global slab index of each local engine (contiguous)
    n_slabs   total slab count
    v0_levels pinned initial velocity per level (used by slab 0)
    guides    per local slab, per level: guide with n_local + 1 frames
    """

    def __init__(self, engines, slab_ids, n_slabs, v0_levels, guides, comm=None, nu1=2, nu2=2, n_coarse=10):
        self.E = engines
        self.ids = list(slab_ids)
        self.P = n_slabs
        self.v0 = v0_levels
        self.guides = guides
        self.comm = comm or SingleComm()
        self.nu1, self.nu2, self.n_coarse = nu1, nu2, n_coarse
        self.L = engines[0].n_levels
        self.halo_bufs = [[e.halo_buffers(l) for l in range(self.L)] for e in engines]

    # ----- halos -----
    def exchange(self, l, states):
        E, S = self.E, len(self.E)
        bufs = [self.halo_bufs[s][l] for s in range(S)]
        # local neighbours: copy the snapshot
        for s in range(S):
            if s > 0:
                E[s].copy_frame(bufs[s]["vprev"], E[s - 1].last_v(states[s - 1]))
            if s < S - 1:
                E[s].copy_frame(bufs[s]["unext"], E[s + 1].first_u(states[s + 1]))
        # remote neighbours
        first, last = self.ids[0], self.ids[-1]
        send_left = E[0].first_u(states[0]) if first > 0 else ()
        send_right = E[-1].last_v(states[-1]) if last < self.P - 1 else ()
        recv_left = bufs[0]["vprev"] if first > 0 else ()
        recv_right = bufs[-1]["unext"] if last < self.P - 1 else ()
        if getattr(self.comm, "host_sync", True):
            E[0].sync()
        self.comm.exchange(send_left, send_right, recv_left, recv_right)
        halos = []
        for s in range(S):
            p = self.ids[s]
            vprev = self.v0[l] if p == 0 else bufs[s]["vprev"]
            unext = bufs[s]["unext"] if p < self.P - 1 else None
            halos.append(Halo(vprev, unext, self.guides[s][l]))
        return halos

    # ----- cycle -----
    def sweep(self, l, states, rhss):
        for c in range(self.E[0].n_colors):
            halos = self.exchange(l, states)
            for s, e in enumerate(self.E):
                e.color_pass(l, c, states[s], rhss[s] if rhss else None, halos[s])

    def residual(self, l, states, rhss):
        halos = self.exchange(l, states)
        return [e.residual(l, states[s], rhss[s] if rhss else None, halos[s]) for s, e in enumerate(self.E)]

    def vcycle(self, states, l=0, rhss=None):
        if l == self.L - 1:
            for _ in range(self.n_coarse):
                self.sweep(l, states, rhss)
            return states
        for _ in range(self.nu1):
            self.sweep(l, states, rhss)
        coarse = [e.restrict_state(l, st) for e, st in zip(self.E, states)]
        coarse0 = [e.copy_state(st) for e, st in zip(self.E, coarse)]
        f = self.residual(l, states, rhss)
        rf = [e.restrict_res(l, r) for e, r in zip(self.E, f)]
        rhs_c = self.residual(l + 1, coarse, rf)
        self.vcycle(coarse, l + 1, rhs_c)
        for e, c0, c, st in zip(self.E, coarse0, coarse, states):
            e.axpby_state(l + 1, c0, c, 1.0, -1.0)     # c0 <- c - c0
            e.prolong_add(l + 1, c0, st)
        for _ in range(self.nu2):
            self.sweep(l, states, rhss)
        return states

    def norms(self, states):
        f = self.residual(0, states, None)
        m, q = 0.0, 0.0
        for e, r in zip(self.E, f):
            a, b = e.norms(r)
            m, q = max(m, a), q + b
        return self.comm.allreduce_max(m), self.comm.allreduce_sum(q) ** 0.5

    def gauge(self, states):
        for e, st in zip(self.E, states):
            e.gauge(st)

    def close(self):
        for e in self.E:
            if hasattr(e, "hier"):
                e.hier.close()

    def solve(self, states, eps=1e-5, relative=False, cycle_budget=50):
        ri, r2 = self.norms(states)
        hist = [(0, ri, r2)]
        tol = eps * ri if relative else eps
        for c in range(1, cycle_budget + 1):
            if ri <= tol:
                break
            self.vcycle(states)
            self.gauge(states)
            ri, r2 = self.norms(states)
            hist.append((c, ri, r2))
        return hist


# ---------------------------------------------------------------------------
# libsmk engine (product path)
# ---------------------------------------------------------------------------


def _level_specs(spec, n):
    out = [spec]
    while len(out) < n:
        out.append(out[-1].coarsen())
    return out


class LibEngine:
    """Per-slab operations on libsmk (one smk_nso handle per slab)."""

    def __init__(self, spec, cfg, t0, t1, n_total, dtype=torch.float64):
        _dev.require_device()
        self.dtype = dtype
        self.t0, self.t1, self.Nl = t0, t1, t1 - t0
        c = StfasConfig(**{**cfg.__dict__})
        self.cfg = c
        self.hier = StfasHierarchy(spec, c, self.Nl, dtype, t0=t0, n_total=n_total)
        self.n_levels = self.hier.levels
        self.specs = _level_specs(spec, self.n_levels)
        self.n_colors = self.hier._L.smk_nso_n_colors(self.hier._h)
        self._L = _lib.load()
        self._dt = _dev._DT[dtype]

    # ---- buffers ----
    def halo_buffers(self, l):
        s = self.specs[l]
        mk = lambda: tuple(torch.zeros(s.face_shape(k), dtype=self.dtype, device="cuda") for k in range(s.dim))
        return {"vprev": mk(), "unext": mk()}

    def last_v(self, st):
        return tuple(c[-1] for c in st.V)

    def first_u(self, st):
        return tuple(c[0] for c in st.U)

    def copy_frame(self, dst, src):
        for d, s in zip(dst, src):
            d.copy_(s)

    def sync(self):
        torch.cuda.current_stream().synchronize()

    def zeros_state(self, l=0):
        return SpacetimeState.zeros(self.specs[l], self.Nl, self.dtype)

    def copy_state(self, st):
        return st.copy()

    # ---- compute ----
    def residual(self, l, st, rhs, halo):
        # k_kkt writes every row (wall rows included), so no zero-fill
        out = SpacetimeResidual.empty(self.specs[l], self.Nl, self.dtype)
        s, o = st.c_struct(), out.c_struct()
        r = rhs.c_struct() if rhs is not None else None
        rc = self._L.smk_nso_level_residual(self.hier._h, l, ctypes.byref(s), _lib.ptrs(halo.vprev),
                                            _lib.ptrs(halo.unext) if halo.unext is not None else None,
                                            _lib.ptrs(halo.vs), ctypes.byref(r) if r is not None else None,
                                            ctypes.byref(o), _dev.stream())
        _lib.check(rc, "level_residual")
        return out

    def color_pass(self, l, colour, st, rhs, halo):
        s = st.c_struct()
        r = rhs.c_struct() if rhs is not None else None
        rc = self._L.smk_nso_level_color_pass(self.hier._h, l, colour, ctypes.byref(s), _lib.ptrs(halo.vprev),
                                              _lib.ptrs(halo.unext) if halo.unext is not None else None,
                                              _lib.ptrs(halo.vs), ctypes.byref(r) if r is not None else None,
                                              _dev.stream())
        _lib.check(rc, "level_color_pass")

    def restrict_state(self, l, st):
        from .nso import restrict
        return restrict(self.specs[l], st)

    def restrict_res(self, l, r):
        from .nso import restrict
        return restrict(self.specs[l], r)

    def restrict_faces(self, l, comps):
        from .fields import restrict_face
        return restrict_face(self.specs[l], comps)

    def prolong_add(self, lc, delta, st):
        g = _dev.grid(self.specs[lc], self.dtype)
        n = self.Nl
        L = self._L
        for src, dst in ((delta.V, st.V), (delta.U, st.U)):
            _lib.check(L.smk_prolong_face(g, n, _lib.ptrs(src), _lib.ptrs(dst), 1, _dev.stream()), "prolong_face")
        for src, dst in ((delta.PB, st.PB), (delta.P, st.P)):
            _lib.check(L.smk_prolong_cell(g, n, src.data_ptr(), dst.data_ptr(), 1, _dev.stream()), "prolong_cell")

    def axpby_state(self, l, y, x, a, b):
        for yy, xx in zip((*y.V, y.PB, *y.U, y.P), (*x.V, x.PB, *x.U, x.P)):
            _lib.check(self._L.smk_axpby(self._dt, yy.data_ptr(), xx.data_ptr(), float(a), float(b), yy.numel(),
                                         _dev.stream()), "axpby")

    def gauge(self, st):
        self.hier.gauge_fix(st)

    def norms(self, r):
        m, q = 0.0, 0.0
        for a in r.arrays():
            v = ctypes.c_double()
            _lib.check(self._L.smk_inf_norm(self._dt, a.data_ptr(), a.numel(), ctypes.byref(v), _dev.stream()))
            m = max(m, v.value)
            _lib.check(self._L.smk_dot(self._dt, a.data_ptr(), a.data_ptr(), a.numel(), ctypes.byref(v),
                                       _dev.stream()))
            q += v.value
        return m, q


def guide_levels(engine, vstar_slab):
    """Per-level guides (n_local + 1 frames) from the level-0 slab guide."""
    out = [tuple(c.contiguous() for c in vstar_slab)]
    for l in range(engine.n_levels - 1):
        out.append(engine.restrict_faces(l, out[-1]))
    return out


def slab_guide(vstar, t0, t1):
    """v*_{t0} .. v*_{t1} (n_local + 1 frames; the frame past the global end,
    never read by the K term, is zero)."""
    out = []
    for c in vstar:
        n = c.shape[0]
        if t1 < n:
            out.append(c[t0:t1 + 1].contiguous())
        else:
            pad = torch.zeros((t1 + 1 - n,) + tuple(c.shape[1:]), dtype=c.dtype, device=c.device)
            out.append(torch.cat([c[t0:], pad], 0).contiguous())
    return tuple(out)


def build_lib_solver(spec, cfg, v0, vstar, slab_ids, n_slabs, n_total, dtype=torch.float64, comm=None):
    """Slab solver on libsmk for the local slabs `slab_ids` of `n_slabs`."""
    ranges = split_frames(n_total, n_slabs)
    vstar = tuple(_dev.as_dev(c, dtype) for c in vstar)
    v0 = tuple(_dev.as_dev(c, dtype) for c in v0)
    engines, guides = [], []
    for p in slab_ids:
        t0, t1 = ranges[p]
        e = LibEngine(spec, cfg, t0, t1, n_total, dtype)
        engines.append(e)
        guides.append(guide_levels(e, slab_guide(vstar, t0, t1)))
    v0_levels = [v0]
    for l in range(engines[0].n_levels - 1):
        v0_levels.append(engines[0].restrict_faces(l, v0_levels[-1]))
    states = [e.zeros_state() for e in engines]
    solver = SlabSolver(engines, slab_ids, n_slabs, v0_levels, guides, comm, cfg.nu1, cfg.nu2, cfg.n_coarse)
    return solver, states


# ---------------------------------------------------------------------------
# the product path: the slab V-cycle in C++ (smk_slabs_*, one CUDA graph per
# V-cycle with the halo copies / NCCL P2P inside; no Python per colour pass)
# ---------------------------------------------------------------------------


class NcclSlabComm:
    """Rank layout of the C++ slab set: world ranks, rank r holds a contiguous
    block of slabs; the NCCL communicator is created inside libsmk from rank
    0's unique id, broadcast here over torch.distributed (any backend)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        buf = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            raw = (ctypes.c_ubyte * 128)()
            _lib.check(_lib.load().smk_nccl_unique_id(ctypes.cast(raw, ctypes.c_void_p), 128), "nccl_unique_id")
            buf = torch.tensor(list(raw), dtype=torch.uint8)
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        b = buf.to(dev)
        dist.broadcast(b, 0, group=group)
        self.uid = bytes(b.cpu().tolist())


class CSlabSolver:
    """Time-slab STFAS on libsmk's C++ slab set: same phases
    and halo semantics as SlabSolver (bitwise the same kernels per slab), the
    whole V-cycle replayed from one CUDA graph."""

    def __init__(self, spec, cfg, v0, vstar, slab_ids, n_slabs, n_total, dtype=torch.float64, comm=None):
        _dev.require_device()
        self.dtype = dtype
        self.spec = spec
        self.ids = list(slab_ids)
        if self.ids != list(range(self.ids[0], self.ids[0] + len(self.ids))):
            raise ValueError("local slabs must be contiguous")
        self._L = _lib.load()
        rank, world, uid = 0, 1, None
        if comm is not None:
            rank, world, uid = comm.rank, comm.world, comm.uid
        self._uid = ctypes.create_string_buffer(uid, 128) if uid else None
        g = _dev.grid(spec, dtype)
        p = cfg.params(n_total)
        h = self._L.smk_slabs_create(ctypes.byref(g), ctypes.byref(p), self.ids[0], len(self.ids), n_slabs, rank,
                                     world, ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None)
        if not h:
            _lib.check(_lib.SMK_ERR_CUDA, "slabs_create")
        self._h = h
        self.L = self._L.smk_slabs_levels(h)
        self.frames = []
        for k in range(len(self.ids)):
            t0, n = ctypes.c_int(), ctypes.c_int()
            _lib.check(self._L.smk_slabs_frames(h, k, ctypes.byref(t0), ctypes.byref(n)), "slabs_frames")
            self.frames.append((t0.value, n.value))
        self.set_guide(v0, vstar)

    def set_guide(self, v0=None, vstar=None):
        """Bind v0 / the full guide v*_0..v*_{N-1} (device copies kept); with
        no arguments, re-read the bound tensors (after an in-place update)."""
        if v0 is not None:
            self._v0 = tuple(_dev.as_dev(c, self.dtype).contiguous() for c in v0)
        if vstar is not None:
            self._vs = tuple(_dev.as_dev(c, self.dtype).contiguous() for c in vstar)
        _lib.check(self._L.smk_slabs_set_guide(self._h, _lib.ptrs(self._v0), _lib.ptrs(self._vs), _dev.stream()),
                   "slabs_set_guide")

    def zero_states(self):
        return [SpacetimeState.zeros(self.spec, n, self.dtype) for _, n in self.frames]

    def _arr(self, states):
        arr = (_lib.smk_state * len(states))()
        for k, st in enumerate(states):
            arr[k] = st.c_struct()
        return arr

    def vcycle(self, states):
        _lib.check(self._L.smk_slabs_vcycle(self._h, self._arr(states), _dev.stream()), "slabs_vcycle")
        return states

    def gauge(self, states):
        _lib.check(self._L.smk_slabs_gauge_fix(self._h, self._arr(states), _dev.stream()), "slabs_gauge")

    def norms(self, states):
        ri, r2 = ctypes.c_double(), ctypes.c_double()
        _lib.check(self._L.smk_slabs_residual_norms(self._h, self._arr(states), ctypes.byref(ri), ctypes.byref(r2),
                                                    _dev.stream()), "slabs_norms")
        return ri.value, r2.value

    def solve(self, states, eps=1e-5, relative=False, cycle_budget=50):
        return SlabSolver.solve(self, states, eps, relative, cycle_budget)

    def device_bytes(self):
        return int(self._L.smk_slabs_device_bytes(self._h))

    # the StfasHierarchy profiling interface, summed over the local slabs
    KERNELS = StfasHierarchy.KERNELS

    @property
    def levels(self):
        return self.L

    def profile(self, enable=True):
        _lib.check(self._L.smk_slabs_profile(self._h, int(bool(enable))), "slabs_profile")

    def profile_read(self, kind=0, level=None):
        ms, n, cells = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_longlong()
        _lib.check(self._L.smk_slabs_profile_read_level(self._h, int(kind), -1 if level is None else int(level),
                                                        ctypes.byref(ms), ctypes.byref(n), ctypes.byref(cells)),
                   "slabs_profile_read")
        return ms.value, n.value, cells.value

    def close(self):
        if self._h:
            self._L.smk_slabs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_c_solver(spec, cfg, v0, vstar, slab_ids, n_slabs, n_total, dtype=torch.float64, comm=None):
    """C++ slab solver for the local slabs `slab_ids` of `n_slabs`, and zero
    states for them."""
    s = CSlabSolver(spec, cfg, v0, vstar, slab_ids, n_slabs, n_total, dtype, comm)
    return s, s.zero_states()
