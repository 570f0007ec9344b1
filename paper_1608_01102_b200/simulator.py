"""Forward step on B200 — drop-in for ``pkg/src/smokectrl/simulator.py``.

One ``smk_sim_step`` call runs the whole step on the device: Taylor density
advection by the pre-step velocity, the Picard-implicit self-advection with a
multigrid projection per sweep, and pressure recovery (``simulator.py:73-110``).
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _dev, _lib
from .advection import DEFAULT_TERM_CAP, DEFAULT_TRUNCATION_TOL
from .errors import NonConvergence
from .fields import ScalarField, StaggeredVectorField


@dataclass
class SimConfig:
    """``simulator.py:28-40``."""

    dt: float
    picard_iters: int = 3
    sim_tol: float = 1e-6
    truncation_tol: float = DEFAULT_TRUNCATION_TOL
    truncation_cap: int = DEFAULT_TERM_CAP

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.picard_iters < 1:
            raise ValueError("picard_iters must be >= 1")


@dataclass
class SimState:
    """``simulator.py:43-53``."""

    v: StaggeredVectorField
    p: ScalarField
    rho: ScalarField

    @classmethod
    def rest(cls, spec, rho0):
        dt = rho0.values.dtype
        return cls(StaggeredVectorField.zeros(spec, dt), ScalarField.zeros(spec, dt), rho0)


def step(state, u, cfg, accept_stall=False):
    """``simulator.py:73-110``."""
    _dev.require_device()
    spec = state.v.spec
    dt = state.v.comps[0].dtype
    v = tuple(_dev.as_dev(c, dt) for c in state.v.comps)
    uu = tuple(_dev.as_dev(c, dt) for c in u.comps)
    rho = _dev.as_dev(state.rho.values, dt)
    v_out = tuple(torch.empty_like(c) for c in v)
    p_out = torch.empty_like(rho)
    rho_out = torch.empty_like(rho)
    k = ctypes.c_int()
    resid = ctypes.c_double()
    L = _lib.load()
    rc = L.smk_sim_step(_dev.grid(spec, dt), _lib.ptrs(v), rho.data_ptr(), _lib.ptrs(uu), float(cfg.dt),
                        int(cfg.picard_iters), float(cfg.sim_tol), float(cfg.truncation_tol),
                        int(cfg.truncation_cap), _lib.ptrs(v_out), p_out.data_ptr(), rho_out.data_ptr(),
                        ctypes.byref(k), ctypes.byref(resid), _dev.stream())
    new_state = SimState(StaggeredVectorField(spec, v_out), ScalarField(spec, p_out), ScalarField(spec, rho_out))
    if rc == _lib.SMK_NONCONVERGENCE and resid.value > cfg.sim_tol:
        if accept_stall:
            return new_state
        err = NonConvergence(f"Picard update stalled at {resid.value:.3e} > sim_tol {cfg.sim_tol:.3e}",
                             residual=resid.value)
        err.state = new_state
        raise err
    _lib.check(rc, "sim_step")
    return new_state


def simulate(state0, forces, cfg, accept_stall=False):
    """``simulator.py:113-122``."""
    states = [state0]
    for i, u in enumerate(forces):
        try:
            states.append(step(states[-1], u, cfg, accept_stall=accept_stall))
        except NonConvergence as e:
            e.context = f"timestep {i}"
            raise
    return states
