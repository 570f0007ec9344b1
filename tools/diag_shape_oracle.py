"""Diagnose GPU sweep vs C oracle on random 3D states (size / recipe sweep)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from oracle import cstfas, stfas
from oracle.grid import Grid
from paper_1608_01102_b200 import _lib, nso
from paper_1608_01102_b200.fields import GridSpec
from conftest import rel_err
_lib.load(); cstfas.load()

def case(n, N, K, r, amp, walls=True, seed=5):
    spec = GridSpec(3, (n, n, n), 1.0 / n, "neumann")
    cfg = nso.StfasConfig(dt=1.0 / N, K=K, r=r, omega=0.8)
    g = torch.Generator().manual_seed(seed)
    shp = lambda k: (N,) + tuple(n + (a == k) for a in range(3))
    V = tuple((amp * torch.randn(shp(k), generator=g, dtype=torch.float64)) for k in range(3))
    U = tuple((amp * torch.randn(shp(k), generator=g, dtype=torch.float64)) for k in range(3))
    PB = amp * torch.randn((N, n, n, n), generator=g, dtype=torch.float64)
    P = amp * torch.randn((N, n, n, n), generator=g, dtype=torch.float64)
    vs = tuple((amp * torch.randn(shp(k), generator=g, dtype=torch.float64)) for k in range(3))
    v0 = tuple(torch.zeros(shp(k)[1:], dtype=torch.float64) for k in range(3))
    if walls:
        for k in range(3):
            for c in (V[k], U[k], vs[k]):
                idx = [slice(None)] * 4; idx[k + 1] = 0; c[tuple(idx)] = 0; idx[k + 1] = -1; c[tuple(idx)] = 0
    dev = nso.SpacetimeState.from_arrays([c.numpy() for c in V], PB.numpy(), [c.numpy() for c in U], P.numpy(), dtype=torch.float64)
    nso.scgs_smooth(spec, cfg, dev, [c.numpy() for c in v0], [c.numpy() for c in vs])
    got = dev.numpy()
    og = Grid(3, (n, n, n), 1.0 / n, "neumann")
    pb = stfas.Problem(og, 1.0 / N, K, r, tuple(c.numpy() for c in v0), tuple(c.numpy() for c in vs))
    st = stfas.State(tuple(c.numpy() for c in V), PB.numpy(), tuple(c.numpy() for c in U), P.numpy())
    want = cstfas.scgs_smooth(pb, st)
    e = {"V": rel_err(tuple(got[0]), want.V), "PB": rel_err(got[1], want.PB), "U": rel_err(tuple(got[2]), want.U), "P": rel_err(got[3], want.P)}
    # the update itself
    dV = tuple(a - b for a, b in zip(got[0], st.V)); wV = tuple(a - b for a, b in zip(want.V, st.V))
    e["dV"] = rel_err(dV, wV)
    print(f"n={n} N={N} K={K} r={r} amp={amp} walls={walls}: " + " ".join(f"{k}={v:.2e}" for k, v in e.items()), flush=True)

for amp in (0.01, 0.03):
    for n in (16, 32, 64):
        try:
            case(n, 6, 1e3, 1e3, amp)
        except Exception as ex:
            print(f"n={n} amp={amp}: {type(ex).__name__}: {ex}", flush=True)
