"""Diagnostic: one red-black sweep per kernel shape x fused/unfused vs the C oracle."""
import os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
SHAPES = {"tm64p1": ("0,0", "0"), "tm32p2": ("1000000000,0", str(1 << 40)), "tm32p4": ("1000000000,1000000000", str(1 << 40))}

def child(n, N, shape, fuse, out):
    import numpy as np, torch
    from paper_1608_01102_b200 import nso
    from paper_1608_01102_b200.fields import GridSpec
    g = torch.Generator().manual_seed(5)
    spec = GridSpec(3, (n, n, n), 1.0 / n, "neumann")
    cfg = nso.StfasConfig(dt=1.0 / N, K=1e3, r=1e3, omega=0.8)
    shp = lambda k: (N,) + tuple(n + (a == k) for a in range(3))
    V = tuple((0.1 * torch.randn(shp(k), generator=g, dtype=torch.float64)) for k in range(3))
    U = tuple((0.1 * torch.randn(shp(k), generator=g, dtype=torch.float64)) for k in range(3))
    PB = 0.1 * torch.randn((N, n, n, n), generator=g, dtype=torch.float64)
    P = 0.1 * torch.randn((N, n, n, n), generator=g, dtype=torch.float64)
    vs = tuple((0.1 * torch.randn(shp(k), generator=g, dtype=torch.float64)) for k in range(3))
    # walls zero
    for k in range(3):
        for c in (V[k], U[k], vs[k]):
            idx = [slice(None)] * 4; idx[k + 1] = 0; c[tuple(idx)] = 0; idx[k + 1] = -1; c[tuple(idx)] = 0
    v0 = tuple(torch.zeros(shp(k)[1:], dtype=torch.float64) for k in range(3))
    dev = nso.SpacetimeState.from_arrays([c.numpy() for c in V], PB.numpy(), [c.numpy() for c in U], P.numpy(), dtype=torch.float64)
    nso.scgs_smooth(spec, cfg, dev, [c.numpy() for c in v0], [c.numpy() for c in vs])
    Vd, PBd, Ud, Pd = dev.numpy()
    np.savez(out, V0=Vd[0], V1=Vd[1], V2=Vd[2], U0=Ud[0], U1=Ud[1], U2=Ud[2], P=Pd, PB=PBd,
             iV0=V[0].numpy(), iV1=V[1].numpy(), iV2=V[2].numpy(), iU0=U[0].numpy(), iU1=U[1].numpy(),
             iU2=U[2].numpy(), iP=P.numpy(), iPB=PB.numpy(), vs0=vs[0].numpy(), vs1=vs[1].numpy(), vs2=vs[2].numpy())

if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5], sys.argv[6]); sys.exit(0)
    import numpy as np
    from oracle import cstfas, stfas
    from oracle.grid import Grid
    for n, N in [(int(a.split("x")[0]), int(a.split("x")[1])) for a in sys.argv[1:]]:
        res = {}
        for shape, (ft, bf) in SHAPES.items():
            for fuse in ("1", "0"):
                env = dict(os.environ, SMK_FWD_THRESH=ft, SMK_BACK_FLAT=bf, SMK_BACK_DEEP="1", SMK_NO_FUSE="0" if fuse == "1" else "1")
                out = f"/tmp/diag_{n}_{shape}_{fuse}.npz"
                subprocess.check_call([sys.executable, __file__, "child", str(n), str(N), shape, fuse, out], env=env)
                res[(shape, fuse)] = np.load(out)
        z = res[("tm64p1", "1")]
        g = Grid(3, (n,) * 3, 1.0 / n, "neumann")
        pb = stfas.Problem(g, 1.0 / N, 1e3, 1e3, tuple(np.zeros(g.face_shape(k)) for k in range(3)), (z["vs0"], z["vs1"], z["vs2"]))
        st = stfas.State((z["iV0"], z["iV1"], z["iV2"]), z["iPB"], (z["iU0"], z["iU1"], z["iU2"]), z["iP"])
        want = cstfas.scgs_smooth(pb, st)
        w = dict(V0=want.V[0], V1=want.V[1], V2=want.V[2], U0=want.U[0], U1=want.U[1], U2=want.U[2], P=want.P, PB=want.PB)
        for key, d in res.items():
            errs = {f: float(np.max(np.abs(d[f] - w[f])) / max(np.max(np.abs(w[f])), 1e-300)) for f in w}
            worst = max(errs, key=errs.get)
            bad = np.argwhere(np.abs(d[worst] - w[worst]) > 1e-6 * np.max(np.abs(w[worst])))
            print(n, N, key, f"max rel {errs[worst]:.2e} in {worst}", "n_bad", len(bad), "first", bad[:4].tolist(), flush=True)
