"""Exercise every colour-pass kernel shape once, small, for compute-sanitizer
(racecheck / synccheck / memcheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_shapes.py

Forward shapes TM 64 / P 1 (compact + fused backward, factored + unpipelined
/ pipelined backward), TM 32 / P 2, TM 32 / P 4 (record hand-off + cp.async
ring backward, and the factored fallback), 2D / 3D, fp32 / fp64, one
V-cycle of a 2-level hierarchy (residual, transfers, both sweeps), the
fused residual-norm stop test and a 2-slab C++ slab V-cycle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

from oracle import stfas  # noqa: E402
from paper_1608_01102_b200 import _lib, nso, slabs  # noqa: E402
from paper_1608_01102_b200.fields import GridSpec  # noqa: E402
from problems import make_problem  # noqa: E402

SHAPES = [("tm64p1-cmp", "0,0", "0", "1"), ("tm64p1-fact", "0,0", str(1 << 40), "1"),
          ("tm32p2", "1000000000,0", str(1 << 40), "1"), ("tm32p4-rec", "1000000000,1000000000", str(1 << 40), "1"),
          ("tm32p4-fact", "1000000000,1000000000", str(1 << 40), "0")]


def main():
    _lib.load()
    for dim, n in ((2, 16), (3, 8)):
        pb = make_problem(dim, n=n, N=3, seed=5)
        g = pb.g
        spec = GridSpec(g.dim, g.res, g.h, g.boundary)
        for dtype in (torch.float64, torch.float32):
            for name, fwd, bf, deep in SHAPES:
                os.environ["SMK_FWD_THRESH"] = fwd
                os.environ["SMK_BACK_FLAT"] = bf
                os.environ["SMK_BACK_DEEP"] = deep
                cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=2)
                h = nso.StfasHierarchy(spec, cfg, pb.N, dtype)
                h.set_guide(pb.v0, pb.vstar)
                s = nso.SpacetimeState.zeros(spec, pb.N, dtype)
                h.vcycle(s)
                h.gauge_fix(s)
                ri, _ = h.residual_norms(s)
                torch.cuda.synchronize()
                h.close()
                print(f"dim={dim} {str(dtype)[6:]} {name}: |f|={ri:.3e}", flush=True)
    for k in ("SMK_FWD_THRESH", "SMK_BACK_FLAT", "SMK_BACK_DEEP"):
        os.environ.pop(k, None)
    pb = make_problem(3, n=8, N=4, seed=6)
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=2)
    cs, st = slabs.build_c_solver(spec, cfg, pb.v0, pb.vstar, [0, 1], 2, pb.N)
    cs.vcycle(st)
    cs.gauge(st)
    print("slabs x2 |f| =", cs.norms(st)[0], flush=True)
    cs.close()


if __name__ == "__main__":
    main()
