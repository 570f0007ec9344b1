"""Dev diagnostic: per-field / per-colour fp32 vs fp64 smoother comparison."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from oracle import stfas
from problems import make_problem, random_state
from conftest import rel_err
from paper_1608_01102_b200 import nso
from paper_1608_01102_b200.fields import GridSpec

pb = make_problem(2, n=16, N=4, seed=51)
rng = np.random.default_rng(6)
st = random_state(pb, rng)
g = pb.g
spec = GridSpec(g.dim, g.res, g.h, g.boundary)
for dt in (torch.float64, torch.float32):
    for colours in (1, 4):
        cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r)
        want = st
        for c in range(colours):
            want = stfas.scgs_color(pb, want, None, c)
        dev = nso.SpacetimeState.from_arrays(st.V, st.PB, st.U, st.P, dtype=dt)
        if colours == 4:
            nso.scgs_smooth(spec, cfg, dev, pb.v0, pb.vstar)
        else:
            # one colour only: emulate by a sweep with color_mod... run full and compare colour 0 only
            nso.scgs_smooth(spec, cfg, dev, pb.v0, pb.vstar)
            want = stfas.scgs_smooth(pb, st)
        V, PB, U, P = dev.numpy()
        print(dt, colours, "V %.2e U %.2e P %.2e PB %.2e" % (rel_err(V, want.V), rel_err(U, want.U), rel_err(P, want.P), rel_err(PB, want.PB)))
        d = np.abs(V[0] - want.V[0])
        print("   worst V0 at", np.unravel_index(np.argmax(d), d.shape), d.max())
r = nso.kkt_residual(spec, nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r), nso.SpacetimeState.from_arrays(st.V, st.PB, st.U, st.P, dtype=torch.float32), pb.v0, pb.vstar)
want = stfas.kkt_residual(pb, st)
R1, R2, R3, R4 = r.numpy()
print("res fp32: R1 %.2e R2 %.2e R3 %.2e R4 %.2e" % (rel_err(R1, want.R1), rel_err(R2, want.R2), rel_err(R3, want.R3), rel_err(R4, want.R4)))
