import sys, time, types
sys.path.insert(0, '.')
import torch
import bench
from paper_1608_01102_b200 import nso, workloads
w = workloads.config(int(sys.argv[1]))
spec = w.spec
vstar = workloads.guide_velocity(w); v0 = workloads.initial_velocity(w)
cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=w.levels)
state = nso.SpacetimeState.zeros(spec, w.N, w.dtype)
hier = nso.StfasHierarchy(spec, cfg, w.N, w.dtype); hier.set_guide(v0, vstar)
for _ in range(3):
    hier.vcycle(state); hier.gauge_fix(state)
torch.cuda.synchronize()
pin = lambda t: t.detach().cpu().pin_memory()
arr = lambda st: [*st.V, st.PB, *st.U, st.P]
h_in = [pin(t) for t in list(vstar) + arr(state)]
out_h = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in arr(state)]
# serial reference of one call
t = time.perf_counter(); hier.set_guide(v0, vstar); hier.vcycle(state); hier.gauge_fix(state); torch.cuda.synchronize()
print("one vcycle wall ms", (time.perf_counter() - t) * 1e3)
ref_state = [x.cpu() for x in arr(state)]
for d, h in zip(list(vstar) + arr(state), h_in):
    d.copy_(h)
torch.cuda.synchronize()
args = types.SimpleNamespace(steps=5)
t = time.perf_counter()
ms, reps = bench.e2e_pipelined(args, spec, cfg, w, v0, vstar, state, hier, h_in, out_h)
wall = (time.perf_counter() - t) * 1e3
print("pipelined ms/call", ms, "reps", reps, "wall total ms", wall)
# expected: out_h = state after one vcycle from h_in's state
h2 = [x.cpu() for x in h_in[len(vstar):]]
hier.set_guide(v0, vstar)
st2 = nso.SpacetimeState(tuple(x.cuda() for x in h2[:3]), h2[3].cuda(), tuple(x.cuda() for x in h2[4:7]), h2[7].cuda())
hier.vcycle(st2); hier.gauge_fix(st2); torch.cuda.synchronize()
want = [x.cpu() for x in arr(st2)]
print("max diff out vs one call", max(float((a - b).abs().max()) for a, b in zip(out_h, want)), "scale", max(float(a.abs().max()) for a in want))
