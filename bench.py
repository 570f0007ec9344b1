#!/usr/bin/env python
"""STFAS V-cycle throughput on B200 (BASELINE.json metric).

metric: spacetime cell-updates/s = n^d * N / (seconds per FAS V-cycle), with
s/V-cycle and HBM GB/s reported beside it.  A "step" is one full STFAS
V-cycle (all levels, PAPER Alg. 2) over the whole spacetime volume, inputs
resident in HBM.  Default workload: BASELINE config 5 (3D 128^3 x 80 fp32,
4 levels), the config the metric's 1/2/4/8-GPU scaling is quoted on.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5]
    python bench.py --impl reference ...   # CPU oracle (port) on host cores

Multi-GPU (N>1, torchrun): the spacetime volume is split into N contiguous
time slabs, one per rank (strong scaling: total work fixed), on libsmk's C++
slab set: the whole V-cycle is one CUDA graph per rank with the halo NCCL
send / recv before every residual / colour pass inside it, ||f|| an NCCL
allreduce -- paper_1608_01102_b200/slabs.py CSlabSolver, DESIGN.md §6.
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# bytes per cell-timestep moved by one smoother sweep: read and
# write the state (s = 2d+2 values) and read the guide (d values)
def sweep_values(dim):
    s = 2 * dim + 2
    return 2 * s + dim


def vcycle_values_per_cts(dim, levels):
    """SURVEY.md §8d algorithmic values per fine cell-timestep per V-cycle."""
    s, g = 2 * dim + 2, dim
    r = s
    per = {}
    l0 = 4 * (2 * s + g) + (s + s / 2 ** dim) + (s + g + s / 2 ** dim) + (2 * s / 2 ** dim + 2 * s)
    lmid = 4 * (2 * s + g + r) + (s + s / 2 ** dim) + (s + g + r + s / 2 ** dim) + (2 * s / 2 ** dim + 2 * s) \
        + (3 * s + g)
    coarsest = 10 * (2 * s + g + r) + (3 * s + g)
    tot = 0.0
    for l in range(levels):
        w = 2.0 ** (-dim * l)
        if l == levels - 1:
            tot += w * coarsest
        elif l == 0:
            tot += w * l0
        else:
            tot += w * lmid
    return tot


def traffic_ref(workload, kernel):
    """Measured DRAM bytes per level-0 launch of `kernel` for `workload` from
    the committed ncu capture summary (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d[workload][kernel]
        return {"bytes_per_launch": float(e["bytes_per_launch"]), "source": e["source"]}
    except Exception:
        return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.strip().split(",") for r in self.f.read().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(w, full=False):
    """The CPU arm's bounded sample of workload w: the config itself for the
    2D configs (or on request), else the config's spatial grid and level
    count on a short time line (the oracle's cost per cell-timestep is
    independent of N: the time-line solve is linear in N)."""
    if full or w.dim == 2:
        return dict(n=w.n, N=w.N, levels=w.levels, same_config=True)
    return dict(n=w.n, N=2, levels=w.levels, same_config=False)


def cpu_vcycle_rate(w, steps=1, warmup=0, full=False, threads=0):
    """Time the C oracle (oracle/cstfas.c: the numpy oracle restated in C,
    OpenMP over the cells of a colour) V-cycle on the host cores.
    Returns (cell-updates/s, s per V-cycle, sample, threads)."""
    import numpy as np
    from oracle import cstfas, stfas
    from oracle.grid import Grid
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from problems import smooth_vector
    sh = cpu_sample(w, full)
    nt = cstfas.set_threads(threads)
    g = Grid(w.dim, (sh["n"],) * w.dim, 1.0 / sh["n"], "neumann")
    rng = np.random.default_rng(1608_01102 + w.index)
    dt = w.dt
    # same recipe as workloads.guide_velocity (band-limited, projected, dt|v*|/h = 1)
    # band-limited guide of the workloads' scale (not projected: the oracle's
    # cost does not depend on the guide's values)
    vs = [smooth_vector(g, rng, g.h / dt) for _ in range(sh["N"])]
    vstar = tuple(np.stack([v[k] for v in vs]) for k in range(w.dim))
    v0 = tuple(np.zeros(g.face_shape(k)) for k in range(w.dim))
    pb = stfas.Problem(g, dt, w.K, w.r, v0, vstar)
    H = cstfas.Hierarchy(pb, sh["levels"])
    st = stfas.zero_state(g, sh["N"])
    for _ in range(warmup):
        st = H.vcycle(st, gauge=True)
    t0 = time.perf_counter()
    for _ in range(steps):
        st = H.vcycle(st, gauge=True)
    sec = (time.perf_counter() - t0) / max(steps, 1)
    H.close()
    cts = sh["n"] ** w.dim * sh["N"]
    sh["levels"] = len(stfas.build_levels(pb, sh["levels"]))
    return cts / sec, sec, sh, nt


def cpu_sample_text(w, sh, nt, sec):
    return (f"C restatement of the oracle (oracle/cstfas.c, fp64, OpenMP over colour cells; the reference "
            f"ships no STFAS) FAS V-cycle on {sh['n']}^{w.dim} x {sh['N']} frames, {sh['levels']} levels"
            f"{' (= the config)' if sh['same_config'] else ' (the config grid on a short time line)'}, "
            f"{nt} host threads, {sec:.2f} s per V-cycle")


def run_reference(args, w, rank, world):
    if rank != 0:
        return 0
    steps, warm = args.steps, args.warmup
    rate, sec, sh, nt = cpu_vcycle_rate(w, steps, warm, full=args.cpu_full)
    line = {
        "impl": "reference", "metric": "STFAS spacetime cell-updates/s (per V-cycle)", "value": rate,
        "unit": "cell-updates/s", "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": 1000.0 * sec,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "config_index": w.index, "cell_timesteps": w.cell_timesteps,
                   "sample_cell_timesteps": sh["n"] ** w.dim * sh["N"], "same_config": sh["same_config"],
                   "parallelism": f"cpu x{nt} threads"},
        "cpu_baseline": {"value": rate, "unit": "cell-updates/s", "cores": nt, "kind": "port",
                         "sample": cpu_sample_text(w, sh, nt, sec)},
        "e2e": {"value": rate, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def time_to_solution(nso, spec, w, v0, vstar, levels, budget):
    """solve_nso from zero to eps (fp64: absolute 1e-5; fp32:
    relative 1e-5 * ||f_0||), every V-cycle + gauge + the
    ||f|| stop test device-timed; returns the record for the bench line."""
    import torch
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=levels)
    hier = nso.StfasHierarchy(spec, cfg, w.N, w.dtype)
    hier.set_guide(v0, vstar)
    st = nso.SpacetimeState.zeros(spec, w.N, w.dtype)
    scratch = st.copy()
    hier.vcycle(scratch)           # graph capture outside the timed solve
    del scratch
    st2 = nso.SpacetimeState.zeros(spec, w.N, w.dtype)
    torch.cuda.synchronize()
    f0, _ = hier.residual_norms(st2)
    rel = w.dtype == torch.float32
    tol = 1e-5 * f0 if rel else 1e-5
    hist, t_ms, reached, stop_ms = [f0], 0.0, None, 0.0
    for c in range(1, budget + 1):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        hier.vcycle(st2)
        hier.gauge_fix(st2)
        e1.record()
        ri, _ = hier.residual_norms(st2)
        e2.record()
        e2.synchronize()
        t_ms += e0.elapsed_time(e2)
        stop_ms += e1.elapsed_time(e2)
        hist.append(ri)
        if ri <= tol:
            reached = c
            break
    out = {"levels": hier.levels, "eps": 1e-5, "eps_kind": "relative" if rel else "absolute", "f0_inf": f0,
           "vcycles_to_eps": reached, "s_to_solution": t_ms / 1000.0 if reached else None,
           "final_residual_inf": hist[-1], "stop_test_ms_per_cycle": stop_ms / max(1, len(hist) - 1),
           "residual_history": [float(f"{x:.4e}") for x in hist],
           "asym_factor": (hist[-1] / hist[-4]) ** (1 / 3) if len(hist) >= 4 and hist[-4] > 0 else None}
    hier.close()
    return out


E2E_LANES = 3


def e2e_pipelined(args, spec, cfg, w, v0, vstar, state, hier, h_in, out_h):
    """End-to-end throughput of a stream of independent solve calls with host
    buffers: each call uploads its inputs (guide + state) from pinned memory,
    runs set_guide + one V-cycle + gauge, and downloads the updated state.
    E2E_LANES buffer lanes (state, guide, hierarchy each) let call k+1's upload
    and call k-1's download (copy engines, both PCIe directions at once) overlap
    call k's V-cycle.  A lane is busy from its upload start to its download end
    (upload + solve + download), so two lanes bound a call at half that sum;
    three leave the period at the slowest of the three legs.  Every call still
    moves all of its bytes inside the timed region (first upload start -> last
    download end, device events)."""
    import torch
    from paper_1608_01102_b200 import nso
    nl = E2E_LANES
    lanes = [(state, list(vstar), hier)]
    extra = []
    for _ in range(nl - 1):
        st1 = nso.SpacetimeState.zeros(spec, w.N, w.dtype)
        vs1 = [torch.empty_like(c) for c in vstar]
        for d, s_ in zip(vs1, vstar):
            d.copy_(s_)
        h1 = nso.StfasHierarchy(spec, cfg, w.N, w.dtype)
        lanes.append((st1, vs1, h1))
        extra.append(h1)
    outs = [out_h] + [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in out_h] for _ in range(nl - 1)]
    sH, sC, sD = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    arrays = lambda st: [*st.V, st.PB, *st.U, st.P]

    def call(k, done):
        st, vs, hr = lanes[k % nl]
        d_in = list(vs) + arrays(st)
        if done[k % nl] is not None:
            sH.wait_event(done[k % nl])
        with torch.cuda.stream(sH):
            for d, h in zip(d_in, h_in):
                d.copy_(h, non_blocking=True)
            eh = torch.cuda.Event()
            eh.record(sH)
        sC.wait_event(eh)
        with torch.cuda.stream(sC):
            hr.set_guide(v0, vs)
            hr.vcycle(st)
            hr.gauge_fix(st)
            ec = torch.cuda.Event()
            ec.record(sC)
        sD.wait_event(ec)
        with torch.cuda.stream(sD):
            for h, d in zip(outs[k % nl], arrays(st)):
                h.copy_(d, non_blocking=True)
            ed = torch.cuda.Event()
            ed.record(sD)
        done[k % nl] = ed

    # untimed: one call per lane (graph capture of each lane's V-cycle)
    done = [None] * nl
    for k in range(nl):
        call(k, done)
    torch.cuda.synchronize()
    reps = max(8 * nl, args.steps)   # a stream of calls: fill (one upload) + drain (one download) amortised over 24
    done = [None] * nl
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(sH)
    for k in range(reps):
        call(k, done)
    sD.wait_event(done[(reps - 1) % nl])
    e1.record(sD)
    e1.synchronize()
    torch.cuda.synchronize()
    for h1 in extra:
        h1.close()
    return e0.elapsed_time(e1) / reps, reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--dtype", default=None, choices=[None, "fp32", "fp64"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true", help="e2e calls back to back (no copy/compute overlap)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="CPU arm on the whole config (3D: minutes)")
    ap.add_argument("--levels", type=int, default=0, help="hierarchy depth (0 = the config's)")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution solves")
    ap.add_argument("--tts-budget", type=int, default=80)
    ap.add_argument("--slabs", type=int, default=0,
                    help="single process: S in-process time slabs on the C++ slab set (the N > 1 code path on one GPU)")
    args = ap.parse_args()

    import torch
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    from paper_1608_01102_b200 import workloads
    dt_override = {"fp32": torch.float32, "fp64": torch.float64}.get(args.dtype)
    w = workloads.config(args.config, dt_override)

    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    import torch.distributed as dist
    from paper_1608_01102_b200 import _lib, nso
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    L = _lib.load()

    spec = w.spec
    vstar = workloads.guide_velocity(w)
    v0 = workloads.initial_velocity(w)
    cfg = nso.StfasConfig(dt=w.dt, K=w.K, r=w.r, n_levels=args.levels or w.levels)
    stream = torch.cuda.current_stream()
    slab = None
    n_slabs = world if world > 1 else max(1, args.slabs)
    if n_slabs > 1:
        # one slab per rank (NCCL halos), or --slabs S in-process slabs on one GPU
        from paper_1608_01102_b200 import slabs
        ids = [rank] if world > 1 else list(range(n_slabs))
        slab, states = slabs.build_c_solver(spec, cfg, v0, vstar, ids, n_slabs, w.N, w.dtype,
                                            comm=slabs.NcclSlabComm() if world > 1 else None)
        hier = slab                      # same profiling interface, summed over the local slabs
        slab_t0 = slab.frames[0][0]
        n_local = sum(n for _, n in slab.frames)
    else:
        state = nso.SpacetimeState.zeros(spec, w.N, w.dtype)
        hier = nso.StfasHierarchy(spec, cfg, w.N, w.dtype)
        hier.set_guide(v0, vstar)
        n_local = w.N
        states = [state]

    def step():
        if slab is not None:
            slab.vcycle(states)
            slab.gauge(states)
        else:
            hier.vcycle(state)
            hier.gauge_fix(state)

    # inputs larger than L2 (126 MB) for configs >= 3; otherwise flush L2
    state_tensors = [t for st in states for t in (*st.V, st.PB, *st.U, st.P)]
    state_bytes = sum(t.numel() * t.element_size() for t in state_tensors)
    guide_bytes = sum(t.numel() * t.element_size() for t in vstar) * n_local // w.N
    flush = None
    if state_bytes + guide_bytes < 4 * 126e6:
        flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device events) ----------------
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local) if rank == 0 else None
    n0 = L.smk_launch_count()
    torch.cuda.profiler.start()   # ncu --profile-from-start off sees only this region
    t_total = 0.0
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        t_total += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    launches = L.smk_launch_count() - n0
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    # per-kernel breakdown: separate, untimed V-cycles with CUDA events around
    # every colour-pass / residual kernel (the events would perturb the timed
    # region, so it runs without them)
    prof_steps = max(1, min(args.steps, 2))
    hier.profile(True)
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize()
    kprof = {name: hier.profile_read(kind) for kind, name in hier.KERNELS.items()}
    kprof_lv = {name: [hier.profile_read(kind, level=l) for l in range(hier.levels)]
                for kind, name in hier.KERNELS.items()}
    hier.profile(False)
    ms = t_total / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    if slab is not None:
        ri, r2 = slab.norms(states)
    else:
        ri, r2 = hier.residual_norms(state)
    value = w.cell_timesteps / (ms / 1000.0)   # strong scaling: the whole volume per V-cycle
    hbm, peak_kind = peaks()
    esz = 4 if w.dtype == torch.float32 else 8
    # dominant kernel: the fine-level forward elimination k_scgs_fwd (level 0).
    # Algorithmic bytes per launch = SURVEY §8d's smoother figure for the cells
    # the launch updates: (2s + g) values per colour cell-timestep (read and
    # write the state, read the guide; level 0 has no rhs) x colour cells x
    # frames.  traffic = measured DRAM bytes per L0 launch from the committed
    # ncu capture of this workload (profiles/traffic.json), or null.
    kname = "k_scgs_fwd"
    k_ms, k_n, k_cells = kprof_lv[kname][0]
    k_avg_ms = k_ms / max(k_n, 1)
    k_bytes_launch = (k_cells / max(k_n, 1)) * sweep_values(w.dim) * esz
    k_achieved = k_bytes_launch / (k_avg_ms / 1000.0) / 1e9 if k_n else 0.0
    traffic = traffic_ref(w.name, kname) if slab is None else None   # the capture is of the whole time line
    kernels = {}
    for k, v in kprof.items():
        kernels[k] = {"ms_per_step": v[0] / prof_steps, "launches_per_step": v[1] / prof_steps,
                      "share_of_step": (v[0] / prof_steps) / ms if ms else None,
                      "ms_per_step_by_level": [round(x[0] / prof_steps, 3) for x in kprof_lv[k]]}
    vc_bytes = vcycle_values_per_cts(w.dim, hier.levels) * esz * w.cell_timesteps
    vc_gbs = vc_bytes / (ms / 1000.0) / 1e9 / world

    # ---------------- end to end through the public API ----------------
    e2e = None
    if not args.no_e2e:
        # each rank: H2D of its inputs (its slab's state and level-0 guide --
        # the whole problem at N = 1), the V-cycle, D2H of the updated state;
        # device-timed, max over ranks
        pin = lambda t: t.detach().cpu().pin_memory()
        if slab is None:
            d_in = list(vstar) + state_tensors
        else:
            # this rank's guide frames v*_{t0} .. v*_{t0+n} (uploaded into the
            # full guide tensor, re-bound by set_guide inside the timed region)
            t1 = min(slab_t0 + n_local + 1, w.N)
            d_in = [c[slab_t0:t1] for c in vstar] + state_tensors
        d_st = state_tensors
        h_in = [pin(t) for t in d_in]
        out_h = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in d_st]
        h2d = sum(t.numel() * t.element_size() for t in h_in)
        d2h = sum(t.numel() * t.element_size() for t in out_h)
        reps = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e_ms = 0.0
        pipelined = slab is None and not args.e2e_serial
        if pipelined:
            e_ms, reps = e2e_pipelined(args, spec, cfg, w, v0, vstar, state, hier, h_in, out_h)
        for _ in range(0 if pipelined else reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for d, h in zip(d_in, h_in):
                d.copy_(h, non_blocking=True)
            if slab is None:
                hier.set_guide(v0, vstar)
            else:
                slab.set_guide()
            step()
            for h, d in zip(out_h, d_st):
                h.copy_(d, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            e_ms += e0.elapsed_time(e1)
        if not pipelined:
            e_ms /= reps
        if world > 1:
            t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
            hb = torch.tensor([float(h2d), float(d2h)], device="cuda", dtype=torch.float64)
            dist.all_reduce(hb, op=dist.ReduceOp.SUM)
            h2d, d2h = hb[0].item(), hb[1].item()
        e2e = {"value": w.cell_timesteps / (e_ms / 1000.0), "unit": "cell-updates/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms,
               "calls": reps, "mode": (f"pipelined: {E2E_LANES} buffer lanes, H2D / solve / D2H on three streams, "
                                       "calls k+1's upload and k-1's download overlap call k's V-cycle")
               if pipelined else "serial"}

    # ---------------- time to solution (V-cycles to eps, seconds) ----------------
    # the config's hierarchy (BASELINE level count) and the full-depth one
    # (coarsest 4^d: the coarsest-level 10-sweep solve is what limits the
    # config's convergence factor)
    tts = None
    if slab is None and not args.no_tts:
        tts = {"config_levels": time_to_solution(nso, spec, w, v0, vstar, w.levels, args.tts_budget),
               "full_depth": time_to_solution(nso, spec, w, v0, vstar, 99, args.tts_budget)}

    cpu = None
    if rank == 0 and slab is None and not args.no_cpu:
        try:
            rate, sec, sh, nt = cpu_vcycle_rate(w, 1)
            cpu = {"value": rate, "unit": "cell-updates/s", "cores": nt, "kind": "port",
                   "same_config": sh["same_config"], "sample": cpu_sample_text(w, sh, nt, sec)}
        except Exception as ex:  # never fail the GPU line on the CPU leg
            cpu = {"value": None, "unit": "cell-updates/s", "cores": 1, "kind": "port", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": "STFAS spacetime cell-updates/s (per V-cycle)",
            "value": value, "unit": "cell-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "s_per_vcycle": ms / 1000.0,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if w.dtype == torch.float32 else "f64", "data": "synthetic",
            "config": {"workload": w.name, "config_index": w.index, "grid": f"{w.n}^{w.dim}", "frames": w.N,
                       "levels": hier.levels, "cell_timesteps": w.cell_timesteps,
                       "parallelism": (f"time-slabs x{world}" if world > 1 else
                                       f"time-slabs x{n_slabs} in-process" if slab is not None else "single"),
                       "l2": "flushed" if flush is not None else "inputs larger than L2",
                       "residual_inf_after": ri},
            "roofline": {"bound": "hbm", "kernel": f"{kname} (level 0)", "achieved": k_achieved, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": k_achieved / hbm,
                         "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_gbs": (traffic["bytes_per_launch"] / (k_avg_ms / 1000.0) / 1e9) if traffic else None,
                         "traffic_frac": (traffic["bytes_per_launch"] / (k_avg_ms / 1000.0) / 1e9 / hbm)
                         if traffic else None,
                         "traffic_source": traffic["source"] if traffic else None,
                         "algorithmic_bytes_per_launch": k_bytes_launch, "avg_launch_ms": k_avg_ms,
                         "launches": k_n, "share_of_step": (k_ms / prof_steps) / ms if ms else None},
            "kernels": kernels,
            "vcycle_hbm": {"achieved_per_gpu": vc_gbs, "peak": hbm, "unit": "GB/s", "frac": vc_gbs / hbm,
                           "algorithmic_bytes": vc_bytes},
            "e2e": e2e,
            "time_to_solution": tts,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    hier.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
