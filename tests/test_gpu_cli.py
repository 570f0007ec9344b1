"""CLI end to end on the B200 and the SPEC.md:529 memory
bound through the memtrack drop-in."""

import json
import os

import numpy as np
import pytest
import torch

from paper_1608_01102_b200 import cli, fileio

pytestmark = pytest.mark.gpu


def test_optimize_translated_blob_writes_frames_and_logs(tmp_path, capsys):
    """optimize on make-benchmark's translated blob 32^2 / N = 10
    exits 0 and writes N + 1 density frames plus logs; re-running reproduces
    bit-identical field files."""
    b = tmp_path / "bench"
    assert cli.main(["make-benchmark", "--name", "translated-blob", "--res", "32", "--frames", "10",
                     "--out", str(b)]) == 0
    outs = []
    for rep in range(2):
        o = tmp_path / f"out{rep}"
        rc = cli.main(["optimize", "--config", str(b / "run.cfg"), "--out", str(o)])
        assert rc == 0, capsys.readouterr().err
        outs.append(o)
    names = sorted(os.listdir(outs[0]))
    assert sum(n.startswith("rho_") for n in names) == 11
    assert sum(n.startswith("u_") for n in names) == 10
    assert {"admm_log.csv", "vcycle_log.csv", "result.json"} <= set(names)
    res = json.load(open(outs[0] / "result.json"))
    assert res["converged"] and res["outer_iterations"] >= 1
    for n in names:
        if n.endswith(".smkf"):
            assert open(outs[0] / n, "rb").read() == open(outs[1] / n, "rb").read(), n
    rows = open(outs[0] / "admm_log.csv").read().splitlines()
    assert rows[0] == "outer_iter,ao_obj,nso_resid,visual_diff,wall_s" and len(rows) >= 2


def test_simulate_rest_state_reproduces_density(tmp_path, capsys):
    """zero forces and zero initial velocity reproduce the
    initial density in every exported frame."""
    b = tmp_path / "bench"
    assert cli.main(["make-benchmark", "--name", "circle-letter", "--res", "32", "--frames", "6",
                     "--out", str(b)]) == 0
    assert cli.main(["simulate", "--config", str(b / "run.cfg"), "--out", str(tmp_path / "sim")]) == 0
    rho0 = fileio.load_smkf(b / "initial.smkf")
    frames = sorted(f for f in os.listdir(tmp_path / "sim") if f.startswith("rho_"))
    assert len(frames) == 7
    for f in frames:
        assert np.array_equal(fileio.load_smkf(tmp_path / "sim" / f), rho0), f
    assert cli.main(["export-frames", "--in", str(tmp_path / "sim"), "--out", str(tmp_path / "pgm")]) == 0
    assert len(os.listdir(tmp_path / "pgm")) == 7


@pytest.mark.parametrize("dim,n,N", [(2, 32, 16), (3, 16, 8)])
def test_solve_nso_payload_memory_bound(dim, n, N):
    """SPEC.md:529 (PAPER §5 'analytical upper bound'): peak field payload
    during solve_nso <= 1.5 * 8 n^d (1 + d) N values (32^2 / N = 16 is the
    SPEC's case; 16^3 / N = 8 the 3D analogue)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
    from problems import make_problem
    from paper_1608_01102_b200 import memtrack, nso
    from paper_1608_01102_b200.fields import GridSpec
    pb = make_problem(dim, n=n, N=N, seed=3)
    g = pb.g
    spec = GridSpec(g.dim, g.res, g.h, g.boundary)
    vstar = tuple(torch.as_tensor(c).cuda() for c in pb.vstar)
    v0 = tuple(torch.as_tensor(c).cuda() for c in pb.v0)
    with memtrack.track_payload() as stats:
        s = nso.SpacetimeState.zeros(spec, N)
        res = nso.solve_nso(spec, nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r), v0, vstar, s=s, eps=1e-5)
        hist = res.history if hasattr(res, "history") else res[1]
    bound = 1.5 * 8 * n ** dim * (1 + dim) * N
    print(f"[memtrack] {dim}D {n}^{dim} x {N}: peak {stats.peak_values} values, bound {bound:.0f} "
          f"({stats.peak_values / bound:.2f} of it), {len(hist) - 1} V-cycles")
    assert stats.peak_values > 0
    assert stats.peak_values <= bound
