"""SPEC.md:474-518 (cli_io) on the host: SMKF field files, PGM keyframes,
the run-config format and the CLI surface that needs no device."""

import json
import os

import numpy as np
import pytest

from paper_1608_01102_b200 import cli, fileio
from paper_1608_01102_b200.errors import FormatError, SpecMismatch
from paper_1608_01102_b200.fields import GridSpec


@pytest.mark.parametrize("dim,bnd", [(2, "neumann"), (3, "periodic")])
def test_smkf_round_trip_bitwise(tmp_path, dim, bnd):
    res = (6, 5) if dim == 2 else (4, 6, 5)
    spec = GridSpec(dim, res, 0.125, bnd)
    rng = np.random.default_rng(1)
    cell = rng.standard_normal(res)
    face = tuple(rng.standard_normal(spec.face_shape(k)) for k in range(dim))
    p1, p2 = tmp_path / "c.smkf", tmp_path / "f.smkf"
    fileio.save_smkf(p1, spec, cell)
    fileio.save_smkf(p2, spec, face)
    s, kind, back = fileio.read_smkf(p1)
    assert kind == fileio.KIND_CELL and back.tobytes() == cell.tobytes()
    assert (s.dim, tuple(s.res), s.h, s.boundary) == (dim, res, 0.125, bnd)
    _, kind, fb = fileio.read_smkf(p2)
    assert kind == fileio.KIND_FACE and all(a.tobytes() == b.tobytes() for a, b in zip(fb, face))
    # save -> load -> save is byte-identical
    fileio.save_smkf(tmp_path / "c2.smkf", spec, fileio.load_smkf(p1, spec))
    assert open(p1, "rb").read() == open(tmp_path / "c2.smkf", "rb").read()


def test_smkf_errors(tmp_path):
    spec = GridSpec(2, (4, 4), 0.25, "neumann")
    p = tmp_path / "a.smkf"
    fileio.save_smkf(p, spec, np.zeros((4, 4)))
    with pytest.raises(SpecMismatch):
        fileio.load_smkf(p, GridSpec(2, (8, 8), 0.125, "neumann"))
    with pytest.raises(SpecMismatch):
        fileio.save_smkf(p, spec, np.zeros((4, 5)))
    raw = open(p, "rb").read()
    (tmp_path / "bad.smkf").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(FormatError):
        fileio.read_smkf(tmp_path / "bad.smkf")
    (tmp_path / "short.smkf").write_bytes(raw[:-8])
    with pytest.raises(FormatError):
        fileio.read_smkf(tmp_path / "short.smkf")


def _pgm(path, w, h, value):
    with open(path, "wb") as f:
        f.write(b"P5\n# comment\n%d %d\n255\n" % (w, h))
        f.write(bytes([value]) * (w * h))


def test_pgm_keyframes(tmp_path):
    """all-black -> zero, all-white 128^2 onto 64^2 -> 1.0."""
    spec = GridSpec(2, (64, 64), 1 / 64, "neumann")
    _pgm(tmp_path / "black.pgm", 32, 32, 0)
    _pgm(tmp_path / "white.pgm", 128, 128, 255)
    assert np.all(fileio.load_keyframe(tmp_path / "black.pgm", spec) == 0.0)
    w = fileio.load_keyframe(tmp_path / "white.pgm", spec)
    assert w.shape == (64, 64) and np.all(w == 1.0)
    with pytest.raises(FormatError):
        fileio.load_keyframe(tmp_path / "white.pgm", GridSpec(3, (8, 8, 8), 1 / 8, "neumann"))


def test_pgm_orientation_and_resample(tmp_path):
    # a ramp along x written and read back; then resampled 2x up is monotone
    spec = GridSpec(2, (8, 4), 1 / 8, "neumann")
    a = np.repeat(np.linspace(0, 1, 8)[:, None], 4, axis=1)
    fileio.write_pgm(tmp_path / "r.pgm", a)
    b = fileio.read_pgm(tmp_path / "r.pgm")
    assert b.shape == (8, 4) and np.max(np.abs(a - b)) <= 0.5 / 255 + 1e-12
    up = fileio.resample(b, (16, 8))
    assert np.all(np.diff(up[:, 0]) >= 0) and np.isclose(up.min(), 0) and np.isclose(up.max(), 1)
    assert fileio.load_keyframe(tmp_path / "r.pgm", spec).shape == (8, 4)


def test_run_config_round_trip(tmp_path):
    cfg = fileio.RunConfig(dim=3, res=(16, 16, 8), frames=12, K=10.0, r=1e-3, fallback=True, eps_admm=0.01,
                           keyframes={12: "k12.smkf", 6: "k6.smkf"})
    t = cfg.dumps()
    back = fileio.RunConfig.loads(t)
    assert back == cfg and back.dumps() == t
    with pytest.raises(FormatError):
        fileio.RunConfig.loads("[grid]\nnope = 1\n")
    with pytest.raises(FormatError):
        fileio.RunConfig.loads("dim = 2\n")
    (tmp_path / "c.cfg").write_text(t)
    with pytest.raises(FormatError):    # keyframe files missing
        fileio.RunConfig.load(tmp_path / "c.cfg")


def test_make_benchmark_deterministic(tmp_path, capsys):
    for name in cli.BENCHMARKS:
        for rep in range(2):
            out = tmp_path / f"{name}{rep}"
            assert cli.main(["make-benchmark", "--name", name, "--res", "32", "--frames", "10",
                             "--out", str(out)]) == 0
        cfg = fileio.RunConfig.load(tmp_path / f"{name}0" / "run.cfg")
        assert cfg.frames == 10 and cfg.keyframes
        for f in os.listdir(tmp_path / f"{name}0"):
            assert open(tmp_path / f"{name}0" / f, "rb").read() == open(tmp_path / f"{name}1" / f, "rb").read()


def test_export_frames(tmp_path, capsys):
    spec = GridSpec(3, (8, 8, 6), 1 / 8, "neumann")
    for i in range(3):
        fileio.save_smkf(tmp_path / f"rho_{i:04d}.smkf", spec, np.full((8, 8, 6), i / 2))
    assert cli.main(["export-frames", "--in", str(tmp_path), "--out", str(tmp_path / "pgm")]) == 0
    names = sorted(os.listdir(tmp_path / "pgm"))
    assert names == ["rho_0000.pgm", "rho_0001.pgm", "rho_0002.pgm"]
    assert np.allclose(fileio.read_pgm(tmp_path / "pgm" / "rho_0002.pgm"), 1.0)


def test_cli_usage_and_errors(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["frobnicate"])
    assert e.value.code == 2
    assert "usage" in capsys.readouterr().err
    rc = cli.main(["optimize", "--config", str(tmp_path / "missing.cfg"), "--out", str(tmp_path / "o")])
    assert rc == 1
    err = json.loads(capsys.readouterr().err.strip().splitlines()[-1])
    assert err["error"] in ("FileNotFoundError", "FormatError")
