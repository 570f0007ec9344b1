"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/smk.h declares (no compute calls: there may be no GPU here)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "smk.h")
LIB = os.path.join(ROOT, "paper_1608_01102_b200", "libsmk.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(smk_[A-Za-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_entry_points():
    names = declared()
    for must in ["smk_div", "smk_grad", "smk_advect", "smk_advect_v_T", "smk_self_adv_jac_T", "smk_sim_step",
                 "smk_kkt_residual", "smk_scgs_sweep", "smk_nso_create", "smk_nso_vcycle", "smk_nso_solve"]:
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libsmk.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libsmk.so not built")
def test_python_binding_matches_header():
    from paper_1608_01102_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared())
    L = _lib.load()
    assert L.smk_version() >= 1


def test_product_path_has_no_cpu_fallback():
    """Without a device the product raises instead of computing on the CPU."""
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1608_01102_b200 import fields
    from paper_1608_01102_b200.errors import ExtensionMissing
    s = fields.GridSpec(2, (8, 8), 0.125)
    with pytest.raises(ExtensionMissing):
        fields.divergence_arrays(s, (np.zeros((9, 8)), np.zeros((8, 9))))


@pytest.mark.skipif(not os.path.exists(LIB), reason="libsmk.so not built")
@pytest.mark.parametrize("res,bnd,rb,mod,ok", [
    ((10, 10), 1, 1, 2, True),     # even periodic: red-black fine (coarsening stops before 5^2)
    ((10, 9), 1, 1, 2, False),     # odd periodic extent: wrap neighbours share a colour
    ((12, 9), 0, 1, 2, False),     # red-black needs an even last-axis extent
    ((12, 9), 0, 0, 2, True),      # mod-2 on a Neumann odd extent is fine
    ((9, 12), 1, 0, 3, True),      # mod-3 on periodic multiples of 3
    ((10, 12), 1, 0, 3, False),    # periodic 10 is not a multiple of 3
])
def test_nso_create_rejects_uncolourable_grids(res, bnd, rb, mod, ok):
    """a colouring whose same-colour cells share a face (odd
    periodic extents) is rejected before any device work."""
    from paper_1608_01102_b200 import _lib
    L = _lib.load()
    g = _lib.smk_grid()
    g.dim = 2
    g.res[0], g.res[1] = res
    g.h = 1.0 / res[0]
    g.boundary = bnd
    g.dtype = _lib.SMK_F64
    p = _lib.smk_nso_params()
    p.n_frames, p.n_levels, p.dt, p.K, p.r, p.omega = 2, 3, 0.5, 1e3, 1e3, 0.8
    p.nu1 = p.nu2 = 2
    p.n_coarse = 10
    p.color_mod = mod
    p.red_black = rb
    h = L.smk_nso_create(ctypes.byref(g), ctypes.byref(p))
    if ok:
        if h:   # only reachable with a device (allocation follows the checks)
            L.smk_nso_destroy(h)
        else:
            assert "colour" not in _lib.last_error() and "periodic" not in _lib.last_error()
    else:
        assert not h
        msg = _lib.last_error()
        assert "colour" in msg or "periodic" in msg, msg
