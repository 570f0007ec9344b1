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
