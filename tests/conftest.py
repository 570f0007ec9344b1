import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def load_golden(name="ref_ops.npz"):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


class GoldenCase:
    """View of one tagged case in a golden npz."""

    def __init__(self, z, tag):
        self.z = z
        self.tag = tag

    def __getitem__(self, name):
        return self.z[f"{self.tag}/{name}"]

    def has(self, name):
        return f"{self.tag}/{name}" in self.z.files

    def comps(self, name):
        out = []
        k = 0
        while self.has(f"{name}{k}"):
            out.append(self[f"{name}{k}"])
            k += 1
        return tuple(out)

    def grid(self):
        from oracle.grid import Grid
        meta = self["meta"]
        dim = int(meta[0])
        res = tuple(int(r) for r in meta[1:1 + dim])
        return Grid(dim, res, float(self["h"]), str(self["bnd"]))


@pytest.fixture(scope="session")
def golden():
    return load_golden()


def rel_err(a, b):
    if isinstance(a, tuple):
        num = max(float(np.max(np.abs(x - y))) if x.size else 0.0 for x, y in zip(a, b))
        den = max(float(np.max(np.abs(y))) if y.size else 0.0 for y in b)
    else:
        num = float(np.max(np.abs(a - b))) if a.size else 0.0
        den = float(np.max(np.abs(b))) if b.size else 0.0
    return num / max(den, 1e-300)


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
