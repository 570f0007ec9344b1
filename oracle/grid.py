"""MAC grid metadata for the oracle (TEST INFRASTRUCTURE ONLY).

Restates ``GridSpec`` (``pkg/src/smokectrl/fields.py:37-89``): ``res`` cells
per axis, uniform ``h``, boundary ``"neumann"`` (face arrays carry ``res+1``
entries along their normal axis, walls pinned to zero) or ``"periodic"``.
"""

from dataclasses import dataclass

NEUMANN = "neumann"
PERIODIC = "periodic"


@dataclass(frozen=True)
class Grid:
    dim: int
    res: tuple
    h: float
    boundary: str = NEUMANN

    def __post_init__(self):
        object.__setattr__(self, "res", tuple(int(r) for r in self.res))
        if self.dim not in (2, 3) or len(self.res) != self.dim:
            raise ValueError("bad dim/res")
        if min(self.res) < 4:
            raise ValueError("res components must be >= 4")
        if not self.h > 0:
            raise ValueError("h must be positive")
        if self.boundary not in (NEUMANN, PERIODIC):
            raise ValueError("bad boundary")

    @property
    def periodic(self):
        return self.boundary == PERIODIC

    @property
    def n_cells(self):
        n = 1
        for r in self.res:
            n *= r
        return n

    def face_shape(self, k):
        # fields.py:74-79
        return tuple(r + (0 if (self.periodic or a != k) else 1)
                     for a, r in enumerate(self.res))

    def coarsen(self):
        # fields.py:84-89: halve while every axis stays even and >= 4 after
        if any(r % 2 or r // 2 < 4 for r in self.res):
            return None
        return Grid(self.dim, tuple(r // 2 for r in self.res), 2.0 * self.h,
                    self.boundary)

    def hierarchy(self, levels=None):
        out = [self]
        while (levels is None or len(out) < levels) and out[-1].coarsen():
            out.append(out[-1].coarsen())
        return out
