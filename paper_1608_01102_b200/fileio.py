"""Files of the CLI (SPEC.md:474-518 cli_io; SMKF field format SPEC.md:80).

* SMKF raw field files: little-endian header -- magic ``SMKF``, int32 dim,
  int32 res[dim], float64 h, int32 boundary code (0 Neumann, 1 periodic),
  int32 field kind (0 cell scalar, 1 staggered face vector) -- followed by
  the float64 payload in row-major (C) order; a face vector stores its dim
  components one after the other, component k in its face shape
  ``GridSpec.face_shape(k)``.  save -> load is bitwise.
* ``load_keyframe``: 8-bit grayscale PGM (P5, or P2 text;
  2D only) mapped linearly to [0, 1] and resampled onto the grid by
  multilinear interpolation at the cell centres, or an SMKF scalar field
  loaded verbatim with spec equality enforced.  Image x (columns) runs along
  axis 0, image rows from the top run down axis 1.
* ``RunConfig``: flat UTF-8 ``key = value`` text in
  ``[sections]``; parse -> serialise -> parse is the identity.

Host-side plumbing: numpy in / numpy out (the fields are read back from the
device by the caller).
"""

import os
import struct
from dataclasses import dataclass, field, fields

import numpy as np

from .errors import FormatError, SpecMismatch
from .fields import GridSpec

MAGIC = b"SMKF"
KIND_CELL, KIND_FACE = 0, 1
_BND = {"neumann": 0, "periodic": 1}
_BND_INV = {v: k for k, v in _BND.items()}


def _np(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().double().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------------------
# SMKF
# ---------------------------------------------------------------------------


def save_smkf(path, spec, values):
    """Write a cell scalar (array of shape spec.res) or a face vector (tuple
    of dim arrays of the face shapes) as one SMKF file."""
    if isinstance(values, (tuple, list)):
        kind = KIND_FACE
        comps = [_np(c) for c in values]
        if len(comps) != spec.dim:
            raise SpecMismatch(f"face vector needs {spec.dim} components, got {len(comps)}")
        for k, c in enumerate(comps):
            if c.shape != tuple(spec.face_shape(k)):
                raise SpecMismatch(f"component {k} shape {c.shape} != {spec.face_shape(k)}")
        payload = b"".join(np.ascontiguousarray(c, dtype="<f8").tobytes() for c in comps)
    else:
        kind = KIND_CELL
        a = _np(values)
        if a.shape != tuple(spec.res):
            raise SpecMismatch(f"scalar shape {a.shape} != res {spec.res}")
        payload = np.ascontiguousarray(a, dtype="<f8").tobytes()
    head = MAGIC + struct.pack("<i", spec.dim) + struct.pack(f"<{spec.dim}i", *spec.res)
    head += struct.pack("<d", float(spec.h)) + struct.pack("<ii", _BND[spec.boundary], kind)
    with open(path, "wb") as f:
        f.write(head + payload)


def read_smkf(path):
    """(GridSpec, kind, values) of an SMKF file; raises FormatError."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != MAGIC:
        raise FormatError(f"{path}: not an SMKF file (magic {raw[:4]!r})")
    try:
        off = 4
        (dim,) = struct.unpack_from("<i", raw, off)
        off += 4
        if dim not in (2, 3):
            raise FormatError(f"{path}: bad dim {dim}")
        res = struct.unpack_from(f"<{dim}i", raw, off)
        off += 4 * dim
        (h,) = struct.unpack_from("<d", raw, off)
        off += 8
        bnd, kind = struct.unpack_from("<ii", raw, off)
        off += 8
    except struct.error as e:
        raise FormatError(f"{path}: truncated header ({e})") from None
    if bnd not in _BND_INV or kind not in (KIND_CELL, KIND_FACE):
        raise FormatError(f"{path}: bad boundary / kind code ({bnd}, {kind})")
    spec = GridSpec(dim, tuple(res), h, _BND_INV[bnd])
    body = raw[off:]
    if kind == KIND_CELL:
        n = int(np.prod(res))
        if len(body) != 8 * n:
            raise FormatError(f"{path}: payload {len(body)} bytes, expected {8 * n}")
        return spec, kind, np.frombuffer(body, dtype="<f8").reshape(res).astype(np.float64)
    comps, o = [], 0
    for k in range(dim):
        shp = tuple(spec.face_shape(k))
        n = int(np.prod(shp))
        if len(body) < o + 8 * n:
            raise FormatError(f"{path}: face payload truncated")
        comps.append(np.frombuffer(body[o:o + 8 * n], dtype="<f8").reshape(shp).astype(np.float64))
        o += 8 * n
    if o != len(body):
        raise FormatError(f"{path}: {len(body) - o} trailing bytes")
    return spec, kind, tuple(comps)


def load_smkf(path, spec=None):
    """Values of an SMKF file; with `spec`, the file's grid must equal it."""
    s, _, vals = read_smkf(path)
    if spec is not None and (s.dim, tuple(s.res), float(s.h), s.boundary) != \
            (spec.dim, tuple(spec.res), float(spec.h), spec.boundary):
        raise SpecMismatch(f"{path}: grid {s.dim}D {s.res} h={s.h} {s.boundary} != "
                           f"{spec.dim}D {spec.res} h={spec.h} {spec.boundary}")
    return vals


# ---------------------------------------------------------------------------
# PGM
# ---------------------------------------------------------------------------


def _pgm_tokens(raw):
    """Header tokens of a PGM (comments skipped) and the payload offset."""
    toks, i, n = [], 0, len(raw)
    while len(toks) < 4:
        while i < n and raw[i:i + 1].isspace():
            i += 1
        if i < n and raw[i:i + 1] == b"#":
            while i < n and raw[i:i + 1] not in (b"\n", b"\r"):
                i += 1
            continue
        j = i
        while j < n and not raw[j:j + 1].isspace():
            j += 1
        if j == i:
            raise FormatError("truncated PGM header")
        toks.append(raw[i:j])
        i = j
    return toks, i + 1


def read_pgm(path):
    """8-bit PGM -> float array in [0, 1], indexed [x, y] (x = column,
    y = 0 at the bottom row)."""
    with open(path, "rb") as f:
        raw = f.read()
    try:
        toks, off = _pgm_tokens(raw)
        magic, w, hgt, mx = toks[0], int(toks[1]), int(toks[2]), int(toks[3])
    except (ValueError, IndexError, FormatError) as e:
        raise FormatError(f"{path}: bad PGM header ({e})") from None
    if not (0 < mx <= 255) or w <= 0 or hgt <= 0:
        raise FormatError(f"{path}: only 8-bit PGM is supported (maxval {mx})")
    if magic == b"P5":
        data = np.frombuffer(raw[off:off + w * hgt], dtype=np.uint8)
        if data.size != w * hgt:
            raise FormatError(f"{path}: PGM payload truncated")
    elif magic == b"P2":
        try:
            data = np.array([int(t) for t in raw[off:].split()[:w * hgt]], dtype=np.int64)
        except ValueError:
            raise FormatError(f"{path}: bad P2 payload") from None
        if data.size != w * hgt:
            raise FormatError(f"{path}: PGM payload truncated")
    else:
        raise FormatError(f"{path}: not a PGM (magic {magic!r})")
    img = data.reshape(hgt, w).astype(np.float64) / mx          # [row, col]
    return np.ascontiguousarray(img[::-1, :].T)                 # [x, y], y up


def write_pgm(path, values):
    """2D array indexed [x, y] -> binary PGM, clamp(values, 0, 1) * 255."""
    a = np.clip(_np(values), 0.0, 1.0)
    img = np.round(a.T[::-1, :] * 255.0).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0]))
        f.write(img.tobytes())


def resample(a, shape):
    """Multilinear resampling at cell centres (clamped at the borders)."""
    out = np.asarray(a, dtype=np.float64)
    for ax, n in enumerate(shape):
        m = out.shape[ax]
        if m == n:
            continue
        pos = np.clip((np.arange(n) + 0.5) * m / n - 0.5, 0.0, m - 1)
        i0 = np.floor(pos).astype(int)
        i1 = np.minimum(i0 + 1, m - 1)
        w = pos - i0
        sh = [1] * out.ndim
        sh[ax] = n
        out = np.take(out, i0, axis=ax) * (1 - w).reshape(sh) + np.take(out, i1, axis=ax) * w.reshape(sh)
    return out


def load_keyframe(path, spec):
    """PGM (2D) or SMKF scalar field onto `spec`."""
    with open(path, "rb") as f:
        head = f.read(4)
    if head == MAGIC:
        s, kind, vals = read_smkf(path)
        if kind != KIND_CELL:
            raise FormatError(f"{path}: keyframe must be a cell scalar field")
        return load_smkf(path, spec)
    if head[:2] in (b"P5", b"P2"):
        if spec.dim != 2:
            raise FormatError(f"{path}: 3D keyframes are SMKF only (SPEC.md:515)")
        return resample(read_pgm(path), spec.res)
    raise FormatError(f"{path}: neither PGM nor SMKF")


# ---------------------------------------------------------------------------
# run configuration
# ---------------------------------------------------------------------------


@dataclass
class RunConfig:
    """SPEC.md:478-481.  Paths are relative to the config file's directory."""

    dim: int = 2
    res: tuple = (32, 32)
    h: float = None                 # None -> 1 / res[0]
    boundary: str = "neumann"
    dt: float = None                # None -> 1 / frames
    frames: int = 16
    initial_density: str = "initial.smkf"
    keyframes: dict = field(default_factory=dict)   # timestep -> path
    K: float = 1e3
    r: float = 1e3
    beta: float = 1.0
    ao_iters: int = 2
    eps_stfas: float = 1e-5
    eps_admm: float = None
    max_outer: int = 60
    fallback: bool = False
    safeguard: bool = False
    lm: bool = False
    n_levels: int = 99
    solver: str = "admm"            # admm | lbfgs
    threads: int = 1
    seed: int = 0
    dtype: str = "float64"

    SECTIONS = {"grid": ("dim", "res", "h", "boundary"), "time": ("dt", "frames"),
                "input": ("initial_density",), "admm": ("K", "r", "beta", "ao_iters", "eps_stfas", "eps_admm",
                                                       "max_outer", "fallback", "safeguard", "lm", "n_levels"),
                "run": ("solver", "threads", "seed", "dtype")}

    def spec(self):
        return GridSpec(self.dim, tuple(self.res), self.h if self.h else 1.0 / self.res[0], self.boundary)

    def timestep(self):
        return self.dt if self.dt else 1.0 / self.frames

    def validate(self, base_dir=None):
        if self.dim not in (2, 3) or len(self.res) != self.dim:
            raise FormatError("grid: dim must be 2 or 3 with dim res entries")
        if self.boundary not in _BND:
            raise FormatError(f"grid: unknown boundary {self.boundary!r}")
        if self.solver not in ("admm", "lbfgs"):
            raise FormatError(f"run: solver must be admm or lbfgs, got {self.solver!r}")
        for t, p in self.keyframes.items():
            if not 1 <= int(t) <= self.frames:
                raise FormatError(f"keyframe timestep {t} outside [1, {self.frames}]")
            if base_dir is not None and not os.path.exists(os.path.join(base_dir, p)):
                raise FormatError(f"keyframe file {p} not found")

    # ---- text form ----
    def dumps(self):
        out = []
        for sec, keys in self.SECTIONS.items():
            out.append(f"[{sec}]")
            for k in keys:
                v = getattr(self, k)
                if v is None:
                    continue
                out.append(f"{k} = {_fmt(v)}")
            out.append("")
        out.append("[keyframes]")
        for t in sorted(self.keyframes, key=int):
            out.append(f"{int(t)} = {self.keyframes[t]}")
        return "\n".join(out) + "\n"

    @classmethod
    def loads(cls, text):
        cfg = cls()
        cfg.keyframes = {}
        types = {f.name: f.type for f in fields(cls)}
        sec = None
        for ln, line in enumerate(text.splitlines(), 1):
            s = line.split("#", 1)[0].strip()
            if not s:
                continue
            if s.startswith("[") and s.endswith("]"):
                sec = s[1:-1].strip()
                if sec not in cls.SECTIONS and sec != "keyframes":
                    raise FormatError(f"line {ln}: unknown section [{sec}]")
                continue
            if "=" not in s or sec is None:
                raise FormatError(f"line {ln}: expected key = value inside a section")
            k, v = (x.strip() for x in s.split("=", 1))
            if sec == "keyframes":
                try:
                    cfg.keyframes[int(k)] = v
                except ValueError:
                    raise FormatError(f"line {ln}: keyframe key must be a timestep") from None
                continue
            if k not in cls.SECTIONS[sec]:
                raise FormatError(f"line {ln}: unknown key {k!r} in [{sec}]")
            setattr(cfg, k, _parse(k, v, types[k], ln))
        return cfg

    @classmethod
    def load(cls, path):
        with open(path, encoding="utf-8") as f:
            cfg = cls.loads(f.read())
        cfg.validate(os.path.dirname(os.path.abspath(path)))
        return cfg

    def save(self, path):
        with open(path, "w", encoding="utf-8") as f:
            f.write(self.dumps())


def _fmt(v):
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (tuple, list)):
        return " ".join(str(x) for x in v)
    if isinstance(v, float):
        return repr(v)
    return str(v)


def _parse(k, v, typ, ln):
    try:
        if k == "res":
            return tuple(int(x) for x in v.split())
        if typ in (bool, "bool"):
            if v.lower() not in ("true", "false", "1", "0", "yes", "no"):
                raise ValueError(v)
            return v.lower() in ("true", "1", "yes")
        if typ in (int, "int"):
            return int(v)
        if typ in (float, "float"):
            return float(v)
        if k in ("h", "dt", "eps_admm"):
            return float(v)
        return v
    except ValueError:
        raise FormatError(f"line {ln}: bad value {v!r} for {k}") from None
