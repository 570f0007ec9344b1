"""Memory / race hygiene of the colour-pass kernels on the B200.

compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing
a reset; profiles/r02h_sanitizer.txt), so its checks are stood in for by:

* racecheck / synccheck: every launch shape is run repeatedly on the same
  input and must be bitwise identical (a shared-memory ring hazard or a
  missing barrier makes the producer / consumer exchange order-dependent);
* initcheck: the smoother's hand-off and delta buffers start as NaN
  (SMK_POISON=1) -- reading an entry that no kernel of the pass wrote
  propagates a NaN, so the results must equal the zero-initialised run bitwise;
* memcheck (writes): the state arrays are carved out of one buffer with
  canary gaps between and around them; a V-cycle, the stop test and a 2-slab
  C++ slab V-cycle must leave every canary intact.
"""

import numpy as np
import pytest
import torch

from problems import make_problem

pytestmark = pytest.mark.gpu

SHAPES = [("tm64p1-cmp", "0,0", "0", "1"), ("tm64p1-fact", "0,0", str(1 << 40), "1"),
          ("tm32p2", "1000000000,0", str(1 << 40), "1"), ("tm32p4-rec", "1000000000,1000000000", str(1 << 40), "1"),
          ("tm32p4-fact", "1000000000,1000000000", str(1 << 40), "0")]


@pytest.fixture(scope="module")
def nso():
    from paper_1608_01102_b200 import _lib, nso
    _lib.load()
    return nso


def spec_of(pb):
    from paper_1608_01102_b200.fields import GridSpec
    g = pb.g
    return GridSpec(g.dim, g.res, g.h, g.boundary)


def run_vcycle(nso, pb, dtype, levels=2):
    spec = spec_of(pb)
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=levels)
    h = nso.StfasHierarchy(spec, cfg, pb.N, dtype)
    h.set_guide(pb.v0, pb.vstar)
    s = nso.SpacetimeState.zeros(spec, pb.N, dtype)
    h.vcycle(s)
    h.vcycle(s)
    ri = h.residual_norms(s)
    torch.cuda.synchronize()
    h.close()
    return np.concatenate([np.asarray(a).ravel() for a in s.numpy()[0] + (s.numpy()[1],) + s.numpy()[2] +
                           (s.numpy()[3],)]), ri


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("shape", SHAPES, ids=[s[0] for s in SHAPES])
def test_shapes_deterministic_and_poison_clean(nso, monkeypatch, shape, dtype):
    name, fwd, bf, deep = shape
    monkeypatch.setenv("SMK_FWD_THRESH", fwd)
    monkeypatch.setenv("SMK_BACK_FLAT", bf)
    monkeypatch.setenv("SMK_BACK_DEEP", deep)
    monkeypatch.setenv("SMK_NO_GRAPH", "1")
    # 3D 32^3 x 6: 16,384 colour cells, many CTAs per SM on every shape;
    # tm64p1-cmp also at 48^3 (55,296 colour cells: the TMA-staged fused
    # backward, which needs 128-cell CTAs and a multiple of 128 cells)
    pb = make_problem(3, n=48 if name == "tm64p1-cmp" else 32, N=6, seed=61)
    ref, ri = run_vcycle(nso, pb, dtype)
    assert np.all(np.isfinite(ref))
    for _ in range(2):
        again, ri2 = run_vcycle(nso, pb, dtype)
        assert np.array_equal(again, ref), f"{name}: nondeterministic result"
        assert ri2 == ri
    monkeypatch.setenv("SMK_POISON", "1")
    poisoned, ri3 = run_vcycle(nso, pb, dtype)
    assert np.array_equal(poisoned, ref), f"{name}: result depends on unwritten scratch"
    assert ri3 == ri


def carve(total, sizes, dtype, canary):
    """One device buffer holding arrays of the given element counts with 1 KiB
    canary gaps before, between and after them."""
    gap = 1024 // torch.tensor([], dtype=dtype).element_size()
    buf = torch.full((total + gap * (len(sizes) + 1),), canary, dtype=dtype, device="cuda")
    views, gaps, off = [], [], gap
    gaps.append((0, gap))
    for n in sizes:
        views.append(buf[off:off + n])
        views[-1].zero_()
        off += n
        gaps.append((off, off + gap))
        off += gap
    return buf, views, gaps


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_no_writes_outside_the_state(nso, dim, dtype):
    from paper_1608_01102_b200 import slabs
    pb = make_problem(dim, n=16 if dim == 2 else 8, N=5, seed=62)
    spec = spec_of(pb)
    g = pb.g
    fshape = [(pb.N,) + g.face_shape(k) for k in range(dim)]
    cshape = (pb.N,) + g.res
    shapes = fshape + [cshape] + fshape + [cshape]
    sizes = [int(np.prod(s)) for s in shapes]
    canary = 7.25
    buf, views, gaps = carve(sum(sizes), sizes, dtype, canary)
    arrs = [v.view(s) for v, s in zip(views, shapes)]
    st = nso.SpacetimeState(tuple(arrs[:dim]), arrs[dim], tuple(arrs[dim + 1:2 * dim + 1]), arrs[2 * dim + 1])
    cfg = nso.StfasConfig(dt=pb.dt, K=pb.K, r=pb.r, n_levels=2)
    h = nso.StfasHierarchy(spec, cfg, pb.N, dtype)
    h.set_guide(pb.v0, pb.vstar)
    h.vcycle(st)
    h.gauge_fix(st)
    h.residual_norms(st)
    torch.cuda.synchronize()
    h.close()
    host = buf.cpu().numpy()
    for a, b in gaps:
        assert np.all(host[a:b] == canary), "hierarchy wrote outside the state arrays"
    # the C++ slab set on carved per-slab states
    cs = slabs.CSlabSolver(spec, cfg, pb.v0, pb.vstar, [0, 1], 2, pb.N, dtype)
    sts, bufs = [], []
    for t0, n in cs.frames:
        shp = [(n,) + g.face_shape(k) for k in range(dim)] + [(n,) + g.res]
        shp = shp[:dim] + [shp[dim]] + shp[:dim] + [shp[dim]]
        sz = [int(np.prod(s)) for s in shp]
        b, vv, gp = carve(sum(sz), sz, dtype, canary)
        a = [v.view(s) for v, s in zip(vv, shp)]
        sts.append(nso.SpacetimeState(tuple(a[:dim]), a[dim], tuple(a[dim + 1:2 * dim + 1]), a[2 * dim + 1]))
        bufs.append((b, gp))
    cs.vcycle(sts)
    cs.gauge(sts)
    cs.norms(sts)
    torch.cuda.synchronize()
    cs.close()
    for b, gp in bufs:
        host = b.cpu().numpy()
        for a, c in gp:
            assert np.all(host[a:c] == canary), "slab set wrote outside the state arrays"
