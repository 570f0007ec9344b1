// Shared device machinery for the STFAS kernels (sm_100a).
//
// Layout (identical to the reference's numpy arrays, fields.py:92-133, so the
// C-ABI is a zero-copy drop-in): every field is a C-order array with an
// optional leading frame axis.  A cell field is (N, n0, n1[, n2]); face
// component k is (N, f0, f1[, f2]) with f_a = n_a + (a == k && neumann).
// 2D grids are handled as 3D with n2 == 1 and no k == 2 component, which keeps
// every offset computation identical to numpy's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

namespace smk {

struct Geo {
  int dim;
  int n[3];        // cells per axis (n[2] == 1 for 2D)
  double h;
  int periodic;
};

// ---------------------------------------------------------------------------
// index helpers (templated on DIM / periodicity so the branches fold away)
// ---------------------------------------------------------------------------

template <int DIM, bool PER>
struct Ix {
  int n0, n1, n2;
  __host__ __device__ Ix(const Geo& g) : n0(g.n[0]), n1(g.n[1]), n2(DIM == 3 ? g.n[2] : 1) {}
  __host__ __device__ __forceinline__ int n(int a) const { return a == 0 ? n0 : (a == 1 ? n1 : n2); }
  // extent of face component k along axis a
  __host__ __device__ __forceinline__ int fe(int k, int a) const { return n(a) + ((!PER && a == k) ? 1 : 0); }
  __host__ __device__ __forceinline__ int64_t cells() const { return (int64_t)n0 * n1 * n2; }
  __host__ __device__ __forceinline__ int64_t faces(int k) const {
    return (int64_t)fe(k, 0) * fe(k, 1) * (DIM == 3 ? fe(k, 2) : 1);
  }
  __host__ __device__ __forceinline__ int64_t cell_off(int i, int j, int l) const {
    return ((int64_t)i * n1 + j) * n2 + l;
  }
  __host__ __device__ __forceinline__ int64_t face_off(int k, int i, int j, int l) const {
    return ((int64_t)i * fe(k, 1) + j) * (DIM == 3 ? fe(k, 2) : 1) + l;
  }
  __host__ __device__ __forceinline__ static int wrap(int i, int n) {
    return i < 0 ? i + n : (i >= n ? i - n : i);
  }
  // bounds-checked reads: zero outside (Neumann) / wrapped (periodic)
  template <class R>
  __device__ __forceinline__ R face(const R* p, int k, int i, int j, int l) const {
    if (PER) {
      i = wrap(i, n0); j = wrap(j, n1); if (DIM == 3) l = wrap(l, n2);
    } else {
      if (i < 0 || j < 0 || l < 0 || i >= fe(k, 0) || j >= fe(k, 1) || (DIM == 3 && l >= fe(k, 2))) return R(0);
    }
    return p[face_off(k, i, j, DIM == 3 ? l : 0)];
  }
  template <class R>
  __device__ __forceinline__ R cell(const R* p, int i, int j, int l) const {
    if (PER) {
      i = wrap(i, n0); j = wrap(j, n1); if (DIM == 3) l = wrap(l, n2);
    } else {
      if (i < 0 || j < 0 || l < 0 || i >= n0 || j >= n1 || (DIM == 3 && l >= n2)) return R(0);
    }
    return p[cell_off(i, j, DIM == 3 ? l : 0)];
  }
  // decode a flat face index of component k
  __device__ __forceinline__ void face_idx(int k, int64_t o, int c[3]) const {
    int e2 = DIM == 3 ? fe(k, 2) : 1, e1 = fe(k, 1);
    c[2] = (int)(o % e2); o /= e2;
    c[1] = (int)(o % e1); o /= e1;
    c[0] = (int)o;
  }
  // 32-bit decodes for per-frame element indices (frame-major launches)
  __device__ __forceinline__ void face_idx32(int k, int o, int c[3]) const {
    int e2 = DIM == 3 ? fe(k, 2) : 1, e1 = fe(k, 1);
    c[2] = o % e2; o /= e2;
    c[1] = o % e1; o /= e1;
    c[0] = o;
  }
  __device__ __forceinline__ void cell_idx32(int o, int c[3]) const {
    c[2] = o % n2; o /= n2;
    c[1] = o % n1; o /= n1;
    c[0] = o;
  }
  __device__ __forceinline__ void cell_idx(int64_t o, int c[3]) const {
    c[2] = (int)(o % n2); o /= n2;
    c[1] = (int)(o % n1); o /= n1;
    c[0] = (int)o;
  }
  // wall face of component k at index c (never true for periodic)
  __device__ __forceinline__ bool wall(int k, const int c[3]) const {
    return !PER && (c[k] == 0 || c[k] == n(k));
  }
};

template <class R>
struct Face3 {  // per-frame pointers to the d face components
  const R* c[3];
};

// Field accessors used by the point stencils: plain memory, or a unit vector.
template <int DIM, bool PER, class R>
struct MemField {
  const Ix<DIM, PER>& ix;
  Face3<R> f;
  __device__ __forceinline__ R operator()(int k, int i, int j, int l) const { return ix.face(f.c[k], k, i, j, l); }
};

template <int DIM, bool PER, class R>
struct UnitField {  // e_{(k*, c*)}: 1 at one face (indices already canonical)
  const Ix<DIM, PER>& ix;
  int k0, i0, j0, l0;
  __device__ __forceinline__ R operator()(int k, int i, int j, int l) const {
    if (k != k0) return R(0);
    if (PER) { i = Ix<DIM, PER>::wrap(i, ix.n0); j = Ix<DIM, PER>::wrap(j, ix.n1); if (DIM == 3) l = Ix<DIM, PER>::wrap(l, ix.n2); }
    return (i == i0 && j == j0 && (DIM == 2 || l == l0)) ? R(1) : R(0);
  }
};

__device__ __forceinline__ void shift(int c[3], int a, int s, int out[3]) {
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[a] += s;
}

// ---------------------------------------------------------------------------
// Register cache of one face field around a cell c.  Every read that S(a,w)
// and J_Adv(v)^T u make at the cell's own 2d faces falls in 4 + 4(d-1)
// offsets per component a:  t e_a (t = -1..2)  and  s e_a +/- e_b
// (s = 0,1; b != a).  Slots are resolved at compile time after inlining
// (offsets relative to c are constants), so the cache lives in registers.
// ---------------------------------------------------------------------------
template <int DIM>
struct NbrSlots {
  static constexpr int NB = 4 + 4 * (DIM - 1);
  // slot of offset d (relative to c) for component a, or -1 (branch-light so
  // it folds to a constant when the offsets are compile-time)
  __host__ __device__ __forceinline__ static int slot(int a, int d0, int d1, int d2) {
    const int da = a == 0 ? d0 : (a == 1 ? d1 : d2);
    // the two other axes in increasing order
    const int b0 = a == 0 ? 1 : 0;
    const int b1 = a == 2 ? 1 : 2;
    const int e0 = b0 == 0 ? d0 : (b0 == 1 ? d1 : d2);
    const int e1 = DIM == 3 ? (b1 == 1 ? d1 : d2) : 0;
    if (DIM == 2 && d2 != 0) return -1;
    if (e0 == 0 && e1 == 0) return (da >= -1 && da <= 2) ? da + 1 : -1;
    if (da != 0 && da != 1) return -1;
    if (e1 == 0 && (e0 == 1 || e0 == -1)) return 4 + 2 * da + (e0 > 0 ? 1 : 0);
    if (DIM == 3 && e0 == 0 && (e1 == 1 || e1 == -1)) return 8 + 2 * da + (e1 > 0 ? 1 : 0);
    return -1;
  }
  __host__ __device__ __forceinline__ static void offset(int a, int sl, int d[3]) {
    d[0] = d[1] = d[2] = 0;
    if (sl < 4) { d[a] = sl - 1; return; }
    int r = sl - 4, bi = r / 4, rem = r % 4;
    int b = bi < a ? bi : bi + 1;
    d[a] = rem / 2;
    d[b] = (rem & 1) ? 1 : -1;
  }
};

// compile-time loop helper
template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// slot of (own-axis offset da of component a, offset db along axis b != a)
template <int DIM>
__host__ __device__ constexpr int nbr_slot(int a, int da, int b, int db) {
  return db == 0 ? da + 1 : 4 + 4 * (b < a ? b : b - 1) + 2 * da + (db > 0 ? 1 : 0);
}

template <int DIM, bool PER, class R>
struct NbrField {
  static constexpr int NB = NbrSlots<DIM>::NB;
  const Ix<DIM, PER>& ix;
  int c0, c1, c2;
  Face3<R> f;
  R val[DIM][NB];
  __device__ __forceinline__ NbrField(const Ix<DIM, PER>& ix_, const int c[3], const Face3<R>& f_)
      : ix(ix_), c0(c[0]), c1(c[1]), c2(c[2]), f(f_) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int sl = 0; sl < NB; ++sl) {
        int d[3];
        NbrSlots<DIM>::offset(a, sl, d);
        val[a][sl] = ix.face(f.c[a], a, c0 + d[0], c1 + d[1], c2 + d[2]);
      }
  }
  __device__ __forceinline__ R operator()(int k, int i, int j, int l) const {
    int sl = NbrSlots<DIM>::slot(k, i - c0, j - c1, DIM == 3 ? l - c2 : 0);
    if (sl < 0) return ix.face(f.c[k], k, i, j, l);   // never taken on the cell's own faces
    return val[k][sl];
  }
};

// ---------------------------------------------------------------------------
// One cell's position with cheap neighbour addressing inside a frame.
// Neumann: a face / cell read at a compile-time offset d from c is in range
// iff, per axis a, (d_a == -1 -> c_a >= 1) and (d_a == +1 across, or +2 along
// the face's own axis -> c_a <= n_a - 2); out-of-range reads are 0, like
// Ix::face / Ix::cell.  Offsets are 32-bit within a frame (a 129*128*128
// face frame is 2.1M elements); the frame base pointer carries the rest.
// Periodic: wrapped through Ix (cold path, not used by the benchmarks).
// ---------------------------------------------------------------------------
// NX > 0: the grid is a compile-time NX^3 Neumann cube, so every stencil
// offset below is an immediate (LDG [R + imm]) and only the cell's own face
// offsets are runtime values.
template <int DIM, bool PER, int NX = 0>
struct Loc {
  static_assert(NX == 0 || (DIM == 3 && !PER), "compile-time extents: 3D Neumann cubes only");
  int c[3];
  bool lo[3], hi[3];
  int of[2 * DIM];   // offsets of the cell's own faces (q = 2k + side)
  int co;            // cell offset
  __device__ __forceinline__ Loc(const Ix<DIM, PER>& ix, const int cc[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      c[a] = cc[a];
      lo[a] = cc[a] >= 1;
      hi[a] = cc[a] <= ix.n(a) - 2;
    }
    co = (int)ix.cell_off(c[0], c[1], c[2]);
#pragma unroll
    for (int k = 0; k < DIM; ++k)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        int f[3] = {c[0], c[1], c[2]};
        f[k] += s;
        if (PER && f[k] >= ix.n(k)) f[k] -= ix.n(k);
        of[2 * k + s] = (int)ix.face_off(k, f[0], f[1], f[2]);
      }
  }
  // stride of face component k along axis a (axis 2 / the 2D last axis: 1)
  __device__ __forceinline__ static int fstride(const Ix<DIM, PER>& ix, int k, int a) {
    if (a == 2) return 1;
    if (NX > 0) return a == 0 ? (NX + (k == 1)) * (NX + (k == 2)) : NX + (k == 2);
    if (DIM == 2) return a == 0 ? ix.fe(k, 1) : 1;
    return a == 0 ? ix.fe(k, 1) * ix.fe(k, 2) : ix.fe(k, 2);
  }
  __device__ __forceinline__ static int cstride(const Ix<DIM, PER>& ix, int a) {
    if (a == 2) return 1;
    if (NX > 0) return a == 0 ? NX * NX : NX;
    if (DIM == 2) return a == 0 ? ix.n1 : 1;
    return a == 0 ? ix.n1 * ix.n2 : ix.n2;
  }
  __device__ __forceinline__ bool ok(int a, int d, int up) const {
    return d < 0 ? lo[a] : (d >= up ? hi[a] : true);
  }
  template <class R>
  __device__ __forceinline__ R face(const Ix<DIM, PER>& ix, const R* __restrict__ p, int k, int d0, int d1,
                                    int d2) const {
    if (PER) return ix.face(p, k, c[0] + d0, c[1] + d1, c[2] + d2);
    bool v = ok(0, d0, k == 0 ? 2 : 1) && ok(1, d1, k == 1 ? 2 : 1) && (DIM == 2 || ok(2, d2, k == 2 ? 2 : 1));
    int o = of[2 * k] + d0 * fstride(ix, k, 0) + d1 * fstride(ix, k, 1) + (DIM == 3 ? d2 : 0);
    return v ? __ldg(p + o) : R(0);
  }
  // address and in-range flag of the face read at offset d (for async copies)
  template <class R>
  __device__ __forceinline__ const R* face_ptr(const Ix<DIM, PER>& ix, const R* p, int k, int d0, int d1, int d2,
                                               bool& v) const {
    if (PER) {
      v = true;
      int i = Ix<DIM, PER>::wrap(c[0] + d0, ix.n0), j = Ix<DIM, PER>::wrap(c[1] + d1, ix.n1);
      int l = DIM == 3 ? Ix<DIM, PER>::wrap(c[2] + d2, ix.n2) : 0;
      return p + ix.face_off(k, i, j, l);
    }
    v = ok(0, d0, k == 0 ? 2 : 1) && ok(1, d1, k == 1 ? 2 : 1) && (DIM == 2 || ok(2, d2, k == 2 ? 2 : 1));
    int o = of[2 * k] + d0 * fstride(ix, k, 0) + d1 * fstride(ix, k, 1) + (DIM == 3 ? d2 : 0);
    return v ? p + o : p;
  }
  // address and in-range flag of the cell read at offset d (for async copies)
  template <class R>
  __device__ __forceinline__ const R* cell_ptr(const Ix<DIM, PER>& ix, const R* p, int d0, int d1, int d2,
                                               bool& v) const {
    if (PER) {
      v = true;
      int i = Ix<DIM, PER>::wrap(c[0] + d0, ix.n0), j = Ix<DIM, PER>::wrap(c[1] + d1, ix.n1);
      int l = DIM == 3 ? Ix<DIM, PER>::wrap(c[2] + d2, ix.n2) : 0;
      return p + ix.cell_off(i, j, l);
    }
    v = ok(0, d0, 1) && ok(1, d1, 1) && (DIM == 2 || ok(2, d2, 1));
    int o = co + d0 * cstride(ix, 0) + d1 * cstride(ix, 1) + (DIM == 3 ? d2 : 0);
    return v ? p + o : p;
  }
  template <class R>
  __device__ __forceinline__ R cell(const Ix<DIM, PER>& ix, const R* __restrict__ p, int d0, int d1, int d2) const {
    if (PER) return ix.cell(p, c[0] + d0, c[1] + d1, c[2] + d2);
    bool v = ok(0, d0, 1) && ok(1, d1, 1) && (DIM == 2 || ok(2, d2, 1));
    int o = co + d0 * cstride(ix, 0) + d1 * cstride(ix, 1) + (DIM == 3 ? d2 : 0);
    return v ? __ldg(p + o) : R(0);
  }
};

// register cache of one face field around a cell (NbrSlots layout), loaded
// through Loc; slots a stencil does not use are dead and never loaded
template <int DIM, bool PER, class R, class LocT>
__device__ __forceinline__ void load_nbr(const Ix<DIM, PER>& ix, const LocT& L, const Face3<R>& f,
                                         R (&val)[DIM][NbrSlots<DIM>::NB]) {
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int sl = 0; sl < NbrSlots<DIM>::NB; ++sl) {
      int d[3];
      NbrSlots<DIM>::offset(a, sl, d);
      val[a][sl] = L.face(ix, f.c[a], a, d[0], d[1], d[2]);
    }
}

// ---------------------------------------------------------------------------
// Closed-form S(v,w)_J, T(v,u)_J at the cell's own J-face f = c + SD e_J from
// register caches (same arithmetic as S_at / Tadj_at, compile-time slots).
// Valid for non-wall faces (Neumann: both cells of the face exist).
// ---------------------------------------------------------------------------
template <int DIM, int J, int SD, class R>
__device__ __forceinline__ R S_cached(R c0, const R (&A)[DIM][NbrSlots<DIM>::NB],
                                      const R (&W)[DIM][NbrSlots<DIM>::NB], bool has_up, bool has_dn) {
  R acc = R(0);
  static_for<DIM>([&](auto kc) {
    constexpr int K = decltype(kc)::value;
    R ap, am, wp, wm;
    if constexpr (K == J) {
      const R aj = A[J][SD + 1];
      ap = has_up ? R(0.5) * (aj + A[J][SD + 2]) : R(0);
      am = has_dn ? R(0.5) * (A[J][SD] + aj) : R(0);
      wp = W[J][SD + 2];
      wm = W[J][SD];
    } else {
      ap = R(0.5) * (A[K][nbr_slot<DIM>(K, 1, J, SD)] + A[K][nbr_slot<DIM>(K, 1, J, SD - 1)]);
      am = R(0.5) * (A[K][nbr_slot<DIM>(K, 0, J, SD)] + A[K][nbr_slot<DIM>(K, 0, J, SD - 1)]);
      wp = W[J][nbr_slot<DIM>(J, SD, K, 1)];
      wm = W[J][nbr_slot<DIM>(J, SD, K, -1)];
    }
    acc += ap * wp - am * wm;
  });
  return c0 * acc;
}

template <int DIM, int J, int SD, class R>
__device__ __forceinline__ R T_cached(R c0, const R (&V)[DIM][NbrSlots<DIM>::NB],
                                      const R (&U)[DIM][NbrSlots<DIM>::NB]) {
  R acc = R(0);
  static_for<DIM>([&](auto jc) {
    constexpr int Q = decltype(jc)::value;
    R s = R(0);
    if constexpr (Q == J) {
      // cells g and g - e_J: gam = c0 (u[c'] v[c'+e] - u[c'+e] v[c'])
      static_for<2>([&](auto sc) {
        constexpr int SIDE = decltype(sc)::value;
        constexpr int lo = SD - SIDE + 1, hi = SD - SIDE + 2;
        s += U[J][lo] * V[J][hi] - U[J][hi] * V[J][lo];
      });
    } else {
      static_for<2>([&](auto sc) {
        constexpr int SIDE = decltype(sc)::value;
        constexpr int f = nbr_slot<DIM>(Q, SIDE, J, SD), fm = nbr_slot<DIM>(Q, SIDE, J, SD - 1);
        s += U[Q][fm] * V[Q][f] - U[Q][f] * V[Q][fm];
      });
    }
    acc += R(0.5) * c0 * s;
  });
  return acc;
}

// ---------------------------------------------------------------------------
// S(a, w)_j at one j-face f  (advection.py:306-365)
//   S_j = (1/2h) sum_k (A+_{jk} w_j[f+e_k] - A-_{jk} w_j[f-e_k]),  wall-masked.
// ---------------------------------------------------------------------------
template <int DIM, bool PER, class R, class FA, class FW>
__device__ __forceinline__ R S_at(const Ix<DIM, PER>& ix, R c0, int j, const int f[3], const FA& a, const FW& w) {
  if (!PER && (f[j] == 0 || f[j] == ix.n(j))) return R(0);
  R acc = R(0);
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    R ap, am;
    int t[3];
    if (k == j) {
      // centre averages of a_j in the cells above / below the face
      int up[3], dn[3];
      shift((int*)f, j, 1, up);
      shift((int*)f, j, -1, dn);
      R aj = a(j, f[0], f[1], f[2]);
      bool has_up = PER || f[j] < ix.n(j);
      bool has_dn = PER || f[j] > 0;
      ap = has_up ? R(0.5) * (aj + a(j, up[0], up[1], up[2])) : R(0);
      am = has_dn ? R(0.5) * (a(j, dn[0], dn[1], dn[2]) + aj) : R(0);
    } else {
      // corners: a_k averaged along j at k-index f_k+1 (plus) / f_k (minus)
      int p0[3], p1[3];
      shift((int*)f, k, 1, p0);          // (f_j, f_k+1)
      shift(p0, j, -1, p1);              // (f_j-1, f_k+1)
      ap = R(0.5) * (a(k, p0[0], p0[1], p0[2]) + a(k, p1[0], p1[1], p1[2]));
      shift((int*)f, j, -1, p1);         // (f_j-1, f_k)
      am = R(0.5) * (a(k, f[0], f[1], f[2]) + a(k, p1[0], p1[1], p1[2]));
    }
    shift((int*)f, k, 1, t);
    R wp = w(j, t[0], t[1], t[2]);
    shift((int*)f, k, -1, t);
    R wm = w(j, t[0], t[1], t[2]);
    acc += ap * wp - am * wm;
  }
  return c0 * acc;
}

// ---------------------------------------------------------------------------
// T(v, u)_k at one k-face g: adjoint of d -> S(d, v) tested against u
// (advection.py:380-434).  J_Adv(v)^T u = T(v, u) - S(v, u) (advection.py:437).
// ---------------------------------------------------------------------------
template <int DIM, bool PER, class R, class FV, class FU>
__device__ __forceinline__ R Tadj_at(const Ix<DIM, PER>& ix, R c0, int k, const int g[3], const FV& v, const FU& u) {
  if (!PER && (g[k] == 0 || g[k] == ix.n(k))) return R(0);
  R acc = R(0);
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    if (j == k) {
      // gam[c] = c0 (u_k[c] v_k[c+e_k] - u_k[c+e_k] v_k[c]) on cells along k;
      // out += 1/2 (gam[cell g] + gam[cell g - e_k])
      R s = R(0);
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        int c[3], cp[3];
        shift((int*)g, k, -side, c);     // cell index (lower face of the cell) = c
        if (!PER && (c[k] < 0 || c[k] >= ix.n(k))) continue;
        shift(c, k, 1, cp);
        s += u(k, c[0], c[1], c[2]) * v(k, cp[0], cp[1], cp[2]) - u(k, cp[0], cp[1], cp[2]) * v(k, c[0], c[1], c[2]);
      }
      acc += R(0.5) * c0 * s;
    } else {
      // gam_jk at (j-face index f_j, corner index f_k along k):
      //   c0 (u_j[f - e_k] v_j[f] - u_j[f] v_j[f - e_k]),  interior f_k only;
      // out_k[g] += 1/2 (gam[f_j = g_j] + gam[f_j = g_j + 1]) at f_k = g_k
      if (!PER && (g[k] == 0 || g[k] == ix.n(k))) continue;
      R s = R(0);
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        int f[3], fm[3];
        shift((int*)g, j, side, f);
        shift(f, k, -1, fm);
        s += u(j, fm[0], fm[1], fm[2]) * v(j, f[0], f[1], f[2]) - u(j, f[0], f[1], f[2]) * v(j, fm[0], fm[1], fm[2]);
      }
      acc += R(0.5) * c0 * s;
    }
  }
  return acc;
}

template <int DIM, bool PER, class R, class FV, class FU>
__device__ __forceinline__ R JT_at(const Ix<DIM, PER>& ix, R c0, int k, const int g[3], const FV& v, const FU& u) {
  return Tadj_at<DIM, PER, R>(ix, c0, k, g, v, u) - S_at<DIM, PER, R>(ix, c0, k, g, v, u);
}

// ---------------------------------------------------------------------------
// Paired arithmetic for the dense per-cell block algebra: fp32 maps to the
// sm_100 packed FFMA2 / FMUL2 (two independent fused multiply-adds per
// instruction, each rounded exactly like the scalar FFMA), fp64 to two DFMAs.
// `a` is broadcast to both lanes.
// ---------------------------------------------------------------------------
template <class R> struct PairOf;
template <> struct PairOf<float> { using T = float2; };
template <> struct PairOf<double> { using T = double2; };
template <class R> using R2 = typename PairOf<R>::T;

__device__ __forceinline__ float2 p2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 p2(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2 fma2s(float a, float2 b, float2 c) { return __ffma2_rn(make_float2(a, a), b, c); }
__device__ __forceinline__ double2 fma2s(double a, double2 b, double2 c) {
  return make_double2(fma(a, b.x, c.x), fma(a, b.y, c.y));
}
__device__ __forceinline__ float2 mul2s(float a, float2 b) { return __fmul2_rn(make_float2(a, a), b); }
__device__ __forceinline__ double2 mul2s(double a, double2 b) { return make_double2(a * b.x, a * b.y); }

// one element global -> shared, asynchronous (cp.async, L1-allocating);
// valid == false zero-fills (src-size 0) without reading the source
template <class R>
__device__ __forceinline__ void cp_async_elem(R* smem, const R* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if constexpr (sizeof(R) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 4 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0) : "memory");
}
// 16-byte copy (L2 only), both addresses 16-byte aligned
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// N consecutive values from 16-byte aligned shared memory, 16 bytes per load
template <class R, int N>
__device__ __forceinline__ void lds_vec(const R* p, R (&o)[N]) {
  if constexpr (sizeof(R) == 4) {
    static_assert(N % 4 == 0, "lds_vec: N % 4");
#pragma unroll
    for (int k = 0; k < N / 4; ++k) {
      const float4 v = reinterpret_cast<const float4*>(p)[k];
      o[4 * k] = v.x; o[4 * k + 1] = v.y; o[4 * k + 2] = v.z; o[4 * k + 3] = v.w;
    }
  } else {
    static_assert(N % 2 == 0, "lds_vec: N % 2");
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
      const double2 v = reinterpret_cast<const double2*>(p)[k];
      o[2 * k] = v.x; o[2 * k + 1] = v.y;
    }
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

// explicit-width |x| (an unqualified abs() on a float can bind to int abs)
__device__ __forceinline__ float rabs(float x) { return fabsf(x); }
__device__ __forceinline__ double rabs(double x) { return fabs(x); }

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ R warp_max(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <class R>
__device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// atomic max of a non-negative value through its bit pattern (order-free,
// hence deterministic)
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  atomicMax((unsigned int*)addr, (unsigned int)__float_as_int(v));
}

template <class R>
__device__ __forceinline__ void block_max_to(R v, R* out) {
  __shared__ R sh[32];
  v = warp_max(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : R(0);
    v = warp_max(v);
    if (lane == 0 && v > R(0)) atomic_max_nonneg(out, v);
  }
}

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  const int64_t cap = 148 * 32;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

// frame-major launch shape: blockIdx.z = frame, blockIdx.y = component (face
// kernels), a 32-bit grid-stride index over one frame's elements
inline dim3 frame_grid(int64_t per_frame, int nframes, int block, int comps = 1) {
  int64_t g = (per_frame + block - 1) / block;
  if (g > 65535) g = 65535;
  if (g < 1) g = 1;
  return dim3((unsigned)g, (unsigned)comps, (unsigned)nframes);
}
#define SMK_FRAME_LOOP(e, n) for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (int)(n); e += gridDim.x * blockDim.x)

#define SMK_GRID_STRIDE(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

}  // namespace smk
