// STFAS / NSO: Eq. 8 KKT residual, coloured time-line SCGS smoother, FAS
// V-cycle hierarchy (PAPER Eq. 8/9, Alg. 2).
//
// Semantics are frozen in DESIGN.md §3 and mirrored by oracle/stfas.py:
//   pair index i = 0..N-1:  U[i]=u_i, P[i]=p_{i+1}, V[i]=v_{i+1}, PB[i]=pbar_{i+1}
//   R3[i] = (v_{i+1}-v_i)/dt + Adv(v_{i+1}) - u_i + grad p_{i+1}
//   R4[i] = div u_i
//   R1[i] = [i<N-1]((K/r)(v_{i+1}-v*_{i+1}) - u_{i+1}/dt) + u_i/dt
//           + J_Adv(v_{i+1})^T u_i + grad pbar_{i+1}
//   R2[i] = div v_{i+1}
// Smoother: per colour, every cell of the colour solves its 2N-block
// (2d faces + 1 scalar) Gauss-Newton time line with the state frozen
// (snapshot reads, writes go to a delta buffer), then the colour's unknowns
// take x += omega * dx.  Same-colour cells own disjoint unknowns, so the
// apply pass is race-free and the sweep is bitwise deterministic.
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <vector>
#include <array>
#include <type_traits>

#include <dlfcn.h>
#include <memory>
#include <nccl.h>

#include "smk_internal.cuh"

namespace smk {

#ifndef SMK_HANDOFF_BLOCKED
#define SMK_HANDOFF_BLOCKED 1
#endif


template <class R>
struct StP {
  R* V[3];
  R* PB;
  R* U[3];
  R* P;
};
template <class R>
struct ResP {
  R* R1[3];
  R* R2;
  R* R3[3];
  R* R4;
};

struct NsoK {  // kernel-side scalars
  int N;
  double dt, kr, omega;
};

template <class R>
__device__ __forceinline__ Face3<R> frame_of(const Face3<R>& base, int fr, const int64_t nf[3]) {
  Face3<R> o;
#pragma unroll
  for (int k = 0; k < 3; ++k) o.c[k] = base.c[k] ? base.c[k] + (int64_t)fr * nf[k] : nullptr;
  return o;
}

// ---------------------------------------------------------------------------
// point residuals (shared by the residual kernel and the smoother)
// ---------------------------------------------------------------------------
template <int DIM, bool PER, class R>
struct KktCtx {
  Ix<DIM, PER> ix;
  R c0, h, dt, kr;
  R ih, idt;       // 1/h, 1/dt (host-rounded; exact for h = 2^-k)
  int N;           // local pairs (this slab)
  int t0, Ng;      // global index of local pair 0, global pair count
  int64_t nf[3], nc;
  Face3<R> V, U, v0, vs;
  Face3<R> un;     // right halo u_{t0+N} (slab mode; unused when t0+N == Ng)
  const R* P;
  const R* PB;

  // K-term / u_{i+1} present for local pair i (global i < Ng-1)
  __device__ __forceinline__ bool inner(int i) const { return t0 + i < Ng - 1; }
  // frame fr of a face stack.  (32-bit frame offsets without the null
  // checks were measured slower: cfg5 V-cycle 145 -> 169 ms.)
  __device__ __forceinline__ Face3<R> frame(const Face3<R>& base, int fr) const { return frame_of(base, fr, nf); }
  __device__ __forceinline__ Face3<R> u_next(int i) const { return i < N - 1 ? frame(U, i + 1) : un; }

};

// ---------------------------------------------------------------------------
// Eq. 8 rows of one cell, shared by the residual kernel and the smoother.
//
// f - rhs of pair i at the cell's own faces q = 2j + sd (sd = 0 always, sd = 1
// when BOTH) and at the cell: yu = (R3, R4) rows, yv = (R1, R2) rows.  Inputs
// are register caches of V_i (VC) and U_i (UC) around the cell and V_{i-1} at
// the own faces (vp).  Wall rows (Neumann, not unknowns): 0 - rhs when
// WALLRHS (the residual, like the masked rows of SPEC kkt_residual), else 0
// (the smoother assembles only unknown rows).  Same term order as
// oracle/stfas.py kkt_residual; 1/h and 1/dt are multiplied, not divided.
// ---------------------------------------------------------------------------
// gathered scalar inputs of one pair's rows (besides the V / U caches)
template <int DIM, class R>
struct RowIn {
  static constexpr int NF = 2 * DIM;
  R pc, pbc;                  // P, PBAR at the cell
  R pn[NF], pbn[NF];          // P, PBAR across each own face
  R vsv[NF], unv[NF];         // guide v*_{i+1} and u_{i+1} at the own faces
  R r1v[NF], r3v[NF], r2c, r4c;   // rhs rows (HR)
};

// the rows from the caches and the gathered inputs (no memory access)
template <int DIM, bool PER, class R, bool BOTH, bool WALLRHS, bool HR>
__device__ __forceinline__ void rows_compute(const KktCtx<DIM, PER, R>& cx, const bool (&wall)[2 * DIM], bool inner,
                                             const R (&VC)[DIM][NbrSlots<DIM>::NB],
                                             const R (&UC)[DIM][NbrSlots<DIM>::NB], const R (&vp)[2 * DIM],
                                             const RowIn<DIM, R>& g, R (&yu)[2 * DIM + 1], R (&yv)[2 * DIM + 1]) {
  constexpr int NF = 2 * DIM;
  static_for<NF>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    constexpr int j = q >> 1, sd = q & 1;
    if constexpr (!BOTH && sd == 1) {
      yu[q] = R(0);
      yv[q] = R(0);
    } else {
      if (wall[q]) {
        yu[q] = (WALLRHS && HR) ? R(0) - g.r3v[q] : R(0);
        yv[q] = (WALLRHS && HR) ? R(0) - g.r1v[q] : R(0);
      } else {
        const R gp = sd ? (g.pn[q] - g.pc) * cx.ih : (g.pc - g.pn[q]) * cx.ih;
        const R gpb = sd ? (g.pbn[q] - g.pbc) * cx.ih : (g.pbc - g.pbn[q]) * cx.ih;
        const R vf = VC[j][sd + 1], uf = UC[j][sd + 1];
        const R adv = S_cached<DIM, j, sd, R>(cx.c0, VC, VC, true, true);
        R a = (((vf - vp[q]) * cx.idt + adv) - uf) + gp;
        R t1 = R(0);
        if (inner) t1 = cx.kr * (vf - g.vsv[q]) - g.unv[q] * cx.idt;
        const R jt = T_cached<DIM, j, sd, R>(cx.c0, VC, UC) - S_cached<DIM, j, sd, R>(cx.c0, VC, UC, true, true);
        R b = ((t1 + uf * cx.idt) + jt) + gpb;
        if (HR) {
          a -= g.r3v[q];
          b -= g.r1v[q];
        }
        yu[q] = a;
        yv[q] = b;
      }
    }
  });
  R dv = R(0), du = R(0);
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    R a = (VC[k][2] - VC[k][1]) * cx.ih;
    R b = (UC[k][2] - UC[k][1]) * cx.ih;
    dv = (k == 0) ? a : dv + a;
    du = (k == 0) ? b : du + b;
  }
  if (HR) {
    du -= g.r4c;
    dv -= g.r2c;
  }
  yu[NF] = du;
  yv[NF] = dv;
}

template <int DIM, bool PER, class R, bool BOTH, bool WALLRHS, bool HR, class LocT>
__device__ __forceinline__ void pair_rows(const KktCtx<DIM, PER, R>& cx, const LocT& L,
                                          const bool (&wall)[2 * DIM], int i,
                                          const R (&VC)[DIM][NbrSlots<DIM>::NB],
                                          const R (&UC)[DIM][NbrSlots<DIM>::NB], const R (&vp)[2 * DIM],
                                          const ResP<R>& rhs, R (&yu)[2 * DIM + 1],
                                          R (&yv)[2 * DIM + 1]) {
  constexpr int NF = 2 * DIM;
  const auto& ix = cx.ix;
  const R* Pi = cx.P + (int64_t)i * cx.nc;
  const R* PBi = cx.PB + (int64_t)i * cx.nc;
  const bool inner = cx.inner(i);
  const Face3<R> Un = inner ? cx.u_next(i) : Face3<R>{};
  const Face3<R> Vs = inner ? cx.frame(cx.vs, i + 1) : Face3<R>{};
  // gather every scalar input first, so all of the pair's loads are in
  // flight together (one memory latency per pair, not one per face)
  RowIn<DIM, R> g;
  g.pc = Pi[L.co];
  g.pbc = PBi[L.co];
  static_for<NF>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    constexpr int j = q >> 1, sd = q & 1;
    constexpr int d = sd ? 1 : -1;
    const bool on = (BOTH || sd == 0);
    const int64_t oo = (int64_t)i * cx.nf[j] + L.of[q];
    g.pn[q] = (on && !wall[q]) ? L.cell(ix, Pi, j == 0 ? d : 0, j == 1 ? d : 0, j == 2 ? d : 0) : R(0);
    g.pbn[q] = (on && !wall[q]) ? L.cell(ix, PBi, j == 0 ? d : 0, j == 1 ? d : 0, j == 2 ? d : 0) : R(0);
    g.vsv[q] = (on && inner && !wall[q]) ? Vs.c[j][L.of[q]] : R(0);
    g.unv[q] = (on && inner && !wall[q]) ? Un.c[j][L.of[q]] : R(0);
    g.r1v[q] = (on && HR && (WALLRHS || !wall[q])) ? rhs.R1[j][oo] : R(0);
    g.r3v[q] = (on && HR && (WALLRHS || !wall[q])) ? rhs.R3[j][oo] : R(0);
  });
  g.r2c = R(0);
  g.r4c = R(0);
  if (HR) {
    const int64_t o = (int64_t)i * cx.nc + L.co;
    g.r4c = rhs.R4[o];
    g.r2c = rhs.R2[o];
  }
  rows_compute<DIM, PER, R, BOTH, WALLRHS, HR>(cx, wall, inner, VC, UC, vp, g, yu, yv);
}

// Eq. 8 residual f(x) - rhs, one thread per (frame, cell): the cell's lower
// faces (R1, R3 of every component), the cell (R2, R4), and under Neumann the
// upper wall face of the last cell along each axis (0 - rhs).  Neighbour
// values come from the register caches (every V / U value the cell's faces
// need is read once per thread, through L1).
// NORM (the stop test): the same values, not stored; each
// block writes max |f| and sum f^2 (fp64) of its entries to part[2 blk ..],
// reduced in a fixed order by k_norm_final -- every residual entry is
// produced by exactly one thread, so this is ||f||_inf / ||f||_2 of the full
// residual without writing it (5.4 GB at cfg5) and reading it back.
// Each thread walks its cell through `fpt` consecutive frames (blockIdx.z =
// frame group): the cell's index math, wall flags and offsets are formed
// once, and V_{i-1} at the own faces is carried from the previous frame's
// register cache instead of being loaded again (the same values: results are
// bitwise those of one thread per cell-frame).  cfg5 level 0: 6.0 -> 5.4 ms,
// the stop test 6.7 -> 4.8 ms (fpt 8; 4: 5.7 / 5.3; 2: 6.4 / 6.0).
#ifndef SMK_KKT_FPT
#define SMK_KKT_FPT 8
#endif
// frames per thread: SMK_KKT_FPT on levels of >= 64^3 cells while the launch
// still has >= 8 blocks per SM, else 1 (smaller levels and the 2D configs are
// latency-bound and measured slower with a frame loop: 32^3 0.24 -> 0.33 ms,
// 256^2 0.13 -> 0.17 ms)
inline int kkt_fpt(int64_t nc, int nframes) {
  if (nc < 262144) return 1;
  int fpt = SMK_KKT_FPT;
  const int64_t bpf = (nc + 255) / 256;
  while (fpt > 1 && bpf * ((nframes + fpt - 1) / fpt) < 148 * 8) fpt >>= 1;
  return fpt;
}
inline dim3 kkt_grid(int64_t nc, int nframes) {
  const int fpt = kkt_fpt(nc, nframes);
  return frame_grid(nc, (nframes + fpt - 1) / fpt, 256);
}
// FL: the frame-loop shape (fpt > 1); !FL is the one-thread-per-cell-frame
// shape of the small levels, unchanged.
template <int DIM, bool PER, class R, bool HR, int NX, bool NORM = false, bool FL = false>
__global__ void __launch_bounds__(256, FL && sizeof(R) == 4 ? 2 : 1) k_kkt(KktCtx<DIM, PER, R> cx, ResP<R> rhs, ResP<R> out,
                                             double* __restrict__ part = nullptr, int fpt = 1) {
  constexpr int NF = 2 * DIM, B = NF + 1, NB = NbrSlots<DIM>::NB;
  const auto& ix = cx.ix;
  const int64_t nc = cx.nc;
  const int i0 = FL ? blockIdx.z * fpt : blockIdx.z;
  const int i1 = FL ? (i0 + fpt < cx.N ? i0 + fpt : cx.N) : i0 + 1;
  R mx = R(0);
  double sq = 0.0;
  auto put = [&](R* dst, int64_t o, R v) {
    if constexpr (NORM) {
      mx = fmax(mx, rabs(v));
      sq += (double)v * (double)v;
    } else {
      dst[o] = v;
    }
  };
  SMK_FRAME_LOOP(e, nc) {
    int c[3];
    ix.cell_idx32(e, c);
    const Loc<DIM, PER, NX> L(ix, c);
    bool wall[NF];
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      wall[2 * k] = !PER && c[k] == 0;
      wall[2 * k + 1] = !PER && c[k] == ix.n(k) - 1;
    }
    R vp[NF];
    if constexpr (FL) {
      const Face3<R> Vp = i0 == 0 ? cx.v0 : cx.frame(cx.V, i0 - 1);
#pragma unroll
      for (int q = 0; q < NF; ++q) vp[q] = (q & 1) ? R(0) : Vp.c[q >> 1][L.of[q]];
    }
    for (int i = i0; i < i1; ++i) {
      R VC[DIM][NB], UC[DIM][NB];
      load_nbr<DIM, PER, R>(ix, L, cx.frame(cx.V, i), VC);
      load_nbr<DIM, PER, R>(ix, L, cx.frame(cx.U, i), UC);
      if constexpr (!FL) {
        const Face3<R> Vp = i == 0 ? cx.v0 : cx.frame(cx.V, i - 1);
#pragma unroll
        for (int q = 0; q < NF; ++q) vp[q] = (q & 1) ? R(0) : Vp.c[q >> 1][L.of[q]];
      }
      R yu[B], yv[B];
      pair_rows<DIM, PER, R, false, true, HR>(cx, L, wall, i, VC, UC, vp, rhs, yu, yv);
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        const int64_t o = (int64_t)i * cx.nf[k] + L.of[2 * k];
        put(out.R3[k], o, yu[2 * k]);
        put(out.R1[k], o, yv[2 * k]);
        if (!PER && wall[2 * k + 1]) {
          const int64_t ou = (int64_t)i * cx.nf[k] + L.of[2 * k + 1];
          put(out.R3[k], ou, HR ? R(0) - rhs.R3[k][ou] : R(0));
          put(out.R1[k], ou, HR ? R(0) - rhs.R1[k][ou] : R(0));
        }
      }
      const int64_t oc = (int64_t)i * nc + L.co;
      put(out.R4, oc, yu[NF]);
      put(out.R2, oc, yv[NF]);
      // V_i at the own lower faces is the next frame's V_{i-1} (slot 1 of the cache)
      if constexpr (FL) {
#pragma unroll
        for (int q = 0; q < NF; q += 2) vp[q] = VC[q >> 1][1];
      }
    }
  }
  if constexpr (NORM) {
    __shared__ double shm[8], shs[8];
    double m = warp_max((double)mx);
    sq = warp_sum(sq);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
      shm[w] = m;
      shs[w] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
        a = fmax(a, shm[k]);
        b += shs[k];
      }
      const int64_t blk = (int64_t)blockIdx.z * gridDim.x + blockIdx.x;
      part[2 * blk] = a;
      part[2 * blk + 1] = b;
    }
  }
}

// fixed-order reduction of the NORM blocks' partials: out = {max, sum}
__global__ void __launch_bounds__(1024) k_norm_final(const double* __restrict__ part, int64_t nblk, double* out) {
  __shared__ double shm[32], shs[32];
  double a = 0.0, b = 0.0;
  for (int64_t k = threadIdx.x; k < nblk; k += blockDim.x) {
    a = fmax(a, part[2 * k]);
    b += part[2 * k + 1];
  }
  a = warp_max(a);
  b = warp_sum(b);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    shm[w] = a;
    shs[w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      x = fmax(x, shm[k]);
      y += shs[k];
    }
    out[0] = isnan(y) ? y : x;   // fmax drops NaN; the sum keeps it
    out[1] = y;
  }
}

// ---------------------------------------------------------------------------
// the time-line SCGS smoother
// ---------------------------------------------------------------------------

// Dense solve S [W | z] = [RHS], B x B with C right-hand sides, in registers.
// PIVOT selects partial pivoting (tournament row swaps, fully unrolled so the
// arrays stay in registers); definite blocks use the natural order.
template <class R, int B, int C, bool PIVOT>
// (tiny is relative to the largest |entry| of A: scale-free SingularBlock test)
__device__ __forceinline__ bool dense_solve(R (&A)[B][B], R (&X)[B][C], R tiny) {
  bool ok = true;
  {
    R amax = R(0);
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) amax = fmax(amax, rabs(A[r][c]));
    tiny *= amax;
  }
  R inv[B];
#pragma unroll
  for (int col = 0; col < B; ++col) {
    if (PIVOT) {
#pragma unroll
      for (int r = col + 1; r < B; ++r) {
        bool sw = rabs(A[r][col]) > rabs(A[col][col]);
#pragma unroll
        for (int c = 0; c < B; ++c) {
          R a = A[col][c], b = A[r][c];
          A[col][c] = sw ? b : a;
          A[r][c] = sw ? a : b;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          R a = X[col][c], b = X[r][c];
          X[col][c] = sw ? b : a;
          X[r][c] = sw ? a : b;
        }
      }
    }
    R piv = A[col][col];
    if (!(rabs(piv) > tiny)) ok = false;
    inv[col] = R(1) / piv;
#pragma unroll
    for (int r = col + 1; r < B; ++r) {
      R fct = A[r][col] * inv[col];
#pragma unroll
      for (int c = col + 1; c < B; ++c) A[r][c] -= fct * A[col][c];
#pragma unroll
      for (int c = 0; c < C; ++c) X[r][c] -= fct * X[col][c];
    }
  }
#pragma unroll
  for (int r = B - 1; r >= 0; --r) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      R s = X[r][c];
#pragma unroll
      for (int q = r + 1; q < B; ++q) s -= A[r][q] * X[q][c];
      X[r][c] = s * inv[r];
    }
  }
  return ok;
}

// 1/x for the pivots: fp32 uses the hardware approximation plus one Newton
// step (<= 1 ulp for the normal, well-scaled pivots of these blocks; no IEEE
// slow-path call sites in the consumer loop), fp64 the IEEE division.
__device__ __forceinline__ float pivot_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r * (2.0f - x * r);
}
__device__ __forceinline__ double pivot_rcp(double x) { return 1.0 / x; }

// In-place LDL^T of a symmetric B x B matrix held in the lower triangle of T
// (natural order, no pivoting -- used for the saddle blocks whose faces part
// is positive definite): on exit T[r][c] (c < r) = L[r][c], dinv = 1 / d.
//
// SingularBlock ("block pivot below 1e-12"), made scale-free:
// the blocks are K' = [[D~, g], [g^T, 0]] with D~ ~ (PM)^T PM + alpha I +
// P / dt^2, so a faces pivot is compared with tf = 1e-12 (1/dt^2 + alpha)
// and the saddle pivot (units |g|^2 / D~) with ts = 1e-12 sigma / (1/dt^2 +
// alpha), sigma = |g|^2 -- per-cell constants, nothing on the elimination's
// critical path.  In fp32 this flags breakdown (zero / denormal / NaN
// pivots), in fp64 the SPEC's degenerate configurations too.
template <class R, int B>
__device__ __forceinline__ bool ldlt(R (&T)[B][B], R (&dinv)[B], R tf, R ts) {
  bool ok = true;
#pragma unroll
  for (int col = 0; col < B; ++col) {
    const R piv = T[col][col];
    if (!(rabs(piv) > (col < B - 1 ? tf : ts))) ok = false;
    dinv[col] = pivot_rcp(piv);
    R l[B];
#pragma unroll
    for (int r = col + 1; r < B; ++r) l[r] = T[r][col] * dinv[col];
#pragma unroll
    for (int r = col + 1; r < B; ++r)
#pragma unroll
      for (int c = col + 1; c <= r; ++c) T[r][c] -= l[r] * T[c][col];
#pragma unroll
    for (int r = col + 1; r < B; ++r) T[r][col] = l[r];
  }
  return ok;
}

// b <- (L diag(d) L^T)^-1 b
template <class R, int B>
__device__ __forceinline__ void ldlt_solve(const R (&T)[B][B], const R (&dinv)[B], R (&b)[B]) {
#pragma unroll
  for (int r = 1; r < B; ++r)
#pragma unroll
    for (int c = 0; c < r; ++c) b[r] -= T[r][c] * b[c];
#pragma unroll
  for (int r = 0; r < B; ++r) b[r] *= dinv[r];
#pragma unroll
  for (int r = B - 2; r >= 0; --r)
#pragma unroll
    for (int c = r + 1; c < B; ++c) b[r] -= T[c][r] * b[c];
}

// The partially pivoted solve runs once per cell line (the last global pair,
// alpha = 0, whose faces block is singular along M^-1 g while the saddle is
// not); it is kept out of line on a local-memory copy so its unrolled row
// swaps do not bloat the consumer loop.
template <class R, int B>
__device__ __noinline__ bool saddle_solve_pivot_mem(R* Tm, R tiny) {
  R A[B][B], X[B][1];
#pragma unroll
  for (int r = 0; r < B; ++r) {
#pragma unroll
    for (int c = 0; c < B; ++c) A[r][c] = Tm[r * (B + 1) + c];
    X[r][0] = Tm[r * (B + 1) + B];
  }
  bool ok = dense_solve<R, B, 1, true>(A, X, tiny);
#pragma unroll
  for (int r = 0; r < B; ++r) Tm[r * (B + 1) + B] = X[r][0];
  return ok;
}

// b <- K'^-1 b for the symmetric K' held in the lower triangle of T
template <class R, int B>
__device__ __forceinline__ bool saddle_solve_pivot(const R (&T)[B][B], R (&b)[B], R tiny) {
  R Tm[B * (B + 1)];
#pragma unroll
  for (int r = 0; r < B; ++r) {
#pragma unroll
    for (int c = 0; c < B; ++c) Tm[r * (B + 1) + c] = c <= r ? T[r][c] : T[c][r];
    Tm[r * (B + 1) + B] = b[r];
  }
  bool ok = saddle_solve_pivot_mem<R, B>(Tm, tiny);
#pragma unroll
  for (int r = 0; r < B; ++r) b[r] = Tm[r * (B + 1) + B];
  return ok;
}

template <int DIM>
struct Slots {
  static constexpr int NF = 2 * DIM;
  static constexpr int B = NF + 1;
  static constexpr int C = NF + 1;  // W columns (faces) + z
};

// Colour cell m -> cell coordinates.  mod > 0: mod-m colouring, colour
// digits (o0, o1, o2), cells o_a + mod * q_a; mod < 0: red-black, colour o0,
// cells with (sum_a c_a) % 2 == o0 -- unit stride on the leading axes, stride
// 2 along the last axis starting at the row's parity (even last extent, so
// every row holds m_last colour cells).
//
// 3D red-black row order (mod = -T, T > 1): consecutive rows (one CTA each
// on the big colours) walk axis 1 inside bands of T rows along axis 0, row
// r -> (c0, c1) = (T (r / (T n1)) + r mod T, (r mod (T n1)) / T).  CTAs start
// in blockIdx order and march through the N pairs independently, so a row's
// stencil neighbours come from L2 only if their CTAs run close in time: with
// the plain order (T = 1) the axis-0 neighbours are n1 rows away (a fifth of
// the resident CTAs at 128^3, ~17 pairs of skew) and every neighbour row was
// re-read from DRAM; with T = 8 the axis-1 neighbours are T rows away, the
// axis-0 ones inside the band 1 row, and only the band edges miss.  A pure
// relabelling of m: the pass's results do not depend on it.
template <int DIM>
__device__ __forceinline__ void color_cell(int64_t m, int o0, int o1, int o2, int mod, int m1, int m2, int (&c)[3]) {
  int64_t q = m;
  const int q2 = (int)(q % m2); q /= m2;
  if (DIM == 3 && mod < -1) {
    const int T = -mod;   // the host only passes T > 1 when T divides n0
    const int64_t bw = (int64_t)T * m1;
    const int64_t band = q / bw;
    const int rem = (int)(q - band * bw);
    c[0] = (int)(band * T) + rem % T;
    c[1] = rem / T;
    c[2] = ((o0 + c[0] + c[1]) & 1) + 2 * q2;
    return;
  }
  const int q1 = (int)(q % m1); q /= m1;
  if (mod > 0) {
    c[0] = o0 + mod * (int)q;
    c[1] = o1 + mod * q1;
    c[2] = DIM == 3 ? o2 + mod * q2 : 0;
  } else if (DIM == 3) {
    c[0] = (int)q;
    c[1] = q1;
    c[2] = ((o0 + c[0] + c[1]) & 1) + 2 * q2;
  } else {
    c[0] = (int)q;
    c[1] = ((o0 + c[0]) & 1) + 2 * q1;
    c[2] = 0;
  }
}

// colour-cell geometry shared by the smoother kernels
template <int DIM, bool PER, class R>
struct CellGeo {
  static constexpr int NF = 2 * DIM;
  int c[3];
  int fidx[NF][3];
  bool wall[NF];
  R gcol[NF];
  __device__ __forceinline__ CellGeo(const Ix<DIM, PER>& ix, R h, int64_t m, int o0, int o1, int o2, int mod, int m1,
                                     int m2) {
    color_cell<DIM>(m, o0, o1, o2, mod, m1, m2, c);
#pragma unroll
    for (int k = 0; k < DIM; ++k)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        int qq = 2 * k + s;
        fidx[qq][0] = c[0]; fidx[qq][1] = c[1]; fidx[qq][2] = c[2];
        fidx[qq][k] += s;
        if (PER && fidx[qq][k] >= ix.n(k)) fidx[qq][k] -= ix.n(k);
        wall[qq] = !PER && (s == 0 ? c[k] == 0 : c[k] == ix.n(k) - 1);
        gcol[qq] = wall[qq] ? R(0) : (s == 0 ? R(1) : R(-1)) / h;
      }
  }
};

// Closed-form local Jacobian of Adv(v) = S(v, v) on the cell's own faces
// (derived from advection.py:306-377 with d = e_g):
//   row (j,s_r), col (j,s_c):  S(v, e_g) gives the opposite-face coupling
//     +/- c0 * vc_j (vc_j = cell-centre average of v_j), S(e_g, v) gives
//     (j,0)(j,0) = c0/2 (v_j[c+e_j] - v_j[c-e_j])   (j,0)(j,1) += c0/2 v_j[c+e_j]
//     (j,1)(j,1) = c0/2 (v_j[c+2e_j] - v_j[c])      (j,1)(j,0) -= c0/2 v_j[c]
//   row (j,s), col (k != j):  (k,1) = +c0/2 v_j[c + s e_j + e_k]
//                             (k,0) = -c0/2 v_j[c + s e_j - e_k]
// Wall rows / columns are zero (not unknowns).  Equal to the probed Jacobian
// of oracle/stfas.local_jacobian up to rounding.
template <int DIM, class R>
__device__ __forceinline__ void jac_cached(R c0, R idt, const R (&v)[DIM][NbrSlots<DIM>::NB],
                                           const bool (&wall)[2 * DIM], R (&J)[2 * DIM][2 * DIM]) {
  constexpr int NF = 2 * DIM;
  const R hc = R(0.5) * c0;
#pragma unroll
  for (int j = 0; j < DIM; ++j) {
    const R vm = v[j][0], v0 = v[j][1], v1 = v[j][2], v2 = v[j][3];
    const R vc = R(0.5) * (v0 + v1);
    J[2 * j][2 * j] = hc * (v1 - vm);
    J[2 * j][2 * j + 1] = c0 * vc + hc * v1;
    J[2 * j + 1][2 * j] = -c0 * vc - hc * v0;
    J[2 * j + 1][2 * j + 1] = hc * (v2 - v0);
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      if (k == j) continue;
#pragma unroll
      for (int sr = 0; sr < 2; ++sr) {
        J[2 * j + sr][2 * k + 1] = hc * v[j][nbr_slot<DIM>(j, sr, k, 1)];
        J[2 * j + sr][2 * k] = -hc * v[j][nbr_slot<DIM>(j, sr, k, -1)];
      }
    }
  }
#pragma unroll
  for (int a = 0; a < NF; ++a)
#pragma unroll
    for (int b = 0; b < NF; ++b)
      if (wall[a] || wall[b]) J[a][b] = R(0);
  // M = I/dt + J on the unknown faces
#pragma unroll
  for (int q = 0; q < NF; ++q)
    if (!wall[q]) J[q][q] += idt;
}

// ---------------------------------------------------------------------------
// One colour pass = k_scgs_fwd (forward elimination) + k_scgs_back (back
// substitution) + k_scgs_apply.  Every cell of the colour solves its 2N-block
// Eq. 9 time line exactly (oracle/stfas.py scgs_color), the
// state is read-only until k_scgs_apply (snapshot semantics).
//
// The u-block of pair i is the constant saddle [[-I, g], [-g^T, 0]] (g = the
// cell's grad column), coupled to v_i by -I/dt and to v_{i+1} by
// M_i = I/dt + J_i.  With P = I - g g^T / sigma (sigma = g^T g):
//     du_i = -c_i - (P/dt) dv_i + P M_i dv_{i+1},   c_i = P yu_i + g yp_i / sigma,
//     dp_{i+1} = (g^T a_i - yp_i) / sigma,   a_i = yu_i + dv_i/dt - M_i dv_{i+1}.
// Substituting into the v-rows leaves a symmetric block-tridiagonal system in
// (dv_{i+1}, dpbar_{i+1}) only (N blocks of 2d+1 instead of 2N):
//     D_i  = (P M_i)^T (P M_i) + alpha_i I + [i+1<N] P/dt^2   (faces; + the g saddle)
//     L_i  = -(P M_i)^T / dt   (to dv_i),   U_i = L_{i+1}^T = -P M_{i+1} / dt
//     rhs  = yv_i + M_i^T c_i - [i+1<N] c_{i+1} / dt.
//
// k_scgs_fwd is warp-specialised.  A CTA owns TM colour cells; warps
// [0, TM/32) are producers, [TM/32, 2TM/32) consumers, one thread of each per
// cell.  Producers stream the state (all the HBM reads of the pass): the
// -(f - rhs) rows of pair i from register caches of the cell's
// neighbourhood, and hand the rows and the V stencil values behind M_i to the
// consumers through an S-stage shared-memory ring (named barriers FULL/EMPTY
// per stage); they also store the u-rows yu_i for the backward pass.  Consumers run the dense elimination (an LDL^T of each pair's
// symmetric saddle block, see below), carrying the Schur-updated D_{i+1}, its
// partial rhs and (P M_{i+1})^T z_i to the next pair.  Per pair the scratch
// holds SE values (L, 1/d, z, yu), layout [pair][entry][m].
// ---------------------------------------------------------------------------
template <int DIM>
struct Line {
  static constexpr int NF = 2 * DIM, B = NF + 1;
  // hand-off of a pair, two formats sharing one scratch stride SE:
  //   compact (big colours): D~ faces block (lower triangle with diagonal), rhs b, yu
  //   factored (small, latency-bound colours): L (strict lower), 1/d, z, yu
  static constexpr int NT = NF * (NF + 1) / 2, NL = B * (B - 1) / 2;
  static constexpr int T0 = 0, B0 = NT, Y0 = NL + 2 * B;
  // compact keeps its yu right after b, so a pair's compact entries are the
  // contiguous rows [0, NCMP) of its tile (one bulk copy per block, k_scgs_back)
  static constexpr int Y0C = NT + B, NCMP = NT + 2 * B;
  static constexpr int L0 = 0, D0 = NL, Z0 = NL + B;
  static constexpr int SE = NL + 3 * B;
  // [i][e][m] formats are stored block-interleaved, [i][m / HB][e][HB]: a
  // pair's entries of HB consecutive colour cells are one contiguous
  // SE x HB tile, so a thread addresses entry e of pair i as
  // base_i + e * HB (an immediate offset on one per-pair pointer) instead of
  // a 64-bit (i SE + e) M + m product per access; every warp access is still
  // one coalesced 128-byte row.
  static constexpr int HB = SMK_HANDOFF_BLOCKED ? 64 : 1;
  __host__ __device__ static int64_t pair_stride(int64_t M) { return ((M + HB - 1) / HB) * SE * HB; }
  __host__ __device__ static int64_t cell_base(int64_t m) { return (m / HB) * SE * HB + (m % HB); }
  // entry stride of the tile (HB = 1: the plain [i][e][m] layout, stride M)
  __host__ __device__ static int64_t entry_stride(int64_t M) { return HB > 1 ? HB : M; }
  // record hand-off (shape-2 colours with the cp.async-ring backward): RS
  // values per (pair, cell) -- M_i (row-major, written by the pair's
  // producer), yu_i (padded to 8), then the consumer's L, 1/d and z -- in
  // 16-byte groups interleaved over the cells, [i][RS / VW][m][VW] with VW =
  // 16 / sizeof(R): one 16-byte store / cp.async per group and thread, a
  // coalesced 512 B per warp
  static constexpr int NY = 8;
  static constexpr int NLDZ = (NL + 2 * B + 3) & ~3;
  static constexpr int R_M = 0, R_Y = NF * NF, R_L = NF * NF + NY, R_D = R_L + NL, R_Z = R_D + B;
  static constexpr int RS = R_L + NLDZ;
  static constexpr int NV = DIM * NbrSlots<DIM>::NB;     // V stencil values behind M
  static constexpr int NE = 2 * B + NV;                  // ring entry: yu, yv, V stencil
  static constexpr int E_YU = 0, E_YV = B, E_VS = 2 * B;
  // prep ring entry (latency-bound shapes: the producers also build the
  // pair's dense inputs): c, yv + M^T c, dpbar-row rhs, P M, D faces block
  static constexpr int NEP = 2 * NF + 1 + NF * NF + NT;
  static constexpr int P_C = 0, P_XR = NF, P_YC = 2 * NF, P_PM = 2 * NF + 1, P_D = 2 * NF + 1 + NF * NF;
};

// record group g0.. of (pair i, cell m): N values, 16 bytes per store
template <class R, int N>
__device__ __forceinline__ void stg_rec(R* scratch, int64_t M, int64_t m, int i, int rs, int e0, const R (&v)[N]) {
  constexpr int VW = 16 / (int)sizeof(R);
  static_assert(N % VW == 0, "stg_rec: N % VW");
  R* p = scratch + (((int64_t)i * (rs / VW) + e0 / VW) * M + m) * VW;
#pragma unroll
  for (int k = 0; k < N / VW; ++k) {
    if constexpr (sizeof(R) == 4)
      *reinterpret_cast<float4*>(p + (int64_t)k * M * VW) = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    else
      *reinterpret_cast<double2*>(p + (int64_t)k * M * VW) = make_double2(v[2 * k], v[2 * k + 1]);
  }
}

// the consumer's dense inputs are built by the producers on the P = 4 shape
__host__ __device__ constexpr bool fwd_prep(int P) { return P == 4; }
template <int DIM>
__host__ __device__ constexpr int fwd_ring_entry(int P) { return fwd_prep(P) ? Line<DIM>::NEP : Line<DIM>::NE; }

__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// per-cell constants shared by the smoother kernels
template <int DIM, bool PER, class R>
struct LineCell {
  static constexpr int NF = 2 * DIM;
  CellGeo<DIM, PER, R> cg;
  R isig;
  __device__ __forceinline__ LineCell(const Ix<DIM, PER>& ix, R h, int64_t m, int o0, int o1, int o2, int mod, int m1,
                                      int m2)
      : cg(ix, h, m, o0, o1, o2, mod, m1, m2) {
    R sigma = R(0);
#pragma unroll
    for (int q = 0; q < NF; ++q) sigma += cg.gcol[q] * cg.gcol[q];
    isig = R(1) / sigma;
    sig = sigma;
  }
  R sig;
  // SingularBlock thresholds of the pairs with shift alpha (see ldlt)
  __device__ __forceinline__ void piv_ref(R idt2, R alpha, R& tf, R& ts) const {
    const R d = idt2 + alpha;
    tf = R(1e-12) * d;
    ts = R(1e-12) * sig / d;
  }
  // P x on the unknown faces (g is zero on walls)
  __device__ __forceinline__ void projP(R (&x)[NF]) const {
    R d = R(0);
#pragma unroll
    for (int q = 0; q < NF; ++q) d += cg.gcol[q] * x[q];
    d *= isig;
#pragma unroll
    for (int q = 0; q < NF; ++q) x[q] = cg.wall[q] ? R(0) : x[q] - cg.gcol[q] * d;
  }
};

// dense per-pair inputs of the time-line elimination (used by the consumer,
// or by the producers in prep mode); FFMA2 lane pairs over columns 2h, 2h+1
template <int DIM, bool PER, class R>
struct PairAlg {
  static constexpr int NF = 2 * DIM, B = NF + 1, NH = NF / 2, NB = NbrSlots<DIM>::NB;
  using P2 = R2<R>;
  __device__ __forceinline__ static R lo_hi(const P2& v, int e) { return e ? v.y : v.x; }
  // c = P yu + g yu_p / sigma
  __device__ __forceinline__ static void cvec(const LineCell<DIM, PER, R>& lc, const R (&yu)[B], R (&cv)[NF]) {
#pragma unroll
    for (int q = 0; q < NF; ++q) cv[q] = yu[q];
    lc.projP(cv);
#pragma unroll
    for (int q = 0; q < NF; ++q) cv[q] += lc.cg.gcol[q] * yu[NF] * lc.isig;
  }
  // M from the V stencil, then P M (column pairs) and xr = yv + M^T c
  __device__ __forceinline__ static void mats(const LineCell<DIM, PER, R>& lc, R c0, R idt, const R (&VC)[DIM][NB],
                                              const R (&yv)[B], const R (&cv)[NF], P2 (&PM)[NF][NH],
                                              R (&xr)[NF]) {
    const auto& cg = lc.cg;
    R Mx[NF][NF];
    jac_cached<DIM, R>(c0, idt, VC, cg.wall, Mx);
    P2 Mp[NF][NH];
#pragma unroll
    for (int t = 0; t < NF; ++t)
#pragma unroll
      for (int h = 0; h < NH; ++h) Mp[t][h] = p2(Mx[t][2 * h], Mx[t][2 * h + 1]);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      P2 s2 = p2(yv[2 * h], yv[2 * h + 1]);
#pragma unroll
      for (int t = 0; t < NF; ++t) s2 = fma2s(cv[t], Mp[t][h], s2);
      xr[2 * h] = s2.x;
      xr[2 * h + 1] = s2.y;
    }
    // P M column pairs: d = isig g^T M, PM = M - g d on the unknown rows
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      P2 d = p2(R(0), R(0));
#pragma unroll
      for (int q = 0; q < NF; ++q) d = fma2s(cg.gcol[q], Mp[q][h], d);
      d = mul2s(lc.isig, d);
#pragma unroll
      for (int a = 0; a < NF; ++a) PM[a][h] = cg.wall[a] ? p2(R(0), R(0)) : fma2s(-cg.gcol[a], d, Mp[a][h]);
    }
  }
  // D faces block (lower triangle): (PM)^T PM + [nx] P/dt^2 + alpha / wall identity
  __device__ __forceinline__ static void diag(const LineCell<DIM, PER, R>& lc, const R (&gs)[NF], R idt2, R alpha,
                                              bool nx, const P2 (&PM)[NF][NH], R (&T)[B][B]) {
    const auto& cg = lc.cg;
#pragma unroll
    for (int a = 0; a < NF; ++a)
#pragma unroll
      for (int h = 0; h <= (a >> 1); ++h) {
        P2 acc = p2(R(0), R(0));
#pragma unroll
        for (int t = 0; t < NF; ++t) acc = fma2s(lo_hi(PM[t][a >> 1], a & 1), PM[t][h], acc);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = 2 * h + e;
          if (b > a) continue;
          R s = lo_hi(acc, e);
          if (nx) s -= cg.gcol[a] * gs[b];
          if (a == b) s += cg.wall[a] ? R(1) : alpha + (nx ? idt2 : R(0));
          T[a][b] = s;
        }
      }
  }
};

// ring stages for P producer groups: a multiple of P, at least 3
__host__ __device__ constexpr int ring_stages(int P) { return P == 1 ? 3 : (P == 2 ? 4 : P); }

// k_scgs_fwd<TM, P>: TM cells per CTA, P producer groups of TM threads
// (group p builds pairs i = p mod P, so the coarse levels -- few cells, long
// time lines -- get P-fold producer parallelism), one consumer group.
// resident CTAs per SM the register budget is sized for
#ifndef SMK_FWD_MINB
#define SMK_FWD_MINB 4
#endif
#ifndef SMK_FWD_MINB_64X2
#define SMK_FWD_MINB_64X2 2
#endif
__host__ __device__ constexpr int fwd_min_blocks_f32(int TM, int P) {
  // 128 registers on P <= 2 (more CTAs spill: measured slower); TM 64 / P 1
  // at SMK_FWD_MINB CTAs per SM (tuning builds)
  return P == 1 ? (TM == 64 ? SMK_FWD_MINB : 512 / (2 * TM)) : (P == 2 ? (TM == 64 ? SMK_FWD_MINB_64X2 : 5) : 2);
}
__host__ __device__ constexpr int fwd_min_blocks(int TM, int P, int esz) {
  return esz == 8 ? (fwd_min_blocks_f32(TM, P) / 2 > 0 ? fwd_min_blocks_f32(TM, P) / 2 : 1) : fwd_min_blocks_f32(TM, P);
}

// FMT: hand-off format 0 factored, 1 compact (both [i][e][m]), 2 record
template <int DIM, bool PER, class R, int TM, int P, bool HR, int NX, int FMT>
__global__ void __launch_bounds__((P + 1) * TM, fwd_min_blocks(TM, P, sizeof(R)))
    k_scgs_fwd(KktCtx<DIM, PER, R> cx, ResP<R> rhs, int o0, int o1, int o2, int mod, int m0, int m1,
               int m2, R* __restrict__ scratch, int* flag) {
  using LN = Line<DIM>;
  using PA = PairAlg<DIM, PER, R>;
  constexpr int NF = LN::NF, B = LN::B, NB = NbrSlots<DIM>::NB;
  constexpr bool PREP = fwd_prep(P);
  constexpr bool CMP = FMT == 1, REC = FMT == 2;
  static_assert(!REC || PREP, "record hand-off needs the prep shape");
  constexpr int NE = fwd_ring_entry<DIM>(P);
  constexpr int S = ring_stages(P);
  constexpr int NT = 2 * TM;   // threads per named barrier: one producer group + the consumers
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* ring = reinterpret_cast<R*>(smem_raw);   // [S][NE][TM]
  const auto& ix = cx.ix;
  const int N = cx.N;
  const int64_t M = (int64_t)m0 * m1 * m2;
  const int grp = threadIdx.x / TM;           // 0..P-1 producers, P consumers
  const bool producer = grp < P;
  const int lane = threadIdx.x - grp * TM;
  const int64_t m = (int64_t)blockIdx.x * TM + lane;
  const bool act = m < M;   // inactive threads still take part in every barrier
  const LineCell<DIM, PER, R> lc(ix, cx.h, act ? m : 0, o0, o1, o2, mod, m1, m2);
  const auto& cg = lc.cg;
  const R c0 = cx.c0;
  const R idt = cx.idt;
#if SMK_HANDOFF_BLOCKED
  R* const hbase = scratch + LN::cell_base(act ? m : 0);
  const int64_t hstride = LN::pair_stride(M);
  auto sc = [&](int i, int e) -> R* { return hbase + (int64_t)i * hstride + e * LN::HB; };
#else
  auto sc = [&](int i, int e) -> R* { return scratch + ((int64_t)i * LN::SE + e) * M + m; };
#endif
  auto slot = [&](int i, int e) -> R* { return ring + ((i % S) * NE + e) * TM + lane; };
  const R idt2 = idt * idt;
  R gs[NF];   // g * idt^2 / sigma: P idt^2 = idt^2 I - g gs^T on the unknown faces
#pragma unroll
  for (int q = 0; q < NF; ++q) gs[q] = cg.gcol[q] * lc.isig * idt2;
  auto alpha_of = [&](int ip) -> R { return (cx.t0 + ip < cx.Ng - 1) ? cx.kr : R(0); };

  if (producer) {
    const Loc<DIM, PER, NX> L(ix, cg.c);
    R vp[NF];   // V_{i-1} at the own faces (carried when one group builds every pair)
    if (P == 1) {
#pragma unroll
      for (int q = 0; q < NF; ++q) vp[q] = act ? cx.v0.c[q >> 1][L.of[q]] : R(0);
    }
    for (int i = grp; i < N; i += P) {
      if (i >= S) nb_sync(1 + S + i % S, NT);   // EMPTY: the consumers released pair i - S
      if (act) {
        if (P > 1) {
          const Face3<R> Vp = i == 0 ? cx.v0 : cx.frame(cx.V, i - 1);
#pragma unroll
          for (int q = 0; q < NF; ++q) vp[q] = Vp.c[q >> 1][L.of[q]];
        }
        R VC[DIM][NB], UC[DIM][NB];
        R yu[B], yv[B];
        load_nbr<DIM, PER, R>(ix, L, cx.frame(cx.V, i), VC);
        load_nbr<DIM, PER, R>(ix, L, cx.frame(cx.U, i), UC);
        pair_rows<DIM, PER, R, true, false, HR>(cx, L, cg.wall, i, VC, UC, vp, rhs, yu, yv);
#pragma unroll
        for (int q = 0; q < B; ++q) {
          yu[q] = -yu[q];
          yv[q] = -yv[q];
          if constexpr (!REC) *sc(i, (CMP ? LN::Y0C : LN::Y0) + q) = yu[q];
        }
        if constexpr (REC) {
          // M_i and yu_i for the backward's step of pair i - 1 (M from the
          // same function and inputs the backward used to rebuild it from)
          R Mx[NF][NF], mr[NF * NF], yr[LN::NY];
          jac_cached<DIM, R>(c0, idt, VC, cg.wall, Mx);
#pragma unroll
          for (int a = 0; a < NF; ++a)
#pragma unroll
            for (int b = 0; b < NF; ++b) mr[a * NF + b] = Mx[a][b];
#pragma unroll
          for (int q = 0; q < LN::NY; ++q) yr[q] = q < B ? yu[q] : R(0);
          stg_rec<R, NF * NF>(scratch, M, m, i, LN::RS, LN::R_M, mr);
          stg_rec<R, LN::NY>(scratch, M, m, i, LN::RS, LN::R_Y, yr);
        }
        if (P == 1) {
#pragma unroll
          for (int q = 0; q < NF; ++q) vp[q] = VC[q >> 1][(q & 1) + 1];
        }
        if constexpr (PREP) {
          R cv[NF], xrv[NF], Dl[B][B];
          typename PA::P2 PM[NF][NF / 2];
          PA::cvec(lc, yu, cv);
          PA::mats(lc, c0, idt, VC, yv, cv, PM, xrv);
          PA::diag(lc, gs, idt2, alpha_of(i), i + 1 < N, PM, Dl);
#pragma unroll
          for (int q = 0; q < NF; ++q) {
            *slot(i, LN::P_C + q) = cv[q];
            *slot(i, LN::P_XR + q) = xrv[q];
          }
          *slot(i, LN::P_YC) = yv[NF];
#pragma unroll
          for (int a = 0; a < NF; ++a)
#pragma unroll
            for (int h = 0; h < NF / 2; ++h) {
              *slot(i, LN::P_PM + a * NF + 2 * h) = PM[a][h].x;
              *slot(i, LN::P_PM + a * NF + 2 * h + 1) = PM[a][h].y;
            }
#pragma unroll
          for (int a = 0; a < NF; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) *slot(i, LN::P_D + a * (a + 1) / 2 + b) = Dl[a][b];
        } else {
#pragma unroll
          for (int q = 0; q < B; ++q) {
            *slot(i, LN::E_YU + q) = yu[q];
            *slot(i, LN::E_YV + q) = yv[q];
          }
#pragma unroll
          for (int a = 0; a < DIM; ++a)
#pragma unroll
            for (int sl = 0; sl < NB; ++sl) *slot(i, LN::E_VS + a * NB + sl) = VC[a][sl];
        }
      }
      nb_arrive(1 + i % S, NT);   // FULL
    }
    return;
  }

  // ---------------- consumers ----------------
  // Per pair, the saddle block K' = [[D~_i, g], [g^T, 0]] (symmetric form of
  // the v-row / dpbar-row block) is factored K' = L diag(d) L^T in place; z_i
  // solves K' z = [rhs; -ycell].  The coupling to the next pair enters only
  // through Y = L^-1 [P M_{i+1}; 0]:  D~_{i+1} = D_{i+1} - Y^T diag(1/d) Y / dt^2,
  // and the back substitution needs W_i dv = K'^-1 [-P M_{i+1} dv / dt; 0],
  // so the pair hands off only D~_i and its rhs -- no explicit W.
  const R tinyv = R(1e-12);   // relative SingularBlock threshold of dense_solve (the alpha = 0 pair)
  R tf, ts;                    // ldlt thresholds of the alpha = K/r pairs
  lc.piv_ref(idt2, cx.kr, tf, ts);
  // The dense block algebra below runs on lane pairs (columns 2h, 2h+1):
  // FFMA2 with a broadcast scalar in fp32, each lane rounded exactly like the
  // scalar FFMA of the same expression (same operand order, same summation
  // order), so the pairing does not change the results.
  constexpr int NH = NF / 2;
  using P2 = R2<R>;
  auto lo_hi = [](const P2& v, int e) -> R { return e ? v.y : v.x; };
  // D faces block of pair ip (lower triangle)
  auto diag_block = [&](int ip, const P2 (&PM)[NF][NH], R (&T)[B][B]) {
    if constexpr (PREP) {
#pragma unroll
      for (int a = 0; a < NF; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) T[a][b] = *slot(ip, LN::P_D + a * (a + 1) / 2 + b);
    } else {
      PA::diag(lc, gs, idt2, alpha_of(ip), ip + 1 < N, PM, T);
    }
  };
  // c = P yu + g yu_p / sigma of pair i
  auto c_of = [&](int i, R (&cv)[NF]) {
    if constexpr (PREP) {
#pragma unroll
      for (int q = 0; q < NF; ++q) cv[q] = *slot(i, LN::P_C + q);
    } else {
      R yu[B];
#pragma unroll
      for (int q = 0; q < B; ++q) yu[q] = *slot(i, LN::E_YU + q);
      PA::cvec(lc, yu, cv);
    }
  };
  // P M_i, the partial rhs yv + M^T c and the dpbar-row rhs of pair i
  auto mats_of = [&](int i, const R (&cv)[NF], P2 (&PM)[NF][NH], R (&xrr)[NF], R& yc) {
    if constexpr (PREP) {
#pragma unroll
      for (int q = 0; q < NF; ++q) xrr[q] = *slot(i, LN::P_XR + q);
      yc = *slot(i, LN::P_YC);
#pragma unroll
      for (int a = 0; a < NF; ++a)
#pragma unroll
        for (int h = 0; h < NH; ++h)
          PM[a][h] = p2(*slot(i, LN::P_PM + a * NF + 2 * h), *slot(i, LN::P_PM + a * NF + 2 * h + 1));
    } else {
      R VC[DIM][NB], yv[B];
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int sl = 0; sl < NB; ++sl) VC[a][sl] = *slot(i, LN::E_VS + a * NB + sl);
#pragma unroll
      for (int q = 0; q < B; ++q) yv[q] = *slot(i, LN::E_YV + q);
      PA::mats(lc, c0, idt, VC, yv, cv, PM, xrr);
      yc = yv[NF];
    }
  };
  R T[B][B];      // lower triangle: D~ of the current pair, then its L
  R xr[NF];       // partial rhs yv + M^T c of the current pair
  R sz[NF];       // (P M)^T z_{i-1}
  R ycell;        // its dpbar-row rhs
  bool ok = true;
  nb_sync(1 + 0, NT);
  {
    P2 PM[NF][NH];
    R cv[NF];
    c_of(0, cv);
    mats_of(0, cv, PM, xr, ycell);
    diag_block(0, PM, T);
#pragma unroll
    for (int a = 0; a < NF; ++a) sz[a] = R(0);
  }
  // rhs of pair i (symmetric form): faces xr - c_{i+1}/dt + sz/dt, -ycell
  auto build_rhs = [&](const R (&cn)[NF], R (&b)[B]) {
#pragma unroll
    for (int a = 0; a < NF; ++a) {
      R s = cg.wall[a] ? R(0) : xr[a] - cn[a] * idt;
      b[a] = s + sz[a] * idt;
    }
    b[NF] = -ycell;
  };
  // hand-off of pair i to the backward pass: the Schur-updated faces block
  // (before the saddle is appended and factored) and the pair's rhs; the
  // backward re-runs the identical factorisation, so this is 35 values per
  // pair instead of L, 1/d and z (42)
  auto store_pair = [&](int i, const R (&b)[B]) {
#pragma unroll
    for (int r = 0; r < NF; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) *sc(i, LN::T0 + r * (r + 1) / 2 + c) = T[r][c];
#pragma unroll
    for (int r = 0; r < B; ++r) *sc(i, LN::B0 + r) = b[r];
  };
  // factored hand-off (small colours): L, 1/d and z of pair i
  auto store_factors = [&](int i, const R (&dinv)[B], const R (&z)[B]) {
    if constexpr (REC) {
      R v[LN::NLDZ];
#pragma unroll
      for (int r = 1; r < B; ++r)
#pragma unroll
        for (int c = 0; c < r; ++c) v[r * (r - 1) / 2 + c] = T[r][c];
#pragma unroll
      for (int r = 0; r < B; ++r) {
        v[LN::NL + r] = dinv[r];
        v[LN::NL + B + r] = z[r];
      }
#pragma unroll
      for (int e = LN::NL + 2 * B; e < LN::NLDZ; ++e) v[e] = R(0);
      stg_rec<R, LN::NLDZ>(scratch, M, m, i, LN::RS, LN::R_L, v);
      return;
    }
#pragma unroll
    for (int r = 1; r < B; ++r)
#pragma unroll
      for (int c = 0; c < r; ++c) *sc(i, LN::L0 + r * (r - 1) / 2 + c) = T[r][c];
#pragma unroll
    for (int r = 0; r < B; ++r) {
      *sc(i, LN::D0 + r) = dinv[r];
      *sc(i, LN::Z0 + r) = z[r];
    }
  };
  auto saddle = [&]() {
#pragma unroll
    for (int a = 0; a < NF; ++a) T[NF][a] = cg.gcol[a];
    T[NF][NF] = R(0);
  };
  for (int i = 0; i < N - 1; ++i) {
    nb_arrive(1 + S + i % S, NT);   // EMPTY: pair i's stage was consumed at step i-1
    nb_sync(1 + (i + 1) % S, NT);   // FULL: pair i+1 ready
    R b[B], dinv[B], cn[NF];
    c_of(i + 1, cn);
    build_rhs(cn, b);
    if (CMP && act) store_pair(i, b);
    saddle();
    ok &= ldlt<R, B>(T, dinv, tf, ts);
    ldlt_solve<R, B>(T, dinv, b);
    if (!CMP && act) store_factors(i, dinv, b);
    P2 PM[NF][NH];
    mats_of(i + 1, cn, PM, xr, ycell);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      P2 s2 = p2(R(0), R(0));
#pragma unroll
      for (int t = 0; t < NF; ++t) s2 = fma2s(b[t], PM[t][h], s2);
      sz[2 * h] = s2.x;
      sz[2 * h + 1] = s2.y;
    }
    // Y = L^-1 [PM; 0] on column pairs (row NF starts at 0)
    P2 Y[B][NH];
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        P2 s2 = r < NF ? PM[r][h] : p2(R(0), R(0));
#pragma unroll
        for (int c = 0; c < r; ++c) s2 = fma2s(-T[r][c], Y[c][h], s2);
        Y[r][h] = s2;
      }
    diag_block(i + 1, PM, T);
    // Schur complement of the eliminated pair: - Y^T diag(1/d) Y / dt^2
#pragma unroll
    for (int k = 0; k < B; ++k) dinv[k] *= idt2;
#pragma unroll
    for (int a = 0; a < NF; ++a) {
      R DY[B];
#pragma unroll
      for (int k = 0; k < B; ++k) DY[k] = lo_hi(Y[k][a >> 1], a & 1) * dinv[k];
#pragma unroll
      for (int h = 0; h <= (a >> 1); ++h) {
        P2 s2 = p2(R(0), R(0));
#pragma unroll
        for (int k = 0; k < B; ++k) s2 = fma2s(DY[k], Y[k][h], s2);
        T[a][2 * h] -= s2.x;
        if (2 * h + 1 <= a) T[a][2 * h + 1] -= s2.y;
      }
    }
  }
  {
    // last pair: no coupling to a next pair; only z is needed
    const int i = N - 1;
    R b[B], cn[NF];
#pragma unroll
    for (int a = 0; a < NF; ++a) cn[a] = R(0);
    build_rhs(cn, b);
    if (CMP && act) store_pair(i, b);
    saddle();
    if (cx.t0 + i < cx.Ng - 1) {
      R dinv[B];
      ok &= ldlt<R, B>(T, dinv, tf, ts);
      ldlt_solve<R, B>(T, dinv, b);
    } else {
      // alpha = 0: D~ is singular along M^-1 g; the saddle is not -> pivot
      ok &= saddle_solve_pivot<R, B>(T, b, tinyv);
    }
    if (REC && act) {
      R v[LN::NLDZ];   // only z is read for the last pair
#pragma unroll
      for (int e = 0; e < LN::NLDZ; ++e) v[e] = R(0);
#pragma unroll
      for (int r = 0; r < B; ++r) v[LN::NL + B + r] = b[r];
      stg_rec<R, LN::NLDZ>(scratch, M, m, i, LN::RS, LN::R_L, v);
    } else if (!CMP && act) {
#pragma unroll
      for (int r = 0; r < B; ++r) *sc(i, LN::Z0 + r) = b[r];
    }
  }
  if (act && !ok) atomicExch(flag, 1);
}

// Back substitution of one colour, pair i = N-1 .. 0:
//   refactor pair i's saddle from the handed-off D~ faces block (the same
//   LDL^T / pivoted solve as the forward pass, so bitwise the same factors),
//   z_i = K'^-1 b_i, then dv, dpbar of pair i = z_i - K'^-1 [-P M_{i+1} dv_{i+1}/dt; 0]
//   (M_{i+1} recomputed from V), then du, dp of pair i+1 from dv_{i+1},
//   dv_{i+2}, yu_{i+1} and the same M_{i+1} dv_{i+2}.
// Writes omega * deltas to xout [2 * pair + (0: u-block, 1: v-block)][entry][m].
// PIPE (small colours, latency-bound): the loads of step i-1 (its hand-off,
// u-rows and V stencil) are issued before step i computes, so one memory
// latency overlaps one step instead of adding to it.

// ---- mbarrier + 1D bulk async copy (TMA engine) helpers -------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n }" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int DIM, class R, bool CMP>
struct BackIn {
  static constexpr int NF = 2 * DIM, B = NF + 1, NB = NbrSlots<DIM>::NB;
  // compact: D~ faces block + rhs; factored: L + 1/d + z
  R t[CMP ? NF * (NF + 1) / 2 : B * (B - 1) / 2], b[B], d[CMP ? 1 : B], yu[B];
  R VC[DIM][NB];
  // FUSE: the in-place targets of the step (U, P of pair i+1, PBAR of pair i),
  // loaded with the step's other inputs so no extra latency joins the chain,
  // and the frame pointers of their stores (one 64-bit product per array and
  // step instead of one per access)
  R uo[NF], po, pbo;
  R* fu[DIM];
  R* fv[DIM];
  R* fp;
  R* fpb;
};

// FUSE (red-black, where every face of the grid has exactly one cell of the
// colour): no delta buffer and no apply pass -- U, P and PBAR take
// x += omega dx in place (no thread of the pass reads them), and V, which the
// pass's stencils read, is written whole into the other buffer of a pair
// (so.V = the pass's output, cx.V its input): Vout = Vin + omega dv at every
// face.  Same arithmetic as k_scgs_apply, so bitwise equal to the unfused
// pass.
// resident CTAs per SM the big-colour (compact) variant is register-capped
// for (tuning builds: -DSMK_BACK_MINB=n)
#ifndef SMK_BACK_MINB
#define SMK_BACK_MINB 1
#endif
// TMA (compact + fused, 128-thread CTAs = two 64-cell hand-off blocks, the
// host launches it only when the colour is a multiple of 128 cells): the
// compact entries of pair i for the CTA's two blocks (2 x 35 x 64 values,
// contiguous per block) arrive by two 1D bulk async copies issued NS - 1 steps
// ahead by thread 0 into an NS-stage shared-memory ring (fp32: 3), completion on an
// mbarrier per stage; the thread reads its t / b / yu from shared memory, so
// the 42 hand-off loads per step and their address math leave the serial
// chain.  One __syncthreads per step frees the stage the next copy targets.
// ring depth of the TMA-staged hand-off: the copy of pair i - (NS - 1) is
// issued at step i, so NS - 1 pairs (2 x 8.96 KB each in fp32) are in flight
// per CTA while a step computes
#ifndef SMK_BACK_STAGES
#define SMK_BACK_STAGES 3
#endif
template <class R>
__host__ __device__ constexpr int back_tma_stages() { return sizeof(R) == 4 ? SMK_BACK_STAGES : 2; }
template <int DIM, class R>
__host__ __device__ constexpr size_t back_tma_smem() {
  return (size_t)back_tma_stages<R>() * 2 * Line<DIM>::NCMP * Line<DIM>::HB * sizeof(R);
}
template <int DIM, bool PER, class R, bool PIPE, int NX, bool CMP, bool FUSE, bool TMA = false>
__global__ void __launch_bounds__(128, CMP ? SMK_BACK_MINB : 1) k_scgs_back(KktCtx<DIM, PER, R> cx, int o0, int o1, int o2, int mod, int m0,
                                                   int m1, int m2, R omega, const R* __restrict__ scratch,
                                                   R* __restrict__ xout, StP<R> so) {
  using LN = Line<DIM>;
  constexpr int NF = LN::NF, B = LN::B, NTT = CMP ? LN::NT : LN::NL;
  static_assert(!TMA || (CMP && FUSE && !PIPE && SMK_HANDOFF_BLOCKED), "TMA: compact fused blocked hand-off only");
  const auto& ix = cx.ix;
  const int N = cx.N;
  const int64_t M = (int64_t)m0 * m1 * m2;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;   // TMA: never taken (M % 128 == 0)
  extern __shared__ __align__(128) unsigned char tsm_raw[];
  constexpr int NS = back_tma_stages<R>();
  __shared__ __align__(8) uint64_t tbar[NS];
  constexpr int NC = LN::NCMP, HB = LN::HB;
  R* const tring = reinterpret_cast<R*>(tsm_raw);   // [stage][block][NC][HB]
  const int tblk = threadIdx.x / HB, tl = threadIdx.x % HB;
  const R* const tr0 = tring + tblk * NC * HB + tl;   // stage 0 of this thread's block; stage s at + 2 s NC HB
  // pair i lives in stage (N - 1 - i) % NS, in the ((N - 1 - i) / NS)-th use of its barrier
  auto tstage = [&](int i) -> int { return (N - 1 - i) % NS; };
  auto tmem = [&](int i, int e) -> R { return tr0[tstage(i) * 2 * NC * HB + e * HB]; };
  auto tissue = [&](int i) {   // thread 0: pair i's compact entries of both blocks
    if (threadIdx.x != 0 || i < 0) return;
    const uint32_t bytes = NC * HB * sizeof(R);
    const int sg = tstage(i);
    uint64_t* bar = &tbar[sg];
    mbar_expect_tx(bar, 2 * bytes);
    const int64_t b0 = (int64_t)blockIdx.x * 2;
    for (int j = 0; j < 2; ++j)
      bulk_g2s(tring + (sg * 2 + j) * NC * HB, scratch + (int64_t)i * LN::pair_stride(M) + (b0 + j) * LN::SE * HB,
               bytes, bar);
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      for (int k = 0; k < NS; ++k) mbar_init(&tbar[k], 1);
      mbar_fence_init();
    }
    __syncthreads();
    for (int k = 0; k < NS - 1; ++k) tissue(N - 1 - k);
  }
  const LineCell<DIM, PER, R> lc(ix, cx.h, m, o0, o1, o2, mod, m1, m2);
  const auto& cg = lc.cg;
  const Loc<DIM, PER, NX> L(ix, cg.c);
  const R idt = cx.idt;
  const R tinyv = R(1e-12);   // relative SingularBlock threshold of dense_solve (the alpha = 0 pair)
#if SMK_HANDOFF_BLOCKED
  const R* const hbase = scratch + LN::cell_base(m);
  const int64_t hstride = LN::pair_stride(M);
  auto sc = [&](int i, int e) -> R { return __ldg(hbase + (int64_t)i * hstride + e * LN::HB); };
#else
  auto sc = [&](int i, int e) -> R { return __ldg(scratch + ((int64_t)i * LN::SE + e) * M + m); };
#endif
  // inputs of step i: hand-off of pair i; u-rows of pair i+1 and the V
  // stencil of frame i+1 (i = -1: only the u-rows / stencil of pair 0)
  auto fetch = [&](int i, BackIn<DIM, R, CMP>& in) {
    if constexpr (TMA) {
      // yu_{i+1} from pair i+1's stage (landed last step), then free that
      // stage and launch pair i-1 into it; the V stencil and the targets by
      // plain loads; pair i's t / b once its copy has landed
      if (i + 1 < N) {
#pragma unroll
        for (int q = 0; q < B; ++q) in.yu[q] = tmem(i + 1, LN::Y0C + q);
      }
      __syncthreads();
      tissue(i - (NS - 1));   // into pair i+1's stage, which every thread has left
      if (i + 1 < N) load_nbr<DIM, PER, R>(ix, L, cx.frame(cx.V, i + 1), in.VC);
      if (i + 1 < N) {
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          in.fu[k] = so.U[k] + (int64_t)(i + 1) * cx.nf[k];
          in.fv[k] = so.V[k] + (int64_t)(i + 1) * cx.nf[k];
        }
        in.fp = so.P + (int64_t)(i + 1) * cx.nc;
#pragma unroll
        for (int q = 0; q < NF; ++q) in.uo[q] = cg.wall[q] ? R(0) : in.fu[q >> 1][L.of[q]];
        in.po = in.fp[L.co];
      }
      if (i >= 0) {
        in.fpb = so.PB + (int64_t)i * cx.nc;
        in.pbo = in.fpb[L.co];
        mbar_wait(&tbar[tstage(i)], (uint32_t)(((N - 1 - i) / NS) & 1));
#pragma unroll
        for (int e = 0; e < NTT; ++e) in.t[e] = tmem(i, LN::T0 + e);
#pragma unroll
        for (int r = 0; r < B; ++r) in.b[r] = tmem(i, LN::B0 + r);
      }
      return;
    }
    if (i >= 0) {
      if (CMP || i + 1 < N) {
#pragma unroll
        for (int e = 0; e < NTT; ++e) in.t[e] = sc(i, (CMP ? LN::T0 : LN::L0) + e);
      }
#pragma unroll
      for (int r = 0; r < B; ++r) in.b[r] = sc(i, (CMP ? LN::B0 : LN::Z0) + r);
      if (!CMP) {
#pragma unroll
        for (int r = 0; r < B; ++r) in.d[r] = sc(i, LN::D0 + r);
      }
    }
    if (i + 1 < N) {
#pragma unroll
      for (int q = 0; q < B; ++q) in.yu[q] = sc(i + 1, (CMP ? LN::Y0C : LN::Y0) + q);
      load_nbr<DIM, PER, R>(ix, L, cx.frame(cx.V, i + 1), in.VC);
    }
    if constexpr (FUSE) {
      if (i + 1 < N) {
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          in.fu[k] = so.U[k] + (int64_t)(i + 1) * cx.nf[k];
          in.fv[k] = so.V[k] + (int64_t)(i + 1) * cx.nf[k];
        }
        in.fp = so.P + (int64_t)(i + 1) * cx.nc;
#pragma unroll
        for (int q = 0; q < NF; ++q) in.uo[q] = cg.wall[q] ? R(0) : in.fu[q >> 1][L.of[q]];
        in.po = in.fp[L.co];
      }
      if (i >= 0) {
        in.fpb = so.PB + (int64_t)i * cx.nc;
        in.pbo = in.fpb[L.co];
      }
    }
  };
  // t = M dv from a V stencil
  auto mdot = [&](const BackIn<DIM, R, CMP>& in, const R (&dv)[NF], R (&t)[NF]) {
    R Mi[NF][NF];
    jac_cached<DIM, R>(cx.c0, idt, in.VC, cg.wall, Mi);
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < NF; ++k) s += Mi[q][k] * dv[k];
      t[q] = s;
    }
  };
  // du, dp of pair ip from dv_ip (dvi), yu_ip and t = M_ip dv_{ip+1}
  auto u_delta = [&](int ip, const BackIn<DIM, R, CMP>& in, const R (&dvi)[NF], const R (&t)[NF]) {
    const auto& yu = in.yu;
    R a[NF];
    R ga = R(0);
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      R s = yu[q] + dvi[q] * idt - t[q];
      a[q] = cg.wall[q] ? R(0) : s;
      ga += cg.gcol[q] * a[q];
    }
    const R dp = (ga - yu[NF]) * lc.isig;
    if constexpr (FUSE) {
#pragma unroll
      for (int q = 0; q < NF; ++q)
        if (!cg.wall[q]) in.fu[q >> 1][L.of[q]] = in.uo[q] + omega * (cg.gcol[q] * dp - a[q]);
      in.fp[L.co] = in.po + omega * dp;
    } else {
      R* xo = xout + (int64_t)(2 * ip) * B * M + m;
#pragma unroll
      for (int q = 0; q < NF; ++q) xo[(int64_t)q * M] = cg.wall[q] ? R(0) : omega * (cg.gcol[q] * dp - a[q]);
      xo[(int64_t)NF * M] = omega * dp;
    }
  };
  // FUSE: V of frame ip (pair ip) = its input value (own faces of the frame's
  // stencil) + omega dv
  auto v_store = [&](int ip, const BackIn<DIM, R, CMP>& in, const R (&dv)[NF]) {
#pragma unroll
    for (int q = 0; q < NF; ++q)
      if (!cg.wall[q]) in.fv[q >> 1][L.of[q]] = in.VC[q >> 1][(q & 1) + 1] + omega * dv[q];
  };
  R xn[NF];   // dv of pair i+1
  R t[NF];    // M_{i+1} dv_{i+1}
#pragma unroll
  for (int q = 0; q < NF; ++q) xn[q] = R(0);
  BackIn<DIM, R, CMP> cur, nxt;
  if (PIPE) fetch(N - 1, nxt);
  for (int i = N - 1; i >= -1; --i) {
    if (PIPE) {
      cur = nxt;
      if (i - 1 >= -1) fetch(i - 1, nxt);
    } else {
      fetch(i, cur);
    }
    if (i + 1 < N) mdot(cur, xn, t);
    if (FUSE && i + 1 < N) v_store(i + 1, cur, xn);
    if (i < 0) {
      R zero[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) zero[q] = R(0);
      u_delta(0, cur, zero, t);   // dv_0 = 0 (pinned / frozen halo)
      break;
    }
    R T[B][B], dinv[B], xb[B];
#pragma unroll
    for (int r = 0; r < B; ++r) xb[r] = cur.b[r];
    if (CMP) {
      // pair i's saddle, refactored exactly as in the forward pass
#pragma unroll
      for (int r = 0; r < NF; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) T[r][c] = cur.t[r * (r + 1) / 2 + c];
#pragma unroll
      for (int a = 0; a < NF; ++a) T[NF][a] = cg.gcol[a];
      T[NF][NF] = R(0);
      if (i + 1 < N || cx.t0 + i < cx.Ng - 1) {
        ldlt<R, B>(T, dinv, R(0), R(0));   // same factors as the forward; its flag is not re-raised
        ldlt_solve<R, B>(T, dinv, xb);
      } else {
        saddle_solve_pivot<R, B>(T, xb, tinyv);
      }
    } else if (i + 1 < N) {
      // stored factors
#pragma unroll
      for (int r = 1; r < B; ++r)
#pragma unroll
        for (int c = 0; c < r; ++c) T[r][c] = cur.t[r * (r - 1) / 2 + c];
#pragma unroll
      for (int r = 0; r < B; ++r) dinv[r] = cur.d[r];
    }
    if (i + 1 < N) {
      R wf[NF], w[B];
#pragma unroll
      for (int q = 0; q < NF; ++q) wf[q] = t[q];
      lc.projP(wf);
#pragma unroll
      for (int q = 0; q < NF; ++q) w[q] = -wf[q] * idt;
      w[NF] = R(0);
      ldlt_solve<R, B>(T, dinv, w);   // K'^-1 w
#pragma unroll
      for (int r = 0; r < B; ++r) xb[r] -= w[r];
    }
    if constexpr (FUSE) {
      cur.fpb[L.co] = cur.pbo + omega * xb[NF];
    } else {
      R* xo = xout + (int64_t)(2 * i + 1) * B * M + m;
#pragma unroll
      for (int r = 0; r < B; ++r) xo[(int64_t)r * M] = omega * xb[r];
    }
    if (i + 1 < N) {
      R dvi[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) dvi[q] = xb[q];
      u_delta(i + 1, cur, dvi, t);
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) xn[q] = xb[q];
  }
}

// record pitch in shared memory (values): 16-byte aligned, and 16-byte
// loads of 8 consecutive lanes land in distinct bank quads
template <class R>
__host__ __device__ constexpr int rec_pitch(int rs) {
  return sizeof(R) == 4 ? (rs % 8 == 4 ? rs : rs + 4) : rs + 2;
}
template <class R>
__host__ __device__ constexpr int back_depth() { return sizeof(R) == 4 ? 4 : 2; }

// Back substitution of a shape-2 colour from the record hand-off: step s
// handles pair i = N - 1 - s; its record (L, 1/d, z of pair i; M_i, yu_i for
// the next step) arrives by 16-byte cp.async, DEPTH - 1 steps ahead.  M and yu
// of pair i + 1 are carried in registers from the previous step, so nothing
// is gathered or rebuilt from the state.  Same arithmetic, in the same order,
// as k_scgs_back.
template <int DIM, bool PER, class R>
__global__ void __launch_bounds__(32) k_scgs_back_deep(KktCtx<DIM, PER, R> cx, int o0, int o1, int o2, int mod,
                                                       int m0, int m1, int m2, R omega,
                                                       const R* __restrict__ scratch, R* __restrict__ xout) {
  using LN = Line<DIM>;
  constexpr int NF = LN::NF, B = LN::B, NL = LN::NL, RS = LN::RS, RP = rec_pitch<R>(RS);
  constexpr int DEPTH = back_depth<R>();
  constexpr int VW = 16 / (int)sizeof(R);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* ring = reinterpret_cast<R*>(smem_raw);   // [DEPTH][32][RP]
  const int N = cx.N;
  const int64_t M = (int64_t)m0 * m1 * m2;
  const int lane = threadIdx.x;
  const int64_t m = (int64_t)blockIdx.x * 32 + lane;
  if (m >= M) return;   // no block-wide synchronisation below
  const LineCell<DIM, PER, R> lc(cx.ix, cx.h, m, o0, o1, o2, mod, m1, m2);
  const auto& cg = lc.cg;
  const R idt = cx.idt;
  auto stage = [&](int st) -> R* { return ring + ((st % DEPTH) * 32 + lane) * RP; };
  auto issue = [&](int st) {
    const int i = N - 1 - st;
    if (i >= 0) {
      const R* src = scratch + ((int64_t)i * (RS / VW) * M + m) * VW;
      R* dst = stage(st);
#pragma unroll
      for (int k = 0; k < RS / VW; ++k) cp_async16(dst + k * VW, src + (int64_t)k * M * VW);
    }
    cp_async_commit();   // one group per step (empty past the end)
  };
  auto u_delta = [&](int ip, const R (&yu)[LN::NY], const R (&dvi)[NF], const R (&t)[NF]) {
    R a[NF];
    R ga = R(0);
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      R s = yu[q] + dvi[q] * idt - t[q];
      a[q] = cg.wall[q] ? R(0) : s;
      ga += cg.gcol[q] * a[q];
    }
    const R dp = (ga - yu[NF]) * lc.isig;
    R* xo = xout + (int64_t)(2 * ip) * B * M + m;
#pragma unroll
    for (int q = 0; q < NF; ++q) xo[(int64_t)q * M] = cg.wall[q] ? R(0) : omega * (cg.gcol[q] * dp - a[q]);
    xo[(int64_t)NF * M] = omega * dp;
  };
#pragma unroll
  for (int st = 0; st < DEPTH - 1; ++st) issue(st);
  R xn[NF], Mn[NF * NF], yun[LN::NY];   // dv, M and yu of pair i + 1
#pragma unroll
  for (int q = 0; q < NF; ++q) xn[q] = R(0);
  for (int st = 0; st <= N; ++st) {
    issue(st + DEPTH - 1);
    cp_async_wait<DEPTH - 1>();   // step st's record has landed
    const int i = N - 1 - st;
    const R* cur = stage(st);
    R t[NF];   // M_{i+1} dv_{i+1}
    if (i + 1 < N) {
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < NF; ++k) s += Mn[q * NF + k] * xn[k];
        t[q] = s;
      }
    }
    if (i < 0) {
      R zero[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) zero[q] = R(0);
      u_delta(0, yun, zero, t);   // dv_0 = 0 (pinned / frozen halo)
      break;
    }
    R ldz[LN::NLDZ];
    lds_vec<R, LN::NLDZ>(cur + LN::R_L, ldz);
    R xb[B];
#pragma unroll
    for (int r = 0; r < B; ++r) xb[r] = ldz[NL + B + r];
    if (i + 1 < N) {
      R T[B][B], dinv[B];
#pragma unroll
      for (int r = 1; r < B; ++r)
#pragma unroll
        for (int c = 0; c < r; ++c) T[r][c] = ldz[r * (r - 1) / 2 + c];
#pragma unroll
      for (int r = 0; r < B; ++r) dinv[r] = ldz[NL + r];
      R wf[NF], w[B];
#pragma unroll
      for (int q = 0; q < NF; ++q) wf[q] = t[q];
      lc.projP(wf);
#pragma unroll
      for (int q = 0; q < NF; ++q) w[q] = -wf[q] * idt;
      w[NF] = R(0);
      ldlt_solve<R, B>(T, dinv, w);   // K'^-1 w
#pragma unroll
      for (int r = 0; r < B; ++r) xb[r] -= w[r];
    }
    R* xo = xout + (int64_t)(2 * i + 1) * B * M + m;
#pragma unroll
    for (int r = 0; r < B; ++r) xo[(int64_t)r * M] = omega * xb[r];
    if (i + 1 < N) {
      R dvi[NF];
#pragma unroll
      for (int q = 0; q < NF; ++q) dvi[q] = xb[q];
      u_delta(i + 1, yun, dvi, t);
    }
#pragma unroll
    for (int q = 0; q < NF; ++q) xn[q] = xb[q];
    // pair i's M and yu, for step st + 1 (before the next issue reuses the stage)
    lds_vec<R, NF * NF>(cur + LN::R_M, Mn);
    lds_vec<R, LN::NY>(cur + LN::R_Y, yun);
  }
  cp_async_wait<0>();
}

// x += omega * dx on the colour's unknowns (disjoint across cells)
// x += omega * dx on the colour's unknowns (disjoint across cells); the
// cell's face / cell offsets are computed once, FPT frames (blockIdx.z +
// u * gridDim.z) per thread (FPT = 1 measured fastest: more frames per
// thread strides the same offsets 8 MB apart and lost bandwidth).
template <int DIM, bool PER, class R, int FPT>
__global__ void __launch_bounds__(256) k_scgs_apply(Ix<DIM, PER> ix, StP<R> s, int N, int o0, int o1, int o2, int mod,
                                                    int m0, int m1, int m2, const R* __restrict__ xout) {
  constexpr int NF = 2 * DIM, B = NF + 1;
  const int64_t M = (int64_t)m0 * m1 * m2;
  const int64_t nf[3] = {ix.faces(0), ix.faces(1), DIM == 3 ? ix.faces(2) : 0};
  const int64_t ncl = ix.cells();
  const int fstride = gridDim.z;
  SMK_FRAME_LOOP(m, M) {
    int c[3];
    color_cell<DIM>(m, o0, o1, o2, mod, m1, m2, c);
    int64_t fo[NF];
    bool w[NF];
#pragma unroll
    for (int k = 0; k < DIM; ++k)
#pragma unroll
      for (int sd = 0; sd < 2; ++sd) {
        const int qq = 2 * k + sd;
        w[qq] = !PER && (sd == 0 ? c[k] == 0 : c[k] == ix.n(k) - 1);
        int f[3] = {c[0], c[1], c[2]};
        f[k] += sd;
        if (PER && f[k] >= ix.n(k)) f[k] -= ix.n(k);
        fo[qq] = ix.face_off(k, f[0], f[1], f[2]);
      }
    const int64_t co = ix.cell_off(c[0], c[1], c[2]);
#pragma unroll
    for (int u = 0; u < FPT; ++u) {
      const int i = blockIdx.z + u * fstride;
      if (i >= N) break;
      const R* xu = xout + (int64_t)(2 * i) * B * M + m;
      const R* xv = xout + (int64_t)(2 * i + 1) * B * M + m;
      // every load first, then the stores: the state pointers may alias as
      // far as the compiler knows, so interleaved += would serialise 14
      // memory round trips per thread
      R du[B], dv[B], ou[NF], ov[NF];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        du[q] = xu[(int64_t)q * M];
        dv[q] = xv[(int64_t)q * M];
      }
#pragma unroll
      for (int k = 0; k < DIM; ++k)
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
          const int qq = 2 * k + sd;
          if (w[qq]) continue;
          const int64_t o = (int64_t)i * nf[k] + fo[qq];
          ou[qq] = s.U[k][o];
          ov[qq] = s.V[k][o];
        }
      const int64_t oc = (int64_t)i * ncl + co;
      const R op = s.P[oc], opb = s.PB[oc];
#pragma unroll
      for (int k = 0; k < DIM; ++k)
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
          const int qq = 2 * k + sd;
          if (w[qq]) continue;
          const int64_t o = (int64_t)i * nf[k] + fo[qq];
          s.U[k][o] = ou[qq] + du[qq];
          s.V[k][o] = ov[qq] + dv[qq];
        }
      s.P[oc] = op + du[NF];
      s.PB[oc] = opb + dv[NF];
    }
  }
}

// ---------------------------------------------------------------------------
// host: hierarchy
// ---------------------------------------------------------------------------
template <class R>
struct Level {
  Geo g;
  StP<R> st{};      // state (levels >= 1 owned; level 0 bound per call)
  StP<R> st0{};     // restricted copy (coarse levels)
  ResP<R> rhs{};    // FAS rhs (levels >= 1)
  ResP<R> f{};      // residual buffer
  R* v0[3] = {nullptr, nullptr, nullptr};
  R* vs[3] = {nullptr, nullptr, nullptr};
  int64_t nc = 0, nf[3] = {0, 0, 0};
};

struct NsoBase {
  virtual ~NsoBase() {}
  virtual int set_guide(const void* const v0[], const void* const vstar[], cudaStream_t st) = 0;
  virtual int vcycle(const smk_state* s, cudaStream_t st) = 0;
  virtual int norms(const smk_state* s, double* ri, double* r2, cudaStream_t st) = 0;
  virtual int gauge(const smk_state* s, cudaStream_t st) = 0;
  virtual int levels() const = 0;
  virtual int set_K(double K) = 0;
  virtual int ncolors() const = 0;
  virtual int level_residual(int l, const smk_state* s, const void* const vprev[], const void* const unext[],
                             const void* const vs[], const smk_residual* rhs, const smk_residual* out,
                             cudaStream_t st) = 0;
  virtual int level_color_pass(int l, int colour, const smk_state* s, const void* const vprev[],
                               const void* const unext[], const void* const vs[], const smk_residual* rhs,
                               cudaStream_t st) = 0;
  virtual int profile(int enable) = 0;
  virtual int profile_read(int kind, int level, double* ms, long long* launches, long long* cells) = 0;
  virtual int64_t bytes() const = 0;
  virtual int64_t payload() const = 0;
};

template <int DIM, bool PER, class R>
struct Nso : NsoBase {
  smk_nso_params prm;
  std::vector<Level<R>> lv;
  Scratch mem;
  int64_t nbytes = 0;
  R* scratch = nullptr;   // smoother fill-in W/z and u-rows (Line<DIM>::SE per pair)
  R* xout = nullptr;      // smoother deltas
  int* flag = nullptr;
  double* parts = nullptr;
  void* scal = nullptr;
  bool ok = true;
  const void* top_v0[3] = {nullptr, nullptr, nullptr};
  const void* top_vs[3] = {nullptr, nullptr, nullptr};
  bool guide_set = false;
  // optional CUDA-event profile of the kernels of each colour pass / residual,
  // per kind and level
  bool prof = false;
  static constexpr int NKIND = 4;  // 0 forward, 1 apply, 2 residual, 3 backward
  struct Ev {
    cudaEvent_t a, b;
    int level;
    int64_t cells;
  };
  std::vector<Ev> ev[NKIND];
  size_t ev_used[NKIND] = {0, 0, 0, 0};

  void prof_begin(int kind, int level, int64_t M, cudaStream_t st) {
    if (!prof) return;
    if (ev_used[kind] == ev[kind].size()) {
      Ev e{};
      cudaEventCreate(&e.a);
      cudaEventCreate(&e.b);
      ev[kind].push_back(e);
    }
    Ev& e = ev[kind][ev_used[kind]];
    e.level = level;
    e.cells = M * prm.n_frames;
    cudaEventRecord(e.a, st);
  }
  void prof_end(int kind, cudaStream_t st) {
    if (!prof) return;
    cudaEventRecord(ev[kind][ev_used[kind]].b, st);
    ++ev_used[kind];
  }

  // field payload values owned by the hierarchy (memtrack.py:1-9 counts
  // field containers, not solver scratch): every allocation except the
  // smoother's hand-off and delta buffers
  int64_t npayload = 0;
  R* alloc(int64_t n, bool payload = true) {
    void* p = mem.get((size_t)n * sizeof(R));
    if (!p) ok = false;
    else cudaMemset(p, 0, (size_t)n * sizeof(R));
    nbytes += n * (int64_t)sizeof(R);
    if (payload) npayload += n;
    return (R*)p;
  }

  // forward-kernel shape thresholds (colour cells): >= fwd_big -> TM 64 (fp32:
  // P 2, 168 registers, 2 CTAs / SM; fp64: P 1), >= fwd_mid -> TM 32 / P 2,
  // else TM 32 / P 4.  SMK_FWD_THRESH="big,mid" overrides them (tuning runs
  // only).  The 64^3 red-black colours (131,072 cells: cfg5 level 1, cfg4
  // level 0) take the TM 64 / P 2 shape with the factored hand-off (cfg5
  // level-1 forward 11.2 -> 9.1 ms per V-cycle vs TM 32 / P 2; TM 64 / P 1
  // there: 14.4 ms; the compact hand-off: forward 8.9 but backward 4.7 -> 5.3).
  int64_t fwd_big = 148 * 64 * 10, fwd_mid = 148 * 32 * 2;
  // shape-0 colours with >= cmp_min cells hand off the compact format
  // (SMK_CMP_MIN overrides)
  int64_t cmp_min = 148 * 64 * 16;
  bool fwd_p1 = false;   // SMK_FWD_P1=1: fp32 TM 64 colours on one producer group
  // backward: colours with >= back_flat cells use the unpipelined variant
  // (occupancy), smaller ones the load-pipelined one.  SMK_BACK_FLAT overrides.
  int64_t back_flat = 148 * 128 * 4;
  // colours below 148*64 cells: cp.async-ring backward (SMK_BACK_DEEP=0 off)
  bool back_deep = getenv("SMK_BACK_DEEP") == nullptr || atoi(getenv("SMK_BACK_DEEP")) != 0;

  Nso(const Geo& g, const smk_nso_params& p) : prm(p) {
    if (const char* e = getenv("SMK_BACK_FLAT")) cmp_min = back_flat = atoll(e);   // tuning / tests: compact from back_flat up
    if (const char* e = getenv("SMK_CMP_MIN")) cmp_min = atoll(e);
    if (const char* e = getenv("SMK_FWD_P1")) fwd_p1 = atoi(e) != 0;

    if (const char* e = getenv("SMK_FWD_THRESH")) {
      long long a = 0, b = 0;
      if (sscanf(e, "%lld,%lld", &a, &b) == 2) {
        fwd_big = a;
        fwd_mid = b;
      }
    }
    int want = p.n_levels < 1 ? 1 : p.n_levels;
    Geo cur = g;
    for (int l = 0; l < want; ++l) {
      Level<R> L;
      L.g = cur;
      L.nc = cells_of(cur);
      for (int k = 0; k < DIM; ++k) L.nf[k] = faces_of(cur, k);
      lv.push_back(L);
      if (!can_coarsen(cur) || !colourable(coarsen(cur))) break;
      cur = coarsen(cur);
    }
    const int N = p.n_frames;
    int64_t maxM = 0;
    for (size_t l = 0; l < lv.size(); ++l) {
      Level<R>& L = lv[l];
      auto face_alloc = [&](R* (&dst)[3], int frames) {
        for (int k = 0; k < 3; ++k) dst[k] = k < DIM ? alloc((int64_t)frames * L.nf[k]) : nullptr;
      };
      if (l > 0) {
        face_alloc(L.st.V, N); L.st.PB = alloc((int64_t)N * L.nc);
        face_alloc(L.st.U, N); L.st.P = alloc((int64_t)N * L.nc);
        face_alloc(L.st0.V, N); L.st0.PB = alloc((int64_t)N * L.nc);
        face_alloc(L.st0.U, N); L.st0.P = alloc((int64_t)N * L.nc);
        face_alloc(L.rhs.R1, N); L.rhs.R2 = alloc((int64_t)N * L.nc);
        face_alloc(L.rhs.R3, N); L.rhs.R4 = alloc((int64_t)N * L.nc);
        face_alloc(L.v0, 1);
        face_alloc(L.vs, N);
      }
      face_alloc(L.f.R1, N); L.f.R2 = alloc((int64_t)N * L.nc);
      face_alloc(L.f.R3, N); L.f.R4 = alloc((int64_t)N * L.nc);
      int o[3], mm[3];
      int64_t M = 0;
      for (int col = 0; col < n_colors(); ++col) {
        const int64_t Mc = color_geometry(L.g, col, o, mm);
        M = Mc > M ? Mc : M;
      }
      maxM = M > maxM ? M : maxM;
    }
    constexpr int B = Slots<DIM>::B;
    // [i][e][m] formats: SE values per pair; record format (shape-2 colours,
    // fewer than fwd_mid cells): RS
    const int64_t rec_m = back_deep ? (maxM < fwd_mid ? maxM : fwd_mid) : 0;
    const int64_t per_pair = std::max(Line<DIM>::pair_stride(maxM), (int64_t)Line<DIM>::RS * rec_m);
    scratch = alloc((int64_t)N * per_pair, false);
    xout = alloc((int64_t)2 * N * B * maxM, false);
    // SMK_POISON=1 (tests): the smoother's hand-off and delta buffers start
    // as NaN, so a kernel reading an entry no kernel of the pass wrote shows
    // up as a NaN in the result (initcheck stand-in; compute-sanitizer is not
    // available on the GPU pool)
    if (ok && getenv("SMK_POISON") && atoi(getenv("SMK_POISON"))) {
      cudaMemset(scratch, 0xFF, (size_t)N * per_pair * sizeof(R));
      cudaMemset(xout, 0xFF, (size_t)2 * N * B * maxM * sizeof(R));
    }
    vswap.resize(lv.size());
    for (size_t l = 0; l < lv.size(); ++l) {
      for (int k = 0; k < 3; ++k)
        vswap[l][k] = (k < DIM && fusable((int)l)) ? alloc((int64_t)N * lv[l].nf[k]) : nullptr;
    }
    flag = (int*)mem.get(64);
    parts = (double*)mem.get(sizeof(double) * 70000);
    scal = mem.get(64);
    if (!flag || !parts || !scal) ok = false;
    else cudaMemset(flag, 0, 64);
  }

  int levels() const override { return (int)lv.size(); }
  int set_K(double K) override {
    if (!(K >= 0)) { set_error("K must be >= 0"); return SMK_ERR_ARG; }
    if (K != prm.K) {
      prm.K = K;
      if (vc_exec) cudaGraphExecDestroy(vc_exec);   // the kernels take K/r by value
      vc_exec = nullptr;
    }
    return SMK_OK;
  }
  int profile(int enable) override {
    prof = enable != 0;
    for (int k = 0; k < NKIND; ++k) ev_used[k] = 0;
    return SMK_OK;
  }
  int profile_read(int kind, int level, double* ms, long long* launches, long long* cells) override {
    if (kind < 0 || kind >= NKIND) { set_error("bad profile kind"); return SMK_ERR_ARG; }
    double tot = 0.0;
    long long n = 0, c = 0;
    for (size_t i = 0; i < ev_used[kind]; ++i) {
      const Ev& e = ev[kind][i];
      if (level >= 0 && e.level != level) continue;
      cudaEventSynchronize(e.b);
      float t = 0.f;
      cudaEventElapsedTime(&t, e.a, e.b);
      tot += t;
      ++n;
      c += e.cells;
    }
    if (ms) *ms = tot;
    if (launches) *launches = n;
    if (cells) *cells = c;
    return cuda_check("nso_profile_read");
  }
  ~Nso() override {
    if (vc_exec) cudaGraphExecDestroy(vc_exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (int k = 0; k < NKIND; ++k)
      for (auto& e : ev[k]) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
      }
  }
  int64_t bytes() const override { return nbytes; }
  int64_t payload() const override { return npayload; }

  // slab halos for the next residual / colour pass (set by the level API)
  const void* halo_vprev[3] = {nullptr, nullptr, nullptr};
  const void* halo_unext[3] = {nullptr, nullptr, nullptr};
  const void* halo_vs[3] = {nullptr, nullptr, nullptr};
  bool use_halo = false;

  KktCtx<DIM, PER, R> ctx(int l, const StP<R>& s) const {
    const Level<R>& L = lv[l];
    KktCtx<DIM, PER, R> c{Ix<DIM, PER>(L.g)};
    c.t0 = prm.t0;
    c.Ng = prm.n_total > 0 ? prm.n_total : prm.n_frames;
    for (int k = 0; k < 3; ++k) c.un.c[k] = use_halo ? (const R*)halo_unext[k] : nullptr;
    c.c0 = (R)(0.5 / L.g.h);
    c.h = (R)L.g.h;
    c.dt = (R)prm.dt;
    c.ih = (R)(1.0 / L.g.h);
    c.idt = (R)(1.0 / prm.dt);
    c.kr = (R)(prm.K / prm.r);
    c.N = prm.n_frames;
    for (int k = 0; k < 3; ++k) c.nf[k] = L.nf[k];
    c.nc = L.nc;
    for (int k = 0; k < 3; ++k) {
      c.V.c[k] = s.V[k];
      c.U.c[k] = s.U[k];
      c.v0.c[k] = use_halo ? (const R*)halo_vprev[k] : (l == 0 ? (const R*)top_v0[k] : L.v0[k]);
      c.vs.c[k] = use_halo ? (const R*)halo_vs[k] : (l == 0 ? (const R*)top_vs[k] : L.vs[k]);
    }
    c.P = s.P;
    c.PB = s.PB;
    return c;
  }

  static StP<R> from_api(const smk_state* s) {
    StP<R> o;
    for (int k = 0; k < 3; ++k) {
      o.V[k] = (R*)s->V[k];
      o.U[k] = (R*)s->U[k];
    }
    o.PB = (R*)s->PB;
    o.P = (R*)s->P;
    return o;
  }

  void residual(int l, const StP<R>& s, const ResP<R>* rhs, const ResP<R>& out, cudaStream_t st) {
    auto c = ctx(l, s);
    ResP<R> r = rhs ? *rhs : ResP<R>{};
    prof_begin(2, l, lv[l].nc, st);
    const dim3 grid = kkt_grid(lv[l].nc, prm.n_frames);
    with_nx(l, [&](auto nxc) {
      constexpr int NXv = decltype(nxc)::value;
      const int fpt = kkt_fpt(lv[l].nc, prm.n_frames);
      if (fpt > 1) {
        if (rhs) k_kkt<DIM, PER, R, true, NXv, false, true><<<grid, 256, 0, st>>>(c, r, out, nullptr, fpt);
        else k_kkt<DIM, PER, R, false, NXv, false, true><<<grid, 256, 0, st>>>(c, r, out, nullptr, fpt);
      } else {
        if (rhs) k_kkt<DIM, PER, R, true, NXv><<<grid, 256, 0, st>>>(c, r, out);
        else k_kkt<DIM, PER, R, false, NXv><<<grid, 256, 0, st>>>(c, r, out);
      }
    });
    count_launch();
    prof_end(2, st);
  }

  int n_colors() const {
    if (prm.red_black) return 2;
    int ncol = 1;
    for (int a = 0; a < DIM; ++a) ncol *= prm.color_mod;
    return ncol;
  }
  // colouring validity: same-colour cells must
  // not share a face -- red-black needs an even last-axis extent (and even
  // periodic extents: the wrap neighbour has the other parity); mod-m needs
  // periodic extents divisible by m
  bool colourable(const Geo& g) const {
    for (int a = 0; a < DIM; ++a) {
      if (prm.red_black && a == DIM - 1 && g.n[a] % 2) return false;
      if (PER && g.n[a] % (prm.red_black ? 2 : prm.color_mod)) return false;
    }
    return true;
  }
  // kernel colour geometry (color_cell): offsets o, extents mm, the kernels'
  // mod argument (-1 = red-black); returns the colour's cell count
  int64_t color_geometry(const Geo& g, int col, int (&o)[3], int (&mm)[3]) const {
    o[0] = o[1] = o[2] = 0;
    mm[0] = mm[1] = mm[2] = 1;
    if (prm.red_black) {
      o[0] = col;
      for (int a = 0; a < DIM; ++a) mm[a] = a == DIM - 1 ? g.n[a] / 2 : g.n[a];
    } else {
      const int mod = prm.color_mod;
      int cc = col;
      for (int a = 0; a < DIM; ++a) {
        o[a] = cc % mod;
        cc /= mod;
        mm[a] = (g.n[a] - o[a] + mod - 1) / mod;
        if (mm[a] < 0) mm[a] = 0;
      }
    }
    return (int64_t)mm[0] * mm[1] * mm[2];
  }
  // 3D red-black: -T selects the banded row order of color_cell (T rows
  // along axis 0 per band, T | n0); SMK_ROW_TILE overrides T (1 = plain)
  int row_tile = getenv("SMK_ROW_TILE") ? atoi(getenv("SMK_ROW_TILE")) : 8;
  int kernel_mod(int l) const {
    if (!prm.red_black) return prm.color_mod;
    if (DIM == 3 && row_tile > 1 && lv[l].g.n[0] % row_tile == 0) return -row_tile;
    return -1;
  }

  // red-black passes whose backward is k_scgs_back run fused (no delta
  // buffer, no apply kernel, V ping-pongs through vswap[l]); the record
  // backward of the small colours keeps deltas + apply.  SMK_NO_FUSE=1 off.
  bool fuse_env = getenv("SMK_NO_FUSE") == nullptr || atoi(getenv("SMK_NO_FUSE")) == 0;
  // the compact fused backward stages its hand-off with bulk async copies
  // (k_scgs_back<..., TMA>); SMK_BACK_TMA=0 off
  bool back_tma = getenv("SMK_BACK_TMA") == nullptr || atoi(getenv("SMK_BACK_TMA")) != 0;
  bool fusable(int l) const {
    if (!prm.red_black || !fuse_env) return false;
    int o[3], mm[3];
    const int64_t M = color_geometry(lv[l].g, 0, o, mm);
    return !(M < fwd_mid && back_deep);
  }
  std::vector<std::array<R*, 3>> vswap;   // per level: the other V buffer of a fused pass pair

  void sweep(int l, const StP<R>& s, const ResP<R>* rhs, cudaStream_t st) {
    if (fusable(l) && n_colors() == 2) {
      StP<R> alt = s;
      for (int k = 0; k < 3; ++k) alt.V[k] = vswap[l][k];
      color_pass(l, 0, s, rhs, st, &alt);   // V: s -> alt
      color_pass(l, 1, alt, rhs, st, &s);   // V: alt -> s
      return;
    }
    for (int col = 0; col < n_colors(); ++col) color_pass(l, col, s, rhs, st);
  }

  // compile-time cube extent of level l for the big-colour kernels (0 = runtime)
  int cube_nx(int l) const {
    if (DIM != 3 || PER) return 0;
    const Geo& g = lv[l].g;
    if (g.n[0] != g.n[1] || g.n[1] != g.n[2]) return 0;
    return (g.n[0] == 64 || g.n[0] == 128) ? g.n[0] : 0;
  }
  template <class F>
  void with_nx(int l, F&& f) {
    if constexpr (DIM == 3 && !PER) {
      const int nx = cube_nx(l);
      if (nx == 128) return f(std::integral_constant<int, 128>{});
      if (nx == 64) return f(std::integral_constant<int, 64>{});
    }
    f(std::integral_constant<int, 0>{});
  }

  template <int TM, int P, bool HR, int NX, int FMT>
  void launch_fwd_t(const KktCtx<DIM, PER, R>& c, const ResP<R>& r, const int o[3], int mod, const int mm[3], int64_t M,
                    cudaStream_t st) {
    const size_t shm = (size_t)ring_stages(P) * fwd_ring_entry<DIM>(P) * TM * sizeof(R);
    auto kern = k_scgs_fwd<DIM, PER, R, TM, P, HR, NX, FMT>;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
      attr = true;
    }
    kern<<<(unsigned)((M + TM - 1) / TM), (P + 1) * TM, shm, st>>>(c, r, o[0], o[1], o[2], mod, mm[0], mm[1], mm[2],
                                                                   scratch, flag);
    count_launch();
  }
  template <int TM, int P, int NX, int FMT>
  void launch_fwd(const KktCtx<DIM, PER, R>& c, const ResP<R>& r, bool hr, const int o[3], int mod, const int mm[3],
                  int64_t M, cudaStream_t st) {
    if (hr) launch_fwd_t<TM, P, true, NX, FMT>(c, r, o, mod, mm, M, st);
    else launch_fwd_t<TM, P, false, NX, FMT>(c, r, o, mod, mm, M, st);
  }

  void color_pass(int l, int col, const StP<R>& s, const ResP<R>* rhs, cudaStream_t st,
                  const StP<R>* fuse_out = nullptr) {
    const Level<R>& L = lv[l];
    const int mod = kernel_mod(l);
    auto c = ctx(l, s);
    ResP<R> r = rhs ? *rhs : ResP<R>{};
    Ix<DIM, PER> ix(L.g);
    int o[3], mm[3];
    const int64_t M = color_geometry(L.g, col, o, mm);
    if (M == 0) return;
    // forward: TM colour cells per CTA (producer + consumer warp per 32);
    // small colours use TM = 32 to spread over all SMs
    prof_begin(0, l, M, st);
    // colour cells per SM decide the shape: many -> one producer group
    // (throughput), few -> more producer groups per cell (latency)
    int shape = M >= fwd_big ? 0 : (M >= fwd_mid ? 1 : 2);
    // big colours (unpipelined backward) hand off the compact D~ / rhs
    // format, small latency-bound ones the factored format
    const bool cmp = M >= back_flat && M >= cmp_min && shape == 0;
    if (shape == 2) {
      if (back_deep) launch_fwd<32, 4, 0, 2>(c, r, rhs != nullptr, o, mod, mm, M, st);
      else launch_fwd<32, 4, 0, 0>(c, r, rhs != nullptr, o, mod, mm, M, st);
    } else {
      with_nx(l, [&](auto nxc) {
        constexpr int NXv = decltype(nxc)::value;
        if (shape == 0) {
          // fp32 compact colours: two producer groups, 2 CTAs / SM at 168
          // registers (cfg5 level-0 forward 60.9 -> 58.2 ms per V-cycle;
          // P = 3 and producer-side prep measured slower: 72.0 / 67.7 ms);
          // SMK_FWD_P1=1 keeps the one-group shape
          if constexpr (sizeof(R) == 4) {
            if (cmp && !fwd_p1) return launch_fwd<64, 2, NXv, 1>(c, r, rhs != nullptr, o, mod, mm, M, st);
            if (!cmp && !fwd_p1) return launch_fwd<64, 2, NXv, 0>(c, r, rhs != nullptr, o, mod, mm, M, st);
          }
          if (cmp) launch_fwd<64, 1, NXv, 1>(c, r, rhs != nullptr, o, mod, mm, M, st);
          else launch_fwd<64, 1, NXv, 0>(c, r, rhs != nullptr, o, mod, mm, M, st);
        } else {
          launch_fwd<32, 2, NXv, 0>(c, r, rhs != nullptr, o, mod, mm, M, st);
        }
      });
    }
    prof_end(0, st);
    prof_begin(3, l, M, st);
    StP<R> so{};
    if (fuse_out) {
      so = s;
      for (int k = 0; k < 3; ++k) so.V[k] = fuse_out->V[k];
    }
    {
      const int tpb = M >= 148 * 128 ? 128 : 32;
      const unsigned gb = (unsigned)((M + tpb - 1) / tpb);
      auto back = [&](auto pipe, auto nxc, auto cmpc) {
        constexpr bool PIPEv = decltype(pipe)::value, CMPv = decltype(cmpc)::value;
        constexpr int NXv = decltype(nxc)::value;
        if constexpr (CMPv && !PIPEv && SMK_HANDOFF_BLOCKED) {
          if (fuse_out && back_tma && tpb == 128 && M % 128 == 0) {
            auto kern = k_scgs_back<DIM, PER, R, false, NXv, true, true, true>;
            const size_t shm = back_tma_smem<DIM, R>();
            static bool attr = false;
            if (!attr) {
              cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
              attr = true;
            }
            kern<<<gb, tpb, shm, st>>>(c, o[0], o[1], o[2], mod, mm[0], mm[1], mm[2], (R)prm.omega, scratch, xout,
                                       so);
            return;
          }
        }
        if (fuse_out)
          k_scgs_back<DIM, PER, R, PIPEv, NXv, CMPv, true><<<gb, tpb, 0, st>>>(
              c, o[0], o[1], o[2], mod, mm[0], mm[1], mm[2], (R)prm.omega, scratch, xout, so);
        else
          k_scgs_back<DIM, PER, R, PIPEv, NXv, CMPv, false><<<gb, tpb, 0, st>>>(
              c, o[0], o[1], o[2], mod, mm[0], mm[1], mm[2], (R)prm.omega, scratch, xout, so);
      };
      using F = std::false_type;
      using T = std::true_type;
      using Z = std::integral_constant<int, 0>;
      if (cmp) {
        with_nx(l, [&](auto nxc) { back(F{}, nxc, T{}); });
      } else if (shape == 2 && back_deep) {   // record hand-off
        const size_t shm = (size_t)back_depth<R>() * 32 * rec_pitch<R>(Line<DIM>::RS) * sizeof(R);
        static bool attr = false;
        if (!attr) {
          cudaFuncSetAttribute(k_scgs_back_deep<DIM, PER, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
          attr = true;
        }
        k_scgs_back_deep<DIM, PER, R><<<(unsigned)((M + 31) / 32), 32, shm, st>>>(c, o[0], o[1], o[2], mod, mm[0], mm[1],
                                                                                  mm[2], (R)prm.omega, scratch, xout);
      } else if (M >= back_flat) {
        back(F{}, Z{}, F{});
      } else {
        back(T{}, Z{}, F{});
      }
      count_launch();
    }
    prof_end(3, st);
    if (fuse_out) return;
    prof_begin(1, l, M, st);
    k_scgs_apply<DIM, PER, R, 1><<<frame_grid(M, prm.n_frames, 256), 256, 0, st>>>(
        ix, s, prm.n_frames, o[0], o[1], o[2], mod, mm[0], mm[1], mm[2], xout);
    count_launch();
    prof_end(1, st);

  }

  void restrict_state(int l, const StP<R>& fine, const StP<R>& coarse, cudaStream_t st) {
    const int N = prm.n_frames;
    Face3<R> a, b;
    FaceW<R> oa, ob;
    for (int k = 0; k < 3; ++k) {
      a.c[k] = fine.V[k]; b.c[k] = fine.U[k];
      oa.c[k] = coarse.V[k]; ob.c[k] = coarse.U[k];
    }
    launch_restrict_face<DIM, PER, R>(lv[l].g, N, a, oa, st);
    launch_restrict_face<DIM, PER, R>(lv[l].g, N, b, ob, st);
    launch_restrict_cell<DIM, PER, R>(lv[l].g, N, fine.PB, coarse.PB, st);
    launch_restrict_cell<DIM, PER, R>(lv[l].g, N, fine.P, coarse.P, st);
  }

  void restrict_res(int l, const ResP<R>& fine, const ResP<R>& coarse, cudaStream_t st) {
    const int N = prm.n_frames;
    Face3<R> a, b;
    FaceW<R> oa, ob;
    for (int k = 0; k < 3; ++k) {
      a.c[k] = fine.R1[k]; b.c[k] = fine.R3[k];
      oa.c[k] = coarse.R1[k]; ob.c[k] = coarse.R3[k];
    }
    launch_restrict_face<DIM, PER, R>(lv[l].g, N, a, oa, st);
    launch_restrict_face<DIM, PER, R>(lv[l].g, N, b, ob, st);
    launch_restrict_cell<DIM, PER, R>(lv[l].g, N, fine.R2, coarse.R2, st);
    launch_restrict_cell<DIM, PER, R>(lv[l].g, N, fine.R4, coarse.R4, st);
  }

  void copy_state(int l, const StP<R>& src, const StP<R>& dst, cudaStream_t st) {
    const int N = prm.n_frames;
    const Level<R>& L = lv[l];
    for (int k = 0; k < DIM; ++k) {
      cudaMemcpyAsync(dst.V[k], src.V[k], (size_t)N * L.nf[k] * sizeof(R), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(dst.U[k], src.U[k], (size_t)N * L.nf[k] * sizeof(R), cudaMemcpyDeviceToDevice, st);
    }
    cudaMemcpyAsync(dst.PB, src.PB, (size_t)N * L.nc * sizeof(R), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(dst.P, src.P, (size_t)N * L.nc * sizeof(R), cudaMemcpyDeviceToDevice, st);
  }

  // dst = a*src + b*dst over the whole state
  void axpby_state(int l, const StP<R>& src, const StP<R>& dst, double a, double b, cudaStream_t st) {
    const int N = prm.n_frames;
    const Level<R>& L = lv[l];
    for (int k = 0; k < DIM; ++k) {
      axpby<R>(dst.V[k], src.V[k], a, b, (int64_t)N * L.nf[k], st);
      axpby<R>(dst.U[k], src.U[k], a, b, (int64_t)N * L.nf[k], st);
    }
    axpby<R>(dst.PB, src.PB, a, b, (int64_t)N * L.nc, st);
    axpby<R>(dst.P, src.P, a, b, (int64_t)N * L.nc, st);
  }

  void prolong_add(int lc, const StP<R>& coarse, const StP<R>& fine, cudaStream_t st) {
    const int N = prm.n_frames;
    Face3<R> a, b;
    FaceW<R> oa, ob;
    for (int k = 0; k < 3; ++k) {
      a.c[k] = coarse.V[k]; b.c[k] = coarse.U[k];
      oa.c[k] = fine.V[k]; ob.c[k] = fine.U[k];
    }
    launch_prolong_face<DIM, PER, R>(lv[lc].g, N, a, oa, 1, st);
    launch_prolong_face<DIM, PER, R>(lv[lc].g, N, b, ob, 1, st);
    launch_prolong_cell<DIM, PER, R>(lv[lc].g, N, coarse.PB, fine.PB, 1, st);
    launch_prolong_cell<DIM, PER, R>(lv[lc].g, N, coarse.P, fine.P, 1, st);
  }

  int set_guide(const void* const v0[], const void* const vstar[], cudaStream_t st) override {
    for (int k = 0; k < 3; ++k) {
      top_v0[k] = k < DIM ? v0[k] : nullptr;
      top_vs[k] = k < DIM ? vstar[k] : nullptr;
    }
    for (size_t l = 1; l < lv.size(); ++l) {
      Face3<R> a, b;
      FaceW<R> oa, ob;
      for (int k = 0; k < 3; ++k) {
        a.c[k] = l == 1 ? (const R*)top_v0[k] : lv[l - 1].v0[k];
        b.c[k] = l == 1 ? (const R*)top_vs[k] : lv[l - 1].vs[k];
        oa.c[k] = lv[l].v0[k];
        ob.c[k] = lv[l].vs[k];
      }
      launch_restrict_face<DIM, PER, R>(lv[l - 1].g, 1, a, oa, st);
      launch_restrict_face<DIM, PER, R>(lv[l - 1].g, prm.n_frames, b, ob, st);
    }
    guide_set = true;
    return cuda_check("nso_set_guide");
  }

  void vcycle_level(int l, const StP<R>& s, const ResP<R>* rhs, cudaStream_t st) {
    if (l == (int)lv.size() - 1) {
      for (int it = 0; it < prm.n_coarse; ++it) sweep(l, s, rhs, st);
      return;
    }
    for (int it = 0; it < prm.nu1; ++it) sweep(l, s, rhs, st);
    Level<R>& C = lv[l + 1];
    restrict_state(l, s, C.st, st);
    copy_state(l + 1, C.st, C.st0, st);
    // f = f(x) - rhs on this level; coarse rhs = f_c(R x) - R f
    residual(l, s, rhs, lv[l].f, st);
    restrict_res(l, lv[l].f, C.f, st);
    residual(l + 1, C.st, &C.f, C.rhs, st);
    vcycle_level(l + 1, C.st, &C.rhs, st);
    // x += P(x_c - R x)
    axpby_state(l + 1, C.st, C.st0, 1.0, -1.0, st);
    prolong_add(l + 1, C.st0, s, st);
    for (int it = 0; it < prm.nu2; ++it) sweep(l, s, rhs, st);
  }

  int check_flag(cudaStream_t st) {
    int h = 0;
    cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    int rc = cuda_check("nso");
    if (rc) return rc;
    if (h) {
      cudaMemsetAsync(flag, 0, sizeof(int), st);
      set_error("SCGS block pivot below threshold (SingularBlock)");
      return SMK_SINGULAR_BLOCK;
    }
    return SMK_OK;
  }

  // One V-cycle is ~1800 launches: it is captured once into a CUDA graph
  // (on a private stream, so the caller may use the legacy stream) and
  // replayed; re-captured when the caller's state / guide buffers change.
  // Profiling runs and SMK_NO_GRAPH=1 launch directly.
  cudaGraphExec_t vc_exec = nullptr;
  cudaStream_t cap_stream = nullptr;
  const void* vc_key[14] = {};
  long long vc_launches = 0;
  bool graph_ok = getenv("SMK_NO_GRAPH") == nullptr;

  int vcycle(const smk_state* s, cudaStream_t st) override {
    if (!guide_set) { set_error("nso: set_guide not called"); return SMK_ERR_ARG; }
    StP<R> top = from_api(s);
    if (!graph_ok || prof) {
      vcycle_level(0, top, nullptr, st);
      return cuda_check("nso_vcycle");
    }
    const void* key[14] = {s->V[0], s->V[1], s->V[2], s->U[0], s->U[1], s->U[2], s->P, s->PB,
                           top_v0[0], top_v0[1], top_v0[2], top_vs[0], top_vs[1], top_vs[2]};
    if (!vc_exec || memcmp(key, vc_key, sizeof(key)) != 0) {
      if (vc_exec) cudaGraphExecDestroy(vc_exec);
      vc_exec = nullptr;
      if (!cap_stream && cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        graph_ok = false;
        return vcycle(s, st);
      }
      const long long n0 = launch_count();
      cudaGraph_t g = nullptr;
      bool ok_cap = cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
      if (ok_cap) vcycle_level(0, top, nullptr, cap_stream);
      ok_cap = ok_cap && cudaStreamEndCapture(cap_stream, &g) == cudaSuccess && g;
      ok_cap = ok_cap && cudaGraphInstantiate(&vc_exec, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
      if (!ok_cap) {
        cudaGetLastError();
        vc_exec = nullptr;
        graph_ok = false;
        return vcycle(s, st);
      }
      vc_launches = launch_count() - n0;   // counted once while capturing
      memcpy(vc_key, key, sizeof(key));
    } else {
      count_launch((int)vc_launches);
    }
    cudaGraphLaunch(vc_exec, st);
    return cuda_check("nso_vcycle");
  }

  int gauge(const smk_state* s, cudaStream_t st) override {
    StP<R> top = from_api(s);
    frame_sub_mean<R>(top.P, lv[0].nc, prm.n_frames, st, parts);
    frame_sub_mean<R>(top.PB, lv[0].nc, prm.n_frames, st, parts);
    return cuda_check("nso_gauge");
  }

  // ||f||_inf and ||f||_2 of the level-0 residual: one fused residual+norm
  // launch (k_kkt<NORM>, nothing stored), a fixed-order final reduction and
  // one read-back together with the SingularBlock flag
  double* nparts = nullptr;
  int64_t nparts_n = 0;
  // launch the fused residual + norm of level 0 (halos as set) and its
  // fixed-order reduction into dev_out[0..1] = {max |f|, sum f^2}
  int norm_launch(const StP<R>& top, double* dev_out, cudaStream_t st) {
    auto c = ctx(0, top);
    const dim3 grid = kkt_grid(lv[0].nc, prm.n_frames);
    const int64_t nblk = (int64_t)grid.x * grid.y * grid.z;
    if (nparts_n < nblk + 1) {
      nparts = (double*)mem.get(sizeof(double) * 2 * (nblk + 1));
      if (!nparts) { nparts_n = 0; set_error("nso: out of device memory (norm partials)"); return SMK_ERR_CUDA; }
      nparts_n = nblk + 1;
    }
    prof_begin(2, 0, lv[0].nc, st);
    with_nx(0, [&](auto nxc) {
      constexpr int NXv = decltype(nxc)::value;
      const int fpt = kkt_fpt(lv[0].nc, prm.n_frames);
      if (fpt > 1) k_kkt<DIM, PER, R, false, NXv, true, true><<<grid, 256, 0, st>>>(c, ResP<R>{}, ResP<R>{}, nparts, fpt);
      else k_kkt<DIM, PER, R, false, NXv, true><<<grid, 256, 0, st>>>(c, ResP<R>{}, ResP<R>{}, nparts);
    });
    count_launch();
    prof_end(2, st);
    k_norm_final<<<1, 1024, 0, st>>>(nparts, nblk, dev_out ? dev_out : nparts + 2 * nblk);
    count_launch();
    return SMK_OK;
  }
  // read the SingularBlock flag after a synchronisation point
  int take_flag(int fl, cudaStream_t st) {
    if (fl) {
      cudaMemsetAsync(flag, 0, sizeof(int), st);
      set_error("SCGS block pivot below threshold (SingularBlock)");
      return SMK_SINGULAR_BLOCK;
    }
    return SMK_OK;
  }
  int norms(const smk_state* s, double* ri, double* r2, cudaStream_t st) override {
    if (!guide_set) { set_error("nso: set_guide not called"); return SMK_ERR_ARG; }
    int rc = norm_launch(from_api(s), nullptr, st);
    if (rc) return rc;
    const dim3 grid = kkt_grid(lv[0].nc, prm.n_frames);
    const int64_t nblk = (int64_t)grid.x * grid.y * grid.z;
    double h[2] = {0.0, 0.0};
    int fl = 0;
    cudaMemcpyAsync(h, nparts + 2 * nblk, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&fl, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    rc = cuda_check("nso_norms");
    if (rc) return rc;
    *ri = h[0];
    if (r2) *r2 = std::sqrt(h[1]);
    return take_flag(fl, st);
  }

  // ---- slab (per-level) API: caller owns the level's state and halos ----
  void set_halo(const void* const vprev[], const void* const unext[], const void* const vs[]) {
    for (int k = 0; k < 3; ++k) {
      halo_vprev[k] = k < DIM ? vprev[k] : nullptr;
      halo_unext[k] = (k < DIM && unext) ? unext[k] : nullptr;
      halo_vs[k] = k < DIM ? vs[k] : nullptr;
    }
    use_halo = true;
  }
  static ResP<R> res_from_api(const smk_residual* r) {
    ResP<R> o{};
    if (!r) return o;
    for (int k = 0; k < 3; ++k) { o.R1[k] = (R*)r->R1[k]; o.R3[k] = (R*)r->R3[k]; }
    o.R2 = (R*)r->R2; o.R4 = (R*)r->R4;
    return o;
  }
  int ncolors() const override { return n_colors(); }
  int level_residual(int l, const smk_state* s, const void* const vprev[], const void* const unext[],
                     const void* const vs[], const smk_residual* rhs, const smk_residual* out,
                     cudaStream_t st) override {
    if (l < 0 || l >= (int)lv.size()) { set_error("bad level"); return SMK_ERR_ARG; }
    set_halo(vprev, unext, vs);
    ResP<R> r = res_from_api(rhs);
    residual(l, from_api(s), rhs ? &r : nullptr, res_from_api(out), st);
    use_halo = false;
    return cuda_check("nso_level_residual");
  }
  int level_color_pass(int l, int colour, const smk_state* s, const void* const vprev[], const void* const unext[],
                       const void* const vs[], const smk_residual* rhs, cudaStream_t st) override {
    if (l < 0 || l >= (int)lv.size()) { set_error("bad level"); return SMK_ERR_ARG; }
    if (colour < 0 || colour >= n_colors()) { set_error("bad colour"); return SMK_ERR_ARG; }
    set_halo(vprev, unext, vs);
    ResP<R> r = res_from_api(rhs);
    color_pass(l, colour, from_api(s), rhs ? &r : nullptr, st);
    use_halo = false;
    return cuda_check("nso_level_color_pass");
  }

  // standalone entry points (level-0 only)
  int residual_api(const smk_state* s, const smk_residual* rhs, const smk_residual* out, cudaStream_t st) {
    StP<R> top = from_api(s);
    ResP<R> o, r;
    for (int k = 0; k < 3; ++k) {
      o.R1[k] = (R*)out->R1[k]; o.R3[k] = (R*)out->R3[k];
      if (rhs) { r.R1[k] = (R*)rhs->R1[k]; r.R3[k] = (R*)rhs->R3[k]; }
    }
    o.R2 = (R*)out->R2; o.R4 = (R*)out->R4;
    if (rhs) { r.R2 = (R*)rhs->R2; r.R4 = (R*)rhs->R4; }
    residual(0, top, rhs ? &r : nullptr, o, st);
    return cuda_check("smk_kkt_residual");
  }
  int sweep_api(const smk_state* s, const smk_residual* rhs, cudaStream_t st) {
    StP<R> top = from_api(s);
    ResP<R> r;
    if (rhs) {
      for (int k = 0; k < 3; ++k) { r.R1[k] = (R*)rhs->R1[k]; r.R3[k] = (R*)rhs->R3[k]; }
      r.R2 = (R*)rhs->R2; r.R4 = (R*)rhs->R4;
    }
    sweep(0, top, rhs ? &r : nullptr, st);
    return check_flag(st);
  }
};


// ---------------------------------------------------------------------------
// Time slabs: this process's contiguous slabs of the spacetime
// volume, each an Nso over its pairs (t0, n_total set), driven through the
// whole FAS V-cycle in C++ with the slab halos refreshed before every
// residual and every colour pass -- local neighbours by device copies,
// remote ones (the ranks holding the slabs on either side) by NCCL
// send / recv on the same stream.  The V-cycle (kernels, copies and NCCL
// P2P) is captured once into a CUDA graph and replayed; no host code runs
// per colour pass.  NCCL is loaded with dlopen on first use (world > 1).
// ---------------------------------------------------------------------------
struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
  bool load() {
    if (so) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names)
      if ((so = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!so) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(so, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(so, "ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))dlsym(so, "ncclCommDestroy");
    GroupStart = (decltype(GroupStart))dlsym(so, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(so, "ncclGroupEnd");
    Send = (decltype(Send))dlsym(so, "ncclSend");
    Recv = (decltype(Recv))dlsym(so, "ncclRecv");
    AllReduce = (decltype(AllReduce))dlsym(so, "ncclAllReduce");
    ErrStr = (decltype(ErrStr))dlsym(so, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && CommDestroy && GroupStart && GroupEnd && Send && Recv && AllReduce;
  }
};
static NcclApi g_nccl;

struct SlabsBase {
  virtual ~SlabsBase() {}
  virtual int set_guide(const void* const v0[], const void* const vstar[], cudaStream_t st) = 0;
  virtual int vcycle(const smk_state* s, cudaStream_t st) = 0;
  virtual int gauge(const smk_state* s, cudaStream_t st) = 0;
  virtual int norms(const smk_state* s, double* ri, double* r2, cudaStream_t st) = 0;
  virtual int levels() const = 0;
  virtual int64_t bytes() const = 0;
  virtual int frames(int k, int* t0, int* n) const = 0;
  virtual int profile(int enable) = 0;
  virtual int profile_read(int kind, int level, double* ms, long long* launches, long long* cells) = 0;
};

template <int DIM, bool PER, class R>
struct Slabs : SlabsBase {
  using NS = Nso<DIM, PER, R>;
  int first, nloc, nslab, rank, world, ntot;
  std::vector<std::unique_ptr<NS>> E;
  std::vector<int> t0s, ns;
  int L = 0;
  Scratch mem;
  int64_t nbytes = 0;
  ncclComm_t comm = nullptr;
  bool nccl_local = false;   // SMK_SLABS_NCCL_LOCAL=1: local-neighbour halos by NCCL self send / recv
  // per level: pinned v0 (slab 0), per local slab: halo frames and guide
  struct H {
    R* vprev[3] = {nullptr, nullptr, nullptr};
    R* unext[3] = {nullptr, nullptr, nullptr};
    R* vs[3] = {nullptr, nullptr, nullptr};
  };
  std::vector<std::array<R*, 3>> v0l;
  std::vector<std::vector<H>> hl;   // [level][local slab]
  double* dnorm = nullptr;           // per local slab {max, sum}, then the combined pair
  bool ok = true, guide_set = false;

  R* alloc(int64_t n) {
    void* p = mem.get((size_t)n * sizeof(R));
    if (!p) { ok = false; return nullptr; }
    cudaMemset(p, 0, (size_t)n * sizeof(R));
    nbytes += n * (int64_t)sizeof(R);
    return (R*)p;
  }

  Slabs(const Geo& g, const smk_nso_params& p, int first_, int nloc_, int nslab_, int rank_, int world_,
        const void* nccl_id)
      : first(first_), nloc(nloc_), nslab(nslab_), rank(rank_), world(world_), ntot(p.n_frames) {
    // split_frames (slabs.py): contiguous, the first (ntot % nslab) slabs one longer
    const int base = ntot / nslab, extra = ntot % nslab;
    int t = 0;
    for (int q = 0; q < nslab; ++q) {
      const int n = base + (q < extra ? 1 : 0);
      if (q >= first && q < first + nloc) {
        t0s.push_back(t);
        ns.push_back(n);
      }
      t += n;
    }
    for (int k = 0; k < nloc; ++k) {
      smk_nso_params q = p;
      q.t0 = t0s[k];
      q.n_frames = ns[k];
      q.n_total = ntot;
      E.emplace_back(new NS(g, q));
      if (!E.back()->ok) ok = false;
      nbytes += E.back()->bytes();
    }
    if (!ok) return;
    L = E[0]->levels();
    v0l.resize(L);
    hl.assign(L, std::vector<H>(nloc));
    for (int l = 0; l < L; ++l) {
      const auto& Lv = E[0]->lv[l];
      for (int c = 0; c < 3; ++c) v0l[l][c] = c < DIM ? alloc(Lv.nf[c]) : nullptr;
      for (int k = 0; k < nloc; ++k)
        for (int c = 0; c < DIM; ++c) {
          hl[l][k].vprev[c] = alloc(Lv.nf[c]);
          hl[l][k].unext[c] = alloc(Lv.nf[c]);
          hl[l][k].vs[c] = alloc((int64_t)(ns[k] + 1) * Lv.nf[c]);
        }
    }
    dnorm = (double*)mem.get(sizeof(double) * 2 * (nloc + 1));
    if (!dnorm) ok = false;
    // a communicator whenever a unique id is given: world > 1 needs one; a
    // one-rank world takes it too (norm allreduce over NCCL -- the path a
    // single-GPU box can exercise, tests/test_gpu_slabs.py)
    if (world > 1 || nccl_id) {
      if (!nccl_id || !g_nccl.load()) {
        set_error("slabs: world > 1 needs NCCL (libnccl.so.2) and a unique id");
        ok = false;
        return;
      }
      ncclUniqueId id;
      memcpy(&id, nccl_id, sizeof(id));
      if (g_nccl.CommInitRank(&comm, world, id, rank) != ncclSuccess) {
        set_error("slabs: ncclCommInitRank failed");
        comm = nullptr;
        ok = false;
      }
      const char* e = getenv("SMK_SLABS_NCCL_LOCAL");   // tests: local halos over NCCL too
      nccl_local = e && atoi(e) != 0;
    }
  }
  ~Slabs() override {
    if (exec) cudaGraphExecDestroy(exec);
    if (cap) cudaStreamDestroy(cap);
    if (comm) g_nccl.CommDestroy(comm);
  }
  int levels() const override { return L; }
  int64_t bytes() const override { return nbytes; }
  int frames(int k, int* t0, int* n) const override {
    if (k < 0 || k >= nloc) { set_error("bad local slab"); return SMK_ERR_ARG; }
    *t0 = t0s[k];
    *n = ns[k];
    return SMK_OK;
  }
  bool global_first(int k) const { return first + k == 0; }
  bool global_last(int k) const { return first + k == nslab - 1; }

  // vstar: the full guide v*_0 .. v*_{ntot-1} (ntot frames); each slab keeps
  // v*_{t0} .. v*_{t0+n} per level (the frame past the global end is zero)
  int set_guide(const void* const v0[], const void* const vstar[], cudaStream_t st) override {
    const auto& L0 = E[0]->lv[0];
    for (int c = 0; c < DIM; ++c)
      cudaMemcpyAsync(v0l[0][c], v0[c], (size_t)L0.nf[c] * sizeof(R), cudaMemcpyDeviceToDevice, st);
    for (int k = 0; k < nloc; ++k)
      for (int c = 0; c < DIM; ++c) {
        const int nfr = std::min(ns[k] + 1, ntot - t0s[k]);
        cudaMemcpyAsync(hl[0][k].vs[c], (const R*)vstar[c] + (int64_t)t0s[k] * L0.nf[c],
                        (size_t)nfr * L0.nf[c] * sizeof(R), cudaMemcpyDeviceToDevice, st);
        if (nfr < ns[k] + 1)
          cudaMemsetAsync(hl[0][k].vs[c] + (int64_t)nfr * L0.nf[c], 0,
                          (size_t)(ns[k] + 1 - nfr) * L0.nf[c] * sizeof(R), st);
      }
    for (int l = 1; l < L; ++l) {
      const Geo& gf = E[0]->lv[l - 1].g;
      Face3<R> a;
      FaceW<R> oa;
      for (int c = 0; c < 3; ++c) { a.c[c] = v0l[l - 1][c]; oa.c[c] = v0l[l][c]; }
      launch_restrict_face<DIM, PER, R>(gf, 1, a, oa, st);
      for (int k = 0; k < nloc; ++k) {
        for (int c = 0; c < 3; ++c) { a.c[c] = hl[l - 1][k].vs[c]; oa.c[c] = hl[l][k].vs[c]; }
        launch_restrict_face<DIM, PER, R>(gf, ns[k] + 1, a, oa, st);
      }
    }
    // the slab Nso's never use their own guide buffers (halo mode), but their
    // entry points check that a guide was bound
    for (auto& e : E) e->guide_set = true;
    guide_set = true;
    return cuda_check("slabs_set_guide");
  }

  // halos of level l from the local slabs' current states (V read from sv[k],
  // U from su[k]); remote neighbours over NCCL
  void exchange(int l, const std::vector<StP<R>>& sv, cudaStream_t st) {
    const auto& Lv = E[0]->lv[l];
    if (comm && nccl_local) {
      // local neighbours through NCCL self send / recv (matched in issue
      // order inside one group): the halo path of a remote neighbour --
      // ncclSend / ncclRecv captured into the V-cycle graph -- on one GPU
      const ncclDataType_t ty = sizeof(R) == 8 ? ncclFloat64 : ncclFloat32;
      g_nccl.GroupStart();
      for (int k = 0; k < nloc; ++k)
        for (int c = 0; c < DIM; ++c) {
          if (k > 0) {
            g_nccl.Send(sv[k - 1].V[c] + (int64_t)(ns[k - 1] - 1) * Lv.nf[c], (size_t)Lv.nf[c], ty, rank, comm, st);
            g_nccl.Recv(hl[l][k].vprev[c], (size_t)Lv.nf[c], ty, rank, comm, st);
          }
          if (k < nloc - 1) {
            g_nccl.Send(sv[k + 1].U[c], (size_t)Lv.nf[c], ty, rank, comm, st);
            g_nccl.Recv(hl[l][k].unext[c], (size_t)Lv.nf[c], ty, rank, comm, st);
          }
        }
      g_nccl.GroupEnd();
    } else
    for (int k = 0; k < nloc; ++k) {
      if (k > 0)
        for (int c = 0; c < DIM; ++c)
          cudaMemcpyAsync(hl[l][k].vprev[c], sv[k - 1].V[c] + (int64_t)(ns[k - 1] - 1) * Lv.nf[c],
                          (size_t)Lv.nf[c] * sizeof(R), cudaMemcpyDeviceToDevice, st);
      if (k < nloc - 1)
        for (int c = 0; c < DIM; ++c)
          cudaMemcpyAsync(hl[l][k].unext[c], sv[k + 1].U[c], (size_t)Lv.nf[c] * sizeof(R), cudaMemcpyDeviceToDevice,
                          st);
    }
    if (world > 1 && comm) {
      const ncclDataType_t ty = sizeof(R) == 8 ? ncclFloat64 : ncclFloat32;
      g_nccl.GroupStart();
      if (!global_first(0))   // left neighbour: send my first U frame, receive its last V frame
        for (int c = 0; c < DIM; ++c) {
          g_nccl.Send(sv[0].U[c], (size_t)Lv.nf[c], ty, rank - 1, comm, st);
          g_nccl.Recv(hl[l][0].vprev[c], (size_t)Lv.nf[c], ty, rank - 1, comm, st);
        }
      if (!global_last(nloc - 1))
        for (int c = 0; c < DIM; ++c) {
          g_nccl.Send(sv[nloc - 1].V[c] + (int64_t)(ns[nloc - 1] - 1) * Lv.nf[c], (size_t)Lv.nf[c], ty, rank + 1,
                      comm, st);
          g_nccl.Recv(hl[l][nloc - 1].unext[c], (size_t)Lv.nf[c], ty, rank + 1, comm, st);
        }
      g_nccl.GroupEnd();
    }
  }
  void bind(int l, int k) {
    const void* vp[3] = {nullptr, nullptr, nullptr};
    const void* un[3] = {nullptr, nullptr, nullptr};
    const void* vs[3] = {nullptr, nullptr, nullptr};
    for (int c = 0; c < DIM; ++c) {
      vp[c] = global_first(k) ? (const void*)v0l[l][c] : (const void*)hl[l][k].vprev[c];
      un[c] = hl[l][k].unext[c];
      vs[c] = hl[l][k].vs[c];
    }
    E[k]->set_halo(vp, global_last(k) ? nullptr : un, vs);
  }
  void unbind(int k) { E[k]->use_halo = false; }

  void sweep(int l, const std::vector<StP<R>>& S, const std::vector<const ResP<R>*>& rhs, cudaStream_t st) {
    NS& e0 = *E[0];
    if (e0.fusable(l) && e0.n_colors() == 2) {
      std::vector<StP<R>> alt = S;
      for (int k = 0; k < nloc; ++k)
        for (int c = 0; c < 3; ++c) alt[k].V[c] = E[k]->vswap[l][c];
      exchange(l, S, st);
      for (int k = 0; k < nloc; ++k) {
        bind(l, k);
        E[k]->color_pass(l, 0, S[k], rhs[k], st, &alt[k]);
        unbind(k);
      }
      exchange(l, alt, st);
      for (int k = 0; k < nloc; ++k) {
        bind(l, k);
        E[k]->color_pass(l, 1, alt[k], rhs[k], st, &S[k]);
        unbind(k);
      }
      return;
    }
    for (int col = 0; col < e0.n_colors(); ++col) {
      exchange(l, S, st);
      for (int k = 0; k < nloc; ++k) {
        bind(l, k);
        E[k]->color_pass(l, col, S[k], rhs[k], st);
        unbind(k);
      }
    }
  }
  void residual(int l, const std::vector<StP<R>>& S, const std::vector<const ResP<R>*>& rhs,
                const std::vector<ResP<R>>& out, cudaStream_t st) {
    exchange(l, S, st);
    for (int k = 0; k < nloc; ++k) {
      bind(l, k);
      E[k]->residual(l, S[k], rhs[k], out[k], st);
      unbind(k);
    }
  }
  void vcycle_level(int l, const std::vector<StP<R>>& S, const std::vector<const ResP<R>*>& rhs, cudaStream_t st) {
    const int n1 = E[0]->prm.nu1, n2 = E[0]->prm.nu2, nc = E[0]->prm.n_coarse;
    if (l == L - 1) {
      for (int it = 0; it < nc; ++it) sweep(l, S, rhs, st);
      return;
    }
    for (int it = 0; it < n1; ++it) sweep(l, S, rhs, st);
    std::vector<StP<R>> C(nloc);
    std::vector<ResP<R>> F(nloc), CF(nloc), CR(nloc);
    std::vector<const ResP<R>*> cfp(nloc), crp(nloc);
    for (int k = 0; k < nloc; ++k) {
      auto& ck = E[k]->lv[l + 1];
      C[k] = ck.st;
      F[k] = E[k]->lv[l].f;
      CF[k] = ck.f;
      CR[k] = ck.rhs;
      cfp[k] = &E[k]->lv[l + 1].f;
      crp[k] = &E[k]->lv[l + 1].rhs;
      E[k]->restrict_state(l, S[k], ck.st, st);
      E[k]->copy_state(l + 1, ck.st, ck.st0, st);
    }
    residual(l, S, rhs, F, st);
    for (int k = 0; k < nloc; ++k) E[k]->restrict_res(l, F[k], CF[k], st);
    residual(l + 1, C, cfp, CR, st);
    vcycle_level(l + 1, C, crp, st);
    for (int k = 0; k < nloc; ++k) {
      auto& ck = E[k]->lv[l + 1];
      E[k]->axpby_state(l + 1, ck.st, ck.st0, 1.0, -1.0, st);
      E[k]->prolong_add(l + 1, ck.st0, S[k], st);
    }
    for (int it = 0; it < n2; ++it) sweep(l, S, rhs, st);
  }

  std::vector<StP<R>> tops(const smk_state* s) const {
    std::vector<StP<R>> S(nloc);
    for (int k = 0; k < nloc; ++k) S[k] = NS::from_api(&s[k]);
    return S;
  }
  // graph of the whole slab V-cycle (re-captured when a state pointer changes)
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  std::vector<const void*> key;
  long long exec_launches = 0;
  bool graph_ok = getenv("SMK_NO_GRAPH") == nullptr;

  // per-kernel CUDA-event profile summed over the local slabs (launched
  // directly, not from the graph, while enabled -- like Nso)
  bool prof = false;
  int profile(int enable) override {
    prof = enable != 0;
    for (auto& e : E) e->profile(enable);
    return SMK_OK;
  }
  int profile_read(int kind, int level, double* ms, long long* launches, long long* cells) override {
    double t = 0.0;
    long long n = 0, c = 0;
    for (auto& e : E) {
      double a = 0.0;
      long long b = 0, d = 0;
      int rc = e->profile_read(kind, level, &a, &b, &d);
      if (rc) return rc;
      t += a;
      n += b;
      c += d;
    }
    if (ms) *ms = t;
    if (launches) *launches = n;
    if (cells) *cells = c;
    return SMK_OK;
  }

  int vcycle(const smk_state* s, cudaStream_t st) override {
    if (!guide_set) { set_error("slabs: set_guide not called"); return SMK_ERR_ARG; }
    const auto S = tops(s);
    const std::vector<const ResP<R>*> none(nloc, nullptr);
    if (!graph_ok || prof) {
      vcycle_level(0, S, none, st);
      return cuda_check("slabs_vcycle");
    }
    std::vector<const void*> kk;
    for (int k = 0; k < nloc; ++k) {
      for (int c = 0; c < 3; ++c) { kk.push_back(s[k].V[c]); kk.push_back(s[k].U[c]); }
      kk.push_back(s[k].P);
      kk.push_back(s[k].PB);
    }
    if (!exec || kk != key) {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
      if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        graph_ok = false;
        return vcycle(s, st);
      }
      // the capture stream must see the caller's prior work
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, st);
      cudaStreamWaitEvent(cap, ev, 0);
      cudaEventDestroy(ev);
      const long long n0 = launch_count();
      cudaGraph_t g = nullptr;
      bool okc = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) == cudaSuccess;
      if (okc) vcycle_level(0, S, none, cap);
      okc = okc && cudaStreamEndCapture(cap, &g) == cudaSuccess && g;
      okc = okc && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
      if (!okc) {
        cudaGetLastError();
        exec = nullptr;
        graph_ok = false;
        return vcycle(s, st);
      }
      exec_launches = launch_count() - n0;
      key = kk;
    } else {
      count_launch((int)exec_launches);
    }
    cudaGraphLaunch(exec, st);
    return cuda_check("slabs_vcycle");
  }
  int gauge(const smk_state* s, cudaStream_t st) override {
    for (int k = 0; k < nloc; ++k) {
      int rc = E[k]->gauge(&s[k], st);
      if (rc) return rc;
    }
    return SMK_OK;
  }
  int norms(const smk_state* s, double* ri, double* r2, cudaStream_t st) override {
    if (!guide_set) { set_error("slabs: set_guide not called"); return SMK_ERR_ARG; }
    const auto S = tops(s);
    exchange(0, S, st);
    for (int k = 0; k < nloc; ++k) {
      bind(0, k);
      int rc = E[k]->norm_launch(S[k], dnorm + 2 * k, st);
      unbind(k);
      if (rc) return rc;
    }
    std::vector<double> h(2 * nloc);
    std::vector<int> fl(nloc, 0);
    cudaMemcpyAsync(h.data(), dnorm, sizeof(double) * 2 * nloc, cudaMemcpyDeviceToHost, st);
    for (int k = 0; k < nloc; ++k) cudaMemcpyAsync(&fl[k], E[k]->flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    int rc = cuda_check("slabs_norms");
    if (rc) return rc;
    double mx = 0.0, sq = 0.0;
    for (int k = 0; k < nloc; ++k) {
      mx = std::isnan(h[2 * k + 1]) ? h[2 * k + 1] : std::max(mx, h[2 * k]);
      sq += h[2 * k + 1];
    }
    if (comm) {
      double both[2] = {mx, sq};
      double* d = dnorm + 2 * nloc;
      cudaMemcpyAsync(d, both, sizeof(both), cudaMemcpyHostToDevice, st);
      g_nccl.GroupStart();
      g_nccl.AllReduce(d, d, 1, ncclFloat64, ncclMax, comm, st);
      g_nccl.AllReduce(d + 1, d + 1, 1, ncclFloat64, ncclSum, comm, st);
      g_nccl.GroupEnd();
      cudaMemcpyAsync(both, d, sizeof(both), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      rc = cuda_check("slabs_norms_allreduce");
      if (rc) return rc;
      mx = both[0];
      sq = both[1];
    }
    *ri = mx;
    if (r2) *r2 = std::sqrt(sq);
    for (int k = 0; k < nloc; ++k) {
      rc = E[k]->take_flag(fl[k], st);
      if (rc) return rc;
    }
    return SMK_OK;
  }
};

}  // namespace smk

using namespace smk;

struct smk_nso {
  NsoBase* impl;
  smk_grid grid;
  smk_nso_params prm;
};

static int check_params(const smk_nso_params* p) {
  if (!p) { set_error("null params"); return SMK_ERR_ARG; }
  if (p->t0 < 0 || p->n_total < 0 || (p->n_total > 0 && p->t0 + p->n_frames > p->n_total)) {
    set_error("bad slab range (t0, n_total)");
    return SMK_ERR_ARG;
  }
  if (p->n_frames < 1) { set_error("n_frames must be >= 1"); return SMK_ERR_ARG; }
  if (!(p->dt > 0) || !(p->r > 0) || !(p->K >= 0)) { set_error("dt, r must be positive, K >= 0"); return SMK_ERR_ARG; }
  if (!p->red_black && p->color_mod < 2) { set_error("color_mod must be >= 2"); return SMK_ERR_ARG; }
  if (p->nu1 < 0 || p->nu2 < 0 || p->n_coarse < 0) { set_error("negative sweep counts"); return SMK_ERR_ARG; }
  return SMK_OK;
}

// the colouring must keep same-colour cells face-disjoint on the top level
// (coarser levels stop before a level that breaks it, Nso::colourable)
static int check_colouring(const smk_grid* g, const smk_nso_params* p) {
  const int mod = p->red_black ? 2 : p->color_mod;
  for (int a = 0; a < g->dim; ++a) {
    if (p->red_black && a == g->dim - 1 && g->res[a] % 2) {
      set_error("red-black colouring needs an even extent along the last axis");
      return SMK_ERR_ARG;
    }
    if (g->boundary == SMK_PERIODIC && g->res[a] % mod) {
      set_error("periodic extents must be divisible by the colouring modulus (%d)", mod);
      return SMK_ERR_ARG;
    }
  }
  return SMK_OK;
}

template <class F>
static NsoBase* make_nso(const smk_grid* g, const smk_nso_params* p) {
  NsoBase* out = nullptr;
  dispatch(g, [&](auto tag) {
    using T = decltype(tag);
    auto* n = new Nso<T::DIM, T::PER, typename T::R>(to_geo(g), *p);
    if (!n->ok) {
      // the operator scratch pool may hold the memory: release it, retry once
      delete n;
      pool_trim();
      n = new Nso<T::DIM, T::PER, typename T::R>(to_geo(g), *p);
    }
    if (!n->ok) {
      delete n;
      set_error("nso: device allocation failed");
      return SMK_ERR_CUDA;
    }
    out = n;
    return SMK_OK;
  });
  return out;
}

struct smk_slabs {
  SlabsBase* impl;
};

extern "C" {

int smk_nccl_unique_id(void* out, int nbytes) {
  if (!out || nbytes < (int)sizeof(ncclUniqueId)) { set_error("need %d bytes", (int)sizeof(ncclUniqueId)); return SMK_ERR_ARG; }
  if (!g_nccl.load()) { set_error("libnccl.so.2 not found"); return SMK_ERR_CUDA; }
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) { set_error("ncclGetUniqueId failed"); return SMK_ERR_CUDA; }
  memcpy(out, &id, sizeof(id));
  return SMK_OK;
}

smk_slabs* smk_slabs_create(const smk_grid* g, const smk_nso_params* p, int first, int n_local, int n_slabs, int rank,
                            int world, const void* nccl_id) {
  if (check_grid(g) || check_params(p) || check_colouring(g, p)) return nullptr;
  if (p->t0 != 0 || (p->n_total != 0 && p->n_total != p->n_frames)) {
    set_error("slabs: n_frames is the global pair count (t0 = 0, n_total = 0)");
    return nullptr;
  }
  if (n_slabs < 1 || n_slabs > p->n_frames || first < 0 || n_local < 1 || first + n_local > n_slabs || world < 1 ||
      rank < 0 || rank >= world) {
    set_error("slabs: bad slab range / rank");
    return nullptr;
  }
  SlabsBase* impl = nullptr;
  dispatch(g, [&](auto tag) {
    using T = decltype(tag);
    auto* s = new Slabs<T::DIM, T::PER, typename T::R>(to_geo(g), *p, first, n_local, n_slabs, rank, world, nccl_id);
    if (!s->ok) {
      delete s;
      return SMK_ERR_CUDA;
    }
    impl = s;
    return SMK_OK;
  });
  if (!impl) return nullptr;
  return new smk_slabs{impl};
}

void smk_slabs_destroy(smk_slabs* h) {
  if (!h) return;
  cudaDeviceSynchronize();
  delete h->impl;
  delete h;
}

int smk_slabs_levels(const smk_slabs* h) { return h ? h->impl->levels() : 0; }
int64_t smk_slabs_device_bytes(const smk_slabs* h) { return h ? h->impl->bytes() : 0; }
int smk_slabs_frames(const smk_slabs* h, int k, int* t0, int* n) {
  if (!h || !t0 || !n) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->frames(k, t0, n);
}
int smk_slabs_set_guide(smk_slabs* h, const void* const v0[], const void* const vstar[], void* stream) {
  if (!h || !v0 || !vstar) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->set_guide(v0, vstar, (cudaStream_t)stream);
}
int smk_slabs_vcycle(smk_slabs* h, const smk_state* states, void* stream) {
  if (!h || !states) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->vcycle(states, (cudaStream_t)stream);
}
int smk_slabs_gauge_fix(smk_slabs* h, const smk_state* states, void* stream) {
  if (!h || !states) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->gauge(states, (cudaStream_t)stream);
}
int smk_slabs_residual_norms(smk_slabs* h, const smk_state* states, double* ri, double* r2, void* stream) {
  if (!h || !states || !ri) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->norms(states, ri, r2, (cudaStream_t)stream);
}
int smk_slabs_profile(smk_slabs* h, int enable) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  return h->impl->profile(enable);
}
int smk_slabs_profile_read_level(smk_slabs* h, int kind, int level, double* ms, long long* launches,
                                 long long* cells) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  return h->impl->profile_read(kind, level, ms, launches, cells);
}

smk_nso* smk_nso_create(const smk_grid* g, const smk_nso_params* p) {
  if (check_grid(g) || check_params(p) || check_colouring(g, p)) return nullptr;
  NsoBase* impl = make_nso<int>(g, p);
  if (!impl) return nullptr;
  smk_nso* h = new smk_nso;
  h->impl = impl;
  h->grid = *g;
  h->prm = *p;
  return h;
}

void smk_nso_destroy(smk_nso* h) {
  if (!h) return;
  cudaDeviceSynchronize();
  delete h->impl;
  delete h;
}

int smk_nso_levels(const smk_nso* h) { return h ? h->impl->levels() : 0; }
int64_t smk_nso_payload_values(const smk_nso* h) { return h ? h->impl->payload() : 0; }
int smk_nso_n_colors(const smk_nso* h) { return h ? h->impl->ncolors() : 0; }

int smk_nso_level_residual(smk_nso* h, int level, const smk_state* s, const void* const vprev[],
                           const void* const unext[], const void* const vs[], const smk_residual* rhs,
                           const smk_residual* out, void* stream) {
  if (!h || !s || !out || !vprev || !vs) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->level_residual(level, s, vprev, unext, vs, rhs, out, (cudaStream_t)stream);
}

int smk_nso_level_color_pass(smk_nso* h, int level, int colour, const smk_state* s, const void* const vprev[],
                             const void* const unext[], const void* const vs[], const smk_residual* rhs,
                             void* stream) {
  if (!h || !s || !vprev || !vs) { set_error("null argument"); return SMK_ERR_ARG; }
  int rc = h->impl->level_color_pass(level, colour, s, vprev, unext, vs, rhs, (cudaStream_t)stream);
  return rc;
}

int smk_axpby(int dtype, void* y, const void* x, double a, double b, int64_t n, void* stream) {
  if (dtype == SMK_F64) axpby<double>((double*)y, (const double*)x, a, b, n, (cudaStream_t)stream);
  else if (dtype == SMK_F32) axpby<float>((float*)y, (const float*)x, a, b, n, (cudaStream_t)stream);
  else { set_error("bad dtype"); return SMK_ERR_ARG; }
  count_launch();
  return cuda_check("smk_axpby");
}

int smk_nso_profile(smk_nso* h, int enable) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  return h->impl->profile(enable);
}

int smk_nso_profile_read(smk_nso* h, int kind, double* ms, long long* launches, long long* cells) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  return h->impl->profile_read(kind, -1, ms, launches, cells);
}

int smk_nso_profile_read_level(smk_nso* h, int kind, int level, double* ms, long long* launches, long long* cells) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  return h->impl->profile_read(kind, level, ms, launches, cells);
}
int64_t smk_nso_device_bytes(const smk_nso* h) { return h ? h->impl->bytes() : 0; }

int smk_nso_set_guide(smk_nso* h, const void* const v0[], const void* const vstar[], void* stream) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  return h->impl->set_guide(v0, vstar, (cudaStream_t)stream);
}

int smk_nso_set_K(smk_nso* h, double K) {
  if (!h) { set_error("null handle"); return SMK_ERR_ARG; }
  int rc = h->impl->set_K(K);
  if (rc == SMK_OK) h->prm.K = K;
  return rc;
}

int smk_nso_vcycle(smk_nso* h, const smk_state* s, void* stream) {
  if (!h || !s) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->vcycle(s, (cudaStream_t)stream);
}

int smk_nso_residual_norms(smk_nso* h, const smk_state* s, double* ri, double* r2, void* stream) {
  if (!h || !s || !ri) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->norms(s, ri, r2, (cudaStream_t)stream);
}

int smk_nso_gauge_fix(smk_nso* h, const smk_state* s, void* stream) {
  if (!h || !s) { set_error("null argument"); return SMK_ERR_ARG; }
  return h->impl->gauge(s, (cudaStream_t)stream);
}

int smk_nso_solve(smk_nso* h, const smk_state* s, double eps, int relative, int budget, int* cycles, double* hist,
                  void* stream) {
  if (!h || !s) { set_error("null argument"); return SMK_ERR_ARG; }
  if (!(eps > 0)) { set_error("eps must be positive"); return SMK_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  double ri = 0, r2 = 0;
  int rc = h->impl->norms(s, &ri, &r2, st);
  if (rc) return rc;
  if (hist) { hist[0] = ri; hist[1] = r2; }
  double tol = relative ? eps * ri : eps;
  if (cycles) *cycles = 0;
  if (ri <= tol) return SMK_OK;
  for (int c = 1; c <= budget; ++c) {
    rc = h->impl->vcycle(s, st);
    if (rc) return rc;
    rc = h->impl->gauge(s, st);
    if (rc) return rc;
    rc = h->impl->norms(s, &ri, &r2, st);
    if (rc) return rc;
    if (hist) { hist[2 * c] = ri; hist[2 * c + 1] = r2; }
    if (cycles) *cycles = c;
    if (ri <= tol) return SMK_OK;
  }
  set_error("STFAS cycle budget exhausted (residual %.3e > %.3e)", ri, tol);
  return SMK_NONCONVERGENCE;
}

int smk_kkt_residual(const smk_grid* g, const smk_nso_params* p, const smk_state* s, const void* const v0[],
                     const void* const vstar[], const smk_residual* rhs, const smk_residual* out, void* stream) {
  if (check_grid(g) || check_params(p)) return SMK_ERR_ARG;
  smk_nso_params q = *p;
  q.n_levels = 1;
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag);
    Nso<T::DIM, T::PER, typename T::R> n(to_geo(g), q);
    if (!n.ok) { set_error("allocation failed"); return SMK_ERR_CUDA; }
    n.set_guide(v0, vstar, (cudaStream_t)stream);
    int rc = n.residual_api(s, rhs, out, (cudaStream_t)stream);
    cudaStreamSynchronize((cudaStream_t)stream);
    return rc;
  });
}

int smk_scgs_sweep(const smk_grid* g, const smk_nso_params* p, const smk_state* s, const void* const v0[],
                   const void* const vstar[], const smk_residual* rhs, void* stream) {
  if (check_grid(g) || check_params(p) || check_colouring(g, p)) return SMK_ERR_ARG;
  smk_nso_params q = *p;
  q.n_levels = 1;
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag);
    Nso<T::DIM, T::PER, typename T::R> n(to_geo(g), q);
    if (!n.ok) { set_error("allocation failed"); return SMK_ERR_CUDA; }
    n.set_guide(v0, vstar, (cudaStream_t)stream);
    int rc = n.sweep_api(s, rhs, (cudaStream_t)stream);
    cudaStreamSynchronize((cudaStream_t)stream);
    return rc;
  });
}

}  // extern "C"
