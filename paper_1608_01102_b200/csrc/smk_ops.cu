// Field-core, transport, transfer, Poisson and forward-step kernels.
//
// Each kernel reproduces one reference raw kernel (cited per function) with
// the same floating-point evaluation order where that is cheap, so fp64
// results agree with the oracle to a few ulps.  All kernels are HBM-bound
// stencils: one thread per output point, grid-stride, coalesced along the
// contiguous axis, neighbours served by L1/L2.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "smk_dispatch.cuh"
#include "smk_internal.cuh"

namespace smk {

static thread_local char g_err[512] = {0};
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ===========================================================================
// field core
// ===========================================================================

template <int DIM, bool PER, class R>
__global__ void k_div(Ix<DIM, PER> ix, R h, Face3<R> v, R* __restrict__ out, int N) {
  const int64_t nc = ix.cells();
  SMK_GRID_STRIDE(t, (int64_t)N * nc) {
    int fr = (int)(t / nc);
    int c[3];
    ix.cell_idx(t - (int64_t)fr * nc, c);
    R acc = R(0);
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const R* p = v.c[k] + (int64_t)fr * ix.faces(k);
      int hi[3];
      shift(c, k, 1, hi);
      R d = (ix.face(p, k, hi[0], hi[1], hi[2]) - p[ix.face_off(k, c[0], c[1], c[2])]) / h;
      acc = (k == 0) ? d : acc + d;
    }
    out[t] = acc;
  }
}

template <int DIM, bool PER, class R>
__global__ void k_grad(Ix<DIM, PER> ix, R h, const R* __restrict__ p, FaceW<R> out, int N) {
  const int k = blockIdx.y;
  const int64_t nf = ix.faces(k), nc = ix.cells();
  SMK_GRID_STRIDE(t, (int64_t)N * nf) {
    int fr = (int)(t / nf);
    int c[3];
    ix.face_idx(k, t - (int64_t)fr * nf, c);
    const R* pp = p + (int64_t)fr * nc;
    R val = R(0);
    if (!ix.wall(k, c)) {
      int lo[3];
      shift(c, k, -1, lo);
      val = (ix.cell(pp, c[0], c[1], c[2]) - ix.cell(pp, lo[0], lo[1], lo[2])) / h;
    }
    out.c[k][t] = val;
  }
}

template <int DIM, bool PER, class R>
__global__ void k_zero_walls(Ix<DIM, PER> ix, FaceW<R> v, int N) {
  const int k = blockIdx.y;
  const int64_t nf = ix.faces(k);
  SMK_GRID_STRIDE(t, (int64_t)N * nf) {
    int c[3];
    ix.face_idx(k, t % nf, c);
    if (ix.wall(k, c)) v.c[k][t] = R(0);
  }
}

// div(grad p) with the reference's evaluation order (fields.py:223-225)
template <int DIM, bool PER, class R>
__device__ __forceinline__ R lap_at(const Ix<DIM, PER>& ix, R h, const R* pp, const int c[3]) {
  R acc = R(0);
  R pc = pp[ix.cell_off(c[0], c[1], c[2])];
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    int hi[3], lo[3];
    shift((int*)c, k, 1, hi);
    shift((int*)c, k, -1, lo);
    bool whi = !PER && hi[k] == ix.n(k);
    bool wlo = !PER && c[k] == 0;
    R gh = whi ? R(0) : (ix.cell(pp, hi[0], hi[1], hi[2]) - pc) / h;
    R gl = wlo ? R(0) : (pc - ix.cell(pp, lo[0], lo[1], lo[2])) / h;
    R d = (gh - gl) / h;
    acc = (k == 0) ? d : acc + d;
  }
  return acc;
}

template <int DIM, bool PER, class R>
__device__ __forceinline__ R lap_diag_at(const Ix<DIM, PER>& ix, R h, const int c[3]) {
  R h2 = h * h;
  R d = R(-2.0 * DIM) / h2;
  if (!PER) {
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      if (c[k] == 0) d += R(1) / h2;
      if (c[k] == ix.n(k) - 1) d += R(1) / h2;
    }
  }
  return d;
}

template <int DIM, bool PER, class R>
__global__ void k_laplacian(Ix<DIM, PER> ix, R h, const R* __restrict__ p, R* __restrict__ out, int N) {
  const int64_t nc = ix.cells();
  SMK_GRID_STRIDE(t, (int64_t)N * nc) {
    int fr = (int)(t / nc);
    int c[3];
    ix.cell_idx(t - (int64_t)fr * nc, c);
    out[t] = lap_at(ix, h, p + (int64_t)fr * nc, c);
  }
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
template <class R>
__global__ void k_absmax(const R* __restrict__ x, int64_t n, R* out) {
  R m = R(0);
  SMK_GRID_STRIDE(i, n) m = max(m, rabs(x[i]));
  block_max_to(m, out);
}

// deterministic two-pass sum: fixed partition into `parts` block partials
template <class R>
__global__ void k_partial_sum(const R* __restrict__ x, const R* __restrict__ y, int64_t n, double* part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += y ? (double)x[i] * (double)y[i] : (double)x[i];
  s = warp_sum(s);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) part[blockIdx.x] = s;
  }
}

__global__ void k_final_sum(const double* part, int n, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) *out = s;
  }
}

// per-frame sums -> subtract the per-frame mean in place (gauge / rhs mean)
template <class R>
__global__ void k_frame_partial(const R* __restrict__ x, int64_t per, int parts, double* part) {
  // grid (parts, nframes)
  __shared__ double sh[32];
  const int fr = blockIdx.y;
  const R* p = x + (int64_t)fr * per;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)parts * blockDim.x)
    s += (double)p[i];
  s = warp_sum(s);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) part[(int64_t)fr * parts + blockIdx.x] = s;
  }
}

template <class R>
__global__ void k_frame_sub_mean(R* __restrict__ x, int64_t per, int parts, const double* part, int nframes) {
  __shared__ double mean;
  const int fr = blockIdx.y;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < parts; ++i) s += part[(int64_t)fr * parts + i];
    mean = s / (double)per;
  }
  __syncthreads();
  R m = (R)mean;
  R* p = x + (int64_t)fr * per;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x)
    p[i] -= m;
}

// ---------------------------------------------------------------------------
// elementwise helpers
// ---------------------------------------------------------------------------
template <class R>
__global__ void k_axpby(R* __restrict__ y, const R* __restrict__ x, R a, R b, int64_t n) {
  SMK_GRID_STRIDE(i, n) y[i] = b * y[i] + a * x[i];
}
template <class R>
__global__ void k_absdiff_max(const R* __restrict__ a, const R* __restrict__ b, int64_t n, R* out) {
  R m = R(0);
  SMK_GRID_STRIDE(i, n) m = max(m, rabs(a[i] - b[i]));
  block_max_to(m, out);
}

// ===========================================================================
// transfers
// ===========================================================================

// restrict_cell: axis-by-axis pair averages (fields.py:243-253)
template <int DIM, bool PER, class R>
__global__ void k_restrict_cell(Ix<DIM, PER> fx, Ix<DIM, PER> cx, const R* __restrict__ x, R* __restrict__ out,
                                int N) {
  const int64_t ncc = cx.cells(), ncf = fx.cells();
  const int fr = blockIdx.z;
  SMK_FRAME_LOOP(e, ncc) {
    const int64_t t = (int64_t)fr * ncc + e;
    int c[3];
    cx.cell_idx32(e, c);
    const R* p = x + (int64_t)fr * ncf;
    R v[2][2];
    int l0 = 2 * c[2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < (DIM == 3 ? 2 : 1); ++e) {
        int j = 2 * c[1] + b, l = DIM == 3 ? l0 + e : 0;
        v[b][e] = R(0.5) * (p[fx.cell_off(2 * c[0], j, l)] + p[fx.cell_off(2 * c[0] + 1, j, l)]);
      }
    R w0 = R(0.5) * (v[0][0] + v[1][0]);
    R res = w0;
    if (DIM == 3) {
      R w1 = R(0.5) * (v[0][1] + v[1][1]);
      res = R(0.5) * (w0 + w1);
    }
    out[t] = res;
  }
}

// 1-D (3/4, 1/4) prolongation weight pair for fine index I along an axis of
// coarse extent n: returns the two coarse indices (clamped / wrapped)
template <bool PER>
__device__ __forceinline__ void pro_idx(int I, int n, int& i0, int& i1) {
  i0 = I >> 1;
  i1 = (I & 1) ? i0 + 1 : i0 - 1;
  if (PER) i1 = i1 < 0 ? i1 + n : (i1 >= n ? i1 - n : i1);
  else i1 = i1 < 0 ? 0 : (i1 > n - 1 ? n - 1 : i1);
}

// prolong_cell with the reference's axis order (fields.py:256-284).
// Launch: x over the last (contiguous) axis, y over the rows of the leading
// axes, z over frames -- the leading-axis coarse rows are block-uniform, so a
// thread does only its own last-axis weights and 2^d coalesced loads.
// Prolongation launch shape (cells and faces): one warp per fine row of the
// leading axes, 4 rows per 128-thread block (y), frame (z).  The warp issues
// the row's old values (accumulate) and the 2^(d-1) coarse rows it
// interpolates from, combines the coarse rows across the leading axes ONCE
// per coarse element into one shared-memory row c (the same expressions, in
// the same axis order, as per fine element), then each lane builds the fine
// pair (2j, 2j+1) along the contiguous axis from c[j-1..j+1]: a few
// instructions per fine element (the per-element leading-axis work made the
// first version issue-bound at 1.6 TB/s).
constexpr int kProlongWarps = 4;
constexpr int kProlongRows = 2;   // fine rows per warp, loads of both issued up front
// fine pairs per lane with prefetched old values: MAXP = 3 (nl <= 192) or 5
// (nl <= 320, longer rows finish in a tail loop), chosen per launch


// fine pair (2j, 2j+1) of a row from the combined coarse row c (cn values):
// normal: 2j copies c[j], 2j+1 averages c[j], c[j+1]; across: (3/4, 1/4)
// with c[j-1] / c[j+1] (clamped, or wrapped when periodic)
template <bool PER, class R>
__device__ __forceinline__ void pro_pair(const R* c, int j, int cn, bool normal, R& f0, R& f1) {
  const R cj = c[j];
  if (normal) {
    int jn = j + 1;
    if (PER && jn >= cn) jn -= cn;
    if (!PER && jn > cn - 1) jn = cn - 1;   // only reached past the row end
    f0 = cj;
    f1 = R(0.5) * cj + R(0.5) * c[jn];
  } else {
    int jm = j - 1, jp = j + 1;
    if (PER) {
      jm = jm < 0 ? jm + cn : jm;
      jp = jp >= cn ? jp - cn : jp;
    } else {
      jm = jm < 0 ? 0 : jm;
      jp = jp > cn - 1 ? cn - 1 : jp;
    }
    f0 = R(0.75) * cj + R(0.25) * c[jm];
    f1 = R(0.75) * cj + R(0.25) * c[jp];
  }
}

// old values of the fine row (issued before the coarse loads)
template <class R, int MAXP>
__device__ __forceinline__ void pro_old(const R* orow, int nl, int lane, int accumulate, R (&old)[MAXP][2]) {
#pragma unroll
  for (int u = 0; u < MAXP; ++u) {
    const int F = 2 * (lane + 32 * u);
    old[u][0] = (accumulate && F < nl) ? orow[F] : R(0);
    old[u][1] = (accumulate && F + 1 < nl) ? orow[F + 1] : R(0);
  }
}
// fine row phase shared by cells and faces: orow[0..nl) (+)= pairs from c
template <bool PER, class R, int MAXP>
__device__ __forceinline__ void pro_row(const R* c, int cn, bool normal, R* orow, int nl, int lane, int accumulate,
                                        const R (&old)[MAXP][2]) {
  const int np = (nl + 1) >> 1;
  auto put = [&](int j, R o0, R o1) {
    R f0, f1;
    pro_pair<PER, R>(c, j, cn, normal, f0, f1);
    const int F = 2 * j;
    orow[F] = accumulate ? o0 + f0 : f0;
    if (F + 1 < nl) orow[F + 1] = accumulate ? o1 + f1 : f1;
  };
  __syncwarp();
#pragma unroll
  for (int u = 0; u < MAXP; ++u) {
    const int j = lane + 32 * u;
    if (j >= np) break;
    put(j, old[u][0], old[u][1]);
  }
  for (int j = lane + 32 * MAXP; j < np; j += 32) {
    const int F = 2 * j;
    put(j, accumulate ? orow[F] : R(0), (accumulate && F + 1 < nl) ? orow[F + 1] : R(0));
  }
}

template <int DIM, bool PER, class R, int MAXP>
__global__ void __launch_bounds__(32 * kProlongWarps) k_prolong_cell(Ix<DIM, PER> cx, Ix<DIM, PER> fx,
                                                                    const R* __restrict__ x, R* __restrict__ out,
                                                                    int N, int accumulate) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nl = DIM == 3 ? fx.n2 : fx.n1, cnl = DIM == 3 ? cx.n2 : cx.n1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RPW = kProlongRows;
  R* crow = reinterpret_cast<R*>(smem_raw) + warp * RPW * cnl;   // this warp's combined coarse rows
  const int64_t ncc = cx.cells(), ncf = fx.cells();
  const int fr = blockIdx.z;
  const int nrows = DIM == 3 ? fx.n0 * fx.n1 : fx.n0;
  const int rowb = (blockIdx.y * kProlongWarps + warp) * RPW;
  if (rowb >= nrows) return;
  const R* p = x + (int64_t)fr * ncc;
  int F0[RPW], F1[RPW];
  R* orow[RPW];
  R old[RPW][MAXP][2];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int row = rowb + r < nrows ? rowb + r : rowb;   // past the end: a duplicate, never stored
    F0[r] = DIM == 3 ? row / fx.n1 : row;
    F1[r] = DIM == 3 ? row - F0[r] * fx.n1 : 0;
    // in-frame offsets in 32 bits (a frame has < 2^31 elements)
    orow[r] = out + (int64_t)fr * ncf + (DIM == 3 ? (F0[r] * fx.n1 + F1[r]) * fx.n2 : F0[r] * fx.n1);
    pro_old<R, MAXP>(orow[r], nl, lane, accumulate, old[r]);
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    R* cr = crow + r * cnl;
    int a0, a1, b0 = 0, b1 = 0;
    pro_idx<PER>(F0[r], cx.n0, a0, a1);
    if (DIM == 3) pro_idx<PER>(F1[r], cx.n1, b0, b1);
    if (DIM == 3) {
      // axis 0 (a), then axis 1 (b): y_b = 3/4 (a0, b) + 1/4 (a1, b); c = 3/4 y_b0 + 1/4 y_b1
      const R *r00 = p + (a0 * cx.n1 + b0) * cx.n2, *r01 = p + (a0 * cx.n1 + b1) * cx.n2;
      const R *r10 = p + (a1 * cx.n1 + b0) * cx.n2, *r11 = p + (a1 * cx.n1 + b1) * cx.n2;
      for (int l = lane; l < cnl; l += 32) {
        const R y0 = R(0.75) * r00[l] + R(0.25) * r10[l];
        const R y1 = R(0.75) * r01[l] + R(0.25) * r11[l];
        cr[l] = R(0.75) * y0 + R(0.25) * y1;
      }
    } else {
      const R *r0 = p + a0 * cx.n1, *r1 = p + a1 * cx.n1;
      for (int l = lane; l < cnl; l += 32) cr[l] = R(0.75) * r0[l] + R(0.25) * r1[l];
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r)
    if (rowb + r < nrows) pro_row<PER, R, MAXP>(crow + r * cnl, cnl, false, orow[r], nl, lane, accumulate, old[r]);
}

template <int DIM, bool PER>
inline dim3 prolong_cell_grid(const Ix<DIM, PER>& fx, int N, int& tpb) {
  tpb = 32 * kProlongWarps;
  const int rows = DIM == 3 ? fx.n0 * fx.n1 : fx.n0;
  return dim3(1, (rows + kProlongWarps * kProlongRows - 1) / (kProlongWarps * kProlongRows), N);
}
template <int DIM, bool PER, class R>
inline size_t prolong_cell_smem(const Ix<DIM, PER>& cx) {
  return (size_t)kProlongWarps * kProlongRows * (DIM == 3 ? cx.n2 : cx.n1) * sizeof(R);
}

// face restriction: along the normal take the coincident (even) face, across
// it average pairs; axes processed in order.  One warp per
// coarse row of the leading axes (component blockIdx.x, frame blockIdx.z):
// the row's 1-4 fine source rows are fixed, so each lane only walks the
// contiguous axis -- a float2 load per fine row when that axis is an across
// axis (even fine row length), a scalar load of the coincident face when it
// is the normal.  Same expressions, same axis order as per-element code.
constexpr int kRestrictWarps = 4;
template <int DIM, bool PER, class R>
__global__ void __launch_bounds__(32 * kRestrictWarps) k_restrict_face(Ix<DIM, PER> fx, Ix<DIM, PER> cx, Face3<R> in,
                                                                      FaceW<R> out, int N) {
  constexpr int L = DIM - 1;   // contiguous axis
  const int k = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ce1 = cx.fe(k, 1), ce2 = DIM == 3 ? cx.fe(k, 2) : 1;
  const int fe1 = fx.fe(k, 1), fe2 = DIM == 3 ? fx.fe(k, 2) : 1;
  const int crows = DIM == 3 ? cx.fe(k, 0) * ce1 : cx.fe(k, 0);
  const int row = blockIdx.y * kRestrictWarps + warp;
  if (row >= crows) return;
  const int fr = blockIdx.z;
  const int C0 = DIM == 3 ? row / ce1 : row;
  const int C1 = DIM == 3 ? row - C0 * ce1 : 0;
  const int cnl = cx.fe(k, L);
  // fine rows: axis 0 picks 2 C0 (+1 across), axis 1 (3D) 2 C1 (+1 across)
  const int n0 = k == 0 ? 1 : 2, n1 = DIM == 3 ? (k == 1 ? 1 : 2) : 1;
  const R* p = in.c[k] + (int64_t)fr * fx.faces(k);
  const R* fr_[2][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
      fr_[x][y] = p + (DIM == 3 ? ((2 * C0 + (x < n0 ? x : 0)) * fe1 + 2 * C1 + (y < n1 ? y : 0)) * fe2
                                 : (2 * C0 + (x < n0 ? x : 0)) * fe1);
  R* o = out.c[k] + (int64_t)fr * cx.faces(k) + (DIM == 3 ? (C0 * ce1 + C1) * ce2 : C0 * ce1);
  const bool across = k != L;   // contiguous axis averages pairs
  for (int l = lane; l < cnl; l += 32) {
    // v[y][e]: axis 0 applied (fine row pair x), fine element 2l + e
    R v[2][2];
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      if (y >= n1) { v[y][0] = v[y][1] = R(0); continue; }
      R a0, a1, b0 = R(0), b1 = R(0);
      if (across) {
        if constexpr (sizeof(R) == 4) {
          const float2 t = reinterpret_cast<const float2*>(fr_[0][y])[l];
          a0 = t.x; a1 = t.y;
          if (n0 == 2) { const float2 u = reinterpret_cast<const float2*>(fr_[1][y])[l]; b0 = u.x; b1 = u.y; }
        } else {
          const double2 t = reinterpret_cast<const double2*>(fr_[0][y])[l];
          a0 = t.x; a1 = t.y;
          if (n0 == 2) { const double2 u = reinterpret_cast<const double2*>(fr_[1][y])[l]; b0 = u.x; b1 = u.y; }
        }
      } else {
        a0 = fr_[0][y][2 * l];
        a1 = R(0);
        if (n0 == 2) b0 = fr_[1][y][2 * l];
      }
      v[y][0] = n0 == 1 ? a0 : R(0.5) * (a0 + b0);
      v[y][1] = n0 == 1 ? a1 : R(0.5) * (a1 + b1);
    }
    const R w0 = n1 == 1 ? v[0][0] : R(0.5) * (v[0][0] + v[1][0]);
    R res = w0;
    if (across) {
      const R w1 = n1 == 1 ? v[0][1] : R(0.5) * (v[0][1] + v[1][1]);
      res = R(0.5) * (w0 + w1);
    }
    o[l] = res;
  }
}

// face prolongation: linear along the normal, (3/4,1/4) across, axis order
template <int DIM, bool PER, class R>
__device__ __forceinline__ void pro_face_axis(int I, int n_c_axis, bool normal, int& i0, int& i1, R& w0, R& w1) {
  if (normal) {
    i0 = I >> 1;
    if (I & 1) {
      i1 = i0 + 1;
      if (PER && i1 >= n_c_axis) i1 -= n_c_axis;
      w0 = R(0.5);
      w1 = R(0.5);
    } else {
      i1 = i0;
      w0 = R(1);
      w1 = R(0);
    }
  } else {
    pro_idx<PER>(I, n_c_axis, i0, i1);
    w0 = R(0.75);
    w1 = R(0.25);
  }
}

// launch shape as k_prolong_cell, one launch per component k
template <int DIM, bool PER, class R, int MAXP>
__global__ void __launch_bounds__(32 * kProlongWarps) k_prolong_face(Ix<DIM, PER> cx, Ix<DIM, PER> fx, int k,
                                                                    const R* __restrict__ in, R* __restrict__ out,
                                                                    int N, int accumulate) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = DIM - 1;                             // last (contiguous) axis
  const int nl = fx.fe(k, L), cnl = cx.fe(k, L);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RPW = kProlongRows;
  R* crow = reinterpret_cast<R*>(smem_raw) + warp * RPW * cnl;   // this warp's combined coarse rows
  const int64_t nfc = cx.faces(k), nff = fx.faces(k);
  const int fr = blockIdx.z;
  const int fe1 = fx.fe(k, 1), fe2 = DIM == 3 ? fx.fe(k, 2) : 1;
  const int ce1 = cx.fe(k, 1), ce2 = DIM == 3 ? cx.fe(k, 2) : 1;
  const int nrows = DIM == 3 ? fx.fe(k, 0) * fe1 : fx.fe(k, 0);
  const int rowb = (blockIdx.y * kProlongWarps + warp) * RPW;
  if (rowb >= nrows) return;
  const R* p = in + (int64_t)fr * nfc;
  int F[RPW][2];
  R* orow[RPW];
  R old[RPW][MAXP][2];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int row = rowb + r < nrows ? rowb + r : rowb;   // past the end: a duplicate, never stored
    F[r][0] = DIM == 3 ? row / fe1 : row;
    F[r][1] = DIM == 3 ? row - F[r][0] * fe1 : 0;
    // in-frame offsets in 32 bits (a frame has < 2^31 elements)
    orow[r] = out + (int64_t)fr * nff + (F[r][0] * fe1 + F[r][1]) * fe2;
    pro_old<R, MAXP>(orow[r], nl, lane, accumulate, old[r]);
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    int i0[2] = {0, 0}, i1[2] = {0, 0};
    R w0[2] = {R(1), R(1)}, w1[2] = {R(0), R(0)};
#pragma unroll
    for (int a = 0; a < DIM - 1; ++a)
      pro_face_axis<DIM, PER, R>(F[r][a], cx.n(a), a == k, i0[a], i1[a], w0[a], w1[a]);
    // sequential axis application over the leading axes (axis 0, then 1); a
    // weight of exactly (1, 0) reproduces numpy's plain copy bit-for-bit
    const R* rr[2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
        rr[x][y] = p + ((x ? i1[0] : i0[0]) * ce1 + (DIM == 3 ? (y ? i1[1] : i0[1]) : 0)) * ce2;
    R* cr = crow + r * cnl;
    for (int l = lane; l < cnl; l += 32) {
      auto ax0 = [&](int y) -> R {
        const R a = rr[0][y][l];
        if (w1[0] == R(0)) return a;
        return w0[0] * a + w1[0] * rr[1][y][l];
      };
      R c = ax0(0);
      if (DIM == 3 && w1[1] != R(0)) c = w0[1] * c + w1[1] * ax0(1);
      cr[l] = c;
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r)
    if (rowb + r < nrows) pro_row<PER, R, MAXP>(crow + r * cnl, cnl, L == k, orow[r], nl, lane, accumulate, old[r]);
}

// ===========================================================================
// transport
// ===========================================================================

// out = s * T(v) x  (T from advection.py:88-97); optional acc += out and
// max |out| reduction.  v has `vframes` frames (1 = broadcast).  `gate`: the
// previous Taylor term's norm -- a term launched speculatively past the
// adaptive stop (*gate < gate_tol, advection.py:157-160) is a no-op and leaves
// its own norm slot at 0, so every later term is skipped too.
template <int DIM, bool PER, class R>
__global__ void k_transport(Ix<DIM, PER> ix, R c0, Face3<R> v, int vframes, const R* __restrict__ x,
                            R* __restrict__ out, R s, R* __restrict__ acc, R* norm, int N,
                            const R* gate = nullptr, R gate_tol = R(0)) {
  if (gate && *gate < gate_tol) return;
  const int64_t nc = ix.cells();
  R m = R(0);
  SMK_GRID_STRIDE(t, (int64_t)N * nc) {
    int fr = (int)(t / nc);
    int c[3];
    ix.cell_idx(t - (int64_t)fr * nc, c);
    const R* xp = x + (int64_t)fr * nc;
    int vf = vframes == 1 ? 0 : fr;
    R o = R(0);
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      const R* vk = v.c[k] + (int64_t)vf * ix.faces(k);
      int hi[3], lo[3];
      shift(c, k, 1, hi);
      shift(c, k, -1, lo);
      R vp = ix.face(vk, k, hi[0], hi[1], hi[2]);
      R vm = vk[ix.face_off(k, c[0], c[1], c[2])];
      o -= c0 * (vp * ix.cell(xp, hi[0], hi[1], hi[2]) - vm * ix.cell(xp, lo[0], lo[1], lo[2]));
    }
    R term = s * o;
    out[t] = term;
    if (acc) acc[t] = acc[t] + term;
    m = max(m, rabs(term));
  }
  if (norm) block_max_to(m, norm);
}

// g_k[f] = -(1/2h)(y_L x_R - y_R x_L)  (advection.py:105-130)
template <int DIM, bool PER, class R>
__global__ void k_stencil_v_adj(Ix<DIM, PER> ix, R c0, const R* __restrict__ x, const R* __restrict__ y,
                                FaceW<R> out, int N) {
  const int k = blockIdx.y;
  const int64_t nf = ix.faces(k), nc = ix.cells();
  SMK_GRID_STRIDE(t, (int64_t)N * nf) {
    int fr = (int)(t / nf);
    int c[3];
    ix.face_idx(k, t - (int64_t)fr * nf, c);
    R val = R(0);
    if (!ix.wall(k, c)) {
      const R* xp = x + (int64_t)fr * nc;
      const R* yp = y + (int64_t)fr * nc;
      int L[3];
      shift(c, k, -1, L);
      R xr = ix.cell(xp, c[0], c[1], c[2]), yr = ix.cell(yp, c[0], c[1], c[2]);
      R xl = ix.cell(xp, L[0], L[1], L[2]), yl = ix.cell(yp, L[0], L[1], L[2]);
      val = -c0 * (yl * xr - yr * xl);
    }
    out.c[k][t] = val;
  }
}

// advect_scalar_v_T face accumulation (advection.py:177-210):
//   out = sum_t coeff_t sum_{s<=t} g(xs[s], ys[t-s])
template <int DIM, bool PER, class R>
__global__ void k_vT_faces(Ix<DIM, PER> ix, R c0, const R* __restrict__ xs, const R* __restrict__ ys, int K,
                           R dt, FaceW<R> out) {
  const int k = blockIdx.y;
  const int64_t nf = ix.faces(k), nc = ix.cells();
  SMK_GRID_STRIDE(t, nf) {
    int c[3];
    ix.face_idx(k, t, c);
    R res = R(0);
    if (!ix.wall(k, c)) {
      int L[3];
      shift(c, k, -1, L);
      int64_t oR = ix.cell_off(Ix<DIM, PER>::wrap(c[0], ix.n0), Ix<DIM, PER>::wrap(c[1], ix.n1),
                               DIM == 3 ? Ix<DIM, PER>::wrap(c[2], ix.n2) : 0);
      int64_t oL = ix.cell_off(Ix<DIM, PER>::wrap(L[0], ix.n0), Ix<DIM, PER>::wrap(L[1], ix.n1),
                               DIM == 3 ? Ix<DIM, PER>::wrap(L[2], ix.n2) : 0);
      R coeff = R(1);
      bool first = true;
      for (int tt = 0; tt < K; ++tt) {
        coeff = coeff * dt / R(tt + 1);
        R acc = R(0);
        for (int s = 0; s <= tt; ++s) {
          const R* xp = xs + (int64_t)s * nc;
          const R* yp = ys + (int64_t)(tt - s) * nc;
          R g = -c0 * (yp[oL] * xp[oR] - yp[oR] * xp[oL]);
          acc = (s == 0) ? g : acc + g;
        }
        R term = coeff * acc;
        res = first ? term : res + term;
        first = false;
      }
    }
    out.c[k][t] = res;
  }
}

// S(a, w), J(v) d = S(v,d)+S(d,v), J(v)^T u  -- one face per thread
enum { FACE_S = 0, FACE_J = 1, FACE_JT = 2 };

template <int DIM, bool PER, class R>
__global__ void k_face_op(Ix<DIM, PER> ix, R c0, Face3<R> a, Face3<R> w, FaceW<R> out, int N, int op) {
  const int j = blockIdx.y;
  const int64_t nf = ix.faces(j);
  SMK_GRID_STRIDE(t, (int64_t)N * nf) {
    int fr = (int)(t / nf);
    int f[3];
    ix.face_idx(j, t - (int64_t)fr * nf, f);
    Face3<R> af, wf;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      af.c[k] = k < DIM ? a.c[k] + (int64_t)fr * ix.faces(k) : nullptr;
      wf.c[k] = k < DIM ? w.c[k] + (int64_t)fr * ix.faces(k) : nullptr;
    }
    MemField<DIM, PER, R> A{ix, af}, W{ix, wf};
    R val;
    if (op == FACE_S) val = S_at<DIM, PER, R>(ix, c0, j, f, A, W);
    else if (op == FACE_J) val = S_at<DIM, PER, R>(ix, c0, j, f, A, W) + S_at<DIM, PER, R>(ix, c0, j, f, W, A);
    else val = JT_at<DIM, PER, R>(ix, c0, j, f, A, W);
    out.c[j][t] = val;
  }
}

// semi_lagrangian (advection.py:264-299)
template <int DIM, bool PER, class R>
__global__ void k_semi_lagrangian(Ix<DIM, PER> ix, R h, Face3<R> v, const R* __restrict__ rho, R dt,
                                  R* __restrict__ out) {
  SMK_GRID_STRIDE(t, ix.cells()) {
    int c[3];
    ix.cell_idx(t, c);
    int i0[3] = {0, 0, 0};
    R fr[3] = {R(0), R(0), R(0)};
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
      int hi[3];
      shift(c, k, 1, hi);
      R vp = ix.face(v.c[k], k, hi[0], hi[1], hi[2]);
      R vm = v.c[k][ix.face_off(k, c[0], c[1], c[2])];
      if (!PER) {  // walls were zeroed by the caller contract (advection.py:268)
        if (hi[k] == ix.n(k)) vp = R(0);
        if (c[k] == 0) vm = R(0);
      }
      R vel = R(0.5) * (vp + vm);
      R s = (R(c[k]) + R(0.5)) - dt * vel / h;
      R q = s - R(0.5);
      R b = floor(q);
      i0[k] = (int)b;
      fr[k] = q - b;
    }
    R acc = R(0);
    for (int corner = 0; corner < (1 << DIM); ++corner) {
      R w = R(1);
      int id[3] = {0, 0, 0};
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        int bit = (corner >> k) & 1;
        int ik = i0[k] + bit;
        int n = ix.n(k);
        if (PER) { ik %= n; if (ik < 0) ik += n; }
        else ik = ik < 0 ? 0 : (ik > n - 1 ? n - 1 : ik);
        id[k] = ik;
        w = w * (bit ? fr[k] : R(1) - fr[k]);
      }
      acc += w * rho[ix.cell_off(id[0], id[1], id[2])];
    }
    out[t] = acc;
  }
}

// ===========================================================================
// Poisson multigrid (fields.py:287-347)
// ===========================================================================

template <int DIM, bool PER, class R>
__global__ void k_jacobi(Ix<DIM, PER> ix, R h, R omega, const R* __restrict__ p, const R* __restrict__ rhs,
                         R* __restrict__ out, int zero_guess) {
  SMK_GRID_STRIDE(t, ix.cells()) {
    int c[3];
    ix.cell_idx(t, c);
    R L = zero_guess ? R(0) : lap_at(ix, h, p, c);
    R pv = zero_guess ? R(0) : p[t];
    out[t] = pv + omega * (rhs[t] - L) / lap_diag_at(ix, h, c);
  }
}

// coarse residual: restrict(rhs - L p) with the reference's averaging order
template <int DIM, bool PER, class R>
__global__ void k_resid_restrict(Ix<DIM, PER> fx, Ix<DIM, PER> cx, R h, const R* __restrict__ p,
                                 const R* __restrict__ rhs, R* __restrict__ out) {
  SMK_GRID_STRIDE(t, cx.cells()) {
    int c[3];
    cx.cell_idx(t, c);
    R v[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < (DIM == 3 ? 2 : 1); ++e) {
        int r0[3] = {2 * c[0], 2 * c[1] + b, DIM == 3 ? 2 * c[2] + e : 0};
        int r1[3] = {2 * c[0] + 1, r0[1], r0[2]};
        R a0 = rhs[fx.cell_off(r0[0], r0[1], r0[2])] - lap_at(fx, h, p, r0);
        R a1 = rhs[fx.cell_off(r1[0], r1[1], r1[2])] - lap_at(fx, h, p, r1);
        v[b][e] = R(0.5) * (a0 + a1);
      }
    R w0 = R(0.5) * (v[0][0] + v[1][0]);
    R res = w0;
    if (DIM == 3) res = R(0.5) * (w0 + R(0.5) * (v[0][1] + v[1][1]));
    out[t] = res;
  }
}

template <int DIM, bool PER, class R>
__global__ void k_resid_absmax(Ix<DIM, PER> ix, R h, const R* __restrict__ p, const R* __restrict__ rhs, R* norm) {
  R m = R(0);
  SMK_GRID_STRIDE(t, ix.cells()) {
    int c[3];
    ix.cell_idx(t, c);
    m = max(m, rabs(rhs[t] - lap_at(ix, h, p, c)));
  }
  block_max_to(m, norm);
}

template <class R>
__global__ void k_dense_matvec(const R* __restrict__ A, const R* __restrict__ x, R* __restrict__ y, int n) {
  // one warp per row; fixed summation order (lane-strided partial + tree)
  int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (row >= n) return;
  R s = R(0);
  for (int j = lane; j < n; j += 32) s += A[(int64_t)row * n + j] * x[j];
  s = warp_sum(s);
  if (lane == 0) y[row] = s;
}

}  // namespace smk

// ===========================================================================
// host side
// ===========================================================================
using namespace smk;

namespace smk {

namespace {
// Process-wide stream-ordered scratch pool: buffers return with an event
// recorded on the releasing stream and are reused by size on the SAME device
// (entries are keyed by (device, rounded size)); at most kPoolCap bytes stay
// pooled per device, and smk_pool_trim() / an allocation failure hands them
// back to the driver.
struct PoolEntry {
  void* p;
  cudaStream_t st;
  cudaEvent_t ev;
};
using PoolKey = std::pair<int, size_t>;
std::mutex g_pool_mu;
std::multimap<PoolKey, PoolEntry> g_pool;
std::map<int, size_t> g_pool_bytes;        // pooled bytes per device
constexpr size_t kPoolMax = size_t(1) << 30;   // largest pooled buffer
constexpr size_t kPoolCap = size_t(4) << 30;   // pooled bytes per device

size_t pool_round(size_t b) {
  b = b < 256 ? 256 : b;
  return (b + 4095) & ~size_t(4095);
}
int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d;
}
// free every pooled buffer of device dev (-1: all devices)
void pool_drop(int dev) {
  std::vector<std::pair<PoolKey, PoolEntry>> drop;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (auto it = g_pool.begin(); it != g_pool.end();) {
      if (dev < 0 || it->first.first == dev) {
        drop.push_back(*it);
        g_pool_bytes[it->first.first] -= it->first.second;
        it = g_pool.erase(it);
      } else {
        ++it;
      }
    }
  }
  const int here = cur_device();
  for (auto& kv : drop) {
    if (kv.first.first != here) cudaSetDevice(kv.first.first);
    cudaEventSynchronize(kv.second.ev);
    cudaEventDestroy(kv.second.ev);
    cudaFree(kv.second.p);
    if (kv.first.first != here) cudaSetDevice(here);
  }
}
}  // namespace

void pool_trim() { pool_drop(-1); }

Scratch::~Scratch() { release(); }
void Scratch::release() {
  const int dev = cur_device();
  for (auto& b : bufs) {
    if (!b.first) continue;
    if (pooled && b.second <= kPoolMax) {
      bool room;
      {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        room = g_pool_bytes[dev] + b.second <= kPoolCap;
      }
      cudaEvent_t ev = nullptr;
      if (room && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess &&
          cudaEventRecord(ev, st) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        g_pool.emplace(PoolKey{dev, b.second}, PoolEntry{b.first, st, ev});
        g_pool_bytes[dev] += b.second;
        continue;
      }
      cudaGetLastError();
      if (ev) cudaEventDestroy(ev);
      cudaStreamSynchronize(st);
    }
    cudaFree(b.first);
  }
  bufs.clear();
}
void* Scratch::get(size_t bytes) {
  const size_t r = pool_round(bytes);
  const int dev = cur_device();
  if (pooled && r <= kPoolMax) {
    PoolEntry e{nullptr, nullptr, nullptr};
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      auto it = g_pool.find(PoolKey{dev, r});
      if (it != g_pool.end()) {
        e = it->second;
        g_pool.erase(it);
        g_pool_bytes[dev] -= r;
      }
    }
    if (e.p) {
      if (e.st != st) cudaStreamWaitEvent(st, e.ev, 0);
      cudaEventDestroy(e.ev);
      bufs.push_back({e.p, r});
      return e.p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, r) != cudaSuccess) {
    cudaGetLastError();
    // out of memory: hand this device's pooled buffers back and retry
    pool_drop(dev);
    if (cudaMalloc(&p, r) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  bufs.push_back({p, r});
  return p;
}

double host_absmax(int dtype, const void* x, int64_t n, cudaStream_t st, void* dev_scalar) {
  cudaMemsetAsync(dev_scalar, 0, 8, st);
  if (n > 0) {
    if (dtype == SMK_F64) k_absmax<double><<<grid_for(n, 256), 256, 0, st>>>((const double*)x, n, (double*)dev_scalar);
    else k_absmax<float><<<grid_for(n, 256), 256, 0, st>>>((const float*)x, n, (float*)dev_scalar);
    count_launch();
  }
  double out = 0.0;
  if (dtype == SMK_F64) {
    cudaMemcpyAsync(&out, dev_scalar, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
  } else {
    float f = 0.f;
    cudaMemcpyAsync(&f, dev_scalar, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    out = f;
  }
  return out;
}

double host_sum(int dtype, const void* x, const void* y, int64_t n, cudaStream_t st, double* dev_parts) {
  const int parts = 256;
  if (dtype == SMK_F64) k_partial_sum<double><<<parts, 256, 0, st>>>((const double*)x, (const double*)y, n, dev_parts);
  else k_partial_sum<float><<<parts, 256, 0, st>>>((const float*)x, (const float*)y, n, dev_parts);
  count_launch();
  k_final_sum<<<1, 256, 0, st>>>(dev_parts, parts, dev_parts + parts); count_launch();
  double out = 0.0;
  cudaMemcpyAsync(&out, dev_parts + parts, 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return out;
}

template <class R>
void frame_sub_mean(R* x, int64_t per, int nframes, cudaStream_t st, double* dev_parts) {
  const int parts = 64;
  dim3 g1(parts, nframes);
  k_frame_partial<R><<<g1, 256, 0, st>>>(x, per, parts, dev_parts); count_launch();
  dim3 g2(grid_for(per, 256) < 64 ? grid_for(per, 256) : 64, nframes);
  k_frame_sub_mean<R><<<g2, 256, 0, st>>>(x, per, parts, dev_parts, nframes); count_launch();
}
template void frame_sub_mean<double>(double*, int64_t, int, cudaStream_t, double*);
template void frame_sub_mean<float>(float*, int64_t, int, cudaStream_t, double*);

template <class R>
void axpby(R* y, const R* x, double a, double b, int64_t n, cudaStream_t st) {
  k_axpby<R><<<grid_for(n, 256), 256, 0, st>>>(y, x, (R)a, (R)b, n); count_launch();
}
template void axpby<double>(double*, const double*, double, double, int64_t, cudaStream_t);
template void axpby<float>(float*, const float*, double, double, int64_t, cudaStream_t);

// ---------------------------------------------------------------------------
// generic launchers (used by the STFAS host code too)
// ---------------------------------------------------------------------------
template <int DIM, bool PER, class R>
void launch_div(const Geo& g, int N, Face3<R> v, R* out, cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  int64_t n = (int64_t)N * ix.cells();
  k_div<DIM, PER, R><<<grid_for(n, 256), 256, 0, st>>>(ix, (R)g.h, v, out, N); count_launch();
}
template <int DIM, bool PER, class R>
void launch_grad(const Geo& g, int N, const R* p, FaceW<R> out, cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  int64_t n = (int64_t)N * ix.faces(0);
  dim3 grid(grid_for(n, 256), DIM);
  k_grad<DIM, PER, R><<<grid, 256, 0, st>>>(ix, (R)g.h, p, out, N); count_launch();
}
template <int DIM, bool PER, class R>
void launch_face_op(const Geo& g, int N, Face3<R> a, Face3<R> w, FaceW<R> out, int op, cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  int64_t n = (int64_t)N * ix.faces(0);
  dim3 grid(grid_for(n, 256), DIM);
  k_face_op<DIM, PER, R><<<grid, 256, 0, st>>>(ix, (R)(0.5 / g.h), a, w, out, N, op); count_launch();
}
template <int DIM, bool PER, class R>
void launch_restrict_cell(const Geo& gf, int N, const R* x, R* out, cudaStream_t st) {
  Geo gc = coarsen(gf);
  Ix<DIM, PER> fx(gf), cx(gc);
  k_restrict_cell<DIM, PER, R><<<frame_grid(cx.cells(), N, 256), 256, 0, st>>>(fx, cx, x, out, N); count_launch();
}
template <int DIM, bool PER, class R>
void prolong_cell_go(const Ix<DIM, PER>& cx, const Ix<DIM, PER>& fx, int N, const R* x, R* out, int acc,
                     cudaStream_t st) {
  int tpb;
  const dim3 grid = prolong_cell_grid(fx, N, tpb);
  const size_t shm = prolong_cell_smem<DIM, PER, R>(cx);
  const int nl = DIM == 3 ? fx.n2 : fx.n1;
  if (nl <= 192) k_prolong_cell<DIM, PER, R, 3><<<grid, tpb, shm, st>>>(cx, fx, x, out, N, acc);
  else k_prolong_cell<DIM, PER, R, 5><<<grid, tpb, shm, st>>>(cx, fx, x, out, N, acc);
  count_launch();
}
template <int DIM, bool PER, class R>
void launch_prolong_cell(const Geo& gc, int N, const R* x, R* out, int acc, cudaStream_t st) {
  Geo gf = refine(gc);
  Ix<DIM, PER> fx(gf), cx(gc);
  prolong_cell_go<DIM, PER, R>(cx, fx, N, x, out, acc, st);
}
template <int DIM, bool PER, class R>
void launch_restrict_face(const Geo& gf, int N, Face3<R> in, FaceW<R> out, cudaStream_t st) {
  Geo gc = coarsen(gf);
  Ix<DIM, PER> fx(gf), cx(gc);
  int rows = 0;
  for (int k = 0; k < DIM; ++k) rows = std::max(rows, DIM == 3 ? cx.fe(k, 0) * cx.fe(k, 1) : cx.fe(k, 0));
  const dim3 grid(DIM, (rows + kRestrictWarps - 1) / kRestrictWarps, N);
  k_restrict_face<DIM, PER, R><<<grid, 32 * kRestrictWarps, 0, st>>>(fx, cx, in, out, N);
  count_launch();
}
template <int DIM, bool PER, class R>
void launch_prolong_face(const Geo& gc, int N, Face3<R> in, FaceW<R> out, int acc, cudaStream_t st) {
  Geo gf = refine(gc);
  Ix<DIM, PER> fx(gf), cx(gc);
  for (int k = 0; k < DIM; ++k) {
    const int rows = DIM == 3 ? fx.fe(k, 0) * fx.fe(k, 1) : fx.fe(k, 0);
    const dim3 grid(1, (rows + kProlongWarps * kProlongRows - 1) / (kProlongWarps * kProlongRows), N);
    const size_t shm = (size_t)kProlongWarps * kProlongRows * cx.fe(k, DIM - 1) * sizeof(R);
    if (shm > 48 * 1024) {
      cudaFuncSetAttribute(k_prolong_face<DIM, PER, R, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
      cudaFuncSetAttribute(k_prolong_face<DIM, PER, R, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    }
    if (fx.fe(k, DIM - 1) <= 192)
      k_prolong_face<DIM, PER, R, 3><<<grid, 32 * kProlongWarps, shm, st>>>(cx, fx, k, in.c[k], out.c[k], N, acc);
    else
      k_prolong_face<DIM, PER, R, 5><<<grid, 32 * kProlongWarps, shm, st>>>(cx, fx, k, in.c[k], out.c[k], N, acc);
    count_launch();
  }
}

#define SMK_INST(DIM, PER, R)                                                                               \
  template void launch_div<DIM, PER, R>(const Geo&, int, Face3<R>, R*, cudaStream_t);                     \
  template void launch_grad<DIM, PER, R>(const Geo&, int, const R*, FaceW<R>, cudaStream_t);              \
  template void launch_face_op<DIM, PER, R>(const Geo&, int, Face3<R>, Face3<R>, FaceW<R>, int, cudaStream_t); \
  template void launch_restrict_cell<DIM, PER, R>(const Geo&, int, const R*, R*, cudaStream_t);           \
  template void launch_prolong_cell<DIM, PER, R>(const Geo&, int, const R*, R*, int, cudaStream_t);       \
  template void launch_restrict_face<DIM, PER, R>(const Geo&, int, Face3<R>, FaceW<R>, cudaStream_t);     \
  template void launch_prolong_face<DIM, PER, R>(const Geo&, int, Face3<R>, FaceW<R>, int, cudaStream_t);
SMK_INST(2, false, double)
SMK_INST(2, true, double)
SMK_INST(3, false, double)
SMK_INST(3, true, double)
SMK_INST(2, false, float)
SMK_INST(2, true, float)
SMK_INST(3, false, float)
SMK_INST(3, true, float)
#undef SMK_INST

Geo coarsen(const Geo& g) {
  Geo c = g;
  for (int a = 0; a < g.dim; ++a) c.n[a] = g.n[a] / 2;
  c.h = 2.0 * g.h;
  return c;
}
Geo refine(const Geo& g) {
  Geo f = g;
  for (int a = 0; a < g.dim; ++a) f.n[a] = g.n[a] * 2;
  f.h = 0.5 * g.h;
  return f;
}
bool can_coarsen(const Geo& g) {
  for (int a = 0; a < g.dim; ++a)
    if (g.n[a] % 2 || g.n[a] / 2 < 4) return false;
  return true;
}

int64_t cells_of(const Geo& g) { return (int64_t)g.n[0] * g.n[1] * (g.dim == 3 ? g.n[2] : 1); }
int64_t faces_of(const Geo& g, int k) {
  int64_t n = 1;
  for (int a = 0; a < g.dim; ++a) n *= g.n[a] + ((!g.periodic && a == k) ? 1 : 0);
  return n;
}

// ---------------------------------------------------------------------------
// Poisson: coarsest pseudo-inverse (symmetric Jacobi eigensolver on host,
// cached per grid), then V(2,2) cycles on device
// ---------------------------------------------------------------------------
static std::vector<double> host_laplacian_matrix(const Geo& g) {
  int64_t n = cells_of(g);
  std::vector<double> A(n * n, 0.0);
  int nn[3] = {g.n[0], g.n[1], g.dim == 3 ? g.n[2] : 1};
  auto off = [&](int i, int j, int l) { return ((int64_t)i * nn[1] + j) * nn[2] + l; };
  double h = g.h;
  for (int64_t col = 0; col < n; ++col) {
    // L e_col evaluated with the same closure as fields.py:_laplacian
    int c[3] = {(int)(col / ((int64_t)nn[1] * nn[2])), (int)((col / nn[2]) % nn[1]), (int)(col % nn[2])};
    for (int k = 0; k < g.dim; ++k) {
      for (int s = -1; s <= 1; s += 2) {
        int q[3] = {c[0], c[1], c[2]};
        q[k] += s;
        bool wall = false;
        if (g.periodic) q[k] = (q[k] + nn[k]) % nn[k];
        else if (q[k] < 0 || q[k] >= nn[k]) wall = true;
        if (wall) continue;
        // face between c and q carries (p_q - p_c)/h (oriented), contributes
        // +1/h^2 to row q ... symmetric 5/7-point stencil
        A[off(q[0], q[1], q[2]) * n + col] += 1.0 / (h * h);
        A[col * n + col] -= 1.0 / (h * h);
      }
    }
  }
  return A;
}

static void jacobi_eigen(std::vector<double>& A, int n, std::vector<double>& w, std::vector<double>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += A[(size_t)p * n + q] * A[(size_t)p * n + q];
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = A[(size_t)p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
          A[(size_t)k * n + p] = c * akp - s * akq;
          A[(size_t)k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
          A[(size_t)p * n + k] = c * apk - s * aqk;
          A[(size_t)q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
          V[(size_t)k * n + p] = c * vkp - s * vkq;
          V[(size_t)k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = A[(size_t)i * n + i];
}

static std::vector<double> host_pinv_laplacian(const Geo& g) {
  int n = (int)cells_of(g);
  std::vector<double> A = host_laplacian_matrix(g), w, V;
  jacobi_eigen(A, n, w, V);
  double wmax = 0.0;
  for (double x : w) wmax = std::max(wmax, std::fabs(x));
  std::vector<double> P((size_t)n * n, 0.0);
  for (int e = 0; e < n; ++e) {
    if (std::fabs(w[e]) <= 1e-12 * wmax) continue;  // numpy pinv rcond=1e-12
    double inv = 1.0 / w[e];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) P[(size_t)i * n + j] += V[(size_t)i * n + e] * inv * V[(size_t)j * n + e];
  }
  return P;
}

struct PinvKey {
  int dev;
  int dim, n0, n1, n2, per, dtype;
  long long hbits;
  bool operator<(const PinvKey& o) const {
    return std::tie(dev, dim, n0, n1, n2, per, dtype, hbits) <
           std::tie(o.dev, o.dim, o.n0, o.n1, o.n2, o.per, o.dtype, o.hbits);
  }
};
static std::mutex g_pinv_mu;
static std::map<PinvKey, void*> g_pinv;

const void* device_pinv(const Geo& g, int dtype) {
  long long hb;
  memcpy(&hb, &g.h, 8);
  PinvKey key{cur_device(), g.dim, g.n[0], g.n[1], g.n[2], g.periodic, dtype, hb};
  std::lock_guard<std::mutex> lk(g_pinv_mu);
  auto it = g_pinv.find(key);
  if (it != g_pinv.end()) return it->second;
  std::vector<double> P = host_pinv_laplacian(g);
  void* d = nullptr;
  size_t es = dtype == SMK_F64 ? 8 : 4;
  if (cudaMalloc(&d, P.size() * es) != cudaSuccess) return nullptr;
  if (dtype == SMK_F64) {
    cudaMemcpy(d, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
  } else {
    std::vector<float> f(P.begin(), P.end());
    cudaMemcpy(d, f.data(), f.size() * 4, cudaMemcpyHostToDevice);
  }
  g_pinv[key] = d;
  return d;
}

template <int DIM, bool PER, class R>
struct PoissonMG {
  std::vector<Geo> lv;
  std::vector<R*> p, rhs, tmp;
  Scratch scratch;
  const R* pinv = nullptr;
  bool ok = true;

  PoissonMG(const Geo& g, cudaStream_t st) : scratch(st) {
    lv.push_back(g);
    while (can_coarsen(lv.back())) lv.push_back(coarsen(lv.back()));
    for (size_t i = 0; i < lv.size(); ++i) {
      size_t b = (size_t)cells_of(lv[i]) * sizeof(R);
      p.push_back((R*)scratch.get(b));
      rhs.push_back((R*)scratch.get(b));
      tmp.push_back((R*)scratch.get(b));
      if (!p.back() || !rhs.back() || !tmp.back()) ok = false;
    }
    pinv = (const R*)device_pinv(lv.back(), sizeof(R) == 8 ? SMK_F64 : SMK_F32);
    if (!pinv) ok = false;
  }

  // one V-cycle at level li on (p[li], rhs[li]); zero initial guess when zg
  void vcycle(size_t li, bool zg, cudaStream_t st) {
    const Geo& g = lv[li];
    Ix<DIM, PER> ix(g);
    int64_t n = ix.cells();
    if (li + 1 == lv.size()) {
      int nn = (int)n;
      k_dense_matvec<R><<<(nn + 7) / 8, 256, 0, st>>>(pinv, rhs[li], p[li], nn); count_launch();
      return;
    }
    R h = (R)g.h, om = (R)0.8;
    int gb = grid_for(n, 256);
    // pre-smoothing (2 damped Jacobi sweeps), ping-pong p <-> tmp
    k_jacobi<DIM, PER, R><<<gb, 256, 0, st>>>(ix, h, om, p[li], rhs[li], tmp[li], zg ? 1 : 0); count_launch();
    k_jacobi<DIM, PER, R><<<gb, 256, 0, st>>>(ix, h, om, tmp[li], rhs[li], p[li], 0); count_launch();
    const Geo& gc = lv[li + 1];
    Ix<DIM, PER> cx(gc);
    k_resid_restrict<DIM, PER, R><<<grid_for(cx.cells(), 256), 256, 0, st>>>(ix, cx, h, p[li], rhs[li], rhs[li + 1]); count_launch();
    vcycle(li + 1, true, st);
    {
      prolong_cell_go<DIM, PER, R>(cx, ix, 1, p[li + 1], p[li], 1, st);
    }
    k_jacobi<DIM, PER, R><<<gb, 256, 0, st>>>(ix, h, om, p[li], rhs[li], tmp[li], 0); count_launch();
    k_jacobi<DIM, PER, R><<<gb, 256, 0, st>>>(ix, h, om, tmp[li], rhs[li], p[li], 0); count_launch();
  }
};

// rhs_in: device array (1 frame).  Writes p_out.  Returns status.
template <int DIM, bool PER, class R>
int poisson_solve(const Geo& g, const R* rhs_in, R* p_out, double tol, int max_cycles, int* cycles,
                  double* residual, cudaStream_t st) {
  PoissonMG<DIM, PER, R> mg(g, st);
  if (!mg.ok) { set_error("poisson: allocation failed"); return SMK_ERR_CUDA; }
  Ix<DIM, PER> ix(g);
  int64_t n = ix.cells();
  Scratch sc(st);
  double* parts = (double*)sc.get(sizeof(double) * 600);
  void* scal = sc.get(16);
  // rhs - mean(rhs)
  cudaMemcpyAsync(mg.rhs[0], rhs_in, n * sizeof(R), cudaMemcpyDeviceToDevice, st);
  frame_sub_mean<R>(mg.rhs[0], n, 1, st, parts);
  double r0 = host_absmax(sizeof(R) == 8 ? SMK_F64 : SMK_F32, mg.rhs[0], n, st, scal);
  if (cycles) *cycles = 0;
  if (r0 <= tol) {
    cudaMemsetAsync(p_out, 0, n * sizeof(R), st);
    if (residual) *residual = r0;
    return cuda_check("poisson");
  }
  cudaMemsetAsync(mg.p[0], 0, n * sizeof(R), st);
  double r = INFINITY;
  for (int it = 0; it < max_cycles; ++it) {
    mg.vcycle(0, it == 0, st);
    cudaMemsetAsync(scal, 0, 8, st);
    k_resid_absmax<DIM, PER, R><<<grid_for(n, 256), 256, 0, st>>>(ix, (R)g.h, mg.p[0], mg.rhs[0], (R*)scal); count_launch();
    R rv;
    cudaMemcpyAsync(&rv, scal, sizeof(R), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    r = (double)rv;
    if (r <= tol) {
      if (cycles) *cycles = it + 1;
      if (residual) *residual = r;
      cudaMemcpyAsync(p_out, mg.p[0], n * sizeof(R), cudaMemcpyDeviceToDevice, st);
      return cuda_check("poisson");
    }
  }
  if (cycles) *cycles = max_cycles;
  if (residual) *residual = r;
  cudaMemcpyAsync(p_out, mg.p[0], n * sizeof(R), cudaMemcpyDeviceToDevice, st);
  set_error("Poisson V-cycle budget exhausted (residual %.3e)", r);
  int rc = cuda_check("poisson");
  return rc ? rc : SMK_NONCONVERGENCE;
}

// project_arrays (fields.py:350-358); in/out may alias
template <int DIM, bool PER, class R>
int project(const Geo& g, Face3<R> in, FaceW<R> out, double tol, int* cycles, double* residual, cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  for (int k = 0; k < DIM; ++k)
    if ((const R*)out.c[k] != in.c[k])
      cudaMemcpyAsync(out.c[k], in.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
  {
    dim3 grid(grid_for(ix.faces(0), 256), DIM);
    k_zero_walls<DIM, PER, R><<<grid, 256, 0, st>>>(ix, out, 1); count_launch();
  }
  Scratch sc(st);
  int64_t n = ix.cells();
  R* dv = (R*)sc.get(n * sizeof(R));
  R* phi = (R*)sc.get(n * sizeof(R));
  void* scal = sc.get(16);
  Face3<R> o3;
  for (int k = 0; k < 3; ++k) o3.c[k] = out.c[k];
  launch_div<DIM, PER, R>(g, 1, o3, dv, st);
  double r0 = host_absmax(sizeof(R) == 8 ? SMK_F64 : SMK_F32, dv, n, st, scal);
  if (cycles) *cycles = 0;
  if (residual) *residual = r0;
  if (r0 <= tol) return cuda_check("project");
  int rc = poisson_solve<DIM, PER, R>(g, dv, phi, tol, 200, cycles, residual, st);
  if (rc != SMK_OK && rc != SMK_NONCONVERGENCE) return rc;
  // out -= grad(phi): gradient into scratch then subtract
  FaceW<R> gr;
  for (int k = 0; k < 3; ++k) gr.c[k] = k < DIM ? (R*)sc.get(ix.faces(k) * sizeof(R)) : nullptr;
  launch_grad<DIM, PER, R>(g, 1, phi, gr, st);
  for (int k = 0; k < DIM; ++k) axpby<R>(out.c[k], gr.c[k], -1.0, 1.0, ix.faces(k), st);
  int rc2 = cuda_check("project");
  return rc2 ? rc2 : rc;
}

// Taylor exp(+-T dt) x (advection.py:144-174).  One launch per term.  The
// adaptive stop (first term with |term|inf < tol) is decided on the device:
// terms are launched in speculative batches, each gated on its predecessor's
// norm, and the host reads the norms once per batch (normally once per call:
// the first batch is as long as the previous call's order).
template <int DIM, bool PER, class R>
int advect(const Geo& g, Face3<R> v, const R* rho, R* out, double dt, double tol, int cap, int k_fixed,
           int transpose, int* k_used, double* last, cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  int64_t n = ix.cells();
  if (cap < 1) { set_error("advect: term cap must be >= 1"); return SMK_ERR_ARG; }
  Scratch sc(st);
  R* t0 = (R*)sc.get(n * sizeof(R));
  R* t1 = (R*)sc.get(n * sizeof(R));
  R* norms = (R*)sc.get(sizeof(R) * (size_t)(cap + 2));
  if (!t0 || !t1 || !norms) { set_error("advect: allocation failed"); return SMK_ERR_CUDA; }
  cudaMemcpyAsync(out, rho, n * sizeof(R), cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(norms, 0, sizeof(R) * (size_t)(cap + 2), st);
  const R* cur = rho;
  R* bufs[2] = {t0, t1};
  R c0 = (R)(0.5 / g.h);
  int gb = grid_for(n, 256);
  const bool adaptive = k_fixed <= 0;
  const int kmax = adaptive ? cap : (k_fixed < cap ? k_fixed : cap);
  static thread_local int hint = 6;
  std::vector<R> hn((size_t)cap + 2, R(0));
  int k = 0;  // terms launched so far
  while (k < kmax) {
    int upto = adaptive ? (k == 0 ? hint : k + 4) : kmax;
    if (upto > kmax) upto = kmax;
    for (++k; k <= upto; ++k) {
      R s = (R)(dt / (double)k);
      if (transpose) s = -s;
      R* nxt = bufs[(k - 1) & 1];
      // reference: term = (dt/k) * stencil(term) with stencil = +-T
      const R* gate = adaptive && k >= 2 ? norms + (k - 2) : nullptr;
      k_transport<DIM, PER, R><<<gb, 256, 0, st>>>(ix, c0, v, 1, cur, nxt, s, out, norms + (k - 1), 1, gate, (R)tol);
      count_launch();
      cur = nxt;
    }
    k = upto;
    cudaMemcpyAsync(hn.data(), norms, sizeof(R) * (size_t)k, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (!adaptive) break;
    for (int j = 1; j <= k; ++j)
      if (hn[j - 1] < (R)tol) {  // the device gate's comparison, same rounding
        hint = j;
        if (k_used) *k_used = j;
        if (last) *last = (double)hn[j - 1];
        return cuda_check("advect");
      }
  }
  if (last) *last = (double)hn[kmax - 1];
  if (k_used) *k_used = kmax;
  if (!adaptive && k_fixed <= cap) return cuda_check("advect");
  set_error("Taylor term cap %d exceeded (dt*|v|/h too large)", cap);
  return SMK_TRUNCATION_OVERFLOW;
}

template <int DIM, bool PER, class R>
int advect_v_T(const Geo& g, Face3<R> v, const R* rho, const R* mu, FaceW<R> out, double dt, int K, cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  int64_t n = ix.cells();
  if (K < 1) { set_error("advect_v_T: k must be >= 1"); return SMK_ERR_ARG; }
  Scratch sc(st);
  R* xs = (R*)sc.get((size_t)K * n * sizeof(R));
  R* ys = (R*)sc.get((size_t)K * n * sizeof(R));
  if (!xs || !ys) { set_error("advect_v_T: allocation failed"); return SMK_ERR_CUDA; }
  cudaMemcpyAsync(xs, rho, n * sizeof(R), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(ys, mu, n * sizeof(R), cudaMemcpyDeviceToDevice, st);
  R c0 = (R)(0.5 / g.h);
  int gb = grid_for(n, 256);
  for (int s = 1; s < K; ++s) {
    k_transport<DIM, PER, R><<<gb, 256, 0, st>>>(ix, c0, v, 1, xs + (s - 1) * n, xs + s * n, R(1), nullptr, nullptr, 1); count_launch();
    k_transport<DIM, PER, R><<<gb, 256, 0, st>>>(ix, c0, v, 1, ys + (s - 1) * n, ys + s * n, R(-1), nullptr, nullptr, 1); count_launch();
  }
  dim3 grid(grid_for(ix.faces(0), 256), DIM);
  k_vT_faces<DIM, PER, R><<<grid, 256, 0, st>>>(ix, c0, xs, ys, K, (R)dt, out); count_launch();
  return cuda_check("advect_v_T");
}

template <int DIM, bool PER, class R>
int sim_step(const Geo& g, Face3<R> v_in, const R* rho, Face3<R> u_in, double dt, int picard_iters, double sim_tol,
             double trunc_tol, int trunc_cap, FaceW<R> v_out, R* p_out, R* rho_out, int* k_used, double* pres,
             cudaStream_t st) {
  Ix<DIM, PER> ix(g);
  Scratch sc(st);
  FaceW<R> v, u, w, wn, adv, tgt;
  auto alloc_face = [&](FaceW<R>& f) {
    for (int k = 0; k < 3; ++k) f.c[k] = k < DIM ? (R*)sc.get(ix.faces(k) * sizeof(R)) : nullptr;
  };
  alloc_face(v); alloc_face(u); alloc_face(w); alloc_face(wn); alloc_face(adv); alloc_face(tgt);
  dim3 fg(grid_for(ix.faces(0), 256), DIM);
  for (int k = 0; k < DIM; ++k) {
    cudaMemcpyAsync(v.c[k], v_in.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(u.c[k], u_in.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
  }
  k_zero_walls<DIM, PER, R><<<fg, 256, 0, st>>>(ix, v, 1); count_launch();
  k_zero_walls<DIM, PER, R><<<fg, 256, 0, st>>>(ix, u, 1); count_launch();
  auto c3 = [](FaceW<R> f) { Face3<R> o; for (int k = 0; k < 3; ++k) o.c[k] = f.c[k]; return o; };
  // density: advected by the pre-step velocity (simulator.py:86-87)
  double lastn = 0;
  int rc = advect<DIM, PER, R>(g, c3(v), rho, rho_out, dt, trunc_tol, trunc_cap, 0, 0, k_used, &lastn, st);
  if (rc) return rc;
  // Picard (simulator.py:56-70)
  for (int k = 0; k < DIM; ++k) cudaMemcpyAsync(w.c[k], v.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
  void* scal = sc.get(16);
  double resid = INFINITY;
  for (int it = 0; it < picard_iters; ++it) {
    launch_face_op<DIM, PER, R>(g, 1, c3(w), c3(w), adv, FACE_S, st);
    // target = v + dt * (u - adv)
    for (int k = 0; k < DIM; ++k) {
      cudaMemcpyAsync(tgt.c[k], u.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
      axpby<R>(tgt.c[k], adv.c[k], -1.0, 1.0, ix.faces(k), st);
      k_axpby<R><<<grid_for(ix.faces(k), 256), 256, 0, st>>>(tgt.c[k], v.c[k], R(1), (R)dt, ix.faces(k)); count_launch();
    }
    int cyc;
    double pr;
    rc = project<DIM, PER, R>(g, c3(tgt), wn, sim_tol, &cyc, &pr, st);
    if (rc != SMK_OK) return rc;
    double m = 0;
    for (int k = 0; k < DIM; ++k) {
      cudaMemsetAsync(scal, 0, 8, st);
      k_absdiff_max<R><<<grid_for(ix.faces(k), 256), 256, 0, st>>>(wn.c[k], w.c[k], ix.faces(k), (R*)scal); count_launch();
      R mv;
      cudaMemcpyAsync(&mv, scal, sizeof(R), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      m = std::max(m, (double)mv);
    }
    resid = m;
    std::swap(w, wn);
    if (resid <= sim_tol) break;
  }
  // pressure recovery (simulator.py:89-99)
  launch_face_op<DIM, PER, R>(g, 1, c3(w), c3(w), adv, FACE_S, st);
  for (int k = 0; k < DIM; ++k) {
    // src = (v - w)/dt + u - adv   (evaluated as ((v - w)/dt + u) - adv)
    cudaMemcpyAsync(tgt.c[k], v.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
    axpby<R>(tgt.c[k], w.c[k], -1.0, 1.0, ix.faces(k), st);
    k_axpby<R><<<grid_for(ix.faces(k), 256), 256, 0, st>>>(tgt.c[k], u.c[k], R(1), (R)(1.0 / dt), ix.faces(k)); count_launch();
    axpby<R>(tgt.c[k], adv.c[k], -1.0, 1.0, ix.faces(k), st);
  }
  int64_t n = ix.cells();
  R* ds = (R*)sc.get(n * sizeof(R));
  double* parts = (double*)sc.get(sizeof(double) * 600);
  launch_div<DIM, PER, R>(g, 1, c3(tgt), ds, st);
  frame_sub_mean<R>(ds, n, 1, st, parts);
  double dn = host_absmax(sizeof(R) == 8 ? SMK_F64 : SMK_F32, ds, n, st, scal);
  if (dn > sim_tol) {
    int cyc;
    double pr;
    rc = poisson_solve<DIM, PER, R>(g, ds, p_out, sim_tol, 200, &cyc, &pr, st);
    if (rc != SMK_OK) return rc;
  } else {
    cudaMemsetAsync(p_out, 0, n * sizeof(R), st);
  }
  for (int k = 0; k < DIM; ++k)
    cudaMemcpyAsync(v_out.c[k], w.c[k], ix.faces(k) * sizeof(R), cudaMemcpyDeviceToDevice, st);
  if (pres) *pres = resid;
  cudaStreamSynchronize(st);
  rc = cuda_check("sim_step");
  if (rc) return rc;
  if (resid > sim_tol) {
    set_error("Picard update stalled at %.3e > sim_tol %.3e", resid, sim_tol);
    return SMK_NONCONVERGENCE;
  }
  return SMK_OK;
}

}  // namespace smk

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* smk_last_error(void) { return smk::g_err; }
int smk_version(void) { return 1; }
void smk_pool_trim(void) { smk::pool_trim(); }
long long smk_launch_count(void) { return smk::g_launches.load(); }

#define ST(s) ((cudaStream_t)(s))

int smk_div(const smk_grid* g, int N, const void* const comps[], void* out, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_div<T::DIM, T::PER, R>(to_geo(g), N, face3<R>(comps, g->dim), (R*)out, ST(stream));
    return cuda_check("smk_div");
  });
}

int smk_grad(const smk_grid* g, int N, const void* p, void* const out[], void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_grad<T::DIM, T::PER, R>(to_geo(g), N, (const R*)p, facew<R>(out, g->dim), ST(stream));
    return cuda_check("smk_grad");
  });
}

int smk_zero_walls(const smk_grid* g, int N, void* const comps[], void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    Ix<T::DIM, T::PER> ix(to_geo(g));
    dim3 grid(grid_for((int64_t)N * ix.faces(0), 256), T::DIM);
    k_zero_walls<T::DIM, T::PER, R><<<grid, 256, 0, ST(stream)>>>(ix, facew<R>(comps, g->dim), N); count_launch();
    return cuda_check("smk_zero_walls");
  });
}

int smk_laplacian(const smk_grid* g, int N, const void* p, void* out, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    Ix<T::DIM, T::PER> ix(to_geo(g));
    int64_t n = (int64_t)N * ix.cells();
    k_laplacian<T::DIM, T::PER, R><<<grid_for(n, 256), 256, 0, ST(stream)>>>(ix, (R)g->h, (const R*)p, (R*)out, N); count_launch();
    return cuda_check("smk_laplacian");
  });
}

int smk_inf_norm(int dtype, const void* x, int64_t n, double* out, void* stream) {
  if (dtype != SMK_F64 && dtype != SMK_F32) { set_error("bad dtype"); return SMK_ERR_ARG; }
  Scratch sc(ST(stream));
  void* scal = sc.get(16);
  *out = host_absmax(dtype, x, n, ST(stream), scal);
  return cuda_check("smk_inf_norm");
}

int smk_dot(int dtype, const void* x, const void* y, int64_t n, double* out, void* stream) {
  if (dtype != SMK_F64 && dtype != SMK_F32) { set_error("bad dtype"); return SMK_ERR_ARG; }
  Scratch sc(ST(stream));
  double* parts = (double*)sc.get(sizeof(double) * 600);
  *out = host_sum(dtype, x, y, n, ST(stream), parts);
  return cuda_check("smk_dot");
}

int smk_restrict_cell(const smk_grid* g, int N, const void* x, void* out, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    for (int a = 0; a < g->dim; ++a)
      if (g->res[a] % 2) { set_error("restriction needs even resolution"); return SMK_ERR_ARG; }
    launch_restrict_cell<T::DIM, T::PER, R>(to_geo(g), N, (const R*)x, (R*)out, ST(stream));
    return cuda_check("smk_restrict_cell");
  });
}

int smk_prolong_cell(const smk_grid* g, int N, const void* x, void* out, int acc, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_prolong_cell<T::DIM, T::PER, R>(to_geo(g), N, (const R*)x, (R*)out, acc, ST(stream));
    return cuda_check("smk_prolong_cell");
  });
}

int smk_restrict_face(const smk_grid* g, int N, const void* const in[], void* const out[], void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    for (int a = 0; a < g->dim; ++a)
      if (g->res[a] % 2) { set_error("restriction needs even resolution"); return SMK_ERR_ARG; }
    launch_restrict_face<T::DIM, T::PER, R>(to_geo(g), N, face3<R>(in, g->dim), facew<R>(out, g->dim), ST(stream));
    return cuda_check("smk_restrict_face");
  });
}

int smk_prolong_face(const smk_grid* g, int N, const void* const in[], void* const out[], int acc, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_prolong_face<T::DIM, T::PER, R>(to_geo(g), N, face3<R>(in, g->dim), facew<R>(out, g->dim), acc,
                                           ST(stream));
    return cuda_check("smk_prolong_face");
  });
}

int smk_poisson_solve(const smk_grid* g, const void* rhs, void* p, double tol, int max_cycles, int* cycles,
                      double* residual, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    return poisson_solve<T::DIM, T::PER, R>(to_geo(g), (const R*)rhs, (R*)p, tol, max_cycles, cycles, residual,
                                            ST(stream));
  });
}

int smk_project(const smk_grid* g, const void* const in[], void* const out[], double tol, int* cycles,
                double* residual, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    return project<T::DIM, T::PER, R>(to_geo(g), face3<R>(in, g->dim), facew<R>(out, g->dim), tol, cycles, residual,
                                      ST(stream));
  });
}

int smk_transport_scalar(const smk_grid* g, int N, const void* const v[], const void* rho, void* out,
                         void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    Ix<T::DIM, T::PER> ix(to_geo(g));
    int64_t n = (int64_t)N * ix.cells();
    k_transport<T::DIM, T::PER, R><<<grid_for(n, 256), 256, 0, ST(stream)>>>(
        ix, (R)(0.5 / g->h), face3<R>(v, g->dim), N, (const R*)rho, (R*)out, R(1), nullptr, nullptr, N); count_launch();
    return cuda_check("smk_transport_scalar");
  });
}

int smk_advect(const smk_grid* g, const void* const v[], const void* rho, void* out, double dt, double tol, int cap,
               int k_fixed, int transpose, int* k_used, double* last_term_norm, void* stream) {
  if (!(dt > 0)) { set_error("dt must be positive"); return SMK_ERR_ARG; }
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    return advect<T::DIM, T::PER, R>(to_geo(g), face3<R>(v, g->dim), (const R*)rho, (R*)out, dt, tol, cap, k_fixed,
                                     transpose, k_used, last_term_norm, ST(stream));
  });
}

int smk_scalar_stencil_v_adjoint(const smk_grid* g, int N, const void* x, const void* y, void* const out[],
                                 void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    Ix<T::DIM, T::PER> ix(to_geo(g));
    dim3 grid(grid_for((int64_t)N * ix.faces(0), 256), T::DIM);
    k_stencil_v_adj<T::DIM, T::PER, R><<<grid, 256, 0, ST(stream)>>>(ix, (R)(0.5 / g->h), (const R*)x, (const R*)y,
                                                                    facew<R>(out, g->dim), N); count_launch();
    return cuda_check("smk_scalar_stencil_v_adjoint");
  });
}

int smk_advect_v_T(const smk_grid* g, const void* const v[], const void* rho, const void* mu, void* const out[],
                   double dt, int k, void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    return advect_v_T<T::DIM, T::PER, R>(to_geo(g), face3<R>(v, g->dim), (const R*)rho, (const R*)mu,
                                         facew<R>(out, g->dim), dt, k, ST(stream));
  });
}

int smk_transport_face(const smk_grid* g, int N, const void* const a[], const void* const w[], void* const out[],
                       void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_face_op<T::DIM, T::PER, R>(to_geo(g), N, face3<R>(a, g->dim), face3<R>(w, g->dim), facew<R>(out, g->dim),
                                      FACE_S, ST(stream));
    return cuda_check("smk_transport_face");
  });
}

int smk_self_adv_jac(const smk_grid* g, int N, const void* const v[], const void* const d[], void* const out[],
                     void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_face_op<T::DIM, T::PER, R>(to_geo(g), N, face3<R>(v, g->dim), face3<R>(d, g->dim), facew<R>(out, g->dim),
                                      FACE_J, ST(stream));
    return cuda_check("smk_self_adv_jac");
  });
}

int smk_self_adv_jac_T(const smk_grid* g, int N, const void* const v[], const void* const u[], void* const out[],
                       void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    launch_face_op<T::DIM, T::PER, R>(to_geo(g), N, face3<R>(v, g->dim), face3<R>(u, g->dim), facew<R>(out, g->dim),
                                      FACE_JT, ST(stream));
    return cuda_check("smk_self_adv_jac_T");
  });
}

int smk_semi_lagrangian(const smk_grid* g, const void* const v[], const void* rho, void* out, double dt,
                        void* stream) {
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    Ix<T::DIM, T::PER> ix(to_geo(g));
    k_semi_lagrangian<T::DIM, T::PER, R><<<grid_for(ix.cells(), 256), 256, 0, ST(stream)>>>(
        ix, (R)g->h, face3<R>(v, g->dim), (const R*)rho, (R)dt, (R*)out); count_launch();
    return cuda_check("smk_semi_lagrangian");
  });
}

int smk_sim_step(const smk_grid* g, const void* const v[], const void* rho, const void* const u[], double dt,
                 int picard_iters, double sim_tol, double trunc_tol, int trunc_cap, void* const v_out[], void* p_out,
                 void* rho_out, int* k_used, double* picard_residual, void* stream) {
  if (!(dt > 0)) { set_error("dt must be positive"); return SMK_ERR_ARG; }
  if (picard_iters < 1) { set_error("picard_iters must be >= 1"); return SMK_ERR_ARG; }
  return dispatch(g, [&](auto tag) {
    using T = decltype(tag); using R = typename T::R;
    return sim_step<T::DIM, T::PER, R>(to_geo(g), face3<R>(v, g->dim), (const R*)rho, face3<R>(u, g->dim), dt,
                                       picard_iters, sim_tol, trunc_tol, trunc_cap, facew<R>(v_out, g->dim),
                                       (R*)p_out, (R*)rho_out, k_used, picard_residual, ST(stream));
  });
}

}  // extern "C"
