// Runtime (dtype, dim, boundary) -> template dispatch and C-ABI plumbing.
#pragma once

#include <cstdio>
#include <string>

#include "../../include/smk.h"
#include "smk_common.cuh"

namespace smk {

template <class R_, int D_, bool P_>
struct Tag {
  using R = R_;
  static constexpr int DIM = D_;
  static constexpr bool PER = P_;
};

void set_error(const char* fmt, ...);

inline Geo to_geo(const smk_grid* g) {
  Geo o;
  o.dim = g->dim;
  o.n[0] = g->res[0];
  o.n[1] = g->res[1];
  o.n[2] = g->dim == 3 ? g->res[2] : 1;
  o.h = g->h;
  o.periodic = g->boundary == SMK_PERIODIC;
  return o;
}

inline int check_grid(const smk_grid* g) {
  if (!g) { set_error("null grid"); return SMK_ERR_ARG; }
  if (g->dim != 2 && g->dim != 3) { set_error("dim must be 2 or 3"); return SMK_ERR_ARG; }
  for (int a = 0; a < g->dim; ++a)
    if (g->res[a] < 4) { set_error("res must be >= 4"); return SMK_ERR_ARG; }
  if (!(g->h > 0)) { set_error("h must be positive"); return SMK_ERR_ARG; }
  if (g->boundary != SMK_NEUMANN && g->boundary != SMK_PERIODIC) { set_error("bad boundary"); return SMK_ERR_ARG; }
  if (g->dtype != SMK_F64 && g->dtype != SMK_F32) { set_error("bad dtype"); return SMK_ERR_ARG; }
  return SMK_OK;
}

template <class F>
int dispatch(const smk_grid* g, F&& f) {
  int rc = check_grid(g);
  if (rc) return rc;
  bool per = g->boundary == SMK_PERIODIC;
  if (g->dtype == SMK_F64) {
    if (g->dim == 2) return per ? f(Tag<double, 2, true>{}) : f(Tag<double, 2, false>{});
    return per ? f(Tag<double, 3, true>{}) : f(Tag<double, 3, false>{});
  }
  if (g->dim == 2) return per ? f(Tag<float, 2, true>{}) : f(Tag<float, 2, false>{});
  return per ? f(Tag<float, 3, true>{}) : f(Tag<float, 3, false>{});
}

inline int cuda_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return SMK_ERR_CUDA;
  }
  return SMK_OK;
}

template <class R>
inline Face3<R> face3(const void* const* p, int dim) {
  Face3<R> f;
  for (int k = 0; k < 3; ++k) f.c[k] = (k < dim) ? (const R*)p[k] : nullptr;
  return f;
}

template <class R>
struct FaceW {  // writable face pointers
  R* c[3];
};

template <class R>
inline FaceW<R> facew(void* const* p, int dim) {
  FaceW<R> f;
  for (int k = 0; k < 3; ++k) f.c[k] = (k < dim) ? (R*)p[k] : nullptr;
  return f;
}

}  // namespace smk
