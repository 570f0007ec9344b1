// Advection-optimisation keyframe metric (pkg/src/smokectrl/ao.py:74-127).
//
// C = sum_j w_j G_j^T G_j with separable per-axis dense filter matrices
// (mirror / wrap folding baked into the matrix, ao.py:55-71).  The host
// composes C x from per-axis passes: y = alpha * op(M) x (+ beta * y), where
// op(M) = M or M^T is applied along the middle axis of x viewed as
// (outer, n, inner).  One thread per output element; a warp runs along the
// contiguous inner axis (every lane reads the same M entry: a broadcast) or,
// for the last axis (inner == 1), along the filtered axis (lanes read one x
// value: a broadcast, M rows through L1).  The sum runs over j ascending in
// the element type, like numpy's tensordot contraction per output.

#include <cuda_runtime.h>

#include "smk.h"
#include "smk_internal.cuh"

namespace smk {
namespace {

template <class R, bool TR, bool ACC>
__global__ void __launch_bounds__(256) k_axis_filter(int64_t total, int n, int64_t inner, const R* __restrict__ M,
                                                     const R* __restrict__ x, R* __restrict__ y, R alpha, R beta) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e % inner;
    const int64_t t = e / inner;
    const int i = (int)(t % n);
    const int64_t a = t / n;
    const R* xs = x + a * n * inner + b;
    R s = R(0);
    if (TR) {
      for (int j = 0; j < n; ++j) s = fma(__ldg(M + (int64_t)j * n + i), __ldg(xs + (int64_t)j * inner), s);
    } else {
      const R* mr = M + (int64_t)i * n;
      for (int j = 0; j < n; ++j) s = fma(__ldg(mr + j), __ldg(xs + (int64_t)j * inner), s);
    }
    y[e] = ACC ? alpha * s + beta * y[e] : alpha * s;
  }
}

template <class R>
void launch_axis_filter(int64_t outer, int n, int64_t inner, const R* M, int tr, double alpha, double beta,
                        const R* x, R* y, cudaStream_t st) {
  const int64_t total = outer * n * inner;
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = (int)(want < 148 * 64 ? want : 148 * 64);
  const bool acc = beta != 0.0;
  count_launch();
  if (tr) {
    if (acc) k_axis_filter<R, true, true><<<blocks, threads, 0, st>>>(total, n, inner, M, x, y, R(alpha), R(beta));
    else k_axis_filter<R, true, false><<<blocks, threads, 0, st>>>(total, n, inner, M, x, y, R(alpha), R(beta));
  } else {
    if (acc) k_axis_filter<R, false, true><<<blocks, threads, 0, st>>>(total, n, inner, M, x, y, R(alpha), R(beta));
    else k_axis_filter<R, false, false><<<blocks, threads, 0, st>>>(total, n, inner, M, x, y, R(alpha), R(beta));
  }
}

}  // namespace
}  // namespace smk

using namespace smk;

extern "C" int smk_axis_filter(int dtype, int64_t outer, int n, int64_t inner, const void* M, int transpose,
                               double alpha, double beta, const void* x, void* y, void* stream) {
  if (dtype != SMK_F64 && dtype != SMK_F32) { set_error("bad dtype"); return SMK_ERR_ARG; }
  if (outer < 0 || n < 1 || inner < 1) { set_error("bad axis_filter extents"); return SMK_ERR_ARG; }
  if (x == y) { set_error("axis_filter cannot run in place"); return SMK_ERR_ARG; }
  if (outer == 0) return SMK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SMK_F64)
    launch_axis_filter<double>(outer, n, inner, (const double*)M, transpose, alpha, beta, (const double*)x,
                               (double*)y, st);
  else
    launch_axis_filter<float>(outer, n, inner, (const float*)M, transpose, alpha, beta, (const float*)x,
                              (float*)y, st);
  return cuda_check("smk_axis_filter");
}
