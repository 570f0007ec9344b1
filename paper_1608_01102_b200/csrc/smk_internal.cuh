// Declarations shared between the translation units of libsmk.
#pragma once

#include <utility>
#include <vector>

#include "smk_dispatch.cuh"

namespace smk {

// device allocations released together.  Scratch(st) is operator-level
// scratch: its buffers come from a process-wide pool and go back to it on
// release with an event recorded on `st`, so a later call reuses them with no
// cudaMalloc / cudaFree (cudaFree synchronises the whole device): on the same
// stream stream order makes reuse safe, on another stream the taker waits on
// the event.  A default-constructed Scratch (long-lived solver memory) owns
// plain cudaMalloc allocations.
struct Scratch {
  std::vector<std::pair<void*, size_t>> bufs;
  cudaStream_t st = nullptr;
  bool pooled = false;
  Scratch() = default;
  explicit Scratch(cudaStream_t s) : st(s), pooled(true) {}
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  void* get(size_t bytes);
  void release();
  ~Scratch();
};

// free the process-wide operator scratch pool (every device)
void pool_trim();
Geo coarsen(const Geo& g);
Geo refine(const Geo& g);
bool can_coarsen(const Geo& g);
int64_t cells_of(const Geo& g);
int64_t faces_of(const Geo& g, int k);

double host_absmax(int dtype, const void* x, int64_t n, cudaStream_t st, void* dev_scalar);
double host_sum(int dtype, const void* x, const void* y, int64_t n, cudaStream_t st, double* dev_parts);
template <class R>
void frame_sub_mean(R* x, int64_t per, int nframes, cudaStream_t st, double* dev_parts);
template <class R>
void axpby(R* y, const R* x, double a, double b, int64_t n, cudaStream_t st);

enum { OP_S = 0, OP_J = 1, OP_JT = 2 };

// launch accounting (gpu_launches in bench.py): every kernel launch site of
// the library calls count_launch()
void count_launch(int n = 1);
long long launch_count();

template <int DIM, bool PER, class R>
void launch_div(const Geo& g, int N, Face3<R> v, R* out, cudaStream_t st);
template <int DIM, bool PER, class R>
void launch_grad(const Geo& g, int N, const R* p, FaceW<R> out, cudaStream_t st);
template <int DIM, bool PER, class R>
void launch_face_op(const Geo& g, int N, Face3<R> a, Face3<R> w, FaceW<R> out, int op, cudaStream_t st);
template <int DIM, bool PER, class R>
void launch_restrict_cell(const Geo& gf, int N, const R* x, R* out, cudaStream_t st);
template <int DIM, bool PER, class R>
void launch_prolong_cell(const Geo& gc, int N, const R* x, R* out, int acc, cudaStream_t st);
template <int DIM, bool PER, class R>
void launch_restrict_face(const Geo& gf, int N, Face3<R> in, FaceW<R> out, cudaStream_t st);
template <int DIM, bool PER, class R>
void launch_prolong_face(const Geo& gc, int N, Face3<R> in, FaceW<R> out, int acc, cudaStream_t st);

}  // namespace smk
