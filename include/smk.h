/*
 * smk.h — C-ABI of the B200 STFAS library (libsmk.so, sm_100a).
 *
 * Drop-in boundary for the reference's operator layer (pure functions on
 * fp64 numpy arrays, pkg/src/smokectrl/fields.py:17-22, advection.py:22-28)
 * and for the STFAS solver the reference specifies but does not ship
 * (SPEC.md:285-374).  Every entry point takes plain C types:
 *
 *   - a grid descriptor (smk_grid), mirroring GridSpec (fields.py:37-89)
 *     plus the element type;
 *   - DEVICE pointers to C-order arrays laid out exactly like the reference's
 *     numpy arrays: a cell field is (nframes, n0, n1[, n2]); face component k
 *     is (nframes, f0, f1[, f2]) with f_a = n_a + (a == k && Neumann)
 *     (fields.py:74-79).  Face fields are passed as arrays of `dim` pointers;
 *   - a CUDA stream (cudaStream_t passed as void*; NULL = legacy stream).
 *
 * Inputs are never mutated unless documented (in-place solver state);
 * outputs are caller-owned.  Results are bitwise deterministic for a given
 * device and launch configuration (no floating-point atomics; colour passes
 * are race-free).
 *
 * Return codes map to the reference exception taxonomy (errors.py:4-56):
 *   SMK_OK, SMK_NONCONVERGENCE (NonConvergence), SMK_TRUNCATION_OVERFLOW
 *   (TruncationOverflow), SMK_SINGULAR_BLOCK (SingularBlock),
 *   SMK_MAX_ITERATIONS (MaxIterations), SMK_ERR_ARG (ValueError),
 *   SMK_ERR_CUDA (CUDA failure).  smk_last_error() returns the message of the
 *   last failure on the calling thread.
 */
#ifndef SMK_H
#define SMK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMK_OK 0
#define SMK_NONCONVERGENCE 1
#define SMK_TRUNCATION_OVERFLOW 2
#define SMK_SINGULAR_BLOCK 3
#define SMK_MAX_ITERATIONS 4
#define SMK_ERR_ARG (-1)
#define SMK_ERR_CUDA (-2)

#define SMK_NEUMANN 0
#define SMK_PERIODIC 1

#define SMK_F64 0
#define SMK_F32 1

/* GridSpec (fields.py:37-89) + element type. res[2] ignored when dim == 2. */
typedef struct smk_grid {
  int dim;
  int res[3];
  double h;
  int boundary; /* SMK_NEUMANN | SMK_PERIODIC */
  int dtype;    /* SMK_F64 | SMK_F32 */
} smk_grid;

const char* smk_last_error(void);
int smk_version(void);
/* number of kernels the library has launched in this process (accounting) */
long long smk_launch_count(void);
/* release the operator scratch pool (stream-ordered buffers the raw operators
 * reuse across calls, keyed by device, <= 4 GiB pooled per device) */
void smk_pool_trim(void);

/* ---------------- field core (fields.py) ---------------- */

/* divergence_arrays, fields.py:163-178 */
int smk_div(const smk_grid* g, int nframes, const void* const comps[], void* out, void* stream);
/* gradient_arrays, fields.py:181-201 */
int smk_grad(const smk_grid* g, int nframes, const void* p, void* const out[], void* stream);
/* zero_boundary_faces, fields.py:145-160 (in place) */
int smk_zero_walls(const smk_grid* g, int nframes, void* const comps[], void* stream);
/* _laplacian, fields.py:223-225 */
int smk_laplacian(const smk_grid* g, int nframes, const void* p, void* out, void* stream);
/* inf_norm / dot_fields, fields.py:204-216 (synchronising; n = element count) */
int smk_inf_norm(int dtype, const void* x, int64_t n, double* out, void* stream);
int smk_dot(int dtype, const void* x, const void* y, int64_t n, double* out, void* stream);
/* restrict_cell / prolong_cell, fields.py:243-284.  `g` is the FINE grid for
 * restriction and the COARSE grid for prolongation; accumulate != 0 adds into
 * `out` instead of overwriting. */
int smk_restrict_cell(const smk_grid* fine, int nframes, const void* x, void* out, void* stream);
int smk_prolong_cell(const smk_grid* coarse, int nframes, const void* x, void* out, int accumulate, void* stream);
/* STFAS face transfers */
int smk_restrict_face(const smk_grid* fine, int nframes, const void* const in[], void* const out[], void* stream);
int smk_prolong_face(const smk_grid* coarse, int nframes, const void* const in[], void* const out[], int accumulate, void* stream);
/* solve_poisson, fields.py:330-347: V(2,2) damped Jacobi + dense pinv on the
 * coarsest level; `p` receives the solution; returns SMK_NONCONVERGENCE when
 * the budget is exhausted (residual in *residual). */
int smk_poisson_solve(const smk_grid* g, const void* rhs, void* p, double tol, int max_cycles,
                      int* cycles, double* residual, void* stream);
/* project_arrays, fields.py:350-358 */
int smk_project(const smk_grid* g, const void* const in[], void* const out[], double tol,
                int* cycles, double* residual, void* stream);

/* ---------------- transport (advection.py) ---------------- */

/* transport_scalar, advection.py:88-97 (batch over frames) */
int smk_transport_scalar(const smk_grid* g, int nframes, const void* const v[], const void* rho, void* out,
                         void* stream);
/* advect_scalar / advect_scalar_rho_T, advection.py:144-174: truncated
 * exp(+-T(v) dt) rho.  k_fixed <= 0 selects the adaptive order. */
int smk_advect(const smk_grid* g, const void* const v[], const void* rho, void* out, double dt, double tol,
               int cap, int k_fixed, int transpose, int* k_used, double* last_term_norm, void* stream);
/* scalar_stencil_v_adjoint, advection.py:105-130 */
int smk_scalar_stencil_v_adjoint(const smk_grid* g, int nframes, const void* x, const void* y, void* const out[],
                                 void* stream);
/* advect_scalar_v_T, advection.py:177-210 (order k from the forward pass) */
int smk_advect_v_T(const smk_grid* g, const void* const v[], const void* rho, const void* mu, void* const out[],
                   double dt, int k, void* stream);
/* transport_face S(a, w), advection.py:353-365 */
int smk_transport_face(const smk_grid* g, int nframes, const void* const a[], const void* const w[],
                       void* const out[], void* stream);
/* self_adv_jacobian_apply, advection.py:373-377 */
int smk_self_adv_jac(const smk_grid* g, int nframes, const void* const v[], const void* const d[],
                     void* const out[], void* stream);
/* self_adv_jacobian_T_apply, advection.py:437-441 */
int smk_self_adv_jac_T(const smk_grid* g, int nframes, const void* const v[], const void* const u[],
                       void* const out[], void* stream);
/* semi_lagrangian, advection.py:264-299 (comparator) */
int smk_semi_lagrangian(const smk_grid* g, const void* const v[], const void* rho, void* out, double dt,
                        void* stream);

/* ---------------- forward step (simulator.py) ---------------- */

/* simulator.step, simulator.py:73-110.  Returns SMK_NONCONVERGENCE when the
 * Picard update stalls above sim_tol (outputs are still written, as the
 * reference attaches the completed state to the exception). */
int smk_sim_step(const smk_grid* g, const void* const v[], const void* rho, const void* const u[], double dt,
                 int picard_iters, double sim_tol, double trunc_tol, int trunc_cap, void* const v_out[],
                 void* p_out, void* rho_out, int* k_used, double* picard_residual, void* stream);

/* ---------------- STFAS / NSO ---------------- */

typedef struct smk_nso_params {
  int n_frames;   /* N */
  int n_levels;   /* spatial levels (>=1; clipped to what the grid allows) */
  double dt;
  double K;
  double r;
  double omega;   /* smoother damping (default 0.8) */
  int nu1, nu2;   /* pre/post sweeps (2, 2) */
  int n_coarse;   /* coarsest sweeps (10) */
  int color_mod;  /* colouring modulus per axis (2: 4/8 colours) */
  int t0;         /* time-slab mode: global index of local pair 0 (0 otherwise) */
  int n_total;    /* time-slab mode: global pair count (0 = n_frames) */
  int red_black;  /* != 0: 2 colours by (sum_k c_k) mod 2 (color_mod ignored);
                     needs an even last-axis extent (periodic: even extents) */
} smk_nso_params;

/* Spacetime state (pair index i = 0..N-1): V[i]=v_{i+1}, PB[i]=pbar_{i+1},
 * U[i]=u_i, P[i]=p_{i+1}; every array has N frames.  Neumann wall faces are
 * not unknowns and must hold zero (zero_boundary_faces, fields.py:145-160);
 * the solver never writes them. */
typedef struct smk_state {
  void* V[3];
  void* PB;
  void* U[3];
  void* P;
} smk_state;

/* Residual blocks of Eq. 8 (same layout as the state). */
typedef struct smk_residual {
  void* R1[3];
  void* R2;
  void* R3[3];
  void* R4;
} smk_residual;

/* kkt_residual: out = f(state) - rhs (rhs may be NULL).
 * v0: pinned initial velocity (1 frame); vstar: v*_0..v*_{N-1} (N frames). */
int smk_kkt_residual(const smk_grid* g, const smk_nso_params* prm, const smk_state* s, const void* const v0[],
                     const void* const vstar[], const smk_residual* rhs, const smk_residual* out, void* stream);
/* One coloured SCGS sweep, in place. */
int smk_scgs_sweep(const smk_grid* g, const smk_nso_params* prm, const smk_state* s, const void* const v0[],
                   const void* const vstar[], const smk_residual* rhs, void* stream);

typedef struct smk_nso smk_nso; /* opaque hierarchy (StfasHierarchy) */

smk_nso* smk_nso_create(const smk_grid* g, const smk_nso_params* prm);
void smk_nso_destroy(smk_nso* h);
int smk_nso_levels(const smk_nso* h);
/* device bytes owned by the hierarchy (memtrack equivalent, memtrack.py:19-59) */
int64_t smk_nso_device_bytes(const smk_nso* h);
/* field-payload values owned by the hierarchy (coarse-level states, FAS rhs,
 * residuals, guides; not the smoother's hand-off / delta scratch) --
 * memtrack.py:1-9's accounting, for SPEC.md:529's memory bound */
int64_t smk_nso_payload_values(const smk_nso* h);
/* Bind the (device) v0 / vstar of the top level; restricts them down the
 * hierarchy.  Must be called before vcycle/solve and again when they change. */
int smk_nso_set_guide(smk_nso* h, const void* const v0[], const void* const vstar[], void* stream);
/* Update K on an existing hierarchy (the LM proximal shift);
 * the next V-cycle re-captures its graph. */
int smk_nso_set_K(smk_nso* h, double K);
/* One FAS V(nu1, nu2) cycle (PAPER Alg. 2) on the caller's top-level state. */
int smk_nso_vcycle(smk_nso* h, const smk_state* s, void* stream);
/* ||f||_inf and ||f||_2 of the top level (synchronising). */
int smk_nso_residual_norms(smk_nso* h, const smk_state* s, double* res_inf, double* res_l2, void* stream);
/* Bracket every colour-pass and residual kernel launch with CUDA events on
 * the launching stream (enable != 0 also resets the record).  profile_read
 * returns, for kernel kind 0 (k_scgs_fwd, forward elimination), 1
 * (k_scgs_apply), 2 (k_kkt, residual) or 3 (k_scgs_back, back substitution),
 * the summed kernel time, the launch count and the cell-timesteps processed
 * (colour cells x frames; all cells x frames for the residual), over all
 * levels; profile_read_level restricts it to one hierarchy level. */
int smk_nso_profile(smk_nso* h, int enable);
int smk_nso_profile_read(smk_nso* h, int kind, double* ms, long long* launches, long long* cell_timesteps);
int smk_nso_profile_read_level(smk_nso* h, int kind, int level, double* ms, long long* launches,
                               long long* cell_timesteps);
/* Subtract per-frame means of p and pbar (gauge). */
int smk_nso_gauge_fix(smk_nso* h, const smk_state* s, void* stream);
/* solve_nso: V-cycles until ||f||_inf <= eps (or
 * eps * ||f_0||_inf when relative != 0).  hist (optional, 2*(budget+1)
 * doubles) receives (res_inf, res_l2) per cycle.  Returns
 * SMK_NONCONVERGENCE if the budget is exhausted. */
int smk_nso_solve(smk_nso* h, const smk_state* s, double eps, int relative, int cycle_budget, int* cycles,
                  double* hist, void* stream);

/* ---- time-slab (multi-GPU) per-level operations ----
 * The caller owns the level's state (n_frames local pairs) and passes the
 * slab halos explicitly: vprev = v at the frame before local pair 0 (the left
 * neighbour's last V frame, or the pinned v0 on the first slab), unext = the
 * right neighbour's first U frame (NULL on the last slab), vs = the level's
 * guide with n_frames + 1 frames (v*_{t0} .. v*_{t0+n_frames}).  The smoother's
 * time line is cut at the slab boundary (neighbour frames frozen). */
int smk_nso_n_colors(const smk_nso* h);
int smk_nso_level_residual(smk_nso* h, int level, const smk_state* s, const void* const vprev[],
                           const void* const unext[], const void* const vs[], const smk_residual* rhs,
                           const smk_residual* out, void* stream);
int smk_nso_level_color_pass(smk_nso* h, int level, int colour, const smk_state* s, const void* const vprev[],
                             const void* const unext[], const void* const vs[], const smk_residual* rhs,
                             void* stream);
/* ---- time slabs in C++ (DESIGN.md §6): the whole slab V-cycle without host
 * code per colour pass (replaces the per-level Python orchestration above on
 * the product path; slabs.py CSlabSolver).  This process holds the
 * contiguous slabs [first, first + n_local) of n_slabs (split_frames order:
 * the first n_frames % n_slabs slabs one pair longer); prm->n_frames is the
 * GLOBAL pair count.  Halos are refreshed before every residual and colour
 * pass: local neighbours by device copies, the slabs of ranks rank - 1 /
 * rank + 1 by NCCL send / recv (world > 1: nccl_id = the 128-byte
 * ncclUniqueId of rank 0, from smk_nccl_unique_id, broadcast by the caller).
 * The V-cycle (kernels, copies, NCCL P2P) is captured into one CUDA graph.
 * states[k] holds local slab k's pairs (smk_slabs_frames). */
typedef struct smk_slabs smk_slabs;
int smk_nccl_unique_id(void* out, int nbytes);
smk_slabs* smk_slabs_create(const smk_grid* g, const smk_nso_params* prm, int first, int n_local, int n_slabs,
                            int rank, int world, const void* nccl_id);
void smk_slabs_destroy(smk_slabs* h);
int smk_slabs_levels(const smk_slabs* h);
int64_t smk_slabs_device_bytes(const smk_slabs* h);
int smk_slabs_frames(const smk_slabs* h, int local, int* t0, int* n_frames);
/* v0: pinned initial velocity (1 frame); vstar: the full guide v*_0..v*_{N-1} */
int smk_slabs_set_guide(smk_slabs* h, const void* const v0[], const void* const vstar[], void* stream);
int smk_slabs_vcycle(smk_slabs* h, const smk_state* states, void* stream);
int smk_slabs_gauge_fix(smk_slabs* h, const smk_state* states, void* stream);
/* ||f||_inf / ||f||_2 over every slab of every rank (synchronising) */
int smk_slabs_residual_norms(smk_slabs* h, const smk_state* states, double* res_inf, double* res_l2, void* stream);
/* smk_nso_profile / _read_level summed over the local slabs (level < 0: all) */
int smk_slabs_profile(smk_slabs* h, int enable);
int smk_slabs_profile_read_level(smk_slabs* h, int kind, int level, double* ms, long long* launches,
                                 long long* cell_timesteps);

/* ---------------- advection optimisation (ao.py) ---------------- */

/* One separable pass of the keyframe metric (GaussianMetric._filter,
 * ao.py:100-104): x viewed as (outer, n, inner), y = alpha * op(M) x along
 * the middle axis + beta * y (y not read when beta == 0), op(M) = M (n x n,
 * C order) or M^T when transpose != 0.  GaussianMetric.apply / quad
 * (ao.py:106-120) are 2*dim such passes per pyramid level.  x != y. */
int smk_axis_filter(int dtype, int64_t outer, int n, int64_t inner, const void* M, int transpose, double alpha,
                    double beta, const void* x, void* y, void* stream);
/* y = a * x + b * y over n elements (state algebra of the slab V-cycle) */
int smk_axpby(int dtype, void* y, const void* x, double a, double b, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SMK_H */
