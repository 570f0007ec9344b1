/*
 * cstfas.c -- fp64 scalar C restatement of the STFAS oracle
 * (TEST INFRASTRUCTURE AND CPU BASELINE ONLY; never on the product path).
 *
 * The same algorithm as oracle/stfas.py (PAPER Eq. 8/9,
 * Alg. 2, frozen in DESIGN.md §3), restated point by point so that it runs at
 * the BASELINE configs' real sizes on the host cores (OpenMP over the cells
 * of a colour / the points of a frame):
 *
 *   - the reference's raw operators, evaluated per point:
 *       div / grad            fields.py:163-201   (oracle/ops.py div, grad)
 *       transport_face S(a,w) advection.py:306-365 (oracle/ops.py adv_samples,
 *                                                    transport_face)
 *       J_Adv(v)^T u          advection.py:380-441 (oracle/ops.py
 *                                                    _samples_adjoint, jac_T_apply)
 *       restrict/prolong cell fields.py:243-284    (oracle/ops.py)
 *       face R/P              DESIGN.md §3.6       (oracle/ops.py restrict_face,
 *                                                    prolong_face)
 *   - kkt_residual (oracle/stfas.py kkt_residual);
 *   - the local Jacobian by unit-vector probing of J_Adv(v) d = S(v,d)+S(d,v)
 *     (oracle/stfas.py local_jacobian) -- NOT the GPU's closed form;
 *   - assemble_line + block_thomas with partially pivoted dense block solves
 *     on the full 2N-block (u, v) time line (oracle/stfas.py) -- NOT the GPU's
 *     Schur / LDL^T elimination;
 *   - scgs_color (snapshot reads, x += omega dx), FAS V-cycle, gauge fix,
 *     solve_nso (oracle/stfas.py vcycle / gauge_fix / solve_nso).
 *
 * Pinned to oracle/stfas.py by tests/test_coracle.py (which is itself pinned
 * to the reference's golden vectors and SPEC's known-answer tests).  Array
 * layout = the reference's numpy layout: C order, frame-major stacks, face
 * component k has extent res[a] + (a == k && Neumann) along axis a.  2D grids
 * are handled as res[2] = 1.  Compile with -ffp-contract=off (numpy rounds
 * every product).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int dim;
  int n[3];
  double h;
  int per;
} cgrid;

typedef struct {
  double* V[3];
  double* PB;
  double* U[3];
  double* P;
} cstate;

typedef struct {
  double* R1[3];
  double* R2;
  double* R3[3];
  double* R4;
} cres;

/* problem of one level (oracle/stfas.py Problem) */
typedef struct {
  cgrid g;
  int N;          /* local pairs */
  double dt, K, r, omega;
  int colors;     /* colouring modulus */
  int t0, Ng;     /* slab: global index of pair 0, global pair count */
  const double* v0[3];     /* 1 frame */
  const double* vstar[3];  /* vs_frames frames */
  int vs_frames;           /* N (v*_0..v*_{N-1}) or N+1 (slab mode) */
  const double* unext[3];  /* right halo (1 frame) or NULL */
  int red_black;           /* 2 colours by parity of sum_k c_k (else mod-`colors`) */
} cprob;

/* ------------------------------------------------------------------ grid */

static inline int ext(const cgrid* g, int k, int a) { /* k = -1: cells */
  if (a >= g->dim) return 1;
  return g->n[a] + ((!g->per && a == k) ? 1 : 0);
}
static inline int64_t fsize(const cgrid* g, int k) {
  return (int64_t)ext(g, k, 0) * ext(g, k, 1) * ext(g, k, 2);
}
static inline int64_t csize(const cgrid* g) { return (int64_t)g->n[0] * (g->dim > 1 ? g->n[1] : 1) * (g->dim > 2 ? g->n[2] : 1); }
/* normalise coordinates on lattice k (wrap / range check); 0 = outside */
static inline int lnorm(const cgrid* g, int k, int* x) {
  for (int a = 0; a < g->dim; ++a) {
    int e = ext(g, k, a);
    if (g->per) {
      x[a] = ((x[a] % e) + e) % e;
    } else if (x[a] < 0 || x[a] >= e) {
      return 0;
    }
  }
  return 1;
}
static inline int64_t lidx(const cgrid* g, int k, const int* x) {
  return ((int64_t)x[0] * ext(g, k, 1) + (g->dim > 1 ? x[1] : 0)) * ext(g, k, 2) + (g->dim > 2 ? x[2] : 0);
}

/* face field of one frame; unit mode = the unit vector e at (uk, uf) */
typedef struct {
  const double* c[3];
  int unit, uk, uf[3];
} ffield;

static inline double fget(const cgrid* g, const ffield* F, int k, int x0, int x1, int x2) {
  int x[3] = {x0, x1, x2};
  if (!lnorm(g, k, x)) return 0.0;
  if (F->unit) {
    if (k != F->uk) return 0.0;
    for (int a = 0; a < g->dim; ++a)
      if (x[a] != F->uf[a]) return 0.0;
    return 1.0;
  }
  return F->c[k][lidx(g, k, x)];
}
static inline double cget(const cgrid* g, const double* p, int x0, int x1, int x2) {
  int x[3] = {x0, x1, x2};
  if (!lnorm(g, -1, x)) return 0.0;
  return p[lidx(g, -1, x)];
}
static inline int on_wall(const cgrid* g, int k, const int* f) {
  return !g->per && (f[k] == 0 || f[k] == g->n[k]);
}
#define OFF(x, a, d) ((a) == 0 ? (x)[0] + (d) : (x)[0]), ((a) == 1 ? (x)[1] + (d) : (x)[1]), ((a) == 2 ? (x)[2] + (d) : (x)[2])

/* ------------------------------------------- transport_face (S(a, w)) */

/* centre average of a_j at cell c (zero outside, Neumann) -- adv_samples k==j */
static inline double ccj(const cgrid* g, const ffield* A, int j, const int* c) {
  int x[3] = {c[0], c[1], c[2]};
  if (!g->per && (x[j] < 0 || x[j] >= g->n[j])) return 0.0;
  double lo = fget(g, A, j, x[0], x[1], x[2]);
  double hi = fget(g, A, j, OFF(x, j, 1));
  return 0.5 * (lo + hi);
}
/* corner sample of a_k on the j-face lattice (k != j) at index f (k-extent n_k+1) */
static inline double corner(const cgrid* g, const ffield* A, int j, int k, const int* f) {
  double a0 = fget(g, A, k, f[0], f[1], f[2]);
  double a1 = fget(g, A, k, OFF(f, j, -1));
  return 0.5 * (a0 + a1);
}
/* S(a, w)_j at j-face f, wall-masked (advection.py:353-365) */
static double sface(const cgrid* g, const ffield* A, const ffield* W, int j, const int* f) {
  if (on_wall(g, j, f)) return 0.0;
  const double c0 = 0.5 / g->h;
  double acc = 0.0;
  for (int k = 0; k < g->dim; ++k) {
    double sp, sm;
    if (k == j) {
      int cm[3] = {f[0], f[1], f[2]};
      cm[j] -= 1;
      sp = ccj(g, A, j, f);
      sm = ccj(g, A, j, cm);
    } else {
      int fp[3] = {f[0], f[1], f[2]};
      fp[k] += 1;
      if (g->per) fp[k] %= g->n[k];
      sp = corner(g, A, j, k, fp);
      sm = corner(g, A, j, k, f);
    }
    double wp = fget(g, W, j, OFF(f, k, 1));
    double wm = fget(g, W, j, OFF(f, k, -1));
    double t = c0 * (sp * wp - sm * wm);
    acc = (k == 0) ? 0.0 + t : acc + t;
  }
  return acc;
}

/* _samples_adjoint(v, u) at m-face f, wall-masked (advection.py:380-434) */
static double sadj(const cgrid* g, const ffield* Vf, const ffield* Uf, int m, const int* f) {
  if (on_wall(g, m, f)) return 0.0;
  const double c0 = 0.5 / g->h;
  double out = 0.0;
  for (int j = 0; j < g->dim; ++j) {
    double term;
    if (j == m) {
      /* gam[c] = c0 (u_m[c] v_m[c+1] - u_m[c+1] v_m[c]) on cells along m */
      double gm[2];
      for (int s = 0; s < 2; ++s) {
        int c[3] = {f[0], f[1], f[2]};
        c[m] -= s; /* s = 0: gam[f], s = 1: gam[f-1] */
        if (!g->per && (c[m] < 0 || c[m] >= g->n[m])) {
          gm[s] = 0.0;
          continue;
        }
        double u0 = fget(g, Uf, m, c[0], c[1], c[2]), v1 = fget(g, Vf, m, OFF(c, m, 1));
        double u1 = fget(g, Uf, m, OFF(c, m, 1)), v0 = fget(g, Vf, m, c[0], c[1], c[2]);
        gm[s] = c0 * (u0 * v1 - u1 * v0);
      }
      term = 0.5 * (gm[0] + gm[1]);
    } else {
      /* term (j, k = m): gam on the j-face lattice (m-extent n_m + 1),
         gam[x] = c0 (u_j[x-e_m] v_j[x] - u_j[x] v_j[x-e_m]) interior in m */
      double gm[2];
      for (int s = 0; s < 2; ++s) {
        int x[3] = {f[0], f[1], f[2]};
        x[j] += s; /* s = 0: gam[f], s = 1: gam[f+e_j] */
        if (g->per) {
          x[j] %= g->n[j];
        } else if (x[m] <= 0 || x[m] >= g->n[m]) {
          gm[s] = 0.0;
          continue;
        }
        double ua = fget(g, Uf, j, OFF(x, m, -1)), vb = fget(g, Vf, j, x[0], x[1], x[2]);
        double ub = fget(g, Uf, j, x[0], x[1], x[2]), va = fget(g, Vf, j, OFF(x, m, -1));
        gm[s] = c0 * (ua * vb - ub * va);
      }
      term = 0.5 * (gm[0] + gm[1]);
    }
    out = (j == 0) ? 0.0 + term : out + term;
  }
  return out;
}

/* grad p at k-face f (fields.py:181-201) */
static inline double gradf(const cgrid* g, const double* p, int k, const int* f) {
  if (!g->per && (f[k] == 0 || f[k] == g->n[k])) return 0.0;
  return (cget(g, p, f[0], f[1], f[2]) - cget(g, p, OFF(f, k, -1))) / g->h;
}
/* div at cell c (fields.py:163-178) */
static inline double divc(const cgrid* g, const ffield* F, const int* c) {
  double out = 0.0;
  for (int k = 0; k < g->dim; ++k) {
    double hi = fget(g, F, k, OFF(c, k, 1)), lo = fget(g, F, k, c[0], c[1], c[2]);
    double t = (hi - lo) / g->h;
    out = (k == 0) ? 0.0 + t : out + t;
  }
  return out;
}

/* ------------------------------------------------------ KKT residual rows */

static inline void frame_ff(const cgrid* g, double* const base[3], int fr, ffield* F) {
  memset(F, 0, sizeof(*F));
  for (int k = 0; k < g->dim; ++k) F->c[k] = base[k] + (int64_t)fr * fsize(g, k);
}
static inline void cframe_ff(const cgrid* g, const double* const base[3], int fr, ffield* F) {
  memset(F, 0, sizeof(*F));
  for (int k = 0; k < g->dim; ++k) F->c[k] = base[k] ? base[k] + (int64_t)fr * fsize(g, k) : NULL;
}

/* R3 / R1 rows of pair i at k-face f (masked), oracle/stfas.py kkt_residual */
static void face_rows(const cprob* pb, const cstate* st, int i, int k, const int* f, double* r3, double* r1) {
  const cgrid* g = &pb->g;
  if (on_wall(g, k, f)) {
    *r3 = 0.0;
    *r1 = 0.0;
    return;
  }
  ffield Vi, Ui, Vp;
  frame_ff(g, st->V, i, &Vi);
  frame_ff(g, st->U, i, &Ui);
  if (i == 0)
    cframe_ff(g, pb->v0, 0, &Vp);
  else
    frame_ff(g, st->V, i - 1, &Vp);
  const int64_t o = lidx(g, k, f);
  const double v = Vi.c[k][o], vp = Vp.c[k][o], u = Ui.c[k][o];
  const double a = sface(g, &Vi, &Vi, k, f);
  const double q = gradf(g, st->P + (int64_t)i * csize(g), k, f);
  *r3 = (((v - vp) / pb->dt + a) - u) + q;
  /* R1 = kmask (kr (v - s) - un/dt) + u/dt + J^T u + grad pbar */
  const double kmask = (pb->t0 + i < pb->Ng - 1) ? 1.0 : 0.0;
  double s = 0.0, un = 0.0;
  if (pb->vs_frames == pb->N + 1)
    s = pb->vstar[k][(int64_t)(i + 1) * fsize(g, k) + o];
  else if (i + 1 < pb->N)
    s = pb->vstar[k][(int64_t)(i + 1) * fsize(g, k) + o];
  if (i + 1 < pb->N)
    un = st->U[k][(int64_t)(i + 1) * fsize(g, k) + o];
  else if (pb->unext[0])
    un = pb->unext[k][o];
  const double kr = pb->K / pb->r;
  const double jt = sadj(g, &Vi, &Ui, k, f) - sface(g, &Vi, &Ui, k, f);
  const double qb = gradf(g, st->PB + (int64_t)i * csize(g), k, f);
  *r1 = ((kmask * (kr * (v - s) - un / pb->dt) + u / pb->dt) + jt) + qb;
}
static void cell_rows(const cprob* pb, const cstate* st, int i, const int* c, double* r4, double* r2) {
  const cgrid* g = &pb->g;
  ffield Vi, Ui;
  frame_ff(g, st->V, i, &Vi);
  frame_ff(g, st->U, i, &Ui);
  *r4 = divc(g, &Ui, c);
  *r2 = divc(g, &Vi, c);
}

static void lat_coords(const cgrid* g, int k, int64_t e, int* x) {
  int e2 = ext(g, k, 2), e1 = ext(g, k, 1);
  x[2] = (int)(e % e2);
  e /= e2;
  x[1] = (int)(e % e1);
  x[0] = (int)(e / e1);
}

/* full residual f(state) - rhs (rhs may be NULL) */
void cst_kkt_residual(const cprob* pb, const cstate* st, const cres* rhs, const cres* out) {
  const cgrid* g = &pb->g;
  const int N = pb->N;
  for (int k = 0; k < g->dim; ++k) {
    const int64_t nf = fsize(g, k);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)N * nf; ++t) {
      int i = (int)(t / nf);
      int x[3];
      lat_coords(g, k, t % nf, x);
      double r3, r1;
      face_rows(pb, st, i, k, x, &r3, &r1);
      if (rhs) {
        r3 = r3 - rhs->R3[k][t];
        r1 = r1 - rhs->R1[k][t];
      }
      out->R3[k][t] = r3;
      out->R1[k][t] = r1;
    }
  }
  const int64_t nc = csize(g);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)N * nc; ++t) {
    int i = (int)(t / nc);
    int x[3];
    lat_coords(g, -1, t % nc, x);
    double r4, r2;
    cell_rows(pb, st, i, x, &r4, &r2);
    if (rhs) {
      r4 = r4 - rhs->R4[t];
      r2 = r2 - rhs->R2[t];
    }
    out->R4[t] = r4;
    out->R2[t] = r2;
  }
}

/* ---------------------------------------------------- dense block algebra */

#define BMAX 7
#define CMAX (BMAX + 1)

/* S X = R, b x b with nc right-hand sides, partial pivoting (LAPACK gesv
   semantics: pivot = largest |.| in the column, first on ties) */
static int solve_pivot(int b, double* S, int nc, double* X) {
  int ok = 1;
  for (int col = 0; col < b; ++col) {
    int p = col;
    double best = fabs(S[col * b + col]);
    for (int r = col + 1; r < b; ++r)
      if (fabs(S[r * b + col]) > best) {
        best = fabs(S[r * b + col]);
        p = r;
      }
    if (p != col) {
      for (int c = 0; c < b; ++c) {
        double t = S[col * b + c];
        S[col * b + c] = S[p * b + c];
        S[p * b + c] = t;
      }
      for (int c = 0; c < nc; ++c) {
        double t = X[col * nc + c];
        X[col * nc + c] = X[p * nc + c];
        X[p * nc + c] = t;
      }
    }
    double piv = S[col * b + col];
    if (!(fabs(piv) > 0.0)) {
      ok = 0;
      piv = 1e-300;
    }
    for (int r = col + 1; r < b; ++r) {
      double fct = S[r * b + col] / piv;
      for (int c = col + 1; c < b; ++c) S[r * b + c] -= fct * S[col * b + c];
      for (int c = 0; c < nc; ++c) X[r * nc + c] -= fct * X[col * nc + c];
    }
  }
  for (int r = b - 1; r >= 0; --r) {
    for (int c = 0; c < nc; ++c) {
      double s = X[r * nc + c];
      for (int q = r + 1; q < b; ++q) s -= S[r * b + q] * X[q * nc + c];
      X[r * nc + c] = s / S[r * b + r];
    }
  }
  return ok;
}

/* per-thread scratch of one cell's time line */
typedef struct {
  double* D;  /* [nb][b][b] */
  double* L;
  double* Up;
  double* y;  /* [nb][b] */
  double* W;  /* [nb][b][b] */
  double* z;  /* [nb][b] */
} line_ws;

/* the cell's own face slots: q = 2k + s */
typedef struct {
  int c[3];
  int fk[6];
  int f[6][3];
  int wall[6];
  double gcol[6];
} cslots;

static void cell_slots(const cgrid* g, const int* c, cslots* s) {
  memset(s, 0, sizeof(*s));
  for (int a = 0; a < 3; ++a) s->c[a] = c[a];
  for (int k = 0; k < g->dim; ++k)
    for (int sd = 0; sd < 2; ++sd) {
      int q = 2 * k + sd;
      s->fk[q] = k;
      for (int a = 0; a < 3; ++a) s->f[q][a] = c[a];
      s->f[q][k] += sd;
      if (g->per) {
        s->f[q][k] %= g->n[k];
        s->wall[q] = 0;
      } else {
        s->wall[q] = sd == 0 ? c[k] == 0 : c[k] == g->n[k] - 1;
      }
      s->gcol[q] = s->wall[q] ? 0.0 : (sd == 0 ? 1.0 : -1.0) / g->h;
    }
}

/* local Jacobian J[qr][qc] = (S(v, e_qc) + S(e_qc, v))_{qr}
   (oracle/stfas.py local_jacobian: unit-vector probing of jac_apply) */
static void local_jac(const cgrid* g, const ffield* Vi, const cslots* s, double J[6][6]) {
  const int nf = 2 * g->dim;
  for (int qr = 0; qr < nf; ++qr)
    for (int qc = 0; qc < nf; ++qc) J[qr][qc] = 0.0;
  for (int qc = 0; qc < nf; ++qc) {
    if (s->wall[qc]) continue;
    ffield E;
    memset(&E, 0, sizeof(E));
    E.unit = 1;
    E.uk = s->fk[qc];
    for (int a = 0; a < 3; ++a) E.uf[a] = s->f[qc][a];
    for (int qr = 0; qr < nf; ++qr) {
      if (s->wall[qr]) continue;
      double a = sface(g, Vi, &E, s->fk[qr], s->f[qr]);
      double b = sface(g, &E, Vi, s->fk[qr], s->f[qr]);
      J[qr][qc] = a + b;
    }
  }
}

/* one cell's time-line solve; x (nb x b) = the line's correction */
static int cell_line(const cprob* pb, const cstate* st, const cres* rhs, const cslots* s, line_ws* w) {
  const cgrid* g = &pb->g;
  const int N = pb->N, nf = 2 * g->dim, b = nf + 1, nb = 2 * N;
  const double dt = pb->dt;
  const int64_t nc = csize(g);
  const int64_t co = lidx(g, -1, s->c);
  memset(w->D, 0, sizeof(double) * nb * b * b);
  memset(w->L, 0, sizeof(double) * nb * b * b);
  memset(w->Up, 0, sizeof(double) * nb * b * b);
  for (int i = 0; i < N; ++i) {
    /* rhs rows -(f - rhs) */
    double* yu = w->y + (2 * i) * b;
    double* yv = w->y + (2 * i + 1) * b;
    for (int q = 0; q < nf; ++q) {
      double r3, r1;
      face_rows(pb, st, i, s->fk[q], s->f[q], &r3, &r1);
      if (rhs) {
        int64_t o = (int64_t)i * fsize(g, s->fk[q]) + lidx(g, s->fk[q], s->f[q]);
        r3 = r3 - rhs->R3[s->fk[q]][o];
        r1 = r1 - rhs->R1[s->fk[q]][o];
      }
      yu[q] = s->wall[q] ? 0.0 : -r3;
      yv[q] = s->wall[q] ? 0.0 : -r1;
    }
    double r4, r2;
    cell_rows(pb, st, i, s->c, &r4, &r2);
    if (rhs) {
      r4 = r4 - rhs->R4[(int64_t)i * nc + co];
      r2 = r2 - rhs->R2[(int64_t)i * nc + co];
    }
    yu[nf] = -r4;
    yv[nf] = -r2;
    /* blocks (assemble_line) */
    ffield Vi;
    frame_ff(g, st->V, i, &Vi);
    double J[6][6];
    local_jac(g, &Vi, s, J);
    const int bu = 2 * i, bv = 2 * i + 1;
    double* Du = w->D + (int64_t)bu * b * b;
    double* Dv = w->D + (int64_t)bv * b * b;
    const double alpha = (pb->t0 + i < pb->Ng - 1) ? pb->K / pb->r : 0.0;
    for (int r = 0; r < nf; ++r) {
      const double er = s->wall[r] ? 0.0 : 1.0;
      Du[r * b + r] = -er;
      Du[r * b + nf] = s->gcol[r];
      Du[nf * b + r] = -s->gcol[r];
      Dv[r * b + r] = alpha * er;
      Dv[r * b + nf] = s->gcol[r];
      Dv[nf * b + r] = -s->gcol[r];
      for (int c = 0; c < nf; ++c) {
        const double e = (r == c && !s->wall[r]) ? 1.0 : 0.0;
        w->Up[((int64_t)bu * b + r) * b + c] = e / dt + J[r][c];
        w->L[((int64_t)bv * b + r) * b + c] = e / dt + J[c][r];
        if (i + 1 < N) {
          w->Up[((int64_t)bv * b + r) * b + c] = -e / dt;
          w->L[((int64_t)(bv + 1) * b + r) * b + c] = -e / dt;
        }
      }
    }
  }
  for (int q = 0; q < nf; ++q)
    if (s->wall[q])
      for (int k = 0; k < nb; ++k) w->D[((int64_t)k * b + q) * b + q] = 1.0;
  /* block Thomas */
  int ok = 1;
  double S[BMAX * BMAX], X[BMAX * CMAX];
  const int ncol = b + 1;
  for (int k = 0; k < nb; ++k) {
    const double* Dk = w->D + (int64_t)k * b * b;
    const double* Lk = w->L + (int64_t)k * b * b;
    const double* Uk = w->Up + (int64_t)k * b * b;
    const double* yk = w->y + (int64_t)k * b;
    for (int r = 0; r < b; ++r) {
      for (int c = 0; c < b; ++c) {
        double v = Dk[r * b + c];
        if (k > 0) {
          double acc = 0.0;
          for (int t = 0; t < b; ++t) acc += Lk[r * b + t] * w->W[((int64_t)(k - 1) * b + t) * b + c];
          v = v - acc;
        }
        S[r * b + c] = v;
      }
      double rv = yk[r];
      if (k > 0) {
        double acc = 0.0;
        for (int t = 0; t < b; ++t) acc += Lk[r * b + t] * w->z[(int64_t)(k - 1) * b + t];
        rv = rv - acc;
      }
      for (int c = 0; c < b; ++c) X[r * ncol + c] = Uk[r * b + c];
      X[r * ncol + b] = rv;
    }
    ok &= solve_pivot(b, S, ncol, X);
    for (int r = 0; r < b; ++r) {
      for (int c = 0; c < b; ++c) w->W[((int64_t)k * b + r) * b + c] = X[r * ncol + c];
      w->z[(int64_t)k * b + r] = X[r * ncol + b];
    }
  }
  /* back substitution in place: z -> x */
  for (int k = nb - 2; k >= 0; --k)
    for (int r = 0; r < b; ++r) {
      double acc = 0.0;
      for (int t = 0; t < b; ++t) acc += w->W[((int64_t)k * b + r) * b + t] * w->z[(int64_t)(k + 1) * b + t];
      w->z[(int64_t)k * b + r] -= acc;
    }
  return ok;
}

static int color_of_cell(const cgrid* g, int mod, int red_black, const int* c) {
  if (red_black) {
    int s = 0;
    for (int k = 0; k < g->dim; ++k) s += c[k];
    return s % 2;
  }
  int col = 0, mul = 1;
  for (int k = 0; k < g->dim; ++k) {
    col += (c[k] % mod) * mul;
    mul *= mod;
  }
  return col;
}

/* One colour pass (snapshot): cells = explicit list (ncells x 3 ints, 2D uses
 * the first two) or, when NULL, every cell of colour `color`.  Deltas
 * (omega * x) are applied in place unless apply == 0; when xout != NULL it
 * receives the raw line solution x [cell][2N][b].  Returns 0 / 3 (singular). */
int cst_color_pass(const cprob* pb, cstate* st, const cres* rhs, int color, const int* cells, int64_t ncells,
                   int apply, double* xout) {
  const cgrid* g = &pb->g;
  const int N = pb->N, nf = 2 * g->dim, b = nf + 1, nb = 2 * N;
  int64_t M = 0;
  int* own = NULL;
  if (!cells) {
    const int64_t nc = csize(g);
    own = (int*)malloc(sizeof(int) * 3 * nc);
    for (int64_t e = 0; e < nc; ++e) {
      int x[3];
      lat_coords(g, -1, e, x);
      if (color_of_cell(g, pb->colors, pb->red_black, x) == color) {
        own[3 * M] = x[0];
        own[3 * M + 1] = x[1];
        own[3 * M + 2] = x[2];
        ++M;
      }
    }
    cells = own;
  } else {
    M = ncells;
  }
  double* xs = xout ? xout : (double*)malloc(sizeof(double) * (size_t)M * nb * b);
  int ok = 1;
#pragma omp parallel reduction(&& : ok)
  {
    line_ws w;
    w.D = (double*)malloc(sizeof(double) * nb * b * b);
    w.L = (double*)malloc(sizeof(double) * nb * b * b);
    w.Up = (double*)malloc(sizeof(double) * nb * b * b);
    w.W = (double*)malloc(sizeof(double) * nb * b * b);
    w.y = (double*)malloc(sizeof(double) * nb * b);
    w.z = (double*)malloc(sizeof(double) * nb * b);
#pragma omp for schedule(dynamic, 16)
    for (int64_t m = 0; m < M; ++m) {
      int c[3] = {cells[3 * m], cells[3 * m + 1], g->dim > 2 ? cells[3 * m + 2] : 0};
      cslots s;
      cell_slots(g, c, &s);
      ok = cell_line(pb, st, rhs, &s, &w) && ok;
      memcpy(xs + (size_t)m * nb * b, w.z, sizeof(double) * nb * b);
    }
    free(w.D);
    free(w.L);
    free(w.Up);
    free(w.W);
    free(w.y);
    free(w.z);
  }
  if (apply) {
    const double om = pb->omega;
    const int64_t nc = csize(g);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
      int c[3] = {cells[3 * m], cells[3 * m + 1], g->dim > 2 ? cells[3 * m + 2] : 0};
      cslots s;
      cell_slots(g, c, &s);
      const double* x = xs + (size_t)m * nb * b;
      const int64_t co = lidx(g, -1, c);
      for (int i = 0; i < N; ++i) {
        const double* xu = x + (2 * i) * b;
        const double* xv = x + (2 * i + 1) * b;
        for (int q = 0; q < nf; ++q) {
          if (s.wall[q]) continue;
          const int k = s.fk[q];
          const int64_t o = (int64_t)i * fsize(g, k) + lidx(g, k, s.f[q]);
          st->U[k][o] += om * xu[q];
          st->V[k][o] += om * xv[q];
        }
        st->P[(int64_t)i * nc + co] += om * xu[nf];
        st->PB[(int64_t)i * nc + co] += om * xv[nf];
      }
    }
  }
  if (!xout) free(xs);
  free(own);
  return ok ? 0 : 3;
}

int cst_sweep(const cprob* pb, cstate* st, const cres* rhs) {
  int nc = 1, rc = 0;
  for (int k = 0; k < pb->g.dim; ++k) nc *= pb->colors;
  if (pb->red_black) nc = 2;
  for (int c = 0; c < nc; ++c) {
    int r = cst_color_pass(pb, st, rhs, c, NULL, 0, 1, NULL);
    if (r) rc = r;
  }
  return rc;
}

/* ----------------------------------------------------------- transfers */

static int coarsenable(const cgrid* g) {
  for (int a = 0; a < g->dim; ++a)
    if (g->n[a] % 2 || g->n[a] / 2 < 4) return 0;
  return 1;
}
/* oracle/stfas.py colourable: same-colour cells share no face */
static int colourable(const cgrid* g, int mod, int red_black) {
  for (int a = 0; a < g->dim; ++a) {
    if (red_black && a == g->dim - 1 && g->n[a] % 2) return 0;
    if (g->per && g->n[a] % (red_black ? 2 : mod)) return 0;
  }
  return 1;
}
static cgrid coarse_of(const cgrid* g) {
  cgrid c = *g;
  for (int a = 0; a < g->dim; ++a) c.n[a] = g->n[a] / 2;
  c.h = 2.0 * g->h;
  return c;
}

/* restrict_cell at coarse cell C (per-axis pair averages, axis 0 first) */
static double rcell_rec(const cgrid* gf, const double* x, int a, int* F) {
  if (a < 0) return x[lidx(gf, -1, F)];
  /* averages along axis a of the array already reduced along axes < a:
     evaluate innermost-last so axis 0 is reduced first */
  int F0[3] = {F[0], F[1], F[2]}, F1[3] = {F[0], F[1], F[2]};
  F1[a] += 1;
  return 0.5 * (rcell_rec(gf, x, a - 1, F0) + rcell_rec(gf, x, a - 1, F1));
}
void cst_restrict_cell(const cgrid* gf, int nframes, const double* x, double* out) {
  cgrid gc = coarse_of(gf);
  const int64_t nf = csize(gf), ncs = csize(&gc);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)nframes * ncs; ++t) {
    int fr = (int)(t / ncs);
    int C[3];
    lat_coords(&gc, -1, t % ncs, C);
    int F[3] = {2 * C[0], 2 * C[1], gf->dim > 2 ? 2 * C[2] : 0};
    out[t] = rcell_rec(gf, x + (int64_t)fr * nf, gf->dim - 1, F);
  }
}
/* restrict_face comp k at coarse face C: along k take the even fine face,
   across average pairs (axis order 0..dim-1) */
static double rface_rec(const cgrid* gf, const double* x, int k, int a, int* F) {
  if (a < 0) return x[lidx(gf, k, F)];
  if (a == k) return rface_rec(gf, x, k, a - 1, F);
  int F0[3] = {F[0], F[1], F[2]}, F1[3] = {F[0], F[1], F[2]};
  F1[a] += 1;
  return 0.5 * (rface_rec(gf, x, k, a - 1, F0) + rface_rec(gf, x, k, a - 1, F1));
}
void cst_restrict_face(const cgrid* gf, int nframes, double* const in[3], double* const out[3]) {
  cgrid gc = coarse_of(gf);
  for (int k = 0; k < gf->dim; ++k) {
    const int64_t nf = fsize(gf, k), ncs = fsize(&gc, k);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)nframes * ncs; ++t) {
      int fr = (int)(t / ncs);
      int C[3];
      lat_coords(&gc, k, t % ncs, C);
      int F[3] = {2 * C[0], 2 * C[1], gf->dim > 2 ? 2 * C[2] : 0};
      out[k][t] = rface_rec(gf, in[k] + (int64_t)fr * nf, k, gf->dim - 1, F);
    }
  }
}
/* prolongation: T_{a+1}[.., F_a, ..] from T_a; k = -1 for cells */
static double pro_rec(const cgrid* gc, const double* x, int k, int a, int* I) {
  /* I: fine indices on axes < a, coarse on axes >= a */
  if (a == 0) return x[lidx(gc, k, I)];
  const int b = a - 1;
  const int Fb = I[b];
  int J0[3] = {I[0], I[1], I[2]}, J1[3] = {I[0], I[1], I[2]};
  if (b == k) {
    /* linear along the face normal: even -> c[i], odd -> (c[i] + c[i+1]) / 2 */
    const int i = Fb / 2;
    J0[b] = i;
    if (Fb % 2 == 0) return pro_rec(gc, x, k, b, J0);
    int ip = i + 1;
    if (gc->per) ip %= gc->n[b];
    J1[b] = ip;
    return 0.5 * (pro_rec(gc, x, k, b, J0) + pro_rec(gc, x, k, b, J1));
  }
  const int i = Fb / 2, n = gc->n[b];
  int j = (Fb % 2 == 0) ? i - 1 : i + 1;
  if (gc->per)
    j = (j + n) % n;
  else
    j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
  J0[b] = i;
  J1[b] = j;
  return 0.75 * pro_rec(gc, x, k, b, J0) + 0.25 * pro_rec(gc, x, k, b, J1);
}
/* out (fine) = P x (accumulate: out += P x) */
void cst_prolong_cell(const cgrid* gc, int nframes, const double* x, double* out, int accumulate) {
  cgrid gf = *gc;
  for (int a = 0; a < gc->dim; ++a) gf.n[a] *= 2;
  gf.h = gc->h / 2;
  const int64_t nf = csize(&gf), ncs = csize(gc);
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)nframes * nf; ++t) {
    int fr = (int)(t / nf);
    int F[3];
    lat_coords(&gf, -1, t % nf, F);
    double v = pro_rec(gc, x + (int64_t)fr * ncs, -1, gc->dim, F);
    out[t] = accumulate ? out[t] + v : v;
  }
}
void cst_prolong_face(const cgrid* gc, int nframes, double* const in[3], double* const out[3], int accumulate) {
  cgrid gf = *gc;
  for (int a = 0; a < gc->dim; ++a) gf.n[a] *= 2;
  gf.h = gc->h / 2;
  for (int k = 0; k < gc->dim; ++k) {
    const int64_t nf = fsize(&gf, k), ncs = fsize(gc, k);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)nframes * nf; ++t) {
      int fr = (int)(t / nf);
      int F[3];
      lat_coords(&gf, k, t % nf, F);
      double v = pro_rec(gc, in[k] + (int64_t)fr * ncs, k, gc->dim, F);
      out[k][t] = accumulate ? out[k][t] + v : v;
    }
  }
}

/* ------------------------------------------------------------ hierarchy */

typedef struct {
  cprob pb;
  double* v0[3];
  double* vs[3];
  cstate st, st0;   /* coarse state and its restricted copy (levels >= 1) */
  cres rhs;         /* FAS rhs (levels >= 1) */
  cres res;         /* residual scratch */
  cres rr;          /* restricted residual (of the next finer level's rows) */
} clevel;

typedef struct {
  int nl;
  clevel lv[8];
  int nu1, nu2, n_coarse;
} chier;

static double* dalloc(int64_t n) {
  double* p = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  return p;
}
static void state_alloc(const cgrid* g, int N, cstate* s) {
  memset(s, 0, sizeof(*s));
  for (int k = 0; k < g->dim; ++k) {
    s->V[k] = dalloc(N * fsize(g, k));
    s->U[k] = dalloc(N * fsize(g, k));
  }
  s->PB = dalloc(N * csize(g));
  s->P = dalloc(N * csize(g));
}
static void state_free(cstate* s) {
  for (int k = 0; k < 3; ++k) {
    free(s->V[k]);
    free(s->U[k]);
  }
  free(s->PB);
  free(s->P);
  memset(s, 0, sizeof(*s));
}
static void res_alloc(const cgrid* g, int N, cres* s) {
  memset(s, 0, sizeof(*s));
  for (int k = 0; k < g->dim; ++k) {
    s->R1[k] = dalloc(N * fsize(g, k));
    s->R3[k] = dalloc(N * fsize(g, k));
  }
  s->R2 = dalloc(N * csize(g));
  s->R4 = dalloc(N * csize(g));
}
static void res_free(cres* s) {
  for (int k = 0; k < 3; ++k) {
    free(s->R1[k]);
    free(s->R3[k]);
  }
  free(s->R2);
  free(s->R4);
  memset(s, 0, sizeof(*s));
}

/* build the hierarchy: level guides by the face restriction (build_levels) */
chier* cst_hier_create(const cprob* top, int n_levels, int nu1, int nu2, int n_coarse) {
  chier* H = (chier*)calloc(1, sizeof(chier));
  H->nu1 = nu1;
  H->nu2 = nu2;
  H->n_coarse = n_coarse;
  H->lv[0].pb = *top;
  H->nl = 1;
  const int N = top->N;
  res_alloc(&top->g, N, &H->lv[0].res);
  while (H->nl < n_levels && H->nl < 8 && coarsenable(&H->lv[H->nl - 1].pb.g)) {
    cgrid gnext = coarse_of(&H->lv[H->nl - 1].pb.g);
    if (!colourable(&gnext, top->colors, top->red_black)) break;
    clevel* f = &H->lv[H->nl - 1];
    clevel* c = &H->lv[H->nl];
    c->pb = f->pb;
    c->pb.g = coarse_of(&f->pb.g);
    const cgrid* gc = &c->pb.g;
    for (int k = 0; k < gc->dim; ++k) {
      c->v0[k] = dalloc(fsize(gc, k));
      c->vs[k] = dalloc((int64_t)f->pb.vs_frames * fsize(gc, k));
    }
    cst_restrict_face(&f->pb.g, 1, (double* const*)f->pb.v0, c->v0);
    cst_restrict_face(&f->pb.g, f->pb.vs_frames, (double* const*)f->pb.vstar, c->vs);
    for (int k = 0; k < 3; ++k) {
      c->pb.v0[k] = c->v0[k];
      c->pb.vstar[k] = c->vs[k];
      c->pb.unext[k] = NULL;
    }
    state_alloc(gc, N, &c->st);
    state_alloc(gc, N, &c->st0);
    res_alloc(gc, N, &c->rhs);
    res_alloc(gc, N, &c->res);
    res_alloc(gc, N, &c->rr);
    H->nl++;
  }
  return H;
}
void cst_hier_destroy(chier* H) {
  if (!H) return;
  res_free(&H->lv[0].res);
  for (int l = 1; l < H->nl; ++l) {
    clevel* c = &H->lv[l];
    for (int k = 0; k < 3; ++k) {
      free(c->v0[k]);
      free(c->vs[k]);
    }
    state_free(&c->st);
    state_free(&c->st0);
    res_free(&c->rhs);
    res_free(&c->res);
    res_free(&c->rr);
  }
  free(H);
}
int cst_hier_levels(const chier* H) { return H->nl; }

static void state_copy(const cgrid* g, int N, const cstate* a, cstate* b) {
  for (int k = 0; k < g->dim; ++k) {
    memcpy(b->V[k], a->V[k], sizeof(double) * N * fsize(g, k));
    memcpy(b->U[k], a->U[k], sizeof(double) * N * fsize(g, k));
  }
  memcpy(b->PB, a->PB, sizeof(double) * N * csize(g));
  memcpy(b->P, a->P, sizeof(double) * N * csize(g));
}

static void restrict_state(const cgrid* gf, int N, const cstate* f, cstate* c) {
  cst_restrict_face(gf, N, f->V, c->V);
  cst_restrict_cell(gf, N, f->PB, c->PB);
  cst_restrict_face(gf, N, f->U, c->U);
  cst_restrict_cell(gf, N, f->P, c->P);
}

/* vcycle (oracle/stfas.py vcycle): level li's state in place */
static int vcycle_rec(chier* H, int li, cstate* st, const cres* rhs) {
  clevel* L = &H->lv[li];
  const cprob* pb = &L->pb;
  const int N = pb->N;
  int rc = 0, r;
  if (li == H->nl - 1 || li >= 7) {
    for (int s = 0; s < H->n_coarse; ++s)
      if ((r = cst_sweep(pb, st, rhs))) rc = r;
    return rc;
  }
  for (int s = 0; s < H->nu1; ++s)
    if ((r = cst_sweep(pb, st, rhs))) rc = r;
  clevel* C = &H->lv[li + 1];
  const cgrid* g = &pb->g;
  const cgrid* gc = &C->pb.g;
  restrict_state(g, N, st, &C->st0);
  /* ff = f(st); rh - ff (rh = 0 when rhs is NULL) */
  cst_kkt_residual(pb, st, NULL, &L->res);
  for (int k = 0; k < g->dim; ++k) {
    const int64_t n = (int64_t)N * fsize(g, k);
    for (int64_t t = 0; t < n; ++t) {
      L->res.R1[k][t] = (rhs ? rhs->R1[k][t] : 0.0) - L->res.R1[k][t];
      L->res.R3[k][t] = (rhs ? rhs->R3[k][t] : 0.0) - L->res.R3[k][t];
    }
  }
  {
    const int64_t n = (int64_t)N * csize(g);
    for (int64_t t = 0; t < n; ++t) {
      L->res.R2[t] = (rhs ? rhs->R2[t] : 0.0) - L->res.R2[t];
      L->res.R4[t] = (rhs ? rhs->R4[t] : 0.0) - L->res.R4[t];
    }
  }
  cst_restrict_face(g, N, L->res.R1, C->rr.R1);
  cst_restrict_cell(g, N, L->res.R2, C->rr.R2);
  cst_restrict_face(g, N, L->res.R3, C->rr.R3);
  cst_restrict_cell(g, N, L->res.R4, C->rr.R4);
  /* rc = f_c(sc0) + R(rh - ff) */
  cst_kkt_residual(&C->pb, &C->st0, NULL, &C->rhs);
  for (int k = 0; k < gc->dim; ++k) {
    const int64_t n = (int64_t)N * fsize(gc, k);
    for (int64_t t = 0; t < n; ++t) {
      C->rhs.R1[k][t] = C->rhs.R1[k][t] + C->rr.R1[k][t];
      C->rhs.R3[k][t] = C->rhs.R3[k][t] + C->rr.R3[k][t];
    }
  }
  {
    const int64_t n = (int64_t)N * csize(gc);
    for (int64_t t = 0; t < n; ++t) {
      C->rhs.R2[t] = C->rhs.R2[t] + C->rr.R2[t];
      C->rhs.R4[t] = C->rhs.R4[t] + C->rr.R4[t];
    }
  }
  state_copy(gc, N, &C->st0, &C->st);
  if ((r = vcycle_rec(H, li + 1, &C->st, &C->rhs))) rc = r;
  /* st += P(sc - sc0) */
  for (int k = 0; k < gc->dim; ++k) {
    const int64_t n = (int64_t)N * fsize(gc, k);
    for (int64_t t = 0; t < n; ++t) {
      C->st.V[k][t] = C->st.V[k][t] + (-1.0) * C->st0.V[k][t];
      C->st.U[k][t] = C->st.U[k][t] + (-1.0) * C->st0.U[k][t];
    }
  }
  {
    const int64_t n = (int64_t)N * csize(gc);
    for (int64_t t = 0; t < n; ++t) {
      C->st.PB[t] = C->st.PB[t] + (-1.0) * C->st0.PB[t];
      C->st.P[t] = C->st.P[t] + (-1.0) * C->st0.P[t];
    }
  }
  cst_prolong_face(gc, N, C->st.V, st->V, 1);
  cst_prolong_cell(gc, N, C->st.PB, st->PB, 1);
  cst_prolong_face(gc, N, C->st.U, st->U, 1);
  cst_prolong_cell(gc, N, C->st.P, st->P, 1);
  for (int s = 0; s < H->nu2; ++s)
    if ((r = cst_sweep(pb, st, rhs))) rc = r;
  return rc;
}

void cst_gauge_fix(const cgrid* g, int N, cstate* st) {
  const int64_t nc = csize(g);
  for (int i = 0; i < N; ++i) {
    double* arrs[2] = {st->PB + (int64_t)i * nc, st->P + (int64_t)i * nc};
    for (int a = 0; a < 2; ++a) {
      double s = 0.0;
      for (int64_t e = 0; e < nc; ++e) s += arrs[a][e];
      const double mean = s / (double)nc;
      for (int64_t e = 0; e < nc; ++e) arrs[a][e] -= mean;
    }
  }
}

int cst_hier_vcycle(chier* H, cstate* st, int gauge) {
  int rc = vcycle_rec(H, 0, st, NULL);
  if (gauge) cst_gauge_fix(&H->lv[0].pb.g, H->lv[0].pb.N, st);
  return rc;
}

/* ||f||_inf and ||f||_2 of the top level */
void cst_hier_norms(chier* H, const cstate* st, double* rinf, double* rl2) {
  clevel* L = &H->lv[0];
  const cgrid* g = &L->pb.g;
  const int N = L->pb.N;
  cst_kkt_residual(&L->pb, st, NULL, &L->res);
  double mx = 0.0, s2 = 0.0;
  const double* arrs[8];
  int64_t lens[8];
  int na = 0;
  for (int k = 0; k < g->dim; ++k) {
    arrs[na] = L->res.R1[k];
    lens[na++] = N * fsize(g, k);
  }
  arrs[na] = L->res.R2;
  lens[na++] = N * csize(g);
  for (int k = 0; k < g->dim; ++k) {
    arrs[na] = L->res.R3[k];
    lens[na++] = N * fsize(g, k);
  }
  arrs[na] = L->res.R4;
  lens[na++] = N * csize(g);
  for (int a = 0; a < na; ++a)
    for (int64_t t = 0; t < lens[a]; ++t) {
      const double v = arrs[a][t];
      if (fabs(v) > mx) mx = fabs(v);
      s2 += v * v;
    }
  *rinf = mx;
  *rl2 = sqrt(s2);
}

/* solve_nso: hist gets (res_inf, res_l2) per cycle (2 * (budget + 1)).
   Returns 0 converged, 1 budget exhausted, 3 singular. */
int cst_hier_solve(chier* H, cstate* st, double eps, int relative, int budget, int* cycles, double* hist) {
  double ri, r2;
  cst_hier_norms(H, st, &ri, &r2);
  if (hist) {
    hist[0] = ri;
    hist[1] = r2;
  }
  *cycles = 0;
  const double tol = relative ? eps * ri : eps;
  if (ri <= tol) return 0;
  for (int c = 1; c <= budget; ++c) {
    int rc = cst_hier_vcycle(H, st, 1);
    cst_hier_norms(H, st, &ri, &r2);
    if (hist) {
      hist[2 * c] = ri;
      hist[2 * c + 1] = r2;
    }
    *cycles = c;
    if (rc == 3) return 3;
    if (ri <= tol) return 0;
  }
  return 1;
}

int cst_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}
