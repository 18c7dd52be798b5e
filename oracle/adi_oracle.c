/*
 * adi_oracle.c — CPU fp64 ORACLE for the Peaceman–Rachford ADI step of
 * Otero, Rojas, Moya & Castillo, arXiv:2006.07583.
 *
 * *** TEST INFRASTRUCTURE ONLY. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_2006_07583_b200/) never links, imports or calls it, and it shares no
 * code, header, table or helper with the CUDA path.
 *
 * It is deliberately plain and slow: every derivative is the paper's
 * operator applied literally (stencil rows of Q, Q̄, D4, G4 as printed, then a
 * Thomas solve with P or P̄ factored once, no pivoting), every ADI stage is the
 * fixed-point loop of eqs. 8–9 / Alg. 3–4 in the paper's order, plain loops,
 * fp64, no FMA contraction (built with -ffp-contract=off), OpenMP over
 * independent grid lines only ("no data dependency among the N linear
 * systems").
 *
 * Citations are PAPER.md line numbers (section / equation / algorithm).
 * Readings of ambiguous passages are SURVEY.md §8c G1–G21 and are listed in
 * DESIGN.md §3; the ones used here are cited inline as [G#].
 *
 * Layout (row index = y, column index = x):
 *   CFD (Alg. 1 Require): nx, ny nodes per direction,
 *       N_x = nx-1 cells.  U is ny x nx (boundary included);
 *       V̄ = rows 1..ny-2 of V, shape (ny-2) x nx;  W̄ = cols 1..nx-2 of W,
 *       shape ny x (nx-2).
 *   MFD ([G13]): U on X_cb⊗Y_cb, (ny+1) x (nx+1);
 *       V̄ = (ny-1) x nx (N_y centres x N_x+1 nodes);
 *       W̄ = ny x (nx-1) (N_y+1 nodes x N_x centres).
 * The edge velocity lines that the paper never updates are not state [G12].
 *
 * NEXT rows: heterogeneous media (f3: per-point alpha, beta in stage_line and
 * or_run, from or_problem.kappa / rv / rw) and the full-matrix CFD variant with a
 * Cerjan layer (f4: or_run_full, stage_line_full).
 *
 * Parity status of each function is listed in DESIGN.md §4, §8.3 and §8.4 (all
 * pinned).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_CFD 0
#define OR_MFD 1

/* ------------------------------------------------------------------------ */
/* Tridiagonal LU without pivoting.                                          */
/* "forward and backward substitutions from the LU decomposition of          */
/*  tridiagonal P and P̄"; "omit any pivoting strategy"       */
/*  (PAPER.md:192); factor once.                              */
/* Row i: a[i]*x[i-1] + b[i]*x[i] + c[i]*x[i+1] = r[i].                      */
/* ------------------------------------------------------------------------ */
int or_tri_factor(int n, const double* a, const double* b, const double* c,
                  double* l, double* d) {
  (void)c;
  d[0] = b[0];
  l[0] = 0.0;
  if (d[0] == 0.0) return -4;
  for (int i = 1; i < n; ++i) {
    l[i] = a[i] / d[i - 1];
    d[i] = b[i] - l[i] * c[i - 1];
    if (d[i] == 0.0) return -4;
  }
  return 0;
}

/* x may alias r. */
void or_tri_solve(int n, const double* l, const double* d, const double* c,
                  const double* r, double* x) {
  /* forward substitution: L y = r */
  x[0] = r[0];
  for (int i = 1; i < n; ++i) x[i] = r[i] - l[i] * x[i - 1];
  /* backward substitution: U x = y */
  x[n - 1] = x[n - 1] / d[n - 1];
  for (int i = n - 2; i >= 0; --i) x[i] = (x[i] - c[i] * x[i + 1]) / d[i];
}

/* ------------------------------------------------------------------------ */
/* CFD operators, Appendix A, n = number of cells.        */
/* ------------------------------------------------------------------------ */
typedef struct {
  int n;          /* cells */
  double h;
  /* P: (n+1)x(n+1), eq. 12 */
  double *Pa, *Pb, *Pc, *Pl, *Pd;
  /* P̄: (n-1)x(n-1), eq. 14; size n-1 [G1] */
  double *Ba, *Bb, *Bc, *Bl, *Bd;
} cfd_ops;

static int cfd_ops_init(cfd_ops* o, int n, double h) {
  o->n = n;
  o->h = h;
  int np = n + 1, nb = n - 1;
  double* mem = (double*)malloc(sizeof(double) * (5 * np + 5 * nb));
  if (!mem) return -2;
  o->Pa = mem; o->Pb = o->Pa + np; o->Pc = o->Pb + np; o->Pl = o->Pc + np; o->Pd = o->Pl + np;
  o->Ba = o->Pd + np; o->Bb = o->Ba + nb; o->Bc = o->Bb + nb; o->Bl = o->Bc + nb; o->Bd = o->Bl + nb;
  /* P4: first row (6, 18), interior (1, 4, 1), last row (18, 6). */
  for (int i = 0; i < np; ++i) { o->Pa[i] = 1.0; o->Pb[i] = 4.0; o->Pc[i] = 1.0; }
  o->Pa[0] = 0.0; o->Pb[0] = 6.0; o->Pc[0] = 18.0;
  o->Pa[n] = 18.0; o->Pb[n] = 6.0; o->Pc[n] = 0.0;
  /* P̄4: first row (6, 6), interior (1, 4, 1), last row (6, 6). */
  for (int i = 0; i < nb; ++i) { o->Ba[i] = 1.0; o->Bb[i] = 4.0; o->Bc[i] = 1.0; }
  o->Ba[0] = 0.0; o->Bb[0] = 6.0; o->Bc[0] = 6.0;
  o->Ba[nb - 1] = 6.0; o->Bb[nb - 1] = 6.0; o->Bc[nb - 1] = 0.0;
  int e1 = or_tri_factor(np, o->Pa, o->Pb, o->Pc, o->Pl, o->Pd);
  int e2 = or_tri_factor(nb, o->Ba, o->Bb, o->Bc, o->Bl, o->Bd);
  return (e1 || e2) ? -4 : 0;
}
static void cfd_ops_free(cfd_ops* o) { free(o->Pa); }

/* Q4 f (eq. 13): (n+1) nodes -> (n+1) nodes. */
void or_cfd_Qf(int n, double h, const double* f, double* out) {
  out[0] = (-17.0 * f[0] + 9.0 * f[1] + 9.0 * f[2] - 1.0 * f[3]) / h;
  for (int i = 1; i < n; ++i) out[i] = (-3.0 * f[i - 1] + 3.0 * f[i + 1]) / h;
  out[n] = (1.0 * f[n - 3] - 9.0 * f[n - 2] - 9.0 * f[n - 1] + 17.0 * f[n]) / h;
}
/* Q̄4 f (eq. 15): (n+1) nodes -> interior nodes 1..n-1. */
void or_cfd_Qbarf(int n, double h, const double* f, double* out) {
  out[0] = (-1.0 * f[0] - 9.0 * f[1] + 9.0 * f[2] + 1.0 * f[3]) / h;
  for (int r = 1; r < n - 2; ++r) out[r] = (-3.0 * f[r] + 3.0 * f[r + 2]) / h;
  out[n - 2] = (-1.0 * f[n - 3] - 9.0 * f[n - 2] + 9.0 * f[n - 1] + 1.0 * f[n]) / h;
}
/* D(f) = P^{-1} Q f : U_x P^T = U Q^T / P U_y = Q U. */
static void cfd_D(const cfd_ops* o, const double* f, double* out) {
  or_cfd_Qf(o->n, o->h, f, out);
  or_tri_solve(o->n + 1, o->Pl, o->Pd, o->Pc, out, out);
}
/* D̄(f) = P̄^{-1} Q̄ f : V̄_x P̄^T = V̄ Q̄^T / P̄ W̄_y = Q̄ W̄ (eq. 2). */
static void cfd_Dbar(const cfd_ops* o, const double* f, double* out) {
  or_cfd_Qbarf(o->n, o->h, f, out);
  or_tri_solve(o->n - 1, o->Bl, o->Bd, o->Bc, out, out);
}

/* ------------------------------------------------------------------------ */
/* MFD operators, Appendix B, alpha=beta=0, gamma=-1/24   */
/* [G15]; bottom rows are the top rows reversed and negated.                 */
/* ------------------------------------------------------------------------ */
static const double D4_row0_num[6] = {-4751.0, 909.0, 6091.0, -1165.0, 129.0, -25.0};
static const double D4_row0_den[6] = {5192.0, 1298.0, 15576.0, 5192.0, 2596.0, 15576.0};
static const double G4_row0_num[6] = {-47888.0, 1790.0, -14545.0, 8997.0, -2335.0, 25.0};
static const double G4_row0_den[6] = {14245.0, 407.0, 9768.0, 16280.0, 22792.0, 9768.0};
static const double G4_row1_num[5] = {16.0, -31.0, 29.0, -3.0, 1.0};
static const double G4_row1_den[5] = {105.0, 24.0, 24.0, 40.0, 168.0};
static const double INT_num[4] = {1.0, -9.0, 9.0, -1.0};
static const double INT_den[4] = {24.0, 8.0, 8.0, 24.0};

/* D4 f: nodes (n+1) -> centres (n).  Row r <-> centre r (x = (r+1/2)h). */
void or_mfd_D4f(int n, double h, const double* f, double* out) {
  double s = 0.0;
  for (int k = 0; k < 6; ++k) s += (D4_row0_num[k] / D4_row0_den[k]) * f[k];
  out[0] = s / h;
  for (int r = 1; r < n - 1; ++r) {
    s = 0.0;
    for (int k = 0; k < 4; ++k) s += (INT_num[k] / INT_den[k]) * f[r - 1 + k];
    out[r] = s / h;
  }
  s = 0.0; /* last row = first row reversed and negated, on nodes n-5..n */
  for (int k = 0; k < 6; ++k) s += (-D4_row0_num[5 - k] / D4_row0_den[5 - k]) * f[n - 5 + k];
  out[n - 1] = s / h;
}
/* G4 f: cb points (n+2: 0, centres, 1) -> nodes (n+1). */
void or_mfd_G4f(int n, double h, const double* f, double* out) {
  double s = 0.0;
  for (int k = 0; k < 6; ++k) s += (G4_row0_num[k] / G4_row0_den[k]) * f[k];
  out[0] = s / h;
  s = 0.0;
  for (int k = 0; k < 5; ++k) s += (G4_row1_num[k] / G4_row1_den[k]) * f[k];
  out[1] = s / h;
  for (int i = 2; i < n - 1; ++i) {
    s = 0.0;
    for (int k = 0; k < 4; ++k) s += (INT_num[k] / INT_den[k]) * f[i - 1 + k];
    out[i] = s / h;
  }
  s = 0.0; /* row n-1: row 1 reversed and negated on cb n-3..n+1 */
  for (int k = 0; k < 5; ++k) s += (-G4_row1_num[4 - k] / G4_row1_den[4 - k]) * f[n - 3 + k];
  out[n - 1] = s / h;
  s = 0.0; /* row n: row 0 reversed and negated on cb n-4..n+1 */
  for (int k = 0; k < 6; ++k) s += (-G4_row0_num[5 - k] / G4_row0_den[5 - k]) * f[n - 4 + k];
  out[n] = s / h;
}

/* ------------------------------------------------------------------------ */
/* One 1-D axis of either method: D maps pressure-with-boundary -> velocity  */
/* points, D̄ maps velocity points -> pressure-interior points.              */
/*   CFD: D = P^{-1}Q (nodes->nodes), D̄ = P̄^{-1}Q̄ (nodes->interior nodes)  */
/*   MFD: D = G4 (cb->nodes),           D̄ = D4 (nodes->centres)            */
/* (eq. 3; eq. 10)                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  int method, n;
  double h;
  cfd_ops cfd;
  int nu;   /* pressure-interior points on the line: n-1 (CFD) / n (MFD) */
  int nub;  /* pressure points incl. the 2 Dirichlet ends: n+1 / n+2     */
  int nv;   /* velocity points on the line: n+1 (both)                    */
} axis_t;

static int axis_init(axis_t* a, int method, int n, double h) {
  a->method = method; a->n = n; a->h = h;
  a->nv = n + 1;
  if (method == OR_CFD) { a->nu = n - 1; a->nub = n + 1; return cfd_ops_init(&a->cfd, n, h); }
  a->nu = n; a->nub = n + 2;
  return 0;
}
static void axis_free(axis_t* a) { if (a->method == OR_CFD) cfd_ops_free(&a->cfd); }
/* D: ub[nub] -> out[nv] */
static void axis_D(const axis_t* a, const double* ub, double* out) {
  if (a->method == OR_CFD) cfd_D(&a->cfd, ub, out); else or_mfd_G4f(a->n, a->h, ub, out);
}
/* D̄: v[nv] -> out[nu] */
static void axis_Dbar(const axis_t* a, const double* v, double* out) {
  if (a->method == OR_CFD) cfd_Dbar(&a->cfd, v, out); else or_mfd_D4f(a->n, a->h, v, out);
}

/* Exported single-line operator entry points (operator pin tests). */
int or_apply_D(int method, int n, double h, const double* ub, double* out) {
  axis_t a; int e = axis_init(&a, method, n, h); if (e) return e;
  axis_D(&a, ub, out); axis_free(&a); return 0;
}
int or_apply_Dbar(int method, int n, double h, const double* v, double* out) {
  axis_t a; int e = axis_init(&a, method, n, h); if (e) return e;
  axis_Dbar(&a, v, out); axis_free(&a); return 0;
}

/* ------------------------------------------------------------------------ */
/* One ADI stage on one line: the fixed-point iteration of eq. 8 / eq. 9,    */
/* Alg. 3/4 with a fixed K sweeps [G10],*/
/* Seidel coupling u before v [G11], initial guess v0 = (V^m | W*) [G7]:      */
/*   repeat K:  u <- s - alpha * D̄(v)                                       */
/*              v <- v0 - beta * D([gL, u, gR])                               */
/* Heterogeneous media (NEXT row f3; Alg. 3/4 "K.*( )", "R.*( )",            */
/* PAPER.md:655-656, 695-696; K, R: grid values of kappa and rho^-1,         */
/* PAPER.md:183): alpha and beta become per-point, alpha_i = dt/2 K_i after  */
/* the derivative [G8], beta_j = dt/2 R_j; av (nu) / bv (nv) hold them, or   */
/* NULL for the scalars alpha / beta.                                        */
/* Returns u (nu), v (nv).                                                    */
/* ------------------------------------------------------------------------ */
#define OR_A(i) (av ? av[i] : alpha)
#define OR_B(i) (bv ? bv[i] : beta)
static void stage_line(const axis_t* a, int K, double alpha, double beta, const double* av,
                       const double* bv, const double* s, const double* v0, double gL, double gR,
                       double* u, double* v, double* ub, double* tmp) {
  for (int i = 0; i < a->nv; ++i) v[i] = v0[i];
  for (int k = 0; k < K; ++k) {
    axis_Dbar(a, v, tmp);
    for (int i = 0; i < a->nu; ++i) u[i] = s[i] - OR_A(i) * tmp[i];
    ub[0] = gL;
    for (int i = 0; i < a->nu; ++i) ub[i + 1] = u[i];
    ub[a->nub - 1] = gR;
    axis_D(a, ub, tmp);
    for (int i = 0; i < a->nv; ++i) v[i] = v0[i] - OR_B(i) * tmp[i];
  }
}

/* The same iteration to kmax sweeps, recording for k = 2..kmax the squared
 * changes du2[k] = sum_i (u_k - u_{k-1})^2, dv2[k] = sum_i (v_k - v_{k-1})^2 of
 * this line (Alg. 3/4 "test"; the Frobenius norms of the
 * whole matrices are the square roots of the sums over the lines). */
static void stage_line_norms(const axis_t* a, int kmax, double alpha, double beta,
                             const double* av, const double* bv, const double* s, const double* v0, double gL, double gR,
                             double* u, double* v, double* ub, double* tmp, double* uold,
                             double* vold, double* du2, double* dv2) {
  for (int i = 0; i < a->nv; ++i) v[i] = v0[i];
  for (int k = 1; k <= kmax; ++k) {
    for (int i = 0; i < a->nu; ++i) uold[i] = u[i];
    for (int i = 0; i < a->nv; ++i) vold[i] = v[i];
    axis_Dbar(a, v, tmp);
    for (int i = 0; i < a->nu; ++i) u[i] = s[i] - OR_A(i) * tmp[i];
    ub[0] = gL;
    for (int i = 0; i < a->nu; ++i) ub[i + 1] = u[i];
    ub[a->nub - 1] = gR;
    axis_D(a, ub, tmp);
    for (int i = 0; i < a->nv; ++i) v[i] = v0[i] - OR_B(i) * tmp[i];
    double su = 0.0, sv = 0.0;
    if (k >= 2) {
      for (int i = 0; i < a->nu; ++i) su += (u[i] - uold[i]) * (u[i] - uold[i]);
      for (int i = 0; i < a->nv; ++i) sv += (v[i] - vold[i]) * (v[i] - vold[i]);
    }
    du2[k] = su;
    dv2[k] = sv;
  }
}

/* Alg. 3/4 stopping rule with the paper's GPU practice:
 * sweeps k = kmin..kmax are tested, test_k = ||U_k - U_{k-1}||_F + ||V_k -
 * V_{k-1}||_F over the whole stage (all lines); the stage stops at the first k
 * with test_k <= eps, else at kmax. */
static int pick_k(const double* su, const double* sv, int kmin, int kmax, double eps, double* tests) {
  int ks = kmax;
  for (int k = kmin; k <= kmax; ++k) {
    const double t = sqrt(su[k]) + sqrt(sv[k]);
    if (tests) tests[k] = t;
    if (t <= eps && ks == kmax) ks = k;
  }
  return ks;
}

/* ------------------------------------------------------------------------ */
/* Problem description (time tables sampled at half steps).      */
/* ------------------------------------------------------------------------ */
typedef struct {
  int method, nx, ny, K;
  double eps; int kmin;          /* Alg. 3/4 stopping rule: eps > 0 tests sweeps kmin..K */
  int* kchosen;                  /* if set: [2 * nsteps] chosen sweeps (rows, columns) */
  double* tests;                 /* if set: [2 * nsteps][K + 1] test values (k >= kmin) */
  double h, dt, c, rho;
  const double* phi;  /* source pattern on pressure-interior points, or NULL */
  int src_ix, src_iy; /* point source (U-array indices), F = g_f / h^2; <0: none */
  const double* gf; int ngf;     /* g_f(t0 + j dt/2), j < ngf; NULL -> 1 */
  const double* edges[4];        /* y0 (U row 0), y1 (U last row), x0 (U col 0), x1 (U last col) */
  const double* gb; int ngb;     /* g_b(t0 + j dt/2); NULL -> 1 */
  /* heterogeneous media (f3): kappa on the U layout (interior used), rho^-1 on
   * the V̄ (rv) and W̄ (rw) layouts; all three set, or all NULL (scalar kappa, rho) */
  const double* kappa; const double* rv; const double* rw;
} or_problem;

static double tab(const double* g, int ng, int j) {
  (void)ng; /* coverage is checked by or_run_flat */
  return g ? g[j] : 1.0;
}

/* F(t) at pressure-interior point (jj, ii) (row, col of the interior block):
 * the A_F term of eq. 4-6. */
static double source_at(const or_problem* p, int nxi, int jj, int ii, double gft) {
  double f = 0.0;
  if (p->phi) f += p->phi[(size_t)jj * nxi + ii] * gft;
  if (p->src_ix >= 1 && p->src_iy >= 1 && ii == p->src_ix - 1 && jj == p->src_iy - 1)
    f += gft / (p->h * p->h);
  return f;
}

/* f3 (heterogeneous media): per-point alpha_i = dt/2 K, beta_j = dt/2 R of one
 * row line jj (K at U(jj+1, i+1), R = rv at V̄(jj, i)) or one column line ii (K at
 * U(r+1, ii+1), R = rw at W̄(r, ii)); Alg. 1/2 lines 8-14 and Alg. 3/4
 * with K, R of PAPER.md:183. */
static void row_coefs(const or_problem* p, int jj, int nxu, int nxi, int nxv, double* av,
                      double* bv) {
  for (int i = 0; i < nxi; ++i) av[i] = p->dt / 2.0 * p->kappa[(size_t)(jj + 1) * nxu + i + 1];
  for (int i = 0; i < nxv; ++i) bv[i] = p->dt / 2.0 * p->rv[(size_t)jj * nxv + i];
}
static void col_coefs(const or_problem* p, int ii, int nxu, int nxi, int nyi, int nyv, double* av,
                      double* bv) {
  for (int r = 0; r < nyi; ++r) av[r] = p->dt / 2.0 * p->kappa[(size_t)(r + 1) * nxu + ii + 1];
  for (int r = 0; r < nyv; ++r) bv[r] = p->dt / 2.0 * p->rw[(size_t)r * nxi + ii];
}

/*
 * or_run: advance (U, V̄, W̄) by nsteps Peaceman–Rachford steps starting at
 * step index m0 (t = m0*dt).  One step is Alg. 1 / Alg. 2 body
 * (PAPER.md:155-171 / 288-306):
 *   a2  W* = W̄ - beta*D_y(U^m)  and  S1 = Ū^m - alpha*D̄_y(W̄^m) + dt/2 F^m
 *       (the A computation, line 8, in derivative form [G6]; W*, line 10 [G2,G14])
 *   a3  ADI-rows: K sweeps, U* boundary at t+dt/2 [G9], V0 = V^m (eq. 8)
 *   a4  S2 = U* - alpha*D̄_x(V*) + dt/2 F^{m+1} (C, line 12 [G3]);
 *       V^{m+1} = V* - beta*D_x(U*) (line 14 [G5])
 *   a6  ADI-columns: K sweeps, boundary g(t^{m+1}), W0 = W* [G7] (eq. 9)
 * alpha = kappa*dt/2, beta = dt/(2 rho), kappa = rho c^2 [G19].
 * Returns 0 or a negative error (-4 zero pivot, -2 no memory).
 */
int or_run(const or_problem* p, double* U, double* Vb, double* Wb, int m0, int nsteps,
           int nthreads) {
  const int method = p->method;
  axis_t ax, ay;
  int ncx = p->nx - 1, ncy = p->ny - 1; /* cells */
  int e = axis_init(&ax, method, ncx, p->h);
  if (e) return e;
  e = axis_init(&ay, method, ncy, p->h);
  if (e) { axis_free(&ax); return e; }
  const int nxu = ax.nub, nyu = ay.nub;   /* U array: nyu rows x nxu cols */
  const int nxi = ax.nu, nyi = ay.nu;     /* pressure interior */
  const int nxv = ax.nv, nyv = ay.nv;     /* V̄: nyi x nxv ; W̄: nyv x nxi */
  const double rho = p->rho, kappa = rho * p->c * p->c;
  const double dt = p->dt;
  const double alpha = kappa * dt / 2.0, beta = dt / (2.0 * rho);
  const int het = p->kappa != NULL;   /* f3: per-point alpha, beta (row_coefs / col_coefs) */
  size_t nS = (size_t)nyi * nxi, nW = (size_t)nyv * nxi;
  double* S1 = (double*)malloc(sizeof(double) * nS);
  double* S2 = (double*)malloc(sizeof(double) * nS);
  double* Ws = (double*)malloc(sizeof(double) * nW);
  if (!S1 || !S2 || !Ws) { free(S1); free(S2); free(Ws); axis_free(&ax); axis_free(&ay); return -2; }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  const int L = (nxu > nyu ? nxu : nyu) + 8;

  for (int st = 0; st < nsteps; ++st) {
    const int m = m0 + st;
    const double gf_m = tab(p->gf, p->ngf, 2 * m), gf_1 = tab(p->gf, p->ngf, 2 * m + 2);
    const double gb_h = tab(p->gb, p->ngb, 2 * m + 1), gb_1 = tab(p->gb, p->ngb, 2 * m + 2);

    /* ---- a2: explicit y-terms, per interior column (lines 8 and 10) ---- */
#pragma omp parallel
    {
      double* col = (double*)malloc(sizeof(double) * 6 * L);
      double *w = col + L, *t1 = col + 2 * L, *t2 = col + 3 * L;
      double *av = het ? col + 4 * L : NULL, *bv = het ? col + 5 * L : NULL;
#pragma omp for schedule(static)
      for (int ii = 0; ii < nxi; ++ii) {
        const int i = ii + 1; /* U column */
        for (int r = 0; r < nyu; ++r) col[r] = U[(size_t)r * nxu + i];
        for (int r = 0; r < nyv; ++r) w[r] = Wb[(size_t)r * nxi + ii];
        axis_D(&ay, col, t1);     /* D_y(U^m(:,i)), Dirichlet rows included */
        axis_Dbar(&ay, w, t2);    /* D̄_y(W̄^m(:,i)) */
        if (het) col_coefs(p, ii, nxu, nxi, nyi, nyv, av, bv);
        for (int r = 0; r < nyv; ++r) Ws[(size_t)r * nxi + ii] = w[r] - OR_B(r) * t1[r];
        for (int r = 0; r < nyi; ++r)
          S1[(size_t)r * nxi + ii] =
              col[r + 1] - OR_A(r) * t2[r] + (dt / 2.0) * source_at(p, nxi, r, ii, gf_m);
      }
      free(col);
    }

    /* ---- a3 + a4: ADI-rows (line 11) then C and V^{m+1} (lines 12, 14) ---- */
    int Kr = p->K;
    if (p->eps > 0.0) {  /* stopping rule: pass 1 over all lines to K sweeps */
      const int K1 = p->K + 1;
      double* lu = (double*)calloc((size_t)nyi * K1 * 2, sizeof(double));
      if (!lu) { free(S1); free(S2); free(Ws); axis_free(&ax); axis_free(&ay); return -2; }
      double* lv = lu + (size_t)nyi * K1;
#pragma omp parallel
      {
        double* buf = (double*)malloc(sizeof(double) * 10 * L);
        double *u = buf, *v = buf + L, *ub = buf + 2 * L, *tmp = buf + 3 * L, *s = buf + 4 * L,
               *v0 = buf + 5 * L, *uo = buf + 6 * L, *vo = buf + 7 * L;
        double *av = het ? buf + 8 * L : NULL, *bv = het ? buf + 9 * L : NULL;
#pragma omp for schedule(static)
        for (int jj = 0; jj < nyi; ++jj) {
          const int j = jj + 1;
          const double gL = (p->edges[2] ? p->edges[2][j] : 0.0) * gb_h;
          const double gR = (p->edges[3] ? p->edges[3][j] : 0.0) * gb_h;
          for (int i = 0; i < nxi; ++i) s[i] = S1[(size_t)jj * nxi + i];
          for (int i = 0; i < nxv; ++i) v0[i] = Vb[(size_t)jj * nxv + i];
          for (int i = 0; i < nxi; ++i) u[i] = 0.0;
          if (het) row_coefs(p, jj, nxu, nxi, nxv, av, bv);
          stage_line_norms(&ax, p->K, alpha, beta, av, bv, s, v0, gL, gR, u, v, ub, tmp, uo, vo,
                           lu + (size_t)jj * K1, lv + (size_t)jj * K1);
        }
        free(buf);
      }
      double* su = (double*)calloc((size_t)K1 * 2, sizeof(double));
      double* sv = su + K1;
      for (int jj = 0; jj < nyi; ++jj)          /* sums in line order */
        for (int k = 0; k < K1; ++k) { su[k] += lu[(size_t)jj * K1 + k]; sv[k] += lv[(size_t)jj * K1 + k]; }
      Kr = pick_k(su, sv, p->kmin, p->K, p->eps, p->tests ? p->tests + (size_t)(2 * st) * K1 : NULL);
      free(su); free(lu);
    }
    if (p->kchosen) p->kchosen[2 * st] = Kr;
#pragma omp parallel
    {
      double* buf = (double*)malloc(sizeof(double) * 8 * L);
      double *u = buf, *v = buf + L, *ub = buf + 2 * L, *tmp = buf + 3 * L, *s = buf + 4 * L,
             *v0 = buf + 5 * L;
      double *av = het ? buf + 6 * L : NULL, *bv = het ? buf + 7 * L : NULL;
#pragma omp for schedule(static)
      for (int jj = 0; jj < nyi; ++jj) {
        const int j = jj + 1; /* U row */
        const double gL = (p->edges[2] ? p->edges[2][j] : 0.0) * gb_h;
        const double gR = (p->edges[3] ? p->edges[3][j] : 0.0) * gb_h;
        for (int i = 0; i < nxi; ++i) s[i] = S1[(size_t)jj * nxi + i];
        for (int i = 0; i < nxv; ++i) v0[i] = Vb[(size_t)jj * nxv + i];
        if (het) row_coefs(p, jj, nxu, nxi, nxv, av, bv);
        stage_line(&ax, Kr, alpha, beta, av, bv, s, v0, gL, gR, u, v, ub, tmp);
        /* C / S2 = U* - alpha D̄_x(V*) + dt/2 F^{m+1} */
        axis_Dbar(&ax, v, tmp);
        for (int i = 0; i < nxi; ++i)
          S2[(size_t)jj * nxi + i] =
              u[i] - OR_A(i) * tmp[i] + (dt / 2.0) * source_at(p, nxi, jj, i, gf_1);
        /* V^{m+1} = V* - beta D_x([g(t+dt/2), U*, g(t+dt/2)]) */
        ub[0] = gL;
        for (int i = 0; i < nxi; ++i) ub[i + 1] = u[i];
        ub[nxu - 1] = gR;
        axis_D(&ax, ub, tmp);
        for (int i = 0; i < nxv; ++i) Vb[(size_t)jj * nxv + i] = v[i] - OR_B(i) * tmp[i];
      }
      free(buf);
    }

    /* ---- a6: ADI-columns (line 15), boundary at t^{m+1} ---- */
    int Kc = p->K;
    if (p->eps > 0.0) {  /* stopping rule: pass 1 over all columns to K sweeps */
      const int K1 = p->K + 1;
      double* lu = (double*)calloc((size_t)nxi * K1 * 2, sizeof(double));
      if (!lu) { free(S1); free(S2); free(Ws); axis_free(&ax); axis_free(&ay); return -2; }
      double* lw = lu + (size_t)nxi * K1;
#pragma omp parallel
      {
        double* buf = (double*)malloc(sizeof(double) * 10 * L);
        double *u = buf, *w = buf + L, *ub = buf + 2 * L, *tmp = buf + 3 * L, *s = buf + 4 * L,
               *w0 = buf + 5 * L, *uo = buf + 6 * L, *wo = buf + 7 * L;
        double *av = het ? buf + 8 * L : NULL, *bv = het ? buf + 9 * L : NULL;
#pragma omp for schedule(static)
        for (int ii = 0; ii < nxi; ++ii) {
          const int i = ii + 1;
          const double gB = (p->edges[0] ? p->edges[0][i] : 0.0) * gb_1;
          const double gT = (p->edges[1] ? p->edges[1][i] : 0.0) * gb_1;
          for (int r = 0; r < nyi; ++r) s[r] = S2[(size_t)r * nxi + ii];
          for (int r = 0; r < nyv; ++r) w0[r] = Ws[(size_t)r * nxi + ii];
          for (int r = 0; r < nyi; ++r) u[r] = 0.0;
          if (het) col_coefs(p, ii, nxu, nxi, nyi, nyv, av, bv);
          stage_line_norms(&ay, p->K, alpha, beta, av, bv, s, w0, gB, gT, u, w, ub, tmp, uo, wo,
                           lu + (size_t)ii * K1, lw + (size_t)ii * K1);
        }
        free(buf);
      }
      double* su = (double*)calloc((size_t)K1 * 2, sizeof(double));
      double* sw = su + K1;
      for (int ii = 0; ii < nxi; ++ii)
        for (int k = 0; k < K1; ++k) { su[k] += lu[(size_t)ii * K1 + k]; sw[k] += lw[(size_t)ii * K1 + k]; }
      Kc = pick_k(su, sw, p->kmin, p->K, p->eps, p->tests ? p->tests + (size_t)(2 * st + 1) * K1 : NULL);
      free(su); free(lu);
    }
    if (p->kchosen) p->kchosen[2 * st + 1] = Kc;
#pragma omp parallel
    {
      double* buf = (double*)malloc(sizeof(double) * 8 * L);
      double *u = buf, *w = buf + L, *ub = buf + 2 * L, *tmp = buf + 3 * L, *s = buf + 4 * L,
             *w0 = buf + 5 * L;
      double *av = het ? buf + 6 * L : NULL, *bv = het ? buf + 7 * L : NULL;
#pragma omp for schedule(static)
      for (int ii = 0; ii < nxi; ++ii) {
        const int i = ii + 1;
        const double gB = (p->edges[0] ? p->edges[0][i] : 0.0) * gb_1;
        const double gT = (p->edges[1] ? p->edges[1][i] : 0.0) * gb_1;
        for (int r = 0; r < nyi; ++r) s[r] = S2[(size_t)r * nxi + ii];
        for (int r = 0; r < nyv; ++r) w0[r] = Ws[(size_t)r * nxi + ii];
        if (het) col_coefs(p, ii, nxu, nxi, nyi, nyv, av, bv);
        stage_line(&ay, Kc, alpha, beta, av, bv, s, w0, gB, gT, u, w, ub, tmp);
        for (int r = 0; r < nyi; ++r) U[(size_t)(r + 1) * nxu + i] = u[r];
        for (int r = 0; r < nyv; ++r) Wb[(size_t)r * nxi + ii] = w[r];
      }
      free(buf);
    }
    /* Dirichlet data of U^{m+1} */
    for (int i = 0; i < nxu; ++i) {
      U[i] = (p->edges[0] ? p->edges[0][i] : 0.0) * gb_1;
      U[(size_t)(nyu - 1) * nxu + i] = (p->edges[1] ? p->edges[1][i] : 0.0) * gb_1;
    }
    for (int r = 0; r < nyu; ++r) {
      U[(size_t)r * nxu] = (p->edges[2] ? p->edges[2][r] : 0.0) * gb_1;
      U[(size_t)r * nxu + nxu - 1] = (p->edges[3] ? p->edges[3][r] : 0.0) * gb_1;
    }
  }
  free(S1); free(S2); free(Ws);
  axis_free(&ax); axis_free(&ay);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT row f4: the full-matrix CFD variant with a Cerjan absorbing layer.   */
/* "By simply replacing reduced operators P̄ and Q̄, and reduced */
/* matrices Ū, V̄, W̄, by their full matrix versions in previous formulation  */
/* steps [...] the boundary wave fields can be also obtained.  These values  */
/* can be further damped by the absorbing technique proposed in [Cerjan]."   */
/* Readings (F1-F2):                                            */
/*  F1  every node is unknown (U, V, W all ny x nx, no Dirichlet data); both   */
/*      the pressure and the velocity derivatives are D = P^{-1} Q (full,     */
/*      n+1 rows, App. A), in both directions; otherwise Alg. 1 / Alg. 3 in   */
/*      their order: a2 W* = W - beta D_y U, S1 = U - alpha D_y W + dt/2 F^m;  */
/*      rows: K sweeps u = S1 - alpha D_x v, v = V - beta D_x u; a4 S2 = u -   */
/*      alpha D_x v + dt/2 F^{m+1}, V^{m+1} = v - beta D_x u; columns: K       */
/*      sweeps u = S2 - alpha D_y w, w = W* - beta D_y u.                      */
/*  F2  after each step U, V, W are multiplied by G(x) G(y), G(k) =            */
/*      exp(-(a (nb - d_k))^2) for d_k = min(k, n - k) < nb, else 1 (the      */
/*      Cerjan et al. 1985 taper; nb, a are parameters).                       */
/* phi (if set) is on all nodes (ny x nx); a point source at U index (ix,iy). */
/* ------------------------------------------------------------------------ */
static void stage_line_full(const axis_t* a, int K, double alpha, double beta, const double* s,
                            const double* v0, double* u, double* v, double* tmp) {
  const int n1 = a->nv; /* n + 1 */
  for (int i = 0; i < n1; ++i) v[i] = v0[i];
  for (int k = 0; k < K; ++k) {
    axis_D(a, v, tmp);
    for (int i = 0; i < n1; ++i) u[i] = s[i] - alpha * tmp[i];
    axis_D(a, u, tmp);
    for (int i = 0; i < n1; ++i) v[i] = v0[i] - beta * tmp[i];
  }
}

static double cerjan(int k, int n, int nb, double a) {
  const int d = k < n - k ? k : n - k;
  if (d >= nb) return 1.0;
  const double t = a * (double)(nb - d);
  return exp(-t * t);
}

static double source_full(const or_problem* p, int nx, int j, int i, double gft) {
  double f = 0.0;
  if (p->phi) f += p->phi[(size_t)j * nx + i] * gft;
  if (p->src_ix >= 0 && p->src_iy >= 0 && i == p->src_ix && j == p->src_iy) f += gft / (p->h * p->h);
  return f;
}

int or_run_full(const or_problem* p, double* U, double* V, double* W, int m0, int nsteps, int nthreads,
                int nb, double ca) {
  axis_t ax, ay;
  int e = axis_init(&ax, OR_CFD, p->nx - 1, p->h);
  if (e) return e;
  e = axis_init(&ay, OR_CFD, p->ny - 1, p->h);
  if (e) { axis_free(&ax); return e; }
  const int nx = p->nx, ny = p->ny;
  const double rho = p->rho, kappa = rho * p->c * p->c, dt = p->dt;
  const double alpha = kappa * dt / 2.0, beta = dt / (2.0 * rho);
  const size_t nn = (size_t)nx * ny;
  double* S1 = (double*)malloc(sizeof(double) * nn);
  double* S2 = (double*)malloc(sizeof(double) * nn);
  double* Ws = (double*)malloc(sizeof(double) * nn);
  if (!S1 || !S2 || !Ws) { free(S1); free(S2); free(Ws); axis_free(&ax); axis_free(&ay); return -2; }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  const int L = (nx > ny ? nx : ny) + 8;
  for (int st = 0; st < nsteps; ++st) {
    const int m = m0 + st;
    const double gf_m = tab(p->gf, p->ngf, 2 * m), gf_1 = tab(p->gf, p->ngf, 2 * m + 2);
    /* a2, per column */
#pragma omp parallel
    {
      double* buf = (double*)malloc(sizeof(double) * 4 * L);
      double *col = buf, *w = buf + L, *t1 = buf + 2 * L, *t2 = buf + 3 * L;
#pragma omp for schedule(static)
      for (int i = 0; i < nx; ++i) {
        for (int r = 0; r < ny; ++r) { col[r] = U[(size_t)r * nx + i]; w[r] = W[(size_t)r * nx + i]; }
        axis_D(&ay, col, t1);
        axis_D(&ay, w, t2);
        for (int r = 0; r < ny; ++r) {
          Ws[(size_t)r * nx + i] = w[r] - beta * t1[r];
          S1[(size_t)r * nx + i] = col[r] - alpha * t2[r] + (dt / 2.0) * source_full(p, nx, r, i, gf_m);
        }
      }
      free(buf);
    }
    /* rows (all of them), then C and V^{m+1} */
#pragma omp parallel
    {
      double* buf = (double*)malloc(sizeof(double) * 4 * L);
      double *u = buf, *v = buf + L, *tmp = buf + 2 * L, *t2 = buf + 3 * L;
#pragma omp for schedule(static)
      for (int j = 0; j < ny; ++j) {
        stage_line_full(&ax, p->K, alpha, beta, S1 + (size_t)j * nx, V + (size_t)j * nx, u, v, tmp);
        axis_D(&ax, v, tmp);
        axis_D(&ax, u, t2);
        for (int i = 0; i < nx; ++i) {
          S2[(size_t)j * nx + i] = u[i] - alpha * tmp[i] + (dt / 2.0) * source_full(p, nx, j, i, gf_1);
          V[(size_t)j * nx + i] = v[i] - beta * t2[i];
        }
      }
      free(buf);
    }
    /* columns (all of them) */
#pragma omp parallel
    {
      double* buf = (double*)malloc(sizeof(double) * 5 * L);
      double *u = buf, *w = buf + L, *tmp = buf + 2 * L, *s = buf + 3 * L, *w0 = buf + 4 * L;
#pragma omp for schedule(static)
      for (int i = 0; i < nx; ++i) {
        for (int r = 0; r < ny; ++r) { s[r] = S2[(size_t)r * nx + i]; w0[r] = Ws[(size_t)r * nx + i]; }
        stage_line_full(&ay, p->K, alpha, beta, s, w0, u, w, tmp);
        for (int r = 0; r < ny; ++r) { U[(size_t)r * nx + i] = u[r]; W[(size_t)r * nx + i] = w[r]; }
      }
      free(buf);
    }
    /* F2: Cerjan taper of all three fields */
    if (nb > 0) {
      for (int r = 0; r < ny; ++r) {
        const double gy = cerjan(r, ny - 1, nb, ca);
        for (int i = 0; i < nx; ++i) {
          const double g = gy * cerjan(i, nx - 1, nb, ca);
          U[(size_t)r * nx + i] *= g;
          V[(size_t)r * nx + i] *= g;
          W[(size_t)r * nx + i] *= g;
        }
      }
    }
  }
  free(S1); free(S2); free(Ws);
  axis_free(&ax); axis_free(&ay);
  return 0;
}

int or_run_full_flat(int nx, int ny, double h, double dt, double c, double rho, int K, const double* phi,
                     int src_ix, int src_iy, const double* gf, int ngf, double* U, double* V, double* W,
                     int m0, int nsteps, int nthreads, int nb, double ca) {
  or_problem p;
  memset(&p, 0, sizeof p);
  p.method = OR_CFD; p.nx = nx; p.ny = ny; p.K = K;
  p.h = h; p.dt = dt; p.c = c; p.rho = rho;
  p.phi = phi; p.src_ix = src_ix; p.src_iy = src_iy;
  p.gf = gf; p.ngf = ngf;
  if (nx < 9 || ny < 9 || K < 1 || m0 < 0 || nsteps < 0 || nb < 0 || 2 * nb > nx || 2 * nb > ny) return -1;
  if (gf && ngf < 2 * (m0 + nsteps) + 1) return -1;
  return or_run_full(&p, U, V, W, m0, nsteps, nthreads, nb, ca);
}

/* One full-variant stage on a single line (exported for the dense-solve pin). */
int or_stage_line_full(int n, double h, int K, double alpha, double beta, const double* s, const double* v0,
                       double* u, double* v) {
  axis_t a;
  int e = axis_init(&a, OR_CFD, n, h);
  if (e) return e;
  double* tmp = (double*)malloc(sizeof(double) * (n + 8));
  stage_line_full(&a, K, alpha, beta, s, v0, u, v, tmp);
  free(tmp);
  axis_free(&a);
  return 0;
}

/* Flat-argument wrapper for ctypes. */
int or_run_flat(int method, int nx, int ny, double h, double dt, double c, double rho, int K,
                const double* phi, int src_ix, int src_iy, const double* gf, int ngf,
                const double* ey0, const double* ey1, const double* ex0, const double* ex1,
                const double* gb, int ngb, double* U, double* Vb, double* Wb, int m0,
                int nsteps, int nthreads, double eps, int kmin, int* kchosen, double* tests,
                const double* kappa, const double* rv, const double* rw) {
  or_problem p;
  if ((kappa != NULL) != (rv != NULL) || (kappa != NULL) != (rw != NULL)) return -1;
  p.kappa = kappa; p.rv = rv; p.rw = rw;
  p.method = method; p.nx = nx; p.ny = ny; p.K = K;
  p.eps = eps; p.kmin = kmin; p.kchosen = kchosen; p.tests = tests;
  if (eps > 0.0 && (kmin < 2 || kmin > K)) return -1;
  p.h = h; p.dt = dt; p.c = c; p.rho = rho;
  p.phi = phi; p.src_ix = src_ix; p.src_iy = src_iy;
  p.gf = gf; p.ngf = ngf;
  p.edges[0] = ey0; p.edges[1] = ey1; p.edges[2] = ex0; p.edges[3] = ex1;
  p.gb = gb; p.ngb = ngb;
  if (nx < 9 || ny < 9 || K < 1 || m0 < 0 || nsteps < 0) return -1;
  /* the time tables must cover t^{m0} .. t^{m0+nsteps} at half steps */
  if (gf && ngf < 2 * (m0 + nsteps) + 1) return -1;
  if (gb && ngb < 2 * (m0 + nsteps) + 1) return -1;
  return or_run(&p, U, Vb, Wb, m0, nsteps, nthreads);
}

/* One ADI stage on a single line (exported for the dense-LU stage pin). */
int or_stage_line(int method, int n, double h, int K, double alpha, double beta,
                  const double* av, const double* bv, const double* s, const double* v0, double gL, double gR,
                  double* u, double* v) {
  axis_t a;
  int e = axis_init(&a, method, n, h);
  if (e) return e;
  double* ub = (double*)malloc(sizeof(double) * 2 * (n + 8));
  stage_line(&a, K, alpha, beta, av, bv, s, v0, gL, gR, u, v, ub, ub + n + 8);
  free(ub);
  axis_free(&a);
  return 0;
}

/* LU factors of P (which=0) or P̄ (which=1) for n cells (pivot pins). */
int or_cfd_factors(int n, int which, double* l, double* d) {
  cfd_ops o;
  int e = cfd_ops_init(&o, n, 1.0);
  if (e) return e;
  if (which == 0) { memcpy(l, o.Pl, sizeof(double) * (n + 1)); memcpy(d, o.Pd, sizeof(double) * (n + 1)); }
  else { memcpy(l, o.Bl, sizeof(double) * (n - 1)); memcpy(d, o.Bd, sizeof(double) * (n - 1)); }
  cfd_ops_free(&o);
  return 0;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
