/*
 * ipm_oracle.h — plain, slow, fp64 CPU oracle of the IPM hot path of
 * Kusch, Wolters, Frank, arXiv 1912.09238 ("PAPER.md" below).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1912_09238_b200/csrc, include/ipm.h).
 *
 * Every function follows the paper's definitions literally: plain loops, no
 * blocking, no fusion, full n x n Hessians, textbook Cholesky.  Where the paper
 * is silent or garbled the reading used is the one listed in DESIGN.md
 * ("Readings"), which is SURVEY.md §8(c) verbatim.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without a pin say
 * "parity unpinned" in their comment (also listed in DESIGN.md).
 */
#ifndef IPM_ORACLE_H
#define IPM_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* closures (App. B) */
enum { ORC_CL_QUADRATIC = 0, ORC_CL_BARRIER = 1, ORC_CL_EULER = 2 };
/* deterministic two-point fluxes g */
enum { ORC_FLUX_LF_GLOBAL = 0, ORC_FLUX_HLL = 1, ORC_FLUX_RUSANOV = 2 };
/* meshes */
enum { ORC_MESH_1D = 0, ORC_MESH_CART2D = 1, ORC_MESH_TRI = 2 };
/* boundary conditions (ghost states at quadrature nodes, reading 16) */
enum { ORC_BC_TRANSMISSIVE = 0, ORC_BC_STATE = 1, ORC_BC_SLIP = 2, ORC_BC_FARFIELD = 3 };
/* characteristic far-field ghost (reading 37): ui interior, uf free stream, n outward unit normal */
void orc_farfield_ghost(double gamma, const double *ui, const double *uf, const double *n, double *ug);
/* state specs (primitive states, possibly xi-dependent) */
enum { ORC_SPEC_AFFINE = 0, ORC_SPEC_FREESTREAM = 1 };
/* IC kinds */
enum { ORC_IC_UNIFORM = 0, ORC_IC_STEP1D = 1, ORC_IC_QUAD2D = 2 };
/* Newton modes / update forms */
enum { ORC_NEWTON_FULL = 0, ORC_NEWTON_ONE_STEP = 1 };
enum { ORC_UPDATE_CONSERVATIVE = 0, ORC_UPDATE_PAPER_C = 1 };
/* per-cell dual-solve status */
enum { ORC_OK = 0, ORC_NONCONVERGENCE = 1, ORC_ILLCONDITIONED = 2, ORC_LINESEARCH = 3, ORC_INADMISSIBLE = 4 };

/* A primitive state as a function of xi.
 *   AFFINE:     q_c(xi) = q0[c] + sum_d q1[c][d] xi_d, primitive components
 *               scalar: (u);  Euler d=1: (rho, v, p);  Euler d=2: (rho, vx, vy, p)
 *   FREESTREAM: rho=q0[0], p=q0[1], Ma = q0[2] + q0[3] xi_{dim_a},
 *               theta(deg) = q0[4] + q0[5] xi_{dim_b}; v = Ma c (cos th, sin th). */
typedef struct {
  int32_t kind;
  int32_t dim_a, dim_b;
  int32_t pad;
  double q0[6];
  double q1[5][3];
} orc_state_spec;

typedef struct {
  /* random space: total degree basis, tensor Gauss-Legendre rule */
  int32_t p, M, q1d;
  /* physics */
  int32_t m, closure, flux;
  double gamma;          /* Euler */
  double umin, umax;     /* barrier */
  /* mesh */
  int32_t mesh_kind;
  int32_t nx, ny;
  int32_t n_vert, n_tri;
  int32_t periodic;          /* 1D / cart: wrap neighbours (conservation pin) */
  double x0, x1, y0, y1;
  const double *vert;        /* [n_vert][2] */
  const int32_t *tri;        /* [n_tri][3], counter-clockwise */
  const int32_t *tri_tag;    /* [n_tri][3]: edge e=(v_e,v_{e+1}) tag, -1 interior */
  /* boundary: index = side (1D: 0 left,1 right; cart: 0 left,1 right,2 bottom,3 top) or tri tag */
  int32_t bc_kind[4];
  orc_state_spec bc_state[4];
  /* Newton */
  double tau, armijo_c;
  int32_t max_newton, max_halvings;
  int32_t newton_mode, update_form;
  double cfl;
  /* adaptivity: n_levels==0 -> off */
  int32_t n_levels;
  int32_t level_M[8];
  int32_t pad1;
  double delta_dec, delta_inc;
  int32_t n_threads;         /* OpenMP threads, 0 = default */
  /* refinement retardation (Alg. 4): stage l caps the level index at
   * retard_level[l] until the steady residual falls below retard_eps[l]; past the last stage no cap.
   * n_retard == 0 -> off (reading 31: Alg. 4's max{., l*} is a cap, min) */
  int32_t n_retard;
  int32_t retard_level[8];
  double retard_eps[8];
  /* quadrature (reading 33): 0 tensor Gauss-Legendre with q1d points per
   * dimension, 1 tensor Clenshaw-Curtis with q1d points, 2 Smolyak sparse grid of nested
   * Clenshaw-Curtis rules of level quad_level */
  int32_t quad_kind, quad_level;
  /* dual-solve direction (reading 35): 0 exact Newton (the
   * Hessian of PAPER.md:169), 1 limited-memory BFGS with the lbfgs_m most recent (s, y) pairs of
   * every cell kept across (pseudo-)time steps and the initial matrix I (x) Jbar^{-1} */
  int32_t hessian_kind, lbfgs_m;
  /* per-level nested quadrature (reading 36): level_q1d[l] > 0
   * gives level l its own tensor Clenshaw-Curtis rule of level_q1d[l] = 2^k + 1 points per dimension,
   * nested in the finest one (quad_kind 1, q1d = level_q1d[n_levels-1]); 0 = one rule for all levels */
  int32_t level_q1d[8];
} orc_problem;

typedef struct {
  int32_t kind;
  int32_t pad;
  double xs0, xs1[3];        /* split x_s(xi) = xs0 + sum_d xs1[d] xi_d */
  double ys0, ys1[3];
  orc_state_spec state[4];   /* STEP1D: left,right; QUAD2D: NE,NW,SW,SE; UNIFORM: [0] */
} orc_ic;

typedef struct orc_ctx orc_ctx;

orc_ctx *orc_create(const orc_problem *P);
size_t orc_problem_size(void); /* sizeof(orc_problem) (binding check) */
int orc_retard_stage(const orc_ctx *c); /* refinement retardation stage (Alg. 4) */
/* Stochastic Collocation: node states U [cells][Q][m] */
void orc_sc_init(const orc_ctx *c, const orc_ic *ic, double *U);
double orc_sc_step(const orc_ctx *c, const double *U, double *Unew, double t_remaining, double *residual);
void orc_sc_moments(const orc_ctx *c, const double *U, double *uhat);
void orc_destroy(orc_ctx *c);
/* sizes */
int orc_N(const orc_ctx *c);
int orc_Q(const orc_ctx *c);
int orc_cells(const orc_ctx *c);

/* random space */
void orc_gauss_legendre(int q, double *x, double *w);
int orc_num_basis(int p, int M);
/* Clenshaw-Curtis nodes x_j = -cos(pi j/(n-1)) (ascending) and weights (sum 2) */
void orc_clenshaw_curtis(int n, double *x, double *w);
/* Smolyak sparse grid of nested Clenshaw-Curtis rules (level L >= p, dimension p): number of points,
 * and (when xi/w are non-NULL) points [Q][p] in lexicographic order of their finest-grid indices,
 * weights summing to 2^p */
int orc_smolyak_cc(int p, int L, double *xi, double *w);
void orc_multi_indices(int p, int M, int32_t *idx);
void orc_get_quadrature(const orc_ctx *c, double *xi, double *omega, double *Phi);
void orc_get_geometry(const orc_ctx *c, int32_t *nbr, double *nrm, double *coef, double *area);

/* closures (App. B) — single node */
int orc_closure_u(const orc_ctx *c, const double *Lam, double *u);
int orc_closure_du(const orc_ctx *c, const double *Lam, double *J);
double orc_closure_sstar(const orc_ctx *c, const double *Lam);
int orc_closure_grad_s(const orc_ctx *c, const double *u, double *Lam);
/* App. B in the paper's own scaling, misprints corrected (readings 9, 10) */
void orc_euler_paper_grad_s(double gamma, int d, const double *u, double *Lam);
int orc_euler_paper_u(double gamma, int d, const double *Lam, double *u);

/* dual problem for one cell at level N_l */
int orc_dual_objective(const orc_ctx *c, int Nl, const double *lam, const double *uhat, double *L);
int orc_dual_gradient(const orc_ctx *c, int Nl, const double *lam, const double *uhat, double *g);
int orc_dual_hessian(const orc_ctx *c, int Nl, const double *lam, double *H);
int orc_dual_solve_cell(const orc_ctx *c, int Nl, int mode, const double *uhat, double *lam,
                        int32_t *iters, double *crit);
/* h(lambda) = <u_s(lambda^T phi) phi^T>_Q^T */
int orc_moments_from_dual(const orc_ctx *c, int Nl, const double *lam, double *uhat);
/* L-BFGS (reading 35): direction d = -H g of the two-loop recursion over cnt pairs (S, Y: [cnt][n],
 * newest first) with H0 = I (x) Jbar(lam)^{-1}; returns 0 if Jbar is not SPD or lam inadmissible */
int orc_lbfgs_direction(const orc_ctx *c, int Nl, const double *lam, const double *g, const double *S,
                        const double *Y, int cnt, double *d);
/* Jbar(lam) = sum_k omega_k grad u_s(lam^T phi(xi_k))  [m][m] */
int orc_lbfgs_jbar(const orc_ctx *c, int Nl, const double *lam, double *Jbar);
/* history of cell j: pairs (newest first) into S, Y [lbfgs_m][N m] (nullable); returns the count */
int orc_lbfgs_history(const orc_ctx *c, int j, double *S, double *Y);
void orc_lbfgs_reset(orc_ctx *c);
/* per-level nested rule of level l (reading 36): its node indices into the finest rule kf [Q_l] and
 * weights w [Q_l] (nullable); returns Q_l (the whole rule when per-level rules are off) */
int orc_level_rule(const orc_ctx *c, int l, int32_t *kf, double *w);

/* two-point flux at one node; dx_over_dt for global LF */
void orc_flux_g(const orc_ctx *c, const double *ul, const double *ur, const double *n,
                double dx_over_dt, double *g);

/* whole-field operations, arrays [cells][N][m] (N = N_max) */
void orc_project_ic(const orc_ctx *c, const orc_ic *ic, double *uhat);
void orc_warm_start(const orc_ctx *c, const double *uhat, double *lam);
void orc_set_levels(orc_ctx *c, const int32_t *levels);
/* smoothness indicator S_l on the first state of h [N][m] at level index lvl */
double orc_indicator(const orc_ctx *c, int lvl, const double *h);
void orc_get_levels(const orc_ctx *c, int32_t *levels);
/* as orc_dual_solve_all, plus per cell the rejected line-search trials and the inadmissible ones */
void orc_dual_solve_all_ls(const orc_ctx *c, const double *uhat, double *lam, int32_t *iters,
                           int32_t *status, double *crit, int32_t *halvings, int32_t *inadmissible);
void orc_dual_solve_all(const orc_ctx *c, const double *uhat, double *lam, int32_t *iters,
                        int32_t *status, double *crit);
double orc_compute_dt(const orc_ctx *c, const double *lam, double t_remaining);
/* per-cell CFL rate (largest wave speed x mesh factor, incl. boundary ghost states); dt = CFL / max */
void orc_cell_rates(const orc_ctx *c, const double *lam, double *rates);
void orc_flux_update(orc_ctx *c, const double *lam, const double *uhat_old, double *uhat_new,
                     double dt);
/* one step of Algorithm 1 / 2 / 3: dual solve, [levels], dt, moment update.
 * returns worst status; writes dt used and (steady) zeroth-moment residual. */
int orc_step(orc_ctx *c, double *uhat, double *lam, double t_remaining, int32_t *iters,
             int32_t *status, double *dt_used, double *residual);

#ifdef __cplusplus
}
#endif
#endif
