/*
 * ipm.h — C-ABI of libipm: the B200 (sm_100a) hot path of the Intrusive Polynomial Moment
 * method, Kusch, Wolters, Frank, arXiv 1912.09238 ("PAPER.md:n" = line n of the paper source).
 *
 * The path, per (pseudo-)time step (Algorithm 1; Algorithm 2, PAPER.md:252-269;
 * Algorithm 3):
 *   1. per spatial cell j, Newton iteration on the convex dual problem
 *        lambda_j = argmin L(lambda; uhat_j),  L = <s_*(lambda^T phi)>_Q - sum_i lambda_i^T uhat_i
 *      (PAPER.md:155-180), to ||grad L|| < tau (FULL) or one step (ONE_STEP),
 *      optionally choosing the cell's next polynomial degree;
 *   2. CFL time step from the reconstructed states u_s(lambda^T phi(xi_k));
 *   3. kinetic-flux finite-volume moment update.
 *
 * Conventions (all entry points):
 *   - d_* arguments are DEVICE pointers on the context's device, caller-owned, contiguous,
 *     fp64 unless stated.  Moment / dual arrays are [cells][N][m] row-major (m fastest),
 *     N = binom(M+p, p) the full basis size; cell order: 1D j; cartesian iy*nx+ix; tri = triangle id.
 *     With adaptivity entries above a cell's level are zero.
 *   - h_* arguments are HOST pointers.
 *   - Calls are asynchronous on the stream given in ipm_config.stream (NULL = legacy default
 *     stream) unless documented as synchronous.  They return IPM_ERR_ARG for invalid arguments,
 *     IPM_ERR_CUDA for launch/runtime errors; per-cell numerical outcomes are written to per-cell
 *     status arrays (ipm_cell_status), never returned by the asynchronous calls.
 *   - The context allocates all its device memory in ipm_init and nothing afterwards.
 *   - One context per device and thread; not thread-safe.
 *   - There is no CPU fallback: without a CUDA device ipm_init returns IPM_ERR_CUDA.
 */
#ifndef IPM_H
#define IPM_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define IPM_API __attribute__((visibility("default")))
#else
#define IPM_API
#endif

typedef struct ipm_ctx ipm_ctx;

typedef enum {
  IPM_OK = 0,
  IPM_ERR_ARG = 1,
  IPM_ERR_CUDA = 2,
  IPM_ERR_NCCL = 3,
  IPM_ERR_UNSUPPORTED = 4, /* size/closure combination not compiled in */
  IPM_ERR_NUMERIC = 5      /* a synchronous call found failed cells (see ipm_cell_status) */
} ipm_status;

/* per-cell outcome of the dual solve (readings 3', 4, 5 in DESIGN.md) */
typedef enum {
  IPM_CELL_OK = 0,
  IPM_CELL_NONCONVERGENCE = 1,     /* max_newton iterations without ||grad L|| < tau */
  IPM_CELL_ILLCONDITIONED = 2,     /* Cholesky of the dual Hessian found a pivot <= 0 / non-finite */
  IPM_CELL_LINESEARCH = 3,         /* Armijo backtracking exhausted max_halvings */
  IPM_CELL_INADMISSIBLE = 4        /* the starting lambda reconstructs a non-admissible state */
} ipm_cell_status;

/* entropy closures: u_s = (grad s)^{-1} */
typedef enum {
  IPM_CLOSURE_QUADRATIC = 0, /* s = |u|^2/2, IPM == stochastic Galerkin */
  IPM_CLOSURE_BARRIER = 1,   /* scalar, u(L) = u- + (u+ - u-)/(1+exp(-L)) (BASELINE cfg 1) */
  IPM_CLOSURE_EULER = 2      /* U = -rho S/(gamma-1) (BASELINE cfg 2; App. B up to scaling) */
} ipm_closure;

/* deterministic two-point fluxes g(u_l, u_r) used inside the kinetic flux */
typedef enum {
  IPM_FLUX_LF_GLOBAL = 0, /* scalar Burgers: (u_l^2+u_r^2)/4 - dx/(2dt)(u_r-u_l) */
  IPM_FLUX_HLL = 1,       /* Euler 1D, Davis wave speeds */
  IPM_FLUX_RUSANOV = 2    /* Euler, local Lax-Friedrichs along the face normal */
} ipm_flux;

typedef enum { IPM_MESH_1D = 0, IPM_MESH_CART2D = 1, IPM_MESH_TRI = 2 } ipm_mesh_kind;
/* IPM_BC_FARFIELD: characteristic far-field ghost (reading 37) from the
 * interior node state and the free stream bc_state: Riemann invariants along the outward normal.
 * Triangle meshes with m = 4 only (ipm_init returns IPM_ERR_ARG otherwise); the CFL rate takes the
 * free-stream state at such faces. */
typedef enum { IPM_BC_TRANSMISSIVE = 0, IPM_BC_STATE = 1, IPM_BC_SLIP = 2, IPM_BC_FARFIELD = 3 } ipm_bc_kind;
typedef enum { IPM_NEWTON_FULL = 0, IPM_NEWTON_ONE_STEP = 1 } ipm_newton_mode;
typedef enum { IPM_UPDATE_CONSERVATIVE = 0, IPM_UPDATE_PAPER_C = 1 } ipm_update_form;
typedef enum { IPM_IC_UNIFORM = 0, IPM_IC_STEP1D = 1, IPM_IC_QUAD2D = 2 } ipm_ic_kind;

/* A primitive state as a function of the random vector xi.
 *   kind 0 (affine):     q_c(xi) = q0[c] + sum_d q1[c][d] xi_d; components (u) | (rho,v,p) | (rho,vx,vy,p)
 *   kind 1 (freestream): rho = q0[0], p = q0[1], Mach = q0[2] + q0[3] xi[dim_a],
 *                        angle(deg) = q0[4] + q0[5] xi[dim_b], v = Mach c (cos, sin). */
typedef struct {
  int32_t kind, dim_a, dim_b, reserved;
  double q0[6];
  double q1[5][3];
} ipm_state;

typedef struct {
  /* random space: total-degree Legendre basis, tensor Gauss-Legendre rule */
  int32_t p, M, q1d;
  /* physics */
  int32_t m;                 /* states per node: 1 (scalar), 3 (Euler 1D), 4 (Euler 2D) */
  int32_t closure, flux;
  double gamma;              /* Euler */
  double u_minus, u_plus;    /* barrier bounds */
  /* mesh (the full, global mesh) */
  int32_t mesh_kind, nx, ny, periodic;
  double x0, x1, y0, y1;
  int32_t n_vert, n_tri;
  const double *h_vert;      /* [n_vert][2] */
  const int32_t *h_tri;      /* [n_tri][3] counter-clockwise */
  const int32_t *h_tri_tag;  /* [n_tri][3] boundary tag of edge (v_e, v_e+1), -1 interior */
  /* boundary conditions, indexed by side (1D: 0 left, 1 right; cart: 0 left, 1 right, 2 bottom,
   * 3 top) or by triangle edge tag */
  int32_t bc_kind[4];
  ipm_state bc_state[4];
  /* Newton */
  double tau, armijo_c;
  int32_t max_newton, max_halvings;
  int32_t newton_mode, update_form;
  double cfl;
  /* adaptivity: n_levels = 0 -> off; level_M ascending, level_M[n_levels-1] == M */
  int32_t n_levels;
  int32_t level_M[8];
  double delta_dec, delta_inc;
  /* distribution: the context owns part (rank) of a px x py block decomposition (cartesian)
   * or of the Morton-ordered cell list (tri); nranks = 1 -> whole mesh */
  int32_t rank, nranks, px, py;
  const void *reserved_ptr;  /* unused (the exchange is performed by the caller) */
  void *stream;              /* cudaStream_t */
  /* refinement retardation (Algorithm 4; n_levels > 0): stage l caps every
   * cell's level index at retard_level[l] until the steady residual of a step falls below
   * retard_eps[l], then the next stage applies; past the last stage no cap.  n_retard = 0 -> off.
   * Reading 31: Algorithm 4's max{DetermineRefinementLevel, l*_l} is read as the cap
   * min{.} the text describes ("maximal refinement levels"). */
  int32_t n_retard;
  int32_t retard_level[8];
  double retard_eps[8];
  /* quadrature (reading 33): 0 tensor Gauss-Legendre with q1d points per dimension
   * (default), 1 tensor Clenshaw-Curtis with q1d points (q1d <= 33), 2 Smolyak sparse grid of nested
   * Clenshaw-Curtis rules of level quad_level (p <= quad_level <= p + 5; negative weights: cells whose
   * Hessian is then indefinite report IPM_CELL_ILLCONDITIONED).  Rules other than 0 need n = N m <= 88. */
  int32_t quad_kind, quad_level;
  /* dual-solve direction (reading 35, "Hessian
   * approximations ... BFGS ... construct the Hessian from previously computed gradients"):
   *   0 exact Newton: H(lambda) of PAPER.md:169, Cholesky (default);
   *   1 limited-memory BFGS: d = -H_l g by the two-loop recursion over the cell's last lbfgs_m pairs
   *     (s, y) of accepted iterates, kept in the context across (pseudo-)time steps (a cell whose basis
   *     size changed starts without pairs), initial matrix I_N (x) Jbar^{-1}, Jbar = sum_k omega_k
   *     grad u_s(Lambda_k); the pairs occupy 2 lbfgs_m N m doubles per cell of device memory.
   *     Supported: lbfgs_m = 8 (0 selects 8), n = N m <= 96, or Euler 2D cells of a 3D tensor Gauss-Legendre
   *     rule without levels with n <= 256 (config 5: CTA per cell, sum-factorised node pass).  Same line search, stopping test, counts
   *     (accepted steps) and statuses as Newton; a cell not converged after max_newton quasi-Newton
   *     steps continues with at most max_newton exact Newton steps from its iterate (its count is the
   *     sum, its pairs are dropped); IPM_CELL_ILLCONDITIONED = Jbar not positive definite. */
  int32_t hessian_kind, lbfgs_m;
  /* per-level nested quadrature (reading 36; PAPER.md:385-398 and 625,
   * "Order 2 uses 5 quadrature points, orders 3 to 6 use 9"): level_q1d[0] > 0 gives adaptive level l
   * (n_levels > 0) its own tensor Clenshaw-Curtis rule of level_q1d[l] points per dimension, nested in
   * the context's rule (quad_kind 1, q1d = level_q1d[n_levels-1]; level_q1d ascending with
   * (q1d - 1) % (level_q1d[l] - 1) == 0).  The dual solve of a cell at level l and the moment update
   * to level l integrate with rule l; the states of the stencil at its nodes come from each cell's
   * duals at its own level (a node pass evaluates every cell at every node of the finest rule).  The
   * IC projection uses the initial level's rule; the CFL rate takes the cells at their own rule's
   * nodes and prescribed (STATE) boundary states at every node of the finest rule.  Needs the bucketed
   * dual launches (Euler 2D, p = 2, degrees 2-5; IPM_ERR_UNSUPPORTED otherwise).  0 = one rule. */
  int32_t level_q1d[8];
} ipm_config;

#define IPM_HIST_BUCKETS 16
typedef struct {
  double dt, t;              /* time step taken, time after the step */
  double residual;           /* sum_j |Omega_j| |uhat_{j,0,0}^{n+1} - uhat_{j,0,0}^n| */
  int64_t newton_iters;      /* accepted Newton steps over all local cells this step */
  int64_t failed_cells;      /* cells with status != IPM_CELL_OK */
  int32_t worst_status;      /* max ipm_cell_status over local cells */
  int32_t reserved;
  /* Newton-count histogram (Alg. 1 lines 7-10 per cell): newton_hist[i] = local cells that took i
   * accepted Newton steps this step, the last bucket counts >= IPM_HIST_BUCKETS - 1 */
  int64_t newton_hist[IPM_HIST_BUCKETS];
  int64_t halvings;          /* rejected Armijo trials (step halvings, reading 3') over all local cells */
  int64_t inadmissible_trials; /* of which the trial state was not admissible (reading 4) */
} ipm_step_info;

/* Create a context: host setup of basis, quadrature and mesh tables, device upload,
 * communicator (nranks > 1).  Synchronous. */
IPM_API ipm_status ipm_init(const ipm_config *cfg, ipm_ctx **out);
IPM_API void ipm_destroy(ipm_ctx *c);
IPM_API const char *ipm_status_string(ipm_status s);
IPM_API const char *ipm_last_error(void);

/* sizes of the local problem: cells (owned), N, Q, m */
IPM_API ipm_status ipm_sizes(const ipm_ctx *c, int64_t *cells, int32_t *N, int32_t *Q, int32_t *m);
/* Node-state storage chosen by ipm_init (host only): *rows = 0 when the context keeps the node states
 * u_s(lambda^T phi(xi_k)) of all cells ([cells + halo][m][Q], written by the dual solve for the flux),
 * else the rows per band of the banded mode (row-major cartesian blocks without levels whose whole
 * buffer would exceed IPM_NODE_BUDGET_GB, default 24 GB, or IPM_BAND_ROWS set): the flux then
 * recomputes each band's node states from lambda (PAPER.md:455-462 needs them only face by face). */
IPM_API ipm_status ipm_node_band_rows(const ipm_ctx *c, int64_t *rows);
/* host copies of the basis tables: h_xi [Q][p], h_omega [Q], h_phi [Q][N] (any may be NULL) */
IPM_API ipm_status ipm_get_basis(const ipm_ctx *c, double *h_xi, double *h_omega, double *h_phi);
/* host copy of the owned cells' global ids [cells] (int64) */
IPM_API ipm_status ipm_get_cell_ids(const ipm_ctx *c, int64_t *h_ids);

/* Dual solve for all owned cells (Alg. 1 lines 4-10; Alg. 2 line 5).
 *   d_uhat   [cells][N][m] in
 *   d_lambda [cells][N][m] in: warm start, out: last accepted iterate
 *   mode     IPM_NEWTON_FULL | IPM_NEWTON_ONE_STEP
 *   d_iters  [cells] int32 out: accepted Newton steps (nullable)
 *   d_status [cells] int32 out: ipm_cell_status (nullable)
 *   d_crit   [cells] out: final sum_a ||grad_{lambda_{.,a}} L||_2 (nullable) */
IPM_API ipm_status ipm_dual_solve(ipm_ctx *c, const double *d_uhat, double *d_lambda, int32_t mode,
                          int32_t *d_iters, int32_t *d_status, double *d_crit);

/* Kinetic-flux moment update from given duals, single-rank contexts only
 * (a distributed context returns IPM_ERR_ARG: its halo duals arrive through ipm_step_flux):
 *   d_lambda    [cells][N][m] in
 *   d_uhat_old  [cells][N][m] in; d_uhat_new [cells][N][m] out (may not alias d_uhat_old)
 *   dt > 0: use it; dt <= 0: CFL step from the reconstructed states, capped by t_end - t.
 *   Uses ipm_config.update_form.  d_dt (nullable, device, 1 double) receives the step used. */
IPM_API ipm_status ipm_flux_update(ipm_ctx *c, const double *d_lambda, const double *d_uhat_old,
                           double *d_uhat_new, double dt, double *d_dt);

/* One full step of Algorithm 1/2/3 in place: dual solve (config newton_mode), refinement level
 * (n_levels > 0), CFL dt capped at t_end - t (t_end <= 0: no cap, steady), moment update.
 * info == NULL: asynchronous.  info != NULL: synchronous; fills info and returns IPM_ERR_NUMERIC
 * if a cell failed (the step is still complete: failed cells keep their last iterate).
 * Small problems (fewer than IPM_GRAPH_MAX_CELLS local cells) replay the step's launches from a
 * CUDA graph captured on first use (re-captured when d_uhat, d_lambda or t_end change; not while
 * kernel timing is enabled): for configs 1 and 2 the per-step launch cost bounds the step. */
#define IPM_GRAPH_MAX_CELLS 65536
IPM_API ipm_status ipm_step(ipm_ctx *c, double *d_uhat, double *d_lambda, double t_end, ipm_step_info *info);

/* ipm_step with the state in HOST memory (the end-to-end path):
 *   h_uhat, h_lambda  [cells][N][m] host, in/out; page-locked (cudaHostAlloc / torch pin_memory)
 *                     for the copies to overlap, pageable memory works but serialises them
 *   d_uhat, d_lambda  [cells][N][m] device work buffers (caller-owned, contents overwritten)
 *   nchunks >= 1      the host->device copies are split into nchunks contiguous cell ranges on a
 *                     copy stream; the dual solve of a range starts when its copy has landed, so
 *                     the copies of later ranges overlap the solves of earlier ones; the duals of a
 *                     range go back to the host right after its solve (no adaptive levels), the
 *                     moments (and duals with adaptive levels) after the flux update.
 * The result equals ipm_step on the same data bit for bit.  Synchronous: returns when h_uhat /
 * h_lambda hold the result; info (nullable) as for ipm_step.  Single-rank contexts only
 * (IPM_ERR_ARG otherwise). */
IPM_API ipm_status ipm_step_host(ipm_ctx *c, double *h_uhat, double *h_lambda, double *d_uhat, double *d_lambda,
                                 double t_end, int32_t nchunks, ipm_step_info *info);

/* Helpers for inputs (not steps of the path):
 *   ipm_project_ic: uhat_j = <ubar_j(xi) phi>_Q with exact cell averages of a piecewise-constant IC
 *                   (Alg. 1 line 2); also resets t = 0 and levels to initial_level.
 *   ipm_warm_start: lambda = e_0 (x) grad s(uhat_0) per cell (reading 6)
 *   ipm_moments_from_dual: uhat = h(lambda) = <u_s(lambda^T phi) phi^T>_Q
 *   ipm_stress_dual: lambda_0 = grad s(d_base[j]); lambda_{i,a} = (rel |lambda_{0,a}| + abs)
 *                    2^{-|i|} d_z[j][i][a], higher modes scaled so max_k Lambda_E <= lambda_{0,E}/2. */
typedef struct {
  int32_t kind, initial_level;
  double xs0, xs1[3], ys0, ys1[3];
  ipm_state state[4];        /* STEP1D: left,right; QUAD2D: NE,NW,SW,SE; UNIFORM: [0] */
} ipm_ic;
IPM_API ipm_status ipm_project_ic(ipm_ctx *c, const ipm_ic *ic, double *d_uhat);

/* Stochastic Collocation: the deterministic finite-volume
 * scheme with the same numerical flux (ipm_config.flux) run at every quadrature node; all nodes
 * advance together with one CFL step (the paper's coupled collocation code).
 *   d_nodes  [cells][m][Q] node states (device, caller-owned)
 *   ipm_sc_init     node states of the IC (the cell averages ipm_project_ic projects); sets t = 0
 *   ipm_sc_step     d_out = d_in - dt r(d_in), dt = CFL / max node rate capped at t_end - t
 *                   (t_end <= 0: no cap); d_in and d_out must not alias.  The step also records the
 *                   CFL rate of d_out; the next call with d_in == that d_out reuses it instead of
 *                   a rate pass, so the states must not be modified between such calls (any other
 *                   d_in, or ipm_sc_init, recomputes it); info (nullable, makes the
 *                   call synchronous): dt, t, residual = sum_j |Omega_j| |change of the mean of the
 *                   first state|, newton_iters = 0
 *   ipm_sc_moments  uhat_i = sum_k w_k u(xi_k) phi_i(xi_k), [cells][N][m]
 * Single-rank contexts only (IPM_ERR_ARG otherwise). */
IPM_API ipm_status ipm_sc_init(ipm_ctx *c, const ipm_ic *ic, double *d_nodes);
IPM_API ipm_status ipm_sc_step(ipm_ctx *c, const double *d_in, double *d_out, double t_end, ipm_step_info *info);
IPM_API ipm_status ipm_sc_moments(ipm_ctx *c, const double *d_nodes, double *d_uhat);
IPM_API ipm_status ipm_warm_start(ipm_ctx *c, const double *d_uhat, double *d_lambda);
IPM_API ipm_status ipm_moments_from_dual(ipm_ctx *c, const double *d_lambda, double *d_uhat);
IPM_API ipm_status ipm_stress_dual(ipm_ctx *c, const double *d_base, const double *d_z, double rel, double abs_,
                           double *d_lambda);

/* L-BFGS (hessian_kind 1): forget every cell's pairs (the next solves start from Jbar^{-1} alone);
 * asynchronous on the ctx stream.  IPM_ERR_ARG for a Newton context. */
IPM_API ipm_status ipm_lbfgs_reset(ipm_ctx *c);
/* L-BFGS history of the owned cells (device, caller-owned, nullable): d_S, d_Y [cells][lbfgs_m][N m]
 * pairs newest first (entries beyond the count / the cell's basis size unspecified), d_count int32
 * [cells].  Asynchronous on the ctx stream.  IPM_ERR_ARG for a Newton context. */
IPM_API ipm_status ipm_lbfgs_history(ipm_ctx *c, double *d_S, double *d_Y, int32_t *d_count);

/* levels (adaptivity): device int32 [cells]; get/set copy from/to the context */
IPM_API ipm_status ipm_get_levels(ipm_ctx *c, int32_t *d_levels);
IPM_API ipm_status ipm_set_levels(ipm_ctx *c, const int32_t *d_levels);
/* per-cell results of the last ipm_step: d_iters, d_status int32 [cells] (device, nullable) */
IPM_API ipm_status ipm_last_cell_stats(ipm_ctx *c, int32_t *d_iters, int32_t *d_status);
/* per-cell line-search record of the last dual solve (ipm_step or ipm_dual_solve): rejected Armijo
 * trials (step halvings) and the inadmissible trials among them, int32 [cells] (device, nullable) */
IPM_API ipm_status ipm_last_cell_linesearch(ipm_ctx *c, int32_t *d_halvings, int32_t *d_inadmissible);
/* Outcome of the last dual solve (ipm_dual_solve, ipm_step, ipm_step_dual): the worst
 * ipm_cell_status over the local cells and the number of cells with status != IPM_CELL_OK.
 * Synchronous (waits for the ctx stream); either pointer may be NULL. */
IPM_API ipm_status ipm_get_status(ipm_ctx *c, int32_t *worst, int64_t *n_failed);
/* simulation time (host, synchronous) */
IPM_API ipm_status ipm_get_time(ipm_ctx *c, double *t);
IPM_API ipm_status ipm_set_time(ipm_ctx *c, double t);

/* Distributed contexts (nranks > 1): the step is split around the exchange, which the caller
 * performs (e.g. torch.distributed over NCCL; the dual problems need no communication, only the
 * flux needs the face neighbours' duals):
 *   ipm_step_dual  dual solve of the owned cells, packs the duals of the cells adjacent to each peer
 *                  into d_sendbuf [nsend][N][m] (grouped by peer, ipm_halo_layout order) and copies
 *                  the local CFL rate (bits of a double >= 0, order-preserving as uint64) to d_rate;
 *   (caller)       send/receive the per-peer slices, all-reduce d_rate with MAX;
 *   ipm_step_flux  node states of the halo cells from d_recvbuf [nrecv][N][m], dt from d_rate,
 *                  moment update of the owned cells; info (if non-NULL) holds LOCAL sums.
 * ipm_step = ipm_step_dual + ipm_step_flux without exchange (single-rank contexts only). */
IPM_API ipm_status ipm_step_dual(ipm_ctx *c, const double *d_uhat, double *d_lambda, double *d_sendbuf,
                                 uint64_t *d_rate);
IPM_API ipm_status ipm_step_flux(ipm_ctx *c, double *d_uhat, double *d_lambda, const double *d_recvbuf,
                                 const uint64_t *d_rate, double t_end, ipm_step_info *info);
/* ipm_step_dual in two parts, so that the halo exchange overlaps the interior dual solves:
 *   ipm_step_dual_boundary  begins the step, solves the owned cells adjacent to a peer, packs d_sendbuf;
 *   (caller)                starts the send / receive of the per-peer slices (asynchronous);
 *   ipm_step_dual_interior  solves the remaining owned cells, copies the local CFL rate to d_rate;
 *   (caller)                waits for the receives, all-reduces d_rate with MAX; then ipm_step_flux.
 * Results equal ipm_step_dual bit for bit (every cell's solve is independent of the launch it is in).
 * Contexts with adaptive levels, or the comparison dual kernels (IPM_DUAL_KERNEL=group|warp), solve
 * every cell in the boundary part (the interior part then only copies the rate). */
IPM_API ipm_status ipm_step_dual_boundary(ipm_ctx *c, const double *d_uhat, double *d_lambda, double *d_sendbuf);
IPM_API ipm_status ipm_step_dual_interior(ipm_ctx *c, const double *d_uhat, double *d_lambda, uint64_t *d_rate);
/* peers (ascending rank) with per-peer send / receive cell counts; arrays sized npeers */
IPM_API ipm_status ipm_halo_layout(const ipm_ctx *c, int32_t *npeers, int64_t *nsend, int64_t *nrecv,
                                   int32_t *h_peers, int32_t *h_send_count, int32_t *h_recv_count);
/* Host-only (no CUDA): the partition ipm_init would build for cfg->rank of cfg->nranks.
 * Pass NULL arrays to query sizes first.  local ids ascending; halo and send ids grouped by peer
 * (ascending rank), ascending within a peer; send list r->s equals halo list of s from r. */
IPM_API ipm_status ipm_partition_query(const ipm_config *cfg, int64_t *cells, int64_t *nhalo, int32_t *npeers,
                                       int64_t *nsend, int64_t *h_local_gid, int64_t *h_halo_gid,
                                       int32_t *h_peers, int32_t *h_send_count, int32_t *h_recv_count,
                                       int64_t *h_send_gid);

/* Timing of the last ipm_step's dual-solve kernel (ms, CUDA events on the ctx stream;
 * synchronous) — used by bench.py for the roofline line. */
IPM_API ipm_status ipm_last_kernel_ms(ipm_ctx *c, float *dual_ms, float *flux_ms);
IPM_API ipm_status ipm_enable_timing(ipm_ctx *c, int32_t on);

/* Name of the dual-solve kernel the last dual launch of this process used ("k_dual_mma",
 * "k_dual_group", "k_dual_warp", "k_dual_big"; "" before the first launch).  Host only, never fails;
 * the string is static. */
IPM_API const char *ipm_last_dual_kernel(void);

/* sizeof(ipm_config), sizeof(ipm_ic), sizeof(ipm_step_info) as compiled into the library (host only;
 * bindings check their struct mirrors against them) */
IPM_API size_t ipm_struct_size(int32_t which /* 0 config, 1 ic, 2 step_info */);

/* Refinement retardation stage (Algorithm 4): ipm_retard_stage reads the current stage
 * (synchronous; 0 when retardation is off).  Single-rank contexts advance the stage on the device
 * after every step from the step's residual; distributed contexts (nranks > 1) do not — the caller
 * passes the global residual of each step to ipm_retard_advance (the Python binding does after its
 * residual all-reduce), which advances the stage when it lies below the stage's tolerance. */
IPM_API ipm_status ipm_retard_stage(ipm_ctx *c, int32_t *stage);
IPM_API ipm_status ipm_retard_advance(ipm_ctx *c, double global_residual);

/* Name of the flux kernel the last flux launch of this process used ("k_flux_strip", "k_flux_cart",
 * "k_flux_warp"; "" before the first launch).  Host only, never fails; the string is static. */
IPM_API const char *ipm_last_flux_kernel(void);

/* Debug: per-phase clock64 cycle totals of the dual kernel (builds with -DIPM_PHASE_TIMERS;
 * zeros otherwise).  h_out[8]: 0 eval/grad/line search, 1 Hessian, 2 Cholesky, 3 back-substitution,
 * 4 final line search, 7 epilogue + cell fetch.  Synchronous; resets the counters. */
IPM_API ipm_status ipm_debug_phase_cycles(uint64_t *h_out);

#ifdef __cplusplus
}
#endif
#endif
