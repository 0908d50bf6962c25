// ipm_internal.h — internal structures shared by the libipm host code and kernels.
#pragma once
#include <cstdint>

namespace ipm {

struct ClParams {
  double gamma, umin, umax, inv_gm1;  // inv_gm1 = 1/(gamma-1)
};

// Basis / quadrature tables as seen by the kernels (device pointers).
//   PhiT  [N][QP]  phi_i(xi_k)           (QP = Q rounded up to an odd stride: bank spread)
//   WPhiT [N][QP]  omega_k phi_i(xi_k)
struct Tables {
  const double* PhiT;
  const double* WPhiT;
  const double* omega;
  const int32_t* deg;  // [N] total degree |i|
  int N, Q, QP, p;
  // sum factorisation over the tensor Gauss-Legendre rule (p == 2):
  //   LL [q1d][npr] = (w_k/2) L_a(x_k) L_b(x_k) for 1D degree pairs a <= b <= M
  //   idx [N][p]    multi-indices
  const double* LL;
  const int32_t* idx;
  int q1d, npr;
  // omega Phi^T in mma.m8n8k4 A-fragment order: WPhiF[(mt * KS + ks) * 32 + l] =
  //   omega_k phi_i(xi_k), i = 8 mt + l/4, k = 4 ks + l%4 (zero outside N x Q); MT = ceil(N/8), KS = ceil(Q/4)
  const double* WPhiF;
  int MT, KS;
  // 1D tables of the tensor Gauss-Legendre rule (sum-factorised node pass of k_dual_lbfgs_big):
  //   L1 [M+1][q1d] orthonormal Legendre L_i(x_k) = sqrt(2i+1) P_i(x_k),  w1h [q1d] = w_k / 2;  npr1 = M + 1
  const double* L1;
  const double* w1h;
  int npr1;
};

// Local mesh: owned cells, face tables (F faces per cell)
//   nbr  [cells][F]  >= 0: cell index into the node-state buffer (owned or halo slot),
//                    < 0: boundary, tag = -1 - nbr
//   nrm  [cells][F][2] outward unit normal (tri only)
//   coef [cells][F]  |e| / |Omega_j|
struct Mesh {
  int kind, F;
  int64_t cells;
  const int32_t* nbr;
  const double* nrm;
  const double* coef;
  const double* area;      // [cells]
  const double* rate_geo;  // [cells] tri: perimeter / area
  double inv_dx, inv_dy;   // 1D / cartesian
  const double* ghost;     // [4][Q][m] STATE boundary node states
  int bc_kind[4];
  int bx, by;  // cartesian: the cells form a row-major bx x by block (verified from nbr on the host), else 0
};

struct Newton {
  double tau, armijo_c;
  int max_newton, max_halvings;
  int mode;
};

// per-level nested quadrature (reading 36): level l integrates with its own
// tensor Clenshaw-Curtis rule, node q of which is node kf[l][q] of the finest rule (Tables T)
struct LevelRules {
  int on;
  int Q[8], QP[8];
  const int32_t* kf[8];    // [Q_l]
  const double* wphit[8];  // [N_l][QP_l]  omega^l_q phi_i(xi_kf(q))
};

struct Adapt {
  LevelRules lq;
  int n_levels;
  int Nl[8];
  int Nprev0;  // basis size of degree level_M[0]-1 (indicator band at the lowest level)
  double delta_dec, delta_inc;
  int n_retard;  // refinement retardation (Alg. 4): 0 = off
  int retard_level[8];
  double retard_eps[8];
};

// Device scalars of one step (ctx-owned).
struct StepScalars {
  unsigned long long rate_bits;  // max over nodes of the CFL rate (as ordered bits of a double >= 0)
  double dt, t, residual;
  unsigned long long newton_iters, failed;
  int worst, work_counter, work_counter2;
  int stage;  // refinement retardation stage (Alg. 4)
  unsigned long long sc_rate_next;  // SC: CFL rate of the last ipm_sc_step output (ordered bits)
  // dual-solve statistics of the step (ipm_step_info): cells per Newton count (last bucket: >= 15),
  // rejected line-search trials and the inadmissible ones among them
  unsigned long long hist[16];
  unsigned long long halvings, inadm_trials;
  // adaptive degree in uniform-degree buckets: cells per level, and a work queue per level's launch
  int lvl_count[8], lvl_queue[8];
  // reading 35: cells of the quasi-Newton pass handed to the Newton fallback, per level, and its queues
  int fb_count[8], fb_queue[8];
};
constexpr int kHistBuckets = 16;

struct DualLaunch {
  const double* uhat;
  double* lam;
  int32_t* iters;
  int32_t* status;
  double* crit;
  double* uq;            // [cells][Q][m] node states at the final iterate (nullable)
  const int32_t* level;  // nullable
  int32_t* level_new;    // nullable
  int64_t cells;
  int mode;
  int want_rate;
  int32_t* halv;   // [cells] rejected line-search trials of the cell (nullable)
  int32_t* inadm;  // [cells] of which inadmissible (non-finite L / closure) (nullable)
  // bucketed launches (k_dual_mma): the cells are list[0 .. *ncells_dev) (device count), the queue a
  // per-launch counter, row the [cells][row] stride of uhat / lambda (0: N m of the tables)
  const int32_t* list;
  const int32_t* ncells_dev;
  int* queue;
  int row;
  // L-BFGS history (hessian_kind 1, reading 35; ctx-owned): pairs newest first
  double* lb_S;     // [cells][lbfgs_m][row]
  double* lb_Y;     // [cells][lbfgs_m][row]
  double* lb_rho;   // [cells][lbfgs_m]  1 / (s^T y)
  int32_t* lb_cnt;  // [cells] stored pairs
  int32_t* lb_n;    // [cells] unknowns the pairs belong to
  // reading 35's Newton fallback: k_dual_lbfgs appends the cells that reach max_newton quasi-Newton
  // steps to fb_list (device count fb_count) and leaves their accounting to the Newton pass over that
  // list, which runs with accumulate = 1 (per-cell counts and line-search records add up)
  int32_t* fb_list;
  int* fb_count;
  int accumulate;
};

struct FluxLaunch {
  const double* uq;  // [cells + halo][Q][m]
  const double* uhat_old;
  double* uhat_new;
  const int32_t* level_new;  // nullable: projection level per cell
  double* lam;               // nullable: duals truncated to the new level after the update
  int update_form;
  double cfl;
  // banded node states (k_flux_warp; zero = the whole-mesh buffer): the cells [cell0, mesh.cells)
  // are updated; the node states of owned cell c live at uq + (c - uq_base) Q m, those of halo cell
  // c >= n_owned at uq_halo + (c - n_owned) Q m
  int64_t cell0, uq_base, n_owned;
  const double* uq_halo;
  // processing order of the cells (k_flux_warp on triangle meshes: Morton order of the centroids, so the
  // node states of a cell's neighbours are read while still in L2; nullable = index order)
  const int32_t* order;
};

// Everything a launcher needs.
struct KernelCtx {
  Tables T;
  Mesh mesh;
  Newton nw;
  Adapt ad;
  ClParams cl;
  int closure, flux, m;
  StepScalars* sc;  // device
  void* stream;     // cudaStream_t
  int sm_count;
  size_t smem_optin;
  int force_warp_kernel;  // 1: always use the warp-per-cell dual kernel (tests, comparison)
  // kernel choices, read once from the environment at ipm_init (comparison paths for the tests and
  // A/B experiments; the defaults are the product path): IPM_DUAL_KERNEL=group|warp, IPM_SUMFACT=0,
  // IPM_MMA_W=4, IPM_MMA_GROUPS=n, IPM_GROUP_T=1, IPM_FLUX_KERNEL=cart|warp|strip
  int dual_group;    // 1: the 4x4-register-block kernel instead of k_dual_mma
  int sumfact;       // 0: direct Hessian sum instead of the sum factorisation
  int mma_w4;        // 1: config 3 with W = 4 warps per cell
  int mma_generic;   // 1: the run-time-shape k_dual_mma instance even where a fixed-shape one exists
  int mma_groups;    // > 0: cap on the groups per CTA of k_dual_mma
  int group_t1;      // 1: one Hessian block per thread in k_dual_group
  int flux_choice;   // 0 default (strip when applicable), 1 cart, 2 warp
  int flux_scalar_proj;  // 1: k_flux_warp projects with scalar dot products (IPM_FLUX_SCALAR_PROJ, comparison)
  double* big_scratch;    // per-CTA scratch of the large-cell dual kernel (config 5), or null
  int big_ctas;
  // adaptive degree bucketed into uniform-degree launches (north star (c); Alg. 3): per-level
  // tables (N_l, its 1D pair table, tile counts; Phi / omega Phi shared by prefix) and cell lists
  int hessian_kind;       // 0 exact Newton (Hessian + Cholesky), 1 L-BFGS (k_dual_lbfgs, reading 35)
  int lbfgs_m;            // L-BFGS pairs per cell
  int lbfgs_pairs_reg;    // 1: k_dual_lbfgs keeps the pairs in registers (IPM_LBFGS_PAIRS=reg), else shared memory
  int32_t* fb_lists;      // [max(1, n_levels)][cells] Newton-fallback cell lists (hessian_kind 1)
  int bucket;             // 1: one k_dual_mma launch per level over that level's cells
  Tables Tl[8];
  int32_t* lists;         // [n_levels][cells]
};

// launchers (ipm_kernels.cu); return 0 on success, else a cudaError_t / -1 unsupported
int launch_step_begin(const KernelCtx& k, double rate0);
size_t big_scratch_doubles(int N, int Q, int m, int q1d, int npr, int p);
int debug_phase_cycles(unsigned long long* out);
int launch_dual(const KernelCtx& k, const DualLaunch& a);
const char* last_dual_kernel();
const char* last_flux_kernel();
int launch_retard(const KernelCtx& k);
int launch_sc_rate(const KernelCtx& k, const double* Uin);
int launch_sc_begin(const KernelCtx& k, double rate0, int use_cached);
int launch_sc_update(const KernelCtx& k, const double* Uin, double* Uout);
int launch_sc_moments(const KernelCtx& k, const double* U, double* uhat);
int launch_dt(const KernelCtx& k, double t_end, double dt_fixed, double cfl);
int launch_flux(const KernelCtx& k, const FluxLaunch& a);
int launch_project_ic(const KernelCtx& k, const double* d_region /*[R][Q][m]*/, const double* d_split /*[Q][2]*/,
                      int ic_kind, int nx, double x0, double y0, double dx, double dy, const int32_t* level,
                      const int64_t* gid, double* uhat, double* unodes = nullptr);
// pack duals of the listed local cells into a contiguous send buffer [n][N][m]
int launch_pack(const KernelCtx& k, const double* lam, const int32_t* idx, int64_t n, double* out);
int launch_warm_start(const KernelCtx& k, const double* uhat, double* lam);
// node pass: uhat = h(lambda) (nullable), node states uq (nullable), CFL rate into sc
// exact = 1: the dual kernels' node-pass instruction sequence (bit-identical states; halo cells)
int launch_nodes(const KernelCtx& k, const double* lam, double* uhat, double* uq, int want_rate, int exact = 0);
int launch_stress(const KernelCtx& k, const double* base, const double* z, double rel, double abs_, double* lam);

}  // namespace ipm
