/*
 * ipm_oracle.c — plain fp64 CPU oracle of the IPM hot path (arXiv 1912.09238).
 *
 * TEST INFRASTRUCTURE ONLY (see ipm_oracle.h).  Citations "PAPER.md:n" are
 * lines of the paper's LaTeX source; "reading k" refers to the numbered
 * readings of SURVEY.md §8(c), copied into DESIGN.md.
 *
 * Style: every routine is the textbook form of the paper's formula.  Loops are
 * written in the paper's index order; nothing is blocked, fused or reordered.
 * OpenMP only distributes independent spatial cells (the dual
 * problem needs no communication).
 */
#include "ipm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PI_ 3.14159265358979323846

struct orc_ctx {
  orc_problem P;
  int N, Q, m, d, F, cells;
  int32_t *idx;   /* [N][p] multi-indices, graded then lexicographically descending */
  double *xi;     /* [Q][p] nodes */
  double *omega;  /* [Q]    w_k f_Xi(xi_k) */
  double *Phi;    /* [Q][N] phi_i(xi_k) */
  int32_t *nbr;   /* [cells][F] neighbour, or -1-tag on the boundary */
  double *nrm;    /* [cells][F][2] outward unit normal */
  double *coef;   /* [cells][F] |e| / |Omega_j| */
  double *area;   /* [cells] */
  double *perim;  /* [cells] */
  double *xc;     /* [cells][2] cell centre (1D/cart) */
  double *bc_u;   /* [4][Q][m] ghost states of STATE boundaries */
  int32_t *level; /* [cells] refinement level index (adaptivity) */
  int retard_stage; /* refinement retardation stage (Alg. 4) */
  int n_levels;
  int Nl[8];      /* N at each level */
  /* L-BFGS history (hessian_kind 1, reading 35): per cell lbfgs_m pairs, newest first */
  double *lb_S, *lb_Y; /* [cells][lbfgs_m][N m] */
  int32_t *lb_cnt;     /* [cells] stored pairs */
  int32_t *lb_n;       /* [cells] unknowns n the pairs belong to (a level change clears them) */
  /* per-level nested rules (reading 36): level l uses the nodes lkf[l][0..lQ[l]) of the finest rule
   * (c->xi, c->Phi) with its own weights lw[l] */
  int lq_on;
  int lQ[8];
  int32_t *lkf[8];
  double *lw[8];
};

/* the quadrature rule of a cell with basis size Nl: node q is node kf[q] of the finest rule (c->xi,
 * c->Phi), weight w[q] (H_l, grad at level l use Q_l) */
typedef struct {
  int Q;
  const int32_t *kf;
  const double *w;
} orc_rule;
static orc_rule rule_of(const orc_ctx *c, int Nl) {
  orc_rule R = {c->Q, NULL, c->omega};
  if (c->lq_on)
    for (int l = 0; l < c->n_levels; ++l)
      if (c->Nl[l] == Nl) {
        R.Q = c->lQ[l];
        R.kf = c->lkf[l];
        R.w = c->lw[l];
      }
  return R;
}
#define RK(R, q) ((R).kf ? (R).kf[q] : (q))

/* ------------------------------------------------------------------------ */
/* Random space: Legendre polynomials, Gauss-Legendre rule, total-degree basis */
/* ------------------------------------------------------------------------ */

/* P_0..P_n at x by the three-term recurrence (k+1)P_{k+1} = (2k+1)x P_k - k P_{k-1}. */
static void legendre_P(int n, double x, double *P) {
  P[0] = 1.0;
  if (n >= 1) P[1] = x;
  for (int k = 1; k < n; ++k) P[k + 1] = ((2.0 * k + 1.0) * x * P[k] - k * P[k - 1]) / (k + 1.0);
}

/* Orthonormal Legendre w.r.t. the density 1/2 on [-1,1]: sqrt(2i+1) P_i. */
static double phi_1d(int i, double x) {
  double P[64];
  legendre_P(i, x, P);
  return sqrt(2.0 * i + 1.0) * P[i];
}

/* Clenshaw-Curtis rule: nodes -cos(pi j / (n-1)), weights by the classical cosine
 * sum w_j = c_j/(n-1) (1 - sum_{k=1}^{(n-1)/2} b_k/(4k^2-1) cos(2 k theta_j)), c_j = 1 at the ends,
 * 2 inside, b_k = 1 for k = (n-1)/2, else 2 (n odd); n = 1: the midpoint with weight 2. */
void orc_clenshaw_curtis(int n, double *x, double *w) {
  if (n == 1) {
    x[0] = 0.0;
    w[0] = 2.0;
    return;
  }
  int Nn = n - 1;
  for (int j = 0; j < n; ++j) {
    double th = PI_ * j / Nn;
    x[j] = -cos(th);
    double s = 0.0;
    for (int k = 1; k <= Nn / 2; ++k) {
      double b = (2 * k == Nn) ? 1.0 : 2.0;
      s += b / (4.0 * k * k - 1.0) * cos(2.0 * k * th);
    }
    double cj = (j == 0 || j == Nn) ? 1.0 : 2.0;
    w[j] = cj / Nn * (1.0 - s);
  }
  if (n % 2 == 1) x[Nn / 2] = 0.0; /* exact midpoint */
}

/* Smolyak formula A(L, p) = sum_{L-p+1 <= |i| <= L} (-1)^{L-|i|} C(p-1, L-|i|) (U^{i_1} x ... x U^{i_p}),
 * i_d >= 1, U^1 the midpoint rule, U^i Clenshaw-Curtis with 2^{i-1}+1 nodes (nested); coincident
 * nodes merged by their index on the finest 1D grid (2^{L-1}+1 nodes). */
static int binom_(int n, int k) {
  if (k < 0 || k > n) return 0;
  int r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}
int orc_smolyak_cc(int p, int L, double *xi, double *w) {
  int F = L - p + 1;                 /* largest 1D level in the sum */
  int nf = F >= 2 ? (1 << (F - 1)) + 1 : 1; /* finest 1D grid */
  int ngrid = 1;
  for (int d = 0; d < p; ++d) ngrid *= nf;
  double *acc = (double *)calloc(ngrid, sizeof(double));
  char *used = (char *)calloc(ngrid, 1);
  int i[3] = {1, 1, 1};
  for (;;) {
    int s = 0;
    for (int d = 0; d < p; ++d) s += i[d];
    if (s >= L - p + 1 && s <= L) {
      int coef = ((L - s) % 2 ? -1 : 1) * binom_(p - 1, L - s);
      double xs[3][129], ws[3][129];
      int ns[3], step[3];
      for (int d = 0; d < p; ++d) {
        ns[d] = i[d] == 1 ? 1 : (1 << (i[d] - 1)) + 1;
        orc_clenshaw_curtis(ns[d], xs[d], ws[d]);
        step[d] = ns[d] == 1 ? 0 : (nf - 1) / (ns[d] - 1);
      }
      int cnt = 1;
      for (int d = 0; d < p; ++d) cnt *= ns[d];
      for (int t = 0; t < cnt; ++t) {
        int r = t, key = 0;
        double wt = coef;
        int jd[3];
        for (int d = p - 1; d >= 0; --d) {
          jd[d] = r % ns[d];
          r /= ns[d];
        }
        for (int d = 0; d < p; ++d) {
          int fi = ns[d] == 1 ? (nf - 1) / 2 : jd[d] * step[d];
          key = key * nf + fi;
          wt *= ws[d][jd[d]];
        }
        acc[key] += wt;
        used[key] = 1;
      }
    }
    int d = p - 1;
    while (d >= 0) {
      if (++i[d] <= L) break;
      i[d] = 1;
      --d;
    }
    if (d < 0) break;
  }
  double xf[129], wf[129];
  orc_clenshaw_curtis(nf, xf, wf);
  int Q = 0;
  for (int key = 0; key < ngrid; ++key) {
    if (!used[key]) continue;
    if (xi) {
      int r = key;
      for (int d = p - 1; d >= 0; --d) {
        xi[Q * p + d] = xf[r % nf];
        r /= nf;
      }
      w[Q] = acc[key];
    }
    ++Q;
  }
  free(acc);
  free(used);
  return Q;
}

/* Gauss-Legendre nodes (ascending) and weights (sum 2): Newton on P_q. */
void orc_gauss_legendre(int q, double *x, double *w) {
  double P[256];
  for (int i = 0; i < q; ++i) {
    double z = cos(PI_ * (i + 0.75) / (q + 0.5));
    for (int it = 0; it < 100; ++it) {
      legendre_P(q, z, P);
      double dP = q * (z * P[q] - P[q - 1]) / (z * z - 1.0);
      double dz = P[q] / dP;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    legendre_P(q, z, P);
    double dP = q * (z * P[q] - P[q - 1]) / (z * z - 1.0);
    x[q - 1 - i] = z;
    w[q - 1 - i] = 2.0 / ((1.0 - z * z) * dP * dP);
  }
}

/* N = binom(M+p, p). */
int orc_num_basis(int p, int M) {
  double r = 1.0;
  for (int k = 1; k <= p; ++k) r = r * (M + k) / k;
  return (int)(r + 0.5);
}

/* All multi-indices |i| <= M, graded by |i|, then lexicographically descending within a degree
 * (reading: SURVEY §8c step 1; e.g. p=2, degree 2 -> (2,0),(1,1),(0,2)). */
static void gen_degree(int p, int pos, int rem, int32_t *cur, int32_t *idx, int *n) {
  if (pos == p - 1) {
    cur[pos] = rem;
    for (int k = 0; k < p; ++k) idx[*n * p + k] = cur[k];
    ++*n;
    return;
  }
  for (int v = rem; v >= 0; --v) {
    cur[pos] = v;
    gen_degree(p, pos + 1, rem - v, cur, idx, n);
  }
}

void orc_multi_indices(int p, int M, int32_t *idx) {
  int n = 0;
  int32_t cur[8];
  for (int deg = 0; deg <= M; ++deg) gen_degree(p, 0, deg, cur, idx, &n);
}

/* ------------------------------------------------------------------------ */
/* Closures: u_s = (grad s)^{-1}, its Jacobian, s_* */
/* ------------------------------------------------------------------------ */

/* BASELINE scaling U = -rho S/(gamma-1), S = ln p - gamma ln rho (reading 11):
 *   ln rho = v1 - |v_m|^2/(2 v_E) - (gamma + ln(-v_E))/(gamma-1), p = rho/(-v_E), w = -v_m/v_E. */
static int euler_u(double gamma, int d, const double *v, double *u) {
  int m = d + 2;
  double vE = v[m - 1];
  if (!(vE < 0.0)) return 0;
  double vm2 = 0.0;
  for (int k = 0; k < d; ++k) vm2 += v[1 + k] * v[1 + k];
  double lnrho = v[0] - vm2 / (2.0 * vE) - (gamma + log(-vE)) / (gamma - 1.0);
  double rho = exp(lnrho);
  double p = rho / (-vE);
  double w2 = 0.0;
  u[0] = rho;
  for (int k = 0; k < d; ++k) {
    double wk = -v[1 + k] / vE;
    u[1 + k] = rho * wk;
    w2 += wk * wk;
  }
  u[m - 1] = p / (gamma - 1.0) + 0.5 * rho * w2;
  for (int k = 0; k < m; ++k)
    if (!isfinite(u[k])) return 0;
  return rho > 0.0;
}

/* du/dv = A0 (symmetric), H = (E+p)/rho, c^2 = gamma p / rho. */
static int euler_du(double gamma, int d, const double *v, double *J) {
  int m = d + 2;
  double u[4];
  if (!euler_u(gamma, d, v, u)) return 0;
  double rho = u[0], E = u[m - 1];
  double mm2 = 0.0;
  for (int k = 0; k < d; ++k) mm2 += u[1 + k] * u[1 + k];
  double p = (gamma - 1.0) * (E - 0.5 * mm2 / rho);
  double H = (E + p) / rho;
  double c2 = gamma * p / rho;
  J[0 * m + 0] = rho;
  for (int k = 0; k < d; ++k) {
    J[0 * m + 1 + k] = u[1 + k];
    J[(1 + k) * m + 0] = u[1 + k];
    for (int l = 0; l < d; ++l) J[(1 + k) * m + 1 + l] = u[1 + k] * u[1 + l] / rho + (k == l ? p : 0.0);
    J[(1 + k) * m + m - 1] = u[1 + k] * H;
    J[(m - 1) * m + 1 + k] = u[1 + k] * H;
  }
  J[0 * m + m - 1] = E;
  J[(m - 1) * m + 0] = E;
  J[(m - 1) * m + m - 1] = rho * H * H - c2 * p / (gamma - 1.0);
  return 1;
}

/* forward map v = grad U(u) (BASELINE scaling). */
static int euler_grad(double gamma, int d, const double *u, double *v) {
  int m = d + 2;
  double rho = u[0];
  double mm2 = 0.0;
  for (int k = 0; k < d; ++k) mm2 += u[1 + k] * u[1 + k];
  double p = (gamma - 1.0) * (u[m - 1] - 0.5 * mm2 / rho);
  if (!(rho > 0.0) || !(p > 0.0)) return 0;
  double S = log(p) - gamma * log(rho);
  double w2 = mm2 / (rho * rho);
  v[0] = (gamma - S) / (gamma - 1.0) - rho * w2 / (2.0 * p);
  for (int k = 0; k < d; ++k) v[1 + k] = rho * (u[1 + k] / rho) / p;
  v[m - 1] = -rho / p;
  return 1;
}

/* App. B, paper scaling s = -rho ln(rho^{-gamma}(E - |m|^2/(2 rho))),
 * with dS/dE corrected to -rho/(E - |m|^2/(2 rho)) (reading 9). */
void orc_euler_paper_grad_s(double gamma, int d, const double *u, double *Lam) {
  int m = d + 2;
  double rho = u[0], E = u[m - 1];
  double mm2 = 0.0;
  for (int k = 0; k < d; ++k) mm2 += u[1 + k] * u[1 + k];
  double eps = E - mm2 / (2.0 * rho);
  Lam[0] = -log(pow(rho, -gamma) * eps) + mm2 / (-2.0 * rho * E + mm2) + gamma;
  for (int k = 0; k < d; ++k) Lam[1 + k] = -2.0 * rho * u[1 + k] / (-2.0 * rho * E + mm2);
  Lam[m - 1] = -rho / eps;
}

/* App. B alpha(Lambda) with the gamma-term sign corrected to +2 Lambda_4 gamma
 * (reading 10). */
int orc_euler_paper_u(double gamma, int d, const double *L, double *u) {
  int m = d + 2;
  double L4 = L[m - 1];
  if (!(L4 < 0.0)) return 0;
  double Lm2 = 0.0;
  for (int k = 0; k < d; ++k) Lm2 += L[1 + k] * L[1 + k];
  double alpha = exp((Lm2 - 2.0 * L[0] * L4 + 2.0 * L4 * gamma) / (2.0 * L4 * (1.0 - gamma))) *
                 pow(-L4, 1.0 / (1.0 - gamma));
  u[0] = alpha;
  for (int k = 0; k < d; ++k) u[1 + k] = -L[1 + k] * alpha / L4;
  u[m - 1] = -alpha * (-Lm2 + 2.0 * L4) / (2.0 * L4 * L4);
  return isfinite(alpha) && alpha > 0.0;
}

static double sigmoid(double L) {
  if (L >= 0.0) return 1.0 / (1.0 + exp(-L));
  double e = exp(L);
  return e / (1.0 + e);
}

int orc_closure_u(const orc_ctx *c, const double *L, double *u) {
  const orc_problem *P = &c->P;
  switch (P->closure) {
    case ORC_CL_QUADRATIC: /* s = u^2/2: u_s(Lambda) = Lambda */
      for (int a = 0; a < c->m; ++a) u[a] = L[a];
      return 1;
    case ORC_CL_BARRIER: /* u_s = u- + (u+ - u-) sigma(Lambda) (BASELINE cfg 1) */
      u[0] = P->umin + (P->umax - P->umin) * sigmoid(L[0]);
      return isfinite(u[0]);
    default:
      return euler_u(P->gamma, c->m - 2, L, u);
  }
}

int orc_closure_du(const orc_ctx *c, const double *L, double *J) {
  const orc_problem *P = &c->P;
  switch (P->closure) {
    case ORC_CL_QUADRATIC:
      for (int a = 0; a < c->m; ++a)
        for (int b = 0; b < c->m; ++b) J[a * c->m + b] = (a == b) ? 1.0 : 0.0;
      return 1;
    case ORC_CL_BARRIER: {
      double s = sigmoid(L[0]);
      J[0] = (P->umax - P->umin) * s * (1.0 - s);
      return 1;
    }
    default:
      return euler_du(P->gamma, c->m - 2, L, J);
  }
}

/* Legendre transform s_* (only used by the dual objective L). */
double orc_closure_sstar(const orc_ctx *c, const double *L) {
  const orc_problem *P = &c->P;
  switch (P->closure) {
    case ORC_CL_QUADRATIC: {
      double s = 0.0;
      for (int a = 0; a < c->m; ++a) s += 0.5 * L[a] * L[a];
      return s;
    }
    case ORC_CL_BARRIER: {
      double D = P->umax - P->umin;
      double softplus = (L[0] > 0.0 ? L[0] : 0.0) + log1p(exp(-fabs(L[0])));
      return P->umin * L[0] + D * softplus - D * log(D);
    }
    default: {
      double u[4];
      if (!euler_u(P->gamma, c->m - 2, L, u)) return NAN;
      return u[0]; /* U_*(v) = rho(v) */
    }
  }
}

int orc_closure_grad_s(const orc_ctx *c, const double *u, double *L) {
  const orc_problem *P = &c->P;
  switch (P->closure) {
    case ORC_CL_QUADRATIC:
      for (int a = 0; a < c->m; ++a) L[a] = u[a];
      return 1;
    case ORC_CL_BARRIER: /* s'(u) = ln((u-u-)/(u+-u)) */
      if (!(u[0] > P->umin && u[0] < P->umax)) return 0;
      L[0] = log((u[0] - P->umin) / (P->umax - u[0]));
      return 1;
    default:
      return euler_grad(P->gamma, c->m - 2, u, L);
  }
}

/* ------------------------------------------------------------------------ */
/* Physics: physical flux, wave speed, two-point numerical fluxes g           */
/* ------------------------------------------------------------------------ */

/* Euler physical flux along unit normal n: (rho v_n, m v_n + p n, (E+p) v_n). */
static void euler_flux_n(double gamma, int d, const double *u, const double *n, double *f,
                         double *vn_out, double *c_out) {
  int m = d + 2;
  double rho = u[0], E = u[m - 1];
  double mm2 = 0.0, vn = 0.0;
  for (int k = 0; k < d; ++k) {
    mm2 += u[1 + k] * u[1 + k];
    vn += u[1 + k] / rho * n[k];
  }
  double p = (gamma - 1.0) * (E - 0.5 * mm2 / rho);
  f[0] = rho * vn;
  for (int k = 0; k < d; ++k) f[1 + k] = u[1 + k] * vn + p * n[k];
  f[m - 1] = (E + p) * vn;
  if (vn_out) *vn_out = vn;
  if (c_out) *c_out = sqrt(gamma * p / rho);
}

/* g(u_l, u_r; n) at one node.  cfg 1: global LF g = (u_l^2+u_r^2)/4 - dx/(2dt) (u_r-u_l)
 * (PAPER.md:870); HLL with Davis speeds (reading 14); Rusanov (reading 14). */
void orc_flux_g(const orc_ctx *c, const double *ul, const double *ur, const double *n,
                double dx_over_dt, double *g) {
  const orc_problem *P = &c->P;
  int m = c->m;
  if (P->flux == ORC_FLUX_LF_GLOBAL) {
    /* scalar Burgers, 1D, n = +1 */
    g[0] = 0.25 * (ul[0] * ul[0] + ur[0] * ur[0]) - 0.5 * dx_over_dt * (ur[0] - ul[0]);
    return;
  }
  int d = m - 2;
  double fl[4], fr[4], vl, vr, cl, cr;
  euler_flux_n(P->gamma, d, ul, n, fl, &vl, &cl);
  euler_flux_n(P->gamma, d, ur, n, fr, &vr, &cr);
  if (P->flux == ORC_FLUX_HLL) {
    double SL = fmin(vl - cl, vr - cr);
    double SR = fmax(vl + cl, vr + cr);
    for (int a = 0; a < m; ++a) {
      if (SL >= 0.0)
        g[a] = fl[a];
      else if (SR <= 0.0)
        g[a] = fr[a];
      else
        g[a] = (SR * fl[a] - SL * fr[a] + SL * SR * (ur[a] - ul[a])) / (SR - SL);
    }
    return;
  }
  double al = fabs(vl) + cl, ar = fabs(vr) + cr;
  double amax = al > ar ? al : ar;
  for (int a = 0; a < m; ++a) g[a] = 0.5 * (fl[a] + fr[a]) - 0.5 * amax * (ur[a] - ul[a]);
}

/* wave speed s = |f'(u)| along one direction (Burgers |u|; Euler |v_n|+c) */
static double wave_speed(const orc_ctx *c, const double *u, const double *n) {
  if (c->P.closure != ORC_CL_EULER && c->m == 1) return fabs(u[0]);
  int d = c->m - 2;
  double f[4], vn, cs;
  euler_flux_n(c->P.gamma, d, u, n, f, &vn, &cs);
  return fabs(vn) + cs;
}

static double speed_norm(const orc_ctx *c, const double *u) {
  if (c->m == 1) return fabs(u[0]);
  int d = c->m - 2;
  double v2 = 0.0;
  for (int k = 0; k < d; ++k) v2 += (u[1 + k] / u[0]) * (u[1 + k] / u[0]);
  double n0[2] = {1.0, 0.0}, f[4], vn, cs;
  euler_flux_n(c->P.gamma, d, u, n0, f, &vn, &cs);
  return sqrt(v2) + cs;
}

/* primitive -> conserved */
static void prim_to_cons(const orc_ctx *c, const double *q, double *u) {
  if (c->m == 1) {
    u[0] = q[0];
    return;
  }
  int d = c->m - 2;
  double rho = q[0], p = q[d + 1], v2 = 0.0;
  u[0] = rho;
  for (int k = 0; k < d; ++k) {
    u[1 + k] = rho * q[1 + k];
    v2 += q[1 + k] * q[1 + k];
  }
  u[d + 1] = p / (c->P.gamma - 1.0) + 0.5 * rho * v2;
}

/* conserved state of a state spec at node xi */
static void spec_state(const orc_ctx *c, const orc_state_spec *s, const double *xi, double *u) {
  int p = c->P.p;
  double q[5] = {0, 0, 0, 0, 0};
  if (s->kind == ORC_SPEC_FREESTREAM) {
    double rho = s->q0[0], pr = s->q0[1];
    double Ma = s->q0[2] + s->q0[3] * xi[s->dim_a];
    double th = (s->q0[4] + s->q0[5] * xi[s->dim_b]) * PI_ / 180.0;
    double cs = sqrt(c->P.gamma * pr / rho);
    q[0] = rho;
    q[1] = Ma * cs * cos(th);
    q[2] = Ma * cs * sin(th);
    q[3] = pr;
  } else {
    int nq = (c->m == 1) ? 1 : c->m;
    for (int k = 0; k < nq; ++k) {
      q[k] = s->q0[k];
      for (int dd = 0; dd < p && dd < 3; ++dd) q[k] += s->q1[k][dd] * xi[dd];
    }
  }
  prim_to_cons(c, q, u);
}

/* characteristic far-field ghost state (reading 37; Riemann invariants of the Euler equations along
 * the outward normal n, the textbook non-reflecting far-field treatment of the paper's far-field
 * boundaries): with v_n the normal velocity and c the sound speed,
 *   R+ = v_n + 2c/(gamma-1) leaves the domain (taken from the interior state ui),
 *   R- = v_n - 2c/(gamma-1) enters it (taken from the free stream uf);
 * v_nb = (R+ + R-)/2, c_b = (gamma-1)(R+ - R-)/4; entropy p/rho^gamma and tangential velocity from
 * the upwind side (free stream where v_nb < 0, interior otherwise).  Supersonic normal flow in the
 * interior (|v_n| >= c): inflow takes the free stream, outflow the interior state.  2D Euler only. */
static void farfield_ghost(double gamma, const double *ui, const double *uf, const double *n, double *ug) {
  double qi[4], qf[4];
  const double *us[2] = {ui, uf};
  double *qs[2] = {qi, qf};
  for (int s = 0; s < 2; ++s) { /* primitives rho, vx, vy, p */
    const double *u = us[s];
    double *q = qs[s];
    q[0] = u[0];
    q[1] = u[1] / u[0];
    q[2] = u[2] / u[0];
    q[3] = (gamma - 1.0) * (u[3] - 0.5 * u[0] * (q[1] * q[1] + q[2] * q[2]));
  }
  double vni = qi[1] * n[0] + qi[2] * n[1], vnf = qf[1] * n[0] + qf[2] * n[1];
  double ci = sqrt(gamma * qi[3] / qi[0]), cf = sqrt(gamma * qf[3] / qf[0]);
  if (vni <= -ci) { memcpy(ug, uf, 4 * sizeof(double)); return; }
  if (vni >= ci) { memcpy(ug, ui, 4 * sizeof(double)); return; }
  double rp = vni + 2.0 * ci / (gamma - 1.0), rm = vnf - 2.0 * cf / (gamma - 1.0);
  double vnb = 0.5 * (rp + rm), cb = 0.25 * (gamma - 1.0) * (rp - rm);
  const double *qu = vnb < 0.0 ? qf : qi; /* upwind side */
  double ent = qu[3] / pow(qu[0], gamma);
  double vnu = qu[1] * n[0] + qu[2] * n[1];
  double vt[2] = {qu[1] - vnu * n[0], qu[2] - vnu * n[1]};
  double rho = pow(cb * cb / (gamma * ent), 1.0 / (gamma - 1.0));
  double p = rho * cb * cb / gamma;
  double vx = vt[0] + vnb * n[0], vy = vt[1] + vnb * n[1];
  ug[0] = rho;
  ug[1] = rho * vx;
  ug[2] = rho * vy;
  ug[3] = p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy);
}

void orc_farfield_ghost(double gamma, const double *ui, const double *uf, const double *n, double *ug) {
  farfield_ghost(gamma, ui, uf, n, ug);
}

/* ghost state at node k for boundary tag t (reading 16; FARFIELD: reading 37) */
static void ghost_state(const orc_ctx *c, int tag, int k, const double *uin, const double *n,
                        double *ug) {
  int m = c->m;
  int kind = c->P.bc_kind[tag];
  if (kind == ORC_BC_STATE) {
    memcpy(ug, c->bc_u + ((size_t)tag * c->Q + k) * m, sizeof(double) * m);
  } else if (kind == ORC_BC_FARFIELD) {
    farfield_ghost(c->P.gamma, uin, c->bc_u + ((size_t)tag * c->Q + k) * m, n, ug);
  } else if (kind == ORC_BC_SLIP) {
    int d = m - 2;
    double mn = 0.0;
    for (int q = 0; q < d; ++q) mn += uin[1 + q] * n[q];
    ug[0] = uin[0];
    for (int q = 0; q < d; ++q) ug[1 + q] = uin[1 + q] - 2.0 * mn * n[q];
    ug[m - 1] = uin[m - 1];
  } else {
    memcpy(ug, uin, sizeof(double) * m);
  }
}

/* ------------------------------------------------------------------------ */
/* Context: basis, quadrature, mesh geometry                                  */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t key;
  int32_t t, e;
} edge_t;

static int edge_cmp(const void *x, const void *y) {
  const edge_t *a = (const edge_t *)x, *b = (const edge_t *)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return (a->t * 3 + a->e) - (b->t * 3 + b->e);
}

static void build_geometry(orc_ctx *c) {
  const orc_problem *P = &c->P;
  int F = c->F, n = c->cells;
  c->nbr = (int32_t *)malloc(sizeof(int32_t) * n * F);
  c->nrm = (double *)calloc((size_t)n * F * 2, sizeof(double));
  c->coef = (double *)malloc(sizeof(double) * n * F);
  c->area = (double *)malloc(sizeof(double) * n);
  c->perim = (double *)malloc(sizeof(double) * n);
  c->xc = (double *)calloc((size_t)n * 2, sizeof(double));
  if (P->mesh_kind == ORC_MESH_1D) {
    double dx = (P->x1 - P->x0) / P->nx;
    for (int j = 0; j < n; ++j) {
      c->nbr[j * 2 + 0] = (j > 0) ? j - 1 : (P->periodic ? n - 1 : -1 - 0);
      c->nbr[j * 2 + 1] = (j < n - 1) ? j + 1 : (P->periodic ? 0 : -1 - 1);
      c->nrm[(j * 2 + 0) * 2] = -1.0;
      c->nrm[(j * 2 + 1) * 2] = 1.0;
      c->coef[j * 2 + 0] = c->coef[j * 2 + 1] = 1.0 / dx;
      c->area[j] = dx;
      c->perim[j] = 2.0;
      c->xc[j * 2] = P->x0 + (j + 0.5) * dx;
    }
  } else if (P->mesh_kind == ORC_MESH_CART2D) {
    double dx = (P->x1 - P->x0) / P->nx, dy = (P->y1 - P->y0) / P->ny;
    for (int iy = 0; iy < P->ny; ++iy)
      for (int ix = 0; ix < P->nx; ++ix) {
        int j = iy * P->nx + ix;
        int nx = P->nx, ny = P->ny;
        c->nbr[j * 4 + 0] = ix > 0 ? j - 1 : (P->periodic ? iy * nx + nx - 1 : -1 - 0);
        c->nbr[j * 4 + 1] = ix < nx - 1 ? j + 1 : (P->periodic ? iy * nx : -1 - 1);
        c->nbr[j * 4 + 2] = iy > 0 ? j - nx : (P->periodic ? (ny - 1) * nx + ix : -1 - 2);
        c->nbr[j * 4 + 3] = iy < ny - 1 ? j + nx : (P->periodic ? ix : -1 - 3);
        double nn[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
        for (int f = 0; f < 4; ++f) {
          c->nrm[(j * 4 + f) * 2 + 0] = nn[f][0];
          c->nrm[(j * 4 + f) * 2 + 1] = nn[f][1];
        }
        c->coef[j * 4 + 0] = c->coef[j * 4 + 1] = 1.0 / dx;
        c->coef[j * 4 + 2] = c->coef[j * 4 + 3] = 1.0 / dy;
        c->area[j] = dx * dy;
        c->perim[j] = 2.0 * (dx + dy);
        c->xc[j * 2] = P->x0 + (ix + 0.5) * dx;
        c->xc[j * 2 + 1] = P->y0 + (iy + 0.5) * dy;
      }
  } else {
    /* triangles: neighbour across edge e = (v_e, v_{e+1}) found by brute-force edge matching
     * (sorted edge keys); outward normal of a counter-clockwise triangle is (dy, -dx)/|e|. */
    int T = P->n_tri;
    edge_t *E = (edge_t *)malloc(sizeof(edge_t) * 3 * T);
    for (int t = 0; t < T; ++t)
      for (int e = 0; e < 3; ++e) {
        int a = P->tri[t * 3 + e], b = P->tri[t * 3 + (e + 1) % 3];
        int lo = a < b ? a : b, hi = a < b ? b : a;
        E[t * 3 + e].key = (int64_t)lo * P->n_vert + hi;
        E[t * 3 + e].t = t;
        E[t * 3 + e].e = e;
      }
    qsort(E, 3 * T, sizeof(edge_t), edge_cmp);
    for (int t = 0; t < T; ++t)
      for (int e = 0; e < 3; ++e) c->nbr[t * 3 + e] = -1 - (P->tri_tag[t * 3 + e] < 0 ? 0 : P->tri_tag[t * 3 + e]);
    for (int i = 0; i + 1 < 3 * T; ++i)
      if (E[i].key == E[i + 1].key) {
        c->nbr[E[i].t * 3 + E[i].e] = E[i + 1].t;
        c->nbr[E[i + 1].t * 3 + E[i + 1].e] = E[i].t;
      }
    free(E);
    for (int t = 0; t < T; ++t) {
      const double *A = P->vert + 2 * P->tri[t * 3 + 0];
      const double *B = P->vert + 2 * P->tri[t * 3 + 1];
      const double *C = P->vert + 2 * P->tri[t * 3 + 2];
      double ar = 0.5 * ((B[0] - A[0]) * (C[1] - A[1]) - (C[0] - A[0]) * (B[1] - A[1]));
      c->area[t] = ar;
      c->perim[t] = 0.0;
      c->xc[t * 2] = (A[0] + B[0] + C[0]) / 3.0;
      c->xc[t * 2 + 1] = (A[1] + B[1] + C[1]) / 3.0;
      for (int e = 0; e < 3; ++e) {
        const double *V0 = P->vert + 2 * P->tri[t * 3 + e];
        const double *V1 = P->vert + 2 * P->tri[t * 3 + (e + 1) % 3];
        double dx = V1[0] - V0[0], dy = V1[1] - V0[1];
        double len = sqrt(dx * dx + dy * dy);
        c->nrm[(t * 3 + e) * 2 + 0] = dy / len;
        c->nrm[(t * 3 + e) * 2 + 1] = -dx / len;
        c->coef[t * 3 + e] = len / ar;
        c->perim[t] += len;
      }
    }
  }
}

orc_ctx *orc_create(const orc_problem *P) {
  orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
  c->P = *P;
  int p = P->p;
  c->N = orc_num_basis(p, P->M);
  c->Q = 1;
  if (P->quad_kind == 2)
    c->Q = orc_smolyak_cc(p, P->quad_level, NULL, NULL);
  else
    for (int d = 0; d < p; ++d) c->Q *= P->q1d;
  c->m = P->m;
  c->d = (P->mesh_kind == ORC_MESH_1D) ? 1 : 2;
  c->F = (P->mesh_kind == ORC_MESH_1D) ? 2 : (P->mesh_kind == ORC_MESH_CART2D ? 4 : 3);
  c->cells = (P->mesh_kind == ORC_MESH_1D) ? P->nx : (P->mesh_kind == ORC_MESH_CART2D ? P->nx * P->ny : P->n_tri);
  int N = c->N, Q = c->Q;
  c->idx = (int32_t *)malloc(sizeof(int32_t) * N * p);
  orc_multi_indices(p, P->M, c->idx);
  /* tensor rule (Gauss-Legendre or Clenshaw-Curtis), last dimension fastest, or the Smolyak sparse
   * grid; omega_k = w_k 2^-p (f_Xi = 2^-p) */
  double x1[129], w1[129];
  if (P->quad_kind == 1)
    orc_clenshaw_curtis(P->q1d, x1, w1);
  else if (P->quad_kind == 0)
    orc_gauss_legendre(P->q1d, x1, w1);
  c->xi = (double *)malloc(sizeof(double) * Q * p);
  c->omega = (double *)malloc(sizeof(double) * Q);
  c->Phi = (double *)malloc(sizeof(double) * Q * N);
  double *wsg = NULL;
  if (P->quad_kind == 2) {
    wsg = (double *)malloc(sizeof(double) * Q);
    orc_smolyak_cc(p, P->quad_level, c->xi, wsg);
  }
  for (int k = 0; k < Q; ++k) {
    double om = 1.0;
    if (P->quad_kind == 2) {
      for (int d = 0; d < p; ++d) om /= 2.0;
      om *= wsg[k];
    } else {
      int r = k;
      for (int d = p - 1; d >= 0; --d) {
        int kd = r % P->q1d;
        r /= P->q1d;
        c->xi[k * p + d] = x1[kd];
        om *= w1[kd] / 2.0;
      }
    }
    c->omega[k] = om;
    for (int i = 0; i < N; ++i) {
      double v = 1.0;
      for (int d = 0; d < p; ++d) v *= phi_1d(c->idx[i * p + d], c->xi[k * p + d]);
      c->Phi[k * N + i] = v;
    }
  }
  free(wsg);
  build_geometry(c);
  c->bc_u = (double *)calloc((size_t)4 * Q * c->m, sizeof(double));
  for (int t = 0; t < 4; ++t)
    if (P->bc_kind[t] == ORC_BC_STATE || P->bc_kind[t] == ORC_BC_FARFIELD)
      for (int k = 0; k < Q; ++k) spec_state(c, &P->bc_state[t], c->xi + k * p, c->bc_u + ((size_t)t * Q + k) * c->m);
  c->level = (int32_t *)calloc(c->cells, sizeof(int32_t));
  c->n_levels = P->n_levels;
  if (c->n_levels > 0) {
    for (int l = 0; l < c->n_levels; ++l) c->Nl[l] = orc_num_basis(p, P->level_M[l]);
  } else {
    c->Nl[0] = N;
  }
  /* per-level nested Clenshaw-Curtis rules (reading 36): level l's 1D points are every
   * (n_f - 1)/(n_l - 1)-th point of the finest rule (n = 2^k + 1 nest), tensor index last dimension
   * fastest, weights prod_d w_l[j_d] / 2 */
  if (c->n_levels > 0 && P->level_q1d[0] > 0) {
    int nf = P->level_q1d[c->n_levels - 1];
    int okq = (P->quad_kind == 1 && P->q1d == nf);
    for (int l = 0; l < c->n_levels && okq; ++l) {
      int nl = P->level_q1d[l];
      okq = nl >= 2 && nl <= nf && (nf - 1) % (nl - 1) == 0 && (l == 0 || nl >= P->level_q1d[l - 1]);
    }
    if (!okq) {
      orc_destroy(c);
      return NULL;
    }
    c->lq_on = 1;
    for (int l = 0; l < c->n_levels; ++l) {
      int nl = P->level_q1d[l], stride = (nf - 1) / (nl - 1), Ql = 1;
      double xl[129], wl[129];
      orc_clenshaw_curtis(nl, xl, wl);
      for (int d = 0; d < p; ++d) Ql *= nl;
      c->lQ[l] = Ql;
      c->lkf[l] = (int32_t *)malloc(sizeof(int32_t) * Ql);
      c->lw[l] = (double *)malloc(sizeof(double) * Ql);
      for (int q = 0; q < Ql; ++q) {
        int r = q, kf = 0, scale = 1;
        double w = 1.0;
        for (int d = p - 1; d >= 0; --d) {
          int jd = r % nl;
          r /= nl;
          kf += jd * stride * scale;
          scale *= nf;
          w *= wl[jd] / 2.0;
        }
        c->lkf[l][q] = kf;
        c->lw[l][q] = w;
      }
    }
  }
  if (P->hessian_kind == 1) {
    size_t per = (size_t)P->lbfgs_m * N * c->m;
    c->lb_S = (double *)calloc((size_t)c->cells * per, sizeof(double));
    c->lb_Y = (double *)calloc((size_t)c->cells * per, sizeof(double));
    c->lb_cnt = (int32_t *)calloc(c->cells, sizeof(int32_t));
    c->lb_n = (int32_t *)calloc(c->cells, sizeof(int32_t));
  }
#ifdef _OPENMP
  if (P->n_threads > 0) omp_set_num_threads(P->n_threads);
#endif
  return c;
}

void orc_destroy(orc_ctx *c) {
  if (!c) return;
  free(c->idx); free(c->xi); free(c->omega); free(c->Phi);
  free(c->lb_S); free(c->lb_Y); free(c->lb_cnt); free(c->lb_n);
  for (int l = 0; l < 8; ++l) {
    free(c->lkf[l]);
    free(c->lw[l]);
  }
  free(c->nbr); free(c->nrm); free(c->coef); free(c->area); free(c->perim); free(c->xc);
  free(c->bc_u); free(c->level);
  free(c);
}

int orc_N(const orc_ctx *c) { return c->N; }
int orc_Q(const orc_ctx *c) { return c->Q; }
int orc_cells(const orc_ctx *c) { return c->cells; }

void orc_get_quadrature(const orc_ctx *c, double *xi, double *omega, double *Phi) {
  if (xi) memcpy(xi, c->xi, sizeof(double) * c->Q * c->P.p);
  if (omega) memcpy(omega, c->omega, sizeof(double) * c->Q);
  if (Phi) memcpy(Phi, c->Phi, sizeof(double) * c->Q * c->N);
}

void orc_get_geometry(const orc_ctx *c, int32_t *nbr, double *nrm, double *coef, double *area) {
  int n = c->cells, F = c->F;
  if (nbr) memcpy(nbr, c->nbr, sizeof(int32_t) * n * F);
  if (nrm) memcpy(nrm, c->nrm, sizeof(double) * n * F * 2);
  if (coef) memcpy(coef, c->coef, sizeof(double) * n * F);
  if (area) memcpy(area, c->area, sizeof(double) * n);
}

static int cell_N(const orc_ctx *c, int j) { return c->n_levels > 0 ? c->Nl[c->level[j]] : c->N; }

/* ------------------------------------------------------------------------ */
/* Dual problem                                           */
/* ------------------------------------------------------------------------ */

/* Lambda_k = sum_i lambda_i phi_i(xi_k)  (lambda^T phi at node k) */
static void reconstruct(const orc_ctx *c, int Nl, const double *lam, int k, double *Lk) {
  int m = c->m, N = c->N;
  for (int a = 0; a < m; ++a) {
    double s = 0.0;
    for (int i = 0; i < Nl; ++i) s += lam[i * m + a] * c->Phi[k * N + i];
    Lk[a] = s;
  }
}

/* L(lambda; uhat) = <s_*(lambda^T phi)>_Q - sum_i lambda_i^T uhat_i */
int orc_dual_objective(const orc_ctx *c, int Nl, const double *lam, const double *uhat, double *L) {
  int m = c->m;
  double Lk[4], s = 0.0;
  orc_rule R = rule_of(c, Nl);
  for (int q = 0; q < R.Q; ++q) {
    reconstruct(c, Nl, lam, RK(R, q), Lk);
    s += R.w[q] * orc_closure_sstar(c, Lk);
  }
  for (int i = 0; i < Nl; ++i)
    for (int a = 0; a < m; ++a) s -= lam[i * m + a] * uhat[i * m + a];
  *L = s;
  return isfinite(s);
}

/* grad L = <u_s(lambda^T phi) phi^T>_Q^T - uhat */
int orc_dual_gradient(const orc_ctx *c, int Nl, const double *lam, const double *uhat, double *g) {
  int m = c->m, N = c->N;
  double Lk[4], uk[4];
  for (int i = 0; i < Nl; ++i)
    for (int a = 0; a < m; ++a) g[i * m + a] = 0.0;
  orc_rule R = rule_of(c, Nl);
  for (int q = 0; q < R.Q; ++q) {
    int k = RK(R, q);
    reconstruct(c, Nl, lam, k, Lk);
    if (!orc_closure_u(c, Lk, uk)) return 0;
    for (int i = 0; i < Nl; ++i)
      for (int a = 0; a < m; ++a) g[i * m + a] += R.w[q] * uk[a] * c->Phi[k * N + i];
  }
  int ok = 1;
  for (int i = 0; i < Nl; ++i)
    for (int a = 0; a < m; ++a) {
      g[i * m + a] -= uhat[i * m + a];
      if (!isfinite(g[i * m + a])) ok = 0;
    }
  return ok;
}

/* h(lambda) = <u_s(lambda^T phi) phi^T>_Q^T */
int orc_moments_from_dual(const orc_ctx *c, int Nl, const double *lam, double *uhat) {
  int n = Nl * c->m;
  double *zero = (double *)calloc(n, sizeof(double));
  int ok = orc_dual_gradient(c, Nl, lam, zero, uhat);
  free(zero);
  return ok;
}

/* H = <grad u_s(lambda^T phi) (x) phi phi^T>_Q^T, full n x n, vec index (i,a) -> i*m+a */
int orc_dual_hessian(const orc_ctx *c, int Nl, const double *lam, double *H) {
  int m = c->m, N = c->N, n = Nl * m;
  double Lk[4], J[16];
  for (int r = 0; r < n * n; ++r) H[r] = 0.0;
  orc_rule R = rule_of(c, Nl);
  for (int q = 0; q < R.Q; ++q) {
    int k = RK(R, q);
    reconstruct(c, Nl, lam, k, Lk);
    if (!orc_closure_du(c, Lk, J)) return 0;
    for (int i = 0; i < Nl; ++i)
      for (int a = 0; a < m; ++a)
        for (int j = 0; j < Nl; ++j)
          for (int b = 0; b < m; ++b)
            H[(i * m + a) * n + (j * m + b)] += R.w[q] * J[a * m + b] * c->Phi[k * N + i] * c->Phi[k * N + j];
  }
  return 1;
}

/* stopping quantity sum_a ||g_{.,a}||_2 (reading 1) */
static double crit_of(const double *g, int Nl, int m) {
  double s = 0.0;
  for (int a = 0; a < m; ++a) {
    double q = 0.0;
    for (int i = 0; i < Nl; ++i) q += g[i * m + a] * g[i * m + a];
    s += sqrt(q);
  }
  return s;
}

/* Textbook Cholesky H = L L^T, then L L^T d = -g */
static int cholesky_solve(double *H, int n, const double *g, double *d) {
  for (int j = 0; j < n; ++j) {
    double s = H[j * n + j];
    for (int k = 0; k < j; ++k) s -= H[j * n + k] * H[j * n + k];
    if (!(s > 0.0) || !isfinite(s)) return 0;
    double Ljj = sqrt(s);
    H[j * n + j] = Ljj;
    for (int i = j + 1; i < n; ++i) {
      double t = H[i * n + j];
      for (int k = 0; k < j; ++k) t -= H[i * n + k] * H[j * n + k];
      H[i * n + j] = t / Ljj;
    }
  }
  /* forward: L y = -g */
  for (int i = 0; i < n; ++i) {
    double t = -g[i];
    for (int k = 0; k < i; ++k) t -= H[i * n + k] * d[k];
    d[i] = t / H[i * n + i];
  }
  /* backward: L^T d = y */
  for (int i = n - 1; i >= 0; --i) {
    double t = d[i];
    for (int k = i + 1; k < n; ++k) t -= H[k * n + i] * d[k];
    d[i] = t / H[i * n + i];
  }
  return 1;
}

/* L together with the magnitude of the terms it sums (rounding scale of L):
 *   scale = <|s_*(lambda^T phi)|>_Q + sum_i |lambda_i^T uhat_i|  */
static int objective_and_scale(const orc_ctx *c, int Nl, const double *lam, const double *uhat,
                               double *L, double *scale) {
  int m = c->m;
  double Lk[4], s = 0.0, sc = 0.0;
  orc_rule R = rule_of(c, Nl);
  for (int q = 0; q < R.Q; ++q) {
    reconstruct(c, Nl, lam, RK(R, q), Lk);
    double sk = orc_closure_sstar(c, Lk);
    s += R.w[q] * sk;
    sc += R.w[q] * fabs(sk);
  }
  for (int i = 0; i < Nl; ++i)
    for (int a = 0; a < m; ++a) {
      s -= lam[i * m + a] * uhat[i * m + a];
      sc += fabs(lam[i * m + a] * uhat[i * m + a]);
    }
  *L = s;
  *scale = sc;
  return isfinite(s);
}

/* ---- L-BFGS direction (reading 35) -----------------------------
 * PAPER.md:843 proposes BFGS Hessian approximations built "from previously computed gradients", with
 * gradients "from a certain number of old time steps ... saved in every spatial cell".  Here: the
 * limited-memory BFGS inverse-Hessian approximation of Nocedal & Wright (the paper's reference
 * [nocedal2006numerical]; two-loop recursion, Alg. 7.4) over the cell's most recent pairs
 * s = lambda^{(l+1)} - lambda^{(l)}, y = grad L(lambda^{(l+1)}) - grad L(lambda^{(l)}), with the initial
 * matrix H0 = I_N (x) Jbar^{-1}, Jbar = <grad u_s(lambda^T phi)>_Q (m x m): the exact inverse Hessian
 * when lambda^T phi does not depend on xi, because <phi phi^T>_Q = I. */
int orc_lbfgs_jbar(const orc_ctx *c, int Nl, const double *lam, double *Jbar) {
  int m = c->m;
  double Lk[4], J[16];
  for (int r = 0; r < m * m; ++r) Jbar[r] = 0.0;
  orc_rule R = rule_of(c, Nl);
  for (int q = 0; q < R.Q; ++q) {
    reconstruct(c, Nl, lam, RK(R, q), Lk);
    if (!orc_closure_du(c, Lk, J)) return 0;
    for (int r = 0; r < m * m; ++r) Jbar[r] += R.w[q] * J[r];
  }
  return 1;
}

int orc_lbfgs_direction(const orc_ctx *c, int Nl, const double *lam, const double *g, const double *S,
                        const double *Y, int cnt, double *d) {
  int m = c->m, n = Nl * m;
  double *q = (double *)malloc(sizeof(double) * n);
  double al[64], Jb[16];
  for (int r = 0; r < n; ++r) q[r] = g[r];
  /* first loop, newest pair first: alpha_i = rho_i s_i^T q, q -= alpha_i y_i */
  for (int i = 0; i < cnt; ++i) {
    const double *si = S + (size_t)i * n, *yi = Y + (size_t)i * n;
    double sy = 0.0, sq = 0.0;
    for (int r = 0; r < n; ++r) {
      sy += si[r] * yi[r];
      sq += si[r] * q[r];
    }
    al[i] = sq / sy;
    for (int r = 0; r < n; ++r) q[r] -= al[i] * yi[r];
  }
  /* r = H0 q: solve Jbar r_i = q_i for every moment i (m x m Cholesky) */
  int ok = orc_lbfgs_jbar(c, Nl, lam, Jb);
  if (ok) {
    double L[16] = {0};
    for (int j = 0; j < m && ok; ++j) {
      double t = Jb[j * m + j];
      for (int k = 0; k < j; ++k) t -= L[j * m + k] * L[j * m + k];
      if (!(t > 0.0) || !isfinite(t)) { ok = 0; break; }
      L[j * m + j] = sqrt(t);
      for (int i = j + 1; i < m; ++i) {
        double v = Jb[i * m + j];
        for (int k = 0; k < j; ++k) v -= L[i * m + k] * L[j * m + k];
        L[i * m + j] = v / L[j * m + j];
      }
    }
    for (int i = 0; i < Nl && ok; ++i) {
      double *qi = q + i * m, y[4];
      for (int a = 0; a < m; ++a) {
        double v = qi[a];
        for (int k = 0; k < a; ++k) v -= L[a * m + k] * y[k];
        y[a] = v / L[a * m + a];
      }
      for (int a = m - 1; a >= 0; --a) {
        double v = y[a];
        for (int k = a + 1; k < m; ++k) v -= L[k * m + a] * qi[k];
        qi[a] = v / L[a * m + a];
      }
    }
  }
  /* second loop, oldest pair first: beta = rho_i y_i^T r, r += s_i (alpha_i - beta) */
  for (int i = cnt - 1; i >= 0 && ok; --i) {
    const double *si = S + (size_t)i * n, *yi = Y + (size_t)i * n;
    double sy = 0.0, yr = 0.0;
    for (int r = 0; r < n; ++r) {
      sy += si[r] * yi[r];
      yr += yi[r] * q[r];
    }
    double be = yr / sy;
    for (int r = 0; r < n; ++r) q[r] += si[r] * (al[i] - be);
  }
  for (int r = 0; r < n; ++r) d[r] = -q[r];
  free(q);
  return ok;
}

/* the pair (s, y) enters the history if s^T y > 1e-10 |s| |y| (curvature condition with a rounding
 * margin; s^T y > 0 holds for every s != 0 in exact arithmetic because L is strictly convex); the
 * oldest pair drops out when lbfgs_m pairs are stored */
static void lbfgs_push(int mh, int n, double *S, double *Y, int32_t *cnt, const double *s, const double *y) {
  double sy = 0.0, ss = 0.0, yy = 0.0;
  for (int r = 0; r < n; ++r) {
    sy += s[r] * y[r];
    ss += s[r] * s[r];
    yy += y[r] * y[r];
  }
  if (!(sy > 1e-10 * sqrt(ss * yy))) return;
  int keep = *cnt < mh ? *cnt : mh - 1;
  for (int i = keep; i > 0; --i) {
    memcpy(S + (size_t)i * n, S + (size_t)(i - 1) * n, sizeof(double) * n);
    memcpy(Y + (size_t)i * n, Y + (size_t)(i - 1) * n, sizeof(double) * n);
  }
  memcpy(S, s, sizeof(double) * n);
  memcpy(Y, y, sizeof(double) * n);
  *cnt = keep + 1;
}

/* Newton iteration lambda^{(l+1)} = d(lambda^{(l)}; uhat) until the stopping
 * criterion holds (FULL, Alg. 1 lines 7-10) or once (ONE_STEP, Alg. 2 line 5),
 * globalised by Armijo backtracking on the dual objective L with a rounding
 * allowance (reading 3'):  accept alpha if the trial is admissible and
 *     L(lambda + alpha d) <= L(lambda) + c alpha grad L . d + 1e-12 scale(L).
 * With lb_S != NULL the direction is the L-BFGS one over the cell's history (reading 35) instead of
 * the exact Newton direction -H^{-1} g; everything else is the same iteration. */
static int dual_solve_cell_impl(const orc_ctx *c, int Nl, int mode, const double *uhat, double *lam,
                                int32_t *iters, double *crit_out, int32_t *halvings, int32_t *inadmissible,
                                double *lb_S, double *lb_Y, int32_t *lb_cnt, int32_t *lb_n) {
  const orc_problem *P = &c->P;
  int m = c->m, n = Nl * m;
  double *g = (double *)malloc(sizeof(double) * n);
  double *g0 = (double *)malloc(sizeof(double) * n);
  double *dd = (double *)malloc(sizeof(double) * n);
  double *lt = (double *)malloc(sizeof(double) * n);
  double *H = lb_S ? NULL : (double *)malloc(sizeof(double) * n * n);
  int status = ORC_OK, l = 0, nhalv = 0, ninad = 0; /* rejected trials; inadmissible among them */
  int cap = P->max_newton;
  double crit = INFINITY;
  if (lb_S && *lb_n != n) { /* history of another basis size (level change): start afresh */
    *lb_cnt = 0;
    *lb_n = n;
  }
  if (!orc_dual_gradient(c, Nl, lam, uhat, g)) {
    status = ORC_INADMISSIBLE;
    goto done;
  }
  for (;;) {
    crit = crit_of(g, Nl, m);
    if (crit < P->tau) break;
    if (mode == ORC_NEWTON_ONE_STEP && l == 1) break;
    /* reading 5: at most max_newton steps.  Reading 35: a quasi-Newton solve that has not converged
     * after max_newton steps continues with (at most max_newton) exact Newton steps from its iterate,
     * and the cell's pairs are dropped (measured on the config-3 stress state: mean 10-18 quasi-Newton
     * steps, p99 18-40; ~2e-4 of the cells stagnate and would not converge in 1600) */
    if (l == cap) {
      if (lb_S) {
        lb_S = NULL;
        *lb_cnt = 0;
        cap = l + P->max_newton;
        H = (double *)malloc(sizeof(double) * n * n);
        continue;
      }
      status = ORC_NONCONVERGENCE;
      break;
    }
    double slope = 0.0;
    if (lb_S) {
      if (!orc_lbfgs_direction(c, Nl, lam, g, lb_S, lb_Y, *lb_cnt, dd)) {
        status = ORC_ILLCONDITIONED;
        break;
      }
      for (int r = 0; r < n; ++r) slope += g[r] * dd[r];
      if (!(slope < 0.0) && *lb_cnt > 0) { /* not a descent direction (rounding): drop the history */
        *lb_cnt = 0;
        orc_lbfgs_direction(c, Nl, lam, g, lb_S, lb_Y, 0, dd);
        slope = 0.0;
        for (int r = 0; r < n; ++r) slope += g[r] * dd[r];
      }
    } else {
      if (!orc_dual_hessian(c, Nl, lam, H) || !cholesky_solve(H, n, g, dd)) {
        status = ORC_ILLCONDITIONED;
        break;
      }
      for (int r = 0; r < n; ++r) slope += g[r] * dd[r];
    }
    double L0, scale;
    objective_and_scale(c, Nl, lam, uhat, &L0, &scale);
    memcpy(g0, g, sizeof(double) * n);
    double alpha = 1.0;
    int accepted = 0;
    for (int h = 0; h <= P->max_halvings; ++h) {
      for (int r = 0; r < n; ++r) lt[r] = lam[r] + alpha * dd[r];
      double Lt, sct;
      int admissible = objective_and_scale(c, Nl, lt, uhat, &Lt, &sct);
      if (admissible && Lt <= L0 + P->armijo_c * alpha * slope + 1e-12 * scale &&
          orc_dual_gradient(c, Nl, lt, uhat, g)) {
        accepted = 1;
        break;
      }
      ++nhalv;
      if (!admissible) ++ninad;
      alpha *= 0.5;
    }
    if (!accepted) {
      memcpy(g, g0, sizeof(double) * n);
      status = ORC_LINESEARCH;
      break;
    }
    if (lb_S) { /* pair s = lt - lam, y = g - g0 */
      for (int r = 0; r < n; ++r) {
        dd[r] = lt[r] - lam[r];
        g0[r] = g[r] - g0[r];
      }
      lbfgs_push(P->lbfgs_m, n, lb_S, lb_Y, lb_cnt, dd, g0);
    }
    memcpy(lam, lt, sizeof(double) * n);
    ++l;
  }
done:
  if (iters) *iters = l;
  if (crit_out) *crit_out = crit;
  if (halvings) *halvings = nhalv;
  if (inadmissible) *inadmissible = ninad;
  free(g); free(g0); free(dd); free(lt); free(H);
  return status;
}

int orc_dual_solve_cell_ls(const orc_ctx *c, int Nl, int mode, const double *uhat, double *lam,
                           int32_t *iters, double *crit_out, int32_t *halvings, int32_t *inadmissible) {
  return dual_solve_cell_impl(c, Nl, mode, uhat, lam, iters, crit_out, halvings, inadmissible, NULL, NULL, NULL,
                              NULL);
}

int orc_lbfgs_history(const orc_ctx *c, int j, double *S, double *Y) {
  if (!c->lb_S) return 0;
  size_t per = (size_t)c->P.lbfgs_m * c->N * c->m;
  int cnt = c->lb_cnt[j], n = c->lb_n[j];
  for (int i = 0; i < cnt; ++i) {
    if (S) memcpy(S + (size_t)i * c->N * c->m, c->lb_S + j * per + (size_t)i * n, sizeof(double) * n);
    if (Y) memcpy(Y + (size_t)i * c->N * c->m, c->lb_Y + j * per + (size_t)i * n, sizeof(double) * n);
  }
  return cnt;
}

int orc_level_rule(const orc_ctx *c, int l, int32_t *kf, double *w) {
  if (!c->lq_on || l < 0 || l >= c->n_levels) {
    for (int k = 0; k < c->Q; ++k) {
      if (kf) kf[k] = k;
      if (w) w[k] = c->omega[k];
    }
    return c->Q;
  }
  if (kf) memcpy(kf, c->lkf[l], sizeof(int32_t) * c->lQ[l]);
  if (w) memcpy(w, c->lw[l], sizeof(double) * c->lQ[l]);
  return c->lQ[l];
}

void orc_lbfgs_reset(orc_ctx *c) {
  if (c->lb_cnt) memset(c->lb_cnt, 0, sizeof(int32_t) * c->cells);
}

int orc_dual_solve_cell(const orc_ctx *c, int Nl, int mode, const double *uhat, double *lam,
                        int32_t *iters, double *crit_out) {
  return orc_dual_solve_cell_ls(c, Nl, mode, uhat, lam, iters, crit_out, NULL, NULL);
}

/* ------------------------------------------------------------------------ */
/* Whole-field operations                                                     */
/* ------------------------------------------------------------------------ */

static double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

/* cell average of the piecewise-constant IC at node xi_k (exact fractions of the cell on each side
 * of the split lines, reading 17) */
static void ic_node_state(const orc_ctx *c, const orc_ic *ic, int j, int k, double *ub) {
  const orc_problem *P = &c->P;
  int m = c->m, p = P->p;
  const double *xi = c->xi + k * p;
  double us[4][4];
  for (int a = 0; a < 4; ++a) ub[a] = 0.0;
  if (ic->kind == ORC_IC_UNIFORM) {
    spec_state(c, &ic->state[0], xi, ub);
    return;
  }
  double xs = ic->xs0, ys = ic->ys0;
  for (int d = 0; d < p && d < 3; ++d) {
    xs += ic->xs1[d] * xi[d];
    ys += ic->ys1[d] * xi[d];
  }
  int nreg = ic->kind == ORC_IC_STEP1D ? 2 : 4;
  for (int r = 0; r < nreg; ++r) spec_state(c, &ic->state[r], xi, us[r]);
  if (P->mesh_kind == ORC_MESH_1D) {
    double dx = (P->x1 - P->x0) / P->nx;
    double xl = P->x0 + j * dx;
    double fl = clamp01((xs - xl) / dx); /* fraction of the cell left of x_s */
    for (int a = 0; a < m; ++a) ub[a] = fl * us[0][a] + (1.0 - fl) * us[1][a];
  } else {
    int ix = j % P->nx, iy = j / P->nx;
    double dx = (P->x1 - P->x0) / P->nx, dy = (P->y1 - P->y0) / P->ny;
    double fx = clamp01((xs - (P->x0 + ix * dx)) / dx); /* fraction with x < x_s */
    double fy = clamp01((ys - (P->y0 + iy * dy)) / dy); /* fraction with y < y_s */
    for (int a = 0; a < m; ++a)
      ub[a] = (1.0 - fx) * (1.0 - fy) * us[0][a] + fx * (1.0 - fy) * us[1][a] + fx * fy * us[2][a] +
              (1.0 - fx) * fy * us[3][a];
  }
}

/* u_j^0 = (1/|Omega_j|) int <u_IC phi>_Q dx with exact cell averages of the piecewise-constant IC
 * at every node (Alg. 1 line 2; reading 17). */
void orc_project_ic(const orc_ctx *c, const orc_ic *ic, double *uhat) {
  int N = c->N, m = c->m;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < c->cells; ++j) {
    int Nl = cell_N(c, j);
    orc_rule R = rule_of(c, Nl); /* Alg. 3 line 3: <u_IC phi_l>_{Q_l} at the initial level */
    double *uj = uhat + (size_t)j * N * m;
    for (int r = 0; r < N * m; ++r) uj[r] = 0.0;
    for (int q = 0; q < R.Q; ++q) {
      int k = RK(R, q);
      double ub[4];
      ic_node_state(c, ic, j, k, ub);
      for (int i = 0; i < Nl; ++i)
        for (int a = 0; a < m; ++a) uj[i * m + a] += R.w[q] * ub[a] * c->Phi[k * N + i];
    }
  }
}

/* lambda^(0) at t=0: e_0 (x) grad s(uhat_0) (reading 6) */
void orc_warm_start(const orc_ctx *c, const double *uhat, double *lam) {
  int N = c->N, m = c->m;
  for (int j = 0; j < c->cells; ++j) {
    double *lj = lam + (size_t)j * N * m;
    for (int r = 0; r < N * m; ++r) lj[r] = 0.0;
    orc_closure_grad_s(c, uhat + (size_t)j * N * m, lj);
  }
}

int orc_retard_stage(const orc_ctx *c) { return c->retard_stage; }
size_t orc_problem_size(void) { return sizeof(orc_problem); }
void orc_set_levels(orc_ctx *c, const int32_t *levels) { memcpy(c->level, levels, sizeof(int32_t) * c->cells); }
void orc_get_levels(const orc_ctx *c, int32_t *levels) { memcpy(levels, c->level, sizeof(int32_t) * c->cells); }

/* Alg. 1 lines 4-10 (FULL) / Alg. 2 line 5 (ONE_STEP) for every cell */
void orc_dual_solve_all_ls(const orc_ctx *c, const double *uhat, double *lam, int32_t *iters,
                           int32_t *status, double *crit, int32_t *halvings, int32_t *inadmissible) {
  int N = c->N, m = c->m;
#pragma omp parallel for schedule(dynamic, 1)
  for (int j = 0; j < c->cells; ++j) {
    int32_t it = 0, hv = 0, ia = 0;
    double cr = 0.0;
    int st;
    if (c->lb_S) { /* L-BFGS with the cell's history (reading 35) */
      size_t per = (size_t)c->P.lbfgs_m * N * m;
      st = dual_solve_cell_impl(c, cell_N(c, j), c->P.newton_mode, uhat + (size_t)j * N * m, lam + (size_t)j * N * m,
                                &it, &cr, &hv, &ia, ((orc_ctx *)c)->lb_S + j * per, ((orc_ctx *)c)->lb_Y + j * per,
                                ((orc_ctx *)c)->lb_cnt + j, ((orc_ctx *)c)->lb_n + j);
    } else {
      st = orc_dual_solve_cell_ls(c, cell_N(c, j), c->P.newton_mode, uhat + (size_t)j * N * m,
                                  lam + (size_t)j * N * m, &it, &cr, &hv, &ia);
    }
    if (iters) iters[j] = it;
    if (status) status[j] = st;
    if (crit) crit[j] = cr;
    if (halvings) halvings[j] = hv;
    if (inadmissible) inadmissible[j] = ia;
  }
}

void orc_dual_solve_all(const orc_ctx *c, const double *uhat, double *lam, int32_t *iters,
                        int32_t *status, double *crit) {
  orc_dual_solve_all_ls(c, uhat, lam, iters, status, crit, NULL, NULL);
}

/* node states u_k^{(j)} = u_s(lambda_j^T phi(xi_k)) for all cells */
static int node_states(const orc_ctx *c, const double *lam, double *U) {
  int N = c->N, m = c->m, Q = c->Q, bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
  for (int j = 0; j < c->cells; ++j) {
    double Lk[4];
    for (int k = 0; k < Q; ++k) {
      reconstruct(c, cell_N(c, j), lam + (size_t)j * N * m, k, Lk);
      if (!orc_closure_u(c, Lk, U + ((size_t)j * Q + k) * m)) bad++;
    }
  }
  return bad == 0;
}

/* CFL rate of cell j: largest wave speed over its nodes and the ghost states of its boundary faces,
 * times the mesh factor (reading 15). */
static double state_rate(const orc_ctx *c, const double *u, int j) {
  const orc_problem *P = &c->P;
  if (P->mesh_kind == ORC_MESH_1D) {
    double n1[2] = {1.0, 0.0};
    return wave_speed(c, u, n1) * c->coef[j * 2];
  }
  if (P->mesh_kind == ORC_MESH_CART2D) {
    double nx[2] = {1.0, 0.0}, ny[2] = {0.0, 1.0};
    return wave_speed(c, u, nx) * c->coef[j * 4 + 0] + wave_speed(c, u, ny) * c->coef[j * 4 + 2];
  }
  return speed_norm(c, u) * c->perim[j] / c->area[j];
}

/* CFL rate of cell j: largest wave speed over its nodes (those of its current level's rule, reading
 * 36) and the ghost states of its boundary faces, times the mesh factor (reading 15); with per-level
 * rules prescribed (STATE) ghost states enter at every node of the finest rule. */
static double cell_rate(const orc_ctx *c, const double *U, int j) {
  const orc_problem *P = &c->P;
  int Q = c->Q, m = c->m, F = c->F;
  double rate = 0.0;
  orc_rule R = rule_of(c, cell_N(c, j));
  for (int q = 0; q < R.Q; ++q) {
    int k = RK(R, q);
    const double *u = U + ((size_t)j * Q + k) * m;
    double r = state_rate(c, u, j);
    if (r > rate) rate = r;
    for (int f = 0; f < F; ++f) {
      int nb = c->nbr[j * F + f];
      if (nb >= 0) continue;
      double ug[4];
      /* reading 37: a far-field face enters the rate with its free-stream state */
      if (P->bc_kind[-1 - nb] == ORC_BC_FARFIELD)
        memcpy(ug, c->bc_u + ((size_t)(-1 - nb) * Q + k) * m, sizeof(double) * m);
      else
        ghost_state(c, -1 - nb, k, u, c->nrm + (j * F + f) * 2, ug);
      double rg = state_rate(c, ug, j);
      if (rg > rate) rate = rg;
    }
  }
  if (c->lq_on)
    for (int f = 0; f < F; ++f) {
      int nb = c->nbr[j * F + f];
      if (nb >= 0 || (P->bc_kind[-1 - nb] != ORC_BC_STATE && P->bc_kind[-1 - nb] != ORC_BC_FARFIELD)) continue;
      for (int k = 0; k < Q; ++k) {
        double rg = state_rate(c, c->bc_u + ((size_t)(-1 - nb) * Q + k) * m, j);
        if (rg > rate) rate = rg;
      }
    }
  return rate;
}

/* Delta t = CFL / max_j rate_j, clipped to the remaining time (reading 15). */
static double dt_from_states(const orc_ctx *c, const double *U, double t_remaining) {
  double rate = 0.0;
  for (int j = 0; j < c->cells; ++j) {
    double r = cell_rate(c, U, j);
    if (r > rate) rate = r;
  }
  double dt = c->P.cfl / rate;
  return dt < t_remaining ? dt : t_remaining;
}

void orc_cell_rates(const orc_ctx *c, const double *lam, double *rates) {
  double *U = (double *)malloc(sizeof(double) * (size_t)c->cells * c->Q * c->m);
  node_states(c, lam, U);
  for (int j = 0; j < c->cells; ++j) rates[j] = cell_rate(c, U, j);
  free(U);
}

double orc_compute_dt(const orc_ctx *c, const double *lam, double t_remaining) {
  double *U = (double *)malloc(sizeof(double) * (size_t)c->cells * c->Q * c->m);
  double dt = node_states(c, lam, U) ? dt_from_states(c, U, t_remaining) : NAN;
  free(U);
  return dt;
}

/* Moment update:
 *   r_{j,k} = 1D:   (g(u_j,u_{j+1}) - g(u_{j-1},u_j)) / dx                        (eq. IPMDiscretization)
 *             cart: (G_{i+1/2}-G_{i-1/2})/dx + (H_{j+1/2}-H_{j-1/2})/dy           (dimension by dimension)
 *             tri:  sum_e |e|/|Omega_j| g(u_j, u_nb; n_e)                          (edge sum)
 *   CONSERVATIVE: uhat^{n+1} = uhat^n - dt <r phi^T>_Q^T                          (reading 13)
 *   PAPER_C:      uhat^{n+1} = <(u^{(j)} - dt r) phi_{l^{n+1}}^T>_Q^T */
/* kinetic-flux residual r_{j,k} of node k of cell j from the node states U [cells][Q][m] (the
 * formulas in the comment above) */
static void node_residual(const orc_ctx *c, const double *U, int j, int k, double dx_over_dt, double *r) {
  const orc_problem *P = &c->P;
  int m = c->m, Q = c->Q, F = c->F;
  const double *uj = U + ((size_t)j * Q + k) * m;
  double nb_u[4][4];
  for (int f = 0; f < F; ++f) {
    int nb = c->nbr[j * F + f];
    if (nb >= 0)
      memcpy(nb_u[f], U + ((size_t)nb * Q + k) * m, sizeof(double) * m);
    else
      ghost_state(c, -1 - nb, k, uj, c->nrm + (j * F + f) * 2, nb_u[f]);
  }
  double gp[4], gm[4];
  for (int a = 0; a < 4; ++a) r[a] = 0.0;
  if (P->mesh_kind == ORC_MESH_1D) {
    double n1[2] = {1.0, 0.0};
    orc_flux_g(c, uj, nb_u[1], n1, dx_over_dt, gp);    /* g_{j+1/2} = g(u_j, u_{j+1}) */
    orc_flux_g(c, nb_u[0], uj, n1, dx_over_dt, gm);    /* g_{j-1/2} = g(u_{j-1}, u_j) */
    for (int a = 0; a < m; ++a) r[a] = (gp[a] - gm[a]) * c->coef[j * 2];
  } else if (P->mesh_kind == ORC_MESH_CART2D) {
    double nx[2] = {1.0, 0.0}, ny[2] = {0.0, 1.0};
    orc_flux_g(c, uj, nb_u[1], nx, 0.0, gp);
    orc_flux_g(c, nb_u[0], uj, nx, 0.0, gm);
    for (int a = 0; a < m; ++a) r[a] = (gp[a] - gm[a]) * c->coef[j * 4 + 0];
    orc_flux_g(c, uj, nb_u[3], ny, 0.0, gp);
    orc_flux_g(c, nb_u[2], uj, ny, 0.0, gm);
    for (int a = 0; a < m; ++a) r[a] += (gp[a] - gm[a]) * c->coef[j * 4 + 2];
  } else {
    for (int f = 0; f < F; ++f) {
      orc_flux_g(c, uj, nb_u[f], c->nrm + (j * F + f) * 2, 0.0, gp);
      for (int a = 0; a < m; ++a) r[a] += c->coef[j * F + f] * gp[a];
    }
  }
}

static void flux_update_states(const orc_ctx *c, const double *U, const int32_t *new_level,
                               const double *uhat_old, double *uhat_new, double dt) {
  const orc_problem *P = &c->P;
  int N = c->N, m = c->m, Q = c->Q;
  double dx_over_dt = (P->mesh_kind == ORC_MESH_1D) ? ((P->x1 - P->x0) / P->nx) / dt : 0.0;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < c->cells; ++j) {
    int Nnew = c->n_levels > 0 ? c->Nl[new_level[j]] : N;
    double *un = uhat_new + (size_t)j * N * m;
    const double *uo = uhat_old + (size_t)j * N * m;
    double acc[224 * 4];
    for (int r = 0; r < N * m; ++r) acc[r] = 0.0;
    /* eq. (adaptiveFVUpdate): the update at level l^{n+1} integrates with Q_{l^{n+1}};
     * the stencil's states at those nodes come from their duals at the old levels (U holds every cell
     * at every node of the finest rule: the neighbours "evaluated at the finer quadrature level",
     * PAPER.md:398) */
    orc_rule R = rule_of(c, Nnew);
    for (int q = 0; q < R.Q; ++q) {
      int k = RK(R, q);
      const double *uj = U + ((size_t)j * Q + k) * m;
      double r[4];
      node_residual(c, U, j, k, dx_over_dt, r);
      for (int i = 0; i < Nnew; ++i)
        for (int a = 0; a < m; ++a) {
          if (P->update_form == ORC_UPDATE_PAPER_C)
            acc[i * m + a] += R.w[q] * (uj[a] - dt * r[a]) * c->Phi[k * N + i];
          else
            acc[i * m + a] += R.w[q] * r[a] * c->Phi[k * N + i];
        }
    }
    for (int i = 0; i < N; ++i)
      for (int a = 0; a < m; ++a) {
        double v;
        if (i >= Nnew)
          v = 0.0;
        else if (P->update_form == ORC_UPDATE_PAPER_C)
          v = acc[i * m + a];
        else
          v = uo[i * m + a] - dt * acc[i * m + a];
        un[i * m + a] = v;
      }
  }
}

void orc_flux_update(orc_ctx *c, const double *lam, const double *uhat_old, double *uhat_new, double dt) {
  double *U = (double *)malloc(sizeof(double) * (size_t)c->cells * c->Q * c->m);
  node_states(c, lam, U);
  flux_update_states(c, U, c->level, uhat_old, uhat_new, dt);
  free(U);
}

/* smoothness indicator on the first state component (reading 19-20):
 *   S = sum_{M_{l-1} < |i| <= M_l} h_{i,0}^2 / sum_{|i| <= M_l} h_{i,0}^2 */
double orc_indicator(const orc_ctx *c, int lvl, const double *h) {
  int m = c->m;
  int Nl = c->Nl[lvl];
  int Nprev = lvl > 0 ? c->Nl[lvl - 1] : orc_num_basis(c->P.p, c->P.level_M[0] - 1);
  double num = 0.0, den = 0.0;
  for (int i = 0; i < Nl; ++i) {
    den += h[i * m] * h[i * m];
    if (i >= Nprev) num += h[i * m] * h[i * m];
  }
  return den > 0.0 ? num / den : 0.0;
}

/* One step of Algorithm 1 (FULL) / 2 (ONE_STEP) / 3-4 structure (levels), PAPER.md:196-217,
 * 252-269, 400-450; refinement retardation (Alg. 4) when n_retard > 0. */
int orc_step(orc_ctx *c, double *uhat, double *lam, double t_remaining, int32_t *iters,
             int32_t *status, double *dt_used, double *residual) {
  int N = c->N, m = c->m, Q = c->Q, cells = c->cells;
  int32_t *st = (int32_t *)malloc(sizeof(int32_t) * cells);
  int32_t *newlev = (int32_t *)malloc(sizeof(int32_t) * cells);
  orc_dual_solve_all(c, uhat, lam, iters, st, NULL);
  int worst = 0;
  for (int j = 0; j < cells; ++j) {
    if (st[j] > worst) worst = st[j];
    if (status) status[j] = st[j];
  }
  /* refinement level l^{n+1} from h(lambda^{n+1}) at level l^n (Alg. 3 line 15) */
  memcpy(newlev, c->level, sizeof(int32_t) * cells);
  if (c->n_levels > 0) {
#pragma omp parallel for schedule(static)
    for (int j = 0; j < cells; ++j) {
      int lvl = c->level[j];
      double h[224 * 4];
      orc_moments_from_dual(c, c->Nl[lvl], lam + (size_t)j * N * m, h);
      double S = orc_indicator(c, lvl, h);
      int nl = lvl;
      /* reading 34: a cell whose dual solve ended INADMISSIBLE (no admissible iterate, h(lambda) is
       * undefined) keeps its level; every other cell follows the indicator */
      if (st[j] == ORC_INADMISSIBLE) nl = lvl;
      else if (S < c->P.delta_dec && lvl > 0) nl = lvl - 1;
      else if (S > c->P.delta_inc && lvl < c->n_levels - 1) nl = lvl + 1;
      /* Alg. 4 line 6: the current stage's maximal level l*_l (reading 31: a cap) */
      if (c->P.n_retard > 0 && c->retard_stage < c->P.n_retard && nl > c->P.retard_level[c->retard_stage])
        nl = c->P.retard_level[c->retard_stage];
      newlev[j] = nl;
    }
  }
  double *U = (double *)malloc(sizeof(double) * (size_t)cells * Q * m);
  if (!node_states(c, lam, U)) {
    if (worst < ORC_INADMISSIBLE) worst = ORC_INADMISSIBLE;
  }
  double dt = dt_from_states(c, U, t_remaining);
  double *unew = (double *)malloc(sizeof(double) * (size_t)cells * N * m);
  flux_update_states(c, U, newlev, uhat, unew, dt);
  /* steady residual on the zeroth moment of the first state (reading 23) */
  double res = 0.0;
  for (int j = 0; j < cells; ++j) res += c->area[j] * fabs(unew[(size_t)j * N * m] - uhat[(size_t)j * N * m]);
  memcpy(uhat, unew, sizeof(double) * (size_t)cells * N * m);
  /* Alg. 4 lines 12-14: next stage once the residual lies below the stage's tolerance */
  if (c->P.n_retard > 0 && c->retard_stage < c->P.n_retard && res < c->P.retard_eps[c->retard_stage])
    c->retard_stage += 1;
  /* lambda zero-padded (refine) or truncated (coarsen) to the new level */
  if (c->n_levels > 0) {
    for (int j = 0; j < cells; ++j) {
      int Nn = c->Nl[newlev[j]];
      for (int r = Nn * m; r < N * m; ++r) lam[(size_t)j * N * m + r] = 0.0;
    }
    memcpy(c->level, newlev, sizeof(int32_t) * cells);
  }
  if (dt_used) *dt_used = dt;
  if (residual) *residual = res;
  free(U); free(unew); free(st); free(newlev);
  return worst;
}


/* ---- Stochastic Collocation (reading 32) -------------
 * The deterministic finite-volume solver with the same numerical flux g runs at every quadrature
 * point; the points advance together with one CFL step (the paper's coupled collocation code,
 * PAPER.md:463), and the moments come from the quadrature rule uhat_i = sum_k w_k u(xi_k) phi_i(xi_k). */
void orc_sc_init(const orc_ctx *c, const orc_ic *ic, double *U) {
  int Q = c->Q, m = c->m;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < c->cells; ++j)
    for (int k = 0; k < Q; ++k) {
      double ub[4];
      ic_node_state(c, ic, j, k, ub);
      for (int a = 0; a < m; ++a) U[((size_t)j * Q + k) * m + a] = ub[a];
    }
}

/* one step: dt = CFL / max rate over all node (and ghost) states, u_k^{n+1} = u_k^n - dt r_k(u^n);
 * residual = sum_j |Omega_j| |sum_k w_k (u_k^{n+1} - u_k^n)_0| (PAPER.md:238-241 on the mean) */
double orc_sc_step(const orc_ctx *c, const double *U, double *Unew, double t_remaining, double *residual) {
  const orc_problem *P = &c->P;
  int Q = c->Q, m = c->m;
  double dt = dt_from_states(c, U, t_remaining);
  double dx_over_dt = (P->mesh_kind == ORC_MESH_1D) ? ((P->x1 - P->x0) / P->nx) / dt : 0.0;
  double res = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : res)
  for (int j = 0; j < c->cells; ++j) {
    double dmean = 0.0;
    for (int k = 0; k < Q; ++k) {
      double r[4];
      node_residual(c, U, j, k, dx_over_dt, r);
      const double *uj = U + ((size_t)j * Q + k) * m;
      double *un = Unew + ((size_t)j * Q + k) * m;
      for (int a = 0; a < m; ++a) un[a] = uj[a] - dt * r[a];
      dmean += c->omega[k] * (un[0] - uj[0]);
    }
    res += c->area[j] * fabs(dmean);
  }
  if (residual) *residual = res;
  return dt;
}

void orc_sc_moments(const orc_ctx *c, const double *U, double *uhat) {
  int N = c->N, Q = c->Q, m = c->m;
  for (int j = 0; j < c->cells; ++j) {
    double *uj = uhat + (size_t)j * N * m;
    for (int r = 0; r < N * m; ++r) uj[r] = 0.0;
    for (int k = 0; k < Q; ++k)
      for (int i = 0; i < N; ++i)
        for (int a = 0; a < m; ++a) uj[i * m + a] += c->omega[k] * U[((size_t)j * Q + k) * m + a] * c->Phi[k * N + i];
  }
}
