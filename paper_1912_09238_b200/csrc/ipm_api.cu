// ipm_api.cu — libipm host side: context setup (basis, quadrature, mesh tables), device memory,
// and the C-ABI declared in include/ipm.h.
//
// Host setup follows the paper's definitions:
//   total-degree basis, N = binom(M+p, p), graded multi-indices
//   orthonormal Legendre phi_i(xi) = prod_n sqrt(2 i_n + 1) P_{i_n}(xi_n) for U(-1,1)^p
//   <h>_Q = sum_k w_k h(xi_k) f_Xi(xi_k) with a tensor Gauss-Legendre rule
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ipm.h"
#include "ipm_host.h"
#include "ipm_internal.h"

namespace {

thread_local std::string g_err;

ipm_status fail(ipm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_OK(expr)                                                                               \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess) return fail(IPM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------------------------
// random space
// ---------------------------------------------------------------------------------------------

// Gauss-Legendre rule on [-1,1] (weights sum to 2): Newton iteration on P_q from the asymptotic
// guess cos(pi (k - 1/4)/(q + 1/2)), P_q and P_q' from the three-term recurrence.
void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w) {
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  for (int k = 1; k <= (q + 1) / 2; ++k) {
    double z = std::cos(M_PI * (k - 0.25) / (q + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 64; ++it) {
      double p0 = 1.0, p1 = z;
      for (int n = 2; n <= q; ++n) {
        const double p2 = ((2.0 * n - 1.0) * z * p1 - (n - 1.0) * p0) / n;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) {
        p1 = z;
        p0 = 1.0;
      }
      dp = q * (z * p1 - p0) / (z * z - 1.0);
      const double step = p1 / dp;
      z -= step;
      if (std::fabs(step) <= 1e-16 * std::max(1.0, std::fabs(z))) break;
    }
    {
      double p0 = 1.0, p1 = z;
      for (int n = 2; n <= q; ++n) {
        const double p2 = ((2.0 * n - 1.0) * z * p1 - (n - 1.0) * p0) / n;
        p0 = p1;
        p1 = p2;
      }
      dp = q * (z * p1 - p0) / (z * z - 1.0);
    }
    const double wk = 2.0 / ((1.0 - z * z) * dp * dp);
    x[k - 1] = -z;
    x[q - k] = z;
    w[k - 1] = wk;
    w[q - k] = wk;
  }
  if (q % 2 == 1) x[q / 2] = 0.0;
}

// Clenshaw-Curtis rule with n points (reading 33): nodes -cos(pi j/(n-1)); weights
// from the exactness conditions sum_j w_j P_k(x_j) = 2 delta_k0, k < n (Legendre moment fitting,
// Gaussian elimination with partial pivoting); n = 1: the midpoint, weight 2.
void clenshaw_curtis(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  if (n == 1) {
    w[0] = 2.0;
    return;
  }
  for (int j = 0; j < n; ++j) x[j] = -std::cos(M_PI * j / (n - 1));
  if (n % 2 == 1) x[(n - 1) / 2] = 0.0;
  std::vector<long double> A((size_t)n * (n + 1));
  for (int j = 0; j < n; ++j) {  // row k: P_k(x_j), Legendre (not normalised) by recurrence
    long double p0 = 1.0L, p1 = x[j];
    A[(size_t)0 * (n + 1) + j] = p0;
    if (n > 1) A[(size_t)1 * (n + 1) + j] = p1;
    for (int k = 2; k < n; ++k) {
      const long double p2 = ((2.0L * k - 1.0L) * x[j] * p1 - (k - 1.0L) * p0) / k;
      A[(size_t)k * (n + 1) + j] = p2;
      p0 = p1;
      p1 = p2;
    }
  }
  for (int k = 0; k < n; ++k) A[(size_t)k * (n + 1) + n] = (k == 0) ? 2.0L : 0.0L;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs((double)A[(size_t)r * (n + 1) + c]) > std::fabs((double)A[(size_t)piv * (n + 1) + c])) piv = r;
    for (int cc = 0; cc <= n; ++cc) std::swap(A[(size_t)c * (n + 1) + cc], A[(size_t)piv * (n + 1) + cc]);
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const long double f = A[(size_t)r * (n + 1) + c] / A[(size_t)c * (n + 1) + c];
      for (int cc = c; cc <= n; ++cc) A[(size_t)r * (n + 1) + cc] -= f * A[(size_t)c * (n + 1) + cc];
    }
  }
  for (int j = 0; j < n; ++j) w[j] = (double)(A[(size_t)j * (n + 1) + n] / A[(size_t)j * (n + 1) + j]);
}

// Smolyak sparse grid of nested Clenshaw-Curtis rules (reading 33): the combination formula
// sum over multi-levels i (i_d >= 1, L-p+1 <= |i| <= L) of (-1)^{L-|i|} C(p-1, L-|i|) times the tensor
// rule of levels i (level 1: midpoint; level l > 1: 2^{l-1}+1 points); coincident points merged by
// their index on the finest 1D grid, listed in lexicographic order of those indices.
void smolyak_cc(int p, int L, std::vector<double>& xi, std::vector<double>& w) {
  const int Fl = L - p + 1, nf = Fl >= 2 ? (1 << (Fl - 1)) + 1 : 1;
  std::vector<double> xf, wf;
  clenshaw_curtis(nf, xf, wf);
  std::map<std::vector<int>, double> acc;
  std::vector<int> lev(p, 1);
  std::function<void(int, int)> rec = [&](int d, int used) {
    if (d == p) {
      if (used < L - p + 1 || used > L) return;
      double coef = ((L - used) % 2) ? -1.0 : 1.0;
      {
        long long b = 1;  // C(p-1, L-used)
        const int kk = L - used;
        for (int t = 1; t <= kk; ++t) b = b * (p - 1 - kk + t) / t;
        coef *= (double)b;
      }
      std::vector<std::vector<double>> ws(p);
      std::vector<int> ns(p), stride(p);
      for (int e = 0; e < p; ++e) {
        ns[e] = lev[e] == 1 ? 1 : (1 << (lev[e] - 1)) + 1;
        std::vector<double> xx;
        clenshaw_curtis(ns[e], xx, ws[e]);
        stride[e] = ns[e] == 1 ? 0 : (nf - 1) / (ns[e] - 1);
      }
      std::vector<int> j(p, 0), key(p);
      for (;;) {
        double wt = coef;
        for (int e = 0; e < p; ++e) {
          key[e] = ns[e] == 1 ? (nf - 1) / 2 : j[e] * stride[e];
          wt *= ws[e][j[e]];
        }
        acc[key] += wt;
        int e = p - 1;
        while (e >= 0 && ++j[e] == ns[e]) j[e--] = 0;
        if (e < 0) break;
      }
      return;
    }
    for (int l = 1; used + l <= L; ++l) {
      lev[d] = l;
      rec(d + 1, used + l);
    }
  };
  rec(0, 0);
  xi.clear();
  w.clear();
  for (const auto& kv : acc) {
    for (int e = 0; e < p; ++e) xi.push_back(xf[kv.first[e]]);
    w.push_back(kv.second);
  }
}

double legendre_orthonormal(int n, double x) {
  double p0 = 1.0, p1 = x;
  if (n == 0) return 1.0;
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  return std::sqrt(2.0 * n + 1.0) * p1;
}

int binom_total(int p, int M) {
  long long r = 1;
  for (int k = 1; k <= p; ++k) r = r * (M + k) / k;
  return (int)r;
}

// graded, then lexicographically descending within one total degree (prefix property per level)
void total_degree_set(int p, int M, std::vector<int>& idx) {
  idx.clear();
  std::vector<int> cur(p, 0);
  for (int deg = 0; deg <= M; ++deg) {
    // odometer over tuples summing to deg, first entry descending
    std::vector<int> t(p, 0);
    t[0] = deg;
    for (;;) {
      idx.insert(idx.end(), t.begin(), t.end());
      // predecessor in lexicographic order among tuples with sum deg
      int j = p - 2;
      while (j >= 0 && t[j] == 0) --j;
      if (j < 0) break;
      t[j] -= 1;
      int rest = 0;
      for (int r = j + 1; r < p; ++r) rest += t[r];
      rest += 1;
      for (int r = j + 1; r < p; ++r) t[r] = 0;
      t[j + 1] = rest;
    }
  }
}

struct HostPrim {
  // primitive state at node xi for an ipm_state
  static void eval(const ipm_state& s, const double* xi, int p, int m, double gamma, double* u) {
    double q[5] = {0, 0, 0, 0, 0};
    if (s.kind == 1) {
      const double rho = s.q0[0], pr = s.q0[1];
      const double mach = s.q0[2] + s.q0[3] * xi[s.dim_a];
      const double th = (s.q0[4] + s.q0[5] * xi[s.dim_b]) * M_PI / 180.0;
      const double c = std::sqrt(gamma * pr / rho);
      q[0] = rho;
      q[1] = mach * c * std::cos(th);
      q[2] = mach * c * std::sin(th);
      q[3] = pr;
    } else {
      const int nq = m;
      for (int c = 0; c < nq; ++c) {
        q[c] = s.q0[c];
        for (int d = 0; d < p && d < 3; ++d) q[c] += s.q1[c][d] * xi[d];
      }
    }
    if (m == 1) {
      u[0] = q[0];
      return;
    }
    const int d = m - 2;
    double v2 = 0.0;
    u[0] = q[0];
    for (int k = 0; k < d; ++k) {
      u[1 + k] = q[0] * q[1 + k];
      v2 += q[1 + k] * q[1 + k];
    }
    u[m - 1] = q[d + 1] / (gamma - 1.0) + 0.5 * q[0] * v2;
  }
};

double host_speed(int m, double gamma, const double* u, int mode /*0 dir x, 1 dir y, 2 norm*/) {
  if (m == 1) return std::fabs(u[0]);
  const int d = m - 2;
  double m2 = 0.0;
  for (int k = 0; k < d; ++k) m2 += u[1 + k] * u[1 + k];
  const double p = (gamma - 1.0) * (u[m - 1] - 0.5 * m2 / u[0]);
  const double c = std::sqrt(gamma * p / u[0]);
  if (mode == 2) return std::sqrt(m2) / u[0] + c;
  return std::fabs(u[1 + mode] / u[0]) + c;
}

template <typename T>
T* dalloc(size_t n, std::vector<void*>& owned) {
  if (n == 0) n = 1;
  void* p = nullptr;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
  owned.push_back(p);
  return (T*)p;
}

}  // namespace

struct ipm_ctx {
  ipm_config cfg;
  int N = 0, Q = 0, QP = 0, m = 0, p = 0, F = 0;
  int64_t cells = 0, halo = 0;
  ipm::Partition part;
  int64_t* d_gid = nullptr;       // [cells] global ids of owned cells
  int32_t* d_send_local = nullptr;  // [nsend] local indices packed for the peers
  std::vector<int> idx, deg;
  std::vector<double> xi, omega, phi;  // phi [Q][N]
  std::vector<int64_t> cell_ids;
  double ghost_rate = 0.0;
  int nl_levels[8] = {0};
  std::vector<void*> owned;
  cudaStream_t stream = nullptr;
  ipm::KernelCtx k{};
  // device buffers
  double *d_uq = nullptr, *d_crit = nullptr;
  int32_t *d_level = nullptr, *d_level_new = nullptr, *d_iters = nullptr, *d_status = nullptr;
  int32_t *d_halv = nullptr, *d_inadm = nullptr;  // per-cell line-search record of the last dual solve
  ipm::StepScalars* d_sc = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  const double* sc_last_out = nullptr;  // ipm_sc_step: output whose CFL rate is cached on the device
  cudaStream_t copy_stream = nullptr;  // ipm_step_host
  std::vector<cudaEvent_t> hev;        // ipm_step_host: per-chunk copy / solve events
  bool timing = false;
  int initial_level = 0;
  // CUDA graph of one ipm_step (small single-rank problems without levels, ipm.h)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  const double *g_uhat = nullptr, *g_lambda = nullptr;
  double g_tend = 0.0;
  bool graph_off = false;
  // banded node states (meshes whose [cells + halo][m][Q] buffer would not fit: config 5 at 4096^2
  // is 537 GB): d_uq holds band_rows + 2 rows of a row-major cartesian block, d_uq_halo the halo cells;
  // the dual kernel then writes no node states, the flux recomputes each band's from lambda
  int64_t band_rows = 0;
  double* d_uq_halo = nullptr;
  // L-BFGS history (hessian_kind 1, reading 35): pairs newest first, 1/(s^T y), counts, basis sizes
  double *d_lbS = nullptr, *d_lbY = nullptr, *d_lbR = nullptr;
  int32_t *d_lbC = nullptr, *d_lbN = nullptr;
  // per-level nested rules (reading 36): each level's tables on its own nodes (no sum factorisation
  // tables; the bucketed launches add them)
  ipm::Tables lq_tables[8] = {};
  // distributed contexts: the owned cells adjacent to a peer (boundary) and the others (interior), local
  // indices ascending, for ipm_step_dual_boundary / ipm_step_dual_interior
  int32_t *d_bnd = nullptr, *d_int = nullptr;
  int64_t n_bnd = 0, n_int = 0;
  // triangle meshes: the flux kernel's processing order (Morton order of the owned cells' centroids)
  int32_t* d_order = nullptr;
};

// the L-BFGS history of cells [r0, ...) for a dual launch (nothing for Newton contexts)
static void lb_attach(const ipm_ctx* c, ipm::DualLaunch& a, int64_t r0) {
  if (c->k.hessian_kind != 1) return;
  const int64_t row = (int64_t)c->N * c->m, mh = c->k.lbfgs_m;
  a.lb_S = c->d_lbS + r0 * mh * row;
  a.lb_Y = c->d_lbY + r0 * mh * row;
  a.lb_rho = c->d_lbR + r0 * mh;
  a.lb_cnt = c->d_lbC + r0;
  a.lb_n = c->d_lbN + r0;
}

extern "C" {

const char* ipm_status_string(ipm_status s) {
  switch (s) {
    case IPM_OK: return "ok";
    case IPM_ERR_ARG: return "invalid argument";
    case IPM_ERR_CUDA: return "CUDA error";
    case IPM_ERR_NCCL: return "NCCL error";
    case IPM_ERR_UNSUPPORTED: return "unsupported configuration";
    case IPM_ERR_NUMERIC: return "failed cells";
  }
  return "unknown";
}

const char* ipm_last_error(void) { return g_err.c_str(); }

void ipm_destroy(ipm_ctx* c) {
  if (!c) return;
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->hev) cudaEventDestroy(e);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (void* p : c->owned) cudaFree(p);
  delete c;
}

ipm_status ipm_init(const ipm_config* cfg, ipm_ctx** out) {
  if (!cfg || !out) return fail(IPM_ERR_ARG, "null argument");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(IPM_ERR_CUDA, "no CUDA device (libipm has no CPU path)");
  const ipm_config& C = *cfg;
  if (C.p < 1 || C.p > 3 || C.M < 0) return fail(IPM_ERR_ARG, "bad random space");
  if (C.quad_kind < 0 || C.quad_kind > 2) return fail(IPM_ERR_ARG, "quad_kind must be 0 (GL), 1 (CC), 2 (Smolyak)");
  if (C.quad_kind != 2 && (C.q1d < 1 || C.q1d > (C.quad_kind == 1 ? 33 : 64))) return fail(IPM_ERR_ARG, "bad q1d");
  if (C.quad_kind == 2 && (C.quad_level < C.p || C.quad_level - C.p + 1 > 6))
    return fail(IPM_ERR_ARG, "Smolyak level must satisfy p <= L <= p + 5");
  if (C.quad_kind != 0 && binom_total(C.p, C.M) * C.m > 88)
    return fail(IPM_ERR_ARG, "non-tensor-GL rules: n = N m <= 88 (the large-cell kernel is sum-factorised)");
  if (!(C.m == 1 || C.m == 3 || C.m == 4)) return fail(IPM_ERR_ARG, "m must be 1, 3 or 4");
  if (C.closure == IPM_CLOSURE_BARRIER && (C.m != 1 || !(C.u_plus > C.u_minus)))
    return fail(IPM_ERR_ARG, "barrier closure needs m = 1 and u+ > u-");
  if (C.closure == IPM_CLOSURE_EULER && C.m == 1) return fail(IPM_ERR_ARG, "Euler closure needs m = 3 or 4");
  if (C.nranks > 1 && (C.rank < 0 || C.rank >= C.nranks)) return fail(IPM_ERR_ARG, "rank out of range");
  if (C.n_levels < 0 || C.n_levels > 8) return fail(IPM_ERR_ARG, "n_levels in [0, 8]");
  if (C.n_levels > 0 && C.level_M[C.n_levels - 1] != C.M) return fail(IPM_ERR_ARG, "level_M[last] must equal M");
  if (C.n_retard < 0 || C.n_retard > 8) return fail(IPM_ERR_ARG, "n_retard must be in [0, 8]");
  for (int t = 0; t < 4; ++t) {
    if (C.bc_kind[t] < IPM_BC_TRANSMISSIVE || C.bc_kind[t] > IPM_BC_FARFIELD) return fail(IPM_ERR_ARG, "bad bc_kind");
    if (C.bc_kind[t] == IPM_BC_FARFIELD && (C.mesh_kind != IPM_MESH_TRI || C.m != 4 || C.closure != IPM_CLOSURE_EULER))
      return fail(IPM_ERR_ARG, "far-field boundaries: triangle meshes, 2D Euler only (reading 37)");
  }
  // per-level nested rules (reading 36): a nested ladder of tensor Clenshaw-Curtis rules, the finest
  // being the context's rule
  const bool level_rules = C.n_levels > 0 && C.level_q1d[0] > 0;
  if (level_rules) {
    const int nf = C.level_q1d[C.n_levels - 1];
    if (C.quad_kind != 1 || C.q1d != nf) return fail(IPM_ERR_ARG, "per-level rules: quad_kind 1 (CC) with q1d = level_q1d[last]");
    for (int l = 0; l < C.n_levels; ++l) {
      const int nl = C.level_q1d[l];
      if (nl < 2 || nl > nf || (nf - 1) % (nl - 1) != 0 || (l > 0 && nl < C.level_q1d[l - 1]))
        return fail(IPM_ERR_ARG, "per-level rules must nest: level_q1d ascending, (q1d_f - 1) % (q1d_l - 1) == 0");
    }
  }
  for (int l = 0; l < C.n_retard && C.n_levels > 0; ++l)
    if (C.retard_level[l] < 0 || C.retard_level[l] >= C.n_levels) return fail(IPM_ERR_ARG, "retard_level out of range");

  ipm_ctx* c = new ipm_ctx();
  c->cfg = C;
  c->stream = (cudaStream_t)C.stream;
  c->p = C.p;
  c->m = C.m;
  c->N = binom_total(C.p, C.M);
  // quadrature (reading 33): tensor Gauss-Legendre (default), tensor Clenshaw-Curtis, or Smolyak
  std::vector<double> sg_xi, sg_w;
  if (C.quad_kind == 2) {
    smolyak_cc(C.p, C.quad_level, sg_xi, sg_w);
    c->Q = (int)sg_w.size();
  } else {
    c->Q = 1;
    for (int d = 0; d < C.p; ++d) c->Q *= C.q1d;
  }
  c->QP = (c->Q % 2 == 0) ? c->Q + 1 : c->Q;
  const int N = c->N, Q = c->Q, QP = c->QP, p = c->p, m = c->m;

  // basis and quadrature
  total_degree_set(p, C.M, c->idx);
  c->deg.resize(N);
  for (int i = 0; i < N; ++i) {
    int s = 0;
    for (int d = 0; d < p; ++d) s += c->idx[i * p + d];
    c->deg[i] = s;
  }
  std::vector<double> x1, w1;
  if (C.quad_kind == 1)
    clenshaw_curtis(C.q1d, x1, w1);
  else if (C.quad_kind == 0)
    gauss_legendre(C.q1d, x1, w1);
  c->xi.resize((size_t)Q * p);
  c->omega.resize(Q);
  c->phi.resize((size_t)Q * N);
  for (int k = 0; k < Q; ++k) {
    double om = 1.0;
    if (C.quad_kind == 2) {
      for (int d = 0; d < p; ++d) {
        c->xi[(size_t)k * p + d] = sg_xi[(size_t)k * p + d];
        om *= 0.5;  // f_Xi = 2^{-p}
      }
      om *= sg_w[k];
    } else {
      int r = k;
      for (int d = p - 1; d >= 0; --d) {
        const int kd = r % C.q1d;
        r /= C.q1d;
        c->xi[(size_t)k * p + d] = x1[kd];
        om *= 0.5 * w1[kd];  // f_Xi = 2^{-p}
      }
    }
    c->omega[k] = om;
    for (int i = 0; i < N; ++i) {
      double v = 1.0;
      for (int d = 0; d < p; ++d) v *= legendre_orthonormal(c->idx[i * p + d], c->xi[(size_t)k * p + d]);
      c->phi[(size_t)k * N + i] = v;
    }
  }
  // 1D pair table for the sum-factorised Hessian: LL[k][pr] = (w_k/2) L_a(x_k) L_b(x_k), a <= b <= M
  // (tensor Gauss-Legendre only: other rules use the direct Hessian sum, q1d = npr = 0 on the device)
  const bool tensor_gl = C.quad_kind == 0;
  const int npr = tensor_gl ? (C.M + 1) * (C.M + 2) / 2 : 0;
  std::vector<double> LL((size_t)std::max(1, (tensor_gl ? C.q1d : 0) * npr), 0.0);
  for (int k = 0; tensor_gl && k < C.q1d; ++k) {
    int pr = 0;
    for (int aa = 0; aa <= C.M; ++aa)
      for (int bb = aa; bb <= C.M; ++bb, ++pr)
        LL[(size_t)k * npr + pr] =
            0.5 * w1[k] * legendre_orthonormal(aa, x1[k]) * legendre_orthonormal(bb, x1[k]);
  }
  std::vector<int32_t> idx32(c->idx.begin(), c->idx.end());
  std::vector<double> PhiT((size_t)N * QP, 0.0), WPhiT((size_t)N * QP, 0.0);
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < Q; ++k) {
      PhiT[(size_t)i * QP + k] = c->phi[(size_t)k * N + i];
      WPhiT[(size_t)i * QP + k] = c->omega[k] * c->phi[(size_t)k * N + i];
    }
  // the same table in DMMA A-fragment order (projection of the flux kernel)
  const int MT = (N + 7) / 8, KS = (Q + 3) / 4;
  std::vector<double> WPhiF((size_t)MT * KS * 32, 0.0);
  for (int mt = 0; mt < MT; ++mt)
    for (int ks = 0; ks < KS; ++ks)
      for (int l = 0; l < 32; ++l) {
        const int i = 8 * mt + l / 4, k = 4 * ks + l % 4;
        if (i < N && k < Q) WPhiF[((size_t)mt * KS + ks) * 32 + l] = WPhiT[(size_t)i * QP + k];
      }

  // mesh face tables (global), this rank's part and its halo
  ipm::MeshTables G, Lm;
  std::string merr;
  if (!ipm::build_mesh(C, G, merr)) {
    delete c;
    return fail(IPM_ERR_ARG, merr);
  }
  const int nranks = C.nranks > 0 ? C.nranks : 1;
  if (!ipm::build_partition(C, G, nranks > 1 ? C.rank : 0, nranks, c->part, merr)) {
    delete c;
    return fail(IPM_ERR_ARG, merr);
  }
  ipm::local_tables(G, c->part, Lm);
  const int F = G.F;
  const int64_t cells = Lm.cells;
  const double inv_dx = G.inv_dx, inv_dy = G.inv_dy;
  std::vector<int32_t>& nbr = Lm.nbr;
  std::vector<double>&nrm = Lm.nrm, &coef = Lm.coef, &area = Lm.area, &rgeo = Lm.rgeo;
  c->F = F;
  c->cells = cells;
  c->halo = (int64_t)c->part.halo_gid.size();
  c->cell_ids = c->part.local_gid;

  // boundary ghost states per node and their CFL contribution
  std::vector<double> ghost((size_t)4 * Q * m, 0.0);
  for (int t = 0; t < 4; ++t)
    if (C.bc_kind[t] == IPM_BC_STATE || C.bc_kind[t] == IPM_BC_FARFIELD)  // FARFIELD: the free stream
      for (int k = 0; k < Q; ++k)
        HostPrim::eval(C.bc_state[t], &c->xi[(size_t)k * p], p, m, C.gamma, &ghost[((size_t)t * Q + k) * m]);
  double grate = 0.0;
  for (int64_t j = 0; j < G.cells; ++j)
    for (int f = 0; f < F; ++f) {
      const int nb = G.nbr[j * F + f];
      if (nb >= 0) continue;
      const int tag = -1 - nb;
      if (C.bc_kind[tag] != IPM_BC_STATE && C.bc_kind[tag] != IPM_BC_FARFIELD) continue;  // reading 37
      for (int k = 0; k < Q; ++k) {
        const double* ug = &ghost[((size_t)tag * Q + k) * m];
        double r;
        if (C.mesh_kind == IPM_MESH_1D)
          r = host_speed(m, C.gamma, ug, 0) * inv_dx;
        else if (C.mesh_kind == IPM_MESH_CART2D)
          r = host_speed(m, C.gamma, ug, 0) * inv_dx + host_speed(m, C.gamma, ug, 1) * inv_dy;
        else
          r = host_speed(m, C.gamma, ug, 2) * G.rgeo[j];
        grate = std::max(grate, r);
      }
    }
  c->ghost_rate = grate;

  // device memory
  auto& O = c->owned;
  double* d_PhiT = dalloc<double>(PhiT.size(), O);
  double* d_WPhiT = dalloc<double>(WPhiT.size(), O);
  double* d_WPhiF = dalloc<double>(WPhiF.size(), O);
  double* d_omega = dalloc<double>(Q, O);
  int32_t* d_deg = dalloc<int32_t>(N, O);
  double* d_LL = dalloc<double>(LL.size(), O);
  int32_t* d_idx = dalloc<int32_t>(idx32.size(), O);
  int32_t* d_nbr = dalloc<int32_t>(nbr.size(), O);
  double* d_nrm = dalloc<double>(nrm.size(), O);
  double* d_coef = dalloc<double>(coef.size(), O);
  double* d_area = dalloc<double>(area.size(), O);
  double* d_rgeo = dalloc<double>(rgeo.size(), O);
  double* d_ghost = dalloc<double>(ghost.size(), O);
  c->d_gid = dalloc<int64_t>(cells, O);
  c->d_send_local = dalloc<int32_t>(c->part.send_local.size(), O);
  c->d_crit = dalloc<double>(cells, O);
  c->d_level = dalloc<int32_t>(cells, O);
  c->d_level_new = dalloc<int32_t>(cells, O);
  c->d_iters = dalloc<int32_t>(cells, O);
  c->d_status = dalloc<int32_t>(cells, O);
  c->d_halv = dalloc<int32_t>(cells, O);
  c->d_inadm = dalloc<int32_t>(cells, O);
  c->d_sc = dalloc<ipm::StepScalars>(1, O);
  if (!d_PhiT || !d_WPhiT || !d_WPhiF || !d_omega || !d_deg || !d_LL || !d_idx || !d_nbr || !d_nrm || !d_coef || !d_area || !d_rgeo || !d_ghost ||
      !c->d_gid || !c->d_send_local || !c->d_crit || !c->d_level || !c->d_level_new || !c->d_iters || !c->d_status || !c->d_halv || !c->d_inadm || !c->d_sc) {
    ipm_destroy(c);
    return fail(IPM_ERR_CUDA, "cudaMalloc failed");
  }
  std::vector<int32_t> deg32(c->deg.begin(), c->deg.end());
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return bytes == 0 ? cudaSuccess : cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  };
  if (up(d_PhiT, PhiT.data(), PhiT.size() * 8) || up(d_WPhiT, WPhiT.data(), WPhiT.size() * 8) ||
      up(d_WPhiF, WPhiF.data(), WPhiF.size() * 8) ||
      up(d_omega, c->omega.data(), Q * 8) || up(d_deg, deg32.data(), N * 4) ||
      up(d_LL, LL.data(), LL.size() * 8) || up(d_idx, idx32.data(), idx32.size() * 4) ||
      up(d_nbr, nbr.data(), nbr.size() * 4) || up(d_nrm, nrm.data(), nrm.size() * 8) ||
      up(d_coef, coef.data(), coef.size() * 8) || up(d_area, area.data(), area.size() * 8) ||
      up(d_rgeo, rgeo.data(), rgeo.size() * 8) || up(d_ghost, ghost.data(), ghost.size() * 8) ||
      up(c->d_gid, c->part.local_gid.data(), cells * 8) ||
      up(c->d_send_local, c->part.send_local.data(), c->part.send_local.size() * 4) ||
      cudaMemset(c->d_sc, 0, sizeof(ipm::StepScalars)) || cudaMemset(c->d_level, 0, cells * 4) ||
      cudaMemset(c->d_level_new, 0, cells * 4) ||
      cudaMemset(c->d_iters, 0, cells * 4) || cudaMemset(c->d_status, 0, cells * 4) ||
      cudaMemset(c->d_halv, 0, cells * 4) || cudaMemset(c->d_inadm, 0, cells * 4)) {
    ipm_destroy(c);
    return fail(IPM_ERR_CUDA, "upload failed");
  }
  for (auto& e : c->ev) cudaEventCreate(&e);

  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);

  ipm::KernelCtx& k = c->k;
  k.T = ipm::Tables{d_PhiT, d_WPhiT, d_omega, d_deg, N, Q, QP, p, d_LL, d_idx, tensor_gl ? C.q1d : 0, npr, d_WPhiF, MT, KS,
                    nullptr, nullptr, 0};
  // 1D tables of the tensor Gauss-Legendre rule (the large-cell quasi-Newton kernel's sum factorisation)
  if (tensor_gl) {
    std::vector<double> L1h((size_t)(C.M + 1) * C.q1d), w1hh(C.q1d);
    for (int i = 0; i <= C.M; ++i)
      for (int kq = 0; kq < C.q1d; ++kq) L1h[(size_t)i * C.q1d + kq] = legendre_orthonormal(i, x1[kq]);
    for (int kq = 0; kq < C.q1d; ++kq) w1hh[kq] = 0.5 * w1[kq];
    double *d_L1 = dalloc<double>(L1h.size(), O), *d_w1h = dalloc<double>(w1hh.size(), O);
    if (!d_L1 || !d_w1h || up(d_L1, L1h.data(), L1h.size() * 8) || up(d_w1h, w1hh.data(), w1hh.size() * 8)) {
      ipm_destroy(c);
      return fail(IPM_ERR_CUDA, "1D table upload failed");
    }
    k.T.L1 = d_L1;
    k.T.w1h = d_w1h;
    k.T.npr1 = C.M + 1;
  }
  k.mesh.kind = C.mesh_kind;
  k.mesh.F = F;
  k.mesh.cells = cells;
  k.mesh.nbr = d_nbr;
  k.mesh.nrm = d_nrm;
  k.mesh.coef = d_coef;
  k.mesh.area = d_area;
  k.mesh.rate_geo = d_rgeo;
  k.mesh.inv_dx = inv_dx;
  k.mesh.inv_dy = inv_dy;
  k.mesh.ghost = d_ghost;
  for (int t = 0; t < 4; ++t) k.mesh.bc_kind[t] = C.bc_kind[t];
  k.mesh.bx = k.mesh.by = 0;
  if (C.mesh_kind == IPM_MESH_CART2D && cells > 0) {
    // row-major block structure of the (local) cells, as the strip flux kernel walks it: row 0 is
    // cells 0..bx-1 (east links), every owned neighbour is the index arithmetic says
    int64_t bx = 1;
    while (bx < cells && nbr[(bx - 1) * 4 + 1] == (int32_t)bx) ++bx;
    bool ok = cells % bx == 0;
    for (int64_t j = 0; ok && j < cells; ++j) {
      const int64_t x = j % bx, y = j / bx, by = cells / bx;
      ok = (x == 0 || nbr[j * 4 + 0] == (int32_t)(j - 1)) && (x == bx - 1 || nbr[j * 4 + 1] == (int32_t)(j + 1)) &&
           (y == 0 || nbr[j * 4 + 2] == (int32_t)(j - bx)) && (y == by - 1 || nbr[j * 4 + 3] == (int32_t)(j + bx));
    }
    if (ok && cells < ((int64_t)1 << 31)) {
      k.mesh.bx = (int)bx;
      k.mesh.by = (int)(cells / bx);
    }
  }
  // node-state buffer: whole mesh, or bands of rows (IPM_BAND_ROWS forces bands of that many rows, e.g.
  // for parity tests; otherwise bands when the whole buffer would exceed IPM_NODE_BUDGET_GB, default 24)
  {
    const size_t per_cell = (size_t)Q * m * 8;
    const double budget = (std::getenv("IPM_NODE_BUDGET_GB") ? std::atof(std::getenv("IPM_NODE_BUDGET_GB")) : 24.0) * 1e9;
    const int64_t forced = std::getenv("IPM_BAND_ROWS") ? std::atoll(std::getenv("IPM_BAND_ROWS")) : 0;
    const bool can_band = k.mesh.bx > 0 && C.n_levels == 0;
    if (can_band && (forced > 0 || (double)(cells + c->halo) * per_cell > budget)) {
      const int64_t rows = forced > 0 ? forced : std::max<int64_t>(1, (int64_t)(budget / ((double)k.mesh.bx * per_cell)) - 2);
      c->band_rows = std::min<int64_t>(rows, k.mesh.by);
      c->d_uq = dalloc<double>((size_t)(c->band_rows + 2) * k.mesh.bx * Q * m, O);
      c->d_uq_halo = dalloc<double>((size_t)std::max<int64_t>(c->halo, 1) * Q * m, O);
      if (!c->d_uq || !c->d_uq_halo || cudaMemset(c->d_uq, 0, (size_t)(c->band_rows + 2) * k.mesh.bx * per_cell) ||
          cudaMemset(c->d_uq_halo, 0, (size_t)std::max<int64_t>(c->halo, 1) * per_cell)) {
        ipm_destroy(c);
        return fail(IPM_ERR_CUDA, "cudaMalloc (node-state bands) failed");
      }
    } else {
      c->d_uq = dalloc<double>((size_t)(cells + c->halo) * Q * m, O);
      // defined before the first dual solve writes them (halo rows: before the first exchange)
      if (!c->d_uq || cudaMemset(c->d_uq, 0, (size_t)(cells + c->halo) * per_cell)) {
        ipm_destroy(c);
        return fail(IPM_ERR_CUDA, "cudaMalloc (node states) failed");
      }
    }
  }
  k.nw = ipm::Newton{C.tau, C.armijo_c, C.max_newton, C.max_halvings, C.newton_mode};
  k.ad.n_levels = C.n_levels;
  for (int l = 0; l < C.n_levels; ++l) k.ad.Nl[l] = binom_total(p, C.level_M[l]);
  k.ad.Nprev0 = C.n_levels > 0 ? (C.level_M[0] > 0 ? binom_total(p, C.level_M[0] - 1) : 0) : 0;
  k.ad.delta_dec = C.delta_dec;
  k.ad.n_retard = C.n_levels > 0 ? C.n_retard : 0;
  for (int l = 0; l < 8; ++l) {
    k.ad.retard_level[l] = l < k.ad.n_retard ? C.retard_level[l] : 0;
    k.ad.retard_eps[l] = l < k.ad.n_retard ? C.retard_eps[l] : 0.0;
  }
  k.ad.delta_inc = C.delta_inc;
  k.cl = ipm::ClParams{C.gamma, C.u_minus, C.u_plus, C.gamma > 1.0 ? 1.0 / (C.gamma - 1.0) : 0.0};
  k.closure = C.closure;
  k.flux = C.flux;
  k.m = m;
  k.sc = c->d_sc;
  k.stream = c->stream;
  k.sm_count = sms;
  k.smem_optin = (size_t)optin;
  // large cells (the on-chip group kernel needs <= 256 threads x 2 blocks): L2-resident scratch
  if (N * (N + 1) / 2 > 512 && m == 4) {
    k.big_ctas = sms;
    const size_t nd = ipm::big_scratch_doubles(N, Q, m, C.q1d, npr, p) * (size_t)sms;
    k.big_scratch = dalloc<double>(nd, c->owned);
    if (!k.big_scratch) {
      ipm_destroy(c);
      return fail(IPM_ERR_CUDA, "cudaMalloc (big-cell scratch) failed");
    }
  }
  // IPM_DUAL_KERNEL=warp selects the warp-per-cell dual kernel (comparison / tests)
  auto env_is = [](const char* name, const char* v) {
    const char* e = std::getenv(name);
    return e && std::strcmp(e, v) == 0;
  };
  k.force_warp_kernel = env_is("IPM_DUAL_KERNEL", "warp") ? 1 : 0;
  k.dual_group = env_is("IPM_DUAL_KERNEL", "group") ? 1 : 0;
  k.sumfact = env_is("IPM_SUMFACT", "0") ? 0 : 1;
  k.mma_w4 = env_is("IPM_MMA_W", "4") ? 1 : 0;
  k.mma_generic = env_is("IPM_MMA_SHAPE", "generic") ? 1 : 0;
  c->graph_off = env_is("IPM_GRAPH", "0");  // comparison: launch small steps kernel by kernel
  k.mma_groups = std::getenv("IPM_MMA_GROUPS") ? std::max(1, std::atoi(std::getenv("IPM_MMA_GROUPS"))) : 0;
  k.group_t1 = env_is("IPM_GROUP_T", "1") ? 1 : 0;
  k.flux_choice = env_is("IPM_FLUX_KERNEL", "cart") ? 1 : env_is("IPM_FLUX_KERNEL", "warp") ? 2 : 0;
  k.flux_scalar_proj = std::getenv("IPM_FLUX_SCALAR_PROJ") ? 1 : 0;
  // per-level nested rules (reading 36): every level's own tables (Phi^T, omega Phi^T, the A-fragment
  // copy, omega) on its Q_l nodes, and the node indices into the finest rule for the flux
  if (level_rules) {
    const int nf = C.level_q1d[C.n_levels - 1];
    k.ad.lq.on = 1;
    for (int l = 0; l < C.n_levels; ++l) {
      const int nl = C.level_q1d[l], stride = (nf - 1) / (nl - 1), Nl = binom_total(p, C.level_M[l]);
      std::vector<double> xl, wl;
      clenshaw_curtis(nl, xl, wl);
      int Ql = 1;
      for (int d = 0; d < p; ++d) Ql *= nl;
      const int QPl = (Ql % 2 == 0) ? Ql + 1 : Ql, MTl = (Nl + 7) / 8, KSl = (Ql + 3) / 4;
      std::vector<int32_t> kf(Ql);
      std::vector<double> om(Ql), PT((size_t)Nl * QPl, 0.0), WT((size_t)Nl * QPl, 0.0), WF((size_t)MTl * KSl * 32, 0.0);
      for (int q = 0; q < Ql; ++q) {
        int r = q, kk = 0, sc = 1;
        double w = 1.0;
        for (int d = p - 1; d >= 0; --d) {
          const int jd = r % nl;
          r /= nl;
          kk += jd * stride * sc;
          sc *= nf;
          w *= 0.5 * wl[jd];
        }
        kf[q] = kk;
        om[q] = w;
        for (int i = 0; i < Nl; ++i) {
          PT[(size_t)i * QPl + q] = c->phi[(size_t)kk * N + i];  // the finest rule's basis values at the node
          WT[(size_t)i * QPl + q] = w * c->phi[(size_t)kk * N + i];
        }
      }
      for (int mt = 0; mt < MTl; ++mt)
        for (int ks = 0; ks < KSl; ++ks)
          for (int ln = 0; ln < 32; ++ln) {
            const int i = 8 * mt + ln / 4, q = 4 * ks + ln % 4;
            if (i < Nl && q < Ql) WF[((size_t)mt * KSl + ks) * 32 + ln] = WT[(size_t)i * QPl + q];
          }
      int32_t* d_kf = dalloc<int32_t>(Ql, O);
      double *d_om = dalloc<double>(Ql, O), *d_PT = dalloc<double>(PT.size(), O), *d_WT = dalloc<double>(WT.size(), O),
             *d_WF = dalloc<double>(WF.size(), O);
      if (!d_kf || !d_om || !d_PT || !d_WT || !d_WF || up(d_kf, kf.data(), Ql * 4) || up(d_om, om.data(), Ql * 8) ||
          up(d_PT, PT.data(), PT.size() * 8) || up(d_WT, WT.data(), WT.size() * 8) || up(d_WF, WF.data(), WF.size() * 8)) {
        ipm_destroy(c);
        return fail(IPM_ERR_CUDA, "per-level rule tables upload failed");
      }
      k.ad.lq.Q[l] = Ql;
      k.ad.lq.QP[l] = QPl;
      k.ad.lq.kf[l] = d_kf;
      k.ad.lq.wphit[l] = d_WT;
      ipm::Tables t = k.T;
      t.PhiT = d_PT;
      t.WPhiT = d_WT;
      t.omega = d_om;
      t.N = Nl;
      t.Q = Ql;
      t.QP = QPl;
      t.WPhiF = d_WF;
      t.MT = MTl;
      t.KS = KSl;
      t.LL = nullptr;
      t.q1d = 0;
      t.npr = 0;
      c->lq_tables[l] = t;
    }
  }
  // adaptive degree bucketed into uniform-degree launches (north star (c)): Euler 2D, tensor
  // Gauss-Legendre sum factorisation, every level's (n = N_l m, degree) among the k_dual_mma shapes
  // (n <= 24 / 40 / 64 / 88 with degrees 2 / 3 / 4 / 5); IPM_BUCKET=0 keeps the single N_max launch
  k.bucket = 0;
  if (C.n_levels > 0 && C.closure == IPM_CLOSURE_EULER && m == 4 && p == 2 && (tensor_gl || level_rules) &&
      !env_is("IPM_BUCKET", "0")) {
    bool ok = true;
    for (int l = 0; l < C.n_levels; ++l) ok = ok && C.level_M[l] >= 2 && C.level_M[l] <= 5;
    if (ok) {
      k.lists = dalloc<int32_t>((size_t)C.n_levels * std::max<int64_t>(cells, 1), c->owned);
      if (!k.lists) {
        ipm_destroy(c);
        return fail(IPM_ERR_CUDA, "cudaMalloc (level lists) failed");
      }
      for (int l = 0; l < C.n_levels; ++l) {
        const int Ml = C.level_M[l], nprl = (Ml + 1) * (Ml + 2) / 2;
        // the level's 1D rule: the context's, or its own nested Clenshaw-Curtis rule (reading 36)
        std::vector<double> xl = x1, wl = w1;
        if (level_rules) clenshaw_curtis(C.level_q1d[l], xl, wl);
        const int q1l = (int)xl.size();
        std::vector<double> LLl((size_t)q1l * nprl);
        for (int kq = 0; kq < q1l; ++kq) {
          int pr = 0;
          for (int aa = 0; aa <= Ml; ++aa)
            for (int bb = aa; bb <= Ml; ++bb, ++pr)
              LLl[(size_t)kq * nprl + pr] = 0.5 * wl[kq] * legendre_orthonormal(aa, xl[kq]) * legendre_orthonormal(bb, xl[kq]);
        }
        double* d_LLl = dalloc<double>(LLl.size(), c->owned);
        if (!d_LLl || cudaMemcpy(d_LLl, LLl.data(), LLl.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
          ipm_destroy(c);
          return fail(IPM_ERR_CUDA, "level tables upload failed");
        }
        ipm::Tables t = level_rules ? c->lq_tables[l] : k.T;
        t.N = binom_total(p, Ml);
        t.MT = (t.N + 7) / 8;
        t.LL = d_LLl;
        t.npr = nprl;
        t.q1d = q1l;
        k.Tl[l] = t;
      }
      k.bucket = 1;
    }
  }
  if (level_rules && !k.bucket) {
    ipm_destroy(c);
    return fail(IPM_ERR_UNSUPPORTED, "per-level rules need the bucketed dual launches (Euler 2D, p = 2, degrees 2-5)");
  }
  // quasi-Newton dual solve (reading 35): per-cell pair history in device memory
  k.hessian_kind = C.hessian_kind;
  k.lbfgs_m = C.lbfgs_m > 0 ? C.lbfgs_m : 8;
  k.lbfgs_pairs_reg = env_is("IPM_LBFGS_PAIRS", "reg") ? 1 : 0;
  if (C.hessian_kind == 1) {
    const bool big_ok = N * m <= 256 && p == 3 && tensor_gl && C.closure == IPM_CLOSURE_EULER && m == 4 && C.n_levels == 0;
    if (k.lbfgs_m != 8 || (N * m > 96 && !big_ok)) {
      ipm_destroy(c);
      return fail(IPM_ERR_UNSUPPORTED, "L-BFGS dual solve: lbfgs_m must be 8 and N m <= 96 (or the 3D tensor-rule Euler "
                                       "cells of config 5, N m <= 256)");
    }
    const size_t row = (size_t)N * m, mh = (size_t)k.lbfgs_m, nc = (size_t)std::max<int64_t>(cells, 1);
    c->d_lbS = dalloc<double>(nc * mh * row, c->owned);
    c->d_lbY = dalloc<double>(nc * mh * row, c->owned);
    c->d_lbR = dalloc<double>(nc * mh, c->owned);
    c->d_lbC = dalloc<int32_t>(nc, c->owned);
    c->d_lbN = dalloc<int32_t>(nc, c->owned);
    k.fb_lists = dalloc<int32_t>(nc * (size_t)std::max(1, C.n_levels), c->owned);
    if (!c->d_lbS || !c->d_lbY || !c->d_lbR || !c->d_lbC || !c->d_lbN || !k.fb_lists ||
        cudaMemset(c->d_lbC, 0, nc * 4) != cudaSuccess || cudaMemset(c->d_lbN, 0, nc * 4) != cudaSuccess) {
      ipm_destroy(c);
      return fail(IPM_ERR_CUDA, "cudaMalloc (L-BFGS history: 2 lbfgs_m N m doubles per cell, " +
                                    std::to_string(16.0 * k.lbfgs_m * row * nc / 1e9) + " GB) failed");
    }
  } else if (C.hessian_kind != 0) {
    ipm_destroy(c);
    return fail(IPM_ERR_ARG, "hessian_kind must be 0 (Newton) or 1 (L-BFGS)");
  }
  if (C.mesh_kind == IPM_MESH_TRI && cells > 0 && !std::getenv("IPM_FLUX_INDEX_ORDER")) {
    std::vector<int32_t> ord;
    ipm::morton_order(std::vector<double>(Lm.cx.begin(), Lm.cx.begin() + cells),
                      std::vector<double>(Lm.cy.begin(), Lm.cy.begin() + cells), ord);
    c->d_order = dalloc<int32_t>(ord.size(), c->owned);
    if (!c->d_order || up(c->d_order, ord.data(), ord.size() * 4)) {
      ipm_destroy(c);
      return fail(IPM_ERR_CUDA, "flux order upload failed");
    }
  }
  // boundary / interior cell lists (distributed contexts without adaptive levels: the list launches use the
  // uniform-degree kernels)
  if (nranks > 1 && C.n_levels == 0 && !c->part.send_local.empty()) {
    std::vector<char> isb(cells, 0);
    for (int32_t l : c->part.send_local) isb[l] = 1;
    std::vector<int32_t> bl, il;
    for (int64_t j = 0; j < cells; ++j) (isb[j] ? bl : il).push_back((int32_t)j);
    c->n_bnd = (int64_t)bl.size();
    c->n_int = (int64_t)il.size();
    c->d_bnd = dalloc<int32_t>(std::max<size_t>(bl.size(), 1), c->owned);
    c->d_int = dalloc<int32_t>(std::max<size_t>(il.size(), 1), c->owned);
    if (!c->d_bnd || !c->d_int || up(c->d_bnd, bl.data(), bl.size() * 4) || up(c->d_int, il.data(), il.size() * 4)) {
      ipm_destroy(c);
      return fail(IPM_ERR_CUDA, "boundary / interior lists upload failed");
    }
  }
  *out = c;
  return IPM_OK;
}

ipm_status ipm_lbfgs_reset(ipm_ctx* c) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (c->k.hessian_kind != 1) return fail(IPM_ERR_ARG, "not an L-BFGS context");
  CUDA_OK(cudaMemsetAsync(c->d_lbC, 0, (size_t)std::max<int64_t>(c->cells, 1) * 4, c->stream));
  return IPM_OK;
}

ipm_status ipm_lbfgs_history(ipm_ctx* c, double* d_S, double* d_Y, int32_t* d_count) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (c->k.hessian_kind != 1) return fail(IPM_ERR_ARG, "not an L-BFGS context");
  const size_t nc = (size_t)c->cells, per = (size_t)c->k.lbfgs_m * c->N * c->m;
  if (d_S) CUDA_OK(cudaMemcpyAsync(d_S, c->d_lbS, nc * per * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (d_Y) CUDA_OK(cudaMemcpyAsync(d_Y, c->d_lbY, nc * per * 8, cudaMemcpyDeviceToDevice, c->stream));
  if (d_count) CUDA_OK(cudaMemcpyAsync(d_count, c->d_lbC, nc * 4, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

ipm_status ipm_sizes(const ipm_ctx* c, int64_t* cells, int32_t* N, int32_t* Q, int32_t* m) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (cells) *cells = c->cells;
  if (N) *N = c->N;
  if (Q) *Q = c->Q;
  if (m) *m = c->m;
  return IPM_OK;
}

ipm_status ipm_node_band_rows(const ipm_ctx* c, int64_t* rows) {
  if (!c || !rows) return fail(IPM_ERR_ARG, "null argument");
  *rows = c->band_rows;
  return IPM_OK;
}

ipm_status ipm_get_basis(const ipm_ctx* c, double* h_xi, double* h_omega, double* h_phi) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (h_xi) std::memcpy(h_xi, c->xi.data(), c->xi.size() * 8);
  if (h_omega) std::memcpy(h_omega, c->omega.data(), c->omega.size() * 8);
  if (h_phi) std::memcpy(h_phi, c->phi.data(), c->phi.size() * 8);
  return IPM_OK;
}

ipm_status ipm_get_cell_ids(const ipm_ctx* c, int64_t* h_ids) {
  if (!c || !h_ids) return fail(IPM_ERR_ARG, "null argument");
  std::memcpy(h_ids, c->cell_ids.data(), c->cell_ids.size() * 8);
  return IPM_OK;
}

// step statistics of the device scalars -> ipm_step_info; IPM_ERR_NUMERIC when a cell failed
static ipm_status fill_info(ipm_step_info* info, const ipm::StepScalars& s) {
  info->dt = s.dt;
  info->t = s.t;
  info->residual = s.residual;
  info->newton_iters = (int64_t)s.newton_iters;
  info->failed_cells = (int64_t)s.failed;
  info->worst_status = s.worst;
  info->reserved = 0;
  for (int i = 0; i < IPM_HIST_BUCKETS; ++i) info->newton_hist[i] = (int64_t)s.hist[i];
  info->halvings = (int64_t)s.halvings;
  info->inadmissible_trials = (int64_t)s.inadm_trials;
  if (s.failed) return fail(IPM_ERR_NUMERIC, "failed cells in step");
  return IPM_OK;
}

static ipm_status launch_rc(int rc, const char* what) {
  if (rc == 0) return IPM_OK;
  if (rc < 0) return fail(IPM_ERR_UNSUPPORTED, std::string(what) + ": combination not compiled in / too large");
  return fail(IPM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString((cudaError_t)rc));
}

ipm_status ipm_dual_solve(ipm_ctx* c, const double* d_uhat, double* d_lambda, int32_t mode, int32_t* d_iters,
                          int32_t* d_status, double* d_crit) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  if (mode != IPM_NEWTON_FULL && mode != IPM_NEWTON_ONE_STEP) return fail(IPM_ERR_ARG, "mode");
  ipm::KernelCtx k = c->k;
  k.nw.mode = mode;
  if (int rc = ipm::launch_step_begin(k, 0.0)) return launch_rc(rc, "step_begin");
  ipm::DualLaunch a{};
  a.uhat = d_uhat;
  a.lam = d_lambda;
  a.iters = d_iters ? d_iters : c->d_iters;
  a.status = d_status ? d_status : c->d_status;
  a.crit = d_crit ? d_crit : c->d_crit;
  a.halv = c->d_halv;
  a.inadm = c->d_inadm;
  a.uq = nullptr;
  a.level = c->cfg.n_levels > 0 ? c->d_level : nullptr;
  a.level_new = nullptr;
  a.cells = c->cells;
  a.mode = mode;
  a.want_rate = 0;
  lb_attach(c, a, 0);
  return launch_rc(ipm::launch_dual(k, a), "dual_solve");
}

// node states of the halo cells from received duals (rows cells .. cells+halo of the node buffer)
static int halo_nodes(ipm_ctx* c, const double* d_recv) {
  if (c->halo == 0) return 0;
  ipm::KernelCtx kh = c->k;
  kh.mesh.cells = c->halo;
  double* dst = c->band_rows ? c->d_uq_halo : c->d_uq + (size_t)c->cells * c->Q * c->m;
  return ipm::launch_nodes(kh, d_recv, nullptr, dst, 0, 1);
}

// the flux update over bands of rows (banded node states): per band, the node states of its rows and
// the rows above and below from lambda (k_nodes), then the flux of the band's cells
static int band_flux(ipm_ctx* c, const double* d_lambda, ipm::FluxLaunch f) {
  const ipm::KernelCtx& k = c->k;
  const int64_t bx = k.mesh.bx, by = k.mesh.by, R = c->band_rows, row = (int64_t)c->N * c->m;
  for (int64_t r0 = 0; r0 < by; r0 += R) {
    const int64_t r1 = std::min(by, r0 + R), n0 = std::max<int64_t>(0, r0 - 1), n1 = std::min(by, r1 + 1);
    ipm::KernelCtx kn = k;
    kn.mesh.cells = (n1 - n0) * bx;
    if (int rc = ipm::launch_nodes(kn, d_lambda + n0 * bx * row, nullptr, c->d_uq, 0)) return rc;
    ipm::KernelCtx kf = k;
    kf.mesh.cells = r1 * bx;
    ipm::FluxLaunch fb = f;
    fb.uq = c->d_uq;
    fb.cell0 = r0 * bx;
    fb.uq_base = n0 * bx;
    fb.n_owned = c->cells;
    fb.uq_halo = c->d_uq_halo;
    if (int rc = ipm::launch_flux(kf, fb)) return rc;
  }
  return 0;
}

ipm_status ipm_flux_update(ipm_ctx* c, const double* d_lambda, const double* d_uhat_old, double* d_uhat_new,
                           double dt, double* d_dt) {
  if (!c || !d_lambda || !d_uhat_old || !d_uhat_new) return fail(IPM_ERR_ARG, "null argument");
  if (c->halo > 0) return fail(IPM_ERR_ARG, "ipm_flux_update needs halo duals: use ipm_step_dual/ipm_step_flux");
  const ipm::KernelCtx& k = c->k;
  if (int rc = ipm::launch_step_begin(k, c->ghost_rate)) return launch_rc(rc, "step_begin");
  if (c->band_rows) {  // the CFL rate of every cell first (no node states kept), then band by band
    if (int rc = ipm::launch_nodes(k, d_lambda, nullptr, nullptr, 1)) return launch_rc(rc, "nodes");
  } else if (int rc = ipm::launch_nodes(k, d_lambda, nullptr, c->d_uq, 1)) {
    return launch_rc(rc, "nodes");
  }
  if (int rc = ipm::launch_dt(k, -1.0, dt, c->cfg.cfl)) return launch_rc(rc, "dt");
  ipm::FluxLaunch f{c->d_uq, d_uhat_old, d_uhat_new, nullptr, nullptr, c->cfg.update_form, c->cfg.cfl};
  f.order = c->d_order;
  if (c->band_rows) {
    if (int rc = band_flux(c, d_lambda, f)) return launch_rc(rc, "flux (bands)");
  } else if (int rc = ipm::launch_flux(k, f)) {
    return launch_rc(rc, "flux");
  }
  if (d_dt) CUDA_OK(cudaMemcpyAsync(d_dt, &c->d_sc->dt, 8, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

ipm_status ipm_step_dual(ipm_ctx* c, const double* d_uhat, double* d_lambda, double* d_sendbuf,
                         uint64_t* d_rate) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  if (!c->part.send_local.empty() && !d_sendbuf) return fail(IPM_ERR_ARG, "send buffer required");
  const ipm::KernelCtx& k = c->k;
  if (int rc = ipm::launch_step_begin(k, c->ghost_rate)) return launch_rc(rc, "step_begin");
  ipm::DualLaunch a{};
  a.uhat = d_uhat;
  a.lam = d_lambda;
  a.iters = c->d_iters;
  a.status = c->d_status;
  a.crit = c->d_crit;
  a.halv = c->d_halv;
  a.inadm = c->d_inadm;
  // banded: the flux recomputes the node states; per-level rules: a node pass on the finest rule
  a.uq = (c->band_rows || c->k.ad.lq.on) ? nullptr : c->d_uq;
  a.level = c->cfg.n_levels > 0 ? c->d_level : nullptr;
  a.level_new = c->cfg.n_levels > 0 ? c->d_level_new : nullptr;
  a.cells = c->cells;
  a.mode = c->cfg.newton_mode;
  a.want_rate = 1;
  lb_attach(c, a, 0);
  if (c->timing) cudaEventRecord(c->ev[0], c->stream);
  if (int rc = ipm::launch_dual(k, a)) return launch_rc(rc, "dual_solve");
  if (c->timing) cudaEventRecord(c->ev[1], c->stream);
  if (!c->part.send_local.empty())
    if (int rc = ipm::launch_pack(k, d_lambda, c->d_send_local, (int64_t)c->part.send_local.size(), d_sendbuf))
      return launch_rc(rc, "pack");
  if (d_rate) CUDA_OK(cudaMemcpyAsync(d_rate, &c->d_sc->rate_bits, 8, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

// the dual solve of one of the two cell lists (boundary first, so its halo duals can travel while the
// interior cells solve); part 0 also begins the step and packs the send buffer, part 1 copies the rate
static ipm_status step_dual_part(ipm_ctx* c, const double* d_uhat, double* d_lambda, double* d_sendbuf,
                                 uint64_t* d_rate, int part) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  if (!c->part.send_local.empty() && !d_sendbuf && part == 0) return fail(IPM_ERR_ARG, "send buffer required");
  ipm::KernelCtx k = c->k;
  // the list launches need a uniform-degree dual kernel that takes cell lists (k_dual_mma, k_dual_big,
  // the quasi-Newton kernels): otherwise part 0 solves every cell and part 1 does nothing
  const bool split = c->d_bnd && !k.force_warp_kernel && !k.dual_group;
  if (part == 0) {
    if (int rc = ipm::launch_step_begin(k, c->ghost_rate)) return launch_rc(rc, "step_begin");
    if (c->timing) cudaEventRecord(c->ev[0], c->stream);
  }
  if (part == 0 || split) {
    ipm::DualLaunch a{};
    a.uhat = d_uhat;
    a.lam = d_lambda;
    a.iters = c->d_iters;
    a.status = c->d_status;
    a.crit = c->d_crit;
    a.halv = c->d_halv;
    a.inadm = c->d_inadm;
    a.uq = (c->band_rows || c->k.ad.lq.on) ? nullptr : c->d_uq;
    a.cells = c->cells;
    a.mode = c->cfg.newton_mode;
    a.want_rate = 1;
    lb_attach(c, a, 0);
    if (split) {
      a.list = part == 0 ? c->d_bnd : c->d_int;
      a.cells = part == 0 ? c->n_bnd : c->n_int;
      a.queue = part == 0 ? &c->d_sc->work_counter : &c->d_sc->work_counter2;
      a.row = c->N * c->m;
    }
    if (a.cells > 0)
      if (int rc = ipm::launch_dual(k, a)) return launch_rc(rc, "dual_solve");
  }
  if (part == 0 && !c->part.send_local.empty())
    if (int rc = ipm::launch_pack(k, d_lambda, c->d_send_local, (int64_t)c->part.send_local.size(), d_sendbuf))
      return launch_rc(rc, "pack");
  if (part == 1) {
    if (c->timing) cudaEventRecord(c->ev[1], c->stream);
    if (d_rate) CUDA_OK(cudaMemcpyAsync(d_rate, &c->d_sc->rate_bits, 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  return IPM_OK;
}

ipm_status ipm_step_dual_boundary(ipm_ctx* c, const double* d_uhat, double* d_lambda, double* d_sendbuf) {
  return step_dual_part(c, d_uhat, d_lambda, d_sendbuf, nullptr, 0);
}

ipm_status ipm_step_dual_interior(ipm_ctx* c, const double* d_uhat, double* d_lambda, uint64_t* d_rate) {
  return step_dual_part(c, d_uhat, d_lambda, nullptr, d_rate, 1);
}

ipm_status ipm_step_flux(ipm_ctx* c, double* d_uhat, double* d_lambda, const double* d_recvbuf,
                         const uint64_t* d_rate, double t_end, ipm_step_info* info) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  if (c->halo > 0 && !d_recvbuf) return fail(IPM_ERR_ARG, "receive buffer required");
  const ipm::KernelCtx& k = c->k;
  if (d_rate) CUDA_OK(cudaMemcpyAsync(&c->d_sc->rate_bits, d_rate, 8, cudaMemcpyDeviceToDevice, c->stream));
  if (int rc = halo_nodes(c, d_recvbuf)) return launch_rc(rc, "halo nodes");
  if (int rc = ipm::launch_dt(k, t_end, -1.0, c->cfg.cfl)) return launch_rc(rc, "dt");
  const int32_t* lvl_new = c->cfg.n_levels > 0 ? c->d_level_new : nullptr;
  ipm::FluxLaunch f{c->d_uq, d_uhat, d_uhat, lvl_new, d_lambda, c->cfg.update_form, c->cfg.cfl};
  f.order = c->d_order;
  if (c->timing) cudaEventRecord(c->ev[2], c->stream);
  // per-level nested rules (reading 36): every owned cell's states at every node of the finest rule
  // from its duals at its old level (the flux of a cell at level l reads the nodes of Q_l)
  if (k.ad.lq.on)
    if (int rc = ipm::launch_nodes(k, d_lambda, nullptr, c->d_uq, 0)) return launch_rc(rc, "nodes (level rules)");
  if (c->band_rows) {
    if (int rc = band_flux(c, d_lambda, f)) return launch_rc(rc, "flux (bands)");
  } else if (int rc = ipm::launch_flux(k, f)) {
    return launch_rc(rc, "flux");
  }
  if (c->timing) cudaEventRecord(c->ev[3], c->stream);
  if (c->cfg.n_levels > 0) std::swap(c->d_level, c->d_level_new);
  if (c->cfg.nranks <= 1)  // distributed: the caller advances with the global residual
    if (int rc = ipm::launch_retard(k)) return launch_rc(rc, "retard");
  if (info) {
    ipm::StepScalars s;
    CUDA_OK(cudaMemcpyAsync(&s, c->d_sc, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    return fill_info(info, s);
  }
  return IPM_OK;
}

// the launches of one single-rank step (no synchronisation, no read-back)
static ipm_status enqueue_step(ipm_ctx* c, double* d_uhat, double* d_lambda, double t_end) {
  if (ipm_status s = ipm_step_dual(c, d_uhat, d_lambda, nullptr, nullptr)) return s;
  return ipm_step_flux(c, d_uhat, d_lambda, nullptr, nullptr, t_end, nullptr);
}

// capture the step's launches into a CUDA graph on a private stream (the ctx stream may be the legacy
// default stream, which cannot be captured); false: not capturable, launch directly from now on
static bool capture_step(ipm_ctx* c, double* d_uhat, double* d_lambda, double t_end) {
  if (c->gexec) {
    cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
  }
  if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) return false;
  void* saved = c->k.stream;
  cudaStream_t saved_s = c->stream;
  c->k.stream = c->cap_stream;
  c->stream = c->cap_stream;
  cudaGraph_t graph = nullptr;
  bool ok = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  const ipm_status st = ok ? enqueue_step(c, d_uhat, d_lambda, t_end) : IPM_ERR_CUDA;
  ok = (cudaStreamEndCapture(c->cap_stream, &graph) == cudaSuccess) && ok && st == IPM_OK && graph;
  c->k.stream = saved;
  c->stream = saved_s;
  if (ok) ok = cudaGraphInstantiate(&c->gexec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();  // a failed capture leaves no sticky error
  if (!ok) {
    c->gexec = nullptr;
    return false;
  }
  c->g_uhat = d_uhat;
  c->g_lambda = d_lambda;
  c->g_tend = t_end;
  return true;
}

ipm_status ipm_step(ipm_ctx* c, double* d_uhat, double* d_lambda, double t_end, ipm_step_info* info) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  if (c->halo > 0 || !c->part.send_local.empty())
    return fail(IPM_ERR_ARG, "distributed context: use ipm_step_dual / exchange / ipm_step_flux");
  const bool graph = !c->graph_off && !c->timing && c->cfg.n_levels == 0 && c->cells < IPM_GRAPH_MAX_CELLS;
  if (graph && (!c->gexec || c->g_uhat != d_uhat || c->g_lambda != d_lambda || c->g_tend != t_end))
    if (!capture_step(c, d_uhat, d_lambda, t_end)) c->graph_off = true;
  if (graph && c->gexec) {
    CUDA_OK(cudaGraphLaunch(c->gexec, c->stream));
  } else if (ipm_status s = enqueue_step(c, d_uhat, d_lambda, t_end)) {
    return s;
  }
  if (info) {
    ipm::StepScalars s;
    CUDA_OK(cudaMemcpyAsync(&s, c->d_sc, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    return fill_info(info, s);
  }
  return IPM_OK;
}

ipm_status ipm_step_host(ipm_ctx* c, double* h_uhat, double* h_lambda, double* d_uhat, double* d_lambda, double t_end,
                         int32_t nchunks, ipm_step_info* info) {
  if (!c || !h_uhat || !h_lambda || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  if (c->halo > 0 || !c->part.send_local.empty())
    return fail(IPM_ERR_ARG, "ipm_step_host: single-rank contexts only");
  if (nchunks < 1) return fail(IPM_ERR_ARG, "nchunks must be >= 1");
  const int64_t cells = c->cells;
  const int nch = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, std::max<int64_t>(cells, 1)));
  if (!c->copy_stream) CUDA_OK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  while ((int)c->hev.size() < 2 * nch + 2) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->hev.push_back(e);
  }
  cudaStream_t ms = c->stream, cs = c->copy_stream;
  const size_t row = (size_t)c->N * c->m;
  const bool adaptive = c->cfg.n_levels > 0;
  const ipm::KernelCtx& k = c->k;
  auto lo = [&](int i) { return cells * i / nch; };
  // the copy stream starts after everything queued on the ctx stream (the previous step)
  CUDA_OK(cudaEventRecord(c->hev[2 * nch], ms));
  CUDA_OK(cudaStreamWaitEvent(cs, c->hev[2 * nch], 0));
  for (int i = 0; i < nch; ++i) {
    const size_t r0 = (size_t)lo(i), nr = (size_t)(lo(i + 1) - lo(i));
    CUDA_OK(cudaMemcpyAsync(d_uhat + r0 * row, h_uhat + r0 * row, nr * row * 8, cudaMemcpyHostToDevice, cs));
    CUDA_OK(cudaMemcpyAsync(d_lambda + r0 * row, h_lambda + r0 * row, nr * row * 8, cudaMemcpyHostToDevice, cs));
    CUDA_OK(cudaEventRecord(c->hev[i], cs));
  }
  if (int rc = ipm::launch_step_begin(k, c->ghost_rate)) return launch_rc(rc, "step_begin");
  for (int i = 0; i < nch; ++i) {
    const int64_t r0 = lo(i), nr = lo(i + 1) - lo(i);
    CUDA_OK(cudaStreamWaitEvent(ms, c->hev[i], 0));
    if (nr == 0) continue;
    // dual solve of cells [r0, r0 + nr): a fresh work queue, pointers offset to the range
    CUDA_OK(cudaMemsetAsync(&c->d_sc->work_counter, 0, sizeof(int), ms));
    ipm::KernelCtx kc = k;
    if (kc.mesh.rate_geo) kc.mesh.rate_geo += r0;
    ipm::DualLaunch a{};
    a.uhat = d_uhat + r0 * row;
    a.lam = d_lambda + r0 * row;
    a.iters = c->d_iters + r0;
    a.status = c->d_status + r0;
    a.crit = c->d_crit + r0;
    a.halv = c->d_halv + r0;
    a.inadm = c->d_inadm + r0;
    a.uq = (c->band_rows || c->k.ad.lq.on) ? nullptr : c->d_uq + (size_t)r0 * c->Q * c->m;
    a.level = adaptive ? c->d_level + r0 : nullptr;
    a.level_new = adaptive ? c->d_level_new + r0 : nullptr;
    a.cells = nr;
    a.mode = c->cfg.newton_mode;
    a.want_rate = 1;
    lb_attach(c, a, r0);
    if (int rc = ipm::launch_dual(kc, a)) return launch_rc(rc, "dual_solve");
    if (!adaptive) {  // final duals of the range go back while later ranges solve
      CUDA_OK(cudaEventRecord(c->hev[nch + i], ms));
      CUDA_OK(cudaStreamWaitEvent(cs, c->hev[nch + i], 0));
      CUDA_OK(cudaMemcpyAsync(h_lambda + r0 * row, d_lambda + r0 * row, (size_t)nr * row * 8, cudaMemcpyDeviceToHost,
                              cs));
    }
  }
  if (ipm_status s = ipm_step_flux(c, d_uhat, d_lambda, nullptr, nullptr, t_end, nullptr)) return s;
  CUDA_OK(cudaMemcpyAsync(h_uhat, d_uhat, (size_t)cells * row * 8, cudaMemcpyDeviceToHost, ms));
  if (adaptive) CUDA_OK(cudaMemcpyAsync(h_lambda, d_lambda, (size_t)cells * row * 8, cudaMemcpyDeviceToHost, ms));
  CUDA_OK(cudaEventRecord(c->hev[2 * nch + 1], cs));
  CUDA_OK(cudaStreamWaitEvent(ms, c->hev[2 * nch + 1], 0));
  ipm::StepScalars s;
  CUDA_OK(cudaMemcpyAsync(&s, c->d_sc, sizeof(s), cudaMemcpyDeviceToHost, ms));
  CUDA_OK(cudaStreamSynchronize(ms));
  if (info) return fill_info(info, s);
  return IPM_OK;
}

ipm_status ipm_retard_stage(ipm_ctx* c, int32_t* stage) {
  if (!c || !stage) return fail(IPM_ERR_ARG, "null argument");
  int st = 0;
  CUDA_OK(cudaMemcpyAsync(&st, &c->d_sc->stage, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  *stage = st;
  return IPM_OK;
}

ipm_status ipm_retard_advance(ipm_ctx* c, double global_residual) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  const ipm::Adapt& ad = c->k.ad;
  if (ad.n_retard <= 0) return IPM_OK;
  int st = 0;
  CUDA_OK(cudaMemcpyAsync(&st, &c->d_sc->stage, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  if (st < ad.n_retard && global_residual < ad.retard_eps[st]) {
    ++st;
    CUDA_OK(cudaMemcpyAsync(&c->d_sc->stage, &st, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
  }
  return IPM_OK;
}

ipm_status ipm_halo_layout(const ipm_ctx* c, int32_t* npeers, int64_t* nsend, int64_t* nrecv, int32_t* h_peers,
                           int32_t* h_send_count, int32_t* h_recv_count) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  const ipm::Partition& P = c->part;
  if (npeers) *npeers = (int32_t)P.peers.size();
  if (nsend) *nsend = (int64_t)P.send_gid.size();
  if (nrecv) *nrecv = (int64_t)P.halo_gid.size();
  for (size_t i = 0; i < P.peers.size(); ++i) {
    if (h_peers) h_peers[i] = P.peers[i];
    if (h_send_count) h_send_count[i] = P.send_count[i];
    if (h_recv_count) h_recv_count[i] = P.recv_count[i];
  }
  return IPM_OK;
}

ipm_status ipm_partition_query(const ipm_config* cfg, int64_t* cells, int64_t* nhalo, int32_t* npeers,
                               int64_t* nsend, int64_t* h_local_gid, int64_t* h_halo_gid, int32_t* h_peers,
                               int32_t* h_send_count, int32_t* h_recv_count, int64_t* h_send_gid) {
  if (!cfg) return fail(IPM_ERR_ARG, "null config");
  ipm::MeshTables G;
  ipm::Partition P;
  std::string err;
  if (!ipm::build_mesh(*cfg, G, err)) return fail(IPM_ERR_ARG, err);
  const int nr = cfg->nranks > 0 ? cfg->nranks : 1;
  if (!ipm::build_partition(*cfg, G, nr > 1 ? cfg->rank : 0, nr, P, err)) return fail(IPM_ERR_ARG, err);
  if (cells) *cells = (int64_t)P.local_gid.size();
  if (nhalo) *nhalo = (int64_t)P.halo_gid.size();
  if (npeers) *npeers = (int32_t)P.peers.size();
  if (nsend) *nsend = (int64_t)P.send_gid.size();
  if (h_local_gid) std::memcpy(h_local_gid, P.local_gid.data(), P.local_gid.size() * 8);
  if (h_halo_gid) std::memcpy(h_halo_gid, P.halo_gid.data(), P.halo_gid.size() * 8);
  if (h_send_gid) std::memcpy(h_send_gid, P.send_gid.data(), P.send_gid.size() * 8);
  for (size_t i = 0; i < P.peers.size(); ++i) {
    if (h_peers) h_peers[i] = P.peers[i];
    if (h_send_count) h_send_count[i] = P.send_count[i];
    if (h_recv_count) h_recv_count[i] = P.recv_count[i];
  }
  return IPM_OK;
}

static ipm_status project_ic_impl(ipm_ctx* c, const ipm_ic* ic, double* d_uhat, double* d_nodes) {
  const ipm_config& C = c->cfg;
  const int Q = c->Q, m = c->m, p = c->p;
  const int R = ic->kind == IPM_IC_UNIFORM ? 1 : (ic->kind == IPM_IC_STEP1D ? 2 : 4);
  if (ic->kind == IPM_IC_STEP1D && C.mesh_kind != IPM_MESH_1D) return fail(IPM_ERR_ARG, "STEP1D needs a 1D mesh");
  if (ic->kind == IPM_IC_QUAD2D && C.mesh_kind != IPM_MESH_CART2D)
    return fail(IPM_ERR_ARG, "QUAD2D needs a cartesian mesh");
  std::vector<double> region((size_t)R * Q * m), split((size_t)Q * 2);
  for (int k = 0; k < Q; ++k) {
    const double* x = &c->xi[(size_t)k * p];
    for (int r = 0; r < R; ++r) HostPrim::eval(ic->state[r], x, p, m, C.gamma, &region[((size_t)r * Q + k) * m]);
    double xs = ic->xs0, ys = ic->ys0;
    for (int d = 0; d < p && d < 3; ++d) {
      xs += ic->xs1[d] * x[d];
      ys += ic->ys1[d] * x[d];
    }
    split[k * 2] = xs;
    split[k * 2 + 1] = ys;
  }
  // temporary device copies (setup helper, synchronous)
  double *d_reg = nullptr, *d_split = nullptr;
  CUDA_OK(cudaMalloc(&d_reg, region.size() * 8));
  CUDA_OK(cudaMalloc(&d_split, split.size() * 8));
  CUDA_OK(cudaMemcpy(d_reg, region.data(), region.size() * 8, cudaMemcpyHostToDevice));
  CUDA_OK(cudaMemcpy(d_split, split.data(), split.size() * 8, cudaMemcpyHostToDevice));
  c->initial_level = ic->initial_level;
  if (C.n_levels > 0) {
    std::vector<int32_t> lv(c->cells, ic->initial_level);
    CUDA_OK(cudaMemcpy(c->d_level, lv.data(), lv.size() * 4, cudaMemcpyHostToDevice));
  }
  const double dx = C.nx > 0 ? (C.x1 - C.x0) / C.nx : 0.0, dy = C.ny > 0 ? (C.y1 - C.y0) / C.ny : 0.0;
  int rc = ipm::launch_project_ic(c->k, d_reg, d_split, ic->kind, C.nx, C.x0, C.y0, dx, dy,
                                  C.n_levels > 0 ? c->d_level : nullptr, c->d_gid, d_uhat, d_nodes);
  ipm::StepScalars s{};
  cudaMemcpy(c->d_sc, &s, sizeof(s), cudaMemcpyHostToDevice);  // t = 0
  cudaStreamSynchronize(c->stream);
  cudaFree(d_reg);
  cudaFree(d_split);
  return launch_rc(rc, "project_ic");
}

ipm_status ipm_project_ic(ipm_ctx* c, const ipm_ic* ic, double* d_uhat) {
  if (!c || !ic || !d_uhat) return fail(IPM_ERR_ARG, "null argument");
  c->sc_last_out = nullptr;
  return project_ic_impl(c, ic, d_uhat, nullptr);
}

// ---- Stochastic Collocation (reading 32) -----------------------------------
ipm_status ipm_sc_init(ipm_ctx* c, const ipm_ic* ic, double* d_nodes) {
  if (!c || !ic || !d_nodes) return fail(IPM_ERR_ARG, "null argument");
  if (c->halo > 0 || !c->part.send_local.empty()) return fail(IPM_ERR_ARG, "SC: single-rank contexts only");
  c->sc_last_out = nullptr;
  return project_ic_impl(c, ic, nullptr, d_nodes);
}

ipm_status ipm_sc_step(ipm_ctx* c, const double* d_in, double* d_out, double t_end, ipm_step_info* info) {
  if (!c || !d_in || !d_out || d_in == d_out) return fail(IPM_ERR_ARG, "null or aliased argument");
  if (c->halo > 0 || !c->part.send_local.empty()) return fail(IPM_ERR_ARG, "SC: single-rank contexts only");
  const ipm::KernelCtx& k = c->k;
  // the CFL rate of d_in: cached by the previous step when d_in is its output, else a rate pass
  const bool cached = d_in == c->sc_last_out;
  if (int rc = ipm::launch_sc_begin(k, c->ghost_rate, cached ? 1 : 0)) return launch_rc(rc, "sc_begin");
  if (!cached)
    if (int rc = ipm::launch_sc_rate(k, d_in)) return launch_rc(rc, "sc_rate");
  if (int rc = ipm::launch_dt(k, t_end, -1.0, c->cfg.cfl)) return launch_rc(rc, "dt");
  if (int rc = ipm::launch_sc_update(k, d_in, d_out)) return launch_rc(rc, "sc_update");
  c->sc_last_out = d_out;
  if (info) {
    ipm::StepScalars s;
    CUDA_OK(cudaMemcpyAsync(&s, c->d_sc, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
    CUDA_OK(cudaStreamSynchronize(c->stream));
    info->dt = s.dt;
    info->t = s.t;
    info->residual = s.residual;
    info->newton_iters = 0;
    info->failed_cells = 0;
    info->worst_status = 0;
  }
  return IPM_OK;
}

ipm_status ipm_sc_moments(ipm_ctx* c, const double* d_nodes, double* d_uhat) {
  if (!c || !d_nodes || !d_uhat) return fail(IPM_ERR_ARG, "null argument");
  return launch_rc(ipm::launch_sc_moments(c->k, d_nodes, d_uhat), "sc_moments");
}

ipm_status ipm_warm_start(ipm_ctx* c, const double* d_uhat, double* d_lambda) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  return launch_rc(ipm::launch_warm_start(c->k, d_uhat, d_lambda), "warm_start");
}

ipm_status ipm_moments_from_dual(ipm_ctx* c, const double* d_lambda, double* d_uhat) {
  if (!c || !d_uhat || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  return launch_rc(ipm::launch_nodes(c->k, d_lambda, d_uhat, nullptr, 0), "moments_from_dual");
}

ipm_status ipm_stress_dual(ipm_ctx* c, const double* d_base, const double* d_z, double rel, double abs_,
                           double* d_lambda) {
  if (!c || !d_base || !d_z || !d_lambda) return fail(IPM_ERR_ARG, "null argument");
  return launch_rc(ipm::launch_stress(c->k, d_base, d_z, rel, abs_, d_lambda), "stress_dual");
}

ipm_status ipm_get_levels(ipm_ctx* c, int32_t* d_levels) {
  if (!c || !d_levels) return fail(IPM_ERR_ARG, "null argument");
  CUDA_OK(cudaMemcpyAsync(d_levels, c->d_level, c->cells * 4, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

ipm_status ipm_set_levels(ipm_ctx* c, const int32_t* d_levels) {
  if (!c || !d_levels) return fail(IPM_ERR_ARG, "null argument");
  CUDA_OK(cudaMemcpyAsync(c->d_level, d_levels, c->cells * 4, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

ipm_status ipm_last_cell_stats(ipm_ctx* c, int32_t* d_iters, int32_t* d_status) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (d_iters) CUDA_OK(cudaMemcpyAsync(d_iters, c->d_iters, c->cells * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (d_status) CUDA_OK(cudaMemcpyAsync(d_status, c->d_status, c->cells * 4, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

ipm_status ipm_last_cell_linesearch(ipm_ctx* c, int32_t* d_halvings, int32_t* d_inadmissible) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (d_halvings) CUDA_OK(cudaMemcpyAsync(d_halvings, c->d_halv, c->cells * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (d_inadmissible)
    CUDA_OK(cudaMemcpyAsync(d_inadmissible, c->d_inadm, c->cells * 4, cudaMemcpyDeviceToDevice, c->stream));
  return IPM_OK;
}

ipm_status ipm_get_status(ipm_ctx* c, int32_t* worst, int64_t* n_failed) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  ipm::StepScalars s;
  CUDA_OK(cudaMemcpyAsync(&s, c->d_sc, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  if (worst) *worst = s.worst;
  if (n_failed) *n_failed = (int64_t)s.failed;
  return IPM_OK;
}

ipm_status ipm_get_time(ipm_ctx* c, double* t) {
  if (!c || !t) return fail(IPM_ERR_ARG, "null argument");
  CUDA_OK(cudaMemcpyAsync(t, &c->d_sc->t, 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  return IPM_OK;
}

ipm_status ipm_set_time(ipm_ctx* c, double t) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  c->sc_last_out = nullptr;
  CUDA_OK(cudaMemcpyAsync(&c->d_sc->t, &t, 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  return IPM_OK;
}


ipm_status ipm_enable_timing(ipm_ctx* c, int32_t on) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  c->timing = on != 0;
  return IPM_OK;
}

ipm_status ipm_last_kernel_ms(ipm_ctx* c, float* dual_ms, float* flux_ms) {
  if (!c) return fail(IPM_ERR_ARG, "null ctx");
  if (!c->timing) return fail(IPM_ERR_ARG, "timing not enabled");
  CUDA_OK(cudaEventSynchronize(c->ev[3]));
  if (dual_ms) CUDA_OK(cudaEventElapsedTime(dual_ms, c->ev[0], c->ev[1]));
  if (flux_ms) CUDA_OK(cudaEventElapsedTime(flux_ms, c->ev[2], c->ev[3]));
  return IPM_OK;
}

const char* ipm_last_dual_kernel(void) { return ipm::last_dual_kernel(); }
size_t ipm_struct_size(int32_t which) {
  return which == 0 ? sizeof(ipm_config) : which == 1 ? sizeof(ipm_ic) : which == 2 ? sizeof(ipm_step_info) : 0;
}
const char* ipm_last_flux_kernel(void) { return ipm::last_flux_kernel(); }

ipm_status ipm_debug_phase_cycles(uint64_t* h_out) {
  if (!h_out) return fail(IPM_ERR_ARG, "null argument");
  unsigned long long v[8];
  if (int rc = ipm::debug_phase_cycles(v)) return launch_rc(rc, "debug_phase_cycles");
  for (int i = 0; i < 8; ++i) h_out[i] = v[i];
  return IPM_OK;
}

}  // extern "C"
