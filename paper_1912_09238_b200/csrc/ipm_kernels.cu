// ipm_kernels.cu — sm_100a kernels of the IPM hot path (fp64).
//
//   k_dual_warp   one warp per spatial cell, persistent CTAs pulling cells from an atomic queue
//                 (Newton counts differ from cell to cell).  Per iteration:
//                   Lambda_k = Phi lambda            (lanes over nodes k)
//                   u_k = u_s(Lambda_k), J_k = grad u_s(Lambda_k), s_*(Lambda_k)
//                   g = Phi^T (omega o u) - uhat     (lanes over outputs (i,a))
//                   H_{(i,a),(j,b)} = sum_k omega_k phi_ki phi_kj J_ab,k   (lanes over pairs i<=j)
//                   packed-lower Cholesky of H in shared memory, d = -H^{-1} g
//                   Armijo backtracking on L (reading 3'), trial = next iterate's node data
//                 epilogue: lambda, iteration count, status, node states u_k (for the flux),
//                 CFL rate, refinement level.
//   k_flux_warp   one warp per cell: kinetic flux at every node of every face (PAPER.md:144-146,
//                 460-462), projection Phi^T(omega o .) and the conservative / c-form update.
//   small kernels: step begin, dt, IC projection, warm start, h(lambda), stress duals.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "ipm_device.cuh"
#include "ipm_internal.h"

namespace ipm {

// ------------------------------------------------------------------------------------------------
// geometry of the per-warp shared-memory workspace of the dual kernel
// ------------------------------------------------------------------------------------------------
template <int MS>
struct DualLayout {
  static constexpr int MM = MS * (MS + 1) / 2;
  static constexpr int NS = ((MS + MM) % 2 == 0) ? MS + MM + 1 : MS + MM;  // odd node stride
  static __host__ __device__ int per_warp(int N, int Q) {
    const int n = N * MS;
    int w = 5 * n + Q * NS + n * (n + 1) / 2;
    return (w + 1) & ~1;  // keep 16-byte alignment between warps
  }
  static __host__ __device__ int tables(int N, int QP) { return 2 * N * QP; }
};

__device__ __forceinline__ int packed(int r, int c) { return r * (r + 1) / 2 + c; }  // r >= c

// node pass: Lambda = Phi lam, closure at every node -> nb, returns admissibility (warp-uniform),
// s1 = sum_k omega_k s_*(Lambda_k), s2 = sum_k omega_k |s_*(Lambda_k)|
template <int CL, int MS>
__device__ __forceinline__ bool warp_eval(const double* __restrict__ lamv, int Nl, const double* __restrict__ sPhiT,
                                          int QP, const double* __restrict__ omega, int Q, double* __restrict__ nb,
                                          const ClParams& cp, double& s1, double& s2, int lane) {
  using L = DualLayout<MS>;
  bool ok = true;
  double a1 = 0.0, a2 = 0.0;
  for (int k = lane; k < Q; k += 32) {
    double Lam[MS];
#pragma unroll
    for (int a = 0; a < MS; ++a) Lam[a] = 0.0;
    for (int i = 0; i < Nl; ++i) {
      const double ph = sPhiT[i * QP + k];
#pragma unroll
      for (int a = 0; a < MS; ++a) Lam[a] = fma(lamv[i * MS + a], ph, Lam[a]);
    }
    double u[MS], J[L::MM], ss;
    const bool okk = Closure<CL, MS>::eval(Lam, u, J, ss, cp);
    ok = ok && okk;
    double* row = nb + k * L::NS;
#pragma unroll
    for (int a = 0; a < MS; ++a) row[a] = u[a];
#pragma unroll
    for (int q = 0; q < L::MM; ++q) row[MS + q] = J[q];
    const double w = omega[k];
    a1 = fma(w, ss, a1);
    a2 = fma(w, fabs(ss), a2);
  }
  ok = __all_sync(FULL_MASK, ok);
  s1 = warp_sum(a1);
  s2 = warp_sum(a2);
  __syncwarp();
  return ok && isfinite(s1);
}

// g = Phi^T(omega o u) - uhat ; returns crit = sum_a ||g_{.,a}||_2 (warp-uniform)
template <int MS>
__device__ __forceinline__ double warp_grad(const double* __restrict__ nb, const double* __restrict__ sWPhiT, int QP,
                                            int Q, int Nl, const double* __restrict__ uh, double* __restrict__ g,
                                            int lane) {
  using L = DualLayout<MS>;
  const int n = Nl * MS;
  double part[MS];
#pragma unroll
  for (int a = 0; a < MS; ++a) part[a] = 0.0;
  for (int r = lane; r < n; r += 32) {
    const int i = r / MS, a = r - i * MS;
    const double* wp = sWPhiT + i * QP;
    double s = 0.0;
    for (int k = 0; k < Q; ++k) s = fma(wp[k], nb[k * L::NS + a], s);
    const double gr = s - uh[r];
    g[r] = gr;
#pragma unroll
    for (int b = 0; b < MS; ++b)
      if (b == a) part[b] = fma(gr, gr, part[b]);
  }
  double crit = 0.0;
#pragma unroll
  for (int a = 0; a < MS; ++a) crit += sqrt(warp_sum(part[a]));
  __syncwarp();
  return crit;
}

// H (packed lower, n x n) = sum_k omega_k J_k (x) phi_k phi_k^T
template <int MS>
__device__ __forceinline__ void warp_hessian(const double* __restrict__ nb, const double* __restrict__ sPhiT,
                                             const double* __restrict__ sWPhiT, int QP, int Q, int Nl,
                                             double* __restrict__ H, int lane) {
  using L = DualLayout<MS>;
  const int NP = Nl * (Nl + 1) / 2;
  for (int pp = lane; pp < NP; pp += 32) {
    int j = (int)((sqrtf(8.0f * pp + 1.0f) - 1.0f) * 0.5f);
    while (j * (j + 1) / 2 > pp) --j;
    while ((j + 1) * (j + 2) / 2 <= pp) ++j;
    const int i = pp - j * (j + 1) / 2;  // i <= j
    double acc[L::MM];
#pragma unroll
    for (int q = 0; q < L::MM; ++q) acc[q] = 0.0;
    const double* wi = sWPhiT + i * QP;
    const double* pj = sPhiT + j * QP;
    for (int k = 0; k < Q; ++k) {
      const double f = wi[k] * pj[k];
      const double* Jk = nb + k * L::NS + MS;
#pragma unroll
      for (int q = 0; q < L::MM; ++q) acc[q] = fma(f, Jk[q], acc[q]);
    }
#pragma unroll
    for (int a = 0; a < MS; ++a)
#pragma unroll
      for (int b = 0; b < MS; ++b) {
        const double v = acc[a <= b ? sym_idx<MS>(a, b) : sym_idx<MS>(b, a)];
        const int r1 = i * MS + a, r2 = j * MS + b;
        if (r1 >= r2)
          H[packed(r1, r2)] = v;
        else
          H[packed(r2, r1)] = v;
      }
  }
  __syncwarp();
}

// in-place Cholesky of packed-lower H, then d = -H^{-1} g.  Returns false on a non-positive pivot.
__device__ __forceinline__ bool warp_chol_solve(double* __restrict__ H, int n, const double* __restrict__ g,
                                                double* __restrict__ d, int lane) {
  for (int k = 0; k < n; ++k) {
    const double piv = H[packed(k, k)];
    if (!(piv > 0.0) || !isfinite(piv)) return false;  // warp-uniform (same address)
    const double Lkk = sqrt(piv);
    __syncwarp();
    if (lane == 0) H[packed(k, k)] = Lkk;
    for (int i = k + 1 + lane; i < n; i += 32) H[packed(i, k)] = H[packed(i, k)] / Lkk;
    __syncwarp();
    for (int i = k + 1 + lane; i < n; i += 32) {
      const double lik = H[packed(i, k)];
      double* row = H + packed(i, 0);
      for (int jj = k + 1; jj <= i; ++jj) row[jj] = fma(-lik, H[packed(jj, k)], row[jj]);
    }
    __syncwarp();
  }
  for (int r = lane; r < n; r += 32) d[r] = -g[r];
  __syncwarp();
  for (int k = 0; k < n; ++k) {  // L y = -g
    const double yk = d[k] / H[packed(k, k)];
    __syncwarp();
    if (lane == 0) d[k] = yk;
    for (int i = k + 1 + lane; i < n; i += 32) d[i] = fma(-H[packed(i, k)], yk, d[i]);
    __syncwarp();
  }
  for (int k = n - 1; k >= 0; --k) {  // L^T d = y
    const double dk = d[k] / H[packed(k, k)];
    __syncwarp();
    if (lane == 0) d[k] = dk;
    for (int i = lane; i < k; i += 32) d[i] = fma(-H[packed(k, i)], dk, d[i]);
    __syncwarp();
  }
  return true;
}

__device__ __forceinline__ double warp_dot(const double* a, const double* b, int n, int lane) {
  double s = 0.0;
  for (int r = lane; r < n; r += 32) s = fma(a[r], b[r], s);
  return warp_sum(s);
}
__device__ __forceinline__ double warp_absdot(const double* a, const double* b, int n, int lane) {
  double s = 0.0;
  for (int r = lane; r < n; r += 32) s += fabs(a[r] * b[r]);
  return warp_sum(s);
}

// CFL rate of a node state (reading 15)
template <int CL, int MS>
__device__ __forceinline__ double node_rate(const double* u, const Mesh& M, int64_t cell, double gamma) {
  if constexpr (MS == 1) {
    return fabs(u[0]) * M.inv_dx;
  } else {
    if (M.kind == MK_1D) return Euler<MS>::speed_dir(u, 0, gamma) * M.inv_dx;
    if (M.kind == MK_CART) {  // (|v_x| + c)/dx + (|v_y| + c)/dy with 1/rho, p and c formed once
      const double irho = rcp_nr(u[0]);
      double m2 = 0.0;
#pragma unroll
      for (int k = 0; k < MS - 2; ++k) m2 = fma(u[1 + k], u[1 + k], m2);
      const double p = (gamma - 1.0) * (u[MS - 1] - 0.5 * m2 * irho);
      const double c = sqrt_nr(gamma * p * irho);
      return (fabs(u[1] * irho) + c) * M.inv_dx + (fabs(u[2] * irho) + c) * M.inv_dy;
    }
    return Euler<MS>::speed_norm(u, gamma) * M.rate_geo[cell];
  }
}

// refinement retardation (Algorithm 4; reading 31): the current stage caps the
// level index
__device__ __forceinline__ int retard_cap(const Adapt& ad, const StepScalars* sc, int nl) {
  if (ad.n_retard > 0) {
    const int st = *(volatile const int*)&sc->stage;
    if (st < ad.n_retard && nl > ad.retard_level[st]) nl = ad.retard_level[st];
  }
  return nl;
}

// per-cell outcome of a dual solve (one thread per cell): per-cell arrays, the step's Newton-count
// histogram and line-search counters (ipm_step_info)
__device__ __forceinline__ void cell_stats(const DualLaunch& A, StepScalars* sc, int64_t cell, int l, int status,
                                           int hv, int ia, double crit) {
  if (A.accumulate) {  // Newton fallback of reading 35: totals over both passes
    if (A.iters) l += A.iters[cell];
    if (A.halv) hv += A.halv[cell];
    if (A.inadm) ia += A.inadm[cell];
  }
  if (A.iters) A.iters[cell] = l;
  if (A.status) A.status[cell] = status;
  if (A.crit) A.crit[cell] = crit;
  if (A.halv) A.halv[cell] = hv;
  if (A.inadm) A.inadm[cell] = ia;
  atomicAdd(&sc->hist[l < kHistBuckets - 1 ? l : kHistBuckets - 1], 1ull);
  if (hv) atomicAdd(&sc->halvings, (unsigned long long)hv);
  if (ia) atomicAdd(&sc->inadm_trials, (unsigned long long)ia);
}

// next refinement level from the indicator S (readings 19, 20): every cell
// whose dual solve ended on an admissible iterate (all but IPM_CELL_INADMISSIBLE, reading 34) moves
// one level down if S < delta_dec, up if S > delta_inc; then the retardation cap (Alg. 4)
__device__ __forceinline__ int next_level(const Adapt& ad, const StepScalars* sc, int lvl, int status, double S) {
  int nl = lvl;
  if (status != 4) {
    if (S < ad.delta_dec && lvl > 0)
      nl = lvl - 1;
    else if (S > ad.delta_inc && lvl < ad.n_levels - 1)
      nl = lvl + 1;
  }
  return retard_cap(ad, sc, nl);
}

struct DualParams {
  Tables T;
  Mesh mesh;
  Newton nw;
  Adapt ad;
  ClParams cl;
  DualLaunch a;
  StepScalars* sc;
};

template <int CL, int MS>
__global__ void __launch_bounds__(512) k_dual_warp(DualParams P) {
  using Lay = DualLayout<MS>;
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, Q = P.T.Q, QP = P.T.QP;
  double* sPhiT = sm;
  double* sWPhiT = sm + N * QP;
  for (int t = threadIdx.x; t < N * QP; t += blockDim.x) {
    sPhiT[t] = P.T.PhiT[t];
    sWPhiT[t] = P.T.WPhiT[t];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nmax = N * MS;
  double* base = sm + Lay::tables(N, QP) + (size_t)warp * Lay::per_warp(N, Q);
  double* lam = base;
  double* lt = lam + nmax;
  double* uh = lt + nmax;
  double* g = uh + nmax;
  double* dd = g + nmax;
  double* nb = dd + nmax;
  double* H = nb + Q * Lay::NS;

  const double* __restrict__ omega = P.T.omega;
  long long my_iters = 0, my_failed = 0;
  int my_worst = 0;
  double my_rate = 0.0;
  const DualLaunch& A = P.a;

  for (;;) {
    int64_t cell = 0;
    if (lane == 0) cell = atomicAdd(&P.sc->work_counter, 1);
    cell = __shfl_sync(FULL_MASK, cell, 0);
    if (cell >= A.cells) break;
    const int lvl = A.level ? A.level[cell] : 0;
    const int Nl = (P.ad.n_levels > 0) ? P.ad.Nl[lvl] : N;
    const int n = Nl * MS;
    const double* gu = A.uhat + cell * nmax;
    double* gl = A.lam + cell * nmax;
    for (int r = lane; r < n; r += 32) {
      uh[r] = gu[r];
      lam[r] = gl[r];
    }
    __syncwarp();

    int status = 0, l = 0, hv = 0, ia = 0;
    double s1, s2, crit = INFINITY;
    bool nb_is_lam = warp_eval<CL, MS>(lam, Nl, sPhiT, QP, omega, Q, nb, P.cl, s1, s2, lane);
    if (!nb_is_lam) {
      status = 4;  // INADMISSIBLE
    } else {
      crit = warp_grad<MS>(nb, sWPhiT, QP, Q, Nl, uh, g, lane);
      double L0 = s1 - warp_dot(lam, uh, n, lane);
      double scale = s2 + warp_absdot(lam, uh, n, lane);
      for (;;) {
        if (crit < P.nw.tau) break;
        if (P.nw.mode == 1 && l == 1) break;
        if (l == P.nw.max_newton) {
          status = 1;
          break;
        }
        warp_hessian<MS>(nb, sPhiT, sWPhiT, QP, Q, Nl, H, lane);
        if (!warp_chol_solve(H, n, g, dd, lane)) {
          status = 2;
          break;
        }
        const double slope = warp_dot(g, dd, n, lane);
        double alpha = 1.0;
        bool accepted = false;
        for (int h = 0; h <= P.nw.max_halvings; ++h) {
          for (int r = lane; r < n; r += 32) lt[r] = lam[r] + alpha * dd[r];
          __syncwarp();
          double t1, t2;
          const bool okt = warp_eval<CL, MS>(lt, Nl, sPhiT, QP, omega, Q, nb, P.cl, t1, t2, lane);
          nb_is_lam = false;
          if (okt) {
            const double Lt = t1 - warp_dot(lt, uh, n, lane);
            if (Lt <= L0 + P.nw.armijo_c * alpha * slope + 1e-12 * scale) {
              const double sct = t2 + warp_absdot(lt, uh, n, lane);
              crit = warp_grad<MS>(nb, sWPhiT, QP, Q, Nl, uh, g, lane);
              for (int r = lane; r < n; r += 32) lam[r] = lt[r];
              __syncwarp();
              nb_is_lam = true;
              L0 = Lt;
              scale = sct;
              accepted = true;
              break;
            }
          }
          ++hv;
          if (!okt) ++ia;
          alpha *= 0.5;
        }
        if (!accepted) {
          status = 3;
          break;
        }
        ++l;
      }
    }
    // ---- epilogue ------------------------------------------------------------------------------
    if (!nb_is_lam && status != 4) {
      double t1, t2;
      warp_eval<CL, MS>(lam, Nl, sPhiT, QP, omega, Q, nb, P.cl, t1, t2, lane);
    }
    int Nnew = Nl;
    if (P.ad.n_levels > 0 && A.level_new) {
      // S_l on the first state of h = g + uhat at level l (readings 19, 20)
      const int Nprev = lvl > 0 ? P.ad.Nl[lvl - 1] : P.ad.Nprev0;
      double num = 0.0, den = 0.0;
      for (int i = lane; i < Nl; i += 32) {
        const double h = g[i * MS] + uh[i * MS];
        den = fma(h, h, den);
        if (i >= Nprev) num = fma(h, h, num);
      }
      num = warp_sum(num);
      den = warp_sum(den);
      const double S = den > 0.0 ? num / den : 0.0;
      const int nl = next_level(P.ad, P.sc, lvl, status, S);
      Nnew = P.ad.Nl[nl];
      if (lane == 0) A.level_new[cell] = nl;
    }
    // lambda zero-padded / truncated to the new level (the node states keep the old level)
    for (int r = lane; r < nmax; r += 32) gl[r] = (r < n) ? lam[r] : 0.0;  // truncated after the flux
    if (lane == 0) cell_stats(A, P.sc, cell, l, status, hv, ia, crit);
    {  // node states at the final iterate (also for INADMISSIBLE cells: the evaluation at lambda)
      double cr = 0.0;
      for (int k = lane; k < Q; k += 32) {
        const double* u = nb + k * Lay::NS;
        if (A.uq) {
          double* o = A.uq + cell * Q * MS + k;  // [cell][state][node]
#pragma unroll
          for (int a = 0; a < MS; ++a) o[a * Q] = u[a];
        }
        if (A.want_rate) cr = fmax(cr, node_rate<CL, MS>(u, P.mesh, cell, P.cl.gamma));
      }
      my_rate = fmax(my_rate, cr);
    }
    my_iters += l;
    if (status != 0) {
      my_failed += 1;
      my_worst = max(my_worst, status);
    }
    __syncwarp();
  }
  my_rate = warp_max(my_rate);
  if (lane == 0) {
    if (A.want_rate) atomicMax(&P.sc->rate_bits, (unsigned long long)__double_as_longlong(my_rate));
    if (my_iters) atomicAdd(&P.sc->newton_iters, (unsigned long long)my_iters);
    if (my_failed) atomicAdd(&P.sc->failed, (unsigned long long)my_failed);
    if (my_worst) atomicMax(&P.sc->worst, my_worst);
  }
}

#include "ipm_dual_group.cuh"
#include "ipm_dual_mma.cuh"
#include "ipm_dual_big.cuh"
#include "ipm_dual_lbfgs.cuh"

// ------------------------------------------------------------------------------------------------
// flux kernel (variant B: node states from the dual kernel)
// ------------------------------------------------------------------------------------------------
struct FluxParams {
  Tables T;
  Mesh mesh;
  ClParams cl;
  Adapt ad;
  FluxLaunch a;
  StepScalars* sc;
  int tables_in_smem;
  int qchunk;  // k_flux_warp, DMMA projection: nodes per chunk of the per-warp buffer (multiple of 4; 0 = Q)
};

// CH: the node loop in chunks of P.qchunk nodes with the DMMA projection accumulated across chunks (16
// accumulator registers live through the loop: config 5, Q = 1 000); otherwise one pass over the rule and
// the projection tile by tile afterwards (config 4: fewer registers, more CTAs per SM)
// Launch bound: the single-pass instance is built for 3 CTAs per SM (80 registers, no spills; 140
// registers and one CTA per SM otherwise): config 4 flux 2.49 -> 1.25 ms (r02ac_ab_fluxwarp_minb3.txt);
// the chunked instance keeps its registers (80 would spill ~600 bytes).
#ifndef IPM_FLUXW_MINB
#define IPM_FLUXW_MINB 3  // CTAs per SM of the single-pass instance (A/B: 1)
#endif
#ifndef IPM_FLUXW_MINB_CH
#define IPM_FLUXW_MINB_CH 2  // CTAs per SM of the chunked instance (128 registers)
#endif
// FF: the instance with the characteristic far-field branch (reading 37), launched only when a boundary
// tag asks for it: inlined into the common instance it cost config 4 1.22 -> 1.49 ms (r02ao) under the
// 80-register bound
template <int FX, int MS, int MK, bool CH, bool FF = false>
__global__ void __launch_bounds__(256, CH ? IPM_FLUXW_MINB_CH : IPM_FLUXW_MINB) k_flux_warp(FluxParams P) {
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, Q = P.T.Q, QP = P.T.QP;
  // basis table staged in shared memory when it fits (P.tables_in_smem), else read from L2
  // tables_in_smem: 1 omega Phi^T [N][QP] (scalar projection: per-level rules), 2 its A-fragment copy
  // [MT][KS][32] (DMMA projection), 0 neither fits (read from L2)
  const double* sWPhiT = P.tables_in_smem == 1 ? sm : P.T.WPhiT;
  const int tabd = P.tables_in_smem == 1 ? N * QP : (P.tables_in_smem == 2 ? P.T.MT * P.T.KS * 32 : 0);
  if (P.tables_in_smem == 1) {
    for (int t = threadIdx.x; t < N * QP; t += blockDim.x) sm[t] = P.T.WPhiT[t];
    __syncthreads();
  } else if (P.tables_in_smem == 2) {
    for (int t = threadIdx.x; t < tabd; t += blockDim.x) sm[t] = P.T.WPhiF[t];
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  // per-warp buffer of the nodes' residuals (or c-form states): the whole rule, or QB-node chunks that the
  // DMMA projection consumes one after the other (config 5: Q = 1000 nodes, 32 KB per warp otherwise)
  const int QB = (P.tables_in_smem != 1 && P.qchunk > 0 && N <= 64) ? P.qchunk : Q;
  double* q = sm + tabd + (size_t)warp * (QB * MS + 1);
  const int nmax = N * MS;
  const double dt = P.sc->dt;
  const double gam = P.cl.gamma;
  const int F = P.mesh.F;
  const FluxLaunch& A = P.a;
  double my_res = 0.0;
  const int64_t total_warps = (int64_t)gridDim.x * nw;
  // node states of cell c: whole-mesh buffer, or a band of owned cells plus a halo buffer
  auto nodes_of = [&](int64_t c) -> const double* {
    if (A.uq_halo && c >= A.n_owned) return A.uq_halo + (c - A.n_owned) * Q * MS;
    return A.uq + (c - A.uq_base) * Q * MS;
  };
  for (int64_t idx = A.cell0 + (int64_t)blockIdx.x * nw + warp; idx < P.mesh.cells; idx += total_warps) {
    const int64_t cell = A.order ? (int64_t)A.order[idx] : idx;
    // per-level nested rules (reading 36): the update at level l^{n+1} integrates with that level's
    // rule, at its nodes kf of the finest rule (eq. adaptiveFVUpdate)
    const int Lq = (P.ad.lq.on && A.level_new) ? A.level_new[cell] : -1;
    const int Qc = Lq >= 0 ? P.ad.lq.Q[Lq] : Q;
    const int32_t* __restrict__ kfc = Lq >= 0 ? P.ad.lq.kf[Lq] : nullptr;
    const int Nnew = (P.ad.n_levels > 0 && A.level_new) ? P.ad.Nl[A.level_new[cell]] : N;
    const bool mma = Lq < 0 && P.tables_in_smem != 1 && N <= 64;
    const int QBc = (mma && CH) ? QB : Qc;
    // DMMA projection accumulators (row tiles mt < MTl <= 8: N <= 64)
    const int MTl = (Nnew + 7) >> 3, bk = lane & 3, bn = lane >> 2;
    constexpr int NACC = CH ? 8 : 1;
    double acc[NACC][2];
#pragma unroll
    for (int mt = 0; mt < NACC; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    for (int k0 = 0; k0 < Qc; k0 += QBc) {
    const int k1 = min(Qc, k0 + QBc);
    for (int kq = k0 + lane; kq < k1; kq += 32) {
      const int k = kfc ? kfc[kq] : kq;
      double uj[MS], r[MS], gneg[MS];
      const double* src = nodes_of(cell) + k;
#pragma unroll
      for (int a = 0; a < MS; ++a) {
        uj[a] = src[a * Q];
        r[a] = 0.0;
      }
      for (int f = 0; f < F; ++f) {
        const int nbc = P.mesh.nbr[cell * F + f];
        double un[MS];
        double nv[2];
        if (MK == MK_TRI) {
          nv[0] = P.mesh.nrm[(cell * F + f) * 2];
          nv[1] = P.mesh.nrm[(cell * F + f) * 2 + 1];
        } else {
          nv[0] = (f >> 1) == 0 ? 1.0 : 0.0;
          nv[1] = (f >> 1) == 1 ? 1.0 : 0.0;
        }
        if (nbc >= 0) {
          const double* s2 = nodes_of(nbc) + k;
#pragma unroll
          for (int a = 0; a < MS; ++a) un[a] = s2[a * Q];
        } else {
          const int tag = -1 - nbc;
          const int kind = P.mesh.bc_kind[tag];
          if (kind == 1) {
            const double* gs = P.mesh.ghost + ((int64_t)tag * Q + k) * MS;
#pragma unroll
            for (int a = 0; a < MS; ++a) un[a] = gs[a];
          } else if (FF && MS == 4 && kind == 3) {  // characteristic far field (reading 37; triangles only)
            farfield_ghost(gam, uj, P.mesh.ghost + ((int64_t)tag * Q + k) * MS, nv, un);
          } else if (kind == 2 && MS > 1) {
            // slip wall: mirror the normal momentum about the outward normal
            const double sgn = (MK == MK_TRI || (f & 1)) ? 1.0 : -1.0;
            const double on[2] = {nv[0] * sgn, nv[1] * sgn};
            double mn = 0.0;
#pragma unroll
            for (int d = 0; d < MS - 2; ++d) mn += uj[1 + d] * on[d];
            un[0] = uj[0];
#pragma unroll
            for (int d = 0; d < MS - 2; ++d) un[1 + d] = uj[1 + d] - 2.0 * mn * on[d];
            un[MS - 1] = uj[MS - 1];
          } else {
#pragma unroll
            for (int a = 0; a < MS; ++a) un[a] = uj[a];
          }
        }
        const double cf = P.mesh.coef[cell * F + f];
        if (MK == MK_TRI) {
          double gf[MS];
          NumFlux<FX, MS>::g(uj, un, nv, gam, 0.0, gf);
#pragma unroll
          for (int a = 0; a < MS; ++a) r[a] = fma(cf, gf[a], r[a]);
        } else if ((f & 1) == 0) {
          // paper form per direction: (g(u_j, u_{j+1}) - g(u_{j-1}, u_j)) / dx;
          // the difference is formed before scaling so a uniform state gives exactly zero
          NumFlux<FX, MS>::g(un, uj, nv, gam, 1.0 / (cf * dt), gneg);
        } else {
          double gpos[MS];
          NumFlux<FX, MS>::g(uj, un, nv, gam, 1.0 / (cf * dt), gpos);
#pragma unroll
          for (int a = 0; a < MS; ++a) r[a] += (gpos[a] - gneg[a]) * cf;
        }
      }
      double* qk = q + (kq - k0) * MS;
      if (A.update_form == 1) {
#pragma unroll
        for (int a = 0; a < MS; ++a) qk[a] = uj[a] - dt * r[a];
      } else {
#pragma unroll
        for (int a = 0; a < MS; ++a) qk[a] = r[a];
      }
    }
    __syncwarp();
    if (mma && CH) {
      // projection Phi^T (omega o q) on the fp64 tensor path, this chunk's k-steps: C[i][a] += sum_k
      // (omega phi_i)(xi_k) q_a(xi_k), A = omega Phi^T in A-fragment order (shared memory when it fits,
      // else L2), B = the chunk's q rows
      const double* __restrict__ sWF = P.tables_in_smem == 2 ? sm : P.T.WPhiF;
      const int KS = P.T.KS;
      const bool bval = bn < MS;
      for (int ks = k0 >> 2; ks < (k1 + 3) >> 2; ++ks) {
        const int k = 4 * ks + bk;
        const double bv = (bval && k < k1) ? q[(k - k0) * MS + bn] : 0.0;
        const double* asrc = sWF + (size_t)ks * 32 + lane;
#pragma unroll
        for (int mt = 0; mt < NACC; ++mt)
          if (mt < MTl) dmma884(acc[mt][0], acc[mt][1], asrc[(size_t)mt * KS * 32], bv);
      }
      __syncwarp();
    }
    }  // node chunks
    const double* uo = A.uhat_old + cell * nmax;
    double* un_ = A.uhat_new + cell * nmax;
    if (mma) {
      const double* __restrict__ sWF = P.tables_in_smem == 2 ? sm : P.T.WPhiF;
      const int KS = P.T.KS;
#pragma unroll 1
      for (int mt = 0; mt < (CH ? 8 : MTl); ++mt) {
        if (mt >= MTl) break;
        double c0, c1;
        if constexpr (CH) {
          c0 = acc[mt < NACC ? mt : 0][0];
          c1 = acc[mt < NACC ? mt : 0][1];
        } else {  // one pass over the whole rule (q holds every node)
          c0 = c1 = 0.0;
          const double* asrc = sWF + (size_t)mt * KS * 32 + lane;
#pragma unroll 4
          for (int ks = 0; ks < KS; ++ks) {
            const int k = 4 * ks + bk;
            const double bv = (bn < MS && k < Qc) ? q[k * MS + bn] : 0.0;
            dmma884(c0, c1, asrc[(size_t)ks * 32], bv);
          }
        }
        const int i = 8 * mt + (lane >> 2);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int a = 2 * (lane & 3) + e;
          if (a < MS && i < Nnew) {
            const int rr = i * MS + a;
            const double old = uo[rr];
            const double sres = e == 0 ? c0 : c1;
            const double out = (A.update_form == 1) ? sres : old - dt * sres;
            un_[rr] = out;
            if (rr == 0) my_res += P.mesh.area[cell] * fabs(out - old);
          }
        }
      }
      for (int rr = Nnew * MS + lane; rr < nmax; rr += 32) {
        un_[rr] = 0.0;
        if (A.lam) A.lam[cell * nmax + rr] = 0.0;  // duals truncated to the new level (Alg. 3)
      }
      __syncwarp();
      continue;
    }
    for (int rr = lane; rr < nmax; rr += 32) {
      const int i = rr / MS, a = rr - i * MS;
      const double old = uo[rr];  // uhat_new may alias uhat_old (only this cell's entries are read)
      double out = 0.0;
      if (i < Nnew) {
        const double* wp = Lq >= 0 ? P.ad.lq.wphit[Lq] + i * P.ad.lq.QP[Lq] : sWPhiT + i * QP;
        double s = 0.0;
        for (int k = 0; k < Qc; ++k) s = fma(wp[k], q[k * MS + a], s);
        out = (A.update_form == 1) ? s : old - dt * s;
      }
      un_[rr] = out;
      if (rr == 0) my_res += P.mesh.area[cell] * fabs(out - old);
      // duals zero-padded / truncated to the new level (Alg. 3: next dual solve at l^{n+1})
      if (A.lam && i >= Nnew) A.lam[cell * nmax + rr] = 0.0;
    }
    __syncwarp();
  }
  my_res = warp_sum(my_res);
  if (lane == 0 && my_res != 0.0) atomicAdd(&P.sc->residual, my_res);
}

// ------------------------------------------------------------------------------------------------
// Stochastic Collocation (reading 32): the deterministic
// finite-volume scheme with the same numerical flux at every quadrature node, all nodes advancing
// with one CFL step. Node states [cells][m][Q] (the flux kernels' layout); warp per cell, lanes over
// nodes; the residual is the change of the mean, sum_j |Omega_j| |sum_k w_k (u^{n+1} - u^n)_0|.
// ------------------------------------------------------------------------------------------------
template <int MS>
__global__ void k_sc_rate(int64_t cells, int Q, Mesh mesh, double gamma, const double* __restrict__ U,
                          StepScalars* sc) {
  double my = 0.0;
  const int64_t n = cells * Q;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = t / Q;
    const int k = (int)(t - cell * Q);
    double u[MS];
#pragma unroll
    for (int a = 0; a < MS; ++a) u[a] = U[cell * Q * MS + a * Q + k];
    my = fmax(my, node_rate<0, MS>(u, mesh, cell, gamma));
  }
  my = warp_max(my);
  if ((threadIdx.x & 31) == 0 && my > 0.0) atomicMax(&sc->rate_bits, (unsigned long long)__double_as_longlong(my));
}

template <int FX, int MS, int MK>
__global__ void __launch_bounds__(256) k_sc_update(FluxParams P, const double* __restrict__ Uin,
                                                   double* __restrict__ Uout) {
  const int Q = P.T.Q;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double dt = P.sc->dt, gam = P.cl.gamma;
  const int F = P.mesh.F;
  double my_res = 0.0, my_rate = 0.0;
  for (int64_t cell = (int64_t)blockIdx.x * nw + warp; cell < P.mesh.cells; cell += (int64_t)gridDim.x * nw) {
    double dmean = 0.0;
    for (int k = lane; k < Q; k += 32) {
      double uj[MS], r[MS], gneg[MS];
      const double* src = Uin + cell * Q * MS + k;
#pragma unroll
      for (int a = 0; a < MS; ++a) {
        uj[a] = src[a * Q];
        r[a] = 0.0;
      }
      for (int f = 0; f < F; ++f) {
        const int nbc = P.mesh.nbr[cell * F + f];
        double un[MS], nv[2];
        if (MK == MK_TRI) {
          nv[0] = P.mesh.nrm[(cell * F + f) * 2];
          nv[1] = P.mesh.nrm[(cell * F + f) * 2 + 1];
        } else {
          nv[0] = (f >> 1) == 0 ? 1.0 : 0.0;
          nv[1] = (f >> 1) == 1 ? 1.0 : 0.0;
        }
        if (nbc >= 0) {
          const double* s2 = Uin + (int64_t)nbc * Q * MS + k;
#pragma unroll
          for (int a = 0; a < MS; ++a) un[a] = s2[a * Q];
        } else {
          const int tag = -1 - nbc;
          const int kind = P.mesh.bc_kind[tag];
          if (kind == 1) {
            const double* gs = P.mesh.ghost + ((int64_t)tag * Q + k) * MS;
#pragma unroll
            for (int a = 0; a < MS; ++a) un[a] = gs[a];
          } else if (MS == 4 && kind == 3) {  // characteristic far field (reading 37; triangles only)
            farfield_ghost(gam, uj, P.mesh.ghost + ((int64_t)tag * Q + k) * MS, nv, un);
          } else if (kind == 2 && MS > 1) {  // slip wall: mirror the normal momentum
            const double sgn = (MK == MK_TRI || (f & 1)) ? 1.0 : -1.0;
            const double on[2] = {nv[0] * sgn, nv[1] * sgn};
            double mn = 0.0;
#pragma unroll
            for (int d = 0; d < MS - 2; ++d) mn += uj[1 + d] * on[d];
            un[0] = uj[0];
#pragma unroll
            for (int d = 0; d < MS - 2; ++d) un[1 + d] = uj[1 + d] - 2.0 * mn * on[d];
            un[MS - 1] = uj[MS - 1];
          } else {
#pragma unroll
            for (int a = 0; a < MS; ++a) un[a] = uj[a];
          }
        }
        const double cf = P.mesh.coef[cell * F + f];
        if (MK == MK_TRI) {
          double gf[MS];
          NumFlux<FX, MS>::g(uj, un, nv, gam, 0.0, gf);
#pragma unroll
          for (int a = 0; a < MS; ++a) r[a] = fma(cf, gf[a], r[a]);
        } else if ((f & 1) == 0) {
          NumFlux<FX, MS>::g(un, uj, nv, gam, 1.0 / (cf * dt), gneg);
        } else {
          double gpos[MS];
          NumFlux<FX, MS>::g(uj, un, nv, gam, 1.0 / (cf * dt), gpos);
#pragma unroll
          for (int a = 0; a < MS; ++a) r[a] += (gpos[a] - gneg[a]) * cf;
        }
      }
      double* dst = Uout + cell * Q * MS + k;
      double u0n = 0.0;
#pragma unroll
      for (int a = 0; a < MS; ++a) {
        const double v = uj[a] - dt * r[a];
        dst[a * Q] = v;
        if (a == 0) u0n = v;
      }
      dmean = fma(P.T.omega[k], u0n - uj[0], dmean);
      {  // CFL rate of the new state, for the next step (ipm_sc_step reuses it when it gets this output)
        double v[MS];
#pragma unroll
        for (int a = 0; a < MS; ++a) v[a] = dst[a * Q];
        my_rate = fmax(my_rate, node_rate<0, MS>(v, P.mesh, cell, gam));
      }
    }
    dmean = warp_sum(dmean);
    if (lane == 0) my_res += P.mesh.area[cell] * fabs(dmean);
  }
  if (lane == 0 && my_res != 0.0) atomicAdd(&P.sc->residual, my_res);
  my_rate = warp_max(my_rate);
  if (lane == 0 && my_rate > 0.0)
    atomicMax(&P.sc->sc_rate_next, (unsigned long long)__double_as_longlong(my_rate));
}

// SC step begin: the rate starts at the ghost states' rate, maxed with the cached rate of the input
// (the previous step's output) when the host knows it is valid
__global__ void k_sc_begin(StepScalars* sc, double rate0, int use_cached) {
  unsigned long long r = (unsigned long long)__double_as_longlong(rate0);
  if (use_cached && sc->sc_rate_next > r) r = sc->sc_rate_next;
  sc->rate_bits = r;
  sc->sc_rate_next = 0ull;
  sc->residual = 0.0;
  sc->newton_iters = 0;
  sc->failed = 0;
  sc->worst = 0;
}

// ------------------------------------------------------------------------------------------------
// flux kernel for 1D / cartesian meshes: CPW = 8/m cells per warp so that the projection
// Phi^T(omega o r) of all of them is one set of DMMAs (columns = (cell, state) pairs):
//   flux    lanes over (cell, node): the node's physical flux along each direction is formed once
//           (Rusanov) and combined with the neighbours' at the two faces of that direction, in the
//           paper's difference form (g(u_j, u_{j+1}) - g(u_{j-1}, u_j)) / dx;
//   project C[i][(c,a)] = sum_k (omega phi_i)(xi_k) r_k[(c,a)], A = WPhiF (fragment order, shared
//           memory), B = r staged per warp;  the update uhat^{n+1} = uhat^n - dt C (CONSERVATIVE) or
//           Phi^T(omega o (u - dt r)) (c-form).
// ------------------------------------------------------------------------------------------------
// Rusanov flux ingredients of one node state along coordinate direction dir (Euler, m = d + 2)
template <int MS>
struct RusNode {
  static constexpr int D = MS - 2;
  double irho, p, c;
  __device__ void init(const double* u, double gamma) {
    irho = rcp_nr(u[0]);
    double m2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) m2 = fma(u[1 + k], u[1 + k], m2);
    p = (gamma - 1.0) * (u[MS - 1] - 0.5 * m2 * irho);
    c = sqrt_nr(gamma * p * irho);
  }
  // F_dir(u) and |v_dir| + c
  __device__ void flux(const double* u, int dir, double* f, double& s) const {
    const double vn = u[1 + dir] * irho;
    f[0] = u[1 + dir];
#pragma unroll
    for (int k = 0; k < D; ++k) f[1 + k] = (k == dir) ? fma(u[1 + k], vn, p) : u[1 + k] * vn;
    f[MS - 1] = (u[MS - 1] + p) * vn;
    s = fabs(vn) + c;
  }
};

template <int FX, int MS, int MK>
#ifndef IPM_FLUX_MINB
#define IPM_FLUX_MINB 2  // measured: 3 blocks per SM (80 registers, spills) is 14 % slower
#endif
__global__ void __launch_bounds__(256, IPM_FLUX_MINB) k_flux_cart(FluxParams P) {
  constexpr int CPW = 8 / MS;              // cells per warp (DMMA columns = CPW * MS <= 8)
  constexpr int F = (MK == MK_CART) ? 4 : 2;
  constexpr int ND = F / 2;                // directions
  constexpr bool FAST = (FX == FX_RUSANOV && MS >= 3);
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, Q = P.T.Q, MT = P.T.MT, KS = P.T.KS;
  double* sA = sm;  // [MT][KS][32]
  for (int x = threadIdx.x; x < MT * KS * 32; x += blockDim.x) sA[x] = P.T.WPhiF[x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* rb = sm + MT * KS * 32 + (size_t)warp * KS * 32;  // [KS*4][8]: rows k >= Q and unused columns stay 0
  for (int x = lane; x < KS * 32; x += 32) rb[x] = 0.0;
  __syncthreads();
  const int nmax = N * MS;
  const double dt = P.sc->dt;
  const double gam = P.cl.gamma;
  const FluxLaunch& A = P.a;
  const int64_t cells = P.mesh.cells;
  double my_res = 0.0;
  const int64_t groups = (cells + CPW - 1) / CPW;
  for (int64_t grp = (int64_t)blockIdx.x * nw + warp; grp < groups; grp += (int64_t)gridDim.x * nw) {
    const int64_t cell0 = grp * CPW;
    // ---- a11: kinetic flux at every node of every face ------------------------------------------
    for (int it = lane; it < CPW * Q; it += 32) {
      const int c = it / Q, k = it - c * Q;
      const int64_t cell = cell0 + c;
      if (cell >= cells) continue;
      double uj[MS], r[MS];
      const double* src = A.uq + cell * Q * MS + k;
#pragma unroll
      for (int a = 0; a < MS; ++a) {
        uj[a] = src[a * Q];
        r[a] = 0.0;
      }
      // all neighbour node states first: their loads are independent and overlap
      double un[F][MS];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int nbc = P.mesh.nbr[cell * F + f];
        if (nbc >= 0) {
          const double* s2 = A.uq + (int64_t)nbc * Q * MS + k;
#pragma unroll
          for (int a = 0; a < MS; ++a) un[f][a] = s2[a * Q];
        } else {
          const int tag = -1 - nbc;
          const int kind = P.mesh.bc_kind[tag];
          if (kind == 1) {
            const double* gs = P.mesh.ghost + ((int64_t)tag * Q + k) * MS;
#pragma unroll
            for (int a = 0; a < MS; ++a) un[f][a] = gs[a];
          } else if (kind == 2 && MS > 1) {
            // slip wall: mirror the normal momentum
#pragma unroll
            for (int a = 0; a < MS; ++a) un[f][a] = uj[a];
            un[f][1 + f / 2] = -uj[1 + f / 2];
          } else {
#pragma unroll
            for (int a = 0; a < MS; ++a) un[f][a] = uj[a];
          }
        }
      }
      RusNode<MS> nj;
      if constexpr (FAST) nj.init(uj, gam);
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        double fj[MS], sj = 0.0, gneg[MS];
        if constexpr (FAST) nj.flux(uj, d, fj, sj);
#pragma unroll
        for (int side = 0; side < 2; ++side) {
          const int f = 2 * d + side;
          const double cf = P.mesh.coef[cell * F + f];
          double gf[MS];
          if constexpr (FAST) {
            RusNode<MS> nn;
            nn.init(un[f], gam);
            double fn[MS], sn;
            nn.flux(un[f], d, fn, sn);
            const double amax = fmax(side == 0 ? sn : sj, side == 0 ? sj : sn);
            // g(uL, uR) = (F(uL) + F(uR))/2 - a (uR - uL)/2, uL = west/south state
#pragma unroll
            for (int a = 0; a < MS; ++a) {
              const double fl = side == 0 ? fn[a] : fj[a], fr = side == 0 ? fj[a] : fn[a];
              const double ul = side == 0 ? un[f][a] : uj[a], ur = side == 0 ? uj[a] : un[f][a];
              gf[a] = 0.5 * (fl + fr) - 0.5 * amax * (ur - ul);
            }
          } else {
            double nv[2] = {d == 0 ? 1.0 : 0.0, d == 1 ? 1.0 : 0.0};
            if (side == 0)
              NumFlux<FX, MS>::g(un[f], uj, nv, gam, 1.0 / (cf * dt), gf);
            else
              NumFlux<FX, MS>::g(uj, un[f], nv, gam, 1.0 / (cf * dt), gf);
          }
          if (side == 0) {
#pragma unroll
            for (int a = 0; a < MS; ++a) gneg[a] = gf[a];
          } else {
#pragma unroll
            for (int a = 0; a < MS; ++a) r[a] += (gf[a] - gneg[a]) * cf;
          }
        }
      }
      double* o = rb + k * 8 + c * MS;
      if (A.update_form == 1) {
#pragma unroll
        for (int a = 0; a < MS; ++a) o[a] = uj[a] - dt * r[a];
      } else {
#pragma unroll
        for (int a = 0; a < MS; ++a) o[a] = r[a];
      }
    }
    __syncwarp();
    // ---- projection on the fp64 tensor path and the update ---------------------------------------
    const int rr = lane >> 2, q = lane & 3;
    for (int mt = 0; mt < MT; ++mt) {
      double c0 = 0.0, c1 = 0.0;
      const double* a = sA + (size_t)mt * KS * 32 + lane;
      const double* b = rb + (lane & 3) * 8 + (lane >> 2);
#pragma unroll 5
      for (int ks = 0; ks < KS; ++ks) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0), "+d"(c1)
                     : "d"(a[ks * 32]), "d"(b[ks * 32]));
      }
      const int i = 8 * mt + rr;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 2 * q + e, c = col / MS, av = col - c * MS;
        const int64_t cell = cell0 + c;
        if (col >= CPW * MS || i >= N || cell >= cells) continue;
        const int Nnew = (P.ad.n_levels > 0 && A.level_new) ? P.ad.Nl[A.level_new[cell]] : N;
        const int64_t idx = cell * nmax + i * MS + av;
        const double old = A.uhat_old[idx];
        double out = 0.0;
        if (i < Nnew) out = (A.update_form == 1) ? (e == 0 ? c0 : c1) : old - dt * (e == 0 ? c0 : c1);
        A.uhat_new[idx] = out;
        if (i == 0 && av == 0) my_res += P.mesh.area[cell] * fabs(out - old);
        if (A.lam && i >= Nnew) A.lam[idx] = 0.0;
      }
    }
    __syncwarp();
  }
  my_res = warp_sum(my_res);
  if (lane == 0 && my_res != 0.0) atomicAdd(&P.sc->residual, my_res);
}

#include "ipm_flux_strip.cuh"

// ------------------------------------------------------------------------------------------------
// small kernels
// ------------------------------------------------------------------------------------------------
__global__ void k_step_begin(StepScalars* sc, double rate0) {
  sc->rate_bits = (unsigned long long)__double_as_longlong(rate0);
  sc->residual = 0.0;
  sc->newton_iters = 0;
  sc->failed = 0;
  sc->worst = 0;
  sc->work_counter = 0;
  sc->work_counter2 = 0;
  for (int i = 0; i < kHistBuckets; ++i) sc->hist[i] = 0;
  sc->halvings = 0;
  sc->inadm_trials = 0;
}

// Algorithm 4 lines 12-14: next retardation stage once the step's residual is below its tolerance
__global__ void k_retard(StepScalars* sc, Adapt ad) {
  if (sc->stage < ad.n_retard && sc->residual < ad.retard_eps[sc->stage]) sc->stage += 1;
}

// dt = min(cfl / rate, t_end - t) (t_end <= 0: no cap), then t += dt
__global__ void k_dt(StepScalars* sc, double t_end, double dt_fixed, double cfl) {
  double dt;
  if (dt_fixed > 0.0) {
    dt = dt_fixed;
  } else {
    const double rate = __longlong_as_double((long long)sc->rate_bits);
    dt = cfl / rate;
    if (t_end > 0.0) dt = fmin(dt, t_end - sc->t);
  }
  sc->dt = dt;
  sc->t = sc->t + dt;
}

// IC projection: uhat_j = sum_k omega_k phi(xi_k) ubar_j(xi_k), exact cell averages of a
// piecewise-constant IC at each node (Alg. 1 line 2; reading 17)
template <int MS>
__global__ void k_project_ic(Tables T, int64_t cells, const double* __restrict__ region,
                             const double* __restrict__ split, int kind, int nx, double x0, double y0, double dx,
                             double dy, const int32_t* __restrict__ level, const int64_t* __restrict__ gid, Adapt ad,
                             double* __restrict__ uhat, double* __restrict__ unodes) {
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int Q = T.Q, N = T.N;
  double* q = sm + warp * (Q * MS + 1);
  for (int64_t cell = (int64_t)blockIdx.x * nw + warp; cell < cells; cell += (int64_t)gridDim.x * nw) {
    for (int k = lane; k < Q; k += 32) {
      double ub[MS];
      if (kind == 0) {
#pragma unroll
        for (int a = 0; a < MS; ++a) ub[a] = region[(0 * Q + k) * MS + a];
      } else if (kind == 1) {
        const double xl = x0 + (double)gid[cell] * dx;
        double fl = (split[k * 2] - xl) / dx;
        fl = fmin(fmax(fl, 0.0), 1.0);
#pragma unroll
        for (int a = 0; a < MS; ++a)
          ub[a] = fl * region[(0 * Q + k) * MS + a] + (1.0 - fl) * region[(1 * Q + k) * MS + a];
      } else {
        const int64_t ix = gid[cell] % nx, iy = gid[cell] / nx;
        double fx = (split[k * 2] - (x0 + ix * dx)) / dx;
        double fy = (split[k * 2 + 1] - (y0 + iy * dy)) / dy;
        fx = fmin(fmax(fx, 0.0), 1.0);
        fy = fmin(fmax(fy, 0.0), 1.0);
        const double w0 = (1.0 - fx) * (1.0 - fy), w1 = fx * (1.0 - fy), w2 = fx * fy, w3 = (1.0 - fx) * fy;
#pragma unroll
        for (int a = 0; a < MS; ++a)
          ub[a] = w0 * region[(0 * Q + k) * MS + a] + w1 * region[(1 * Q + k) * MS + a] +
                  w2 * region[(2 * Q + k) * MS + a] + w3 * region[(3 * Q + k) * MS + a];
      }
#pragma unroll
      for (int a = 0; a < MS; ++a) q[k * MS + a] = ub[a];
      if (unodes) {  // Stochastic Collocation: the node states themselves, [cell][state][node]
#pragma unroll
        for (int a = 0; a < MS; ++a) unodes[cell * Q * MS + a * Q + k] = ub[a];
      }
    }
    __syncwarp();
    if (!uhat) continue;
    const int Nl = (ad.n_levels > 0 && level) ? ad.Nl[level[cell]] : N;
    const int Lq = (ad.lq.on && level) ? level[cell] : -1;  // Alg. 3 line 3: the initial level's rule
    for (int r = lane; r < N * MS; r += 32) {
      const int i = r / MS, a = r - i * MS;
      double s = 0.0;
      if (i < Nl) {
        if (Lq >= 0) {
          const double* wp = ad.lq.wphit[Lq] + i * ad.lq.QP[Lq];
          const int32_t* kf = ad.lq.kf[Lq];
          for (int kq = 0; kq < ad.lq.Q[Lq]; ++kq) s = fma(wp[kq], q[kf[kq] * MS + a], s);
        } else {
          for (int k = 0; k < Q; ++k) s = fma(T.WPhiT[i * T.QP + k], q[k * MS + a], s);
        }
      }
      uhat[cell * N * MS + r] = s;
    }
    __syncwarp();
  }
}

template <int CL, int MS>
__global__ void k_warm_start(int64_t cells, int N, ClParams cp, const double* __restrict__ uhat,
                             double* __restrict__ lam, StepScalars* sc) {
  const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= cells) return;
  double u[MS], L[MS];
#pragma unroll
  for (int a = 0; a < MS; ++a) u[a] = uhat[cell * N * MS + a];
  const bool ok = Closure<CL, MS>::grad_s(u, L, cp);
  if (!ok) atomicMax(&sc->worst, 4);
  for (int r = 0; r < N * MS; ++r) lam[cell * N * MS + r] = (r < MS) ? (ok ? L[r] : NAN) : 0.0;
}

// node pass for given duals (warp per cell): optional uhat = h(lambda), node states
// u_s(lambda^T phi(xi_k)) and CFL rate
template <int CL, int MS>
__global__ void k_nodes(Tables T, Mesh mesh, ClParams cp, const double* __restrict__ lam_g, double* __restrict__ uhat,
                        double* __restrict__ uq, StepScalars* sc, int tables_in_smem, int want_rate) {
  using Lay = DualLayout<MS>;
  extern __shared__ __align__(16) double sm[];
  const int N = T.N, Q = T.Q, QP = T.QP;
  const double* sPhiT = tables_in_smem ? sm : T.PhiT;
  const double* sWPhiT = tables_in_smem ? sm + N * QP : T.WPhiT;
  if (tables_in_smem) {
    for (int t = threadIdx.x; t < N * QP; t += blockDim.x) {
      sm[t] = T.PhiT[t];
      sm[N * QP + t] = T.WPhiT[t];
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* lam = sm + (tables_in_smem ? 2 * N * QP : 0) + (size_t)warp * (N * MS + Q * Lay::NS + 1);
  double* nb = lam + N * MS;
  double my_rate = 0.0;
  int bad = 0;
  for (int64_t cell = (int64_t)blockIdx.x * nw + warp; cell < mesh.cells; cell += (int64_t)gridDim.x * nw) {
    for (int r = lane; r < N * MS; r += 32) lam[r] = lam_g[cell * N * MS + r];
    __syncwarp();
    double s1, s2;
    if (!warp_eval<CL, MS>(lam, N, sPhiT, QP, T.omega, Q, nb, cp, s1, s2, lane)) bad = 1;
    if (uhat) {
      double* out = uhat + cell * N * MS;
      for (int r = lane; r < N * MS; r += 32) {
        const int i = r / MS, a = r - i * MS;
        double s = 0.0;
        for (int k = 0; k < Q; ++k) s = fma(sWPhiT[i * QP + k], nb[k * Lay::NS + a], s);
        out[r] = s;
      }
    }
    for (int k = lane; k < Q; k += 32) {
      const double* u = nb + k * Lay::NS;
      if (uq) {
        double* o = uq + cell * Q * MS + k;  // [cell][state][node]
#pragma unroll
        for (int a = 0; a < MS; ++a) o[a * Q] = u[a];
      }
      if (want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(u, mesh, cell, cp.gamma));
    }
    __syncwarp();
  }
  my_rate = warp_max(my_rate);
  if (lane == 0 && sc) {
    if (want_rate) atomicMax(&sc->rate_bits, (unsigned long long)__double_as_longlong(my_rate));
    if (bad) atomicMax(&sc->worst, 4);
  }
}

// node states only (no h(lambda)): u_s(Phi lambda) of C cells per warp written straight to uq
// [cell][state][node] — no per-warp node buffer (config 5: Q (m + m(m+1)/2) doubles = 120 KB per warp
// left k_nodes one warp per SM), each basis value read once for the C cells.  Same fma order over i as
// the dual kernels' node pass, so the states are bit-identical to the ones they write.
template <int CL, int MS, int C>
__global__ void __launch_bounds__(256) k_nodes_out(Tables T, Mesh mesh, ClParams cp, const double* __restrict__ lam_g,
                                                   double* __restrict__ uq, StepScalars* sc, int tables_in_smem,
                                                   int want_rate) {
  extern __shared__ __align__(16) double sm[];
  const int N = T.N, Q = T.Q, QP = T.QP, n = N * MS;
  const double* sPhiT = tables_in_smem ? sm : T.PhiT;
  if (tables_in_smem) {
    for (int t = threadIdx.x; t < N * QP; t += blockDim.x) sm[t] = T.PhiT[t];
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* lam = sm + (tables_in_smem ? N * QP : 0) + (size_t)warp * (C * n);
  double my_rate = 0.0;
  int bad = 0;
  for (int64_t c0 = ((int64_t)blockIdx.x * nw + warp) * C; c0 < mesh.cells; c0 += (int64_t)gridDim.x * nw * C) {
    const int nc = (int)min((int64_t)C, mesh.cells - c0);
    for (int r = lane; r < C * n; r += 32) lam[r] = (r < nc * n) ? lam_g[c0 * n + r] : 0.0;
    __syncwarp();
    for (int k = lane; k < Q; k += 32) {
      double Lam[C][MS];
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int a = 0; a < MS; ++a) Lam[c][a] = 0.0;
#pragma unroll 2
      for (int i = 0; i < N; ++i) {
        const double ph = sPhiT[(size_t)i * QP + k];
#pragma unroll
        for (int c = 0; c < C; ++c)
#pragma unroll
          for (int a = 0; a < MS; ++a) Lam[c][a] = fma(lam[c * n + i * MS + a], ph, Lam[c][a]);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (c < nc) {
          double u[MS], J[MS * (MS + 1) / 2], ss;
          if (!Closure<CL, MS>::eval(Lam[c], u, J, ss, cp)) bad = 1;
          double* o = uq + (c0 + c) * Q * MS + k;
#pragma unroll
          for (int a = 0; a < MS; ++a) o[a * Q] = u[a];
          if (want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(u, mesh, c0 + c, cp.gamma));
        }
      }
    }
    __syncwarp();
  }
  my_rate = warp_max(my_rate);
  if (lane == 0 && sc) {
    if (want_rate) atomicMax(&sc->rate_bits, (unsigned long long)__double_as_longlong(my_rate));
    if (bad) atomicMax(&sc->worst, 4);
  }
}

// stress duals: lambda_0 = grad s(base); higher (rel|l0| + abs) 2^-|i| z; Euler: scale
// higher modes so that max_k sum_{i>=1} lambda_{i,E} phi_i(xi_k) <= |lambda_{0,E}|/2
template <int CL, int MS>
__global__ void k_stress(Tables T, int64_t cells, ClParams cp, const double* __restrict__ basev,
                         const double* __restrict__ z, double rel, double abs_, double* __restrict__ lam) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int N = T.N, Q = T.Q;
  for (int64_t cell = (int64_t)blockIdx.x * nw + warp; cell < cells; cell += (int64_t)gridDim.x * nw) {
    double u[MS], L0[MS];
#pragma unroll
    for (int a = 0; a < MS; ++a) u[a] = basev[cell * MS + a];
    Closure<CL, MS>::grad_s(u, L0, cp);
    double* out = lam + cell * N * MS;
    for (int r = lane; r < N * MS; r += 32) {
      const int i = r / MS, a = r - i * MS;
      double v;
      if (i == 0) {
        v = L0[a];
      } else {
        double amp = 0.0;
#pragma unroll
        for (int b = 0; b < MS; ++b)
          if (b == a) amp = rel * fabs(L0[b]) + abs_;
        v = amp * exp2(-(double)T.deg[i]) * z[cell * N * MS + r];
      }
      out[r] = v;
    }
    __syncwarp();
    if (CL == CL_EULER) {
      double mx = -INFINITY;
      for (int k = lane; k < Q; k += 32) {
        double s = 0.0;
        for (int i = 1; i < N; ++i) s = fma(T.PhiT[i * T.QP + k], out[i * MS + MS - 1], s);
        mx = fmax(mx, s);
      }
      mx = warp_max(mx);
      const double lim = 0.5 * fabs(L0[MS - 1]);
      if (mx > lim) {
        const double f = lim / mx;
        for (int r = MS + lane; r < N * MS; r += 32) out[r] *= f;
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------------------------------------
// launchers and dispatch
// ------------------------------------------------------------------------------------------------
static inline cudaStream_t S(const KernelCtx& k) { return (cudaStream_t)k.stream; }

// Launch configuration, cached on the host: the dynamic shared-memory attribute is raised only when a
// launch needs more than the kernel has on this device, and the occupancy query runs once per
// (kernel, device, block size, shared memory) — not on every launch (host-side cost on the small,
// launch-bound configurations).  Contexts are single-threaded (ipm.h), so is this cache.
struct LaunchCfgEntry {
  const void* f;
  int dev, threads;
  size_t smem;
  int per_sm;
};
template <class K>
static int configure(K kern, int threads, size_t smem) {
  static std::vector<LaunchCfgEntry> occ;
  static std::vector<LaunchCfgEntry> attr;  // per (kernel, device): largest smem attribute set
  int dev = 0;
  cudaGetDevice(&dev);
  const void* f = (const void*)kern;
  bool have = false;
  for (auto& e : attr)
    if (e.f == f && e.dev == dev) {
      if (smem > e.smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e.smem = smem;
      }
      have = true;
    }
  if (!have) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr.push_back({f, dev, 0, smem, 0});
  }
  if (threads <= 0) return 1;
  for (const auto& e : occ)
    if (e.f == f && e.dev == dev && e.threads == threads && e.smem == smem) return e.per_sm;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  occ.push_back({f, dev, threads, smem, per_sm});
  return per_sm;
}


int debug_phase_cycles(unsigned long long* out) {
#ifdef IPM_PHASE_TIMERS
  cudaError_t e = cudaMemcpyFromSymbol(out, g_phase_cycles, 8 * sizeof(unsigned long long));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  return (int)e;
#else
  for (int i = 0; i < 8; ++i) out[i] = 0;
  return 0;
#endif
}

int launch_sc_begin(const KernelCtx& k, double rate0, int use_cached) {
  k_sc_begin<<<1, 1, 0, S(k)>>>(k.sc, rate0, use_cached);
  return (int)cudaGetLastError();
}

int launch_step_begin(const KernelCtx& k, double rate0) {
  k_step_begin<<<1, 1, 0, S(k)>>>(k.sc, rate0);
  return (int)cudaGetLastError();
}

int launch_dt(const KernelCtx& k, double t_end, double dt_fixed, double cfl) {
  k_dt<<<1, 1, 0, S(k)>>>(k.sc, t_end, dt_fixed, cfl);
  return (int)cudaGetLastError();
}

template <int CL, int MS>
static int dual_impl(const KernelCtx& k, const DualLaunch& a) {
  using Lay = DualLayout<MS>;
  const size_t tab = (size_t)Lay::tables(k.T.N, k.T.QP) * 8, pw = (size_t)Lay::per_warp(k.T.N, k.T.Q) * 8;
  if (tab + pw > k.smem_optin) return -1;
  int warps = (int)((k.smem_optin - tab) / pw);
  warps = warps > 16 ? 16 : warps;
  const size_t smem = tab + warps * pw;
  auto kern = k_dual_warp<CL, MS>;
  int per_sm = configure(kern, warps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t want = (a.cells + warps - 1) / warps;
  int grid = (int)std::min<int64_t>(want, (int64_t)k.sm_count * per_sm);
  if (grid < 1) grid = 1;
  DualParams P{k.T, k.mesh, k.nw, k.ad, k.cl, a, k.sc};
  kern<<<grid, warps * 32, smem, S(k)>>>(P);
  return (int)cudaGetLastError();
}

template <int CL, int MS, int G, int SF, int T>
static int dual_group_impl(const KernelCtx& k, const DualLaunch& a) {
  using Lay = GroupLayout<MS>;
  const int npr = SF * (SF + 1) / 2;
  const size_t tab = ((size_t)2 * k.T.N * k.T.QP + (SF > 0 ? ((k.T.q1d * npr + 1) & ~1) : 0)) * 8;
  const size_t pg = (size_t)Lay::per_group(k.T.N, k.T.Q, G, SF, k.T.q1d) * 8;
  if (tab + pg > k.smem_optin) return -1;
  int groups = (int)((k.smem_optin - tab) / pg);
  groups = std::min(groups, IPM_GROUP_THREADS / G);
  const size_t smem = tab + groups * pg;
  auto kern = k_dual_group<CL, MS, G, SF, T>;
  int per_sm = configure(kern, groups * G, smem);
  if (per_sm < 1) return -1;
  const int64_t want = (a.cells + groups - 1) / groups;
  int grid = (int)std::min<int64_t>(want, (int64_t)k.sm_count * per_sm);
  if (grid < 1) grid = 1;
  DualParams P{k.T, k.mesh, k.nw, k.ad, k.cl, a, k.sc};
  kern<<<grid, groups * G, smem, S(k)>>>(P);
  return (int)cudaGetLastError();
}

// group size G and blocks per thread T: T = 2 (fewer threads per cell, more cells per SM) with the
// smallest G such that G T covers every m x m Hessian block; IPM_GROUP_T=1 forces one block per thread
static void group_shape(int N, int t1, int& G, int& T) {
  const int NP = N * (N + 1) / 2;
  const int tmax = t1 ? 1 : 2;
  G = 0;
  T = 0;
  for (int t = tmax; t >= 1 && G == 0; --t)
    for (int g : {32, 64, 128, 256})
      if (NP <= g * t) {
        G = g;
        T = t;
        break;
      }
}

size_t big_scratch_doubles(int N, int Q, int m, int q1d, int npr, int p) {
  return m == 4 ? BigLayout<4>::scratch(N, Q, q1d, npr, p) : 0;
}

template <int CL, int MS, int NB, int W, int SF, int QC = 0, int NC = 0, int Q1C = 0>
static int dual_mma_impl(const KernelCtx& k, const DualLaunch& a) {
  using Lay = MmaLayout<MS>;
  constexpr int G = 32 * W;
  const int npr = SF * (SF + 1) / 2;
  const size_t tab = ((size_t)2 * k.T.N * k.T.QP + (SF > 0 ? ((k.T.q1d * npr + 1) & ~1) : 0) +
                      (size_t)k.T.MT * k.T.KS * 32 + ((size_t)k.T.N * (k.T.N + 1) / 2 + 3) / 4 * 2 +
                      (SF > 0 ? (size_t)((k.T.q1d + 3) / 4) * ((npr + 7) / 8) * 32 : 0) +  // + sLLF
                      (SF > 0 ? (size_t)Lay::pairlist_doubles(k.T.N, npr) : 0)) * 8;    // + stage-2 list
  const size_t pg = (size_t)Lay::per_group(k.T.N, k.T.Q, W, SF, k.T.q1d, NB) * 8;
  if (tab + pg > k.smem_optin) return -1;
  int groups = (int)((k.smem_optin - tab) / pg);
  groups = std::min(groups, std::min(512 / G, 15));  // named barriers 1..15 (0 = __syncthreads)
  if (k.mma_groups > 0) groups = std::min(groups, k.mma_groups);  // experiments
  const size_t smem = tab + groups * pg;
  auto kern = k_dual_mma<CL, MS, NB, W, SF, QC, NC, Q1C>;
  int per_sm = configure(kern, groups * G, smem);
  if (per_sm < 1) return -1;
  const int64_t want = (a.cells + groups - 1) / groups;
  int grid = (int)std::min<int64_t>(want, (int64_t)k.sm_count * per_sm);
  if (grid < 1) grid = 1;
  DualParams P{k.T, k.mesh, k.nw, k.ad, k.cl, a, k.sc};
  kern<<<grid, groups * G, smem, S(k)>>>(P);
  return (int)cudaGetLastError();
}

// DMMA-Cholesky kernel: 8x8 blocks of the padded n x n Hessian, W warps per cell so that the
// register blocks fit (<= 18 blocks per warp)
int dual_mma_dispatch(const KernelCtx& k, const DualLaunch& a, int SF) {
  const int n = k.T.N * k.m, NB = (n + 7) / 8;
  const int key = ((k.closure * 10 + k.m) * 100 + NB) * 10 + SF;
  if (k.mma_w4 && key == ((CL_EULER * 10 + 4) * 100 + 8) * 10 + 5)
    return dual_mma_impl<CL_EULER, 4, 8, 4, 5>(k, a);
  // the BASELINE configurations' shapes: compile-time-shape instances (Q, N, q1d constants)
  if (!k.mma_generic && (k.ad.n_levels == 0 || a.list)) {  // uniform N over the launch
    const int q1 = SF > 0 ? k.T.q1d : 0;
#define IPM_FCASE(CLV, MSV, NBV, WV, SFV, QV, NV, Q1V)                                                 \
  if (key == ((CLV * 10 + MSV) * 100 + NBV) * 10 + SFV && k.T.Q == QV && k.T.N == NV && q1 == Q1V) \
    return dual_mma_impl<CLV, MSV, NBV, WV, SFV, QV, NV, Q1V>(k, a);
    IPM_FCASE(CL_BARRIER, 1, 1, 1, 0, 20, 6, 0)   // config 1
    IPM_FCASE(CL_EULER, 3, 4, 1, 0, 30, 10, 0)    // config 2
    IPM_FCASE(CL_EULER, 4, 8, 2, 5, 100, 15, 10)  // config 3
    IPM_FCASE(CL_EULER, 4, 11, 4, 6, 144, 21, 12) // config 4 (degree 5)
    IPM_FCASE(CL_EULER, 4, 3, 1, 3, 144, 6, 12)   // config 4 degree-2 bucket
    IPM_FCASE(CL_EULER, 4, 5, 1, 4, 144, 10, 12)  // config 4 degree-3 bucket
    IPM_FCASE(CL_EULER, 4, 8, 2, 5, 144, 15, 12)  // config 4 degree-4 bucket
#undef IPM_FCASE
  }
  switch (key) {
#define IPM_MCASE(CLV, MSV, NBV, WV, SFV) \
  case ((CLV * 10 + MSV) * 100 + NBV) * 10 + SFV: return dual_mma_impl<CLV, MSV, NBV, WV, SFV>(k, a);
    IPM_MCASE(CL_BARRIER, 1, 1, 1, 0)
    IPM_MCASE(CL_QUADRATIC, 1, 1, 1, 0)
    IPM_MCASE(CL_EULER, 3, 4, 1, 0)
    IPM_MCASE(CL_EULER, 4, 3, 1, 3)
    IPM_MCASE(CL_EULER, 4, 5, 1, 4)
    IPM_MCASE(CL_EULER, 4, 8, 2, 5)
    IPM_MCASE(CL_EULER, 4, 8, 2, 0)
    IPM_MCASE(CL_EULER, 4, 11, 4, 6)
#undef IPM_MCASE
  }
  return -1;
}

static const char* g_last_dual = "";
const char* last_dual_kernel() { return g_last_dual; }

// the large-cell Newton kernel (config 5): CTA per cell, L2-resident scratch; also the Newton fallback of
// the large-cell quasi-Newton kernel (a.list)
static int launch_big(const KernelCtx& k, const DualLaunch& a) {
  if (!k.big_scratch || k.closure != CL_EULER || k.m != 4) return -1;
  constexpr int NT = 512;
  const size_t smem0 = ((size_t)5 * k.T.N * 4 + 8 * (NT / 32) + ((k.T.q1d * k.T.npr + 1) & ~1) + 8) * 8;
  const size_t nb8 = (size_t)(k.T.N * 4 + 7) / 8;
  const size_t hbl = (nb8 * (nb8 + 1) / 2 * 64 + 64) * 8;  // 8 x 8 blocks + Linv operand
  const int hb_in_smem = (smem0 + hbl <= k.smem_optin) ? 1 : 0;
  const size_t smem = smem0 + (hb_in_smem ? hbl : 0);
  auto kern = hb_in_smem ? k_dual_big<CL_EULER, 4, NT, true> : k_dual_big<CL_EULER, 4, NT, false>;
  configure(kern, 0, smem);
  const int grid = (int)std::min<int64_t>(a.cells, (int64_t)k.big_ctas);
  DualParams P{k.T, k.mesh, k.nw, k.ad, k.cl, a, k.sc};
  kern<<<grid, NT, smem, S(k)>>>(P, k.big_scratch);
  return (int)cudaGetLastError();
}

// quasi-Newton dual solve (reading 35): one warp per cell, as many warps per CTA as shared memory and
// registers allow, one persistent CTA per SM
template <int CL, int MS, int NR, int MH, bool PSM, int QC = 0, int NC = 0>
static int dual_lbfgs_impl(const KernelCtx& k, const DualLaunch& a) {
  const size_t tab = (((size_t)k.T.N * k.T.QP + (size_t)k.T.MT * k.T.KS * 32 + 1) & ~(size_t)1) * 8;
  const size_t pw = (size_t)LbfgsLayout<MS>::per_warp(32 * NR, k.T.Q, PSM ? MH : 0) * 8;
  if (tab + pw > k.smem_optin) return -1;
  int warps = (int)((k.smem_optin - tab) / pw);
  warps = std::min(warps, (PSM ? 512 : 384) / 32);
  auto kern = k_dual_lbfgs<CL, MS, NR, MH, PSM, QC, NC>;
  const size_t smem = tab + warps * pw;
  int per_sm = configure(kern, warps * 32, smem);
  if (per_sm < 1) return -1;
  const int64_t want = (a.cells + warps - 1) / warps;
  int grid = (int)std::min<int64_t>(want, (int64_t)k.sm_count * per_sm);
  if (grid < 1) grid = 1;
  DualParams P{k.T, k.mesh, k.nw, k.ad, k.cl, a, k.sc};
  kern<<<grid, warps * 32, smem, S(k)>>>(P);
  g_last_dual = "k_dual_lbfgs";
  return (int)cudaGetLastError();
}

static int dual_lbfgs_dispatch(const KernelCtx& k, const DualLaunch& a) {
  const int n = k.T.N * k.m, NR = (n + 31) / 32;
  if (k.lbfgs_m != 8) return -1;
  if (n > 96) {  // large cells (config 5): CTA per cell, sum-factorised node pass over the 3D tensor rule
    constexpr int NT = 256;
    if (!(k.closure == CL_EULER && k.m == 4 && k.T.p == 3 && k.T.L1 && n <= NT && k.ad.n_levels == 0)) return -1;
    const size_t smem = (size_t)LbfgsBigLayout<4>::doubles(n, k.T.Q, k.T.npr1 - 1, k.T.q1d, NT / 32) * 8;
    if (smem > k.smem_optin) return -1;
    // config 5's shape (q1d 10, degree 5, p = 3) at compile time
    auto kern = (k.T.q1d == 10 && k.T.npr1 == 6) ? k_dual_lbfgs_big<CL_EULER, 4, 8, NT, 10, 5>
                                                 : k_dual_lbfgs_big<CL_EULER, 4, 8, NT>;
    int per_sm = configure(kern, NT, smem);
    if (per_sm < 1) return -1;
    const int grid = (int)std::min<int64_t>(a.cells, (int64_t)k.sm_count * per_sm);
    DualParams P{k.T, k.mesh, k.nw, k.ad, k.cl, a, k.sc};
    kern<<<std::max(grid, 1), NT, smem, S(k)>>>(P);
    g_last_dual = "k_dual_lbfgs_big";
    return (int)cudaGetLastError();
  }
  // (compile-time Q, N instances of this kernel, as k_dual_mma has, measured 8 % slower on config 3 and
  // 4 % on config 4: r02u_*_lbfgs_fixed.json — the generic instance is the product path)
  switch ((k.closure * 10 + k.m) * 10 + NR) {
// pairs in shared memory (PSM) unless IPM_LBFGS_PAIRS=reg (read at ipm_init: k.lbfgs_pairs_reg)
#define IPM_LCASE(CLV, MSV, NRV)                                                                         \
  case (CLV * 10 + MSV) * 10 + NRV:                                                                      \
    return k.lbfgs_pairs_reg ? dual_lbfgs_impl<CLV, MSV, NRV, 8, false>(k, a)                          \
                             : dual_lbfgs_impl<CLV, MSV, NRV, 8, true>(k, a);
    IPM_LCASE(CL_QUADRATIC, 1, 1)
    IPM_LCASE(CL_BARRIER, 1, 1)
    IPM_LCASE(CL_EULER, 3, 1)
    IPM_LCASE(CL_EULER, 4, 1)
    IPM_LCASE(CL_EULER, 4, 2)
    IPM_LCASE(CL_EULER, 4, 3)
#undef IPM_LCASE
  }
  return -1;
}

// cells -> per-level lists (warp-aggregated atomics; the order inside a list is irrelevant: every
// cell's solve is independent of the others)
__global__ void k_bucket(const int32_t* __restrict__ level, int64_t cells, int32_t* __restrict__ lists,
                         StepScalars* sc) {
  const int lane = threadIdx.x & 31;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < cells; j0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    const bool live = j < cells;
    const int l = live ? level[j] : -1;
    const unsigned peers = __match_any_sync(FULL_MASK, l);
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (live && lane == leader) base = atomicAdd(&sc->lvl_count[l], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    if (live) lists[(int64_t)l * cells + base + __popc(peers & ((1u << lane) - 1))] = (int32_t)j;
  }
}

int dual_mma_dispatch(const KernelCtx& k, const DualLaunch& a, int SF);

// adaptive degree in uniform-degree buckets (north star (c); Alg. 3): one k_dual_mma launch per
// level with that level's basis size N_l (its own register-block shape and warps per cell) over the
// level's cells, instead of one launch at N_max looping over each cell's level
static int launch_dual_bucketed(const KernelCtx& k, const DualLaunch& a) {
  const int L = k.ad.n_levels;
  cudaMemsetAsync(&k.sc->lvl_count[0], 0, sizeof(int) * 16, S(k));
  if (k.hessian_kind == 1) cudaMemsetAsync(&k.sc->fb_count[0], 0, sizeof(int) * 16, S(k));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((a.cells + 255) / 256, (int64_t)k.sm_count * 8));
  k_bucket<<<grid, 256, 0, S(k)>>>(a.level, a.cells, k.lists, k.sc);
  for (int l = 0; l < L; ++l) {
    KernelCtx kl = k;
    kl.T = k.Tl[l];
    kl.bucket = 0;
    DualLaunch al = a;
    al.list = k.lists + (int64_t)l * a.cells;
    al.ncells_dev = &k.sc->lvl_count[l];
    al.queue = &k.sc->lvl_queue[l];
    al.row = k.T.N * k.m;
    const int SF = (k.T.p == 2 && k.sumfact) ? (int)std::lround((std::sqrt(8.0 * kl.T.npr + 1) - 1) / 2) : 0;
    if (k.hessian_kind == 1) {
      al.fb_list = k.fb_lists + (int64_t)l * a.cells;
      al.fb_count = &k.sc->fb_count[l];
      if (const int rc = dual_lbfgs_dispatch(kl, al)) return rc;
      // reading 35: Newton from the iterate for the cells that reached max_newton quasi-Newton steps
      DualLaunch af = al;
      af.list = al.fb_list;
      af.ncells_dev = al.fb_count;
      af.queue = &k.sc->fb_queue[l];
      af.accumulate = 1;
      af.fb_list = nullptr;
      if (const int rc = dual_mma_dispatch(kl, af, SF)) return rc;
    } else if (const int rc = dual_mma_dispatch(kl, al, SF)) {
      return rc;
    }
  }
  g_last_dual = k.hessian_kind == 1 ? "k_dual_lbfgs" : "k_dual_mma";
  return (int)cudaGetLastError();
}

int launch_dual(const KernelCtx& k, const DualLaunch& a) {
  if (a.cells == 0) return 0;
  if (k.hessian_kind == 1 && !(k.bucket && a.level && !a.list)) {
    cudaMemsetAsync(&k.sc->fb_count[0], 0, sizeof(int) * 16, S(k));
    DualLaunch al = a;
    al.fb_list = k.fb_lists;
    al.fb_count = &k.sc->fb_count[0];
    if (const int rc = dual_lbfgs_dispatch(k, al)) return rc;
    // reading 35: Newton from the iterate for the cells that reached max_newton quasi-Newton steps
    DualLaunch af = a;
    af.list = k.fb_lists;
    af.ncells_dev = &k.sc->fb_count[0];
    af.queue = &k.sc->fb_queue[0];
    af.accumulate = 1;
    af.row = a.row ? a.row : k.T.N * k.m;
    const char* qn = g_last_dual;
    int rc;
    if (k.T.N * k.m > 96) {
      rc = launch_big(k, af);  // (k_dual_big: the Newton kernel of the large cells)
    } else {
      const int SF = (k.T.p == 2 && k.sumfact) ? (int)std::lround((std::sqrt(8.0 * k.T.npr + 1) - 1) / 2) : 0;
      rc = dual_mma_dispatch(k, af, SF);  // (every warp-kernel L-BFGS shape has a k_dual_mma instance)
    }
    g_last_dual = qn;
    return rc;
  }
  if (k.bucket && a.level && !a.list && (k.hessian_kind == 1 || (!k.force_warp_kernel && !k.dual_group)))
    return launch_dual_bucketed(k, a);
  // default: the DMMA-Cholesky kernel where it is instantiated; IPM_DUAL_KERNEL=group selects the
  // 4x4-register-block kernel (comparison, tests)
  if (!k.force_warp_kernel && !k.dual_group) {
    const int SF = (k.T.p == 2 && k.sumfact) ? (int)std::lround((std::sqrt(8.0 * k.T.npr + 1) - 1) / 2) : 0;
    const int rc = dual_mma_dispatch(k, a, SF);
    if (rc != -1) {
      g_last_dual = "k_dual_mma";
      return rc;
    }
  }
  if (!k.force_warp_kernel) {
    int G, T;
    group_shape(k.T.N, k.group_t1, G, T);
    // sum factorisation for p = 2 tensor rules (SF = M + 1); IPM_SUMFACT=0 selects the direct sum
    const int SF = (k.T.p == 2 && k.sumfact) ? (int)std::lround((std::sqrt(8.0 * k.T.npr + 1) - 1) / 2) : 0;
    const int key = (((k.closure * 10 + k.m) * 1000 + G) * 10 + SF) * 10 + T;
    int rc = -1;
    switch (key) {
#define IPM_GCASE(CLV, MSV, GV, SFV, TV) \
  case (((CLV * 10 + MSV) * 1000 + GV) * 10 + SFV) * 10 + TV: rc = dual_group_impl<CLV, MSV, GV, SFV, TV>(k, a); break;
      IPM_GCASE(CL_BARRIER, 1, 32, 0, 1)
      IPM_GCASE(CL_BARRIER, 1, 32, 0, 2)
      IPM_GCASE(CL_QUADRATIC, 1, 32, 0, 1)
      IPM_GCASE(CL_EULER, 3, 32, 0, 2)
      IPM_GCASE(CL_EULER, 3, 64, 0, 1)
      IPM_GCASE(CL_EULER, 4, 64, 0, 2)
      IPM_GCASE(CL_EULER, 4, 64, 5, 2)
      IPM_GCASE(CL_EULER, 4, 128, 0, 1)
      IPM_GCASE(CL_EULER, 4, 128, 5, 1)
      IPM_GCASE(CL_EULER, 4, 128, 0, 2)
      IPM_GCASE(CL_EULER, 4, 128, 6, 2)
      IPM_GCASE(CL_EULER, 4, 256, 6, 1)
      IPM_GCASE(CL_EULER, 4, 32, 3, 2)
      IPM_GCASE(CL_EULER, 4, 64, 4, 2)
#undef IPM_GCASE
    }
    if (rc != -1) {
      g_last_dual = "k_dual_group";
      return rc;
    }
    // cells too large for the on-chip group kernel (config 5): CTA per cell, L2-resident scratch
    if (k.big_scratch && k.closure == CL_EULER && k.m == 4) {
      const int rc = launch_big(k, a);
      g_last_dual = "k_dual_big";
      return rc;
    }
  }
  g_last_dual = "k_dual_warp";
  switch (k.closure * 10 + k.m) {
    case CL_QUADRATIC * 10 + 1: return dual_impl<CL_QUADRATIC, 1>(k, a);
    case CL_QUADRATIC * 10 + 3: return dual_impl<CL_QUADRATIC, 3>(k, a);
    case CL_QUADRATIC * 10 + 4: return dual_impl<CL_QUADRATIC, 4>(k, a);
    case CL_BARRIER * 10 + 1: return dual_impl<CL_BARRIER, 1>(k, a);
    case CL_EULER * 10 + 3: return dual_impl<CL_EULER, 3>(k, a);
    case CL_EULER * 10 + 4: return dual_impl<CL_EULER, 4>(k, a);
  }
  return -1;
}

template <int FX, int MS, int MK>
static int flux_impl(const KernelCtx& k, const FluxLaunch& a) {
  // per-level rules: the scalar projection with omega Phi^T (1); otherwise the DMMA projection with the
  // A-fragment table (2), staged in shared memory when it fits next to 4 warps' buffers
  const bool scalar = k.ad.lq.on || k.flux_scalar_proj || k.T.N > 64;
  const size_t tab = scalar ? (size_t)k.T.N * k.T.QP * 8 : (size_t)k.T.MT * k.T.KS * 32 * 8;
  // DMMA projection: the per-warp buffer holds the whole rule up to 256 nodes (config 4: one chunk of
  // 144, measured 1.56 ms against 2.23 ms in chunks of 128), chunks of 128 beyond (config 5: 1 000)
  const int q4 = (k.T.Q + 3) & ~3;
  const int qchunk = scalar ? 0 : (q4 <= 256 ? q4 : 128);
  const size_t pw = (size_t)((scalar ? k.T.Q : qchunk) * MS + 1) * 8;
  int in_smem = (tab + 4 * pw <= k.smem_optin) ? (scalar ? 1 : 2) : 0;
  const size_t base = in_smem ? tab : 0;
  int warps = (int)std::min<size_t>(8, (k.smem_optin - base) / pw);
  if (warps < 1) return -1;
  const size_t smem = base + warps * pw;
  const bool ch = qchunk > 0 && qchunk < k.T.Q;
  void (*kern)(FluxParams) = ch ? k_flux_warp<FX, MS, MK, true> : k_flux_warp<FX, MS, MK, false>;
  if constexpr (MS == 4 && MK == MK_TRI) {
    bool ff = false;
    for (int t = 0; t < 4; ++t) ff = ff || k.mesh.bc_kind[t] == 3;
    if (ff) kern = ch ? k_flux_warp<FX, MS, MK, true, true> : k_flux_warp<FX, MS, MK, false, true>;
  }
  int per_sm = configure(kern, warps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (k.mesh.cells - a.cell0 + warps - 1) / warps;
  int grid = (int)std::min<int64_t>(want, (int64_t)k.sm_count * per_sm * 4);
  if (grid < 1) grid = 1;
  FluxParams P{k.T, k.mesh, k.cl, k.ad, a, k.sc, in_smem, qchunk};
  kern<<<grid, warps * 32, smem, S(k)>>>(P);
  return (int)cudaGetLastError();
}

template <int FX, int MS, int MK>
static int flux_cart_impl(const KernelCtx& k, const FluxLaunch& a) {
  constexpr int CPW = 8 / MS;
  const size_t tab = (size_t)k.T.MT * k.T.KS * 32 * 8, pw = (size_t)k.T.KS * 32 * 8;
  if (tab + pw > k.smem_optin) return -1;
  const int warps = (int)std::min<size_t>(8, (k.smem_optin - tab) / pw);
  const size_t smem = tab + warps * pw;
  auto kern = k_flux_cart<FX, MS, MK>;
  int per_sm = configure(kern, warps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t groups = (k.mesh.cells + CPW - 1) / CPW;
  const int64_t want = (groups + warps - 1) / warps;
  int grid = (int)std::min<int64_t>(want, (int64_t)k.sm_count * per_sm);
  if (grid < 1) grid = 1;
  FluxParams P{k.T, k.mesh, k.cl, k.ad, a, k.sc, 1};
  kern<<<grid, warps * 32, smem, S(k)>>>(P);
  return (int)cudaGetLastError();
}

// strip kernel (row-major cartesian block, Euler 2D Rusanov, Q = QC): -1 when not applicable
template <int TX, int NT, int MINB, int QC, bool SC = false>
static int flux_strip_impl(const KernelCtx& k, const FluxLaunch& a) {
  if (k.mesh.kind != MK_CART || k.m != 4 || k.flux != FX_RUSANOV || k.mesh.bx <= 0 || k.T.Q != QC) return -1;
  const strip::Layout<TX, QC> lay(k.T.MT, k.T.N * 4);
  const size_t smem = lay.total * 8;
  if (smem > k.smem_optin) return -1;
  auto kern = k_flux_strip<TX, NT, MINB, QC, SC>;
  int per_sm = configure(kern, NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t rows = (int64_t)((k.mesh.bx + TX - 1) / TX) * k.mesh.by;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)k.sm_count * per_sm));
  FluxParams P{k.T, k.mesh, k.cl, k.ad, a, k.sc, 1};
  kern<<<grid, NT, smem, S(k)>>>(P);
  return (int)cudaGetLastError();
}

int launch_retard(const KernelCtx& k) {
  if (k.ad.n_retard <= 0) return 0;
  k_retard<<<1, 1, 0, S(k)>>>(k.sc, k.ad);
  return (int)cudaGetLastError();
}

static const char* g_last_flux = "";
const char* last_flux_kernel() { return g_last_flux; }

int launch_flux(const KernelCtx& k, const FluxLaunch& a) {
  if (k.mesh.cells <= a.cell0) return 0;
  const int key = (k.flux * 10 + k.m) * 10 + k.mesh.kind;
  // banded node states, or per-level rules (reading 36): the cell-range kernel only
  const bool banded = a.uq_halo != nullptr || k.ad.lq.on;
  if (k.flux_choice == 0 && !banded) {
#ifndef IPM_STRIP_NT
#define IPM_STRIP_NT 512
#endif
    const int rc = flux_strip_impl<8, IPM_STRIP_NT, 1, 100>(k, a);
    if (rc != -1) {
      g_last_flux = "k_flux_strip";
      return rc;
    }
  }
  if (k.flux_choice != 2 && !banded) {
    int rc = -1;
    switch (key) {
      case (FX_LF_GLOBAL * 10 + 1) * 10 + MK_1D: rc = flux_cart_impl<FX_LF_GLOBAL, 1, MK_1D>(k, a); break;
      case (FX_HLL * 10 + 3) * 10 + MK_1D: rc = flux_cart_impl<FX_HLL, 3, MK_1D>(k, a); break;
      case (FX_RUSANOV * 10 + 3) * 10 + MK_1D: rc = flux_cart_impl<FX_RUSANOV, 3, MK_1D>(k, a); break;
      case (FX_RUSANOV * 10 + 4) * 10 + MK_CART: rc = flux_cart_impl<FX_RUSANOV, 4, MK_CART>(k, a); break;
      case (FX_HLL * 10 + 4) * 10 + MK_CART: rc = flux_cart_impl<FX_HLL, 4, MK_CART>(k, a); break;
    }
    if (rc != -1) {
      g_last_flux = "k_flux_cart";
      return rc;
    }
  }
  g_last_flux = "k_flux_warp";
  switch (key) {
    case (FX_LF_GLOBAL * 10 + 1) * 10 + MK_1D: return flux_impl<FX_LF_GLOBAL, 1, MK_1D>(k, a);
    case (FX_HLL * 10 + 3) * 10 + MK_1D: return flux_impl<FX_HLL, 3, MK_1D>(k, a);
    case (FX_RUSANOV * 10 + 3) * 10 + MK_1D: return flux_impl<FX_RUSANOV, 3, MK_1D>(k, a);
    case (FX_RUSANOV * 10 + 4) * 10 + MK_CART: return flux_impl<FX_RUSANOV, 4, MK_CART>(k, a);
    case (FX_HLL * 10 + 4) * 10 + MK_CART: return flux_impl<FX_HLL, 4, MK_CART>(k, a);
    case (FX_RUSANOV * 10 + 4) * 10 + MK_TRI: return flux_impl<FX_RUSANOV, 4, MK_TRI>(k, a);
  }
  return -1;
}

template <int FX, int MS, int MK>
static int sc_impl(const KernelCtx& k, const double* Uin, double* Uout) {
  const int threads = 256;
  const int64_t n = k.mesh.cells * k.T.Q;
  const int rgrid = (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)k.sm_count * 8));
  k_sc_rate<MS><<<rgrid, threads, 0, S(k)>>>(k.mesh.cells, k.T.Q, k.mesh, k.cl.gamma, Uin, k.sc);
  return (int)cudaGetLastError();
}
template <int FX, int MS, int MK>
static int sc_update_impl(const KernelCtx& k, const double* Uin, double* Uout) {
  const int64_t want = (k.mesh.cells + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)k.sm_count * 8));
  FluxParams P{k.T, k.mesh, k.cl, k.ad, FluxLaunch{}, k.sc, 0};
  k_sc_update<FX, MS, MK><<<grid, 256, 0, S(k)>>>(P, Uin, Uout);
  return (int)cudaGetLastError();
}
#define IPM_SC_DISPATCH(FN)                                                                          \
  switch ((k.flux * 10 + k.m) * 10 + k.mesh.kind) {                                                 \
    case (FX_LF_GLOBAL * 10 + 1) * 10 + MK_1D: return FN<FX_LF_GLOBAL, 1, MK_1D>(k, Uin, Uout);     \
    case (FX_HLL * 10 + 3) * 10 + MK_1D: return FN<FX_HLL, 3, MK_1D>(k, Uin, Uout);                 \
    case (FX_RUSANOV * 10 + 3) * 10 + MK_1D: return FN<FX_RUSANOV, 3, MK_1D>(k, Uin, Uout);         \
    case (FX_RUSANOV * 10 + 4) * 10 + MK_CART: return FN<FX_RUSANOV, 4, MK_CART>(k, Uin, Uout);     \
    case (FX_HLL * 10 + 4) * 10 + MK_CART: return FN<FX_HLL, 4, MK_CART>(k, Uin, Uout);             \
    case (FX_RUSANOV * 10 + 4) * 10 + MK_TRI: return FN<FX_RUSANOV, 4, MK_TRI>(k, Uin, Uout);       \
  }                                                                                                  \
  return -1;
int launch_sc_rate(const KernelCtx& k, const double* Uin) {
  double* Uout = nullptr;
  IPM_SC_DISPATCH(sc_impl)
}
int launch_sc_update(const KernelCtx& k, const double* Uin, double* Uout) {
  if (k.flux_choice == 0) {  // the strip walk (cartesian blocks, Euler Rusanov, Q = 100)
    FluxLaunch a{};
    a.uq = Uin;
    a.uhat_new = Uout;
    const int rc = flux_strip_impl<8, IPM_STRIP_NT, 1, 100, true>(k, a);
    if (rc != -1) return rc;
  }
  IPM_SC_DISPATCH(sc_update_impl)
}

template <int MS>
__global__ void k_sc_moments(Tables T, int64_t cells, const double* __restrict__ U, double* __restrict__ uhat) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int N = T.N, Q = T.Q;
  for (int64_t cell = (int64_t)blockIdx.x * nw + warp; cell < cells; cell += (int64_t)gridDim.x * nw)
    for (int r = lane; r < N * MS; r += 32) {
      const int i = r / MS, a = r - i * MS;
      double s = 0.0;
      for (int k = 0; k < Q; ++k) s = fma(T.WPhiT[i * T.QP + k], U[cell * Q * MS + a * Q + k], s);
      uhat[cell * N * MS + r] = s;
    }
}
int launch_sc_moments(const KernelCtx& k, const double* U, double* uhat) {
  const int64_t want = (k.mesh.cells + 7) / 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)k.sm_count * 8));
  switch (k.m) {
    case 1: k_sc_moments<1><<<grid, 256, 0, S(k)>>>(k.T, k.mesh.cells, U, uhat); break;
    case 3: k_sc_moments<3><<<grid, 256, 0, S(k)>>>(k.T, k.mesh.cells, U, uhat); break;
    case 4: k_sc_moments<4><<<grid, 256, 0, S(k)>>>(k.T, k.mesh.cells, U, uhat); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}

template <int MS>
static int ic_impl(const KernelCtx& k, const double* region, const double* split, int kind, int nx, double x0,
                   double y0, double dx, double dy, const int32_t* level, const int64_t* gid, double* uhat,
                   double* unodes) {
  const size_t pw = (size_t)(k.T.Q * MS + 1) * 8;
  const int warps = (int)std::min<size_t>(8, k.smem_optin / pw);
  if (warps < 1) return -1;
  const size_t smem = (size_t)warps * pw;
  auto kern = k_project_ic<MS>;
  configure(kern, 0, smem);
  const int64_t want = (k.mesh.cells + warps - 1) / warps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)k.sm_count * 8));
  kern<<<grid, warps * 32, smem, S(k)>>>(k.T, k.mesh.cells, region, split, kind, nx, x0, y0, dx, dy, level, gid,
                                         k.ad, uhat, unodes);
  return (int)cudaGetLastError();
}

int launch_project_ic(const KernelCtx& k, const double* region, const double* split, int kind, int nx, double x0,
                      double y0, double dx, double dy, const int32_t* level, const int64_t* gid, double* uhat,
                      double* unodes) {
  switch (k.m) {
    case 1: return ic_impl<1>(k, region, split, kind, nx, x0, y0, dx, dy, level, gid, uhat, unodes);
    case 3: return ic_impl<3>(k, region, split, kind, nx, x0, y0, dx, dy, level, gid, uhat, unodes);
    case 4: return ic_impl<4>(k, region, split, kind, nx, x0, y0, dx, dy, level, gid, uhat, unodes);
  }
  return -1;
}

template <int CL, int MS>
static int warm_impl(const KernelCtx& k, const double* uhat, double* lam) {
  const int64_t n = k.mesh.cells;
  k_warm_start<CL, MS><<<(unsigned)((n + 127) / 128), 128, 0, S(k)>>>(n, k.T.N, k.cl, uhat, lam, k.sc);
  return (int)cudaGetLastError();
}

template <int CL, int MS>
static int nodes_impl(const KernelCtx& k, const double* lam, double* uhat, double* uq, int want_rate, int exact) {
  // node states only: k_nodes_out; exact = 1 (halo cells of distributed contexts) keeps the dual
  // kernels' instruction sequence (warp_eval), so a virtual-rank run equals one context bit for bit
  if (!uhat && uq && !exact) {
    constexpr int C = (MS == 4) ? 4 : 2, W = 8;
    const size_t tab = (size_t)k.T.N * k.T.QP * 8, pw = (size_t)C * k.T.N * MS * 8;
    const int in_smem = (tab + W * pw <= k.smem_optin / 2) ? 1 : 0;  // (leave room for 2 CTAs per SM)
    const size_t smem = (in_smem ? tab : 0) + W * pw;
    auto kern = k_nodes_out<CL, MS, C>;
    int per_sm = configure(kern, W * 32, smem);
    if (per_sm < 1) return -1;
    const int64_t want = (k.mesh.cells + W * C - 1) / (W * C);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)k.sm_count * per_sm));
    kern<<<grid, W * 32, smem, S(k)>>>(k.T, k.mesh, k.cl, lam, uq, k.sc, in_smem, want_rate);
    return (int)cudaGetLastError();
  }
  using Lay = DualLayout<MS>;
  const size_t tab = (size_t)2 * k.T.N * k.T.QP * 8, pw = (size_t)(k.T.N * MS + k.T.Q * Lay::NS + 1) * 8;
  const int in_smem = (tab + 4 * pw <= k.smem_optin) ? 1 : 0;
  const size_t base = in_smem ? tab : 0;
  const int warps = (int)std::min<size_t>(4, (k.smem_optin - base) / pw);
  if (warps < 1) return -1;
  const size_t smem = base + warps * pw;
  auto kern = k_nodes<CL, MS>;
  configure(kern, 0, smem);
  const int64_t want = (k.mesh.cells + warps - 1) / warps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)k.sm_count * 4));
  kern<<<grid, warps * 32, smem, S(k)>>>(k.T, k.mesh, k.cl, lam, uhat, uq, k.sc, in_smem, want_rate);
  return (int)cudaGetLastError();
}

template <int CL, int MS>
static int stress_impl(const KernelCtx& k, const double* base, const double* z, double rel, double abs_,
                       double* lam) {
  const int warps = 8;
  const int64_t want = (k.mesh.cells + warps - 1) / warps;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)k.sm_count * 16));
  k_stress<CL, MS><<<grid, warps * 32, 0, S(k)>>>(k.T, k.mesh.cells, k.cl, base, z, rel, abs_, lam);
  return (int)cudaGetLastError();
}

#define IPM_DISPATCH_CL(FN, ...)                                                \
  switch (k.closure * 10 + k.m) {                                               \
    case CL_QUADRATIC * 10 + 1: return FN<CL_QUADRATIC, 1>(k, __VA_ARGS__);     \
    case CL_QUADRATIC * 10 + 3: return FN<CL_QUADRATIC, 3>(k, __VA_ARGS__);     \
    case CL_QUADRATIC * 10 + 4: return FN<CL_QUADRATIC, 4>(k, __VA_ARGS__);     \
    case CL_BARRIER * 10 + 1: return FN<CL_BARRIER, 1>(k, __VA_ARGS__);         \
    case CL_EULER * 10 + 3: return FN<CL_EULER, 3>(k, __VA_ARGS__);             \
    case CL_EULER * 10 + 4: return FN<CL_EULER, 4>(k, __VA_ARGS__);             \
  }                                                                             \
  return -1;

int launch_warm_start(const KernelCtx& k, const double* uhat, double* lam) { IPM_DISPATCH_CL(warm_impl, uhat, lam) }
int launch_nodes(const KernelCtx& k, const double* lam, double* uhat, double* uq, int want_rate, int exact) {
  IPM_DISPATCH_CL(nodes_impl, lam, uhat, uq, want_rate, exact)
}

__global__ void k_pack(const double* __restrict__ lam, const int32_t* __restrict__ idx, int64_t n, int row,
                       double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * row) return;
  const int64_t s = e / row, r = e - s * row;
  out[e] = lam[(int64_t)idx[s] * row + r];
}

int launch_pack(const KernelCtx& k, const double* lam, const int32_t* idx, int64_t n, double* out) {
  if (n == 0) return 0;
  const int row = k.T.N * k.m;
  const int64_t tot = n * row;
  k_pack<<<(unsigned)((tot + 255) / 256), 256, 0, S(k)>>>(lam, idx, n, row, out);
  return (int)cudaGetLastError();
}
int launch_stress(const KernelCtx& k, const double* base, const double* z, double rel, double abs_, double* lam) {
  IPM_DISPATCH_CL(stress_impl, base, z, rel, abs_, lam)
}

}  // namespace ipm
