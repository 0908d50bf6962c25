// ipm_dual_group.cuh — cell-per-thread-group dual solve (sm_100a, fp64).
//
// A CTA holds GROUPS groups of G threads; each group solves one spatial cell at a time (cells pulled
// from an atomic queue: Newton counts differ from cell to cell).  The basis tables Phi, omega Phi
// are staged once per CTA and shared by all groups; groups synchronise with named barriers.
//
// Per Newton iteration, for a cell with N_l basis functions and m states:
//   eval      Lambda_k = Phi lambda, u_k = u_s(Lambda_k), J_k = grad u_s(Lambda_k), s_*   (threads over k)
//   gradient  g = Phi^T(omega o u) - uhat, crit = sum_a ||g_.a||                       (threads over (i,a))
//   Hessian   thread t owns the m x m block H_{(I,.),(J,.)} of basis pair (I >= J), built in registers:
//             H_IJ = sum_k omega_k phi_kI phi_kJ J_k
//   Cholesky  blocked right-looking over block columns K; the blocks never leave registers until
//             finished (L_IK is published to shared memory for the trailing updates)
//   solves    L y = -g, L^T d = y (one warp, column-oriented)
//   Armijo    on L(lambda) with the rounding allowance of reading 3'; the accepted trial's node data
//             and gradient are the next iteration's.
#pragma once
// (included inside namespace ipm by ipm_kernels.cu, after DualParams and node_rate)

template <int MS>
struct GroupLayout {
  static constexpr int MM = MS * (MS + 1) / 2;
  static constexpr int NS = ((MS + MM) % 2 == 0) ? MS + MM + 1 : MS + MM;
  static constexpr int TB = MS * MS;  // doubles per block (stored column-major)
  static constexpr int RS = MS > 2 ? MS : 2;  // values per reduction slot
  // doubles per group: 5 vectors + union(node buffer, L blocks) + reduction scratch + control
  static __host__ __device__ int per_group(int N, int Q, int G) {
    const int n = N * MS, NP = N * (N + 1) / 2;
    const int nb = Q * NS, lb = NP * TB;
    int w = 5 * n + (nb > lb ? nb : lb) + 2 * RS * (G / 32) + 4;
    return (w + 1) & ~1;
  }
};

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int CL, int MS, int G>
__global__ void __launch_bounds__(768) k_dual_group(DualParams P) {
  using Lay = GroupLayout<MS>;
  constexpr int NW = G / 32;
  constexpr int MM = Lay::MM, NS = Lay::NS, TB = Lay::TB;
#define LIDX(a, b) ((b) * MS + (a))  // element (a, b) of a column-major block
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, Q = P.T.Q, QP = P.T.QP;
  double* sPhiT = sm;
  double* sWPhiT = sm + N * QP;
  for (int x = threadIdx.x; x < N * QP; x += blockDim.x) {
    sPhiT[x] = P.T.PhiT[x];
    sWPhiT[x] = P.T.WPhiT[x];
  }
  __syncthreads();
  const int grp = threadIdx.x / G, t = threadIdx.x - grp * G;
  const int wig = t >> 5, lane = t & 31;
  const int bar = 1 + grp;
  const int nmax = N * MS;
  double* base = sm + 2 * N * QP + (size_t)grp * Lay::per_group(N, Q, G);
  double* lam = base;
  double* lt = lam + nmax;
  double* uh = lt + nmax;
  double* g = uh + nmax;
  double* dd = g + nmax;
  double* nb = dd + nmax;  // node buffer, union with the L blocks
  double* Ls = nb;
  const int nbsize = Q * NS > (N * (N + 1) / 2) * TB ? Q * NS : (N * (N + 1) / 2) * TB;
  double* red = nb + nbsize;  // [2 slots][RS][NW]
  int* ctl = (int*)(red + 2 * Lay::RS * NW);

  const double* __restrict__ omega = P.T.omega;
  const DualLaunch& A = P.a;
  long long my_iters = 0, my_failed = 0;
  int my_worst = 0;
  double my_rate = 0.0;
  int slot = 0;

  auto gsync = [&]() { named_sync(bar, G); };
  // group-wide sums of MS values (alternating scratch slots)
  auto gsum_vec = [&](double* v) {
    double* r = red + slot * Lay::RS * NW;
    slot ^= 1;
#pragma unroll
    for (int a = 0; a < MS; ++a) {
      const double s = warp_sum(v[a]);
      if (lane == 0) r[a * NW + wig] = s;
    }
    gsync();
#pragma unroll
    for (int a = 0; a < MS; ++a) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += r[a * NW + w];
      v[a] = s;
    }
  };
  auto gsum2 = [&](double& x, double& y) {
    double v[MS > 1 ? MS : 2];
    v[0] = x;
    v[1] = y;
#pragma unroll
    for (int a = 2; a < (MS > 1 ? MS : 2); ++a) v[a] = 0.0;
    if constexpr (MS >= 2) {
      gsum_vec(v);
    } else {
      double* r = red + slot * Lay::RS * NW;
      slot ^= 1;
      const double s0 = warp_sum(v[0]), s1 = warp_sum(v[1]);
      if (lane == 0) {
        r[wig] = s0;
        r[NW + wig] = s1;
      }
      gsync();
      v[0] = 0.0;
      v[1] = 0.0;
      for (int w = 0; w < NW; ++w) {
        v[0] += r[w];
        v[1] += r[NW + w];
      }
    }
    x = v[0];
    y = v[1];
  };

  // eval(lamv) -> nb; returns admissible; s1 = <s_*>, s2 = <|s_*|>
  auto eval = [&](const double* lamv, int Nl, double& s1, double& s2) -> bool {
    double a1 = 0.0, a2 = 0.0, bad = 0.0;
    for (int k = t; k < Q; k += G) {
      double Lam[MS];
#pragma unroll
      for (int a = 0; a < MS; ++a) Lam[a] = 0.0;
      for (int i = 0; i < Nl; ++i) {
        const double ph = sPhiT[i * QP + k];
#pragma unroll
        for (int a = 0; a < MS; ++a) Lam[a] = fma(lamv[i * MS + a], ph, Lam[a]);
      }
      double u[MS], J[MM], ss;
      const bool ok = Closure<CL, MS>::eval(Lam, u, J, ss, P.cl);
      if (!ok) bad = 1.0;
      double* row = nb + k * NS;
#pragma unroll
      for (int a = 0; a < MS; ++a) row[a] = u[a];
#pragma unroll
      for (int q = 0; q < MM; ++q) row[MS + q] = J[q];
      const double w = omega[k];
      a1 = fma(w, ss, a1);
      a2 = fma(w, fabs(ss), a2);
    }
    // bad flag folded into the second sum as +inf
    if (bad != 0.0) a2 = INFINITY;
    gsum2(a1, a2);
    s1 = a1;
    s2 = a2;
    return isfinite(a2) && isfinite(a1);
  };

  auto grad = [&](int Nl) -> double {
    const int n = Nl * MS;
    double part[MS];
#pragma unroll
    for (int a = 0; a < MS; ++a) part[a] = 0.0;
    for (int r = t; r < n; r += G) {
      const int i = r / MS, a = r - i * MS;
      const double* wp = sWPhiT + i * QP;
      double s = 0.0;
      for (int k = 0; k < Q; ++k) s = fma(wp[k], nb[k * NS + a], s);
      const double gr = s - uh[r];
      g[r] = gr;
#pragma unroll
      for (int b = 0; b < MS; ++b)
        if (b == a) part[b] = fma(gr, gr, part[b]);
    }
    gsum_vec(part);
    double crit = 0.0;
#pragma unroll
    for (int a = 0; a < MS; ++a) crit += sqrt(part[a]);
    return crit;
  };

  auto dot2 = [&](const double* x, const double* y, int n, double& d, double& ad) {
    double s = 0.0, sa = 0.0;
    for (int r = t; r < n; r += G) {
      const double v = x[r] * y[r];
      s += v;
      sa += fabs(v);
    }
    gsum2(s, sa);
    d = s;
    ad = sa;
  };

  // block (I, J) owned by this thread: row-major lower enumeration p = I(I+1)/2 + J
  int bI = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while (bI * (bI + 1) / 2 > t) --bI;
  while ((bI + 1) * (bI + 2) / 2 <= t) ++bI;
  const int bJ = t - bI * (bI + 1) / 2;

  for (;;) {
    if (t == 0) ctl[0] = atomicAdd(&P.sc->work_counter, 1);
    gsync();
    const int64_t cell = ctl[0];
    if (cell >= A.cells) break;
    const int lvl = A.level ? A.level[cell] : 0;
    const int Nl = (P.ad.n_levels > 0) ? P.ad.Nl[lvl] : N;
    const int n = Nl * MS;
    const int NPl = Nl * (Nl + 1) / 2;
    const bool own = t < NPl;
    const double* gu = A.uhat + cell * nmax;
    double* gl = A.lam + cell * nmax;
    for (int r = t; r < n; r += G) {
      uh[r] = gu[r];
      lam[r] = gl[r];
    }
    gsync();

    int status = 0, l = 0;
    double s1, s2, crit = INFINITY;
    bool nb_is_lam = eval(lam, Nl, s1, s2);
    if (!nb_is_lam) {
      status = 4;
    } else {
      crit = grad(Nl);
      double L0, scale;
      {
        double d1, d2;
        dot2(lam, uh, n, d1, d2);
        L0 = s1 - d1;
        scale = s2 + d2;
      }
      for (;;) {
        if (crit < P.nw.tau) break;
        if (P.nw.mode == 1 && l == 1) break;
        if (l == P.nw.max_newton) {
          status = 1;
          break;
        }
        // ---- Hessian block in registers -------------------------------------------------------
        double blk[MS][MS];
        if (own) {
          double acc[MM];
#pragma unroll
          for (int q = 0; q < MM; ++q) acc[q] = 0.0;
          const double* wi = sWPhiT + bI * QP;
          const double* pj = sPhiT + bJ * QP;
          for (int k = 0; k < Q; ++k) {
            const double f = wi[k] * pj[k];
            const double* Jk = nb + k * NS + MS;
#pragma unroll
            for (int q = 0; q < MM; ++q) acc[q] = fma(f, Jk[q], acc[q]);
          }
#pragma unroll
          for (int a = 0; a < MS; ++a)
#pragma unroll
            for (int b = 0; b < MS; ++b) blk[a][b] = acc[a <= b ? sym_idx<MS>(a, b) : sym_idx<MS>(b, a)];
        }
        gsync();  // node buffer dead from here: L blocks reuse it
        // ---- blocked Cholesky ------------------------------------------------------------------
        bool chol_ok = true;
        for (int K = 0; K < Nl; ++K) {
          if (own && bI == K && bJ == K) {
            bool ok = true;
#pragma unroll
            for (int c = 0; c < MS; ++c) {
              double s = blk[c][c];
#pragma unroll
              for (int x = 0; x < c; ++x) s = fma(-blk[c][x], blk[c][x], s);
              if (!(s > 0.0) || !isfinite(s)) ok = false;
              const double lcc = sqrt(s);
              const double inv = 1.0 / lcc;
              blk[c][c] = lcc;
#pragma unroll
              for (int r = c + 1; r < MS; ++r) {
                double v = blk[r][c];
#pragma unroll
                for (int x = 0; x < c; ++x) v = fma(-blk[r][x], blk[c][x], v);
                blk[r][c] = v * inv;
              }
            }
            double* o = Ls + (size_t)t * TB;
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) o[LIDX(a, b)] = (b <= a) ? blk[a][b] : 0.0;
            ctl[1] = ok ? 0 : 1;
          }
          gsync();
          if (ctl[1]) {
            chol_ok = false;
            break;
          }
          const double* Lkk = Ls + (size_t)(K * (K + 1) / 2 + K) * TB;
          if (own && bJ == K && bI > K) {
            // X = A_IK L_KK^{-T}: x_c = (a_c - sum_{x<c} x_x L_KK[c][x]) / L_KK[c][c]
            double inv[MS];
#pragma unroll
            for (int c = 0; c < MS; ++c) inv[c] = 1.0 / Lkk[LIDX(c, c)];
#pragma unroll
            for (int r = 0; r < MS; ++r)
#pragma unroll
              for (int c = 0; c < MS; ++c) {
                double v = blk[r][c];
#pragma unroll
                for (int x = 0; x < c; ++x) v = fma(-blk[r][x], Lkk[LIDX(c, x)], v);
                blk[r][c] = v * inv[c];
              }
            double* o = Ls + (size_t)t * TB;
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) o[LIDX(a, b)] = blk[a][b];
          }
          gsync();
          if (own && bJ > K) {
            const double* Lik = Ls + (size_t)(bI * (bI + 1) / 2 + K) * TB;
            const double* Ljk = Ls + (size_t)(bJ * (bJ + 1) / 2 + K) * TB;
            // rank-1 updates by column x of L_IK and L_JK (contiguous in column-major blocks)
#pragma unroll
            for (int x = 0; x < MS; ++x) {
              double ci[MS], cj[MS];
#pragma unroll
              for (int a = 0; a < MS; ++a) {
                ci[a] = Lik[LIDX(a, x)];
                cj[a] = Ljk[LIDX(a, x)];
              }
#pragma unroll
              for (int r = 0; r < MS; ++r)
#pragma unroll
                for (int c = 0; c < MS; ++c) blk[r][c] = fma(-ci[r], cj[c], blk[r][c]);
            }
          }
        }
        if (!chol_ok) {
          status = 2;
          break;
        }
        // ---- triangular solves by warp 0: L y = -g, L^T d = y ---------------------------------
        if (wig == 0) {
          for (int r = lane; r < n; r += 32) dd[r] = -g[r];
          __syncwarp();
          for (int K = 0; K < Nl; ++K) {
            const double* Lkk = Ls + (size_t)(K * (K + 1) / 2 + K) * TB;
            double y[MS];
#pragma unroll
            for (int c = 0; c < MS; ++c) {
              double v = dd[K * MS + c];
#pragma unroll
              for (int x = 0; x < c; ++x) v = fma(-Lkk[LIDX(c, x)], y[x], v);
              y[c] = v / Lkk[LIDX(c, c)];
            }
            __syncwarp();
            if (lane < MS) {
#pragma unroll
              for (int c = 0; c < MS; ++c)
                if (c == lane) dd[K * MS + c] = y[c];
            }
            for (int e = lane; e < (Nl - 1 - K) * MS; e += 32) {
              const int I = K + 1 + e / MS, c = e - (e / MS) * MS;
              const double* Lik = Ls + (size_t)(I * (I + 1) / 2 + K) * TB;
              double v = dd[I * MS + c];
#pragma unroll
              for (int x = 0; x < MS; ++x) v = fma(-Lik[LIDX(c, x)], y[x], v);
              dd[I * MS + c] = v;
            }
            __syncwarp();
          }
          for (int K = Nl - 1; K >= 0; --K) {
            const double* Lkk = Ls + (size_t)(K * (K + 1) / 2 + K) * TB;
            double x_[MS];
#pragma unroll
            for (int c = MS - 1; c >= 0; --c) {
              double v = dd[K * MS + c];
#pragma unroll
              for (int x = c + 1; x < MS; ++x) v = fma(-Lkk[LIDX(x, c)], x_[x], v);
              x_[c] = v / Lkk[LIDX(c, c)];
            }
            __syncwarp();
            if (lane < MS) {
#pragma unroll
              for (int c = 0; c < MS; ++c)
                if (c == lane) dd[K * MS + c] = x_[c];
            }
            for (int e = lane; e < K * MS; e += 32) {
              const int J = e / MS, c = e - J * MS;
              const double* Lkj = Ls + (size_t)(K * (K + 1) / 2 + J) * TB;
              double v = dd[J * MS + c];
#pragma unroll
              for (int x = 0; x < MS; ++x) v = fma(-Lkj[LIDX(x, c)], x_[x], v);
              dd[J * MS + c] = v;
            }
            __syncwarp();
          }
        }
        gsync();
        // ---- Armijo backtracking on L (reading 3') ---------------------------------------------
        double slope, dummy;
        dot2(g, dd, n, slope, dummy);
        double alpha = 1.0;
        bool accepted = false;
        for (int h = 0; h <= P.nw.max_halvings; ++h) {
          for (int r = t; r < n; r += G) lt[r] = lam[r] + alpha * dd[r];
          gsync();
          double t1, t2;
          const bool okt = eval(lt, Nl, t1, t2);
          nb_is_lam = false;
          if (okt) {
            double d1, d2;
            dot2(lt, uh, n, d1, d2);
            const double Lt = t1 - d1;
            if (Lt <= L0 + P.nw.armijo_c * alpha * slope + 1e-12 * scale) {
              crit = grad(Nl);
              for (int r = t; r < n; r += G) lam[r] = lt[r];
              nb_is_lam = true;
              L0 = Lt;
              scale = t2 + d2;
              accepted = true;
              break;
            }
          }
          alpha *= 0.5;
        }
        if (!accepted) {
          status = 3;
          break;
        }
        ++l;
        gsync();
      }
    }
    // ---- epilogue ------------------------------------------------------------------------------
    gsync();
    if (!nb_is_lam && status != 4) {
      double t1, t2;
      eval(lam, Nl, t1, t2);
    }
    int Nnew = Nl;
    if (P.ad.n_levels > 0 && A.level_new) {
      const int Nprev = lvl > 0 ? P.ad.Nl[lvl - 1] : P.ad.Nprev0;
      double num = 0.0, den = 0.0;
      for (int i = t; i < Nl; i += G) {
        const double h = g[i * MS] + uh[i * MS];
        den = fma(h, h, den);
        if (i >= Nprev) num = fma(h, h, num);
      }
      gsum2(num, den);
      const double S = den > 0.0 ? num / den : 0.0;
      int nl = lvl;
      if (status == 0 || P.nw.mode == 1) {
        if (S < P.ad.delta_dec && lvl > 0)
          nl = lvl - 1;
        else if (S > P.ad.delta_inc && lvl < P.ad.n_levels - 1)
          nl = lvl + 1;
      }
      Nnew = P.ad.Nl[nl];
      if (t == 0) A.level_new[cell] = nl;
    }
    for (int r = t; r < nmax; r += G) gl[r] = (r < Nnew * MS) ? lam[r] : 0.0;
    if (t == 0) {
      if (A.iters) A.iters[cell] = l;
      if (A.status) A.status[cell] = status;
      if (A.crit) A.crit[cell] = crit;
      my_iters += l;
      if (status != 0) {
        my_failed += 1;
        my_worst = max(my_worst, status);
      }
    }
    if (status != 4) {
      for (int k = t; k < Q; k += G) {
        const double* u = nb + k * NS;
        if (A.uq) {
          double* o = A.uq + (cell * Q + k) * MS;
#pragma unroll
          for (int a = 0; a < MS; ++a) o[a] = u[a];
        }
        if (A.want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(u, P.mesh, cell, P.cl.gamma));
      }
    }
    gsync();
  }
  my_rate = warp_max(my_rate);
  if (lane == 0) {
    if (A.want_rate) atomicMax(&P.sc->rate_bits, (unsigned long long)__double_as_longlong(my_rate));
    if (t == 0) {
      if (my_iters) atomicAdd(&P.sc->newton_iters, (unsigned long long)my_iters);
      if (my_failed) atomicAdd(&P.sc->failed, (unsigned long long)my_failed);
      if (my_worst) atomicMax(&P.sc->worst, my_worst);
    }
  }
}

#undef LIDX
