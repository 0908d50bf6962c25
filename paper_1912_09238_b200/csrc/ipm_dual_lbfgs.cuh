// ipm_dual_lbfgs.cuh — quasi-Newton (limited-memory BFGS) dual solve, one warp per cell (sm_100a, fp64).
//
// SURVEY 8(f) NEXT-4; reading 35.  PAPER.md:843 proposes to replace the exact dual Hessian
// by BFGS approximations "which construct the Hessian from previously computed gradients", the
// gradients of old time steps kept in every spatial cell.  Per cell, the direction is
//   d = -H_l g,  H_l = the L-BFGS inverse-Hessian approximation (two-loop recursion) over the cell's
//                      last MH pairs s = lambda^{(l+1)} - lambda^{(l)}, y = g^{(l+1)} - g^{(l)},
//                      kept across (pseudo-)time steps in HBM,
//   initial matrix H0 = I_N (x) Jbar^{-1},  Jbar = sum_k omega_k grad u_s(Lambda_k)  (m x m),
// the exact inverse Hessian of a xi-independent state because <phi phi^T>_Q = I.
// Everything else is the Newton iteration of k_dual_mma: node pass, gradient on DMMA, Armijo on L
// with the rounding allowance (reading 3'), stopping test, epilogue.  Per iteration
// there is no Hessian and no Cholesky: the node pass, one DMMA gradient and 2 cnt dot products.
//
// Layout: one warp per cell (no group barriers), lanes own unknowns r = lane + 32 e (e < NR) for the
// vector work and the pairs, which live in REGISTERS (S, Y: MH x NR per lane, newest first; shifted
// on insertion so every index is a compile-time constant); lambda, trial, uhat, g, the direction and
// the node buffer u[a][k] live in the warp's shared-memory slice (the node pass reads lambda by
// broadcast).  Tables as k_dual_mma: Phi^T [N][QP], omega Phi^T in A-fragment order.
#pragma once
// (included inside namespace ipm by ipm_kernels.cu, after ipm_dual_mma.cuh)

template <int MS>
struct LbfgsLayout {
  // per warp: lam, lt, uh, g, q (direction / two-loop vector)  [5][NV]  + node buffer u [MS][Q]
  //           (+ the pairs S, Y [MH][NV] when they live in shared memory, PSM)
  static __host__ __device__ int per_warp(int NV, int Q, int pairs = 0) {
    return ((5 * NV + MS * Q + 2 * pairs * NV) + 1) & ~1;
  }
};

// PSM: the pairs in shared memory (fewer registers: 16 warps per SM) instead of registers (12 warps)
// QC, NC: compile-time Q and N of the launch (0 = from the tables at run time), as k_dual_mma's
// fixed-shape instances (loop bounds and tile counts fold to constants)
template <int CL, int MS, int NR, int MH, bool PSM, int QC = 0, int NC = 0>
__global__ void __launch_bounds__(PSM ? 512 : 384, 1) k_dual_lbfgs(DualParams P) {
  extern __shared__ __align__(16) double sm[];
  constexpr int MM = MS * (MS + 1) / 2;
  constexpr int NV = 32 * NR;
  const int N = NC ? NC : P.T.N, Q = QC ? QC : P.T.Q;
  const int QP = QC ? ((QC % 2) ? QC : QC + 1) : P.T.QP, KS = QC ? (QC + 3) / 4 : P.T.KS;
  double* sPhiT = sm;
  double* sWF = sm + N * QP;  // [MT][KS][32]
  const int MTT = NC ? (NC + 7) / 8 : P.T.MT;
  const int tabsz = (N * QP + MTT * KS * 32 + 1) & ~1;
  for (int x = threadIdx.x; x < N * QP; x += blockDim.x) sPhiT[x] = P.T.PhiT[x];
  for (int x = threadIdx.x; x < MTT * KS * 32; x += blockDim.x) sWF[x] = P.T.WPhiF[x];
  __syncthreads();
  const int wig = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* base = sm + tabsz + (size_t)wig * LbfgsLayout<MS>::per_warp(NV, Q, PSM ? MH : 0);
  double* lam = base;
  double* lt = lam + NV;
  double* uh = lt + NV;
  double* g = uh + NV;
  double* qv = g + NV;
  double* nb = qv + NV;  // u[a][k] at nb[a Q + k]
  double* sS = nb + MS * Q;  // PSM: [MH][NV], column r of lane r % 32
  double* sY = sS + MH * NV;

  const double* __restrict__ omega = P.T.omega;
  const DualLaunch& A = P.a;
  const int nmax = A.row ? A.row : N * MS;
  const int64_t ncells = A.ncells_dev ? (int64_t)*A.ncells_dev : A.cells;
  int* const queue = A.queue ? A.queue : &P.sc->work_counter;
  long long my_iters = 0, my_failed = 0;
  int my_worst = 0;
  double my_rate = 0.0;

  for (;;) {
    int ci = 0;
    if (lane == 0) ci = atomicAdd(queue, 1);
    ci = __shfl_sync(FULL_MASK, ci, 0);
    if (ci >= ncells) break;
    const int64_t cell = A.list ? (int64_t)A.list[ci] : (int64_t)ci;
    const int lvl = A.level ? A.level[cell] : 0;
    const int Nl = NC ? NC : ((P.ad.n_levels > 0 && !A.list) ? P.ad.Nl[lvl] : N);
    const int n = Nl * MS;
    // ---- load the cell: uhat, lambda, the L-BFGS history (pairs of another size are dropped) ----
    {
      const double* gu = A.uhat + cell * nmax;
      const double* gl = A.lam + cell * nmax;
      for (int r = lane; r < NV; r += 32) {
        uh[r] = r < n ? gu[r] : 0.0;
        lam[r] = r < n ? gl[r] : 0.0;
      }
    }
    int cnt = A.lb_cnt[cell];
    if (A.lb_n[cell] != n) cnt = 0;
    double rho[MH];
#define PS(i, e) (*(PSM ? &sS[(i) * NV + lane + 32 * (e)] : &S[PSM ? 0 : (i)][PSM ? 0 : (e)]))
#define PY(i, e) (*(PSM ? &sY[(i) * NV + lane + 32 * (e)] : &Y[PSM ? 0 : (i)][PSM ? 0 : (e)]))
    double S[PSM ? 1 : MH][PSM ? 1 : NR], Y[PSM ? 1 : MH][PSM ? 1 : NR];
    {
      const double* gS = A.lb_S + cell * (int64_t)MH * nmax;
      const double* gY = A.lb_Y + cell * (int64_t)MH * nmax;
#pragma unroll
      for (int i = 0; i < MH; ++i) {
        rho[i] = (i < cnt) ? A.lb_rho[cell * MH + i] : 0.0;
#pragma unroll
        for (int e = 0; e < NR; ++e) {
          const int r = lane + 32 * e;
          const bool v = i < cnt && r < n;
          PS(i, e) = v ? gS[(int64_t)i * nmax + r] : 0.0;
          PY(i, e) = v ? gY[(int64_t)i * nmax + r] : 0.0;
        }
      }
    }
    __syncwarp();

    int status = 0, l = 0, h = 0, mode = 0, hv = 0, ia = 0;
    double crit = INFINITY, L0 = 0.0, scale = 0.0, slope = 0.0, alpha = 1.0;
    bool nb_is_lam = false;
    double gold[NR], dreg[NR];
#pragma unroll
    for (int e = 0; e < NR; ++e) gold[e] = dreg[e] = 0.0;
    for (;;) {
      const double* x = (mode == 1) ? lt : lam;
      // ---- a2: Lambda = Phi x, u = u_s(Lambda), s_*, and the lane's part of sum_k omega_k J_k -------
      double sv0 = 0.0, sv1 = 0.0, jac[MM];
#pragma unroll
      for (int z = 0; z < MM; ++z) jac[z] = 0.0;
      bool bad = false;
      for (int k = lane; k < Q; k += 32) {
        double Lam[MS];
#pragma unroll
        for (int a = 0; a < MS; ++a) Lam[a] = 0.0;
#pragma unroll 4
        for (int i = 0; i < Nl; ++i) {
          const double ph = sPhiT[i * QP + k];
#pragma unroll
          for (int a = 0; a < MS; ++a) Lam[a] = fma(x[i * MS + a], ph, Lam[a]);
        }
        double u[MS], J[MM], ss;
        if (!Closure<CL, MS>::eval(Lam, u, J, ss, P.cl)) bad = true;
#pragma unroll
        for (int a = 0; a < MS; ++a) nb[a * Q + k] = u[a];
        const double w = omega[k];
#pragma unroll
        for (int z = 0; z < MM; ++z) jac[z] = fma(w, J[z], jac[z]);
        sv0 = fma(w, ss, sv0);
        sv1 = fma(w, fabs(ss), sv1);
      }
      if (bad) sv1 = INFINITY;
      double dv0 = 0.0, dv1 = 0.0;
#pragma unroll
      for (int e = 0; e < NR; ++e) {
        const int r = lane + 32 * e;
        const double v = x[r] * uh[r];  // zero beyond n
        dv0 += v;
        dv1 += fabs(v);
      }
      sv0 = warp_sum(sv0);
      sv1 = warp_sum(sv1);
      dv0 = warp_sum(dv0);
      dv1 = warp_sum(dv1);
      __syncwarp();  // node buffer complete
      if (mode == 2) {
        nb_is_lam = true;
        break;
      }
      const bool ok = isfinite(sv0) && isfinite(sv1);
      const double Lt = sv0 - dv0;
      bool accept;
      if (mode == 0) {
        if (!ok) {
          status = 4;
          break;
        }
        accept = true;
      } else {
        accept = ok && (Lt <= L0 + P.nw.armijo_c * alpha * slope + 1e-12 * scale);
      }
      bool finish = false;
      if (accept) {
        // ---- a3: gradient g = Phi^T (omega o u) - uhat on DMMA (A = omega Phi^T fragments) ----------
        double part[MS];
#pragma unroll
        for (int a = 0; a < MS; ++a) part[a] = 0.0;
        {
          const int MTl = (Nl + 7) >> 3, bn = lane >> 2, bk = lane & 3;
          const bool bval = bn < MS;
          const double* bsrc = nb + (bval ? bn : 0) * Q + bk;
#pragma unroll 1
          for (int mt = 0; mt < MTl; ++mt) {
            double c0 = 0.0, c1 = 0.0;
            const double* asrc = sWF + mt * KS * 32 + lane;
#pragma unroll 5
            for (int ks = 0; ks < KS; ++ks) {
              const double bv = (bval && 4 * ks + bk < Q) ? bsrc[4 * ks] : 0.0;
              dmma884(c0, c1, asrc[ks * 32], bv);
            }
            const int i = 8 * mt + (lane >> 2);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int a = 2 * (lane & 3) + e;
              if (a < MS && i < Nl) {
                const int rr = i * MS + a;
                const double gr = (e == 0 ? c0 : c1) - uh[rr];
                g[rr] = gr;
#pragma unroll
                for (int b = 0; b < MS; ++b)
                  if (b == a) part[b] = fma(gr, gr, part[b]);
              }
            }
          }
        }
        __syncwarp();
        double gr_[NR];
#pragma unroll
        for (int e = 0; e < NR; ++e) {
          const int r = lane + 32 * e;
          gr_[e] = r < n ? g[r] : 0.0;
        }
        if (mode == 1) {
          // accepted trial: pair s = lt - lam, y = g_new - g_old (reading 35), then lam = lt
          double sy = 0.0, ss2 = 0.0, yy = 0.0, sn[NR], yn[NR];
#pragma unroll
          for (int e = 0; e < NR; ++e) {
            const int r = lane + 32 * e;
            sn[e] = lt[r] - lam[r];
            yn[e] = gr_[e] - gold[e];
            sy = fma(sn[e], yn[e], sy);
            ss2 = fma(sn[e], sn[e], ss2);
            yy = fma(yn[e], yn[e], yy);
          }
          sy = warp_sum(sy);
          ss2 = warp_sum(ss2);
          yy = warp_sum(yy);
          if (sy > 1e-10 * sqrt(ss2 * yy)) {  // curvature condition with a rounding margin
#pragma unroll
            for (int i = MH - 1; i > 0; --i) {
              rho[i] = rho[i - 1];
#pragma unroll
              for (int e = 0; e < NR; ++e) {
                PS(i, e) = PS(i - 1, e);
                PY(i, e) = PY(i - 1, e);
              }
            }
            rho[0] = 1.0 / sy;
#pragma unroll
            for (int e = 0; e < NR; ++e) {
              PS(0, e) = sn[e];
              PY(0, e) = yn[e];
            }
            cnt = cnt < MH ? cnt + 1 : MH;
          }
#pragma unroll
          for (int e = 0; e < NR; ++e) {
            const int r = lane + 32 * e;
            lam[r] = lt[r];
          }
          ++l;
        }
#pragma unroll
        for (int e = 0; e < NR; ++e) gold[e] = gr_[e];
#pragma unroll
        for (int a = 0; a < MS; ++a) part[a] = warp_sum(part[a]);
        crit = 0.0;
#pragma unroll
        for (int a = 0; a < MS; ++a) crit += sqrt(part[a]);
        nb_is_lam = true;
        L0 = Lt;
        scale = sv1 + dv1;
        // ---- a7: stopping tests ---------------------------------------------------------------------
        if (crit < P.nw.tau || (P.nw.mode == 1 && l == 1)) break;
        if (l == P.nw.max_newton) {  // reading 35: Newton takes over (fallback pass)
          status = 1;
          break;
        }
        // ---- L-BFGS direction (two-loop recursion, H0 = I (x) Jbar^{-1}) ------------------------------
        double Jb[MM];
#pragma unroll
        for (int z = 0; z < MM; ++z) Jb[z] = warp_sum(jac[z]);
        // Cholesky of Jbar (m x m, every lane redundantly): Lc packed lower by rows
        double Lc[MS][MS], Li[MS];  // Cholesky factor of Jbar and the reciprocals of its diagonal
        bool spd = true;
#pragma unroll
        for (int j = 0; j < MS; ++j) {
          double t = Jb[sym_idx<MS>(j, j)];
#pragma unroll
          for (int k = 0; k < j; ++k) t = fma(-Lc[j][k], Lc[j][k], t);
          if (!(t > 0.0) || !isfinite(t)) spd = false;
          Lc[j][j] = sqrt(t);
          const double inv = 1.0 / Lc[j][j];
          Li[j] = inv;
#pragma unroll
          for (int i = j + 1; i < MS; ++i) {
            double v = Jb[sym_idx<MS>(j, i)];
#pragma unroll
            for (int k = 0; k < j; ++k) v = fma(-Lc[i][k], Lc[j][k], v);
            Lc[i][j] = v * inv;
          }
        }
        if (!spd) {
          status = 2;
          finish = true;
        } else {
          for (int pass = 0; pass < 2; ++pass) {
            // first loop, newest pair first
            double q[NR], al[MH];
#pragma unroll
            for (int e = 0; e < NR; ++e) q[e] = gr_[e];
#pragma unroll
            for (int i = 0; i < MH; ++i) {
              al[i] = 0.0;
              if (i < cnt) {
                double t = 0.0;
#pragma unroll
                for (int e = 0; e < NR; ++e) t = fma(PS(i, e), q[e], t);
                al[i] = rho[i] * warp_sum(t);
#pragma unroll
                for (int e = 0; e < NR; ++e) q[e] = fma(-al[i], PY(i, e), q[e]);
              }
            }
            // r = H0 q: Jbar r_i = q_i per moment i (the m states of moment i through shared memory)
#pragma unroll
            for (int e = 0; e < NR; ++e) qv[lane + 32 * e] = q[e];
            __syncwarp();
#pragma unroll
            for (int e = 0; e < NR; ++e) {
              const int r = lane + 32 * e;
              const int rc = r < n ? r : 0;  // (lanes beyond n: a valid moment, result discarded)
              const int i = rc / MS, a = rc - i * MS;
              double y[MS], z[MS];
#pragma unroll
              for (int b = 0; b < MS; ++b) {
                double v = qv[i * MS + b];
#pragma unroll
                for (int k = 0; k < b; ++k) v = fma(-Lc[b][k], y[k], v);
                y[b] = v * Li[b];
              }
#pragma unroll
              for (int b = MS - 1; b >= 0; --b) {
                double v = y[b];
#pragma unroll
                for (int k = b + 1; k < MS; ++k) v = fma(-Lc[k][b], z[k], v);
                z[b] = v * Li[b];
              }
              double rv = 0.0;
#pragma unroll
              for (int b = 0; b < MS; ++b)
                if (b == a) rv = z[b];
              q[e] = (r < n) ? rv : 0.0;
            }
            __syncwarp();
            // second loop, oldest pair first
#pragma unroll
            for (int i = MH - 1; i >= 0; --i) {
              if (i < cnt) {
                double t = 0.0;
#pragma unroll
                for (int e = 0; e < NR; ++e) t = fma(PY(i, e), q[e], t);
                const double be = rho[i] * warp_sum(t);
#pragma unroll
                for (int e = 0; e < NR; ++e) q[e] = fma(PS(i, e), al[i] - be, q[e]);
              }
            }
            double sl = 0.0;
#pragma unroll
            for (int e = 0; e < NR; ++e) {
              dreg[e] = -q[e];
              sl = fma(gr_[e], dreg[e], sl);
            }
            slope = warp_sum(sl);
            if (slope < 0.0 || cnt == 0) break;
            cnt = 0;  // not a descent direction (rounding): drop the history, H0 alone
          }
          alpha = 1.0;
          h = 0;
        }
      } else {
        nb_is_lam = false;
        ++hv;
        if (!ok) ++ia;
        alpha *= 0.5;
        if (++h > P.nw.max_halvings) {
          status = 3;
          finish = true;
        }
      }
      if (finish) {
        if (nb_is_lam) break;
        mode = 2;  // re-evaluate the last accepted iterate
      } else {
#pragma unroll
        for (int e = 0; e < NR; ++e) {
          const int r = lane + 32 * e;
          lt[r] = (r < n) ? lam[r] + alpha * dreg[e] : 0.0;
        }
        mode = 1;
      }
      __syncwarp();
    }
    __syncwarp();
    // ---- epilogue: level (adaptive), lambda, history, statistics, node states, CFL rate ------------
    if (P.ad.n_levels > 0 && A.level_new) {
      const int Nprev = lvl > 0 ? P.ad.Nl[lvl - 1] : P.ad.Nprev0;
      double nd0 = 0.0, nd1 = 0.0;
      for (int i = lane; i < Nl; i += 32) {
        const double hv_ = g[i * MS] + uh[i * MS];
        nd1 = fma(hv_, hv_, nd1);
        if (i >= Nprev) nd0 = fma(hv_, hv_, nd0);
      }
      nd0 = warp_sum(nd0);
      nd1 = warp_sum(nd1);
      const double Sv = nd1 > 0.0 ? nd0 / nd1 : 0.0;
      const int nl = next_level(P.ad, P.sc, lvl, status, Sv);
      if (lane == 0) A.level_new[cell] = nl;
    }
    {
      double* gl = A.lam + cell * nmax;
      for (int r = lane; r < nmax; r += 32) gl[r] = (r < n) ? lam[r] : 0.0;
      double* gS = A.lb_S + cell * (int64_t)MH * nmax;
      double* gY = A.lb_Y + cell * (int64_t)MH * nmax;
#pragma unroll
      for (int i = 0; i < MH; ++i) {
        if (i < cnt) {
#pragma unroll
          for (int e = 0; e < NR; ++e) {
            const int r = lane + 32 * e;
            if (r < n) {
              gS[(int64_t)i * nmax + r] = PS(i, e);
              gY[(int64_t)i * nmax + r] = PY(i, e);
            }
          }
          if (lane == 0) A.lb_rho[cell * MH + i] = rho[i];
        }
      }
      if (lane == 0) {
        A.lb_cnt[cell] = (status == 1 && A.fb_list != nullptr) ? 0 : cnt;
        A.lb_n[cell] = n;
      }
    }
    // reading 35: a cell at max_newton quasi-Newton steps goes to the Newton fallback pass, which does
    // its accounting (counts add up there) and its node states / CFL rate; its pairs are dropped
    const bool handoff = status == 1 && A.fb_list != nullptr;
    if (lane == 0) {
      if (handoff) {
        if (A.iters) A.iters[cell] = l;
        if (A.halv) A.halv[cell] = hv;
        if (A.inadm) A.inadm[cell] = ia;
        A.lb_cnt[cell] = 0;
        A.fb_list[atomicAdd(A.fb_count, 1)] = (int32_t)cell;
      } else {
        cell_stats(A, P.sc, cell, l, status, hv, ia, crit);
        if (status != 0) {
          my_failed += 1;
          my_worst = max(my_worst, status);
        }
      }
      my_iters += l;
    }
    for (int k = lane; k < Q && !handoff; k += 32) {  // node states at the final iterate (variant B)
      double u[MS];
#pragma unroll
      for (int a = 0; a < MS; ++a) u[a] = nb[a * Q + k];
      if (A.uq) {
        double* o = A.uq + cell * Q * MS + k;  // [cell][state][node]
#pragma unroll
        for (int a = 0; a < MS; ++a) o[a * Q] = u[a];
      }
      if (A.want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(u, P.mesh, cell, P.cl.gamma));
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
#undef PS
#undef PY

// ---- large cells (config 5: N = 56, m = 4, n = 224, Q = 10^3, p = 3) -------------------------------------
// The same quasi-Newton iteration (reading 35) with one CTA of NT threads per cell.  Thread t owns the
// unknown r = t (n <= NT) and its MH pairs in registers.  The node pass and the gradient are
// sum-factorised over the tensor Gauss-Legendre rule (the basis is a product of 1D orthonormal
// Legendre polynomials, the weights a product of 1D weights):
//   T1[i1 i2][k3] = sum_i3 lambda_(i1,i2,i3) L_i3(x_k3)      T2[i1][k2][k3] = sum_i2 T1[i1 i2][k3] L_i2(x_k2)
//   (stored state-major: T1[i1 i2][a][k3], T2[i1][a][k2][k3])
//   Lambda(k1,k2,k3) = sum_i1 T2[i1][k2][k3] L_i1(x_k1)
// and the transpose for g = Phi^T (omega o u) - uhat — about 35 k fmas each instead of 224 k, with
// 1D tables in shared memory instead of the 448 KB Phi read from L2.  Everything per cell lives in
// shared memory (~68 KB).  No adaptive levels (config 5 has none).
template <int MS>
struct LbfgsBigLayout {
  // doubles: vectors [5][n], u [MS][Q], T1 [npr2][q][MS], T2 [M+1][q][q][MS], L1 [M+1][q], w1h [q],
  // reductions [2][16][NW]; then ints: basis index of (i1, i2, i3) [(M+1)^3]
  static __host__ __device__ int doubles(int n, int Q, int M, int q, int NW) {
    const int npr2 = (M + 1) * (M + 2) / 2;
    const int t1 = npr2 * q * MS, t2 = (M + 1) * q * q * MS;
    return 5 * n + MS * Q + t1 + t2 + 2 * (M + 1) * q + q + 2 * 16 * NW + ((M + 1) * (M + 1) * (M + 1) + 1) / 2 + 8 +
           2 * 8 * n;  // + the pairs S, Y [MH <= 8][n]; WL1 [M+1][q] = (w_k / 2) L_i(x_k)
  }
};

// Q1, MD: compile-time 1D points and degree (config 5: 10, 5; 0 = from the tables): the stage loops'
// index arithmetic (divisions by q, m) folds to constants
template <int CL, int MS, int MH, int NT, int Q1 = 0, int MD = 0>
__global__ void __launch_bounds__(NT, 2) k_dual_lbfgs_big(DualParams P) {
  extern __shared__ __align__(16) double sm[];
  constexpr int MM = MS * (MS + 1) / 2, NW = NT / 32;
  const int q = Q1 ? Q1 : P.T.q1d, M = MD ? MD : P.T.npr1 - 1;  // npr1 = M + 1 (1D degrees)
  const int N = MD ? (MD + 1) * (MD + 2) * (MD + 3) / 6 : P.T.N, Q = Q1 ? Q1 * Q1 * Q1 : P.T.Q;
  const int n = N * MS, npr2 = (M + 1) * (M + 2) / 2;
  double* lam = sm;
  double* lt = lam + n;
  double* uh = lt + n;
  double* g = uh + n;
  double* qv = g + n;
  double* u = qv + n;                      // [MS][Q]
  // stage buffers state-major (a before the node index), so that consecutive threads, which walk the
  // node index, read consecutive doubles (with the state innermost the node pass read T2 at a 4-double
  // stride: 4-way bank conflicts)
  double* T1 = u + MS * Q;                 // [npr2][MS][q]  (also R2 of the gradient)
  double* T2 = T1 + npr2 * q * MS;         // [M+1][MS][q][q] (also R1)
  double* L1 = T2 + (M + 1) * q * q * MS;  // [M+1][q]
  double* w1h = L1 + (M + 1) * q;          // [q]
  double* WL1 = w1h + q;                   // [M+1][q] (w_k / 2) L_i(x_k): the gradient stages' 1D table
  // [2][16][NW], 16-byte aligned (double2 reads of the partials); the layout has slack for it
  double* red = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(WL1 + (M + 1) * q) + 15) & ~(uintptr_t)15);
  int* bidx = reinterpret_cast<int*>(red + 2 * 16 * NW);  // [(M+1)^3] -> basis index or -1
  // the cell's pairs, newest first, column t owned by thread t (shared memory: registers would spill)
  double* sS = red + 2 * 16 * NW + ((M + 1) * (M + 1) * (M + 1) + 1) / 2 + 8;  // [MH][n]
  double* sY = sS + MH * n;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int x = t; x < (M + 1) * q; x += NT) L1[x] = P.T.L1[x];
  for (int x = t; x < q; x += NT) w1h[x] = P.T.w1h[x];
  for (int x = t; x < (M + 1) * q; x += NT) WL1[x] = P.T.w1h[x % q] * P.T.L1[x];
  for (int x = t; x < (M + 1) * (M + 1) * (M + 1); x += NT) bidx[x] = -1;
  __syncthreads();
  for (int i = t; i < N; i += NT) bidx[(P.T.idx[i * 3] * (M + 1) + P.T.idx[i * 3 + 1]) * (M + 1) + P.T.idx[i * 3 + 2]] = i;
  __syncthreads();
  // pair (i1, i2), i1 + i2 <= M, enumerated i1-major: offset of i1's row
  auto prow = [&](int i1) { return i1 * (M + 1) - i1 * (i1 - 1) / 2; };
  int slot = 0;
  auto bsum = [&](double* v, int cnt) {  // block-wide sums of cnt (<= 16) values
    double* r = red + slot * 16 * NW;
    slot ^= 1;
    for (int a = 0; a < cnt; ++a) {
      const double s = warp_sum(v[a]);
      if (lane == 0) r[a * NW + wid] = s;
    }
    __syncthreads();
    for (int a = 0; a < cnt; ++a) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; w += 2) {
        const double2 x = *reinterpret_cast<const double2*>(r + a * NW + w);
        s += x.x + x.y;
      }
      v[a] = s;
    }
  };

  const DualLaunch& A = P.a;
  const int nmax = A.row ? A.row : n;
  const int64_t ncells = A.ncells_dev ? (int64_t)*A.ncells_dev : A.cells;
  int* const queue = A.queue ? A.queue : &P.sc->work_counter;
  long long my_iters = 0, my_failed = 0;
  int my_worst = 0;
  double my_rate = 0.0;
  __shared__ int s_ci;
  for (;;) {
    if (t == 0) s_ci = atomicAdd(queue, 1);
    __syncthreads();
    const int64_t ci = s_ci;
    __syncthreads();
    if (ci >= ncells) break;
    const int64_t cell = A.list ? (int64_t)A.list[ci] : ci;
    for (int r = t; r < n; r += NT) {
      uh[r] = A.uhat[cell * nmax + r];
      lam[r] = A.lam[cell * nmax + r];
    }
    int cnt = A.lb_cnt[cell];
    if (A.lb_n[cell] != n) cnt = 0;
    double rho[MH];
    const bool own = t < n;
#pragma unroll
    for (int i = 0; i < MH; ++i) {
      rho[i] = (i < cnt) ? A.lb_rho[cell * MH + i] : 0.0;
      if (own) {
        sS[i * n + t] = (i < cnt) ? A.lb_S[(cell * MH + i) * (int64_t)nmax + t] : 0.0;
        sY[i * n + t] = (i < cnt) ? A.lb_Y[(cell * MH + i) * (int64_t)nmax + t] : 0.0;
      }
    }
    __syncthreads();
    int status = 0, l = 0, h = 0, mode = 0, hv = 0, ia = 0;
    double crit = INFINITY, L0 = 0.0, scale = 0.0, slope = 0.0, alpha = 1.0, gold = 0.0, dreg = 0.0;
    bool nb_is_lam = false;
    for (;;) {
      const double* x = (mode == 1) ? lt : lam;
      // ---- a2 sum-factorised: stages A, B into T1, T2; stage C + closure per node ----------------------
      for (int o = t; o < npr2 * q * MS; o += NT) {
        const int k3 = o % q, a = (o / q) % MS, pr = o / (MS * q);
        int i1 = 0;
        while (pr >= prow(i1 + 1)) ++i1;
        const int i2 = pr - prow(i1);
        double s = 0.0;
        for (int i3 = 0; i3 <= M - i1 - i2; ++i3) {
          const int bi = bidx[(i1 * (M + 1) + i2) * (M + 1) + i3];
          s = fma(x[bi * MS + a], L1[i3 * q + k3], s);
        }
        T1[o] = s;
      }
      __syncthreads();
      for (int o = t; o < (M + 1) * q * q * MS; o += NT) {
        const int k3 = o % q, k2 = (o / q) % q, a = (o / (q * q)) % MS, i1 = o / (MS * q * q);
        double s = 0.0;
        for (int i2 = 0; i2 <= M - i1; ++i2) s = fma(T1[((prow(i1) + i2) * MS + a) * q + k3], L1[i2 * q + k2], s);
        T2[o] = s;
      }
      __syncthreads();
      double sv[2] = {0.0, 0.0}, jac[MM];
#pragma unroll
      for (int z = 0; z < MM; ++z) jac[z] = 0.0;
      bool bad = false;
      for (int k = t; k < Q; k += NT) {
        const int k1 = k / (q * q), k23 = k - k1 * q * q;
        double Lam[MS];
#pragma unroll
        for (int a = 0; a < MS; ++a) Lam[a] = 0.0;
        for (int i1 = 0; i1 <= M; ++i1) {
          const double lv = L1[i1 * q + k1];
#pragma unroll
          for (int a = 0; a < MS; ++a) Lam[a] = fma(T2[(i1 * MS + a) * q * q + k23], lv, Lam[a]);
        }
        double uk[MS], J[MM], ss;
        if (!Closure<CL, MS>::eval(Lam, uk, J, ss, P.cl)) bad = true;
#pragma unroll
        for (int a = 0; a < MS; ++a) u[a * Q + k] = uk[a];
        const double w = P.T.omega[k];
#pragma unroll
        for (int z = 0; z < MM; ++z) jac[z] = fma(w, J[z], jac[z]);
        sv[0] = fma(w, ss, sv[0]);
        sv[1] = fma(w, fabs(ss), sv[1]);
      }
      if (bad) sv[1] = INFINITY;
      double red4[4] = {sv[0], sv[1], 0.0, 0.0};
      if (own) {
        const double v = x[t] * uh[t];
        red4[2] = v;
        red4[3] = fabs(v);
      }
      bsum(red4, 4);  // (its barrier also completes the node buffer)
      if (mode == 2) {
        nb_is_lam = true;
        break;
      }
      const bool ok = isfinite(red4[0]) && isfinite(red4[1]);
      const double Lt = red4[0] - red4[2];
      bool accept;
      if (mode == 0) {
        if (!ok) {
          status = 4;
          break;
        }
        accept = true;
      } else {
        accept = ok && (Lt <= L0 + P.nw.armijo_c * alpha * slope + 1e-12 * scale);
      }
      bool finish = false;
      if (accept) {
        // ---- a3 sum-factorised: R1 (into T2), R2 (into T1), g ----------------------------------------
        for (int o = t; o < (M + 1) * q * q * MS; o += NT) {
          const int k23 = o % (q * q), a = (o / (q * q)) % MS, i1 = o / (MS * q * q);
          double s = 0.0;
          for (int k1 = 0; k1 < q; ++k1) s = fma(WL1[i1 * q + k1], u[a * Q + k1 * q * q + k23], s);
          T2[o] = s;
        }
        __syncthreads();
        for (int o = t; o < npr2 * q * MS; o += NT) {
          const int k3 = o % q, a = (o / q) % MS, pr = o / (MS * q);
          int i1 = 0;
          while (pr >= prow(i1 + 1)) ++i1;
          const int i2 = pr - prow(i1);
          double s = 0.0;
          for (int k2 = 0; k2 < q; ++k2) s = fma(WL1[i2 * q + k2], T2[((i1 * MS + a) * q + k2) * q + k3], s);
          T1[o] = s;
        }
        __syncthreads();
        double gr = 0.0;
        if (own) {
          const int i = t / MS, a = t - i * MS;
          const int i1 = P.T.idx[i * 3], i2 = P.T.idx[i * 3 + 1], i3 = P.T.idx[i * 3 + 2];
          double s = 0.0;
          for (int k3 = 0; k3 < q; ++k3) s = fma(WL1[i3 * q + k3], T1[((prow(i1) + i2) * MS + a) * q + k3], s);
          gr = s - uh[t];
          g[t] = gr;
        }
        double part[MS + 3];
#pragma unroll
        for (int a = 0; a < MS + 3; ++a) part[a] = 0.0;
        if (own) {
          const int a = t % MS;
#pragma unroll
          for (int b = 0; b < MS; ++b)
            if (b == a) part[b] = gr * gr;
        }
        if (mode == 1) {  // accepted trial: the pair (reading 35), then lambda = trial
          const double sn = own ? lt[t] - lam[t] : 0.0, yn = own ? gr - gold : 0.0;
          part[MS] = sn * yn;
          part[MS + 1] = sn * sn;
          part[MS + 2] = yn * yn;
          bsum(part, MS + 3);
          if (part[MS] > 1e-10 * sqrt(part[MS + 1] * part[MS + 2])) {
#pragma unroll
            for (int i = MH - 1; i > 0; --i) {
              rho[i] = rho[i - 1];
              if (own) {
                sS[i * n + t] = sS[(i - 1) * n + t];
                sY[i * n + t] = sY[(i - 1) * n + t];
              }
            }
            rho[0] = 1.0 / part[MS];
            if (own) {
              sS[t] = sn;
              sY[t] = yn;
            }
            cnt = cnt < MH ? cnt + 1 : MH;
          }
          if (own) lam[t] = lt[t];
          ++l;
        } else {
          bsum(part, MS);
        }
        gold = gr;
        crit = 0.0;
#pragma unroll
        for (int a = 0; a < MS; ++a) crit += sqrt(part[a]);
        nb_is_lam = true;
        L0 = Lt;
        scale = red4[1] + red4[3];
        if (crit < P.nw.tau || (P.nw.mode == 1 && l == 1)) break;
        if (l == P.nw.max_newton) {  // reading 35: Newton takes over (fallback pass)
          status = 1;
          break;
        }
        // ---- L-BFGS direction: Jbar, two-loop recursion ----------------------------------------------
        bsum(jac, MM);
        double Lc[MS][MS], Li[MS];  // Cholesky factor of Jbar and the reciprocals of its diagonal
        bool spd = true;
#pragma unroll
        for (int j = 0; j < MS; ++j) {
          double tt = jac[sym_idx<MS>(j, j)];
#pragma unroll
          for (int kk = 0; kk < j; ++kk) tt = fma(-Lc[j][kk], Lc[j][kk], tt);
          if (!(tt > 0.0) || !isfinite(tt)) spd = false;
          Lc[j][j] = sqrt(tt);
          const double inv = 1.0 / Lc[j][j];
          Li[j] = inv;
#pragma unroll
          for (int i = j + 1; i < MS; ++i) {
            double v = jac[sym_idx<MS>(j, i)];
#pragma unroll
            for (int kk = 0; kk < j; ++kk) v = fma(-Lc[i][kk], Lc[j][kk], v);
            Lc[i][j] = v * inv;
          }
        }
        if (!spd) {
          status = 2;
          finish = true;
        } else {
          for (int pass = 0; pass < 2; ++pass) {
            double qq = gr, al[MH];
#pragma unroll
            for (int i = 0; i < MH; ++i) {
              al[i] = 0.0;
              if (i < cnt) {
                double tt[1] = {own ? sS[i * n + t] * qq : 0.0};
                bsum(tt, 1);
                al[i] = rho[i] * tt[0];
                if (own) qq = fma(-al[i], sY[i * n + t], qq);
              }
            }
            if (own) qv[t] = qq;
            __syncthreads();
            double rv = 0.0;
            if (own) {
              const int i = t / MS, a = t - i * MS;
              double y[MS], z[MS];
#pragma unroll
              for (int b = 0; b < MS; ++b) {
                double v = qv[i * MS + b];
#pragma unroll
                for (int kk = 0; kk < b; ++kk) v = fma(-Lc[b][kk], y[kk], v);
                y[b] = v * Li[b];
              }
#pragma unroll
              for (int b = MS - 1; b >= 0; --b) {
                double v = y[b];
#pragma unroll
                for (int kk = b + 1; kk < MS; ++kk) v = fma(-Lc[kk][b], z[kk], v);
                z[b] = v * Li[b];
              }
#pragma unroll
              for (int b = 0; b < MS; ++b)
                if (b == a) rv = z[b];
            }
            qq = rv;
#pragma unroll
            for (int i = MH - 1; i >= 0; --i) {
              if (i < cnt) {
                double tt[1] = {own ? sY[i * n + t] * qq : 0.0};
                bsum(tt, 1);
                if (own) qq = fma(sS[i * n + t], al[i] - rho[i] * tt[0], qq);
              }
            }
            dreg = -qq;
            double sl[1] = {own ? gr * dreg : 0.0};
            bsum(sl, 1);
            slope = sl[0];
            if (slope < 0.0 || cnt == 0) break;
            cnt = 0;  // not a descent direction (rounding): drop the history, H0 alone
          }
          alpha = 1.0;
          h = 0;
        }
      } else {
        nb_is_lam = false;
        ++hv;
        if (!ok) ++ia;
        alpha *= 0.5;
        if (++h > P.nw.max_halvings) {
          status = 3;
          finish = true;
        }
      }
      if (finish) {
        if (nb_is_lam) break;
        mode = 2;
      } else {
        if (own) lt[t] = lam[t] + alpha * dreg;
        mode = 1;
      }
      __syncthreads();
    }
    __syncthreads();
    const bool handoff = status == 1 && A.fb_list != nullptr;
    for (int r = t; r < nmax; r += NT) A.lam[cell * nmax + r] = (r < n) ? lam[r] : 0.0;
#pragma unroll
    for (int i = 0; i < MH; ++i)
      if (i < cnt && own) {
        A.lb_S[(cell * MH + i) * (int64_t)nmax + t] = sS[i * n + t];
        A.lb_Y[(cell * MH + i) * (int64_t)nmax + t] = sY[i * n + t];
      }
    if (t == 0) {
      for (int i = 0; i < cnt; ++i) A.lb_rho[cell * MH + i] = rho[i];
      A.lb_cnt[cell] = handoff ? 0 : cnt;
      A.lb_n[cell] = n;
      if (handoff) {
        if (A.iters) A.iters[cell] = l;
        if (A.halv) A.halv[cell] = hv;
        if (A.inadm) A.inadm[cell] = ia;
        A.fb_list[atomicAdd(A.fb_count, 1)] = (int32_t)cell;
      } else {
        cell_stats(A, P.sc, cell, l, status, hv, ia, crit);
        if (status != 0) {
          my_failed += 1;
          my_worst = max(my_worst, status);
        }
      }
      my_iters += l;
    }
    for (int k = t; k < Q && !handoff; k += NT) {  // node states at the final iterate
      double uk[MS];
#pragma unroll
      for (int a = 0; a < MS; ++a) uk[a] = u[a * Q + k];
      if (A.uq) {
#pragma unroll
        for (int a = 0; a < MS; ++a) A.uq[cell * Q * MS + a * Q + k] = uk[a];
      }
      if (A.want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(uk, P.mesh, cell, P.cl.gamma));
    }
    __syncthreads();
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
