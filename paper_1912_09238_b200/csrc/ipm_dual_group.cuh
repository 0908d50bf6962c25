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
#ifndef IPM_GROUP_THREADS
#define IPM_GROUP_THREADS 512  // CTA size bound: 512 -> <= 128 registers / thread
#endif
// (included inside namespace ipm by ipm_kernels.cu, after DualParams and node_rate)

template <int MS>
struct GroupLayout {
  static constexpr int MM = MS * (MS + 1) / 2;
  // node-buffer row stride: even (16-byte aligned rows for vector loads), not a multiple of 16 doubles
  static constexpr int NS0 = (MS + MM + 1) & ~1;
  static constexpr int NS = (NS0 % 16 == 0) ? NS0 + 2 : NS0;
  static constexpr int TB = MS * MS;  // doubles per block (stored column-major)
  // block stride in shared memory: padded so that lanes reading the same element of different
  // blocks fall into different banks (a 128-byte stride would put them all in one bank)
  static constexpr int TBP = (TB % 2 == 0) ? ((TB % 16 == 0) ? TB + 2 : TB) : TB + 1;
  static constexpr int RS = MS > 2 ? MS : 2;  // values per reduction slot
  // doubles per group: 5 vectors + node buffer / L blocks / sum-factorisation stage + reduction + control
  //   direct (SF = 0): union(node buffer, L blocks)
  //   SF > 0:          node buffer, then union(T stage [q][npr][MM], L blocks)
  // sum factorisation builds T_ab[k1][pr][ab] in NCH chunks of CHW ab-components so that
  // (node buffer + one T chunk) fits where the L blocks go later
  static constexpr int NCH = (MM >= 6) ? 2 : 1;
  static constexpr int CHW = (MM + NCH - 1) / NCH;
  static __host__ __device__ int region(int N, int Q, int SF, int q1d) {
    const int NP = N * (N + 1) / 2;
    const int nb = Q * NS, lb = NP * TBP;
    const int used = (SF == 0) ? nb : nb + q1d * (SF * (SF + 1) / 2) * CHW;
    return used > lb ? used : lb;
  }
  static __host__ __device__ int per_group(int N, int Q, int G, int SF = 0, int q1d = 0) {
    const int n = N * MS;
    int w = 5 * n + region(N, Q, SF, q1d) + N * TBP + 2 * RS * (G / 32) + 4;
    return (w + 1) & ~1;
  }
};

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

#ifdef IPM_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[8];
#define PHASE_MARK(i)                                  \
  do {                                                 \
    const long long now_ = clock64();                  \
    if (t == 0) ph_acc[i] += (unsigned long long)(now_ - ph_t0); \
    ph_t0 = now_;                                      \
  } while (0)
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#endif

template <int CL, int MS, int G, int SF, int T>
__global__ void __launch_bounds__(IPM_GROUP_THREADS) k_dual_group(DualParams P) {
#ifdef IPM_PHASE_TIMERS
  unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t0 = clock64();
#endif
  using Lay = GroupLayout<MS>;
  constexpr int NW = G / 32;
  constexpr int MM = Lay::MM, NS = Lay::NS, TB = Lay::TBP;
#define LIDX(a, b) ((b) * MS + (a))  // element (a, b) of a column-major block
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, Q = P.T.Q, QP = P.T.QP;
  double* sPhiT = sm;
  double* sWPhiT = sm + N * QP;
  constexpr int NPR = SF * (SF + 1) / 2;
  double* sLL = sm + 2 * N * QP;  // [q1d][NPR] (SF > 0)
  const int q1 = P.T.q1d;
  const int tabsz = 2 * N * QP + ((SF > 0) ? ((q1 * NPR + 1) & ~1) : 0);
  for (int x = threadIdx.x; x < N * QP; x += blockDim.x) {
    sPhiT[x] = P.T.PhiT[x];
    sWPhiT[x] = P.T.WPhiT[x];
  }
  if (SF > 0)
    for (int x = threadIdx.x; x < q1 * NPR; x += blockDim.x) sLL[x] = P.T.LL[x];
  __syncthreads();
  const int grp = threadIdx.x / G, t = threadIdx.x - grp * G;
  const int wig = t >> 5, lane = t & 31;
  const int bar = 1 + grp;
  const int nmax = N * MS;
  double* base = sm + tabsz + (size_t)grp * Lay::per_group(N, Q, G, SF, q1);
  double* lam = base;
  double* lt = lam + nmax;
  double* uh = lt + nmax;
  double* g = uh + nmax;
  double* dd = g + nmax;
  double* nb = dd + nmax;                   // node buffer
  double* Ls = nb;           // L blocks (union with the node buffer and the T stage)
  double* Tt = nb + Q * NS;  // sum-factorisation stage chunk T[k1][pr][c] (SF > 0)
  double* Linv = nb + Lay::region(N, Q, SF, q1);  // [N] inverses of the diagonal Cholesky blocks
  double* red = Linv + (size_t)N * TB;  // [2 slots][RS][NW]
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

  // blocks (I, J) owned by this thread: rank r = t + s G in the order J descending, then I
  // ascending.  The blocks still updated in late Cholesky steps (large J) are then packed into the
  // first threads, so the other warps skip those phases instead of issuing them for idle lanes.
  // Shared-memory blocks are stored at the row-major lower index I(I+1)/2 + J.
  int bIa[T], bJa[T];
  auto assign_blocks = [&](int Nl) {
#pragma unroll
    for (int q = 0; q < T; ++q) {
      int r = t + q * G, J = Nl - 1;
      while (J > 0 && r >= Nl - J) {
        r -= Nl - J;
        --J;
      }
      bJa[q] = J;
      bIa[q] = J + r;
    }
  };

  for (;;) {
    if (t == 0) ctl[0] = atomicAdd(&P.sc->work_counter, 1);
    gsync();
    const int64_t cell = ctl[0];
    if (cell >= A.cells) break;
    PHASE_MARK(7);
    const int lvl = A.level ? A.level[cell] : 0;
    const int Nl = (P.ad.n_levels > 0) ? P.ad.Nl[lvl] : N;
    const int n = Nl * MS;
    const int NPl = Nl * (Nl + 1) / 2;
    bool owna[T];
#pragma unroll
    for (int q = 0; q < T; ++q) owna[q] = (t + q * G) < NPl;
    assign_blocks(Nl);
    const double* gu = A.uhat + cell * nmax;
    double* gl = A.lam + cell * nmax;
    for (int r = t; r < n; r += G) {
      uh[r] = gu[r];
      lam[r] = gl[r];
    }
    gsync();

    int status = 0, l = 0, hv = 0, ia = 0;
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
        PHASE_MARK(0);  // eval / gradient / line search of the previous iteration
        // ---- Hessian block in registers -------------------------------------------------------
        double blk[T][MS][MS];
        if constexpr (SF > 0) {
          // sum factorisation over the tensor rule (p = 2), k = k1 q + k2, in ab-chunks:
          //   T_ab[k1][(i2,j2)] = sum_k2 LL[k2][(i2,j2)] J_ab(k1,k2)
          //   H_ab[I][J]       = sum_k1 LL[k1][(i1,j1)] T_ab[k1][(i2,j2)]
          constexpr int NCH = Lay::NCH, CHW = Lay::CHW;
          double acc[T][MM];
#pragma unroll
          for (int q = 0; q < T; ++q)
#pragma unroll
            for (int z = 0; z < MM; ++z) acc[q][z] = 0.0;
          int pr1[T], pr2[T];
#pragma unroll
          for (int q = 0; q < T; ++q) {
            const int I = owna[q] ? bIa[q] : 0, J = owna[q] ? bJa[q] : 0;
            int a1 = P.T.idx[I * 2], a2 = P.T.idx[I * 2 + 1], b1 = P.T.idx[J * 2], b2 = P.T.idx[J * 2 + 1];
            if (a1 > b1) { const int x = a1; a1 = b1; b1 = x; }
            if (a2 > b2) { const int x = a2; a2 = b2; b2 = x; }
            pr1[q] = a1 * SF - a1 * (a1 - 1) / 2 + (b1 - a1);
            pr2[q] = a2 * SF - a2 * (a2 - 1) / 2 + (b2 - a2);
          }
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int ab0 = ch * CHW;
            const int nab = (MM - ab0) < CHW ? (MM - ab0) : CHW;
            for (int e = t; e < q1 * nab; e += G) {
              const int k1 = e / nab, c = e - k1 * nab;
              double at[NPR];
#pragma unroll
              for (int pr = 0; pr < NPR; ++pr) at[pr] = 0.0;
              const double* jrow = nb + (k1 * q1) * NS + MS + ab0 + c;
              for (int k2 = 0; k2 < q1; ++k2) {
                const double jv = jrow[k2 * NS];
                const double* ll = sLL + k2 * NPR;
#pragma unroll
                for (int pr = 0; pr < NPR; ++pr) at[pr] = fma(ll[pr], jv, at[pr]);
              }
#pragma unroll
              for (int pr = 0; pr < NPR; ++pr) Tt[(k1 * NPR + pr) * CHW + c] = at[pr];
            }
            gsync();
#pragma unroll
            for (int q = 0; q < T; ++q) {
              if (!owna[q]) continue;
              for (int k1 = 0; k1 < q1; ++k1) {
                const double lv = sLL[k1 * NPR + pr1[q]];
                const double* Tk = Tt + (k1 * NPR + pr2[q]) * CHW;
#pragma unroll
                for (int c = 0; c < CHW; ++c)
                  if (ab0 + c < MM) acc[q][ab0 + c] = fma(lv, Tk[c], acc[q][ab0 + c]);
              }
            }
            if (ch + 1 < NCH) gsync();  // T chunk is rewritten by the next chunk
          }
#pragma unroll
          for (int q = 0; q < T; ++q)
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b)
                blk[q][a][b] = acc[q][a <= b ? sym_idx<MS>(a, b) : sym_idx<MS>(b, a)];
        } else {
          // direct: H_IJ = sum_k (omega_k phi_kI phi_kJ) J_k; the J_k row is loaded once for all of
          // this thread's blocks
          double acc[T][MM];
#pragma unroll
          for (int q = 0; q < T; ++q)
#pragma unroll
            for (int z = 0; z < MM; ++z) acc[q][z] = 0.0;
          const double* wi[T];
          const double* pj[T];
#pragma unroll
          for (int q = 0; q < T; ++q) {
            wi[q] = sWPhiT + (owna[q] ? bIa[q] : 0) * QP;
            pj[q] = sPhiT + (owna[q] ? bJa[q] : 0) * QP;
          }
          for (int k = 0; k < Q; ++k) {
            const double* Jk = nb + k * NS + MS;
            double jv[MM];
#pragma unroll
            for (int z = 0; z < MM; ++z) jv[z] = Jk[z];
#pragma unroll
            for (int q = 0; q < T; ++q) {
              const double f = wi[q][k] * pj[q][k];
#pragma unroll
              for (int z = 0; z < MM; ++z) acc[q][z] = fma(f, jv[z], acc[q][z]);
            }
          }
#pragma unroll
          for (int q = 0; q < T; ++q)
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b)
                blk[q][a][b] = acc[q][a <= b ? sym_idx<MS>(a, b) : sym_idx<MS>(b, a)];
        }
        for (int r = t; r < n; r += G) dd[r] = -g[r];
        gsync();  // node buffer / T stage dead from here: L blocks reuse them
        PHASE_MARK(1);
        // ---- blocked Cholesky with the forward solve folded in ---------------------------------
        // step K: (1) owner of (K,K): L_KK = chol(A_KK), Linv_K = L_KK^{-1}, y_K = Linv_K b_K
        //         (2) owners of (I,K), I > K: L_IK = A_IK Linv_K^T, b_I -= L_IK y_K
        //         (3) owners of (I,J), I >= J > K: A_IJ -= L_IK L_JK^T
        // b = -g lives in dd and becomes y = L^{-1}(-g) in place.
        // diagonal step: owner of (K,K) factors its (fully updated) block, publishes L_KK and
        // Linv_K, and turns b_K into y_K = Linv_K b_K.  Called for K = 0 up front and for K + 1
        // inside the trailing phase of step K (look-ahead), right after that block's own update.
        auto diag_step = [&](int q, int K) {
          bool ok = true;
          double inv[MS];
#pragma unroll
          for (int c = 0; c < MS; ++c) {
            double sv = blk[q][c][c];
#pragma unroll
            for (int x = 0; x < c; ++x) sv = fma(-blk[q][c][x], blk[q][c][x], sv);
            if (!(sv > 0.0) || !isfinite(sv)) ok = false;
            const double rs = rsqrt(sv);
            inv[c] = rs;
            blk[q][c][c] = sv * rs;
#pragma unroll
            for (int r = c + 1; r < MS; ++r) {
              double v = blk[q][r][c];
#pragma unroll
              for (int x = 0; x < c; ++x) v = fma(-blk[q][r][x], blk[q][c][x], v);
              blk[q][r][c] = v * rs;
            }
          }
          // Linv (lower): Linv[c][c] = 1/L[c][c]; Linv[r][c] = -Linv[r][r] sum_{x=c}^{r-1} L[r][x] Linv[x][c]
          double li[MS][MS];
#pragma unroll
          for (int c = 0; c < MS; ++c) {
            li[c][c] = inv[c];
#pragma unroll
            for (int r = c + 1; r < MS; ++r) {
              double v = 0.0;
#pragma unroll
              for (int x = c; x < r; ++x) v = fma(blk[q][r][x], li[x][c], v);
              li[r][c] = -inv[r] * v;
            }
          }
          double* o = Ls + (size_t)(bIa[q] * (bIa[q] + 1) / 2 + bJa[q]) * TB;
          double* oi = Linv + (size_t)K * TB;
#pragma unroll
          for (int aa = 0; aa < MS; ++aa)
#pragma unroll
            for (int bb = 0; bb < MS; ++bb) {
              o[LIDX(aa, bb)] = (bb <= aa) ? blk[q][aa][bb] : 0.0;
              oi[LIDX(aa, bb)] = (bb <= aa) ? li[aa][bb] : 0.0;
            }
          double bk[MS];
#pragma unroll
          for (int aa = 0; aa < MS; ++aa) bk[aa] = dd[K * MS + aa];
#pragma unroll
          for (int aa = 0; aa < MS; ++aa) {
            double v = 0.0;
#pragma unroll
            for (int x = 0; x <= aa; ++x) v = fma(li[aa][x], bk[x], v);
            dd[K * MS + aa] = v;
          }
          ctl[1] = ok ? 0 : 1;
        };
        bool chol_ok = true;
#pragma unroll
        for (int q = 0; q < T; ++q)
          if (owna[q] && bIa[q] == 0 && bJa[q] == 0) diag_step(q, 0);
        gsync();
        for (int K = 0; K < Nl; ++K) {
          if (ctl[1]) {
            chol_ok = false;
            break;
          }
          // (2) panel
          const double* Li = Linv + (size_t)K * TB;
#pragma unroll
          for (int q = 0; q < T; ++q) {
            if (!(owna[q] && bJa[q] == K && bIa[q] > K)) continue;
            double X[MS][MS];
#pragma unroll
            for (int r = 0; r < MS; ++r)
#pragma unroll
              for (int c = 0; c < MS; ++c) {
                double v = 0.0;
#pragma unroll
                for (int x = 0; x <= c; ++x) v = fma(blk[q][r][x], Li[LIDX(c, x)], v);
                X[r][c] = v;
              }
            double yk[MS];
#pragma unroll
            for (int x = 0; x < MS; ++x) yk[x] = dd[K * MS + x];
            double* o = Ls + (size_t)(bIa[q] * (bIa[q] + 1) / 2 + bJa[q]) * TB;
            const int bI = bIa[q];
#pragma unroll
            for (int r = 0; r < MS; ++r) {
              double v = dd[bI * MS + r];
#pragma unroll
              for (int c = 0; c < MS; ++c) {
                o[LIDX(r, c)] = X[r][c];
                v = fma(-X[r][c], yk[c], v);
              }
              dd[bI * MS + r] = v;
            }
          }
          gsync();
          // (3) trailing update; the owner of (K+1,K+1) then factors it at once (look-ahead)
#pragma unroll
          for (int q = 0; q < T; ++q) {
            if (!(owna[q] && bJa[q] > K)) continue;
            const double* Lik = Ls + (size_t)(bIa[q] * (bIa[q] + 1) / 2 + K) * TB;
            const double* Ljk = Ls + (size_t)(bJa[q] * (bJa[q] + 1) / 2 + K) * TB;
#pragma unroll
            for (int x = 0; x < MS; ++x) {
              double ci[MS], cj[MS];
#pragma unroll
              for (int aa = 0; aa < MS; ++aa) {
                ci[aa] = Lik[LIDX(aa, x)];
                cj[aa] = Ljk[LIDX(aa, x)];
              }
#pragma unroll
              for (int r = 0; r < MS; ++r)
#pragma unroll
                for (int c = 0; c < MS; ++c) blk[q][r][c] = fma(-ci[r], cj[c], blk[q][r][c]);
            }
            if (bIa[q] == K + 1 && bJa[q] == K + 1) diag_step(q, K + 1);
          }
          gsync();
        }
        if (!chol_ok) {
          status = 2;
          break;
        }
        PHASE_MARK(2);
        // ---- back substitution L^T d = y by warp 0 (column oriented, Linv_K^T per block) ------
        if (wig == 0) {
          for (int K = Nl - 1; K >= 0; --K) {
            const double* Li = Linv + (size_t)K * TB;
            double dk[MS];
#pragma unroll
            for (int c = 0; c < MS; ++c) {
              double v = 0.0;
#pragma unroll
              for (int x = c; x < MS; ++x) v = fma(Li[LIDX(x, c)], dd[K * MS + x], v);
              dk[c] = v;
            }
            __syncwarp();
            if (lane < MS) {
#pragma unroll
              for (int c = 0; c < MS; ++c)
                if (c == lane) dd[K * MS + c] = dk[c];
            }
            for (int e = lane; e < K * MS; e += 32) {
              const int J = e / MS, c = e - J * MS;
              const double* Lkj = Ls + (size_t)(K * (K + 1) / 2 + J) * TB;
              double v = dd[J * MS + c];
#pragma unroll
              for (int x = 0; x < MS; ++x) v = fma(-Lkj[LIDX(x, c)], dk[x], v);
              dd[J * MS + c] = v;
            }
            __syncwarp();
          }
        }
        gsync();
        PHASE_MARK(3);
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
          ++hv;
          if (!okt) ++ia;
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
    PHASE_MARK(4);
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
      const int nl = next_level(P.ad, P.sc, lvl, status, S);
      Nnew = P.ad.Nl[nl];
      if (t == 0) A.level_new[cell] = nl;
    }
    for (int r = t; r < nmax; r += G) gl[r] = (r < n) ? lam[r] : 0.0;  // truncated to the new level after the flux
    if (t == 0) {
      cell_stats(A, P.sc, cell, l, status, hv, ia, crit);
      my_iters += l;
      if (status != 0) {
        my_failed += 1;
        my_worst = max(my_worst, status);
      }
    }
    {  // node states at the final iterate (also for INADMISSIBLE cells: the evaluation at lambda)
      for (int k = t; k < Q; k += G) {
        const double* u = nb + k * NS;
        if (A.uq) {
          double* o = A.uq + cell * Q * MS + k;  // [cell][state][node]
#pragma unroll
          for (int a = 0; a < MS; ++a) o[a * Q] = u[a];
        }
        if (A.want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(u, P.mesh, cell, P.cl.gamma));
      }
    }
    gsync();
  }
  PHASE_MARK(5);
#ifdef IPM_PHASE_TIMERS
  if (t == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&g_phase_cycles[i], ph_acc[i]);
#endif
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
