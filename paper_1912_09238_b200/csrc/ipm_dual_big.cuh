// ipm_dual_big.cuh — dual solve for large cells (config 5: N = 56, m = 4, n = 224, Q = 1000).
// (included inside namespace ipm by ipm_kernels.cu)
//
// One CTA (NT threads) per cell, persistent over an atomic cell queue.  The per-cell working set
// (node data Q x (m + m(m+1)/2), Hessian blocks N(N+1)/2 x m^2, diagonal inverses) does not fit on
// chip, so it lives in a per-CTA global scratch slice that stays L2-resident (148 CTAs x ~330 KB);
// the basis tables are read from global memory (L2).  Vectors (lambda, trial, uhat, g, d) are in
// shared memory.  Same method as k_dual_group: eval / gradient / Hessian blocks / blocked Cholesky
// with the forward solve folded in / back substitution / Armijo on L (reading 3').
#pragma once

template <int MS>
struct BigLayout {
  static constexpr int MM = MS * (MS + 1) / 2;
  static constexpr int NS = MS + MM;
  static constexpr int TB = MS * MS;
  // per-CTA global scratch (doubles): node data, Hessian blocks (also the first sum-factorisation
  // stage T1, which fits inside them), diagonal inverses, second stage T2 (p = 3)
  static __host__ __device__ size_t hb_size(int N, int q1, int npr, int p) {
    const size_t hb = (size_t)(N * (N + 1) / 2) * TB;
    const size_t t1 = (p == 3) ? (size_t)q1 * q1 * npr * MM : 0;
    return hb > t1 ? hb : t1;
  }
  static __host__ __device__ size_t t2_size(int q1, int npr, int p) {
    return (p == 3) ? (size_t)q1 * npr * npr * MM : 0;
  }
  static __host__ __device__ size_t scratch(int N, int Q, int q1, int npr, int p) {
    return (size_t)Q * NS + hb_size(N, q1, npr, p) + (size_t)N * TB + t2_size(q1, npr, p) + 64;
  }
};

template <int CL, int MS, int NT, bool HBS>
__global__ void __launch_bounds__(NT) k_dual_big(DualParams P, double* __restrict__ scratch) {
  using Lay = BigLayout<MS>;
  constexpr int NW = NT / 32;
  constexpr int MM = Lay::MM, NS = Lay::NS, TB = Lay::TB;
#define BIDX(a, b) ((b) * MS + (a))
  // shared-memory blocks: element index XOR-swizzled by the block index, so that threads touching the
  // same element of consecutive blocks hit different banks (a 128-byte block stride would put them all
  // in one bank)
#define SW(pb, x) (HBS ? ((x) ^ ((pb) & 15)) : (x))
  // HBS 8 x 8 blocks (and linvf): element (r, c) at r * 8 + (c ^ 4 (r & 2)) — the two column halves of
  // rows 2, 3, 6, 7 swapped, so the A/B-fragment loads (lane: row l/4, columns l%4 and l%4 + 4) of a
  // half-warp spread over all banks (plain rows put rows r and r + 2 on the same banks: 2-way
  // conflicts); the double2 C-fragment accesses stay aligned and conflict-free
//   and the whole element index XOR (2 b) & 14 for block b (a bijection inside the block that keeps both
//   properties), so that the Hessian scatter (one thread per basis pair, consecutive lanes in
//   consecutive blocks 64 doubles apart) spreads over 8 bank groups instead of hitting one
#ifdef IPM_BIG_NOSWZ
#define BE8(r, c) ((r) * 8 + (c))
#define BX(b) 0
#else
#define BE8(r, c) ((r) * 8 + ((c) ^ (((r) & 2) << 1)))
#define BX(b) ((int)(((b) * 2) & 14))
#endif
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, Q = P.T.Q, QP = P.T.QP;
  const double* __restrict__ PhiT = P.T.PhiT;
  const double* __restrict__ WPhiT = P.T.WPhiT;
  const double* __restrict__ omega = P.T.omega;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int nmax = N * MS;
  double* lam = sm;
  double* lt = lam + nmax;
  double* uh = lt + nmax;
  double* g = uh + nmax;
  double* dd = g + nmax;
  double* red = dd + nmax;  // [2][4][NW]
  double* sLL = red + 8 * NW;  // [q1][npr] 1D pair table (sum factorisation)
  int* ctl = (int*)(sLL + ((P.T.q1d * P.T.npr + 1) & ~1));
  for (int x = threadIdx.x; x < P.T.q1d * P.T.npr; x += NT) sLL[x] = P.T.LL[x];
  __syncthreads();
  const int q1 = P.T.q1d, npr = P.T.npr, pdim = P.T.p;
  double* nb = scratch + (size_t)blockIdx.x * Lay::scratch(N, Q, q1, npr, pdim);
  double* T1 = nb + (size_t)Q * NS;                 // [k1 k2][pr3][ab] (p = 3); Hb when not in smem
  double* Linv = T1 + Lay::hb_size(N, q1, npr, pdim);
  double* T2 = Linv + (size_t)N * TB;               // [k1][pr2][pr3][ab] (p = 3)
  // Hessian blocks (row-major lower enumeration): in shared memory when they fit (config 5: 204 KB),
  // so the blocked Cholesky works on-chip; else in the L2-resident scratch slice
  // HBS (compile time): the Hessian as 8 x 8 blocks (row-major, lower block triangle, 64 doubles each)
  // in shared memory, factored with DMMA (as k_dual_mma, blocks in shared memory instead of
  // registers); otherwise 4 x 4 blocks in the L2-resident scratch slice
  double* Hb = HBS ? sLL + ((P.T.q1d * P.T.npr + 1) & ~1) + 8 : T1;  // after ctl (8 doubles)
  const int NB8 = (N * MS + 7) / 8;
  double* linvf = Hb + (size_t)(NB8 * (NB8 + 1) / 2) * 64;  // HBS: Linv_K row-major (panel operand)

  const DualLaunch& A = P.a;
  long long my_iters = 0, my_failed = 0;
  int my_worst = 0;
  double my_rate = 0.0;
  int slot = 0;

  auto bsum = [&](double* v, int cnt) {  // block-wide sums of cnt (<= 4) values
    double* r = red + slot * 4 * NW;
    slot ^= 1;
    for (int a = 0; a < cnt; ++a) {
      const double s = warp_sum(v[a]);
      if (lane == 0) r[a * NW + wid] = s;
    }
    __syncthreads();
    for (int a = 0; a < cnt; ++a) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += r[a * NW + w];
      v[a] = s;
    }
  };
  auto eval = [&](const double* lamv, int Nl, double& s1, double& s2) -> bool {
    double v[2] = {0.0, 0.0};
    bool bad = false;
    for (int k = t; k < Q; k += NT) {
      double Lam[MS];
#pragma unroll
      for (int a = 0; a < MS; ++a) Lam[a] = 0.0;
      for (int i = 0; i < Nl; ++i) {
        const double ph = PhiT[(size_t)i * QP + k];
#pragma unroll
        for (int a = 0; a < MS; ++a) Lam[a] = fma(lamv[i * MS + a], ph, Lam[a]);
      }
      double u[MS], J[MM], ss;
      if (!Closure<CL, MS>::eval(Lam, u, J, ss, P.cl)) bad = true;
      double* row = nb + (size_t)k * NS;
#pragma unroll
      for (int a = 0; a < MS; ++a) row[a] = u[a];
#pragma unroll
      for (int q = 0; q < MM; ++q) row[MS + q] = J[q];
      v[0] = fma(omega[k], ss, v[0]);
      v[1] = fma(omega[k], fabs(ss), v[1]);
    }
    if (bad) v[1] = INFINITY;
    bsum(v, 2);
    s1 = v[0];
    s2 = v[1];
    return isfinite(v[0]) && isfinite(v[1]);
  };
  auto grad = [&](int Nl) -> double {
    const int n = Nl * MS;
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    if (HBS && ((Nl + 7) >> 3) <= 8) {
      // on the fp64 tensor path: C[i][a] = sum_k (omega phi_i)(xi_k) u_a(xi_k), A = omega Phi^T in
      // fragment order (Tables::WPhiF, L2), B = the node buffer's u; the node range is split over
      // the warps and the partial C tiles are summed through shared memory (the Hessian blocks of
      // the previous iteration are dead here)
      constexpr int NWp = NT / 32;
      const int MTg = (Nl + 7) >> 3, KS = P.T.KS;
      const int rr = lane >> 2, qq = lane & 3;
      double acc[8][2];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
      for (int ks = wid; ks < KS; ks += NWp) {
        const int k = 4 * ks + qq;
        const double bv = (rr < MS && k < Q) ? nb[(size_t)k * NS + rr] : 0.0;
        const double* af = P.T.WPhiF + (size_t)ks * 32 + lane;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
          if (mt < MTg) dmma884(acc[mt][0], acc[mt][1], af[(size_t)mt * KS * 32], bv);
      }
      double* red_c = Hb;  // [NWp][8][64]
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
        if (mt < MTg)
          *reinterpret_cast<double2*>(red_c + ((size_t)wid * 8 + mt) * 64 + 2 * lane) =
              make_double2(acc[mt][0], acc[mt][1]);
      __syncthreads();
      for (int r = t; r < n; r += NT) {
        const int i = r / MS, a = r - i * MS, mt = i >> 3;
        const int off = mt * 64 + ((i & 7) * 4 + (a >> 1)) * 2 + (a & 1);
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < NWp; ++w) sum += red_c[(size_t)w * 8 * 64 + off];
        const double gr = sum - uh[r];
        g[r] = gr;
        part[a] = fma(gr, gr, part[a]);
      }
      bsum(part, MS);
      double crit = 0.0;
      for (int a = 0; a < MS; ++a) crit += sqrt(part[a]);
      return crit;
    }
    // two threads per output (halves of the node range, combined by a shuffle): a 1000-node dot
    // product per output is a long latency chain
    const int Qh = (Q + 1) / 2;
    for (int base = 0; base < 2 * n; base += NT) {
      const int idx = base + t, r = idx >> 1, half = idx & 1;
      double s0 = 0.0, s1 = 0.0;
      if (idx < 2 * n) {
        const int i = r / MS, a = r - i * MS;
        const double* wp = WPhiT + (size_t)i * QP;
        const int k0 = half * Qh, k1 = half ? Q : Qh;
        int k = k0;
        for (; k + 1 < k1; k += 2) {
          s0 = fma(wp[k], nb[(size_t)k * NS + a], s0);
          s1 = fma(wp[k + 1], nb[(size_t)(k + 1) * NS + a], s1);
        }
        if (k < k1) s0 = fma(wp[k], nb[(size_t)k * NS + a], s0);
      }
      double sum = s0 + s1;
      sum += __shfl_xor_sync(FULL_MASK, sum, 1);
      if (idx < 2 * n && half == 0) {
        const int a = r % MS;
        const double gr = sum - uh[r];
        g[r] = gr;
        part[a] = fma(gr, gr, part[a]);
      }
    }
    bsum(part, MS);
    double crit = 0.0;
    for (int a = 0; a < MS; ++a) crit += sqrt(part[a]);
    return crit;
  };
  auto dot2 = [&](const double* x, const double* y, int n, double& d, double& ad) {
    double v[2] = {0.0, 0.0};
    for (int r = t; r < n; r += NT) {
      const double p = x[r] * y[r];
      v[0] += p;
      v[1] += fabs(p);
    }
    bsum(v, 2);
    d = v[0];
    ad = v[1];
  };
  // write the m x m block of basis pair (I >= J) of the Hessian (unique entries acc[ab])
  auto hput = [&](int p, int I, int J, const double* acc) {
#pragma unroll
    for (int a = 0; a < MS; ++a)
#pragma unroll
      for (int b = 0; b < MS; ++b) {
        const double v = acc[a <= b ? sym_idx<MS>(a, b) : sym_idx<MS>(b, a)];
        if constexpr (HBS) {
          const int R = I * MS + a, C = J * MS + b, bi = R >> 3, bj = C >> 3;
          Hb[(size_t)(bi * (bi + 1) / 2 + bj) * 64 + (BE8(R & 7, C & 7) ^ BX(bi * (bi + 1) / 2 + bj))] = v;
        } else {
          Hb[(size_t)p * TB + BIDX(a, b)] = v;
        }
      }
  };
  auto blk_ij = [](int p, int& I, int& J) {
    I = (int)((sqrtf(8.0f * p + 1.0f) - 1.0f) * 0.5f);
    while (I * (I + 1) / 2 > p) --I;
    while ((I + 1) * (I + 2) / 2 <= p) ++I;
    J = p - I * (I + 1) / 2;
  };

  // Cholesky of the 8 x 8-blocked Hessian in shared memory on the fp64 tensor path (HBS), forward
  // solve folded in, then the back substitution; dd: in -g (padded), out: the Newton direction.
  // Block (I, J) is row-major; after step J it holds L_IJ, the diagonal slot holds Linv_J.
  //   fragments (mma.m8n8k4.f64, lane = 4r + q): A (r, q + 4kk), B (q + 4kk, r), C (r, 2q + e)
  auto chol8 = [&](int n) -> bool {
    constexpr int NWp = NT / 32;
    const int NBl = (n + 7) >> 3, r = lane >> 2, q = lane & 3;
    auto blk = [&](int I, int J) -> double* { return Hb + (size_t)(I * (I + 1) / 2 + J) * 64; };
    auto bg = [&](int I, int J) -> int { return BX(I * (I + 1) / 2 + J); };
    // diagonal block K (warp 0): L_KK by quad shuffles, Linv_K (into linvf and the diagonal slot),
    // y_K = Linv_K b_K
    auto diag = [&](int K) {
      double* D = blk(K, K);
      const int gD = bg(K, K);
      double a0 = D[BE8(r, 2 * q) ^ gD], a1 = D[(BE8(r, 2 * q) ^ gD) + 1];
      const bool ok = blk8_diag_factor(a0, a1, lane, min(8, n - 8 * K));
      __syncwarp();
      *reinterpret_cast<double2*>(linvf + BE8(r, 2 * q)) = make_double2(a0, a1);
      *reinterpret_cast<double2*>(D + (BE8(r, 2 * q) ^ gD)) = make_double2(a0, a1);
      __syncwarp();
      const double f0 = linvf[BE8(r, q)], f1 = linvf[BE8(r, q + 4)];
      const double b0 = lane < 4 ? dd[K * 8 + lane] : 0.0, b1 = lane < 4 ? dd[K * 8 + 4 + lane] : 0.0;
      double y0 = 0.0, y1 = 0.0;
      dmma884(y0, y1, f0, b0);
      dmma884(y0, y1, f1, b1);
      __syncwarp();
      if (q == 0) dd[K * 8 + r] = y0;
      if (lane == 0 && !ok) ctl[1] = 1;
    };
    // A_IJ -= L_IK L_JK^T for the row I, columns J in [j0, j1]
    auto row_update = [&](int K, int I, int j0, int j1) {
      const double* Lik = blk(I, K);
      const int gik = bg(I, K);
      const double a0 = dneg(Lik[BE8(r, q) ^ gik]), a1 = dneg(Lik[BE8(r, q + 4) ^ gik]);
      for (int J = j0; J <= j1; ++J) {
        const double* Ljk = blk(J, K);
        double* C = blk(I, J);
        const int gjk = bg(J, K), gij = bg(I, J);
        double2 c = *reinterpret_cast<const double2*>(C + (BE8(r, 2 * q) ^ gij));
        dmma884(c.x, c.y, a0, Ljk[BE8(r, q) ^ gjk]);
        dmma884(c.x, c.y, a1, Ljk[BE8(r, q + 4) ^ gjk]);
        *reinterpret_cast<double2*>(C + (BE8(r, 2 * q) ^ gij)) = c;
      }
    };
    if (t == 0) ctl[1] = 0;
    if (wid == 0) diag(0);
    __syncthreads();
    for (int K = 0; K < NBl; ++K) {
      if (ctl[1]) return false;
      {  // panel: L_IK = A_IK Linv_K^T, b_I -= L_IK y_K
        const double lf0 = linvf[BE8(r, q)], lf1 = linvf[BE8(r, q + 4)];
        const double yf0 = lane < 4 ? dd[K * 8 + lane] : 0.0, yf1 = lane < 4 ? dd[K * 8 + 4 + lane] : 0.0;
        for (int I = K + 1 + wid; I < NBl; I += NWp) {
          double* B = blk(I, K);
          const int gB = bg(I, K);
          double f0 = B[BE8(r, q) ^ gB], f1 = B[BE8(r, q + 4) ^ gB];
          double x0 = 0.0, x1 = 0.0;
          dmma884(x0, x1, f0, lf0);
          dmma884(x0, x1, f1, lf1);
          __syncwarp();
          *reinterpret_cast<double2*>(B + (BE8(r, 2 * q) ^ gB)) = make_double2(x0, x1);
          __syncwarp();
          f0 = B[BE8(r, q) ^ gB];
          f1 = B[BE8(r, q + 4) ^ gB];
          double v0 = 0.0, v1 = 0.0;
          dmma884(v0, v1, f0, yf0);
          dmma884(v0, v1, f1, yf1);
          if (q == 0) dd[I * 8 + r] -= v0;
        }
      }
      __syncthreads();
      // trailing update by rows (the row's L_IK operand is loaded once); warp 0 first updates and
      // factors the next diagonal block (look-ahead), the other warps share the remaining rows
      if (K + 1 < NBl) {
        if (wid == 0) {
          row_update(K, K + 1, K + 1, K + 1);
          diag(K + 1);
        }
        // rows I = K+2 .. NBl-1 (row K+1 is only the diagonal block), cyclic over warps 1..NWp-1
        if (wid > 0)
          for (int idx = wid; idx < NBl - 1 - K; idx += NWp - 1) row_update(K, K + 1 + idx, K + 1, K + 1 + idx);
      }
      __syncthreads();
    }
    // back substitution: d_K = Linv_K^T z_K, z_J -= L_KJ^T d_K (row-vector DMMAs)
    for (int K = NBl - 1; K >= 0; --K) {
      if (wid == 0) {
        const double* D = blk(K, K);
        const int gD = bg(K, K);
        const double z0 = lane < 4 ? dd[K * 8 + lane] : 0.0, z1 = lane < 4 ? dd[K * 8 + 4 + lane] : 0.0;
        double v0 = 0.0, v1 = 0.0;
        dmma884(v0, v1, z0, D[BE8(q, r) ^ gD]);
        dmma884(v0, v1, z1, D[BE8(q + 4, r) ^ gD]);
        __syncwarp();
        if (lane < 4) {
          dd[K * 8 + 2 * q] = v0;
          dd[K * 8 + 2 * q + 1] = v1;
        }
      }
      __syncthreads();
      if (K == 0) break;
      const double d0 = lane < 4 ? dd[K * 8 + lane] : 0.0, d1 = lane < 4 ? dd[K * 8 + 4 + lane] : 0.0;
      for (int J = wid; J < K; J += NWp) {
        const double* L = blk(K, J);
        const int gL = bg(K, J);
        double v0 = 0.0, v1 = 0.0;
        dmma884(v0, v1, d0, L[BE8(q, r) ^ gL]);
        dmma884(v0, v1, d1, L[BE8(q + 4, r) ^ gL]);
        if (lane < 4) {
          dd[J * 8 + 2 * q] -= v0;
          dd[J * 8 + 2 * q + 1] -= v1;
        }
      }
      __syncthreads();
    }
    return true;
  };

  // cells from the work queue, or a device-built list (the Newton fallback of k_dual_lbfgs_big)
  const int64_t ncells = A.ncells_dev ? (int64_t)*A.ncells_dev : A.cells;
  int* const queue = A.queue ? A.queue : &P.sc->work_counter;
  for (;;) {
    if (t == 0) ctl[0] = atomicAdd(queue, 1);
    __syncthreads();
    const int64_t ci = ctl[0];
    if (ci >= ncells) break;
    const int64_t cell = A.list ? (int64_t)A.list[ci] : ci;
    const int lvl = A.level ? A.level[cell] : 0;
    const int Nl = (P.ad.n_levels > 0) ? P.ad.Nl[lvl] : N;
    const int n = Nl * MS, NPl = Nl * (Nl + 1) / 2;
    const double* gu = A.uhat + cell * nmax;
    double* gl = A.lam + cell * nmax;
    for (int r = t; r < n; r += NT) {
      uh[r] = gu[r];
      lam[r] = gl[r];
    }
    __syncthreads();
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
        // Hessian blocks H_IJ = sum_k omega_k phi_kI phi_kJ J_k
        if (pdim == 3 && npr <= 32) {
          // sum factorisation over the tensor rule, k = (k1 q1 + k2) q1 + k3, LL[k][(a,b)] =
          // (w_k/2) L_a L_b (x_k):  T1 = sum_k3 LL J,  T2 = sum_k2 LL T1,  H = sum_k1 LL T2
          const int SF = (int)((sqrtf(8.0f * npr + 1.0f) - 1.0f) * 0.5f + 0.5f);
          if (npr <= 24 && q1 <= 12) {
            // stages 1 and 2 on the fp64 tensor path: both contract a 1D node index with LL, so the
            // A operand LL^T[pr][k] (pr < 24, k < 12: 3 x 3 fragments) stays in registers
            constexpr int NWp = NT / 32;
            const int rr = lane >> 2, qq = lane & 3;
            double lla[3][3];
#pragma unroll
            for (int mt = 0; mt < 3; ++mt)
#pragma unroll
              for (int ks = 0; ks < 3; ++ks) {
                const int pr = 8 * mt + rr, k = 4 * ks + qq;
                lla[mt][ks] = (pr < npr && k < q1) ? sLL[k * npr + pr] : 0.0;
              }
            // stage 1: per (k1 k2): T1[k12][pr3][ab] = sum_k3 LL[k3][pr3] J_ab(k12 q1 + k3)
            for (int u = wid; u < q1 * q1 * 2; u += NWp) {
              const int k12 = u >> 1, nt = u & 1, ab = 8 * nt + rr;
              double bfr[3];
#pragma unroll
              for (int ks = 0; ks < 3; ++ks) {
                const int k3 = 4 * ks + qq;
                bfr[ks] = (k3 < q1 && ab < MM) ? nb[((size_t)k12 * q1 + k3) * NS + MS + ab] : 0.0;
              }
#pragma unroll
              for (int mt = 0; mt < 3; ++mt) {
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) dmma884(c0, c1, lla[mt][ks], bfr[ks]);
                const int pr3 = 8 * mt + rr, abo = 8 * nt + 2 * qq;
                if (pr3 < npr) {
                  double* o = T1 + ((size_t)k12 * npr + pr3) * MM + abo;
                  if (abo + 1 < MM)
                    *reinterpret_cast<double2*>(o) = make_double2(c0, c1);
                  else if (abo < MM)
                    o[0] = c0;
                }
              }
            }
            __syncthreads();
            // stage 2: per k1: T2[k1][pr2][col] = sum_k2 LL[k2][pr2] T1[k1 q1 + k2][col], col = pr3 MM + ab
            const int ncol = npr * MM, ntl = (ncol + 7) >> 3;
            for (int u = wid; u < q1 * ntl; u += NWp) {
              const int k1 = u / ntl, nt = u - k1 * ntl, col = 8 * nt + rr;
              double bfr[3];
#pragma unroll
              for (int ks = 0; ks < 3; ++ks) {
                const int k2 = 4 * ks + qq;
                bfr[ks] = (k2 < q1 && col < ncol) ? T1[((size_t)k1 * q1 + k2) * ncol + col] : 0.0;
              }
#pragma unroll
              for (int mt = 0; mt < 3; ++mt) {
                double c0 = 0.0, c1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 3; ++ks) dmma884(c0, c1, lla[mt][ks], bfr[ks]);
                const int pr2 = 8 * mt + rr, co = 8 * nt + 2 * qq;
                if (pr2 < npr) {
                  double* o = T2 + ((size_t)k1 * npr + pr2) * ncol + co;
                  if (co + 1 < ncol)
                    *reinterpret_cast<double2*>(o) = make_double2(c0, c1);
                  else if (co < ncol)
                    o[0] = c0;
                }
              }
            }
            __syncthreads();
          } else {
          for (int e = t; e < q1 * q1 * MM; e += NT) {
            const int k12 = e / MM, ab = e - k12 * MM;
            double at[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) at[x] = 0.0;
            const double* jr = nb + (size_t)k12 * q1 * NS + MS + ab;
            for (int k3 = 0; k3 < q1; ++k3) {
              const double jv = jr[(size_t)k3 * NS];
              const double* ll = sLL + k3 * npr;
#pragma unroll
              for (int x = 0; x < 32; ++x)
                if (x < npr) at[x] = fma(ll[x], jv, at[x]);
            }
#pragma unroll
            for (int x = 0; x < 32; ++x)
              if (x < npr) T1[((size_t)k12 * npr + x) * MM + ab] = at[x];
          }
          __syncthreads();
          for (int e = t; e < q1 * npr * MM; e += NT) {
            const int k1 = e / (npr * MM), rem = e - k1 * npr * MM, pr3 = rem / MM, ab = rem - pr3 * MM;
            double at[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) at[x] = 0.0;
            for (int k2 = 0; k2 < q1; ++k2) {
              const double tv = T1[(((size_t)k1 * q1 + k2) * npr + pr3) * MM + ab];
              const double* ll = sLL + k2 * npr;
#pragma unroll
              for (int x = 0; x < 32; ++x)
                if (x < npr) at[x] = fma(ll[x], tv, at[x]);
            }
#pragma unroll
            for (int x = 0; x < 32; ++x)
              if (x < npr) T2[(((size_t)k1 * npr + x) * npr + pr3) * MM + ab] = at[x];
          }
          __syncthreads();
          }
          for (int p = t; p < NPl; p += NT) {
            int I, J;
            blk_ij(p, I, J);
            int pr[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              int a = P.T.idx[I * 3 + d], b = P.T.idx[J * 3 + d];
              if (a > b) {
                const int x = a;
                a = b;
                b = x;
              }
              pr[d] = a * SF - a * (a - 1) / 2 + (b - a);
            }
            double acc[MM];
#pragma unroll
            for (int z = 0; z < MM; ++z) acc[z] = 0.0;
            for (int k1 = 0; k1 < q1; ++k1) {
              const double lv = sLL[k1 * npr + pr[0]];
              const double* tv = T2 + (((size_t)k1 * npr + pr[1]) * npr + pr[2]) * MM;
              if constexpr (MM % 2 == 0) {  // rows of MM doubles start 16-byte aligned: vector loads
#pragma unroll
                for (int z = 0; z < MM; z += 2) {
                  const double2 v2 = *reinterpret_cast<const double2*>(tv + z);
                  acc[z] = fma(lv, v2.x, acc[z]);
                  acc[z + 1] = fma(lv, v2.y, acc[z + 1]);
                }
              } else {
#pragma unroll
                for (int z = 0; z < MM; ++z) acc[z] = fma(lv, tv[z], acc[z]);
              }
            }
            hput(p, I, J, acc);
          }
        } else
        for (int p = t; p < NPl; p += NT) {
          int I, J;
          blk_ij(p, I, J);
          double acc[MM];
#pragma unroll
          for (int z = 0; z < MM; ++z) acc[z] = 0.0;
          const double* wi = WPhiT + (size_t)I * QP;
          const double* pj = PhiT + (size_t)J * QP;
          for (int k = 0; k < Q; ++k) {
            const double f = wi[k] * pj[k];
            const double* Jk = nb + (size_t)k * NS + MS;
#pragma unroll
            for (int z = 0; z < MM; ++z) acc[z] = fma(f, Jk[z], acc[z]);
          }
          hput(p, I, J, acc);
        }
        // identity padding of the last 8 x 8 block row beyond n (HBS), right-hand side -g
        if constexpr (HBS) {
          const int NBl = (n + 7) >> 3;
          if (n < NBl * 8) {
            const int I = NBl - 1;
            for (int e = t; e < NBl * 64; e += NT) {
              const int J = e >> 6, rr = (e >> 3) & 7, cc = e & 7;
              const int R = 8 * I + rr, C = 8 * J + cc;
              if (R >= n || C >= n) Hb[(size_t)(I * (I + 1) / 2 + J) * 64 + (BE8(rr, cc) ^ BX(I * (I + 1) / 2 + J))] = (R == C) ? 1.0 : 0.0;
            }
          }
          for (int r = t; r < NBl * 8; r += NT) dd[r] = (r < n) ? -g[r] : 0.0;
        } else {
          for (int r = t; r < n; r += NT) dd[r] = -g[r];
        }
        __syncthreads();
        bool chol_ok = true;
        if constexpr (HBS) {
          chol_ok = chol8(n);
        } else {
        // blocked right-looking Cholesky, blocks resident in the scratch slice; forward solve folded
        for (int K = 0; K < Nl; ++K) {
          if (t == 0) {
            const int pk = K * (K + 1) / 2 + K;
            double* Bk = Hb + (size_t)pk * TB;
            double L[MS][MS], li[MS][MS], inv[MS];
            bool ok = true;
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) L[a][b] = Bk[SW(pk, BIDX(a, b))];
#pragma unroll
            for (int c = 0; c < MS; ++c) {
              double sv = L[c][c];
#pragma unroll
              for (int x = 0; x < c; ++x) sv = fma(-L[c][x], L[c][x], sv);
              if (!(sv > 0.0) || !isfinite(sv)) ok = false;
              const double rs = rsqrt(sv);
              inv[c] = rs;
              L[c][c] = sv * rs;
#pragma unroll
              for (int r = c + 1; r < MS; ++r) {
                double v = L[r][c];
#pragma unroll
                for (int x = 0; x < c; ++x) v = fma(-L[r][x], L[c][x], v);
                L[r][c] = v * rs;
              }
            }
#pragma unroll
            for (int c = 0; c < MS; ++c) {
              li[c][c] = inv[c];
#pragma unroll
              for (int r = c + 1; r < MS; ++r) {
                double v = 0.0;
#pragma unroll
                for (int x = c; x < r; ++x) v = fma(L[r][x], li[x][c], v);
                li[r][c] = -inv[r] * v;
              }
            }
            double* oi = Linv + (size_t)K * TB;
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) {
                Bk[SW(pk, BIDX(a, b))] = (b <= a) ? L[a][b] : 0.0;
                oi[SW(K, BIDX(a, b))] = (b <= a) ? li[a][b] : 0.0;
              }
            double bk[MS];
#pragma unroll
            for (int a = 0; a < MS; ++a) bk[a] = dd[K * MS + a];
#pragma unroll
            for (int a = 0; a < MS; ++a) {
              double v = 0.0;
#pragma unroll
              for (int x = 0; x <= a; ++x) v = fma(li[a][x], bk[x], v);
              dd[K * MS + a] = v;
            }
            ctl[1] = ok ? 0 : 1;
          }
          __syncthreads();
          if (ctl[1]) {
            chol_ok = false;
            break;
          }
          const double* Li = Linv + (size_t)K * TB;
          for (int I = K + 1 + t; I < Nl; I += NT) {
            const int pik = I * (I + 1) / 2 + K;
            double* Bik = Hb + (size_t)pik * TB;
            double A_[MS][MS], X[MS][MS], yk[MS];
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) A_[a][b] = Bik[SW(pik, BIDX(a, b))];
#pragma unroll
            for (int r = 0; r < MS; ++r)
#pragma unroll
              for (int c = 0; c < MS; ++c) {
                double v = 0.0;
#pragma unroll
                for (int x = 0; x <= c; ++x) v = fma(A_[r][x], Li[SW(K, BIDX(c, x))], v);
                X[r][c] = v;
              }
#pragma unroll
            for (int x = 0; x < MS; ++x) yk[x] = dd[K * MS + x];
#pragma unroll
            for (int r = 0; r < MS; ++r) {
              double v = dd[I * MS + r];
#pragma unroll
              for (int c = 0; c < MS; ++c) {
                Bik[SW(pik, BIDX(r, c))] = X[r][c];
                v = fma(-X[r][c], yk[c], v);
              }
              dd[I * MS + r] = v;
            }
          }
          __syncthreads();
          // trailing: blocks (I, J) with I >= J > K
          const int R = Nl - 1 - K, ntr = R * (R + 1) / 2;
          for (int e = t; e < ntr; e += NT) {
            int a_, b_;
            blk_ij(e, a_, b_);
            const int I = K + 1 + a_, J = K + 1 + b_;
            const int pik = I * (I + 1) / 2 + K, pjk = J * (J + 1) / 2 + K, pij = I * (I + 1) / 2 + J;
            const double* Lik = Hb + (size_t)pik * TB;
            const double* Ljk = Hb + (size_t)pjk * TB;
            double* Bij = Hb + (size_t)pij * TB;
            double acc[MS][MS];
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) acc[a][b] = Bij[SW(pij, BIDX(a, b))];
#pragma unroll
            for (int x = 0; x < MS; ++x) {
              double ci[MS], cj[MS];
#pragma unroll
              for (int a = 0; a < MS; ++a) {
                ci[a] = Lik[SW(pik, BIDX(a, x))];
                cj[a] = Ljk[SW(pjk, BIDX(a, x))];
              }
#pragma unroll
              for (int r = 0; r < MS; ++r)
#pragma unroll
                for (int c = 0; c < MS; ++c) acc[r][c] = fma(-ci[r], cj[c], acc[r][c]);
            }
#pragma unroll
            for (int a = 0; a < MS; ++a)
#pragma unroll
              for (int b = 0; b < MS; ++b) Bij[SW(pij, BIDX(a, b))] = acc[a][b];
          }
          __syncthreads();
        }
          if (chol_ok) {
        // back substitution L^T d = y (warp 0)
        if (wid == 0) {
          for (int K = Nl - 1; K >= 0; --K) {
            const double* Li = Linv + (size_t)K * TB;
            double dk[MS];
#pragma unroll
            for (int c = 0; c < MS; ++c) {
              double v = 0.0;
#pragma unroll
              for (int x = c; x < MS; ++x) v = fma(Li[SW(K, BIDX(x, c))], dd[K * MS + x], v);
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
              const int pkj = K * (K + 1) / 2 + J;
              const double* Lkj = Hb + (size_t)pkj * TB;
              double v = dd[J * MS + c];
#pragma unroll
              for (int x = 0; x < MS; ++x) v = fma(-Lkj[SW(pkj, BIDX(x, c))], dk[x], v);
              dd[J * MS + c] = v;
            }
            __syncwarp();
          }
        }
        __syncthreads();
          }
        }
        if (!chol_ok) {
          status = 2;
          break;
        }
        __syncthreads();
        double slope, dummy;
        dot2(g, dd, n, slope, dummy);
        double alpha = 1.0;
        bool accepted = false;
        for (int h = 0; h <= P.nw.max_halvings; ++h) {
          for (int r = t; r < n; r += NT) lt[r] = lam[r] + alpha * dd[r];
          __syncthreads();
          double t1, t2;
          const bool okt = eval(lt, Nl, t1, t2);
          nb_is_lam = false;
          if (okt) {
            double d1, d2;
            dot2(lt, uh, n, d1, d2);
            const double Lt = t1 - d1;
            if (Lt <= L0 + P.nw.armijo_c * alpha * slope + 1e-12 * scale) {
              crit = grad(Nl);
              for (int r = t; r < n; r += NT) lam[r] = lt[r];
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
        __syncthreads();
      }
    }
    __syncthreads();
    if (!nb_is_lam && status != 4) {
      double t1, t2;
      eval(lam, Nl, t1, t2);
    }
    int Nnew = Nl;
    if (P.ad.n_levels > 0 && A.level_new) {
      const int Nprev = lvl > 0 ? P.ad.Nl[lvl - 1] : P.ad.Nprev0;
      double v[2] = {0.0, 0.0};
      for (int i = t; i < Nl; i += NT) {
        const double h = g[i * MS] + uh[i * MS];
        v[1] = fma(h, h, v[1]);
        if (i >= Nprev) v[0] = fma(h, h, v[0]);
      }
      bsum(v, 2);
      const double S = v[1] > 0.0 ? v[0] / v[1] : 0.0;
      const int nl = next_level(P.ad, P.sc, lvl, status, S);
      Nnew = P.ad.Nl[nl];
      if (t == 0) A.level_new[cell] = nl;
    }
    for (int r = t; r < nmax; r += NT) gl[r] = (r < n) ? lam[r] : 0.0;  // truncated to the new level after the flux
    if (t == 0) {
      cell_stats(A, P.sc, cell, l, status, hv, ia, crit);
      my_iters += l;
      if (status != 0) {
        my_failed += 1;
        my_worst = max(my_worst, status);
      }
    }
    {  // node states at the final iterate (also for INADMISSIBLE cells: the evaluation at lambda)
      for (int k = t; k < Q; k += NT) {
        const double* u = nb + (size_t)k * NS;
        if (A.uq) {
          double* o = A.uq + cell * Q * MS + k;  // [cell][state][node]
#pragma unroll
          for (int a = 0; a < MS; ++a) o[a * Q] = u[a];
        }
        if (A.want_rate) my_rate = fmax(my_rate, node_rate<CL, MS>(u, P.mesh, cell, P.cl.gamma));
      }
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
#undef BIDX
#undef SW
}
