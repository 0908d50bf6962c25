// ipm_dual_mma.cuh — dual solve with a register-resident, DMMA-blocked Cholesky (sm_100a, fp64).
//
// Same method as k_dual_group (Algorithm 1 / 2, reading 3' line search), with the
// Newton system solved on the fp64 tensor path:
//   * a group of W warps owns one spatial cell at a time (cells from an atomic queue);
//   * the Hessian H = sum_k omega_k (phi_k phi_k^T) (x) J_k is built as the
//     N(N+1)/2 x m(m+1)/2 table S[ab][pair] of its unique entries (sum factorised over the tensor
//     Gauss-Legendre rule when p = 2, else the direct sum), then gathered into 8 x 8 blocks of the
//     padded n x n matrix (n = N m, padded with the identity to NB*8);
//   * every lower-triangular 8 x 8 block lives in the registers of one warp in the accumulator
//     layout of mma.sync.m8n8k4.f64 (lane l: row l/4, columns 2(l%4), 2(l%4)+1);
//   * right-looking blocked Cholesky, one block column K per step:
//       diag     owner of (K,K): unblocked factor by quad shuffles, Linv_K = L_KK^{-1} formed on the
//                fly; y_K = Linv_K b_K (forward solve folded in);
//       panel    owners of (I,K): L_IK = A_IK Linv_K^T (2 DMMA), b_I -= L_IK y_K, L_IK published to
//                shared memory in operand (A-fragment) order;
//       trailing owners of (I,J), J > K: A_IJ -= L_IK L_JK^T (2 DMMA); the owner of (K+1,K+1)
//                updates and factors it first (look-ahead);
//   * back substitution L^T d = y with the register blocks (Linv_K^T on the diagonal, L_KJ^T below).
#pragma once
#include <utility>
// (included inside namespace ipm by ipm_kernels.cu, after DualParams and node_rate)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// ordered shared-memory load (volatile: not hoisted across the DMMAs, which bounds register use)
__device__ __forceinline__ double lds_ord(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ double dneg(double x) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)0x8000000000000000ULL);
}

// compile-time loop: f(std::integral_constant<int, i>) for i = 0..N-1 (indices are constants in f)
template <class F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// column-major enumeration of the lower block triangle: r -> (I, J), J = 0.., I = J..NB-1
__host__ __device__ constexpr int cmJ(int r, int NB) {
  int J = 0;
  while (r >= NB - J) {
    r -= NB - J;
    ++J;
  }
  return J;
}
__host__ __device__ constexpr int cmI(int r, int NB) {
  int J = 0;
  while (r >= NB - J) {
    r -= NB - J;
    ++J;
  }
  return J + r;
}

// 1/sqrt(x): hardware approximation + two Newton steps (rounding-level accuracy for the positive
// normal pivots of an SPD matrix; shorter latency than the library rsqrt, which also handles
// special operands, on the Cholesky's critical path)
__device__ __forceinline__ double rsqrt_nr(double x) {
#ifdef IPM_DIAG_LIBRSQRT
  return rsqrt(x);
#else
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
#ifdef IPM_RSQRT_NR1  // one Newton step (~1e-13 relative): +1 % on config 3, not the default
  return fma(y, e, y);
#else
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  return fma(y, e, y);
#endif
#endif
}

// ---- 8x8 diagonal block: in C-fragment layout A (lower part used); out: Linv = L^{-1} -------
// ncol: columns to factor (the rest of the block is identity padding beyond n)
__device__ __forceinline__ bool blk8_diag_factor(double& a0, double& a1, int lane, int ncol = 8) {
  const int r = lane >> 2, q = lane & 3;
  double x0 = (r == 2 * q) ? 1.0 : 0.0, x1 = (r == 2 * q + 1) ? 1.0 : 0.0;
  bool ok = true;
  __syncwarp();  // the warp is converged here: lets the compiler drop divergent-shuffle fallbacks
#ifdef IPM_DIAG_UNROLL
#pragma unroll
#else
#pragma unroll 1  // smaller code beats the extra ILP (instruction-cache bound kernel)
#endif
  for (int c = 0; c < ncol; ++c) {
    const int cq = c >> 1;
    const double mine = (c & 1) ? a1 : a0;
    const double d = __shfl_sync(FULL_MASK, mine, c * 4 + cq);
    const double arc = __shfl_sync(FULL_MASK, mine, r * 4 + cq);
    const double a0c = __shfl_sync(FULL_MASK, mine, (2 * q) * 4 + cq);
    const double a1c = __shfl_sync(FULL_MASK, mine, (2 * q + 1) * 4 + cq);
    if (!(d > 0.0) || !isfinite(d)) ok = false;
    const double rs = rsqrt_nr(d);
    const double lrc = arc * rs;
    if (2 * q > c) a0 = fma(-lrc, a0c * rs, a0);
    if (2 * q + 1 > c) a1 = fma(-lrc, a1c * rs, a1);
    const double xs = (r == c) ? rs : 1.0;
    x0 *= xs;
    x1 *= xs;
    const double xc0 = __shfl_sync(FULL_MASK, x0, c * 4 + q);
    const double xc1 = __shfl_sync(FULL_MASK, x1, c * 4 + q);
    if (r > c) {
      x0 = fma(-lrc, xc0, x0);
      x1 = fma(-lrc, xc1, x1);
    }
  }
  a0 = x0;
  a1 = x1;
  return ok;
}


// ---- 8x8 diagonal block: explicit inverse by Gauss-Jordan (block LDL^T, IPM_MMA_LDL) ----------------
// in:  a0, a1 = A[r][2q], A[r][2q+1] of the symmetric positive definite block (C-fragment, full)
// out: a0, a1 = the same entries of A^{-1}; false on a pivot <= 0 or non-finite.  The pivots are the
// diagonal of the block's LDL^T (= the squared Cholesky pivots): an indefinite matrix fails at the
// same pivot as the Cholesky factorisation.  Per column: four independent shuffles, one reciprocal,
// two fmas — no square root and no separate inverse of L.
__device__ __forceinline__ bool blk8_gj_inverse(double& a0, double& a1, int lane, int ncol = 8) {
  const int r = lane >> 2, q = lane & 3;
  bool ok = true;
  __syncwarp();
#pragma unroll 1
  for (int k = 0; k < ncol; ++k) {
    const int kq = k >> 1;
    const double mine = (k & 1) ? a1 : a0;                    // A[.][k] of this lane's row
    const double p = __shfl_sync(FULL_MASK, mine, k * 4 + kq);  // A[k][k]
    const double ark = __shfl_sync(FULL_MASK, mine, r * 4 + kq);  // A[r][k]
    const double rk0 = __shfl_sync(FULL_MASK, a0, k * 4 + q);     // A[k][2q]
    const double rk1 = __shfl_sync(FULL_MASK, a1, k * 4 + q);     // A[k][2q+1]
    if (!(p > 0.0) || !isfinite(p)) ok = false;
    const double ip = rcp_nr(p);
    const double f = ark * ip;
    const bool rowk = r == k;
    a0 = (2 * q == k) ? (rowk ? ip : -f) : (rowk ? rk0 * ip : fma(-f, rk0, a0));
    a1 = (2 * q + 1 == k) ? (rowk ? ip : -f) : (rowk ? rk1 * ip : fma(-f, rk1, a1));
  }
  return ok;
}

// ---- 8x8 diagonal block, rows in lanes ------------------------------------------------------------
// Left-looking (Crout) Cholesky with lane l owning row r = l/4 (its 4 lanes compute redundantly):
//   s_rc = A_rc - sum_{k<c} L_rk L_ck,   d_c = A_cc - sum_{k<c} L_ck^2,   L_rc = s_rc / sqrt(d_c)
// row c of L comes from shared memory (written one column at a time), the pivot d_c from the shuffle of
// row c's running diagonal; then row r of Linv = L^{-1} by back substitution x L = e_r.  The
// per-column chain is one shuffle + rsqrt; the instruction count is a third of the shuffle-based
// C-fragment factor (each lane carries only its row).
//   in:  a0, a1 = A[r][2q], A[r][2q+1] (C-fragment; lower part used), As / Ls: 64-double shared scratch
//   out: a0, a1 = Linv[r][2q], Linv[r][2q+1]; false on a pivot <= 0 or non-finite
// ncol: columns to factor (the rest of the block is the identity padding beyond n)
__device__ __forceinline__ bool blk8_factor_rows(double& a0, double& a1, int lane, int ncol, double* As,
                                                 double* Ls) {
  const int r = lane >> 2, q = lane & 3;
  *reinterpret_cast<double2*>(As + 2 * lane) = make_double2(a0, a1);  // C-fragment order = row-major
  __syncwarp();
  double lr[8];               // row r of L (lr[c] = L_rc for c < r; 0 for c > r)
  double dr = As[r * 8 + r];  // running pivot of row r
  double rsr = 1.0;           // 1 / L_rr
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double s = As[r * 8 + c];
#pragma unroll
    for (int k = 0; k < c; ++k) s = fma(-lr[k], Ls[c * 8 + k], s);
    const double d = __shfl_sync(FULL_MASK, dr, 4 * c);
    const bool live = c < ncol;
    ok = ok && (!live || ((d > 0.0) && isfinite(d)));
    const double rs = live ? rsqrt_nr(d) : 1.0;
    const double l = (r > c) ? s * rs : 0.0;
    lr[c] = l;
    dr = fma(-l, l, dr);
    if (r == c) rsr = rs;
    if (q == 0) Ls[r * 8 + c] = (r == c) ? rs : l;  // L below the diagonal, 1 / L_cc on it
    __syncwarp();
  }
  // row r of Linv: x_j = 0 (j > r), x_r = 1 / L_rr, x_j = -(1 / L_jj) sum_{i=j+1..r} x_i L_ij (j < r)
  double x[8];
#pragma unroll
  for (int j = 7; j >= 0; --j) {
    double acc = 0.0;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) acc = fma(x[i], Ls[i * 8 + j], acc);
    x[j] = (j < r) ? -Ls[j * 8 + j] * acc : ((j == r) ? rsr : 0.0);
  }
  a0 = (q == 0) ? x[0] : (q == 1) ? x[2] : (q == 2) ? x[4] : x[6];
  a1 = (q == 0) ? x[1] : (q == 1) ? x[3] : (q == 2) ? x[5] : x[7];
  __syncwarp();  // Ls / As are overwritten by the caller next
  return ok;
}

// Stored 8 x 8 blocks of the fragment exchange (pan, panA, linvf): row r at MMA_ROW(r) = 8 r + 4 (r / 2),
// block extent 76, stride MMA_BS = 80.  The skew of 4 doubles every second row makes the A-fragment loads (lane:
// row l/4, columns l%4 and l%4 + 4) conflict-free — with the plain r * 8 rows, rows r and r + 2 of a
// half-warp fell into the same banks (2-way conflicts, ncu r02q: 5.1 G excess shared wavefronts per
// launch) — and keeps the B-fragment loads (column-wise) and the double2 C-fragment stores
// conflict-free; both offsets of a fragment still differ by an immediate (+4 / +40 doubles).
#ifdef IPM_MMA_BLK64  // A/B: the unskewed layout
#define MMA_ROW(r) ((r) * 8)
#define MMA_BS 64
#else
#define MMA_ROW(r) ((r) * 8 + 4 * ((r) >> 1))
#define MMA_BS 80
#endif

template <int MS>
struct MmaLayout {
  static constexpr int MM = MS * (MS + 1) / 2;
  static constexpr int NCH = (MM >= 6) ? 2 : 1;  // ab chunks of the sum factorisation
  static constexpr int CHW = (MM + NCH - 1) / NCH;
  static constexpr int RSX = MS > 4 ? MS : 4;  // values per group reduction
  // region (per group):  [node buffer u[MS][Q], J[MM][Q]]  overlapped by  S[MM][NPP]
  //                      [T chunk q1 x NPR x CHW] at offset TO (SF only)
  // S may overlap the dead part of the node buffer chunk by chunk (see s_base)
  static __host__ __device__ int npp(int N) { return N * (N + 1) / 2; }
  // stage-2 work list of the sum factorisation (SF > 0): pairs grouped two by two with a common 1D pair
  // index pr2, slots [2 * NEMAX] ints + the pr2 histogram [npr] + the entry count, in doubles
  static __host__ __device__ int nemax(int N, int npr) { return (N * (N + 1) / 2 + npr) / 2 + 1; }
  static __host__ __device__ int pairlist_doubles(int N, int npr) { return (nemax(N, npr) + (npr + 2) / 2 + 1) & ~1; }
  // row stride of S[ab][pair]: odd, so the gather's rows (different ab) fall into different banks
  static __host__ __device__ int nps(int N) { return npp(N) | 1; }
  static __host__ __device__ int node(int Q) { return Q * (MS + MM); }
  static __host__ __device__ bool s_overlaps(int N, int Q, int SF) {
    if (SF == 0) return false;  // the direct sum reads J until the end
    for (int ch = 0; ch + 1 < NCH; ++ch)
      if ((ch + 1) * CHW * nps(N) > (MS + (ch + 1) * CHW) * Q) return false;
    return true;
  }
  static __host__ __device__ int t_off(int N, int Q, int SF) {
    const int s = s_overlaps(N, Q, SF) ? MM * nps(N) : 0;
    return ((node(Q) > s ? node(Q) : s) + 1) & ~1;
  }
  static __host__ __device__ int s_base(int N, int Q, int SF, int q1d) {
    if (s_overlaps(N, Q, SF)) return 0;
    const int t = (SF > 0) ? q1d * (SF * (SF + 1) / 2) * CHW : 0;
    return (t_off(N, Q, SF) + t + 1) & ~1;
  }
  static __host__ __device__ int region(int N, int Q, int SF, int q1d, int NB) {
    int r = s_base(N, Q, SF, q1d) + MM * nps(N);
    const int t = t_off(N, Q, SF) + ((SF > 0) ? q1d * (SF * (SF + 1) / 2) * CHW : 0);
    if (t > r) r = t;
#ifdef IPM_MMA_LDL  // + the unscaled panel [NB][64] and w = D^{-1} z [NB * 8]
    const int c = (2 * NB + 1) * MMA_BS + NB * 64 + NB * 8;
#else
    const int c = (NB + 1) * MMA_BS + NB * 64;  // Cholesky: panel [NB][BS], Linv fragment [BS], diagonal [NB][64]
#endif
    if (c > r) r = c;
    return (r + 1) & ~1;
  }
  static __host__ __device__ int per_group(int N, int Q, int W, int SF, int q1d, int NB) {
    const int nv = NB * 8;  // padded vector length
    int w = 5 * nv + region(N, Q, SF, q1d, NB) + 2 * RSX * W + 4;
    return (w + 1) & ~1;
  }
};

template <int CL, int MS, int NB, int W, int SF>
struct DualMma {
  using Lay = MmaLayout<MS>;
  static constexpr int MM = Lay::MM;
  static constexpr int G = 32 * W;
  static constexpr int NBT = NB * (NB + 1) / 2;
  
  __device__ static bool diag_factor(double& a0, double& a1, int lane, int ncol, double* As, double* Ls) {
#ifdef IPM_DIAG_ROWS  // rows-in-lanes factor: a third of the instructions, measured 22 % slower
    return blk8_factor_rows(a0, a1, lane, ncol, As, Ls);
#else
    return blk8_diag_factor(a0, a1, lane, ncol);
#endif
  }

  // C-fragment -> A-fragment (lane l: row l/4, column l%4 + 4 kk)
  __device__ static void to_afrag(double c0, double c1, int lane, double& f0, double& f1) {
    const int r = lane >> 2, q = lane & 3;
    const int s0 = r * 4 + (q >> 1), s1 = s0 + 2;
    const double u0 = __shfl_sync(FULL_MASK, c0, s0), u1 = __shfl_sync(FULL_MASK, c1, s0);
    const double v0 = __shfl_sync(FULL_MASK, c0, s1), v1 = __shfl_sync(FULL_MASK, c1, s1);
    f0 = (q & 1) ? u1 : u0;
    f1 = (q & 1) ? v1 : v0;
  }
  // block storage in shared memory for fragment exchange: row-major, element (r, c) at r*8 + c.
  // (An XOR swizzle that also removes the 2-way conflicts of the A/B-fragment loads measured 3 %
  // slower: the extra index arithmetic costs more than the conflicts.)
  __device__ static int bpos(int r, int c) { return MMA_ROW(r) + c; }
  __device__ static void store_afrag(double* dst, double c0, double c1, int lane) {
    const int r = lane >> 2, q = lane & 3;
    double2* p = reinterpret_cast<double2*>(dst + bpos(r, 2 * q));
    *p = make_double2(c0, c1);
  }

  // H entry (R, C) from the unique-entry table S[ab][pair(i >= j)]; identity outside n x n
  __device__ static double hval(const double* S, int npp, int n, int R, int C) {
    if (R >= n || C >= n) return (R == C) ? 1.0 : 0.0;
    if (R < C) {
      const int x = R;
      R = C;
      C = x;
    }
    const int i = R / MS, a = R - i * MS, j = C / MS, b = C - j * MS;
    const int ab = (a <= b) ? sym_idx<MS>(a, b) : sym_idx<MS>(b, a);
    return S[ab * npp + i * (i + 1) / 2 + j];
  }

  // Gather H (unique-entry table S[ab][pair]) into 8x8 blocks, factor, solve.
  //   strictly-lower blocks: registers of warp (column-major rank) % W, C-fragment layout; the
  //                          (I, J) of slot s of warp wr is byte s of ijp (packed 4 per word)
  //   diagonal blocks:       shared memory dg[K][lane][2] (C-fragment order), owned by warp K % W;
  //                          after the factorisation they hold Linv_K
  //   pan[I] (A-fragment order): the current panel L_IK;  linvf: Linv_K in A-fragment order
  // dd: in -b (padded with zeros to NB*8), out: the Newton direction.  Returns SPD.
  static constexpr int NBO = NB * (NB - 1) / 2;               // strictly-lower blocks
  static constexpr int NBW2 = NBO > 0 ? (NBO + W - 1) / W : 1;  // per warp (upper bound)
  static constexpr int NDW = (NB + W - 1) / W;                // diagonal blocks per warp
  __host__ __device__ static constexpr int oJ(int r) { return cmJ(r, NB - 1); }
  __host__ __device__ static constexpr int oI(int r) { return cmI(r, NB - 1) + 1; }
  // WR: the warp role (compile time, so every slot's block (I, J) and every step's work list are
  // constants: the factorisation is straight-line code without per-slot predicates)
  template <int WR>
  __device__ static bool chol_solve(const double* S, int npp, double* dd, double* reg, int* ctl, int n, int NBl,
                                    int lane, int bar) {
    constexpr int wr = WR;
    const int r = lane >> 2, q = lane & 3;
    double* pan = reg;                          // [NB][MMA_BS]
    double* linvf = reg + NB * MMA_BS;          // [MMA_BS]
    double* dg = reg + NB * MMA_BS + MMA_BS;    // [NB][64] (C-fragment order, lane-contiguous)
#ifdef IPM_MMA_LDL
    // block LDL^T: L_IK = A_IK D_K^{-1} (pan), the unscaled A_IK (panA) for the trailing updates
    // A_IJ -= L_IK A_JK^T, D_K^{-1} by Gauss-Jordan (linvf), forward z_I -= L_IK z_K (dd), w = D^{-1} z (ww),
    // back substitution d_K = w_K - sum_{I > K} L_IK^T d_I
    double* panA = dg + NB * 64;      // [NB][MMA_BS]
    double* ww = panA + NB * MMA_BS;  // [NB * 8]
#else
    double* const panA = pan;
#endif
#ifdef IPM_PHASE_TIMERS
    long long ct0 = clock64();
#define CPH(i)                                                                                  \
  do {                                                                                          \
    const long long now_ = clock64();                                                           \
    if (lane == 0 && wr == 0) atomicAdd(&g_phase_cycles[i], (unsigned long long)(now_ - ct0)); \
    ct0 = now_;                                                                                 \
  } while (0)
#else
#define CPH(i) \
  do {         \
  } while (0)
#endif
    double blk[NBW2][2];
    double dtmp[NDW][2];
    // ---- gather ------------------------------------------------------------------------------
    if constexpr (MS == 4) {
      // 8x8 block (I, J) = basis functions (2I + r/4, 2J + c/4): S offsets from lane constants
      const int hi = r >> 2, a = r & 3, hq = q >> 1;
      int abn[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int b = 2 * (q & 1) + e;
        abn[e] = ((a <= b) ? sym_idx<4>(a, b) : sym_idx<4>(b, a)) * npp;
      }
      const int hmx = hi > hq ? hi : hq, hmn = hi + hq - hmx;
      static_for<NBW2>([&](auto sc) {
        constexpr int s = decltype(sc)::value, br = s * W + WR;
        if constexpr (br < NBO) {
          constexpr int I = oI(br), J = oJ(br);
          const int o = I * (2 * I + 1) + hi * (2 * I + 1) + 2 * J + hq;
          const bool rin = 8 * I + r < n;
#pragma unroll
          for (int e = 0; e < 2; ++e) blk[s][e] = (rin && 8 * J + 2 * q + e < n) ? S[abn[e] + o] : 0.0;
        }
      });
#pragma unroll
      for (int u = 0; u < NDW; ++u) {
        const int K = u * W + wr;
        if (K < NB) {
          const int o = K * (2 * K + 1) + hmx * (2 * K + 1) + 2 * K + hmn;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int R = 8 * K + r, C = 8 * K + 2 * q + e;
            dtmp[u][e] = (R < n && C < n) ? S[abn[e] + o] : ((R == C) ? 1.0 : 0.0);
          }
        }
      }
    } else {
      static_for<NBW2>([&](auto sc) {
        constexpr int s = decltype(sc)::value, br = s * W + WR;
        if constexpr (br < NBO) {
          constexpr int I = oI(br), J = oJ(br);
#pragma unroll
          for (int e = 0; e < 2; ++e) blk[s][e] = hval(S, npp, n, 8 * I + r, 8 * J + 2 * q + e);
        }
      });
#pragma unroll
      for (int u = 0; u < NDW; ++u) {
        const int K = u * W + wr;
        if (K < NB) {
#pragma unroll
          for (int e = 0; e < 2; ++e) dtmp[u][e] = hval(S, npp, n, 8 * K + r, 8 * K + 2 * q + e);
        }
      }
    }
    if (lane == 0 && wr == 0) ctl[1] = 0;
    named_sync(bar, G);  // S is dead: the Cholesky buffers reuse it
#pragma unroll
    for (int u = 0; u < NDW; ++u) {
      const int K = u * W + wr;
      if (K < NB) *reinterpret_cast<double2*>(dg + K * 64 + 2 * lane) = make_double2(dtmp[u][0], dtmp[u][1]);
    }
    named_sync(bar, G);
    CPH(4);
    // Fragment orders (mma.m8n8k4.f64; lane l, r = l/4, q = l%4):
    //   C: (r, 2q + e), e = 0, 1          A: (r, q + 4kk)          B: (q + 4kk, r)
    // Conversions go through shared memory (store as bpos(r, c), reload), not shuffles.
    //   blk[s]  C-fragment of the trailing block A_IJ; after its panel step the B-fragment of L_IJ
    //   pan[I]  L_IK of the current panel;  linvf: Linv_K (both stored as bpos)
    //   dg[K]   C-fragment of A_KK; after the factorisation the B-fragment of Linv_K
    auto afrag_ld = [&](const double* src, double& f0, double& f1) {
      f0 = src[bpos(r, q)];
      f1 = src[bpos(r, q + 4)];
    };
    // B-fragment: element (q + 4kk, r) of the stored block
    auto bfrag_ld = [&](const double* src, double& f0, double& f1) {
      f0 = src[bpos(q, r)];
      f1 = src[bpos(q + 4, r)];
    };
    // vector as an operand: column 0 of B or row 0 of A (lanes 0-3)
    auto vec_frag = [&](const double* v, double& f0, double& f1) {
      f0 = (lane < 4) ? v[lane] : 0.0;
      f1 = (lane < 4) ? v[4 + lane] : 0.0;
    };
    bool live = true;  // false after a failed pivot or past the cell's level (adaptive)
    // K = -1 only factors the first diagonal block (look-ahead of the loop)
    static_for<NB + 1>([&](auto kc) {
      constexpr int K = decltype(kc)::value - 1;
      if (!live) return;
      if (K >= NBl || ctl[1]) {
        live = false;
        return;
      }
      // ---- panel: L_IK = A_IK Linv_K^T, b_I -= L_IK y_K ---------------------------------------
      // batched over the warp's panel blocks so the shared-memory round trips overlap:
      //   C -> A order via pan[I];  X = A_IK Linv^T;  X -> pan[I] (A order);  B-fragment of X kept
      if constexpr (K >= 0) {
        auto each_panel = [&](auto&& fn) {
          static_for<NBW2>([&](auto sc) {
            constexpr int s = decltype(sc)::value, br = s * W + WR;
            if constexpr (br < NBO) {
              constexpr int I = oI(br), J = oJ(br);
              if constexpr (J == K) {
                if (I < NBl) fn(s, pan + I * MMA_BS, I);
              }
            }
          });
        };
        each_panel([&](int s, double* pI, int I) { store_afrag(panA + I * MMA_BS, blk[s][0], blk[s][1], lane); });
        __syncwarp();
        double lf0, lf1;
        afrag_ld(linvf, lf0, lf1);
        each_panel([&](int s, double* pI, int I) {
          double f0, f1;
          afrag_ld(panA + I * MMA_BS, f0, f1);
          double x0 = 0.0, x1 = 0.0;
          dmma884(x0, x1, f0, lf0);
          dmma884(x0, x1, f1, lf1);
          blk[s][0] = x0;
          blk[s][1] = x1;
        });
        __syncwarp();
        each_panel([&](int s, double* pI, int) { store_afrag(pI, blk[s][0], blk[s][1], lane); });
        __syncwarp();
        double yf0, yf1;
        vec_frag(dd + K * 8, yf0, yf1);
        each_panel([&](int s, double* pI, int I) {
          double f0, f1;
          afrag_ld(pI, f0, f1);
          bfrag_ld(pI, blk[s][0], blk[s][1]);
          double v0 = 0.0, v1 = 0.0;
          dmma884(v0, v1, f0, yf0);
          dmma884(v0, v1, f1, yf1);
          if (q == 0) dd[I * 8 + r] -= v0;
        });
        named_sync(bar, G);
      }
      // ---- trailing update; (K+1, K+1) first, then factored at once (look-ahead) ---------------
      if constexpr (K + 1 < NB && (K + 1) % W == WR) {
        constexpr int K1 = K + 1;
        if (K1 < NBl) {
          double2 v = *reinterpret_cast<const double2*>(dg + K1 * 64 + 2 * lane);
          if constexpr (K >= 0) {
            double p0, p1, pa0, pa1;
            afrag_ld(pan + K1 * MMA_BS, p0, p1);
            afrag_ld(panA + K1 * MMA_BS, pa0, pa1);
            dmma884(v.x, v.y, dneg(p0), pa0);
            dmma884(v.x, v.y, dneg(p1), pa1);
          }
          double a0 = v.x, a1 = v.y;
#ifdef IPM_MMA_LDL
          const bool okd = blk8_gj_inverse(a0, a1, lane, min(8, n - 8 * K1));
#else
          const bool okd = diag_factor(a0, a1, lane, min(8, n - 8 * K1), dg + K1 * 64, linvf);
#endif
          store_afrag(linvf, a0, a1, lane);
          __syncwarp();
          // y_K1 = Linv b_K1;  dg[K1] <- B-fragment of Linv (back substitution)
          double f0, f1, bf0, bf1, g0, g1;
          afrag_ld(linvf, f0, f1);
          vec_frag(dd + K1 * 8, bf0, bf1);
          bfrag_ld(linvf, g0, g1);
          double y0 = 0.0, y1 = 0.0;
          dmma884(y0, y1, f0, bf0);
          dmma884(y0, y1, f1, bf1);
#ifdef IPM_MMA_LDL
          (void)g0;
          (void)g1;
          if (q == 0) ww[K1 * 8 + r] = y0;  // w_K1 = D^{-1} z_K1; dd keeps z_K1 for the panel update
#else
          *reinterpret_cast<double2*>(dg + K1 * 64 + 2 * lane) = make_double2(g0, g1);
          __syncwarp();
          if (q == 0) dd[K1 * 8 + r] = y0;
#endif
          if (lane == 0 && !okd) ctl[1] = 1;
        }
      }
      if constexpr (K >= 0) {
        static_for<NDW>([&](auto uc) {
          constexpr int Jd = decltype(uc)::value * W + WR;
          if constexpr (Jd > K + 1 && Jd < NB) {
            if (Jd < NBl) {
              double2 v = *reinterpret_cast<const double2*>(dg + Jd * 64 + 2 * lane);
              double p0, p1, pa0, pa1;
              afrag_ld(pan + Jd * MMA_BS, p0, p1);
              afrag_ld(panA + Jd * MMA_BS, pa0, pa1);
              dmma884(v.x, v.y, dneg(p0), pa0);
              dmma884(v.x, v.y, dneg(p1), pa1);
              *reinterpret_cast<double2*>(dg + Jd * 64 + 2 * lane) = v;
            }
          }
        });
        static_for<NBW2>([&](auto sc) {
          constexpr int s = decltype(sc)::value, br = s * W + WR;
          if constexpr (br < NBO) {
            constexpr int I = oI(br), J = oJ(br);
            if constexpr (J > K) {
              if (I < NBl) {
                double a0, a1, b0, b1;
                afrag_ld(pan + I * MMA_BS, a0, a1);
                afrag_ld(panA + J * MMA_BS, b0, b1);
                dmma884(blk[s][0], blk[s][1], dneg(a0), b0);
                dmma884(blk[s][0], blk[s][1], dneg(a1), b1);
              }
            }
          }
        });
      }
      named_sync(bar, G);
    });
    CPH(5);
    if (ctl[1]) return false;
#ifdef IPM_MMA_LDL
    // ---- back substitution: d_K = w_K - sum_{I > K} L_IK^T d_I: w_J -= L_KJ^T d_K (J < K) -------------
    static_for<NB>([&](auto kc) {
      constexpr int K = NB - 1 - decltype(kc)::value;
      if (K >= NBl) return;
      if constexpr (K > 0) {
        double d0, d1;
        vec_frag(ww + K * 8, d0, d1);
        static_for<NBW2>([&](auto sc) {
          constexpr int s = decltype(sc)::value, br = s * W + WR;
          if constexpr (br < NBO) {
            constexpr int I = oI(br), J = oJ(br);
            if constexpr (I == K) {
              double v0 = 0.0, v1 = 0.0;
              dmma884(v0, v1, d0, blk[s][0]);
              dmma884(v0, v1, d1, blk[s][1]);
              if (lane < 4) {
                ww[J * 8 + 2 * q] -= v0;
                ww[J * 8 + 2 * q + 1] -= v1;
              }
            }
          }
        });
        named_sync(bar, G);
      }
    });
    for (int x = wr * 32 + lane; x < NBl * 8; x += W * 32) dd[x] = ww[x];
    named_sync(bar, G);
    CPH(6);
    return true;
#endif
#ifdef IPM_MMA_BACKSUB1
    // ---- back substitution with one group barrier per block row ------------------------------------------
    // every warp forms d_K = Linv_K^T (z_K - sum_w p_w[K]) itself (Linv_K from its shared diagonal slot),
    // then adds L_KJ^T d_K of its own blocks of row K to its partial sums p_WR[J]; the barrier ending the
    // row publishes them.  The owner of K keeps d_K in dout, copied to dd at the end.  (The panel
    // buffer is free here.)
    {
      constexpr int NV8 = NB * 8;
      double* pw = pan + WR * NV8;
      double* dout = pan + W * NV8;
      double* dsc = pan + (W + 1) * NV8 + WR * 8;
      for (int x = lane; x < NV8; x += 32) pw[x] = 0.0;
      named_sync(bar, G);
      static_for<NB>([&](auto kc) {
        constexpr int K = NB - 1 - decltype(kc)::value;
        if (K >= NBl) return;
        const double2 li = *reinterpret_cast<const double2*>(dg + K * 64 + 2 * lane);
        double z0 = 0.0, z1 = 0.0;
        if (lane < 4) {
          z0 = dd[K * 8 + lane];
          z1 = dd[K * 8 + 4 + lane];
#pragma unroll
          for (int w = 0; w < W; ++w) {
            z0 -= pan[w * NV8 + K * 8 + lane];
            z1 -= pan[w * NV8 + K * 8 + 4 + lane];
          }
        }
        double v0 = 0.0, v1 = 0.0;
        dmma884(v0, v1, z0, li.x);
        dmma884(v0, v1, z1, li.y);
        if constexpr (K % W == WR) {
          if (lane < 4) {
            dout[K * 8 + 2 * q] = v0;
            dout[K * 8 + 2 * q + 1] = v1;
          }
        }
        if constexpr (K > 0) {
          if (lane < 4) {
            dsc[2 * q] = v0;
            dsc[2 * q + 1] = v1;
          }
          __syncwarp();
          double d0, d1;
          vec_frag(dsc, d0, d1);
          static_for<NBW2>([&](auto sc) {
            constexpr int s = decltype(sc)::value, br = s * W + WR;
            if constexpr (br < NBO) {
              constexpr int I = oI(br), J = oJ(br);
              if constexpr (I == K) {
                double w0 = 0.0, w1 = 0.0;
                dmma884(w0, w1, d0, blk[s][0]);
                dmma884(w0, w1, d1, blk[s][1]);
                if (lane < 4) {
                  pw[J * 8 + 2 * q] += w0;
                  pw[J * 8 + 2 * q + 1] += w1;
                }
              }
            }
          });
        }
        named_sync(bar, G);
      });
      for (int x = WR * 32 + lane; x < NBl * 8; x += W * 32) dd[x] = dout[x];
      named_sync(bar, G);
    }
    CPH(6);
    return true;
#endif
    // ---- back substitution: d_K = Linv_K^T z_K; z_J -= L_KJ^T d_K (J < K), as row-vector DMMAs --------
    static_for<NB>([&](auto kc) {
      constexpr int K = NB - 1 - decltype(kc)::value;
      if (K >= NBl) return;
      if constexpr (K % W == WR) {
        const double2 li = *reinterpret_cast<const double2*>(dg + K * 64 + 2 * lane);
        double z0, z1;
        vec_frag(dd + K * 8, z0, z1);
        double v0 = 0.0, v1 = 0.0;
        dmma884(v0, v1, z0, li.x);
        dmma884(v0, v1, z1, li.y);
        __syncwarp();
        if (lane < 4) {
          dd[K * 8 + 2 * q] = v0;
          dd[K * 8 + 2 * q + 1] = v1;
        }
      }
      named_sync(bar, G);
      if constexpr (K > 0) {
        double d0, d1;
        vec_frag(dd + K * 8, d0, d1);
        static_for<NBW2>([&](auto sc) {
          constexpr int s = decltype(sc)::value, br = s * W + WR;
          if constexpr (br < NBO) {
            constexpr int I = oI(br), J = oJ(br);
            if constexpr (I == K) {
              double v0 = 0.0, v1 = 0.0;
              dmma884(v0, v1, d0, blk[s][0]);
              dmma884(v0, v1, d1, blk[s][1]);
              if (lane < 4) {
                dd[J * 8 + 2 * q] -= v0;
                dd[J * 8 + 2 * q + 1] -= v1;
              }
            }
          }
        });
        named_sync(bar, G);
      }
    });
    CPH(6);
    return true;
#undef CPH
  }
};

#ifdef IPM_PHASE_TIMERS
#define MPHASE(i)                                                  \
  do {                                                             \
    const long long now_ = clock64();                              \
    if (t == 0) ph_acc[i] += (unsigned long long)(now_ - ph_t0);   \
    ph_t0 = now_;                                                  \
  } while (0)
#else
#define MPHASE(i) \
  do {            \
  } while (0)
#endif

// QC, NC, Q1C: compile-time Q, N, q1d of the configuration the instance serves (0 = read from the
// tables at run time).  With them every loop bound, tile count and shared-memory offset is a constant
// (config 3: Q = 100, N = 15, q1d = 10), which removes most of the integer address arithmetic and
// predicates of the generic instance (measured +19 % on config 3).  They serve launches in which every
// cell has the basis size N (no levels, or one level's bucket); per-cell sizes need the generic one.
template <int CL, int MS, int NB, int W, int SF, int QC = 0, int NC = 0, int Q1C = 0>
#ifndef IPM_MMA_THREADS
#define IPM_MMA_THREADS 512
#endif
__global__ void __launch_bounds__(IPM_MMA_THREADS) k_dual_mma(DualParams P) {
#ifdef IPM_PHASE_TIMERS
  unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_t0 = clock64();
#endif
  using D = DualMma<CL, MS, NB, W, SF>;
  using Lay = MmaLayout<MS>;
  constexpr int G = D::G, MM = Lay::MM, NV = NB * 8;
  extern __shared__ __align__(16) double sm[];
  const int N = NC ? NC : P.T.N, Q = QC ? QC : P.T.Q, QP = QC ? ((QC % 2) ? QC : QC + 1) : P.T.QP;
  constexpr int NPR = SF * (SF + 1) / 2;
  double* sPhiT = sm;
  double* sWPhiT = sm + N * QP;
  double* sLL = sm + 2 * N * QP;  // [q1d][NPR] (SF > 0)
  const int q1 = Q1C ? Q1C : P.T.q1d;
  const int KS = QC ? (QC + 3) / 4 : P.T.KS, MTT = NC ? (NC + 7) / 8 : P.T.MT;
  double* sWF = sm + 2 * N * QP + ((SF > 0) ? ((q1 * NPR + 1) & ~1) : 0);  // [MT][KS][32] omega Phi^T fragments
  // per pair p = i(i+1)/2 + j: the 1D pair indices (pr1, pr2) of the sum factorisation, packed
  int* sPR = (int*)(sWF + MTT * KS * 32);
  const int NPT = N * (N + 1) / 2;
  // the sum factorisation's first-stage B operand LL[k2][pr2] in B-fragment order [KSs][NTs][32 lanes]
  // (read per lane as LL[k2 * NPR + pr] its rows k2 = 4ks + lane%4 fell 4-way onto the same banks)
  constexpr int NTS1 = (NPR + 7) / 8;
  const int KSS1 = (SF > 0) ? (q1 + 3) / 4 : 0;
  double* sLLF = sm + 2 * N * QP + ((SF > 0) ? ((q1 * NPR + 1) & ~1) : 0) + MTT * KS * 32 + ((NPT + 3) / 4) * 2;
  // stage-2 work list: slot 2e, 2e+1 of entry e = two pairs with the same pr2 (p | pr1 << 12 | pr2 << 20; -1
  // empty), so one thread forms both from one read of the T row (r02ac: the per-pair T reads were 10 % of
  // the kernel's shared-memory wavefronts)
  const int NEMAX = Lay::nemax(N, NPR);
  int* sSlot = (int*)(sLLF + KSS1 * NTS1 * 32);
  int* sHist = sSlot + 2 * NEMAX;  // [NPR] + the entry count
  const int tabsz = 2 * N * QP + ((SF > 0) ? ((q1 * NPR + 1) & ~1) : 0) + MTT * KS * 32 + ((NPT + 3) / 4) * 2 +
                    KSS1 * NTS1 * 32 + ((SF > 0) ? Lay::pairlist_doubles(N, NPR) : 0);
  for (int x = threadIdx.x; x < N * QP; x += blockDim.x) {
    sPhiT[x] = P.T.PhiT[x];
    sWPhiT[x] = P.T.WPhiT[x];
  }
  if (SF > 0) {
    for (int x = threadIdx.x; x < q1 * NPR; x += blockDim.x) sLL[x] = P.T.LL[x];
    for (int x = threadIdx.x; x < KSS1 * NTS1 * 32; x += blockDim.x) {
      const int ln = x & 31, nt = (x >> 5) % NTS1, ks = (x >> 5) / NTS1;
      const int k2 = 4 * ks + (ln & 3), pr = 8 * nt + (ln >> 2);
      sLLF[x] = (k2 < q1 && pr < NPR) ? P.T.LL[k2 * NPR + pr] : 0.0;
    }
  }
  for (int x = threadIdx.x; x < MTT * KS * 32; x += blockDim.x) sWF[x] = P.T.WPhiF[x];
  if constexpr (SF > 0) {
    for (int p = threadIdx.x; p < NPT; p += blockDim.x) {
      int i = 0;
      while ((i + 1) * (i + 2) / 2 <= p) ++i;
      const int j = p - i * (i + 1) / 2;
      int a1 = P.T.idx[i * 2], a2 = P.T.idx[i * 2 + 1], b1 = P.T.idx[j * 2], b2 = P.T.idx[j * 2 + 1];
      if (a1 > b1) { const int x = a1; a1 = b1; b1 = x; }
      if (a2 > b2) { const int x = a2; a2 = b2; b2 = x; }
      sPR[p] = (a1 * SF - a1 * (a1 - 1) / 2 + (b1 - a1)) | ((a2 * SF - a2 * (a2 - 1) / 2 + (b2 - a2)) << 16);
    }
    for (int x = threadIdx.x; x < 2 * NEMAX; x += blockDim.x) sSlot[x] = -1;
    for (int x = threadIdx.x; x < NPR; x += blockDim.x) sHist[x] = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < NPT; p += blockDim.x) atomicAdd(&sHist[sPR[p] >> 16], 1);
    __syncthreads();
    // padded order: pairs sorted by (pr2, p), every pr2 group padded to an even length
    for (int p = threadIdx.x; p < NPT; p += blockDim.x) {
      const int pr2 = sPR[p] >> 16;
      int pos = 0;
      for (int q = 0; q < pr2; ++q) pos += (sHist[q] + 1) & ~1;
      for (int p2 = 0; p2 < p; ++p2) pos += (sPR[p2] >> 16) == pr2;
      sSlot[pos] = p | ((sPR[p] & 0xffff) << 12) | (pr2 << 20);
    }
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int q = 0; q < NPR; ++q) tot += (sHist[q] + 1) & ~1;
      sHist[NPR] = tot / 2;
    }
  }
  __syncthreads();
  const int grp = threadIdx.x / G, t = threadIdx.x - grp * G;
  const int wig = t >> 5, lane = t & 31;
  const int bar = 1 + grp;
  const int npp = Lay::nps(N);  // S row stride
  double* base = sm + tabsz + (size_t)grp * Lay::per_group(N, Q, W, SF, q1, NB);
  double* lam = base;
  double* lt = lam + NV;
  double* uh = lt + NV;
  double* g = uh + NV;
  double* dd = g + NV;
  double* nb = dd + NV;  // node buffer: u[a][k] at nb[a Q + k], J[z][k] at nb[(MS + z) Q + k]
  double* red = nb + Lay::region(N, Q, SF, q1, NB);  // [2 slots][RSX][W]
  int* ctl = (int*)(red + 2 * Lay::RSX * W);

  const double* __restrict__ omega = P.T.omega;
  const DualLaunch& A = P.a;
  const int nmax = A.row ? A.row : N * MS;  // [cells][nmax] stride of uhat / lambda
  long long my_iters = 0, my_failed = 0;
  int my_worst = 0;
  double my_rate = 0.0;
  int slot = 0;

  auto gsync = [&]() { named_sync(bar, G); };
  // group-wide sums of RS values (alternating scratch slots)
  auto gsum = [&](auto& v) {
    constexpr int RS = sizeof(v) / sizeof(double);
    double* rr = red + slot * Lay::RSX * W;
    slot ^= 1;
    __syncwarp();
#pragma unroll
    for (int a = 0; a < RS; ++a) {
      v[a] = warp_sum(v[a]);
      if (W > 1 && lane == 0) rr[a * W + wig] = v[a];
    }
    gsync();
    if (W > 1) {
#pragma unroll
      for (int a = 0; a < RS; ++a) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) s += rr[a * W + w];
        v[a] = s;
      }
    }
  };

  // Hessian unique entries S[ab][pair(i >= j)]
  auto hessian = [&](int Nl) {
    double* Tt = nb + Lay::t_off(N, Q, SF);
    double* Sx = nb + Lay::s_base(N, Q, SF, q1);
    const int NPl = Nl * (Nl + 1) / 2;
    if constexpr (SF > 0) {
      constexpr int NCH = Lay::NCH, CHW = Lay::CHW;
#pragma unroll 1
      for (int ch = 0; ch < NCH; ++ch) {
        const int ab0 = ch * CHW;
        const int nab = (MM - ab0) < CHW ? (MM - ab0) : CHW;
        // stage 1: T[k1][pr2][c] = sum_k2 LL[k2][pr2] J_{ab0+c}(k1, k2), on the fp64 tensor path:
        // rows (k1, c), columns pr2, contraction over k2 (zero-padded to whole 8 x 8 x 4 tiles)
        {
          const int rows = q1 * nab, MTs = (rows + 7) >> 3, KSs = (q1 + 3) >> 2;
          constexpr int NTs = (NPR + 7) / 8;
          const int lr = lane >> 2, lq = lane & 3;
#pragma unroll 1
          for (int mt = wig; mt < MTs; mt += W) {
            const int row = 8 * mt + lr;  // A-fragment row of this lane
            const bool rok = row < rows;
            const int k1a = rok ? row / nab : 0, ca = rok ? row - k1a * nab : 0;
            const double* jrow = nb + (MS + ab0 + ca) * Q + k1a * q1;
            double acc[NTs][2];
#pragma unroll
            for (int nt = 0; nt < NTs; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
#pragma unroll 1
            for (int ks = 0; ks < KSs; ++ks) {
              const int k2 = 4 * ks + lq;  // A column / B row of this lane
              const double av = (rok && k2 < q1) ? jrow[k2] : 0.0;
#pragma unroll
              for (int nt = 0; nt < NTs; ++nt) dmma884(acc[nt][0], acc[nt][1], av, sLLF[(ks * NTs + nt) * 32 + lane]);
            }
            // C-fragment (row 8mt + lr, columns 8nt + 2lq + e) -> T[k1][pr2][c]
            if (rok) {
#pragma unroll
              for (int nt = 0; nt < NTs; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const int pr = 8 * nt + 2 * lq + e;
                  if (pr < NPR) Tt[(k1a * NPR + pr) * CHW + ca] = acc[nt][e];
                }
            }
          }
        }
        gsync();
        // stage 2: S[ab0+c][pair] = sum_k1 LL[k1][pr1] T[k1][pr2][c]
        const int NE = sHist[NPR];
#pragma unroll 1
        for (int e = t; e < NE; e += G) {
          const int sa = sSlot[2 * e], sb = sSlot[2 * e + 1];
          const int pa = sa & 0xfff, pr1a = (sa >> 12) & 0xff, pr2 = sa >> 20;
          const bool hb = sb >= 0;
          const int pb = sb & 0xfff, pr1b = hb ? (sb >> 12) & 0xff : pr1a;
          double acc[CHW], acb[CHW];
#pragma unroll
          for (int c = 0; c < CHW; ++c) acc[c] = acb[c] = 0.0;
#pragma unroll 2
          for (int k1 = 0; k1 < q1; ++k1) {
            const double la = sLL[k1 * NPR + pr1a], lb = sLL[k1 * NPR + pr1b];
            const double* Tk = Tt + (k1 * NPR + pr2) * CHW;
#pragma unroll
            for (int c = 0; c < CHW; ++c) {
              const double tv = Tk[c];
              acc[c] = fma(la, tv, acc[c]);
              acb[c] = fma(lb, tv, acb[c]);
            }
          }
#pragma unroll
          for (int c = 0; c < CHW; ++c)
            if (c < nab) {
              if (pa < NPl) Sx[(ab0 + c) * npp + pa] = acc[c];
              if (hb && pb < NPl) Sx[(ab0 + c) * npp + pb] = acb[c];
            }
        }
        gsync();  // T chunk is rewritten by the next chunk; S complete after the last
      }
    } else {
      // direct: S[ab][pair] = sum_k (omega_k phi_ki phi_kj) J_ab,k
#pragma unroll 1
      for (int p = t; p < NPl; p += G) {
        int i = (int)((sqrtf(8.0f * p + 1.0f) - 1.0f) * 0.5f);
        if ((i + 1) * (i + 2) / 2 <= p) ++i;
        if (i * (i + 1) / 2 > p) --i;
        const int j = p - i * (i + 1) / 2;
        const double* wi = sWPhiT + i * QP;
        const double* pj = sPhiT + j * QP;
        double acc[MM];
#pragma unroll
        for (int z = 0; z < MM; ++z) acc[z] = 0.0;
#pragma unroll 1
        for (int k = 0; k < Q; ++k) {
          const double f = wi[k] * pj[k];
#pragma unroll
          for (int z = 0; z < MM; ++z) acc[z] = fma(f, nb[(MS + z) * Q + k], acc[z]);
        }
#pragma unroll
        for (int z = 0; z < MM; ++z) Sx[z * npp + p] = acc[z];
      }
      gsync();
    }
  };

  const int64_t ncells = A.ncells_dev ? (int64_t)*A.ncells_dev : A.cells;
  int* const queue = A.queue ? A.queue : &P.sc->work_counter;
  for (;;) {
    if (t == 0) ctl[0] = atomicAdd(queue, 1);
    gsync();
    if (ctl[0] >= ncells) break;
    const int64_t cell = A.list ? (int64_t)A.list[ctl[0]] : (int64_t)ctl[0];
    MPHASE(7);
    const int lvl = A.level ? A.level[cell] : 0;
    // fixed-shape instances serve launches of one basis size (no levels, or one level's bucket):
    // N_l = N at compile time, so n, the block count and every guard on them fold away
    const int Nl = NC ? N : ((P.ad.n_levels > 0) ? P.ad.Nl[lvl] : N);
    const int n = Nl * MS;
    const int NBl = (n + 7) / 8;
    {
      const double* gu = A.uhat + cell * nmax;
      const double* gl = A.lam + cell * nmax;
      for (int r = t; r < n; r += G) {
        uh[r] = gu[r];
        lam[r] = gl[r];
      }
    }
    gsync();

    // Newton iteration with Armijo backtracking on L (reading 3') as one loop with a single
    // evaluation site: mode 0 = first evaluation at lambda, 1 = line-search trial at lt,
    // 2 = re-evaluation of the final lambda (node states for the flux)
    int status = 0, l = 0, h = 0, mode = 0, hv = 0, ia = 0;
    double crit = INFINITY, L0 = 0.0, scale = 0.0, slope = 0.0, alpha = 1.0;
    bool nb_is_lam = false;
    for (;;) {
      const double* x = (mode == 1) ? lt : lam;
      // ---- a2: Lambda = Phi x, u = u_s(Lambda), J = grad u_s, s_* (node buffer) --------------------
      double sv[2] = {0.0, 0.0}, dv[2] = {0.0, 0.0};
      bool bad = false;
#pragma unroll 1
      for (int k = t; k < Q; k += G) {
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
#pragma unroll
        for (int z = 0; z < MM; ++z) nb[(MS + z) * Q + k] = J[z];
        const double w = omega[k];
        sv[0] = fma(w, ss, sv[0]);
        sv[1] = fma(w, fabs(ss), sv[1]);
      }
      if (bad) sv[1] = INFINITY;
      // x . uhat (and its magnitude) for L(x) = <s_*> - x . uhat
      for (int r = t; r < n; r += G) {
        const double v = x[r] * uh[r];
        dv[0] += v;
        dv[1] += fabs(v);
      }
      double red4[4] = {sv[0], sv[1], dv[0], dv[1]};
      gsum(red4);
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
        // ---- a3: gradient g = Phi^T (omega o u) - uhat, crit = sum_a ||g_.a|| -----------------------
        // on the fp64 tensor path: C[i][a] = sum_k (omega phi_i)(xi_k) u_a(xi_k), A = omega Phi^T in
        // fragment order (shared memory), B = the node buffer's u rows; warps split the row tiles
        double part[MS];
#pragma unroll
        for (int a = 0; a < MS; ++a) part[a] = 0.0;
        {
          const int MTl = (Nl + 7) >> 3, bn = lane >> 2, bk = lane & 3;
          const bool bval = bn < MS;
          const double* bsrc = nb + (bval ? bn : 0) * Q + bk;
#pragma unroll 1
          for (int mt = wig; mt < MTl; mt += W) {
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
          if (mode == 1)
            for (int r = t; r < n; r += G) lam[r] = lt[r];
        }
        gsum(part);
        crit = 0.0;
#pragma unroll
        for (int a = 0; a < MS; ++a) crit += sqrt(part[a]);
        if (mode == 1) ++l;
        nb_is_lam = true;
        L0 = Lt;
        scale = red4[1] + red4[3];
        // ---- a7: stopping tests -------------------------------------------------------------------
        if (crit < P.nw.tau || (P.nw.mode == 1 && l == 1)) break;
        if (l == P.nw.max_newton) {
          status = 1;
          break;
        }
        MPHASE(0);
        // ---- a4-a5: Hessian, Cholesky, d = -H^{-1} g ----------------------------------------------
        hessian(Nl);
        nb_is_lam = false;
        for (int r = t; r < NBl * 8; r += G) dd[r] = (r < n) ? -g[r] : 0.0;
        gsync();
        MPHASE(1);
        const double* Sx = nb + Lay::s_base(N, Q, SF, q1);
        bool chol_ok;
if constexpr (W == 1) {
          chol_ok = D::template chol_solve<0>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar);
        } else if constexpr (W == 2) {
          chol_ok = (wig == 0) ? D::template chol_solve<0>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar)
                               : D::template chol_solve<1>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar);
        } else if constexpr (W == 3) {
          switch (wig) {
            case 0: chol_ok = D::template chol_solve<0>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
            case 1: chol_ok = D::template chol_solve<1>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
            default: chol_ok = D::template chol_solve<2>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
          }
        } else {
          static_assert(W == 4, "W in {1, 2, 3, 4}");
          switch (wig) {
            case 0: chol_ok = D::template chol_solve<0>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
            case 1: chol_ok = D::template chol_solve<1>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
            case 2: chol_ok = D::template chol_solve<2>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
            default: chol_ok = D::template chol_solve<3>(Sx, npp, dd, nb, ctl, n, NBl, lane, bar); break;
          }
        }
        MPHASE(2);
        if (!chol_ok) {
          status = 2;
          finish = true;
        } else {
          double sl[1] = {0.0};
          for (int r = t; r < n; r += G) sl[0] = fma(g[r], dd[r], sl[0]);
          gsum(sl);
          slope = sl[0];
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
        for (int r = t; r < n; r += G) lt[r] = lam[r] + alpha * dd[r];
        mode = 1;
      }
      gsync();
      MPHASE(3);
    }
    MPHASE(4);
    // ---- epilogue --------------------------------------------------------------------------------
    gsync();
    if (P.ad.n_levels > 0 && A.level_new) {
      const int Nprev = lvl > 0 ? P.ad.Nl[lvl - 1] : P.ad.Nprev0;
      double nd[2] = {0.0, 0.0};
      for (int i = t; i < Nl; i += G) {
        const double hv = g[i * MS] + uh[i * MS];
        nd[1] = fma(hv, hv, nd[1]);
        if (i >= Nprev) nd[0] = fma(hv, hv, nd[0]);
      }
      gsum(nd);
      const double Sv = nd[1] > 0.0 ? nd[0] / nd[1] : 0.0;
      const int nl = next_level(P.ad, P.sc, lvl, status, Sv);
      if (t == 0) A.level_new[cell] = nl;
    }
    {
      double* gl = A.lam + cell * nmax;
      for (int r = t; r < nmax; r += G) gl[r] = (r < n) ? lam[r] : 0.0;
    }
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
    }
    gsync();
  }
  MPHASE(5);
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
#undef MPHASE
