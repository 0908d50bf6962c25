// Strip-marching kinetic-flux kernel for row-major cartesian blocks (Euler 2D, Rusanov; m = 4).
// Included by ipm_kernels.cu after RusNode / FluxParams.
//
// What it computes is k_flux_cart's a11 + projection (PAPER.md:130 difference form per direction,
// PAPER.md:182-185 update forms), with every node's Rusanov ingredients formed ONCE and every face
// flux formed ONCE (k_flux_cart forms five ingredient sets and four faces per node):
//   * a CTA owns a strip of TX = 8 cell columns and walks its rows y = ya..yb-1 (a contiguous share
//     of all strip rows, so every CTA gets the same number of rows);
//   * the node states of the row's 8 cells and its two x-halo cells are TMA bulk copies (one per
//     cell: the node states are stored [cell][state][node]) into a 4-row shared-memory ring, three
//     rows ahead, completing on an mbarrier;
//   * compute warps: lane = (column c, node kk of a group of 4); each thread holds two node groups
//     for the whole walk and carries, per item, the current node state, its ingredients (1/rho, p,
//     c) and the y-face flux g_{y-1/2}; it forms the next row's ingredients and g_{y+1/2}, the east
//     x face from its east neighbour's (u, F_x, s_x) by warp shuffles, the west one by a shuffle of
//     that face (the strip's edge columns take the halo ingredients from shared memory), and then
//     r = (g_E - g_W)/dx + (g_N - g_S)/dy;
//   * halo warps form the x-halo ingredients of the next row (boundary states: ghost / slip wall /
//     outflow copy, k_flux_cart's rules); the last NPW warps (one per SM sub-partition) project the
//     previous row, Phi^T(omega o r), on DMMA with A = r^T (rows (cell, state), K = nodes) and
//     B = the WPhiF fragments, and write the update;
//   * one CTA barrier per row.

#ifndef IPM_FLUX_STRIP_CUH
#define IPM_FLUX_STRIP_CUH

namespace strip {

__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src) : "memory");
}
// TMA bulk copies (global -> shared) completing on an mbarrier
__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE;\n"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

constexpr int UNUSED = -2147483647 - 1;

__host__ __device__ constexpr int KS_(int QC) { return (QC + 3) / 4; }

template <int TX, int QC>
struct Layout {
  static constexpr int NC = TX + 2;  // ring columns: west halo, TX owned, east halo
  static constexpr int CT = TX / 2;  // DMMA row tiles of r^T (8 rows = 2 cells x 4 states)
  // ring column stride: 4 Q doubles + padding so that 4 columns x 4 nodes fall into distinct banks
  static constexpr int QMP = 4 * QC + ((4 - (4 * QC) % 16) + 16) % 16;
  // r^T row stride: room for the per-column k shift (4 (c & 3) doubles, bank spreading of the stores)
  // and = 4 mod 16 (the A-fragment loads of 8 rows x 4 k fill 16 banks per half warp)
  static constexpr int KP = ((KS_(QC) * 4 + 12 + 11) / 16) * 16 + 4;
  static constexpr int KS = KS_(QC), RB = CT * 8 * KP, HXS = 2 * 4 * QC;
  int MT;
  size_t a, ring, hx, rb, idx, bar, dm, total;  // offsets in doubles
  __host__ __device__ Layout(int MT_, int) : MT(MT_) {
    a = 0;
    ring = a + (size_t)MT * KS * 32;
    hx = ring + (size_t)4 * NC * QMP;
    rb = hx + (size_t)2 * HXS;
    idx = rb + (size_t)2 * RB;
    bar = idx + (8 * NC + 1) / 2;
    dm = bar + 4;  // SC mode: change of the mean per owned cell of the last two rows [2][TX]
    total = dm + 2 * TX;
  }
};

// Rusanov flux g(uL, uR) = (F(uL) + F(uR))/2 - max(sL, sR) (uR - uL)/2 (k_flux_cart's formula)
__device__ __forceinline__ void face(const double* fl, double sl, const double* ul, const double* fr, double sr,
                                     const double* ur, double* g) {
  const double amax = fmax(sl, sr);
#pragma unroll
  for (int a = 0; a < 4; ++a) g[a] = 0.5 * fma(-amax, ur[a] - ul[a], fl[a] + fr[a]);
}

// boundary node state for a face whose neighbour code is a boundary tag (k_flux_cart's rules)
__device__ __forceinline__ void bstate(const FluxParams& P, int code, int f, int k, const double* uref, double* ub) {
  const int tag = -1 - code;
  const int kind = P.mesh.bc_kind[tag];
  if (kind == 1) {
    const double* gs = P.mesh.ghost + ((int64_t)tag * P.T.Q + k) * 4;
#pragma unroll
    for (int a = 0; a < 4; ++a) ub[a] = gs[a];
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) ub[a] = uref[a];
    if (kind == 2) ub[1 + f / 2] = -uref[1 + f / 2];
  }
}

// node state of one node from a ring column [state][Q] (lanes over nodes: conflict-free)
template <int Q>
__device__ __forceinline__ void ld4(const double* p, double* u) {
#pragma unroll
  for (int a = 0; a < 4; ++a) u[a] = p[a * Q];
}

}  // namespace strip

#ifdef IPM_STRIP_PROF
#define STRIP_STAMP(n) \
  if (blockIdx.x == 0 && lane == 0 && it >= 20 && it < 24) st[(it - 20) * 4 + (n)] = clock64();
#else
#define STRIP_STAMP(n)
#endif

// SC = true: the Stochastic Collocation node update (reading 32) on the same walk: every node state
// is advanced, u_k - dt r_k -> P.a.uhat_new [cells][m][Q], instead of projected; the change of each
// cell's mean goes to the residual and the CFL rate of the new states to sc_rate_next.
template <int TX, int NT, int MINB, int QC, bool SC = false>
__global__ void __launch_bounds__(NT, MINB) k_flux_strip(FluxParams P) {
  using L = strip::Layout<TX, QC>;
  constexpr int NC = L::NC, CT = L::CT, QMP = L::QMP, KS = L::KS, KP = L::KP, RB = L::RB, HXS = L::HXS;
  constexpr int Q = QC, G = (QC + 3) / 4;  // node groups of 4 (one per 4 lanes x 8 columns warp slot)
#ifndef IPM_STRIP_SLOTS
#define IPM_STRIP_SLOTS 2
#endif
  constexpr int SL = IPM_STRIP_SLOTS;      // node groups per compute thread
  constexpr int CW = (G + SL - 1) / SL;    // compute warps
  constexpr int NW = NT / 32, HT0 = CW * 32, NTH = NT - HT0;  // halo threads [HT0, NT)
  constexpr int NPW = 4;                                       // projection warps: the last NPW
  static_assert(TX == 8 && NTH >= 32 && CW <= NW - 1 && CT % NPW == 0, "strip kernel geometry");
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, MT = P.T.MT, nmax = N * 4;
  const L lay(MT, nmax);
  double* sA = sm + lay.a;
  double* ring = sm + lay.ring;  // [4 rows][NC][4][Q] (+pad): node states of the row's cells
  double* HX = sm + lay.hx;      // [2 rows][2 sides][4][Q]: x fluxes at the strip's west / east faces
  double* rbT = sm + lay.rb;     // [2 rows][CT][8][KP]: r^T
  int* sidx = reinterpret_cast<int*>(sm + lay.idx);  // [8 rows][NC] cell codes
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + lay.bar);
  double* dmean = sm + lay.dm;  // SC
  double my_rate = 0.0;         // SC
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int b = 0; b < 4; ++b) strip::mbar_init(mbar + b, 1);
    strip::fence_mbar_init();
  }
  unsigned rows_done = 0;  // ring rows issued by this CTA before the current segment (mbarrier phases)
  for (int x = tid; x < MT * KS * 32; x += NT) sA[x] = P.T.WPhiF[x];
  for (int x = tid; x < 2 * RB; x += NT) rbT[x] = 0.0;  // K padding (k >= Q) stays 0
  if (tid < 2 * TX) dmean[tid] = 0.0;
  __syncthreads();

  const int bx = P.mesh.bx, by = P.mesh.by;
  const int nstrips = (bx + TX - 1) / TX;
  const int64_t R = (int64_t)nstrips * by;
  const int64_t g1 = R * (blockIdx.x + 1) / gridDim.x;
  const double dt = P.sc->dt, gam = P.cl.gamma;
  const double cfx = P.mesh.inv_dx, cfy = P.mesh.inv_dy;
  const FluxLaunch& A = P.a;
  const int32_t* nbr = P.mesh.nbr;
  const bool cform = A.update_form == 1;
  double my_res = 0.0;

  // compute-warp items: column c, node k = 4 (2 warp + sl) + kk
  const int c = lane >> 2;
  int kq[SL];  // node, clamped to a valid one for idle items (they only feed shuffles)
  bool kv[SL];
#pragma unroll
  for (int sl = 0; sl < SL; ++sl) {
    const int k = 4 * (SL * warp + sl) + (lane & 3);
    kv[sl] = warp < CW && k < Q;
    kq[sl] = k < Q ? k : Q - 1;
  }
  // r^T rows of tile ct = c/2: (cell c&1, state a) -> row 4 (c&1) + a; column c's node k is stored at
  // k + 4 (c & 3), so that the 8 columns' stores of one state fall into 4 distinct bank groups (the
  // projection's A-fragment loads add the same shift)
  const int bo = (c >> 1) * 8 * KP + (c & 1) * 4 * KP + 4 * (c & 3);  // row block + k shift
#ifdef IPM_STRIP_PROF
  long long st[16];
  bool first_seg = true;
#endif

  // Work split. With at least one CTA per strip (gridDim >= nstrips) the first nstrips CTAs walk rows
  // [0, RA) of strip b side by side, so the x-halo cells one CTA reads were just read by its
  // neighbour (L2 hits); the other CTAs share the rows [RA, by) of all strips, contiguous in
  // strip-major order; RA = the rows per CTA of an even split.  Otherwise: contiguous strip-major
  // shares of all strip rows.
  const bool banded = (int64_t)gridDim.x >= nstrips && gridDim.x > 1;
  const int64_t RA0 = (R + gridDim.x - 1) / gridDim.x;
  const int RA = banded ? (int)(RA0 < by ? RA0 : by) : 0;
  int64_t ga, gb;  // this CTA's range in its ordering
  if (!banded) {
    ga = R * blockIdx.x / gridDim.x;
    gb = g1;
  } else if ((int)blockIdx.x < nstrips) {
    ga = 0;
    gb = 0;  // band A handled below
  } else {
    const int64_t RB = (int64_t)nstrips * (by - RA), G2 = gridDim.x - nstrips, b2 = blockIdx.x - nstrips;
    ga = RB * b2 / G2;
    gb = RB * (b2 + 1) / G2;
  }
  const bool bandA = banded && (int)blockIdx.x < nstrips && RA > 0;
  for (int64_t g = bandA ? -1 : ga; bandA ? g < 0 : g < gb;) {
    int s, ya, yb;
    if (bandA) {
      s = blockIdx.x;
      ya = 0;
      yb = RA;
      g = 0;
    } else if (banded) {  // band B: rows RA..by-1 of every strip
      const int hb = by - RA;
      s = (int)(g / hb);
      ya = RA + (int)(g - (int64_t)s * hb);
      const int64_t ybl = ya + (gb - g);
      yb = ybl < by ? (int)ybl : by;
      g += yb - ya;
    } else {
      s = (int)(g / by);
      ya = (int)(g - (int64_t)s * by);
      const int64_t ybl = ya + (gb - g);
      yb = ybl < by ? (int)ybl : by;
      g += yb - ya;
    }
    const int x0 = s * TX, tw = min(TX, bx - x0);
    const int LR = yb - ya + 2;  // ring rows ya-1 .. yb

    // cell index (>= 0), boundary code (< 0) or UNUSED of ring row it (y = ya-1+it), column slot j
    auto row_code = [&](int it, int j) -> int {
      const int y = ya - 1 + it;
      if (j == 0 || j == tw + 1) {
        if (y < ya || y >= yb) return strip::UNUSED;
        const int64_t edge = (int64_t)y * bx + (j == 0 ? x0 : x0 + tw - 1);
        return nbr[edge * 4 + (j == 0 ? 0 : 1)];
      }
      if (j > tw) return strip::UNUSED;
      const int x = x0 + j - 1;
      if (y >= 0 && y < by) return y * bx + x;
      if (y < 0) return nbr[(int64_t)x * 4 + 2];
      return nbr[((int64_t)(by - 1) * bx + x) * 4 + 3];
    };
    // one thread: TMA bulk copies of ring row it (node states of its cells)
    auto issue_row = [&](int it) {
      const int* code = sidx + (it & 7) * NC;
      double* dst = ring + (it & 3) * NC * QMP;
      unsigned long long* bar = mbar + ((rows_done + it) & 3);
      unsigned bytes = 0;
      for (int col = 0; col < NC; ++col)
        if (code[col] >= 0) bytes += 4 * Q * 8;
      strip::mbar_expect_tx(bar, bytes);
      for (int col = 0; col < NC; ++col)
        if (code[col] >= 0) strip::bulk_g2s(dst + col * QMP, A.uq + (int64_t)code[col] * 4 * Q, 4 * Q * 8, bar);
    };
    auto wait_row = [&](int it) {
      const unsigned gi = rows_done + it;
      strip::mbar_wait(mbar + (gi & 3), (gi >> 2) & 1);
    };
    // projection of ring row itp: C^T = r^T (omega Phi^T) on DMMA, then the update of its cells
    auto project = [&](int itp) {
      const int y = ya - 1 + itp;
      const double* rb = rbT + (itp & 1) * RB;
      const int rr = lane >> 2, q = lane & 3, pw = warp - (NW - NPW);
      for (int ct = pw; ct < CT; ct += NPW) {
        const int av = rr & 3;
        const int cl = ct * 2 + (rr >> 2);
        const bool cv_ = cl < tw;
        const int64_t cell = (int64_t)y * bx + x0 + cl;
        const double area = (cv_ && q == 0 && av == 0) ? P.mesh.area[cell] : 0.0;
        const int Nnew = (cv_ && P.ad.n_levels > 0 && A.level_new) ? P.ad.Nl[A.level_new[cell]] : N;
        for (int mt0 = 0; mt0 < MT; mt0 += 2) {
          const bool two = mt0 + 1 < MT;
          double old[2][2];
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * (mt0 + m) + 2 * q + e;
              old[m][e] = (cv_ && i < N) ? A.uhat_old[cell * nmax + i * 4 + av] : 0.0;
            }
          double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
          const double* a = rb + ct * 8 * KP + rr * KP + q + 4 * ((2 * ct + (rr >> 2)) & 3);
          const double* b = sA + mt0 * KS * 32 + lane;
#pragma unroll 5
          for (int ks = 0; ks < KS; ++ks) {
            const double af = a[ks * 4];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[0][0]), "+d"(acc[0][1])
                         : "d"(af), "d"(b[ks * 32]));
            if (two)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                           : "+d"(acc[1][0]), "+d"(acc[1][1])
                           : "d"(af), "d"(b[(KS + ks) * 32]));
          }
          if (!cv_) continue;
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int i = 8 * (mt0 + m) + 2 * q + e;
              if (i >= N) continue;
              const int64_t idx = cell * nmax + i * 4 + av;
              double out = 0.0;
              if (i < Nnew) out = cform ? acc[m][e] : old[m][e] - dt * acc[m][e];
              A.uhat_new[idx] = out;
              if (i == 0 && av == 0) my_res += area * fabs(out - old[m][e]);
              if (A.lam && i >= Nnew) A.lam[idx] = 0.0;
            }
        }
      }
    };

    // SC: residual contribution of ring row itp, sum |Omega_j| |change of the mean|, then clear
    auto sc_residual = [&](int itp) {
      if (lane < tw) {
        double* d = dmean + (itp & 1) * TX + lane;
        my_res += P.mesh.area[(int64_t)(ya - 1 + itp) * bx + x0 + lane] * fabs(*d);
        *d = 0.0;
      }
    };

    int pend = 0;  // codes are loaded one iteration before they are stored (nbr latency off the barrier path)
    if (tid < NC) {
      for (int it = 0; it < 4 && it < LR; ++it) sidx[it * NC + tid] = row_code(it, tid);
      if (4 < LR) pend = row_code(4, tid);
    }
    __syncthreads();
    if (tid == NT - 1)
      for (int it = 0; it < 3 && it < LR; ++it) issue_row(it);

    // per-item carried state: node state, its ingredients, the south face flux
    double cu[SL][4], cir[SL], cp[SL], cc_[SL], gS[SL][4];
    bool act[SL];
#pragma unroll
    for (int sl = 0; sl < SL; ++sl) act[sl] = kv[sl] && c < tw;
    const int ro0 = ((c < tw ? c : tw - 1) + 1) * QMP;  // idle columns read the last owned one

    for (int it = 0; it + 1 < LR; ++it) {
      if (it == 0) wait_row(0);
      wait_row(it + 1);
      __syncthreads();  // rows <= it+1 in the ring; halo of row it in HX; r^T of row it-1 complete
      STRIP_STAMP(0)
      if (tid == NT - 1 && it + 3 < LR) issue_row(it + 3);
      if (tid < NC && it + 4 < LR) {
        sidx[((it + 4) & 7) * NC + tid] = pend;
        if (it + 5 < LR) pend = row_code(it + 5, tid);
      }
      const int* codeC = sidx + (it & 7) * NC;
      const int* codeN = sidx + ((it + 1) & 7) * NC;
      const double* rC = ring + (it & 3) * NC * QMP;
      const double* rN = ring + ((it + 1) & 3) * NC * QMP;
      const bool own_row = it > 0;
      const bool general = it == 0 || it + 2 == LR;  // rows that may hold boundary states

      if (warp < CW) {
        const double* hxr = HX + (it & 1) * HXS;  // strip-edge x fluxes of the current row
        double* rb = rbT + (it & 1) * RB;
        double un[SL][4];
        if (!general) {
#pragma unroll
          for (int sl = 0; sl < SL; ++sl) strip::ld4<Q>(rN + ro0 + kq[sl], un[sl]);
        } else {
#pragma unroll
          for (int sl = 0; sl < SL; ++sl) {
            const int k = kq[sl];
            if (it == 0) {
              if (act[sl]) {
                if (codeC[c + 1] >= 0) {
                  strip::ld4<Q>(rC + ro0 + k, cu[sl]);
                } else {  // the current row is the south boundary row
                  double ur[4];
                  strip::ld4<Q>(rN + ro0 + k, ur);
                  strip::bstate(P, codeC[c + 1], 2, k, ur, cu[sl]);
                }
              } else {
#pragma unroll
                for (int a = 0; a < 4; ++a) cu[sl][a] = a == 0 ? 1.0 : (a == 3 ? 2.5 : 0.0);
              }
              RusNode<4> n0;
              n0.init(cu[sl], gam);
              cir[sl] = n0.irho;
              cp[sl] = n0.p;
              cc_[sl] = n0.c;
            }
            if (act[sl] && codeN[c + 1] < 0)
              strip::bstate(P, codeN[c + 1], 3, k, cu[sl], un[sl]);
            else
              strip::ld4<Q>(rN + ro0 + k, un[sl]);
          }
        }
#pragma unroll
        for (int sl = 0; sl < SL; ++sl) {
          RusNode<4> ncur, nnx;
          ncur.irho = cir[sl];
          ncur.p = cp[sl];
          ncur.c = cc_[sl];
          nnx.init(un[sl], gam);
          double fc[4], fn[4], sc, sn, gN[4];
          ncur.flux(cu[sl], 1, fc, sc);
          nnx.flux(un[sl], 1, fn, sn);
          strip::face(fc, sc, cu[sl], fn, sn, un[sl], gN);
          if (own_row) {
            double fx[4], sx, ue[4], fe[4], gE[4], gW[4];
            ncur.flux(cu[sl], 0, fx, sx);
            // east face from column c+1's (u, F_x, s_x) by shuffle; the strip's edge faces come from
            // the halo warps (shared memory)
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              ue[a] = __shfl_down_sync(0xffffffffu, cu[sl][a], 4);
              fe[a] = __shfl_down_sync(0xffffffffu, fx[a], 4);
            }
            const double se = __shfl_down_sync(0xffffffffu, sx, 4);
            strip::face(fx, sx, cu[sl], fe, se, ue, gE);
            if (c == tw - 1) {
#pragma unroll
              for (int a = 0; a < 4; ++a) gE[a] = hxr[(4 + a) * Q + kq[sl]];
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) gW[a] = __shfl_up_sync(0xffffffffu, gE[a], 4);
            if (c == 0) {
#pragma unroll
              for (int a = 0; a < 4; ++a) gW[a] = hxr[a * Q + kq[sl]];
            }
            if (act[sl]) {
              if constexpr (SC) {
                const int64_t cell = (int64_t)(ya - 1 + it) * bx + x0 + c;
                double* o = A.uhat_new + cell * 4 * Q + kq[sl];
                double v[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                  double r = 0.0;
                  r += (gE[a] - gW[a]) * cfx;
                  r += (gN[a] - gS[sl][a]) * cfy;
                  v[a] = cu[sl][a] - dt * r;
                  o[a * Q] = v[a];
                }
                atomicAdd(dmean + (it & 1) * TX + c, P.T.omega[kq[sl]] * (v[0] - cu[sl][0]));
                my_rate = fmax(my_rate, node_rate<0, 4>(v, P.mesh, cell, gam));
              } else {
                double* o = rb + bo + kq[sl];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                  double r = 0.0;
                  r += (gE[a] - gW[a]) * cfx;
                  r += (gN[a] - gS[sl][a]) * cfy;
                  o[a * KP] = cform ? cu[sl][a] - dt * r : r;
                }
              }
            }
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            gS[sl][a] = gN[a];
            cu[sl][a] = un[sl][a];
          }
          cir[sl] = nnx.irho;
          cp[sl] = nnx.p;
          cc_[sl] = nnx.c;
        }
      } else if (it + 2 < LR) {
        // x fluxes at the strip's west and east faces of the next row (an owned row)
        double* hxn = HX + ((it + 1) & 1) * HXS;
        for (int h = tid - HT0; h < 2 * Q; h += NTH) {
          const int side = h >= Q, k = h - side * Q;
          const int hcol = side ? tw + 1 : 0, icol = side ? tw : 1;  // halo / inner column
          double ui[4], uh[4];
          strip::ld4<Q>(rN + icol * QMP + k, ui);
          if (codeN[hcol] >= 0)
            strip::ld4<Q>(rN + hcol * QMP + k, uh);
          else
            strip::bstate(P, codeN[hcol], side, k, ui, uh);
          RusNode<4> ni, nh;
          ni.init(ui, gam);
          nh.init(uh, gam);
          double fi[4], fh[4], si, sh, gf[4];
          ni.flux(ui, 0, fi, si);
          nh.flux(uh, 0, fh, sh);
          if (side)
            strip::face(fi, si, ui, fh, sh, uh, gf);
          else
            strip::face(fh, sh, uh, fi, si, ui, gf);
#pragma unroll
          for (int a = 0; a < 4; ++a) hxn[(side * 4 + a) * Q + k] = gf[a];
        }
      }
      STRIP_STAMP(1)
      if constexpr (SC) {
        if (warp == NW - 1 && it >= 2) sc_residual(it - 1);
      } else {
        if (warp >= NW - NPW && it >= 2) project(it - 1);
      }
      STRIP_STAMP(2)
    }
#ifdef IPM_STRIP_PROF
    if (blockIdx.x == 0 && first_seg && lane == 0)
      for (int r = 0; r < 4; ++r)
        printf("PROF warp %d row %d work %lld proj %lld\n", warp, r, st[r * 4 + 1] - st[r * 4], st[r * 4 + 2] - st[r * 4 + 1]);
    first_seg = false;
#endif
    __syncthreads();
    if constexpr (SC) {
      if (warp == NW - 1) sc_residual(LR - 2);
    } else {
      if (warp >= NW - NPW) project(LR - 2);
    }
    rows_done += LR;
    __syncthreads();
  }
  my_res = warp_sum(my_res);
  if (lane == 0 && my_res != 0.0) atomicAdd(&P.sc->residual, my_res);
  if constexpr (SC) {
    my_rate = warp_max(my_rate);
    if (lane == 0 && my_rate > 0.0)
      atomicMax(&P.sc->sc_rate_next, (unsigned long long)__double_as_longlong(my_rate));
  }
}

#endif
