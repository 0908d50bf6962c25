// Strip-marching kinetic-flux kernel for row-major cartesian blocks (Euler 2D, Rusanov; m = 4).
// Included by ipm_kernels.cu after RusNode / FluxParams.
//
// What it computes is k_flux_cart's a11 + projection (PAPER.md:130 difference form per direction,
// PAPER.md:182-185 update forms), with every node's Rusanov ingredients formed ONCE and every face
// flux formed once per node (y faces) or twice (x faces, by both cells) instead of five ingredient
// evaluations and four faces per node:
//   * a CTA owns a strip of TX cell columns and walks its rows y = ya..yb-1 (a contiguous share of
//     all strip rows, so every CTA gets the same number of rows);
//   * the node states of the TX cells of a row plus the two x-halo cells are copied into a 3-row
//     shared-memory ring with cp.async two rows ahead (every cell's Q x m block is contiguous);
//   * thread items (column j, node k), two per thread, fixed for the whole walk: the item carries the
//     ingredients (1/rho, p, c) of its current row and the y-face flux g_{y-1/2} from the previous
//     row, forms the next row's ingredients and g_{y+1/2}, publishes (F_x, s_x) of its current node
//     for the x neighbours, and then r = (g_E - g_W)/dx + (g_N - g_S)/dy;
//   * the projection Phi^T(omega o r) of the row's TX cells is a set of DMMAs with A = r^T (rows =
//     (cell, state), K = nodes; written conflict-free by the items) and B = the WPhiF fragments.
// Boundary states (ghost / slip wall / outflow copy) follow k_flux_cart exactly; x-halo boundary
// states are materialised in the ring's halo column by the halo threads.

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

// K stride of the r^T rows: >= KS*4 and = 4 mod 8 doubles so that the 8 rows x 4 k of an A fragment
// fall into distinct banks
__host__ __device__ constexpr int kp(int KS) { return (KS * 4) % 8 == 4 ? KS * 4 : KS * 4 + 4; }

constexpr int UNUSED = -2147483647 - 1;

template <int TX, int QC>
struct Layout {
  static constexpr int NC = TX + 2;  // ring columns: west halo, TX owned, east halo
  static constexpr int CT = TX / 2;  // DMMA row tiles of r^T (8 rows = 2 cells x 4 states)
  static constexpr int QM = QC * 4, KS = (QC + 3) / 4, KP = kp(KS), RB = CT * 8 * KP;
  int MT, NM, RS;
  size_t a, ring, row, xs, rb, idx, bar, total;  // offsets in doubles
  // per ring row besides the node states: uhat_old of the TX cells [TX][NM]
  __host__ __device__ Layout(int MT_, int NM_) : MT(MT_), NM(NM_), RS(TX * NM_) {
    a = 0;
    ring = a + (size_t)MT * KS * 32;
    row = ring + (size_t)4 * NC * QM;
    xs = row + (size_t)5 * RS;
    rb = xs + (((size_t)NC * 5 * QC + 1) & ~(size_t)1);
    idx = rb + (size_t)RB;
    bar = idx + (8 * NC + 1) / 2;
    total = bar + 4;
  }
};

// Rusanov flux g(uL, uR) = (F(uL) + F(uR))/2 - max(sL, sR) (uR - uL)/2 (k_flux_cart's formula)
__device__ __forceinline__ void face(const double* fl, double sl, const double* ul, const double* fr, double sr,
                                     const double* ur, double* g) {
  const double amax = fmax(sl, sr);
#pragma unroll
  for (int a = 0; a < 4; ++a) g[a] = 0.5 * (fl[a] + fr[a]) - 0.5 * amax * (ur[a] - ul[a]);
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
__device__ int g_strip_prof_done = 0;
#define STRIP_STAMP(n) \
  if (prof && lane == 0 && it >= 20 && it < 24) st[(it - 20) * 4 + (n)] = clock64();
#else
#define STRIP_STAMP(n)
#endif

template <int TX, int NT, int MINB, int QC>
__global__ void __launch_bounds__(NT, MINB) k_flux_strip(FluxParams P) {
  using L = strip::Layout<TX, QC>;
  constexpr int NC = L::NC, CT = L::CT, QM = L::QM, KS = L::KS, KP = L::KP, RB = L::RB;
  constexpr int Q = QC, OT = TX * QC / 2;  // owned-item threads (2 items each); [OT, OT+Q): x-halo items
  constexpr int NW = NT / 32, PW0 = (OT + 31) / 32;  // warps [PW0, NW) hold no owned items
#ifndef IPM_STRIP_NPW
#define IPM_STRIP_NPW 4
#endif
  constexpr int NPW = IPM_STRIP_NPW;  // projection warps: the last NPW, one per SM sub-partition (DMMA pipe)
  static_assert(OT + QC <= NT && PW0 - 1 <= NW - NPW && CT % NPW == 0, "strip kernel: not enough threads");
  extern __shared__ __align__(16) double sm[];
  const int N = P.T.N, MT = P.T.MT, nmax = N * 4;
  const L lay(MT, nmax);
  const int RS = lay.RS;
  double* sA = sm + lay.a;
  double* ring = sm + lay.ring;  // [4 rows][NC][4][Q] (node states are stored [cell][state][node])
  double* rowd = sm + lay.row;   // [5 rows][TX][nmax] uhat_old
  double* XS = sm + lay.xs;      // [NC][5][Q]: F_x, s_x of the current row
  double* rbT = sm + lay.rb;     // [CT][8][KP]: r^T of the current row
  int* sidx = reinterpret_cast<int*>(sm + lay.idx);  // [8 rows][NC] cell codes
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + lay.bar);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int b = 0; b < 4; ++b) strip::mbar_init(mbar + b, 1);
    strip::fence_mbar_init();
  }
  unsigned rows_done = 0;  // ring rows issued by this CTA before the current segment (mbarrier phases)
  for (int x = tid; x < MT * KS * 32; x += NT) sA[x] = P.T.WPhiF[x];
  for (int x = tid; x < RB; x += NT) rbT[x] = 0.0;  // K padding (k >= Q) stays 0
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

  // fixed per-thread item offsets (ring row, XS, r^T)
  int jj[2], ro[2], xo[2], bo[2];
#pragma unroll
  for (int sl = 0; sl < 2; ++sl) {
    const int i = tid + sl * OT, j = i / Q, k = i - j * Q;
    jj[sl] = tid < OT ? j : TX;
    ro[sl] = (j + 1) * QM + k;
    xo[sl] = (j + 1) * 5 * Q + k;
    bo[sl] = (j >> 1) * 8 * KP + (j & 1) * 4 * KP + k;
  }
  const int hk = tid - OT;  // halo node
#ifdef IPM_STRIP_PROF
  long long st[16];
  const bool prof = blockIdx.x == 0 && g_strip_prof_done == 0;
  bool first_seg = true;
#endif

  for (int64_t g = R * blockIdx.x / gridDim.x; g < g1;) {
    const int s = (int)(g / by);
    const int ya = (int)(g - (int64_t)s * by);
    const int64_t ybl = ya + (g1 - g);
    const int yb = ybl < by ? (int)ybl : by;
    g += yb - ya;
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
    // one thread: TMA bulk copies of ring row it (node states of its cells, uhat_old of owned rows)
    auto issue_row = [&](int it) {
      const int* code = sidx + (it & 7) * NC;
      double* dst = ring + (it & 3) * NC * QM;
      unsigned long long* bar = mbar + ((rows_done + it) & 3);
      const int yr = ya - 1 + it;
      const bool owned = yr >= ya && yr < yb;
      unsigned bytes = owned ? (unsigned)(tw * nmax * 8) : 0u;
      for (int col = 0; col < NC; ++col)
        if (code[col] >= 0) bytes += QM * 8;
      strip::fence_proxy_async();  // generic writes into the ring (boundary states) before the async ones
      strip::mbar_expect_tx(bar, bytes);
      for (int col = 0; col < NC; ++col)
        if (code[col] >= 0) strip::bulk_g2s(dst + col * QM, A.uq + (int64_t)code[col] * QM, QM * 8, bar);
      if (owned)
        strip::bulk_g2s(rowd + (it % 5) * RS, A.uhat_old + ((int64_t)yr * bx + x0) * nmax, (unsigned)(tw * nmax * 8),
                        bar);
    };
    auto wait_row = [&](int it) {
      const unsigned gi = rows_done + it;
      strip::mbar_wait(mbar + (gi & 3), (gi >> 2) & 1);
    };
    // projection C^T = r^T (omega Phi^T) on DMMA (two accumulator chains) and the update of ring row
    // itp's cells (projection warps)
    // projection warps: the last NPW warps; for MT == 2 each holds CT/NPW column tiles x both row tiles
    // of C^T in registers, so every A fragment (r^T) and B fragment (omega Phi) is loaded once per k step
    auto project = [&](int itp) {
      const int y = ya - 1 + itp;
      const double* rd = rowd + (itp % 5) * RS;
      const int rr = lane >> 2, q = lane & 3, pw = warp - (NW - NPW);
      auto epilogue = [&](int mt, int ct, double c0, double c1) {
        const int cl = ct * 2 + (rr >> 2), av = rr & 3;
        if (cl >= tw) return;
        const int64_t cell = (int64_t)y * bx + x0 + cl;
        const int Nnew = (P.ad.n_levels > 0 && A.level_new) ? P.ad.Nl[A.level_new[cell]] : N;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 8 * mt + 2 * q + e;
          if (i >= N) continue;
          const int64_t idx = cell * nmax + i * 4 + av;
          const double old = rd[cl * nmax + i * 4 + av];
          const double cv = e == 0 ? c0 : c1;
          double out = 0.0;
          if (i < Nnew) out = cform ? cv : old - dt * cv;
          A.uhat_new[idx] = out;
          if (i == 0 && av == 0) my_res += P.mesh.area[cell] * fabs(out - old);
          if (A.lam && i >= Nnew) A.lam[idx] = 0.0;
        }
      };
      if (MT == 2) {
        constexpr int NCT = CT / NPW;
        double acc[2][NCT][2];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int c = 0; c < NCT; ++c) acc[m][c][0] = acc[m][c][1] = 0.0;
        const double* a = rbT + rr * KP + q;
        const double* b = sA + lane;
#pragma unroll 3
        for (int ks = 0; ks < KS; ++ks) {
          double bf[2], af[NCT];
#pragma unroll
          for (int m = 0; m < 2; ++m) bf[m] = b[(m * KS + ks) * 32];
#pragma unroll
          for (int c = 0; c < NCT; ++c) af[c] = a[(pw + c * NPW) * 8 * KP + ks * 4];
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int c = 0; c < NCT; ++c)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                           : "+d"(acc[m][c][0]), "+d"(acc[m][c][1])
                           : "d"(af[c]), "d"(bf[m]));
        }
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int c = 0; c < NCT; ++c) epilogue(m, pw + c * NPW, acc[m][c][0], acc[m][c][1]);
      } else {
        for (int tile = pw; tile < MT * CT; tile += NPW) {
          const int mt = tile / CT, ct = tile - mt * CT;
          double c0 = 0.0, c1 = 0.0;
          const double* a = rbT + ct * 8 * KP + rr * KP + q;
          const double* b = sA + mt * KS * 32 + lane;
#pragma unroll 5
          for (int ks = 0; ks < KS; ++ks)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c0), "+d"(c1)
                         : "d"(a[ks * 4]), "d"(b[ks * 32]));
          epilogue(mt, ct, c0, c1);
        }
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

    // per-item carried state (two items per owned thread)
    double cir[2], cp[2], cc_[2], gS[2][4];
    const int hro = (tw + 1) * QM + hk, hxo = (tw + 1) * 5 * Q + hk;

    for (int it = 0; it + 1 < LR; ++it) {
      if (it == 0) wait_row(0);
      wait_row(it + 1);
      __syncthreads();  // rows <= it+1 in the ring; F2 of row it-1 done (r^T, XS free)
      STRIP_STAMP(0)
      if (tid == NT - 1 && it + 3 < LR) issue_row(it + 3);
      if (tid < NC && it + 4 < LR) {
        sidx[((it + 4) & 7) * NC + tid] = pend;
        if (it + 5 < LR) pend = row_code(it + 5, tid);
      }
      const int* codeC = sidx + (it & 7) * NC;
      const int* codeN = sidx + ((it + 1) & 7) * NC;
      double* rC = ring + (it & 3) * NC * QM;
      const double* rN = ring + ((it + 1) & 3) * NC * QM;
      const bool own_row = it > 0;
      const bool general = it == 0 || it + 2 == LR;  // rows that may hold boundary states

      // ---- phase 1: next-row ingredients, y face, x ingredients | x halo | projection of row it-1 ----
      double nir[2], np[2], nc[2], gN[2][4];
      if (tid < OT) {
        if (!general) {
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            double cu[4], un[4];
            strip::ld4<Q>(rC + ro[sl], cu);
            strip::ld4<Q>(rN + ro[sl], un);
            RusNode<4> ncur, nnx;
            ncur.irho = cir[sl];
            ncur.p = cp[sl];
            ncur.c = cc_[sl];
            nnx.init(un, gam);
            nir[sl] = nnx.irho;
            np[sl] = nnx.p;
            nc[sl] = nnx.c;
            double fc[4], fn[4], sc, sn, fx[4], sx;
            ncur.flux(cu, 1, fc, sc);
            nnx.flux(un, 1, fn, sn);
            strip::face(fc, sc, cu, fn, sn, un, gN[sl]);
            ncur.flux(cu, 0, fx, sx);
            if (jj[sl] < tw) {
              double* xs = XS + xo[sl];
#pragma unroll
              for (int a = 0; a < 4; ++a) xs[a * Q] = fx[a];
              xs[4 * Q] = sx;
            }
          }
        } else {
#pragma unroll
          for (int sl = 0; sl < 2; ++sl) {
            if (jj[sl] >= tw) continue;
            const int col = jj[sl] + 1, k = ro[sl] - col * QM;
            double cu[4], un[4];
            if (codeC[col] >= 0) {
              strip::ld4<Q>(rC + ro[sl], cu);
            } else {  // current row is the south boundary row
              double ur[4];
              strip::ld4<Q>(rN + ro[sl], ur);
              strip::bstate(P, codeC[col], 2, k, ur, cu);
            }
            if (!own_row) {
              RusNode<4> n0;
              n0.init(cu, gam);
              cir[sl] = n0.irho;
              cp[sl] = n0.p;
              cc_[sl] = n0.c;
            }
            if (codeN[col] >= 0)
              strip::ld4<Q>(rN + ro[sl], un);
            else
              strip::bstate(P, codeN[col], 3, k, cu, un);
            RusNode<4> ncur, nnx;
            ncur.irho = cir[sl];
            ncur.p = cp[sl];
            ncur.c = cc_[sl];
            nnx.init(un, gam);
            nir[sl] = nnx.irho;
            np[sl] = nnx.p;
            nc[sl] = nnx.c;
            double fc[4], fn[4], sc, sn;
            ncur.flux(cu, 1, fc, sc);
            nnx.flux(un, 1, fn, sn);
            strip::face(fc, sc, cu, fn, sn, un, gN[sl]);
            if (own_row) {
              double fx[4], sx;
              ncur.flux(cu, 0, fx, sx);
              double* xs = XS + xo[sl];
#pragma unroll
              for (int a = 0; a < 4; ++a) xs[a * Q] = fx[a];
              xs[4 * Q] = sx;
            }
          }
        }
      } else {
        if (tid < OT + Q && own_row) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const int col = side ? tw + 1 : 0;
            double* up = rC + (side ? hro : hk);
            double u[4];
            if (codeC[col] >= 0) {
              strip::ld4<Q>(up, u);
            } else {
              double ur[4];
              strip::ld4<Q>(up + (side ? -QM : QM), ur);
              strip::bstate(P, codeC[col], side, hk, ur, u);
#pragma unroll
              for (int a = 0; a < 4; ++a) up[a * Q] = u[a];
            }
            RusNode<4> h;
            h.init(u, gam);
            double fx[4], sx;
            h.flux(u, 0, fx, sx);
            double* xs = XS + (side ? hxo : hk);
#pragma unroll
            for (int a = 0; a < 4; ++a) xs[a * Q] = fx[a];
            xs[4 * Q] = sx;
          }
        }
      }
#ifndef IPM_STRIP_NOPROJ
      if (warp >= NW - NPW && it >= 2) project(it - 1);
#endif
      STRIP_STAMP(1)
      __syncthreads();
      STRIP_STAMP(2)

      // ---- phase 2: x faces, the residual r and r^T (owned items) ------------------------------------
      if (tid < OT) {
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
#ifdef IPM_STRIP_NOF2
          if (false) {
#else
          if (own_row) {
#endif
            const double* pc = rC + ro[sl];
            double cu[4], uw[4], ue[4], fw[4], fc[4], fe[4];
            strip::ld4<Q>(pc, cu);
            strip::ld4<Q>(pc - QM, uw);
            strip::ld4<Q>(pc + QM, ue);
            const double* xc = XS + xo[sl];
            const double* xw = xc - 5 * Q;
            const double* xe = xc + 5 * Q;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              fw[a] = xw[a * Q];
              fc[a] = xc[a * Q];
              fe[a] = xe[a * Q];
            }
            double gw[4], ge[4], r[4];
            strip::face(fw, xw[4 * Q], uw, fc, xc[4 * Q], cu, gw);
            strip::face(fc, xc[4 * Q], cu, fe, xe[4 * Q], ue, ge);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              r[a] = 0.0;
              r[a] += (ge[a] - gw[a]) * cfx;
              r[a] += (gN[sl][a] - gS[sl][a]) * cfy;
            }
            if (jj[sl] < tw) {
              double* o = rbT + bo[sl];
#pragma unroll
              for (int a = 0; a < 4; ++a) o[a * KP] = cform ? cu[a] - dt * r[a] : r[a];
            }
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) gS[sl][a] = gN[sl][a];
          cir[sl] = nir[sl];
          cp[sl] = np[sl];
          cc_[sl] = nc[sl];
        }
      }
      STRIP_STAMP(3)
    }
#ifdef IPM_STRIP_PROF
    if (prof && first_seg && lane == 0)
      for (int r = 0; r < 4; ++r)
        printf("PROF warp %d row %d t0 %lld p1 %lld syncA %lld p2 %lld\n", warp, r, 0LL, st[r * 4 + 1] - st[r * 4],
               st[r * 4 + 2] - st[r * 4], st[r * 4 + 3] - st[r * 4]);
    first_seg = false;
#endif
    __syncthreads();
    if (warp >= NW - NPW) project(LR - 2);
    rows_done += LR;
    __syncthreads();
  }
  my_res = warp_sum(my_res);
  if (lane == 0 && my_res != 0.0) atomicAdd(&P.sc->residual, my_res);
}

#endif
