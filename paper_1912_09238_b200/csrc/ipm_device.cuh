// ipm_device.cuh — device-side closures, fluxes and warp helpers of libipm (sm_100a, fp64).
//
// Closures u_s = (grad s)^{-1} and grad u_s:
//   QUADRATIC  s = |u|^2/2                  -> u_s = Lambda, grad u_s = I
//   BARRIER    u_s = u- + (u+ - u-) sigma(Lambda)                          (BASELINE cfg 1)
//   EULER      U = -rho S/(gamma-1): ln rho = v1 - |v_m|^2/(2 v_E) - (gamma + ln(-v_E))/(gamma-1),
//              p = rho/(-v_E), w = -v_m/v_E, grad u_s = A0 (symmetric)   (App. B, readings 9-11)
// Two-point fluxes g (reading 14).
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "ipm_internal.h"

namespace ipm {

constexpr unsigned FULL_MASK = 0xffffffffu;

enum { CL_QUADRATIC = 0, CL_BARRIER = 1, CL_EULER = 2 };
enum { FX_LF_GLOBAL = 0, FX_HLL = 1, FX_RUSANOV = 2 };
enum { MK_1D = 0, MK_CART = 1, MK_TRI = 2 };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// Fast reciprocal and square root for positive normal operands (densities, pressures, pivots of an SPD
// matrix): the hardware approximation refined by Newton steps to about one ulp, without the special-
// operand handling of the IEEE routines (which costs ~20-30 instructions per call in the flux kernels)
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double sqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  e = fma(-h * y, y, 0.5);
  y = fma(y, e, y);
  const double s = x * y;                 // sqrt(x) to ~1e-16
  return fma(0.5 * y, fma(-s, s, x), s);  // one correction: ~0.5 ulp
}

// packed symmetric index of (a, b), a <= b, row-major upper triangle of an m x m matrix
template <int MS>
__host__ __device__ constexpr int sym_idx(int a, int b) {
  return a * MS - a * (a - 1) / 2 + (b - a);
}

// ---------------------------------------------------------------------------------------------
// closures: eval() returns admissibility, fills u[MS], J[MS(MS+1)/2] (packed upper), s_*(Lambda)
// ---------------------------------------------------------------------------------------------
template <int CL, int MS>
struct Closure;

template <int MS>
struct Closure<CL_QUADRATIC, MS> {
  static constexpr int MM = MS * (MS + 1) / 2;
  __device__ static bool eval(const double* L, double* u, double* J, double& sstar, const ClParams&) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < MS; ++a) {
      u[a] = L[a];
      s += 0.5 * L[a] * L[a];
    }
#pragma unroll
    for (int a = 0; a < MS; ++a)
#pragma unroll
      for (int b = a; b < MS; ++b) J[sym_idx<MS>(a, b)] = (a == b) ? 1.0 : 0.0;
    sstar = s;
    return true;
  }
  __device__ static bool grad_s(const double* u, double* L, const ClParams&) {
#pragma unroll
    for (int a = 0; a < MS; ++a) L[a] = u[a];
    return true;
  }
};

template <>
struct Closure<CL_BARRIER, 1> {
  static constexpr int MM = 1;
  __device__ static bool eval(const double* L, double* u, double* J, double& sstar, const ClParams& c) {
    const double x = L[0], D = c.umax - c.umin;
    // numerically stable logistic
    double sg;
    if (x >= 0.0) {
      sg = 1.0 / (1.0 + exp(-x));
    } else {
      const double e = exp(x);
      sg = e / (1.0 + e);
    }
    u[0] = c.umin + D * sg;
    J[0] = D * sg * (1.0 - sg);
    sstar = c.umin * x + D * (fmax(x, 0.0) + log1p(exp(-fabs(x)))) - D * log(D);
    return isfinite(u[0]);
  }
  __device__ static bool grad_s(const double* u, double* L, const ClParams& c) {
    if (!(u[0] > c.umin && u[0] < c.umax)) return false;
    L[0] = log((u[0] - c.umin) / (c.umax - u[0]));
    return true;
  }
};

template <int MS>
struct Closure<CL_EULER, MS> {
  static_assert(MS == 3 || MS == 4, "Euler closure needs m = d + 2 with d in {1, 2}");
  static constexpr int D = MS - 2;
  static constexpr int MM = MS * (MS + 1) / 2;
  __device__ static bool eval(const double* v, double* u, double* J, double& sstar, const ClParams& c) {
    // branch-free (an early exit would leave u, J partly unwritten and force them to local memory);
    // vE >= 0 makes log(-vE) NaN and the state inadmissible
    const double g = c.gamma, vE = v[MS - 1];
    double vm2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) vm2 = fma(v[1 + k], v[1 + k], vm2);
    const double inv_vE = rcp_nr(vE);  // vE < 0 on the admissible set (checked below)
    const double igm1 = c.inv_gm1;
    const double lnrho = v[0] - 0.5 * vm2 * inv_vE - (g + log(-vE)) * igm1;
    const double rho = exp(lnrho);
    const double p = -rho * inv_vE;
    double w[D], w2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      w[k] = -v[1 + k] * inv_vE;
      w2 = fma(w[k], w[k], w2);
    }
    const double E = p * igm1 + 0.5 * rho * w2;
    u[0] = rho;
#pragma unroll
    for (int k = 0; k < D; ++k) u[1 + k] = rho * w[k];
    u[MS - 1] = E;
    sstar = rho;
    // A0 = du/dv: H = (E+p)/rho, c^2 = gamma p / rho
    const double irho = rcp_nr(rho);
    const double H = (E + p) * irho;
    J[sym_idx<MS>(0, 0)] = rho;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      J[sym_idx<MS>(0, 1 + k)] = u[1 + k];
#pragma unroll
      for (int l = k; l < D; ++l) J[sym_idx<MS>(1 + k, 1 + l)] = u[1 + k] * w[l] + (k == l ? p : 0.0);
      J[sym_idx<MS>(1 + k, MS - 1)] = u[1 + k] * H;
    }
    J[sym_idx<MS>(0, MS - 1)] = E;
    J[sym_idx<MS>(MS - 1, MS - 1)] = rho * H * H - g * p * p * irho * igm1;
    return vE < 0.0 && rho > 0.0 && isfinite(rho) && isfinite(E);
  }
  // v = ((gamma - S)/(gamma-1) - rho|w|^2/(2p), rho w/p, -rho/p), S = ln p - gamma ln rho
  __device__ static bool grad_s(const double* u, double* v, const ClParams& c) {
    const double g = c.gamma, rho = u[0];
    double m2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) m2 += u[1 + k] * u[1 + k];
    const double p = (g - 1.0) * (u[MS - 1] - 0.5 * m2 / rho);
    if (!(rho > 0.0) || !(p > 0.0)) return false;
    const double S = log(p) - g * log(rho);
    const double beta = rho / p;
    v[0] = (g - S) / (g - 1.0) - 0.5 * beta * m2 / (rho * rho);
#pragma unroll
    for (int k = 0; k < D; ++k) v[1 + k] = beta * u[1 + k] / rho;
    v[MS - 1] = -beta;
    return true;
  }
};

// ---------------------------------------------------------------------------------------------
// physics: flux along a unit normal, wave speeds
// ---------------------------------------------------------------------------------------------
template <int MS>
struct Euler {
  static constexpr int D = MS - 2;
  // F(u).n, normal velocity, sound speed
  __device__ static void flux_n(const double* u, const double* n, double gamma, double* f, double& vn, double& c) {
    const double irho = rcp_nr(u[0]);
    double m2 = 0.0, mn = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      m2 = fma(u[1 + k], u[1 + k], m2);
      mn = fma(u[1 + k], n[k], mn);
    }
    const double p = (gamma - 1.0) * (u[MS - 1] - 0.5 * m2 * irho);
    vn = mn * irho;
    c = sqrt_nr(gamma * p * irho);
    f[0] = mn;
#pragma unroll
    for (int k = 0; k < D; ++k) f[1 + k] = fma(u[1 + k], vn, p * n[k]);
    f[MS - 1] = (u[MS - 1] + p) * vn;
  }
  __device__ static double speed_norm(const double* u, double gamma) {
    const double rho = u[0], irho = 1.0 / rho;
    double m2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) m2 = fma(u[1 + k], u[1 + k], m2);
    const double p = (gamma - 1.0) * (u[MS - 1] - 0.5 * m2 * irho);
    return sqrt(m2) * irho + sqrt(gamma * p * irho);
  }
  // |v.e_dir| + c along a coordinate direction
  __device__ static double speed_dir(const double* u, int dir, double gamma) {
    const double rho = u[0], irho = 1.0 / rho;
    double m2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) m2 = fma(u[1 + k], u[1 + k], m2);
    const double p = (gamma - 1.0) * (u[MS - 1] - 0.5 * m2 * irho);
    return fabs(u[1 + dir] * irho) + sqrt(gamma * p * irho);
  }
};

template <int FX, int MS>
struct NumFlux;

// scalar Burgers, global Lax-Friedrichs with dx/(2dt)
template <>
struct NumFlux<FX_LF_GLOBAL, 1> {
  __device__ static void g(const double* ul, const double* ur, const double*, double, double dx_over_dt, double* out) {
    out[0] = 0.25 * (ul[0] * ul[0] + ur[0] * ur[0]) - 0.5 * dx_over_dt * (ur[0] - ul[0]);
  }
};

template <int MS>
struct NumFlux<FX_HLL, MS> {
  __device__ static void g(const double* ul, const double* ur, const double* n, double gamma, double, double* out) {
    double fl[MS], fr[MS], vl, vr, cl, cr;
    Euler<MS>::flux_n(ul, n, gamma, fl, vl, cl);
    Euler<MS>::flux_n(ur, n, gamma, fr, vr, cr);
    const double SL = fmin(vl - cl, vr - cr), SR = fmax(vl + cl, vr + cr);
    if (SL >= 0.0) {
#pragma unroll
      for (int a = 0; a < MS; ++a) out[a] = fl[a];
    } else if (SR <= 0.0) {
#pragma unroll
      for (int a = 0; a < MS; ++a) out[a] = fr[a];
    } else {
      const double inv = 1.0 / (SR - SL), sls = SL * SR;
#pragma unroll
      for (int a = 0; a < MS; ++a) out[a] = (SR * fl[a] - SL * fr[a] + sls * (ur[a] - ul[a])) * inv;
    }
  }
};

template <int MS>
struct NumFlux<FX_RUSANOV, MS> {
  __device__ static void g(const double* ul, const double* ur, const double* n, double gamma, double, double* out) {
    double fl[MS], fr[MS], vl, vr, cl, cr;
    Euler<MS>::flux_n(ul, n, gamma, fl, vl, cl);
    Euler<MS>::flux_n(ur, n, gamma, fr, vr, cr);
    const double a = fmax(fabs(vl) + cl, fabs(vr) + cr);
#pragma unroll
    for (int k = 0; k < MS; ++k) out[k] = 0.5 * (fl[k] + fr[k]) - 0.5 * a * (ur[k] - ul[k]);
  }
};

// Characteristic far-field ghost state (reading 37), 2D Euler: the
// outgoing Riemann invariant v_n + 2c/(g-1) from the interior node state ui, the incoming one
// v_n - 2c/(g-1) from the free-stream node state uf; entropy p/rho^g and tangential velocity from the
// upwind side; supersonic normal flow in the interior takes uf (inflow) or ui (outflow).  n: outward unit
// normal.  Full-precision sqrt / pow (no fast approximations: the host libm's results to ~1 ulp).
__device__ __forceinline__ void farfield_ghost(double g, const double* ui, const double* uf, const double* n,
                                               double* ug) {
  const double ri = ui[0], vxi = ui[1] / ri, vyi = ui[2] / ri;
  const double pi = (g - 1.0) * (ui[3] - 0.5 * ri * (vxi * vxi + vyi * vyi));
  const double rf = uf[0], vxf = uf[1] / rf, vyf = uf[2] / rf;
  const double pf = (g - 1.0) * (uf[3] - 0.5 * rf * (vxf * vxf + vyf * vyf));
  const double vni = vxi * n[0] + vyi * n[1], vnf = vxf * n[0] + vyf * n[1];
  const double ci = sqrt(g * pi / ri), cf = sqrt(g * pf / rf);
  if (vni <= -ci || vni >= ci) {
    const double* src = vni <= -ci ? uf : ui;
#pragma unroll
    for (int a = 0; a < 4; ++a) ug[a] = src[a];
    return;
  }
  const double igm = 1.0 / (g - 1.0);
  const double rp = vni + 2.0 * ci * igm, rm = vnf - 2.0 * cf * igm;
  const double vnb = 0.5 * (rp + rm), cb = 0.25 * (g - 1.0) * (rp - rm);
  const bool in = vnb < 0.0;
  const double ru = in ? rf : ri, vxu = in ? vxf : vxi, vyu = in ? vyf : vyi, pu = in ? pf : pi;
  const double ent = pu / pow(ru, g);
  const double vnu = vxu * n[0] + vyu * n[1];
  const double vx = (vxu - vnu * n[0]) + vnb * n[0], vy = (vyu - vnu * n[1]) + vnb * n[1];
  const double rho = pow(cb * cb / (g * ent), igm);
  const double p = rho * cb * cb / g;
  ug[0] = rho;
  ug[1] = rho * vx;
  ug[2] = rho * vy;
  ug[3] = p * igm + 0.5 * rho * (vx * vx + vy * vy);
}

}  // namespace ipm
