// omb_math.cuh -- FP64 point operations of the hydro step, shared by every
// kernel.  Each function restates one piece of the reference with the SAME
// association of every + - * / so that, compiled with -fmad=false (no
// contraction), results are bit-identical to the reference CPU path:
//
//   iface / mono / contact / fallback : _core.pyx:76-155 (reconstruct)
//   kt_state / kt_axis                : _core.pyx:180-220 (_kt_point)
//   quadrature combine                : _core.pyx:310-346
//   prim_cell                         : _kernels/reference.py:30-45
//   update_cell                       : hydro/step.py:243-288, eos.py:50-61, sources.py:8-35
//   speed_cell                        : hydro/step.py:81-92, eos.py:28-44
//
// Everything is OMB_HD so the same code also builds for the host (the CPU
// emulation harness in tests/ runs the fused kernel logic under g++).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define OMB_HD __host__ __device__ __forceinline__
#else
#define OMB_HD inline
#endif

#include "omb_pow.cuh"  // glibc's pow, bit for bit (tau: reference.py:39, eos.py:50-61)

namespace omb {

constexpr int NF = 6;
constexpr int NLINES = 13;

// geometry.py:24-41 -- line directions, packed 2 bits per line (component+1)
// so the lookups are branch-free shifts of a constant
constexpr unsigned LDX_BITS = 0x2A96A96u;  // lines 0..12: 1,0,0,1,1,1,1,0,0,1,1,1,1
constexpr unsigned LDY_BITS = 0x2A9499u;   // 0,1,0,1,-1,0,0,1,1,1,1,-1,-1
constexpr unsigned LDZ_BITS = 0x888965u;   // 0,0,1,0,0,1,-1,1,-1,1,-1,1,-1
OMB_HD int ldx(int l) { return (int)((LDX_BITS >> (2 * l)) & 3u) - 1; }
OMB_HD int ldy(int l) { return (int)((LDY_BITS >> (2 * l)) & 3u) - 1; }
OMB_HD int ldz(int l) { return (int)((LDZ_BITS >> (2 * l)) & 3u) - 1; }

// the rarely taken exact operations (named so the call sites read as the rare branches they are;
// as out-of-line calls they measured neutral, profiles/r02/ab16_noinline_rare.txt)
OMB_HD double rare_div(double a, double b) { return a / b; }
OMB_HD double rare_pow(double x, double y) { return pow_glibc(x, y); }

// IEEE a/b that never takes CUDA's division slow path for a zero numerator
// (CUDA routes 0/b through a called subroutine; zero momenta and zero
// deviations are everywhere in the Sedov ambient).  For a == 0 the quotient
// t = 2^-100/b is finite for every b != 0 (even subnormal) and a*t carries
// 0/b's sign (t underflowing to +-0 for huge b keeps it); b = 0, inf, NaN
// give 0*inf = NaN, +-0, NaN as IEEE does -- branch-free, bit-identical.
OMB_HD double div_nz(double a, double b) {
  bool z = (a == 0.0);
  double q = (z ? 0x1p-100 : a) / b;
  return z ? a * q : q;
}

// IEEE a/b from a precomputed y = RN(1/b) (Markstein): q0 = a*y, then two
// fma corrections q <- q + (a - b q) y.  q1 is within 1 ulp of a/b, so the
// second correction returns the correctly rounded quotient (Markstein's
// theorem, given y normal, a normal quotient and an exact residual a - b q,
// whose grid 2^(e_b + e_q - 104) must not fall below 2^-1074).  With the
// divisor in [2^-100, 2^100] (checked once per divisor, or guaranteed by the
// caller) those premises hold whenever |q1| is in (2^-860, 2^1000): then
// |a| > 2^-960.  A zero numerator returns a*y, the signed zero (y finite).
// Straight-line; anything else sets `rare` and the caller redoes the
// quotient with IEEE division (kt_axis does that once for all six fields).
// Checked bitwise against IEEE division on 2^30 random pairs covering every
// exponent (omb_selftest_div, tests/test_gpu_parity.py).
OMB_HD bool div_range_ok(double b) { return b > 0x1p-100 && b < 0x1p+100; }  // b > 0
OMB_HD double div_fast(double a, double b, double y, unsigned& rare) {
  double q0 = a * y;
  double q1 = fma(fma(-b, q0, a), y, q0);
  double q2 = fma(fma(-b, q1, a), y, q1);
  bool zero = (a == 0.0);
  double m = fabs(q1);
  rare |= (unsigned)!(zero || (m > 0x1p-860 && m < 0x1p+1000));
  return zero ? q0 : q2;
}
// single quotient by a divisor in [2^-100, 2^100] (caller's guarantee: the
// EOS's gamma-1 -- checked on the host -- and the Simpson weight 36), with
// its own rarely taken IEEE fallback
// A zero numerator returns q0 = a*y (the signed zero) before the range test:
// zero Simpson deviations are everywhere in the Sedov ambient, and the IEEE
// division of the rare branch must not be reached (or speculated) for them --
// CUDA routes 0/b through its out-of-line division subroutine (ncu: 1.4 M
// warp-level calls per c2 launch, 5 % of k_stage's instructions, before this).
OMB_HD double div_by(double a, double b, double y) {
  double q0 = a * y;
  if (a == 0.0) return q0;
  double q1 = fma(fma(-b, q0, a), y, q0);
  double q2 = fma(fma(-b, q1, a), y, q1);
  double m = fabs(q1);
  if (!(m > 0x1p-860 && m < 0x1p+1000)) {
    double aa = a;
#ifdef __CUDA_ARCH__
    asm volatile("" : "+d"(aa));  // keep the IEEE division inside this rare branch
#endif
    q2 = rare_div(aa, b);
  }
  return q2;
}

// NaN-faithful helpers: C fmin/fmax semantics (IEEE minNum/maxNum), as libm.
OMB_HD double dmin(double a, double b) { return fmin(a, b); }
OMB_HD double dmax(double a, double b) { return fmax(a, b); }

// ---------------------------------------------------------------------------
// PPM reconstruction pieces (_core.pyx:76-106)
// ---------------------------------------------------------------------------

// interface value between cells a (=c) and ap1 (=c+d), stencil c-d .. c+2d
// The clamp bounds use glibc's fmin/fmax tie rule ((x<y)?x:y, (x>y)?x:y) as
// plain selects: NaN handling cannot matter here because any NaN among the
// four inputs already makes v7 NaN, which no comparison changes.
OMB_HD double iface(double am1, double a, double ap1, double ap2) {
  double v7 = (7.0 / 12.0) * (a + ap1) - (1.0 / 12.0) * (am1 + ap2);
  double mn = a < ap1 ? a : ap1, mx = a > ap1 ? a : ap1;
  if (v7 < mn) v7 = mn;
  if (v7 > mx) v7 = mx;
  return v7;
}

// Colella-Woodward monotonisation of (lv, hv) around the cell value a.
// `diff*diff/6.0` only feeds two comparisons, so it is evaluated as a
// multiply by RN(1/6) and the exact IEEE division is taken only when the
// comparison margin is within a guard band of 8 ulp -- the branch outcomes
// (hence the outputs) are identical to the reference's.
OMB_HD void mono(double a, double& lv, double& hv) {
  if ((hv - a) * (a - lv) <= 0.0) {
    lv = a;
    hv = a;
    return;
  }
  double diff = hv - lv;
  double mid = a - 0.5 * (lv + hv);
  double dm = diff * mid;
  double d2 = diff * diff;
  double q = d2 * (1.0 / 6.0);
  double band = 0x1p-49 * fabs(q) + 0x1p-1000;
  if (!(fabs(dm - q) > band) || !(fabs(dm + q) > band)) {
    double dd = d2;
#ifdef __CUDA_ARCH__
    // keep the exact division inside this rare branch: without the opaque
    // copy the compiler speculates the IEEE division for every field
    asm volatile("" : "+d"(dd));
#endif
    q = rare_div(dd, 6.0);
  }
  double nlv = lv, nhv = hv;
  if (dm > q) nlv = 3.0 * a - 2.0 * hv;
  if (-q > dm) nhv = 3.0 * a - 2.0 * nlv;
  lv = nlv;
  hv = nhv;
}

// _core.pyx:159-173
OMB_HD double mc_slope(double am1, double a, double ap1) {
  double dc = 0.5 * (ap1 - am1);
  double dl = 2.0 * (a - am1);
  double dr = 2.0 * (ap1 - a);
  if (dl * dr <= 0.0) return 0.0;
  double mag = dmin(fabs(dc), dmin(fabs(dl), fabs(dr)));
  return dc < 0.0 ? -mag : mag;
}

// _core.pyx:107-142 for one cell of one line; r[k] = rho at c+(k-2)d,
// pm1/pp1 = pressure at c-d / c+d.  Modifies lo/hi of rho in place.
OMB_HD void contact_steepen(const double r[5], double pm1, double pp1, double gamma, double& lo, double& hi) {
  double am1 = r[1], ap1 = r[3];
  double dr = ap1 - am1;
  if (fabs(dr) <= 1e-300) return;
  double d2m = r[2] - 2.0 * am1 + r[0];
  double d2p = r[4] - 2.0 * ap1 + r[2];
  if (d2m * d2p >= 0.0) return;
  if (fabs(dr) - 0.01 * dmin(fabs(ap1), fabs(am1)) <= 0.0) return;
  double pmin = dmin(pp1, pm1);
  double rmin = dmin(fabs(ap1), fabs(am1));
  if (fabs(pp1 - pm1) / pmin >= 0.1 * gamma * fabs(dr) / rmin) return;
  double eta_t = (d2m - d2p) / (6.0 * dr);
  double eta = 20.0 * (eta_t - 0.05);
  if (eta <= 0.0) return;
  if (eta > 1.0) eta = 1.0;
  double sm = mc_slope(r[0], r[1], r[2]);
  double sp = mc_slope(r[2], r[3], r[4]);
  lo = lo * (1.0 - eta) + (am1 + 0.5 * sm) * eta;
  hi = hi * (1.0 - eta) + (ap1 - 0.5 * sp) * eta;
}

// ---------------------------------------------------------------------------
// Central-upwind flux (_core.pyx:180-220), split into the per-state part
// (shared by every axis an interface serves) and the per-axis part.
// ---------------------------------------------------------------------------
struct KtState {
  double r, v[3], p, u[NF];  // primitive rho, v, p; conserved u
  double c;                  // sqrt(gamma p / rho)
};

OMB_HD void kt_state(const double* w, double gamma, double gm1, double inv_gm1, KtState& s) {
  s.r = w[0];
  s.v[0] = w[1];
  s.v[1] = w[2];
  s.v[2] = w[3];
  s.p = w[4];
  s.c = sqrt(div_nz(gamma * s.p, s.r));
  double kin = 0.5 * s.r * (s.v[0] * s.v[0] + s.v[1] * s.v[1] + s.v[2] * s.v[2]);
  s.u[0] = s.r;
  s.u[1] = s.r * s.v[0];
  s.u[2] = s.r * s.v[1];
  s.u[3] = s.r * s.v[2];
  s.u[4] = div_by(s.p, gm1, inv_gm1) + kin;
  s.u[5] = w[5];
}

// Flux through an `axis` face across the interface P -> Q (P = cell the
// `hi` state belongs to, Q = P + line direction, whose `lo` state is used).
// When the line runs against the face normal (`flip`) the reference swaps
// the roles: left = Q, right = P (_core.pyx:299-306).  The swap is folded
// into scalar coefficients instead of selecting whole states:
//   ap*fl - am*fr + (ap*am)*(ur-ul)
//     = cP*fP + cQ*fQ + s*(uQ-uP),  (cP,cQ,s) = (ap,-am,ap*am) or (-am,ap,-(ap*am))
// which is bit-identical (IEEE + commutes, x-y = x+(-y), products negate
// exactly).  Returns the signal speed max(a+, -a-).
// physical flux of field v through an `axis` face for state S (normal velocity vn)
OMB_HD double kt_phys(const KtState& S, double vn, int axis, int v) {
  double f = S.u[v] * vn;
  if (v == 1 || v == 2 || v == 3) f = (v == 1 + axis) ? f + S.p : f;  // normal momentum picks up p
  if (v == 4) f = f + S.p * vn;
  return f;
}
// Results go to out[v * stride] as they are computed (no array kept live);
// the six quotients run straight-line (independent chains) with one
// rare-case test for all of them (div_fast), whose redo recomputes.
OMB_HD double kt_axis(const KtState& P, const KtState& Q, int axis, bool flip, double* out, int stride = 1) {
  double vnP = axis == 0 ? P.v[0] : (axis == 1 ? P.v[1] : P.v[2]);
  double vnQ = axis == 0 ? Q.v[0] : (axis == 1 ? Q.v[1] : Q.v[2]);
  double eP = vnP + P.c, eQ = vnQ + Q.c;
  double mP = vnP - P.c, mQ = vnQ - Q.c;
  double ap = dmax(0.0, flip ? dmax(eQ, eP) : dmax(eP, eQ));
  double am = dmin(0.0, flip ? dmin(mQ, mP) : dmin(mP, mQ));
  double denom = ap - am;
  double apam = ap * am;
  double rden = 1.0 / denom;  // one IEEE reciprocal for the six quotients
  double cP = flip ? -am : ap;
  double cQ = flip ? ap : -am;
  double sg = flip ? -apam : apam;
  bool ok = denom > 0.0;
  unsigned rare = !div_range_ok(denom);
#pragma unroll
  for (int v = 0; v < NF; v++) {
    double fP = kt_phys(P, vnP, axis, v), fQ = kt_phys(Q, vnQ, axis, v);
    double num = (cP * fP + cQ * fQ) + sg * (Q.u[v] - P.u[v]);
    double q = div_fast(num, denom, rden, rare);
    out[v * stride] = ok ? q : (flip ? fQ : fP);
  }
  if (ok && rare) {
#pragma unroll
    for (int v = 0; v < NF; v++) {
      double fP = kt_phys(P, vnP, axis, v), fQ = kt_phys(Q, vnQ, axis, v);
      out[v * stride] = ((cP * fP + cQ * fQ) + sg * (Q.u[v] - P.u[v])) / denom;
    }
  }
  return dmax(ap, -am);
}

// Simpson face value in the reference's deviation form (_core.pyx:322-346):
// F = C + (4 edev + vdev)/36 with edev = (e0+e1)+(e2+e3), e_i = 0.5 acc_i - C
OMB_HD double pdev_edge(double acc, double c) { return 0.5 * acc - c; }
OMB_HD double pdev_vert(double acc, double c) { return 0.25 * acc - c; }
OMB_HD double face_final(double c, double edev, double vdev) { return c + div_by(4.0 * edev + vdev, 36.0, 1.0 / 36.0); }
// point accumulators exactly as the Cython loop builds them
OMB_HD double edge_acc(double f0, double f1) { return (0.0 + f0) + f1; }
OMB_HD double vert_acc(double f0, double f1, double f2, double f3) { return (0.0 + (f0 + f1)) + (f2 + f3); }

// ---------------------------------------------------------------------------
// primitives (reference.py:30-45); pow only on the tau branch
// ---------------------------------------------------------------------------
OMB_HD void prim_cell(const double* u, double gamma, double gm1, double eta, double* w) {
  double rho = u[0];
  double inv = 1.0 / rho;
  double vx = u[1] * inv, vy = u[2] * inv, vz = u[3] * inv;
  double kin = 0.5 * ((u[1] * vx + u[2] * vy) + u[3] * vz);
  double e1 = u[4] - kin;
  double eint = (e1 >= eta * u[4]) ? e1 : rare_pow(u[5], gamma);
  w[0] = rho;
  w[1] = vx;
  w[2] = vy;
  w[3] = vz;
  w[4] = gm1 * eint;
  w[5] = u[5];
}

// passive-scalar pass (omb_scalar_input built u = (rho, sx, sy, sz, p, X)): the
// velocities exactly as prim_cell forms them, the pressure and the scalar as given
OMB_HD void prim_cell_scalar(const double* u, double* w) {
  double inv = 1.0 / u[0];
  w[0] = u[0];
  w[1] = u[1] * inv;
  w[2] = u[2] * inv;
  w[3] = u[3] * inv;
  w[4] = u[4];
  w[5] = u[5];
}

// ---------------------------------------------------------------------------
// CFL wave speed of one cell (step.py:86-88 via eos.py:28-44); NaN-propagating
// ---------------------------------------------------------------------------
OMB_HD double nanmax(double a, double b) {
  if (a != a || b != b) return a + b;  // NaN
  return a > b ? a : b;
}
OMB_HD double speed_cell(const double* u, double gamma, double gm1, double eta) {
  double rho = u[0];
  double vm = nanmax(nanmax(div_nz(fabs(u[1]), rho), div_nz(fabs(u[2]), rho)), div_nz(fabs(u[3]), rho));
  double kin = div_nz(0.5 * ((u[1] * u[1] + u[2] * u[2]) + u[3] * u[3]), rho);
  double e1 = u[4] - kin;
  double eint = (e1 >= eta * u[4]) ? e1 : pow_glibc(u[5], gamma);
  double p = gm1 * eint;
  return vm + sqrt(gamma * p / rho);
}

// ---------------------------------------------------------------------------
// conservative update of one cell (step.py:249-265 + eos.py:50-61 +
// step.py:269-288).  rhs already holds ((0 - dFx/dx) - dFy/dx) - dFz/dx.
// ---------------------------------------------------------------------------
struct UpdateParams {
  double dt, a, b;
  double gamma, eta, inv_gamma;
  double omega;
  double floor_rho, floor_tau, floor_vmax;
  int has_src, has_grav;
};

// first part: sources and the RK combination -> nw
OMB_HD void update_cell_rk(const UpdateParams& P, const double* u, const double* u0, double* r, double x, double y,
                           const double* g /* gx gy gz dphi_dt or null */, double* nw) {
  if (P.has_src) {
    if (P.omega != 0.0) {
      double w2 = P.omega * P.omega;
      double ds1 = 2.0 * P.omega * u[2] + u[0] * w2 * x;
      double ds2 = -2.0 * P.omega * u[1] + u[0] * w2 * y;
      double ds4 = w2 * (x * u[1] + y * u[2]);
      r[0] = r[0] + 0.0;
      r[1] = r[1] + ds1;
      r[2] = r[2] + ds2;
      r[3] = r[3] + 0.0;
      r[4] = r[4] + ds4;
      r[5] = r[5] + 0.0;
    }
    if (P.has_grav) {
      double ds4 = u[1] * g[0] + u[2] * g[1] + u[3] * g[2] + 0.5 * u[0] * g[3];
      r[0] = r[0] + 0.0;
      r[1] = r[1] + u[0] * g[0];
      r[2] = r[2] + u[0] * g[1];
      r[3] = r[3] + u[0] * g[2];
      r[4] = r[4] + ds4;
      r[5] = r[5] + 0.0;
    }
  }
#pragma unroll
  for (int v = 0; v < NF; v++) {
    double st = u[v] + P.dt * r[v];
    nw[v] = (P.a != 0.0) ? P.a * u0[v] + P.b * st : st;
  }
}

// second part: dual-energy resync and floors (nw in, out)
OMB_HD void update_cell_fin(const UpdateParams& P, double* nw, double* out) {
  {  // dual_energy_sync
    double kin = div_nz(0.5 * ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]), nw[0]);
    double e1 = nw[4] - kin;
    if (e1 >= P.eta * nw[4]) nw[5] = pow_glibc(fabs(e1), P.inv_gamma);
  }
  if (P.floor_rho > 0.0 && nw[0] < P.floor_rho) nw[0] = P.floor_rho;
  if (P.floor_vmax > 0.0 && P.floor_rho > 0.0) {
    bool thin = nw[0] < 100.0 * P.floor_rho;
    double v2 = ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / (nw[0] * nw[0]);
    if (thin && v2 > P.floor_vmax * P.floor_vmax) {
      double scale = P.floor_vmax / sqrt(v2 > 1e-300 ? v2 : 1e-300);
      double kin_old = 0.5 * ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / nw[0];
      nw[1] *= scale;
      nw[2] *= scale;
      nw[3] *= scale;
      double kin_new = 0.5 * ((nw[1] * nw[1] + nw[2] * nw[2]) + nw[3] * nw[3]) / nw[0];
      nw[4] += kin_new - kin_old;
    }
  }
  if (P.floor_tau > 0.0 && nw[5] < P.floor_tau) nw[5] = P.floor_tau;
#pragma unroll
  for (int v = 0; v < NF; v++) out[v] = nw[v];
}

OMB_HD void update_cell(const UpdateParams& P, const double* u, const double* u0, double* r, double x, double y,
                        const double* g /* gx gy gz dphi_dt or null */, double* out) {
  double nw[NF];
  update_cell_rk(P, u, u0, r, x, y, g, nw);
  update_cell_fin(P, nw, out);
}

}  // namespace omb
