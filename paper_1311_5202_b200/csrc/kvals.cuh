// kvals.cuh -- complex helpers and the kernel values K(x, n_x; y, n_y) shared by the apply kernels (kernels.cu)
// and the locally corrected Nystrom weights (nystrom.cu).
#pragma once
#include <cuda_runtime.h>

namespace fda {

#define FDA_INV4PI 0.079577471545947667884

// ---------------------------------------------------------------- complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

// ---------------------------------------------------------------- kernel values
// K = dG/dn_y + alpha d2G/dn_x dn_y at d = x - y (eq_hmat), combined form:
//   K = -E/r^3 [ (ikr-1)(b + alpha c) + alpha (3 - 3ikr - k^2 r^2) a b / r^2 ],
//   E = e^{ikr}/(4 pi), a = d.n_x, b = d.n_y, c = n_x.n_y
__device__ __forceinline__ double2 bm_h(double dx, double dy, double dz, double nxx, double nxy, double nxz,
                                        double nyx, double nyy, double nyz, double k, double2 alpha) {
  const double r2 = dx * dx + dy * dy + dz * dz;
  const double ir = rsqrt(r2);
  const double r = r2 * ir;
  const double kr = k * r;
  double sn, cs;
  sincos(kr, &sn, &cs);
  const double a = dx * nxx + dy * nxy + dz * nxz;
  const double b = dx * nyx + dy * nyy + dz * nyz;
  const double c = nxx * nyx + nxy * nyy + nxz * nyz;
  const double ir2 = ir * ir;
  // u = ikr - 1 ; v = 3 - k^2 r^2 - 3ikr
  const double2 u = make_double2(-1.0, kr);
  const double2 v = make_double2(3.0 - kr * kr, -3.0 * kr);
  const double2 t1 = make_double2(b + alpha.x * c, alpha.y * c);       // b + alpha c
  double2 inner = cmul(u, t1);
  const double2 av = cmul(alpha, v);
  const double ab = a * b * ir2;
  inner.x = fma(av.x, ab, inner.x);
  inner.y = fma(av.y, ab, inner.y);
  const double f = -FDA_INV4PI * ir2 * ir;                               // -1/(4 pi r^3)
  const double2 E = make_double2(cs * f, sn * f);
  return cmul(E, inner);
}

// dG/dn_y(a, y) at d = a - y:  -e^{ikr}(ikr - 1)(d.n_y)/(4 pi r^3)    (S2M E_up, eq_evas2mh)
__device__ __forceinline__ double2 dg_dny(double dx, double dy, double dz, double nyx, double nyy, double nyz,
                                          double k) {
  const double r2 = dx * dx + dy * dy + dz * dz;
  const double ir = rsqrt(r2);
  const double r = r2 * ir;
  const double kr = k * r;
  double sn, cs;
  sincos(kr, &sn, &cs);
  const double b = (dx * nyx + dy * nyy + dz * nyz) * (-FDA_INV4PI) * ir * ir * ir;
  // e^{ikr}(ikr - 1) = (cs + i sn)(-1 + i kr) = (-cs - kr sn) + i(kr cs - sn)
  return make_double2((-cs - kr * sn) * b, (kr * cs - sn) * b);
}

// G at d = a - y: e^{ikr}/(4 pi r)   (S2M E_up of the single layer, BM_G plans)
__device__ __forceinline__ double2 g_only(double dx, double dy, double dz, double k) {
  const double r2 = dx * dx + dy * dy + dz * dz;
  const double ir = rsqrt(r2);
  const double kr = k * r2 * ir;
  double sn, cs;
  sincos(kr, &sn, &cs);
  const double f = FDA_INV4PI * ir;
  return make_double2(cs * f, sn * f);
}

// G + alpha dG/dn_x at d = x - y:  e^{ikr}/(4 pi r) [1 + alpha (ikr - 1)(d.n_x)/r^2]   (eq_eval2t)
__device__ __forceinline__ double2 bm_g(double dx, double dy, double dz, double nxx, double nxy, double nxz,
                                        double k, double2 alpha) {
  const double r2 = dx * dx + dy * dy + dz * dz;
  const double ir = rsqrt(r2);
  const double r = r2 * ir;
  const double kr = k * r;
  double sn, cs;
  sincos(kr, &sn, &cs);
  const double a = (dx * nxx + dy * nxy + dz * nxz) * ir * ir;
  // 1 + alpha (ikr - 1) a
  const double2 ua = make_double2(-a, kr * a);
  const double2 t = cmul(alpha, ua);
  const double f = FDA_INV4PI * ir;
  return cmul(make_double2(cs * f, sn * f), make_double2(1.0 + t.x, t.y));
}

}  // namespace fda
