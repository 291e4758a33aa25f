// nystrom.cu -- locally corrected Nystrom weights on the device.
//
// For a field point x and an element Delta of its local region D_i that does not contain x, the
// corrected weights wbar_j^Delta(K; x) solve (eq:local correction)
//     sum_j wbar_j phi^(n)(xi_j) = I_n = int_Delta K(x, y) phi^(n)(y) dy,   phi^(n) = xi1^p xi2^q, p + q <= 2,
// and the moments I_n, nearly singular when x is close to Delta, are computed "by using a recursive subdivision
// quadrature".  The paper gives neither the subdivision criterion nor the rule; reading R27
// (DESIGN.md): a sub-triangle of the reference triangle is split at its edge mid-points while its largest mapped
// edge h exceeds theta x the distance from x to the nearest of its mapped corners and centroid, or while the map
// is not flat enough on it (|y(G) - mean of the mapped corners| > gamma h: strongly curved elements, where the
// element map rather than the distance limits the smoothness of the integrand); a leaf is integrated by the
// nq x nq Gauss-Legendre product rule on the collapsed square.
//
// One warp per (field point, element) pair: the subdivision is an explicit depth-first stack in shared memory
// (every lane takes the same decisions), the nq^2 points of a leaf are spread over the lanes, the six complex
// moments are reduced by shuffles, lanes 0-5 apply the inverse moment matrix and write wbar_j (and the delta
// CSR value wbar_j - w_j K(x, y_j) of reading R4).  Fixed evaluation order: results are deterministic.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "fda.h"
#include "kvals.cuh"

namespace fda {
namespace {

constexpr int NY_WARPS = 4;        // warps (pairs) per CTA
constexpr int NY_MAXQ = 16;        // largest Gauss-Legendre order
constexpr int NY_MAXDEPTH = 20;    // deepest subdivision
constexpr int NY_STACK = 3 * NY_MAXDEPTH + 4;

struct NyConst {
  double gu[NY_MAXQ], gw[NY_MAXQ];  // Gauss-Legendre nodes / weights on [0, 1]
  double minv[6][6];                // inverse of M[n][j] = phi^(n)(xi_j): wbar_j = sum_n minv[j][n] I_n
  double xi[6][2], wref[6];         // the element's quadrature points and reference weights (sum 1/2)
};
__constant__ NyConst c_ny;

// The 6-node triangle (corners 1 2 3, mid-edges 12 23 31) as a quadratic polynomial in (a, b):
//   y = c0 + c1 a + c2 b + c3 a^2 + c4 a b + c5 b^2   (the shape functions N_q(a, b) expanded in monomials)
__device__ __forceinline__ void ny_coeffs(const double* __restrict__ P, double (&C)[18]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double p1 = P[c], p2 = P[3 + c], p3 = P[6 + c], p4 = P[9 + c], p5 = P[12 + c], p6 = P[15 + c];
    C[c] = p1;
    C[3 + c] = -3.0 * p1 - p2 + 4.0 * p4;
    C[6 + c] = -3.0 * p1 - p3 + 4.0 * p6;
    C[9 + c] = 2.0 * p1 + 2.0 * p2 - 4.0 * p4;
    C[12 + c] = 4.0 * (p1 - p4 + p5 - p6);
    C[15 + c] = 2.0 * p1 + 2.0 * p3 - 4.0 * p6;
  }
}
// y(a, b), and optionally the unit normal t1 x t2 / J and J (t1 = dy/da, t2 = dy/db)
__device__ __forceinline__ void ny_map(const double (&C)[18], double a, double b, double (&y)[3], double* nv,
                                       double* J) {
  const double aa = a * a, ab = a * b, bb = b * b;
#pragma unroll
  for (int c = 0; c < 3; ++c)
    y[c] = fma(C[15 + c], bb, fma(C[12 + c], ab, fma(C[9 + c], aa, fma(C[6 + c], b, fma(C[3 + c], a, C[c])))));
  if (nv) {
    double t1[3], t2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      t1[c] = fma(2.0 * C[9 + c], a, fma(C[12 + c], b, C[3 + c]));
      t2[c] = fma(2.0 * C[15 + c], b, fma(C[12 + c], a, C[6 + c]));
    }
    const double cx = t1[1] * t2[2] - t1[2] * t2[1], cy = t1[2] * t2[0] - t1[0] * t2[2],
                 cz = t1[0] * t2[1] - t1[1] * t2[0];
    const double j2 = cx * cx + cy * cy + cz * cz, ij = rsqrt(j2);
    *J = j2 * ij;
    nv[0] = cx * ij, nv[1] = cy * ij, nv[2] = cz * ij;
  }
}

__device__ __forceinline__ double ny_dist(const double (&a)[3], const double (&b)[3]) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return sqrt(dx * dx + dy * dy + dz * dz);
}

template <int KERNEL>
__device__ __forceinline__ double2 ny_kernel(const double (&x)[3], const double (&nx)[3], const double (&y)[3],
                                             const double (&ny)[3], double k, double2 alpha) {
  const double dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
  if (KERNEL == FDA_KERNEL_BMH) return bm_h(dx, dy, dz, nx[0], nx[1], nx[2], ny[0], ny[1], ny[2], k, alpha);
  if (KERNEL == FDA_KERNEL_BMG) return bm_g(dx, dy, dz, nx[0], nx[1], nx[2], k, alpha);
  // FDA_KERNEL_T1: G + alpha dG/dn_y
  const double2 g = g_only(dx, dy, dz, k), d = dg_dny(dx, dy, dz, ny[0], ny[1], ny[2], k);
  const double2 ad = cmul(alpha, d);
  return make_double2(g.x + ad.x, g.y + ad.y);
}

struct NyTri {
  double a0, a1, b0, b1, c0, c1;
  int depth;
};

// flag bits: 1 = pair index out of range, 2 = field point on the element (subdivision unresolved at max_depth)
template <int KERNEL>
__global__ void __launch_bounds__(32 * NY_WARPS, 4)
    k_nystrom_weights(const double* __restrict__ elem, int64_t ne, const double* __restrict__ tx,
                      const double* __restrict__ tn, int64_t nt, const int64_t* __restrict__ pair_t,
                      const int64_t* __restrict__ pair_e, int64_t npairs, double k, double2 alpha, int nq,
                      double theta, double gamma, int max_depth, double2* __restrict__ wbar,
                      double2* __restrict__ delta, int* __restrict__ flag, unsigned long long* __restrict__ next) {
  __shared__ NyTri stack[NY_WARPS][NY_STACK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Persistent warps take pairs from a device counter: the work per pair varies by two orders of magnitude
  // with the distance of the field point (a far element of D_i is one leaf, an adjacent one ~50), so a fixed
  // pair -> warp map leaves most resident warps idle (ncu: 6.6 of 64 warps active per SM, 26 Mpairs/s).
  // The result of a pair does not depend on which warp computes it.
  for (;;) {
    long long p = 0;
    if (lane == 0) p = (long long)atomicAdd(next, 1ull);
    p = __shfl_sync(0xffffffffu, p, 0);
    if (p >= npairs) return;
    const int64_t t = pair_t[p], e = pair_e[p];
    if (t < 0 || t >= nt || e < 0 || e >= ne) {
      if (lane == 0) atomicOr(flag, 1);
      continue;
    }
    double P[18], x[3], nx[3];  // P: the element's monomial coefficients
    ny_coeffs(elem + 18 * e, P);
#pragma unroll
    for (int c = 0; c < 3; ++c) x[c] = tx[3 * t + c], nx[c] = tn[3 * t + c];

    double2 mom[6];
#pragma unroll
    for (int n = 0; n < 6; ++n) mom[n] = make_double2(0.0, 0.0);
    NyTri* st = stack[warp];
    int top = 0;
    if (lane == 0) st[0] = NyTri{0.0, 0.0, 1.0, 0.0, 0.0, 1.0, 0};
    __syncwarp();
    top = 1;
    bool touching = false;
    const int nq2 = nq * nq;
    while (top > 0) {
      const NyTri T = st[--top];
      __syncwarp();
      // lane & 3 selects one of the corners A, B, C or the centroid G: one map per lane instead of four, the
      // distances combined by shuffles inside each group of four lanes (every group holds the same values, so the
      // decision stays uniform over the warp)
      const int sel = lane & 3;
      const double pa = sel == 0 ? T.a0 : sel == 1 ? T.b0 : sel == 2 ? T.c0 : (T.a0 + T.b0 + T.c0) / 3.0;
      const double pb = sel == 0 ? T.a1 : sel == 1 ? T.b1 : sel == 2 ? T.c1 : (T.a1 + T.b1 + T.c1) / 3.0;
      double ys[3], yn[3];
      ny_map(P, pa, pb, ys, nullptr, nullptr);
      const int nxt = (lane & ~3) | (sel == 2 ? 0 : sel + 1);  // A -> B -> C -> A (G: unused)
#pragma unroll
      for (int c = 0; c < 3; ++c) yn[c] = __shfl_sync(0xffffffffu, ys[c], nxt);
      double h = sel == 3 ? 0.0 : ny_dist(ys, yn);
      double d = ny_dist(x, ys);
      // flatness of the mapped sub-triangle: |y(G) - (y(A) + y(B) + y(C)) / 3|, the quadratic part of the map
      double cs[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) cs[c] = sel == 3 ? 0.0 : ys[c];
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        h = fmax(h, __shfl_xor_sync(0xffffffffu, h, o));
        d = fmin(d, __shfl_xor_sync(0xffffffffu, d, o));
#pragma unroll
        for (int c = 0; c < 3; ++c) cs[c] += __shfl_xor_sync(0xffffffffu, cs[c], o);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) cs[c] *= (1.0 / 3.0);
      const double flat = __shfl_sync(0xffffffffu, ny_dist(ys, cs), lane | 3);
      if ((h > theta * d || flat > gamma * h) && T.depth < max_depth) {
        if (lane == 0) {
          const double ab0 = 0.5 * (T.a0 + T.b0), ab1 = 0.5 * (T.a1 + T.b1);
          const double bc0 = 0.5 * (T.b0 + T.c0), bc1 = 0.5 * (T.b1 + T.c1);
          const double ca0 = 0.5 * (T.c0 + T.a0), ca1 = 0.5 * (T.c1 + T.a1);
          const int dd = T.depth + 1;
          st[top + 0] = NyTri{ab0, ab1, bc0, bc1, ca0, ca1, dd};
          st[top + 1] = NyTri{ca0, ca1, bc0, bc1, T.c0, T.c1, dd};
          st[top + 2] = NyTri{ab0, ab1, T.b0, T.b1, bc0, bc1, dd};
          st[top + 3] = NyTri{T.a0, T.a1, ab0, ab1, ca0, ca1, dd};
        }
        top += 4;
        __syncwarp();
        continue;
      }
      // still unresolved at the deepest level: the field point lies on the element (or closer to it than
      // 2^-max_depth side lengths / theta) -- the singular case this routine does not cover
      if (!(h <= theta * d)) touching = true;
      const double area2 = fabs((T.b0 - T.a0) * (T.c1 - T.a1) - (T.b1 - T.a1) * (T.c0 - T.a0));
      for (int q = lane; q < nq2; q += 32) {
        const int ia = q / nq, ib = q - ia * nq;
        const double u = c_ny.gu[ia], v = c_ny.gu[ib];
        const double s1 = T.a0 + u * ((T.b0 - T.a0) + v * (T.c0 - T.b0));
        const double s2 = T.a1 + u * ((T.b1 - T.a1) + v * (T.c1 - T.b1));
        double y[3], nyv[3], J;
        ny_map(P, s1, s2, y, nyv, &J);
        const double2 kv = ny_kernel<KERNEL>(x, nx, y, nyv, k, alpha);
        const double wq = c_ny.gw[ia] * c_ny.gw[ib] * u * area2 * J;
        const double2 f = make_double2(kv.x * wq, kv.y * wq);
        const double m[6] = {1.0, s1, s2, s1 * s1, s1 * s2, s2 * s2};
#pragma unroll
        for (int n = 0; n < 6; ++n) mom[n].x = fma(f.x, m[n], mom[n].x), mom[n].y = fma(f.y, m[n], mom[n].y);
      }
    }
#pragma unroll
    for (int n = 0; n < 6; ++n)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mom[n].x += __shfl_xor_sync(0xffffffffu, mom[n].x, o);
        mom[n].y += __shfl_xor_sync(0xffffffffu, mom[n].y, o);
      }
    if (touching) {
      if (lane == 0) atomicOr(flag, 2);
      continue;
    }
    if (lane < 6) {
      double2 w = make_double2(0.0, 0.0);
#pragma unroll
      for (int n = 0; n < 6; ++n) w.x = fma(c_ny.minv[lane][n], mom[n].x, w.x), w.y = fma(c_ny.minv[lane][n], mom[n].y, w.y);
      if (wbar) wbar[6 * p + lane] = w;
      if (delta) {  // wbar_j - w_j K(x, y_j): what the correction CSR holds next to the plain far quadrature (R4)
        double y[3], nyv[3], J;
        ny_map(P, c_ny.xi[lane][0], c_ny.xi[lane][1], y, nyv, &J);
        const double2 kv = ny_kernel<KERNEL>(x, nx, y, nyv, k, alpha);
        const double wj = c_ny.wref[lane] * J;
        delta[6 * p + lane] = make_double2(w.x - wj * kv.x, w.y - wj * kv.y);
      }
    }
    __syncwarp();
  }  // next pair
}

// Gauss-Legendre nodes and weights on [0, 1] (Newton iteration on P_n from the Chebyshev-like initial guess)
void gauss_legendre01(int n, double* x, double* w) {
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < n; ++i) {
    double z = std::cos(pi * (i + 0.75) / (n + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int j = 2; j <= n; ++j) {
        const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
        p0 = p1, p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    {  // derivative at the converged node
      double p0 = 1.0, p1 = z;
      for (int j = 2; j <= n; ++j) {
        const double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
        p0 = p1, p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
    }
    x[i] = 0.5 * (z + 1.0);
    w[i] = 1.0 / ((1.0 - z * z) * dp * dp);  // = (2 / ((1 - z^2) P_n'(z)^2)) / 2 on [0, 1]
  }
}

// inverse of the 6 x 6 moment matrix by Gauss-Jordan with partial pivoting; false if singular
bool invert6(double (&A)[6][6], double (&inv)[6][6]) {
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) inv[i][j] = i == j ? 1.0 : 0.0;
  for (int c = 0; c < 6; ++c) {
    int piv = c;
    for (int r = c + 1; r < 6; ++r)
      if (std::fabs(A[r][c]) > std::fabs(A[piv][c])) piv = r;
    if (std::fabs(A[piv][c]) < 1e-14) return false;
    for (int q = 0; q < 6; ++q) std::swap(A[c][q], A[piv][q]), std::swap(inv[c][q], inv[piv][q]);
    const double d = 1.0 / A[c][c];
    for (int q = 0; q < 6; ++q) A[c][q] *= d, inv[c][q] *= d;
    for (int r = 0; r < 6; ++r) {
      if (r == c) continue;
      const double f = A[r][c];
      for (int q = 0; q < 6; ++q) A[r][q] -= f * A[c][q], inv[r][q] -= f * inv[c][q];
    }
  }
  return true;
}

bool on_device(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// device view of a caller array (host arrays are copied into a scratch allocation)
struct DevIn {
  const void* ptr = nullptr;
  void* owned = nullptr;
  cudaError_t get(const void* src, size_t bytes) {
    if (bytes == 0 || on_device(src)) {
      ptr = src;
      return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(&owned, bytes);
    if (e != cudaSuccess) return e;
    ptr = owned;
    return cudaMemcpy(owned, src, bytes, cudaMemcpyHostToDevice);
  }
  ~DevIn() {
    if (owned) cudaFree(owned);
  }
};

}  // namespace
}  // namespace fda

extern "C" fda_status fda_nystrom_weights(int kernel, double k, double alpha_re, double alpha_im,
                                          const double* elem_nodes, int64_t ne, const double* xi, const double* wref,
                                          const double* tx, const double* tn, int64_t nt, const int64_t* pair_t,
                                          const int64_t* pair_e, int64_t npairs, int nq, double theta, double gamma,
                                          int max_depth, double* wbar, double* delta) {
  using namespace fda;
  if (kernel != FDA_KERNEL_BMH && kernel != FDA_KERNEL_BMG && kernel != FDA_KERNEL_T1) return FDA_ERR_INVALID_ARG;
  if (!(k >= 0.0) || !std::isfinite(k) || !std::isfinite(alpha_re) || !std::isfinite(alpha_im)) return FDA_ERR_INVALID_ARG;
  if (ne < 0 || nt < 0 || npairs < 0 || !xi || !wref || (!wbar && !delta)) return FDA_ERR_INVALID_ARG;
  if (nq == 0) nq = 8;
  // without the flatness split, nq = 8 reaches 5e-13 on gently curved elements but only 8e-7 on the tip
  // elements of a 10:1:1 spheroid, where the element map, not the distance, limits the smoothness (R27)
  if (gamma == 0.0) gamma = 0.05;
  if (theta == 0.0) theta = 0.5;
  if (max_depth == 0) max_depth = 16;
  if (nq < 2 || nq > NY_MAXQ || !(theta > 0.0 && theta <= 1.0) || !(gamma > 0.0) || max_depth < 1 || max_depth > NY_MAXDEPTH)
    return FDA_ERR_INVALID_ARG;
  if (npairs == 0) return FDA_OK;
  if (!elem_nodes || !tx || !tn || !pair_t || !pair_e || ne == 0 || nt == 0) return FDA_ERR_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return FDA_ERR_CUDA;  // no CPU fallback
  }
  // the rule constants live in one __constant__ block: concurrent calls are serialised
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  NyConst C{};
  gauss_legendre01(nq, C.gu, C.gw);
  double hxi[12], hw[6];
  if (on_device(xi)) {
    if (cudaMemcpy(hxi, xi, sizeof hxi, cudaMemcpyDeviceToHost) != cudaSuccess) return FDA_ERR_CUDA;
  } else
    for (int i = 0; i < 12; ++i) hxi[i] = xi[i];
  if (on_device(wref)) {
    if (cudaMemcpy(hw, wref, sizeof hw, cudaMemcpyDeviceToHost) != cudaSuccess) return FDA_ERR_CUDA;
  } else
    for (int i = 0; i < 6; ++i) hw[i] = wref[i];
  double M[6][6];
  for (int j = 0; j < 6; ++j) {
    const double a = hxi[2 * j], b = hxi[2 * j + 1];
    if (!std::isfinite(a) || !std::isfinite(b) || !(hw[j] > 0.0)) return FDA_ERR_INVALID_ARG;
    M[0][j] = 1.0, M[1][j] = a, M[2][j] = b, M[3][j] = a * a, M[4][j] = a * b, M[5][j] = b * b;
    C.xi[j][0] = a, C.xi[j][1] = b, C.wref[j] = hw[j];
  }
  if (!invert6(M, C.minv)) return FDA_ERR_INVALID_ARG;  // the six points do not determine the quadratic moments
  if (cudaMemcpyToSymbol(c_ny, &C, sizeof C) != cudaSuccess) return FDA_ERR_CUDA;

  DevIn de, dx, dn, dt, dpe;
  cudaError_t e = de.get(elem_nodes, (size_t)ne * 18 * sizeof(double));
  if (e == cudaSuccess) e = dx.get(tx, (size_t)nt * 3 * sizeof(double));
  if (e == cudaSuccess) e = dn.get(tn, (size_t)nt * 3 * sizeof(double));
  if (e == cudaSuccess) e = dt.get(pair_t, (size_t)npairs * sizeof(int64_t));
  if (e == cudaSuccess) e = dpe.get(pair_e, (size_t)npairs * sizeof(int64_t));
  const size_t obytes = (size_t)npairs * 6 * sizeof(double2);
  double2 *dw = nullptr, *dd = nullptr;
  void *ow = nullptr, *od = nullptr;
  int* dflag = nullptr;  // flag word, then the 8-byte pair counter
  auto cleanup = [&] {
    if (ow) cudaFree(ow);
    if (od) cudaFree(od);
    if (dflag) cudaFree(dflag);
  };
  auto fail = [&](cudaError_t err) {
    cleanup();
    cudaGetLastError();
    return err == cudaErrorMemoryAllocation ? FDA_ERR_OOM : FDA_ERR_CUDA;
  };
  if (e != cudaSuccess) return fail(e);
  if (wbar) {
    if (on_device(wbar))
      dw = reinterpret_cast<double2*>(wbar);
    else if ((e = cudaMalloc(&ow, obytes)) != cudaSuccess)
      return fail(e);
    else
      dw = static_cast<double2*>(ow);
  }
  if (delta) {
    if (on_device(delta))
      dd = reinterpret_cast<double2*>(delta);
    else if ((e = cudaMalloc(&od, obytes)) != cudaSuccess)
      return fail(e);
    else
      dd = static_cast<double2*>(od);
  }
  if ((e = cudaMalloc(&dflag, 16)) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(dflag, 0, 16)) != cudaSuccess) return fail(e);
  unsigned long long* dnext = reinterpret_cast<unsigned long long*>(dflag + 2);
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // persistent grid: the resident CTAs of every SM (launch bounds: 4 per SM), never more CTAs than pairs
  const unsigned grid = (unsigned)std::min<int64_t>((npairs + NY_WARPS - 1) / NY_WARPS, (int64_t)std::max(1, nsm) * 4);
  const double2 alpha = make_double2(alpha_re, alpha_im);
  auto launch = [&](auto kern) {
    kern<<<grid, 32 * NY_WARPS>>>(static_cast<const double*>(de.ptr), ne, static_cast<const double*>(dx.ptr),
                                  static_cast<const double*>(dn.ptr), nt, static_cast<const int64_t*>(dt.ptr),
                                  static_cast<const int64_t*>(dpe.ptr), npairs, k, alpha, nq, theta, gamma, max_depth, dw,
                                  dd, dflag, dnext);
  };
  if (kernel == FDA_KERNEL_BMH)
    launch(k_nystrom_weights<FDA_KERNEL_BMH>);
  else if (kernel == FDA_KERNEL_BMG)
    launch(k_nystrom_weights<FDA_KERNEL_BMG>);
  else
    launch(k_nystrom_weights<FDA_KERNEL_T1>);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  int flag = 0;
  if ((e = cudaMemcpy(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e);
  if (ow && (e = cudaMemcpy(wbar, ow, obytes, cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e);
  if (od && (e = cudaMemcpy(delta, od, obytes, cudaMemcpyDeviceToHost)) != cudaSuccess) return fail(e);
  cleanup();
  return flag ? FDA_ERR_INVALID_ARG : FDA_OK;
}
