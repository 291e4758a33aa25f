// kernels.cu -- device kernels of the FDA Burton-Miller apply.  See kernels.cuh.
#include "kernels.cuh"
#include "kvals.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace fda {

__device__ __forceinline__ int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// ---------------------------------------------------------------- H1 / H9
__global__ void k_permute_scale(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ w,
                                const double2* __restrict__ phi, double2* __restrict__ q, double2* __restrict__ phim) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n) return;
  const double2 v = phi[perm[m]];
  phim[m] = v;
  const double ww = w[m];
  q[m] = make_double2(ww * v.x, ww * v.y);
}
void launch_permute_scale(int64_t n, const int32_t* perm, const double* w, const double2* phi, double2* q,
                          double2* phim, cudaStream_t st) {
  if (n <= 0) return;
  k_permute_scale<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, perm, w, phi, q, phim);
}

__global__ void k_unpermute(int64_t n, const int32_t* __restrict__ perm, const double2* __restrict__ outm,
                            double2* __restrict__ out) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n) return;
  out[perm[m]] = outm[m];
}
void launch_unpermute(int64_t n, const int32_t* perm, const double2* outm, double2* out, cudaStream_t st) {
  if (n <= 0) return;
  k_unpermute<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, perm, outm, out);
}

// ---------------------------------------------------------------- multi-GPU expansion exchange
// pack: warp per send entry, buf[boff[e] + k] = X[xoff[e] + k], k < len[e]
__global__ void k_xpack(int64_t nent, const int64_t* __restrict__ xoff, const int32_t* __restrict__ len,
                        const int64_t* __restrict__ boff, const double2* __restrict__ X, double2* __restrict__ buf) {
  const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  if (e >= nent) return;
  const int lane = threadIdx.x & 31;
  const double2* src = X + xoff[e];
  double2* dst = buf + boff[e];
  for (int k = lane; k < len[e]; k += 32) dst[k] = src[k];
}
void launch_xpack(int64_t nent, const int64_t* xoff, const int32_t* len, const int64_t* boff, const double2* X,
                  double2* buf, cudaStream_t st) {
  if (nent <= 0) return;
  k_xpack<<<(unsigned)((nent * 32 + 255) / 256), 256, 0, st>>>(nent, xoff, len, boff, X, buf);
}
// unpack: warp per destination slot, X[xoff[d] + k] += sum over its received partials (peer order), so the
// sum is deterministic and needs no atomics
__global__ void k_xunpack(int64_t ndst, const int64_t* __restrict__ xoff, const int32_t* __restrict__ len,
                          const int64_t* __restrict__ rptr, const int64_t* __restrict__ roff,
                          const double2* __restrict__ buf, double2* __restrict__ X) {
  const int64_t d = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  if (d >= ndst) return;
  const int lane = threadIdx.x & 31;
  double2* dst = X + xoff[d];
  const int64_t pb = rptr[d], pe = rptr[d + 1];
  for (int k = lane; k < len[d]; k += 32) {
    double2 a = dst[k];
    for (int64_t p = pb; p < pe; ++p) a = cadd(a, buf[roff[p] + k]);
    dst[k] = a;
  }
}
void launch_xunpack(int64_t ndst, const int64_t* xoff, const int32_t* len, const int64_t* rptr, const int64_t* roff,
                    const double2* buf, double2* X, cudaStream_t st) {
  if (ndst <= 0) return;
  k_xunpack<<<(unsigned)((ndst * 32 + 255) / 256), 256, 0, st>>>(ndst, xoff, len, rptr, roff, buf, X);
}

// ---------------------------------------------------------------- H2 P2P near field
#define P2P_T 128
#define P2P_MAXL 256
template <int KIND>
__global__ void __launch_bounds__(P2P_T) k_p2p(const int64_t* __restrict__ leaf_ptr, const int64_t* __restrict__ p2p_ptr,
                                               const int32_t* __restrict__ p2p_src, Points P,
                                               const double2* __restrict__ q, double k, double2 alpha,
                                               double2* __restrict__ outm, int64_t leaf0) {
  __shared__ double sx[P2P_T], sy[P2P_T], sz[P2P_T], snx[P2P_T], sny[P2P_T], snz[P2P_T];
  __shared__ double2 sq[P2P_T];
  __shared__ int64_t sj[P2P_T];
  __shared__ int64_t lpre[P2P_MAXL + 1], lbeg[P2P_MAXL];
  __shared__ double2 red[P2P_T];
  const int64_t t = leaf0 + blockIdx.x;
  const int64_t tb = leaf_ptr[t], te = leaf_ptr[t + 1];
  const int nt = (int)(te - tb);
  const int ntp = nt >= P2P_T ? P2P_T : next_pow2(nt);
  const int nsl = P2P_T / ntp;
  const int my_t = threadIdx.x % ntp, my_sl = threadIdx.x / ntp;
  const int64_t sb0 = p2p_ptr[t], se0 = p2p_ptr[t + 1];
  for (int t0 = 0; t0 < nt; t0 += ntp) {
    const int64_t i = tb + t0 + my_t;
    const bool act = (t0 + my_t) < nt;
    double xi = 0, yi = 0, zi = 0, nxi = 0, nyi = 0, nzi = 0;
    if (act) xi = P.x[i], yi = P.y[i], zi = P.z[i], nxi = P.nx[i], nyi = P.ny[i], nzi = P.nz[i];
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t sb = sb0; sb < se0; sb += P2P_MAXL) {
      const int nl = (int)min((int64_t)P2P_MAXL, se0 - sb);
      __syncthreads();
      for (int l = threadIdx.x; l < nl; l += P2P_T) {
        const int64_t s = p2p_src[sb + l];
        lbeg[l] = leaf_ptr[s];
        lpre[l + 1] = leaf_ptr[s + 1] - leaf_ptr[s];
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        lpre[0] = 0;
        for (int l = 0; l < nl; ++l) lpre[l + 1] += lpre[l];
      }
      __syncthreads();
      const int64_t tot = lpre[nl];
      for (int64_t s0 = 0; s0 < tot; s0 += P2P_T) {
        const int64_t jj = s0 + threadIdx.x;
        if (jj < tot) {
          int lo = 0, hi = nl - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (lpre[mid] <= jj) lo = mid;
            else hi = mid - 1;
          }
          const int64_t j = lbeg[lo] + (jj - lpre[lo]);
          sx[threadIdx.x] = P.x[j], sy[threadIdx.x] = P.y[j], sz[threadIdx.x] = P.z[j];
          snx[threadIdx.x] = P.nx[j], sny[threadIdx.x] = P.ny[j], snz[threadIdx.x] = P.nz[j];
          sq[threadIdx.x] = q[j];
          sj[threadIdx.x] = j;
        }
        __syncthreads();
        const int cnt = (int)min((int64_t)P2P_T, tot - s0);
        if (act) {
          for (int u = my_sl; u < cnt; u += nsl) {
            if (sj[u] == i) continue;
            // KIND 1: G + alpha dG/dn_x; KIND 2: G + alpha dG/dn_y = the same form with n_x -> -n_y
            const double2 kv =
                KIND == 0   ? bm_h(xi - sx[u], yi - sy[u], zi - sz[u], nxi, nyi, nzi, snx[u], sny[u], snz[u], k, alpha)
                : KIND == 1 ? bm_g(xi - sx[u], yi - sy[u], zi - sz[u], nxi, nyi, nzi, k, alpha)
                            : bm_g(xi - sx[u], yi - sy[u], zi - sz[u], -snx[u], -sny[u], -snz[u], k, alpha);
            cfma(acc, kv, sq[u]);
          }
        }
        __syncthreads();
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (my_sl == 0 && act) {
      double2 s = red[my_t];
      for (int sl = 1; sl < nsl; ++sl) s = cadd(s, red[my_t + sl * ntp]);
      outm[i] = s;
    }
    __syncthreads();
  }
}
// Symmetric P2P for the BM_H kernel (single-rank plans): the near-field list is symmetric (leaf pair (T, S) is
// P2P iff (S, T) is, R20), and K_ij, K_ji share r, e^{ikr} and the alpha term: with d = x_i - x_j,
// a = d.n_i, b = d.n_j, c = n_i.n_j, E = e^{ikr}/(4 pi), u = ikr - 1,
//   C    = alpha ((3 - 3ikr - k^2 r^2) a b / r^5 + u c / r^3)
//   K_ij = -E (u b / r^3 + C),   K_ji = -E (-u a / r^3 + C)          (eq_hmat)
// The CTA of leaf T takes the pairs with source leaves S > T in both directions (the source side is reduced
// over the targets of the warp segment by shuffles, then one FP64 reduction per source point) and its own
// leaf S = T one way (j != i); outputs accumulate with FP64 reductions into the zeroed outm.
__device__ __forceinline__ void bm_h_pair(double dx, double dy, double dz, double nxx, double nxy, double nxz,
                                          double nyx, double nyy, double nyz, double k, double2 alpha, double2& kij,
                                          double2& kji) {
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
  const double2 u = make_double2(-1.0, kr);
  const double2 v = make_double2(3.0 - kr * kr, -3.0 * kr);
  // alpha (v a b / r^2 + u c)  (the common 1/r^3 is in f)
  double2 w = make_double2(u.x * c, u.y * c);
  const double ab = a * b * ir2;
  w.x = fma(v.x, ab, w.x);
  w.y = fma(v.y, ab, w.y);
  const double2 C = cmul(alpha, w);
  const double f = -FDA_INV4PI * ir2 * ir;  // -1/(4 pi r^3)
  const double2 E = make_double2(cs * f, sn * f);
  kij = cmul(E, make_double2(fma(u.x, b, C.x), fma(u.y, b, C.y)));
  kji = cmul(E, make_double2(fma(-u.x, a, C.x), fma(-u.y, a, C.y)));
}

__global__ void __launch_bounds__(P2P_T) k_p2p_sym(const int64_t* __restrict__ leaf_ptr,
                                                   const int64_t* __restrict__ p2p_ptr,
                                                   const int32_t* __restrict__ p2p_src, Points P,
                                                   const double2* __restrict__ q, double k, double2 alpha,
                                                   double2* __restrict__ outm) {
  __shared__ double sx[P2P_T], sy[P2P_T], sz[P2P_T], snx[P2P_T], sny[P2P_T], snz[P2P_T];
  __shared__ double2 sq[P2P_T];
  __shared__ int64_t sj[P2P_T];
  __shared__ int64_t lpre[P2P_MAXL + 1], lbeg[P2P_MAXL];
  __shared__ int lself[P2P_MAXL];
  __shared__ char sself[P2P_T];
  __shared__ double2 red[P2P_T];
  const int64_t t = blockIdx.x;
  const int64_t tb = leaf_ptr[t], te = leaf_ptr[t + 1];
  const int nt = (int)(te - tb);
  const int ntp = nt >= 32 ? 32 : next_pow2(nt);  // targets per segment: a power of two within one warp
  const int nsl = P2P_T / ntp;
  const int my_t = threadIdx.x % ntp, my_sl = threadIdx.x / ntp;
  const int64_t sb0 = p2p_ptr[t], se0 = p2p_ptr[t + 1];
  for (int t0 = 0; t0 < nt; t0 += ntp) {
    const int64_t i = tb + t0 + my_t;
    const bool act = (t0 + my_t) < nt;
    double xi = 0, yi = 0, zi = 0, nxi = 0, nyi = 0, nzi = 0;
    double2 qi = make_double2(0.0, 0.0);
    if (act) xi = P.x[i], yi = P.y[i], zi = P.z[i], nxi = P.nx[i], nyi = P.ny[i], nzi = P.nz[i], qi = q[i];
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t sb = sb0; sb < se0; sb += P2P_MAXL) {
      const int nl = (int)min((int64_t)P2P_MAXL, se0 - sb);
      __syncthreads();
      for (int l = threadIdx.x; l < nl; l += P2P_T) {
        const int64_t s = p2p_src[sb + l];
        lbeg[l] = leaf_ptr[s];
        lpre[l + 1] = s >= t ? leaf_ptr[s + 1] - leaf_ptr[s] : 0;  // source leaves S >= T only
        lself[l] = s == t;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        lpre[0] = 0;
        for (int l = 0; l < nl; ++l) lpre[l + 1] += lpre[l];
      }
      __syncthreads();
      const int64_t tot = lpre[nl];
      for (int64_t s0 = 0; s0 < tot; s0 += P2P_T) {
        const int64_t jj = s0 + threadIdx.x;
        if (jj < tot) {
          int lo = 0, hi = nl - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (lpre[mid] <= jj) lo = mid;
            else hi = mid - 1;
          }
          const int64_t j = lbeg[lo] + (jj - lpre[lo]);
          sx[threadIdx.x] = P.x[j], sy[threadIdx.x] = P.y[j], sz[threadIdx.x] = P.z[j];
          snx[threadIdx.x] = P.nx[j], sny[threadIdx.x] = P.ny[j], snz[threadIdx.x] = P.nz[j];
          sq[threadIdx.x] = q[j];
          sj[threadIdx.x] = j;
          sself[threadIdx.x] = (char)lself[lo];
        }
        __syncthreads();
        const int cnt = (int)min((int64_t)P2P_T, tot - s0);
        // uniform trip count over the slices of a warp (the source-side reduction shuffles need every lane)
        for (int m = 0; m * nsl < cnt; ++m) {
          const int u = m * nsl + my_sl;
          const bool on = u < cnt;
          double2 kij = make_double2(0.0, 0.0), kji = kij;
          bool self = false;
          if (on) {
            self = sself[u] != 0;
            if (act && sj[u] != i)
              bm_h_pair(xi - sx[u], yi - sy[u], zi - sz[u], nxi, nyi, nzi, snx[u], sny[u], snz[u], k, alpha, kij,
                        kji);
            cfma(acc, kij, sq[u]);
          }
          // source side (S > T): sum over this segment's targets of K_ji q_i, one reduction per source point
          double2 v = make_double2(0.0, 0.0);
          if (on && !self) cfma(v, kji, qi);
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1)
            if (o < ntp) {
              v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
              v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
            }
          if (on && !self && my_t == 0) {
            atomicAdd(&outm[sj[u]].x, v.x);
            atomicAdd(&outm[sj[u]].y, v.y);
          }
        }
        __syncthreads();
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (my_sl == 0 && act) {
      double2 s = red[my_t];
      for (int sl = 1; sl < nsl; ++sl) s = cadd(s, red[my_t + sl * ntp]);
      atomicAdd(&outm[i].x, s.x);
      atomicAdd(&outm[i].y, s.y);
    }
    __syncthreads();
  }
}
void launch_p2p_sym(int64_t nleaf, const int64_t* leaf_ptr, const int64_t* p2p_ptr, const int32_t* p2p_src, Points P,
                    const double2* q, double k, double2 alpha, double2* outm, cudaStream_t st) {
  if (nleaf <= 0) return;
  k_p2p_sym<<<(unsigned)nleaf, P2P_T, 0, st>>>(leaf_ptr, p2p_ptr, p2p_src, P, q, k, alpha, outm);
}

void launch_p2p(int kind, int64_t nleaf, const int64_t* leaf_ptr, const int64_t* p2p_ptr, const int32_t* p2p_src,
                Points P, const double2* q, double k, double2 alpha, double2* outm, int64_t leaf0, cudaStream_t st) {
  if (nleaf <= 0) return;
  if (kind == 0)
    k_p2p<0><<<(unsigned)nleaf, P2P_T, 0, st>>>(leaf_ptr, p2p_ptr, p2p_src, P, q, k, alpha, outm, leaf0);
  else if (kind == 1)
    k_p2p<1><<<(unsigned)nleaf, P2P_T, 0, st>>>(leaf_ptr, p2p_ptr, p2p_src, P, q, k, alpha, outm, leaf0);
  else
    k_p2p<2><<<(unsigned)nleaf, P2P_T, 0, st>>>(leaf_ptr, p2p_ptr, p2p_src, P, q, k, alpha, outm, leaf0);
}

// ---------------------------------------------------------------- H3 correction SpMV (warp per row)
__global__ void k_csr(int64_t r0, int64_t r1, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                      const double2* __restrict__ val, const double2* __restrict__ phim, double2* __restrict__ outm) {
  const int64_t row = r0 + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= r1) return;
  double2 acc = make_double2(0.0, 0.0);
  const int64_t e = rp[row + 1];
  for (int64_t p = rp[row] + lane; p < e; p += 32) cfma(acc, __ldg(&val[p]), __ldg(&phim[__ldg(&col[p])]));
  for (int o = 16; o; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if (lane == 0) {
    double2 v = outm[row];
    outm[row] = cadd(v, acc);
  }
}
void launch_csr(int64_t r0, int64_t r1, const int64_t* rp, const int32_t* col, const double2* val,
                const double2* phim, double2* outm, cudaStream_t st) {
  if (r1 <= r0) return;
  const int64_t warps = r1 - r0;
  k_csr<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(r0, r1, rp, col, val, phim, outm);
}

// ---------------------------------------------------------------- H4 S2M (dipole check potentials)
// chk[leaf][i] = sum_{j in leaf} dG/dn_y(a_i, y_j) q_j  on the leaf's outgoing check surface
// (E_up of eq_evas2mh).  The reduction x~ = Sigma^-1 U^H chk (eq_cmps) is one
// dense group of the grouped-translation kernel (all leaves of a level share S).
#define S2M_T 128
#define S2M_MAXC 3
template <int KIND>
__global__ void __launch_bounds__(S2M_T) k_s2m_check(const int32_t* __restrict__ leaf_ids, LeafGeom L, Points P,
                                                     const double2* __restrict__ q, const double* __restrict__ surf,
                                                     int nsurf, double k, double2 alpha, double2* __restrict__ chk) {
  __shared__ double sx[S2M_T], sy[S2M_T], sz[S2M_T], snx[S2M_T], sny[S2M_T], snz[S2M_T];
  __shared__ double2 sq[S2M_T];
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t pb = L.ptr[leaf], pe = L.ptr[leaf + 1];
  const double cx = L.cx[leaf], cy = L.cy[leaf], cz = L.cz[leaf];
  double2* out = chk + (int64_t)blockIdx.x * nsurf;
  for (int i0 = 0; i0 < nsurf; i0 += S2M_T * S2M_MAXC) {  // check-point blocks (one pass for nsurf <= 384)
    double ax[S2M_MAXC], ay[S2M_MAXC], az[S2M_MAXC];
    double2 acc[S2M_MAXC];
#pragma unroll
    for (int c = 0; c < S2M_MAXC; ++c) {
      const int i = i0 + threadIdx.x + c * S2M_T;
      acc[c] = make_double2(0.0, 0.0);
      ax[c] = ay[c] = az[c] = 0.0;
      if (i < nsurf) ax[c] = cx + surf[3 * i], ay[c] = cy + surf[3 * i + 1], az[c] = cz + surf[3 * i + 2];
    }
    for (int64_t s0 = pb; s0 < pe; s0 += S2M_T) {
      const int64_t j = s0 + threadIdx.x;
      __syncthreads();
      if (j < pe) {
        sx[threadIdx.x] = P.x[j], sy[threadIdx.x] = P.y[j], sz[threadIdx.x] = P.z[j];
        snx[threadIdx.x] = P.nx[j], sny[threadIdx.x] = P.ny[j], snz[threadIdx.x] = P.nz[j];
        sq[threadIdx.x] = q[j];
      }
      __syncthreads();
      const int cnt = (int)min((int64_t)S2M_T, pe - s0);
#pragma unroll
      for (int c = 0; c < S2M_MAXC; ++c) {
        const int i = i0 + threadIdx.x + c * S2M_T;
        if (i >= nsurf) break;
        for (int u = 0; u < cnt; ++u)
          cfma(acc[c],
               KIND == 0   ? dg_dny(ax[c] - sx[u], ay[c] - sy[u], az[c] - sz[u], snx[u], sny[u], snz[u], k)
               : KIND == 1 ? g_only(ax[c] - sx[u], ay[c] - sy[u], az[c] - sz[u], k)
                           : bm_g(ax[c] - sx[u], ay[c] - sy[u], az[c] - sz[u], -snx[u], -sny[u], -snz[u], k, alpha),
               sq[u]);
      }
    }
#pragma unroll
    for (int c = 0; c < S2M_MAXC; ++c) {
      const int i = i0 + threadIdx.x + c * S2M_T;
      if (i < nsurf) out[i] = acc[c];
    }
  }
}
void launch_s2m_check(int kind, int64_t nleaves, const int32_t* leaf_ids, LeafGeom L, Points P, const double2* q,
                      const double* surf, int nsurf, double k, double2 alpha, double2* chk, cudaStream_t st) {
  if (nleaves <= 0) return;
  if (kind == 0)
    k_s2m_check<0><<<(unsigned)nleaves, S2M_T, 0, st>>>(leaf_ids, L, P, q, surf, nsurf, k, alpha, chk);
  else if (kind == 1)
    k_s2m_check<1><<<(unsigned)nleaves, S2M_T, 0, st>>>(leaf_ids, L, P, q, surf, nsurf, k, alpha, chk);
  else
    k_s2m_check<2><<<(unsigned)nleaves, S2M_T, 0, st>>>(leaf_ids, L, P, q, surf, nsurf, k, alpha, chk);
}

// ---------------------------------------------------------------- grouped translation (H5/H6/H7)
// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) complex GEMM per (item, group, chunk of GT_P pairs):
//   dense   : Y[out] += A X[in]                  A  : s_out x s_in
//   low rank: Y[out] += U (V X[in])               V  : r x s_in,  U : s_out x r      (eq_lrdk)
// Complex products by the 3M scheme: P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi);
// re = P1 - P2, im = P3 - P1 - P2 (3 real MMAs per complex MMA instead of 4).
// Matrices live in global memory in fragment order (api.cu frag_append): tile (mt, kt) of 8 x 4
// holds 32 real parts in lane order (lane -> row mt*8 + lane/4, col kt*4 + lane%4) then 32
// imaginary parts, so each A-fragment load of a warp is one coalesced 256-byte read (L2 / L1).
// The gathered input columns X (and the low-rank intermediate T) are B operands in shared memory,
// double2 (re, im) column-major with a leading dimension = 4 (mod 8) double2 (conflict-free
// 128-bit fragment loads).  X is gathered with cp.async into a double buffer: the next chunk's
// columns are in flight while the current chunk computes.
#define GT_T 256
#define GT_W (GT_T / 32)
// A warp unit computes (8 rows) x (CT 8-column tiles); CT = GT_P/8 (all the chunk's columns: each A
// fragment feeds 3*CT DMMAs) for the T stage and the atomic output, CT = 2 for owned outputs (more
// units -> better balance across warps when the output has few row tiles).

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// TMA bulk reduction (SASS UBLKRED): dst[0 .. bytes/8) += src[...] in FP64, shared -> global, element-wise
// atomic at L2; one instruction per output column instead of 2 s_out per-lane REDG atomics (the LSU issue
// rate of those bounded the translations: ~1.3 cycles per lane and SM).
__device__ __forceinline__ void bulk_red_f64(double2* gdst, const double2* ssrc, unsigned bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(gdst), "r"(sa),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// one lane per column of the staged tile Ys (ld s_out) issues its bulk reduction into Y[out slot]
__device__ __forceinline__ void bulk_issue_cols(double2* Y, const double2* Ys, const int* sOut, int s_out, int nb,
                                                int lane) {
  for (int c = lane; c < nb; c += 32) bulk_red_f64(Y + (int64_t)sOut[c] * s_out, Ys + c * s_out, (unsigned)s_out * 16u);
  bulk_commit();
}

// sector-complete reductions in the atomic epilogue (kernels.cu gt_stage; FDA_GT_SECTOR=1 enables them)
__constant__ int gt_sector_red = 0;
// diagnostics only (FDA_GT_NORED=1|2): drop the atomic output of the translations / replace it by plain stores,
// to measure what the FP64 reductions cost (results are wrong then)
__constant__ int gt_nored = 0;

__host__ __device__ __forceinline__ int gt_ld(int k) { return ((k + 3) / 8) * 8 + 4; }  // >= k, = 4 mod 8

// One GEMM stage: C (Mt*8 x GT_P) = A (Mt*8 x Kt*4, fragment order) x B (Kt*4 x GT_P, smem double2).
// Work units (row tile, column group, k split) are spread over the CTA's warps.
// mode 0: C into the smem tile Ts (ldt) (ksplit must be 1: shared-memory FP64 atomics are CAS loops);
// mode 3: rows < s_out of C into the smem tile Ts (ldt = s_out), for a bulk reduction into Y (ksplit 1);
// mode 1: Y[sOut[col]*s_out + row] += C (plain RMW; Y loaded before the k loop so the load latency
//         overlaps the MMAs); mode 2: same with global atomics.
template <int GT_P, int MODE, int GT_CT, bool ASM = false>
__device__ __forceinline__ void gt_stage(const double* __restrict__ Ag, int Mt, int Kt, int ksplit, const double2* Bs,
                                         int ldb, double2* Ts, int ldt, double2* __restrict__ Y, const int* sOut,
                                         int s_out, int nb, int lda_kt = 0, int wbase = 0, int nw = GT_W) {
  if (lda_kt == 0) lda_kt = Kt;  // k tiles per row tile in the fragment-order storage of A
  // the units are spread over warps [wbase, wbase + nw) of the CTA
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) - wbase;
  const int CG = GT_P / 8 / GT_CT;
  const int nunits = Mt * CG * ksplit;
  const int g = lane >> 2, t = lane & 3;
  for (int u = warp; u < nunits; u += nw) {
    const int ks = u % ksplit, rest = u / ksplit;
    const int mt = rest / CG, cg = rest - mt * CG;
    const int kb = (ks * Kt) / ksplit, ke = ((ks + 1) * Kt) / ksplit;
    const int row = mt * 8 + g;
    double2 yv[GT_CT][2];
    if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < GT_CT; ++c)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int col = (cg * GT_CT + c) * 8 + 2 * t + i;
          yv[c][i] = (row < s_out && col < nb) ? Y[(int64_t)sOut[col] * s_out + row] : make_double2(0.0, 0.0);
        }
    }
    double acc[GT_CT][3][2];
#pragma unroll
    for (int c = 0; c < GT_CT; ++c)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc[c][q][0] = acc[c][q][1] = 0.0;
    const double* ap = Ag + (size_t)mt * lda_kt * 64 + lane;
    const double2* bp = Bs + (cg * GT_CT * 8 + g) * ldb + t;
#pragma unroll 4
    for (int kt = kb; kt < ke; ++kt) {
      const double ar = ASM ? ap[kt * 64] : __ldg(ap + kt * 64), ai = ASM ? ap[kt * 64 + 32] : __ldg(ap + kt * 64 + 32);
      const double as = ar + ai;
#pragma unroll
      for (int c = 0; c < GT_CT; ++c) {
        const double2 b = bp[c * 8 * ldb + kt * 4];
        dmma(acc[c][0][0], acc[c][0][1], ar, b.x);
        dmma(acc[c][1][0], acc[c][1][1], ai, b.y);
        dmma(acc[c][2][0], acc[c][2][1], as, b.x + b.y);
      }
    }
    if (MODE == 2 && gt_sector_red && !(s_out & 1)) {
      // Sector-complete FP64 reductions.  The L2 applies REDs per 32-byte sector; a lane's own values
      // (real / imaginary part of one row for two columns) cover half of a sector per instruction.  The
      // values are redistributed by shuffles so that in each of the 4 instructions per column tile the 4
      // lanes 4q..4q+3 add (re, im) of rows 2h and 2h+1 of one column -- one full, 32-byte aligned sector
      // (s_out even: every Y row pair starts on a sector).  Halves the L2 sector operations.
#pragma unroll
      for (int c = 0; c < GT_CT; ++c) {
        double rr[2], mm[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          rr[i] = acc[c][0][i] - acc[c][1][i];
          mm[i] = acc[c][2][i] - acc[c][0][i] - acc[c][1][i];
        }
        const int q = lane >> 2, e = lane & 3, tt = q & 3;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = j >> 1, h = 2 * (j & 1) + (q >> 2);
          const int r = 2 * h + (e >> 1), src = r * 4 + tt;
          const double vre = __shfl_sync(0xffffffffu, rr[i], src);
          const double vim = __shfl_sync(0xffffffffu, mm[i], src);
          const double v = (e & 1) ? vim : vre;
          const int col = (cg * GT_CT + c) * 8 + 2 * tt + i, rw = mt * 8 + r;
          if (rw < s_out && col < nb && v != 0.0)
            atomicAdd(reinterpret_cast<double*>(Y + (int64_t)sOut[col] * s_out + rw) + (e & 1), v);
        }
      }
      continue;
    }
#pragma unroll
    for (int c = 0; c < GT_CT; ++c)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = (cg * GT_CT + c) * 8 + 2 * t + i;
        const double re = acc[c][0][i] - acc[c][1][i];
        const double im = acc[c][2][i] - acc[c][0][i] - acc[c][1][i];
        if (MODE == 0) {
          Ts[col * ldt + row] = make_double2(re, im);
        } else if (MODE == 3) {
          if (row < s_out) Ts[col * ldt + row] = make_double2(re, im);
        } else if (row < s_out && col < nb) {
          double2* y = Y + (int64_t)sOut[col] * s_out + row;
          if (MODE == 2) {
            // rows past the group's own expansion length (an HF wedge shorter than the level's padded s)
            // are exact zeros: no atomic for them
            if (gt_nored) {  // diagnostics (FDA_GT_NORED): 1 no output, 2 plain stores instead of reductions
              if (gt_nored == 2 || re == 1.2345e300) *y = make_double2(re, im);
            } else if (re != 0.0 || im != 0.0) {
              atomicAdd(&y->x, re);
              atomicAdd(&y->y, im);
            }
          } else {
            *y = make_double2(yv[c][i].x + re, yv[c][i].y + im);
          }
        }
      }
  }
}

// k split of an atomic Y stage with units = Mt row tiles (all columns; each split adds its partial sums
// with global atomics): the fewest splits that give every warp a unit, >= 3 k tiles each.
__device__ __forceinline__ int gt_ksplit_y(int Mt, int Kt) {
  if (Mt >= GT_W) return 1;
  return max(1, min((GT_W + Mt - 1) / Mt, Kt / 3));
}

// Column tiles per warp unit for a stage with Mt row tiles (x ksplit): the CT in {P/8, .., 2, 1} whose
// unit count fills the warps best (ties -> the larger CT: each A fragment feeds more MMAs).
template <int GT_P>
__device__ __forceinline__ int gt_pick_ct(int Mt, int ks) {
  int best = GT_P / 8;
  double beff = -1.0;
  for (int ct = GT_P / 8; ct >= 1; ct >>= 1) {
    const int n = Mt * ks * (GT_P / 8 / ct);
    const double eff = (double)n / (double)(GT_W * ((n + GT_W - 1) / GT_W));
    if (eff > beff + 0.05) beff = eff, best = ct;
  }
  return best;
}
// dispatch a stage on a runtime CT
template <int GT_P, int MODE, bool ASM>
__device__ __forceinline__ void gt_stage_ct(int ct, const double* __restrict__ Ag, int Mt, int Kt, int ksplit,
                                            const double2* Bs, int ldb, double2* Ts, int ldt,
                                            double2* __restrict__ Y, const int* sOut, int s_out, int nb,
                                            int lda_kt = 0, int wbase = 0, int nw = GT_W) {
  if (ct >= 4 && GT_P / 8 >= 4)
    gt_stage<GT_P, MODE, (GT_P / 8 >= 4 ? 4 : 1), ASM>(Ag, Mt, Kt, ksplit, Bs, ldb, Ts, ldt, Y, sOut, s_out, nb, lda_kt,
                                                      wbase, nw);
  else if (ct >= 2 && GT_P / 8 >= 2)
    gt_stage<GT_P, MODE, (GT_P / 8 >= 2 ? 2 : 1), ASM>(Ag, Mt, Kt, ksplit, Bs, ldb, Ts, ldt, Y, sOut, s_out, nb, lda_kt, wbase, nw);
  else
    gt_stage<GT_P, MODE, 1, ASM>(Ag, Mt, Kt, ksplit, Bs, ldb, Ts, ldt, Y, sOut, s_out, nb, lda_kt, wbase, nw);
}

// One CTA per work item.  Per chunk of GT_P pairs two barriers: [C] after the chunk's gather has
// landed (cp.async), [D] between the low-rank stages.  The next chunk's gather is issued right after
// [C] into the other buffer (NBUF = 2) or, with one buffer, after [D] (X is dead once T = V X) or
// after the dense stage; pair indices are triple-buffered and fetched two chunks ahead.
template <int GT_P, int NBUF, bool STAGE, bool YB>
__global__ void __launch_bounds__(GT_T, 2) k_gtrans(GTrans T, const double2* __restrict__ X, double2* __restrict__ Y) {
  extern __shared__ double2 gsm2[];
  const int s_in = T.s_in, s_out = T.s_out;
  const int kin = (s_in + 3) / 4, mout = (s_out + 7) / 8;  // k tiles of the input, m tiles of the output
  const int ldx = gt_ld(kin * 4), ldt = gt_ld(T.rmax8);
  double2* Ts = gsm2 + NBUF * GT_P * ldx;
  // YB (atomic items): the chunk's output tile (GT_P columns of s_out), bulk-reduced into Y per column
  double2* Ys = Ts + GT_P * ldt;
  // STAGE: the current group's fragment-order matrix block is copied (cp.async, contiguous) into shared
  // memory once per group and read from there by every chunk of the item
  double* Ms = reinterpret_cast<double*>(Ys + (YB ? GT_P * s_out : 0));
  __shared__ int sOut[3][GT_P], sIn[3][GT_P];  // pair indices of chunks i, i+1, i+2 (mod 3)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Persistent CTAs: CTA b walks the items item_order[b], item_order[b + G], ... (G = gridDim.x) as one
  // stream of chunks, so the next item's first gather overlaps the current item's last chunk and the
  // items resident at any time stay the consecutive block of the launch order (Morton locality).
  struct Cur {
    int64_t j, e, e_end, c;  // item slot j, entry e in [item start, e_end), first pair c of the chunk
  };
  auto item_at = [&](Cur& u) {
    while (u.j < T.n_items) {
      const int64_t it = T.item_order[u.j];
      u.e = T.item_ptr[it], u.e_end = T.item_ptr[it + 1];
      if (u.e < u.e_end) {
        u.c = T.ig_pb[u.e];
        return;
      }
      u.j += gridDim.x;
    }
  };
  auto valid = [&](const Cur& u) { return u.j < T.n_items; };
  auto advance = [&](Cur& u) {
    u.c += GT_P;
    if (u.c >= T.ig_pe[u.e]) {
      if (++u.e < u.e_end) {
        u.c = T.ig_pb[u.e];
      } else {
        u.j += gridDim.x;
        item_at(u);
      }
    }
  };
  Cur cur{(int64_t)blockIdx.x, 0, 0, 0};
  item_at(cur);
  if (!valid(cur)) return;
  // zero the X buffers once: the padding rows k in [s_in, 4 kin) are never written by the gather
  for (int i = tid; i < NBUF * GT_P * ldx; i += GT_T) gsm2[i] = make_double2(0.0, 0.0);
  auto load_idx = [&](int ib, const Cur& u) {
    if (tid < GT_P) {
      const int64_t p = u.c + tid;
      const bool v = p < T.ig_pe[u.e];
      sOut[ib][tid] = v ? T.out[p] : 0;
      sIn[ib][tid] = v ? T.in[p] : -1;
    }
  };
  // per-group expansion lengths (HF wedges are shorter than the level's padded s; their tails are zero):
  // k tiles of the input / row tiles of the output actually used, and the gathered length
  auto kin_of = [&](int grp) { return T.gsi ? (T.gsi[grp] + 3) / 4 : kin; };
  auto mout_of = [&](int grp) { return T.gso ? (T.gso[grp] + 7) / 8 : mout; };
  auto issue_x = [&](int xbuf, int ib, int grp) {  // warp per pair column, lanes along k (no division)
    double2* xb = gsm2 + xbuf * GT_P * ldx;
    const int len = min(4 * kin_of(grp), s_in);
    for (int c = warp; c < GT_P; c += GT_W) {
      const int src = sIn[ib][c];
      if (src < 0) continue;
      const double2* xs = X + (int64_t)src * s_in;
      for (int k = lane; k < len; k += 32) cp_async16(xb + c * ldx + k, xs + k);
    }
    cp_async_commit();
  };
  auto stage_m = [&](int grp) {
    const int rank = T.grank[grp], rt = (rank + 7) / 8;
    const double* src = T.pool + T.gmat[grp];
    const int nd = rank >= 0 ? (rt * kin + mout * 2 * rt) * 64 : mout * kin * 64;  // doubles, multiple of 64
    for (int i = tid; i < nd / 2; i += GT_T) cp_async16(Ms + 2 * i, src + 2 * i);
    cp_async_commit();
  };
  // prologue: indices of chunks 0 and 1, matrix of chunk 0, gather of chunk 0
  Cur c1 = cur;
  advance(c1);
  load_idx(0, cur);
  if (valid(c1)) load_idx(1, c1);
  if (STAGE) stage_m(T.ig_group[cur.e]);
  __syncthreads();
  issue_x(0, 0, T.ig_group[cur.e]);
  int xbuf = 0, ib = 0;
  bool ypend = false;  // YB: a bulk reduction of Ys is in flight (issued by warp 0)
  while (valid(cur)) {
    Cur nx = cur;
    advance(nx);
    const bool has_next = valid(nx);
    Cur n2 = nx;
    if (has_next) advance(n2);
    const bool has_next2 = has_next && valid(n2);
    const int64_t e = cur.e, c0 = cur.c;
    const int ib1 = ib == 2 ? 0 : ib + 1, ib2 = ib1 == 2 ? 0 : ib1 + 1;
    const int grp = T.ig_group[e];
    const int rank = T.grank[grp];
    const int rt = (rank + 7) / 8;  // low rank: m tiles of V = k-tile pairs of U
    // T stage work units = (row tile, column tiles): no k split (shared-memory FP64 atomics are CAS
    // loops on sm_100a); 2 column tiles per unit when >= half the warps get a unit, else 1
    int ct1 = T.ct1;
    if (ct1 <= 0) ct1 = rt * (GT_P / 16) >= GT_W / 2 ? 2 : 1;
    cp_async_wait<0>();
    if (YB && ypend && warp == 0) bulk_wait_read();  // the bulk engine has read the previous chunk's Ys
    __syncthreads();  // [C] X (and Ms) of this chunk visible; previous chunk finished everywhere
    const int nb = (int)min((int64_t)GT_P, T.ig_pe[e] - c0);
    const double* Mg = STAGE ? Ms : T.pool + T.gmat[grp];
    const double2* xb = gsm2 + xbuf * GT_P * ldx;
    const int kin_g = T.atomic ? kin_of(grp) : kin, mout_g = T.atomic ? mout_of(grp) : mout;
    if (NBUF == 2 && has_next) issue_x(xbuf ^ 1, ib1, T.ig_group[nx.e]);  // the other buffer was last read by chunk i-1
    if (rank >= 0) {
      gt_stage_ct<GT_P, 0, STAGE>(ct1, Mg, rt, kin_g, 1, xb, ldx, Ts, ldt, nullptr, nullptr, 0, 0, kin);
      __syncthreads();  // [D] T complete, X of this chunk no longer read
      if (NBUF == 1 && has_next) issue_x(0, ib1, T.ig_group[nx.e]);
      if (has_next2) load_idx(ib2, n2);  // buffer ib2 held chunk i-1's indices (done at [C])
      const double* U = Mg + (size_t)rt * kin * 64;
      const int kt2 = (rank + 3) / 4;  // U is stored with pad8(r) columns; ceil(r/4) k tiles are non-zero
      if (YB) {  // atomic items, mout >= GT_W (no k split)
        gt_stage_ct<GT_P, 3, STAGE>(T.ct2 > 0 ? T.ct2 : GT_P / 8, U, mout_g, kt2, 1, Ts, ldt, Ys, s_out, nullptr, nullptr,
                                    s_out, nb, 2 * rt);
        fence_async_smem();
        __syncthreads();
        if (warp == 0) bulk_issue_cols(Y, Ys, sOut[ib], s_out, nb, lane);
        ypend = true;
      } else if (T.atomic) {
        const int ks = gt_ksplit_y(mout, kt2);
        gt_stage_ct<GT_P, 2, STAGE>(T.ct2 > 0 ? T.ct2 : (T.ct2 < 0 ? gt_pick_ct<GT_P>(mout, ks) : GT_P / 8), U, mout_g,
                                    kt2, ks, Ts, ldt, nullptr, 0, Y, sOut[ib], s_out, nb, 2 * rt);
      } else
        gt_stage<GT_P, 1, 2, STAGE>(U, mout, kt2, 1, Ts, ldt, nullptr, 0, Y, sOut[ib], s_out, nb, 2 * rt);
    } else {
      if (YB) {
        gt_stage_ct<GT_P, 3, STAGE>(T.ct2 > 0 ? T.ct2 : GT_P / 8, Mg, mout_g, kin_g, 1, xb, ldx, Ys, s_out, nullptr,
                                    nullptr, s_out, nb, kin);
        fence_async_smem();
        __syncthreads();
        if (warp == 0) bulk_issue_cols(Y, Ys, sOut[ib], s_out, nb, lane);
        ypend = true;
      } else if (T.atomic) {
        const int ks = gt_ksplit_y(mout, kin_g);
        gt_stage_ct<GT_P, 2, STAGE>(T.ct2 > 0 ? T.ct2 : (T.ct2 < 0 ? gt_pick_ct<GT_P>(mout, ks) : GT_P / 8), Mg,
                                    mout_g, kin_g, ks, xb, ldx, nullptr, 0, Y, sOut[ib], s_out, nb, kin);
      } else
        gt_stage<GT_P, 1, 2, STAGE>(Mg, mout, kin, 1, xb, ldx, nullptr, 0, Y, sOut[ib], s_out, nb);
      if (has_next2) load_idx(ib2, n2);
      if (NBUF == 1 && has_next) {
        __syncthreads();  // X buffer free
        issue_x(0, ib1, T.ig_group[nx.e]);
      }
    }
    if (STAGE && has_next && T.ig_group[nx.e] != grp) {
      __syncthreads();  // every warp is done with Ms
      stage_m(T.ig_group[nx.e]);
    }
    cur = nx, ib = ib1;
    if (NBUF == 2) xbuf ^= 1;
  }
  if (YB && warp == 0) bulk_wait_all();
}

// Warp-specialised variant for items whose groups are all low rank (atomic items): warps 0-3 run the
// first stage T = V X of chunk i+1 while warps 4-7 run the second stage Y += U T of chunk i (T double
// buffered), so neither stage's few work units leave half the CTA idle at a barrier.  One CTA
// barrier per chunk; the stage-1 warps own the gather (cp.async) and wait for it with a named
// barrier among themselves, overlapping the stage-2 warps' work.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
// NT threads: 256 (two CTAs per SM) or 512 (one CTA per SM: 227 KB of shared memory, so the LF levels'
// operators can be staged too; 8 + 8 warps)
// OWN: owned items (T.atomic == 0: an item owns its output slots and walks several groups): plain
// read-modify-write of Y instead of FP64 atomics; the operators are read from L2 (no staging) and the full
// expansion lengths are used.
template <int GT_P, bool STAGE, bool YB, int NT, bool OWN = false>
__global__ void __launch_bounds__(NT, NT == 256 ? 2 : 1) k_gtrans_ws(GTrans T, const double2* __restrict__ X,
                                                      double2* __restrict__ Y) {
  extern __shared__ double2 gsm2[];
  const int s_in = T.s_in, s_out = T.s_out;
  const int kin = (s_in + 3) / 4, mout = (s_out + 7) / 8;
  const int ldx = gt_ld(kin * 4), ldt = gt_ld(T.rmax8);
  double2* Xs = gsm2;
  double2* const T0 = gsm2 + GT_P * ldx;  // T double buffer: T0 (even chunks), T0 + GT_P ldt (odd)
  // YB: the stage-2 output tile (GT_P columns of s_out), bulk-reduced into Y (one UBLKRED per column)
  double2* Ys = T0 + 2 * GT_P * ldt;
  double* Ms = reinterpret_cast<double*>(Ys + (YB ? GT_P * s_out : 0));
  __shared__ int sOut[3][GT_P], sIn[3][GT_P];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool grpA = warp < (NT / 64);  // stage-1 warps (and the gather); the rest run stage 2
  const int64_t item = T.item_order[blockIdx.x];
  const int64_t e_beg = T.item_ptr[item], e_end = T.item_ptr[item + 1];
  if (e_beg >= e_end) return;
  for (int i = tid; i < GT_P * ldx; i += NT) Xs[i] = make_double2(0.0, 0.0);
  // chunk list of the item: entries (groups) e, pairs [c, c + GT_P)
  auto advance = [&](int64_t& e, int64_t& c) {
    c += GT_P;
    if (c >= T.ig_pe[e]) {
      ++e;
      c = e < e_end ? T.ig_pb[e] : 0;
    }
  };
  auto load_idx = [&](int ib, int64_t e, int64_t c) {  // by warp 0
    if (tid < GT_P) {
      const int64_t p = c + tid;
      const bool v = p < T.ig_pe[e];
      sOut[ib][tid] = v ? T.out[p] : 0;
      sIn[ib][tid] = v ? T.in[p] : -1;
    }
  };
  // all groups of an atomic item are one group; stage its matrix once (all threads)
  const int grp0 = T.ig_group[e_beg];
  // the group's own expansion lengths (HF wedges shorter than the level's padded s; their tails are zero)
  const int kin_g = (T.gsi && !OWN) ? (T.gsi[grp0] + 3) / 4 : kin, mout_g = (T.gso && !OWN) ? (T.gso[grp0] + 7) / 8 : mout;
  const int xlen = min(4 * kin_g, s_in);
  auto issue_x = [&](int ib) {  // by the stage-1 warps
    for (int c = warp; c < GT_P; c += (NT / 64)) {
      const int src = sIn[ib][c];
      if (src < 0) continue;
      const double2* xs = X + (int64_t)src * s_in;
      for (int k = lane; k < xlen; k += 32) cp_async16(Xs + c * ldx + k, xs + k);
    }
    cp_async_commit();
  };
  if (STAGE) {
    const int rank = T.grank[grp0], rt = (rank + 7) / 8;
    const double* src = T.pool + T.gmat[grp0];
    const int nd = (rt * kin + mout * 2 * rt) * 64;
    for (int i = tid; i < nd / 2; i += NT) cp_async16(Ms + 2 * i, src + 2 * i);
    cp_async_commit();
  }
  int64_t ea = e_beg, ca = T.ig_pb[e_beg];  // chunk of the stage-1 warps (i)
  int64_t e1 = ea, c1 = ca;
  advance(e1, c1);
  load_idx(0, ea, ca);
  if (e1 < e_end) load_idx(1, e1, c1);
  cp_async_wait<0>();
  __syncthreads();
  if (grpA) issue_x(0);
  int64_t eb = -1, cb = 0;  // chunk of the stage-2 warps (i - 1); -1: none yet
  bool ypend = false;       // YB: a bulk reduction of Ys is in flight (issued by warp GT_W/2)
  int i = 0;
  while (ea < e_end || eb >= 0) {
    const int ia = i % 3, ibb = (i + 2) % 3;  // index buffers of chunks i and i - 1
    if (grpA && ea < e_end) {
      const int grp = T.ig_group[ea];
      const int rank = T.grank[grp], rt = (rank + 7) / 8;
      const double* Mg = STAGE ? Ms : T.pool + T.gmat[grp];
      cp_async_wait<0>();
      named_bar(1, (NT / 2));  // X of chunk i visible to the stage-1 warps
      // units = rt x (GT_P / 8 / ct1): a multiple of the NT / 64 stage-1 warps where possible
      const int ct1 = (NT == 256 && rt % 2 == 0 && GT_P >= 16) ? 2 : 1;
      gt_stage_ct<GT_P, 0, STAGE>(ct1, Mg, rt, kin_g, 1, Xs, ldx, T0 + (i & 1) * GT_P * ldt, ldt, nullptr, nullptr, 0,
                                  0, kin, 0, (NT / 64));
    }
    (void)ia;
    if (!grpA && eb >= 0) {
      // stage 2 of chunk i-1 on warps 4-7 (static units: letting the stage-1 warps claim stage-2 units
      // from a shared counter measured slower -- 312 vs 300 ms at config 5, more L2 traffic)
      const int grp = T.ig_group[eb];
      const int rank = T.grank[grp], rt = (rank + 7) / 8;
      const double* Mg = STAGE ? Ms : T.pool + T.gmat[grp];
      const double* U = Mg + (size_t)rt * kin * 64;
      const int kt2 = (rank + 3) / 4;
      const int nb = (int)min((int64_t)GT_P, T.ig_pe[eb] - cb);
      if (YB) {
        if (ypend && warp == (NT / 64)) bulk_wait_read();  // Ys of the previous chunk read by the bulk engine
        named_bar(2, (NT / 2));
        gt_stage_ct<GT_P, 3, STAGE>(T.ct2 > 0 ? T.ct2 : GT_P / 8, U, mout_g, kt2, 1, T0 + ((i + 1) & 1) * GT_P * ldt,
                                    ldt, Ys, s_out, nullptr, nullptr, s_out, nb, 2 * rt, (NT / 64), (NT / 64));
        fence_async_smem();
        named_bar(2, (NT / 2));
        if (warp == (NT / 64)) bulk_issue_cols(Y, Ys, sOut[ibb], s_out, nb, lane);
        ypend = true;
      } else {
        gt_stage_ct<GT_P, OWN ? 1 : 2, STAGE>(T.ct2 > 0 ? T.ct2 : GT_P / 8, U, mout_g, kt2, 1,
                                              T0 + ((i + 1) & 1) * GT_P * ldt, ldt, nullptr, 0, Y, sOut[ibb], s_out,
                                              nb, 2 * rt, (NT / 64), (NT / 64));
      }
    }
    __syncthreads();  // chunk i's T written, chunk i-1's outputs issued; X and index buffer ibb free
    // advance: stage 2 takes chunk i, stage 1 takes chunk i + 1
    eb = ea < e_end ? ea : -1, cb = ca;
    if (ea < e_end) advance(ea, ca);
    if (ea < e_end) {
      int64_t e2 = ea, c2 = ca;
      advance(e2, c2);
      if (grpA) issue_x((i + 1) % 3);             // indices of chunk i+1 were loaded a chunk ago
      if (e2 < e_end) load_idx((i + 2) % 3, e2, c2);  // buffer of chunk i-1 (done)
    }
    ++i;
  }
  if (YB && warp == (NT / 64)) bulk_wait_all();
}

static size_t gt_smem_ws(const GTrans& T, int p, bool stage, bool yb) {
  const int kin = (T.s_in + 3) / 4;
  return (size_t)(p * gt_ld(kin * 4) + 2 * p * gt_ld(T.rmax8) + (yb ? p * T.s_out : 0)) * sizeof(double2) +
         (stage ? (size_t)T.mmax * sizeof(double) : 0);
}
// bulk-reduced outputs (FDA_GT_BULK=1; default: per-lane FP64 atomics).  Measured at config 5 (round 2,
// FDA_TRACE per-level times): the TMA bulk reduction is slower than the REDG atomics on every level
// (LF M2L 151 vs 114 ms with the 16-column tile it needs for two CTAs per SM, 163 ms with 32 columns and
// one CTA per SM; HF levels +8%), so the reduction payload at L2, not the SM-side atomic issue, bounds
// the accumulation.
static bool gt_bulk() {
  static const bool on = getenv("FDA_GT_BULK") && getenv("FDA_GT_BULK")[0] == '1';
  return on;
}
static bool gt_yb(const GTrans& T) { return gt_bulk() && T.atomic && (T.s_out + 7) / 8 >= GT_W; }

// bulk-reduced outputs apply to atomic items whose output has >= GT_W row tiles (no k split)
static bool gt_yb(const GTrans& T);
static size_t gt_smem(const GTrans& T, int p, int nbuf, bool stage) {
  const int kin = (T.s_in + 3) / 4;
  return (size_t)(nbuf * p * gt_ld(kin * 4) + p * gt_ld(T.rmax8) + (gt_yb(T) ? p * T.s_out : 0)) * sizeof(double2) +
         (stage ? (size_t)T.mmax * sizeof(double) : 0);
}
// opt-in shared-memory limit per CTA of the current device (227 KB on B200)
static size_t smem_optin() {
  static size_t v = 0;
  if (!v) {
    int dev = 0, b = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&b, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || b <= 0) {
      cudaGetLastError();
      b = 227 * 1024;
    }
    v = (size_t)b;
  }
  return v;
}
// chunk width, buffering and matrix staging: the first candidate that keeps two CTAs per SM
// (FDA_GT_STAGE=0 disables staging); else the widest single-buffered chunk that fits one CTA per SM
// (large expansions at small eps: s_in ~ 1000 surface points); 8 columns as the last resort.
static void gt_cfg(const GTrans& T, int* p, int* nbuf, bool* stage) {
  static const bool allow = !(getenv("FDA_GT_STAGE") && getenv("FDA_GT_STAGE")[0] == '0');
  const int cand[6][3] = {{32, 1, 1}, {32, 2, 0}, {32, 1, 0}, {16, 1, 1}, {16, 2, 0}, {16, 1, 0}};
  static const size_t budget = getenv("FDA_GT_SMEM_KB") ? (size_t)atoi(getenv("FDA_GT_SMEM_KB")) * 1024
                                                         : (size_t)GT_SMEM_BUDGET;
  // FDA_GT_CFG=p,nbuf,stage (experiments): the first candidate at or after it in this list
  static const int force = [] {
    const char* f = getenv("FDA_GT_CFG");
    int a = 0, b = 0, c = 0;
    if (!f || sscanf(f, "%d,%d,%d", &a, &b, &c) != 3) return -1;
    const int cl[6][3] = {{32, 1, 1}, {32, 2, 0}, {32, 1, 0}, {16, 1, 1}, {16, 2, 0}, {16, 1, 0}};
    for (int i = 0; i < 6; ++i)
      if (cl[i][0] == a && cl[i][1] == b && cl[i][2] == c) return i;
    return -1;
  }();
  int ci = 0;
  for (auto& c : cand) {
    if (ci++ < force) continue;
    if (c[2] && !allow) continue;
    if (gt_smem(T, c[0], c[1], c[2]) <= budget) {
      *p = c[0], *nbuf = c[1], *stage = c[2];
      return;
    }
  }
  for (int pp : {32, 16})
    if (gt_smem(T, pp, 1, false) <= smem_optin()) {
      *p = pp, *nbuf = 1, *stage = false;
      return;
    }
  *p = 8, *nbuf = 1, *stage = false;
}
size_t smem_optin_bytes() { return smem_optin(); }
size_t gtrans_smem(const GTrans& T) {
  int p, nb;
  bool stg;
  gt_cfg(T, &p, &nb, &stg);
  return gt_smem(T, p, nb, stg);
}
bool gtrans_fits(const GTrans& T) { return T.n_items <= 0 || m2l_warp_fits(T) || gtrans_smem(T) <= smem_optin(); }
int gtrans_cols(const GTrans& T) {
  int p, nb;
  bool stg;
  gt_cfg(T, &p, &nb, &stg);
  return p;
}

template <int P, int NB, bool STG, bool YB>
static cudaError_t gt_launch_k(const GTrans& T, const double2* X, double2* Y, size_t sm, cudaStream_t st) {
  if (sm > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_gtrans<P, NB, STG, YB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  // One CTA per item (the hardware block scheduler keeps the resident items a compact window of the
  // Morton launch order).  FDA_GT_PERSIST=1: persistent CTAs streaming items b, b+G, ... -- measured
  // slower at config 5 (348 vs 336 ms: the CTAs drift apart in the item order and the L2 window grows).
  static const bool persist = getenv("FDA_GT_PERSIST") && getenv("FDA_GT_PERSIST")[0] == '1';
  int64_t grid = T.n_items;
  if (persist) {
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gtrans<P, NB, STG, YB>, GT_T, sm);
    grid = std::min<int64_t>(T.n_items, (int64_t)std::max(1, per_sm) * nsm);
  }
  k_gtrans<P, NB, STG, YB><<<(unsigned)grid, GT_T, sm, st>>>(T, X, Y);
  return cudaGetLastError();
}
template <int P, int NB, bool STG>
static cudaError_t gt_launch(const GTrans& T, const double2* X, double2* Y, size_t sm, cudaStream_t st) {
  return gt_yb(T) ? gt_launch_k<P, NB, STG, true>(T, X, Y, sm, st) : gt_launch_k<P, NB, STG, false>(T, X, Y, sm, st);
}

// largest pad8 rank for which the warp-specialised kernel fits the two-CTAs-per-SM budget: 32 columns with
// per-lane atomic outputs, 16 columns with the bulk output tile
int gtrans_ws_rmax(int s_in) {
  const int kin = (s_in + 3) / 4;
  const int p = gt_bulk() ? 16 : 32;
  int best = 0;
  for (int r8 = 8; r8 <= 512; r8 += 8)
    if ((size_t)(p * gt_ld(kin * 4) + 2 * p * gt_ld(r8) + (gt_bulk() ? p * s_in : 0)) * sizeof(double2) <=
        (size_t)GT_SMEM_BUDGET)
      best = r8;
  return best;
}

template <int P, bool STG, bool YB, int NT = 256, bool OWN = false>
static cudaError_t gt_launch_ws(const GTrans& T, const double2* X, double2* Y, size_t sm, cudaStream_t st) {
  if (sm > 48 * 1024) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_gtrans_ws<P, STG, YB, NT, OWN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  k_gtrans_ws<P, STG, YB, NT, OWN><<<(unsigned)T.n_items, NT, sm, st>>>(T, X, Y);
  return cudaGetLastError();
}

cudaError_t launch_gtrans(const GTrans& T, const double2* X, double2* Y, cudaStream_t st) {
  if (T.n_items <= 0) return cudaSuccess;
  static const bool sector_on = [] {
    const bool on = getenv("FDA_GT_SECTOR") && getenv("FDA_GT_SECTOR")[0] == '1';
    if (on) {
      const int one = 1;
      cudaMemcpyToSymbol(gt_sector_red, &one, sizeof(int));
    }
    return on;
  }();
  (void)sector_on;
  static const bool nored_on = [] {
    const int v = getenv("FDA_GT_NORED") ? atoi(getenv("FDA_GT_NORED")) : 0;
    if (v) cudaMemcpyToSymbol(gt_nored, &v, sizeof(int));
    return v != 0;
  }();
  (void)nored_on;
  // low-rank M2L items: warp-independent tasks with the operator in shared memory (m2l_warp.cu)
  if (m2l_warp_fits(T)) return launch_m2l_warp(T, X, Y, st);
  // warp-specialised kernel for all-low-rank atomic items (FDA_GT_WS=0 disables it)
  static const bool ws_ok = !(getenv("FDA_GT_WS") && getenv("FDA_GT_WS")[0] == '0');
  // owned low-rank items (FDA_GT_MODE=owned): the warp-specialised kernel with plain read-modify-write outputs
  if (ws_ok && !T.atomic && T.all_lowrank && gt_smem_ws(T, 32, false, false) <= GT_SMEM_BUDGET)
    return gt_launch_ws<32, false, false, 256, true>(T, X, Y, gt_smem_ws(T, 32, false, false), st);
  if (ws_ok && T.atomic && T.all_lowrank) {
    static const size_t budget = getenv("FDA_GT_SMEM_KB") ? (size_t)atoi(getenv("FDA_GT_SMEM_KB")) * 1024
                                                           : (size_t)GT_SMEM_BUDGET;
    // FDA_GT_WSP=32|16: chunk width of the warp-specialised kernel (default: the widest that keeps two CTAs
    // per SM; 32 columns with bulk outputs may take one CTA per SM with FDA_GT_WSP=32)
    static const int wsp = getenv("FDA_GT_WSP") ? atoi(getenv("FDA_GT_WSP")) : 0;
    const bool yb = gt_bulk();
    // FDA_GT_WS512=1: operators too large to stage next to two CTAs per SM run as one 512-thread CTA per SM
    // with the operator staged in shared memory.  Measured slower at config 5 (HF level 7: 42.5 vs 35.3 ms;
    // the LF level's operators do not fit even then), so off by default.
    static const bool ws512 = getenv("FDA_GT_WS512") && getenv("FDA_GT_WS512")[0] == '1';
    if (ws512 && !yb && !wsp && gt_smem_ws(T, 32, true, false) > budget &&
        gt_smem_ws(T, 32, true, false) <= smem_optin())
      return gt_launch_ws<32, true, false, 512>(T, X, Y, gt_smem_ws(T, 32, true, false), st);
    for (int p : {32, 16}) {
      if (wsp && p != wsp) continue;
      const size_t lim = wsp == p ? smem_optin() : budget;
      for (bool stg : {true, false}) {
        const size_t sm = gt_smem_ws(T, p, stg, yb);
        if (sm > lim) continue;
        if (p == 32 && stg) return yb ? gt_launch_ws<32, true, true>(T, X, Y, sm, st) : gt_launch_ws<32, true, false>(T, X, Y, sm, st);
        if (p == 32) return yb ? gt_launch_ws<32, false, true>(T, X, Y, sm, st) : gt_launch_ws<32, false, false>(T, X, Y, sm, st);
        if (stg) return yb ? gt_launch_ws<16, true, true>(T, X, Y, sm, st) : gt_launch_ws<16, true, false>(T, X, Y, sm, st);
        return yb ? gt_launch_ws<16, false, true>(T, X, Y, sm, st) : gt_launch_ws<16, false, false>(T, X, Y, sm, st);
      }
    }
  }
  int p, nb;
  bool stg;
  gt_cfg(T, &p, &nb, &stg);
  const size_t sm = gt_smem(T, p, nb, stg);
  if (p == 32 && nb == 1 && stg) return gt_launch<32, 1, true>(T, X, Y, sm, st);
  if (p == 32 && nb == 2) return gt_launch<32, 2, false>(T, X, Y, sm, st);
  if (p == 32) return gt_launch<32, 1, false>(T, X, Y, sm, st);
  if (p == 16 && stg) return gt_launch<16, 1, true>(T, X, Y, sm, st);
  if (p == 16 && nb == 2) return gt_launch<16, 2, false>(T, X, Y, sm, st);
  if (p == 16) return gt_launch<16, 1, false>(T, X, Y, sm, st);
  return gt_launch<8, 1, false>(T, X, Y, sm, st);
}

// ---------------------------------------------------------------- stored leaf S2M / L2T matrices
// "In the FDBEM, the S2M and L2T matrices are precomputed and saved in memory": per leaf,
//   S_leaf = (Sigma^-1 U^H) E_up  (s x n_leaf; eq_cmps x eq_evas2mh)   rows stored per source point: Sm[j][c]
//   T_leaf = E_dn (conj(U) Sigma^-1) (n_leaf x s; eq_eval2t x eq_cmpt) rows stored per target point: Tm[i][c]
// so the apply's S2M is x~[slot] = S_leaf q_leaf and its L2T out_i += T_leaf[i] y~[slot]: one HBM read of the
// matrices instead of the kernel evaluations on the check / equivalent surfaces.
#define LM_T 128
template <int KIND>
__global__ void __launch_bounds__(LM_T) k_leafmat_s2m(const int32_t* __restrict__ leaf_ids, const int64_t* __restrict__ pofs,
                                                      LeafGeom L, Points P, const double* __restrict__ surf, int nsurf,
                                                      double k, double2 alpha, const double2* __restrict__ Sred, int s,
                                                      double2* __restrict__ Sm) {
  extern __shared__ double2 e[];  // nsurf kernel values of one source point
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t pb = L.ptr[leaf], pe = L.ptr[leaf + 1];
  const double cx = L.cx[leaf], cy = L.cy[leaf], cz = L.cz[leaf];
  for (int64_t j = pb; j < pe; ++j) {
    const double yx = P.x[j], yy = P.y[j], yz = P.z[j], nyx = P.nx[j], nyy = P.ny[j], nyz = P.nz[j];
    __syncthreads();
    for (int a = threadIdx.x; a < nsurf; a += LM_T) {
      const double ax = cx + surf[3 * a], ay = cy + surf[3 * a + 1], az = cz + surf[3 * a + 2];
      e[a] = KIND == 0   ? dg_dny(ax - yx, ay - yy, az - yz, nyx, nyy, nyz, k)
             : KIND == 1 ? g_only(ax - yx, ay - yy, az - yz, k)
                         : bm_g(ax - yx, ay - yy, az - yz, -nyx, -nyy, -nyz, k, alpha);
    }
    __syncthreads();
    double2* row = Sm + (pofs[blockIdx.x] + (j - pb)) * s;
    for (int c = threadIdx.x; c < s; c += LM_T) {  // Sred column-major s x nsurf
      double2 acc = make_double2(0.0, 0.0);
      for (int a = 0; a < nsurf; ++a) cfma(acc, Sred[c + (int64_t)a * s], e[a]);
      row[c] = acc;
    }
  }
}
__global__ void __launch_bounds__(LM_T) k_leafmat_l2t(const int32_t* __restrict__ leaf_ids, const int64_t* __restrict__ pofs,
                                                      LeafGeom L, Points P, const double* __restrict__ surf, int nsurf,
                                                      double k, double2 alpha, const double2* __restrict__ TredT, int s,
                                                      double2* __restrict__ Tm) {
  extern __shared__ double2 e[];  // nsurf kernel values of one target point
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t pb = L.ptr[leaf], pe = L.ptr[leaf + 1];
  const double cx = L.cx[leaf], cy = L.cy[leaf], cz = L.cz[leaf];
  for (int64_t i = pb; i < pe; ++i) {
    const double xi = P.x[i] - cx, yi = P.y[i] - cy, zi = P.z[i] - cz, nxi = P.nx[i], nyi = P.ny[i], nzi = P.nz[i];
    __syncthreads();
    for (int b = threadIdx.x; b < nsurf; b += LM_T)
      e[b] = bm_g(xi - surf[3 * b], yi - surf[3 * b + 1], zi - surf[3 * b + 2], nxi, nyi, nzi, k, alpha);
    __syncthreads();
    double2* row = Tm + (pofs[blockIdx.x] + (i - pb)) * s;
    for (int c = threadIdx.x; c < s; c += LM_T) {  // TredT row-major nsurf x s (the transpose of T's storage)
      double2 acc = make_double2(0.0, 0.0);
      for (int b = 0; b < nsurf; ++b) cfma(acc, e[b], TredT[(int64_t)b * s + c]);
      row[c] = acc;
    }
  }
}
void launch_leafmat(int kind, int64_t nleaves, const int32_t* leaf_ids, const int64_t* pofs, LeafGeom L, Points P,
                    const double* surf, int nsurf, double k, double2 alpha, double2 alpha_dn, const double2* Sred,
                    const double2* TredT, int s, double2* Sm, double2* Tm, cudaStream_t st) {
  if (nleaves <= 0) return;
  const size_t sm = (size_t)nsurf * sizeof(double2);
  if (kind == 0)
    k_leafmat_s2m<0><<<(unsigned)nleaves, LM_T, sm, st>>>(leaf_ids, pofs, L, P, surf, nsurf, k, alpha, Sred, s, Sm);
  else if (kind == 1)
    k_leafmat_s2m<1><<<(unsigned)nleaves, LM_T, sm, st>>>(leaf_ids, pofs, L, P, surf, nsurf, k, alpha, Sred, s, Sm);
  else
    k_leafmat_s2m<2><<<(unsigned)nleaves, LM_T, sm, st>>>(leaf_ids, pofs, L, P, surf, nsurf, k, alpha, Sred, s, Sm);
  k_leafmat_l2t<<<(unsigned)nleaves, LM_T, sm, st>>>(leaf_ids, pofs, L, P, surf, nsurf, k, alpha_dn, TredT, s, Tm);
}

// apply: x~[slot] = sum_j Sm[j] q_j (threads over the expansion index; each row read once, coalesced)
__global__ void __launch_bounds__(LM_T) k_leaf_s2m(const int32_t* __restrict__ leaf_ids, const int64_t* __restrict__ pofs,
                                                   const int32_t* __restrict__ slot, const int64_t* __restrict__ lptr,
                                                   const double2* __restrict__ q, const double2* __restrict__ Sm, int s,
                                                   double2* __restrict__ X) {
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t pb = lptr[leaf], pe = lptr[leaf + 1];
  const double2* rows = Sm + pofs[blockIdx.x] * s;
  double2* x = X + (int64_t)slot[blockIdx.x] * s;
  for (int c = threadIdx.x; c < s; c += LM_T) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t j = pb; j < pe; ++j) cfma(acc, __ldg(rows + (j - pb) * s + c), __ldg(q + j));
    x[c] = acc;
  }
}
// apply: out_i += Tm[i] . y~[slot] (a warp per target point, lanes along the expansion, shuffle reduction)
__global__ void __launch_bounds__(LM_T) k_leaf_l2t(const int32_t* __restrict__ leaf_ids, const int64_t* __restrict__ pofs,
                                                   const int32_t* __restrict__ slot, const int64_t* __restrict__ lptr,
                                                   const double2* __restrict__ Y, const double2* __restrict__ Tm, int s,
                                                   double2* __restrict__ outm) {
  extern __shared__ double2 y[];
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t pb = lptr[leaf], pe = lptr[leaf + 1];
  const double2* yl = Y + (int64_t)slot[blockIdx.x] * s;
  for (int c = threadIdx.x; c < s; c += LM_T) y[c] = yl[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2* rows = Tm + pofs[blockIdx.x] * s;
  for (int64_t i = pb + warp; i < pe; i += LM_T / 32) {
    const double2* r = rows + (i - pb) * s;
    double2 acc = make_double2(0.0, 0.0);
    for (int c = lane; c < s; c += 32) cfma(acc, __ldg(r + c), y[c]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) outm[i] = cadd(outm[i], acc);
  }
}
void launch_leaf_s2m(int64_t nleaves, const int32_t* leaf_ids, const int64_t* pofs, const int32_t* slot,
                     const int64_t* lptr, const double2* q, const double2* Sm, int s, double2* X, cudaStream_t st) {
  if (nleaves <= 0) return;
  k_leaf_s2m<<<(unsigned)nleaves, LM_T, 0, st>>>(leaf_ids, pofs, slot, lptr, q, Sm, s, X);
}
void launch_leaf_l2t(int64_t nleaves, const int32_t* leaf_ids, const int64_t* pofs, const int32_t* slot,
                     const int64_t* lptr, const double2* Y, const double2* Tm, int s, double2* outm, cudaStream_t st) {
  if (nleaves <= 0) return;
  k_leaf_l2t<<<(unsigned)nleaves, LM_T, (size_t)s * sizeof(double2), st>>>(leaf_ids, pofs, slot, lptr, Y, Tm, s, outm);
}

// ---------------------------------------------------------------- H8 L2T
// out_i += sum_b [G(x_i, b) + alpha dG/dn_x(x_i, b)] rho[leaf][b] over the leaf's incoming equivalent
// surface (E_dn of eq_eval2t).  rho = conj(U) Sigma^-1 y~ (eq_cmpt) comes from the
// grouped-translation kernel.
#define L2T_T 128
__global__ void __launch_bounds__(L2T_T) k_l2t_eval(const int32_t* __restrict__ leaf_ids, LeafGeom L, Points P,
                                                    const double* __restrict__ surf, int nsurf, double k,
                                                    double2 alpha, const double2* __restrict__ rhoall,
                                                    double2* __restrict__ outm) {
  extern __shared__ double2 rho[];  // nsurf (+ 3 nsurf doubles of surface points)
  double* sp = reinterpret_cast<double*>(rho + nsurf);
  __shared__ double2 red[L2T_T];
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t pb = L.ptr[leaf], pe = L.ptr[leaf + 1];
  const double cx = L.cx[leaf], cy = L.cy[leaf], cz = L.cz[leaf];
  const double2* rl = rhoall + (int64_t)blockIdx.x * nsurf;
  for (int i = threadIdx.x; i < nsurf; i += L2T_T) rho[i] = rl[i];
  for (int i = threadIdx.x; i < 3 * nsurf; i += L2T_T) sp[i] = surf[i];
  __syncthreads();
  const int nt = (int)(pe - pb);
  const int ntp = nt >= L2T_T ? L2T_T : next_pow2(nt);
  const int nsl = L2T_T / ntp;
  const int my_t = threadIdx.x % ntp, my_sl = threadIdx.x / ntp;
  for (int t0 = 0; t0 < nt; t0 += ntp) {
    const int64_t i = pb + t0 + my_t;
    const bool act = (t0 + my_t) < nt;
    double2 acc = make_double2(0.0, 0.0);
    if (act) {
      const double xi = P.x[i] - cx, yi = P.y[i] - cy, zi = P.z[i] - cz;
      const double nxi = P.nx[i], nyi = P.ny[i], nzi = P.nz[i];
      for (int b = my_sl; b < nsurf; b += nsl)
        cfma(acc, bm_g(xi - sp[3 * b], yi - sp[3 * b + 1], zi - sp[3 * b + 2], nxi, nyi, nzi, k, alpha), rho[b]);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (my_sl == 0 && act) {
      double2 sum = red[my_t];
      for (int sl = 1; sl < nsl; ++sl) sum = cadd(sum, red[my_t + sl * ntp]);
      outm[i] = cadd(outm[i], sum);
    }
    __syncthreads();
  }
}
void launch_l2t_eval(int64_t nleaves, const int32_t* leaf_ids, LeafGeom L, Points P, const double* surf, int nsurf,
                     double k, double2 alpha, const double2* rho, double2* outm, cudaStream_t st) {
  if (nleaves <= 0) return;
  k_l2t_eval<<<(unsigned)nleaves, L2T_T, nsurf * (sizeof(double2) + 3 * sizeof(double)), st>>>(
      leaf_ids, L, P, surf, nsurf, k, alpha, rho, outm);
}

}  // namespace fda
