// kernels.cu -- device kernels of the FDA Burton-Miller apply.  See kernels.cuh.
#include "kernels.cuh"

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

// ---------------------------------------------------------------- H2 P2P near field
#define P2P_T 128
#define P2P_MAXL 256
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
            const double2 kv = bm_h(xi - sx[u], yi - sy[u], zi - sz[u], nxi, nyi, nzi, snx[u], sny[u], snz[u], k, alpha);
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
void launch_p2p(int64_t nleaf, const int64_t* leaf_ptr, const int64_t* p2p_ptr, const int32_t* p2p_src, Points P,
                const double2* q, double k, double2 alpha, double2* outm, int64_t leaf0, cudaStream_t st) {
  if (nleaf <= 0) return;
  k_p2p<<<(unsigned)nleaf, P2P_T, 0, st>>>(leaf_ptr, p2p_ptr, p2p_src, P, q, k, alpha, outm, leaf0);
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

// ---------------------------------------------------------------- H4 S2M (dipole check potentials + reduction)
#define S2M_T 128
#define S2M_MAXC 4
__global__ void __launch_bounds__(S2M_T) k_s2m(const int32_t* __restrict__ leaf_ids, const int32_t* __restrict__ slots,
                                               LeafGeom L, Points P, const double2* __restrict__ q,
                                               const double* __restrict__ surf, int nsurf, const double2* __restrict__ S,
                                               int s, double k, double2* __restrict__ X) {
  extern __shared__ double2 chk[];  // nsurf
  __shared__ double sx[S2M_T], sy[S2M_T], sz[S2M_T], snx[S2M_T], sny[S2M_T], snz[S2M_T];
  __shared__ double2 sq[S2M_T];
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t slot = slots[blockIdx.x];
  const int64_t pb = L.ptr[leaf], pe = L.ptr[leaf + 1];
  const double cx = L.cx[leaf], cy = L.cy[leaf], cz = L.cz[leaf];
  double ax[S2M_MAXC], ay[S2M_MAXC], az[S2M_MAXC];
  double2 acc[S2M_MAXC];
#pragma unroll
  for (int c = 0; c < S2M_MAXC; ++c) {
    const int i = threadIdx.x + c * S2M_T;
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
      const int i = threadIdx.x + c * S2M_T;
      if (i >= nsurf) break;
      for (int u = 0; u < cnt; ++u)
        cfma(acc[c], dg_dny(ax[c] - sx[u], ay[c] - sy[u], az[c] - sz[u], snx[u], sny[u], snz[u], k), sq[u]);
    }
  }
#pragma unroll
  for (int c = 0; c < S2M_MAXC; ++c) {
    const int i = threadIdx.x + c * S2M_T;
    if (i < nsurf) chk[i] = acc[c];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < s; r += S2M_T) {
    double2 x = make_double2(0.0, 0.0);
    for (int i = 0; i < nsurf; ++i) cfma(x, S[r + (int64_t)i * s], chk[i]);
    X[slot * s + r] = x;
  }
}
void launch_s2m(int64_t nleaves, const int32_t* leaf_ids, const int32_t* slots, LeafGeom L, Points P,
                const double2* q, const double* surf, int nsurf, const double2* S, int s, double k, double2* X,
                cudaStream_t st) {
  if (nleaves <= 0) return;
  k_s2m<<<(unsigned)nleaves, S2M_T, nsurf * sizeof(double2), st>>>(leaf_ids, slots, L, P, q, surf, nsurf, S, s, k, X);
}

// ---------------------------------------------------------------- H5 M2M / H7 L2L
__global__ void k_m2m(const int64_t* __restrict__ up_ptr, const int32_t* __restrict__ up_child,
                      const int32_t* __restrict__ up_mat, const double2* __restrict__ pool, int sp, int sc,
                      const double2* __restrict__ Xc, double2* __restrict__ Xp) {
  extern __shared__ double2 xs[];
  const int64_t slot = blockIdx.x;
  const int i = threadIdx.x;
  // a leaf's slot has no children: its expansion came from S2M, leave it alone
  if (up_ptr[slot] == up_ptr[slot + 1]) return;
  double2 acc = make_double2(0.0, 0.0);
  const int64_t msz = (int64_t)sp * sc;
  for (int64_t e = up_ptr[slot]; e < up_ptr[slot + 1]; ++e) {
    const int64_t c = up_child[e];
    const double2* M = pool + up_mat[e] * msz;
    __syncthreads();
    for (int j = threadIdx.x; j < sc; j += blockDim.x) xs[j] = Xc[c * sc + j];
    __syncthreads();
    if (i < sp)
      for (int j = 0; j < sc; ++j) cfma(acc, M[i + (int64_t)j * sp], xs[j]);
  }
  if (i < sp) Xp[slot * sp + i] = acc;
}
void launch_m2m(int64_t nparent, const int64_t* up_ptr, const int32_t* up_child, const int32_t* up_mat,
                const double2* pool, int sp, int sc, const double2* Xc, double2* Xp, cudaStream_t st) {
  if (nparent <= 0) return;
  const int th = ((sp + 31) / 32) * 32;
  k_m2m<<<(unsigned)nparent, th, sc * sizeof(double2), st>>>(up_ptr, up_child, up_mat, pool, sp, sc, Xc, Xp);
}

__global__ void k_l2l(const int64_t* __restrict__ dn_ptr, const int32_t* __restrict__ dn_parent,
                      const int32_t* __restrict__ dn_mat, const double2* __restrict__ poolT, int sp, int sc,
                      const double2* __restrict__ Yp, double2* __restrict__ Yc) {
  extern __shared__ double2 ys[];
  const int64_t slot = blockIdx.x;
  const int j = threadIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  const int64_t msz = (int64_t)sp * sc;
  for (int64_t e = dn_ptr[slot]; e < dn_ptr[slot + 1]; ++e) {
    const int64_t p = dn_parent[e];
    const double2* M = poolT + dn_mat[e] * msz;  // sc x sp column-major (= M~^T)
    __syncthreads();
    for (int i = threadIdx.x; i < sp; i += blockDim.x) ys[i] = Yp[p * sp + i];
    __syncthreads();
    if (j < sc)
      for (int i = 0; i < sp; ++i) cfma(acc, M[j + (int64_t)i * sc], ys[i]);
  }
  if (j < sc) Yc[slot * sc + j] = cadd(Yc[slot * sc + j], acc);
}
void launch_l2l(int64_t nchild, const int64_t* dn_ptr, const int32_t* dn_parent, const int32_t* dn_mat,
                const double2* poolT, int sp, int sc, const double2* Yp, double2* Yc, cudaStream_t st) {
  if (nchild <= 0) return;
  const int th = ((sc + 31) / 32) * 32;
  k_l2l<<<(unsigned)nchild, th, sp * sizeof(double2), st>>>(dn_ptr, dn_parent, dn_mat, poolT, sp, sc, Yp, Yc);
}

// ---------------------------------------------------------------- H6 M2L (group = one offset)
#define M2L_PB 8
__global__ void k_m2l(const int64_t* __restrict__ gbeg, const int64_t* __restrict__ gend,
                      const int32_t* __restrict__ grank, const int64_t* __restrict__ gmat,
                      const int32_t* __restrict__ tgt, const int32_t* __restrict__ src,
                      const double2* __restrict__ pool, int s, const double2* __restrict__ X, double2* __restrict__ Y) {
  extern __shared__ double2 sm[];
  double2* xs = sm;                 // PB x s
  double2* ts = sm + M2L_PB * s;    // PB x s (low-rank intermediate)
  const int64_t g = blockIdx.x;
  const int rank = grank[g];
  const double2* M = pool + gmat[g];
  const int i = threadIdx.x;
  for (int64_t p0 = gbeg[g]; p0 < gend[g]; p0 += M2L_PB) {
    const int np = (int)min((int64_t)M2L_PB, gend[g] - p0);
    __syncthreads();
    for (int e = threadIdx.x; e < np * s; e += blockDim.x) {
      const int pp = e / s, j = e % s;
      xs[pp * s + j] = X[(int64_t)src[p0 + pp] * s + j];
    }
    __syncthreads();
    double2 y[M2L_PB];
#pragma unroll
    for (int pp = 0; pp < M2L_PB; ++pp) y[pp] = make_double2(0.0, 0.0);
    if (rank < 0) {
      if (i < s) {
        for (int j = 0; j < s; ++j) {
          const double2 m = M[i + (int64_t)j * s];
#pragma unroll
          for (int pp = 0; pp < M2L_PB; ++pp) cfma(y[pp], m, xs[pp * s + j]);
        }
      }
    } else {
      const double2* U = M;                      // s x rank
      const double2* Vh = M + (int64_t)s * rank; // rank x s
      if (i < rank) {
        double2 t[M2L_PB];
#pragma unroll
        for (int pp = 0; pp < M2L_PB; ++pp) t[pp] = make_double2(0.0, 0.0);
        for (int j = 0; j < s; ++j) {
          const double2 m = Vh[i + (int64_t)j * rank];
#pragma unroll
          for (int pp = 0; pp < M2L_PB; ++pp) cfma(t[pp], m, xs[pp * s + j]);
        }
#pragma unroll
        for (int pp = 0; pp < M2L_PB; ++pp) ts[pp * s + i] = t[pp];
      }
      __syncthreads();
      if (i < s) {
        for (int c = 0; c < rank; ++c) {
          const double2 m = U[i + (int64_t)c * s];
#pragma unroll
          for (int pp = 0; pp < M2L_PB; ++pp) cfma(y[pp], m, ts[pp * s + c]);
        }
      }
    }
    if (i < s) {
      for (int pp = 0; pp < np; ++pp) {
        double* dst = reinterpret_cast<double*>(Y + (int64_t)tgt[p0 + pp] * s + i);
        atomicAdd(dst, y[pp].x);
        atomicAdd(dst + 1, y[pp].y);
      }
    }
  }
}
void launch_m2l(int64_t ngroups, const int64_t* gbeg, const int64_t* gend, const int32_t* grank, const int64_t* gmat,
                const int32_t* tgt, const int32_t* src, const double2* pool, int s, const double2* X, double2* Y,
                cudaStream_t st) {
  if (ngroups <= 0) return;
  const int th = ((s + 31) / 32) * 32;
  const size_t sm = 2 * M2L_PB * s * sizeof(double2);
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_m2l, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_m2l<<<(unsigned)ngroups, th, sm, st>>>(gbeg, gend, grank, gmat, tgt, src, pool, s, X, Y);
}

// ---------------------------------------------------------------- grouped translation (H5/H6/H7)
// Register-tiled complex FP64 GEMM on 128 threads: output tile TM rows x GT_NB pair columns,
// each thread RM rows x RN columns; A streamed from global through shared memory in
// GT_KC-deep slices, B (the gathered input vectors) resident in shared memory.
#define GT_T 128
#define GT_NB 16
#define GT_NBP (GT_NB + 1)   // padded column stride of the shared B / T tiles (bank spread)
#define GT_KC 16

template <int TM, int TX, int RM, int RN>
__device__ __forceinline__ void gt_tile(const double2* __restrict__ A, int64_t lda, int row0, int M, int K,
                                        const double2* Bs, double2* As, double2 (&acc)[RM][RN]) {
  const int tid = threadIdx.x, ty = tid / TX, tx = tid % TX;
#pragma unroll
  for (int r = 0; r < RM; ++r)
#pragma unroll
    for (int c = 0; c < RN; ++c) acc[r][c] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < K; k0 += GT_KC) {
    __syncthreads();
    for (int e = tid; e < GT_KC * TM; e += GT_T) {
      const int kk = e / TM, i = e % TM;
      const int row = row0 + i, k = k0 + kk;
      As[e] = (row < M && k < K) ? __ldg(&A[row + (int64_t)k * lda]) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int kmax = min(GT_KC, K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      double2 a[RM], b[RN];
#pragma unroll
      for (int r = 0; r < RM; ++r) a[r] = As[kk * TM + ty * RM + r];
#pragma unroll
      for (int c = 0; c < RN; ++c) b[c] = Bs[(k0 + kk) * GT_NBP + tx * RN + c];
#pragma unroll
      for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int c = 0; c < RN; ++c) cfma(acc[r][c], a[r], b[c]);
    }
  }
}

__global__ void __launch_bounds__(GT_T) k_gtrans(GTrans T, const double2* __restrict__ X, double2* __restrict__ Y) {
  extern __shared__ double2 gsm[];
  const int s_in = T.s_in, s_out = T.s_out;
  double2* Xs = gsm;                              // s_in x NBP
  double2* Ts = Xs + (size_t)s_in * GT_NBP;       // rmax x NBP
  double2* As = Ts + (size_t)T.rmax * GT_NBP;     // KC x 64
  __shared__ int sOut[GT_NB];
  const int tid = threadIdx.x;
  const int64_t item = T.item_order[blockIdx.x];
  for (int64_t e = T.item_ptr[item]; e < T.item_ptr[item + 1]; ++e) {
    const int g = T.ig_group[e];
    const int rank = T.grank[g];
    const double2* Mg = T.pool + T.gmat[g];
    const int64_t pe = T.ig_pe[e];
    for (int64_t c0 = T.ig_pb[e]; c0 < pe; c0 += GT_NB) {
      const int nb = (int)min((int64_t)GT_NB, pe - c0);
      __syncthreads();
      if (tid < GT_NB) sOut[tid] = tid < nb ? T.out[c0 + tid] : -1;
      for (int idx = tid; idx < s_in * GT_NB; idx += GT_T) {
        const int c = idx / s_in, k = idx - c * s_in;
        Xs[k * GT_NBP + c] = c < nb ? X[(int64_t)T.in[c0 + c] * s_in + k] : make_double2(0.0, 0.0);
      }
      __syncthreads();
      const double2* Bs = Xs;
      const double2* U = Mg;
      int kin = s_in;
      if (rank >= 0) {
        // stage 1: T = Vh (r x s_in) X
        const double2* Vh = Mg + (int64_t)s_out * rank;
        for (int row0 = 0; row0 < rank; row0 += 32) {
          double2 acc[4][1];
          gt_tile<32, 16, 4, 1>(Vh, rank, row0, rank, s_in, Xs, As, acc);
          const int ty = tid / 16, tx = tid % 16;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = row0 + ty * 4 + r;
            if (row < rank) Ts[row * GT_NBP + tx] = acc[r][0];
          }
        }
        __syncthreads();
        Bs = Ts;
        kin = rank;
      }
      // stage 2 (or dense): Y += A (s_out x kin) B
      for (int row0 = 0; row0 < s_out; row0 += 64) {
        double2 acc[4][2];
        gt_tile<64, 8, 4, 2>(U, s_out, row0, s_out, kin, Bs, As, acc);
        const int ty = tid / 8, tx = tid % 8;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int col = tx * 2 + c;
          if (col >= nb) continue;
          double2* y = Y + (int64_t)sOut[col] * s_out;
          if (T.atomic) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = row0 + ty * 4 + r;
              if (row < s_out) {
                atomicAdd(&y[row].x, acc[r][c].x);
                atomicAdd(&y[row].y, acc[r][c].y);
              }
            }
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int row = row0 + ty * 4 + r;
              if (row < s_out) y[row] = cadd(y[row], acc[r][c]);
            }
          }
        }
      }
    }
  }
}
void launch_gtrans(const GTrans& T, const double2* X, double2* Y, cudaStream_t st) {
  if (T.n_items <= 0) return;
  const size_t sm = ((size_t)T.s_in * GT_NBP + (size_t)T.rmax * GT_NBP + (size_t)GT_KC * 64) * sizeof(double2);
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_gtrans, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_gtrans<<<(unsigned)T.n_items, GT_T, sm, st>>>(T, X, Y);
}

// ---------------------------------------------------------------- H8 L2T
#define L2T_T 128
__global__ void __launch_bounds__(L2T_T) k_l2t(const int32_t* __restrict__ leaf_ids, const int32_t* __restrict__ slots,
                                               LeafGeom L, Points P, const double* __restrict__ surf, int nsurf,
                                               const double2* __restrict__ T, int s, double k, double2 alpha,
                                               const double2* __restrict__ Y, double2* __restrict__ outm) {
  extern __shared__ double2 rho[];  // nsurf
  __shared__ double2 red[L2T_T];
  const int64_t leaf = leaf_ids[blockIdx.x];
  const int64_t slot = slots[blockIdx.x];
  const int64_t pb = L.ptr[leaf], pe = L.ptr[leaf + 1];
  const double cx = L.cx[leaf], cy = L.cy[leaf], cz = L.cz[leaf];
  const double2* y = Y + slot * s;
  for (int i = threadIdx.x; i < nsurf; i += L2T_T) {
    double2 v = make_double2(0.0, 0.0);
    for (int r = 0; r < s; ++r) cfma(v, T[i + (int64_t)r * nsurf], y[r]);
    rho[i] = v;
  }
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
        cfma(acc, bm_g(xi - surf[3 * b], yi - surf[3 * b + 1], zi - surf[3 * b + 2], nxi, nyi, nzi, k, alpha), rho[b]);
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
void launch_l2t(int64_t nleaves, const int32_t* leaf_ids, const int32_t* slots, LeafGeom L, Points P,
                const double* surf, int nsurf, const double2* T, int s, double k, double2 alpha, const double2* Y,
                double2* outm, cudaStream_t st) {
  if (nleaves <= 0) return;
  k_l2t<<<(unsigned)nleaves, L2T_T, nsurf * sizeof(double2), st>>>(leaf_ids, slots, L, P, surf, nsurf, T, s, k, alpha,
                                                                   Y, outm);
}

}  // namespace fda
