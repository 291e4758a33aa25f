#include <cstdio>
#include <cstdlib>
// plan_dev.cu -- device builders of the translation operators.  See plan_dev.cuh.
#include "plan_dev.cuh"

#include <algorithm>
#include <vector>

namespace fda {

#define PD_INV4PI 0.079577471545947667884
#define OP_T 256
#define OP_W (OP_T / 32)

__device__ __forceinline__ double2 pd_g(double k, double dx, double dy, double dz) {
  const double r = sqrt(dx * dx + dy * dy + dz * dz);
  double s, c;
  sincos(k * r, &s, &c);
  const double f = PD_INV4PI / r;
  return make_double2(c * f, s * f);
}
__device__ __forceinline__ void pd_fma(double2& acc, double2 a, double2 b) {  // acc += a b
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ void pd_fmac(double2& acc, double2 a, double2 b) {  // acc += conj(a) b
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
}
__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Write an M x K operator a(i, j) (zero outside [0, Mr) x [0, Kr)) in the DMMA fragment order of
// kernels.cuh GTrans, padded to Mp x Kp: tiles (mt, kt) of 8 x 4, row-tile-major, each 32 real parts in
// lane order (lane -> row mt*8 + lane/4, col kt*4 + lane%4) then 32 imaginary parts.
template <class F>
__device__ void frag_write(double* dst, int Mr, int Kr, int Mp, int Kp, F a) {
  const int kt_n = Kp / 4, ntile = (Mp / 8) * kt_n;
  for (int e = threadIdx.x; e < ntile * 32; e += blockDim.x) {
    const int tile = e >> 5, l = e & 31;
    const int i = (tile / kt_n) * 8 + (l >> 2), j = (tile % kt_n) * 4 + (l & 3);
    const double2 v = (i < Mr && j < Kr) ? a(i, j) : make_double2(0.0, 0.0);
    dst[(int64_t)tile * 64 + l] = v.x;
    dst[(int64_t)tile * 64 + 32 + l] = v.y;
  }
}
__host__ __device__ __forceinline__ int pd_pad8(int v) { return (v + 7) / 8 * 8; }
__host__ __device__ __forceinline__ int pd_pad4(int v) { return (v + 3) / 4 * 4; }

// Block-wide argmax of val[j] over j < n with flag[j] == 0 (first index on ties); result in *bv, *bj.
__device__ void block_argmax(const double* val, const unsigned char* flag, int n, double* red_v, int* red_j, double* bv,
                             int* bj) {
  double v = -1.0;
  int jj = -1;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    if (!flag[j] && val[j] > v) v = val[j], jj = j;
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, jj, o);
    if (v2 > v || (v2 == v && j2 >= 0 && (jj < 0 || j2 < jj))) v = v2, jj = j2;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red_v[w] = v, red_j[w] = jj;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bvv = -1.0;
    int bjj = -1;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
      if (red_v[i] > bvv || (red_v[i] == bvv && red_j[i] >= 0 && (bjj < 0 || red_j[i] < bjj))) bvv = red_v[i], bjj = red_j[i];
    *bv = bvv, *bj = bjj;
  }
  __syncthreads();
}

// One CTA per operator (grid-stride).  Workspace per CTA: G (maxn^2), T (maxn maxs), O, Q, W, V, U (maxs^2 each).
__global__ void __launch_bounds__(OP_T) k_opjob(OpJob J, int pass, double2* ws, size_t ws_per) {
  extern __shared__ double pd_sm[];
  double* nrm = pd_sm;                                                  // maxs
  double* sig = nrm + J.maxs;                                           // maxs
  int* piv = reinterpret_cast<int*>(sig + J.maxs);                      // maxs
  int* sel = piv + J.maxs;                                              // maxs
  unsigned char* used = reinterpret_cast<unsigned char*>(sel + J.maxs);  // maxs
  __shared__ double red_v[OP_W];
  __shared__ int red_j[OP_W];
  __shared__ double s_best;
  __shared__ int s_jb, s_rot, s_np, s_rank;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int maxn = J.maxn, maxs = J.maxs;
  double2* Gk = ws + (size_t)blockIdx.x * ws_per;
  double2* T = Gk + (size_t)maxn * maxn;
  double2* O = T + (size_t)maxn * maxs;
  double2* Q = O + (size_t)maxs * maxs;
  double2* W = Q + (size_t)maxs * maxs;
  double2* V = W + (size_t)maxs * maxs;
  double2* U = V + (size_t)maxs * maxs;
  for (int it = blockIdx.x; it < J.n_items; it += gridDim.x) {
    const DevSet A = J.sets[J.a[it]], B = J.sets[J.b[it]];
    const double sx = J.shift[3 * it], sy = J.shift[3 * it + 1], sz = J.shift[3 * it + 2];
    const int nA = A.n, nB = B.n, sA = A.s, sB = B.s;
    // G(P_A - Q_B + shift)
    for (int e = tid; e < nA * nB; e += OP_T) {
      const int i = e % nA, j = e / nA;
      Gk[e] = pd_g(J.k, A.pts[3 * i] - B.pts[3 * j] + sx, A.pts[3 * i + 1] - B.pts[3 * j + 1] + sy,
                   A.pts[3 * i + 2] - B.pts[3 * j + 2] + sz);
    }
    __syncthreads();
    // T = G Rf_B (nA x sB)
    for (int e = tid; e < nA * sB; e += OP_T) {
      const int i = e % nA, c = e / nA;
      double2 acc = make_double2(0.0, 0.0);
      const double2* rb = B.Rf + (size_t)c * nB;
      for (int j = 0; j < nB; ++j) pd_fma(acc, Gk[i + (size_t)j * nA], rb[j]);
      T[e] = acc;
    }
    __syncthreads();
    // O = Lf_A T (sA x sB)
    for (int e = tid; e < sA * sB; e += OP_T) {
      const int a = e % sA, c = e / sA;
      double2 acc = make_double2(0.0, 0.0);
      for (int i = 0; i < nA; ++i) pd_fma(acc, A.Lf[a + (size_t)i * sA], T[i + (size_t)c * nA]);
      O[e] = acc;
    }
    __syncthreads();
    int rank = -1, np_ = 0;
    if (J.compress) {
      // the MGS works on a copy C of O (in the G workspace, free once T is built): O stays K~ for a dense group
      double2* C = Gk;
      for (int e = tid; e < sA * sB; e += OP_T) C[e] = O[e];
      __syncthreads();
      // ---- pivoted MGS (re-orthogonalised) of O's columns, tol 0.1 eps_lr of the largest column norm
      for (int j = warp; j < sB; j += OP_W) {
        double s = 0;
        for (int a = lane; a < sA; a += 32) s += C[a + (size_t)j * sA].x * C[a + (size_t)j * sA].x +
                                                  C[a + (size_t)j * sA].y * C[a + (size_t)j * sA].y;
        s = wsum(s);
        if (lane == 0) nrm[j] = s;
      }
      for (int j = tid; j < sB; j += OP_T) used[j] = 0;
      __syncthreads();
      block_argmax(nrm, used, sB, red_v, red_j, &s_best, &s_jb);
      const double n0 = sqrt(fmax(s_best, 0.0)), tol = 0.1 * J.eps_lr;
      const int rmax = min(sA, sB);
      int t = 0;
      for (; t < rmax; ++t) {
        if (t > 0) block_argmax(nrm, used, sB, red_v, red_j, &s_best, &s_jb);
        const int jb = s_jb;
        if (jb < 0 || s_best <= 0.0 || sqrt(s_best) <= tol * n0) break;
        // q = a_jb / |a_jb|  (warp 0), stored as column t of Q
        if (warp == 0) {
          double s = 0;
          for (int a = lane; a < sA; a += 32) {
            const double2 v = C[a + (size_t)jb * sA];
            s += v.x * v.x + v.y * v.y;
          }
          s = wsum(s);
          const double inv = 1.0 / sqrt(s);
          for (int a = lane; a < sA; a += 32) {
            const double2 v = C[a + (size_t)jb * sA];
            Q[a + (size_t)t * sA] = make_double2(v.x * inv, v.y * inv);
          }
          if (lane == 0) piv[t] = jb, used[jb] = 1;
        }
        __syncthreads();
        const double2* q = Q + (size_t)t * sA;
        for (int j = warp; j < sB; j += OP_W) {
          if (used[j] && j != jb) {
            if (lane == 0) W[j + (size_t)t * sB] = make_double2(0.0, 0.0);  // W = R^H
            continue;
          }
          double2* aj = C + (size_t)j * sA;
          double2 tot = make_double2(0.0, 0.0);
          for (int pass2 = 0; pass2 < 2; ++pass2) {
            double2 c = make_double2(0.0, 0.0);
            for (int a = lane; a < sA; a += 32) pd_fmac(c, q[a], aj[a]);
            c.x = wsum(c.x), c.y = wsum(c.y);
            for (int a = lane; a < sA; a += 32) {
              const double2 v = aj[a], qa = q[a];
              aj[a] = make_double2(v.x - (c.x * qa.x - c.y * qa.y), v.y - (c.x * qa.y + c.y * qa.x));
            }
            __syncwarp();
            tot.x += c.x, tot.y += c.y;
          }
          double s = 0;
          for (int a = lane; a < sA; a += 32) s += aj[a].x * aj[a].x + aj[a].y * aj[a].y;
          s = wsum(s);
          if (lane == 0) {
            W[j + (size_t)t * sB] = make_double2(tot.x, -tot.y);
            nrm[j] = j == jb ? 0.0 : s;
          }
        }
        __syncthreads();
      }
      np_ = t;
      // ---- one-sided Jacobi on W = R^H (sB x np_), V (np_ x np_) = I
      for (int e = tid; e < np_ * np_; e += OP_T) V[e] = make_double2((e % np_) == (e / np_) ? 1.0 : 0.0, 0.0);
      __syncthreads();
      const int M = np_ + (np_ & 1);
      for (int sweep = 0; sweep < 60 && np_ > 1; ++sweep) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int rd = 0; rd < M - 1; ++rd) {
          for (int pi = warp; pi < M / 2; pi += OP_W) {
            int p = pi == 0 ? rd % (M - 1) : (rd + pi) % (M - 1);
            int qq = pi == 0 ? M - 1 : (rd - pi + M - 1) % (M - 1);
            if (p > qq) {
              const int tmp = p;
              p = qq, qq = tmp;
            }
            if (qq >= np_) continue;
            double2* wp = W + (size_t)p * sB;
            double2* wq = W + (size_t)qq * sB;
            double al = 0, be = 0;
            double2 g = make_double2(0.0, 0.0);
            for (int a = lane; a < sB; a += 32) {
              al += wp[a].x * wp[a].x + wp[a].y * wp[a].y;
              be += wq[a].x * wq[a].x + wq[a].y * wq[a].y;
              pd_fmac(g, wp[a], wq[a]);
            }
            al = wsum(al), be = wsum(be), g.x = wsum(g.x), g.y = wsum(g.y);
            const double ga = sqrt(g.x * g.x + g.y * g.y);
            if (al == 0.0 || be == 0.0 || ga <= 1e-15 * sqrt(al * be)) continue;
            if (lane == 0) s_rot = 1;
            const double zeta = (be - al) / (2.0 * ga);
            const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
            const double phr = g.x / ga, phi = -g.y / ga;  // conj(g / |g|)
            for (int a = lane; a < sB; a += 32) {
              const double2 ap = wp[a], aq0 = wq[a];
              const double2 aq = make_double2(aq0.x * phr - aq0.y * phi, aq0.x * phi + aq0.y * phr);
              wp[a] = make_double2(c * ap.x - s * aq.x, c * ap.y - s * aq.y);
              wq[a] = make_double2(s * ap.x + c * aq.x, s * ap.y + c * aq.y);
            }
            double2* vp = V + (size_t)p * np_;
            double2* vq = V + (size_t)qq * np_;
            for (int a = lane; a < np_; a += 32) {
              const double2 ap = vp[a], aq0 = vq[a];
              const double2 aq = make_double2(aq0.x * phr - aq0.y * phi, aq0.x * phi + aq0.y * phr);
              vp[a] = make_double2(c * ap.x - s * aq.x, c * ap.y - s * aq.y);
              vq[a] = make_double2(s * ap.x + c * aq.x, s * ap.y + c * aq.y);
            }
            __syncwarp();
          }
          __syncthreads();
        }
        if (!s_rot) break;
        __syncthreads();
      }
      // singular values, order, rank
      for (int tt = warp; tt < np_; tt += OP_W) {
        double s = 0;
        for (int a = lane; a < sB; a += 32) s += W[a + (size_t)tt * sB].x * W[a + (size_t)tt * sB].x +
                                                  W[a + (size_t)tt * sB].y * W[a + (size_t)tt * sB].y;
        s = wsum(s);
        if (lane == 0) sig[tt] = sqrt(s);
      }
      __syncthreads();
      if (tid == 0) {
        for (int i = 0; i < np_; ++i) sel[i] = i;
        for (int i = 1; i < np_; ++i) {  // stable insertion sort, descending sigma
          const int v = sel[i];
          int j = i - 1;
          while (j >= 0 && sig[sel[j]] < sig[v]) sel[j + 1] = sel[j], --j;
          sel[j + 1] = v;
        }
        int r = 0;
        const double s1 = np_ ? sig[sel[0]] : 0.0;
        for (int i = 0; i < np_; ++i)
          if (sig[sel[i]] >= J.eps_lr * s1 && sig[sel[i]] > 0.0) ++r;
        // low rank iff r < s/2 (eq_lrdk); the kernel computes with r rounded up to 8 (its tile height), so
        // the rank is rounded up too -- more accuracy at no extra work (R23)
        const int rr = J.rank_round > 1 ? J.rank_round : 1;
        const int r8 = min((r + rr - 1) / rr * rr, np_);
        s_rank = (2 * r < max(sA, sB)) ? (2 * r8 < max(sA, sB) ? r8 : r) : -1;
      }
      __syncthreads();
      rank = s_rank;
    }
    if (pass == 1) {
      if (tid == 0) J.rank[it] = rank;
      __syncthreads();
      continue;
    }
    double* dst = J.pool + J.off[it];
    if (J.compress && J.rank_in) rank = J.rank_in[it];
    if (rank < 0) {
      frag_write(dst, sA, sB, pd_pad8(J.s_out), pd_pad4(J.s_in), [&](int i, int j) { return O[i + (size_t)j * sA]; });
      if (J.poolT) {
        double* dT = J.poolT + (int64_t)it * ((int64_t)pd_pad8(J.s_in) / 8) * (pd_pad4(J.s_out) / 4) * 64;
        frag_write(dT, sB, sA, pd_pad8(J.s_in), pd_pad4(J.s_out), [&](int i, int j) { return O[j + (size_t)i * sA]; });
      }
    } else {
      // U^ = (Q V)[:, sel] (sA x r), V^ = W[:, sel]^H (r x sB)
      for (int e = tid; e < sA * rank; e += OP_T) {
        const int a = e % sA, c = e / sA;
        double2 acc = make_double2(0.0, 0.0);
        const int sc = sel[c];
        for (int tt = 0; tt < np_; ++tt) pd_fma(acc, Q[a + (size_t)tt * sA], V[tt + (size_t)sc * np_]);
        U[e] = acc;
      }
      __syncthreads();
      frag_write(dst, rank, sB, pd_pad8(rank), pd_pad4(J.s_in), [&](int i, int j) {
        const double2 w = W[j + (size_t)sel[i] * sB];
        return make_double2(w.x, -w.y);
      });
      double* du = dst + (int64_t)(pd_pad8(rank) / 8) * (pd_pad4(J.s_in) / 4) * 64;
      frag_write(du, sA, rank, pd_pad8(J.s_out), pd_pad8(rank), [&](int i, int j) { return U[i + (size_t)j * sA]; });
    }
    __syncthreads();
  }
}

cudaError_t launch_opjob(const OpJob& J, int pass, cudaStream_t st) {
  if (J.n_items <= 0) return cudaSuccess;
  const size_t per = (size_t)J.maxn * J.maxn + (size_t)J.maxn * J.maxs + 5 * (size_t)J.maxs * J.maxs;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // 2 CTAs per SM, bounded by a 4 GB workspace
  int64_t grid = std::min<int64_t>(J.n_items, 2 * (int64_t)nsm);
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, (int64_t)((4ull << 30) / (per * sizeof(double2)))));
  double2* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, (size_t)grid * per * sizeof(double2), st);
  if (e != cudaSuccess) {
    if (getenv("FDA_DEBUG"))
      fprintf(stderr, "fda: k_opjob workspace of %zu B failed (maxn %d maxs %d)\n", (size_t)grid * per * sizeof(double2),
              J.maxn, J.maxs);
    return e;
  }
  const size_t smem = (size_t)J.maxs * (2 * sizeof(double) + 2 * sizeof(int) + 1) + 16;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_opjob, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_opjob<<<(unsigned)grid, OP_T, smem, st>>>(J, pass, ws, per);
  e = cudaGetLastError();
  if (e != cudaSuccess && getenv("FDA_DEBUG"))
    fprintf(stderr, "fda: k_opjob pass %d launch failed (%s): items %d grid %lld smem %zu maxn %d maxs %d ws %zu B\n", pass,
            cudaGetErrorString(e), J.n_items, (long long)grid, smem, J.maxn, J.maxs, (size_t)grid * per * sizeof(double2));
  cudaFreeAsync(ws, st);
  return e;
}

// ---------------------------------------------------------------- HF directional sets (pivoted column selection)
__global__ void k_gmat(double2* A, const double* X, int64_t m, const double* Y, int64_t n, const double* rs,
                       const double* cs, double k) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * n) return;
  const int64_t i = e % m, j = e / m;
  double2 v = pd_g(k, X[3 * i] - Y[3 * j], X[3 * i + 1] - Y[3 * j + 1], X[3 * i + 2] - Y[3 * j + 2]);
  if (rs) v.x *= rs[i], v.y *= rs[i];
  if (cs) v.x *= cs[j], v.y *= cs[j];
  A[e] = v;
}
void launch_gmat(double2* A, const double* X, int64_t m, const double* Y, int64_t n, const double* rs, const double* cs,
                 double k, cudaStream_t st) {
  if (m * n <= 0) return;
  k_gmat<<<(unsigned)((m * n + 255) / 256), 256, 0, st>>>(A, X, m, Y, n, rs, cs, k);
}

// column norms (block per column)
__global__ void k_colnrm(const double2* A, int64_t m, int64_t n, double* nrm) {
  __shared__ double red[8];
  const int64_t j = blockIdx.x;
  double s = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double2 v = A[i + j * m];
    s += v.x * v.x + v.y * v.y;
  }
  s = wsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    nrm[j] = t;
  }
}
// argmax over unused columns -> out[0] = best (as double), out[1] = index (as double)
__global__ void k_argmax(const double* nrm, const unsigned char* used, int64_t n, double* out) {
  __shared__ double red_v[32];
  __shared__ int red_j[32];
  double v = -1.0;
  int jj = -1;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
    if (!used[j] && nrm[j] > v) v = nrm[j], jj = (int)j;
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int j2 = __shfl_xor_sync(0xffffffffu, jj, o);
    if (v2 > v || (v2 == v && j2 >= 0 && (jj < 0 || j2 < jj))) v = v2, jj = j2;
  }
  if ((threadIdx.x & 31) == 0) red_v[threadIdx.x >> 5] = v, red_j[threadIdx.x >> 5] = jj;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = -1.0;
    int bj = -1;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      if (red_v[w] > b || (red_v[w] == b && red_j[w] >= 0 && (bj < 0 || red_j[w] < bj))) b = red_v[w], bj = red_j[w];
    out[0] = b, out[1] = (double)bj;
  }
}
// q = a_jb / |a_jb| (one block); used[jb] = 1
__global__ void k_makeq(const double2* A, int64_t m, const double* amx, double2* q, unsigned char* used) {
  __shared__ double red[32];
  __shared__ double s_inv;
  const int64_t jb = (int64_t)amx[1];
  double s = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double2 v = A[i + jb * m];
    s += v.x * v.x + v.y * v.y;
  }
  s = wsum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    s_inv = 1.0 / sqrt(t);
    used[jb] = 1;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double2 v = A[i + jb * m];
    q[i] = make_double2(v.x * s_inv, v.y * s_inv);
  }
}
// project q out of every active column (twice), update its norm (block per column)
__global__ void k_project(double2* A, int64_t m, const double2* q, const unsigned char* used, const double* amx,
                          double* nrm) {
  __shared__ double rx[8], ry[8];
  __shared__ double2 s_c;
  const int64_t j = blockIdx.x, jb = (int64_t)amx[1];
  if (used[j] && j != jb) return;
  double2* a = A + j * m;
  for (int pass = 0; pass < 2; ++pass) {
    double2 c = make_double2(0.0, 0.0);
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) pd_fmac(c, q[i], a[i]);
    c.x = wsum(c.x), c.y = wsum(c.y);
    if ((threadIdx.x & 31) == 0) rx[threadIdx.x >> 5] = c.x, ry[threadIdx.x >> 5] = c.y;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 t = make_double2(0.0, 0.0);
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t.x += rx[w], t.y += ry[w];
      s_c = t;
    }
    __syncthreads();
    const double2 cc = s_c;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
      const double2 v = a[i], qi = q[i];
      a[i] = make_double2(v.x - (cc.x * qi.x - cc.y * qi.y), v.y - (cc.x * qi.y + cc.y * qi.x));
    }
    __syncthreads();
  }
  double s = 0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += a[i].x * a[i].x + a[i].y * a[i].y;
  s = wsum(s);
  if ((threadIdx.x & 31) == 0) rx[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += rx[w];
    nrm[j] = j == jb ? 0.0 : t;
  }
}

cudaError_t pivoted_columns(double2* A, int64_t m, int64_t n, double tol, int64_t maxrank, int64_t* piv, int64_t* npiv,
                            cudaStream_t st) {
  *npiv = 0;
  if (m <= 0 || n <= 0) return cudaSuccess;
  double *nrm = nullptr, *amx = nullptr;
  double2* q = nullptr;
  unsigned char* used = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&nrm, n * sizeof(double), st)) != cudaSuccess) return e;
  cudaMallocAsync(&amx, 2 * sizeof(double), st);
  cudaMallocAsync(&q, m * sizeof(double2), st);
  cudaMallocAsync(&used, n, st);
  cudaMemsetAsync(used, 0, n, st);
  k_colnrm<<<(unsigned)n, 256, 0, st>>>(A, m, n, nrm);
  const int64_t rmax = std::min<int64_t>({maxrank, m, n});
  double n0 = -1, hb[2];
  for (int64_t t = 0; t < rmax; ++t) {
    k_argmax<<<1, 1024, 0, st>>>(nrm, used, n, amx);
    if ((e = cudaMemcpyAsync(hb, amx, 2 * sizeof(double), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
    if (n0 < 0) n0 = std::sqrt(std::max(hb[0], 0.0));
    if (hb[1] < 0 || hb[0] <= 0.0 || std::sqrt(hb[0]) <= tol * n0) break;
    piv[(*npiv)++] = (int64_t)hb[1];
    k_makeq<<<1, 1024, 0, st>>>(A, m, amx, q, used);
    k_project<<<(unsigned)n, 256, 0, st>>>(A, m, q, used, amx, nrm);
  }
  cudaFreeAsync(nrm, st);
  cudaFreeAsync(amx, st);
  cudaFreeAsync(q, st);
  cudaFreeAsync(used, st);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

}  // namespace fda
