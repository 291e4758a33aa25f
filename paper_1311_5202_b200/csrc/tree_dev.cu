// tree_dev.cu -- Morton sort and adaptive octree on the device.  See tree_dev.cuh.
#include "tree_dev.cuh"

#include <cub/cub.cuh>

#include <cmath>

#include "plan.hpp"

namespace fda {

namespace {

constexpr int TD_MAXD = 21;  // Morton bits per axis
constexpr double TD_PI = 3.14159265358979323846;

struct TdFail {
  std::string what;
};
inline void tck(cudaError_t e) {
  if (e != cudaSuccess) throw TdFail{"CUDA"};
}

__device__ __forceinline__ uint64_t td_spread3(uint64_t v) {
  v &= 0x1fffff;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// per point: validity (finite, |n| = 1 to 1e-10, w > 0) and the block's bounding box
__global__ void k_validate_box(int64_t n, const double* __restrict__ x, const double* __restrict__ nr,
                               const double* __restrict__ w, int* bad, double* box /* per block: 6 */) {
  __shared__ double red[6][8];
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  int b = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double nn = sqrt(nr[3 * i] * nr[3 * i] + nr[3 * i + 1] * nr[3 * i + 1] + nr[3 * i + 2] * nr[3 * i + 2]);
    bool ok = isfinite(w[i]) && w[i] > 0 && isfinite(nn) && fabs(nn - 1.0) <= 1e-10;
    for (int d = 0; d < 3; ++d) {
      const double v = x[3 * i + d];
      ok = ok && isfinite(v);
      lo[d] = fmin(lo[d], v), hi[d] = fmax(hi[d], v);
    }
    b |= !ok;
  }
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  if ((threadIdx.x & 31) == 0)
    for (int d = 0; d < 3; ++d) red[d][threadIdx.x >> 5] = lo[d], red[3 + d][threadIdx.x >> 5] = hi[d];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int d = 0; d < 3; ++d) {
      double a = 1e300, c = -1e300;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) a = fmin(a, red[d][q]), c = fmax(c, red[3 + d][q]);
      box[6 * blockIdx.x + d] = a, box[6 * blockIdx.x + 3 + d] = c;
    }
  }
}

__global__ void k_morton(int64_t n, const double* __restrict__ x, double lo0, double lo1, double lo2, double scale,
                         uint64_t* key, int32_t* idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo[3] = {lo0, lo1, lo2};
  uint64_t c[3];
  for (int d = 0; d < 3; ++d) {
    int64_t v = (int64_t)floor((x[3 * i + d] - lo[d]) * scale);
    v = v < 0 ? 0 : (v > (1 << TD_MAXD) - 1 ? (1 << TD_MAXD) - 1 : v);
    c[d] = (uint64_t)v;
  }
  key[i] = (td_spread3(c[0]) << 2) | (td_spread3(c[1]) << 1) | td_spread3(c[2]);
  idx[i] = (int32_t)i;
}

__global__ void k_gather_soa(int64_t n, const int32_t* __restrict__ perm, const double* __restrict__ x,
                             const double* __restrict__ nr, const double* __restrict__ w, DevGeom g) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t i = perm[t];
  g.x[t] = x[3 * i], g.y[t] = x[3 * i + 1], g.z[t] = x[3 * i + 2];
  g.nx[t] = nr[3 * i], g.ny[t] = nr[3 * i + 1], g.nz[t] = nr[3 * i + 2];
  g.w[t] = w[i];
  g.perm[t] = perm[t];
}

__global__ void k_coincident(int64_t n, const uint64_t* __restrict__ skey, DevGeom g, double tol, int* bad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < 1 || t >= n || skey[t] != skey[t - 1]) return;
  const double dx = g.x[t] - g.x[t - 1], dy = g.y[t] - g.y[t - 1], dz = g.z[t] - g.z[t - 1];
  if (sqrt(dx * dx + dy * dy + dz * dz) < tol) atomicOr(bad, 1);
}

// level step: children of the split cubes of level l are the distinct level-(l+1) prefixes of their points
__global__ void k_child_flags(int64_t n, const uint64_t* __restrict__ skey, const int32_t* __restrict__ cop,
                              const int64_t* __restrict__ pbeg, const unsigned char* __restrict__ split, int shift,
                              int32_t* flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = cop[i];
  int32_t f = 0;
  if (c >= 0 && split[c]) f = (i == pbeg[c]) || ((skey[i] >> shift) != (skey[i - 1] >> shift));
  flag[i] = f;
}
__global__ void k_child_make(int64_t n, const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                             const int32_t* __restrict__ cop, int64_t* cpbeg, int32_t* cpar, int32_t* cop_next) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = cop[i];
  if (flag[i]) cpbeg[pos[i]] = i, cpar[pos[i]] = c;
  // points of a split cube belong to the child that starts at or before them (pos + flag - 1); points of a
  // leaf are no longer tracked
  cop_next[i] = (c >= 0 && (flag[i] || pos[i] > 0)) ? pos[i] + flag[i] - 1 : -1;
}
__global__ void k_child_end(int64_t nch, const int64_t* __restrict__ cpbeg, const int32_t* __restrict__ cpar,
                            const int64_t* __restrict__ pend, int64_t* cpend) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nch) return;
  cpend[c] = (c + 1 < nch && cpar[c + 1] == cpar[c]) ? cpbeg[c + 1] : pend[cpar[c]];
}
__global__ void k_fix_cop(int64_t n, const int32_t* __restrict__ cop, const unsigned char* __restrict__ split,
                          int32_t* cop_next) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t c = cop[i];
  if (c < 0 || !split[c]) cop_next[i] = -1;
}
__global__ void k_split(int64_t nc, const int64_t* __restrict__ pbeg, const int64_t* __restrict__ pend, int np,
                        int force, int none, unsigned char* split) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc) return;
  split[c] = !none && (force || pend[c] - pbeg[c] > np);
}
__global__ void k_cube_keys(int64_t nc, const int64_t* __restrict__ pbeg, const uint64_t* __restrict__ skey,
                            int shift, uint64_t* ck) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < nc) ck[c] = skey[pbeg[c]] >> shift;
}

inline unsigned nb(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

template <class T>
T* dmalloc(size_t count, cudaStream_t st) {
  void* p = nullptr;
  tck(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st));
  return (T*)p;
}

}  // namespace

std::string build_tree_device(int64_t n, const double* pts, const double* nrm, const double* w, double k, int np,
                              int single_leaf, int max_depth, const DevGeom& g, TreeIn& out, cudaStream_t st) {
  std::vector<void*> tmp;
  auto alloc = [&](auto* tag, size_t count) {
    using T = std::remove_pointer_t<decltype(tag)>;
    T* p = dmalloc<T>(count, st);
    tmp.push_back(p);
    return p;
  };
  try {
    // ---- P0: validation, bounding cube
    const int nblk = 2 * 148;
    int* bad = alloc((int*)nullptr, 2);
    double* box = alloc((double*)nullptr, 6 * nblk);
    tck(cudaMemsetAsync(bad, 0, 2 * sizeof(int), st));
    k_validate_box<<<nblk, 256, 0, st>>>(n, pts, nrm, w, bad, box);
    std::vector<double> hb(6 * nblk);
    int hbad[2];
    tck(cudaMemcpyAsync(hb.data(), box, hb.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    tck(cudaMemcpyAsync(hbad, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    tck(cudaStreamSynchronize(st));
    if (hbad[0]) throw TdFail{"INVALID_ARG"};
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int b = 0; b < nblk; ++b)
      for (int d = 0; d < 3; ++d) lo[d] = std::min(lo[d], hb[6 * b + d]), hi[d] = std::max(hi[d], hb[6 * b + 3 + d]);
    double W = 0;
    for (int d = 0; d < 3; ++d) W = std::max(W, hi[d] - lo[d]);
    if (W <= 0) W = 1.0;
    W *= (1.0 + 1e-6);  // root = bounding cube x (1 + 1e-6)   (R13)
    for (int d = 0; d < 3; ++d) out.root_lo[d] = 0.5 * (lo[d] + hi[d]) - 0.5 * W;
    out.root_w = W;
    // ---- Morton keys, stable radix sort (equal keys keep the caller order, as std::stable_sort)
    uint64_t* key = alloc((uint64_t*)nullptr, n);
    uint64_t* skey = alloc((uint64_t*)nullptr, n);
    int32_t* idx = alloc((int32_t*)nullptr, n);
    int32_t* perm = alloc((int32_t*)nullptr, n);
    k_morton<<<nb(n), 256, 0, st>>>(n, pts, out.root_lo[0], out.root_lo[1], out.root_lo[2], (double)(1 << TD_MAXD) / W,
                                     key, idx);
    size_t tb = 0;
    tck(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, skey, idx, perm, (int)n, 0, 3 * TD_MAXD, st));
    void* tbuf = alloc((char*)nullptr, tb);
    tck(cub::DeviceRadixSort::SortPairs(tbuf, tb, key, skey, idx, perm, (int)n, 0, 3 * TD_MAXD, st));
    k_gather_soa<<<nb(n), 256, 0, st>>>(n, perm, pts, nrm, w, g);
    k_coincident<<<nb(n), 256, 0, st>>>(n, skey, g, 1e-14 * W, bad + 1);
    out.perm.resize(n);
    tck(cudaMemcpyAsync(out.perm.data(), perm, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    tck(cudaMemcpyAsync(hbad, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    tck(cudaStreamSynchronize(st));
    if (hbad[1]) throw TdFail{"COINCIDENT_POINTS"};

    // ---- P1: levels
    const double lambda = k > 0 ? 2.0 * TD_PI / k : INFINITY;
    int32_t* cop = alloc((int32_t*)nullptr, n);       // cube (index within the level) of each tracked point
    int32_t* cop2 = alloc((int32_t*)nullptr, n);
    int32_t* flag = alloc((int32_t*)nullptr, n);
    int32_t* pos = alloc((int32_t*)nullptr, n);
    tck(cudaMemsetAsync(cop, 0, n * sizeof(int32_t), st));
    size_t sb = 0;
    tck(cub::DeviceScan::ExclusiveSum(nullptr, sb, flag, pos, (int)n, st));
    void* sbuf = alloc((char*)nullptr, sb);
    // level 0: the root
    int64_t* pbeg = alloc((int64_t*)nullptr, 1);
    int64_t* pend = alloc((int64_t*)nullptr, 1);
    const int64_t zero = 0;
    tck(cudaMemcpyAsync(pbeg, &zero, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    tck(cudaMemcpyAsync(pend, &n, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    int64_t nc = 1;
    out.level.assign(1, 0), out.pbeg.assign(1, 0), out.pend.assign(1, n), out.parent.assign(1, -1);
    out.key.assign(1, 0);
    out.leaf.assign(1, 1);
    int64_t base = 0;  // global id of the level's first cube
    for (int l = 0; l < max_depth; ++l) {
      const bool hf = k > 0 && W / (double)(1LL << l) >= lambda;  // HF iff w >= lambda (R13)
      unsigned char* split = alloc((unsigned char*)nullptr, nc);
      k_split<<<nb(nc), 256, 0, st>>>(nc, pbeg, pend, np, hf ? 1 : 0, single_leaf, split);
      const int shift = 3 * (TD_MAXD - l - 1);
      k_child_flags<<<nb(n), 256, 0, st>>>(n, skey, cop, pbeg, split, shift, flag);
      tck(cub::DeviceScan::ExclusiveSum(sbuf, sb, flag, pos, (int)n, st));
      int32_t last[2];
      tck(cudaMemcpyAsync(&last[0], pos + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      tck(cudaMemcpyAsync(&last[1], flag + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      std::vector<unsigned char> hs(nc);
      tck(cudaMemcpyAsync(hs.data(), split, nc, cudaMemcpyDeviceToHost, st));
      tck(cudaStreamSynchronize(st));
      for (int64_t c = 0; c < nc; ++c) out.leaf[base + c] = !hs[c];
      const int64_t nch = (int64_t)last[0] + last[1];
      if (nch == 0) break;
      int64_t* cpbeg = alloc((int64_t*)nullptr, nch);
      int64_t* cpend = alloc((int64_t*)nullptr, nch);
      int32_t* cpar = alloc((int32_t*)nullptr, nch);
      uint64_t* ckey = alloc((uint64_t*)nullptr, nch);
      k_child_make<<<nb(n), 256, 0, st>>>(n, flag, pos, cop, cpbeg, cpar, cop2);
      k_fix_cop<<<nb(n), 256, 0, st>>>(n, cop, split, cop2);
      k_child_end<<<nb(nch), 256, 0, st>>>(nch, cpbeg, cpar, pend, cpend);
      k_cube_keys<<<nb(nch), 256, 0, st>>>(nch, cpbeg, skey, shift, ckey);
      std::vector<int64_t> hb2(nch), he2(nch);
      std::vector<int32_t> hp(nch);
      std::vector<uint64_t> hk(nch);
      tck(cudaMemcpyAsync(hb2.data(), cpbeg, nch * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      tck(cudaMemcpyAsync(he2.data(), cpend, nch * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      tck(cudaMemcpyAsync(hp.data(), cpar, nch * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      tck(cudaMemcpyAsync(hk.data(), ckey, nch * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      tck(cudaStreamSynchronize(st));
      const int64_t nbase = base + nc;
      for (int64_t c = 0; c < nch; ++c) {
        out.level.push_back(l + 1);
        out.pbeg.push_back(hb2[c]), out.pend.push_back(he2[c]);
        out.parent.push_back(base + hp[c]);
        out.key.push_back((int64_t)hk[c]);
        out.leaf.push_back(1);
      }
      base = nbase;
      nc = nch;
      pbeg = cpbeg, pend = cpend;
      std::swap(cop, cop2);
    }
  } catch (const TdFail& f) {
    for (void* p : tmp) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaGetLastError();
    return f.what;
  }
  for (void* p : tmp) cudaFreeAsync(p, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return "CUDA";
  return "";
}

// ---------------------------------------------------------------- correction CSR into Morton order
namespace {
__global__ void k_csr_rows_ok(int64_t n, const int64_t* __restrict__ rp, int* bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && rp[i + 1] < rp[i]) atomicOr(bad, 1);
}
__global__ void k_csr_cols_ok(int64_t nnz, int64_t n, const int32_t* __restrict__ col, int* bad) {
  int b = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    b |= col[p] < 0 || col[p] >= n;
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void k_inv_perm(int64_t n, const int32_t* __restrict__ perm, int32_t* inv) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m < n) inv[perm[m]] = (int32_t)m;
}
__global__ void k_csr_len(int64_t r0, int64_t nr, const int32_t* __restrict__ perm, const int64_t* __restrict__ rp,
                          int64_t* len) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > nr) return;
  if (j == nr) {
    len[j] = 0;
    return;
  }
  const int64_t i = perm[r0 + j];
  len[j] = rp[i + 1] - rp[i];
}
// warp per Morton row: copy the caller row perm[m] with its columns mapped to Morton order
__global__ void k_csr_permute(int64_t r0, int64_t nr, const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                              const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double2* __restrict__ val, const int64_t* __restrict__ mp, int32_t* ocol,
                              double2* oval) {
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  if (j >= nr) return;
  const int lane = threadIdx.x & 31;
  const int64_t i = perm[r0 + j];
  const int64_t b = rp[i], e = rp[i + 1], o = mp[j];
  for (int64_t p = b + lane; p < e; p += 32) {
    ocol[o + (p - b)] = inv[col[p]];
    oval[o + (p - b)] = val[p];
  }
}
__global__ void k_csr_ptr(int64_t r0, int64_t nr, const int64_t* __restrict__ mp, int64_t* optr) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j <= nr) optr[r0 + j] = mp[j];
}
}  // namespace

std::string permute_csr_device(int64_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const double2* val,
                               const int32_t* perm, int64_t r0, int64_t r1, int64_t* optr, int32_t** ocol,
                               double2** oval, int64_t* onnz, cudaStream_t st) {
  std::vector<void*> tmp;
  try {
    int* bad = dmalloc<int>(1, st);
    tmp.push_back(bad);
    tck(cudaMemsetAsync(bad, 0, sizeof(int), st));
    int64_t ends[2];
    tck(cudaMemcpyAsync(&ends[0], rp, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    tck(cudaMemcpyAsync(&ends[1], rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    k_csr_rows_ok<<<nb(n), 256, 0, st>>>(n, rp, bad);
    k_csr_cols_ok<<<4 * 148, 256, 0, st>>>(nnz, n, col, bad);
    int hbad = 0;
    tck(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    tck(cudaStreamSynchronize(st));
    if (hbad || ends[0] != 0 || ends[1] != nnz) throw TdFail{"INVALID_ARG"};
    const int64_t nr = r1 - r0;
    int32_t* inv = dmalloc<int32_t>(n, st);
    tmp.push_back(inv);
    int64_t* len = dmalloc<int64_t>(nr + 1, st);
    tmp.push_back(len);
    int64_t* mp = dmalloc<int64_t>(nr + 1, st);
    tmp.push_back(mp);
    k_inv_perm<<<nb(n), 256, 0, st>>>(n, perm, inv);
    k_csr_len<<<nb(nr + 1), 256, 0, st>>>(r0, nr, perm, rp, len);
    size_t sb = 0;
    tck(cub::DeviceScan::ExclusiveSum(nullptr, sb, len, mp, (int)(nr + 1), st));
    void* sbuf = dmalloc<char>(sb, st);
    tmp.push_back(sbuf);
    tck(cub::DeviceScan::ExclusiveSum(sbuf, sb, len, mp, (int)(nr + 1), st));
    tck(cudaMemcpyAsync(onnz, mp + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    tck(cudaStreamSynchronize(st));
    tck(cudaMalloc(ocol, std::max<int64_t>(1, *onnz) * sizeof(int32_t)));
    tck(cudaMalloc(oval, std::max<int64_t>(1, *onnz) * sizeof(double2)));
    k_csr_permute<<<nb(nr * 32), 256, 0, st>>>(r0, nr, perm, inv, rp, col, val, mp, *ocol, *oval);
    k_csr_ptr<<<nb(nr + 1), 256, 0, st>>>(r0, nr, mp, optr);
  } catch (const TdFail& f) {
    for (void* p : tmp) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaGetLastError();
    return f.what;
  }
  for (void* p : tmp) cudaFreeAsync(p, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return "CUDA";
  return "";
}

}  // namespace fda
