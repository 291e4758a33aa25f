// lists_dev.cu -- P2P lists, interaction lists and expansion slots on the device.  See lists_dev.cuh.
#include "lists_dev.cuh"

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include "plan.hpp"

namespace fda {

namespace {

struct LdFail {};
inline void lck(cudaError_t e) {
  if (e != cudaSuccess) throw LdFail{};
}
inline unsigned ld_nb(int64_t n) { return (unsigned)((n + 255) / 256); }

__host__ __device__ inline uint64_t ld_spread3(uint64_t v) {
  v &= 0x1fffff;
  v = (v | (v << 32)) & 0x1f00000000ffffull;
  v = (v | (v << 16)) & 0x1f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}
__host__ __device__ inline uint64_t ld_key(int64_t i, int64_t j, int64_t k) {
  return (ld_spread3((uint64_t)i) << 2) | (ld_spread3((uint64_t)j) << 1) | ld_spread3((uint64_t)k);
}

struct DevLevelT {
  int64_t nc = 0;
  const uint64_t* key = nullptr;        // Morton key of the cube's ijk (ascending: the level's Morton order)
  const int64_t* ijk = nullptr;         // 3 per cube
  const unsigned char* leaf = nullptr;
  const int32_t* child = nullptr;       // 8 per cube: local index at the next level or -1
  const int64_t* pbeg = nullptr;
  const int64_t* pend = nullptr;
};

__device__ int64_t ld_find(const DevLevelT& L, uint64_t key) {
  int64_t lo = 0, hi = L.nc - 1;
  while (lo <= hi) {
    const int64_t mid = (lo + hi) >> 1;
    const uint64_t v = L.key[mid];
    if (v == key) return mid;
    if (v < key) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}
__device__ int64_t ld_lower(const int64_t* a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ---- P2P lists (R20): pass 0 counts, pass 1 writes (unsorted within a leaf)
__global__ void k_p2p_lists(int pass, int64_t nl, const int32_t* __restrict__ leaf_level,
                            const int64_t* __restrict__ leaf_local, const DevLevelT* __restrict__ lv,
                            const int64_t* __restrict__ leaf_pbeg, int64_t* cnt, const int64_t* __restrict__ ptr,
                            int32_t* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nl) return;
  const int lt = leaf_level[t];
  const DevLevelT L = lv[lt];
  const int64_t c = leaf_local[t];
  const int64_t i0 = L.ijk[3 * c], j0 = L.ijk[3 * c + 1], k0 = L.ijk[3 * c + 2];
  int64_t n = 0, o = pass ? ptr[t] : 0;
  const int64_t lim = 1LL << lt;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        const int64_t i = i0 + dx, j = j0 + dy, k = k0 + dz;
        if (i < 0 || j < 0 || k < 0 || i >= lim || j >= lim || k >= lim) continue;
        const int64_t a = ld_find(L, ld_key(i, j, k));
        if (a < 0) continue;
        // the leaf descendants of cube a: the leaves whose points start inside its point range
        const int64_t lo = ld_lower(leaf_pbeg, nl, L.pbeg[a]), hi = ld_lower(leaf_pbeg, nl, L.pend[a]);
        if (pass)
          for (int64_t q = lo; q < hi; ++q) out[o++] = (int32_t)q;
        n += hi - lo;
      }
  for (int la = lt - 1; la >= 0; --la) {  // leaves adjacent to an ancestor
    const DevLevelT A = lv[la];
    const int sh = lt - la;
    const int64_t ai = i0 >> sh, aj = j0 >> sh, ak = k0 >> sh, alim = 1LL << la;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          if (!dx && !dy && !dz) continue;
          const int64_t i = ai + dx, j = aj + dy, k = ak + dz;
          if (i < 0 || j < 0 || k < 0 || i >= alim || j >= alim || k >= alim) continue;
          const int64_t a = ld_find(A, ld_key(i, j, k));
          if (a < 0 || !A.leaf[a]) continue;
          if (pass) out[o++] = (int32_t)ld_lower(leaf_pbeg, nl, A.pbeg[a]);
          ++n;
        }
  }
  if (!pass) cnt[t] = n;
}

// ---- interaction lists of level l: parents Lp (level l-1), children at level l.  nq candidates per parent:
// the (2 Rp + 1)^3 offsets, or every parent (brute).  pass 0 counts, pass 1 writes (key << 32 | B, C).
__global__ void k_vlist(int pass, int64_t npar, int64_t nq, int brute, DevLevelT Lp, int Rp, int Rc, int span, int D,
                        int64_t* cnt, const int64_t* __restrict__ off, uint64_t* okey, int32_t* oc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= npar * nq) return;
  const int64_t pi = t / nq, q = t % nq;
  int64_t n = 0;
  if (!Lp.leaf[pi]) {
    const int64_t pi0 = Lp.ijk[3 * pi], pj0 = Lp.ijk[3 * pi + 1], pk0 = Lp.ijk[3 * pi + 2];
    int64_t qi = -1;
    if (brute) {
      const int64_t dm = max(max(llabs(Lp.ijk[3 * q] - pi0), llabs(Lp.ijk[3 * q + 1] - pj0)), llabs(Lp.ijk[3 * q + 2] - pk0));
      if (dm <= Rp) qi = q;
    } else {
      const int64_t w = 2 * Rp + 1;
      const int64_t dx = q / (w * w) - Rp, dy = (q / w) % w - Rp, dz = q % w - Rp;
      const int64_t i = pi0 + dx, j = pj0 + dy, k = pk0 + dz;
      // out-of-range cubes have keys beyond every cube of the level: not found
      if (i >= 0 && j >= 0 && k >= 0) qi = ld_find(Lp, ld_key(i, j, k));
    }
    if (qi >= 0 && !Lp.leaf[qi]) {
      const int64_t qi0 = Lp.ijk[3 * qi], qj0 = Lp.ijk[3 * qi + 1], qk0 = Lp.ijk[3 * qi + 2];
      int64_t o = pass ? off[t] : 0;
      for (int ob = 0; ob < 8; ++ob) {
        const int32_t B = Lp.child[pi * 8 + ob];
        if (B < 0) continue;
        const int64_t bi = 2 * pi0 + ((ob >> 2) & 1), bj = 2 * pj0 + ((ob >> 1) & 1), bk = 2 * pk0 + (ob & 1);
        for (int ocx = 0; ocx < 8; ++ocx) {
          const int32_t C = Lp.child[qi * 8 + ocx];
          if (C < 0) continue;
          const int64_t d0 = bi - (2 * qi0 + ((ocx >> 2) & 1)), d1 = bj - (2 * qj0 + ((ocx >> 1) & 1)),
                        d2 = bk - (2 * qk0 + (ocx & 1));
          const int64_t dm = max(max(llabs(d0), llabs(d1)), llabs(d2));
          if (dm <= Rc) continue;  // near at this level
          if (pass) {
            const uint64_t key = (uint64_t)(((d0 + span) * D + (d1 + span)) * D + (d2 + span));
            okey[o] = (key << 32) | (uint64_t)(uint32_t)B;
            oc[o] = C;
            ++o;
          }
          ++n;
        }
      }
    }
  }
  if (!pass) cnt[t] = n;
}

__global__ void k_split_key(int64_t n, const uint64_t* __restrict__ okey, uint32_t* gk, int32_t* b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  gk[i] = (uint32_t)(okey[i] >> 32);
  b[i] = (int32_t)(okey[i] & 0xffffffffu);
}

__device__ inline int ld_anti_dir(int d, int m) {
  const int f = d / (m * m), rem = d % (m * m), a = rem / m, b = rem % m;
  return ((f ^ 1) * m + (m - 1 - a)) * m + (m - 1 - b);
}
__device__ inline int ld_child_dir(int d, int mp) {
  const int f = d / (mp * mp), rem = d % (mp * mp), a = rem / mp, b = rem % mp, mc = mp / 2;
  return (f * mc + a / 2) * mc + b / 2;
}

// group of every pair (binary search in the run offsets)
__device__ int64_t ld_run(const int64_t* roff, int64_t nruns, int64_t p) {
  int64_t lo = 0, hi = nruns - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (roff[mid] <= p) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
// HF slot marks from the pairs: out (C, d), in (B, antipode of d)
__global__ void k_mark_pairs(int64_t np, const int64_t* __restrict__ roff, int64_t nruns, const int32_t* __restrict__ gdir,
                             const int32_t* __restrict__ b, const int32_t* __restrict__ c, int m, int ndir,
                             unsigned char* omark, unsigned char* imark) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int d = gdir[ld_run(roff, nruns, p)];
  omark[(int64_t)c[p] * ndir + d] = 1;
  imark[(int64_t)b[p] * ndir + ld_anti_dir(d, m)] = 1;
}
// closure from the parent level's slots: every child of a parent with slot (pc, d) gets (child, child_dir(d))
__global__ void k_mark_closure(int64_t npar, int ndirp, int mp, const int32_t* __restrict__ child,
                               const unsigned char* __restrict__ pom, const unsigned char* __restrict__ pim, int ndir,
                               unsigned char* omark, unsigned char* imark) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= npar * ndirp) return;
  const bool o = pom[e], i = pim[e];
  if (!o && !i) return;
  const int64_t pc = e / ndirp;
  const int cd = ld_child_dir((int)(e % ndirp), mp);
  for (int oc = 0; oc < 8; ++oc) {
    const int32_t cl = child[pc * 8 + oc];
    if (cl < 0) continue;
    if (o) omark[(int64_t)cl * ndir + cd] = 1;
    if (i) imark[(int64_t)cl * ndir + cd] = 1;
  }
}
__global__ void k_u8_to_i64(int64_t n, const unsigned char* __restrict__ a, int64_t* o) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i];
}
// slot numbers (cube-major) from the exclusive scan of the marks; slot -> (cube, dir)
__global__ void k_number(int64_t n, int ndir, const unsigned char* __restrict__ mark, const int64_t* __restrict__ pos,
                         int64_t* slot, int64_t* scube, int32_t* sdir) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  if (!mark[e]) {
    slot[e] = -1;
    return;
  }
  const int64_t s = pos[e];
  slot[e] = s;
  scube[s] = e / ndir;
  sdir[s] = (int32_t)(e % ndir);
}
__global__ void k_pair_slots(int64_t np, const int64_t* __restrict__ roff, int64_t nruns, const int32_t* __restrict__ gdir,
                             const int32_t* __restrict__ b, const int32_t* __restrict__ c, int m, int ndir, int hf,
                             const int64_t* __restrict__ islot, const int64_t* __restrict__ oslot, int32_t* tgt,
                             int32_t* src) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  const int d = hf ? gdir[ld_run(roff, nruns, p)] : 0, t = hf ? ld_anti_dir(d, m) : 0;
  tgt[p] = (int32_t)islot[(int64_t)b[p] * ndir + t];
  src[p] = (int32_t)oslot[(int64_t)c[p] * ndir + d];
}

template <class T>
struct DBuf {  // device buffer freed on scope exit
  T* p = nullptr;
  explicit DBuf(size_t n) { lck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
  ~DBuf() { cudaFree(p); }
  DBuf(const DBuf&) = delete;
};
template <class T>
T* up(std::vector<void*>& keep, const std::vector<T>& v) {
  T* p = nullptr;
  lck(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)));
  keep.push_back(p);
  if (!v.empty()) lck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// device -> host copy of a large result: the destination pages are pinned for the copy (DMA at full PCIe
// rate instead of the staged pageable path)
void d2h_pinned(void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  const bool pinned = cudaHostRegister(dst, bytes, cudaHostRegisterDefault) == cudaSuccess;
  if (!pinned) cudaGetLastError();
  lck(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  if (pinned) cudaHostUnregister(dst);
}

// exclusive scan of n int64 values into out (n + 1 entries: out[n] = total)
void scan_i64(const int64_t* in, int64_t* out, int64_t n) {
  size_t tb = 0;
  lck(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n + 1));
  DBuf<char> tmp(tb);
  lck(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n + 1));
}

}  // namespace

static double ld_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::string build_lists_device(HostPlan& P) {
  std::vector<void*> keep;
  double t0 = ld_now(), t_tab = 0, t_p2p = 0, t_gen = 0, t_slots = 0, t_pairs = 0;
  auto lap = [&](double& acc) {
    cudaDeviceSynchronize();
    const double t = ld_now();
    acc += t - t0;
    t0 = t;
  };
  try {
    const int nlev = (int)P.levels.size();
    // ---- per-level cube tables on the device
    std::vector<DevLevelT> hl(nlev);
    for (int l = 0; l < nlev; ++l) {
      const Level& L = P.levels[l];
      const int64_t nc = (int64_t)L.cubes.size();
      std::vector<uint64_t> key(nc);
      std::vector<int64_t> ijk(3 * nc), pb(nc), pe(nc);
      std::vector<unsigned char> leaf(nc);
      std::vector<int32_t> child(8 * nc, -1);
      for (int64_t c = 0; c < nc; ++c) {
        const Cube& C = P.cubes[L.cubes[c]];
        key[c] = ld_key(C.ijk[0], C.ijk[1], C.ijk[2]);
        for (int d = 0; d < 3; ++d) ijk[3 * c + d] = C.ijk[d];
        pb[c] = C.pbeg, pe[c] = C.pend, leaf[c] = C.leaf;
        for (int o = 0; o < 8; ++o)
          if (C.child[o] >= 0) child[8 * c + o] = (int32_t)P.cubes[C.child[o]].local;
      }
      hl[l].nc = nc;
      hl[l].key = up(keep, key), hl[l].ijk = up(keep, ijk), hl[l].leaf = up(keep, leaf);
      hl[l].child = up(keep, child), hl[l].pbeg = up(keep, pb), hl[l].pend = up(keep, pe);
    }
    const DevLevelT* dlv = up(keep, hl);
    lap(t_tab);

    // ---- P2P lists
    {
      const int64_t nl = (int64_t)P.leaves.size();
      std::vector<int32_t> ll(nl);
      std::vector<int64_t> lloc(nl), lpb(nl);
      for (int64_t t = 0; t < nl; ++t) {
        const Cube& C = P.cubes[P.leaves[t]];
        ll[t] = C.level, lloc[t] = C.local, lpb[t] = C.pbeg;
      }
      const int32_t* dll = up(keep, ll);
      const int64_t *dloc = up(keep, lloc), *dpb = up(keep, lpb);
      DBuf<int64_t> cnt(nl + 1), ptr(nl + 1);
      lck(cudaMemset(cnt.p + nl, 0, sizeof(int64_t)));
      k_p2p_lists<<<ld_nb(nl), 256>>>(0, nl, dll, dloc, dlv, dpb, cnt.p, nullptr, nullptr);
      scan_i64(cnt.p, ptr.p, nl);
      int64_t tot = 0;
      lck(cudaMemcpy(&tot, ptr.p + nl, sizeof(int64_t), cudaMemcpyDeviceToHost));
      DBuf<int32_t> src(tot), srt(tot);
      k_p2p_lists<<<ld_nb(nl), 256>>>(1, nl, dll, dloc, dlv, dpb, nullptr, ptr.p, src.p);
      size_t tb = 0;
      lck(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, src.p, srt.p, (int64_t)tot, (int64_t)nl, ptr.p, ptr.p + 1));
      {
        DBuf<char> tmp(tb);
        lck(cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, src.p, srt.p, (int64_t)tot, (int64_t)nl, ptr.p, ptr.p + 1));
      }
      P.p2p_ptr.resize(nl + 1);
      std::vector<int32_t> hs(tot);
      lck(cudaMemcpy(P.p2p_ptr.data(), ptr.p, (nl + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost));
      lck(cudaMemcpy(hs.data(), srt.p, tot * sizeof(int32_t), cudaMemcpyDeviceToHost));
      P.p2p_src.assign(hs.begin(), hs.end());
    }
    lap(t_p2p);

    // ---- interaction lists, slots, M2L pairs, level by level
    P.lmin = -1;
    P.m2l_groups.clear(), P.m2l_tgt.clear(), P.m2l_src.clear();
    std::vector<unsigned char*> om(nlev, nullptr), im(nlev, nullptr);  // slot marks (device)
    std::vector<std::vector<void*>> lvl_keep(nlev);
    auto dalloc_keep = [&](int l, size_t bytes) {
      void* p = nullptr;
      lck(cudaMalloc(&p, std::max<size_t>(bytes, 1)));
      lvl_keep[l].push_back(p);
      return p;
    };
    for (int l = 0; l < nlev; ++l) {
      Level& L = P.levels[l];
      const int64_t nc = (int64_t)L.cubes.size();
      L.out_slot.assign(nc * L.ndir, -1);
      L.in_slot.assign(nc * L.ndir, -1);
      L.n_out = L.n_in = 0;
      L.out_cube.clear(), L.out_dir.clear(), L.in_cube.clear(), L.in_dir.clear();
      // pairs of level l (parents at l - 1)
      int64_t np = 0, nruns = 0;
      DBuf<uint64_t>* okey = nullptr;
      std::unique_ptr<DBuf<uint64_t>> okey_s, okey_o;
      std::unique_ptr<DBuf<int32_t>> oc_s, oc_o, bb;
      std::vector<uint32_t> rk;
      std::vector<int64_t> rcnt;
      int span = 0, D = 0;
      if (l >= 1) {
        const Level& Lp = P.levels[l - 1];
        const int Rp = Lp.R, Rc = L.R;
        span = (int)std::min<int64_t>(2 * Rp + 1, (1LL << l) - 1);
        D = 2 * span + 1;
        const int64_t npar = (int64_t)Lp.cubes.size();
        const int64_t w = 2 * Rp + 1;
        const bool brute = w * w * w > npar;
        const int64_t nq = brute ? npar : w * w * w;
        DBuf<int64_t> cnt(npar * nq + 1), off(npar * nq + 1);
        lck(cudaMemset(cnt.p + npar * nq, 0, sizeof(int64_t)));
        k_vlist<<<ld_nb(npar * nq), 256>>>(0, npar, nq, brute, hl[l - 1], Rp, Rc, span, D, cnt.p, nullptr, nullptr,
                                             nullptr);
        scan_i64(cnt.p, off.p, npar * nq);
        lck(cudaMemcpy(&np, off.p + npar * nq, sizeof(int64_t), cudaMemcpyDeviceToHost));
        if (np > 0) {
          okey_o.reset(new DBuf<uint64_t>(np));
          oc_o.reset(new DBuf<int32_t>(np));
          k_vlist<<<ld_nb(npar * nq), 256>>>(1, npar, nq, brute, hl[l - 1], Rp, Rc, span, D, nullptr, off.p,
                                               okey_o->p, oc_o->p);
          // sort by (offset key, target), stable: equal keys keep the generation order
          okey_s.reset(new DBuf<uint64_t>(np));
          oc_s.reset(new DBuf<int32_t>(np));
          int kb = 1;
          while ((1LL << kb) < (int64_t)D * D * D) ++kb;
          size_t tb = 0;
          lck(cub::DeviceRadixSort::SortPairs(nullptr, tb, okey_o->p, okey_s->p, oc_o->p, oc_s->p, np, 0, 32 + kb));
          {
            DBuf<char> tmp(tb);
            lck(cub::DeviceRadixSort::SortPairs(tmp.p, tb, okey_o->p, okey_s->p, oc_o->p, oc_s->p, np, 0, 32 + kb));
          }
          okey_o.reset(), oc_o.reset();
          okey = okey_s.get();
          DBuf<uint32_t> gk(np), uk(np);
          bb.reset(new DBuf<int32_t>(np));
          k_split_key<<<ld_nb(np), 256>>>(np, okey->p, gk.p, bb->p);
          DBuf<int64_t> rc(np), nr(1);
          tb = 0;
          lck(cub::DeviceRunLengthEncode::Encode(nullptr, tb, gk.p, uk.p, rc.p, nr.p, np));
          {
            DBuf<char> tmp(tb);
            lck(cub::DeviceRunLengthEncode::Encode(tmp.p, tb, gk.p, uk.p, rc.p, nr.p, np));
          }
          lck(cudaMemcpy(&nruns, nr.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
          rk.resize(nruns), rcnt.resize(nruns);
          lck(cudaMemcpy(rk.data(), uk.p, nruns * sizeof(uint32_t), cudaMemcpyDeviceToHost));
          lck(cudaMemcpy(rcnt.data(), rc.p, nruns * sizeof(int64_t), cudaMemcpyDeviceToHost));
          if (P.lmin < 0) P.lmin = l;
        }
      }
      lap(t_gen);
      const int lmin = P.lmin;
      if (lmin < 0 || l < lmin) continue;
      // groups: offsets and (HF) source wedges
      std::vector<int32_t> gdir(std::max<int64_t>(nruns, 1), 0);
      std::vector<std::array<int, 3>> goff(nruns);
      std::vector<int64_t> roff(nruns + 1, 0);
      for (int64_t r = 0; r < nruns; ++r) {
        const int kk = (int)rk[r];
        goff[r] = {kk / (D * D) - span, (kk / D) % D - span, kk % D - span};
        if (L.hf) {
          const double v[3] = {(double)goff[r][0], (double)goff[r][1], (double)goff[r][2]};
          gdir[r] = face_dir(v, L.m);
        }
        roff[r + 1] = roff[r] + rcnt[r];
      }
      const int32_t* dgdir = up(lvl_keep[l], gdir);
      const int64_t* droff = up(lvl_keep[l], roff);
      // slot marks
      const int64_t ne = nc * L.ndir;
      om[l] = (unsigned char*)dalloc_keep(l, ne);
      im[l] = (unsigned char*)dalloc_keep(l, ne);
      if (!L.hf) {
        lck(cudaMemset(om[l], 1, ne));
        lck(cudaMemset(im[l], 1, ne));
      } else {
        lck(cudaMemset(om[l], 0, ne));
        lck(cudaMemset(im[l], 0, ne));
        if (np > 0)
          k_mark_pairs<<<ld_nb(np), 256>>>(np, droff, nruns, dgdir, bb->p, oc_s->p, L.m, L.ndir, om[l], im[l]);
        if (l - 1 >= lmin && P.levels[l - 1].hf) {
          const Level& Lp = P.levels[l - 1];
          const int64_t npe = (int64_t)Lp.cubes.size() * Lp.ndir;
          k_mark_closure<<<ld_nb(npe), 256>>>((int64_t)Lp.cubes.size(), Lp.ndir, Lp.m, hl[l - 1].child, om[l - 1],
                                              im[l - 1], L.ndir, om[l], im[l]);
        }
      }
      // numbering (cube-major)
      DBuf<int64_t> oslot(ne), islot(ne);
      for (int io = 0; io < 2; ++io) {
        unsigned char* mk = io ? im[l] : om[l];
        DBuf<int64_t> m64(ne + 1), pos(ne + 1);
        lck(cudaMemset(m64.p + ne, 0, sizeof(int64_t)));
        k_u8_to_i64<<<ld_nb(ne), 256>>>(ne, mk, m64.p);
        scan_i64(m64.p, pos.p, ne);
        int64_t ns = 0;
        lck(cudaMemcpy(&ns, pos.p + ne, sizeof(int64_t), cudaMemcpyDeviceToHost));
        DBuf<int64_t> scube(ns);
        DBuf<int32_t> sdir(ns);
        int64_t* sl = io ? islot.p : oslot.p;
        k_number<<<ld_nb(ne), 256>>>(ne, L.ndir, mk, pos.p, sl, scube.p, sdir.p);
        std::vector<int64_t>& tab = io ? L.in_slot : L.out_slot;
        lck(cudaMemcpy(tab.data(), sl, ne * sizeof(int64_t), cudaMemcpyDeviceToHost));
        std::vector<int64_t>& vc = io ? L.in_cube : L.out_cube;
        std::vector<int>& vd = io ? L.in_dir : L.out_dir;
        std::vector<int32_t> hd(ns);
        vc.resize(ns);
        lck(cudaMemcpy(vc.data(), scube.p, ns * sizeof(int64_t), cudaMemcpyDeviceToHost));
        lck(cudaMemcpy(hd.data(), sdir.p, ns * sizeof(int32_t), cudaMemcpyDeviceToHost));
        vd.assign(hd.begin(), hd.end());
        (io ? L.n_in : L.n_out) = ns;
      }
      lap(t_slots);
      // M2L pairs -> (target in slot, source out slot), groups
      if (np > 0) {
        DBuf<int32_t> tg(np), sr(np);
        k_pair_slots<<<ld_nb(np), 256>>>(np, droff, nruns, dgdir, bb->p, oc_s->p, L.m, L.ndir, L.hf ? 1 : 0, islot.p,
                                         oslot.p, tg.p, sr.p);
        const int64_t base = (int64_t)P.m2l_tgt.size();
        P.m2l_tgt.resize(base + np), P.m2l_src.resize(base + np);
        d2h_pinned(P.m2l_tgt.data() + base, tg.p, np * sizeof(int32_t));
        d2h_pinned(P.m2l_src.data() + base, sr.p, np * sizeof(int32_t));
        for (int64_t r = 0; r < nruns; ++r) {
          HostPlan::M2LGroup G;
          G.level = l;
          G.off[0] = goff[r][0], G.off[1] = goff[r][1], G.off[2] = goff[r][2];
          G.dir = L.hf ? gdir[r] : 0;
          G.rank = -2;
          G.mat_off = 0;
          G.pbeg = base + roff[r], G.pend = base + roff[r + 1];
          P.m2l_groups.push_back(G);
        }
      }
      lap(t_pairs);
      // the parent level's marks are no longer needed
      if (l >= 1)
        for (void* p : lvl_keep[l - 1]) cudaFree(p);
      if (l >= 1) lvl_keep[l - 1].clear();
    }
    for (auto& v : lvl_keep)
      for (void* p : v) cudaFree(p);
    lck(cudaDeviceSynchronize());
    char buf[256];
    snprintf(buf, sizeof buf, "lists (device): tables %.3fs p2p %.3fs v-lists %.3fs slots %.3fs pairs %.3fs\n", t_tab,
             t_p2p, t_gen, t_slots, t_pairs);
    P.log += buf;
  } catch (const LdFail&) {
    for (void* p : keep) cudaFree(p);
    cudaGetLastError();
    return "CUDA";
  }
  for (void* p : keep) cudaFree(p);
  return "";
}

}  // namespace fda
