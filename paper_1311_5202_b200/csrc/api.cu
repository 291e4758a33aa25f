// api.cu -- the C ABI (include/fda.h): plan upload, apply orchestration, diagnostics.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/fda.h"
#include "kernels.cuh"
#include "plan.hpp"

using fda::cplx;

namespace {

struct DevLevel {
  int s = 0;
  int64_t n_out = 0, n_in = 0;
  double2* X = nullptr;
  double2* Y = nullptr;
  fda::GTrans m2l;   // H6 (groups of rank <= the warp-specialised kernel's limit, or all)
  fda::GTrans m2l2;  // H6, remaining groups (higher rank / dense), when the level is split
};
struct DevTrans {
  int lp = 0, sp = 0, sc = 0;
  fda::GTrans up;   // H5 M2M: child X -> parent X
  fda::GTrans dn;   // H7 L2L: parent Y -> child Y
};
struct DevLeafOps {
  int level = 0, s = 0, nsurf = 0;
  int64_t nleaves = 0;       // all leaves of the level (S2M)
  int64_t nleaves_own = 0;   // owned leaves (L2T)
  int32_t *leaf = nullptr, *leaf_own = nullptr;
  double* surf = nullptr;
  fda::GTrans s2m;           // H4 reduction: X[slot] += S chk[t]            (S = Sigma^-1 U^H, eq_cmps)
  fda::GTrans l2t;           // H8 reduction: rho[t'] += T Y[slot]           (T = conj(U) Sigma^-1, eq_cmpt)
};

}  // namespace

struct fda_plan_s {
  fda::HostPlan H;
  int dev = 0;
  cudaStream_t stream = 0;
  bool sticky_error = false;
  bool host_only = false;
  std::vector<void*> allocs;
  int64_t bytes = 0;
  // geometry
  int64_t n = 0, nleaf = 0;
  double *px, *py, *pz, *nx, *ny, *nz, *w;
  int32_t* perm;
  int64_t* leaf_ptr;
  double *lcx, *lcy, *lcz;
  int64_t *p2p_ptr;
  int32_t* p2p_src;
  double2 *q, *phim, *outm, *phi_buf, *out_buf;
  // ownership (multi-GPU)
  int nranks = 1;
  int kind = 0;  // FDA_KERNEL_BMH / FDA_KERNEL_BMG
  int64_t leaf_b = 0, leaf_e = 0, pt_b = 0, pt_e = 0;
  // correction
  int64_t nnz = 0;
  int64_t* c_ptr = nullptr;
  int32_t* c_col = nullptr;
  double2* c_val = nullptr;
  // far field
  std::vector<DevLevel> lv;
  std::vector<DevTrans> tr;
  std::vector<DevLeafOps> lo;
  double2* surfbuf = nullptr;  // check potentials (S2M) / equivalent densities (L2T) of one level's leaves
  int64_t surfbuf_n = 0;
  fda_stats st{};
  std::string logstr;
  int64_t last_launches = 0;  // kernels launched by the last apply
};

namespace {

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct CudaFail {
  fda_status s;
};

void ck(cudaError_t e) {
  if (e == cudaErrorMemoryAllocation) throw CudaFail{FDA_ERR_OOM};
  if (e != cudaSuccess) throw CudaFail{FDA_ERR_CUDA};
}

template <class T>
T* dalloc(fda_plan P, size_t count) {
  if (count == 0) count = 1;
  void* p = nullptr;
  ck(cudaMalloc(&p, count * sizeof(T)));
  P->allocs.push_back(p);
  P->bytes += (int64_t)(count * sizeof(T));
  return (T*)p;
}
template <class T>
T* upload(fda_plan P, const T* h, size_t count) {
  T* d = dalloc<T>(P, count);
  if (count) ck(cudaMemcpy(d, h, count * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}
template <class T>
T* upload(fda_plan P, const std::vector<T>& v) {
  return upload(P, v.data(), v.size());
}
int32_t* upload_i32(fda_plan P, const std::vector<int64_t>& v) {
  std::vector<int32_t> t(v.begin(), v.end());
  return upload(P, t);
}

// copy an input array (host or device) to a host vector
template <class T>
std::vector<T> to_host(const T* p, size_t count) {
  std::vector<T> h(count);
  if (!count) return h;
  if (is_device_ptr(p)) ck(cudaMemcpy(h.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost));
  else std::memcpy(h.data(), p, count * sizeof(T));
  return h;
}

void free_plan(fda_plan P) {
  for (void* p : P->allocs) cudaFree(p);
  P->allocs.clear();
}

// Pairs (out slot, in slot) in group-major order; each group one translation matrix.
struct GroupedPairs {
  std::vector<int64_t> gptr{0};
  std::vector<int64_t> out, in;
  std::vector<int32_t> rank;
  std::vector<int64_t> mat;
};

// Split the output slots into work items that own them exclusively (direction x Morton slab of
// cubes), so the grouped-translation kernel accumulates without atomics; each item walks its
// groups in order.  Slab count: enough pairs per (item, group) to amortise the matrix
// (>= ~32) and enough items to fill the GPU (>= 2 CTAs per SM).
// Append matrix A (M x K; element (i, j) = a(i, j)) in DMMA fragment order, padded to Mp x Kp
// (kernels.cuh GTrans): tiles (mt, kt) of 8 x 4, each 32 real parts in lane order then 32 imaginary.
template <class F>
void frag_append(std::vector<double>& out, int M, int K, int Mp, int Kp, F a) {
  for (int mt = 0; mt < Mp / 8; ++mt)
    for (int kt = 0; kt < Kp / 4; ++kt) {
      double re[32], im[32];
      for (int l = 0; l < 32; ++l) {
        const int i = mt * 8 + l / 4, j = kt * 4 + l % 4;
        const cplx v = (i < M && j < K) ? a(i, j) : cplx(0.0);
        re[l] = v.real(), im[l] = v.imag();
      }
      out.insert(out.end(), re, re + 32);
      out.insert(out.end(), im, im + 32);
    }
}
inline int pad8(int v) { return (v + 7) / 8 * 8; }
inline int pad4(int v) { return (v + 3) / 4 * 4; }

// Fragment-order pool of the groups' matrices.  raw: the plan's column-major pool; a dense group is
// s_out x s_in (ld s_out) at G.mat[g]; a low-rank group is U (s_out x r, ld s_out) then V (r x s_in, ld r).
// Rewrites G.mat to offsets (doubles) into the returned pool.
std::vector<double> frag_pool(GroupedPairs& G, const cplx* raw, int s_out, int s_in, int* rmax8, int64_t* mmax) {
  std::vector<double> pool;
  *rmax8 = 0;
  *mmax = 0;
  for (size_t g = 0; g < G.rank.size(); ++g) {
    const size_t before = pool.size();
    const cplx* A = raw + G.mat[g];
    const int r = G.rank[g];
    G.mat[g] = (int64_t)pool.size();
    if (r < 0) {
      frag_append(pool, s_out, s_in, pad8(s_out), pad4(s_in), [&](int i, int j) { return A[i + (int64_t)j * s_out]; });
    } else {
      const cplx* V = A + (int64_t)s_out * r;
      frag_append(pool, r, s_in, pad8(r), pad4(s_in), [&](int i, int j) { return V[i + (int64_t)j * r]; });
      frag_append(pool, s_out, r, pad8(s_out), pad8(r), [&](int i, int j) { return A[i + (int64_t)j * s_out]; });
      *rmax8 = std::max(*rmax8, pad8(r));
    }
    *mmax = std::max<int64_t>(*mmax, (int64_t)(pool.size() - before));
  }
  return pool;
}

fda::GTrans make_items(fda_plan P, GroupedPairs& G, const std::vector<int64_t>& out_cube,
                       const std::vector<int>& out_dir, int64_t ncubes, int s_out, int s_in, const cplx* raw) {
  fda::GTrans T;
  const int64_t ng = (int64_t)G.rank.size(), np = (int64_t)G.out.size();
  if (np == 0) return T;
  {
    int rmax8 = 0;
    int64_t mmax = 0;
    std::vector<double> pool = frag_pool(G, raw, s_out, s_in, &rmax8, &mmax);
    T.mmax = mmax;
    T.pool = upload(P, pool);
    T.rmax8 = rmax8;
    T.s_out = s_out, T.s_in = s_in;
    T.all_lowrank = 1;
    for (int32_t r : G.rank) T.all_lowrank &= (r >= 0);
    if (getenv("FDA_GT_CT1")) T.ct1 = atoi(getenv("FDA_GT_CT1"));
    if (getenv("FDA_GT_CT2")) T.ct2 = atoi(getenv("FDA_GT_CT2"));
  }
  const int cols = fda::gtrans_cols(T);
  std::unordered_map<int, int64_t> dix;
  for (int64_t p = 0; p < np; ++p) dix.emplace(out_dir[G.out[p]], (int64_t)dix.size());
  const int64_t nd = (int64_t)dix.size();
  const double ppg = (double)np / (double)std::max<int64_t>(ng, 1);
  // parallelism first (>= 8 items per SM), then ~2 chunks of pairs per (item, group) where the groups allow
  int64_t S = std::max<int64_t>((int64_t)(ppg / (2 * cols)), (8 * 148 + nd - 1) / nd);
  S = std::max<int64_t>(1, std::min<int64_t>({S, 4096, ncubes}));
  // FDA_GT_MODE=atomic|owned forces the item kind (experiments); FDA_GT_CHUNK: pairs per atomic item
  const char* gm = getenv("FDA_GT_MODE");
  // Default: group-major items of <= 1024 pairs with atomic accumulation (measured at config 5: 400 ms
  // apply vs 440 ms with the automatic choice and 509 ms with owned items only; 1024 vs 256 pairs:
  // 332 vs 336 ms).
  // pairs per atomic item: up to 1024, but enough items to give every SM ~16 CTAs over the launch
  const int64_t chunk = getenv("FDA_GT_CHUNK")
                            ? std::max(1, atoi(getenv("FDA_GT_CHUNK")))
                            : std::max<int64_t>(32, std::min<int64_t>(1024, (np / (16 * 148) + 31) / 32 * 32));
  const bool force_owned = gm && !strcmp(gm, "owned"), use_auto = gm && !strcmp(gm, "auto");
  if (!force_owned && (!use_auto || ppg / (double)S < 0.75 * cols)) {
    // Few pairs per group: owned items would reload each matrix for ~1 pair.  Group-major items
    // (chunks of <= 128 pairs of one group) reuse the matrix; outputs then need atomics.
    std::vector<int64_t> iptr{0}, igpb, igpe;
    std::vector<int32_t> igg, order;
    std::vector<double> cost;
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t p = G.gptr[g]; p < G.gptr[g + 1]; p += chunk) {
        const int64_t q = std::min<int64_t>(p + chunk, G.gptr[g + 1]);
        igg.push_back((int32_t)g), igpb.push_back(p), igpe.push_back(q);
        iptr.push_back((int64_t)igg.size());
        const int r = G.rank[g];
        cost.push_back((double)(q - p) * (r < 0 ? (double)s_out * s_in : (double)r * (s_out + s_in)));
        order.push_back((int32_t)order.size());
      }
    std::vector<int32_t> pout(G.out.begin(), G.out.end()), pin(G.in.begin(), G.in.end());
    // Launch order: by the first output slot of the item (pairs of a group are sorted by output slot,
    // slots are numbered in Morton order), so the items resident at any time cover a narrow Morton
    // window of targets -- their y rows and nearby x rows stay in L2 -- across all groups.
    // FDA_ITEM_ORDER=cost: largest item first (group-major).
    const char* io = getenv("FDA_ITEM_ORDER");
    if (io && !strcmp(io, "cost"))
      std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
    else
      std::stable_sort(order.begin(), order.end(),
                       [&](int32_t a, int32_t b) { return pout[igpb[a]] < pout[igpb[b]]; });
    T.n_items = (int64_t)order.size();
    T.item_order = upload(P, order);
    T.item_ptr = upload(P, iptr);
    T.ig_group = upload(P, igg);
    T.ig_pb = upload(P, igpb);
    T.ig_pe = upload(P, igpe);
    T.out = upload(P, pout);
    T.in = upload(P, pin);
    T.grank = upload(P, G.rank);
    T.gmat = upload(P, G.mat);
    T.s_out = s_out, T.s_in = s_in, T.atomic = 1;
    return T;
  }
  const int64_t nitems = nd * S;
  std::vector<int64_t> item(np);
  std::vector<int64_t> cnt(nitems + 1, 0);
  for (int64_t p = 0; p < np; ++p) {
    const int64_t o = G.out[p];
    item[p] = dix[out_dir[o]] * S + (out_cube[o] * S) / std::max<int64_t>(ncubes, 1);
    cnt[item[p] + 1]++;
  }
  for (int64_t i = 0; i < nitems; ++i) cnt[i + 1] += cnt[i];
  std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
  std::vector<int32_t> pout(np), pin(np), pg(np);
  for (int64_t g = 0; g < ng; ++g)
    for (int64_t p = G.gptr[g]; p < G.gptr[g + 1]; ++p) {
      const int64_t pos = fill[item[p]]++;
      pout[pos] = (int32_t)G.out[p];
      pin[pos] = (int32_t)G.in[p];
      pg[pos] = (int32_t)g;
    }
  std::vector<int64_t> iptr(nitems + 1, 0), igpb, igpe;
  std::vector<int32_t> igg;
  std::vector<double> cost(nitems, 0.0);
  for (int64_t i = 0; i < nitems; ++i) {
    for (int64_t p = cnt[i]; p < cnt[i + 1];) {
      int64_t q = p;
      while (q < cnt[i + 1] && pg[q] == pg[p]) ++q;
      igg.push_back(pg[p]);
      igpb.push_back(p);
      igpe.push_back(q);
      const int r = G.rank[pg[p]];
      cost[i] += (double)(q - p) * (r < 0 ? (double)s_out * s_in : (double)r * (s_out + s_in)) + 2000.0;
      p = q;
    }
    iptr[i + 1] = (int64_t)igg.size();
  }
  std::vector<int32_t> order;
  for (int64_t i = 0; i < nitems; ++i)
    if (cnt[i + 1] > cnt[i]) order.push_back((int32_t)i);
  // Launch order: largest item first (measured at config 5: 10-30% faster per M2L level than the
  // (direction, Morton slab) order, profiles/r01_m2l_order.md; FDA_ITEM_ORDER=morton selects the latter).
  const char* io = getenv("FDA_ITEM_ORDER");
  if (!(io && !strcmp(io, "morton")))
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
  T.n_items = (int64_t)order.size();
  T.item_order = upload(P, order);
  T.item_ptr = upload(P, iptr);
  T.ig_group = upload(P, igg);
  T.ig_pb = upload(P, igpb);
  T.ig_pe = upload(P, igpe);
  T.out = upload(P, pout);
  T.in = upload(P, pin);
  T.grank = upload(P, G.rank);
  T.gmat = upload(P, G.mat);
  T.s_out = s_out;
  T.s_in = s_in;
  return T;
}

// Ownership (multi-GPU): rank r of R owns the contiguous leaf range whose points
// start at or after floor(n r / R) and before floor(n (r+1) / R) (leaves are never split).
void set_ownership(fda_plan P, const fda_options& o) {
  const fda::HostPlan& H = P->H;
  const int64_t n = H.n, nl = (int64_t)H.leaves.size();
  std::vector<int64_t> lp(nl + 1, 0);
  for (int64_t t = 0; t < nl; ++t) lp[t] = H.cubes[H.leaves[t]].pbeg;
  lp[nl] = n;
  const int R = std::max(1, o.nranks), r = std::min(std::max(0, o.rank), R - 1);
  const int64_t pb = (n * r) / R, pe = (n * (r + 1)) / R;
  int64_t lb = std::lower_bound(lp.begin(), lp.begin() + nl, pb) - lp.begin();
  int64_t le = std::lower_bound(lp.begin(), lp.begin() + nl, pe) - lp.begin();
  if (r == R - 1) le = nl;
  if (r == 0) lb = 0;
  P->nranks = R;
  P->nleaf = nl;
  P->leaf_b = lb, P->leaf_e = le;
  P->pt_b = lp[lb], P->pt_e = lp[le];
  P->st.owned_begin = P->pt_b, P->st.owned_end = P->pt_e;
  P->st.owned_leaf_begin = lb, P->st.owned_leaf_end = le;
  P->st.n = n;
  P->st.nleaves = nl;
  P->st.nlevels = (int64_t)H.levels.size();
  P->st.lmin = H.lmin;
}

fda_status upload_plan(fda_plan P, const fda_options& o) {
  fda::HostPlan& H = P->H;
  const int64_t n = H.n;
  P->n = n;
  P->px = upload(P, H.px), P->py = upload(P, H.py), P->pz = upload(P, H.pz);
  P->nx = upload(P, H.nx), P->ny = upload(P, H.ny), P->nz = upload(P, H.nz);
  P->w = upload(P, H.w);
  P->perm = upload(P, H.perm);
  const int64_t nl = (int64_t)H.leaves.size();
  P->nleaf = nl;
  std::vector<int64_t> lp(nl + 1);
  std::vector<double> cx(nl), cy(nl), cz(nl);
  for (int64_t t = 0; t < nl; ++t) {
    const fda::Cube& c = H.cubes[H.leaves[t]];
    lp[t] = c.pbeg;
    lp[t + 1] = c.pend;
    const double wl = H.root_w / (double)(1LL << c.level);
    cx[t] = H.root_lo[0] + (c.ijk[0] + 0.5) * wl;
    cy[t] = H.root_lo[1] + (c.ijk[1] + 0.5) * wl;
    cz[t] = H.root_lo[2] + (c.ijk[2] + 0.5) * wl;
  }
  P->leaf_ptr = upload(P, lp);
  P->lcx = upload(P, cx), P->lcy = upload(P, cy), P->lcz = upload(P, cz);
  P->p2p_ptr = upload(P, H.p2p_ptr);
  P->p2p_src = upload_i32(P, H.p2p_src);
  P->q = dalloc<double2>(P, n), P->phim = dalloc<double2>(P, n), P->outm = dalloc<double2>(P, n);
  P->phi_buf = dalloc<double2>(P, n), P->out_buf = dalloc<double2>(P, n);
  const int R = P->nranks;
  auto owned_cube = [&](int64_t gid) {
    const fda::Cube& c = H.cubes[gid];
    return c.pend > P->pt_b && c.pbeg < P->pt_e;
  };
  // levels
  const int nlev = (int)H.levels.size();
  P->lv.assign(nlev, DevLevel());
  for (int l = 0; l < nlev; ++l) {
    const fda::Level& L = H.levels[l];
    DevLevel& D = P->lv[l];
    D.s = L.s, D.n_out = L.n_out, D.n_in = L.n_in;
    if (L.n_out) D.X = dalloc<double2>(P, (size_t)L.n_out * L.s);
    if (L.n_in) D.Y = dalloc<double2>(P, (size_t)L.n_in * L.s);
  }
  // M2L: pairs filtered to owned targets, grouped by offset, split into owned work items
  for (int l = 0; l < nlev; ++l) {
    const fda::Level& L = H.levels[l];
    GroupedPairs G;
    for (const auto& g : H.m2l_groups) {
      if (g.level != l) continue;
      const size_t b0 = G.out.size();
      for (int64_t p = g.pbeg; p < g.pend; ++p) {
        const int64_t ts = H.m2l_tgt[p];
        if (R > 1 && !owned_cube(L.cubes[L.in_cube[ts]])) continue;
        G.out.push_back(ts);
        G.in.push_back(H.m2l_src[p]);
      }
      if (G.out.size() == b0) continue;
      G.gptr.push_back((int64_t)G.out.size());
      G.rank.push_back(g.rank);
      G.mat.push_back(g.mat_off);
      const double np = (double)(G.out.size() - b0);
      P->st.m2l_pairs += (int64_t)np;
      P->st.m2l_groups += 1;
      P->st.m2l_lowrank_groups += g.rank >= 0;
      P->st.flops_m2l += np * (g.rank < 0 ? 8.0 * L.s * L.s : 16.0 * g.rank * L.s);
    }
    if (G.out.empty()) continue;
    // Groups whose rank fits the warp-specialised kernel's shared memory run there; the others (few,
    // the nearest offsets) go to a second launch of the general kernel.
    const int rlim = fda::gtrans_ws_rmax(L.s);
    GroupedPairs G1, G2;
    for (size_t g = 0; g < G.rank.size(); ++g) {
      GroupedPairs& D = (G.rank[g] >= 0 && G.rank[g] <= rlim) ? G1 : G2;
      for (int64_t q = G.gptr[g]; q < G.gptr[g + 1]; ++q) D.out.push_back(G.out[q]), D.in.push_back(G.in[q]);
      D.gptr.push_back((int64_t)D.out.size());
      D.rank.push_back(G.rank[g]);
      D.mat.push_back(G.mat[g]);
    }
    if (!G1.out.empty() && !G2.out.empty()) {
      P->lv[l].m2l = make_items(P, G1, L.in_cube, L.in_dir, (int64_t)L.cubes.size(), L.s, L.s, H.m2l_pool[l].data());
      P->lv[l].m2l2 = make_items(P, G2, L.in_cube, L.in_dir, (int64_t)L.cubes.size(), L.s, L.s, H.m2l_pool[l].data());
    } else {
      P->lv[l].m2l = make_items(P, G, L.in_cube, L.in_dir, (int64_t)L.cubes.size(), L.s, L.s, H.m2l_pool[l].data());
    }
  }
  // transitions: M2M items own parent out slots (groups = (dir, octant) matrices),
  // L2L items own child in slots (groups = the same matrices, transposed layout)
  for (const auto& T : H.trans) {
    DevTrans D;
    const fda::Level& Lp = H.levels[T.lp];
    const fda::Level& Lc = H.levels[T.lp + 1];
    D.lp = T.lp, D.sp = T.sp, D.sc = T.sc;
    const int64_t nmat = (int64_t)(T.pool.size() / std::max<size_t>(1, (size_t)T.sp * T.sc));
    auto grouped = [&](const std::vector<int64_t>& ptr, const std::vector<int64_t>& other,
                       const std::vector<int64_t>& mat) {
      // CSR by output slot -> group-major pairs
      GroupedPairs G;
      std::vector<int64_t> cnt(nmat + 1, 0);
      for (int64_t m : mat) cnt[T.mat_index[m] + 1]++;
      for (int64_t g = 0; g < nmat; ++g) cnt[g + 1] += cnt[g];
      G.out.assign(other.size(), 0);
      G.in.assign(other.size(), 0);
      std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
      for (int64_t s = 0; s + 1 < (int64_t)ptr.size(); ++s)
        for (int64_t e = ptr[s]; e < ptr[s + 1]; ++e) {
          const int64_t pos = fill[T.mat_index[mat[e]]]++;
          G.out[pos] = s;
          G.in[pos] = other[e];
        }
      for (int64_t g = 0; g < nmat; ++g) {
        G.gptr.push_back(cnt[g + 1]);
        G.rank.push_back(-1);
        G.mat.push_back(g * (int64_t)T.sp * T.sc);
      }
      return G;
    };
    if (!T.up_child.empty()) {
      GroupedPairs G = grouped(T.up_ptr, T.up_child, T.up_mat);
      D.up = make_items(P, G, Lp.out_cube, Lp.out_dir, (int64_t)Lp.cubes.size(), T.sp, T.sc, T.pool.data());
    }
    if (!T.dn_parent.empty()) {
      GroupedPairs G = grouped(T.dn_ptr, T.dn_parent, T.dn_mat);
      D.dn = make_items(P, G, Lc.in_cube, Lc.in_dir, (int64_t)Lc.cubes.size(), T.sc, T.sp, T.poolT.data());
    }
    P->st.flops_m2m += 8.0 * T.sp * T.sc * (double)T.up_child.size();
    P->st.flops_l2l += 8.0 * T.sp * T.sc * (double)T.dn_parent.size();
    P->tr.push_back(D);
  }
  // leaf operators
  for (const auto& O : H.leafops) {
    const fda::Level& L = H.levels[O.level];
    DevLeafOps D;
    D.level = O.level, D.s = L.s, D.nsurf = L.nsurf;
    D.nleaves = (int64_t)O.leaf.size();
    D.leaf = upload_i32(P, O.leaf);
    std::vector<int64_t> lo_, so_;
    for (size_t t = 0; t < O.leaf.size(); ++t)
      if (O.leaf[t] >= P->leaf_b && O.leaf[t] < P->leaf_e) lo_.push_back(O.leaf[t]), so_.push_back(O.slot[t]);
    D.nleaves_own = (int64_t)lo_.size();
    D.leaf_own = upload_i32(P, lo_);
    std::vector<double> sf;
    for (const auto& p : L.ck_pts) sf.insert(sf.end(), {p[0], p[1], p[2]});
    D.surf = upload(P, sf);
    {  // S2M reduction: pairs (out = leaf slot, in = leaf row t of the check-potential buffer)
      GroupedPairs G;
      G.out = O.slot;
      G.in.resize(O.leaf.size());
      for (size_t t = 0; t < O.leaf.size(); ++t) G.in[t] = (int64_t)t;
      G.gptr.push_back((int64_t)G.out.size());
      G.rank.push_back(-1);
      G.mat.push_back(0);
      D.s2m = make_items(P, G, L.out_cube, L.out_dir, (int64_t)L.cubes.size(), L.s, L.nsurf, O.S.data());
    }
    if (!lo_.empty()) {  // L2T reduction: pairs (out = owned leaf row t', in = leaf slot)
      GroupedPairs G;
      G.in = so_;
      G.out.resize(lo_.size());
      std::vector<int64_t> oc(lo_.size());
      for (size_t t = 0; t < lo_.size(); ++t) G.out[t] = (int64_t)t, oc[t] = L.in_cube[so_[t]];
      std::vector<int> od(lo_.size(), 0);
      G.gptr.push_back((int64_t)G.out.size());
      G.rank.push_back(-1);
      G.mat.push_back(0);
      D.l2t = make_items(P, G, oc, od, (int64_t)L.cubes.size(), L.nsurf, L.s, O.T.data());
    }
    P->surfbuf_n = std::max(P->surfbuf_n, (int64_t)O.leaf.size() * L.nsurf);
    for (int64_t t = 0; t < D.nleaves; ++t) {
      const double npt = (double)(lp[O.leaf[t] + 1] - lp[O.leaf[t]]);
      P->st.flops_s2m += npt * L.nsurf * 40.0 + 8.0 * L.s * L.nsurf;
    }
    for (size_t t = 0; t < lo_.size(); ++t) {
      const double npt = (double)(lp[lo_[t] + 1] - lp[lo_[t]]);
      P->st.flops_l2t += npt * L.nsurf * 45.0 + 8.0 * L.s * L.nsurf;
    }
    P->lo.push_back(D);
  }
  if (P->surfbuf_n) P->surfbuf = dalloc<double2>(P, (size_t)P->surfbuf_n);
  // stats
  fda_stats& s = P->st;
  s.n = n;
  s.nleaves = nl;
  s.nlevels = nlev;
  s.lmin = H.lmin;
  s.p2p_leaf_pairs = (int64_t)H.p2p_src.size();
  for (int64_t t = P->leaf_b; t < P->leaf_e; ++t)
    for (int64_t e = H.p2p_ptr[t]; e < H.p2p_ptr[t + 1]; ++e)
      s.p2p_point_pairs += (lp[t + 1] - lp[t]) * (lp[H.p2p_src[e] + 1] - lp[H.p2p_src[e]]);
  s.flops_p2p = 100.0 * (double)s.p2p_point_pairs;
  for (int l = 0; l < nlev; ++l) s.out_slots += H.levels[l].n_out, s.in_slots += H.levels[l].n_in;
  s.owned_begin = P->pt_b, s.owned_end = P->pt_e;
  s.setup_tree_s = H.t_tree, s.setup_lists_s = H.t_lists, s.setup_ops_s = H.t_ops;
  return FDA_OK;
}

bool finite3(const std::vector<double>& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

}  // namespace

extern "C" {

void fda_options_default(fda_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  fda::Options d;
  o->leaf_size = 0;
  o->eps_internal = 0;
  o->lf_p_low = d.lf_p_low;
  o->lf_p_high = d.lf_p_high;
  o->lf_p_switch = d.lf_p_switch;
  o->lowrank = 1;
  o->single_leaf = 0;
  o->hf_max_rows = d.hf_max_rows;
  o->hf_spacing = d.hf_spacing;
  o->rank = 0;
  o->nranks = 1;
  o->verbose = 0;
}

const char* fda_status_str(fda_status s) {
  switch (s) {
    case FDA_OK: return "FDA_OK";
    case FDA_ERR_INVALID_ARG: return "FDA_ERR_INVALID_ARG";
    case FDA_ERR_COINCIDENT_POINTS: return "FDA_ERR_COINCIDENT_POINTS";
    case FDA_ERR_ALIAS: return "FDA_ERR_ALIAS";
    case FDA_ERR_CUDA: return "FDA_ERR_CUDA";
    case FDA_ERR_OOM: return "FDA_ERR_OOM";
    case FDA_ERR_SETUP_ACCURACY: return "FDA_ERR_SETUP_ACCURACY";
    case FDA_ERR_NCCL: return "FDA_ERR_NCCL";
    case FDA_ERR_STATE: return "FDA_ERR_STATE";
  }
  return "FDA_ERR_UNKNOWN";
}

fda_status fda_plan_create_ex(int64_t n, const double* points, const double* normals, const double* quad_weights,
                              double k, double alpha_re, double alpha_im, double eps, const fda_options* opt,
                              fda_plan* out) {
  if (!out) return FDA_ERR_INVALID_ARG;
  *out = nullptr;
  if (n < 1 || !points || !normals || !quad_weights) return FDA_ERR_INVALID_ARG;
  if (!std::isfinite(k) || k < 0 || !std::isfinite(alpha_re) || !std::isfinite(alpha_im)) return FDA_ERR_INVALID_ARG;
  if (k == 0 && (alpha_re != 0 || alpha_im != 0)) return FDA_ERR_INVALID_ARG;
  if (!(eps >= 1e-10 && eps <= 1e-1)) return FDA_ERR_INVALID_ARG;
  if (n > (int64_t)INT32_MAX) return FDA_ERR_INVALID_ARG;
  fda_options o;
  fda_options_default(&o);
  if (opt) o = *opt;
  int ndev = 0;
  if (!o.host_only && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)) {
    cudaGetLastError();
    return FDA_ERR_CUDA;
  }
  std::unique_ptr<fda_plan_s> P(new fda_plan_s());
  try {
    if (!o.host_only) cudaGetDevice(&P->dev);
    std::vector<double> x = to_host(points, (size_t)n * 3), nr = to_host(normals, (size_t)n * 3),
                        w = to_host(quad_weights, (size_t)n);
    if (!finite3(x) || !finite3(nr) || !finite3(w)) return FDA_ERR_INVALID_ARG;
    for (int64_t i = 0; i < n; ++i) {
      const double nn = std::sqrt(nr[3 * i] * nr[3 * i] + nr[3 * i + 1] * nr[3 * i + 1] + nr[3 * i + 2] * nr[3 * i + 2]);
      if (std::fabs(nn - 1.0) > 1e-10 || !(w[i] > 0)) return FDA_ERR_INVALID_ARG;
    }
    fda::Options fo;
    fo.np = o.leaf_size;
    fo.eps_int = o.eps_internal;
    fo.eps_lr = o.eps_lowrank;
    if (o.lf_p_low > 1) fo.lf_p_low = o.lf_p_low;
    if (o.lf_p_high > 1) fo.lf_p_high = o.lf_p_high;
    if (o.lf_p_switch > 0) fo.lf_p_switch = o.lf_p_switch;
    fo.lowrank = o.lowrank;
    fo.single_leaf = o.single_leaf;
    if (o.hf_max_rows > 0) fo.hf_max_rows = o.hf_max_rows;
    if (o.hf_spacing > 0) fo.hf_spacing = o.hf_spacing;
    fo.verbose = o.verbose;
    std::string err = fda::build_plan(P->H, n, x.data(), nr.data(), w.data(), k, cplx(alpha_re, alpha_im), eps, fo);
    if (err == "COINCIDENT_POINTS") return FDA_ERR_COINCIDENT_POINTS;
    if (!err.empty()) return FDA_ERR_INVALID_ARG;
    P->host_only = o.host_only != 0;
    P->logstr = P->H.log;
    set_ownership(P.get(), o);
    if (o.kernel != FDA_KERNEL_BMH && o.kernel != FDA_KERNEL_BMG && o.kernel != FDA_KERNEL_T1) return FDA_ERR_INVALID_ARG;
    P->kind = o.kernel;
    if (P->host_only) {
      *out = P.release();
      return FDA_OK;
    }
    const double t0 = now();
    fda_status s = upload_plan(P.get(), o);
    if (s != FDA_OK) {
      free_plan(P.get());
      return s;
    }
    ck(cudaDeviceSynchronize());
    P->st.setup_upload_s = now() - t0;
    P->st.device_bytes = P->bytes;
    P->logstr = P->H.log;
    // the host copies of the big pools are no longer needed
    std::vector<std::vector<cplx>>().swap(P->H.m2l_pool);
    for (auto& T : P->H.trans) std::vector<cplx>().swap(T.pool), std::vector<cplx>().swap(T.poolT);
  } catch (const CudaFail& f) {
    free_plan(P.get());
    cudaGetLastError();
    return f.s;
  } catch (const std::bad_alloc&) {
    free_plan(P.get());
    return FDA_ERR_OOM;
  }
  *out = P.release();
  return FDA_OK;
}

fda_status fda_plan_create(int64_t n, const double* points, const double* normals, const double* quad_weights,
                           double k, double alpha_re, double alpha_im, double eps, fda_plan* out) {
  return fda_plan_create_ex(n, points, normals, quad_weights, k, alpha_re, alpha_im, eps, nullptr, out);
}

fda_status fda_plan_set_stream(fda_plan P, void* stream) {
  if (!P) return FDA_ERR_INVALID_ARG;
  P->stream = (cudaStream_t)stream;
  return FDA_OK;
}

fda_status fda_plan_set_correction(fda_plan P, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                                   const double* val) {
  if (!P) return FDA_ERR_INVALID_ARG;
  if (P->host_only) return FDA_ERR_STATE;
  if (P->sticky_error) return FDA_ERR_CUDA;
  if (nnz < 0) return FDA_ERR_INVALID_ARG;
  if (nnz > 0 && (!row_ptr || !col || !val)) return FDA_ERR_INVALID_ARG;
  try {
    if (P->c_ptr) {
      // release the old correction
      for (void* p : {(void*)P->c_ptr, (void*)P->c_col, (void*)P->c_val}) {
        auto it = std::find(P->allocs.begin(), P->allocs.end(), p);
        if (it != P->allocs.end()) P->allocs.erase(it);
        cudaFree(p);
      }
      P->c_ptr = nullptr, P->c_col = nullptr, P->c_val = nullptr, P->nnz = 0;
    }
    if (nnz == 0) return FDA_OK;
    const int64_t n = P->n;
    std::vector<int64_t> rp = to_host(row_ptr, (size_t)n + 1);
    if (rp[0] != 0 || rp[n] != nnz) return FDA_ERR_INVALID_ARG;
    for (int64_t i = 0; i < n; ++i)
      if (rp[i + 1] < rp[i]) return FDA_ERR_INVALID_ARG;
    std::vector<int32_t> cl = to_host(col, (size_t)nnz);
    for (int64_t p = 0; p < nnz; ++p)
      if (cl[p] < 0 || cl[p] >= n) return FDA_ERR_INVALID_ARG;
    std::vector<double> vl = to_host(val, (size_t)nnz * 2);
    // permute into Morton order: row m = caller row perm[m]; columns through the inverse permutation
    const std::vector<int32_t>& perm = P->H.perm;
    std::vector<int32_t> inv(n);
    for (int64_t m = 0; m < n; ++m) inv[perm[m]] = (int32_t)m;
    std::vector<int64_t> mp(n + 1, 0);
    for (int64_t m = 0; m < n; ++m) mp[m + 1] = mp[m] + (rp[perm[m] + 1] - rp[perm[m]]);
    std::vector<int32_t> mc(nnz);
    std::vector<double> mv((size_t)nnz * 2);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t m = 0; m < n; ++m) {
      const int64_t i = perm[m];
      int64_t o = mp[m];
      for (int64_t p = rp[i]; p < rp[i + 1]; ++p, ++o) {
        mc[o] = inv[cl[p]];
        mv[2 * o] = vl[2 * p];
        mv[2 * o + 1] = vl[2 * p + 1];
      }
    }
    P->c_ptr = upload(P, mp);
    P->c_col = upload(P, mc);
    P->c_val = upload(P, reinterpret_cast<const double2*>(mv.data()), (size_t)nnz);
    P->nnz = nnz;
    P->st.csr_nnz = nnz;
    int64_t own = mp[P->pt_e] - mp[P->pt_b];
    P->st.bytes_csr = 20.0 * (double)own + 48.0 * (double)(P->pt_e - P->pt_b);
    P->st.device_bytes = P->bytes;
  } catch (const CudaFail& f) {
    P->sticky_error = true;
    return f.s;
  } catch (const std::bad_alloc&) {
    return FDA_ERR_OOM;
  }
  return FDA_OK;
}

static fda_status apply_impl(fda_plan P, uint32_t mask, const double* phi, double* out, float* phase_ms) {
  if (!P || !phi || !out) return FDA_ERR_INVALID_ARG;
  if (P->host_only) return FDA_ERR_STATE;
  if (P->sticky_error) return FDA_ERR_CUDA;
  if ((const void*)phi == (const void*)out) return FDA_ERR_ALIAS;
  const int64_t n = P->n;
  cudaStream_t st = P->stream;
  const bool dphi = is_device_ptr(phi), dout = is_device_ptr(out);
  if (phase_ms && (!dphi || !dout)) return FDA_ERR_INVALID_ARG;
  try {
    const double2* d_phi = reinterpret_cast<const double2*>(phi);
    double2* d_out = reinterpret_cast<double2*>(out);
    if (!dphi) {
      ck(cudaMemcpyAsync(P->phi_buf, phi, (size_t)n * sizeof(double2), cudaMemcpyHostToDevice, st));
      d_phi = P->phi_buf;
    }
    if (!dout) d_out = P->out_buf;
    cudaEvent_t ev[10];
    if (phase_ms)
      for (int i = 0; i < 10; ++i) ck(cudaEventCreate(&ev[i]));
    auto mark = [&](int i) {
      if (phase_ms) ck(cudaEventRecord(ev[i], st));
    };
    fda::Points Pt{P->px, P->py, P->pz, P->nx, P->ny, P->nz, P->w};
    fda::LeafGeom Lg{P->leaf_ptr, P->lcx, P->lcy, P->lcz};
    const double k = P->H.k;
    const double2 alpha = make_double2(P->H.alpha.real(), P->H.alpha.imag());
    mark(0);
    fda::launch_permute_scale(n, P->perm, P->w, d_phi, P->q, P->phim, st);
    mark(1);
    const bool partial = P->leaf_b > 0 || P->leaf_e < P->nleaf;
    if (!(mask & FDA_PHASE_NEAR) || partial) ck(cudaMemsetAsync(P->outm, 0, (size_t)n * sizeof(double2), st));
    if (mask & FDA_PHASE_NEAR)
      fda::launch_p2p(P->kind, P->leaf_e - P->leaf_b, P->leaf_ptr, P->p2p_ptr, P->p2p_src, Pt, P->q, k, alpha, P->outm,
                      P->leaf_b, st);
    mark(2);
    if ((mask & FDA_PHASE_CORR) && P->nnz > 0)
      fda::launch_csr(P->pt_b, P->pt_e, P->c_ptr, P->c_col, P->c_val, P->phim, P->outm, st);
    mark(3);
    const bool far = (mask & FDA_PHASE_FAR) && P->H.lmin >= 0;
    // FDA_TRACE=1: synchronise after every far-field launch and print its wall time (diagnostics only)
    static const bool trace = getenv("FDA_TRACE") != nullptr;
    double tlast = now();
    auto tr = [&](const char* what, int l) {
      if (!trace) return;
      ck(cudaStreamSynchronize(st));
      const double t = now();
      fprintf(stderr, "[fda trace] %-4s level %d  %.3f ms\n", what, l, 1e3 * (t - tlast));
      tlast = t;
    };
    if (far) {
      tr("pre", -1);
      // M2M accumulates into the non-leaf slots: clear every level's outgoing expansions first
      for (auto& D : P->lv)
        if (D.n_out) ck(cudaMemsetAsync(D.X, 0, (size_t)D.n_out * D.s * sizeof(double2), st));
      for (const auto& O : P->lo) {
        fda::launch_s2m_check(P->kind, O.nleaves, O.leaf, Lg, Pt, P->q, O.surf, O.nsurf, k, alpha, P->surfbuf, st);
        fda::launch_gtrans(O.s2m, P->surfbuf, P->lv[O.level].X, st);
        tr("s2m", O.level);
      }
    }
    mark(4);
    if (far) {
      for (int t = (int)P->tr.size() - 1; t >= 0; --t) {
        const DevTrans& T = P->tr[t];
        fda::launch_gtrans(T.up, P->lv[T.lp + 1].X, P->lv[T.lp].X, st);
        tr("m2m", T.lp);
      }
    }
    mark(5);
    if (far) {
      for (auto& D : P->lv)
        if (D.n_in) ck(cudaMemsetAsync(D.Y, 0, (size_t)D.n_in * D.s * sizeof(double2), st));
      for (size_t l = 0; l < P->lv.size(); ++l) {
        fda::launch_gtrans(P->lv[l].m2l, P->lv[l].X, P->lv[l].Y, st);
        fda::launch_gtrans(P->lv[l].m2l2, P->lv[l].X, P->lv[l].Y, st);
        if (P->lv[l].m2l.n_items) tr("m2l", (int)l);
      }
    }
    mark(6);
    if (far) {
      for (const auto& T : P->tr) {
        fda::launch_gtrans(T.dn, P->lv[T.lp].Y, P->lv[T.lp + 1].Y, st);
        tr("l2l", T.lp);
      }
    }
    mark(7);
    if (far) {
      for (const auto& O : P->lo) {
        if (!O.nleaves_own) continue;
        ck(cudaMemsetAsync(P->surfbuf, 0, (size_t)O.nleaves_own * O.nsurf * sizeof(double2), st));
        fda::launch_gtrans(O.l2t, P->lv[O.level].Y, P->surfbuf, st);
        // E_dn = G + alpha dG/dn_x (BM_H, BM_G: PAPER.md eq_eval2t); the Table-1 kernel has no target
        // derivative: E_dn = G
        const double2 alpha_dn = P->kind == FDA_KERNEL_T1 ? make_double2(0.0, 0.0) : alpha;
        fda::launch_l2t_eval(O.nleaves_own, O.leaf_own, Lg, Pt, O.surf, O.nsurf, k, alpha_dn, P->surfbuf, P->outm, st);
        tr("l2t", O.level);
      }
    }
    mark(8);
    fda::launch_unpermute(n, P->perm, P->outm, d_out, st);
    mark(9);
    ck(cudaGetLastError());
    {
      int64_t L = 3;  // permute, p2p, unpermute
      if ((mask & FDA_PHASE_CORR) && P->nnz > 0) ++L;
      if (far) {
        for (const auto& O : P->lo) L += 2 * (O.nleaves > 0) + 2 * (O.nleaves_own > 0);
        for (const auto& T : P->tr) L += (T.up.n_items > 0) + (T.dn.n_items > 0);
        for (const auto& D : P->lv) L += (D.m2l.n_items > 0) + (D.m2l2.n_items > 0);
      }
      P->last_launches = L;
    }
    if (!dout) {
      ck(cudaMemcpyAsync(out, d_out, (size_t)n * sizeof(double2), cudaMemcpyDeviceToHost, st));
      ck(cudaStreamSynchronize(st));
    }
    if (phase_ms) {
      ck(cudaEventSynchronize(ev[9]));
      for (int i = 0; i < 9; ++i) ck(cudaEventElapsedTime(&phase_ms[i], ev[i], ev[i + 1]));
      for (int i = 0; i < 10; ++i) cudaEventDestroy(ev[i]);
    }
  } catch (const CudaFail& f) {
    P->sticky_error = true;
    return f.s;
  }
  return FDA_OK;
}

fda_status fda_apply(fda_plan P, const double* phi, double* out) { return apply_impl(P, FDA_PHASE_ALL, phi, out, nullptr); }
fda_status fda_apply_phases(fda_plan P, uint32_t mask, const double* phi, double* out) {
  return apply_impl(P, mask, phi, out, nullptr);
}
fda_status fda_apply_timed(fda_plan P, uint32_t mask, const double* phi, double* out, float* phase_ms) {
  if (!phase_ms) return FDA_ERR_INVALID_ARG;
  return apply_impl(P, mask, phi, out, phase_ms);
}

fda_status fda_plan_stats(fda_plan P, fda_stats* s) {
  if (!P || !s) return FDA_ERR_INVALID_ARG;
  *s = P->st;
  return FDA_OK;
}

const char* fda_plan_log(fda_plan P) { return P ? P->logstr.c_str() : ""; }

int64_t fda_plan_launches(fda_plan P) { return P ? P->last_launches : -1; }

fda_status fda_plan_export_leaves(fda_plan P, int64_t* nleaves, int32_t* leaf_of_point, int32_t* leaf_level,
                                  int64_t* leaf_ijk) {
  if (!P || !nleaves) return FDA_ERR_INVALID_ARG;
  const fda::HostPlan& H = P->H;
  *nleaves = (int64_t)H.leaves.size();
  for (size_t t = 0; t < H.leaves.size(); ++t) {
    const fda::Cube& c = H.cubes[H.leaves[t]];
    if (leaf_of_point)
      for (int64_t m = c.pbeg; m < c.pend; ++m) leaf_of_point[H.perm[m]] = (int32_t)t;
    if (leaf_level) leaf_level[t] = c.level;
    if (leaf_ijk)
      for (int d = 0; d < 3; ++d) leaf_ijk[3 * t + d] = c.ijk[d];
  }
  return FDA_OK;
}

fda_status fda_plan_export_p2p(fda_plan P, int64_t* npairs, int32_t* tgt, int32_t* src) {
  if (!P || !npairs) return FDA_ERR_INVALID_ARG;
  const fda::HostPlan& H = P->H;
  *npairs = (int64_t)H.p2p_src.size();
  if (tgt && src) {
    for (size_t t = 0; t + 1 < H.p2p_ptr.size(); ++t)
      for (int64_t e = H.p2p_ptr[t]; e < H.p2p_ptr[t + 1]; ++e) tgt[e] = (int32_t)t, src[e] = (int32_t)H.p2p_src[e];
  }
  return FDA_OK;
}

fda_status fda_plan_export_m2l(fda_plan P, int64_t* npairs, int32_t* level, int64_t* tgt_ijk, int64_t* src_ijk) {
  if (!P || !npairs) return FDA_ERR_INVALID_ARG;
  const fda::HostPlan& H = P->H;
  *npairs = (int64_t)H.m2l_tgt.size();
  if (level && tgt_ijk && src_ijk) {
    for (const auto& G : H.m2l_groups) {
      const fda::Level& L = H.levels[G.level];
      for (int64_t p = G.pbeg; p < G.pend; ++p) {
        const fda::Cube& B = H.cubes[L.cubes[L.in_cube[H.m2l_tgt[p]]]];
        const fda::Cube& C = H.cubes[L.cubes[L.out_cube[H.m2l_src[p]]]];
        level[p] = G.level;
        for (int d = 0; d < 3; ++d) tgt_ijk[3 * p + d] = B.ijk[d], src_ijk[3 * p + d] = C.ijk[d];
      }
    }
  }
  return FDA_OK;
}

fda_status fda_plan_destroy(fda_plan P) {
  if (!P) return FDA_ERR_INVALID_ARG;
  free_plan(P);
  delete P;
  return FDA_OK;
}

}  // extern "C"
