// api.cu -- the C ABI (include/fda.h): plan upload, apply orchestration, diagnostics.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <map>
#include <unordered_map>
#include <vector>

#include "../../include/fda.h"
#include "kernels.cuh"
#include "nccl_dl.hpp"
#include "plan.hpp"
#include "plan_dev.cuh"
#include "lists_dev.cuh"
#include "tree_dev.cuh"

using fda::cplx;

// FP64 flops per kernel evaluation (P2P point pair; S2M / L2T surface evaluation) by operator kind
// (BM_H, BM_G, T1): (2 x DFMA + DADD + DMUL) thread instructions per evaluation, counted by ncu
// (smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum) over k_p2p / k_s2m_check / k_l2t_eval
// of a config-3 apply divided by the plan's evaluation counts (profiles/r02/ncu_alu_counts_c3.csv):
// BM_H P2P 109.8, S2M (dipole) 77.1, L2T 86.1.  The BM_G / T1 entries are estimates (not measured).
static const double FLOP_P2P[3] = {109.8, 75.0, 75.0};
static const double FLOP_S2M[3] = {77.1, 60.0, 86.1};
static const double FLOP_L2T = 86.1;

namespace {

struct DevLevel {
  int s = 0;
  int64_t n_out = 0, n_in = 0;
  double2* X = nullptr;  // = Xall + xoff of this level (all levels' outgoing expansions are one allocation)
  double2* Y = nullptr;
  fda::GTrans m2l;   // H6 (groups of rank <= the warp-specialised kernel's limit, or all)
  fda::GTrans m2l2;  // H6, remaining groups (higher rank / dense), when the level is split
  fda::BTrans m2lb;  // H6, low-rank groups (pad8(r) <= 24) with target-owned outputs (m2l_block.cu), launched first
};
struct DevTrans {
  int lp = 0, sp = 0, sc = 0;
  fda::GTrans up;   // H5 M2M: child X -> parent X
  fda::GTrans dn;   // H7 L2L: parent Y -> child Y
};
struct DevLeafOps {
  int level = 0, s = 0, nsurf = 0;
  int64_t nleaves_own = 0;   // owned leaves of the level (S2M and L2T)
  int32_t* leaf_own = nullptr;
  double* surf = nullptr;
  fda::GTrans s2m;           // H4 reduction: X[slot] += S chk[t]            (S = Sigma^-1 U^H, eq_cmps)
  fda::GTrans l2t;           // H8 reduction: rho[t'] += T Y[slot]           (T = conj(U) Sigma^-1, eq_cmpt)
  // stored leaf matrices (kernels.cuh launch_leafmat), null when not stored
  int64_t* pofs = nullptr;   // owned leaf t -> first row (point) of its matrices
  int32_t* slot = nullptr;   // owned leaf t -> its out (= in) slot
  double2* Sm = nullptr;     // rows per source point: S_leaf = Sigma^-1 U^H E_up
  double2* Tm = nullptr;     // rows per target point: T_leaf = E_dn conj(U) Sigma^-1
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
  double *px = nullptr, *py = nullptr, *pz = nullptr, *nx = nullptr, *ny = nullptr, *nz = nullptr, *w = nullptr;
  int32_t* perm = nullptr;
  int64_t* leaf_ptr;
  double *lcx, *lcy, *lcz;
  int64_t *p2p_ptr;
  int32_t* p2p_src;
  double2 *q, *phim, *outm, *phi_buf, *out_buf;
  // ownership (multi-GPU): rank q owns Morton leaves [rank_leaf[q], rank_leaf[q+1]) = points
  // [rank_pt[q], rank_pt[q+1])
  int nranks = 1, rank = 0;
  int kind = 0;  // FDA_KERNEL_BMH / FDA_KERNEL_BMG / FDA_KERNEL_T1
  int64_t leaf_b = 0, leaf_e = 0, pt_b = 0, pt_e = 0;
  std::vector<int64_t> rank_pt, rank_leaf;
  // expansion exchange: send entries (peer-major, (level, slot) ascending) and received partial sums
  struct Xchg {
    std::vector<std::vector<std::pair<int, int64_t>>> send, recv;  // per peer: (level, out slot)
    std::vector<int64_t> send_cnt, recv_cnt;                       // per peer, complex128 elements
    int64_t send_tot = 0, recv_tot = 0, nsend = 0, ndst = 0;
    int64_t *s_xoff = nullptr, *s_boff = nullptr, *d_xoff = nullptr, *d_rptr = nullptr, *d_roff = nullptr;
    int32_t *s_len = nullptr, *d_len = nullptr;
    double2 *sendbuf = nullptr, *recvbuf = nullptr;
  } xc;
  double2* Xall = nullptr;
  std::vector<int64_t> xoff;
  std::vector<fda::DevSet> dev_sets;  // point sets / factors of the device-built operators  // per level offset (complex128 elements) into Xall
  ncclComm_t comm = nullptr;  // fda_plan_create_dist
  cudaStream_t xstream = nullptr;
  cudaEvent_t ev_up = nullptr, ev_x = nullptr;
  cudaStream_t nstream = nullptr;  // near field (P2P, correction), concurrent with the far field
  cudaEvent_t ev_perm = nullptr, ev_near = nullptr;
  // CUDA graph of the apply's device-resident middle (near field, upward pass, M2L, L2L, L2T): captured once per
  // phase mask on the plan's capture stream, replayed on the caller's stream between the permute and the
  // unpermute (which take the caller's pointers).  fda_options.graph / FDA_GRAPH; single-rank plans.
  bool graph_on = false;
  bool deterministic = false;  // fda_options.deterministic: owned items everywhere, one-sided P2P
  cudaStream_t gstream = nullptr;
  std::map<uint32_t, cudaGraphExec_t> gexec;
  std::map<uint32_t, int> gcalls;  // applies per mask so far (the capture is the second one: lazy setup done)
  // correction
  int64_t nnz = 0;
  int64_t* c_ptr = nullptr;
  int32_t* c_col = nullptr;
  double2* c_val = nullptr;
  // far field
  std::vector<DevLevel> lv;
  std::vector<DevTrans> tr;
  std::vector<DevLeafOps> lo;
  double2* tbuf = nullptr;     // two-pass M2L: T = V X of one level's block groups (m2l_block.cu)
  int64_t tbuf_n = 0;          // complex128 elements (max over levels)
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
void drop_graphs(fda_plan P);

// FDA_DEBUG=1: report the failing call site on stderr
void ck_at(cudaError_t e, int line) {
  if (e == cudaSuccess) return;
  if (getenv("FDA_DEBUG")) fprintf(stderr, "fda: CUDA error %s at api.cu:%d\n", cudaGetErrorString(e), line);
  if (e == cudaErrorMemoryAllocation) throw CudaFail{FDA_ERR_OOM};
  throw CudaFail{FDA_ERR_CUDA};
}
#define ck(e) ck_at((e), __LINE__)

template <class T>
T* dalloc(fda_plan P, size_t count) {
  if (count == 0) count = 1;
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess && getenv("FDA_DEBUG"))
    fprintf(stderr, "fda: cudaMalloc of %zu bytes failed (plan holds %lld bytes)\n", count * sizeof(T),
            (long long)P->bytes);
  ck(e);
  P->allocs.push_back(p);
  P->bytes += (int64_t)(count * sizeof(T));
  return (T*)p;
}
template <class T>
T* upload(fda_plan P, const T* h, size_t count) {
  T* d = dalloc<T>(P, count);
  if (!count) return d;
  // large host arrays: pin their pages for the copy (DMA at full PCIe rate instead of the staged path)
  const size_t bytes = count * sizeof(T);
  const bool pin = bytes >= (64u << 20) &&
                   cudaHostRegister(const_cast<T*>(h), bytes, cudaHostRegisterReadOnly) == cudaSuccess;
  if (bytes >= (64u << 20) && !pin) cudaGetLastError();
  ck(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  if (pin) cudaHostUnregister(const_cast<T*>(h));
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
  std::vector<int32_t> out, in;
  std::vector<int32_t> rank;
  std::vector<int64_t> mat;
  std::vector<int16_t> so, si;  // optional: the group's own output / input expansion lengths
};

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

// Fragment-order size (doubles) of a group's operator: dense s_out x s_in, or V (r x s_in) then U (s_out x r).
int64_t frag_size(int rank, int s_out, int s_in) {
  if (rank < 0) return (int64_t)(pad8(s_out) / 8) * (pad4(s_in) / 4) * 64;
  return (int64_t)(pad8(rank) / 8) * (pad4(s_in) / 4) * 64 + (int64_t)(pad8(s_out) / 8) * (pad8(rank) / 4) * 64;
}

// Operators shared by symmetry (HF levels).  The point sets of wedge d are g_d applied to the sets of its
// orbit representative ("obtained by rotation ... R_up^+ remain the same"; g_d = dir_sym[d],
// a signed coordinate permutation M_d).  The M2L group (offset delta, source wedge d, target wedge t) has
//   K[i][j] = G(|delta w + M_t a_i - M_d b_j|) = G(|M_d^T delta w + (M_d^T M_t) a_i - b_j|)
// (a: target representative's points, b: source representative's), and both reduced bases are the
// representatives' (R16), so K~ depends only on (rep t, rep d, M_d^T delta, M_d^T M_t): groups with
// the same key have the same operator, which is built and stored once and applied to the union of their
// pairs.  LF levels: one point set for every offset, so no sharing.  FDA_M2L_NOSHARE=1 disables it.
// Returns, per group q of lg, the first q' with the same key (q itself if none).
std::vector<int32_t> m2l_symmetry_classes(const fda::Level& L, const fda::HostPlan& H, const std::vector<int64_t>& lg,
                                          const std::vector<int64_t>& cnt) {
  std::vector<int32_t> cls(lg.size());
  for (size_t q = 0; q < lg.size(); ++q) cls[q] = (int32_t)q;
  if (!L.hf || L.dir_sym.empty() || (getenv("FDA_M2L_NOSHARE") && getenv("FDA_M2L_NOSHARE")[0] == '1')) return cls;
  auto mat = [](const fda::Sym& g, int M[3][3]) {  // (g v)_i = sign_i v_perm_i
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M[i][j] = (g.perm[i] == j) ? g.sign[i] : 0;
  };
  std::map<std::pair<uint64_t, uint64_t>, int32_t> first;
  for (size_t q = 0; q < lg.size(); ++q) {
    if (!cnt[q]) continue;
    const auto& g = H.m2l_groups[lg[q]];
    const int d = g.dir, t = fda::anti_dir(d, L.m);
    int Md[3][3], Mt[3][3];
    mat(L.dir_sym[d], Md), mat(L.dir_sym[t], Mt);
    const uint64_t reps = (uint64_t)L.dir_rep[d] << 32 | (uint64_t)(uint32_t)L.dir_rep[t];
    uint64_t key = 0;  // per axis: the offset component (16 bits) and a row of M_d^T M_t (3 trits): 3 x 21 bits
    for (int i = 0; i < 3; ++i) {
      int dp = 0;
      for (int k = 0; k < 3; ++k) dp += Md[k][i] * g.off[k];
      key = key * (1u << 16) + (uint64_t)(dp + 32768);
      for (int j = 0; j < 3; ++j) {
        int h = 0;
        for (int k = 0; k < 3; ++k) h += Md[k][i] * Mt[k][j];
        key = key * 3u + (uint64_t)(h + 1);
      }
    }
    cls[q] = first.emplace(std::make_pair(reps, key), (int32_t)q).first->second;
  }
  return cls;
}

fda::Points points_of(fda_plan P);
fda::LeafGeom leaves_of(fda_plan P);
double2 alpha_of(fda_plan P);

// Work items of a grouped translation.  raw != nullptr: the groups' matrices are the host column-major pool
// raw (G.mat offsets), converted to fragment order and uploaded; raw == nullptr: they are already in the
// device pool dpool in fragment order (G.mat = offsets in doubles, plan_dev.cu).
fda::GTrans make_items(fda_plan P, GroupedPairs& G, const std::vector<int64_t>& out_cube,
                       const std::vector<int>& out_dir, int64_t ncubes, int s_out, int s_in, const cplx* raw,
                       const double* dpool = nullptr, const char* mode = nullptr, int win = 0) {
  fda::GTrans T;
  const int64_t ng = (int64_t)G.rank.size(), np = (int64_t)G.out.size();
  if (np == 0) return T;
  {
    int rmax8 = 0;
    int64_t mmax = 0;
    if (raw) {
      std::vector<double> pool = frag_pool(G, raw, s_out, s_in, &rmax8, &mmax);
      T.pool = upload(P, pool);
    } else {
      for (int32_t r : G.rank) {
        if (r >= 0) rmax8 = std::max(rmax8, pad8(r));
        mmax = std::max<int64_t>(mmax, frag_size(r, s_out, s_in));
      }
      T.pool = dpool;
    }
    T.mmax = mmax;
    T.rmax8 = rmax8;
    T.s_out = s_out, T.s_in = s_in;
    T.all_lowrank = 1;
    for (int32_t r : G.rank) T.all_lowrank &= (r >= 0);
    if (getenv("FDA_GT_CT1")) T.ct1 = atoi(getenv("FDA_GT_CT1"));
    if (getenv("FDA_GT_CT2")) T.ct2 = atoi(getenv("FDA_GT_CT2"));
  }
  const int cols = fda::gtrans_cols(T);
  const double ppg = (double)np / (double)std::max<int64_t>(ng, 1);
  // FDA_GT_MODE=atomic|owned|auto forces the item kind (experiments); FDA_GT_CHUNK: pairs per atomic item
  const char* gm = P->deterministic ? "owned" : mode ? mode : getenv("FDA_GT_MODE");
  // Default: group-major items of <= 1024 pairs with atomic accumulation (measured at config 5: 400 ms
  // apply vs 440 ms with the automatic choice and 509 ms with owned items only; 1024 vs 256 pairs:
  // 332 vs 336 ms).
  // pairs per atomic item: up to 1024, but enough items to give every SM ~16 CTAs over the launch
  const int64_t chunk = getenv("FDA_GT_CHUNK")
                            ? std::max(1, atoi(getenv("FDA_GT_CHUNK")))
                            : std::max<int64_t>(32, std::min<int64_t>(1024, (np / (16 * 148) + 31) / 32 * 32));
  const bool force_owned = gm && !strcmp(gm, "owned"), use_auto = gm && !strcmp(gm, "auto");
  // owned items: (output direction) x (Morton slab of cubes); parallelism first (>= 8 items per SM), then
  // ~2 chunks of pairs per (item, group) where the groups allow
  std::unordered_map<int, int64_t> dix;
  int64_t S = 1;
  if (force_owned || use_auto) {
    for (int64_t p = 0; p < np; ++p) dix.emplace(out_dir[G.out[p]], (int64_t)dix.size());
    const int64_t nd = (int64_t)dix.size();
    S = std::max<int64_t>((int64_t)(ppg / (2 * cols)), (8 * 148 + nd - 1) / nd);
    // FDA_GT_SLABS=n: n Morton slabs per output direction (experiments)
    if (getenv("FDA_GT_SLABS")) S = std::max(1, atoi(getenv("FDA_GT_SLABS")) / (int)std::max<int64_t>(1, nd));
    S = std::max<int64_t>(1, std::min<int64_t>({S, 4096, ncubes}));
  }
  if (!force_owned && (!use_auto || ppg / (double)S < 0.75 * cols)) {
    // Few pairs per group: owned items would reload each matrix for ~1 pair.  Group-major items
    // (chunks of <= 128 pairs of one group) reuse the matrix; outputs then need atomics.
    std::vector<int64_t> iptr{0}, igpb, igpe;
    std::vector<int32_t> igg, order;
    std::vector<double> cost;
    // FDA_GT_WIN=W: items also end at the boundaries of W Morton windows of output cubes (equal cube
    // counts), so the items resident at any time touch the Y rows (and the nearby X rows) of ~one window
    // and those stay in L2 (experiment)
    const int64_t W = win > 0 ? win : getenv("FDA_GT_WIN") ? std::max(1, atoi(getenv("FDA_GT_WIN"))) : 1;
    auto win = [&](int64_t p) { return W == 1 ? 0 : (out_cube[G.out[p]] * W) / std::max<int64_t>(ncubes, 1); };
    std::vector<int64_t> iwin;
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t p = G.gptr[g], q; p < G.gptr[g + 1]; p = q) {
        q = std::min<int64_t>(p + chunk, G.gptr[g + 1]);
        if (W > 1) {
          const int64_t w0 = win(p);
          if (win(q - 1) != w0) q = std::partition_point(G.out.begin() + p, G.out.begin() + q, [&](int32_t o) {
                                      return (out_cube[o] * W) / std::max<int64_t>(ncubes, 1) == w0;
                                    }) - G.out.begin();
          iwin.push_back(w0);
        }
        igg.push_back((int32_t)g), igpb.push_back(p), igpe.push_back(q);
        iptr.push_back((int64_t)igg.size());
        const int r = G.rank[g];
        cost.push_back((double)(q - p) * (r < 0 ? (double)s_out * s_in : (double)r * (s_out + s_in)));
        order.push_back((int32_t)order.size());
      }
    const std::vector<int32_t>& pout = G.out;
    const std::vector<int32_t>& pin = G.in;
    // Launch order: by the first output slot of the item (pairs of a group are sorted by output slot,
    // slots are numbered in Morton order), so the items resident at any time cover a narrow Morton
    // window of targets -- their y rows and nearby x rows stay in L2 -- across all groups.
    // FDA_ITEM_ORDER=cost: largest item first (group-major).
    const char* io = getenv("FDA_ITEM_ORDER");
    if (io && !strcmp(io, "cost"))
      std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cost[a] > cost[b]; });
    else if (W > 1)  // window-major, then Morton (FDA_ITEM_ORDER=group: then the group, then Morton)
      std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
        if (iwin[a] != iwin[b]) return iwin[a] < iwin[b];
        if (io && !strcmp(io, "group") && igg[a] != igg[b]) return igg[a] < igg[b];
        return pout[igpb[a]] < pout[igpb[b]];
      });
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
    if (!G.so.empty()) T.gso = upload(P, G.so), T.gsi = upload(P, G.si);
    T.s_out = s_out, T.s_in = s_in, T.atomic = 1;
    return T;
  }
  const int64_t nitems = (int64_t)dix.size() * S;
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

// Split a group-major pair set into the groups pred(g) accepts and the others (order kept).
template <class F>
void split_groups(const GroupedPairs& G, F pred, GroupedPairs& A, GroupedPairs& B) {
  const size_t ng = G.rank.size();
  std::vector<char> ina(ng);
  std::vector<int64_t> dst(ng);
  int64_t oa = 0, ob = 0;
  for (size_t g = 0; g < ng; ++g) {
    ina[g] = pred(g) ? 1 : 0;
    GroupedPairs& D = ina[g] ? A : B;
    const int64_t n = G.gptr[g + 1] - G.gptr[g];
    D.gptr.push_back(D.gptr.back() + n);
    D.rank.push_back(G.rank[g]);
    D.mat.push_back(G.mat[g]);
    if (!G.so.empty()) D.so.push_back(G.so[g]), D.si.push_back(G.si[g]);
    dst[g] = ina[g] ? oa : ob;
    (ina[g] ? oa : ob) += n;
  }
  A.out.resize(oa), A.in.resize(oa), B.out.resize(ob), B.in.resize(ob);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t g = 0; g < (int64_t)ng; ++g) {
    GroupedPairs& D = ina[g] ? A : B;
    std::copy(G.out.begin() + G.gptr[g], G.out.begin() + G.gptr[g + 1], D.out.begin() + dst[g]);
    std::copy(G.in.begin() + G.gptr[g], G.in.begin() + G.gptr[g + 1], D.in.begin() + dst[g]);
  }
}

// Target blocks of a level's low-rank M2L groups (kernels.cuh BTrans).  The output slots that receive
// pairs are ordered by (direction, slot) -- slots are numbered cube-major in Morton order, so the slots of
// one direction are Morton-ordered -- and cut into blocks of <= bmax slots of one direction; the pairs of a
// block keep the group-major order of G (so they are sorted by group) and are cut into chunks of <= 32
// pairs of one group.  Blocks launch in the Morton order of their first cube (L2 window of X).
fda::BTrans make_blocks(fda_plan P, const GroupedPairs& G, const std::vector<int64_t>& out_cube,
                        const std::vector<int>& out_dir, int s_out, int s_in, const double* dpool) {
  fda::BTrans B;
  const int64_t np = (int64_t)G.out.size(), ng = (int64_t)G.rank.size();
  if (np == 0) return B;
  int rmax8 = 8;  // >= one row tile (rank-0 groups contribute nothing but keep their chunks)
  for (int32_t r : G.rank) rmax8 = std::max(rmax8, pad8(r));
  int bmax = fda::m2l_block_bmax(s_out, rmax8, fda::smem_optin_bytes());
  if (getenv("FDA_M2L_BMAX")) bmax = std::max(1, std::min(bmax, atoi(getenv("FDA_M2L_BMAX"))));
  if (bmax <= 0) {
    fprintf(stderr, "fda: target-block M2L: no block fits (s_out %d, rmax8 %d)\n", s_out, rmax8);
    throw CudaFail{FDA_ERR_SETUP_ACCURACY};
  }
  const int64_t nslot = (int64_t)out_dir.size();
  std::vector<int64_t> cnt(nslot, 0);
  for (int64_t p = 0; p < np; ++p) cnt[G.out[p]]++;
  std::vector<int32_t> act;
  for (int64_t sl = 0; sl < nslot; ++sl)
    if (cnt[sl]) act.push_back((int32_t)sl);
  std::stable_sort(act.begin(), act.end(), [&](int32_t a, int32_t b) { return out_dir[a] < out_dir[b]; });
  std::vector<int64_t> sptr{0};
  std::vector<int32_t> bslot, blk_of(nslot, -1);
  std::vector<uint8_t> loc_of(nslot, 0);
  for (size_t i = 0; i < act.size(); ++i) {
    const int32_t sl = act[i];
    const int64_t cur = (int64_t)bslot.size() - sptr.back();
    if (cur == bmax || (cur > 0 && out_dir[bslot.back()] != out_dir[sl])) sptr.push_back((int64_t)bslot.size());
    blk_of[sl] = (int32_t)(sptr.size() - 1);
    loc_of[sl] = (uint8_t)((int64_t)bslot.size() - sptr.back());
    bslot.push_back(sl);
  }
  sptr.push_back((int64_t)bslot.size());
  const int64_t nb = (int64_t)sptr.size() - 1;
  // pairs by block, stable: group-major inside each block
  std::vector<int64_t> bp(nb + 1, 0);
  for (int64_t p = 0; p < np; ++p) bp[blk_of[G.out[p]] + 1]++;
  for (int64_t b = 0; b < nb; ++b) bp[b + 1] += bp[b];
  std::vector<int64_t> fill(bp.begin(), bp.end() - 1);
  std::vector<int32_t> pg(np);
  std::vector<uint8_t> ploc(np);
  std::vector<int32_t> p1out(np);  // pass-1 pair (G order) -> pass-2 position
  for (int64_t g = 0; g < ng; ++g)
    for (int64_t p = G.gptr[g]; p < G.gptr[g + 1]; ++p) {
      const int32_t o = G.out[p];
      const int64_t q = fill[blk_of[o]]++;
      ploc[q] = loc_of[o], pg[q] = (int32_t)g, p1out[p] = (int32_t)q;
    }
  std::vector<int64_t> cptr(nb + 1, 0), chp;
  std::vector<int32_t> chg;
  std::vector<uint8_t> chl;
  for (int64_t b = 0; b < nb; ++b) {
    for (int64_t p = bp[b]; p < bp[b + 1];) {
      int64_t q = p;
      while (q < bp[b + 1] && pg[q] == pg[p] && q - p < 32) ++q;
      chp.push_back(p), chg.push_back(pg[p]);
      for (int64_t e = 0; e < 32; ++e) chl.push_back(p + e < q ? ploc[p + e] : (uint8_t)0);
      p = q;
    }
    cptr[b + 1] = (int64_t)chg.size();
  }
  chp.push_back(np);
  std::vector<int32_t> order(nb);
  for (int64_t b = 0; b < nb; ++b) order[b] = (int32_t)b;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    const int64_t ca = out_cube[bslot[sptr[a]]], cb = out_cube[bslot[sptr[b]]];
    return ca != cb ? ca < cb : out_dir[bslot[sptr[a]]] < out_dir[bslot[sptr[b]]];
  });
  // pass-1 items: (group, <= 512 consecutive pairs of G -- sorted by target slot within the group), launched
  // in the order of their first target: the items resident at any time read the x columns of a narrow Morton
  // window of sources (L2-resident), while each item reuses its staged V over its pairs
  std::vector<int32_t> itg0;
  std::vector<int64_t> itp0;
  for (int64_t g = 0; g < ng; ++g)
    for (int64_t p = G.gptr[g]; p < G.gptr[g + 1]; p += 512) itg0.push_back((int32_t)g), itp0.push_back(p);
  std::vector<int32_t> iord(itg0.size());
  for (size_t i = 0; i < iord.size(); ++i) iord[i] = (int32_t)i;
  std::stable_sort(iord.begin(), iord.end(), [&](int32_t a, int32_t b) { return G.out[itp0[a]] < G.out[itp0[b]]; });
  std::vector<int32_t> itg(iord.size());
  std::vector<int64_t> itp(iord.size() + 1);  // item i: pairs [itp[i], itp_end[i])
  std::vector<int64_t> ite(iord.size());
  for (size_t i = 0; i < iord.size(); ++i) {
    const int32_t k = iord[i];
    itg[i] = itg0[k], itp[i] = itp0[k];
    ite[i] = std::min<int64_t>(itp0[k] + 512, G.gptr[itg0[k] + 1]);
  }
  itp.pop_back();
  B.n_blocks = nb;
  B.n_chunks = (int64_t)chg.size();
  B.n_pairs = np;
  B.n_items1 = (int64_t)itg.size();
  B.blk_order = upload(P, order);
  B.blk_sptr = upload(P, sptr);
  B.blk_slot = upload(P, bslot);
  B.blk_cptr = upload(P, cptr);
  B.ch_ptr = upload(P, chp);
  B.ch_group = upload(P, chg);
  B.ch_loc = upload(P, chl);
  B.it_group = upload(P, itg);
  B.it_ptr = upload(P, itp);
  B.it_end = upload(P, ite);
  B.p1_in = upload(P, G.in);
  B.p1_out = upload(P, p1out);
  B.grank = upload(P, G.rank);
  B.gmat = upload(P, G.mat);
  B.pool = dpool;
  if (!G.so.empty()) B.gso = upload(P, G.so), B.gsi = upload(P, G.si);
  B.s_out = s_out, B.s_in = s_in, B.rmax8 = rmax8, B.bmax = bmax;
  B.ldt = fda::m2l_block_ldt(rmax8);
  return B;
}

// Ownership (multi-GPU): the leaves (Morton order) are cut into nranks contiguous ranges of
// about equal estimated work -- P2P point pairs x 100 flop + the M2L flops into every ancestor cube, shared
// among the cube's leaves by points + the leaf's S2M / L2T surface work.  Leaves are never
// split, so a rank owns whole leaves and the point range they span.
void set_ownership(fda_plan P, const fda_options& o) {
  const fda::HostPlan& H = P->H;
  const int64_t n = H.n, nl = (int64_t)H.leaves.size();
  std::vector<int64_t> lp(nl + 1, 0);
  for (int64_t t = 0; t < nl; ++t) lp[t] = H.cubes[H.leaves[t]].pbeg;
  lp[nl] = n;
  const int R = std::max(1, o.nranks), r = std::min(std::max(0, o.rank), R - 1);
  std::vector<int64_t> rl(R + 1, 0);
  rl[R] = nl;
  if (R > 1) {
    std::vector<double> cost(nl, 0.0);
    for (int64_t t = 0; t < nl; ++t) {
      double src = 0;
      for (int64_t e = H.p2p_ptr[t]; e < H.p2p_ptr[t + 1]; ++e) src += (double)(lp[H.p2p_src[e] + 1] - lp[H.p2p_src[e]]);
      const double nt = (double)(lp[t + 1] - lp[t]);
      const fda::Level& L = H.levels[H.cubes[H.leaves[t]].level];
      cost[t] = 100.0 * nt * src + 2.0 * (40.0 * nt * L.nsurf + 8.0 * L.s * L.nsurf);
    }
    // M2L flops per target cube (global cube id), spread over the cube's leaves by points
    std::vector<double> cf(H.cubes.size(), 0.0);
    for (const auto& g : H.m2l_groups) {
      const fda::Level& L = H.levels[g.level];
      // device-built operators have no rank yet (-2): estimate r = s / 6 (config 5 measures 13-15 at s = 58-136)
      const double r = g.rank == -2 ? L.s / 6.0 : g.rank;
      const double f = g.rank == -1 ? 8.0 * L.s * L.s : 16.0 * r * L.s;
      for (int64_t p = g.pbeg; p < g.pend; ++p) cf[L.cubes[L.in_cube[H.m2l_tgt[p]]]] += f;
    }
    for (int64_t t = 0; t < nl; ++t) {
      const double nt = (double)(lp[t + 1] - lp[t]);
      for (int64_t c = H.leaves[t]; c >= 0; c = H.cubes[c].parent)
        if (cf[c] > 0) cost[t] += cf[c] * nt / (double)(H.cubes[c].pend - H.cubes[c].pbeg);
    }
    std::vector<double> pre(nl + 1, 0.0);
    for (int64_t t = 0; t < nl; ++t) pre[t + 1] = pre[t] + cost[t];
    for (int q = 1; q < R; ++q) {
      const double target = pre[nl] * (double)q / (double)R;
      rl[q] = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
      rl[q] = std::min(std::max(rl[q], rl[q - 1]), nl);
    }
  }
  P->nranks = R;
  P->rank = r;
  P->nleaf = nl;
  P->rank_leaf = rl;
  P->rank_pt.assign(R + 1, 0);
  for (int q = 0; q <= R; ++q) P->rank_pt[q] = lp[rl[q]];
  P->leaf_b = rl[r], P->leaf_e = rl[r + 1];
  P->pt_b = P->rank_pt[r], P->pt_e = P->rank_pt[r + 1];
  P->st.owned_begin = P->pt_b, P->st.owned_end = P->pt_e;
  P->st.owned_leaf_begin = P->leaf_b, P->st.owned_leaf_end = P->leaf_e;
  P->st.n = n;
  P->st.nleaves = nl;
  P->st.nlevels = (int64_t)H.levels.size();
  P->st.lmin = H.lmin;
}

// does the cube (global id) contain points of rank q?
inline bool cube_on_rank(fda_plan P, int64_t gid, int q) {
  const fda::Cube& c = P->H.cubes[gid];
  return P->rank_pt[q] < P->rank_pt[q + 1] && c.pend > P->rank_pt[q] && c.pbeg < P->rank_pt[q + 1];
}
// ranks [*a, *b] whose point ranges meet the cube (empty ranks inside the interval are skipped by callers)
inline void cube_ranks(fda_plan P, int64_t gid, int* a, int* b) {
  const fda::Cube& c = P->H.cubes[gid];
  *a = (int)(std::upper_bound(P->rank_pt.begin(), P->rank_pt.end(), c.pbeg) - P->rank_pt.begin()) - 1;
  *b = (int)(std::upper_bound(P->rank_pt.begin(), P->rank_pt.end(), c.pend - 1) - P->rank_pt.begin()) - 1;
  *a = std::min(std::max(*a, 0), P->nranks - 1);
  *b = std::min(std::max(*b, 0), P->nranks - 1);
}

// Exchange lists.  Every rank runs S2M on its own leaves and M2M on the cubes that contain
// its points, so its outgoing expansion of a cube is the partial sum over its own points (M2M is linear);
// the full expansion is the sum of the partials of the cube's ranks.  Rank q needs the full expansion of
// every source slot of an M2L pair whose target cube contains points of q.  So rank r sends its partial of
// slot s to every q != r that needs s, and receives from every other rank of cube(s) the slots it needs.
// Both sides enumerate (level, slot) in ascending order, so the lists agree without negotiation.
void build_exchange(fda_plan P) {
  const fda::HostPlan& H = P->H;
  const int R = P->nranks, r = P->rank;
  auto& X = P->xc;
  X.send.assign(R, {});
  X.recv.assign(R, {});
  if (R == 1) return;
  const int nlev = (int)H.levels.size();
  std::vector<std::vector<int64_t>> grp_by_level(nlev);
  for (size_t g = 0; g < H.m2l_groups.size(); ++g) grp_by_level[H.m2l_groups[g].level].push_back((int64_t)g);
  for (int l = 0; l < nlev; ++l) {
    const fda::Level& L = H.levels[l];
    if (grp_by_level[l].empty() || L.n_out == 0) continue;
    // need[s]: bit q set iff rank q needs out slot s (R <= 64)
    std::vector<uint64_t> need(L.n_out, 0);
    std::vector<uint64_t> tmask(L.n_in, 0);
    for (int64_t t = 0; t < L.n_in; ++t) {
      const int64_t gid = L.cubes[L.in_cube[t]];
      int a, b;
      cube_ranks(P, gid, &a, &b);
      for (int q = a; q <= b; ++q)
        if (cube_on_rank(P, gid, q)) tmask[t] |= 1ull << q;
    }
    for (int64_t g : grp_by_level[l]) {
      const auto& G = H.m2l_groups[g];
      for (int64_t p = G.pbeg; p < G.pend; ++p) need[H.m2l_src[p]] |= tmask[H.m2l_tgt[p]];
    }
    for (int64_t s = 0; s < L.n_out; ++s) {
      if (!need[s]) continue;
      const int64_t gid = L.cubes[L.out_cube[s]];
      int a, b;
      cube_ranks(P, gid, &a, &b);
      if (cube_on_rank(P, gid, r))
        for (int q = 0; q < R; ++q)
          if (q != r && ((need[s] >> q) & 1)) X.send[q].push_back({l, s});
      if ((need[s] >> r) & 1)
        for (int q = a; q <= b; ++q)
          if (q != r && cube_on_rank(P, gid, q)) X.recv[q].push_back({l, s});
    }
  }
  X.send_cnt.assign(R, 0);
  X.recv_cnt.assign(R, 0);
  for (int q = 0; q < R; ++q) {
    for (auto& e : X.send[q]) X.send_cnt[q] += H.levels[e.first].s;
    for (auto& e : X.recv[q]) X.recv_cnt[q] += H.levels[e.first].s;
    X.send_tot += X.send_cnt[q];
    X.recv_tot += X.recv_cnt[q];
  }
  P->st.xchg_send_bytes = 16 * X.send_tot;
  P->st.xchg_recv_bytes = 16 * X.recv_tot;
}

// device arrays of the exchange (after Xall / xoff exist)
void upload_exchange(fda_plan P);

fda_status upload_plan(fda_plan P, const fda_options& o) {
  fda::HostPlan& H = P->H;
  const int64_t n = H.n;
  P->n = n;
  P->deterministic = o.deterministic != 0;
  if (!P->px) {  // host-built tree (the device tree leaves the Morton-ordered geometry in place)
    P->px = upload(P, H.px), P->py = upload(P, H.py), P->pz = upload(P, H.pz);
    P->nx = upload(P, H.nx), P->ny = upload(P, H.ny), P->nz = upload(P, H.nz);
    P->w = upload(P, H.w);
    P->perm = upload(P, H.perm);
  }
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
  auto owned_cube = [&](int64_t gid) { return R == 1 || cube_on_rank(P, gid, P->rank); };
  // levels: all outgoing expansions in one allocation (the exchange addresses them by one offset)
  const int nlev = (int)H.levels.size();
  P->lv.assign(nlev, DevLevel());
  P->xoff.assign(nlev + 1, 0);
  for (int l = 0; l < nlev; ++l) P->xoff[l + 1] = P->xoff[l] + H.levels[l].n_out * (int64_t)H.levels[l].s;
  if (P->xoff[nlev]) P->Xall = dalloc<double2>(P, (size_t)P->xoff[nlev]);
  for (int l = 0; l < nlev; ++l) {
    const fda::Level& L = H.levels[l];
    DevLevel& D = P->lv[l];
    D.s = L.s, D.n_out = L.n_out, D.n_in = L.n_in;
    if (L.n_out) D.X = P->Xall + P->xoff[l];
    if (L.n_in) D.Y = dalloc<double2>(P, (size_t)L.n_in * L.s);
  }
  std::ostringstream tlog;  // setup timings of the upload (plan log)
  double tu = now();
  auto lap = [&](const char* what) {
    cudaDeviceSynchronize();
    const double t = now();
    tlog << what << " " << t - tu << "s ";
    tu = t;
  };
  lap("geometry");
  // device point sets and factors of every level's directions (plan_dev.cuh DevSet), for the operators
  const bool dev_ops = H.opt.dev_ops;
  std::vector<std::vector<int>> bset(nlev), aset(nlev);
  fda::DevSet* d_sets = nullptr;
  if (dev_ops) {
    std::vector<fda::DevSet> hs;
    auto up_c = [&](const std::vector<cplx>& v) { return reinterpret_cast<const double2*>(upload(P, v)); };
    for (int l = std::max(H.lmin, 0); H.lmin >= 0 && l < nlev; ++l) {
      const fda::Level& L = H.levels[l];
      if (L.s == 0 || (L.n_out == 0 && L.n_in == 0)) continue;
      const int nd = L.hf ? L.ndir : 1;
      bset[l].assign(nd, -1), aset[l].assign(nd, -1);
      // factors per representative (HF) or of the LF surface: V, V^T (M2L left), Sigma^-1 U^H (M2M left)
      const int nrep = L.hf ? (int)L.reps.size() : 1;
      std::vector<const double2*> fV(nrep), fVT(nrep), fSU(nrep);
      std::vector<int> fs(nrep);
      for (int ri = 0; ri < nrep; ++ri) {
        const fda::Mat& U = L.hf ? L.reps[ri].U : L.lfU;
        const fda::Mat& V = L.hf ? L.reps[ri].V : L.lfV;
        const std::vector<double>& sg = L.hf ? L.reps[ri].sig : L.lfsig;
        const int sr = (int)sg.size();
        if (!L.orig) {
          std::vector<cplx> vt((size_t)sr * V.m), su((size_t)sr * U.m);
          for (int64_t i = 0; i < V.m; ++i)
            for (int r = 0; r < sr; ++r) vt[r + (size_t)i * sr] = V(i, r);
          for (int64_t i = 0; i < U.m; ++i)
            for (int r = 0; r < sr; ++r) su[r + (size_t)i * sr] = std::conj(U(i, r)) / sg[r];
          fV[ri] = up_c(V.a), fVT[ri] = up_c(vt), fSU[ri] = up_c(su), fs[ri] = sr;
        } else {
          // original mode (Table 1): the expansion is the equivalent density itself -- identity reduction,
          // M2M left factor R^+ = V Sigma^-1 U^H (n_b x n_a)
          const int nb_ = (int)V.m;
          std::vector<cplx> id((size_t)nb_ * nb_, 0.0), rp((size_t)nb_ * U.m, 0.0);
          for (int b = 0; b < nb_; ++b) id[b + (size_t)b * nb_] = 1.0;
          for (int64_t i = 0; i < U.m; ++i)
            for (int b = 0; b < nb_; ++b) {
              cplx v = 0;
              for (int r = 0; r < sr; ++r) v += V(b, r) * std::conj(U(i, r)) / sg[r];
              rp[b + (size_t)i * nb_] = v;
            }
          fV[ri] = up_c(id), fVT[ri] = fV[ri], fSU[ri] = up_c(rp), fs[ri] = nb_;
        }
      }
      for (int d = 0; d < nd; ++d) {
        if (L.hf && L.dir_rep[d] < 0) continue;
        const int ri = L.hf ? L.dir_rep[d] : 0;
        auto pts = [&](bool check) {
          std::vector<double> f;
          for (const auto& p : fda::dir_points(L, d, check)) f.insert(f.end(), {p[0], p[1], p[2]});
          return f;
        };
        const std::vector<double> pb = pts(false), pa = pts(true);
        bset[l][d] = (int)hs.size();
        hs.push_back(fda::DevSet{(int)pb.size() / 3, fs[ri], upload(P, pb), fVT[ri], fV[ri]});
        aset[l][d] = (int)hs.size();
        hs.push_back(fda::DevSet{(int)pa.size() / 3, fs[ri], upload(P, pa), fSU[ri], nullptr});
      }
    }
    d_sets = upload(P, hs);
    P->dev_sets = hs;
  }
  auto set_max = [&](const std::vector<int>& ids, int* maxn) {
    for (int i : ids)  // (directions without a set have id -1)
      if (i >= 0) *maxn = std::max(*maxn, P->dev_sets[i].n);
  };
  lap("sets");
  // M2L: pairs filtered to owned targets, grouped by offset; operators built on the device
  for (int l = 0; l < nlev; ++l) {
    const fda::Level& L = H.levels[l];
    // groups of the level with pairs into this rank's target cubes, counted in parallel, then filled in
    // parallel (group-major, pairs in the plan's order)
    std::vector<int64_t> lg;  // group indices of the level
    for (size_t gi = 0; gi < H.m2l_groups.size(); ++gi)
      if (H.m2l_groups[gi].level == l) lg.push_back((int64_t)gi);
    std::vector<int64_t> cntg(lg.size(), 0);
    auto keep_pair = [&](int64_t p) { return R == 1 || owned_cube(L.cubes[L.in_cube[H.m2l_tgt[p]]]); };
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t q = 0; q < (int64_t)lg.size(); ++q) {
      const auto& g = H.m2l_groups[lg[q]];
      int64_t c = 0;
      for (int64_t p = g.pbeg; p < g.pend; ++p) c += keep_pair(p);
      cntg[q] = c;
    }
    // HF levels: groups whose operators are equal by the cube symmetry share one operator (below)
    const std::vector<int32_t> cls = m2l_symmetry_classes(L, H, lg, cntg);
    GroupedPairs G;
    std::vector<int64_t> gid;                 // canonical group (index in H.m2l_groups) of each operator
    std::vector<std::vector<int64_t>> memb;   // member groups of each operator (level-local indices q)
    {
      std::vector<int32_t> slot(lg.size(), -1);
      for (size_t q = 0; q < lg.size(); ++q) {
        if (!cntg[q]) continue;
        int32_t& sl = slot[cls[q]];
        if (sl < 0) {
          sl = (int32_t)gid.size();
          gid.push_back(lg[q]);
          memb.emplace_back();
        }
        memb[sl].push_back((int64_t)q);
      }
    }
    for (size_t g = 0; g < gid.size(); ++g) {
      const auto& hg = H.m2l_groups[gid[g]];
      int64_t n = 0;
      for (int64_t q : memb[g]) n += cntg[q];
      G.gptr.push_back(G.gptr.back() + n);
      G.rank.push_back(hg.rank);
      G.mat.push_back(hg.mat_off);
      G.so.push_back((int16_t)L.sdir(L.hf ? fda::anti_dir(hg.dir, L.m) : 0));
      G.si.push_back((int16_t)L.sdir(hg.dir));
    }
    G.out.resize(G.gptr.back()), G.in.resize(G.gptr.back());
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t g = 0; g < (int64_t)gid.size(); ++g) {
      int64_t o = G.gptr[g];
      for (int64_t q : memb[g]) {
        const auto& hg = H.m2l_groups[lg[q]];
        for (int64_t p = hg.pbeg; p < hg.pend; ++p)
          if (keep_pair(p)) G.out[o] = (int32_t)H.m2l_tgt[p], G.in[o] = (int32_t)H.m2l_src[p], ++o;
      }
      // a shared operator's pairs in output-slot (Morton) order, as within one group
      if (memb[g].size() > 1) {
        std::vector<std::pair<int32_t, int32_t>> pr;
        pr.reserve(G.gptr[g + 1] - G.gptr[g]);
        for (int64_t e = G.gptr[g]; e < G.gptr[g + 1]; ++e) pr.emplace_back(G.out[e], G.in[e]);
        std::sort(pr.begin(), pr.end());
        for (int64_t e = G.gptr[g]; e < G.gptr[g + 1]; ++e) G.out[e] = pr[e - G.gptr[g]].first, G.in[e] = pr[e - G.gptr[g]].second;
      }
    }
    P->st.m2l_ops += (int64_t)gid.size();
    if (G.out.empty()) continue;
    const double* dpool = nullptr;
    if (dev_ops) {
      // K~ of every group on the device: pass 1 ranks, offsets, pass 2 the fragment-order pool
      const int ng = (int)gid.size();
      std::vector<int32_t> ia(ng), ib(ng);
      std::vector<double> sh(3 * (size_t)ng);
      std::vector<int> used_sets;
      for (int g = 0; g < ng; ++g) {
        const auto& hg = H.m2l_groups[gid[g]];
        const int d = L.hf ? hg.dir : 0, t = L.hf ? fda::anti_dir(hg.dir, L.m) : 0;
        ia[g] = bset[l][t], ib[g] = bset[l][d];
        for (int c = 0; c < 3; ++c) sh[3 * g + c] = hg.off[c] * L.w;  // G(delta w + b_t - b_s)
      }
      fda::OpJob J;
      J.n_items = ng;
      J.a = upload(P, ia), J.b = upload(P, ib), J.shift = upload(P, sh);
      J.sets = d_sets, J.k = H.k, J.s_out = L.s, J.s_in = L.s;
      J.compress = H.opt.lowrank ? 1 : 0, J.eps_lr = H.eps_lr_level(L);
      // FDA_RANK_ROUND=n (experiments): round the low ranks up to a multiple of n instead of 8
      if (getenv("FDA_RANK_ROUND")) J.rank_round = std::max(1, atoi(getenv("FDA_RANK_ROUND")));
      set_max(bset[l], &J.maxn);
      J.maxs = L.s;
      std::vector<int32_t> rk(ng, -1);
      if (J.compress) {
        int32_t* d_rank = dalloc<int32_t>(P, ng);
        J.rank = d_rank;
        ck(fda::launch_opjob(J, 1, 0));
        ck(cudaMemcpy(rk.data(), d_rank, ng * sizeof(int32_t), cudaMemcpyDeviceToHost));
        J.rank_in = d_rank;
      }
      std::vector<int64_t> off(ng);
      int64_t tot = 0;
      for (int g = 0; g < ng; ++g) {
        off[g] = tot;
        tot += frag_size(rk[g], L.s, L.s);
        G.rank[g] = rk[g], G.mat[g] = off[g];
        for (int64_t q : memb[g]) P->H.m2l_groups[lg[q]].rank = rk[g];
      }
      double* pool = dalloc<double>(P, (size_t)tot);
      J.off = upload(P, off), J.pool = pool;
      ck(fda::launch_opjob(J, 2, 0));
      dpool = pool;
    }
    for (size_t g = 0; g < G.rank.size(); ++g) {
      const auto& hg = H.m2l_groups[gid[g]];
      const double np = (double)(G.gptr[g + 1] - G.gptr[g]);
      P->st.m2l_pairs += (int64_t)np;
      P->st.m2l_groups += (int64_t)memb[g].size();
      P->st.m2l_lowrank_groups += G.rank[g] >= 0 ? (int64_t)memb[g].size() : 0;
      // algorithmic flops with the wedges' own expansion lengths (the pool pads them to the level's max)
      const double ss = L.sdir(hg.dir), st_ = L.sdir(L.hf ? fda::anti_dir(hg.dir, L.m) : 0);
      P->st.flops_m2l += np * (G.rank[g] < 0 ? 8.0 * st_ * ss : 8.0 * G.rank[g] * (st_ + ss));
    }
    const cplx* raw = dev_ops ? nullptr : H.m2l_pool[l].data();
    // FDA_M2L_BLOCK=1: the low-rank groups with pad8(r) <= 24 (device operators) run as the two-pass M2L with
    // target-owned outputs (m2l_block.cu: T = V X stored, then Y += U T per target block in shared memory) --
    // deterministic, but measured slower than the group-major atomic kernels at config 5, so
    // off by default
    const bool blk_on = getenv("FDA_M2L_BLOCK") && getenv("FDA_M2L_BLOCK")[0] == '1';  // read per plan (tests toggle it)
    if (blk_on && dpool) {
      GroupedPairs Gb, Gr;
      // (a level whose expansions are too long for the block kernel's shared memory keeps every group in Gr)
      const bool blk_fits = fda::m2l_block_bmax(L.s, 24, fda::smem_optin_bytes()) > 0;
      split_groups(G, [&](size_t g) { return blk_fits && G.rank[g] >= 0 && pad8(G.rank[g]) <= 24; }, Gb, Gr);
      {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) cudaGetLastError(), fr = 0;
        if ((double)Gb.out.size() * fda::m2l_block_ldt(24) * sizeof(double2) > 0.3 * (double)fr) {
          Gb = GroupedPairs();
          Gr = G;
        }
      }
      P->lv[l].m2lb = make_blocks(P, Gb, L.in_cube, L.in_dir, L.s, L.s, dpool);
      P->tbuf_n = std::max<int64_t>(P->tbuf_n, P->lv[l].m2lb.n_pairs * (int64_t)P->lv[l].m2lb.ldt);
      if (H.opt.verbose && P->lv[l].m2lb.n_blocks) {
        const fda::BTrans& Bt = P->lv[l].m2lb;
        std::ostringstream os;
        os << "m2l blocks L" << l << ": groups " << Gb.rank.size() << "/" << G.rank.size() << " pairs " << Gb.out.size()
           << " blocks " << Bt.n_blocks << " (<= " << Bt.bmax << " slots) chunks " << Bt.n_chunks << " ("
           << (double)Gb.out.size() / (double)std::max<int64_t>(1, Bt.n_chunks) << " pairs/chunk) rmax8 " << Bt.rmax8 << "\n";
        H.log += os.str();
      }
      G = std::move(Gr);
      if (G.out.empty()) continue;
    }
    // FDA_M2L_MODE=owned|atomic: the item kind of the M2L launches only (experiments; FDA_GT_MODE: all)
    const char* m2l_mode = getenv("FDA_M2L_MODE");
    // Groups whose rank fits the warp-specialised kernel's shared memory run there; the others (few,
    // the nearest offsets) go to a second launch of the general kernel.
    const bool warp = fda::m2l_warp_on();
    // (warp-task kernel: ranks <= 24 whose operator keeps two CTAs per SM go to the first launch, the others to
    // the second; measured at config 5 (profiles/r02/ab_c5.log): M2L 158.2 ms with the split at 24, 162.8 ms with
    // the ranks <= 16 in a three-CTAs-per-SM launch of their own; FDA_M2L_RLIM overrides it)
    int rlim = warp ? std::max(8, std::min(24, fda::m2l_warp_rmax(L.s, L.s, GT_SMEM_BUDGET))) : fda::gtrans_ws_rmax(L.s);
    if (warp && getenv("FDA_M2L_RLIM")) rlim = std::max(8, atoi(getenv("FDA_M2L_RLIM")));
    GroupedPairs G1, G2;
    {
      std::vector<char> in1(G.rank.size());
      for (size_t g = 0; g < G.rank.size(); ++g) {
        in1[g] = G.rank[g] >= 0 && G.rank[g] <= rlim;
        GroupedPairs& D = in1[g] ? G1 : G2;
        D.gptr.push_back(D.gptr.back() + (G.gptr[g + 1] - G.gptr[g]));
        D.rank.push_back(G.rank[g]);
        D.mat.push_back(G.mat[g]);
        D.so.push_back(G.so[g]), D.si.push_back(G.si[g]);
      }
      if (!G1.rank.empty() && !G2.rank.empty()) {
        G1.out.resize(G1.gptr.back()), G1.in.resize(G1.gptr.back());
        G2.out.resize(G2.gptr.back()), G2.in.resize(G2.gptr.back());
        std::vector<int64_t> dst(G.rank.size());
        int64_t o1 = 0, o2 = 0;
        for (size_t g = 0; g < G.rank.size(); ++g) {
          dst[g] = in1[g] ? o1 : o2;
          (in1[g] ? o1 : o2) += G.gptr[g + 1] - G.gptr[g];
        }
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t g = 0; g < (int64_t)G.rank.size(); ++g) {
          GroupedPairs& D = in1[g] ? G1 : G2;
          std::copy(G.out.begin() + G.gptr[g], G.out.begin() + G.gptr[g + 1], D.out.begin() + dst[g]);
          std::copy(G.in.begin() + G.gptr[g], G.in.begin() + G.gptr[g + 1], D.in.begin() + dst[g]);
        }
      }
    }
    // FDA_M2L_WIN=W (experiment): the LF levels' items end at W Morton windows of target cubes (L2 residency of Y)
    const int win = (!L.hf && getenv("FDA_M2L_WIN")) ? atoi(getenv("FDA_M2L_WIN")) : 0;
    if (H.opt.verbose) {
      std::map<int, int64_t> hist;  // pad8 rank -> pairs
      for (size_t g = 0; g < G.rank.size(); ++g) hist[G.rank[g] < 0 ? -1 : pad8(G.rank[g])] += G.gptr[g + 1] - G.gptr[g];
      std::ostringstream os;
      os << "m2l L" << l << " (s " << L.s << ", split at rank " << rlim << "): pairs by pad8 rank:";
      for (const auto& kv : hist) os << " " << kv.first << ":" << kv.second;
      H.log += os.str() + "\n";
    }
    if (!G1.rank.empty() && !G2.rank.empty()) {
      P->lv[l].m2l = make_items(P, G1, L.in_cube, L.in_dir, (int64_t)L.cubes.size(), L.s, L.s, raw, dpool, m2l_mode, win);
      P->lv[l].m2l2 = make_items(P, G2, L.in_cube, L.in_dir, (int64_t)L.cubes.size(), L.s, L.s, raw, dpool, m2l_mode, win);
    } else {
      P->lv[l].m2l = make_items(P, G, L.in_cube, L.in_dir, (int64_t)L.cubes.size(), L.s, L.s, raw, dpool, m2l_mode, win);
    }
    P->lv[l].m2l.warp_tasks = P->lv[l].m2l2.warp_tasks = warp ? 1 : 0;
    P->lv[l].m2l.sector = P->lv[l].m2l2.sector = 0;  // measured slower at config 5 (ab_c5.log: +4.7 ms)
  }
  if (P->tbuf_n) P->tbuf = dalloc<double2>(P, (size_t)P->tbuf_n);
  lap("m2l");
  // transitions: M2M items own parent out slots (groups = (dir, octant) matrices),
  // L2L items own child in slots (groups = the same matrices, transposed layout)
  for (const auto& T : H.trans) {
    DevTrans D;
    const fda::Level& Lp = H.levels[T.lp];
    const fda::Level& Lc = H.levels[T.lp + 1];
    D.lp = T.lp, D.sp = T.sp, D.sc = T.sc;
    const int64_t nmat = (int64_t)T.need.size();
    // CSR by output slot -> group-major pairs, keeping the pairs keep(out slot, in slot) accepts
    auto grouped = [&](const std::vector<int64_t>& ptr, const std::vector<int64_t>& other,
                       const std::vector<int64_t>& mat, auto keep) {
      GroupedPairs G;
      std::vector<int64_t> cnt(nmat + 1, 0);
      for (int64_t s = 0; s + 1 < (int64_t)ptr.size(); ++s)
        for (int64_t e = ptr[s]; e < ptr[s + 1]; ++e)
          if (keep(s, other[e])) cnt[T.mat_index[mat[e]] + 1]++;
      for (int64_t g = 0; g < nmat; ++g) cnt[g + 1] += cnt[g];
      G.out.assign(cnt[nmat], 0);
      G.in.assign(cnt[nmat], 0);
      std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
      for (int64_t s = 0; s + 1 < (int64_t)ptr.size(); ++s)
        for (int64_t e = ptr[s]; e < ptr[s + 1]; ++e) {
          if (!keep(s, other[e])) continue;
          const int64_t pos = fill[T.mat_index[mat[e]]]++;
          G.out[pos] = (int32_t)s;
          G.in[pos] = (int32_t)other[e];
        }
      for (int64_t g = 0; g < nmat; ++g) {
        G.gptr.push_back(cnt[g + 1]);
        G.rank.push_back(-1);
        G.mat.push_back(g * (int64_t)T.sp * T.sc);
      }
      return G;
    };
    // the (parent direction, child direction) expansion lengths of every M2M matrix
    auto sizes = [&](GroupedPairs& G, bool up) {
      for (int64_t g = 0; g < nmat; ++g) {
        const int d = T.need[g].first, sp_ = Lp.sdir(Lp.hf ? d : 0), sc_ = Lc.sdir(Lc.hf ? fda::child_dir(d, Lp.m) : 0);
        G.so.push_back((int16_t)(up ? sp_ : sc_)), G.si.push_back((int16_t)(up ? sc_ : sp_));
      }
    };
    // multi-GPU: M2M only from child cubes with points of this rank (partial sums); L2L only
    // into child cubes with points of this rank (their local expansions are complete here)
    double fup = 0, fdn = 0;  // algorithmic flops with the directions' own expansion lengths
    auto up_keep = [&](int64_t ps, int64_t cs) {
      if (!owned_cube(Lc.cubes[Lc.out_cube[cs]])) return false;
      fup += 8.0 * Lp.sdir(Lp.out_dir[ps]) * Lc.sdir(Lc.out_dir[cs]);
      return true;
    };
    auto dn_keep = [&](int64_t cs, int64_t ps) {
      if (!owned_cube(Lc.cubes[Lc.in_cube[cs]])) return false;
      fdn += 8.0 * Lp.sdir(Lp.in_dir[ps]) * Lc.sdir(Lc.in_dir[cs]);
      return true;
    };
    // M2M (and its transpose, L2L) operators on the device: one per (parent direction, child octant)
    const double *dup = nullptr, *ddn = nullptr;
    if (dev_ops && nmat > 0) {
      std::vector<int32_t> ia(nmat), ib(nmat);
      std::vector<double> sh(3 * (size_t)nmat);
      for (int64_t t = 0; t < nmat; ++t) {
        const int d = T.need[t].first, oc = T.need[t].second;
        ia[t] = aset[T.lp][Lp.hf ? d : 0];
        ib[t] = bset[T.lp + 1][Lc.hf ? fda::child_dir(d, Lp.m) : 0];
        const double o[3] = {(((oc >> 2) & 1) ? 0.5 : -0.5) * Lc.w, (((oc >> 1) & 1) ? 0.5 : -0.5) * Lc.w,
                             ((oc & 1) ? 0.5 : -0.5) * Lc.w};
        for (int c = 0; c < 3; ++c) sh[3 * t + c] = -o[c];  // E_up = G(a_P - (b_C + o))
      }
      fda::OpJob J;
      J.n_items = (int)nmat;
      J.a = upload(P, ia), J.b = upload(P, ib), J.shift = upload(P, sh);
      J.sets = d_sets, J.k = H.k, J.s_out = T.sp, J.s_in = T.sc;
      set_max(aset[T.lp], &J.maxn);
      set_max(bset[T.lp + 1], &J.maxn);
      J.maxs = std::max(T.sp, T.sc);
      const int64_t szu = frag_size(-1, T.sp, T.sc), szd = frag_size(-1, T.sc, T.sp);
      std::vector<int64_t> off(nmat);
      for (int64_t t = 0; t < nmat; ++t) off[t] = t * szu;
      double* pu = dalloc<double>(P, (size_t)(nmat * szu));
      double* pd = dalloc<double>(P, (size_t)(nmat * szd));
      J.off = upload(P, off), J.pool = pu, J.poolT = pd;
      ck(fda::launch_opjob(J, 2, 0));
      dup = pu, ddn = pd;
    }
    if (!T.up_child.empty()) {
      GroupedPairs G = grouped(T.up_ptr, T.up_child, T.up_mat, up_keep);
      sizes(G, true);
      if (dev_ops)
        for (auto& m : G.mat) m = (m / ((int64_t)T.sp * T.sc)) * frag_size(-1, T.sp, T.sc);
      D.up = make_items(P, G, Lp.out_cube, Lp.out_dir, (int64_t)Lp.cubes.size(), T.sp, T.sc,
                        dev_ops ? nullptr : T.pool.data(), dup);
    }
    if (!T.dn_parent.empty()) {
      GroupedPairs G = grouped(T.dn_ptr, T.dn_parent, T.dn_mat, dn_keep);
      sizes(G, false);
      if (dev_ops)
        for (auto& m : G.mat) m = (m / ((int64_t)T.sp * T.sc)) * frag_size(-1, T.sc, T.sp);
      D.dn = make_items(P, G, Lc.in_cube, Lc.in_dir, (int64_t)Lc.cubes.size(), T.sc, T.sp,
                        dev_ops ? nullptr : T.poolT.data(), ddn);
    }
    P->st.flops_m2m += 0.5 * fup;  // keep() runs twice per pair (count, fill)
    P->st.flops_l2l += 0.5 * fdn;
    P->tr.push_back(D);
  }
  lap("m2m/l2l");
  // leaf operators: S2M and L2T on this rank's leaves
  for (const auto& O : H.leafops) {
    const fda::Level& L = H.levels[O.level];
    DevLeafOps D;
    D.level = O.level, D.s = L.s, D.nsurf = L.nsurf;
    std::vector<int64_t> lo_, so_;
    for (size_t t = 0; t < O.leaf.size(); ++t)
      if (O.leaf[t] >= P->leaf_b && O.leaf[t] < P->leaf_e) lo_.push_back(O.leaf[t]), so_.push_back(O.slot[t]);
    D.nleaves_own = (int64_t)lo_.size();
    if (lo_.empty()) continue;
    D.leaf_own = upload_i32(P, lo_);
    std::vector<double> sf;
    for (const auto& p : L.ck_pts) sf.insert(sf.end(), {p[0], p[1], p[2]});
    D.surf = upload(P, sf);
    {  // S2M reduction: pairs (out = leaf slot, in = owned-leaf row t of the check-potential buffer)
      GroupedPairs G;
      G.out.assign(so_.begin(), so_.end());
      G.in.resize(lo_.size());
      for (size_t t = 0; t < lo_.size(); ++t) G.in[t] = (int32_t)t;
      G.gptr.push_back((int64_t)G.out.size());
      G.rank.push_back(-1);
      G.mat.push_back(0);
      D.s2m = make_items(P, G, L.out_cube, L.out_dir, (int64_t)L.cubes.size(), L.s, L.nsurf, O.S.data());
    }
    {  // L2T reduction: pairs (out = owned-leaf row t, in = leaf slot)
      GroupedPairs G;
      G.in.assign(so_.begin(), so_.end());
      G.out.resize(lo_.size());
      std::vector<int64_t> oc(lo_.size());
      for (size_t t = 0; t < lo_.size(); ++t) G.out[t] = (int32_t)t, oc[t] = L.in_cube[so_[t]];
      std::vector<int> od(lo_.size(), 0);
      G.gptr.push_back((int64_t)G.out.size());
      G.rank.push_back(-1);
      G.mat.push_back(0);
      D.l2t = make_items(P, G, oc, od, (int64_t)L.cubes.size(), L.nsurf, L.s, O.T.data());
    }
    // "In the FDBEM, the S2M and L2T matrices are precomputed and saved in memory": the
    // per-leaf matrices S_leaf (s x n) and T_leaf (n x s) are built here once when they take <= 40% of the free
    // device memory (FDA_LEAF_MATS=0: never; then the apply evaluates the kernels on the surfaces every time)
    std::vector<int64_t> pofs(lo_.size() + 1, 0);
    for (size_t t = 0; t < lo_.size(); ++t) pofs[t + 1] = pofs[t] + (lp[lo_[t] + 1] - lp[lo_[t]]);
    const double mat_bytes = 2.0 * (double)pofs.back() * L.s * sizeof(double2);
    bool mats = !(getenv("FDA_LEAF_MATS") && getenv("FDA_LEAF_MATS")[0] == '0');
    if (mats) {
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) cudaGetLastError(), fr = 0;
      mats = mat_bytes <= 0.4 * (double)fr;
    }
    if (mats) {
      D.pofs = upload(P, pofs);
      std::vector<int32_t> sl(so_.begin(), so_.end());
      D.slot = upload(P, sl);
      D.Sm = dalloc<double2>(P, (size_t)pofs.back() * L.s);
      D.Tm = dalloc<double2>(P, (size_t)pofs.back() * L.s);
      std::vector<double> sred(2 * O.S.size()), tredt(2 * O.T.size());
      for (size_t i = 0; i < O.S.size(); ++i) sred[2 * i] = O.S[i].real(), sred[2 * i + 1] = O.S[i].imag();
      for (int b = 0; b < L.nsurf; ++b)  // O.T: nsurf x s column-major -> row-major
        for (int c = 0; c < L.s; ++c) {
          const cplx v = O.T[b + (size_t)c * L.nsurf];
          tredt[2 * ((size_t)b * L.s + c)] = v.real(), tredt[2 * ((size_t)b * L.s + c) + 1] = v.imag();
        }
      const double* d_sred = upload(P, sred);
      const double* d_tredt = upload(P, tredt);
      const double2 alpha_dn = P->kind == FDA_KERNEL_T1 ? make_double2(0.0, 0.0) : alpha_of(P);
      fda::launch_leafmat(P->kind, (int64_t)lo_.size(), D.leaf_own, D.pofs, leaves_of(P), points_of(P), D.surf,
                          L.nsurf, H.k, alpha_of(P), alpha_dn, reinterpret_cast<const double2*>(d_sred),
                          reinterpret_cast<const double2*>(d_tredt), L.s, D.Sm, D.Tm, 0);
      ck(cudaGetLastError());
      P->st.bytes_s2m += (double)pofs.back() * L.s * sizeof(double2);
      P->st.bytes_l2t += (double)pofs.back() * L.s * sizeof(double2);
      P->st.flops_s2m += 8.0 * (double)pofs.back() * L.s;  // x~ = S_leaf q
      P->st.flops_l2t += 8.0 * (double)pofs.back() * L.s;
    } else {
      P->surfbuf_n = std::max(P->surfbuf_n, (int64_t)lo_.size() * L.nsurf);
      for (size_t t = 0; t < lo_.size(); ++t) {
        const int64_t npt = lp[lo_[t] + 1] - lp[lo_[t]];
        P->st.s2m_evals += npt * L.nsurf;
        P->st.l2t_evals += npt * L.nsurf;
        P->st.flops_s2m += 8.0 * L.s * L.nsurf;  // the reduction x~ = S chk (eq_cmps); the evaluations are counted apart
        P->st.flops_l2t += 8.0 * L.s * L.nsurf;
      }
    }
    P->lo.push_back(D);
  }
  if (P->surfbuf_n) P->surfbuf = dalloc<double2>(P, (size_t)P->surfbuf_n);
  // every translation launch must fit the device's shared memory (large expansions at small eps)
  {
    bool fits = true;
    for (const auto& D : P->lv) fits &= fda::gtrans_fits(D.m2l) && fda::gtrans_fits(D.m2l2);
    for (const auto& T : P->tr) fits &= fda::gtrans_fits(T.up) && fda::gtrans_fits(T.dn);
    for (const auto& O : P->lo) fits &= fda::gtrans_fits(O.s2m) && fda::gtrans_fits(O.l2t);
    if (!fits) {
      fprintf(stderr, "fda: a translation launch exceeds the device's shared memory per CTA\n");
      return FDA_ERR_SETUP_ACCURACY;
    }
  }
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
  const int kk = std::min(std::max(P->kind, 0), 2);
  s.flops_p2p = FLOP_P2P[kk] * (double)s.p2p_point_pairs;
  s.flops_s2m += FLOP_S2M[kk] * (double)s.s2m_evals;
  s.flops_l2t += FLOP_L2T * (double)s.l2t_evals;
  for (int l = 0; l < nlev; ++l) s.out_slots += H.levels[l].n_out, s.in_slots += H.levels[l].n_in;
  s.owned_begin = P->pt_b, s.owned_end = P->pt_e;
  s.setup_tree_s = H.t_tree, s.setup_lists_s = H.t_lists, s.setup_ops_s = H.t_ops;
  upload_exchange(P);
  lap("leaf/exchange");
  if (o.verbose) P->H.log += "upload: " + tlog.str() + "\n";
  return FDA_OK;
}

void upload_exchange(fda_plan P) {
  auto& X = P->xc;
  const int R = P->nranks;
  if (R == 1) return;
  const fda::HostPlan& H = P->H;
  std::vector<int64_t> sx, sb;
  std::vector<int32_t> sl;
  int64_t off = 0;
  for (int q = 0; q < R; ++q)
    for (auto& e : X.send[q]) {
      const int s_ = H.levels[e.first].s;
      sx.push_back(P->xoff[e.first] + e.second * s_), sl.push_back(s_), sb.push_back(off);
      off += s_;
    }
  X.nsend = (int64_t)sx.size();
  // received entries grouped by destination (level, slot), partials in peer order
  std::vector<std::pair<std::pair<int, int64_t>, std::pair<int, int64_t>>> rv;  // ((level, slot), (peer, buf off))
  off = 0;
  for (int q = 0; q < R; ++q)
    for (auto& e : X.recv[q]) {
      rv.push_back({e, {q, off}});
      off += H.levels[e.first].s;
    }
  std::stable_sort(rv.begin(), rv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<int64_t> dx, dp{0}, ro;
  std::vector<int32_t> dl;
  for (size_t i = 0; i < rv.size(); ++i) {
    if (i == 0 || rv[i].first != rv[i - 1].first) {
      if (i) dp.push_back((int64_t)ro.size());
      const int s_ = H.levels[rv[i].first.first].s;
      dx.push_back(P->xoff[rv[i].first.first] + rv[i].first.second * s_), dl.push_back(s_);
    }
    ro.push_back(rv[i].second.second);
  }
  if (!rv.empty()) dp.push_back((int64_t)ro.size());
  X.ndst = (int64_t)dx.size();
  X.s_xoff = upload(P, sx), X.s_len = upload(P, sl), X.s_boff = upload(P, sb);
  X.d_xoff = upload(P, dx), X.d_len = upload(P, dl), X.d_rptr = upload(P, dp), X.d_roff = upload(P, ro);
  X.sendbuf = dalloc<double2>(P, (size_t)std::max<int64_t>(1, X.send_tot));
  X.recvbuf = dalloc<double2>(P, (size_t)std::max<int64_t>(1, X.recv_tot));
}

// Pivoted column selection of the HF directional sets on the device (plan.hpp Options::select).
std::vector<int64_t> dev_select(const std::vector<std::array<double, 3>>& X, const std::vector<std::array<double, 3>>& Y,
                                const std::vector<double>& rs, const std::vector<double>& cs, double k, double tol,
                                int64_t maxrank) {
  const int64_t m = (int64_t)X.size(), n = (int64_t)Y.size();
  std::vector<int64_t> piv(std::min<int64_t>({m, n, maxrank}) + 1);
  int64_t np = 0;
  double *dx, *dy, *drs = nullptr, *dcs = nullptr;
  double2* A;
  ck(cudaMalloc(&dx, 3 * m * sizeof(double)));
  ck(cudaMalloc(&dy, 3 * n * sizeof(double)));
  ck(cudaMalloc(&A, (size_t)m * n * sizeof(double2)));
  ck(cudaMemcpy(dx, X.data(), 3 * m * sizeof(double), cudaMemcpyHostToDevice));
  ck(cudaMemcpy(dy, Y.data(), 3 * n * sizeof(double), cudaMemcpyHostToDevice));
  if (!rs.empty()) {
    ck(cudaMalloc(&drs, m * sizeof(double)));
    ck(cudaMemcpy(drs, rs.data(), m * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (!cs.empty()) {
    ck(cudaMalloc(&dcs, n * sizeof(double)));
    ck(cudaMemcpy(dcs, cs.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  }
  fda::launch_gmat(A, dx, m, dy, n, drs, dcs, k, 0);
  const cudaError_t e = fda::pivoted_columns(A, m, n, tol, maxrank, piv.data(), &np, 0);
  for (void* p : {(void*)dx, (void*)dy, (void*)A, (void*)drs, (void*)dcs})
    if (p) cudaFree(p);
  ck(e);
  piv.resize(np);
  return piv;
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
  o->lf_p_low = 0;  // eps-dependent default
  o->lf_p_high = 0;
  o->lf_p_switch = d.lf_p_switch;
  o->lowrank = 1;
  o->single_leaf = 0;
  o->hf_max_rows = d.hf_max_rows;
  o->hf_spacing = d.hf_spacing;
  o->rank = 0;
  o->nranks = 1;
  o->verbose = 0;
  o->graph = 1;
  o->deterministic = 0;
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
  if (o.kernel != FDA_KERNEL_BMH && o.kernel != FDA_KERNEL_BMG && o.kernel != FDA_KERNEL_T1) return FDA_ERR_INVALID_ARG;
  if (o.nranks < 1 || o.nranks > 64 || o.rank < 0 || o.rank >= o.nranks) return FDA_ERR_INVALID_ARG;
  int ndev = 0;
  if (!o.host_only && (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)) {
    cudaGetLastError();
    return FDA_ERR_CUDA;
  }
  std::unique_ptr<fda_plan_s> P(new fda_plan_s());
  try {
    if (!o.host_only) cudaGetDevice(&P->dev);
    std::vector<double> x, nr, w;
    const bool dev_tree = !o.host_only && !(getenv("FDA_HOST_TREE") && getenv("FDA_HOST_TREE")[0] == '1');
    if (!dev_tree) {
      x = to_host(points, (size_t)n * 3), nr = to_host(normals, (size_t)n * 3), w = to_host(quad_weights, (size_t)n);
      if (!finite3(x) || !finite3(nr) || !finite3(w)) return FDA_ERR_INVALID_ARG;
      for (int64_t i = 0; i < n; ++i) {
        const double nn = std::sqrt(nr[3 * i] * nr[3 * i] + nr[3 * i + 1] * nr[3 * i + 1] + nr[3 * i + 2] * nr[3 * i + 2]);
        if (std::fabs(nn - 1.0) > 1e-10 || !(w[i] > 0)) return FDA_ERR_INVALID_ARG;
      }
    }
    fda::Options fo;
    fo.np = o.leaf_size;
    fo.eps_int = o.eps_internal;
    fo.eps_lr = o.eps_lowrank;
    fo.lf_p_low = o.lf_p_low > 1 ? o.lf_p_low : 0;  // 0: the eps-dependent default (plan.cpp, R17)
    fo.lf_p_high = o.lf_p_high > 1 ? o.lf_p_high : 0;
    if (o.lf_p_switch > 0) fo.lf_p_switch = o.lf_p_switch;
    fo.lowrank = o.lowrank;
    fo.single_leaf = o.single_leaf;
    if (o.hf_max_rows > 0) fo.hf_max_rows = o.hf_max_rows;
    if (o.hf_spacing > 0) fo.hf_spacing = o.hf_spacing;
    fo.verbose = o.verbose;
    fo.original = o.original != 0;
    if (fo.original) fo.lowrank = 0;  // the original FDA has no low-rank M2L
    // operators and HF directional sets on the device (plan_dev.cu); host-only plans (list audits) skip the
    // operators; FDA_HOST_OPS=1 builds them on the host (linalg.cpp) instead, for cross-checks
    const bool host_ops = getenv("FDA_HOST_OPS") && getenv("FDA_HOST_OPS")[0] == '1';
    fo.dev_ops = o.host_only || !host_ops || fo.original;
    if (!o.host_only && !host_ops) fo.select = dev_select;
    // P2 on the device (lists_dev.cu); FDA_HOST_LISTS=1 keeps the host lists (cross-checks)
    const bool host_lists = getenv("FDA_HOST_LISTS") && getenv("FDA_HOST_LISTS")[0] == '1';
    if (!o.host_only && !host_lists && !host_ops) fo.lists = fda::build_lists_device;
    std::string err;
    fda::TreeIn tin;
    const double t_dev0 = now();
    if (dev_tree) {
      // rows a-P0 / a-P1 on the device (tree_dev.cu): validation, Morton sort, octree; the Morton-ordered
      // geometry becomes the plan's
      const double *dp = points, *dn = normals, *dw = quad_weights;
      std::vector<void*> staged;
      auto stage = [&](const double* h, size_t count) {
        double* d = nullptr;
        ck(cudaMalloc(&d, count * sizeof(double)));
        staged.push_back(d);
        ck(cudaMemcpy(d, h, count * sizeof(double), cudaMemcpyHostToDevice));
        return (const double*)d;
      };
      if (!is_device_ptr(dp)) dp = stage(dp, (size_t)n * 3);
      if (!is_device_ptr(dn)) dn = stage(dn, (size_t)n * 3);
      if (!is_device_ptr(dw)) dw = stage(dw, (size_t)n);
      fda_plan Pp = P.get();
      Pp->px = dalloc<double>(Pp, n), Pp->py = dalloc<double>(Pp, n), Pp->pz = dalloc<double>(Pp, n);
      Pp->nx = dalloc<double>(Pp, n), Pp->ny = dalloc<double>(Pp, n), Pp->nz = dalloc<double>(Pp, n);
      Pp->w = dalloc<double>(Pp, n);
      Pp->perm = dalloc<int32_t>(Pp, n);
      const fda::DevGeom g{Pp->px, Pp->py, Pp->pz, Pp->nx, Pp->ny, Pp->nz, Pp->w, Pp->perm};
      err = fda::build_tree_device(n, dp, dn, dw, k, fda::leaf_size_for(eps, fo.np), fo.single_leaf, fo.max_depth, g,
                                   tin, 0);
      for (void* p : staged) cudaFree(p);
      if (err == "CUDA") throw CudaFail{FDA_ERR_CUDA};
      if (!err.empty()) {
        free_plan(Pp);
        return err == "COINCIDENT_POINTS" ? FDA_ERR_COINCIDENT_POINTS : FDA_ERR_INVALID_ARG;
      }
    }
    const double t_dev = now() - t_dev0;  // device P0 / P1 (with the input staging)
    err = fda::build_plan(P->H, n, x.data(), nr.data(), w.data(), k, cplx(alpha_re, alpha_im), eps, fo,
                          dev_tree ? &tin : nullptr);
    P->H.t_tree += t_dev;
    if (!err.empty()) {
      free_plan(P.get());
      if (err == "SETUP_ACCURACY") return FDA_ERR_SETUP_ACCURACY;
      return err == "COINCIDENT_POINTS" ? FDA_ERR_COINCIDENT_POINTS : FDA_ERR_INVALID_ARG;
    }
    P->host_only = o.host_only != 0;
    P->logstr = P->H.log;
    P->kind = o.kernel;
    set_ownership(P.get(), o);
    build_exchange(P.get());
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
    {  // return the plan builder's stream-ordered scratch (cudaMallocAsync pool) to the device
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, P->dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
      cudaGetLastError();
    }
    ck(cudaStreamCreateWithFlags(&P->nstream, cudaStreamNonBlocking));
    ck(cudaEventCreateWithFlags(&P->ev_perm, cudaEventDisableTiming));
    ck(cudaEventCreateWithFlags(&P->ev_near, cudaEventDisableTiming));
    P->graph_on = o.graph != 0 && !(getenv("FDA_GRAPH") && getenv("FDA_GRAPH")[0] == '0');
    if (P->graph_on) ck(cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking));
    ck(cudaDeviceSynchronize());
    P->st.setup_upload_s = now() - t0;
    P->st.device_bytes = P->bytes;
    P->logstr = P->H.log;
    if (o.verbose) P->logstr += fda::level_summary(P->H);
    // the host copies of the big pools are no longer needed
    std::vector<std::vector<cplx>>().swap(P->H.m2l_pool);
    for (auto& T : P->H.trans) std::vector<cplx>().swap(T.pool), std::vector<cplx>().swap(T.poolT);
  } catch (const CudaFail& f) {
    free_plan(P.get());
    cudaGetLastError();
    return f.s;
  } catch (const std::bad_alloc&) {
    if (getenv("FDA_DEBUG")) fprintf(stderr, "fda: host allocation failed in the plan upload\n");
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
  drop_graphs(P);  // the captured applies hold the old correction's pointers
  try {
    const int64_t n = P->n;
    int64_t* n_ptr = nullptr;
    int32_t* n_col = nullptr;
    double2* n_val = nullptr;
    int64_t own = 0;
    if (nnz > 0) {
      // validate and permute on the device into NEW buffers first: on any error the plan keeps its current
      // correction.  Host arrays are staged to the device.
      std::vector<void*> staged;
      auto stage = [&](const void* h, size_t bytes) -> const void* {
        if (is_device_ptr(h)) return h;
        void* d = nullptr;
        ck(cudaMalloc(&d, bytes));
        staged.push_back(d);
        ck(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
        return d;
      };
      auto unstage = [&] {
        for (void* p : staged) cudaFree(p);
        staged.clear();
      };
      try {
        const int64_t* drp = (const int64_t*)stage(row_ptr, (size_t)(n + 1) * sizeof(int64_t));
        const int32_t* dcol = (const int32_t*)stage(col, (size_t)nnz * sizeof(int32_t));
        const double2* dval = (const double2*)stage(val, (size_t)nnz * sizeof(double2));
        n_ptr = dalloc<int64_t>(P, (size_t)n + 1);
        const std::string err = fda::permute_csr_device(n, nnz, drp, dcol, dval, P->perm, P->pt_b, P->pt_e, n_ptr,
                                                        &n_col, &n_val, &own, 0);
        unstage();
        if (err == "CUDA") throw CudaFail{FDA_ERR_CUDA};
        if (!err.empty()) {
          auto it = std::find(P->allocs.begin(), P->allocs.end(), (void*)n_ptr);
          if (it != P->allocs.end()) P->allocs.erase(it);
          cudaFree(n_ptr);
          return FDA_ERR_INVALID_ARG;
        }
        P->allocs.push_back(n_col), P->allocs.push_back(n_val);
        P->bytes += own * (int64_t)(sizeof(int32_t) + sizeof(double2));
      } catch (...) {
        unstage();
        throw;
      }
    }
    if (P->c_ptr) {  // release the old correction only now that the new one is in place
      for (void* p : {(void*)P->c_ptr, (void*)P->c_col, (void*)P->c_val}) {
        auto it = std::find(P->allocs.begin(), P->allocs.end(), p);
        if (it != P->allocs.end()) P->allocs.erase(it);
        cudaFree(p);
      }
    }
    P->c_ptr = n_ptr, P->c_col = n_col, P->c_val = n_val;
    P->nnz = nnz;
    P->st.csr_nnz = nnz;
    P->st.bytes_csr = nnz ? 20.0 * (double)own + 48.0 * (double)(P->pt_e - P->pt_b) : 0.0;
    P->st.device_bytes = P->bytes;
  } catch (const CudaFail& f) {
    P->sticky_error = true;
    return f.s;
  } catch (const std::bad_alloc&) {
    return FDA_ERR_OOM;
  }
  return FDA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- apply
// Phases (fda_apply_timed indices): 0 permute, 1 p2p, 2 csr, 3 s2m, 4 m2m, 5 m2l, 6 l2l, 7 l2t, 8 unpermute,
// 9 exchange.  The stages below are stream-ordered on st; none synchronises the host.
namespace {

struct Marks {
  cudaEvent_t ev[2 * FDA_NPHASES] = {};
  bool on = false;
  cudaStream_t st = 0;
  void begin(int ph) {
    if (on) ck(cudaEventRecord(ev[2 * ph], st));
  }
  void end(int ph) {
    if (on) ck(cudaEventRecord(ev[2 * ph + 1], st));
  }
};

// FDA_TRACE=1: synchronise after every far-field launch and print its wall time (diagnostics only)
struct Trace {
  bool on = getenv("FDA_TRACE") != nullptr;
  double t = now();
  void operator()(cudaStream_t st, const char* what, int l) {
    if (!on) return;
    ck(cudaStreamSynchronize(st));
    const double t1 = now();
    fprintf(stderr, "[fda trace] %-4s level %d  %.3f ms\n", what, l, 1e3 * (t1 - t));
    t = t1;
  }
};

fda::Points points_of(fda_plan P) { return fda::Points{P->px, P->py, P->pz, P->nx, P->ny, P->nz, P->w}; }
fda::LeafGeom leaves_of(fda_plan P) { return fda::LeafGeom{P->leaf_ptr, P->lcx, P->lcy, P->lcz}; }
double2 alpha_of(fda_plan P) { return make_double2(P->H.alpha.real(), P->H.alpha.imag()); }
bool has_far(fda_plan P, uint32_t mask) { return (mask & FDA_PHASE_FAR) && P->H.lmin >= 0; }

// H1: q = w phi, phi and q in Morton order
void stage_permute(fda_plan P, const double2* d_phi, cudaStream_t st, Marks& mk) {
  mk.begin(0);
  fda::launch_permute_scale(P->n, P->perm, P->w, d_phi, P->q, P->phim, st);
  mk.end(0);
}

// upward pass (H4 S2M on this rank's leaves, H5 M2M on cubes with this rank's points) + pack of the
// partial expansions other ranks need into sendbuf
void stage_up(fda_plan P, uint32_t mask, double2* sendbuf, cudaStream_t st, Marks& mk, Trace& tr) {
  const fda::Points Pt = points_of(P);
  const fda::LeafGeom Lg = leaves_of(P);
  if (!has_far(P, mask)) return;
  mk.begin(3);
  // M2M accumulates into the non-leaf slots: clear every level's outgoing expansions first
  if (P->xoff.back()) ck(cudaMemsetAsync(P->Xall, 0, (size_t)P->xoff.back() * sizeof(double2), st));
  for (const auto& O : P->lo) {
    if (O.Sm) {  // stored S_leaf
      fda::launch_leaf_s2m(O.nleaves_own, O.leaf_own, O.pofs, O.slot, P->leaf_ptr, P->q, O.Sm, O.s, P->lv[O.level].X,
                           st);
    } else {
      fda::launch_s2m_check(P->kind, O.nleaves_own, O.leaf_own, Lg, Pt, P->q, O.surf, O.nsurf, P->H.k, alpha_of(P),
                            P->surfbuf, st);
      ck(fda::launch_gtrans(O.s2m, P->surfbuf, P->lv[O.level].X, st));
    }
    tr(st, "s2m", O.level);
  }
  mk.end(3);
  mk.begin(4);
  for (int t = (int)P->tr.size() - 1; t >= 0; --t) {
    const DevTrans& T = P->tr[t];
    ck(fda::launch_gtrans(T.up, P->lv[T.lp + 1].X, P->lv[T.lp].X, st));
    tr(st, "m2m", T.lp);
  }
  if (P->nranks > 1)
    fda::launch_xpack(P->xc.nsend, P->xc.s_xoff, P->xc.s_len, P->xc.s_boff, P->Xall, sendbuf, st);
  mk.end(4);
}

// H2 P2P + H3 correction on this rank's rows (outm of the other rows is cleared when they are not computed)
void stage_near(fda_plan P, uint32_t mask, cudaStream_t st, Marks& mk) {
  const bool partial = P->leaf_b > 0 || P->leaf_e < P->nleaf;
  mk.begin(1);
  // symmetric P2P (each leaf pair once, both directions; BM_H on a single-rank plan; FDA_P2P_SYM=0: off)
  const bool sym = (mask & FDA_PHASE_NEAR) && !partial && P->kind == 0 && !P->deterministic &&
                   !(getenv("FDA_P2P_SYM") && getenv("FDA_P2P_SYM")[0] == '0');
  if (!(mask & FDA_PHASE_NEAR) || partial || sym) ck(cudaMemsetAsync(P->outm, 0, (size_t)P->n * sizeof(double2), st));
  if (sym)
    fda::launch_p2p_sym(P->nleaf, P->leaf_ptr, P->p2p_ptr, P->p2p_src, points_of(P), P->q, P->H.k, alpha_of(P),
                        P->outm, st);
  else if (mask & FDA_PHASE_NEAR)
    fda::launch_p2p(P->kind, P->leaf_e - P->leaf_b, P->leaf_ptr, P->p2p_ptr, P->p2p_src, points_of(P), P->q, P->H.k,
                    alpha_of(P), P->outm, P->leaf_b, st);
  mk.end(1);
  mk.begin(2);
  if ((mask & FDA_PHASE_CORR) && P->nnz > 0)
    fda::launch_csr(P->pt_b, P->pt_e, P->c_ptr, P->c_col, P->c_val, P->phim, P->outm, st);
  mk.end(2);
}

// unpack of the received partial expansions, then H6 M2L, H7 L2L, H8 L2T into this rank's rows
void stage_down(fda_plan P, uint32_t mask, const double2* recvbuf, cudaStream_t st, Marks& mk, Trace& tr,
                cudaEvent_t near_done = nullptr) {
  if (!has_far(P, mask)) return;
  const fda::Points Pt = points_of(P);
  const fda::LeafGeom Lg = leaves_of(P);
  mk.begin(5);
  if (P->nranks > 1)
    fda::launch_xunpack(P->xc.ndst, P->xc.d_xoff, P->xc.d_len, P->xc.d_rptr, P->xc.d_roff, recvbuf, P->Xall, st);
  for (auto& D : P->lv)
    if (D.n_in) ck(cudaMemsetAsync(D.Y, 0, (size_t)D.n_in * D.s * sizeof(double2), st));
  for (size_t l = 0; l < P->lv.size(); ++l) {
    // stores: before the atomic launches into the same Y
    if (P->lv[l].m2lb.n_blocks) {
      ck(fda::launch_m2l_block(P->lv[l].m2lb, P->lv[l].X, P->tbuf, P->lv[l].Y, st, 1));
      tr(st, "m2l-pass1", (int)l);
      ck(fda::launch_m2l_block(P->lv[l].m2lb, P->lv[l].X, P->tbuf, P->lv[l].Y, st, 2));
      tr(st, "m2l-pass2", (int)l);
    }
    ck(fda::launch_gtrans(P->lv[l].m2l, P->lv[l].X, P->lv[l].Y, st));
    ck(fda::launch_gtrans(P->lv[l].m2l2, P->lv[l].X, P->lv[l].Y, st));
    if (P->lv[l].m2l.n_items || P->lv[l].m2lb.n_blocks) tr(st, "m2l", (int)l);
  }
  mk.end(5);
  mk.begin(6);
  for (const auto& T : P->tr) {
    ck(fda::launch_gtrans(T.dn, P->lv[T.lp].Y, P->lv[T.lp + 1].Y, st));
    tr(st, "l2l", T.lp);
  }
  mk.end(6);
  mk.begin(7);
  if (near_done) ck(cudaStreamWaitEvent(st, near_done, 0));  // L2T adds into the rows P2P / CSR wrote
  for (const auto& O : P->lo) {
    if (O.Tm) {  // stored T_leaf
      fda::launch_leaf_l2t(O.nleaves_own, O.leaf_own, O.pofs, O.slot, P->leaf_ptr, P->lv[O.level].Y, O.Tm, O.s,
                           P->outm, st);
      tr(st, "l2t", O.level);
      continue;
    }
    ck(cudaMemsetAsync(P->surfbuf, 0, (size_t)O.nleaves_own * O.nsurf * sizeof(double2), st));
    ck(fda::launch_gtrans(O.l2t, P->lv[O.level].Y, P->surfbuf, st));
    // E_dn = G + alpha dG/dn_x (BM_H, BM_G: PAPER.md eq_eval2t); the Table-1 kernel has no target
    // derivative: E_dn = G
    const double2 alpha_dn = P->kind == FDA_KERNEL_T1 ? make_double2(0.0, 0.0) : alpha_of(P);
    fda::launch_l2t_eval(O.nleaves_own, O.leaf_own, Lg, Pt, O.surf, O.nsurf, P->H.k, alpha_dn, P->surfbuf, P->outm,
                         st);
    tr(st, "l2t", O.level);
  }
  mk.end(7);
}

// kernels one apply launches (memsets excluded)
int64_t count_launches(fda_plan P, uint32_t mask) {
  int64_t L = 3;  // permute, p2p, unpermute
  if ((mask & FDA_PHASE_CORR) && P->nnz > 0) ++L;
  if (has_far(P, mask)) {
    for (const auto& O : P->lo) L += (O.Sm ? 2 : 4) * (O.nleaves_own > 0);
    for (const auto& T : P->tr) L += (T.up.n_items > 0) + (T.dn.n_items > 0);
    for (const auto& D : P->lv) L += (D.m2l.n_items > 0) + (D.m2l2.n_items > 0) + 2 * (D.m2lb.n_blocks > 0);
    if (P->nranks > 1) L += (P->xc.nsend > 0) + (P->xc.ndst > 0);
  }
  return L;
}

// multi-GPU exchange over NCCL: grouped send / receive of the partial expansions with every peer
void nccl_exchange(fda_plan P, cudaStream_t st) {
  const fda::Nccl& N = fda::nccl();
  auto& X = P->xc;
  auto nck = [](ncclResult_t r) {
    if (r != ncclSuccess) throw CudaFail{FDA_ERR_NCCL};
  };
  nck(N.GroupStart());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < P->nranks; ++q) {
    if (X.send_cnt[q]) nck(N.Send(X.sendbuf + so, 2 * (size_t)X.send_cnt[q], ncclDouble, q, P->comm, st));
    if (X.recv_cnt[q]) nck(N.Recv(X.recvbuf + ro, 2 * (size_t)X.recv_cnt[q], ncclDouble, q, P->comm, st));
    so += X.send_cnt[q], ro += X.recv_cnt[q];
  }
  nck(N.GroupEnd());
}
// multi-GPU output assembly: every rank broadcasts its own (contiguous, Morton-order) rows of outm
void nccl_allgather_out(fda_plan P, cudaStream_t st) {
  const fda::Nccl& N = fda::nccl();
  auto nck = [](ncclResult_t r) {
    if (r != ncclSuccess) throw CudaFail{FDA_ERR_NCCL};
  };
  nck(N.GroupStart());
  for (int q = 0; q < P->nranks; ++q) {
    const int64_t b = P->rank_pt[q], e = P->rank_pt[q + 1];
    if (e > b) nck(N.Broadcast(P->outm + b, P->outm + b, 2 * (size_t)(e - b), ncclDouble, q, P->comm, st));
  }
  nck(N.GroupEnd());
}

// the apply between the permute of phi and the unpermute of out: it touches plan buffers only
void apply_middle(fda_plan P, uint32_t mask, cudaStream_t st, Marks& mk, Trace& tr) {
  const bool xchg = P->nranks > 1 && has_far(P, mask);
  // the near field (P2P, correction: H2, H3) runs on the plan's side stream, concurrent with the far
  // field; L2T (which adds into the same rows) waits for it.  Timed applies run the phases in sequence.
  const bool overlap = !mk.on && !tr.on && has_far(P, mask);
  if (overlap) {
    ck(cudaEventRecord(P->ev_perm, st));
    ck(cudaStreamWaitEvent(P->nstream, P->ev_perm, 0));
    stage_near(P, mask, P->nstream, mk);
    ck(cudaEventRecord(P->ev_near, P->nstream));
  }
  stage_up(P, mask, P->xc.sendbuf, st, mk, tr);
  if (xchg && !mk.on) {
    // the exchange runs on the plan's exchange stream
    ck(cudaEventRecord(P->ev_up, st));
    ck(cudaStreamWaitEvent(P->xstream, P->ev_up, 0));
    nccl_exchange(P, P->xstream);
    ck(cudaEventRecord(P->ev_x, P->xstream));
    if (!overlap) stage_near(P, mask, st, mk);
    ck(cudaStreamWaitEvent(st, P->ev_x, 0));
  } else {
    mk.begin(9);
    if (xchg) nccl_exchange(P, st);
    mk.end(9);
    if (!overlap) stage_near(P, mask, st, mk);
  }
  stage_down(P, mask, P->xc.recvbuf, st, mk, tr, overlap ? P->ev_near : nullptr);
}

void drop_graphs(fda_plan P) {
  for (auto& kv : P->gexec) cudaGraphExecDestroy(kv.second);
  P->gexec.clear();
  P->gcalls.clear();
}

// replay (capturing it on first use) the CUDA graph of apply_middle for this mask on st; false: run it plainly.
// The first apply of a mask runs plainly (one-time launch setup: shared-memory attributes, constants), the
// second one is captured on the plan's capture stream.  A failed capture turns graphs off for the plan.
bool apply_graph(fda_plan P, uint32_t mask, cudaStream_t st) {
  auto it = P->gexec.find(mask);
  if (it == P->gexec.end()) {
    if (P->gcalls[mask]++ < 1) return false;
    Marks mk0;
    Trace tr0;
    tr0.on = false;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    ck(cudaStreamBeginCapture(P->gstream, cudaStreamCaptureModeRelaxed));
    bool ok = true;
    try {
      apply_middle(P, mask, P->gstream, mk0, tr0);
    } catch (const CudaFail&) {
      ok = false;
    }
    const cudaError_t e = cudaStreamEndCapture(P->gstream, &g);
    if (ok && e == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
      it = P->gexec.emplace(mask, ex).first;
    } else {
      ok = false;
    }
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      cudaGetLastError();
      P->graph_on = false;
      P->logstr += "CUDA graph capture of the apply failed; applies run without a graph\n";
      return false;
    }
  }
  ck(cudaGraphLaunch(it->second, st));
  return true;
}

fda_status check_apply_args(fda_plan P, const void* phi, const void* out) {
  if (!P || !phi || !out) return FDA_ERR_INVALID_ARG;
  if (P->host_only) return FDA_ERR_STATE;
  if (P->sticky_error) return FDA_ERR_CUDA;
  if (phi == out) return FDA_ERR_ALIAS;
  return FDA_OK;
}

}  // namespace

extern "C" {

static fda_status apply_impl(fda_plan P, uint32_t mask, const double* phi, double* out, float* phase_ms) {
  fda_status cs = check_apply_args(P, phi, out);
  if (cs != FDA_OK) return cs;
  // a partitioned plan without a communicator computes only its own rows and needs the expansions of the
  // other ranks: it is driven through fda_apply_up / fda_apply_down
  if (P->nranks > 1 && !P->comm) return FDA_ERR_STATE;
  const int64_t n = P->n;
  cudaStream_t st = P->stream;
  const bool dphi = is_device_ptr(phi), dout = is_device_ptr(out);
  if (phase_ms && (!dphi || !dout)) return FDA_ERR_INVALID_ARG;
  Marks mk;
  mk.st = st;
  mk.on = phase_ms != nullptr;
  try {
    const double2* d_phi = reinterpret_cast<const double2*>(phi);
    double2* d_out = reinterpret_cast<double2*>(out);
    if (!dphi) {
      ck(cudaMemcpyAsync(P->phi_buf, phi, (size_t)n * sizeof(double2), cudaMemcpyHostToDevice, st));
      // pinned host memory makes the copy asynchronous: the caller may reuse phi once we return, so wait
      // for it here when nothing below synchronises (device output)
      if (dout) ck(cudaStreamSynchronize(st));
      d_phi = P->phi_buf;
    }
    if (!dout) d_out = P->out_buf;
    if (mk.on)
      for (auto& e : mk.ev) ck(cudaEventCreate(&e));
    Trace tr;
    stage_permute(P, d_phi, st, mk);
    // CUDA graph of the middle on single-rank plans (untimed, untraced applies)
    const bool graph = P->graph_on && !mk.on && !tr.on && P->nranks == 1 && !P->comm;
    if (!(graph && apply_graph(P, mask, st))) apply_middle(P, mask, st, mk, tr);
    mk.begin(8);
    if (P->comm) nccl_allgather_out(P, st);
    fda::launch_unpermute(n, P->perm, P->outm, d_out, st);
    mk.end(8);
    ck(cudaGetLastError());
    P->last_launches = count_launches(P, mask);
    if (!dout) {
      ck(cudaMemcpyAsync(out, d_out, (size_t)n * sizeof(double2), cudaMemcpyDeviceToHost, st));
      ck(cudaStreamSynchronize(st));
    }
    if (mk.on) {
      ck(cudaEventSynchronize(mk.ev[2 * 8 + 1]));
      for (int i = 0; i < FDA_NPHASES; ++i) {
        phase_ms[i] = 0.f;
        if (cudaEventQuery(mk.ev[2 * i + 1]) == cudaSuccess &&
            cudaEventElapsedTime(&phase_ms[i], mk.ev[2 * i], mk.ev[2 * i + 1]) != cudaSuccess)
          phase_ms[i] = 0.f;
      }
      cudaGetLastError();
      for (auto& e : mk.ev) cudaEventDestroy(e);
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

fda_status fda_dist_counts(fda_plan P, int64_t* send_counts, int64_t* recv_counts) {
  if (!P || !send_counts || !recv_counts) return FDA_ERR_INVALID_ARG;
  for (int q = 0; q < P->nranks; ++q) {
    send_counts[q] = P->nranks > 1 ? P->xc.send_cnt[q] : 0;
    recv_counts[q] = P->nranks > 1 ? P->xc.recv_cnt[q] : 0;
  }
  return FDA_OK;
}

fda_status fda_apply_up(fda_plan P, const double* phi, double* sendbuf) {
  if (!P || !phi) return FDA_ERR_INVALID_ARG;
  if (P->host_only) return FDA_ERR_STATE;
  if (P->sticky_error) return FDA_ERR_CUDA;
  if (!is_device_ptr(phi) || (P->nranks > 1 && P->xc.send_tot > 0 && (!sendbuf || !is_device_ptr(sendbuf))))
    return FDA_ERR_INVALID_ARG;
  try {
    Marks mk;
    Trace tr;
    stage_permute(P, reinterpret_cast<const double2*>(phi), P->stream, mk);
    stage_up(P, FDA_PHASE_ALL, reinterpret_cast<double2*>(sendbuf), P->stream, mk, tr);
    ck(cudaGetLastError());
  } catch (const CudaFail& f) {
    P->sticky_error = true;
    return f.s;
  }
  return FDA_OK;
}

fda_status fda_apply_down(fda_plan P, const double* recvbuf, double* out) {
  if (!P || !out) return FDA_ERR_INVALID_ARG;
  if (P->host_only) return FDA_ERR_STATE;
  if (P->sticky_error) return FDA_ERR_CUDA;
  if (!is_device_ptr(out) || (P->nranks > 1 && P->xc.recv_tot > 0 && (!recvbuf || !is_device_ptr(recvbuf))))
    return FDA_ERR_INVALID_ARG;
  try {
    Marks mk;
    Trace tr;
    cudaStream_t st = P->stream;
    stage_near(P, FDA_PHASE_ALL, st, mk);
    stage_down(P, FDA_PHASE_ALL, reinterpret_cast<const double2*>(recvbuf), st, mk, tr);
    fda::launch_unpermute(P->n, P->perm, P->outm, reinterpret_cast<double2*>(out), st);
    ck(cudaGetLastError());
    P->last_launches = count_launches(P, FDA_PHASE_ALL);
  } catch (const CudaFail& f) {
    P->sticky_error = true;
    return f.s;
  }
  return FDA_OK;
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

fda_status fda_nccl_unique_id(char* id) {
  if (!id) return FDA_ERR_INVALID_ARG;
  const fda::Nccl& N = fda::nccl();
  if (!N.ok) return FDA_ERR_NCCL;
  ncclUniqueId u;
  if (N.GetUniqueId(&u) != ncclSuccess) return FDA_ERR_NCCL;
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return FDA_OK;
}

fda_status fda_plan_create_dist(int64_t n, const double* points, const double* normals, const double* quad_weights,
                                double k, double alpha_re, double alpha_im, double eps, const fda_options* opt,
                                const char* nccl_id, int rank, int nranks, fda_plan* out) {
  if (!out || !nccl_id || nranks < 1 || rank < 0 || rank >= nranks || nranks > 64) return FDA_ERR_INVALID_ARG;
  *out = nullptr;
  fda_options o;
  fda_options_default(&o);
  if (opt) o = *opt;
  if (o.host_only) return FDA_ERR_INVALID_ARG;
  o.rank = rank, o.nranks = nranks;
  const fda::Nccl& N = fda::nccl();
  if (!N.ok) return FDA_ERR_NCCL;
  fda_plan P = nullptr;
  fda_status s = fda_plan_create_ex(n, points, normals, quad_weights, k, alpha_re, alpha_im, eps, &o, &P);
  if (s != FDA_OK) return s;
  ncclUniqueId u;
  std::memcpy(u.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
  if (N.CommInitRank(&P->comm, nranks, u, rank) != ncclSuccess) {
    P->comm = nullptr;
    fda_plan_destroy(P);
    return FDA_ERR_NCCL;
  }
  if (cudaStreamCreateWithFlags(&P->xstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_up, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&P->ev_x, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    fda_plan_destroy(P);
    return FDA_ERR_CUDA;
  }
  *out = P;
  return FDA_OK;
}

fda_status fda_plan_export_exchange(fda_plan P, int peer, int recv, int64_t* count, int32_t* level, int64_t* slot,
                                    int64_t* cube_ijk) {
  if (!P || !count || peer < 0 || peer >= P->nranks) return FDA_ERR_INVALID_ARG;
  if (P->nranks == 1) {
    *count = 0;
    return FDA_OK;
  }
  const auto& v = recv ? P->xc.recv[peer] : P->xc.send[peer];
  *count = (int64_t)v.size();
  for (size_t i = 0; i < v.size(); ++i) {
    const fda::Level& L = P->H.levels[v[i].first];
    if (level) level[i] = v[i].first;
    if (slot) slot[i] = v[i].second;
    if (cube_ijk)
      for (int d = 0; d < 3; ++d) cube_ijk[3 * i + d] = P->H.cubes[L.cubes[L.out_cube[v[i].second]]].ijk[d];
  }
  return FDA_OK;
}

fda_status fda_plan_destroy(fda_plan P) {
  if (!P) return FDA_ERR_INVALID_ARG;
  if (P->comm) fda::nccl().CommDestroy(P->comm);
  if (P->ev_up) cudaEventDestroy(P->ev_up);
  if (P->ev_x) cudaEventDestroy(P->ev_x);
  if (P->xstream) cudaStreamDestroy(P->xstream);
  drop_graphs(P);
  if (P->gstream) cudaStreamDestroy(P->gstream);
  if (P->ev_perm) cudaEventDestroy(P->ev_perm);
  if (P->ev_near) cudaEventDestroy(P->ev_near);
  if (P->nstream) cudaStreamDestroy(P->nstream);
  free_plan(P);
  delete P;
  return FDA_OK;
}

}  // extern "C"
