// kernels.cuh -- device kernels of the FDA Burton-Miller apply (sm_100a, FP64).
//
// Notation:
//   H1 permute+weight   H2 P2P near   H3 correction SpMV   H4 S2M (dipole E_up)
//   H5 M2M   H6 M2L (dense / low-rank)   H7 L2L (= M2M^T)   H8 L2T (E_dn = G + alpha dG/dn_x)
//   H9 unpermute
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GT_SMEM_BUDGET (112 * 1024)  // shared memory per CTA of the translation kernels: two CTAs (16 warps) per SM

namespace fda {

struct LeafGeom {        // leaves in Morton order; leaf t owns points [ptr[t], ptr[t+1])
  const int64_t* ptr;
  const double* cx;      // leaf centres
  const double* cy;
  const double* cz;
};

struct Points {
  const double *x, *y, *z, *nx, *ny, *nz, *w;
};

void launch_permute_scale(int64_t n, const int32_t* perm, const double* w, const double2* phi, double2* q,
                          double2* phim, cudaStream_t st);
void launch_unpermute(int64_t n, const int32_t* perm, const double2* outm, double2* out, cudaStream_t st);
// multi-GPU expansion exchange: gather send entries of the concatenated outgoing expansions X into buf;
// add each destination slot's received partial sums (CSR rptr/roff into buf, peer order) into X
void launch_xpack(int64_t nent, const int64_t* xoff, const int32_t* len, const int64_t* boff, const double2* X,
                  double2* buf, cudaStream_t st);
void launch_xunpack(int64_t ndst, const int64_t* xoff, const int32_t* len, const int64_t* rptr, const int64_t* roff,
                    const double2* buf, double2* X, cudaStream_t st);
// kind 0: BM_H kernel (dG/dn_y + alpha d2G/dn_x dn_y), 1: BM_G kernel (G + alpha dG/dn_x),
// 2: Table-1 kernel (G + alpha dG/dn_y)
void launch_p2p(int kind, int64_t nleaf, const int64_t* leaf_ptr, const int64_t* p2p_ptr, const int32_t* p2p_src,
                Points P, const double2* q, double k, double2 alpha, double2* outm, int64_t tgt_leaf_begin,
                cudaStream_t st);
// symmetric P2P of the BM_H kernel over the whole plan (single rank): outm must be zeroed first (FP64 reductions)
void launch_p2p_sym(int64_t nleaf, const int64_t* leaf_ptr, const int64_t* p2p_ptr, const int32_t* p2p_src, Points P,
                    const double2* q, double k, double2 alpha, double2* outm, cudaStream_t st);
void launch_csr(int64_t row_begin, int64_t row_end, const int64_t* rp, const int32_t* col, const double2* val,
                const double2* phim, double2* outm, cudaStream_t st);
// H4: check potentials chk[t][i] of leaf leaf_ids[t] on its check surface (nsurf points, relative):
// kind 0 dipole sources (dG/dn_y), 1 monopole sources (G), 2 monopole + alpha dipole (G + alpha dG/dn_y)
void launch_s2m_check(int kind, int64_t nleaves, const int32_t* leaf_ids, LeafGeom L, Points P, const double2* q,
                      const double* surf, int nsurf, double k, double2 alpha, double2* chk, cudaStream_t st);
// H8: out += E_dn rho over the leaves' equivalent surfaces; rho[t][b] for leaf leaf_ids[t]
void launch_l2t_eval(int64_t nleaves, const int32_t* leaf_ids, LeafGeom L, Points P, const double* surf, int nsurf,
                     double k, double2 alpha, const double2* rho, double2* outm, cudaStream_t st);
// Stored leaf S2M / L2T matrices ("precomputed and saved in memory"): rows per point of the
// owned leaves of one LF level, pofs[t] = first row of owned leaf t.  launch_leafmat builds Sm = (Sigma^-1 U^H)
// E_up (Sred: s x nsurf column-major) and Tm = E_dn (conj(U) Sigma^-1) (TredT: nsurf x s row-major); the apply
// kernels then compute X[slot] = S_leaf q and out += T_leaf Y[slot].
void launch_leafmat(int kind, int64_t nleaves, const int32_t* leaf_ids, const int64_t* pofs, LeafGeom L, Points P,
                    const double* surf, int nsurf, double k, double2 alpha, double2 alpha_dn, const double2* Sred,
                    const double2* TredT, int s, double2* Sm, double2* Tm, cudaStream_t st);
void launch_leaf_s2m(int64_t nleaves, const int32_t* leaf_ids, const int64_t* pofs, const int32_t* slot,
                     const int64_t* lptr, const double2* q, const double2* Sm, int s, double2* X, cudaStream_t st);
void launch_leaf_l2t(int64_t nleaves, const int32_t* leaf_ids, const int64_t* pofs, const int32_t* slot,
                     const int64_t* lptr, const double2* Y, const double2* Tm, int s, double2* outm, cudaStream_t st);
// Grouped translation (H5 M2M, H6 M2L, H7 L2L): one CTA per work item; an item owns a
// disjoint set of output slots and walks a list of groups, each group = one matrix
// (dense s_out x s_in, or low-rank U (s_out x r) V (r x s_in)) applied to its pairs:
//   Y[out_slot] += A X[in_slot]   (no atomics: outputs are owned by the item)
// Matrices are stored in DMMA fragment order (8x4 tiles, 32 re then 32 im doubles per tile,
// tiles row-tile-major); a low-rank group stores V (pad8(r) x pad4(s_in)) then U (pad8(s_out) x pad8(r)).
struct GTrans {
  int64_t n_items = 0;
  const int32_t* item_order = nullptr;  // launch order (largest first)
  const int64_t* item_ptr = nullptr;    // item -> [ig begin, ig end)
  const int32_t* ig_group = nullptr;    // item-group entry -> group
  const int64_t* ig_pb = nullptr;       // item-group entry -> pair range
  const int64_t* ig_pe = nullptr;
  const int32_t* out = nullptr;         // pair -> output slot
  const int32_t* in = nullptr;          // pair -> input slot
  const int32_t* grank = nullptr;       // group -> -1 (dense) or r
  const int64_t* gmat = nullptr;        // group -> matrix offset (doubles) into pool
  const double* pool = nullptr;         // fragment-order matrices
  const int16_t* gso = nullptr;         // group -> its own output / input expansion length (<= s_out / s_in;
  const int16_t* gsi = nullptr;         //   the rest of the padded operator is zero); null: s_out / s_in
  int s_out = 0, s_in = 0, rmax8 = 0;   // rmax8: largest low rank rounded up to 8
  int64_t mmax = 0;                     // largest matrix block of a group (doubles): shared-memory staging
  int all_lowrank = 0;                  // every group low rank (warp-specialised kernel)
  int ct1 = 0, ct2 = 0;                 // warp-unit column tiles (experiments: FDA_GT_CT1 / FDA_GT_CT2; 0 = default, -1 = balance)
  int atomic = 0;   // 1: items are (group, pair chunk) and accumulate with atomics (few pairs per group)
  int warp_tasks = 0;  // 1: low-rank M2L items for the warp-task kernel (m2l_warp.cu; chosen at plan time)
  int sector = 0;      // warp-task kernel: sector-complete FP64 reductions (the plan sets it on the LF levels)
};
cudaError_t launch_gtrans(const GTrans& T, const double2* X, double2* Y, cudaStream_t st);

// Two-pass M2L of the low-rank groups (m2l_block.cu).  Pass 1: items (group, <= 2048 pairs) compute
// T_p = V_o x_s and store it at the pair's position in pass-2 order (ld = ldt).  Pass 2: a block is <= bmax
// output slots of one direction (Morton-consecutive); its pairs, sorted by group, are cut into chunks of <= 32
// pairs of one group.  One CTA per block keeps the block's Y rows in shared memory and stores them once:
// Y[slot] = sum over the block's pairs of U_o T_p (overwrites -- launch it before any atomic contribution to
// the same Y).
struct BTrans {
  int64_t n_blocks = 0, n_chunks = 0, n_pairs = 0, n_items1 = 0;
  // pass 2
  const int32_t* blk_order = nullptr;  // launch order (Morton order of the block's first cube)
  const int64_t* blk_sptr = nullptr;   // block -> [begin, end) into blk_slot
  const int32_t* blk_slot = nullptr;   // output slots; local index = position - blk_sptr[block]
  const int64_t* blk_cptr = nullptr;   // block -> [begin, end) into the chunks
  const int64_t* ch_ptr = nullptr;     // chunk -> [begin, end) into the pass-2 pairs (<= 32) = T columns
  const int32_t* ch_group = nullptr;   // chunk -> group
  const uint8_t* ch_loc = nullptr;     // chunk -> 32 local output indices (block-relative) of its pairs
  // pass 1
  const int32_t* it_group = nullptr;   // item -> group
  const int64_t* it_ptr = nullptr;     // item -> [it_ptr, it_end) into the pass-1 pairs (group-major)
  const int64_t* it_end = nullptr;
  const int32_t* p1_in = nullptr;      // pass-1 pair -> input slot
  const int32_t* p1_out = nullptr;     // pass-1 pair -> T column (its pass-2 position)
  // groups
  const int32_t* grank = nullptr;      // group -> low rank r (pad8(r) <= 24)
  const int64_t* gmat = nullptr;       // group -> V (pad8(r) x pad4(s_in)) then U, fragment order (as GTrans)
  const double* pool = nullptr;
  const int16_t* gso = nullptr;        // group -> own output / input expansion length (null: s_out / s_in)
  const int16_t* gsi = nullptr;
  int s_out = 0, s_in = 0, rmax8 = 0, bmax = 0, ldt = 0;  // ldt: T column stride (complex128), = 4 mod 8
};
// pass 1 into T (ldt x n_pairs complex128), then pass 2 into Y (passes: bit 0 pass 1, bit 1 pass 2)
cudaError_t launch_m2l_block(const BTrans& B, const double2* X, double2* T, double2* Y, cudaStream_t st,
                             int passes = 3);
size_t m2l_block_smem(int s_out, int rmax8, int bmax);
int m2l_block_ldt(int rmax8);
// largest block (output slots) whose Y rows fit next to the T ring within smem_limit; 0 if rmax8 > 24
// (those groups stay with launch_gtrans)
int m2l_block_bmax(int s_out, int rmax8, size_t smem_limit);
// Low-rank M2L with warp-independent 8-pair tasks and the group's operator staged in shared memory
// (m2l_warp.cu); launch_gtrans takes it for all-low-rank atomic items when m2l_warp_fits (FDA_M2L_WARP=0: off)
bool m2l_warp_on();
bool m2l_warp_fits(const GTrans& T);
int m2l_warp_rmax(int s_out, int s_in, size_t smem_limit);  // largest pad8 rank whose operator fits smem_limit
cudaError_t launch_m2l_warp(const GTrans& T, const double2* X, double2* Y, cudaStream_t st);
size_t gtrans_smem(const GTrans& T);  // dynamic shared memory of one CTA
bool gtrans_fits(const GTrans& T);    // gtrans_smem(T) within the device's opt-in shared-memory limit
int gtrans_cols(const GTrans& T);     // pair columns per chunk (16 or 32)
int gtrans_ws_rmax(int s_in);         // largest (pad8) low rank the warp-specialised kernel takes
size_t smem_optin_bytes();            // opt-in shared memory per CTA of the current device

}  // namespace fda
