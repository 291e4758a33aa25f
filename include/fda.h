/*
 * fda.h -- C ABI of the B200 FDA Burton-Miller apply (libfda.so).
 *
 * The library applies the Nystrom-discretised Burton-Miller operator H of
 * Cao, Wen, Xiao & Liu (arXiv 1311.5202) with the fast directional algorithm:
 *
 *   out_i = sum_{j != i} w_j K(x_i, n_i; x_j, n_j) phi_j + sum_{p in row i} val_p phi_{col_p}
 *
 *   K = dG/dn_y + alpha d2G/(dn_x dn_y),  G = e^{ikr}/(4 pi r)      PAPER.md:352-355 (eq_hmat), 210-212
 *   (or, with fda_options.kernel = FDA_KERNEL_BMG, K = G + alpha dG/dn_x, PAPER.md:356-358 eq_gmat)
 *   far quadrature w_j K(x_i, y_j)                                  PAPER.md:291-297 (eq:far field)
 *   locally corrected kernel K-bar inside D_i, supplied by the caller
 *   as a delta CSR (the "val" term)                                 PAPER.md:329-341 (eq:sum, kcorrection)
 *
 * The first term is approximated by the FDA (near-field P2P + S2M / M2M /
 * M2L / L2L / L2T) to the accuracy eps;
 * the CSR term is exact.  Targets are the sources themselves (Nystrom
 * collocation).  Everything of the apply runs in this library's CUDA kernels
 * (sm_100a); there is no CPU fallback: without a CUDA device every call that
 * needs one returns FDA_ERR_CUDA.
 *
 * Layout and ownership
 *   points, normals : n x 3 doubles, xyz interleaved, caller order; normals unit, outward.
 *   quad_weights    : n doubles, > 0 (rule weight x Jacobian).
 *   phi, out        : n complex128 (2n doubles, re/im interleaved), caller order.
 *   Any array argument may be host memory (pageable or pinned) or device memory
 *   of the current device; the library detects which (cudaPointerGetAttributes).
 *   fda_plan_create / fda_plan_set_correction COPY their inputs: the caller may
 *   free them on return.  The plan owns all device workspace.
 *
 * Errors: every function returns an fda_status; nothing throws across the ABI.
 *   FDA_ERR_INVALID_ARG   bad sizes / null pointers / non-finite values / |n| != 1 (1e-10) /
 *                         w <= 0 / eps not in [1e-10, 1e-1] / k < 0 / (k == 0 and alpha != 0) /
 *                         CSR with non-monotone row_ptr or col outside [0, n) / unknown kernel kind /
 *                         rank not in [0, nranks) or nranks not in [1, 64]
 *   FDA_ERR_COINCIDENT_POINTS  two distinct points closer than 1e-14 x root width
 *   FDA_ERR_ALIAS         phi and out are the same buffer
 *   FDA_ERR_CUDA          a CUDA error (sticky: destroy the plan)
 *   FDA_ERR_OOM           device allocation failed
 *   FDA_ERR_SETUP_ACCURACY the plan cannot reach eps on this device (a translation launch needs more shared
 *                         memory than the device has, at very small eps)
 *   FDA_ERR_NCCL          NCCL missing or a collective failed (multi-GPU plans)
 *   FDA_ERR_STATE         call not valid for this plan (host_only plan; fda_apply on a partitioned plan
 *                         without communicator)
 * Threading: one apply in flight per plan; the device-pointer apply is ordered on
 * the plan's stream (fda_plan_set_stream) and does not synchronise the host.
 */
#ifndef FDA_H
#define FDA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fda_plan_s* fda_plan;

typedef enum {
  FDA_OK = 0,
  FDA_ERR_INVALID_ARG = 1,
  FDA_ERR_COINCIDENT_POINTS = 2,
  FDA_ERR_ALIAS = 3,
  FDA_ERR_CUDA = 4,
  FDA_ERR_OOM = 5,
  FDA_ERR_SETUP_ACCURACY = 6,
  FDA_ERR_NCCL = 7,
  FDA_ERR_STATE = 8
} fda_status;

/* number of phase times fda_apply_timed writes */
#define FDA_NPHASES 10

/* phase mask for fda_apply_phases (tests / diagnostics) */
#define FDA_PHASE_NEAR 1u /* P2P over the plan's near leaf pairs (H2)             */
#define FDA_PHASE_CORR 2u /* correction CSR (H3)                                   */
#define FDA_PHASE_FAR 4u  /* S2M, M2M, M2L, L2L, L2T (H4-H8)                        */
#define FDA_PHASE_ALL 7u

/* operator of the plan (fda_options.kernel) */
#define FDA_KERNEL_BMH 0 /* Burton-Miller H: dipole sources, target (1 + alpha d/dn_x)    */
#define FDA_KERNEL_BMG 1 /* Burton-Miller G: monopole sources, target (1 + alpha d/dn_x)  */
#define FDA_KERNEL_T1 2  /* Table-1 summation kernel G + alpha dG/dn_y (eq_sum):
                            monopole + dipole sources, no target derivative                */

/* Plan knobs (all optional; fda_options_default fills the defaults). */
typedef struct {
  int32_t leaf_size;       /* N_p; 0 -> max(30, 50(-log10 eps - 3))  (eq_npleaf, sign-corrected) */
  double eps_internal;     /* expansion truncation (R+ SVDs, HF interpolative selection); 0 -> eps / 100 (R11) */
  int32_t lf_p_low;        /* LF surface points per cube edge below lf_p_switch; 0 (default) -> 6 + dp (7 + dp
                              below w = lambda / 4) with dp = round(log10(1e-4 / eps)) for eps < 1e-4, else 0
                              (R17); a value > 1 is used verbatim */
  int32_t lf_p_high;       /* ... at or above lf_p_switch wavelengths; 0 (default) -> 8 + dp */
  double lf_p_switch;      /* w / lambda switch (default 0.75) */
  int32_t lowrank;         /* low-rank M2L when rank < s/2, default 1 */
  int32_t single_leaf;     /* debug: no far field, every pair P2P (default 0) */
  int32_t hf_max_rows;     /* HF directional-set sample rows; 0 (default): 6000 x (1 + decades of eps below 1e-4) */
  double hf_spacing;       /* HF candidate spacing in wavelengths (default 0.25) */
  int32_t rank, nranks;    /* multi-GPU: this rank owns the rank-th of nranks Morton ranges of leaves (default 0/1);
                              nranks <= 64; see fda_plan_create_dist / fda_apply_up */
  int32_t verbose;         /* plan log (fda_plan_log) */
  double eps_lowrank;      /* low-rank M2L truncation sigma_i < eps_lowrank sigma_1; 0 -> eps, 10x tighter
                              on the low-frequency LF levels (R23) */
  int32_t kernel;          /* FDA_KERNEL_BMH (default): K = dG/dn_y + alpha d2G/dn_x dn_y (eq_hmat);
                              FDA_KERNEL_BMG: K = G + alpha dG/dn_x (eq_gmat);
                              FDA_KERNEL_T1: K = G + alpha dG/dn_y (eq_sum; Table 1 mode,
                              SURVEY §8(f) row 2: pass unit weights and no correction for the paper's summation) */
  int32_t host_only;       /* diagnostics: build the host plan only (tree, lists, operators), no device;
                              fda_apply* then returns FDA_ERR_STATE.  Lets CPU tests audit the lists. */
  int32_t original;        /* 1: the paper's "original" FDA for Table 1: expansions are the
                              equivalent densities (no SVD reduction of the basis), dense unreduced M2L, no low
                              rank (R24); default 0 = the improved FDA */
  int32_t graph;           /* 1 (default): fda_apply replays a CUDA graph of its device-resident middle (near field,
                              upward pass, M2L, L2L, L2T; captured on the second apply of a phase mask, single-rank
                              plans; fda_plan_set_correction drops it); 0 (or env FDA_GRAPH=0): plain launches */
  int32_t deterministic;   /* 1: bit-reproducible applies -- every translation runs as owned items (an item owns its
                              output slots: plain read-modify-write in a fixed order instead of FP64 reductions) and
                              the P2P one-sided; equal to the default apply to rounding (3e-16) and 2.6x slower at
                              config 5 (565 vs 218 ms); default 0 */
} fda_options;

typedef struct {
  int64_t n, nleaves, nlevels, lmin;
  int64_t p2p_leaf_pairs, p2p_point_pairs;
  int64_t m2l_pairs, m2l_groups, m2l_lowrank_groups;
  int64_t out_slots, in_slots;
  int64_t csr_nnz;
  int64_t device_bytes;
  int64_t owned_begin, owned_end; /* owned points, Morton order */
  int64_t owned_leaf_begin, owned_leaf_end; /* owned leaves (Morton leaf ids of fda_plan_export_leaves) */
  double setup_tree_s, setup_lists_s, setup_ops_s, setup_upload_s;
  double flops_p2p, flops_m2l, flops_m2m, flops_l2l, flops_s2m, flops_l2t; /* algorithmic flops per apply */
  double bytes_csr;                                                        /* algorithmic bytes of H3 per apply */
  int64_t s2m_evals, l2t_evals;               /* kernel evaluations of the S2M / L2T surface phases per apply */
  int64_t xchg_send_bytes, xchg_recv_bytes;   /* multi-GPU: expansion bytes this rank sends / receives per apply */
  int64_t m2l_ops;  /* distinct M2L operators stored: (offset, wedge) groups related by a cube symmetry share one
                       (the wedges' point sets are rotations of one set), m2l_ops <= m2l_groups */
  double bytes_s2m, bytes_l2t;  /* algorithmic bytes per apply of the stored leaf S2M / L2T matrices (PAPER.md:979-980:
                                   "precomputed and saved in memory"); 0 when the kernels are evaluated on the fly */
} fda_stats;

void fda_options_default(fda_options* opt);

/* Build a plan (tree, lists, wedges, translation operators) and upload it.
 * k >= 0 wavenumber; alpha = alpha_re + i alpha_im (Burton-Miller coupling, i/k in the paper);
 * eps in [1e-10, 1e-1] target accuracy of the far field. */
fda_status fda_plan_create(int64_t n, const double* points, const double* normals, const double* quad_weights,
                           double k, double alpha_re, double alpha_im, double eps, fda_plan* out);
fda_status fda_plan_create_ex(int64_t n, const double* points, const double* normals, const double* quad_weights,
                              double k, double alpha_re, double alpha_im, double eps, const fda_options* opt,
                              fda_plan* out);

/* Singular-correction CSR in caller order: row_ptr (n+1, int64, row_ptr[0] = 0, monotone, row_ptr[n] = nnz),
 * col (nnz, int32 in [0,n)), val (nnz complex128, interleaved).  Copied into the plan (Morton order).
 * nnz = 0 removes it. */
fda_status fda_plan_set_correction(fda_plan plan, int64_t nnz, const int64_t* row_ptr, const int32_t* col,
                                   const double* val);

/* out = H phi.  phi / out: n complex128 each, caller order, host or device. */
fda_status fda_apply(fda_plan plan, const double* phi, double* out);
/* Same, restricted to the phases in mask (FDA_PHASE_*). */
fda_status fda_apply_phases(fda_plan plan, uint32_t mask, const double* phi, double* out);
/* Same as fda_apply_phases, with CUDA-event time per phase written to phase_ms[0..FDA_NPHASES-1]:
 * permute, p2p, csr, s2m, m2m (+ pack), m2l (+ unpack), l2l, l2t, unpermute (+ output all-gather), exchange
 * (device pointers only; synchronises; phases run one after another, without the exchange overlap). */
fda_status fda_apply_timed(fda_plan plan, uint32_t mask, const double* phi, double* out, float* phase_ms);

/* Order the plan's device work on this cudaStream_t (default: the legacy default stream). */
fda_status fda_plan_set_stream(fda_plan plan, void* stream);
fda_status fda_plan_stats(fda_plan plan, fda_stats* stats);
const char* fda_plan_log(fda_plan plan);
/* Number of CUDA kernels the last apply on this plan launched (memsets excluded); -1 for a null plan. */
int64_t fda_plan_launches(fda_plan plan);

/* Diagnostics for the list audit (host arrays; pass NULL arrays to query sizes).
 * leaf_of_point: n (caller order); leaf_level / leaf_ijk: per leaf (ijk: 3 int64). */
fda_status fda_plan_export_leaves(fda_plan plan, int64_t* nleaves, int32_t* leaf_of_point, int32_t* leaf_level,
                                  int64_t* leaf_ijk);
/* The exact (target leaf, source leaf) pairs the P2P phase sums. */
fda_status fda_plan_export_p2p(fda_plan plan, int64_t* npairs, int32_t* tgt_leaf, int32_t* src_leaf);
/* The M2L cube pairs: level, target cube ijk (3), source cube ijk (3). */
fda_status fda_plan_export_m2l(fda_plan plan, int64_t* npairs, int32_t* level, int64_t* tgt_ijk, int64_t* src_ijk);

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU.  Rank q of R owns a contiguous Morton range of leaves (cut by estimated work) and
 * computes the rows of out in it: P2P, correction, S2M on its leaves, M2M on the cubes holding its points
 * (partial expansions: M2M is linear), M2L into target cubes holding its points, L2L, L2T.  Before M2L each
 * rank receives from the other ranks of every source cube it reads their partial outgoing expansions
 * (the upward pass of PAPER.md:519-523 split by points, summed on arrival) -- one grouped NCCL
 * send/receive per apply, overlapped with P2P and the correction -- and after L2T the ranks' rows are
 * all-gathered, so every rank returns the full out. */

/* 128-byte NCCL unique id (ncclGetUniqueId); rank 0 makes it, the caller distributes it.
 * FDA_ERR_NCCL if libnccl.so.2 cannot be loaded. */
fda_status fda_nccl_unique_id(char* id);
/* Collective over the nranks processes (each on its own current device): builds the same plan on every rank
 * (opt->rank / opt->nranks are overridden) and the NCCL communicator.  fda_apply on the plan then returns the
 * full out on every rank.  Errors as fda_plan_create_ex, FDA_ERR_NCCL if the communicator fails. */
fda_status fda_plan_create_dist(int64_t n, const double* points, const double* normals, const double* quad_weights,
                                double k, double alpha_re, double alpha_im, double eps, const fda_options* opt,
                                const char* nccl_id, int rank, int nranks, fda_plan* out);

/* The exchange without NCCL (tests, other transports).  A plan made by fda_plan_create_ex with
 * opt.nranks > 1 (no communicator) rejects fda_apply (FDA_ERR_STATE) and is applied in two halves:
 *   fda_dist_counts: complex128 elements this rank sends to / receives from each peer (nranks entries each);
 *   fda_apply_up:    permute + S2M + M2M, packs the partial expansions into sendbuf (device, peer-major);
 *   fda_apply_down:  adds recvbuf (device, peer-major; the bytes peer q sent to this rank, in q order), then
 *                    P2P, correction, M2L, L2L, L2T; out (device, caller order) holds this rank's rows, the
 *                    other rows zero.
 * Device pointers only (FDA_ERR_INVALID_ARG otherwise); stream-ordered like fda_apply. */
fda_status fda_dist_counts(fda_plan plan, int64_t* send_counts, int64_t* recv_counts);
fda_status fda_apply_up(fda_plan plan, const double* phi, double* sendbuf);
fda_status fda_apply_down(fda_plan plan, const double* recvbuf, double* out);
/* Diagnostics (also for host_only plans): the exchange list with peer (recv = 0: what this rank sends to peer,
 * 1: what it receives from peer) in buffer order: level, out slot and cube ijk (3 per entry). */
fda_status fda_plan_export_exchange(fda_plan plan, int peer, int recv, int64_t* count, int32_t* level, int64_t* slot,
                                    int64_t* cube_ijk);

/* Locally corrected Nystrom weights on the device.
 * For every listed pair (field point t, element e) with the field point OFF the element, the six weights
 *   wbar_j^Delta(K; x_t),  sum_j wbar_j phi^(n)(xi_j) = int_Delta K(x_t, y) phi^(n)(y) dy,
 *   phi^(n) = xi1^p xi2^q, p + q <= 2, (p,q) = (0,0),(1,0),(0,1),(2,0),(1,1),(0,2)
 * with the nearly singular moments computed by recursive subdivision quadrature: a sub-triangle of
 * the reference triangle is split at its edge mid-points while its largest mapped edge h exceeds theta x the
 * distance from x_t to the nearest of its mapped corners and centroid, or while the element map is not flat on it
 * (|y(centroid) - mean of the mapped corners| > gamma h); leaves take the nq x nq Gauss-Legendre product rule on
 * the collapsed square (R27).  The self element (x_t on Delta) is singular / hyper-
 * singular and needs the method of [rjj_int], which the paper does not give: such a pair
 * makes the call return FDA_ERR_INVALID_ARG (outputs then unspecified).
 *   kernel        FDA_KERNEL_BMH / _BMG / _T1; k >= 0; alpha = alpha_re + i alpha_im
 *   elem_nodes    ne x 6 x 3 doubles: corners 1 2 3 then mid-edge nodes 12 23 31 of each quadratic triangle
 *                 (counter-clockwise seen from outside: n_y = t_1 x t_2 / |t_1 x t_2|)
 *   xi, wref      the element rule: 6 x 2 intrinsic coordinates (xi1, xi2) on the reference triangle
 *                 xi1, xi2 >= 0, xi1 + xi2 <= 1, and 6 reference weights (sum 1/2; w_j = wref_j J(xi_j))
 *   tx, tn        nt x 3 field points and their unit normals
 *   pair_t/pair_e npairs indices into tx / elem_nodes (int64)
 *   nq, theta, gamma, max_depth   0 selects the defaults 8, 0.5, 0.05, 16; limits nq <= 16, theta in (0, 1],
 *                 gamma > 0 (a large value switches the flatness split off), max_depth <= 20
 *   wbar          npairs x 6 complex128 (12 doubles per pair), the weights; may be NULL
 *   delta         npairs x 6 complex128, wbar_j - w_j K(x_t, y_j): the value the correction CSR of
 *                 fda_plan_set_correction holds for (row t, column of node j of e); may be NULL (not both)
 * Arrays may be host or device memory; the call runs on the default stream and synchronises (concurrent calls are
 * serialised).  Errors: FDA_ERR_INVALID_ARG (arguments, an index
 * out of range, a field point on its element), FDA_ERR_CUDA (no device / CUDA error), FDA_ERR_OOM. */
fda_status fda_nystrom_weights(int kernel, double k, double alpha_re, double alpha_im, const double* elem_nodes,
                               int64_t ne, const double* xi, const double* wref, const double* tx, const double* tn,
                               int64_t nt, const int64_t* pair_t, const int64_t* pair_e, int64_t npairs, int nq,
                               double theta, double gamma, int max_depth, double* wbar, double* delta);

fda_status fda_plan_destroy(fda_plan plan);
const char* fda_status_str(fda_status s);

#ifdef __cplusplus
}
#endif
#endif /* FDA_H */
