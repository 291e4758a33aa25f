// plan.hpp -- host-side plan of the FDA Burton-Miller apply.
//
// The plan holds everything that depends on the geometry, k, alpha and eps but
// not on the density phi ("the matrices of the M2M, M2L and
// L2L translations are computed only once and then stored"):
//   P0  Morton order of the points, each leaf a contiguous range
//   P1  adaptive octree, N_p split, LF/HF regimes, HF cubes split
//   P2  near (P2P) lists, interaction lists I^C = N^P \ N^C, wedges
//   P3  translation operators: LF surfaces, HF directional sets,
//       truncated-SVD pseudo-inverses, reduced S~ M~ K~ T~, low-rank K~
// It is built on the host (C++/OpenMP) once and uploaded; see DESIGN.md.
#pragma once
#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "linalg.hpp"

namespace fda {

struct Options {
  int np = 0;               // leaf threshold N_p; 0 -> from eps (eq_npleaf, sign-corrected)
  double eps_int = 0;       // expansion truncation tolerance; 0 -> eps / 100 (R11)
  double eps_lr = 0;        // low-rank M2L truncation tolerance; 0 -> eps (R23)
  int lf_p_low = 0;         // LF surface points per edge for w/lambda < lf_p_switch; 0 -> 6 + dp(eps)
  int lf_p_high = 0;        // ... for w/lambda >= lf_p_switch; 0 -> 8 + dp(eps)  (R17)
  double lf_p_switch = 0.75;
  int lowrank = 1;          // low-rank M2L (eq_lrdk) on/off
  int single_leaf = 0;      // debug: no far field, root is the only leaf (everything P2P)
  int max_depth = 20;
  int hf_max_rows = 0;      // HF interpolative-selection sample rows per direction representative; 0: 6000 per
                            // decade of eps from 1e-4 (6000 at eps >= 1e-4)
  double hf_spacing = 0.25; // HF candidate spacing in wavelengths
  int verbose = 0;
  // Translation operators (M2M / L2L / M2L matrices) built on the device (plan_dev.cu) after the host plan:
  // build_plan then only records which operators are needed (Trans::need, M2LGroup with rank = -2).
  bool dev_ops = false;
  // P2 (P2P lists, interaction lists, slots, M2L pairs) built elsewhere (lists_dev.cu); empty: the host code
  std::function<std::string(struct HostPlan&)> lists;
  // The paper's "original" FDA (Table 1): no SVD reduction of the expansion basis, dense unreduced M2L
  // (requires dev_ops; low rank off)
  bool original = false;
  // Pivoted column selection on A[i, j] = G(X_i - Y_j) rs_i cs_j (empty rs / cs: 1) with tolerance tol relative
  // to the largest column, at most maxrank pivots (R16).  Empty: the host pivoted QR (linalg.cpp).
  std::function<std::vector<int64_t>(const std::vector<std::array<double, 3>>& X,
                                     const std::vector<std::array<double, 3>>& Y, const std::vector<double>& rs,
                                     const std::vector<double>& cs, double k, double tol, int64_t maxrank)>
      select;
};

struct Cube {
  int level;
  int64_t ijk[3];
  int64_t pbeg, pend;   // point range (Morton order)
  int64_t parent;       // global cube index, -1 for root
  int64_t child[8];     // global cube index or -1
  int64_t local;        // index within its level
  bool leaf;
};

// group element of the cube symmetry group: (g v)_i = sign[i] * v[perm[i]]
struct Sym {
  int perm[3];
  int sign[3];
};

struct DirRep {         // HF directional point sets of one orbit representative
  int dir;              // representative direction id
  Mat b, a;             // equivalent points (nb x 3, stored as real parts) / check points (na x 3)
  std::vector<std::array<double, 3>> bp, ap;
  Mat U, V;             // truncated SVD of R_up = G(a, b): U (na x s), V (nb x s)
  std::vector<double> sig;
  double verr = 0;      // relative error of the expansion on held-out far-field samples (build_plan)
};

struct Level {
  int l = 0;
  double w = 0;          // cube width
  bool hf = false;       // w >= lambda
  int R = 1;             // near radius in cube units (LF: 1; HF: floor(1 + k w / pi))
  int m = 0;             // HF face-grid cells per face edge
  int ndir = 1;          // 6 m^2 (HF) or 1 (LF)
  int s = 0;             // (padded) reduced expansion length
  std::vector<int64_t> cubes;     // global cube ids in Morton order
  // slots: dense tables cube_local * ndir + dir -> slot (or -1)
  std::vector<int64_t> out_slot, in_slot;
  int64_t n_out = 0, n_in = 0;
  std::vector<int64_t> out_cube, in_cube;  // slot -> cube local index
  std::vector<int> out_dir, in_dir;         // slot -> dir
  // LF surfaces (unit cube surface grid scaled by w)
  int p = 0, nsurf = 0;
  std::vector<std::array<double, 3>> eq_pts, ck_pts;  // 1.05 w and 2.95 w surfaces (relative)
  Mat lfU, lfV;
  std::vector<double> lfsig;
  // HF direction data
  std::vector<int> dir_rep;      // dir -> index into reps
  std::vector<Sym> dir_sym;      // dir -> g with P_dir = g P_rep
  std::vector<DirRep> reps;
  bool orig = false;  // original (unreduced) mode: expansions are equivalent densities (Options::original)
  // the expansion length of direction d (HF wedges are truncated separately; s is their maximum)
  int sdir(int d) const {
    if (!hf || reps.empty()) return s;
    return orig ? (int)reps[dir_rep[d]].bp.size() : (int)reps[dir_rep[d]].sig.size();
  }
};

struct HostPlan {
  // inputs (Morton order)
  int64_t n = 0;
  double k = 0;
  std::complex<double> alpha;
  double eps = 1e-4, eps_int = 1e-5, eps_lr = 1e-5;
  int np = 50;
  Options opt;
  std::vector<double> px, py, pz, nx, ny, nz, w;
  std::vector<int32_t> perm;      // Morton position -> caller index
  double root_lo[3], root_w;
  // tree
  std::vector<Cube> cubes;
  std::vector<Level> levels;
  std::vector<int64_t> leaves;    // global cube ids of leaves, Morton order
  std::vector<int64_t> leaf_of_cube;
  // P2P: target leaf -> source leaves
  std::vector<int64_t> p2p_ptr, p2p_src;
  int lmin = -1;                  // coarsest level with a non-empty interaction list
  // M2L (per level): groups by offset
  struct M2LGroup {
    int level;
    int off[3];
    int dir;          // source direction (HF) or 0
    int64_t pbeg, pend;  // into pair arrays
    int rank;         // -1: dense K~, else low-rank rank r; -2: not computed on the host (Options::dev_ops)
    int64_t mat_off;  // offset (complex elements) into the M2L matrix pool of the level
  };
  std::vector<M2LGroup> m2l_groups;
  std::vector<int32_t> m2l_tgt, m2l_src;    // slots (in / out) at the group's level
  std::vector<std::vector<cplx>> m2l_pool;  // per level
  // M2M / L2L per transition (parent level l): matrices per (dir, octant)
  struct Trans {
    int lp;                          // parent level
    int sp, sc;                      // padded sizes
    std::vector<int64_t> mat_index;  // dir * 8 + oct -> matrix id or -1
    std::vector<cplx> pool;          // matrices, each sp x sc column-major (M2M layout)
    std::vector<cplx> poolT;         // the same transposed: sc x sp column-major (L2L layout)
    // M2M: per parent out slot CSR of (child out slot, matrix id)
    std::vector<int64_t> up_ptr, up_child, up_mat;
    // L2L: per child in slot CSR of (parent in slot, matrix id)
    std::vector<int64_t> dn_ptr, dn_parent, dn_mat;
    std::vector<std::pair<int, int>> need;  // matrix id -> (parent direction, child octant)
  };
  std::vector<Trans> trans;
  // S2M / L2T: per LF level, leaves (global leaf index) with their slots
  struct LeafOps {
    int level;
    std::vector<int64_t> leaf, slot;
    std::vector<cplx> S;   // s x nsurf column-major  (Sigma^-1 U^H)
    std::vector<cplx> T;   // nsurf x s column-major  (conj(U) Sigma^-1)
  };
  std::vector<LeafOps> leafops;
  // low-rank M2L truncation of a level (R23): eps_lr, tightened 10x on the low-frequency LF levels
  // (w < lambda / 4), whose far fields of mean-zero densities cancel most (measured: kD = 1 far-field error
  // 2.1e-3 at eps / 3, 5.8e-4 at eps / 30, profiles/r02)
  double eps_lr_level(const Level& L) const {
    const bool lowf = !L.hf && (k <= 0 || L.w * k / (2.0 * 3.14159265358979323846) < 0.25);
    return lowf && opt.eps_lr <= 0 ? eps_lr / 10.0 : eps_lr;
  }
  // stats
  double t_tree = 0, t_lists = 0, t_ops = 0;
  std::string log;
};

// P0 / P1 built on the device (tree_dev.cu): root box, Morton permutation and every cube, level-major
// (the level's cubes in Morton order), as the host builder would number them.
struct TreeIn {
  double root_lo[3] = {0, 0, 0}, root_w = 1;
  std::vector<int32_t> perm;                // Morton position -> caller index
  std::vector<int> level;                   // per cube
  std::vector<int64_t> key;                 // per cube: Morton prefix (3 bits per level)
  std::vector<int64_t> pbeg, pend, parent;  // per cube (parent: global id, -1 for the root)
  std::vector<unsigned char> leaf;
};

// Build the plan.  x/nrm interleaved xyz (n x 3), w (n), all host, caller order.  With tin (the device-built
// tree) the host P0 / P1 are skipped and x / nrm / w are not read (the geometry stays on the device).
// Returns "" on success, else an error message.
std::string build_plan(HostPlan& P, int64_t n, const double* x, const double* nrm, const double* w,
                       double k, std::complex<double> alpha, double eps, const Options& opt,
                       const TreeIn* tin = nullptr);

// equivalent (check = false) or check (check = true) points of direction d of a level, relative to the cube
// centre (HF: the representative's set mapped by the direction's cube symmetry; LF: the surfaces)
std::vector<std::array<double, 3>> dir_points(const Level& L, int d, bool check);

// N_p = max(30, 50 (-log10 eps - 3)) (eq_npleaf, sign-corrected; R12), or np_opt > 0
int leaf_size_for(double eps, int np_opt);

// per-level summary lines of the plan log (sizes, M2L pairs, ranks, flops)
std::string level_summary(const HostPlan& P);

// direction helpers (face grid, R15)
int face_dir(const double v[3], int m);
void dir_center(int d, int m, double out[3]);
int anti_dir(int d, int m);
int child_dir(int d, int m_parent);  // parent-level direction -> child-level (coarser grid) direction

}  // namespace fda
