// plan_dev.cuh -- device builders of the plan's translation operators (row a-P3 of SURVEY.md §8(a)).
//
//   M2L  K~ = V_t^T G(delta w + b_t, b_s) V_s                (eq_cmpk)
//        low rank K~ ~ U^ V^ when r < s/2, r = #{sigma_i >= eps_lr sigma_1}   (eq_lrdk)
//   M2M  M~ = Sigma^-1 U_P^H G(a_P, b_C + o) V_C              (eq_cmpm, R18)
//   L2L  L~ = M~^T
//   HF directional sets: pivoted-QR (interpolative) column selection (R16)
//
// Every operator is "out = Lf_A G(P_A - Q_B + shift) Rf_B" for a pair of point sets with factors, so one
// batched kernel builds them all (one CTA per operator, the chain in a per-CTA global workspace that stays
// in L2); the M2L ones are then compressed in the same CTA (pivoted MGS + one-sided Jacobi SVD of R) and
// every operator is written straight into the DMMA fragment order the apply reads (kernels.cuh GTrans), so
// no operator ever goes through host memory.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fda {

// One point set with its factors (a direction of an HF level, or the LF surface of an LF level).
struct DevSet {
  int n = 0;                    // points
  int s = 0;                    // expansion length of this set (<= the level's padded s)
  const double* pts = nullptr;  // n x 3 (relative to the cube centre)
  const double2* Lf = nullptr;  // left factor  s x n, column-major (V^T for M2L targets, Sigma^-1 U^H for M2M parents)
  const double2* Rf = nullptr;  // right factor n x s, column-major (V)
};

struct OpJob {
  int n_items = 0;
  const int32_t* a = nullptr;    // item -> left set
  const int32_t* b = nullptr;    // item -> right set
  const double* shift = nullptr; // item -> 3 doubles added to P_A - Q_B
  const DevSet* sets = nullptr;
  double k = 0;
  // output layout (kernels.cuh GTrans fragment order)
  int s_out = 0, s_in = 0;       // padded sizes of the level(s)
  // M2L compression
  int compress = 0;              // 1: pivoted MGS + SVD, low rank iff 2 r < max(s_A, s_B)
  double eps_lr = 0;
  int rank_round = 8;            // the rank is rounded up to a multiple of this (R23)
  int32_t* rank = nullptr;       // pass 1 output: r, or -1 for dense
  const int32_t* rank_in = nullptr;  // pass 2 input (from pass 1)
  const int64_t* off = nullptr;  // pass 2: item -> offset (doubles) into pool
  double* pool = nullptr;        // pass 2 output
  double* poolT = nullptr;       // M2M only: the transposed operator (L2L) at the same offsets
  // workspace
  int maxn = 0, maxs = 0;        // largest set size / expansion length of the job
};

// pass 1 (compress): ranks only; pass 2: write the operators.  M2M jobs (compress = 0) only run pass 2.
cudaError_t launch_opjob(const OpJob& J, int pass, cudaStream_t st);

// Pivoted (modified Gram-Schmidt, re-orthogonalised) column selection of a device m x n complex matrix A
// (column-major, overwritten): the columns in pivot order until the largest remaining column norm drops
// below tol x the largest initial one, at most maxrank (R16).  Returns the pivots.
cudaError_t pivoted_columns(double2* A, int64_t m, int64_t n, double tol, int64_t maxrank, int64_t* piv, int64_t* npiv,
                            cudaStream_t st);
// A[i, j] = G(X_i - Y_j) rs_i cs_j (column-major, m x n; null rs / cs: 1), G = e^{ikr}/(4 pi r)
void launch_gmat(double2* A, const double* X, int64_t m, const double* Y, int64_t n, const double* rs, const double* cs,
                 double k, cudaStream_t st);

}  // namespace fda
