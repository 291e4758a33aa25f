// linalg.hpp -- small dense complex linear algebra for the plan builder (host).
//
// Column-major storage (element (i, j) of an m x n matrix at i + j*m).
// Used once per plan to build the translation operators:
//   * truncated SVD  R = U S V^H, keep sigma_i >= eps sigma_1   (eq_svdr, eq_invr)
//   * column-pivoted QR (interpolative selection of the directional
//     equivalent / check points, reading R16)
//   * low-rank factors of the reduced M2L matrices (eq_lrdk)
#pragma once
#include <complex>
#include <cstdint>
#include <vector>

namespace fda {

using cplx = std::complex<double>;

struct Mat {
  int64_t m = 0, n = 0;
  std::vector<cplx> a;
  Mat() = default;
  Mat(int64_t m_, int64_t n_) : m(m_), n(n_), a((size_t)(m_ * n_)) {}
  cplx& operator()(int64_t i, int64_t j) { return a[(size_t)(i + j * m)]; }
  const cplx& operator()(int64_t i, int64_t j) const { return a[(size_t)(i + j * m)]; }
  cplx* col(int64_t j) { return a.data() + j * m; }
  const cplx* col(int64_t j) const { return a.data() + j * m; }
};

// C = op(A) * op(B); op = 'N' (none), 'T' (transpose), 'C' (conjugate transpose)
Mat gemm(const Mat& A, char opa, const Mat& B, char opb);

struct SVD {
  Mat U;                  // m x r
  std::vector<double> s;  // r, descending
  Mat V;                  // n x r  (A ~ U diag(s) V^H)
};

// Full thin SVD by one-sided Jacobi, then truncation sigma_i >= eps * sigma_1 (eps <= 0: none).
SVD svd_truncated(const Mat& A, double eps);

// Column-pivoted QR (modified Gram-Schmidt with re-orthogonalisation), stopped when
// the largest remaining column norm drops below tol * (largest initial column norm)
// or after maxrank steps.  Returns the pivot order of the selected columns; if Q / R
// are non-null they receive Q (m x r) and R (r x n) with A(:, piv) ~ Q R(:, 0..r) and
// R in the ORIGINAL column order (A ~ Q R).
std::vector<int64_t> pivoted_qr(const Mat& A, double tol, int64_t maxrank, Mat* Q = nullptr,
                                Mat* R = nullptr);

}  // namespace fda
