// linalg.cpp -- see linalg.hpp.
#include "linalg.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace fda {

static Mat materialize(const Mat& A, char op) {
  if (op == 'N') return A;
  Mat T(A.n, A.m);
  for (int64_t j = 0; j < A.n; ++j)
    for (int64_t i = 0; i < A.m; ++i) T(j, i) = (op == 'C') ? std::conj(A(i, j)) : A(i, j);
  return T;
}

Mat gemm(const Mat& A0, char opa, const Mat& B0, char opb) {
  const Mat A = materialize(A0, opa);
  const Mat B = materialize(B0, opb);
  Mat C(A.m, B.n);
  const int64_t m = A.m, k = A.n, n = B.n;
  for (int64_t j = 0; j < n; ++j) {
    cplx* c = C.col(j);
    for (int64_t l = 0; l < k; ++l) {
      const cplx b = B(l, j);
      const double br = b.real(), bi = b.imag();
      if (br == 0.0 && bi == 0.0) continue;
      const cplx* a = A.col(l);
      for (int64_t i = 0; i < m; ++i) {
        const double ar = a[i].real(), ai = a[i].imag();
        c[i] = cplx(c[i].real() + ar * br - ai * bi, c[i].imag() + ar * bi + ai * br);
      }
    }
  }
  return C;
}

static inline cplx dotc(const cplx* x, const cplx* y, int64_t m) {  // x^H y
  double re = 0, im = 0;
  for (int64_t i = 0; i < m; ++i) {
    const double xr = x[i].real(), xi = x[i].imag(), yr = y[i].real(), yi = y[i].imag();
    re += xr * yr + xi * yi;
    im += xr * yi - xi * yr;
  }
  return cplx(re, im);
}

static inline double nrm2sq(const cplx* x, int64_t m) {
  double s = 0;
  for (int64_t i = 0; i < m; ++i) s += std::norm(x[i]);
  return s;
}

// One-sided (Hestenes) Jacobi on a tall matrix W (m >= n): W V = U S.
static void jacobi_tall(Mat& W, Mat& V) {
  const int64_t m = W.m, n = W.n;
  V = Mat(n, n);
  for (int64_t i = 0; i < n; ++i) V(i, i) = 1.0;
  std::vector<double> nrm(n);
  for (int64_t j = 0; j < n; ++j) nrm[j] = nrm2sq(W.col(j), m);
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int64_t p = 0; p < n - 1; ++p) {
      for (int64_t q = p + 1; q < n; ++q) {
        const double alpha = nrm[p], beta = nrm[q];
        if (alpha == 0.0 || beta == 0.0) continue;
        const cplx g = dotc(W.col(p), W.col(q), m);
        const double ga = std::abs(g);
        if (ga <= tol * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const cplx ph = g / ga;  // e^{i phi}
        const double zeta = (beta - alpha) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        // a_q' = a_q e^{-i phi}; [a_p, a_q'] <- [c a_p - s a_q', s a_p + c a_q']
        const cplx phc = std::conj(ph);
        cplx* wp = W.col(p);
        cplx* wq = W.col(q);
        for (int64_t i = 0; i < m; ++i) {
          const cplx ap = wp[i], aq = wq[i] * phc;
          wp[i] = c * ap - s * aq;
          wq[i] = s * ap + c * aq;
        }
        cplx* vp = V.col(p);
        cplx* vq = V.col(q);
        for (int64_t i = 0; i < n; ++i) {
          const cplx ap = vp[i], aq = vq[i] * phc;
          vp[i] = c * ap - s * aq;
          vq[i] = s * ap + c * aq;
        }
        nrm[p] = nrm2sq(wp, m);
        nrm[q] = nrm2sq(wq, m);
      }
    }
    if (!rotated) break;
  }
}

SVD svd_truncated(const Mat& A, double eps) {
  const bool wide = A.m < A.n;
  Mat W = wide ? materialize(A, 'C') : A;  // tall
  Mat V;
  jacobi_tall(W, V);
  const int64_t n = W.n, m = W.m;
  std::vector<double> s(n);
  for (int64_t j = 0; j < n; ++j) s[j] = std::sqrt(nrm2sq(W.col(j), m));
  std::vector<int64_t> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return s[a] > s[b]; });
  int64_t r = 0;
  const double s1 = n ? s[ord[0]] : 0.0;
  for (int64_t t = 0; t < n; ++t) {
    const double v = s[ord[t]];
    if (v <= 0.0) break;
    if (eps > 0 && v < eps * s1) break;
    ++r;
  }
  SVD out;
  Mat Ut(m, r), Vt(n, r);
  out.s.resize(r);
  for (int64_t t = 0; t < r; ++t) {
    const int64_t j = ord[t];
    out.s[t] = s[j];
    for (int64_t i = 0; i < m; ++i) Ut(i, t) = W(i, j) / s[j];
    for (int64_t i = 0; i < n; ++i) Vt(i, t) = V(i, j);
  }
  // W = A (tall case): A V = U S  ->  A = U S V^H.
  // wide case: W = A^H, A^H V = U S -> A = V S U^H: swap roles.
  if (!wide) {
    out.U = std::move(Ut);
    out.V = std::move(Vt);
  } else {
    out.U = std::move(Vt);
    out.V = std::move(Ut);
  }
  return out;
}

std::vector<int64_t> pivoted_qr(const Mat& A0, double tol, int64_t maxrank, Mat* Qout, Mat* Rout) {
  Mat A = A0;
  const int64_t m = A.m, n = A.n;
  std::vector<double> nrm(n);
  double n0 = 0;
  for (int64_t j = 0; j < n; ++j) {
    nrm[j] = nrm2sq(A.col(j), m);
    n0 = std::max(n0, nrm[j]);
  }
  n0 = std::sqrt(n0);
  std::vector<int64_t> piv;
  std::vector<char> used(n, 0);
  const int64_t rmax = std::min<int64_t>({maxrank, m, n});
  std::vector<std::vector<cplx>> Qc;
  std::vector<std::vector<cplx>> Rr;  // rows of R (length n)
  for (int64_t step = 0; step < rmax; ++step) {
    int64_t jb = -1;
    double best = -1;
    for (int64_t j = 0; j < n; ++j)
      if (!used[j] && nrm[j] > best) best = nrm[j], jb = j;
    if (jb < 0 || std::sqrt(std::max(best, 0.0)) <= tol * n0 || best <= 0.0) break;
    used[jb] = 1;
    piv.push_back(jb);
    std::vector<cplx> q(A.col(jb), A.col(jb) + m);
    const double qn = std::sqrt(nrm2sq(q.data(), m));
    for (auto& v : q) v /= qn;
    std::vector<cplx> rrow(n, cplx(0));
    // project the remaining columns (twice: re-orthogonalisation)
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
      if (used[j] && j != jb) continue;
      cplx* a = A.col(j);
      cplx tot = 0;
      for (int pass = 0; pass < 2; ++pass) {
        const cplx c = dotc(q.data(), a, m);
        tot += c;
        for (int64_t i = 0; i < m; ++i) a[i] -= c * q[i];
      }
      rrow[j] = tot;
      nrm[j] = nrm2sq(a, m);
    }
    nrm[jb] = 0;
    Qc.push_back(std::move(q));
    Rr.push_back(std::move(rrow));
  }
  const int64_t r = (int64_t)piv.size();
  if (Qout) {
    *Qout = Mat(m, r);
    for (int64_t t = 0; t < r; ++t)
      for (int64_t i = 0; i < m; ++i) (*Qout)(i, t) = Qc[t][i];
  }
  if (Rout) {
    // R(t, j) = q_t^H a_j accumulated over the steps where column j was still active;
    // columns selected at step t' have R(t, j) = 0 for t > t'.
    *Rout = Mat(r, n);
    for (int64_t t = 0; t < r; ++t)
      for (int64_t j = 0; j < n; ++j) (*Rout)(t, j) = Rr[t][j];
    for (int64_t t = 0; t < r; ++t)
      for (int64_t t2 = t + 1; t2 < r; ++t2) (*Rout)(t2, piv[t]) = 0.0;
  }
  return piv;
}

}  // namespace fda
