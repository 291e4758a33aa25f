/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously correct CPU reference for the FDA Burton-Miller apply.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code with the CUDA path
 * (paper_1311_5202_b200/csrc) and neither includes the other.
 *
 * What it computes (the plain definition the FDA approximates):
 *
 *   out_i = sum_{j != i} w_j K(x_i, n_i; y_j, n_j) phi_j  +  sum_{p in row i} val_p phi_{col_p}
 *
 *   K = dG/dn_y + alpha d2G/(dn_x dn_y)                         PAPER.md:352-355 (eq_hmat)
 *   G = e^{ikr} / (4 pi r)                                      PAPER.md:210-212 (eq:fundsol)
 *   far quadrature: integral ~ sum_j w_j K(x_i, y_j) u_j        PAPER.md:291-297 (eq:far field)
 *   corrected summation kernel K-bar (weights inside D_i)       PAPER.md:334-341 (kcorrection),
 *       realised as the plain sum plus a caller-owned delta CSR (reading R3/R4)
 *   self term j = i excluded from the plain sum (singular)      PAPER.md:325-326 (R3)
 *
 * The kernel derivatives are written the way they are defined: with g(r) =
 * e^{ikr}/(4 pi r) and r = |x - y|, rhat = (x - y)/r,
 *   grad_x G = g'(r) rhat,  grad_y G = -g'(r) rhat,
 *   dG/dn_y  = -g'(r) (rhat . n_y)
 *   dG/dn_x  =  g'(r) (rhat . n_x)
 *   d2G/dn_x dn_y = n_x . grad_x ( -g'(r) rhat . n_y )
 *                 = -[ g''(r) (rhat.n_x)(rhat.n_y) + g'(r)/r ( n_x.n_y - (rhat.n_x)(rhat.n_y) ) ]
 *   g'(r)  = e^{ikr} (ikr - 1) / (4 pi r^2)
 *   g''(r) = e^{ikr} (2 - 2ikr - k^2 r^2) / (4 pi r^3)
 * (PAPER.md:216-231 eq:operator defines the operators; the paper prints no
 * derivative formulas -- DESIGN.md reading R1; the SPEC.md:142 sign of the
 * hypersingular kernel is wrong.)  Pinned by tests/test_oracle_pins.py.
 *
 * IEEE FP64 throughout, libm exp/sin/cos/sqrt, serial ascending-j inner loop,
 * OpenMP over target rows only.  Build: gcc -O3 -march=native -fopenmp (no fast-math).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define PI 3.14159265358979323846

typedef double complex cplx;

/* kind: 0 = G, 1 = dG/dn_y (double layer), 2 = dG/dn_x (adjoint),
 *       3 = d2G/dn_x dn_y (hypersingular), 4 = BM_H = 1 + alpha*3, 5 = BM_G = 0 + alpha*2,
 *       6 = Table-1 summation kernel G + alpha dG/dn_y (eq_sum) = 0 + alpha*1 */
static cplx kernel(int kind, const double *x, const double *nx, const double *y, const double *ny,
                   double k, cplx alpha) {
    double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
    double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    double rh[3] = {d[0] / r, d[1] / r, d[2] / r};
    cplx e = cexp(I * k * r);
    cplx g = e / (4.0 * PI * r);
    cplx g1 = e * (I * k * r - 1.0) / (4.0 * PI * r * r);
    cplx g2 = e * (2.0 - 2.0 * I * k * r - k * k * r * r) / (4.0 * PI * r * r * r);
    double a = 0, b = 0, c = 0;
    if (nx) a = rh[0] * nx[0] + rh[1] * nx[1] + rh[2] * nx[2];
    if (ny) b = rh[0] * ny[0] + rh[1] * ny[1] + rh[2] * ny[2];
    if (nx && ny) c = nx[0] * ny[0] + nx[1] * ny[1] + nx[2] * ny[2];
    cplx dny = -g1 * b;
    cplx dnx = g1 * a;
    cplx hyp = -(g2 * a * b + (g1 / r) * (c - a * b));
    switch (kind) {
    case 0: return g;
    case 1: return dny;
    case 2: return dnx;
    case 3: return hyp;
    case 4: return dny + alpha * hyp;
    case 5: return g + alpha * dnx;
    case 6: return g + alpha * dny;
    }
    return 0;
}

/* single kernel value (for pins) */
void oracle_kernel(int kind, const double *x, const double *nx, const double *y, const double *ny,
                   double k, double ar, double ai, double *out) {
    cplx v = kernel(kind, x, nx, y, ny, k, ar + I * ai);
    out[0] = creal(v);
    out[1] = cimag(v);
}

/*
 * Rows of the discrete BM_H operator (or any kernel kind) at on-surface targets.
 *   n points pts (n x 3), normals nrm (n x 3), weights w (n); density phi (2n interleaved)
 *   nrows target row ids rows[]; out (2 nrows)
 *   row_ptr/col/val: optional correction CSR (NULL to skip); val interleaved complex.
 * out_r = sum_{j != rows[r]} w_j K(x_i, n_i; x_j, n_j) phi_j + (C phi)_i
 */
void oracle_rows(int kind, int64_t n, const double *pts, const double *nrm, const double *w,
                 double k, double ar, double ai, const double *phi, int64_t nrows, const int64_t *rows,
                 const int64_t *row_ptr, const int32_t *col, const double *val, double *out) {
    cplx alpha = ar + I * ai;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        cplx acc = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            cplx kij = kernel(kind, pts + 3 * i, nrm + 3 * i, pts + 3 * j, nrm + 3 * j, k, alpha);
            acc += w[j] * kij * (phi[2 * j] + I * phi[2 * j + 1]);
        }
        if (row_ptr) {
            for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
                int64_t j = col[p];
                acc += (val[2 * p] + I * val[2 * p + 1]) * (phi[2 * j] + I * phi[2 * j + 1]);
            }
        }
        out[2 * r] = creal(acc);
        out[2 * r + 1] = cimag(acc);
    }
}

/*
 * Near-field-only reference (kernel kind as in oracle_rows): the same sum restricted to the pairs (i, j) with
 * i in target leaf t, j in source leaf s, for the leaf pairs (t, s) listed,
 * j != i.  Leaves are given as point-index lists: leaf_ptr (nleaf+1), leaf_pts.
 * Pairs are grouped by target leaf: pair_ptr (nleaf+1), pair_src.
 * out (2n) is overwritten for every point (zero where no pair contributes).
 */
void oracle_near(int kind, int64_t n, const double *pts, const double *nrm, const double *w,
                 double k, double ar, double ai, const double *phi,
                 int64_t nleaf, const int64_t *leaf_ptr, const int64_t *leaf_pts,
                 const int64_t *pair_ptr, const int64_t *pair_src, double *out) {
    cplx alpha = ar + I * ai;
    for (int64_t i = 0; i < 2 * n; ++i) out[i] = 0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < nleaf; ++t) {
        for (int64_t a = leaf_ptr[t]; a < leaf_ptr[t + 1]; ++a) {
            int64_t i = leaf_pts[a];
            cplx acc = 0;
            for (int64_t p = pair_ptr[t]; p < pair_ptr[t + 1]; ++p) {
                int64_t s = pair_src[p];
                for (int64_t b = leaf_ptr[s]; b < leaf_ptr[s + 1]; ++b) {
                    int64_t j = leaf_pts[b];
                    if (j == i) continue;
                    cplx kij = kernel(kind, pts + 3 * i, nrm + 3 * i, pts + 3 * j, nrm + 3 * j, k, alpha);
                    acc += w[j] * kij * (phi[2 * j] + I * phi[2 * j + 1]);
                }
            }
            out[2 * i] = creal(acc);
            out[2 * i + 1] = cimag(acc);
        }
    }
}

/*
 * Off-surface targets (for the pins): out_t = sum_j w_j K(kind; t, tn_t; y_j, n_j) dens_j.
 * tn may be NULL for kinds without a target normal.
 */
void oracle_targets(int kind, int64_t m, const double *tx, const double *tn, int64_t n,
                    const double *pts, const double *nrm, const double *w, double k, double ar,
                    double ai, const double *dens, double *out) {
    cplx alpha = ar + I * ai;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t t = 0; t < m; ++t) {
        cplx acc = 0;
        for (int64_t j = 0; j < n; ++j) {
            cplx kij = kernel(kind, tx + 3 * t, tn ? tn + 3 * t : NULL, pts + 3 * j, nrm + 3 * j, k, alpha);
            acc += w[j] * kij * (dens[2 * j] + I * dens[2 * j + 1]);
        }
        out[2 * t] = creal(acc);
        out[2 * t + 1] = cimag(acc);
    }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
