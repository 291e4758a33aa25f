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

/*
 * Locally corrected Nystrom weights of one (field point, element) pair -- SURVEY.md §8(f) row 4,
 * PAPER.md:299-323.  The element is a 6-node quadratic triangle (corners 1, 2, 3, mid-edges 12, 23, 31,
 * SPEC.md:82) with intrinsic coordinates (xi1, xi2) on the reference triangle xi1, xi2 >= 0, xi1 + xi2 <= 1:
 *   y(xi) = sum_a N_a(xi) P_a,  t_1 = dy/dxi1,  t_2 = dy/dxi2,  J = |t_1 x t_2|,  n_y = t_1 x t_2 / J.
 * Moments (right-hand side of PAPER.md:313-317, eq:local correction):
 *   I_n = int_Delta K(x, y) phi^(n)(y) dy = int_ref K(x, n_x; y(xi), n_y(xi)) xi1^p xi2^q J(xi) dxi,
 *   phi^(n) = xi1^p xi2^q, p + q <= 2, ordered (p,q) = (0,0),(1,0),(0,1),(2,0),(1,1),(0,2).
 * They are "nearly singular when x is close to the element, and ... computed by using a recursive
 * subdivision quadrature": a sub-triangle A, B, C of the reference triangle is split into its
 * four mid-point children while its largest mapped edge exceeds theta times the distance from x to the
 * nearest of y(A), y(B), y(C), y(centroid) (the paper gives no criterion -- DESIGN.md reading R27); otherwise
 * it is integrated by the nq x nq Gauss-Legendre product rule on the collapsed square,
 *   xi(u, v) = A + u [(B - A) + v (C - B)],  dxi = 2 |T| u du dv,  (u, v) in [0,1]^2.
 * The Gauss-Legendre nodes and weights on [0,1] are inputs (gu, gw; numpy.polynomial.legendre.leggauss in the
 * wrapper).  The field point must not lie on the element (the singular self-element integrals need the method
 * of [rjj_int], which the paper does not give: out of scope).
 * The weights solve the 6 x 6 system  sum_j wbar_j phi^(n)(xi_j) = I_n  (eq:local correction) at the element's
 * six quadrature points xi_j (inputs), by Gaussian elimination with partial pivoting.
 */
static void elem_map(const double *P, double a, double b, double *y, double *nv, double *J) {
    double l1 = 1.0 - a - b, l2 = a, l3 = b;
    double N[6] = {l1 * (2 * l1 - 1), l2 * (2 * l2 - 1), l3 * (2 * l3 - 1), 4 * l1 * l2, 4 * l2 * l3, 4 * l3 * l1};
    double d1[6] = {-(4 * l1 - 1), 4 * l2 - 1, 0, 4 * (l1 - l2), 4 * l3, -4 * l3};
    double d2[6] = {-(4 * l1 - 1), 0, 4 * l3 - 1, -4 * l2, 4 * l2, 4 * (l1 - l3)};
    double t1[3] = {0, 0, 0}, t2[3] = {0, 0, 0};
    for (int c = 0; c < 3; ++c) {
        y[c] = 0;
        for (int q = 0; q < 6; ++q) {
            y[c] += N[q] * P[3 * q + c];
            t1[c] += d1[q] * P[3 * q + c];
            t2[c] += d2[q] * P[3 * q + c];
        }
    }
    if (nv) {
        double cr[3] = {t1[1] * t2[2] - t1[2] * t2[1], t1[2] * t2[0] - t1[0] * t2[2], t1[0] * t2[1] - t1[1] * t2[0]};
        *J = sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
        for (int c = 0; c < 3; ++c) nv[c] = cr[c] / *J;
    }
}

static double dist3(const double *a, const double *b) {
    return sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]) + (a[2] - b[2]) * (a[2] - b[2]));
}

static void moments_rec(int kind, const double *P, const double *x, const double *nx, double k, cplx alpha,
                        int nq, const double *gu, const double *gw, double theta, int depth, int maxdepth,
                        const double *A, const double *B, const double *C, cplx *I6) {
    double yA[3], yB[3], yC[3], yG[3];
    elem_map(P, A[0], A[1], yA, NULL, NULL);
    elem_map(P, B[0], B[1], yB, NULL, NULL);
    elem_map(P, C[0], C[1], yC, NULL, NULL);
    elem_map(P, (A[0] + B[0] + C[0]) / 3.0, (A[1] + B[1] + C[1]) / 3.0, yG, NULL, NULL);
    double h = fmax(dist3(yA, yB), fmax(dist3(yB, yC), dist3(yC, yA)));
    double d = fmin(fmin(dist3(x, yA), dist3(x, yB)), fmin(dist3(x, yC), dist3(x, yG)));
    if (h > theta * d && depth < maxdepth) {
        double AB[2] = {0.5 * (A[0] + B[0]), 0.5 * (A[1] + B[1])};
        double BC[2] = {0.5 * (B[0] + C[0]), 0.5 * (B[1] + C[1])};
        double CA[2] = {0.5 * (C[0] + A[0]), 0.5 * (C[1] + A[1])};
        moments_rec(kind, P, x, nx, k, alpha, nq, gu, gw, theta, depth + 1, maxdepth, A, AB, CA, I6);
        moments_rec(kind, P, x, nx, k, alpha, nq, gu, gw, theta, depth + 1, maxdepth, AB, B, BC, I6);
        moments_rec(kind, P, x, nx, k, alpha, nq, gu, gw, theta, depth + 1, maxdepth, CA, BC, C, I6);
        moments_rec(kind, P, x, nx, k, alpha, nq, gu, gw, theta, depth + 1, maxdepth, AB, BC, CA, I6);
        return;
    }
    double area2 = fabs((B[0] - A[0]) * (C[1] - A[1]) - (B[1] - A[1]) * (C[0] - A[0])); /* 2 |T| */
    for (int a = 0; a < nq; ++a)
        for (int b = 0; b < nq; ++b) {
            double u = gu[a], v = gu[b];
            double s1 = A[0] + u * ((B[0] - A[0]) + v * (C[0] - B[0]));
            double s2 = A[1] + u * ((B[1] - A[1]) + v * (C[1] - B[1]));
            double y[3], ny[3], J;
            elem_map(P, s1, s2, y, ny, &J);
            cplx f = kernel(kind, x, nx, y, ny, k, alpha) * (gw[a] * gw[b] * u * area2 * J);
            I6[0] += f;
            I6[1] += f * s1;
            I6[2] += f * s2;
            I6[3] += f * s1 * s1;
            I6[4] += f * s1 * s2;
            I6[5] += f * s2 * s2;
        }
}

/* moments I_n of npairs (field point, element) pairs: elem (ne x 6 x 3), tx / tn (nt x 3), pair_t / pair_e */
void oracle_moments(int kind, const double *elem, const double *tx, const double *tn, int64_t npairs,
                    const int64_t *pair_t, const int64_t *pair_e, double k, double ar, double ai, int nq,
                    const double *gu, const double *gw, double theta, int maxdepth, double *out) {
    cplx alpha = ar + I * ai;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < npairs; ++p) {
        cplx I6[6] = {0, 0, 0, 0, 0, 0};
        const double A[2] = {0, 0}, B[2] = {1, 0}, C[2] = {0, 1};
        moments_rec(kind, elem + 18 * pair_e[p], tx + 3 * pair_t[p], tn + 3 * pair_t[p], k, alpha, nq, gu, gw, theta,
                    0, maxdepth, A, B, C, I6);
        for (int n = 0; n < 6; ++n) out[12 * p + 2 * n] = creal(I6[n]), out[12 * p + 2 * n + 1] = cimag(I6[n]);
    }
}

/* wbar (npairs x 6 complex) from the moments: sum_j wbar_j xi1_j^p xi2_j^q = I_n; xi (6 x 2) quadrature points */
void oracle_weights_from_moments(const double *xi, int64_t npairs, const double *mom, double *wbar) {
    for (int64_t p = 0; p < npairs; ++p) {
        double M[6][6];
        cplx rhs[6];
        for (int j = 0; j < 6; ++j) {
            double a = xi[2 * j], b = xi[2 * j + 1];
            M[0][j] = 1, M[1][j] = a, M[2][j] = b, M[3][j] = a * a, M[4][j] = a * b, M[5][j] = b * b;
        }
        for (int n = 0; n < 6; ++n) rhs[n] = mom[12 * p + 2 * n] + I * mom[12 * p + 2 * n + 1];
        for (int c = 0; c < 6; ++c) {
            int piv = c;
            for (int r = c + 1; r < 6; ++r)
                if (fabs(M[r][c]) > fabs(M[piv][c])) piv = r;
            for (int q = 0; q < 6; ++q) { double t = M[c][q]; M[c][q] = M[piv][q]; M[piv][q] = t; }
            cplx t = rhs[c]; rhs[c] = rhs[piv]; rhs[piv] = t;
            for (int r = c + 1; r < 6; ++r) {
                double f = M[r][c] / M[c][c];
                for (int q = c; q < 6; ++q) M[r][q] -= f * M[c][q];
                rhs[r] -= f * rhs[c];
            }
        }
        for (int r = 5; r >= 0; --r) {
            cplx s = rhs[r];
            for (int q = r + 1; q < 6; ++q) s -= M[r][q] * (wbar[12 * p + 2 * q] + I * wbar[12 * p + 2 * q + 1]);
            s /= M[r][r];
            wbar[12 * p + 2 * r] = creal(s), wbar[12 * p + 2 * r + 1] = cimag(s);
        }
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
