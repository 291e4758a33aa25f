/*
 * csynth.c -- seeded synthetic-input helpers (geometry bookkeeping only).
 *
 * This file is part of the INPUT GENERATOR, shared by the oracle tests and the
 * CUDA path.  It contains none of the method's arithmetic (no Green's function,
 * no kernel, no translation): only
 *   (1) the local-region pattern D_i of PAPER.md:285 ("D_i consists of all the
 *       elements whose distance to x_i is not larger than 2 times of their
 *       largest side length"), with dist(x_i, Delta) read as the minimum over
 *       Delta's 6 nodes and 6 quadrature points (R5),
 *   (2) seeded synthetic values for the correction CSR (DESIGN.md "input
 *       recipe"), drawn from a counter-based generator (splitmix64) so that
 *       any (seed, i, j) entry can be regenerated independently.
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC csynth.c -o libcsynth.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* uniform double in [-1, 1) from a 64-bit counter */
static inline double u11(uint64_t h) {
    return ((double)(h >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

/* Exported for tests: the counter-based generator. */
double csynth_u11(uint64_t seed, uint64_t i, uint64_t j, uint64_t lane) {
    uint64_t h = splitmix64(seed ^ splitmix64(i * 0x100000001B3ull + splitmix64(j + (lane << 56))));
    return u11(h);
}

typedef struct { int64_t *data; int64_t n, cap; } vec64;

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/*
 * Count / fill the D_i element lists.
 *  ne        number of elements
 *  samples   ne x 12 x 3 doubles: the 6 nodes then the 6 quadrature points of each element
 *  hmax      ne doubles: largest side length of each element
 *  n         number of collocation points (= 6 ne); x: n x 3
 *  elem_ptr  out, n+1 (int64): prefix sums of |D_i|
 *  elem_idx  out (may be NULL on the counting pass): element ids, ascending per row
 * Returns total number of (i, element) incidences, or -1 on allocation failure.
 */
int64_t csynth_local_regions(int64_t ne, const double *samples, const double *hmax,
                             int64_t n, const double *x, int64_t *elem_ptr, int32_t *elem_idx) {
    /* uniform grid over element centroids; cell = max over elements of (2 h + element radius) */
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    double *cen = (double *)malloc(sizeof(double) * 3 * ne);
    double *rad = (double *)malloc(sizeof(double) * ne);
    if (!cen || !rad) return -1;
    double reach = 0.0;
    for (int64_t e = 0; e < ne; ++e) {
        double c[3] = {0, 0, 0};
        for (int s = 0; s < 12; ++s)
            for (int d = 0; d < 3; ++d) c[d] += samples[(e * 12 + s) * 3 + d] / 12.0;
        double r = 0;
        for (int s = 0; s < 12; ++s) {
            double dd = 0;
            for (int d = 0; d < 3; ++d) {
                double t = samples[(e * 12 + s) * 3 + d] - c[d];
                dd += t * t;
            }
            if (dd > r) r = dd;
        }
        r = sqrt(r);
        for (int d = 0; d < 3; ++d) {
            cen[e * 3 + d] = c[d];
            if (c[d] < lo[d]) lo[d] = c[d];
            if (c[d] > hi[d]) hi[d] = c[d];
        }
        rad[e] = r;
        double rr = 2.0 * hmax[e] + r;
        if (rr > reach) reach = rr;
    }
    double cell = reach * 1.0000001;
    int64_t g[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] -= cell;
        g[d] = (int64_t)((hi[d] + cell - lo[d]) / cell) + 1;
    }
    int64_t ncell = g[0] * g[1] * g[2];
    int64_t *cstart = (int64_t *)calloc(ncell + 1, sizeof(int64_t));
    int64_t *corder = (int64_t *)malloc(sizeof(int64_t) * ne);
    int64_t *ecell = (int64_t *)malloc(sizeof(int64_t) * ne);
    if (!cstart || !corder || !ecell) return -1;
    for (int64_t e = 0; e < ne; ++e) {
        int64_t ci[3];
        for (int d = 0; d < 3; ++d) ci[d] = (int64_t)((cen[e * 3 + d] - lo[d]) / cell);
        ecell[e] = (ci[0] * g[1] + ci[1]) * g[2] + ci[2];
        cstart[ecell[e] + 1]++;
    }
    for (int64_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * ncell);
        memcpy(fill, cstart, sizeof(int64_t) * ncell);
        for (int64_t e = 0; e < ne; ++e) corder[fill[ecell[e]]++] = e; /* ascending e within a cell */
        free(fill);
    }
    int64_t total = 0;
    int fail = 0;
#pragma omp parallel reduction(+ : total)
    {
        int64_t cap = 1024, *buf = (int64_t *)malloc(sizeof(int64_t) * cap);
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; ++i) {
            const double *xi = x + i * 3;
            int64_t ci[3];
            for (int d = 0; d < 3; ++d) ci[d] = (int64_t)((xi[d] - lo[d]) / cell);
            int64_t cnt = 0;
            for (int64_t a = ci[0] - 1; a <= ci[0] + 1; ++a)
                for (int64_t b = ci[1] - 1; b <= ci[1] + 1; ++b)
                    for (int64_t c = ci[2] - 1; c <= ci[2] + 1; ++c) {
                        if (a < 0 || b < 0 || c < 0 || a >= g[0] || b >= g[1] || c >= g[2]) continue;
                        int64_t cc = (a * g[1] + b) * g[2] + c;
                        for (int64_t t = cstart[cc]; t < cstart[cc + 1]; ++t) {
                            int64_t e = corder[t];
                            double lim = 2.0 * hmax[e];
                            double best = 1e300;
                            for (int s = 0; s < 12; ++s) {
                                const double *p = samples + (e * 12 + s) * 3;
                                double dx = p[0] - xi[0], dy = p[1] - xi[1], dz = p[2] - xi[2];
                                double dd = dx * dx + dy * dy + dz * dz;
                                if (dd < best) best = dd;
                            }
                            if (best <= lim * lim) {
                                if (cnt == cap) {
                                    cap *= 2;
                                    buf = (int64_t *)realloc(buf, sizeof(int64_t) * cap);
                                }
                                buf[cnt++] = e;
                            }
                        }
                    }
            if (elem_idx) {
                qsort(buf, cnt, sizeof(int64_t), cmp_i64);
                int64_t o = elem_ptr[i];
                if (elem_ptr[i + 1] - o != cnt) fail = 1;
                for (int64_t t = 0; t < cnt; ++t) elem_idx[o + t] = (int32_t)buf[t];
            } else {
                elem_ptr[i + 1] = cnt;
            }
            total += cnt;
        }
        free(buf);
    }
    if (!elem_idx) {
        elem_ptr[0] = 0;
        for (int64_t i = 0; i < n; ++i) elem_ptr[i + 1] += elem_ptr[i];
    }
    free(cen); free(rad); free(cstart); free(corder); free(ecell);
    return fail ? -2 : total;
}

/*
 * Expand the element lists into the point-level CSR pattern (each element
 * contributes its 6 collocation points 6e..6e+5; columns ascending) and fill
 * synthetic values (correction CSR):
 *   val_ij = scale_i * w_j * xi_ij            (j != i)
 *   val_ii = 0.5 + scale_i * w_i * xi_ii
 *   scale_i = 0.1 / (4 pi kref h_i^3),  h_i = hmax of the element owning i,
 *   xi_ij   = u11(seed,i,j,0) + i u11(seed,i,j,1).
 * row_ptr (n+1) is 6 * elem_ptr.  val is interleaved complex (2 * nnz doubles).
 */
void csynth_fill_csr(int64_t n, const int64_t *elem_ptr, const int32_t *elem_idx,
                     const double *w, const double *hmax, double kref, uint64_t seed,
                     int64_t *row_ptr, int32_t *col, double *val) {
    for (int64_t i = 0; i <= n; ++i) row_ptr[i] = 6 * elem_ptr[i];
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
        double h = hmax[i / 6];
        double scale = 0.1 / (4.0 * 3.14159265358979323846 * kref * h * h * h);
        int64_t o = row_ptr[i];
        for (int64_t t = elem_ptr[i]; t < elem_ptr[i + 1]; ++t) {
            int64_t e = elem_idx[t];
            for (int q = 0; q < 6; ++q, ++o) {
                int64_t j = 6 * e + q;
                col[o] = (int32_t)j;
                double re = csynth_u11(seed, (uint64_t)i, (uint64_t)j, 0);
                double im = csynth_u11(seed, (uint64_t)i, (uint64_t)j, 1);
                val[2 * o] = scale * w[j] * re + (j == i ? 0.5 : 0.0);
                val[2 * o + 1] = scale * w[j] * im;
            }
        }
    }
}
