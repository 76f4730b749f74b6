/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, called by,
 * or shipped with the product path (paper_1302_7193_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Plain-C restatement of the reference (arXiv 1302.7193, "anisocg") hot path,
 * written from the reference's specification and pinned bit-for-bit against
 * the reference itself compiled from /root/reference (oracle/_ref, see
 * tests/test_oracle.py) and against the reference unit tests' frozen values.
 * Compiled with -ffp-contract=off like the reference (proj/CMakeLists.txt:15-18)
 * so every expression below is the plain IEEE sequence.
 *
 * Citations are /root/reference/proj/... file:line.
 *
 * Conventions shared with the reference:
 *   layout 0 = VerticalContiguous   l = n_z*(m*i + j) + k   (field.hpp:23-28)
 *   layout 1 = HorizontalContiguous l = m*(n_z*j + k) + i
 *   per-column partials are indexed col = i*m + j and combined with the
 *   fixed pairwise tree (parallel.hpp:11-20).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ setup */

/* grid.cpp:10-24 — r_k = 1 + (k/n_z)^2 * H */
int orc_vertical_grid(int n_z, double h, double *r) {
    if (n_z < 1 || !(h > 0.0)) return 1;
    for (int k = 0; k <= n_z; ++k) {
        double t = (double)k / n_z;
        r[k] = 1.0 + t * t * h;
    }
    return 0;
}

typedef struct { double x, y, z; } v3;

static v3 v3_cross(v3 a, v3 b) {
    v3 c = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return c;
}
static double v3_dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
/* grid.cpp:48-51 gnomonic projection of (X, Y) onto the unit sphere */
static v3 gno(double X, double Y) {
    double s = sqrt(1.0 + X * X + Y * Y);
    v3 v = {X / s, Y / s, 1.0 / s};
    return v;
}
/* grid.cpp:54 great-circle angle */
static double arc(v3 a, v3 b) {
    v3 c = v3_cross(a, b);
    return atan2(sqrt(v3_dot(c, c)), v3_dot(a, b));
}
/* grid.cpp:58-62 solid angle of a geodesic triangle */
static double tri_omega(v3 a, v3 b, v3 c) {
    double num = v3_dot(a, v3_cross(b, c));
    double den = 1.0 + v3_dot(a, b) + v3_dot(b, c) + v3_dot(c, a);
    return 2.0 * atan2(num, den);
}

/* grid.cpp:72-79 alpha_diag: fixed order west, east, south, north */
static void diag_sum(int m, const double *east, const double *north, double *diag) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            double s = 0.0;
            if (i > 0) s += east[(size_t)(i - 1) * m + j];
            if (i < m - 1) s += east[(size_t)i * m + j];
            if (j > 0) s += north[(size_t)i * (m - 1) + j - 1];
            if (j < m - 1) s += north[(size_t)i * (m - 1) + j];
            diag[(size_t)i * m + j] = s;
        }
}

/* grid.cpp:88-125 */
int orc_cubed_sphere_panel(int m, double *area, double *east, double *north, double *diag) {
    if (m < 1) return 1;
    double *X = malloc(sizeof(double) * (m + 1)), *C = malloc(sizeof(double) * m);
    for (int i = 0; i <= m; ++i) X[i] = -1.0 + 2.0 * (double)i / m;
    for (int i = 0; i < m; ++i) C[i] = 0.5 * (X[i] + X[i + 1]);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            v3 a = gno(X[i], X[j]), b = gno(X[i + 1], X[j]);
            v3 c = gno(X[i + 1], X[j + 1]), d = gno(X[i], X[j + 1]);
            area[(size_t)i * m + j] = tri_omega(a, b, c) + tri_omega(a, c, d);
        }
    for (int i = 0; i + 1 < m; ++i)
        for (int j = 0; j < m; ++j)
            east[(size_t)i * m + j] = arc(gno(X[i + 1], X[j]), gno(X[i + 1], X[j + 1])) /
                                      arc(gno(C[i], C[j]), gno(C[i + 1], C[j]));
    for (int i = 0; i < m; ++i)
        for (int j = 0; j + 1 < m; ++j)
            north[(size_t)i * (m - 1) + j] = arc(gno(X[i], X[j + 1]), gno(X[i + 1], X[j + 1])) /
                                             arc(gno(C[i], C[j]), gno(C[i], C[j + 1]));
    diag_sum(m, east, north, diag);
    free(X);
    free(C);
    return 0;
}

/* grid.cpp:127-139 */
int orc_planar_panel(int m, double extent, double *area, double *east, double *north,
                     double *diag) {
    if (m < 1 || !(extent > 0.0)) return 1;
    double h = extent / m;
    for (size_t l = 0; l < (size_t)m * m; ++l) area[l] = h * h;
    for (size_t l = 0; l < (size_t)(m - 1) * m; ++l) east[l] = 1.0, north[l] = 1.0;
    diag_sum(m, east, north, diag);
    return 0;
}

/* profile.cpp:7-48 */
int orc_vertical_profile(int n_z, const double *r, double omega2, double lambda2, double *ap,
                         double *bp, double *cp, double *d) {
    if (!(omega2 > 0.0) || lambda2 < 0.0) return 1;
    double *a = malloc(sizeof(double) * n_z), *b = malloc(sizeof(double) * n_z);
    double *c = malloc(sizeof(double) * n_z);
    for (int k = 0; k < n_z; ++k) {
        double v = (r[k + 1] * r[k + 1] * r[k + 1] - r[k] * r[k] * r[k]) / 3.0;
        a[k] = v;
        d[k] = -omega2 * v;
    }
    for (int k = 0; k + 1 < n_z; ++k) {
        double delta = 0.5 * (r[k + 2] + r[k + 1]) - 0.5 * (r[k + 1] + r[k]);
        b[k] = -omega2 * lambda2 * r[k + 1] * r[k + 1] / delta;
    }
    b[n_z - 1] = 0.0;
    c[0] = 0.0;
    for (int k = 1; k < n_z; ++k) c[k] = b[k - 1];
    for (int k = 0; k < n_z; ++k) {
        ap[k] = a[k] / d[k];
        bp[k] = b[k] / d[k];
        cp[k] = c[k] / d[k];
    }
    bp[n_z - 1] = 0.0;
    cp[0] = 0.0;
    free(a);
    free(b);
    free(c);
    return 0;
}

/* grid.cpp:141-156 gamma^2 in column order (i*m+j)*n_z+k */
void orc_anisotropy(int m, const double *area, int n_z, const double *r, double lambda2,
                    double *out) {
    for (size_t col = 0; col < (size_t)m * m; ++col)
        for (int k = 0; k < n_z; ++k) {
            double dz = r[k + 1] - r[k];
            out[col * n_z + k] = lambda2 * area[col] / (dz * dz);
        }
}

/* ---------------------------------------------------------------- context */

/* Precision-converted operator data, operator.hpp:32-44: every double is
 * converted to T once; the kernels then work purely in T. */
typedef struct {
    int m, n_z;
    double *ap, *bp, *cp, *d, *area, *east, *north, *diag; /* double copies */
    float *fap, *fbp, *fcp, *fd, *farea, *feast, *fnorth, *fdiag;
} orc_ctx;

static double *dup_d(const double *s, size_t n) {
    double *p = malloc(sizeof(double) * (n ? n : 1));
    if (n) memcpy(p, s, sizeof(double) * n);
    return p;
}
static float *dup_f(const double *s, size_t n) {
    float *p = malloc(sizeof(float) * (n ? n : 1));
    for (size_t l = 0; l < n; ++l) p[l] = (float)s[l];
    return p;
}

orc_ctx *orc_ctx_create(int m, int n_z, const double *ap, const double *bp, const double *cp,
                        const double *d, const double *area, const double *east,
                        const double *north, const double *diag) {
    if (m < 1 || n_z < 1) return NULL;
    orc_ctx *c = calloc(1, sizeof(orc_ctx));
    size_t mm = (size_t)m * m, me = (size_t)(m - 1) * m;
    c->m = m;
    c->n_z = n_z;
    c->ap = dup_d(ap, n_z), c->bp = dup_d(bp, n_z), c->cp = dup_d(cp, n_z), c->d = dup_d(d, n_z);
    c->area = dup_d(area, mm), c->east = dup_d(east, me), c->north = dup_d(north, me);
    c->diag = dup_d(diag, mm);
    c->fap = dup_f(ap, n_z), c->fbp = dup_f(bp, n_z), c->fcp = dup_f(cp, n_z);
    c->fd = dup_f(d, n_z);
    c->farea = dup_f(area, mm), c->feast = dup_f(east, me), c->fnorth = dup_f(north, me);
    c->fdiag = dup_f(diag, mm);
    return c;
}

void orc_ctx_destroy(orc_ctx *c) {
    if (!c) return;
    void *ps[] = {c->ap,   c->bp,   c->cp,    c->d,     c->area, c->east, c->north, c->diag,
                  c->fap,  c->fbp,  c->fcp,   c->fd,    c->farea, c->feast, c->fnorth,
                  c->fdiag};
    for (size_t l = 0; l < sizeof(ps) / sizeof(ps[0]); ++l) free(ps[l]);
    free(c);
}

/* field.hpp:23-28 */
static size_t lin(int layout, int i, int j, int k, int m, int n_z) {
    if (layout == 0) return (size_t)n_z * ((size_t)m * i + j) + k;
    return (size_t)m * ((size_t)n_z * j + k) + i;
}

/* splitmix64 draw sequence in canonical (i, j, k) order, field.hpp:180-196 */
static uint64_t smix(uint64_t *s) {
    *s += 0x9e3779b97f4a7c15ull;
    uint64_t z = *s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static ptrdiff_t kstride(int layout, int m) { return layout == 0 ? 1 : m; }

/* -------------------------------------------- precision-generic kernels */
#define ORC_T double
#define ORC_SFX(name) name##_f64
#define ORC_CTX(c, field) (c)->field
#define ORC_SQRT sqrt
#include "acg_oracle_body.inc"
#undef ORC_T
#undef ORC_SFX
#undef ORC_CTX
#undef ORC_SQRT

#define ORC_T float
#define ORC_SFX(name) name##_f32
#define ORC_CTX(c, field) (c)->f##field
#define ORC_SQRT sqrtf
#include "acg_oracle_body.inc"
