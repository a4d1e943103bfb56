/*
 * lamfast_oracle.c -- TEST INFRASTRUCTURE (the checker), never the product.
 *
 * A plain-C restatement of the reference lamfast assembly path
 * (/root/reference/proj, arXiv 1905.05417).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  Each function cites the
 * reference file:line it restates.  Parity of this restatement is pinned
 * (tests/test_oracle.py) against
 *   - the known-answer values frozen in the reference's own tests, and
 *   - the UNMODIFIED reference sources compiled here (oracle/_ref), on small
 *     problems and on tests/golden fixtures generated from them.
 *
 * Differences from the reference that are not algorithmic:
 *   - dense 6x6 inverse / LU use textbook partial pivoting instead of
 *     Eigen's kernels, and the small GEMMs are plain loops: last-bit
 *     differences only;
 *   - the CSR is produced directly in sorted order, computing positions in
 *     closed form, instead of triplets + stable_sort (sparse.cpp:30-55).  For
 *     the fast path every block is produced once; for the standard path the
 *     duplicates are accumulated in the same insertion order the stable sort
 *     preserves, so the sums are formed in the same order;
 *   - a slab mode restricts output to thickness rows [t_begin, t_end).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lamfast_cuda.h"

#define ORC_MAXP 8
#define ORC_MAXQ 16

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int orc_fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---------------------------------------------------------------------- */
/* splines (splines.cpp)                                                    */

typedef struct {
    int p, nk, n;
    const double* t;
} orc_kv;

/* KnotVector ctor validation (splines.cpp:10-25). */
static int kv_init(orc_kv* kv, int p, int nk, const double* t) {
    kv->p = p;
    kv->nk = nk;
    kv->t = t;
    kv->n = nk - p - 1;
    if (p < 1)
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "KnotVector: degree must be >= 1");
    if (nk < 2 * (p + 1))
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "KnotVector: too few knots");
    for (int i = 1; i < nk; ++i)
        if (t[i] < t[i - 1])
            return orc_fail(LF_ERR_INVALID_ARGUMENT, "KnotVector: knots must be nondecreasing");
    for (int i = 0; i <= p; ++i)
        if (t[i] != 0.0 || t[nk - 1 - i] != 1.0)
            return orc_fail(LF_ERR_INVALID_ARGUMENT, "KnotVector: clamped ends required");
    return LF_OK;
}

/* KnotVector::findSpan (splines.cpp:37-51). */
static int kv_find_span(const orc_kv* kv, double x) {
    const int p = kv->p, n = kv->n;
    if (x >= 1.0) {
        int k = n - 1;
        while (k > p && kv->t[k] >= 1.0)
            --k;
        return k;
    }
    /* upper_bound over t[p .. n] */
    int lo = p, hi = n + 1;
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (kv->t[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo - 1;
}

/* KnotVector::evaluate (splines.cpp:53-101): triangular Cox-de Boor. */
static int kv_eval(const orc_kv* kv, double x, double* vals, double* ders) {
    const int p = kv->p;
    const double* t = kv->t;
    const int span = kv_find_span(kv, x);
    double low[ORC_MAXP + 1], left[ORC_MAXP + 1], right[ORC_MAXP + 1];
    for (int r = 0; r <= p; ++r)
        vals[r] = low[r] = left[r] = right[r] = 0.0;
    vals[0] = 1.0;
    for (int level = 1; level <= p; ++level) {
        if (level == p)
            for (int r = 0; r <= p; ++r)
                low[r] = vals[r];
        left[level] = x - t[span + 1 - level];
        right[level] = t[span + level] - x;
        double saved = 0.0;
        for (int r = 0; r < level; ++r) {
            const double denom = right[r + 1] + left[level - r];
            const double tmp = denom > 0.0 ? vals[r] / denom : 0.0;
            vals[r] = saved + right[r + 1] * tmp;
            saved = left[level - r] * tmp;
        }
        vals[level] = saved;
    }
    const int first = span - p;
    for (int r = 0; r <= p; ++r) {
        const int i = first + r;
        double d = 0.0;
        if (r >= 1) {
            const double den = t[i + p] - t[i];
            if (den > 0.0)
                d += low[r - 1] / den;
        }
        if (r <= p - 1) {
            const double den = t[i + p + 1] - t[i + 1];
            if (den > 0.0)
                d -= low[r] / den;
        }
        ders[r] = p * d;
    }
    return first;
}

int orc_basis_eval(int p, int nk, const double* t, double x, int* first, double* vals,
                   double* ders) {
    orc_kv kv;
    int st = kv_init(&kv, p, nk, t);
    if (st)
        return st;
    if (p > ORC_MAXP)
        return orc_fail(LF_ERR_UNSUPPORTED, "oracle: degree too high");
    if (x < 0.0 || x > 1.0)
        return orc_fail(LF_ERR_DOMAIN, "KnotVector: point outside [0,1]");
    *first = kv_eval(&kv, x, vals, ders);
    return LF_OK;
}

typedef struct {
    double begin, end;
    int first;
} orc_span;

/* KnotVector::elementSpans (splines.cpp:103-112); returns count. */
static int kv_spans(const orc_kv* kv, orc_span* out) {
    int c = 0;
    for (int k = kv->p; k <= kv->n - 1; ++k)
        if (kv->t[k + 1] > kv->t[k]) {
            out[c].begin = kv->t[k];
            out[c].end = kv->t[k + 1];
            out[c].first = k - kv->p;
            ++c;
        }
    return c;
}

/* ---------------------------------------------------------------------- */
/* quadrature (quadrature.cpp)                                              */

/* gaussLegendre(n) then mapped to [a, b] (quadrature.cpp:9-57). */
void orc_gauss(int n, double a, double b, double* pts, double* wts) {
    const int half = (n + 1) / 2;
    const double pi = 3.141592653589793238462643383279502884;
    for (int i = 0; i < half; ++i) {
        double x = cos(pi * (i + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int iter = 0; iter < 100; ++iter) {
            double p0 = 1.0, p1 = x;
            for (int k = 2; k <= n; ++k) {
                const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / dp;
            x -= dx;
            if (fabs(dx) < 1e-15)
                break;
        }
        const double w = 2.0 / ((1.0 - x * x) * dp * dp);
        pts[i] = -x;
        pts[n - 1 - i] = x;
        wts[i] = w;
        wts[n - 1 - i] = w;
    }
    if (n % 2 == 1)
        pts[half - 1] = 0.0;
    const double mid = 0.5 * (a + b), hw = 0.5 * (b - a);
    for (int i = 0; i < n; ++i) {
        pts[i] = mid + hw * pts[i];
        wts[i] *= hw;
    }
}

typedef struct {
    double lo, hi;
    int layer, span;
    double pts[ORC_MAXQ], wts[ORC_MAXQ];
} orc_cell;

/* layerwiseThicknessRule (quadrature.cpp:59-87); returns count or -1. */
static int thickness_cells(const orc_kv* kt, int n_layers, const double* ifc, int npts,
                           orc_cell** out) {
    if (n_layers < 1 || ifc[0] != 0.0 || ifc[n_layers] != 1.0)
        return -orc_fail(LF_ERR_INVALID_ARGUMENT, "layerwiseThicknessRule: interfaces 0..1");
    for (int i = 1; i <= n_layers; ++i)
        if (!(ifc[i] > ifc[i - 1]))
            return -orc_fail(LF_ERR_INVALID_ARGUMENT, "interfaces must be strictly increasing");
    orc_span* spans = malloc(sizeof(orc_span) * (size_t)kt->nk);
    const int ns = kv_spans(kt, spans);
    orc_cell* cells = malloc(sizeof(orc_cell) * (size_t)(ns + n_layers));
    int c = 0;
    for (int s = 0; s < ns; ++s)
        for (int l = 0; l < n_layers; ++l) {
            const double lo = spans[s].begin > ifc[l] ? spans[s].begin : ifc[l];
            const double hi = spans[s].end < ifc[l + 1] ? spans[s].end : ifc[l + 1];
            if (hi <= lo)
                continue;
            cells[c].lo = lo;
            cells[c].hi = hi;
            cells[c].layer = l;
            cells[c].span = s;
            orc_gauss(npts, lo, hi, cells[c].pts, cells[c].wts);
            ++c;
        }
    free(spans);
    *out = cells;
    return c;
}

/* ---------------------------------------------------------------------- */
/* materials (materials.cpp)                                                */

static const int kVoigtIndex[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
static const int kVoigtPair[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};

/* LU with partial pivoting; solves A X = B in place (A n x n row-major, B n x m). */
static int lu_solve(int n, double* a, int m, double* b, double* det_out) {
    double det = 1.0;
    for (int k = 0; k < n; ++k) {
        int piv = k;
        for (int i = k + 1; i < n; ++i)
            if (fabs(a[i * n + k]) > fabs(a[piv * n + k]))
                piv = i;
        if (piv != k) {
            for (int j = 0; j < n; ++j) {
                double t = a[k * n + j];
                a[k * n + j] = a[piv * n + j];
                a[piv * n + j] = t;
            }
            for (int j = 0; j < m; ++j) {
                double t = b[k * m + j];
                b[k * m + j] = b[piv * m + j];
                b[piv * m + j] = t;
            }
            det = -det;
        }
        det *= a[k * n + k];
        if (a[k * n + k] == 0.0) {
            if (det_out)
                *det_out = 0.0;
            return -1;
        }
        for (int i = k + 1; i < n; ++i) {
            const double l = a[i * n + k] / a[k * n + k];
            a[i * n + k] = l;
            for (int j = k + 1; j < n; ++j)
                a[i * n + j] -= l * a[k * n + j];
            for (int j = 0; j < m; ++j)
                b[i * m + j] -= l * b[k * m + j];
        }
    }
    for (int j = 0; j < m; ++j)
        for (int i = n - 1; i >= 0; --i) {
            double s = b[i * m + j];
            for (int k = i + 1; k < n; ++k)
                s -= a[i * n + k] * b[k * m + j];
            b[i * m + j] = s / a[i * n + i];
        }
    if (det_out)
        *det_out = det;
    return 0;
}

/* voigtFromConstants (materials.cpp:73-95). */
int orc_voigt_from_constants(const lf_orthotropic* c, double d[36]) {
    if (c->E1 <= 0 || c->E2 <= 0 || c->E3 <= 0 || c->G12 <= 0 || c->G13 <= 0 || c->G23 <= 0)
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "voigtFromConstants: moduli must be positive");
    double s[36] = {0};
    s[0] = 1.0 / c->E1;
    s[7] = 1.0 / c->E2;
    s[14] = 1.0 / c->E3;
    s[1] = s[6] = -c->nu12 / c->E1;
    s[2] = s[12] = -c->nu13 / c->E1;
    s[8] = s[13] = -c->nu23 / c->E2;
    s[21] = 1.0 / c->G12;
    s[28] = 1.0 / c->G13;
    s[35] = 1.0 / c->G23;
    double inv[36] = {0};
    for (int i = 0; i < 6; ++i)
        inv[i * 6 + i] = 1.0;
    lu_solve(6, s, 6, inv, NULL);
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j)
            d[i * 6 + j] = 0.5 * (inv[i * 6 + j] + inv[j * 6 + i]);
    /* LLT positivity check (materials.cpp:91-93). */
    double l[36] = {0};
    for (int j = 0; j < 6; ++j) {
        double dd = d[j * 6 + j];
        for (int k = 0; k < j; ++k)
            dd -= l[j * 6 + k] * l[j * 6 + k];
        if (!(dd > 0.0))
            return orc_fail(LF_ERR_INVALID_ARGUMENT, "voigtFromConstants: non-SPD stiffness");
        l[j * 6 + j] = sqrt(dd);
        for (int i = j + 1; i < 6; ++i) {
            double s2 = d[i * 6 + j];
            for (int k = 0; k < j; ++k)
                s2 -= l[i * 6 + k] * l[j * 6 + k];
            l[i * 6 + j] = s2 / l[j * 6 + j];
        }
    }
    return LF_OK;
}

/* rotateInplane = fromVoigt -> rotated -> toVoigt (materials.cpp:26-61, 112-117). */
void orc_rotate_inplane(const double d[36], double theta, double out[36]) {
    double c4[81], r[9];
    const double cs = cos(theta), sn = sin(theta);
    r[0] = cs; r[1] = -sn; r[2] = 0.0;
    r[3] = sn; r[4] = cs;  r[5] = 0.0;
    r[6] = 0.0; r[7] = 0.0; r[8] = 1.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l)
                    c4[((i * 3 + j) * 3 + k) * 3 + l] = d[kVoigtIndex[i][j] * 6 + kVoigtIndex[k][l]];
    double rot[81];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) {
                    double sum = 0.0;
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b)
                            for (int c = 0; c < 3; ++c)
                                for (int e = 0; e < 3; ++e)
                                    sum += r[i * 3 + a] * r[j * 3 + b] * r[k * 3 + c] *
                                           r[l * 3 + e] * c4[((a * 3 + b) * 3 + c) * 3 + e];
                    rot[((i * 3 + j) * 3 + k) * 3 + l] = sum;
                }
    for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b)
            out[a * 6 + b] = rot[((kVoigtPair[a][0] * 3 + kVoigtPair[a][1]) * 3 +
                                  kVoigtPair[b][0]) * 3 + kVoigtPair[b][1]];
}

/* angleDecomposition (materials.cpp:119-149). */
int orc_angle_decomposition(const lf_orthotropic* c, double out[180]) {
    double d[36];
    int st = orc_voigt_from_constants(c, d);
    if (st)
        return st;
    const double angles[5] = {0.12, 0.53, 0.97, 1.31, 1.49};
    double m[25], rhs[180];
    for (int k = 0; k < 5; ++k) {
        const double cs = cos(angles[k]), sn = sin(angles[k]);
        m[k * 5 + 0] = 1.0;
        m[k * 5 + 1] = cs * cs * cs * cs;
        m[k * 5 + 2] = cs * cs * cs * sn;
        m[k * 5 + 3] = cs * cs;
        m[k * 5 + 4] = cs * sn;
        double rot[36];
        orc_rotate_inplane(d, angles[k], rot);
        for (int e = 0; e < 36; ++e)
            rhs[k * 36 + e] = rot[e];
    }
    double det = 0.0;
    lu_solve(5, m, 36, rhs, &det);
    if (fabs(det) < 1e-12)
        return orc_fail(LF_ERR_RUNTIME, "angleDecomposition: singular sampling system");
    memcpy(out, rhs, sizeof rhs);
    return LF_OK;
}

static int constants_equal(const lf_orthotropic* a, const lf_orthotropic* b) {
    return a->E1 == b->E1 && a->E2 == b->E2 && a->E3 == b->E3 && a->G12 == b->G12 &&
           a->G13 == b->G13 && a->G23 == b->G23 && a->nu12 == b->nu12 && a->nu13 == b->nu13 &&
           a->nu23 == b->nu23;
}

/* Layup ctor: validation + dedup by exact (constants, angle) (materials.cpp:151-183). */
int orc_layup(const lf_problem* p, int* n_cfg, int* layer_cfg, double* cfg_d) {
    if (p->n_layers < 1)
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "Layup: need at least one layer");
    if (p->interfaces[0] != 0.0 || p->interfaces[p->n_layers] != 1.0)
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "Layup: interfaces must run from 0 to 1");
    for (int i = 1; i <= p->n_layers; ++i)
        if (!(p->interfaces[i] > p->interfaces[i - 1]))
            return orc_fail(LF_ERR_INVALID_ARGUMENT, "Layup: interfaces strictly increasing");
    int nc = 0;
    int* rep = malloc(sizeof(int) * (size_t)p->n_layers);
    for (int l = 0; l < p->n_layers; ++l) {
        int id = -1;
        for (int c = 0; c < nc; ++c) {
            const lf_layer* r = &p->layers[rep[c]];
            if (constants_equal(&r->constants, &p->layers[l].constants) &&
                r->angle == p->layers[l].angle) {
                id = c;
                break;
            }
        }
        if (id < 0) {
            double d[36];
            int st = orc_voigt_from_constants(&p->layers[l].constants, d);
            if (st) {
                free(rep);
                return st;
            }
            orc_rotate_inplane(d, p->layers[l].angle, cfg_d + 36 * nc);
            rep[nc] = l;
            id = nc++;
        }
        layer_cfg[l] = id;
    }
    free(rep);
    *n_cfg = nc;
    return LF_OK;
}

/* ---------------------------------------------------------------------- */
/* geometry (geometry.cpp)                                                  */

/* ExtrudedGeometry::frameAt (geometry.cpp:74-85) for the built-in surfaces
 * (geometry.cpp:8-31); out = df col-major(9), dfit col-major(9), det. */
int orc_frame_at(const lf_problem* p, double u, double v, double out[19]) {
    double su[3], sv[3];
    const double* g = p->geometry;
    if (p->geometry_kind == LF_GEOM_PLANAR) {
        su[0] = g[0]; su[1] = 0.0; su[2] = 0.0;
        sv[0] = 0.0; sv[1] = g[1]; sv[2] = 0.0;
    } else if (p->geometry_kind == LF_GEOM_BILINEAR) {
        for (int k = 0; k < 3; ++k) {
            su[k] = (1 - v) * (g[3 + k] - g[0 + k]) + v * (g[9 + k] - g[6 + k]);
            sv[k] = (1 - u) * (g[6 + k] - g[0 + k]) + u * (g[9 + k] - g[3 + k]);
        }
    } else {
        return orc_fail(LF_ERR_UNSUPPORTED, "oracle: frame tables are not restated");
    }
    double* df = out;
    for (int k = 0; k < 3; ++k) {
        df[k] = su[k];
        df[3 + k] = sv[k];
        df[6 + k] = p->direction[k];
    }
#define M(i, j) df[3 * (j) + (i)]
    const double det = M(0, 0) * (M(1, 1) * M(2, 2) - M(2, 1) * M(1, 2)) -
                       M(1, 0) * (M(0, 1) * M(2, 2) - M(2, 1) * M(0, 2)) +
                       M(2, 0) * (M(0, 1) * M(1, 2) - M(1, 1) * M(0, 2));
    if (det < 1e-14)
        return orc_fail(LF_ERR_DOMAIN, "ExtrudedGeometry: degenerate Jacobian");
    double inv[9]; /* row-major inverse */
    inv[0] = (M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1)) / det;
    inv[1] = (M(0, 2) * M(2, 1) - M(0, 1) * M(2, 2)) / det;
    inv[2] = (M(0, 1) * M(1, 2) - M(0, 2) * M(1, 1)) / det;
    inv[3] = (M(1, 2) * M(2, 0) - M(1, 0) * M(2, 2)) / det;
    inv[4] = (M(0, 0) * M(2, 2) - M(0, 2) * M(2, 0)) / det;
    inv[5] = (M(0, 2) * M(1, 0) - M(0, 0) * M(1, 2)) / det;
    inv[6] = (M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0)) / det;
    inv[7] = (M(0, 1) * M(2, 0) - M(0, 0) * M(2, 1)) / det;
    inv[8] = (M(0, 0) * M(1, 1) - M(0, 1) * M(1, 0)) / det;
#undef M
    /* dfit(r, c) = inv(c, r); stored col-major: dfit[3c + r] = inv[3c + r]. */
    for (int k = 0; k < 9; ++k)
        out[9 + k] = inv[k];
    out[18] = det;
    return LF_OK;
}

/* ---------------------------------------------------------------------- */
/* shared space bookkeeping                                                 */

typedef struct {
    orc_kv ku, kv, kt;
    int nu, nv, nt, ns;
    int pu, pv, pt;
    int nspu, nspv, nspt;
    orc_span *spu, *spv, *spt;
    int nqu, nqv, nqt;
    double ru[ORC_MAXQ], wu[ORC_MAXQ], rv[ORC_MAXQ], wv[ORC_MAXQ];
} orc_space;

static void space_free(orc_space* s) {
    free(s->spu);
    free(s->spv);
    free(s->spt);
}

static int space_init(orc_space* s, const lf_problem* p) {
    memset(s, 0, sizeof *s);
    int st;
    if ((st = kv_init(&s->ku, p->degree_u, p->n_knots_u, p->knots_u)))
        return st;
    if ((st = kv_init(&s->kv, p->degree_v, p->n_knots_v, p->knots_v)))
        return st;
    if ((st = kv_init(&s->kt, p->degree_t, p->n_knots_t, p->knots_t)))
        return st;
    if (p->degree_u > ORC_MAXP || p->degree_v > ORC_MAXP || p->degree_t > ORC_MAXP)
        return orc_fail(LF_ERR_UNSUPPORTED, "oracle: degree too high");
    s->pu = p->degree_u;
    s->pv = p->degree_v;
    s->pt = p->degree_t;
    s->nu = s->ku.n;
    s->nv = s->kv.n;
    s->nt = s->kt.n;
    s->ns = s->nu * s->nv;
    s->spu = malloc(sizeof(orc_span) * (size_t)p->n_knots_u);
    s->spv = malloc(sizeof(orc_span) * (size_t)p->n_knots_v);
    s->spt = malloc(sizeof(orc_span) * (size_t)p->n_knots_t);
    s->nspu = kv_spans(&s->ku, s->spu);
    s->nspv = kv_spans(&s->kv, s->spv);
    s->nspt = kv_spans(&s->kt, s->spt);
    /* inplanePointCount / thicknessPointCount (assembly.cpp:106-112). */
    s->nqu = p->inplane_points > 0 ? p->inplane_points : s->pu + 1;
    s->nqv = p->inplane_points > 0 ? p->inplane_points : s->pv + 1;
    s->nqt = p->thickness_points > 0 ? p->thickness_points : s->pt + 1;
    if (s->nqu > ORC_MAXQ || s->nqv > ORC_MAXQ || s->nqt > ORC_MAXQ)
        return orc_fail(LF_ERR_UNSUPPORTED, "oracle: too many quadrature points");
    orc_gauss(s->nqu, -1.0, 1.0, s->ru, s->wu);
    orc_gauss(s->nqv, -1.0, 1.0, s->rv, s->wv);
    return LF_OK;
}

/* Local quadrature data of one in-plane element (assembly.cpp:14-67). */
typedef struct {
    int funcs[(ORC_MAXP + 1) * (ORC_MAXP + 1)];
    int first_u, first_v;
    int npts;
    double weight[ORC_MAXQ * ORC_MAXQ];
    double frame[ORC_MAXQ * ORC_MAXQ][19];
    double val[ORC_MAXQ * ORC_MAXQ][(ORC_MAXP + 1) * (ORC_MAXP + 1)];
    double du[ORC_MAXQ * ORC_MAXQ][(ORC_MAXP + 1) * (ORC_MAXP + 1)];
    double dv[ORC_MAXQ * ORC_MAXQ][(ORC_MAXP + 1) * (ORC_MAXP + 1)];
} orc_elem;

static int build_elem(const orc_space* s, const lf_problem* p, int eu, int ev, orc_elem* el) {
    const orc_span* su = &s->spu[eu];
    const orc_span* sv = &s->spv[ev];
    el->first_u = su->first;
    el->first_v = sv->first;
    int a = 0;
    for (int jv = 0; jv <= s->pv; ++jv)
        for (int ju = 0; ju <= s->pu; ++ju)
            el->funcs[a++] = (el->first_v + jv) * s->nu + el->first_u + ju;
    const double mid_u = 0.5 * (su->begin + su->end), half_u = 0.5 * (su->end - su->begin);
    const double mid_v = 0.5 * (sv->begin + sv->end), half_v = 0.5 * (sv->end - sv->begin);
    int q = 0;
    for (int qv = 0; qv < s->nqv; ++qv) {
        const double v = mid_v + half_v * s->rv[qv];
        double bvv[ORC_MAXP + 1], bvd[ORC_MAXP + 1];
        kv_eval(&s->kv, v, bvv, bvd);
        for (int qu = 0; qu < s->nqu; ++qu, ++q) {
            const double u = mid_u + half_u * s->ru[qu];
            double buv[ORC_MAXP + 1], bud[ORC_MAXP + 1];
            kv_eval(&s->ku, u, buv, bud);
            el->weight[q] = s->wu[qu] * half_u * s->wv[qv] * half_v;
            if (p->geometry_kind == LF_GEOM_FRAMES) {
                const int e = ev * s->nspu + eu;
                memcpy(el->frame[q], p->frames + ((size_t)e * s->nqu * s->nqv + q) * 19,
                       19 * sizeof(double));
            } else {
                int st = orc_frame_at(p, u, v, el->frame[q]);
                if (st)
                    return st;
            }
            for (int jv = 0; jv <= s->pv; ++jv)
                for (int ju = 0; ju <= s->pu; ++ju) {
                    const int aa = jv * (s->pu + 1) + ju;
                    el->val[q][aa] = buv[ju] * bvv[jv];
                    el->du[q][aa] = bud[ju] * bvv[jv];
                    el->dv[q][aa] = buv[ju] * bvd[jv];
                }
        }
    }
    el->npts = q;
    return LF_OK;
}

/* writeStrainColumns (assembly.cpp:125-130): W is 6 x ncols, row-major. */
static void strain_cols(double* w, int ncols, int a, const double g[3]) {
    const int c0 = 3 * a, c1 = 3 * a + 1, c2 = 3 * a + 2;
    for (int r = 0; r < 6; ++r)
        w[r * ncols + c0] = w[r * ncols + c1] = w[r * ncols + c2] = 0.0;
    w[0 * ncols + c0] = g[0];
    w[3 * ncols + c0] = g[1];
    w[4 * ncols + c0] = g[2];
    w[1 * ncols + c1] = g[1];
    w[3 * ncols + c1] = g[0];
    w[5 * ncols + c1] = g[2];
    w[2 * ncols + c2] = g[2];
    w[4 * ncols + c2] = g[0];
    w[5 * ncols + c2] = g[1];
}

/* m += W^T (scale D) W, W 6 x n row-major, m n x n row-major. */
static void accumulate_wdw(int n, const double* w, const double* d, double scale, double* m,
                           double* dw) {
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < n; ++c) {
            double s = 0.0;
            for (int k = 0; k < 6; ++k)
                s += (scale * d[r * 6 + k]) * w[k * n + c];
            dw[r * n + c] = s;
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < 6; ++k)
                s += w[k * n + i] * dw[k * n + j];
            m[i * n + j] += s;
        }
}

/* ---------------------------------------------------------------------- */
/* in-plane operators (fast.cpp:13-168)                                     */

typedef struct {
    int nu, nv, pu, pv, bu, bv, ns;
    double* blocks; /* [4][ns][bv][bu][9] */
    char* flags;    /* [ns][bv][bu] */
} orc_pset;

static size_t pset_slot(const orc_pset* ps, int is, int js) {
    const int iu = is % ps->nu, iv = is / ps->nu, ju = js % ps->nu, jv = js / ps->nu;
    return ((size_t)is * ps->bv + (size_t)(jv - iv + ps->pv)) * ps->bu + (size_t)(ju - iu + ps->pu);
}

/* Element-local m = sum_q W^T (w |det| D) W of element e (fast.cpp:98-124). */
static int element_matrix(const orc_space* s, const lf_problem* p, const double* d, int e, orc_elem* el,
                          double* w, double* dw, double* m) {
    const int nl = (s->pu + 1) * (s->pv + 1);
    const int n = 6 * nl;
    const int eu = e % s->nspu, ev = e / s->nspu;
    int st = build_elem(s, p, eu, ev, el);
    if (st)
        return st;
    memset(m, 0, sizeof(double) * (size_t)n * n);
    for (int q = 0; q < el->npts; ++q) {
        const double* G = el->frame[q] + 9; /* dfit col-major: G(r,c) = G[3c+r] */
        for (int js = 0; js < nl; ++js) {
            double g1[3], g2[3];
            for (int r = 0; r < 3; ++r) {
                g1[r] = G[r] * el->du[q][js] + G[3 + r] * el->dv[q][js] + G[6 + r] * 0.0;
                g2[r] = el->val[q][js] * G[6 + r];
            }
            strain_cols(w, n, js, g1);
            strain_cols(w, n, nl + js, g2);
        }
        accumulate_wdw(n, w, d, el->weight[q] * el->frame[q][18], m, dw);
    }
    return LF_OK;
}

/* computeInplaneOperators (fast.cpp:54-168).  Element matrices are formed in
 * parallel (OpenMP) in batches and scattered serially in element order, so
 * every block is summed in the reference's element order whatever the thread
 * count.  want_values = 0: only the occupancy flags (the pattern). */
static int inplane_operators(const orc_space* s, const lf_problem* p, const double* d,
                             orc_pset* ps, int want_values) {
    ps->nu = s->nu;
    ps->nv = s->nv;
    ps->pu = s->pu;
    ps->pv = s->pv;
    ps->bu = 2 * s->pu + 1;
    ps->bv = 2 * s->pv + 1;
    ps->ns = s->ns;
    const size_t per = (size_t)ps->ns * ps->bv * ps->bu;
    ps->blocks = want_values ? calloc(4 * per * 9, sizeof(double)) : NULL;
    ps->flags = calloc(per, 1);
    const int nl = (s->pu + 1) * (s->pv + 1);
    const int n = 6 * nl;
    const int nel = s->nspu * s->nspv;
    if (!want_values) {
        for (int e = 0; e < nel; ++e) {
            const orc_span* su = &s->spu[e % s->nspu];
            const orc_span* sv = &s->spv[e / s->nspu];
            for (int as = 0; as < nl; ++as)
                for (int bs = 0; bs < nl; ++bs) {
                    const int is = (sv->first + as / (s->pu + 1)) * s->nu + su->first + as % (s->pu + 1);
                    const int js = (sv->first + bs / (s->pu + 1)) * s->nu + su->first + bs % (s->pu + 1);
                    ps->flags[pset_slot(ps, is, js)] = 1;
                }
        }
        return LF_OK;
    }
    const int batch = 1024;
    double* mats = malloc(sizeof(double) * (size_t)batch * n * n);
    int* funcs = malloc(sizeof(int) * (size_t)batch * nl);
    int* est = malloc(sizeof(int) * (size_t)batch);
    int st = LF_OK;
    for (int e0 = 0; e0 < nel && !st; e0 += batch) {
        const int nb = nel - e0 < batch ? nel - e0 : batch;
#pragma omp parallel
        {
            orc_elem* el = malloc(sizeof(orc_elem));
            double* w = calloc((size_t)6 * n, sizeof(double));
            double* dw = calloc((size_t)6 * n, sizeof(double));
#pragma omp for schedule(dynamic, 4)
            for (int k = 0; k < nb; ++k) {
                est[k] = element_matrix(s, p, d, e0 + k, el, w, dw, mats + (size_t)k * n * n);
                memcpy(funcs + (size_t)k * nl, el->funcs, sizeof(int) * (size_t)nl);
            }
            free(el);
            free(w);
            free(dw);
        }
        for (int k = 0; k < nb && !st; ++k) {
            if (est[k]) { /* first failing element in element order: redo it serially for its message */
                orc_elem* el = malloc(sizeof(orc_elem));
                st = build_elem(s, p, (e0 + k) % s->nspu, (e0 + k) / s->nspu, el);
                free(el);
                if (!st)
                    st = est[k];
                break;
            }
            const double* m = mats + (size_t)k * n * n;
            const int* fk = funcs + (size_t)k * nl;
            for (int as = 0; as < nl; ++as)
                for (int bs = 0; bs < nl; ++bs) {
                    const int is = fk[as], js = fk[bs];
                    const size_t slot = pset_slot(ps, is, js);
                    for (int ab = 0; ab < 4; ++ab) {
                        const int ra = ab < 2 ? 3 * as : 3 * (nl + as);
                        const int cb = ab % 2 == 0 ? 3 * bs : 3 * (nl + bs);
                        double* blk = ps->blocks + ((size_t)ab * per + slot) * 9;
                        for (int r = 0; r < 3; ++r)
                            for (int c = 0; c < 3; ++c)
                                blk[3 * r + c] += m[(ra + r) * n + cb + c];
                    }
                    ps->flags[slot] = 1;
                }
        }
    }
    free(mats);
    free(funcs);
    free(est);
    return st;
}

int orc_inplane_operators(const lf_problem* p, const double d[36], double* blocks, char* flags) {
    orc_space s;
    int st = space_init(&s, p);
    if (st) {
        space_free(&s);
        return st;
    }
    orc_pset ps;
    st = inplane_operators(&s, p, d, &ps, 1);
    if (!st) {
        const size_t per = (size_t)ps.ns * ps.bv * ps.bu;
        memcpy(blocks, ps.blocks, 4 * per * 9 * sizeof(double));
        memcpy(flags, ps.flags, per);
    }
    free(ps.blocks);
    free(ps.flags);
    space_free(&s);
    return st;
}

/* ---------------------------------------------------------------------- */
/* thickness operators (fast.cpp:170-209)                                   */

/* Per-layer thickness integrals Q_l (fast.cpp:170-209), each held as the
 * dense block of the functions its cells touch: block[l] covers functions
 * [lo[l], lo[l] + w[l]) and stores [4][w][w].  Accumulation order per entry
 * is the reference's (cells in order, points in order). */
typedef struct {
    int n_layers;
    int* lo;
    int* w;
    double** q;
} orc_tblocks;

static void tblocks_free(orc_tblocks* b) {
    for (int l = 0; l < b->n_layers; ++l)
        free(b->q[l]);
    free(b->q);
    free(b->lo);
    free(b->w);
}

static int thickness_blocks(const orc_kv* kt, int n_layers, const double* ifc, int npts, orc_tblocks* tb,
                            char* occ /* [nt][nt] */) {
    const int nt = kt->n, p = kt->p;
    memset(tb, 0, sizeof *tb);
    memset(occ, 0, (size_t)nt * nt);
    orc_cell* cells = NULL;
    const int nc = thickness_cells(kt, n_layers, ifc, npts, &cells);
    if (nc < 0)
        return -nc;
    tb->n_layers = n_layers;
    tb->lo = malloc(sizeof(int) * (size_t)n_layers);
    tb->w = calloc((size_t)n_layers, sizeof(int));
    tb->q = calloc((size_t)n_layers, sizeof(double*));
    int* hi = malloc(sizeof(int) * (size_t)n_layers);
    for (int l = 0; l < n_layers; ++l) {
        tb->lo[l] = nt;
        hi[l] = -1;
    }
    /* function range of each layer's cells */
    for (int c = 0; c < nc; ++c)
        for (int k = 0; k < npts; ++k) {
            double v[ORC_MAXP + 1], dd[ORC_MAXP + 1];
            const int first = kv_eval(kt, cells[c].pts[k], v, dd);
            const int l = cells[c].layer;
            if (first < tb->lo[l])
                tb->lo[l] = first;
            if (first + p > hi[l])
                hi[l] = first + p;
        }
    for (int l = 0; l < n_layers; ++l) {
        if (hi[l] < tb->lo[l])
            tb->lo[l] = 0, hi[l] = -1;
        tb->w[l] = hi[l] - tb->lo[l] + 1;
        tb->q[l] = calloc((size_t)4 * tb->w[l] * tb->w[l] + 1, sizeof(double));
    }
    free(hi);
    for (int c = 0; c < nc; ++c) {
        const int l = cells[c].layer, w = tb->w[l], lo = tb->lo[l];
        double* fam = tb->q[l];
        const size_t ww = (size_t)w * w;
        for (int k = 0; k < npts; ++k) {
            const double wq = cells[c].wts[k];
            double v[ORC_MAXP + 1], dd[ORC_MAXP + 1];
            const int first = kv_eval(kt, cells[c].pts[k], v, dd);
            for (int a = 0; a <= p; ++a)
                for (int b = 0; b <= p; ++b) {
                    const size_t ij = (size_t)(first + a - lo) * w + (first + b - lo);
                    fam[0 * ww + ij] += wq * v[a] * v[b];
                    fam[1 * ww + ij] += wq * v[a] * dd[b];
                    fam[2 * ww + ij] += wq * dd[a] * v[b];
                    fam[3 * ww + ij] += wq * dd[a] * dd[b];
                    occ[(size_t)(first + a) * nt + (first + b)] = 1;
                }
        }
    }
    free(cells);
    return LF_OK;
}

/* thick[(f * nt + i) * nt + j] += weight * Q_l (family-major dense [4][nt][nt]). */
static void add_layer_block(const orc_tblocks* tb, int l, double weight, int nt, double* thick) {
    const int w = tb->w[l], lo = tb->lo[l];
    const size_t nn = (size_t)nt * nt, ww = (size_t)w * w;
    for (int f = 0; f < 4; ++f)
        for (int i = 0; i < w; ++i)
            for (int j = 0; j < w; ++j)
                thick[f * nn + (size_t)(lo + i) * nt + (lo + j)] += weight * tb->q[l][f * ww + (size_t)i * w + j];
}

static int thickness_operators(const orc_kv* kt, int n_layers, const double* ifc, int npts,
                               double* q /* [L][4][nt][nt] */, char* occ /* [nt][nt] */) {
    const int nt = kt->n;
    orc_tblocks tb;
    const int st = thickness_blocks(kt, n_layers, ifc, npts, &tb, occ);
    if (st)
        return st;
    memset(q, 0, sizeof(double) * (size_t)n_layers * 4 * nt * nt);
    for (int l = 0; l < n_layers; ++l)
        add_layer_block(&tb, l, 1.0, nt, q + (size_t)l * 4 * nt * nt);
    tblocks_free(&tb);
    return LF_OK;
}

int orc_thickness_operators(int p, int nk, const double* t, int n_ifc, const double* ifc,
                            int npts, double* q, char* occ) {
    orc_kv kt;
    int st = kv_init(&kt, p, nk, t);
    if (st)
        return st;
    if (npts > ORC_MAXQ || p > ORC_MAXP)
        return orc_fail(LF_ERR_UNSUPPORTED, "oracle: limits");
    return thickness_operators(&kt, n_ifc - 1, ifc, npts, q, occ);
}

/* ---------------------------------------------------------------------- */
/* fast assembly: assembleFast + combineOperators (fast.cpp:211-339)        */

static int layer_active(const lf_problem* p, int l) {
    if (p->n_active_layers <= 0)
        return 1;
    for (int k = 0; k < p->n_active_layers; ++k)
        if (p->active_layers[k] == l)
            return 1;
    return 0;
}

typedef struct {
    int n;
    orc_pset* ps;     /* n operator sets */
    double* thick;    /* [n][4][nt][nt] */
} orc_terms;

static void terms_free(orc_terms* t) {
    for (int k = 0; k < t->n; ++k) {
        free(t->ps[k].blocks);
        free(t->ps[k].flags);
    }
    free(t->ps);
    free(t->thick);
}

/* Operator terms of assembleFast (fast.cpp:283-336) or assembleVoigtFree's
 * equivalent (here with strain-form P; both produce the same operators). */
static int build_terms(const orc_space* s, const lf_problem* p, orc_terms* terms, char* occ,
                       lf_stats* stats, int want_values) {
    const int nt = s->nt, L = p->n_layers;
    int* cfg = malloc(sizeof(int) * (size_t)L);
    double* cd = malloc(sizeof(double) * 36 * (size_t)L);
    int ncfg = 0;
    int st = orc_layup(p, &ncfg, cfg, cd);
    orc_tblocks tb;
    memset(&tb, 0, sizeof tb);
    memset(terms, 0, sizeof *terms);
    if (st)
        goto done;
    if ((st = thickness_blocks(&s->kt, L, p->interfaces, s->nqt, &tb, occ)))
        goto done;
    const size_t nn = (size_t)nt * nt;
    if (!p->decompose_angles) {
        terms->n = ncfg;
        terms->ps = calloc((size_t)ncfg, sizeof(orc_pset));
        terms->thick = calloc((size_t)ncfg * 4 * nn, sizeof(double));
        for (int c = 0; c < ncfg && !st; ++c) {
            st = inplane_operators(s, p, cd + 36 * c, &terms->ps[c], want_values);
            for (int l = 0; l < L; ++l) {
                if (cfg[l] != c || !layer_active(p, l))
                    continue;
                add_layer_block(&tb, l, 1.0, nt, terms->thick + (size_t)c * 4 * nn);
            }
        }
    } else {
        /* groups of distinct constants in config order (fast.cpp:308-311) */
        int* grp = malloc(sizeof(int) * (size_t)L);
        int ng = 0;
        for (int c = 0; c < ncfg; ++c) {
            int rep = -1;
            for (int l = 0; l < L; ++l)
                if (cfg[l] == c) {
                    rep = l;
                    break;
                }
            int found = 0;
            for (int g = 0; g < ng; ++g)
                if (constants_equal(&p->layers[grp[g]].constants, &p->layers[rep].constants))
                    found = 1;
            if (!found)
                grp[ng++] = rep;
        }
        terms->n = 5 * ng;
        terms->ps = calloc((size_t)terms->n, sizeof(orc_pset));
        terms->thick = calloc((size_t)terms->n * 4 * nn, sizeof(double));
        for (int g = 0; g < ng && !st; ++g) {
            double basis[180];
            if ((st = orc_angle_decomposition(&p->layers[grp[g]].constants, basis)))
                break;
            for (int k = 0; k < 5 && !st; ++k) {
                const int t = 5 * g + k;
                st = inplane_operators(s, p, basis + 36 * k, &terms->ps[t], want_values);
                for (int l = 0; l < L; ++l) {
                    if (!constants_equal(&p->layers[l].constants, &p->layers[grp[g]].constants) ||
                        !layer_active(p, l))
                        continue;
                    const double c = cos(p->layers[l].angle), sn = sin(p->layers[l].angle);
                    const double weight[5] = {1.0, c * c * c * c, c * c * c * sn, c * c, c * sn};
                    add_layer_block(&tb, l, weight[k], nt, terms->thick + (size_t)t * 4 * nn);
                }
            }
        }
        free(grp);
    }
    if (stats && !st) {
        const int64_t per = (int64_t)s->nspu * s->nspv * s->nqu * s->nqv;
        stats->qpoint_visits += per * terms->n;
        stats->frame_evaluations += per * terms->n;
        stats->operator_builds += terms->n;
    }
done:
    if (tb.q)
        tblocks_free(&tb);
    free(cfg);
    free(cd);
    return st;
}

/* combineOperators (fast.cpp:211-264) in slab mode; CSR emitted in sorted
 * order.  With values == NULL only counts rows/nnz.  Row block (it, is) holds
 * 3 rows of occ(it) x band(is) x 3 entries each (the triplets addBlock emits
 * for that function, sparse.cpp:15-21); its offset is the prefix sum of the
 * block sizes, so blocks are filled independently (OpenMP) with the same
 * values and columns as the serial loop. */
static int combine(const orc_space* s, const orc_terms* terms, const char* occ, int t0, int t1,
                   int64_t* row_ptr, int32_t* cols, double* values, int64_t* nnz_out) {
    const int nt = s->nt, ns = s->ns;
    const orc_pset* pat = &terms->ps[0];
    const size_t per = (size_t)pat->ns * pat->bv * pat->bu;
    const size_t nn = (size_t)nt * nt;
    const int bmax = pat->bu * pat->bv;
    int* bandcols = malloc(sizeof(int) * (size_t)ns * bmax); /* occupied js of each is, ascending */
    int* nband = malloc(sizeof(int) * (size_t)ns);
    for (int is = 0; is < ns; ++is) {
        const int iu = is % s->nu, iv = is / s->nu;
        int nb = 0;
        for (int jv = iv - s->pv < 0 ? 0 : iv - s->pv; jv <= (iv + s->pv < s->nv - 1 ? iv + s->pv : s->nv - 1); ++jv)
            for (int ju = iu - s->pu < 0 ? 0 : iu - s->pu; ju <= (iu + s->pu < s->nu - 1 ? iu + s->pu : s->nu - 1); ++ju) {
                const int js = jv * s->nu + ju;
                if (pat->flags[pset_slot(pat, is, js)])
                    bandcols[(size_t)is * bmax + nb++] = js;
            }
        nband[is] = nb;
    }
    const int nslab = t1 - t0;
    int* tcols = malloc(sizeof(int) * (size_t)(nslab > 0 ? nslab : 1) * nt); /* occupied jt of each it */
    int* ntc = malloc(sizeof(int) * (size_t)(nslab > 0 ? nslab : 1));
    for (int it = t0; it < t1; ++it) {
        int c = 0;
        for (int jt = 0; jt < nt; ++jt)
            if (occ[(size_t)it * nt + jt])
                tcols[(size_t)(it - t0) * nt + c++] = jt;
        ntc[it - t0] = c;
    }
    const size_t nblk = (size_t)(nslab > 0 ? nslab : 0) * ns;
    int64_t* boff = malloc(sizeof(int64_t) * (nblk + 1));
    boff[0] = 0;
    for (size_t bk = 0; bk < nblk; ++bk)
        boff[bk + 1] = boff[bk] + 9LL * ntc[bk / ns] * nband[bk % ns];
    if (row_ptr) {
        row_ptr[0] = 0;
        for (size_t bk = 0; bk < nblk; ++bk) {
            const int64_t len = 3LL * ntc[bk / ns] * nband[bk % ns];
            for (int a = 0; a < 3; ++a)
                row_ptr[3 * bk + a + 1] = boff[bk] + (a + 1) * len;
        }
    }
    if (values) {
#pragma omp parallel for schedule(dynamic, 64)
        for (long long bk = 0; bk < (long long)nblk; ++bk) {
            const int it = t0 + (int)(bk / ns), is = (int)(bk % ns);
            const int* jts = tcols + (size_t)(it - t0) * nt;
            const int njt = ntc[it - t0], nb = nband[is];
            int64_t k = boff[bk];
            for (int a = 0; a < 3; ++a)
                for (int x = 0; x < njt; ++x) {
                    const int jt = jts[x];
                    for (int y = 0; y < nb; ++y) {
                        const int js = bandcols[(size_t)is * bmax + y];
                        const size_t slot = pset_slot(pat, is, js);
                        for (int b = 0; b < 3; ++b, ++k) {
                            double blk = 0.0;
                            for (int t = 0; t < terms->n; ++t)
                                for (int ab = 0; ab < 4; ++ab)
                                    blk += terms->ps[t].blocks[((size_t)ab * per + slot) * 9 + 3 * a + b] *
                                           terms->thick[((size_t)t * 4 + ab) * nn + (size_t)it * nt + jt];
                            values[k] = 0.0 + blk; /* finalize: sum = 0.0; sum += v */
                            cols[k] = 3 * (jt * ns + js) + b;
                        }
                    }
                }
        }
    }
    *nnz_out = boff[nblk];
    free(boff);
    free(tcols);
    free(ntc);
    free(bandcols);
    free(nband);
    return LF_OK;
}

static int check_slab(const orc_space* s, int* t0, int* t1) {
    if (*t1 < 0)
        *t1 = s->nt;
    if (*t0 < 0 || *t0 > *t1 || *t1 > s->nt)
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "oracle: bad slab");
    return LF_OK;
}

/* The operator terms of one problem, built once and combined into any
 * number of row slabs (the checker of a full-size problem compares several
 * slabs; building P is the expensive part). */
typedef struct orc_fast {
    orc_space s;
    orc_terms terms;
    char* occ;
    lf_stats stats;
} orc_fast;

int orc_fast_create(const lf_problem* p, int want_values, orc_fast** out) {
    *out = NULL;
    orc_fast* f = calloc(1, sizeof(orc_fast));
    int st = space_init(&f->s, p);
    if (!st && p->n_layers < 1)
        st = orc_fail(LF_ERR_INVALID_ARGUMENT, "assembleFast: empty layup");
    if (st) {
        space_free(&f->s);
        free(f);
        return st;
    }
    f->occ = malloc((size_t)f->s.nt * f->s.nt);
    st = build_terms(&f->s, p, &f->terms, f->occ, &f->stats, want_values);
    if (!st && f->terms.n == 0)
        st = orc_fail(LF_ERR_INVALID_ARGUMENT, "combineOperators: no operator terms");
    if (st) {
        terms_free(&f->terms);
        free(f->occ);
        space_free(&f->s);
        free(f);
        return st;
    }
    *out = f;
    return LF_OK;
}

void orc_fast_destroy(orc_fast* f) {
    if (!f)
        return;
    terms_free(&f->terms);
    free(f->occ);
    space_free(&f->s);
    free(f);
}

/* Rows of thickness functions [t0, t1); values == NULL: only *nnz (and
 * row_ptr when given).  The handle must have been created with values. */
int orc_fast_slab(const orc_fast* f, int t0, int t1, int64_t* row_ptr, int32_t* cols, double* values,
                  int64_t* nnz) {
    int st = check_slab(&f->s, &t0, &t1);
    if (st)
        return st;
    if (values && !f->terms.ps[0].blocks)
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "oracle: handle built without values");
    return combine(&f->s, &f->terms, f->occ, t0, t1, row_ptr, cols, values, nnz);
}

/* assembleFast (fast.cpp:266-339), rows of thickness functions [t0, t1).
 * values == NULL: only *nnz (and row_ptr when given) are produced. */
int orc_assemble_fast(const lf_problem* p, int t0, int t1, int64_t* row_ptr, int32_t* cols,
                      double* values, int64_t* nnz, lf_stats* stats) {
    orc_fast* f = NULL;
    int st = orc_fast_create(p, values != NULL, &f);
    if (st)
        return st;
    st = orc_fast_slab(f, t0, t1, row_ptr, cols, values, nnz);
    if (!st && values && stats) {
        stats->qpoint_visits += f->stats.qpoint_visits;
        stats->frame_evaluations += f->stats.frame_evaluations;
        stats->operator_builds += f->stats.operator_builds;
    }
    orc_fast_destroy(f);
    return st;
}

/* ---------------------------------------------------------------------- */
/* standard assembly (assembly.cpp:69-104, 134-245)                         */

typedef struct {
    int first;  /* first active thickness function of the span */
    int ncells; /* unmasked cells */
    int cell0;  /* index into the compacted cell list */
} orc_tspan;

/* Thickness adjacency of the standard path: functions sharing a span that
 * has at least one unmasked cell (assembly.cpp:184-186). */
static void std_thickness_adj(const orc_space* s, const orc_tspan* ts, int* lo, int* len) {
    for (int i = 0; i < s->nt; ++i) {
        int l = 1 << 30, h = -1;
        for (int k = 0; k < s->nspt; ++k) {
            if (ts[k].ncells == 0)
                continue;
            if (ts[k].first <= i && i <= ts[k].first + s->pt) {
                if (ts[k].first < l)
                    l = ts[k].first;
                if (ts[k].first + s->pt > h)
                    h = ts[k].first + s->pt;
            }
        }
        lo[i] = h < 0 ? 0 : l;
        len[i] = h < 0 ? 0 : h - l + 1;
    }
}

static void inplane_adj(const orc_span* sp, int nsp, int p, int n, int* lo, int* len) {
    for (int i = 0; i < n; ++i) {
        int l = 1 << 30, h = -1;
        for (int k = 0; k < nsp; ++k)
            if (sp[k].first <= i && i <= sp[k].first + p) {
                if (sp[k].first < l)
                    l = sp[k].first;
                if (sp[k].first + p > h)
                    h = sp[k].first + p;
            }
        lo[i] = h < 0 ? 0 : l;
        len[i] = h < 0 ? 0 : h - l + 1;
    }
}

int orc_assemble_standard(const lf_problem* p, int t0, int t1, int64_t* row_ptr, int32_t* cols,
                          double* values, int64_t* nnz, lf_stats* stats) {
    orc_space s;
    int st = space_init(&s, p);
    if (!st)
        st = check_slab(&s, &t0, &t1);
    if (st) {
        space_free(&s);
        return st;
    }
    if (p->n_layers < 1) {
        space_free(&s);
        return orc_fail(LF_ERR_INVALID_ARGUMENT, "assembleStandard: empty layup");
    }
    const int L = p->n_layers;
    int* cfg = malloc(sizeof(int) * (size_t)L);
    double* cd = malloc(sizeof(double) * 36 * (size_t)L);
    int ncfg = 0;
    orc_cell* cells = NULL;
    int ncells = 0;
    st = orc_layup(p, &ncfg, cfg, cd);
    if (!st) {
        ncells = thickness_cells(&s.kt, L, p->interfaces, s.nqt, &cells);
        if (ncells < 0)
            st = -ncells;
    }
    if (st) {
        free(cfg);
        free(cd);
        space_free(&s);
        return st;
    }
    /* buildThicknessData: group unmasked cells by span (assembly.cpp:69-104). */
    orc_tspan* ts = calloc((size_t)s.nspt, sizeof(orc_tspan));
    int* order = malloc(sizeof(int) * (size_t)(ncells + 1));
    int no = 0;
    for (int k = 0; k < s.nspt; ++k) {
        ts[k].first = s.spt[k].first;
        ts[k].cell0 = no;
        for (int c = 0; c < ncells; ++c)
            if (cells[c].span == k && layer_active(p, cells[c].layer))
                order[no++] = c;
        ts[k].ncells = no - ts[k].cell0;
    }
    /* closed-form pattern of the standard path */
    int *lou = malloc(sizeof(int) * (size_t)s.nu), *lnu = malloc(sizeof(int) * (size_t)s.nu);
    int *lov = malloc(sizeof(int) * (size_t)s.nv), *lnv = malloc(sizeof(int) * (size_t)s.nv);
    int *lot = malloc(sizeof(int) * (size_t)s.nt), *lnt = malloc(sizeof(int) * (size_t)s.nt);
    inplane_adj(s.spu, s.nspu, s.pu, s.nu, lou, lnu);
    inplane_adj(s.spv, s.nspv, s.pv, s.nv, lov, lnv);
    std_thickness_adj(&s, ts, lot, lnt);
    const int64_t rows = (int64_t)3 * s.ns * (t1 - t0);
    int64_t* rp = row_ptr ? row_ptr : malloc(sizeof(int64_t) * (size_t)(rows + 1));
    rp[0] = 0;
    int64_t r = 0;
    for (int it = t0; it < t1; ++it)
        for (int is = 0; is < s.ns; ++is)
            for (int a = 0; a < 3; ++a, ++r)
                rp[r + 1] = rp[r] + (int64_t)3 * lnt[it] * lnu[is % s.nu] * lnv[is / s.nu];
    *nnz = rp[rows];
    if (values) {
        /* columns in sorted order */
        r = 0;
        for (int it = t0; it < t1; ++it)
            for (int is = 0; is < s.ns; ++is) {
                const int iu = is % s.nu, iv = is / s.nu;
                for (int a = 0; a < 3; ++a, ++r) {
                    int64_t k = rp[r];
                    for (int jt = lot[it]; jt < lot[it] + lnt[it]; ++jt)
                        for (int jv = lov[iv]; jv < lov[iv] + lnv[iv]; ++jv)
                            for (int ju = lou[iu]; ju < lou[iu] + lnu[iu]; ++ju)
                                for (int b = 0; b < 3; ++b) {
                                    cols[k] = 3 * (jt * s.ns + jv * s.nu + ju) + b;
                                    values[k++] = 0.0;
                                }
                }
            }
        const int pt = s.pt, nls = (s.pu + 1) * (s.pv + 1), nl = nls * (pt + 1);
        const int n = 3 * nl;
        double* w = calloc((size_t)6 * n, sizeof(double));
        double* dw = calloc((size_t)6 * n, sizeof(double));
        double* kl = calloc((size_t)n * n, sizeof(double));
        double* tv = malloc(sizeof(double) * (size_t)(no + 1) * s.nqt * (pt + 1));
        double* td = malloc(sizeof(double) * (size_t)(no + 1) * s.nqt * (pt + 1));
        for (int c = 0; c < no; ++c)
            for (int q = 0; q < s.nqt; ++q)
                kv_eval(&s.kt, cells[order[c]].pts[q], tv + ((size_t)c * s.nqt + q) * (pt + 1),
                        td + ((size_t)c * s.nqt + q) * (pt + 1));
        orc_elem* el = malloc(sizeof(orc_elem));
        int64_t visits = 0;
        for (int e = 0; e < s.nspu * s.nspv && !st; ++e) {
            if ((st = build_elem(&s, p, e % s.nspu, e / s.nspu, el)))
                break;
            for (int k = 0; k < s.nspt; ++k) {
                if (ts[k].ncells == 0)
                    continue;
                memset(kl, 0, sizeof(double) * (size_t)n * n);
                for (int q2 = 0; q2 < el->npts; ++q2) {
                    const double* G = el->frame[q2] + 9;
                    for (int cc = ts[k].cell0; cc < ts[k].cell0 + ts[k].ncells; ++cc) {
                        const orc_cell* cell = &cells[order[cc]];
                        const double* d = cd + 36 * cfg[cell->layer];
                        for (int q3 = 0; q3 < s.nqt; ++q3) {
                            ++visits;
                            const double* T = tv + ((size_t)cc * s.nqt + q3) * (pt + 1);
                            const double* Td = td + ((size_t)cc * s.nqt + q3) * (pt + 1);
                            for (int jt = 0; jt <= pt; ++jt)
                                for (int js = 0; js < nls; ++js) {
                                    const double gh[3] = {el->du[q2][js] * T[jt],
                                                          el->dv[q2][js] * T[jt],
                                                          el->val[q2][js] * Td[jt]};
                                    double g[3];
                                    for (int rr = 0; rr < 3; ++rr)
                                        g[rr] = G[rr] * gh[0] + G[3 + rr] * gh[1] + G[6 + rr] * gh[2];
                                    strain_cols(w, n, jt * nls + js, g);
                                }
                            accumulate_wdw(n, w, d, el->weight[q2] * cell->wts[q3] * el->frame[q2][18],
                                           kl, dw);
                        }
                    }
                }
                /* scatter (assembly.cpp:217-231) in insertion order */
                for (int at = 0; at <= pt; ++at)
                    for (int as = 0; as < nls; ++as) {
                        const int it = ts[k].first + at;
                        if (it < t0 || it >= t1)
                            continue;
                        const int is = el->funcs[as];
                        const int iu = is % s.nu, iv = is / s.nu;
                        for (int bt = 0; bt <= pt; ++bt)
                            for (int bs = 0; bs < nls; ++bs) {
                                const int jt = ts[k].first + bt, js = el->funcs[bs];
                                const int ju = js % s.nu, jv = js / s.nu;
                                const int64_t off =
                                    ((int64_t)(jt - lot[it]) * lnv[iv] + (jv - lov[iv])) * lnu[iu] +
                                    (ju - lou[iu]);
                                for (int a = 0; a < 3; ++a) {
                                    const int64_t rr = ((int64_t)(it - t0) * s.ns + is) * 3 + a;
                                    for (int b = 0; b < 3; ++b)
                                        values[rp[rr] + 3 * off + b] +=
                                            kl[(3 * (at * nls + as) + a) * n + 3 * (bt * nls + bs) + b];
                                }
                            }
                    }
            }
        }
        if (stats && !st) {
            stats->qpoint_visits += visits;
            stats->frame_evaluations += (int64_t)s.nspu * s.nspv * s.nqu * s.nqv;
        }
        free(w);
        free(dw);
        free(kl);
        free(tv);
        free(td);
        free(el);
    }
    if (!row_ptr)
        free(rp);
    free(lou);
    free(lnu);
    free(lov);
    free(lnv);
    free(lot);
    free(lnt);
    free(ts);
    free(order);
    free(cells);
    free(cfg);
    free(cd);
    space_free(&s);
    return st;
}
