// Host-side setup; see setup.hpp.  Reference citations are relative to
// /root/reference/proj.
#include "setup.hpp"

#if defined(__SSE2__)
#include <immintrin.h>
#endif

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace lfb {

namespace {

constexpr int kVoigtIndex[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
constexpr int kVoigtPair[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};

/// Dense LU with partial (or complete) pivoting, A n x n row-major, B n x m.
/// Returns the determinant.
double luSolve(int n, double* a, int m, double* b, bool full_pivot) {
    std::vector<int> colperm(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i)
        colperm[static_cast<std::size_t>(i)] = i;
    double det = 1.0;
    for (int k = 0; k < n; ++k) {
        int pr = k, pc = k;
        double best = -1.0;
        for (int i = k; i < n; ++i)
            for (int j = full_pivot ? k : k; j < (full_pivot ? n : k + 1); ++j)
                if (std::abs(a[i * n + j]) > best) {
                    best = std::abs(a[i * n + j]);
                    pr = i;
                    pc = j;
                }
        if (pr != k) {
            for (int j = 0; j < n; ++j)
                std::swap(a[k * n + j], a[pr * n + j]);
            for (int j = 0; j < m; ++j)
                std::swap(b[k * m + j], b[pr * m + j]);
            det = -det;
        }
        if (pc != k) {
            for (int i = 0; i < n; ++i)
                std::swap(a[i * n + k], a[i * n + pc]);
            std::swap(colperm[static_cast<std::size_t>(k)], colperm[static_cast<std::size_t>(pc)]);
            det = -det;
        }
        det *= a[k * n + k];
        if (a[k * n + k] == 0.0)
            continue;
        for (int i = k + 1; i < n; ++i) {
            const double l = a[i * n + k] / a[k * n + k];
            a[i * n + k] = l;
            for (int j = k + 1; j < n; ++j)
                a[i * n + j] -= l * a[k * n + j];
            for (int j = 0; j < m; ++j)
                b[i * m + j] -= l * b[k * m + j];
        }
    }
    std::vector<double> x(static_cast<std::size_t>(n));
    for (int j = 0; j < m; ++j) {
        for (int i = n - 1; i >= 0; --i) {
            double s = b[i * m + j];
            for (int k = i + 1; k < n; ++k)
                s -= a[i * n + k] * x[static_cast<std::size_t>(k)];
            x[static_cast<std::size_t>(i)] = a[i * n + i] != 0.0 ? s / a[i * n + i] : 0.0;
        }
        for (int i = 0; i < n; ++i)
            b[colperm[static_cast<std::size_t>(i)] * m + j] = x[static_cast<std::size_t>(i)];
    }
    return det;
}

double tensorFromVoigt(const double d[36], int i, int j, int k, int l) {
    return d[kVoigtIndex[i][j] * 6 + kVoigtIndex[k][l]];
}

} // namespace

Knots makeKnots(int degree, int n_knots, const double* knots, const char* which) {
    Knots kv;
    kv.p = degree;
    if (degree < 1)
        raise(LF_ERR_INVALID_ARGUMENT, std::string("KnotVector(") + which + "): degree must be >= 1");
    if (knots == nullptr || n_knots < 2 * (degree + 1))
        raise(LF_ERR_INVALID_ARGUMENT,
              std::string("KnotVector(") + which + "): too few knots for degree " + std::to_string(degree));
    kv.t.assign(knots, knots + n_knots);
    if (!std::is_sorted(kv.t.begin(), kv.t.end()))
        raise(LF_ERR_INVALID_ARGUMENT, std::string("KnotVector(") + which + "): knots must be nondecreasing");
    for (int i = 0; i <= degree; ++i) {
        if (kv.t[static_cast<std::size_t>(i)] != 0.0)
            raise(LF_ERR_INVALID_ARGUMENT, "KnotVector: first degree+1 knots must equal 0");
        if (kv.t[kv.t.size() - 1 - static_cast<std::size_t>(i)] != 1.0)
            raise(LF_ERR_INVALID_ARGUMENT, "KnotVector: last degree+1 knots must equal 1");
    }
    if (degree > kMaxDegree)
        raise(LF_ERR_UNSUPPORTED, "degree above " + std::to_string(kMaxDegree) +
                                      " is not compiled into the device kernels");
    kv.n = n_knots - degree - 1;
    return kv;
}

int evaluateBasis(const Knots& kv, double x, double* vals, double* ders) {
    if (x < 0.0 || x > 1.0)
        raise(LF_ERR_DOMAIN, "KnotVector: point outside [0,1]");
    const int p = kv.p, n = kv.n;
    const std::vector<double>& t = kv.t;
    int span;
    if (x >= 1.0) {
        span = n - 1;
        while (span > p && t[static_cast<std::size_t>(span)] >= 1.0)
            --span;
    } else {
        span = static_cast<int>(std::upper_bound(t.begin() + p, t.begin() + n + 1, x) - t.begin()) - 1;
    }
    double low[kMaxDegree + 2] = {0}, left[kMaxDegree + 2] = {0}, right[kMaxDegree + 2] = {0};
    for (int r = 0; r <= p; ++r)
        vals[r] = 0.0;
    vals[0] = 1.0;
    for (int level = 1; level <= p; ++level) {
        if (level == p)
            for (int r = 0; r <= p; ++r)
                low[r] = vals[r];
        left[level] = x - t[static_cast<std::size_t>(span + 1 - level)];
        right[level] = t[static_cast<std::size_t>(span + level)] - x;
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
        const std::size_t i = static_cast<std::size_t>(first + r);
        double d = 0.0;
        if (r >= 1 && t[i + p] - t[i] > 0.0)
            d += low[r - 1] / (t[i + p] - t[i]);
        if (r <= p - 1 && t[i + p + 1] - t[i + 1] > 0.0)
            d -= low[r] / (t[i + p + 1] - t[i + 1]);
        ders[r] = p * d;
    }
    return first;
}

std::vector<Span> elementSpans(const Knots& kv) {
    std::vector<Span> s;
    for (int k = kv.p; k <= kv.n - 1; ++k)
        if (kv.t[static_cast<std::size_t>(k) + 1] > kv.t[static_cast<std::size_t>(k)])
            s.push_back({kv.t[static_cast<std::size_t>(k)], kv.t[static_cast<std::size_t>(k) + 1], k - kv.p});
    return s;
}

void gaussLegendre(int n, double a, double b, double* pts, double* wts) {
    if (n < 1)
        raise(LF_ERR_INVALID_ARGUMENT, "gaussLegendre: need at least one point");
    const double pi = 3.141592653589793238462643383279502884;
    const int half = (n + 1) / 2;
    for (int i = 0; i < half; ++i) {
        double x = std::cos(pi * (i + 0.75) / (n + 0.5));
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
            if (std::abs(dx) < 1e-15)
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

std::vector<Cell> thicknessCells(const Knots&, const std::vector<Span>& spans,
                                 const std::vector<double>& ifc) {
    if (ifc.size() < 2 || ifc.front() != 0.0 || ifc.back() != 1.0)
        raise(LF_ERR_INVALID_ARGUMENT, "layerwiseThicknessRule: interfaces must run from 0 to 1");
    for (std::size_t i = 1; i < ifc.size(); ++i)
        if (!(ifc[i] > ifc[i - 1]))
            raise(LF_ERR_INVALID_ARGUMENT, "layerwiseThicknessRule: interfaces must be strictly increasing");
    std::vector<Cell> cells;
    const int nl = static_cast<int>(ifc.size()) - 1;
    for (int s = 0; s < static_cast<int>(spans.size()); ++s) {
        // layers overlapping the span: a contiguous range, found by bisection
        const Span& sp = spans[static_cast<std::size_t>(s)];
        int l = static_cast<int>(std::upper_bound(ifc.begin(), ifc.end(), sp.begin) - ifc.begin()) - 1;
        l = std::max(0, l);
        for (; l < nl; ++l) {
            const double lo = std::max(sp.begin, ifc[static_cast<std::size_t>(l)]);
            const double hi = std::min(sp.end, ifc[static_cast<std::size_t>(l) + 1]);
            if (ifc[static_cast<std::size_t>(l)] >= sp.end)
                break;
            if (hi <= lo)
                continue; // zero-measure intersection
            cells.push_back({lo, hi, l, s});
        }
    }
    return cells;
}

void voigtFromConstants(const lf_orthotropic& c, double d[36]) {
    if (c.E1 <= 0 || c.E2 <= 0 || c.E3 <= 0 || c.G12 <= 0 || c.G13 <= 0 || c.G23 <= 0)
        raise(LF_ERR_INVALID_ARGUMENT, "voigtFromConstants: moduli must be positive");
    double s[36] = {0};
    s[0] = 1.0 / c.E1;
    s[7] = 1.0 / c.E2;
    s[14] = 1.0 / c.E3;
    s[1] = s[6] = -c.nu12 / c.E1;
    s[2] = s[12] = -c.nu13 / c.E1;
    s[8] = s[13] = -c.nu23 / c.E2;
    s[21] = 1.0 / c.G12;
    s[28] = 1.0 / c.G13;
    s[35] = 1.0 / c.G23;
    double inv[36] = {0};
    for (int i = 0; i < 6; ++i)
        inv[i * 6 + i] = 1.0;
    luSolve(6, s, 6, inv, false);
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j)
            d[i * 6 + j] = 0.5 * (inv[i * 6 + j] + inv[j * 6 + i]);
    // LLT success check (materials.cpp:91-93)
    double l[36] = {0};
    for (int j = 0; j < 6; ++j) {
        double dd = d[j * 6 + j];
        for (int k = 0; k < j; ++k)
            dd -= l[j * 6 + k] * l[j * 6 + k];
        if (!(dd > 0.0))
            raise(LF_ERR_INVALID_ARGUMENT, "voigtFromConstants: constants give a non-SPD stiffness");
        l[j * 6 + j] = std::sqrt(dd);
        for (int i = j + 1; i < 6; ++i) {
            double s2 = d[i * 6 + j];
            for (int k = 0; k < j; ++k)
                s2 -= l[i * 6 + k] * l[j * 6 + k];
            l[i * 6 + j] = s2 / l[j * 6 + j];
        }
    }
}

void rotateInplane(const double d[36], double theta, double out[36]) {
    const double cs = std::cos(theta), sn = std::sin(theta);
    const double r[9] = {cs, -sn, 0.0, sn, cs, 0.0, 0.0, 0.0, 1.0};
    double c4[81], rot[81];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l)
                    c4[((i * 3 + j) * 3 + k) * 3 + l] = tensorFromVoigt(d, i, j, k, l);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) {
                    double sum = 0.0;
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b)
                            for (int c = 0; c < 3; ++c)
                                for (int e = 0; e < 3; ++e)
                                    sum += r[i * 3 + a] * r[j * 3 + b] * r[k * 3 + c] * r[l * 3 + e] *
                                           c4[((a * 3 + b) * 3 + c) * 3 + e];
                    rot[((i * 3 + j) * 3 + k) * 3 + l] = sum;
                }
    for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b)
            out[a * 6 + b] = rot[((kVoigtPair[a][0] * 3 + kVoigtPair[a][1]) * 3 + kVoigtPair[b][0]) * 3 +
                                 kVoigtPair[b][1]];
}

void angleDecomposition(const lf_orthotropic& c, double out[180]) {
    double d[36];
    voigtFromConstants(c, d);
    const double angles[5] = {0.12, 0.53, 0.97, 1.31, 1.49};
    double m[25], rhs[180];
    for (int k = 0; k < 5; ++k) {
        const double cs = std::cos(angles[k]), sn = std::sin(angles[k]);
        m[k * 5 + 0] = 1.0;
        m[k * 5 + 1] = cs * cs * cs * cs;
        m[k * 5 + 2] = cs * cs * cs * sn;
        m[k * 5 + 3] = cs * cs;
        m[k * 5 + 4] = cs * sn;
        double rot[36];
        rotateInplane(d, angles[k], rot);
        for (int e = 0; e < 36; ++e)
            rhs[k * 36 + e] = rot[e];
    }
    const double det = luSolve(5, m, 36, rhs, false);
    if (std::abs(det) < 1e-12)
        raise(LF_ERR_RUNTIME, "angleDecomposition: singular sampling system");
    std::memcpy(out, rhs, sizeof rhs);
}

namespace {

/// basisTensorEntry (voigt_free.cpp:29-49) with m1 = e1 e1', m2 = e2 e2'.
double basisTensorEntry(int which, int i, int j, int k, int l) {
    auto id = [](int a, int b) { return a == b ? 1.0 : 0.0; };
    auto m1 = [](int a, int b) { return (a == 0 && b == 0) ? 1.0 : 0.0; };
    auto m2 = [](int a, int b) { return (a == 1 && b == 1) ? 1.0 : 0.0; };
    auto sym = [&](auto m) {
        return m(i, k) * id(j, l) + m(i, l) * id(j, k) + id(i, k) * m(j, l) + id(i, l) * m(j, k);
    };
    switch (which) {
    case 0: return id(i, j) * id(k, l);
    case 1: return id(i, k) * id(j, l) + id(i, l) * id(j, k);
    case 2: return m1(i, j) * m1(k, l);
    case 3: return m2(i, j) * m2(k, l);
    case 4: return sym(m1);
    case 5: return sym(m2);
    case 6: return id(i, j) * m1(k, l) + m1(i, j) * id(k, l);
    case 7: return id(i, j) * m2(k, l) + m2(i, j) * id(k, l);
    default: return m1(i, j) * m2(k, l) + m2(i, j) * m1(k, l);
    }
}

} // namespace

void bracketParameters(const lf_orthotropic& c, double out[9]) {
    double d[36];
    voigtFromConstants(c, d);
    constexpr int kEntries[9][4] = {{0, 0, 0, 0}, {1, 1, 1, 1}, {2, 2, 2, 2},
                                    {0, 0, 1, 1}, {0, 0, 2, 2}, {1, 1, 2, 2},
                                    {0, 1, 0, 1}, {0, 2, 0, 2}, {1, 2, 1, 2}};
    double sys[81], rhs[9];
    for (int r = 0; r < 9; ++r) {
        const int i = kEntries[r][0], j = kEntries[r][1], k = kEntries[r][2], l = kEntries[r][3];
        for (int q = 0; q < 9; ++q)
            sys[r * 9 + q] = basisTensorEntry(q, i, j, k, l);
        rhs[r] = tensorFromVoigt(d, i, j, k, l);
    }
    luSolve(9, sys, 1, rhs, true);
    std::memcpy(out, rhs, sizeof rhs);
}

void contractionTable(const double prm[9], double angle, double table[81]) {
    const double lambda = prm[0], mu = prm[1];
    const double* al = prm + 2;
    const double a1[3] = {std::cos(angle), std::sin(angle), 0.0};
    const double a2[3] = {-std::sin(angle), std::cos(angle), 0.0};
    double m1[9], m2[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            m1[3 * r + c] = a1[r] * a1[c];
            m2[3 * r + c] = a2[r] * a2[c];
        }
    auto id = [](int a, int b) { return a == b ? 1.0 : 0.0; };
    for (int i = 0; i < 3; ++i) {
        double a1i[3], a2i[3];
        for (int r = 0; r < 3; ++r) {
            a1i[r] = m1[3 * r + i];
            a2i[r] = m2[3 * r + i];
        }
        for (int j = 0; j < 3; ++j) {
            double a1j[3], a2j[3];
            for (int r = 0; r < 3; ++r) {
                a1j[r] = m1[3 * r + j];
                a2j[r] = m2[3 * r + j];
            }
            const double dij = id(i, j);
            const double ei_a1j = a1j[i], ei_a2j = a2j[i];
            double* e = table + (3 * i + j) * 9;
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    // isotropicEntry (voigt_free.cpp:82-87)
                    double v = lambda * id(r, i) * id(c, j) + mu * (dij * id(r, c) + id(r, j) * id(c, i));
                    v += al[0] * a1i[r] * a1j[c];
                    v += al[1] * a2i[r] * a2j[c];
                    v += al[2] * (ei_a1j * id(r, c) + dij * m1[3 * r + c] + id(r, j) * a1i[c] + a1j[r] * id(c, i));
                    v += al[3] * (ei_a2j * id(r, c) + dij * m2[3 * r + c] + id(r, j) * a2i[c] + a2j[r] * id(c, i));
                    v += al[4] * (id(r, i) * a1j[c] + a1i[r] * id(c, j));
                    v += al[5] * (id(r, i) * a2j[c] + a2i[r] * id(c, j));
                    v += al[6] * (a1i[r] * a2j[c] + a2i[r] * a1j[c]);
                    e[3 * r + c] = v;
                }
        }
    }
}

void tableFromVoigt(const double d[36], double table[81]) {
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            for (int i = 0; i < 3; ++i)
                for (int k = 0; k < 3; ++k)
                    table[(3 * j + l) * 9 + 3 * i + k] = tensorFromVoigt(d, i, j, k, l);
}

bool sameConstants(const lf_orthotropic& a, const lf_orthotropic& b) {
    return a.E1 == b.E1 && a.E2 == b.E2 && a.E3 == b.E3 && a.G12 == b.G12 && a.G13 == b.G13 &&
           a.G23 == b.G23 && a.nu12 == b.nu12 && a.nu13 == b.nu13 && a.nu23 == b.nu23;
}

LayupInfo buildLayup(const lf_problem& p) {
    if (p.n_layers < 1 || p.layers == nullptr || p.interfaces == nullptr)
        raise(LF_ERR_INVALID_ARGUMENT, "Layup: need at least one layer");
    if (p.interfaces[0] != 0.0 || p.interfaces[p.n_layers] != 1.0)
        raise(LF_ERR_INVALID_ARGUMENT, "Layup: interfaces must run from 0 to 1");
    for (int i = 1; i <= p.n_layers; ++i)
        if (!(p.interfaces[i] > p.interfaces[i - 1]))
            raise(LF_ERR_INVALID_ARGUMENT, "Layup: interfaces must be strictly increasing");
    LayupInfo L;
    for (int l = 0; l < p.n_layers; ++l) {
        int id = -1;
        for (int c = 0; c < L.n_configs; ++c) {
            const lf_layer& r = p.layers[L.rep_layer[static_cast<std::size_t>(c)]];
            if (sameConstants(r.constants, p.layers[l].constants) && r.angle == p.layers[l].angle) {
                id = c;
                break;
            }
        }
        if (id < 0) {
            std::array<double, 36> d0{}, d{};
            voigtFromConstants(p.layers[l].constants, d0.data());
            rotateInplane(d0.data(), p.layers[l].angle, d.data());
            L.D.push_back(d);
            L.rep_layer.push_back(l);
            id = L.n_configs++;
        }
        L.layer_config.push_back(id);
    }
    return L;
}

Frame frameAt(const lf_problem& p, double u, double v) {
    double su[3], sv[3];
    const double* g = p.geometry;
    if (p.geometry_kind == LF_GEOM_PLANAR) {
        if (g[0] <= 0.0 || g[1] <= 0.0)
            raise(LF_ERR_INVALID_ARGUMENT, "PlanarRectangle: side lengths must be positive");
        su[0] = g[0], su[1] = 0.0, su[2] = 0.0;
        sv[0] = 0.0, sv[1] = g[1], sv[2] = 0.0;
    } else if (p.geometry_kind == LF_GEOM_BILINEAR) {
        for (int k = 0; k < 3; ++k) {
            su[k] = (1 - v) * (g[3 + k] - g[k]) + v * (g[9 + k] - g[6 + k]);
            sv[k] = (1 - u) * (g[6 + k] - g[k]) + u * (g[9 + k] - g[3 + k]);
        }
    } else {
        raise(LF_ERR_INVALID_ARGUMENT, "frameAt: frame tables carry their own frames");
    }
    Frame f;
    for (int k = 0; k < 3; ++k) {
        f.df[k] = su[k];
        f.df[3 + k] = sv[k];
        f.df[6 + k] = p.direction[k];
    }
    const double* m = f.df; // col-major: m(i,j) = m[3j+i]
#define M(i, j) m[3 * (j) + (i)]
    f.det = M(0, 0) * (M(1, 1) * M(2, 2) - M(2, 1) * M(1, 2)) - M(1, 0) * (M(0, 1) * M(2, 2) - M(2, 1) * M(0, 2)) +
            M(2, 0) * (M(0, 1) * M(1, 2) - M(1, 1) * M(0, 2));
    if (f.det < 1e-14)
        raise(LF_ERR_DOMAIN, "ExtrudedGeometry: degenerate or orientation-reversing Jacobian");
    // inverse(i,j) (row i, col j); dfit(r,c) = inverse(c,r); col-major dfit[3c+r]
    double inv[3][3];
    inv[0][0] = (M(1, 1) * M(2, 2) - M(1, 2) * M(2, 1)) / f.det;
    inv[0][1] = (M(0, 2) * M(2, 1) - M(0, 1) * M(2, 2)) / f.det;
    inv[0][2] = (M(0, 1) * M(1, 2) - M(0, 2) * M(1, 1)) / f.det;
    inv[1][0] = (M(1, 2) * M(2, 0) - M(1, 0) * M(2, 2)) / f.det;
    inv[1][1] = (M(0, 0) * M(2, 2) - M(0, 2) * M(2, 0)) / f.det;
    inv[1][2] = (M(0, 2) * M(1, 0) - M(0, 0) * M(1, 2)) / f.det;
    inv[2][0] = (M(1, 0) * M(2, 1) - M(1, 1) * M(2, 0)) / f.det;
    inv[2][1] = (M(0, 1) * M(2, 0) - M(0, 0) * M(2, 1)) / f.det;
    inv[2][2] = (M(0, 0) * M(1, 1) - M(0, 1) * M(1, 0)) / f.det;
#undef M
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            f.dfit[3 * c + r] = inv[c][r];
    return f;
}

Adjacency adjacency(int p, int n, const std::vector<Span>& spans, const std::vector<char>* enabled) {
    Adjacency a;
    a.lo.assign(static_cast<std::size_t>(n), 0);
    a.len.assign(static_cast<std::size_t>(n), 0);
    a.pre.assign(static_cast<std::size_t>(n) + 1, 0);
    std::vector<int> lo(static_cast<std::size_t>(n), 1 << 30), hi(static_cast<std::size_t>(n), -1);
    for (std::size_t s = 0; s < spans.size(); ++s) {
        if (enabled && !(*enabled)[s])
            continue;
        const int f = spans[s].first;
        for (int i = f; i <= f + p && i < n; ++i) {
            lo[static_cast<std::size_t>(i)] = std::min(lo[static_cast<std::size_t>(i)], f);
            hi[static_cast<std::size_t>(i)] = std::max(hi[static_cast<std::size_t>(i)], f + p);
        }
    }
    for (int i = 0; i < n; ++i) {
        const std::size_t k = static_cast<std::size_t>(i);
        if (hi[k] >= 0) {
            a.lo[k] = lo[k];
            a.len[k] = hi[k] - lo[k] + 1;
        }
        a.pre[k + 1] = a.pre[k] + a.len[k];
        a.max_len = std::max(a.max_len, a.len[k]);
    }
    a.total = a.pre[static_cast<std::size_t>(n)];
    return a;
}

namespace {

void spaceCommon(Setup& s, const lf_problem& p) {
    s.ku = makeKnots(p.degree_u, p.n_knots_u, p.knots_u, "u");
    s.kv = makeKnots(p.degree_v, p.n_knots_v, p.knots_v, "v");
    s.kt = makeKnots(p.degree_t, p.n_knots_t, p.knots_t, "thickness");
    s.spu = elementSpans(s.ku);
    s.spv = elementSpans(s.kv);
    s.spt = elementSpans(s.kt);
    s.n_u = s.ku.n;
    s.n_v = s.kv.n;
    s.n_t = s.kt.n;
    s.n_s = s.n_u * s.n_v;
    // inplanePointCount / thicknessPointCount (assembly.cpp:106-112)
    s.nqu = p.inplane_points > 0 ? p.inplane_points : s.ku.p + 1;
    s.nqv = p.inplane_points > 0 ? p.inplane_points : s.kv.p + 1;
    s.nqt = p.thickness_points > 0 ? p.thickness_points : s.kt.p + 1;
    if (s.nqu > kMaxPoints || s.nqv > kMaxPoints || s.nqt > kMaxPoints)
        raise(LF_ERR_UNSUPPORTED, "more than " + std::to_string(kMaxPoints) + " Gauss points per direction");
    s.ru.resize(static_cast<std::size_t>(s.nqu));
    s.wu.resize(static_cast<std::size_t>(s.nqu));
    s.rv.resize(static_cast<std::size_t>(s.nqv));
    s.wv.resize(static_cast<std::size_t>(s.nqv));
    gaussLegendre(s.nqu, -1.0, 1.0, s.ru.data(), s.wu.data());
    gaussLegendre(s.nqv, -1.0, 1.0, s.rv.data(), s.wv.data());
    s.au = adjacency(s.ku.p, s.n_u, s.spu);
    s.av = adjacency(s.kv.p, s.n_v, s.spv);
    s.S_s = s.au.total * s.av.total;
    s.es_pre.assign(static_cast<std::size_t>(s.n_s) + 1, 0);
    for (int is = 0; is < s.n_s; ++is) {
        const int iu = is % s.n_u, iv = is / s.n_u;
        // P_s(i_s) = P_v(i_v) S_u + L_v(i_v) P_u(i_u)
        s.es_pre[static_cast<std::size_t>(is)] =
            9 * (s.av.pre[static_cast<std::size_t>(iv)] * s.au.total +
                 static_cast<int64_t>(s.av.len[static_cast<std::size_t>(iv)]) * s.au.pre[static_cast<std::size_t>(iu)]);
    }
    s.es_pre[static_cast<std::size_t>(s.n_s)] = 9 * s.S_s;
}

void geometryCommon(Setup& s, const lf_problem& p) {
    const double dn = std::sqrt(p.direction[0] * p.direction[0] + p.direction[1] * p.direction[1] +
                                p.direction[2] * p.direction[2]);
    if (dn == 0.0)
        raise(LF_ERR_INVALID_ARGUMENT, "ExtrudedGeometry: extrusion direction must be nonzero");
    const std::size_t n_el = s.spu.size() * s.spv.size();
    const int nq = s.nqu * s.nqv;
    if (p.geometry_kind == LF_GEOM_PLANAR) {
        s.affine = true;
        s.frame0 = frameAt(p, 0.5, 0.5);
        return;
    }
    s.affine = false;
    s.frames.resize(n_el * static_cast<std::size_t>(nq) * 19);
    if (p.geometry_kind == LF_GEOM_FRAMES) {
        if (p.frames == nullptr)
            raise(LF_ERR_INVALID_ARGUMENT, "LF_GEOM_FRAMES needs a frame table");
        std::memcpy(s.frames.data(), p.frames, s.frames.size() * sizeof(double));
        for (std::size_t k = 0; k < n_el * static_cast<std::size_t>(nq); ++k)
            if (s.frames[k * 19 + 18] < 1e-14)
                raise(LF_ERR_DOMAIN, "ExtrudedGeometry: degenerate or orientation-reversing Jacobian");
        return;
    }
    if (p.geometry_kind != LF_GEOM_BILINEAR)
        raise(LF_ERR_INVALID_ARGUMENT, "unknown geometry kind");
    for (std::size_t e = 0; e < n_el; ++e) {
        const Span& su = s.spu[e % s.spu.size()];
        const Span& sv = s.spv[e / s.spu.size()];
        const double mu = 0.5 * (su.begin + su.end), hu = 0.5 * (su.end - su.begin);
        const double mv = 0.5 * (sv.begin + sv.end), hv = 0.5 * (sv.end - sv.begin);
        for (int qv = 0; qv < s.nqv; ++qv)
            for (int qu = 0; qu < s.nqu; ++qu) {
                const Frame f = frameAt(p, mu + hu * s.ru[static_cast<std::size_t>(qu)],
                                        mv + hv * s.rv[static_cast<std::size_t>(qv)]);
                double* o = s.frames.data() + (e * static_cast<std::size_t>(nq) + static_cast<std::size_t>(qv * s.nqu + qu)) * 19;
                std::memcpy(o, f.df, 9 * sizeof(double));
                std::memcpy(o + 9, f.dfit, 9 * sizeof(double));
                o[18] = f.det;
            }
    }
}

} // namespace

Setup buildSpaceSetup(const lf_problem& p, bool need_geometry) {
    Setup s;
    spaceCommon(s, p);
    if (need_geometry)
        geometryCommon(s, p);
    return s;
}

int64_t functionOffset(const Setup& s, int64_t f) {
    const int64_t F = static_cast<int64_t>(s.n_t) * s.n_s;
    if (f >= F)
        return 9 * s.S_s * s.at.pre[static_cast<std::size_t>(s.n_t)];
    const int t = static_cast<int>(f / s.n_s), is = static_cast<int>(f % s.n_s);
    return 9 * s.S_s * s.at.pre[static_cast<std::size_t>(t)] +
           static_cast<int64_t>(s.at.len[static_cast<std::size_t>(t)]) * s.es_pre[static_cast<std::size_t>(is)];
}

namespace {

/// Streaming writer of consecutive int32 runs: 16-byte non-temporal stores
/// (no read-for-ownership of the destination lines, which would double the
/// host memory traffic while the values' DMA is writing the same memory).
struct ColumnWriter {
    int32_t* p;
    alignas(16) int32_t buf[4];
    int n = 0;
    explicit ColumnWriter(int32_t* dst) : p(dst) {}
    void put(int32_t v) {
#if defined(__SSE2__)
        if (n == 0 && (reinterpret_cast<std::uintptr_t>(p) & 15) != 0) { // head: align the destination
            *p++ = v;
            return;
        }
        buf[n++] = v;
        if (n == 4) {
            _mm_stream_si128(reinterpret_cast<__m128i*>(p), _mm_load_si128(reinterpret_cast<const __m128i*>(buf)));
            p += 4;
            n = 0;
        }
#else
        *p++ = v;
#endif
    }
    /// c0, c0 + 1, ..., c0 + len - 1
    void run(int32_t c0, int len) {
#if defined(__SSE2__)
        while (len > 0 && (n != 0 || (reinterpret_cast<std::uintptr_t>(p) & 15) != 0)) {
            put(c0++);
            --len;
        }
        const __m128i step = _mm_set_epi32(3, 2, 1, 0);
        for (; len >= 4; len -= 4, c0 += 4, p += 4)
            _mm_stream_si128(reinterpret_cast<__m128i*>(p), _mm_add_epi32(_mm_set1_epi32(c0), step));
#endif
        for (; len > 0; --len)
            put(c0++);
    }
    void finish() {
        for (int i = 0; i < n; ++i)
            *p++ = buf[i];
        n = 0;
#if defined(__SSE2__)
        _mm_sfence();
#endif
    }
};

} // namespace

void fillColumns(const Setup& s, int64_t f_lo, int64_t f_hi, int32_t* cols) {
    // row block of function f = (i_t, i_s): rows a = 0..2, each L_t segments
    // (neighbour j_t) of 3 L_s columns ordered (j_s, b); for a
    // fixed (a, j_t, j_v) the 3 L_u columns are consecutive integers
    const int nu = s.n_u, ns = s.n_s;
    ColumnWriter w(cols);
    for (int64_t f = f_lo; f < f_hi; ++f) {
        const int it = static_cast<int>(f / ns), is = static_cast<int>(f % ns);
        const int iu = is % nu, iv = is / nu;
        const int Lt = s.at.len[static_cast<std::size_t>(it)], lot = s.at.lo[static_cast<std::size_t>(it)];
        const int Lu = s.au.len[static_cast<std::size_t>(iu)], lou = s.au.lo[static_cast<std::size_t>(iu)];
        const int Lv = s.av.len[static_cast<std::size_t>(iv)], lov = s.av.lo[static_cast<std::size_t>(iv)];
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < Lt; ++k)
                for (int sv = 0; sv < Lv; ++sv)
                    w.run(3 * ((lot + k) * ns + (lov + sv) * nu + lou), 3 * Lu);
    }
    w.finish();
}

Range rangeOf(const Setup& s, int64_t f0, int64_t f1) {
    const int64_t F = static_cast<int64_t>(s.n_t) * s.n_s;
    if (f1 < 0)
        f1 = F;
    if (f0 < 0 || f0 > f1 || f1 > F)
        raise(LF_ERR_INVALID_ARGUMENT, "row slab out of range");
    Range r;
    r.f0 = f0;
    r.f1 = f1;
    r.rows = 3 * (f1 - f0);
    r.row_begin = 3 * f0;
    r.nnz_begin = functionOffset(s, f0);
    if (f0 == f1) { // empty slab
        r.t0 = r.t1 = static_cast<int>(std::min<int64_t>(f0 / s.n_s, s.n_t));
        r.s0 = 0;
        r.s1 = s.n_s;
        return r;
    }
    r.t0 = static_cast<int>(f0 / s.n_s);
    r.s0 = static_cast<int>(f0 % s.n_s);
    r.t1 = static_cast<int>((f1 + s.n_s - 1) / s.n_s);
    r.s1 = static_cast<int>(f1 - static_cast<int64_t>(r.t1 - 1) * s.n_s);
    r.out_base = static_cast<int64_t>(s.at.len[static_cast<std::size_t>(r.t0)]) * s.es_pre[static_cast<std::size_t>(r.s0)];
    r.n_pairs = s.at.pre[static_cast<std::size_t>(r.t1)] - s.at.pre[static_cast<std::size_t>(r.t0)];
    r.nnz = functionOffset(s, f1) - r.nnz_begin;
    return r;
}

void applyRange(Setup& s, int64_t f0, int64_t f1) {
    const Range r = rangeOf(s, f0, f1);
    s.f0 = r.f0;
    s.f1 = r.f1;
    s.t0 = r.t0;
    s.t1 = r.t1;
    s.s0 = r.s0;
    s.s1 = r.s1;
    s.out_base = r.out_base;
    s.rows = r.rows;
    s.row_begin = r.row_begin;
    s.n_pairs = r.n_pairs;
    s.nnz_begin = r.nnz_begin;
    s.nnz = r.nnz;
}

Setup buildSetupRange(const lf_problem& p, int backend, int64_t f0, int64_t f1) {
    Setup s = buildSetup(p, backend, 0, -1);
    applyRange(s, f0, f1);
    return s;
}

Setup buildSetup(const lf_problem& p, int backend, int t0, int t1) {
    if (backend != LF_BACKEND_FAST && backend != LF_BACKEND_STANDARD && backend != LF_BACKEND_VOIGT_FREE)
        raise(LF_ERR_INVALID_ARGUMENT, "unknown backend");
    Setup s;
    s.backend = backend;
    spaceCommon(s, p);
    s.layup = buildLayup(p);
    geometryCommon(s, p);
    const int L = p.n_layers;
    s.interfaces.assign(p.interfaces, p.interfaces + L + 1);
    s.layer_active.assign(static_cast<std::size_t>(L), p.n_active_layers > 0 ? 0 : 1);
    for (int k = 0; k < p.n_active_layers; ++k)
        if (p.active_layers[k] >= 0 && p.active_layers[k] < L)
            s.layer_active[static_cast<std::size_t>(p.active_layers[k])] = 1;

    // thickness cells (all cells for fast; unmasked cells for standard)
    std::vector<Cell> all = thicknessCells(s.kt, s.spt, s.interfaces);
    const bool standard = backend == LF_BACKEND_STANDARD;
    std::vector<char> span_enabled(s.spt.size(), standard ? 0 : 1);
    s.span_cell0.assign(s.spt.size() + 1, 0);
    for (const Cell& c : all) {
        if (standard && !s.layer_active[static_cast<std::size_t>(c.layer)])
            continue; // buildThicknessData drops masked cells (assembly.cpp:82-84)
        s.cells.push_back(c);
        s.span_cell0[static_cast<std::size_t>(c.span) + 1]++;
        span_enabled[static_cast<std::size_t>(c.span)] = 1;
    }
    for (std::size_t k = 0; k < s.spt.size(); ++k)
        s.span_cell0[k + 1] += s.span_cell0[k];
    for (const Span& sp : s.spt)
        s.spt_first.push_back(sp.first);
    const std::size_t nc = s.cells.size();
    s.cell_pts.resize(nc * static_cast<std::size_t>(s.nqt));
    s.cell_wts.resize(nc * static_cast<std::size_t>(s.nqt));
    for (std::size_t c = 0; c < nc; ++c) {
        gaussLegendre(s.nqt, s.cells[c].lo, s.cells[c].hi, s.cell_pts.data() + c * static_cast<std::size_t>(s.nqt),
                      s.cell_wts.data() + c * static_cast<std::size_t>(s.nqt));
        s.cell_first.push_back(s.spt[static_cast<std::size_t>(s.cells[c].span)].first);
        s.cell_layer.push_back(s.cells[c].layer);
    }
    // thickness adjacency: q.occupied for fast (fast.cpp:203); active spans
    // only for standard (assembly.cpp:184-186)
    s.at = adjacency(s.kt.p, s.n_t, s.spt, &span_enabled);

    // operator terms
    const int nc_cfg = s.layup.n_configs;
    int stat_terms = -1; // terms the work counters report when they differ from n_terms
    if (backend == LF_BACKEND_FAST && p.decompose_angles) {
        std::vector<int> groups; // representative layer per distinct constants, config order
        for (int c = 0; c < nc_cfg; ++c) {
            const int rep = s.layup.rep_layer[static_cast<std::size_t>(c)];
            bool found = false;
            for (int g : groups)
                found = found || sameConstants(p.layers[g].constants, p.layers[rep].constants);
            if (!found)
                groups.push_back(rep);
        }
        s.n_terms = 5 * static_cast<int>(groups.size());
        s.term_table.assign(static_cast<std::size_t>(s.n_terms) * 81, 0.0);
        s.lam.assign(static_cast<std::size_t>(s.n_terms) * L, 0.0);
        s.lam_on.assign(static_cast<std::size_t>(s.n_terms) * L, 0);
        for (std::size_t g = 0; g < groups.size(); ++g) {
            double basis[180];
            angleDecomposition(p.layers[groups[g]].constants, basis);
            for (int k = 0; k < 5; ++k) {
                const std::size_t t = 5 * g + static_cast<std::size_t>(k);
                tableFromVoigt(basis + 36 * k, s.term_table.data() + 81 * t);
                for (int l = 0; l < L; ++l) {
                    if (!sameConstants(p.layers[l].constants, p.layers[groups[g]].constants) ||
                        !s.layer_active[static_cast<std::size_t>(l)])
                        continue;
                    const double c = std::cos(p.layers[l].angle), sn = std::sin(p.layers[l].angle);
                    const double w[5] = {1.0, c * c * c * c, c * c * c * sn, c * c, c * sn};
                    s.lam[t * static_cast<std::size_t>(L) + static_cast<std::size_t>(l)] = w[k];
                    s.lam_on[t * static_cast<std::size_t>(L) + static_cast<std::size_t>(l)] = 1;
                }
            }
        }
        stat_terms = s.n_terms; // the five builds per material the option stands for (fast.cpp:285-336)
        const char* fold = std::getenv("LAMFAST_FOLD_DECOMPOSE");
        if (s.affine && !(fold && fold[0] == '0')) {
            // Constant frame: the in-plane operators are never built (P is
            // formed in registers from the 1D integrals and C~), and every
            // term's contribution is linear in its contraction table.  The
            // five basis tables of a material are therefore summed per
            // distinct (material, angle) configuration with that ply's
            // multipliers BEFORE the combine,
            //     table(config) = sum_k w_k(angle) basis_k(material),
            // which leaves one term per configuration -- the direct form's
            // term count, with the decomposition's arithmetic for the ply
            // stiffness -- instead of ten terms under a vertex function.
            std::vector<double> tab(static_cast<std::size_t>(nc_cfg) * 81, 0.0);
            std::vector<double> lam(static_cast<std::size_t>(nc_cfg) * L, 0.0);
            std::vector<uint8_t> on(static_cast<std::size_t>(nc_cfg) * L, 0);
            for (int c = 0; c < nc_cfg; ++c) {
                const lf_layer& rep = p.layers[s.layup.rep_layer[static_cast<std::size_t>(c)]];
                std::size_t g = 0;
                while (g < groups.size() && !sameConstants(p.layers[groups[g]].constants, rep.constants))
                    ++g;
                const double cs = std::cos(rep.angle), sn = std::sin(rep.angle);
                const double w[5] = {1.0, cs * cs * cs * cs, cs * cs * cs * sn, cs * cs, cs * sn};
                for (int k = 0; k < 5; ++k)
                    for (int e = 0; e < 81; ++e)
                        tab[static_cast<std::size_t>(c) * 81 + e] +=
                            w[k] * s.term_table[(5 * g + static_cast<std::size_t>(k)) * 81 + e];
                for (int l = 0; l < L; ++l)
                    if (s.layup.layer_config[static_cast<std::size_t>(l)] == c &&
                        s.layer_active[static_cast<std::size_t>(l)]) {
                        lam[static_cast<std::size_t>(c) * L + static_cast<std::size_t>(l)] = 1.0;
                        on[static_cast<std::size_t>(c) * L + static_cast<std::size_t>(l)] = 1;
                    }
            }
            s.n_terms = nc_cfg;
            s.term_table = std::move(tab);
            s.lam = std::move(lam);
            s.lam_on = std::move(on);
        }
    } else {
        s.n_terms = nc_cfg;
        s.term_table.assign(static_cast<std::size_t>(s.n_terms) * 81, 0.0);
        s.lam.assign(static_cast<std::size_t>(s.n_terms) * L, 0.0);
        s.lam_on.assign(static_cast<std::size_t>(s.n_terms) * L, 0);
        std::vector<lf_orthotropic> fitted;
        std::vector<std::array<double, 9>> params;
        for (int c = 0; c < nc_cfg; ++c) {
            double* tab = s.term_table.data() + 81 * static_cast<std::size_t>(c);
            const lf_layer& rep = p.layers[s.layup.rep_layer[static_cast<std::size_t>(c)]];
            if (backend == LF_BACKEND_VOIGT_FREE) {
                // coefficient fit shared by configs with equal constants (voigt_free.cpp:270-279)
                std::size_t k = 0;
                while (k < fitted.size() && !sameConstants(fitted[k], rep.constants))
                    ++k;
                if (k == fitted.size()) {
                    fitted.push_back(rep.constants);
                    params.emplace_back();
                    bracketParameters(rep.constants, params.back().data());
                }
                contractionTable(params[k].data(), rep.angle, tab);
            } else {
                tableFromVoigt(s.layup.D[static_cast<std::size_t>(c)].data(), tab);
            }
            for (int l = 0; l < L; ++l)
                if (s.layup.layer_config[static_cast<std::size_t>(l)] == c &&
                    (standard || s.layer_active[static_cast<std::size_t>(l)])) {
                    s.lam[static_cast<std::size_t>(c) * L + static_cast<std::size_t>(l)] = 1.0;
                    s.lam_on[static_cast<std::size_t>(c) * L + static_cast<std::size_t>(l)] = 1;
                }
        }
    }

    // slab
    if (t1 < 0)
        t1 = s.n_t;
    if (t0 < 0 || t0 > t1 || t1 > s.n_t)
        raise(LF_ERR_INVALID_ARGUMENT, "row slab out of range");
    applyRange(s, static_cast<int64_t>(t0) * s.n_s, static_cast<int64_t>(t1) * s.n_s);

    // analytic AssemblyStats (test_fast.cpp:343-351, test_assembly.cpp:249-253)
    const int64_t per_build = static_cast<int64_t>(s.spu.size() * s.spv.size()) * s.nqu * s.nqv;
    if (standard) {
        s.stats.qpoint_visits = per_build * static_cast<int64_t>(nc) * s.nqt;
        s.stats.frame_evaluations = per_build;
    } else {
        const int counted = stat_terms >= 0 ? stat_terms : s.n_terms;
        s.stats.qpoint_visits = per_build * counted;
        s.stats.frame_evaluations = per_build * counted;
        s.stats.operator_builds = counted;
    }
    if (!standard && s.n_terms == 0)
        raise(LF_ERR_INVALID_ARGUMENT, "combineOperators: no operator terms");
    return s;
}

void slabBounds(const Setup& s, int n_parts, int part, int* t0, int* t1) {
    if (n_parts < 1 || part < 0 || part >= n_parts)
        raise(LF_ERR_INVALID_ARGUMENT, "slab: bad part");
    // cut at thickness-function boundaries, balanced by nnz (prefix of pairs)
    auto cut = [&](int k) {
        if (k == 0)
            return 0;
        if (k == n_parts)
            return s.n_t;
        const double target = static_cast<double>(s.at.total) * k / n_parts;
        int best = 0;
        double bestd = 1e300;
        for (int t = 0; t <= s.n_t; ++t) {
            const double d = std::abs(static_cast<double>(s.at.pre[static_cast<std::size_t>(t)]) - target);
            if (d < bestd) {
                bestd = d;
                best = t;
            }
        }
        return best;
    };
    *t0 = cut(part);
    *t1 = std::max(*t0, cut(part + 1));
}

void slabBoundsFunctions(const Setup& s, int n_parts, int part, int64_t* f0, int64_t* f1) {
    if (n_parts < 1 || part < 0 || part >= n_parts)
        raise(LF_ERR_INVALID_ARGUMENT, "slab: bad part");
    // cut at function boundaries, balanced by nnz: the prefix functionOffset
    // is nondecreasing in f, so the closest cut is found by bisection
    const int64_t F = static_cast<int64_t>(s.n_t) * s.n_s;
    const int64_t total = functionOffset(s, F);
    auto cut = [&](int k) -> int64_t {
        if (k == 0)
            return 0;
        if (k == n_parts)
            return F;
        const long double target = static_cast<long double>(total) * k / n_parts;
        int64_t lo = 0, hi = F; // first f with offset >= target lies in [lo, hi]
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (static_cast<long double>(functionOffset(s, mid)) < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        if (lo > 0 && target - functionOffset(s, lo - 1) < functionOffset(s, lo) - target)
            --lo;
        return lo;
    };
    *f0 = cut(part);
    *f1 = std::max(*f0, cut(part + 1));
}

} // namespace lfb
