// lamfast C++ API over the B200 C ABI (include/lamfast/lamfast_b200.hpp).
//
// Host-side containers and setup live here; every assembly entry point
// (assembleFast, assembleStandard, assembleVoigtFree, computeInplaneOperators,
// computeInplaneOperatorsBracket, computeThicknessOperators, combineOperators)
// converts its arguments to an lf_problem and calls the CUDA library.  lf_status
// codes are rethrown as the exception types the reference throws.
#include <sys/mman.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "lamfast/lamfast_b200.hpp"
#include "lamfast_cuda.h"

namespace lamfast {

namespace {

int g_device = -1;

[[noreturn]] void rethrow(int status) {
    const std::string msg = lf_last_error();
    switch (status) {
    case LF_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LF_ERR_DOMAIN: throw std::domain_error(msg);
    case LF_ERR_LOGIC: throw std::logic_error(msg);
    case LF_ERR_OUT_OF_MEMORY: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
    }
}

void ok(int status) {
    if (status != LF_OK)
        rethrow(status);
}

/// Sets v's size to n <= capacity() without touching the elements (T trivial):
/// the three-pointer representation {begin, end, end of storage} that
/// libstdc++ and libc++ share is read back against data() / size() /
/// capacity() first, and anything else leaves v alone (false).  This is the
/// library-specific "resize without initialisation" that std::vector itself
/// does not offer before a whole-array overwrite.
template <class T>
bool setSizeUninitialized(std::vector<T>& v, std::size_t n) {
    static_assert(std::is_trivial_v<T>, "elements are overwritten, never constructed");
    struct Rep {
        T *begin, *end, *cap;
    };
    if constexpr (sizeof(std::vector<T>) != sizeof(Rep)) {
        return false;
    } else {
        if (n > v.capacity() || v.data() == nullptr)
            return false;
        Rep r;
        std::memcpy(&r, static_cast<const void*>(&v), sizeof r);
        if (r.begin != v.data() || r.end != r.begin + v.size() || r.cap != r.begin + v.capacity())
            return false;
        r.end = r.begin + n;
        std::memcpy(static_cast<void*>(&v), &r, sizeof r);
        return v.size() == n;
    }
}

/// A std::vector of n elements for a CSR array (the reference's
/// StiffnessMatrix type) that the assembly call overwrites completely.
/// - Large arrays ask for transparent huge pages between the allocation and
///   the first touch, so the pages fault in as 2 MB instead of 4 KB: with 4 KB
///   faults a fresh C4 result (23 GB) cost 8.4 s on the GPU box against 0.41 s
///   for the whole device assembly into pinned memory.
/// - The elements are not zero-filled (setSizeUninitialized): a value-
///   initialising resize is a single-threaded 23 GB fill (2.7 of the 3.2 s a
///   drop-in C4 call took with it), while the assembly's host threads touch
///   and fill disjoint ranges in parallel.  LAMFAST_DROPIN_ZERO_FILL=1, or a
///   standard library with another vector layout, takes the plain resize.
template <class T>
std::vector<T> csrArray(std::size_t n) {
    std::vector<T> v;
    v.reserve(n);
    constexpr std::uintptr_t huge = std::uintptr_t(2) << 20;
    if (n * sizeof(T) >= 4 * huge) {
        const auto p = reinterpret_cast<std::uintptr_t>(v.data());
        const std::uintptr_t a = (p + huge - 1) & ~(huge - 1), e = (p + n * sizeof(T)) & ~(huge - 1);
        if (e > a)
            madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE); // advisory: ignored where THP is off
        static const bool zero_fill = [] {
            const char* e = std::getenv("LAMFAST_DROPIN_ZERO_FILL");
            return e && *e && *e != '0';
        }();
        if (!zero_fill && setSizeUninitialized(v, n))
            return v;
    }
    v.resize(n);
    return v;
}

lf_orthotropic toC(const OrthotropicConstants& c) {
    return {c.E1, c.E2, c.E3, c.G12, c.G13, c.G23, c.nu12, c.nu13, c.nu23};
}

VoigtMatrix fromRowMajor(const double* d) {
    VoigtMatrix m;
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c)
            m(r, c) = d[6 * r + c];
    return m;
}

void toRowMajor(const VoigtMatrix& m, double* d) {
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c)
            d[6 * r + c] = m(r, c);
}

/// Owns the arrays an lf_problem points to.
struct CProblem {
    lf_problem p{};
    std::vector<lf_layer> layers;
    std::vector<double> frames;
    std::vector<int32_t> active;
};

void fillSpace(CProblem& cp, const TensorProductSpace& s) {
    cp.p.degree_u = s.inplaneU().degree();
    cp.p.degree_v = s.inplaneV().degree();
    cp.p.degree_t = s.thickness().degree();
    cp.p.n_knots_u = static_cast<int32_t>(s.inplaneU().knots().size());
    cp.p.n_knots_v = static_cast<int32_t>(s.inplaneV().knots().size());
    cp.p.n_knots_t = static_cast<int32_t>(s.thickness().knots().size());
    cp.p.knots_u = s.inplaneU().knots().data();
    cp.p.knots_v = s.inplaneV().knots().data();
    cp.p.knots_t = s.thickness().knots().data();
}

void fillOptions(CProblem& cp, const AssemblyOptions& o) {
    cp.p.inplane_points = o.inplane_points;
    cp.p.thickness_points = o.thickness_points;
    cp.active.assign(o.active_layers.begin(), o.active_layers.end());
    cp.p.n_active_layers = static_cast<int32_t>(cp.active.size());
    cp.p.active_layers = cp.active.empty() ? nullptr : cp.active.data();
    cp.p.decompose_angles = o.decompose_angles ? 1 : 0;
    cp.p.threads = o.threads;
}

/// Built-in surfaces go to the device by kind; any other SurfaceMap is
/// evaluated here, on the host, at every in-plane quadrature point.
void fillGeometry(CProblem& cp, const TensorProductSpace& s, const ExtrudedGeometry& g, const AssemblyOptions& o) {
    for (int k = 0; k < 3; ++k)
        cp.p.direction[k] = g.direction()[k];
    if (const auto* pr = dynamic_cast<const PlanarRectangle*>(&g.surface())) {
        cp.p.geometry_kind = LF_GEOM_PLANAR;
        cp.p.geometry[0] = pr->lx();
        cp.p.geometry[1] = pr->ly();
        return;
    }
    if (const auto* bq = dynamic_cast<const BilinearQuad*>(&g.surface())) {
        cp.p.geometry_kind = LF_GEOM_BILINEAR;
        for (int c = 0; c < 4; ++c)
            for (int k = 0; k < 3; ++k)
                cp.p.geometry[3 * c + k] = bq->corner(c)[k];
        return;
    }
    cp.p.geometry_kind = LF_GEOM_FRAMES;
    const int nqu = o.inplane_points > 0 ? o.inplane_points : s.inplaneU().degree() + 1;
    const int nqv = o.inplane_points > 0 ? o.inplane_points : s.inplaneV().degree() + 1;
    const QuadratureRule ru = gaussLegendre(nqu), rv = gaussLegendre(nqv);
    const std::vector<Span> su = s.inplaneU().elementSpans(), sv = s.inplaneV().elementSpans();
    cp.frames.clear();
    cp.frames.reserve(su.size() * sv.size() * static_cast<std::size_t>(nqu * nqv) * 19);
    for (const Span& b : sv)
        for (const Span& a : su)
            for (int qv = 0; qv < nqv; ++qv)
                for (int qu = 0; qu < nqu; ++qu) {
                    const double u = 0.5 * (a.begin + a.end) + 0.5 * (a.end - a.begin) * ru.points[static_cast<std::size_t>(qu)];
                    const double v = 0.5 * (b.begin + b.end) + 0.5 * (b.end - b.begin) * rv.points[static_cast<std::size_t>(qv)];
                    const GeometryFrame f = g.frameAt(u, v);
                    for (int c = 0; c < 3; ++c)
                        for (int r = 0; r < 3; ++r)
                            cp.frames.push_back(f.df(r, c));
                    for (int c = 0; c < 3; ++c)
                        for (int r = 0; r < 3; ++r)
                            cp.frames.push_back(f.df_inv_transpose(r, c));
                    cp.frames.push_back(f.det);
                }
    cp.p.frames = cp.frames.data();
}

void fillLayup(CProblem& cp, const Layup& layup) {
    cp.layers.clear();
    for (int l = 0; l < layup.numLayers(); ++l) {
        const MaterialConfig& c = layup.configOf(l);
        cp.layers.push_back({toC(c.constants), c.angle});
    }
    cp.p.n_layers = static_cast<int32_t>(cp.layers.size());
    cp.p.layers = cp.layers.data();
    cp.p.interfaces = layup.interfaces().data();
}

void accumulate(AssemblyStats* stats, const lf_stats& st) {
    if (!stats)
        return;
    stats->qpoint_visits += st.qpoint_visits;
    stats->frame_evaluations += st.frame_evaluations;
    stats->operator_builds += st.operator_builds;
}

StiffnessMatrix assembleOnDevice(int backend, const ProblemSetup& setup, const AssemblyOptions& options,
                                 AssemblyStats* stats) {
    if (setup.layup.numLayers() < 1)
        throw std::invalid_argument("assemble: empty layup");
    CProblem cp;
    fillSpace(cp, setup.space);
    fillGeometry(cp, setup.space, setup.geom, options);
    fillLayup(cp, setup.layup);
    fillOptions(cp, options);
    int64_t dim = 0, nnz = 0;
    ok(lf_pattern_size(&cp.p, backend, &dim, &nnz));
    std::vector<std::int64_t> rp = csrArray<std::int64_t>(static_cast<std::size_t>(dim) + 1);
    std::vector<int> cols = csrArray<int>(static_cast<std::size_t>(nnz));
    std::vector<double> vals = csrArray<double>(static_cast<std::size_t>(nnz));
    lf_stats st{};
    ok(lf_assemble(&cp.p, backend, device(), rp.data(), cols.data(), vals.data(), &st));
    accumulate(stats, st);
    return StiffnessMatrix::fromCsr(static_cast<int>(dim), std::move(rp), std::move(cols), std::move(vals));
}

InPlaneOperatorSet operatorsFromBanded(const TensorProductSpace& s, const std::vector<double>& blocks,
                                       const std::vector<char>& flags) {
    const int nu = s.numU(), nv = s.numV(), pu = s.inplaneU().degree(), pv = s.inplaneV().degree();
    InPlaneOperatorSet set{{InPlaneOperator(nu, nv, pu, pv), InPlaneOperator(nu, nv, pu, pv),
                            InPlaneOperator(nu, nv, pu, pv), InPlaneOperator(nu, nv, pu, pv)}};
    const int bu = 2 * pu + 1, bv = 2 * pv + 1;
    const std::size_t per = static_cast<std::size_t>(nu) * nv * bu * bv;
    for (int is = 0; is < nu * nv; ++is) {
        const int iu = is % nu, iv = is / nu;
        for (int js : set.op[0].bandColumns(is)) {
            const int ju = js % nu, jv = js / nu;
            const std::size_t slot = (static_cast<std::size_t>(is) * bv + (jv - iv + pv)) * bu + (ju - iu + pu);
            if (!flags[slot])
                continue;
            for (int f = 0; f < 4; ++f) {
                Eigen::Matrix3d& b = set.op[static_cast<std::size_t>(f)].block(is, js);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c)
                        b(r, c) = blocks[(f * per + slot) * 9 + 3 * r + c];
                set.op[static_cast<std::size_t>(f)].markOccupied(is, js);
            }
        }
    }
    return set;
}

InPlaneOperatorSet inplaneOnDevice(const TensorProductSpace& space, const ExtrudedGeometry& geom,
                                   const double* voigt, const double* table, const AssemblyOptions& options,
                                   AssemblyStats* stats) {
    CProblem cp;
    fillSpace(cp, space);
    fillGeometry(cp, space, geom, options);
    fillOptions(cp, options);
    const std::size_t per = static_cast<std::size_t>(space.numInplane()) * (2 * space.inplaneU().degree() + 1) *
                            (2 * space.inplaneV().degree() + 1);
    std::vector<double> blocks(4 * per * 9);
    std::vector<char> flags(per);
    lf_stats st{};
    if (voigt)
        ok(lf_inplane_operators(&cp.p, voigt, device(), blocks.data(), flags.data(), &st));
    else
        ok(lf_inplane_operators_bracket(&cp.p, table, device(), blocks.data(), flags.data(), &st));
    accumulate(stats, st);
    return operatorsFromBanded(space, blocks, flags);
}

} // namespace

// ---- device selection ---------------------------------------------------------

void setDevice(int d) { g_device = d; }

int device() {
    if (g_device < 0) {
        const char* env = std::getenv("LAMFAST_DEVICE");
        g_device = env ? std::atoi(env) : 0;
    }
    return g_device;
}

// ---- splines -------------------------------------------------------------------

KnotVector::KnotVector(int degree, std::vector<double> knots) : p_(degree), t_(std::move(knots)) {
    if (p_ < 1)
        throw std::invalid_argument("KnotVector: degree must be >= 1");
    if (static_cast<int>(t_.size()) < 2 * (p_ + 1))
        throw std::invalid_argument("KnotVector: too few knots for degree " + std::to_string(p_));
    if (!std::is_sorted(t_.begin(), t_.end()))
        throw std::invalid_argument("KnotVector: knots must be nondecreasing");
    for (int k = 0; k <= p_; ++k)
        if (t_[static_cast<std::size_t>(k)] != 0.0 || t_[t_.size() - 1 - static_cast<std::size_t>(k)] != 1.0)
            throw std::invalid_argument("KnotVector: the first and last degree+1 knots must be 0 and 1");
}

KnotVector KnotVector::uniform(int degree, int n_elements) {
    if (n_elements < 1)
        throw std::invalid_argument("KnotVector::uniform: n_elements must be >= 1");
    std::vector<double> k(static_cast<std::size_t>(degree) + 1, 0.0);
    for (int e = 1; e < n_elements; ++e)
        k.push_back(static_cast<double>(e) / n_elements);
    k.resize(k.size() + static_cast<std::size_t>(degree) + 1, 1.0);
    return KnotVector(degree, std::move(k));
}

int KnotVector::findSpan(double x) const {
    if (x < 0.0 || x > 1.0)
        throw std::domain_error("KnotVector: point outside [0,1]");
    const int n = numFunctions();
    if (x >= 1.0) {
        int k = n - 1;
        while (k > p_ && t_[static_cast<std::size_t>(k)] >= 1.0)
            --k;
        return k;
    }
    return static_cast<int>(std::upper_bound(t_.begin() + p_, t_.begin() + n + 1, x) - t_.begin()) - 1;
}

BasisEval1D KnotVector::evaluate(double x) const {
    BasisEval1D out;
    out.point = x;
    out.values.resize(static_cast<std::size_t>(p_) + 1);
    out.derivs.resize(static_cast<std::size_t>(p_) + 1);
    if (x < 0.0 || x > 1.0)
        throw std::domain_error("KnotVector: point outside [0,1]");
    int32_t first = 0;
    ok(lf_basis_eval(p_, static_cast<int32_t>(t_.size()), t_.data(), x, &first, out.values.data(),
                     out.derivs.data()));
    out.first_active = first;
    return out;
}

std::vector<Span> KnotVector::elementSpans() const {
    std::vector<Span> s;
    for (int k = p_; k < numFunctions(); ++k)
        if (t_[static_cast<std::size_t>(k) + 1] > t_[static_cast<std::size_t>(k)])
            s.push_back({t_[static_cast<std::size_t>(k)], t_[static_cast<std::size_t>(k) + 1], k - p_});
    return s;
}

TensorProductSpace::TensorProductSpace(KnotVector inplane_u, KnotVector inplane_v, KnotVector thickness)
    : ku_(std::move(inplane_u)), kv_(std::move(inplane_v)), kt_(std::move(thickness)) {}

std::array<int, 3> TensorProductSpace::split(int i) const {
    const int is = i % numInplane();
    return {is % numU(), is / numU(), i / numInplane()};
}

// ---- quadrature ---------------------------------------------------------------

QuadratureRule gaussLegendre(int n) { return gaussLegendre(n, -1.0, 1.0); }

QuadratureRule gaussLegendre(int n, double a, double b) {
    if (n < 1)
        throw std::invalid_argument("gaussLegendre: need at least one point");
    QuadratureRule r;
    r.points.resize(static_cast<std::size_t>(n));
    r.weights.resize(static_cast<std::size_t>(n));
    ok(lf_gauss_legendre(n, a, b, r.points.data(), r.weights.data()));
    return r;
}

std::vector<ThicknessCell> layerwiseThicknessRule(const KnotVector& kv, const std::vector<double>& z, int n_points) {
    if (z.size() < 2 || z.front() != 0.0 || z.back() != 1.0)
        throw std::invalid_argument("layerwiseThicknessRule: interfaces must run from 0 to 1");
    for (std::size_t i = 1; i < z.size(); ++i)
        if (!(z[i] > z[i - 1]))
            throw std::invalid_argument("layerwiseThicknessRule: interfaces must be strictly increasing");
    std::vector<ThicknessCell> out;
    const std::vector<Span> spans = kv.elementSpans();
    for (std::size_t s = 0; s < spans.size(); ++s)
        for (std::size_t l = 0; l + 1 < z.size(); ++l) {
            ThicknessCell c;
            c.lo = std::max(spans[s].begin, z[l]);
            c.hi = std::min(spans[s].end, z[l + 1]);
            if (!(c.hi > c.lo))
                continue;
            c.layer = static_cast<int>(l);
            c.span = static_cast<int>(s);
            c.rule = gaussLegendre(n_points, c.lo, c.hi);
            out.push_back(std::move(c));
        }
    return out;
}

// ---- geometry -------------------------------------------------------------------

PlanarRectangle::PlanarRectangle(double lx, double ly) : a_(lx), b_(ly) {
    if (!(lx > 0.0) || !(ly > 0.0))
        throw std::invalid_argument("PlanarRectangle: side lengths must be positive");
}

SurfacePoint PlanarRectangle::evaluate(double u, double v) const {
    SurfacePoint s;
    s.position = Eigen::Vector3d(a_ * u, b_ * v, 0.0);
    s.du = Eigen::Vector3d(a_, 0.0, 0.0);
    s.dv = Eigen::Vector3d(0.0, b_, 0.0);
    return s;
}

BilinearQuad::BilinearQuad(Eigen::Vector3d c00, Eigen::Vector3d c10, Eigen::Vector3d c01, Eigen::Vector3d c11)
    : c_{std::move(c00), std::move(c10), std::move(c01), std::move(c11)} {}

SurfacePoint BilinearQuad::evaluate(double u, double v) const {
    SurfacePoint s;
    s.position = (1 - u) * (1 - v) * c_[0] + u * (1 - v) * c_[1] + (1 - u) * v * c_[2] + u * v * c_[3];
    s.du = (1 - v) * (c_[1] - c_[0]) + v * (c_[3] - c_[2]);
    s.dv = (1 - u) * (c_[2] - c_[0]) + u * (c_[3] - c_[1]);
    return s;
}

SplineSurface::SplineSurface(KnotVector ku, KnotVector kv, std::vector<Eigen::Vector3d> controls)
    : bu_(std::move(ku)), bv_(std::move(kv)), net_(std::move(controls)) {
    if (net_.size() != static_cast<std::size_t>(bu_.numFunctions()) * static_cast<std::size_t>(bv_.numFunctions()))
        throw std::invalid_argument("SplineSurface: control net size does not match the bases");
}

SurfacePoint SplineSurface::evaluate(double u, double v) const {
    const BasisEval1D eu = bu_.evaluate(u), ev = bv_.evaluate(v);
    SurfacePoint s;
    const int nu = bu_.numFunctions();
    for (int b = 0; b <= bv_.degree(); ++b)
        for (int a = 0; a <= bu_.degree(); ++a) {
            const Eigen::Vector3d& c =
                net_[static_cast<std::size_t>((ev.first_active + b) * nu + eu.first_active + a)];
            const double nu_ = eu.values[static_cast<std::size_t>(a)], nv_ = ev.values[static_cast<std::size_t>(b)];
            s.position += (nu_ * nv_) * c;
            s.du += (eu.derivs[static_cast<std::size_t>(a)] * nv_) * c;
            s.dv += (nu_ * ev.derivs[static_cast<std::size_t>(b)]) * c;
        }
    return s;
}

ExtrudedGeometry::ExtrudedGeometry(std::shared_ptr<const SurfaceMap> surface, Eigen::Vector3d direction)
    : surf_(std::move(surface)), dir_(std::move(direction)) {
    if (!surf_)
        throw std::invalid_argument("ExtrudedGeometry: surface must not be null");
    if (dir_.norm() == 0.0)
        throw std::invalid_argument("ExtrudedGeometry: extrusion direction must be nonzero");
}

Eigen::Vector3d ExtrudedGeometry::position(double u, double v, double w) const {
    return surf_->evaluate(u, v).position + w * dir_;
}

GeometryFrame ExtrudedGeometry::frameAt(double u, double v) const {
    const SurfacePoint s = surf_->evaluate(u, v);
    GeometryFrame f;
    f.df.col(0) = s.du;
    f.df.col(1) = s.dv;
    f.df.col(2) = dir_;
    f.det = f.df.determinant();
    if (f.det < 1e-14)
        throw std::domain_error("ExtrudedGeometry: degenerate or orientation-reversing Jacobian");
    f.df_inv_transpose = f.df.inverse().transpose();
    return f;
}

// ---- materials ------------------------------------------------------------------

OrthotropicConstants OrthotropicConstants::isotropic(double e, double nu) {
    OrthotropicConstants c;
    c.E1 = c.E2 = c.E3 = e;
    c.G12 = c.G13 = c.G23 = e / (2.0 * (1.0 + nu));
    c.nu12 = c.nu13 = c.nu23 = nu;
    return c;
}

namespace {
constexpr int kVI[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
constexpr int kVP[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};
} // namespace

ElasticityTensor ElasticityTensor::fromVoigt(const VoigtMatrix& d) {
    ElasticityTensor t;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l)
                    t(i, j, k, l) = d(kVI[i][j], kVI[k][l]);
    return t;
}

VoigtMatrix ElasticityTensor::toVoigt() const {
    VoigtMatrix d;
    for (int a = 0; a < 6; ++a)
        for (int b = 0; b < 6; ++b)
            d(a, b) = (*this)(kVP[a][0], kVP[a][1], kVP[b][0], kVP[b][1]);
    return d;
}

ElasticityTensor ElasticityTensor::rotated(const Eigen::Matrix3d& r) const {
    // two-index-at-a-time contraction: C'_ijkl = R_ia R_jb R_kc R_ld C_abcd
    ElasticityTensor a, b;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int c = 0; c < 3; ++c)
                for (int d = 0; d < 3; ++d) {
                    double s = 0.0;
                    for (int p = 0; p < 3; ++p)
                        for (int q = 0; q < 3; ++q)
                            s += r(i, p) * r(j, q) * (*this)(p, q, c, d);
                    a(i, j, c, d) = s;
                }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) {
                    double s = 0.0;
                    for (int p = 0; p < 3; ++p)
                        for (int q = 0; q < 3; ++q)
                            s += r(k, p) * r(l, q) * a(i, j, p, q);
                    b(i, j, k, l) = s;
                }
    return b;
}

double ElasticityTensor::quadraticForm(const Eigen::Matrix3d& eps) const {
    double s = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l)
                    s += eps(i, j) * (*this)(i, j, k, l) * eps(k, l);
    return s;
}

VoigtMatrix voigtFromConstants(const OrthotropicConstants& c) {
    const lf_orthotropic cc = toC(c);
    double d[36];
    ok(lf_voigt_from_constants(&cc, d));
    return fromRowMajor(d);
}

OrthotropicConstants constantsFromVoigt(const VoigtMatrix& d) {
    const VoigtMatrix s = d.inverse();
    OrthotropicConstants c;
    c.E1 = 1.0 / s(0, 0);
    c.E2 = 1.0 / s(1, 1);
    c.E3 = 1.0 / s(2, 2);
    c.nu12 = -s(0, 1) * c.E1;
    c.nu13 = -s(0, 2) * c.E1;
    c.nu23 = -s(1, 2) * c.E2;
    c.G12 = 1.0 / s(3, 3);
    c.G13 = 1.0 / s(4, 4);
    c.G23 = 1.0 / s(5, 5);
    return c;
}

VoigtMatrix rotateInplane(const VoigtMatrix& d, double theta) {
    double in[36], out[36];
    toRowMajor(d, in);
    ok(lf_rotate_inplane(in, theta, out));
    return fromRowMajor(out);
}

std::array<VoigtMatrix, 5> angleDecomposition(const OrthotropicConstants& c) {
    const lf_orthotropic cc = toC(c);
    double out[180];
    ok(lf_angle_decomposition(&cc, out));
    std::array<VoigtMatrix, 5> r;
    for (int k = 0; k < 5; ++k)
        r[static_cast<std::size_t>(k)] = fromRowMajor(out + 36 * k);
    return r;
}

Layup::Layup(std::vector<double> interfaces, const std::vector<LayerSpec>& layers) : z_(std::move(interfaces)) {
    if (layers.empty())
        throw std::invalid_argument("Layup: need at least one layer");
    if (z_.size() != layers.size() + 1)
        throw std::invalid_argument("Layup: need one more interface than layers");
    if (z_.front() != 0.0 || z_.back() != 1.0)
        throw std::invalid_argument("Layup: interfaces must run from 0 to 1");
    for (std::size_t i = 1; i < z_.size(); ++i)
        if (!(z_[i] > z_[i - 1]))
            throw std::invalid_argument("Layup: interfaces must be strictly increasing");
    for (const LayerSpec& spec : layers) {
        auto it = std::find_if(cfgs_.begin(), cfgs_.end(),
                               [&](const MaterialConfig& m) { return m.matches(spec.constants, spec.angle); });
        if (it == cfgs_.end()) {
            MaterialConfig m;
            m.constants = spec.constants;
            m.angle = spec.angle;
            m.id = static_cast<int>(cfgs_.size());
            m.stiffness = rotateInplane(voigtFromConstants(spec.constants), spec.angle);
            cfgs_.push_back(m);
            it = cfgs_.end() - 1;
        }
        cfg_of_layer_.push_back(it->id);
    }
}

Layup Layup::equalLayers(const std::vector<LayerSpec>& layers) {
    const int m = static_cast<int>(layers.size());
    std::vector<double> z;
    for (int l = 0; l <= m; ++l)
        z.push_back(static_cast<double>(l) / m);
    return Layup(std::move(z), layers);
}

int Layup::layerAt(double xi3) const {
    if (xi3 < 0.0 || xi3 > 1.0)
        throw std::domain_error("Layup: thickness coordinate outside [0,1]");
    const auto it = std::upper_bound(z_.begin(), z_.end(), xi3);
    return it == z_.end() ? numLayers() - 1 : static_cast<int>(it - z_.begin()) - 1;
}

// ---- sparse -------------------------------------------------------------------

SparseMatrixBuilder::SparseMatrixBuilder(int n_functions) : n_(n_functions) {
    if (n_functions < 1)
        throw std::invalid_argument("SparseMatrixBuilder: need at least one function");
}

void SparseMatrixBuilder::addBlock(int i, int j, const Eigen::Matrix3d& block) {
    if (i < 0 || j < 0 || i >= n_ || j >= n_)
        throw std::invalid_argument("SparseMatrixBuilder: block index out of range");
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
            entries_.push_back({3 * i + r, 3 * j + c, block(r, c)});
}

void SparseMatrixBuilder::merge(SparseMatrixBuilder&& other) {
    if (other.n_ != n_)
        throw std::invalid_argument("SparseMatrixBuilder: merging builders of different size");
    entries_.insert(entries_.end(), other.entries_.begin(), other.entries_.end());
    other.entries_.clear();
}

StiffnessMatrix SparseMatrixBuilder::finalize() const {
    if (entries_.empty())
        throw std::logic_error("SparseMatrixBuilder: nothing accumulated");
    std::vector<Triplet> t = entries_;
    std::stable_sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
        return a.row < b.row || (a.row == b.row && a.col < b.col);
    });
    StiffnessMatrix m;
    m.n_ = dim();
    m.ptr_.assign(static_cast<std::size_t>(dim()) + 1, 0);
    for (std::size_t k = 0; k < t.size();) {
        double sum = 0.0;
        const int r = t[k].row, c = t[k].col;
        for (; k < t.size() && t[k].row == r && t[k].col == c; ++k)
            sum += t[k].value;
        m.col_.push_back(c);
        m.val_.push_back(sum);
        m.ptr_[static_cast<std::size_t>(r) + 1]++;
    }
    for (std::size_t r = 0; r < static_cast<std::size_t>(dim()); ++r)
        m.ptr_[r + 1] += m.ptr_[r];
    return m;
}

StiffnessMatrix StiffnessMatrix::fromCsr(int dim, std::vector<std::int64_t> row_offsets, std::vector<int> cols,
                                         std::vector<double> values) {
    if (row_offsets.size() != static_cast<std::size_t>(dim) + 1 || cols.size() != values.size() ||
        static_cast<std::size_t>(row_offsets.back()) != values.size())
        throw std::invalid_argument("StiffnessMatrix::fromCsr: inconsistent arrays");
    StiffnessMatrix m;
    m.n_ = dim;
    m.ptr_ = std::move(row_offsets);
    m.col_ = std::move(cols);
    m.val_ = std::move(values);
    return m;
}

double StiffnessMatrix::at(int row, int col) const {
    const auto b = col_.begin() + ptr_[static_cast<std::size_t>(row)];
    const auto e = col_.begin() + ptr_[static_cast<std::size_t>(row) + 1];
    const auto it = std::lower_bound(b, e, col);
    return (it != e && *it == col) ? val_[static_cast<std::size_t>(it - col_.begin())] : 0.0;
}

double StiffnessMatrix::frobeniusNorm() const {
    double s = 0.0;
    for (double v : val_)
        s += v * v;
    return std::sqrt(s);
}

double StiffnessMatrix::symmetryRelError() const {
    double s = 0.0;
    for (int r = 0; r < n_; ++r)
        for (std::int64_t k = ptr_[static_cast<std::size_t>(r)]; k < ptr_[static_cast<std::size_t>(r) + 1]; ++k) {
            const int c = col_[static_cast<std::size_t>(k)];
            const auto b = col_.begin() + ptr_[static_cast<std::size_t>(c)];
            const auto e = col_.begin() + ptr_[static_cast<std::size_t>(c) + 1];
            const auto it = std::lower_bound(b, e, r);
            const bool has = it != e && *it == r;
            const double d = val_[static_cast<std::size_t>(k)] - (has ? val_[static_cast<std::size_t>(it - col_.begin())] : 0.0);
            s += has ? d * d : 2 * d * d; // an absent mirror slot differs too
        }
    const double n = frobeniusNorm();
    return n == 0.0 ? 0.0 : std::sqrt(s) / n;
}

Eigen::VectorXd StiffnessMatrix::apply(const Eigen::VectorXd& x) const {
    if (x.size() != n_)
        throw std::invalid_argument("StiffnessMatrix: vector length mismatch");
    Eigen::VectorXd y = Eigen::VectorXd::Zero(n_);
    for (int r = 0; r < n_; ++r) {
        double s = 0.0;
        for (std::int64_t k = ptr_[static_cast<std::size_t>(r)]; k < ptr_[static_cast<std::size_t>(r) + 1]; ++k)
            s += val_[static_cast<std::size_t>(k)] * x[col_[static_cast<std::size_t>(k)]];
        y[r] = s;
    }
    return y;
}

double frobeniusRelDiff(const StiffnessMatrix& a, const StiffnessMatrix& b) {
    if (a.dim() != b.dim())
        throw std::invalid_argument("frobeniusRelDiff: dimension mismatch");
    double s = 0.0;
    for (int r = 0; r < a.dim(); ++r) {
        std::int64_t i = a.rowOffsets()[static_cast<std::size_t>(r)], j = b.rowOffsets()[static_cast<std::size_t>(r)];
        const std::int64_t ie = a.rowOffsets()[static_cast<std::size_t>(r) + 1];
        const std::int64_t je = b.rowOffsets()[static_cast<std::size_t>(r) + 1];
        while (i < ie || j < je) {
            const int ca = i < ie ? a.colIndices()[static_cast<std::size_t>(i)] : a.dim();
            const int cb = j < je ? b.colIndices()[static_cast<std::size_t>(j)] : b.dim();
            const double d = ca == cb ? a.values()[static_cast<std::size_t>(i++)] - b.values()[static_cast<std::size_t>(j++)]
                             : ca < cb ? a.values()[static_cast<std::size_t>(i++)]
                                       : -b.values()[static_cast<std::size_t>(j++)];
            s += d * d;
        }
    }
    const double den = std::max(a.frobeniusNorm(), b.frobeniusNorm());
    return den == 0.0 ? 0.0 : std::sqrt(s) / den;
}

void writeMatrixMarket(const StiffnessMatrix& m, std::ostream& out) {
    out << "%%MatrixMarket matrix coordinate real general\n" << m.dim() << ' ' << m.dim() << ' ' << m.nnz() << '\n';
    out.precision(17);
    for (int r = 0; r < m.dim(); ++r)
        for (std::int64_t k = m.rowOffsets()[static_cast<std::size_t>(r)];
             k < m.rowOffsets()[static_cast<std::size_t>(r) + 1]; ++k)
            out << r + 1 << ' ' << m.colIndices()[static_cast<std::size_t>(k)] + 1 << ' '
                << m.values()[static_cast<std::size_t>(k)] << '\n';
}

// ---- in-plane operator storage ---------------------------------------------------------

InPlaneOperator::InPlaneOperator(int n_u, int n_v, int degree_u, int degree_v)
    : nu_(n_u), nv_(n_v), pu_(degree_u), pv_(degree_v) {
    const std::size_t n = static_cast<std::size_t>(n_u) * n_v * (2 * degree_u + 1) * (2 * degree_v + 1);
    blk_.assign(n, Eigen::Matrix3d::Zero());
    occ_.assign(n, 0);
}

std::size_t InPlaneOperator::slot(int is, int js) const {
    const int du = js % nu_ - is % nu_ + pu_, dv = js / nu_ - is / nu_ + pv_;
    return (static_cast<std::size_t>(is) * (2 * pv_ + 1) + static_cast<std::size_t>(dv)) * (2 * pu_ + 1) +
           static_cast<std::size_t>(du);
}

bool InPlaneOperator::inBand(int is, int js) const {
    return std::abs(is % nu_ - js % nu_) <= pu_ && std::abs(is / nu_ - js / nu_) <= pv_;
}

bool InPlaneOperator::occupied(int is, int js) const { return inBand(is, js) && occ_[slot(is, js)] != 0; }

std::vector<int> InPlaneOperator::bandColumns(int is) const {
    std::vector<int> out;
    const int iu = is % nu_, iv = is / nu_;
    for (int jv = std::max(0, iv - pv_); jv <= std::min(nv_ - 1, iv + pv_); ++jv)
        for (int ju = std::max(0, iu - pu_); ju <= std::min(nu_ - 1, iu + pu_); ++ju)
            out.push_back(jv * nu_ + ju);
    return out;
}

// ---- assembly entry points (GPU) -------------------------------------------------------

StiffnessMatrix assembleStandard(const ProblemSetup& setup, const AssemblyOptions& options, AssemblyStats* stats) {
    return assembleOnDevice(LF_BACKEND_STANDARD, setup, options, stats);
}

StiffnessMatrix assembleFast(const ProblemSetup& setup, const AssemblyOptions& options, AssemblyStats* stats) {
    return assembleOnDevice(LF_BACKEND_FAST, setup, options, stats);
}

StiffnessMatrix assembleVoigtFree(const ProblemSetup& setup, const AssemblyOptions& options, AssemblyStats* stats) {
    return assembleOnDevice(LF_BACKEND_VOIGT_FREE, setup, options, stats);
}

double referenceBilinear(const ProblemSetup& setup, const Eigen::VectorXd& v, const Eigen::VectorXd& u,
                         const AssemblyOptions& options) {
    // v' K u by full 3D quadrature on the device, without forming K (K8)
    const int n = 3 * setup.space.numFunctions();
    if (v.size() != n || u.size() != n)
        throw std::invalid_argument("referenceBilinear: coefficient length mismatch");
    if (setup.layup.numLayers() < 1)
        throw std::invalid_argument("referenceBilinear: empty layup");
    CProblem cp;
    fillSpace(cp, setup.space);
    fillGeometry(cp, setup.space, setup.geom, options);
    fillLayup(cp, setup.layup);
    fillOptions(cp, options);
    const std::vector<double> hv(v.data(), v.data() + n), hu(u.data(), u.data() + n);
    double out = 0.0;
    ok(lf_reference_bilinear(&cp.p, hv.data(), hu.data(), device(), &out));
    return out;
}

InPlaneOperatorSet computeInplaneOperators(const TensorProductSpace& space, const ExtrudedGeometry& geom,
                                           const VoigtMatrix& material, const AssemblyOptions& options,
                                           AssemblyStats* stats) {
    double d[36];
    toRowMajor(material, d);
    return inplaneOnDevice(space, geom, d, nullptr, options, stats);
}

ThicknessOperators computeThicknessOperators(const KnotVector& thickness, const std::vector<double>& interfaces,
                                             int pts_per_cell) {
    const int nt = thickness.numFunctions();
    const int L = static_cast<int>(interfaces.size()) - 1;
    if (L < 1)
        throw std::invalid_argument("layerwiseThicknessRule: interfaces must run from 0 to 1");
    std::vector<double> q(static_cast<std::size_t>(L) * 4 * nt * nt);
    std::vector<char> occ(static_cast<std::size_t>(nt) * nt);
    ok(lf_thickness_operators(thickness.degree(), static_cast<int32_t>(thickness.knots().size()),
                              thickness.knots().data(), static_cast<int32_t>(interfaces.size()), interfaces.data(),
                              pts_per_cell, device(), q.data(), occ.data()));
    ThicknessOperators out;
    out.per_layer.resize(static_cast<std::size_t>(L));
    for (int l = 0; l < L; ++l)
        for (int f = 0; f < 4; ++f) {
            Eigen::MatrixXd m(nt, nt);
            for (int i = 0; i < nt; ++i)
                for (int j = 0; j < nt; ++j)
                    m(i, j) = q[((static_cast<std::size_t>(l) * 4 + f) * nt + i) * nt + j];
            out.per_layer[static_cast<std::size_t>(l)][static_cast<std::size_t>(f)] = std::move(m);
        }
    out.occupied = Eigen::Matrix<char, Eigen::Dynamic, Eigen::Dynamic>::Zero(nt, nt);
    for (int i = 0; i < nt; ++i)
        for (int j = 0; j < nt; ++j)
            out.occupied(i, j) = occ[static_cast<std::size_t>(i) * nt + j];
    return out;
}

StiffnessMatrix combineOperators(const TensorProductSpace& space, const std::vector<OperatorTerm>& terms,
                                 const Eigen::Matrix<char, Eigen::Dynamic, Eigen::Dynamic>& thickness_occupied,
                                 const AssemblyOptions& options) {
    (void)options;
    if (terms.empty())
        throw std::invalid_argument("combineOperators: no operator terms");
    CProblem cp;
    fillSpace(cp, space);
    const int nu = space.numU(), nv = space.numV(), nt = space.numThickness();
    const int pu = space.inplaneU().degree(), pv = space.inplaneV().degree();
    const int bu = 2 * pu + 1, bv = 2 * pv + 1;
    const std::size_t per = static_cast<std::size_t>(nu) * nv * bu * bv;
    std::vector<double> blocks(terms.size() * 4 * per * 9, 0.0);
    std::vector<char> flags(per, 0);
    std::vector<double> th(terms.size() * 4 * static_cast<std::size_t>(nt) * nt);
    std::vector<char> occ(static_cast<std::size_t>(nt) * nt);
    for (int is = 0; is < nu * nv; ++is)
        for (int js : terms[0].inplane.op[0].bandColumns(is)) {
            const std::size_t slot =
                (static_cast<std::size_t>(is) * bv + (js / nu - is / nu + pv)) * bu + (js % nu - is % nu + pu);
            flags[slot] = terms[0].inplane.op[0].occupied(is, js) ? 1 : 0;
            for (std::size_t t = 0; t < terms.size(); ++t)
                for (int f = 0; f < 4; ++f) {
                    const Eigen::Matrix3d& b = terms[t].inplane.op[static_cast<std::size_t>(f)].block(is, js);
                    for (int r = 0; r < 3; ++r)
                        for (int c = 0; c < 3; ++c)
                            blocks[((t * 4 + f) * per + slot) * 9 + 3 * r + c] = b(r, c);
                }
        }
    for (std::size_t t = 0; t < terms.size(); ++t)
        for (int f = 0; f < 4; ++f)
            for (int i = 0; i < nt; ++i)
                for (int j = 0; j < nt; ++j)
                    th[((t * 4 + f) * nt + i) * nt + j] = terms[t].thickness[static_cast<std::size_t>(f)](i, j);
    for (int i = 0; i < nt; ++i)
        for (int j = 0; j < nt; ++j)
            occ[static_cast<std::size_t>(i) * nt + j] = thickness_occupied(i, j) ? 1 : 0;
    int64_t nnz = 0;
    const int32_t nterm = static_cast<int32_t>(terms.size());
    ok(lf_combine(&cp.p, nterm, blocks.data(), flags.data(), th.data(), occ.data(), device(), &nnz, nullptr, nullptr,
                  nullptr));
    const int dim = 3 * space.numFunctions();
    std::vector<std::int64_t> rp = csrArray<std::int64_t>(static_cast<std::size_t>(dim) + 1);
    std::vector<int> cols = csrArray<int>(static_cast<std::size_t>(nnz));
    std::vector<double> vals = csrArray<double>(static_cast<std::size_t>(nnz));
    ok(lf_combine(&cp.p, nterm, blocks.data(), flags.data(), th.data(), occ.data(), device(), &nnz, rp.data(),
                  cols.data(), vals.data()));
    return StiffnessMatrix::fromCsr(dim, std::move(rp), std::move(cols), std::move(vals));
}

BracketParameters bracketParameters(const OrthotropicConstants& constants) {
    const lf_orthotropic c = toC(constants);
    double out[9];
    ok(lf_bracket_parameters(&c, out));
    BracketParameters b;
    b.lambda = out[0];
    b.mu = out[1];
    for (int k = 0; k < 7; ++k)
        b.alpha[static_cast<std::size_t>(k)] = out[2 + k];
    return b;
}

Eigen::Matrix3d ContractionTable::isotropicEntry(double lambda, double mu, int i, int j) {
    Eigen::Matrix3d m = Eigen::Matrix3d::Zero();
    m(i, j) += lambda;
    m(j, i) += mu;
    if (i == j)
        for (int k = 0; k < 3; ++k)
            m(k, k) += mu;
    return m;
}

ContractionTable::ContractionTable(const BracketParameters& params, double angle) {
    double prm[9] = {params.lambda, params.mu};
    for (int k = 0; k < 7; ++k)
        prm[2 + k] = params.alpha[static_cast<std::size_t>(k)];
    double t[81];
    ok(lf_contraction_table(prm, angle, t));
    for (int e = 0; e < 9; ++e)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                tab_[static_cast<std::size_t>(e)](r, c) = t[9 * e + 3 * r + c];
}

std::array<Eigen::Matrix3d, 9> pullbackContractionTable(const ContractionTable& table, const GeometryFrame& frame) {
    std::array<Eigen::Matrix3d, 9> out;
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            Eigen::Matrix3d s = Eigen::Matrix3d::Zero();
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j)
                    s += table.entry(i, j) * (frame.df_inv_transpose(i, a) * frame.df_inv_transpose(j, b));
            out[static_cast<std::size_t>(3 * a + b)] = s;
        }
    return out;
}

InPlaneOperatorSet computeInplaneOperatorsBracket(const TensorProductSpace& space, const ExtrudedGeometry& geom,
                                                  const ContractionTable& table, const AssemblyOptions& options,
                                                  AssemblyStats* stats) {
    double t[81];
    for (int e = 0; e < 9; ++e)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                t[9 * e + 3 * r + c] = table.entry(e / 3, e % 3)(r, c);
    return inplaneOnDevice(space, geom, nullptr, t, options, stats);
}

std::string backendName(Backend b) {
    switch (b) {
    case Backend::Standard: return "standard";
    case Backend::Fast: return "fast";
    case Backend::VoigtFree: return "voigt_free";
    }
    throw std::logic_error("backendName: unknown backend");
}

Backend backendFromName(const std::string& name) {
    if (name == "standard")
        return Backend::Standard;
    if (name == "fast")
        return Backend::Fast;
    if (name == "voigt_free" || name == "voigt-free")
        return Backend::VoigtFree;
    throw std::invalid_argument("unknown backend '" + name + "'");
}

StiffnessMatrix assembleWith(Backend backend, const ProblemSetup& setup, const AssemblyOptions& options,
                             AssemblyStats* stats) {
    switch (backend) {
    case Backend::Standard: return assembleStandard(setup, options, stats);
    case Backend::Fast: return assembleFast(setup, options, stats);
    case Backend::VoigtFree: return assembleVoigtFree(setup, options, stats);
    }
    throw std::logic_error("assembleWith: unknown backend");
}

std::string layupFamilyName(LayupFamily family) {
    switch (family) {
    case LayupFamily::CrossPly: return "cross_ply_0_90";
    case LayupFamily::QuadPly: return "quad_ply_0_p45_m45_90";
    case LayupFamily::Custom: return "custom";
    }
    throw std::logic_error("layupFamilyName: unknown family");
}

LayupFamily layupFamilyFromName(const std::string& name) {
    static const std::pair<const char*, LayupFamily> names[] = {
        {"cross_ply_0_90", LayupFamily::CrossPly}, {"cross_ply", LayupFamily::CrossPly},
        {"quad_ply_0_p45_m45_90", LayupFamily::QuadPly}, {"quad_ply", LayupFamily::QuadPly},
        {"custom", LayupFamily::Custom}};
    for (const auto& [n, f] : names)
        if (name == n)
            return f;
    throw std::invalid_argument("unknown layup family '" + name + "'");
}

std::vector<double> familyAngles(LayupFamily family, int m) {
    if (m < 1)
        throw std::invalid_argument("familyAngles: need at least one layer");
    if (family == LayupFamily::Custom)
        throw std::invalid_argument("familyAngles: the custom family has no fixed angles");
    constexpr double pi = 3.14159265358979323846;
    const std::vector<double> cycle = family == LayupFamily::CrossPly
                                          ? std::vector<double>{0.0, 0.5 * pi}
                                          : std::vector<double>{0.0, 0.25 * pi, -0.25 * pi, 0.5 * pi};
    std::vector<double> angles(static_cast<std::size_t>(m));
    for (int l = 0; l < m; ++l)
        angles[static_cast<std::size_t>(l)] = cycle[static_cast<std::size_t>(l) % cycle.size()];
    return angles;
}

OrthotropicConstants paganoConstants() {
    OrthotropicConstants c;
    c.E1 = 25.0;
    c.E2 = c.E3 = 1.0;
    c.G12 = c.G13 = 0.2;
    c.G23 = 0.5;
    c.nu12 = c.nu13 = c.nu23 = 0.25;
    return c;
}

ProblemSetup paganoSetup(const std::vector<double>& angles, int degree, int elements_x, int elements_y,
                         int thickness_elements, const PlateDimensions& plate) {
    std::vector<LayerSpec> layers;
    for (const double a : angles)
        layers.push_back(LayerSpec{paganoConstants(), a});
    TensorProductSpace space(KnotVector::uniform(degree, elements_x), KnotVector::uniform(degree, elements_y),
                             KnotVector::uniform(degree, thickness_elements));
    ExtrudedGeometry geometry(std::make_shared<PlanarRectangle>(plate.lx, plate.ly),
                              Eigen::Vector3d(0.0, 0.0, plate.thickness));
    return ProblemSetup{std::move(space), std::move(geometry), Layup::equalLayers(layers)};
}

ProblemSetup paganoSetup(int m, LayupFamily family, int degree, int elements) {
    return paganoSetup(familyAngles(family, m), degree, elements, elements);
}

} // namespace lamfast
