// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// extern "C" shim around the UNMODIFIED reference sources
// (/root/reference/proj/src/{splines,quadrature,geometry,materials,assembly,
// fast,sparse,voigt_free}.cpp), compiled by oracle/build_ref.sh against the
// from-scratch Eigen subset into oracle/_ref/libref_lamfast.so.  Python tests
// use it to pin the C restatement (oracle/lamfast_oracle.c) and the GPU path
// against the reference's own output, and bench.py --impl reference times it.
// The problem descriptor is the product's lf_problem (include/lamfast_cuda.h)
// so every checker consumes byte-identical inputs.

#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lamfast/assembly.hpp"
#include "lamfast/fast.hpp"
#include "lamfast/geometry.hpp"
#include "lamfast/materials.hpp"
#include "lamfast/quadrature.hpp"
#include "lamfast/sparse.hpp"
#include "lamfast/splines.hpp"
#include "lamfast/voigt_free.hpp"
#include "lamfast_cuda.h"

using namespace lamfast;

namespace {

thread_local std::string g_error;

int fail(int code, const char* what) {
    g_error = what;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LF_OK;
    } catch (const std::invalid_argument& e) {
        return fail(LF_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::domain_error& e) {
        return fail(LF_ERR_DOMAIN, e.what());
    } catch (const std::logic_error& e) {
        return fail(LF_ERR_LOGIC, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(LF_ERR_OUT_OF_MEMORY, e.what());
    } catch (const std::exception& e) {
        return fail(LF_ERR_RUNTIME, e.what());
    }
}

KnotVector knots(int degree, int n, const double* k) {
    return KnotVector(degree, std::vector<double>(k, k + n));
}

OrthotropicConstants constants(const lf_orthotropic& c) {
    OrthotropicConstants o;
    o.E1 = c.E1;
    o.E2 = c.E2;
    o.E3 = c.E3;
    o.G12 = c.G12;
    o.G13 = c.G13;
    o.G23 = c.G23;
    o.nu12 = c.nu12;
    o.nu13 = c.nu13;
    o.nu23 = c.nu23;
    return o;
}

ExtrudedGeometry geometry(const lf_problem& p) {
    const Eigen::Vector3d dir(p.direction[0], p.direction[1], p.direction[2]);
    const double* g = p.geometry;
    if (p.geometry_kind == LF_GEOM_PLANAR)
        return ExtrudedGeometry(std::make_shared<PlanarRectangle>(g[0], g[1]), dir);
    if (p.geometry_kind == LF_GEOM_BILINEAR)
        return ExtrudedGeometry(
            std::make_shared<BilinearQuad>(Eigen::Vector3d(g[0], g[1], g[2]),
                                           Eigen::Vector3d(g[3], g[4], g[5]),
                                           Eigen::Vector3d(g[6], g[7], g[8]),
                                           Eigen::Vector3d(g[9], g[10], g[11])),
            dir);
    throw std::invalid_argument("ref_capi: only planar and bilinear geometry are wired");
}

TensorProductSpace space(const lf_problem& p) {
    return TensorProductSpace(knots(p.degree_u, p.n_knots_u, p.knots_u),
                              knots(p.degree_v, p.n_knots_v, p.knots_v),
                              knots(p.degree_t, p.n_knots_t, p.knots_t));
}

ProblemSetup setup(const lf_problem& p) {
    std::vector<LayerSpec> layers;
    for (int l = 0; l < p.n_layers; ++l)
        layers.push_back({constants(p.layers[l].constants), p.layers[l].angle});
    std::vector<double> interfaces(p.interfaces, p.interfaces + p.n_layers + 1);
    return ProblemSetup{space(p), geometry(p), Layup(std::move(interfaces), layers)};
}

AssemblyOptions options(const lf_problem& p, int threads) {
    AssemblyOptions o;
    o.threads = threads;
    o.inplane_points = p.inplane_points;
    o.thickness_points = p.thickness_points;
    for (int k = 0; k < p.n_active_layers; ++k)
        o.active_layers.push_back(p.active_layers[k]);
    o.decompose_angles = p.decompose_angles != 0;
    return o;
}

VoigtMatrix voigt(const double* d) {
    VoigtMatrix m;
    for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c)
            m(r, c) = d[6 * r + c];
    return m;
}

void exportOperators(const InPlaneOperatorSet& set, const TensorProductSpace& sp, double* blocks,
                     char* flags) {
    const int nu = sp.numU(), n_s = sp.numInplane();
    const int pu = sp.inplaneU().degree(), pv = sp.inplaneV().degree();
    const int bu = 2 * pu + 1, bv = 2 * pv + 1;
    const std::size_t per = static_cast<std::size_t>(n_s) * bv * bu;
    std::memset(flags, 0, per);
    std::memset(blocks, 0, 4 * per * 9 * sizeof(double));
    for (int is = 0; is < n_s; ++is) {
        const int iu = is % nu, iv = is / nu;
        for (int js : set.op[0].bandColumns(is)) {
            const int ju = js % nu, jv = js / nu;
            const std::size_t slot =
                (static_cast<std::size_t>(is) * bv + (jv - iv + pv)) * bu + (ju - iu + pu);
            flags[slot] = set.op[0].occupied(is, js) ? 1 : 0;
            for (int f = 0; f < 4; ++f) {
                const Eigen::Matrix3d& b = set.op[f].block(is, js);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c)
                        blocks[(f * per + slot) * 9 + 3 * r + c] = b(r, c);
            }
        }
    }
}

} // namespace

extern "C" {

struct ref_csr {
    int64_t dim;
    int64_t nnz;
    int64_t* row_ptr;
    int32_t* cols;
    double* values;
};

const char* ref_last_error(void) { return g_error.c_str(); }

void ref_csr_free(ref_csr* m) {
    std::free(m->row_ptr);
    std::free(m->cols);
    std::free(m->values);
    m->row_ptr = nullptr;
    m->cols = nullptr;
    m->values = nullptr;
}

static void exportMatrix(const StiffnessMatrix& k, ref_csr* out) {
    out->dim = k.dim();
    out->nnz = k.nnz();
    out->row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (out->dim + 1)));
    out->cols = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (out->nnz + 1)));
    out->values = static_cast<double*>(std::malloc(sizeof(double) * (out->nnz + 1)));
    std::memcpy(out->row_ptr, k.rowOffsets().data(), sizeof(int64_t) * (out->dim + 1));
    std::memcpy(out->cols, k.colIndices().data(), sizeof(int32_t) * out->nnz);
    std::memcpy(out->values, k.values().data(), sizeof(double) * out->nnz);
}

/// assembleWith(backend, setup, options, stats) (bench.cpp:53-61).
int ref_assemble(const lf_problem* p, int backend, int threads, ref_csr* out, lf_stats* stats) {
    return guarded([&] {
        const ProblemSetup s = setup(*p);
        const AssemblyOptions o = options(*p, threads);
        AssemblyStats st;
        StiffnessMatrix k;
        if (backend == LF_BACKEND_STANDARD)
            k = assembleStandard(s, o, &st);
        else if (backend == LF_BACKEND_FAST)
            k = assembleFast(s, o, &st);
        else if (backend == LF_BACKEND_VOIGT_FREE)
            k = assembleVoigtFree(s, o, &st);
        else
            throw std::invalid_argument("unknown backend");
        exportMatrix(k, out);
        if (stats) {
            stats->qpoint_visits += st.qpoint_visits;
            stats->frame_evaluations += st.frame_evaluations;
            stats->operator_builds += st.operator_builds;
        }
    });
}

/// KnotVector::evaluate (splines.cpp:53-101).
int ref_basis_eval(int degree, int n_knots, const double* k, double x, int* first, double* vals,
                   double* ders) {
    return guarded([&] {
        const BasisEval1D e = knots(degree, n_knots, k).evaluate(x);
        *first = e.first_active;
        for (int r = 0; r <= degree; ++r) {
            vals[r] = e.values[static_cast<std::size_t>(r)];
            ders[r] = e.derivs[static_cast<std::size_t>(r)];
        }
    });
}

/// gaussLegendre(n, a, b) (quadrature.cpp:48-57).
int ref_gauss(int n, double a, double b, double* pts, double* wts) {
    return guarded([&] {
        const QuadratureRule r = gaussLegendre(n, a, b);
        for (int i = 0; i < n; ++i) {
            pts[i] = r.points[static_cast<std::size_t>(i)];
            wts[i] = r.weights[static_cast<std::size_t>(i)];
        }
    });
}

/// rotateInplane(voigtFromConstants(c), angle) (materials.cpp:73-117).
int ref_stiffness(const lf_orthotropic* c, double angle, double out[36]) {
    return guarded([&] {
        const VoigtMatrix d = rotateInplane(voigtFromConstants(constants(*c)), angle);
        for (int r = 0; r < 6; ++r)
            for (int q = 0; q < 6; ++q)
                out[6 * r + q] = d(r, q);
    });
}

/// angleDecomposition (materials.cpp:119-149).
int ref_angle_decomposition(const lf_orthotropic* c, double out[180]) {
    return guarded([&] {
        const auto basis = angleDecomposition(constants(*c));
        for (int k = 0; k < 5; ++k)
            for (int r = 0; r < 6; ++r)
                for (int q = 0; q < 6; ++q)
                    out[36 * k + 6 * r + q] = basis[static_cast<std::size_t>(k)](r, q);
    });
}

/// bracketParameters (voigt_free.cpp:52-80): lambda, mu, alpha[7].
int ref_bracket_parameters(const lf_orthotropic* c, double out[9]) {
    return guarded([&] {
        const BracketParameters b = bracketParameters(constants(*c));
        out[0] = b.lambda;
        out[1] = b.mu;
        for (int k = 0; k < 7; ++k)
            out[2 + k] = b.alpha[static_cast<std::size_t>(k)];
    });
}

/// ContractionTable(params(c), angle) entries (voigt_free.cpp:89-123).
int ref_contraction_table(const lf_orthotropic* c, double angle, double out[81]) {
    return guarded([&] {
        const ContractionTable t(bracketParameters(constants(*c)), angle);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                for (int r = 0; r < 3; ++r)
                    for (int q = 0; q < 3; ++q)
                        out[(3 * i + j) * 9 + 3 * r + q] = t.entry(i, j)(r, q);
    });
}

/// computeThicknessOperators (fast.cpp:170-209): q[layer][4][n_t][n_t].
int ref_thickness_operators(int degree, int n_knots, const double* k, int n_interfaces,
                            const double* interfaces, int pts, double* q, char* occupied) {
    return guarded([&] {
        const KnotVector kt = knots(degree, n_knots, k);
        const ThicknessOperators t = computeThicknessOperators(
            kt, std::vector<double>(interfaces, interfaces + n_interfaces), pts);
        const int n = kt.numFunctions();
        for (std::size_t l = 0; l < t.per_layer.size(); ++l)
            for (int f = 0; f < 4; ++f)
                for (int i = 0; i < n; ++i)
                    for (int j = 0; j < n; ++j)
                        q[((l * 4 + f) * n + i) * n + j] = t.per_layer[l][f](i, j);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                occupied[i * n + j] = t.occupied(i, j);
    });
}

/// computeInplaneOperators (fast.cpp:54-168) in the banded export layout.
int ref_inplane_operators(const lf_problem* p, const double material[36], double* blocks,
                          char* flags, lf_stats* stats) {
    return guarded([&] {
        const TensorProductSpace sp = space(*p);
        AssemblyStats st;
        const InPlaneOperatorSet set =
            computeInplaneOperators(sp, geometry(*p), voigt(material), options(*p, 1), &st);
        exportOperators(set, sp, blocks, flags);
        if (stats) {
            stats->qpoint_visits += st.qpoint_visits;
            stats->frame_evaluations += st.frame_evaluations;
            stats->operator_builds += st.operator_builds;
        }
    });
}

/// computeInplaneOperatorsBracket (voigt_free.cpp:142-248).
int ref_inplane_operators_bracket(const lf_problem* p, const lf_orthotropic* c, double angle,
                                  double* blocks, char* flags) {
    return guarded([&] {
        const TensorProductSpace sp = space(*p);
        const ContractionTable table(bracketParameters(constants(*c)), angle);
        const InPlaneOperatorSet set =
            computeInplaneOperatorsBracket(sp, geometry(*p), table, options(*p, 1), nullptr);
        exportOperators(set, sp, blocks, flags);
    });
}

/// ExtrudedGeometry::frameAt (geometry.cpp:74-85): df, dfit (col-major), det.
int ref_frame_at(const lf_problem* p, double u, double v, double out[19]) {
    return guarded([&] {
        const GeometryFrame f = geometry(*p).frameAt(u, v);
        for (int c = 0; c < 3; ++c)
            for (int r = 0; r < 3; ++r) {
                out[3 * c + r] = f.df(r, c);
                out[9 + 3 * c + r] = f.df_inv_transpose(r, c);
            }
        out[18] = f.det;
    });
}

/// referenceBilinear (assembly.cpp:247-318).
int ref_bilinear(const lf_problem* p, const double* v, const double* u, int64_t n, double* out) {
    return guarded([&] {
        Eigen::VectorXd ev(n), eu(n);
        for (int64_t k = 0; k < n; ++k) {
            ev[k] = v[k];
            eu[k] = u[k];
        }
        *out = referenceBilinear(setup(*p), ev, eu, options(*p, 1));
    });
}

} // extern "C"
