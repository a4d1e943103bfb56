// Drop-in check: code written against the reference's lamfast C++ API,
// compiled against include/lamfast (B200 edition) and linked with
// liblamfast.so.  Cases follow the reference tests (file:line given per
// case).  `--host-only` runs the cases that need no GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "lamfast/assembly.hpp"
#include "lamfast/bench.hpp"
#include "lamfast/fast.hpp"
#include "lamfast/geometry.hpp"
#include "lamfast/materials.hpp"
#include "lamfast/quadrature.hpp"
#include "lamfast/sparse.hpp"
#include "lamfast/splines.hpp"
#include "lamfast/voigt_free.hpp"

using namespace lamfast;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                 \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(cond)) {                                                              \
            ++g_fail;                                                               \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
        }                                                                           \
    } while (0)

static OrthotropicConstants pagano() {
    OrthotropicConstants c;
    c.E1 = 25.0;
    c.E2 = c.E3 = 1.0;
    c.G12 = c.G13 = 0.2;
    c.G23 = 0.5;
    c.nu12 = c.nu13 = c.nu23 = 0.25;
    return c;
}

static Layup paganoLayup(const std::vector<double>& angles) {
    std::vector<LayerSpec> layers;
    for (double a : angles)
        layers.push_back({pagano(), a});
    return Layup::equalLayers(layers);
}

static TensorProductSpace cube(int p, int e, int et) {
    return TensorProductSpace(KnotVector::uniform(p, e), KnotVector::uniform(p, e), KnotVector::uniform(p, et));
}

static ExtrudedGeometry flat(double lx, double ly, double h) {
    return ExtrudedGeometry(std::make_shared<PlanarRectangle>(lx, ly), Eigen::Vector3d(0, 0, h));
}

static ExtrudedGeometry skewed() {
    return ExtrudedGeometry(std::make_shared<BilinearQuad>(Eigen::Vector3d(0, 0, 0), Eigen::Vector3d(1.2, 0.1, 0.05),
                                                           Eigen::Vector3d(-0.1, 0.9, -0.02),
                                                           Eigen::Vector3d(1.0, 1.1, 0.08)),
                            Eigen::Vector3d(0.03, -0.02, 0.2));
}

/// A user SurfaceMap the device cannot evaluate: the drop-in ships its
/// frames as a host table.  Same map as the skewed BilinearQuad.
class UserQuad : public SurfaceMap {
public:
    SurfacePoint evaluate(double u, double v) const override { return inner_.evaluate(u, v); }

private:
    BilinearQuad inner_{Eigen::Vector3d(0, 0, 0), Eigen::Vector3d(1.2, 0.1, 0.05), Eigen::Vector3d(-0.1, 0.9, -0.02),
                        Eigen::Vector3d(1.0, 1.1, 0.08)};
};

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void hostOnly() {
    // test_splines.cpp:64-84
    KnotVector kv(3, {0, 0, 0, 0, 0.5, 1, 1, 1, 1});
    const BasisEval1D e = kv.evaluate(0.3);
    CHECK(e.first_active == 0);
    CHECK(std::abs(e.values[1] - 0.55799999999999994) <= 1e-14);
    CHECK(std::abs(e.derivs[2] - 1.4399999999999997) <= 1e-13);
    CHECK(throws<std::domain_error>([&] { kv.evaluate(1.5); }));
    CHECK(throws<std::invalid_argument>([] { KnotVector(2, {0, 0, 1, 1}); }));
    CHECK(kv.findSpan(1.0) == 4);
    // test_quadrature.cpp: exactness
    const QuadratureRule r = gaussLegendre(4, 0.0, 2.0);
    double s = 0.0;
    for (int i = 0; i < r.size(); ++i)
        s += r.weights[static_cast<std::size_t>(i)] * std::pow(r.points[static_cast<std::size_t>(i)], 7);
    CHECK(std::abs(s - 32.0) <= 1e-12);
    CHECK(layerwiseThicknessRule(KnotVector::uniform(2, 2), {0.0, 0.3, 1.0}, 3).size() == 3);
    // test_materials.cpp:44-63
    const VoigtMatrix d = voigtFromConstants(pagano());
    CHECK(std::abs(d(0, 0) - 25.16778523489933) <= 1e-12);
    CHECK(std::abs(d(5, 5) - 0.5) <= 1e-14);
    const OrthotropicConstants back = constantsFromVoigt(d);
    CHECK(std::abs(back.E1 - 25.0) <= 1e-11);
    const VoigtMatrix d90 = rotateInplane(d, 1.5707963267948966);
    CHECK(std::abs(d90(1, 1) - d(0, 0)) <= 1e-12);
    const auto basis = angleDecomposition(pagano());
    const double th = 0.37, c = std::cos(th), sn = std::sin(th);
    const VoigtMatrix rec = basis[0] + c * c * c * c * basis[1] + c * c * c * sn * basis[2] + c * c * basis[3] +
                            c * sn * basis[4];
    CHECK((rec - rotateInplane(d, th)).norm() <= 1e-10);
    const ElasticityTensor t = ElasticityTensor::fromVoigt(d);
    CHECK((t.rotated(Eigen::Matrix3d::Identity()).toVoigt() - d).norm() <= 1e-13);
    // test_materials.cpp:170-224
    const Layup lay = paganoLayup({0.0, 1.5707963267948966, 0.0, 1.5707963267948966});
    CHECK(lay.numDistinctConfigs() == 2);
    CHECK(lay.layerAt(0.25) == 1 && lay.layerAt(1.0) == 3);
    CHECK(throws<std::invalid_argument>([] { Layup({0.0, 0.5}, {LayerSpec{}}); }));
    // test_voigt_free.cpp:77-88
    const BracketParameters b = bracketParameters(pagano());
    CHECK(std::abs(b.lambda - 0.07114093959731704) <= 1e-12);
    CHECK(std::abs(b.alpha[0] - 24.767785234899335) <= 1e-10);
    const Eigen::Matrix3d e11 = ContractionTable::isotropicEntry(0.0, 0.5, 0, 0);
    CHECK(std::abs(e11(0, 0) - 1.0) <= 1e-15 && std::abs(e11(1, 1) - 0.5) <= 1e-15);
    // test_sparse.cpp: builder sums duplicates, symmetry, SpMV
    SparseMatrixBuilder sb(2);
    Eigen::Matrix3d blk = Eigen::Matrix3d::Identity();
    sb.addBlock(0, 1, blk);
    sb.addBlock(0, 1, blk);
    sb.addBlock(1, 0, 2.0 * blk);
    const StiffnessMatrix m = sb.finalize();
    CHECK(m.nnz() == 18 && m.at(0, 3) == 2.0 && m.at(0, 4) == 0.0);
    CHECK(m.symmetryRelError() <= 1e-15);
    Eigen::VectorXd x = Eigen::VectorXd::Zero(6);
    x[3] = 1.0;
    CHECK(m.apply(x)[0] == 2.0);
    CHECK(frobeniusRelDiff(m, m) == 0.0);
    std::ostringstream mm;
    writeMatrixMarket(m, mm);
    CHECK(mm.str().rfind("%%MatrixMarket", 0) == 0);
    CHECK(throws<std::logic_error>([] { SparseMatrixBuilder(3).finalize(); }));
    CHECK(backendFromName("voigt-free") == Backend::VoigtFree && backendName(Backend::Fast) == "fast");
    // problem builders (bench.hpp:22-46)
    const auto quad = familyAngles(LayupFamily::QuadPly, 5);
    CHECK(quad.size() == 5 && quad[1] == 0.25 * 3.14159265358979323846 && quad[2] == -quad[1] && quad[4] == 0.0);
    CHECK(familyAngles(LayupFamily::CrossPly, 3)[1] == 0.5 * 3.14159265358979323846);
    CHECK(throws<std::invalid_argument>([] { familyAngles(LayupFamily::Custom, 2); }));
    CHECK(throws<std::invalid_argument>([] { familyAngles(LayupFamily::CrossPly, 0); }));
    CHECK(layupFamilyFromName(layupFamilyName(LayupFamily::QuadPly)) == LayupFamily::QuadPly &&
          layupFamilyFromName("cross_ply") == LayupFamily::CrossPly);
    CHECK(throws<std::invalid_argument>([] { layupFamilyFromName("angle_ply"); }));
    CHECK(paganoConstants().E1 == 25.0 && paganoConstants().G23 == 0.5 && paganoConstants().G12 == 0.2);
    const ProblemSetup ps = paganoSetup(4, LayupFamily::CrossPly, 2, 3);
    CHECK(ps.space.numU() == 5 && ps.space.numV() == 5 && ps.layup.numDistinctConfigs() == 2);
}

static StiffnessMatrix hexOracle(double E, double nu) {
    // test_assembly.cpp:73-125: trilinear brick, built through the builder
    const double lam = E * nu / ((1 + nu) * (1 - 2 * nu)), mu = E / (2 * (1 + nu));
    Eigen::Matrix<double, 6, 6> D = Eigen::Matrix<double, 6, 6>::Zero();
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j)
            D(i, j) = lam;
        D(i, i) = lam + 2 * mu;
        D(3 + i, 3 + i) = mu;
    }
    const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};
    auto hv = [](int w, double t) { return w == 0 ? 1.0 - t : t; };
    auto hd = [](int w) { return w == 0 ? -1.0 : 1.0; };
    SparseMatrixBuilder sb(8);
    for (double x : gp)
        for (double y : gp)
            for (double z : gp) {
                std::vector<Eigen::Matrix<double, 6, 3>> B(8);
                for (int n = 0; n < 8; ++n) {
                    const int ix = n % 2, iy = (n / 2) % 2, iz = n / 4;
                    const double g[3] = {hd(ix) * hv(iy, y) * hv(iz, z), hv(ix, x) * hd(iy) * hv(iz, z),
                                         hv(ix, x) * hv(iy, y) * hd(iz)};
                    Eigen::Matrix<double, 6, 3> b = Eigen::Matrix<double, 6, 3>::Zero();
                    b(0, 0) = g[0], b(1, 1) = g[1], b(2, 2) = g[2];
                    b(3, 0) = g[1], b(3, 1) = g[0], b(4, 0) = g[2], b(4, 2) = g[0], b(5, 1) = g[2], b(5, 2) = g[1];
                    B[static_cast<std::size_t>(n)] = b;
                }
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j)
                        sb.addBlock(i, j, 0.125 * (B[static_cast<std::size_t>(i)].transpose() * D *
                                                   B[static_cast<std::size_t>(j)]));
            }
    return sb.finalize();
}

static void gpuCases() {
    // test_assembly.cpp:129-141 + acceptance.cpp:249-303: hexahedron, all backends
    {
        ProblemSetup s{cube(1, 1, 1), flat(1, 1, 1), Layup::equalLayers({{OrthotropicConstants::isotropic(1.0, 0.3), 0.0}})};
        const StiffnessMatrix oracle = hexOracle(1.0, 0.3);
        for (Backend b : {Backend::Standard, Backend::Fast, Backend::VoigtFree})
            CHECK(frobeniusRelDiff(assembleWith(b, s), oracle) <= 1e-13);
    }
    // test_fast.cpp:310-333
    const std::vector<std::vector<double>> layups = {
        {0.0}, {0.0, 1.5707963267948966, 0.0}, {0.0, 0.7853981633974483, -0.7853981633974483, 1.5707963267948966}};
    for (int k = 0; k < 3; ++k) {
        ProblemSetup s{cube(k + 1, k == 0 ? 1 : 2, 1), k == 1 ? skewed() : flat(1, 1, 0.1), paganoLayup(layups[k])};
        const StiffnessMatrix st = assembleStandard(s), fa = assembleFast(s), vf = assembleVoigtFree(s);
        CHECK(fa.nnz() == st.nnz());
        CHECK(frobeniusRelDiff(fa, st) <= 1e-12);
        CHECK(frobeniusRelDiff(vf, st) <= 1e-12);
        CHECK(fa.symmetryRelError() <= 1e-13);
        // acceptance.cpp:95-104: rigid translations are annihilated
        for (int dir = 0; dir < 3; ++dir) {
            Eigen::VectorXd u = Eigen::VectorXd::Zero(fa.dim());
            for (int f = 0; f < s.space.numFunctions(); ++f)
                u[3 * f + dir] = 1.0;
            CHECK(fa.apply(u).lpNorm<Eigen::Infinity>() / fa.frobeniusNorm() <= 1e-12);
        }
    }
    // user SurfaceMap (host frame table) == BilinearQuad (device frames)
    {
        ProblemSetup a{cube(2, 2, 1), skewed(), paganoLayup({0.0, 0.9})};
        ProblemSetup u{cube(2, 2, 1), ExtrudedGeometry(std::make_shared<UserQuad>(), Eigen::Vector3d(0.03, -0.02, 0.2)),
                       paganoLayup({0.0, 0.9})};
        CHECK(frobeniusRelDiff(assembleFast(a), assembleFast(u)) <= 1e-15);
        CHECK(frobeniusRelDiff(assembleStandard(a), assembleStandard(u)) <= 1e-15);
    }
    // SplineSurface (curved shell) through the frame table: fast == standard
    {
        const KnotVector ku = KnotVector::uniform(2, 2), kv = KnotVector::uniform(2, 2);
        std::vector<Eigen::Vector3d> net;
        for (int j = 0; j < kv.numFunctions(); ++j)
            for (int i = 0; i < ku.numFunctions(); ++i)
                net.emplace_back(0.3 * i, 0.3 * j, 0.05 * std::sin(1.0 * i + 0.5 * j));
        ProblemSetup s{cube(2, 2, 1), ExtrudedGeometry(std::make_shared<SplineSurface>(ku, kv, net),
                                                       Eigen::Vector3d(0, 0, 0.1)),
                       paganoLayup({0.0, 0.6, 1.2})};
        CHECK(frobeniusRelDiff(assembleFast(s), assembleStandard(s)) <= 1e-12);
    }
    // arrays past the drop-in's large-array threshold (std::vectors sized without a
    // zero fill, filled by the assembly's host threads): every element is written
    {
        ProblemSetup s{TensorProductSpace(KnotVector::uniform(2, 24), KnotVector::uniform(2, 24),
                                          KnotVector::uniform(2, 8)),
                       flat(1.0, 1.0, 0.1), paganoLayup({0.0, 1.5707963267948966, 0.7, -0.7, 0.0, 0.3, 1.2, 0.0})};
        const StiffnessMatrix fa = assembleFast(s), st = assembleStandard(s);
        CHECK(fa.nnz() > (std::int64_t(8) << 20) / 4); // the column array alone is past 8 MB
        CHECK(fa.rowOffsets().size() == static_cast<std::size_t>(fa.dim()) + 1);
        CHECK(fa.rowOffsets().back() == fa.nnz());
        CHECK(fa.colIndices().size() == static_cast<std::size_t>(fa.nnz()));
        CHECK(fa.values().size() == static_cast<std::size_t>(fa.nnz()));
        CHECK(frobeniusRelDiff(fa, st) <= 1e-12);
        CHECK(fa.symmetryRelError() <= 1e-12);
    }
    // test_fast.cpp:335-352 work accounting
    {
        std::vector<double> angles;
        for (int l = 0; l < 32; ++l)
            angles.push_back(l % 2 == 0 ? 0.0 : 1.5707963267948966);
        ProblemSetup s{cube(3, 2, 1), flat(1, 1, 0.1), paganoLayup(angles)};
        AssemblyStats fs, ss;
        (void)assembleFast(s, {}, &fs);
        (void)assembleStandard(s, {}, &ss);
        CHECK(fs.operator_builds == 2 && fs.qpoint_visits == 2 * 4 * 16);
        CHECK(ss.qpoint_visits == 32 * 4 * 16 * 4);
    }
    // test_fast.cpp:390-425 angle decomposition
    {
        std::mt19937 rng(99u);
        std::uniform_real_distribution<double> dist(-1.6, 1.6);
        std::vector<double> angles;
        for (int l = 0; l < 9; ++l)
            angles.push_back(dist(rng));
        ProblemSetup s{cube(2, 2, 1), skewed(), paganoLayup(angles)};
        AssemblyStats a, b;
        const StiffnessMatrix direct = assembleFast(s, {}, &a);
        AssemblyOptions o;
        o.decompose_angles = true;
        const StiffnessMatrix dec = assembleFast(s, o, &b);
        CHECK(a.operator_builds == 9 && b.operator_builds == 5);
        CHECK(frobeniusRelDiff(dec, direct) <= 1e-12);
    }
    // test_fast.cpp:268-276, 291-308: operators
    {
        const InPlaneOperatorSet set = computeInplaneOperators(cube(1, 1, 1), flat(1, 1, 1),
                                                               voigtFromConstants(OrthotropicConstants::isotropic(1.0, 0.0)));
        CHECK((set.op[3].block(0, 0) - Eigen::Vector3d(1.0 / 18, 1.0 / 18, 1.0 / 9).asDiagonal()).cwiseAbs().maxCoeff() <= 1e-15);
        const InPlaneOperatorSet sk = computeInplaneOperators(cube(2, 2, 1), skewed(), rotateInplane(voigtFromConstants(pagano()), 1.1));
        double worst = 0.0;
        for (int is = 0; is < 16; ++is)
            for (int js : sk.op[1].bandColumns(is))
                if (sk.op[1].occupied(is, js))
                    worst = std::max(worst, (sk.op[1].block(is, js) - sk.op[2].block(js, is).transpose()).cwiseAbs().maxCoeff());
        CHECK(worst <= 1e-14);
        // bracket P == strain P (test_voigt_free.cpp:186-212)
        const InPlaneOperatorSet br =
            computeInplaneOperatorsBracket(cube(2, 2, 1), skewed(), ContractionTable(bracketParameters(pagano()), 1.1));
        double d = 0.0, sc = 0.0;
        for (int f = 0; f < 4; ++f)
            for (int is = 0; is < 16; ++is)
                for (int js : br.op[f].bandColumns(is))
                    if (br.op[f].occupied(is, js)) {
                        d = std::max(d, (br.op[f].block(is, js) - sk.op[f].block(is, js)).cwiseAbs().maxCoeff());
                        sc = std::max(sc, sk.op[f].block(is, js).cwiseAbs().maxCoeff());
                    }
        CHECK(d <= 25e-13 * sc);
    }
    // test_fast.cpp:171-188, 354-375: thickness operators and the long form
    {
        const ThicknessOperators q = computeThicknessOperators(KnotVector::uniform(1, 1), {0.0, 1.0}, 2);
        CHECK(std::abs(q.per_layer[0][0](0, 1) - 1.0 / 6) <= 1e-15 && std::abs(q.per_layer[0][3](0, 1) + 1.0) <= 1e-15);
        ProblemSetup s{cube(2, 2, 2), flat(1.3, 0.8, 0.2), paganoLayup({0.0, 1.5707963267948966, 1.5707963267948966, 0.0})};
        const StiffnessMatrix reduced = assembleFast(s);
        const ThicknessOperators tq = computeThicknessOperators(s.space.thickness(), s.layup.interfaces(), 3);
        std::vector<InPlaneOperatorSet> per;
        for (const MaterialConfig& cfg : s.layup.distinctConfigs())
            per.push_back(computeInplaneOperators(s.space, s.geom, cfg.stiffness));
        std::vector<OperatorTerm> terms;
        for (int l = 0; l < s.layup.numLayers(); ++l)
            terms.push_back({per[static_cast<std::size_t>(s.layup.configIndexOf(l))], tq.per_layer[static_cast<std::size_t>(l)]});
        const StiffnessMatrix lf = combineOperators(s.space, terms, tq.occupied);
        CHECK(lf.nnz() == reduced.nnz() && frobeniusRelDiff(lf, reduced) <= 1e-14);
    }
    // referenceBilinear == v' K u  (test_assembly.cpp:200-212)
    {
        ProblemSetup s{cube(2, 2, 1), skewed(), paganoLayup({0.0, 0.7})};
        const StiffnessMatrix k = assembleFast(s);
        std::mt19937 rng(5u);
        std::uniform_real_distribution<double> dist(-1, 1);
        Eigen::VectorXd v(k.dim()), u(k.dim());
        for (int i = 0; i < k.dim(); ++i) {
            v[i] = dist(rng);
            u[i] = dist(rng);
        }
        const double a = referenceBilinear(s, v, u), b2 = v.dot(k.apply(u));
        CHECK(std::abs(a - b2) <= 1e-11 * std::abs(b2));
    }
    // a benchmark-family problem through the drop-in builders, fast vs standard
    {
        const ProblemSetup ps = paganoSetup(8, LayupFamily::QuadPly, 3, 2);
        CHECK(frobeniusRelDiff(assembleFast(ps), assembleStandard(ps)) <= 1e-12);
    }
    // exceptions (test_assembly.cpp:256-262)
    {
        ProblemSetup bad{cube(1, 1, 1), ExtrudedGeometry(std::make_shared<PlanarRectangle>(1, 1), Eigen::Vector3d(1, 0, 0)),
                         paganoLayup({0.0})};
        CHECK(throws<std::domain_error>([&] { assembleFast(bad); }));
        CHECK(throws<std::domain_error>([&] { assembleStandard(bad); }));
        CHECK(throws<std::invalid_argument>([] { combineOperators(cube(1, 1, 1), {}, {}); }));
    }
}

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
    try {
        hostOnly();
        if (!host_only)
            gpuCases();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "uncaught exception: %s\n", e.what());
        return 2;
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
