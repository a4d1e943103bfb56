// lamfast C++ API, B200 edition.
//
// Drop-in replacement for the public C++ interface of the reference library
// `lamfast` (/root/reference/proj/include/lamfast/*.hpp): the same namespace,
// class and function names, argument and return types, and the same
// exception types.  The assembly entry points run on the GPU through the C ABI
// of include/lamfast_cuda.h (liblamfast_b200.so); everything here is host-side
// setup, containers and result accessors.
//
// The per-module headers (lamfast/fast.hpp, lamfast/assembly.hpp, ...) the
// reference's users include all resolve to this file.
//
// Additions over the reference API (ABI-compatible for callers):
//   * StiffnessMatrix::fromCsr(...)       adopt a CSR produced on the device
//   * PlanarRectangle::lx()/ly(), BilinearQuad::corner(k)   geometry accessors
//   * lamfast::setDevice(int) / device()  CUDA device used by the assemblers
#pragma once

#include <array>
#include <cstdint>
#include <iosfwd>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include <Eigen/Dense>

namespace lamfast {

// =====================================================================
// B-spline bases (reference splines.hpp)
// =====================================================================

/// Active basis functions at one parametric point: p+1 values and first
/// derivatives, starting at global index first_active.
struct BasisEval1D {
    double point = 0.0;
    int first_active = 0;
    std::vector<double> values;
    std::vector<double> derivs;
};

/// A nonempty knot span [begin, end); functions first_active..first_active+p live on it.
struct Span {
    double begin = 0.0;
    double end = 0.0;
    int first_active = 0;
};

/// Clamped (open) knot vector on [0, 1]; interior multiplicity may be up to p.
class KnotVector {
public:
    KnotVector(int degree, std::vector<double> knots);
    static KnotVector uniform(int degree, int n_elements);

    int degree() const { return p_; }
    int numFunctions() const { return static_cast<int>(t_.size()) - p_ - 1; }
    const std::vector<double>& knots() const { return t_; }

    int findSpan(double x) const;
    BasisEval1D evaluate(double x) const;
    std::vector<Span> elementSpans() const;

    bool operator==(const KnotVector&) const = default;

private:
    int p_;
    std::vector<double> t_;
};

/// u x v x thickness space; global index i = i_t * n_s + i_v * n_u + i_u.
class TensorProductSpace {
public:
    TensorProductSpace(KnotVector inplane_u, KnotVector inplane_v, KnotVector thickness);

    const KnotVector& inplaneU() const { return ku_; }
    const KnotVector& inplaneV() const { return kv_; }
    const KnotVector& thickness() const { return kt_; }
    int numU() const { return ku_.numFunctions(); }
    int numV() const { return kv_.numFunctions(); }
    int numThickness() const { return kt_.numFunctions(); }
    int numInplane() const { return numU() * numV(); }
    int numFunctions() const { return numInplane() * numThickness(); }
    int flattenInplane(int iu, int iv) const { return iv * numU() + iu; }
    int flatten(int iu, int iv, int it) const { return it * numInplane() + flattenInplane(iu, iv); }
    std::array<int, 3> split(int i) const;

private:
    KnotVector ku_, kv_, kt_;
};

// =====================================================================
// Quadrature (reference quadrature.hpp)
// =====================================================================

struct QuadratureRule {
    std::vector<double> points;
    std::vector<double> weights;
    int size() const { return static_cast<int>(points.size()); }
};

QuadratureRule gaussLegendre(int n);
QuadratureRule gaussLegendre(int n, double a, double b);

/// span intersected with layer, with its Gauss rule.
struct ThicknessCell {
    double lo = 0.0;
    double hi = 0.0;
    int layer = 0;
    int span = 0;
    QuadratureRule rule;
};

std::vector<ThicknessCell> layerwiseThicknessRule(const KnotVector& kv,
                                                  const std::vector<double>& interfaces,
                                                  int n_points);

// =====================================================================
// Geometry (reference geometry.hpp)
// =====================================================================

struct SurfacePoint {
    Eigen::Vector3d position = Eigen::Vector3d::Zero();
    Eigen::Vector3d du = Eigen::Vector3d::Zero();
    Eigen::Vector3d dv = Eigen::Vector3d::Zero();
};

/// Midsurface S(u, v) on the unit square.  Subclasses other than the
/// built-in ones are evaluated on the host and shipped as a frame table.
class SurfaceMap {
public:
    virtual ~SurfaceMap() = default;
    virtual SurfacePoint evaluate(double u, double v) const = 0;
};

class PlanarRectangle : public SurfaceMap {
public:
    PlanarRectangle(double lx, double ly);
    SurfacePoint evaluate(double u, double v) const override;
    double lx() const { return a_; }
    double ly() const { return b_; }

private:
    double a_, b_;
};

class BilinearQuad : public SurfaceMap {
public:
    BilinearQuad(Eigen::Vector3d c00, Eigen::Vector3d c10, Eigen::Vector3d c01, Eigen::Vector3d c11);
    SurfacePoint evaluate(double u, double v) const override;
    /// corners in constructor order c00, c10, c01, c11
    const Eigen::Vector3d& corner(int k) const { return c_[static_cast<std::size_t>(k)]; }

private:
    std::array<Eigen::Vector3d, 4> c_;
};

class SplineSurface : public SurfaceMap {
public:
    SplineSurface(KnotVector ku, KnotVector kv, std::vector<Eigen::Vector3d> controls);
    SurfacePoint evaluate(double u, double v) const override;

private:
    KnotVector bu_, bv_;
    std::vector<Eigen::Vector3d> net_;
};

struct GeometryFrame {
    Eigen::Matrix3d df = Eigen::Matrix3d::Identity();
    Eigen::Matrix3d df_inv_transpose = Eigen::Matrix3d::Identity();
    double det = 1.0;
    Eigen::Vector3d covariant(int i) const { return df.col(i); }
    Eigen::Vector3d contravariant(int i) const { return df_inv_transpose.col(i); }
};

/// F(u, v, w) = S(u, v) + w a.
class ExtrudedGeometry {
public:
    ExtrudedGeometry(std::shared_ptr<const SurfaceMap> surface, Eigen::Vector3d direction);
    GeometryFrame frameAt(double u, double v) const;
    Eigen::Vector3d position(double u, double v, double w) const;
    const Eigen::Vector3d& direction() const { return dir_; }
    const SurfaceMap& surface() const { return *surf_; }

private:
    std::shared_ptr<const SurfaceMap> surf_;
    Eigen::Vector3d dir_;
};

inline Eigen::Vector3d pullbackGradient(const GeometryFrame& frame, const Eigen::Vector3d& grad_hat) {
    return frame.df_inv_transpose * grad_hat;
}

// =====================================================================
// Materials (reference materials.hpp)
// =====================================================================

/// 6x6 stiffness, Voigt order (11, 22, 33, 12, 13, 23), engineering shear.
using VoigtMatrix = Eigen::Matrix<double, 6, 6>;

struct OrthotropicConstants {
    double E1 = 1.0, E2 = 1.0, E3 = 1.0;
    double G12 = 0.5, G13 = 0.5, G23 = 0.5;
    double nu12 = 0.0, nu13 = 0.0, nu23 = 0.0;
    static OrthotropicConstants isotropic(double e, double nu);
    bool operator==(const OrthotropicConstants&) const = default;
};

class ElasticityTensor {
public:
    ElasticityTensor() { c_.fill(0.0); }
    double& operator()(int i, int j, int k, int l) { return c_[idx(i, j, k, l)]; }
    double operator()(int i, int j, int k, int l) const { return c_[idx(i, j, k, l)]; }
    static ElasticityTensor fromVoigt(const VoigtMatrix& d);
    VoigtMatrix toVoigt() const;
    ElasticityTensor rotated(const Eigen::Matrix3d& r) const;
    double quadraticForm(const Eigen::Matrix3d& eps) const;

private:
    static std::size_t idx(int i, int j, int k, int l) {
        return static_cast<std::size_t>(27 * i + 9 * j + 3 * k + l);
    }
    std::array<double, 81> c_;
};

VoigtMatrix voigtFromConstants(const OrthotropicConstants& c);
OrthotropicConstants constantsFromVoigt(const VoigtMatrix& d);
VoigtMatrix rotateInplane(const VoigtMatrix& d, double theta);
std::array<VoigtMatrix, 5> angleDecomposition(const OrthotropicConstants& c);

struct MaterialConfig {
    OrthotropicConstants constants;
    double angle = 0.0;
    int id = 0;
    VoigtMatrix stiffness = VoigtMatrix::Zero();
    bool matches(const OrthotropicConstants& c, double theta) const {
        return constants == c && angle == theta;
    }
};

struct LayerSpec {
    OrthotropicConstants constants;
    double angle = 0.0;
};

class Layup {
public:
    Layup(std::vector<double> interfaces, const std::vector<LayerSpec>& layers);
    static Layup equalLayers(const std::vector<LayerSpec>& layers);

    int numLayers() const { return static_cast<int>(cfg_of_layer_.size()); }
    const std::vector<double>& interfaces() const { return z_; }
    int layerAt(double xi3) const;
    int configIndexOf(int layer) const { return cfg_of_layer_[static_cast<std::size_t>(layer)]; }
    const MaterialConfig& configOf(int layer) const {
        return cfgs_[static_cast<std::size_t>(configIndexOf(layer))];
    }
    const MaterialConfig& materialAt(double xi3) const { return configOf(layerAt(xi3)); }
    const std::vector<MaterialConfig>& distinctConfigs() const { return cfgs_; }
    int numDistinctConfigs() const { return static_cast<int>(cfgs_.size()); }

private:
    std::vector<double> z_;
    std::vector<int> cfg_of_layer_;
    std::vector<MaterialConfig> cfgs_;
};

// =====================================================================
// Sparse storage (reference sparse.hpp)
// =====================================================================

struct Triplet {
    int row = 0;
    int col = 0;
    double value = 0.0;
};

class StiffnessMatrix;

class SparseMatrixBuilder {
public:
    explicit SparseMatrixBuilder(int n_functions);
    int numFunctions() const { return n_; }
    int dim() const { return 3 * n_; }
    std::size_t numTriplets() const { return entries_.size(); }
    void addBlock(int i, int j, const Eigen::Matrix3d& block);
    void merge(SparseMatrixBuilder&& other);
    void reserve(std::size_t n) { entries_.reserve(n); }
    StiffnessMatrix finalize() const;

private:
    int n_;
    std::vector<Triplet> entries_;
};

class StiffnessMatrix {
public:
    StiffnessMatrix() = default;
    /// Adopts a CSR (row offsets dim+1, sorted columns, values).  Addition.
    static StiffnessMatrix fromCsr(int dim, std::vector<std::int64_t> row_offsets,
                                   std::vector<int> cols, std::vector<double> values);

    int dim() const { return n_; }
    std::int64_t nnz() const { return static_cast<std::int64_t>(val_.size()); }
    double at(int row, int col) const;
    double frobeniusNorm() const;
    double symmetryRelError() const;
    Eigen::VectorXd apply(const Eigen::VectorXd& x) const;
    const std::vector<std::int64_t>& rowOffsets() const { return ptr_; }
    const std::vector<int>& colIndices() const { return col_; }
    const std::vector<double>& values() const { return val_; }

private:
    friend class SparseMatrixBuilder;
    int n_ = 0;
    std::vector<std::int64_t> ptr_;
    std::vector<int> col_;
    std::vector<double> val_;
};

double frobeniusRelDiff(const StiffnessMatrix& a, const StiffnessMatrix& b);
void writeMatrixMarket(const StiffnessMatrix& m, std::ostream& out);

// =====================================================================
// Assembly (reference assembly.hpp, fast.hpp, voigt_free.hpp, bench.hpp)
// =====================================================================

struct ProblemSetup {
    TensorProductSpace space;
    ExtrudedGeometry geom;
    Layup layup;
};

struct AssemblyOptions {
    int threads = 1;          ///< accepted and ignored on the GPU
    int inplane_points = 0;   ///< 0: degree + 1
    int thickness_points = 0; ///< 0: degree + 1
    std::vector<int> active_layers;
    bool decompose_angles = false;
};

struct AssemblyStats {
    std::int64_t qpoint_visits = 0;
    std::int64_t frame_evaluations = 0;
    int operator_builds = 0;
};

/// CUDA device used by the assembly entry points (default 0, or the
/// LAMFAST_DEVICE environment variable).  Addition.
void setDevice(int device);
int device();

StiffnessMatrix assembleStandard(const ProblemSetup& setup, const AssemblyOptions& options = {},
                                 AssemblyStats* stats = nullptr);
double referenceBilinear(const ProblemSetup& setup, const Eigen::VectorXd& v, const Eigen::VectorXd& u,
                         const AssemblyOptions& options = {});

class InPlaneOperator {
public:
    InPlaneOperator(int n_u, int n_v, int degree_u, int degree_v);
    int numInplane() const { return nu_ * nv_; }
    int bandU() const { return 2 * pu_ + 1; }
    int bandV() const { return 2 * pv_ + 1; }
    bool inBand(int is, int js) const;
    bool occupied(int is, int js) const;
    void markOccupied(int is, int js) { occ_[slot(is, js)] = 1; }
    Eigen::Matrix3d& block(int is, int js) { return blk_[slot(is, js)]; }
    const Eigen::Matrix3d& block(int is, int js) const { return blk_[slot(is, js)]; }
    std::vector<int> bandColumns(int is) const;

private:
    std::size_t slot(int is, int js) const;
    int nu_, nv_, pu_, pv_;
    std::vector<Eigen::Matrix3d> blk_;
    std::vector<char> occ_;
};

struct InPlaneOperatorSet {
    std::array<InPlaneOperator, 4> op;
};

struct ThicknessOperators {
    std::vector<std::array<Eigen::MatrixXd, 4>> per_layer;
    Eigen::Matrix<char, Eigen::Dynamic, Eigen::Dynamic> occupied;
};

InPlaneOperatorSet computeInplaneOperators(const TensorProductSpace& space, const ExtrudedGeometry& geom,
                                           const VoigtMatrix& material, const AssemblyOptions& options = {},
                                           AssemblyStats* stats = nullptr);
ThicknessOperators computeThicknessOperators(const KnotVector& thickness, const std::vector<double>& interfaces,
                                             int pts_per_cell);

struct OperatorTerm {
    InPlaneOperatorSet inplane;
    std::array<Eigen::MatrixXd, 4> thickness;
};

StiffnessMatrix combineOperators(const TensorProductSpace& space, const std::vector<OperatorTerm>& terms,
                                 const Eigen::Matrix<char, Eigen::Dynamic, Eigen::Dynamic>& thickness_occupied,
                                 const AssemblyOptions& options = {});
StiffnessMatrix assembleFast(const ProblemSetup& setup, const AssemblyOptions& options = {},
                             AssemblyStats* stats = nullptr);

struct BracketParameters {
    double lambda = 0.0;
    double mu = 0.0;
    std::array<double, 7> alpha = {0, 0, 0, 0, 0, 0, 0};
};

BracketParameters bracketParameters(const OrthotropicConstants& constants);

class ContractionTable {
public:
    static Eigen::Matrix3d isotropicEntry(double lambda, double mu, int i, int j);
    ContractionTable(const BracketParameters& params, double angle);
    const Eigen::Matrix3d& entry(int i, int j) const { return tab_[static_cast<std::size_t>(3 * i + j)]; }

private:
    std::array<Eigen::Matrix3d, 9> tab_;
};

std::array<Eigen::Matrix3d, 9> pullbackContractionTable(const ContractionTable& table, const GeometryFrame& frame);
InPlaneOperatorSet computeInplaneOperatorsBracket(const TensorProductSpace& space, const ExtrudedGeometry& geom,
                                                  const ContractionTable& table,
                                                  const AssemblyOptions& options = {},
                                                  AssemblyStats* stats = nullptr);
StiffnessMatrix assembleVoigtFree(const ProblemSetup& setup, const AssemblyOptions& options = {},
                                  AssemblyStats* stats = nullptr);

enum class Backend { Standard, Fast, VoigtFree };
std::string backendName(Backend backend);
Backend backendFromName(const std::string& name);
StiffnessMatrix assembleWith(Backend backend, const ProblemSetup& setup, const AssemblyOptions& options = {},
                             AssemblyStats* stats = nullptr);

// Problem builders of the reference's benchmark header (bench.hpp:22-46): the
// callers' side of the path.  The sweep harness itself (BenchConfig, runBench,
// the JSON config parser) is not part of this edition; its CSV/JSON report
// format is reproduced by paper_1905_05417_b200/report.py.
enum class LayupFamily { CrossPly, QuadPly, Custom };
std::string layupFamilyName(LayupFamily family);
LayupFamily layupFamilyFromName(const std::string& name);
/// Cross-ply alternates {0, 90} deg, quad-ply cycles {0, 45, -45, 90} deg;
/// throws std::invalid_argument for the custom family or m < 1.
std::vector<double> familyAngles(LayupFamily family, int m);

struct PlateDimensions {
    double lx = 1.0, ly = 1.0, thickness = 0.1;
};

/// Pagano's material: E1 = 25, E2 = E3 = 1, G12 = G13 = 0.2, G23 = 0.5, nu = 0.25.
OrthotropicConstants paganoConstants();
/// Equal Pagano layers at `angles`, an lx x ly plate extruded along
/// (0, 0, thickness), uniform maximum-continuity knots of `degree` everywhere.
ProblemSetup paganoSetup(const std::vector<double>& angles, int degree, int elements_x, int elements_y,
                         int thickness_elements = 1, const PlateDimensions& plate = {});
ProblemSetup paganoSetup(int m, LayupFamily family, int degree, int elements);

} // namespace lamfast
