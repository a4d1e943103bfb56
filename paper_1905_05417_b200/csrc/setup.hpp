// Host-side setup of the B200 assembler: validation, knot spans, Gauss rules,
// thickness cells, material tables, layup de-duplication, adjacency and the
// closed-form CSR pattern tables.  Everything here is O(size of the 1D / 2D
// inputs); the O(nnz) work runs on the device (kernels_*.cu).
//
// This is the host half of the reference's L0 layer, restated
// B200-side: splines.cpp, quadrature.cpp, geometry.cpp, materials.cpp and the
// coefficient fit of voigt_free.cpp.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "lamfast_cuda.h"

namespace lfb {

constexpr int kMaxDegree = 6;   // device arrays are sized for p <= 6
constexpr int kMaxPoints = 10;  // Gauss points per direction per element / cell
constexpr int kMaxTermsPerPass = 8;

/// Error carrying an lf_status; the C ABI layer maps it back to the status.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

struct Knots {
    int p = 0;
    std::vector<double> t;
    int n = 0; // number of functions
};
/// KnotVector ctor checks (splines.cpp:10-25).
Knots makeKnots(int degree, int n_knots, const double* knots, const char* which);

/// KnotVector::findSpan + evaluate (splines.cpp:37-101) on the host; returns
/// first_active.  Throws LF_ERR_DOMAIN outside [0, 1].
int evaluateBasis(const Knots& kv, double x, double* vals, double* ders);

struct Span {
    double begin, end;
    int first;
};
/// KnotVector::elementSpans (splines.cpp:103-112).
std::vector<Span> elementSpans(const Knots& kv);

/// gaussLegendre(n) on [-1,1] (quadrature.cpp:9-46), mapped to [a,b] (48-57).
void gaussLegendre(int n, double a, double b, double* pts, double* wts);

struct Cell {
    double lo, hi;
    int layer, span;
};
/// layerwiseThicknessRule cell list (quadrature.cpp:59-87), without rules.
std::vector<Cell> thicknessCells(const Knots& kt, const std::vector<Span>& spans,
                                 const std::vector<double>& interfaces);

// ---- materials (materials.cpp) ------------------------------------------
void voigtFromConstants(const lf_orthotropic& c, double d[36]);
void rotateInplane(const double d[36], double theta, double out[36]);
void angleDecomposition(const lf_orthotropic& c, double out[180]);
/// bracketParameters (voigt_free.cpp:52-80): lambda, mu, alpha[7].
void bracketParameters(const lf_orthotropic& c, double out[9]);
/// ContractionTable(params, angle) (voigt_free.cpp:89-123):
/// table[(3i+j)*9 + 3r + c] = C{e_i, e_j}(r, c).
void contractionTable(const double params[9], double angle, double table[81]);
/// The same contraction-table layout from a Voigt matrix: C{e_j,e_l}(i,k) =
/// C_ijkl = D(V(i,j), V(k,l)) (materials.cpp:26-33), so that both P
/// formulations share one device kernel.
void tableFromVoigt(const double d[36], double table[81]);

bool sameConstants(const lf_orthotropic& a, const lf_orthotropic& b);

struct LayupInfo {
    int n_configs = 0;
    std::vector<int> layer_config;        // per layer
    std::vector<std::array<double, 36>> D; // per config, rotated stiffness
    std::vector<int> rep_layer;           // first layer of each config
};
/// Layup ctor (materials.cpp:151-183).
LayupInfo buildLayup(const lf_problem& p);

/// GeometryFrame (geometry.hpp:61-67): df, dfit col-major, det.
struct Frame {
    double df[9], dfit[9], det;
};
/// ExtrudedGeometry::frameAt for the built-in surfaces (geometry.cpp:8-31,74-85).
Frame frameAt(const lf_problem& p, double u, double v);

/// 1D adjacency of a knot direction: function j is adjacent to i iff both
/// are active on a common (enabled) span.  Always a contiguous interval.
struct Adjacency {
    std::vector<int32_t> lo, len;
    std::vector<int64_t> pre; // prefix sums of len, size n+1
    int64_t total = 0;
    int max_len = 0;
};
Adjacency adjacency(int p, int n, const std::vector<Span>& spans,
                    const std::vector<char>* span_enabled = nullptr);

/// Everything a plan needs, computed once on the host.
struct Setup {
    int backend = LF_BACKEND_FAST;
    Knots ku, kv, kt;
    std::vector<Span> spu, spv, spt;
    int nqu = 0, nqv = 0, nqt = 0;
    std::vector<double> ru, wu, rv, wv; // reference Gauss rules on [-1, 1]
    std::vector<double> interfaces;
    std::vector<Cell> cells;            // all cells (fast) or unmasked (standard), span-major
    std::vector<double> cell_pts, cell_wts; // [n_cells][nqt]
    std::vector<int32_t> cell_first;    // first active thickness function of the cell's span
    std::vector<int32_t> cell_layer;
    std::vector<int32_t> span_cell0;    // [n_spans_t + 1] cell ranges per span
    std::vector<int32_t> spt_first;     // [n_spans_t]
    LayupInfo layup;
    std::vector<char> layer_active;
    // operator terms: contraction tables and per-layer multipliers
    int n_terms = 0;
    std::vector<double> term_table;     // [T][81]
    std::vector<double> lam;            // [T][L]
    std::vector<uint8_t> lam_on;        // [T][L]
    // geometry
    bool affine = false;                // constant frame (PlanarRectangle)
    Frame frame0{};                     // the constant frame when affine
    std::vector<double> frames;         // [n_el][nqu*nqv][19] when !affine
    // pattern
    Adjacency au, av, at;
    int64_t S_s = 0;                    // in-plane pairs
    std::vector<int64_t> es_pre;        // [n_s + 1] = 9 * P_s(i_s)
    int n_u = 0, n_v = 0, n_t = 0, n_s = 0;
    // slab: the functions f = i_t * n_s + i_s in [f0, f1) (rows 3 f0 .. 3 f1);
    // they cover the thickness rows [t0, t1), the first from in-plane
    // function s0, the last up to s1 (exclusive); out_base = L_t(t0) *
    // es_pre[s0] is the offset of (t0, s0) inside thickness row t0's block
    int t0 = 0, t1 = 0, s0 = 0, s1 = 0;
    int64_t f0 = 0, f1 = 0, out_base = 0;
    int64_t rows = 0, nnz = 0, row_begin = 0, nnz_begin = 0, n_pairs = 0;
    // stats of one assembly (analytic)
    lf_stats stats{};
};

/// Builds the setup of `backend` for thickness rows [t0, t1) (t1 < 0: all).
Setup buildSetup(const lf_problem& p, int backend, int t0, int t1);
/// The same for the functions [f0, f1) (f = i_t * n_s + i_s; f1 < 0: all):
/// row slabs cut inside a thickness row.
Setup buildSetupRange(const lf_problem& p, int backend, int64_t f0, int64_t f1);
/// Sizes and offsets of the functions [f0, f1) of a full setup (f1 < 0: to the end).
struct Range {
    int t0 = 0, t1 = 0, s0 = 0, s1 = 0;
    int64_t f0 = 0, f1 = 0, out_base = 0, rows = 0, row_begin = 0, nnz = 0, nnz_begin = 0, n_pairs = 0;
};
Range rangeOf(const Setup& s, int64_t f0, int64_t f1);
/// Restricts a setup to the functions [f0, f1) (slab sizes and offsets).
void applyRange(Setup& s, int64_t f0, int64_t f1);
/// Global CSR offset of the first entry of function f (f = n_t * n_s: nnz).
int64_t functionOffset(const Setup& s, int64_t f);

/// Host writer of the closed-form CSR columns of the functions [f_lo, f_hi)
/// (the same pattern k_pattern_cols writes), into cols[0 ..).
void fillColumns(const Setup& s, int64_t f_lo, int64_t f_hi, int32_t* cols);

/// Space-only setup (knots, spans, quadrature, adjacency) used by the
/// operator-level entry points.
Setup buildSpaceSetup(const lf_problem& p, bool need_geometry);

/// Row slab of n_parts balanced by nnz at thickness-function boundaries.
void slabBounds(const Setup& full, int n_parts, int part, int* t0, int* t1);
/// Row slab of n_parts balanced by nnz at function boundaries (cuts inside
/// thickness rows): functions [f0, f1).
void slabBoundsFunctions(const Setup& full, int n_parts, int part, int64_t* f0, int64_t* f1);

} // namespace lfb
