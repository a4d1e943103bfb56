/*
 * lamfast_cuda.h — C ABI of the B200-native laminate stiffness assembler.
 *
 * Drop-in boundary for the assembly path of the reference library `lamfast`
 * (arXiv 1905.05417).  The reference exposes a C++ API only (no C ABI, no
 * FFI); every entry point here replaces one of its functions and says which
 * (reference file:line, relative to /root/reference/proj):
 *
 *   lf_assemble(.., LF_BACKEND_FAST, ..)       assembleFast        include/lamfast/fast.hpp:95-96
 *   lf_assemble(.., LF_BACKEND_STANDARD, ..)   assembleStandard    include/lamfast/assembly.hpp:52-53
 *   lf_assemble(.., LF_BACKEND_VOIGT_FREE, ..) assembleVoigtFree   include/lamfast/voigt_free.hpp:69-70
 *   lf_assemble(backend, ..)                   assembleWith        include/lamfast/bench.hpp:19-20
 *   lf_inplane_operators                       computeInplaneOperators         fast.hpp:65-69
 *   lf_inplane_operators_bracket               computeInplaneOperatorsBracket  voigt_free.hpp:60-64
 *   lf_thickness_operators                     computeThicknessOperators       fast.hpp:73-75
 *   lf_combine                                 combineOperators                fast.hpp:86-90
 *   lf_voigt_from_constants / lf_rotate_inplane / lf_angle_decomposition
 *                                              materials.hpp:55,62,68 (host setup, shared)
 *   lf_bracket_parameters                      bracketParameters  voigt_free.hpp:26
 *   lf_contraction_table                       ContractionTable   voigt_free.hpp:41
 *   lf_gauss_legendre / lf_basis_eval          gaussLegendre quadrature.hpp:20-23,
 *                                              KnotVector::evaluate splines.hpp:45
 *   lf_csr_* (device verification)             StiffnessMatrix::{frobeniusNorm,symmetryRelError,apply},
 *                                              frobeniusRelDiff   sparse.hpp:45-69,83
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types.  Device pointers
 *    are named d_*; everything else is host memory.
 *  - Every function returns an lf_status.  Codes map 1:1 back onto the
 *    exception types the reference throws:
 *      LF_ERR_INVALID_ARGUMENT -> std::invalid_argument
 *      LF_ERR_DOMAIN           -> std::domain_error
 *      LF_ERR_LOGIC            -> std::logic_error
 *      LF_ERR_RUNTIME / LF_ERR_CUDA -> std::runtime_error
 *      LF_ERR_OUT_OF_MEMORY    -> std::bad_alloc
 *    lf_last_error() returns the thread-local message of the last failure.
 *  - CSR layout is the reference StiffnessMatrix (sparse.hpp:78-81): int64
 *    row offsets (dim+1), int32 column indices sorted ascending per row, FP64
 *    values; all 9 entries of each coupled 3x3 block are stored.
 *  - There is no CPU fallback: when no CUDA device is usable every compute
 *    entry point fails with LF_ERR_CUDA.
 */
#ifndef LAMFAST_CUDA_H
#define LAMFAST_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LF_ABI_VERSION 1

typedef enum lf_status {
    LF_OK = 0,
    LF_ERR_INVALID_ARGUMENT = 1,
    LF_ERR_DOMAIN = 2,
    LF_ERR_LOGIC = 3,
    LF_ERR_RUNTIME = 4,
    LF_ERR_CUDA = 5,
    LF_ERR_OUT_OF_MEMORY = 6,
    LF_ERR_UNSUPPORTED = 7
} lf_status;

/* Same order as lamfast::Backend (bench.hpp:14). */
typedef enum lf_backend {
    LF_BACKEND_STANDARD = 0,
    LF_BACKEND_FAST = 1,
    LF_BACKEND_VOIGT_FREE = 2
} lf_backend;

/* Built-in SurfaceMap kinds (geometry.hpp:25-58) plus a host-evaluated
 * frame table for any other SurfaceMap subclass (its virtual evaluate is
 * host-only, geometry.hpp:20-24). */
typedef enum lf_geometry_kind {
    LF_GEOM_PLANAR = 0,   /* PlanarRectangle(lx, ly): geometry[0..1] */
    LF_GEOM_BILINEAR = 1, /* BilinearQuad(c00, c10, c01, c11): geometry[0..11] */
    LF_GEOM_FRAMES = 2    /* frames[] table, see lf_problem.frames */
} lf_geometry_kind;

/* OrthotropicConstants (materials.hpp:17-25). */
typedef struct lf_orthotropic {
    double E1, E2, E3;
    double G12, G13, G23;
    double nu12, nu13, nu23;
} lf_orthotropic;

/* LayerSpec (materials.hpp:84-87): angle in radians about the extrusion axis. */
typedef struct lf_layer {
    lf_orthotropic constants;
    double angle;
} lf_layer;

/* ProblemSetup + AssemblyOptions (assembly.hpp:17-36) as plain data. */
typedef struct lf_problem {
    /* TensorProductSpace(u, v, thickness): open knot vectors on [0, 1]. */
    int32_t degree_u, degree_v, degree_t;
    int32_t n_knots_u, n_knots_v, n_knots_t;
    const double* knots_u;
    const double* knots_v;
    const double* knots_t;
    /* Layup(interfaces, layers); identical (constants, angle) pairs share
     * one material configuration, by exact equality, in first-appearance
     * order (materials.cpp:151-183). */
    int32_t n_layers;
    const double* interfaces; /* n_layers + 1, 0 = t0 < ... < tm = 1 */
    const lf_layer* layers;   /* n_layers */
    /* ExtrudedGeometry(surface, direction). */
    int32_t geometry_kind;
    double geometry[12];
    double direction[3];
    /* LF_GEOM_FRAMES: one record of 19 doubles per in-plane quadrature
     * point, elements in (e_v, e_u) order (e_u fastest), points in (q_v, q_u)
     * order (q_u fastest): DF column-major (9), DF^{-T} column-major (9),
     * det (1) -- i.e. GeometryFrame (geometry.hpp:61-67). */
    const double* frames;
    /* AssemblyOptions. */
    int32_t inplane_points;   /* 0 = degree + 1 */
    int32_t thickness_points; /* 0 = degree + 1 */
    int32_t n_active_layers;  /* 0 = all layers active */
    const int32_t* active_layers;
    int32_t decompose_angles; /* fast backend only */
    int32_t threads;          /* accepted, ignored (the device grid replaces std::thread) */
} lf_problem;

/* AssemblyStats (assembly.hpp:39-48); accumulated (+=), never reset. */
typedef struct lf_stats {
    int64_t qpoint_visits;
    int64_t frame_evaluations;
    int32_t operator_builds;
    int32_t reserved;
} lf_stats;

int lf_abi_version(void);
const char* lf_status_name(int status);
const char* lf_last_error(void);
/* Number of usable CUDA devices (0 on a host without a GPU). */
int lf_device_count(void);

/* ---- host-side setup shared with the drop-in C++ layer ---------------- */
int lf_voigt_from_constants(const lf_orthotropic* c, double d_out[36]);
int lf_rotate_inplane(const double d[36], double theta, double d_out[36]);
int lf_angle_decomposition(const lf_orthotropic* c, double out[5 * 36]);
int lf_bracket_parameters(const lf_orthotropic* c, double out[9]);
/* gaussLegendre(n, a, b) (quadrature.cpp:9-57). */
int lf_gauss_legendre(int32_t n, double a, double b, double* points, double* weights);
/* KnotVector::evaluate (splines.cpp:53-101): p+1 values/derivatives at x. */
int lf_basis_eval(int32_t degree, int32_t n_knots, const double* knots, double x,
                  int32_t* first_active, double* values, double* derivs);
/* ContractionTable(params, angle) entries, table[(3i+j)*9 + 3r + c]
 * (voigt_free.cpp:89-123); params = lambda, mu, alpha[7]. */
int lf_contraction_table(const double params[9], double angle, double table[81]);
/* Distinct configurations of the layup: n_configs, per-layer config id,
 * rotated stiffness per config (row-major 6x6).  Arrays sized n_layers. */
int lf_layup_configs(const lf_problem* p, int32_t* n_configs, int32_t* layer_config,
                     double* config_stiffness);

/* ---- closed-form CSR pattern ----------------------------------------- */
/* Host-side view of the operator terms a plan of this problem combines (no
 * device work): their number -- distinct ply configurations, or five per
 * material with decompose_angles on a non-affine map; on an affine map the
 * decomposition's basis tables are summed per configuration first --, their
 * 81-entry contraction tables (tables, [n_terms][81], may be NULL), and the
 * slot schedule of the slot form of the combine: n_slots = 2 or 3 and, per
 * thickness function i_t, the term each slot holds or -1 (slot_term,
 * [n_t][n_slots] with room for 3 per row, may be NULL); n_slots = 0 when some
 * thickness row sees more than three terms.  fast.cpp:285-336 (the terms),
 * fast.cpp:241-258 (which terms a thickness pair sums). */
int lf_operator_terms(const lf_problem* p, int backend, int32_t* n_terms, double* tables, int32_t* n_slots,
                      int32_t* slot_term);
/* Matrix dimension (3 x number of functions) and number of stored entries
 * produced by `backend` (the standard backend drops thickness spans whose
 * cells are all masked by active_layers, assembly.cpp:184-186). */
int lf_pattern_size(const lf_problem* p, int backend, int64_t* dim, int64_t* nnz);
/* Column indices of the CSR rows of the functions [f_begin, f_end) (rows
 * 3 f_begin .. 3 f_end; f_end < 0: to the end), written on the host into
 * cols[0 .. *nnz) -- the same closed form k_pattern_cols writes on the device
 * (the column half of SparseMatrixBuilder::finalize, sparse.cpp:30-55).
 * cols == NULL: only *nnz.  One-shot calls into host arrays use it so that
 * the columns do not cross PCIe.  Host-only: no device is needed. */
int lf_pattern_columns(const lf_problem* p, int backend, int64_t f_begin, int64_t f_end, int32_t* cols,
                       int64_t* nnz);
/* Row slab `part` of `n_parts`, cut at thickness-function boundaries and
 * balanced by nnz.  Rows [row_begin, row_end) hold entries
 * [nnz_begin, nnz_end) of the global CSR. */
int lf_slab_bounds(const lf_problem* p, int backend, int n_parts, int part, int32_t* t_begin,
                   int32_t* t_end, int64_t* row_begin, int64_t* row_end, int64_t* nnz_begin,
                   int64_t* nnz_end);

/* Row slab `part` of `n_parts` cut at FUNCTION boundaries (a function is
 * f = i_t * n_s + i_s, rows 3f .. 3f+2), balanced by nnz to within one
 * function's row block: slabs may start and end inside a thickness row.
 * Functions [f_begin, f_end) = rows [row_begin, row_end) hold entries
 * [nnz_begin, nnz_end) of the global CSR. */
int lf_slab_bounds_functions(const lf_problem* p, int backend, int n_parts, int part,
                             int64_t* f_begin, int64_t* f_end, int64_t* row_begin,
                             int64_t* row_end, int64_t* nnz_begin, int64_t* nnz_end);

/* ---- device-resident plan (bench / multi-GPU slab path) --------------- */
typedef struct lf_plan lf_plan;
/* Uploads the problem tables to `device` and sizes the workspace for the
 * row slab of thickness functions [t_begin, t_end) (t_end < 0: all).
 * `cuda_stream` is a cudaStream_t (NULL = a private stream). */
int lf_plan_create(const lf_problem* p, int backend, int device, void* cuda_stream,
                   int32_t t_begin, int32_t t_end, lf_plan** out);
/* The same for the functions [f_begin, f_end) (f_end < 0: all), i.e. rows
 * [3 f_begin, 3 f_end): a slab cut inside thickness rows. */
int lf_plan_create_range(const lf_problem* p, int backend, int device, void* cuda_stream,
                         int64_t f_begin, int64_t f_end, lf_plan** out);
int lf_plan_destroy(lf_plan* plan);
/* Local slab sizes: rows, nnz, and their global offsets. */
int lf_plan_info(const lf_plan* plan, int64_t* rows, int64_t* nnz, int64_t* row_begin,
                 int64_t* nnz_begin);
/* Writes the slab's CSR pattern (row offsets rebased to 0, global column
 * indices) into device buffers of rows+1 and nnz entries. */
int lf_plan_build_pattern(lf_plan* plan, int64_t* d_row_ptr, int32_t* d_cols);
/* The hot path: every stage from device-resident inputs to the slab's FP64
 * values in d_values (nnz entries, pattern order).  Asynchronous on the
 * plan's stream. */
int lf_plan_assemble(lf_plan* plan, double* d_values);
/* Kernels one lf_plan_assemble enqueues, and the dominant kernel's name. */
int lf_plan_launch_count(const lf_plan* plan);
/* Form of the combine kernel the plan chose for its operator terms (fast and
 * Voigt-free backends): 0 per-term (k_combine), 1 slots (k_combine_slots),
 * 2 coefficient (k_combine_coef); -1 for a standard plan or a null plan. */
int lf_plan_combine_form(const lf_plan* plan);
/* CUDA events around the dominant (combine) kernel of the most recent
 * lf_plan_assemble; cumulative milliseconds and launch count since reset. */
int lf_plan_kernel_time(lf_plan* plan, int reset, double* ms_total, int64_t* launches);
int lf_plan_stats(const lf_plan* plan, lf_stats* stats);
int lf_plan_synchronize(lf_plan* plan);

/* ---- one-shot, host buffers (what the drop-in C++ entry points call) -- */
/* Assembles the full matrix; host arrays must hold dim+1 / nnz / nnz
 * entries (query lf_pattern_size).  The CSR is produced in chunks of at
 * most ~2 GiB (or half the free device memory): each chunk's pattern and
 * values are computed on the device while the previous chunk is copied out,
 * so the matrix only has to fit in host memory, not in HBM.  Pinned host
 * arrays receive the copies directly at full PCIe speed; pageable ones are
 * filled from pinned staging buffers by host threads. */
int lf_assemble(const lf_problem* p, int backend, int device, int64_t* row_ptr, int32_t* cols,
                double* values, lf_stats* stats);
/* The row slab of thickness functions [t_begin, t_end) (lf_slab_bounds) of
 * the same matrix, one-shot into host arrays of rows+1 / nnz / nnz entries
 * (lf_plan_create + lf_plan_rows/nnz give the sizes): row offsets rebased to
 * 0, global columns -- what one rank of a multi-GPU assembly returns.  No
 * reference counterpart (the reference is single-process). */
int lf_assemble_slab(const lf_problem* p, int backend, int device, int32_t t_begin, int32_t t_end,
                     int64_t* row_ptr, int32_t* cols, double* values, lf_stats* stats);
/* The same for the functions [f_begin, f_end) (lf_slab_bounds_functions). */
int lf_assemble_range(const lf_problem* p, int backend, int device, int64_t f_begin, int64_t f_end,
                      int64_t* row_ptr, int32_t* cols, double* values, lf_stats* stats);
/* Receives one chunk of rows of a streamed assembly: global rows
 * [row_begin, row_begin + rows) holding global entries [nnz_begin, nnz_begin
 * + nnz); row_ptr (rows + 1 entries) is chunk-local (starts at 0), columns
 * are global.  The arrays are pinned staging memory valid only during the
 * call; while it runs the device computes and copies the next chunk.
 * Return 0 to continue, non-zero to abort (the assembly then fails with
 * LF_ERR_RUNTIME). */
typedef int (*lf_chunk_sink)(void* user, int64_t row_begin, int64_t rows, int64_t nnz_begin, int64_t nnz,
                             const int64_t* row_ptr, const int32_t* cols, const double* values);
/* The whole matrix streamed through `sink` in row order, in chunks of at most
 * max_chunk_nnz values (0: the library's default): a CSR larger than both
 * HBM and host memory can be written out, reduced or verified chunk by chunk.
 * No reference counterpart (the reference returns one StiffnessMatrix). */
int lf_assemble_stream(const lf_problem* p, int backend, int device, int64_t max_chunk_nnz,
                       lf_chunk_sink sink, void* user, lf_stats* stats);

/* v^T K u by full 3D quadrature without forming K (referenceBilinear,
 * include/lamfast/assembly.hpp; assembly.cpp:247-318): host coefficient
 * arrays of 3 * (number of functions) doubles, result in *out. */
int lf_reference_bilinear(const lf_problem* p, const double* v, const double* u, int device, double* out);

/* ---- operator-level entry points -------------------------------------- */
/* InPlaneOperatorSet in the reference's banded layout (fast.cpp:13-32):
 * blocks[4][n_s][2p_v+1][2p_u+1][9] (3x3 row-major), flags[n_s][2p_v+1][2p_u+1]. */
int lf_inplane_operators(const lf_problem* p, const double material[36], int device,
                         double* blocks, char* flags, lf_stats* stats);
/* Same, from a contraction table C{e_i,e_j} (voigt_free.hpp:32-49):
 * table[(3i+j)*9 + 3r + c] = entry(i,j)(r,c). */
int lf_inplane_operators_bracket(const lf_problem* p, const double table[81], int device,
                                 double* blocks, char* flags, lf_stats* stats);
/* ThicknessOperators: q[n_layers][4][n_t][n_t] (row-major), occupied[n_t][n_t]. */
int lf_thickness_operators(int32_t degree_t, int32_t n_knots_t, const double* knots_t,
                           int32_t n_interfaces, const double* interfaces, int32_t pts_per_cell,
                           int device, double* q, char* occupied);
/* combineOperators over arbitrary terms: blocks/flags per term in the banded
 * layout above, thickness[n_terms][4][n_t][n_t], thickness_occupied[n_t][n_t].
 * Only the space fields of p are read.  Output arrays as for lf_assemble;
 * pass NULL row_ptr/cols/values to query *nnz only. */
int lf_combine(const lf_problem* p, int32_t n_terms, const double* blocks, const char* flags,
               const double* thickness, const char* thickness_occupied, int device,
               int64_t* nnz, int64_t* row_ptr, int32_t* cols, double* values);

/* ---- device-side verification (sparse.cpp:66-139), device pointers ---- */
int lf_csr_frobenius_sq(int64_t rows, const int64_t* d_row_ptr, const double* d_values,
                        void* cuda_stream, double* out);
int lf_csr_spmv(int64_t rows, const int64_t* d_row_ptr, const int32_t* d_cols,
                const double* d_values, const double* d_x, double* d_y, void* cuda_stream);
/* Sum of squared differences over the union pattern of two CSR matrices of
 * the same row count (frobeniusRelDiff numerator, sparse.cpp:108-139). */
int lf_csr_diff_sq(int64_t rows, const int64_t* d_ra, const int32_t* d_ca, const double* d_va,
                   const int64_t* d_rb, const int32_t* d_cb, const double* d_vb,
                   void* cuda_stream, double* out);
/* ||K - K^T||_F^2 numerator of symmetryRelError (sparse.cpp:73-95) for a
 * full CSR of `rows` rows; LF_ERR_INVALID_ARGUMENT if a column lies outside
 * the matrix (a row slab: use lf_csr_symmetry_sq_slab). */
int lf_csr_symmetry_sq(int64_t rows, const int64_t* d_row_ptr, const int32_t* d_cols,
                       const double* d_values, void* cuda_stream, double* out);
/* The same numerator restricted to a row slab holding global rows
 * [row_begin, row_begin + rows) (row offsets rebased to 0, global columns):
 * sum over the slab's entries (r, c) whose mirror row c is also in the slab.
 * *n_skipped (may be NULL) receives the number of entries whose mirror row
 * lies outside.  For row_begin = 0 and the whole matrix it equals
 * lf_csr_symmetry_sq. */
int lf_csr_symmetry_sq_slab(int64_t rows, int64_t row_begin, const int64_t* d_row_ptr,
                            const int32_t* d_cols, const double* d_values, void* cuda_stream,
                            double* out, int64_t* n_skipped);
/* Symmetry numerator of a plan's slab values (pattern order, as written by
 * lf_plan_assemble) from the closed-form pattern: no binary searches, every
 * value read once.  Same slab convention as lf_csr_symmetry_sq_slab. */
int lf_plan_symmetry_sq(lf_plan* plan, const double* d_values, double* out);
/* Returns the library's cached device memory (its private stream-ordered
 * pool, kept across one-shot calls) to the driver. */
int lf_release_memory(int device);

#ifdef __cplusplus
}
#endif

#endif /* LAMFAST_CUDA_H */
