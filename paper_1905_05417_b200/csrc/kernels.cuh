// Device-side tables and kernel launchers of the B200 assembler.
//
// Data layout in HBM:
//   in-plane entry space  e in [0, E), E = 9 * S_s: for in-plane function i_s,
//       entries es_pre[i_s] .. es_pre[i_s+1]) ordered (a, slot, b) with
//       slot = (j_v - lo_v(i_v)) * L_u(i_u) + (j_u - lo_u(i_u)) -- exactly the
//       order of one CSR row block, so thread e writes output entries
//       base_t(i_t) + L_t(i_t) * (es_pre[i_s] + a*3L_s) + k*3L_s + (3*slot + b)
//       for every thickness row i_t and neighbour k.
//   thickness pairs p in [0, n_pairs): (i_t, j_t = lo_t(i_t) + k) of the slab in
//       CSR order; W[p][term][family] are the layer-reduced q~ weights and
//       Wmask[pass][p] flags the terms that have any contributing cell.
#pragma once

#include <cstdint>
#ifdef LF_DEBUG_CHECKS
#include <cstdio>
#endif

namespace lfb {

// Device-side bounds checks (debug builds: make EXTRA=-DLF_DEBUG_CHECKS).  The
// pool's compute-sanitizer is unavailable, so every index a kernel writes
// through is checked against its buffer and a violation traps the kernel.
#ifdef LF_DEBUG_CHECKS
#define LF_CHECK(cond)                                                                                         \
    do {                                                                                                       \
        if (!(cond)) {                                                                                         \
            printf("LF_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                               \
            __trap();                                                                                          \
        }                                                                                                      \
    } while (0)
#else
#define LF_CHECK(cond) \
    do {               \
    } while (0)
#endif

struct DevTables {
    // degrees / sizes
    int pu, pv, pt;
    int nu, nv, nt, ns;
    int nspu, nspv, nspt;
    int nqu, nqv, nqt;
    int ncells, n_layers, n_terms, n_passes;
    int bu, bv; // band widths 2p+1 of the U/V tables
    // knots
    const double *ku, *kv, *kt;
    int nku, nkv, nkt;
    // spans + reference Gauss rules on [-1, 1]
    const int *spu_first, *spv_first, *spt_first;
    const double *spu_lo, *spu_hi, *spv_lo, *spv_hi;
    const double *ru, *wu, *rv, *wv;
    // thickness cells (span-major), their Gauss rules, span -> cell range
    const double *cell_pts, *cell_wts;
    const int *cell_first, *cell_layer, *span_cell0;
    // operator terms
    const double* term_table; // [T][81] contraction tables C{e_j,e_l}(i,k)
    const double* lam;        // [T][L]
    const unsigned char* lam_on;
    const int* layer_config;  // [L]
    // adjacency / pattern
    const int *lo_u, *len_u, *lo_v, *len_v, *lo_t, *len_t;
    const long long *pre_u, *pre_v, *pre_t;
    const long long* es_pre; // [ns + 1]
    const int* blk_is;       // [ceil(E / 256)] i_s of each 256-entry block's first entry
    int lt_max;              // max L_t over all thickness rows
    // every term table has major symmetry C[(3j+l)9 + 3a+b] = C[(3l+j)9 + 3b+a]:
    // the standard kernel (K6) then computes pairs al <= be and mirrors them
    int sym;
    long long S_s, S_u;
    // geometry
    int affine;
    double G[9]; // constant DF^{-T} (col-major) when affine
    double det;
    const double* frames; // [n_el][nqu*nqv][19] when !affine
    // workspace
    double *Bu_val, *Bu_der, *Bv_val, *Bv_der; // [nsp * nq][p+1]
    double *Bt_val, *Bt_der;                   // [ncells * nqt][pt+1]
    int* Bt_first;                             // [ncells * nqt]
    double *U, *V;                             // [n][b][4]
    double* Ct;                                // [T][81]
    double* W;                                 // [n_pairs][T][4]
    unsigned* Wmask;                           // [n_passes][n_pairs]
    double* Pg;                                // [T][4][E] (general geometry)
    // coefficient form of the combine (affine geometry, many terms): per
    // thickness pair E[pair][ab][xy] = sum_t Ct[t][xy][ab] W[pair][t][f(xy)],
    // padded to kEStride doubles per ab; nullptr -> the per-term form
    double* Etab;
    double* Pe;     // element-local P of a batch of pe_terms terms: [term][el][4][nl2][3][nl2][3]
    int pe_terms;   // terms per batch
    // two-phase standard assembly (K6): element-local blocks of a batch of
    // ks_batch thickness spans, Ks[span][el][pair][9] (pair: al <= be when sym)
    double* Ks;
    int ks_batch;
    const int* spt_first_h; // host copy of spt_first (the launcher's batch bounds)
    // combine launches: 1 = grid x runs over the row chunks, y over the entry blocks (k_combine.cu)
    int grid_swap;
    // slot form of the per-term combine (k_combine_slots): per thickness row
    // (absolute i_t) the term held by each of n_slots register slots, -1: slot
    // not used by the row; n_slots = 0: per-term / coefficient forms
    const int* slot_term;
    int n_slots;
    // output range: the functions f = i_t * ns + i_s in [f0, f1), covering
    // thickness rows [t0, t1) -- row t0 from in-plane function s0, row t1 - 1
    // up to s1 (exclusive).  Entry (it, is, ...) of the range is written at
    // 9 S_s (pre_t[it] - pre_t[t0]) + L_t(it) es_pre[is] + ... - out_base;
    // row offsets get rp_base added (0: slab-local CSR).
    int t0, t1, s0, s1;
    long long f0, f1, out_base, rp_base;
    // thickness rows whose pair weights W / Wmask hold (the plan's slab;
    // a streamed sub-range reads the plan's W)
    int w_t0, w_t1;
    long long n_pairs, E;
    long long nnz_slab; // values of this range (bounds checks in LF_DEBUG_CHECKS builds)
};

/// Pulled-back contraction tables of an affine map without the in-plane
/// weight, det G C G per material configuration, passed to K6 phase 1 as a
/// kernel parameter (constant bank: no shared-memory loads in its inner loop).
constexpr int kK6MaxCfg = 16;
struct K6Const {
    int n_cfg; // 0: not available (non-affine map or too many configurations)
    double C[kK6MaxCfg][81];
};

constexpr int kEStride = 10; // doubles per (pair, ab) row of Etab (9 used; 16-byte rows)
constexpr int kEPair = 9 * kEStride;

// Launchers (all asynchronous on `stream`).  Return cudaError_t as int.
int launch_basis(const DevTables& d, bool with_ct, cudaStream_t stream);
int launch_thickness_pairs(const DevTables& d, cudaStream_t stream);
/// Affine fast path: U, V, thickness pairs and Ct in one launch.
int launch_prepare_affine(const DevTables& d, cudaStream_t stream);
int launch_integrals_1d(const DevTables& d, cudaStream_t stream);
/// General-geometry in-plane operators into Pg (two-phase: Pe, then the gather).
int launch_inplane_general(const DevTables& d, cudaStream_t stream);
int inplane_general_launches(const DevTables& d);
int launch_affine_export(const DevTables& d, cudaStream_t stream);
/// Combine: one launch per pass of <= 8 terms.  `t_chunk` thickness rows per
/// block row; returns the number of kernels launched via *launches.
int launch_combine(const DevTables& d, double* out, int t_chunk, cudaStream_t stream,
                   int* launches);
/// Coefficient form: Etab from W and Ct (after the setup kernels).
int launch_pair_coeffs(const DevTables& d, cudaStream_t stream);
int launch_pattern(const DevTables& d, long long* row_ptr, int* cols, cudaStream_t stream);
int launch_standard(const DevTables& d, double* values, long long nnz, cudaStream_t stream,
                    int* launches, const K6Const* cst = nullptr);

/// Matrix-free v^T K u (referenceBilinear, assembly.cpp:247-318); partial holds
/// nspu * nspv * nspt doubles, *out (device) the result.
int launch_bilinear(const DevTables& d, const double* u, const double* v, double* partial, double* out,
                    cudaStream_t stream);

// Verification (sparse.cpp:66-139)
int launch_frobenius_sq(long long rows, const long long* rp, const double* v, double* out,
                        cudaStream_t stream);
int launch_spmv(long long rows, const long long* rp, const int* c, const double* v,
                const double* x, double* y, cudaStream_t stream);
int launch_diff_sq(long long rows, const long long* ra, const int* ca, const double* va,
                   const long long* rb, const int* cb, const double* vb, double* out,
                   cudaStream_t stream);
/// rows [row_begin, row_begin + rows) of a CSR; mirrors outside are skipped
/// and counted into *outside (device)
int launch_symmetry_sq(long long rows, long long row_begin, const long long* rp, const int* c,
                       const double* v, double* out, unsigned long long* outside, cudaStream_t stream);
/// closed-form symmetry numerator of a plan's slab values (pattern order)
int launch_plan_symmetry(const DevTables& d, const double* v, double* out, cudaStream_t stream);

} // namespace lfb
