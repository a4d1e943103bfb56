// Operator, cross-check, pattern and verification kernels of the B200
// laminate assembler (sm_100a).
//
//  K2a k_integrals_1d     1D basis-product integrals U, V (sum-factorised P
//                         for affine geometry; fast.cpp:54-168 restated)
//  K2b k_inplane_elem +   per-element P for non-affine geometry, two-phase
//      k_inplane_gather   (fast.cpp:54-168 / voigt_free.cpp:142-248)
//  (K4 k_combine, the hot kernel, is in k_combine.cu)
//  K5  k_pattern_*        closed-form CSR row offsets and columns
//  K6  k_standard_local + full 3D quadrature cross-check, two-phase
//      k_standard_gather
//                         (assembly.cpp:134-245)
//  K7  verification       ||K||_F, K x, ||A-B||_F, ||K-K^T||_F (sparse.cpp:66-139)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "combine_common.cuh"

namespace lfb {

namespace {

// ---------------------------------------------------------------------------
// K2a: U[i][slot][2d+e] = sum over spans and Gauss points of
//      (w h) N_i^{(d)} N_j^{(e)},  j = lo(i) + slot.
// With a constant frame the 2D in-plane integrals factor exactly:
//      I_xy(i_s, j_s) = U_{du_x du_y}(i_u, j_u) * V_{dv_x dv_y}(i_v, j_v).
__global__ void k_integrals_1d(DevTables d) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int nu_slots = d.nu * d.bu, nv_slots = d.nv * d.bv;
    if (g >= nu_slots + nv_slots)
        return;
    const bool is_u = g < nu_slots;
    const int h = is_u ? g : g - nu_slots;
    const int b = is_u ? d.bu : d.bv;
    const int i = h / b, slot = h % b;
    const int p = is_u ? d.pu : d.pv;
    const int* lo = is_u ? d.lo_u : d.lo_v;
    const int* len = is_u ? d.len_u : d.len_v;
    const int* first = is_u ? d.spu_first : d.spv_first;
    const double* slo = is_u ? d.spu_lo : d.spv_lo;
    const double* shi = is_u ? d.spu_hi : d.spv_hi;
    const double* wref = is_u ? d.wu : d.wv;
    const double* bval = is_u ? d.Bu_val : d.Bv_val;
    const double* bder = is_u ? d.Bu_der : d.Bv_der;
    const int nsp = is_u ? d.nspu : d.nspv, nq = is_u ? d.nqu : d.nqv;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (slot < len[i]) {
        const int j = lo[i] + slot;
        const int mn = min(i, j), mx = max(i, j);
        for (int s = 0; s < nsp; ++s) {
            const int f = first[s];
            if (f > mn || mx > f + p)
                continue;
            const double half = 0.5 * (shi[s] - slo[s]);
            for (int q = 0; q < nq; ++q) {
                const long long row = ((long long)s * nq + q) * (p + 1);
                const double w = wref[q] * half;
                const double vi = bval[row + i - f], di = bder[row + i - f];
                const double vj = bval[row + j - f], dj = bder[row + j - f];
                acc[0] += w * vi * vj;
                acc[1] += w * vi * dj;
                acc[2] += w * di * vj;
                acc[3] += w * di * dj;
            }
        }
    }
    double* out = (is_u ? d.U : d.V) + (long long)h * 4;
    out[0] = acc[0];
    out[1] = acc[1];
    out[2] = acc[2];
    out[3] = acc[3];
}

/// Exports P of every term in the entry layout Pg[t][f][e] (affine path),
/// for the operator-level entry point.
__global__ void k_affine_export(const DevTables d) {
    const long long e = (long long)blockIdx.x * kBlock + threadIdx.x;
    if (e >= d.E)
        return;
    const int is = find_is(d.es_pre, d.ns, e);
    const int r = (int)(e - d.es_pre[is]);
    const int iu = is % d.nu, iv = is / d.nu;
    const int Lu = d.len_u[iu], Lv = d.len_v[iv];
    const int B = 3 * Lu * Lv;
    const int a = r / B, rem = r - a * B;
    const int s = rem / 3, b = rem % 3;
    const int sv = s / Lu, su = s - sv * Lu;
    for (int t = 0; t < d.n_terms; ++t) {
        double P[1][4];
        affine_p<1>(d, iu, iv, su, sv, 3 * a + b, t, P);
        for (int f = 0; f < 4; ++f)
            d.Pg[((long long)t * 4 + f) * d.E + e] = P[0][f];
    }
}

// ---------------------------------------------------------------------------
// Shared per-element prologue: gradient tables and quadrature weights.
struct ElemInfo {
    int eu, ev, fu, fv, nl2, nq2;
    double hu, hv;
};

__device__ __forceinline__ void element_tables(const DevTables& d, const ElemInfo& el, double* gh,
                                               double* w2) {
    // gh[(q*nl2 + a)*3 + {0,1,2}] = (du, dv, val) of local function a at in-plane point q
    for (int idx = threadIdx.x; idx < el.nq2 * el.nl2; idx += blockDim.x) {
        const int q = idx / el.nl2, a = idx % el.nl2;
        const int qv = q / d.nqu, qu = q % d.nqu;
        const int jv = a / (d.pu + 1), ju = a % (d.pu + 1);
        const long long ru = ((long long)el.eu * d.nqu + qu) * (d.pu + 1) + ju;
        const long long rv = ((long long)el.ev * d.nqv + qv) * (d.pv + 1) + jv;
        const double bu = d.Bu_val[ru], bud = d.Bu_der[ru];
        const double bv = d.Bv_val[rv], bvd = d.Bv_der[rv];
        gh[idx * 3 + 0] = bud * bv;
        gh[idx * 3 + 1] = bu * bvd;
        gh[idx * 3 + 2] = bu * bv;
    }
    for (int q = threadIdx.x; q < el.nq2; q += blockDim.x) {
        const int qv = q / d.nqu, qu = q % d.nqu;
        w2[q] = d.wu[qu] * el.hu * d.wv[qv] * el.hv; // assembly.cpp:44-45
    }
}

/// Ctq[q][3x+y][3i+k] = scale_q * sum_{j,l} G_q(j,x) G_q(l,y) C{e_j,e_l}(i,k)
/// (pullbackContractionTable, voigt_free.cpp:125-140).
__device__ __forceinline__ void pullback_tables(const DevTables& d, int e_index, int nq2,
                                                const double* w2, const double* table, double* ctq) {
    // layout [q][xy][10]: ik padded to 10 so the consumers load 16-byte pairs
    for (int idx = threadIdx.x; idx < nq2 * 90; idx += blockDim.x) {
        const int q = idx / 90, xy = (idx % 90) / 10, ik = idx % 10;
        if (ik == 9) {
            ctq[idx] = 0.0;
            continue;
        }
        const int x = xy / 3, y = xy % 3;
        const double* G;
        double det;
        if (d.affine) {
            G = d.G;
            det = d.det;
        } else {
            const double* f = d.frames + ((long long)e_index * nq2 + q) * 19;
            G = f + 9;
            det = f[18];
        }
        double s = 0.0;
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l)
                s += G[3 * x + j] * G[3 * y + l] * table[(3 * j + l) * 9 + ik];
        ctq[idx] = w2[q] * det * s;
    }
}


// ---------------------------------------------------------------------------
// K2b, two-phase form (default): phase 1 computes every element's local P
// for a batch of terms into Pe -- all elements in one launch, coalesced
// writes, no colours, no read-modify-write; phase 2 gathers each in-plane
// entry's contributions from the <= (p+1)^2 elements that contain both of
// its functions, in a fixed element order (deterministic), and writes Pg
// once.  The coloured in-place form it replaced (tools/experiments/
// k2b_variants.cu) re-read and re-wrote most of Pg in each of its (p+1)^2
// launches with 24-byte pieces (C3: 141 MB read + 57 MB written per launch,
// profiles/r1_ncu_inplane_general_c3.txt).

/// Offset of value (f, al, a, be, b) inside one element's block of Pe.
__device__ __forceinline__ long long pe_local(int f, int al, int a, int be, int b, int nl2) {
    return ((((long long)f * nl2 + al) * 3 + a) * nl2 + be) * 3 + b;
}

/// Phase 1: one block per (element, term); a thread takes one family f, one
/// al and kK2bPairs consecutive be, so every broadcast load of a C~ row
/// (warp-uniform f) feeds kK2bPairs x 9 FMA (the one-pair form loaded a row
/// per 9 FMA: C3 1.10 ms, FP64 pipe 4%, profiles/r1_k2b.txt).
#ifndef LF_K2B_PAIRS
#define LF_K2B_PAIRS 4
#endif
#ifndef LF_K2B_MINB
#define LF_K2B_MINB 2
#endif
constexpr int kK2bPairs = LF_K2B_PAIRS;

__host__ __device__ inline int k2b_family_slots(int nl2) {
    return (nl2 * ((nl2 + kK2bPairs - 1) / kK2bPairs) + 31) / 32 * 32;
}

__global__ void __launch_bounds__(256, LF_K2B_MINB) k_inplane_elem(const DevTables d, int t0) {
    extern __shared__ double sm[];
    const int e_index = blockIdx.x;
    const int t = t0 + blockIdx.y;
    if (t >= d.n_terms)
        return;
    ElemInfo el;
    el.eu = e_index % d.nspu;
    el.ev = e_index / d.nspu;
    el.fu = d.spu_first[el.eu];
    el.fv = d.spv_first[el.ev];
    el.nl2 = (d.pu + 1) * (d.pv + 1);
    el.nq2 = d.nqu * d.nqv;
    el.hu = 0.5 * (d.spu_hi[el.eu] - d.spu_lo[el.eu]);
    el.hv = 0.5 * (d.spv_hi[el.ev] - d.spv_lo[el.ev]);
    double* gh = sm;
    double* w2 = gh + el.nq2 * el.nl2 * 3;
    double* ctq = sm + ((el.nq2 * el.nl2 * 3 + el.nq2 + 1) & ~1);
    element_tables(d, el, gh, w2);
    __syncthreads();
    pullback_tables(d, e_index, el.nq2, w2, d.term_table + (long long)t * 81, ctq);
    __syncthreads();
    const int nel = d.nspu * d.nspv;
    const long long per_el = 36LL * el.nl2 * el.nl2;
    double* pe = d.Pe + ((long long)blockIdx.y * nel + e_index) * per_el;
    const int ngroup = (el.nl2 + kK2bPairs - 1) / kK2bPairs;
    const int fslots = k2b_family_slots(el.nl2);
    for (int idx = threadIdx.x; idx < 4 * fslots; idx += blockDim.x) {
        const int f = idx / fslots;
        const int g = idx - f * fslots;
        if (g >= el.nl2 * ngroup)
            continue;
        const int al = g / ngroup, be0 = (g - al * ngroup) * kK2bPairs;
        const int nxy = f == 0 ? 4 : f == 3 ? 1 : 2;
        int xys[4];
        xys[0] = f == 0 ? 0 : f == 1 ? 2 : f == 2 ? 6 : 8;
        xys[1] = f == 0 ? 1 : f == 1 ? 5 : 7;
        xys[2] = 3;
        xys[3] = 4;
        int bes[kK2bPairs];
#pragma unroll
        for (int p = 0; p < kK2bPairs; ++p)
            bes[p] = min(be0 + p, el.nl2 - 1);
        double acc[kK2bPairs][9];
#pragma unroll
        for (int p = 0; p < kK2bPairs; ++p)
#pragma unroll
            for (int k = 0; k < 9; ++k)
                acc[p][k] = 0.0;
        for (int q = 0; q < el.nq2; ++q) {
            const double* ga = gh + (q * el.nl2 + al) * 3;
            const double* C = ctq + q * 90;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (u < nxy) {
                    const int xy = xys[u];
                    const double gx = ga[xy / 3];
                    const double2* C2 = reinterpret_cast<const double2*>(C + xy * 10);
                    const double2 c0 = C2[0], c1 = C2[1], c2 = C2[2], c3 = C2[3], c4 = C2[4];
#pragma unroll
                    for (int p = 0; p < kK2bPairs; ++p) {
                        const double sxy = gx * gh[(q * el.nl2 + bes[p]) * 3 + xy % 3];
                        acc[p][0] = fma(c0.x, sxy, acc[p][0]);
                        acc[p][1] = fma(c0.y, sxy, acc[p][1]);
                        acc[p][2] = fma(c1.x, sxy, acc[p][2]);
                        acc[p][3] = fma(c1.y, sxy, acc[p][3]);
                        acc[p][4] = fma(c2.x, sxy, acc[p][4]);
                        acc[p][5] = fma(c2.y, sxy, acc[p][5]);
                        acc[p][6] = fma(c3.x, sxy, acc[p][6]);
                        acc[p][7] = fma(c3.y, sxy, acc[p][7]);
                        acc[p][8] = fma(c4.x, sxy, acc[p][8]);
                    }
                }
            }
        }
#pragma unroll
        for (int p = 0; p < kK2bPairs; ++p) {
            if (be0 + p >= el.nl2)
                continue;
            LF_CHECK(pe_local(f, al, 2, be0 + p, 2, el.nl2) < per_el);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    pe[pe_local(f, al, a, be0 + p, b, el.nl2)] = acc[p][3 * a + b];
        }
    }
}


/// First span index s with first[s] >= lo (first[] strictly increasing).
__device__ __forceinline__ int span_lower(const int* first, int nsp, int lo) {
    int a = 0, b = nsp;
    while (a < b) {
        const int m = (a + b) >> 1;
        if (first[m] < lo)
            a = m + 1;
        else
            b = m;
    }
    return a;
}

/// K2b phase 2: Pg[t][f][e] = sum over the elements containing both functions
/// of entry e (ev outer, eu inner: a fixed order), from Pe; one thread per
/// entry and term computes the four families (the entry decode and element
/// search are shared).  PU/PV > 0: the (PU+1)(PV+1) candidate elements are
/// unrolled so their loads issue together; 0: runtime degrees.
template <int PU, int PV>
__global__ void k_inplane_gather(const DevTables d, int t0) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    const int t = t0 + y;
    if (e >= d.E || t >= d.n_terms)
        return;
    const int pu = PU > 0 ? PU : d.pu, pv = PV > 0 ? PV : d.pv;
    int is = __ldg(d.blk_is + e / kBlock);
    while (__ldg(d.es_pre + is + 1) <= e)
        ++is;
    const int r = (int)(e - __ldg(d.es_pre + is));
    const int iu = is % d.nu, iv = is / d.nu;
    const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
    const int B = 3 * Lu * Lv;
    const int a = r / B, rem = r - a * B;
    const int s = rem / 3, b = rem - 3 * s;
    const int sv = s / Lu, su = s - sv * Lu;
    const int ju = __ldg(d.lo_u + iu) + su, jv = __ldg(d.lo_v + iv) + sv;
    const int pu1 = pu + 1, nl2 = pu1 * (pv + 1);
    const int nel = d.nspu * d.nspv;
    const long long per_el = 36LL * nl2 * nl2;
    const long long fstride = 9LL * nl2 * nl2; // pe_local(f + 1, ...) - pe_local(f, ...)
    const double* pe = d.Pe + (long long)y * nel * per_el;
    // elements (spans) containing both functions: first <= min and first + p >= max
    const int u_lo = span_lower(d.spu_first, d.nspu, max(iu, ju) - pu);
    const int v_lo = span_lower(d.spv_first, d.nspv, max(iv, jv) - pv);
    const int umin = min(iu, ju), vmin = min(iv, jv);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if constexpr (PU > 0 && PV > 0) {
        int fu[PU + 1];
        bool uok[PU + 1];
#pragma unroll
        for (int i = 0; i <= PU; ++i) {
            const int eu = u_lo + i;
            fu[i] = eu < d.nspu ? __ldg(d.spu_first + eu) : 0x7fffffff;
            uok[i] = fu[i] <= umin;
        }
#pragma unroll
        for (int j = 0; j <= PV; ++j) {
            const int ev = v_lo + j;
            const int fv = ev < d.nspv ? __ldg(d.spv_first + ev) : 0x7fffffff;
            const bool vok = fv <= vmin;
            double v[PU + 1][4];
#pragma unroll
            for (int i = 0; i <= PU; ++i) {
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    v[i][f] = 0.0;
                if (vok && uok[i]) {
                    const int al = (iv - fv) * pu1 + (iu - fu[i]), be = (jv - fv) * pu1 + (ju - fu[i]);
                    const double* src = pe + (long long)(ev * d.nspu + u_lo + i) * per_el +
                                        pe_local(0, al, a, be, b, nl2);
#pragma unroll
                    for (int f = 0; f < 4; ++f)
                        v[i][f] = __ldg(src + f * fstride);
                }
            }
#pragma unroll
            for (int i = 0; i <= PU; ++i)
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    acc[f] += v[i][f];
        }
    } else {
        for (int ev = v_lo; ev < d.nspv && __ldg(d.spv_first + ev) <= vmin; ++ev) {
            const int fv = __ldg(d.spv_first + ev);
            for (int eu = u_lo; eu < d.nspu && __ldg(d.spu_first + eu) <= umin; ++eu) {
                const int fu = __ldg(d.spu_first + eu);
                const int al = (iv - fv) * pu1 + (iu - fu), be = (jv - fv) * pu1 + (ju - fu);
                const double* src = pe + (long long)(ev * d.nspu + eu) * per_el + pe_local(0, al, a, be, b, nl2);
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    acc[f] += __ldg(src + f * fstride);
            }
        }
    }
    LF_CHECK(((long long)t * 4 + 3) * d.E + e < (long long)d.n_terms * 4 * d.E);
#pragma unroll
    for (int f = 0; f < 4; ++f)
        d.Pg[((long long)t * 4 + f) * d.E + e] = acc[f];
}

// ---------------------------------------------------------------------------
// K6: standard full-3D quadrature (assembly.cpp:134-245), the reference's
// element loop with its full in-plane quadrature, in two phases (below).
//
// The local block of a pair (al, be) = ((at, as), (bt, bs)) is
//   K[ab] = sum_cells sum_q2 sum_q3 sum_xy Ct_q2[xy][ab] X_al[x] X_be[y] w3,
//   X_al = (du N_as T_at, dv N_as T_at, N_as T'_at)   (assembly.cpp:203-206).
// The 3D Gauss rule is a tensor product and the pulled-back Ct of a cell
// does not vary with q3, so the thickness points are summed first, exactly:
//   sum_q3 X_al[x] X_be[y] w3 = g_as[x] g_bs[y] tau[at][bt][x==2][y==2],
//   tau[at][bt][i][j] = sum_q3 T^(i)_at T^(j)_bt w3     (per cell, 36 values),
// so a (pair, q2) costs 18 products + 81 FMA, with no thickness loop.  Each
// thread takes a group of KP pairs sharing al (KP consecutive be), so every
// broadcast load of a Ct row feeds KP x 9 FMA (ncu, the one-pair form: FP64
// pipe 43%, shared-memory loads as the second stall; profiles/r1_ncu_standard_c3.txt).
// Measured (C3 / C4 ms, profiles/r2_k6_*.txt): round 1 (one pair per thread,
// q3 loop, 48 coloured launches of += into the CSR) 87 / 88; tau + KP = 2,
// coloured, 78 / 85 (KP = 3, 4 at 197-228 registers: 120-200, the += needs
// warps to hide its loads), + L2 prefetch of the += targets 76.5 / 81.5;
// two-phase 62.6 / 82.0, with the pair-symmetric gather (every stored block
// read once) 60.1 / 80.7 (KP = 3, 4 at 8 warps/SM: 76-78 / 99-106).
// Pairs per thread and blocks per SM are template parameters of phase 1:
// p = 3 (nl3 = 48) runs best at KP = 2, 16 warps/SM (C3 56.3 ms against 67.3
// at KP = 1, 32 warps); p <= 2 (nl3 = 27) the other way round (C4 67.7
// against 75.7 ms), profiles/r2_k6_occ.txt.

/// Pair group g of an element block: al and the first be of KP consecutive
/// be (be >= al when the tables are symmetric).
template <int KP>
__device__ __forceinline__ void k6_group(int g, int nl3, bool sym, int& al, int& be0) {
    if (sym) {
        al = 0;
        int per = (nl3 + KP - 1) / KP;
        while (g >= per) {
            g -= per;
            ++al;
            per = (nl3 - al + KP - 1) / KP;
        }
        be0 = al + g * KP;
    } else {
        const int per = (nl3 + KP - 1) / KP;
        al = g / per;
        be0 = (g % per) * KP;
    }
}

template <int KP>
__host__ __device__ inline int k6_groups(int nl3, bool sym) {
    if (!sym)
        return nl3 * ((nl3 + KP - 1) / KP);
    int n = 0;
    for (int al = 0; al < nl3; ++al)
        n += (nl3 - al + KP - 1) / KP;
    return n;
}

// ---------------------------------------------------------------------------
// K6, two-phase form: phase 1 (k_standard_local) computes every (element,
// span) block's local pairs into the scratch Ks -- all elements and spans of
// a batch in one launch, coalesced stores, no colours, no read-modify-write
// of the CSR; phase 2 (k_standard_gather) has one thread per (row block,
// in-plane pair) sum, for each thickness neighbour, the <= (pt+1)(pu+1)(pv+1)
// local blocks that contain both functions in a fixed (span, ev, eu) order
// (deterministic) and add the 9 values into the CSR once per batch.

/// Triangular index of the local pair (al, be), al <= be, or the full one.
__device__ __forceinline__ int k6_pair_index(int al, int be, int nl3, bool sym) {
    return sym ? al * nl3 - (al * (al - 1)) / 2 + (be - al) : al * nl3 + be;
}

/// CONSTC: affine map, the per-configuration tables det G C G come in the
/// kernel parameter `cst`, so a cell's pulled-back table is w2[q] times one
/// of them (one product per entry) instead of the frame contraction of
/// pullback_tables (9 products and the frame loads per entry).  The inner
/// loop reads the table from shared memory either way: reading it from the
/// constant bank measured C4 71.5 ms but C3 65.1 against 60.1 ms (the
/// register-indexed constant loads set the pace), profiles/r2_k6_const.txt.
template <bool CONSTC, int KP, int MINB>
__global__ void __launch_bounds__(256, MINB) k_standard_local(const DevTables d, int ks0,
                                                                    const __grid_constant__ K6Const cst) {
    extern __shared__ double sm[];
    ElemInfo el;
    const int e_index = blockIdx.x;
    el.eu = e_index % d.nspu;
    el.ev = e_index / d.nspu;
    const int ks = ks0 + blockIdx.y;
    if (ks >= d.nspt)
        return;
    const int c0 = d.span_cell0[ks], c1 = d.span_cell0[ks + 1];
    if (c0 == c1)
        return; // span with no unmasked cell: phase 2 skips it
    if (d.spt_first[ks] + d.pt < d.t0 || d.spt_first[ks] >= d.t1)
        return; // no row of this span lies in the slab
    el.fu = d.spu_first[el.eu];
    el.fv = d.spv_first[el.ev];
    el.nl2 = (d.pu + 1) * (d.pv + 1);
    el.nq2 = d.nqu * d.nqv;
    el.hu = 0.5 * (d.spu_hi[el.eu] - d.spu_lo[el.eu]);
    el.hv = 0.5 * (d.spv_hi[el.ev] - d.spv_lo[el.ev]);
    const int ft = d.spt_first[ks];
    const int ntl = d.pt + 1;
    const int nl3 = el.nl2 * ntl;
    double* gh = sm;
    double* w2 = gh + el.nq2 * el.nl2 * 3;
    double* ctq = sm + ((el.nq2 * el.nl2 * 3 + el.nq2 + 1) & ~1); // nq2 * 90, 16-byte aligned
    double* tv = ctq + el.nq2 * 90;
    double* td = tv + d.nqt * ntl;
    double* w3 = td + d.nqt * ntl;
    double* tau = w3 + d.nqt; // [at][bt][i][j]
    element_tables(d, el, gh, w2);
    const bool sym = d.sym != 0;
    const int ngroup = k6_groups<KP>(nl3, sym);
    const long long per_blk = 9LL * (sym ? nl3 * (nl3 + 1) / 2 : nl3 * nl3);
    double* kb = d.Ks + ((long long)blockIdx.y * (d.nspu * d.nspv) + e_index) * per_blk;
    for (int c = c0; c < c1; ++c) {
        __syncthreads();
        const int cfg = d.layer_config[d.cell_layer[c]];
        if constexpr (CONSTC) { // affine: the pulled-back table is w2[q] times the configuration's
            const double* Cc = cst.C[cfg];
            for (int idx = threadIdx.x; idx < el.nq2 * 90; idx += blockDim.x) {
                const int q = idx / 90, r = idx - 90 * q, xy = r / 10, ik = r - 10 * xy;
                ctq[idx] = ik == 9 ? 0.0 : w2[q] * Cc[xy * 9 + ik];
            }
        } else {
            pullback_tables(d, e_index, el.nq2, w2, d.term_table + (long long)cfg * 81, ctq);
        }
        for (int idx = threadIdx.x; idx < d.nqt * ntl; idx += blockDim.x) {
            const int q = idx / ntl, a = idx % ntl;
            const long long h = (long long)c * d.nqt + q;
            const int sh = ft - d.Bt_first[h]; // 0 unless a point rounds onto a knot
            const int aa = a + sh;
            const bool ok = aa >= 0 && aa <= d.pt;
            tv[idx] = ok ? d.Bt_val[h * ntl + aa] : 0.0;
            td[idx] = ok ? d.Bt_der[h * ntl + aa] : 0.0;
        }
        for (int q = threadIdx.x; q < d.nqt; q += blockDim.x)
            w3[q] = d.cell_wts[(long long)c * d.nqt + q];
        __syncthreads();
        for (int idx = threadIdx.x; idx < ntl * ntl * 4; idx += blockDim.x) {
            const int a = idx / (4 * ntl), b = (idx / 4) % ntl, i = (idx >> 1) & 1, j = idx & 1;
            double s = 0.0;
            for (int q3 = 0; q3 < d.nqt; ++q3)
                s += (i ? td : tv)[q3 * ntl + a] * (j ? td : tv)[q3 * ntl + b] * w3[q3];
            tau[idx] = s;
        }
        __syncthreads();
        for (int g = threadIdx.x; g < ngroup; g += blockDim.x) {
            int al, be0;
            k6_group<KP>(g, nl3, sym, al, be0);
            const int at = al / el.nl2, as = al % el.nl2;
            int bs[KP], bt[KP];
            bool pv[KP];
#pragma unroll
            for (int p = 0; p < KP; ++p) {
                const int be = be0 + p;
                pv[p] = be < nl3;
                const int bec = pv[p] ? be : al;
                bt[p] = bec / el.nl2;
                bs[p] = bec % el.nl2;
            }
            double acc[KP][9];
            double tp[KP][4];
#pragma unroll
            for (int p = 0; p < KP; ++p) {
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    acc[p][k] = 0.0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    tp[p][k] = tau[(at * ntl + bt[p]) * 4 + k];
            }
            for (int q2 = 0; q2 < el.nq2; ++q2) {
                const double* ga = gh + (q2 * el.nl2 + as) * 3;
                const double a0 = ga[0], a1 = ga[1], a2 = ga[2];
                double gb[KP][3];
#pragma unroll
                for (int p = 0; p < KP; ++p) {
                    const double* b = gh + (q2 * el.nl2 + bs[p]) * 3;
                    gb[p][0] = b[0];
                    gb[p][1] = b[1];
                    gb[p][2] = b[2];
                }
                const double2* C2 = reinterpret_cast<const double2*>(ctq + q2 * 90);
#pragma unroll
                for (int xy = 0; xy < 9; ++xy) {
                    const int x = xy / 3, y = xy % 3;
                    const double gx = x == 0 ? a0 : x == 1 ? a1 : a2;
                    const double2 r0 = C2[xy * 5], r1 = C2[xy * 5 + 1], r2 = C2[xy * 5 + 2], r3 = C2[xy * 5 + 3],
                                  r4 = C2[xy * 5 + 4];
#pragma unroll
                    for (int p = 0; p < KP; ++p) {
                        const double s = gx * gb[p][y] * tp[p][(x == 2 ? 2 : 0) + (y == 2 ? 1 : 0)];
                        acc[p][0] = fma(r0.x, s, acc[p][0]);
                        acc[p][1] = fma(r0.y, s, acc[p][1]);
                        acc[p][2] = fma(r1.x, s, acc[p][2]);
                        acc[p][3] = fma(r1.y, s, acc[p][3]);
                        acc[p][4] = fma(r2.x, s, acc[p][4]);
                        acc[p][5] = fma(r2.y, s, acc[p][5]);
                        acc[p][6] = fma(r3.x, s, acc[p][6]);
                        acc[p][7] = fma(r3.y, s, acc[p][7]);
                        acc[p][8] = fma(r4.x, s, acc[p][8]);
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < KP; ++p) {
                if (!pv[p])
                    continue;
                double* o = kb + 9LL * k6_pair_index(al, be0 + p, nl3, sym);
                LF_CHECK(o >= kb && o + 9 <= kb + per_blk);
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    o[k] = c == c0 ? acc[p][k] : o[k] + acc[p][k]; // a block's own scratch: no race
            }
        }
    }
}

/// Phase 2: thread per (thickness row it of the batch, in-plane pair
/// (i_s, slot)); for every neighbour j_t of it, the 3x3 block K(i, j) is the
/// sum over the batch's spans and the elements containing both in-plane
/// functions of the local blocks in Ks, added into the CSR.  With symmetric
/// tables only blocks al <= be are stored; local order follows the global
/// function order, so the thread with i < j reads its blocks directly
/// (consecutive slots: consecutive blocks) and also adds the transpose into
/// row block j, the thread with i > j does nothing unless j lies outside the
/// output range (then it reads the transposed blocks itself): every stored
/// block is read once.
__global__ void __launch_bounds__(256) k_standard_gather(const DevTables d, double* __restrict__ values, int ks0,
                                                         int ks1, int it_lo) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; // in-plane pair
    const int it = it_lo + blockIdx.y;
    if (q >= d.S_s || it < d.t0 || it >= d.t1)
        return;
    const long long e = 9 * q;
    int is = __ldg(d.blk_is + e / kBlock);
    while (__ldg(d.es_pre + is + 1) <= e)
        ++is;
    const long long gi = (long long)it * d.ns + is;
    if (gi < d.f0 || gi >= d.f1)
        return; // partial first / last row of a function range
    const int slot = (int)((e - __ldg(d.es_pre + is)) / 9);
    const int iu = is % d.nu, iv = is / d.nu;
    const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
    const int sv = slot / Lu, su = slot - sv * Lu;
    const int ju = __ldg(d.lo_u + iu) + su, jv = __ldg(d.lo_v + iv) + sv;
    const int js = jv * d.nu + ju;
    const int B = 3 * Lu * Lv;
    const int nl2 = (d.pu + 1) * (d.pv + 1), ntl = d.pt + 1, nl3 = nl2 * ntl;
    const bool sym = d.sym != 0;
    const long long per_blk = 9LL * (sym ? nl3 * (nl3 + 1) / 2 : nl3 * nl3);
    const int nel = d.nspu * d.nspv;
    // elements containing both in-plane functions: first[e] <= min, max <= first[e] + p
    const int umin = min(iu, ju), umax = max(iu, ju), vmin = min(iv, jv), vmax = max(iv, jv);
    const int eu_lo = span_lower(d.spu_first, d.nspu, umax - d.pu);
    const int ev_lo = span_lower(d.spv_first, d.nspv, vmax - d.pv);
    const int Lt = __ldg(d.len_t + it), lot = __ldg(d.lo_t + it);
    const long long pre0 = __ldg(d.pre_t + d.t0), nine_S = 9 * d.S_s;
    const long long row0 = nine_S * (__ldg(d.pre_t + it) - pre0) + (long long)Lt * __ldg(d.es_pre + is) + 3 * slot -
                           d.out_base;
    for (int k = 0; k < Lt; ++k) {
        const int jt = lot + k;
        const long long gj = (long long)jt * d.ns + js;
        const bool j_in = gj >= d.f0 && gj < d.f1;
        // which blocks this thread writes: K(i,j) always (row i is ours), K(j,i)
        // too when i < j and row j is ours; a thread with i > j and row j ours
        // leaves both to that row's thread
        if (sym && gi > gj && j_in)
            continue;
        const bool mirror = sym && gi < gj && j_in;
        const bool transposed = sym && gi > gj; // stored block is (be, al)
        const int tmin = min(it, jt), tmax = max(it, jt);
        double acc[9];
#pragma unroll
        for (int x = 0; x < 9; ++x)
            acc[x] = 0.0;
        bool any = false;
        for (int ks = max(ks0, span_lower(d.spt_first, d.nspt, tmax - d.pt)); ks < ks1; ++ks) {
            const int ft = __ldg(d.spt_first + ks);
            if (ft > tmin)
                break;
            if (__ldg(d.span_cell0 + ks) == __ldg(d.span_cell0 + ks + 1))
                continue; // masked span (assembly.cpp:185-186)
            const int at = it - ft, bt = jt - ft;
            for (int ev = ev_lo; ev < d.nspv && __ldg(d.spv_first + ev) <= vmin; ++ev) {
                const int fv = __ldg(d.spv_first + ev);
                for (int eu = eu_lo; eu < d.nspu && __ldg(d.spu_first + eu) <= umin; ++eu) {
                    const int fu = __ldg(d.spu_first + eu);
                    const int al = at * nl2 + (iv - fv) * (d.pu + 1) + (iu - fu);
                    const int be = bt * nl2 + (jv - fv) * (d.pu + 1) + (ju - fu);
                    const double* kb = d.Ks + ((long long)(ks - ks0) * nel + ev * d.nspu + eu) * per_blk;
                    any = true;
                    if (!transposed) {
                        const double* src = kb + 9LL * k6_pair_index(al, be, nl3, sym);
#pragma unroll
                        for (int x = 0; x < 9; ++x)
                            acc[x] += __ldg(src + x);
                    } else { // K(i,j) = K(j,i)^T
                        const double* src = kb + 9LL * k6_pair_index(be, al, nl3, sym);
#pragma unroll
                        for (int a = 0; a < 3; ++a)
#pragma unroll
                            for (int b = 0; b < 3; ++b)
                                acc[3 * a + b] += __ldg(src + 3 * b + a);
                    }
                }
            }
        }
        if (!any)
            continue;
        const long long pos = row0 + (long long)k * B;
        LF_CHECK(pos >= 0 && pos + 2LL * Lt * B + 2 < d.nnz_slab);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                values[pos + (long long)a * Lt * B + b] += acc[3 * a + b];
        if (mirror) { // K(j,i)[b][a] = K(i,j)[a][b], in row block j
            const int Luj = __ldg(d.len_u + ju), Lvj = __ldg(d.len_v + jv);
            const int Bj = 3 * Luj * Lvj, Ltj = __ldg(d.len_t + jt);
            const int slot_m = (iv - __ldg(d.lo_v + jv)) * Luj + (iu - __ldg(d.lo_u + ju));
            const long long posj = nine_S * (__ldg(d.pre_t + jt) - pre0) + (long long)Ltj * __ldg(d.es_pre + js) +
                                   (long long)(it - __ldg(d.lo_t + jt)) * Bj + 3 * slot_m - d.out_base;
            LF_CHECK(posj >= 0 && posj + 2LL * Ltj * Bj + 2 < d.nnz_slab);
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    values[posj + (long long)b * Ltj * Bj + a] += acc[3 * a + b];
        }
    }
}

// ---------------------------------------------------------------------------
// K8: matrix-free v^T K u by full 3D quadrature (referenceBilinear,
// assembly.cpp:247-318): no matrix is formed.  One block per (element,
// thickness span); the element's local coefficients of u and v sit in shared
// memory, each thread takes quadrature points, forms the reference-space
// gradients G(a, x) = sum_al c[al][a] dN_al/dx and adds
// sum_{a,b,x,y} Gv(a,x) Ct_q[xy][ab] Gu(b,y) w3 (Ct_q = pulled-back C with
// the in-plane weight and |det|: the same tables as K6).  Block partials go to
// partial[block]; k_bilinear_final sums them in block order (deterministic).
__global__ void __launch_bounds__(128) k_bilinear(const DevTables d, const double* __restrict__ u,
                                                  const double* __restrict__ v, double* __restrict__ partial) {
    extern __shared__ double sm[];
    const long long bid = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    ElemInfo el;
    el.eu = blockIdx.x;
    el.ev = blockIdx.y;
    const int ks = blockIdx.z;
    el.fu = d.spu_first[el.eu];
    el.fv = d.spv_first[el.ev];
    el.nl2 = (d.pu + 1) * (d.pv + 1);
    el.nq2 = d.nqu * d.nqv;
    el.hu = 0.5 * (d.spu_hi[el.eu] - d.spu_lo[el.eu]);
    el.hv = 0.5 * (d.spv_hi[el.ev] - d.spv_lo[el.ev]);
    const int ft = d.spt_first[ks];
    const int ntl = d.pt + 1;
    const int nl3 = el.nl2 * ntl;
    double* gh = sm;
    double* w2 = gh + el.nq2 * el.nl2 * 3;
    double* ctq = sm + ((el.nq2 * el.nl2 * 3 + el.nq2 + 1) & ~1); // nq2 * 90
    double* tv = ctq + el.nq2 * 90;                                 // nqt * ntl values, then derivatives
    double* td = tv + d.nqt * ntl;
    double* w3 = td + d.nqt * ntl;
    double* cu = w3 + d.nqt; // [nl3][3] local coefficients of u, then v
    double* cv = cu + 3 * nl3;
    double* red = cv + 3 * nl3; // [warps]
    const int c0 = d.span_cell0[ks], c1 = d.span_cell0[ks + 1];
    double acc = 0.0;
    if (c0 < c1) {
        element_tables(d, el, gh, w2);
        for (int idx = threadIdx.x; idx < 3 * nl3; idx += blockDim.x) {
            const int l = idx / 3, comp = idx - 3 * l;
            const int at = l / el.nl2, as = l - at * el.nl2;
            const int iu = el.fu + as % (d.pu + 1), iv = el.fv + as / (d.pu + 1);
            const long long gi = (long long)(ft + at) * d.ns + (long long)iv * d.nu + iu;
            cu[idx] = u[3 * gi + comp];
            cv[idx] = v[3 * gi + comp];
        }
        const int e_index = el.ev * d.nspu + el.eu;
        for (int c = c0; c < c1; ++c) {
            __syncthreads();
            const int cfg = d.layer_config[d.cell_layer[c]];
            pullback_tables(d, e_index, el.nq2, w2, d.term_table + (long long)cfg * 81, ctq);
            for (int idx = threadIdx.x; idx < d.nqt * ntl; idx += blockDim.x) {
                const int q = idx / ntl, a = idx % ntl;
                const long long h = (long long)c * d.nqt + q;
                const int sh = ft - d.Bt_first[h]; // 0 unless a point rounds onto a knot
                const int aa = a + sh;
                const bool ok = aa >= 0 && aa <= d.pt;
                tv[idx] = ok ? d.Bt_val[h * ntl + aa] : 0.0;
                td[idx] = ok ? d.Bt_der[h * ntl + aa] : 0.0;
            }
            for (int q = threadIdx.x; q < d.nqt; q += blockDim.x)
                w3[q] = d.cell_wts[(long long)c * d.nqt + q];
            __syncthreads();
            for (int ip = threadIdx.x; ip < el.nq2 * d.nqt; ip += blockDim.x) {
                const int q2 = ip / d.nqt, q3 = ip - q2 * d.nqt;
                double Gu[3][3] = {}, Gv[3][3] = {}; // [component][reference direction]
                for (int l = 0; l < nl3; ++l) {
                    const int at = l / el.nl2, as = l - at * el.nl2;
                    const double* g = gh + (q2 * el.nl2 + as) * 3;
                    const double T = tv[q3 * ntl + at], Td = td[q3 * ntl + at];
                    const double gx[3] = {g[0] * T, g[1] * T, g[2] * Td}; // (du T, dv T, val T')
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const double ua = cu[3 * l + a], va = cv[3 * l + a];
#pragma unroll
                        for (int x = 0; x < 3; ++x) {
                            Gu[a][x] += ua * gx[x];
                            Gv[a][x] += va * gx[x];
                        }
                    }
                }
                const double* C = ctq + q2 * 90;
                double form = 0.0;
#pragma unroll
                for (int x = 0; x < 3; ++x)
#pragma unroll
                    for (int y = 0; y < 3; ++y)
#pragma unroll
                        for (int a = 0; a < 3; ++a)
#pragma unroll
                            for (int b = 0; b < 3; ++b)
                                form += Gv[a][x] * C[(3 * x + y) * 10 + 3 * a + b] * Gu[b][y];
                acc += form * w3[q3];
            }
        }
    }
    // block reduction in a fixed order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            s += red[w];
        partial[bid] = s;
    }
}

__global__ void k_bilinear_final(const double* __restrict__ partial, long long n, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x)
        s += partial[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            t += red[w];
        *out = t;
    }
}

// ---------------------------------------------------------------------------
// K5: closed-form CSR pattern, slab-local row offsets.
__global__ void k_pattern_rows(const DevTables d, long long* __restrict__ row_ptr, long long rows) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > rows)
        return;
    if (r == rows) {
        row_ptr[rows] = d.rp_base + d.nnz_slab;
        return;
    }
    const long long g = d.f0 + r / 3; // function i_t * ns + i_s of row r
    const int it = (int)(g / d.ns), is = (int)(g % d.ns), a = (int)(r % 3);
    const int iu = is % d.nu, iv = is / d.nu;
    const int B = 3 * d.len_u[iu] * d.len_v[iv];
    const int Lt = d.len_t[it];
    row_ptr[r] = d.rp_base + 9 * d.S_s * (d.pre_t[it] - d.pre_t[d.t0]) +
                 (long long)Lt * (d.es_pre[is] + (long long)a * B) - d.out_base;
}

/// Columns of the slab's CSR.  Thread slots are warp-contiguous (a warp owns
/// 32 * kColsEpt consecutive entries, so its kColsEpt stores per (row, k) are
/// adjacent 128-byte runs) and the stores stream (st.global.cs).  16 entries
/// per thread on large slabs (C4 1.63 -> 1.45 ms), 8 on small ones (C2: 16
/// leaves too few blocks); profiles/r1_pattern_ept.txt.
template <int kColsEpt>
__global__ void __launch_bounds__(kBlock) k_pattern_cols(const DevTables d, int* __restrict__ cols,
                                                         int t_chunk) {
    // per entry: row-segment length B, offset in the segment, in-plane entry
    // base A (< E < 2^31, checked by the launcher) and column; 32-bit each
    int B[kColsEpt], col_s[kColsEpt], rem_x[kColsEpt], A[kColsEpt];
    // bit x: entry x is live / its function is >= s0 / < s1 (partial first and
    // last rows); packed so that 16 entries per thread stay within 255 registers
    // without spilling (three bool arrays took the C4 build from 1.44 to 2.2 ms)
    unsigned live = 0, in_s0 = 0, in_s1 = 0;
#pragma unroll
    for (int x = 0; x < kColsEpt; ++x) {
        const long long e = (long long)blockIdx.x * kBlock * kColsEpt + (threadIdx.x >> 5) * 32 * kColsEpt +
                            x * 32 + (threadIdx.x & 31);
        live |= (e < d.E ? 1u : 0u) << x;
        const long long ec = e < d.E ? e : d.E - 1;
        int is = __ldg(d.blk_is + ec / kBlock);
        while (__ldg(d.es_pre + is + 1) <= ec)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(ec - ebase);
        in_s0 |= (is >= d.s0 ? 1u : 0u) << x;
        in_s1 |= (is < d.s1 ? 1u : 0u) << x;
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        B[x] = 3 * Lu * Lv;
        const int a = r / B[x], rem = r - a * B[x];
        const int s = rem / 3, b = rem % 3;
        const int jv = __ldg(d.lo_v + iv) + s / Lu, ju = __ldg(d.lo_u + iu) + s % Lu;
        col_s[x] = 3 * (jv * d.nu + ju) + b;
        A[x] = (int)(ebase + (long long)a * B[x]);
        rem_x[x] = rem;
    }
    const int it_begin = d.t0 + blockIdx.y * t_chunk;
    const int it_end = min(d.t1, it_begin + t_chunk);
    const long long pre0 = __ldg(d.pre_t + d.t0);
    for (int it = it_begin; it < it_end; ++it) {
        const int Lt = __ldg(d.len_t + it);
        const long long base = 9 * d.S_s * (__ldg(d.pre_t + it) - pre0) - d.out_base;
        const int c0 = 3 * d.ns * __ldg(d.lo_t + it);
        const int edge = row_edge(d, it);
        const unsigned lv = live & ((edge & 1) ? in_s0 : ~0u) & ((edge & 2) ? in_s1 : ~0u);
#pragma unroll
        for (int x = 0; x < kColsEpt; ++x)
            LF_CHECK(!((lv >> x) & 1u) || (base + (long long)Lt * A[x] + rem_x[x] >= 0 &&
                                base + (long long)Lt * A[x] + (long long)(Lt - 1) * B[x] + rem_x[x] <
                                    d.nnz_slab));
        for (int k = 0; k < Lt; ++k) {
#pragma unroll
            for (int x = 0; x < kColsEpt; ++x)
                if ((lv >> x) & 1u)
                    __stcs(cols + base + (long long)Lt * A[x] + (long long)k * B[x] + rem_x[x],
                           c0 + 3 * d.ns * k + col_s[x]);
        }
    }
}

// ---------------------------------------------------------------------------
// K7: verification reductions (deterministic two-pass).
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    if (threadIdx.x < 32)
        for (int o = 16; o > 0; o >>= 1)
            v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__global__ void k_sumsq(const double* v, long long n, double* partial) {
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s += v[i] * v[i];
    s = block_sum(s);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = s;
}

__global__ void k_final_sum(const double* partial, int n, double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        s += partial[i];
    s = block_sum(s);
    if (threadIdx.x == 0)
        *out = s;
}

__global__ void k_spmv(long long rows, const long long* rp, const int* c, const double* v, const double* x,
                       double* y) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows)
        return;
    double s = 0.0;
    for (long long k = rp[r]; k < rp[r + 1]; ++k)
        s += v[k] * x[c[k]];
    y[r] = s;
}

__global__ void k_diff_rows(long long rows, const long long* ra, const int* ca, const double* va,
                            const long long* rb, const int* cb, const double* vb, double* partial) {
    double s = 0.0;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (long long)gridDim.x * blockDim.x) {
        long long ka = ra[r], kb = rb[r];
        const long long ea = ra[r + 1], eb = rb[r + 1];
        while (ka < ea || kb < eb) {
            const long long xa = ka < ea ? ca[ka] : (1LL << 40);
            const long long xb = kb < eb ? cb[kb] : (1LL << 40);
            double dd;
            if (xa == xb) {
                dd = va[ka++] - vb[kb++];
            } else if (xa < xb) {
                dd = va[ka++];
            } else {
                dd = -vb[kb++];
            }
            s += dd * dd;
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = s;
}

/// symmetryRelError numerator (sparse.cpp:73-95) of a CSR holding the rows
/// [row_begin, row_begin + rows) of a matrix: one warp per row, the row's
/// entries loaded coalesced, each lane's mirror found by a binary search of
/// its column's row.  Entries whose mirror row lies outside the rows held are
/// not counted (a row slab cannot see them); *outside counts them, so the
/// full-matrix entry point can reject a slab passed as a whole matrix.
__global__ void __launch_bounds__(256) k_symmetry_rows(long long rows, long long row_begin, const long long* rp,
                                                       const int* c, const double* v, double* partial,
                                                       unsigned long long* outside) {
    double s = 0.0;
    unsigned long long n_out = 0;
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w0; r < rows; r += nw) {
        const long long gr = r + row_begin;
        const long long k1 = __ldg(rp + r + 1);
        for (long long k = __ldg(rp + r) + lane; k < k1; k += 32) {
            const long long lr = (long long)__ldg(c + k) - row_begin;
            if (lr < 0 || lr >= rows) {
                ++n_out;
                continue;
            }
            long long lo = __ldg(rp + lr), hi = __ldg(rp + lr + 1);
            const long long end = hi;
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if ((long long)__ldg(c + mid) < gr)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            const bool mirrored = lo < end && (long long)__ldg(c + lo) == gr;
            const double dd = __ldg(v + k) - (mirrored ? __ldg(v + lo) : 0.0);
            s += dd * dd;
            if (!mirrored)
                s += dd * dd; // the structurally absent mirror slot counts too (sparse.cpp:87-90)
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = s;
    if (n_out)
        atomicAdd(outside, n_out);
}

/// Closed-form symmetry numerator of a plan's slab: one
/// thread per in-plane pair (i_s, slot) and thickness chunk.  For every
/// coupled block (i, j) with i <= j whose mirror row block j lies in the slab,
/// the 9 values of K_ij and the 9 of K_ji are read at their closed-form
/// positions and sum_ab (K_ij[a][b] - K_ji[b][a])^2 is added once for i = j
/// and twice for i < j (the reference visits both blocks).  The pattern is
/// structurally symmetric, so no mirror slot is absent.  Reads each value
/// once: consecutive threads take consecutive slots, so the K_ij rows load as
/// contiguous 768-byte runs per warp.
__global__ void __launch_bounds__(256) k_plan_symmetry(const DevTables d, const double* __restrict__ v,
                                                       int t_chunk, double* partial) {
    double s = 0.0;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; // in-plane pair
    if (q < d.S_s) {
        const long long e = 9 * q;
        int is = __ldg(d.blk_is + e / kBlock);
        while (__ldg(d.es_pre + is + 1) <= e)
            ++is;
        const int slot = (int)((e - __ldg(d.es_pre + is)) / 9);
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        const int sv = slot / Lu, su = slot - sv * Lu;
        const int ju = __ldg(d.lo_u + iu) + su, jv = __ldg(d.lo_v + iv) + sv;
        const int js = jv * d.nu + ju;
        const int Luj = __ldg(d.len_u + ju), Lvj = __ldg(d.len_v + jv);
        const int slot_m = (iv - __ldg(d.lo_v + jv)) * Luj + (iu - __ldg(d.lo_u + ju));
        const long long Bi = 3LL * Lu * Lv, Bj = 3LL * Luj * Lvj;
        const long long esi = __ldg(d.es_pre + is), esj = __ldg(d.es_pre + js);
        const long long pre0 = __ldg(d.pre_t + d.t0), nine_S = 9 * d.S_s;
        const int it0 = d.t0 + blockIdx.y * t_chunk, it1 = min(d.t1, it0 + t_chunk);
        for (int it = it0; it < it1; ++it) {
            const long long gi = (long long)it * d.ns + is;
            if (gi < d.f0 || gi >= d.f1)
                continue; // partial first / last row
            const int Lt = __ldg(d.len_t + it), lot = __ldg(d.lo_t + it);
            const long long base_i = nine_S * (__ldg(d.pre_t + it) - pre0) - d.out_base;
            for (int k = 0; k < Lt; ++k) {
                const int jt = lot + k;
                const long long gj = (long long)jt * d.ns + js;
                if (gj < d.f0 || gj >= d.f1)
                    continue; // mirror row block outside the slab
                if (gi > gj)
                    continue;
                const int Ltj = __ldg(d.len_t + jt);
                const long long base_j = nine_S * (__ldg(d.pre_t + jt) - pre0) - d.out_base;
                const double* own = v + base_i + (long long)Lt * esi + (long long)k * Bi + 3 * slot;
                const double* mir = v + base_j + (long long)Ltj * esj + (long long)(it - __ldg(d.lo_t + jt)) * Bj +
                                    3 * slot_m;
                double blk = 0.0;
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) {
                        const double x = __ldg(own + (long long)a * Lt * Bi + b);
                        const double y = __ldg(mir + (long long)b * Ltj * Bj + a);
                        blk += (x - y) * (x - y);
                    }
                s += gi == gj ? blk : 2.0 * blk;
            }
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0)
        partial[(long long)blockIdx.y * gridDim.x + blockIdx.x] = s;
}

int reduce_launch(int blocks, double* partial, double* out, cudaStream_t stream) {
    k_final_sum<<<1, 1024, 0, stream>>>(partial, blocks, out);
    return (int)cudaGetLastError();
}

} // namespace

int launch_integrals_1d(const DevTables& d, cudaStream_t stream) {
    const int n = d.nu * d.bu + d.nv * d.bv;
    k_integrals_1d<<<(n + 127) / 128, 128, 0, stream>>>(d);
    return (int)cudaGetLastError();
}

int launch_affine_export(const DevTables& d, cudaStream_t stream) {
    if (d.E == 0)
        return 0;
    k_affine_export<<<(unsigned)((d.E + kBlock - 1) / kBlock), kBlock, 0, stream>>>(d);
    return (int)cudaGetLastError();
}

int launch_inplane_general(const DevTables& d, cudaStream_t stream) {
    // two-phase: element-local P (one launch per term batch), then the gather
    const int nl2 = (d.pu + 1) * (d.pv + 1), nq2 = d.nqu * d.nqv;
    const size_t smem = sizeof(double) * ((size_t)nq2 * nl2 * 3 + nq2 + 1 + (size_t)nq2 * 90);
    const int threads = std::min(256, 4 * k2b_family_slots(nl2)); // one thread per (family, al, be group)
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_inplane_elem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned nel = (unsigned)(d.nspu * d.nspv);
    for (int t0 = 0; t0 < d.n_terms; t0 += d.pe_terms) {
        const int tb = std::min(d.pe_terms, d.n_terms - t0);
        k_inplane_elem<<<dim3(nel, (unsigned)tb), threads, smem, stream>>>(d, t0);
        const dim3 grid((unsigned)((d.E + kBlock - 1) / kBlock), (unsigned)tb);
        if (d.pu == d.pv && d.pu == 2)
            k_inplane_gather<2, 2><<<grid, kBlock, 0, stream>>>(d, t0);
        else if (d.pu == d.pv && d.pu == 3)
            k_inplane_gather<3, 3><<<grid, kBlock, 0, stream>>>(d, t0);
        else if (d.pu == d.pv && d.pu == 1)
            k_inplane_gather<1, 1><<<grid, kBlock, 0, stream>>>(d, t0);
        else if (d.pu == d.pv && d.pu == 4)
            k_inplane_gather<4, 4><<<grid, kBlock, 0, stream>>>(d, t0);
        else
            k_inplane_gather<0, 0><<<grid, kBlock, 0, stream>>>(d, t0);
    }
    return (int)cudaGetLastError();
}

int inplane_general_launches(const DevTables& d) { return 2 * ((d.n_terms + d.pe_terms - 1) / d.pe_terms); }

int launch_pattern(const DevTables& d, long long* row_ptr, int* cols, cudaStream_t stream) {
    const long long rows = 3 * (d.f1 - d.f0);
    if (d.E >= (1LL << 31))
        return (int)cudaErrorInvalidValue; // in-plane entry space beyond 32-bit offsets
    k_pattern_rows<<<(unsigned)((rows + 1 + 255) / 256), 256, 0, stream>>>(d, row_ptr, rows);
    if (cols && d.E > 0 && d.t1 > d.t0) { // cols == nullptr: row offsets only
        const int nt = d.t1 - d.t0;
        auto launch = [&](auto kern, int ept) {
            const long long nblk = (d.E + (long long)kBlock * ept - 1) / ((long long)kBlock * ept);
            long long nchunks = std::max(1LL, std::min<long long>((148LL * 16 + nblk - 1) / nblk, nt));
            const int t_chunk = (int)((nt + nchunks - 1) / nchunks);
            const dim3 grid((unsigned)nblk, (unsigned)((nt + t_chunk - 1) / t_chunk));
            kern<<<grid, kBlock, 0, stream>>>(d, cols, t_chunk);
        };
        const long long blocks16 = (d.E + kBlock * 16LL - 1) / (kBlock * 16LL) * nt;
        if (blocks16 >= 148LL * 32)
            launch(k_pattern_cols<16>, 16);
        else
            launch(k_pattern_cols<8>, 8);
    }
    return (int)cudaGetLastError();
}

int launch_standard(const DevTables& d, double* values, long long nnz, cudaStream_t stream, int* launches,
                    const K6Const* cst) {
    cudaMemsetAsync(values, 0, sizeof(double) * (size_t)nnz, stream);
    const int nl2 = (d.pu + 1) * (d.pv + 1), nq2 = d.nqu * d.nqv, ntl = d.pt + 1;
    const size_t smem = sizeof(double) * ((size_t)nq2 * nl2 * 3 + nq2 + 1 + (size_t)nq2 * 90 +
                                          2 * (size_t)d.nqt * ntl + d.nqt + 4 * (size_t)ntl * ntl);
    if (!d.Ks)
        return (int)cudaErrorInvalidValue; // the plan allocates the scratch for every standard assembly
    // two-phase: batches of ks_batch spans, local blocks then the gather
    const bool constc = cst && cst->n_cfg > 0;
    static const K6Const none{}; // n_cfg = 0
    const bool small = (d.pu + 1) * (d.pv + 1) * (d.pt + 1) <= 32; // nl3: p <= 2 layouts
    auto local = [&](auto kern, unsigned nel, int ks0, int nks) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<dim3(nel, (unsigned)nks), 256, smem, stream>>>(d, ks0, constc ? *cst : none);
    };
    // spans with a row in the slab
    int ks_lo = 0, ks_hi = d.nspt;
    while (ks_lo < d.nspt && d.spt_first_h[ks_lo] + d.pt < d.t0)
        ++ks_lo;
    while (ks_hi > ks_lo && d.spt_first_h[ks_hi - 1] >= d.t1)
        --ks_hi;
    const unsigned nel = (unsigned)(d.nspu * d.nspv);
    // batches aligned to absolute multiples of ks_batch (bitwise-identical sums on any slab)
    for (int ks0 = ks_lo; ks0 < ks_hi;) {
        const int ks1 = std::min(ks_hi, (ks0 / d.ks_batch + 1) * d.ks_batch);
        if (small)
            constc ? local(k_standard_local<true, 1, 4>, nel, ks0, ks1 - ks0)
                   : local(k_standard_local<false, 1, 4>, nel, ks0, ks1 - ks0);
        else
            constc ? local(k_standard_local<true, 2, 2>, nel, ks0, ks1 - ks0)
                   : local(k_standard_local<false, 2, 2>, nel, ks0, ks1 - ks0);
        // rows of the batch's spans inside the slab
        const int it_lo = std::max(d.t0, d.spt_first_h[ks0]);
        const int it_hi = std::min(d.t1, d.spt_first_h[ks1 - 1] + d.pt + 1);
        if (it_hi > it_lo) {
            const dim3 grid((unsigned)((d.S_s + 255) / 256), (unsigned)(it_hi - it_lo));
            k_standard_gather<<<grid, 256, 0, stream>>>(d, values, ks0, ks1, it_lo);
        }
        if (launches)
            *launches += 2;
        ks0 = ks1;
    }
    return (int)cudaGetLastError();
}

int launch_bilinear(const DevTables& d, const double* u, const double* v, double* partial, double* out,
                    cudaStream_t stream) {
    const int nl2 = (d.pu + 1) * (d.pv + 1), nq2 = d.nqu * d.nqv, ntl = d.pt + 1, nl3 = nl2 * ntl;
    const size_t smem = sizeof(double) * ((size_t)nq2 * nl2 * 3 + nq2 + 1 + (size_t)nq2 * 90 +
                                          2 * (size_t)d.nqt * ntl + d.nqt + 6 * (size_t)nl3 + 4 + 1);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_bilinear, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 grid(d.nspu, d.nspv, d.nspt);
    k_bilinear<<<grid, 128, smem, stream>>>(d, u, v, partial);
    k_bilinear_final<<<1, 1024, 0, stream>>>(partial, (long long)d.nspu * d.nspv * d.nspt, out);
    return (int)cudaGetLastError();
}

int launch_frobenius_sq(long long rows, const long long* rp, const double* v, double* out, cudaStream_t stream) {
    long long nnz = 0;
    cudaMemcpyAsync(&nnz, rp + rows, sizeof nnz, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    const int blocks = 1024;
    double* partial = nullptr;
    cudaMallocAsync(&partial, sizeof(double) * blocks, stream);
    k_sumsq<<<blocks, 256, 0, stream>>>(v, nnz, partial);
    reduce_launch(blocks, partial, out, stream);
    cudaFreeAsync(partial, stream);
    return (int)cudaGetLastError();
}

int launch_spmv(long long rows, const long long* rp, const int* c, const double* v, const double* x, double* y,
                cudaStream_t stream) {
    k_spmv<<<(unsigned)((rows + 255) / 256), 256, 0, stream>>>(rows, rp, c, v, x, y);
    return (int)cudaGetLastError();
}

int launch_diff_sq(long long rows, const long long* ra, const int* ca, const double* va, const long long* rb,
                   const int* cb, const double* vb, double* out, cudaStream_t stream) {
    const int blocks = 1024;
    double* partial = nullptr;
    cudaMallocAsync(&partial, sizeof(double) * blocks, stream);
    k_diff_rows<<<blocks, 256, 0, stream>>>(rows, ra, ca, va, rb, cb, vb, partial);
    reduce_launch(blocks, partial, out, stream);
    cudaFreeAsync(partial, stream);
    return (int)cudaGetLastError();
}

int launch_symmetry_sq(long long rows, long long row_begin, const long long* rp, const int* c, const double* v,
                       double* out, unsigned long long* outside, cudaStream_t stream) {
    const int blocks = 148 * 8;
    double* partial = nullptr;
    cudaMallocAsync(&partial, sizeof(double) * blocks, stream);
    cudaMemsetAsync(outside, 0, sizeof(unsigned long long), stream);
    k_symmetry_rows<<<blocks, 256, 0, stream>>>(rows, row_begin, rp, c, v, partial, outside);
    reduce_launch(blocks, partial, out, stream);
    cudaFreeAsync(partial, stream);
    return (int)cudaGetLastError();
}

int launch_plan_symmetry(const DevTables& d, const double* v, double* out, cudaStream_t stream) {
    const int nt = d.t1 - d.t0;
    if (d.S_s == 0 || nt <= 0) {
        cudaMemsetAsync(out, 0, sizeof(double), stream);
        return (int)cudaGetLastError();
    }
    const unsigned gx = (unsigned)((d.S_s + 255) / 256);
    // ~16 blocks per SM in total, chunks of whole thickness rows
    const int nchunk = (int)std::max(1LL, std::min<long long>(nt, (148LL * 16 + gx - 1) / gx));
    const int t_chunk = (nt + nchunk - 1) / nchunk;
    const unsigned gy = (unsigned)((nt + t_chunk - 1) / t_chunk);
    const int blocks = (int)(gx * gy);
    double* partial = nullptr;
    cudaMallocAsync(&partial, sizeof(double) * blocks, stream);
    k_plan_symmetry<<<dim3(gx, gy), 256, 0, stream>>>(d, v, t_chunk, partial);
    reduce_launch(blocks, partial, out, stream);
    cudaFreeAsync(partial, stream);
    return (int)cudaGetLastError();
}

} // namespace lfb
