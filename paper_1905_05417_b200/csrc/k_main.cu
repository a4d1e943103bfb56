// Main kernels of the B200 laminate assembler (sm_100a).
//
//  K2a k_integrals_1d     1D basis-product integrals U, V (sum-factorised P
//                         for affine geometry; fast.cpp:54-168 restated)
//  K2b k_inplane_general  per-element P for non-affine geometry, coloured
//                         (fast.cpp:54-168 / voigt_free.cpp:142-248)
//  K4  k_combine          P (x) q~ straight into the CSR value array
//                         (fast.cpp:211-264 + sparse.cpp:30-55)       <- hot
//  K5  k_pattern_*        closed-form CSR row offsets and columns
//  K6  k_standard         full 3D quadrature cross-check, coloured
//                         (assembly.cpp:134-245)
//  K7  verification       ||K||_F, K x, ||A-B||_F, ||K-K^T||_F (sparse.cpp:66-139)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "kernels.cuh"

namespace lfb {

namespace {

constexpr int kBlock = 256;

/// Output store of the combine kernel: st.global.cs (evict-first), the
/// values are written once and never re-read by this kernel (measured
/// 3.24 -> 3.15 ms on C4, profiles/round1.md).
__device__ __forceinline__ void store_value(double* p, double v) {
#ifdef LF_PLAIN_STORES
    *p = v;
#else
    __stcs(p, v);
#endif
}

__device__ __forceinline__ int find_is(const long long* es_pre, int ns, long long e) {
    int lo = 0, hi = ns; // es_pre[lo] <= e < es_pre[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(es_pre + mid) <= e)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

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

/// Affine P of one in-plane entry for `nt` terms starting at term t0:
/// P_{t,f}(a,b) = sum_{(x,y) in family f} Ct[t][3x+y][3a+b] * I_xy.
template <int NT>
__device__ __forceinline__ void affine_p(const DevTables& d, int iu, int iv, int su, int sv, int ab,
                                         int t0, double (&P)[NT][4]) {
    const double* U = d.U + ((long long)iu * d.bu + su) * 4;
    const double* V = d.V + ((long long)iv * d.bv + sv) * 4;
    const double u0 = __ldg(U), u1 = __ldg(U + 1), u2 = __ldg(U + 2), u3 = __ldg(U + 3);
    const double v0 = __ldg(V), v1 = __ldg(V + 1), v2 = __ldg(V + 2), v3 = __ldg(V + 3);
    // x -> (u-derivative, v-derivative): 0 -> (1,0) [d/du], 1 -> (0,1) [d/dv], 2 -> (0,0) [value]
    const double I00 = u3 * v0, I01 = u2 * v1, I10 = u1 * v2, I11 = u0 * v3;
    const double I02 = u2 * v0, I12 = u0 * v2, I20 = u1 * v0, I21 = u0 * v1, I22 = u0 * v0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const double* C = d.Ct + (long long)(t0 + t) * 81 + ab;
        P[t][0] = __ldg(C + 0) * I00 + __ldg(C + 9) * I01 + __ldg(C + 27) * I10 + __ldg(C + 36) * I11;
        P[t][1] = __ldg(C + 18) * I02 + __ldg(C + 45) * I12;
        P[t][2] = __ldg(C + 54) * I20 + __ldg(C + 63) * I21;
        P[t][3] = __ldg(C + 72) * I22;
    }
}

// ---------------------------------------------------------------------------
// K4: the hot kernel.  Each thread owns EPT in-plane entries (i_s, a, slot, b)
// (entries e and e + 256 of a 256*EPT block), keeps their P_{t,f} for the
// pass's terms in registers and streams over the thickness rows of its
// block-row chunk, writing one FP64 value per (entry, thickness pair).
// Consecutive lanes hold consecutive entries of one CSR row segment, so every
// warp store is a contiguous 256-byte run.
//
// Per staged sub-chunk of thickness rows, the pair weights (warp-uniform) sit
// in shared memory as s_w[row][k][term][4]; each row carries the union mask of
// its terms and, per term, the neighbour range [k_lo, k_hi) holding that
// term's contributing pairs.  A row is processed with a compile-time
// neighbour count (switch on L_t) so the accumulators stay in registers; a
// term absent from the row is a skipped uniform branch, and pairs outside the
// term's range are predicated off (no shared-memory wavefront, no FMA).  With
// EPT = 2 every weight load feeds two outputs.
struct RowInfo {
    long long base; // 9 S_s (pre_t[it] - pre_t[t0]): slab offset of row block it
    int lt;         // L_t(it)
    unsigned mask;  // union of term masks over the row's pairs (this pass)
};

template <int NT, int EPT, int LT, bool ACCUM, bool SMEM = false>
__device__ __forceinline__ void combine_row(const double (&P)[EPT][NT][4], const double4* __restrict__ w,
                                            unsigned mask, const unsigned char* __restrict__ kr,
                                            double* const (&o)[EPT], const int (&B)[EPT], const bool (&live)[EPT]) {
    double acc[EPT][LT];
#pragma unroll
    for (int x = 0; x < EPT; ++x)
#pragma unroll
        for (int k = 0; k < LT; ++k)
            acc[x][k] = (ACCUM && live[x]) ? o[x][(long long)k * B[x]] : 0.0;
#ifdef LF_STORE_ONLY
    // diagnostic build: identical store pattern, no weight loads / FMAs
    mask = 0;
#endif
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        if (mask & (1u << t)) {
            const int klo = kr[2 * t], khi = kr[2 * t + 1];
#pragma unroll
            for (int k = 0; k < LT; ++k) {
#ifdef LF_NO_KRANGE
                if (true) {
#else
                if (k >= klo && k < khi) {
#endif
                    const double4 ww = w[k * NT + t];
#pragma unroll
                    for (int x = 0; x < EPT; ++x) {
                        acc[x][k] = fma(P[x][t][0], ww.x, acc[x][k]);
                        acc[x][k] = fma(P[x][t][1], ww.y, acc[x][k]);
                        acc[x][k] = fma(P[x][t][2], ww.z, acc[x][k]);
                        acc[x][k] = fma(P[x][t][3], ww.w, acc[x][k]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < EPT; ++x)
        if (live[x])
#pragma unroll
            for (int k = 0; k < LT; ++k) {
                if constexpr (SMEM)
                    o[x][k * B[x]] = acc[x][k];
                else
                    store_value(o[x] + (long long)k * B[x], acc[x][k]);
            }
}

/// k-outer form of combine_row: one neighbour at a time, all its terms, then
/// the store -- EPT live accumulators instead of EPT * LT (register relief for
/// the wide variants).
template <int NT, int EPT, int LT, bool ACCUM>
__device__ __forceinline__ void combine_row_k(const double (&P)[EPT][NT][4], const double4* __restrict__ w,
                                              unsigned mask, const unsigned char* __restrict__ kr,
                                              double* const (&o)[EPT], const int (&B)[EPT], const bool (&live)[EPT]) {
    int klo[NT], khi[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        klo[t] = (mask & (1u << t)) ? kr[2 * t] : LT;
        khi[t] = kr[2 * t + 1];
    }
#pragma unroll
    for (int k = 0; k < LT; ++k) {
        double acc[EPT];
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            acc[x] = (ACCUM && live[x]) ? o[x][(long long)k * B[x]] : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (k >= klo[t] && k < khi[t]) {
                const double4 ww = w[k * NT + t];
#pragma unroll
                for (int x = 0; x < EPT; ++x) {
                    acc[x] = fma(P[x][t][0], ww.x, acc[x]);
                    acc[x] = fma(P[x][t][1], ww.y, acc[x]);
                    acc[x] = fma(P[x][t][2], ww.z, acc[x]);
                    acc[x] = fma(P[x][t][3], ww.w, acc[x]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            if (live[x])
                store_value(o[x] + (long long)k * B[x], acc[x]);
    }
}

template <int NT, int EPT, int LT, bool ACCUM>
__device__ __forceinline__ void row_dispatch(const double (&P)[EPT][NT][4], const double4* __restrict__ w,
                                             unsigned mask, const unsigned char* __restrict__ kr,
                                             double* const (&o)[EPT], const int (&B)[EPT], const bool (&live)[EPT]) {
    if constexpr (EPT >= 2)
        combine_row_k<NT, EPT, LT, ACCUM>(P, w, mask, kr, o, B, live);
    else
        combine_row<NT, EPT, LT, ACCUM>(P, w, mask, kr, o, B, live);
}

template <int NT, int EPT, bool ACCUM, bool SMEM = false>
__device__ __forceinline__ void combine_row_dyn(const double (&P)[EPT][NT][4], const double4* __restrict__ w,
                                                int lt, unsigned mask, double* const (&o)[EPT], const int (&B)[EPT],
                                                const bool (&live)[EPT]) {
    for (int k = 0; k < lt; ++k) {
        double acc[EPT];
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            acc[x] = (ACCUM && live[x]) ? o[x][(long long)k * B[x]] : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (mask & (1u << t)) {
                const double4 ww = w[k * NT + t];
#pragma unroll
                for (int x = 0; x < EPT; ++x) {
                    acc[x] = fma(P[x][t][0], ww.x, acc[x]);
                    acc[x] = fma(P[x][t][1], ww.y, acc[x]);
                    acc[x] = fma(P[x][t][2], ww.z, acc[x]);
                    acc[x] = fma(P[x][t][3], ww.w, acc[x]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            if (live[x]) {
                if constexpr (SMEM)
                    o[x][k * B[x]] = acc[x];
                else
                    store_value(o[x] + (long long)k * B[x], acc[x]);
            }
    }
}

/// Stages `nrow` thickness rows starting at it0 for the block: RowInfo, the
/// per-term neighbour ranges [k_lo, k_hi) and the weights s_w[row][k][term].
template <int NT>
__device__ __forceinline__ void stage_rows_block(const DevTables& d, int it0, int nrow, int pass, int lt_max,
                                                 RowInfo* s_row, unsigned char* s_kr, double4* s_w, int tid,
                                                 int nthreads) {
    const int t_first = pass * 8;
    const long long pre0 = __ldg(d.pre_t + d.t0);
    const long long nine_S = 9 * d.S_s;
    const unsigned* mask_base = d.Wmask + (long long)pass * d.n_pairs;
    const int T = d.n_terms;
    // stage rows: RowInfo, per-term neighbour ranges, weights s_w[row][k][t]
    for (int rr = tid; rr < nrow; rr += nthreads) {
        const int it = it0 + rr;
        const long long pfx = __ldg(d.pre_t + it) - pre0;
        const int lt = __ldg(d.len_t + it);
        unsigned m = 0;
        unsigned char lo[NT], hi[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            lo[t] = 255;
            hi[t] = 0;
        }
        for (int k = 0; k < lt; ++k) {
            const unsigned mk = __ldg(mask_base + pfx + k);
            m |= mk;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (mk & (1u << t)) {
                    lo[t] = min((int)lo[t], k);
                    hi[t] = (unsigned char)(k + 1);
                }
        }
        s_row[rr].base = nine_S * pfx;
        s_row[rr].lt = lt;
        s_row[rr].mask = m;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            s_kr[(rr * NT + t) * 2] = lo[t] == 255 ? 0 : lo[t];
            s_kr[(rr * NT + t) * 2 + 1] = hi[t];
        }
    }
    const int nw = nrow * lt_max * NT;
    for (int idx = tid; idx < nw; idx += nthreads) {
        const int rr = idx / (lt_max * NT);
        const int k = (idx / NT) % lt_max;
        const int t = idx % NT;
        const int it = it0 + rr;
        double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
        if (k < __ldg(d.len_t + it)) {
            const long long q = __ldg(d.pre_t + it) - pre0 + k;
            const double2* src = reinterpret_cast<const double2*>(d.W + ((q * T) + t_first + t) * 4);
            const double2 lo2 = __ldg(src), hi2 = __ldg(src + 1);
            v = make_double4(lo2.x, lo2.y, hi2.x, hi2.y);
        }
        s_w[idx] = v;
    }
}

template <int NT, int EPT, bool AFFINE, bool ACCUM, int BT>
__device__ __forceinline__ void combine_body(const DevTables& d, double* __restrict__ out, int pass, int t_chunk,
                                             int stage_rows, int lt_max) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RowInfo* s_row = reinterpret_cast<RowInfo*>(smem_raw);
    unsigned char* s_kr = smem_raw + stage_rows * sizeof(RowInfo); // [row][NT][2]
    double4* s_w = reinterpret_cast<double4*>(
        smem_raw + ((stage_rows * (sizeof(RowInfo) + 2 * NT) + 31) & ~31));

    const int t_first = pass * 8;
    double P[EPT][NT][4];
    double* o_thread[EPT];
    long long A[EPT];
    int B[EPT];
    bool live[EPT];
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
        // entry of slot x: 'strided' e = (blockIdx*EPT + x)*256 + tid, or
        // 'contiguous' (d.contig) e = blockIdx*256*EPT + warp*32*EPT + x*32 + lane,
        // where a warp's EPT stores per (row, k) are adjacent 256-byte runs
        const long long e = d.contig ? (long long)blockIdx.x * BT * EPT + (threadIdx.x >> 5) * 32 * EPT + x * 32 +
                                           (threadIdx.x & 31)
                                     : (long long)(blockIdx.x * EPT + x) * BT + threadIdx.x;
        live[x] = e < d.E;
        const long long ec = live[x] ? e : d.E - 1;
        int is = __ldg(d.blk_is + ec / kBlock);
        while (__ldg(d.es_pre + is + 1) <= ec)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(ec - ebase);
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        B[x] = 3 * Lu * Lv; // row segment length per thickness neighbour
        const int a = r / B[x];
        const int rem = r - a * B[x];
        A[x] = ebase + (long long)a * B[x];
        o_thread[x] = out + (long long)rem;
        if constexpr (AFFINE) {
            const int s = rem / 3, b = rem - 3 * (rem / 3);
            const int sv = s / Lu, su = s - sv * Lu;
            affine_p<NT>(d, iu, iv, su, sv, 3 * a + b, t_first, P[x]);
        } else {
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    P[x][t][f] = __ldg(d.Pg + ((long long)(t_first + t) * 4 + f) * d.E + ec);
        }
    }

    const int it_begin = d.t0 + blockIdx.y * t_chunk;
    const int it_end = min(d.t1, it_begin + t_chunk);
    bool any_live = false;
#pragma unroll
    for (int x = 0; x < EPT; ++x)
        any_live |= live[x];

    for (int it0 = it_begin; it0 < it_end; it0 += stage_rows) {
        const int nrow = min(stage_rows, it_end - it0);
        if (it0 != it_begin)
            __syncthreads();
        stage_rows_block<NT>(d, it0, nrow, pass, lt_max, s_row, s_kr, s_w, threadIdx.x, BT);
        __syncthreads();
        if (!any_live)
            continue;
        for (int rr = 0; rr < nrow; ++rr) {
            const RowInfo ri = s_row[rr];
            double* o[EPT];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                o[x] = o_thread[x] + ri.base + (long long)ri.lt * A[x];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                LF_CHECK(!live[x] || (o[x] >= out && o[x] + (long long)(ri.lt - 1) * B[x] < out + d.nnz_slab));
            const double4* w = s_w + rr * lt_max * NT;
            const unsigned char* kr = s_kr + rr * NT * 2;
            // EPT >= 2: k-outer rows (EPT live accumulators; C4 2.66 -> 2.53 ms,
            // C3 1.39 -> 1.33 ms with two entries per thread); EPT = 1: the
            // LT-unrolled form keeps more independent FMA chains in flight
            switch (ri.lt) {
            case 1: row_dispatch<NT, EPT, 1, ACCUM>(P, w, ri.mask, kr, o, B, live); break;
            case 2: row_dispatch<NT, EPT, 2, ACCUM>(P, w, ri.mask, kr, o, B, live); break;
            case 3: row_dispatch<NT, EPT, 3, ACCUM>(P, w, ri.mask, kr, o, B, live); break;
            case 4: row_dispatch<NT, EPT, 4, ACCUM>(P, w, ri.mask, kr, o, B, live); break;
            case 5: row_dispatch<NT, EPT, 5, ACCUM>(P, w, ri.mask, kr, o, B, live); break;
            case 7: row_dispatch<NT, EPT, 7, ACCUM>(P, w, ri.mask, kr, o, B, live); break;
            default: combine_row_dyn<NT, EPT, ACCUM>(P, w, ri.lt, ri.mask, o, B, live); break;
            }
        }
    }
}



// k_combine: 256-thread blocks and the compiler's own register choice (one
// entry per thread, 80-128 registers); k_combine_b: explicit bounds (two
// entries per thread, <= 128 registers so that 2 blocks of 256 fit per SM).
template <int NT, int EPT, bool AFFINE, bool ACCUM>
__global__ void __launch_bounds__(kBlock) k_combine(const DevTables d, double* __restrict__ out, int pass,
                                                    int t_chunk, int stage_rows, int lt_max) {
    combine_body<NT, EPT, AFFINE, ACCUM, kBlock>(d, out, pass, t_chunk, stage_rows, lt_max);
}

template <int NT, int EPT, bool AFFINE, bool ACCUM, int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB) k_combine_b(const DevTables d, double* __restrict__ out, int pass,
                                                        int t_chunk, int stage_rows, int lt_max) {
    combine_body<NT, EPT, AFFINE, ACCUM, BT>(d, out, pass, t_chunk, stage_rows, lt_max);
}

// ---------------------------------------------------------------------------
// K4, team/bulk variant (opt-in: LAMFAST_TEAM, see upload_teams in capi.cu).  The direct kernel above
// writes each warp's 32 values as a 256-byte run at 8-byte alignment: the CSR
// row segments are 3 L_s = 75 / 147 values long, so almost every warp store
// splits a 128-byte line with another warp, and that caps it near 85% of the
// HBM write rate (tools/store_pattern_bench.cu: 4.3-5.7 vs 7.1 TB/s).
//
// Here a team of `team` warps owns whole row-segment groups (i_s, a) of the
// entry space, packed up to 32*team*EPT entries (d.tm_e0 / d.tm_is).  For one
// thickness row the team's output is then ONE contiguous range of
// L_t * (e1 - e0) values.  The threads compute exactly as in k_combine but
// store into the team's shared-memory slot (3 slots, row i -> slot i % 3);
// after a team barrier one elected thread writes the range with a single
// cp.async.bulk (TMA bulk copy, 16-byte aligned body; an 8-byte head/tail,
// if any, with plain stores).  Slot reuse: after issuing row i the elected
// thread waits until at most one copy is still reading shared memory, i.e.
// the copy of row i-1 is done, before it reaches the barrier of row i+1; so
// when any thread starts row i+2 (slot (i+2)%3 = slot of row i-1) that slot
// is free.  Store-only microbenchmark: 7.1 TB/s (profiles/r1_store_modes.md).
__device__ __forceinline__ void team_barrier(int id, int nthreads) {
    if (nthreads == 32)
        __syncwarp();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void sts64(unsigned addr, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

/// Per-row record of the team kernel: code = L_t | mask << 8, kr = per term t
/// (k_lo | k_hi << 4) << 8t, base = slab offset of the row block.
struct TeamRow {
    unsigned code, kr;
    long long base;
};

/// One thickness row of the team kernel.  `code` and `kr` are broadcast from
/// lane 0 so the compiler treats them as warp-uniform: the term / neighbour
/// tests become uniform branches instead of divergent ones.  Stores are
/// unconditional (dead entries write to a scratch line of the slot).
template <int NT, int EPT, int LT, bool KR>
__device__ __forceinline__ void team_row(const double (&P)[EPT][NT][4], const double4* __restrict__ w, unsigned mask,
                                         unsigned kr, const unsigned (&o)[EPT], const unsigned (&Bb)[EPT]) {
    double acc[EPT][LT];
#pragma unroll
    for (int x = 0; x < EPT; ++x)
#pragma unroll
        for (int k = 0; k < LT; ++k)
            acc[x][k] = 0.0;
#ifdef LF_STORE_ONLY
    mask = 0; // diagnostic build: identical stores, no weight loads / FMAs
#endif
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        if (mask & (1u << t)) {
            const unsigned klo = (kr >> (8 * t)) & 15u, khi = (kr >> (8 * t + 4)) & 15u;
#pragma unroll
            for (int k = 0; k < LT; ++k) {
                if (!KR || (k >= (int)klo && k < (int)khi)) {
                    const double4 ww = w[k * NT + t];
#pragma unroll
                    for (int x = 0; x < EPT; ++x) {
                        acc[x][k] = fma(P[x][t][0], ww.x, acc[x][k]);
                        acc[x][k] = fma(P[x][t][1], ww.y, acc[x][k]);
                        acc[x][k] = fma(P[x][t][2], ww.z, acc[x][k]);
                        acc[x][k] = fma(P[x][t][3], ww.w, acc[x][k]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < EPT; ++x)
#pragma unroll
        for (int k = 0; k < LT; ++k)
            sts64(o[x] + k * Bb[x], acc[x][k]);
}

template <int NT, int EPT>
__device__ __forceinline__ void team_row_dyn(const double (&P)[EPT][NT][4], const double4* __restrict__ w, int lt,
                                             unsigned mask, const unsigned (&o)[EPT], const unsigned (&Bb)[EPT]) {
    for (int k = 0; k < lt; ++k) {
        double acc[EPT];
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            acc[x] = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (mask & (1u << t)) {
                const double4 ww = w[k * NT + t];
#pragma unroll
                for (int x = 0; x < EPT; ++x) {
                    acc[x] = fma(P[x][t][0], ww.x, acc[x]);
                    acc[x] = fma(P[x][t][1], ww.y, acc[x]);
                    acc[x] = fma(P[x][t][2], ww.z, acc[x]);
                    acc[x] = fma(P[x][t][3], ww.w, acc[x]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            sts64(o[x] + k * Bb[x], acc[x]);
    }
}

/// Stages `nrow` rows for the team kernel: TeamRow records and the weights
/// s_w[row][k][term] (zero beyond L_t).
template <int NT>
__device__ __forceinline__ void stage_team_rows(const DevTables& d, int it0, int nrow, int lt_max, TeamRow* s_row,
                                                double4* s_w, int tid, int nthreads) {
    const long long pre0 = __ldg(d.pre_t + d.t0);
    for (int rr = tid; rr < nrow; rr += nthreads) {
        const int it = it0 + rr;
        const long long pfx = __ldg(d.pre_t + it) - pre0;
        const int lt = __ldg(d.len_t + it);
        unsigned m = 0, kr = 0;
        int lo[NT], hi[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            lo[t] = 15;
            hi[t] = 0;
        }
        for (int k = 0; k < lt; ++k) {
            const unsigned mk = __ldg(d.Wmask + pfx + k);
            m |= mk;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (mk & (1u << t)) {
                    lo[t] = min(lo[t], k);
                    hi[t] = k + 1;
                }
        }
#pragma unroll
        for (int t = 0; t < NT; ++t)
            kr |= (unsigned)((lo[t] == 15 ? 0 : lo[t]) | (hi[t] << 4)) << (8 * t);
        TeamRow r;
        r.code = (unsigned)lt | (m << 8);
        r.kr = kr;
        r.base = 9 * d.S_s * pfx;
        s_row[rr] = r;
    }
    const int T = d.n_terms;
    const int nw = nrow * lt_max * NT;
    for (int idx = tid; idx < nw; idx += nthreads) {
        const int rr = idx / (lt_max * NT);
        const int k = (idx / NT) % lt_max;
        const int t = idx % NT;
        const int it = it0 + rr;
        double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
        if (k < __ldg(d.len_t + it)) {
            const long long q = __ldg(d.pre_t + it) - pre0 + k;
            const double2* src = reinterpret_cast<const double2*>(d.W + ((q * T) + t) * 4);
            const double2 lo2 = __ldg(src), hi2 = __ldg(src + 1);
            v = make_double4(lo2.x, lo2.y, hi2.x, hi2.y);
        }
        s_w[idx] = v;
    }
}

template <int NT, int EPT, bool AFFINE, bool KR>
__global__ void __launch_bounds__(kBlock) k_combine_team(const DevTables d, double* __restrict__ out, int t_chunk,
                                                          int stage_rows, int lt_max, int team, int slot_len) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nthreads = blockDim.x;
    TeamRow* s_row = reinterpret_cast<TeamRow*>(smem_raw);
    double4* s_w = reinterpret_cast<double4*>(smem_raw + ((stage_rows * sizeof(TeamRow) + 31) & ~size_t(31)));
    double* s_slots = reinterpret_cast<double*>(s_w + stage_rows * lt_max * NT);

    const int team_threads = team * 32;
    const int tib = threadIdx.x / team_threads; // team index in the block
    const int tl = threadIdx.x - tib * team_threads;
    const long long tm = (long long)blockIdx.x * (nthreads / team_threads) + tib;
    const bool team_live = tm < d.n_team;
    const long long e0 = team_live ? __ldg(d.tm_e0 + tm) : 0;
    const long long e1 = team_live ? __ldg(d.tm_e0 + tm + 1) : 0;
    const int ne = (int)(e1 - e0);
    // 3 slots of slot_len doubles; the last 32*team doubles of each slot are
    // the scratch line that dead entries write to
    double* slots = s_slots + (size_t)tib * 3 * slot_len;
    const unsigned slots_sh = (unsigned)__cvta_generic_to_shared(slots);
    const int bar_id = 1 + tib;
    const bool elected = tl == 0;

    double P[EPT][NT][4];
    unsigned loc[EPT], rem8[EPT], Bb[EPT]; // group start, 8*rem, 8*B (0 for dead entries)
    int is = team_live ? __ldg(d.tm_is + tm) : 0;
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
        const long long e = e0 + tl + (long long)x * team_threads;
        const bool live = e < e1;
        const long long ec = live ? e : (team_live ? e1 - 1 : 0);
        while (__ldg(d.es_pre + is + 1) <= ec)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(ec - ebase);
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        const int B = 3 * Lu * Lv;
        const int a = r / B;
        const int rem = r - a * B;
        loc[x] = live ? (unsigned)(ebase + (long long)a * B - e0) : 0u;
        rem8[x] = live ? 8u * rem : 8u * (slot_len - team_threads + tl);
        Bb[x] = live ? 8u * B : 0u;
        if constexpr (AFFINE) {
            const int s = rem / 3, b = rem - 3 * (rem / 3);
            const int sv = s / Lu, su = s - sv * Lu;
            affine_p<NT>(d, iu, iv, su, sv, 3 * a + b, 0, P[x]);
        } else {
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    P[x][t][f] = __ldg(d.Pg + ((long long)t * 4 + f) * d.E + ec);
        }
    }
    // dead entries must not be scaled by L_t: their loc is 0, rem8 the scratch

    const int it_begin = d.t0 + blockIdx.y * t_chunk;
    const int it_end = min(d.t1, it_begin + t_chunk);
    int slot_i = 0; // slot ring position
    for (int it0 = it_begin; it0 < it_end; it0 += stage_rows) {
        const int nrow = min(stage_rows, it_end - it0);
        if (it0 != it_begin)
            __syncthreads();
        stage_team_rows<NT>(d, it0, nrow, lt_max, s_row, s_w, threadIdx.x, nthreads);
        __syncthreads();
        if (!team_live)
            continue;
        for (int rr = 0; rr < nrow; ++rr) {
            const TeamRow ri = s_row[rr];
            // warp-uniform copies (lane 0 broadcast) for the branch structure
            const unsigned code = __shfl_sync(0xffffffffu, ri.code, 0);
            const unsigned kr = __shfl_sync(0xffffffffu, ri.kr, 0);
            const int lt = (int)(code & 255u);
            const unsigned mask = code >> 8;
            double* gdst = out + ri.base + (long long)lt * e0;
            const unsigned par = (unsigned)(reinterpret_cast<uintptr_t>(gdst) >> 3) & 1u; // 16-byte phase
            const unsigned slot = slots_sh + 8u * ((unsigned)slot_i * (unsigned)slot_len + par);
            unsigned o[EPT];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                o[x] = slot + 8u * (unsigned)lt * loc[x] + rem8[x] - (Bb[x] ? 0u : 8u * par);
            const double4* w = s_w + rr * lt_max * NT;
            switch (lt) {
            case 1: team_row<NT, EPT, 1, KR>(P, w, mask, kr, o, Bb); break;
            case 2: team_row<NT, EPT, 2, KR>(P, w, mask, kr, o, Bb); break;
            case 3: team_row<NT, EPT, 3, KR>(P, w, mask, kr, o, Bb); break;
            case 4: team_row<NT, EPT, 4, KR>(P, w, mask, kr, o, Bb); break;
            case 5: team_row<NT, EPT, 5, KR>(P, w, mask, kr, o, Bb); break;
            case 7: team_row<NT, EPT, 7, KR>(P, w, mask, kr, o, Bb); break;
            default: team_row_dyn<NT, EPT>(P, w, lt, mask, o, Bb); break;
            }
            // generic-proxy smem writes -> visible to the bulk-copy (async) proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            team_barrier(bar_id, team_threads);
            if (elected) {
                const double* sl = slots + (size_t)slot_i * slot_len + par;
                const int n = lt * ne;
                const int nb = (n - (int)par) & ~1; // 16-byte body
                if (par)
                    __stcs(gdst, sl[0]);
                if (n - (int)par - nb)
                    __stcs(gdst + n - 1, sl[n - 1]);
                if (nb > 0) {
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst + par),
                                 "r"(slot + 8u * par), "r"(nb * 8)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            slot_i = slot_i == 2 ? 0 : slot_i + 1;
        }
    }
    if (elected)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// K4, warp-specialised variant (default when the row segments pack): the
// direct-store k_combine writes each warp's 32 values as a 256-byte run at
// 8-byte alignment, and that misalignment -- not the access order -- is what
// keeps it below the fill rate (tools/store_pattern_bench.cu: 4.3 vs 7.1 TB/s).
// Here every block owns whole CSR row-segment groups (all entries (a, slot, b)
// of one row segment of i_s), so its output for one thickness row is ONE
// contiguous range of L_t x (#entries) values.
//   * NP producer warps (EPT entries per thread, P in registers) compute a
//     row and write it into a shared-memory copy of that range (slot of a
//     3-deep ring, lanes -> consecutive words);
//   * NC consumer warps stream the slot out with 16-byte stores aligned to
//     128-byte lines (scalar head/tail), st.global.cs;
//   * slots are handed over with named barriers (bar.arrive / bar.sync):
//     FULL[s] = 1 + s, EMPTY[s] = 4 + s -- no block-wide barrier in the loop.
// Weights of the whole row chunk are staged once, before the roles split.
constexpr int kWsSlots = 3;

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Per-row data of the combine in the constant bank.  A combine launch covers
// a segment of thickness rows whose image fits here; the producers read the
// weights with uniform loads (LDCU into uniform registers, consumed directly
// by DFMA): no shared-memory or LSU traffic for the warp-uniform weights.
struct RowC {
    long long base;          // 9 S_s (pre_t[it] - pre_t[t0])
    int lt;                  // L_t(it)
    unsigned mask;           // union of term masks over the row's pairs
    unsigned char kr[16];    // per term: neighbour range [k_lo, k_hi)
};
constexpr int kConstRows = 256;
constexpr int kConstW = 1600; // double4 -> 51.2 KB
__constant__ RowC c_rows[kConstRows];
__constant__ double4 c_w[kConstW];

/// Packs RowC and the padded weights [row][k][term] of the slab into global
/// images (copied per segment into the constant bank).
__global__ void k_pack_rows(const DevTables d, RowC* __restrict__ g_rows, double4* __restrict__ g_w, int nt,
                            int lt_max) {
    const int nrow = d.t1 - d.t0;
    const long long pre0 = d.pre_t[d.t0];
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int nw = nrow * lt_max * nt;
    if (idx < nw) {
        const int rr = idx / (lt_max * nt), k = (idx / nt) % lt_max, t = idx % nt;
        const int it = d.t0 + rr;
        double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
        if (k < d.len_t[it]) {
            const long long q = d.pre_t[it] - pre0 + k;
            const double* src = d.W + (q * d.n_terms + t) * 4;
            v = make_double4(src[0], src[1], src[2], src[3]);
        }
        g_w[idx] = v;
    }
    if (idx < nrow) {
        const int it = d.t0 + idx;
        const long long pfx = d.pre_t[it] - pre0;
        const int lt = d.len_t[it];
        RowC r;
        r.base = 9 * d.S_s * pfx;
        r.lt = lt;
        unsigned m = 0;
        for (int t = 0; t < 16; ++t)
            r.kr[t] = 0;
        for (int t = 0; t < nt && t < 8; ++t) {
            int lo = 255, hi = 0;
            for (int k = 0; k < lt; ++k)
                if (d.Wmask[pfx + k] & (1u << t)) {
                    lo = min(lo, k);
                    hi = k + 1;
                }
            if (hi > 0)
                m |= 1u << t;
            r.kr[2 * t] = (unsigned char)(lo == 255 ? 0 : lo);
            r.kr[2 * t + 1] = (unsigned char)hi;
        }
        r.mask = m;
        g_rows[idx] = r;
    }
}

template <int NT, int EPT, int LT>
__device__ __forceinline__ void combine_row_const(const double (&P)[EPT][NT][4], int wbase, const RowC& ri,
                                                  double* sbuf, const int (&loc)[EPT], const int (&rem)[EPT],
                                                  const int (&B)[EPT], const bool (&live)[EPT]) {
    double acc[EPT][LT];
#pragma unroll
    for (int x = 0; x < EPT; ++x)
#pragma unroll
        for (int k = 0; k < LT; ++k)
            acc[x][k] = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        if (ri.mask & (1u << t)) {
            const int klo = ri.kr[2 * t], khi = ri.kr[2 * t + 1];
#pragma unroll
            for (int k = 0; k < LT; ++k) {
                if (k >= klo && k < khi) {
                    const double4 ww = c_w[wbase + k * NT + t];
#pragma unroll
                    for (int x = 0; x < EPT; ++x) {
                        acc[x][k] = fma(P[x][t][0], ww.x, acc[x][k]);
                        acc[x][k] = fma(P[x][t][1], ww.y, acc[x][k]);
                        acc[x][k] = fma(P[x][t][2], ww.z, acc[x][k]);
                        acc[x][k] = fma(P[x][t][3], ww.w, acc[x][k]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int x = 0; x < EPT; ++x)
        if (live[x])
#pragma unroll
            for (int k = 0; k < LT; ++k)
                sbuf[LT * loc[x] + k * B[x] + rem[x]] = acc[x][k];
}

template <int NT, int EPT>
__device__ __forceinline__ void combine_row_const_dyn(const double (&P)[EPT][NT][4], int wbase, const RowC& ri,
                                                      double* sbuf, const int (&loc)[EPT], const int (&rem)[EPT],
                                                      const int (&B)[EPT], const bool (&live)[EPT]) {
    for (int k = 0; k < ri.lt; ++k) {
        double acc[EPT];
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            acc[x] = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (ri.mask & (1u << t)) {
                const double4 ww = c_w[wbase + k * NT + t];
#pragma unroll
                for (int x = 0; x < EPT; ++x) {
                    acc[x] = fma(P[x][t][0], ww.x, acc[x]);
                    acc[x] = fma(P[x][t][1], ww.y, acc[x]);
                    acc[x] = fma(P[x][t][2], ww.z, acc[x]);
                    acc[x] = fma(P[x][t][3], ww.w, acc[x]);
                }
            }
        }
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            if (live[x])
                sbuf[ri.lt * loc[x] + k * B[x] + rem[x]] = acc[x];
    }
}

/// Warp-specialised combine over the segment of rows [seg_r0, seg_r0 +
/// seg_rows) of the slab (row data in the constant bank, chunked by y).
template <int NT, int EPT, int NP, int NC, bool AFFINE>
__global__ void __launch_bounds__((NP + NC) * 32) k_combine_ws(const DevTables d, double* __restrict__ out,
                                                               int seg_rows, int t_chunk, int lt_max) {
    constexpr int kProd = NP * 32, kAll = (NP + NC) * 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int slot_len = lt_max * kProd * EPT + 2;
    double* s_out = reinterpret_cast<double*>(smem_raw);

    const long long e0 = __ldg(d.gbw_e0 + blockIdx.x), e1 = __ldg(d.gbw_e0 + blockIdx.x + 1);
    const int ne = (int)(e1 - e0);
    const int r_begin = blockIdx.y * t_chunk; // local to the segment
    const int r_end = min(seg_rows, r_begin + t_chunk);
    const int nrow = r_end - r_begin;
    // warp index made provably warp-uniform, so the role branches stay on the
    // uniform datapath (constant-bank weights via LDCU -> uniform registers)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);

    if (warp < NP) {
        // ---- producers ----
        double P[EPT][NT][4];
        int loc[EPT], rem[EPT], B[EPT];
        bool live[EPT];
        int is = __ldg(d.gbw_is + blockIdx.x);
#pragma unroll
        for (int x = 0; x < EPT; ++x) {
            const long long e = e0 + x * kProd + threadIdx.x;
            live[x] = e < e1;
            const long long ec = live[x] ? e : e1 - 1;
            while (__ldg(d.es_pre + is + 1) <= ec)
                ++is;
            const long long ebase = __ldg(d.es_pre + is);
            const int r = (int)(ec - ebase);
            const int iu = is % d.nu, iv = is / d.nu;
            const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
            B[x] = 3 * Lu * Lv;
            const int a = r / B[x];
            rem[x] = r - a * B[x];
            // (row, k) position inside the block's range: L_t * loc + k * B + rem
            loc[x] = (int)(ebase + (long long)a * B[x] - e0);
            if constexpr (AFFINE) {
                const int s = rem[x] / 3, b = rem[x] - 3 * (rem[x] / 3);
                const int sv = s / Lu, su = s - sv * Lu;
                affine_p<NT>(d, iu, iv, su, sv, 3 * a + b, 0, P[x]);
            } else {
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int f = 0; f < 4; ++f)
                        P[x][t][f] = __ldg(d.Pg + ((long long)t * 4 + f) * d.E + ec);
            }
        }
        for (int i = 0; i < nrow; ++i) {
            const int slot = i % kWsSlots;
            if (i >= kWsSlots)
                named_sync(1 + kWsSlots + slot, kAll); // consumers released the slot
            const int rr = r_begin + i;
            const RowC ri = c_rows[rr];
            const long long dst = ri.base + (long long)ri.lt * e0;
            double* sbuf = s_out + (size_t)slot * slot_len + (int)((reinterpret_cast<uintptr_t>(out + dst) >> 3) & 1);
            const int wbase = rr * lt_max * NT;
            switch (ri.lt) {
            case 1: combine_row_const<NT, EPT, 1>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            case 2: combine_row_const<NT, EPT, 2>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            case 3: combine_row_const<NT, EPT, 3>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            case 4: combine_row_const<NT, EPT, 4>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            case 5: combine_row_const<NT, EPT, 5>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            case 7: combine_row_const<NT, EPT, 7>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            default: combine_row_const_dyn<NT, EPT>(P, wbase, ri, sbuf, loc, rem, B, live); break;
            }
            named_arrive(1 + slot, kAll); // slot full
        }
    } else {
        // ---- consumers: 128-byte aligned 16-byte stores of each full slot ----
        const int ct = threadIdx.x - kProd;
        for (int i = 0; i < nrow; ++i) {
            const int slot = i % kWsSlots;
            named_sync(1 + slot, kAll);
            const RowC ri = c_rows[r_begin + i];
            const long long dst = ri.base + (long long)ri.lt * e0;
            const long long phase = (long long)((reinterpret_cast<uintptr_t>(out + dst) >> 3) & 15); // in doubles
            const double* sbuf = s_out + (size_t)slot * slot_len + (int)(phase & 1);
            const int n = ri.lt * ne;
            double* g = out + dst;
            const int head = (int)min((long long)n, (16 - phase) & 15);
            if (ct < head)
                __stcs(g + ct, sbuf[ct]);
            const int body = (n - head) >> 1;
            const double2* sv = reinterpret_cast<const double2*>(sbuf + head);
            double2* gv = reinterpret_cast<double2*>(g + head);
            int v = ct;
            for (; v + 3 * NC * 32 < body; v += 4 * NC * 32) { // 4 loads in flight per lane
                const double2 a0 = sv[v], a1 = sv[v + NC * 32], a2 = sv[v + 2 * NC * 32], a3 = sv[v + 3 * NC * 32];
                __stcs(gv + v, a0);
                __stcs(gv + v + NC * 32, a1);
                __stcs(gv + v + 2 * NC * 32, a2);
                __stcs(gv + v + 3 * NC * 32, a3);
            }
            for (; v < body; v += NC * 32)
                __stcs(gv + v, sv[v]);
            if (((n - head) & 1) && ct == NC * 32 - 1)
                __stcs(g + n - 1, sbuf[n - 1]);
            if (i + kWsSlots < nrow)
                named_arrive(1 + kWsSlots + slot, kAll); // slot free
        }
    }
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

// K2b: in-plane operators of every term for one element colour.  Elements of
// one colour share no basis function, so plain += is race-free and the
// result is deterministic.
__global__ void k_inplane_general(const DevTables d, int cu, int cv) {
    extern __shared__ double sm[];
    ElemInfo el;
    el.eu = cu + blockIdx.x * (d.pu + 1);
    el.ev = cv + blockIdx.y * (d.pv + 1);
    if (el.eu >= d.nspu || el.ev >= d.nspv)
        return;
    el.fu = d.spu_first[el.eu];
    el.fv = d.spv_first[el.ev];
    el.nl2 = (d.pu + 1) * (d.pv + 1);
    el.nq2 = d.nqu * d.nqv;
    el.hu = 0.5 * (d.spu_hi[el.eu] - d.spu_lo[el.eu]);
    el.hv = 0.5 * (d.spv_hi[el.ev] - d.spv_lo[el.ev]);
    double* gh = sm;                    // nq2 * nl2 * 3
    double* w2 = gh + el.nq2 * el.nl2 * 3; // nq2
    double* ctq = sm + ((el.nq2 * el.nl2 * 3 + el.nq2 + 1) & ~1); // nq2 * 90, 16-byte aligned
    element_tables(d, el, gh, w2);
    const int e_index = el.ev * d.nspu + el.eu;
    {
        const int t = blockIdx.z; // one block per (element, term): 4x the blocks per colour
        __syncthreads();
        pullback_tables(d, e_index, el.nq2, w2, d.term_table + (long long)t * 81, ctq);
        __syncthreads();
        // one thread per (local pair, family f): 9 accumulators and a 9-value
        // read-modify-write each, so many more warps hide the latency of the
        // coloured accumulation into Pg (the bound of this kernel).  Threads of
        // a warp share f (warp-aligned quarters), so the C~ loads broadcast.
        const int npair = el.nl2 * el.nl2;
        const int qstride = (npair + 31) & ~31;
        for (int idx = threadIdx.x; idx < 4 * qstride; idx += blockDim.x) {
            const int f = idx / qstride;
            const int pr = idx - f * qstride;
            if (pr >= npair)
                continue;
            const int al = pr / el.nl2, be = pr % el.nl2;
            // P11 <- C~00,01,10,11; P12 <- 02,12; P21 <- 20,21; P22 <- 22 (layout [q][xy][10])
            const int nxy = f == 0 ? 4 : f == 3 ? 1 : 2;
            int xys[4];
            xys[0] = f == 0 ? 0 : f == 1 ? 2 : f == 2 ? 6 : 8;
            xys[1] = f == 0 ? 1 : f == 1 ? 5 : 7;
            xys[2] = 3;
            xys[3] = 4;
            double acc[9];
#pragma unroll
            for (int k = 0; k < 9; ++k)
                acc[k] = 0.0;
            for (int q = 0; q < el.nq2; ++q) {
                const double* ga = gh + (q * el.nl2 + al) * 3;
                const double* gb = gh + (q * el.nl2 + be) * 3;
                const double* C = ctq + q * 90;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (u < nxy) {
                        const int xy = xys[u];
                        const double sxy = ga[xy / 3] * gb[xy % 3];
                        const double2* C2 = reinterpret_cast<const double2*>(C + xy * 10);
#pragma unroll
                        for (int h = 0; h < 5; ++h) {
                            const double2 c = C2[h];
                            acc[2 * h] += c.x * sxy;
                            if (2 * h + 1 < 9)
                                acc[2 * h + 1] += c.y * sxy;
                        }
                    }
                }
            }
            const int iu = el.fu + al % (d.pu + 1), iv = el.fv + al / (d.pu + 1);
            const int ju = el.fu + be % (d.pu + 1), jv = el.fv + be / (d.pu + 1);
            const int is = iv * d.nu + iu;
            const int Lu = d.len_u[iu], Lv = d.len_v[iv];
            const int slot = (jv - d.lo_v[iv]) * Lu + (ju - d.lo_u[iu]);
            const long long base = d.es_pre[is] + 3 * slot;
            const int B = 3 * Lu * Lv;
            double* dst = d.Pg + ((long long)t * 4 + f) * d.E + base;
            LF_CHECK(base >= 0 && base + 2LL * B + 2 < d.E && t < d.n_terms);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    dst[(long long)a * B + b] += acc[3 * a + b];
        }
    }
}

// ---------------------------------------------------------------------------
// K6: standard full-3D quadrature (assembly.cpp:134-245), one block per
// (element, thickness span) of one colour, accumulated straight into the
// precomputed CSR (the duplicate summation of sparse.cpp:30-55).
__global__ void k_standard(const DevTables d, double* __restrict__ values, int cu, int cv, int ct, int nchunk) {
    extern __shared__ double sm[];
    ElemInfo el;
    el.eu = cu + blockIdx.x * (d.pu + 1);
    el.ev = cv + blockIdx.y * (d.pv + 1);
    // blockIdx.z = (span of this thickness colour, chunk of the local pairs):
    // few elements per colour (small plates, many plies per span) still fill
    // the GPU; chunks own disjoint pairs, so their writes never overlap
    const int chunk = blockIdx.z % nchunk;
    const int ks = ct + (blockIdx.z / nchunk) * (d.pt + 1);
    if (el.eu >= d.nspu || el.ev >= d.nspv || ks >= d.nspt)
        return;
    const int c0 = d.span_cell0[ks], c1 = d.span_cell0[ks + 1];
    if (c0 == c1)
        return; // span with no unmasked cell (assembly.cpp:185-186)
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
    double* tv = ctq + el.nq2 * 90; // nqt * ntl values, then derivatives
    double* td = tv + d.nqt * ntl;
    double* w3 = td + d.nqt * ntl;
    element_tables(d, el, gh, w2);
    const int e_index = el.ev * d.nspu + el.eu;
    const long long pre0 = d.pre_t[d.t0];
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
        const int npair = d.sym ? nl3 * (nl3 + 1) / 2 : nl3 * nl3;
        const int per = (npair + nchunk - 1) / nchunk;
        const int p_end = min(npair, (chunk + 1) * per);
        for (int pr = chunk * per + threadIdx.x; pr < p_end; pr += blockDim.x) {
            int al, be;
            if (d.sym) { // triangular index: be >= al
                al = 0;
                int rest = pr;
                while (rest >= nl3 - al) {
                    rest -= nl3 - al;
                    ++al;
                }
                be = al + rest;
            } else {
                al = pr / nl3;
                be = pr % nl3;
            }
            const int at = al / el.nl2, as = al % el.nl2;
            const int bt = be / el.nl2, bs = be % el.nl2;
            const int it = ft + at, jt = ft + bt;
            const bool row_i = it >= d.t0 && it < d.t1;
            const bool row_j = d.sym && al != be && jt >= d.t0 && jt < d.t1;
            if (!row_i && !row_j)
                continue;
            double acc[9];
#pragma unroll
            for (int k = 0; k < 9; ++k)
                acc[k] = 0.0;
            for (int q2 = 0; q2 < el.nq2; ++q2) {
                const double* ga = gh + (q2 * el.nl2 + as) * 3;
                const double* gb = gh + (q2 * el.nl2 + bs) * 3;
                // the thickness points of the cell share the in-plane C~: sum the
                // 9 gradient products over q3 first, then contract once with C~
                double S[9];
#pragma unroll
                for (int xy = 0; xy < 9; ++xy)
                    S[xy] = 0.0;
                for (int q3 = 0; q3 < d.nqt; ++q3) {
                    const double Ta = tv[q3 * ntl + at], Tda = td[q3 * ntl + at];
                    const double Tb = tv[q3 * ntl + bt], Tdb = td[q3 * ntl + bt];
                    // grad_hat = (du T, dv T, val T') (assembly.cpp:203-206)
                    const double xa[3] = {ga[0] * Ta, ga[1] * Ta, ga[2] * Tda};
                    const double xb[3] = {gb[0] * Tb * w3[q3], gb[1] * Tb * w3[q3], gb[2] * Tdb * w3[q3]};
#pragma unroll
                    for (int x = 0; x < 3; ++x)
#pragma unroll
                        for (int y = 0; y < 3; ++y)
                            S[3 * x + y] += xa[x] * xb[y];
                }
                const double2* C2 = reinterpret_cast<const double2*>(ctq + q2 * 90);
#pragma unroll
                for (int xy = 0; xy < 9; ++xy) {
#pragma unroll
                    for (int h = 0; h < 5; ++h) {
                        const double2 c = C2[xy * 5 + h];
                        acc[2 * h] += c.x * S[xy];
                        if (2 * h + 1 < 9)
                            acc[2 * h + 1] += c.y * S[xy];
                    }
                }
            }
            // K(i,j)[a][b] into row block i; with symmetric tables also
            // K(j,i)[b][a] = K(i,j)[a][b] into row block j (same element, so the
            // colouring still makes the += race-free)
            for (int side = 0; side < 2; ++side) {
                if (side == 0 ? !row_i : !row_j)
                    continue;
                const int ls = side ? bs : as, ms = side ? as : bs;
                const int rt = side ? jt : it, ct_ = side ? it : jt;
                const int iu = el.fu + ls % (d.pu + 1), iv = el.fv + ls / (d.pu + 1);
                const int ju = el.fu + ms % (d.pu + 1), jv = el.fv + ms / (d.pu + 1);
                const int is = iv * d.nu + iu;
                const int Lu = d.len_u[iu], Lv = d.len_v[iv];
                const int B = 3 * Lu * Lv;
                const int slot = (jv - d.lo_v[iv]) * Lu + (ju - d.lo_u[iu]);
                const int Lt = d.len_t[rt];
                const long long pos = 9 * d.S_s * (d.pre_t[rt] - pre0) + (long long)Lt * d.es_pre[is] +
                                      (long long)(ct_ - d.lo_t[rt]) * B + 3 * slot;
                LF_CHECK(pos >= 0 && pos + 2LL * Lt * B + 2 < d.nnz_slab && ct_ >= d.lo_t[rt] &&
                         ct_ < d.lo_t[rt] + Lt);
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b)
                        values[pos + (long long)a * Lt * B + b] += side ? acc[3 * b + a] : acc[3 * a + b];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K5: closed-form CSR pattern, slab-local row offsets.
__global__ void k_pattern_rows(const DevTables d, long long* __restrict__ row_ptr, long long rows) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > rows)
        return;
    if (r == rows) {
        row_ptr[rows] = 9 * d.S_s * (d.pre_t[d.t1] - d.pre_t[d.t0]);
        return;
    }
    const long long per_t = 3LL * d.ns;
    const int it = d.t0 + (int)(r / per_t);
    const long long rr = r % per_t;
    const int is = (int)(rr / 3), a = (int)(rr % 3);
    const int iu = is % d.nu, iv = is / d.nu;
    const int B = 3 * d.len_u[iu] * d.len_v[iv];
    const int Lt = d.len_t[it];
    row_ptr[r] = 9 * d.S_s * (d.pre_t[it] - d.pre_t[d.t0]) + (long long)Lt * (d.es_pre[is] + (long long)a * B);
}

constexpr int kColsEpt = 4; // entries per thread of k_pattern_cols

/// Columns of the slab's CSR.  Thread slots are warp-contiguous (a warp owns
/// 32 * kColsEpt consecutive entries, so its kColsEpt stores per (row, k) are
/// adjacent 128-byte runs) and the stores stream (st.global.cs).
__global__ void __launch_bounds__(kBlock) k_pattern_cols(const DevTables d, int* __restrict__ cols,
                                                         int t_chunk) {
    int* o0[kColsEpt];
    int B[kColsEpt], col_s[kColsEpt];
    long long A[kColsEpt];
    bool live[kColsEpt];
#pragma unroll
    for (int x = 0; x < kColsEpt; ++x) {
        const long long e = (long long)blockIdx.x * kBlock * kColsEpt + (threadIdx.x >> 5) * 32 * kColsEpt +
                            x * 32 + (threadIdx.x & 31);
        live[x] = e < d.E;
        const long long ec = live[x] ? e : d.E - 1;
        int is = __ldg(d.blk_is + ec / kBlock);
        while (__ldg(d.es_pre + is + 1) <= ec)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(ec - ebase);
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        B[x] = 3 * Lu * Lv;
        const int a = r / B[x], rem = r - a * B[x];
        const int s = rem / 3, b = rem % 3;
        const int jv = __ldg(d.lo_v + iv) + s / Lu, ju = __ldg(d.lo_u + iu) + s % Lu;
        col_s[x] = 3 * (jv * d.nu + ju) + b;
        A[x] = ebase + (long long)a * B[x];
        o0[x] = cols + rem;
    }
    const int it_begin = d.t0 + blockIdx.y * t_chunk;
    const int it_end = min(d.t1, it_begin + t_chunk);
    const long long pre0 = __ldg(d.pre_t + d.t0);
    for (int it = it_begin; it < it_end; ++it) {
        const int Lt = __ldg(d.len_t + it);
        const long long base = 9 * d.S_s * (__ldg(d.pre_t + it) - pre0);
        const int c0 = 3 * d.ns * __ldg(d.lo_t + it);
#pragma unroll
        for (int x = 0; x < kColsEpt; ++x)
            LF_CHECK(!live[x] || (base + (long long)Lt * A[x] + (o0[x] - cols) >= 0 &&
                                  base + (long long)Lt * A[x] + (long long)(Lt - 1) * B[x] + (o0[x] - cols) <
                                      d.nnz_slab));
        for (int k = 0; k < Lt; ++k) {
#pragma unroll
            for (int x = 0; x < kColsEpt; ++x)
                if (live[x])
                    __stcs(o0[x] + base + (long long)Lt * A[x] + (long long)k * B[x], c0 + 3 * d.ns * k + col_s[x]);
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

__global__ void k_symmetry_rows(long long rows, const long long* rp, const int* c, const double* v,
                                double* partial) {
    double s = 0.0;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (long long)gridDim.x * blockDim.x) {
        for (long long k = rp[r]; k < rp[r + 1]; ++k) {
            const int col = c[k];
            long long lo = rp[col], hi = rp[col + 1];
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if (c[mid] < r)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            const bool mirrored = lo < rp[col + 1] && c[lo] == r;
            const double dd = v[k] - (mirrored ? v[lo] : 0.0);
            s += dd * dd;
            if (!mirrored)
                s += dd * dd; // symmetryRelError counts the absent mirror slot (sparse.cpp:87-90)
        }
    }
    s = block_sum(s);
    if (threadIdx.x == 0)
        partial[blockIdx.x] = s;
}

int reduce_launch(int blocks, double* partial, double* out, cudaStream_t stream) {
    k_final_sum<<<1, 1024, 0, stream>>>(partial, blocks, out);
    return (int)cudaGetLastError();
}

template <int NT>
constexpr int entries_per_thread() { return NT <= 4 ? 2 : 1; } // two entries: 64 P registers at 4 terms

/// TMA-bulk variant for a first pass; false when it does not apply (group
/// wider than a block, or staging buffers too large for two blocks per SM).
/// One event per device orders every use of the constant-bank row images
/// (c_rows / c_w are per device, not per stream).
cudaEvent_t const_bank_event(int device) {
    static std::mutex mu;
    static cudaEvent_t ev[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (device < 0 || device >= 64)
        return nullptr;
    if (!ev[device])
        cudaEventCreateWithFlags(&ev[device], cudaEventDisableTiming);
    return ev[device];
}

/// Warp-specialised combine for a single pass of <= 4 terms; false when it
/// does not apply (no group packing for this problem, or staging too large).
/// ws_variant (LAMFAST_WS): 1 = 7 producer + 1 consumer warps, 2 = 6 + 2,
/// 3 = 8 + 2; two entries per producer thread.
template <int NT>
bool combine_ws(const DevTables& d, double* out, int lt_max, cudaStream_t s, int* launches) {
    if constexpr (NT > 4) {
        return false;
    } else {
        if (d.ws_variant == 0 || d.n_gbw <= 0 || !d.g_rows || !d.g_w)
            return false;
        const int np = d.ws_variant == 1 ? 7 : d.ws_variant == 2 ? 6 : 8;
        const int nc = d.ws_variant == 1 ? 1 : 2;
        const size_t slot_len = (size_t)lt_max * np * 32 * 2 + 2;
        const size_t smem = kWsSlots * slot_len * sizeof(double) + 64;
        const int seg_rows = std::min(kConstRows, kConstW / (lt_max * NT));
        if (smem > 112 * 1024 || seg_rows < 1)
            return false;
        const int nrow = d.t1 - d.t0;
        RowC* g_rows = static_cast<RowC*>(d.g_rows);
        double4* g_w = static_cast<double4*>(d.g_w);
        const int npack = std::max(nrow, nrow * lt_max * NT);
        k_pack_rows<<<(npack + 255) / 256, 256, 0, s>>>(d, g_rows, g_w, NT, lt_max);
        if (launches)
            ++*launches;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaEvent_t bank = const_bank_event(dev);
        auto kern = d.affine ? (d.ws_variant == 1 ? k_combine_ws<NT, 2, 7, 1, true>
                                : d.ws_variant == 2 ? k_combine_ws<NT, 2, 6, 2, true>
                                                    : k_combine_ws<NT, 2, 8, 2, true>)
                             : (d.ws_variant == 1 ? k_combine_ws<NT, 2, 7, 1, false>
                                : d.ws_variant == 2 ? k_combine_ws<NT, 2, 6, 2, false>
                                                    : k_combine_ws<NT, 2, 8, 2, false>);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int r0 = 0; r0 < nrow; r0 += seg_rows) {
            const int rows = std::min(seg_rows, nrow - r0);
            if (bank)
                cudaStreamWaitEvent(s, bank, 0);
            cudaMemcpyToSymbolAsync(c_rows, g_rows + r0, sizeof(RowC) * rows, 0, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyToSymbolAsync(c_w, g_w + (size_t)r0 * lt_max * NT, sizeof(double4) * rows * lt_max * NT, 0,
                                    cudaMemcpyDeviceToDevice, s);
            // chunks of <= 64 rows, balanced in multiples of 16
            int nchunk = (rows + 63) / 64;
            while (nchunk < rows / 16 && (long long)d.n_gbw * nchunk < 148LL * 2 * 4)
                ++nchunk;
            const int t_chunk = std::min(rows, ((rows + nchunk - 1) / nchunk + 15) / 16 * 16);
            const dim3 grid((unsigned)d.n_gbw, (unsigned)((rows + t_chunk - 1) / t_chunk));
            // rows of this segment start at slab row r0: offset the output base
            // through the constant image (RowC::base is slab-global)
            kern<<<grid, (np + nc) * 32, smem, s>>>(d, out, rows, t_chunk, lt_max);
            if (launches)
                ++*launches;
            if (bank)
                cudaEventRecord(bank, s);
        }
        return true;
    }
}


/// Team/bulk combine for a single pass of <= 4 terms; false when it does not
/// apply (no team layout for this plan, or the slots do not fit).
template <int NT>
bool combine_team(const DevTables& d, double* out, int t_chunk_req, int lt_max, cudaStream_t s, int* launches) {
    if constexpr (NT > 4) {
        return false;
    } else {
        if (d.n_team <= 0 || d.tm_team <= 0)
            return false;
        const int team = d.tm_team, ept = d.tm_ept;
        static const int tpb_env = [] {
            const char* e = std::getenv("LAMFAST_TEAM_TPB");
            return e ? std::atoi(e) : 0;
        }();
        const int teams_per_block = tpb_env > 0 ? std::min(tpb_env, 8 / team) : std::max(1, 8 / team);
        const int threads = teams_per_block * team * 32;
        const int cap = 32 * team * ept;
        const int slot_len = (lt_max * cap + 2 + team * 32 + 1) & ~1; // data + phase pad + scratch line
        const size_t slots = (size_t)teams_per_block * 3 * slot_len * sizeof(double);
        const int nt = d.t1 - d.t0;
        const long long nblk = (d.n_team + teams_per_block - 1) / teams_per_block;
        int t_chunk = t_chunk_req;
        if (t_chunk <= 0) {
            t_chunk = std::min(nt, 64);
            while (t_chunk > 32 && nblk * ((nt + t_chunk - 1) / t_chunk) < 148LL * 2 * 4)
                t_chunk /= 2;
            const int nchunks = (nt + t_chunk - 1) / t_chunk;
            t_chunk = std::min(nt, ((nt + nchunks - 1) / nchunks + 15) / 16 * 16);
        }
        int stage_rows = (int)((16 * 1024) / ((size_t)lt_max * NT * sizeof(double4)));
        stage_rows = std::max(1, std::min(stage_rows, t_chunk));
        const size_t smem = ((stage_rows * sizeof(TeamRow) + 31) & ~size_t(31)) +
                            (size_t)stage_rows * lt_max * NT * sizeof(double4) + slots;
        if (smem > 200 * 1024)
            return false;
        // per-term neighbour ranges off by default here: uniform all-k loops
        // measured faster in this kernel (C4 3.18 -> 3.05 ms)
        static const bool kr = [] {
            const char* e = std::getenv("LAMFAST_TEAM_KR");
            return e && std::atoi(e) != 0;
        }();
        auto pick = [&](auto kr_tag) {
            constexpr bool KR = decltype(kr_tag)::value;
            return d.affine ? (ept == 1   ? k_combine_team<NT, 1, true, KR>
                               : ept == 2 ? k_combine_team<NT, 2, true, KR>
                                          : k_combine_team<NT, 3, true, KR>)
                            : (ept == 1   ? k_combine_team<NT, 1, false, KR>
                               : ept == 2 ? k_combine_team<NT, 2, false, KR>
                                          : k_combine_team<NT, 3, false, KR>);
        };
        auto kern = kr ? pick(std::true_type{}) : pick(std::false_type{});
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const dim3 grid((unsigned)nblk, (unsigned)((nt + t_chunk - 1) / t_chunk));
        kern<<<grid, threads, smem, s>>>(d, out, t_chunk, stage_rows, lt_max, team, slot_len);
        if (launches)
            ++*launches;
        return true;
    }
}

template <int NT>
void combine_one(const DevTables& d, double* out, int pass, int t_chunk, int stage_rows, int lt_max,
                 unsigned nchunk, cudaStream_t s, bool accum) {
    constexpr int EPT = entries_per_thread<NT>();
    // two entries per thread: explicit bounds (<= 128 registers, 2 blocks of
    // 256 per SM); one entry: the compiler's own choice (80-128 registers)
    constexpr int BT = kBlock;
    constexpr int MINB = 2;
    constexpr bool bounded = EPT >= 2;
    const size_t smem = ((stage_rows * (sizeof(RowInfo) + 2 * NT) + 31) & ~size_t(31)) +
                        (size_t)stage_rows * lt_max * NT * sizeof(double4);
    const dim3 grid((unsigned)((d.E + (long long)BT * EPT - 1) / ((long long)BT * EPT)), nchunk);
    auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, BT, smem, s>>>(d, out, pass, t_chunk, stage_rows, lt_max);
    };
    if constexpr (!bounded) {
        if (d.affine)
            accum ? launch(k_combine<NT, EPT, true, true>) : launch(k_combine<NT, EPT, true, false>);
        else
            accum ? launch(k_combine<NT, EPT, false, true>) : launch(k_combine<NT, EPT, false, false>);
    } else {
        if (d.affine)
            accum ? launch(k_combine_b<NT, EPT, true, true, BT, MINB>)
                  : launch(k_combine_b<NT, EPT, true, false, BT, MINB>);
        else
            accum ? launch(k_combine_b<NT, EPT, false, true, BT, MINB>)
                  : launch(k_combine_b<NT, EPT, false, false, BT, MINB>);
    }
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
    const int nl2 = (d.pu + 1) * (d.pv + 1), nq2 = d.nqu * d.nqv;
    const size_t smem = sizeof(double) * ((size_t)nq2 * nl2 * 3 + nq2 + 1 + (size_t)nq2 * 90);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_inplane_general, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const dim3 grid((d.nspu + d.pu) / (d.pu + 1), (d.nspv + d.pv) / (d.pv + 1), d.n_terms);
    const int threads = std::min(512, 4 * ((nl2 * nl2 + 31) / 32 * 32)); // one thread per (local pair, family)
    for (int cv = 0; cv <= d.pv; ++cv)
        for (int cu = 0; cu <= d.pu; ++cu)
            k_inplane_general<<<grid, threads, smem, stream>>>(d, cu, cv);
    return (int)cudaGetLastError();
}

int launch_combine(const DevTables& d, double* out, int t_chunk, cudaStream_t stream, int* launches) {
    if (d.E == 0 || d.t1 <= d.t0)
        return 0;
    const long long nblk = (d.E + kBlock - 1) / kBlock; // 256-entry sub-blocks
    const int nt = d.t1 - d.t0;
    if (t_chunk <= 0) {
        if (const char* env = std::getenv("LAMFAST_TCHUNK"))
            t_chunk = std::atoi(env);
    }
    const int t_chunk_req = t_chunk;
    if (t_chunk <= 0) {
        // 64 thickness rows per block amortise the per-block prologue (P in
        // registers, entry decode, staging); shorter chunks (down to 32) only
        // while the grid is under ~4 waves of 2 resident blocks on 148 SMs.
        // Measured sweep: profiles/r1_tchunk_sweep.txt.
        const long long blocks_x = (nblk + 1) / 2; // two entries per thread for <= 4 terms
        // general geometry loads P from HBM once per block: whole-slab chunks
        // (measured C3 bilinear 1.47 -> 1.38 ms); affine P is recomputed, so
        // shorter chunks balance better (profiles/r1_tchunk_sweep.txt)
        t_chunk = d.affine ? std::min(nt, 64) : nt;
        while (!d.affine && t_chunk > 64 && blocks_x * ((nt + t_chunk - 1) / t_chunk) < 148LL * 2 * 4)
            t_chunk = (t_chunk + 1) / 2;
        while (t_chunk > 32 && blocks_x * ((nt + t_chunk - 1) / t_chunk) < 148LL * 2 * 4)
            t_chunk /= 2;
        const int nchunks = (nt + t_chunk - 1) / t_chunk; // balance, in multiples of 16 rows
        t_chunk = std::min(nt, ((nt + nchunks - 1) / nchunks + 15) / 16 * 16);
    }
    const unsigned nchunk = (unsigned)((nt + t_chunk - 1) / t_chunk);
    const int lt_max = std::max(1, d.lt_max);
    if (d.n_passes == 1) {
        bool done = false;
        switch (d.n_terms) {
        case 1: done = combine_team<1>(d, out, t_chunk_req, lt_max, stream, launches); break;
        case 2: done = combine_team<2>(d, out, t_chunk_req, lt_max, stream, launches); break;
        case 3: done = combine_team<3>(d, out, t_chunk_req, lt_max, stream, launches); break;
        case 4: done = combine_team<4>(d, out, t_chunk_req, lt_max, stream, launches); break;
        default: break;
        }
        if (done)
            return (int)cudaGetLastError();
        switch (d.n_terms) {
        case 1: done = combine_ws<1>(d, out, lt_max, stream, launches); break;
        case 2: done = combine_ws<2>(d, out, lt_max, stream, launches); break;
        case 3: done = combine_ws<3>(d, out, lt_max, stream, launches); break;
        case 4: done = combine_ws<4>(d, out, lt_max, stream, launches); break;
        default: break;
        }
        if (done)
            return (int)cudaGetLastError();
    }
    for (int pass = 0; pass < d.n_passes; ++pass) {
        const int nterm = std::min(8, d.n_terms - 8 * pass);
        const bool accum = pass > 0;
        // rows per staged sub-chunk: ~24 KB of weights, at most the chunk
        int stage_rows = (int)((24 * 1024) / ((size_t)lt_max * nterm * sizeof(double4)));
        stage_rows = std::max(1, std::min(stage_rows, t_chunk));
        switch (nterm) {
        case 1: combine_one<1>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        case 2: combine_one<2>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        case 3: combine_one<3>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        case 4: combine_one<4>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        case 5: combine_one<5>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        case 6: combine_one<6>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        case 7: combine_one<7>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        default: combine_one<8>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, stream, accum); break;
        }
        if (launches)
            ++*launches;
    }
    return (int)cudaGetLastError();
}

int launch_pattern(const DevTables& d, long long* row_ptr, int* cols, cudaStream_t stream) {
    const long long rows = 3LL * d.ns * (d.t1 - d.t0);
    k_pattern_rows<<<(unsigned)((rows + 1 + 255) / 256), 256, 0, stream>>>(d, row_ptr, rows);
    if (d.E > 0 && d.t1 > d.t0) {
        const long long nblk = (d.E + (long long)kBlock * kColsEpt - 1) / ((long long)kBlock * kColsEpt);
        const int nt = d.t1 - d.t0;
        long long nchunks = std::max(1LL, std::min<long long>((148LL * 16 + nblk - 1) / nblk, nt));
        const int t_chunk = (int)((nt + nchunks - 1) / nchunks);
        const dim3 grid((unsigned)nblk, (unsigned)((nt + t_chunk - 1) / t_chunk));
        k_pattern_cols<<<grid, kBlock, 0, stream>>>(d, cols, t_chunk);
    }
    return (int)cudaGetLastError();
}

int launch_standard(const DevTables& d, double* values, long long nnz, cudaStream_t stream, int* launches) {
    cudaMemsetAsync(values, 0, sizeof(double) * (size_t)nnz, stream);
    const int nl2 = (d.pu + 1) * (d.pv + 1), nq2 = d.nqu * d.nqv, ntl = d.pt + 1;
    const size_t smem = sizeof(double) * ((size_t)nq2 * nl2 * 3 + nq2 + 1 + (size_t)nq2 * 90 +
                                          2 * (size_t)d.nqt * ntl + d.nqt);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_standard, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int gx = (d.nspu + d.pu) / (d.pu + 1), gy = (d.nspv + d.pv) / (d.pv + 1), gz = (d.nspt + d.pt) / (d.pt + 1);
    // split the local pairs of each (element, span) over enough blocks for
    // ~4 blocks per SM per colour launch (chunks of >= 256 pairs)
    const int nl3 = nl2 * ntl;
    const int npair = d.sym ? nl3 * (nl3 + 1) / 2 : nl3 * nl3;
    const long long blocks = (long long)gx * gy * gz;
    int nchunk = (int)std::min<long long>((148LL * 4 + blocks - 1) / blocks, (npair + 255) / 256);
    nchunk = std::max(1, std::min(nchunk, 65535 / std::max(1, gz)));
    const dim3 grid(gx, gy, gz * nchunk);
    for (int ct = 0; ct <= d.pt; ++ct)
        for (int cv = 0; cv <= d.pv; ++cv)
            for (int cu = 0; cu <= d.pu; ++cu) {
                k_standard<<<grid, 256, smem, stream>>>(d, values, cu, cv, ct, nchunk);
                if (launches)
                    ++*launches;
            }
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

int launch_symmetry_sq(long long rows, const long long* rp, const int* c, const double* v, double* out,
                       cudaStream_t stream) {
    const int blocks = 1024;
    double* partial = nullptr;
    cudaMallocAsync(&partial, sizeof(double) * blocks, stream);
    k_symmetry_rows<<<blocks, 256, 0, stream>>>(rows, rp, c, v, partial);
    reduce_launch(blocks, partial, out, stream);
    cudaFreeAsync(partial, stream);
    return (int)cudaGetLastError();
}

} // namespace lfb
