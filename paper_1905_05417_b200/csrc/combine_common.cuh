// Device helpers shared by the combine kernels (K4 and its store variants):
// entry decode, affine P in registers, the per-row FMA forms and the
// per-block staging of thickness rows.  Everything here has internal linkage
// (anonymous namespace): each translation unit gets its own inlined copy.
#pragma once

#include <cuda_runtime.h>

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

/// Predicated streaming store (no branch around it).
__device__ __forceinline__ void store_value_if(double* p, double v, unsigned pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cs.f64 [%0], %1;\n\t}" ::"l"(p),
                 "d"(v), "r"(pred)
                 : "memory");
}

/// 16-byte global -> shared asynchronous copy (L2 only), zero-filled when !ok.
__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc, bool ok) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gsrc), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
/// all but the most recent committed group have landed (this thread's copies)
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

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
    long long base; // 9 S_s (pre_t[it] - pre_t[t0]) - out_base: range offset of row block it
    int lt;         // L_t(it) | edge << 8 (edge bit 0: row t0 starts at s0; bit 1: row t1-1 ends at s1)
    unsigned mask;  // union of term masks over the row's pairs (this pass)
};

/// Row of a range that starts or ends inside it (see DevTables::s0 / s1).
__device__ __forceinline__ int row_edge(const DevTables& d, int it) {
    return (it == d.t0 && d.s0 > 0 ? 1 : 0) | (it == d.t1 - 1 && d.s1 < d.ns ? 2 : 0);
}

template <int NT, int EPT, int LT, bool ACCUM, bool SMEM = false, typename WP = const double4*>
__device__ __forceinline__ void combine_row(const double (&P)[EPT][NT][4], WP w,
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
template <int NT, int EPT, int LT, bool ACCUM, typename WP = const double4*>
__device__ __forceinline__ void combine_row_k(const double (&P)[EPT][NT][4], WP w,
                                              unsigned mask, const unsigned char* __restrict__ kr,
                                              double* const (&o)[EPT], const int (&B)[EPT], const bool (&live)[EPT]) {
    int klo[NT], khi[NT];
#ifdef LF_STORE_ONLY
    mask = 0; // diagnostic build: identical store pattern, no weight loads / FMAs
#endif
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

/// Rows whose active terms are the compile-time set M: straight-line FMAs
/// over all LT neighbours, no per-(neighbour, term) range tests.  A pair a
/// term of M does not reach has exactly zero weights (W accumulates only
/// contributing cells, k_prepare_affine / k_thickness_pairs), so the extra
/// products add zeros.  The range tests and their branches were ~29% of the
/// instructions of the k-outer rows (ncu source page, C3: ISETP 19%, BRA 9%,
/// DFMA 17%); fully unrolled, the LT neighbours' chains are independent.
template <int NT, int EPT, int LT, unsigned M, typename WP = const double4*>
__device__ __forceinline__ void combine_row_m(const double (&P)[EPT][NT][4], WP w,
                                              double* const (&o)[EPT], const int (&B)[EPT], const bool (&live)[EPT]) {
    static_assert(M != 0u && ((M & (M - 1u)) & ((M & (M - 1u)) - 1u)) == 0u, "at most two terms");
    constexpr int t_first = __builtin_ctz(M), t_last = 31 - __builtin_clz(M); // M has <= 2 bits
#pragma unroll
    for (int k = 0; k < LT; ++k) {
        double acc[EPT];
        {
            const double4 ww = w[k * NT + t_first];
#pragma unroll
            for (int x = 0; x < EPT; ++x) {
                acc[x] = P[x][t_first][0] * ww.x;
                acc[x] = fma(P[x][t_first][1], ww.y, acc[x]);
                acc[x] = fma(P[x][t_first][2], ww.z, acc[x]);
                acc[x] = fma(P[x][t_first][3], ww.w, acc[x]);
            }
        }
        if constexpr (t_last != t_first) {
            const double4 ww = w[k * NT + t_last];
#pragma unroll
            for (int x = 0; x < EPT; ++x) {
                acc[x] = fma(P[x][t_last][0], ww.x, acc[x]);
                acc[x] = fma(P[x][t_last][1], ww.y, acc[x]);
                acc[x] = fma(P[x][t_last][2], ww.z, acc[x]);
                acc[x] = fma(P[x][t_last][3], ww.w, acc[x]);
            }
        }
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            if (live[x])
                store_value(o[x] + (long long)k * B[x], acc[x]);
    }
}

/// Selects combine_row_m for a row whose union term mask has at most two
/// terms (every row of a C0 thickness space with one element per ply: a
/// vertex function spans two plies, a bubble one); false -> generic rows.
template <int NT, int EPT, int LT, typename WP = const double4*>
__device__ __forceinline__ bool row_masked(unsigned mask, const double (&P)[EPT][NT][4],
                                           WP w, double* const (&o)[EPT],
                                           const int (&B)[EPT], const bool (&live)[EPT]) {
#ifdef LF_STORE_ONLY
    return false;
#endif
    switch (mask) {
#define LF_ROW_M(m)                                                  \
    case m:                                                          \
        if constexpr ((m >> NT) == 0u) {                             \
            combine_row_m<NT, EPT, LT, m>(P, w, o, B, live);         \
            return true;                                             \
        }                                                            \
        break;
        LF_ROW_M(1u) LF_ROW_M(2u) LF_ROW_M(3u) LF_ROW_M(4u) LF_ROW_M(5u)
        LF_ROW_M(6u) LF_ROW_M(8u) LF_ROW_M(9u) LF_ROW_M(10u) LF_ROW_M(12u)
#undef LF_ROW_M
    default:
        break;
    }
    return false;
}

template <int NT, int EPT, int LT, bool ACCUM, typename WP = const double4*>
__device__ __forceinline__ void row_dispatch(const double (&P)[EPT][NT][4], WP w,
                                             unsigned mask, const unsigned char* __restrict__ kr,
                                             double* const (&o)[EPT], const int (&B)[EPT], const bool (&live)[EPT]) {
    if constexpr (EPT >= 2)
        combine_row_k<NT, EPT, LT, ACCUM>(P, w, mask, kr, o, B, live);
    else
        combine_row<NT, EPT, LT, ACCUM>(P, w, mask, kr, o, B, live);
}

template <int NT, int EPT, bool ACCUM, bool SMEM = false, typename WP = const double4*>
__device__ __forceinline__ void combine_row_dyn(const double (&P)[EPT][NT][4], WP w,
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
    const long long preW = __ldg(d.pre_t + d.w_t0); // W / Wmask index base (the plan's rows)
    const long long nine_S = 9 * d.S_s;
    const unsigned* mask_base = d.Wmask + (long long)pass * d.n_pairs;
    const int T = d.n_terms;
    // stage rows: RowInfo, per-term neighbour ranges, weights s_w[row][k][t]
    for (int rr = tid; rr < nrow; rr += nthreads) {
        const int it = it0 + rr;
        const long long pfx = __ldg(d.pre_t + it) - preW;
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
        s_row[rr].base = nine_S * (__ldg(d.pre_t + it) - pre0) - d.out_base;
        s_row[rr].lt = lt | row_edge(d, it) << 8;
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
            const long long q = __ldg(d.pre_t + it) - preW + k;
            const double2* src = reinterpret_cast<const double2*>(d.W + ((q * T) + t_first + t) * 4);
            const double2 lo2 = __ldg(src), hi2 = __ldg(src + 1);
            v = make_double4(lo2.x, lo2.y, hi2.x, hi2.y);
        }
        s_w[idx] = v;
    }
}

} // namespace
} // namespace lfb
