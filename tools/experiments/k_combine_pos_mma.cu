// K4, position-owned form on the FP64 tensor cores: P (x) q~ straight into
// the CSR value array (fast.cpp:211-264 + sparse.cpp:30-55) with line-aligned
// 256-bit stores.
//
// The values of one thickness row i_t are one contiguous range of
// L_t(i_t) * E doubles (E = 9 S_s in-plane entries), ordered
// (i_s, a, k, slot, b).  k_combine (k_combine.cu) gives a thread one in-plane
// entry and lets it write that entry's L_t values of every row: its warp
// stores are 256-byte runs at the 8-byte alignment the odd row-segment length
// 3 L_s dictates, and that store pattern alone sets the kernel's time
// (profiles/r2_storeonly.txt).
//
// Here a POSITION of the row range is owned instead.  A class holds the
// thickness rows with the same L_t and the same phase phi = (address of the
// row range / 8) mod A; position tau of a class is value
// values[base(i_t) - phi + tau] of every row of the class, and its in-plane
// entry and neighbour (i_s, a, k, slot, b) do not depend on the row.  For a
// fixed neighbour k the values of (rows x positions) are a small dense
// product,
//     K[row, pos] = sum_t sum_f W[(row, k)][t][f] * P[pos][t][f],
// which a warp evaluates with mma.sync.m8n8k4.f64: one DMMA per (8 rows,
// 8 positions, term) with the four operator families as the contraction
// index.  A = the pair weights (one 8-byte shared load per lane, reused by
// every position tile of the warp), B = the positions' P (registers, formed
// once per block from U, V, C~ as in k_combine; lane j of a quad holds family
// j), D = 8 rows x 8 positions.  Tile columns are mapped to positions so that
// a lane ends up with four consecutive positions of one row: one 256-bit
// store per lane, a full 128-byte line per (row, quad), 1 KB per warp store.
// A scalar position-owned form (tools/experiments/k_combine_pos_scalar.cu)
// reached the fill rate store-only (7.16 TB/s) but was bound by the LSU pipe
// with its per-value weight loads (ncu: 80% LSU wavefronts, C4 3.2 ms); the
// DMMA form needs one weight load per 64-256 values.
//
// A warp's positions are consecutive, so they span a few neighbours k at
// most; per k the positions of other neighbours enter with B = 0 (exact
// zeros).  Terms outside the union mask of a row tile are skipped; a pair a
// term does not reach has exactly zero weights (k_prepare_affine /
// k_thickness_pairs accumulate contributing cells only).
//
// Classes, their row lists and the block -> (class, row chunk) map are built
// on the host per launch and travel as a kernel parameter (no upload).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

#include "combine_common.cuh"

namespace lfb {

namespace {

constexpr int kPosMaxJobs = 256;
constexpr int kPosMaxRows = 4096;

struct PosJob {
    int first_block;           // first block of the job in the flat grid
    unsigned short row0, nrow; // the job's rows: rows[row0 .. row0 + nrow)
    unsigned short L, phi;     // neighbour count and phase of the class
};

struct PosParams {
    int n_jobs;
    PosJob jobs[kPosMaxJobs];
    unsigned short rows[kPosMaxRows]; // thickness rows i_t, class by class
};

struct PosRow {
    long long base; // range offset of the row block minus the class phase
    unsigned mask;  // union of the term masks of the row's pairs
    int edge;       // row_edge() of a partial first / last row; 4: padding row (not written)
};

/// doubles per staged row of weights [k][term][family], padded so that the
/// eight rows of a tile start 8 banks apart (conflict-free quads)
__host__ __device__ inline int pos_row_stride(int L, int NT) {
    const int n = L * NT * 4;
    return n + ((4 - n % 16) + 16) % 16;
}

/// D (8x8, rows x positions) += A (8x4, rows x families) * B (4x8, families x positions)
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

/// four consecutive values, 32-byte aligned, streaming
__device__ __forceinline__ void store_value4(double* p, double v0, double v1, double v2, double v3, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
                 "d"(v0), "d"(v1), "d"(v2), "d"(v3), "r"((unsigned)pred)
                 : "memory");
}

// decoded position: k | (3a + b) << 8 | (i_s >= s0) << 12 | (i_s < s1) << 13 | live << 14
struct PosDec {
    int info, uo, vo, ec;
};

__device__ __forceinline__ PosDec decode_position(const DevTables& d, long long o, int L, long long EL) {
    PosDec r;
    const bool live = o >= 0 && o < EL;
    const unsigned oc = live ? (unsigned)o : 0u; // E L < 2^31 (launcher)
    const unsigned e1 = oc / (unsigned)L;        // lies inside the entry range of the position's i_s
    int is = __ldg(d.blk_is + e1 / kBlock);
    while (__ldg(d.es_pre + is + 1) <= (long long)e1)
        ++is;
    const int ebase = (int)__ldg(d.es_pre + is);
    const int rr = (int)oc - L * ebase; // offset inside the (i_t, i_s) row block
    const int iu = is % d.nu, iv = is / d.nu;
    const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
    const int B = 3 * Lu * Lv; // row segment length per thickness neighbour
    const int a = rr / (L * B);
    const int r2 = rr - a * (L * B);
    const int k = r2 / B;
    const int rem = r2 - k * B;
    const int s = rem / 3, b = rem - 3 * s;
    const int sv = s / Lu, su = s - sv * Lu;
    r.info = k | (3 * a + b) << 8 | (is >= d.s0 ? 1 << 12 : 0) | (is < d.s1 ? 1 << 13 : 0) | (live ? 1 << 14 : 0);
    r.uo = (iu * d.bu + su) * 4;
    r.vo = (iv * d.bv + sv) * 4;
    r.ec = ebase + a * B + rem;
    return r;
}

/// Running decode of a lane's position across the consecutive 32-position
/// groups of its warp: the in-plane function, row component, neighbour and
/// offset inside the row segment advance by 32 values without a search or a
/// division by a run-time row length.
struct PosState {
    int is, iu, iv, Lu, Lv, B; // in-plane function of the position, its neighbour counts, segment length 3 Lu Lv
    int ebase;                 // first in-plane entry of is
    int a, k, rem;             // row component, neighbour, offset inside the row segment
    bool live;
};

__device__ __forceinline__ PosState start_position(const DevTables& d, long long o, int L, long long EL) {
    PosState st;
    st.live = o >= 0 && o < EL;
    const unsigned oc = st.live ? (unsigned)o : 0u; // E L < 2^31 (launcher)
    const unsigned e1 = oc / (unsigned)L;           // lies inside the entry range of the position's i_s
    int is = __ldg(d.blk_is + e1 / kBlock);
    while (__ldg(d.es_pre + is + 1) <= (long long)e1)
        ++is;
    st.is = is;
    st.ebase = (int)__ldg(d.es_pre + is);
    const int rr = (int)oc - L * st.ebase; // offset inside the (i_t, i_s) row block
    st.iu = is % d.nu;
    st.iv = is / d.nu;
    st.Lu = __ldg(d.len_u + st.iu);
    st.Lv = __ldg(d.len_v + st.iv);
    st.B = 3 * st.Lu * st.Lv;
    st.a = rr / (L * st.B);
    const int r2 = rr - st.a * (L * st.B);
    st.k = r2 / st.B;
    st.rem = r2 - st.k * st.B;
    return st;
}

/// 32 positions further (the position stays inside the class range: o + 32 < E L)
__device__ __forceinline__ void advance_position(const DevTables& d, PosState& st, int L) {
    st.rem += 32;
    while (st.rem >= st.B) {
        st.rem -= st.B;
        if (++st.k == L) {
            st.k = 0;
            if (++st.a == 3) {
                st.a = 0;
                st.ebase += 3 * st.B; // 9 Lu Lv entries per in-plane function
                ++st.is;
                if (++st.iu == d.nu) {
                    st.iu = 0;
                    ++st.iv;
                    st.Lv = __ldg(d.len_v + st.iv);
                }
                st.Lu = __ldg(d.len_u + st.iu);
                st.B = 3 * st.Lu * st.Lv;
            }
        }
    }
}

__device__ __forceinline__ PosDec state_fields(const DevTables& d, const PosState& st) {
    PosDec r;
    const int s = st.rem / 3, b = st.rem - 3 * s;
    const int sv = s / st.Lu, su = s - sv * st.Lu;
    r.info = st.k | (3 * st.a + b) << 8 | (st.is >= d.s0 ? 1 << 12 : 0) | (st.is < d.s1 ? 1 << 13 : 0) |
             (st.live ? 1 << 14 : 0);
    r.uo = (st.iu * d.bu + su) * 4;
    r.vo = (st.iv * d.bv + sv) * 4;
    r.ec = st.ebase + st.a * st.B + st.rem;
    return r;
}

/// Affine P of family j of one in-plane entry for NT terms (affine_p,
/// combine_common.cuh, one family per lane): s_ct = C~ in shared memory.
template <int NT>
__device__ __forceinline__ void family_p(const DevTables& d, const double* s_ct, int uo, int vo, int ab, int j,
                                         double (&P)[NT]) {
    const double2 ua = __ldg(reinterpret_cast<const double2*>(d.U + uo));
    const double2 ub = __ldg(reinterpret_cast<const double2*>(d.U + uo + 2));
    const double2 va = __ldg(reinterpret_cast<const double2*>(d.V + vo));
    const double2 vb = __ldg(reinterpret_cast<const double2*>(d.V + vo + 2));
    const double u0 = ua.x, u1 = ua.y, u2 = ub.x, u3 = ub.y;
    const double v0 = va.x, v1 = va.y, v2 = vb.x, v3 = vb.y;
    // x -> (u-derivative, v-derivative): 0 -> d/du, 1 -> d/dv, 2 -> value; I_xy index xy = 3x + y
    // family 0: xy 0, 1, 3, 4; family 1: xy 2, 5; family 2: xy 6, 7; family 3: xy 8
    const double Ia = j == 0 ? u3 * v0 : j == 1 ? u2 * v0 : j == 2 ? u1 * v0 : u0 * v0;
    const double Ib = j == 0 ? u2 * v1 : j == 1 ? u0 * v2 : j == 2 ? u0 * v1 : 0.0;
    const double Ic = j == 0 ? u1 * v2 : 0.0;
    const double Id = j == 0 ? u0 * v3 : 0.0;
    const int xa = j == 0 ? 0 : j == 1 ? 18 : j == 2 ? 54 : 72;
    const int xb = j == 0 ? 9 : j == 1 ? 45 : j == 2 ? 63 : 72;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const double* C = s_ct + t * 81 + ab;
        P[t] = C[xa] * Ia + C[xb] * Ib + C[27] * Ic + C[36] * Id;
    }
}

// position q (0 .. 8 NTILE) of the warp window held by column n of tile tl:
// tiles 2h and 2h + 1 interleave so that lane (g, j) -- D columns 2j, 2j + 1
// of both -- holds positions 16 h + 4 j .. + 3
__device__ __forceinline__ int tile_position(int tl, int n) {
    return 16 * (tl >> 1) + 4 * (n >> 1) + 2 * (tl & 1) + (n & 1);
}

/// 32-bit shared-window address and loads through it: the row loop keeps no
/// generic pointer to shared memory (the generic form rematerialised the
/// window base, S2UR SR_CgaCtaId, once per row tile).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds_u128(unsigned a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

/// Rows of one job for the warp's current positions and the neighbours
/// (k0, k1): Pa / Pb are the B operands of the positions with neighbour k0 /
/// k1 (exact zeros elsewhere), so a tile that holds both neighbours takes one
/// DMMA per neighbour and nothing is selected inside the loop.  TWO = false:
/// every position of the warp has neighbour k0.
template <int NT, int NTILE, bool TWO>
__device__ __forceinline__ void mma_rows(const DevTables& d, double* __restrict__ out, double* const o_lane,
                                         const double (&Pa)[NTILE][NT], const double (&Pb)[NTILE][NT],
                                         unsigned pair_a, unsigned pair_b, unsigned srow_a, unsigned sw_a0,
                                         unsigned sw_a1, int nrow8, int rs, bool fast_store, const int (&qinfo)[NTILE / 2][4],
                                         int k0, int k1) {
    const unsigned w_step = (unsigned)rs * 8u * (unsigned)sizeof(double);
    for (int rt = 0; rt < nrow8; rt += 8, srow_a += 8u * (unsigned)sizeof(PosRow), sw_a0 += w_step, sw_a1 += w_step) {
        const uint4 ri = lds_u128(srow_a); // base (lo, hi), term mask of the tile, edge | tile edges << 8
        const unsigned tmask = ri.z;
        double D[NTILE][2];
#pragma unroll
        for (int tl = 0; tl < NTILE; ++tl)
            D[tl][0] = D[tl][1] = 0.0;
#ifndef LF_STORE_ONLY
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if (tmask & (1u << t)) {
                const double a0 = lds_f64(sw_a0 + t * 32);
                if constexpr (!TWO) {
#pragma unroll
                    for (int tl = 0; tl < NTILE; ++tl)
                        dmma_884(D[tl][0], D[tl][1], a0, Pa[tl][t]);
                } else {
                    const double a1 = lds_f64(sw_a1 + t * 32);
#pragma unroll
                    for (int h = 0; h < NTILE / 2; ++h) {
                        if (pair_a & (1u << h)) {
                            dmma_884(D[2 * h][0], D[2 * h][1], a0, Pa[2 * h][t]);
                            dmma_884(D[2 * h + 1][0], D[2 * h + 1][1], a0, Pa[2 * h + 1][t]);
                        }
                        if (pair_b & (1u << h)) {
                            dmma_884(D[2 * h][0], D[2 * h][1], a1, Pb[2 * h][t]);
                            dmma_884(D[2 * h + 1][0], D[2 * h + 1][1], a1, Pb[2 * h + 1][t]);
                        }
                    }
                }
            }
#endif
        const long long base = (long long)(((unsigned long long)ri.y << 32) | ri.x);
        const int edge = (int)(ri.w & 0xffu);
        if (fast_store && (ri.w >> 8) == 0) {
            const bool row_ok = edge == 0; // padding rows of the last tile are not written
            double* const p = o_lane + base;
#pragma unroll
            for (int h = 0; h < NTILE / 2; ++h) {
                LF_CHECK(!row_ok || (p + 16 * h >= out && p + 16 * h + 3 < out + d.nnz_slab));
                store_value4(p + 16 * h, D[2 * h][0], D[2 * h][1], D[2 * h + 1][0], D[2 * h + 1][1], row_ok);
            }
        } else {
            // warps at the ends of the class range, warps with a third
            // neighbour, and tiles with a partial first / last row of a
            // function range: one predicated store per value
#pragma unroll
            for (int h = 0; h < NTILE / 2; ++h)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int info = qinfo[h][c];
                    const unsigned flags = (info >> 12) & 3u;
                    const int k = info & 0xff;
                    const bool pred = ((info >> 14) & 1) && (k == k0 || k == k1) && edge < 4 &&
                                      ((unsigned)edge & ~flags) == 0;
                    double* const p = o_lane + base + 16 * h + c;
                    LF_CHECK(!pred || (p >= out && p < out + d.nnz_slab));
                    store_value_if(p, D[2 * h + (c >> 1)][c & 1], pred);
                }
        }
    }
}

template <int NT, int NTILE, bool AFFINE, int BT, int MINB, int G>
__global__ void __launch_bounds__(BT, MINB)
    k_combine_mma(const __grid_constant__ DevTables d, const __grid_constant__ PosParams pp,
                  double* __restrict__ out) {
    static_assert(NTILE == 4, "32 positions per warp and group");
    constexpr int WP = 8 * NTILE; // positions per warp and group
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // job of this block
    int jlo = 0, jhi = pp.n_jobs; // jobs[jlo].first_block <= blockIdx.x < jobs[jhi].first_block
    while (jhi - jlo > 1) {
        const int mid = (jlo + jhi) >> 1;
        if (pp.jobs[mid].first_block <= (int)blockIdx.x)
            jlo = mid;
        else
            jhi = mid;
    }
    const int L = pp.jobs[jlo].L, phi = pp.jobs[jlo].phi;
    const int nrow = pp.jobs[jlo].nrow, row0 = pp.jobs[jlo].row0;
    const int nrow8 = (nrow + 7) & ~7;
    const long long xb = (long long)((int)blockIdx.x - pp.jobs[jlo].first_block);
    const int rs = pos_row_stride(L, NT);
    PosRow* s_row = reinterpret_cast<PosRow*>(smem_raw);
    double* s_w = reinterpret_cast<double*>(smem_raw + nrow8 * sizeof(PosRow));
    double* s_ct = s_w + (size_t)nrow8 * rs; // C~ [NT][81] (affine maps)

    const int lane = threadIdx.x & 31, g = lane >> 2, j = lane & 3;
    const long long EL = d.E * L;

    // stage C~, the job's rows and their weights s_w[row][k][term][family]
    if constexpr (AFFINE)
        for (int idx = threadIdx.x; idx < NT * 81; idx += BT)
            s_ct[idx] = __ldg(d.Ct + idx);
    {
        const long long pre0 = __ldg(d.pre_t + d.t0);
        const long long preW = __ldg(d.pre_t + d.w_t0); // W / Wmask index base (the plan's rows)
        const long long nine_S = 9 * d.S_s;
        for (int rr = threadIdx.x; rr < nrow8; rr += BT) {
            PosRow ri;
            ri.base = 0;
            ri.edge = 4;
            // term mask and edge bits of the row's 8-row tile
            unsigned m = 0, te = 0;
            for (int r8 = rr & ~7; r8 < (rr & ~7) + 8 && r8 < nrow; ++r8) {
                const int it = pp.rows[row0 + r8];
                const long long pre = __ldg(d.pre_t + it);
                for (int k = 0; k < L; ++k)
                    m |= __ldg(d.Wmask + (pre - preW) + k);
                te |= (unsigned)row_edge(d, it);
            }
            if (rr < nrow) {
                const int it = pp.rows[row0 + rr];
                ri.base = nine_S * (__ldg(d.pre_t + it) - pre0) - d.out_base - phi;
                ri.edge = row_edge(d, it);
            }
            ri.mask = m;
            ri.edge |= (int)(te << 8);
            s_row[rr] = ri;
        }
        // a row's weights [k][term][family] are contiguous in W (single pass: n_terms = NT)
        const int per_row = L * NT * 2; // 16-byte pieces
        for (int rr = threadIdx.x >> 5; rr < nrow8; rr += BT / 32) {
            const double2* src = nullptr;
            if (rr < nrow)
                src = reinterpret_cast<const double2*>(d.W) +
                      (__ldg(d.pre_t + pp.rows[row0 + rr]) - preW) * (NT * 2);
            double* dst = s_w + (size_t)rr * rs;
            for (int c = lane; c < per_row; c += 32)
                cp_async16(dst + 2 * c, src ? reinterpret_cast<const double*>(src + c) : d.W, src != nullptr);
        }
        cp_async_commit();
        cp_async_wait0();
    }
    __syncthreads(); // C~, rows and weights visible; no block-wide barrier below

    const unsigned srow_a = smem_u32(s_row) + (unsigned)g * (unsigned)sizeof(PosRow);
    const unsigned sw_g = smem_u32(s_w) + (unsigned)(g * rs + j) * (unsigned)sizeof(double);

    // a warp owns G consecutive 32-position groups
    const long long tau_w0 = (xb * (BT / 32) + (threadIdx.x >> 5)) * (long long)(G * WP);
    PosState st;
    st.live = false;
    for (int grp = 0; grp < G; ++grp) {
        const long long tau_w = tau_w0 + grp * WP; // first position of the warp in this group
        if (tau_w - phi >= EL)
            break;
        // decode the warp's positions, one per lane: a full decode for the
        // first group (and for lanes before the start of the class range),
        // 32 values further after that
        {
            const long long o = tau_w + lane - phi;
            if (grp == 0 || !st.live)
                st = start_position(d, o, L, EL);
            else if (o < EL)
                advance_position(d, st, L);
            else
                st.live = false;
        }
        const PosDec dec = state_fields(d, st);
        const bool lv0 = (dec.info >> 14) & 1;
        const unsigned kmask = __reduce_or_sync(0xffffffffu, lv0 ? 1u << (dec.info & 0xff) : 0u);
        const bool all_live = __all_sync(0xffffffffu, lv0);
        if (kmask == 0)
            continue; // no live position in this warp

        // positions of the lane's tile columns and of its stored values
        int tinfo[NTILE], tuo[NTILE], tvo[NTILE];
#pragma unroll
        for (int tl = 0; tl < NTILE; ++tl) {
            const int src = tile_position(tl, g);
            tinfo[tl] = __shfl_sync(0xffffffffu, dec.info, src);
            tuo[tl] = __shfl_sync(0xffffffffu, AFFINE ? dec.uo : dec.ec, src);
            tvo[tl] = __shfl_sync(0xffffffffu, dec.vo, src);
        }
        int qinfo[NTILE / 2][4];
#pragma unroll
        for (int h = 0; h < NTILE / 2; ++h)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                qinfo[h][c] = __shfl_sync(0xffffffffu, dec.info, 16 * h + 4 * j + c);
        double* const o_lane = out + tau_w + 4 * j; // + 16 h: the lane's four positions of tile pair h

        // neighbours two at a time (a warp's 32 consecutive positions hold one
        // or two; three only where the row segments are shorter than 32 values)
        bool first = true;
        for (unsigned kleft = kmask; kleft; first = false) {
            const int k0 = __ffs(kleft) - 1;
            kleft &= kleft - 1;
            const bool two = kleft != 0;
            const int k1 = two ? __ffs(kleft) - 1 : k0;
            kleft &= kleft - 1;
            const bool fast_store = all_live && first && kleft == 0;

            // B operands: lane (g, j) holds family j of the position in column g of every tile
            double Pa[NTILE][NT], Pb[NTILE][NT];
            unsigned pair_a = 0, pair_b = 0;
#pragma unroll
            for (int tl = 0; tl < NTILE; ++tl) {
                const int info = tinfo[tl];
                const bool lv = (info >> 14) & 1;
                const int k = lv ? (info & 0xff) : -1;
                double P[NT];
                if constexpr (AFFINE) {
                    family_p<NT>(d, s_ct, tuo[tl], tvo[tl], (info >> 8) & 15, j, P);
                } else {
#pragma unroll
                    for (int t = 0; t < NT; ++t)
                        P[t] = __ldg(d.Pg + ((long long)t * 4 + j) * d.E + tuo[tl]);
                }
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    Pa[tl][t] = k == k0 ? P[t] : 0.0;
                    Pb[tl][t] = (two && k == k1) ? P[t] : 0.0;
                }
                pair_a |= __any_sync(0xffffffffu, k == k0) ? 1u << (tl >> 1) : 0u;
                pair_b |= __any_sync(0xffffffffu, two && k == k1) ? 1u << (tl >> 1) : 0u;
            }
            const unsigned sw_a0 = sw_g + (unsigned)(k0 * NT * 4) * (unsigned)sizeof(double);
            const unsigned sw_a1 = sw_g + (unsigned)(k1 * NT * 4) * (unsigned)sizeof(double);
            if (two)
                mma_rows<NT, NTILE, true>(d, out, o_lane, Pa, Pb, pair_a, pair_b, srow_a, sw_a0, sw_a1, nrow8, rs,
                                          fast_store, qinfo, k0, k1);
            else
                mma_rows<NT, NTILE, false>(d, out, o_lane, Pa, Pb, pair_a, pair_b, srow_a, sw_a0, sw_a1, nrow8, rs,
                                           fast_store, qinfo, k0, k1);
        }
    }
}

struct PosConfig {
    int align;     // phase granularity A in values, a multiple of 4 (16: full 128-byte lines per quad store)
    int min_rows;  // classes with fewer rows join the largest class of their L_t (unaligned there)
    size_t smem;   // shared-memory budget per block (rows per job)
};

/// Classes (L_t, phase), row chunks and the flat block map of one launch.
/// false: outside the limits of the kernel-parameter tables (the entry-owned
/// k_combine then takes the launch).
bool build_pos_params(const DevTables& d, const double* out, int NT, int threads_x, const PosConfig& cfg,
                      PosParams& pp, long long& total_blocks, size_t& smem_max) {
    if (!d.pre_t_h || !d.len_t_h || d.t1 - d.t0 > kPosMaxRows || d.t1 > 65535 ||
        d.E * std::max(1, d.lt_max) >= (1LL << 31))
        return false;
    const long long A = cfg.align;
    const long long addr0 = (long long)(reinterpret_cast<uintptr_t>(out) / sizeof(double));
    // rows by (L, phi)
    std::map<std::pair<int, int>, std::vector<int>> cls;
    for (int it = d.t0; it < d.t1; ++it) {
        const int L = d.len_t_h[it];
        if (L <= 0)
            continue;
        if (L > 32)
            return false; // the kernel keeps a warp's neighbours in a 32-bit mask
        const long long base = 9 * d.S_s * (d.pre_t_h[it] - d.pre_t_h[d.t0]) - d.out_base;
        const long long ph = (((addr0 + base) % A) + A) % A;
        cls[{L, (int)ph}].push_back(it);
    }
    // small classes join the largest class of the same L (their stores lose the alignment, nothing else)
    for (auto it = cls.begin(); it != cls.end();) {
        if ((int)it->second.size() >= cfg.min_rows) {
            ++it;
            continue;
        }
        auto best = cls.end();
        for (auto jt = cls.begin(); jt != cls.end(); ++jt)
            if (jt != it && jt->first.first == it->first.first &&
                (jt->first.second - it->first.second) % 4 == 0 && // the 256-bit stores stay 32-byte aligned
                (best == cls.end() || jt->second.size() > best->second.size()))
                best = jt;
        if (best == cls.end() || best->second.size() < it->second.size()) {
            ++it;
            continue;
        }
        best->second.insert(best->second.end(), it->second.begin(), it->second.end());
        std::sort(best->second.begin(), best->second.end());
        it = cls.erase(it);
    }
    // rows of a class ordered by their term mask: the 8-row tiles then skip the terms none of their rows has
    if (d.row_mask_h)
        for (auto& c : cls)
            std::stable_sort(c.second.begin(), c.second.end(),
                             [&](int x, int y) { return d.row_mask_h[x] < d.row_mask_h[y]; });
    // rows per job from the shared-memory budget; more, shorter jobs while the grid is under ~4 waves
    size_t budget = cfg.smem;
    for (;;) {
        int n_jobs = 0, n_rows = 0;
        total_blocks = 0;
        smem_max = 0;
        bool fits = true;
        for (const auto& c : cls) {
            const int L = c.first.first, phi = c.first.second, R = (int)c.second.size();
            const size_t per_row = sizeof(PosRow) + (size_t)pos_row_stride(L, NT) * sizeof(double);
            const int cap = std::max(8, (int)((budget - (size_t)NT * 81 * sizeof(double)) / per_row) / 8 * 8);
            const int nchunks = (R + cap - 1) / cap;
            const int per_job = (R + nchunks - 1) / nchunks;
            const long long nblk = (d.E * L + phi + threads_x - 1) / threads_x;
            for (int r0 = 0; r0 < R; r0 += per_job) {
                const int nr = std::min(per_job, R - r0);
                if (n_jobs >= kPosMaxJobs) {
                    fits = false;
                    break;
                }
                PosJob& j = pp.jobs[n_jobs++];
                j.first_block = (int)total_blocks;
                j.row0 = (unsigned short)(n_rows + r0);
                j.nrow = (unsigned short)nr;
                j.L = (unsigned short)L;
                j.phi = (unsigned short)phi;
                total_blocks += nblk;
                smem_max = std::max(smem_max, (size_t)((nr + 7) & ~7) * per_row + (size_t)NT * 81 * sizeof(double));
            }
            if (!fits)
                break;
            for (int r = 0; r < R; ++r)
                pp.rows[n_rows + r] = (unsigned short)c.second[(size_t)r];
            n_rows += R;
        }
        if (!fits || total_blocks > 0x7fffffffLL)
            return false;
        pp.n_jobs = n_jobs;
        if (total_blocks >= 148LL * 2 * 4 || budget <= 2048)
            break;
        budget /= 2;
    }
    return pp.n_jobs > 0;
}

template <int NT, int NTILE>
int combine_pos_launch(const DevTables& d, double* out, const PosConfig& cfg, cudaStream_t s) {
#ifndef LF_POS_BT
#define LF_POS_BT 256
#endif
#ifndef LF_POS_MINB
#define LF_POS_MINB 2
#endif
#ifndef LF_POS_G
#define LF_POS_G 4 // 32-position groups per warp: the staged rows and weights serve G * 256 positions
#endif
    constexpr int BT = LF_POS_BT, MINB = LF_POS_MINB, G = LF_POS_G;
    static thread_local PosParams pp;
    long long total_blocks = 0;
    size_t smem = 0;
    if (!build_pos_params(d, out, NT, G * (BT / 32) * 8 * NTILE, cfg, pp, total_blocks, smem))
        return -1;
    if (std::getenv("LAMFAST_POS_DEBUG")) {
        std::fprintf(stderr, "combine_pos: NT=%d NTILE=%d align=%d jobs=%d blocks=%lld smem=%zu\n", NT, NTILE,
                     cfg.align, pp.n_jobs, total_blocks, smem);
        for (int j = 0; j < pp.n_jobs; ++j)
            std::fprintf(stderr, "  job %d: L=%d phi=%d rows=%d (first i_t %d) first_block=%d\n", j, pp.jobs[j].L,
                         pp.jobs[j].phi, pp.jobs[j].nrow, pp.rows[pp.jobs[j].row0], pp.jobs[j].first_block);
    }
    auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)total_blocks, BT, smem, s>>>(d, pp, out);
    };
    if (d.affine)
        launch(k_combine_mma<NT, NTILE, true, BT, MINB, G>);
    else
        launch(k_combine_mma<NT, NTILE, false, BT, MINB, G>);
    return (int)cudaGetLastError();
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

} // namespace

/// Position-owned combine of a single-pass per-term plan (<= 7 terms).
/// Returns -1 when the launch is outside this form's limits (more rows or
/// classes than the parameter tables hold, no host copy of the thickness
/// adjacency): the caller falls back to the entry-owned kernel.
int launch_combine_pos(const DevTables& d, double* out, cudaStream_t stream) {
    if (d.n_passes != 1 || d.n_terms < 1 || d.n_terms > 4 || d.Etab)
        return -1;
    PosConfig cfg;
    cfg.align = env_int("LAMFAST_POS_ALIGN", 0);
    cfg.min_rows = env_int("LAMFAST_POS_MIN_ROWS", 8);
    cfg.smem = (size_t)env_int("LAMFAST_POS_SMEM_KB", 72) * 1024;
    if (cfg.align <= 0) {
        // rows per class first (they amortise a warp's position decode and P),
        // then the widest phase granularity that keeps them: 96 rows per
        // class on average, or what 32-byte phases already give
        cfg.align = 4;
        if (d.pre_t_h && d.len_t_h) {
            const long long addr0 = (long long)(reinterpret_cast<uintptr_t>(out) / sizeof(double));
            auto rows_per_class = [&](int A) {
                std::map<std::pair<int, long long>, int> cnt;
                for (int it = d.t0; it < d.t1; ++it) {
                    const long long base = 9 * d.S_s * (d.pre_t_h[it] - d.pre_t_h[d.t0]) - d.out_base;
                    ++cnt[{d.len_t_h[it], (((addr0 + base) % A) + A) % A}];
                }
                int big = 0, big_rows = 0; // classes that survive the merge, and their rows
                for (const auto& c : cnt)
                    if (c.second >= cfg.min_rows) {
                        ++big;
                        big_rows += c.second;
                    }
                return big ? (double)big_rows / big : 0.0;
            };
            const double want = std::min(96.0, rows_per_class(4));
            for (int A = 32; A > 4; A /= 2)
                if (rows_per_class(A) >= want) {
                    cfg.align = A;
                    break;
                }
        }
    }
    cfg.align = std::max(4, cfg.align / 4 * 4); // 256-bit stores need 32-byte aligned quads
#ifndef LF_POS_NTILE
#define LF_POS_NTILE 4 // 8-position tiles per warp (4: 32 positions, 8: 64)
#endif
    switch (d.n_terms) {
    case 1: return combine_pos_launch<1, LF_POS_NTILE>(d, out, cfg, stream);
    case 2: return combine_pos_launch<2, LF_POS_NTILE>(d, out, cfg, stream);
    case 3: return combine_pos_launch<3, LF_POS_NTILE>(d, out, cfg, stream);
    case 4: return combine_pos_launch<4, LF_POS_NTILE>(d, out, cfg, stream);
    default: return -1; // more terms: the split B operands would not fit the register file
    }
}

} // namespace lfb
