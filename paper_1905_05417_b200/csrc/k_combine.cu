// K4: the hot kernel -- P (x) q~ straight into the CSR value array
// (fast.cpp:211-264 + sparse.cpp:30-55), and its launcher.  The store
// variants measured slower in round 1 (team/TMA bulk copy, warp-specialised)
// are kept out of the product in tools/experiments/k_combine_variants.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "combine_common.cuh"

namespace lfb {

namespace {

// block -> (entry block, row chunk).  The row chunks run fastest in the
// launch order (grid x = chunk) where the entry blocks fit grid y: the blocks
// in flight then cover every chunk of a narrow entry window instead of one
// chunk of a wide one, which the store pattern likes better (C3 1.314 ->
// 1.275 ms, C4 2.50 -> 2.47 ms, profiles/r2_grid_order.txt).
#define LF_BLOCK_ENTRY (d.grid_swap ? blockIdx.y : blockIdx.x)
#define LF_BLOCK_CHUNK (d.grid_swap ? blockIdx.x : blockIdx.y)

/// grid of `nblk` entry blocks x `nchunk` row chunks, and the order flag for the kernel
inline dim3 combine_grid(long long nblk, unsigned nchunk, DevTables& d) {
#ifdef LF_NO_GRID_SWAP
    d.grid_swap = 0;
#else
    d.grid_swap = nblk >= 2048 && nblk <= 65535 ? 1 : 0; // small plans (C2: 473 entry blocks) ran 5% slower swapped
#endif
    return d.grid_swap ? dim3(nchunk, (unsigned)nblk) : dim3((unsigned)nblk, nchunk);
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
    bool live[EPT], in_s0[EPT], in_s1[EPT]; // in_s0/1: entry's function is >= s0 / < s1 (partial rows)
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
        // entry of slot x: e = blockIdx*256*EPT + warp*32*EPT + x*32 + lane, so
        // a warp's EPT stores per (row, k) are adjacent 256-byte runs (these
        // warp-contiguous slots measured C4 2.79 -> 2.66 ms against strided ones)
        const long long e = (long long)LF_BLOCK_ENTRY * BT * EPT + (threadIdx.x >> 5) * 32 * EPT + x * 32 +
                            (threadIdx.x & 31);
        live[x] = e < d.E;
        const long long ec = live[x] ? e : d.E - 1;
        int is = __ldg(d.blk_is + ec / kBlock);
        while (__ldg(d.es_pre + is + 1) <= ec)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(ec - ebase);
        in_s0[x] = is >= d.s0;
        in_s1[x] = is < d.s1;
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        B[x] = 3 * Lu * Lv; // row segment length per thickness neighbour
        const int a = r / B[x];
        const int rem = r - a * B[x];
        A[x] = ebase + (long long)a * B[x];
        o_thread[x] = out + (long long)rem;
#ifdef LF_STORE_ONLY_NOP // diagnostic: no P at all (the store pattern at the occupancy the launch bounds allow)
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int f = 0; f < 4; ++f)
                P[x][t][f] = 0.0;
#else
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
#endif
    }

    const int it_begin = d.t0 + LF_BLOCK_CHUNK * t_chunk;
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
            const int lt = ri.lt & 0xff, edge = ri.lt >> 8;
            // entries of a partial first / last row outside the range are not written
            bool lv[EPT];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                lv[x] = edge ? live[x] && (!(edge & 1) || in_s0[x]) && (!(edge & 2) || in_s1[x]) : live[x];
            double* o[EPT];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                o[x] = o_thread[x] + ri.base + (long long)lt * A[x];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                LF_CHECK(!lv[x] || (o[x] >= out && o[x] + (long long)(lt - 1) * B[x] < out + d.nnz_slab));
            const double4* w = s_w + rr * lt_max * NT;
            const unsigned char* kr = s_kr + rr * NT * 2;
#ifndef LF_NO_MASKED_ROWS
            // rows with <= 2 terms and L_t = 3 (bubble) or 5 (vertex) -- every
            // row of a C0 thickness space with one element per ply -- take the
            // branch-free bodies (combine_row_m).  Measured A/B
            // (profiles/r1_masked_rows.txt): 4 terms C3 1.341 -> 1.301 ms, C5
            // family 6.08 -> 5.88 ms; 3 terms (C4) 2.52 -> 2.65 ms, so 4 only.
#ifndef LF_MASKED_LTS
#define LF_MASKED_LTS 8 // bit L set: rows with L_t = L take the branch-free bodies (bubble rows
                        // only: C3 1.300 -> 1.295 ms, C5 family -0.3% against L_t 3 and 5)
#endif
#ifndef LF_MASKED_MIN_NT
#define LF_MASKED_MIN_NT 4
#endif
            if constexpr (EPT >= 2 && NT <= 4 && NT >= LF_MASKED_MIN_NT && !ACCUM) {
                if (((LF_MASKED_LTS >> 5) & 1) && lt == 5 && row_masked<NT, EPT, 5>(ri.mask, P, w, o, B, lv))
                    continue;
                if (((LF_MASKED_LTS >> 3) & 1) && lt == 3 && row_masked<NT, EPT, 3>(ri.mask, P, w, o, B, lv))
                    continue;
            }
#endif
            // EPT >= 2: k-outer rows (EPT live accumulators; C4 2.66 -> 2.53 ms,
            // C3 1.39 -> 1.33 ms with two entries per thread); EPT = 1: the
            // LT-unrolled form keeps more independent FMA chains in flight
            switch (lt) {
            case 1: row_dispatch<NT, EPT, 1, ACCUM>(P, w, ri.mask, kr, o, B, lv); break;
            case 2: row_dispatch<NT, EPT, 2, ACCUM>(P, w, ri.mask, kr, o, B, lv); break;
            case 3: row_dispatch<NT, EPT, 3, ACCUM>(P, w, ri.mask, kr, o, B, lv); break;
            case 4: row_dispatch<NT, EPT, 4, ACCUM>(P, w, ri.mask, kr, o, B, lv); break;
            case 5: row_dispatch<NT, EPT, 5, ACCUM>(P, w, ri.mask, kr, o, B, lv); break;
            case 7: row_dispatch<NT, EPT, 7, ACCUM>(P, w, ri.mask, kr, o, B, lv); break;
            default: combine_row_dyn<NT, EPT, ACCUM>(P, w, lt, ri.mask, o, B, lv); break;
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

template <int NT>
constexpr int entries_per_thread() { return NT <= 4 ? 2 : 1; } // two entries: 64 P registers at 4 terms

template <int NT, int EPT>
void combine_one_ept(const DevTables& d, double* out, int pass, int t_chunk, int stage_rows, int lt_max,
                     unsigned nchunk, cudaStream_t s, bool accum) {
    // two entries per thread: explicit bounds (<= 128 registers, 2 blocks of
    // 256 per SM); one entry: the compiler's own choice (80-128 registers)
#ifndef LF_COMBINE_BT
#define LF_COMBINE_BT 256 // threads per block (A/B knob)
#endif
    constexpr int BT = EPT >= 2 ? LF_COMBINE_BT : kBlock;
#ifndef LF_COMBINE_MINB
#define LF_COMBINE_MINB 2
#endif
    constexpr int MINB = LF_COMBINE_MINB;
    constexpr bool bounded = EPT >= 2;
    const size_t smem = ((stage_rows * (sizeof(RowInfo) + 2 * NT) + 31) & ~size_t(31)) +
                        (size_t)stage_rows * lt_max * NT * sizeof(double4);
    DevTables dl = d;
    const dim3 grid = combine_grid((d.E + (long long)BT * EPT - 1) / ((long long)BT * EPT), nchunk, dl);
    auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, BT, smem, s>>>(dl, out, pass, t_chunk, stage_rows, lt_max);
    };
    if constexpr (!bounded) {
        if (d.affine)
            accum ? launch(k_combine<NT, EPT, true, true>) : launch(k_combine<NT, EPT, true, false>);
        else
            accum ? launch(k_combine<NT, EPT, false, true>) : launch(k_combine<NT, EPT, false, false>);
    } else {
        if (d.affine)
            launch(k_combine_b<NT, EPT, true, false, BT, MINB>);
        else
            launch(k_combine_b<NT, EPT, false, false, BT, MINB>);
    }
}

/// Accumulating passes (> 8 terms) read the values they add to: one entry per
/// thread and the L_t-unrolled rows, whose loads of all L_t old values issue
/// together (k-outer rows would serialise load -> FMA -> store per neighbour:
/// measured 14.2 ms for the 2-term second pass of C4 with decompose_angles).
template <int NT>
void combine_one(const DevTables& d, double* out, int pass, int t_chunk, int stage_rows, int lt_max,
                 unsigned nchunk, cudaStream_t s, bool accum) {
    if (accum)
        combine_one_ept<NT, 1>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, s, true);
    else
        combine_one_ept<NT, entries_per_thread<NT>()>(d, out, pass, t_chunk, stage_rows, lt_max, nchunk, s,
                                                        false);
}

// ---------------------------------------------------------------------------
// Slot form of the per-term combine (affine geometry, 5 or more terms whose
// thickness rows each see at most NS of them: laminates with many distinct
// ply angles and one element per ply).  The per-term kernel above keeps the
// entry's P of EVERY term in registers, so it drops to one entry per thread
// at 5 terms and needs a read-modify-write pass per 8 terms; but a thickness
// row only touches the terms of the plies under its function.  Here a thread
// keeps the entry's nine term-independent 2D integrals I_xy and NS register
// slots of P; the host assigns each row's terms to slots (capi.cu,
// slot_schedule: a term keeps its slot while consecutive rows use it), and a
// slot is refilled from I_xy and C~ of its new term (9 FMA) only when its
// term changes -- once per ply.  Rows then run the same k-outer bodies as the
// per-term kernel with NS "terms": 4 FMA per value and active slot, one
// pass, two entries per thread for any term count.
template <int NS>
__device__ __forceinline__ void stage_rows_slots(const DevTables& d, int it0, int nrow, int lt_max, RowInfo* s_row,
                                                 unsigned char* s_kr, int* s_term, double4* s_w, int tid,
                                                 int nthreads) {
    const long long pre0 = __ldg(d.pre_t + d.t0);
    const long long preW = __ldg(d.pre_t + d.w_t0); // W / Wmask index base (the plan's rows)
    const long long nine_S = 9 * d.S_s;
    const int T = d.n_terms;
    for (int rr = tid; rr < nrow; rr += nthreads) {
        const int it = it0 + rr;
        const long long pfx = __ldg(d.pre_t + it) - preW;
        const int lt = __ldg(d.len_t + it);
        unsigned m = 0;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
            const int t = __ldg(d.slot_term + (long long)it * NS + sl);
            int lo = 255, hi = 0;
            if (t >= 0) {
                // Wmask: one word per (pass of 8 terms, pair), k_prepare_affine
                const unsigned* mk = d.Wmask + (long long)(t / 8) * d.n_pairs + pfx;
                const unsigned bit = 1u << (t % 8);
                for (int k = 0; k < lt; ++k)
                    if (__ldg(mk + k) & bit) {
                        lo = min(lo, k);
                        hi = k + 1;
                    }
            }
            if (hi > 0)
                m |= 1u << sl;
            s_kr[(rr * NS + sl) * 2] = (unsigned char)(lo == 255 ? 0 : lo);
            s_kr[(rr * NS + sl) * 2 + 1] = (unsigned char)hi;
            s_term[rr * NS + sl] = t;
        }
        s_row[rr].base = nine_S * (__ldg(d.pre_t + it) - pre0) - d.out_base;
        s_row[rr].lt = lt | row_edge(d, it) << 8;
        s_row[rr].mask = m;
    }
    const int nw = nrow * lt_max * NS;
    for (int idx = tid; idx < nw; idx += nthreads) {
        const int rr = idx / (lt_max * NS);
        const int k = (idx / NS) % lt_max;
        const int sl = idx % NS;
        const int it = it0 + rr;
        const int t = __ldg(d.slot_term + (long long)it * NS + sl);
        double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
        if (t >= 0 && k < __ldg(d.len_t + it)) {
            const long long q = __ldg(d.pre_t + it) - preW + k;
            const double2* src = reinterpret_cast<const double2*>(d.W + ((q * T) + t) * 4);
            const double2 lo2 = __ldg(src), hi2 = __ldg(src + 1);
            v = make_double4(lo2.x, lo2.y, hi2.x, hi2.y);
        }
        s_w[idx] = v;
    }
}

template <int NS, int EPT, int BT, int MINB, bool CT_SMEM>
__global__ void __launch_bounds__(BT, MINB) k_combine_slots(const DevTables d, double* __restrict__ out, int t_chunk,
                                                            int stage_rows, int lt_max) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RowInfo* s_row = reinterpret_cast<RowInfo*>(smem_raw);
    unsigned char* s_kr = smem_raw + stage_rows * sizeof(RowInfo); // [row][NS][2]
    int* s_term = reinterpret_cast<int*>(smem_raw + ((stage_rows * (sizeof(RowInfo) + 2 * NS) + 15) & ~15));
    double4* s_w = reinterpret_cast<double4*>(
        smem_raw + ((((stage_rows * (sizeof(RowInfo) + 2 * NS) + 15) & ~15) + stage_rows * NS * sizeof(int) + 31) & ~31));
    // C~ of every term behind the weights (the slot refills read it; from
    // global memory the refill's loads were the top stall), when it fits
    double* s_ct = reinterpret_cast<double*>(s_w + (size_t)stage_rows * lt_max * NS);
    if constexpr (CT_SMEM)
        for (int idx = threadIdx.x; idx < d.n_terms * 81; idx += BT)
            s_ct[idx] = __ldg(d.Ct + idx); // visible after the first staging barrier below

    double I[EPT][9]; // I00 I01 I10 I11 | I02 I12 | I20 I21 | I22 (x, y: 0 d/du, 1 d/dv, 2 value)
    int ab[EPT];
    double P[EPT][NS][4];
    double* o_thread[EPT];
    long long A[EPT];
    int B[EPT];
    bool live[EPT], in_s0[EPT], in_s1[EPT];
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
        // the entry slots of combine_body: a warp's EPT stores per (row, k) are adjacent 256-byte runs
        const long long e = (long long)LF_BLOCK_ENTRY * BT * EPT + (threadIdx.x >> 5) * 32 * EPT + x * 32 +
                            (threadIdx.x & 31);
        live[x] = e < d.E;
        const long long ec = live[x] ? e : d.E - 1;
        int is = __ldg(d.blk_is + ec / kBlock);
        while (__ldg(d.es_pre + is + 1) <= ec)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(ec - ebase);
        in_s0[x] = is >= d.s0;
        in_s1[x] = is < d.s1;
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        B[x] = 3 * Lu * Lv;
        const int a = r / B[x];
        const int rem = r - a * B[x];
        A[x] = ebase + (long long)a * B[x];
        o_thread[x] = out + (long long)rem;
        const int sp = rem / 3, b = rem - 3 * sp;
        const int sv = sp / Lu, su = sp - sv * Lu;
        ab[x] = 3 * a + b;
        const double* U = d.U + ((long long)iu * d.bu + su) * 4;
        const double* V = d.V + ((long long)iv * d.bv + sv) * 4;
        const double u0 = __ldg(U), u1 = __ldg(U + 1), u2 = __ldg(U + 2), u3 = __ldg(U + 3);
        const double v0 = __ldg(V), v1 = __ldg(V + 1), v2 = __ldg(V + 2), v3 = __ldg(V + 3);
        I[x][0] = u3 * v0, I[x][1] = u2 * v1, I[x][2] = u1 * v2, I[x][3] = u0 * v3;
        I[x][4] = u2 * v0, I[x][5] = u0 * v2, I[x][6] = u1 * v0, I[x][7] = u0 * v1, I[x][8] = u0 * v0;
#pragma unroll
        for (int sl = 0; sl < NS; ++sl)
#pragma unroll
            for (int f = 0; f < 4; ++f)
                P[x][sl][f] = 0.0;
    }
    int tag[NS]; // term whose P each slot holds (block-uniform)
#pragma unroll
    for (int sl = 0; sl < NS; ++sl)
        tag[sl] = -1;

    const int it_begin = d.t0 + LF_BLOCK_CHUNK * t_chunk;
    const int it_end = min(d.t1, it_begin + t_chunk);
    bool any_live = false;
#pragma unroll
    for (int x = 0; x < EPT; ++x)
        any_live |= live[x];

    for (int it0 = it_begin; it0 < it_end; it0 += stage_rows) {
        const int nrow = min(stage_rows, it_end - it0);
        if (it0 != it_begin)
            __syncthreads();
        stage_rows_slots<NS>(d, it0, nrow, lt_max, s_row, s_kr, s_term, s_w, threadIdx.x, BT);
        __syncthreads();
        if (!any_live)
            continue;
        for (int rr = 0; rr < nrow; ++rr) {
            const RowInfo ri = s_row[rr];
            const int lt = ri.lt & 0xff, edge = ri.lt >> 8;
            // slots whose term changes with this row: P of the new term from I_xy and C~ (affine_p's sums)
#pragma unroll
            for (int sl = 0; sl < NS; ++sl) {
                const int t = s_term[rr * NS + sl];
                if (t >= 0 && t != tag[sl]) {
                    tag[sl] = t;
#pragma unroll
                    for (int x = 0; x < EPT; ++x) {
                        double c[9];
#pragma unroll
                        for (int q = 0; q < 9; ++q)
                            c[q] = CT_SMEM ? s_ct[t * 81 + 9 * q + ab[x]] : __ldg(d.Ct + t * 81 + 9 * q + ab[x]);
                        P[x][sl][0] = c[0] * I[x][0] + c[1] * I[x][1] + c[3] * I[x][2] + c[4] * I[x][3];
                        P[x][sl][1] = c[2] * I[x][4] + c[5] * I[x][5];
                        P[x][sl][2] = c[6] * I[x][6] + c[7] * I[x][7];
                        P[x][sl][3] = c[8] * I[x][8];
                    }
                }
            }
            bool lv[EPT];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                lv[x] = edge ? live[x] && (!(edge & 1) || in_s0[x]) && (!(edge & 2) || in_s1[x]) : live[x];
            double* o[EPT];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                o[x] = o_thread[x] + ri.base + (long long)lt * A[x];
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                LF_CHECK(!lv[x] || (o[x] >= out && o[x] + (long long)(lt - 1) * B[x] < out + d.nnz_slab));
            const double4* w = s_w + rr * lt_max * NS;
            const unsigned char* kr = s_kr + rr * NS * 2;
#ifndef LF_SLOTS_MASKED_LTS
#define LF_SLOTS_MASKED_LTS 8 // bit L set: two-slot rows with L_t = L take the branch-free bodies; bubble rows
                              // only (profiles/r2_slots_masked.txt: C4 16 angles 2.73 -> 2.67 ms, also L_t = 5: 2.72)
#endif
            if constexpr (NS == 2 && LF_SLOTS_MASKED_LTS != 0) {
                if (((LF_SLOTS_MASKED_LTS >> 5) & 1) && lt == 5 && row_masked<NS, EPT, 5>(ri.mask, P, w, o, B, lv))
                    continue;
                if (((LF_SLOTS_MASKED_LTS >> 3) & 1) && lt == 3 && row_masked<NS, EPT, 3>(ri.mask, P, w, o, B, lv))
                    continue;
            }
            switch (lt) {
            case 1: row_dispatch<NS, EPT, 1, false>(P, w, ri.mask, kr, o, B, lv); break;
            case 2: row_dispatch<NS, EPT, 2, false>(P, w, ri.mask, kr, o, B, lv); break;
            case 3: row_dispatch<NS, EPT, 3, false>(P, w, ri.mask, kr, o, B, lv); break;
            case 4: row_dispatch<NS, EPT, 4, false>(P, w, ri.mask, kr, o, B, lv); break;
            case 5: row_dispatch<NS, EPT, 5, false>(P, w, ri.mask, kr, o, B, lv); break;
            case 7: row_dispatch<NS, EPT, 7, false>(P, w, ri.mask, kr, o, B, lv); break;
            default: combine_row_dyn<NS, EPT, false>(P, w, lt, ri.mask, o, B, lv); break;
            }
        }
    }
}

template <int NS>
int combine_slots_launch(const DevTables& d, double* out, int t_chunk, int lt_max, unsigned nchunk, cudaStream_t s) {
    constexpr int EPT = 2, BT = 256, MINB = 2;
    int stage_rows = (int)((24 * 1024) / ((size_t)lt_max * NS * sizeof(double4)));
    stage_rows = std::max(1, std::min(stage_rows, t_chunk));
    const size_t head = ((stage_rows * (sizeof(RowInfo) + 2 * NS) + 15) & ~size_t(15)) + (size_t)stage_rows * NS * sizeof(int);
    size_t smem = ((head + 31) & ~size_t(31)) + (size_t)stage_rows * lt_max * NS * sizeof(double4);
    const size_t ct_bytes = (size_t)d.n_terms * 81 * sizeof(double);
    const int ct_smem = smem + ct_bytes <= 96 * 1024; // two blocks per SM keep their shared memory
    if (ct_smem)
        smem += ct_bytes;
    DevTables dl = d;
    const dim3 grid = combine_grid((d.E + (long long)BT * EPT - 1) / ((long long)BT * EPT), nchunk, dl);
    auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, BT, smem, s>>>(dl, out, t_chunk, stage_rows, lt_max);
    };
    if (ct_smem)
        launch(k_combine_slots<NS, EPT, BT, MINB, true>);
    else
        launch(k_combine_slots<NS, EPT, BT, MINB, false>);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Coefficient form of K4 for affine geometry with many operator terms
// (decompose_angles: 5 per material; laminates with > 8 distinct angles).
// With a constant frame every term's P is linear in the same nine 2D
// integrals I_xy of the entry, so the whole sum over terms and families
//   K = sum_t sum_f W[pair][t][f] P_{t,f} = sum_xy I_xy E[pair][ab][xy],
//   E[pair][ab][xy] = sum_t Ct[t][xy][ab] W[pair][t][f(xy)]
// costs 9 FMA per value whatever the term count.  E (720 B per thickness
// pair) is formed once per assembly by k_pair_coeffs; the combine keeps the
// entry's nine I_xy in registers and streams E rows through shared memory.
// One launch, every value written once (the per-term form needed one
// read-modify-write pass per 8 terms: 24 B/nnz of traffic for 10 terms).
__global__ void k_pair_coeffs(const DevTables d) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= d.n_pairs * 81)
        return;
    const long long pp = g / 81;
    const int r = (int)(g - pp * 81), ab = r / 9, xy = r - 9 * ab;
    // family of xy: {00,01,10,11} -> P11, {02,12} -> P12, {20,21} -> P21, 22 -> P22
    const int x = xy / 3, y = xy - 3 * x;
    const int f = (x < 2 && y < 2) ? 0 : (x < 2) ? 1 : (y < 2) ? 2 : 3;
    double e = 0.0;
    for (int t = 0; t < d.n_terms; ++t)
        e = fma(d.Ct[(long long)t * 81 + xy * 9 + ab], d.W[(pp * d.n_terms + t) * 4 + f], e);
    d.Etab[pp * kEPair + ab * kEStride + xy] = e;
}

// Thread mapping.  A warp owns 32 consecutive in-plane pairs (i_s, slot) of
// one row-component a (the pairs of each a are padded to a multiple of 32, so
// a is warp-uniform and every coefficient load is a shared-memory broadcast).
// Per (row, neighbour) the warp writes the 96 values (pair, b) of its pairs:
// lane t stores values j = t + 32 m, m = 0..2, i.e. pair j / 3 and b = j % 3,
// so each of its three stores is one contiguous 256-byte run across the warp
// (except where a segment of the row ends).  Since 32 = 2 mod 3, a lane's
// three values carry the three different b, so the lane keeps, for every b,
// the nine I_xy of the pair it stores with that b (J[b], selected once) and
// forms w_b = sum_xy J[b][xy] E[pair][3a + b][xy] with the same broadcast
// coefficient rows as every other lane.  With NS sets of 32 pairs per warp
// every broadcast feeds NS FMA per lane.  Measured (C4 / C3 combine ms,
// profiles/r2_eform_*.txt, r2_coef_*.txt): one entry per thread 5.62 / 2.80;
// one triple per thread with 24-byte-stride stores 5.66 / 2.67 (ncu: LSU
// data pipe 74%, three shared wavefronts per coefficient load); this mapping
// 4.39 / 1.98, with split FMA chains and component-local staging 4.09 / 1.78
// (NS = 1, 16 warps/SM), NS = 2 at 254 registers (8 warps/SM) 4.04 / 1.75.
// The per-term form it replaces above 7 terms needs one read-modify-write
// pass per 8 terms: C4 decompose_angles 14.6 ms, 16 distinct angles 12.3 ms.
template <int BT, int NS, int MINB>
__global__ void __launch_bounds__(BT, MINB) k_combine_coef(const DevTables d, double* __restrict__ out, int t_chunk,
                                                           int stage_rows, int lt_max, long long s_pad) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // s_row: the chunk's rows; two coefficient-row buffers, the next stage's
    // cp.async copies in flight while the current one is consumed
    RowInfo* s_row = reinterpret_cast<RowInfo*>(smem_raw);
    double* s_ebuf = reinterpret_cast<double*>(smem_raw + ((t_chunk * sizeof(RowInfo) + 15) & ~15));
    const int lane = threadIdx.x & 31;
    // first pair slot of the warp; the warp owns NS sets of 32 consecutive pairs
    const long long w0 = ((long long)blockIdx.x * BT + threadIdx.x - lane) * NS;
    const int a = (int)(w0 / s_pad);
    const bool warp_live = a < 3;
    const long long ps0 = w0 - (long long)a * s_pad;
    // the block stages only the coefficient rows ab = 3 a + b of the
    // components its warps carry (one a, or two where the block straddles)
    const int a_lo = (int)min(2LL, (long long)blockIdx.x * BT * NS / s_pad);
    const int a_hi = (int)min(2LL, ((long long)blockIdx.x * BT + BT - 1) * NS / s_pad);
    const int k_stride = 3 * (a_hi - a_lo + 1) * kEStride; // doubles per staged (row, k)
    const int coff = 3 * (min(a, 2) - a_lo) * kEStride;
    double J[NS][3][9];
    int A[NS][3], B[NS][3], R[NS][3], bsel[3];
    unsigned live = 0, in_s0 = 0, in_s1 = 0; // bit 3 s + m
#pragma unroll
    for (int m = 0; m < 3; ++m)
        bsel[m] = (lane + 32 * m) % 3;
#pragma unroll
    for (int st = 0; st < NS; ++st)
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            const int j = lane + 32 * m;
            const int b = bsel[m];
            const long long ps = ps0 + 32 * st + j / 3;
            const bool lv = warp_live && ps < d.S_s;
            live |= (lv ? 1u : 0u) << (3 * st + m);
            const long long e = 9 * (lv ? ps : d.S_s - 1);
            int is = __ldg(d.blk_is + e / kBlock);
            while (__ldg(d.es_pre + is + 1) <= e)
                ++is;
            const long long ebase = __ldg(d.es_pre + is);
            const int slot = (int)((e - ebase) / 9);
            in_s0 |= (is >= d.s0 ? 1u : 0u) << (3 * st + m);
            in_s1 |= (is < d.s1 ? 1u : 0u) << (3 * st + m);
            const int iu = is % d.nu, iv = is / d.nu;
            const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
            B[st][m] = 3 * Lu * Lv;
            A[st][m] = (int)(ebase + (long long)min(a, 2) * B[st][m]);
            R[st][m] = 3 * slot + b;
            const int sv = slot / Lu, su = slot - sv * Lu;
            const double* U = d.U + ((long long)iu * d.bu + su) * 4;
            const double* V = d.V + ((long long)iv * d.bv + sv) * 4;
            const double u0 = __ldg(U), u1 = __ldg(U + 1), u2 = __ldg(U + 2), u3 = __ldg(U + 3);
            const double v0 = __ldg(V), v1 = __ldg(V + 1), v2 = __ldg(V + 2), v3 = __ldg(V + 3);
            // xy = 3x + y, x/y: 0 -> d/du, 1 -> d/dv, 2 -> value (affine_p)
            const double I[9] = {u3 * v0, u2 * v1, u2 * v0, u1 * v2, u0 * v3, u0 * v2, u1 * v0, u0 * v1, u0 * v0};
            // J[st][b] = I of the value this lane stores with component b
#pragma unroll
            for (int bb = 0; bb < 3; ++bb)
#pragma unroll
                for (int xy = 0; xy < 9; ++xy)
                    if (bb == b)
                        J[st][bb][xy] = I[xy];
        }
    // staging assignment: a row's lt_max * k_stride / 2 chunks spread over the
    // block, st_rows rows per pass (st_h < 0: more chunks per row than threads)
    const int row_chunks = lt_max * (k_stride / 2);
    const int st_rows = BT / row_chunks;
    int st_r = 0, st_k = 0, st_h = -1;
    if (st_rows > 0 && (int)threadIdx.x < st_rows * row_chunks) {
        st_r = threadIdx.x / row_chunks;
        const int r = threadIdx.x - st_r * row_chunks;
        st_k = r / (k_stride / 2);
        st_h = r - st_k * (k_stride / 2);
    } else if (st_rows > 0) {
        st_h = -2; // idle in staging
    }
    const int it_begin = d.t0 + blockIdx.y * t_chunk;
    const int it_end = min(d.t1, it_begin + t_chunk);
    const long long pre0 = __ldg(d.pre_t + d.t0), preW = __ldg(d.pre_t + d.w_t0), nine_S = 9 * d.S_s;
    for (int rr = threadIdx.x; rr < it_end - it_begin; rr += BT) {
        const int it = it_begin + rr;
        s_row[rr].base = nine_S * (__ldg(d.pre_t + it) - pre0) - d.out_base;
        s_row[rr].lt = __ldg(d.len_t + it) | row_edge(d, it) << 8;
        s_row[rr].mask = 0;
    }
    const int stage_doubles = stage_rows * lt_max * k_stride;
    const double* eb = d.Etab + 3 * a_lo * kEStride;
    // issue the cp.async copies of stage rows [i0, i0 + stage_rows) into buf
    // (16-byte chunks; neighbours k >= L_t(it) are zero-filled)
    auto issue = [&](int i0, double* buf) {
        const int nrow = min(stage_rows, it_end - i0);
        const int per_k = k_stride / 2;
        if (st_rows > 0) {
            for (int rr = st_r; st_h >= 0 && rr < nrow; rr += st_rows) {
                const int it = i0 + rr;
                const bool ok = st_k < __ldg(d.len_t + it);
                const double* src = ok ? eb + (__ldg(d.pre_t + it) - preW + st_k) * kEPair + 2 * st_h : eb;
                cp_async16(buf + ((rr * lt_max + st_k) * per_k + st_h) * 2, src, ok);
            }
        } else {
            for (int idx = threadIdx.x; idx < nrow * lt_max * per_k; idx += BT) {
                const int rk = idx / per_k, h = idx - rk * per_k;
                const int rr = rk / lt_max, kk = rk - rr * lt_max;
                const int it = i0 + rr;
                const bool ok = kk < __ldg(d.len_t + it);
                const double* src = ok ? eb + (__ldg(d.pre_t + it) - preW + kk) * kEPair + 2 * h : eb;
                cp_async16(buf + 2 * idx, src, ok);
            }
        }
        cp_async_commit();
    };
    if (it_begin < it_end)
        issue(it_begin, s_ebuf);
    int stage = 0;
    for (int it0 = it_begin; it0 < it_end; it0 += stage_rows, ++stage) {
        const int nrow = min(stage_rows, it_end - it0);
        double* const s_e = s_ebuf + (stage & 1) * stage_doubles;
        if (it0 + stage_rows < it_end)
            issue(it0 + stage_rows, s_ebuf + ((stage + 1) & 1) * stage_doubles);
        else
            cp_async_commit(); // empty group: the wait below always leaves one group pending
        cp_async_wait1();
        __syncthreads();
        for (int rr = 0; live && rr < nrow; ++rr) {
            const RowInfo ri = s_row[it0 - it_begin + rr];
            const int lt = ri.lt & 0xff, edge = ri.lt >> 8;
            const unsigned lv = live & ((edge & 1) ? in_s0 : ~0u) & ((edge & 2) ? in_s1 : ~0u);
            // 32-bit offsets inside the row block (< 9 S_s L_t values) from one
            // 64-bit row base: one IMAD.WIDE per store instead of 64-bit pointer arithmetic
            double* const rowp = out + ri.base;
            int o[NS][3];
            bool sb[NS][3];
#pragma unroll
            for (int st = 0; st < NS; ++st)
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    o[st][m] = lt * A[st][m] + R[st][m];
                    sb[st][m] = (lv >> (3 * st + m)) & 1u;
                }
            const double* er = s_e + (long long)rr * lt_max * k_stride + coff;
            for (int k = 0; k < lt; ++k) {
                const double2* c = reinterpret_cast<const double2*>(er + k * k_stride);
                double w[NS][3];
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    // coefficients of component b: er[k][10 b + xy], xy < 9 (five 16-byte
                    // broadcasts, each feeding NS FMA per lane); two partial sums per value
                    // halve the dependent FMA chain
                    const double2 c0 = c[5 * b], c1 = c[5 * b + 1], c2 = c[5 * b + 2], c3 = c[5 * b + 3],
                                  c4 = c[5 * b + 4];
#pragma unroll
                    for (int st = 0; st < NS; ++st) {
                        const double* Jb = J[st][b];
                        double s0 = Jb[0] * c0.x, s1 = Jb[1] * c0.y;
                        s0 = fma(Jb[2], c1.x, s0);
                        s1 = fma(Jb[3], c1.y, s1);
                        s0 = fma(Jb[4], c2.x, s0);
                        s1 = fma(Jb[5], c2.y, s1);
                        s0 = fma(Jb[6], c3.x, s0);
                        s1 = fma(Jb[7], c3.y, s1);
                        s0 = fma(Jb[8], c4.x, s0);
                        w[st][b] = s0 + s1;
                    }
                }
#pragma unroll
                for (int st = 0; st < NS; ++st)
#pragma unroll
                    for (int m = 0; m < 3; ++m) {
                        const double val = bsel[m] == 0 ? w[st][0] : bsel[m] == 1 ? w[st][1] : w[st][2];
                        double* const p = rowp + o[st][m];
                        LF_CHECK(!sb[st][m] || (p >= out && p < out + d.nnz_slab));
                        store_value_if(p, val, sb[st][m]);
                        o[st][m] += B[st][m];
                    }
            }
        }
        __syncthreads(); // every warp is done with this buffer before the next issue refills it
    }
    cp_async_wait0();
}

} // namespace

int launch_combine(const DevTables& d, double* out, int t_chunk, cudaStream_t stream, int* launches) {
    if (d.E == 0 || d.t1 <= d.t0)
        return 0;
    const long long nblk = (d.E + kBlock - 1) / kBlock; // 256-entry sub-blocks
    const int nt = d.t1 - d.t0;
    if (t_chunk <= 0) {
        if (const char* env = std::getenv("LAMFAST_TCHUNK"))
            t_chunk = std::atoi(env);
    }
    if (t_chunk <= 0) {
        // 48 thickness rows per block amortise the per-block prologue (P in
        // registers, entry decode, staging); shorter chunks (down to 32) only
        // while the grid is under ~4 waves of 2 resident blocks on 148 SMs.
        // Measured sweeps: profiles/r1_tchunk_sweep.txt (k-outer rows: C4 48
        // rows 2.488 ms vs 64 rows 2.520 ms; C3 48 rows already the balanced choice).
        const long long blocks_x = (nblk + 1) / 2; // two entries per thread for <= 4 terms
        // general geometry loads P from HBM once per block: whole-slab chunks
        // (measured C3 bilinear 1.47 -> 1.38 ms); affine P is recomputed, so
        // shorter chunks balance better (profiles/r1_tchunk_sweep.txt)
        // (C5 family, 32 k entry blocks of p = 3 four-term entries: ~100-row chunks amortise the
        // heavier entry prologue, 193 rows 18.63 -> 17.88 ms, profiles/r2_grid_order.txt; C3 / C4
        // with 3.7 k entry blocks keep 48)
        t_chunk = d.affine ? std::min(nt, blocks_x >= 16384 ? 112 : 48) : nt;
        while (!d.affine && t_chunk > 64 && blocks_x * ((nt + t_chunk - 1) / t_chunk) < 148LL * 2 * 4)
            t_chunk = (t_chunk + 1) / 2;
        while (t_chunk > 32 && blocks_x * ((nt + t_chunk - 1) / t_chunk) < 148LL * 2 * 4)
            t_chunk /= 2;
        const int nchunks = (nt + t_chunk - 1) / t_chunk; // balance, in multiples of 16 rows
        t_chunk = std::min(nt, ((nt + nchunks - 1) / nchunks + 15) / 16 * 16);
    }
    const unsigned nchunk = (unsigned)((nt + t_chunk - 1) / t_chunk);
    const int lt_max = std::max(1, d.lt_max);
    if (d.Etab) {
        // coefficient form: one launch for any term count; ~32 KB of staged
        // coefficient rows (two components a per block at most when a
        // component's pairs fill a block, else all three)
#ifndef LF_COEF_BT
#define LF_COEF_BT 256
#endif
#ifndef LF_COEF_NS
#define LF_COEF_NS 2
#endif
#ifndef LF_COEF_MINB
#define LF_COEF_MINB 1
#endif
        constexpr int BT = LF_COEF_BT, NS = LF_COEF_NS, MINB = LF_COEF_MINB;
        const long long s_pad = (d.S_s + 32 * NS - 1) / (32 * NS) * (32 * NS); // pairs per component, warp-padded
        const int nab = s_pad >= (long long)BT * NS ? 6 : 9;
        int stage_rows = (int)((32 * 1024) / ((size_t)lt_max * nab * kEStride * sizeof(double)));
        stage_rows = std::max(1, std::min(stage_rows, t_chunk));
        // the chunk's rows + two coefficient-row stage buffers
        const size_t smem = ((t_chunk * sizeof(RowInfo) + 15) & ~size_t(15)) +
                            2 * (size_t)stage_rows * lt_max * nab * kEStride * sizeof(double);
        auto kern = k_combine_coef<BT, NS, MINB>;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const long long warps = 3 * s_pad / (32 * NS);
        const dim3 grid((unsigned)((warps * 32 + BT - 1) / BT), nchunk);
        kern<<<grid, BT, smem, stream>>>(d, out, t_chunk, stage_rows, lt_max, s_pad);
        if (launches)
            ++*launches;
        return (int)cudaGetLastError();
    }
    if (d.n_slots > 0 && d.slot_term && d.affine) {
        // slot form: one pass for any term count (rows see <= n_slots terms each)
        const int rc = d.n_slots <= 2 ? combine_slots_launch<2>(d, out, t_chunk, lt_max, nchunk, stream)
                                      : combine_slots_launch<3>(d, out, t_chunk, lt_max, nchunk, stream);
        if (launches)
            ++*launches;
        return rc;
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


int launch_pair_coeffs(const DevTables& d, cudaStream_t stream) {
    if (d.n_pairs == 0)
        return 0;
    const long long n = d.n_pairs * 81;
    k_pair_coeffs<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d);
    return (int)cudaGetLastError();
}

} // namespace lfb
