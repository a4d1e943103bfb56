// Opt-in store variants of K4 (profiles/r1_store_modes.md): the team/TMA
// bulk-copy combine (LAMFAST_TEAM) and the warp-specialised combine
// (LAMFAST_WS).  Both are parity-tested and measured slower than the default
// direct-store k_combine; they stay as documented experiments.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "combine_common.cuh"

namespace lfb {
namespace {

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
    extern __shared__ __align__(128) unsigned char smem_raw[];
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

} // namespace

bool launch_combine_variant(const DevTables& d, double* out, int t_chunk_req, int lt_max, cudaStream_t stream,
                            int* launches) {
    bool done = false;
    switch (d.n_terms) {
    case 1: done = combine_team<1>(d, out, t_chunk_req, lt_max, stream, launches); break;
    case 2: done = combine_team<2>(d, out, t_chunk_req, lt_max, stream, launches); break;
    case 3: done = combine_team<3>(d, out, t_chunk_req, lt_max, stream, launches); break;
    case 4: done = combine_team<4>(d, out, t_chunk_req, lt_max, stream, launches); break;
    default: break;
    }
    if (done)
        return true;
    switch (d.n_terms) {
    case 1: done = combine_ws<1>(d, out, lt_max, stream, launches); break;
    case 2: done = combine_ws<2>(d, out, lt_max, stream, launches); break;
    case 3: done = combine_ws<3>(d, out, lt_max, stream, launches); break;
    case 4: done = combine_ws<4>(d, out, lt_max, stream, launches); break;
    default: break;
    }
    return done;
}

} // namespace lfb
