// K4, position-owned form: P (x) q~ straight into the CSR value array
// (fast.cpp:211-264 + sparse.cpp:30-55) with line-aligned warp stores.
//
// The values of one thickness row i_t are one contiguous range of
// L_t(i_t) * E doubles (E = 9 S_s in-plane entries), ordered
// (i_s, a, k, slot, b).  k_combine (k_combine.cu) gives a thread one in-plane
// entry and lets it write that entry's L_t values of every row: its warp
// stores are 256-byte runs at the 8-byte alignment the odd row-segment length
// 3 L_s dictates, and the store pattern alone sets that kernel's time
// (profiles/r2_storeonly.txt; tools/store_pattern_bench.cu: 4.3 TB/s for that
// pattern against 7.05 TB/s for 256-byte-aligned pieces).
//
// Here a thread owns a POSITION of the row range instead: thread tau of a
// class of rows writes values[base(i_t) - phi + tau] for every row of the
// class, where a class holds the rows with the same L_t and the same phase
// phi = (address of the row range / 8) mod A.  Every warp store is then one
// contiguous 256-byte run aligned to 8 A bytes, a block writes 4 KB
// contiguous pieces, and nothing is staged.  The position's in-plane entry
// and neighbour (i_s, a, k, slot, b) are the same for every row of the class,
// so the thread keeps that entry's P_{t,f} in registers as before and reads
// the weights of pair (i_t, k) from shared memory (a warp spans at most a few
// different k).  Per-(neighbour, term) range tests are gone: a pair a term
// does not reach has exactly zero weights (k_prepare_affine /
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
    unsigned mask;  // union of the term masks of the row's pairs (this pass)
    int edge;       // row_edge(): partial first / last row of a function range
};

#ifndef LF_POS_SWITCH_NT
#define LF_POS_SWITCH_NT 4 // term counts whose rows take one straight-line body per term set
#endif

/// Value of EPT positions for a row whose active terms are the compile-time
/// set M: all weight loads first, one FMA chain per term, then their sum.
template <int NT, int EPT, unsigned M>
__device__ __forceinline__ void pos_row_m(const double (&P)[EPT][NT][4], const double4* __restrict__ w,
                                          const int (&koff)[EPT], double (&acc)[EPT]) {
    double4 ww[EPT][NT];
#pragma unroll
    for (int t = 0; t < NT; ++t)
        if ((M >> t) & 1u) {
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                ww[x][t] = w[koff[x] + t];
        }
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
        double sum = 0.0;
        bool first = true;
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if ((M >> t) & 1u) {
                double c = P[x][t][0] * ww[x][t].x;
                c = fma(P[x][t][1], ww[x][t].y, c);
                c = fma(P[x][t][2], ww[x][t].z, c);
                c = fma(P[x][t][3], ww[x][t].w, c);
                sum = first ? c : sum + c;
                first = false;
            }
        acc[x] = sum;
    }
}

template <int NT, int EPT, bool AFFINE, int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB)
    k_combine_pos(const __grid_constant__ DevTables d, const __grid_constant__ PosParams pp,
                  double* __restrict__ out, int pass) {
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
    const long long xb = (long long)((int)blockIdx.x - pp.jobs[jlo].first_block);
    PosRow* s_row = reinterpret_cast<PosRow*>(smem_raw);
    double4* s_w = reinterpret_cast<double4*>(smem_raw + ((nrow * sizeof(PosRow) + 31) & ~size_t(31)));

    const int t_first = pass * 8;
    const long long EL = d.E * L;
    double P[EPT][NT][4];
    double* op[EPT];
    int koff[EPT];
    unsigned flags[EPT]; // bit 0: i_s >= s0, bit 1: i_s < s1
    bool live[EPT];
    bool any_live = false;
#pragma unroll
    for (int x = 0; x < EPT; ++x) {
        // a warp's EPT stores per row are adjacent 256-byte runs
        const long long tau = xb * (BT * EPT) + (threadIdx.x >> 5) * (32 * EPT) + x * 32 + (threadIdx.x & 31);
        const long long o = tau - phi;
        live[x] = o >= 0 && o < EL;
        any_live |= live[x];
        const long long oc = live[x] ? o : 0;
        const long long e1 = oc / L; // lies inside the entry range of the position's i_s
        int is = __ldg(d.blk_is + e1 / kBlock);
        while (__ldg(d.es_pre + is + 1) <= e1)
            ++is;
        const long long ebase = __ldg(d.es_pre + is);
        const int r = (int)(oc - (long long)L * ebase); // offset inside the (i_t, i_s) row block
        flags[x] = (is >= d.s0 ? 1u : 0u) | (is < d.s1 ? 2u : 0u);
        const int iu = is % d.nu, iv = is / d.nu;
        const int Lu = __ldg(d.len_u + iu), Lv = __ldg(d.len_v + iv);
        const int B = 3 * Lu * Lv; // row segment length per thickness neighbour
        const int a = r / (L * B);
        const int r2 = r - a * (L * B);
        const int k = r2 / B;
        const int rem = r2 - k * B;
        koff[x] = k * NT;
        op[x] = out + tau;
        if constexpr (AFFINE) {
            const int s = rem / 3, b = rem - 3 * s;
            const int sv = s / Lu, su = s - sv * Lu;
            affine_p<NT>(d, iu, iv, su, sv, 3 * a + b, t_first, P[x]);
        } else {
            const long long ec = ebase + (long long)a * B + rem;
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    P[x][t][f] = __ldg(d.Pg + ((long long)(t_first + t) * 4 + f) * d.E + ec);
        }
    }

    // stage the job's rows: PosRow and the weights s_w[row][k][term]
    {
        const long long pre0 = __ldg(d.pre_t + d.t0);
        const long long preW = __ldg(d.pre_t + d.w_t0); // W / Wmask index base (the plan's rows)
        const long long nine_S = 9 * d.S_s;
        const unsigned* mask_base = d.Wmask + (long long)pass * d.n_pairs;
        for (int rr = threadIdx.x; rr < nrow; rr += BT) {
            const int it = pp.rows[row0 + rr];
            const long long pre = __ldg(d.pre_t + it);
            unsigned m = 0;
            for (int k = 0; k < L; ++k)
                m |= __ldg(mask_base + (pre - preW) + k);
            PosRow ri;
            ri.base = nine_S * (pre - pre0) - d.out_base - phi;
            ri.mask = m;
            ri.edge = row_edge(d, it);
            s_row[rr] = ri;
        }
        const int per_row = L * NT, nw = nrow * per_row;
        for (int idx = threadIdx.x; idx < nw; idx += BT) {
            const int rr = idx / per_row;
            const int kt = idx - rr * per_row;
            const int k = kt / NT, t = kt - k * NT;
            const int it = pp.rows[row0 + rr];
            const long long q = __ldg(d.pre_t + it) - preW + k;
            const double2* src = reinterpret_cast<const double2*>(d.W + ((q * d.n_terms) + t_first + t) * 4);
            const double2 lo2 = __ldg(src), hi2 = __ldg(src + 1);
            s_w[idx] = make_double4(lo2.x, lo2.y, hi2.x, hi2.y);
        }
    }
    __syncthreads();
    if (!any_live)
        return;

    const double4* w = s_w;
    for (int rr = 0; rr < nrow; ++rr, w += L * NT) {
        const PosRow ri = s_row[rr];
        double acc[EPT];
#ifdef LF_STORE_ONLY
#pragma unroll
        for (int x = 0; x < EPT; ++x)
            acc[x] = 0.0;
#else
        if constexpr (NT <= LF_POS_SWITCH_NT) {
            // one straight-line body per term set of the row: every weight load
            // issues before the first FMA, one independent FMA chain per term
            switch (ri.mask) {
#define LF_POS_M(m)                                          \
    case m:                                                  \
        if constexpr (((m) >> NT) == 0u)                     \
            pos_row_m<NT, EPT, m>(P, w, koff, acc);          \
        break;
                LF_POS_M(1u) LF_POS_M(2u) LF_POS_M(3u) LF_POS_M(4u) LF_POS_M(5u) LF_POS_M(6u) LF_POS_M(7u)
                LF_POS_M(8u) LF_POS_M(9u) LF_POS_M(10u) LF_POS_M(11u) LF_POS_M(12u) LF_POS_M(13u)
                LF_POS_M(14u) LF_POS_M(15u)
#undef LF_POS_M
            default:
#pragma unroll
                for (int x = 0; x < EPT; ++x)
                    acc[x] = 0.0;
                break;
            }
        } else {
#pragma unroll
            for (int x = 0; x < EPT; ++x)
                acc[x] = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (ri.mask & (1u << t)) {
#pragma unroll
                    for (int x = 0; x < EPT; ++x) {
                        const double4 ww = w[koff[x] + t];
                        acc[x] = fma(P[x][t][0], ww.x, acc[x]);
                        acc[x] = fma(P[x][t][1], ww.y, acc[x]);
                        acc[x] = fma(P[x][t][2], ww.z, acc[x]);
                        acc[x] = fma(P[x][t][3], ww.w, acc[x]);
                    }
                }
            }
        }
#endif
#pragma unroll
        for (int x = 0; x < EPT; ++x) {
            // positions of a partial first / last row outside the range are not written
            const unsigned pred = live[x] && (ri.edge & ~flags[x]) == 0;
            double* const p = op[x] + ri.base;
            LF_CHECK(!pred || (p >= out && p < out + d.nnz_slab));
            store_value_if(p, acc[x], pred);
        }
    }
}

struct PosConfig {
    int align;     // phase granularity A in values (32: 256-byte aligned warp stores)
    int min_rows;  // classes with fewer rows join the largest class of their L_t (unaligned there)
    size_t smem;   // shared-memory budget per block (rows per job)
};

/// Classes (L_t, phase), row chunks and the flat block map of one launch.
/// false: outside the limits of the kernel-parameter tables (the entry-owned
/// k_combine then takes the launch).
bool build_pos_params(const DevTables& d, const double* out, int NT, int threads_x, const PosConfig& cfg,
                      PosParams& pp, long long& total_blocks, size_t& smem_max) {
    if (!d.pre_t_h || !d.len_t_h || d.t1 - d.t0 > kPosMaxRows || d.t1 > 65535)
        return false;
    const long long A = cfg.align;
    const long long addr0 = (long long)(reinterpret_cast<uintptr_t>(out) / sizeof(double));
    // rows by (L, phi)
    std::map<std::pair<int, int>, std::vector<int>> cls;
    for (int it = d.t0; it < d.t1; ++it) {
        const int L = d.len_t_h[it];
        if (L <= 0)
            continue;
        if (L > 65535)
            return false;
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
    // rows per job from the shared-memory budget; more, shorter jobs while the grid is under ~4 waves
    size_t budget = cfg.smem;
    for (;;) {
        int n_jobs = 0, n_rows = 0;
        total_blocks = 0;
        smem_max = 0;
        bool fits = true;
        for (const auto& c : cls) {
            const int L = c.first.first, phi = c.first.second, R = (int)c.second.size();
            const size_t per_row = sizeof(PosRow) + (size_t)L * NT * sizeof(double4);
            const int cap = (int)std::max<size_t>(1, (budget - 32) / per_row);
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
                smem_max = std::max(smem_max, ((nr * sizeof(PosRow) + 31) & ~size_t(31)) +
                                                  (size_t)nr * L * NT * sizeof(double4));
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

template <int NT, int EPT>
int combine_pos_launch(const DevTables& d, double* out, int pass, const PosConfig& cfg, cudaStream_t s) {
#ifndef LF_POS_BT
#define LF_POS_BT 256
#endif
#ifndef LF_POS_MINB
#define LF_POS_MINB 2
#endif
    constexpr int BT = LF_POS_BT, MINB = LF_POS_MINB;
    static thread_local PosParams pp;
    long long total_blocks = 0;
    size_t smem = 0;
    if (!build_pos_params(d, out, NT, BT * EPT, cfg, pp, total_blocks, smem))
        return -1;
    if (std::getenv("LAMFAST_POS_DEBUG")) {
        std::fprintf(stderr, "combine_pos: NT=%d EPT=%d align=%d jobs=%d blocks=%lld smem=%zu\n", NT, EPT, cfg.align,
                     pp.n_jobs, total_blocks, smem);
        for (int j = 0; j < pp.n_jobs; ++j)
            std::fprintf(stderr, "  job %d: L=%d phi=%d rows=%d (first i_t %d) first_block=%d\n", j, pp.jobs[j].L,
                         pp.jobs[j].phi, pp.jobs[j].nrow, pp.rows[pp.jobs[j].row0], pp.jobs[j].first_block);
    }
    auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)total_blocks, BT, smem, s>>>(d, pp, out, pass);
    };
    if (d.affine)
        launch(k_combine_pos<NT, EPT, true, BT, MINB>);
    else
        launch(k_combine_pos<NT, EPT, false, BT, MINB>);
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
    if (d.n_passes != 1 || d.n_terms < 1 || d.n_terms > 7 || d.Etab)
        return -1;
    PosConfig cfg;
    cfg.align = env_int("LAMFAST_POS_ALIGN", 0);
    cfg.min_rows = env_int("LAMFAST_POS_MIN_ROWS", 8);
    cfg.smem = (size_t)env_int("LAMFAST_POS_SMEM_KB", 40) * 1024;
    if (cfg.align <= 0) {
        // widest phase granularity that leaves the classes enough rows to
        // amortise a thread's entry decode and P (>= 24 rows per class on average)
        const int nt = d.t1 - d.t0;
        cfg.align = 1;
        if (d.pre_t_h && d.len_t_h)
            for (int A = 32; A > 1; A /= 2) {
                std::map<std::pair<int, long long>, int> cnt;
                const long long addr0 = (long long)(reinterpret_cast<uintptr_t>(out) / sizeof(double));
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
                if (big == 0 || big_rows >= 24 * big || nt < 24) {
                    cfg.align = A;
                    break;
                }
            }
    }
    switch (d.n_terms) {
#ifndef LF_POS_EPT
#define LF_POS_EPT 2 // positions per thread up to 4 terms
#endif
    case 1: return combine_pos_launch<1, LF_POS_EPT>(d, out, 0, cfg, stream);
    case 2: return combine_pos_launch<2, LF_POS_EPT>(d, out, 0, cfg, stream);
    case 3: return combine_pos_launch<3, LF_POS_EPT>(d, out, 0, cfg, stream);
    case 4: return combine_pos_launch<4, LF_POS_EPT>(d, out, 0, cfg, stream);
    case 5: return combine_pos_launch<5, 1>(d, out, 0, cfg, stream);
    case 6: return combine_pos_launch<6, 1>(d, out, 0, cfg, stream);
    default: return combine_pos_launch<7, 1>(d, out, 0, cfg, stream);
    }
}

} // namespace lfb
