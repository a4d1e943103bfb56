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

template <int NT, int NTILE, bool AFFINE, int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB)
    k_combine_mma(const __grid_constant__ DevTables d, const __grid_constant__ PosParams pp,
                  double* __restrict__ out) {
    static_assert(NTILE == 4 || NTILE == 8, "32 or 64 positions per warp");
    constexpr int WP = 8 * NTILE;   // positions per warp
    constexpr int ND = NTILE / 4;   // positions decoded per lane
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
    const long long tau_w = xb * ((BT / 32) * WP) + (threadIdx.x >> 5) * WP; // first position of the warp

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
            ri.mask = 0;
            ri.edge = 4;
            if (rr < nrow) {
                const int it = pp.rows[row0 + rr];
                const long long pre = __ldg(d.pre_t + it);
                unsigned m = 0;
                for (int k = 0; k < L; ++k)
                    m |= __ldg(d.Wmask + (pre - preW) + k);
                ri.base = nine_S * (pre - pre0) - d.out_base - phi;
                ri.mask = m;
                ri.edge = row_edge(d, it);
            }
            s_row[rr] = ri;
        }
        // a row's weights [k][term][family] are contiguous in W (single pass: n_terms = NT)
        const int per_row = L * NT * 2; // 16-byte pieces
        for (int rr = threadIdx.x >> 5; rr < nrow8; rr += BT / 32) {
            const double2* src = nullptr;
            if (rr < nrow)
                src = reinterpret_cast<const double2*>(d.W) +
                      (__ldg(d.pre_t + pp.rows[row0 + rr]) - preW) * (NT * 2);
            double2* dst = reinterpret_cast<double2*>(s_w + (size_t)rr * rs);
            for (int c = lane; c < per_row; c += 32)
                dst[c] = src ? __ldg(src + c) : make_double2(0.0, 0.0);
        }
    }

    // decode the warp's positions, one (or two) per lane
    PosDec dec[ND];
#pragma unroll
    for (int x = 0; x < ND; ++x)
        dec[x] = decode_position(d, tau_w + 32 * x + lane - phi, L, EL);
    unsigned kmask = 0, all_live = 1;
#pragma unroll
    for (int x = 0; x < ND; ++x) {
        const bool lv = (dec[x].info >> 14) & 1;
        kmask |= __reduce_or_sync(0xffffffffu, lv ? 1u << (dec[x].info & 0xff) : 0u);
        all_live &= __all_sync(0xffffffffu, lv) ? 1u : 0u;
    }
    __syncthreads(); // s_ct (and the staged rows) visible
    if (kmask == 0)
        return; // no live position in this warp

    // B operands: lane (g, j) holds family j of the position in column g of every tile
    double P[NTILE][NT];
    int ksel[NTILE];
    unsigned tk[NTILE]; // neighbours present in the tile (bit k)
#pragma unroll
    for (int tl = 0; tl < NTILE; ++tl) {
        const int q = tile_position(tl, g);
        const int src = q & 31, x = q >> 5;
        int info = 0, uo = 0, vo = 0, ec = 0;
#pragma unroll
        for (int xx = 0; xx < ND; ++xx) {
            const int i0 = __shfl_sync(0xffffffffu, dec[xx].info, src);
            const int i1 = __shfl_sync(0xffffffffu, AFFINE ? dec[xx].uo : dec[xx].ec, src);
            const int i2 = __shfl_sync(0xffffffffu, dec[xx].vo, src);
            if (xx == x) {
                info = i0;
                uo = ec = i1;
                vo = i2;
            }
        }
        const bool lv = (info >> 14) & 1;
        ksel[tl] = lv ? (info & 0xff) : -1;
        tk[tl] = __reduce_or_sync(0xffffffffu, lv ? 1u << (info & 0xff) : 0u);
        if constexpr (AFFINE) {
            family_p<NT>(d, s_ct, uo, vo, (info >> 8) & 15, j, P[tl]);
        } else {
#pragma unroll
            for (int t = 0; t < NT; ++t)
                P[tl][t] = __ldg(d.Pg + ((long long)t * 4 + j) * d.E + ec);
        }
        if (!lv) {
#pragma unroll
            for (int t = 0; t < NT; ++t)
                P[tl][t] = 0.0;
        }
    }
    const bool one_k = (kmask & (kmask - 1)) == 0; // every position of the warp has the same neighbour

    double* const o_lane = out + tau_w + 4 * j; // + 16 h: the lane's four positions of tile pair h
    for (int rt = 0; rt < nrow8; rt += 8) {
        const PosRow ri = s_row[rt + g];
        const unsigned tmask = __reduce_or_sync(0xffffffffu, ri.mask);
        const unsigned edge = __reduce_or_sync(0xffffffffu, (unsigned)ri.edge & 3u);
        double D[NTILE][2];
#pragma unroll
        for (int tl = 0; tl < NTILE; ++tl)
            D[tl][0] = D[tl][1] = 0.0;
        const double* wrow = s_w + (size_t)(rt + g) * rs + j;
        if (one_k) {
            const double* wk = wrow + (31 - __clz(kmask)) * (NT * 4);
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (tmask & (1u << t)) {
                    const double a = wk[t * 4];
#pragma unroll
                    for (int tl = 0; tl < NTILE; ++tl)
                        dmma_884(D[tl][0], D[tl][1], a, P[tl][t]);
                }
        } else {
            for (unsigned km = kmask; km; km &= km - 1) {
                const int k = __ffs(km) - 1;
                const double* wk = wrow + k * (NT * 4);
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    if (tmask & (1u << t)) {
                        const double a = wk[t * 4];
#pragma unroll
                        for (int tl = 0; tl < NTILE; ++tl)
                            if (tk[tl] & (1u << k))
                                dmma_884(D[tl][0], D[tl][1], a, ksel[tl] == k ? P[tl][t] : 0.0);
                    }
            }
        }
        if (all_live && edge == 0) {
            const bool row_ok = ri.edge == 0; // padding rows of the last tile are not written
            double* const p = o_lane + ri.base;
#pragma unroll
            for (int h = 0; h < NTILE / 2; ++h) {
                LF_CHECK(!row_ok || (p + 16 * h >= out && p + 16 * h + 3 < out + d.nnz_slab));
                store_value4(p + 16 * h, D[2 * h][0], D[2 * h][1], D[2 * h + 1][0], D[2 * h + 1][1], row_ok);
            }
        } else {
            // warps at the ends of the class range, and tiles with a partial
            // first / last row of a function range: one predicated store per value
#pragma unroll
            for (int h = 0; h < NTILE / 2; ++h)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int q = 16 * h + 4 * j + c;
                    int info = 0;
#pragma unroll
                    for (int xx = 0; xx < ND; ++xx) {
                        const int i0 = __shfl_sync(0xffffffffu, dec[xx].info, q & 31);
                        if (xx == (q >> 5))
                            info = i0;
                    }
                    const unsigned flags = (info >> 12) & 3u;
                    const bool pred = ((info >> 14) & 1) && ri.edge < 4 && ((unsigned)ri.edge & ~flags) == 0;
                    double* const p = o_lane + ri.base + 16 * h + c;
                    LF_CHECK(!pred || (p >= out && p < out + d.nnz_slab));
                    store_value_if(p, D[2 * h + (c >> 1)][c & 1], pred);
                }
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
#define LF_POS_MINB 3
#endif
    constexpr int BT = LF_POS_BT, MINB = NT * NTILE <= 20 ? LF_POS_MINB : 2; // 80 registers up to 5 terms
    static thread_local PosParams pp;
    long long total_blocks = 0;
    size_t smem = 0;
    if (!build_pos_params(d, out, NT, (BT / 32) * 8 * NTILE, cfg, pp, total_blocks, smem))
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
        launch(k_combine_mma<NT, NTILE, true, BT, MINB>);
    else
        launch(k_combine_mma<NT, NTILE, false, BT, MINB>);
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
    cfg.smem = (size_t)env_int("LAMFAST_POS_SMEM_KB", 72) * 1024;
    if (cfg.align <= 0) {
        // widest phase granularity that leaves the classes enough rows to
        // amortise a warp's position decode and P (>= 24 rows per class on average)
        const int nt = d.t1 - d.t0;
        cfg.align = 4;
        if (d.pre_t_h && d.len_t_h)
            for (int A = 32; A > 4; A /= 2) {
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
    cfg.align = std::max(4, cfg.align / 4 * 4); // 256-bit stores need 32-byte aligned quads
#ifndef LF_POS_NTILE
#define LF_POS_NTILE 4 // 8-position tiles per warp (4: 32 positions, 8: 64)
#endif
    switch (d.n_terms) {
    case 1: return combine_pos_launch<1, LF_POS_NTILE>(d, out, cfg, stream);
    case 2: return combine_pos_launch<2, LF_POS_NTILE>(d, out, cfg, stream);
    case 3: return combine_pos_launch<3, LF_POS_NTILE>(d, out, cfg, stream);
    case 4: return combine_pos_launch<4, LF_POS_NTILE>(d, out, cfg, stream);
    case 5: return combine_pos_launch<5, LF_POS_NTILE>(d, out, cfg, stream);
    case 6: return combine_pos_launch<6, LF_POS_NTILE>(d, out, cfg, stream);
    default: return combine_pos_launch<7, LF_POS_NTILE>(d, out, cfg, stream);
    }
}

} // namespace lfb
