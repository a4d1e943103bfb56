// EXPERIMENTS, not built into the product library (moved out of
// paper_1905_05417_b200/csrc/k_ops.cu in round 2).  Two alternative forms of
// K2b phase 1 (general-geometry in-plane operators), both parity-green in
// round 1 and both measured slower than the default two-phase scalar kernel
// (k_inplane_elem + k_inplane_gather):
//   * k_inplane_general: coloured, in-place accumulation into Pg
//     (C3: 16 launches x 97 us, 141 MB read + 57 MB written per launch,
//     profiles/r1_ncu_inplane_general_c3.txt);
//   * k_inplane_elem_mma: the element contraction on the FP64 tensor cores
//     (mma.sync.m8n8k4.f64): FP64 pipe 4%, same 1.1 ms as the scalar kernel on
//     C3, slower at p = 2 (profiles/r1_k2b.txt).
// They depend on the helpers of k_ops.cu (ElemInfo, element_tables,
// pullback_tables, pe_local) and are kept as the record of those A/B runs.
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

/// Shared-memory layout of the DMMA element kernel (doubles).
struct ElemMmaLayout {
    int nl2, nq2, m, mpad, npad, kmax, ldh, ldb;
    long long gh, w2, ctq, h, b, total;
    __host__ __device__ ElemMmaLayout(int pu, int pv, int nqu, int nqv) {
        nl2 = (pu + 1) * (pv + 1);
        nq2 = nqu * nqv;
        m = 9 * nl2;
        mpad = (m + 7) & ~7;
        npad = (nl2 + 7) & ~7;
        kmax = (2 * nq2 + 3) & ~3;
        ldh = kmax + ((4 - kmax % 16) + 16) % 16;  // ldh = 4 (mod 16): conflict-free A fragments
        ldb = npad + ((8 - npad % 16) + 16) % 16;  // ldb = 8 (mod 16): conflict-free B fragments
        gh = 0;
        w2 = gh + (long long)nq2 * nl2 * 3;
        ctq = (w2 + nq2 + 1) & ~1LL;
        h = ctq + (long long)nq2 * 90;
        b = h + (long long)mpad * ldh;
        total = b + (long long)kmax * ldb;
    }
};

__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

/// K2b phase 1 on the FP64 tensor cores: for each family f the element's
/// P_f is a dense contraction over (Gauss point, derivative direction y):
///   P_f[(al, ab), be] = sum_{q, y in Y_f} H_f[(al, ab), (q, y)] * g_y(be, q),
///   H_f[(al, ab), (q, y)] = sum_{x in X_f} Ct_q[xy][ab] g_x(al, q)
/// (P11 <- xy in {0,1}^2, P12 <- x in {0,1}, y = 2, P21 <- x = 2, y in {0,1},
/// P22 <- x = y = 2).  H_f and g are staged in shared memory, padded to
/// 8 x 8 x 4 tiles, and multiplied with mma.sync.m8n8k4.f64 (DMMA): one warp
/// instruction per 256 multiply-adds instead of 8 DFMA, with the operands
/// loaded once per k-step.  Opt-in (LAMFAST_K2B=mma), while the layout fits
/// shared memory (p <= 4): per element the contraction is small (p = 3: 864
/// DMMA per family set), so the staging and the scattered Pe stores set the
/// time -- ncu shows the FP64 pipe at 4% and the same 1.1 ms as the scalar
/// element kernel on C3, and the 8x8 padding of nl2 = 9 makes it slower at
/// p = 2 (profiles/r1_k2b.txt).
__global__ void __launch_bounds__(256) k_inplane_elem_mma(const DevTables d, int t0) {
    extern __shared__ double sm[];
    const int e_index = blockIdx.x;
    const int t = t0 + blockIdx.y;
    if (t >= d.n_terms)
        return;
    const ElemMmaLayout L(d.pu, d.pv, d.nqu, d.nqv);
    ElemInfo el;
    el.eu = e_index % d.nspu;
    el.ev = e_index / d.nspu;
    el.fu = d.spu_first[el.eu];
    el.fv = d.spv_first[el.ev];
    el.nl2 = L.nl2;
    el.nq2 = L.nq2;
    el.hu = 0.5 * (d.spu_hi[el.eu] - d.spu_lo[el.eu]);
    el.hv = 0.5 * (d.spv_hi[el.ev] - d.spv_lo[el.ev]);
    double* gh = sm + L.gh;
    double* w2 = sm + L.w2;
    double* ctq = sm + L.ctq;
    double* H = sm + L.h;
    double* Bm = sm + L.b;
    element_tables(d, el, gh, w2);
    __syncthreads();
    pullback_tables(d, e_index, el.nq2, w2, d.term_table + (long long)t * 81, ctq);
    const int nel = d.nspu * d.nspv;
    const long long per_el = 36LL * L.nl2 * L.nl2;
    double* pe = d.Pe + ((long long)blockIdx.y * nel + e_index) * per_el;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int nl2 = L.nl2, nq2 = L.nq2;
    for (int f = 0; f < 4; ++f) {
        const int ny = (f == 0 || f == 2) ? 2 : 1;  // y in {0,1} or {2}
        const int y0 = (f == 0 || f == 2) ? 0 : 2;
        const int nx = (f <= 1) ? 2 : 1;            // x in {0,1} or {2}
        const int x0 = (f <= 1) ? 0 : 2;
        const int K = nq2 * ny, kpad = (K + 3) & ~3;
        __syncthreads(); // ctq ready / previous family's tiles consumed
        // H_f: one item per (al, k) produces the 9 values (al, ab = 0..8, k); lanes
        // take consecutive k, so the shared stores of a warp are contiguous
        for (int idx = threadIdx.x; idx < kpad * L.mpad / 9 + kpad; idx += blockDim.x) {
            const int al = idx / kpad, k = idx - al * kpad;
            if (9 * al >= L.mpad)
                continue;
            double v[9];
#pragma unroll
            for (int ab = 0; ab < 9; ++ab)
                v[ab] = 0.0;
            if (al < nl2 && k < K) {
                const int q = ny == 2 ? k >> 1 : k, y = y0 + (ny == 2 ? (k & 1) : 0);
                const double* g = gh + (q * nl2 + al) * 3;
                const double* c = ctq + q * 90 + (3 * x0 + y) * 10;
                const double g0 = g[x0];
#pragma unroll
                for (int ab = 0; ab < 9; ++ab)
                    v[ab] = c[ab] * g0;
                if (nx == 2) {
                    const double g1 = g[x0 + 1];
#pragma unroll
                    for (int ab = 0; ab < 9; ++ab)
                        v[ab] += c[30 + ab] * g1;
                }
            }
#pragma unroll
            for (int ab = 0; ab < 9; ++ab)
                if (9 * al + ab < L.mpad)
                    H[(9 * al + ab) * L.ldh + k] = v[ab];
        }
        for (int k = warp; k < kpad; k += nwarp) {
            const int q = ny == 2 ? k >> 1 : k, y = y0 + (ny == 2 ? (k & 1) : 0);
            for (int n = lane; n < L.npad; n += 32)
                Bm[k * L.ldb + n] = (k < K && n < nl2) ? gh[(q * nl2 + n) * 3 + y] : 0.0;
        }
        __syncthreads();
        const int mtiles = L.mpad >> 3, ntiles = L.npad >> 3;
        for (int mt = warp; mt < mtiles; mt += nwarp) {
            double acc[4][2];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
                acc[nt][0] = acc[nt][1] = 0.0;
            const double* ha = H + (mt * 8 + (lane >> 2)) * L.ldh + (lane & 3);
            const double* bb = Bm + (lane & 3) * L.ldb + (lane >> 2);
            for (int k0 = 0; k0 < kpad; k0 += 4) {
                const double a = ha[k0];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                    if (nt < ntiles)
                        dmma_m8n8k4(acc[nt], a, bb[k0 * L.ldb + nt * 8]);
            }
            const int m = mt * 8 + (lane >> 2);
            if (m < L.m) {
                const int al = m / 9, ab = m - 9 * al, a = ab / 3, b = ab - 3 * a;
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
                    if (nt < ntiles)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int be = nt * 8 + 2 * (lane & 3) + h;
                            if (be < nl2) {
                                LF_CHECK(pe_local(f, al, a, be, b, nl2) < per_el);
                                pe[pe_local(f, al, a, be, b, nl2)] = acc[nt][h];
                            }
                        }
            }
        }
    }
}
