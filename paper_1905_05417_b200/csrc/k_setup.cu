// Small setup kernels of the fast path, compiled with --fmad=false so that
// their arithmetic is formed exactly as the reference forms it (separately
// rounded products and sums): B-spline evaluation at Gauss points (K1,
// splines.cpp:53-101) and the per-ply thickness integrals reduced per
// operator term (K3, fast.cpp:170-209 + 285-302).  Both are O(thickness
// pairs x cells) -- microseconds -- so exactness costs nothing here.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace lfb {

namespace {

constexpr int kMaxP = 6;

/// KnotVector::findSpan (splines.cpp:37-51).
__device__ int find_span(const double* t, int p, int n, double x) {
    if (x >= 1.0) {
        int k = n - 1;
        while (k > p && t[k] >= 1.0)
            --k;
        return k;
    }
    int lo = p, hi = n + 1; // upper_bound over t[p .. n]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (t[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo - 1;
}

/// KnotVector::evaluate (splines.cpp:53-101): values and first derivatives
/// of the p+1 active functions; returns first_active.
__device__ int eval_basis(const double* t, int p, int n, double x, double* vals, double* ders) {
    const int span = find_span(t, p, n, x);
    double low[kMaxP + 1], left[kMaxP + 1], right[kMaxP + 1];
    for (int r = 0; r <= p; ++r)
        vals[r] = low[r] = left[r] = right[r] = 0.0;
    vals[0] = 1.0;
    for (int level = 1; level <= p; ++level) {
        if (level == p)
            for (int r = 0; r <= p; ++r)
                low[r] = vals[r];
        left[level] = x - t[span + 1 - level];
        right[level] = t[span + level] - x;
        double saved = 0.0;
        for (int r = 0; r < level; ++r) {
            const double denom = right[r + 1] + left[level - r];
            const double tmp = denom > 0.0 ? vals[r] / denom : 0.0;
            vals[r] = saved + right[r + 1] * tmp;
            saved = left[level - r] * tmp;
        }
        vals[level] = saved;
    }
    const int first = span - p;
    for (int r = 0; r <= p; ++r) {
        const int i = first + r;
        double d = 0.0;
        if (r >= 1) {
            const double den = t[i + p] - t[i];
            if (den > 0.0)
                d += low[r - 1] / den;
        }
        if (r <= p - 1) {
            const double den = t[i + p + 1] - t[i + 1];
            if (den > 0.0)
                d -= low[r] / den;
        }
        ders[r] = p * d;
    }
    return first;
}

__global__ void k_basis(DevTables d, int with_ct) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nu_pts = (long long)d.nspu * d.nqu;
    const long long nv_pts = (long long)d.nspv * d.nqv;
    const long long nt_pts = (long long)d.ncells * d.nqt;
    double v[kMaxP + 1], dd[kMaxP + 1];
    if (g < nu_pts) {
        // in-plane u points: u = mid + half * ref (assembly.cpp:30-40)
        const int s = (int)(g / d.nqu), q = (int)(g % d.nqu);
        const double mid = 0.5 * (d.spu_lo[s] + d.spu_hi[s]), half = 0.5 * (d.spu_hi[s] - d.spu_lo[s]);
        eval_basis(d.ku, d.pu, d.nku - d.pu - 1, mid + half * d.ru[q], v, dd);
        for (int r = 0; r <= d.pu; ++r) {
            d.Bu_val[g * (d.pu + 1) + r] = v[r];
            d.Bu_der[g * (d.pu + 1) + r] = dd[r];
        }
        return;
    }
    long long h = g - nu_pts;
    if (h < nv_pts) {
        const int s = (int)(h / d.nqv), q = (int)(h % d.nqv);
        const double mid = 0.5 * (d.spv_lo[s] + d.spv_hi[s]), half = 0.5 * (d.spv_hi[s] - d.spv_lo[s]);
        eval_basis(d.kv, d.pv, d.nkv - d.pv - 1, mid + half * d.rv[q], v, dd);
        for (int r = 0; r <= d.pv; ++r) {
            d.Bv_val[h * (d.pv + 1) + r] = v[r];
            d.Bv_der[h * (d.pv + 1) + r] = dd[r];
        }
        return;
    }
    h -= nv_pts;
    if (h < nt_pts) {
        // thickness cell points (fast.cpp:188-190)
        const int first = eval_basis(d.kt, d.pt, d.nkt - d.pt - 1, d.cell_pts[h], v, dd);
        d.Bt_first[h] = first;
        for (int r = 0; r <= d.pt; ++r) {
            d.Bt_val[h * (d.pt + 1) + r] = v[r];
            d.Bt_der[h * (d.pt + 1) + r] = dd[r];
        }
        return;
    }
    h -= nt_pts;
    if (with_ct && h < (long long)d.n_terms * 81) {
        // Constant-frame pulled-back contraction table (affine geometry):
        // Ct[t][3x+y][3i+k] = det * sum_{j,l} G(j,x) G(l,y) C_t{e_j,e_l}(i,k)
        // (voigt_free.cpp:125-140 with the Jacobian folded in).
        const int t = (int)(h / 81), xy = (int)(h % 81) / 9, ik = (int)(h % 9);
        const int x = xy / 3, y = xy % 3;
        const double* tab = d.term_table + (long long)t * 81;
        double s = 0.0;
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l)
                s += d.G[3 * x + j] * d.G[3 * y + l] * tab[(3 * j + l) * 9 + ik];
        d.Ct[(long long)t * 81 + xy * 9 + ik] = d.det * s;
    }
}

/// Thickness integrals per pair, reduced per term (fast.cpp:170-209 and the
/// q~ pre-reduction fast.cpp:285-302 / 303-336), from the tabulated basis
/// (general geometry path).  One warp per thickness pair of the slab; each
/// lane takes cells round-robin and adds each cell's Q with its layer's term
/// multiplier (term.thickness += w * Q_l, distributed over the layer's cells),
/// then a fixed xor tree combines the lanes (deterministic).
__global__ void k_thickness_pairs(DevTables d) {
    // one warp per pair (lanes over the pair's cells), as thickness_pair_warp
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= d.n_pairs)
        return;
    const long long pp = gw;
    // locate (it, k): pre_t[it] - pre_t[w_t0] <= pp < pre_t[it+1] - pre_t[w_t0]
    const long long target = pp + d.pre_t[d.w_t0];
    int lo = d.w_t0, hi = d.w_t1; // it in [w_t0, w_t1)
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (d.pre_t[mid] <= target)
            lo = mid;
        else
            hi = mid;
    }
    const int it = lo;
    const int jt = d.lo_t[it] + (int)(target - d.pre_t[it]);
    const int mn = min(it, jt), mx = max(it, jt);
    constexpr int kChunk = 8;
    for (int t0 = 0; t0 < d.n_terms; t0 += kChunk) {
        const int tn = min(kChunk, d.n_terms - t0);
        double acc[kChunk][4];
        unsigned on = 0;
        for (int t = 0; t < kChunk; ++t)
            acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0;
        for (int s = 0; s < d.nspt; ++s) {
            const int f0 = d.spt_first[s];
            if (f0 > mn || mx > f0 + d.pt)
                continue;
            for (int c = d.span_cell0[s] + lane; c < d.span_cell0[s + 1]; c += 32) {
                double ql[4] = {0.0, 0.0, 0.0, 0.0};
                for (int q = 0; q < d.nqt; ++q) {
                    const long long h = (long long)c * d.nqt + q;
                    const int first = d.Bt_first[h];
                    const int a = it - first, b = jt - first;
                    if (a < 0 || a > d.pt || b < 0 || b > d.pt)
                        continue;
                    const double wq = d.cell_wts[h];
                    const double va = d.Bt_val[h * (d.pt + 1) + a], da = d.Bt_der[h * (d.pt + 1) + a];
                    const double vb = d.Bt_val[h * (d.pt + 1) + b], db = d.Bt_der[h * (d.pt + 1) + b];
                    ql[0] += wq * va * vb;
                    ql[1] += wq * va * db;
                    ql[2] += wq * da * vb;
                    ql[3] += wq * da * db;
                }
                const int layer = d.cell_layer[c];
                for (int t = 0; t < tn; ++t) {
                    const long long tl = (long long)(t0 + t) * d.n_layers + layer;
                    if (!d.lam_on[tl])
                        continue;
                    const double w = d.lam[tl];
                    for (int f = 0; f < 4; ++f)
                        acc[t][f] += w * ql[f];
                    on |= 1u << t;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int t = 0; t < kChunk; ++t)
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    acc[t][f] += __shfl_xor_sync(0xffffffffu, acc[t][f], o);
            on |= __shfl_xor_sync(0xffffffffu, on, o);
        }
        if (lane == 0) {
            for (int t = 0; t < tn; ++t)
                for (int f = 0; f < 4; ++f)
                    d.W[(pp * d.n_terms + t0 + t) * 4 + f] = acc[t][f];
            d.Wmask[(long long)(t0 / kChunk) * d.n_pairs + pp] = on;
        }
    }
}

/// Cox-de Boor on a known span (splines.cpp:53-101 after findSpan): the
/// evaluation points of the fused setup are Gauss points strictly inside the
/// span, so findSpan would return `span`.  Compile-time degree keeps every
/// array in registers.  Returns values/derivatives of functions i and j
/// (global indices); false when either is inactive on the span.
template <int P>
__device__ __forceinline__ bool eval_pair(const double* t, int span, double x, int i, int j, double& vi, double& di,
                                          double& vj, double& dj) {
    double vals[P + 1], low[P + 1], left[P + 1], right[P + 1];
#pragma unroll
    for (int r = 0; r <= P; ++r)
        vals[r] = low[r] = left[r] = right[r] = 0.0;
    vals[0] = 1.0;
#pragma unroll
    for (int level = 1; level <= P; ++level) {
        if (level == P)
#pragma unroll
            for (int r = 0; r <= P; ++r)
                low[r] = vals[r];
        left[level] = x - t[span + 1 - level];
        right[level] = t[span + level] - x;
        double saved = 0.0;
#pragma unroll
        for (int r = 0; r < level; ++r) {
            const double denom = right[r + 1] + left[level - r];
            const double tmp = denom > 0.0 ? vals[r] / denom : 0.0;
            vals[r] = saved + right[r + 1] * tmp;
            saved = left[level - r] * tmp;
        }
        vals[level] = saved;
    }
    const int first = span - P;
    const int a = i - first, b = j - first;
    if (a < 0 || a > P || b < 0 || b > P)
        return false;
    vi = vj = di = dj = 0.0;
#pragma unroll
    for (int r = 0; r <= P; ++r) {
        const int g = first + r;
        double d = 0.0;
        if (r >= 1) {
            const double den = t[g + P] - t[g];
            if (den > 0.0)
                d += low[r - 1] / den;
        }
        if (r <= P - 1) {
            const double den = t[g + P + 1] - t[g + 1];
            if (den > 0.0)
                d -= low[r] / den;
        }
        d = P * d;
        if (r == a) {
            vi = vals[r];
            di = d;
        }
        if (r == b) {
            vj = vals[r];
            dj = d;
        }
    }
    return true;
}

/// 1D in-plane integrals U/V of one (i, slot) (see k_integrals_1d).
template <int P>
__device__ void integral_1d(const double* kn, const int* first, const double* slo, const double* shi,
                            const double* rref, const double* wref, int nsp, int nq, int i, int j, double* acc) {
    const int mn = min(i, j), mx = max(i, j);
    int s0 = 0, s1 = nsp; // first[] strictly increasing: spans with first in [mx - P, mn]
    while (s0 < s1) {
        const int m = (s0 + s1) >> 1;
        if (first[m] < mx - P)
            s0 = m + 1;
        else
            s1 = m;
    }
    for (int s = s0; s < nsp && first[s] <= mn; ++s) {
        const double mid = 0.5 * (slo[s] + shi[s]), half = 0.5 * (shi[s] - slo[s]);
        for (int q = 0; q < nq; ++q) {
            double vi, di, vj, dj;
            if (!eval_pair<P>(kn, first[s] + P, mid + half * rref[q], i, j, vi, di, vj, dj))
                continue;
            const double w = wref[q] * half;
            acc[0] += w * vi * vj;
            acc[1] += w * vi * dj;
            acc[2] += w * di * vj;
            acc[3] += w * di * dj;
        }
    }
}

/// Thickness integrals of one pair reduced per term (see k_thickness_pairs),
/// one warp per pair: the lanes take the pair's cells round-robin, each cell's
/// Q is added with its layer's term multiplier (q~ = sum_l w_l Q_l, with the
/// layer sums distributed over cells), and the lanes' partial sums are combined
/// by a fixed xor tree -- deterministic, and independent of the ply count in
/// latency (a 64-ply single thickness element no longer walks 256 points in
/// one thread).
template <int P>
__device__ void thickness_pair_warp(const DevTables& d, long long pp, int lane) {
    const long long target = pp + d.pre_t[d.w_t0];
    int lo = d.w_t0, hi = d.w_t1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (d.pre_t[mid] <= target)
            lo = mid;
        else
            hi = mid;
    }
    const int it = lo;
    const int jt = d.lo_t[it] + (int)(target - d.pre_t[it]);
    const int mn = min(it, jt), mx = max(it, jt);
    int s0 = 0, s1 = d.nspt;
    while (s0 < s1) {
        const int m = (s0 + s1) >> 1;
        if (d.spt_first[m] < mx - P)
            s0 = m + 1;
        else
            s1 = m;
    }
    int s_end = s0;
    while (s_end < d.nspt && d.spt_first[s_end] <= mn)
        ++s_end;
    const int c_begin = d.span_cell0[s0], c_end = d.span_cell0[s_end];
    constexpr int kChunk = 8;
    for (int t0 = 0; t0 < d.n_terms; t0 += kChunk) {
        const int tn = min(kChunk, d.n_terms - t0);
        double acc[kChunk][4];
        unsigned on = 0;
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0;
        int s = s0;
        for (int c = c_begin + lane; c < c_end; c += 32) {
            while (d.span_cell0[s + 1] <= c)
                ++s;
            const int span = d.spt_first[s] + P;
            double ql[4] = {0.0, 0.0, 0.0, 0.0};
            for (int q = 0; q < d.nqt; ++q) {
                const long long hq = (long long)c * d.nqt + q;
                double va, da, vb, db;
                if (!eval_pair<P>(d.kt, span, d.cell_pts[hq], it, jt, va, da, vb, db))
                    continue;
                const double wq = d.cell_wts[hq];
                ql[0] += wq * va * vb;
                ql[1] += wq * va * db;
                ql[2] += wq * da * vb;
                ql[3] += wq * da * db;
            }
            const int layer = d.cell_layer[c];
#pragma unroll
            for (int t = 0; t < kChunk; ++t) {
                if (t >= tn)
                    break;
                const long long tl = (long long)(t0 + t) * d.n_layers + layer;
                if (!d.lam_on[tl])
                    continue;
                const double w = d.lam[tl];
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    acc[t][f] += w * ql[f];
                on |= 1u << t;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int t = 0; t < kChunk; ++t)
#pragma unroll
                for (int f = 0; f < 4; ++f)
                    acc[t][f] += __shfl_xor_sync(0xffffffffu, acc[t][f], o);
            on |= __shfl_xor_sync(0xffffffffu, on, o);
        }
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < kChunk; ++t)
                if (t < tn)
                    for (int f = 0; f < 4; ++f)
                        d.W[(pp * d.n_terms + t0 + t) * 4 + f] = acc[t][f];
            d.Wmask[(long long)(t0 / kChunk) * d.n_pairs + pp] = on;
        }
    }
}

#define LF_DISPATCH_P(p, CALL)                                  \
    switch (p) {                                                \
    case 1: { constexpr int PP = 1; CALL; } break;              \
    case 2: { constexpr int PP = 2; CALL; } break;              \
    case 3: { constexpr int PP = 3; CALL; } break;              \
    case 4: { constexpr int PP = 4; CALL; } break;              \
    case 5: { constexpr int PP = 5; CALL; } break;              \
    default: { constexpr int PP = 6; CALL; } break;             \
    }

/// Fused setup of the affine fast path: one launch computes
///   [0, nU)            U[i][slot][4]   1D in-plane integrals, u direction (thread per item)
///   [nU, nU+nV)        V[i][slot][4]   v direction
///   [uv, +32 n_pairs)  W / Wmask       thickness integrals reduced per term (warp per pair;
///                                      uv = nU + nV rounded up to a warp)
///   [.., +T*81)        Ct              constant-frame pulled-back tables
/// with the same arithmetic as k_integrals_1d / k_thickness_pairs / k_basis.
__global__ void __launch_bounds__(64) k_prepare_affine(DevTables d) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nU = (long long)d.nu * d.bu, nV = (long long)d.nv * d.bv;
    if (g < nU + nV) {
        const bool is_u = g < nU;
        const int h = (int)(is_u ? g : g - nU);
        const int b = is_u ? d.bu : d.bv;
        const int i = h / b, slot = h % b;
        const int* lo = is_u ? d.lo_u : d.lo_v;
        const int* len = is_u ? d.len_u : d.len_v;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (slot < len[i]) {
            const int j = lo[i] + slot;
            if (is_u) {
                LF_DISPATCH_P(d.pu, (integral_1d<PP>(d.ku, d.spu_first, d.spu_lo, d.spu_hi, d.ru, d.wu, d.nspu,
                                                     d.nqu, i, j, acc)))
            } else {
                LF_DISPATCH_P(d.pv, (integral_1d<PP>(d.kv, d.spv_first, d.spv_lo, d.spv_hi, d.rv, d.wv, d.nspv,
                                                     d.nqv, i, j, acc)))
            }
        }
        double* out = (is_u ? d.U : d.V) + (long long)h * 4;
        out[0] = acc[0];
        out[1] = acc[1];
        out[2] = acc[2];
        out[3] = acc[3];
        return;
    }
    // thickness pairs: one warp per pair, region start aligned to a warp
    const long long uv = (nU + nV + 31) / 32 * 32;
    if (g < uv)
        return;
    long long h = g - uv;
    if (h < d.n_pairs * 32) {
        LF_DISPATCH_P(d.pt, (thickness_pair_warp<PP>(d, h >> 5, (int)(h & 31))))
        return;
    }
    h -= d.n_pairs * 32;
    if (h < (long long)d.n_terms * 81) {
        const int t = (int)(h / 81), xy = (int)(h % 81) / 9, ik = (int)(h % 9);
        const int x = xy / 3, y = xy % 3;
        const double* tab = d.term_table + (long long)t * 81;
        double s = 0.0;
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l)
                s += d.G[3 * x + j] * d.G[3 * y + l] * tab[(3 * j + l) * 9 + ik];
        d.Ct[(long long)t * 81 + xy * 9 + ik] = d.det * s;
    }
}

} // namespace

int launch_prepare_affine(const DevTables& d, cudaStream_t stream) {
    const long long uv = ((long long)d.nu * d.bu + (long long)d.nv * d.bv + 31) / 32 * 32;
    const long long n = uv + d.n_pairs * 32 + (long long)d.n_terms * 81;
    const int block = 64; // few items: spread them over more SMs
    k_prepare_affine<<<(unsigned)((n + block - 1) / block), block, 0, stream>>>(d);
    return (int)cudaGetLastError();
}

int launch_basis(const DevTables& d, bool with_ct, cudaStream_t stream) {
    const long long n = (long long)d.nspu * d.nqu + (long long)d.nspv * d.nqv +
                        (long long)d.ncells * d.nqt + (with_ct ? (long long)d.n_terms * 81 : 0);
    if (n == 0)
        return 0;
    const int block = 128;
    k_basis<<<(unsigned)((n + block - 1) / block), block, 0, stream>>>(d, with_ct ? 1 : 0);
    return (int)cudaGetLastError();
}

int launch_thickness_pairs(const DevTables& d, cudaStream_t stream) {
    if (d.n_pairs == 0)
        return 0;
    const int block = 128; // 4 pairs (warps) per block
    k_thickness_pairs<<<(unsigned)((d.n_pairs * 32 + block - 1) / block), block, 0, stream>>>(d);
    return (int)cudaGetLastError();
}

} // namespace lfb
