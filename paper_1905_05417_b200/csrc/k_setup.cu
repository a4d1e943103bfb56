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
/// q~ pre-reduction fast.cpp:285-302 / 303-336).  One thread per thickness
/// pair of the slab.  Cells are visited in the reference order (span-major;
/// each layer's cells are consecutive), Q_l is completed per layer and then
/// added with the term multiplier, as `term.thickness += w * Q_l` does.
__global__ void k_thickness_pairs(DevTables d) {
    const long long pp = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pp >= d.n_pairs)
        return;
    // locate (it, k): pre_t[it] - pre_t[t0] <= pp < pre_t[it+1] - pre_t[t0]
    const long long target = pp + d.pre_t[d.t0];
    int lo = d.t0, hi = d.t1; // it in [t0, t1)
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
        double ql[4] = {0.0, 0.0, 0.0, 0.0};
        int cur = -1;
        auto flush = [&](int layer) {
            if (layer < 0)
                return;
            for (int t = 0; t < tn; ++t) {
                const long long tl = (long long)(t0 + t) * d.n_layers + layer;
                if (!d.lam_on[tl])
                    continue;
                const double w = d.lam[tl];
                for (int f = 0; f < 4; ++f)
                    acc[t][f] += w * ql[f];
                on |= 1u << t;
            }
        };
        for (int s = 0; s < d.nspt; ++s) {
            const int f0 = d.spt_first[s];
            if (f0 > mn || mx > f0 + d.pt)
                continue;
            for (int c = d.span_cell0[s]; c < d.span_cell0[s + 1]; ++c) {
                const int layer = d.cell_layer[c];
                if (layer != cur) {
                    flush(cur);
                    cur = layer;
                    ql[0] = ql[1] = ql[2] = ql[3] = 0.0;
                }
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
            }
        }
        flush(cur);
        for (int t = 0; t < tn; ++t)
            for (int f = 0; f < 4; ++f)
                d.W[(pp * d.n_terms + t0 + t) * 4 + f] = acc[t][f];
        // pass masks: pass = term / 8, bit = term % 8 (chunk == pass width)
        d.Wmask[(long long)(t0 / kChunk) * d.n_pairs + pp] = on;
    }
}

} // namespace

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
    const int block = 128;
    k_thickness_pairs<<<(unsigned)((d.n_pairs + block - 1) / block), block, 0, stream>>>(d);
    return (int)cudaGetLastError();
}

} // namespace lfb
