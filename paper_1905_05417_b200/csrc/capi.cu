// C ABI of the B200 assembler (include/lamfast_cuda.h).  Host orchestration
// only: validation and setup tables come from setup.cpp, all O(nnz) and
// O(elements) work runs in the kernels of k_setup.cu / k_ops.cu / k_combine.cu.  No CPU
// fallback exists: without a usable CUDA device every compute entry point
// fails with LF_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "kernels.cuh"
#include "lamfast_cuda.h"
#include "setup.hpp"

using lfb::raise;

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LF_OK;
    } catch (const lfb::Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_error = e.what();
        return LF_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_error = e.what();
        return LF_ERR_RUNTIME;
    }
}

void cuda_check(cudaError_t st, const char* what) {
    if (st != cudaSuccess) {
        const std::string msg = std::string(what) + ": " + cudaGetErrorString(st);
        if (st == cudaErrorMemoryAllocation)
            raise(LF_ERR_OUT_OF_MEMORY, msg);
        raise(LF_ERR_CUDA, msg);
    }
}
#define CK(x) cuda_check((x), #x)

void use_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        raise(LF_ERR_CUDA, "no CUDA device available (the B200 assembler has no CPU fallback)");
    }
    if (device < 0 || device >= n)
        raise(LF_ERR_INVALID_ARGUMENT, "device index out of range");
    CK(cudaSetDevice(device));
}

/// The library's own stream-ordered memory pool per device.  Its release
/// threshold is unlimited, so one-shot calls reuse the buffers the previous
/// call freed (no fresh mappings of a 23 GB CSR per call), but it is private:
/// torch's caching allocator and other users of the device's default pool
/// never see it, and lf_release_memory() returns it to the driver.
cudaMemPool_t lib_pool(int device) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lock(mu);
    if (static_cast<int>(pools.size()) <= device)
        pools.resize(static_cast<std::size_t>(device) + 1, nullptr);
    cudaMemPool_t& pool = pools[static_cast<std::size_t>(device)];
    if (!pool) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        CK(cudaMemPoolCreate(&pool, &props));
        uint64_t threshold = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    }
    return pool;
}

int current_device() {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    return dev;
}

void* pool_alloc(std::size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    CK(cudaMallocFromPoolAsync(&p, std::max<std::size_t>(bytes, 8), lib_pool(current_device()), s));
    return p;
}

/// Device allocations owned by a plan.  With a stream set (plans), they come
/// from the stream-ordered pool and go back to it without a device-wide
/// synchronisation: per-call cudaMalloc/cudaFree of the ~50 table buffers
/// measured as 40-370 ms outliers of plan creation / destruction on the box
/// (tools/e2e_phases.py).  Without a stream: plain cudaMalloc/cudaFree.
struct DeviceArena {
    std::vector<void*> ptrs;
    cudaStream_t s = nullptr;
    ~DeviceArena() { clear(); }
    void clear() {
        for (void* p : ptrs)
            s ? cudaFreeAsync(p, s) : cudaFree(p);
        ptrs.clear();
    }
    template <typename T>
    T* alloc(std::size_t n) {
        void* p = nullptr;
        const std::size_t bytes = std::max<std::size_t>(1, n) * sizeof(T);
        if (s)
            p = pool_alloc(bytes, s);
        else
            CK(cudaMalloc(&p, bytes));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <typename T>
    T* upload(const T* src, std::size_t n) {
        T* d = alloc<T>(n);
        if (n) {
            if (s) { // stream-ordered; the caller synchronises before the host data dies
                CK(cudaMemcpyAsync(d, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
            } else {
                CK(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice));
            }
        }
        return d;
    }
    template <typename T>
    T* upload(const std::vector<T>& v) {
        return upload(v.data(), v.size());
    }
};

/// Uploads the space part of a setup (knots, spans, rules, adjacency) and
/// allocates the basis / 1D-integral workspace.
void upload_space(const lfb::Setup& s, DeviceArena& ar, lfb::DevTables& d) {
    std::memset(&d, 0, sizeof d);
    d.pu = s.ku.p;
    d.pv = s.kv.p;
    d.pt = s.kt.p;
    d.nu = s.n_u;
    d.nv = s.n_v;
    d.nt = s.n_t;
    d.ns = s.n_s;
    d.nspu = static_cast<int>(s.spu.size());
    d.nspv = static_cast<int>(s.spv.size());
    d.nspt = static_cast<int>(s.spt.size());
    d.nqu = s.nqu;
    d.nqv = s.nqv;
    d.nqt = s.nqt;
    d.bu = 2 * d.pu + 1;
    d.bv = 2 * d.pv + 1;
    d.ku = ar.upload(s.ku.t);
    d.kv = ar.upload(s.kv.t);
    d.kt = ar.upload(s.kt.t);
    d.nku = static_cast<int>(s.ku.t.size());
    d.nkv = static_cast<int>(s.kv.t.size());
    d.nkt = static_cast<int>(s.kt.t.size());
    auto spans = [&](const std::vector<lfb::Span>& sp, const int** first, const double** lo, const double** hi) {
        std::vector<int> f;
        std::vector<double> l, h;
        for (const auto& x : sp) {
            f.push_back(x.first);
            l.push_back(x.begin);
            h.push_back(x.end);
        }
        *first = ar.upload(f);
        *lo = ar.upload(l);
        *hi = ar.upload(h);
    };
    spans(s.spu, &d.spu_first, &d.spu_lo, &d.spu_hi);
    spans(s.spv, &d.spv_first, &d.spv_lo, &d.spv_hi);
    d.ru = ar.upload(s.ru);
    d.wu = ar.upload(s.wu);
    d.rv = ar.upload(s.rv);
    d.wv = ar.upload(s.wv);
    d.lo_u = ar.upload(s.au.lo);
    d.len_u = ar.upload(s.au.len);
    d.pre_u = reinterpret_cast<const long long*>(ar.upload(s.au.pre));
    d.lo_v = ar.upload(s.av.lo);
    d.len_v = ar.upload(s.av.len);
    d.pre_v = reinterpret_cast<const long long*>(ar.upload(s.av.pre));
    d.es_pre = reinterpret_cast<const long long*>(ar.upload(s.es_pre));
    {
        // first in-plane function of every 256-entry block of the entry space
        const long long E = 9 * s.S_s;
        std::vector<int> blk(static_cast<std::size_t>((E + 255) / 256) + 1, 0);
        int is = 0;
        for (std::size_t b = 0; b + 1 < blk.size(); ++b) {
            const long long e0 = static_cast<long long>(b) * 256;
            while (is + 1 < s.n_s && s.es_pre[static_cast<std::size_t>(is) + 1] <= e0)
                ++is;
            blk[b] = is;
        }
        d.blk_is = ar.upload(blk);
    }
    d.S_s = s.S_s;
    d.S_u = s.au.total;
    d.E = 9 * s.S_s;
    d.Bu_val = ar.alloc<double>(static_cast<std::size_t>(d.nspu) * d.nqu * (d.pu + 1));
    d.Bu_der = ar.alloc<double>(static_cast<std::size_t>(d.nspu) * d.nqu * (d.pu + 1));
    d.Bv_val = ar.alloc<double>(static_cast<std::size_t>(d.nspv) * d.nqv * (d.pv + 1));
    d.Bv_der = ar.alloc<double>(static_cast<std::size_t>(d.nspv) * d.nqv * (d.pv + 1));
    d.U = ar.alloc<double>(static_cast<std::size_t>(d.nu) * d.bu * 4);
    d.V = ar.alloc<double>(static_cast<std::size_t>(d.nv) * d.bv * 4);
}

void upload_geometry(const lfb::Setup& s, DeviceArena& ar, lfb::DevTables& d) {
    d.affine = s.affine ? 1 : 0;
    if (s.affine) {
        std::memcpy(d.G, s.frame0.dfit, sizeof d.G);
        d.det = s.frame0.det;
    } else {
        d.frames = ar.upload(s.frames);
    }
}

void upload_thickness(const lfb::Setup& s, DeviceArena& ar, lfb::DevTables& d, const lfb::Adjacency& at) {
    d.ncells = static_cast<int>(s.cells.size());
    d.cell_pts = ar.upload(s.cell_pts);
    d.cell_wts = ar.upload(s.cell_wts);
    d.cell_first = ar.upload(s.cell_first);
    d.cell_layer = ar.upload(s.cell_layer);
    d.span_cell0 = ar.upload(s.span_cell0);
    d.spt_first = ar.upload(s.spt_first);
    d.lo_t = ar.upload(at.lo);
    d.len_t = ar.upload(at.len);
    d.pre_t = reinterpret_cast<const long long*>(ar.upload(at.pre));
    d.lt_max = at.max_len;
    const std::size_t ntp = static_cast<std::size_t>(d.ncells) * d.nqt;
    d.Bt_val = ar.alloc<double>(ntp * (d.pt + 1));
    d.Bt_der = ar.alloc<double>(ntp * (d.pt + 1));
    d.Bt_first = ar.alloc<int>(ntp);
}

void upload_terms(DeviceArena& ar, lfb::DevTables& d, int n_terms, int n_layers, const std::vector<double>& table,
                  const std::vector<double>& lam, const std::vector<uint8_t>& lam_on) {
    d.n_terms = n_terms;
    d.n_layers = n_layers;
    d.n_passes = (n_terms + lfb::kMaxTermsPerPass - 1) / lfb::kMaxTermsPerPass;
    d.term_table = ar.upload(table);
    d.lam = ar.upload(lam);
    d.lam_on = ar.upload(lam_on);
    d.Ct = ar.alloc<double>(static_cast<std::size_t>(std::max(1, n_terms)) * 81);
}


} // namespace

struct lf_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    lfb::Setup setup;
    DeviceArena arena;
    lfb::DevTables d{};
    lfb::K6Const k6c{}; // standard backend, affine map: K6 phase-1 tables (n_cfg = 0: not used)
    int launches = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> free_events, pending;
    double kernel_ms = 0.0;
    int64_t kernel_launches = 0;
    // CUDA-graph replay of the per-step launch sequence (small, launch-bound
    // plans): captured once per output pointer, replayed by one cudaGraphLaunch
    bool use_graph = false;
    cudaGraphExec_t graph = nullptr;
    double* graph_values = nullptr;
    int graph_launches = 0;

    ~lf_plan() {
        if (stream)
            cudaStreamSynchronize(stream);
        if (graph)
            cudaGraphExecDestroy(graph);
        for (auto& e : free_events) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        for (auto& e : pending) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
        arena.clear(); // stream-ordered frees, before the stream goes away
        if (own_stream && stream)
            cudaStreamDestroy(stream);
    }

    void harvest() {
        CK(cudaStreamSynchronize(stream));
        for (auto& e : pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e.first, e.second));
            kernel_ms += ms;
            ++kernel_launches;
            free_events.push_back(e);
        }
        pending.clear();
    }
};

namespace {

/// Element-local scratch of the two-phase general in-plane kernel (K2b):
/// as many terms per batch as fit in ~2 GB (one at least).
void alloc_element_scratch(DeviceArena& ar, lfb::DevTables& d, int n_terms) {
    const std::size_t nl2 = static_cast<std::size_t>(d.pu + 1) * (d.pv + 1);
    const std::size_t per_term = static_cast<std::size_t>(d.nspu) * d.nspv * 36 * nl2 * nl2;
    const std::size_t budget = (std::size_t(2) << 30) / sizeof(double);
    d.pe_terms = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(n_terms, budget / std::max<std::size_t>(1, per_term))));
    d.Pe = ar.alloc<double>(per_term * static_cast<std::size_t>(d.pe_terms));
}

/// Functions per thickness row (n_u n_v) of a problem, 0 if its in-plane knot
/// counts are not valid (the setup then reports the error).
int64_t functions_per_row(const lf_problem* p) {
    if (!p)
        return 0;
    const int64_t nu = p->n_knots_u - p->degree_u - 1, nv = p->n_knots_v - p->degree_v - 1;
    return nu > 0 && nv > 0 ? nu * nv : 0;
}

/// Function range of the thickness rows [t0, t1) (t1 < 0: all).
std::pair<int64_t, int64_t> thickness_range(const lf_problem* p, int t0, int t1) {
    const int64_t ns = functions_per_row(p);
    return {static_cast<int64_t>(t0) * ns, t1 < 0 ? -1 : static_cast<int64_t>(t1) * ns};
}

/// Smallest term count that takes the coefficient form of the combine
/// (affine geometry).  Below it the per-term form keeps the entry's P in
/// registers (4 FMA per active term and value); the coefficient form costs
/// 9 FMA per value whatever the term count, and from 9 terms on the
/// per-term form would need a second read-modify-write pass.  Measured
/// crossover (profiles/r2_coef_threshold.txt): per-term faster up to 6-7
/// distinct angles on C4 and C3, the coefficient form from 8.
/// LAMFAST_EFORM_MIN_TERMS overrides it (A/B runs).
int eform_min_terms() {
    if (const char* e = std::getenv("LAMFAST_EFORM_MIN_TERMS"))
        return std::max(1, std::atoi(e));
    return 8;
}

/// Smallest term count that takes the slot form of the per-term combine
/// (k_combine_slots; affine geometry, every thickness row seeing <= 3 terms).
/// From 5 terms on the per-term kernel drops to one entry per thread
/// (profiles/r2_coef_threshold.txt: C4 3.75 ms at 5 terms, 4.16 at 7) and the
/// coefficient form takes 4.0 ms; the slot form keeps two entries per thread
/// for any term count.  LAMFAST_SLOTS_MIN_TERMS overrides it (A/B runs, tests).
int slots_min_terms() {
    if (const char* e = std::getenv("LAMFAST_SLOTS_MIN_TERMS"))
        return std::max(1, std::atoi(e));
    return 5;
}

/// Slot schedule of the slot form: for every thickness row (absolute i_t) the
/// term each of the n register slots holds, -1 where the row does not use the
/// slot.  A row's terms are those switched on (lam_on) in a layer of a cell
/// under its function.  Rows are walked in order; a term already in a slot
/// keeps it, a new term takes the least recently used slot the row does not
/// need, so with one element per ply each ply's term is formed once.
/// Returns n (2 or 3), or 0 when some row sees more than max_slots terms.
int slot_schedule(const lfb::Setup& s, int max_slots, std::vector<int32_t>& sched) {
    const int T = s.n_terms, nt = s.n_t;
    const int L = T > 0 ? static_cast<int>(s.lam_on.size() / static_cast<std::size_t>(T)) : 0;
    std::vector<std::vector<int>> row_terms(static_cast<std::size_t>(nt));
    {
        std::vector<uint8_t> on(static_cast<std::size_t>(nt) * T, 0);
        for (std::size_t c = 0; c < s.cell_first.size(); ++c)
            for (int t = 0; t < T; ++t)
                if (s.lam_on[static_cast<std::size_t>(t) * L + s.cell_layer[c]])
                    for (int i = s.cell_first[c]; i <= s.cell_first[c] + s.kt.p && i < nt; ++i)
                        on[static_cast<std::size_t>(i) * T + t] = 1;
        for (int i = 0; i < nt; ++i)
            for (int t = 0; t < T; ++t)
                if (on[static_cast<std::size_t>(i) * T + t])
                    row_terms[static_cast<std::size_t>(i)].push_back(t);
    }
    std::size_t most = 0;
    for (const auto& r : row_terms)
        most = std::max(most, r.size());
    if (most > static_cast<std::size_t>(max_slots))
        return 0;
    const int n = most <= 2 ? 2 : 3;
    sched.assign(static_cast<std::size_t>(nt) * n, -1);
    std::vector<int> cur(static_cast<std::size_t>(n), -1), used(static_cast<std::size_t>(n), -1); // term, last row
    for (int i = 0; i < nt; ++i) {
        const auto& terms = row_terms[static_cast<std::size_t>(i)];
        for (int t : terms) // terms that stay where they are
            for (int k = 0; k < n; ++k)
                if (cur[static_cast<std::size_t>(k)] == t)
                    used[static_cast<std::size_t>(k)] = i;
        for (int t : terms) {
            if (std::find(cur.begin(), cur.end(), t) != cur.end())
                continue;
            int best = -1;
            for (int k = 0; k < n; ++k)
                if (used[static_cast<std::size_t>(k)] != i &&
                    (best < 0 || used[static_cast<std::size_t>(k)] < used[static_cast<std::size_t>(best)]))
                    best = k;
            cur[static_cast<std::size_t>(best)] = t; // most <= n: a free slot exists
            used[static_cast<std::size_t>(best)] = i;
        }
        for (int k = 0; k < n; ++k)
            if (used[static_cast<std::size_t>(k)] == i)
                sched[static_cast<std::size_t>(i) * n + k] = cur[static_cast<std::size_t>(k)];
    }
    return n;
}

/// Output-range fields of the device tables (row offsets slab-local).
void set_range(const lfb::Range& r, lfb::DevTables& d) {
    d.t0 = r.t0;
    d.t1 = r.t1;
    d.s0 = r.s0;
    d.s1 = r.s1;
    d.f0 = r.f0;
    d.f1 = r.f1;
    d.out_base = r.out_base;
    d.rp_base = 0;
    d.nnz_slab = r.nnz;
}

void plan_init(lf_plan* plan, const lf_problem* p, int backend, int device, void* stream, int64_t f0, int64_t f1,
               bool want_values = true) {
    if (!p)
        raise(LF_ERR_INVALID_ARGUMENT, "null problem");
    plan->setup = lfb::buildSetupRange(*p, backend, f0, f1);
    use_device(device);
    plan->device = device;
    if (stream) {
        plan->stream = static_cast<cudaStream_t>(stream);
    } else {
        CK(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
        plan->own_stream = true;
    }
    const lfb::Setup& s = plan->setup;
    lfb::DevTables& d = plan->d;
    DeviceArena& ar = plan->arena;
    ar.s = plan->stream;
    upload_space(s, ar, d);
    upload_geometry(s, ar, d);
    upload_thickness(s, ar, d, s.at);
    upload_terms(ar, d, s.n_terms, p->n_layers, s.term_table, s.lam, s.lam_on);
    {
        // major symmetry of every term table (exact up to 1e-15 relative):
        // lets K6 compute half the local pairs and mirror them
        double amax = 0.0, dmax = 0.0;
        for (std::size_t t = 0; t * 81 < s.term_table.size(); ++t)
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l)
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) {
                            const double x = s.term_table[t * 81 + (3 * j + l) * 9 + 3 * a + b];
                            const double y = s.term_table[t * 81 + (3 * l + j) * 9 + 3 * b + a];
                            amax = std::max(amax, std::fabs(x));
                            dmax = std::max(dmax, std::fabs(x - y));
                        }
        d.sym = (dmax <= 1e-15 * amax && !std::getenv("LAMFAST_NO_SYM")) ? 1 : 0;
    }
    d.layer_config = ar.upload(s.layup.layer_config);
    set_range(lfb::rangeOf(s, s.f0, s.f1), d);
    d.w_t0 = s.t0;
    d.w_t1 = s.t1;
    d.n_pairs = s.n_pairs;
    if (backend == LF_BACKEND_STANDARD) {
        d.spt_first_h = s.spt_first.data();
        // affine map: det G C G per configuration for K6 phase 1 (kernel parameter)
        const int n_cfg = static_cast<int>(s.term_table.size() / 81);
        const char* kc = std::getenv("LAMFAST_K6_CONST");
        if (d.affine && n_cfg <= lfb::kK6MaxCfg && !(kc && kc[0] == '0')) {
            plan->k6c.n_cfg = n_cfg;
            for (int c = 0; c < n_cfg; ++c)
                for (int xy = 0; xy < 9; ++xy)
                    for (int ik = 0; ik < 9; ++ik) {
                        const int x = xy / 3, y = xy % 3;
                        double acc = 0.0; // pullback_tables' order (k_ops.cu), without the in-plane weight
                        for (int j = 0; j < 3; ++j)
                            for (int l = 0; l < 3; ++l)
                                acc += d.G[3 * x + j] * d.G[3 * y + l] *
                                       s.term_table[static_cast<std::size_t>(c) * 81 + (3 * j + l) * 9 + ik];
                        plan->k6c.C[c][xy * 9 + ik] = d.det * acc;
                    }
        }
        if (want_values) {
            // two-phase K6: element-local blocks of as many spans per batch as
            // fit 4 GB, one span at least.  The batch size depends on the
            // problem only (not on free memory) and batches are aligned to
            // absolute span multiples (launch_standard), so a row slab sums
            // its entries exactly as the whole matrix does: bitwise equal rows
            // on any partition.
            const std::size_t nl3 = static_cast<std::size_t>(d.pu + 1) * (d.pv + 1) * (d.pt + 1);
            const std::size_t per_blk = 9 * (d.sym ? nl3 * (nl3 + 1) / 2 : nl3 * nl3);
            const std::size_t per_span = static_cast<std::size_t>(d.nspu) * d.nspv * per_blk * sizeof(double);
            const std::size_t budget = std::size_t(4) << 30;
            d.ks_batch = static_cast<int>(std::max<std::size_t>(
                1, std::min<std::size_t>(static_cast<std::size_t>(d.nspt), budget / std::max<std::size_t>(1, per_span))));
            d.Ks = ar.alloc<double>(per_span / sizeof(double) * static_cast<std::size_t>(d.ks_batch));
        }
    }
    if (backend != LF_BACKEND_STANDARD) {
        d.W = ar.alloc<double>(static_cast<std::size_t>(std::max<long long>(1, d.n_pairs)) * d.n_terms * 4);
        d.Wmask = ar.alloc<unsigned>(static_cast<std::size_t>(std::max<long long>(1, d.n_pairs)) * d.n_passes);
        if (!d.affine) {
            d.Pg = ar.alloc<double>(static_cast<std::size_t>(d.n_terms) * 4 * static_cast<std::size_t>(d.E));
            alloc_element_scratch(ar, d, d.n_terms);
        } else if (std::vector<int32_t> sched;
                   d.n_terms >= slots_min_terms() && (d.n_slots = slot_schedule(s, 3, sched)) > 0) {
            // slot form of the per-term combine: rows see <= 3 terms each
            d.slot_term = ar.upload(sched);
        } else if (d.n_terms >= eform_min_terms()) {
            // coefficient form of the combine: one pass for any term count
            d.Etab = ar.alloc<double>(static_cast<std::size_t>(std::max<long long>(1, d.n_pairs)) * lfb::kEPair);
        }
    }
    if (backend != LF_BACKEND_STANDARD && std::getenv("LAMFAST_DEBUG_FORM"))
        std::fprintf(stderr, "lamfast: combine form %s (%d terms, %d slots)\n",
                     d.n_slots > 0 ? "slots" : d.Etab ? "coefficient" : "per-term", d.n_terms, d.n_slots);
    // graph replay for launch-bound plans (<= 64M values, or any standard plan:
    // its colour launches are many and short)
    const char* ge = std::getenv("LAMFAST_GRAPH");
    const bool small = s.nnz <= (64LL << 20) || backend == LF_BACKEND_STANDARD;
    plan->use_graph = ge ? std::atoi(ge) != 0 : small;
    CK(cudaStreamSynchronize(plan->stream)); // the uploads' host sources are temporaries
}

/// Setup kernels of one assembly, everything before the values: basis and
/// thickness weights (W), the 1D integrals / C~ (affine) or the general P.
/// Asynchronous on `s`; returns the number of kernels launched.
int plan_prepare(lf_plan* plan, cudaStream_t s) {
    const lfb::DevTables& d = plan->d;
    int launches = 0;
    if (plan->setup.backend == LF_BACKEND_STANDARD) {
        CK(static_cast<cudaError_t>(lfb::launch_basis(d, false, s)));
        return 1;
    }
    if (d.affine) {
        // one fused setup launch: U, V, thickness-pair weights, Ct
        CK(static_cast<cudaError_t>(lfb::launch_prepare_affine(d, s)));
        if (!d.Etab)
            return 1;
        CK(static_cast<cudaError_t>(lfb::launch_pair_coeffs(d, s)));
        return 2;
    }
    CK(static_cast<cudaError_t>(lfb::launch_basis(d, false, s)));
    ++launches;
    if (d.n_pairs > 0) {
        CK(static_cast<cudaError_t>(lfb::launch_thickness_pairs(d, s)));
        ++launches;
    }
    CK(static_cast<cudaError_t>(lfb::launch_inplane_general(d, s)));
    return launches + lfb::inplane_general_launches(d);
}

/// The value kernels of the output range of `d` (the plan's own range or a
/// sub-range of it) into `values`, after plan_prepare.
int plan_values(lf_plan* plan, const lfb::DevTables& d, double* values, cudaStream_t s) {
    int launches = 0;
    if (plan->setup.backend == LF_BACKEND_STANDARD)
        CK(static_cast<cudaError_t>(lfb::launch_standard(d, values, d.nnz_slab, s, &launches, &plan->k6c)));
    else
        CK(static_cast<cudaError_t>(lfb::launch_combine(d, values, 0, s, &launches)));
    return launches;
}

int plan_launch(lf_plan* plan, double* values, bool timed = true) {
    cudaStream_t s = plan->stream;
    int launches = plan_prepare(plan, s);
    if (!timed)
        return launches + plan_values(plan, plan->d, values, s);
    // CUDA events around the dominant kernels (combine, or the coloured standard launches)
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!plan->free_events.empty()) {
        ev = plan->free_events.back();
        plan->free_events.pop_back();
    } else {
        CK(cudaEventCreate(&ev.first));
        CK(cudaEventCreate(&ev.second));
    }
    CK(cudaEventRecord(ev.first, s));
    launches += plan_values(plan, plan->d, values, s);
    CK(cudaEventRecord(ev.second, s));
    plan->pending.push_back(ev);
    if (plan->pending.size() > 4096)
        plan->harvest();
    return launches;
}

/// One step through the captured graph: the events bracket the whole step
/// (setup + combine), which is what a launch-bound plan's time is.
int plan_launch_graph(lf_plan* plan, double* values) {
    cudaStream_t s = plan->stream;
    if (!plan->graph || plan->graph_values != values) {
        if (plan->graph) {
            CK(cudaGraphExecDestroy(plan->graph));
            plan->graph = nullptr;
        }
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int n = 0;
        try {
            n = plan_launch(plan, values, false);
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g)
                cudaGraphDestroy(g);
            throw;
        }
        CK(cudaStreamEndCapture(s, &g));
        const cudaError_t e = cudaGraphInstantiate(&plan->graph, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        plan->graph_values = values;
        plan->graph_launches = n;
    }
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!plan->free_events.empty()) {
        ev = plan->free_events.back();
        plan->free_events.pop_back();
    } else {
        CK(cudaEventCreate(&ev.first));
        CK(cudaEventCreate(&ev.second));
    }
    CK(cudaEventRecord(ev.first, s));
    CK(cudaGraphLaunch(plan->graph, s));
    CK(cudaEventRecord(ev.second, s));
    plan->pending.push_back(ev);
    if (plan->pending.size() > 4096)
        plan->harvest();
    return plan->graph_launches;
}

void copy_d2h(void* dst, const void* src, std::size_t bytes, cudaStream_t s) {
    if (bytes)
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
}

struct DeviceBuffer {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DeviceBuffer(std::size_t bytes, cudaStream_t st) : s(st) { p = pool_alloc(bytes, st); }
    ~DeviceBuffer() {
        if (p)
            cudaFreeAsync(p, s);
    }
};

/// Entry-layout P (Pg[t][f][e]) -> banded InPlaneOperator blocks (fast.cpp:13-32).
void export_banded(const lfb::Setup& s, const std::vector<double>& pg, int n_terms, double* blocks, char* flags) {
    const int pu = s.ku.p, pv = s.kv.p, bu = 2 * pu + 1, bv = 2 * pv + 1;
    const std::size_t per = static_cast<std::size_t>(s.n_s) * bv * bu;
    const long long E = 9 * s.S_s;
    std::memset(flags, 0, per);
    std::memset(blocks, 0, sizeof(double) * per * 9 * 4 * n_terms);
    for (int is = 0; is < s.n_s; ++is) {
        const int iu = is % s.n_u, iv = is / s.n_u;
        const int Lu = s.au.len[static_cast<std::size_t>(iu)], Lv = s.av.len[static_cast<std::size_t>(iv)];
        const long long B = 3LL * Lu * Lv;
        for (int sv = 0; sv < Lv; ++sv)
            for (int su = 0; su < Lu; ++su) {
                const int jv = s.av.lo[static_cast<std::size_t>(iv)] + sv, ju = s.au.lo[static_cast<std::size_t>(iu)] + su;
                const std::size_t slot = (static_cast<std::size_t>(is) * bv + (jv - iv + pv)) * bu + (ju - iu + pu);
                flags[slot] = 1;
                const long long e0 = s.es_pre[static_cast<std::size_t>(is)] + 3LL * (sv * Lu + su);
                for (int t = 0; t < n_terms; ++t)
                    for (int f = 0; f < 4; ++f)
                        for (int a = 0; a < 3; ++a)
                            for (int b = 0; b < 3; ++b)
                                blocks[((static_cast<std::size_t>(t) * 4 + f) * per + slot) * 9 + 3 * a + b] =
                                    pg[(static_cast<std::size_t>(t) * 4 + f) * E + e0 + a * B + b];
            }
    }
}

} // namespace

extern "C" {

int lf_abi_version(void) { return LF_ABI_VERSION; }

const char* lf_status_name(int status) {
    switch (status) {
    case LF_OK: return "ok";
    case LF_ERR_INVALID_ARGUMENT: return "invalid_argument";
    case LF_ERR_DOMAIN: return "domain_error";
    case LF_ERR_LOGIC: return "logic_error";
    case LF_ERR_RUNTIME: return "runtime_error";
    case LF_ERR_CUDA: return "cuda_error";
    case LF_ERR_OUT_OF_MEMORY: return "out_of_memory";
    case LF_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown";
    }
}

const char* lf_last_error(void) { return g_error.c_str(); }

int lf_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int lf_voigt_from_constants(const lf_orthotropic* c, double d_out[36]) {
    return guarded([&] { lfb::voigtFromConstants(*c, d_out); });
}

int lf_rotate_inplane(const double d[36], double theta, double d_out[36]) {
    return guarded([&] { lfb::rotateInplane(d, theta, d_out); });
}

int lf_angle_decomposition(const lf_orthotropic* c, double out[180]) {
    return guarded([&] { lfb::angleDecomposition(*c, out); });
}

int lf_bracket_parameters(const lf_orthotropic* c, double out[9]) {
    return guarded([&] { lfb::bracketParameters(*c, out); });
}

int lf_gauss_legendre(int32_t n, double a, double b, double* points, double* weights) {
    return guarded([&] { lfb::gaussLegendre(n, a, b, points, weights); });
}

int lf_basis_eval(int32_t degree, int32_t n_knots, const double* knots, double x, int32_t* first_active,
                  double* values, double* derivs) {
    return guarded([&] {
        const lfb::Knots kv = lfb::makeKnots(degree, n_knots, knots, "evaluate");
        *first_active = lfb::evaluateBasis(kv, x, values, derivs);
    });
}

int lf_contraction_table(const double params[9], double angle, double table[81]) {
    return guarded([&] { lfb::contractionTable(params, angle, table); });
}

int lf_layup_configs(const lf_problem* p, int32_t* n_configs, int32_t* layer_config, double* config_stiffness) {
    return guarded([&] {
        const lfb::LayupInfo L = lfb::buildLayup(*p);
        *n_configs = L.n_configs;
        for (int l = 0; l < p->n_layers; ++l)
            layer_config[l] = L.layer_config[static_cast<std::size_t>(l)];
        if (config_stiffness)
            for (int c = 0; c < L.n_configs; ++c)
                std::memcpy(config_stiffness + 36 * c, L.D[static_cast<std::size_t>(c)].data(), 36 * sizeof(double));
    });
}

/// Whether one-shot calls into host arrays write the columns on the host
/// (default) instead of building them on the device and copying them over
/// PCIe.  The columns are a closed form of the adjacency tables (4 B/nnz, a
/// third of the CSR); host threads write them into the destination while the
/// values (8 B/nnz) and row offsets cross PCIe.  LAMFAST_HOST_COLS=0 restores
/// the device pattern (A/B runs, tests).
static bool host_columns_enabled() {
    const char* e = std::getenv("LAMFAST_HOST_COLS");
    return !(e && e[0] == '0');
}

/// Host threads writing the columns of the functions [f0, f1) into `cols`
/// (offset 0 = the first entry of f0), cut into equal-nnz pieces.
struct HostColumns {
    std::vector<std::thread> th;
    /// background: the columns of a whole one-shot call, written while its
    /// values cross PCIe into the same host memory.  They only have to finish
    /// before the copy does, and every extra thread takes memory bandwidth
    /// from the DMA: on the 16-core GPU box 4 threads give 273 ms per C4 call
    /// (a plain D2H of the same bytes: 271 ms), 16 threads 288 ms, 2 threads
    /// 403 ms (profiles/r2_e2e_col_threads.txt).  A quarter of the cores, at
    /// least 4.  Otherwise (a chunk's columns that its sink waits for, or a
    /// plain lf_pattern_columns call): up to 16 threads.
    /// chunk: one chunk's columns into its pinned staging slot while the
    /// chunk's values cross PCIe (lf_assemble_stream); they must be there when
    /// the chunk's copy ends.  3/8 of the cores, at least 6: C5's 203 GB CSR
    /// streams in 2.39 s with 6 threads, 2.45 s with 8, 2.56 s with 16
    /// (profiles/r2_c5_stream_threads.txt).
    HostColumns(const lfb::Setup& s, int64_t f0, int64_t f1, int32_t* cols, bool background = false,
                bool chunk = false) {
        const int64_t base = lfb::functionOffset(s, f0), total = lfb::functionOffset(s, f1) - base;
        const unsigned cores = std::max(1u, std::thread::hardware_concurrency());
        unsigned hw = background ? std::min(16u, std::max(4u, cores / 4))
                      : chunk    ? std::min(16u, std::max(6u, 3 * cores / 8))
                                 : std::min(16u, cores);
        if (const char* e = std::getenv("LAMFAST_COL_THREADS")) // A/B knob: host threads writing the columns
            hw = static_cast<unsigned>(std::max(1, std::atoi(e)));
        const unsigned nt = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(hw, total >> 22)));
        std::vector<int64_t> cut{f0};
        for (unsigned t = 1; t < nt; ++t) { // first function whose offset reaches t/nt of the entries
            const int64_t target = base + total * t / nt;
            int64_t lo = cut.back(), hi = f1;
            while (lo < hi) {
                const int64_t mid = lo + (hi - lo) / 2;
                if (lfb::functionOffset(s, mid) < target)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            cut.push_back(lo);
        }
        cut.push_back(f1);
        try {
            for (unsigned t = 0; t < nt; ++t) {
                const int64_t a = cut[t], b = cut[t + 1];
                if (a < b)
                    th.emplace_back(
                        [&s, a, b, cols, base] { lfb::fillColumns(s, a, b, cols + (lfb::functionOffset(s, a) - base)); });
            }
        } catch (...) { // no thread left running if one cannot be started
            join();
            throw;
        }
    }
    void join() {
        for (auto& x : th)
            if (x.joinable())
                x.join();
    }
    ~HostColumns() { join(); }
};

int lf_pattern_size(const lf_problem* p, int backend, int64_t* dim, int64_t* nnz) {
    return guarded([&] {
        const lfb::Setup s = lfb::buildSetup(*p, backend, 0, -1);
        *dim = 3LL * s.n_s * s.n_t;
        *nnz = s.nnz;
    });
}

int lf_operator_terms(const lf_problem* p, int backend, int32_t* n_terms, double* tables, int32_t* n_slots,
                      int32_t* slot_term) {
    return guarded([&] {
        if (!p || !n_terms || !n_slots)
            raise(LF_ERR_INVALID_ARGUMENT, "lf_operator_terms: null argument");
        if (backend == LF_BACKEND_STANDARD)
            raise(LF_ERR_INVALID_ARGUMENT, "lf_operator_terms: the standard backend has no operator terms");
        const lfb::Setup s = lfb::buildSetup(*p, backend, 0, -1);
        *n_terms = s.n_terms;
        if (tables)
            std::copy(s.term_table.begin(), s.term_table.end(), tables);
        std::vector<int32_t> sched;
        *n_slots = slot_schedule(s, 3, sched);
        if (slot_term && *n_slots > 0)
            std::copy(sched.begin(), sched.end(), slot_term);
    });
}

int lf_pattern_columns(const lf_problem* p, int backend, int64_t f_begin, int64_t f_end, int32_t* cols,
                       int64_t* nnz) {
    return guarded([&] {
        if (!p || !nnz)
            raise(LF_ERR_INVALID_ARGUMENT, "lf_pattern_columns: null argument");
        const lfb::Setup s = lfb::buildSetup(*p, backend, 0, -1);
        const lfb::Range r = lfb::rangeOf(s, f_begin, f_end);
        *nnz = r.nnz;
        if (cols)
            HostColumns(s, r.f0, r.f1, cols).join();
    });
}

int lf_slab_bounds(const lf_problem* p, int backend, int n_parts, int part, int32_t* t_begin, int32_t* t_end,
                   int64_t* row_begin, int64_t* row_end, int64_t* nnz_begin, int64_t* nnz_end) {
    return guarded([&] {
        const lfb::Setup s = lfb::buildSetup(*p, backend, 0, -1);
        int t0 = 0, t1 = 0;
        lfb::slabBounds(s, n_parts, part, &t0, &t1);
        *t_begin = t0;
        *t_end = t1;
        *row_begin = 3LL * s.n_s * t0;
        *row_end = 3LL * s.n_s * t1;
        *nnz_begin = 9 * s.S_s * s.at.pre[static_cast<std::size_t>(t0)];
        *nnz_end = 9 * s.S_s * s.at.pre[static_cast<std::size_t>(t1)];
    });
}

int lf_slab_bounds_functions(const lf_problem* p, int backend, int n_parts, int part, int64_t* f_begin,
                             int64_t* f_end, int64_t* row_begin, int64_t* row_end, int64_t* nnz_begin,
                             int64_t* nnz_end) {
    return guarded([&] {
        const lfb::Setup s = lfb::buildSetup(*p, backend, 0, -1);
        int64_t f0 = 0, f1 = 0;
        lfb::slabBoundsFunctions(s, n_parts, part, &f0, &f1);
        *f_begin = f0;
        *f_end = f1;
        *row_begin = 3 * f0;
        *row_end = 3 * f1;
        *nnz_begin = lfb::functionOffset(s, f0);
        *nnz_end = lfb::functionOffset(s, f1);
    });
}

int lf_plan_create(const lf_problem* p, int backend, int device, void* cuda_stream, int32_t t_begin, int32_t t_end,
                   lf_plan** out) {
    return guarded([&] {
        auto plan = std::make_unique<lf_plan>();
        const auto r = thickness_range(p, t_begin, t_end);
        plan_init(plan.get(), p, backend, device, cuda_stream, r.first, r.second);
        *out = plan.release();
    });
}

int lf_plan_create_range(const lf_problem* p, int backend, int device, void* cuda_stream, int64_t f_begin,
                         int64_t f_end, lf_plan** out) {
    return guarded([&] {
        auto plan = std::make_unique<lf_plan>();
        plan_init(plan.get(), p, backend, device, cuda_stream, f_begin, f_end);
        *out = plan.release();
    });
}

int lf_plan_destroy(lf_plan* plan) {
    return guarded([&] {
        if (plan)
            cudaSetDevice(plan->device);
        delete plan;
    });
}

int lf_plan_info(const lf_plan* plan, int64_t* rows, int64_t* nnz, int64_t* row_begin, int64_t* nnz_begin) {
    return guarded([&] {
        if (rows)
            *rows = plan->setup.rows;
        if (nnz)
            *nnz = plan->setup.nnz;
        if (row_begin)
            *row_begin = plan->setup.row_begin;
        if (nnz_begin)
            *nnz_begin = plan->setup.nnz_begin;
    });
}

int lf_plan_build_pattern(lf_plan* plan, int64_t* d_row_ptr, int32_t* d_cols) {
    return guarded([&] {
        CK(cudaSetDevice(plan->device));
        CK(static_cast<cudaError_t>(lfb::launch_pattern(plan->d, reinterpret_cast<long long*>(d_row_ptr),
                                                        reinterpret_cast<int*>(d_cols), plan->stream)));
    });
}

int lf_plan_assemble(lf_plan* plan, double* d_values) {
    return guarded([&] {
        CK(cudaSetDevice(plan->device));
        plan->launches = plan->use_graph ? plan_launch_graph(plan, d_values) : plan_launch(plan, d_values);
    });
}

int lf_plan_launch_count(const lf_plan* plan) { return plan ? plan->launches : -1; }
int lf_plan_combine_form(const lf_plan* plan) {
    if (!plan || plan->setup.backend == LF_BACKEND_STANDARD)
        return -1;
    return plan->d.n_slots > 0 ? 1 : plan->d.Etab ? 2 : 0;
}

int lf_plan_kernel_time(lf_plan* plan, int reset, double* ms_total, int64_t* launches) {
    return guarded([&] {
        CK(cudaSetDevice(plan->device));
        plan->harvest();
        if (ms_total)
            *ms_total = plan->kernel_ms;
        if (launches)
            *launches = plan->kernel_launches;
        if (reset) {
            plan->kernel_ms = 0.0;
            plan->kernel_launches = 0;
        }
    });
}

int lf_plan_stats(const lf_plan* plan, lf_stats* stats) {
    return guarded([&] {
        stats->qpoint_visits += plan->setup.stats.qpoint_visits;
        stats->frame_evaluations += plan->setup.stats.frame_evaluations;
        stats->operator_builds += plan->setup.stats.operator_builds;
    });
}

int lf_plan_synchronize(lf_plan* plan) {
    return guarded([&] {
        CK(cudaSetDevice(plan->device));
        CK(cudaStreamSynchronize(plan->stream));
    });
}

/// One-shot calls run on a per-(thread, device) pair of streams kept for the
/// thread's lifetime, so the device buffers a call frees are reused by the
/// next call's stream-ordered allocations on the same stream (no fresh
/// mappings of the 23 GB of a C4 CSR).
struct OneShotStreams {
    cudaStream_t main = nullptr, side = nullptr;
};

static OneShotStreams& one_shot_streams(int device) {
    thread_local std::vector<OneShotStreams> per_device;
    if (static_cast<int>(per_device.size()) <= device)
        per_device.resize(static_cast<std::size_t>(device) + 1);
    OneShotStreams& st = per_device[static_cast<std::size_t>(device)];
    if (!st.main) {
        CK(cudaStreamCreateWithFlags(&st.main, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&st.side, cudaStreamNonBlocking));
    }
    return st;
}

/// Pinned host staging of one-shot calls whose destination is pageable (or
/// a chunk sink): two slots, kept per (thread, device) and grown on demand,
/// so a call does not pay for pinning fresh host pages.
struct Staging {
    void* slot[2] = {nullptr, nullptr};
    std::size_t bytes = 0;
    ~Staging() {
        for (void* p : slot)
            if (p)
                cudaFreeHost(p);
    }
    void reserve(std::size_t n) {
        if (n <= bytes)
            return;
        for (void*& p : slot) {
            if (p)
                CK(cudaFreeHost(p));
            p = nullptr;
        }
        bytes = 0;
        for (void*& p : slot)
            CK(cudaHostAlloc(&p, n, cudaHostAllocDefault));
        bytes = n;
    }
};

static Staging& host_staging(int device) {
    thread_local std::vector<std::unique_ptr<Staging>> per_device;
    if (static_cast<int>(per_device.size()) <= device)
        per_device.resize(static_cast<std::size_t>(device) + 1);
    auto& st = per_device[static_cast<std::size_t>(device)];
    if (!st)
        st = std::make_unique<Staging>();
    return *st;
}

static bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

/// memcpy of several (dst, src, bytes) pieces on up to 16 host threads: a
/// pageable destination takes ~50 GB/s only with several cores copying.
static void parallel_copy(const std::vector<std::tuple<void*, const void*, std::size_t>>& jobs) {
    std::size_t total = 0;
    for (const auto& j : jobs)
        total += std::get<2>(j);
    unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (const char* e = std::getenv("LAMFAST_COPY_THREADS")) // A/B knob: host threads emptying a staging slot
        hw = static_cast<unsigned>(std::max(1, std::atoi(e)));
    const unsigned nt = static_cast<unsigned>(std::max<std::size_t>(1, std::min<std::size_t>(hw, total >> 24)));
    if (nt <= 1) {
        for (const auto& j : jobs)
            std::memcpy(std::get<0>(j), std::get<1>(j), std::get<2>(j));
        return;
    }
    // cut the concatenated byte range into nt equal pieces
    auto work = [&](unsigned t) {
        const std::size_t lo = total * t / nt, hi = total * (t + 1) / nt;
        std::size_t off = 0;
        for (const auto& j : jobs) {
            const std::size_t n = std::get<2>(j);
            const std::size_t a = std::max(lo, off), b = std::min(hi, off + n);
            if (a < b)
                std::memcpy(static_cast<char*>(std::get<0>(j)) + (a - off),
                            static_cast<const char*>(std::get<1>(j)) + (a - off), b - a);
            off += n;
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t)
        th.emplace_back(work, t);
    work(0);
    for (auto& x : th)
        x.join();
}

/// Function cuts [f0 = c_0 < c_1 < ... < c_K = f1] of chunks holding at most
/// max_nnz values each (at least one function per chunk).
static std::vector<int64_t> chunk_cuts(const lfb::Setup& s, int64_t f0, int64_t f1, int64_t max_nnz) {
    std::vector<int64_t> cuts{f0};
    int64_t cur = f0;
    while (cur < f1) {
        const int64_t base = lfb::functionOffset(s, cur);
        int64_t lo = cur + 1, hi = f1;
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo + 1) / 2;
            if (lfb::functionOffset(s, mid) - base <= max_nnz)
                lo = mid;
            else
                hi = mid - 1;
        }
        cur = lo;
        cuts.push_back(cur);
    }
    return cuts;
}

/// Destination of a one-shot assembly: the caller's host arrays for the whole
/// range (row offsets from 0 at the range start), or a chunk sink.
struct OneShotOut {
    int64_t* row_ptr = nullptr;
    int32_t* cols = nullptr;
    double* values = nullptr;
    lf_chunk_sink sink = nullptr;
    void* user = nullptr;
};

/// The one-shot pipeline: the range is cut into chunks of at most
/// `chunk_nnz` values; each chunk's pattern and values are computed into one
/// of two device slots on the plan's stream while the other slot's chunk
/// crosses PCIe on the side stream, so the CSR may be larger than HBM (it
/// only has to fit the host).  Pinned destinations receive the D2H directly;
/// pageable ones (and sinks) go through two pinned staging slots, emptied by
/// host threads while the next chunk is copied.
static void run_one_shot(lf_plan& plan, OneShotStreams& st, int64_t chunk_nnz, const OneShotOut& out) {
    const lfb::Setup& s = plan.setup;
    const std::vector<int64_t> cuts = chunk_cuts(s, s.f0, s.f1, chunk_nnz);
    const std::size_t K = cuts.size() - 1;
    std::vector<lfb::Range> rg(K);
    int64_t max_rows = 0, max_nnz = 0;
    for (std::size_t k = 0; k < K; ++k) {
        rg[k] = lfb::rangeOf(s, cuts[k], cuts[k + 1]);
        max_rows = std::max(max_rows, rg[k].rows);
        max_nnz = std::max(max_nnz, rg[k].nnz);
    }
    const bool host_cols = host_columns_enabled();
    const bool staged =
        out.sink || !(is_pinned(out.row_ptr) && (host_cols || is_pinned(out.cols)) && is_pinned(out.values));
    // device slots (two only when there is more than one chunk)
    const int nslot = K > 1 ? 2 : 1;
    const std::size_t rp_bytes = sizeof(int64_t) * static_cast<std::size_t>(max_rows + 1);
    const std::size_t col_bytes = sizeof(int32_t) * static_cast<std::size_t>(std::max<int64_t>(1, max_nnz));
    const std::size_t val_bytes = sizeof(double) * static_cast<std::size_t>(std::max<int64_t>(1, max_nnz));
    std::vector<std::unique_ptr<DeviceBuffer>> drp, dcols, dvals;
    for (int b = 0; b < nslot; ++b) {
        drp.push_back(std::make_unique<DeviceBuffer>(rp_bytes, plan.stream));
        dcols.push_back(std::make_unique<DeviceBuffer>(host_cols ? sizeof(int32_t) : col_bytes, plan.stream));
        dvals.push_back(std::make_unique<DeviceBuffer>(val_bytes, plan.stream));
    }
    // staging slot layout: values | columns | row offsets (8-byte aligned)
    const std::size_t so_cols = val_bytes, so_rp = val_bytes + ((col_bytes + 7) & ~std::size_t(7));
    Staging* stg = nullptr;
    if (staged) {
        stg = &host_staging(plan.device);
        stg->reserve(so_rp + rp_bytes);
    }
    struct Events {
        cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
        ~Events() {
            for (auto x : e)
                if (x)
                    cudaEventDestroy(x);
        }
    } ev;
    for (auto& x : ev.e)
        CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    cudaEvent_t* ready = ev.e;    // [2] slot computed (plan stream)
    cudaEvent_t* drained = ev.e + 2; // [2] slot copied out (side stream)
    cudaStream_t cs = plan.stream, xs = st.side;
    // columns on the host, concurrently with the whole device pipeline (host
    // arrays), or per chunk into the staging slot while the chunk's values
    // cross PCIe (sinks)
    std::unique_ptr<HostColumns> hc, slot_hc[2];
    if (host_cols && !out.sink)
        // pinned arrays: few threads (they compete with the DMA); pageable arrays: all of them, the
        // first touch of fresh pages is the writer's cost there (drop-in C4: 552 ms with 16, 622 ms with 4)
        hc = std::make_unique<HostColumns>(s, s.f0, s.f1, out.cols, /*background=*/!staged);
    plan_prepare(&plan, cs);
    auto finish = [&](std::size_t j) { // host side of chunk j (staged only)
        const int b = static_cast<int>(j % 2);
        CK(cudaEventSynchronize(drained[b]));
        const lfb::Range& r = rg[j];
        const char* base = static_cast<const char*>(stg->slot[b]);
        const double* v = reinterpret_cast<const double*>(base);
        const int32_t* c = reinterpret_cast<const int32_t*>(base + so_cols);
        const int64_t* rp = reinterpret_cast<const int64_t*>(base + so_rp);
        if (slot_hc[b])
            slot_hc[b]->join();
        if (out.sink) {
            if (out.sink(out.user, r.row_begin, r.rows, r.nnz_begin, r.nnz, rp, c, v) != 0)
                raise(LF_ERR_RUNTIME, "lf_assemble_stream: the chunk sink aborted the assembly");
            return;
        }
        const std::size_t ro = static_cast<std::size_t>(r.row_begin - s.row_begin);
        const std::size_t zo = static_cast<std::size_t>(r.nnz_begin - s.nnz_begin);
        if (host_cols)
            parallel_copy({{out.values + zo, v, sizeof(double) * static_cast<std::size_t>(r.nnz)},
                           {out.row_ptr + ro, rp, sizeof(int64_t) * static_cast<std::size_t>(r.rows + 1)}});
        else
            parallel_copy({{out.values + zo, v, sizeof(double) * static_cast<std::size_t>(r.nnz)},
                           {out.cols + zo, c, sizeof(int32_t) * static_cast<std::size_t>(r.nnz)},
                           {out.row_ptr + ro, rp, sizeof(int64_t) * static_cast<std::size_t>(r.rows + 1)}});
    };
    for (std::size_t k = 0; k < K; ++k) {
        const int b = static_cast<int>(k % 2);
        const lfb::Range& r = rg[k];
        lfb::DevTables d = plan.d;
        set_range(r, d);
        d.rp_base = out.sink ? 0 : r.nnz_begin - s.nnz_begin; // sinks get chunk-local row offsets
        if (k >= 2)
            CK(cudaStreamWaitEvent(cs, drained[b], 0)); // the slot's previous chunk has left the device
        auto* rpd = static_cast<long long*>(drp[static_cast<std::size_t>(b % nslot)]->p);
        auto* cd = static_cast<int*>(dcols[static_cast<std::size_t>(b % nslot)]->p);
        auto* vd = static_cast<double*>(dvals[static_cast<std::size_t>(b % nslot)]->p);
        CK(static_cast<cudaError_t>(lfb::launch_pattern(d, rpd, host_cols ? nullptr : cd, cs)));
        if (r.nnz > 0)
            plan_values(&plan, d, vd, cs);
        CK(cudaEventRecord(ready[b], cs));
        CK(cudaStreamWaitEvent(xs, ready[b], 0));
        const std::size_t nv = static_cast<std::size_t>(r.nnz), nr = static_cast<std::size_t>(r.rows + 1);
        if (staged) {
            char* base = static_cast<char*>(stg->slot[b]);
            copy_d2h(base, vd, sizeof(double) * nv, xs);
            if (!host_cols)
                copy_d2h(base + so_cols, cd, sizeof(int32_t) * nv, xs);
            copy_d2h(base + so_rp, rpd, sizeof(int64_t) * nr, xs);
        } else {
            const std::size_t ro = static_cast<std::size_t>(r.row_begin - s.row_begin);
            const std::size_t zo = static_cast<std::size_t>(r.nnz_begin - s.nnz_begin);
            copy_d2h(out.values + zo, vd, sizeof(double) * nv, xs);
            if (!host_cols)
                copy_d2h(out.cols + zo, cd, sizeof(int32_t) * nv, xs);
            copy_d2h(out.row_ptr + ro, rpd, sizeof(int64_t) * nr, xs);
        }
        CK(cudaEventRecord(drained[b], xs));
        if (host_cols && out.sink) // this chunk's columns, into its staging slot, while its values cross PCIe
            slot_hc[b] = std::make_unique<HostColumns>(
                s, r.f0, r.f1, reinterpret_cast<int32_t*>(static_cast<char*>(stg->slot[b]) + so_cols),
                /*background=*/false, /*chunk=*/true);
        if (staged && k >= 1)
            finish(k - 1);
    }
    if (staged && K > 0)
        finish(K - 1);
    CK(cudaStreamSynchronize(xs));
    CK(cudaStreamSynchronize(cs));
    if (hc)
        hc->join();
    CK(cudaGetLastError());
}

/// Values per chunk of a one-shot call: whole range in one chunk when its CSR
/// fits half the free device memory and 2 GiB, else chunks of that size (so
/// the D2H of one overlaps the compute of the next).  `requested` > 0 caps it.
static int64_t default_chunk_nnz(int64_t requested) {
    std::size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const double per_nnz = 12.5; // value + column + a share of the row offsets
    const double slot = std::min<double>(2.0 * (1ull << 30), 0.45 * static_cast<double>(free_b));
    int64_t n = std::max<int64_t>(1 << 20, static_cast<int64_t>(slot / per_nnz));
    if (requested > 0)
        n = std::min(n, requested);
    return n;
}

static int assemble_one_shot(const lf_problem* p, int backend, int device, int64_t f0, int64_t f1, bool whole,
                             const OneShotOut& out, int64_t chunk_nnz, lf_stats* stats) {
    return guarded([&] {
        use_device(device);
        OneShotStreams& streams = one_shot_streams(device);
        lf_plan plan;
        plan_init(&plan, p, backend, device, streams.main, f0, f1);
        const lfb::Setup& s = plan.setup;
        if (s.nnz == 0) {
            if (whole) // the whole matrix: SparseMatrixBuilder::finalize (sparse.cpp:15-18)
                raise(LF_ERR_LOGIC, "SparseMatrixBuilder: nothing accumulated");
            if (out.sink) {
                std::vector<int64_t> zeros(static_cast<std::size_t>(s.rows + 1), 0);
                if (out.sink(out.user, s.row_begin, s.rows, s.nnz_begin, 0, zeros.data(), nullptr, nullptr) != 0)
                    raise(LF_ERR_RUNTIME, "lf_assemble_stream: the chunk sink aborted the assembly");
            } else {
                std::fill(out.row_ptr, out.row_ptr + s.rows + 1, int64_t(0)); // an empty slab: every row empty
            }
            return;
        }
        run_one_shot(plan, streams, default_chunk_nnz(chunk_nnz), out);
        if (stats) {
            stats->qpoint_visits += s.stats.qpoint_visits;
            stats->frame_evaluations += s.stats.frame_evaluations;
            stats->operator_builds += s.stats.operator_builds;
        }
    });
}

int lf_assemble(const lf_problem* p, int backend, int device, int64_t* row_ptr, int32_t* cols, double* values,
                lf_stats* stats) {
    OneShotOut out;
    out.row_ptr = row_ptr;
    out.cols = cols;
    out.values = values;
    return assemble_one_shot(p, backend, device, 0, -1, true, out, 0, stats);
}

int lf_assemble_slab(const lf_problem* p, int backend, int device, int32_t t_begin, int32_t t_end, int64_t* row_ptr,
                     int32_t* cols, double* values, lf_stats* stats) {
    OneShotOut out;
    out.row_ptr = row_ptr;
    out.cols = cols;
    out.values = values;
    const auto r = thickness_range(p, t_begin, t_end);
    return assemble_one_shot(p, backend, device, r.first, r.second, false, out, 0, stats);
}

int lf_assemble_range(const lf_problem* p, int backend, int device, int64_t f_begin, int64_t f_end,
                      int64_t* row_ptr, int32_t* cols, double* values, lf_stats* stats) {
    OneShotOut out;
    out.row_ptr = row_ptr;
    out.cols = cols;
    out.values = values;
    return assemble_one_shot(p, backend, device, f_begin, f_end, false, out, 0, stats);
}

int lf_assemble_stream(const lf_problem* p, int backend, int device, int64_t max_chunk_nnz, lf_chunk_sink sink,
                       void* user, lf_stats* stats) {
    if (!sink) {
        g_error = "lf_assemble_stream: null sink";
        return LF_ERR_INVALID_ARGUMENT;
    }
    OneShotOut out;
    out.sink = sink;
    out.user = user;
    return assemble_one_shot(p, backend, device, 0, -1, true, out, max_chunk_nnz, stats);
}

int lf_reference_bilinear(const lf_problem* p, const double* v, const double* u, int device, double* out) {
    return guarded([&] {
        if (!p || !v || !u || !out)
            raise(LF_ERR_INVALID_ARGUMENT, "referenceBilinear: null argument");
        lf_plan plan;
        plan_init(&plan, p, LF_BACKEND_STANDARD, device, nullptr, 0, -1, false);
        const lfb::DevTables& d = plan.d;
        const std::size_t n = 3 * static_cast<std::size_t>(plan.setup.n_s) * static_cast<std::size_t>(d.nt);
        const std::size_t nblk = static_cast<std::size_t>(d.nspu) * d.nspv * d.nspt;
        DeviceBuffer du(sizeof(double) * n, plan.stream), dv(sizeof(double) * n, plan.stream),
            dpart(sizeof(double) * std::max<std::size_t>(1, nblk), plan.stream), dout(sizeof(double), plan.stream);
        CK(cudaMemcpyAsync(du.p, u, sizeof(double) * n, cudaMemcpyHostToDevice, plan.stream));
        CK(cudaMemcpyAsync(dv.p, v, sizeof(double) * n, cudaMemcpyHostToDevice, plan.stream));
        CK(static_cast<cudaError_t>(lfb::launch_basis(d, false, plan.stream)));
        CK(static_cast<cudaError_t>(lfb::launch_bilinear(d, static_cast<const double*>(du.p),
                                                         static_cast<const double*>(dv.p),
                                                         static_cast<double*>(dpart.p),
                                                         static_cast<double*>(dout.p), plan.stream)));
        CK(cudaMemcpyAsync(out, dout.p, sizeof(double), cudaMemcpyDeviceToHost, plan.stream));
        CK(cudaStreamSynchronize(plan.stream));
    });
}

static int inplane_common(const lf_problem* p, const double table[81], int device, double* blocks, char* flags,
                          lf_stats* stats) {
    return guarded([&] {
        if (!p)
            raise(LF_ERR_INVALID_ARGUMENT, "null problem");
        const lfb::Setup s = lfb::buildSpaceSetup(*p, true);
        use_device(device);
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        {
            DeviceArena ar;
            ar.s = st; // uploads ordered on the kernels' stream (a non-blocking stream does not wait for legacy copies)
            lfb::DevTables d{};
            upload_space(s, ar, d);
            upload_geometry(s, ar, d);
            std::vector<double> tab(table, table + 81), lam(1, 1.0);
            std::vector<uint8_t> on(1, 1);
            upload_terms(ar, d, 1, 1, tab, lam, on);
            d.Pg = ar.alloc<double>(4 * static_cast<std::size_t>(d.E));
            CK(cudaMemsetAsync(d.Pg, 0, sizeof(double) * 4 * d.E, st));
            if (!d.affine)
                alloc_element_scratch(ar, d, 1);
            CK(static_cast<cudaError_t>(lfb::launch_basis(d, d.affine != 0, st)));
            if (d.affine) {
                CK(static_cast<cudaError_t>(lfb::launch_integrals_1d(d, st)));
                CK(static_cast<cudaError_t>(lfb::launch_affine_export(d, st)));
            } else {
                CK(static_cast<cudaError_t>(lfb::launch_inplane_general(d, st)));
            }
            std::vector<double> pg(4 * static_cast<std::size_t>(d.E));
            CK(cudaMemcpyAsync(pg.data(), d.Pg, pg.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            export_banded(s, pg, 1, blocks, flags);
        }
        cudaStreamDestroy(st);
        if (stats) {
            const int64_t per = static_cast<int64_t>(s.spu.size() * s.spv.size()) * s.nqu * s.nqv;
            stats->qpoint_visits += per;
            stats->frame_evaluations += per;
            stats->operator_builds += 1;
        }
    });
}

int lf_inplane_operators(const lf_problem* p, const double material[36], int device, double* blocks, char* flags,
                         lf_stats* stats) {
    double table[81];
    lfb::tableFromVoigt(material, table);
    return inplane_common(p, table, device, blocks, flags, stats);
}

int lf_inplane_operators_bracket(const lf_problem* p, const double table[81], int device, double* blocks,
                                 char* flags, lf_stats* stats) {
    return inplane_common(p, table, device, blocks, flags, stats);
}

int lf_thickness_operators(int32_t degree_t, int32_t n_knots_t, const double* knots_t, int32_t n_interfaces,
                           const double* interfaces, int32_t pts_per_cell, int device, double* q, char* occupied) {
    return guarded([&] {
        lfb::Setup s;
        s.kt = lfb::makeKnots(degree_t, n_knots_t, knots_t, "thickness");
        s.spt = lfb::elementSpans(s.kt);
        s.n_t = s.kt.n;
        s.nqt = pts_per_cell;
        if (pts_per_cell < 1 || pts_per_cell > lfb::kMaxPoints)
            raise(LF_ERR_INVALID_ARGUMENT, "computeThicknessOperators: bad point count");
        s.interfaces.assign(interfaces, interfaces + n_interfaces);
        const int L = n_interfaces - 1;
        s.cells = lfb::thicknessCells(s.kt, s.spt, s.interfaces);
        s.span_cell0.assign(s.spt.size() + 1, 0);
        for (const auto& c : s.cells)
            s.span_cell0[static_cast<std::size_t>(c.span) + 1]++;
        for (std::size_t k = 0; k < s.spt.size(); ++k)
            s.span_cell0[k + 1] += s.span_cell0[k];
        for (const auto& sp : s.spt)
            s.spt_first.push_back(sp.first);
        s.cell_pts.resize(s.cells.size() * static_cast<std::size_t>(s.nqt));
        s.cell_wts.resize(s.cells.size() * static_cast<std::size_t>(s.nqt));
        for (std::size_t c = 0; c < s.cells.size(); ++c) {
            lfb::gaussLegendre(s.nqt, s.cells[c].lo, s.cells[c].hi, s.cell_pts.data() + c * s.nqt,
                               s.cell_wts.data() + c * s.nqt);
            s.cell_first.push_back(s.spt[static_cast<std::size_t>(s.cells[c].span)].first);
            s.cell_layer.push_back(s.cells[c].layer);
        }
        s.at = lfb::adjacency(s.kt.p, s.n_t, s.spt);
        use_device(device);
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        {
            DeviceArena ar;
            ar.s = st; // uploads ordered on the kernels' stream
            lfb::DevTables d{};
            std::memset(&d, 0, sizeof d);
            d.pt = s.kt.p;
            d.nt = s.n_t;
            d.nqt = s.nqt;
            d.nspt = static_cast<int>(s.spt.size());
            d.kt = ar.upload(s.kt.t);
            d.nkt = static_cast<int>(s.kt.t.size());
            upload_thickness(s, ar, d, s.at);
            // one term per layer, identity multipliers: W[pair][l] = Q_l(pair)
            std::vector<double> tab(static_cast<std::size_t>(L) * 81, 0.0), lam(static_cast<std::size_t>(L) * L, 0.0);
            std::vector<uint8_t> on(static_cast<std::size_t>(L) * L, 0);
            for (int l = 0; l < L; ++l) {
                lam[static_cast<std::size_t>(l) * L + l] = 1.0;
                on[static_cast<std::size_t>(l) * L + l] = 1;
            }
            upload_terms(ar, d, L, L, tab, lam, on);
            d.t0 = d.w_t0 = 0;
            d.t1 = d.w_t1 = s.n_t;
            d.n_pairs = s.at.total;
            d.W = ar.alloc<double>(static_cast<std::size_t>(d.n_pairs) * L * 4);
            d.Wmask = ar.alloc<unsigned>(static_cast<std::size_t>(d.n_pairs) * d.n_passes);
            CK(static_cast<cudaError_t>(lfb::launch_basis(d, false, st)));
            CK(static_cast<cudaError_t>(lfb::launch_thickness_pairs(d, st)));
            std::vector<double> w(static_cast<std::size_t>(d.n_pairs) * L * 4);
            CK(cudaMemcpyAsync(w.data(), d.W, w.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const int nt = s.n_t;
            std::memset(q, 0, sizeof(double) * static_cast<std::size_t>(L) * 4 * nt * nt);
            std::memset(occupied, 0, static_cast<std::size_t>(nt) * nt);
            for (int it = 0; it < nt; ++it)
                for (int k = 0; k < s.at.len[static_cast<std::size_t>(it)]; ++k) {
                    const int jt = s.at.lo[static_cast<std::size_t>(it)] + k;
                    const std::size_t pr = static_cast<std::size_t>(s.at.pre[static_cast<std::size_t>(it)] + k);
                    occupied[static_cast<std::size_t>(it) * nt + jt] = 1;
                    for (int l = 0; l < L; ++l)
                        for (int f = 0; f < 4; ++f)
                            q[((static_cast<std::size_t>(l) * 4 + f) * nt + it) * nt + jt] = w[(pr * L + l) * 4 + f];
                }
        }
        cudaStreamDestroy(st);
    });
}

int lf_combine(const lf_problem* p, int32_t n_terms, const double* blocks, const char* flags, const double* thickness,
               const char* thickness_occupied, int device, int64_t* nnz_out, int64_t* row_ptr, int32_t* cols,
               double* values) {
    return guarded([&] {
        if (n_terms < 1)
            raise(LF_ERR_INVALID_ARGUMENT, "combineOperators: no operator terms");
        lfb::Setup s = lfb::buildSpaceSetup(*p, false);
        const int pu = s.ku.p, pv = s.kv.p, bu = 2 * pu + 1, bv = 2 * pv + 1;
        // the in-plane pattern of term 0 / family 0 must be the tensor adjacency
        for (int is = 0; is < s.n_s; ++is) {
            const int iu = is % s.n_u, iv = is / s.n_u;
            for (int dv = -pv; dv <= pv; ++dv)
                for (int du = -pu; du <= pu; ++du) {
                    const int ju = iu + du, jv = iv + dv;
                    if (ju < 0 || ju >= s.n_u || jv < 0 || jv >= s.n_v)
                        continue;
                    const bool adj = ju >= s.au.lo[static_cast<std::size_t>(iu)] &&
                                     ju < s.au.lo[static_cast<std::size_t>(iu)] + s.au.len[static_cast<std::size_t>(iu)] &&
                                     jv >= s.av.lo[static_cast<std::size_t>(iv)] &&
                                     jv < s.av.lo[static_cast<std::size_t>(iv)] + s.av.len[static_cast<std::size_t>(iv)];
                    const std::size_t slot = (static_cast<std::size_t>(is) * bv + (dv + pv)) * bu + (du + pu);
                    if ((flags[slot] != 0) != adj)
                        raise(LF_ERR_UNSUPPORTED, "combineOperators: in-plane occupancy is not the span adjacency");
                }
        }
        // thickness pattern from the occupancy matrix (rows must be intervals)
        const int nt = s.n_t;
        lfb::Adjacency at;
        at.lo.assign(static_cast<std::size_t>(nt), 0);
        at.len.assign(static_cast<std::size_t>(nt), 0);
        at.pre.assign(static_cast<std::size_t>(nt) + 1, 0);
        for (int it = 0; it < nt; ++it) {
            int lo = -1, hi = -1;
            for (int jt = 0; jt < nt; ++jt)
                if (thickness_occupied[static_cast<std::size_t>(it) * nt + jt]) {
                    if (lo < 0)
                        lo = jt;
                    else if (hi != jt - 1)
                        raise(LF_ERR_UNSUPPORTED, "combineOperators: thickness occupancy row is not an interval");
                    hi = jt;
                }
            at.lo[static_cast<std::size_t>(it)] = lo < 0 ? 0 : lo;
            at.len[static_cast<std::size_t>(it)] = lo < 0 ? 0 : hi - lo + 1;
            at.pre[static_cast<std::size_t>(it) + 1] = at.pre[static_cast<std::size_t>(it)] + at.len[static_cast<std::size_t>(it)];
        }
        at.total = at.pre[static_cast<std::size_t>(nt)];
        const int64_t nnz = 9 * s.S_s * at.total;
        *nnz_out = nnz;
        if (!row_ptr && !cols && !values)
            return;
        if (nnz == 0)
            raise(LF_ERR_LOGIC, "SparseMatrixBuilder: nothing accumulated");
        use_device(device);
            cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        {
            DeviceArena ar;
            ar.s = st; // uploads ordered on the kernels' stream
            lfb::DevTables d{};
            upload_space(s, ar, d);
            d.lo_t = ar.upload(at.lo);
            d.len_t = ar.upload(at.len);
            d.pre_t = reinterpret_cast<const long long*>(ar.upload(at.pre));
            d.lt_max = 0;
            for (int it = 0; it < nt; ++it)
                d.lt_max = std::max(d.lt_max, at.len[static_cast<std::size_t>(it)]);
            d.nt = nt;
            d.n_terms = n_terms;
            d.n_passes = (n_terms + 7) / 8;
            d.affine = 0;
            d.t0 = d.w_t0 = 0;
            d.t1 = d.w_t1 = nt;
            d.s0 = 0;
            d.s1 = s.n_s;
            d.f0 = 0;
            d.f1 = static_cast<long long>(nt) * s.n_s;
            d.out_base = d.rp_base = 0;
            d.n_pairs = at.total;
            d.nnz_slab = nnz;
            // P: banded -> entry layout
            const std::size_t per = static_cast<std::size_t>(s.n_s) * bv * bu;
            std::vector<double> pg(static_cast<std::size_t>(n_terms) * 4 * d.E);
            for (int is = 0; is < s.n_s; ++is) {
                const int iu = is % s.n_u, iv = is / s.n_u;
                const int Lu = s.au.len[static_cast<std::size_t>(iu)], Lv = s.av.len[static_cast<std::size_t>(iv)];
                const long long B = 3LL * Lu * Lv;
                for (int sv = 0; sv < Lv; ++sv)
                    for (int su = 0; su < Lu; ++su) {
                        const int jv = s.av.lo[static_cast<std::size_t>(iv)] + sv, ju = s.au.lo[static_cast<std::size_t>(iu)] + su;
                        const std::size_t slot = (static_cast<std::size_t>(is) * bv + (jv - iv + pv)) * bu + (ju - iu + pu);
                        const long long e0 = s.es_pre[static_cast<std::size_t>(is)] + 3LL * (sv * Lu + su);
                        for (int t = 0; t < n_terms; ++t)
                            for (int f = 0; f < 4; ++f)
                                for (int a = 0; a < 3; ++a)
                                    for (int b = 0; b < 3; ++b)
                                        pg[(static_cast<std::size_t>(t) * 4 + f) * d.E + e0 + a * B + b] =
                                            blocks[((static_cast<std::size_t>(t) * 4 + f) * per + slot) * 9 + 3 * a + b];
                    }
            }
            d.Pg = ar.upload(pg);
            std::vector<double> w(static_cast<std::size_t>(at.total) * n_terms * 4);
            std::vector<unsigned> mask(static_cast<std::size_t>(at.total) * d.n_passes, 0u);
            for (int it = 0; it < nt; ++it)
                for (int k = 0; k < at.len[static_cast<std::size_t>(it)]; ++k) {
                    const int jt = at.lo[static_cast<std::size_t>(it)] + k;
                    const std::size_t pr = static_cast<std::size_t>(at.pre[static_cast<std::size_t>(it)] + k);
                    for (int t = 0; t < n_terms; ++t) {
                        for (int f = 0; f < 4; ++f)
                            w[(pr * n_terms + t) * 4 + f] =
                                thickness[((static_cast<std::size_t>(t) * 4 + f) * nt + it) * nt + jt];
                        mask[static_cast<std::size_t>(t / 8) * at.total + pr] |= 1u << (t % 8);
                    }
                }
            d.W = ar.upload(w);
            d.Wmask = ar.upload(mask);
            const std::size_t rows = static_cast<std::size_t>(3LL * s.n_s * nt);
            DeviceBuffer drp(sizeof(int64_t) * (rows + 1), st), dcols(sizeof(int32_t) * nnz, st),
                dvals(sizeof(double) * nnz, st);
            CK(static_cast<cudaError_t>(lfb::launch_pattern(d, static_cast<long long*>(drp.p),
                                                            static_cast<int*>(dcols.p), st)));
            CK(static_cast<cudaError_t>(lfb::launch_combine(d, static_cast<double*>(dvals.p), 0, st, nullptr)));
            if (row_ptr)
                copy_d2h(row_ptr, drp.p, sizeof(int64_t) * (rows + 1), st);
            if (cols)
                copy_d2h(cols, dcols.p, sizeof(int32_t) * nnz, st);
            if (values)
                copy_d2h(values, dvals.p, sizeof(double) * nnz, st);
            CK(cudaStreamSynchronize(st));
        }
        cudaStreamDestroy(st);
    });
}

static double fetch_scalar(double* d_out, cudaStream_t st) {
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, d_out, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return h;
}

int lf_csr_frobenius_sq(int64_t rows, const int64_t* d_row_ptr, const double* d_values, void* cuda_stream,
                        double* out) {
    return guarded([&] {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        DeviceBuffer d_out(sizeof(double), st);
        CK(static_cast<cudaError_t>(lfb::launch_frobenius_sq(rows, reinterpret_cast<const long long*>(d_row_ptr),
                                                             d_values, static_cast<double*>(d_out.p), st)));
        *out = fetch_scalar(static_cast<double*>(d_out.p), st);
    });
}

int lf_csr_spmv(int64_t rows, const int64_t* d_row_ptr, const int32_t* d_cols, const double* d_values,
                const double* d_x, double* d_y, void* cuda_stream) {
    return guarded([&] {
        CK(static_cast<cudaError_t>(lfb::launch_spmv(rows, reinterpret_cast<const long long*>(d_row_ptr),
                                                     reinterpret_cast<const int*>(d_cols), d_values, d_x, d_y,
                                                     static_cast<cudaStream_t>(cuda_stream))));
    });
}

int lf_csr_diff_sq(int64_t rows, const int64_t* d_ra, const int32_t* d_ca, const double* d_va, const int64_t* d_rb,
                   const int32_t* d_cb, const double* d_vb, void* cuda_stream, double* out) {
    return guarded([&] {
        cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
        DeviceBuffer d_out(sizeof(double), st);
        CK(static_cast<cudaError_t>(lfb::launch_diff_sq(
            rows, reinterpret_cast<const long long*>(d_ra), reinterpret_cast<const int*>(d_ca), d_va,
            reinterpret_cast<const long long*>(d_rb), reinterpret_cast<const int*>(d_cb), d_vb,
            static_cast<double*>(d_out.p), st)));
        *out = fetch_scalar(static_cast<double*>(d_out.p), st);
    });
}

static double symmetry_sq(int64_t rows, int64_t row_begin, const int64_t* d_row_ptr, const int32_t* d_cols,
                          const double* d_values, cudaStream_t st, unsigned long long* n_outside) {
    DeviceBuffer d_out(sizeof(double), st), d_cnt(sizeof(unsigned long long), st);
    CK(static_cast<cudaError_t>(lfb::launch_symmetry_sq(
        rows, row_begin, reinterpret_cast<const long long*>(d_row_ptr), reinterpret_cast<const int*>(d_cols),
        d_values, static_cast<double*>(d_out.p), static_cast<unsigned long long*>(d_cnt.p), st)));
    CK(cudaMemcpyAsync(n_outside, d_cnt.p, sizeof *n_outside, cudaMemcpyDeviceToHost, st));
    return fetch_scalar(static_cast<double*>(d_out.p), st);
}

int lf_csr_symmetry_sq(int64_t rows, const int64_t* d_row_ptr, const int32_t* d_cols, const double* d_values,
                       void* cuda_stream, double* out) {
    return guarded([&] {
        unsigned long long outside = 0;
        const double v = symmetry_sq(rows, 0, d_row_ptr, d_cols, d_values, static_cast<cudaStream_t>(cuda_stream),
                                     &outside);
        if (outside)
            raise(LF_ERR_INVALID_ARGUMENT, "symmetryRelError: column index outside the matrix (a row slab? use "
                                           "lf_csr_symmetry_sq_slab)");
        *out = v;
    });
}

int lf_csr_symmetry_sq_slab(int64_t rows, int64_t row_begin, const int64_t* d_row_ptr, const int32_t* d_cols,
                            const double* d_values, void* cuda_stream, double* out, int64_t* n_skipped) {
    return guarded([&] {
        if (row_begin < 0)
            raise(LF_ERR_INVALID_ARGUMENT, "symmetry: negative row_begin");
        unsigned long long outside = 0;
        *out = symmetry_sq(rows, row_begin, d_row_ptr, d_cols, d_values, static_cast<cudaStream_t>(cuda_stream),
                           &outside);
        if (n_skipped)
            *n_skipped = static_cast<int64_t>(outside);
    });
}

int lf_plan_symmetry_sq(lf_plan* plan, const double* d_values, double* out) {
    return guarded([&] {
        CK(cudaSetDevice(plan->device));
        DeviceBuffer d_out(sizeof(double), plan->stream);
        CK(static_cast<cudaError_t>(lfb::launch_plan_symmetry(plan->d, d_values, static_cast<double*>(d_out.p),
                                                              plan->stream)));
        *out = fetch_scalar(static_cast<double*>(d_out.p), plan->stream);
    });
}

int lf_release_memory(int device) {
    return guarded([&] {
        use_device(device);
        CK(cudaDeviceSynchronize());
        CK(cudaMemPoolTrimTo(lib_pool(device), 0));
    });
}

} // extern "C"
