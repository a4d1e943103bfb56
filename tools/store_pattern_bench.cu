// Microbenchmark: HBM write bandwidth of the combine kernel's store pattern vs
// simpler patterns, 15.4 GB buffer (C4 values).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/store_bench tools/store_pattern_bench.cu
// Variants:
//   fill        warp w writes 256 B at 256*w (grid-stride)             -- ideal
//   pattern     thread = entry of a row segment of length B; per row it writes
//               L_t values at base + L_t*A + k*B + rem (the combine layout),
//               B = 75 (C4 interior), L_t alternating 3 / 5
//   pattern96   same with B = 96 (every warp piece 256-byte aligned)
//   pattern_cs  'pattern' with st.global.cs
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fill(double* out, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = 1.0;
}

template <bool CS>
__global__ void pattern(double* out, long long E, int B, int nrows, int chunk) {
    const long long e = (long long)blockIdx.x * 256 + threadIdx.x;
    if (e >= E)
        return;
    const long long A = e / B * B;
    const int rem = (int)(e - A);
    const int r0 = blockIdx.y * chunk, r1 = min(nrows, r0 + chunk);
    // row r has L_t = 3 (odd) or 5 (even); base = 8*E per pair-row prefix
    for (int r = r0; r < r1; ++r) {
        const int lt = (r & 1) ? 3 : 5;
        const long long pfx = (long long)(r / 2) * 8 + ((r & 1) ? 5 : 0);
        double* o = out + pfx * E + (long long)lt * A + rem;
        for (int k = 0; k < lt; ++k) {
            if (CS)
                __stcs(o + (long long)k * B, 1.0);
            else
                o[(long long)k * B] = 1.0;
        }
    }
}

// Two adjacent entries per lane, one 16-byte store per (row, k): B even keeps
// every piece 16-byte aligned (128-byte alignment still varies with k).
__global__ void pattern_v2(double* out, long long E, int B, int nrows, int chunk) {
    const long long e = ((long long)blockIdx.x * 256 + threadIdx.x) * 2;
    if (e >= E)
        return;
    const long long A = e / B * B;
    const int rem = (int)(e - A);
    const int r0 = blockIdx.y * chunk, r1 = min(nrows, r0 + chunk);
    for (int r = r0; r < r1; ++r) {
        const int lt = (r & 1) ? 3 : 5;
        const long long pfx = (long long)(r / 2) * 8 + ((r & 1) ? 5 : 0);
        double* o = out + pfx * E + (long long)lt * A + rem;
        for (int k = 0; k < lt; ++k)
            __stcs(reinterpret_cast<double2*>(o + (long long)k * B), make_double2(1.0, 1.0));
    }
}

// Warp-specialised staging: NP producer warps write the block's contiguous
// row range into a smem slot, NC consumer warps copy it out with 128-byte
// aligned 16-byte stores; named barriers hand slots over (no block barrier).
template <int NP, int NC, int NSLOT>
__global__ void __launch_bounds__((NP + NC) * 32) ws_pattern(double* out, long long E, int B, int nrows, int chunk,
                                                              int cap) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x / 32;
    const int nthreads = (NP + NC) * 32;
    // block owns whole groups: entries [e0, e1)
    const long long e0 = (long long)blockIdx.x * (cap / B) * B;
    const long long e1 = min(E, e0 + (long long)(cap / B) * B);
    const int ne = (int)(e1 - e0);
    const int slot_len = 5 * cap + 32;
    const int r0 = blockIdx.y * chunk, r1 = min(nrows, r0 + chunk);
    if (warp < NP) {
        for (int r = r0, i = 0; r < r1; ++r, ++i) {
            const int slot = i % NSLOT;
            if (i >= NSLOT) // wait until consumers released this slot
                asm volatile("bar.sync %0, %1;" ::"r"(1 + NSLOT + slot), "r"(nthreads));
            const int lt = (r & 1) ? 3 : 5;
            const long long pfx = (long long)(r / 2) * 8 + ((r & 1) ? 5 : 0);
            const long long dst = pfx * E + (long long)lt * e0;
            double* sb = smem + slot * slot_len + (int)(dst & 1);
            for (int x = threadIdx.x; x < ne; x += NP * 32) {
                const int loc = x / B * B, rem = x - loc;
                for (int k = 0; k < lt; ++k)
                    sb[lt * loc + k * B + rem] = 1.0;
            }
            asm volatile("bar.arrive %0, %1;" ::"r"(1 + slot), "r"(nthreads));
        }
    } else {
        const int ct = threadIdx.x - NP * 32;
        for (int r = r0, i = 0; r < r1; ++r, ++i) {
            const int slot = i % NSLOT;
            asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(nthreads));
            const int lt = (r & 1) ? 3 : 5;
            const long long pfx = (long long)(r / 2) * 8 + ((r & 1) ? 5 : 0);
            const long long dst = pfx * E + (long long)lt * e0;
            const double* sb = smem + slot * slot_len + (int)(dst & 1);
            const int n = lt * ne;
            double* g = out + dst;
            const int head = (int)min((long long)n, (16 - (dst & 15)) & 15);
            if (ct < head)
                __stcs(g + ct, sb[ct]);
            const int body = (n - head) >> 1;
            const double2* sv = reinterpret_cast<const double2*>(sb + head);
            double2* gv = reinterpret_cast<double2*>(g + head);
            for (int v = ct; v < body; v += NC * 32)
                __stcs(gv + v, sv[v]);
            if (((n - head) & 1) && ct == 0)
                __stcs(g + n - 1, sb[n - 1]);
            if (r + NSLOT < r1) // release the slot for the producers' row i + NSLOT
                asm volatile("bar.arrive %0, %1;" ::"r"(1 + NSLOT + slot), "r"(nthreads));
        }
    }
}

// Warp-private staging: warp w owns one whole row segment group (B entries,
// lanes hold entries lane + 32x), writes its L_t*B values per row into its own
// double-buffered smem slice, then copies the contiguous region out with
// 16-byte stores whose warp footprint starts on a 128-byte line.  Only
// __syncwarp, no block barriers.  MINB forces the blocks/SM of the real kernel.
template <int EPT, int MINB, int GPW = 1, bool TMA = false>
__global__ void __launch_bounds__(256, MINB) wp_pattern(double* out, long long E, int B, int nrows, int chunk) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long g = (long long)blockIdx.x * 8 + warp;
    const long long g0 = g * B * GPW;
    if (g0 >= E)
        return;
    const int W = B * GPW; // entries of this warp
    const int slot_len = (5 * W + 3) & ~1;
    double* buf = smem + warp * 2 * slot_len;
    const int r0 = blockIdx.y * chunk, r1 = min(nrows, r0 + chunk);
    for (int r = r0, i = 0; r < r1; ++r, ++i) {
        const int lt = (r & 1) ? 3 : 5;
        const long long pfx = (long long)(r / 2) * 8 + ((r & 1) ? 5 : 0);
        const long long G = pfx * E + (long long)lt * g0;
        double* sb = buf + (i & 1) * slot_len + (int)(G & 1);
#pragma unroll
        for (int x = 0; x < EPT; ++x) {
            const int ent = lane + 32 * x;
            const int grp = ent / B, rem = ent - grp * B;
            if (ent < W)
                for (int k = 0; k < lt; ++k)
                    sb[lt * B * grp + k * B + rem] = 1.0;
        }
        const int n = lt * W;
        if constexpr (TMA) {
            double* gp = out + G;
            const int h = (int)(G & 1);
            const int nb = (n - h) & ~1;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (h)
                    __stcs(gp, sb[0]);
                if (n - h - nb)
                    __stcs(gp + n - 1, sb[n - 1]);
                // the buffer written two rows ago must have been read
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gp + h),
                             "r"((unsigned)__cvta_generic_to_shared(sb + h)), "r"(nb * 8)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
            __syncwarp();
            continue;
        }
        __syncwarp();
        double* gp = out + G;
        const int head = (int)min((long long)n, (16 - (G & 15)) & 15);
        if (lane < head)
            __stcs(gp + lane, sb[lane]);
        const int body = (n - head) >> 1;
        const double2* sv = reinterpret_cast<const double2*>(sb + head);
        double2* gv = reinterpret_cast<double2*>(gp + head);
        for (int v = lane; v < body; v += 32)
            __stcs(gv + v, sv[v]);
        if (((n - head) & 1) && lane == 0)
            __stcs(gp + n - 1, sb[n - 1]);
    }
    if (TMA && lane == 0)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Warp owns a contiguous sub-range of one group: `parts` warps split each group
// (entries [part*B/parts, (part+1)*B/parts)); per row the warp stages its
// L_t pieces and issues one bulk copy per piece (8-byte head/tail scalar).
template <int EPT>
__global__ void __launch_bounds__(256, 1) wp_part_pattern(double* out, long long E, int B, int nrows, int chunk,
                                                         int parts) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * 8 + warp;
    const long long g = gw / parts;
    const int part = (int)(gw % parts);
    const long long g0 = g * B;
    if (g0 >= E)
        return;
    const int lo = part * B / parts, hi = (part + 1) * B / parts, W = hi - lo;
    const int slot_len = (5 * (W + 2) + 3) & ~1;
    double* buf = smem + warp * 2 * slot_len;
    const int r0 = blockIdx.y * chunk, r1 = min(nrows, r0 + chunk);
    for (int r = r0, i = 0; r < r1; ++r, ++i) {
        const int lt = (r & 1) ? 3 : 5;
        const long long pfx = (long long)(r / 2) * 8 + ((r & 1) ? 5 : 0);
        const long long G = pfx * E + (long long)lt * g0 + lo;
        double* sb = buf + (i & 1) * slot_len;
        // piece k starts at G + k*B; staged at sb + k*(W+2) + ((G + k*B) & 1)
#pragma unroll
        for (int x = 0; x < EPT; ++x) {
            const int ent = lane + 32 * x;
            if (ent < W)
                for (int k = 0; k < lt; ++k)
                    sb[k * ((W + 3) & ~1) + (int)((G + (long long)k * B) & 1) + ent] = 1.0;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < lt) {
            const int k = lane;
            const long long Gk = G + (long long)k * B;
            double* gp = out + Gk;
            const double* sk = sb + k * ((W + 3) & ~1) + (int)(Gk & 1);
            const int h = (int)(Gk & 1);
            const int nb = (W - h) & ~1;
            if (h)
                __stcs(gp, sk[0]);
            if (W - h - nb)
                __stcs(gp + W - 1, sk[W - 1]);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gp + h),
                         "r"((unsigned)__cvta_generic_to_shared(sk + h)), "r"(nb * 8)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncwarp();
    }
    if (lane < 5)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int nrows = 257;
    long long E = 1884000; // ~C4 entry count
    const long long pairs = (long long)(nrows / 2) * 8 + 5;
    double* buf;
    const long long n = pairs * E;
    if (cudaMalloc(&buf, n * sizeof(double)) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i)
            launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        printf("%-12s %8.3f ms  %7.1f GB/s  (%s)\n", name, ms, n * 8.0 / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    timeit("fill", [&] { fill<<<148 * 16, 256>>>(buf, n); });
    for (int B : {75, 96}) {
        const long long EB = E / B * B;
        dim3 grid((unsigned)((EB + 255) / 256), 5);
        const int chunk = (nrows + 4) / 5;
        char nm[32];
        snprintf(nm, sizeof nm, "pattern%d", B);
        timeit(nm, [&] { pattern<false><<<grid, 256>>>(buf, EB, B, nrows, chunk); });
        snprintf(nm, sizeof nm, "pattern%d_cs", B);
        timeit(nm, [&] { pattern<true><<<grid, 256>>>(buf, EB, B, nrows, chunk); });
    }
    for (int B : {74, 146}) {
        const long long EB = E / B * B;
        dim3 grid((unsigned)((EB / 2 + 255) / 256), 5);
        const int chunk = (nrows + 4) / 5;
        char nm[32];
        snprintf(nm, sizeof nm, "v2_B%d", B);
        timeit(nm, [&] { pattern_v2<<<grid, 256>>>(buf, EB, B, nrows, chunk); });
        dim3 grid1((unsigned)((EB + 255) / 256), 5);
        snprintf(nm, sizeof nm, "scalar_B%d", B);
        timeit(nm, [&] { pattern<true><<<grid1, 256>>>(buf, EB, B, nrows, chunk); });
    }
    for (int B : {75, 147}) {
        const int cap = 512;
        const long long EB = E / B * B;
        const long long per = cap / B * B;
        const int chunk = 52;
        dim3 grid((unsigned)((EB + per - 1) / per), (nrows + chunk - 1) / chunk);
        const size_t smem = 3 * (5 * cap + 32) * sizeof(double);
        char nm[32];
        snprintf(nm, sizeof nm, "ws8+2_B%d", B);
        cudaFuncSetAttribute(ws_pattern<8, 2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        timeit(nm, [&] { ws_pattern<8, 2, 3><<<grid, 320, smem>>>(buf, EB, B, nrows, chunk, cap); });
        snprintf(nm, sizeof nm, "ws8+4_B%d", B);
        cudaFuncSetAttribute(ws_pattern<8, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        timeit(nm, [&] { ws_pattern<8, 4, 3><<<grid, 384, smem>>>(buf, EB, B, nrows, chunk, cap); });
    }
    for (int B : {75, 147}) {
        const long long EB = E / B * B;
        const long long ng = EB / B;
        const int chunk = 52;
        dim3 grid((unsigned)((ng + 7) / 8), (nrows + chunk - 1) / chunk);
        const size_t smem = 8 * 2 * ((5 * B * 2 + 3) & ~1) * sizeof(double);
        char nm[32];
        auto run = [&](auto kern, const char* tag) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            snprintf(nm, sizeof nm, "wp_%s_B%d", tag, B);
            timeit(nm, [&] { kern<<<grid, 256, smem>>>(buf, EB, B, nrows, chunk); });
        };
        if (B == 75) {
            run(wp_pattern<3, 1>, "m1");
            run(wp_pattern<3, 1, 1, true>, "tma");
        } else {
            run(wp_pattern<5, 1>, "m1");
            run(wp_pattern<5, 1, 1, true>, "tma");
        }
        dim3 grid2((unsigned)((ng / 2 + 7) / 8), (nrows + chunk - 1) / chunk);
        auto run2 = [&](auto kern, const char* tag) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            snprintf(nm, sizeof nm, "wp2_%s_B%d", tag, B);
            timeit(nm, [&] { kern<<<grid2, 256, smem>>>(buf, EB / (2 * B) * 2 * B, B, nrows, chunk); });
        };
        if (B == 75) {
            run2(wp_pattern<5, 1, 2>, "m1");
            run2(wp_pattern<5, 1, 2, true>, "tma");
        } else {
            run2(wp_pattern<10, 1, 2>, "m1");
            run2(wp_pattern<10, 1, 2, true>, "tma");
        }
    }
    for (int B : {75, 147}) {
        const long long EB = E / B * B;
        const long long ng = EB / B;
        const int chunk = 52;
        for (int parts : {1, 2, 3}) {
            dim3 grid((unsigned)((ng * parts + 7) / 8), (nrows + chunk - 1) / chunk);
            const int W = (B + parts - 1) / parts;
            const size_t smem = 8 * 2 * ((5 * (W + 2) + 3) & ~1) * sizeof(double);
            char nm[32];
            snprintf(nm, sizeof nm, "part%d_B%d", parts, B);
            auto kern = W <= 96 ? wp_part_pattern<3> : wp_part_pattern<5>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            timeit(nm, [&] { kern<<<grid, 256, smem>>>(buf, EB, B, nrows, chunk, parts); });
        }
    }
    cudaFree(buf);
    return 0;
}
