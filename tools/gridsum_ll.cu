// Microbenchmark: flag-in-word ("LL") grid sums at the fused PCG's launch
// shape (148 blocks x 1024 threads), against the counter barrier.
//   B   counter barrier only (red.release + relaxed poll + acquire)
//   L0  LL: warp k posts component k ({epoch|half} x 2 words), every block
//       polls all blocks' slots (slots packed 16 B apart)
//   L1  L0 + release/acquire fences (the ordering sum of the CG)
//   L2  L0 with slots 256 B apart (spread over L2 slices)
//   L3  leader: block 0 collects, publishes the total in one flag slot,
//       the other blocks poll that slot
// Each iteration first runs a store phase (every thread writes `spw` doubles)
// so the fences have outstanding stores to drain, as in the CG's P2.
// usage: nvcc -O3 -arch=sm_100a -o /tmp/gl tools/gridsum_ll.cu && /tmp/gl
#include <cstdint>
#include <cstdio>
constexpr int T = 1024;

#ifndef LLSCOPE
#define LLSCOPE "volatile"
#endif
__device__ __forceinline__ void st_ll(uint64_t *p, double v, unsigned e) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long hi = (unsigned long long)e << 32;
    asm volatile("st." LLSCOPE ".global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(hi | (b & 0xffffffffull)),
                 "l"(hi | (b >> 32))
                 : "memory");
}
// publish through the L2 atomic unit: epoch in the high half, so max wins
__device__ __forceinline__ void red_ll(uint64_t *p, double v, unsigned e) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long hi = (unsigned long long)e << 32;
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(hi | (b & 0xffffffffull)) : "memory");
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p + 1), "l"(hi | (b >> 32)) : "memory");
}
__device__ __forceinline__ void xch_ll(uint64_t *p, double v, unsigned e) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned long long hi = (unsigned long long)e << 32;
    unsigned long long o;
    asm volatile("atom.relaxed.gpu.global.exch.b64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(hi | (b & 0xffffffffull)) : "memory");
    asm volatile("atom.relaxed.gpu.global.exch.b64 %0, [%1], %2;" : "=l"(o) : "l"(p + 1), "l"(hi | (b >> 32)) : "memory");
}
__device__ __forceinline__ bool ld_ll(const uint64_t *p, unsigned e, double &v) {
    unsigned long long lo, hi;
    asm volatile("ld." LLSCOPE ".global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
    if ((unsigned)(lo >> 32) != e || (unsigned)(hi >> 32) != e) return false;
    v = __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
    return true;
}
__device__ __forceinline__ double warp_sum(double t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(~0u, t, o));
    return t;
}
template <int K>
__device__ __forceinline__ double block_stage(const double (&v)[K], double (*s_val)[T]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) s_val[k][threadIdx.x] = v[k];
    __syncthreads();
    double t = 0.0;
    if (warp < K) {
#pragma unroll
        for (int j = 0; j < 32; ++j) t = __dadd_rn(t, s_val[warp][lane + 32 * j]);
        t = warp_sum(t);
    }
    return t;
}
template <int STRIDE>
__device__ __forceinline__ double collect(const uint64_t *row, int G, unsigned e) {
    const int lane = threadIdx.x & 31;
    double w[8];
    unsigned pend = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        w[j] = 0.0;
        if (lane + 32 * j < G) pend |= 1u << j;
    }
    while (pend) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (pend & (1u << j))
                if (ld_ll(row + (size_t)(lane + 32 * j) * STRIDE, e, w[j])) pend &= ~(1u << j);
    }
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t = __dadd_rn(t, w[j]);
    return warp_sum(t);
}

template <int V, int K>
__global__ void __launch_bounds__(T, 1)
    kern(unsigned *bar, uint64_t *part, double *sink, int iters, int spw, double *out, int *bad) {
    __shared__ __align__(16) double s_val[4][T];
    __shared__ double s_tot[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x;
    unsigned target = 0, e = 0;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        for (int s = 0; s < spw; ++s) sink[((size_t)s * G + blockIdx.x) * T + threadIdx.x] = i;
        double v[K];
        for (int k = 0; k < K; ++k) v[k] = (double)(threadIdx.x + k + i + blockIdx.x);
        ++e;
        const int set = i & 1;
        if (V == 0) {  // barrier
            __syncthreads();
            target += G;
            if (threadIdx.x == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
                unsigned x;
                do {
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(bar) : "memory");
                } while ((int)(x - target) < 0);
                asm volatile("{\n\t.reg .u32 t;\n\tld.acquire.gpu.global.u32 t, [%0];\n\t}" ::"l"(bar) : "memory");
            }
            __syncthreads();
            continue;
        }
        if (V == 5) {
            const double t5 = block_stage<K>(v, s_val);
            if (warp < K && lane == 0) s_tot[warp] = t5;
            __syncthreads();
            continue;
        }
        const double t = V >= 6 ? v[0] : block_stage<K>(v, s_val);
        constexpr int STRIDE = V == 3 ? 32 : 2;  // words between slots
        if (V == 1 || V == 2 || V == 3 || V >= 6) {
            if (warp < K) {
                uint64_t *row = part + (size_t)(set * 8 + warp) * 1024 * 32;
                if (lane == 0) {
                    if (V == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    if (V == 7) red_ll(row + (size_t)blockIdx.x * STRIDE, t, e);
                    else if (V == 8) xch_ll(row + (size_t)blockIdx.x * STRIDE, t, e);
                    else st_ll(row + (size_t)blockIdx.x * STRIDE, t, e);
                }
                const double tot = collect<STRIDE>(row, G, e);
                if (V == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
                if (lane == 0) s_tot[warp] = tot;
            }
        } else if (V == 4) {  // leader
            if (warp < K) {
                uint64_t *row = part + (size_t)(set * 8 + warp) * 1024 * 32;
                uint64_t *bc = part + (size_t)(16 + set * 8 + warp) * 1024 * 32;
                if (lane == 0) st_ll(row + (size_t)blockIdx.x * 2, t, e);
                double tot;
                if (blockIdx.x == 0) {
                    tot = collect<2>(row, G, e);
                    if (lane == 0) st_ll(bc, tot, e);
                } else {
                    if (lane == 0)
                        while (!ld_ll(bc, e, tot)) {
                        }
                }
                if (lane == 0) s_tot[warp] = tot;
            }
        }
        __syncthreads();
        for (int k = 0; k < K; ++k) v[k] = s_tot[k];
        if (V >= 6) continue;
        const double Gd = G;
        for (int k = 0; k < K; ++k) {
            const double ex = Gd * (T * (T - 1) / 2.0) + T * (Gd * (Gd - 1) / 2.0) + Gd * T * (k + i);
            if (v[k] != ex && threadIdx.x == 0) atomicAdd(bad, 1);
        }
        acc += v[0];
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

template <int V, int K>
void run(unsigned *bar, uint64_t *part, double *sink, double *out, int *bad, int spw, int grid = 148) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 4000;
    void *args[] = {&bar, &part, &sink, &iters, &spw, &out, &bad};
    float ms = 0, base = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 64);
        cudaMemset(bad, 0, 4);
        cudaMemset(part, 0, 48 * 1024 * 32 * 8);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((const void *)kern<V, K>, grid, T, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    int hb;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("grid %d V%d K=%d spw=%d: %.3f us/iter  wrong=%d (%s)\n", grid, V, K, spw, 1e3 * ms / iters, hb,
           cudaGetErrorString(cudaGetLastError()));
    (void)base;
}
int main() {
    unsigned *bar;
    uint64_t *part;
    double *out, *sink;
    int *bad;
    cudaMalloc(&bar, 64);
    cudaMalloc(&part, 48 * 1024 * 32 * 8);
    cudaMalloc(&sink, (size_t)4 * 148 * T * 8);
    cudaMalloc(&out, 8);
    cudaMalloc(&bad, 4);
    for (int g : {148, 74, 37, 16, 8}) {
        run<0, 1>(bar, part, sink, out, bad, 0, g);
        run<1, 1>(bar, part, sink, out, bad, 0, g);
        run<2, 4>(bar, part, sink, out, bad, 0, g);
        run<4, 1>(bar, part, sink, out, bad, 0, g);
    }
    return 0;
}
