// Microbenchmark: grid barrier variants at 148 x 1024 threads (one CTA/SM).
//   B0 red.release + relaxed poll + fence.acq_rel (the fused PCG's barrier)
//   B1 red.release + relaxed poll + one ld.acquire re-read (no fence)
//   B2 fence.acq_rel + red.relaxed + relaxed poll + fence.acq_rel
//   B3 red.relaxed + relaxed poll, no fences (NOT a valid barrier: floor only)
//   B4 as B0 with stores outstanding (each thread stores 8 doubles first)
//   B5/B6/B7 as B1 with the arrivals split over 4/8/16 counters (block b ->
//        counter b % S, one 128-B line each); lanes 0..S-1 of warp 0 poll
//        one counter each and sum with shuffles, then acquire-re-read
//        their counter (fewer same-address atomics at the L2).
//        B200: B1 1.16, B5 1.28, B6 1.35, B7 1.36 us/barrier
#include <cstdio>
constexpr int T = 1024;
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <int S> __device__ __forceinline__ void barrier_split(unsigned *bar, unsigned &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        if (lane == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 32 * (blockIdx.x % S)) : "memory");
        unsigned *mine = bar + 32 * (lane % S);
        while (true) {
            unsigned c = lane < S ? ld_relaxed(mine) : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(~0u, c, o);
            if ((int)(c - target) >= 0) break;
        }
        if (lane < S) (void)ld_acquire(mine);
        __syncwarp();
    }
    __syncthreads();
}
template <int B> __device__ __forceinline__ void barrier(unsigned *bar, unsigned &target) {
    if (B == 5) { barrier_split<4>(bar, target); return; }
    if (B == 6) { barrier_split<8>(bar, target); return; }
    if (B == 7) { barrier_split<16>(bar, target); return; }
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        if (B == 0 || B == 1 || B == 4) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        if (B == 2) asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        if (B == 3) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while ((int)(ld_relaxed(bar) - target) < 0) {}
        if (B == 0 || B == 2 || B == 4) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (B == 1) (void)ld_acquire(bar);
    }
    __syncthreads();
}
template <int B> __global__ void __launch_bounds__(T, 1) kern(unsigned *bar, double *sink, int iters) {
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        if (B == 4)
#pragma unroll
            for (int k = 0; k < 8; ++k) sink[((size_t)k * gridDim.x + blockIdx.x) * T + threadIdx.x] = i;
        barrier<B>(bar, target);
    }
}
template <int B> void run(unsigned *bar, double *sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 10000, grid = 148;
    void *args[] = {&bar, &sink, &iters};
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 16 * 128);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((const void *)kern<B>, grid, T, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    printf("B%d: %.3f us/barrier (%s)\n", B, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    unsigned *bar;
    double *sink;
    cudaMalloc(&bar, 16 * 128);
    cudaMalloc(&sink, (size_t)8 * 148 * T * 8);
    run<0>(bar, sink); run<1>(bar, sink); run<2>(bar, sink); run<3>(bar, sink); run<4>(bar, sink);
    run<5>(bar, sink); run<6>(bar, sink); run<7>(bar, sink);
    return 0;
}
