// Microbenchmark: cost of a device-wide barrier (+ K-double deterministic
// reduction) inside a persistent cooperative kernel on B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bar_mine(unsigned *bar, unsigned &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned old = atomicAdd(bar, 1u);
        if (old == gridDim.x - 1) { atomicExch(bar, 0u); __threadfence(); st_release(bar + 1, gen + 1); }
        else while (ld_acquire(bar + 1) == gen) {}
    }
    ++gen;
    __syncthreads();
}
// red.release + flag-per-generation variant: counter grows monotonically
__device__ __forceinline__ void bar_mono(unsigned *bar, unsigned &target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        target += gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while ((int)(ld_acquire(bar) - target) < 0) {}
    }
    __syncthreads();
}
template <int MODE>
__global__ void k(unsigned *bar, int iters, double *part, double *out) {
    unsigned gen = ld_acquire(bar + 1);
    unsigned target = 0;
    if (MODE == 2) target = ld_acquire(bar + 2) ; // not used for mono: assume start 0
    cg::grid_group g = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) g.sync();
        else if (MODE == 1) bar_mine(bar, gen);
        else if (MODE == 2) bar_mono(bar + 4, target);
        else if (MODE == 3) {  // barrier + 5-value reduction read by every block
            if (threadIdx.x < 5) part[threadIdx.x * gridDim.x + blockIdx.x] = i + threadIdx.x;
            bar_mine(bar, gen);
            if (threadIdx.x < 32) {
                double s = 0;
                for (int k5 = 0; k5 < 5; ++k5)
                    for (int j = threadIdx.x; j < gridDim.x; j += 32) s += __ldcg(part + k5 * gridDim.x + j);
                for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
                acc += s;
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}
int main() {
    unsigned *bar; double *part, *out;
    cudaMalloc(&bar, 64); cudaMemset(bar, 0, 64);
    cudaMalloc(&part, 1 << 20); cudaMalloc(&out, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 2000;
    for (int mode = 0; mode < 4; ++mode)
        for (int threads : {256, 512, 1024})
            for (int per : {1, 2, 4}) {
                const void *fn = mode == 0 ? (const void *)k<0> : mode == 1 ? (const void *)k<1> : mode == 2 ? (const void *)k<2> : (const void *)k<3>;
                int maxper = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxper, fn, threads, 0);
                if (per > maxper) continue;
                int grid = 148 * per;
                cudaMemset(bar, 0, 64);
                void *args[] = {&bar, &iters, &part, &out};
                cudaLaunchCooperativeKernel(fn, grid, threads, args, 0, 0);
                cudaMemset(bar, 0, 64);
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel(fn, grid, threads, args, 0, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                printf("mode %d (%s) threads %4d grid %4d: %.3f us/barrier  err=%s\n", mode,
                       mode == 0 ? "cg::grid.sync" : mode == 1 ? "atomic+gen" : mode == 2 ? "red.release mono" : "atomic+gen+5red",
                       threads, grid, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
