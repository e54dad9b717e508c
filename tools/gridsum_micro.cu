// Microbenchmark: the fused PCG's deterministic grid_sum<K> (barrier +
// block-major partials + parallel read + fixed trees) on B200, per call,
// for K = 1, 2, 4, 5 at the kernel's launch shape (512 threads, 2 blocks/SM).
#include <cstdio>
#include <cstdint>
constexpr int CG_THREADS = 512;

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while ((int)(ld_relaxed(bar) - target) < 0) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}
template <int K> __device__ __forceinline__ void warp_tree(double (&t)[K]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __shfl_xor_sync(~0u, t[k], o));
}
template <int K> __device__ __forceinline__ void warp0_combine(const double (*s_warp)[5], double (&t)[K]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = lane < CG_THREADS / 32 ? s_warp[lane][k] : 0.0;
    warp_tree<K>(t);
}
template <int K>
__device__ __forceinline__ void grid_sum(double (&v)[K], double *part, unsigned *bar, unsigned &target,
                                         double (*s_warp)[5], double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    warp_tree<K>(v);
    if (lane == 0)
        for (int k = 0; k < K; ++k) s_warp[warp][k] = v[k];
    __syncthreads();
    if (warp == 0) {
        double t[K];
        warp0_combine<K>(s_warp, t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) part[blockIdx.x * 8 + k] = t[k];
    }
    grid_barrier(bar, target);
    double t[K];
    for (int k = 0; k < K; ++k) t[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += CG_THREADS)
        for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __ldcg(part + b * 8 + k));
    warp_tree<K>(t);
    if (lane == 0)
        for (int k = 0; k < K; ++k) s_warp[warp][k] = t[k];
    __syncthreads();
    if (warp == 0) {
        warp0_combine<K>(s_warp, t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}
template <int K>
__global__ void __launch_bounds__(CG_THREADS, 2) kern(unsigned *bar, double *part, int iters, double *out) {
    __shared__ double s_warp[CG_THREADS / 32][5];
    __shared__ double s_tot[5];
    unsigned target = 0;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        double v[K];
        for (int k = 0; k < K; ++k) v[k] = (double)(threadIdx.x + k + i);
        grid_sum<K>(v, part, bar, target, s_warp, s_tot);
        acc += v[0];
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}
template <int K> void run(unsigned *bar, double *part, double *out, int grid) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int iters = 2000;
    void *args[] = {&bar, &part, &iters, &out};
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(bar, 0, 64);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((const void *)kern<K>, grid, CG_THREADS, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid_sum<%d> grid %d: %.3f us/call (%s)\n", K, grid, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    unsigned *bar; double *part, *out;
    cudaMalloc(&bar, 64); cudaMalloc(&part, 1 << 20); cudaMalloc(&out, 8);
    for (int grid : {148, 205, 296}) {
        run<1>(bar, part, out, grid); run<2>(bar, part, out, grid); run<4>(bar, part, out, grid); run<5>(bar, part, out, grid);
    }
    return 0;
}
