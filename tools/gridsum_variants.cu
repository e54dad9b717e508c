// Microbenchmark: grid-wide deterministic sums at the fused PCG's launch
// shape (148 blocks x 1024 threads, one per SM), three designs:
//   V0  counter barrier (red.release + relaxed poll + fence), then every
//       block reads all partials with 1024 threads, two smem trees;
//   V1  same barrier, warp 0 alone reads the partials and reduces them;
//   V2  no counter: the partials are their own flags.  Three rotating
//       partial sets; a slot holds a signalling-NaN sentinel until written;
//       warp 0 polls the slots (relaxed) and fences once.  The block that
//       owns a slot re-arms it two reductions ahead.
// usage: nvcc -O3 -arch=sm_100a gridsum_variants.cu && ./a.out
#include <cstdint>
#include <cstdio>
constexpr int T = 1024;
constexpr unsigned long long SENT = 0x7ff4dead0badf00dull;  // sNaN: arithmetic never produces it

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ld_relaxed_v2(const double *p, unsigned long long &a, unsigned long long &b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_relaxed(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
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
template <int K> __device__ __forceinline__ void block_partial(double (&v)[K], double (*s_warp)[5], double (&t)[K]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    warp_tree<K>(v);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) s_warp[warp][k] = v[k];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] = s_warp[lane][k];
        warp_tree<K>(t);
    }
}

template <int K>
__device__ void sum_v0(double (&v)[K], double *part, unsigned *bar, unsigned &target, double (*s_warp)[5],
                       double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double t[K];
    block_partial<K>(v, s_warp, t);
    if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) part[blockIdx.x * 8 + k] = t[k];
    grid_barrier(bar, target);
    for (int k = 0; k < K; ++k) t[k] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += T)
        for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __ldcg(part + b * 8 + k));
    warp_tree<K>(t);
    if (lane == 0)
        for (int k = 0; k < K; ++k) s_warp[warp][k] = t[k];
    __syncthreads();
    if (warp == 0) {
        for (int k = 0; k < K; ++k) t[k] = s_warp[lane][k];
        warp_tree<K>(t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

template <int K>
__device__ void sum_v1(double (&v)[K], double *part, unsigned *bar, unsigned &target, double (*s_warp)[5],
                       double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double t[K];
    block_partial<K>(v, s_warp, t);
    if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) part[blockIdx.x * 8 + k] = t[k];
    grid_barrier(bar, target);
    if (warp == 0) {
        for (int k = 0; k < K; ++k) t[k] = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32)
            for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __ldcg(part + b * 8 + k));
        warp_tree<K>(t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

template <int K>
__device__ void sum_v3(double (&v)[K], double *part, unsigned *bar, unsigned &target, double (*s_warp)[5],
                       double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double t[K];
    block_partial<K>(v, s_warp, t);
    if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) part[blockIdx.x * 8 + k] = t[k];
    grid_barrier(bar, target);
    if (warp == 0) {
        constexpr int J = 5;  // ceil(148 / 32)
        double w[J][K];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int b = lane + 32 * j;
#pragma unroll
            for (int k = 0; k < K; ++k) w[j][k] = b < (int)gridDim.x ? __ldcg(part + b * 8 + k) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            t[k] = w[0][k];
#pragma unroll
            for (int j = 1; j < J; ++j) t[k] = __dadd_rn(t[k], w[j][k]);
        }
        warp_tree<K>(t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

template <int K>
__device__ void sum_v4(double (&v)[K], double *part, unsigned &gen, double (*s_warp)[5], double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = gridDim.x;
    double t[K];
    block_partial<K>(v, s_warp, t);
    const int set = gen % 3, next = (gen + 1) % 3;
    ++gen;
    __syncthreads();
    if (warp == 0) {
        if (lane < K) {
            double tv = t[0];
#pragma unroll
            for (int k = 1; k < K; ++k)
                if (lane == k) tv = t[k];
            st_relaxed(part + ((size_t)next * G + blockIdx.x) * 4 + lane, __longlong_as_double(SENT));
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            st_relaxed(part + ((size_t)set * G + blockIdx.x) * 4 + lane, tv);
        }
        constexpr int J = 5;
        unsigned long long w[J][4];
        unsigned pending = 0;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            w[j][0] = w[j][1] = w[j][2] = w[j][3] = 0;
            if (lane + 32 * j < G) pending |= 1u << j;
        }
        while (pending) {
#pragma unroll
            for (int j = 0; j < J; ++j)
                if (pending >> j & 1) {
                    const double *s = part + ((size_t)set * G + lane + 32 * j) * 4;
                    ld_relaxed_v2(s, w[j][0], w[j][1]);
                    if (K > 2) ld_relaxed_v2(s + 2, w[j][2], w[j][3]);
                }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                bool ok = w[j][0] != SENT && (K < 2 || w[j][1] != SENT) && (K < 3 || w[j][2] != SENT) &&
                          (K < 4 || w[j][3] != SENT);
                if (ok) pending &= ~(1u << j);
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
        for (int k = 0; k < K; ++k) {
            t[k] = lane < G ? __longlong_as_double(w[0][k]) : 0.0;
#pragma unroll
            for (int j = 1; j < J; ++j)
                t[k] = __dadd_rn(t[k], lane + 32 * j < G ? __longlong_as_double(w[j][k]) : 0.0);
        }
        warp_tree<K>(t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

// V5: barrier only; V6: block partial (trees) only
template <int K>
__device__ void sum_v5(double (&v)[K], unsigned *bar, unsigned &target) {
    grid_barrier(bar, target);
}
template <int K>
__device__ void sum_v6(double (&v)[K], double (*s_warp)[5], double *s_tot) {
    double t[K];
    block_partial<K>(v, s_warp, t);
    if (threadIdx.x == 0)
        for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    __syncthreads();
}

// V7: smem block partial (warp k owns component k) + per-component post stage
template <int K>
__device__ void block_partial_smem(double (&v)[K], double (*s_val)[T], double (&t)) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) s_val[k][threadIdx.x] = v[k];
    __syncthreads();
    if (warp < K) {
        // lane i sums threads i, i+32, i+64, ... of component `warp` in order (conflict-free)
        const double *col = &s_val[warp][lane];
        double x[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = col[32 * j];
        double acc = x[0];
#pragma unroll
        for (int j = 1; j < 32; ++j) acc = __dadd_rn(acc, x[j]);
        double tt[1] = {acc};
        warp_tree<1>(tt);
        t = tt[0];
    }
}
template <int K>
__device__ void sum_v7(double (&v)[K], double *part, unsigned *bar, unsigned &target, double (*s_val)[T],
                       double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double t;
    block_partial_smem<K>(v, s_val, t);
    if (warp < K && lane == 0) part[blockIdx.x * 8 + warp] = t;
    grid_barrier(bar, target);
    if (warp < K) {
        constexpr int J = 5;
        double w[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int b = lane + 32 * j;
            w[j] = b < (int)gridDim.x ? __ldcg(part + b * 8 + warp) : 0.0;
        }
        double tt[1] = {w[0]};
#pragma unroll
        for (int j = 1; j < J; ++j) tt[0] = __dadd_rn(tt[0], w[j]);
        warp_tree<1>(tt);
        if (lane == 0) s_tot[warp] = tt[0];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}
// V8: barrier + warp 0 loading the partials (no trees)
template <int K>
__device__ void sum_v8(double (&v)[K], double *part, unsigned *bar, unsigned &target, double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    grid_barrier(bar, target);
    if (warp == 0) {
        double a = 0;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int b = lane + 32 * j;
#pragma unroll
            for (int k = 0; k < K; ++k) a += b < (int)gridDim.x ? __ldcg(part + b * 8 + k) : 0.0;
        }
        if (lane == 0) s_tot[0] = a;
    }
    __syncthreads();
}

// V2: slot b of set s at part + (s*G + b)*4 (32 B, K <= 4)
template <int K>
__device__ void sum_v2(double (&v)[K], double *part, unsigned &gen, double (*s_warp)[5], double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = gridDim.x;
    double t[K];
    block_partial<K>(v, s_warp, t);  // t valid in warp 0
    const int set = gen % 3, next = (gen + 1) % 3;
    ++gen;
    __syncthreads();  // every thread's prior stores precede the release below
    if (warp == 0) {
        if (lane < K) {
            double tv = t[0];
#pragma unroll
            for (int k = 1; k < K; ++k)
                if (lane == k) tv = t[k];
            // re-arm our slot of the set used two reductions ahead ...
            st_relaxed(part + ((size_t)next * G + blockIdx.x) * 4 + lane, __longlong_as_double(SENT));
            // ... then publish (release orders the re-arm and the block's stores)
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            st_relaxed(part + ((size_t)set * G + blockIdx.x) * 4 + lane, tv);
        }
        for (int k = 0; k < K; ++k) t[k] = 0.0;
        for (int b = lane; b < G; b += 32) {
            const double *s = part + ((size_t)set * G + b) * 4;
            unsigned long long a0, a1, a2 = 0, a3 = 0;
            for (;;) {
                ld_relaxed_v2(s, a0, a1);
                if (K > 2) ld_relaxed_v2(s + 2, a2, a3);
                bool ok = a0 != SENT && (K < 2 || a1 != SENT) && (K < 3 || a2 != SENT) && (K < 4 || a3 != SENT);
                if (ok) break;
            }
            const unsigned long long w[4] = {a0, a1, a2, a3};
#pragma unroll
            for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __longlong_as_double(w[k]));
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        warp_tree<K>(t);
        if (lane == 0)
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
    }
    __syncthreads();
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

template <int V, int K>
__global__ void __launch_bounds__(T, 1) kern(unsigned *bar, double *part, int iters, double *out, int *bad) {
    __shared__ double s_warp[T / 32][5];
    __shared__ double s_tot[5];
    __shared__ __align__(16) double s_val[V == 7 ? K : 1][T];
    unsigned target = 0, gen = 0;
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        double v[K];
        for (int k = 0; k < K; ++k) v[k] = (double)(threadIdx.x + k + i + blockIdx.x);
        if (V == 0) sum_v0<K>(v, part, bar, target, s_warp, s_tot);
        if (V == 1) sum_v1<K>(v, part, bar, target, s_warp, s_tot);
        if (V == 2) sum_v2<K>(v, part, gen, s_warp, s_tot);
        if (V == 3) sum_v3<K>(v, part, bar, target, s_warp, s_tot);
        if (V == 4) sum_v4<K>(v, part, gen, s_warp, s_tot);
        if (V == 5) sum_v5<K>(v, bar, target);
        if (V == 7) sum_v7<K>(v, part, bar, target, s_val, s_tot);
        if (V == 8) { sum_v8<K>(v, part, bar, target, s_tot); continue; }
        if (V == 6) sum_v6<K>(v, s_warp, s_tot);
        if (V >= 5) continue;
        // exact expected sum (small integers): sum over blocks and threads
        const double G = gridDim.x;
        for (int k = 0; k < K; ++k) {
            const double e = G * (T * (T - 1) / 2.0) + T * (G * (G - 1) / 2.0) + G * T * (k + i);
            if (v[k] != e && threadIdx.x == 0) atomicAdd(bad, 1);
        }
        acc += v[0];
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = acc;
}

template <int V, int K> void run(unsigned *bar, double *part, double *out, int *bad, int grid) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 4000;
    void *args[] = {&bar, &part, &iters, &out, &bad};
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 64);
        cudaMemset(bad, 0, 4);
        // sentinel-fill the V2 sets (3 x grid slots x 4 doubles)
        static unsigned long long h[3 * 1024 * 4];
        for (auto &x : h) x = SENT;
        cudaMemcpy(part, h, sizeof h, cudaMemcpyHostToDevice);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((const void *)kern<V, K>, grid, T, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    int hb;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("V%d K=%d grid %d: %.3f us/sum  wrong=%d (%s)\n", V, K, grid, 1e3 * ms / iters, hb,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    unsigned *bar;
    double *part, *out;
    int *bad;
    cudaMalloc(&bar, 64);
    cudaMalloc(&part, 1 << 20);
    cudaMalloc(&out, 8);
    cudaMalloc(&bad, 4);
    for (int grid : {148}) {
        run<5, 1>(bar, part, out, bad, grid);
        run<8, 1>(bar, part, out, bad, grid);
        run<8, 4>(bar, part, out, bad, grid);
        run<0, 2>(bar, part, out, bad, grid);
        run<3, 2>(bar, part, out, bad, grid);
        run<7, 2>(bar, part, out, bad, grid);
        run<0, 4>(bar, part, out, bad, grid);
        run<3, 4>(bar, part, out, bad, grid);
        run<7, 4>(bar, part, out, bad, grid);
    }
    return 0;
}
