// Microbenchmark: how fast can one producer warp per SM stream contiguous
// chunks from HBM into a shared-memory ring (the k_cg1t pattern)?
//   mode 0: 32 lanes issue 16-B cp.async, arrive.noinc on the slot barrier
//   mode 1: lane 0 issues one cp.async.bulk per chunk (mbarrier tx count)
// Consumers (15 warps) wait for each slot, optionally read it (work=1: every
// consumer thread sums its share of the slot from shared memory), release.
// usage: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/rb tools/ring_bench.cu && /tmp/rb
#include <cstdint>
#include <cstdio>
constexpr int TT = 512, NSLOT = 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     smem_u32(b)),
                 "r"(par)
                 : "memory");
}

template <int MODE, int WORK>
__global__ void __launch_bounds__(TT, 1) kern(const double *src, size_t per_block, int chunk, double *out) {
    extern __shared__ __align__(128) uint8_t dyn[];
    double *ring = (double *)dyn;
    uint64_t *bars = (uint64_t *)(dyn + (size_t)NSLOT * chunk * 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int q = 0; q < NSLOT; ++q) {
            mbar_init(bars + q, MODE == 0 ? 32 : 1);
            mbar_init(bars + NSLOT + q, TT / 32 - 1);
        }
    }
    __syncthreads();
    const double *g = src + (size_t)blockIdx.x * per_block;
    const int nch = (int)(per_block / chunk);
    double acc = 0;
    if (warp == 0) {
        for (int f = 0; f < nch; ++f) {
            const int q = f % NSLOT;
            if (f >= NSLOT) mbar_wait(bars + NSLOT + q, ((f - NSLOT) / NSLOT) & 1);
            const double *s = g + (size_t)f * chunk;
            const uint32_t d = smem_u32(ring + (size_t)q * chunk);
            if (MODE == 0) {
                for (int c = lane; c < chunk / 2; c += 32)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16 * c), "l"(s + 2 * c) : "memory");
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bars + q)) : "memory");
            } else if (lane == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + q)),
                             "r"(chunk * 8)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                    "l"(s), "r"(chunk * 8), "r"(smem_u32(bars + q))
                    : "memory");
            }
        }
    } else {
        for (int f = 0; f < nch; ++f) {
            const int q = f % NSLOT;
            mbar_wait(bars + q, (f / NSLOT) & 1);
            if (WORK)
                for (int c = threadIdx.x - 32; c < chunk; c += TT - 32) acc += ring[(size_t)q * chunk + c];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bars + NSLOT + q)) : "memory");
        }
    }
    if (acc == 12345.0) *out = acc;
}

template <int MODE, int WORK>
void run(const double *src, size_t per_block, int chunk, double *out) {
    const size_t smem = (size_t)NSLOT * chunk * 8 + 2 * NSLOT * 8;
    cudaFuncSetAttribute(kern<MODE, WORK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        kern<MODE, WORK><<<148, TT, smem>>>(src, per_block, chunk, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
    }
    const double bytes = 148.0 * per_block * 8;
    printf("mode %d work %d chunk %6d B: %7.1f GB/s (%s)\n", MODE, WORK, chunk * 8, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const size_t per_block = (size_t)1 << 21;  // 16 MB per block, 2.4 GB total
    double *src, *out;
    cudaMalloc(&src, 148 * per_block * 8);
    cudaMemset(src, 0, 148 * per_block * 8);
    cudaMalloc(&out, 8);
    for (int chunk : {512, 1024, 2048, 4096}) {
        run<0, 0>(src, per_block, chunk, out);
        run<1, 0>(src, per_block, chunk, out);
        run<0, 1>(src, per_block, chunk, out);
        run<1, 1>(src, per_block, chunk, out);
    }
    return 0;
}
