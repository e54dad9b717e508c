// vs_cc.cu -- periodic face-adjacency connected components on the GPU
// (geometry.py:183-222 connected_components; the check in operators.py:224-230).
//
// Lock-free union-find over the cell index (int32: n^dim < 2^31): every
// fluid cell unites with its +e_a periodic neighbours, always hooking the
// larger root under the smaller one (atomicCAS), so the final root of a
// component is its minimum cell index -- its first cell in row-major order.
// Dense ids in first-appearance order are then the rank of each root among
// the roots (an exclusive scan of the root flags), exactly the host
// labelling's ids.
#include <cub/device/device_scan.cuh>

#include "vs_internal.h"

namespace vs {
namespace {

// Reads go to L2 (__ldcg), where the atomicCAS hooks of other SMs land.
__device__ __forceinline__ int cc_find(int *lab, int x) {
    // path halving while roots are still being hooked: a write only ever
    // replaces a parent by one of its ancestors
    int p = __ldcg(lab + x);
    while (p != x) {
        const int gp = __ldcg(lab + p);
        if (gp != p) lab[x] = gp;
        x = p;
        p = gp;
    }
    return x;
}

// read-only root search for after the hooks (no halving writes: a stale
// write could replace a cell's final root pointer by a non-root ancestor)
__device__ __forceinline__ int cc_root(const int *lab, int x) {
    int p = __ldcg(lab + x);
    while (p != x) {
        x = p;
        p = __ldcg(lab + x);
    }
    return x;
}

__device__ __forceinline__ void cc_unite(int *lab, int a, int b) {
    while (true) {
        a = cc_find(lab, a);
        b = cc_find(lab, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicCAS(lab + b, b, a);  // hook root b under the smaller root a
        if (old == b) return;
        b = old;  // b got a parent meanwhile: retry from there
    }
}

__global__ void k_cc_init(const uint8_t *__restrict__ f, int *lab, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
        lab[i] = f[i] ? (int)i : -1;
}

__global__ void k_cc_hook(const uint8_t *__restrict__ f, int *lab, int dim, int n, int64_t N) {
    const int64_t st[3] = {dim == 3 ? (int64_t)n * n : (int64_t)n, dim == 3 ? (int64_t)n : 1, 1};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (!f[i]) continue;
        for (int a = 0; a < dim; ++a) {
            const int64_t s = st[a];
            const int64_t coord = (i / s) % n;
            const int64_t j = coord == n - 1 ? i - (int64_t)(n - 1) * s : i + s;
            if (f[j]) cc_unite(lab, (int)i, (int)j);
        }
    }
}

// point every fluid cell at its root (roots are final after the hook
// kernel; writing an ancestor is safe against concurrent path halving) and
// flag the roots
__global__ void k_cc_flatten(int *lab, int *is_root, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        if (lab[i] < 0) {
            is_root[i] = 0;
            continue;
        }
        const int r = cc_root(lab, (int)i);
        lab[i] = r;
        is_root[i] = r == (int)i;
    }
}

// root index -> dense id (every fluid lab[] is its root after the flatten)
__global__ void k_cc_finish(int *lab, const int *rank, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = lab[i];
        if (r >= 0) lab[i] = rank[r];
    }
}

}  // namespace

// Labels (nullable device output, -1 on solid, dense ids in first row-major
// appearance) and the component count of a device mask; `work` holds 3 N
// ints + scan temp (cc_work_bytes).  Returns the count (host sync).
size_t cc_work_bytes(int64_t N) {
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, (int *)nullptr, (int *)nullptr, (int)N);
    return ((size_t)3 * N * sizeof(int) + temp + 255) & ~(size_t)255;
}

int64_t cc_label_device(const uint8_t *d_fluid, int dim, int n, int *d_labels, void *work, size_t work_bytes,
                        cudaStream_t s) {
    const int64_t N = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    int *lab = reinterpret_cast<int *>(work);
    int *flag = lab + N, *rank = flag + N;
    void *temp = rank + N;
    size_t temp_bytes = work_bytes - (size_t)3 * N * sizeof(int);
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((N + threads - 1) / threads, 148 * 32);
    k_cc_init<<<blocks, threads, 0, s>>>(d_fluid, lab, N);
    k_cc_hook<<<blocks, threads, 0, s>>>(d_fluid, lab, dim, n, N);
    k_cc_flatten<<<blocks, threads, 0, s>>>(lab, flag, N);
    // exclusive scan of the root flags: the dense id of each root
    cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flag, rank, (int)N, s);
    int last[2] = {0, 0};
    cudaMemcpyAsync(last, flag + N - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(last + 1, rank + N - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (d_labels) {
        k_cc_finish<<<blocks, threads, 0, s>>>(lab, rank, N);
        cudaMemcpyAsync(d_labels, lab, N * sizeof(int), cudaMemcpyDeviceToDevice, s);
    }
    cudaStreamSynchronize(s);
    return (int64_t)last[0] + last[1];
}

}  // namespace vs
