// vs_cg.cu -- K8: the fused persistent PCG of the inner solves (krylov.py:76-182).
//
// One cooperative launch runs a whole inner solve.  Per CG iteration:
//   P1  d = (z - mu) + beta d_old        (z stored by P2, mean-projected for S_hat)
//       q = op(d), neighbour d recomputed from z/d_old -> no extra pass
//       partial d.q                                              -> barrier 1
//   P2  q = op(d) from the stored d; x -= alpha d; r -= alpha q;
//       z = M^-1 r (stored); partials r.z, z.z, r.r, sum z, sum r -> barrier 2
// Scalars live in registers of every block: each block reduces the same
// per-block partials in the same fixed order, so alpha/beta/mu and the
// convergence decision are bitwise identical everywhere (deterministic for
// a given grid).  The mean projection z - mean(z) (krylov.py:152-153) is
// folded into the sums: r.(z-mu) = r.z - mu sum r, |z-mu|^2 = z.z - mu sum z.
// Every elementwise update keeps the reference's operation order
// (x -= alpha*d is dsub(x, dmul(alpha, d)), d = z + beta*d is
// dadd(z, dmul(beta, d))) with explicit round-to-nearest intrinsics.
//
// DRAM bytes per DOF per iteration (8 B each): P1 reads z, d_old, record and
// writes d; P2 reads d, x, r, record and writes x, r, z  -> 88 B (plus
// L2-resident bitmask words for the neighbour ranks).
#include "vs_device.cuh"
#include "vs_internal.h"

namespace vs {

__device__ __forceinline__ uint32_t rank_of(const uint2 *__restrict__ meta, int nw, int L, int z) {
    const uint2 m = __ldg(meta + (L * nw + (z >> 5)));
    const uint32_t b = (uint32_t)z & 31u;
    const uint32_t rk = m.y + (uint32_t)__popc(m.x & ((1u << b) - 1u));
    return ((m.x >> b) & 1u) ? rk : ABSENT;
}

// ranks of the 2*DIM neighbours in the reference slot order
// (x+, x-, [y+, y-,] z+, z-)   (operators.py:269-271: d = 0..dim-1, s = +1, -1)
template <int DIM>
__device__ __forceinline__ void neighbour_ranks(const uint2 *__restrict__ meta, int nw, int n, uint64_t rc,
                                                uint32_t (&nr)[2 * DIM]) {
    const int z = rec_z(rc), y = rec_y(rc), x = rec_x(rc);
    const int sx = DIM == 3 ? n : 1;
    const int L = DIM == 3 ? x * n + y : x;
    const int Lxp = (x == n - 1) ? L - (n - 1) * sx : L + sx;
    const int Lxm = (x == 0) ? L + (n - 1) * sx : L - sx;
    nr[0] = rank_of(meta, nw, Lxp, z);
    nr[1] = rank_of(meta, nw, Lxm, z);
    if (DIM == 3) {
        const int Lyp = (y == n - 1) ? L - (n - 1) : L + 1;
        const int Lym = (y == 0) ? L + (n - 1) : L - 1;
        nr[2] = rank_of(meta, nw, Lyp, z);
        nr[3] = rank_of(meta, nw, Lym, z);
    }
    const int zp = (z == n - 1) ? 0 : z + 1, zm = (z == 0) ? n - 1 : z - 1;
    nr[2 * DIM - 2] = rank_of(meta, nw, L, zp);
    nr[2 * DIM - 1] = rank_of(meta, nw, L, zm);
}

struct Tabs {
    const double *diag;  // velocity diag by raw code (smem)
    const double *inv;   // velocity 1/diag by raw code (smem)
    const double *invA;  // face weight by encoded code (smem)
    const double *__restrict__ invS;  // S_hat Jacobi by 18-bit key (global)
};

// op(v) at one DOF; v_nb[] = values at the neighbour slots (0.0 if absent).
// A: operators.py:131-135.  S_hat: schur.py:234-240 (see vs_device.cuh).
template <int DIM, int OP>
__device__ __forceinline__ double op_value(uint64_t rc, double vi, const double (&vn)[2 * DIM], const Tabs &T,
                                           double inv_h, double inv_h2) {
    if (OP == 0) {
        double acc = vn[0];
#pragma unroll
        for (int s = 1; s < 2 * DIM; ++s) acc = __dadd_rn(acc, vn[s]);
        return __dsub_rn(__dmul_rn(T.diag[rec_vcode(rc)], vi), __dmul_rn(inv_h2, acc));
    } else {
        double out = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            // slot 2a = +e_a neighbour (out face), 2a+1 = -e_a neighbour (in face)
            const int ci = rec_pin(rc, a), co = rec_pout(rc, a);
            const double wi = ci ? __dmul_rn(__dmul_rn(__dsub_rn(vi, vn[2 * a + 1]), inv_h), T.invA[ci]) : 0.0;
            const double wo = co ? __dmul_rn(__dmul_rn(__dsub_rn(vn[2 * a], vi), inv_h), T.invA[co]) : 0.0;
            out = __dadd_rn(out, __dsub_rn(wi, wo));
        }
        return __dmul_rn(out, inv_h);
    }
}

template <int OP>
__device__ __forceinline__ double jacobi_inv(uint64_t rc, const Tabs &T) {
    return OP == 0 ? T.inv[rec_vcode(rc)] : __ldg(T.invS + rec_pkey(rc));
}

template <int OP>
__device__ __forceinline__ const uint2 *family_meta(const CgParams &P, uint64_t rc) {
    if (OP == 1) return P.g.pmeta;
    const int c = rec_comp(rc);
    return c == 0 ? P.g.vmeta[0] : (c == 1 ? P.g.vmeta[1] : P.g.vmeta[2]);
}

// ------------------------------------------------------------- grid barrier
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// bar[0] = arrival count, bar[1] = generation.  All blocks co-resident
// (cooperative launch).  The last arriver resets the count and bumps the
// generation; everyone else polls the generation with acquire loads.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned old = atomicAdd(bar, 1u);
        if (old == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            st_release(bar + 1, gen + 1);
        } else {
            while (ld_acquire(bar + 1) == gen) {
            }
        }
    }
    ++gen;
    __syncthreads();
}

template <int K>
__device__ __forceinline__ void grid_sum(double (&v)[K], double *part, unsigned *bar, unsigned &gen,
                                         double (*s_warp)[5], double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(~0u, x, o));
        if (lane == 0) s_warp[warp][k] = x;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < CG_THREADS / 32; ++w) s = __dadd_rn(s, s_warp[w][threadIdx.x]);
        part[threadIdx.x * gridDim.x + blockIdx.x] = s;
    }
    grid_barrier(bar, gen);
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int j = lane; j < (int)gridDim.x; j += 32) s = __dadd_rn(s, __ldcg(part + k * gridDim.x + j));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(~0u, s, o));
            if (lane == 0) s_tot[k] = s;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
    __syncthreads();
}

// ------------------------------------------------------------------ kernel
template <int DIM, int OP>
__global__ void __launch_bounds__(CG_THREADS, 2) k_pcg(const CgParams P) {
    constexpr bool PROJ = (OP == 1);
    constexpr int NS = 2 * DIM;
    __shared__ double s_tab[40];
    __shared__ double s_warp[CG_THREADS / 32][5];
    __shared__ double s_tot[5];
    if (threadIdx.x < 16) {
        s_tab[threadIdx.x] = P.diag_code[threadIdx.x];
        s_tab[16 + threadIdx.x] = P.inv_code[threadIdx.x];
        if (threadIdx.x < 8) s_tab[32 + threadIdx.x] = P.invA_enc[threadIdx.x];
    }
    unsigned gen = ld_acquire(P.bar + 1);
    __syncthreads();
    const Tabs T{s_tab, s_tab + 16, s_tab + 32, P.invS};
    const int n = P.g.n, nw = P.g.nw;
    const uint32_t m = (uint32_t)P.m;
    const uint32_t tid = blockIdx.x * CG_THREADS + threadIdx.x;
    const uint32_t stride = gridDim.x * CG_THREADS;
    const uint64_t *__restrict__ rec = P.rec;
    double *x = P.x, *r = P.r, *z = P.z;
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;

    // ---- setup (krylov.py:102-119): project rhs; r = op(x0) - rhs; z = M^-1 r
    double mu_rhs = 0.0, mu = 0.0, rz = 0.0, rp0 = 0.0, ru0 = 0.0;
    if (PROJ) {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], P.rhs[i]);
        grid_sum<1>(v, P.part, P.bar, gen, s_warp, s_tot);
        mu_rhs = v[0] / (double)P.m;
    }
    {
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double *x0 = P.x0;
        for (uint32_t i = tid; i < m; i += stride) {
            const uint64_t rc = rec[i];
            double ax = 0.0, xi = 0.0;
            if (x0) {
                xi = x0[i];
                uint32_t nr[NS];
                neighbour_ranks<DIM>(family_meta<OP>(P, rc), nw, n, rc, nr);
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) vn[s] = nr[s] != ABSENT ? x0[nr[s]] : 0.0;
                ax = op_value<DIM, OP>(rc, xi, vn, T, inv_h, inv_h2);
                if (x0 != x) x[i] = xi;
            } else {
                x[i] = 0.0;
            }
            const double b = PROJ ? __dsub_rn(P.rhs[i], mu_rhs) : P.rhs[i];
            const double ri = __dsub_rn(ax, b);
            const double zi = __dmul_rn(ri, jacobi_inv<OP>(rc, T));
            r[i] = ri;
            z[i] = zi;
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
            v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
            v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
            v[3] = __dadd_rn(v[3], zi);
            v[4] = __dadd_rn(v[4], ri);
        }
        grid_sum<5>(v, P.part + 8 * gridDim.x, P.bar, gen, s_warp, s_tot);
        if (PROJ) {
            mu = v[3] / (double)P.m;
            v[0] = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
            v[1] = __dsub_rn(v[1], __dmul_rn(mu, v[3]));
        }
        rz = v[0];
        rp0 = sqrt(v[1]);
        ru0 = sqrt(v[2]);
    }
    const double ref = P.norm_prec ? rp0 : ru0;
    double beta = 0.0, rp_last = rp0, ru_last = ru0, sval = 0.0;
    int status = 0;
    int64_t sat = 0, its = 0;
    bool conv = (ref == 0.0);
    double *dold = P.d0, *dnew = P.d1;
    if (!conv) {
        for (int64_t k = 0; k < P.max_iter; ++k) {
            if (rz < 0.0) { status = 1; sval = rz; sat = k; break; }
            if (rz == 0.0) { conv = true; break; }
            const bool first = (k == 0);
            // ---- P1: d = z - mu + beta d_old, q = op(d), d.q
            double v1[1] = {0.0};
            uint64_t rc_next = tid < m ? rec[tid] : 0;
            for (uint32_t i = tid; i < m; i += stride) {
                const uint64_t rc = rc_next;
                if (i + stride < m) rc_next = rec[i + stride];
                uint32_t nr[NS];
                neighbour_ranks<DIM>(family_meta<OP>(P, rc), nw, n, rc, nr);
                double zc = z[i];
                if (PROJ) zc = __dsub_rn(zc, mu);
                const double di = first ? zc : __dadd_rn(zc, __dmul_rn(beta, dold[i]));
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    double zj = 0.0, dj = 0.0;
                    if (nr[s] != ABSENT) {
                        zj = z[nr[s]];
                        if (!first) dj = dold[nr[s]];
                    }
                    if (PROJ) zj = __dsub_rn(zj, mu);
                    vn[s] = nr[s] == ABSENT ? 0.0 : (first ? zj : __dadd_rn(zj, __dmul_rn(beta, dj)));
                }
                const double qi = op_value<DIM, OP>(rc, di, vn, T, inv_h, inv_h2);
                dnew[i] = di;
                v1[0] = __dadd_rn(v1[0], __dmul_rn(di, qi));
            }
            grid_sum<1>(v1, P.part + 16 * gridDim.x, P.bar, gen, s_warp, s_tot);
            const double dq = v1[0];
            if (dq <= 0.0) { status = 2; sval = dq; sat = k; break; }
            const double alpha = rz / dq;
            // ---- P2: q = op(d); x -= alpha d; r -= alpha q; z = M^-1 r; sums
            double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
            rc_next = tid < m ? rec[tid] : 0;
            for (uint32_t i = tid; i < m; i += stride) {
                const uint64_t rc = rc_next;
                if (i + stride < m) rc_next = rec[i + stride];
                uint32_t nr[NS];
                neighbour_ranks<DIM>(family_meta<OP>(P, rc), nw, n, rc, nr);
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) vn[s] = nr[s] != ABSENT ? dnew[nr[s]] : 0.0;
                const double di = dnew[i];
                const double qi = op_value<DIM, OP>(rc, di, vn, T, inv_h, inv_h2);
                const double xi = __dsub_rn(x[i], __dmul_rn(alpha, di));
                const double ri = __dsub_rn(r[i], __dmul_rn(alpha, qi));
                const double zi = __dmul_rn(ri, jacobi_inv<OP>(rc, T));
                x[i] = xi;
                r[i] = ri;
                z[i] = zi;
                v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
                v[3] = __dadd_rn(v[3], zi);
                v[4] = __dadd_rn(v[4], ri);
            }
            grid_sum<5>(v, P.part + 24 * gridDim.x, P.bar, gen, s_warp, s_tot);
            if (PROJ) {
                mu = v[3] / (double)P.m;
                v[0] = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
                v[1] = __dsub_rn(v[1], __dmul_rn(mu, v[3]));
            }
            const double rz_new = v[0];
            beta = rz_new / rz;
            rz = rz_new;
            const double nz = sqrt(v[1]), nrr = sqrt(v[2]);
            if (!(isfinite(nz) && isfinite(nrr))) { status = 3; sat = k + 1; break; }
            its = k + 1;
            rp_last = nz;
            ru_last = nrr;
            double *t = dold; dold = dnew; dnew = t;
            if ((P.norm_prec ? nz : nrr) / ref < P.tol) { conv = true; break; }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        CgOut *o = P.out;
        o->iterations = its;
        o->converged = conv ? 1 : 0;
        o->status = status;
        o->value = sval;
        o->at_iter = sat;
        o->res_prec0 = rp0;
        o->res_unprec0 = ru0;
        o->res_prec_last = rp_last;
        o->res_unprec_last = ru_last;
    }
}

static const void *pcg_fn(int dim, int op) {
    if (dim == 3) return op == 0 ? (const void *)k_pcg<3, 0> : (const void *)k_pcg<3, 1>;
    return op == 0 ? (const void *)k_pcg<2, 0> : (const void *)k_pcg<2, 1>;
}

int pcg_max_grid(int dim, int op, int device) {
    int per_sm = 0, nsm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_fn(dim, op), CG_THREADS, 0);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    return per_sm * nsm;
}

cudaError_t launch_pcg(int dim, int op, CgParams &P, int grid, cudaStream_t s) {
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel(pcg_fn(dim, op), dim3(grid), dim3(CG_THREADS), args, 0, s);
}

}  // namespace vs
