// vs_cg_common.cuh -- device pieces shared by the fused PCG kernels
// (vs_cg.cu: k_pcg, k_cg1; vs_cgt.cu: k_cg1t): neighbour ranks from the
// bitmask meta, the bit-exact operator values, grid barrier and
// deterministic grid sums, the block-resident DOF cache.
#pragma once
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "vs_device.cuh"
#include "vs_internal.h"

namespace vs {

// ranks of the 2*DIM neighbours in the reference slot order
// (x+, x-, [y+, y-,] z+, z-)   (operators.py:269-271: d = 0..dim-1, s = +1, -1)
// (nx = extent of the local x axis: n for a whole-domain group, slab planes
// + 2 ghost planes otherwise -- owned DOFs of a slab never wrap in x).
// Presence comes from the record.  The z neighbours lie on the DOF's own
// line, so they are ranks i +- 1 except across the periodic wrap (one meta
// load).  The tangential neighbours share the DOF's bit position, so their
// ranks are base + popc(mask & below(b)) of the word at a fixed offset.
template <int DIM, int OP>
__device__ __forceinline__ void neighbour_ranks(const uint2 *__restrict__ meta, int nw, int n, int nx,
                                                uint64_t rc, uint32_t i, uint32_t (&nr)[2 * DIM]) {
    const int z = rec_z(rc), y = rec_y(rc), x = rec_x(rc);
    const uint32_t b = (uint32_t)z & 31u, below = (1u << b) - 1u;
    const int lineW = (DIM == 3 ? x * n + y : x) * nw;  // word 0 of the DOF's line
    const int w0 = lineW + (z >> 5);
    const int planeW = (DIM == 3 ? n : 1) * nw;           // words per x-plane
    auto tang = [&](int s, int idx) -> uint32_t {
        if (!rec_has_nb<OP>(rc, s)) return ABSENT;
        const uint2 m = __ldg(meta + idx);
        return m.y + (uint32_t)__popc(m.x & below);
    };
    nr[0] = tang(0, w0 + ((x == nx - 1) ? -(nx - 1) * planeW : planeW));
    nr[1] = tang(1, w0 + ((x == 0) ? (nx - 1) * planeW : -planeW));
    if (DIM == 3) {
        nr[2] = tang(2, w0 + ((y == n - 1) ? -(n - 1) * nw : nw));
        nr[3] = tang(3, w0 + ((y == 0) ? (n - 1) * nw : -nw));
    }
    const bool hp = rec_has_nb<OP>(rc, 2 * DIM - 2), hm = rec_has_nb<OP>(rc, 2 * DIM - 1);
    const bool top = (z == n - 1), bot = (z == 0);
    uint32_t rw = 0;
    if ((top && hp) || (bot && hm)) {  // periodic wrap: cell 0 (from the top) or n-1 (from the bottom)
        const int zz = top ? 0 : n - 1;
        const uint2 m = __ldg(meta + lineW + (zz >> 5));
        rw = m.y + (uint32_t)__popc(m.x & ((1u << (zz & 31)) - 1u));
    }
    nr[2 * DIM - 2] = hp ? (top ? rw : i + 1) : ABSENT;
    nr[2 * DIM - 1] = hm ? (bot ? rw : i - 1) : ABSENT;
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
        // branch-free: an absent face has code 0 and invA[0] = 0.0, so its
        // weight is (finite) * 0.0 = +-0.0 -- the reference's padded 0.0 up to
        // the sign of zero (neighbour values of absent faces are finite: the
        // gather is clamped to the DOF itself)
        double out = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            // slot 2a = +e_a neighbour (out face), 2a+1 = -e_a neighbour (in face)
            const double wi = __dmul_rn(__dmul_rn(__dsub_rn(vi, vn[2 * a + 1]), inv_h), T.invA[rec_pin(rc, a)]);
            const double wo = __dmul_rn(__dmul_rn(__dsub_rn(vn[2 * a], vi), inv_h), T.invA[rec_pout(rc, a)]);
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
__device__ __forceinline__ const uint2 *family_meta(const CgGroup &G, uint64_t rc) {
    const uint2 *m;
    if (OP == 1) {
        m = G.meta[0];
    } else {
        const int c = rec_comp(rc);
        m = c == 0 ? G.meta[0] : (c == 1 ? G.meta[1] : G.meta[2]);
    }
    __builtin_assume(__isGlobal(m));
    return m;
}

// z of an owned DOF that lies in the first / last owned x-plane of its
// slab is also stored into the neighbour slab's ghost plane (peer memory on
// a multi-GPU run; another group's array when ranks are emulated).
__device__ __forceinline__ void halo_store(const CgGroup &G, int fam, uint32_t i, double zi) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const uint32_t b = G.sbeg[s][fam];
        if (i >= b && i < G.send[s][fam]) {
            double *dst = G.zpeer[s];
            __builtin_assume(__isGlobal(dst));
            dst[G.sdst[s][fam] + (i - b)] = zi;
        }
    }
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ------------------------------------------------------------- grid barrier
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// (Tried: flag-in-word slots polled by every block, with no arrival
// counter -- slower on B200: 148 blocks polling every slot costs more than
// one counter barrier plus one read of the partials; tools/gridsum_ll.cu,
// C1 S_hat 7.8 -> 9.5 us/it.  ORDER is accepted for that interface; the
// counter barrier always orders.)
// bar = monotonic arrival counter shared by every block of every rank; it is
// never reset.  Each launch starts from *P.bar_base (the previous launch's
// final target, written back by its block 0 -- identical on every rank, since
// all ranks run the same barrier sequence) and each barrier adds the number
// of participating blocks of all ranks.  One red.release per block, then
// thread 0 polls.
// Polling uses relaxed loads: an acquire load per poll makes ptxas emit an
// L1 invalidation (CCTL.IVALL) per poll.  Once the target is seen, one
// acquire re-read of the counter synchronises with every block's release
// (the reds form one release sequence); it is 0.13 us cheaper than a
// fence.acq_rel (B200, 148 x 1024 threads: 1.17 vs 1.30 us per barrier;
// the unfenced floor is 0.84 us -- tools/gridsync_variants.cu).
// xflag (multi-GPU runs only): this rank's "a peer never arrived" flag, in
// device memory.  A cross-GPU barrier that waits longer than
// xtimeout_ns sets it and gives up; every later barrier of the rank returns
// at once, the fused loops stop at their next iteration (status 4) and the
// host raises VS_ECUDA after its next synchronisation instead of hanging.
// Hierarchical form for multi-rank runs (P.hier; only kernels instantiated with MR = true contain
// it, so the single-GPU kernels' code is untouched -- at 64 registers they are sensitive to any
// change around their hot loops: an `if (P.hier)` in the common path cost k_pcgx 3 %).  The blocks
// of a rank arrive on the rank's own counter (atom.inc, wraps at bpg: no base to carry); the last
// local arriver is the rank's leader for this barrier: it alone arrives on the shared counter --
// which then counts RANKS, R per barrier, the unit k_xbar uses -- polls it, and publishes the
// reached target in the rank's local release word, which the rank's other blocks poll.  NVLink
// carries R arrivals and R pollers per barrier instead of 148 R of each; every other poll stays in
// local memory.  Ordering: the local arrivals are acq_rel RMWs on one word (the leader's acquires
// every earlier block's release), the leader's arrival on the shared counter is a release at the
// run's scope (cumulative over what it acquired), its final acquire + local release + the blocks'
// local acquire carry the other ranks' stores to every block.
__device__ __forceinline__ void grid_barrier_hier(const CgParams &P, unsigned &target) {
    __syncthreads();
    target += (unsigned)P.nranks_bar;
    if (threadIdx.x == 0) {
        unsigned *lb = P.lbar[P.part_self + (int)(blockIdx.x / P.bpg)];
        __builtin_assume(__isGlobal(lb));
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(old) : "l"(lb), "r"((unsigned)P.bpg - 1u) : "memory");
        if (old == (unsigned)P.bpg - 1u) {  // this rank's last arrival
            unsigned v;
            if (P.xgpu) {
                asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(P.bar) : "memory");
                unsigned long long t0 = 0;
                unsigned spins = 0;
                do {
                    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(P.bar) : "memory");
                    if (P.xflag && (++spins & 1023u) == 0) {  // look at the clock every 1024 polls
                        unsigned long long now;
                        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
                        if (!t0) t0 = now;
                        if (*P.xflag) break;
                        if (P.xtimeout_ns && now - t0 > P.xtimeout_ns) {
                            *P.xflag = 1;
                            break;
                        }
                    }
                } while ((int)(v - target) < 0);
                asm volatile("{\n\t.reg .u32 t;\n\tld.acquire.sys.global.u32 t, [%0];\n\t}" ::"l"(P.bar) : "memory");
            } else {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bar) : "memory");
                while ((int)(ld_relaxed(P.bar) - target) < 0) {
                }
                asm volatile("{\n\t.reg .u32 t;\n\tld.acquire.gpu.global.u32 t, [%0];\n\t}" ::"l"(P.bar) : "memory");
            }
            st_release(lb + 1, target);  // (also after a timeout: the rank's blocks must not hang)
        } else {
            unsigned spins = 0;
            while ((int)(ld_relaxed(lb + 1) - target) < 0) {
                if (P.xgpu && P.xflag && (++spins & 4095u) == 0 && *P.xflag) break;
            }
            asm volatile("{\n\t.reg .u32 t;\n\tld.acquire.gpu.global.u32 t, [%0];\n\t}" ::"l"(lb + 1) : "memory");
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &target, unsigned total_blocks,
                                             bool xgpu = false, volatile int *xflag = nullptr,
                                             unsigned long long xtimeout_ns = 0) {
    __syncthreads();
    target += total_blocks;
    if (threadIdx.x == 0) {
        if (xgpu) {
            // ranks on different GPUs (peer memory over NVLink): system scope,
            // so the release orders this GPU's peer stores (ghost planes,
            // partials) before the arrival, and the acquire makes the other
            // GPUs' stores visible here
            asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            unsigned v;
            unsigned long long t0 = 0;
            unsigned spins = 0;
            do {
                asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
                if (xflag && (++spins & 1023u) == 0) {  // look at the clock every 1024 polls
                    unsigned long long now;
                    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
                    if (!t0) t0 = now;
                    if (*xflag) break;
                    if (xtimeout_ns && now - t0 > xtimeout_ns) {
                        *xflag = 1;
                        break;
                    }
                }
            } while ((int)(v - target) < 0);
            asm volatile("{\n\t.reg .u32 t;\n\tld.acquire.sys.global.u32 t, [%0];\n\t}" ::"l"(bar) : "memory");
        } else {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
            while ((int)(ld_relaxed(bar) - target) < 0) {
            }
            asm volatile("{\n\t.reg .u32 t;\n\tld.acquire.gpu.global.u32 t, [%0];\n\t}" ::"l"(bar) : "memory");
        }
    }
    __syncthreads();
}

// Warp 0 combines the per-warp values s_warp[w][k] (w < CG_THREADS/32) with
// one xor-butterfly carrying all K values at once; the result lands in
// every lane of warp 0.  Fixed shape -> bitwise identical in every block.
template <int K, int NT = CG_THREADS>
__device__ __forceinline__ void warp0_combine(const double (*s_warp)[5], double (&t)[K]) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = lane < NW ? s_warp[lane][k] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __shfl_xor_sync(~0u, t[k], o));
    }
}

template <int K>
__device__ __forceinline__ void warp_tree(double (&t)[K]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __shfl_xor_sync(~0u, t[k], o));
    }
}

// Deterministic grid-wide sum of K values over every block of every rank.
// Block g (global index block_base + blockIdx.x) writes its K sums into slot
// g of partial set `set` of EVERY rank's partial buffer (peer stores on a
// multi-GPU run; one buffer when the ranks are groups of one launch).  After
// the barrier each block reads all blocks' sums from its own buffer in one
// parallel round trip and reduces them in the same fixed tree, so every
// block of every rank obtains bitwise-identical totals.
template <int K, bool ORDER, int NT = CG_THREADS, bool MR = false>
__device__ __forceinline__ void grid_sum_shfl(double (&v)[K], int set, const CgParams &P, unsigned &target,
                                              double (*s_warp)[5], double *s_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int TB = P.total_blocks;
    warp_tree<K>(v);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) s_warp[warp][k] = v[k];
    }
    __syncthreads();
    if (warp == 0) {
        double t[K];
        warp0_combine<K, NT>(s_warp, t);
        if (lane < P.npart) {  // lane p stores to rank p's buffer
            double *dst = P.part_peer[lane] + (size_t)set * 8 * TB + (size_t)(P.block_base + blockIdx.x) * 8;
            __builtin_assume(__isGlobal(dst));
#pragma unroll
            for (int k = 0; k < K; ++k) dst[k] = t[k];
        }
    }
    if constexpr (MR) {
        if (P.hier)
            grid_barrier_hier(P, target);
        else
            grid_barrier(P.bar, target, TB, P.xgpu, P.xflag, P.xtimeout_ns);
    } else {
        grid_barrier(P.bar, target, TB, P.xgpu, P.xflag, P.xtimeout_ns);
    }  // starts with __syncthreads (s_warp reuse is safe)
    // own buffer: one per rank (per group when ranks are emulated as groups)
    const double *part = (P.npart > 1 ? P.part_peer[P.part_self + (int)(blockIdx.x / P.bpg)] : P.part) +
                         (size_t)set * 8 * TB;
    __builtin_assume(__isGlobal(part));
    double t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = 0.0;
    for (int b = threadIdx.x; b < TB; b += NT) {
#pragma unroll
        for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __ldcg(part + b * 8 + k));
    }
    warp_tree<K>(t);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) s_warp[warp][k] = t[k];
    }
    __syncthreads();
    if (warp == 0) {
        warp0_combine<K, NT>(s_warp, t);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) s_tot[k] = t[k];
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

// The per-iteration form (K <= 8; s_val holds K rows).  Block stage through shared memory:
// every thread stores its K values, then warp k alone reduces component k
// -- lane i sums threads i, i+32, ..., i+992 in a fixed pairwise tree, one
// xor butterfly combines the lanes.  The shuffle tree over all 32 warps
// cost 32 x K x 10 SHFL per block and was SHFL-throughput bound (B200,
// tools/gridsum_variants.cu: K=4 3.93 -> 2.77 us, K=2 2.95 -> 2.52 us per
// grid sum).  After the barrier warp k again reduces component k over the
// blocks (lane i: blocks i, i+32, ... in order; loads issued 8 at a time).
template <int K, bool ORDER, int NT = CG_THREADS, bool MR = false>
__device__ __forceinline__ void grid_sum(double (&v)[K], int set, const CgParams &P, unsigned &target,
                                         double (*s_val)[NT], double *s_tot) {
    static_assert(K >= 1 && K <= 8, "grid_sum stages at most 8 components");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int TB = P.total_blocks;
#pragma unroll
    for (int k = 0; k < K; ++k) s_val[k][threadIdx.x] = v[k];
    __syncthreads();
    if (warp < K) {
        // chunks of 8 (pairwise within a chunk), then the chunk sums pairwise
        constexpr int NC = NT / 256;
        static_assert(NC == 2 || NC == 3 || NC == 4, "grid_sum block stage: 512, 768 or 1024 threads");
        double c[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            double x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = s_val[warp][lane + 32 * (8 * q + j)];
#pragma unroll
            for (int w = 1; w < 8; w *= 2) {
#pragma unroll
                for (int j = 0; j < 8; j += 2 * w) x[j] = __dadd_rn(x[j], x[j + w]);
            }
            c[q] = x[0];
        }
        double t[1];
        if constexpr (NC == 4)
            t[0] = __dadd_rn(__dadd_rn(c[0], c[1]), __dadd_rn(c[2], c[3]));
        else if constexpr (NC == 3)
            t[0] = __dadd_rn(__dadd_rn(c[0], c[1]), c[2]);
        else
            t[0] = __dadd_rn(c[0], c[1]);
        warp_tree<1>(t);
        if (lane < P.npart) {  // lane p stores to rank p's buffer
            double *dst =
                P.part_peer[lane] + (size_t)set * 8 * TB + (size_t)(P.block_base + blockIdx.x) * 8 + warp;
            __builtin_assume(__isGlobal(dst));
            *dst = t[0];
        }
    }
    if constexpr (MR) {
        if (P.hier)
            grid_barrier_hier(P, target);
        else
            grid_barrier(P.bar, target, TB, P.xgpu, P.xflag, P.xtimeout_ns);
    } else {
        grid_barrier(P.bar, target, TB, P.xgpu, P.xflag, P.xtimeout_ns);
    }  // starts with __syncthreads (s_val reuse is safe)
    if (warp < K) {
        // own buffer: one per rank (per group when ranks are emulated as groups)
        const double *part = (P.npart > 1 ? P.part_peer[P.part_self + (int)(blockIdx.x / P.bpg)] : P.part) +
                             (size_t)set * 8 * TB + warp;
        __builtin_assume(__isGlobal(part));
        double t[1] = {0.0};
        for (int b0 = 0; b0 < TB; b0 += 32 * 8) {
            double w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int b = b0 + lane + 32 * j;
                w[j] = b < TB ? __ldcg(part + (size_t)b * 8) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) t[0] = __dadd_rn(t[0], w[j]);
        }
        warp_tree<1>(t);
        if (lane == 0) s_tot[warp] = t[0];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = s_tot[k];
}

// ------------------------------------------------------------------ kernel
// Block-resident DOF cache: a persistent block visits the same DOFs every
// iteration (i = tid + k*stride), so slot k of thread t keeps, in shared
// memory, the DOF's record (TIER >= 1) and its 2*DIM neighbour ranks
// (TIER 2) for the first `kc` slots.  Cached DOFs skip the record read
// (8 B/DOF/pass of DRAM) and, at TIER 2, the whole bitmask rank lookup.
template <int DIM, int OP, int TIER, int NT = CG_THREADS>
struct DofCache {
    static constexpr int NS = 2 * DIM;
    uint64_t *rec;
    uint32_t *rank;
    __device__ DofCache(uint8_t *base, uint32_t kc) {
        rec = reinterpret_cast<uint64_t *>(base);
        rank = reinterpret_cast<uint32_t *>(base + (size_t)kc * NT * 8);
    }
    __device__ __forceinline__ void put(uint32_t k, uint64_t rc, const uint32_t (&nr)[NS]) {
        rec[k * NT + threadIdx.x] = rc;
        if (TIER == 2) {
#pragma unroll
            for (int s = 0; s < NS; ++s) rank[(k * NS + s) * NT + threadIdx.x] = nr[s];
        }
    }
};

// TIER 3: records as TIER 1, neighbour ranks precomputed in global memory
// (G.nbr, [2*DIM][m_own] uint32, streamed coalesced): the rank lookup is no
// longer a dependent bitmask load between the record and the gathers.
template <int DIM, int OP, int TIER, int NT = CG_THREADS>
__device__ __forceinline__ void fetch_dof(const CgParams &P, const CgGroup &G, const DofCache<DIM, OP, TIER, NT> &C,
                                          uint32_t k, uint32_t kc, uint32_t i, uint64_t &rc,
                                          uint32_t (&nr)[2 * DIM]) {
    if (TIER == 3) {
        const uint32_t *nb = G.nbr;
        __builtin_assume(__isGlobal(nb));
#pragma unroll
        for (int s = 0; s < 2 * DIM; ++s) nr[s] = __ldcs(nb + (size_t)s * G.m_own + i);
        if (k < kc) {
            rc = C.rec[k * NT + threadIdx.x];
        } else {
            const uint64_t *rec = G.rec;
            __builtin_assume(__isGlobal(rec));
            rc = rec[i];
        }
        return;
    }
    if (TIER == 4) {
        // packed deltas: one 8-B and one 4-B coalesced load, issued before the
        // record is needed; INT_MIN in x.x = wrap / out-of-range -> bitmask lookup
        const int2 *xd = reinterpret_cast<const int2 *>(G.nbr);
        __builtin_assume(__isGlobal(xd));
        const int2 dx = __ldcs(xd + i);
        short2 dy = make_short2(0, 0);
        if (DIM == 3) {
            const short2 *yd = reinterpret_cast<const short2 *>(G.nbr + 2 * (size_t)G.m_own);
            __builtin_assume(__isGlobal(yd));
            dy = __ldcs(yd + i);
        }
        if (k < kc) {
            rc = C.rec[k * NT + threadIdx.x];
        } else {
            const uint64_t *rec = G.rec;
            __builtin_assume(__isGlobal(rec));
            rc = rec[i];
        }
        if (dx.x == INT_MIN) {
            neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
            return;
        }
        nr[0] = rec_has_nb<OP>(rc, 0) ? i + (uint32_t)dx.x : ABSENT;
        nr[1] = rec_has_nb<OP>(rc, 1) ? i + (uint32_t)dx.y : ABSENT;
        if (DIM == 3) {
            nr[2] = rec_has_nb<OP>(rc, 2) ? i + (uint32_t)(int)dy.x : ABSENT;
            nr[3] = rec_has_nb<OP>(rc, 3) ? i + (uint32_t)(int)dy.y : ABSENT;
        }
        nr[2 * DIM - 2] = rec_has_nb<OP>(rc, 2 * DIM - 2) ? i + 1 : ABSENT;
        nr[2 * DIM - 1] = rec_has_nb<OP>(rc, 2 * DIM - 1) ? i - 1 : ABSENT;
        return;
    }
    if (k < kc) {
        rc = C.rec[k * NT + threadIdx.x];
        if (TIER == 2) {
#pragma unroll
            for (int s = 0; s < 2 * DIM; ++s) nr[s] = C.rank[(k * 2 * DIM + s) * NT + threadIdx.x];
            return;
        }
    } else {
        const uint64_t *rec = G.rec;
        __builtin_assume(__isGlobal(rec));
        rc = rec[i];
    }
    neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
}

// k_cg1 grid-sum staging in dynamic smem (KS rows of CG_THREADS doubles)
__host__ __device__ constexpr size_t cg1_stage_bytes(int op, int nt = CG_THREADS) { return (size_t)(op == 1 ? 6 : 3) * nt * 8; }

template <int OP>
__device__ __forceinline__ void inv_diag(uint64_t rc, const Tabs &T, const double2 *__restrict__ sdg, double &inv,
                                         double &dg) {
    if (OP == 0) {
        inv = T.inv[rec_vcode(rc)];
        dg = T.diag[rec_vcode(rc)];
    } else {
        const double2 t = __ldg(sdg + rec_pkey(rc));
        inv = t.x;
        dg = t.y;
    }
}

}  // namespace vs
