// vs_cgx.cu -- k_pcgx: the fused inner PCG (krylov.py:76-182) with the search
// direction taken out of the stencil pass and the solution update batched --
// the HBM-regime kernel with the fewest bytes per DOF-iteration.
//
// k_pcgm (vs_cgm.cu, qrec form) moves 98 B per DOF and CG iteration: P1 reads
// z, d_old, s_old and the descriptor and writes d and s; P2 reads d, s, x, z
// and writes x, z.  It streams those bytes at 84-91 % of the copy peak, so
// the bytes are what is left to cut.  Two observations remove 20-26 of them:
//
//  * d'q does not need d.  With delta = z'.A z' (z' = z - mu) the CG identity
//        d'A d = delta - beta gamma / alpha_prev         (gamma = r.z')
//    gives alpha from sums over z alone -- the recurrence k_cg1 (vs_cg.cu)
//    already uses, parity-pinned at C1.  The stencil pass P1 then reads
//    z, s_old and the descriptor and writes s = M A z + beta s_old: 32 B,
//    no d_old read, no d write.
//  * d and x are a slave recurrence: d_k = z'_k + beta_k d_{k-1},
//    x -= alpha_k d_k need only z_k and scalars known after P1's sum, and
//    nothing else in the iteration reads them.  So z is kept in a ring of M
//    buffers (P2 of iteration k reads z_k from buffer k mod M and writes
//    z_{k+1} to buffer (k+1) mod M), and d, x are brought up to date only
//    every M-th iteration ("heavy" P2: reads the M-1 older z, d, x; applies
//    the M updates in order, in registers, with the recorded
//    (mu, beta, alpha) of each; writes d, x).  The operations and their order
//    are exactly those of an every-iteration update, so x is bitwise the
//    same for every M.  The other P2s ("light") read z, s and the 2-B code
//    index and write z: 26 B.  At the end of the solve the pending updates
//    are applied from the ring.
//
//    bytes per DOF-iteration: 32 (P1) + 26 (P2) + (32 + 8 (M-1)) / M
//      M = 1: 90    M = 2: 78    M = 3: 74    M = 4: 72        (k_pcgm: 98)
//
// The M-scaled recurrences use fused multiply-adds (this form is not bitwise
// the reference's operation order anyway -- k_pcg keeps that role); parity is
// the solve bar: p, u, k within 1e-8, iteration counts within 2 %.
// Barrier, deterministic grid sums, slab groups and ghost planes are
// vs_cg_common.cuh's; the ghost stores go to the peers' ring buffer that the
// next P1 reads.
#include "vs_cg_common.cuh"
#include "vs_desc.cuh"

namespace vs {

// a*b + c.  Rounded twice, as numpy rounds it, unless the build contracts (-DVS_X_FMA=bits:
// 1 the stencil, 2 the sums, 4 the vector updates): with every contraction the tiny golden
// cases, where CG nearly terminates finitely, drift off the reference's iteration counts
// (pack3d/SIMPLE: 280/176 against the reference's 272/163; 272/162 without)
#ifndef VS_X_FMA
#define VS_X_FMA 0
#endif
#ifndef VS_X_W  // DOFs per thread and step of the stream pass (1 or 2)
#define VS_X_W 1
#endif
#ifndef VS_X_PFMASK  // stream pass: lanes with (lane & mask) == 0 issue the L2 hints
#define VS_X_PFMASK 0
#endif
#ifndef VS_X_CARRY  // stencil pass: own z, s_old loaded a step ahead
#define VS_X_CARRY 0
#endif
#ifndef VS_X_TMA  // own streams of P1 and of the light P2 staged in shared memory by cp.async.bulk
#define VS_X_TMA 0
#endif
// ---- bulk-copy pipeline (VS_X_TMA): PS stages of one 1024-DOF chunk each, chunk k + PD issued at step k
#ifndef VS_X_PS
#define VS_X_PS 4
#endif
constexpr int PS = VS_X_PS, PD = PS - 2;
constexpr uint32_t ST_Z = 0, ST_S = (1024 + 4) * 8, ST_D = ST_S + 1024 * 8;  // z (+ 2 halo each side), s, descriptors / code indices
constexpr uint32_t ST_BYTES = (ST_D + 1024 * 8 + 127) / 128 * 128;
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

#ifndef VS_X_BPF  // L2 prefetch of the next chunks by cp.async.bulk.prefetch (one instruction per stream and step)
#define VS_X_BPF 1
#endif
#ifndef VS_X_WL  // DOFs per thread and step of the LIGHT stream pass (1 or 2)
#define VS_X_WL VS_X_W
#endif
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

template <int BIT>
__device__ __forceinline__ double xfma(double a, double b, double c) {
    if ((VS_X_FMA & BIT) != 0) return fma(a, b, c);
    return __dadd_rn(__dmul_rn(a, b), c);
}
constexpr int FS = 1, FD = 2, FU = 4;  // stencil, dot products, updates

template <int DIM, int OP, int M, int NT>
__global__ void __launch_bounds__(NT, 1) k_pcgx(const CgParams P) {
    if (P.gate && *P.gate) {  // enqueued ahead of the host, and the outer loop is already over
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            CgOut *o = P.out;
            o->iterations = 0;
            o->converged = 1;
            o->status = 0;
            o->value = 0.0;
            o->at_iter = 0;
            o->res_prec0 = o->res_unprec0 = o->res_prec_last = o->res_unprec_last = 0.0;
        }
        return;
    }
    constexpr bool PROJ = (OP == 1);
    constexpr int NS = 2 * DIM;
    __shared__ double s_tab[48];  // [40..47]: S_hat face weights times inv_h^2
    __shared__ double s_warp[NT / 32][5];
    __shared__ double s_tot[5];
    __shared__ __align__(16) double s_val[4][NT];  // grid_sum staging
    __shared__ CgGroup G;
    constexpr bool TMA = VS_X_TMA != 0;
    extern __shared__ __align__(128) unsigned char s_pipe[];  // TMA: PS stages of ST_BYTES
    __shared__ __align__(8) uint64_t s_full[PS], s_empty[PS];
    const int grp = P.group_base + blockIdx.x / P.bpg;
    if (threadIdx.x == 0) {
        G = P.groups[grp];
        if (TMA) {
#pragma unroll
            for (int q = 0; q < PS; ++q) {
                mbar_init(s_full + q, 1);         // the producer's expect_tx arrival
                mbar_init(s_empty + q, NT / 32);  // one arrival per consumer warp
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
    }
    if (threadIdx.x < 16) {
        s_tab[threadIdx.x] = P.diag_code[threadIdx.x];
        s_tab[16 + threadIdx.x] = P.inv_code[threadIdx.x];
        if (threadIdx.x < 8) {
            s_tab[32 + threadIdx.x] = P.invA_enc[threadIdx.x];
            s_tab[40 + threadIdx.x] = __dmul_rn(P.invA_enc[threadIdx.x], P.inv_h2);
        }
    }
    unsigned gen = __ldcg(P.bar_base);
    __syncthreads();
    const Tabs T{s_tab, s_tab + 16, s_tab + 32, P.invS};
    const double *wS = s_tab + 40;
    const double2 *sdg = P.sdiag2;
    const double2 *ctab = P.ctab;
    __builtin_assume(__isGlobal(ctab));
    const uint32_t m = G.m_own;
    const uint32_t blk0 = (blockIdx.x % P.bpg) * NT;  // first DOF of this block's chunk in stride 0
    const uint32_t tid = blk0 + threadIdx.x;
    const uint32_t stride = P.bpg * NT;
    double *x = G.x, *sv = G.q, *dv = G.d0;
    const uint64_t *desc = G.desc;
    const uint16_t *cidx = G.cidx;
    const uint64_t *rec = G.rec;
    const int2 *xb = G.xb;
    const bool halo = G.zpeer[0] != nullptr;
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(sv));
    __builtin_assume(__isGlobal(dv));
    __builtin_assume(__isGlobal(desc));
    __builtin_assume(__isGlobal(cidx));
    __builtin_assume(__isGlobal(rec));
    __builtin_assume(__isGlobal(xb));
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // L2 prefetch distances in grid strides, per pass (experiment overrides in VOXSCHUR_DBG:
    // bits 4-7 P1, 8-11 light P2, 12-15 heavy P2)
    const uint32_t pfd = (((P.dbg >> 4) & 15u) ? ((P.dbg >> 4) & 15u) : P.pf_dist) * stride;
    const uint32_t pfd_l = (((P.dbg >> 8) & 15u) ? ((P.dbg >> 8) & 15u) : P.pf_dist) * stride;
    const uint32_t pfd_h = (((P.dbg >> 12) & 15u) ? ((P.dbg >> 12) & 15u) : P.pf_dist) * stride;
    constexpr bool carry_own = VS_X_CARRY != 0;

    // first / last owned plane of a slab -> the neighbour slab's ghost plane of ring buffer b
    auto halo_to = [&](int b, int fam, uint32_t i, double zi) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const uint32_t b0 = G.sbeg[s][fam];
            if (i >= b0 && i < G.send[s][fam]) {
                double *dst = G.zrp[s][b];
                __builtin_assume(__isGlobal(dst));
                dst[G.sdst[s][fam] + (i - b0)] = zi;
            }
        }
    };
    // descriptor -> record bits, gather indices (an absent neighbour reads the
    // DOF itself) and the presence mask (A zeroes absent slots)
    auto decode = [&](uint64_t d, uint32_t i, int2 cb, uint64_t &rc, uint32_t (&j)[NS], uint32_t &pres) {
        const uint32_t fx = (uint32_t)(d >> SH_XP) & DX_MASK;
        if (fx == DX_ESC) {  // escape: the record and the bitmask lookups
            rc = rec[i];
            uint32_t nr[NS];
            neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
            pres = 0;
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                j[s] = nr[s] != ABSENT ? nr[s] : i;
                pres |= (nr[s] != ABSENT ? 1u : 0u) << s;
            }
            return;
        }
        rc = desc_rec<OP>(d);
        pres = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) pres |= (rec_has_nb<OP>(rc, s) ? 1u : 0u) << s;
        j[0] = (pres & 1u) ? i + (uint32_t)cb.x + fx : i;
        j[1] = (pres & 2u) ? i + (uint32_t)cb.y + ((uint32_t)(d >> SH_XM) & DX_MASK) : i;
        if (DIM == 3) {  // absent y slots carry distance 0
            j[2] = i + ((uint32_t)(d >> SH_YP) & DY_MASK);
            j[3] = i - ((uint32_t)(d >> SH_YM) & DY_MASK);
        }
        j[NS - 2] = i + ((pres >> (NS - 2)) & 1u);
        j[NS - 1] = i - ((pres >> (NS - 1)) & 1u);
    };
    // L2 prefetch of the block's chunk pf_dist strides ahead: one line per lane,
    // warp w covers half (w & 1) of stream (w >> 1)
    auto prefetch_chunk = [&](uint32_t c0, const void *base, int sh) {
        const uint32_t per_line = 128u >> sh;
        const uint32_t i = c0 + ((uint32_t)(warp & 1) * 32u + (uint32_t)lane) * per_line;
        if (base && i < c0 + NT && i < m) prefetch_l2(reinterpret_cast<const char *>(base) + ((size_t)i << sh));
    };

    // the same by the copy engine: warp w < nstr (lane 0) prefetches stream w's chunk of `cnt`
    // elements starting at element c0 (a multiple of 16 B) -- one instruction per stream and step
    constexpr bool BPF = VS_X_BPF != 0;
    auto bulk_pf = [&](uint32_t c0, uint32_t cnt, const void *base, int sh) {
        if (base && c0 < m) {
            const uint32_t n = min(cnt, m - c0);
            bulk_prefetch_l2(reinterpret_cast<const char *>(base) + ((size_t)c0 << sh), ((n << sh) + 15u) & ~15u);
        }
    };

    // ---- bulk-copy pipeline.  A pass over this block's chunks (chunk k = DOFs [blk0 + k stride,
    // + 1024)) takes its own streams from shared memory: thread 0 issues chunk k + PD at step k
    // (cp.async.bulk, completion on s_full[stage]); a stage is reused once every warp has
    // arrived on s_empty[stage].  pq counts the chunks this block has consumed so far (all
    // passes): stage = pq mod PS, use = pq / PS gives the barrier parities.
    uint32_t pq = 0;
    const uint32_t nsteps = blk0 < m ? (m - blk0 + stride - 1) / stride : 0;
    const uint32_t m_pad = (m + 1u) & ~1u;  // vectors are allocated in 256-B units: reading z[m] is in bounds
    auto stage_ptr = [&](uint32_t q) { return s_pipe + (size_t)(q % PS) * ST_BYTES; };
    // kind 0: P1 (z with a 2-element halo each side, s_old unless first, descriptors); 1: light P2 (z, s, code indices)
    auto pipe_issue = [&](int kind, bool with_s, uint32_t k, const double *zsrc) {  // thread 0 only
        const uint32_t q = pq + k, st = q % PS, use = q / PS;
        if (use >= 1) mbar_wait(s_empty + st, (use - 1) & 1u);
        unsigned char *sp = stage_ptr(q);
        const uint32_t c = blk0 + k * stride;
        const uint32_t cnt = min(1024u, m - c);
        const uint32_t b8 = ((cnt * 8u) + 15u) & ~15u;
        if (kind == 0) {
            const uint32_t lo = c >= 2 ? c - 2 : 0, hi = min(c + 1026u, m_pad);
            const uint32_t bz = (hi - lo) * 8u;
            mbar_expect(s_full + st, bz + (with_s ? b8 : 0u) + b8);
            bulk_g2s(sp + ST_Z + (size_t)(lo - (c - 2)) * 8u, zsrc + lo, bz, s_full + st);
            if (with_s) bulk_g2s(sp + ST_S, sv + c, b8, s_full + st);
            bulk_g2s(sp + ST_D, desc + c, b8, s_full + st);
        } else {
            const uint32_t b2 = ((cnt * 2u) + 15u) & ~15u;
            mbar_expect(s_full + st, 2 * b8 + b2);
            bulk_g2s(sp + ST_Z, zsrc + c, b8, s_full + st);
            bulk_g2s(sp + ST_S, sv + c, b8, s_full + st);
            bulk_g2s(sp + ST_D, cidx + c, b2, s_full + st);
        }
    };
    auto pipe_begin = [&](int kind, bool with_s, const double *zsrc) {
        if (threadIdx.x == 0) {
            // the other blocks' stores of the previous pass (generic proxy, ordered by the grid
            // barrier) precede these copies (async proxy)
            asm volatile("fence.proxy.async;" ::: "memory");
            for (uint32_t k = 0; k < (uint32_t)PD && k < nsteps; ++k) pipe_issue(kind, with_s, k, zsrc);
        }
    };
    auto pipe_wait = [&](uint32_t k) -> unsigned char * {
        const uint32_t q = pq + k;
        mbar_wait(s_full + (q % PS), (q / PS) & 1u);
        return stage_ptr(q);
    };
    auto pipe_release = [&](uint32_t k) {
        __syncwarp();
        if (lane == 0) mbar_arrive(s_empty + ((pq + k) % PS));
    };

    // ---- setup (krylov.py:102-119): project rhs; r = op(x0) - rhs; z = M^-1 r; d = 0
    double mu_rhs = 0.0, mu = 0.0, rz = 0.0, rp0 = 0.0, ru0 = 0.0;
    if (PROJ) {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], G.rhs[i]);
        grid_sum<1, false, NT>(v, 0, P, gen, s_val, s_tot);
        mu_rhs = v[0] / P.m_global;
    }
    {
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double *x0 = G.x0;
        double *z0 = G.zr[0];
        __builtin_assume(__isGlobal(z0));
        for (uint32_t i = tid; i < m; i += stride) {
            const uint64_t rc = rec[i];
            double ax = 0.0, xi = 0.0;
            if (x0) {
                uint32_t nr[NS];
                neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
                xi = x0[i];
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) vn[s] = nr[s] != ABSENT ? x0[nr[s]] : 0.0;
                ax = op_value<DIM, OP>(rc, xi, vn, T, inv_h, inv_h2);
                if (x0 != x) x[i] = xi;
            } else {
                x[i] = 0.0;
            }
            dv[i] = 0.0;  // d_0 = z'_0 + beta_0 d_{-1} with beta_0 = 0: the value read must be finite
            const double b = PROJ ? __dsub_rn(G.rhs[i], mu_rhs) : G.rhs[i];
            const double ri = __dsub_rn(ax, b);
            const double zi = __dmul_rn(ri, jacobi_inv<OP>(rc, T));
            z0[i] = zi;
            if (halo) halo_to(0, OP == 0 ? rec_comp(rc) : 0, i, zi);
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
            v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
            v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
            v[3] = __dadd_rn(v[3], zi);
            v[4] = __dadd_rn(v[4], ri);
        }
        grid_sum_shfl<5, true, NT>(v, 1, P, gen, s_warp, s_tot);
        if (PROJ) {
            mu = v[3] / P.m_global;
            v[0] = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
            v[1] = __dsub_rn(v[1], __dmul_rn(mu, v[3]));
        }
        rz = v[0];
        rp0 = sqrt(v[1]);
        ru0 = sqrt(v[2]);
    }
    const double ref = rp0;  // inner solves stop on the preconditioned norm (schur.py:207-210, :259-262)
    double beta = 0.0, alpha_prev = 0.0, rp_last = rp0, sval = 0.0;
    int status = 0;
    int64_t sat = 0, its = 0;
    bool conv = (ref == 0.0);
    // pending (d, x) updates: their scalars, oldest first; fbase = ring buffer of the oldest pending z
    // (shared memory: every thread writes the same values, and block barriers of the grid sums
    // lie between a write and the reads -- nothing is carried in registers across P1)
    __shared__ double s_hist[3][PCGX_MAX_DEPTH];
    int pend = 0, fbase = 0, cur = 0;
    unsigned long long ph[4] = {0, 0, 0, 0};
    if (!conv) {
        for (int64_t it = 0; it < P.max_iter; ++it) {
            if (rz < 0.0) { status = 1; sval = rz; sat = it; break; }
            if (rz == 0.0) { conv = true; break; }
            if (P.xgpu && *P.xflag) { status = 4; sat = it; break; }  // a peer rank never arrived
            const int nxt = (cur + 1 == M) ? 0 : cur + 1;
            const double *zc_ = G.zr[cur];
            double *zn_ = G.zr[nxt];
            __builtin_assume(__isGlobal(zc_));
            __builtin_assume(__isGlobal(zn_));
            const uint64_t t0 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            // ---- P1: s = M A z + beta s_old; sums z.Az (, sum Az)
            constexpr int K1 = PROJ ? 2 : 1;
            double v1[K1];
#pragma unroll
            for (int s = 0; s < K1; ++s) v1[s] = 0.0;
            auto pass1 = [&](auto first_c) {
                constexpr bool first = decltype(first_c)::value;
                const int ps = warp >> 1;  // this warp's prefetch stream: z, descriptors, s_old
                const void *pfb = ps == 0 ? (const void *)zc_
                                : ps == 1 ? (const void *)desc
                                : (!first && ps == 2) ? (const void *)sv : nullptr;
                uint64_t dn_ = 0;  // the next step's descriptor and chunk base, carried across the step
                int2 cbn_ = make_int2(0, 0);
                double zcn_ = 0.0, son_ = 0.0;  // and its own z, s_old (VS_X_CARRY)
                if (!TMA && tid < m) {
                    dn_ = __ldcs(desc + tid);
                    cbn_ = __ldg(xb + (tid >> CHUNK_SHIFT));
                    if (carry_own) {
                        zcn_ = zc_[tid];
                        if (!first) son_ = sv[tid];
                    }
                }
                if (TMA) pipe_begin(0, !first, zc_);
                uint32_t c0 = blk0, k = 0;
                for (uint32_t i = tid; TMA ? (c0 < m) : (i < m); i += stride, c0 += stride, ++k) {
                    uint64_t d;
                    int2 cb;
                    double zc, so, zlo = 0.0, zhi = 0.0;
                    if (TMA) {
                        if (threadIdx.x == 0 && k + PD < nsteps) pipe_issue(0, !first, k + PD, zc_);
                        cb = __ldg(xb + (c0 >> CHUNK_SHIFT));
                        const unsigned char *sp = pipe_wait(k);
                        const double *zs = reinterpret_cast<const double *>(sp + ST_Z) + 2 + threadIdx.x;
                        zc = zs[0];
                        zlo = zs[-1];
                        zhi = zs[1];
                        so = first ? 0.0 : reinterpret_cast<const double *>(sp + ST_S)[threadIdx.x];
                        d = reinterpret_cast<const uint64_t *>(sp + ST_D)[threadIdx.x];
                    } else {
                        if (BPF) {
                            if (pfd && lane == 0 && warp < 3)
                                bulk_pf(c0 + pfd, NT, warp == 0 ? (const void *)zc_ : warp == 1 ? (const void *)desc
                                                      : first ? nullptr : (const void *)sv, 3);
                        } else if (pfd) {
                            prefetch_chunk(c0 + pfd, pfb, 3);
                        }
                        d = dn_;
                        cb = cbn_;
                        zc = zcn_;
                        so = son_;
                        if (i + stride < m) {  // issued first: a whole step to arrive
                            dn_ = __ldcs(desc + i + stride);
                            cbn_ = __ldg(xb + ((i + stride) >> CHUNK_SHIFT));
                            if (carry_own) {
                                zcn_ = zc_[i + stride];
                                if (!first) son_ = sv[i + stride];
                            }
                        }
                        if (!carry_own) {
                            zc = zc_[i];
                            so = first ? 0.0 : sv[i];
                        }
                    }
                    if (!TMA || i < m) {  // (the tail of the last chunk computes nothing but still releases its stage)
                    uint64_t rc;
                    uint32_t j[NS], pres;
                    decode(d, i, cb, rc, j, pres);
                    double zn[NS];
#pragma unroll
                    for (int s = 0; s < NS - 2; ++s) zn[s] = zc_[j[s]];
                    if (TMA) {
                        // z+-: ranks i +- 1 (or i when absent) are in the staged window; an escape
                        // (periodic wrap) reads global memory
                        const bool esc = ((uint32_t)(d >> SH_XP) & DX_MASK) == DX_ESC;
                        zn[NS - 2] = esc ? zc_[j[NS - 2]] : (((pres >> (NS - 2)) & 1u) ? zhi : zc);
                        zn[NS - 1] = esc ? zc_[j[NS - 1]] : (((pres >> (NS - 1)) & 1u) ? zlo : zc);
                    } else {
                        zn[NS - 2] = zc_[j[NS - 2]];
                        zn[NS - 1] = zc_[j[NS - 1]];
                    }
                    double inv, dg;
                    inv_diag<OP>(rc, T, sdg, inv, dg);
                    double w;
                    if (OP == 1) {
                        // S_hat z = sum_a (z_i - z_in) W_in - (z_out - z_i) W_out, face weights
                        // pre-multiplied by inv_h^2 (schur.py:234-240 up to rounding); differences
                        // only, so the mean mu cancels and raw z is used; an absent face has weight 0
                        w = 0.0;
#pragma unroll
                        for (int a = 0; a < DIM; ++a) {
                            w = xfma<FS>(__dsub_rn(zc, zn[2 * a + 1]), wS[rec_pin(rc, a)], w);
                            w = xfma<FS>(__dsub_rn(zc, zn[2 * a]), wS[rec_pout(rc, a)], w);
                        }
                    } else {
                        double vn[NS];
#pragma unroll
                        for (int s = 0; s < NS; ++s) vn[s] = ((pres >> s) & 1u) ? zn[s] : 0.0;
                        w = op_value<DIM, OP>(rc, zc, vn, T, inv_h, inv_h2);
                    }
                    const double mw = __dmul_rn(w, inv);
                    sv[i] = first ? mw : xfma<FU>(beta, so, mw);
                    v1[0] = xfma<FD>(zc, w, v1[0]);
                    if (PROJ) v1[1] = __dadd_rn(v1[1], w);
                    }
                    if (TMA) pipe_release(k);
                }
                if (TMA) pq += nsteps;
            };
            if (it == 0)
                pass1(std::true_type{});
            else
                pass1(std::false_type{});
            const uint64_t t1 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            grid_sum<K1, false, NT>(v1, 2, P, gen, s_val, s_tot);
            const uint64_t t2 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            const double delta = PROJ ? __dsub_rn(v1[0], __dmul_rn(mu, v1[PROJ ? 1 : 0])) : v1[0];
            const double dq = it == 0 ? delta : __dsub_rn(delta, __dmul_rn(beta, rz) / alpha_prev);
            if (dq <= 0.0) { status = 2; sval = dq; sat = it; break; }
            const double alpha = rz / dq, nalpha = -alpha;
            // ---- P2: z_next = z - alpha s; sums r.z = sum diag z^2, z.z (+ sum z, sum r);
            // heavy (every M-th): d and x brought up to date from the ring
            constexpr int KL = PROJ ? 4 : 2;
            double v[KL];
#pragma unroll
            for (int s = 0; s < KL; ++s) v[s] = 0.0;
            auto pass2 = [&](auto heavy_c) {
                constexpr bool heavy = decltype(heavy_c)::value;
                const double *zo_[M > 1 ? M - 1 : 1];  // the older z of the pending updates, oldest first
#pragma unroll
                for (int q = 0; q < M - 1; ++q) {
                    const int b = fbase + q;
                    zo_[q] = G.zr[b >= M ? b - M : b];
                    __builtin_assume(__isGlobal(zo_[q]));
                }
                // the stream pass: thread t of a block step owns W consecutive DOFs of the step's
                // W*NT chunk (W = 2: 16-B loads and stores)
                // (every pass ends in a grid barrier, so the passes need not agree on who owns a DOF)
                constexpr int W = heavy ? VS_X_W : VS_X_WL;
                static_assert(W == 1 || W == 2, "stream-pass width");
                if (TMA && !heavy) {  // the light pass from the bulk-copy pipeline: z, s and the code index staged
                    pipe_begin(1, true, zc_);
                    uint32_t c0 = blk0, k = 0;
                    for (uint32_t i = tid; c0 < m; i += stride, c0 += stride, ++k) {
                        if (threadIdx.x == 0 && k + PD < nsteps) pipe_issue(1, true, k + PD, zc_);
                        const unsigned char *sp = pipe_wait(k);
                        if (i < m) {
                            const double zo = reinterpret_cast<const double *>(sp + ST_Z)[threadIdx.x];
                            const double si = reinterpret_cast<const double *>(sp + ST_S)[threadIdx.x];
                            const uint32_t ci = reinterpret_cast<const uint16_t *>(sp + ST_D)[threadIdx.x];
                            const double dg = __ldg(ctab + (OP == 0 ? (ci & 0xFFu) : ci)).y;
                            const double zi = xfma<FU>(nalpha, si, zo);
                            zn_[i] = zi;
                            if (halo) halo_to(nxt, OP == 0 ? (int)(ci >> 8) : 0, i, zi);
                            const double ri = __dmul_rn(dg, zi);
                            v[0] = xfma<FD>(ri, zi, v[0]);
                            v[1] = xfma<FD>(zi, zi, v[1]);
                            if (PROJ) {
                                v[2] = __dadd_rn(v[2], zi);
                                v[3] = __dadd_rn(v[3], ri);
                            }
                        }
                        pipe_release(k);
                    }
                    pq += nsteps;
                    return;
                }
                auto ldw = [&](const double *p, uint32_t i, bool two, double (&o)[W]) {
                    if (W == 2 && two) {
                        const double2 t = *reinterpret_cast<const double2 *>(p + i);
                        o[0] = t.x;
                        o[W - 1] = t.y;
                    } else {
                        o[0] = p[i];
                        if (W == 2) o[W - 1] = 0.0;
                    }
                };
                auto stw = [&](double *p, uint32_t i, bool two, const double (&o)[W]) {
                    if (W == 2 && two)
                        *reinterpret_cast<double2 *>(p + i) = make_double2(o[0], o[W - 1]);
                    else
                        p[i] = o[0];
                };
                auto ldc = [&](uint32_t i) -> uint32_t {  // W 2-B code indices
                    return (W == 2 && i + 1 < m) ? *reinterpret_cast<const uint32_t *>(cidx + i)
                                                 : (uint32_t)__ldcs(cidx + i);
                };
                const uint32_t i0 = W * tid, sw = W * stride, pfw = W * (heavy ? pfd_h : pfd_l);
                uint32_t cin_ = i0 < m ? ldc(i0) : 0u;  // the next step's code indices, carried
                // this warp's prefetch stream (BPF): z, s, code indices; heavy: d, x, the older z
                const void *pfs = nullptr;
                if (BPF && lane == 0) {
                    pfs = warp == 0 ? (const void *)zc_ : warp == 1 ? (const void *)sv : warp == 2 ? (const void *)cidx : nullptr;
                    if (heavy) {
                        if (warp == 3) pfs = dv;
                        if (warp == 4) pfs = x;
#pragma unroll
                        for (int q = 0; q < M - 1; ++q)
                            if (warp == 5 + q) pfs = zo_[q];
                    }
                }
                uint32_t cb0 = W * blk0;
                for (uint32_t i = i0; i < m; i += sw, cb0 += sw) {
                    const bool two = W == 2 && i + 1 < m;
                    const uint32_t ip = i + pfw;
                    if (BPF) {
                        if (pfw && pfs) bulk_pf(cb0 + pfw, W * NT, pfs, warp == 2 ? 1 : 3);
                    } else if (pfw && ip < m && (lane & VS_X_PFMASK) == 0) {
                        prefetch_l2(zc_ + ip);
                        prefetch_l2(sv + ip);
                        if (heavy) {
                            prefetch_l2(dv + ip);
                            prefetch_l2(x + ip);
#pragma unroll
                            for (int q = 0; q < M - 1; ++q) prefetch_l2(zo_[q] + ip);
                        }
                    }
                    const uint32_t ci2 = cin_;
                    uint32_t ci[W];
                    double dg[W];
#pragma unroll
                    for (int e = 0; e < W; ++e) {
                        ci[e] = e == 0 ? (ci2 & 0xFFFFu) : (ci2 >> 16);
                        dg[e] = __ldg(ctab + (OP == 0 ? (ci[e] & 0xFFu) : ci[e])).y;
                    }
                    if (i + sw < m) cin_ = ldc(i + sw);
                    double zo[W], si[W], dd[W], xx[W], zh[M > 1 ? M - 1 : 1][W], zi[W];
                    ldw(zc_, i, two, zo);
                    ldw(sv, i, two, si);
                    if (heavy) {
#pragma unroll
                        for (int q = 0; q < M - 1; ++q) ldw(zo_[q], i, two, zh[q]);  // before z_next overwrites the oldest
                        ldw(dv, i, two, dd);
                        ldw(x, i, two, xx);
                    }
#pragma unroll
                    for (int e = 0; e < W; ++e) zi[e] = xfma<FU>(nalpha, si[e], zo[e]);
                    stw(zn_, i, two, zi);
                    if (halo) {
                        halo_to(nxt, OP == 0 ? (int)(ci[0] >> 8) : 0, i, zi[0]);
                        if (two) halo_to(nxt, OP == 0 ? (int)(ci[W - 1] >> 8) : 0, i + 1, zi[W - 1]);
                    }
#pragma unroll
                    for (int e = 0; e < W; ++e) {  // a missing second DOF contributes zeros
                        const double ri = __dmul_rn(dg[e], zi[e]);
                        v[0] = xfma<FD>(ri, zi[e], v[0]);
                        v[1] = xfma<FD>(zi[e], zi[e], v[1]);
                        if (PROJ) {
                            v[2] = __dadd_rn(v[2], zi[e]);
                            v[3] = __dadd_rn(v[3], ri);
                        }
                    }
                    if (heavy) {
#pragma unroll
                        for (int e = 0; e < W; ++e) {
#pragma unroll
                            for (int q = 0; q < M - 1; ++q) {
                                // the recorded scalars: uniform shared-memory reads, not 6 (M-1) registers
                                dd[e] = xfma<FU>(s_hist[1][q], dd[e], PROJ ? __dsub_rn(zh[q][e], s_hist[0][q]) : zh[q][e]);
                                xx[e] = xfma<FU>(s_hist[2][q], dd[e], xx[e]);
                            }
                            dd[e] = xfma<FU>(beta, dd[e], PROJ ? __dsub_rn(zo[e], mu) : zo[e]);
                            xx[e] = xfma<FU>(nalpha, dd[e], xx[e]);
                        }
                        stw(dv, i, two, dd);
                        stw(x, i, two, xx);
                    }
                }
            };
            if (pend + 1 == M) {
                pass2(std::true_type{});
                pend = 0;
            } else {
                pass2(std::false_type{});
                if (pend == 0) fbase = cur;
                s_hist[0][pend] = mu;
                s_hist[1][pend] = beta;
                s_hist[2][pend] = nalpha;
                ++pend;
            }
            const uint64_t t3 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            grid_sum<KL, true, NT>(v, 3, P, gen, s_val, s_tot);
            if (P.phase_ns && threadIdx.x == 0) {
                const uint64_t t4 = gtimer();
                ph[0] += t1 - t0;
                ph[1] += t2 - t1;
                ph[2] += t3 - t2;
                ph[3] += t4 - t3;
            }
            if (PROJ) {
                mu = v[2] / P.m_global;
                v[0] = __dsub_rn(v[0], __dmul_rn(mu, v[3]));
                v[1] = __dsub_rn(v[1], __dmul_rn(mu, v[2]));
            }
            const double rz_new = v[0];
            beta = rz_new / rz;
            rz = rz_new;
            alpha_prev = alpha;
            cur = nxt;
            const double nz = sqrt(v[1]);
            if (!isfinite(nz)) { status = 3; sat = it + 1; break; }
            its = it + 1;
            rp_last = nz;
            if (nz / ref < P.tol) { conv = true; break; }
        }
    }
    // ---- the pending (d, x) updates, oldest first (each thread reads only what it wrote)
    if (M > 1 && pend > 0) {
        for (uint32_t i0 = VS_X_W * tid; i0 < m; i0 += VS_X_W * stride) {  // P2's mapping
#pragma unroll
            for (int e = 0; e < VS_X_W; ++e) {
                const uint32_t i = i0 + e;
                if (i >= m) break;
                double dd = dv[i], xx = x[i];
#pragma unroll
                for (int q = 0; q < M - 1; ++q)
                    if (q < pend) {
                        const int b = fbase + q;
                        const double *zq = G.zr[b >= M ? b - M : b];
                        __builtin_assume(__isGlobal(zq));
                        const double zj = zq[i];
                        dd = xfma<FU>(s_hist[1][q], dd, PROJ ? __dsub_rn(zj, s_hist[0][q]) : zj);
                        xx = xfma<FU>(s_hist[2][q], dd, xx);
                    }
                x[i] = xx;
            }
        }
    }
    if (P.phase_ns && threadIdx.x == 0) {  // [0..3] block 0, [4..7] max, [8..11] sum over blocks
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            if (blockIdx.x == 0) P.phase_ns[p] += ph[p];
            atomicMax(P.phase_ns + 4 + p, ph[p]);
            atomicAdd(P.phase_ns + 8 + p, ph[p]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *P.bar_base = gen;  // the next launch on this stream starts from here
        CgOut *o = P.out;
        o->iterations = its;
        o->converged = conv ? 1 : 0;
        o->status = status;
        o->value = sval;
        o->at_iter = sat;
        o->res_prec0 = rp0;
        o->res_unprec0 = ru0;
        o->res_prec_last = rp_last;
        o->res_unprec_last = ru0;
    }
}

template <int DIM, int OP>
static const void *pcgx_fn_t(int depth) {
    switch (depth) {
        case 1: return (const void *)k_pcgx<DIM, OP, 1, CG_THREADS>;
        case 3: return (const void *)k_pcgx<DIM, OP, 3, CG_THREADS>;
        case 4: return (const void *)k_pcgx<DIM, OP, 4, CG_THREADS>;
        default: return (const void *)k_pcgx<DIM, OP, 2, CG_THREADS>;
    }
}
static const void *pcgx_fn(int dim, int op, int depth) {
    if (dim == 3) return op == 0 ? pcgx_fn_t<3, 0>(depth) : pcgx_fn_t<3, 1>(depth);
    return op == 0 ? pcgx_fn_t<2, 0>(depth) : pcgx_fn_t<2, 1>(depth);
}

// Plan: one block per SM (per group); no dynamic shared memory.  `unroll` carries the
// ring depth M (1..4; VOXSCHUR_X_DEPTH).
CgPlan pcgx_plan(int dim, int op, int64_t m, int groups, int device, int sms) {
    CgPlan pl{};
    pl.alg = CG_TWO_SUM_MX;
    int depth = PCGX_DEPTH_DEFAULT;
    if (const char *e = getenv("VOXSCHUR_X_DEPTH"))
        if (atoi(e) >= 1 && atoi(e) <= PCGX_MAX_DEPTH) depth = atoi(e);
    pl.unroll = depth;
    pl.tier = 5;
    pl.threads = CG_THREADS;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    if (sms > 0 && sms < nsm) nsm = sms;
    pl.smem = VS_X_TMA ? (size_t)PS * ST_BYTES : 0;  // the bulk-copy pipeline's stages
    if (pl.smem) cudaFuncSetAttribute(pcgx_fn(dim, op, depth), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcgx_fn(dim, op, depth), pl.threads, pl.smem);
    if (per_sm < 1) per_sm = 1;
    pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * nsm / groups, (m + pl.threads - 1) / pl.threads));
    pl.slots = 0;
    return pl;
}

cudaError_t launch_pcgx(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s) {
    P.cache_slots = 0;
    P.bpg = pl.grid;
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel(pcgx_fn(dim, op, pl.unroll), dim3(pl.grid * groups), dim3(pl.threads), args,
                                       pl.smem, s);
}

}  // namespace vs
