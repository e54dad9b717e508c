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
//    are exactly those of an every-iteration update (the depths differ only in
//    how the grid sums round: the light and the heavy pass map DOFs to threads
//    differently).  The other P2s ("light") read z, s and the 2-B code
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
#ifndef VS_X_WL  // DOFs per thread and step of the LIGHT stream pass (1 or 2)
#define VS_X_WL 2
#endif
#ifndef VS_X_LU  // light stream pass: 2 = two pair-steps per loop trip, all loads first
#define VS_X_LU 2
#endif
#ifndef VS_X_NT2  // threads of a block that take part in the stream passes of HBM-sized operators
#define VS_X_NT2 768
#endif
#ifndef VS_X_U2  // stencil pass: two steps per loop trip (carried words ping-ponged)
#define VS_X_U2 1
#endif
#ifndef VS_X_BPF2  // stream pass: L2 prefetch by the copy engine too (measured slower there: P2 182 -> 195 us)
#define VS_X_BPF2 0
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

template <int DIM, int OP, int M, int NT, bool MR>
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
    const int grp = P.group_base + blockIdx.x / P.bpg;
    if (threadIdx.x == 0) {
        G = P.groups[grp];
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
    // (P1 looks three strides ahead: against one, C4 S_hat P1 232 -> 218, A 463 -> 402 us; three
    // against two, same call: S_hat 389.8 -> 389.2, A 784.6 -> 780.0 us/it)
    const uint32_t pf1 = (((P.dbg >> 4) & 15u) ? ((P.dbg >> 4) & 15u) : 3u * P.pf_dist) * stride;
    const uint32_t pfd_l = (((P.dbg >> 8) & 15u) ? ((P.dbg >> 8) & 15u) : P.pf_dist) * stride;
    const uint32_t pfd_h = (((P.dbg >> 12) & 15u) ? ((P.dbg >> 12) & 15u) : P.pf_dist) * stride;

    // Threads of a block that take part in the stream passes.  With all 1024 streaming from HBM the
    // SMs get unequal shares of the bandwidth and a pass ends 8 % after its mean block (C4 512^3:
    // P2 160 -> 153 us, the grid sum after it 34 -> 15); operators whose vectors largely stay in L2
    // want every thread (C2 256^3: P2 13.1 vs 13.9 us).
    const uint32_t nt2 = (P.m_global > 8.0e6 && VS_X_NT2 < NT) ? VS_X_NT2 : NT;

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
        if (fx == DX_ESC) {  // escape (periodic wrap in y or z, a distance outside its field)
            const uint64_t eo = d >> SH_EORD;
            if (eo) {  // the gather indices from the escape table: one round trip, no record, no bitmask words
                const uint4 *et = G.esc + 2 * (eo - 1);  // (pointer re-read from shared memory: not held in a register)
                __builtin_assume(__isGlobal(et));
                const uint4 a = __ldg(et), b = __ldg(et + 1);
                j[0] = a.x;
                j[1] = a.y;
                j[2] = a.z;
                j[3] = a.w;
                if (DIM == 3) {
                    j[NS - 2] = b.x;
                    j[NS - 1] = b.y;
                }
                rc = desc_rec<OP>(d);
                pres = 0;
#pragma unroll
                for (int s = 0; s < NS; ++s) pres |= (rec_has_nb<OP>(rc, s) ? 1u : 0u) << s;
                return;
            }
            const uint64_t *rp = G.rec;
            __builtin_assume(__isGlobal(rp));
            rc = rp[i];  // the table was full: the record and the bitmask lookups
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
    // L2 prefetch by the copy engine: one thread prefetches a stream's chunk of `cnt` elements
    // starting at element c0 (a multiple of 16 B) -- one instruction per stream and step instead of
    // one hint per 128-B line (P1: 214 -> 205 us at C4; hints issued in bursts are dropped under load)
    auto bulk_pf = [&](uint32_t c0, uint32_t cnt, const void *base, int sh) {
        if (base && c0 < m) {
            const uint32_t n = min(cnt, m - c0);
            bulk_prefetch_l2(reinterpret_cast<const char *>(base) + ((size_t)c0 << sh), ((n << sh) + 15u) & ~15u);
        }
    };

    // The scalars of the iteration live in shared memory, not in registers: thread 0 writes them
    // after a grid sum, a block barrier follows, and a pass reads what it needs into locals.  Held
    // in registers (~40 of the 64) they made ptxas split P1's six gathers into dependent batches.
    __shared__ struct {
        double mu, rz, rp0, ru0, beta, alpha_prev, rp_last, sval;
        long long sat, its;
        unsigned long long t[4], ph[4];
        int status, conv;
    } S;
    // ---- setup (krylov.py:102-119): project rhs; r = op(x0) - rhs; z = M^-1 r; d = 0
    double mu_rhs = 0.0;
    if (PROJ) {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], G.rhs[i]);
        grid_sum<1, false, NT, MR>(v, 0, P, gen, s_val, s_tot);
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
        grid_sum_shfl<5, true, NT, MR>(v, 1, P, gen, s_warp, s_tot);
        if (threadIdx.x == 0) {
            double mu = 0.0;
            if (PROJ) {
                mu = v[3] / P.m_global;
                v[0] = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
                v[1] = __dsub_rn(v[1], __dmul_rn(mu, v[3]));
            }
            S.mu = mu;
            S.rz = v[0];
            S.rp0 = S.rp_last = sqrt(v[1]);  // inner solves stop on the preconditioned norm (schur.py:207-210, :259-262)
            S.ru0 = sqrt(v[2]);
            S.beta = S.alpha_prev = S.sval = 0.0;
            S.sat = S.its = 0;
            S.status = 0;
            S.conv = (S.rp0 == 0.0);
#pragma unroll
            for (int q = 0; q < 4; ++q) S.ph[q] = 0;
        }
        __syncthreads();
    }
    // pending (d, x) updates: their scalars, oldest first; fbase = ring buffer of the oldest pending z
    // (shared memory: every thread writes the same values, and block barriers of the grid sums
    // lie between a write and the reads -- nothing is carried in registers across P1)
    __shared__ double s_hist[3][PCGX_MAX_DEPTH];
    int pend = 0, fbase = 0, cur = 0;
    const bool t0_ = threadIdx.x == 0;
    if (!S.conv) {
        for (int64_t it = 0; it < P.max_iter; ++it) {
            {
                const double rz = S.rz;
                if (rz < 0.0) { if (t0_) { S.status = 1; S.sval = rz; S.sat = it; } break; }
                if (rz == 0.0) { if (t0_) S.conv = 1; break; }
            }
            if (P.xgpu && *P.xflag) { if (t0_) { S.status = 4; S.sat = it; } break; }  // a peer rank never arrived
            const int nxt = (cur + 1 == M) ? 0 : cur + 1;
            const double *zc_ = G.zr[cur];
            double *zn_ = G.zr[nxt];
            __builtin_assume(__isGlobal(zc_));
            __builtin_assume(__isGlobal(zn_));
            if (P.phase_ns && t0_) S.t[0] = gtimer();
            // ---- P1: s = M A z + beta s_old; sums z.Az (, sum Az)
            constexpr int K1 = PROJ ? 2 : 1;
            double v1[K1];
#pragma unroll
            for (int s = 0; s < K1; ++s) v1[s] = 0.0;
            auto pass1 = [&](auto first_c) {
                constexpr bool first = decltype(first_c)::value;
                const double beta = first ? 0.0 : S.beta;
                // one step: DOF i of the block's chunk c0, its descriptor d and chunk base cb already in
                // registers; the next step's are loaded into (dn_, cbn_) first -- a whole step to arrive
                auto step = [&](uint32_t i, uint32_t c0, const uint64_t d, const int2 cb, uint64_t &dn_, int2 &cbn_) {
                    // L2 prefetch of the block's chunk pf1 strides ahead: z, descriptors, s_old
                    if (pf1 && lane == 0 && warp < 3)
                        bulk_pf(c0 + pf1, NT, warp == 0 ? (const void *)zc_ : warp == 1 ? (const void *)desc
                                              : first ? nullptr : (const void *)sv, 3);
                    if (i + stride < m) {  // issued first
                        dn_ = __ldcs(desc + i + stride);
                        cbn_ = __ldg(xb + ((i + stride) >> CHUNK_SHIFT));
                    }
                    const double zc = zc_[i];
                    const double so = first ? 0.0 : sv[i];
                    uint64_t rc;
                    uint32_t j[NS], pres;
                    decode(d, i, cb, rc, j, pres);
                    double zn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) zn[s] = zc_[j[s]];
                    double inv, dg;
                    inv_diag<OP>(rc, T, sdg, inv, dg);
                    double w;
                    if (OP == 1) {
                        // S_hat z = sum_a (z_i - z_in) W_in - (z_out - z_i) W_out, face weights
                        // pre-multiplied by inv_h^2 (schur.py:234-240 up to rounding); differences
                        // only, so the mean mu cancels and raw z is used; an absent face has weight 0.
                        // (The weights are looked up where they are used: loading all six first, or in
                        // pairs, costs registers and ptxas then splits the gathers into more dependent
                        // batches -- P1 205 -> 235 us at C4.)
                        // (the 3-bit face codes sit at bits 8 + 3f of the record's high word: one
                        // shift and one mask give the byte offset into the 8-entry weight table)
                        const uint32_t hi = (uint32_t)(rc >> 32);
                        auto wgt = [&](int f) {
                            return *reinterpret_cast<const double *>(reinterpret_cast<const char *>(s_tab) + 40 * 8 +
                                                                     ((hi >> (5 + 3 * f)) & 0x38u));
                        };
                        w = 0.0;
#pragma unroll
                        for (int a = 0; a < DIM; ++a) {
                            w = xfma<FS>(__dsub_rn(zc, zn[2 * a + 1]), wgt(a), w);      // in face: code a
                            w = xfma<FS>(__dsub_rn(zc, zn[2 * a]), wgt(3 + a), w);      // out face: code 3 + a
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
                };
                // two steps per trip, the carried words ping-ponged between two register sets (no moves)
                uint64_t da = 0, db = 0;
                int2 ca = make_int2(0, 0), cb2 = ca;
                if (tid < m) {
                    da = __ldcs(desc + tid);
                    ca = __ldg(xb + (tid >> CHUNK_SHIFT));
                }
                uint32_t c0 = blk0;
                for (uint32_t i = tid; i < m; i += stride, c0 += stride) {
                    step(i, c0, da, ca, db, cb2);
                    if (VS_X_U2) {
                        i += stride;
                        c0 += stride;
                        if (i >= m) break;
                        step(i, c0, db, cb2, da, ca);
                    } else {
                        da = db;
                        ca = cb2;
                    }
                }
            };
            if (it == 0)
                pass1(std::true_type{});
            else
                pass1(std::false_type{});
            if (P.phase_ns && t0_) S.t[1] = gtimer();
            grid_sum<K1, false, NT, MR>(v1, 2, P, gen, s_val, s_tot);
            if (P.phase_ns && t0_) S.t[2] = gtimer();
            double nalpha;
            {
                const double delta = PROJ ? __dsub_rn(v1[0], __dmul_rn(S.mu, v1[PROJ ? 1 : 0])) : v1[0];
                const double dq = it == 0 ? delta : __dsub_rn(delta, __dmul_rn(S.beta, S.rz) / S.alpha_prev);
                if (dq <= 0.0) { if (t0_) { S.status = 2; S.sval = dq; S.sat = it; } break; }
                nalpha = -(S.rz / dq);
            }
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
                // (every pass ends in a grid barrier, so the passes need not agree on who owns a DOF)
                if (!heavy && VS_X_LU == 2) {
                    // the light pass, two pair-steps per trip: thread t owns DOFs 2t, 2t+1 of the
                    // 2*NT chunks at i and i + 2 stride; all four 16-B loads are issued before the
                    // first use (26 B per DOF need twice the bytes in flight of one pair-step to
                    // stream at the heavy pass's rate)
                    // (only the block's first NT2 threads stream: with all 1024 the SMs get unequal
                    // shares of the bandwidth and the pass ends 8 % after its mean block)
                    const uint32_t NT2 = nt2;
                    if (threadIdx.x >= NT2) return;
                    const uint32_t tid = (blockIdx.x % P.bpg) * NT2 + threadIdx.x, stride = P.bpg * NT2;
                    const uint32_t sw = 2 * stride, pfw = 2 * (pfd_l / NT) * NT2;
                    auto cix = [&](uint32_t i) -> uint32_t {
                        return i + 1 < m ? *reinterpret_cast<const uint32_t *>(cidx + i) : (i < m ? (uint32_t)cidx[i] : 0u);
                    };
                    auto ldp = [&](const double *p, uint32_t i) {
                        return i + 1 < m ? *reinterpret_cast<const double2 *>(p + i)
                                         : make_double2(i < m ? p[i] : 0.0, 0.0);
                    };
                    uint32_t ca_ = cix(2 * tid), cb_ = cix(2 * tid + sw);  // the next trip's code indices, carried
                    for (uint32_t i = 2 * tid; i < m; i += 2 * sw) {
                        const uint32_t ib = i + sw;
                        if (pfw) {
                            if (i + 2 * pfw < m) {
                                prefetch_l2(zc_ + i + 2 * pfw);
                                prefetch_l2(sv + i + 2 * pfw);
                            }
                            if (ib + 2 * pfw < m) {
                                prefetch_l2(zc_ + ib + 2 * pfw);
                                prefetch_l2(sv + ib + 2 * pfw);
                            }
                        }
                        const uint32_t cc[2] = {ca_, cb_};
                        double dgv[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint32_t ci = (e & 1) ? (cc[e >> 1] >> 16) : (cc[e >> 1] & 0xFFFFu);
                            dgv[e] = __ldg(ctab + (OP == 0 ? (ci & 0xFFu) : ci)).y;
                        }
                        ca_ = cix(i + 2 * sw);
                        cb_ = cix(ib + 2 * sw);
                        const double2 za = ldp(zc_, i), sa = ldp(sv, i), zb = ldp(zc_, ib), sb = ldp(sv, ib);
                        const double zo[4] = {za.x, za.y, zb.x, zb.y}, si[4] = {sa.x, sa.y, sb.x, sb.y};
                        double zi[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) zi[e] = xfma<FU>(nalpha, si[e], zo[e]);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t ih = h ? ib : i;
                            if (ih + 1 < m)
                                *reinterpret_cast<double2 *>(zn_ + ih) = make_double2(zi[2 * h], zi[2 * h + 1]);
                            else if (ih < m)
                                zn_[ih] = zi[2 * h];
                            if (halo) {
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const uint32_t ci = e ? (cc[h] >> 16) : (cc[h] & 0xFFFFu);
                                    if (ih + e < m) halo_to(nxt, OP == 0 ? (int)(ci >> 8) : 0, ih + e, zi[2 * h + e]);
                                }
                            }
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {  // a missing DOF contributes zeros
                            const double ri = __dmul_rn(dgv[e], zi[e]);
                            v[0] = xfma<FD>(ri, zi[e], v[0]);
                            v[1] = xfma<FD>(zi[e], zi[e], v[1]);
                            if (PROJ) {
                                v[2] = __dadd_rn(v[2], zi[e]);
                                v[3] = __dadd_rn(v[3], ri);
                            }
                        }
                    }
                    return;
                }
                // the stream pass: thread t of a block step owns W consecutive DOFs of the step's
                // W*NT chunk (W = 2: 16-B loads and stores)
                constexpr int W = heavy ? VS_X_W : VS_X_WL;
                static_assert(W == 1 || W == 2, "stream-pass width");
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
                const double beta_h = S.beta, mu_h = S.mu;  // (heavy)
                const uint32_t NTH = nt2;  // threads that take part (see the light pass)
                if (threadIdx.x >= NTH) return;
                const uint32_t tid = (blockIdx.x % P.bpg) * NTH + threadIdx.x, stride = P.bpg * NTH;
                const uint32_t blk0 = (blockIdx.x % P.bpg) * NTH;
                const uint32_t i0 = W * tid, sw = W * stride, pfw = W * ((heavy ? pfd_h : pfd_l) / NT) * NTH;
                uint32_t cin_ = i0 < m ? ldc(i0) : 0u;  // the next step's code indices, carried
                // this warp's prefetch stream (BPF): z, s, code indices; heavy: d, x, the older z
                constexpr bool BPF2 = VS_X_BPF2 != 0;
                const void *pfs = nullptr;
                if (BPF2 && lane == 0) {
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
                    if (BPF2) {
                        if (pfw && pfs) bulk_pf(cb0 + pfw, W * NT, pfs, warp == 2 ? 1 : 3);
                    } else if (pfw && ip < m) {
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
                            dd[e] = xfma<FU>(beta_h, dd[e], PROJ ? __dsub_rn(zo[e], mu_h) : zo[e]);
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
                if (t0_) {  // (read only after the next grid sum's block barriers)
                    s_hist[0][pend] = S.mu;
                    s_hist[1][pend] = S.beta;
                    s_hist[2][pend] = nalpha;
                }
                ++pend;
            }
            if (P.phase_ns && t0_) S.t[3] = gtimer();
            grid_sum<KL, true, NT, MR>(v, 3, P, gen, s_val, s_tot);
            if (P.phase_ns && t0_) {
                const uint64_t t4 = gtimer();
                S.ph[0] += S.t[1] - S.t[0];
                S.ph[1] += S.t[2] - S.t[1];
                S.ph[2] += S.t[3] - S.t[2];
                S.ph[3] += t4 - S.t[3];
            }
            double mu_n = 0.0;
            if (PROJ) {
                mu_n = v[2] / P.m_global;
                v[0] = __dsub_rn(v[0], __dmul_rn(mu_n, v[3]));
                v[1] = __dsub_rn(v[1], __dmul_rn(mu_n, v[2]));
            }
            cur = nxt;
            const double nz = sqrt(v[1]);
            const bool bad = !isfinite(nz), done = !bad && nz / S.rp0 < P.tol;
            // (the old scalars were last read before this grid sum's block barriers; rp0 never changes)
            if (t0_) {
                if (bad) {
                    S.status = 3;
                    S.sat = it + 1;
                } else {
                    S.mu = mu_n;
                    S.beta = v[0] / S.rz;
                    S.rz = v[0];
                    S.alpha_prev = -nalpha;
                    S.its = it + 1;
                    S.rp_last = nz;
                    if (done) S.conv = 1;
                }
            }
            __syncthreads();
            if (bad || done) break;
        }
    }
    __syncthreads();  // thread 0's status words of a break before the loop's last barrier
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
            if (blockIdx.x == 0) P.phase_ns[p] += S.ph[p];
            atomicMax(P.phase_ns + 4 + p, S.ph[p]);
            atomicAdd(P.phase_ns + 8 + p, S.ph[p]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *P.bar_base = gen;  // the next launch on this stream starts from here
        CgOut *o = P.out;
        o->iterations = S.its;
        o->converged = S.conv ? 1 : 0;
        o->status = S.status;
        o->value = S.sval;
        o->at_iter = S.sat;
        o->res_prec0 = S.rp0;
        o->res_unprec0 = S.ru0;
        o->res_prec_last = S.rp_last;
        o->res_unprec_last = S.ru0;
    }
}

template <int DIM, int OP, bool MR>
static const void *pcgx_fn_m(int depth) {
    switch (depth) {
        case 1: return (const void *)k_pcgx<DIM, OP, 1, CG_THREADS, MR>;
        case 2: return (const void *)k_pcgx<DIM, OP, 2, CG_THREADS, MR>;
        case 3: return (const void *)k_pcgx<DIM, OP, 3, CG_THREADS, MR>;
        default: return (const void *)k_pcgx<DIM, OP, 4, CG_THREADS, MR>;
    }
}
// (768-thread blocks -- 24 warps of 80 registers -- were measured and lost: C4 S_hat 394.6 vs 392.1 us/it)
// mr: the multi-rank instantiation (hierarchical barrier, vs_cg_common.cuh); the single-GPU one does not contain it
template <int DIM, int OP>
static const void *pcgx_fn_t(int depth, int mr) {
    return mr ? pcgx_fn_m<DIM, OP, true>(depth) : pcgx_fn_m<DIM, OP, false>(depth);
}
static const void *pcgx_fn(int dim, int op, int depth, int mr) {
    if (dim == 3) return op == 0 ? pcgx_fn_t<3, 0>(depth, mr) : pcgx_fn_t<3, 1>(depth, mr);
    return op == 0 ? pcgx_fn_t<2, 0>(depth, mr) : pcgx_fn_t<2, 1>(depth, mr);
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
    pl.smem = 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcgx_fn(dim, op, depth, 0), pl.threads, pl.smem);
    if (per_sm < 1) per_sm = 1;
    pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * nsm / groups, (m + pl.threads - 1) / pl.threads));
    pl.slots = 0;
    return pl;
}

cudaError_t launch_pcgx(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s) {
    P.cache_slots = 0;
    P.bpg = pl.grid;
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel(pcgx_fn(dim, op, pl.unroll, P.hier), dim3(pl.grid * groups), dim3(pl.threads), args,
                                       pl.smem, s);
}

}  // namespace vs
