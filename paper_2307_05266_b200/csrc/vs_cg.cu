// vs_cg.cu -- K8: the fused persistent PCG of the inner solves (krylov.py:76-182).
//
// One cooperative launch runs a whole inner solve.  Per CG iteration:
//   P1  d = (z - mu) + beta d_old        (z stored by P2, mean-projected for S_hat)
//       q = op(d), neighbour d recomputed from z/d_old -> no extra pass
//       partial d.q                                              -> barrier 1
//   P2  x -= alpha d; r -= alpha q (q stored by P1: P2 is a pure stream, no
//       gathers or rank lookups); z = M^-1 r (stored);
//       partials r.z, z.z (+ sum z, sum r when projected)       -> barrier 2
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
// writes d, q; P2 reads d, q, x, r, record and writes x, r, z  -> 104 B (less
// whatever stays in L2 and the smem DOF cache), plus the L2-resident bitmask
// words for the neighbour ranks.  Storing q costs 16 B/DOF but halves the
// rank lookups and stencil work, which bound the passes (issue-bound at
// ~280 SASS instructions per DOF per pass before; 36 % of them rank lookups,
// ncu source counters, profiles/).
#include "vs_cg_common.cuh"

namespace vs {


// QR: q by recurrence, q = A(z - mu) + beta q_old (A applied to the projected
// z, then the reference's d-recurrence carried over to q by linearity; the
// same recurrence k_cg1 uses for s = M q).  P1 then gathers the neighbours'
// z only (6 loads instead of 12 in 3D) and reads its own q_old; neighbour d
// is never needed, so the ghost-plane d recompute goes too.  Rounding
// differs from q = A d at the last bits (not bitwise the reference's order).
// U (QR only): DOFs per step of P1's grid-stride loop; U = 2 issues both
// DOFs' loads before either's arithmetic (twice the independent load chains
// per thread).  The per-DOF arithmetic and the order of the d.q partial are
// unchanged, so U = 1 and U = 2 give bitwise the same results.
template <int DIM, int OP, int TIER, bool QR = false, int U_ = 1>
__global__ void __launch_bounds__(CG_THREADS, 1) k_pcg(const CgParams P) {
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
    constexpr int U = U_ > 0 ? U_ : 1;  // U_ == 0: P1 with carried delta words (TIER 4)
    constexpr bool PROJ = (OP == 1);
    constexpr int NS = 2 * DIM;
    extern __shared__ __align__(16) uint8_t dyn_smem[];
    __shared__ double s_tab[40];
    __shared__ double s_warp[CG_THREADS / 32][5];
    __shared__ double s_tot[5];
    __shared__ __align__(16) double s_val[4][CG_THREADS];  // grid_sum staging (32 KB)
    __shared__ CgGroup G;  // this block's slab (group)
    const int grp = P.group_base + blockIdx.x / P.bpg;
    if (threadIdx.x == 0) G = P.groups[grp];
    if (threadIdx.x < 16) {
        s_tab[threadIdx.x] = P.diag_code[threadIdx.x];
        s_tab[16 + threadIdx.x] = P.inv_code[threadIdx.x];
        if (threadIdx.x < 8) s_tab[32 + threadIdx.x] = P.invA_enc[threadIdx.x];
    }
    unsigned gen = __ldcg(P.bar_base);  // barrier target: where the previous launch left the counter
    const uint32_t kc = P.cache_slots;
    DofCache<DIM, OP, TIER> cache(dyn_smem, kc);
    __syncthreads();
    const Tabs T{s_tab, s_tab + 16, s_tab + 32, P.invS};
    const uint32_t m = G.m_own;       // owned DOFs of this slab
    const uint32_t m_all = G.m_all;   // + ghost-plane DOFs
    const int fam_p = 0;
    const uint32_t tid = (blockIdx.x % P.bpg) * CG_THREADS + threadIdx.x;
    const uint32_t stride = P.bpg * CG_THREADS;
    double *x = G.x, *r = G.r, *z = G.z, *q = G.q;
    const bool halo = G.zpeer[0] != nullptr;  // multi-slab run: ghost-plane exchange
    // pointers come from shared memory: tell the compiler they are global
    // (LDG/STG instead of generic LD/ST)
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(r));
    __builtin_assume(__isGlobal(z));
    __builtin_assume(__isGlobal(q));
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;

    // ---- setup (krylov.py:102-119): project rhs; r = op(x0) - rhs; z = M^-1 r;
    //      fill the DOF cache
    double mu_rhs = 0.0, mu = 0.0, rz = 0.0, rp0 = 0.0, ru0 = 0.0;
    if (PROJ) {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], G.rhs[i]);
        grid_sum<1, false>(v, 0, P, gen, s_val, s_tot);
        mu_rhs = v[0] / P.m_global;
    }
    {
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double *x0 = G.x0;
        uint32_t k = 0;
        for (uint32_t i = tid; i < m; i += stride, ++k) {
            const uint64_t rc = G.rec[i];
            uint32_t nr[NS];
            if (x0 || (TIER == 2 && k < kc))
                neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
            if (k < kc) cache.put(k, rc, nr);
            double ax = 0.0, xi = 0.0;
            if (x0) {
                xi = x0[i];
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) vn[s] = nr[s] != ABSENT ? x0[nr[s]] : 0.0;
                ax = op_value<DIM, OP>(rc, xi, vn, T, inv_h, inv_h2);
                if (x0 != x) x[i] = xi;
            } else {
                x[i] = 0.0;
            }
            const double b = PROJ ? __dsub_rn(G.rhs[i], mu_rhs) : G.rhs[i];
            const double ri = __dsub_rn(ax, b);
            const double zi = __dmul_rn(ri, jacobi_inv<OP>(rc, T));
            r[i] = ri;
            z[i] = zi;
            if (halo) halo_store(G, OP == 0 ? rec_comp(rc) : fam_p, i, zi);
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
            v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
            v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
            v[3] = __dadd_rn(v[3], zi);
            v[4] = __dadd_rn(v[4], ri);
        }
        grid_sum_shfl<5, true>(v, 1, P, gen, s_warp, s_tot);
        if (PROJ) {
            mu = v[3] / P.m_global;
            v[0] = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
            v[1] = __dsub_rn(v[1], __dmul_rn(mu, v[3]));
        }
        rz = v[0];
        rp0 = sqrt(v[1]);
        ru0 = sqrt(v[2]);
    }
    const double ref = rp0;  // inner solves: preconditioned norm (schur.py:207-210, :259-262)
    double beta = 0.0, rp_last = rp0, ru_last = ru0, sval = 0.0;
    int status = 0;
    int64_t sat = 0, its = 0;
    bool conv = (ref == 0.0);
    double *dold = G.d0, *dnew = G.d1;
    __builtin_assume(__isGlobal(dold));
    __builtin_assume(__isGlobal(dnew));
    unsigned long long ph[4] = {0, 0, 0, 0};  // this block's phase sums (thread 0)
    if (!conv) {
        for (int64_t it = 0; it < P.max_iter; ++it) {
            if (rz < 0.0) { status = 1; sval = rz; sat = it; break; }
            if (rz == 0.0) { conv = true; break; }
            if (P.xgpu && *P.xflag) { status = 4; sat = it; break; }  // a peer rank never arrived
            const uint64_t t0 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            // ---- P1: d = z - mu + beta d_old, q = op(d), d.q  (instantiated
            // separately for the first iteration, where d = z - mu)
            double v1[1] = {0.0};
            auto pass1 = [&](auto first_c) {
                const bool first = first_c;  // constant-folded for std::bool_constant
                uint32_t k = 0;
                for (uint32_t i = tid; i < m; i += stride, ++k) {
                    const uint32_t ip = i + P.pf_dist * stride;
                    if (P.pf_dist && ip < m) {  // stream the centre vectors pf_dist strides ahead
                        if (k + 2 >= kc) prefetch_l2(G.rec + ip);
                        prefetch_l2(z + ip);
                        if (!first) prefetch_l2(dold + ip);
                    }
                    double zc = z[i];
                    const double dc = first ? 0.0 : dold[i];
                    const double qo = (QR && !first) ? q[i] : 0.0;
                    uint64_t rc;
                    uint32_t nr[NS];
                    fetch_dof<DIM, OP, TIER>(P, G, cache, k, kc, i, rc, nr);
                    double zn[NS], dn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {  // unconditional loads (absent -> own index)
                        const uint32_t j = nr[s] != ABSENT ? nr[s] : i;
                        zn[s] = z[j];
                        dn[s] = (first || QR) ? 0.0 : dold[j];
                    }
                    if (PROJ) zc = __dsub_rn(zc, mu);
                    const double di = first ? zc : __dadd_rn(zc, __dmul_rn(beta, dc));
                    double vn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        double zj = zn[s];
                        if (PROJ) zj = __dsub_rn(zj, mu);
                        const double dj = (first || QR) ? zj : __dadd_rn(zj, __dmul_rn(beta, dn[s]));
                        // A needs 0.0 at absent slots (left fold); S_hat's absent faces
                        // carry weight 0.0 (op_value), so the clamped value is harmless
                        vn[s] = (OP == 0 && nr[s] == ABSENT) ? 0.0 : dj;
                    }
                    double qi;
                    if (QR) {
                        const double wi = op_value<DIM, OP>(rc, zc, vn, T, inv_h, inv_h2);
                        qi = first ? wi : __dadd_rn(wi, __dmul_rn(beta, qo));
                    } else {
                        qi = op_value<DIM, OP>(rc, di, vn, T, inv_h, inv_h2);
                    }
                    dnew[i] = di;
                    q[i] = qi;
                    v1[0] = __dadd_rn(v1[0], __dmul_rn(di, qi));
                }
                // ghost-plane d, recomputed exactly as the owning slab computes it
                // (QR reads neighbour z only)
                if (!QR)
                for (uint32_t i = m + tid; i < m_all; i += stride) {
                    double zc = z[i];
                    if (PROJ) zc = __dsub_rn(zc, mu);
                    dnew[i] = first ? zc : __dadd_rn(zc, __dmul_rn(beta, dold[i]));
                }
            };
            // P1 of the QR form: neighbour z only, U DOFs per step
            auto pass1q = [&](bool first) {
                uint32_t k = 0;
                for (uint32_t i0 = tid; i0 < m; i0 += U * stride, k += U) {
                    uint32_t ii[U], kk[U];
                    bool ok[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {  // a DOF past the end repeats DOF 0 (not stored)
                        ok[u] = (i0 + u * stride) < m;
                        ii[u] = ok[u] ? i0 + u * stride : i0;
                        kk[u] = ok[u] ? k + u : k;
                    }
                    const uint32_t ip = i0 + P.pf_dist * U * stride;
                    if (P.pf_dist && ip < m) {  // the own streams pf_dist steps ahead (L2, no registers)
                        prefetch_l2(z + ip);
                        if (!first) {
                            prefetch_l2(dold + ip);
                            prefetch_l2(q + ip);
                        }
                        if (k + U * P.pf_dist >= kc) prefetch_l2(G.rec + ip);
                        if (TIER == 4) {
                            prefetch_l2(reinterpret_cast<const int2 *>(G.nbr) + ip);
                            if (DIM == 3) prefetch_l2(reinterpret_cast<const short2 *>(G.nbr + 2 * (size_t)G.m_own) + ip);
                        }
                    }
                    double zc[U], dc[U], qo[U];
                    uint64_t rc[U];
                    uint32_t nr[U][NS];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        zc[u] = z[ii[u]];
                        dc[u] = first ? 0.0 : dold[ii[u]];
                        qo[u] = first ? 0.0 : q[ii[u]];
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) fetch_dof<DIM, OP, TIER>(P, G, cache, kk[u], kc, ii[u], rc[u], nr[u]);
                    double zn[U][NS];
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int s = 0; s < NS; ++s) zn[u][s] = z[nr[u][s] != ABSENT ? nr[u][s] : ii[u]];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (!ok[u]) break;
                        const double zp = PROJ ? __dsub_rn(zc[u], mu) : zc[u];
                        const double di = first ? zp : __dadd_rn(zp, __dmul_rn(beta, dc[u]));
                        double vn[NS];
#pragma unroll
                        for (int s = 0; s < NS; ++s) {
                            const double zj = PROJ ? __dsub_rn(zn[u][s], mu) : zn[u][s];
                            vn[s] = (OP == 0 && nr[u][s] == ABSENT) ? 0.0 : zj;
                        }
                        const double wi = op_value<DIM, OP>(rc[u], zp, vn, T, inv_h, inv_h2);
                        const double qi = first ? wi : __dadd_rn(wi, __dmul_rn(beta, qo[u]));
                        dnew[ii[u]] = di;
                        q[ii[u]] = qi;
                        v1[0] = __dadd_rn(v1[0], __dmul_rn(di, qi));
                    }
                }
            };
            // P1 of the QR form at TIER 4 with the next DOF's delta words and
            // record carried across the step (U == 0): the rank decode of a step
            // waits on nothing, and the gathers issue with the own loads
            auto pass1c = [&](bool first) {
                const int2 *xd = reinterpret_cast<const int2 *>(G.nbr);
                const short2 *yd = reinterpret_cast<const short2 *>(G.nbr + 2 * (size_t)G.m_own);
                __builtin_assume(__isGlobal(xd));
                __builtin_assume(__isGlobal(yd));
                const uint64_t *rec = G.rec;
                __builtin_assume(__isGlobal(rec));
                int2 dxn = make_int2(0, 0);
                short2 dyn = make_short2(0, 0);
                uint64_t rcn = 0;
                auto words = [&](uint32_t i, uint32_t kk) {
                    dxn = __ldcs(xd + i);
                    if (DIM == 3) dyn = __ldcs(yd + i);
                    rcn = kk < kc ? cache.rec[kk * CG_THREADS + threadIdx.x] : rec[i];
                };
                if (tid < m) words(tid, 0);
                uint32_t k = 0;
                for (uint32_t i = tid; i < m; i += stride, ++k) {
                    const uint32_t ip = i + P.pf_dist * stride;
                    if (P.pf_dist && ip < m) {
                        prefetch_l2(z + ip);
                        if (!first) {
                            prefetch_l2(dold + ip);
                            prefetch_l2(q + ip);
                        }
                        if (k + P.pf_dist >= kc) prefetch_l2(rec + ip);
                        prefetch_l2(xd + ip);
                        if (DIM == 3) prefetch_l2(yd + ip);
                    }
                    const int2 dx = dxn;
                    const short2 dy = dyn;
                    const uint64_t rc = rcn;
                    const double zc = z[i];
                    const double dc = first ? 0.0 : dold[i];
                    const double qo = first ? 0.0 : q[i];
                    uint32_t nr[NS];
                    if (dx.x == INT_MIN) {
                        neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
                    } else {
                        nr[0] = rec_has_nb<OP>(rc, 0) ? i + (uint32_t)dx.x : ABSENT;
                        nr[1] = rec_has_nb<OP>(rc, 1) ? i + (uint32_t)dx.y : ABSENT;
                        if (DIM == 3) {
                            nr[2] = rec_has_nb<OP>(rc, 2) ? i + (uint32_t)(int)dy.x : ABSENT;
                            nr[3] = rec_has_nb<OP>(rc, 3) ? i + (uint32_t)(int)dy.y : ABSENT;
                        }
                        nr[NS - 2] = rec_has_nb<OP>(rc, NS - 2) ? i + 1 : ABSENT;
                        nr[NS - 1] = rec_has_nb<OP>(rc, NS - 1) ? i - 1 : ABSENT;
                    }
                    double zn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) zn[s] = z[nr[s] != ABSENT ? nr[s] : i];
                    if (i + stride < m) words(i + stride, k + 1);
                    const double zp = PROJ ? __dsub_rn(zc, mu) : zc;
                    const double di = first ? zp : __dadd_rn(zp, __dmul_rn(beta, dc));
                    double vn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        const double zj = PROJ ? __dsub_rn(zn[s], mu) : zn[s];
                        vn[s] = (OP == 0 && nr[s] == ABSENT) ? 0.0 : zj;
                    }
                    const double wi = op_value<DIM, OP>(rc, zp, vn, T, inv_h, inv_h2);
                    const double qi = first ? wi : __dadd_rn(wi, __dmul_rn(beta, qo));
                    dnew[i] = di;
                    q[i] = qi;
                    v1[0] = __dadd_rn(v1[0], __dmul_rn(di, qi));
                }
            };
            // peeling the first iteration pays for S_hat (B200, C2: 63.8 -> 57.3
            // us/it) but not for A (131.5 -> 137 us/it: register allocation)
            if (QR && U_ == 0 && TIER == 4)
                pass1c(it == 0);
            else if (QR)
                pass1q(it == 0);
            else if (OP == 1 && it == 0)
                pass1(std::true_type{});
            else if (OP == 1)
                pass1(std::false_type{});
            else
                pass1(it == 0);
            const uint64_t t1 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            grid_sum<1, false>(v1, 2, P, gen, s_val, s_tot);
            const uint64_t t2 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            const double dq = v1[0];
            if (dq <= 0.0) { status = 2; sval = dq; sat = it; break; }
            const double alpha = rz / dq;
            // ---- P2: x -= alpha d; r -= alpha q; z = M^-1 r; sums
            // per-iteration sums: r.z, z.z (+ sum z, sum r when projected).
            // Inner solves stop on the preconditioned norm (schur.py:207-210),
            // so |r| is not needed: z = r * (positive finite inverse diagonal)
            // is non-finite exactly when r is, which keeps krylov.py:159-160.
            constexpr int KL = PROJ ? 4 : 2;
            double v[KL];
#pragma unroll
            for (int s = 0; s < KL; ++s) v[s] = 0.0;
            uint32_t k = 0;
            for (uint32_t i = tid; i < m; i += stride, ++k) {
                const uint32_t ip = i + P.pf_dist * stride;
                if (P.pf_dist && ip < m) {
                    if (k + 2 >= kc) prefetch_l2(G.rec + ip);
                    prefetch_l2(dnew + ip);
                    prefetch_l2(q + ip);
                    prefetch_l2(x + ip);
                    prefetch_l2(r + ip);
                }
                const double di = dnew[i], qi = q[i], xo = x[i], ro = r[i];
                uint64_t rc;
                if (k < kc) {
                    rc = cache.rec[k * CG_THREADS + threadIdx.x];
                } else {
                    const uint64_t *rec = G.rec;
                    __builtin_assume(__isGlobal(rec));
                    rc = rec[i];
                }
                const double xi = __dsub_rn(xo, __dmul_rn(alpha, di));
                const double ri = __dsub_rn(ro, __dmul_rn(alpha, qi));
                const double zi = __dmul_rn(ri, jacobi_inv<OP>(rc, T));
                x[i] = xi;
                r[i] = ri;
                z[i] = zi;
                if (halo) halo_store(G, OP == 0 ? rec_comp(rc) : fam_p, i, zi);
                v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                if (PROJ) {
                    v[2] = __dadd_rn(v[2], zi);
                    v[3] = __dadd_rn(v[3], ri);
                }
            }
            const uint64_t t3 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            grid_sum<KL, true>(v, 3, P, gen, s_val, s_tot);
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
            const double nz = sqrt(v[1]);
            if (!isfinite(nz)) { status = 3; sat = it + 1; break; }
            its = it + 1;
            rp_last = nz;
            double *t = dold; dold = dnew; dnew = t;
            if (nz / ref < P.tol) { conv = true; break; }
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
        o->res_unprec_last = ru_last;
    }
}

// ===================================================================
// k_cg1 -- the same Jacobi-PCG with ONE grid reduction per iteration
// (Chronopoulos-Gear form of krylov.py:76-182, M-scaled recurrences).
//
// The two-reduction loop above keeps the reference's exact elementwise
// operation order but pays two grid-wide sums per iteration (~2.5-4 us each
// on B200, tools/gridsum_ll.cu), which dominates small solves.  With
//   zr = M r (unprojected), z = zr - mu, w = A zr, u = M w, s = M q,
//   gamma = r.z, delta = z.w,
// the recurrences (exact arithmetic identical to the reference's CG)
//   beta_i  = gamma_i / gamma_{i-1},  alpha_i = gamma_i / (delta_i - beta_i gamma_i / alpha_{i-1})
//   d_i = z_i + beta_i d_{i-1},  s_i = u_i + beta_i s_{i-1}
//   x_{i+1} = x_i - alpha_i d_i,  zr_{i+1} = zr_i - alpha_i s_i
//   w_{i+1} = A zr_{i+1},  u_{i+1} = M w_{i+1}
// need the sums gamma_{i+1}, delta_{i+1}, |z_{i+1}| only after the pass
// that produces zr_{i+1}: one pass, one reduction.  A neighbour's zr_{i+1}
// is recomputed from its zr_i, u_i, s_{i-1} (no second pass; M of the
// neighbour is never needed because u and s are stored M-scaled).  For the
// projected S_hat solve, A annihilates constants, so w = A zr = A z and
// delta = zr.w - mu sum w; r = zr * diag(S_hat).
// zr, u, s are double-buffered (neighbours read the old values while the
// pass writes the new); x and d are per-DOF and updated in place.
// DRAM bytes per DOF per iteration: read x, d, zr, u, s; write x, d, zr,
// u, s -> 80 B (+ the record when not smem-cached).
// Parity: values and iteration counts agree with the reference's
// two-reduction form to rounding (tests/test_gpu_scale.py: counts within
// 2 %, solutions within 1e-8); elementwise order is no longer bitwise.
template <int DIM, int OP, int TIER, int NT>
__global__ void __launch_bounds__(NT, 1) k_cg1(const CgParams P) {
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
    constexpr int KS = PROJ ? 6 : 3;  // per-iteration sums
    extern __shared__ __align__(16) uint8_t dyn_smem[];
    __shared__ double s_tab[40];
    __shared__ double s_warp[NT / 32][5];
    __shared__ double s_tot[8];
    __shared__ CgGroup G;
    // dynamic smem: [grid-sum staging KS x NT doubles | DOF cache]
    double(*s_val)[NT] = reinterpret_cast<double(*)[NT]>(dyn_smem);
    if (threadIdx.x == 0) G = P.groups[P.group_base + blockIdx.x / P.bpg];
    if (threadIdx.x < 16) {
        s_tab[threadIdx.x] = P.diag_code[threadIdx.x];
        s_tab[16 + threadIdx.x] = P.inv_code[threadIdx.x];
        if (threadIdx.x < 8) s_tab[32 + threadIdx.x] = P.invA_enc[threadIdx.x];
    }
    unsigned ep = __ldcg(P.bar_base);
    const uint32_t kc = P.cache_slots;
    DofCache<DIM, OP, TIER, NT> cache(dyn_smem + cg1_stage_bytes(OP, NT), kc);
    __syncthreads();
    const Tabs T{s_tab, s_tab + 16, s_tab + 32, P.invS};
    const double2 *sdg = P.sdiag2;
    const uint32_t m = G.m_own;
    const uint32_t tid = (blockIdx.x % P.bpg) * NT + threadIdx.x;
    const uint32_t stride = P.bpg * NT;
    double *x = G.x, *dv = G.d0;
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(dv));
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;
    int cur = 0;  // zb/ub/sb[cur] hold zr_i, u_i, s_{i-1}
    auto buf = [&](double *const(&b)[2], int k) -> double * {
        double *p = b[k];
        __builtin_assume(__isGlobal(p));
        return p;
    };

    // ---- setup 1 (krylov.py:102-119): project rhs; r0 = op(x0) - rhs;
    //      zr0 = M r0; fill the DOF cache
    double mu_rhs = 0.0;
    if (PROJ) {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], G.rhs[i]);
        grid_sum<1, false, NT>(v, 0, P, ep, s_val, s_tot);
        mu_rhs = v[0] / P.m_global;
    }
    double mu, gamma, rp0, ru0;
    {
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double *x0 = G.x0;
        double *zr = buf(G.zb, 0);
        uint32_t k = 0;
        for (uint32_t i = tid; i < m; i += stride, ++k) {
            const uint64_t rc = G.rec[i];
            uint32_t nr[NS];
            if (x0 || (TIER == 2 && k < kc))
                neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), P.nw, P.n, G.nx, rc, i, nr);
            if (k < kc) cache.put(k, rc, nr);
            double ax = 0.0, xi = 0.0;
            if (x0) {
                xi = x0[i];
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) vn[s] = nr[s] != ABSENT ? x0[nr[s]] : 0.0;
                ax = op_value<DIM, OP>(rc, xi, vn, T, inv_h, inv_h2);
            }
            x[i] = xi;
            const double b = PROJ ? __dsub_rn(G.rhs[i], mu_rhs) : G.rhs[i];
            const double ri = __dsub_rn(ax, b);
            double inv, dg;
            inv_diag<OP>(rc, T, sdg, inv, dg);
            const double zi = __dmul_rn(ri, inv);
            zr[i] = zi;
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
            v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
            v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
            v[3] = __dadd_rn(v[3], zi);
            v[4] = __dadd_rn(v[4], ri);
        }
        grid_sum_shfl<5, true, NT>(v, 1, P, ep, s_warp, s_tot);
        mu = PROJ ? v[3] / P.m_global : 0.0;
        gamma = PROJ ? __dsub_rn(v[0], __dmul_rn(mu, v[4])) : v[0];
        rp0 = sqrt(PROJ ? __dsub_rn(v[1], __dmul_rn(mu, v[3])) : v[1]);
        ru0 = sqrt(v[2]);
    }
    // ---- setup 2: w0 = A zr0, u0 = M w0; delta0 = z0.w0
    double delta;
    {
        double v[2] = {0.0, 0.0};
        const double *zr = buf(G.zb, 0);
        double *u = buf(G.ub, 0);
        uint32_t k = 0;
        for (uint32_t i = tid; i < m; i += stride, ++k) {
            uint64_t rc;
            uint32_t nr[NS];
            fetch_dof<DIM, OP, TIER, NT>(P, G, cache, k, kc, i, rc, nr);
            const double zi = zr[i];
            double vn[NS];
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const uint32_t j = nr[s] != ABSENT ? nr[s] : i;
                const double zj = zr[j];
                vn[s] = (OP == 0 && nr[s] == ABSENT) ? 0.0 : zj;
            }
            const double w = op_value<DIM, OP>(rc, zi, vn, T, inv_h, inv_h2);
            double inv, dg;
            inv_diag<OP>(rc, T, sdg, inv, dg);
            u[i] = __dmul_rn(w, inv);
            v[0] = __dadd_rn(v[0], __dmul_rn(zi, w));
            v[1] = __dadd_rn(v[1], w);
        }
        grid_sum<2, true, NT>(v, 2, P, ep, s_val, s_tot);
        delta = PROJ ? __dsub_rn(v[0], __dmul_rn(mu, v[1])) : v[0];
    }
    const double ref = rp0;
    double gamma_prev = 0.0, alpha_prev = 0.0, rp_last = rp0, sval = 0.0;
    int status = 0;
    int64_t sat = 0, its = 0;
    bool conv = (ref == 0.0);
    unsigned long long ph[4] = {0, 0, 0, 0};
    if (!conv) {
        for (int64_t it = 0; it < P.max_iter; ++it) {
            if (gamma < 0.0) { status = 1; sval = gamma; sat = it; break; }
            if (gamma == 0.0) { conv = true; break; }
            if (P.xgpu && *P.xflag) { status = 4; sat = it; break; }  // a peer rank never arrived
            double beta, dq;
            if (it == 0) {
                beta = 0.0;
                dq = delta;
            } else {
                beta = gamma / gamma_prev;
                dq = __dsub_rn(delta, __dmul_rn(beta, gamma) / alpha_prev);
            }
            if (dq <= 0.0) { status = 2; sval = dq; sat = it; break; }
            const double alpha = gamma / dq;
            const uint64_t t0 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            double v[KS];
#pragma unroll
            for (int q = 0; q < KS; ++q) v[q] = 0.0;
            auto pass = [&](auto first_c) {
                constexpr bool first = decltype(first_c)::value;
                const double *zr = buf(G.zb, cur), *u = buf(G.ub, cur), *so = buf(G.sb, cur);
                double *zn_o = buf(G.zb, cur ^ 1), *un_o = buf(G.ub, cur ^ 1), *sn_o = buf(G.sb, cur ^ 1);
                uint32_t k = 0;
                for (uint32_t i = tid; i < m; i += stride, ++k) {
                    uint64_t rc;
                    uint32_t nr[NS];
                    fetch_dof<DIM, OP, TIER, NT>(P, G, cache, k, kc, i, rc, nr);
                    const double zc = zr[i], uc = u[i], xc = x[i];
                    const double sc = first ? 0.0 : so[i], dc = first ? 0.0 : dv[i];
                    double vn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {  // unconditional loads (absent -> own index)
                        const uint32_t j = nr[s] != ABSENT ? nr[s] : i;
                        const double zj = zr[j], uj = u[j];
                        const double sj = first ? uj : __dadd_rn(uj, __dmul_rn(beta, so[j]));
                        const double zn = __dsub_rn(zj, __dmul_rn(alpha, sj));
                        vn[s] = (OP == 0 && nr[s] == ABSENT) ? 0.0 : zn;
                    }
                    const double z0 = PROJ ? __dsub_rn(zc, mu) : zc;
                    const double di = first ? z0 : __dadd_rn(z0, __dmul_rn(beta, dc));
                    const double si = first ? uc : __dadd_rn(uc, __dmul_rn(beta, sc));
                    const double zi = __dsub_rn(zc, __dmul_rn(alpha, si));
                    const double w = op_value<DIM, OP>(rc, zi, vn, T, inv_h, inv_h2);
                    double inv, dg;
                    inv_diag<OP>(rc, T, sdg, inv, dg);
                    x[i] = __dsub_rn(xc, __dmul_rn(alpha, di));
                    dv[i] = di;
                    sn_o[i] = si;
                    zn_o[i] = zi;
                    un_o[i] = __dmul_rn(w, inv);
                    const double ri = __dmul_rn(zi, dg);
                    v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                    v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                    v[2] = __dadd_rn(v[2], __dmul_rn(zi, w));
                    if (PROJ) {
                        v[3] = __dadd_rn(v[3], zi);
                        v[4] = __dadd_rn(v[4], ri);
                        v[5] = __dadd_rn(v[5], w);
                    }
                }
            };
            if (it == 0)
                pass(std::true_type{});
            else
                pass(std::false_type{});
            const uint64_t t1 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            // consecutive grid sums must use different partial sets: a block that
            // is one pass ahead writes the next sum while a slow block may still
            // read this one (same set -> diverging scalars -> barrier deadlock)
            grid_sum<KS, true, NT>(v, 3 - (int)(it & 1), P, ep, s_val, s_tot);
            if (P.phase_ns && threadIdx.x == 0) {
                const uint64_t t2 = gtimer();
                ph[0] += t1 - t0;
                ph[1] += t2 - t1;
            }
            gamma_prev = gamma;
            alpha_prev = alpha;
            cur ^= 1;
            double nz2;
            if (PROJ) {
                mu = v[3] / P.m_global;
                gamma = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
                nz2 = __dsub_rn(v[1], __dmul_rn(mu, v[3]));
                delta = __dsub_rn(v[2], __dmul_rn(mu, v[5]));
            } else {
                gamma = v[0];
                nz2 = v[1];
                delta = v[2];
            }
            const double nz = sqrt(nz2);
            if (!isfinite(nz)) { status = 3; sat = it + 1; break; }
            its = it + 1;
            rp_last = nz;
            if (nz / ref < P.tol) { conv = true; break; }
        }
    }
    if (P.phase_ns && threadIdx.x == 0) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            if (blockIdx.x == 0) P.phase_ns[p] += ph[p];
            atomicMax(P.phase_ns + 4 + p, ph[p]);
            atomicAdd(P.phase_ns + 8 + p, ph[p]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *P.bar_base = ep;
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
__global__ void k_build_nbr(const CgGroup G, int n, int nw, uint32_t *out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.m_own) return;
    const uint64_t rc = G.rec[i];
    uint32_t nr[2 * DIM];
    neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), nw, n, G.nx, rc, i, nr);
#pragma unroll
    for (int s = 0; s < 2 * DIM; ++s) out[(size_t)s * G.m_own + i] = nr[s];
}
// TIER 4 table: neighbour ranks as deltas from the DOF's own rank -- x+/x-
// as int32 (always fit), y+/y- as int16; a DOF whose y-delta does not fit
// or whose z-neighbour wraps is flagged (x.x = INT_MIN) for the bitmask
// lookup.  Absent slots store 0 (the record's presence bits decide).
template <int DIM, int OP>
__global__ void k_build_dnb(const CgGroup G, int n, int nw, uint32_t *out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.m_own) return;
    const uint64_t rc = G.rec[i];
    uint32_t nr[2 * DIM];
    neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), nw, n, G.nx, rc, i, nr);
    auto delta = [&](int s) -> int64_t { return nr[s] == ABSENT ? 0 : (int64_t)nr[s] - (int64_t)i; };
    bool flag = (nr[2 * DIM - 2] != ABSENT && nr[2 * DIM - 2] != i + 1) ||
                (nr[2 * DIM - 1] != ABSENT && nr[2 * DIM - 1] != i - 1);
    int2 dx = make_int2((int)delta(0), (int)delta(1));
    if (DIM == 3) {
        const int64_t a = delta(2), b = delta(3);
        flag |= a < -32767 || a > 32767 || b < -32767 || b > 32767;
        reinterpret_cast<short2 *>(out + 2 * (size_t)G.m_own)[i] = make_short2((short)a, (short)b);
    }
    if (flag) dx.x = INT_MIN;
    reinterpret_cast<int2 *>(out)[i] = dx;
}

void launch_build_nbr(int dim, int op, const CgGroup &G, int n, int nw, uint32_t *out, cudaStream_t s,
                      int tier) {
    if (!G.m_own) return;
    const unsigned nb = (G.m_own + 255) / 256;
    if (tier == 4) {
        if (dim == 3)
            op == 0 ? k_build_dnb<3, 0><<<nb, 256, 0, s>>>(G, n, nw, out) : k_build_dnb<3, 1><<<nb, 256, 0, s>>>(G, n, nw, out);
        else
            op == 0 ? k_build_dnb<2, 0><<<nb, 256, 0, s>>>(G, n, nw, out) : k_build_dnb<2, 1><<<nb, 256, 0, s>>>(G, n, nw, out);
        return;
    }
    if (dim == 3)
        op == 0 ? k_build_nbr<3, 0><<<nb, 256, 0, s>>>(G, n, nw, out) : k_build_nbr<3, 1><<<nb, 256, 0, s>>>(G, n, nw, out);
    else
        op == 0 ? k_build_nbr<2, 0><<<nb, 256, 0, s>>>(G, n, nw, out) : k_build_nbr<2, 1><<<nb, 256, 0, s>>>(G, n, nw, out);
}

template <int DIM, int OP, int NT>
static const void *cg1_fn_t(int tier) {
    return tier == 3 ? (const void *)k_cg1<DIM, OP, 3, NT>
                     : (tier == 2 ? (const void *)k_cg1<DIM, OP, 2, NT> : (const void *)k_cg1<DIM, OP, 1, NT>);
}
template <int DIM, int OP>
static const void *pcg_fn_t(int tier, int alg, int nt, int u) {
    if (alg == CG_ONE_SUM) return nt == 512 ? cg1_fn_t<DIM, OP, 512>(tier) : cg1_fn_t<DIM, OP, CG_THREADS>(tier);
    if (tier == 4)
        return alg == CG_TWO_SUM_QREC ? (u == 0 ? (const void *)k_pcg<DIM, OP, 4, true, 0> : (const void *)k_pcg<DIM, OP, 4, true>)
                                      : (const void *)k_pcg<DIM, OP, 4>;
    if (alg == CG_TWO_SUM_QREC) {
        return tier == 3 ? (const void *)k_pcg<DIM, OP, 3, true>
                         : (tier == 2 ? (const void *)k_pcg<DIM, OP, 2, true> : (const void *)k_pcg<DIM, OP, 1, true>);
    }
    return tier == 3 ? (const void *)k_pcg<DIM, OP, 3>
                     : (tier == 2 ? (const void *)k_pcg<DIM, OP, 2> : (const void *)k_pcg<DIM, OP, 1>);
}
static const void *pcg_fn(int dim, int op, int tier, int alg, int nt, int u) {
    if (dim == 3) return op == 0 ? pcg_fn_t<3, 0>(tier, alg, nt, u) : pcg_fn_t<3, 1>(tier, alg, nt, u);
    return op == 0 ? pcg_fn_t<2, 0>(tier, alg, nt, u) : pcg_fn_t<2, 1>(tier, alg, nt, u);
}

// Plan one launch: blocks per group (all groups co-resident on one device),
// cache tier and slots, smem.  m = the largest owned DOF count of a group.
CgPlan pcg_plan(int dim, int op, int64_t m, int groups, int device, int alg, int nbr_tier, int sms) {
    CgPlan pl{};
    pl.alg = alg;
    // P1 DOFs per step: 1.  (U = 2 -- both DOFs' loads issued first -- spills
    // 100-156 B at 64 registers: B200 C2 A 124.7 -> 130.6, S_hat 59.0 -> 63.8
    // us/it; the template keeps it for experiments.)
    pl.unroll = 1;
    // k_pcg_qrec at TIER 4 carries the next DOF's delta words across the P1
    // step (unroll 0; B200: C2 S_hat 56.3 -> 53.5, C4 512^3 651 -> 634 us/it,
    // despite 56-88 B of spills); VOXSCHUR_P1CARRY=0 turns it off
    if (alg == CG_TWO_SUM_QREC) {
        const char *e = getenv("VOXSCHUR_P1CARRY");
        if (!e || atoi(e) == 1) pl.unroll = 0;
    }
    // k_cg1 on the projected S_hat runs 512-thread blocks (B200, C1: 7.2 -> 6.1
    // us/it: half the block-stage work in its 6-component grid sum); the A
    // solve and k_pcg keep 1024 (k_pcg at 512: C2 S_hat 57 -> 83 us/it)
    int nt = (alg == CG_ONE_SUM && op == 1) ? 512 : CG_THREADS;
    if (const char *e = getenv("VOXSCHUR_CG1_THREADS"))
        if (alg == CG_ONE_SUM && (atoi(e) == 512 || atoi(e) == CG_THREADS)) nt = atoi(e);
    pl.threads = nt;
    int nsm = 0, maxopt = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (sms > 0 && sms < nsm) nsm = sms;  // a share of the device (concurrent solves)
    const int ns = 2 * dim;
    // nbr_tier: 0 (bitmask lookups), 3 (32-bit ranks in HBM), 4 (packed deltas;
    // k_pcg only)
    const int alt = (nbr_tier == 3 || (nbr_tier == 4 && alg != CG_ONE_SUM)) ? nbr_tier : 1;
    for (int tier : {2, alt}) {
        const void *fn = pcg_fn(dim, op, tier, alg, nt, pl.unroll);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, fn);  // static smem (grid_sum staging, tables)
        const size_t stage = alg == CG_ONE_SUM ? cg1_stage_bytes(op, nt) : 0;  // dynamic grid-sum staging
        size_t total = std::min<size_t>(CG_SMEM_BUDGET + stage, (size_t)maxopt - fa.sharedSizeBytes);
        if (const char *e = getenv("VOXSCHUR_SMEM_KB")) total = std::min<size_t>(total, (size_t)atoi(e) * 1024 + stage);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)total);
        const size_t budget = total - stage;  // DOF cache
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, total);
        if (per_sm < 1) per_sm = 1;
        int grid = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)per_sm * nsm / groups, (m + nt - 1) / nt));
        const int64_t stride = (int64_t)grid * nt;
        const int64_t slots = (m + stride - 1) / stride;
        const size_t per_slot = (size_t)nt * (tier == 2 ? 8 + 4 * ns : 8);
        if (tier == 2 && (size_t)slots * per_slot > budget) continue;
        pl.tier = tier;
        pl.grid = grid;
        pl.slots = (uint32_t)std::min<int64_t>(slots, (int64_t)(budget / per_slot));
        pl.smem = stage + pl.slots * per_slot;
        return pl;
    }
    return pl;
}

// launches `groups` x pl.grid blocks (one cooperative grid over all groups)
cudaError_t launch_pcg(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s) {
    P.cache_slots = pl.slots;
    P.bpg = pl.grid;
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel(pcg_fn(dim, op, pl.tier, pl.alg, pl.threads, pl.unroll), dim3(pl.grid * groups), dim3(pl.threads), args,
                                       pl.smem, s);
}

}  // namespace vs
