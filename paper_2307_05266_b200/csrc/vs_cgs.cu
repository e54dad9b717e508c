// vs_cgs.cu -- k_pcgs: k_pcgm's arithmetic (vs_cgm.cu: M-scaled two-reduction
// PCG over 8-byte descriptors, "qrec" and "rc" forms) on an x-SWEEP schedule.
//
// Why.  k_pcgm visits its DOFs grid-stride (i = tid + k * stride): a block's
// consecutive chunks lie a whole stride apart, so every x+- neighbour it
// gathers was loaded by another SM and comes from L2 at L2 latency, in the
// middle of the step's dependent chain (ncu, profiles/r02d_c4_mq.txt: 57 %
// long-scoreboard stalls, and 335 warp instructions per 32 DOFs of which 28
// find the DOF's segment and 32 are per-thread prefetches).  Here the work is
// cut into units (component, strip j of S, plane x) -- strip j of a plane is
// the j-th S-th of its rank range, at most 1024 DOFs -- and a block owns a run
// of units with x running fastest: it sweeps its strip plane by plane.  The
// x+ neighbours a unit gathers are the own DOFs of the block's next unit and
// the x- neighbours those of its previous one, so after the first touch they
// are L1 hits on lines this SM loaded itself; each vector comes up from L2
// about once per pass.  The unit table ({first rank, length, segment, x+
// base, x- base}) sits in shared memory (no segment search), and the own
// ranges of the unit two steps ahead are prefetched to L2 by a few warps with
// one line per lane (no per-thread prefetch instructions).
//
// The schedule is static, so every sum is reduced in a fixed order:
// deterministic for a given grid, like every other fused CG here.
#include "vs_cg_common.cuh"

namespace vs {

constexpr int SW_NT = CG_THREADS;  // threads per block = DOFs per unit at most
constexpr int DXB = 13, DYB = 10;  // descriptor fields (vs_cgm.cu)
constexpr uint32_t DXM = (1u << DXB) - 1u, DYM = (1u << DYB) - 1u, DXE = DXM;
constexpr int S_XP = 18, S_XM = S_XP + DXB, S_YP = S_XM + DXB, S_YM = S_YP + DYB;

template <int OP>
__device__ __forceinline__ uint64_t sdesc_rec(uint64_t d) {
    const uint64_t c = d & 0x3FFFFull;
    if (OP == 1) return c << 40;
    return ((c & 0xF) << 36) | (((c >> 4) & 0x3F) << 40) | (((c >> 10) & 0x3) << 33);
}

template <int DIM, int OP, bool RC>
__global__ void __launch_bounds__(SW_NT, 1) k_pcgs(const CgParams P) {
    constexpr bool PROJ = (OP == 1);
    constexpr int NS = 2 * DIM;
    constexpr int NT = SW_NT;
    extern __shared__ __align__(16) uint8_t dyn_smem[];  // unit table
    __shared__ double s_tab[40];
    __shared__ double s_warp[NT / 32][5];
    __shared__ double s_tot[5];
    __shared__ __align__(16) double s_val[4][NT];  // grid_sum staging
    __shared__ CgGroup G;
    const int grp = P.group_base + blockIdx.x / P.bpg;
    if (threadIdx.x == 0) G = P.groups[grp];
    if (threadIdx.x < 16) {
        s_tab[threadIdx.x] = P.diag_code[threadIdx.x];
        s_tab[16 + threadIdx.x] = P.inv_code[threadIdx.x];
        if (threadIdx.x < 8) s_tab[32 + threadIdx.x] = P.invA_enc[threadIdx.x];
    }
    unsigned gen = __ldcg(P.bar_base);
    __syncthreads();
    // ---- this block's units: [u0, u1) of the group's U = nseg * S, x fastest
    uint4 *s_unit = reinterpret_cast<uint4 *>(dyn_smem);  // {first rank, length | segment << 16, x+ base, x- base}
    const uint32_t nxs = (uint32_t)G.nx, S = (uint32_t)G.nstrip;
    const uint32_t U = (uint32_t)G.nseg * S;
    const uint32_t bl = blockIdx.x % P.bpg;
    const uint32_t u0 = (uint32_t)(((uint64_t)U * bl) / P.bpg), u1 = (uint32_t)(((uint64_t)U * (bl + 1)) / P.bpg);
    const uint32_t nu = u1 - u0;
    for (uint32_t k = threadIdx.x; k < nu; k += NT) {
        const uint32_t u = u0 + k, x = u % nxs, t = u / nxs, j = t % S, c = t / S;
        const uint32_t seg = c * nxs + x;
        const uint32_t s0 = G.segstart[seg], L = G.segstart[seg + 1] - s0;
        const uint32_t a = s0 + (uint32_t)(((uint64_t)L * j) / S), b = s0 + (uint32_t)(((uint64_t)L * (j + 1)) / S);
        s_unit[k] = make_uint4(a, (b - a) | (seg << 16), (uint32_t)G.xp[seg], (uint32_t)G.xm[seg]);
    }
    __syncthreads();
    const Tabs T{s_tab, s_tab + 16, s_tab + 32, P.invS};
    const double2 *sdg = P.sdiag2;
    const double2 *ctab = P.ctab;
    __builtin_assume(__isGlobal(ctab));
    const uint32_t m = G.m_own, m_all = G.m_all;
    const uint32_t tid = bl * NT + threadIdx.x;
    const uint32_t stride = P.bpg * NT;
    double *x = G.x, *z = G.z, *sv = G.q;
    const uint64_t *desc = G.desc;
    const uint16_t *cidx = G.cidx;
    const uint64_t *rec = G.rec;
    const bool halo = G.zpeer[0] != nullptr;
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(z));
    __builtin_assume(__isGlobal(sv));
    __builtin_assume(__isGlobal(desc));
    __builtin_assume(__isGlobal(cidx));
    __builtin_assume(__isGlobal(rec));
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t PF = P.pf_dist;

    // descriptor -> record bits, gather indices (an absent neighbour reads the
    // DOF itself) and the presence mask (A zeroes absent slots)
    auto decode = [&](uint64_t d, uint32_t i, uint32_t xpb, uint32_t xmb, uint64_t &rc, uint32_t (&j)[NS],
                      uint32_t &pres) {
        const uint32_t fx = (uint32_t)(d >> S_XP) & DXM;
        if (fx == DXE) {  // escape: the record and the bitmask lookups
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
        rc = sdesc_rec<OP>(d);
        pres = 0;
#pragma unroll
        for (int s = 0; s < NS; ++s) pres |= (rec_has_nb<OP>(rc, s) ? 1u : 0u) << s;
        j[0] = (pres & 1u) ? i + xpb + fx : i;
        j[1] = (pres & 2u) ? i + xmb + ((uint32_t)(d >> S_XM) & DXM) : i;
        if (DIM == 3) {  // absent y slots carry distance 0
            j[2] = i + ((uint32_t)(d >> S_YP) & DYM);
            j[3] = i - ((uint32_t)(d >> S_YM) & DYM);
        }
        j[NS - 2] = i + ((pres >> (NS - 2)) & 1u);
        j[NS - 1] = i - ((pres >> (NS - 1)) & 1u);
    };
    // one L2 prefetch per lane, 128 B apart: warp w covers half (w & 1) of stream (w >> 1)
    // of the unit PF steps ahead (streams of 8-B elements; `sh` = 3, or 1 for the 2-B indices)
    auto prefetch_unit = [&](uint32_t k, const void *base, int sh) {
        if (k + PF < nu && base) {
            const uint4 e = s_unit[k + PF];
            const uint32_t per_line = 128u >> sh;
            const uint32_t off = ((uint32_t)(warp & 1) * 32u + (uint32_t)lane) * per_line;
            if (off < (e.y & 0xFFFFu)) prefetch_l2(reinterpret_cast<const char *>(base) + (((size_t)e.x + off) << sh));
        }
    };

    // ---- setup (krylov.py:102-119): project rhs; r = op(x0) - rhs; z = M^-1 r
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
            const double b = PROJ ? __dsub_rn(G.rhs[i], mu_rhs) : G.rhs[i];
            const double ri = __dsub_rn(ax, b);
            const double zi = __dmul_rn(ri, jacobi_inv<OP>(rc, T));
            z[i] = zi;
            if (halo) halo_store(G, OP == 0 ? rec_comp(rc) : 0, i, zi);
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
    double beta = 0.0, rp_last = rp0, sval = 0.0;
    int status = 0;
    int64_t sat = 0, its = 0;
    bool conv = (ref == 0.0);
    double *dold = G.d0, *dnew = G.d1;
    unsigned long long ph[4] = {0, 0, 0, 0};
    if (!conv) {
        for (int64_t it = 0; it < P.max_iter; ++it) {
            if (rz < 0.0) { status = 1; sval = rz; sat = it; break; }
            if (rz == 0.0) { conv = true; break; }
            if (P.xgpu && *P.xflag) { status = 4; sat = it; break; }  // a peer rank never arrived
            __builtin_assume(__isGlobal(dold));
            __builtin_assume(__isGlobal(dnew));
            const uint64_t t0 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            // ---- P1: d = (z - mu) + beta d_old; d.q
            double v1[1] = {0.0};
            auto pass1 = [&](auto first_c) {
                constexpr bool first = decltype(first_c)::value;
                // prefetch streams of this pass: z, descriptors, d_old (, s_old)
                const int ps = warp >> 1;
                const void *pfb = ps == 0 ? (const void *)z
                                : ps == 1 ? (const void *)desc
                                : (!first && ps == 2) ? (const void *)dold
                                : (!first && !RC && ps == 3) ? (const void *)sv : nullptr;
                uint64_t dn_ = 0;  // the next unit's descriptor, carried across the step
                if (nu) {
                    const uint4 e = s_unit[0];
                    if (threadIdx.x < (e.y & 0xFFFFu)) dn_ = __ldcs(desc + e.x + threadIdx.x);
                }
                for (uint32_t k = 0; k < nu; ++k) {
                    const uint4 e = s_unit[k];
                    if (PF) prefetch_unit(k, pfb, 3);
                    const bool live = threadIdx.x < (e.y & 0xFFFFu);
                    const uint32_t i = e.x + threadIdx.x;
                    const uint64_t d = dn_;
                    double zc = 0.0, dc = 0.0, so = 0.0;
                    uint64_t rc = 0;
                    uint32_t j[NS], pres = 0;
                    double zn[NS], dn[NS];
                    if (live) {
                        zc = z[i];
                        if (!first) dc = dold[i];
                        if (!RC && !first) so = sv[i];
                        decode(d, i, e.z, e.w, rc, j, pres);
#pragma unroll
                        for (int s = 0; s < NS; ++s) {
                            zn[s] = z[j[s]];
                            dn[s] = (RC && !first) ? dold[j[s]] : 0.0;
                        }
                    }
                    if (k + 1 < nu) {
                        const uint4 e2 = s_unit[k + 1];
                        if (threadIdx.x < (e2.y & 0xFFFFu)) dn_ = __ldcs(desc + e2.x + threadIdx.x);
                    }
                    if (!live) continue;
                    const double zp = PROJ ? __dsub_rn(zc, mu) : zc;
                    const double di = first ? zp : __dadd_rn(zp, __dmul_rn(beta, dc));
                    double vn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        double zj = PROJ ? __dsub_rn(zn[s], mu) : zn[s];
                        if (RC && !first) zj = __dadd_rn(zj, __dmul_rn(beta, dn[s]));
                        // A needs 0.0 at absent slots (left fold); S_hat's absent faces
                        // carry weight 0.0 (op_value), so the DOF's own value is harmless
                        vn[s] = (OP == 0 && !((pres >> s) & 1u)) ? 0.0 : zj;
                    }
                    dnew[i] = di;
                    if (RC) {
                        const double qi = op_value<DIM, OP>(rc, di, vn, T, inv_h, inv_h2);
                        v1[0] = __dadd_rn(v1[0], __dmul_rn(di, qi));
                    } else {
                        double inv, dg;
                        inv_diag<OP>(rc, T, sdg, inv, dg);
                        const double mw = __dmul_rn(op_value<DIM, OP>(rc, zp, vn, T, inv_h, inv_h2), inv);
                        const double si = first ? mw : __dadd_rn(mw, __dmul_rn(beta, so));
                        sv[i] = si;
                        v1[0] = __dadd_rn(v1[0], __dmul_rn(di, __dmul_rn(dg, si)));
                    }
                }
                // ghost-plane d, recomputed exactly as the owning slab computes it
                if (RC)
                    for (uint32_t i = m + tid; i < m_all; i += stride) {
                        double zc = z[i];
                        if (PROJ) zc = __dsub_rn(zc, mu);
                        dnew[i] = first ? zc : __dadd_rn(zc, __dmul_rn(beta, dold[i]));
                    }
            };
            if (it == 0)
                pass1(std::true_type{});
            else
                pass1(std::false_type{});
            const uint64_t t1 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            grid_sum<1, false, NT>(v1, 2, P, gen, s_val, s_tot);
            const uint64_t t2 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            const double dq = v1[0];
            if (dq <= 0.0) { status = 2; sval = dq; sat = it; break; }
            const double alpha = rz / dq;
            // ---- P2: x -= alpha d; z -= alpha M q; sums r.z = sum diag z^2, z.z
            // (+ sum z, sum r when projected)
            constexpr int KL = PROJ ? 4 : 2;
            double v[KL];
#pragma unroll
            for (int s = 0; s < KL; ++s) v[s] = 0.0;
            if (RC) {
                const int ps = warp >> 1;
                const void *pfb = ps == 0 ? (const void *)dnew : ps == 1 ? (const void *)desc
                                : ps == 2 ? (const void *)x : ps == 3 ? (const void *)z : nullptr;
                uint64_t dn_ = 0;
                if (nu) {
                    const uint4 e = s_unit[0];
                    if (threadIdx.x < (e.y & 0xFFFFu)) dn_ = __ldcs(desc + e.x + threadIdx.x);
                }
                for (uint32_t k = 0; k < nu; ++k) {
                    const uint4 e = s_unit[k];
                    if (PF) prefetch_unit(k, pfb, 3);
                    const bool live = threadIdx.x < (e.y & 0xFFFFu);
                    const uint32_t i = e.x + threadIdx.x;
                    const uint64_t d = dn_;
                    double di = 0.0, xo = 0.0, zo = 0.0, vn[NS];
                    uint64_t rc = 0;
                    uint32_t j[NS], pres = 0;
                    if (live) {
                        di = dnew[i];
                        xo = x[i];
                        zo = z[i];
                        decode(d, i, e.z, e.w, rc, j, pres);
#pragma unroll
                        for (int s = 0; s < NS; ++s) {
                            const double dj = dnew[j[s]];
                            vn[s] = (OP == 0 && !((pres >> s) & 1u)) ? 0.0 : dj;
                        }
                    }
                    if (k + 1 < nu) {
                        const uint4 e2 = s_unit[k + 1];
                        if (threadIdx.x < (e2.y & 0xFFFFu)) dn_ = __ldcs(desc + e2.x + threadIdx.x);
                    }
                    if (!live) continue;
                    double inv, dg;
                    inv_diag<OP>(rc, T, sdg, inv, dg);
                    const double qi = op_value<DIM, OP>(rc, di, vn, T, inv_h, inv_h2);
                    const double xi = __dsub_rn(xo, __dmul_rn(alpha, di));
                    const double zi = __dsub_rn(zo, __dmul_rn(alpha, __dmul_rn(qi, inv)));
                    x[i] = xi;
                    z[i] = zi;
                    if (halo) halo_store(G, OP == 0 ? rec_comp(rc) : 0, i, zi);
                    const double ri = __dmul_rn(dg, zi);
                    v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                    v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                    if (PROJ) {
                        v[2] = __dadd_rn(v[2], zi);
                        v[3] = __dadd_rn(v[3], ri);
                    }
                }
            } else {
                const int ps = warp >> 1;
                const void *pfb = ps == 0 ? (const void *)dnew : ps == 1 ? (const void *)sv
                                : ps == 2 ? (const void *)x : ps == 3 ? (const void *)z
                                : ps == 4 ? (const void *)cidx : nullptr;
                const int pfs = ps == 4 ? 1 : 3;
                for (uint32_t k = 0; k < nu; ++k) {
                    const uint4 e = s_unit[k];
                    if (PF) prefetch_unit(k, pfb, pfs);
                    if (threadIdx.x >= (e.y & 0xFFFFu)) continue;
                    const uint32_t i = e.x + threadIdx.x;
                    const double di = dnew[i], si = sv[i], xo = x[i], zo = z[i];
                    const uint32_t ci = __ldcs(cidx + i);
                    const double2 t = __ldg(ctab + (OP == 0 ? (ci & 0xFFu) : ci));
                    const double xi = __dsub_rn(xo, __dmul_rn(alpha, di));
                    const double zi = __dsub_rn(zo, __dmul_rn(alpha, si));
                    x[i] = xi;
                    z[i] = zi;
                    if (halo) halo_store(G, OP == 0 ? (int)(ci >> 8) : 0, i, zi);
                    const double ri = __dmul_rn(t.y, zi);
                    v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                    v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                    if (PROJ) {
                        v[2] = __dadd_rn(v[2], zi);
                        v[3] = __dadd_rn(v[3], ri);
                    }
                }
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
        o->res_unprec_last = ru0;
    }
}

template <int DIM, int OP>
static const void *pcgs_fn_t(bool rc) {
    return rc ? (const void *)k_pcgs<DIM, OP, true> : (const void *)k_pcgs<DIM, OP, false>;
}
static const void *pcgs_fn(int dim, int op, bool rc) {
    if (dim == 3) return op == 0 ? pcgs_fn_t<3, 0>(rc) : pcgs_fn_t<3, 1>(rc);
    return op == 0 ? pcgs_fn_t<2, 0>(rc) : pcgs_fn_t<2, 1>(rc);
}

// Plan: one block per SM (per group); the unit table (16 B per unit of the
// block's run) in dynamic smem.  units_max = the largest nseg * nstrip of a group.
CgPlan pcgs_plan(int dim, int op, int64_t m, int groups, int device, int alg, int64_t units_max, int sms) {
    CgPlan pl{};
    pl.alg = alg;
    pl.unroll = 1;
    pl.tier = 5;
    pl.threads = SW_NT;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    if (sms > 0 && sms < nsm) nsm = sms;
    pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm / groups, (m + SW_NT - 1) / SW_NT));
    pl.smem = (size_t)(units_max / pl.grid + 2) * sizeof(uint4);
    pl.slots = 0;
    return pl;
}

// false: the unit table of a block does not fit shared memory
bool pcgs_fits(int dim, int op, const CgPlan &pl, int device) {
    int maxopt = 0;
    cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, pcgs_fn(dim, op, pl.alg == CG_SWEEP_MRC));
    return pl.smem + fa.sharedSizeBytes <= (size_t)maxopt;
}

cudaError_t launch_pcgs(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s) {
    P.cache_slots = 0;
    P.bpg = pl.grid;
    const void *fn = pcgs_fn(dim, op, pl.alg == CG_SWEEP_MRC);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel(fn, dim3(pl.grid * groups), dim3(pl.threads), args, pl.smem, s);
}

}  // namespace vs
