// vs_cgm.cu -- k_pcgm: the two-reduction inner PCG (krylov.py:76-182) in
// M-scaled form over 8-byte DOF descriptors -- the HBM-regime kernel.
//
// Why.  At 512^3 the two-reduction loop of vs_cg.cu (k_pcg<QR>, packed
// deltas) already streams at ~5.9 TB/s of DRAM (ncu, profiles/r02a_c4_full.txt)
// but moves 124 B per DOF per iteration against the 64-B algorithmic figure:
// x, r, z, d, q are all read and written, the 8-B record is read in both
// passes and the 12-B neighbour deltas in P1.  This kernel cuts the bytes:
//
//  * no r vector.  z = M r is the only residual stored: z -= alpha (M q)
//    (the recurrence k_cg1 already uses), r_i = diag_i z_i where a sum needs
//    it (r.z = sum diag z^2).  Rounding differs from r -= alpha q; z = M r in
//    the last bits; counts and solutions stay inside the parity bar.
//  * one 8-B descriptor per DOF replaces record + deltas (20 B): 18 bits of
//    integer codes (S_hat: the six 3-bit face codes; A: no-slip code,
//    neighbour presence, component), the x+- neighbour ranks as 13-bit
//    residuals against the base of the DOF's 1024-rank chunk (an int2 per
//    chunk, one warp-uniform load), the y+- ranks as 10-bit distances,
//    z+- = i +- 1.  A DOF whose deltas do
//    not fit, or whose z/y neighbour wraps, carries an escape mark and takes
//    the record + bitmask lookup of vs_cg_common.cuh (about 1 % at 512^3).
//  * two forms of the operator product:
//    RC = false ("qrec"): s = M q by recurrence, s = M A(z - mu) + beta s_old:
//         P1 reads z, d_old, s_old, descriptor and gathers 6 neighbour z;
//         P2 is a pure stream (d, s, x, z and a 2-B code index)  -> 98 B;
//    RC = true  ("rc"):  q = A d recomputed in both passes from the stored d
//         (bitwise the same value twice), nothing but x, z, d stored:
//         P1 reads z, d_old, descriptor (+ 12 gathers), writes d;
//         P2 reads d, x, z, descriptor (+ 6 gathers), writes x, z   -> 80 B.
//    Gathers are L1/L2 hits (a neighbour is at most one x-plane away, and the
//    grid sweeps the vectors front to back), so DRAM sees each value once.
//
// Everything else -- the persistent cooperative launch, the deterministic
// grid sums, the barrier, slab groups and ghost planes -- is vs_cg.cu's.
#include "vs_cg_common.cuh"
#include "vs_desc.cuh"

namespace vs {


// ---- descriptor build (once per context and operator) --------------------
// pass 1: the smallest x+ / x- rank distance inside every chunk (the bases
// the residuals are taken from)
template <int DIM, int OP>
__global__ void k_desc_scan(const CgGroup G, int n, int nw, int2 *xb) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // a warp lies inside one chunk
    int dp = INT_MAX, dm = INT_MAX;
    if (i < G.m_own) {
        const uint64_t rc = G.rec[i];
        uint32_t nr[2 * DIM];
        neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), nw, n, G.nx, rc, i, nr);
        if (nr[0] != ABSENT) dp = (int)(nr[0] - i);
        if (nr[1] != ABSENT) dm = (int)(nr[1] - i);
    }
    const int mp = __reduce_min_sync(~0u, dp), mm = __reduce_min_sync(~0u, dm);
    if ((threadIdx.x & 31) == 0 && i < G.m_own) {
        int *b = reinterpret_cast<int *>(xb + (i >> CHUNK_SHIFT));
        if (mp != INT_MAX) atomicMin(b, mp);
        if (mm != INT_MAX) atomicMin(b + 1, mm);
    }
}
// pass 2: pack
template <int DIM, int OP>
__global__ void k_desc_pack(const CgGroup G, int n, int nw, const int2 *xb, uint64_t *desc, uint16_t *cidx,
                            unsigned long long *n_escape, int force_escape, uint32_t *esc_tab, uint32_t esc_cap) {
    constexpr int NS = 2 * DIM;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.m_own) return;
    const uint64_t rc = G.rec[i];
    uint32_t nr[NS];
    neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), nw, n, G.nx, rc, i, nr);
    const int2 cb = xb[i >> CHUNK_SHIFT];
    bool esc = false;
    uint64_t ex0 = 0, ex1 = 0, dy0 = 0, dy1 = 0;
    if (nr[0] != ABSENT) {
        const int64_t e = (int64_t)(int)(nr[0] - i) - cb.x;
        if (e < 0 || e >= (int64_t)DX_ESC) esc = true; else ex0 = (uint64_t)e;
    }
    if (nr[1] != ABSENT) {
        const int64_t e = (int64_t)(int)(nr[1] - i) - cb.y;
        if (e < 0 || e > (int64_t)DX_MASK) esc = true; else ex1 = (uint64_t)e;
    }
    if (DIM == 3) {
        if (nr[2] != ABSENT) {
            const int64_t e = (int64_t)nr[2] - (int64_t)i;
            if (e < 1 || e > (int64_t)DY_MASK) esc = true; else dy0 = (uint64_t)e;
        }
        if (nr[3] != ABSENT) {
            const int64_t e = (int64_t)i - (int64_t)nr[3];
            if (e < 1 || e > (int64_t)DY_MASK) esc = true; else dy1 = (uint64_t)e;
        }
    }
    if (nr[NS - 2] != ABSENT && nr[NS - 2] != i + 1) esc = true;
    if (nr[NS - 1] != ABSENT && nr[NS - 1] != i - 1) esc = true;
    if (force_escape) esc = true;  // test hook: every DOF through the record + bitmask lookup
    if (esc) {
        ex0 = DX_ESC;
        const unsigned long long e = atomicAdd(n_escape, 1ull);
        ex1 = dy0 = dy1 = 0;
        if (esc_tab && e < esc_cap) {  // the gather indices, for k_pcgx (slot order is arbitrary, the content is not)
            uint32_t *t = esc_tab + 8 * e;
#pragma unroll
            for (int s = 0; s < 8; ++s) t[s] = (s < NS && nr[s] != ABSENT) ? nr[s] : i;
            ex1 = e + 1;  // bits SH_EORD.. (33 bits)
        }
    }
    desc[i] = rec_codes<OP>(rc) | (ex0 << SH_XP) | (ex1 << SH_XM) | (dy0 << SH_YP) | (dy1 << SH_YM);
    cidx[i] = (uint16_t)rec_cidx<DIM, OP>(rc);
}
// {1/diag, diag} by code index
__global__ void k_build_ctab(int op, const double2 *sdiag2, const double *diag_code, double2 *ctab, int count) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    if (op == 0) {
        const double d = diag_code[k & 15];
        ctab[k] = make_double2(d != 0.0 ? 1.0 / d : 0.0, d);  // krylov.py:213
        return;
    }
    uint32_t v = (uint32_t)k, key = 0;
    for (int f = 0; f < 6; ++f) {
        key |= (v % 6u) << (3 * f);
        v /= 6u;
    }
    ctab[k] = sdiag2[key];
}

void launch_desc_scan(int dim, int op, const CgGroup &G, int n, int nw, int2 *xb, cudaStream_t s) {
    if (!G.m_own) return;
    const unsigned nb = (G.m_own + 255) / 256;
    if (dim == 3)
        op == 0 ? k_desc_scan<3, 0><<<nb, 256, 0, s>>>(G, n, nw, xb) : k_desc_scan<3, 1><<<nb, 256, 0, s>>>(G, n, nw, xb);
    else
        op == 0 ? k_desc_scan<2, 0><<<nb, 256, 0, s>>>(G, n, nw, xb) : k_desc_scan<2, 1><<<nb, 256, 0, s>>>(G, n, nw, xb);
}
void launch_desc_pack(int dim, int op, const CgGroup &G, int n, int nw, const int2 *xb, uint64_t *desc,
                      uint16_t *cidx, unsigned long long *n_escape, uint32_t *esc_tab, uint32_t esc_cap,
                      cudaStream_t s) {
    if (!G.m_own) return;
    const unsigned nb = (G.m_own + 255) / 256;
    const char *ee = getenv("VOXSCHUR_DESC_ESCAPE");  // test hook: 1 = mark every DOF as an escape
    const int fe = ee && atoi(ee) == 1;
    if (dim == 3)
        op == 0 ? k_desc_pack<3, 0><<<nb, 256, 0, s>>>(G, n, nw, xb, desc, cidx, n_escape, fe, esc_tab, esc_cap)
                : k_desc_pack<3, 1><<<nb, 256, 0, s>>>(G, n, nw, xb, desc, cidx, n_escape, fe, esc_tab, esc_cap);
    else
        op == 0 ? k_desc_pack<2, 0><<<nb, 256, 0, s>>>(G, n, nw, xb, desc, cidx, n_escape, fe, esc_tab, esc_cap)
                : k_desc_pack<2, 1><<<nb, 256, 0, s>>>(G, n, nw, xb, desc, cidx, n_escape, fe, esc_tab, esc_cap);
}
void launch_build_ctab(int op, const double2 *sdiag2, const double *diag_code, double2 *ctab, int count,
                       cudaStream_t s) {
    k_build_ctab<<<(count + 255) / 256, 256, 0, s>>>(op, sdiag2, diag_code, ctab, count);
}

// ---- the kernel -----------------------------------------------------------
template <int DIM, int OP, bool RC, int NT>
__global__ void __launch_bounds__(NT, 1) k_pcgm(const CgParams P) {
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
    __shared__ double s_tab[48];  // [40..47]: S_hat face weights times inv_h^2 (qrec form)
    __shared__ double s_warp[NT / 32][5];
    __shared__ double s_tot[5];
    __shared__ __align__(16) double s_val[4][NT];  // grid_sum staging
    __shared__ CgGroup G;
    const int grp = P.group_base + blockIdx.x / P.bpg;
    if (threadIdx.x == 0) G = P.groups[grp];
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
    const uint32_t m = G.m_own, m_all = G.m_all;
    const uint32_t blk0 = (blockIdx.x % P.bpg) * NT;  // first DOF of this block's chunk in stride 0
    const uint32_t tid = blk0 + threadIdx.x;
    const uint32_t stride = P.bpg * NT;
    double *x = G.x, *z = G.z, *sv = G.q;
    const uint64_t *desc = G.desc;
    const uint16_t *cidx = G.cidx;
    const uint64_t *rec = G.rec;
    const int2 *xb = G.xb;
    const bool halo = G.zpeer[0] != nullptr;
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(z));
    __builtin_assume(__isGlobal(sv));
    __builtin_assume(__isGlobal(desc));
    __builtin_assume(__isGlobal(cidx));
    __builtin_assume(__isGlobal(rec));
    __builtin_assume(__isGlobal(xb));
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pfd = P.pf_dist * stride;

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
    // warp w covers half (w & 1) of stream (w >> 1) -- one instruction per thread
    // and step instead of one per thread and stream (sh = log2 of the element size)
    auto prefetch_chunk = [&](uint32_t c0, const void *base, int sh) {
        const uint32_t per_line = 128u >> sh;
        const uint32_t i = c0 + ((uint32_t)(warp & 1) * 32u + (uint32_t)lane) * per_line;
        if (base && i < c0 + NT && i < m) {
            const char *p = reinterpret_cast<const char *>(base) + ((size_t)i << sh);
            if (P.dbg & 2u)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
            else
                prefetch_l2(p);
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
            // ---- P1: d = (z - mu) + beta d_old; d.q  (the first iteration,
            // where d = z - mu and nothing old is read, is its own instantiation)
            double v1[1] = {0.0};
            auto pass1 = [&](auto first_c) {
                constexpr bool first = decltype(first_c)::value;
                // this warp's prefetch stream: z, descriptors, d_old (, s_old)
                const int ps = warp >> 1;
                const void *pfb = ps == 0 ? (const void *)z
                                : ps == 1 ? (const void *)desc
                                : (!first && ps == 2) ? (const void *)dold
                                : (!first && !RC && ps == 3) ? (const void *)sv : nullptr;
                // the next step's descriptor and chunk base, carried across the step
                uint64_t dn_ = 0;
                int2 cbn_ = make_int2(0, 0);
                if (tid < m) {
                    dn_ = __ldcs(desc + tid);
                    cbn_ = __ldg(xb + (tid >> CHUNK_SHIFT));
                }
                uint32_t c0 = blk0;
                for (uint32_t i = tid; i < m; i += stride, c0 += stride) {
                    if (pfd) prefetch_chunk(c0 + pfd, pfb, 3);
                    const uint64_t d = dn_;
                    const int2 cb = cbn_;
                    if (i + stride < m) {  // issued first: a whole step to arrive
                        dn_ = __ldcs(desc + i + stride);
                        cbn_ = __ldg(xb + ((i + stride) >> CHUNK_SHIFT));
                    }
                    const double zc = z[i];
                    const double dc = first ? 0.0 : dold[i];
                    const double so = (RC || first) ? 0.0 : sv[i];
                    uint64_t rc;
                    uint32_t j[NS], pres;
                    decode(d, i, cb, rc, j, pres);
                    double zn[NS], dn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        zn[s] = z[j[s]];
                        dn[s] = (RC && !first) ? dold[j[s]] : 0.0;
                    }
                    const double zp = PROJ ? __dsub_rn(zc, mu) : zc;
                    const double di = first ? zp : __dadd_rn(zp, __dmul_rn(beta, dc));
                    double vn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        // qrec S_hat: the stencil takes differences only, so mu cancels
                        double zj = (PROJ && RC) ? __dsub_rn(zn[s], mu) : zn[s];
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
                        double w;
                        if (OP == 1) {
                            // S_hat z = sum_a (z_i - z_in) W_in - (z_out - z_i) W_out with the
                            // face weights pre-multiplied by inv_h^2 (schur.py:234-240 up to
                            // rounding: this form is M-scaled, not bitwise the reference's)
                            w = 0.0;
#pragma unroll
                            for (int a = 0; a < DIM; ++a) {
                                const double wi = __dmul_rn(__dsub_rn(zc, vn[2 * a + 1]), wS[rec_pin(rc, a)]);
                                const double wo = __dmul_rn(__dsub_rn(vn[2 * a], zc), wS[rec_pout(rc, a)]);
                                w = __dadd_rn(w, __dsub_rn(wi, wo));
                            }
                        } else {
                            w = op_value<DIM, OP>(rc, zp, vn, T, inv_h, inv_h2);
                        }
                        const double mw = __dmul_rn(w, inv);
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
                int2 cbn_ = make_int2(0, 0);
                if (tid < m) {
                    dn_ = __ldcs(desc + tid);
                    cbn_ = __ldg(xb + (tid >> CHUNK_SHIFT));
                }
                uint32_t c0 = blk0;
                for (uint32_t i = tid; i < m; i += stride, c0 += stride) {
                    if (pfd) prefetch_chunk(c0 + pfd, pfb, 3);
                    const uint64_t d = dn_;
                    const int2 cb = cbn_;
                    if (i + stride < m) {
                        dn_ = __ldcs(desc + i + stride);
                        cbn_ = __ldg(xb + ((i + stride) >> CHUNK_SHIFT));
                    }
                    const double di = dnew[i], xo = x[i], zo = z[i];
                    uint64_t rc;
                    uint32_t j[NS], pres;
                    decode(d, i, cb, rc, j, pres);
                    double vn[NS];
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        const double dj = dnew[j[s]];
                        vn[s] = (OP == 0 && !((pres >> s) & 1u)) ? 0.0 : dj;
                    }
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
                // a pure stream, not issue-bound: every thread prefetches its own next
                // elements (B200, C4 512^3: the one-line-per-lane bursts of P1 cost this
                // pass 70 us/it -- hints issued in bursts are dropped under load)
                uint32_t cin_ = tid < m ? (uint32_t)__ldcs(cidx + tid) : 0u;  // the next step's code index, carried
                for (uint32_t i = tid; i < m; i += stride) {
                    const uint32_t ip = i + pfd;
                    if (pfd && ip < m) {
                        prefetch_l2(dnew + ip);
                        prefetch_l2(sv + ip);
                        prefetch_l2(x + ip);
                        prefetch_l2(z + ip);
                    }
                    const uint32_t ci = cin_;
                    const double2 t = __ldg(ctab + (OP == 0 ? (ci & 0xFFu) : ci));  // no load ahead of this lookup
                    if (i + stride < m) cin_ = (uint32_t)__ldcs(cidx + i + stride);
                    const double di = dnew[i], si = sv[i], xo = x[i], zo = z[i];
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
static const void *pcgm_fn_t(bool rc, int nt) {
    if (nt == 512) return rc ? (const void *)k_pcgm<DIM, OP, true, 512> : (const void *)k_pcgm<DIM, OP, false, 512>;
    return rc ? (const void *)k_pcgm<DIM, OP, true, CG_THREADS> : (const void *)k_pcgm<DIM, OP, false, CG_THREADS>;
}
static const void *pcgm_fn(int dim, int op, bool rc, int nt) {
    if (dim == 3) return op == 0 ? pcgm_fn_t<3, 0>(rc, nt) : pcgm_fn_t<3, 1>(rc, nt);
    return op == 0 ? pcgm_fn_t<2, 0>(rc, nt) : pcgm_fn_t<2, 1>(rc, nt);
}

// Plan: one block per SM (per group); no dynamic shared memory.
CgPlan pcgm_plan(int dim, int op, int64_t m, int groups, int device, int alg, int sms) {
    CgPlan pl{};
    pl.alg = alg;
    pl.unroll = 1;
    pl.tier = 5;
    int nt = CG_THREADS;
    if (const char *e = getenv("VOXSCHUR_M_THREADS"))
        if (atoi(e) == 512 || atoi(e) == CG_THREADS) nt = atoi(e);
    pl.threads = nt;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    if (sms > 0 && sms < nsm) nsm = sms;
    const void *fn = pcgm_fn(dim, op, alg == CG_TWO_SUM_MRC, nt);  // CG_BLOCKED plans like the qrec form
    pl.smem = 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, pl.smem);
    if (per_sm < 1) per_sm = 1;
    if (const char *e = getenv("VOXSCHUR_M_BLOCKS_PER_SM"))
        if (atoi(e) >= 1 && atoi(e) < per_sm) per_sm = atoi(e);
    pl.grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * nsm / groups, (m + nt - 1) / nt));
    pl.slots = 0;
    return pl;
}

cudaError_t launch_pcgm(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s) {
    P.cache_slots = 0;
    P.bpg = pl.grid;
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel(pcgm_fn(dim, op, pl.alg == CG_TWO_SUM_MRC, pl.threads), dim3(pl.grid * groups),
                                       dim3(pl.threads), args, pl.smem, s);
}

}  // namespace vs
