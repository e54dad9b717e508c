// vs_cgb.cu -- k_pcgb: k_pcgm's qrec arithmetic (vs_cgm.cu) for the S_hat solve
// on a BLOCKED internal DOF order with the neighbour values staged in shared
// memory.
//
// Why it was built.  In the reference's packed order a DOF's x+- neighbours lie a
// whole plane away, so P1's gathers come from L2; a reading of the k_pcgm
// measurements suggested that those gathers cost as much as DRAM bytes.  Here
// the pressure DOFs are stored tile by tile -- a tile is TB x TB lines (x, y)
// with all their z -- and P1 works through one tile at a time: the tile's z
// values and the one-plane / one-line halos around it are copied into shared
// memory (each line padded with its own two ends, so that the periodic z wrap
// is index +-1 too), and all six neighbours of a DOF are shared-memory reads
// at tile-local distances held in the same 8-byte descriptor.
//
// What it showed.  Parity-green and 28 % slower than k_pcgm (B200, C4 512^3:
// 615 vs 482 us/it).  A later timing experiment (all gathers of k_pcgm redirected
// to the DOF's own index) put the whole cost of the gathers at 19 us of P1's
// 248: there was never more than 4 % to win here.  Kept as
// an opt-in experiment (VOXSCHUR_CG=6).
//
// Scope: S_hat (projected), 3D, one slab, n a multiple of TB; everything else
// keeps k_pcgm.  The vectors live in the blocked order for the length of one
// inner solve: the right-hand side is permuted in, the solution out.
#include "vs_cg_common.cuh"

namespace vs {

constexpr int TB = 8;                    // tile edge in lines
constexpr int TS = TB + 2;               // line slots per tile edge (halo included)
constexpr int NSLOT = TS * TS;           // 100
constexpr int BX = 13, BY = 10;          // descriptor fields (as in vs_cgm.cu)
constexpr uint32_t BXM = (1u << BX) - 1u, BYM = (1u << BY) - 1u;
constexpr int B_XP = 18, B_XM = B_XP + BX, B_YP = B_XM + BX, B_YM = B_YP + BY;

// 2-B code index (the six face codes in base 6; vs_cgm.cu)
__device__ __forceinline__ uint32_t blk_cidx(uint64_t rc) {
    uint32_t v = 0;
#pragma unroll
    for (int a = 2; a >= 0; --a) v = v * 6 + (uint32_t)rec_pout(rc, a);
#pragma unroll
    for (int a = 2; a >= 0; --a) v = v * 6 + (uint32_t)rec_pin(rc, a);
    return v;
}

// ---- build: per pressure DOF (reference rank i) its blocked rank, its index in
// the tile's shared-memory window, the window distances of its neighbours
__global__ void k_blk_build(const CgGroup G, int n, int nw, const uint32_t *lineR, const uint32_t *lineI,
                            const uint16_t *tl_v, uint64_t *desc, uint16_t *vidx, uint16_t *cidx, int *bad) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= G.m_own) return;
    const uint64_t rc = G.rec[i];
    uint32_t nr[6];
    neighbour_ranks<3, 1>(G.meta[0], nw, n, G.nx, rc, i, nr);
    const int x = rec_x(rc), y = rec_y(rc);
    const int nt = n / TB, t = (x / TB) * nt + (y / TB), px = x % TB, py = y % TB;
    const uint32_t kl = i - lineR[x * n + y];
    const uint32_t j = lineI[x * n + y] + kl;
    const uint16_t *tv = tl_v + (size_t)t * NSLOT;
    const int v = (int)tv[(px + 1) * TS + (py + 1)] + (int)kl;
    const int xp = (x + 1) % n, xm = (x + n - 1) % n, yp = (y + 1) % n, ym = (y + n - 1) % n;
    uint64_t dxp = 0, dxm = 0, dyp = 0, dym = 0;
    bool ok = true;
    if (nr[0] != ABSENT) {
        const int d = (int)tv[(px + 2) * TS + (py + 1)] + (int)(nr[0] - lineR[xp * n + y]) - v;
        ok &= d > 0 && d <= (int)BXM;
        dxp = (uint64_t)d;
    }
    if (nr[1] != ABSENT) {
        const int d = v - ((int)tv[px * TS + (py + 1)] + (int)(nr[1] - lineR[xm * n + y]));
        ok &= d > 0 && d <= (int)BXM;
        dxm = (uint64_t)d;
    }
    if (nr[2] != ABSENT) {
        const int d = (int)tv[(px + 1) * TS + (py + 2)] + (int)(nr[2] - lineR[x * n + yp]) - v;
        ok &= d > 0 && d <= (int)BYM;
        dyp = (uint64_t)d;
    }
    if (nr[3] != ABSENT) {
        const int d = v - ((int)tv[(px + 1) * TS + py] + (int)(nr[3] - lineR[x * n + ym]));
        ok &= d > 0 && d <= (int)BYM;
        dym = (uint64_t)d;
    }
    if (!ok) atomicExch(bad, 1);
    desc[j] = ((rc >> 40) & 0x3FFFFull) | (dxp << B_XP) | (dxm << B_XM) | (dyp << B_YP) | (dym << B_YM);
    vidx[j] = (uint16_t)v;
    cidx[j] = (uint16_t)blk_cidx(rc);
}

// reference order <-> blocked order
__global__ void k_blk_perm(const uint64_t *rec, int n, const uint32_t *lineR, const uint32_t *lineI, uint32_t m,
                           const double *in, double *out, int to_blocked) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t rc = rec[i];
    const int l = rec_x(rc) * n + rec_y(rc);
    const uint32_t j = lineI[l] + (i - lineR[l]);
    if (to_blocked) out[j] = in[i];
    else out[i] = in[j];
}

void launch_blk_build(const CgGroup &G, int n, int nw, const uint32_t *lineR, const uint32_t *lineI,
                      const uint16_t *tl_v, uint64_t *desc, uint16_t *vidx, uint16_t *cidx, int *bad, cudaStream_t s) {
    if (G.m_own) k_blk_build<<<(G.m_own + 255) / 256, 256, 0, s>>>(G, n, nw, lineR, lineI, tl_v, desc, vidx, cidx, bad);
}
void launch_blk_perm(const uint64_t *rec, int n, const uint32_t *lineR, const uint32_t *lineI, uint32_t m,
                     const double *in, double *out, int to_blocked, cudaStream_t s) {
    if (m) k_blk_perm<<<(m + 255) / 256, 256, 0, s>>>(rec, n, lineR, lineI, m, in, out, to_blocked);
}

// ---- the kernel -----------------------------------------------------------
// All vectors (rhs, x, z, d0, d1, q) are in the blocked order.
__global__ void __launch_bounds__(CG_THREADS, 1) k_pcgb(const CgParams P) {
    constexpr int NT = CG_THREADS;
    constexpr int KL = 4;
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
    extern __shared__ __align__(16) double dyn_v[];  // the tile window V[vcap], then the slot tables
    __shared__ double s_w[8];
    __shared__ double s_warp[NT / 32][5];
    __shared__ double s_tot[5];
    __shared__ __align__(16) double s_val[4][NT];  // grid_sum staging
    __shared__ CgGroup G;
    if (threadIdx.x == 0) G = P.groups[P.group_base];
    if (threadIdx.x < 8) s_w[threadIdx.x] = __dmul_rn(P.invA_enc[threadIdx.x], P.inv_h2);
    unsigned gen = __ldcg(P.bar_base);
    __syncthreads();
    double *V = dyn_v;
    const int nbuf = G.vbuf;  // 2 windows when they fit, else 1
    const uint32_t vstride = (uint32_t)G.vcap;
    uint32_t *s_src = reinterpret_cast<uint32_t *>(dyn_v + (size_t)nbuf * G.vcap);  // [2][NSLOT] each
    uint16_t *s_len = reinterpret_cast<uint16_t *>(s_src + 2 * NSLOT);
    uint16_t *s_vst = s_len + 2 * NSLOT;
    const double2 *ctab = P.ctab;
    __builtin_assume(__isGlobal(ctab));
    const uint32_t m = G.m_own;
    const uint32_t bl = blockIdx.x, nb = P.bpg;
    const uint32_t tid = bl * NT + threadIdx.x, stride = nb * NT;
    double *x = G.x, *z = G.z, *sv = G.q;
    const uint64_t *desc = G.desc;
    const uint16_t *cidx = G.cidx, *vidx = G.vidx;
    const uint32_t *tile0 = G.tile0;
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(z));
    __builtin_assume(__isGlobal(sv));
    __builtin_assume(__isGlobal(desc));
    __builtin_assume(__isGlobal(cidx));
    __builtin_assume(__isGlobal(vidx));
    __builtin_assume(__isGlobal(tile0));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pfd = P.pf_dist * stride;

    // ---- setup (krylov.py:102-119, x0 = 0): rhs -= mean; r = -rhs; z = M^-1 r
    double mu_rhs, mu, rz, rp0, ru0;
    {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], G.rhs[i]);
        grid_sum<1, false, NT>(v, 0, P, gen, s_val, s_tot);
        mu_rhs = v[0] / P.m_global;
    }
    {
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (uint32_t i = tid; i < m; i += stride) {
            const double2 t = __ldg(ctab + cidx[i]);
            x[i] = 0.0;
            const double ri = __dsub_rn(0.0, __dsub_rn(G.rhs[i], mu_rhs));
            const double zi = __dmul_rn(ri, t.x);
            z[i] = zi;
            v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
            v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
            v[2] = __dadd_rn(v[2], __dmul_rn(ri, ri));
            v[3] = __dadd_rn(v[3], zi);
            v[4] = __dadd_rn(v[4], ri);
        }
        grid_sum_shfl<5, true, NT>(v, 1, P, gen, s_warp, s_tot);
        mu = v[3] / P.m_global;
        rz = __dsub_rn(v[0], __dmul_rn(mu, v[4]));
        rp0 = sqrt(__dsub_rn(v[1], __dmul_rn(mu, v[3])));
        ru0 = sqrt(v[2]);
    }
    const double ref = rp0;
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
            __builtin_assume(__isGlobal(dold));
            __builtin_assume(__isGlobal(dnew));
            const bool first = it == 0;
            const uint64_t t0 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            // ---- P1, tile by tile: d = (z - mu) + beta d_old; s = M S_hat z + beta s_old; d.q
            double v1[1] = {0.0};
            // Two windows: while the block computes tile t out of one, the copies of its
            // next tile (t + nb) land in the other (cp.async, 8 B per lane: in flight
            // without registers; each thread waits for its own, the block barrier makes
            // them visible).
            auto load_tables = [&](uint32_t t, int b) {
                if (threadIdx.x < NSLOT) {
                    s_src[b * NSLOT + threadIdx.x] = G.tl_src[(size_t)t * NSLOT + threadIdx.x];
                    s_len[b * NSLOT + threadIdx.x] = G.tl_len[(size_t)t * NSLOT + threadIdx.x];
                    s_vst[b * NSLOT + threadIdx.x] = G.tl_v[(size_t)t * NSLOT + threadIdx.x];
                }
            };
            auto issue_copies = [&](int b) {  // every line slot, padded with the line's own two ends
                double *W = V + (size_t)b * vstride;
                for (int slot = warp; slot < NSLOT; slot += NT / 32) {
                    const uint32_t ln = s_len[b * NSLOT + slot];
                    if (!ln) continue;
                    const double *src = z + s_src[b * NSLOT + slot];
                    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(W + s_vst[b * NSLOT + slot]);
                    for (uint32_t e = lane; e < ln; e += 32)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + e * 8u), "l"(src + e) : "memory");
                    if (lane == 0)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst - 8u), "l"(src + ln - 1) : "memory");
                    if (lane == 1)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + ln * 8u), "l"(src) : "memory");
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            int buf = 0;
            if (bl < (uint32_t)G.ntiles) {
                load_tables(bl, 0);
                __syncthreads();
                issue_copies(0);
            }
            for (uint32_t t = bl; t < (uint32_t)G.ntiles; t += nb, buf ^= nbuf - 1) {
                const uint32_t tn = t + nb;
                const bool more = tn < (uint32_t)G.ntiles;
                const uint32_t T0 = tile0[t], len = tile0[t + 1] - T0;
                if (nbuf == 2) {
                    if (more) {
                        load_tables(tn, buf ^ 1);
                        __syncthreads();
                        issue_copies(buf ^ 1);
                        asm volatile("cp.async.wait_group 1;" ::: "memory");
                    } else {
                        asm volatile("cp.async.wait_group 0;" ::: "memory");
                    }
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                if (pfd && more) {  // the tile after the next one's z lines aside, the own streams -> L2
                    const uint32_t N0 = tile0[tn], nlen = tile0[tn + 1] - N0;
                    for (uint32_t k = threadIdx.x; k < nlen; k += NT) {
                        prefetch_l2(desc + N0 + k);
                        if (!first) {
                            prefetch_l2(dold + N0 + k);
                            prefetch_l2(sv + N0 + k);
                        }
                    }
                }
                __syncthreads();  // tile t's window is complete and visible
                const double *W = V + (size_t)buf * vstride;
                // the next step's own values are loaded a step ahead (issued before this
                // step's arithmetic, carried in registers)
                uint64_t dn_ = 0;
                uint32_t vn_ = 0;
                double dcn_ = 0.0, son_ = 0.0;
                if (threadIdx.x < len) {
                    const uint32_t i0 = T0 + threadIdx.x;
                    dn_ = __ldcs(desc + i0);
                    vn_ = vidx[i0];
                    if (!first) {
                        dcn_ = dold[i0];
                        son_ = sv[i0];
                    }
                }
                for (uint32_t k = threadIdx.x; k < len; k += NT) {
                    const uint32_t i = T0 + k;
                    const uint64_t d = dn_;
                    const uint32_t v = vn_;
                    const double dc = dcn_, so = son_;
                    if (k + NT < len) {
                        dn_ = __ldcs(desc + i + NT);
                        vn_ = vidx[i + NT];
                        if (!first) {
                            dcn_ = dold[i + NT];
                            son_ = sv[i + NT];
                        }
                    }
                    const double zc = W[v];
                    const double zxp = W[v + ((uint32_t)(d >> B_XP) & BXM)], zxm = W[v - ((uint32_t)(d >> B_XM) & BXM)];
                    const double zyp = W[v + ((uint32_t)(d >> B_YP) & BYM)], zym = W[v - ((uint32_t)(d >> B_YM) & BYM)];
                    const double zzp = W[v + 1], zzm = W[v - 1];
                    const uint32_t c = (uint32_t)d & 0x3FFFFu;
                    // S_hat z = sum_a (z_i - z_in) W_in - (z_out - z_i) W_out; an absent face has
                    // weight 0 (and, for x/y, distance 0: it reads the DOF itself)
                    double w = 0.0;
                    {
                        const double wi = __dmul_rn(__dsub_rn(zc, zxm), s_w[c & 7u]);
                        const double wo = __dmul_rn(__dsub_rn(zxp, zc), s_w[(c >> 9) & 7u]);
                        w = __dadd_rn(w, __dsub_rn(wi, wo));
                    }
                    {
                        const double wi = __dmul_rn(__dsub_rn(zc, zym), s_w[(c >> 3) & 7u]);
                        const double wo = __dmul_rn(__dsub_rn(zyp, zc), s_w[(c >> 12) & 7u]);
                        w = __dadd_rn(w, __dsub_rn(wi, wo));
                    }
                    {
                        const double wi = __dmul_rn(__dsub_rn(zc, zzm), s_w[(c >> 6) & 7u]);
                        const double wo = __dmul_rn(__dsub_rn(zzp, zc), s_w[(c >> 15) & 7u]);
                        w = __dadd_rn(w, __dsub_rn(wi, wo));
                    }
                    const double2 td = __ldg(P.sdiag2 + c);  // {1/diag, diag} by the 18-bit key
                    const double zp = __dsub_rn(zc, mu);
                    const double di = first ? zp : __dadd_rn(zp, __dmul_rn(beta, dc));
                    const double mw = __dmul_rn(w, td.x);
                    const double si = first ? mw : __dadd_rn(mw, __dmul_rn(beta, so));
                    dnew[i] = di;
                    sv[i] = si;
                    v1[0] = __dadd_rn(v1[0], __dmul_rn(di, __dmul_rn(td.y, si)));
                }
                if (nbuf == 1) {
                    __syncthreads();  // single window: everyone is done with it before the next copies
                    if (more) {
                        load_tables(tn, 0);
                        __syncthreads();
                        issue_copies(0);
                    }
                } else {
                    __syncthreads();  // this window is the target of the copies issued next round
                }
            }
            const uint64_t t1 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            grid_sum<1, false, NT>(v1, 2, P, gen, s_val, s_tot);
            const uint64_t t2 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            const double dq = v1[0];
            if (dq <= 0.0) { status = 2; sval = dq; sat = it; break; }
            const double alpha = rz / dq;
            // ---- P2: x -= alpha d; z -= alpha s; sums (a pure stream over the blocked order)
            double v[KL] = {0.0, 0.0, 0.0, 0.0};
            uint32_t cin_ = tid < m ? (uint32_t)__ldcs(cidx + tid) : 0u;
            for (uint32_t i = tid; i < m; i += stride) {
                const uint32_t ip = i + pfd;
                if (pfd && ip < m) {
                    prefetch_l2(dnew + ip);
                    prefetch_l2(sv + ip);
                    prefetch_l2(x + ip);
                    prefetch_l2(z + ip);
                }
                const uint32_t ci = cin_;
                const double2 t = __ldg(ctab + ci);
                if (i + stride < m) cin_ = (uint32_t)__ldcs(cidx + i + stride);
                const double di = dnew[i], si = sv[i], xo = x[i], zo = z[i];
                const double xi = __dsub_rn(xo, __dmul_rn(alpha, di));
                const double zi = __dsub_rn(zo, __dmul_rn(alpha, si));
                x[i] = xi;
                z[i] = zi;
                const double ri = __dmul_rn(t.y, zi);
                v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                v[2] = __dadd_rn(v[2], zi);
                v[3] = __dadd_rn(v[3], ri);
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
            mu = v[2] / P.m_global;
            const double rz_new = __dsub_rn(v[0], __dmul_rn(mu, v[3]));
            beta = rz_new / rz;
            rz = rz_new;
            const double nz = sqrt(__dsub_rn(v[1], __dmul_rn(mu, v[2])));
            if (!isfinite(nz)) { status = 3; sat = it + 1; break; }
            its = it + 1;
            rp_last = nz;
            double *tp = dold; dold = dnew; dnew = tp;
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
        *P.bar_base = gen;
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

size_t pcgb_smem(int vcap, int nbuf) { return (size_t)nbuf * vcap * sizeof(double) + 2 * NSLOT * (4 + 2 + 2); }

// windows that fit next to the kernel's static shared memory: 2, 1 or 0 (does not fit)
int pcgb_fits(int vcap, int device) {
    int maxopt = 0;
    cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, (const void *)k_pcgb);
    for (int nbuf = 2; nbuf >= 1; --nbuf)
        if (pcgb_smem(vcap, nbuf) + fa.sharedSizeBytes <= (size_t)maxopt) return nbuf;
    return 0;
}

cudaError_t launch_pcgb(const CgPlan &pl, CgParams &P, int vcap, int nbuf, cudaStream_t s) {
    P.cache_slots = 0;
    P.bpg = pl.grid;
    const size_t smem = pcgb_smem(vcap, nbuf);
    cudaError_t e = cudaFuncSetAttribute((const void *)k_pcgb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {&P};
    return cudaLaunchCooperativeKernel((const void *)k_pcgb, dim3(pl.grid), dim3(CG_THREADS), args, smem, s);
}

}  // namespace vs
