// vs_cgt.cu -- k_cg1t: the one-reduction fused PCG of vs_cg.cu (k_cg1's
// arithmetic, krylov.py:76-182 in Chronopoulos-Gear form) with every
// neighbour value staged in shared memory.
//
// Why: the gather form (k_pcg / k_cg1) is latency-bound on B200 -- a
// chain record -> bitmask word -> 12-18 scattered loads per DOF with 64
// registers per thread keeps too few loads in flight (ncu, C2: 41 % issue
// active, 62 % long-scoreboard stalls, DRAM at 41 % of peak).
//
// Layout.  The DOFs of a family are packed in (x, y, z) order, z fastest, so
// the own lines [ya, ya + H) of plane x together with one halo line on each
// side are ONE contiguous rank run (two across the periodic y wrap).  A
// block owns units (family, line range, plane run) and sweeps its planes in
// x.  An NSLOT-slot ring in shared memory holds, per plane, that window of
// zr = M r, u = M A zr, s = M q plus its bitmask words; planes x-1, x, x+1 are
// resident while plane x is computed and the next planes are in flight.
// Warp 0 is the producer: its lanes stream each window in with 16-B
// cp.async and arrive on the slot's "full" mbarrier; warps 1.. consume,
// reading neighbours from shared memory only (rank from the staged bitmask
// word + a per-slot offset), and release slots on an "empty" mbarrier.  The
// own-DOF streams (record, x, d) are read coalesced one plane ahead into
// registers.
//
// Bytes per DOF per iteration: window reads (3 x 8 B, ~1.3x for the halo
// lines, re-used for x-1/x+1 from shared memory), record/x/d reads (24 B),
// x/d/zr/u/s writes (40 B): ~88 B of DRAM traffic when nothing stays in L2.
#include <cstdio>
#include <vector>

#include "vs_cg_common.cuh"

namespace vs {

// threads per block of the tiled kernel: 512 leaves 128 registers per thread
// (1024 x 64 spilled the per-DOF state to local memory)
constexpr int TT = 512;
constexpr int TNJ = 2;  // own DOFs per consumer thread and plane (own slice <= (TT - 32) * TNJ)
constexpr int NSLOT = 8, LSLOT = 3;  // ring slots (planes x-1, x, x+1 in use, the rest in flight)
constexpr double OWN_TARGET = 0.8 * (TT - 32);  // own DOFs per plane the planner aims at

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// dynamic shared memory layout (byte offsets), identical on host and device
struct TileSmem {
    size_t own, meta, vd, desc, bar, total;
};
__host__ __device__ inline TileSmem tile_smem(uint32_t capg, uint32_t capo, uint32_t capm, uint32_t wlmax,
                                              uint32_t dmax) {
    TileSmem L{};
    L.own = (size_t)NSLOT * 3 * capg * 8;                   // ring: slots x window {zr, u, s}
    L.meta = L.own + (size_t)NSLOT * 3 * capo * 8;          // ring: slots x own {rec, x, d}
    L.vd = L.meta + (size_t)NSLOT * capm * 8;               // ring: slots x bitmask words
    L.desc = L.vd + 32;                                     // 4 slots x 2 piece offsets
    L.bar = L.desc + ((size_t)dmax * sizeof(PlaneDesc) + 15) / 16 * 16;
    L.total = L.bar + (2 * NSLOT + 1) * 8;
    return L;
}

template <int OP>
__global__ void __launch_bounds__(TT, 1) k_cg1t(const CgParams P, const TileParams TP) {
    constexpr int DIM = 3;
    constexpr bool PROJ = (OP == 1);
    constexpr int NS = 2 * DIM;
    constexpr int KS = PROJ ? 6 : 3;
    extern __shared__ __align__(128) uint8_t dyn[];
    __shared__ double s_tab[40];
    __shared__ double s_warp[TT / 32][5];
    __shared__ double s_tot[8];
    __shared__ CgGroup G;
    __shared__ TileUnit sU;
    const uint32_t capg = TP.capg, capm = TP.capm, wlmax = TP.wlmax;
    const TileSmem SL = tile_smem(capg, TP.capo, capm, wlmax, TP.dmax);
    const uint32_t capo = TP.capo;
    double *ring = reinterpret_cast<double *>(dyn);
    double *oring = reinterpret_cast<double *>(dyn + SL.own);  // slot q: rec | x | d, capo each
    uint2 *smeta = reinterpret_cast<uint2 *>(dyn + SL.meta);
    PlaneDesc *sdesc = reinterpret_cast<PlaneDesc *>(dyn + SL.desc);  // every descriptor of the block
    uint64_t *bars = reinterpret_cast<uint64_t *>(dyn + SL.bar);  // full[4], empty[4], descriptors
    double(*s_val)[TT] = reinterpret_cast<double(*)[TT]>(dyn);  // grid sums (ring idle)

    if (threadIdx.x == 0) {
        G = P.groups[0];
        for (int q = 0; q < NSLOT; ++q) {
            mbar_init(bars + q, 1);                   // full: the producer's expect_tx arrival + bytes
            mbar_init(bars + NSLOT + q, TT / 32 - 1); // empty: one arrival per consumer warp
        }
        mbar_init(bars + 2 * NSLOT, 1);               // the block's plane descriptors (one bulk copy)
        fence_async_smem();
    }
    if (threadIdx.x < 16) {
        s_tab[threadIdx.x] = P.diag_code[threadIdx.x];
        s_tab[16 + threadIdx.x] = P.inv_code[threadIdx.x];
        if (threadIdx.x < 8) s_tab[32 + threadIdx.x] = P.invA_enc[threadIdx.x];
    }
    unsigned gen = __ldcg(P.bar_base);
    __syncthreads();
    const Tabs T{s_tab, s_tab + 16, s_tab + 32, P.invS};
    const double2 *sdg = P.sdiag2;
    const uint32_t m = G.m_own;
    const uint32_t tid = blockIdx.x * TT + threadIdx.x;
    const uint32_t stride = gridDim.x * TT;
    const int n = P.n, nw = P.nw;
    double *x = G.x, *dv = G.d0;
    __builtin_assume(__isGlobal(x));
    __builtin_assume(__isGlobal(dv));
    const double inv_h = P.inv_h, inv_h2 = P.inv_h2;
    int cur = 0;
    auto buf = [&](double *const(&b)[2], int k) -> double * {
        double *p = b[k];
        __builtin_assume(__isGlobal(p));
        return p;
    };
    auto gdof = [&](uint32_t i, uint64_t &rc, uint32_t (&nr)[NS]) {
        const uint64_t *rec = G.rec;
        __builtin_assume(__isGlobal(rec));
        rc = rec[i];
        neighbour_ranks<DIM, OP>(family_meta<OP>(G, rc), nw, n, G.nx, rc, i, nr);
    };

    // ---- setup (as k_cg1, grid-strided with global gathers: once per solve)
    double mu_rhs = 0.0;
    if (PROJ) {
        double v[1] = {0.0};
        for (uint32_t i = tid; i < m; i += stride) v[0] = __dadd_rn(v[0], G.rhs[i]);
        grid_sum<1, false, TT>(v, 0, P, gen, s_val, s_tot);
        mu_rhs = v[0] / P.m_global;
    }
    double mu, gamma, rp0, ru0;
    {
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        const double *x0 = G.x0;
        double *zr = buf(G.zb, 0);
        for (uint32_t i = tid; i < m; i += stride) {
            uint64_t rc;
            uint32_t nr[NS];
            double ax = 0.0, xi = 0.0;
            if (x0) {
                gdof(i, rc, nr);
                xi = x0[i];
                double vn[NS];
#pragma unroll
                for (int s = 0; s < NS; ++s) vn[s] = nr[s] != ABSENT ? x0[nr[s]] : 0.0;
                ax = op_value<DIM, OP>(rc, xi, vn, T, inv_h, inv_h2);
            } else {
                rc = G.rec[i];
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
        grid_sum_shfl<5, true, TT>(v, 1, P, gen, s_warp, s_tot);
        mu = PROJ ? v[3] / P.m_global : 0.0;
        gamma = PROJ ? __dsub_rn(v[0], __dmul_rn(mu, v[4])) : v[0];
        rp0 = sqrt(PROJ ? __dsub_rn(v[1], __dmul_rn(mu, v[3])) : v[1]);
        ru0 = sqrt(v[2]);
    }
    double delta;
    {
        double v[2] = {0.0, 0.0};
        const double *zr = buf(G.zb, 0);
        double *u = buf(G.ub, 0);
        for (uint32_t i = tid; i < m; i += stride) {
            uint64_t rc;
            uint32_t nr[NS];
            gdof(i, rc, nr);
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
        grid_sum<2, true, TT>(v, 2, P, gen, s_val, s_tot);
        delta = PROJ ? __dsub_rn(v[0], __dmul_rn(mu, v[1])) : v[0];
    }

    // ---- the plane sweep: warp 0 stages planes, warps 1.. compute them
    // Ring protocol over a flat plane counter fc (continues across units and
    // iterations): plane f lives in slot f % NSLOT; full[slot] completes when
    // the producer's copies of f have landed (phase f / NSLOT), empty[slot]
    // when every consumer warp has released f.  Consumers release plane f
    // after computing plane f + 1, and the last two planes of a unit at its
    // end, so the producer runs up to NSLOT - 3 planes ahead of the slowest
    // warp.  (4 slots left one plane of lookahead: consumers waited 35 % of
    // the sweep for data and the producer 17 % for free slots, B200 C2.)
    const uint32_t ub0 = TP.blk_unit[blockIdx.x], ub1 = TP.blk_unit[blockIdx.x + 1];
    uint64_t *full = bars, *empty = bars + NSLOT, *dbar = bars + 2 * NSLOT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d0 = ub0 < ub1 ? TP.units[ub0].desc0 : 0u;  // the block's descriptors are contiguous
    if (ub0 < ub1 && threadIdx.x == 0) {
        const TileUnit Ul = TP.units[ub1 - 1];
        const unsigned bytes = ((Ul.desc0 + Ul.nplanes - d0) * (unsigned)sizeof(PlaneDesc) + 15u) & ~15u;
        mbar_expect(dbar, bytes);
        bulk_g2s(sdesc, TP.planes + d0, bytes, dbar);
    }
    if (ub0 < ub1) mbar_wait(dbar, 0);
    uint32_t fc = 0;  // flat plane counter (identical in every warp)
    // producer warp: stage plane descriptor D of family meta mf into slot q.
    // One cp.async.bulk per contiguous segment, issued by one lane each
    // (window zr, u, s and bitmask words per piece; own record, x, d), all
    // completing on full[q] through its transaction count.  (16-B cp.async
    // by the 32 lanes streamed at 2.9-4.9 TB/s with 4-8 KB per slot against
    // 5.0-7.1 TB/s for bulk copies: tools/ring_bench.cu.)
    auto issue = [&](const PlaneDesc &D, int npc, int pw1, const uint2 *mf, uint32_t q, const double *zr,
                     const double *u, const double *so, bool first_it) {
        const uint32_t o0 = D.own_start & ~1u;
        const uint32_t olen = D.own_len ? ((D.own_start + D.own_len + 1u) & ~1u) - o0 : 0u;
        const int nown = D.own_len ? (first_it ? 2 : 3) : 0;
        if (lane == 0) {
            unsigned bytes = nown * olen * 8u;
            for (int p = 0; p < npc; ++p) bytes += (3 * D.vlen[p] + D.mlen[p]) * 8u;
            mbar_expect(full + q, bytes);
        }
        __syncwarp();
        const int nseg = 4 * npc + nown;
        if (lane < nseg) {
            void *dst;
            const void *src;
            uint32_t bytes;
            if (lane < 4 * npc) {
                const int p = lane >> 2, v = lane & 3;
                if (v < 3) {
                    dst = ring + (size_t)(q * 3 + v) * capg + (p ? D.vlen[0] : 0u);
                    src = (v == 0 ? zr : (v == 1 ? u : so)) + D.vstart[p];
                    bytes = D.vlen[p] * 8u;
                } else {
                    dst = smeta + (size_t)q * capm + (size_t)(p ? pw1 : 0) * nw;
                    src = mf + D.mstart[p];
                    bytes = D.mlen[p] * 8u;
                }
            } else {
                const int v = lane - 4 * npc;
                dst = oring + (size_t)(q * 3 + v) * capo;
                src = v == 0 ? (const void *)(G.rec + o0) : (v == 1 ? (const void *)(x + o0) : (const void *)(dv + o0));
                bytes = olen * 8u;
            }
            if (bytes) bulk_g2s(dst, src, bytes, full + q);
        }
    };
    auto release = [&](uint32_t f) {  // consumer warp: done with plane f
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + (f & (NSLOT - 1)))) : "memory");
    };
    // ring offset of rank r in piece p of the slot of flat plane f (descriptor D)
    auto piece_base = [&](const PlaneDesc &D, uint32_t f, int p) -> uint32_t {
        const uint32_t q = f & (NSLOT - 1);
        return p == 0 ? q * 3 * capg - D.vstart[0] : q * 3 * capg + D.vlen[0] - D.vstart[1];
    };
    unsigned long long tw = 0, tis = 0;  // phase timing: consumer waits / producer waits (thread 0, 32)

    const double ref = rp0;
    double gamma_prev = 0.0, alpha_prev = 0.0, rp_last = rp0, sval = 0.0;
    int status = 0;
    int64_t sat = 0, its = 0;
    bool conv = (ref == 0.0);
    unsigned long long phn[4] = {0, 0, 0, 0};
    if (!conv) {
        for (int64_t it = 0; it < P.max_iter; ++it) {
            if (gamma < 0.0) { status = 1; sval = gamma; sat = it; break; }
            if (gamma == 0.0) { conv = true; break; }
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
            const double *zr = buf(G.zb, cur), *u = buf(G.ub, cur), *so = buf(G.sb, cur);
            double *zn_o = buf(G.zb, cur ^ 1), *un_o = buf(G.ub, cur ^ 1), *sn_o = buf(G.sb, cur ^ 1);
            if (warp == 0) {
                // the previous iteration's stores (ordered by the grid barrier) and
                // the grid-sum staging in the ring (generic) precede these copies
                asm volatile("fence.proxy.async;" ::: "memory");
                for (uint32_t un = ub0; un < ub1; ++un) {
                    const TileUnit U = TP.units[un];
                    const uint2 *mf = OP == 1 ? G.meta[0] : G.meta[U.fam];
                    for (int k = 0; k < U.nplanes; ++k, ++fc) {
                        if (fc >= NSLOT) {  // slot reuse: every consumer warp released plane fc - NSLOT
                            const uint64_t a0 = (P.phase_ns && lane == 0) ? gtimer() : 0;
                            mbar_wait(empty + (fc & (NSLOT - 1)), ((fc - NSLOT) >> LSLOT) & 1u);
                            if (P.phase_ns && lane == 0) tis += gtimer() - a0;
                        }
                        issue(sdesc[U.desc0 - d0 + k], U.npc, U.pwl1, mf, fc & (NSLOT - 1), zr, u, so, it == 0);
                    }
                }
            } else {
                const uint32_t ct = threadIdx.x - 32;  // consumer thread
                auto sweep = [&](auto first_c) {
                    constexpr bool first = decltype(first_c)::value;
                    for (uint32_t un = ub0; un < ub1; ++un) {
                        const TileUnit U = TP.units[un];
                        const int nplanes = U.nplanes, ya = U.ya, wrapw = U.wrap, pwl1 = U.pwl1;
                        const PlaneDesc *Ds = sdesc + (U.desc0 - d0);
                        const uint32_t f0 = fc;
                        auto wait_full = [&](uint32_t f) {
                            const uint64_t a0 = (P.phase_ns && threadIdx.x == 32) ? gtimer() : 0;
                            mbar_wait(full + (f & (NSLOT - 1)), (f >> LSLOT) & 1u);
                            if (P.phase_ns && threadIdx.x == 32) tw += gtimer() - a0;
                        };
                        wait_full(f0);
                        wait_full(f0 + 1);
                        for (int k = 1; k + 1 < nplanes; ++k) {
                            wait_full(f0 + k + 1);
                            const uint32_t own_start = Ds[k].own_start, own_len = Ds[k].own_len;
                            const uint32_t fm = f0 + k - 1, fcur = f0 + k, fp = f0 + k + 1;
                            const uint32_t cm = fm & (NSLOT - 1), cc = fcur & (NSLOT - 1), cp = fp & (NSLOT - 1);
                            // own streams of this plane (slot cc): rank own_start + j at index j + ooff
                            const uint32_t ooff = own_start & 1u;
                            const uint64_t *orec = reinterpret_cast<const uint64_t *>(oring + (size_t)cc * 3 * capo);
                            const double *ox = oring + (size_t)cc * 3 * capo + capo, *od = ox + capo;
                            const uint32_t pb[3][2] = {{piece_base(Ds[k - 1], fm, 0), piece_base(Ds[k - 1], fm, 1)},
                                                       {piece_base(Ds[k], fcur, 0), piece_base(Ds[k], fcur, 1)},
                                                       {piece_base(Ds[k + 1], fp, 0), piece_base(Ds[k + 1], fp, 1)}};
#pragma unroll
                            for (int jj = 0; jj < TNJ; ++jj) {
                                const uint32_t j = ct + jj * (TT - 32);
                                if (j >= own_len) continue;
                                const uint64_t rc = orec[j + ooff];
                                const uint32_t i = own_start + j;
                                const int z = rec_z(rc), y = rec_y(rc);
                                const int w = z >> 5;
                                const uint32_t below = (1u << (z & 31)) - 1u;
                                const int wl = wrapw ? y : y - ya + 1;
                                // ring offset base of window line wl2 in slot position sp (0: x-1, 1: x, 2: x+1)
                                auto vdo = [&](int sp, int wl2) -> uint32_t { return pb[sp][wl2 >= pwl1 ? 1 : 0]; };
                                const uint32_t oc = i + vdo(1, wl);
                                // neighbour ring offsets first (independent), then every load, then the math
                                uint32_t o[NS];
#pragma unroll
                                for (int s = 0; s < 4; ++s) {  // x+, x-, y+, y-: bitmask word of the neighbour line
                                    const int sp = s == 0 ? 2 : (s == 1 ? 0 : 1);
                                    const uint32_t q = s == 0 ? cp : (s == 1 ? cm : cc);
                                    const int wl2 = s < 2 ? wl
                                                   : (s == 2 ? (wrapw && wl == n - 1 ? 0 : wl + 1)
                                                             : (wrapw && wl == 0 ? n - 1 : wl - 1));
                                    const uint2 mw = smeta[q * capm + wl2 * nw + w];
                                    o[s] = rec_has_nb<OP>(rc, s) ? mw.y + vdo(sp, wl2) + (uint32_t)__popc(mw.x & below)
                                                                 : oc;
                                }
#pragma unroll
                                for (int s = 4; s < 6; ++s) {  // z+, z-: the DOF's own line
                                    const bool up = (s == 4);
                                    uint32_t off = up ? oc + 1 : oc - 1;
                                    if (up ? (z == n - 1) : (z == 0)) {  // periodic wrap along the line
                                        const int zz = up ? 0 : n - 1;
                                        const uint2 mw = smeta[cc * capm + wl * nw + (zz >> 5)];
                                        off = mw.y + vdo(1, wl) + (uint32_t)__popc(mw.x & ((1u << (zz & 31)) - 1u));
                                    }
                                    o[s] = rec_has_nb<OP>(rc, s) ? off : oc;
                                }
                                const double zc = ring[oc], uc = ring[oc + capg];
                                const double sc = first ? 0.0 : ring[oc + 2 * capg];
                                double zj[NS], uj[NS], sj[NS];
#pragma unroll
                                for (int s = 0; s < NS; ++s) {
                                    zj[s] = ring[o[s]];
                                    uj[s] = ring[o[s] + capg];
                                    sj[s] = first ? 0.0 : ring[o[s] + 2 * capg];
                                }
                                const double z0 = PROJ ? __dsub_rn(zc, mu) : zc;
                                const double di = first ? z0 : __dadd_rn(z0, __dmul_rn(beta, od[j + ooff]));
                                const double si = first ? uc : __dadd_rn(uc, __dmul_rn(beta, sc));
                                const double zi = __dsub_rn(zc, __dmul_rn(alpha, si));
                                double vn[NS];
#pragma unroll
                                for (int s = 0; s < NS; ++s) {
                                    const double sn = first ? uj[s] : __dadd_rn(uj[s], __dmul_rn(beta, sj[s]));
                                    const double znj = __dsub_rn(zj[s], __dmul_rn(alpha, sn));
                                    vn[s] = (OP == 0 && !rec_has_nb<OP>(rc, s)) ? 0.0 : znj;
                                }
                                const double wv = op_value<DIM, OP>(rc, zi, vn, T, inv_h, inv_h2);
                                double inv, dg;
                                inv_diag<OP>(rc, T, sdg, inv, dg);
                                x[i] = __dsub_rn(ox[j + ooff], __dmul_rn(alpha, di));
                                dv[i] = di;
                                sn_o[i] = si;
                                zn_o[i] = zi;
                                un_o[i] = __dmul_rn(wv, inv);
                                const double ri = __dmul_rn(zi, dg);
                                v[0] = __dadd_rn(v[0], __dmul_rn(ri, zi));
                                v[1] = __dadd_rn(v[1], __dmul_rn(zi, zi));
                                v[2] = __dadd_rn(v[2], __dmul_rn(zi, wv));
                                if (PROJ) {
                                    v[3] = __dadd_rn(v[3], zi);
                                    v[4] = __dadd_rn(v[4], ri);
                                    v[5] = __dadd_rn(v[5], wv);
                                }
                            }
                            release(fm);
                        }
                        release(f0 + nplanes - 2);
                        release(f0 + nplanes - 1);
                        fc += nplanes;
                    }
                };
                if (it == 0)
                    sweep(std::true_type{});
                else
                    sweep(std::false_type{});
            }
            __syncthreads();  // the ring is idle: the grid sum stages through it
            const uint64_t t1 = (P.phase_ns && threadIdx.x == 0) ? gtimer() : 0;
            // alternate partial sets (see k_cg1): consecutive sums never share one
            grid_sum<KS, true, TT>(v, 3 - (int)(it & 1), P, gen, s_val, s_tot);
            if (P.phase_ns && threadIdx.x == 0) {
                const uint64_t t2 = gtimer();
                phn[0] += t1 - t0;
                phn[1] += t2 - t1;
                phn[3] = tis;  // producer lane 0: its waits on empty slots
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
    if (P.phase_ns && threadIdx.x == 32) phn[2] = tw;  // consumer thread 32: its waits on full slots
    if (P.phase_ns && (threadIdx.x == 0 || threadIdx.x == 32)) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            if ((p == 2) != (threadIdx.x == 32)) continue;
            if (blockIdx.x == 0) P.phase_ns[p] += phn[p];
            atomicMax(P.phase_ns + 4 + p, phn[p]);
            atomicAdd(P.phase_ns + 8 + p, phn[p]);
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

// ------------------------------------------------------------ planning
__global__ void k_line_stats(const uint2 *meta, int64_t nlines, int nw, uint32_t *cnt, uint32_t *start) {
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= nlines) return;
    const uint2 *mw = meta + l * nw;
    uint32_t c = 0;
    for (int w = 0; w < nw; ++w) c += __popc(mw[w].x);
    cnt[l] = c;
    start[l] = mw[0].y;
}

TilePlan tile_plan(int op, int n, int nw, int nfam, const uint2 *const *meta, const int64_t *m_fam, int device,
                   cudaStream_t s) {
    TilePlan TPl;
    if (n < 8 || (nw & 1) || nfam < 1) return TPl;
    int nsm = 0, maxopt = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const void *fn = op == 0 ? (const void *)k_cg1t<0> : (const void *)k_cg1t<1>;
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return TPl;
    const size_t limit = (size_t)maxopt - fa.sharedSizeBytes;
    const int64_t nl = (int64_t)n * n;
    // per-line DOF counts and first ranks of every family
    std::vector<std::vector<uint32_t>> cnt(nfam), lst(nfam);
    {
        uint32_t *d = nullptr;
        if (cudaMalloc(&d, 2 * nl * sizeof(uint32_t)) != cudaSuccess) return TPl;
        for (int f = 0; f < nfam; ++f) {
            cnt[f].resize(nl);
            lst[f].resize(nl);
            k_line_stats<<<(unsigned)((nl + 255) / 256), 256, 0, s>>>(meta[f], nl, nw, d, d + nl);
            cudaMemcpyAsync(cnt[f].data(), d, nl * 4, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(lst[f].data(), d + nl, nl * 4, cudaMemcpyDeviceToHost, s);
        }
        cudaStreamSynchronize(s);
        cudaFree(d);
        if (cudaGetLastError() != cudaSuccess) return TPl;
    }
    int64_t m_tot = 0;
    for (int f = 0; f < nfam; ++f) m_tot += m_fam[f];
    if (m_tot == 0) return TPl;
    // lines per unit: ~0.8 x TT x TNJ own DOFs per plane, shrunk until the ring fits
    double scale = 1.0;
    for (int attempt = 0; attempt < 24; ++attempt, scale *= 0.85) {
        int H[3];
        bool any_small = false;
        for (int f = 0; f < nfam; ++f) {
            const double L = std::max(1e-9, (double)m_fam[f] / (double)nl);
            int h = (int)std::lround(scale * OWN_TARGET / L);
            h = std::max(1, std::min(h, n));
            if (h >= n - 1) h = n;
            H[f] = h;
            any_small |= (h < 1);
        }
        if (any_small) break;
        // slices (family, line range, plane) in order, with their DOF counts
        struct Col { int f, ya, yb; };
        std::vector<Col> cols;
        for (int f = 0; f < nfam; ++f) {  // equal line ranges (sizes differ by at most one line)
            const int nyr = (n + H[f] - 1) / H[f], base = n / nyr, rem = n % nyr;
            for (int r = 0, ya = 0; r < nyr; ++r) {
                const int h = base + (r < rem ? 1 : 0);
                cols.push_back({f, ya, ya + h});
                ya += h;
            }
        }
        auto own_cnt = [&](const Col &c, int x) {
            uint64_t t = 0;
            for (int y = c.ya; y < c.yb; ++y) t += cnt[c.f][(int64_t)x * n + y];
            return t;
        };
        // cut the slice list into nsm chunks of equal DOFs -> units
        std::vector<TileUnit> units;
        std::vector<uint32_t> blk(nsm + 1, 0);
        std::vector<PlaneDesc> planes;
        uint32_t capg = 2, capo = 2, wlmax = 1, dmax = 1;
        bool fail = false;
        // chunk cost: own DOFs + a per-plane step overhead (sync, issue, halo)
        constexpr double PLANE_COST = 256.0;
        double c_tot = 0.0;
        for (const Col &c : cols)
            for (int x = 0; x < n; ++x) c_tot += (double)own_cnt(c, x) + PLANE_COST;
        const double per = c_tot / nsm;
        int b = 0;
        double acc = 0.0;
        auto end_line = [&](int f, int x, int y) -> uint32_t {  // rank one past line (x, y)
            return lst[f][(int64_t)x * n + y] + cnt[f][(int64_t)x * n + y];
        };
        auto add_unit = [&](const Col &c, int x0, int x1) {
            TileUnit U{};
            U.fam = c.f;
            U.ya = c.ya;
            U.wrap = (c.yb - c.ya == n) ? 1 : 0;
            const int P = x1 - x0 + 1;
            U.nplanes = P + 2;
            U.desc0 = (uint32_t)planes.size();
            int lo[2], hi[2];  // window pieces as line ranges (inclusive)
            if (U.wrap) {
                U.nwl = n;
                U.npc = 1;
                lo[0] = 0;
                hi[0] = n - 1;
            } else {
                U.nwl = c.yb - c.ya + 2;
                if (c.ya == 0) {
                    U.npc = 2;
                    lo[0] = hi[0] = n - 1;
                    lo[1] = 0;
                    hi[1] = c.yb;
                } else if (c.yb == n) {
                    U.npc = 2;
                    lo[0] = c.ya - 1;
                    hi[0] = n - 1;
                    lo[1] = hi[1] = 0;
                } else {
                    U.npc = 1;
                    lo[0] = c.ya - 1;
                    hi[0] = c.yb;
                }
            }
            U.pwl1 = U.npc == 2 ? hi[0] - lo[0] + 1 : U.nwl;
            for (int k = 0; k < U.nplanes; ++k) {
                const int xx = ((x0 - 1 + k) % n + n) % n;
                PlaneDesc D{};
                D.own_start = lst[c.f][(int64_t)xx * n + c.ya];
                D.own_len = (uint32_t)own_cnt(c, xx);
                if (k > 0 && k + 1 < U.nplanes) {
                    if (D.own_len > (uint32_t)((TT - 32) * TNJ)) fail = true;
                    capo = std::max(capo, (D.own_len + 3u) & ~1u);
                }
                uint32_t tot = 0;
                for (int p = 0; p < U.npc; ++p) {
                    const uint32_t r0 = lst[c.f][(int64_t)xx * n + lo[p]], r1 = end_line(c.f, xx, hi[p]);
                    D.vstart[p] = r0 & ~1u;
                    D.vlen[p] = ((r1 + 1u) & ~1u) - D.vstart[p];
                    D.mstart[p] = (uint32_t)(((int64_t)xx * n + lo[p]) * nw);
                    D.mlen[p] = (uint32_t)((hi[p] - lo[p] + 1) * nw);
                    tot += D.vlen[p];
                }
                capg = std::max(capg, (tot + 1u) & ~1u);
                planes.push_back(D);
            }
            wlmax = std::max<uint32_t>(wlmax, U.nwl);
            units.push_back(U);
        };
        for (const Col &c : cols) {
            int x0 = 0;
            for (int x = 0; x < n; ++x) {
                acc += (double)own_cnt(c, x) + PLANE_COST;
                // close this block's chunk once it reaches its share
                if (b < nsm - 1 && acc >= per * (b + 1)) {
                    add_unit(c, x0, x);
                    x0 = x + 1;
                    blk[++b] = (uint32_t)units.size();
                }
            }
            if (x0 < n) add_unit(c, x0, n - 1);
        }
        while (b < nsm) blk[++b] = (uint32_t)units.size();
        if (fail) continue;
        for (int bb = 0; bb < nsm; ++bb) {  // every descriptor of a block is resident
            uint32_t t = 0;
            for (uint32_t uu = blk[bb]; uu < blk[bb + 1]; ++uu) t += units[uu].nplanes;
            dmax = std::max(dmax, t);
        }
        const uint32_t capm = wlmax * nw;
        const TileSmem SL = tile_smem(capg, capo, capm, wlmax, dmax);
        if (SL.total > limit) continue;
        if ((size_t)NSLOT * 3 * capg * 8 < (size_t)(op == 1 ? 6 : 3) * TT * 8) capg = ((op == 1 ? 6 : 3) * TT / (3 * NSLOT) + 1) & ~1u;
        const TileSmem SL2 = tile_smem(capg, capo, capm, wlmax, dmax);
        if (SL2.total > limit) continue;
        if (getenv("VOXSCHUR_TILE_DEBUG")) {
            fprintf(stderr, "tile_plan op %d: H", op);
            for (int f = 0; f < nfam; ++f) fprintf(stderr, " %d", H[f]);
            fprintf(stderr, " capg %u capo %u wlmax %u dmax %u units %zu smem %zu\n", capg, capo, wlmax, dmax, units.size(),
                    tile_smem(capg, capo, capm, wlmax, dmax).total);
            for (int bb = 0; bb < nsm; bb += 1) {
                uint64_t dofs = 0, pl = 0, mx = 0;
                for (uint32_t u = blk[bb]; u < blk[bb + 1]; ++u) {
                    pl += units[u].nplanes;
                    for (int k = 1; k + 1 < units[u].nplanes; ++k) {
                        dofs += planes[units[u].desc0 + k].own_len;
                        mx = std::max<uint64_t>(mx, planes[units[u].desc0 + k].own_len);
                    }
                }
                if (bb < 4 || bb % 37 == 0 || bb == nsm - 1)
                    fprintf(stderr, "  blk %d: units %u planes %llu dofs %llu max_own %llu\n", bb, blk[bb + 1] - blk[bb],
                            (unsigned long long)pl, (unsigned long long)dofs, (unsigned long long)mx);
            }
        }
        // device copy: units | blk | planes (+1 slack descriptor for the 16-B rounded copy)
        const size_t bu = units.size() * sizeof(TileUnit), bb = blk.size() * 4,
                     bp = (planes.size() + 1) * sizeof(PlaneDesc);
        const size_t ou = 0, ob = (bu + 255) / 256 * 256, op_ = ob + (bb + 255) / 256 * 256;
        char *mem = nullptr;
        if (cudaMalloc(&mem, op_ + bp) != cudaSuccess) return TPl;
        planes.push_back(PlaneDesc{});
        cudaMemcpyAsync(mem + ou, units.data(), bu, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(mem + ob, blk.data(), bb, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(mem + op_, planes.data(), bp, cudaMemcpyHostToDevice, s);
        cudaStreamSynchronize(s);
        TPl.ok = true;
        TPl.grid = nsm;
        TPl.smem = SL2.total;
        for (int f = 0; f < nfam; ++f) TPl.H[f] = H[f];
        TPl.units = (int64_t)units.size();
        TPl.mem = mem;
        TPl.tp.units = (const TileUnit *)(mem + ou);
        TPl.tp.blk_unit = (const uint32_t *)(mem + ob);
        TPl.tp.planes = (const PlaneDesc *)(mem + op_);
        TPl.tp.capg = capg;
        TPl.tp.capo = capo;
        TPl.tp.capm = capm;
        TPl.tp.wlmax = wlmax;
        TPl.tp.dmax = dmax;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TPl.smem);
        return TPl;
    }
    return TPl;
}

cudaError_t launch_cg1t(int op, const TilePlan &tp, CgParams &P, cudaStream_t s) {
    TileParams T = tp.tp;
    P.bpg = tp.grid;
    P.cache_slots = 0;
    void *args[] = {&P, &T};
    const void *fn = op == 0 ? (const void *)k_cg1t<0> : (const void *)k_cg1t<1>;
    return cudaLaunchCooperativeKernel(fn, dim3(tp.grid), dim3(TT), args, tp.smem, s);
}

}  // namespace vs
