// vs_kernels.cu -- sm_100a kernels of the Schur-complement Stokes path.
//
//   K1  geometry build   (operators.py:232-297)  integer, bit-exact
//   K2-K6 operator applies (operators.py:131-206, schur.py:234-240) bit-exact
//   (K8, the fused persistent PCG, lives in vs_cg.cu)
//   outer-loop vector kernels + deterministic reductions (schur.py:291-385)
#include <cub/cub.cuh>

#include "vs_device.cuh"
#include "vs_internal.h"

namespace vs {

// ------------------------------------------------------------ K1 geometry

__device__ __forceinline__ Cell word_cell(const Geo &g, int64_t word, int b) {
    const int L = (int)(word / g.nw);
    const int w = (int)(word % g.nw);
    Cell c;
    if (g.dim == 3) { c.x = L / g.n; c.y = L % g.n; } else { c.x = L; c.y = 0; }
    c.z = w * 32 + b;
    return c;
}

__global__ void k_pack_fluid(const uint8_t *fluid, Geo g, int64_t nwords, uint32_t *fbits) {
    const int64_t word = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (word >= nwords) return;
    const int64_t L = word / g.nw;
    const int w = (int)(word % g.nw);
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b) {
        const int z = w * 32 + b;
        if (z < g.n && fluid[L * g.n + z]) bits |= 1u << b;
    }
    fbits[word] = bits;
}

// face (a, I) carries a DOF iff fluid[I] && fluid[I - e_a]  (operators.py:232)
__global__ void k_face_bits(Geo g, int a, int64_t nwords, uint32_t *out) {
    const int64_t word = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (word >= nwords) return;
    const int ia = iaxis(g.dim, a);
    uint32_t fb = g.fbits[word], bits = 0;
    while (fb) {
        const int b = __ffs(fb) - 1;
        fb &= fb - 1;
        const Cell c = word_cell(g, word, b);
        if (fluid_at(g, shifted(c, ia, -1, g))) bits |= 1u << b;
    }
    out[word] = bits;
}

__global__ void k_popc(const uint32_t *bits, int64_t nwords, uint32_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nwords) cnt[i] = __popc(bits[i]);
}

__global__ void k_make_meta(const uint32_t *bits, const uint32_t *base, uint32_t off,
                            int64_t nwords, uint2 *meta) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nwords) meta[i] = make_uint2(bits[i], base[i] + off);
}

// integer no-slip code of the existing face (a, c) (operators.py:268-281)
__device__ int face_code(const Geo &g, int a, Cell c) {
    const int ia = iaxis(g.dim, a);
    int code = 0;
    for (int d = 0; d < g.dim; ++d) {
        const int id = iaxis(g.dim, d);
        for (int si = 0; si < 2; ++si) {
            if (d == a) { code += 1; continue; }
            const Cell cn = shifted(c, id, si == 0 ? 1 : -1, g);
            const bool hi = fluid_at(g, cn);
            const bool lo = fluid_at(g, shifted(cn, ia, -1, g));
            const bool nb_face = hi && lo;
            code += (!nb_face && !hi && !lo) ? 2 : 1;
        }
    }
    return code;
}

__global__ void k_vel_records(Geo g, int a, int64_t nwords, uint64_t *rec) {
    const int64_t word = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (word >= nwords) return;
    const uint2 m = g.vmeta[a][word];
    uint32_t bits = m.x, k = 0;
    while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const Cell c = word_cell(g, word, b);
        const int code = face_code(g, a, c);
        // presence of the 2*dim same-component neighbour faces, slot order
        // (d, s = +1, -1) -> bits 40 + 2d + (s < 0) (the fused CG's rank lookups)
        uint64_t pres = 0;
        for (int dd = 0; dd < g.dim; ++dd)
            for (int si = 0; si < 2; ++si)
                if (rank_at(g.vmeta[a], g, shifted(c, iaxis(g.dim, dd), si == 0 ? 1 : -1, g)) != ABSENT)
                    pres |= 1ull << (40 + 2 * dd + si);
        rec[m.y + k] = make_rec(c.x, c.y, c.z, a) | ((uint64_t)code << 36) | pres;
        ++k;
    }
}

__global__ void k_p_records(Geo g, int64_t nwords, uint64_t *rec) {
    const int64_t word = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (word >= nwords) return;
    const uint2 m = g.pmeta[word];
    const int cbase = 2 * g.dim - 1;
    uint32_t bits = m.x, k = 0;
    while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const Cell c = word_cell(g, word, b);
        uint64_t r = make_rec(c.x, c.y, c.z, 0);
        for (int a = 0; a < g.dim; ++a) {
            const int ia = iaxis(g.dim, a);
            if (fluid_at(g, shifted(c, ia, -1, g)))
                r |= (uint64_t)(face_code(g, a, c) - cbase) << (40 + 3 * a);
            const Cell cp = shifted(c, ia, 1, g);
            if (fluid_at(g, cp))
                r |= (uint64_t)(face_code(g, a, cp) - cbase) << (49 + 3 * a);
        }
        rec[m.y + k] = r;
        ++k;
    }
}

__global__ void k_bits_to_u8(const uint2 *meta, const uint32_t *bits_plain, Geo g, int64_t ncells,
                             uint8_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ncells) return;
    const int64_t L = i / g.n;
    const int z = (int)(i % g.n);
    const uint32_t w = meta ? meta[L * g.nw + (z >> 5)].x : bits_plain[L * g.nw + (z >> 5)];
    out[i] = (w >> (z & 31)) & 1u;
}

__global__ void k_vcodes(const uint64_t *rec, int64_t m, uint8_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = (uint8_t)rec_vcode(rec[i]);
}

// any fluid cell with no velocity face at all -> diag(S_hat) == 0
__global__ void k_zero_sdiag(const uint64_t *prec, int64_t m, int *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m && rec_pkey(prec[i]) == 0) atomicOr(flag, 1);
}

// ------------------------------------------------------ slab decomposition
// Local meta of one family for a slab: local plane p in [0, P+2) is global
// plane (x_lo - 1 + p) mod n; base shifted by the plane's local offset.
__global__ void k_slab_meta(const uint2 *gmeta, uint2 *lmeta, int64_t words_per_plane, int x_lo, int P, int n,
                            int64_t delta_glo, int64_t delta_own, int64_t delta_ghi) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= words_per_plane * (P + 2)) return;
    const int p = (int)(i / words_per_plane);
    const int64_t w = i % words_per_plane;
    const int x = ((x_lo - 1 + p) % n + n) % n;
    const uint2 m = gmeta[(int64_t)x * words_per_plane + w];
    const int64_t d = p == 0 ? delta_glo : (p == P + 1 ? delta_ghi : delta_own);
    lmeta[i] = make_uint2(m.x, (uint32_t)((int64_t)m.y + d));
}

// Owned records of a slab: copy a global rank range, x -> local plane.
__global__ void k_slab_rec(const uint64_t *grec, uint64_t *lrec, int64_t count, int x_lo) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint64_t r = grec[i];
    const uint64_t xl = (uint64_t)(((r >> 22) & 0x7FF) - x_lo + 1);
    lrec[i] = (r & ~(0x7FFull << 22)) | (xl << 22);
}

// --------------------------------------------------------- operator applies

__global__ void k_apply_A(Geo g, const uint64_t *rec, const double *u, double *out, int64_t m,
                          const double *diag_code, double inv_h2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t r = rec[i];
    out[i] = apply_A_at(g, r, u[i], diag_code[rec_vcode(r)], inv_h2,
                        [&](uint32_t j) { return u[j]; });
}

// B (operators.py:137-144): out = 0; out += u_in - u_out per axis; * inv_h
__global__ void k_apply_div(Geo g, const uint64_t *prec, const double *u, double *out, int64_t m,
                            double inv_h, const int *gate) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m || (gate && *gate)) return;
    const uint64_t r = prec[i];
    const Cell c = rec_cell(r);
    double acc = 0.0;
    for (int a = 0; a < g.dim; ++a) {
        const double vin = rec_pin(r, a) ? u[rank_at(g.vmeta[a], g, c)] : 0.0;
        const double vout =
            rec_pout(r, a) ? u[rank_at(g.vmeta[a], g, shifted(c, iaxis(g.dim, a), 1, g))] : 0.0;
        acc = __dadd_rn(acc, __dsub_rn(vin, vout));
    }
    out[i] = __dmul_rn(acc, inv_h);
}

// B^T (operators.py:146-153): (p[I] - p[I - e_a]) * inv_h
__global__ void k_apply_grad(Geo g, const uint64_t *vrec, const double *p, double *out, int64_t m,
                             double inv_h, const int *gate) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m || (gate && *gate)) return;
    const uint64_t r = vrec[i];
    const Cell c = rec_cell(r);
    const int a = rec_comp(r);
    const double hi = p[rank_at(g.pmeta, g, c)];
    const double lo = p[rank_at(g.pmeta, g, shifted(c, iaxis(g.dim, a), -1, g))];
    out[i] = __dmul_rn(__dsub_rn(hi, lo), inv_h);
}

__global__ void k_apply_S(Geo g, const uint64_t *prec, const double *p, double *out, int64_t m,
                          const double *invA_enc, double inv_h) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    out[i] = apply_S_at(g, prec[i], p[i], invA_enc, inv_h, [&](uint32_t j) { return p[j]; });
}

// diag(B W B^T) (operators.py:194-206): out += w_in + w_out; * inv_h2
__global__ void k_dwd(Geo g, const uint64_t *prec, const double *w, double *out, int64_t m,
                      double inv_h2) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t r = prec[i];
    const Cell c = rec_cell(r);
    double acc = 0.0;
    for (int a = 0; a < g.dim; ++a) {
        const double vin = rec_pin(r, a) ? w[rank_at(g.vmeta[a], g, c)] : 0.0;
        const double vout =
            rec_pout(r, a) ? w[rank_at(g.vmeta[a], g, shifted(c, iaxis(g.dim, a), 1, g))] : 0.0;
        acc = __dadd_rn(acc, __dadd_rn(vin, vout));
    }
    out[i] = __dmul_rn(acc, inv_h2);
}

// ------------------------------------------------------ outer vector ops

// kind: 0 out=a-s ; 1 a-=s*b ; 2 a+=s*b ; 3 out=b+s*a (d = z + beta d) ; 4 out=a-b
// s comes from the device scalar *sp when sp != nullptr (outer loop state)
// gate (here and in the other outer-loop kernels): when the outer loop is enqueued several
// iterations ahead of the host, *gate != 0 (converged or failed: OuterState.stop) turns
// every later kernel into a no-op
__global__ void k_vec(int kind, double *out, double *a, const double *b, double s0, const double *sp, int64_t m,
                      const int *gate) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m || (gate && *gate)) return;
    const double s = sp ? *sp : s0;
    switch (kind) {
        case 0: out[i] = __dsub_rn(a[i], s); break;
        case 1: a[i] = __dsub_rn(a[i], __dmul_rn(s, b[i])); break;
        case 2: a[i] = __dadd_rn(a[i], __dmul_rn(s, b[i])); break;
        case 3: out[i] = __dadd_rn(b[i], __dmul_rn(s, a[i])); break;
        case 4: out[i] = __dsub_rn(a[i], b[i]); break;
    }
}

// force vector: 1.0 on [lo, lo+cnt), 0 elsewhere (operators.py:109-113);
// with sub != nullptr: out = force - sub (schur.py:353)
__global__ void k_force(double *out, const double *sub, int64_t lo, int64_t cnt, int64_t m) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double f = (i >= lo && i < lo + cnt) ? 1.0 : 0.0;
    out[i] = sub ? __dsub_rn(f, sub[i]) : f;
}

// deterministic two-stage reduction: kind 0 sum(a), 1 dot(a, b)
__global__ void __launch_bounds__(RED_THREADS) k_reduce1(int kind, const double *a, const double *b,
                                                         int64_t m, double *part, const int *gate) {
    __shared__ double sw[RED_THREADS / 32];
    if (gate && *gate) return;  // uniform over the grid
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RED_THREADS + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * RED_THREADS)
        acc = __dadd_rn(acc, kind ? __dmul_rn(a[i], b[i]) : a[i]);
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(~0u, acc, o));
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < RED_THREADS / 32; ++w) s = __dadd_rn(s, sw[w]);
        part[blockIdx.x] = s;
    }
}

__global__ void k_reduce2(const double *part, int nparts, double *out, const int *gate) {
    if (gate && *gate) return;
    double acc = 0.0;
    for (int j = threadIdx.x; j < nparts; j += 32) acc = __dadd_rn(acc, part[j]);
    for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(~0u, acc, o));
    if (threadIdx.x == 0) *out = acc;
}

// ------------------------------------------------------------ launchers

static inline unsigned nblk(int64_t m, int t = 256) { return (unsigned)((m + t - 1) / t); }

void launch_pack_fluid(const uint8_t *fluid, const Geo &g, int64_t nwords, uint32_t *fbits, cudaStream_t s) {
    k_pack_fluid<<<nblk(nwords), 256, 0, s>>>(fluid, g, nwords, fbits);
}
void launch_face_bits(const Geo &g, int a, int64_t nwords, uint32_t *out, cudaStream_t s) {
    k_face_bits<<<nblk(nwords), 256, 0, s>>>(g, a, nwords, out);
}
cudaError_t build_meta(const uint32_t *bits, int64_t nwords, uint32_t off, uint2 *meta, uint32_t *scratch_cnt,
                       uint32_t *scratch_base, void *temp, size_t temp_bytes, cudaStream_t s) {
    k_popc<<<nblk(nwords), 256, 0, s>>>(bits, nwords, scratch_cnt);
    size_t tb = temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, scratch_cnt, scratch_base, (int64_t)nwords, s);
    if (e != cudaSuccess) return e;
    k_make_meta<<<nblk(nwords), 256, 0, s>>>(bits, scratch_base, off, nwords, meta);
    return cudaGetLastError();
}
size_t scan_temp_bytes(int64_t nwords) {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)nwords);
    return tb;
}
void launch_vel_records(const Geo &g, int a, int64_t nwords, uint64_t *rec, cudaStream_t s) {
    k_vel_records<<<nblk(nwords), 256, 0, s>>>(g, a, nwords, rec);
}
void launch_p_records(const Geo &g, int64_t nwords, uint64_t *rec, cudaStream_t s) {
    k_p_records<<<nblk(nwords), 256, 0, s>>>(g, nwords, rec);
}
void launch_bits_to_u8(const uint2 *meta, const uint32_t *bits, const Geo &g, int64_t ncells, uint8_t *out,
                       cudaStream_t s) {
    k_bits_to_u8<<<nblk(ncells), 256, 0, s>>>(meta, bits, g, ncells, out);
}
void launch_vcodes(const uint64_t *rec, int64_t m, uint8_t *out, cudaStream_t s) {
    if (m) k_vcodes<<<nblk(m), 256, 0, s>>>(rec, m, out);
}
void launch_zero_sdiag(const uint64_t *prec, int64_t m, int *flag, cudaStream_t s) {
    if (m) k_zero_sdiag<<<nblk(m), 256, 0, s>>>(prec, m, flag);
}
void launch_slab_meta(const uint2 *gmeta, uint2 *lmeta, int64_t words_per_plane, int x_lo, int P, int n,
                      int64_t dlo, int64_t down, int64_t dhi, cudaStream_t s) {
    k_slab_meta<<<nblk(words_per_plane * (P + 2)), 256, 0, s>>>(gmeta, lmeta, words_per_plane, x_lo, P, n, dlo,
                                                               down, dhi);
}
void launch_slab_rec(const uint64_t *grec, uint64_t *lrec, int64_t count, int x_lo, cudaStream_t s) {
    if (count) k_slab_rec<<<nblk(count), 256, 0, s>>>(grec, lrec, count, x_lo);
}
void launch_apply_A(const Geo &g, const uint64_t *rec, const double *u, double *out, int64_t m,
                    const double *diag_code, double inv_h2, cudaStream_t s) {
    if (m) k_apply_A<<<nblk(m), 256, 0, s>>>(g, rec, u, out, m, diag_code, inv_h2);
}
void launch_apply_div(const Geo &g, const uint64_t *prec, const double *u, double *out, int64_t m, double inv_h,
                      cudaStream_t s, const int *gate) {
    if (m) k_apply_div<<<nblk(m), 256, 0, s>>>(g, prec, u, out, m, inv_h, gate);
}
void launch_apply_grad(const Geo &g, const uint64_t *vrec, const double *p, double *out, int64_t m,
                       double inv_h, cudaStream_t s, const int *gate) {
    if (m) k_apply_grad<<<nblk(m), 256, 0, s>>>(g, vrec, p, out, m, inv_h, gate);
}
void launch_apply_S(const Geo &g, const uint64_t *prec, const double *p, double *out, int64_t m,
                    const double *invA_enc, double inv_h, cudaStream_t s) {
    if (m) k_apply_S<<<nblk(m), 256, 0, s>>>(g, prec, p, out, m, invA_enc, inv_h);
}
void launch_dwd(const Geo &g, const uint64_t *prec, const double *w, double *out, int64_t m, double inv_h2,
                cudaStream_t s) {
    if (m) k_dwd<<<nblk(m), 256, 0, s>>>(g, prec, w, out, m, inv_h2);
}
void launch_vec(int kind, double *out, double *a, const double *b, double sc, const double *sp, int64_t m,
                cudaStream_t s, const int *gate) {
    if (m) k_vec<<<nblk(m), 256, 0, s>>>(kind, out, a, b, sc, sp, m, gate);
}

// ---- device-side scalar steps of the outer PCG (krylov.py:102-182, schur.py:288)
__device__ __forceinline__ double slab_sum(const double *scal, int q, int R) {
    double t = scal[q * R];
    for (int s = 1; s < R; ++s) t = t + scal[q * R + s];
    return t;
}

__global__ void k_outer(int op, OuterState *st, const double *scal, int R, double arg, int64_t k, double eps,
                        int use_prec, double *hist, const int *gate) {
    if (gate && *gate) return;
    // hist layout: [0] alpha, [1] beta, [2] res_prec, [3] res_unprec, [4] perm; stride HSTRIDE
    double *h_alpha = hist, *h_beta = hist + st->hstride, *h_rp = hist + 2 * st->hstride,
           *h_ru = hist + 3 * st->hstride, *h_perm = hist + 4 * st->hstride;
    auto flag = [&](int code, double val, int64_t at) {
        if (!st->status) { st->status = code; st->value = val; st->at = at; }
    };
    switch (op) {
        case SO_MEAN: st->mu = slab_sum(scal, Q_MU, R) / arg; break;  // arg = m
        case SO_PERM: h_perm[k + 1] = arg * slab_sum(scal, Q_PERM, R); break;  // arg = h**dim
        case SO_INIT: {  // krylov.py:120-128
            const double rp = sqrt(slab_sum(scal, Q_ZZ, R)), ru = sqrt(slab_sum(scal, Q_RR, R));
            h_rp[0] = rp;
            h_ru[0] = ru;
            st->ref = use_prec ? rp : ru;
            st->converged = st->ref == 0.0;
            st->rz = slab_sum(scal, Q_RZ, R);
            st->its = 0;
            if (!st->converged) {
                if (st->rz < 0.0) flag(1, st->rz, 0);
                else if (st->rz == 0.0) st->converged = 1;
            }
            break;
        }
        case SO_ALPHA: {  // krylov.py:139-146
            const double dq = slab_sum(scal, Q_DQ, R);
            if (dq <= 0.0) flag(2, dq, k);
            st->alpha = st->rz / dq;
            h_alpha[k] = st->alpha;
            break;
        }
        case SO_BETA: {  // krylov.py:154-169, then the next iteration's r'z checks (:131-137)
            const double rz_new = slab_sum(scal, Q_RZ, R);
            st->beta = rz_new / st->rz;
            st->rz = rz_new;
            const double nz = sqrt(slab_sum(scal, Q_ZZ, R)), nr = sqrt(slab_sum(scal, Q_RR, R));
            if (!(isfinite(nz) && isfinite(nr))) { flag(3, 0.0, k + 1); break; }
            h_beta[k] = st->beta;
            h_rp[k + 1] = nz;
            h_ru[k + 1] = nr;
            st->its = k + 1;
            if ((use_prec ? nz : nr) / st->ref < eps) { st->converged = 1; break; }
            if (st->rz < 0.0) flag(1, st->rz, k + 1);
            else if (st->rz == 0.0) st->converged = 1;
            break;
        }
    }
    st->stop = (st->converged || st->status) ? 1 : 0;
}

// cross-rank barrier for the outer loop: one arrival per rank on the
// counter the fused CG uses (its base carried in *bar_base).  The ranks are
// processes on different GPUs, so release/acquire are at system scope.
__global__ void k_xbar(unsigned *bar, unsigned *bar_base, int nranks, volatile int *xflag,
                       unsigned long long timeout_ns) {
    const unsigned target = *bar_base + (unsigned)nranks;
    asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v, spins = 0;
    unsigned long long t0 = 0;
    do {
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        if (xflag && (++spins & 1023u) == 0) {  // a peer that never arrives must not hang the stream
            unsigned long long now;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
            if (!t0) t0 = now;
            if (*xflag) break;
            if (timeout_ns && now - t0 > timeout_ns) {
                *xflag = 1;
                break;
            }
        }
    } while ((int)(v - target) < 0);
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    *bar_base = target;
}
void launch_xbar(unsigned *bar, unsigned *bar_base, int nranks, volatile int *xflag, unsigned long long timeout_ns,
                 cudaStream_t s) {
    k_xbar<<<1, 1, 0, s>>>(bar, bar_base, nranks, xflag, timeout_ns);
}

void launch_outer(int op, OuterState *st, const double *scal, int R, double arg, int64_t k, double eps,
                  int use_prec, double *hist, cudaStream_t s, const int *gate) {
    k_outer<<<1, 1, 0, s>>>(op, st, scal, R, arg, k, eps, use_prec, hist, gate);
}
void launch_force(double *out, const double *sub, int64_t lo, int64_t cnt, int64_t m, cudaStream_t s) {
    if (m) k_force<<<nblk(m), 256, 0, s>>>(out, sub, lo, cnt, m);
}
int launch_reduce(int kind, const double *a, const double *b, int64_t m, double *part, double *out,
                  cudaStream_t s, const int *gate) {
    int nb = (int)std::min<int64_t>(RED_MAX_BLOCKS, std::max<int64_t>(1, (m + 4 * RED_THREADS - 1) / (4 * RED_THREADS)));
    k_reduce1<<<nb, RED_THREADS, 0, s>>>(kind, a, b, m, part, gate);
    k_reduce2<<<1, 32, 0, s>>>(part, nb, out, gate);
    return 2;
}

}  // namespace vs
