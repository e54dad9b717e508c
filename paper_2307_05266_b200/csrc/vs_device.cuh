// vs_device.cuh -- device data layout and bit-exact MAC operator stencils.
//
// Layout in HBM:
//   * Every DOF family F (velocity component a = 0..dim-1, pressure) is a
//     packed FP64 vector in the reference's order (operators.py:239-249).
//   * Geometry is kept as bitmasks along the fastest (last) axis: one
//     32-cell word per (line, w), line = (x, y) in 3D or x in 2D.  Each
//     word carries {mask, base} (uint2, 8 B / 32 cells) where base is the
//     global vector rank of the word's first set bit.  The rank of any
//     cell is base + popc(mask & lanemask_below(z)) -- one L1/L2-resident
//     load per neighbour, no neighbour index tables (the reference keeps
//     48 B/DOF of int64 tables, operators.py:260-297).
//   * One uint64 record per DOF: coordinates + the integer no-slip code(s)
//     (velocity: its diagonal code, operators.py:268-285; pressure: the six
//     face codes of B diag(A)^-1 B^T, schur.py:234-240).  Every FP constant
//     is a table lookup on those small integers, so results are bitwise the
//     reference's.
//   * All FP arithmetic uses explicit __d{add,sub,mul}_rn: numpy never
//     contracts a*b-c*d into an FMA, so neither do we.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vs {

constexpr uint32_t ABSENT = 0xFFFFFFFFu;

// ---- record bit layout ------------------------------------------------
// z:0..10  y:11..21  x:22..32  comp:33..34  vcode:36..39
// velocity: neighbour presence 40..45 (slot order x+, x-, [y+, y-,] z+, z-)
// pressure: face codes 40..57 (nonzero <=> the neighbour cell is fluid)
__host__ __device__ __forceinline__ uint64_t make_rec(int x, int y, int z, int comp) {
    return (uint64_t)z | ((uint64_t)y << 11) | ((uint64_t)x << 22) | ((uint64_t)comp << 33);
}
__device__ __forceinline__ int rec_z(uint64_t r) { return (int)(r & 0x7FF); }
__device__ __forceinline__ int rec_y(uint64_t r) { return (int)((r >> 11) & 0x7FF); }
__device__ __forceinline__ int rec_x(uint64_t r) { return (int)((r >> 22) & 0x7FF); }
__device__ __forceinline__ int rec_comp(uint64_t r) { return (int)((r >> 33) & 0x3); }
__device__ __forceinline__ int rec_vcode(uint64_t r) { return (int)((r >> 36) & 0xF); }
// pressure: encoded face code (0 = no face) of face (a, I) ("in") and
// face (a, I + e_a) ("out"); enc = code - (2*dim - 1) in 1..(2*dim-1)
__device__ __forceinline__ int rec_pin(uint64_t r, int a) { return (int)((r >> (40 + 3 * a)) & 7); }
__device__ __forceinline__ int rec_pout(uint64_t r, int a) { return (int)((r >> (49 + 3 * a)) & 7); }
__device__ __forceinline__ uint32_t rec_pkey(uint64_t r) { return (uint32_t)((r >> 40) & 0x3FFFF); }
// neighbour in slot s = 2a + (minus) present? (OP 0 velocity, OP 1 pressure)
template <int OP>
__device__ __forceinline__ bool rec_has_nb(uint64_t r, int s) {
    if (OP == 0) return (r >> (40 + s)) & 1u;
    return (s & 1) ? rec_pin(r, s >> 1) != 0 : rec_pout(r, s >> 1) != 0;
}

struct Geo {
    int dim, n, nw, nlines;
    int nx;                  // extent of the (local) x axis: n, or slab planes + 2 ghosts
    const uint32_t *fbits;   // fluid bits [nlines * nw]
    const uint2 *vmeta[3];   // velocity component meta
    const uint2 *pmeta;      // pressure meta
};

// internal axis of reference axis a: 0 -> x, 1 -> y (3D) / z (2D), 2 -> z
__device__ __forceinline__ int iaxis(int dim, int a) { return (dim == 3) ? a : (a == 0 ? 0 : 2); }

struct Cell { int x, y, z; };

__device__ __forceinline__ Cell shifted(Cell c, int ia, int s, const Geo &g) {
    const int n = g.n;
    if (ia == 0) { c.x += s; c.x = c.x < 0 ? g.nx - 1 : (c.x >= g.nx ? 0 : c.x); }
    else if (ia == 1) { c.y += s; c.y = c.y < 0 ? n - 1 : (c.y >= n ? 0 : c.y); }
    else { c.z += s; c.z = c.z < 0 ? n - 1 : (c.z >= n ? 0 : c.z); }
    return c;
}
__device__ __forceinline__ int line_of(const Geo &g, Cell c) { return g.dim == 3 ? c.x * g.n + c.y : c.x; }

// global rank of cell c in the family described by meta, or ABSENT
__device__ __forceinline__ uint32_t rank_at(const uint2 *meta, const Geo &g, Cell c) {
    const uint2 m = meta[(size_t)line_of(g, c) * g.nw + (c.z >> 5)];
    const uint32_t b = (uint32_t)c.z & 31u;
    if (!((m.x >> b) & 1u)) return ABSENT;
    return m.y + (uint32_t)__popc(m.x & ((1u << b) - 1u));
}

__device__ __forceinline__ bool fluid_at(const Geo &g, Cell c) {
    return (g.fbits[(size_t)line_of(g, c) * g.nw + (c.z >> 5)] >> (c.z & 31)) & 1u;
}

__device__ __forceinline__ Cell rec_cell(uint64_t r) { return Cell{rec_x(r), rec_y(r), rec_z(r)}; }

// ---- A = -Laplacian (operators.py:131-135) ------------------------------
// diag*u - inv_h2 * ((((v0 + v1) + v2) + v3) + v4) + v5 over the slots
// (d=0,+1), (d=0,-1), (d=1,+1), ...; absent neighbours read as 0.0.
template <class Load>
__device__ __forceinline__ double apply_A_at(const Geo &g, uint64_t rec, double ui, double diag,
                                             double inv_h2, Load ld) {
    const Cell c = rec_cell(rec);
    const uint2 *meta = g.vmeta[rec_comp(rec)];
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (d >= g.dim) break;
        const int ia = iaxis(g.dim, d);
#pragma unroll
        for (int si = 0; si < 2; ++si) {
            const Cell cn = shifted(c, ia, si == 0 ? 1 : -1, g);
            const uint32_t rk = rank_at(meta, g, cn);
            const double v = (rk != ABSENT) ? ld(rk) : 0.0;
            acc = (d == 0 && si == 0) ? v : __dadd_rn(acc, v);
        }
    }
    return __dsub_rn(__dmul_rn(diag, ui), __dmul_rn(inv_h2, acc));
}

// ---- S_hat = B diag(A)^-1 B^T (schur.py:234-240) at a pressure cell ------
// out = sum_a (w_in - w_out) starting from 0.0, times inv_h, with
// w_in = ((p_I - p_{I-e_a}) * inv_h) * invA(face a,I)          (:146-153)
// w_out = ((p_{I+e_a} - p_I) * inv_h) * invA(face a,I+e_a)     (:137-144)
template <class Load>
__device__ __forceinline__ double apply_S_at(const Geo &g, uint64_t rec, double pi,
                                             const double *invA_enc, double inv_h, Load ld) {
    const Cell c = rec_cell(rec);
    double out = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (a >= g.dim) break;
        const int ia = iaxis(g.dim, a);
        const int ci = rec_pin(rec, a), co = rec_pout(rec, a);
        double wi = 0.0, wo = 0.0;
        if (ci) {
            const uint32_t rk = rank_at(g.pmeta, g, shifted(c, ia, -1, g));
            wi = __dmul_rn(__dmul_rn(__dsub_rn(pi, ld(rk)), inv_h), invA_enc[ci]);
        }
        if (co) {
            const uint32_t rk = rank_at(g.pmeta, g, shifted(c, ia, 1, g));
            wo = __dmul_rn(__dmul_rn(__dsub_rn(ld(rk), pi), inv_h), invA_enc[co]);
        }
        out = __dadd_rn(out, __dsub_rn(wi, wo));
    }
    return __dmul_rn(out, inv_h);
}

}  // namespace vs
