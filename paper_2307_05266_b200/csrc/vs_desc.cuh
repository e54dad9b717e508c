// vs_desc.cuh -- the 8-byte DOF descriptor shared by the descriptor-driven
// fused PCG kernels (k_pcgm in vs_cgm.cu, k_pcgx in vs_cgx.cu): field layout,
// the code bits as a record, the 2-B code index.  See vs_cgm.cu for the format.
#pragma once
#include "vs_cg_common.cuh"

namespace vs {

constexpr int DX_BITS = 13, DY_BITS = 10;
constexpr uint32_t DX_MASK = (1u << DX_BITS) - 1u, DY_MASK = (1u << DY_BITS) - 1u;
constexpr uint32_t DX_ESC = DX_MASK;  // x+ field all ones: take the record + bitmask lookup
constexpr int SH_XP = 18, SH_XM = SH_XP + DX_BITS, SH_YP = SH_XM + DX_BITS, SH_YM = SH_YP + DY_BITS;
static_assert(SH_YM + DY_BITS == 64, "descriptor is 64 bits");

// the descriptor's 18 code bits as a record the shared helpers understand
// (coordinates zero: only the escape path needs them, and it reads G.rec)
template <int OP>
__device__ __forceinline__ uint64_t desc_rec(uint64_t d) {
    const uint64_t c = d & 0x3FFFFull;
    if (OP == 1) return c << 40;
    return ((c & 0xF) << 36) | (((c >> 4) & 0x3F) << 40) | (((c >> 10) & 0x3) << 33);
}
template <int OP>
__device__ __forceinline__ uint64_t rec_codes(uint64_t rc) {
    if (OP == 1) return (rc >> 40) & 0x3FFFFull;
    return (uint64_t)rec_vcode(rc) | (((rc >> 40) & 0x3F) << 4) | ((uint64_t)rec_comp(rc) << 10);
}
// 2-B code index of P2's stream: A: no-slip code | component << 8;
// S_hat: the six face codes in base 6 (46656 values)
template <int DIM, int OP>
__device__ __forceinline__ uint32_t rec_cidx(uint64_t rc) {
    if (OP == 0) return (uint32_t)rec_vcode(rc) | ((uint32_t)rec_comp(rc) << 8);
    uint32_t v = 0;
#pragma unroll
    for (int a = 2; a >= 0; --a) v = v * 6 + (uint32_t)rec_pout(rc, a);
#pragma unroll
    for (int a = 2; a >= 0; --a) v = v * 6 + (uint32_t)rec_pin(rc, a);
    return v;
}
// An escape descriptor (x+ field = DX_ESC) keeps its 18 code bits; the 33 bits from SH_XM up hold
// 1 + the DOF's slot in the escape table (8 x uint32 per slot: its 2*DIM gather indices, an
// absent neighbour's = the DOF itself), or 0 when the table was full -- k_pcgx reads the slot
// instead of the record + bitmask words (k_pcgm ignores the field).
constexpr int SH_EORD = SH_XM;
constexpr int CHUNK_SHIFT = 10;  // x-bases are kept per chunk of 1024 consecutive ranks

}  // namespace vs
