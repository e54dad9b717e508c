// vs_internal.h -- host-side declarations shared by the API and the kernels.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "vs_device.cuh"

namespace vs {

#ifndef VS_CG_THREADS
#define VS_CG_THREADS 1024
#endif
constexpr int CG_THREADS = VS_CG_THREADS;
constexpr int RED_THREADS = 256;
constexpr int RED_MAX_BLOCKS = 592;
constexpr int VS_MAX_SLABS = 16;

struct CgOut {
    int64_t iterations;
    int32_t converged;
    int32_t status;  // 0 ok, 1 r'z < 0, 2 d'q <= 0, 3 non-finite
    double value;
    int64_t at_iter;
    double res_prec0, res_unprec0, res_prec_last, res_unprec_last;
};

// One slab of the decomposition (one rank); a whole-domain run is 1 group.
// Local vectors hold [owned DOFs | ghost-plane DOFs]; ranks in meta are local.
struct CgGroup {
    const uint2 *meta[3];   // velocity components (op 0) or meta[0] = pressure (op 1)
    const uint64_t *rec;    // records of the owned DOFs (x = local plane)
    int nx;                 // local x extent (n when the group is the whole domain)
    uint32_t m_own, m_all;  // owned DOFs, owned + ghost
    const double *rhs, *x0;
    double *x, *r, *z, *d0, *d1, *q;
    double *zb[2], *ub[2], *sb[2];  // k_cg1: double-buffered zr = M r, u = M A zr, s = M q
    // k_pcgx (vs_cgx.cu): the ring of z buffers (iteration k lives in zr[k mod M]) and, per
    // halo side, the neighbour slab's buffers (ghost planes)
    double *zr[4];
    double *zrp[2][4];
    // k_pcgm (vs_cgm.cu): 8-B descriptors, 2-B code indices and the x+ / x-
    // rank-distance bases per chunk of 1024 ranks
    const uint64_t *desc;
    const uint16_t *cidx;
    const int2 *xb;
    const uint4 *esc;  // escape table (vs_desc.cuh): two uint4 per slot
    // k_pcgb (vs_cgb.cu): blocked order -- tile starts [ntiles + 1], per tile and line slot
    // the line's first blocked rank, its DOFs and its offset in the shared-memory window;
    // per DOF its index in the window; window capacity in doubles
    const uint32_t *tile0, *tl_src;
    const uint16_t *tl_len, *tl_v, *vidx;
    int ntiles, vcap, vbuf;
    const uint32_t *nbr;            // TIER 3: neighbour ranks [2*dim][m_own] (ABSENT if none);
                                    // TIER 4: int2 x-deltas [m_own], then short2 y-deltas [m_own] (3D)
    // halo: side s = 0 sends the first owned plane to the lower neighbour's
    // ghost_hi, s = 1 the last owned plane to the upper neighbour's ghost_lo;
    // per family f, local range [sbeg, send) -> zpeer[s][sdst + (i - sbeg)]
    uint32_t sbeg[2][3], send[2][3], sdst[2][3];
    double *zpeer[2];
};

struct CgParams {
    const CgGroup *groups;  // device array, one per group
    int group_base, bpg;    // group of block b = group_base + b / bpg
    int n, nw;
    double m_global;        // DOFs summed over groups (for the mean projection)
    double *part;           // this rank's partial buffer: 4 sets x 8 slots x total_blocks
    unsigned *bar;          // grid barrier counter (rank 0's on a multi-GPU run)
    unsigned *bar_base;     // local: counter value reached by the previous launch
    int total_blocks;       // blocks of all ranks in this solve
    int block_base;         // global index of this launch's block 0
    int npart;              // ranks whose partial buffers receive this launch's sums
    int xgpu;               // ranks are processes on different GPUs: system-scope barrier
    volatile int *xflag;    // xgpu: set when a cross-GPU barrier timed out (device memory, read back by the host after a sync)
    unsigned long long xtimeout_ns;
    int part_self;          // index in part_peer of the first local group's own buffer
    double *part_peer[VS_MAX_SLABS];
    // hierarchical barrier of multi-rank runs (npart > 1): per rank a local arrival counter
    // (wraps at bpg) and a local release word in the rank's OWN arena; only the rank's last
    // arriver crosses to the shared counter.  Indexed like part_peer (own entries valid).
    unsigned *lbar[VS_MAX_SLABS];
    int hier;               // 1: ranks arrive through their leaders (bar counts ranks, not blocks)
    int nranks_bar;         // ranks that take part in a barrier
    CgOut *out;
    double tol;
    int64_t max_iter;
    int norm_prec;
    double inv_h, inv_h2;
    double diag_code[16];
    double inv_code[16];
    double invA_enc[8];
    const double *invS;
    const double2 *sdiag2;         // S_hat {1/diag, diag} by 18-bit key (k_cg1)
    const double2 *ctab;           // {1/diag, diag} by 2-B code index (k_pcgm)
    uint32_t cache_slots;
    uint32_t pf_dist;              // L2 prefetch distance in grid strides (0 = off)
    const int *gate;               // outer-loop gate (OuterState.stop): != 0 -> this solve is a no-op
    unsigned long long *phase_ns;  // optional [12] accumulators
    uint32_t dbg;                  // VOXSCHUR_DBG bits (timing experiments only; results are wrong):
                                   // 1 = P1 gathers read the DOF's own value
};


void launch_pack_fluid(const uint8_t *fluid, const Geo &g, int64_t nwords, uint32_t *fbits, cudaStream_t s);
void launch_face_bits(const Geo &g, int a, int64_t nwords, uint32_t *out, cudaStream_t s);
cudaError_t build_meta(const uint32_t *bits, int64_t nwords, uint32_t off, uint2 *meta, uint32_t *scratch_cnt,
                       uint32_t *scratch_base, void *temp, size_t temp_bytes, cudaStream_t s);
size_t scan_temp_bytes(int64_t nwords);
void launch_vel_records(const Geo &g, int a, int64_t nwords, uint64_t *rec, cudaStream_t s);
void launch_p_records(const Geo &g, int64_t nwords, uint64_t *rec, cudaStream_t s);
void launch_bits_to_u8(const uint2 *meta, const uint32_t *bits, const Geo &g, int64_t ncells, uint8_t *out,
                       cudaStream_t s);
void launch_vcodes(const uint64_t *rec, int64_t m, uint8_t *out, cudaStream_t s);
void launch_zero_sdiag(const uint64_t *prec, int64_t m, int *flag, cudaStream_t s);
void launch_slab_meta(const uint2 *gmeta, uint2 *lmeta, int64_t words_per_plane, int x_lo, int P, int n,
                      int64_t dlo, int64_t down, int64_t dhi, cudaStream_t s);
void launch_slab_rec(const uint64_t *grec, uint64_t *lrec, int64_t count, int x_lo, cudaStream_t s);
void launch_apply_A(const Geo &g, const uint64_t *rec, const double *u, double *out, int64_t m,
                    const double *diag_code, double inv_h2, cudaStream_t s);
void launch_apply_div(const Geo &g, const uint64_t *prec, const double *u, double *out, int64_t m, double inv_h,
                      cudaStream_t s, const int *gate = nullptr);
void launch_apply_grad(const Geo &g, const uint64_t *vrec, const double *p, double *out, int64_t m,
                       double inv_h, cudaStream_t s, const int *gate = nullptr);
void launch_apply_S(const Geo &g, const uint64_t *prec, const double *p, double *out, int64_t m,
                    const double *invA_enc, double inv_h, cudaStream_t s);
void launch_dwd(const Geo &g, const uint64_t *prec, const double *w, double *out, int64_t m, double inv_h2,
                cudaStream_t s);
void launch_vec(int kind, double *out, double *a, const double *b, double sc, const double *sp, int64_t m,
                cudaStream_t s, const int *gate = nullptr);

// device-side state of the outer PCG (vs_api.cu drives it, one sync per outer iteration)
struct OuterState {
    double rz, alpha, beta, mu, ref, value;
    int32_t status, converged;  // status: 1 r'z < 0, 2 d'q <= 0, 3 non-finite
    int32_t stop, _pad;         // converged or failed: the gate of kernels enqueued ahead of the host
    int64_t at, its, hstride;
};
enum { SO_MEAN, SO_PERM, SO_INIT, SO_ALPHA, SO_BETA };
enum { Q_DQ, Q_PERM, Q_MU, Q_RZ, Q_ZZ, Q_RR, Q_HOST, Q_COUNT };  // reduction slots (x R slabs)
void launch_xbar(unsigned *bar, unsigned *bar_base, int nranks, volatile int *xflag, unsigned long long timeout_ns,
                 cudaStream_t s);
void launch_outer(int op, OuterState *st, const double *scal, int R, double arg, int64_t k, double eps,
                  int use_prec, double *hist, cudaStream_t s, const int *gate = nullptr);
void launch_force(double *out, const double *sub, int64_t lo, int64_t cnt, int64_t m, cudaStream_t s);
int launch_reduce(int kind, const double *a, const double *b, int64_t m, double *part, double *out,
                  cudaStream_t s, const int *gate = nullptr);
// connected components on the GPU (vs_cc.cu)
constexpr int64_t CC_DEVICE_CELLS = (int64_t)1 << 22;  // assemble checks larger grids on the device
size_t cc_work_bytes(int64_t N);
int64_t cc_label_device(const uint8_t *d_fluid, int dim, int n, int *d_labels, void *work, size_t work_bytes,
                        cudaStream_t s);
constexpr size_t CG_SMEM_BUDGET = 200 * 1024;  // dynamic smem per block (1 block / SM)
// k_pcg (reference order) | k_cg1 (one reduction) | k_pcg with q = A z + beta q_old
// (value 3: 2 is the k_cg1t kernel id in vs_kstat)
// 4, 5: k_pcgm (vs_cgm.cu), M-scaled over 8-B descriptors: s = M q by
// recurrence / q = A d recomputed in both passes
// 6: k_pcgb (vs_cgb.cu), the qrec form on the blocked order with shared-memory windows (S_hat, 3D, one slab)
// 7: k_pcgx (vs_cgx.cu): alpha from the z sums (no d in the stencil pass), z in a ring of
//    M buffers, d and x brought up to date every M-th iteration: 90 / 78 / 74 / 72 B per
//    DOF-iteration for M = 1..4
enum CgAlg {
    CG_TWO_SUM = 0, CG_ONE_SUM = 1, CG_TWO_SUM_QREC = 3, CG_TWO_SUM_MQ = 4, CG_TWO_SUM_MRC = 5, CG_BLOCKED = 6,
    CG_TWO_SUM_MX = 7
};
constexpr int PCGX_MAX_DEPTH = 4, PCGX_DEPTH_DEFAULT = 4;
struct CgPlan {
    int alg;
    int unroll;   // DOFs per P1 step (k_pcg<QR> only)
    int threads;  // block size of the launch
    int tier, grid;
    uint32_t slots;
    size_t smem;
};
CgPlan pcg_plan(int dim, int op, int64_t m, int groups, int device, int alg, int nbr_tier = 0,
                int sms = 0);
// fill the TIER-3 neighbour-rank table of one group's owned DOFs
void launch_build_nbr(int dim, int op, const CgGroup &G, int n, int nw, uint32_t *out, cudaStream_t s,
                      int tier = 3);
cudaError_t launch_pcg(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s);
// k_pcgm (vs_cgm.cu)
CgPlan pcgm_plan(int dim, int op, int64_t m, int groups, int device, int alg, int sms = 0);
cudaError_t launch_pcgm(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s);
void launch_desc_scan(int dim, int op, const CgGroup &G, int n, int nw, int2 *xb, cudaStream_t s);
void launch_desc_pack(int dim, int op, const CgGroup &G, int n, int nw, const int2 *xb, uint64_t *desc,
                      uint16_t *cidx, unsigned long long *n_escape, uint32_t *esc_tab, uint32_t esc_cap,
                      cudaStream_t s);
// k_pcgx (vs_cgx.cu); the plan's `unroll` carries the ring depth M
CgPlan pcgx_plan(int dim, int op, int64_t m, int groups, int device, int sms = 0);
cudaError_t launch_pcgx(int dim, int op, const CgPlan &pl, int groups, CgParams &P, cudaStream_t s);
// k_pcgb (vs_cgb.cu)
void launch_blk_build(const CgGroup &G, int n, int nw, const uint32_t *lineR, const uint32_t *lineI,
                      const uint16_t *tl_v, uint64_t *desc, uint16_t *vidx, uint16_t *cidx, int *bad, cudaStream_t s);
void launch_blk_perm(const uint64_t *rec, int n, const uint32_t *lineR, const uint32_t *lineI, uint32_t m,
                     const double *in, double *out, int to_blocked, cudaStream_t s);
size_t pcgb_smem(int vcap, int nbuf);
int pcgb_fits(int vcap, int device);
cudaError_t launch_pcgb(const CgPlan &pl, CgParams &P, int vcap, int nbuf, cudaStream_t s);
void launch_build_ctab(int op, const double2 *sdiag2, const double *diag_code, double2 *ctab, int count,
                       cudaStream_t s);

// ---- k_cg1t: plane-sweep tiles staged by TMA (vs_cgt.cu) ----------------
// A unit = one DOF family (velocity component / pressure), a run of own
// lines [ya, ya + H) of every plane in [x0, x1]; the block sweeps its
// planes in x with the window (own lines +- 1 line) of planes x-1, x, x+1
// resident in shared memory.
struct TileUnit {
    int32_t fam;     // family: velocity component (A) or 0 (S_hat)
    int32_t ya;      // first own line
    int32_t wrap;    // 1: the window is the whole plane (y neighbours wrap inside it)
    int32_t nwl;     // window lines
    int32_t npc;     // window pieces (contiguous rank runs): 1 or 2
    int32_t pwl1;    // first window line of piece 1
    int32_t nplanes; // descriptors: halo plane, compute planes, halo plane
    uint32_t desc0;  // index of the first descriptor
};
struct PlaneDesc {               // 48 B (a multiple of 16: bulk-copied), one per plane of a unit
    uint32_t own_start, own_len; // own DOFs (ranks) of the plane
    uint32_t vstart[2], vlen[2]; // window pieces in doubles (even start and length)
    uint32_t mstart[2], mlen[2]; // window pieces in meta words (even start and length)
    uint32_t pad[2];
};
static_assert(sizeof(PlaneDesc) % 16 == 0, "PlaneDesc is bulk-copied");
struct TileParams {
    const TileUnit *units;
    const uint32_t *blk_unit;  // block b runs units [blk_unit[b], blk_unit[b + 1])
    const PlaneDesc *planes;
    uint32_t capg;             // window capacity per slot and vector (doubles, even)
    uint32_t capo;             // own-slice capacity per slot and stream (8-B words, even)
    uint32_t capm;             // meta words per slot (even)
    uint32_t wlmax;            // window lines (max)
    uint32_t dmax;             // descriptors per unit (max)
};
struct TilePlan {
    bool ok = false;
    int grid = 0;
    size_t smem = 0;
    int H[3] = {0, 0, 0};
    int64_t units = 0;
    TileParams tp{};
    void *mem = nullptr;       // device copy of units, blk_unit, planes
};
// Plan the tiles of one operator's families on `device` (meta/m per family,
// one slab, 3D, nw even).  Returns ok = false when the shapes do not fit.
TilePlan tile_plan(int op, int n, int nw, int nfam, const uint2 *const *meta, const int64_t *m_fam, int device,
                   cudaStream_t s);
cudaError_t launch_cg1t(int op, const TilePlan &tp, CgParams &P, cudaStream_t s);

}  // namespace vs
