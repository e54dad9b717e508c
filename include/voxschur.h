/*
 * voxschur.h -- C ABI of the B200-native pressure-Schur-complement Stokes path.
 *
 * Drop-in boundary for the reference package `voxstokes`
 * (/root/reference/pkg/src/voxstokes).  The reference is pure Python, so the
 * binding a maintainer adds is a ctypes stub; the Python
 * mirror of the reference API in paper_2307_05266_b200/ is that stub.
 *
 * Conventions
 *   - every function returns an int status: VS_OK, VS_EVALUE (the reference
 *     raises ValueError), VS_ERUNTIME (the reference raises RuntimeError),
 *     VS_ECUDA (device/internal failure).  On failure the message is written
 *     to the thread-local buffer returned by vs_last_error(); messages for
 *     VS_EVALUE / VS_ERUNTIME are byte-identical to the reference's.
 *   - host pointers in, host pointers out (caller owns them); the library
 *     owns all device memory inside an opaque context.  No callbacks.
 *   - vectors use the reference DOF order: velocity axis-major, then C-order
 *     of the face position (last axis fastest); pressure C-order over fluid
 *     voxels (operators.py:239-249).
 *   - one context = one device + one CUDA stream; contexts are independent
 *     and may be used from different threads.
 */
#ifndef VOXSCHUR_H
#define VOXSCHUR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VS_OK 0
#define VS_EVALUE 1
#define VS_ERUNTIME 2
#define VS_ECUDA 3
#define VS_EOS 4      /* open/read/write failed; message = errno (the reference raises OSError) */
#define VS_EDECODE 5  /* file is not UTF-8 (the reference raises UnicodeDecodeError) */

typedef struct vs_ctx vs_ctx;

/* Scalars of one Schur solve (schur.py:113-136 SolveReport, minus arrays). */
typedef struct {
    double k_value;              /* permeability of the refreshed velocity  */
    int64_t iters_outer;
    int32_t converged;
    int32_t _pad;
    int64_t inner_velocity;      /* inner_iter_totals["velocity"]           */
    int64_t inner_preconditioner;/* inner_iter_totals["preconditioner"]     */
    int64_t uf_iters;            /* discarded u_f solve count (schur.py:230) */
    int64_t n_hist;              /* entries written to each history array   */
    double device_ms;            /* CUDA-event time of the device solve     */
} vs_report;

/* Solve settings (schur.py:64-75 SchurConfig) + host-computed constants. */
typedef struct {
    int32_t prec;                /* 0 = uzawa, 1 = simple                   */
    int32_t outer_norm;          /* 0 = preconditioned, 1 = unpreconditioned*/
    double eps_S, eps_A, eps_Shat;
    int64_t max_iter;
    double h_pow_dim;            /* h**dim as Python computes it (schur.py:288) */
} vs_schur_cfg;

/* Thread-local message of the last failing call. */
const char *vs_last_error(void);

/* Library build string (arch, version). */
const char *vs_version(void);

/* Visible CUDA devices (0 when there is no device or driver); the sweep
 * driver binds one worker per device. */
int vs_device_count(int *count);

/* Periodic face-adjacency components of a mask (geometry.py:183-222).
 * labels (nullable) receives ids in first row-major appearance, -1 on solid. */
int vs_components(const uint8_t *fluid, int dim, int n, int32_t *labels,
                  int64_t *n_components);

/* The same labelling on the GPU `device` (lock-free union-find, roots at
 * the minimum cell index, dense ids by a scan of the roots): identical
 * labels and count.  assemble uses it for grids of >= 2^22 cells. */
int vs_components_device(const uint8_t *fluid, int dim, int n, int device, int32_t *labels,
                         int64_t *n_components);

/* Percolation along `axis` on the periodic box: a component percolates iff it
 * holds a closed path of non-zero winding along that axis.  Union-find over
 * the fluid cells carrying the unwrapped axis offset (the periodic merge of
 * geometry.py:183-222 extended as SURVEY App. B-3 asks; host C++).  Returns
 * the number of periodic components and how many of them wind. */
int vs_winding(const uint8_t *fluid, int dim, int n, int axis, int64_t *n_components,
               int64_t *n_winding);

/* voxgeo text IO (geometry.py:243-339), multithreaded host C++.
 * vs_grid_header: dim and size from the three header lines only (to size
 * the caller's buffer); vs_read_grid: the whole file with the reference's
 * checks and messages, into fluid (C-order (x,y,z), 1 = fluid; cap bytes;
 * fluid may be NULL to validate only); vs_write_grid: the reference's exact
 * bytes. */
int vs_grid_header(const char *path, int *dim, int64_t *n);
int vs_read_grid(const char *path, uint8_t *fluid, int64_t cap, int *dim, int64_t *n);
int vs_write_grid(const char *path, const uint8_t *fluid, int dim, int64_t n);

/* Seeded synthetic geometry (BASELINE configs; not a reference function):
 * solidify, in order, the periodic balls (or, with prism_axis >= 0,
 * cylinders along that axis) of the given centres/radii (cell-index
 * coordinates, minimum-image distance <= r) until the fluid count drops
 * to target_fluid or the list ends.  *used = balls consumed.  *n_fluid is
 * in/out: on entry the current fluid count of the mask, or < 0 to count
 * it; on return the count after stamping. */
int vs_stamp_balls(uint8_t *fluid, int dim, int n, const double *centers,
                   const double *radii, int64_t count, int64_t target_fluid,
                   int prism_axis, int64_t *used, int64_t *n_fluid);

/* assemble() (operators.py:209-302): validation, connectivity check, and
 * the on-device geometry build (face masks, DOF ranks, diag codes).
 * inv_h = 1.0/h and inv_h2 = 1.0/h**2 as the reference computes them
 * (operators.py:107-108); the diagonal scale (n/1.0)**2 is exact. */
int vs_ctx_create(const uint8_t *fluid, int dim, int n, int flow_dir,
                  int check_connectivity, int require_walls, int device,
                  double inv_h, double inv_h2, vs_ctx **out);
void vs_ctx_destroy(vs_ctx *ctx);

/* As vs_ctx_create, decomposed into `slabs` x-slabs (1..16, <= n): slab s
 * owns reference x-planes [s*n/slabs, (s+1)*n/slabs) plus one ghost plane
 * per side; the fused inner PCG runs all slabs as groups of one cooperative
 * grid that exchange z ghost planes every iteration and reduce in a fixed
 * slab-major order.  On one GPU this emulates a multi-GPU run of `slabs`
 * ranks (same kernel, same halo/reduction schedule). */
int vs_ctx_create2(const uint8_t *fluid, int dim, int n, int flow_dir,
                   int check_connectivity, int require_walls, int device,
                   double inv_h, double inv_h2, int slabs, vs_ctx **out);
int vs_slab_count(vs_ctx *ctx);

/* Plan the fused inner solves of a single-slab context on `sms` SMs
 * (0 = the whole device), so that independent solves on separate contexts
 * (e.g. the two preconditioners, or a sweep's geometries) run concurrently
 * on disjoint SM shares, each on its context's own stream.  No reference
 * counterpart: the reference runs independent solves in a process pool
 * (cli.py:205-212). */
int vs_ctx_limit_sms(vs_ctx *ctx, int sms);
int vs_ctx_sms(vs_ctx *ctx);
/* Device time (CUDA events) from the start of the last vs_solve_schur on
 * `first` to the end of the last one on `last` (same device): the span of
 * concurrent solves is the max over pairs. */
int vs_solve_span_ms(vs_ctx *first, vs_ctx *last, double *ms);

/* Multi-GPU, one process per GPU: context for rank `rank` of `nranks`
 * (slab decomposition as vs_ctx_create2 with slabs = nranks, but this process
 * holds only its own slab, in one device arena).  Exchange the 64-byte
 * vs_ipc_handle of every rank (e.g. torch.distributed all_gather_object),
 * then vs_ipc_attach with all handles in rank order; afterwards every rank
 * calls the same solves -- the fused kernels exchange ghost planes and
 * reduction partials through peer-mapped NVLink memory and share rank 0's
 * barrier counter.  Host vectors in/out carry only this rank's owned DOFs
 * (in reference positions). */
int vs_ctx_create_rank(const uint8_t *fluid, int dim, int n, int flow_dir,
                       int check_connectivity, int require_walls, int device,
                       double inv_h, double inv_h2, int rank, int nranks,
                       vs_ctx **out);
int vs_ipc_handle(vs_ctx *ctx, void *handle64);
int vs_ipc_attach(vs_ctx *ctx, const void *handles);

/* Host-only slab plan of a mask (no device needed): for each slab 42 int64 =
 * x_lo, x_hi; per family (velocity 0, 1, 2, pressure): own, own_off,
 * glo_off, glo_cnt, ghi_off, ghi_cnt, first_cnt, last_cnt, gstart; then
 * m_own[vel, p], m_all[vel, p].  Local vectors are [owned | ghost planes]. */
int vs_slab_plan(const uint8_t *fluid, int dim, int n, int slabs, int64_t *out);

/* DofMap sizes (operators.py:233-235, :247). */
int vs_counts(vs_ctx *ctx, int64_t *m_u, int64_t *m_p, int64_t axis_counts[3]);

/* Geometry export for parity tests: per-component face masks and the
 * pressure mask as n^dim uint8 grids (nullable), and the integer no-slip
 * diagonal code of every velocity DOF (laplacian_diag = code * n^2). */
int vs_export_geometry(vs_ctx *ctx, uint8_t *face_mask0, uint8_t *face_mask1,
                       uint8_t *face_mask2, uint8_t *pressure_mask,
                       uint8_t *diag_code);

/* Single operator applies, bitwise equal to the reference. */
int vs_apply_laplacian(vs_ctx *ctx, const double *u, double *out);   /* operators.py:131 */
int vs_apply_divergence(vs_ctx *ctx, const double *u, double *out);  /* operators.py:137 */
int vs_apply_gradient(vs_ctx *ctx, const double *p, double *out);    /* operators.py:146 */
int vs_divergence_weighted_diagonal(vs_ctx *ctx, const double *w, double *out); /* :194 */
int vs_apply_simple(vs_ctx *ctx, const double *p, double *out);      /* schur.py:234 */

/* Inner solves (schur.py:200-219, :243-272): fused device PCG.
 * x0 nullable (zeros).  *iters receives the iteration count. */
int vs_solve_velocity(vs_ctx *ctx, const double *rhs, const double *x0,
                      double eps, double *x, int64_t *iters);
int vs_solve_simple(vs_ctx *ctx, const double *r, double eps, double *z,
                    int64_t *iters);

/* solve_schur (schur.py:291-385).  pressure/velocity nullable (stay on the
 * device).  History arrays (nullable) need capacity max_iter+1; alpha/beta
 * capacity max_iter. */
int vs_solve_schur(vs_ctx *ctx, const vs_schur_cfg *cfg, double *pressure,
                   double *velocity, vs_report *rep, double *res_prec,
                   double *res_unprec, double *perm_history, double *alpha,
                   double *beta);

/* The same outer PCG on S with the caller's right-hand side g (m_p values)
 * in place of B A^-1 f -- i.e. krylov.py:76 pcg(outer_op, outer_prec, g) with
 * the operator and preconditioner closures of schur.py:312-327.  For the
 * flow-aligned prismatic C3 geometries g = B A^-1 f is exactly 0, the
 * reference does 0 outer iterations and reports no Lanczos estimate
 * (schur.py:359-362); SURVEY App. B-4 asks for a labelled supplementary
 * estimate from a seeded zero-mean g.  alpha/beta are the CG coefficients
 * lanczos_condition_estimate (krylov.py:185-205) takes.  pressure receives
 * the solution S^-1 g; velocity / perm_history / k_value follow the same
 * code path (u_f + sum alpha w, then the refresh) and carry no physical
 * meaning for an arbitrary g. */
int vs_solve_schur_rhs(vs_ctx *ctx, const vs_schur_cfg *cfg, const double *g,
                       double *pressure, double *velocity, vs_report *rep,
                       double *res_prec, double *res_unprec, double *perm_history,
                       double *alpha, double *beta);

/* Bench hooks: CUDA-event timing of the fused persistent CG launches of the
 * most recent vs_solve_schur / inner solve, split by operator.  dof_iters =
 * sum over launches of (iterations x vector length); launches counts kernel
 * launches of the library in that call (all kernels, not only CG). */
typedef struct {
    int64_t launches;     /* persistent CG launches for this operator   */
    int64_t iterations;   /* CG iterations summed over those launches   */
    int64_t dof_iters;    /* iterations x DOFs summed over launches     */
    double ms;            /* summed CUDA-event duration of the launches */
    int32_t kernel;       /* which fused CG ran: 0 k_pcg (two grid sums per
                             iteration, reference operation order), 1 k_cg1
                             (one grid sum), 2 k_cg1t (one grid sum, tiled), 3 k_pcg
                             with q by recurrence, 4 / 5 k_pcgm (M-scaled over 8-B
                             descriptors; s = M q by recurrence / q recomputed), 6 k_pcgb
                             (experimental: S_hat on a blocked order with shared-memory
                             windows), 7 k_pcgx (the default at scale: alpha from the z
                             sums, z in a ring of buffers, d and x updated every M-th
                             iteration) */
    int32_t reserved;     /* k_pcgx: the ring depth M; k_pcg<QR>: DOFs per P1 step */
    int32_t tier;         /* where the fused CG took its neighbour ranks from:
                             1 bitmask lookups (records smem-cached), 2 ranks in
                             the smem DOF cache, 3 32-bit ranks streamed from
                             HBM, 4 packed deltas streamed from HBM, 5 8-B
                             descriptors streamed from HBM (k_pcgm, k_pcgx) */
    int32_t escape_ppm;   /* tier 5 (8-B descriptors): DOFs per million whose neighbour
                             distances do not fit the descriptor; k_pcgm takes their
                             ranks from the record + bitmask lookup, k_pcgx from its
                             escape table */
} vs_kstat;

int vs_kernel_stats(vs_ctx *ctx, vs_kstat *velocity_cg, vs_kstat *simple_cg,
                    int64_t *total_kernel_launches);

/* Debug: with VOXSCHUR_PHASE_TIMING set at context creation, %globaltimer
 * nanoseconds spent in {P1 pass, reduction 1, P2 pass, reduction 2} since
 * the last call (then reset): ns12[0..3] block 0, [4..7] max over blocks,
 * [8..11] sum over blocks.  Zeros otherwise. */
int vs_phase_timing(vs_ctx *ctx, double *ns12);

#ifdef __cplusplus
}
#endif
#endif /* VOXSCHUR_H */
