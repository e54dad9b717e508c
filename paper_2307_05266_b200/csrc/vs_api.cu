// vs_api.cu -- C ABI (include/voxschur.h): context, geometry build, unit
// applies, inner solves and the host-driven outer Schur loop.
//
// The outer loop restates solve_schur (schur.py:291-385) step by step; the
// inner solves are one persistent cooperative launch each (vs_kernels.cu
// k_pcg).  The host synchronises once per inner solve (iteration count and
// status are needed for inner_iter_totals and the reference's errors) and
// once per outer reduction -- O(outer iterations) syncs per solve.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/voxschur.h"
#include "vs_internal.h"

using namespace vs;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

struct CudaFail {
    cudaError_t e;
    const char *what;
};

#define CK(call)                                                  \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) throw CudaFail{e_, #call};         \
    } while (0)

struct Status {
    int code;
    std::string msg;
};

}  // namespace

namespace vs {
void set_last_error(const std::string &msg) { g_err = msg; }
}  // namespace vs

namespace {
// The device's default stream-ordered pool keeps freed memory instead of
// returning it to the driver at each synchronisation, so a context built
// after another one was destroyed allocates without driver calls.
void keep_pool(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
}
}  // namespace

namespace {

// ----------------------------------------------------------------- slabs
// Vector slots of a slab.  Velocity slots have m_all[0] entries, pressure
// slots m_all[1]; owned DOFs first, ghost-plane DOFs after.
enum USlot { U_RHS, U_W, U_ITER, U_F, U_R, U_Z, U_D0, U_D1, U_CQ, U_S0, U_S1, U_TMP, U_IN, NU };
enum PSlot { P_X, P_R, P_D, P_Z, P_Q, P_B, P_SR, P_SZ, P_SD0, P_SD1, P_SQ, P_SS0, P_SS1, P_TMP, P_IN, NP };
constexpr int FP = 3;  // family index of the pressure (velocity components are 0..dim-1)

// One group of the decomposition: a slab of x-planes [x_lo, x_hi) with one
// ghost plane on each side.  With a single group it is the whole periodic
// domain (nx = n, no ghosts, local numbering == reference numbering).
struct Slab {
    int x_lo = 0, x_hi = 0, P = 0, nx = 0;
    int64_t own[4] = {0, 0, 0, 0}, own_off[4] = {0, 0, 0, 0};
    int64_t glo_off[4] = {0, 0, 0, 0}, glo_cnt[4] = {0, 0, 0, 0};
    int64_t ghi_off[4] = {0, 0, 0, 0}, ghi_cnt[4] = {0, 0, 0, 0};
    int64_t first_cnt[4] = {0, 0, 0, 0}, last_cnt[4] = {0, 0, 0, 0};
    int64_t gstart[4] = {0, 0, 0, 0};  // global rank of the first owned DOF per family
    int64_t m_own[2] = {0, 0}, m_all[2] = {0, 0};
    uint2 *meta[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t *vrec = nullptr, *prec = nullptr;
    uint32_t *nbr[2] = {nullptr, nullptr};  // TIER-3 neighbour ranks (A, S_hat), built on first use
    // k_pcgm descriptors (A, S_hat), built on first use
    uint64_t *desc[2] = {nullptr, nullptr};
    uint16_t *cidx[2] = {nullptr, nullptr};
    int2 *xb[2] = {nullptr, nullptr};  // x+ / x- rank-distance bases per chunk of 1024 ranks
    unsigned *lbar = nullptr;  // hierarchical barrier: this slab's local arrival counter and release word (in its arena)
    uint32_t *esc[2] = {nullptr, nullptr};  // escape table: the gather indices of the DOFs outside the descriptor format
    // k_pcgb (S_hat, blocked order): 0 = not built, 1 = built, -1 = not applicable here
    int blk_state = 0;
    uint32_t *blk_lineR = nullptr, *blk_lineI = nullptr, *blk_tile0 = nullptr, *blk_tl_src = nullptr;
    uint16_t *blk_tl_len = nullptr, *blk_tl_v = nullptr, *blk_vidx = nullptr, *blk_cidx = nullptr;
    uint64_t *blk_desc = nullptr;
    int blk_ntiles = 0, blk_vcap = 0, blk_vbuf = 1;
    int64_t n_escape[2] = {0, 0};
    double *u[NU] = {}, *p[NP] = {};
    Geo geo{};
};

}  // namespace

struct vs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int dim = 0, n = 0, nw = 0, nlines = 0, flow_dir = 0, R = 1;
    int64_t nwords = 0, ncells = 0;
    int64_t m_u = 0, m_p = 0, vcount[3] = {0, 0, 0}, voff[3] = {0, 0, 0};
    double inv_h = 0, inv_h2 = 0, diag_scale = 0;
    double diag_code[16] = {0}, inv_code[16] = {0}, invA_enc[8] = {0};
    bool sdiag_ok = true;
    std::vector<void *> allocs, ipc_allocs;
    // global geometry (reference numbering)
    uint32_t *fbits = nullptr;
    uint2 *vmeta[3] = {nullptr, nullptr, nullptr};
    uint2 *pmeta = nullptr;
    uint64_t *vrec = nullptr, *prec = nullptr;
    double2 *sdiag2 = nullptr;
    double2 *ctab[2] = {nullptr, nullptr};  // k_pcgm: {1/diag, diag} by code index
    double *invS = nullptr, *d_diag_code = nullptr, *d_invA_enc = nullptr;
    std::vector<int64_t> pstart[4];  // global rank of the first DOF of plane x, x in [0, n]
    std::vector<Slab> slabs;
    CgGroup *d_groups = nullptr, *h_groups = nullptr;  // [R] device / pinned staging
    unsigned *bar = nullptr;
    unsigned long long *phase_ns = nullptr;  // VOXSCHUR_PHASE_TIMING=1
    double *part = nullptr, *red_part = nullptr, *scal = nullptr;
    CgOut *cgout = nullptr;
    // async inner solves: CgOut log + event pool (read back once per outer iteration)
    CgOut *cglog = nullptr, *h_cglog = nullptr;
    int ncglog = 0, cglog_cap = 0;
    std::vector<cudaEvent_t> evpool;
    std::vector<int> log_op;
    OuterState *ost = nullptr, *h_ost = nullptr;
    double *hist = nullptr;
    int64_t hist_cap = 0;
    double *h_scal = nullptr;  // pinned
    CgOut *h_cg = nullptr;     // pinned
    CgPlan plan_A{}, plan_S{};
    int64_t mu_max = 0, mp_max = 0;  // largest slab's owned DOFs (the plans' sizes)
    int sms = 0;                     // SMs the fused solves are planned on
    TilePlan tile_A{}, tile_S{};  // k_cg1t plans (one slab, 3D); used when use_tile[op]
    bool use_tile[2] = {false, false};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;
    vs_kstat st_A{}, st_S{};  // stats of the last top-level call
    int64_t launches = 0;
    // L2 prefetch of k_pcg's own streams one grid stride ahead (B200, C4 512^3:
    // S_hat 756 -> 652, A 1551 -> 1444 us/it; C2: A 123 -> 110; distance 2
    // and 4 are worse); VOXSCHUR_PREFETCH overrides (0 = off)
    uint32_t pf_dist = 1;
    bool pf_forced = false;

    Geo geo() const {
        Geo g;
        g.dim = dim; g.n = n; g.nw = nw; g.nlines = nlines; g.nx = n;
        g.fbits = fbits;
        for (int a = 0; a < 3; ++a) g.vmeta[a] = vmeta[a];
        g.pmeta = pmeta;
        return g;
    }
    // Device memory comes from the device's stream-ordered pool (released
    // back to the pool, not the driver, on destroy): building and destroying
    // contexts costs no device-wide synchronisation and reuses the memory of
    // earlier contexts.  The slab arena of a multi-process context is an
    // ordinary allocation (it is exported with cudaIpcGetMemHandle).
    template <class T>
    T *alloc(size_t count) {
        void *p = nullptr;
        CK(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), stream));
        allocs.push_back(p);
        return (T *)p;
    }
    template <class T>
    T *alloc_ipc(size_t count) {
        void *p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        ipc_allocs.push_back(p);
        return (T *)p;
    }
    ~vs_ctx() {
        if (device >= 0) cudaSetDevice(device);
        if (tile_A.mem) cudaFree(tile_A.mem);
        if (tile_S.mem) cudaFree(tile_S.mem);
        for (void *p : allocs) cudaFreeAsync(p, stream);
        for (void *p : ipc_allocs) cudaFree(p);
        if (h_scal) cudaFreeHost(h_scal);
        if (h_cg) cudaFreeHost(h_cg);
        if (h_groups) cudaFreeHost(h_groups);
        if (h_cglog) cudaFreeHost(h_cglog);
        if (h_ost) cudaFreeHost(h_ost);
        for (cudaEvent_t e : evpool) cudaEventDestroy(e);
        for (void *p : peer_arena)
            if (p) cudaIpcCloseMemHandle(p);
        for (cudaEvent_t e : {ev0, ev1, evs0, evs1})
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
    // multi-GPU runs: a cross-GPU barrier that gave up sets *xflag_dev (device memory, read back after a sync)
    int *xflag_dev = nullptr;
    unsigned long long xtimeout_ns = 0;
    void sync() {
        CK(cudaStreamSynchronize(stream));
        if (xflag_dev) {
            int h = 0;
            CK(cudaMemcpy(&h, xflag_dev, sizeof h, cudaMemcpyDeviceToHost));
            if (h) {
                char buf[200];
                snprintf(buf, sizeof buf, "cross-rank barrier timed out after %.0f s: a peer rank never arrived "
                         "(this context is unusable; destroy it on every rank)", (double)xtimeout_ns * 1e-9);
                throw Status{VS_ECUDA, buf};
            }
        }
    }
    int nfam() const { return dim; }
    // ---- slab-distributed helpers.  Slabs [s0, s1) are local (all of them
    // in one process, or this rank's one on a multi-process run); remote
    // slabs' vectors are peer-mapped pointers.  Loops run in slab order.
    int s0 = 0, s1 = 1;                 // local slabs
    int rank = 0, nranks = 1;           // process-level decomposition (nranks > 1: one slab per process)
    double *scal_peer[VS_MAX_SLABS] = {};  // every rank's reduction slots
    double *part_peer[VS_MAX_SLABS] = {};  // every rank's CG partial buffer
    unsigned *bar_base = nullptr;       // local: value of the barrier counter after the last launch
    char *arena = nullptr;              // this process's first local slab arena (IPC-exported)
    void *peer_arena[VS_MAX_SLABS] = {};  // opened IPC mappings (closed on destroy)
    int64_t tb_max = 0;
    int npart = 1;
    bool hier_barrier = false;          // multi-rank runs: ranks arrive through leaders (VOXSCHUR_HIER_BARRIER=0|1 overrides)
    bool mp() const { return nranks > 1; }
    // cross-rank device barrier (one arrival per rank; same counter as the CG)
    void xbar() {
        if (!mp()) return;
        launch_xbar(bar, bar_base, nranks, xflag_dev, xtimeout_ns, stream);
        ++launches;
    }
    // make this rank's reduction slots [q0, q1) visible in every rank's scal
    void publish(int q0, int q1) {
        if (!mp()) return;
        for (int r = 0; r < nranks; ++r) {
            if (r == rank) continue;
            for (int q = q0; q < q1; ++q)
                CK(cudaMemcpyAsync(scal_peer[r] + q * R + rank, scal + q * R + rank, sizeof(double),
                                   cudaMemcpyDeviceToDevice, stream));
        }
        xbar();
    }
    // deterministic reduction over the owned DOFs of every slab, result on host
    double reduce(int space, int kind, int a, int b, int64_t lo_fam = -1) {
        reduce_dev(space, kind, a, b, Q_HOST, lo_fam);
        publish(Q_HOST, Q_HOST + 1);
        CK(cudaMemcpyAsync(h_scal, scal + Q_HOST * R, R * sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
        double tot = h_scal[0];
        for (int s = 1; s < R; ++s) tot = tot + h_scal[s];
        return tot;
    }
    double dot(int space, int a, int b) { return reduce(space, 1, a, b); }
    double sum(int space, int a) { return reduce(space, 0, a, -1); }
    double mean(int space, int a) { return sum(space, a) / (double)(space == 0 ? m_u : m_p); }
    // outer-loop gate: while vs_solve_schur enqueues several outer iterations ahead of
    // the host, every kernel of the loop gets &ost->stop and turns into a no-op once the
    // outer PCG has converged or failed; nullptr everywhere else
    const int *gate = nullptr;
    void vec(int space, int kind, int out, int a, int b, double sc, const double *sp = nullptr) {
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            double **v = space == 0 ? S.u : S.p;
            launch_vec(kind, out < 0 ? nullptr : v[out], v[a], b < 0 ? nullptr : v[b], sc, sp, S.m_own[space],
                       stream, gate);
            ++launches;
        }
    }
    // device-resident reduction into slot q (scal[q*R + s]); no host sync
    // (callers publish() before a k_outer step reads the slots of all slabs)
    void reduce_dev(int space, int kind, int a, int b, int q, int64_t lo_fam = -1) {
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            const double *pa = space == 0 ? S.u[a] : S.p[a];
            const double *pb = b < 0 ? nullptr : (space == 0 ? S.u[b] : S.p[b]);
            int64_t off = 0, m = S.m_own[space];
            if (lo_fam >= 0) { off = S.own_off[lo_fam]; m = S.own[lo_fam]; }
            launches += launch_reduce(kind, pa + off, pb ? pb + off : nullptr, m, red_part, scal + q * R + s, stream,
                                      gate);
        }
    }
    void copy(int space, int dst, int src) {
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            double **v = space == 0 ? S.u : S.p;
            if (S.m_own[space])
                CK(cudaMemcpyAsync(v[dst], v[src], S.m_own[space] * sizeof(double), cudaMemcpyDeviceToDevice,
                                   stream));
        }
    }
    // push every local slab's boundary planes into the neighbours' ghost
    // planes (first owned plane -> lower slab's ghost_hi, last -> upper's
    // ghost_lo); peer stores over NVLink on a multi-process run
    void halo(int space, int slot) {
        if (R == 1) return;
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s], &lo = slabs[(s - 1 + R) % R], &hi = slabs[(s + 1) % R];
            const int nf = space == 0 ? dim : 1;
            const double *src = space == 0 ? S.u[slot] : S.p[slot];
            double *dlo = space == 0 ? lo.u[slot] : lo.p[slot];
            double *dhi = space == 0 ? hi.u[slot] : hi.p[slot];
            for (int k = 0; k < nf; ++k) {
                const int f = space == 0 ? k : FP;
                if (S.first_cnt[f])
                    CK(cudaMemcpyAsync(dlo + lo.ghi_off[f], src + S.own_off[f], S.first_cnt[f] * sizeof(double),
                                       cudaMemcpyDeviceToDevice, stream));
                if (S.last_cnt[f])
                    CK(cudaMemcpyAsync(dhi + hi.glo_off[f], src + S.own_off[f] + S.own[f] - S.last_cnt[f],
                                       S.last_cnt[f] * sizeof(double), cudaMemcpyDeviceToDevice, stream));
            }
        }
        xbar();  // every rank's pushes land before anyone reads its ghosts
    }
    // host (reference order) -> local slabs, owned and ghost planes
    void upload(int space, int slot, const double *h) {
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            double *dst = space == 0 ? S.u[slot] : S.p[slot];
            const int nf = space == 0 ? dim : 1;
            for (int k = 0; k < nf; ++k) {
                const int f = space == 0 ? k : FP;
                auto put = [&](int64_t loff, int64_t goff, int64_t cnt) {
                    if (cnt) CK(cudaMemcpyAsync(dst + loff, h + goff, cnt * sizeof(double), cudaMemcpyHostToDevice,
                                                stream));
                };
                put(S.own_off[f], S.gstart[f], S.own[f]);
                if (R > 1) {
                    put(S.glo_off[f], pstart[f][(S.x_lo - 1 + n) % n], S.glo_cnt[f]);
                    put(S.ghi_off[f], pstart[f][S.x_hi % n], S.ghi_cnt[f]);
                }
            }
        }
    }
    // local slabs' owned DOFs -> host vector (reference order)
    void download(int space, int slot, double *h) {
        if (!h) return;
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            const double *src = space == 0 ? S.u[slot] : S.p[slot];
            const int nf = space == 0 ? dim : 1;
            for (int k = 0; k < nf; ++k) {
                const int f = space == 0 ? k : FP;
                if (S.own[f])
                    CK(cudaMemcpyAsync(h + S.gstart[f], src + S.own_off[f], S.own[f] * sizeof(double),
                                       cudaMemcpyDeviceToHost, stream));
            }
        }
    }
    // ---- outer operators on every local slab (ghosts of the input refreshed first)
    void grad(int p_in, int u_out) {  // B^T: needs p at I - e_a
        halo(1, p_in);
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            launch_apply_grad(S.geo, S.vrec, S.p[p_in], S.u[u_out], S.m_own[0], inv_h, stream, gate);
            ++launches;
        }
    }
    void div(int u_in, int p_out) {  // B: needs u at I + e_a
        halo(0, u_in);
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            launch_apply_div(S.geo, S.prec, S.u[u_in], S.p[p_out], S.m_own[1], inv_h, stream, gate);
            ++launches;
        }
    }
    void force(int out, int sub) {  // out = force (- sub)
        for (int s = s0; s < s1; ++s) {
            Slab &S = slabs[s];
            launch_force(S.u[out], sub < 0 ? nullptr : S.u[sub], S.own_off[flow_dir], S.own[flow_dir], S.m_own[0],
                         stream);
            ++launches;
        }
    }
};

namespace {

// ------------------------------------------------------------ components

struct UF {
    std::vector<int64_t> p;
    explicit UF(int64_t n) : p(n) { std::iota(p.begin(), p.end(), 0); }
    int64_t find(int64_t i) {
        while (p[i] != i) { p[i] = p[p[i]]; i = p[i]; }
        return i;
    }
    void unite(int64_t a, int64_t b) {
        a = find(a); b = find(b);
        if (a != b) { if (a < b) p[b] = a; else p[a] = b; }
    }
};

// periodic face-adjacency labelling, ids in first C-order appearance
// (geometry.py:183-222: ndimage.label + periodic union-find)
int64_t label_components(const uint8_t *f, int dim, int n, int32_t *labels) {
    const int64_t N = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    UF uf(N);
    const int64_t strides[3] = {dim == 3 ? (int64_t)n * n : (int64_t)n, dim == 3 ? (int64_t)n : 1, 1};
    for (int64_t i = 0; i < N; ++i) {
        if (!f[i]) continue;
        int64_t rem = i;
        for (int a = 0; a < dim; ++a) {
            const int64_t s = strides[a];
            const int64_t coord = (rem / s) % n;
            const int64_t j = coord == n - 1 ? i - (int64_t)(n - 1) * s : i + s;
            if (f[j]) uf.unite(i, j);
        }
    }
    std::vector<int32_t> id(labels ? 0 : N, -1);
    int32_t *ids = labels ? labels : id.data();
    // first pass: assign ids to roots in first-appearance order
    std::vector<int32_t> rootid;
    int32_t next = 0;
    for (int64_t i = 0; i < N; ++i) ids[i] = -1;
    for (int64_t i = 0; i < N; ++i) {
        if (!f[i]) continue;
        const int64_t r = uf.find(i);
        if (ids[r] < 0 && r <= i) {
            // the root is the minimum index of its class, so it is the class's
            // first cell in C-order: it is always visited first
            ids[r] = next++;
        }
        ids[i] = ids[r];
    }
    return next;
}

Status cg_status_to_error(const CgOut &o, int which) {
    char buf[512];
    if (o.status == 1) {
        snprintf(buf, sizeof buf, "preconditioner not SPD on subspace: r'z = %.3e at iteration %lld", o.value,
                 (long long)o.at_iter);
        return {VS_ERUNTIME, buf};
    }
    if (o.status == 2) {
        snprintf(buf, sizeof buf, "operator not SPD on subspace: d'q = %.3e at iteration %lld", o.value,
                 (long long)o.at_iter);
        return {VS_ERUNTIME, buf};
    }
    if (o.status == 3) {
        snprintf(buf, sizeof buf, "non-finite residual at iteration %lld", (long long)o.at_iter);
        return {VS_ERUNTIME, buf};
    }
    if (o.status == 4) return {VS_ECUDA, "cross-rank barrier timed out inside a fused inner solve"};
    if (!o.converged) {
        // schur.py:214-218 / :266-271
        snprintf(buf, sizeof buf,
                 which == 0 ? "inner velocity solve did not converge: relative residual %.3e after %lld iterations"
                            : "inner pressure preconditioner solve did not converge: relative residual %.3e after "
                              "%lld iterations",
                 o.res_prec_last / o.res_prec0, (long long)o.iterations);
        return {VS_ERUNTIME, buf};
    }
    return {VS_OK, ""};
}

inline bool is_m_alg(int alg) {
    return alg == CG_TWO_SUM_MQ || alg == CG_TWO_SUM_MRC || alg == CG_BLOCKED || alg == CG_TWO_SUM_MX;
}

// k_pcgm descriptors of one slab and operator (vs_cgm.cu): the x-bases per
// chunk of 1024 ranks, then the packed descriptors.  Runs once, on the first
// solve that needs it.
void build_descriptors(vs_ctx *c, Slab &S, const CgGroup &G, int op) {
    const int64_t m = std::max<int64_t>(1, S.m_own[op]);
    const int64_t nchunk = (m + 1023) / 1024;
    int2 *xb = c->alloc<int2>(nchunk);
    CK(cudaMemsetAsync(xb, 0x7F, (size_t)nchunk * sizeof(int2), c->stream));  // 0x7F7F7F7F: "no such neighbour here"
    launch_desc_scan(c->dim, op, G, c->n, c->nw, xb, c->stream);
    CK(cudaGetLastError());
    S.desc[op] = c->alloc<uint64_t>(m + 16);  // k_pcgx's bulk copies round a chunk's size up to 16 B
    S.cidx[op] = c->alloc<uint16_t>(m + 16);
    unsigned long long *cnt = c->alloc<unsigned long long>(1);
    CK(cudaMemsetAsync(cnt, 0, sizeof *cnt, c->stream));
    // escape table: room for 1/16 of the DOFs (C4 512^3: 0.6 % escape; every DOF under the test
    // hook VOXSCHUR_DESC_ESCAPE, where the slots run out and the rest take the record path)
    uint32_t esc_cap = (uint32_t)std::min<int64_t>(m / 16 + 4096, (int64_t)1 << 30);
    if (const char *e = getenv("VOXSCHUR_ESC_CAP"))  // test hook: a small table, so that both escape paths run
        if (atoll(e) >= 0) esc_cap = (uint32_t)std::min<int64_t>(atoll(e), esc_cap);
    S.esc[op] = c->alloc<uint32_t>((size_t)8 * esc_cap + 8);
    launch_desc_pack(c->dim, op, G, c->n, c->nw, xb, S.desc[op], S.cidx[op], cnt, S.esc[op], esc_cap, c->stream);
    CK(cudaGetLastError());
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, cnt, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    S.n_escape[op] = (int64_t)h;
    S.xb[op] = xb;
    if (!c->ctab[op]) {
        const int count = op == 0 ? 16 : 46656;
        c->ctab[op] = c->alloc<double2>(count);
        launch_build_ctab(op, c->sdiag2, c->d_diag_code, c->ctab[op], count, c->stream);
        CK(cudaGetLastError());
    }
}

// k_pcgb tables of the (single) slab's pressure family: line starts in both orders,
// tiles, line slots and window offsets (host), then the per-DOF descriptors (device).
// Leaves S.blk_state = -1 where the blocked kernel does not apply.
void build_blocked(vs_ctx *c, Slab &S, const CgGroup &G) {
    constexpr int TB = 8, TS = 10, NSLOT = 100;
    const int n = c->n;
    S.blk_state = -1;
    if (c->dim != 3 || c->R != 1 || n % TB || n < 2 * TB || !S.m_own[1]) return;
    const size_t nl = (size_t)n * n;
    std::vector<uint32_t> R(nl + 1), I(nl);
    // meta[(x*n + y) * nw].y = reference rank of the line's first DOF
    CK(cudaMemcpy2DAsync(R.data(), sizeof(uint32_t), reinterpret_cast<const char *>(c->pmeta) + sizeof(uint32_t),
                         (size_t)c->nw * sizeof(uint2), sizeof(uint32_t), nl, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    R[nl] = (uint32_t)S.m_own[1];
    const int nt = n / TB, ntiles = nt * nt;
    std::vector<uint32_t> tile0(ntiles + 1), tl_src((size_t)ntiles * NSLOT, 0);
    std::vector<uint16_t> tl_len((size_t)ntiles * NSLOT, 0), tl_v((size_t)ntiles * NSLOT, 0);
    uint32_t run = 0;
    for (int X = 0; X < nt; ++X)
        for (int Y = 0; Y < nt; ++Y) {
            tile0[X * nt + Y] = run;
            for (int px = 0; px < TB; ++px)
                for (int py = 0; py < TB; ++py) {
                    const size_t l = (size_t)(X * TB + px) * n + (Y * TB + py);
                    I[l] = run;
                    run += R[l + 1] - R[l];
                }
        }
    tile0[ntiles] = run;
    int vcap = 0;
    for (int X = 0; X < nt; ++X)
        for (int Y = 0; Y < nt; ++Y) {
            const size_t t = (size_t)X * nt + Y;
            uint32_t cur = 0;
            for (int px = -1; px <= TB; ++px)
                for (int py = -1; py <= TB; ++py) {
                    if ((px < 0 || px == TB) && (py < 0 || py == TB)) continue;  // corners: no neighbour there
                    const size_t l = (size_t)((X * TB + px + n) % n) * n + (size_t)((Y * TB + py + n) % n);
                    const uint32_t L = R[l + 1] - R[l];
                    const size_t k = t * NSLOT + (size_t)(px + 1) * TS + (py + 1);
                    if (!L) continue;
                    if (L > 500) return;  // y distances must fit 10 bits
                    cur += 1;  // pad: the line's last DOF (periodic z wrap)
                    tl_src[k] = I[l];
                    tl_len[k] = (uint16_t)L;
                    tl_v[k] = (uint16_t)cur;
                    cur += L + 1;  // + pad: the line's first DOF
                    if (cur > 60000) return;
                }
            vcap = std::max<int>(vcap, (int)cur + 2);
        }
    vcap = (vcap + 1) & ~1;  // windows 16-B aligned
    const int vbuf = pcgb_fits(vcap, c->device);
    if (!vbuf) return;
    S.blk_vbuf = (getenv("VOXSCHUR_BLK_BUFS") && atoi(getenv("VOXSCHUR_BLK_BUFS")) == 1) ? 1 : vbuf;
    auto up = [&](auto *&dst, const auto &v) {
        using T = typename std::remove_reference<decltype(v[0])>::type;
        dst = c->alloc<typename std::remove_const<T>::type>(v.size());
        CK(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    };
    up(S.blk_lineR, R);
    up(S.blk_lineI, I);
    up(S.blk_tile0, tile0);
    up(S.blk_tl_src, tl_src);
    up(S.blk_tl_len, tl_len);
    up(S.blk_tl_v, tl_v);
    const int64_t m = S.m_own[1];
    S.blk_desc = c->alloc<uint64_t>(m);
    S.blk_vidx = c->alloc<uint16_t>(m);
    S.blk_cidx = c->alloc<uint16_t>(m);
    int *bad = c->alloc<int>(1);
    CK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    launch_blk_build(G, n, c->nw, S.blk_lineR, S.blk_lineI, S.blk_tl_v, S.blk_desc, S.blk_vidx, S.blk_cidx, bad,
                     c->stream);
    CK(cudaGetLastError());
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();  // the host tables must outlive their uploads
    if (hbad) return;  // a window distance did not fit its field
    if (!c->ctab[1]) {
        c->ctab[1] = c->alloc<double2>(46656);
        launch_build_ctab(1, c->sdiag2, c->d_diag_code, c->ctab[1], 46656, c->stream);
        CK(cudaGetLastError());
    }
    S.blk_ntiles = ntiles;
    S.blk_vcap = vcap;
    S.blk_state = 1;
}

constexpr int GROUP_RING = 8;  // group-table staging slots (>= launches between syncs)

// Launch one fused device PCG solve over all slabs (one cooperative launch)
// without waiting: its CgOut goes to log slot c->ncglog (returned), its
// launch time to an event pair of the pool.  op 0: velocity A (x0
// allowed), op 1: S_hat (projected).  Slots index the slab vectors.
int cg_async(vs_ctx *c, int op, int rhs, int x0, double eps, int x) {
    const int64_t m = op == 0 ? c->m_u : c->m_p;
    const int R = c->R;
    if (c->ncglog >= c->cglog_cap) throw Status{VS_ECUDA, "inner-solve log overflow"};
    const int li = c->ncglog++;
    c->log_op.resize(c->ncglog);
    c->log_op[li] = op;
    if (m == 0) {
        CK(cudaMemsetAsync(c->cglog + li, 0, sizeof(CgOut), c->stream));
        return li;
    }
    if (x0 >= 0) c->halo(op == 0 ? 0 : 1, x0);  // A x0 needs x0 on the ghost planes
    // k_pcgb (S_hat on the blocked order): built on first use; where it does not apply
    // (2D, slabs, n not a multiple of 8, ...) the solve takes k_pcgm
    bool use_blocked = false;
    if (op == 1 && c->plan_S.alg == CG_BLOCKED && x0 < 0 && !c->use_tile[1]) {
        Slab &S0 = c->slabs[c->s0];
        if (S0.blk_state == 0) {
            CgGroup G0{};
            memset(&G0, 0, sizeof G0);
            G0.meta[0] = S0.meta[FP];
            G0.rec = S0.prec;
            G0.nx = S0.nx;
            G0.m_own = (uint32_t)S0.m_own[1];
            build_blocked(c, S0, G0);
        }
        use_blocked = S0.blk_state == 1;
    }
    const int ring = li % GROUP_RING;
    const int nloc = c->s1 - c->s0;
    CgGroup *hg = c->h_groups + ring * nloc;
    for (int s = c->s0; s < c->s1; ++s) {
        Slab &S = c->slabs[s];
        CgGroup &G = hg[s - c->s0];
        memset(&G, 0, sizeof G);
        double **v = op == 0 ? S.u : S.p;
        if (op == 0) {
            for (int a = 0; a < 3; ++a) G.meta[a] = S.meta[a];
        } else {
            G.meta[0] = S.meta[FP];
        }
        G.rec = op == 0 ? S.vrec : S.prec;
        G.nx = S.nx;
        G.m_own = (uint32_t)S.m_own[op];
        G.m_all = (uint32_t)S.m_all[op];
        G.rhs = v[rhs];
        G.x0 = x0 >= 0 ? v[x0] : nullptr;
        G.x = v[x];
        G.r = op == 0 ? S.u[U_R] : S.p[P_SR];
        G.z = op == 0 ? S.u[U_Z] : S.p[P_SZ];
        G.d0 = op == 0 ? S.u[U_D0] : S.p[P_SD0];
        G.d1 = op == 0 ? S.u[U_D1] : S.p[P_SD1];
        G.q = op == 0 ? S.u[U_CQ] : S.p[P_SQ];
        const int tier = (op == 0 ? c->plan_A : c->plan_S).tier;
        if (tier == 3 || tier == 4) {  // TIER 3 rank / TIER 4 delta table, built on first use
            uint32_t *&nb = S.nbr[op];
            if (!nb) {
                // TIER 3: 2*dim ranks; TIER 4: int2 x-deltas (+ short2 y-deltas in 3D)
                const size_t words = tier == 4 ? (c->dim == 3 ? 3 : 2) : 2 * c->dim;
                nb = c->alloc<uint32_t>(words * std::max<int64_t>(1, S.m_own[op]));
                launch_build_nbr(c->dim, op, G, c->n, c->nw, nb, c->stream, tier);
                CK(cudaGetLastError());
            }
            G.nbr = nb;
        }
        if (is_m_alg((op == 0 ? c->plan_A : c->plan_S).alg) && !use_blocked) {
            if (!S.desc[op]) build_descriptors(c, S, G, op);
            G.desc = S.desc[op];
            G.cidx = S.cidx[op];
            G.xb = S.xb[op];
            G.esc = reinterpret_cast<const uint4 *>(S.esc[op]);
        }
        if (use_blocked) {  // k_pcgb: the solve runs in the blocked order
            G.desc = S.blk_desc;
            G.cidx = S.blk_cidx;
            G.vidx = S.blk_vidx;
            G.tile0 = S.blk_tile0;
            G.tl_src = S.blk_tl_src;
            G.tl_len = S.blk_tl_len;
            G.tl_v = S.blk_tl_v;
            G.ntiles = S.blk_ntiles;
            G.vcap = S.blk_vcap;
            G.vbuf = S.blk_vbuf;
            launch_blk_perm(S.prec, c->n, S.blk_lineR, S.blk_lineI, (uint32_t)S.m_own[1], v[rhs], S.p[P_SR], 1,
                            c->stream);
            ++c->launches;
            G.rhs = S.p[P_SR];
            G.x = S.p[P_SS0];
        }
        // k_cg1 buffers (the same slots, paired)
        G.zb[0] = G.z;
        G.zb[1] = G.r;
        G.ub[0] = G.d1;
        G.ub[1] = G.q;
        G.sb[0] = op == 0 ? S.u[U_S0] : S.p[P_SS0];
        G.sb[1] = op == 0 ? S.u[U_S1] : S.p[P_SS1];
        // k_pcgx: the z ring (d = d0, s = q as in k_pcgm)
        static const int ring_u[4] = {U_Z, U_R, U_D1, U_S0}, ring_p[4] = {P_SZ, P_SR, P_SD1, P_SS0};
        for (int b = 0; b < 4; ++b) G.zr[b] = op == 0 ? S.u[ring_u[b]] : S.p[ring_p[b]];
        if (R > 1) {
            Slab &lo = c->slabs[(s - 1 + R) % R], &hi = c->slabs[(s + 1) % R];
            G.zpeer[0] = op == 0 ? lo.u[U_Z] : lo.p[P_SZ];
            G.zpeer[1] = op == 0 ? hi.u[U_Z] : hi.p[P_SZ];
            for (int b = 0; b < 4; ++b) {
                G.zrp[0][b] = op == 0 ? lo.u[ring_u[b]] : lo.p[ring_p[b]];
                G.zrp[1][b] = op == 0 ? hi.u[ring_u[b]] : hi.p[ring_p[b]];
            }
            const int nf = op == 0 ? c->dim : 1;
            for (int k = 0; k < nf; ++k) {
                const int f = op == 0 ? k : FP;
                G.sbeg[0][k] = (uint32_t)S.own_off[f];
                G.send[0][k] = (uint32_t)(S.own_off[f] + S.first_cnt[f]);
                G.sdst[0][k] = (uint32_t)lo.ghi_off[f];
                G.sbeg[1][k] = (uint32_t)(S.own_off[f] + S.own[f] - S.last_cnt[f]);
                G.send[1][k] = (uint32_t)(S.own_off[f] + S.own[f]);
                G.sdst[1][k] = (uint32_t)hi.glo_off[f];
            }
        }
    }
    CgGroup *dg = c->d_groups + ring * nloc;
    CK(cudaMemcpyAsync(dg, hg, nloc * sizeof(CgGroup), cudaMemcpyHostToDevice, c->stream));
    CgParams P{};
    memset(&P, 0, sizeof P);
    P.groups = dg;
    P.group_base = 0;  // groups[] holds this process's slabs only
    P.n = c->n;
    P.nw = c->nw;
    P.m_global = (double)m;
    P.part = c->part;
    P.bar = c->bar;
    P.bar_base = c->bar_base;
    P.npart = c->npart;
    P.xgpu = c->mp() ? 1 : 0;
    P.xflag = c->xflag_dev;
    P.xtimeout_ns = c->xtimeout_ns;
    P.part_self = c->mp() ? c->rank : 0;
    for (int r = 0; r < c->npart; ++r) P.part_peer[r] = c->part_peer[r];
    // hierarchical barrier (multi-rank runs): the local words live in each local slab's arena
    P.hier = (c->npart > 1 && c->hier_barrier && (op == 0 ? c->plan_A : c->plan_S).alg == CG_TWO_SUM_MX) ? 1 : 0;  // k_pcgx<MR> carries it
    P.nranks_bar = c->npart;
    for (int q = c->s0; q < c->s1; ++q) P.lbar[P.part_self + (q - c->s0)] = c->slabs[q].lbar;
    P.phase_ns = c->phase_ns;
    P.gate = c->gate;
    if (const char *e = getenv("VOXSCHUR_DBG")) P.dbg = (uint32_t)atoi(e);
    P.out = c->cglog + li;
    P.tol = eps;
    P.max_iter = std::max<int64_t>(1000, 2 * m);  // schur.py:196-197
    // test hook: a lower cap, to drive the "did not converge" paths of
    // schur.py:214-218 / :266-271 (the reference's cap cannot be reached on
    // an SPD operator in exact arithmetic)
    if (const char *e = getenv("VOXSCHUR_INNER_MAXIT"))
        if (atoll(e) > 0) P.max_iter = std::min<int64_t>(P.max_iter, atoll(e));
    P.norm_prec = 1;
    P.inv_h = c->inv_h;
    P.inv_h2 = c->inv_h2;
    memcpy(P.diag_code, c->diag_code, sizeof P.diag_code);
    memcpy(P.inv_code, c->inv_code, sizeof P.inv_code);
    memcpy(P.invA_enc, c->invA_enc, sizeof P.invA_enc);
    P.invS = c->invS;
    P.sdiag2 = c->sdiag2;
    P.ctab = c->ctab[op];
    // prefetch only where the operator's vectors leave L2 (C1 64^3, L2-resident,
    // on a 46-SM share: A 7.6 -> 8.2 us/it with it); the env value applies as given
    P.pf_dist = (c->pf_forced || m > (int64_t(1) << 20)) ? c->pf_dist : 0;
    const CgPlan &pl = op == 0 ? c->plan_A : c->plan_S;
    P.total_blocks = pl.grid * R;          // blocks of every rank
    P.block_base = pl.grid * c->s0;        // global index of this launch's block 0
    while ((int)c->evpool.size() < 2 * c->ncglog) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->evpool.push_back(e);
    }
    CK(cudaEventRecord(c->evpool[2 * li], c->stream));
    if (c->use_tile[op]) {
        const TilePlan &tp = op == 0 ? c->tile_A : c->tile_S;
        P.total_blocks = tp.grid;
        P.block_base = 0;
        CK(launch_cg1t(op, tp, P, c->stream));
    } else if (use_blocked) {
        Slab &S0 = c->slabs[c->s0];
        CK(launch_pcgb(pl, P, S0.blk_vcap, S0.blk_vbuf, c->stream));
        // the solution back into the reference order
        launch_blk_perm(S0.prec, c->n, S0.blk_lineR, S0.blk_lineI, (uint32_t)S0.m_own[1], S0.p[P_SS0], S0.p[x], 0,
                        c->stream);
        ++c->launches;
    } else if (is_m_alg(pl.alg)) {
        CgPlan pm = pl;
        if (pm.alg == CG_BLOCKED) pm.alg = CG_TWO_SUM_MQ;  // k_pcgb does not apply here
        if (pm.alg == CG_TWO_SUM_MX)
            CK(launch_pcgx(c->dim, op, pm, nloc, P, c->stream));
        else
            CK(launch_pcgm(c->dim, op, pm, nloc, P, c->stream));
    } else {
        CK(launch_pcg(c->dim, op, pl, nloc, P, c->stream));
    }
    CK(cudaEventRecord(c->evpool[2 * li + 1], c->stream));
    ++c->launches;
    return li;
}

// After a host sync: account the logged inner solves [from, ncglog) and
// raise the first failure in program order.  Returns the iteration sum per op.
void drain_log(vs_ctx *c, int from, int64_t *its_op) {
    const int n = c->ncglog - from;
    if (n <= 0) return;
    for (int li = from; li < c->ncglog; ++li) {
        const CgOut &o = c->h_cglog[li];
        const int op = c->log_op[li];
        const int64_t m = op == 0 ? c->m_u : c->m_p;
        float ms = 0;
        if (m) CK(cudaEventElapsedTime(&ms, c->evpool[2 * li], c->evpool[2 * li + 1]));
        vs_kstat &st = op == 0 ? c->st_A : c->st_S;
        st.launches += m ? 1 : 0;
        st.iterations += o.iterations;
        st.dof_iters += o.iterations * m;
        st.ms += ms;
        st.kernel = c->use_tile[op] ? 2 : (op == 0 ? c->plan_A.alg : c->plan_S.alg);
        if (st.kernel == CG_BLOCKED && c->slabs[c->s0].blk_state != 1) st.kernel = CG_TWO_SUM_MQ;
        st.reserved = op == 0 ? c->plan_A.unroll : c->plan_S.unroll;  // P1 DOFs per step
        st.tier = op == 0 ? c->plan_A.tier : c->plan_S.tier;
        {
            int64_t esc = 0;
            for (int q = c->s0; q < c->s1; ++q) esc += c->slabs[q].n_escape[op];
            st.escape_ppm = m ? (int32_t)(1000000.0 * (double)esc / (double)m) : 0;
        }
        if (its_op) its_op[li - from] = o.iterations;
        if (m) {
            Status s = cg_status_to_error(o, op);
            if (s.code != VS_OK) throw s;
        }
    }
}

// fetch log slots [from, ncglog) to the host (async, before a sync)
void fetch_log(vs_ctx *c, int from) {
    const int n = c->ncglog - from;
    if (n > 0)
        CK(cudaMemcpyAsync(c->h_cglog + from, c->cglog + from, n * sizeof(CgOut), cudaMemcpyDeviceToHost, c->stream));
}

// Synchronous inner solve: returns the iteration count; throws on errors.
int64_t cg_solve(vs_ctx *c, int op, int rhs, int x0, double eps, int x) {
    c->ncglog = 0;
    cg_async(c, op, rhs, x0, eps, x);
    fetch_log(c, 0);
    c->sync();
    int64_t its = 0;
    drain_log(c, 0, &its);
    c->ncglog = 0;
    return its;
}

void reset_stats(vs_ctx *c) {
    c->st_A = vs_kstat{};
    c->st_S = vs_kstat{};
    c->launches = 0;
}

template <class F>
int guarded(vs_ctx *c, F &&f) {
    try {
        if (c) {
            CK(cudaSetDevice(c->device));
            c->gate = nullptr;  // a call that failed inside a gated batch must not gate this one
        }
        f();
        return VS_OK;
    } catch (const Status &s) {
        g_err = s.msg;
        return s.code;
    } catch (const CudaFail &e) {
        return fail(VS_ECUDA, "CUDA error %s in %s", cudaGetErrorString(e.e), e.what);
    } catch (const std::bad_alloc &) {
        return fail(VS_ECUDA, "host allocation failed");
    }
}

// Layout of every slab from the per-family plane starts (host only; shared
// by the device build and the vs_slab_plan ABI used by the CPU tests).
void plan_slabs(const std::vector<int64_t> (&pstart)[4], int n, int dim, int R, std::vector<Slab> &slabs) {
    auto cnt = [&](int f, int x) { x = (x % n + n) % n; return pstart[f][x + 1] - pstart[f][x]; };
    slabs.assign(R, Slab());
    for (int s = 0; s < R; ++s) {
        Slab &S = slabs[s];
        S.x_lo = (int)((int64_t)s * n / R);
        S.x_hi = (int)((int64_t)(s + 1) * n / R);
        S.P = S.x_hi - S.x_lo;
        S.nx = R == 1 ? n : S.P + 2;
        int64_t off = 0;
        for (int f = 0; f < dim; ++f) {
            S.gstart[f] = pstart[f][S.x_lo];
            S.own[f] = pstart[f][S.x_hi] - pstart[f][S.x_lo];
            S.own_off[f] = off;
            off += S.own[f];
        }
        S.m_own[0] = off;
        for (int f = 0; f < dim; ++f) {
            if (R == 1) continue;
            S.glo_off[f] = off;
            S.glo_cnt[f] = cnt(f, S.x_lo - 1);
            off += S.glo_cnt[f];
            S.ghi_off[f] = off;
            S.ghi_cnt[f] = cnt(f, S.x_hi);
            off += S.ghi_cnt[f];
        }
        S.m_all[0] = off;
        S.gstart[FP] = pstart[FP][S.x_lo];
        S.own[FP] = pstart[FP][S.x_hi] - pstart[FP][S.x_lo];
        S.own_off[FP] = 0;
        S.m_own[1] = S.own[FP];
        off = S.own[FP];
        if (R > 1) {
            S.glo_off[FP] = off;
            S.glo_cnt[FP] = cnt(FP, S.x_lo - 1);
            off += S.glo_cnt[FP];
            S.ghi_off[FP] = off;
            S.ghi_cnt[FP] = cnt(FP, S.x_hi);
            off += S.ghi_cnt[FP];
        }
        S.m_all[1] = off;
        for (int f = 0; f < 4; ++f) {
            if (f < 3 && f >= dim) continue;
            S.first_cnt[f] = cnt(f, S.x_lo);
            S.last_cnt[f] = cnt(f, S.x_hi - 1);
        }
    }
}

// Device arena of one slab: every vector slot, the CG partial buffer, the
// reduction slots and the barrier words in ONE allocation, laid out by a
// formula every rank can evaluate for every slab -- so a single CUDA IPC
// handle per rank maps a neighbour's whole slab (vs_ipc_attach).
struct ArenaLayout {
    size_t u[NU], p[NP], part, scal, bar, bytes;
};
ArenaLayout arena_layout(const Slab &S, int64_t tb_max, int R) {
    ArenaLayout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    for (int k = 0; k < NU; ++k) L.u[k] = take(std::max<int64_t>(1, S.m_all[0]) * sizeof(double));
    for (int k = 0; k < NP; ++k) L.p[k] = take(std::max<int64_t>(1, S.m_all[1]) * sizeof(double));
    L.part = take((size_t)4 * 8 * tb_max * sizeof(double));
    L.scal = take((size_t)Q_COUNT * R * sizeof(double));
    L.bar = take(4 * sizeof(unsigned));
    L.bytes = off;
    return L;
}

void bind_arena(Slab &S, char *base, const ArenaLayout &L) {
    for (int k = 0; k < NU; ++k) S.u[k] = (double *)(base + L.u[k]);
    for (int k = 0; k < NP; ++k) S.p[k] = (double *)(base + L.p[k]);
}

void plan_solvers(vs_ctx *C, int64_t mu_max, int64_t mp_max, int sms);

// Build the decomposition from the global geometry: R slabs in total, of
// which this process holds [s0, s1) (all of them, or `rank`'s one).
void build_slabs(vs_ctx *C, int R, int rank, int nranks) {
    const int n = C->n, dim = C->dim;
    const int64_t wpp = (int64_t)(dim == 3 ? n : 1) * C->nw;  // meta words per x-plane
    // plane starts per family, from the first word of each plane
    for (int f = 0; f < 4; ++f) {
        if (f < 3 && f >= dim) continue;
        const uint2 *gm = f == FP ? C->pmeta : C->vmeta[f];
        std::vector<uint2> first(n);
        for (int x = 0; x < n; ++x)
            CK(cudaMemcpyAsync(&first[x], gm + (int64_t)x * wpp, sizeof(uint2), cudaMemcpyDeviceToHost, C->stream));
        C->sync();
        C->pstart[f].resize(n + 1);
        for (int x = 0; x < n; ++x) C->pstart[f][x] = first[x].y;
        C->pstart[f][n] = f == FP ? C->m_p : C->voff[f] + C->vcount[f];
    }
    C->R = R;
    C->rank = rank;
    C->nranks = nranks;
    C->s0 = nranks > 1 ? rank : 0;
    C->s1 = nranks > 1 ? rank + 1 : R;
    const int nloc = C->s1 - C->s0;
    plan_slabs(C->pstart, n, dim, R, C->slabs);
    // plans from the largest slab of the whole decomposition, so every rank
    // launches the same grid (the barrier counts all ranks' blocks)
    int64_t mu_max = 0, mp_max = 0;
    for (auto &S : C->slabs) {
        mu_max = std::max(mu_max, S.m_own[0]);
        mp_max = std::max(mp_max, S.m_own[1]);
    }
    C->mu_max = mu_max;
    C->mp_max = mp_max;
    plan_solvers(C, mu_max, mp_max, 0);
    // plane-sweep TMA tiles (k_cg1t): VOXSCHUR_TILED=1 turns them on
    const char *et = getenv("VOXSCHUR_TILED");
    if (et && atoi(et) == 1 && dim == 3 && R == 1 && !(C->nw & 1)) {
        const uint2 *mA[3] = {C->vmeta[0], C->vmeta[1], C->vmeta[2]};
        const int64_t fA[3] = {C->vcount[0], C->vcount[1], C->vcount[2]};
        C->tile_A = tile_plan(0, n, C->nw, 3, mA, fA, C->device, C->stream);
        const uint2 *mS[1] = {C->pmeta};
        const int64_t fS[1] = {C->m_p};
        C->tile_S = tile_plan(1, n, C->nw, 1, mS, fS, C->device, C->stream);
        C->use_tile[0] = C->tile_A.ok;
        C->use_tile[1] = C->tile_S.ok;
        CK(cudaGetLastError());
    }
    C->tb_max = (int64_t)std::max(C->plan_A.grid, C->plan_S.grid) * R;
    for (int s = C->s0; s < C->s1; ++s) {
        Slab &S = C->slabs[s];
        // geometry
        if (R == 1) {
            for (int a = 0; a < 3; ++a) S.meta[a] = C->vmeta[a];
            S.meta[FP] = C->pmeta;
            S.vrec = C->vrec;
            S.prec = C->prec;
        } else {
            for (int f = 0; f < 4; ++f) {
                if (f < 3 && f >= dim) continue;
                const uint2 *gm = f == FP ? C->pmeta : C->vmeta[f];
                S.meta[f] = C->alloc<uint2>(wpp * (S.P + 2));
                const int64_t xlo_m = ((S.x_lo - 1) % n + n) % n, xhi_m = S.x_hi % n;
                launch_slab_meta(gm, S.meta[f], wpp, S.x_lo, S.P, n, S.glo_off[f] - C->pstart[f][xlo_m],
                                 S.own_off[f] - C->pstart[f][S.x_lo], S.ghi_off[f] - C->pstart[f][xhi_m],
                                 C->stream);
            }
            S.vrec = C->alloc<uint64_t>(S.m_own[0]);
            for (int f = 0; f < dim; ++f)
                launch_slab_rec(C->vrec + S.gstart[f], S.vrec + S.own_off[f], S.own[f], S.x_lo, C->stream);
            S.prec = C->alloc<uint64_t>(S.m_own[1]);
            launch_slab_rec(C->prec + S.gstart[FP], S.prec, S.own[FP], S.x_lo, C->stream);
            CK(cudaGetLastError());
        }
        S.geo.dim = dim;
        S.geo.n = n;
        S.geo.nw = C->nw;
        S.geo.nlines = (dim == 3 ? n : 1) * S.nx;
        S.geo.nx = S.nx;
        S.geo.fbits = nullptr;
        for (int a = 0; a < 3; ++a) S.geo.vmeta[a] = S.meta[a];
        S.geo.pmeta = S.meta[FP];
        const ArenaLayout L = arena_layout(S, C->tb_max, R);
        char *base = nranks > 1 ? C->alloc_ipc<char>(L.bytes) : C->alloc<char>(L.bytes);
        bind_arena(S, base, L);
        if (s == C->s0) {
            C->arena = base;
            C->part = (double *)(base + L.part);
            C->scal = (double *)(base + L.scal);
            C->bar = (unsigned *)(base + L.bar);  // rank 0's counter replaces it on attach
            C->bar_base = C->bar + 1;
            CK(cudaMemsetAsync(C->bar, 0, 4 * sizeof(unsigned), C->stream));
        }
        // words 2, 3 of every slab's barrier block: the rank-local arrival counter and release
        // word of the hierarchical barrier (vs_cg_common.cuh)
        CK(cudaMemsetAsync(base + L.bar + 2 * sizeof(unsigned), 0, 2 * sizeof(unsigned), C->stream));
        S.lbar = (unsigned *)(base + L.bar) + 2;

    }
    C->npart = 1;
    C->part_peer[0] = C->part;
    // ranks on different GPUs arrive through their leaders; ranks emulated on one GPU keep the
    // flat barrier unless asked (there the second level only adds a local round trip: C2 on 4
    // emulated ranks 43.4 -> 46.3 us/it) -- the tests ask, so that the protocol runs
    C->hier_barrier = nranks > 1;
    if (const char *hb = getenv("VOXSCHUR_HIER_BARRIER")) C->hier_barrier = atoi(hb) != 0;
    // VOXSCHUR_EMULATE_RANKS=1: slabs of one process use the multi-process
    // data flow (a partial buffer per slab arena, every block broadcasting
    // its sums to all of them), so one GPU exercises that protocol
    const char *em = getenv("VOXSCHUR_EMULATE_RANKS");
    if (em && atoi(em) && nranks == 1 && R > 1) {
        for (int s = 0; s < R; ++s) {
            const ArenaLayout L = arena_layout(C->slabs[s], C->tb_max, R);
            C->part_peer[s] = (double *)((char *)C->slabs[s].u[0] - L.u[0] + L.part);
        }
        C->npart = R;
    }
    C->scal_peer[C->rank] = C->scal;
    C->d_groups = C->alloc<CgGroup>(nloc * GROUP_RING);
    CK(cudaMallocHost(&C->h_groups, nloc * GROUP_RING * sizeof(CgGroup)));
    CK(cudaFreeHost(C->h_scal));
    CK(cudaMallocHost(&C->h_scal, std::max(8, Q_COUNT * R) * sizeof(double)));
    C->cglog_cap = 16;
    C->cglog = C->alloc<CgOut>(C->cglog_cap);
    CK(cudaMallocHost(&C->h_cglog, C->cglog_cap * sizeof(CgOut)));
    C->ost = C->alloc<OuterState>(1);
    CK(cudaMallocHost(&C->h_ost, sizeof(OuterState)));
}

// Fused-PCG plans of both inner operators on `sms` SMs (0: the whole device).
// One-reduction CG (k_cg1) on a single slab where the grid sums dominate (a
// few DOFs per thread; B200 C1 64^3: A 12.4 -> 9.7, S_hat 9.6 -> 8.5 us/it);
// on large solves its 18 gathers per DOF cost more than the saved sum (C2
// S_hat 57.6 -> 63.3), and the slab decomposition keeps the two-reduction
// loop (its halo exchange is built for it).  VOXSCHUR_CG=1 / =2 forces the
// one- / two-reduction loop.  TIER 3 (neighbour ranks precomputed in HBM)
// instead of bitmask lookups when the ranks do not fit the smem DOF cache:
// VOXSCHUR_NBR=1.
void plan_solvers(vs_ctx *C, int64_t mu_max, int64_t mp_max, int sms) {
    const int R = C->R, dim = C->dim;
    const int nloc = C->s1 - C->s0;
    const char *ea = getenv("VOXSCHUR_CG");
    const int force = ea ? atoi(ea) : 0;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, C->device));
    if (sms > 0 && sms < nsm) nsm = sms;
    // Small operators (at most 4 DOFs per thread): k_cg1, one grid sum per
    // iteration.  Everything larger, and every slab-decomposed run: k_pcgx (vs_cgx.cu:
    // two grid sums, M-scaled, 8-B descriptors, alpha from the z sums, d and x brought
    // up to date every 4th iteration from a ring of z buffers: 72 B per DOF-iteration).
    // B200, us per CG iteration, against the previous default k_pcgm qrec (98 B):
    // C4 512^3 S_hat 463 -> 403, A 1149 -> 822; C2 256^3 S_hat 47.3 -> 42.6, A 86.8 -> 79.0
    // (profiles/r02x_*).  VOXSCHUR_CG forces a kernel: 1 k_cg1, 2 k_pcg (reference
    // operation order), 3 k_pcg<QR>, 4 k_pcgm qrec, 5 k_pcgm rc (q recomputed in both
    // passes, 80 B), 6 k_pcgb, 7 k_pcgx.
    auto pick = [&](int64_t m, int op) {
        if (force == 6) return op == 1 ? (int)CG_BLOCKED : (int)CG_TWO_SUM_MQ;
        if (force == 7) return (int)CG_TWO_SUM_MX;
        if (force == 4) return (int)CG_TWO_SUM_MQ;
        if (force == 5) return (int)CG_TWO_SUM_MRC;
        if (force == 3) return (int)CG_TWO_SUM_QREC;
        if (force == 2) return (int)CG_TWO_SUM;
        if (R == 1 && (force == 1 || (force == 0 && m <= (int64_t)4 * nsm * CG_THREADS)))
            return (int)CG_ONE_SUM;
        return (int)CG_TWO_SUM_MX;
    };
    const char *en = getenv("VOXSCHUR_NBR");
    // VOXSCHUR_NBR=1: TIER 3 (32-bit ranks), =2: TIER 4 (packed deltas)
    const int nbr = en ? (atoi(en) == 1 && R == 1 ? 3 : atoi(en) == 2 ? 4 : 0) : 0;
    // Two-reduction solves on one slab read packed neighbour deltas (TIER 4)
    // instead of the bitmask lookups when the ranks do not fit the smem DOF
    // cache (B200, with the recurrence: S_hat C2 58.2 -> 55.1, C4 512^3 794 ->
    // 755 us/it; A-solves gain only together with the carried delta words
    // and the L2 prefetch: C2 110.9 -> 102.7, C4 1448 -> 1371).
    // VOXSCHUR_NBR=0 turns it off.  (Ignored by k_cg1.)
    const int nbr_A = en ? nbr : 4;
    const int nbr_S = nbr_A;
    auto plan = [&](int op, int64_t m, int nbr_tier) {
        const int alg = pick(m, op);
        if (is_m_alg(alg)) {
            // an operator whose neighbour ranks fit the shared-memory DOF cache (TIER 2:
            // no descriptor stream, no rank arithmetic) keeps k_pcg<QR> -- e.g. the C1
            // A-solve on a 46-SM share: 14.9 vs 17.9 us/it with k_pcgm (B200)
            if (force == 0) {
                const CgPlan q = pcg_plan(dim, op, m, nloc, C->device, CG_TWO_SUM_QREC, 0, nsm);
                if (q.tier == 2) return q;
            }
            if (alg == CG_TWO_SUM_MX) return pcgx_plan(dim, op, m, nloc, C->device, nsm);
            return pcgm_plan(dim, op, m, nloc, C->device, alg, nsm);
        }
        return pcg_plan(dim, op, m, nloc, C->device, alg, nbr_tier, nsm);
    };
    C->plan_A = plan(0, mu_max, nbr_A);
    C->plan_S = plan(1, mp_max, nbr_S);
    C->sms = nsm;
}

}  // namespace

// =================================================================== ABI

extern "C" {

const char *vs_last_error(void) { return g_err.c_str(); }

const char *vs_version(void) { return "voxschur 0.2 sm_100a (fp64, fused persistent PCG, x-slab groups)"; }

int vs_device_count(int *count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) c = 0;
    else if (e != cudaSuccess) return fail(VS_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    *count = c;
    return VS_OK;
}

int vs_components(const uint8_t *fluid, int dim, int n, int32_t *labels, int64_t *n_components) {
    if ((dim != 2 && dim != 3) || n < 1) return fail(VS_EVALUE, "grid dimension must be 2 or 3, got %d", dim);
    try {
        *n_components = label_components(fluid, dim, n, labels);
    } catch (const std::bad_alloc &) {
        return fail(VS_ECUDA, "host allocation failed");
    }
    return VS_OK;
}

int vs_components_device(const uint8_t *fluid, int dim, int n, int device, int32_t *labels, int64_t *n_components) {
    if ((dim != 2 && dim != 3) || n < 1) return fail(VS_EVALUE, "grid dimension must be 2 or 3, got %d", dim);
    const int64_t N = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    if (N >= ((int64_t)1 << 31)) return fail(VS_EVALUE, "grid of %lld cells exceeds the int32 labelling", (long long)N);
    try {
        CK(cudaSetDevice(device));
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        uint8_t *d_f = nullptr;
        int *d_lab = nullptr;
        void *work = nullptr;
        const size_t wb = cc_work_bytes(N);
        CK(cudaMallocAsync(&d_f, N, s));
        CK(cudaMallocAsync(&work, wb, s));
        if (labels) CK(cudaMallocAsync(&d_lab, N * sizeof(int), s));
        CK(cudaMemcpyAsync(d_f, fluid, N, cudaMemcpyHostToDevice, s));
        *n_components = cc_label_device(d_f, dim, n, d_lab, work, wb, s);
        if (labels) CK(cudaMemcpyAsync(labels, d_lab, N * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaFreeAsync(d_f, s));
        CK(cudaFreeAsync(work, s));
        if (d_lab) CK(cudaFreeAsync(d_lab, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamDestroy(s));
        CK(cudaGetLastError());
    } catch (const CudaFail &e) {
        return fail(VS_ECUDA, "CUDA error %s in %s", cudaGetErrorString(e.e), e.what);
    }
    return VS_OK;
}

int vs_stamp_balls(uint8_t *fluid, int dim, int n, const double *centers, const double *radii, int64_t count,
                   int64_t target_fluid, int prism_axis, int64_t *used, int64_t *n_fluid) {
    if ((dim != 2 && dim != 3) || n < 2) return fail(VS_EVALUE, "bad grid for vs_stamp_balls");
    const int64_t N = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    // *n_fluid >= 0 on entry: the caller's running fluid count (a batched
    // caller passes back the previous call's result; recounting n^3 cells
    // per batch dominated 1024^3 generation)
    int64_t nf = *n_fluid;
    if (nf < 0) {
        nf = 0;
        for (int64_t i = 0; i < N; ++i) nf += fluid[i] ? 1 : 0;
    }
    int64_t k = 0;
    const int64_t st[3] = {dim == 3 ? (int64_t)n * n : (int64_t)n, dim == 3 ? (int64_t)n : 1, 1};
    constexpr int WMAX = 4096;  // window positions per axis of the hoisted path
    std::vector<int64_t> woff_v(3 * WMAX);
    std::vector<double> wd2_v(3 * WMAX);
    int64_t *woff[3] = {woff_v.data(), woff_v.data() + WMAX, woff_v.data() + 2 * WMAX};
    double *wd2[3] = {wd2_v.data(), wd2_v.data() + WMAX, wd2_v.data() + 2 * WMAX};
    for (; k < count && nf > target_fluid; ++k) {
        const double r = radii[k], r2 = r * r;
        const double *c = centers + k * dim;
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) {
            if (a == prism_axis) { lo[a] = 0; hi[a] = n - 1; continue; }
            lo[a] = (int)std::floor(c[a] - r) - 1;
            hi[a] = (int)std::ceil(c[a] + r) + 1;
            if (hi[a] - lo[a] + 1 > n) { lo[a] = 0; hi[a] = n - 1; }
        }
        if (dim == 2) { lo[2] = hi[2] = 0; }
        // per axis: wrapped index offset and squared minimum-image distance
        // of every window position (same operations as per cell, hoisted)
        int len[3] = {1, 1, 1};
        bool small = true;
        for (int a = 0; a < 3; ++a) {
            len[a] = hi[a] - lo[a] + 1;
            if (len[a] > WMAX) small = false;
        }
        if (small) {
            for (int a = 0; a < dim; ++a)
                for (int t = 0; t < len[a]; ++t) {
                    const int w = (((lo[a] + t) % n) + n) % n;
                    woff[a][t] = (int64_t)w * st[dim == 3 ? a : (a == 0 ? 0 : 2)];
                    double dd = std::fabs((double)w - c[a]);
                    dd = std::min(dd, (double)n - dd);
                    wd2[a][t] = a == prism_axis ? 0.0 : dd * dd;
                }
            if (dim == 2) { woff[2][0] = 0; wd2[2][0] = 0.0; }
            for (int ti = 0; ti < len[0]; ++ti)
                for (int tj = 0; tj < len[1]; ++tj) {
                    // d2 accumulates axis by axis from 0.0, as below (a prism
                    // axis contributes nothing: adding 0.0 is exact)
                    const double d01 = (0.0 + wd2[0][ti]) + wd2[1][tj];
                    const int64_t o01 = woff[0][ti] + woff[1][tj];
                    for (int tl = 0; tl < len[2]; ++tl) {
                        const double d2 = dim == 3 ? d01 + wd2[2][tl] : d01;
                        const int64_t off = o01 + woff[2][tl];
                        if (d2 <= r2 && fluid[off]) { fluid[off] = 0; --nf; }
                    }
                }
        } else {
            for (int i = lo[0]; i <= hi[0]; ++i)
                for (int j = lo[1]; j <= hi[1]; ++j)
                    for (int l = lo[2]; l <= hi[2]; ++l) {
                        const int idx[3] = {i, j, l};
                        double d2 = 0.0;
                        int64_t off = 0;
                        for (int a = 0; a < dim; ++a) {
                            const int w = ((idx[a] % n) + n) % n;  // periodic wrap of the window
                            off += w * st[dim == 3 ? a : (a == 0 ? 0 : 2)];
                            if (a == prism_axis) continue;
                            double dd = std::fabs((double)w - c[a]);
                            dd = std::min(dd, (double)n - dd);  // minimum image
                            d2 += dd * dd;
                        }
                        if (d2 <= r2 && fluid[off]) { fluid[off] = 0; --nf; }
                    }
        }
        if (nf <= target_fluid) { ++k; break; }
    }
    *used = k;
    *n_fluid = nf;
    return VS_OK;
}

// Host-only slab plan of a mask (no device): per slab 42 int64 =
// x_lo, x_hi, then per family f in (0,1,2,pressure): own, own_off, glo_off,
// glo_cnt, ghi_off, ghi_cnt, first_cnt, last_cnt, gstart; then m_own[2], m_all[2].
int vs_slab_plan(const uint8_t *fluid, int dim, int n, int slabs, int64_t *out) {
    if ((dim != 2 && dim != 3) || n < 2) return fail(VS_EVALUE, "bad grid for vs_slab_plan");
    if (slabs < 1 || slabs > VS_MAX_SLABS || slabs > n)
        return fail(VS_EVALUE, "slab count %d out of range [1, min(%d, n)]", slabs, VS_MAX_SLABS);
    const int64_t plane = dim == 3 ? (int64_t)n * n : n;
    const int64_t st[3] = {plane, dim == 3 ? (int64_t)n : 1, 1};
    std::vector<int64_t> ps[4];
    std::vector<int64_t> c(n);
    int64_t off = 0;
    for (int f = 0; f < 4; ++f) {
        if (f < 3 && f >= dim) continue;
        std::fill(c.begin(), c.end(), 0);
        for (int x = 0; x < n; ++x)
            for (int64_t q = 0; q < plane; ++q) {
                const int64_t i = (int64_t)x * plane + q;
                if (!fluid[i]) continue;
                if (f == FP) { ++c[x]; continue; }
                // face (f, I): fluid[I] && fluid[I - e_f] (operators.py:232)
                const int64_t coord = (i / st[f]) % n;
                const int64_t j = coord == 0 ? i + (int64_t)(n - 1) * st[f] : i - st[f];
                if (fluid[j]) ++c[x];
            }
        ps[f].assign(n + 1, 0);
        int64_t acc = f == FP ? 0 : off;
        for (int x = 0; x < n; ++x) { ps[f][x] = acc; acc += c[x]; }
        ps[f][n] = acc;
        if (f != FP) off = acc;
    }
    std::vector<Slab> sl;
    plan_slabs(ps, n, dim, slabs, sl);
    for (int s = 0; s < slabs; ++s) {
        const Slab &S = sl[s];
        int64_t *o = out + (int64_t)s * 42;
        o[0] = S.x_lo;
        o[1] = S.x_hi;
        for (int f = 0; f < 4; ++f) {
            int64_t *q = o + 2 + 9 * f;
            q[0] = S.own[f]; q[1] = S.own_off[f]; q[2] = S.glo_off[f]; q[3] = S.glo_cnt[f];
            q[4] = S.ghi_off[f]; q[5] = S.ghi_cnt[f]; q[6] = S.first_cnt[f]; q[7] = S.last_cnt[f];
            q[8] = S.gstart[f];
        }
        o[38] = S.m_own[0]; o[39] = S.m_own[1]; o[40] = S.m_all[0]; o[41] = S.m_all[1];
    }
    return VS_OK;
}

static int create_common(const uint8_t *fluid, int dim, int n, int flow_dir, int check_connectivity,
                         int require_walls, int device, double inv_h, double inv_h2, int slabs, int rank,
                         int nranks, vs_ctx **out) {
    *out = nullptr;
    if (dim != 2 && dim != 3) return fail(VS_EVALUE, "grid dimension must be 2 or 3, got %d", dim);
    if (n < 2) return fail(VS_EVALUE, "grid extent must be at least 2, got %d", n);
    if (n > 2047) return fail(VS_EVALUE, "grid extent %d exceeds the record layout limit 2047", n);
    // cell indices, component labels and the meta prefix counts are 32-bit
    // (3D: n <= 1290); a larger grid must be decomposed before it gets here
    if ((dim == 3 ? (int64_t)n * n * n : (int64_t)n * n) >= ((int64_t)1 << 31))
        return fail(VS_EVALUE, "grid of %lld cells exceeds the 32-bit cell index (n <= 1290 in 3D)",
                    (long long)(dim == 3 ? (int64_t)n * n * n : (int64_t)n * n));
    if (flow_dir < 0 || flow_dir >= dim) return fail(VS_EVALUE, "flow axis %d out of range for dim %d", flow_dir, dim);
    if (slabs < 1 || slabs > VS_MAX_SLABS || slabs > n)
        return fail(VS_EVALUE, "slab count %d out of range [1, min(%d, n)]", slabs, VS_MAX_SLABS);
    const int64_t ncells = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    // operators.py:220-230 -- host-side validation and connectivity
    int64_t nfluid = 0;
    for (int64_t i = 0; i < ncells; ++i) nfluid += fluid[i] ? 1 : 0;
    if (nfluid == 0) return fail(VS_EVALUE, "empty fluid domain");
    if (require_walls && nfluid == ncells) return fail(VS_EVALUE, "velocity operator singular: no no-slip boundary");
    // small grids: host union-find before any device work; large grids
    // (>= CC_DEVICE_CELLS): the same labelling on the GPU after the mask
    // upload (vs_cc.cu; 1024^3 on the host took seconds per pass)
    const bool cc_on_device = check_connectivity && ncells >= CC_DEVICE_CELLS;
    if (check_connectivity && !cc_on_device) {
        int64_t nc = 0;
        try {
            nc = label_components(fluid, dim, n, nullptr);
        } catch (const std::bad_alloc &) {
            return fail(VS_ECUDA, "host allocation failed");
        }
        if (nc > 1)
            return fail(VS_EVALUE,
                        "fluid domain is disconnected (%lld components); run enforce_connectivity first",
                        (long long)nc);
    }
    std::unique_ptr<vs_ctx> c(new vs_ctx());
    c->device = device;
    c->dim = dim;
    c->n = n;
    c->nw = (n + 31) / 32;
    c->nlines = dim == 3 ? n * n : n;
    c->nwords = (int64_t)c->nlines * c->nw;
    c->ncells = ncells;
    c->flow_dir = flow_dir;
    c->inv_h = inv_h;
    c->inv_h2 = inv_h2;
    c->diag_scale = ((double)n / 1.0) * ((double)n / 1.0);  // (n/1.0)**2, exact
    vs_ctx *C = c.get();
    int rc = guarded(C, [&] {
        CK(cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking));
        keep_pool(device);
        for (cudaEvent_t *e : {&C->ev0, &C->ev1, &C->evs0, &C->evs1}) CK(cudaEventCreate(e));
        CK(cudaMallocHost(&C->h_scal, 8 * sizeof(double)));
        CK(cudaMallocHost(&C->h_cg, sizeof(CgOut)));
        const int64_t nw = C->nwords;
        // ---- K1: mask -> bits -> face bits -> ranks -> records
        uint8_t *d_fluid = C->alloc<uint8_t>(ncells);
        CK(cudaMemcpyAsync(d_fluid, fluid, ncells, cudaMemcpyHostToDevice, C->stream));
        if (cc_on_device) {  // operators.py:224-230
            const size_t wb = cc_work_bytes(ncells);
            void *work = nullptr;
            CK(cudaMallocAsync(&work, wb, C->stream));
            const int64_t nc = cc_label_device(d_fluid, dim, n, nullptr, work, wb, C->stream);
            CK(cudaFreeAsync(work, C->stream));
            CK(cudaGetLastError());
            if (nc > 1) {
                char buf[160];
                snprintf(buf, sizeof buf,
                         "fluid domain is disconnected (%lld components); run enforce_connectivity first",
                         (long long)nc);
                throw Status{VS_EVALUE, buf};
            }
        }
        C->fbits = C->alloc<uint32_t>(nw);
        Geo g = C->geo();
        launch_pack_fluid(d_fluid, g, nw, C->fbits, C->stream);
        g = C->geo();
        uint32_t *cnt = C->alloc<uint32_t>(nw), *base = C->alloc<uint32_t>(nw);
        const size_t tb = scan_temp_bytes(nw);
        void *temp = C->alloc<uint8_t>(tb);
        std::vector<uint32_t *> fb(dim);
        for (int a = 0; a < dim; ++a) {
            fb[a] = C->alloc<uint32_t>(nw);
            launch_face_bits(g, a, nw, fb[a], C->stream);
        }
        uint32_t off = 0;
        for (int a = 0; a < dim; ++a) {
            C->vmeta[a] = C->alloc<uint2>(nw);
            CK(build_meta(fb[a], nw, off, C->vmeta[a], cnt, base, temp, tb, C->stream));
            uint2 lastm;
            CK(cudaMemcpyAsync(&lastm, C->vmeta[a] + nw - 1, sizeof(uint2), cudaMemcpyDeviceToHost, C->stream));
            C->sync();
            C->vcount[a] = (int64_t)lastm.y + __builtin_popcount(lastm.x) - off;
            C->voff[a] = off;
            if ((uint64_t)off + C->vcount[a] > 0x7FFFFFF0ull) throw Status{VS_EVALUE, "too many velocity DOFs"};
            off += (uint32_t)C->vcount[a];
        }
        C->m_u = off;
        C->pmeta = C->alloc<uint2>(nw);
        CK(build_meta(C->fbits, nw, 0, C->pmeta, cnt, base, temp, tb, C->stream));
        {
            uint2 lastm;
            CK(cudaMemcpyAsync(&lastm, C->pmeta + nw - 1, sizeof(uint2), cudaMemcpyDeviceToHost, C->stream));
            C->sync();
            C->m_p = (int64_t)lastm.y + __builtin_popcount(lastm.x);
        }
        if (require_walls && C->m_u == 0) throw Status{VS_EVALUE, "no velocity unknowns: every face touches solid"};
        g = C->geo();
        C->vrec = C->alloc<uint64_t>(C->m_u);
        C->prec = C->alloc<uint64_t>(C->m_p);
        for (int a = 0; a < dim; ++a) launch_vel_records(g, a, nw, C->vrec, C->stream);
        launch_p_records(g, nw, C->prec, C->stream);
        CK(cudaGetLastError());
        // ---- tables: every FP constant is computed exactly as the reference does
        for (int code = 0; code < 16; ++code) {
            C->diag_code[code] = (double)code * C->diag_scale;          // operators.py:285
            C->inv_code[code] = code ? 1.0 / C->diag_code[code] : 0.0;  // krylov.py:213
        }
        const int cbase = 2 * dim - 1;
        for (int e = 0; e < 8; ++e)
            C->invA_enc[e] = e ? 1.0 / ((double)(e + cbase) * C->diag_scale) : 0.0;  // schur.py:235
        // diag(S_hat) by the packed face codes, summed in reference order
        const int nkey = 1 << 18;
        std::vector<double> invS(nkey, 0.0);
        std::vector<double2> sdiag2(nkey, double2{0.0, 0.0});
        for (int key = 0; key < nkey; ++key) {
            double acc = 0.0;  // operators.py:202-206
            bool ok = true;
            for (int a = 0; a < dim; ++a) {
                const int ci = (key >> (3 * a)) & 7, co = (key >> (9 + 3 * a)) & 7;
                if (ci > 2 * dim - 1 || co > 2 * dim - 1) ok = false;
                const double wi = ci ? C->invA_enc[ci] : 0.0, wo = co ? C->invA_enc[co] : 0.0;
                acc = acc + (wi + wo);
            }
            const double dS = acc * C->inv_h2;
            invS[key] = (ok && dS > 0) ? 1.0 / dS : 0.0;  // krylov.py:213
            sdiag2[key] = double2{invS[key], (ok && dS > 0) ? dS : 0.0};
        }
        C->sdiag2 = C->alloc<double2>(nkey);
        CK(cudaMemcpyAsync(C->sdiag2, sdiag2.data(), nkey * sizeof(double2), cudaMemcpyHostToDevice, C->stream));
        C->invS = C->alloc<double>(nkey);
        CK(cudaMemcpyAsync(C->invS, invS.data(), nkey * sizeof(double), cudaMemcpyHostToDevice, C->stream));
        C->d_diag_code = C->alloc<double>(16);
        C->d_invA_enc = C->alloc<double>(8);
        CK(cudaMemcpyAsync(C->d_diag_code, C->diag_code, 16 * sizeof(double), cudaMemcpyHostToDevice, C->stream));
        CK(cudaMemcpyAsync(C->d_invA_enc, C->invA_enc, 8 * sizeof(double), cudaMemcpyHostToDevice, C->stream));
        int *flag = C->alloc<int>(1);
        CK(cudaMemsetAsync(flag, 0, sizeof(int), C->stream));
        launch_zero_sdiag(C->prec, C->m_p, flag, C->stream);
        int hflag = 0;
        CK(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, C->stream));
        C->sync();
        C->sdiag_ok = hflag == 0;
        // ---- decomposition into x-slabs (1 = whole domain), work vectors, plans
        build_slabs(C, slabs, rank, nranks);
        if (nranks > 1) {
            // cross-GPU barriers give up after VOXSCHUR_XBAR_TIMEOUT_S seconds (default 60)
            C->xflag_dev = C->alloc<int>(1);
            CK(cudaMemsetAsync(C->xflag_dev, 0, sizeof(int), C->stream));
            const char *et = getenv("VOXSCHUR_XBAR_TIMEOUT_S");
            const double secs = et && atof(et) > 0 ? atof(et) : 60.0;
            C->xtimeout_ns = (unsigned long long)(secs * 1e9);
        }
        if (const char *pf = getenv("VOXSCHUR_PREFETCH")) {
            C->pf_dist = (uint32_t)atoi(pf);
            C->pf_forced = true;
        }
        if (getenv("VOXSCHUR_PHASE_TIMING")) {
            C->phase_ns = C->alloc<unsigned long long>(12);
            CK(cudaMemsetAsync(C->phase_ns, 0, 12 * sizeof(unsigned long long), C->stream));
        }
        C->red_part = C->alloc<double>(RED_MAX_BLOCKS);
        C->cgout = C->alloc<CgOut>(1);
        C->sync();
    });
    if (rc != VS_OK) return rc;
    *out = c.release();
    return VS_OK;
}

int vs_ctx_create2(const uint8_t *fluid, int dim, int n, int flow_dir, int check_connectivity, int require_walls,
                   int device, double inv_h, double inv_h2, int slabs, vs_ctx **out) {
    return create_common(fluid, dim, n, flow_dir, check_connectivity, require_walls, device, inv_h, inv_h2, slabs, 0,
                         1, out);
}

int vs_ctx_create(const uint8_t *fluid, int dim, int n, int flow_dir, int check_connectivity, int require_walls,
                  int device, double inv_h, double inv_h2, vs_ctx **out) {
    return create_common(fluid, dim, n, flow_dir, check_connectivity, require_walls, device, inv_h, inv_h2, 1, 0, 1,
                         out);
}

int vs_ctx_create_rank(const uint8_t *fluid, int dim, int n, int flow_dir, int check_connectivity,
                       int require_walls, int device, double inv_h, double inv_h2, int rank, int nranks,
                       vs_ctx **out) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(VS_EVALUE, "rank %d out of range for %d ranks", rank, nranks);
    return create_common(fluid, dim, n, flow_dir, check_connectivity, require_walls, device, inv_h, inv_h2, nranks,
                         rank, nranks, out);
}

// CUDA IPC: the local slab's arena handle (64 bytes) for the other ranks
int vs_ipc_handle(vs_ctx *c, void *handle64) {
    return guarded(c, [&] {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, c->arena));
        memcpy(handle64, &h, sizeof h);
    });
}

// CUDA IPC: map every other rank's slab arena (handles: nranks x 64 bytes in
// rank order), bind the remote slabs' vectors, CG partial buffers and
// reduction slots to peer pointers, and use rank 0's barrier counter.
int vs_ipc_attach(vs_ctx *c, const void *handles) {
    return guarded(c, [&] {
        if (!c->mp()) throw Status{VS_EVALUE, "vs_ipc_attach needs a context from vs_ctx_create_rank with nranks > 1"};
        const int R = c->R;
        for (int r = 0; r < R; ++r) {
            Slab &S = c->slabs[r];
            const ArenaLayout L = arena_layout(S, c->tb_max, R);
            char *base = nullptr;
            if (r == c->rank) {
                base = c->arena;
            } else {
                cudaIpcMemHandle_t h;
                memcpy(&h, (const char *)handles + (size_t)r * sizeof h, sizeof h);
                void *p = nullptr;
                CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
                c->peer_arena[r] = p;
                base = (char *)p;
                bind_arena(S, base, L);
            }
            c->part_peer[r] = (double *)(base + L.part);
            c->scal_peer[r] = (double *)(base + L.scal);
            if (r == 0) c->bar = (unsigned *)(base + L.bar);  // the shared counter lives on rank 0
        }
        c->npart = R;
        c->sync();
    });
}

void vs_ctx_destroy(vs_ctx *ctx) { delete ctx; }

int vs_counts(vs_ctx *c, int64_t *m_u, int64_t *m_p, int64_t axis_counts[3]) {
    *m_u = c->m_u;
    *m_p = c->m_p;
    for (int a = 0; a < 3; ++a) axis_counts[a] = c->vcount[a];
    return VS_OK;
}

int vs_export_geometry(vs_ctx *c, uint8_t *fm0, uint8_t *fm1, uint8_t *fm2, uint8_t *pm, uint8_t *code) {
    return guarded(c, [&] {
        uint8_t *tmp = nullptr;
        CK(cudaMalloc(&tmp, std::max<int64_t>(c->ncells, c->m_u) + 1));
        const Geo g = c->geo();
        uint8_t *outs[4] = {fm0, fm1, fm2, pm};
        for (int k = 0; k < 4; ++k) {
            if (!outs[k] || (k < 3 && k >= c->dim)) continue;
            launch_bits_to_u8(k < 3 ? c->vmeta[k] : c->pmeta, nullptr, g, c->ncells, tmp, c->stream);
            CK(cudaMemcpyAsync(outs[k], tmp, c->ncells, cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        if (code && c->m_u) {
            launch_vcodes(c->vrec, c->m_u, tmp, c->stream);
            CK(cudaMemcpyAsync(code, tmp, c->m_u, cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        cudaFree(tmp);
    });
}

// unit applies run on every slab (bitwise independent of the decomposition)
static int apply_common(vs_ctx *c, int which, const double *in, double *out) {
    return guarded(c, [&] {
        const bool in_u = (which == 0 || which == 1 || which == 3);
        const bool out_u = (which == 0 || which == 2);
        c->upload(in_u ? 0 : 1, in_u ? (int)U_IN : (int)P_IN, in);  // owned + ghost planes from the host vector
        for (int s = c->s0; s < c->s1; ++s) {
            Slab &S = c->slabs[s];
            const double *din = in_u ? S.u[U_IN] : S.p[P_IN];
            double *dout = out_u ? S.u[U_TMP] : S.p[P_TMP];
            switch (which) {
                case 0: launch_apply_A(S.geo, S.vrec, din, dout, S.m_own[0], c->d_diag_code, c->inv_h2, c->stream); break;
                case 1: launch_apply_div(S.geo, S.prec, din, dout, S.m_own[1], c->inv_h, c->stream); break;
                case 2: launch_apply_grad(S.geo, S.vrec, din, dout, S.m_own[0], c->inv_h, c->stream); break;
                case 3: launch_dwd(S.geo, S.prec, din, dout, S.m_own[1], c->inv_h2, c->stream); break;
                case 4: launch_apply_S(S.geo, S.prec, din, dout, S.m_own[1], c->d_invA_enc, c->inv_h, c->stream); break;
            }
        }
        CK(cudaGetLastError());
        c->download(out_u ? 0 : 1, out_u ? (int)U_TMP : (int)P_TMP, out);
        c->sync();
    });
}

int vs_apply_laplacian(vs_ctx *c, const double *u, double *out) { return apply_common(c, 0, u, out); }
int vs_apply_divergence(vs_ctx *c, const double *u, double *out) { return apply_common(c, 1, u, out); }
int vs_apply_gradient(vs_ctx *c, const double *p, double *out) { return apply_common(c, 2, p, out); }
int vs_divergence_weighted_diagonal(vs_ctx *c, const double *w, double *out) { return apply_common(c, 3, w, out); }
int vs_apply_simple(vs_ctx *c, const double *p, double *out) { return apply_common(c, 4, p, out); }

int vs_solve_velocity(vs_ctx *c, const double *rhs, const double *x0, double eps, double *x, int64_t *iters) {
    return guarded(c, [&] {
        reset_stats(c);
        c->upload(0, U_RHS, rhs);
        if (x0) c->upload(0, U_TMP, x0);
        *iters = cg_solve(c, 0, U_RHS, x0 ? U_TMP : -1, eps, U_W);
        c->download(0, U_W, x);
        c->sync();
    });
}

int vs_solve_simple(vs_ctx *c, const double *r, double eps, double *z, int64_t *iters) {
    return guarded(c, [&] {
        if (!c->sdiag_ok) throw Status{VS_EVALUE, "nonpositive diagonal entry in jacobi preconditioner"};
        reset_stats(c);
        c->upload(1, P_B, r);
        *iters = cg_solve(c, 1, P_B, -1, eps, P_Z);
        c->download(1, P_Z, z);
        c->sync();
    });
}

// ------------------------------------------------------------ solve_schur
// The outer PCG (krylov.py:76-182) over S = B A^-1 B^T with the SIMPLE or
// identity preconditioner (schur.py:291-385).  Every vector op, reduction
// and scalar update runs on the device in the reference's order; the host
// enqueues one outer iteration and synchronises once at its end to read the
// scalar state (convergence / error flags) and the inner-solve log.

static int solve_schur_impl(vs_ctx *c, const vs_schur_cfg *cfg, const double *g_override, double *pressure,
                            double *velocity, vs_report *rep, double *res_prec, double *res_unprec,
                            double *perm_history, double *alpha_out, double *beta_out) {
    return guarded(c, [&] {
        if (cfg->prec == 1 && !c->sdiag_ok)
            throw Status{VS_EVALUE, "nonpositive diagonal entry in jacobi preconditioner"};
        reset_stats(c);
        memset(rep, 0, sizeof *rep);
        cudaStream_t s = c->stream;
        const int R = c->R;
        const int use_prec = cfg->outer_norm == 0;
        // device histories: alpha, beta, res_prec, res_unprec, perm (stride max_iter + 2)
        const int64_t hs = cfg->max_iter + 2;
        if (hs > c->hist_cap) {
            c->hist = c->alloc<double>(5 * hs);
            c->hist_cap = hs;
        }
        OuterState init{};
        init.hstride = hs;
        CK(cudaMemcpyAsync(c->ost, &init, sizeof init, cudaMemcpyHostToDevice, s));
        double *mu = &c->ost->mu, *alpha = &c->ost->alpha, *beta = &c->ost->beta;
        CK(cudaEventRecord(c->ev0, s));
        auto perm = [&](int slot, int64_t k) {  // schur.py:288 -> hist perm[k + 1]
            c->reduce_dev(0, 0, slot, -1, Q_PERM, c->flow_dir);
            c->publish(Q_PERM, Q_PERM + 1);
            launch_outer(SO_PERM, c->ost, c->scal, R, cfg->h_pow_dim, k, 0, 0, c->hist, s, c->gate);
            ++c->launches;
        };
        auto mean_into_mu = [&](int slot) {
            c->reduce_dev(1, 0, slot, -1, Q_MU);
            c->publish(Q_MU, Q_MU + 1);
            launch_outer(SO_MEAN, c->ost, c->scal, R, (double)c->m_p, 0, 0, 0, c->hist, s, c->gate);
            ++c->launches;
        };
        int64_t tot_vel = 0, tot_pre = 0;
        std::vector<int> vel_logs;  // log slots counted in inner_iter_totals["velocity"]
        // drain the log + state after a sync; raise the first failure in program order
        auto settle = [&](int failure_stage_state) {
            fetch_log(c, 0);
            CK(cudaMemcpyAsync(c->h_ost, c->ost, sizeof(OuterState), cudaMemcpyDeviceToHost, s));
            c->sync();
            std::vector<int64_t> its(c->ncglog);
            // inner failures and outer flags interleave in program order: the
            // velocity solve precedes d'q, the preconditioner solve precedes
            // the r'z / norm checks
            for (int li = 0; li < c->ncglog; ++li) {
                const OuterState &o = *c->h_ost;
                if (c->log_op[li] == 1 && o.status == 2) break;  // d'q failed before the S_hat solve
                (void)failure_stage_state;
                const int save = c->ncglog;
                c->ncglog = li + 1;
                drain_log(c, li, &its[li]);
                c->ncglog = save;
            }
            for (int li = 0; li < c->ncglog; ++li) {
                if (c->log_op[li] == 0) tot_vel += its[li];
                else tot_pre += its[li];
            }
            const OuterState &o = *c->h_ost;
            char buf[256];
            if (o.status == 1) {
                snprintf(buf, sizeof buf, "preconditioner not SPD on subspace: r'z = %.3e at iteration %lld", o.value,
                         (long long)o.at);
                throw Status{VS_ERUNTIME, buf};
            }
            if (o.status == 2) {
                snprintf(buf, sizeof buf, "operator not SPD on subspace: d'q = %.3e at iteration %lld", o.value,
                         (long long)o.at);
                throw Status{VS_ERUNTIME, buf};
            }
            if (o.status == 3) {
                snprintf(buf, sizeof buf, "non-finite residual at iteration %lld", (long long)o.at);
                throw Status{VS_ERUNTIME, buf};
            }
            c->ncglog = 0;
        };
        // g, u_f = schur_rhs (schur.py:228-231, :308); the u_f solve is not counted (:230)
        c->ncglog = 0;
        c->force(U_RHS, -1);
        cg_async(c, 0, U_RHS, -1, cfg->eps_A, U_F);
        c->div(U_F, P_B);  // g -> P_B
        if (g_override) c->upload(1, P_B, g_override);  // vs_solve_schur_rhs: the caller's right-hand side
        // outer_op(p) = B A^-1 B^T p, last_w kept (schur.py:312-316)
        auto outer_op = [&](int p, int q) {
            c->grad(p, U_RHS);
            cg_async(c, 0, U_RHS, -1, cfg->eps_A, U_W);
            c->div(U_W, q);
        };
        // z = prec(r); z -= mean(z)   (schur.py:324-327, krylov.py:117-119, :151-153)
        auto outer_prec = [&](int r, int z) {
            if (cfg->prec == 1) {
                cg_async(c, 1, r, -1, cfg->eps_Shat, P_TMP);
                mean_into_mu(P_TMP);
                c->vec(1, 0, z, P_TMP, -1, 0.0, mu);
            } else {
                mean_into_mu(r);
                c->vec(1, 0, z, r, -1, 0.0, mu);
            }
        };
        auto norms = [&]() {  // r.z, z.z, r.r (krylov.py:141, :154-158)
            c->reduce_dev(1, 1, P_R, P_Z, Q_RZ);
            c->reduce_dev(1, 1, P_Z, P_Z, Q_ZZ);
            c->reduce_dev(1, 1, P_R, P_R, Q_RR);
            c->publish(Q_RZ, Q_RR + 1);
        };
        // u = u_f.copy(); perm_history = [k(u)]
        c->copy(0, U_ITER, U_F);
        perm(U_ITER, -1);
        // ---- outer pcg setup with project_nullspace=True (krylov.py:102-128)
        mean_into_mu(P_B);
        c->vec(1, 0, P_B, P_B, -1, 0.0, mu);  // rhs -= mean(rhs)
        for (int q = c->s0; q < c->s1; ++q)  // x = 0
            CK(cudaMemsetAsync(c->slabs[q].p[P_X], 0, c->slabs[q].m_all[1] * sizeof(double), s));
        outer_op(P_X, P_Q);
        c->vec(1, 4, P_R, P_Q, P_B, 0.0);  // r = op(x) - rhs
        outer_prec(P_R, P_Z);
        norms();
        launch_outer(SO_INIT, c->ost, c->scal, R, 0, 0, cfg->eps_S, use_prec, c->hist, s, c->gate);
        ++c->launches;
        c->copy(1, P_D, P_Z);
        {
            // the u_f solve (log slot 0) is discarded from the totals
            fetch_log(c, 0);
            CK(cudaMemcpyAsync(c->h_ost, c->ost, sizeof(OuterState), cudaMemcpyDeviceToHost, s));
            c->sync();
            int64_t its[16] = {0};
            drain_log(c, 0, its);
            rep->uf_iters = its[0];
            for (int li = 1; li < c->ncglog; ++li) {
                if (c->log_op[li] == 0) tot_vel += its[li];
                else tot_pre += its[li];
            }
            c->ncglog = 0;
            const OuterState &o = *c->h_ost;
            if (o.status == 1) {
                char buf[256];
                snprintf(buf, sizeof buf, "preconditioner not SPD on subspace: r'z = %.3e at iteration %lld", o.value,
                         (long long)o.at);
                throw Status{VS_ERUNTIME, buf};
            }
        }
        // Small operators: an outer iteration is a few hundred microseconds of kernels,
        // and a host round trip per iteration (read the state, enqueue the next ~20
        // launches) leaves the GPU idle for about a third as long.  There, `batch`
        // iterations are enqueued per synchronisation, every kernel gated on the
        // device-side stop flag (set with `converged` / `status` by k_outer), so the
        // iterations enqueued past convergence are no-ops and the results are the ones of
        // the one-by-one loop.  VOXSCHUR_OUTER_BATCH overrides (1 = one by one).
        int batch = (R == 1 && !c->mp() && !c->use_tile[0] && !c->use_tile[1] && c->m_u <= ((int64_t)1 << 21)) ? 4 : 1;
        if (const char *eb = getenv("VOXSCHUR_OUTER_BATCH")) batch = std::max(1, std::min(atoi(eb), GROUP_RING / 2));
        if (R > 1 || c->mp()) batch = 1;  // halo copies and cross-rank barriers are not gated
        int in_batch = 0;
        for (int64_t k = 0; k < cfg->max_iter && !c->h_ost->converged; ++k) {
            c->gate = batch > 1 ? &c->ost->stop : nullptr;
            outer_op(P_D, P_Q);
            c->reduce_dev(1, 1, P_D, P_Q, Q_DQ);
            c->publish(Q_DQ, Q_DQ + 1);
            launch_outer(SO_ALPHA, c->ost, c->scal, R, 0, k, 0, 0, c->hist, s, c->gate);  // alpha = rz / d'q
            ++c->launches;
            c->vec(1, 1, -1, P_X, P_D, 0.0, alpha);    // x -= alpha d
            c->vec(1, 1, -1, P_R, P_Q, 0.0, alpha);    // r -= alpha q
            c->vec(0, 2, -1, U_ITER, U_W, 0.0, alpha);  // u += alpha w (schur.py:334-336)
            perm(U_ITER, k);
            outer_prec(P_R, P_Z);
            norms();
            launch_outer(SO_BETA, c->ost, c->scal, R, 0, k, cfg->eps_S, use_prec, c->hist, s, c->gate);
            ++c->launches;
            c->vec(1, 3, P_D, P_D, P_Z, 0.0, beta);  // d = z + beta d (unused once converged)
            c->gate = nullptr;
            if (++in_batch == batch || k + 1 == cfg->max_iter) {
                settle(0);
                in_batch = 0;
            }
        }
        c->gate = nullptr;
        const int64_t its = c->h_ost->its;
        const bool conv = c->h_ost->converged != 0;
        // refresh: A u = f - B^T p, warm start from u (schur.py:352-357)
        c->grad(P_X, U_TMP);
        c->force(U_RHS, U_TMP);
        cg_async(c, 0, U_RHS, U_ITER, cfg->eps_A, U_ITER);
        c->reduce_dev(0, 0, U_ITER, -1, Q_PERM, c->flow_dir);
        c->publish(Q_PERM, Q_PERM + 1);
        CK(cudaMemcpyAsync(c->h_scal, c->scal, Q_COUNT * R * sizeof(double), cudaMemcpyDeviceToHost, s));
        settle(0);
        double ksum = c->h_scal[Q_PERM * R];
        for (int q = 1; q < R; ++q) ksum = ksum + c->h_scal[Q_PERM * R + q];
        const double kval = cfg->h_pow_dim * ksum;
        CK(cudaEventRecord(c->ev1, s));
        c->download(1, P_X, pressure);
        c->download(0, U_ITER, velocity);
        std::vector<double> h(5 * hs);
        CK(cudaMemcpyAsync(h.data(), c->hist, 5 * hs * sizeof(double), cudaMemcpyDeviceToHost, s));
        c->sync();
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        h[4 * hs + its] = kval;  // perm_history[-1] = k of the refreshed velocity (schur.py:357)
        rep->k_value = kval;
        rep->iters_outer = its;
        rep->converged = conv ? 1 : 0;
        rep->inner_velocity = tot_vel;
        rep->inner_preconditioner = tot_pre;
        rep->n_hist = its + 1;
        rep->device_ms = ms;
        auto put = [&](double *dst, int which, int64_t cnt) {
            if (dst && cnt > 0) memcpy(dst, h.data() + which * hs, cnt * sizeof(double));
        };
        put(alpha_out, 0, its);
        put(beta_out, 1, its);
        put(res_prec, 2, its + 1);
        put(res_unprec, 3, its + 1);
        put(perm_history, 4, its + 1);
    });
}

int vs_solve_schur(vs_ctx *c, const vs_schur_cfg *cfg, double *pressure, double *velocity, vs_report *rep,
                   double *res_prec, double *res_unprec, double *perm_history, double *alpha_out,
                   double *beta_out) {
    return solve_schur_impl(c, cfg, nullptr, pressure, velocity, rep, res_prec, res_unprec, perm_history,
                            alpha_out, beta_out);
}

int vs_solve_schur_rhs(vs_ctx *c, const vs_schur_cfg *cfg, const double *g, double *pressure, double *velocity,
                       vs_report *rep, double *res_prec, double *res_unprec, double *perm_history,
                       double *alpha_out, double *beta_out) {
    if (!g) return fail(VS_EVALUE, "vs_solve_schur_rhs needs a right-hand side");
    return solve_schur_impl(c, cfg, g, pressure, velocity, rep, res_prec, res_unprec, perm_history, alpha_out,
                            beta_out);
}

int vs_phase_timing(vs_ctx *c, double *ns12) {
    return guarded(c, [&] {
        unsigned long long h[12] = {0};
        if (c->phase_ns) {
            CK(cudaMemcpyAsync(h, c->phase_ns, sizeof h, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemsetAsync(c->phase_ns, 0, sizeof h, c->stream));
            c->sync();
        }
        for (int k = 0; k < 12; ++k) ns12[k] = (double)h[k];
    });
}

int vs_kernel_stats(vs_ctx *c, vs_kstat *a, vs_kstat *s, int64_t *launches) {
    if (a) *a = c->st_A;
    if (s) *s = c->st_S;
    if (launches) *launches = c->launches;
    return VS_OK;
}

int vs_slab_count(vs_ctx *c) { return c->R; }

int vs_ctx_limit_sms(vs_ctx *c, int sms) {
    if (sms < 0) return fail(VS_EVALUE, "sms must be >= 0, got %d", sms);
    if (c->R > 1 || c->use_tile[0] || c->use_tile[1])
        return fail(VS_EVALUE, "SM limit applies to single-slab contexts without tiled solves");
    // grids only shrink, so the buffers sized for tb_max still fit
    return guarded(c, [&] { plan_solvers(c, c->mu_max, c->mp_max, sms); });
}

int vs_ctx_sms(vs_ctx *c) { return c->sms; }

int vs_solve_span_ms(vs_ctx *first, vs_ctx *last, double *ms) {
    return guarded(first, [&] {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, first->ev0, last->ev1));
        *ms = t;
    });
}

}  // extern "C"
