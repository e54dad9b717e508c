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

struct vs_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int dim = 0, n = 0, nw = 0, nlines = 0, flow_dir = 0;
    int64_t nwords = 0, ncells = 0;
    int64_t m_u = 0, m_p = 0, vcount[3] = {0, 0, 0}, voff[3] = {0, 0, 0};
    double inv_h = 0, inv_h2 = 0, diag_scale = 0;
    double diag_code[16] = {0}, inv_code[16] = {0}, invA_enc[8] = {0};
    bool sdiag_ok = true;
    std::vector<void *> allocs;
    // geometry
    uint32_t *fbits = nullptr;
    uint2 *vmeta[3] = {nullptr, nullptr, nullptr};
    uint2 *pmeta = nullptr;
    uint64_t *vrec = nullptr, *prec = nullptr;
    double *invS = nullptr, *d_diag_code = nullptr, *d_invA_enc = nullptr;
    // velocity work vectors
    double *u_rhs, *u_w, *u_iter, *u_f, *u_r, *u_z, *u_d0, *u_d1, *u_tmp;
    // pressure work vectors
    double *p_x, *p_r, *p_d, *p_z, *p_q, *p_b, *p_sr, *p_sz, *p_sd0, *p_sd1, *p_tmp;
    unsigned *bar = nullptr;
    unsigned long long *phase_ns = nullptr;  // VOXSCHUR_PHASE_TIMING=1
    double *part = nullptr, *red_part = nullptr, *scal = nullptr;
    CgOut *cgout = nullptr;
    double *h_scal = nullptr;  // pinned
    CgOut *h_cg = nullptr;     // pinned
    CgPlan plan_A{}, plan_S{};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs0 = nullptr, evs1 = nullptr;
    // stats of the last top-level call
    vs_kstat st_A{}, st_S{};
    int64_t launches = 0;

    Geo geo() const {
        Geo g;
        g.dim = dim; g.n = n; g.nw = nw; g.nlines = nlines;
        g.fbits = fbits;
        for (int a = 0; a < 3; ++a) g.vmeta[a] = vmeta[a];
        g.pmeta = pmeta;
        return g;
    }
    template <class T>
    T *alloc(size_t count) {
        void *p = nullptr;
        CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
        allocs.push_back(p);
        return (T *)p;
    }
    ~vs_ctx() {
        if (device >= 0) cudaSetDevice(device);
        for (void *p : allocs) cudaFree(p);
        if (h_scal) cudaFreeHost(h_scal);
        if (h_cg) cudaFreeHost(h_cg);
        for (cudaEvent_t e : {ev0, ev1, evs0, evs1})
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }
    void sync() { CK(cudaStreamSynchronize(stream)); }
    // deterministic device reduction, result on host
    double reduce(int kind, const double *a, const double *b, int64_t m) {
        if (m == 0) return 0.0;
        launches += launch_reduce(kind, a, b, m, red_part, scal, stream);
        CK(cudaMemcpyAsync(h_scal, scal, sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
        return h_scal[0];
    }
    double dot(const double *a, const double *b, int64_t m) { return reduce(1, a, b, m); }
    double sum(const double *a, int64_t m) { return reduce(0, a, nullptr, m); }
    double mean(const double *a, int64_t m) { return sum(a, m) / (double)m; }
    void vec(int kind, double *out, double *a, const double *b, double s, int64_t m) {
        launch_vec(kind, out, a, b, s, m, stream);
        ++launches;
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

// One fused device PCG solve.  op 0: velocity A (x0 allowed), op 1: S_hat
// (projected).  Returns the iteration count; throws Status on errors.
int64_t cg_solve(vs_ctx *c, int op, const double *rhs, const double *x0, double eps, double *x) {
    const int64_t m = op == 0 ? c->m_u : c->m_p;
    if (m == 0) return 0;
    CgParams P;
    memset(&P, 0, sizeof P);
    P.g = c->geo();
    P.m = m;
    P.rec = op == 0 ? c->vrec : c->prec;
    P.rhs = rhs;
    P.x0 = x0;
    P.x = x;
    P.r = op == 0 ? c->u_r : c->p_sr;
    P.z = op == 0 ? c->u_z : c->p_sz;
    P.bar = c->bar;
    P.phase_ns = c->phase_ns;
    P.d0 = op == 0 ? c->u_d0 : c->p_sd0;
    P.d1 = op == 0 ? c->u_d1 : c->p_sd1;
    P.part = c->part;
    P.out = c->cgout;
    P.tol = eps;
    P.max_iter = std::max<int64_t>(1000, 2 * m);  // schur.py:196-197
    P.norm_prec = 1;
    P.inv_h = c->inv_h;
    P.inv_h2 = c->inv_h2;
    memcpy(P.diag_code, c->diag_code, sizeof P.diag_code);
    memcpy(P.inv_code, c->inv_code, sizeof P.inv_code);
    memcpy(P.invA_enc, c->invA_enc, sizeof P.invA_enc);
    P.invS = c->invS;
    const CgPlan &pl = op == 0 ? c->plan_A : c->plan_S;
    CK(cudaMemsetAsync(c->bar, 0, sizeof(unsigned), c->stream));
    ++c->launches;
    CK(cudaEventRecord(c->evs0, c->stream));
    CK(launch_pcg(c->dim, op, pl, P, c->stream));
    CK(cudaEventRecord(c->evs1, c->stream));
    ++c->launches;
    CK(cudaMemcpyAsync(c->h_cg, c->cgout, sizeof(CgOut), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, c->evs0, c->evs1));
    const CgOut o = *c->h_cg;
    vs_kstat &st = op == 0 ? c->st_A : c->st_S;
    st.launches += 1;
    st.iterations += o.iterations;
    st.dof_iters += o.iterations * m;
    st.ms += ms;
    Status s = cg_status_to_error(o, op);
    if (s.code != VS_OK) throw s;
    return o.iterations;
}

void reset_stats(vs_ctx *c) {
    c->st_A = vs_kstat{};
    c->st_S = vs_kstat{};
    c->launches = 0;
}

template <class F>
int guarded(vs_ctx *c, F &&f) {
    try {
        if (c) CK(cudaSetDevice(c->device));
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

void h2d_tmp_upload(vs_ctx *c, double *dst, const double *src, int64_t m) {
    if (m) CK(cudaMemcpyAsync(dst, src, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
}
void d2h(vs_ctx *c, double *dst, const double *src, int64_t m) {
    if (m && dst) CK(cudaMemcpyAsync(dst, src, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
}

}  // namespace

// =================================================================== ABI

extern "C" {

const char *vs_last_error(void) { return g_err.c_str(); }

const char *vs_version(void) { return "voxschur 0.1 sm_100a (fp64, fused persistent PCG)"; }

int vs_components(const uint8_t *fluid, int dim, int n, int32_t *labels, int64_t *n_components) {
    if ((dim != 2 && dim != 3) || n < 1) return fail(VS_EVALUE, "grid dimension must be 2 or 3, got %d", dim);
    try {
        *n_components = label_components(fluid, dim, n, labels);
    } catch (const std::bad_alloc &) {
        return fail(VS_ECUDA, "host allocation failed");
    }
    return VS_OK;
}

int vs_stamp_balls(uint8_t *fluid, int dim, int n, const double *centers, const double *radii, int64_t count,
                   int64_t target_fluid, int prism_axis, int64_t *used, int64_t *n_fluid) {
    if ((dim != 2 && dim != 3) || n < 2) return fail(VS_EVALUE, "bad grid for vs_stamp_balls");
    const int64_t N = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    int64_t nf = 0;
    for (int64_t i = 0; i < N; ++i) nf += fluid[i] ? 1 : 0;
    int64_t k = 0;
    const int64_t st[3] = {dim == 3 ? (int64_t)n * n : (int64_t)n, dim == 3 ? (int64_t)n : 1, 1};
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
        if (nf <= target_fluid) { ++k; break; }
    }
    *used = k;
    *n_fluid = nf;
    return VS_OK;
}

int vs_ctx_create(const uint8_t *fluid, int dim, int n, int flow_dir, int check_connectivity, int require_walls,
                  int device, double inv_h, double inv_h2, vs_ctx **out) {
    *out = nullptr;
    if (dim != 2 && dim != 3) return fail(VS_EVALUE, "grid dimension must be 2 or 3, got %d", dim);
    if (n < 2) return fail(VS_EVALUE, "grid extent must be at least 2, got %d", n);
    if (n > 2047) return fail(VS_EVALUE, "grid extent %d exceeds the record layout limit 2047", n);
    if (flow_dir < 0 || flow_dir >= dim) return fail(VS_EVALUE, "flow axis %d out of range for dim %d", flow_dir, dim);
    const int64_t ncells = dim == 3 ? (int64_t)n * n * n : (int64_t)n * n;
    // operators.py:220-230 -- host-side validation and connectivity
    int64_t nfluid = 0;
    for (int64_t i = 0; i < ncells; ++i) nfluid += fluid[i] ? 1 : 0;
    if (nfluid == 0) return fail(VS_EVALUE, "empty fluid domain");
    if (require_walls && nfluid == ncells) return fail(VS_EVALUE, "velocity operator singular: no no-slip boundary");
    if (check_connectivity) {
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
        for (cudaEvent_t *e : {&C->ev0, &C->ev1, &C->evs0, &C->evs1}) CK(cudaEventCreate(e));
        CK(cudaMallocHost(&C->h_scal, 8 * sizeof(double)));
        CK(cudaMallocHost(&C->h_cg, sizeof(CgOut)));
        const int64_t nw = C->nwords;
        // ---- K1: mask -> bits -> face bits -> ranks -> records
        uint8_t *d_fluid = C->alloc<uint8_t>(ncells);
        CK(cudaMemcpyAsync(d_fluid, fluid, ncells, cudaMemcpyHostToDevice, C->stream));
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
        // counts per family: popc on host-visible totals via the scans
        uint32_t off = 0;
        for (int a = 0; a < dim; ++a) {
            C->vmeta[a] = C->alloc<uint2>(nw);
            CK(build_meta(fb[a], nw, off, C->vmeta[a], cnt, base, temp, tb, C->stream));
            uint32_t last[2];
            uint2 lastm;
            CK(cudaMemcpyAsync(&lastm, C->vmeta[a] + nw - 1, sizeof(uint2), cudaMemcpyDeviceToHost, C->stream));
            C->sync();
            last[0] = lastm.y;
            last[1] = __builtin_popcount(lastm.x);
            C->vcount[a] = (int64_t)last[0] + last[1] - off;
            C->voff[a] = off;
            if ((uint64_t)off + C->vcount[a] > 0xFFFFFFF0ull) throw Status{VS_EVALUE, "too many velocity DOFs"};
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
            C->diag_code[code] = (double)code * C->diag_scale;       // operators.py:285
            C->inv_code[code] = code ? 1.0 / C->diag_code[code] : 0.0;  // krylov.py:213
        }
        const int cbase = 2 * dim - 1;
        for (int e = 0; e < 8; ++e)
            C->invA_enc[e] = e ? 1.0 / ((double)(e + cbase) * C->diag_scale) : 0.0;  // schur.py:235
        // diag(S_hat) by the packed face codes, summed in reference order
        const int nkey = 1 << 18;
        std::vector<double> invS(1 << 18, 0.0);
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
        }
        C->invS = C->alloc<double>(1 << 18);
        CK(cudaMemcpyAsync(C->invS, invS.data(), (1 << 18) * sizeof(double), cudaMemcpyHostToDevice, C->stream));
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
        // ---- work vectors
        const int64_t mu = C->m_u, mp = C->m_p;
        for (double **v : {&C->u_rhs, &C->u_w, &C->u_iter, &C->u_f, &C->u_r, &C->u_z, &C->u_d0, &C->u_d1, &C->u_tmp})
            *v = C->alloc<double>(mu);
        for (double **v : {&C->p_x, &C->p_r, &C->p_d, &C->p_z, &C->p_q, &C->p_b, &C->p_sr, &C->p_sz, &C->p_sd0,
                           &C->p_sd1, &C->p_tmp})
            *v = C->alloc<double>(mp);
        C->plan_A = pcg_plan(dim, 0, C->m_u, device);
        C->plan_S = pcg_plan(dim, 1, C->m_p, device);
        C->bar = C->alloc<unsigned>(2);
        if (getenv("VOXSCHUR_PHASE_TIMING")) {
            C->phase_ns = C->alloc<unsigned long long>(12);
            CK(cudaMemsetAsync(C->phase_ns, 0, 12 * sizeof(unsigned long long), C->stream));
        }
        CK(cudaMemsetAsync(C->bar, 0, 2 * sizeof(unsigned), C->stream));
        C->part = C->alloc<double>((size_t)4 * 8 * std::max(C->plan_A.grid, C->plan_S.grid));
        C->red_part = C->alloc<double>(RED_MAX_BLOCKS);
        C->scal = C->alloc<double>(8);
        C->cgout = C->alloc<CgOut>(1);
        C->sync();
    });
    if (rc != VS_OK) return rc;
    *out = c.release();
    return VS_OK;
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

static int apply_common(vs_ctx *c, int which, const double *in, double *out) {
    return guarded(c, [&] {
        const bool in_u = (which == 0 || which == 1 || which == 3);
        const bool out_u = (which == 0 || which == 2);
        const int64_t mi = in_u ? c->m_u : c->m_p, mo = out_u ? c->m_u : c->m_p;
        double *din = in_u ? c->u_tmp : c->p_tmp;
        double *dout = out_u ? c->u_rhs : c->p_b;
        h2d_tmp_upload(c, din, in, mi);
        const Geo g = c->geo();
        switch (which) {
            case 0: launch_apply_A(g, c->vrec, din, dout, c->m_u, c->d_diag_code, c->inv_h2, c->stream); break;
            case 1: launch_apply_div(g, c->prec, din, dout, c->m_p, c->inv_h, c->stream); break;
            case 2: launch_apply_grad(g, c->vrec, din, dout, c->m_u, c->inv_h, c->stream); break;
            case 3: launch_dwd(g, c->prec, din, dout, c->m_p, c->inv_h2, c->stream); break;
            case 4: launch_apply_S(g, c->prec, din, dout, c->m_p, c->d_invA_enc, c->inv_h, c->stream); break;
        }
        CK(cudaGetLastError());
        d2h(c, out, dout, mo);
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
        h2d_tmp_upload(c, c->u_rhs, rhs, c->m_u);
        if (x0) h2d_tmp_upload(c, c->u_tmp, x0, c->m_u);
        *iters = cg_solve(c, 0, c->u_rhs, x0 ? c->u_tmp : nullptr, eps, c->u_w);
        d2h(c, x, c->u_w, c->m_u);
        c->sync();
    });
}

int vs_solve_simple(vs_ctx *c, const double *r, double eps, double *z, int64_t *iters) {
    return guarded(c, [&] {
        if (!c->sdiag_ok) throw Status{VS_EVALUE, "nonpositive diagonal entry in jacobi preconditioner"};
        reset_stats(c);
        h2d_tmp_upload(c, c->p_b, r, c->m_p);
        *iters = cg_solve(c, 1, c->p_b, nullptr, eps, c->p_z);
        d2h(c, z, c->p_z, c->m_p);
        c->sync();
    });
}

// ------------------------------------------------------------ solve_schur

int vs_solve_schur(vs_ctx *c, const vs_schur_cfg *cfg, double *pressure, double *velocity, vs_report *rep,
                   double *res_prec, double *res_unprec, double *perm_history, double *alpha_out,
                   double *beta_out) {
    return guarded(c, [&] {
        if (cfg->prec == 1 && !c->sdiag_ok)
            throw Status{VS_EVALUE, "nonpositive diagonal entry in jacobi preconditioner"};
        reset_stats(c);
        memset(rep, 0, sizeof *rep);
        const int64_t mu = c->m_u, mp = c->m_p;
        const int64_t flo = c->voff[c->flow_dir], fcnt = c->vcount[c->flow_dir];
        const Geo g = c->geo();
        cudaStream_t s = c->stream;
        CK(cudaEventRecord(c->ev0, s));
        auto perm = [&](const double *u) { return cfg->h_pow_dim * c->sum(u + flo, fcnt); };  // schur.py:288
        int64_t tot_vel = 0, tot_pre = 0;
        // g, u_f = schur_rhs (schur.py:228-231, :308)
        launch_force(c->u_rhs, nullptr, flo, fcnt, mu, s);
        ++c->launches;
        rep->uf_iters = cg_solve(c, 0, c->u_rhs, nullptr, cfg->eps_A, c->u_f);
        launch_apply_div(g, c->prec, c->u_f, c->p_b, mp, c->inv_h, s);  // g -> p_b
        ++c->launches;
        // outer_op(p) = B A^-1 B^T p, last_w kept (schur.py:312-316)
        auto outer_op = [&](const double *p, double *q) {
            launch_apply_grad(g, c->vrec, p, c->u_rhs, mu, c->inv_h, s);
            ++c->launches;
            tot_vel += cg_solve(c, 0, c->u_rhs, nullptr, cfg->eps_A, c->u_w);
            launch_apply_div(g, c->prec, c->u_w, q, mp, c->inv_h, s);
            ++c->launches;
        };
        // z = prec(r); z -= mean(z)   (schur.py:324-327, krylov.py:117-119)
        auto outer_prec = [&](double *r, double *z) {
            if (cfg->prec == 1) {
                tot_pre += cg_solve(c, 1, r, nullptr, cfg->eps_Shat, c->p_tmp);
                const double m = c->mean(c->p_tmp, mp);
                c->vec(0, z, c->p_tmp, nullptr, m, mp);
            } else {
                const double m = c->mean(r, mp);
                c->vec(0, z, r, nullptr, m, mp);
            }
        };
        // u = u_f.copy(); perm_history = [k(u)]
        CK(cudaMemcpyAsync(c->u_iter, c->u_f, mu * sizeof(double), cudaMemcpyDeviceToDevice, s));
        std::vector<double> ph, rp, ru, al, be;
        ph.push_back(perm(c->u_iter));
        // ---- outer pcg (krylov.py:76-182) with project_nullspace=True
        const bool use_prec = cfg->outer_norm == 0;
        {
            const double mg = c->mean(c->p_b, mp);
            c->vec(0, c->p_b, c->p_b, nullptr, mg, mp);       // rhs -= mean(rhs)
            CK(cudaMemsetAsync(c->p_x, 0, mp * sizeof(double), s));  // x = 0 (- mean 0)
        }
        outer_op(c->p_x, c->p_q);
        c->vec(4, c->p_r, c->p_q, c->p_b, 0.0, mp);  // r = op(x) - rhs
        outer_prec(c->p_r, c->p_z);
        rp.push_back(std::sqrt(c->dot(c->p_z, c->p_z, mp)));
        ru.push_back(std::sqrt(c->dot(c->p_r, c->p_r, mp)));
        const double ref = use_prec ? rp[0] : ru[0];
        bool conv = ref == 0.0;
        int64_t its = 0;
        if (!conv) {
            CK(cudaMemcpyAsync(c->p_d, c->p_z, mp * sizeof(double), cudaMemcpyDeviceToDevice, s));
            double rz = c->dot(c->p_r, c->p_z, mp);
            char buf[256];
            for (int64_t k = 0; k < cfg->max_iter; ++k) {
                if (rz < 0.0) {
                    snprintf(buf, sizeof buf, "preconditioner not SPD on subspace: r'z = %.3e at iteration %lld", rz,
                             (long long)k);
                    throw Status{VS_ERUNTIME, buf};
                }
                if (rz == 0.0) { conv = true; break; }
                outer_op(c->p_d, c->p_q);
                const double dq = c->dot(c->p_d, c->p_q, mp);
                if (dq <= 0.0) {
                    snprintf(buf, sizeof buf, "operator not SPD on subspace: d'q = %.3e at iteration %lld", dq,
                             (long long)k);
                    throw Status{VS_ERUNTIME, buf};
                }
                const double alpha = rz / dq;
                c->vec(1, nullptr, c->p_x, c->p_d, alpha, mp);  // x -= alpha d
                c->vec(1, nullptr, c->p_r, c->p_q, alpha, mp);  // r -= alpha q
                c->vec(2, nullptr, c->u_iter, c->u_w, alpha, mu);  // u += alpha w (schur.py:334-336)
                ph.push_back(perm(c->u_iter));
                outer_prec(c->p_r, c->p_z);
                const double rz_new = c->dot(c->p_r, c->p_z, mp);
                const double beta = rz_new / rz;
                rz = rz_new;
                const double nz = std::sqrt(c->dot(c->p_z, c->p_z, mp));
                const double nr = std::sqrt(c->dot(c->p_r, c->p_r, mp));
                if (!(std::isfinite(nz) && std::isfinite(nr))) {
                    snprintf(buf, sizeof buf, "non-finite residual at iteration %lld", (long long)(k + 1));
                    throw Status{VS_ERUNTIME, buf};
                }
                al.push_back(alpha);
                be.push_back(beta);
                rp.push_back(nz);
                ru.push_back(nr);
                its = k + 1;
                if ((use_prec ? nz : nr) / ref < cfg->eps_S) { conv = true; break; }
                c->vec(3, c->p_d, c->p_d, c->p_z, beta, mp);  // d = z + beta d
            }
        }
        // refresh: A u = f - B^T p, warm start from u (schur.py:352-357)
        launch_apply_grad(g, c->vrec, c->p_x, c->u_tmp, mu, c->inv_h, s);
        launch_force(c->u_rhs, c->u_tmp, flo, fcnt, mu, s);
        c->launches += 2;
        tot_vel += cg_solve(c, 0, c->u_rhs, c->u_iter, cfg->eps_A, c->u_iter);
        const double kval = perm(c->u_iter);
        ph.back() = kval;
        CK(cudaEventRecord(c->ev1, s));
        d2h(c, pressure, c->p_x, mp);
        d2h(c, velocity, c->u_iter, mu);
        c->sync();
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        rep->k_value = kval;
        rep->iters_outer = its;
        rep->converged = conv ? 1 : 0;
        rep->inner_velocity = tot_vel;
        rep->inner_preconditioner = tot_pre;
        rep->n_hist = (int64_t)ph.size();
        rep->device_ms = ms;
        auto put = [](double *dst, const std::vector<double> &v) {
            if (dst && !v.empty()) memcpy(dst, v.data(), v.size() * sizeof(double));
        };
        put(res_prec, rp);
        put(res_unprec, ru);
        put(perm_history, ph);
        put(alpha_out, al);
        put(beta_out, be);
    });
}

int vs_phase_timing(vs_ctx *c, double *ns4) {
    return guarded(c, [&] {
        unsigned long long h[12] = {0};
        if (c->phase_ns) {
            CK(cudaMemcpyAsync(h, c->phase_ns, sizeof h, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemsetAsync(c->phase_ns, 0, sizeof h, c->stream));
            c->sync();
        }
        for (int k = 0; k < 12; ++k) ns4[k] = (double)h[k];
    });
}

int vs_kernel_stats(vs_ctx *c, vs_kstat *a, vs_kstat *s, int64_t *launches) {
    if (a) *a = c->st_A;
    if (s) *s = c->st_S;
    if (launches) *launches = c->launches;
    return VS_OK;
}

}  // extern "C"
