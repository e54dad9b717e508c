"""CPU oracle for the Schur-complement Stokes path (TEST INFRASTRUCTURE ONLY).

This module is a numpy restatement of the reference algorithm
(`voxstokes`, /root/reference/pkg/src/voxstokes) for the one hot path this
repository rebuilds: ``assemble`` -> ``solve_schur`` (Uzawa | SIMPLE) ->
velocity refresh -> permeability.  It exists to CHECK the CUDA library;
only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product
package (``paper_2307_05266_b200``) never imports it and has no CPU
fallback.

Every function cites the reference file:line it restates.  The discrete
contract is restated from the boolean mask alone,
not from the reference's index tables, and the floating-point operation
order is kept identical to the reference so that single operator applies
are bitwise equal.  The oracle is pinned against fixtures produced by the
reference itself (``tests/golden/make_golden.py``, checked by
``tests/test_oracle_golden.py``).
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

__all__ = [
    "OracleSystem",
    "build_system",
    "face_masks",
    "diag_codes",
    "pcg",
    "lanczos",
    "solve_schur",
    "connected_components",
    "enforce_connectivity",
    "simple_inverse_diag",
]


# --------------------------------------------------------------- geometry


def face_masks(fluid: np.ndarray) -> list:
    """Face (a, I) carries a DOF iff fluid[I] and fluid[I - e_a].

    Restates operators.py:232.
    """
    return [fluid & np.roll(fluid, 1, axis=a) for a in range(fluid.ndim)]


def diag_codes(fluid: np.ndarray, masks: list) -> list:
    """Per velocity component, the integer no-slip diagonal code of each DOF.

    Slot order (d, s) = (0,+1), (0,-1), (1,+1), ... as in
    operators.py:268-281: a same-axis slot adds 1; a tangential slot adds
    2 when the neighbour face is absent and both voxels beside it are
    solid, else 1.  Returned in DOF order (C-order of the face mask).
    """
    dim = fluid.ndim
    out = []
    for a in range(dim):
        mask = masks[a]
        code = np.zeros(int(mask.sum()), dtype=np.int64)
        for d in range(dim):
            for s in (1, -1):
                if d == a:
                    code += 1
                    continue
                nb_face = np.roll(mask, -s, axis=d)[mask]
                hi = np.roll(fluid, -s, axis=d)
                lo = np.roll(np.roll(fluid, 1, axis=a), -s, axis=d)
                both_solid = (~hi & ~lo)[mask]
                code += np.where(~nb_face & both_solid, 2, 1)
        out.append(code)
    return out


def connected_components(fluid: np.ndarray):
    """Periodic face-adjacency labelling, ids in first row-major appearance.

    Restates geometry.py:183-222 (ndimage.label + union-find across the
    periodic faces).  Returns (labels, n_components); labels -1 on solid.
    """
    from scipy import ndimage

    structure = ndimage.generate_binary_structure(fluid.ndim, 1)
    raw, n_raw = ndimage.label(fluid, structure=structure)
    if n_raw == 0:
        return np.full(fluid.shape, -1, dtype=np.int64), 0
    parent = np.arange(n_raw + 1)

    def find(i):
        while parent[i] != i:
            parent[i] = parent[parent[i]]
            i = parent[i]
        return i

    for axis in range(fluid.ndim):
        lo = np.take(raw, 0, axis=axis).ravel()
        hi = np.take(raw, -1, axis=axis).ravel()
        both = (lo > 0) & (hi > 0)
        for a, b in zip(lo[both].tolist(), hi[both].tolist()):
            ra, rb = find(a), find(b)
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
    remap = np.full(n_raw + 1, -1, dtype=np.int64)
    nxt = 0
    for lab in range(1, n_raw + 1):
        root = find(lab)
        if remap[root] < 0:
            remap[root] = nxt
            nxt += 1
        remap[lab] = remap[root]
    return remap[raw], nxt


def enforce_connectivity(fluid: np.ndarray):
    """Keep the largest component, ties to the lowest id (geometry.py:225-240)."""
    labels, n = connected_components(fluid)
    if n == 0:
        raise ValueError("empty fluid domain")
    if n == 1:
        return fluid.copy(), 0
    sizes = np.bincount(labels[labels >= 0], minlength=n)
    keep = labels == int(np.argmax(sizes))
    return keep, int(fluid.sum() - keep.sum())


# --------------------------------------------------------------- operators


@dataclass
class OracleSystem:
    """Matrix-free MAC operators restated from the mask.

    Mirrors StaggeredSystem (operators.py:86-206).  Gather tables are
    built here (sentinel index = m for an absent DOF, read as 0.0) but the
    arithmetic order is the reference's.
    """

    fluid: np.ndarray
    flow_dir: int
    n: int
    dim: int
    masks: list
    axis_counts: tuple
    axis_offsets: tuple
    m_u: int
    m_p: int
    codes: np.ndarray  # int64 per velocity DOF
    laplacian_diag: np.ndarray
    nb: list  # per slot, int64 gather index into padded velocity
    div_in: list
    div_out: list
    grad_hi: list
    grad_lo: list
    h: float
    inv_h: float
    inv_h2: float
    force: np.ndarray

    # A: operators.py:131-135 -- diag*u - inv_h2 * (left fold over slots)
    def apply_laplacian(self, u):
        u = np.asarray(u, dtype=float)
        pad = np.append(u, 0.0)
        acc = pad[self.nb[0]]
        for col in self.nb[1:]:
            acc = acc + pad[col]
        return self.laplacian_diag * u - self.inv_h2 * acc

    # B: operators.py:137-144
    def apply_divergence(self, u):
        pad = np.append(np.asarray(u, dtype=float), 0.0)
        out = np.zeros(self.m_p)
        for a in range(self.dim):
            out += pad[self.div_in[a]] - pad[self.div_out[a]]
        return out * self.inv_h

    # B^T: operators.py:146-153
    def apply_gradient(self, p):
        p = np.asarray(p, dtype=float)
        return np.concatenate(
            [(p[self.grad_hi[a]] - p[self.grad_lo[a]]) * self.inv_h for a in range(self.dim)]
        )

    # diag(B W B^T): operators.py:194-206
    def divergence_weighted_diagonal(self, w):
        pad = np.append(np.asarray(w, dtype=float), 0.0)
        out = np.zeros(self.m_p)
        for a in range(self.dim):
            out += pad[self.div_in[a]] + pad[self.div_out[a]]
        return out * self.inv_h2

    # SIMPLE operator: schur.py:234-240
    def apply_simple(self, p):
        inv_diag = 1.0 / self.laplacian_diag
        return self.apply_divergence(self.apply_gradient(p) * inv_diag)

    def permeability(self, u):
        """schur.py:275-288 -- h**dim * pairwise sum of the flow block."""
        lo = self.axis_offsets[self.flow_dir]
        cnt = self.axis_counts[self.flow_dir]
        return self.h ** self.dim * float(np.asarray(u)[lo : lo + cnt].sum())

    def face_ids(self, a):
        ids = np.full(self.fluid.shape, -1, dtype=np.int64)
        ids[self.masks[a]] = self.axis_offsets[a] + np.arange(self.axis_counts[a])
        return ids


def build_system(fluid, flow_dir: int = 0, check_connectivity: bool = True,
                 require_walls: bool = True) -> OracleSystem:
    """Restates assemble() (operators.py:209-302) from the mask."""
    fluid = np.ascontiguousarray(fluid, dtype=bool)
    dim = fluid.ndim
    n = fluid.shape[0]
    if not fluid.any():
        raise ValueError("empty fluid domain")
    if require_walls and fluid.all():
        raise ValueError("velocity operator singular: no no-slip boundary")
    if check_connectivity:
        _, ncomp = connected_components(fluid)
        if ncomp > 1:
            raise ValueError(
                f"fluid domain is disconnected ({ncomp} components); "
                "run enforce_connectivity first"
            )
    masks = face_masks(fluid)
    counts = tuple(int(m.sum()) for m in masks)
    m_u = sum(counts)
    offsets = tuple(sum(counts[:a]) for a in range(dim))
    if require_walls and m_u == 0:
        raise ValueError("no velocity unknowns: every face touches solid")
    ids = []
    for a in range(dim):
        g = np.full(fluid.shape, m_u, dtype=np.int64)  # sentinel = m_u
        g[masks[a]] = offsets[a] + np.arange(counts[a])
        ids.append(g)
    pid = np.full(fluid.shape, -1, dtype=np.int64)
    m_p = int(fluid.sum())
    pid[fluid] = np.arange(m_p)

    codes = np.concatenate(diag_codes(fluid, masks)) if m_u else np.zeros(0, np.int64)
    inv_h2_diag = (n / 1.0) ** 2  # operators.py:260 (exact for integer n)
    diag = codes.astype(float) * inv_h2_diag

    nb = []
    for d in range(dim):
        for s in (1, -1):
            nb.append(np.concatenate(
                [np.roll(ids[a], -s, axis=d)[masks[a]] for a in range(dim)]))
    div_in = [ids[a][fluid] for a in range(dim)]
    div_out = [np.roll(ids[a], -1, axis=a)[fluid] for a in range(dim)]
    grad_hi = [pid[masks[a]] for a in range(dim)]
    grad_lo = [np.roll(pid, 1, axis=a)[masks[a]] for a in range(dim)]

    h = 1.0 / n  # operators.py:100 (physical_length fixed to 1.0)
    force = np.zeros(m_u)
    force[offsets[flow_dir] : offsets[flow_dir] + counts[flow_dir]] = 1.0
    return OracleSystem(
        fluid=fluid, flow_dir=flow_dir, n=n, dim=dim, masks=masks,
        axis_counts=counts, axis_offsets=offsets, m_u=m_u, m_p=m_p,
        codes=codes, laplacian_diag=diag, nb=nb, div_in=div_in,
        div_out=div_out, grad_hi=grad_hi, grad_lo=grad_lo, h=h,
        inv_h=1.0 / h, inv_h2=1.0 / h**2, force=force,
    )


def simple_inverse_diag(sys: OracleSystem):
    """Jacobi diagonal of the SIMPLE operator (schur.py:320-322)."""
    return sys.divergence_weighted_diagonal(1.0 / sys.laplacian_diag)


# ------------------------------------------------------------------ Krylov


@dataclass
class PcgOut:
    solution: np.ndarray
    iterations: int
    alpha: np.ndarray
    beta: np.ndarray
    res_prec: np.ndarray
    res_unprec: np.ndarray
    converged: bool


def _exact_dot(a, b):
    import math

    return math.fsum(np.asarray(a) * np.asarray(b))


# dot product used by pcg: the reference's (numpy/BLAS) or, for the parity
# tests' rounding-sensitivity probe, an exactly rounded one (math.fsum)
_DOT = [lambda a, b: float(a @ b)]


def pcg(op, prec, rhs, x0=None, tol=1e-6, norm_kind="preconditioned",
        max_iter=10000, project=False, record=True, step_hook=None) -> PcgOut:
    """Preconditioned CG with r = op(x) - rhs, x -= alpha d (krylov.py:76-182)."""
    dot = _DOT[0]
    rhs = np.array(rhs, dtype=float)
    x = np.zeros_like(rhs) if x0 is None else np.array(x0, dtype=float)
    if prec is None:
        prec = lambda v: v  # noqa: E731
    if project:
        rhs = rhs - rhs.mean()
        x = x - x.mean()
    use_prec = norm_kind == "preconditioned"
    r = op(x) - rhs
    z = prec(r)
    if project:
        z = z - z.mean()
    rp = [float(np.sqrt(dot(z, z)))]
    ru = [float(np.sqrt(dot(r, r)))]
    ref = rp[0] if use_prec else ru[0]
    alphas, betas = [], []
    its = 0
    conv = ref == 0.0
    if not conv:
        d = z.copy()
        rz = dot(r, z)
        for k in range(max_iter):
            if rz < 0.0:
                raise RuntimeError(
                    f"preconditioner not SPD on subspace: r'z = {rz:.3e} at iteration {k}")
            if rz == 0.0:
                conv = True
                break
            q = op(d)
            dq = dot(d, q)
            if dq <= 0.0:
                raise RuntimeError(
                    f"operator not SPD on subspace: d'q = {dq:.3e} at iteration {k}")
            alpha = rz / dq
            x -= alpha * d
            r -= alpha * q
            if step_hook is not None:
                step_hook(k, alpha, x)
            z = prec(r)
            if project:
                z = z - z.mean()
            rz_new = dot(r, z)
            beta = rz_new / rz
            rz = rz_new
            nz = float(np.sqrt(dot(z, z)))
            nr = float(np.sqrt(dot(r, r)))
            if not (np.isfinite(nz) and np.isfinite(nr)):
                raise RuntimeError(f"non-finite residual at iteration {k + 1}")
            alphas.append(alpha)
            betas.append(beta)
            rp.append(nz)
            ru.append(nr)
            its = k + 1
            if (nz if use_prec else nr) / ref < tol:
                conv = True
                break
            d = z + beta * d
    if not record:
        alphas, betas = [], []
    return PcgOut(x, its, np.asarray(alphas), np.asarray(betas),
                  np.asarray(rp), np.asarray(ru), conv)


def lanczos(alpha, beta):
    """Extreme eigenvalues from CG coefficients (krylov.py:185-205)."""
    import scipy.linalg

    alpha = np.asarray(alpha, dtype=float)
    beta = np.asarray(beta, dtype=float)
    diag = 1.0 / alpha + np.concatenate(([0.0], beta[: alpha.size - 1] / alpha[:-1]))
    off = np.sqrt(np.maximum(beta[: alpha.size - 1], 0.0)) / alpha[:-1]
    eigs = scipy.linalg.eigvalsh_tridiagonal(diag, off)
    lo, hi = float(eigs[0]), float(eigs[-1])
    return lo, hi, hi / lo


# ----------------------------------------------------------- Schur driver


def _inner_max(m):
    return max(1000, 2 * m)  # schur.py:196-197


def solve_velocity(sys, rhs, eps, x0=None):
    """schur.py:200-219."""
    inv = 1.0 / sys.laplacian_diag
    res = pcg(sys.apply_laplacian, lambda r: r * inv, rhs, x0, eps,
              "preconditioned", _inner_max(sys.m_u), False, False)
    if not res.converged:
        raise RuntimeError(
            "inner velocity solve did not converge: relative residual "
            f"{res.res_prec[-1] / res.res_prec[0]:.3e} after {res.iterations} iterations")
    return res.solution, res.iterations


def solve_simple(sys, r, eps, inv_s=None):
    """schur.py:243-272 (projected Jacobi-PCG on B diag(A)^-1 B^T)."""
    if inv_s is None:
        dS = simple_inverse_diag(sys)
        if np.any(dS <= 0):
            raise ValueError("nonpositive diagonal entry in jacobi preconditioner")
        inv_s = 1.0 / dS
    res = pcg(sys.apply_simple, lambda v: v * inv_s, r, None, eps,
              "preconditioned", _inner_max(sys.m_p), True, False)
    if not res.converged:
        raise RuntimeError(
            "inner pressure preconditioner solve did not converge: relative "
            f"residual {res.res_prec[-1] / res.res_prec[0]:.3e} after "
            f"{res.iterations} iterations")
    return res.solution, res.iterations


def solve_schur(sys: OracleSystem, prec="simple", eps_S=1e-3,
                outer_norm="preconditioned", eps_A=1e-6, eps_Shat=1e-6,
                max_iter=1000, k_ref=None, exact_dots=False) -> dict:
    """Outer PCG on S p = g (schur.py:291-385); exact_dots=True re-runs the
    same algorithm with exactly rounded dot products (rounding-sensitivity
    probe for the parity tests)."""
    if exact_dots:
        old = _DOT[0]
        _DOT[0] = _exact_dot
        try:
            return solve_schur(sys, prec, eps_S, outer_norm, eps_A, eps_Shat, max_iter, k_ref)
        finally:
            _DOT[0] = old
    return _solve_schur(sys, prec, eps_S, outer_norm, eps_A, eps_Shat, max_iter, k_ref)


def _solve_schur(sys, prec, eps_S, outer_norm, eps_A, eps_Shat, max_iter, k_ref) -> dict:
    """Outer PCG on S p = g with velocity iterate and refresh (schur.py:291-385).

    Returns a dict with the SolveReport fields (plus ``uf_iters``, the
    discarded iteration count of the u_f solve, for byte accounting).
    """
    t0 = time.perf_counter()
    totals = {"velocity": 0, "preconditioner": 0}
    u_f, uf_its = solve_velocity(sys, sys.force, eps_A)
    g = sys.apply_divergence(u_f)
    last_w = [None]

    def outer_op(p):
        w, its = solve_velocity(sys, sys.apply_gradient(p), eps_A)
        totals["velocity"] += its
        last_w[0] = w
        return sys.apply_divergence(w)

    if prec == "simple":
        dS = simple_inverse_diag(sys)
        if np.any(dS <= 0):
            raise ValueError("nonpositive diagonal entry in jacobi preconditioner")
        inv_s = 1.0 / dS

        def outer_prec(r):
            z, its = solve_simple(sys, r, eps_Shat, inv_s)
            totals["preconditioner"] += its
            return z
    else:
        outer_prec = None

    u = u_f.copy()
    perm = [sys.permeability(u)]

    def hook(_k, alpha, _x):
        u[:] += alpha * last_w[0]
        perm.append(sys.permeability(u))

    outer = pcg(outer_op, outer_prec, g, None, eps_S, outer_norm, max_iter,
                True, True, hook)
    p = outer.solution
    vel, its = solve_velocity(sys, sys.force - sys.apply_gradient(p), eps_A, x0=u)
    totals["velocity"] += its
    k = sys.permeability(vel)
    perm[-1] = k
    if outer.alpha.size >= 2:
        lo, hi, cond = lanczos(outer.alpha, outer.beta)
    else:
        lo = hi = cond = None
    perm = np.asarray(perm)
    return dict(
        pressure=p, velocity=vel, k_value=k, iters_outer=outer.iterations,
        converged=outer.converged, res_prec=outer.res_prec,
        res_unprec=outer.res_unprec, perm_history=perm,
        perm_err_history=None if k_ref is None else np.abs(perm - k_ref) / k_ref,
        cond_est_outer=cond, lambda_min_est=lo, lambda_max_est=hi,
        inner_iter_totals=totals, wall_time=time.perf_counter() - t0,
        alpha=outer.alpha, beta=outer.beta, uf_iters=uf_its,
    )
