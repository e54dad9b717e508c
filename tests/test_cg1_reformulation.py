"""The one-reduction (Chronopoulos-Gear) PCG that k_cg1 / k_cg1t run, restated
in numpy and checked against the oracle's two-reduction PCG (the reference's
krylov.py:76-182) on the golden geometries: same iteration counts to within
2 %, same solutions to the solve tolerance.  This is the CPU half of the
argument that the reformulation keeps parity; the GPU
half is tests/test_gpu_parity.py run with both kernels.

The recurrences (vs_cg.cu, k_cg1): zr = M r (unprojected), z = zr - mu,
w = A zr, u = M w, s = M q, gamma = r.z, delta = z.w;
beta = gamma/gamma_prev, alpha = gamma / (delta - beta gamma / alpha_prev),
d = z + beta d, s = u + beta s, x -= alpha d, zr -= alpha s.
"""
import numpy as np
import pytest

from conftest import load_golden
from oracle import voxoracle as vo


def pcg_one_sum(op, inv, rhs, tol, project, max_iter):
    diag = 1.0 / inv
    rhs = np.array(rhs, float)
    x = np.zeros_like(rhs)
    m = rhs.size
    if project:
        rhs = rhs - rhs.mean()
    r = op(x) - rhs
    zr = r * inv
    mu = zr.sum() / m if project else 0.0
    w = op(zr)
    u = w * inv
    gamma = r @ zr - mu * r.sum()
    nz2 = zr @ zr - mu * zr.sum()
    delta = zr @ w - mu * w.sum()
    ref = np.sqrt(nz2)
    if ref == 0.0:
        return x, 0
    d = np.zeros_like(x)
    s = np.zeros_like(x)
    g_prev = a_prev = None
    for it in range(max_iter):
        if it == 0:
            beta, dq = 0.0, delta
        else:
            beta = gamma / g_prev
            dq = delta - beta * gamma / a_prev
        assert gamma > 0 and dq > 0
        alpha = gamma / dq
        d = (zr - mu) + beta * d
        s = u + beta * s
        x = x - alpha * d
        zr = zr - alpha * s
        w = op(zr)
        u = w * inv
        rr = zr * diag
        mu = zr.sum() / m if project else 0.0
        g_prev, a_prev = gamma, alpha
        gamma = rr @ zr - mu * rr.sum()
        nz2 = zr @ zr - mu * zr.sum()
        delta = zr @ w - mu * w.sum()
        if np.sqrt(nz2) / ref < tol:
            return x, it + 1
    raise AssertionError("no convergence")


def within_2pct(a, b):
    return abs(int(a) - int(b)) <= max(1, int(np.ceil(0.02 * int(b))))


@pytest.mark.parametrize("name", ["pack2d", "pack3d", "rand3d", "disks2d", "spheres3d"])
def test_inner_solves_match_two_sum_pcg(name):
    g = load_golden(name)
    sys_ = vo.build_system(g["fluid"], int(g["flow_dir"]))
    inv = 1.0 / sys_.laplacian_diag
    x1, i1 = pcg_one_sum(sys_.apply_laplacian, inv, sys_.force, 1e-12, False, vo._inner_max(sys_.m_u))
    x2, i2 = vo.solve_velocity(sys_, sys_.force, 1e-12)
    assert within_2pct(i1, i2), (i1, i2)
    assert np.linalg.norm(x1 - x2) <= 1e-10 * np.linalg.norm(x2)
    p = g["p_in"] - g["p_in"].mean()
    inv_s = 1.0 / vo.simple_inverse_diag(sys_)
    z1, j1 = pcg_one_sum(sys_.apply_simple, inv_s, p, 1e-12, True, vo._inner_max(sys_.m_p))
    z2, j2 = vo.solve_simple(sys_, p, 1e-12, inv_s)
    assert within_2pct(j1, j2), (j1, j2)
    assert np.linalg.norm(z1 - z2) <= 1e-9 * np.linalg.norm(z2)
