"""Pin the CPU oracle to the reference's own outputs (tests/golden)."""
import numpy as np
import pytest

from conftest import load_golden
from oracle import voxoracle as vo

TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)


def test_geometry_and_applies_bitwise(golden):
    name, g = golden
    sys = vo.build_system(g["fluid"], int(g["flow_dir"]))
    assert sys.m_u == g["m_u"] and sys.m_p == g["m_p"]
    assert tuple(sys.axis_counts) == tuple(g["axis_counts"])
    for a in range(sys.dim):
        assert np.array_equal(sys.masks[a], g[f"face_mask{a}"])
    assert np.array_equal(sys.laplacian_diag, g["diag"])
    assert np.array_equal(sys.force, g["force"])
    assert np.array_equal(sys.apply_laplacian(g["u_in"]), g["Au"])
    assert np.array_equal(sys.apply_divergence(g["u_in"]), g["Bu"])
    assert np.array_equal(sys.apply_gradient(g["p_in"]), g["Btp"])
    assert np.array_equal(sys.apply_simple(g["p_in"]), g["Sp"])
    assert np.array_equal(sys.divergence_weighted_diagonal(1.0 / sys.laplacian_diag), g["dwd"])


def test_inner_solves_bitwise(golden):
    name, g = golden
    sys = vo.build_system(g["fluid"], int(g["flow_dir"]))
    uf, _ = vo.solve_velocity(sys, sys.force, 1e-12)
    assert np.array_equal(uf, g["u_f"])
    assert np.array_equal(sys.apply_divergence(uf), g["g"])
    if "simple_inv" in g:
        p = g["p_in"] - g["p_in"].mean()
        z, _ = vo.solve_simple(sys, p, 1e-12)
        assert np.array_equal(z, g["simple_inv"])


def _check_solve(rep, g, prefix):
    assert rep["iters_outer"] == g[prefix + "iters_outer"]
    assert rep["inner_iter_totals"]["velocity"] == g[prefix + "inner_velocity"]
    assert rep["inner_iter_totals"]["preconditioner"] == g[prefix + "inner_preconditioner"]
    assert bool(rep["converged"]) == bool(g[prefix + "converged"])
    # same machine, same numpy/BLAS thread count -> expected bitwise
    np.testing.assert_allclose(rep["pressure"], g[prefix + "pressure"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(rep["velocity"], g[prefix + "velocity"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(rep["perm_history"], g[prefix + "perm_history"], rtol=1e-12)
    np.testing.assert_allclose(rep["res_prec"], g[prefix + "res_prec"], rtol=1e-10)


@pytest.mark.parametrize("name", ["pack2d", "pack3d", "rand3d", "disks2d", "wrap2", "channel16"])
@pytest.mark.parametrize("prec", ["uzawa", "simple"])
def test_full_solve_matches_reference(name, prec):
    g = load_golden(name)
    sys = vo.build_system(g["fluid"], int(g["flow_dir"]))
    rep = vo.solve_schur(sys, prec, **TOL)
    _check_solve(rep, g, f"{prec}_")


def test_paper2d_profile_and_exhaustion():
    g = load_golden("pack2d")
    sys = vo.build_system(g["fluid"], 0)
    for prec in ("uzawa", "simple"):
        rep = vo.solve_schur(sys, prec, eps_S=1e-3, outer_norm="unpreconditioned",
                             eps_A=1e-13, eps_Shat=1e-13)
        _check_solve(rep, g, f"p2d_{prec}_")
    g = load_golden("exhaust")
    sys = vo.build_system(g["fluid"], 0)
    rep = vo.solve_schur(sys, "uzawa", eps_S=1e-9, outer_norm="unpreconditioned",
                         eps_A=1e-13, eps_Shat=1e-13, max_iter=2)
    _check_solve(rep, g, "exh_")
    assert not rep["converged"]


def test_components_match_reference():
    g = load_golden("components")
    for i in range(3):
        labels, n = vo.connected_components(g[f"fluid{i}"])
        assert n == g[f"ncomp{i}"]
        assert np.array_equal(labels, g[f"labels{i}"])
        kept, removed = vo.enforce_connectivity(g[f"fluid{i}"])
        assert np.array_equal(kept, g[f"kept{i}"]) and removed == g[f"removed{i}"]
