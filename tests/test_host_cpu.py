"""CPU-only checks: the C ABI library loads and exports every declared symbol,
the native host logic (periodic connectivity) matches the reference's
golden labels, and the Python mirror of the reference API validates like
the reference (no GPU compute here)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import _lib  # noqa: E402


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "voxschur.h")).read()
    return sorted(set(re.findall(r"\b(vs_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_library_is_sm100a():
    path = _lib.LIB_PATH
    assert os.path.exists(path)
    assert b"sm_100a" in _lib.lib.vs_version()


def test_components_match_reference_labels():
    g = load_golden("components")
    for i in range(3):
        grid = vx.VoxelGrid(g[f"fluid{i}"])
        labels, n = vx.connected_components(grid)
        assert n == g[f"ncomp{i}"]
        assert np.array_equal(labels, g[f"labels{i}"])
        kept, removed = vx.enforce_connectivity(grid)
        assert np.array_equal(kept.fluid, g[f"kept{i}"]) and removed == g[f"removed{i}"]


def test_components_golden_geometries_connected(golden):
    name, g = golden
    _, n = vx.connected_components(vx.VoxelGrid(g["fluid"]))
    assert n == 1


def test_assemble_host_validation_errors():
    # these are raised before any device work, as in operators.py:220-230
    with pytest.raises(ValueError, match="no no-slip boundary"):
        vx.assemble(vx.VoxelGrid(np.ones((4, 4), dtype=bool)))
    with pytest.raises(ValueError, match="empty fluid"):
        vx.assemble(vx.VoxelGrid(np.zeros((4, 4), dtype=bool)))
    fluid = np.zeros((6, 6), dtype=bool)
    fluid[1, 1] = fluid[4, 4] = True
    with pytest.raises(ValueError, match="disconnected \\(2 components\\); run enforce_connectivity"):
        vx.assemble(vx.VoxelGrid(fluid))


def test_voxelgrid_validation():
    with pytest.raises(ValueError, match="dimension"):
        vx.VoxelGrid(np.ones(4, dtype=bool))
    with pytest.raises(ValueError, match="cubic"):
        vx.VoxelGrid(np.ones((4, 5), dtype=bool))
    with pytest.raises(ValueError, match="at least 2"):
        vx.VoxelGrid(np.ones((1, 1), dtype=bool))
    g = vx.VoxelGrid(np.ones((3, 3, 3), dtype=bool))
    assert g.dim == 3 and g.n == 3 and not g.fluid.flags.writeable


def test_axis_index():
    assert vx.axis_index("x", 2) == 0
    assert vx.axis_index("Z", 3) == 2
    with pytest.raises(ValueError, match="out of range"):
        vx.axis_index("z", 2)
    with pytest.raises(ValueError, match="unknown axis"):
        vx.axis_index("w", 2)


def test_config_validation_and_profiles():
    with pytest.raises(ValueError, match="prec"):
        vx.SchurConfig(prec="ilu")
    with pytest.raises(ValueError, match="outer_norm"):
        vx.SchurConfig(prec="uzawa", outer_norm="energy")
    with pytest.raises(ValueError, match="eps_S"):
        vx.SchurConfig(prec="uzawa", eps_S=0.0)
    with pytest.raises(ValueError, match="eps_A"):
        vx.SchurConfig(prec="uzawa", eps_A=1.5)
    with pytest.raises(ValueError, match="max_iter"):
        vx.SchurConfig(prec="uzawa", max_iter=0)
    with pytest.warns(UserWarning, match="eps_A"):
        vx.SchurConfig(prec="uzawa", eps_S=1e-8, eps_A=1e-6)
    cfg = vx.profile_config("paper2d", "uzawa")
    assert cfg.outer_norm == "unpreconditioned" and cfg.eps_A == 1e-13
    with pytest.raises(ValueError, match="profile"):
        vx.profile_config("paper4d", "uzawa")


# ---- the generic host Krylov seam (krylov.py:76-214) --------------------


def test_pcg_identity_and_exact_start():
    rng = np.random.default_rng(0)
    rhs, x0 = rng.standard_normal(15), rng.standard_normal(15)
    res = vx.pcg(lambda v: v, None, rhs, x0, vx.PcgConfig(tol=1e-12))
    assert res.converged and res.iterations == 1
    assert np.allclose(res.solution, rhs, atol=1e-14)
    rhs = np.arange(1.0, 6.0)
    res = vx.pcg(lambda v: 2.0 * v, None, rhs, rhs / 2.0, vx.PcgConfig(tol=1e-12))
    assert res.converged and res.iterations == 0


def test_pcg_matches_oracle_on_projected_neumann():
    from oracle import voxoracle as vo

    n = 32
    op = lambda v: 2 * v - np.roll(v, 1) - np.roll(v, -1)  # noqa: E731
    rhs = np.random.default_rng(1).standard_normal(n)
    res = vx.pcg(op, None, rhs, None, vx.PcgConfig(tol=1e-11, project_nullspace=True, max_iter=500))
    orc = vo.pcg(op, None, rhs, None, 1e-11, "preconditioned", 500, True)
    assert res.iterations == orc.iterations
    assert np.array_equal(res.solution, orc.solution)


def test_pcg_errors_and_lanczos():
    with pytest.raises(RuntimeError, match="not SPD"):
        vx.pcg(lambda v: np.array([1.0, -1.0, 2.0]) * v, None, np.array([0.0, 1.0, 0.0]), None,
               vx.PcgConfig(tol=1e-10))
    with pytest.raises(TypeError):
        vx.pcg(lambda v: v, None, np.ones(3), None, None)
    a = np.diag([1.0, 4.0])
    res = vx.pcg(lambda v: a @ v, None, np.array([1.0, 1.0]), None,
                 vx.PcgConfig(tol=1e-14, max_iter=2))
    lo, hi, cond = vx.lanczos_condition_estimate(res.alpha, res.beta)
    assert lo == pytest.approx(1.0, abs=1e-8) and hi == pytest.approx(4.0, abs=1e-8)
    with pytest.raises(ValueError, match="nonpositive"):
        vx.jacobi_prec(np.array([1.0, 0.0]))


# ---- seeded config generator (configs.py, native stamper) -----------------


def _stamp_numpy(n, dim, centers, radii, target, prism_axis=-1):
    """Plain restatement of the stamping rule: in order, every cell whose
    minimum-image distance (squared, summed axis by axis from 0.0, the prism
    axis skipped) to a ball centre is <= r^2 becomes solid, until the fluid
    count drops to ``target``."""
    fluid = np.ones((n,) * dim, dtype=bool)
    idx = np.indices(fluid.shape)
    nf = fluid.size
    used = 0
    for c, r in zip(centers, radii):
        if nf <= target:
            break
        d2 = np.zeros(fluid.shape)
        for a in range(dim):
            if a == prism_axis:
                continue
            dd = np.abs(idx[a].astype(float) - c[a])
            dd = np.minimum(dd, n - dd)
            d2 = d2 + dd * dd
        hit = (d2 <= r * r) & fluid
        fluid[hit] = False
        nf -= int(hit.sum())
        used += 1
    return fluid, used, nf


@pytest.mark.parametrize("dim,n,prism", [(3, 24, -1), (3, 20, 0), (2, 40, -1)])
def test_stamp_balls_matches_rule(dim, n, prism):
    from paper_2307_05266_b200 import configs

    rng = np.random.default_rng(3)
    c = rng.uniform(0, n, size=(60, dim))
    r = rng.uniform(1.5, 4.5, size=60)
    target = int(0.5 * n**dim)
    ref, used_ref, nf_ref = _stamp_numpy(n, dim, c, r, target, prism)
    fl = np.ones((n,) * dim, dtype=np.uint8)
    used, nf = configs._stamp(fl, c, r, target, prism)           # counts the mask itself
    assert (used, nf) == (used_ref, nf_ref) and np.array_equal(fl.astype(bool), ref)
    fl2 = np.ones((n,) * dim, dtype=np.uint8)
    half = 30
    u1, nf1 = configs._stamp(fl2, c[:half], r[:half], target, prism)  # batched, running count
    if nf1 > target:
        u2, nf1 = configs._stamp(fl2, c[half:], r[half:], target, prism, nf1)
    assert nf1 == nf_ref and np.array_equal(fl2.astype(bool), ref)
