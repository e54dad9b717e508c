"""Generate golden fixtures by running the REFERENCE package itself.

Run inside the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports ``voxstokes`` from /root/reference/pkg/src, builds a handful of
small seeded geometries, and records the reference's own outputs
(geometry, operator applies on seeded vectors, full Schur solves) into
``tests/golden/*.npz``.  The fixtures travel with the repo; the reference
does not.  Nothing under tests/ reads /root/reference at run time.
"""
from __future__ import annotations

import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from voxstokes.geometry import (  # noqa: E402
    PackingParams, VoxelGrid, connected_components, enforce_connectivity,
    generate_packing,
)
from voxstokes.operators import assemble  # noqa: E402
from voxstokes.schur import (  # noqa: E402
    SchurConfig, apply_simple_inverse, profile_config, schur_rhs, solve_schur,
)

BASE_TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)


def balls(n, dim, count, rmin, rmax, seed):
    """Small seeded disk/sphere packing (solid = union of periodic balls)."""
    rng = np.random.default_rng(seed)
    solid = np.zeros((n,) * dim, dtype=bool)
    grids = np.meshgrid(*[np.arange(n)] * dim, indexing="ij")
    for _ in range(count):
        c = rng.uniform(0, n, size=dim)
        r = rng.uniform(rmin, rmax)
        d2 = np.zeros(solid.shape)
        for ax in range(dim):
            dd = np.abs(grids[ax] - c[ax])
            dd = np.minimum(dd, n - dd)
            d2 += dd * dd
        solid |= d2 <= r * r
    grid, _ = enforce_connectivity(VoxelGrid(~solid))
    return grid.fluid


def cases():
    out = {}
    out["pack2d"] = (generate_packing(
        PackingParams(N=2, n_c=10, n_avg=4, n_min=2, seed=11)).fluid, 0)
    out["pack3d"] = (generate_packing(
        PackingParams(N=1, n_c=6, n_avg=2, n_min=2, seed=0, dim=3)).fluid, 2)
    rng = np.random.default_rng(5)
    f = rng.random((14, 14, 14)) < 0.62
    out["rand3d"] = (enforce_connectivity(VoxelGrid(f))[0].fluid, 0)
    out["wrap2"] = (np.array([[True, True], [True, False]]), 0)
    ch = np.zeros((16, 16), dtype=bool)
    ch[:, 4:12] = True
    out["channel16"] = (ch, 0)
    out["disks2d"] = (balls(40, 2, 6, 4, 7, seed=3), 0)
    out["spheres3d"] = (balls(20, 3, 12, 2, 4, seed=4), 0)
    out["exhaust"] = (generate_packing(
        PackingParams(N=1, n_c=10, n_avg=4, n_min=2, seed=1)).fluid, 0)
    return out


def solve_record(prefix, rep, rec):
    rec[prefix + "pressure"] = rep.pressure
    rec[prefix + "velocity"] = rep.velocity
    rec[prefix + "k_value"] = rep.k_value
    rec[prefix + "iters_outer"] = rep.iters_outer
    rec[prefix + "converged"] = rep.converged
    rec[prefix + "res_prec"] = rep.res_prec
    rec[prefix + "res_unprec"] = rep.res_unprec
    rec[prefix + "perm_history"] = rep.perm_history
    rec[prefix + "inner_velocity"] = rep.inner_iter_totals["velocity"]
    rec[prefix + "inner_preconditioner"] = rep.inner_iter_totals["preconditioner"]
    nan = float("nan")
    rec[prefix + "cond"] = nan if rep.cond_est_outer is None else rep.cond_est_outer
    rec[prefix + "lmin"] = nan if rep.lambda_min_est is None else rep.lambda_min_est
    rec[prefix + "lmax"] = nan if rep.lambda_max_est is None else rep.lambda_max_est


def main():
    warnings.simplefilter("ignore")
    for name, (fluid, flow) in cases().items():
        grid = VoxelGrid(fluid)
        sys_ = assemble(grid, flow_dir=flow)
        dm = sys_.dof_map
        rec = dict(
            fluid=fluid, flow_dir=flow, m_u=dm.m_u, m_p=dm.m_p,
            axis_counts=np.array(dm.axis_counts), axis_offsets=np.array(dm.axis_offsets),
            diag=sys_.laplacian_diag, force=sys_.force,
        )
        for a in range(grid.dim):
            rec[f"face_mask{a}"] = dm.face_ids[a] >= 0
        rec["pressure_mask"] = dm.pressure_ids >= 0
        rng = np.random.default_rng(123)
        u = rng.standard_normal(dm.m_u)
        p = rng.standard_normal(dm.m_p)
        rec["u_in"], rec["p_in"] = u, p
        rec["Au"] = sys_.apply_laplacian(u)
        rec["Bu"] = sys_.apply_divergence(u)
        rec["Btp"] = sys_.apply_gradient(p)
        inv = 1.0 / sys_.laplacian_diag
        rec["Sp"] = sys_.apply_divergence(sys_.apply_gradient(p) * inv)
        rec["dwd"] = sys_.divergence_weighted_diagonal(inv)
        # inner solves through the reference seams
        g, uf = schur_rhs(sys_, 1e-12)
        rec["g"], rec["u_f"] = g, uf
        if name != "channel16":
            pz = p - p.mean()
            rec["simple_inv"] = apply_simple_inverse(sys_, pz, 1e-12)
        if name == "exhaust":
            cfg = SchurConfig(prec="uzawa", eps_S=1e-9, outer_norm="unpreconditioned",
                              eps_A=1e-13, eps_Shat=1e-13, max_iter=2)
            solve_record("exh_", solve_schur(sys_, cfg), rec)
        else:
            for prec in ("uzawa", "simple"):
                rep = solve_schur(sys_, SchurConfig(prec=prec, **BASE_TOL))
                solve_record(f"{prec}_", rep, rec)
            if name == "pack2d":
                for prec in ("uzawa", "simple"):
                    rep = solve_schur(sys_, profile_config("paper2d", prec))
                    solve_record(f"p2d_{prec}_", rep, rec)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
        print(name, dm.m_u, dm.m_p, {k: v for k, v in rec.items()
                                      if k.endswith("iters_outer")})

    # connectivity labelling fixtures (geometry.py:183-240)
    rng = np.random.default_rng(9)
    lab = {}
    for i, shape in enumerate([(24, 24), (12, 12, 12), (9, 9, 9)]):
        f = rng.random(shape) < 0.45
        labels, ncomp = connected_components(VoxelGrid(f))
        kept, removed = enforce_connectivity(VoxelGrid(f))
        lab[f"fluid{i}"] = f
        lab[f"labels{i}"] = labels
        lab[f"ncomp{i}"] = ncomp
        lab[f"kept{i}"] = kept.fluid
        lab[f"removed{i}"] = removed
    np.savez_compressed(os.path.join(HERE, "components.npz"), **lab)


if __name__ == "__main__":
    main()
