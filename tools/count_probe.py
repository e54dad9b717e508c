"""Inner/outer iteration counts of the golden full solves under several fused-CG kernels
(VOXSCHUR_CG / VOXSCHUR_X_DEPTH), next to the reference's.  usage: python tools/count_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
variants = sys.argv[1:] or ["1", "4", "7/1", "7/2"]
for name in ["pack2d", "pack3d", "rand3d", "disks2d", "spheres3d"]:
    g = dict(np.load(os.path.join(G, name + ".npz")))
    for prec in ["uzawa", "simple"]:
        pre = prec + "_"
        row = [f"{name:10s} {prec:6s} ref {int(g[pre + 'iters_outer'])}/{int(g[pre + 'inner_velocity'])}/{int(g[pre + 'inner_preconditioner'])}"]
        for v in variants:
            cg, _, depth = v.partition("/")
            os.environ["VOXSCHUR_CG"] = cg
            if depth:
                os.environ["VOXSCHUR_X_DEPTH"] = depth
            s = vx.assemble(vx.VoxelGrid(g["fluid"]), int(g["flow_dir"]), device=0)
            try:
                rep = vx.solve_schur(s, vx.SchurConfig(prec=prec, eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12))
            except RuntimeError as e:
                row.append(f"[{v}] FAILED {e}")
                continue
            dk = abs(rep.k_value - float(g[pre + "k_value"])) / abs(float(g[pre + "k_value"]))
            row.append(f"[{v}] {rep.iters_outer}/{rep.inner_iter_totals['velocity']}/{rep.inner_iter_totals['preconditioner']} dk {dk:.0e}")
        print("  ".join(row), flush=True)
