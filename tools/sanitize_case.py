"""Small end-to-end case for compute-sanitizer: applies, inner solves and a
SIMPLE + Uzawa solve_schur on a 3D golden geometry, single and 2-slab."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2307_05266_b200 as vx  # noqa: E402

with np.load(os.path.join(ROOT, "tests", "golden", "rand3d.npz")) as z:
    fluid = z["fluid"]
for slabs in (1, 2):
    s = vx.assemble(vx.VoxelGrid(fluid), 0, slabs=slabs)
    u = np.random.default_rng(0).standard_normal(s.m_u)
    p = np.random.default_rng(1).standard_normal(s.m_p)
    s.apply_laplacian(u), s.apply_divergence(u), s.apply_gradient(p), s.apply_simple(p)
    for prec in ("uzawa", "simple"):
        rep = vx.solve_schur(s, vx.SchurConfig(prec=prec, eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12))
        print(slabs, prec, rep.iters_outer, rep.k_value)
