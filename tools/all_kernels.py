"""Touch every kernel of the path once at a config's size (an ncu target):
assemble (geometry build, connected components), the five single applies,
and one capped solve_schur (fused CG + outer-loop kernels).
usage: VOXSCHUR_INNER_MAXIT=40 python tools/all_kernels.py C4"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
grid = configs.make_geometry(key, device=0)
s = vx.assemble(grid, 0, check_connectivity=configs.CONFIGS[key].check_connectivity)
rng = np.random.default_rng(0)
u, p = rng.standard_normal(s.m_u), rng.standard_normal(s.m_p)
s.apply_laplacian(u)
s.apply_divergence(u)
s.apply_gradient(p)
s.apply_simple(p)
s.divergence_weighted_diagonal(1.0 / s.laplacian_diag)
try:
    vx.solve_schur(s, vx.SchurConfig(prec="simple", eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12, max_iter=1),
                   return_fields=False)
except RuntimeError as e:  # capped inner solves end in the reference's error: the kernels still ran
    print("capped:", e)
print("done", s.m_u, s.m_p)
