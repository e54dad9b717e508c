"""Per-iteration rates of the fused inner solves at a large config (one GPU).

usage: python tools/scale_probe.py C4 [slabs]
Builds the seeded geometry, assembles on the GPU, times one inner A-solve
(rhs = grad of a seeded zero-mean p) and one inner S_hat-solve capped by the
reference's tolerance 1e-12 (the S_hat solve is long at 512^3, so it is run
once), and prints algorithmic GB/s (64 B per DOF per CG iteration).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("VOXSCHUR_PHASE_TIMING", "1")
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import _lib, configs, schur  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
slabs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
eps_s = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-12
t0 = time.perf_counter()
grid = configs.make_geometry(key)
t_gen = time.perf_counter() - t0
t0 = time.perf_counter()
s = vx.assemble(grid, 0, check_connectivity=configs.CONFIGS[key].check_connectivity, slabs=slabs)
t_asm = time.perf_counter() - t0
out = dict(config=key, n=grid.n, porosity=float(grid.fluid.mean()), m_u=s.m_u, m_p=s.m_p, slabs=slabs,
           gen_s=t_gen, assemble_s=t_asm)
rng = np.random.default_rng(1)
p = rng.standard_normal(s.m_p)
p -= p.mean()
rhs = s.apply_gradient(p)
ph = np.zeros(12)
for rep in range(2):
    _, its = schur._solve_velocity(s, rhs, 1e-12)
    st = vx.last_kernel_stats(s)["velocity_cg"]
    _lib.lib.vs_phase_timing(s._ctx, ph)
out["A"] = dict(iterations=its, ms=st["ms"], us_per_it=1e3 * st["ms"] / its,
                alg_GBps=64 * st["dof_iters"] / st["ms"] / 1e6,
                phases_us_block0=list(np.round(ph[:4] / its / 1e3, 2)),
                phases_us_maxblock=list(np.round(ph[4:8] / its / 1e3, 2)))
z = vx.apply_simple_inverse(s, p, eps_s)
st = vx.last_kernel_stats(s)["simple_cg"]
_lib.lib.vs_phase_timing(s._ctx, ph)
its = st["iterations"]
out["S"] = dict(iterations=its, eps=eps_s, ms=st["ms"], us_per_it=1e3 * st["ms"] / its,
                alg_GBps=64 * st["dof_iters"] / st["ms"] / 1e6,
                phases_us_block0=list(np.round(ph[:4] / its / 1e3, 2)),
                phases_us_maxblock=list(np.round(ph[4:8] / its / 1e3, 2)))
print(json.dumps(out))
