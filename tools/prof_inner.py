"""Time (and, under ncu, profile) one inner A-solve and one inner S_hat-solve
of a config through the C ABI.  usage: python tools/prof_inner.py C1 [reps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--no-phases" not in sys.argv:
    os.environ.setdefault("VOXSCHUR_PHASE_TIMING", "1")
sys.argv = [a for a in sys.argv if a != "--no-phases"]
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import _lib  # noqa: E402
from paper_2307_05266_b200 import configs, schur  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
grid = configs.make_geometry(key)
s = vx.assemble(grid, 0, check_connectivity=configs.CONFIGS[key].check_connectivity)
print(f"{key}: n={grid.n} m_u={s.m_u} m_p={s.m_p}", flush=True)
rng = np.random.default_rng(1)
p = rng.standard_normal(s.m_p)
p -= p.mean()
rhs_u = s.apply_gradient(p)
for _ in range(reps):
    x, its = schur._solve_velocity(s, rhs_u, 1e-12)
    st = vx.last_kernel_stats(s)["velocity_cg"]
    ph = np.zeros(12)
    _lib.lib.vs_phase_timing(s._ctx, ph)
    grid = {"A": None}
    print("   phases us/it (P1, sum1, P2, sum2) block0:", np.round(ph[:4] / its / 1e3, 2),
          "max-block:", np.round(ph[4:8] / its / 1e3, 2), "mean-block:", np.round(ph[8:12] / its / 1e3 / 148, 2))
    print(f"A-solve [{st['kernel']} u{st['p1_unroll']}]: {its} its, {st['ms']:.3f} ms, {1e3 * st['ms'] / its:.2f} us/it, "
          f"{64 * st['dof_iters'] / st['ms'] / 1e6:.1f} GB/s alg", flush=True)
    z = vx.apply_simple_inverse(s, p, 1e-12)
    st = vx.last_kernel_stats(s)["simple_cg"]
    its = st["iterations"]
    _lib.lib.vs_phase_timing(s._ctx, ph)
    print("   phases us/it (P1, sum1, P2, sum2) block0:", np.round(ph[:4] / its / 1e3, 2),
          "max-block:", np.round(ph[4:8] / its / 1e3, 2), "mean-block:", np.round(ph[8:12] / its / 1e3 / 148, 2))
    print(f"S-solve [{st['kernel']} u{st['p1_unroll']}]: {its} its, {st['ms']:.3f} ms, {1e3 * st['ms'] / its:.2f} us/it, "
          f"{64 * st['dof_iters'] / st['ms'] / 1e6:.1f} GB/s alg", flush=True)
