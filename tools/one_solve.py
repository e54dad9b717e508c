"""Run one inner S_hat solve (and one A solve) of a config at a given
tolerance through the C ABI -- a short target for ncu captures.
usage: python tools/one_solve.py C2 [eps] [S|A|SA]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs, schur  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C2"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
which = sys.argv[3] if len(sys.argv) > 3 else "SA"
grid = configs.make_geometry(key)
s = vx.assemble(grid, 0, check_connectivity=configs.CONFIGS[key].check_connectivity)
rng = np.random.default_rng(1)
p = rng.standard_normal(s.m_p)
p -= p.mean()
def guarded(fn):
    """With VOXSCHUR_INNER_MAXIT set the capped solve ends in the reference's
    'did not converge' error: the launch still ran (what an ncu capture needs)."""
    try:
        return fn()
    except RuntimeError as e:
        print("capped:", e, flush=True)
        return None, 0


if "S" in which:
    guarded(lambda: (vx.apply_simple_inverse(s, p, eps), 0))
    st = vx.last_kernel_stats(s)["simple_cg"]
    print(f"S: {st['iterations']} its, {1e3 * st['ms'] / max(1, st['iterations']):.2f} us/it", flush=True)
if "A" in which:
    guarded(lambda: schur._solve_velocity(s, s.apply_gradient(p), eps))
    st = vx.last_kernel_stats(s)["velocity_cg"]
    its = st["iterations"]
    print(f"A: {its} its, {1e3 * st['ms'] / max(1, its):.2f} us/it", flush=True)
