"""Where the C4 e2e step's wall time goes beyond the device span: assemble (connectivity check,
H2D of the mask, geometry build), the first solve's one-off table builds, D2H of p and u.
usage: python tools/e2e_c4_probe.py [C4]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C4"
grid = configs.make_geometry(key, device=0)
cfg = vx.SchurConfig(prec="simple", eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12, max_iter=1)
for rnd in range(3):
    t0 = time.perf_counter()
    s = vx.assemble(grid, 0)
    t1 = time.perf_counter()
    rep = vx.solve_schur(s, cfg)
    t2 = time.perf_counter()
    st = vx.last_kernel_stats(s)
    dev = st["velocity_cg"]["ms"] + st["simple_cg"]["ms"]
    rep2 = vx.solve_schur(s, cfg)
    t3 = time.perf_counter()
    del s
    t4 = time.perf_counter()
    print(f"[{rnd}] assemble {1e3 * (t1 - t0):.0f} ms; first solve wall {1e3 * (t2 - t1):.0f} ms (fused-CG kernels {dev:.0f} ms, "
          f"report wall_time {1e3 * rep.wall_time:.0f}); second solve wall {1e3 * (t3 - t2):.0f} ms; destroy {1e3 * (t4 - t3):.0f} ms",
          flush=True)
