"""Split a full solve_schur's device time into fused-CG kernel time and
outer-loop overhead (C1 by default).  usage: python tools/outer_overhead.py [C1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
grid = configs.make_geometry(key)
s = vx.assemble(grid, 0)
for prec in ("uzawa", "simple"):
    for _ in range(2):
        t0 = time.perf_counter()
        rep = vx.solve_schur(s, vx.SchurConfig(prec=prec, eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12),
                             return_fields=False)
        wall = (time.perf_counter() - t0) * 1e3
    st = vx.last_kernel_stats(s)
    cg = st["velocity_cg"]["ms"] + st["simple_cg"]["ms"]
    print(f"{prec}: outer {rep.iters_outer}, device {rep.device_ms:.1f} ms, wall {wall:.1f} ms, "
          f"cg kernels {cg:.1f} ms ({st['velocity_cg']['launches']} A + {st['simple_cg']['launches']} S "
          f"launches, {st['velocity_cg']['iterations']} + {st['simple_cg']['iterations']} its), "
          f"outer overhead {rep.device_ms - cg:.1f} ms = "
          f"{(rep.device_ms - cg) / max(1, rep.iters_outer) * 1e3:.0f} us/outer it, "
          f"launches {st['kernel_launches']}")
