"""C1 Uzawa + SIMPLE: sequential on the whole device vs concurrent on SM
shares (solve_schur_concurrent).  usage: python tools/concurrent_probe.py [C1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs, schur  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)
grid = configs.make_geometry(key)
su = vx.assemble(grid, 0)
ss = vx.assemble(grid, 0)
cu = vx.SchurConfig(prec="uzawa", **TOL)
cs = vx.SchurConfig(prec="simple", **TOL)
for rnd in range(2):
    su.limit_sms(0); ss.limit_sms(0)
    ru = vx.solve_schur(su, cu, return_fields=False)
    rs = vx.solve_schur(ss, cs, return_fields=False)
    print(f"seq full: uzawa {ru.device_ms:.1f} ms simple {rs.device_ms:.1f} ms total {ru.device_ms + rs.device_ms:.1f}"
          f"  k {ru.k_value:.12e} {rs.k_value:.12e} its {ru.iters_outer},{rs.iters_outer} "
          f"{ru.inner_iter_totals} {rs.inner_iter_totals}", flush=True)
    for ws in (0.5, 0.6, 0.65, 0.7, 0.75, 0.8):
        t0 = time.perf_counter()
        ru, rs = schur.solve_schur_concurrent([(su, cu), (ss, cs)], weights=[1 - ws, ws], return_fields=False)
        wall = 1e3 * (time.perf_counter() - t0)
        span = schur.concurrent_span_ms([su, ss])
        print(f"conc w_S={ws:.2f} sms {su.sms}/{ss.sms}: span {span:.1f} ms (wall {wall:.1f}) uzawa {ru.device_ms:.1f} "
              f"simple {rs.device_ms:.1f} k {ru.k_value:.12e} {rs.k_value:.12e} its {ru.iters_outer},{rs.iters_outer} "
              f"{ru.inner_iter_totals} {rs.inner_iter_totals}", flush=True)
