"""Where the e2e step's time goes beyond the device span: assemble,
first solve on a fresh system, D2H.  usage: python tools/e2e_probe.py [C1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs, schur  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C1"
TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)
grid = configs.make_geometry(key)
cfgs = [vx.SchurConfig(prec="uzawa", **TOL), vx.SchurConfig(prec="simple", **TOL)]
from paper_2307_05266_b200 import geometry  # noqa: E402
t0 = time.perf_counter()
for _ in range(5):
    geometry.connected_components(grid)
print(f"host connectivity labelling: {1e3 * (time.perf_counter() - t0) / 5:.1f} ms", flush=True)
for _ in range(3):
    t0 = time.perf_counter()
    s0 = vx.assemble(grid, 0, check_connectivity=False)
    t1 = time.perf_counter()
    del s0
    print(f"assemble without connectivity {1e3 * (t1 - t0):.1f} ms, destroy {1e3 * (time.perf_counter() - t1):.1f} ms")
for rnd in range(3):
    t0 = time.perf_counter()
    sy = [vx.assemble(grid, 0) for _ in cfgs]
    t1 = time.perf_counter()
    reps = schur.solve_schur_concurrent(list(zip(sy, cfgs)), weights=[188, 395], return_fields=True)
    t2 = time.perf_counter()
    span = schur.concurrent_span_ms(sy)
    reps2 = schur.solve_schur_concurrent(list(zip(sy, cfgs)), weights=[188, 395], return_fields=True)
    t3 = time.perf_counter()
    span2 = schur.concurrent_span_ms(sy)
    t4 = time.perf_counter()
    del sy
    t5 = time.perf_counter()
    print(f"assemble x2 {1e3*(t1-t0):.1f} ms; fresh solve wall {1e3*(t2-t1):.1f} (span {span:.1f}, "
          f"wall-per-solve {[round(r.wall_time*1e3,1) for r in reps]}); second solve wall {1e3*(t3-t2):.1f} "
          f"(span {span2:.1f}); destroy {1e3*(t5-t4):.1f}", flush=True)
