"""Connected-component labelling host vs GPU, and assemble time, on the big
configs.  usage: python tools/cc_probe.py [C4 [C4L]]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

for key in sys.argv[1:] or ["C4"]:
    spec = configs.CONFIGS[key]
    t0 = time.perf_counter()
    fluid = configs.balls(spec.n, spec.dim, spec.rmin, spec.rmax, porosity=spec.porosity, seed=0)
    t1 = time.perf_counter()
    grid = vx.VoxelGrid(fluid)
    t2 = time.perf_counter()
    kept_d, rm_d = vx.enforce_connectivity(grid, device=0)
    t3 = time.perf_counter()
    line = f"{key} n={spec.n}: stamp {t1 - t0:.1f}s  enforce_connectivity GPU {t3 - t2:.2f}s (removed {rm_d})"
    if spec.n <= 512:
        kept_h, rm_h = vx.enforce_connectivity(grid)
        t4 = time.perf_counter()
        line += f"  host {t4 - t3:.2f}s  same={np.array_equal(kept_h.fluid, kept_d.fluid) and rm_h == rm_d}"
    print(line, flush=True)
    del fluid, grid
    t5 = time.perf_counter()
    s = vx.assemble(kept_d, 0)
    t6 = time.perf_counter()
    print(f"   assemble (device connectivity check + geometry build): {t6 - t5:.2f}s  m_u={s.m_u} m_p={s.m_p}",
          flush=True)
    del s
