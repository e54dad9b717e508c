"""Inner solves of a config on R emulated ranks of one GPU (slab groups of one cooperative launch,
per-rank partial buffers: VOXSCHUR_EMULATE_RANKS=1), with the hierarchical and the flat barrier.
usage: python tools/slab_emulate_probe.py C2 4"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["VOXSCHUR_EMULATE_RANKS"] = "1"
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C2"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 4
grid = configs.make_geometry(key, device=0 if configs.CONFIGS[key].n >= 256 else None)
p = np.random.default_rng(1).standard_normal(int(grid.fluid.sum()))
p -= p.mean()
ref = None
for hier in ("1", "0", "1", "0"):
    os.environ["VOXSCHUR_HIER_BARRIER"] = hier
    s = vx.assemble(grid, 0, slabs=R)
    z = vx.apply_simple_inverse(s, p, 1e-12)
    st = vx.last_kernel_stats(s)["simple_cg"]
    same = "" if ref is None else f" bitwise same as the first run: {np.array_equal(z, ref)}"
    ref = z if ref is None else ref
    print(f"{key} R={R} hier={hier}: [{st['kernel']}] {st['iterations']} its, {1e3 * st['ms'] / st['iterations']:.2f} us/it{same}", flush=True)
    del s
