"""Same-process A/B of kernel variants on one config's inner solves: the mask
is generated once, then every variant (environment settings read when the
context is built) assembles its own system and runs one inner A-solve and one
inner S_hat-solve to 1e-12 through the C ABI.  Two alternating rounds.

usage: python tools/ab_variants.py C4 "base:" "mq:VOXSCHUR_CG=4" "rc512:VOXSCHUR_CG=5,VOXSCHUR_M_THREADS=512"
       [--phases] [--ops SA] [--rounds 2]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
args = [a for a in sys.argv[1:] if not a.startswith("--")]
phases = "--phases" in sys.argv
ops = sys.argv[sys.argv.index("--ops") + 1] if "--ops" in sys.argv else "SA"
rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 2
args = [a for a in args if a not in (ops, str(rounds))] if ("--ops" in sys.argv or "--rounds" in sys.argv) else args
if phases:
    os.environ["VOXSCHUR_PHASE_TIMING"] = "1"
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import _lib, configs, schur  # noqa: E402

key, variants = args[0], args[1:]
t0 = time.time()
grid = configs.make_geometry(key, device=0 if configs.CONFIGS[key].n >= 256 else None)
print(f"{key}: n={grid.n} generated in {time.time() - t0:.1f} s", flush=True)
rng = np.random.default_rng(1)
ref = {}
for rnd in range(rounds):
    for spec in variants:
        label, _, envs = spec.partition(":")
        sets = dict(kv.split("=", 1) for kv in envs.split(",") if kv)
        old = {k: os.environ.get(k) for k in sets}
        os.environ.update(sets)
        try:
            s = vx.assemble(grid, 0, check_connectivity=configs.CONFIGS[key].check_connectivity)
            if rnd == 0 and spec == variants[0]:
                print(f"m_u={s.m_u} m_p={s.m_p}", flush=True)
            p = np.random.default_rng(1).standard_normal(s.m_p)
            p -= p.mean()
            ph = np.zeros(12)
            if "S" in ops:
                try:
                    z = vx.apply_simple_inverse(s, p, 1e-12)
                except RuntimeError as e:  # capped by VOXSCHUR_INNER_MAXIT: the timing still stands
                    z = np.zeros(s.m_p)
                st = vx.last_kernel_stats(s)["simple_cg"]
                its = st["iterations"]
                extra = ""
                if phases:
                    _lib.lib.vs_phase_timing(s._ctx, ph)
                    extra = f" phases us/it max-block {np.round(ph[4:8] / its / 1e3, 1)}"
                zn = float(np.linalg.norm(z))
                dev = ""
                if "S" in ref:
                    dev = f" |z-z0|/|z0| {np.linalg.norm(z - ref['S']) / np.linalg.norm(ref['S']):.1e}"
                else:
                    ref["S"] = z
                print(f"[{rnd}] {label:14s} S-solve [{st['kernel']} t{st['tier']} esc {st['escape_ppm']}ppm]: {its} its, "
                      f"{1e3 * st['ms'] / its:8.2f} us/it, {64 * st['dof_iters'] / st['ms'] / 1e6:7.1f} GB/s alg, "
                      f"|z| {zn:.12e}{dev}{extra}", flush=True)
            if "A" in ops:
                rhs_u = s.apply_gradient(p)
                try:
                    x, its = schur._solve_velocity(s, rhs_u, 1e-12)
                except RuntimeError as e:
                    x, its = np.zeros(s.m_u), 0
                st = vx.last_kernel_stats(s)["velocity_cg"]
                its = st["iterations"]
                extra = ""
                if phases:
                    _lib.lib.vs_phase_timing(s._ctx, ph)
                    extra = f" phases us/it max-block {np.round(ph[4:8] / its / 1e3, 1)}"
                dev = ""
                if "A" in ref:
                    dev = f" |x-x0|/|x0| {np.linalg.norm(x - ref['A']) / np.linalg.norm(ref['A']):.1e}"
                else:
                    ref["A"] = x
                print(f"[{rnd}] {label:14s} A-solve [{st['kernel']} t{st['tier']} esc {st['escape_ppm']}ppm]: {its} its, "
                      f"{1e3 * st['ms'] / its:8.2f} us/it, {64 * st['dof_iters'] / st['ms'] / 1e6:7.1f} GB/s alg"
                      f"{dev}{extra}", flush=True)
            del s
        except Exception as e:  # keep going: the other variants still measure
            print(f"[{rnd}] {label}: FAILED {type(e).__name__}: {e}", flush=True)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
