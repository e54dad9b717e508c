"""Full Schur solves of the BASELINE configs on one GPU (C0-C4), one JSON
line per (config, preconditioner): outer/inner iteration counts, k, the
Lanczos condition estimate of the preconditioned S, time to tolerance, and
-- for the slit geometries -- the discrete known answer (a 1D
tridiagonal per slit, interior code 6 -> 2u - u+ - u-, wall code 7 ->
3u - u+).  C4 runs capped at a few outer iterations (time per outer
iteration reported, time-to-tol projected from the C2 outer count).

usage: python tools/config_report.py [keys...] [--cap-c4 N] > profiles/r01_configs.jsonl
"""
import json
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_05266_b200 as vx  # noqa: E402
from paper_2307_05266_b200 import configs  # noqa: E402

TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)


def slit_k(n: int, w: int, wall: int = 4) -> float:
    """k = (n_slits / n) * sum_j u_j with (n^2 T) u = 1 (codes 7 at the walls)."""
    T = np.zeros((w, w))
    for j in range(w):
        T[j, j] = 2.0
        if j > 0:
            T[j, j - 1] = -1.0
        if j < w - 1:
            T[j, j + 1] = -1.0
    T[0, 0] = T[-1, -1] = 3.0
    u = np.linalg.solve(n * n * T, np.ones(w))
    h = 1.0 / n
    nslits = n // (w + wall)
    # permeability = h^3 * sum over flow-direction faces of u = h^3 * n^2 * nslits * sum_j u_j
    return h ** 3 * n * n * nslits * float(u.sum())


def main():
    argv = sys.argv[1:]
    if "--cap-c4" in argv:  # drop the option and its value
        i = argv.index("--cap-c4")
        argv = argv[:i] + argv[i + 2:]
    args = [a for a in argv if not a.startswith("--")]
    cap = 3
    if "--cap-c4" in sys.argv:
        cap = int(sys.argv[sys.argv.index("--cap-c4") + 1])
    keys = args or ["C0", "C1", "C2", "C3s2", "C3s4", "C3s8", "C3s16", "C3s32", "C3c", "C4"]
    # clocks and throttle reasons sampled over the whole run (one record at the end)
    smi = None
    try:
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                                "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                                "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "500",
                                "-i", "0"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except OSError:
        pass
    try:
        run(keys, cap)
    finally:
        if smi is not None:
            smi.terminate()
            out = smi.communicate()[0].splitlines()
            sm = sorted(float(ln.split(",")[0]) for ln in out if ln.strip())
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = sorted({nm for ln in out for nm, v in zip(names, ln.split(",")[2:6]) if v.strip().startswith("Active")})
            print(json.dumps({"clocks": {"samples": len(sm), "sm_mhz_median": sm[len(sm) // 2] if sm else None,
                                         "sm_mhz_min": sm[0] if sm else None,
                                         "sm_max_mhz": float(out[0].split(",")[1]) if out else None,
                                         "reasons": reasons}}), flush=True)


def run(keys, cap):
    for key in keys:
        spec = configs.CONFIGS[key]
        t0 = time.perf_counter()
        grid = configs.make_geometry(key)
        t_gen = time.perf_counter() - t0
        t0 = time.perf_counter()
        s = vx.assemble(grid, 0, check_connectivity=spec.check_connectivity)
        t_asm = time.perf_counter() - t0
        precs = spec.precs if not key.startswith("C3") else ("uzawa", "simple")
        for prec in precs:
            max_iter = spec.max_iter
            if key == "C2" and prec == "uzawa":
                max_iter = 5000  # BASELINE configs[2]: Uzawa capped at 5000 outer iterations
            capped = key.startswith("C4") and cap < spec.max_iter
            if capped:
                max_iter = cap
            cfg = vx.SchurConfig(prec=prec, max_iter=max_iter, **TOL)
            rep = vx.solve_schur(s, cfg, return_fields=False)
            st = vx.last_kernel_stats(s)
            line = dict(config=key, name=spec.name, n=grid.n, porosity=float(grid.fluid.mean()),
                        m_u=s.m_u, m_p=s.m_p, prec=prec, max_iter=max_iter, capped=capped,
                        iters_outer=rep.iters_outer, converged=bool(rep.converged),
                        inner=rep.inner_iter_totals, k=rep.k_value,
                        cond_est_outer=rep.cond_est_outer, lambda_min_est=rep.lambda_min_est,
                        lambda_max_est=rep.lambda_max_est, device_ms=rep.device_ms,
                        wall_s=rep.wall_time, gen_s=t_gen, assemble_s=t_asm,
                        kernels={"A": st["velocity_cg"]["kernel"], "S_hat": st["simple_cg"]["kernel"]},
                        us_per_it={"A": 1e3 * st["velocity_cg"]["ms"] / max(1, st["velocity_cg"]["iterations"]),
                                   "S_hat": 1e3 * st["simple_cg"]["ms"] / max(1, st["simple_cg"]["iterations"])})
            if spec.kind == "slits":
                kk = slit_k(grid.n, spec.width)
                line["k_known"] = kk
                line["k_rel_err"] = abs(rep.k_value - kk) / kk
            if capped and rep.iters_outer:
                line["ms_per_outer"] = rep.device_ms / rep.iters_outer
            if rep.iters_outer == 0 and rep.cond_est_outer is None:
                # flow-aligned prisms: g == 0, the reference reports no estimate
                # (schur.py:359-362); the labelled supplement of SURVEY App. B-4
                try:
                    est = vx.supplementary_condition_estimate(s, cfg, seed=0)
                    line["supplementary"] = {k: est[k] for k in ("label", "seed", "iters_outer", "converged",
                                                                 "cond_est_outer", "lambda_min_est",
                                                                 "lambda_max_est", "inner_iter_totals", "device_ms")}
                except RuntimeError as e:
                    line["supplementary"] = {"error": str(e)}
            print(json.dumps(line), flush=True)
        del s


if __name__ == "__main__":
    main()
