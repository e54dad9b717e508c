"""Pin the BASELINE configs (C0-C4) to the REFERENCE package itself.

Run inside the build container (where /root/reference exists), one config
and preconditioner per process so the long ones can run side by side:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py C1 simple
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py C2 simple --max-iter 2
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_config_golden.py C4 simple --max-iter 1

It builds the seeded mask with the pure-numpy generator (oracle/stamper.py;
the product library is not loaded), runs the reference's own ``assemble``
and ``solve_schur`` (/root/reference/pkg/src/voxstokes/operators.py:209,
schur.py:291) unmodified, and writes ``tests/golden/cfg_<key>_<prec>[_capK].npz``.
The reference's module-level ``schur_rhs`` / ``_solve_velocity`` /
``_solve_simple`` are wrapped by observers that record g, u_f, the first
preconditioner solve and every inner iteration count as they happen; a
``..._partial.npz`` is rewritten after each stage so a run that is cut off
still leaves the stages it finished.

Small configs (C0, C1) store p and u in full; from 256^3 up a fixture keeps
norms, seeded projections and a fixed sample (vecsum.py).
"""
from __future__ import annotations

import argparse
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import voxstokes.schur as rs  # noqa: E402
from voxstokes.geometry import VoxelGrid  # noqa: E402
from voxstokes.operators import assemble  # noqa: E402

from oracle import stamper  # noqa: E402
import vecsum  # noqa: E402

TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("key")
    ap.add_argument("prec", choices=["uzawa", "simple"])
    ap.add_argument("--max-iter", type=int, default=None)
    ap.add_argument("--n", type=int, default=None, help="override the grid size (tests)")
    ap.add_argument("--nproj", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    warnings.simplefilter("ignore")

    spec = stamper.SPECS[args.key]
    n = spec[0] if args.n is None else args.n
    full = n ** spec[1] <= 64 ** 3
    nproj = args.nproj if args.nproj is not None else (64 if n <= 256 else 16)
    name = f"cfg_{args.key}" + (f"_n{n}" if args.n else "") + f"_{args.prec}"
    if args.max_iter is not None:
        name += f"_cap{args.max_iter}"
    out = os.path.join(HERE, name + ".npz")
    partial = os.path.join(HERE, name + "_partial.npz")

    t0 = time.perf_counter()
    fluid = stamper.make_fluid(args.key, args.seed, n)
    t_gen = time.perf_counter() - t0
    check_conn = spec[2] == "balls"
    t0 = time.perf_counter()
    sys_ = assemble(VoxelGrid(fluid), flow_dir=0, check_connectivity=check_conn)
    t_asm = time.perf_counter() - t0
    rec = dict(key=args.key, prec=args.prec, seed=args.seed, n=n, dim=fluid.ndim,
               digest=stamper.mask_digest(fluid), m_u=sys_.m_u, m_p=sys_.m_p,
               porosity=float(fluid.mean()), nproj=nproj,
               max_iter=-1 if args.max_iter is None else args.max_iter,
               gen_time=t_gen, assemble_time=t_asm, **TOL)
    print(name, "n", n, "m_u", sys_.m_u, "m_p", sys_.m_p, f"gen {t_gen:.1f}s asm {t_asm:.1f}s",
          flush=True)

    def flush_partial(stage):
        np.savez_compressed(partial, stage=stage, **rec)
        print(f"  [{time.perf_counter() - t_run:9.1f}s] {stage}", flush=True)

    # observers around the reference's own inner solves (the solver code is untouched)
    a_counts, s_counts, s_times, a_times = [], [], [], []
    orig_rhs, orig_vel, orig_simple = rs.schur_rhs, rs._solve_velocity, rs._solve_simple

    def obs_vel(sys, rhs, eps, x0=None):
        t = time.perf_counter()
        sol, its = orig_vel(sys, rhs, eps, x0)
        a_times.append(time.perf_counter() - t)
        a_counts.append(its)
        rec["inner_A_counts"] = np.array(a_counts)
        rec["inner_A_times"] = np.array(a_times)
        if n >= 256:
            flush_partial(f"A-solve #{len(a_counts)}: {its} its")
        return sol, its

    def obs_rhs(sys, eps_A):
        g, u_f = orig_rhs(sys, eps_A)
        vecsum.summarize("g", g, nproj, rec, full)
        vecsum.summarize("u_f", u_f, nproj, rec, full)
        flush_partial("schur_rhs")
        return g, u_f

    def obs_simple(sys, op, prec, r, eps):
        t = time.perf_counter()
        z, its = orig_simple(sys, op, prec, r, eps)
        s_times.append(time.perf_counter() - t)
        s_counts.append(its)
        rec["inner_S_counts"] = np.array(s_counts)
        rec["inner_S_times"] = np.array(s_times)
        if len(s_counts) == 1:
            # the first preconditioner solve: z0 = S_hat^-1 (0 - (g - mean g))
            vecsum.summarize("z0", z, nproj, rec, full)
        if n >= 256:
            flush_partial(f"S_hat-solve #{len(s_counts)}: {its} its")
        return z, its

    rs._solve_velocity, rs.schur_rhs, rs._solve_simple = obs_vel, obs_rhs, obs_simple
    kw = dict(TOL)
    if args.max_iter is not None:
        kw["max_iter"] = args.max_iter
    elif args.key == "C2" and args.prec == "uzawa":
        kw["max_iter"] = 5000
    t_run = time.perf_counter()
    rep = rs.solve_schur(sys_, rs.SchurConfig(prec=args.prec, **kw))
    rec["wall_time"] = rep.wall_time
    rec["k_value"] = rep.k_value
    rec["iters_outer"] = rep.iters_outer
    rec["converged"] = rep.converged
    rec["res_prec"] = np.asarray(rep.res_prec)
    rec["res_unprec"] = np.asarray(rep.res_unprec)
    rec["perm_history"] = np.asarray(rep.perm_history)
    rec["inner_velocity"] = rep.inner_iter_totals["velocity"]
    rec["inner_preconditioner"] = rep.inner_iter_totals["preconditioner"]
    nan = float("nan")
    rec["cond"] = nan if rep.cond_est_outer is None else rep.cond_est_outer
    rec["lmin"] = nan if rep.lambda_min_est is None else rep.lambda_min_est
    rec["lmax"] = nan if rep.lambda_max_est is None else rep.lambda_max_est
    vecsum.summarize("p", rep.pressure, nproj, rec, full)
    vecsum.summarize("u", rep.velocity, nproj, rec, full)
    np.savez_compressed(out, **rec)
    if os.path.exists(partial):
        os.remove(partial)
    print(name, "done: outer", rep.iters_outer, "converged", rep.converged, "k", rep.k_value,
          "inner", rep.inner_iter_totals, f"wall {rep.wall_time:.1f}s", flush=True)


if __name__ == "__main__":
    main()
