#!/usr/bin/env python
"""Benchmark of the Schur-complement Stokes path (BASELINE.json metric).

Workload (N=1): BASELINE configs[1] -- 64^3 periodic sphere packing
(radii U[4,8], porosity 0.4, x-percolating component), f=(1,0,0), solved
once with Uzawa and once with SIMPLE at eps_S=1e-8, eps_A=eps_Shat=1e-12
(SURVEY Appendix B).  One "step" = those two full Schur solves to tolerance,
run concurrently on one GPU, each on its own system and share of the SMs
(solve_schur_concurrent; the split is tuned in untimed warm-up steps, see
"sm_split_tuning_ms"; --sequential runs them one after another).

* value     -- masked-stencil Gcell/s = n^3 * (I_A + I_S) / t_device, I_A
               counting every inner A-iteration (incl. the u_f solve),
               I_S every inner S_hat-iteration; t_device = CUDA-event time
               span of the step's solves (first start to last end) with
               the geometry resident in HBM.
* e2e       -- same metric through the public API with host buffers:
               assemble(host mask) (H2D + device geometry build) and
               solve_schur returning p, u (D2H) inside the timed region.
* roofline  -- dominant kernel (fused persistent PCG): algorithmic bytes
               64 B per DOF per CG iteration x DOF-iterations
               / summed CUDA-event launch time, vs MEASURED_PEAKS hbm_gbs.
* cpu_baseline / --impl reference -- the CPU oracle port (oracle/, the
               reference algorithm restated in numpy) on the host cores.

Multi-GPU (torchrun): replicas only for now -- each rank solves its own
copy (no data-path collective); value sums the ranks' work over the max
device time ("scaling": "weak").
"""
from __future__ import annotations

import os

# the CPU legs are single-threaded numpy by design (multi-threaded
# OpenBLAS under contention is ~28x slower); pin before numpy is imported, so
# spawned worker processes inherit it too
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import json
import math
import multiprocessing as mp
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)
BYTES_PER_DOF_ITER = 64  # x, r, d read+write, r and d re-read
METRIC = "masked-stencil Gcell/s & HBM GB/s (vs 8 TB/s); Schur solve time-to-tol at 1-8 GPU"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.dev)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------- CPU oracle leg
def _oracle_sample(args):
    """One bounded sample of the workload on the CPU oracle: a SIMPLE
    solve_schur capped at one outer iteration (u_f solve, initial S_hat
    solve, one outer step = A-solve + S_hat-solve, refresh)."""
    key, seed = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, ROOT)
    from oracle import voxoracle as vo
    from paper_2307_05266_b200 import configs

    grid = configs.make_geometry(key, seed)
    s = vo.build_system(grid.fluid, 0)
    t0 = time.perf_counter()
    rep = vo.solve_schur(s, "simple", max_iter=1, **TOL)
    dt = time.perf_counter() - t0
    ia = rep["inner_iter_totals"]["velocity"] + rep["uf_iters"]
    isx = rep["inner_iter_totals"]["preconditioner"]
    # the initial preconditioner solve is inside solve_schur too
    return dict(cells_iters=grid.fluid.size * (ia + isx), seconds=dt, I_A=ia, I_S=isx)


def cpu_sample(key, seed, procs):
    if procs <= 1:
        res = [_oracle_sample((key, seed))]
    else:
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            res = pool.map(_oracle_sample, [(key, seed)] * procs)
    tmax = max(r["seconds"] for r in res)
    tot = sum(r["cells_iters"] for r in res)
    return tot / tmax / 1e9, res


def usable_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------ reference arm
def run_reference(a):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    cores = usable_cores()
    vals, secs = [], []
    for i in range(a.warmup + a.steps):
        v, res = cpu_sample(a.config, a.seed, cores)
        if i >= a.warmup:
            vals.append(v)
            secs.append(max(r["seconds"] for r in res))
    val = statistics.median(vals)
    spec = __import__("paper_2307_05266_b200.configs", fromlist=["CONFIGS"]).CONFIGS[a.config]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Gcell/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": spec.name, "seed": a.seed, "precs": list(spec.precs)},
        "cpu_baseline": {"value": val, "unit": "Gcell/s", "cores": cores, "kind": "port",
                         "sample": "per process: oracle SIMPLE solve_schur capped at 1 outer "
                                   "iteration on the same geometry; one process per core"},
        "e2e": {"value": val, "unit": "Gcell/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def run_ours(a):
    rank, local, world = env_rank()
    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        torch.cuda.set_device(local)
        dist_mod.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist = dist_mod
    dev = local
    torch.cuda.set_device(dev)
    import paper_2307_05266_b200 as vx
    from paper_2307_05266_b200 import configs

    spec = configs.CONFIGS[a.config]
    grid = configs.make_geometry(a.config, a.seed)
    ncell = grid.fluid.size
    cfgs = [vx.SchurConfig(prec=p, max_iter=spec.max_iter, **TOL) for p in spec.precs]
    # one system (context: work vectors + stream) per preconditioner, so the
    # step's independent solves can run concurrently on SM shares
    systems = [vx.assemble(grid, 0, check_connectivity=spec.check_connectivity, device=dev) for _ in cfgs]
    sys_ = systems[0]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{dev}")  # 256 MB > L2

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    def one_step(shares):
        agg = dict(ms=0.0, IA=0, IS=0, dofA=0, dofS=0, msA=0.0, msS=0.0, launches=0,
                   lA=0, lS=0, reps=[], per_kernel={})
        if shares is None:  # sequential, each solve on the whole device
            reps = []
            for s, cfg in zip(systems, cfgs):
                s.limit_sms(0)
                reps.append(vx.solve_schur(s, cfg, return_fields=False))
            agg["ms"] = sum(r.device_ms for r in reps)
        else:
            reps = vx.solve_schur_concurrent(list(zip(systems, cfgs)), sms=shares, return_fields=False)
            agg["ms"] = vx.schur.concurrent_span_ms(systems)
        for s, cfg, rep in zip(systems, cfgs, reps):
            st = vx.last_kernel_stats(s)
            rtot = rep.inner_iter_totals
            agg["IA"] += st["velocity_cg"]["iterations"]
            agg["IS"] += st["simple_cg"]["iterations"]
            agg["dofA"] += st["velocity_cg"]["dof_iters"]
            agg["dofS"] += st["simple_cg"]["dof_iters"]
            agg["msA"] += st["velocity_cg"]["ms"]
            agg["msS"] += st["simple_cg"]["ms"]
            agg["lA"] += st["velocity_cg"]["launches"]
            agg["lS"] += st["simple_cg"]["launches"]
            agg["launches"] += st["kernel_launches"]
            # per fused-CG kernel and operator (a split can run the same
            # operator through different kernels in the two systems)
            for key, op in (("velocity_cg", "A"), ("simple_cg", "S_hat,proj")):
                if st[key]["launches"]:
                    kk = agg["per_kernel"].setdefault(f"{st[key]['kernel']}<{op}>", [0, 0.0, 0, 0])
                    kk[0] += st[key]["dof_iters"]
                    kk[1] += st[key]["ms"]
                    kk[2] += st[key]["launches"]
                    kk[3] = s.sms
            agg["reps"].append(dict(prec=cfg.prec, iters_outer=rep.iters_outer, sms=s.sms,
                                    inner=rtot, k=rep.k_value, converged=rep.converged,
                                    device_ms=rep.device_ms))
        return agg

    # warm-up 1 runs the solves one after another on the whole device.  With
    # two solves, untimed tuning steps then pick the SM split: a coarse scan
    # around the split in proportion to the stand-alone times, then a fine
    # one around the best (per-iteration time steps with the DOFs per thread
    # of the fused CG, so the best split is not the proportional one).
    seq = one_step(None)
    shares, tuning = None, []
    if len(cfgs) == 2 and not a.sequential:
        total = systems[0].sms
        t = [r["device_ms"] for r in seq["reps"]]
        prop = int(round(total * t[1] / (t[0] + t[1])))
        tried = {}

        def trial(k1):
            k1 = min(max(k1, 1), total - 1)
            if k1 not in tried:
                tried[k1] = one_step([total - k1, k1])["ms"]
            return tried[k1]

        # the scan costs ~19 steps: only for steps that take seconds at most
        # (C1); longer workloads use the proportional split
        if max(t) < 2000.0:
            for k1 in range(prop - 24, prop + 25, 4):
                trial(k1)
            best = min(tried, key=tried.get)
            for k1 in range(best - 3, best + 4):
                trial(k1)
        else:
            trial(prop)
        best = min(tried, key=tried.get)
        shares = [total - best, best]
        tuning = sorted(([total - k, k, round(v, 1)] for k, v in tried.items()), key=lambda r: r[1])
    for _ in range(a.warmup - 1):
        one_step(shares)
    barrier()
    steps = []
    with ClockSampler(dev) as clk:
        for _ in range(a.steps):
            flush.zero_()
            torch.cuda.synchronize(dev)
            steps.append(one_step(shares))
        barrier()
    tot = {k: sum(st[k] for st in steps) for k in
           ("ms", "IA", "IS", "dofA", "dofS", "msA", "msS", "launches", "lA", "lS")}
    t_dev = tot["ms"] / 1e3
    cells_iters = ncell * (tot["IA"] + tot["IS"])
    # whole-job aggregate over ranks, max device time over ranks
    if dist is not None:
        tt = torch.tensor([t_dev, cells_iters], dtype=torch.float64, device=f"cuda:{dev}")
        tmax = tt[0:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:2], op=dist.ReduceOp.SUM)
        t_job, cells_job = float(tmax.item()), float(tt[1].item())
    else:
        t_job, cells_job = t_dev, cells_iters
    value = cells_job / t_job / 1e9
    alg_bytes = BYTES_PER_DOF_ITER * (tot["dofA"] + tot["dofS"])
    hbm_alg = alg_bytes / t_dev / 1e9

    # e2e through the public API with host buffers (H2D mask, D2H p, u)
    e2e_t, e2e_cells, h2d, d2h = 0.0, 0, 0, 0
    for _ in range(max(1, a.steps)):
        flush.zero_()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        sy2 = [vx.assemble(grid, 0, check_connectivity=spec.check_connectivity, device=dev) for _ in cfgs]
        if shares is None:
            reps = [vx.solve_schur(s, cfg, return_fields=True) for s, cfg in zip(sy2, cfgs)]
        else:
            reps = vx.solve_schur_concurrent(list(zip(sy2, cfgs)), sms=shares, return_fields=True)
        for s, rep in zip(sy2, reps):
            st = vx.last_kernel_stats(s)
            e2e_cells += ncell * (st["velocity_cg"]["iterations"] + st["simple_cg"]["iterations"])
            d2h += rep.pressure.nbytes + rep.velocity.nbytes + 5 * 8 * (rep.iters_outer + 1)
        e2e_t += time.perf_counter() - t0
        print(f"e2e step {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)
        h2d += grid.fluid.size * len(cfgs)  # uint8 mask, one upload per system
        del sy2
    nsteps_e2e = max(1, a.steps)
    e2e = {"value": e2e_cells / e2e_t / 1e9, "unit": "Gcell/s",
           "h2d_bytes_per_step": h2d // nsteps_e2e, "d2h_bytes_per_step": d2h // nsteps_e2e,
           "ms_per_step": 1e3 * e2e_t / nsteps_e2e,
           "includes": "assemble of one system per solve (host connectivity check + H2D mask + device "
                    "geometry build) + solves (concurrent as in the timed steps) + D2H p,u,histories"}

    peak, peak_kind = measured_peak()

    # dominant kernel: the fused persistent PCG (kernel, operator) with the
    # largest summed launch time over the timed steps
    perk = {}
    for st in steps:
        for k, (d, ms, l, nsm) in st["per_kernel"].items():
            acc = perk.setdefault(k, [0, 0.0, 0, 0])
            acc[0] += d
            acc[1] += ms
            acc[2] += l
            acc[3] = nsm
    kname = max(perk, key=lambda k: perk[k][1])
    dof_k, ms_k, l_k, sms_k = perk[kname]
    achieved = BYTES_PER_DOF_ITER * dof_k / (ms_k / 1e3) / 1e9 if ms_k > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get(a.config, {}).get(kname)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": f"{kname} (fused persistent PCG)",
                "launches": l_k, "avg_launch_ms": ms_k / max(1, l_k),
                "bytes_per_launch": BYTES_PER_DOF_ITER * dof_k / max(1, l_k),
                "peak_kind": peak_kind, "frac_vs_8TBs": achieved / 8000.0,
                # kernel time / step span; above 1 when the step's solves overlap
                "share_of_step": (ms_k / tot["ms"]) if tot["ms"] else None,
                # the kernel runs on its solve's SM share, not the whole device
                "sms": sms_k,
                "kernels": {k: {"launches": v[2], "ms": round(v[1], 3), "sms": v[3],
                                "achieved_gbs": BYTES_PER_DOF_ITER * v[0] / (v[1] / 1e3) / 1e9 if v[1] else 0.0}
                            for k, v in perk.items()}}

    # HBM regime: the same fused kernels on C2 (256^3, working set > L2), one
    # inner A-solve and one inner S_hat-solve (SURVEY 8d per-iteration roofline)
    hbm = None
    if not a.no_hbm:
        g2 = configs.make_geometry("C2", a.seed)
        s2 = vx.assemble(g2, 0, device=dev)
        rng = np.random.default_rng(1)
        pz = rng.standard_normal(s2.m_p)
        pz -= pz.mean()
        rhs = s2.apply_gradient(pz)
        for _ in range(2):  # first = warm-up
            flush.zero_()
            torch.cuda.synchronize(dev)
            vx.schur._solve_velocity(s2, rhs, 1e-12)
            stA = vx.last_kernel_stats(s2)["velocity_cg"]
            flush.zero_()
            torch.cuda.synchronize(dev)
            vx.apply_simple_inverse(s2, pz, 1e-12)
            stS = vx.last_kernel_stats(s2)["simple_cg"]
        tj = {}
        if os.path.exists(os.path.join(ROOT, "profiles", "traffic.json")):
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tj = json.load(f).get("C2", {})

        def rl(st, op):
            ach = BYTES_PER_DOF_ITER * st["dof_iters"] / (st["ms"] / 1e3) / 1e9
            return {"kernel": st["kernel"], "iterations": st["iterations"],
                    "us_per_iteration": 1e3 * st["ms"] / st["iterations"], "achieved": ach, "frac": ach / peak,
                    "algorithmic_bytes": BYTES_PER_DOF_ITER * st["dof_iters"],
                    "traffic": tj.get(f"{st['kernel']}<{op}>")}
        hbm = {"workload": "C2 256^3 spheres phi0.15 (m_u %d, m_p %d): one inner A-solve and one inner "
                           "S_hat-solve to 1e-12" % (s2.m_u, s2.m_p),
               "unit": "GB/s", "peak": peak, "k_pcg_A": rl(stA, "A"), "k_pcg_S": rl(stS, "S_hat,proj")}
        del s2

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu:
            cv, res = cpu_sample(a.config, a.seed, 1)
            cpu = {"value": cv, "unit": "Gcell/s", "cores": 1, "kind": "port",
                   "sample": f"oracle (numpy port of the reference) SIMPLE solve_schur capped at 1 outer "
                             f"iteration on the same geometry: {res[0]['I_A']} A-its + {res[0]['I_S']} "
                             f"S_hat-its in {res[0]['seconds']:.1f} s, 1 core"}
        last = steps[-1]["reps"]
        line = {
            "metric": METRIC, "value": value, "unit": "Gcell/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t_job / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": spec.name, "seed": a.seed, "n": grid.n,
                       "porosity": float(grid.fluid.mean()), "m_u": sys_.m_u, "m_p": sys_.m_p,
                       "precs": list(spec.precs), "tolerances": TOL,
                       "step": "one full solve_schur to tolerance per preconditioner"
                               + (", run concurrently on SM shares (solve_schur_concurrent); step time = "
                                  "device span from the first start to the last end (CUDA events)"
                                  if shares else ", one after another"),
                       "sm_shares": {r["prec"]: r["sms"] for r in steps[-1]["reps"]},
                       "sm_split_tuning_ms": tuning,
                       "l2": "256 MB buffer written between timed steps (L2 flushed)",
                       "parallelism": f"replicas{world}" if world > 1 else "single"},
            "hbm_gbs_algorithmic": hbm_alg,
            # each solve alone on the whole device (warm-up 1, CUDA events)
            "time_to_tol_ms": {r["prec"]: r["device_ms"] for r in seq["reps"]},
            "solves": last,
            "inner_iterations_per_step": {"A": tot["IA"] // a.steps, "S_hat": tot["IS"] // a.steps},
            "roofline": roofline, "roofline_hbm_regime": hbm, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": tot["launches"], "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-hbm", action="store_true", help="skip the C2 HBM-regime kernel measurement")
    ap.add_argument("--sequential", action="store_true",
                    help="run the step's solves one after another on the whole device")
    a = ap.parse_args()
    if a.warmup < 3:
        print("warning: the timing rules require --warmup >= 3", file=sys.stderr)
    sys.exit(run_reference(a) if a.impl == "reference" else run_ours(a))


if __name__ == "__main__":
    main()
