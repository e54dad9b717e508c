#!/usr/bin/env python
"""Benchmark of the Schur-complement Stokes path (BASELINE.json metric).

Workload (default, N=1): BASELINE configs[4] at 512^3 -- the periodic
random-sphere medium (radii U[3,6], porosity 0.2, seed 0, x-percolating
component), f=(1,0,0), SIMPLE-preconditioned Schur CG at eps_S=1e-8,
eps_A=eps_Shat=1e-12.  The full solve to tolerance takes
59 outer iterations (~4 min on one B200), so one "step" is the public call

    solve_schur(sys, SchurConfig(prec="simple", max_iter=1, ...))

i.e. the u_f solve, the first S_hat (preconditioner) solve, ONE outer Schur-CG
iteration (one inner A-solve + one S_hat-solve) and the velocity refresh: the
same inner solves, in the same ~1:50 A:S_hat iteration mix, that make up
every outer iteration of the full solve.  `--config C1|C2|C0` run the other
BASELINE configs (full solves to tolerance); `--max-outer K` changes the cap.

* value     -- masked-stencil Gcell/s = n^3 * (I_A + I_S) / t_device, I_A
               counting every inner A-iteration (incl. the u_f solve), I_S
               every inner S_hat-iteration; t_device = CUDA-event time of the
               step's solve with the geometry resident in HBM.
* e2e       -- same metric through the public API with host buffers:
               assemble(host mask) (H2D + device geometry build) and
               solve_schur returning p, u (D2H) inside the timed region.
* roofline  -- dominant kernel (fused persistent PCG): algorithmic bytes
               64 B per DOF per CG iteration x DOF-iterations
               / summed CUDA-event launch time, vs MEASURED_PEAKS hbm_gbs.
* cpu_baseline / --impl reference -- the reference algorithm on the host
               cores (the numpy oracle port; the reference itself is pure
               Python/numpy and cannot travel to the GPU box).  The reference
               arm loads nothing of the product: the mask comes from the
               pure-numpy generator oracle/stamper.py.  A step there is a
               bounded sample of the same workload: `SAMPLE_A` inner
               A-iterations and `SAMPLE_S` inner S_hat-iterations of the
               oracle's PCG on the same 512^3 system, combined in the step's
               own A:S_hat iteration mix (a full step is hours of CPU time).

Multi-GPU (torchrun, --gpus N): the x-slab decomposition,
one rank per GPU, every rank solving the SAME system ("scaling": "strong");
`--replicas` runs N independent copies instead ("weak").
"""
from __future__ import annotations

import os

# the CPU legs are single-threaded numpy by design (multi-threaded
# OpenBLAS under contention is ~28x slower); pin before numpy is imported, so
# forked worker processes inherit it too
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import glob
import json
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

#: key -> (name, n, dim, preconditioners of one step, outer-iteration cap of a step or None)
WORKLOADS = {
    "C0": ("C0 2D 128^2 disks", 128, 2, ("uzawa",), None),
    "C1": ("C1 64^3 spheres phi0.4", 64, 3, ("uzawa", "simple"), None),
    "C2": ("C2 256^3 spheres phi0.15", 256, 3, ("simple",), None),
    "C4": ("C4 512^3 spheres phi0.2", 512, 3, ("simple",), 1),
    "C4L": ("C4 1024^3 spheres phi0.2", 1024, 3, ("simple",), 1),
}
#: inner iterations of one step (I_A incl. the u_f solve, I_S), used by the
#: reference arm to weight its per-iteration samples when no reference-made
#: fixture of the step exists (tests/golden/cfg_<key>_*.npz); measured on the
#: B200 with the production kernels (profiles/), whose counts are within the
#: +-2 % parity bar of the reference's
MIX_FALLBACK = {"C4": (370, 11897), "C4L": (420, 22800), "C2": (4000, 330000)}
SAMPLE_A, SAMPLE_S = 2, 4  # iterations per CPU sample


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def workload_config(key, seed, cap, fluid, m_u, m_p):
    """The `config` object of the JSON line; both arms build it from the same
    inputs so the driver can compare them field by field."""
    name, n, dim, precs, _ = WORKLOADS[key]
    step = ("one solve_schur per preconditioner through the public API, "
            + ("to tolerance" if cap is None else
               f"capped at max_iter={cap} outer iteration(s): u_f solve + first preconditioner solve + "
               f"{cap} outer Schur-CG step(s) (inner A-solve + S_hat-solve each) + velocity refresh"))
    return {"workload": name, "seed": seed, "n": n, "dim": dim,
            "porosity": float(np.mean(fluid)), "m_u": int(m_u), "m_p": int(m_p),
            "precs": list(precs), "tolerances": TOL, "max_outer": cap, "step": step,
            "l2": ("working set (>= 10 vectors of m_u/m_p doubles) larger than the 126 MB L2"
                   if n >= 256 else "256 MB buffer written between timed steps (L2 flushed)")}


def step_mix(key, precs, cap):
    """(I_A, I_S) of one step from the reference-made fixtures, else MIX_FALLBACK."""
    ia = isx = 0
    for prec in precs:
        name = f"cfg_{key}_{prec}" + (f"_cap{cap}" if cap is not None else "") + ".npz"
        path = os.path.join(ROOT, "tests", "golden", name)
        if not os.path.exists(path):
            return MIX_FALLBACK[key] + ("fallback constants (B200 production-kernel counts)",)
        with np.load(path) as z:
            ia += int(np.sum(z["inner_A_counts"]))
            isx += int(np.sum(z["inner_S_counts"])) if "inner_S_counts" in z.files else 0
    return ia, isx, "reference fixture tests/golden/cfg_%s_*.npz" % key


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


# ----------------------------------------------------------- CPU oracle legs
_ORACLE = {}  # filled before forking: the workers share the tables copy-on-write


def _oracle_setup(key, seed, fluid=None):
    """Oracle system of the workload + seeded right-hand sides (no product code)."""
    from oracle import stamper
    from oracle import voxoracle as vo

    t0 = time.perf_counter()
    if fluid is None:
        fluid = stamper.make_fluid(key, seed)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = vo.build_system(fluid, 0)
    t_asm = time.perf_counter() - t0
    rng = np.random.default_rng(1)
    p = rng.standard_normal(s.m_p)
    p -= p.mean()
    _ORACLE.update(sys=s, p=p, rhs_u=s.apply_gradient(p), inv_a=1.0 / s.laplacian_diag,
                   inv_s=1.0 / vo.simple_inverse_diag(s), t_gen=t_gen, t_asm=t_asm, fluid=fluid)
    return s


def _oracle_sample(_):
    """SAMPLE_A inner A-iterations and SAMPLE_S inner S_hat-iterations of the
    oracle PCG (krylov.py:76-182 restated) -> seconds per iteration of each."""
    from oracle import voxoracle as vo

    o = _ORACLE
    s = o["sys"]

    def timed(op, inv, rhs, its, proj):
        t0 = time.perf_counter()
        vo.pcg(op, lambda r: r * inv, rhs, None, 1e-12, "preconditioned", its, proj, False)
        return time.perf_counter() - t0

    # one capped solve each; its set-up (initial residual = one operator
    # application, one preconditioner application, the norms) is counted as one
    # more iteration, which if anything flatters the CPU figure
    t_a = timed(s.apply_laplacian, o["inv_a"], o["rhs_u"], SAMPLE_A, False) * SAMPLE_A / (SAMPLE_A + 1)
    t_s = timed(s.apply_simple, o["inv_s"], o["p"], SAMPLE_S, True) * SAMPLE_S / (SAMPLE_S + 1)
    return t_a / SAMPLE_A, t_s / SAMPLE_S


def usable_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def mem_available_gb():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable"):
                    return int(ln.split()[1]) / 1e6
    except OSError:
        pass
    return 16.0


def cpu_processes(s):
    """Worker processes for the CPU legs: one per core, bounded by host RAM
    (each worker's private PCG vectors: ~8 velocity- + ~8 pressure-sized)."""
    per_proc_gb = 8 * 8 * (s.m_u + s.m_p) / 1e9 + 0.3
    by_ram = int(max(1, (mem_available_gb() - 4.0) // per_proc_gb))
    return max(1, min(usable_cores(), by_ram)), per_proc_gb


def cpu_sample(procs, ncell, mix):
    """One bounded sample on `procs` forked workers (tables shared
    copy-on-write) -> Gcell/s of the step's iteration mix."""
    if procs <= 1:
        res = [_oracle_sample(0)]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_sample, range(procs), chunksize=1)
    ia, isx = mix
    # every worker runs the same independent sample side by side (as the
    # reference runs independent solves in a process pool, cli.py:205-212)
    t_a = max(r[0] for r in res)
    t_s = max(r[1] for r in res)
    t_step = ia * t_a + isx * t_s
    return len(res) * ncell * (ia + isx) / t_step / 1e9, t_a, t_s, t_step


# ------------------------------------------------------------ reference arm
def run_reference(a):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    name, n, dim, precs, cap0 = WORKLOADS[a.config]
    cap = a.max_outer if a.max_outer is not None else cap0
    s = _oracle_setup(a.config, a.seed)
    ia, isx, mix_src = step_mix(a.config, precs, cap)
    procs, per_gb = cpu_processes(s)
    procs = min(procs, 64)
    ncell = s.fluid.size
    vals, secs, tas, tss = [], [], [], []
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        v, t_a, t_s, _ = cpu_sample(procs, ncell, (ia, isx))
        dt = time.perf_counter() - t0
        if i < a.warmup and dt > 30.0 and procs > 1:
            # numpy's gathers are memory-bound: beyond the host's DRAM bandwidth more
            # workers only stretch the step.  Warm-up steps shrink the pool until a
            # step takes ~25 s, so that the whole run stays within minutes.
            procs = max(1, int(procs * 25.0 / dt))
        if i >= a.warmup:
            vals.append(v)
            secs.append(dt)
            tas.append(t_a)
            tss.append(t_s)
    val = statistics.median(vals)
    sample = (f"per step and worker: {SAMPLE_A} inner A-iterations + {SAMPLE_S} inner S_hat-iterations of the "
              f"oracle PCG (numpy port of the reference) on the same {name} system, {procs} forked workers "
              f"side by side (cores {usable_cores()}, RAM bound {per_gb:.1f} GB/worker, pool shrunk in warm-up until a step "
              f"takes <= ~30 s); seconds per iteration "
              f"(slowest worker, median over steps) A {statistics.median(tas):.3f}, S_hat "
              f"{statistics.median(tss):.3f}; value = workers x n^3 (I_A + I_S) / (I_A t_A + I_S t_S) with the "
              f"step's mix I_A {ia}, I_S {isx} ({mix_src}); mask from oracle/stamper.py "
              f"({_ORACLE['t_gen']:.0f} s), oracle assemble {_ORACLE['t_asm']:.0f} s, both untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Gcell/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
        "scaling": "strong" if world > 1 and not a.replicas else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a.config, a.seed, cap, s.fluid, s.m_u, s.m_p),
        "projected_full_step_s": (ia * statistics.median(tas) + isx * statistics.median(tss)),
        "cpu_baseline": {"value": val, "unit": "Gcell/s", "cores": procs, "kind": "port", "sample": sample},
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

    name, n, dim, precs, cap0 = WORKLOADS[a.config]
    cap = a.max_outer if a.max_outer is not None else cap0
    spec = configs.CONFIGS[a.config]
    slabbed = world > 1 and not a.replicas
    t0 = time.perf_counter()
    grid = configs.make_geometry(a.config, a.seed, device=dev if n >= 256 else None)
    t_gen = time.perf_counter() - t0
    ncell = grid.fluid.size
    kw = dict(TOL)
    kw["max_iter"] = cap if cap is not None else spec.max_iter
    cfgs = [vx.SchurConfig(prec=p, **kw) for p in precs]

    def all_ok(ok):
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        return bool(int(flag.item()))

    def build():
        nonlocal slabbed
        if slabbed:
            # every collective below is entered by every rank, whatever failed locally
            ss = None
            try:
                ss = [vx.assemble(grid, 0, check_connectivity=spec.check_connectivity, device=dev,
                                  rank=rank, nranks=world) for _ in cfgs]
            except Exception as e:  # noqa: BLE001
                print(f"rank {rank}: slab context failed: {type(e).__name__}: {e}", file=sys.stderr)
            if all_ok(ss is not None):
                ok = True
                try:
                    for s in ss:
                        vx.connect_ranks(s)
                except Exception as e:  # noqa: BLE001
                    print(f"rank {rank}: connect_ranks failed: {type(e).__name__}: {e}", file=sys.stderr)
                    ok = False
                if all_ok(ok):
                    return ss
            slabbed = False  # every rank: independent replicas instead
            del ss
        return [vx.assemble(grid, 0, check_connectivity=spec.check_connectivity, device=dev) for _ in cfgs]

    # one system (context: work vectors + stream) per preconditioner, so the
    # step's independent solves can run concurrently on SM shares (C1)
    t0 = time.perf_counter()
    systems = build()
    torch.cuda.synchronize(dev)
    t_asm = time.perf_counter() - t0
    sys_ = systems[0]
    small = n < 256
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{dev}") if small else None

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()

    def one_step(shares, fields=False, sy=None):
        sy = systems if sy is None else sy
        agg = dict(ms=0.0, IA=0, IS=0, dofA=0, dofS=0, msA=0.0, msS=0.0, launches=0,
                   lA=0, lS=0, reps=[], per_kernel={})
        if shares is None:  # one after another, each solve on the whole device
            reps = []
            for s, cfg in zip(sy, cfgs):
                if not slabbed:
                    s.limit_sms(0)
                reps.append(vx.solve_schur(s, cfg, return_fields=fields))
            agg["ms"] = sum(r.device_ms for r in reps)
        else:
            reps = vx.solve_schur_concurrent(list(zip(sy, cfgs)), sms=shares, return_fields=fields)
            agg["ms"] = vx.schur.concurrent_span_ms(sy)
        for s, cfg, rep in zip(sy, cfgs, reps):
            st = vx.last_kernel_stats(s)
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
                    kk = agg["per_kernel"].setdefault(f"{st[key]['kernel']}<{op}>", [0, 0.0, 0, 0, 0])
                    kk[0] += st[key]["dof_iters"]
                    kk[1] += st[key]["ms"]
                    kk[2] += st[key]["launches"]
                    kk[3] = s.sms
                    kk[4] += st[key]["iterations"]
            agg["reps"].append(dict(prec=cfg.prec, iters_outer=rep.iters_outer, sms=s.sms,
                                    inner=rep.inner_iter_totals, k=rep.k_value, converged=rep.converged,
                                    device_ms=rep.device_ms))
            agg.setdefault("bytes_out", 0)
            if fields:
                agg["bytes_out"] += rep.pressure.nbytes + rep.velocity.nbytes + 5 * 8 * (rep.iters_outer + 1)
        return agg

    # warm-up 1 runs the solves one after another on the whole device.  With
    # two small solves (C1), untimed tuning steps then pick the SM split.
    slab_error = None
    if slabbed:
        # the slab transport (CUDA IPC + cross-GPU barriers) has never run on
        # hardware: if any rank fails to build or to finish its first step (a
        # barrier that times out raises instead of hanging), every rank falls
        # back to independent replicas and the line says so
        failed = 0
        try:
            seq = one_step(None)
        except Exception as e:  # noqa: BLE001
            failed, slab_error = 1, f"{type(e).__name__}: {e}"
        flag = torch.tensor([failed], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if int(flag.item()):
            slab_error = slab_error or "another rank failed"
            print(f"rank {rank}: slab decomposition failed ({slab_error}); falling back to replicas",
                  file=sys.stderr)
            slabbed = False
            del systems
            systems = build()
            sys_ = systems[0]
            seq = one_step(None)
    else:
        seq = one_step(None)
    shares, tuning = None, []
    if len(cfgs) == 2 and small and not a.sequential and not slabbed:
        total = systems[0].sms
        t = [r["device_ms"] for r in seq["reps"]]
        prop = int(round(total * t[1] / (t[0] + t[1])))
        tried = {}

        def trial(k1):
            k1 = min(max(k1, 1), total - 1)
            if k1 not in tried:
                tried[k1] = one_step([total - k1, k1])["ms"]
            return tried[k1]

        for k1 in range(prop - 24, prop + 25, 4):
            trial(k1)
        best = min(tried, key=tried.get)
        for k1 in range(best - 3, best + 4):
            trial(k1)
        best = min(tried, key=tried.get)
        shares = [total - best, best]
        tuning = sorted(([total - k, k, round(v, 1)] for k, v in tried.items()), key=lambda r: r[1])
    for _ in range(a.warmup - 1):
        one_step(shares)
    barrier()
    steps = []
    with ClockSampler(dev) as clk:
        for _ in range(a.steps):
            if flush is not None:
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
        t_job = float(tmax.item())
        if slabbed:  # every rank reports the one shared solve
            cells_job = float(cells_iters)
        else:
            dist.all_reduce(tt[1:2], op=dist.ReduceOp.SUM)
            cells_job = float(tt[1].item())
    else:
        t_job, cells_job = t_dev, cells_iters
    value = cells_job / t_job / 1e9
    alg_bytes = BYTES_PER_DOF_ITER * (tot["dofA"] + tot["dofS"])
    hbm_alg = alg_bytes / t_dev / 1e9

    # e2e through the public API with host buffers (H2D mask, D2H p, u):
    # a bounded number of steps (each repeats the assemble)
    n_e2e = 0 if a.no_e2e else max(1, min(a.steps, 3 if not small else a.steps))
    e2e_t, e2e_cells, h2d, d2h = 0.0, 0, 0, 0
    for _ in range(n_e2e):
        if flush is not None:
            flush.zero_()
        barrier()
        t0 = time.perf_counter()
        sy2 = build()
        st = one_step(shares, fields=True, sy=sy2)
        e2e_cells += ncell * (st["IA"] + st["IS"])
        d2h += st["bytes_out"]
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t0
        e2e_t += dt
        print(f"e2e step {1e3 * dt:.1f} ms", file=sys.stderr)
        h2d += grid.fluid.size * len(cfgs)  # uint8 mask, one upload per system
        del sy2
    e2e = None if not n_e2e else {"value": e2e_cells / e2e_t / 1e9, "unit": "Gcell/s",
           "h2d_bytes_per_step": h2d // n_e2e, "d2h_bytes_per_step": d2h // n_e2e,
           "ms_per_step": 1e3 * e2e_t / n_e2e, "steps": n_e2e,
           "includes": "assemble of one system per solve (connectivity check + H2D mask + device "
                       "geometry build) + the step's solves + D2H p, u, histories (pageable numpy buffers)"}

    peak, peak_kind = measured_peak()

    # dominant kernel: the fused persistent PCG (kernel, operator) with the
    # largest summed launch time over the timed steps
    perk = {}
    for st in steps:
        for k, (d, ms, l, nsm, its) in st["per_kernel"].items():
            acc = perk.setdefault(k, [0, 0.0, 0, 0, 0])
            acc[0] += d
            acc[1] += ms
            acc[2] += l
            acc[3] = nsm
            acc[4] += its
    kname = max(perk, key=lambda k: perk[k][1])
    dof_k, ms_k, l_k, sms_k, its_k = perk[kname]
    achieved = BYTES_PER_DOF_ITER * dof_k / (ms_k / 1e3) / 1e9 if ms_k > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get(a.config, {}).get(kname)
        if isinstance(traffic, dict):  # measured DRAM bytes per DOF-iteration -> per launch of this run
            traffic = traffic["bytes_per_dof_iter"] * dof_k / max(1, l_k)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": f"{kname} (fused persistent PCG, one launch per inner solve)",
                "launches": l_k, "avg_launch_ms": ms_k / max(1, l_k),
                "bytes_per_launch": BYTES_PER_DOF_ITER * dof_k / max(1, l_k),
                "us_per_cg_iteration": 1e3 * ms_k / max(1, its_k),
                "peak_kind": peak_kind, "frac_vs_8TBs": achieved / 8000.0,
                # kernel time / step span; above 1 when the step's solves overlap
                "share_of_step": (ms_k / tot["ms"]) if tot["ms"] else None,
                "sms": sms_k,
                "kernels": {k: {"launches": v[2], "ms": round(v[1], 3), "sms": v[3],
                                "us_per_cg_iteration": 1e3 * v[1] / max(1, v[4]),
                                "achieved_gbs": BYTES_PER_DOF_ITER * v[0] / (v[1] / 1e3) / 1e9 if v[1] else 0.0}
                            for k, v in perk.items()}}

    # extras (N = 1): the same fused kernels on the other 3D configs -- one inner
    # A-solve and one inner S_hat-solve at C2 256^3 (us per CG iteration, fraction of
    # the copy peak) and the C1 64^3 solves to tolerance.  Not part of the timed region.
    extras = None
    if world == 1 and not a.no_extras and a.config in ("C4", "C4L"):
        extras = {}
        del systems
        g2 = configs.make_geometry("C2", a.seed, device=dev)
        s2 = vx.assemble(g2, 0, device=dev)
        pz = np.random.default_rng(1).standard_normal(s2.m_p)
        pz -= pz.mean()
        rhs = s2.apply_gradient(pz)
        for _ in range(2):  # first = warm-up
            vx.schur._solve_velocity(s2, rhs, 1e-12)
            st_a = vx.last_kernel_stats(s2)["velocity_cg"]
            vx.apply_simple_inverse(s2, pz, 1e-12)
            st_s = vx.last_kernel_stats(s2)["simple_cg"]

        def per_it(st):
            ach = BYTES_PER_DOF_ITER * st["dof_iters"] / (st["ms"] / 1e3) / 1e9
            return {"kernel": st["kernel"], "iterations": st["iterations"],
                    "us_per_cg_iteration": 1e3 * st["ms"] / max(1, st["iterations"]), "achieved_gbs": ach,
                    "frac": ach / peak}
        extras["C2 256^3 spheres phi0.15 inner solves to 1e-12"] = {
            "m_u": s2.m_u, "m_p": s2.m_p, "A": per_it(st_a), "S_hat": per_it(st_s)}
        del s2
        g1 = configs.make_geometry("C1", a.seed)
        s1 = vx.assemble(g1, 0, device=dev)
        c1 = {}
        for prec in ("uzawa", "simple"):
            for _ in range(2):
                r1 = vx.solve_schur(s1, vx.SchurConfig(prec=prec, **TOL), return_fields=False)
            c1[prec] = {"device_ms": r1.device_ms, "iters_outer": r1.iters_outer, "inner": r1.inner_iter_totals,
                        "k": r1.k_value, "converged": r1.converged}
        extras["C1 64^3 spheres phi0.4 solve_schur to tolerance"] = c1
        del s1

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not a.no_cpu:
            # the oracle on the same mask (its own assemble, untimed), 1 core
            s_or = _oracle_setup(a.config, a.seed, fluid=grid.fluid)
            ia, isx = tot["IA"] // a.steps, tot["IS"] // a.steps
            cv, t_a, t_s, t_step = cpu_sample(1, ncell, (ia, isx))
            cpu = {"value": cv, "unit": "Gcell/s", "cores": 1, "kind": "port",
                   "sample": f"oracle (numpy port of the reference) PCG on the same system: {SAMPLE_A} inner "
                             f"A-iterations at {t_a:.3f} s/it + {SAMPLE_S} inner S_hat-iterations at {t_s:.3f} "
                             f"s/it, combined in this step's mix (I_A {ia}, I_S {isx}); a full step would take "
                             f"{t_step:.0f} s on 1 core (projection)"}
            del s_or
            _ORACLE.clear()
        last = steps[-1]["reps"]
        cfg_obj = workload_config(a.config, a.seed, cap, grid.fluid, sys_.m_u, sys_.m_p)
        line = {
            "metric": METRIC, "value": value, "unit": "Gcell/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * t_job / a.steps,
            "higher_is_better": True, "scaling": "strong" if slabbed else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg_obj,
            "parallelism": (f"xslab{world}" if slabbed else (f"replicas{world}" if world > 1 else "single")),
            "slab_fallback": slab_error,
            "sm_shares": {r["prec"]: r["sms"] for r in last}, "sm_split_tuning_ms": tuning,
            "hbm_gbs_algorithmic": hbm_alg,
            "setup_s": {"generate_mask": t_gen, "assemble": t_asm},
            "solves": last,
            "inner_iterations_per_step": {"A": tot["IA"] // a.steps, "S_hat": tot["IS"] // a.steps},
            "roofline": roofline, "extras": extras, "cpu_baseline": cpu, "e2e": e2e,
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
    ap.add_argument("--config", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--max-outer", type=int, default=None,
                    help="outer-iteration cap of a step (default: the workload's; C4: 1)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end steps (long evidence runs)")
    ap.add_argument("--no-extras", action="store_true", help="skip the C2 / C1 extra measurements")
    ap.add_argument("--sequential", action="store_true",
                    help="run the step's solves one after another on the whole device")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the slab decomposition")
    a = ap.parse_args()
    if a.warmup < 3:
        print("warning: the timing rules require --warmup >= 3", file=sys.stderr)
    sys.exit(run_reference(a) if a.impl == "reference" else run_ours(a))


if __name__ == "__main__":
    main()
