"""Record how sensitive the REFERENCE's own full solves are to the rounding of
its dot products, for the golden geometries (tests/golden/sensitivity.json).

Run inside the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_sensitivity.py

For every golden case and preconditioner the reference's ``solve_schur``
(schur.py:291-385) is run twice more with its ``pcg`` (krylov.py:76-182)
recompiled from its own source with ``r @ z``, ``d @ q`` and the two
``np.linalg.norm`` calls replaced by (a) exactly rounded sums (math.fsum) and
(b) a 256-wide pairwise tree -- nothing else changes (SURVEY Appendix C,
"parity calibration").  The recorded number is the largest relative
difference of p, u (2-norm) and k between those runs and the stock run the
fixture holds.  Where it exceeds 1e-8, no implementation with its own
reduction order can match the fixture to 1e-8, and the GPU test allows 3x the
recorded value for that case instead (tests/test_gpu_parity.py); everywhere
else the bar stays 1e-8.
"""
from __future__ import annotations

import inspect
import json
import math
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import voxstokes.krylov as rk  # noqa: E402
import voxstokes.schur as rs  # noqa: E402
from voxstokes.geometry import VoxelGrid  # noqa: E402
from voxstokes.operators import assemble  # noqa: E402

TOL = dict(eps_S=1e-8, eps_A=1e-12, eps_Shat=1e-12)
CASES = ["pack2d", "pack3d", "rand3d", "wrap2", "channel16", "disks2d", "spheres3d"]


def _fsum_dot(a, b):
    return math.fsum(np.asarray(a) * np.asarray(b))


def _tree_dot(a, b):
    v = np.asarray(a) * np.asarray(b)
    pad = (-v.size) % 256
    w = np.concatenate([v, np.zeros(pad)]).reshape(-1, 256)
    while w.shape[1] > 1:
        w = w[:, 0::2] + w[:, 1::2]
    s = w[:, 0]
    while s.size > 1:
        if s.size % 2:
            s = np.concatenate([s, [0.0]])
        s = s[0::2] + s[1::2]
    return float(s[0]) if s.size else 0.0


def recompiled_pcg(dot):
    """The reference's pcg with its reductions routed through ``dot``."""
    src = inspect.getsource(rk.pcg)
    for old, new in (("float(r @ z)", "_dot(r, z)"), ("float(d @ q)", "_dot(d, q)"),
                     ("float(np.linalg.norm(z))", "float(np.sqrt(_dot(z, z)))"),
                     ("float(np.linalg.norm(r))", "float(np.sqrt(_dot(r, r)))")):
        assert old in src, old
        src = src.replace(old, new)
    ns = dict(vars(rk))
    ns["_dot"] = dot
    exec(compile(src, "<recompiled reference pcg>", "exec"), ns)
    return ns["pcg"]


def rel(a, b):
    den = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / (den if den > 0 else 1.0))


def main():
    warnings.simplefilter("ignore")
    stock = rs.pcg
    out = {}
    for name in CASES:
        with np.load(os.path.join(HERE, f"{name}.npz")) as z:
            g = {k: z[k] for k in z.files}
        sys_ = assemble(VoxelGrid(g["fluid"]), flow_dir=int(g["flow_dir"]))
        for prec in ("uzawa", "simple"):
            pre = f"{prec}_"
            worst = dict(p=0.0, u=0.0, k=0.0)
            for dot in (_fsum_dot, _tree_dot):
                rs.pcg = recompiled_pcg(dot)
                try:
                    rep = rs.solve_schur(sys_, rs.SchurConfig(prec=prec, **TOL))
                finally:
                    rs.pcg = stock
                kref = float(g[pre + "k_value"])
                worst["p"] = max(worst["p"], rel(rep.pressure, g[pre + "pressure"]))
                worst["u"] = max(worst["u"], rel(rep.velocity, g[pre + "velocity"]))
                worst["k"] = max(worst["k"], abs(rep.k_value - kref) / abs(kref))
            out[f"{name}/{prec}"] = worst
            print(name, prec, worst, flush=True)
    with open(os.path.join(HERE, "sensitivity.json"), "w") as f:
        json.dump({"_doc": "largest relative change of the reference's own p, u, k when only the rounding of "
                           "its pcg dot products changes (make_sensitivity.py)", **out}, f, indent=1)


if __name__ == "__main__":
    main()
