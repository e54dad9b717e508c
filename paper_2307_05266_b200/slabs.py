"""x-slab decomposition plan (host side, no device needed).

Slab s of R owns reference x-planes [s*n//R, (s+1)*n//R) of every DOF family
and keeps one ghost plane on each side (periodic).  Local vectors are laid
out [owned DOFs (velocity components in order) | ghost_lo_f | ghost_hi_f ...];
the first owned plane of slab s is the ghost_hi plane of slab s-1 and its
last owned plane the ghost_lo plane of slab s+1, in identical DOF order, so a
halo exchange is a contiguous copy per family.  The plan comes from the
native planner (vs_slab_plan) that also lays out the device slabs.
"""
from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["slab_plan", "FAMILY_FIELDS"]

FAMILY_FIELDS = ("own", "own_off", "glo_off", "glo_cnt", "ghi_off", "ghi_cnt",
                 "first_cnt", "last_cnt", "gstart")


def slab_plan(fluid: np.ndarray, slabs: int) -> list:
    """Per-slab layout dicts; family keys 0..dim-1 (velocity) and 'p'."""
    fluid = np.ascontiguousarray(fluid, dtype=np.uint8)
    dim, n = fluid.ndim, fluid.shape[0]
    out = np.zeros(slabs * 42, dtype=np.int64)
    _lib.check(_lib.lib.vs_slab_plan(fluid.ravel(), dim, n, slabs, _lib.ptr(out)))
    plans = []
    for s in range(slabs):
        o = out[s * 42 : (s + 1) * 42]
        fams = {}
        for f, key in enumerate([0, 1, 2, "p"]):
            if key != "p" and key >= dim:
                continue
            fams[key] = dict(zip(FAMILY_FIELDS, (int(v) for v in o[2 + 9 * f : 11 + 9 * f])))
        plans.append(dict(x_lo=int(o[0]), x_hi=int(o[1]), fam=fams,
                          m_own=(int(o[38]), int(o[39])), m_all=(int(o[40]), int(o[41]))))
    return plans
