"""Pure-numpy geometry generator for the BASELINE configs (TEST INFRASTRUCTURE ONLY).

A second, independent statement of ``paper_2307_05266_b200.configs`` (whose
stamping runs in libvoxschur.so): the same seeded draws, the same
minimum-image distance test, the same stopping rule.  It exists so that

* the golden-fixture generator (``tests/golden/make_config_golden.py``) and
  ``bench.py --impl reference`` can build the BASELINE masks without
  loading the product library, and
* the product stamper can be checked bitwise against it
  (``tests/test_host_cpu.py::test_stamper_matches_oracle``).

Only ``tests/``, ``tests/golden/*.py``, ``__graft_entry__.smoke()`` and the
CPU legs of ``bench.py`` may import this module; the product package never
does.  The reference has no generator for these geometries (its only one is
the square/cube packing, geometry.py:134-156), so there is no reference
line to cite for the stamping itself; the connectivity rule restates
geometry.py:183-240 (see ``voxoracle.enforce_connectivity``).
"""
from __future__ import annotations

import hashlib

import numpy as np

from . import voxoracle as vo

BATCH = 4096

#: key -> (n, dim, kind, rmin, rmax, porosity, count, width)
SPECS = {
    "C0": (128, 2, "balls", 8.0, 16.0, None, 20, 0),
    "C1": (64, 3, "balls", 4.0, 8.0, 0.4, None, 0),
    "C2": (256, 3, "balls", 2.0, 4.0, 0.15, None, 0),
    "C3c": (256, 3, "cylinders", 3.0, 3.0, 0.3, None, 0),
    "C4": (512, 3, "balls", 3.0, 6.0, 0.2, None, 0),
    "C4L": (1024, 3, "balls", 3.0, 6.0, 0.2, None, 0),
}
for _w in (2, 4, 8, 16, 32):
    SPECS[f"C3s{_w}"] = (256, 3, "slits", 0.0, 0.0, None, None, _w)


def _stamp(fluid: np.ndarray, centers, radii, target: int, prism_axis: int, nf: int):
    """Stamp balls in order while the fluid count is above ``target``.

    A cell (integer index) turns solid when its squared minimum-image
    distance to the centre, accumulated axis by axis from 0.0, is <= r*r.
    Returns (balls used, fluid count).
    """
    n, dim = fluid.shape[0], fluid.ndim
    k = 0
    for k in range(len(radii)):
        if nf <= target:
            return k, nf
        r = float(radii[k])
        r2 = r * r
        idx, d2 = [], []
        for a in range(dim):
            c = float(centers[k, a])
            if a == prism_axis:
                lo, hi = 0, n - 1
            else:
                lo = int(np.floor(c - r)) - 1
                hi = int(np.ceil(c + r)) + 1
                if hi - lo + 1 > n:
                    lo, hi = 0, n - 1
            w = np.arange(lo, hi + 1) % n
            dd = np.abs(w.astype(np.float64) - c)
            dd = np.minimum(dd, float(n) - dd)
            idx.append(w)
            d2.append(np.zeros(len(w)) if a == prism_axis else dd * dd)
        if dim == 2:
            tot = (0.0 + d2[0][:, None]) + d2[1][None, :]
        else:
            tot = ((0.0 + d2[0][:, None, None]) + d2[1][None, :, None]) + d2[2][None, None, :]
        sel = np.ix_(*idx)
        win = fluid[sel]
        hit = (tot <= r2) & win
        nf -= int(hit.sum())
        fluid[sel] = win & ~hit
    else:
        k = len(radii)
    return k, nf


def balls(n, dim, rmin, rmax, *, porosity=None, count=None, seed=0, prism_axis=-1):
    """Fluid mask (bool) of a periodic box with seeded solid balls / cylinders."""
    rng = np.random.default_rng(seed)
    fluid = np.ones((n,) * dim, dtype=bool)
    if count is not None:
        c = rng.uniform(0, n, size=(count, dim))
        r = rng.uniform(rmin, rmax, size=count)
        _stamp(fluid, c, r, -1, prism_axis, fluid.size)
        return fluid
    target = int(np.floor(porosity * fluid.size))
    nf = fluid.size
    while True:
        c = rng.uniform(0, n, size=(BATCH, dim))
        r = rng.uniform(rmin, rmax, size=BATCH)
        _, nf = _stamp(fluid, c, r, target, prism_axis, nf)
        if nf <= target:
            return fluid


def slits(n: int, w: int, wall: int = 4) -> np.ndarray:
    """Slits normal to z of width w between solid walls of ``wall`` voxels; the
    tail that does not fit a whole period stays solid."""
    fluid = np.zeros((n, n, n), dtype=bool)
    period = w + wall
    for k in range(n // period):
        fluid[:, :, k * period:k * period + w] = True
    return fluid


def make_fluid(key: str, seed: int = 0, n: int | None = None) -> np.ndarray:
    """The fluid mask of config ``key`` (same rule as configs.make_geometry)."""
    n0, dim, kind, rmin, rmax, phi, count, width = SPECS[key]
    n = n0 if n is None else n
    if kind == "slits":
        return slits(n, width)
    if kind == "cylinders":
        # x-prisms: every fluid component winds in x, so all are kept
        return balls(n, dim, rmin, rmax, porosity=phi, seed=seed, prism_axis=0)
    fluid = balls(n, dim, rmin, rmax, porosity=phi, count=count, seed=seed)
    kept, _ = vo.enforce_connectivity(fluid)
    return kept


def mask_digest(fluid: np.ndarray) -> str:
    """sha256 of the bit-packed mask plus its shape (fixture identity)."""
    h = hashlib.sha256()
    h.update(repr(tuple(fluid.shape)).encode())
    h.update(np.packbits(np.ascontiguousarray(fluid, dtype=bool)).tobytes())
    return h.hexdigest()
