"""Seeded synthetic geometries for the BASELINE.json configs (C0-C4).

BASELINE's inputs are synthetic: seeded disks / spheres / slits /
cylinders on a periodic box.  The reference has no generator for them
(its only one is the square/cube packing, geometry.py:134-156), so this
module defines them once, deterministically:

* RNG: ``numpy.random.default_rng(seed)`` (PCG64, as the reference uses).
  Balls are drawn in batches of ``BATCH``: ``uniform(0, n, (BATCH, dim))``
  centres, then ``uniform(rmin, rmax, BATCH)`` radii.
* A cell (integer index i) is solid if its minimum-image distance to a
  ball centre is <= r (cylinders: distance in the cross-section).  Balls
  are stamped in order until porosity <= the target (native stamper,
  vs_stamp_balls), or exactly ``count`` balls when a count is given.
* "Fluid = connected component percolating in x": keep the largest
  periodic component (the reference's enforce_connectivity rule,
  geometry.py:225-240) and assert that it percolates in x -- that it holds a
  closed path of non-zero x-winding (``winding``: the periodic union-find of
  geometry.py:183-222 carrying the unwrapped x-offset);
  generation fails loudly otherwise (the seed is never silently changed).
* Slits and x-cylinders are x-prismatic: every fluid component percolates
  in x, so all of them are kept (``check_connectivity=False`` at assemble,
  as the reference needs for multi-component masks, operators.py:224-230)
  and the winding check asserts exactly that.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import VoxelGrid, enforce_connectivity

__all__ = ["ConfigSpec", "CONFIGS", "make_geometry", "balls", "slits", "winding", "x_percolates"]

BATCH = 4096


def _stamp(fluid: np.ndarray, centers, radii, target: int, prism_axis: int, n_fluid: int = -1):
    used, nf = C.c_int64(), C.c_int64(n_fluid)
    flat = fluid.reshape(-1)
    _lib.check(_lib.lib.vs_stamp_balls(
        _lib.ptr(flat), fluid.ndim, fluid.shape[0], _lib.ptr(np.ascontiguousarray(centers)),
        _lib.ptr(np.ascontiguousarray(radii)), len(radii), int(target), int(prism_axis),
        C.byref(used), C.byref(nf)))
    return int(used.value), int(nf.value)


def balls(n: int, dim: int, rmin: float, rmax: float, *, porosity: float | None = None,
          count: int | None = None, seed: int = 0, prism_axis: int = -1) -> np.ndarray:
    """Fluid mask (bool) of a box with seeded solid balls / cylinders."""
    rng = np.random.default_rng(seed)
    fluid = np.ones((n,) * dim, dtype=np.uint8)
    if count is not None:
        c = rng.uniform(0, n, size=(count, dim))
        r = rng.uniform(rmin, rmax, size=count)
        _stamp(fluid, c, r, -1, prism_axis)
        return fluid.astype(bool)
    target = int(np.floor(porosity * fluid.size))
    nf = fluid.size
    while True:
        c = rng.uniform(0, n, size=(BATCH, dim))
        r = rng.uniform(rmin, rmax, size=BATCH)
        used, nf = _stamp(fluid, c, r, target, prism_axis, nf)
        if nf <= target:
            return fluid.astype(bool)


def slits(n: int, w: int, wall: int = 4) -> np.ndarray:
    """Parallel-plate slits normal to z (last axis): width w, solid walls of
    ``wall`` voxels; the tail that does not fit a full period is solid so
    the periodic seam never merges two slits."""
    fluid = np.zeros((n, n, n), dtype=bool)
    period = w + wall
    for k in range(n // period):
        fluid[:, :, k * period : k * period + w] = True
    return fluid


def winding(fluid: np.ndarray, axis: int = 0) -> tuple[int, int]:
    """(periodic components, components that percolate along ``axis``).

    A component percolates iff it contains a closed path whose unwrapped
    displacement along ``axis`` is a non-zero multiple of n (vs_winding:
    union-find over the fluid cells that carries the axis offset)."""
    f = np.ascontiguousarray(fluid, dtype=np.uint8)
    nc, nw = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib.vs_winding(f.reshape(-1), f.ndim, f.shape[0], int(axis),
                                   C.byref(nc), C.byref(nw)))
    return int(nc.value), int(nw.value)


def x_percolates(fluid: np.ndarray) -> bool:
    """True when every periodic fluid component of the mask percolates in x."""
    nc, nw = winding(fluid, 0)
    return nc > 0 and nc == nw


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n: int
    dim: int
    kind: str           # balls | cylinders | slits
    rmin: float = 0.0
    rmax: float = 0.0
    porosity: float | None = None
    count: int | None = None
    width: int = 0
    precs: tuple = ("uzawa", "simple")
    max_iter: int = 1000
    check_connectivity: bool = True


CONFIGS = {
    "C0": ConfigSpec("C0 2D 128^2 disks", 128, 2, "balls", 8, 16, count=20, precs=("uzawa",)),
    "C1": ConfigSpec("C1 64^3 spheres phi0.4", 64, 3, "balls", 4, 8, porosity=0.4),
    "C2": ConfigSpec("C2 256^3 spheres phi0.15", 256, 3, "balls", 2, 4, porosity=0.15,
                     precs=("simple", "uzawa")),
    "C3c": ConfigSpec("C3 256^3 x-cylinders r3 phi0.3", 256, 3, "cylinders", 3, 3, porosity=0.3,
                      check_connectivity=False),
    "C4": ConfigSpec("C4 512^3 spheres phi0.2", 512, 3, "balls", 3, 6, porosity=0.2,
                     precs=("simple",)),
    "C4L": ConfigSpec("C4 1024^3 spheres phi0.2", 1024, 3, "balls", 3, 6, porosity=0.2,
                      precs=("simple",)),
}
for _w in (2, 4, 8, 16, 32):
    CONFIGS[f"C3s{_w}"] = ConfigSpec(f"C3 256^3 slits w{_w}", 256, 3, "slits", width=_w,
                                     check_connectivity=False)


def make_geometry(key: str, seed: int = 0, n: int | None = None, device: int | None = None) -> VoxelGrid:
    """The fluid grid of config ``key`` (optionally at a different n, for tests).
    ``device``: run the connected-component labelling on that GPU."""
    spec = CONFIGS[key]
    n = spec.n if n is None else n
    if spec.kind == "slits":
        grid = VoxelGrid(slits(n, spec.width))
    elif spec.kind == "cylinders":
        # x-prisms: every fluid component percolates in x, so all are kept
        grid = VoxelGrid(balls(n, spec.dim, spec.rmin, spec.rmax, porosity=spec.porosity, seed=seed,
                               prism_axis=0))
    else:
        fluid = balls(n, spec.dim, spec.rmin, spec.rmax, porosity=spec.porosity,
                      count=spec.count, seed=seed)
        grid, _ = enforce_connectivity(VoxelGrid(fluid), device)
    nc, nw = winding(grid.fluid, 0)
    if nc == 0 or nw != nc:
        raise ValueError(f"{key} seed {seed}: {nc - nw} of {nc} kept fluid components do not "
                         "percolate in x")
    return grid
