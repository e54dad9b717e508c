"""Voxel geometry input type, periodic connectivity, stats, the packing
generator and the voxgeo text IO (host side).

``VoxelGrid`` mirrors geometry.py:29-66 (validation and immutability);
``connected_components`` / ``enforce_connectivity`` mirror
geometry.py:183-240 and run in the native library (vs_components, a
periodic union-find in C++, or its GPU twin).  ``read_grid`` /
``write_grid`` (geometry.py:243-339) run in the library's multithreaded
C++ reader/writer (vs_io.cpp) with the reference's messages.
``PackingParams`` / ``generate_packing`` / ``stats`` / ``periodize``
(geometry.py:69-180, :243-255) are the callers the CLI needs.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["VoxelGrid", "GeometryStats", "PackingParams", "generate_packing", "stats",
           "connected_components", "enforce_connectivity", "periodize", "read_grid",
           "write_grid"]


@dataclass(frozen=True)
class VoxelGrid:
    """Immutable binary voxel image; True where the voxel is fluid."""

    fluid: np.ndarray
    physical_length: float = 1.0

    def __post_init__(self):
        arr = np.ascontiguousarray(self.fluid, dtype=bool).copy()
        if arr.ndim not in (2, 3):
            raise ValueError(f"grid dimension must be 2 or 3, got {arr.ndim}")
        if len(set(arr.shape)) != 1:
            raise ValueError(f"grid must be cubic, got shape {arr.shape}")
        if arr.shape[0] < 2:
            raise ValueError(f"grid extent must be at least 2, got {arr.shape[0]}")
        if self.physical_length != 1.0:
            raise ValueError("physical_length is fixed to 1.0")
        arr.setflags(write=False)
        object.__setattr__(self, "fluid", arr)

    @property
    def dim(self) -> int:
        return self.fluid.ndim

    @property
    def n(self) -> int:
        return self.fluid.shape[0]


def connected_components(grid: VoxelGrid, device: int | None = None):
    """Label fluid components under periodic face adjacency.

    Returns ``(labels, n_components)``; labels are -1 on solid and dense
    ids in first row-major appearance on fluid (geometry.py:183-190).
    With ``device`` the labelling runs on that GPU (same labels).
    """
    labels, n = _labels32(grid, device)
    return labels.astype(np.int64), n


def _labels32(grid: VoxelGrid, device: int | None):
    f = np.ascontiguousarray(grid.fluid, dtype=np.uint8)
    labels = np.empty(f.shape, dtype=np.int32)
    n = C.c_int64()
    if device is None:
        _lib.check(_lib.lib.vs_components(f.ravel(), grid.dim, grid.n, _lib.ptr(labels), C.byref(n)))
    else:
        _lib.check(_lib.lib.vs_components_device(f.ravel(), grid.dim, grid.n, int(device), _lib.ptr(labels),
                                                 C.byref(n)))
    return labels, int(n.value)


def enforce_connectivity(grid: VoxelGrid, device: int | None = None):
    """Solidify everything outside the largest component (ties: lowest id)."""
    labels, n = _labels32(grid, device)
    if n == 0:
        raise ValueError("empty fluid domain")
    if n == 1:
        return grid, 0
    sizes = np.bincount(labels[labels >= 0], minlength=n)
    fluid = labels == int(np.argmax(sizes))
    return VoxelGrid(fluid), int(grid.fluid.sum() - fluid.sum())


@dataclass(frozen=True)
class GeometryStats:
    """Exact integer counts and derived percentages (geometry.py:69-78)."""

    v_fluid: int
    v_surf: int
    porosity_pct: float
    stv_pct: float
    n_components: int


@dataclass(frozen=True)
class PackingParams:
    """Shifted-obstacle packing parameters, validated as geometry.py:81-131."""

    N: int
    n_c: int
    n_avg: int
    n_min: int
    seed: int
    dim: int = 2

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise ValueError(f"dim must be 2 or 3, got {self.dim}")
        if self.N < 1:
            raise ValueError(f"cell count N must be at least 1, got {self.N}")
        if self.n_min < 1:
            raise ValueError(f"n_min must be at least 1, got {self.n_min}")
        if self.n_avg < self.n_min:
            raise ValueError(f"n_avg ({self.n_avg}) must be at least n_min ({self.n_min})")
        if self.n_c <= self.n_avg:
            raise ValueError(f"cell side n_c ({self.n_c}) must exceed n_avg ({self.n_avg})")
        if self.n_avg % 2 != 0:
            raise ValueError(f"n_avg must be even, got {self.n_avg}")
        if (self.n_avg - self.n_min) % 2 != 0:
            raise ValueError(f"n_avg - n_min must be even, got {self.n_avg - self.n_min}")
        if not 0 <= self.seed < 2**64:
            raise ValueError("seed must be a 64-bit unsigned integer")

    @property
    def extent(self) -> int:
        return self.N * self.n_c

    @property
    def shift_range(self) -> int:
        return (self.n_avg - self.n_min) // 2


def generate_packing(params: PackingParams) -> VoxelGrid:
    """One solid square/cube of side n_c - n_avg per cell, shifted by a
    PCG64 draw per cell in row-major cell order (geometry.py:134-156).

    All shift vectors are drawn first (the same stream as one draw per
    cell), then every obstacle is cleared as a slice; the mask is
    bit-identical to the reference's.
    """
    half = params.shift_range
    side = params.n_c - params.n_avg
    d, cells = params.dim, params.N ** params.dim
    fluid = np.ones((params.extent,) * d, dtype=bool)
    rng = np.random.default_rng(params.seed)
    shifts = [rng.integers(-half, half + 1, size=d) for _ in range(cells)]
    for cell, r in zip(np.ndindex(*(params.N,) * d), shifts):
        lo = [c * params.n_c + params.n_avg // 2 + int(x) for c, x in zip(cell, r)]
        fluid[tuple(slice(a, a + side) for a in lo)] = False
    return VoxelGrid(fluid)


def stats(grid: VoxelGrid, device: int | None = None) -> GeometryStats:
    """Porosity, no-slip surface voxel count and component count
    (geometry.py:159-180); components from the native labelling."""
    fluid = grid.fluid
    v_fluid = int(np.count_nonzero(fluid))
    if v_fluid == 0:
        raise ValueError("empty fluid domain")
    near = np.zeros_like(fluid)
    for axis in range(grid.dim):
        near |= np.roll(fluid, 1, axis)
        near |= np.roll(fluid, -1, axis)
    v_surf = int(np.count_nonzero(near & ~fluid))
    _, n_components = _labels32(grid, device)
    return GeometryStats(
        v_fluid=v_fluid,
        v_surf=v_surf,
        porosity_pct=100.0 * v_fluid / fluid.size,
        stv_pct=100.0 * v_surf / v_fluid,
        n_components=n_components,
    )


def periodize(grid: VoxelGrid) -> VoxelGrid:
    """Mirror across every axis, doubling the extent (geometry.py:243-255)."""
    fluid = grid.fluid
    for axis in range(grid.dim):
        fluid = np.concatenate([fluid, np.flip(fluid, axis=axis)], axis=axis)
    return VoxelGrid(fluid)


def _io_check(rc: int, path) -> None:
    if rc == _lib.VS_EOS:
        err = int(_lib.lib.vs_last_error().decode())
        raise OSError(err, os.strerror(err), os.fspath(path))
    if rc == _lib.VS_EDECODE:
        # the reference fails while decoding the file: raise that exact error
        with open(path, "r", encoding="utf-8", newline="") as handle:
            handle.read()
        raise ValueError("file is not valid UTF-8")
    _lib.check(rc)


def read_grid(path) -> VoxelGrid:
    """Parse a voxgeo file (geometry.py:271-317) in vs_io.cpp.

    Same accepted files, same ValueError messages (line/column info)."""
    p = os.fsencode(path)
    dim, n = C.c_int(), C.c_int64()
    fluid = None
    if _lib.lib.vs_grid_header(p, C.byref(dim), C.byref(n)) == _lib.VS_OK:
        fluid = np.empty((n.value,) * dim.value, dtype=np.uint8)
        rc = _lib.lib.vs_read_grid(p, _lib.ptr(fluid), fluid.size, C.byref(dim), C.byref(n))
    else:  # the full read produces the reference's error for this file
        rc = _lib.lib.vs_read_grid(p, None, 0, C.byref(dim), C.byref(n))
        if rc == _lib.VS_OK:
            fluid = np.empty((n.value,) * dim.value, dtype=np.uint8)
            rc = _lib.lib.vs_read_grid(p, _lib.ptr(fluid), fluid.size, C.byref(dim), C.byref(n))
    _io_check(rc, path)
    return VoxelGrid(fluid.view(bool))


def write_grid(grid: VoxelGrid, path) -> None:
    """Write the reference's voxgeo bytes (geometry.py:258-268) from C++."""
    f = np.ascontiguousarray(grid.fluid, dtype=np.uint8)
    _io_check(_lib.lib.vs_write_grid(os.fsencode(path), _lib.ptr(f), grid.dim, grid.n), path)
