"""Voxel geometry input type and periodic connectivity (host side).

``VoxelGrid`` mirrors geometry.py:29-66 (validation and immutability);
``connected_components`` / ``enforce_connectivity`` mirror
geometry.py:183-240 and run in the native library (vs_components, a
periodic union-find in C++).  Generators, stats and the voxgeo text IO of
the reference are outside this repository's hot-path scope.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["VoxelGrid", "connected_components", "enforce_connectivity"]


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
