"""Device-backed staggered (MAC) system -- drop-in for operators.py.

``assemble`` (operators.py:209-302) validates on the host, then builds the
geometry on the GPU (vs_ctx_create: bit-packed fluid mask -> per-component
face bitmasks -> DOF ranks -> per-DOF records with the integer no-slip
codes).  ``StaggeredSystem`` exposes the reference's duck-typed surface
(operators.py:86-206): counts, ``dof_map``, ``laplacian_diag``, ``force``,
``h`` and the four applies, each a bitwise-equal CUDA kernel.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _lib
from .geometry import VoxelGrid

__all__ = ["DofMap", "StaggeredSystem", "assemble", "axis_index", "connect_ranks"]

_AXIS_NAMES = {"x": 0, "y": 1, "z": 2}


def axis_index(flow_dir, dim: int) -> int:
    """Normalize an axis given as 0/1/2 or 'x'/'y'/'z' (operators.py:48-58)."""
    if isinstance(flow_dir, str):
        try:
            flow_dir = _AXIS_NAMES[flow_dir.lower()]
        except KeyError:
            raise ValueError(f"unknown axis name {flow_dir!r}") from None
    flow_dir = int(flow_dir)
    if not 0 <= flow_dir < dim:
        raise ValueError(f"flow axis {flow_dir} out of range for dim {dim}")
    return flow_dir


@dataclass(frozen=True)
class DofMap:
    """Dense deterministic numbering (operators.py:61-83), rebuilt on the
    host from the device face masks."""

    face_ids: tuple
    pressure_ids: np.ndarray
    axis_counts: tuple
    axis_offsets: tuple
    m_u: int
    m_p: int

    def velocity_coords(self, axis: int) -> np.ndarray:
        return np.argwhere(self.face_ids[axis] >= 0)

    def pressure_coords(self) -> np.ndarray:
        return np.argwhere(self.pressure_ids >= 0)


class StaggeredSystem:
    """Matrix-free discrete Stokes operators resident on one GPU."""

    def __init__(self, grid: VoxelGrid, flow_dir: int, ctx, device: int):
        self.grid = grid
        self.flow_dir = flow_dir
        self.device = device
        self._ctx = ctx
        self.h = grid.physical_length / grid.n
        self._inv_h2 = 1.0 / self.h**2
        self._inv_h = 1.0 / self.h
        mu, mp = C.c_int64(), C.c_int64()
        ac = (C.c_int64 * 3)()
        _lib.check(_lib.lib.vs_counts(ctx, C.byref(mu), C.byref(mp), ac))
        self._m_u, self._m_p = int(mu.value), int(mp.value)
        self._axis_counts = tuple(int(ac[a]) for a in range(grid.dim))
        self._axis_offsets = tuple(sum(self._axis_counts[:a]) for a in range(grid.dim))
        force = np.zeros(self._m_u)
        lo = self._axis_offsets[flow_dir]
        force[lo : lo + self._axis_counts[flow_dir]] = 1.0
        force.setflags(write=False)
        self.force = force

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx:
            _lib.lib.vs_ctx_destroy(ctx)
            self._ctx = None

    @property
    def m_u(self) -> int:
        return self._m_u

    @property
    def m_p(self) -> int:
        return self._m_p

    # -------------------------------------------------------- geometry views
    def _export(self):
        n, dim = self.grid.n, self.grid.dim
        masks = [np.zeros((n,) * dim, dtype=np.uint8) for _ in range(dim)]
        pm = np.zeros((n,) * dim, dtype=np.uint8)
        codes = np.zeros(max(self._m_u, 1), dtype=np.uint8)
        m3 = [_lib.ptr(masks[a]) if a < dim else None for a in range(3)]
        _lib.check(_lib.lib.vs_export_geometry(self._ctx, m3[0], m3[1], m3[2], _lib.ptr(pm),
                                               _lib.ptr(codes)))
        return [m.astype(bool) for m in masks], pm.astype(bool), codes[: self._m_u]

    @cached_property
    def _geometry(self):
        return self._export()

    @cached_property
    def dof_map(self) -> DofMap:
        masks, pm, _ = self._geometry
        face_ids = []
        for a, mask in enumerate(masks):
            ids = np.full(mask.shape, -1, dtype=np.int64)
            ids[mask] = self._axis_offsets[a] + np.arange(self._axis_counts[a], dtype=np.int64)
            ids.setflags(write=False)
            face_ids.append(ids)
        pids = np.full(pm.shape, -1, dtype=np.int64)
        pids[pm] = np.arange(self._m_p, dtype=np.int64)
        pids.setflags(write=False)
        return DofMap(tuple(face_ids), pids, self._axis_counts, self._axis_offsets,
                      self._m_u, self._m_p)

    @cached_property
    def diag_codes(self) -> np.ndarray:
        """Integer no-slip codes per velocity DOF (laplacian_diag / n^2)."""
        return self._geometry[2].astype(np.int64)

    @cached_property
    def laplacian_diag(self) -> np.ndarray:
        inv_h2 = (self.grid.n / self.grid.physical_length) ** 2  # operators.py:260
        d = self.diag_codes.astype(float) * inv_h2
        d.setflags(write=False)
        return d

    # ---------------------------------------------------------------- applies
    def _check(self, vec, m, what):
        vec = np.ascontiguousarray(vec, dtype=float)
        if vec.shape != (m,):
            raise ValueError(f"{what} vector length mismatch: expected {m}, got {vec.shape}")
        return vec

    def _apply(self, fn, vec, m_in, m_out, what):
        vec = self._check(vec, m_in, what)
        out = np.empty(m_out)
        if m_in and m_out:
            _lib.check(fn(self._ctx, vec, out))
        elif m_out:
            out[:] = 0.0
        return out

    def apply_laplacian(self, u) -> np.ndarray:
        """Negative vector Laplacian with no-slip walls (operators.py:131-135)."""
        return self._apply(_lib.lib.vs_apply_laplacian, u, self._m_u, self._m_u, "velocity")

    def apply_divergence(self, u) -> np.ndarray:
        """Negative discrete divergence (operators.py:137-144)."""
        return self._apply(_lib.lib.vs_apply_divergence, u, self._m_u, self._m_p, "velocity")

    def apply_gradient(self, p) -> np.ndarray:
        """Pressure gradient on velocity faces (operators.py:146-153)."""
        return self._apply(_lib.lib.vs_apply_gradient, p, self._m_p, self._m_u, "pressure")

    def divergence_weighted_diagonal(self, face_weights) -> np.ndarray:
        """Diagonal of B W B^T (operators.py:194-206)."""
        return self._apply(_lib.lib.vs_divergence_weighted_diagonal, face_weights,
                           self._m_u, self._m_p, "face weight")

    def limit_sms(self, sms: int) -> None:
        """Plan this system's fused inner solves on ``sms`` SMs (0 = all).

        For independent solves on separate systems that run concurrently
        (``solve_schur_concurrent``); no reference counterpart."""
        _lib.check(_lib.lib.vs_ctx_limit_sms(self._ctx, int(sms)))

    @property
    def sms(self) -> int:
        """SMs the fused inner solves are planned on."""
        return int(_lib.lib.vs_ctx_sms(self._ctx))

    def apply_simple(self, p) -> np.ndarray:
        """B diag(A)^-1 B^T p in one kernel (schur.py:234-240)."""
        return self._apply(_lib.lib.vs_apply_simple, p, self._m_p, self._m_p, "pressure")


def _default_device() -> int:
    return int(os.environ.get("VOXSCHUR_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def assemble(grid: VoxelGrid, flow_dir=0, *, check_connectivity: bool = True,
             require_walls: bool = True, device: int | None = None,
             slabs: int = 1, rank: int | None = None, nranks: int = 1) -> StaggeredSystem:
    """Build the staggered operators for a voxel grid on the GPU.

    Same signature and errors as operators.py:209-230 plus the backend
    selectors ``device`` (default $VOXSCHUR_DEVICE, else $LOCAL_RANK, else 0)
    and ``slabs``: decompose into that many x-slabs (ranks) with ghost-plane
    exchange inside the fused solver; on one device the
    ranks run as groups of one cooperative grid.  With ``rank``/``nranks``
    (one process per GPU) this process holds only slab ``rank``; call
    ``connect_ranks`` on every rank before solving.
    """
    if not isinstance(grid, VoxelGrid):
        grid = VoxelGrid(np.asarray(grid))
    flow_dir = axis_index(flow_dir, grid.dim)
    dev = _default_device() if device is None else int(device)
    h = grid.physical_length / grid.n
    ctx = C.c_void_p()
    fl = np.ascontiguousarray(grid.fluid, dtype=np.uint8).ravel()
    if rank is not None and nranks > 1:
        _lib.check(_lib.lib.vs_ctx_create_rank(fl, grid.dim, grid.n, flow_dir, int(check_connectivity),
                                               int(require_walls), dev, 1.0 / h, 1.0 / h**2, int(rank),
                                               int(nranks), C.byref(ctx)))
    else:
        _lib.check(_lib.lib.vs_ctx_create2(fl, grid.dim, grid.n, flow_dir, int(check_connectivity),
                                           int(require_walls), dev, 1.0 / h, 1.0 / h**2, int(slabs),
                                           C.byref(ctx)))
    sys_ = StaggeredSystem(grid, flow_dir, ctx, dev)
    sys_.rank, sys_.nranks = (int(rank), int(nranks)) if rank is not None else (0, 1)
    return sys_


def connect_ranks(sys_: StaggeredSystem, group=None) -> None:
    """Map every rank's slab into this process (CUDA IPC over NVLink).

    Collective over the ``torch.distributed`` group: each rank contributes
    its 64-byte arena handle; afterwards the fused solver exchanges ghost
    planes and reduction partials through peer memory.
    """
    import torch.distributed as dist

    h = (C.c_char * 64)()
    _lib.check(_lib.lib.vs_ipc_handle(sys_._ctx, h))
    handles = [None] * sys_.nranks
    dist.all_gather_object(handles, bytes(h), group=group)
    blob = b"".join(handles)
    _lib.check(_lib.lib.vs_ipc_attach(sys_._ctx, blob))
