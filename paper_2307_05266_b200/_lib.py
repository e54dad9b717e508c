"""ctypes binding of libvoxschur.so (include/voxschur.h).

This is the reference-side binding a maintainer of ``voxstokes`` would add
(INTEGRATION.md).  There is no CPU fallback: if the library is missing the
import fails loudly, and if no CUDA device is present every compute call
raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VOXSCHUR_LIB", os.path.join(_HERE, "libvoxschur.so"))

VS_OK, VS_EVALUE, VS_ERUNTIME, VS_ECUDA, VS_EOS, VS_EDECODE = 0, 1, 2, 3, 4, 5


class VsReport(C.Structure):
    _fields_ = [
        ("k_value", C.c_double),
        ("iters_outer", C.c_int64),
        ("converged", C.c_int32),
        ("_pad", C.c_int32),
        ("inner_velocity", C.c_int64),
        ("inner_preconditioner", C.c_int64),
        ("uf_iters", C.c_int64),
        ("n_hist", C.c_int64),
        ("device_ms", C.c_double),
    ]


class VsSchurCfg(C.Structure):
    _fields_ = [
        ("prec", C.c_int32),
        ("outer_norm", C.c_int32),
        ("eps_S", C.c_double),
        ("eps_A", C.c_double),
        ("eps_Shat", C.c_double),
        ("max_iter", C.c_int64),
        ("h_pow_dim", C.c_double),
    ]


class VsKstat(C.Structure):
    _fields_ = [
        ("launches", C.c_int64),
        ("iterations", C.c_int64),
        ("dof_iters", C.c_int64),
        ("ms", C.c_double),
        ("kernel", C.c_int32),
        ("reserved", C.c_int32),
        ("tier", C.c_int32),
        ("escape_ppm", C.c_int32),
    ]


class CudaError(RuntimeError):
    """A device or driver failure (not a reference-level error)."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c \"import __graft_entry__ as g; g.build()\"` "
            "(make -C paper_2307_05266_b200/csrc). There is no CPU fallback."
        )
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
    u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
    i64p = C.POINTER(C.c_int64)
    sig = {
        "vs_last_error": (C.c_char_p, []),
        "vs_version": (C.c_char_p, []),
        "vs_components": (C.c_int, [u8, C.c_int, C.c_int, P, i64p]),
        "vs_components_device": (C.c_int, [u8, C.c_int, C.c_int, C.c_int, P, i64p]),
        "vs_winding": (C.c_int, [u8, C.c_int, C.c_int, C.c_int, i64p, i64p]),
        "vs_stamp_balls": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_int64, C.c_int64, C.c_int,
                                     i64p, i64p]),
        "vs_ctx_create": (C.c_int, [u8, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_double, C.c_double, C.POINTER(P)]),
        "vs_ctx_create2": (C.c_int, [u8, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_double, C.c_int, C.POINTER(P)]),
        "vs_slab_count": (C.c_int, [P]),
        "vs_ctx_limit_sms": (C.c_int, [P, C.c_int]),
        "vs_ctx_sms": (C.c_int, [P]),
        "vs_solve_span_ms": (C.c_int, [P, P, C.POINTER(C.c_double)]),
        "vs_slab_plan": (C.c_int, [u8, C.c_int, C.c_int, C.c_int, P]),
        "vs_ctx_create_rank": (C.c_int, [u8, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(P)]),
        "vs_ipc_handle": (C.c_int, [P, P]),
        "vs_ipc_attach": (C.c_int, [P, P]),
        "vs_ctx_destroy": (None, [P]),
        "vs_counts": (C.c_int, [P, i64p, i64p, i64p]),
        "vs_export_geometry": (C.c_int, [P, P, P, P, P, P]),
        "vs_apply_laplacian": (C.c_int, [P, dp, dp]),
        "vs_apply_divergence": (C.c_int, [P, dp, dp]),
        "vs_apply_gradient": (C.c_int, [P, dp, dp]),
        "vs_divergence_weighted_diagonal": (C.c_int, [P, dp, dp]),
        "vs_apply_simple": (C.c_int, [P, dp, dp]),
        "vs_solve_velocity": (C.c_int, [P, dp, P, C.c_double, dp, i64p]),
        "vs_solve_simple": (C.c_int, [P, dp, C.c_double, dp, i64p]),
        "vs_solve_schur": (C.c_int, [P, C.POINTER(VsSchurCfg), P, P, C.POINTER(VsReport),
                                     P, P, P, P, P]),
        "vs_solve_schur_rhs": (C.c_int, [P, C.POINTER(VsSchurCfg), dp, P, P, C.POINTER(VsReport),
                                         P, P, P, P, P]),
        "vs_kernel_stats": (C.c_int, [P, C.POINTER(VsKstat), C.POINTER(VsKstat), i64p]),
        "vs_phase_timing": (C.c_int, [P, dp]),
        "vs_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "vs_grid_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), i64p]),
        "vs_read_grid": (C.c_int, [C.c_char_p, P, C.c_int64, C.POINTER(C.c_int), i64p]),
        "vs_write_grid": (C.c_int, [C.c_char_p, P, C.c_int, C.c_int64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)  # AttributeError here = the ABI is incomplete
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
EXPORTED = (
    "vs_last_error", "vs_version", "vs_components", "vs_components_device", "vs_winding", "vs_stamp_balls", "vs_ctx_create", "vs_ctx_create2", "vs_slab_count", "vs_ctx_limit_sms", "vs_ctx_sms", "vs_solve_span_ms", "vs_slab_plan", "vs_ctx_create_rank", "vs_ipc_handle", "vs_ipc_attach",
    "vs_ctx_destroy",
    "vs_counts", "vs_export_geometry", "vs_apply_laplacian", "vs_apply_divergence",
    "vs_apply_gradient", "vs_divergence_weighted_diagonal", "vs_apply_simple",
    "vs_solve_velocity", "vs_solve_simple", "vs_solve_schur", "vs_solve_schur_rhs", "vs_kernel_stats",
    "vs_phase_timing", "vs_device_count", "vs_grid_header", "vs_read_grid", "vs_write_grid",
)


def check(rc: int) -> None:
    """Map an ABI status to the exception type the reference raises."""
    if rc == VS_OK:
        return
    msg = lib.vs_last_error().decode()
    if rc == VS_EVALUE:
        raise ValueError(msg)
    if rc == VS_ERUNTIME:
        raise RuntimeError(msg)
    raise CudaError(msg)


def ptr(a) -> C.c_void_p:
    """Raw data pointer of a numpy array (or NULL for None)."""
    return None if a is None else C.c_void_p(a.ctypes.data)
