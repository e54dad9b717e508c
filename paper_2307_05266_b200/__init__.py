"""B200-native drop-in for the `voxstokes` Schur-complement Stokes path.

Same public names as the reference package for the hot path
(geometry input type, assemble, the Krylov seam, the Schur driver);
every apply and solve runs in libvoxschur.so (sm_100a CUDA).
"""
from .geometry import (
    GeometryStats,
    PackingParams,
    VoxelGrid,
    connected_components,
    enforce_connectivity,
    generate_packing,
    periodize,
    read_grid,
    stats,
    write_grid,
)
from .krylov import PcgConfig, PcgResult, jacobi_prec, lanczos_condition_estimate, pcg
from .operators import DofMap, StaggeredSystem, assemble, axis_index, connect_ranks
from .schur import (
    TOLERANCE_PROFILES,
    SchurConfig,
    SolveReport,
    apply_schur,
    apply_simple_inverse,
    last_kernel_stats,
    permeability,
    profile_config,
    schur_rhs,
    solve_schur,
    solve_schur_concurrent,
    supplementary_condition_estimate,
)

__version__ = "0.1.0"

__all__ = [
    "VoxelGrid", "connected_components", "enforce_connectivity",
    "PcgConfig", "PcgResult", "jacobi_prec", "lanczos_condition_estimate", "pcg",
    "DofMap", "StaggeredSystem", "assemble", "axis_index", "connect_ranks",
    "TOLERANCE_PROFILES", "SchurConfig", "SolveReport", "apply_schur", "apply_simple_inverse",
    "last_kernel_stats", "permeability", "profile_config", "schur_rhs", "solve_schur",
    "solve_schur_concurrent", "supplementary_condition_estimate",
    "GeometryStats", "PackingParams", "generate_packing", "periodize", "read_grid", "stats",
    "write_grid",
    "__version__",
]
