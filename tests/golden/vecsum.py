"""Size-independent summaries of a solution vector, shared by the fixture
generator (make_config_golden.py) and the GPU parity tests.

At 256^3 and above the full p and u are too large to commit, so a fixture
keeps: the 2-norm, NPROJ seeded random projections, and a fixed sample of
entries (evenly spaced plus both ends).  For a random w the projection
w.e has variance |e|^2, so the rms of the projection differences estimates
|v_gpu - v_ref| itself.
"""
from __future__ import annotations

import numpy as np

NSAMPLE = 4096
NEDGE = 512


def sample_index(m: int) -> np.ndarray:
    idx = np.concatenate([
        np.linspace(0, m - 1, NSAMPLE).astype(np.int64),
        np.arange(min(NEDGE, m), dtype=np.int64),
        np.arange(max(0, m - NEDGE), m, dtype=np.int64),
    ])
    return np.unique(idx)


def projections(v: np.ndarray, nproj: int, seed0: int = 1000) -> np.ndarray:
    out = np.empty(nproj)
    for j in range(nproj):
        w = np.random.default_rng(seed0 + j).standard_normal(v.shape[0])
        out[j] = float(w @ v)
    return out


def summarize(prefix: str, v: np.ndarray, nproj: int, rec: dict, full: bool = False) -> None:
    v = np.asarray(v, dtype=np.float64)
    rec[prefix + "_norm"] = float(np.sqrt(v @ v))
    rec[prefix + "_sum"] = float(v.sum())
    rec[prefix + "_proj"] = projections(v, nproj)
    rec[prefix + "_sample"] = v[sample_index(v.shape[0])]
    if full:
        rec[prefix + "_full"] = v


def compare(prefix: str, v: np.ndarray, rec, rtol: float = 1e-8) -> dict:
    """Relative differences of ``v`` against the fixture's summary of the
    reference vector; raises AssertionError when any exceeds ``rtol``."""
    v = np.asarray(v, dtype=np.float64)
    norm = float(rec[prefix + "_norm"])
    scale = norm if norm > 0 else 1.0
    out = {}
    out["norm"] = abs(float(np.sqrt(v @ v)) - norm) / scale
    ref_proj = np.asarray(rec[prefix + "_proj"])
    dp = projections(v, len(ref_proj)) - ref_proj
    out["proj_rms"] = float(np.sqrt(np.mean(dp * dp))) / scale
    idx = sample_index(v.shape[0])
    ref_s = np.asarray(rec[prefix + "_sample"])
    ds = v[idx] - ref_s
    s_scale = float(np.sqrt(ref_s @ ref_s))
    out["sample"] = float(np.sqrt(ds @ ds)) / (s_scale if s_scale > 0 else 1.0)
    if prefix + "_full" in rec:
        ref = np.asarray(rec[prefix + "_full"])
        out["full"] = float(np.linalg.norm(v - ref)) / scale
    bad = {k: x for k, x in out.items() if not x <= rtol}
    assert not bad, f"{prefix}: relative difference above {rtol:g}: {bad} (all: {out})"
    return out
