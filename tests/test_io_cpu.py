"""voxgeo IO (vs_io.cpp), the packing generator and stats against the
reference's own outputs (tests/golden/io_cases.json, made by
tests/golden/make_io_golden.py from the reference package).  Host code
only: runs without a GPU."""
import base64
import dataclasses
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2307_05266_b200 as vx
from paper_2307_05266_b200 import geometry as G

with open(os.path.join(GOLDEN, "io_cases.json")) as _fh:
    CASES = json.load(_fh)


@pytest.mark.parametrize("case", CASES["read"], ids=lambda c: c["name"])
def test_read_grid_matches_reference(case, tmp_path):
    path = tmp_path / "g.vox"
    path.write_bytes(base64.b64decode(case["data_b64"]))
    if case["ok"]:
        grid = G.read_grid(path)
        assert list(grid.fluid.shape) == case["shape"]
        assert np.packbits(grid.fluid.ravel()).tobytes().hex() == case["bits"]
    else:
        with pytest.raises(Exception) as info:
            G.read_grid(path)
        assert type(info.value).__name__ == case["type"]
        assert str(info.value) == case["message"]


def test_read_missing_file():
    with pytest.raises(FileNotFoundError) as info:
        G.read_grid("does-not-exist.vox")
    assert str(info.value) == "[Errno 2] No such file or directory: 'does-not-exist.vox'"


@pytest.mark.parametrize("case", CASES["packing"], ids=lambda c: str(c["params"]))
def test_packing_stats_and_file_bytes(case, tmp_path):
    grid = G.generate_packing(G.PackingParams(**case["params"]))
    assert hashlib.sha256(np.ascontiguousarray(grid.fluid).tobytes()).hexdigest() == case["mask_sha256"]
    assert dataclasses.asdict(G.stats(grid)) == case["stats"]
    path = tmp_path / "g.vox"
    G.write_grid(grid, path)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == case["file_sha256"]
    back = G.read_grid(path)
    assert np.array_equal(back.fluid, grid.fluid)


@pytest.mark.parametrize("case", CASES["packing_rejected"], ids=lambda c: str(c["params"]))
def test_packing_params_rejections(case):
    with pytest.raises(ValueError) as info:
        G.PackingParams(**case["params"])
    assert str(info.value) == case["message"]


@pytest.mark.parametrize("n,dim", [(2, 2), (3, 3), (65, 2), (130, 3)])
def test_write_read_round_trip(n, dim, tmp_path):
    """Ragged tile edges (n not a multiple of the 64-column tile) and the
    threaded path (130^3 > 2^20 symbols) round-trip bitwise."""
    rng = np.random.default_rng(n)
    fluid = rng.random((n,) * dim) < 0.5
    path = tmp_path / "g.vox"
    G.write_grid(vx.VoxelGrid(fluid), path)
    lines = path.read_bytes().split(b"\n")
    assert lines[:3] == [b"voxgeo 1", f"dim {dim}".encode(), f"size {n}".encode()]
    # the file is x fastest, then y, then z (geometry.py:258-268)
    row = 1 if dim == 2 else n + 1  # (y=1) or (y=1, z=1)
    idx = (slice(None), 1) if dim == 2 else (slice(None), 1, 1)
    assert lines[3 + row] == "".join("1" if v else "0" for v in fluid[idx]).encode()
    assert np.array_equal(G.read_grid(path).fluid, fluid)


def test_periodize():
    fluid = np.zeros((3, 3), dtype=bool)
    fluid[0, 1] = True
    g = G.periodize(vx.VoxelGrid(fluid))
    assert g.n == 6 and g.fluid[0, 1] and g.fluid[5, 1] and g.fluid[0, 4] and g.fluid[5, 4]
    assert g.fluid.sum() == 4
