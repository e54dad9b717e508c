"""Golden vectors for the voxgeo IO, the packing generator, stats and the
CLI report formats, made by running the REFERENCE package itself.

Run inside the build container (where /root/reference exists):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_io_golden.py

Writes ``tests/golden/io_cases.json``:

* ``read``: voxgeo file contents (valid and malformed: header, counts,
  trailing content, lengths, symbols, CRLF, non-ASCII, invalid UTF-8,
  underscores/signs in header integers) with what the reference's
  ``read_grid`` returned — the mask as a hex bit string, or the exception
  type and message;
* ``packing``: ``generate_packing`` masks (sha256 of the bool bytes) and
  ``stats`` for a few parameter sets, plus ``PackingParams`` rejections;
* ``write``: sha256 of ``write_grid``'s bytes for those packings.

Nothing under tests/ reads /root/reference at run time.
"""
from __future__ import annotations

import base64
import dataclasses
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from voxstokes.geometry import (  # noqa: E402
    PackingParams, VoxelGrid, generate_packing, read_grid, stats, write_grid,
)

H = "voxgeo 1\n"


def grid_text(fluid):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.vox")
        write_grid(VoxelGrid(fluid), p)
        with open(p, "rb") as f:
            return f.read()


def read_cases():
    rng = np.random.default_rng(5)
    f2 = rng.random((6, 6)) < 0.5
    f3 = rng.random((5, 5, 5)) < 0.5
    good2, good3 = grid_text(f2), grid_text(f3)
    lines3 = good3.split(b"\n")
    c = {
        "valid2d": good2,
        "valid3d": good3,
        "valid3d_no_final_newline": good3.rstrip(b"\n"),
        "valid3d_trailing_blank_lines": good3 + b"\n\n\n",
        "header_spaces": good3.replace(b"dim 3\n", b"  dim \t 3 \n").replace(b"size 5", b"size\t+0_5"),
        "empty": b"",
        "bad_magic": good3.replace(b"voxgeo 1", b"voxgeo 2"),
        "magic_crlf": good3.replace(b"voxgeo 1\n", b"voxgeo 1\r\n"),
        "missing_dim": b"voxgeo 1",
        "missing_size": b"voxgeo 1\ndim 3",
        "dim_wrong_key": H.encode() + b"dims 3\nsize 5\n",
        "dim_three_parts": H.encode() + b"dim 3 3\nsize 5\n",
        "dim_not_int": H.encode() + b"dim 3x\nsize 5\n",
        "dim_quote": H.encode() + b"dim 3'\nsize 5\n",
        "dim_4": H.encode() + b"dim 4\nsize 5\n",
        "dim_neg0": H.encode() + b"dim -0\nsize 5\n",
        "size_1": H.encode() + b"dim 2\nsize 1\n",
        "size_neg": H.encode() + b"dim 2\nsize -007\n",
        "size_double_underscore": H.encode() + b"dim 2\nsize 1__0\n",
        "size_huge": H.encode() + b"dim 3\nsize 123456789012345678901234\n0101\n",
        "size_big_short": H.encode() + b"dim 3\nsize 1048576\n0101\n",
        "size_short_2d": H.encode() + b"dim 2\nsize 3\n010\n",
        "too_few_lines": b"\n".join(lines3[:10]) + b"\n",
        "empty_data_line": b"\n".join(lines3[:5] + [b""] + lines3[6:]),
        "trailing_content": good3 + b"junk\n",
        "trailing_after_blank": good3 + b"\n\n0\n",
        "short_line": b"\n".join(lines3[:7] + [lines3[7][:-1]] + lines3[8:]),
        "long_line": b"\n".join(lines3[:7] + [lines3[7] + b"1"] + lines3[8:]),
        "bad_symbol": b"\n".join(lines3[:8] + [lines3[8][:2] + b"x" + lines3[8][3:]] + lines3[9:]),
        "bad_symbol_backslash": b"\n".join(lines3[:8] + [b"\\" + lines3[8][1:]] + lines3[9:]),
        "bad_symbol_tab": b"\n".join(lines3[:8] + [lines3[8][:4] + b"\t"] + lines3[9:]),
        "bad_symbol_quote": b"\n".join(lines3[:8] + [lines3[8][:4] + b"'"] + lines3[9:]),
        "bad_symbol_ctrl": b"\n".join(lines3[:8] + [lines3[8][:4] + b"\x1b"] + lines3[9:]),
        "crlf_data": good3.replace(b"\n", b"\r\n").replace(b"voxgeo 1\r\n", b"voxgeo 1\n"),
        "non_ascii_symbol": b"\n".join(lines3[:8] + [lines3[8][:3] + "é".encode() + lines3[8][4:]] + lines3[9:]),
        "non_ascii_nbsp": b"\n".join(lines3[:8] + [lines3[8][:3] + " ".encode() + lines3[8][4:]] + lines3[9:]),
        "non_ascii_long": b"\n".join(lines3[:8] + [lines3[8] + "é".encode()] + lines3[9:]),
        "bad_after_short": b"\n".join(lines3[:5] + [b"0x000"] + lines3[6:8] + [b"0"] + lines3[9:]),
        "invalid_utf8": good3.replace(lines3[6], b"\xff" + lines3[6][1:]),
        "bom": b"\xef\xbb\xbf" + good3,
    }
    out = []
    for name, data in c.items():
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "g.vox")
            with open(p, "wb") as fh:
                fh.write(data)
            try:
                g = read_grid(p)
                res = {"ok": True, "shape": list(g.fluid.shape),
                       "bits": np.packbits(g.fluid.ravel()).tobytes().hex()}
            except Exception as exc:  # noqa: BLE001
                res = {"ok": False, "type": type(exc).__name__, "message": str(exc)}
        out.append({"name": name, "data_b64": base64.b64encode(data).decode(), **res})
    return out


def packing_cases():
    params = [
        dict(N=7, n_c=50, n_avg=4, n_min=2, seed=42),
        dict(N=2, n_c=10, n_avg=6, n_min=2, seed=3),
        dict(N=1, n_c=10, n_avg=4, n_min=2, seed=7),
        dict(N=3, n_c=12, n_avg=4, n_min=2, seed=11, dim=3),
        dict(N=2, n_c=9, n_avg=6, n_min=2, seed=2**64 - 1, dim=3),
    ]
    out = []
    for prm in params:
        g = generate_packing(PackingParams(**prm))
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "g.vox")
            write_grid(g, p)
            with open(p, "rb") as fh:
                file_sha = hashlib.sha256(fh.read()).hexdigest()
        out.append({
            "params": prm,
            "mask_sha256": hashlib.sha256(np.ascontiguousarray(g.fluid).tobytes()).hexdigest(),
            "stats": dataclasses.asdict(stats(g)),
            "file_sha256": file_sha,
        })
    bad = [
        dict(N=1, n_c=10, n_avg=3, n_min=2, seed=0),
        dict(N=0, n_c=10, n_avg=4, n_min=2, seed=0),
        dict(N=1, n_c=4, n_avg=4, n_min=2, seed=0),
        dict(N=1, n_c=10, n_avg=4, n_min=1, seed=0),
        dict(N=1, n_c=10, n_avg=4, n_min=6, seed=0),
        dict(N=1, n_c=10, n_avg=4, n_min=0, seed=0),
        dict(N=1, n_c=10, n_avg=4, n_min=2, seed=-1),
        dict(N=1, n_c=10, n_avg=4, n_min=2, seed=0, dim=4),
    ]
    rej = []
    for prm in bad:
        try:
            PackingParams(**prm)
            rej.append({"params": prm, "message": None})
        except ValueError as exc:
            rej.append({"params": prm, "message": str(exc)})
    return out, rej


def cli_cases():
    """The reference CLI's sweep and solve outputs on the sizes its own
    tests use (test_cli.py:17-25, :155-160); the ``time`` column and
    ``wall_time`` are dropped."""
    from voxstokes.cli import main as ref_main, read_csv_rows

    out = {}
    with tempfile.TemporaryDirectory() as d:
        g = os.path.join(d, "g.vox")
        assert ref_main(["gen", "--N", "1", "--nc", "10", "--navg", "4", "--nmin", "2",
                         "--seed", "7", "-o", g]) == 0
        solves = {}
        for name, extra in (("simple_paper2d", ["--prec", "simple", "--profile", "paper2d"]),
                            ("uzawa_unprec", ["--prec", "uzawa", "--eps-s", "1e-3", "--norm",
                                              "unprec", "--eps-a", "1e-13"])):
            base = os.path.join(d, name)
            assert ref_main(["solve", g, *extra, "-o", base]) == 0
            with open(base + ".json") as fh:
                rep = json.load(fh)
            rep.pop("wall_time")
            solves[name] = {"argv": extra, "report": rep}
        out["solve"] = solves
        sd = os.path.join(d, "sweep")
        argv = ["sweep", "--N", "2", "--nc", "10", "--nmin", "2", "--navg", "4", "6", "--seed",
                "3", "--prec", "both", "--profile", "paper2d", "--jobs", "1", "-o", sd]
        assert ref_main(argv) == 0
        sweep = {"argv": argv[:-2]}
        for name in ("summary", "thresholds", "correlation"):
            rows = read_csv_rows(os.path.join(sd, f"{name}.csv"))
            for row in rows:
                row.pop("time", None)
            sweep[name] = rows
        out["sweep"] = sweep
    return out


def spectra_cases():
    """analyze_spectrum (both pencils) and nev_formula_check of the
    reference on desk-scale packings (spectra.py:203-262)."""
    from voxstokes.spectra import analyze_spectrum, nev_formula_check

    out = {"analyze": [], "nev": []}
    for prm in (dict(N=1, n_c=10, n_avg=4, n_min=2, seed=7),
                dict(N=2, n_c=8, n_avg=4, n_min=2, seed=1),
                dict(N=1, n_c=8, n_avg=4, n_min=2, seed=3, dim=3)):
        grid = generate_packing(PackingParams(**prm))
        for prec in ("none", "simple"):
            rep = analyze_spectrum(grid, prec=prec)
            out["analyze"].append({"params": prm, "prec": prec, "report": rep.to_json_dict(),
                                   "eigenvalues": [float(v) for v in rep.eigenvalues]})
    configs = [PackingParams(N=n, n_c=nc, n_avg=4, n_min=2, seed=0) for n in (1, 2) for nc in (8, 12)]
    for row in nev_formula_check(configs, seeds=[0, 1]):
        out["nev"].append({k: (bool(v) if isinstance(v, (bool, np.bool_)) else int(v))
                           for k, v in row.items()})
    return out


def main():
    packing, rejected = packing_cases()
    doc = {"read": read_cases(), "packing": packing, "packing_rejected": rejected,
           "cli": cli_cases(), "spectra": spectra_cases()}
    with open(os.path.join(HERE, "io_cases.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")
    print(f"{len(doc['read'])} read cases, {len(packing)} packings")


if __name__ == "__main__":
    main()
