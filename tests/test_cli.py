"""The CLI on the GPU backend, modelled on the reference's test_cli.py, with
the reference CLI's own outputs (tests/golden/io_cases.json, ``cli``) as
the parity target: iteration counts exact or within the +-2 % bar, values
within 1e-8 relative."""
import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

from paper_2307_05266_b200.cli import main, read_csv_rows

with open(os.path.join(GOLDEN, "io_cases.json")) as _fh:
    GOLD = json.load(_fh)["cli"]


def run_cli(argv):
    return main(list(argv))


@pytest.fixture()
def small_geom(tmp_path):
    path = tmp_path / "g.vox"
    assert run_cli(["gen", "--N", "1", "--nc", "10", "--navg", "4", "--nmin", "2", "--seed", "7",
                    "-o", str(path)]) == 0
    return path


def close(a, b, rtol=1e-8):
    a, b = float(a), float(b)
    return abs(a - b) <= rtol * max(abs(a), abs(b), 1e-300)


def counts_close(a, b):
    a, b = int(a), int(b)
    return abs(a - b) <= max(1, round(0.02 * b))


# ----------------------------------------------------------------- CPU


def test_gen_stats_full_scale(tmp_path, capsys):
    geom = tmp_path / "g.vox"
    assert run_cli(["gen", "--N", "7", "--nc", "50", "--navg", "4", "--nmin", "2", "--seed", "42",
                    "-o", str(geom)]) == 0
    capsys.readouterr()
    out = tmp_path / "s.json"
    assert run_cli(["stats", str(geom), "-o", str(out)]) == 0
    data = json.loads(capsys.readouterr().out)
    assert data["porosity_pct"] == pytest.approx(15.36, abs=1e-12)
    assert data["n_components"] == 1
    assert set(data) == {"v_fluid", "v_surf", "porosity_pct", "stv_pct", "n_components"}
    assert json.loads(out.read_text()) == data


def test_missing_file_error(capsys):
    assert run_cli(["stats", "does-not-exist.vox"]) == 1
    err = capsys.readouterr().err.strip()
    assert err == "error: [Errno 2] No such file or directory: 'does-not-exist.vox'"


def test_invalid_params_error(tmp_path, capsys):
    assert run_cli(["gen", "--N", "1", "--nc", "10", "--navg", "3", "--nmin", "2",
                    "-o", str(tmp_path / "g.vox")]) == 1
    assert capsys.readouterr().err == "error: n_avg must be even, got 3\n"


def test_malformed_geometry_error(tmp_path, capsys):
    path = tmp_path / "bad.vox"
    path.write_text("voxgeo 1\ndim 2\nsize 2\n01\n0x\n")
    assert run_cli(["stats", str(path)]) == 1
    assert capsys.readouterr().err == "error: line 5, column 2: non-binary voxel symbol 'x'\n"


def test_module_entry_point():
    env = dict(os.environ, PYTHONPATH=ROOT)
    proc = subprocess.run([sys.executable, "-m", "paper_2307_05266_b200", "stats", "missing.vox"],
                          capture_output=True, text=True, env=env)
    assert proc.returncode == 1
    assert proc.stderr.startswith("error:")


# ----------------------------------------------------------------- GPU


def _check_report(got: dict, want: dict):
    assert got["converged"] == want["converged"]
    assert got["iters_outer"] == want["iters_outer"]
    for k, v in want["inner_iter_totals"].items():
        assert counts_close(got["inner_iter_totals"][k], v), (k, got["inner_iter_totals"], v)
    assert close(got["k_value"], want["k_value"])
    for key in ("perm_history",):
        assert len(got[key]) == len(want[key])
        assert all(close(a, b) for a, b in zip(got[key], want[key]))
    assert got["config"] == want["config"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD["solve"]))
def test_solve_matches_reference_cli(name, small_geom, tmp_path, capsys):
    case = GOLD["solve"][name]
    base = tmp_path / "rep"
    assert run_cli(["solve", str(small_geom), *case["argv"], "-o", str(base)]) == 0
    stdout = json.loads(capsys.readouterr().out)
    _check_report(stdout, case["report"])
    on_disk = json.loads((tmp_path / "rep.json").read_text())
    assert on_disk["k_value"] == stdout["k_value"]
    lines = (tmp_path / "rep.csv").read_text().strip().split("\n")
    assert lines[0] == "iter,res_prec,res_unprec,k,e_k"
    assert len(lines) == stdout["iters_outer"] + 2


@pytest.mark.gpu
def test_solve_csv_reruns_byte_identical(small_geom, tmp_path, capsys):
    for name in ("a", "b"):
        assert run_cli(["solve", str(small_geom), "--prec", "uzawa", "--eps-s", "1e-3", "--norm",
                        "unprec", "--eps-a", "1e-13", "-o", str(tmp_path / name)]) == 0
    capsys.readouterr()
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()


def sweep_args(out_dir, jobs):
    return [*GOLD["sweep"]["argv"][:-2], "--jobs", str(jobs), "-o", str(out_dir)]


def drop_time_column(path):
    rows = read_csv_rows(path)
    for row in rows:
        row.pop("time", None)
    return rows


@pytest.mark.gpu
def test_sweep_matches_reference(tmp_path, capsys):
    out = tmp_path / "sweep1"
    assert run_cli(sweep_args(out, jobs=1)) == 0
    capsys.readouterr()
    summary = drop_time_column(out / "summary.csv")
    want = GOLD["sweep"]["summary"]
    assert [(r["n_avg"], r["prec"], r["status"]) for r in summary] == \
        [(r["n_avg"], r["prec"], r["status"]) for r in want]
    for got, ref in zip(summary, want):
        assert got["stv_pct"] == ref["stv_pct"]
        assert counts_close(got["iters"], ref["iters"])
        assert close(got["k_final"], ref["k_final"])
        assert close(got["cond_est"], ref["cond_est"], 1e-6)
        assert close(got["e_final"], ref["e_final"], 1e-4)  # a difference of two close k's
    thresholds = read_csv_rows(out / "thresholds.csv")
    assert len(thresholds) == len(GOLD["sweep"]["thresholds"]) == 12
    for got, ref in zip(thresholds, GOLD["sweep"]["thresholds"]):
        assert (got["n_avg"], got["threshold"], got["prec"], got["norm_kind"], got["iter"]) == \
            (ref["n_avg"], ref["threshold"], ref["prec"], ref["norm_kind"], ref["iter"])
        if ref["k_at_threshold"]:
            assert close(got["k_at_threshold"], ref["k_at_threshold"])
    correlation = read_csv_rows(out / "correlation.csv")
    assert len(correlation) == 2
    for got, ref in zip(correlation, GOLD["sweep"]["correlation"]):
        assert got["stv_pct"] == ref["stv_pct"]
        assert close(got["cond_S"], ref["cond_S"], 1e-6)
        assert close(got["cond_precond"], ref["cond_precond"], 1e-6)
    for name in ("navg4_uzawa.json", "navg6_simple.csv", "navg4_reference.json"):
        assert (out / name).exists()


@pytest.mark.gpu
def test_sweep_deterministic_and_parallel(tmp_path, capsys):
    out1, out2, out3 = (tmp_path / f"s{i}" for i in (1, 2, 3))
    assert run_cli(sweep_args(out1, jobs=1)) == 0
    assert run_cli(sweep_args(out2, jobs=1)) == 0
    assert run_cli(sweep_args(out3, jobs=2)) == 0
    capsys.readouterr()
    for other in (out2, out3):
        assert drop_time_column(out1 / "summary.csv") == drop_time_column(other / "summary.csv")
        for name in ("thresholds.csv", "correlation.csv"):
            assert (out1 / name).read_bytes() == (other / name).read_bytes()
