"""Dense spectra on the GPU (spectra.py) against the reference's own
analyze_spectrum / nev_formula_check outputs (tests/golden/io_cases.json,
``spectra``), modelled on the reference's test_spectra.py / test_cli.py."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2307_05266_b200 as vx
from paper_2307_05266_b200 import spectra as sp
from paper_2307_05266_b200.cli import main, read_csv_rows

with open(os.path.join(GOLDEN, "io_cases.json")) as _fh:
    GOLD = json.load(_fh)["spectra"]

# eigenvalues from a dense Cholesky/syevd vs the reference's sparse LU/LAPACK:
# both are backward-stable direct methods on an O(1)-scaled matrix
EIG_ATOL = 1e-10


def _grid(prm):
    return vx.generate_packing(vx.PackingParams(**prm))


# ----------------------------------------------------------------- CPU


@pytest.mark.parametrize("case", GOLD["analyze"], ids=lambda c: f"{c['params']}-{c['prec']}")
def test_classify_reproduces_reference_report(case):
    rep = sp.classify_eigenvalues(case["eigenvalues"], prec=case["prec"])
    assert rep.to_json_dict() == case["report"]


def test_classify_edge_cases():
    rep = sp.classify_eigenvalues([0.0, 0.0])
    assert rep.n_zero == 2 and rep.lambda_min_nonzero is None and rep.cond_eff is None
    assert rep.tau_null == 1e-10  # absolute fallback for an all-zero spectrum
    with pytest.raises(ValueError, match="empty spectrum"):
        sp.classify_eigenvalues([])


def test_mean_complement_basis():
    q = sp._mean_complement_basis(7)
    assert q.shape == (7, 6)
    assert np.allclose(q.T @ q, np.eye(6), atol=1e-14)
    assert np.allclose(q.T @ np.ones(7), 0.0, atol=1e-14)
    with pytest.raises(ValueError, match="at least 2"):
        sp._mean_complement_basis(1)


def test_eig_sym_validation():
    with pytest.raises(ValueError, match="square matrix"):
        sp.eig_sym(np.zeros((2, 3)))
    with pytest.raises(ValueError, match="not symmetric"):
        sp.eig_sym(np.array([[1.0, 2.0], [0.0, 1.0]]))


def test_report_writers(tmp_path):
    rep = sp.classify_eigenvalues([0.0, 0.5, 1.0])
    rep.write_json(tmp_path / "r.json")
    rep.write_csv(tmp_path / "r.csv")
    assert json.loads((tmp_path / "r.json").read_text()) == rep.to_json_dict()
    assert (tmp_path / "r.csv").read_text() == "index,eigenvalue\n0,0\n1,0.5\n2,1\n"


# ----------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["analyze"], ids=lambda c: f"{c['params']}-{c['prec']}")
def test_analyze_spectrum_vs_reference(case):
    rep = sp.analyze_spectrum(_grid(case["params"]), prec=case["prec"])
    want = case["report"]
    got = rep.to_json_dict()
    for key in ("prec", "m_p", "n_zero", "n_ev"):
        assert got[key] == want[key], key
    assert np.allclose(rep.eigenvalues, case["eigenvalues"], rtol=0, atol=EIG_ATOL)
    for key in ("lambda_min_nonzero", "lambda_max", "cond_eff", "tau_null"):
        assert abs(got[key] - want[key]) <= 1e-8 * abs(want[key]), key


@pytest.mark.gpu
def test_dense_schur_properties():
    s_ = vx.assemble(_grid(GOLD["analyze"][0]["params"]), 0, require_walls=False)
    s = sp.dense_schur(s_)
    assert np.array_equal(s, s.T)
    assert np.abs(s @ np.ones(s_.m_p)).max() < 1e-10  # S 1 = 0 (test_schur.py:84-88)
    # columns agree with the iterative apply_schur
    e = np.zeros(s_.m_p)
    e[3] = 1.0
    col, _ = vx.apply_schur(s_, e - e.mean(), 1e-13)
    assert np.allclose(s @ (e - e.mean()), col, atol=1e-9)
    with pytest.raises(ValueError, match="requires eps_A"):
        sp.dense_schur(s_, eps_A=1e-6)
    with pytest.raises(ValueError, match="dense cap exceeded"):
        sp.dense_schur(s_, cap=5)


@pytest.mark.gpu
def test_nev_formula_check_vs_reference():
    configs = [vx.PackingParams(N=n, n_c=nc, n_avg=4, n_min=2, seed=0) for n in (1, 2) for nc in (8, 12)]
    rows = sp.nev_formula_check(configs, seeds=[0, 1])
    assert [{k: (bool(v) if isinstance(v, (bool, np.bool_)) else int(v)) for k, v in r.items()}
            for r in rows] == GOLD["nev"]


@pytest.fixture()
def small_geom(tmp_path):
    path = tmp_path / "g.vox"
    assert main(["gen", "--N", "1", "--nc", "10", "--navg", "4", "--nmin", "2", "--seed", "7",
                 "-o", str(path)]) == 0
    return path


@pytest.mark.gpu
def test_spectrum_cli(small_geom, tmp_path, capsys):
    base = tmp_path / "spec"
    assert main(["spectrum", str(small_geom), "-o", str(base)]) == 0
    data = json.loads(capsys.readouterr().out)
    assert data["n_zero"] == 1
    rows = read_csv_rows(tmp_path / "spec.csv")
    assert len(rows) == data["m_p"]
    assert float(rows[-1]["eigenvalue"]) == pytest.approx(data["lambda_max"])


@pytest.mark.gpu
def test_spectrum_over_cap(small_geom, capsys):
    assert main(["spectrum", str(small_geom), "--cap", "5"]) == 1
    err = capsys.readouterr().err.strip()
    assert err.startswith("error: dense cap exceeded")
    assert "\n" not in err


@pytest.mark.gpu
def test_nev_check_cli(tmp_path, capsys):
    out = tmp_path / "nev.csv"
    assert main(["nev-check", "--N", "1", "--nc", "8", "--seeds", "0", "1", "-o", str(out)]) == 0
    assert "match 2/2" in capsys.readouterr().err
    rows = read_csv_rows(out)
    assert len(rows) == 2
    for row in rows:
        assert row["match"] == "true"
        assert int(row["n_ev_measured"]) == int(row["n_ev_formula"])
