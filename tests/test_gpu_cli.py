"""The CLI end to end on the GPU against the reference CLI's own outputs
(make_golden.py cli): `fit` (rank-only: GLM-SVD start, aSGD, B1) writes the
same factors and report, exit 3 for max_epochs without convergence;
`cv --criterion scree` the same eigenvalues and pick; `eval` metrics."""
import numpy as np
import pytest

from conftest import golden, normwise

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")


@pytest.fixture(autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_cli_fit_and_scree_match_reference(tmp_path):
    from paper_2412_20509_b200 import cli
    from paper_2412_20509_b200 import io as gio
    g = golden("cli")
    ycsv = tmp_path / "y.csv"
    gio.write_dense_csv(ycsv, g["y"].astype(float))
    rc = cli.main(["fit", "--y", str(ycsv), "--rank", "2", "--family", "neg_binomial",
                   "--nb-shape", "1.5", "--max-epochs", "15", "--mb-rows", "40", "--mb-cols", "40",
                   "--tol", "1e-30", "--out", str(tmp_path / "fit")])
    assert rc == int(g["fit_rc"]) == 3
    u = gio.read_dense_csv(tmp_path / "fit" / "U.csv")[0]
    v = gio.read_dense_csv(tmp_path / "fit" / "V.csv")[0]
    assert normwise(u @ v.T, g["U"] @ g["V"].T) < 1e-7
    rep = gio.read_json(tmp_path / "fit" / "fit_report.json")
    assert normwise(rep["objective_trace"], g["trace"]) < 1e-8
    assert rep["final_objective"] == pytest.approx(float(g["final_objective"]), rel=1e-8)
    man = gio.read_json(tmp_path / "fit" / "manifest.json")
    assert man["command"] == "fit" and str(ycsv) in man["input_checksums"]
    rc = cli.main(["cv", "--y", str(ycsv), "--ranks", "1:3", "--criterion", "scree",
                   "--out", str(tmp_path / "cv")])
    assert rc == int(g["cv_rc"]) == 0
    rr = gio.read_json(tmp_path / "cv" / "rank_report.json")
    assert normwise(rr["scree_eigenvalues"], g["scree"]) < 1e-9
    assert rr["chosen"]["scree"] == int(g["scree_pick"])


def test_cli_eval(tmp_path):
    from paper_2412_20509_b200 import cli
    from paper_2412_20509_b200 import io as gio
    rng = np.random.default_rng(3)
    y = rng.poisson(3.0, (20, 6)).astype(float)
    mu = np.full_like(y, 3.1)
    test = rng.uniform(size=y.shape) < 0.3
    gio.write_dense_csv(tmp_path / "y.csv", y)
    gio.write_dense_csv(tmp_path / "mu.csv", mu)
    gio.write_mask_file(tmp_path / "t.txt", ~test)
    assert cli.main(["eval", "--y", str(tmp_path / "y.csv"), "--mu", str(tmp_path / "mu.csv"),
                     "--test", str(tmp_path / "t.txt"), "--out", str(tmp_path / "ev")]) == 0
    res = gio.read_json(tmp_path / "ev" / "metrics.json")
    ybar = float(y[~test].mean())
    assert res["n_test"] == int(test.sum()) and res["train_mean"] == pytest.approx(ybar)
    d0 = 2 * (np.where(y[test] > 0, y[test] * np.log(y[test] / 3.1), 0) - (y[test] - 3.1))
    db = 2 * (np.where(y[test] > 0, y[test] * np.log(y[test] / ybar), 0) - (y[test] - ybar))
    assert res["rel_deviance"] == pytest.approx(d0.sum() / db.sum(), rel=1e-10)
