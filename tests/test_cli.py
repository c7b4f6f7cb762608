"""CLI and file formats on the host (gmfkit cli.py, io.py:42-200): argument
and config handling, exit codes for input errors, CSV / JSON / mask-list
round trips.  The fits themselves run in tests/test_gpu_cli.py."""
import json
import os

import numpy as np
import pytest

from paper_2412_20509_b200 import cli
from paper_2412_20509_b200 import io as gio


def test_dense_csv_round_trip_is_exact(tmp_path):
    a = np.random.default_rng(0).normal(size=(5, 3))
    a[1, 2] = np.nan
    p = tmp_path / "a.csv"
    gio.write_dense_csv(p, a, [f"row{i}" for i in range(5)], ["a", "b", "c"])
    b, rn, cn = gio.read_dense_csv(p)
    assert rn == [f"row{i}" for i in range(5)] and cn == ["a", "b", "c"]
    np.testing.assert_array_equal(np.isnan(a), np.isnan(b))
    np.testing.assert_array_equal(a[~np.isnan(a)], b[~np.isnan(b)])   # 17 digits: exact
    assert p.read_text().splitlines()[0] == ",a,b,c"


def test_dense_csv_reports_line_and_column(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text(",c1,c2\nr1,1,2\nr2,3,x\n")
    with pytest.raises(Exception, match="line 3: column 3: not a number"):
        gio.read_dense_csv(p)


def test_mask_list_round_trip(tmp_path):
    mask = np.random.default_rng(1).uniform(size=(6, 4)) > 0.3
    p = tmp_path / "m.txt"
    gio.write_mask_file(p, mask)
    np.testing.assert_array_equal(gio.read_mask_file(p, mask.shape), mask)


def test_json_is_sorted_and_byte_stable(tmp_path):
    p, q = tmp_path / "a.json", tmp_path / "b.json"
    obj = {"b": np.float64(1.5), "a": [np.int64(2), 3.0], "c": np.arange(3)}
    gio.write_json(p, obj)
    gio.write_json(q, obj)
    assert p.read_bytes() == q.read_bytes()
    assert json.loads(p.read_text()) == {"a": [2, 3.0], "b": 1.5, "c": [0, 1, 2]}


def test_exit_code_1_on_input_errors(tmp_path):
    ycsv = tmp_path / "y.csv"
    gio.write_dense_csv(ycsv, np.ones((4, 3)))
    assert cli.main(["fit", "--y", str(tmp_path / "missing.csv"), "--rank", "1",
                     "--out", str(tmp_path)]) == 1                        # no such file
    assert cli.main(["fit", "--y", str(ycsv), "--out", str(tmp_path)]) == 1   # no rank
    cfg = tmp_path / "c.toml"
    cfg.write_text("rank = 1\nbogus = 3\n")
    assert cli.main(["fit", "--y", str(ycsv), "--config", str(cfg),
                     "--out", str(tmp_path)]) == 1                        # unknown key
    assert cli.main(["fit", "--y", str(ycsv), "--rank", "1", "--algorithm", "asgd",
                     "--max-epochs", "0", "--out", str(tmp_path)]) == 1   # SgdConfig check


def test_flags_override_config(tmp_path):
    cfg = tmp_path / "c.toml"
    cfg.write_text('rank = 2\nmax_epochs = 7\nfamily = "neg_binomial"\n')
    args = cli.build_parser().parse_args(["fit", "--y", "y.csv", "--config", str(cfg),
                                          "--max-epochs", "9", "--seed", "4"])
    merged = cli._merge(args, cli._SGD_KEYS + ["rank", "family"])
    assert merged == {"rank": 2, "max_epochs": 9, "family": "neg_binomial", "seed": 4}
    assert cli._ranks("2:4") == [2, 3, 4] and cli._ranks("1,5") == [1, 5]
