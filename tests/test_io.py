"""CSR-native MatrixMarket reader (reference io.py:96-139).

Host code in libgmf_asgd.so (no GPU needed): every fixture under
tests/golden/mm/ must read to exactly the reference's dense array
(tests/golden/mm.npz, written by gmfkit.io.read_matrix_market), and the
error behaviour follows the reference's ConfigError contract."""
import os

import numpy as np
import pytest

from conftest import golden

gk = pytest.importorskip("paper_2412_20509_b200")
from paper_2412_20509_b200 import io as gio  # noqa: E402

MM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mm")


@pytest.mark.parametrize("name", ["counts", "sym_pattern", "dups"])
def test_read_matches_reference(name):
    g = golden("mm")
    path = os.path.join(MM, f"{name}.mtx")
    np.testing.assert_array_equal(gio.read_matrix_market(path), g[name])
    rm = gio.read_matrix_market_csr(path)
    assert rm.shape == g[name].shape
    indptr, indices, counts = rm.csr
    for i in range(rm.n):
        cols = indices[indptr[i]:indptr[i + 1]]
        assert np.all(np.diff(cols) > 0)                    # column-sorted, no duplicates
    dense = np.zeros(rm.shape)
    dense[np.repeat(np.arange(rm.n), np.diff(indptr)), indices] = counts
    np.testing.assert_array_equal(dense, g[name])
    assert np.all(counts > 0)                               # explicit zeros dropped


def test_roundtrip_write_read(tmp_path):
    rng = np.random.default_rng(3)
    y = rng.poisson(0.3, (40, 30)).astype(float)
    p = tmp_path / "y.mtx"
    gio.write_matrix_market(p, y)
    np.testing.assert_array_equal(gio.read_matrix_market(p), y)


@pytest.mark.parametrize("body,exc", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", NotImplementedError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.5\n", gk.DomainError),
    ("%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 1 -3\n", gk.DomainError),
    ("%%MatrixMarket matrix coordinate integer general\n2 2 1\n3 1 1\n", gk.ConfigError),
    ("%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 1 1\n", gk.ConfigError),
    ("%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 x 1\n", gk.ConfigError),
    ("not a matrix market file\n", gk.ConfigError),
])
def test_errors(tmp_path, body, exc):
    p = tmp_path / "bad.mtx"
    p.write_text(body)
    with pytest.raises(exc):
        gio.read_matrix_market_csr(p)


def test_missing_file(tmp_path):
    with pytest.raises(gk.ConfigError):
        gio.read_matrix_market_csr(tmp_path / "absent.mtx")


def test_mask_file(tmp_path):
    p = tmp_path / "mask.txt"
    p.write_text("% unobserved\n1 2\n3 1\n")
    mask = gio.read_mask_file(p, (3, 2))
    assert mask.sum() == 4 and not mask[0, 1] and not mask[2, 0]
    p.write_text("4 1\n")
    with pytest.raises(gk.ConfigError):
        gio.read_mask_file(p, (3, 2))
