"""Time the native MatrixMarket -> CSR reader against the reference read (build container only: imports gmfkit from /root/reference)."""
import sys, time, os
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2412_20509_b200 import io as gio
rng = np.random.default_rng(0)
n, m = 50_000, 500
nnz = int(n * m * 0.08)
key = np.unique(rng.integers(0, n * m, nnz)); rows, cols = key // m, key % m; nnz = key.size
vals = rng.integers(1, 20, nnz)
path = "/tmp/c4like.mtx"
if not os.path.exists(path):
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate integer general\n")
        fh.write(f"{n} {m} {nnz}\n")
        np.savetxt(fh, np.column_stack([rows + 1, cols + 1, vals]), fmt="%d")
sz = os.path.getsize(path)
t0 = time.perf_counter(); rm = gio.read_matrix_market_csr(path); t1 = time.perf_counter()
sys.path.insert(0, "/root/reference/pkg/src")
import gmfkit.io as rio
t2 = time.perf_counter(); dense = rio.read_matrix_market(path); t3 = time.perf_counter()
ip, ix, ct = rm.csr
d2 = np.zeros((n, m)); d2[np.repeat(np.arange(n), np.diff(ip)), ix] = ct
assert np.array_equal(d2, dense)
print(f"file {sz/1e6:.0f} MB, {nnz} entries: native CSR read {t1-t0:.2f} s ({nnz/(t1-t0)/1e6:.1f} M entries/s), reference mmread+todense {t3-t2:.2f} s, identical")
