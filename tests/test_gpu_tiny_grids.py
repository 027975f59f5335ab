"""GPU: the distributed drivers on tiny and degenerate grids:
0-row slices (a coarse block with fewer than lambda rows, block_bounds at
partition.cpp:74-81), 0-nnz tiles that still cost (rows+1)*4 wire bytes
(netmodel.hpp:37-39), rectangular operands. The device C must equal the serial
reference product bit for bit and the per-rank ledger must equal the
reference engine's (algorithms.cpp:24-174) for the same grid.

The reference itself cannot partition a matrix whose trailing row slices are
empty: `block_of` (partition.cpp:17-20) maps a slice that starts at nrows to
index nslices, one past `slice_ranks` (partition.cpp:171), and the process
crashes. Those cases (ref=False) are checked against the serial reference
product and the host ledger mirror (`trident_ledger`, itself pinned to the
reference engine on every grid the reference can run, tests/test_host.py)."""
import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg

pytestmark = pytest.mark.gpu


def same(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64))
            and np.array_equal(a.values, b.values))


CASES = [
    # (m, k, n, density, seed, algo, P, lambda, reference can run it)
    (6, 6, 6, 0.4, 1, "trident", 16, 4, False),  # trailing 0-row slices, empty tiles
    (8, 8, 8, 0.3, 2, "trident", 16, 4, True),   # 1-row slices
    (5, 9, 3, 0.5, 3, "trident", 8, 2, True),    # rectangular, uneven slices
    (3, 3, 3, 0.0, 4, "trident", 4, 1, True),    # all tiles empty (still (rows+1)*4 wire bytes)
    (7, 4, 9, 0.5, 5, "summa", 4, 2, True),      # rectangular SUMMA with uneven blocks
    (2, 2, 2, 0.9, 6, "summa", 4, 1, True),      # 1-row / 1-column blocks
    (6, 6, 6, 0.4, 7, "oned", 8, 2, False),      # 1D driver, trailing 0-row slices
]


def rect_er(m, k, density, seed):
    if density == 0.0:
        return spg.CsrMatrix.zeros(m, k)
    return spg.CsrMatrix.of(O.port_gen_erdos_renyi_rect(m, k, density, seed))


@pytest.mark.parametrize("m,k,n,d,seed,algo,P,lam,ref_ok", CASES)
def test_tiny_grid(m, k, n, d, seed, algo, P, lam, ref_ok):
    a = rect_er(m, k, d, seed)
    b = rect_er(k, n, d, seed + 11)
    dr = spg.run_algo(algo, a, b, P, lam)
    assert same(dr.c, O.port_spgemm(a, b))
    led = np.asarray(dr.ledger).reshape(P, 2, 2, 3)
    if ref_ok and O.ref_available():
        ref = O.ref_run_algo(algo, a, b, P, lam)
        assert spg.pattern_equal(dr.c, ref["c"]) and spg.allclose(dr.c, ref["c"], 1e-12)
        assert np.array_equal(led, ref["ledger"])
    elif algo == "trident":
        g = spg.TridentGrid.create(P, lam)
        ta, _ = spg.partition(a, "trident", P, lam)
        tb, _ = spg.partition(b, "trident", P, lam)
        host = spg.trident_ledger(g, [(t.nrows, t.nnz) for t in ta], [(t.nrows, t.nnz) for t in tb])
        assert np.array_equal(led, np.asarray(host).reshape(P, 2, 2, 3))
