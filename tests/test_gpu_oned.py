"""GPU: the sparsity-aware 1D driver (reference
oned_spgemm, algorithms.cpp:176-269) through the C ABI. Each rank multiplies
its A row block by the gathered B (its own block + exactly the remote rows its
columns name) in ascending k, so C is bit-identical to the serial product; the
ledger (one request + one transfer per (rank, owner)) must equal the
reference engine's, run here through oracle/_ref."""
import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def same(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64))
            and np.array_equal(a.values, b.values))


@pytest.mark.parametrize("P,lam", [(1, 1), (2, 2), (3, 1), (4, 2), (5, 2), (8, 4), (8, 1)])
def test_oned_parity(P, lam):
    a, b = O.port_gen_erdos_renyi(400, 0.02, 1), O.port_gen_erdos_renyi(400, 0.02, 2)
    r = spg.oned_spgemm(a, b, P, lam)
    assert same(r.c, O.port_spgemm(a, b))
    assert r.rounds == 1 and r.timeline.shape == (P, 1, 4)


@needs_ref
@pytest.mark.parametrize("P,lam", [(2, 2), (3, 1), (4, 2), (8, 4), (8, 1)])
def test_oned_ledger_matches_reference(P, lam):
    a, b = O.port_gen_erdos_renyi(300, 0.01, 5), O.port_gen_erdos_renyi(300, 0.03, 6)
    r = spg.run_algo("oned", a, b, P, lam)
    ref = O.ref_run_algo("oned", a, b, P, lam)
    assert same(r.c, ref["c"])
    assert np.array_equal(r.ledger, ref["ledger"])


@needs_ref
def test_oned_rectangular_and_sparse_columns():
    # A 300x200 (columns concentrated in a few owners' ranges) times B 200x150
    a = O.port_gen_erdos_renyi_rect(300, 200, 0.004, 7)
    b = O.port_gen_erdos_renyi_rect(200, 150, 0.05, 8)
    for P, lam in [(4, 2), (7, 7)]:
        r = spg.oned_spgemm(a, b, P, lam)
        ref = O.ref_run_algo("oned", a, b, P, lam)
        assert same(r.c, ref["c"])
        assert np.array_equal(r.ledger, ref["ledger"])


def test_oned_errors():
    a = O.port_gen_erdos_renyi(50, 0.1, 1)
    b = O.port_gen_erdos_renyi_rect(40, 50, 0.1, 2)
    with pytest.raises(spg.SpgError) as e:
        spg.oned_spgemm(a, b, 2, 1)
    assert e.value.kind == "DimensionError"
    with pytest.raises(spg.SpgError) as e:
        spg.oned_spgemm(a, a, 0, 1)
    assert e.value.kind == "GridError"
