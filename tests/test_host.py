"""CPU: host-side logic of the product (generators, tiling, ledger) against
the reference's golden outputs and, where built, the reference itself."""
import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg
from golden_io import csr, grids, z


def same(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(a.colind, b.colind) and np.array_equal(a.values, b.values))


def test_generator_bit_exact_vs_golden():
    for s in (1, 2, 3):
        assert same(spg.gen_erdos_renyi(40, 0.15, s), csr(f"er40_s{s}_A"))
    assert same(spg.gen_erdos_renyi(3, 0.7, 11), csr("identity3_B"))
    assert same(spg.gen_erdos_renyi(20, 1.0, 4), csr("dense20_A"))
    assert same(spg.gen_erdos_renyi(300, 0.03, 3), csr("er300_p3_A"))


@pytest.mark.parametrize("n,d,seed", [(16384, 8.0 / 16384, 1), (5000, 0.001, 9), (100, 0.5, 3), (0, 0.1, 1), (7, 1.0, 2)])
def test_generator_bit_exact_vs_port(n, d, seed):
    assert same(spg.gen_erdos_renyi(n, d, seed), O.port_gen_erdos_renyi(n, d, seed))


def test_generator_errors():
    for bad in [(10, 0.0, 1), (10, 1.5, 1), (-1, 0.5, 1)]:
        with pytest.raises(spg.SpgError):
            spg.gen_erdos_renyi(*bad)


def test_rect_generator_matches_port_and_transpose():
    a = spg.gen_erdos_renyi_rect(1000, 300, 0.01, 5)
    assert same(a, O.port_gen_erdos_renyi_rect(1000, 300, 0.01, 5))
    t = spg.transpose(a)
    assert t.is_canonical() and t.nrows == 300 and t.ncols == 1000
    d = np.zeros((1000, 300))
    for i in range(1000):
        d[i, a.colind[a.rowptr[i]:a.rowptr[i + 1]]] = a.values[a.rowptr[i]:a.rowptr[i + 1]]
    dt = np.zeros((300, 1000))
    for i in range(300):
        dt[i, t.colind[t.rowptr[i]:t.rowptr[i + 1]]] = t.values[t.rowptr[i]:t.rowptr[i + 1]]
    assert np.array_equal(d.T, dt)


def test_rmat_deterministic_and_canonical():
    a = spg.gen_rmat(10, 8, 1, 2)
    b = spg.gen_rmat(10, 8, 1, 2)
    assert same(a, b)
    a.check_canonical()
    assert a.nrows == 1024 and 0 < a.nnz <= 8 * 1024
    assert not same(a, spg.gen_rmat(10, 8, 3, 2))


@pytest.mark.parametrize("P,lam", grids())
def test_partition_matches_reference(P, lam):
    a = csr("er300_p3_A")
    tiles, tm = spg.partition(a, "trident", P, lam)
    assert np.array_equal(tm.tiles, z()[f"part_P{P}_L{lam}_rects"])
    assert [t.nnz for t in tiles] == z()[f"part_P{P}_L{lam}_nnz"].tolist()
    assert same(spg.reassemble(tiles, tm), a)


def test_tile_map_spec_pins():
    tm = spg.make_tile_map(8, 8, "trident", 16, 4)
    assert tm.row_bounds.tolist() == list(range(9)) and tm.col_bounds.tolist() == [0, 4, 8]
    assert spg.block_bounds(10, 3).tolist() == [0, 4, 7, 10]
    tm = spg.make_tile_map(2, 5, "trident", 16, 4)  # zero-row slices
    assert (tm.tiles[:, 1] - tm.tiles[:, 0]).min() == 0
    with pytest.raises(spg.SpgError):
        spg.make_tile_map(4, 4, "grid2d", 8, 1)


def test_reassemble_rejects_bad_tiles():
    a = csr("er300_p3_A")
    tiles, tm = spg.partition(a, "trident", 4, 1)
    with pytest.raises(spg.SpgError) as e:
        spg.reassemble(tiles[:3], tm)
    assert e.value.kind == "IncompleteTileSet"


@pytest.mark.parametrize("P,lam", grids())
def test_trident_ledger_matches_reference(P, lam):
    a, b = csr("er300_p3_A"), csr("er300_p3_B")
    g = spg.TridentGrid.create(P, lam)
    ta, _ = spg.partition(a, "trident", P, lam)
    tb, _ = spg.partition(b, "trident", P, lam)
    L = spg.trident_ledger(g, [(t.nrows, t.nnz) for t in ta], [(t.nrows, t.nnz) for t in tb])
    assert np.array_equal(L, z()[f"trident_P{P}_L{lam}_ledger"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_prop1_exactness_uniform_stride():
    # uniform stride at P=16, lambda=4: GI recv per rank = 2(q-1)nnz/P
    n, k = 256, 16
    rows = np.repeat(np.arange(n), k)
    cols = ((np.arange(n)[:, None] + np.arange(k)[None, :] * (n // k)) % n).ravel()
    vals = 1.0 + ((rows + cols) % 7) * 0.125
    a = O.ref_from_triplets(n, n, rows, cols, vals)
    g = spg.TridentGrid.create(16, 4)
    ta, _ = spg.partition(a, "trident", 16, 4)
    L = spg.trident_ledger(g, [(t.nrows, t.nnz) for t in ta], [(t.nrows, t.nnz) for t in ta])
    ref = O.ref_run_algo("trident", a, a, 16, 4, want_c=False)["ledger"]
    assert np.array_equal(L, ref)
    assert (L[:, 1, 1, 1] == 512).all() and (L[:, 1, 0, 1] == 1536).all()


def test_csr_canonical_checker():
    m = spg.CsrMatrix(2, 2, np.array([0, 2, 2]), np.array([0, 0]), np.ones(2))
    assert not m.is_canonical()
    m = spg.CsrMatrix(2, 2, np.array([0, 1, 1]), np.array([5]), np.ones(1))
    assert not m.is_canonical()
    assert spg.gen_erdos_renyi(50, 0.2, 1).is_canonical()


@pytest.mark.parametrize("P,lam", grids())
def test_capi_tile_rects_match_reference(P, lam):
    # spg_tile_rects (the C ABI's make_tile_map, used by the device tile store)
    a = csr("er300_p3_A")
    assert np.array_equal(spg.tile_rects(int(a.nrows), int(a.ncols), "trident", P, lam), z()[f"part_P{P}_L{lam}_rects"])


@pytest.mark.parametrize("shape", [(8, 8), (2, 5), (300, 7), (0, 4), (17, 1)])
@pytest.mark.parametrize("scheme,P,lam", [("trident", 16, 4), ("trident", 8, 2), ("trident", 4, 1), ("grid2d", 9, 1),
                                          ("grid2d", 4, 1), ("rows1d", 5, 1), ("rows1d", 1, 1)])
def test_capi_tile_rects_match_make_tile_map(shape, scheme, P, lam):
    tm = spg.make_tile_map(*shape, scheme, P, lam)
    assert np.array_equal(spg.tile_rects(*shape, scheme, P, lam), tm.tiles)


def test_capi_tile_rects_grid_errors():
    for args in [(4, 4, "grid2d", 8, 1), (4, 4, "trident", 6, 4), (4, 4, "trident", 8, 1), (4, 4, "rows1d", 0, 1)]:
        with pytest.raises(spg.SpgError) as e:
            spg.tile_rects(*args)
        assert e.value.kind == "GridError"
    with pytest.raises(spg.SpgError) as e:
        spg.tile_rects(4, 4, "bogus", 4, 1)
    assert e.value.kind == "ParameterError"


REPORT_KEYS = ["config", "rounds", "makespan_seconds", "aggregate", "per_process", "result", "verified"]
PER_PROCESS_KEYS = ["rank", "node"] + [p + k for p in ("gi_", "li_") for k in
                                       ("messages", "nnz_sent", "bytes_sent", "nnz_recv", "bytes_recv")] + \
    ["completion_time"]


def test_make_report_layout_and_ledger_fields():
    # RunReport::to_json key order (report.cpp:34-83) filled from a measured result
    import json
    P, lam = 8, 2
    a = csr("er300_p3_A")
    g = spg.TridentGrid.create(P, lam)
    L = z()[f"trident_P{P}_L{lam}_ledger"]
    tl = np.arange(P * g.q * 4, dtype=np.float64).reshape(P, g.q, 4)
    dr = spg.DriverResult(a, L, tl, 1.25, g.q, (int(a.nnz), 0xDEADBEEF))
    tm = spg.make_tile_map(300, 300, "trident", P, lam)
    rep = spg.make_report(dr, "trident", P, lam, tilemap=tm, verified=True)
    assert list(rep)[:len(REPORT_KEYS)] == REPORT_KEYS and "tilemap" in rep and "timeline" in rep
    assert [list(r) for r in rep["per_process"]] == [PER_PROCESS_KEYS] * P
    for r, row in enumerate(rep["per_process"]):
        assert row["gi_bytes_recv"] == int(L[r, 1, 1, 2]) and row["li_nnz_sent"] == int(L[r, 0, 0, 1])
        assert row["completion_time"] == pytest.approx(tl[r, :, 1:].sum() * 1e-3)
    assert rep["aggregate"]["gi"]["bytes_sent"] == int(L[:, 0, 1, 2].sum())
    assert rep["result"] == {"nrows": 300, "ncols": 300, "nnz": int(a.nnz), "checksum": "0x00000000deadbeef"}
    assert json.loads(spg.report_json(rep)) == rep


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_port_result_checksum_vs_reference():
    # report.cpp:11-26, incl. negative values, halves and an empty matrix
    for s in (1, 2):
        a = O.port_gen_erdos_renyi(500, 0.02, s)
        assert O.port_result_checksum(a) == O.ref_result_checksum(a)
    m = O.Csr(3, 4, np.array([0, 2, 2, 5], np.int64), np.array([0, 3, 1, 2, 3], np.int64),
              np.array([-1.5e-9, 2.5e-9, -0.25, 7.0, 0.0]))
    assert O.port_result_checksum(m) == O.ref_result_checksum(m)
    assert O.port_result_checksum(spg.CsrMatrix.zeros(5, 5)) == O.ref_result_checksum(spg.CsrMatrix.zeros(5, 5))
