"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: rowptr/colind bit-exact; values bit-exact for the local multiply (the
kernel sums each entry in ascending k with separate mul/add, like the
reference) and within 1e-12 relative where the summation order legitimately
differs (trident q>=2 partial-C merge, like the reference's own trident)."""
import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg
from golden_io import csr, spgemm_cases, z

pytestmark = pytest.mark.gpu
REL_TOL = 1e-12  # north_star: fp64 values within 1e-12 relative


def same(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64))
            and np.array_equal(a.values, b.values))


def gpu_mul(dev, a, b, check=True):
    da, db = dev.upload(a), dev.upload(b)
    dc = dev.spgemm(da, db)
    if check:
        dc.check()
    return dc.download()


@pytest.mark.parametrize("name", spgemm_cases())
def test_spgemm_golden_bit_exact(dev, name):
    c = gpu_mul(dev, csr(f"{name}_A"), csr(f"{name}_B"))
    assert same(c, csr(f"{name}_C"))


@pytest.mark.parametrize("n,d,seed", [(2000, 0.004, 1), (3000, 0.01, 2), (64, 0.5, 3), (1, 1.0, 1), (500, 0.2, 4),
                                      (20000, 0.0012, 5), (4096, 0.03, 6)])
def test_spgemm_random_vs_oracle(dev, n, d, seed):
    a, b = O.port_gen_erdos_renyi(n, d, seed), O.port_gen_erdos_renyi(n, d, seed + 7)
    ref = O.port_spgemm(a, b)
    assert same(gpu_mul(dev, a, b), ref)


def test_config1_full_parity(dev):
    a = spg.gen_erdos_renyi(16384, 8.0 / 16384, 1)
    c = gpu_mul(dev, a, a)
    ref = O.ref_spgemm_local(a, a) if O.ref_available() else O.port_spgemm(a, a)
    assert c.nnz == 1038646
    assert same(c, ref)


def test_edge_cases(dev):
    I64 = np.int64
    # empty matrices and K = 0
    for (m, k, n) in [(0, 0, 0), (3, 0, 4), (0, 5, 2), (4, 4, 0)]:
        a = spg.CsrMatrix.zeros(m, k)
        b = spg.CsrMatrix.zeros(k, n)
        c = gpu_mul(dev, a, b)
        assert c.nrows == m and c.ncols == n and c.nnz == 0 and len(c.rowptr) == m + 1
    # A entries pointing at empty B rows -> zero products
    a = spg.CsrMatrix(2, 3, np.array([0, 2, 3], I64), np.array([0, 2, 1], I64), np.array([1.0, 2.0, 3.0]))
    b = spg.CsrMatrix(3, 2, np.array([0, 0, 1, 1], I64), np.array([1], I64), np.array([5.0]))
    assert same(gpu_mul(dev, a, b), O.port_spgemm(a, b))
    # ncols = 1 and explicit zero from cancellation
    a = O.Csr(1, 2, np.array([0, 2], I64), np.array([0, 1], I64), np.array([1.0, 1.0]))
    b = O.Csr(2, 1, np.array([0, 1, 2], I64), np.array([0, 0], I64), np.array([1.0, -1.0]))
    c = gpu_mul(dev, a, b)
    assert c.nnz == 1 and c.values[0] == 0.0
    # dimension mismatch
    with pytest.raises(spg.SpgError) as e:
        dev.spgemm(dev.upload(spg.CsrMatrix.zeros(2, 3)), dev.upload(spg.CsrMatrix.zeros(2, 2)))
    assert e.value.kind == "DimensionError"


def test_heavy_and_skewed_rows(dev):
    # a row with many entries (heavy by entries), a hub row (heavy by products),
    # clustered columns (banded) and hub columns (many duplicates per column)
    n = 3000
    rng = np.random.default_rng(0)
    rows, cols = [], []
    rows += [0] * 2000; cols += list(rng.choice(n, 2000, replace=False))           # heavy row by entries
    rows += list(range(1, n)); cols += list(rng.integers(0, 5, n - 1))             # hub columns 0..4
    for i in range(1, 200):                                                        # banded block
        for j in range(max(0, i - 20), min(n, i + 20)):
            rows.append(i); cols.append(j)
    vals = rng.random(len(rows)) + 0.5
    a = O.ref_from_triplets(n, n, rows, cols, vals) if O.ref_available() else None
    if a is None:
        pytest.skip("needs oracle/_ref for from_triplets")
    ref = O.port_spgemm(a, a)
    assert same(gpu_mul(dev, a, a), ref)
    r = spg.gen_rmat(12, 16, 1, 2)
    ref = O.port_spgemm(r, r)
    assert same(gpu_mul(dev, r, r), ref)


def _rows_with(products_per_row, entries, ncols_b, seed, b_len=None):
    """A (one row per target) x B with B rows of b_len entries over ncols_b
    columns: row r gets entries[r] A entries whose B rows sum to products_per_row[r]."""
    rng = np.random.default_rng(seed)
    nb_rows = 4096
    b_rp = [0]
    b_ci, b_va = [], []
    lens = rng.integers(1, 40, nb_rows) if b_len is None else np.full(nb_rows, b_len)
    for k in range(nb_rows):
        L = int(min(lens[k], ncols_b))
        cols = np.sort(rng.choice(ncols_b, L, replace=False))
        b_ci += list(cols); b_va += list(rng.random(L) + 0.25); b_rp.append(len(b_ci))
    b_rp = np.array(b_rp, np.int64)
    blen = np.diff(b_rp)
    a_rp, a_ci = [0], []
    for p, e in zip(products_per_row, entries):
        # greedy: pick e distinct B rows whose lengths sum to p (last one adjusted via a row of the exact length)
        ks = []
        left = p
        cand = rng.permutation(nb_rows)
        for k in cand:
            if len(ks) == e - 1:
                break
            if blen[k] <= left - (e - 1 - len(ks)):
                ks.append(int(k)); left -= int(blen[k])
        exact = [int(k) for k in np.nonzero(blen == left)[0] if int(k) not in ks]
        if left > 0 and exact:
            ks.append(exact[0])
        a_ci += sorted(ks); a_rp.append(len(a_ci))
    a_rp = np.array(a_rp, np.int64)
    a = O.Csr(len(products_per_row), nb_rows, a_rp, np.array(a_ci, np.int64), rng.random(len(a_ci)) + 0.5)
    b = O.Csr(nb_rows, ncols_b, b_rp, np.array(b_ci, np.int64), np.array(b_va))
    return a, b


@pytest.mark.parametrize("ncols_b", [64, 700, 1 << 20])
def test_row_class_boundaries_and_duplicates(dev, ncols_b):
    # products per row around the class edges (256/257, 512/513, 4096/4097) with
    # 1..33 entries; small ncols_b makes nearly every product a duplicate
    targets = [1, 2, 31, 32, 33, 255, 256, 257, 300, 511, 512, 513, 1000, 4095, 4096, 4097, 6000]
    ents = [1, 2, 5, 16, 32, 33, 8, 31, 32, 20, 32, 33, 40, 32, 200, 300, 500]
    rows, es = [], []
    for t in targets:
        for e in ents:
            if e <= t:
                rows.append(t); es.append(e)
    a, b = _rows_with(rows, es, ncols_b, seed=ncols_b)
    ref = O.port_spgemm(a, b)
    assert same(gpu_mul(dev, a, b), ref)


def test_big_rows_without_products(dev):
    # BIG rows (more entries than a worker row takes) whose B rows are all
    # empty, beside SMALL rows: zero-product rows on the side path
    I64 = np.int64
    nb = 400
    b_rp = np.zeros(nb + 1, I64)
    b_rp[301:] = np.arange(1, 101)          # rows 0..299 empty, rows 300..399 one entry
    b = O.Csr(nb, 50, b_rp, np.arange(100, dtype=I64) % 50, np.linspace(0.5, 1.5, 100))
    rows = [np.arange(0, 200), np.array([300, 301]), np.arange(0, 300), np.arange(250, 400)]
    a_rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(I64)
    a_ci = np.concatenate(rows).astype(I64)
    a = O.Csr(len(rows), nb, a_rp, a_ci, np.linspace(1, 2, len(a_ci)))
    assert same(gpu_mul(dev, a, b), O.port_spgemm(a, b))


def test_all_one_column(dev):
    # every product of every row lands in the same column (one bucket)
    n = 600
    a = O.port_gen_erdos_renyi(n, 0.05, 3)
    b = O.Csr(n, 3, np.arange(n + 1, dtype=np.int64), np.full(n, 1, np.int64), np.linspace(-1, 1, n))
    assert same(gpu_mul(dev, a, b), O.port_spgemm(a, b))


def test_rectangular_and_transpose(dev):
    a = spg.gen_erdos_renyi_rect(4096, 512, 0.01, 5)
    at = spg.transpose(a)
    assert same(gpu_mul(dev, a, at), O.port_spgemm(a, at))
    assert same(gpu_mul(dev, at, a), O.port_spgemm(at, a))


def test_products_count(dev):
    a = spg.gen_erdos_renyi(5000, 0.002, 3)
    assert dev.products(dev.upload(a), dev.upload(a)) == O.port_products(a, a)


def test_spgeam_golden_and_random(dev):
    z_ = dev.spgeam(dev.upload(csr("geam_X")), dev.upload(csr("geam_Y"))).download()
    assert same(z_, csr("geam_Z"))
    for n, d, s in [(1000, 0.01, 1), (100, 0.3, 2), (5, 1.0, 3), (2000, 0.05, 4)]:
        a, b = O.port_gen_erdos_renyi(n, d, s), O.port_gen_erdos_renyi(n, d, s + 1)
        assert same(dev.spgeam(dev.upload(a), dev.upload(b)).download(), O.port_spgeam(a, b))
    a = O.port_gen_erdos_renyi(300, 0.1, 9)
    neg = O.Csr(a.nrows, a.ncols, a.rowptr, a.colind, -a.values)
    zz = dev.spgeam(dev.upload(a), dev.upload(neg)).download()
    assert spg.pattern_equal(zz, a) and (zz.values == 0).all()
    assert same(dev.spgeam(dev.upload(a), dev.zeros(300, 300)).download(), a)


def test_vconcat_and_extract(dev):
    a = spg.gen_erdos_renyi(1000, 0.01, 8)
    da = dev.upload(a)
    parts = [dev.extract(da, r0, r1, 0, 1000) for r0, r1 in [(0, 300), (300, 300), (300, 1000)]]
    assert same(dev.vconcat(parts).download(), a)
    t = dev.extract(da, 100, 700, 250, 900).download()
    assert same(t, O.port_extract(a, np.array([100, 700, 250, 900])))


def test_normalize_prune_bit_exact(dev):
    m = spg.gen_erdos_renyi(3000, 0.003, 1)
    dm = dev.upload(m)
    dev.column_normalize(dm)
    nm = dm.download()
    ref = O.port_column_normalize(m)
    assert same(nm, ref)
    p = dev.prune(dm, 0.2).download()
    assert same(p, O.port_prune(ref, 0.2))


def test_determinism(dev):
    a = spg.gen_erdos_renyi(20000, 0.0008, 11)
    c1 = gpu_mul(dev, a, a, check=False)
    c2 = gpu_mul(dev, a, a, check=False)
    assert same(c1, c2)


@pytest.mark.parametrize("merge", [False, True])
@pytest.mark.parametrize("P,lam", [(1, 1), (2, 2), (4, 1), (4, 4), (8, 2), (16, 4)])
def test_trident_parity_and_ledger(P, lam, merge, monkeypatch):
    """Default: a rank's q rounds are one multiply of its A tiles side by side
    (k order) times the stacked B blocks, so C is bit-identical to the serial
    reference. SPG_ROUND_MERGE=1: the reference structure (multiply per round
    + spgeam), within 1e-12 of the serial product like the reference's own."""
    if merge:
        monkeypatch.setenv("SPG_ROUND_MERGE", "1")
    a, b = csr("er300_p3_A"), csr("er300_p3_B")
    r = spg.trident_spgemm(a, b, spg.TridentGrid.create(P, lam))
    ref_c = csr("er300_p3_C")
    assert spg.pattern_equal(r.c, ref_c)
    assert spg.allclose(r.c, ref_c, REL_TOL)
    if not merge:
        assert same(r.c, ref_c)
    assert np.array_equal(r.c.values, z()[f"trident_P{P}_L{lam}_Cvalues"]) or spg.allclose(
        r.c, O.Csr(ref_c.nrows, ref_c.ncols, ref_c.rowptr, ref_c.colind, z()[f"trident_P{P}_L{lam}_Cvalues"]),
        REL_TOL)
    assert np.array_equal(r.ledger, z()[f"trident_P{P}_L{lam}_ledger"])
    assert r.rounds == spg.TridentGrid.create(P, lam).q


@pytest.mark.parametrize("P", [1, 4])
def test_summa_parity_and_ledger(P):
    a, b = csr("er300_p3_A"), csr("er300_p3_B")
    r = spg.summa_spgemm(a, b, P, 2)
    assert spg.allclose(r.c, csr("er300_p3_C"), REL_TOL)
    assert same(r.c, csr("er300_p3_C"))  # stages as one k-ordered multiply
    assert np.array_equal(r.ledger, z()[f"summa_P{P}_ledger"])


def test_trident_rectangular_kmer_shape():
    a = spg.gen_erdos_renyi_rect(3000, 400, 0.01, 5)
    at = spg.transpose(a)
    r = spg.trident_spgemm(a, at, spg.TridentGrid.create(8, 2))
    c = O.port_spgemm(a, at)
    assert spg.pattern_equal(r.c, c) and spg.allclose(r.c, c, REL_TOL)
    assert same(r.c, c)


@pytest.mark.parametrize("shared", [True, False])
def test_spgemm_host_entry(dev, shared):
    """spg_spgemm_host (host buffers in, C on the device): C = A*A with the same
    host arrays passed twice (uploaded once) and C = A*B with distinct ones."""
    import ctypes as C
    from paper_2603_21444_b200 import _capi
    L = _capi.lib()
    a = O.port_gen_erdos_renyi(3000, 0.004, 11)
    b = a if shared else O.port_gen_erdos_renyi(3000, 0.004, 12)
    arrs = []
    for m in (a, b):
        arrs.append((np.ascontiguousarray(m.rowptr, np.int64), np.ascontiguousarray(np.asarray(m.colind), np.int32),
                     np.ascontiguousarray(m.values, np.float64)))
    if shared:
        arrs[1] = arrs[0]
    (arp, aci, ava), (brp, bci, bva) = arrs
    h = C.c_void_p()
    _capi.check(L.spg_spgemm_host(dev.ctx, int(a.nrows), int(a.ncols), arp.ctypes.data, aci.ctypes.data,
                                  ava.ctypes.data, int(b.nrows), int(b.ncols), brp.ctypes.data, bci.ctypes.data,
                                  bva.ctypes.data, 4, C.byref(h)))
    c = spg.DeviceCsr(dev, h.value).download()
    assert same(c, O.port_spgemm(a, b))


@pytest.mark.parametrize("which", ["er", "rmat", "dups"])
def test_repeated_multiplies_are_identical(dev, which):
    """Race stress (compute-sanitizer is not available on the GPU pool): the
    tile kernel's look-back, relaxed status words and barrier-free pair
    ranking must give the same bytes on every run, equal to the oracle's."""
    if which == "er":
        a = b = spg.gen_erdos_renyi(16384, 8.0 / 16384, 1)
    elif which == "rmat":
        a = b = spg.gen_rmat(11, 16, 1, 2)
    else:  # 3000 x 40 times 40 x 40: nearly every product is a duplicate
        if not O.ref_available():
            pytest.skip("needs oracle/_ref for from_triplets")
        g = O.port_gen_erdos_renyi(3000, 0.01, 3)
        rows = np.repeat(np.arange(g.nrows), np.diff(np.asarray(g.rowptr)))
        a = O.ref_from_triplets(g.nrows, 40, rows, np.asarray(g.colind) % 40, np.asarray(g.values))
        b = O.port_gen_erdos_renyi(40, 0.5, 4)
    ref = O.port_spgemm(a, b)
    da = dev.upload(a)
    db = da if b is a else dev.upload(b)
    for _ in range(12):
        c = dev.spgemm(da, db).download()
        assert same(c, ref)


def _hub_case(ncols, seed):
    """A mix the hub path must get right: rows with thousands of entries over
    long and short B rows, a row whose products all hit one column (a bucket
    of thousands in k_tile terms), rows that reach the last column of the
    window, and ordinary rows."""
    rng = np.random.default_rng(seed)
    nb = 3000
    # B: mostly short rows, some long ones, a few spanning the whole width
    lens = rng.integers(0, 12, nb)
    lens[rng.choice(nb, 40, replace=False)] = rng.integers(200, 2000, 40)
    lens = np.minimum(lens, ncols)
    b_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    b_ci = np.concatenate([np.sort(rng.choice(ncols, int(l), replace=False)) for l in lens]).astype(np.int64)
    b_ci[b_rp[5]:b_rp[6]] = np.arange(ncols - lens[5], ncols) if lens[5] else b_ci[b_rp[5]:b_rp[6]]
    b_va = rng.uniform(-1, 1, int(b_rp[-1]))
    b = O.Csr(nb, ncols, b_rp, b_ci, b_va)
    rows = [np.sort(rng.choice(nb, 1500, replace=False)),          # a hub row over long and short B rows
            np.sort(rng.choice(nb, 400, replace=False)),
            np.array([5, 6, 7]),                                    # reaches the last column
            np.sort(rng.choice(nb, 8, replace=False)),              # an ordinary row
            np.arange(0, 2500, 3)]
    a_rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    a_ci = np.concatenate(rows).astype(np.int64)
    a = O.Csr(len(rows), nb, a_rp, a_ci, rng.uniform(-2, 2, len(a_ci)))
    return a, b


@pytest.mark.parametrize("ncols", [1000, 262144, 262145])
@pytest.mark.parametrize("seed", [1, 2])
def test_hub_rows_bit_exact(dev, ncols, seed):
    """BIG and MEDIUM rows: the dense hub accumulator (B up to 2^18 columns)
    and the sort-based ESC (wider B) against the oracle, bit-exact; 262144 is
    the widest B the hub takes, 262145 the narrowest that goes to the ESC."""
    a, b = _hub_case(ncols, seed)
    assert same(gpu_mul(dev, a, b), O.port_spgemm(a, b))


def test_hub_and_esc_agree(dev):
    """The same hub-path product through both side paths (SPG_BIG_ESC=1 is
    read once per process, so the ESC run is a child process)."""
    import subprocess
    import sys
    code = """
import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np, oracle as O, paper_2603_21444_b200 as spg
from test_gpu_parity import _hub_case
a, b = _hub_case(5000, 3)
d = spg.Device(0)
c = d.spgemm(d.upload(a), d.upload(b)).download()
np.save(%r, np.concatenate([np.asarray(c.rowptr, np.float64), np.asarray(c.colind, np.float64), np.asarray(c.values)]))
"""
    import os
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for esc in ("0", "1"):
        f = os.path.join(tempfile.mkdtemp(), "c.npy")
        env = dict(os.environ, SPG_BIG_ESC=esc)
        r = subprocess.run([sys.executable, "-c", code % (root, os.path.join(root, "tests"), f)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_tile_geometries_bit_exact():
    """Both compiled tile geometries (wide: 2048 window, 2 CTAs/SM; small:
    1536 window, 3 CTAs/SM — picked by B's mean row length) give the
    oracle's C bit-exact on short-row B, long-row B, A*A^T (a duplicate in
    every row) and MEDIUM rows that fit one geometry's tiles but not the
    other's. SPG_TILE_GEO is read once per process: one child per geometry."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import sys; sys.path.insert(0, {root!r})
import numpy as np, oracle as O, paper_2603_21444_b200 as spg
d = spg.Device(0)
def same(a, b):
    return (np.array_equal(a.rowptr, b.rowptr) and np.array_equal(np.asarray(a.colind, np.int64),
            np.asarray(b.colind, np.int64)) and np.array_equal(a.values, b.values))
cases = []
a = O.port_gen_erdos_renyi(3000, 0.005, 41); cases.append((a, a))                      # short B rows
a = O.port_gen_erdos_renyi_rect(6000, 600, 4 / 600, 42)
cases.append((a, O.port_gen_erdos_renyi_rect(600, 6000, 64 / 6000, 43)))                # long B rows
import scipy.sparse as sp
t = sp.csr_matrix((a.values, a.colind, a.rowptr), shape=(a.nrows, a.ncols)).T.tocsr()
t.sort_indices()
cases.append((a, O.Csr(a.ncols, a.nrows, t.indptr.astype(np.int64), t.indices.astype(np.int32),
                       t.data.astype(np.float64))))                                     # A*A^T
# rows of 1200-3700 products (weights around both geometries' PMAX, 2308 and
# 2820) over a B wider than the hub takes: MEDIUM tiles in one geometry are
# BIG (ESC) rows in the other
a = O.port_gen_erdos_renyi_rect(400, 4000, 40 / 4000, 44)
cases.append((a, O.port_gen_erdos_renyi_rect(4000, 300000, 60 / 300000, 45)))
for i, (a, b) in enumerate(cases):
    c = d.spgemm(d.upload(a), d.upload(b))
    c.check()
    assert same(c.download(), O.port_spgemm(a, b)), i
print("GEO_OK")
"""
    for geo in ("wide", "small"):
        env = dict(os.environ, SPG_TILE_GEO=geo)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (geo, r.stderr[-2000:])
        assert "GEO_OK" in r.stdout
