"""GPU: the MCL post-step on device through the C ABI
against the reference's own column_normalize / prune / elementwise_power
(oracle/_ref, csr.cpp:224-255) composed as in mcl (apps.cpp:79-82).

Bar: structure (rowptr, colind) bit-exact (the prune decision precedes the
power, so it never depends on pow); values bit-exact for exponent 1 and within
1e-12 relative otherwise (north_star's fp64 tolerance): the reference calls
glibc's pow, which is within ~0.52 ulp but not correctly rounded (it differs
from the correctly rounded v*v in ~0.1% of squares), while the device uses the
correctly rounded square for exponent 2 and CUDA's pow otherwise."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg

pytestmark = pytest.mark.gpu
REL_TOL = 1e-12
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def structure_equal(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64)))


def close(a, b, tol=REL_TOL):
    x, y = np.asarray(a.values), np.asarray(b.values)
    return x.shape == y.shape and bool(np.all(np.abs(x - y) <= tol * np.maximum(np.abs(x), np.abs(y))))


def expansion(dev, n, d, seed):
    m = O.port_column_normalize(O.port_gen_erdos_renyi(n, d, seed))
    dm = dev.upload(m)
    return dev.spgemm(dm, dm)


@needs_ref
@pytest.mark.parametrize("r", [2.0, 1.0, 3.0, 1.5, 0.5])
def test_elementwise_power_vs_reference(dev, r):
    a = O.port_gen_erdos_renyi(700, 0.02, 3)
    dm = dev.upload(a)
    dev.elementwise_power(dm, r)
    got, ref = dm.download(), O.ref_elementwise_power(a, r)
    assert structure_equal(got, ref)
    if r == 1.0:
        assert np.array_equal(got.values, ref.values)
    assert close(got, ref)


@needs_ref
@pytest.mark.parametrize("n,d,seed,theta,r", [(2000, 0.004, 1, 0.002, 2.0), (3000, 0.003, 2, 0.01, 2.0),
                                              (500, 0.02, 3, 0.0, 2.0), (1500, 0.005, 4, 0.005, 1.7),
                                              (800, 0.01, 5, 0.5, 2.0)])  # theta 0.5 prunes almost everything
def test_mcl_poststep_vs_reference(dev, n, d, seed, theta, r):
    dc = expansion(dev, n, d, seed)
    c = dc.download()
    got = dev.mcl_poststep(dc, theta, r)
    got.check()
    got = got.download()
    ref = O.ref_mcl_poststep(c, theta, r)
    assert structure_equal(got, ref)
    assert close(got, ref)
    # c is not modified by the fused step
    assert np.array_equal(dc.download().values, c.values)


def test_mcl_poststep_matches_unfused_device_steps(dev):
    dc = expansion(dev, 2500, 0.004, 7)
    fused = dev.mcl_poststep(dc, 0.003, 2.0).download()
    x = dev.copy(dc)
    dev.column_normalize(x)
    p = dev.prune(x, 0.003)
    dev.elementwise_power(p, 2.0)
    dev.column_normalize(p)
    assert structure_equal(fused, p.download()) and np.array_equal(fused.values, p.download().values)


def test_mcl_poststep_errors_and_empty(dev):
    dc = expansion(dev, 300, 0.01, 1)
    with pytest.raises(spg.SpgError) as e:
        dev.mcl_poststep(dc, -1.0, 2.0)
    assert e.value.kind == "ParameterError"
    z = dev.mcl_poststep(dev.zeros(40, 40), 0.002, 2.0).download()
    assert z.nnz == 0 and z.rowptr.tolist() == [0] * 41


@pytest.mark.slow
def test_config4_mcl_step_full_size(dev):
    """Config 4 at full size: C = M*M (537M entries), then the fused post-step,
    against the digest of the reference's own post-step (tests/golden/config4.json
    "mcl_step", made by make_golden.py mcl4)."""
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config4.json")) as f:
        g = json.load(f)
    if "mcl_step" not in g:
        pytest.skip("config4.json has no mcl_step digest")
    g = g["mcl_step"]
    m = spg.gen_erdos_renyi(1 << 21, 16.0 / (1 << 21), 1)
    dm = dev.upload(m)
    dev.column_normalize(dm)
    dc = dev.spgemm(dm, dm)
    s = dev.mcl_poststep(dc, g["params"]["prune_threshold"], g["params"]["inflation"]).download()
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert int(s.nnz) == g["nnz"]
    assert sha(np.asarray(s.rowptr, np.int64)) == g["sha_rowptr"]
    assert sha(np.asarray(s.colind, np.int64)) == g["sha_colind"]
    for i, row in g["sample_rows"].items():
        lo, hi = int(s.rowptr[int(i)]), int(s.rowptr[int(i) + 1])
        assert s.colind[lo:hi].tolist() == row["cols"]
        got, ref = np.asarray(s.values[lo:hi]), np.asarray(row["vals"])
        assert np.all(np.abs(got - ref) <= REL_TOL * np.maximum(np.abs(got), np.abs(ref))), f"row {i}"
