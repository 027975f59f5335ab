"""CPU: pin the oracle before trusting it.

The plain-C restatement (oracle/cpu_oracle.c) must reproduce the reference's
own outputs bit for bit: the golden vectors in tests/golden/small.npz were
produced by the reference itself (tests/golden/make_golden.py over
oracle/_ref/libspgref.so), and where the reference library is present we also
compare directly on fresh random inputs.
"""
import numpy as np
import pytest

import oracle as O
from golden_io import csr, spgemm_cases, z


def same(a, b):
    return (a.nrows == b.nrows and a.ncols == b.ncols and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(a.colind, b.colind) and np.array_equal(a.values, b.values))


@pytest.mark.parametrize("name", spgemm_cases())
def test_port_spgemm_matches_golden_bit_exact(name):
    c = O.port_spgemm(csr(f"{name}_A"), csr(f"{name}_B"))
    assert same(c, csr(f"{name}_C"))


def test_golden_known_answers():
    # test_csr.cpp:31-33 frozen product [[0,3],[8,0]]
    c = csr("frozen2x2_C")
    assert c.rowptr.tolist() == [0, 1, 2] and c.colind.tolist() == [1, 0] and c.values.tolist() == [3.0, 8.0]
    # test_csr.cpp:27 I*A == A
    assert same(csr("identity3_C"), csr("identity3_B"))
    # test_csr.cpp:74-81 explicit zero kept
    c = csr("cancel_C")
    assert c.nnz == 1 and c.values[0] == 0.0
    # test_csr.cpp:36-41 empty row
    c = csr("emptyrow_C")
    assert c.rowptr[1] == c.rowptr[2]


def test_port_spgeam_and_vconcat_match_golden():
    assert same(O.port_spgeam(csr("geam_X"), csr("geam_Y")), csr("geam_Z"))
    f = csr("geam_frozen")
    assert f.colind.tolist() == [0, 1, 1] and f.values.tolist() == [1.0, 2.0, 2.0]
    a = csr("vcat_A")
    parts, start = [], 0
    for size in (6, 6, 5):
        parts.append(O.port_extract(a, np.array([start, start + size, 0, a.ncols])))
        start += size
    assert same(O.port_vconcat(parts), a)


def test_port_generator_matches_golden_inputs():
    for s in (1, 2, 3):
        assert same(O.port_gen_erdos_renyi(40, 0.15, s), csr(f"er40_s{s}_A"))
    assert same(O.port_gen_erdos_renyi(20, 1.0, 4), csr("dense20_A"))


def test_port_dimension_errors():
    a = O.Csr(2, 3, np.zeros(3, np.int64), np.zeros(0, np.int64), np.zeros(0))
    b = O.Csr(2, 2, np.zeros(3, np.int64), np.zeros(0, np.int64), np.zeros(0))
    with pytest.raises(O.OracleError) as e:
        O.port_spgemm(a, b)
    assert e.value.code == 2
    with pytest.raises(O.OracleError):
        O.port_spgeam(b, a)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,d,seed", [(500, 0.02, 7), (2000, 0.004, 9), (64, 0.3, 1), (1, 1.0, 3), (0, 0.5, 1)])
def test_port_vs_reference_random(n, d, seed):
    a = O.ref_gen_erdos_renyi(n, d, seed)
    b = O.ref_gen_erdos_renyi(n, d, seed + 1)
    assert same(O.port_gen_erdos_renyi(n, d, seed), a)
    assert same(O.port_spgemm(a, b), O.ref_spgemm_local(a, b))
    assert same(O.port_spgeam(a, b), O.ref_spgeam(a, b))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_config1_products():
    a = O.ref_gen_erdos_renyi(16384, 8.0 / 16384, 1)
    assert a.nnz == 130618
    assert O.port_products(a, a) == 1040687
    c = O.port_spgemm(a, a)
    assert c.nnz == 1038646


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("r", [2.0, 1.5, 1.0])
def test_port_mcl_poststep_vs_reference(r):
    # apps.cpp:79-82 post-step: the port against the reference's own functions
    a = O.port_column_normalize(O.port_gen_erdos_renyi(400, 0.02, 11))
    c = O.port_spgemm(a, a)
    got, ref = O.port_mcl_poststep(c, 0.003, r), O.ref_mcl_poststep(c, 0.003, r)
    assert O.pattern_equal(got, ref)
    assert np.array_equal(got.values, ref.values)
    assert np.array_equal(O.port_elementwise_power(c, r).values, O.ref_elementwise_power(c, r).values)
