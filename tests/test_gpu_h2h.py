"""GPU parity of the host-to-host local multiply (spg_spgemm_host_to_host: the
whole of spgemm_local, csr.cpp:132-165, host CSR in and out, A in row batches
whose downloads overlap the next batch's multiply) against the CPU oracle and
the reference's golden products. Bar: rowptr/colind/values bit-exact (each
batch is the same per-row kernel; rows never straddle batches)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg
from paper_2603_21444_b200 import _capi
from golden_io import csr, spgemm_cases

pytestmark = pytest.mark.gpu


def same(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64))
            and np.array_equal(a.values, b.values))


@pytest.mark.parametrize("name", spgemm_cases())
def test_h2h_golden_bit_exact(dev, name):
    for batches in (1, 3):
        c = dev.spgemm_host_to_host(csr(f"{name}_A"), csr(f"{name}_B"), batches=batches)
        assert same(c, csr(f"{name}_C"))


@pytest.mark.parametrize("batches", [1, 2, 7, 8, 64])
def test_h2h_random_vs_oracle(dev, batches):
    a = O.port_gen_erdos_renyi(3000, 0.01, 2)
    b = O.port_gen_erdos_renyi(3000, 0.01, 9)
    ref = O.port_spgemm(a, b)
    assert same(dev.spgemm_host_to_host(a, b, batches=batches), ref)
    # C = A*A: the shared host matrix is uploaded once
    assert same(dev.spgemm_host_to_host(a, a, batches=batches), O.port_spgemm(a, a))


def test_h2h_rectangular_and_empty_rows(dev):
    a = O.port_gen_erdos_renyi(400, 0.02, 3)
    # zero out a band of rows (empty rows across batch cuts)
    a = spg.CsrMatrix.of(a)
    keep = np.ones(a.nnz, bool)
    keep[a.rowptr[100]:a.rowptr[250]] = False
    cnt = np.diff(a.rowptr).copy()
    cnt[100:250] = 0
    a = spg.CsrMatrix(400, 400, np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64), a.colind[keep],
                      a.values[keep])
    b = spg.CsrMatrix.of(O.port_gen_erdos_renyi(400, 0.05, 4))
    b = spg.CsrMatrix(400, 400, b.rowptr, b.colind, b.values)
    ref = O.port_spgemm(a, b)
    for batches in (1, 5, 400, 1000):
        assert same(dev.spgemm_host_to_host(a, b, batches=batches), ref)


def test_h2h_empty_and_cap(dev):
    z = spg.CsrMatrix.zeros(5, 7)
    b = spg.CsrMatrix.zeros(7, 3)
    c = dev.spgemm_host_to_host(z, b, batches=4)
    assert c.nrows == 5 and c.ncols == 3 and c.nnz == 0 and np.array_equal(c.rowptr, np.zeros(6, np.int64))
    # too small a capacity: SPG_PARAMETER_ERROR with the needed nnz; the wrapper retries
    a = O.port_gen_erdos_renyi(300, 0.05, 5)
    ref = O.port_spgemm(a, a)
    assert same(dev.spgemm_host_to_host(a, a, batches=3, cap=1), ref)
    lib = _capi.lib()
    a = spg.CsrMatrix.of(a)
    rp = np.empty(a.nrows + 1, np.int64)
    ci = np.empty(1, np.int64)
    va = np.empty(1, np.float64)
    nnz = C.c_int64()
    st = lib.spg_spgemm_host_to_host(dev.ctx, a.nrows, a.ncols, a.rowptr.ctypes.data, a.colind.ctypes.data,
                                     a.values.ctypes.data, a.nrows, a.ncols, a.rowptr.ctypes.data,
                                     a.colind.ctypes.data, a.values.ctypes.data, 8, 2, 1, rp.ctypes.data,
                                     ci.ctypes.data, va.ctypes.data, C.byref(nnz))
    assert _capi.STATUS[st] == "SPG_PARAMETER_ERROR"
    assert nnz.value == ref.nnz
    # inner-dimension mismatch -> DimensionError
    with pytest.raises(spg.SpgError):
        dev.spgemm_host_to_host(spg.CsrMatrix.zeros(3, 4), spg.CsrMatrix.zeros(5, 2))
