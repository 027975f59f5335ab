"""GPU: result_checksum on the device (report.cpp:11-26) equals the
reference's, and a measured RunReport of each driver carries the reference's
ledger fields and result checksum."""
import json

import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_device_checksum_matches_reference(dev):
    for n, d, s in [(500, 0.02, 1), (3000, 0.004, 2), (1, 1.0, 3)]:
        a = O.port_gen_erdos_renyi(n, d, s)
        c = O.port_spgemm(a, a)
        assert dev.upload(c).checksum() == O.ref_result_checksum(c)
    m = O.Csr(3, 4, np.array([0, 2, 2, 5], np.int64), np.array([0, 3, 1, 2, 3], np.int64),
              np.array([-1.5e-9, 2.5e-9, -0.25, 7.0, 0.0]))
    assert dev.upload(m).checksum() == O.ref_result_checksum(m)
    assert dev.zeros(7, 7).checksum() == (0, 0)


@needs_ref
@pytest.mark.parametrize("algo,P,lam", [("trident", 8, 2), ("summa", 4, 2), ("oned", 4, 2)])
def test_measured_report_vs_reference(algo, P, lam):
    a, b = O.port_gen_erdos_renyi(300, 0.03, 3), O.port_gen_erdos_renyi(300, 0.03, 4)
    dr = spg.run_algo(algo, a, b, P, lam)
    ref = O.ref_run_algo(algo, a, b, P, lam)
    assert dr.checksum == O.ref_result_checksum(ref["c"])
    rep = spg.make_report(dr, algo, P, lam, matrix_a="er300", matrix_b="er300b")
    L = ref["ledger"]
    for r, row in enumerate(rep["per_process"]):
        for pfx, c in (("gi_", 1), ("li_", 0)):
            assert row[pfx + "messages"] == int(L[r, 0, c, 0])
            assert row[pfx + "bytes_sent"] == int(L[r, 0, c, 2])
            assert row[pfx + "bytes_recv"] == int(L[r, 1, c, 2])
    assert rep["result"]["checksum"] == f"0x{O.ref_result_checksum(ref['c'])[1]:016x}"
    assert rep["makespan_seconds"] > 0 and json.loads(spg.report_json(rep))["rounds"] == dr.rounds
