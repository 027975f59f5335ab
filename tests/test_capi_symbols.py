"""CPU: the drop-in libraries load and export every symbol their headers
declare; with no GPU the product fails loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2603_21444_b200 as spg
from paper_2603_21444_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spg", "capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spg_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    assert sorted(_capi.EXPORTS) == decl


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_cxx_library_exports_drop_in_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", _capi.CXX_LIB_PATH], capture_output=True, text=True).stdout
    for sym in ["spgsim::spgemm_local(", "spgsim::spgeam(", "spgsim::vconcat(", "spgsim::partition(",
                "spgsim::reassemble(", "spgsim::trident_spgemm(", "spgsim::summa_spgemm(", "spgsim::run_algo(",
                "spgsim::make_tile_map(", "spgsim::block_bounds(", "spgsim::TridentGrid::create(",
                "spgsim::gen_erdos_renyi(", "spgsim::CommLedger::record_transfer(", "spgsim::predict_trident_volume("]:
        assert sym in out, sym


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    n = ctypes.c_int(-1)
    _capi.check(_capi.lib().spg_device_count(ctypes.byref(n)))
    if n.value > 0:
        pytest.skip("a GPU is visible")
    ctx = ctypes.c_void_p()
    st = _capi.lib().spg_init(0, ctypes.byref(ctx))
    assert st == 22  # SPG_NO_DEVICE
    with pytest.raises(spg.SpgError):
        spg.spgemm_local(spg.CsrMatrix.identity(2), spg.CsrMatrix.identity(2))


def test_trident_grid_is_host_logic():
    g = spg.TridentGrid.create(16, 4)
    assert g.q == 2 and g.coords_of(7) == (0, 1, 3)
    with pytest.raises(spg.SpgError) as e:
        spg.TridentGrid.create(12, 4)
    assert e.value.kind == "GridError"
    for P, lam, q in [(1, 1, 1), (2, 2, 1), (4, 4, 1), (4, 1, 2), (8, 2, 2)]:
        assert spg.TridentGrid.create(P, lam).q == q
