"""TEST INFRASTRUCTURE ONLY — the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package, and only as the checker or the
timed CPU baseline — never as the product path.

Two back ends, both loaded with ctypes:

* ``ref_*``  — the reference simulator itself (``/root/reference/proj`` sources
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libspgref.so`` with the
  namespace renamed). Present wherever it was built (it travels with gpurun).
* ``port_*`` — our plain-C restatement (``oracle/cpu_oracle.c``) pinned against
  the reference and against ``tests/golden/``.

Matrices are exchanged as :class:`Csr` (int64 rowptr/colind, float64 values),
mirroring ``CsrMatrix`` (``csr.hpp:18-35``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import math

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libspgref.so")
PORT_SO = os.path.join(_HERE, "lib", "libspgoracle.so")

I64P = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


@dataclass
class Csr:
    nrows: int
    ncols: int
    rowptr: np.ndarray
    colind: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1]) if len(self.rowptr) else 0


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# ---------------------------------------------------------------- reference
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _R():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (run make -C oracle ref where /root/reference exists)")
        lib = C.CDLL(REF_SO)
        vp, i64, f64, u64, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_uint64, C.c_int
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_csr_new.restype = vp
        lib.ref_csr_new.argtypes = [i64, i64, I64P, I64P, F64P]
        lib.ref_csr_free.argtypes = [vp]
        lib.ref_csr_info.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        for f in ("ref_csr_rowptr", "ref_csr_colind"):
            getattr(lib, f).restype = C.POINTER(i64)
            getattr(lib, f).argtypes = [vp]
        lib.ref_csr_values.restype = C.POINTER(f64)
        lib.ref_csr_values.argtypes = [vp]
        lib.ref_csr_is_canonical.argtypes = [vp]
        lib.ref_gen_erdos_renyi.argtypes = [i64, f64, u64, C.POINTER(vp)]
        lib.ref_identity.argtypes = [i64, C.POINTER(vp)]
        lib.ref_from_triplets.argtypes = [i64, i64, i64, I64P, I64P, F64P, C.POINTER(vp)]
        lib.ref_permute_random.argtypes = [vp, u64, C.POINTER(vp)]
        lib.ref_column_normalize.argtypes = [vp, C.POINTER(vp)]
        lib.ref_prune.argtypes = [vp, f64, C.POINTER(vp)]
        lib.ref_elementwise_power.argtypes = [vp, f64, C.POINTER(vp)]
        lib.ref_result_checksum.argtypes = [vp, C.POINTER(i64), C.POINTER(C.c_uint64)]
        lib.ref_spgemm_local.argtypes = [vp, vp, C.POINTER(vp)]
        lib.ref_spgemm_local_timed.argtypes = [vp, vp, C.POINTER(f64), C.POINTER(i64), C.POINTER(vp)]
        lib.ref_spgeam.argtypes = [vp, vp, C.POINTER(vp)]
        lib.ref_vconcat.argtypes = [C.POINTER(vp), i32, C.POINTER(vp)]
        lib.ref_partition.argtypes = [vp, i32, i32, i32, C.POINTER(vp), I64P]
        lib.ref_reassemble.argtypes = [C.POINTER(vp), i32, i64, i64, i32, i32, C.POINTER(vp)]
        lib.ref_run_algo.argtypes = [i32, vp, vp, i32, i32, C.POINTER(vp),
                                     np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS"),
                                     C.POINTER(f64), I64P]
        lib.ref_grid.argtypes = [i32, i32, C.POINTER(i32)]
        lib.ref_predict_volume.argtypes = [i64, i32, i32, F64P]
        _ref = lib
    return _ref


def _chk(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, _R().ref_last_error().decode())


class RefHandle:
    """Owns one reference ``CsrMatrix`` living in the reference library."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        if getattr(self, "ptr", None) and _ref is not None:
            _ref.ref_csr_free(self.ptr)
            self.ptr = None

    @classmethod
    def from_csr(cls, m) -> "RefHandle":
        rp = np.ascontiguousarray(m.rowptr, dtype=np.int64)
        ci = np.ascontiguousarray(m.colind, dtype=np.int64)
        va = np.ascontiguousarray(m.values, dtype=np.float64)
        if len(ci) == 0:
            ci = np.zeros(1, np.int64)
            va = np.zeros(1, np.float64)
        return cls(_R().ref_csr_new(int(m.nrows), int(m.ncols), rp, ci, va))

    def to_csr(self) -> Csr:
        L = _R()
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        L.ref_csr_info(self.ptr, C.byref(nr), C.byref(nc), C.byref(nz))
        nr, nc, nz = nr.value, nc.value, nz.value
        rp = np.ctypeslib.as_array(L.ref_csr_rowptr(self.ptr), shape=(nr + 1,)).copy() if nr + 1 > 0 else np.zeros(1, np.int64)
        ci = np.ctypeslib.as_array(L.ref_csr_colind(self.ptr), shape=(nz,)).copy() if nz else np.zeros(0, np.int64)
        va = np.ctypeslib.as_array(L.ref_csr_values(self.ptr), shape=(nz,)).copy() if nz else np.zeros(0, np.float64)
        return Csr(nr, nc, rp, ci, va)


def _h(m) -> RefHandle:
    return m if isinstance(m, RefHandle) else RefHandle.from_csr(m)


def _out(fn, *args) -> RefHandle:
    o = C.c_void_p()
    _chk(fn(*args, C.byref(o)))
    return RefHandle(o.value)


def ref_gen_erdos_renyi(n: int, density: float, seed: int, handle: bool = False):
    h = _out(_R().ref_gen_erdos_renyi, n, density, seed)
    return h if handle else h.to_csr()


def ref_identity(n: int) -> Csr:
    return _out(_R().ref_identity, n).to_csr()


def ref_from_triplets(nrows, ncols, rows, cols, vals) -> Csr:
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    n = len(rows)
    if n == 0:
        rows, cols, vals = np.zeros(1, np.int64), np.zeros(1, np.int64), np.zeros(1)
    return _out(_R().ref_from_triplets, nrows, ncols, n, rows, cols, vals).to_csr()


def ref_permute_random(m, seed: int, handle: bool = False):
    hm = _h(m)
    h = _out(_R().ref_permute_random, hm.ptr, seed)
    return h if handle else h.to_csr()


def ref_elementwise_power(m, r: float, handle: bool = False):
    """csr.cpp:251-255 (the reference itself)."""
    hm = _h(m)
    h = _out(_R().ref_elementwise_power, hm.ptr, float(r))
    return h if handle else h.to_csr()


def ref_result_checksum(m):
    """report.cpp:11-26 (the reference itself) -> (nnz, hash)."""
    hm = _h(m)
    n, h = C.c_int64(), C.c_uint64()
    _chk(_R().ref_result_checksum(hm.ptr, C.byref(n), C.byref(h)))
    return n.value, h.value


def port_result_checksum(m):
    """report.cpp:11-26 restated in numpy: sum over entries (mod 2^64) of
    mix64(mix64(mix64(row + K) ^ col) ^ llround(v * 1e9))."""
    M1, M2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)

    def mix64(x):
        x = (x ^ (x >> np.uint64(30))) * M1
        x = (x ^ (x >> np.uint64(27))) * M2
        return x ^ (x >> np.uint64(31))

    rp = np.asarray(m.rowptr, np.int64)
    rows = np.repeat(np.arange(int(m.nrows), dtype=np.uint64), np.diff(rp))
    v = np.asarray(m.values, np.float64) * 1e9
    q = np.where(v >= 0, np.floor(v + 0.5), np.ceil(v - 0.5))  # llround: halves away from zero
    # (v + 0.5 is exact for |v| < 2^52; beyond that v is already an integer)
    q = np.where(np.abs(v) >= 2.0 ** 52, v, q).astype(np.int64).view(np.uint64)
    with np.errstate(over="ignore"):
        h = mix64(rows + np.uint64(0x51ED270B9A3E51EB))
        h = mix64(h ^ np.asarray(m.colind, np.int64).view(np.uint64))
        h = mix64(h ^ q)
        return int(rp[-1]), int(np.sum(h, dtype=np.uint64))


def ref_mcl_poststep(c, theta: float, r: float) -> Csr:
    """apps.cpp:79-82 with the reference's own functions."""
    m = ref_column_normalize(c, handle=True)
    m = ref_prune(m, theta, handle=True)
    m = ref_elementwise_power(m, r, handle=True)
    return ref_column_normalize(m)


def ref_column_normalize(m, handle: bool = False):
    hm = _h(m)
    h = _out(_R().ref_column_normalize, hm.ptr)
    return h if handle else h.to_csr()


def ref_prune(m, theta: float, handle: bool = False):
    hm = _h(m)
    h = _out(_R().ref_prune, hm.ptr, theta)
    return h if handle else h.to_csr()


def ref_spgemm_local(a, b, handle: bool = False):
    ha, hb = _h(a), _h(b)
    h = _out(_R().ref_spgemm_local, ha.ptr, hb.ptr)
    return h if handle else h.to_csr()


def ref_spgemm_local_timed(a, b, keep: bool = False):
    """(seconds, nnz(C), C or None): std::chrono around the reference call."""
    ha, hb = _h(a), _h(b)
    s, nz, o = C.c_double(), C.c_int64(), C.c_void_p()
    _chk(_R().ref_spgemm_local_timed(ha.ptr, hb.ptr, C.byref(s), C.byref(nz),
                                     C.byref(o) if keep else None))
    return s.value, nz.value, (RefHandle(o.value).to_csr() if keep else None)


def ref_spgeam(a, b) -> Csr:
    ha, hb = _h(a), _h(b)
    return _out(_R().ref_spgeam, ha.ptr, hb.ptr).to_csr()


def ref_vconcat(slices) -> Csr:
    hs = [_h(s) for s in slices]
    arr = (C.c_void_p * max(1, len(hs)))(*[h.ptr for h in hs])
    return _out(_R().ref_vconcat, arr, len(hs)).to_csr()


SCHEMES = {"trident": 0, "grid2d": 1, "rows1d": 2}


def ref_partition(m, scheme: str, procs: int, gpus_per_node: int):
    """-> (tiles: list[Csr], rects: (procs,4) int64)"""
    arr = (C.c_void_p * procs)()
    rects = np.zeros(procs * 4, np.int64)
    hm = _h(m)
    _chk(_R().ref_partition(hm.ptr, SCHEMES[scheme], procs, gpus_per_node, arr, rects))
    tiles = [RefHandle(arr[r]).to_csr() for r in range(procs)]
    return tiles, rects.reshape(procs, 4)


def ref_reassemble(tiles, nrows, ncols, scheme, procs, gpus_per_node) -> Csr:
    hs = [_h(t) for t in tiles]
    arr = (C.c_void_p * max(1, len(hs)))(*[h.ptr for h in hs])
    return _out(_R().ref_reassemble, arr, len(hs), nrows, ncols, SCHEMES[scheme], gpus_per_node).to_csr()


ALGOS = {"trident": 0, "summa": 1, "oned": 2}


def ref_run_algo(algo: str, a, b, procs: int, gpus_per_node: int, want_c: bool = True):
    """-> dict(c, ledger[(procs,2,2,3)], makespan, events[5]).

    ledger[rank, dir(0 sent / 1 received), class(0 LI / 1 GI)] = (messages, nnz, bytes)."""
    led = np.zeros(procs * 12, np.uint64)
    ev = np.zeros(5, np.int64)
    ms = C.c_double()
    o = C.c_void_p()
    ha, hb = _h(a), _h(b)
    _chk(_R().ref_run_algo(ALGOS[algo], ha.ptr, hb.ptr, procs, gpus_per_node,
                           C.byref(o) if want_c else None, led, C.byref(ms), ev))
    return {"c": RefHandle(o.value).to_csr() if want_c else None, "ledger": led.reshape(procs, 2, 2, 3),
            "makespan": ms.value, "events": ev}


def ref_timeline_jsonl(algo: str, a, b, procs: int, gpus_per_node: int, node_start_delay=None) -> str:
    """The reference's dr.timeline.to_jsonl() (engine.cpp:25-41) of run_algo."""
    ha, hb = _h(a), _h(b)
    d = np.asarray(node_start_delay if node_start_delay is not None else [], np.float64)
    n = C.c_size_t()
    L = _R()
    L.ref_timeline_jsonl.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                     C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
    _chk(L.ref_timeline_jsonl(ALGOS[algo], ha.ptr, hb.ptr, procs, gpus_per_node, d.ctypes.data, len(d), None, 0,
                              C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _chk(L.ref_timeline_jsonl(ALGOS[algo], ha.ptr, hb.ptr, procs, gpus_per_node, d.ctypes.data, len(d), buf,
                              n.value + 1, C.byref(n)))
    return buf.value.decode()


def ref_grid_q(procs: int, gpus_per_node: int) -> int:
    q = C.c_int()
    _chk(_R().ref_grid(procs, gpus_per_node, C.byref(q)))
    return q.value


def ref_predict_volume(nnz: int, procs: int, gpus_per_node: int) -> np.ndarray:
    out = np.zeros(6)
    _chk(_R().ref_predict_volume(nnz, procs, gpus_per_node, out))
    return out


# --------------------------------------------------------------- C restatement
class _OCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("rowptr", C.POINTER(C.c_int64)),
                ("colind", C.POINTER(C.c_int64)), ("values", C.POINTER(C.c_double))]


_port = None


def _P():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise FileNotFoundError(f"{PORT_SO} not built (make -C oracle)")
        lib = C.CDLL(PORT_SO)
        P = C.POINTER(_OCsr)
        lib.oracle_free.argtypes = [P]
        lib.oracle_products.restype = C.c_int64
        lib.oracle_products.argtypes = [P, P, C.c_void_p]
        lib.oracle_spgemm.argtypes = [P, P, P]
        lib.oracle_spgeam.argtypes = [P, P, P]
        lib.oracle_vconcat.argtypes = [C.POINTER(P), C.c_int, P]
        lib.oracle_gen_erdos_renyi.argtypes = [C.c_int64, C.c_double, C.c_uint64, P]
        lib.oracle_gen_erdos_renyi_rect.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, P]
        lib.oracle_trident_rect.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, I64P]
        lib.oracle_extract.argtypes = [P, I64P, P]
        lib.oracle_column_normalize.argtypes = [P]
        lib.oracle_prune.argtypes = [P, C.c_double, P]
        _port = lib
    return _port


def _to_o(m):
    rp = np.ascontiguousarray(m.rowptr, np.int64)
    ci = np.ascontiguousarray(m.colind, np.int64)
    va = np.ascontiguousarray(m.values, np.float64)
    o = _OCsr(int(m.nrows), int(m.ncols), rp.ctypes.data_as(C.POINTER(C.c_int64)),
              ci.ctypes.data_as(C.POINTER(C.c_int64)), va.ctypes.data_as(C.POINTER(C.c_double)))
    o._keep = (rp, ci, va)
    return o


def _from_o(o: _OCsr) -> Csr:
    nr = o.nrows
    nz = o.rowptr[nr] if nr >= 0 else 0
    rp = np.ctypeslib.as_array(o.rowptr, shape=(nr + 1,)).copy()
    ci = np.ctypeslib.as_array(o.colind, shape=(nz,)).copy() if nz else np.zeros(0, np.int64)
    va = np.ctypeslib.as_array(o.values, shape=(nz,)).copy() if nz else np.zeros(0)
    _P().oracle_free(C.byref(o))
    return Csr(nr, o.ncols, rp, ci, va)


def _pchk(rc: int, what: str) -> None:
    if rc == -2:
        raise OracleError(2, f"{what}: dimension mismatch")
    if rc == -3:
        raise OracleError(3, f"{what}: parameter out of range")
    if rc != 0:
        raise OracleError(1, f"{what}: failed ({rc})")


def port_products(a, b, per_row: bool = False):
    oa, ob = _to_o(a), _to_o(b)
    if per_row:
        out = np.zeros(int(a.nrows), np.int64)
        tot = _P().oracle_products(C.byref(oa), C.byref(ob), out.ctypes.data)
        return tot, out
    return _P().oracle_products(C.byref(oa), C.byref(ob), None)


def port_spgemm(a, b) -> Csr:
    oa, ob, oc = _to_o(a), _to_o(b), _OCsr()
    _pchk(_P().oracle_spgemm(C.byref(oa), C.byref(ob), C.byref(oc)), "spgemm")
    return _from_o(oc)


def port_spgeam(a, b) -> Csr:
    oa, ob, oc = _to_o(a), _to_o(b), _OCsr()
    _pchk(_P().oracle_spgeam(C.byref(oa), C.byref(ob), C.byref(oc)), "spgeam")
    return _from_o(oc)


def port_vconcat(slices) -> Csr:
    os_ = [_to_o(s) for s in slices]
    arr = (C.POINTER(_OCsr) * max(1, len(os_)))(*[C.pointer(o) for o in os_])
    oc = _OCsr()
    _pchk(_P().oracle_vconcat(arr, len(os_), C.byref(oc)), "vconcat")
    return _from_o(oc)


def port_gen_erdos_renyi(n: int, density: float, seed: int) -> Csr:
    o = _OCsr()
    _pchk(_P().oracle_gen_erdos_renyi(n, density, seed, C.byref(o)), "gen_erdos_renyi")
    return _from_o(o)


def port_gen_erdos_renyi_rect(nrows: int, ncols: int, density: float, seed: int) -> Csr:
    o = _OCsr()
    _pchk(_P().oracle_gen_erdos_renyi_rect(nrows, ncols, density, seed, C.byref(o)), "gen_er_rect")
    return _from_o(o)


def port_trident_rect(nrows, ncols, q, lam, rank) -> np.ndarray:
    r = np.zeros(4, np.int64)
    _P().oracle_trident_rect(nrows, ncols, q, lam, rank, r)
    return r


def port_extract(m, rect) -> Csr:
    o, t = _to_o(m), _OCsr()
    _pchk(_P().oracle_extract(C.byref(o), np.ascontiguousarray(rect, np.int64), C.byref(t)), "extract")
    return _from_o(t)


def port_column_normalize(m) -> Csr:
    c = Csr(m.nrows, m.ncols, np.array(m.rowptr, np.int64), np.array(m.colind, np.int64),
            np.array(m.values, np.float64))
    o = _to_o(c)
    _P().oracle_column_normalize(C.byref(o))
    return c


def port_elementwise_power(m, r: float) -> Csr:
    """csr.cpp:251-255: v = std::pow(v, r) per stored value. math.pow is the
    host libm's pow, bit-identical to the reference's (numpy's own power is
    not, and neither is the correctly rounded v*v for r = 2: glibc's pow is
    within ~0.52 ulp, not correctly rounded)."""
    v = np.array(m.values, np.float64)
    out = np.fromiter((math.pow(x, r) for x in v), np.float64, count=v.size)
    return Csr(m.nrows, m.ncols, np.array(m.rowptr, np.int64), np.array(m.colind, np.int64), out)


def port_mcl_poststep(c, theta: float, r: float) -> Csr:
    """apps.cpp:79-82 composed from the port's own steps."""
    return port_column_normalize(port_elementwise_power(port_prune(port_column_normalize(c), theta), r))


def port_prune(m, theta: float) -> Csr:
    o, r = _to_o(m), _OCsr()
    _pchk(_P().oracle_prune(C.byref(o), theta, C.byref(r)), "prune")
    return _from_o(r)


# ------------------------------------------------------------- comparisons
def pattern_equal(a, b) -> bool:
    """csr.cpp:365-368."""
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols)
            and np.array_equal(np.asarray(a.rowptr, np.int64), np.asarray(b.rowptr, np.int64))
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64)))


def allclose(a, b, rel_tol: float) -> bool:
    """csr.cpp:370-379: pattern equal and |x-y| <= tol*max(|x|,|y|) (purely relative)."""
    if not pattern_equal(a, b):
        return False
    x = np.asarray(a.values, np.float64)
    y = np.asarray(b.values, np.float64)
    ok = (x == y) | (np.abs(x - y) <= rel_tol * np.maximum(np.abs(x), np.abs(y)))
    return bool(ok.all())


def max_rel_err(a, b) -> float:
    x = np.asarray(a.values, np.float64)
    y = np.asarray(b.values, np.float64)
    if len(x) == 0:
        return 0.0
    d = np.abs(x - y)
    s = np.maximum(np.abs(x), np.abs(y))
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(d == 0, 0.0, d / s)
    return float(r.max())
