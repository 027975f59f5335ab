"""B200-native hot path of Trident (arXiv 2603.21444): local CSR x CSR SpGEMM,
trident / Sparse-SUMMA tile exchange and partial-C merge on sm_100a.

This module is the Python mirror of the reference's C++ interface for that path
(``/root/reference/proj/include/spgsim/{csr,partition,netmodel,algorithms}.hpp``):
same names, argument meaning and error behaviour. Every kernel runs on a B200
through the C ABI of ``lib/libspgb200.so`` (``include/spg/capi.h``); with no
library or no device the calls raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import SpgError, check

__all__ = [
    "CsrMatrix", "Device", "DeviceCsr", "SpgError", "spgemm_local", "spgeam", "vconcat", "column_normalize",
    "prune", "elementwise_power", "mcl_poststep", "pattern_equal", "allclose", "gen_erdos_renyi", "gen_erdos_renyi_rect", "gen_rmat", "transpose",
    "TridentGrid", "TopologySpec", "block_bounds", "make_tile_map", "partition", "reassemble", "trident_spgemm",
    "summa_spgemm", "oned_spgemm", "run_algo", "DriverResult", "make_report", "report_json", "trident_ledger", "payload_bytes", "default_device",
]

I64 = np.int64


# ----------------------------------------------------------------- CsrMatrix
@dataclass(eq=False)
class CsrMatrix:
    """Canonical CSR (csr.hpp:12-35): int64 rowptr/colind, float64 values."""

    nrows: int = 0
    ncols: int = 0
    rowptr: np.ndarray = field(default_factory=lambda: np.zeros(1, I64))
    colind: np.ndarray = field(default_factory=lambda: np.zeros(0, I64))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1]) if len(self.rowptr) else 0

    @staticmethod
    def zeros(nrows: int, ncols: int) -> "CsrMatrix":
        return CsrMatrix(int(nrows), int(ncols), np.zeros(int(nrows) + 1, I64))

    @staticmethod
    def identity(n: int) -> "CsrMatrix":
        return CsrMatrix(n, n, np.arange(n + 1, dtype=I64), np.arange(n, dtype=I64), np.ones(n))

    @staticmethod
    def of(m) -> "CsrMatrix":
        """Adopt any object with nrows/ncols/rowptr/colind/values."""
        if isinstance(m, CsrMatrix):
            return m
        return CsrMatrix(int(m.nrows), int(m.ncols), np.asarray(m.rowptr, I64), np.asarray(m.colind, I64),
                         np.asarray(m.values, np.float64))

    def check_canonical(self) -> None:
        """csr.cpp:30-50; raises SpgError(kind='Error')."""
        def bad(msg):
            raise SpgError(1, msg)
        if self.nrows < 0 or self.ncols < 0:
            bad("negative dimension")
        rp, ci = np.asarray(self.rowptr), np.asarray(self.colind)
        if len(rp) != self.nrows + 1:
            bad("rowptr length != nrows+1")
        if rp[0] != 0:
            bad("rowptr[0] != 0")
        if len(ci) != len(self.values):
            bad("colind/values length mismatch")
        if rp[-1] != len(ci):
            bad("rowptr[nrows] != nnz")
        d = np.diff(rp)
        if (d < 0).any():
            bad(f"rowptr not non-decreasing at row {int(np.argmax(d < 0))}")
        if len(ci):
            rows = np.repeat(np.arange(self.nrows), d)
            oob = (ci < 0) | (ci >= self.ncols)
            if oob.any():
                bad(f"column index out of range in row {int(rows[np.argmax(oob)])}")
            same_row = rows[1:] == rows[:-1]
            dec = same_row & (ci[1:] <= ci[:-1])
            if dec.any():
                bad(f"columns not strictly increasing in row {int(rows[1:][np.argmax(dec)])}")

    def is_canonical(self) -> bool:
        try:
            self.check_canonical()
            return True
        except SpgError:
            return False

    def __eq__(self, o) -> bool:
        return (self.nrows == o.nrows and self.ncols == o.ncols and np.array_equal(self.rowptr, o.rowptr)
                and np.array_equal(self.colind, o.colind) and np.array_equal(self.values, o.values))


def pattern_equal(a, b) -> bool:
    """csr.cpp:365-368."""
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols)
            and np.array_equal(np.asarray(a.rowptr, I64), np.asarray(b.rowptr, I64))
            and np.array_equal(np.asarray(a.colind, I64), np.asarray(b.colind, I64)))


def allclose(a, b, rel_tol: float) -> bool:
    """csr.cpp:370-379 (purely relative tolerance)."""
    if not pattern_equal(a, b):
        return False
    x, y = np.asarray(a.values, np.float64), np.asarray(b.values, np.float64)
    return bool(((x == y) | (np.abs(x - y) <= rel_tol * np.maximum(np.abs(x), np.abs(y)))).all())


# -------------------------------------------------------------- device layer
def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


class DeviceCsr:
    """Owning handle of a device CSR (int64 rowptr, int32 colind, f64 values)."""

    def __init__(self, dev: "Device", handle: int):
        self.dev = dev
        self.h = C.c_void_p(handle)

    @property
    def shape3(self):
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        check(_capi.lib().spg_csr_shape(self.h, C.byref(r), C.byref(c), C.byref(n)))
        return r.value, c.value, n.value

    @property
    def nnz(self) -> int:
        return self.shape3[2]

    def download(self, colind_width: int = 8) -> CsrMatrix:
        r, c, n = self.shape3
        rp = np.empty(r + 1, I64)
        ci = np.empty(n, I64 if colind_width == 8 else np.int32)
        va = np.empty(n, np.float64)
        check(_capi.lib().spg_csr_download(self.dev.ctx, self.h, _ptr(rp), _ptr(ci) or None, colind_width,
                                           _ptr(va) or None))
        return CsrMatrix(r, c, rp, ci.astype(I64, copy=False), va)

    def check(self) -> None:
        check(_capi.lib().spg_csr_check(self.dev.ctx, self.h))

    def checksum(self):
        """report.cpp:11-26 result_checksum on the device -> (nnz, hash)."""
        n, h = C.c_int64(), C.c_uint64()
        check(_capi.lib().spg_result_checksum(self.dev.ctx, self.h, C.byref(n), C.byref(h)))
        return n.value, h.value

    def free(self) -> None:
        if self.h and self.h.value:
            _capi.lib().spg_csr_free(self.h)
            self.h = C.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Device:
    """One B200 context: stream, memory pool and kernel timers (spg_ctx)."""

    def __init__(self, device: int = 0):
        ctx = C.c_void_p()
        check(_capi.lib().spg_init(device, C.byref(ctx)))
        self.ctx = ctx
        self.index = device

    @staticmethod
    def count() -> int:
        n = C.c_int()
        check(_capi.lib().spg_device_count(C.byref(n)))
        return n.value

    @property
    def stream(self) -> int:
        return _capi.lib().spg_ctx_stream(self.ctx) or 0

    def synchronize(self) -> None:
        check(_capi.lib().spg_ctx_synchronize(self.ctx))

    def upload(self, m, colind_width: int = 8) -> DeviceCsr:
        m = CsrMatrix.of(m) if not isinstance(m, CsrMatrix) else m
        rp = np.ascontiguousarray(m.rowptr, I64)
        ci = np.ascontiguousarray(m.colind, I64 if colind_width == 8 else np.int32)
        va = np.ascontiguousarray(m.values, np.float64)
        h = C.c_void_p()
        check(_capi.lib().spg_csr_upload(self.ctx, int(m.nrows), int(m.ncols), _ptr(rp), _ptr(ci) or None,
                                         colind_width, _ptr(va) or None, C.byref(h)))
        return DeviceCsr(self, h.value)

    def zeros(self, nrows: int, ncols: int) -> DeviceCsr:
        h = C.c_void_p()
        check(_capi.lib().spg_csr_zeros(self.ctx, nrows, ncols, C.byref(h)))
        return DeviceCsr(self, h.value)

    def _out(self, fn, *args) -> DeviceCsr:
        h = C.c_void_p()
        check(fn(self.ctx, *args, C.byref(h)))
        return DeviceCsr(self, h.value)

    def spgemm(self, a: DeviceCsr, b: DeviceCsr) -> DeviceCsr:
        return self._out(_capi.lib().spg_spgemm, a.h, b.h)

    def spgemm_host_to_host(self, a, b, batches: int = 0, cap: int | None = None) -> CsrMatrix:
        """spgemm_local (csr.cpp:132-165) host to host through spg_spgemm_host_to_host:
        A in row batches, each batch's download overlapping the next batch's
        multiply. cap = room for C's entries (default: the product count, an
        upper bound); retried once with the exact nnz if it was too small."""
        a, b = CsrMatrix.of(a), CsrMatrix.of(b)
        same = a is b
        ar, ac, av = (np.ascontiguousarray(a.rowptr, I64), np.ascontiguousarray(a.colind, I64),
                      np.ascontiguousarray(a.values, np.float64))
        br, bc, bv = (ar, ac, av) if same else (np.ascontiguousarray(b.rowptr, I64),
                                                np.ascontiguousarray(b.colind, I64),
                                                np.ascontiguousarray(b.values, np.float64))
        if cap is None:
            blen = np.diff(br)
            cap = int(blen[ac].sum()) if len(ac) else 0
        lib = _capi.lib()
        for _ in range(2):
            rp = np.empty(int(a.nrows) + 1, I64)
            ci = np.empty(max(1, cap), I64)
            va = np.empty(max(1, cap), np.float64)
            nnz = C.c_int64()
            st = lib.spg_spgemm_host_to_host(self.ctx, int(a.nrows), int(a.ncols), _ptr(ar), _ptr(ac) or None,
                                             _ptr(av) or None, int(b.nrows), int(b.ncols), _ptr(br),
                                             _ptr(bc) or None, _ptr(bv) or None, 8, int(batches), int(cap),
                                             _ptr(rp), _ptr(ci), _ptr(va), C.byref(nnz))
            if st == 0:
                return CsrMatrix(int(a.nrows), int(b.ncols), rp, ci[:nnz.value].copy(), va[:nnz.value].copy())
            if nnz.value <= cap:
                check(st)
            cap = nnz.value
        check(st)

    def products(self, a: DeviceCsr, b: DeviceCsr) -> int:
        p = C.c_int64()
        check(_capi.lib().spg_spgemm_products(self.ctx, a.h, b.h, C.byref(p)))
        return p.value

    def spgeam(self, a: DeviceCsr, b: DeviceCsr) -> DeviceCsr:
        return self._out(_capi.lib().spg_spgeam, a.h, b.h)

    def vconcat(self, slices) -> DeviceCsr:
        arr = (C.c_void_p * max(1, len(slices)))(*[s.h.value for s in slices])
        return self._out(_capi.lib().spg_vconcat, arr, len(slices))

    def extract(self, m: DeviceCsr, r0, r1, c0, c1) -> DeviceCsr:
        return self._out(_capi.lib().spg_csr_extract, m.h, r0, r1, c0, c1)

    def copy(self, m: DeviceCsr) -> DeviceCsr:
        return self._out(_capi.lib().spg_csr_copy, m.h)

    def partition(self, m: DeviceCsr, scheme: str, procs: int, gpus_per_node: int, devices=None):
        """Device tile store: partition.cpp:161-222 on the GPU (spg_partition).
        m lives on this device; tile r is built on devices[r % len(devices)]
        (default: this device). -> (tiles, TileMap)."""
        devs = list(devices) if devices else [self]
        ctxs = (C.c_void_p * len(devs))(*[d.ctx.value for d in devs])
        out = (C.c_void_p * max(1, procs))()
        check(_capi.lib().spg_partition(ctxs, len(devs), m.h, _SCHEMES.get(scheme, -1), procs, gpus_per_node, out))
        r, c, _ = m.shape3
        return [DeviceCsr(devs[t % len(devs)], out[t]) for t in range(procs)], make_tile_map(r, c, scheme, procs,
                                                                                                 gpus_per_node)

    def reassemble(self, tiles, tm: "TileMap") -> DeviceCsr:
        """Device tile store: partition.cpp:224-261 on the GPU (spg_reassemble);
        tiles may live on any device, the result on this one."""
        arr = (C.c_void_p * max(1, len(tiles)))(*[t.h.value for t in tiles])
        return self._out(_capi.lib().spg_reassemble, arr, len(tiles), int(tm.nrows), int(tm.ncols),
                         _SCHEMES.get(tm.scheme, -1), tm.procs, int(tm.gpus_per_node) if tm.scheme == "trident" else 1)

    def column_normalize(self, m: DeviceCsr) -> None:
        check(_capi.lib().spg_column_normalize(self.ctx, m.h))

    def prune(self, m: DeviceCsr, theta: float) -> DeviceCsr:
        return self._out(_capi.lib().spg_prune, m.h, float(theta))

    def elementwise_power(self, m: DeviceCsr, exponent: float) -> None:
        check(_capi.lib().spg_elementwise_power(self.ctx, m.h, float(exponent)))

    def mcl_poststep(self, c: DeviceCsr, prune_threshold: float, inflation: float) -> DeviceCsr:
        """apps.cpp:79-82: column_normalize(power(prune(column_normalize(c)))), fused."""
        return self._out(_capi.lib().spg_mcl_poststep, c.h, float(prune_threshold), float(inflation))

    # kernel timing (CUDA events on the context stream)
    def timing(self, on: bool = True) -> None:
        check(_capi.lib().spg_timing_enable(self.ctx, 1 if on else 0))

    def timing_reset(self) -> None:
        check(_capi.lib().spg_timing_reset(self.ctx))

    def timing_read(self) -> dict:
        cap = 64
        names = C.create_string_buffer(8192)
        launches = (C.c_int64 * cap)()
        ms = (C.c_double * cap)()
        n = _capi.lib().spg_timing_read(self.ctx, names, 8192, launches, ms, cap)
        if n < 0:
            check(1)
        keys = names.raw.split(b"\0")[:n]
        return {k.decode(): (int(launches[i]), float(ms[i])) for i, k in enumerate(keys)}

    def close(self) -> None:
        if self.ctx and self.ctx.value:
            _capi.lib().spg_finalize(self.ctx)
            self.ctx = C.c_void_p(0)


_devices: dict = {}


def default_device(index: int = 0) -> Device:
    if index not in _devices:
        _devices[index] = Device(index)
    return _devices[index]


# ------------------------------------------------------------ host-facing API
def spgemm_local(a, b) -> CsrMatrix:
    """csr.hpp:64 — C = A*B on the B200 (pattern and values identical to the reference)."""
    if int(a.ncols) != int(b.nrows):
        raise SpgError(2, f"spgemm: a.ncols={a.ncols} != b.nrows={b.nrows}")
    d = default_device()
    da, db = d.upload(a), d.upload(b)
    return d.spgemm(da, db).download()


def spgeam(a, b) -> CsrMatrix:
    """csr.hpp:67 — C = A + B on the B200."""
    if int(a.nrows) != int(b.nrows) or int(a.ncols) != int(b.ncols):
        raise SpgError(2, "spgeam: shape mismatch")
    d = default_device()
    return d.spgeam(d.upload(a), d.upload(b)).download()


def column_normalize(a) -> CsrMatrix:
    d = default_device()
    m = d.upload(a)
    d.column_normalize(m)
    return m.download()


def prune(a, threshold: float) -> CsrMatrix:
    if threshold < 0:
        raise SpgError(3, "prune: negative threshold")
    d = default_device()
    return d.prune(d.upload(a), threshold).download()


def elementwise_power(a, exponent: float) -> CsrMatrix:
    """csr.cpp:251-255."""
    d = default_device()
    m = d.upload(a)
    d.elementwise_power(m, exponent)
    return m.download()


def mcl_poststep(c, prune_threshold: float = 0.002, inflation: float = 2.0) -> CsrMatrix:
    """The post-step of one MCL iteration (apps.cpp:79-82) on the GPU."""
    d = default_device()
    return d.mcl_poststep(d.upload(c), prune_threshold, inflation).download()


def vconcat(slices) -> CsrMatrix:
    """csr.cpp:348-363 data effect (host arrays)."""
    if not slices:
        return CsrMatrix(0, 0)
    nc = int(slices[0].ncols)
    if any(int(s.ncols) != nc for s in slices):
        raise SpgError(2, "vconcat: column count mismatch")
    rp = [np.zeros(1, I64)]
    base = 0
    for s in slices:
        rp.append(np.asarray(s.rowptr[1:], I64) + base)
        base += int(s.rowptr[-1])
    return CsrMatrix(sum(int(s.nrows) for s in slices), nc, np.concatenate(rp),
                     np.concatenate([np.asarray(s.colind, I64) for s in slices]),
                     np.concatenate([np.asarray(s.values, np.float64) for s in slices]))


# ---------------------------------------------------------------- generators
class _XCsr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("rowptr", C.POINTER(C.c_int64)), ("colind", C.POINTER(C.c_int64)),
                ("values", C.POINTER(C.c_double))]


_xlib = None


def _x():
    global _xlib
    if _xlib is None:
        if not os.path.exists(_capi.CXX_LIB_PATH):
            raise RuntimeError(f"{_capi.CXX_LIB_PATH} not built; run make")
        L = C.CDLL(_capi.CXX_LIB_PATH)
        L.spgx_last_error.restype = C.c_char_p
        P = C.POINTER(_XCsr)
        L.spgx_free.argtypes = [P]
        L.spgx_gen_erdos_renyi.argtypes = [C.c_int64, C.c_double, C.c_uint64, P]
        L.spgx_gen_erdos_renyi_rect.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, P]
        L.spgx_gen_rmat.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64, P]
        L.spgx_transpose.argtypes = [P, P]
        _xlib = L
    return _xlib


def _take(x: _XCsr) -> CsrMatrix:
    rp = np.ctypeslib.as_array(x.rowptr, shape=(x.nrows + 1,)).copy()
    ci = np.ctypeslib.as_array(x.colind, shape=(x.nnz,)).copy() if x.nnz else np.zeros(0, I64)
    va = np.ctypeslib.as_array(x.values, shape=(x.nnz,)).copy() if x.nnz else np.zeros(0)
    _x().spgx_free(C.byref(x))
    return CsrMatrix(x.nrows, x.ncols, rp, ci, va)


def _gen(fn, *args) -> CsrMatrix:
    x = _XCsr()
    rc = fn(*args, C.byref(x))
    if rc != 0:
        raise SpgError(3, _x().spgx_last_error().decode())
    return _take(x)


def gen_erdos_renyi(n: int, density: float, seed: int) -> CsrMatrix:
    """csr.cpp:257-279 (same SplitMix64 stream, same matrix), multithreaded."""
    return _gen(_x().spgx_gen_erdos_renyi, n, density, seed)


def gen_erdos_renyi_rect(nrows: int, ncols: int, density: float, seed: int) -> CsrMatrix:
    return _gen(_x().spgx_gen_erdos_renyi_rect, nrows, ncols, density, seed)


def gen_rmat(scale: int, edge_factor: int = 16, seed: int = 1, perm_seed: int = 2) -> CsrMatrix:
    return _gen(_x().spgx_gen_rmat, scale, edge_factor, seed, perm_seed)


def transpose(a) -> CsrMatrix:
    a = CsrMatrix.of(a)
    rp, ci, va = (np.ascontiguousarray(a.rowptr, I64), np.ascontiguousarray(a.colind, I64),
                  np.ascontiguousarray(a.values, np.float64))
    xin = _XCsr(a.nrows, a.ncols, a.nnz, rp.ctypes.data_as(C.POINTER(C.c_int64)),
                ci.ctypes.data_as(C.POINTER(C.c_int64)), va.ctypes.data_as(C.POINTER(C.c_double)))
    x = _XCsr()
    if _x().spgx_transpose(C.byref(xin), C.byref(x)) != 0:
        raise SpgError(1, _x().spgx_last_error().decode())
    return _take(x)


# ------------------------------------------------------------- partitioning
def _isqrt_exact(v: int) -> int:
    r = math.isqrt(v) if v >= 0 else -1
    return r if r >= 0 and r * r == v else -1


@dataclass
class TridentGrid:
    """partition.hpp:18-35: q x q x lambda grid, rank = (i*q + j)*lambda + k."""

    procs: int
    gpus_per_node: int
    q: int

    @staticmethod
    def create(procs: int, gpus_per_node: int) -> "TridentGrid":
        q = C.c_int()
        check(_capi.lib().spg_trident_grid(procs, gpus_per_node, C.byref(q)))
        return TridentGrid(procs, gpus_per_node, q.value)

    def rank_of(self, i, j, k) -> int:
        return (i * self.q + j) * self.gpus_per_node + k

    def coords_of(self, rank):
        node = rank // self.gpus_per_node
        return node // self.q, node % self.q, rank % self.gpus_per_node

    def node_of(self, rank) -> int:
        return rank // self.gpus_per_node

    def rounds(self) -> int:
        return self.q


@dataclass
class TopologySpec:
    """Wire widths of netmodel.hpp:24-25 (the alpha-beta clock is not modeled)."""

    gpus_per_node: int = 4
    index_width: int = 4
    value_width: int = 8

    def payload_bytes(self, rows: int, nnz: int) -> int:
        return payload_bytes(rows, nnz, self.index_width, self.value_width)


def payload_bytes(rows: int, nnz: int, iw: int = 4, vw: int = 8) -> int:
    """netmodel.hpp:37-39."""
    return nnz * (iw + vw) + (rows + 1) * iw


def block_bounds(dim: int, nblocks: int) -> np.ndarray:
    """partition.cpp:74-81 — first dim % nblocks blocks get one extra."""
    sizes = np.full(nblocks, dim // nblocks, I64)
    sizes[: dim % nblocks] += 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(I64)


@dataclass
class TileMap:
    scheme: str
    procs: int
    gpus_per_node: int
    nrows: int
    ncols: int
    row_bounds: np.ndarray
    col_bounds: np.ndarray
    tiles: np.ndarray  # (procs, 4): row_begin, row_end, col_begin, col_end


_SCHEMES = {"trident": 0, "grid2d": 1, "summa": 1, "rows1d": 2, "oned": 2}


def tile_rects(nrows: int, ncols: int, scheme: str, procs: int, gpus_per_node: int) -> np.ndarray:
    """The rectangles of make_tile_map as computed by the C ABI (spg_tile_rects)."""
    out = np.zeros((max(procs, 1), 4), I64)
    check(_capi.lib().spg_tile_rects(nrows, ncols, _SCHEMES.get(scheme, -1), procs, gpus_per_node,
                                     out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out[:procs]


def make_tile_map(nrows: int, ncols: int, scheme: str, procs: int, gpus_per_node: int) -> TileMap:
    """partition.cpp:95-159."""
    if procs <= 0:
        raise SpgError(4, "partition: process count must be positive")
    tiles = np.zeros((procs, 4), I64)
    if scheme == "trident":
        g = TridentGrid.create(procs, gpus_per_node)
        coarse = block_bounds(nrows, g.q)
        cb = block_bounds(ncols, g.q)
        rb = [0]
        for i in range(g.q):
            fine = block_bounds(int(coarse[i + 1] - coarse[i]), g.gpus_per_node)
            rb += [int(coarse[i] + fine[k]) for k in range(1, g.gpus_per_node + 1)]
        rb = np.array(rb, I64)
        for r in range(procs):
            i, j, k = g.coords_of(r)
            f = i * g.gpus_per_node + k
            tiles[r] = (rb[f], rb[f + 1], cb[j], cb[j + 1])
        lam = gpus_per_node
    elif scheme == "grid2d":
        pr = _isqrt_exact(procs)
        if pr < 0:
            raise SpgError(4, f"grid2d: P={procs} is not a perfect square")
        rb, cb = block_bounds(nrows, pr), block_bounds(ncols, pr)
        for r in range(procs):
            tiles[r] = (rb[r // pr], rb[r // pr + 1], cb[r % pr], cb[r % pr + 1])
        lam = 1
    else:
        rb, cb = block_bounds(nrows, procs), np.array([0, ncols], I64)
        for r in range(procs):
            tiles[r] = (rb[r], rb[r + 1], 0, ncols)
        lam = 1
    return TileMap(scheme, procs, lam, nrows, ncols, rb, cb, tiles)


def extract(m, rect) -> CsrMatrix:
    """One tile of partition.cpp:161-222 (local indices)."""
    r0, r1, c0, c1 = (int(x) for x in rect)
    rp = np.asarray(m.rowptr, I64)
    lo, hi = int(rp[r0]), int(rp[r1])
    ci = np.asarray(m.colind, I64)[lo:hi]
    va = np.asarray(m.values, np.float64)[lo:hi]
    rows = np.repeat(np.arange(r1 - r0), np.diff(rp[r0:r1 + 1]))
    keep = (ci >= c0) & (ci < c1)
    cnt = np.bincount(rows[keep], minlength=r1 - r0)
    return CsrMatrix(r1 - r0, c1 - c0, np.concatenate([[0], np.cumsum(cnt)]).astype(I64), ci[keep] - c0, va[keep])


def partition(m, scheme: str, procs: int, gpus_per_node: int):
    """-> (tiles, TileMap)."""
    tm = make_tile_map(int(m.nrows), int(m.ncols), scheme, procs, gpus_per_node)
    return [extract(m, tm.tiles[r]) for r in range(procs)], tm


def reassemble(tiles, tm: TileMap) -> CsrMatrix:
    """partition.cpp:224-261."""
    if len(tiles) != tm.procs:
        raise SpgError(5, f"reassemble: expected {tm.procs} tiles, got {len(tiles)}")
    for r, t in enumerate(tiles):
        r0, r1, c0, c1 = tm.tiles[r]
        if int(t.nrows) != r1 - r0 or int(t.ncols) != c1 - c0:
            raise SpgError(5, f"reassemble: tile {r} does not match its map rectangle")
    rows_l, cols_l, vals_l = [], [], []
    for r, t in enumerate(tiles):
        r0, _, c0, _ = tm.tiles[r]
        rp = np.asarray(t.rowptr, I64)
        rows_l.append(np.repeat(np.arange(int(t.nrows), dtype=I64) + r0, np.diff(rp)))
        cols_l.append(np.asarray(t.colind, I64) + c0)
        vals_l.append(np.asarray(t.values, np.float64))
    rows = np.concatenate(rows_l) if rows_l else np.zeros(0, I64)
    cols = np.concatenate(cols_l) if cols_l else np.zeros(0, I64)
    vals = np.concatenate(vals_l) if vals_l else np.zeros(0)
    order = np.lexsort((cols, rows))
    cnt = np.bincount(rows, minlength=tm.nrows)
    return CsrMatrix(tm.nrows, tm.ncols, np.concatenate([[0], np.cumsum(cnt)]).astype(I64), cols[order], vals[order])


# ---------------------------------------------------------- ledger (host)
def trident_ledger(grid: TridentGrid, a_shapes, b_shapes, iw: int = 4, vw: int = 8) -> np.ndarray:
    """Reference CommLedger of trident_spgemm (engine.cpp:228-302 for the plan of
    algorithms.cpp:53-74). a_shapes/b_shapes: per rank (rows, nnz).
    -> uint64 array [rank, dir(0 sent,1 recv), class(0 LI,1 GI), (messages, nnz, bytes)]."""
    P, lam, q = grid.procs, grid.gpus_per_node, grid.q
    L = np.zeros((P, 2, 2, 3), np.uint64)
    node = lambda r: r // lam  # noqa: E731

    def cls(s, r):
        return 0 if node(s) == node(r) else 1

    def transfer(s, r, rows, nnz):
        if s == r:
            return
        c = cls(s, r)
        b = payload_bytes(rows, nnz, iw, vw)
        L[s, 0, c] += np.array([1, nnz, b], np.uint64)
        L[r, 1, c] += np.array([1, nnz, b], np.uint64)

    def control(s, r):
        if s == r:
            return
        c = cls(s, r)
        L[s, 0, c, 0] += 1
        L[r, 1, c, 0] += 1

    for rnd in range(q):
        for rank in range(P):
            i, j, k = grid.coords_of(rank)
            s = (rnd + i + j) % q
            oa, ob = grid.rank_of(i, s, k), grid.rank_of(s, j, k)
            for o, shp in ((oa, a_shapes), (ob, b_shapes)):
                if o != rank:
                    control(rank, o)
                    transfer(o, rank, *shp[o])
        for nd in range(q * q):
            for k in range(lam):
                for k2 in range(lam):
                    if k == k2:
                        continue
                    send, recv = nd * lam + k2, nd * lam + k
                    i, j, kk = grid.coords_of(send)
                    ob = grid.rank_of((rnd + i + j) % q, j, kk)
                    transfer(send, recv, *b_shapes[ob])
    return L


EVENT_NAMES = ("enqueue-request", "serve-request", "transfer-complete", "allgather-complete", "compute-complete")
LINK_NAMES = ("SELF", "LI", "GI")


@dataclass
class DriverResult:
    """algorithms.hpp:32-38; ledger as the uint64 array of trident_ledger,
    built from the tiles the ranks actually consumed; timeline: (procs,
    rounds, 4) ms [exchange, exposed wait, multiply, merge]; events: the
    measured TimelineEvents (engine.hpp:25-38) as dicts, times in seconds from
    each rank's start; xfer: (procs, 4) [device bytes pulled, pull span ms,
    tiles pulled, tiles of other ranks read in place]."""

    c: CsrMatrix
    ledger: np.ndarray
    timeline: np.ndarray
    makespan: float
    rounds: int
    checksum: tuple | None = None  # (nnz, hash) of C, result_checksum computed on the device
    events: list = field(default_factory=list)
    xfer: np.ndarray | None = None

    def to_jsonl(self) -> str:
        """EventTimeline::to_jsonl (engine.cpp:25-41): one JSON object per
        event, keys in the reference's order."""
        out = []
        for e in self.events:
            out.append(json.dumps({"type": e["type"], "actors": [e["src"], e["dst"]], "round": e["round"],
                                   "t_start": e["t_start"], "t_end": e["t_end"], "bytes": e["bytes"],
                                   "operand": e["operand"], "link": e["link"], "nnz": e["nnz"]},
                                  separators=(",", ":")))
        return "".join(x + "\n" for x in out)


def _devices_for(procs: int):
    n = Device.count()
    if n == 0:
        raise SpgError(22, "no CUDA device")
    return [default_device(d) for d in range(min(n, procs))]


def _run_driver(fn, a, b, procs, lam, scheme, cmap, rounds, topo, delays=None) -> DriverResult:
    """Device tile store end to end: ONE upload of each global operand, the
    tiles split on the GPUs (spg_partition), the driver, the C tiles merged on
    device 0 (spg_reassemble) and ONE download of C. fn: the _ex driver
    (measured ledger + events) for trident / summa, spg_oned_spgemm else."""
    devs = _devices_for(procs)
    nctx = len(devs)
    plam = lam if scheme == "trident" else 1
    ga = devs[0].upload(a)
    gb = ga if b is a else devs[0].upload(b)
    da, _ = devs[0].partition(ga, scheme, procs, plam, devices=devs)
    db, _ = devs[0].partition(gb, scheme, procs, plam, devices=devs)
    del ga, gb
    ctxs = (C.c_void_p * nctx)(*[d.ctx.value for d in devs])
    ha = (C.c_void_p * procs)(*[x.h.value for x in da])
    hb = (C.c_void_p * procs)(*[x.h.value for x in db])
    hc = (C.c_void_p * procs)()
    cells = (_capi.LedgerCell * (procs * 4))()
    tl = (C.c_double * (procs * rounds * 4))()
    L = _capi.lib()
    events, xfer = [], None
    if fn in (L.spg_trident_spgemm_ex, L.spg_summa_spgemm_ex):
        cap = procs * rounds * 8 + 16
        ev = (_capi.Event * cap)()
        nev = C.c_int()
        xf = (C.c_double * (procs * 4))()
        if fn == L.spg_trident_spgemm_ex:
            d = np.asarray(delays if delays is not None else [], np.float64)
            dp = d.ctypes.data_as(C.POINTER(C.c_double)) if len(d) else None
            check(fn(ctxs, nctx, ha, hb, procs, lam, topo.index_width, topo.value_width, dp, len(d), hc, cells, tl,
                     ev, cap, C.byref(nev), xf))
        else:
            check(fn(ctxs, nctx, ha, hb, procs, lam, topo.index_width, topo.value_width, hc, cells, tl, ev, cap,
                     C.byref(nev), xf))
        for x in ev[:nev.value]:
            events.append({"type": EVENT_NAMES[x.type], "src": x.src, "dst": x.dst, "round": x.round,
                           "operand": "AB"[x.operand], "link": LINK_NAMES[x.link], "t_start": x.t_start,
                           "t_end": x.t_end, "nnz": x.nnz, "bytes": x.bytes})
        xfer = np.ctypeslib.as_array(xf).reshape(procs, 4).copy()
    else:
        check(fn(ctxs, nctx, ha, hb, procs, lam, topo.index_width, topo.value_width, hc, cells, tl))
    dc = [DeviceCsr(devs[r % nctx], hc[r]) for r in range(procs)]
    gc = devs[0].reassemble(dc, cmap)
    cs = gc.checksum()
    c = gc.download()
    led = np.array([[x.messages, x.nnz, x.bytes] for x in cells], np.uint64).reshape(procs, 2, 2, 3)
    tla = np.ctypeslib.as_array(tl).reshape(procs, rounds, 4).copy()
    makespan = float((tla[:, :, 1:].sum(axis=(1, 2))).max()) * 1e-3
    return DriverResult(c, led, tla, makespan, rounds, cs, events, xfer)


def trident_spgemm(a, b, grid: TridentGrid, topo: TopologySpec | None = None,
                   node_start_delay=None) -> DriverResult:
    """algorithms.cpp:24-101 on the GPUs of this box (rank r -> device r % ndev).
    node_start_delay: seconds per virtual node; that node's ranks start their
    pulls that much later on the device (engine.cpp:217-221)."""
    if int(a.ncols) != int(b.nrows):
        raise SpgError(2, f"trident_spgemm: a.ncols={a.ncols} != b.nrows={b.nrows}")
    topo = topo or TopologySpec(grid.gpus_per_node)
    cmap = make_tile_map(int(a.nrows), int(b.ncols), "trident", grid.procs, grid.gpus_per_node)
    if node_start_delay is not None and any(not (float(x) >= 0.0) for x in node_start_delay):
        raise SpgError(3, "trident_spgemm: node_start_delay must be >= 0")
    return _run_driver(_capi.lib().spg_trident_spgemm_ex, a, b, grid.procs, grid.gpus_per_node, "trident", cmap,
                       grid.q, topo, node_start_delay)


def summa_spgemm(a, b, procs: int, gpus_per_node: int, topo: TopologySpec | None = None) -> DriverResult:
    """algorithms.cpp:103-174."""
    if int(a.ncols) != int(b.nrows):
        raise SpgError(2, f"summa_spgemm: a.ncols={a.ncols} != b.nrows={b.nrows}")
    pr = _isqrt_exact(procs)
    if pr < 0:
        raise SpgError(4, f"summa: P={procs} is not a perfect square")
    topo = topo or TopologySpec(gpus_per_node)
    cmap = make_tile_map(int(a.nrows), int(b.ncols), "grid2d", procs, 1)
    return _run_driver(_capi.lib().spg_summa_spgemm_ex, a, b, procs, gpus_per_node, "grid2d", cmap, pr, topo)


def oned_spgemm(a, b, procs: int, gpus_per_node: int, topo: TopologySpec | None = None) -> DriverResult:
    """algorithms.cpp:176-269: sparsity-aware 1D (row-selective B fetch)."""
    if int(a.ncols) != int(b.nrows):
        raise SpgError(2, f"oned_spgemm: a.ncols={a.ncols} != b.nrows={b.nrows}")
    if procs <= 0:
        raise SpgError(4, "oned: P must be positive")
    topo = topo or TopologySpec(gpus_per_node)
    cmap = make_tile_map(int(a.nrows), int(b.ncols), "rows1d", procs, 1)
    return _run_driver(_capi.lib().spg_oned_spgemm, a, b, procs, gpus_per_node, "rows1d", cmap, 1, topo)


def make_report(dr: DriverResult, algo: str, procs: int, gpus_per_node: int, topo: TopologySpec | None = None,
                matrix_a: str = "", matrix_b: str = "", square: bool = False, seed: int = 0,
                tilemap: TileMap | None = None, verified: bool | None = None) -> dict:
    """RunReport (report.hpp, report.cpp:34-99) of a MEASURED run, same keys as
    the reference's to_json: config, rounds, makespan_seconds (measured device
    time, not the alpha-beta model), aggregate and per_process ledger,
    result {nrows, ncols, nnz, checksum} (result_checksum computed on the
    device), verified, tilemap. Added: "timeline" — per rank and round the
    measured [exchange_ms, exposed_wait_ms, multiply_ms, merge_ms], so measured
    timelines can be diffed against the modeled schedule."""
    topo = topo or TopologySpec(gpus_per_node)
    L = np.asarray(dr.ledger, np.uint64)
    P = L.shape[0]
    GI, LI = 1, 0
    rep = {"config": {"algo": algo, "procs": procs, "gpus_per_node": gpus_per_node, "matrix_a": matrix_a,
                      "matrix_b": matrix_b, "square": square, "seed": seed,
                      "topology": {"nodes": max(1, procs // max(1, gpus_per_node)), "gpus_per_node": gpus_per_node,
                                   "alpha_li": None, "alpha_gi": None, "beta_li": None, "beta_gi": None,
                                   "index_width": topo.index_width, "value_width": topo.value_width}},
           "rounds": dr.rounds, "makespan_seconds": dr.makespan}
    rep["aggregate"] = {name: {"messages": int(L[:, 0, c, 0].sum()), "nnz_sent": int(L[:, 0, c, 1].sum()),
                               "bytes_sent": int(L[:, 0, c, 2].sum())} for name, c in (("gi", GI), ("li", LI))}
    per = []
    done = np.asarray(dr.timeline)[:, :, 1:].sum(axis=(1, 2)) * 1e-3
    for r in range(P):
        row = {"rank": r, "node": r // max(1, gpus_per_node)}
        for pfx, c in (("gi_", GI), ("li_", LI)):
            row[pfx + "messages"] = int(L[r, 0, c, 0])
            row[pfx + "nnz_sent"] = int(L[r, 0, c, 1])
            row[pfx + "bytes_sent"] = int(L[r, 0, c, 2])
            row[pfx + "nnz_recv"] = int(L[r, 1, c, 1])
            row[pfx + "bytes_recv"] = int(L[r, 1, c, 2])
        row["completion_time"] = float(done[r])
        per.append(row)
    rep["per_process"] = per
    nnz, h = dr.checksum if dr.checksum is not None else (int(dr.c.nnz), None)
    rep["result"] = {"nrows": int(dr.c.nrows), "ncols": int(dr.c.ncols), "nnz": int(nnz),
                     "checksum": None if h is None else f"0x{h:016x}"}
    rep["verified"] = verified
    if tilemap is not None:
        rep["tilemap"] = {"scheme": tilemap.scheme, "procs": tilemap.procs, "gpus_per_node": tilemap.gpus_per_node,
                          "nrows": tilemap.nrows, "ncols": tilemap.ncols,
                          "row_bounds": [int(x) for x in tilemap.row_bounds],
                          "col_bounds": [int(x) for x in tilemap.col_bounds]}
    rep["timeline"] = [[[float(x) for x in rnd] for rnd in rank] for rank in np.asarray(dr.timeline)]
    return rep


def report_json(rep: dict) -> str:
    """RunReport::to_json layout (two-space indent, keys in the reference's order)."""
    import json
    return json.dumps(rep, indent=2)


def run_algo(algo: str, a, b, procs: int, gpus_per_node: int, topo: TopologySpec | None = None) -> DriverResult:
    """algorithms.cpp:271-280."""
    if algo == "trident":
        return trident_spgemm(a, b, TridentGrid.create(procs, gpus_per_node), topo)
    if algo == "summa":
        return summa_spgemm(a, b, procs, gpus_per_node, topo)
    if algo == "oned":
        return oned_spgemm(a, b, procs, gpus_per_node, topo)
    raise SpgError(3, f"run_algo: unknown algorithm '{algo}'")
