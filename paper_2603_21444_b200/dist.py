"""One process per GPU: the trident exchange over CUDA IPC + NVLink.

Plumbing only: ``torch.distributed`` (gloo or nccl process group) carries the
256-byte IPC descriptors of every rank's tiles; after that each rank pulls its
peers' tiles straight out of their HBM inside ``spg_trident_rank`` (C ABI), so
the data path has no collective. Mirrors the rank-local part of
``trident_spgemm`` (reference algorithms.cpp:53-92).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import check
from . import CsrMatrix, DeviceCsr, Device, TridentGrid, extract, make_tile_map, trident_ledger


def grid_for_gpus(n: int) -> tuple[int, int]:
    """(procs, gpus_per_node) used for an n-GPU box: the legal trident grids of
    SURVEY §0.3 item 8 — 1:(1,1) 2:(2,2) 4:(4,4) 8:(8,2)."""
    return {1: (1, 1), 2: (2, 2), 4: (4, 4), 8: (8, 2)}.get(n, (n, n))


def rank_tiles(a, b, grid: TridentGrid, rank: int):
    """This rank's A and B tiles (trident partition, local indices)."""
    ta = make_tile_map(int(a.nrows), int(a.ncols), "trident", grid.procs, grid.gpus_per_node)
    tb = make_tile_map(int(b.nrows), int(b.ncols), "trident", grid.procs, grid.gpus_per_node)
    return extract(a, ta.tiles[rank]), extract(b, tb.tiles[rank])


def all_shapes(a, b, grid: TridentGrid):
    """Per-rank (rows, nnz) of every A and B tile, computed from the global
    matrices without materialising the tiles (for the ledger)."""
    out = []
    for m in (a, b):
        tm = make_tile_map(int(m.nrows), int(m.ncols), "trident", grid.procs, grid.gpus_per_node)
        rp, ci = np.asarray(m.rowptr), np.asarray(m.colind)
        shp = []
        for r0, r1, c0, c1 in tm.tiles:
            lo, hi = int(rp[r0]), int(rp[r1])
            cols = ci[lo:hi]
            shp.append((int(r1 - r0), int(((cols >= c0) & (cols < c1)).sum())))
        out.append(shp)
    return out


class RankExchange:
    """Owns this rank's shareable tiles and the IPC views of every peer's."""

    def __init__(self, dev: Device, a_tile, b_tile, rank: int, world: int, allgather_bytes):
        """``allgather_bytes(b: bytes) -> list[bytes]`` gathers one blob per rank
        (e.g. torch.distributed.all_gather_object)."""
        self.dev, self.rank, self.world = dev, rank, world
        L = _capi.lib()
        da, db = dev.upload(a_tile), dev.upload(b_tile)
        self.own = []
        for d in (da, db):
            h = C.c_void_p()
            check(L.spg_csr_make_shareable(dev.ctx, d.h, C.byref(h)))
            self.own.append(DeviceCsr(dev, h.value))
        blobs = []
        for d in self.own:
            buf = C.create_string_buffer(_capi.IPC_BYTES)
            check(L.spg_csr_ipc_export(d.h, buf))
            blobs.append(buf.raw)
        gathered = allgather_bytes(b"".join(blobs))
        self.views_a, self.views_b = [], []
        for r, g in enumerate(gathered):
            if r == rank:
                self.views_a.append(self.own[0])
                self.views_b.append(self.own[1])
                continue
            for k, lst in ((0, self.views_a), (1, self.views_b)):
                h = C.c_void_p()
                blob = g[k * _capi.IPC_BYTES:(k + 1) * _capi.IPC_BYTES]
                check(L.spg_csr_ipc_open(dev.ctx, blob, C.byref(h)))
                lst.append(DeviceCsr(dev, h.value))

    def trident_step(self, procs: int, gpus_per_node: int, q: int):
        """One trident C tile for this rank -> (DeviceCsr, timeline[q,4] ms)."""
        L = _capi.lib()
        va = (C.c_void_p * procs)(*[v.h.value for v in self.views_a])
        vb = (C.c_void_p * procs)(*[v.h.value for v in self.views_b])
        out = C.c_void_p()
        tl = (C.c_double * (q * 4))()
        check(L.spg_trident_rank(self.dev.ctx, self.rank, procs, gpus_per_node, va, vb, C.byref(out), tl))
        return DeviceCsr(self.dev, out.value), np.ctypeslib.as_array(tl).reshape(q, 4).copy()

    def reload(self, a_host, b_host):
        """Refill this rank's shareable A/B tiles from host arrays (pinned by
        the caller) in place, so the peers' IPC views stay valid (e2e leg).

        Contract: the peers may still be pulling this rank's tiles for the
        previous trident_step; the caller must order the reload after every
        rank's step (bench.py: a dist.barrier() once each rank has its C tile
        downloaded, which the stream-synchronous download implies)."""
        L = _capi.lib()
        for d, m in zip(self.own, (a_host, b_host)):
            check(L.spg_csr_upload_into(self.dev.ctx, d.h, m[0].ctypes.data, m[1].ctypes.data, m[2].ctypes.data))

    def close(self):
        for lst in (self.views_a, self.views_b):
            for i, v in enumerate(lst):
                if i != self.rank:
                    v.free()
        for d in self.own:
            d.free()


def rank_products(a, b, grid: TridentGrid, rank: int) -> int:
    """Products of all of this rank's local multiplies (sum over its q rounds
    of products(A_{i,s,k}, B_{s,j})), from the global matrices (host numpy)."""
    q, lam = grid.q, grid.gpus_per_node
    i, j, k = grid.coords_of(rank)
    tm_a = make_tile_map(int(a.nrows), int(a.ncols), "trident", grid.procs, lam)
    tm_b = make_tile_map(int(b.nrows), int(b.ncols), "trident", grid.procs, lam)
    cb = np.asarray(tm_b.col_bounds, np.int64)
    brp, bci = np.asarray(b.rowptr, np.int64), np.asarray(b.colind, np.int64)
    brow = np.repeat(np.arange(int(b.nrows)), np.diff(brp))
    lo, hi = cb[j], cb[j + 1]
    keep = (bci >= lo) & (bci < hi)
    blen = np.bincount(brow[keep], minlength=int(b.nrows))  # nnz of B rows inside column block j
    total = 0
    for r in range(q):
        s = (r + i + j) % q
        r0, r1, c0, c1 = tm_a.tiles[grid.rank_of(i, s, k)]
        arp, aci = np.asarray(a.rowptr, np.int64), np.asarray(a.colind, np.int64)
        cols = aci[int(arp[r0]):int(arp[r1])]
        cols = cols[(cols >= c0) & (cols < c1)]
        total += int(blen[cols].sum())
    return total


def ledger_for(a, b, grid: TridentGrid, iw: int = 4, vw: int = 8) -> np.ndarray:
    sa, sb = all_shapes(a, b, grid)
    return trident_ledger(grid, sa, sb, iw, vw)


__all__ = ["grid_for_gpus", "rank_tiles", "all_shapes", "rank_products", "RankExchange", "ledger_for", "CsrMatrix"]
