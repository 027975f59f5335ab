"""The one-process-per-GPU host path (paper_2603_21444_b200/dist.py) under
torch.distributed with the gloo backend, world_size 2, on CPU: each rank's
trident tiles equal the reference partition (partition.cpp:161-222), the
descriptor all-gather that RankExchange uses carries every rank's blob, the
per-rank products of the trident rounds add up to products(A, B), and the
per-rank ledger equals the reference CommLedger (algorithms.cpp:53-74)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle as O
    import paper_2603_21444_b200 as spg
    from paper_2603_21444_b200 import dist as sd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        a = O.port_gen_erdos_renyi(600, 0.02, 3)
        b = O.port_gen_erdos_renyi(600, 0.02, 4)
        res = {}
        # the N=2 grid of bench.py: (P, lambda) = (2, 2), q = 1
        procs, lam = sd.grid_for_gpus(WORLD)
        grid = spg.TridentGrid.create(procs, lam)
        at, bt = sd.rank_tiles(a, b, grid, rank)
        ref_a, _ = O.ref_partition(a, "trident", procs, lam) if O.ref_available() else (None, None)
        if ref_a is not None:
            ra = ref_a[rank]
            res["tile_equal"] = bool(np.array_equal(at.rowptr, ra.rowptr) and np.array_equal(at.colind, ra.colind)
                                     and np.array_equal(at.values, ra.values))
        # the descriptor exchange RankExchange performs (256 bytes per tile)
        blob = bytes([rank]) * 256 + bytes([rank + 100]) * 256
        got = [None] * WORLD
        dist.all_gather_object(got, blob)
        res["blobs_ok"] = all(g == bytes([r]) * 256 + bytes([r + 100]) * 256 for r, g in enumerate(got))
        # products of every rank's rounds, for the 2- and 8-rank grids
        for P, L in ((2, 2), (4, 1), (8, 2)):
            g = spg.TridentGrid.create(P, L)
            mine = [sd.rank_products(a, b, g, r) for r in range(P) if r % WORLD == rank]
            tot = [0] * WORLD
            dist.all_gather_object(tot, sum(mine))
            res[f"products_P{P}"] = int(sum(tot))
        res["products_ref"] = int(O.port_products(a, b))
        # per-rank ledger rows vs the reference simulator's CommLedger
        if O.ref_available():
            led = sd.ledger_for(a, b, grid)
            ref = O.ref_run_algo("trident", a, b, procs, lam, want_c=False)["ledger"]
            res["ledger_equal"] = bool(np.array_equal(led, ref))
        np.save(os.path.join(out_dir, f"r{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_trident_host_path(tmp_path):
    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    for r in range(WORLD):
        res = np.load(tmp_path / f"r{r}.npy", allow_pickle=True).item()
        assert res["blobs_ok"]
        for P in (2, 4, 8):
            assert res[f"products_P{P}"] == res["products_ref"], (P, res)
        if "tile_equal" in res:
            assert res["tile_equal"]
        if "ledger_equal" in res:
            assert res["ledger_equal"]
