"""One process per GPU (paper_2603_21444_b200/dist.py + spg_trident_rank over
CUDA IPC): every rank owns its trident tiles in its own GPU's HBM, exports
them, opens its peers' over NVLink and runs its rounds; rank 0 gathers the C
tiles and reassembles C. C must equal the reference's spgemm_local product
(csr.cpp:132-165) — bit-exact, since a rank's rounds run as one k-ordered
multiply — for the N=2 grid (P, lambda) = (2, 2) and, on a 4-GPU box, the
N=4 grid (4, 4) and the q=2 grid (4, 1). Skips with fewer GPUs than ranks.
Each grid runs with the peer slices pulled by the copy engines
(SPG_PULL_CE=1) and by the SM pull kernel (SPG_PULL_CE=0); by default
vconcat picks the SMs for >= 3 remote slices."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, pickle
sys.path.insert(0, {root!r})
import numpy as np
import torch.distributed as dist
import oracle as O
import paper_2603_21444_b200 as spg
from paper_2603_21444_b200 import dist as sd
rank, world = int(sys.argv[1]), int(sys.argv[2])
P, lam, out = int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
dist.init_process_group("gloo", rank=rank, world_size=world)
a = O.port_gen_erdos_renyi(3000, 0.004, 21)
b = O.port_gen_erdos_renyi(3000, 0.004, 22)
grid = spg.TridentGrid.create(P, lam)
dev = spg.Device(rank)
at, bt = sd.rank_tiles(a, b, grid, rank)
def ag(x):
    o = [None] * world
    dist.all_gather_object(o, x)
    return o
ex = sd.RankExchange(dev, at, bt, rank, world, ag)
dist.barrier()
c, tl = ex.trident_step(P, lam, grid.q)
ch = c.download()
c.free()
dist.barrier()  # every peer is done pulling this rank's tiles
tiles = [None] * world
dist.all_gather_object(tiles, (ch.nrows, ch.ncols, np.asarray(ch.rowptr), np.asarray(ch.colind), np.asarray(ch.values)))
ex.close()
if rank == 0:
    with open(out, "wb") as f:
        pickle.dump(tiles, f)
dist.destroy_process_group()
'''


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("pull", ["1", "0"], ids=["copy_engines", "sm_pulls"])
@pytest.mark.parametrize("P,lam", [(2, 2), (4, 4), (4, 1)])
def test_trident_rank_ipc_matches_reference(tmp_path, P, lam, pull):
    if spg.Device.count() < P:
        pytest.skip(f"needs {P} GPUs (one process per GPU)")
    import pickle
    out = str(tmp_path / "tiles.pkl")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), SPG_PULL_CE=pull)
    code = WORKER.format(root=ROOT)
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r), str(P), str(P), str(lam), out], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(P)]
    for p in procs:
        o, e = p.communicate(timeout=600)
        assert p.returncode == 0, e[-3000:]
    with open(out, "rb") as f:
        tiles = pickle.load(f)
    ct = [spg.CsrMatrix(int(nr), int(nc), rp, ci, va) for nr, nc, rp, ci, va in tiles]
    a = O.port_gen_erdos_renyi(3000, 0.004, 21)
    b = O.port_gen_erdos_renyi(3000, 0.004, 22)
    c = spg.reassemble(ct, spg.make_tile_map(3000, 3000, "trident", P, lam))
    ref = O.port_spgemm(a, b)
    assert np.array_equal(np.asarray(c.rowptr), np.asarray(ref.rowptr))
    assert np.array_equal(np.asarray(c.colind), np.asarray(ref.colind))
    assert np.array_equal(np.asarray(c.values), np.asarray(ref.values))
