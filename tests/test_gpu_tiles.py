"""GPU: the device tile store — spg_partition and
spg_reassemble through the C ABI against the reference's partition /
reassemble (partition.cpp:161-261): tiles bit-identical to the reference's
(golden rectangles and tile nnz from the reference itself, and the host mirror
on random inputs), and reassemble(partition(m)) == m bit for bit, tiles spread
over every GPU of the box."""
import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg
from golden_io import csr, grids, z

pytestmark = pytest.mark.gpu


def same(a, b):
    return (int(a.nrows) == int(b.nrows) and int(a.ncols) == int(b.ncols) and np.array_equal(a.rowptr, b.rowptr)
            and np.array_equal(np.asarray(a.colind, np.int64), np.asarray(b.colind, np.int64))
            and np.array_equal(a.values, b.values))


def all_devices():
    return [spg.default_device(d) for d in range(spg.Device.count())]


@pytest.mark.parametrize("P,lam", grids())
def test_device_partition_matches_reference(dev, P, lam):
    a = csr("er300_p3_A")
    da = dev.upload(a)
    tiles, tm = dev.partition(da, "trident", P, lam, devices=all_devices())
    host, _ = spg.partition(a, "trident", P, lam)
    assert [t.nnz for t in tiles] == z()[f"part_P{P}_L{lam}_nnz"].tolist()
    for t, h in zip(tiles, host):
        t.check()
        assert same(t.download(), h)
    back = dev.reassemble(tiles, tm)
    back.check()
    assert same(back.download(), a)


CASES = [((300, 300, 0.03, 1), "trident", 16, 4), ((300, 300, 0.03, 2), "trident", 8, 2),
         ((1000, 700, 0.01, 3), "trident", 4, 1), ((1000, 700, 0.01, 4), "grid2d", 9, 1),
         ((513, 129, 0.05, 5), "grid2d", 4, 1), ((777, 333, 0.02, 6), "rows1d", 5, 1),
         ((6, 9, 0.3, 7), "trident", 16, 4),   # zero-row slices and empty tiles
         ((40, 40, 0.0, 8), "trident", 4, 4),  # no entries at all
         ((0, 12, 0.0, 9), "rows1d", 3, 1)]    # no rows


@pytest.mark.parametrize("gen,scheme,P,lam", CASES)
def test_device_partition_roundtrip(dev, gen, scheme, P, lam):
    m, n, d, seed = gen
    a = O.port_gen_erdos_renyi_rect(m, n, d, seed) if d > 0 else spg.CsrMatrix.zeros(m, n)
    da = dev.upload(a)
    tiles, tm = dev.partition(da, scheme, P, lam, devices=all_devices())
    host, htm = spg.partition(a, scheme, P, lam)
    assert np.array_equal(tm.tiles, htm.tiles)
    for t, h in zip(tiles, host):
        assert same(t.download(), h)
    back = dev.reassemble(tiles, tm)
    assert same(back.download(), a)
    # reassembling host-built tiles uploaded to the devices gives the same matrix
    devs = all_devices()
    up = [devs[r % len(devs)].upload(h) for r, h in enumerate(host)]
    assert same(dev.reassemble(up, tm).download(), spg.reassemble(host, htm))


def test_device_reassemble_errors(dev):
    a = csr("er300_p3_A")
    tiles, tm = dev.partition(dev.upload(a), "trident", 4, 1)
    with pytest.raises(spg.SpgError) as e:
        dev.reassemble(tiles[:3], tm)
    assert e.value.kind == "IncompleteTileSet"
    with pytest.raises(spg.SpgError) as e:
        dev.reassemble([tiles[1], tiles[0], tiles[2], tiles[3]], spg.make_tile_map(301, 300, "trident", 4, 1))
    assert e.value.kind == "IncompleteTileSet"
    with pytest.raises(spg.SpgError) as e:
        dev.partition(dev.upload(a), "trident", 8, 1)
    assert e.value.kind == "GridError"


@pytest.mark.slow
def test_device_partition_config2_size(dev):
    """Config 2 (ER n=2^22, 16/row) at the P=8 (lambda=2) trident map: the
    device round trip is bit-exact, tile nnz are the reference's (SURVEY
    §8(e): A tiles of 8,387,223-8,395,762 nnz)."""
    a = spg.gen_erdos_renyi(1 << 22, 16.0 / (1 << 22), 1)
    da = dev.upload(a)
    tiles, tm = dev.partition(da, "trident", 8, 2, devices=all_devices())
    nnz = [t.nnz for t in tiles]
    assert sum(nnz) == a.nnz and min(nnz) == 8387223 and max(nnz) == 8395762
    back = dev.reassemble(tiles, tm).download()
    assert same(back, a)
