"""The measured exchange record of the distributed drivers against the
reference engine (engine.cpp:228-302, algorithms.cpp:24-174, run through
oracle/_ref = the reference compiled from /root/reference).

* The ledger is built from the tiles each rank actually consumed (pulled or
  read in place), booked along the reference's routes. It must equal the
  reference's CommLedger, and a deliberately doubled pull
  (SPG_DEBUG_DOUBLE_PULL=1: the first remote A tile copied twice) must break
  that equality.
* The events (engine.hpp TimelineEvent) must equal the reference's
  dr.timeline.to_jsonl() event for event, as a multiset over (type, actors,
  round, operand, link, nnz, bytes); only the times differ (measured CUDA
  event seconds vs the modeled alpha-beta clock).
* node_start_delay (engine.cpp:217-221) delays a virtual node's pulls on the
  device.
When the box has >= 2 GPUs the ranks spread over them (rank r -> device
r % ndev), so the peer-copy branches run."""
import collections
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg

pytestmark = pytest.mark.gpu

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref (the reference library)")
GRIDS = [(4, 1), (4, 4), (8, 2), (16, 4), (9, 1), (2, 2)]


def key(e):
    return (e["type"], tuple(e["actors"]) if "actors" in e else (e["src"], e["dst"]), e["round"], e["operand"],
            e["link"], e["nnz"], e["bytes"])


def ours_multiset(r):
    return collections.Counter(key(json.loads(x)) for x in r.to_jsonl().splitlines())


def ref_multiset(algo, a, b, P, lam, delays=None):
    return collections.Counter(key(json.loads(x)) for x in O.ref_timeline_jsonl(algo, a, b, P, lam, delays).splitlines())


def mats(seed=3, n=600):
    return O.port_gen_erdos_renyi(n, 0.01, seed), O.port_gen_erdos_renyi(n, 0.01, seed + 1)


@needs_ref
@pytest.mark.parametrize("P,lam", GRIDS)
def test_trident_ledger_and_events_equal_reference(P, lam):
    a, b = mats()
    r = spg.trident_spgemm(a, b, spg.TridentGrid.create(P, lam))
    ref = O.ref_run_algo("trident", a, b, P, lam)
    assert spg.pattern_equal(r.c, ref["c"]) and spg.allclose(r.c, ref["c"], 1e-12)
    assert np.array_equal(r.ledger, ref["ledger"])
    assert ours_multiset(r) == ref_multiset("trident", a, b, P, lam)
    # every event has measured, ordered times
    assert all(e["t_end"] >= e["t_start"] >= 0.0 for e in r.events)


@needs_ref
@pytest.mark.parametrize("P", [1, 4, 9])
def test_summa_ledger_and_events_equal_reference(P):
    a, b = mats(5)
    r = spg.summa_spgemm(a, b, P, 2)
    ref = O.ref_run_algo("summa", a, b, P, 2)
    assert spg.allclose(r.c, ref["c"], 1e-12)
    assert np.array_equal(r.ledger, ref["ledger"])
    assert ours_multiset(r) == ref_multiset("summa", a, b, P, 2)


@needs_ref
@pytest.mark.parametrize("algo", ["trident", "summa"])
def test_double_pull_breaks_the_ledger(monkeypatch, algo):
    """A wrong exchange (one tile pulled twice) must show in the ledger: the
    ledger counts what was pulled, it does not restate the schedule. (The
    fault hook is read once per process, so the run happens in a child.)"""
    import subprocess
    import sys
    code = f"""
import sys; sys.path.insert(0, {os.getcwd()!r})
import numpy as np, oracle as O, paper_2603_21444_b200 as spg
a, b = O.port_gen_erdos_renyi(600, 0.01, 3), O.port_gen_erdos_renyi(600, 0.01, 4)
r = spg.trident_spgemm(a, b, spg.TridentGrid.create(8, 2)) if {algo!r} == "trident" else spg.summa_spgemm(a, b, 4, 2)
ref = O.ref_run_algo({algo!r}, a, b, 8 if {algo!r} == "trident" else 4, 2)
assert spg.pattern_equal(r.c, ref["c"])  # C is unaffected by a redundant copy
print("LEDGER_EQUAL" if np.array_equal(r.ledger, ref["ledger"]) else "LEDGER_DIFFERS")
print("XFER", r.xfer[:, 2].sum())
"""
    env = dict(os.environ, SPG_DEBUG_DOUBLE_PULL="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "LEDGER_DIFFERS" in out.stdout
    env.pop("SPG_DEBUG_DOUBLE_PULL")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "LEDGER_EQUAL" in out.stdout


@needs_ref
def test_node_start_delay_on_the_device():
    """Node 1 of the (8, 2) grid starts 50 ms late: its ranks' pull events
    start >= 50 ms after their start; node 0's start at once. Ledger and event
    multiset stay the reference's (the reference's delay only shifts times)."""
    a, b = mats(7)
    grid = spg.TridentGrid.create(8, 2)
    delays = [0.0, 0.05, 0.0, 0.0]
    r = spg.trident_spgemm(a, b, grid, node_start_delay=delays)
    ref = O.ref_run_algo("trident", a, b, 8, 2)
    assert np.array_equal(r.ledger, ref["ledger"])
    assert ours_multiset(r) == ref_multiset("trident", a, b, 8, 2, delays)
    pulls = [e for e in r.events if e["type"] == "transfer-complete"]
    first = {}
    for e in pulls:
        first[e["dst"]] = min(first.get(e["dst"], 1e9), e["t_start"])
    # every rank of node 1 starts pulling after its 50 ms delay; node 0's ranks
    # start at once (later pulls of theirs may queue behind a delayed owner's
    # copies on a multi-GPU box, so only the first pull is compared)
    assert all(first[r] >= 0.05 for r in (2, 3))
    assert all(first[r] < 0.05 for r in (0, 1))
    with pytest.raises(spg.SpgError):
        spg.trident_spgemm(a, b, grid, node_start_delay=[-1.0])


def test_xfer_stats_count_the_pulls():
    """xfer[rank] = [device bytes pulled, pull span ms, tiles pulled, tiles
    read in place]: every remote tile a rank consumed is either pulled or
    read in place, and pulled tiles move rowptr (8 B/row) + 12 B/entry."""
    a, b = mats(9)
    P, lam = 8, 2
    r = spg.trident_spgemm(a, b, spg.TridentGrid.create(P, lam))
    grid = spg.TridentGrid.create(P, lam)
    for rank in range(P):
        i, j, k = grid.coords_of(rank)
        remote = 0
        for rnd in range(grid.q):
            s = (rnd + i + j) % grid.q
            remote += grid.rank_of(i, s, k) != rank
            remote += sum(grid.rank_of(s, j, k2) != rank for k2 in range(lam))
        assert r.xfer[rank, 2] + r.xfer[rank, 3] == remote
        if spg.Device.count() == 1:  # every tile of every rank lives on device 0
            assert r.xfer[rank, 2] <= remote


@pytest.mark.skipif(spg.Device.count() < 2, reason="needs >= 2 GPUs (tiles on distinct devices, peer copies)")
@needs_ref
@pytest.mark.parametrize("P,lam", [(2, 2), (4, 4), (8, 2), (4, 1)])
def test_trident_tiles_on_distinct_devices(P, lam):
    """Ranks on different GPUs: the A pulls and B slice pulls take the
    cudaMemcpyPeerAsync branches; C and ledger still equal the reference's,
    and every remote tile on another device is pulled (none read in place)."""
    a, b = mats(11, 2000)
    r = spg.trident_spgemm(a, b, spg.TridentGrid.create(P, lam))
    ref = O.ref_run_algo("trident", a, b, P, lam)
    assert spg.pattern_equal(r.c, ref["c"]) and spg.allclose(r.c, ref["c"], 1e-12)
    assert np.array_equal(r.ledger, ref["ledger"])
    assert ours_multiset(r) == ref_multiset("trident", a, b, P, lam)
    assert r.xfer[:, 2].sum() > 0 and r.xfer[:, 0].sum() > 0


@pytest.mark.skipif(spg.Device.count() < 2, reason="needs >= 2 GPUs (tiles on distinct devices, peer pulls)")
@needs_ref
@pytest.mark.parametrize("pull", ["1", "0"], ids=["copy_engines", "sm_pulls"])
def test_peer_pull_modes_bit_exact(pull):
    """vconcat's two ways of pulling a peer's B slice — copy engines
    (cudaMemcpyPeerAsync) and the SM pull kernel (k_pull_slice, loads over
    NVLink) — give the same C as the reference and the same ledger, with
    slices whose destination offsets are not 16-byte aligned (odd nnz per
    slice). The mode is read once per process, so the run is in a child."""
    import subprocess
    import sys
    code = f"""
import sys; sys.path.insert(0, {os.getcwd()!r})
import numpy as np, oracle as O, paper_2603_21444_b200 as spg
for P, lam, n in ((4, 4, 1999), (8, 2, 2001), (2, 2, 777)):
    a, b = O.port_gen_erdos_renyi(n, 0.006, 31), O.port_gen_erdos_renyi(n, 0.006, 32)
    r = spg.trident_spgemm(a, b, spg.TridentGrid.create(P, lam))
    ref = O.ref_run_algo("trident", a, b, P, lam)
    assert spg.pattern_equal(r.c, ref["c"]) and spg.allclose(r.c, ref["c"], 1e-12), (P, lam)
    # a rank's rounds are one k-ordered multiply: bit-identical to the serial
    # product (the reference's trident adds partial Cs at q = 2)
    assert np.array_equal(np.asarray(r.c.values), np.asarray(O.port_spgemm(a, b).values)), (P, lam)
    assert np.array_equal(r.ledger, ref["ledger"]), (P, lam)
    assert r.xfer[:, 2].sum() > 0
print("PULL_OK")
"""
    env = dict(os.environ, SPG_PULL_CE=pull)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "PULL_OK" in out.stdout
