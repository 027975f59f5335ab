"""CPU: the measured timeline's JSONL (DriverResult.to_jsonl, Python mirror of
EventTimeline::to_jsonl) has the reference's schema — the same keys in the
same order and the same value types as the reference's own
dr.timeline.to_jsonl() (engine.cpp:25-41, run through oracle/_ref)."""
import json

import numpy as np
import pytest

import oracle as O
import paper_2603_21444_b200 as spg


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref")
@pytest.mark.parametrize("algo,P,lam", [("trident", 8, 2), ("summa", 4, 2)])
def test_jsonl_schema_matches_reference(algo, P, lam):
    a, b = O.port_gen_erdos_renyi(120, 0.05, 1), O.port_gen_erdos_renyi(120, 0.05, 2)
    ref_lines = [json.loads(x, object_pairs_hook=list) for x in O.ref_timeline_jsonl(algo, a, b, P, lam).splitlines()]
    assert ref_lines
    ref_keys = [k for k, _ in ref_lines[0]]
    ev = []
    for pairs in ref_lines:  # the reference's events, re-serialised by our writer
        d = dict(pairs)
        ev.append({"type": d["type"], "src": d["actors"][0], "dst": d["actors"][1], "round": d["round"],
                   "operand": d["operand"], "link": d["link"], "t_start": d["t_start"], "t_end": d["t_end"],
                   "nnz": d["nnz"], "bytes": d["bytes"]})
    dr = spg.DriverResult(c=None, ledger=np.zeros(0), timeline=np.zeros(0), makespan=0.0, rounds=1, events=ev)
    ours = [json.loads(x, object_pairs_hook=list) for x in dr.to_jsonl().splitlines()]
    assert len(ours) == len(ref_lines)
    for o, r in zip(ours, ref_lines):
        assert [k for k, _ in o] == ref_keys
        assert dict(o) == dict(r)
