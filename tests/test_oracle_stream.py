"""Pins of the streamed trace replay (NEXT-f3, DESIGN R57; SURVEY f3 "streamed
with double-buffered chunked H2D copies"; the paper feeds the trace per cycle,
P:L233, L276-277).  Nothing here compares the oracle with itself run the same
way: a script pushed in pieces is checked against the definition it must
reduce to -- the whole script given at create -- and against hand-derived
single-event timelines.
  * pieces pushed before their events are due == the whole script at create,
    for random UR and LSPD scripts, interleaved with runs and a drain;
  * an event pushed after its cycle is consumed at the node's next generation
    opportunity (hand-derived: generated, delivered, latency = distance);
  * per-node order is enforced; ranges are checked;
  * a trace file read in chunks (workloads.trace_chunks) == the file loaded
    whole (workloads.load_trace)."""
import os
import random

import pytest

from oracle import Oracle, OracleError, DBG_INVARIANTS
from paper_1508_03235_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def pieces_by_cycle(script, bounds):
    """Split a script at cycle bounds: piece k holds the events with cycle in
    [bounds[k-1], bounds[k])."""
    out = [[] for _ in range(len(bounds) + 1)]
    for e in script:
        k = sum(1 for b in bounds if e[0] >= b)
        out[k].append(e)
    return out


@pytest.mark.parametrize("mode", [W.MODE_UR, W.MODE_LSPD])
def test_pushed_in_pieces_equals_script_at_create(mode):
    if mode == W.MODE_UR:
        cfg = W.make(mesh_w=6, mesh_h=5, mode=W.MODE_UR, thr_inj=0, sendq_cap=16)
    else:
        cfg = W.lspd(6, 5, thr_inj=0, sendq_cap=64, l2_sets=2, mem_lat=20)
    script = W.random_script(cfg, 900, 1200, seed=21)
    whole = Oracle(cfg, script=script, debug=DBG_INVARIANTS)
    parts = pieces_by_cycle(script, [200, 450, 451, 800])
    streamed = Oracle(cfg, script=parts[0], debug=DBG_INVARIANTS)
    # piece k is pushed before the run that reaches its first cycle
    t = 0
    for k, stop in enumerate([200, 450, 451, 800, 1500]):
        if k + 1 < len(parts):
            streamed.push_script(parts[k + 1])
        streamed.run(stop - t)
        whole.run(stop - t)
        t = stop
        assert streamed.state_hash() == whole.state_hash(), stop
    assert whole.drain(100000) == streamed.drain(100000)
    assert streamed.stats() == whole.stats() and streamed.state_hash() == whole.state_hash()
    assert streamed.stats()[0]["generated" if mode == W.MODE_UR else "accesses"] > 0


def test_late_event_consumed_at_next_opportunity():
    """UR 4x4, nothing scripted at create: an event (cycle 3, node 0 -> node 5)
    pushed at cycle 10 is generated at cycle 10 (the node's next generation
    opportunity, DESIGN 3.3: the first unconsumed event with cycle <= t) and
    delivered after Manhattan distance 2 (R8, R11): one probe, latency 2."""
    cfg = W.make(mode=W.MODE_UR, thr_inj=0)
    o = Oracle(cfg)
    o.run(10)
    o.push_script([(3, 0, 5)])
    assert o.stats()[0]["generated"] == 0
    o.run(1)
    assert o.stats()[0]["generated"] == 1
    o.run(10)
    st, hl, _, _ = o.stats()
    assert st["probes_delivered"] == 1 and hl[2] == 1


def test_order_and_range_checks():
    cfg = W.make(mode=W.MODE_UR, thr_inj=0)
    o = Oracle(cfg, script=[(50, 1, 2)])
    with pytest.raises(OracleError):
        o.push_script([(40, 1, 3)])          # precedes node 1's event of cycle 50
    o.push_script([(50, 1, 3), (7, 2, 1)])   # same cycle, and another node: fine
    with pytest.raises(OracleError):
        o.push_script([(60, 16, 0)])         # node out of range
    with pytest.raises(OracleError):
        o.push_script([(60, 4, 4)])          # probe to itself
    o.run(100)
    assert o.stats()[0]["generated"] == 3


def test_trace_file_in_chunks_equals_whole_trace():
    cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32)
    path = os.path.join(GOLDEN, "trace_4x4.txt")
    whole = Oracle(cfg, script=W.load_trace(path, cfg))
    chunks = list(W.trace_chunks(path, cfg, 3))
    assert sum(len(c) for c in chunks) == len(W.load_trace(path, cfg)) and len(chunks) > 1
    streamed = Oracle(cfg)
    for c in chunks:          # every record has cycle 0 (due at once): pushed before the first run
        streamed.push_script(c)
    whole.run(2000)
    streamed.run(2000)
    assert streamed.stats() == whole.stats() and streamed.state_hash() == whole.state_hash()


def test_pieces_interleaved_with_runs_random():
    """Random LSPD script, random piece sizes pushed at random times, each
    piece before its events are due: equal to the script at create."""
    rng = random.Random(5)
    cfg = W.lspd(5, 4, thr_inj=0, sendq_cap=64, l2_sets=2, mem_lat=15, l1_sets=2, l1_ways=2)
    script = W.random_script(cfg, 600, 3000, seed=8)
    bounds = sorted(rng.sample(range(50, 3000), 9))
    parts = pieces_by_cycle(script, bounds)
    whole = Oracle(cfg, script=script)
    streamed = Oracle(cfg, script=parts[0])
    t = 0
    for k, b in enumerate(bounds):
        streamed.push_script(parts[k + 1])
        stop = b - rng.randrange(0, 20)
        stop = max(stop, t)
        streamed.run(stop - t)
        whole.run(stop - t)
        t = stop
    streamed.push_script([])
    streamed.run(3500 - t)
    whole.run(3500 - t)
    assert streamed.stats() == whole.stats() and streamed.state_hash() == whole.state_hash()
