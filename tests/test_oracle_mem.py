"""Pins of memory on the mesh (NEXT-f3 memory at the directory node, NEXT-f4
memory-controller nodes; DESIGN R54-R56; Table I B2;
SPEC S:L333-334) and of the hub send-FIFO capacity.  Nothing here
compares the oracle with itself:
  * hand-derived zero-load latencies (tests/golden/mem_timelines.txt) of the
    controller path, a local controller, a trap, the fill from the home's
    memory and from the central directory node's memory -- the controller
    positions are pinned through their distances;
  * a writeback pinned by counting: one eviction sends one B2 block of nfl_b2
    flits that the memory node absorbs;
  * invariants every cycle and message conservation on random configurations;
  * the hub FIFO: a central directory that overflows an 8-packet FIFO under
    load runs clean with a larger hub FIFO, whose occupancy exceeds 8."""
import collections
import os

import pytest

from oracle import Oracle, DBG_INVARIANTS, OracleError
from paper_1508_03235_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def man(a, b, w=4):
    return abs(a % w - b % w) + abs(a // w - b // w)


def rows(name):
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            yield [c.strip() for c in line.split("|")]


def test_mem_timelines():
    n = 0
    for case, mm, S, home, holder, D, lat, setup in rows("mem_timelines.txt"):
        S, home, mm = int(S), int(home), int(mm)
        T = 112 + home
        kw = dict(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32, mem_mode=mm, mem_ctrls=4)
        if D != "-":
            kw.update(dir_mode=W.DIR_CENTRAL, dir_node=int(D))
        script = [(0, S, T)] if holder == "-" else [(0, int(holder), T), (40, S, T)]
        o = Oracle(W.make(**kw), script=script, debug=DBG_INVARIANTS)
        o.run(600)
        st, _, _, ha = o.stats()
        got = collections.Counter({b: c for b, c in enumerate(ha) if c})
        want = collections.Counter([int(lat)] + ([] if setup == "-" else [int(setup)]))
        assert got == want, (case, dict(got), dict(want))
        assert st["deflections"] == 0, case
        remote_fills = st["mem_fills_received"]
        assert st["mem_fills_sent"] == remote_fills
        if case == "ctrl_trap":
            assert st["traps_received"] == 1 and remote_fills == 2
        n += 1
    assert n == 6


def test_closed_forms_match_the_fixture():
    """The fixture's numbers restated from the closed forms of its header."""
    ctrl = lambda T: [1, 3, 13, 15][T % 4]
    mem, b2 = 100, 16
    assert 2 * man(0, 5) + 2 * man(0, ctrl(117)) + 2 + b2 + mem == 128
    assert 2 * man(13, 6) + 1 + mem == 107 and ctrl(118) == 13
    assert 2 * man(0, 3) + 2 * man(0, 12) + 2 * man(0, ctrl(115)) + 4 + b2 + mem == 144
    assert 2 * man(12, 3) + 2 * man(12, ctrl(115)) + 2 + b2 + mem == 136
    assert 2 * man(0, 10) + b2 + mem == 124
    assert 2 * man(0, 5) + b2 + mem == 120


def test_writeback_of_an_evicted_block():
    """Node 0 fills three blocks of one set of its 2-way slice: the third
    install evicts the LRU block, which goes back to its controller as one B2
    block (Table I "L2 Blk Replacement" B2 = 16 flits) besides the EV."""
    Ts = [112 + 5, 112 + 5 + 64, 112 + 5 + 128]        # T mod 4 sets -> one set, homes differ
    cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32, mem_mode=W.MEM_CTRLS,
                 mem_ctrls=4, tags_per_node=128)
    o = Oracle(cfg, script=[(0, 0, Ts[0]), (300, 0, Ts[1]), (600, 0, Ts[2])], debug=DBG_INVARIANTS)
    o.run(1200)
    used, drained = o.drain(10000)
    assert drained
    st = o.stats()[0]
    assert st["evictions"] == 1 and st["evs_sent"] == 1
    assert st["mem_wbs_sent"] == 1 and st["mem_wb_flits"] == 16
    assert st["mem_requests"] == 3 and st["installs"] == 3


CASES = [
    ("ctrl8x8", W.lspd(8, 8, lam=0.1, mem_mode=W.MEM_CTRLS, mem_ctrls=4, sendq_cap=64, hub_sendq_cap=256,
                       l2_sets=4, seed=3, mem_lat=30)),
    ("ctrl6x5_l1_xy", W.lspd(6, 5, lam=0.2, mem_mode=W.MEM_CTRLS, mem_ctrls=3, sendq_cap=64, hub_sendq_cap=256,
                             l2_sets=2, seed=5, mem_lat=20, l1_sets=2, l1_ways=2, route=W.ROUTE_XY, nfl_b2=5)),
    ("home7x6", W.lspd(7, 6, lam=0.2, mem_mode=W.MEM_HOME, sendq_cap=64, l2_sets=2, seed=9, mem_lat=25,
                       nfl_b2=8)),
    ("central6x6", W.lspd(6, 6, lam=0.05, mem_mode=W.MEM_HOME, dir_mode=W.DIR_CENTRAL, dir_node=14,
                          sendq_cap=16, hub_sendq_cap=1024, l2_sets=2, seed=2, mem_lat=15, nfl_b2=4)),
    ("ctrl5x5_fillall", W.lspd(5, 5, lam=0.2, mem_mode=W.MEM_CTRLS, mem_ctrls=2, sendq_cap=64, hub_sendq_cap=512,
                               l2_sets=2, seed=13, mem_lat=10, inject_mode=2, nfl_b2=6)),
]


@pytest.mark.parametrize("name,cfg", CASES)
def test_memory_nodes_invariants_and_conservation(name, cfg):
    """Every cycle: conservation, exclusivity, degree, top-priority progress,
    single copy and directory checks (debug mode); after a drain: every memory
    request got its fill, every writeback block arrived in full, every access
    completed."""
    o = Oracle(cfg, debug=DBG_INVARIANTS)
    o.run(2500)
    used, drained = o.drain(200000)
    assert drained
    st = o.stats()[0]
    assert st["accesses"] == st["completed"]
    assert st["mem_fills_sent"] == st["mem_fills_received"] > 0
    assert st["mem_wb_flits"] == cfg["nfl_b2"] * st["mem_wbs_sent"]
    assert st["mem_wbs_sent"] > 0
    assert st["requests_made"] == st["requests_received"]
    assert st["injected"] == st["ejected"]


def test_hub_fifo_capacity():
    """NEXT-f3: under load the central directory node's 8-packet
    send FIFO overflows (an error in LSPD mode, R21); with a 256-packet hub
    FIFO the same run is clean and the directory node's queue holds more than
    8 packets at some cycle."""
    base = dict(lam=0.2, dir_mode=W.DIR_CENTRAL, dir_node=27, sendq_cap=8, l2_sets=4, seed=4, mem_lat=20)
    o = Oracle(W.lspd(8, 8, **base))
    with pytest.raises(OracleError):
        o.run(3000)
    o = Oracle(W.lspd(8, 8, hub_sendq_cap=256, **base), debug=DBG_INVARIANTS)
    peak = 0
    for _ in range(60):
        o.run(50)
        peak = max(peak, len(o.fifo(27)[1]))
    assert peak > 8
    used, drained = o.drain(100000)
    assert drained


@pytest.mark.parametrize("bad", [
    dict(mem_mode=3), dict(mem_mode=W.MEM_CTRLS, mem_ctrls=0), dict(mem_mode=W.MEM_CTRLS, mem_ctrls=65),
    dict(mem_mode=W.MEM_CTRLS, mem_ctrls=9), dict(mem_mode=W.MEM_HOME, mig_hist=4),
    dict(hub_sendq_cap=24), dict(hub_sendq_cap=4), dict(hub_sendq_cap=2048),
])
def test_memory_config_limits(bad):
    cfg = W.lspd(4, 4, sendq_cap=8, **bad)
    with pytest.raises(OracleError):
        Oracle(cfg)
