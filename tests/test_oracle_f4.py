"""Pins of the NEXT-f4 fill-all injection mode (inject_mode 2, DESIGN R53;
SPEC S:L145 "pending flits from the node's send queue are injected into input
slots left free, oldest-queued first").  Nothing here compares the
oracle with itself:
  * SPEC's worked example ("empty network, node with 2 queued flits,
    4 free inputs -> both injected same cycle") on a remote-hit reply;
  * a hand-derived zero-load timeline in which the two flits of that reply
    meet again at the requester and one is deflected there;
  * the brute-force arbitration (serial dictatorship over all injective
    assignments) on routers holding several flits injected in one cycle,
    ranked by the R53 tie-break;
  * per-cycle invariants and drain conservation on random configurations."""
import random

import pytest

import oracle
from oracle import Oracle, DBG_INVARIANTS
from paper_1508_03235_b200 import workloads as W
from test_oracle import brute_force, exists, X_, check_case

N = 16


def man(a, b, w=4):
    return abs(a % w - b % w) + abs(a // w - b // w)


def remote_hit(inject_mode, S=0, holder=5, home=10, nfl_ra=2):
    """4x4 LSPD, zero load: the holder fetches T (homed at `home`) first, then
    S reads it (remote hit, Fig. 4).  Returns the per-cycle injected
    counts between the two accesses' start and the end, the stats and the
    access-latency histogram."""
    T = 16 * 7 + home
    cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32, nfl_ra=nfl_ra,
                 inject_mode=inject_mode)
    o = Oracle(cfg, script=[(0, holder, T), (400, S, T)], debug=DBG_INVARIANTS)
    o.run(400)
    per_cycle = []
    last = o.stats()[0]["injected"]
    for _ in range(100):
        o.run(1)
        cur = o.stats()[0]["injected"]
        per_cycle.append(cur - last)
        last = cur
    st, _, _, ha = o.stats()
    return per_cycle, st, {b: c for b, c in enumerate(ha) if c}


def test_spec_example_two_queued_flits_injected_in_one_cycle():
    """the 2-flit RA reply at the degree-4 holder (node 5 of 4x4) is
    injected in one cycle under fill-all, over two cycles under R7."""
    p2, st2, _ = remote_hit(2)
    p0, st0, _ = remote_hit(0)
    assert max(p0) == 1 and max(p2) == 2
    assert p2.count(2) == 1                      # exactly the reply's two flits together
    assert sum(p2) == sum(p0) == 1 + 1 + 1 + 2   # DA + DR + RQ + RA (Table I, nfl_ra = 2)
    # the reply goes out in the cycle after the RQ is served (R22, R27) in
    # both modes: the cycle mode 0 injects the first RA flit
    k = p2.index(2)
    assert p0[k] == 1 and p0[k + 1] == 1


def test_fill_all_remote_hit_timeline_with_deflection_at_the_requester():
    """Hand-derived (zero load, 4x4, S = 0, holder 5 = (1,1), home 10 = (2,2)):
    under R7 the RA flits leave node 5 one cycle apart, both through the x-port
    W, and arrive at S on consecutive cycles: latency 2 d1 + 2 d2 + 2 + nfl_ra
    = 16.  Under fill-all both leave in the same cycle, fid 0 through the
    x-port W (node 4), fid 1 through the y-port N (node 1, PMDR's second
    productive port); both reach S in the same cycle, fid 0 ranks first (equal
    age, inj and src: R53 tie-break) and ejects, fid 1 is deflected to S's
    first free existing port in N,S,E,W (S = node 4, age 1), comes back the
    cycle after and ejects: one deflection, latency 16 + 1."""
    d1, d2, nfl = man(0, 10), man(0, 5), 2
    base = 2 * d1 + 2 * d2 + 2 + nfl
    mem = 100
    setup = 2 * man(5, 10) + 1 + mem            # the holder's own fetch (NDR path)
    _, st0, h0 = remote_hit(0)
    _, st2, h2 = remote_hit(2)
    assert h0 == {setup: 1, base: 1} and st0["deflections"] == 0
    assert h2 == {setup: 1, base + 1: 1} and st2["deflections"] == 1


def rank_key7(f, prio):
    dst, src, age, inj, fid, kind, pay = f
    head = (-age, inj, src) if prio == W.PRIO_DEFLECT else (inj, src)
    return head + (fid, kind, dst, pay)


def brute7(w, h, n, prio, flits, route):
    """brute_force of test_oracle with the R53 tie-break in the ranking."""
    import test_oracle as T
    saved = T.rank_key
    T.rank_key = lambda f, p: rank_key7(f, p)
    try:
        return brute_force(w, h, n, prio, flits, route)
    finally:
        T.rank_key = saved


@pytest.mark.parametrize("route", [W.ROUTE_PMDR, W.ROUTE_XY])
@pytest.mark.parametrize("prio", [W.PRIO_DEFLECT, W.PRIO_OLDEST])
def test_arbitration_with_several_flits_injected_in_one_cycle(prio, route):
    """Routers of a 3x3 mesh (corner, edge, centre) holding link flits plus
    1..degree flits injected by the node this cycle (src = node, inj = t, age
    0), and routers a cycle or more later holding flits that one node injected
    together (equal age, inj, src): the oracle's greedy equals the brute force
    ranked by (age, inj, src, fid, kind, dst, payload) (R53)."""
    rng = random.Random(53 + prio + 2 * route)
    w = h = 3
    t = 9
    for node in (0, 1, 4):
        deg = sum(exists(w, h, node, p) for p in range(4))
        for _ in range(3000):
            nl = rng.randrange(deg)
            ninj = rng.randrange(1, deg - nl + 1)
            flits = []
            srcs = rng.sample([s for s in range(9) if s != node], 8)
            for _k in range(nl):
                flits.append((rng.randrange(9), srcs.pop(), rng.randrange(3), rng.randrange(t - 3, t),
                              rng.randrange(8), rng.randrange(8), rng.randrange(4)))
            for j in range(ninj):
                flits.append((rng.choice([d for d in range(9) if d != node]), node, 0, t,
                              rng.randrange(8), rng.randrange(8), rng.randrange(4)))
            got = oracle.arbitrate(w, h, node, prio, flits, route)
            assert got == brute7(w, h, node, prio, flits, route), (node, flits)
            # later: a group of flits from one source with equal age and inj
            src = rng.choice([s for s in range(9) if s != node])
            k = rng.randrange(2, deg + 1)
            grp = [(rng.randrange(9), src, 1, t - 2, rng.randrange(8), rng.randrange(8), rng.randrange(4))
                   for _ in range(k)]
            got = oracle.arbitrate(w, h, node, prio, grp, route)
            assert got == brute7(w, h, node, prio, grp, route), (node, grp)
            ports = got[0]
            assert len(set(ports)) == len(ports) and all(p == X_ or exists(w, h, node, p) for p in ports)


def test_mode0_arbitration_unchanged_by_the_tie_break():
    """With at most one injected flit per node and cycle, (age, inj, src) is
    unique and the extra keys never decide: 4-field and 7-field calls agree."""
    rng = random.Random(7)
    for _ in range(2000):
        node = rng.choice([0, 1, 4])
        deg = sum(exists(3, 3, node, p) for p in range(4))
        srcs = rng.sample(range(9), deg)
        fl = [(rng.randrange(9), srcs[i], rng.randrange(3), rng.randrange(4)) for i in range(deg)]
        ext = [f + (rng.randrange(8), rng.randrange(8), rng.randrange(9)) for f in fl]
        assert oracle.arbitrate(3, 3, node, W.PRIO_DEFLECT, fl) == oracle.arbitrate(3, 3, node, W.PRIO_DEFLECT, ext)


CASES = [
    ("ur6x5", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_UR, lam=0.3, inject_mode=2, sendq_cap=16)),
    ("ur8x8_oldest", W.make(mesh_w=8, mesh_h=8, mode=W.MODE_UR, lam=0.2, inject_mode=2, prio=W.PRIO_OLDEST)),
    ("lspd6x5", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.2,
                       sendq_cap=32, seed=7, mem_lat=30, inject_mode=2)),
    ("lspd5x4_xy_l1", W.make(mesh_w=5, mesh_h=4, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.3,
                             sendq_cap=32, seed=3, mem_lat=20, inject_mode=2, route=W.ROUTE_XY,
                             l1_sets=2, l1_ways=2)),
    ("lspd6x6_mig", W.make(mesh_w=6, mesh_h=6, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.2,
                           sendq_cap=64, seed=11, mem_lat=20, inject_mode=2, mig_hist=6, nfl_b2=16)),
]


@pytest.mark.parametrize("name,cfg", CASES)
def test_fill_all_invariants_and_drain(name, cfg):
    """Conservation, port exclusivity, flits <= degree, top-priority progress
    every cycle (the oracle's debug checks), and delivery of everything."""
    o = Oracle(cfg, debug=DBG_INVARIANTS)
    o.run(2500)
    used, drained = o.drain(200000)
    assert drained
    st = o.stats()[0]
    assert st["injected"] == st["ejected"]
    if cfg["mode"] == W.MODE_LSPD:
        assert st["accesses"] == st["completed"]
        assert st["requests_made"] == st["requests_received"]
