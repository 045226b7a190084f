"""Pins of the CPU oracle against what the paper and mathematics fix.

Every test here runs on CPU (no GPU marker).  None of them compares the
oracle with itself: each checks a closed form, a worked example from
PAPER.md (fixtures under tests/golden/, each with its citation), an
invariant, a special case, a textbook routine, or a brute-force search
written independently in this file.
"""
import collections
import itertools
import math
import os
import random

import pytest

import oracle
from oracle import Oracle, DBG_INVARIANTS, DBG_REVERSE
from paper_1508_03235_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
N_, S_, E_, W_, X_ = 0, 1, 2, 3, 4
PORT = {"N": 0, "S": 1, "E": 2, "W": 3, "X": 4}


def golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([c.strip() for c in line.split("|")])
    return rows


# ---------------------------------------------------------------- generator
def test_philox_known_answers():
    """Random123 KAT vectors (R25)."""
    for row in golden("philox_kat.txt"):
        k = [int(v, 16) for v in row[0].split()]
        c = [int(v, 16) for v in row[1].split()]
        r = [int(v, 16) for v in row[2].split()]
        assert oracle.philox(k, c) == tuple(r)


def test_bernoulli_rate_within_5_sigma():
    """Open-loop UR generation: generated ~ Binomial(N*T, lambda) (R25, R35)."""
    lam, T = 0.01, 20000
    cfg = W.make(mesh_w=16, mesh_h=16, mode=W.MODE_UR, lam=lam, sendq_cap=64)
    o = Oracle(cfg)
    o.run(T)
    n = 256 * T
    p = W.thr(lam) / 2 ** 32
    mean, sd = n * p, math.sqrt(n * p * (1 - p))
    assert abs(o.stats()[0]["generated"] - mean) < 5 * sd


# ---------------------------------------------------------------- routing
def manhattan(a, b, w):
    return abs(a % w - b % w) + abs(a // w - b // w)


@pytest.mark.parametrize("w,h", [(2, 2), (3, 3), (4, 4), (5, 3), (3, 6), (8, 8)])
def test_zero_load_latency_is_manhattan_all_pairs(w, h):
    """A lone flit never contends, so latency = |dx|+|dy| hops of 1 cycle
    (P:L116 PMDR, R11).  Every (src, dst) pair, one at a time."""
    n = w * h
    gap = w + h + 2
    pairs = [(s, d) for s in range(n) for d in range(n) if s != d]
    script = [(k * gap, s, d) for k, (s, d) in enumerate(pairs)]
    cfg = W.make(mesh_w=w, mesh_h=h, mode=W.MODE_UR, thr_inj=0, sendq_cap=4)
    o = Oracle(cfg, script=script, debug=DBG_INVARIANTS if n <= 16 else 0)
    o.run(len(pairs) * gap + 1)
    st, hl, hd, _ = o.stats()
    want = collections.Counter(manhattan(s, d, w) for s, d in pairs)
    got = {b: c for b, c in enumerate(hl) if c}
    assert got == dict(want)
    assert st["deflections"] == 0 and hd[0] == len(pairs)
    assert st["hops"] == sum(manhattan(s, d, w) for s, d in pairs)
    assert st["ejected"] == st["probes_delivered"] == len(pairs)


def test_zero_load_random_pairs_large_mesh():
    rng = random.Random(7)
    w, h = 32, 24
    n = w * h
    gap = w + h + 2
    pairs = []
    for _ in range(200):
        s = rng.randrange(n)
        d = rng.randrange(n - 1)
        pairs.append((s, d + (d >= s)))
    script = [(k * gap, s, d) for k, (s, d) in enumerate(pairs)]
    o = Oracle(W.make(mesh_w=w, mesh_h=h, mode=W.MODE_UR, thr_inj=0), script=script)
    o.run(len(pairs) * gap)
    hl = o.stats()[1]
    assert {b: c for b, c in enumerate(hl) if c} == dict(
        collections.Counter(manhattan(s, d, w) for s, d in pairs))


def test_example_path_4x4():
    """4x4: (0,0) -> (3,2) = node 11 goes E,E,E,S,S and ejects after 5 cycles."""
    o = Oracle(W.make(mode=W.MODE_UR, thr_inj=0), script=[(3, 0, 11)])
    o.run(3 + 5)   # injected at t=3, at node 11 at t=8 -> ejected in cycle 8
    assert o.stats()[0]["ejected"] == 0
    o.run(1)
    st, hl, _, _ = o.stats()
    assert st["ejected"] == 1 and hl[5] == 1 and st["hops"] == 5


# ---------------------------------------------------------------- arbitration
def rank_key(f, prio):
    dst, src, age, inj = f
    return (-age, inj, src) if prio == W.PRIO_DEFLECT else (inj, src)


def exists(w, h, n, p):
    x, y = n % w, n // w
    return {N_: y > 0, S_: y < h - 1, E_: x < w - 1, W_: x > 0}[p]


def productive(w, n, dst):
    x, y, dx, dy = n % w, n // w, dst % w, dst // w
    ports = []
    if dx != x:
        ports.append(E_ if dx > x else W_)
    if dy != y:
        ports.append(S_ if dy > y else N_)
    return ports


def brute_force(w, h, n, prio, flits, route=W.ROUTE_PMDR):
    """Lexicographically least vector of preference indices, in rank order,
    over all injective assignments (serial dictatorship): found by a
    depth-first search that tries options in preference order.  Preference
    lists: PMDR (R3, R5) = productive ports x then y, then the other existing
    ports in N,S,E,W; strict XY (NEXT-f4) = the XY port,
    then the other existing ports in N,E,S,W."""
    order = sorted(range(len(flits)), key=lambda i: rank_key(flits[i], prio))
    scan = (N_, S_, E_, W_) if route == W.ROUTE_PMDR else (N_, E_, S_, W_)
    prefs = []
    for i in order:
        dst = flits[i][0]
        if dst == n:
            lst = [X_] + [p for p in scan if exists(w, h, n, p)]
        else:
            lst = productive(w, n, dst)
            if route == W.ROUTE_XY:
                lst = lst[:1]
            lst += [p for p in scan if exists(w, h, n, p) and p not in lst]
        prefs.append(lst)
    assign = [None] * len(order)

    def dfs(k, used):
        if k == len(order):
            return True
        for p in prefs[k]:
            if p not in used:
                assign[k] = p
                if dfs(k + 1, used | {p}):
                    return True
        return False

    assert dfs(0, frozenset())
    ports = [None] * len(flits)
    ages = [None] * len(flits)
    for k, i in enumerate(order):
        p = assign[k]
        dst = flits[i][0]
        good = productive(w, n, dst) if route == W.ROUTE_PMDR else productive(w, n, dst)[:1]
        ok = (p == X_) if dst == n else (p in good)
        ports[i] = p
        ages[i] = flits[i][2] + (0 if ok else 1)
    return ports, ages


def check_case(w, h, n, prio, flits, route=W.ROUTE_PMDR):
    got = oracle.arbitrate(w, h, n, prio, flits, route)
    assert got == brute_force(w, h, n, prio, flits, route), (w, h, n, prio, flits, route)
    ports = got[0]
    assert len(set(ports)) == len(ports)                         # one flit per port
    assert all(p == X_ or exists(w, h, n, p) for p in ports)     # never off the mesh


def random_flit(rng, nn, src_pool):
    return (rng.randrange(nn), src_pool.pop(), rng.randrange(3), rng.randrange(2))


def test_arbitration_hand_cases():
    for case, node, fl, ports, ages in golden("arbitration_cases.txt"):
        flits = [tuple(int(v) for v in f.split(",")) for f in fl.split(";")]
        got = oracle.arbitrate(3, 3, int(node), W.PRIO_DEFLECT, flits)
        assert got[0] == [PORT[p] for p in ports.split()], case
        assert got[1] == [int(a) for a in ages.split()], case


def test_arbitration_hand_cases_strict_xy():
    """NEXT-f4 compatibility mode against hand-worked decisions."""
    for case, node, fl, ports, ages, route in golden("arbitration_cases_xy.txt"):
        flits = [tuple(int(v) for v in f.split(",")) for f in fl.split(";")]
        got = oracle.arbitrate(3, 3, int(node), W.PRIO_DEFLECT, flits, int(route))
        assert got[0] == [PORT[p] for p in ports.split()], case
        assert got[1] == [int(a) for a in ages.split()], case


@pytest.mark.parametrize("route", [W.ROUTE_PMDR, W.ROUTE_XY])
@pytest.mark.parametrize("prio", [W.PRIO_DEFLECT, W.PRIO_OLDEST])
def test_arbitration_exhaustive_corner(prio, route):
    """Every degree-2 case at the 3x3 corner (0,0): each input empty or a flit
    with dst in 9 nodes x age 0..2 x inj 0..1, both src orders, plus the
    injected flit (age 0, inj 2) whenever an input is free (R7)."""
    w = h = 3
    n = 0
    slot_opts = [None] + [(d, a, j) for d in range(9) for a in range(3) for j in range(2)]
    count = 0
    for s1, s2 in itertools.product(slot_opts, repeat=2):
        occ = [s for s in (s1, s2) if s is not None]
        inj_opts = [None] + (list(range(9)) if len(occ) < 2 else [])
        for srcs in itertools.permutations((4, 7), len(occ)):
            base = [(d, srcs[i], a, j) for i, (d, a, j) in enumerate(occ)]
            for inj in inj_opts:
                flits = base + ([(inj, n, 0, 2)] if inj is not None else [])
                if not flits:
                    continue
                check_case(w, h, n, prio, flits, route)
                count += 1
    assert count > 5000


@pytest.mark.parametrize("route", [W.ROUTE_PMDR, W.ROUTE_XY])
@pytest.mark.parametrize("prio", [W.PRIO_DEFLECT, W.PRIO_OLDEST])
@pytest.mark.parametrize("node", [1, 4])
def test_arbitration_random_edge_and_centre(prio, node, route):
    """Degree-3 (edge) and degree-4 (centre) routers of a 3x3 mesh: random
    cases against the brute force."""
    rng = random.Random(1000 + node + 10 * prio)
    w = h = 3
    deg = sum(exists(w, h, node, p) for p in range(4))
    for _ in range(6000):
        k = rng.randrange(deg + 1)
        pool = rng.sample(range(20), 5)
        flits = [random_flit(rng, 9, pool) for _ in range(k)]
        if k < deg and rng.random() < 0.7:
            flits.append((rng.randrange(9), node, 0, 2))
        if flits:
            check_case(w, h, node, prio, flits, route)


def test_arbitration_rejects_overfull_router():
    with pytest.raises(ValueError):
        oracle.arbitrate(3, 3, 0, 0, [(1, 1, 0, 0)] * 3)


# ---------------------------------------------------------------- whole-network invariants
INV_CFGS = [
    ("ur5x3", W.make(mesh_w=5, mesh_h=3, mode=W.MODE_UR, lam=0.3)),
    ("ur4x4_oldest", W.c1a(prio=W.PRIO_OLDEST, lam=0.4)),
    ("lspd4x4", W.c1b()),
    ("lspd4x4_oldest", W.c1b(prio=W.PRIO_OLDEST, seed=3)),
    ("lspd6x5", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.2,
                       sendq_cap=32, seed=2, mem_lat=30)),
    # NEXT-f4 strict-XY compatibility mode
    ("ur5x3_xy", W.make(mesh_w=5, mesh_h=3, mode=W.MODE_UR, lam=0.3, route=W.ROUTE_XY)),
    ("lspd6x5_xy", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.2,
                          sendq_cap=32, seed=2, mem_lat=30, route=W.ROUTE_XY)),
    # NEXT-f1 private L1 (Table III 32,2,32 scaled down) in front of the slices
    ("lspd6x5_l1", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.2,
                          sendq_cap=32, seed=5, mem_lat=30, l1_sets=2, l1_ways=2, l1_miss_lat=3)),
    # NEXT-f3 centralized directory at the centre node (2,2) of a 6x5 mesh
    ("lspd6x5_central", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.05,
                               sendq_cap=64, seed=4, mem_lat=30, dir_mode=W.DIR_CENTRAL, dir_node=14)),
]


@pytest.mark.parametrize("name,cfg", INV_CFGS)
def test_invariants_every_cycle(name, cfg):
    """Conservation, <=1 flit per link, flits <= degree, top-priority progress,
    single copy, holder NONE => pend 0, checked inside the
    oracle after every cycle; then drain and check the Table II equalities
     and directory agreement at quiescence."""
    o = Oracle(cfg, debug=DBG_INVARIANTS)
    o.run(3000)
    k, _ = o.links_occupied()
    st = o.stats()[0]
    assert st["injected"] == st["ejected"] + k
    used, drained = o.drain(200000)
    assert drained
    st = o.stats()[0]
    assert st["injected"] == st["ejected"]
    assert o.links_occupied()[0] == 0 and o.fifo_packets() == 0 and o.cores_busy() == 0
    assert st["requests_made"] == st["requests_received"]
    assert st["replies_sent"] == st["replies_received"]
    assert st["traps_sent"] == st["traps_received"]
    assert st["evs_sent"] == st["evs_received"]
    assert st["accesses"] == st["completed"]
    assert st["dir_searches"] == st["l2_misses"]
    assert st["mem_requests"] + st["replies_received"] == st["l2_misses"]
    assert o.directory_quiescent_ok()
    if cfg["mode"] == W.MODE_LSPD:
        assert st["accesses"] > 0 and st["replies_sent"] > 0 and st["evictions"] > 0


def test_table2_equality_pattern_in_paper():
    """The paper's own Table II has Req made == Req Rcved and Reply sent ==
    Reply Rcvd in every row: the pattern test_invariants_every_cycle asserts."""
    for row in golden("table2_counters.txt"):
        assert row[1] == row[2] and row[3] == row[4]


@pytest.mark.parametrize("prio", [W.PRIO_DEFLECT, W.PRIO_OLDEST])
def test_saturated_network_drains(prio):
    """Delivery / livelock freedom: a saturated UR mesh drains once
    generation stops."""
    o = Oracle(W.make(mesh_w=8, mesh_h=8, mode=W.MODE_UR, lam=0.5, prio=prio))
    o.run(2000)
    used, drained = o.drain(100000)
    st = o.stats()[0]
    assert drained and st["injected"] == st["ejected"] and o.fifo_packets() == 0


@pytest.mark.parametrize("w", [8, 16])
def test_throughput_below_bisection_bound(w):
    """Uniform random traffic: accepted throughput <= 4/k flits/node/cycle."""
    o = Oracle(W.make(mesh_w=w, mesh_h=w, mode=W.MODE_UR, lam=0.5))
    o.run(1500)
    o2 = o.stats()[0]["ejected"]
    o.run(1500)
    acc = (o.stats()[0]["ejected"] - o2) / (w * w * 1500)
    assert 0 < acc <= 4 / w


def test_age_equals_deflection_count():
    """Age = number of deflections: total deflections = sum of
    ages of ejected flits + ages of flits still in flight."""
    o = Oracle(W.make(mesh_w=8, mesh_h=8, mode=W.MODE_UR, lam=0.3))
    o.run(3000)
    st, _, hd, _ = o.stats()
    assert hd[-1] == 0
    k, inflight_age = o.links_occupied()
    assert st["deflections"] == sum(b * c for b, c in enumerate(hd)) + inflight_age
    assert st["deflections"] > 0


def test_node_order_does_not_matter():
    """Stages read only the previous cycle's links and write node-owned state
    or next-cycle link slots: reversing the node order in every
    phase leaves the state hash unchanged."""
    for cfg in (W.c1a(), W.c1b(), W.make(mesh_w=7, mesh_h=5, mode=W.MODE_LSPD, lam=0.3,
                                         l2_sets=2, l2_ways=2, sendq_cap=32, mem_lat=20)):
        a, b = Oracle(cfg), Oracle(cfg, debug=DBG_REVERSE)
        a.run(2500)
        b.run(2500)
        assert a.state_hash() == b.state_hash()
        assert a.stats() == b.stats()


def test_split_run_invariance():
    for cfg in (W.c1a(), W.c1b()):
        a, b = Oracle(cfg), Oracle(cfg)
        a.run(3000)
        b.run(1234)
        b.run(1766)
        assert a.state_hash() == b.state_hash()


def test_hash_sensitive_to_seed_and_cycle():
    a, b = Oracle(W.c1b(seed=1)), Oracle(W.c1b(seed=2))
    a.run(500)
    b.run(500)
    assert a.state_hash() != b.state_hash()
    h = a.state_hash()
    a.run(1)
    assert a.state_hash() != h


def test_lambda_zero_is_inert():
    """lambda = 0: nothing is generated; the state is independent of the seed."""
    for mode in (W.MODE_UR, W.MODE_LSPD):
        a = Oracle(W.make(mode=mode, thr_inj=0, seed=1))
        b = Oracle(W.make(mode=mode, thr_inj=0, seed=99))
        a.run(777)
        b.run(777)
        st = a.stats()[0]
        assert all(v == 0 for k, v in st.items() if k != "cycle")
        assert a.state_hash() == b.state_hash()


def test_private_working_set_that_fits_never_evicts():
    """PRIV <= SETS*WAYS and SETS | TPN with all accesses private: no eviction,
    and every access after a tag's first touch hits."""
    cfg = W.make(mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, priv_tags=8, thr_priv=2 ** 32 - 1,
                 lam=0.1, sendq_cap=32)
    o = Oracle(cfg, debug=DBG_INVARIANTS)
    o.run(60000)
    st = o.stats()[0]
    assert st["evictions"] == 0
    assert st["l2_misses"] == 16 * 8
    assert st["l2_hits"] == st["accesses"] - 16 * 8


# ---------------------------------------------------------------- LRU
def lru_replay(tags, sets, ways):
    """Textbook LRU per set: invalid ways first, else least recently used."""
    cache = [collections.OrderedDict() for _ in range(sets)]
    hits = misses = ev = 0
    for t in tags:
        c = cache[t % sets]
        if t in c:
            hits += 1
            c.move_to_end(t)
        else:
            misses += 1
            if len(c) == ways:
                c.popitem(last=False)
                ev += 1
            c[t] = True
    return [set(c) for c in cache], hits, misses, ev


@pytest.mark.parametrize("sets,ways", [(1, 1), (1, 4), (3, 2), (2, 3)])
def test_lru_matches_brute_force_replay(sets, ways):
    """All accesses by node 0 of a 2x2 mesh to tags homed at node 0 (T mod 4 =
    0): the whole protocol is loopback (R28), accesses are serialised,
    so the slice must behave as a textbook LRU (R23)."""
    rng = random.Random(sets * 100 + ways)
    for trial in range(40):
        pool = [4 * rng.randrange(60) for _ in range(rng.randrange(1, 3 * ways * sets + 2))]
        tags = [rng.choice(pool) for _ in range(rng.randrange(1, 40))]
        cfg = W.make(mesh_w=2, mesh_h=2, mode=W.MODE_LSPD, l2_sets=sets, l2_ways=ways,
                     thr_inj=0, mem_lat=3, l2_hit_lat=1, sendq_cap=8)
        # one access per 5 cycles (> mem_lat): no two touches share a cycle stamp
        o = Oracle(cfg, script=[(5 * i, 0, t) for i, t in enumerate(tags)])
        o.run(len(tags) * 5 + 10)
        st = o.stats()[0]
        want_sets, hits, misses, ev = lru_replay(tags, sets, ways)
        assert st["completed"] == len(tags)
        assert (st["l2_hits"], st["l2_misses"], st["evictions"]) == (hits, misses, ev)
        for s in range(sets):
            got = {o.l2_line(0, s, w)[1] for w in range(ways) if o.l2_line(0, s, w)[0]}
            assert got == want_sets[s]
        assert st["injected"] == 0


# ---------------------------------------------------------------- Fig. 4 protocol timelines
def tag_homed_at(home, n=16, k=7):
    return 16 * k + home


def fig4_scenario(case, S, home, holder):
    """Script for one Fig. 4 case on 4x4; returns (script, expected extra
    latencies of the set-up accesses)."""
    T = tag_homed_at(home)
    mem, nfl = 100, 4
    if case == "local_hit":
        return [(0, S, T), (400, S, T)], [2 * manhattan(S, home, 4) + 1 + mem]
    if case in ("remote_hit", "loopback_remote"):
        # holder fetches T from memory first (NDR path), then S asks for it
        return [(0, holder, T), (400, S, T)], [2 * manhattan(holder, home, 4) + 1 + mem
                                               if holder != home else mem]
    if case in ("memory", "memory_far", "loopback_memory"):
        return [(0, S, T)], []
    if case == "trap":
        # holder's fill is still outstanding (MEMWAIT) when S's request reaches it
        return [(0, holder, T), (20, S, T)], [2 * manhattan(holder, home, 4) + 1 + mem]
    raise KeyError(case)


def test_fig4_timelines():
    """Zero-load latencies of every Fig. 4 path against the hand-derived
    closed forms in tests/golden/fig4_timelines.txt."""
    for case, S, home, holder, lat in golden("fig4_timelines.txt"):
        S = int(S)
        home = int(home) if home != "-" else S
        holder = int(holder) if holder != "-" else None
        script, setup = fig4_scenario(case, S, home, holder)
        cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32)
        o = Oracle(cfg, script=script, debug=DBG_INVARIANTS)
        o.run(1000)
        st, _, hd, ha = o.stats()
        got = collections.Counter({b: c for b, c in enumerate(ha) if c})
        want = collections.Counter(setup + [int(lat)])
        assert got == want, (case, dict(got), dict(want))
        assert st["deflections"] == 0
        if case == "trap":
            assert st["traps_sent"] == st["traps_received"] == 1
        if case in ("remote_hit", "loopback_remote"):
            assert st["replies_received"] == 1 and st["requests_made"] == 1


def test_fig4_timelines_centralized_directory():
    """NEXT-f3: with the directory at one node D (R40), every
    access's directory leg goes to D whatever the tag, against the closed forms
    of tests/golden/fig4_timelines_central.txt."""
    for case, S, D, homed, holder, lat in golden("fig4_timelines_central.txt"):
        S, D, homed = int(S), int(D), int(homed)
        holder = int(holder) if holder != "-" else None
        T = tag_homed_at(homed)
        mem = 100
        if case == "remote_hit":
            script, setup = [(0, holder, T), (400, S, T)], [2 * manhattan(holder, D, 4) + 1 + mem]
        elif case == "trap":
            script, setup = [(0, holder, T), (20, S, T)], [2 * manhattan(holder, D, 4) + 1 + mem]
        else:
            script, setup = [(0, S, T)], []
        cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32,
                     dir_mode=W.DIR_CENTRAL, dir_node=D)
        o = Oracle(cfg, script=script, debug=DBG_INVARIANTS)
        o.run(1000)
        st, _, _, ha = o.stats()
        got = collections.Counter({b: c for b, c in enumerate(ha) if c})
        assert got == collections.Counter(setup + [int(lat)]), (case, S, D, dict(got))
        assert st["deflections"] == 0


def test_table1_flit_division_of_remote_hit():
    """Table I: DA, DR = 1 flit, remote L2 access RA = 4 flits.  A
    remote hit moves DA + DR + RQ + RA = 1 + 1 + 1 + 4 flits (R18)."""
    t1 = {r[1]: int(r[2]) for r in golden("table1_flits.txt")}
    T = tag_homed_at(5)
    cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, nfl_ra=t1["RA"])
    o = Oracle(cfg, script=[(0, 15, T)])
    o.run(400)
    before = o.stats()[0]["injected"]
    assert before == t1["DA"] + t1["DR"]          # holder's DA + negative reply
    o2 = Oracle(cfg, script=[(0, 15, T), (400, 0, T)])
    o2.run(800)
    st = o2.stats()[0]
    assert st["injected"] - before == t1["DA"] + t1["DR"] + 1 + t1["RA"]
    assert st["replies_received"] == 1


def test_directory_example_tag_100_at_row2_col4():
    """Fig. 2: tag 100 held by the node at row 2, column 4.  Node
    (x=4, y=2) of a 5x3 mesh fetches tag 100; the location array records it."""
    g = {r[0]: int(r[1]) for r in golden("directory.txt")}
    w, h = 5, 3
    node = g["example_row"] * w + g["example_col"]
    cfg = W.make(mesh_w=w, mesh_h=h, mode=W.MODE_LSPD, thr_inj=0)
    o = Oracle(cfg, script=[(0, node, g["example_tag"])])
    o.run(300)
    holder, pend = o.loc(g["example_tag"])
    assert (holder // w, holder % w) == (g["example_row"], g["example_col"]) and pend == 0
    # and the sizing of the paper's location array (reading R36)
    entries = g["mem_bytes"] // g["line_bytes"]
    assert entries == g["location_array_entries"] == 2 ** 24
    assert entries * g["entry_bytes"] == g["location_array_bytes"]
    assert g["onchip_bytes"] // g["line_bytes"] * g["entry_bytes"] == g["associative_bytes"]


def test_miss_under_miss_not_allowed():
    """while a node waits for a remote block it issues no new access:
    every node has at most one outstanding access at any cycle."""
    o = Oracle(W.c1b(lam=0.9))
    for _ in range(50):
        o.run(37)
        st = o.stats()[0]
        assert st["accesses"] - st["completed"] == o.cores_busy() <= 16


def test_trace_loader_grammar_and_replay():
    """NEXT-f3 trace replay input: the SPEC line grammar (comments, blank lines,
    optional R/W) parses to per-node streams, tag = address // line mod TPN*N
    (R41); malformed lines are rejected; a replay drains with the Table II
    equalities and each record starts exactly one access."""
    cfg = W.c1b(thr_inj=0)
    ev = W.load_trace(os.path.join(GOLDEN, "trace_4x4.txt"), cfg)
    assert ev == [(0, 0, 0), (0, 0, 128), (0, 5, 5), (0, 5, 5), (0, 15, 1), (0, 3, 15),
                  (0, 12, (0x3fffe0 // 32) % (128 * 16))]
    o = Oracle(cfg, script=ev, debug=DBG_INVARIANTS)
    o.run(2000)
    st = o.stats()[0]
    assert st["accesses"] == len(ev) == st["completed"]
    assert st["l2_hits"] == 1
    bad = os.path.join(os.path.dirname(GOLDEN), "_bad_trace.txt")
    for text in ("0 zz\n", "99 0x10\n", "1 0x10 X\n"):
        with open(bad, "w") as f:
            f.write(text)
        with pytest.raises(ValueError):
            W.load_trace(bad, cfg)
    os.unlink(bad)


def test_l1_timelines_and_writebacks():
    """NEXT-f1 private L1 (R42) against the closed forms of
    tests/golden/l1_timelines.txt: an L1 hit is served at once, a miss waits
    l1_miss_lat before the local L2 / Fig. 4 sequence, and every L1 victim is
    written back to the slice that supplied it."""
    for case, S, accs, lats, wbs in golden("l1_timelines.txt"):
        S = int(S)
        script, want = [], []
        cyc = 0
        holders = []
        for a in accs.split():
            if a.startswith("r"):        # remote block: first fetched by its holder
                holder, home = (int(v) for v in a[1:].split("@"))
                T = tag_homed_at(home, k=9)
                if holder not in holders:
                    script.append((cyc, holder, T))
                    want.append(2 * manhattan(holder, home, 4) + 1 + 100 + 2)
                    holders.append(holder)
                    cyc += 300
                script.append((cyc, S, T))
            else:
                script.append((cyc, S, tag_homed_at(int(a))))
            cyc += 300
        want += [int(v) for v in lats.split()]
        cfg = W.make(mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, sendq_cap=32,
                     l1_sets=1, l1_ways=1, l1_miss_lat=2)
        o = Oracle(cfg, script=script, debug=DBG_INVARIANTS)
        o.run(cyc + 300)
        st, _, _, ha = o.stats()
        got = collections.Counter({b: c for b, c in enumerate(ha) if c})
        assert got == collections.Counter(want), (case, dict(got), want)
        sent, local = (int(v) for v in wbs.split())
        assert st["deflections"] == 0
        assert st["wb_sent"] == st["wb_received"] == sent, case
        assert st["l1_hits"] + st["l1_misses"] == st["accesses"]


def test_l1_off_is_the_base_model():
    """l1_sets = 0 leaves every counter, histogram and the hash of the base
    model unchanged whatever the other L1 knobs say."""
    a = Oracle(W.c1b(seed=2))
    b = Oracle(W.c1b(seed=2, l1_ways=4, l1_miss_lat=7))
    a.run(3000)
    b.run(3000)
    assert a.stats() == b.stats() and a.state_hash() == b.state_hash()
    assert a.stats()[0]["l1_hits"] == a.stats()[0]["l1_misses"] == 0


@pytest.mark.parametrize("mode,injected", [(0, 2), (1, 3)])
def test_inject_when_eject_frees_a_slot(mode, injected):
    """NEXT-f4 injection mode (R43).  2x2 mesh, cycle 0: node 1
    sends a probe to node 2 (XY: through node 0) and node 2 one to node 0; at
    cycle 1 both sit at node 0 (degree 2), one of them ejecting, while node 0
    queues a probe to node 3.  Under R7 node 0 cannot inject at cycle 1 (two
    flits = degree); when an ejecting flit frees its port it can."""
    cfg = W.make(mesh_w=2, mesh_h=2, mode=W.MODE_UR, thr_inj=0, inject_mode=mode)
    o = Oracle(cfg, script=[(0, 1, 2), (0, 2, 0), (1, 0, 3)], debug=DBG_INVARIANTS)
    o.run(2)
    assert o.stats()[0]["injected"] == injected
    o.run(20)
    st = o.stats()[0]
    assert st["injected"] == st["ejected"] == 3 and st["deflections"] == 0


def test_arbitration_degree_plus_one_with_an_ejecting_flit():
    """Under the NEXT-f4 injection mode a router holds up to degree + 1 flits
    when one ejects: the greedy still equals the brute force and never drops a
    flit (random degree-2/3/4 cases of a 3x3 mesh, both routings)."""
    rng = random.Random(77)
    w = h = 3
    for node in (0, 1, 4):
        deg = sum(exists(w, h, node, p) for p in range(4))
        for route in (W.ROUTE_PMDR, W.ROUTE_XY):
            for _ in range(3000):
                pool = rng.sample(range(20), 6)
                flits = [random_flit(rng, 9, pool) for _ in range(deg)]
                k = rng.randrange(deg)
                flits[k] = (node,) + flits[k][1:]                 # one of them at its destination
                flits.append((rng.choice([d for d in range(9) if d != node]), node, 0, 2))   # injected
                check_case(w, h, node, W.PRIO_DEFLECT, flits, route)


@pytest.mark.parametrize("name,cfg", [
    ("ur6x5_inj", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_UR, lam=0.4, inject_mode=1)),
    ("lspd6x5_inj", W.make(mesh_w=6, mesh_h=5, mode=W.MODE_LSPD, l2_sets=4, l2_ways=2, lam=0.2,
                           sendq_cap=32, seed=7, mem_lat=30, inject_mode=1)),
])
def test_inject_mode_invariants_and_drain(name, cfg):
    """Conservation / exclusivity / top-priority progress every cycle and
    delivery of everything under the NEXT-f4 injection mode."""
    o = Oracle(cfg, debug=DBG_INVARIANTS)
    o.run(3000)
    used, drained = o.drain(200000)
    assert drained
    st = o.stats()[0]
    assert st["injected"] == st["ejected"]
