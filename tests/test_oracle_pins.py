"""Pins of the oracle parts that round 1 left free: the canonical state hash
(the parity witness of every GPU test) and the generator's draw mappings.

Nothing here compares the oracle with itself:
  * the state hash is re-evaluated in Python, from DESIGN.md section 3.7's
    written definition (splitmix64 finalizer, tuple fold, domains, indices and
    canonicalisation rules), over the raw state peeked field by field from the
    oracle -- a dropped domain, a wrong index or tuple order, or a hashed dead
    field makes the two disagree; every single-field mutation must change the
    oracle's hash and agree with the Python evaluation of the mutated state;
  * the draw mappings are checked against the distributions SURVEY 8(d.1) /
    DESIGN 5 state (uniform over the N-1 other nodes; private blocks uniform
    over the node's PRIV window; shared blocks uniform over the N*(TPN-PRIV)
    pool), and against what the simulation actually generated.
"""
import collections
import math

import pytest

from oracle import Oracle
from paper_1508_03235_b200 import workloads as W

M64 = (1 << 64) - 1


# ---------------------------------------------------------------- DESIGN 3.7
def mix(x):
    """splitmix64 finalizer (DESIGN 3.7)."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def tup(vals):
    """tuple(v0..vk-1): h = k; h = mix(h ^ vi) for each i."""
    h = len(vals)
    for v in vals:
        h = mix(h ^ (v & M64))
    return h


def term(dom, idx, vals):
    return mix(mix(((dom << 56) ^ idx) & M64) ^ tup(vals))


LINK, FIFO, FIFONEXT, CORE, L2, LOC, CNT, HIST, CYCLE, SCRIPT, L1, L2MIG, LOCMIG, MIGRX = range(1, 15)
IDLE, L2WAIT, WAIT_DIR, WAIT_DATA, MEMWAIT, L1WAIT, MEMFETCH = range(7)


def snapshot(o, cfg):
    """The raw state, field by field, through the oracle's peeks."""
    N = cfg["mesh_w"] * cfg["mesh_h"]
    lspd = cfg["mode"] == W.MODE_LSPD
    st = {"links": {}, "fifo": {}, "core": {}, "l2": {}, "l1": {}, "loc": {}, "script": {},
          "l2mig": {}, "locmig": {}, "migrx": {}}
    mig = lspd and cfg.get("mig_hist", 0) > 0
    for n in range(N):
        for d in range(4):
            f = o.link(n, d)
            if f is not None:
                st["links"][(n, d)] = f
        st["fifo"][n] = o.fifo(n)
        st["core"][n] = o.core(n)
        st["script"][n] = o.script_used(n)
        if mig:
            for k in range(4):
                st["migrx"][(n, k)] = o.migrx(n, k)
        if lspd:
            for s in range(cfg["l2_sets"]):
                for w in range(cfg["l2_ways"]):
                    st["l2"][(n, s, w)] = o.l2_line(n, s, w)
                    if mig:
                        st["l2mig"][(n, s, w)] = o.l2_mig(n, s, w) + (o.l2_hist(n, s, w),)
            if cfg["l1_sets"]:
                for s in range(cfg["l1_sets"]):
                    for w in range(cfg["l1_ways"]):
                        st["l1"][(n, s, w)] = o.l1_line(n, s, w)
    if lspd:
        for T in range(cfg["tags_per_node"] * N):
            st["loc"][T] = o.loc(T)
            if mig:
                st["locmig"][T] = o.loc_mig(T)
    cnt, hl, hd, ha = o.stats()
    st["cnt"], st["hist"], st["cycle"] = cnt, (hl, hd, ha), cnt["cycle"]
    return st


def design_hash(st, cfg):
    """DESIGN 3.7, written out from its table."""
    H = 0
    add = lambda dom, idx, vals: term(dom, idx, vals)
    terms = []
    for (n, d), f in st["links"].items():     # occupied input slots of the next cycle
        terms.append(add(LINK, n * 4 + d, [f["dst"], f["src"], f["kind"], f["fid"], f["payload"],
                                          f["age"], f["inj"]]))
    for n, (nxt, pkts) in st["fifo"].items():
        for k, (kind, dst, payload, nfl) in enumerate(pkts):   # position from the head
            terms.append(add(FIFO, (n << 16) + k, [kind, dst, payload, nfl]))
        if nxt:
            terms.append(add(FIFONEXT, n, [nxt]))
    live = {L2WAIT: ("ready", "start"), WAIT_DIR: ("tag", "start"), WAIT_DATA: ("tag", "start", "rx"),
            MEMWAIT: ("ready", "tag", "install", "start"), L1WAIT: ("ready", "tag", "start"),
            MEMFETCH: ("tag", "install", "start", "rx")}
    for n, c in st["core"].items():
        if c["mode"] == IDLE:
            continue
        keep = live[c["mode"]]
        v = [c["mode"]] + [c[k] if k in keep else 0 for k in ("ready", "tag", "install", "start", "rx")]
        terms.append(add(CORE, n, v))
    S, Wy = cfg["l2_sets"], cfg["l2_ways"]
    for (n, s, w), (valid, tag, stamp) in st["l2"].items():
        if valid:
            terms.append(add(L2, (n * S + s) * Wy + w, [tag, stamp]))
    S1, W1 = cfg["l1_sets"], cfg["l1_ways"]
    for (n, s, w), (valid, tag, stamp, owner) in st["l1"].items():
        if valid:
            terms.append(add(L1, (n * S1 + s) * W1 + w, [tag, stamp, owner]))
    for T, (holder, pend) in st["loc"].items():
        hv = 0 if holder == 0xFFFFFFFF else holder + 1
        if hv or pend:
            terms.append(add(LOC, T, [hv, pend]))
    names = list(W_COUNTERS)
    for i, name in enumerate(names):
        terms.append(add(CNT, i, [st["cnt"][name] & M64]))
    for h, hist in enumerate(st["hist"]):
        for b, v in enumerate(hist):
            if v:
                terms.append(add(HIST, (h << 32) + b, [v]))
    terms.append(add(CYCLE, 0, [st["cycle"]]))
    # NEXT-f2 (DESIGN 3.7 domains 12-14): line migration state and history,
    # directory transit flags, inbound migration reassembly slots
    for (n, s_, w), (mstate, mtarget, hcount, hist) in st["l2mig"].items():
        valid, tag = st["l2"][(n, s_, w)][:2]
        if mstate == 0 and (not valid or hcount == 0):
            continue
        terms.append(add(L2MIG, (n * S + s_) * Wy + w, [mstate, tag, mtarget, hcount] + list(hist)))
    for T, (transit, early) in st["locmig"].items():
        if transit or early:
            terms.append(add(LOCMIG, T, [transit, early]))
    for (n, k), (used, tag, count) in st["migrx"].items():
        if used:
            terms.append(add(MIGRX, (n << 2) + k, [tag, count]))
    for n, used in st["script"].items():
        if used:
            terms.append(add(SCRIPT, n, [used]))
    for x in terms:
        H = (H + x) & M64
    return H


# counters in the order of DESIGN 3.6 (hash index 0..46)
W_COUNTERS = ("generated", "packets_enqueued", "injected", "ejected", "hops", "deflections",
              "probes_delivered", "accesses", "completed", "l2_hits", "l2_misses",
              "dir_searches", "requests_made", "requests_received", "replies_sent",
              "replies_received", "traps_sent", "traps_received", "mem_requests",
              "installs", "evictions", "evs_sent", "evs_received",
              "drops_probe", "drops_da", "drops_dr", "drops_ndr", "drops_rq", "drops_ra",
              "drops_trap", "drops_ev", "l1_hits", "l1_misses", "wb_sent", "wb_received",
              "mig_requests", "mig_nacks", "migrations", "mig_installs", "dir_updates", "invalidations",
              "redirections", "rr_received",
              "mem_fills_sent", "mem_fills_received", "mem_wbs_sent", "mem_wb_flits")


def _busy_lspd(w, h, **kw):
    kw.setdefault("lam", 0.3)
    kw.setdefault("sendq_cap", 8)
    return W.make(mesh_w=w, mesh_h=h, mode=W.MODE_LSPD, l2_sets=2, l2_ways=2, tags_per_node=8,
                  priv_tags=4, mem_lat=7, hist_bins=64, **kw)


HASH_CASES = {
    "ur2x2": W.make(mesh_w=2, mesh_h=2, mode=W.MODE_UR, lam=0.6, sendq_cap=4, hist_bins=32),
    "ur3x3_oldest": W.make(mesh_w=3, mesh_h=3, mode=W.MODE_UR, lam=0.5, prio=W.PRIO_OLDEST,
                           sendq_cap=4, hist_bins=32, seed=7),
    "lspd2x2": _busy_lspd(2, 2),
    "lspd3x3": _busy_lspd(3, 3, seed=3),
    "lspd3x3_l1": _busy_lspd(3, 3, seed=5, l1_sets=1, l1_ways=2, l1_miss_lat=2),
    "lspd3x3_central": _busy_lspd(3, 3, seed=2, dir_mode=W.DIR_CENTRAL, dir_node=4),
    "lspd3x3_mig": _busy_lspd(3, 3, seed=6, mig_hist=3, nfl_b2=5, sendq_cap=64),
    "lspd3x3_memctrl": _busy_lspd(3, 3, seed=4, mem_mode=W.MEM_CTRLS, mem_ctrls=2, nfl_b2=3,
                                  sendq_cap=32, hub_sendq_cap=64),
    "lspd3x3_memhome": _busy_lspd(3, 3, seed=8, mem_mode=W.MEM_HOME, nfl_b2=2, sendq_cap=32,
                                  dir_mode=W.DIR_CENTRAL, dir_node=4, hub_sendq_cap=64),
}


@pytest.mark.parametrize("name", sorted(HASH_CASES))
def test_state_hash_equals_design_definition(name):
    """orc_state_hash == DESIGN 3.7 evaluated in Python over the peeked state,
    at several points of a busy run (flits on links, queued packets with a
    partly sent head, every core mode, valid lines, directory entries)."""
    cfg = HASH_CASES[name]
    script = None
    if name == "lspd3x3":
        script = W.random_script(cfg, 12, 40, seed=11)     # SCRIPT domain
    o = Oracle(cfg, script=script)
    seen_domains = collections.Counter()
    for step in (0, 1, 3, 7, 19, 40, 77):
        o.run(step)
        st = snapshot(o, cfg)
        assert o.state_hash() == design_hash(st, cfg), "at cycle %d" % st["cycle"]
        seen_domains["link"] += len(st["links"])
        seen_domains["fifo"] += sum(len(p) for _, p in st["fifo"].values())
        seen_domains["fifonext"] += sum(1 for nx, _ in st["fifo"].values() if nx)
        seen_domains["core"] += sum(1 for c in st["core"].values() if c["mode"])
        seen_domains["script"] += sum(1 for v in st["script"].values() if v)
        seen_domains["memfetch"] += sum(1 for c in st["core"].values() if c["mode"] == MEMFETCH)
    assert seen_domains["link"] > 0 and seen_domains["fifo"] > 0
    if cfg["mode"] == W.MODE_LSPD:
        assert seen_domains["core"] > 0
    if name == "lspd3x3":
        assert seen_domains["script"] > 0
    if name.startswith("lspd3x3_mem"):
        assert seen_domains["memfetch"] > 0 or name == "lspd3x3_memhome"


def _first(d, pred):
    for k, v in d.items():
        if pred(v):
            return k
    return None


def test_every_field_mutation_changes_the_hash():
    """Each hashed field, mutated alone (orc_poke), changes the oracle's hash
    and the new value still equals DESIGN 3.7 over the mutated state; a dead
    core field (not live in the current mode, DESIGN 3.7) does not."""
    cfg = HASH_CASES["lspd3x3_l1"]
    o = Oracle(cfg)
    o.run(30)
    st = snapshot(o, cfg)
    (ln, ld) = next(iter(st["links"]))
    n_fifo = _first(st["fifo"], lambda v: len(v[1]) > 0)
    n_busy = _first(st["core"], lambda c: c["mode"] in (WAIT_DIR, WAIT_DATA, MEMWAIT))
    l2k = _first(st["l2"], lambda v: v[0])
    l1k = _first(st["l1"], lambda v: v[0])
    T = _first(st["loc"], lambda v: v[0] != 0xFFFFFFFF)
    assert None not in (n_fifo, n_busy, l2k, l1k, T)
    pokes = [(0, ln, ld, 0, 1), (1, ln, ld, 0, 5), (2, n_busy, 0, 0, 3), (3, n_busy, 0, 0, IDLE),
             (4, l2k[0], l2k[1], l2k[2], 2), (5, T, 0, 0, 1), (6, n_fifo, 0, 0, 9), (7, n_fifo, 0, 0, 1),
             (8, 0, 4, 0, 1), (8, 0, 34, 0, 1), (9, 0, 0, 3, 1), (9, 0, 2, 5, 1), (10, 0, 0, 0, 1),
             (11, l1k[0], l1k[1], l1k[2], 1)]
    for field, n, i, j, v in pokes:
        before = o.state_hash()
        o.poke(field, n, i, j, v)
        after = o.state_hash()
        assert after != before, "field %d not hashed" % field
        assert after == design_hash(snapshot(o, cfg), cfg), "field %d" % field
    # rx is dead in WAIT_DIR / MEMWAIT (DESIGN 3.7): mutating it must not matter
    n_dead = _first(snapshot(o, cfg)["core"], lambda c: c["mode"] in (WAIT_DIR, MEMWAIT))
    if n_dead is not None:
        before = o.state_hash()
        o.poke(12, n_dead, 0, 0, 1)
        assert o.state_hash() == before


# ---------------------------------------------------------------- generator mappings
def chi2_ok(counts, expected, dof):
    """Pearson chi-square below mean + 6 sd (dof + 6*sqrt(2 dof))."""
    x = sum((c - expected) ** 2 / expected for c in counts)
    return x < dof + 6 * math.sqrt(2 * dof)


def test_ur_destination_uniform_over_other_nodes():
    """UR probes (R25): the destination is never the source and
    is uniform over the N-1 other nodes."""
    cfg = W.make(mesh_w=5, mesh_h=4, mode=W.MODE_UR, thr_inj=(1 << 32) - 1)
    o = Oracle(cfg)
    N, T = 20, 6000
    for n in (0, 7, 19):
        cnt = collections.Counter()
        for t in range(T):
            fired, d = o.gen(n, t)
            assert fired and d != n and 0 <= d < N
            cnt[d] += 1
        assert chi2_ok([cnt[d] for d in range(N) if d != n], T / (N - 1), N - 2)


def test_lspd_private_and_shared_blocks_uniform():
    """LSPD addresses (DESIGN 5): private with probability
    p_priv, uniform over the node's PRIV-block window n*TPN + [0, PRIV);
    shared uniform over the pool {m*TPN + PRIV + j}: owner m uniform over all
    N nodes, offset j uniform over [0, TPN-PRIV), independently."""
    N, TPN, PRIV = 12, 16, 10
    cfg = W.make(mesh_w=4, mesh_h=3, mode=W.MODE_LSPD, tags_per_node=TPN, priv_tags=PRIV,
                 thr_inj=(1 << 32) - 1, p_priv=0.3)
    o = Oracle(cfg)
    n, T = 5, 30000
    priv, owner, off, joint = collections.Counter(), collections.Counter(), collections.Counter(), \
        collections.Counter()
    npriv = 0
    for t in range(T):
        fired, tag = o.gen(n, t)
        assert fired and 0 <= tag < TPN * N
        m, j = divmod(tag, TPN)
        if j < PRIV:
            assert m == n, "a private-window block of another node"
            npriv += 1
            priv[j] += 1
        else:
            owner[m] += 1
            off[j - PRIV] += 1
            joint[(m, j - PRIV)] += 1
    p = W.thr(0.3) / 2 ** 32
    assert abs(npriv - T * p) < 5 * math.sqrt(T * p * (1 - p))
    ns = T - npriv
    assert chi2_ok([priv[j] for j in range(PRIV)], npriv / PRIV, PRIV - 1)
    assert chi2_ok([owner[m] for m in range(N)], ns / N, N - 1)
    assert chi2_ok([off[j] for j in range(TPN - PRIV)], ns / (TPN - PRIV), TPN - PRIV - 1)
    cells = N * (TPN - PRIV)
    assert chi2_ok([joint[(m, j)] for m in range(N) for j in range(TPN - PRIV)], ns / cells, cells - 1)


def test_generator_fire_rate_and_simulation_use_it():
    """The generation the simulation performs is this mapping: UR `generated`
    equals the number of fired draws over all (node, cycle), and an LSPD
    access started at cycle s by node n has tag = the draw of (n, s)."""
    cfg = W.make(mesh_w=3, mesh_h=3, mode=W.MODE_UR, lam=0.2, sendq_cap=64)
    o = Oracle(cfg)
    o.run(300)
    fired = sum(o.gen(n, t)[0] for n in range(9) for t in range(300))
    st = o.stats()[0]
    assert st["generated"] == fired and st["drops_probe"] == 0
    cfg = _busy_lspd(3, 3, seed=9)
    o = Oracle(cfg)
    checked = 0
    for _ in range(60):
        o.run(5)
        for n in range(9):
            c = o.core(n)
            if c["mode"] in (WAIT_DIR, WAIT_DATA, MEMWAIT):
                f, tag = o.gen(n, c["start"])
                assert f and tag == c["tag"]
                checked += 1
    assert checked > 20


def test_state_hash_definition_through_migrations():
    """The NEXT-f2 domains (line migration state and history, directory
    transit flags, inbound reassembly slots) at every third cycle of a run
    with migrations in flight: DESIGN 3.7 equals the oracle's hash."""
    cfg = HASH_CASES["lspd3x3_mig"]
    o = Oracle(cfg)
    seen = collections.Counter()
    for _ in range(60):
        o.run(3)
        st = snapshot(o, cfg)
        assert o.state_hash() == design_hash(st, cfg)
        seen["line"] += sum(1 for v in st["l2mig"].values() if v[0] > 0)
        seen["loc"] += sum(1 for v in st["locmig"].values() if v[0] or v[1])
        seen["rx"] += sum(1 for v in st["migrx"].values() if v[0])
    assert seen["line"] and seen["loc"] and seen["rx"] and o.stats()[0]["migrations"] > 0
