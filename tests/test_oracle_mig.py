"""Pins of the NEXT-f2 oracle extension: migration + redirection (P:L54,
P:L75-80, L85, Table I; readings R44-R52 of
DESIGN.md).  Nothing here compares the oracle with itself:
  * the migration decision against SPEC's worked examples (golden fixture);
  * hand-derived zero-load timelines: the cycle the directory update lands at
    home, the local hit that follows, and the latency of a redirected access
    (2 d1 + 2 d2 + 2 d3 + 4 + nfl_RA);
  * invariants every cycle (single copy plus at most one source copy in
    transit, directory agreement at quiescence) and message conservation on
    random configurations."""
import os
import random

import pytest

import oracle
from oracle import Oracle, DBG_INVARIANTS
from paper_1508_03235_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_migration_decision_spec_examples():
    rows = 0
    for line in open(os.path.join(GOLDEN, "migration_decision.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        hist, holder, want, _src = [c.strip() for c in line.split("|")]
        hist = [int(v) for v in hist.split()]
        got = oracle.mig_target(hist, int(holder))
        assert got == (None if want == "none" else int(want)), line
        rows += 1
    assert rows == 7


def man(a, b, w):
    return abs(a % w - b % w) + abs(a // w - b // w)


def mig_cfg(**kw):
    base = dict(mesh_w=6, mesh_h=6, mode=W.MODE_LSPD, thr_inj=0, l2_sets=4, l2_ways=2, mig_hist=2,
                nfl_b2=16, sendq_cap=64)
    base.update(kw)
    return W.make(**base)


def test_zero_load_migration_and_redirection_timeline():
    """6x6, zero load.  B fetches T (home H); S reads T twice remotely: with a
    2-entry history the second read makes S the majority accessor, so B asks
    H (MR), gets the grant (MG), sends the 16-flit block (two 8-flit parts),
    S installs it and its directory update (DU) reaches H at
        t_DU = t_B + 23 + 2 d(B,H) + d(B,S) + d(S,H),
    t_B = the cycle B served S's request = 600 + 2 d(S,H) + 2 + d(S,B)
    (RA 4 flits, then MR, one flit per cycle; MG back; 16 flits; DU).  A
    third node C whose directory access lands at H just before t_DU gets
    DR(B); its request reaches B after the invalidation, so B redirects it
    (RR) to S: latency 2 d(C,H) + 2 d(C,B) + 2 d(C,S) + 4 + nfl_RA."""
    w = 6
    B, S, H, C = 7, 22, 30, 35
    T = H + 36 * 2
    cfg = mig_cfg()
    dSH, dSB, dBH, dBS = man(S, H, w), man(S, B, w), man(B, H, w), man(B, S, w)
    tB = 600 + 2 * dSH + 2 + dSB
    tDU = tB + 23 + 2 * dBH + dBS + dSH
    dCH, dCB, dCS = man(C, H, w), man(C, B, w), man(C, S, w)
    tC = tDU - 1 - dCH            # C's DA is ejected at H one cycle before the DU
    script = [(0, B, T), (300, S, T), (600, S, T), (tC, C, T), (tDU + 200, S, T)]
    o = Oracle(cfg, script=script, debug=DBG_INVARIANTS)
    o.run(tDU)
    st = o.stats()[0]
    assert st["migrations"] == 1 and st["dir_updates"] == 0
    o.run(1)
    st = o.stats()[0]
    assert st["dir_updates"] == 1 and st["mig_installs"] == 1
    assert o.loc(T)[0] == S
    o.run(2000)
    st, hl, hd, ha = o.stats()
    assert st["redirections"] == 1 and st["rr_received"] == 1 and st["invalidations"] == 1
    lat = {b for b, v in enumerate(ha) if v}
    # B's memory fill, S's two remote reads, C's redirected read, S's local hit
    want_c = 2 * dCH + 2 * dCB + 2 * dCS + 4 + cfg["nfl_ra"]
    assert want_c in lat
    assert cfg["l2_hit_lat"] in lat                   # S now reads T locally
    assert 2 * dSH + 2 * dSB + 2 + cfg["nfl_ra"] in lat   # the remote reads (Fig. 4 form)
    assert st["accesses"] == st["completed"] == 5
    # B keeps a forwarding ghost pointing at S; S holds the block
    s = T % 4
    ghosts = [o.l2_mig(B, s, way) for way in range(2)]
    assert (3, S, 0) in ghosts
    assert any(o.l2_line(S, s, way)[:2] == (1, T) for way in range(2))
    assert o.directory_quiescent_ok()


def test_local_majority_keeps_the_block():
    """With a 10-entry history a single remote reader never outvotes the
    holder's own accesses (P:L78 'If a local node have accessed it most time
    than there is no need of migration')."""
    B, S, T = 7, 22, 30 + 72
    script = [(0, B, T)] + [(300 + 200 * k, B, T) for k in range(5)] + [(1500 + 300 * k, S, T) for k in range(4)]
    o = Oracle(mig_cfg(mig_hist=10), script=script, debug=DBG_INVARIANTS)
    o.run(4000)
    st = o.stats()[0]
    assert st["mig_requests"] == 0 and o.loc(T)[0] == B
    # a fifth remote read makes S the majority (5 S > 5 B is false: tie keeps it) ...
    o2 = Oracle(mig_cfg(mig_hist=10), script=script + [(2800 + 300 * k, S, T) for k in range(2)],
                debug=DBG_INVARIANTS)
    o2.run(6000)
    # ... and the sixth (6 S vs 4 B in the last 10) moves it
    assert o2.stats()[0]["migrations"] == 1 and o2.loc(T)[0] == S


def _random_mig_cfgs(n, seed):
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        out.append(W.make(
            mesh_w=rng.randint(2, 7), mesh_h=rng.randint(2, 7), mode=W.MODE_LSPD,
            l2_sets=rng.choice([1, 2, 4]), l2_ways=rng.choice([1, 2, 3]), lam=rng.choice([0.1, 0.3, 0.7, 1.0]),
            p_priv=rng.choice([0, 0.2, 0.5]), sendq_cap=512, mig_hist=rng.choice([1, 2, 3, 5, 10, 16]),
            seed=rng.randint(1, 10 ** 6), tags_per_node=rng.choice([3, 4, 8]), priv_tags=1,
            mem_lat=rng.choice([1, 3, 10]), nfl_b2=rng.choice([1, 3, 8, 9, 16]), l2_hit_lat=rng.choice([0, 1, 2]),
            dir_mode=rng.choice([0, 0, 1]), dir_node=0, l1_sets=rng.choice([0, 0, 1, 2]), l1_ways=1,
            prio=rng.choice([0, 1])))
    return out


@pytest.mark.parametrize("k,cfg", list(enumerate(_random_mig_cfgs(24, 7))))
def test_migration_invariants_and_conservation(k, cfg):
    """Every cycle: one valid copy per block outside the sources still
    serving a block in transit, holder NONE => pend 0; after a drain: every
    access completed, the directory names each block's unique holder with no
    migration in transit, every granted migration delivered, installed,
    registered and invalidated, every redirection received, requests made =
    received (Table II pattern)."""
    o = Oracle(cfg, debug=DBG_INVARIANTS)
    o.run(3000)
    used, drained = o.drain(200000)
    st = o.stats()[0]
    assert drained and o.directory_quiescent_ok()
    assert st["accesses"] == st["completed"]
    assert st["migrations"] == st["mig_installs"] == st["dir_updates"] == st["invalidations"]
    assert st["mig_requests"] >= st["migrations"] + st["mig_nacks"]
    assert st["redirections"] == st["rr_received"]
    assert st["requests_made"] == st["requests_received"]
    assert st["evs_sent"] == st["evs_received"]


def test_migration_off_is_the_base_model():
    """mig_hist = 0 leaves every counter, histogram and the hash unchanged
    whatever nfl_b2 says, and never migrates."""
    a = Oracle(W.c1b(seed=4))
    b = Oracle(W.c1b(seed=4, nfl_b2=3))
    a.run(3000)
    b.run(3000)
    assert a.stats() == b.stats() and a.state_hash() == b.state_hash()
    assert a.stats()[0]["mig_requests"] == 0
