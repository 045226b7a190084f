"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact on every counter, the three histograms and the canonical state
hash (the model is integer and deterministic, DESIGN 3).
All tests need a B200 (sm_100a).
"""
import collections
import os
import random

import pytest

import paper_1508_03235_b200 as nb
from paper_1508_03235_b200 import workloads as W
from oracle import Oracle

pytestmark = pytest.mark.gpu

ENGINES = [nb.ENGINE_STEP, nb.ENGINE_PERSIST, nb.ENGINE_TILED, nb.ENGINE_TILED4]
TILED_ENGINES = [nb.ENGINE_TILED, nb.ENGINE_TILED4]


def both(cfg, cycles, engine=nb.ENGINE_AUTO, script=None, drain=None, split=None):
    g = nb.NocSim(cfg, script=script, engine=engine)
    o = Oracle(cfg, script=script)
    for k in (split or [cycles]):
        g.run(k)
        o.run(k)
    if drain is not None:
        assert g.drain(drain) == o.drain(drain)
    return g, o


def assert_same(g, o):
    gs, os_ = g.stats(), o.stats()
    assert gs[0] == os_[0], {k: (gs[0][k], os_[0][k]) for k in gs[0] if gs[0][k] != os_[0][k]}
    for i, name in ((1, "lat"), (2, "defl"), (3, "acc")):
        if gs[i] != os_[i]:
            diff = {b: (x, y) for b, (x, y) in enumerate(zip(gs[i], os_[i])) if x != y}
            raise AssertionError("hist %s differs at %s" % (name, dict(list(diff.items())[:10])))
    assert g.state_hash() == o.state_hash()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1a_uniform_random_4x4(engine, seed):
    """BASELINE configs[0]: 4x4, 0.1 flits/node/cycle, 10k cycles."""
    g, o = both(W.c1a(seed=seed), 10_000, engine)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1b_lspd_4x4(engine, seed):
    g, o = both(W.c1b(seed=seed), 10_000, engine)
    assert_same(g, o)
    st = g.stats()[0]
    assert st["replies_sent"] > 0 and st["traps_sent"] > 0 and st["evictions"] > 0


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("prio", [W.PRIO_DEFLECT, W.PRIO_OLDEST])
def test_saturated_ur_with_drops(engine, prio):
    """Saturated 16x16 UR (deflection regime, FIFO overflow drops)."""
    cfg = W.make(mesh_w=16, mesh_h=16, mode=W.MODE_UR, lam=0.5, prio=prio, sendq_cap=4)
    g, o = both(cfg, 3000, engine)
    assert_same(g, o)
    assert g.stats()[0]["drops_probe"] > 0


@pytest.mark.parametrize("engine", ENGINES)
def test_c2_64x64_lspd(engine):
    """BASELINE configs[1] geometry (64x64 LSPD), shortened run (oracle time)."""
    g, o = both(W.c2(), 6000, engine)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
def test_c3_208x208_lspd_bench_config(engine):
    """The bench workload (208x208 LSPD, seed 1) in the launch configuration
    bench.py times, oracle-checked over a window the oracle finishes in
    seconds."""
    g, o = both(W.c3(), 1500, engine)
    assert_same(g, o)


def test_c4_saturated_208():
    cfg = W.c4(0.3)
    g, o = both(cfg, 400, nb.ENGINE_PERSIST)
    assert_same(g, o)


@pytest.mark.parametrize("cfg", [
    W.make(mesh_w=2, mesh_h=2, mode=W.MODE_UR, lam=0.7),
    W.make(mesh_w=2, mesh_h=37, mode=W.MODE_UR, lam=0.3, prio=W.PRIO_OLDEST),
    W.make(mesh_w=53, mesh_h=3, mode=W.MODE_LSPD, lam=0.2, l2_sets=3, l2_ways=3, sendq_cap=32),
    W.make(mesh_w=5, mesh_h=7, mode=W.MODE_LSPD, lam=0.5, l2_hit_lat=0, nfl_ra=1, sendq_cap=32),
    W.make(mesh_w=6, mesh_h=6, mode=W.MODE_LSPD, lam=0.3, nfl_ra=8, sendq_cap=4, hist_bins=1),
    W.make(mesh_w=9, mesh_h=4, mode=W.MODE_LSPD, lam=1.0, l2_sets=1, l2_ways=16, sendq_cap=64,
           tags_per_node=4, priv_tags=1, mem_lat=1),
    W.make(mesh_w=300, mesh_h=7, mode=W.MODE_LSPD, lam=0.1, hist_bins=64, seed=2 ** 40 + 7),
], ids=["2x2", "2x37-oldest", "53x3", "hitlat0-nfl1", "nfl8-q4-nb1", "1set16way", "300x7-bigseed"])
@pytest.mark.parametrize("engine", ENGINES)
def test_edge_configurations(cfg, engine):
    g, o = both(cfg, 2500, engine)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
def test_split_runs_and_drain(engine):
    """run(a); run(b) == run(a+b) and drain (R30) on both sides."""
    cfg = W.make(mesh_w=12, mesh_h=10, mode=W.MODE_LSPD, lam=0.2, sendq_cap=32, l2_sets=4)
    g, o = both(cfg, None, engine, split=[1, 700, 1299], drain=100000)
    assert_same(g, o)
    st = g.stats()[0]
    assert st["requests_made"] == st["requests_received"] and st["accesses"] == st["completed"]
    g.run(500)
    o.run(500)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
def test_drain_cap_and_already_quiescent(engine):
    cfg = W.make(mesh_w=8, mesh_h=8, mode=W.MODE_UR, lam=0.5)
    g, o = both(cfg, 1000, engine)
    assert g.drain(3) == o.drain(3) == (3, False)
    assert_same(g, o)
    r = g.drain(10 ** 6)
    assert r == o.drain(10 ** 6) and r[1]
    assert g.drain(10) == o.drain(10) == (0, True)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
def test_scripted_events(engine):
    for cfg in (W.make(mesh_w=10, mesh_h=9, mode=W.MODE_UR, lam=0.05),
                W.make(mesh_w=10, mesh_h=9, mode=W.MODE_LSPD, lam=0.05, sendq_cap=32)):
        script = W.random_script(cfg, 3000, 2000, seed=5)
        g, o = both(cfg, 2500, engine, script=script)
        assert_same(g, o)


def test_engines_agree_on_hash():
    cfg = W.lspd(40, 33, lam=0.1, seed=9)
    hs = []
    for e in ENGINES:
        g = nb.NocSim(cfg, engine=e)
        g.run(3000)
        hs.append(g.state_hash())
    assert len(set(hs)) == 1


def test_zero_load_latency_208():
    """Closed form at the full bench mesh: lone flits take Manhattan hops."""
    rng = random.Random(3)
    w = h = 208
    n = w * h
    gap = w + h + 2
    pairs = []
    for _ in range(300):
        s = rng.randrange(n)
        d = rng.randrange(n - 1)
        pairs.append((s, d + (d >= s)))
    script = [(k * gap, s, d) for k, (s, d) in enumerate(pairs)]
    g = nb.NocSim(W.make(mesh_w=w, mesh_h=h, mode=W.MODE_UR, thr_inj=0), script=script)
    g.run(len(pairs) * gap)
    hl = g.stats()[1]
    want = collections.Counter(abs(s % w - d % w) + abs(s // w - d // w) for s, d in pairs)
    assert {b: c for b, c in enumerate(hl) if c} == dict(want)


def test_c3_long_run_properties():
    """Full-length properties at the bench size (any length): conservation
    after drain and the Table II equalities; no FIFO drops."""
    g = nb.NocSim(W.c3())
    g.run(20_000)
    used, drained = g.drain(100_000)
    st = g.stats()[0]
    assert drained
    assert st["injected"] == st["ejected"]
    assert st["requests_made"] == st["requests_received"]
    assert st["replies_sent"] == st["replies_received"]
    assert st["traps_sent"] == st["traps_received"]
    assert st["evs_sent"] == st["evs_received"]
    assert st["accesses"] == st["completed"]
    assert sum(v for k, v in st.items() if k.startswith("drops_")) == 0


def test_auto_engine_is_tiled_at_bench_size():
    g = nb.NocSim(W.c3())
    info = g.info()
    assert info["engine"] in TILED_ENGINES and info["grid"] <= 2 * info["sm_count"]


@pytest.mark.parametrize("engine", TILED_ENGINES)
@pytest.mark.parametrize("w,h", [(13, 11), (148, 2), (2, 300), (31, 29)])
def test_tiled_odd_tilings(w, h, engine):
    """Tilings with 1-wide tiles, single-row bands and ragged tile sizes."""
    cfg = W.make(mesh_w=w, mesh_h=h, mode=W.MODE_LSPD, lam=0.3, sendq_cap=32, l2_sets=4, mem_lat=20)
    g, o = both(cfg, 1500, engine)
    assert_same(g, o)
    cfg = W.make(mesh_w=w, mesh_h=h, mode=W.MODE_UR, lam=0.2)
    g, o = both(cfg, 1500, engine)
    assert_same(g, o)


@pytest.mark.parametrize("tiling", ["3x4", "13x1", "1x11"])
def test_small_mesh_forced_tilings(tiling, monkeypatch):
    """A mesh that fits one CTA runs as one tile (no cross-tile exchange);
    the NOCSIM_TILING hook still forces a multi-tile layout on it, which must
    give the same results (ragged, 1-wide and 1-tall tiles)."""
    cfg = W.make(mesh_w=13, mesh_h=11, mode=W.MODE_LSPD, lam=0.3, sendq_cap=32, l2_sets=4, mem_lat=20)
    g1 = nb.NocSim(cfg, engine=nb.ENGINE_TILED)
    assert g1.info()["grid"] == 1
    monkeypatch.setenv("NOCSIM_TILING", tiling)
    g, o = both(cfg, 1500, nb.ENGINE_TILED)
    a, b = (int(v) for v in tiling.split("x"))
    assert g.info()["grid"] == a * b
    assert_same(g, o)
    g1.run(1500)
    assert g1.state_hash() == o.state_hash()


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode", [W.MODE_UR, W.MODE_LSPD])
def test_launch_boundaries(engine, mode):
    """State carried across many short launches (links spilled / reloaded,
    deferred services finished) equals one long run and the oracle."""
    cfg = (W.make(mesh_w=16, mesh_h=16, mode=mode, lam=0.3) if mode == W.MODE_UR
           else W.lspd(24, 20, lam=0.2))
    g, o = both(cfg, None, engine, split=[1, 1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233])
    assert_same(g, o)
    g.drain(7)
    o.drain(7)
    g.run(100)
    o.run(100)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
def test_c3_drain_window(engine):
    """Drain (generation off) at the bench size, checked against the oracle
    mid-drain: multi-warp tiles exchange links through shared memory."""
    cfg = W.c3()
    g, o = both(cfg, 1200, engine)
    for k in (37, 200):
        assert g.drain(k) == o.drain(k)
        assert_same(g, o)


@pytest.mark.parametrize("engine", TILED_ENGINES + [nb.ENGINE_PERSIST])
@pytest.mark.parametrize("bands", [2, 3, 5, 8])
@pytest.mark.parametrize("mode", [W.MODE_UR, W.MODE_LSPD])
def test_virtual_bands_match_oracle(bands, mode, engine):
    """Row bands (the multi-GPU partition, DESIGN 8) simulated on one GPU:
    results identical to the oracle and to the unpartitioned run."""
    cfg = (W.make(mesh_w=18, mesh_h=16, mode=mode, lam=0.3) if mode == W.MODE_UR
           else W.lspd(22, 19, lam=0.2, mem_lat=30))
    script = W.random_script(cfg, 400, 900, seed=11)
    g = nb.NocSim(cfg, script=script, engine=engine, bands=bands)
    o = Oracle(cfg, script=script)
    for k in (1, 999, 600):
        g.run(k)
        o.run(k)
    assert_same(g, o)
    assert g.drain(50000) == o.drain(50000)
    assert_same(g, o)
    g.run(300)
    o.run(300)
    assert_same(g, o)


@pytest.mark.parametrize("bands", [2, 3, 4])
@pytest.mark.parametrize("mode", [W.MODE_UR, W.MODE_LSPD])
def test_virtual_ranks_band_streams(bands, mode):
    """"Virtual ranks" (band_streams): each band advanced by its own launches
    on its own stream with the multi-process launch sequence (refresh,
    cross-band barrier, launch, barrier; events instead of NCCL) -- the
    world_size > 1 host logic on one GPU -- bit-exact against the oracle,
    across many launch boundaries and a drain."""
    if mode == W.MODE_UR:
        cfg = W.make(mesh_w=40, mesh_h=37, mode=W.MODE_UR, lam=0.3, band_streams=1)
    else:
        cfg = W.lspd(40, 37, lam=0.2, band_streams=1)
    g = nb.NocSim(cfg, bands=bands, engine=nb.ENGINE_TILED)
    o = Oracle(cfg)
    for k in (1, 5, 250, 744, 1000):
        g.run(k)
        o.run(k)
    assert g.drain(20000) == o.drain(20000)
    g.run(300)
    o.run(300)
    assert_same(g, o)


def test_virtual_ranks_c3():
    """The bench mesh as 2 virtual ranks, in the bench's launch split."""
    cfg = W.c3(band_streams=1)
    g = nb.NocSim(cfg, bands=2, engine=nb.ENGINE_TILED)
    o = Oracle(cfg)
    for _ in range(2):
        g.run(500)
        o.run(500)
        assert_same(g, o)


def test_virtual_bands_c3():
    cfg = W.c3()
    g = nb.NocSim(cfg, bands=2)
    o = Oracle(cfg)
    g.run(1000)
    o.run(1000)
    assert_same(g, o)


@pytest.mark.parametrize("mode", [W.MODE_LSPD, W.MODE_UR])
def test_c5_1024x1024(mode):
    """BASELINE configs[4] on one GPU (1,048,576 nodes; AUTO picks PERSIST,
    more than 512 nodes per SM): 300 cycles bit-exact against the oracle,
    then the state after a drain window."""
    cfg = W.c5(mode=mode)
    g, o = both(cfg, 300)
    assert g.info()["engine"] == nb.ENGINE_PERSIST
    assert_same(g, o)
    assert g.drain(20) == o.drain(20)
    assert_same(g, o)


@pytest.mark.parametrize("bands", [2, 4, 8])
def test_c5_virtual_bands(bands):
    """BASELINE configs[4] partitioned into 1024/P-row bands (the 2/4/8-GPU
    decomposition, DESIGN 8) on one GPU: PERSIST bands, band-edge links written
    into the neighbour band's arrays, bit-exact against the oracle."""
    cfg = W.c5()
    g = nb.NocSim(cfg, bands=bands)
    assert g.info()["engine"] == nb.ENGINE_PERSIST
    o = Oracle(cfg)
    for k in (150, 150):
        g.run(k)
        o.run(k)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("cfg", [
    W.c1a(route=W.ROUTE_XY, lam=0.3),
    W.c1b(route=W.ROUTE_XY, seed=2),
    W.make(mesh_w=16, mesh_h=16, mode=W.MODE_UR, lam=0.4, route=W.ROUTE_XY, prio=W.PRIO_OLDEST),
    W.lspd(24, 20, lam=0.2, route=W.ROUTE_XY),
], ids=["c1a", "c1b", "ur16_oldest", "lspd24x20"])
def test_strict_xy_compat_mode(cfg, engine):
    """NEXT-f4: SPEC's strict-XY preference with N,E,S,W deflection scan, on
    every engine, bit-exact against the oracle (saturated UR exercises the
    deflection order)."""
    g, o = both(cfg, 3000, engine)
    assert_same(g, o)
    assert g.stats()[0]["deflections"] > 0


def test_strict_xy_c3_and_bands():
    cfg = W.c3(route=W.ROUTE_XY)
    g, o = both(cfg, 800)
    assert_same(g, o)
    g = nb.NocSim(W.lspd(22, 19, lam=0.3, route=W.ROUTE_XY), bands=3)
    o = Oracle(W.lspd(22, 19, lam=0.3, route=W.ROUTE_XY))
    g.run(1500)
    o.run(1500)
    assert_same(g, o)


@pytest.mark.parametrize("mode,lam", [(W.MODE_UR, 0.05), (W.MODE_UR, 0.5), (W.MODE_LSPD, 0.05),
                                      (W.MODE_LSPD, 0.5)])
def test_c4_sweep_endpoints(mode, lam):
    """BASELINE configs[3]: the ends of the 208x208 injection sweep (AUTO
    engine) bit-exact against the oracle."""
    g, o = both(W.c4(lam, mode=mode), 600)
    assert_same(g, o)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("cfg", [
    W.c1b(dir_mode=W.DIR_CENTRAL, dir_node=5, lam=0.05),
    W.lspd(24, 20, lam=0.02, dir_mode=W.DIR_CENTRAL, dir_node=10 * 24 + 12, sendq_cap=512),
], ids=["c1b", "lspd24x20"])
def test_centralized_directory(cfg, engine):
    """NEXT-f3: the paper's centralized location array (R40)
    at one node, on every engine, bit-exact against the oracle."""
    g, o = both(cfg, 4000, engine)
    assert_same(g, o)
    st = g.stats()[0]
    assert st["dir_searches"] > 0 and st["evs_received"] > 0
    # the directory node's FIFO holds up to one reply per requester (R19), so
    # sendq_cap >= N + 2 never overflows; a smaller one would poison the run
    # on both sides (R21, test_lspd_fifo_overflow_is_an_error_on_both_sides)
    assert sum(v for k, v in st.items() if k.startswith("drops_")) == 0


def test_centralized_directory_c3_and_bands():
    """C3 with the directory at the centre node (the hot spot the paper warns
    about), and the same across 4 virtual bands (the directory band
    receives every DA over band edges)."""
    cfg = W.c3(lam=0.002, dir_mode=W.DIR_CENTRAL, dir_node=104 * 208 + 104, sendq_cap=1024)
    g, o = both(cfg, 600)
    assert_same(g, o)
    cfg = W.lspd(22, 19, lam=0.02, dir_mode=W.DIR_CENTRAL, dir_node=9 * 22 + 11, sendq_cap=512)
    for engine in (nb.ENGINE_TILED, nb.ENGINE_PERSIST):
        g = nb.NocSim(cfg, bands=4, engine=engine)
        o = Oracle(cfg)
        g.run(2000)
        o.run(2000)
        assert_same(g, o)


def test_trace_replay_central_directory():
    """NEXT-f3 end to end: a trace file (SPEC grammar) replayed with the
    directory at one node, on every engine, against the oracle."""
    import os
    cfg = W.c1b(thr_inj=0, dir_mode=W.DIR_CENTRAL, dir_node=10)
    ev = W.load_trace(os.path.join(os.path.dirname(__file__), "golden", "trace_4x4.txt"), cfg)
    rng = random.Random(5)
    ev += [(rng.randrange(3000), rng.randrange(16), rng.randrange(128 * 16)) for _ in range(400)]
    for engine in ENGINES:
        g, o = both(cfg, 5000, engine, script=ev)
        assert_same(g, o)
        assert g.stats()[0]["accesses"] == len(ev)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("cfg", [
    W.c1b(l1_sets=2, l1_ways=2, l1_miss_lat=3, seed=3),
    W.lspd(24, 20, lam=0.2, l1_sets=4, l1_ways=2, l1_miss_lat=2),
    W.lspd(16, 16, lam=0.3, l1_sets=1, l1_ways=1, l1_miss_lat=1, l2_hit_lat=0, dir_mode=W.DIR_CENTRAL,
           dir_node=8 * 16 + 8, sendq_cap=128),
], ids=["c1b", "lspd24x20", "lspd16_direct_central"])
def test_private_l1(cfg, engine):
    """NEXT-f1: private write-through L1 with the miss countdown and victim
    writebacks (R42) on every engine, bit-exact against
    the oracle, then drained (every writeback delivered)."""
    g, o = both(cfg, 3000, engine, drain=200000)
    assert_same(g, o)
    st = g.stats()[0]
    assert st["l1_hits"] > 0 and st["l1_misses"] > 0 and st["wb_sent"] > 0
    assert st["wb_sent"] == st["wb_received"]


def test_private_l1_c3_table3_geometry():
    """C3 with Table III's 43k-core L1 (32 sets x 2 ways)."""
    cfg = W.c3(l1_sets=32, l1_ways=2, l1_miss_lat=2)
    g, o = both(cfg, 800)
    assert_same(g, o)
    g = nb.NocSim(W.lspd(22, 19, lam=0.3, l1_sets=2, l1_ways=2), bands=3)
    o = Oracle(W.lspd(22, 19, lam=0.3, l1_sets=2, l1_ways=2))
    g.run(1500)
    o.run(1500)
    assert_same(g, o)


@pytest.mark.parametrize("engine", [nb.ENGINE_STEP, nb.ENGINE_PERSIST, nb.ENGINE_TILED])
@pytest.mark.parametrize("cfg", [
    W.make(mesh_w=16, mesh_h=16, mode=W.MODE_UR, lam=0.4, inject_mode=1),
    W.lspd(24, 20, lam=0.3, inject_mode=1, l1_sets=2, l1_ways=2),
    W.c1b(inject_mode=1, route=W.ROUTE_XY),
], ids=["ur16_sat", "lspd24x20_l1", "c1b_xy"])
def test_inject_when_eject_frees_a_slot_gpu(cfg, engine):
    """NEXT-f4 injection mode (R43) on the engines with five flit lanes per
    router, bit-exact against the oracle."""
    g, o = both(cfg, 3000, engine)
    assert_same(g, o)


def test_inject_mode_c3_and_tiled4_rejected():
    g, o = both(W.c3(inject_mode=1), 600)
    assert_same(g, o)
    with pytest.raises(nb.NocSimError):
        nb.NocSim(W.c1b(inject_mode=1), engine=nb.ENGINE_TILED4)


@pytest.mark.parametrize("cfg,cycles", [
    (W.make(mesh_w=2048, mesh_h=1023, mode=W.MODE_UR, lam=0.02), 30),           # N = 2^21 - 2049: the node-id limit (R32)
    (W.make(mesh_w=2, mesh_h=2048, mode=W.MODE_LSPD, lam=0.2, sendq_cap=32, l2_sets=4), 600),
    (W.make(mesh_w=2048, mesh_h=2, mode=W.MODE_LSPD, lam=0.2, sendq_cap=32, l2_sets=4), 600),
], ids=["max-nodes-ur", "2x2048", "2048x2"])
def test_maximum_sizes(cfg, cycles):
    """The largest meshes the ABI accepts (R9, R32: sides up to 2048, N < 2^21):
    AUTO engine against the oracle."""
    g, o = both(cfg, cycles)
    assert_same(g, o)


MIG_CASES = {
    "c1b_mig1": W.c1b(mig_hist=1, seed=2),
    "lspd16_mig2_b2x3": W.lspd(16, 16, lam=0.3, mig_hist=2, nfl_b2=3, sendq_cap=128, l2_sets=4, tags_per_node=16,
                               priv_tags=8, mem_lat=20),
    "stress5x6": W.make(mesh_w=5, mesh_h=6, mode=W.MODE_LSPD, l2_sets=2, l2_ways=2, lam=0.7, p_priv=0.0,
                        sendq_cap=512, mig_hist=3, nfl_b2=16, tags_per_node=4, priv_tags=1, mem_lat=3, seed=9),
    "central_l1_mig": W.lspd(12, 10, lam=0.3, mig_hist=4, nfl_b2=16, dir_mode=W.DIR_CENTRAL, dir_node=55,
                             sendq_cap=256, l1_sets=2, l1_ways=1, tags_per_node=8, priv_tags=4, mem_lat=10),
}


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name", sorted(MIG_CASES))
def test_migration_and_redirection(name, engine):
    """NEXT-f2 (R44-R52): accessor histories, home-granted migrations of
    16-flit blocks, directory updates, invalidations, forwarding ghosts and
    redirections on every engine, bit-exact against the oracle, then drained
    (every migration completed)."""
    cfg = MIG_CASES[name]
    g, o = both(cfg, 3000, engine, drain=200000)
    assert_same(g, o)
    st = g.stats()[0]
    assert st["migrations"] > 0 and st["migrations"] == st["mig_installs"] == st["dir_updates"]
    g.run(700)
    o.run(700)
    assert_same(g, o)


def test_migration_c3_and_bands():
    """C3 with migration (1-entry histories: a remote reader outvotes the holder, 16-flit blocks) on the default
    engine, and a 22x19 mesh with migration over 3 virtual bands."""
    cfg = W.c3(mig_hist=1)
    g, o = both(cfg, 1500)
    assert_same(g, o)
    assert g.stats()[0]["migrations"] > 0
    cfg = W.lspd(22, 19, lam=0.3, mig_hist=3, tags_per_node=8, priv_tags=4, sendq_cap=256)
    for engine in (nb.ENGINE_TILED, nb.ENGINE_PERSIST):
        g = nb.NocSim(cfg, bands=3, engine=engine)
        o = Oracle(cfg)
        g.run(1500)
        o.run(1500)
        assert_same(g, o)


@pytest.mark.parametrize("engine", [nb.ENGINE_STEP, nb.ENGINE_PERSIST, nb.ENGINE_TILED])
@pytest.mark.parametrize("cfg", [
    W.make(mesh_w=16, mesh_h=16, mode=W.MODE_UR, lam=0.4, inject_mode=2),
    W.make(mesh_w=13, mesh_h=11, mode=W.MODE_UR, lam=0.2, inject_mode=2, prio=W.PRIO_OLDEST),
    W.lspd(24, 20, lam=0.3, inject_mode=2, l1_sets=2, l1_ways=2),
    W.c1b(inject_mode=2, route=W.ROUTE_XY),
    W.lspd(20, 18, lam=0.2, inject_mode=2, mig_hist=6, nfl_b2=16, sendq_cap=64),
], ids=["ur16_sat", "ur13x11_oldest", "lspd24x20_l1", "c1b_xy", "lspd20x18_mig"])
def test_fill_all_injection_gpu(cfg, engine):
    """NEXT-f4 fill-all injection (R53): several flits per node and cycle,
    ranking ties broken by (fid, kind, dst, payload) -- bit-exact against the
    oracle, with a drain."""
    g, o = both(cfg, 3000, engine, drain=200000)
    assert_same(g, o)


def test_fill_all_c3_bands_and_tiled4_rejected():
    g, o = both(W.c3(inject_mode=2), 800, split=[300, 499, 1])
    assert_same(g, o)
    cfg = W.lspd(40, 37, lam=0.3, inject_mode=2)
    g = nb.NocSim(cfg, bands=3, engine=nb.ENGINE_TILED)
    o = Oracle(cfg)
    for k in (7, 400, 993):
        g.run(k)
        o.run(k)
    assert_same(g, o)
    with pytest.raises(nb.NocSimError):
        nb.NocSim(W.c1b(inject_mode=2), engine=nb.ENGINE_TILED4)


MEM_CASES = {
    "ctrl8x8": W.lspd(8, 8, lam=0.1, mem_mode=W.MEM_CTRLS, mem_ctrls=4, sendq_cap=64, hub_sendq_cap=256,
                      l2_sets=4, seed=3, mem_lat=30),
    "ctrl16x12_l1_xy": W.lspd(16, 12, lam=0.2, mem_mode=W.MEM_CTRLS, mem_ctrls=7, sendq_cap=64,
                              hub_sendq_cap=1024, l2_sets=2, seed=5, mem_lat=20, l1_sets=2, l1_ways=2,
                              route=W.ROUTE_XY, nfl_b2=5),
    "home24x20": W.lspd(24, 20, lam=0.2, mem_mode=W.MEM_HOME, sendq_cap=64, l2_sets=2, seed=9, mem_lat=25,
                        nfl_b2=8),
    "central12x12": W.lspd(12, 12, lam=0.03, mem_mode=W.MEM_HOME, dir_mode=W.DIR_CENTRAL, dir_node=77,
                           sendq_cap=16, hub_sendq_cap=1024, l2_sets=2, seed=2, mem_lat=15, nfl_b2=4),
}


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name", sorted(MEM_CASES))
def test_memory_nodes_gpu(name, engine):
    """Memory on the mesh (R54-R56): controller nodes with B2 fills and
    writebacks, memory at the home / central directory node, hub FIFOs --
    bit-exact against the oracle on every engine, with a drain."""
    g, o = both(MEM_CASES[name], 2500, engine, split=[1, 999, 1500], drain=200000)
    assert_same(g, o)
    assert g.stats()[0]["mem_fills_received"] > 0


def test_memory_nodes_c3_and_bands():
    """C3 with memory at every home node (B2 fills and writebacks over the
    whole mesh), in the bench's launch split; a 40x37 mesh with 6 memory
    controllers and hub FIFOs as 3 and 5 virtual bands (the controllers of the
    top and bottom rows live in different bands).  A handful of controllers
    cannot serve C3: each ejects one flit per cycle, so its FIFO overflows."""
    cfg = W.c3(mem_mode=W.MEM_HOME, sendq_cap=32)
    g, o = both(cfg, 1200, split=[600, 600])
    assert_same(g, o)
    cfg = W.lspd(40, 37, lam=0.02, mem_mode=W.MEM_CTRLS, mem_ctrls=6, hub_sendq_cap=1024, sendq_cap=64)
    for bands in (3, 5):
        g = nb.NocSim(cfg, bands=bands, engine=nb.ENGINE_TILED)
        o = Oracle(cfg)
        for k in (7, 400, 993):
            g.run(k)
            o.run(k)
        assert_same(g, o)


def _pieces(script, bounds):
    out = [[] for _ in range(len(bounds) + 1)]
    for e in script:
        out[sum(1 for b in bounds if e[0] >= b)].append(e)
    return out


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("mode", [W.MODE_UR, W.MODE_LSPD])
def test_streamed_script_gpu(mode, engine):
    """NEXT-f3 streamed trace replay (R57): a script pushed in pieces (some
    before their events are due, merged before the run; some well ahead,
    merged after it while their copy overlapped the run; one late, after its
    events were due) -- bit-exact against the oracle fed the same pushes."""
    if mode == W.MODE_UR:
        cfg = W.make(mesh_w=24, mesh_h=20, mode=W.MODE_UR, thr_inj=0, sendq_cap=16)
    else:
        cfg = W.lspd(24, 20, thr_inj=0, sendq_cap=64, l2_sets=2, mem_lat=20)
    script = W.random_script(cfg, 6000, 3000, seed=33)
    parts = _pieces(script, [300, 900, 1000, 2200])
    g = nb.NocSim(cfg, script=parts[0], engine=engine)
    o = Oracle(cfg, script=parts[0])
    plan = [(parts[1], 250), (parts[2], 640), (parts[3], 150), ([], 300), (parts[4], 2000)]
    for piece, k in plan:
        g.push_script(piece)
        o.push_script(piece)
        g.run(k)
        o.run(k)
    assert g.drain(100000) == o.drain(100000)
    assert_same(g, o)


def test_streamed_script_bands_and_trace_chunks():
    """Pushed pieces on 3 virtual bands (each band keeps its nodes' events) and
    a trace file streamed in chunks, against the oracle."""
    cfg = W.lspd(40, 37, thr_inj=0, sendq_cap=64, l2_sets=4, mem_lat=30)
    script = W.random_script(cfg, 20000, 4000, seed=4)
    parts = _pieces(script, [1000, 2500])
    for bands, engine in ((3, nb.ENGINE_TILED), (2, nb.ENGINE_PERSIST)):
        g = nb.NocSim(cfg, script=parts[0], bands=bands, engine=engine)
        o = Oracle(cfg, script=parts[0])
        for piece, k in ((parts[1], 900), (parts[2], 1700), ([], 2000)):
            g.push_script(piece)
            o.push_script(piece)
            g.run(k)
            o.run(k)
        assert_same(g, o)
    cfg = W.c1b(thr_inj=0)
    path = os.path.join(os.path.dirname(__file__), "golden", "trace_4x4.txt")
    g = nb.NocSim(cfg)
    o = Oracle(cfg)
    for c in W.trace_chunks(path, cfg, 4):
        g.push_script(c)
        o.push_script(c)
    g.run(3000)
    o.run(3000)
    assert_same(g, o)


@pytest.mark.parametrize("cfg", [W.c2(), W.make(mesh_w=40, mesh_h=30, mode=W.MODE_UR, lam=0.2),
                                 W.lspd(31, 29, lam=0.2, l1_sets=2, l1_ways=2), W.c2(mem_mode=W.MEM_HOME)],
                         ids=["c2", "ur40x30", "lspd31x29_l1", "c2_memhome"])
def test_cluster_exchange(cfg, monkeypatch):
    """The opt-in cluster exchange of the TILED engine (NOCSIM_CLUSTER=1: the
    band as one thread-block cluster, DSMEM links, cluster barrier), across
    launch boundaries and a drain, bit-exact against the oracle."""
    monkeypatch.setenv("NOCSIM_CLUSTER", "1")
    g, o = both(cfg, 2600, nb.ENGINE_TILED, split=[1, 600, 1999], drain=100000)
    assert g.info()["cluster"] > 1
    assert_same(g, o)


@pytest.mark.parametrize("engine", [nb.ENGINE_PERSIST, nb.ENGINE_TILED])
def test_streamed_script_many_merges(engine):
    """120 pushed pieces, each merged right before its events fall due (the
    merge allocates, zeroes and fills count / offset buffers each time):
    regression for a pushed piece lost when a buffer's legacy-stream zeroing
    landed after the copy that filled it on the library's non-blocking stream.
    Bit-exact against the oracle."""
    cfg = W.lspd(16, 12, thr_inj=0, sendq_cap=64, l2_sets=2, mem_lat=20)
    script = W.random_script(cfg, 6000, 2400, seed=71)
    bounds = list(range(20, 2400, 20))
    parts = _pieces(script, bounds)
    g = nb.NocSim(cfg, script=parts[0], engine=engine)
    o = Oracle(cfg, script=parts[0])
    for piece in parts[1:]:
        g.push_script(piece)
        o.push_script(piece)
        g.run(20)
        o.run(20)
    g.run(400)
    o.run(400)
    assert o.stats()[0]["accesses"] > 3000
    assert_same(g, o)
