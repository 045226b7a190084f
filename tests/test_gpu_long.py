"""GPU parity over the windows the bench times, at the lengths SURVEY 8(d.1)
asks for, and the edge cases of the field widths (R32) and the bounded FIFO
(R21).  Bit-exact against the CPU oracle (DESIGN 3).

Oracle time on one host core: C3 12k cycles ~1 min, C2 100k ~35 s, each C4
point 5k ~20-70 s, C5 1k ~4 min.
"""
import pytest

import paper_1508_03235_b200 as nb
from paper_1508_03235_b200 import workloads as W
from oracle import Oracle, OracleError

pytestmark = pytest.mark.gpu


def assert_same(g, o, where=""):
    gs, os_ = g.stats(), o.stats()
    assert gs[0] == os_[0], (where, {k: (gs[0][k], os_[0][k]) for k in gs[0] if gs[0][k] != os_[0][k]})
    for i, name in ((1, "lat"), (2, "defl"), (3, "acc")):
        assert gs[i] == os_[i], (where, "histogram " + name)
    assert g.state_hash() == o.state_hash(), where


def test_c3_steady_state_in_bench_launch_split():
    """C3 (the bench workload) for 12,000 cycles on the default engine, in the
    2000-cycle launches bench.py times, compared after every launch: by then
    the L2 slices are full (tens of thousands of evictions, local and remote
    hits, traps), the steady state of the timed window (cycles 10k-50k)."""
    cfg = W.c3()
    g, o = nb.NocSim(cfg), Oracle(cfg)
    assert g.info()["engine"] in (nb.ENGINE_TILED, nb.ENGINE_TILED4)
    for k in range(6):
        g.run(2000)
        o.run(2000)
        assert_same(g, o, "after launch %d" % k)
    st = g.stats()[0]
    assert st["evictions"] > 50_000 and st["l2_hits"] > 30_000
    assert st["replies_sent"] > 0 and st["traps_sent"] > 0 and st["evs_received"] > 0


def test_c2_full_length():
    """BASELINE configs[1] (64x64 LSPD) for the full 100,000 cycles of
    SURVEY 8(d.1), compared every 20,000 cycles."""
    cfg = W.c2()
    g, o = nb.NocSim(cfg), Oracle(cfg)
    for k in range(5):
        g.run(20_000)
        o.run(20_000)
        assert_same(g, o, "after %d cycles" % (20_000 * (k + 1)))


@pytest.mark.parametrize("mode,lam", [(W.MODE_UR, 0.3), (W.MODE_LSPD, 0.5)])
def test_c4_sweep_points_5k(mode, lam):
    """BASELINE configs[3] sweep points at the 5,000 oracle cycles of
    SURVEY 8(d.1) (saturated UR with FIFO drops; self-throttled LSPD)."""
    cfg = W.c4(lam, mode=mode)
    g, o = nb.NocSim(cfg), Oracle(cfg)
    g.run(5000)
    o.run(5000)
    assert_same(g, o)


def test_c5_1k_cycles():
    """BASELINE configs[4] (1024x1024 LSPD) for the 1,000 oracle cycles of
    SURVEY 8(d.1), on the engine AUTO picks for one GPU."""
    cfg = W.c5()
    g, o = nb.NocSim(cfg), Oracle(cfg)
    for k in (400, 600):
        g.run(k)
        o.run(k)
    assert_same(g, o)


ENGINES = [nb.ENGINE_STEP, nb.ENGINE_PERSIST, nb.ENGINE_TILED, nb.ENGINE_TILED4]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("cfg", [
    W.make(mesh_w=12, mesh_h=9, mode=W.MODE_UR, lam=0.4, age_base=2040, sendq_cap=8),
    W.make(mesh_w=10, mesh_h=10, mode=W.MODE_UR, lam=0.4, age_base=4090, prio=W.PRIO_OLDEST, hist_bins=8192),
    W.lspd(14, 11, lam=0.3, age_base=30000, hist_bins=65536),
], ids=["ur-2040", "ur-oldest-4090", "lspd-30000"])
def test_ages_across_the_split_age_field(cfg, engine):
    """Flit ages >= 2048 (the GPU record splits the age over two words,
    common.cuh) at parity: the age_base test knob starts every injected flit
    at a high age (every age shifts equally, so the ranking is the paper's)."""
    g, o = nb.NocSim(cfg, engine=engine), Oracle(cfg)
    g.run(1500)
    o.run(1500)
    assert_same(g, o)
    hd = g.stats()[2]
    top = max(b for b, v in enumerate(hd) if v)
    assert top >= min(cfg["hist_bins"] - 1, 2048)


@pytest.mark.parametrize("engine", ENGINES)
def test_age_overflow_is_reported_on_both_sides(engine):
    """R32: a deflection past age 65535 is NOC_EOVERFLOW on the GPU and
    ORC_EOVERFLOW in the oracle, in the same run call; the handle is then
    poisoned."""
    cfg = W.make(mesh_w=8, mesh_h=8, mode=W.MODE_UR, lam=0.5, age_base=65530)
    g, o = nb.NocSim(cfg, engine=engine), Oracle(cfg)
    with pytest.raises(OracleError) as eo:
        o.run(500)
    assert eo.value.code == -5
    with pytest.raises(nb.NocSimError) as eg:
        g.run(500)
    assert eg.value.code == nb.NOC_EOVERFLOW
    with pytest.raises(nb.NocSimError):
        g.run(1)


@pytest.mark.parametrize("engine", ENGINES)
def test_lspd_fifo_overflow_is_an_error_on_both_sides(engine):
    """R21: in LSPD mode a full send FIFO would drop a protocol message and
    leave a core or directory entry waiting for ever, so both sides poison the
    run with an overflow error (a 6x6 mesh with 2-packet FIFOs and 8-flit
    replies overflows within 2,000 cycles)."""
    cfg = W.make(mesh_w=6, mesh_h=6, mode=W.MODE_LSPD, lam=0.3, nfl_ra=8, sendq_cap=2, hist_bins=1)
    g, o = nb.NocSim(cfg, engine=engine), Oracle(cfg)
    with pytest.raises(OracleError) as eo:
        o.run(2500)
    assert eo.value.code == -5
    with pytest.raises(nb.NocSimError) as eg:
        g.run(2500)
    assert eg.value.code == nb.NOC_EOVERFLOW
