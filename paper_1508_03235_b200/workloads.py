"""Seeded synthetic workload definitions (the "input generator" module).

Shared by the CUDA path, the oracle tests and bench.py.  It holds NONE of the
method's arithmetic: it only states the configurations C1a..C5 of DESIGN.md
section 5 as plain integer dictionaries, converts a
rate p in [0, 1] into the integer threshold floor(p * 2^32) that both sides
compare Philox draws against (reading R25), and builds seeded script event
lists for scripted tests.
"""
from __future__ import annotations

import random
from fractions import Fraction

MODE_UR, MODE_LSPD = 0, 1
PRIO_DEFLECT, PRIO_OLDEST = 0, 1
ROUTE_PMDR, ROUTE_XY = 0, 1   # NEXT-f4: strict XY + N,E,S,W deflection
DIR_DISTRIBUTED, DIR_CENTRAL = 0, 1   # NEXT-f3: one node holds the whole directory
MEM_OFFMESH, MEM_HOME, MEM_CTRLS = 0, 1, 2   # memory placement (R54): off-mesh, at the home node, controller nodes


def thr(p) -> int:
    """floor(p * 2^32), clamped to 2^32 - 1 (exact, via Fraction)."""
    v = int(Fraction(str(p)) * (1 << 32))
    return max(0, min(v, (1 << 32) - 1))


BASE = dict(
    mesh_w=4, mesh_h=4, mode=MODE_UR, prio=PRIO_DEFLECT,
    l2_sets=4, l2_ways=2, l2_line_bytes=32,
    tags_per_node=128, priv_tags=96,
    thr_inj=thr(0.1), thr_priv=thr(0.5),
    l2_hit_lat=1, mem_lat=100, nfl_ra=4,
    sendq_cap=16, hist_bins=4096, seed=1, route=0, dir_mode=0, dir_node=0,
    l1_sets=0, l1_ways=2, l1_miss_lat=2, inject_mode=0, age_base=0, band_streams=0,
    mig_hist=0, nfl_b2=16, mem_mode=0, mem_ctrls=4, hub_sendq_cap=0,
)


def make(**kw) -> dict:
    """A config dict: BASE overridden by kw (lam / p_priv accepted as rates)."""
    cfg = dict(BASE)
    if "lam" in kw:
        cfg["thr_inj"] = thr(kw.pop("lam"))
    if "p_priv" in kw:
        cfg["thr_priv"] = thr(kw.pop("p_priv"))
    for k in kw:
        if k not in cfg:
            raise KeyError("unknown config key %r" % k)
    cfg.update(kw)
    return cfg


def c1a(seed=1, **kw):
    """4x4 uniform random, 0.1 flits/node/cycle (BASELINE configs[0])."""
    kw.setdefault("lam", 0.1)
    return make(mesh_w=4, mesh_h=4, mode=MODE_UR, sendq_cap=16, seed=seed, **kw)


def c1b(seed=1, **kw):
    """4x4 LSPD, small L2 (4 sets x 2 ways x 32 B), p_priv 0.5, lambda 0.1."""
    kw.setdefault("lam", 0.1)
    kw.setdefault("p_priv", 0.5)
    return make(mesh_w=4, mesh_h=4, mode=MODE_LSPD, l2_sets=4, l2_ways=2, sendq_cap=32,
                seed=seed, **kw)


def lspd(w, h, seed=1, lam=0.05, **kw):
    """LSPD with the Table III rows 3-4 slice (32 sets x 2 ways x 32 B) by default."""
    kw.setdefault("p_priv", 0.5)
    kw.setdefault("sendq_cap", 32)
    kw.setdefault("l2_sets", 32)
    kw.setdefault("l2_ways", 2)
    return make(mesh_w=w, mesh_h=h, mode=MODE_LSPD, lam=lam, seed=seed, **kw)


def c2(seed=1, **kw):
    """64x64 LSPD (BASELINE configs[1])."""
    return lspd(64, 64, seed=seed, **kw)


def c3(seed=1, **kw):
    """208x208 LSPD, the paper's largest mesh (BASELINE configs[2])."""
    return lspd(208, 208, seed=seed, **kw)


def c4(lam, mode=MODE_UR, seed=1, **kw):
    """208x208 injection sweep point (BASELINE configs[3])."""
    if mode == MODE_UR:
        return make(mesh_w=208, mesh_h=208, mode=MODE_UR, lam=lam, sendq_cap=16, seed=seed, **kw)
    return lspd(208, 208, seed=seed, lam=lam, **kw)


def c5(mode=MODE_LSPD, lam=0.05, seed=1, **kw):
    """1024x1024 (BASELINE configs[4])."""
    if mode == MODE_UR:
        return make(mesh_w=1024, mesh_h=1024, mode=MODE_UR, lam=lam, sendq_cap=16, seed=seed, **kw)
    return lspd(1024, 1024, seed=seed, lam=lam, **kw)


NAMED = {
    "c1a": c1a, "c1b": c1b, "c2": c2, "c3": c3,
}

# cycles per config: (timing, oracle parity) -- SURVEY 8(d.1)
CYCLES = {"c1a": (10_000, 10_000), "c1b": (10_000, 10_000), "c2": (100_000, 100_000),
          "c3": (100_000, 100_000), "c4": (20_000, 5_000), "c5": (10_000, 1_000)}


def random_script(cfg: dict, n_events: int, max_cycle: int, seed: int):
    """Seeded script events (cycle, node, value) valid for cfg's mode."""
    rng = random.Random(seed)
    N = cfg["mesh_w"] * cfg["mesh_h"]
    ev = []
    for _ in range(n_events):
        node = rng.randrange(N)
        cyc = rng.randrange(max_cycle)
        if cfg["mode"] == MODE_UR:
            v = rng.randrange(N - 1)
            v += v >= node
        else:
            v = rng.randrange(cfg["tags_per_node"] * N)
        ev.append((cyc, node, v))
    return ev


def _trace_records(path: str, cfg: dict):
    N = cfg["mesh_w"] * cfg["mesh_h"]
    space = cfg["tags_per_node"] * N
    line_bytes = max(1, int(cfg.get("l2_line_bytes", 32)))
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            body = line.split("#", 1)[0].strip()
            if not body:
                continue
            tok = body.split()
            if len(tok) not in (2, 3) or (len(tok) == 3 and tok[2] not in ("R", "W")):
                raise ValueError("%s:%d: expected '<node> <hex_address> [R|W]'" % (path, ln))
            node = int(tok[0], 10)
            addr = int(tok[1], 16)
            if not 0 <= node < N or addr < 0:
                raise ValueError("%s:%d: node or address out of range" % (path, ln))
            yield (0, node, (addr // line_bytes) % space)


def load_trace(path: str, cfg: dict):
    """Trace replay input (grammar of SPEC S:L533-534):
    one record per line, `<node_linear_id> <hex_address> [R|W]`, `#` comments
    and blank lines ignored.  Each node's records become its address stream in
    file order: script events (0, node, tag) with tag = (address // line bytes)
    mod TPN*N (reading R41), consumed one per generation opportunity in place
    of the Philox draw (DESIGN 3.3; the paper feeds a trace per cycle, P:L233,
    L276).  R/W is accepted and ignored (the model has no dirty state).
    Returns the event list; raises ValueError on a malformed line."""
    return list(_trace_records(path, cfg))


def trace_chunks(path: str, cfg: dict, records: int):
    """The same trace read lazily in chunks of `records` records, for the
    streamed replay (NocSim.push_script, DESIGN R57): only one chunk is held
    in host memory, and pushed chunks are merged on the device as they are
    needed.  Every record has cycle 0, so each node's queue stays in file order."""
    chunk = []
    for r in _trace_records(path, cfg):
        chunk.append(r)
        if len(chunk) == records:
            yield chunk
            chunk = []
    if chunk:
        yield chunk
