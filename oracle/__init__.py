"""CPU oracle of the bufferless-NoC + LSPD-L2 simulation (arXiv 1508.03235).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1508_03235_b200``) never imports it, and it
never imports the product path: the two share no code.  The C source
(``noc_oracle.c``) follows PAPER.md's serial loop and the readings
listed in DESIGN.md section 3; every function there cites its passage.

This module is argument marshalling for ``liboracle.so`` (ctypes) plus a
``build()`` that compiles it with gcc.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "noc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

COUNTER_NAMES = (
    "generated", "packets_enqueued", "injected", "ejected", "hops", "deflections",
    "probes_delivered", "accesses", "completed", "l2_hits", "l2_misses",
    "dir_searches", "requests_made", "requests_received", "replies_sent",
    "replies_received", "traps_sent", "traps_received", "mem_requests",
    "installs", "evictions", "evs_sent", "evs_received",
)
KIND_NAMES = ("probe", "da", "dr", "ndr", "rq", "ra", "trap", "ev")
L1_COUNTER_NAMES = ("l1_hits", "l1_misses", "wb_sent", "wb_received")   # NEXT-f1 (R42)
MIG_COUNTER_NAMES = ("mig_requests", "mig_nacks", "migrations", "mig_installs",
                     "dir_updates", "invalidations", "redirections", "rr_received")   # NEXT-f2
MEM_COUNTER_NAMES = ("mem_fills_sent", "mem_fills_received", "mem_wbs_sent", "mem_wb_flits")   # memory nodes (R55)

MODE_UR, MODE_LSPD = 0, 1
PRIO_DEFLECT, PRIO_OLDEST = 0, 1
DBG_REVERSE, DBG_INVARIANTS = 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "noc_oracle.h"))):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Event(C.Structure):
    _fields_ = [("cycle", C.c_uint64), ("node", C.c_uint32), ("value", C.c_uint32)]


class _Config(C.Structure):
    _fields_ = [
        ("mesh_w", C.c_uint32), ("mesh_h", C.c_uint32), ("mode", C.c_uint32), ("prio", C.c_uint32),
        ("l2_sets", C.c_uint32), ("l2_ways", C.c_uint32), ("tags_per_node", C.c_uint32),
        ("priv_tags", C.c_uint32), ("thr_inj", C.c_uint32), ("thr_priv", C.c_uint32),
        ("l2_hit_lat", C.c_uint32), ("mem_lat", C.c_uint32), ("nfl_ra", C.c_uint32),
        ("sendq_cap", C.c_uint32), ("hist_bins", C.c_uint32), ("seed", C.c_uint64),
        ("script", C.POINTER(_Event)), ("n_script", C.c_uint64), ("route", C.c_uint32),
        ("dir_mode", C.c_uint32), ("dir_node", C.c_uint32),
        ("l1_sets", C.c_uint32), ("l1_ways", C.c_uint32), ("l1_miss_lat", C.c_uint32),
        ("inject_mode", C.c_uint32), ("age_base", C.c_uint32),
        ("mig_hist", C.c_uint32), ("nfl_b2", C.c_uint32),
        ("mem_mode", C.c_uint32), ("mem_ctrls", C.c_uint32), ("hub_sendq_cap", C.c_uint32),
    ]


class _Counters(C.Structure):
    _fields_ = [("cycle", C.c_int64)] + [(n, C.c_int64) for n in COUNTER_NAMES] + [
        ("drops", C.c_int64 * 8)] + [(n, C.c_int64) for n in L1_COUNTER_NAMES + MIG_COUNTER_NAMES + MEM_COUNTER_NAMES]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.orc_create.argtypes = [C.POINTER(_Config), C.POINTER(C.c_void_p)]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_set_debug.argtypes = [C.c_void_p, C.c_int]
        L.orc_run.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_drain.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        L.orc_push_script.argtypes = [C.c_void_p, C.POINTER(_Event), C.c_uint64]
        L.orc_stats.argtypes = [C.c_void_p, C.POINTER(_Counters), C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_uint32]
        L.orc_state_hash.argtypes = [C.c_void_p]
        L.orc_state_hash.restype = C.c_uint64
        L.orc_last_error.restype = C.c_char_p
        L.orc_philox.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_arbitrate.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                    C.POINTER(C.c_uint64)]
        L.orc_arbitrate_ex.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                       C.POINTER(C.c_uint64)]
        L.orc_links_occupied.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_links_occupied.restype = C.c_int64
        L.orc_fifo_packets.argtypes = [C.c_void_p]
        L.orc_fifo_packets.restype = C.c_int64
        L.orc_cores_busy.argtypes = [C.c_void_p]
        L.orc_cores_busy.restype = C.c_int64
        L.orc_check_directory_quiescent.argtypes = [C.c_void_p]
        L.orc_core.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_l2_line.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_uint64)]
        L.orc_loc.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_link.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_fifo.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64)]
        L.orc_l1_line.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_script_used.argtypes = [C.c_void_p, C.c_uint32]
        L.orc_script_used.restype = C.c_int64
        L.orc_gen.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_poke.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]
        L.orc_l2_mig.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_loc_mig.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_mig_target.argtypes = [C.POINTER(C.c_uint32), C.c_uint32, C.c_uint32]
        L.orc_l2_hist.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
        L.orc_migrx.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.orc_mig_target.restype = C.c_uint32
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("oracle error %d: %s" % (code, msg))
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())
    return rc


def philox(key, ctr):
    """Philox4x32-10 of the oracle: key = (k0, k1), ctr = 4 u32 words."""
    c = (C.c_uint32 * 4)(*ctr)
    o = (C.c_uint32 * 4)()
    lib().orc_philox(key[0] & 0xFFFFFFFF, key[1] & 0xFFFFFFFF, c, o)
    return tuple(o)


def arbitrate(mesh_w, mesh_h, node, prio, flits, route=0):
    """One router decision.  flits = [(dst, src, age, inj), ...] or
    [(dst, src, age, inj, fid, kind, payload), ...] (the last three break ties
    between flits one node injected in the same cycle, R53).
    Returns ([port...], [age_after...]); port 0..3 = N,S,E,W, 4 = eject.
    route: 0 = PMDR (R3, R5), 1 = strict XY with N,E,S,W deflection (NEXT-f4)."""
    nf = len(flits)
    k = 7 if nf and len(flits[0]) == 7 else 4
    arr = (C.c_uint64 * (k * max(nf, 1)))()
    for i, f in enumerate(flits):
        for j in range(k):
            arr[k * i + j] = f[j]
    ports = (C.c_int * 5)()
    ages = (C.c_uint64 * 5)()
    rc = lib().orc_arbitrate_ex(mesh_w, mesh_h, node, prio, route, nf, k, arr, ports, ages)
    if rc != 0:
        raise ValueError("more flits than router degree")
    return list(ports[:nf]), list(ages[:nf])


class Oracle:
    """One oracle simulation.  cfg: dict with the keys of workloads.py."""

    def __init__(self, cfg: dict, script=None, debug: int = 0):
        L = lib()
        self.cfg = dict(cfg)
        c = _Config()
        for name, _ in _Config._fields_:
            if name in ("script", "n_script"):
                continue
            setattr(c, name, int(cfg[name]))
        self._events = None
        if script:
            ev = (_Event * len(script))()
            for i, (cy, node, val) in enumerate(script):
                ev[i].cycle, ev[i].node, ev[i].value = cy, node, val
            self._events = ev
            c.script = C.cast(ev, C.POINTER(_Event))
            c.n_script = len(script)
        h = C.c_void_p()
        _check(L.orc_create(C.byref(c), C.byref(h)))
        self._h = h
        self.nbins = int(cfg["hist_bins"])
        if debug:
            L.orc_set_debug(self._h, debug)

    def close(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    __del__ = close

    def run(self, n_cycles: int):
        _check(lib().orc_run(self._h, int(n_cycles)))

    def push_script(self, events):
        """Append scripted events [(cycle, node, value), ...] (R57)."""
        events = list(events)
        ev = (_Event * max(len(events), 1))()
        for i, (cy, node, val) in enumerate(events):
            ev[i].cycle, ev[i].node, ev[i].value = cy, node, val
        _check(lib().orc_push_script(self._h, ev, len(events)))

    def drain(self, max_cycles: int):
        used = C.c_uint64()
        dr = C.c_int()
        _check(lib().orc_drain(self._h, int(max_cycles), C.byref(used), C.byref(dr)))
        return int(used.value), bool(dr.value)

    def stats(self):
        """Returns (counters dict, hist_lat, hist_defl, hist_acc)."""
        cnt = _Counters()
        nb = self.nbins
        hl, hd, ha = (C.c_uint64 * nb)(), (C.c_uint64 * nb)(), (C.c_uint64 * nb)()
        _check(lib().orc_stats(self._h, C.byref(cnt), hl, hd, ha, nb))
        d = {"cycle": cnt.cycle}
        for n in COUNTER_NAMES:
            d[n] = getattr(cnt, n)
        for i, k in enumerate(KIND_NAMES):
            d["drops_" + k] = cnt.drops[i]
        for n in L1_COUNTER_NAMES + MIG_COUNTER_NAMES + MEM_COUNTER_NAMES:
            d[n] = getattr(cnt, n)
        return d, list(hl), list(hd), list(ha)

    def state_hash(self) -> int:
        return int(lib().orc_state_hash(self._h))

    # peeks -------------------------------------------------------------
    def links_occupied(self):
        a = C.c_int64()
        k = lib().orc_links_occupied(self._h, C.byref(a))
        return int(k), int(a.value)

    def fifo_packets(self):
        return int(lib().orc_fifo_packets(self._h))

    def cores_busy(self):
        return int(lib().orc_cores_busy(self._h))

    def directory_quiescent_ok(self):
        return lib().orc_check_directory_quiescent(self._h) == 0

    def core(self, n):
        o = (C.c_uint64 * 6)()
        _check(lib().orc_core(self._h, n, o))
        return dict(zip(("mode", "ready", "tag", "install", "start", "rx"), o))

    def l2_line(self, n, s, w):
        o = (C.c_uint64 * 3)()
        _check(lib().orc_l2_line(self._h, n, s, w, o))
        return tuple(o)

    def loc(self, T):
        o = (C.c_uint64 * 2)()
        _check(lib().orc_loc(self._h, T, o))
        return tuple(o)

    def link(self, n, d):
        """Input slot d of node n for the next cycle: None or a dict of the flit."""
        o = (C.c_uint64 * 8)()
        _check(lib().orc_link(self._h, n, d, o))
        if not o[0]:
            return None
        return dict(zip(("dst", "src", "kind", "fid", "payload", "age", "inj"), o[1:]))

    def fifo(self, n):
        """(next-flit index, [packet (kind, dst, payload, nfl) from the head ...])."""
        ctl = (C.c_uint64 * 2)()
        pkt = (C.c_uint64 * 4)()
        _check(lib().orc_fifo(self._h, n, 0xFFFFFFFF, ctl, pkt))
        out = []
        for k in range(int(ctl[0])):
            _check(lib().orc_fifo(self._h, n, k, ctl, pkt))
            out.append(tuple(int(x) for x in pkt))
        return int(ctl[1]), out

    def l1_line(self, n, s, w):
        o = (C.c_uint64 * 4)()
        _check(lib().orc_l1_line(self._h, n, s, w, o))
        return tuple(o)

    def script_used(self, n):
        return int(lib().orc_script_used(self._h, n))

    def gen(self, n, t):
        """The simulation's generator call for (node, cycle): (fired, dst or tag)."""
        o = (C.c_uint64 * 2)()
        _check(lib().orc_gen(self._h, n, t, o))
        return bool(o[0]), int(o[1])

    def poke(self, field, n=0, i=0, j=0, value=1):
        """Test-only single-field mutation (fields listed at orc_poke)."""
        _check(lib().orc_poke(self._h, field, n, i, j, value & 0xFFFFFFFFFFFFFFFF))

    def l2_mig(self, n, s_, w):
        """NEXT-f2: (mstate, mtarget, hcount) of L2 line (n, set, way); mstate 0 NORMAL,
        1 MIGREQ, 2 MIGSENT, 3 FWD (forwarding ghost)."""
        o = (C.c_uint64 * 3)()
        _check(lib().orc_l2_mig(self._h, n, s_, w, o))
        return tuple(int(x) for x in o)

    def l2_hist(self, n, s_, w):
        """NEXT-f2: accessor history of L2 line (n, set, way), oldest first."""
        o = (C.c_uint32 * 16)()
        k = lib().orc_l2_hist(self._h, n, s_, w, o)
        return list(o[:max(k, 0)])

    def migrx(self, n, k):
        o = (C.c_uint64 * 3)()
        _check(lib().orc_migrx(self._h, n, k, o))
        return tuple(int(x) for x in o)

    def loc_mig(self, T):
        o = (C.c_uint64 * 2)()
        _check(lib().orc_loc_mig(self._h, T, o))
        return tuple(int(x) for x in o)


def mig_target(history, holder):
    """NEXT-f2 migration decision (R46) on an accessor history (oldest first):
    the target node or None."""
    arr = (C.c_uint32 * max(1, len(history)))(*history)
    r = lib().orc_mig_target(arr, len(history), holder)
    return None if r == 0xFFFFFFFF else int(r)
