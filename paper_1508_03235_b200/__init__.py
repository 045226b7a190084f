"""B200-native simulator of the bufferless-NoC + LSPD-L2 hot path of
Kumar & Sahu, arXiv 1508.03235.

This module is the thin Python binding of ``libnocsim.so`` (C-ABI declared in
``include/noc_sim.h``): argument marshalling only.  Every simulated cycle runs
in the library's CUDA kernels; if the library or a CUDA device is missing the
calls raise -- there is no CPU fallback.  Function names mirror the C-ABI.
"""
from __future__ import annotations

import ctypes as C
import os

from . import workloads  # noqa: F401  (seeded configs)

_HERE = os.path.dirname(os.path.abspath(__file__))
# NOCSIM_LIB selects another in-tree build of the same library (A/B timing
# of kernel variants, tools/); default: the one build() writes
LIB_PATH = os.environ.get("NOCSIM_LIB") or os.path.join(_HERE, "libnocsim.so")

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

NOC_OK, NOC_EINVAL, NOC_ENOMEM, NOC_ECUDA, NOC_ENCCL, NOC_EOVERFLOW, NOC_ESTATE = 0, -1, -2, -3, -4, -5, -6
ENGINE_AUTO, ENGINE_STEP, ENGINE_PERSIST, ENGINE_TILED, ENGINE_TILED4 = 0, 1, 2, 3, 4


class noc_sim_event(C.Structure):
    _fields_ = [("cycle", C.c_uint64), ("node", C.c_uint32), ("value", C.c_uint32)]


class noc_sim_config(C.Structure):
    _fields_ = [
        ("mesh_w", C.c_uint32), ("mesh_h", C.c_uint32), ("mode", C.c_uint32), ("prio", C.c_uint32),
        ("l2_sets", C.c_uint32), ("l2_ways", C.c_uint32), ("l2_line_bytes", C.c_uint32),
        ("tags_per_node", C.c_uint32), ("priv_tags", C.c_uint32),
        ("thr_inj", C.c_uint32), ("thr_priv", C.c_uint32),
        ("l2_hit_lat", C.c_uint32), ("mem_lat", C.c_uint32), ("nfl_ra", C.c_uint32),
        ("sendq_cap", C.c_uint32), ("hist_bins", C.c_uint32), ("seed", C.c_uint64),
        ("script", C.POINTER(noc_sim_event)), ("n_script", C.c_uint64),
        ("device", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
        ("engine", C.c_uint32), ("nccl_id", C.c_uint8 * 128), ("bands", C.c_uint32),
        ("route", C.c_uint32), ("dir_mode", C.c_uint32), ("dir_node", C.c_uint32),
        ("l1_sets", C.c_uint32), ("l1_ways", C.c_uint32), ("l1_miss_lat", C.c_uint32),
        ("inject_mode", C.c_uint32), ("age_base", C.c_uint32), ("band_streams", C.c_uint32),
        ("mig_hist", C.c_uint32), ("nfl_b2", C.c_uint32),
        ("mem_mode", C.c_uint32), ("mem_ctrls", C.c_uint32), ("hub_sendq_cap", C.c_uint32),
    ]


class noc_sim_counters(C.Structure):
    _fields_ = [("cycle", C.c_int64)] + [(n, C.c_int64) for n in COUNTER_NAMES] + [
        ("drops", C.c_int64 * 8)] + [(n, C.c_int64) for n in L1_COUNTER_NAMES + MIG_COUNTER_NAMES + MEM_COUNTER_NAMES]


class noc_sim_info(C.Structure):
    _fields_ = [
        ("engine", C.c_uint32), ("grid", C.c_uint32), ("block", C.c_uint32),
        ("nodes_local", C.c_uint32), ("row0", C.c_uint32), ("rows", C.c_uint32),
        ("device_bytes", C.c_uint64), ("loc_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint64), ("cycles_run", C.c_uint64),
        ("sm_count", C.c_int32), ("cluster", C.c_uint32), ("reserved", C.c_int32 * 6),
    ]


class NocSimError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("noc_sim error %d: %s" % (code, msg))
        self.code = code


_lib = None


def lib():
    """Load libnocsim.so (built by build.build()).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NocSimError(NOC_ECUDA, "libnocsim.so not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.noc_sim_abi_version.restype = C.c_uint32
        L.noc_sim_create.argtypes = [C.POINTER(noc_sim_config), C.POINTER(P)]
        L.noc_sim_run.argtypes = [P, C.c_uint64]
        L.noc_sim_run_timed.argtypes = [P, C.c_uint64, C.POINTER(C.c_double)]
        L.noc_sim_drain.argtypes = [P, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
        L.noc_sim_push_script.argtypes = [P, C.POINTER(noc_sim_event), C.c_uint64]
        L.noc_sim_band_rows.argtypes = [C.c_uint32, C.c_int32, C.c_int32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.noc_sim_stats.argtypes = [P, C.POINTER(noc_sim_counters), P, P, P, C.c_uint32]
        L.noc_sim_state_hash.argtypes = [P, C.POINTER(C.c_uint64)]
        L.noc_sim_get_info.argtypes = [P, C.POINTER(noc_sim_info)]
        L.noc_sim_destroy.argtypes = [P]
        L.noc_sim_last_error.restype = C.c_char_p
        L.noc_sim_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        if L.noc_sim_abi_version() != 6:   # include/noc_sim.h NOC_SIM_ABI_VERSION
            raise NocSimError(NOC_EINVAL, "ABI version mismatch")
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise NocSimError(rc, lib().noc_sim_last_error().decode())
    return rc


def make_config(cfg: dict, script=None, device: int = 0, engine: int = ENGINE_AUTO,
                world_size: int = 1, rank: int = 0, nccl_id: bytes = b"", bands: int = 0):
    """Marshal a workloads.py dict (+ script events) into noc_sim_config.
    Returns (config, keepalive)."""
    c = noc_sim_config()
    for name, _ in noc_sim_config._fields_:
        if name in cfg:
            setattr(c, name, int(cfg[name]))
    keep = None
    if script:
        ev = (noc_sim_event * len(script))()
        for i, (cy, node, val) in enumerate(script):
            ev[i].cycle, ev[i].node, ev[i].value = cy, node, val
        c.script = C.cast(ev, C.POINTER(noc_sim_event))
        c.n_script = len(script)
        keep = ev
    c.device, c.engine, c.world_size, c.rank, c.bands = device, engine, world_size, rank, bands
    for i, b in enumerate(nccl_id[:128]):
        c.nccl_id[i] = b
    return c, keep


def noc_sim_create(cfg: dict, script=None, device: int = 0, engine: int = ENGINE_AUTO,
                   world_size: int = 1, rank: int = 0, nccl_id: bytes = b"", bands: int = 0):
    c, _keep = make_config(cfg, script, device, engine, world_size, rank, nccl_id, bands)
    h = C.c_void_p()
    _check(lib().noc_sim_create(C.byref(c), C.byref(h)))
    return h


def noc_sim_run(h, n_cycles: int):
    _check(lib().noc_sim_run(h, int(n_cycles)))


def noc_sim_run_timed(h, n_cycles: int) -> float:
    ms = C.c_double()
    _check(lib().noc_sim_run_timed(h, int(n_cycles), C.byref(ms)))
    return float(ms.value)


def noc_sim_drain(h, max_cycles: int):
    used, dr = C.c_uint64(), C.c_int()
    _check(lib().noc_sim_drain(h, int(max_cycles), C.byref(used), C.byref(dr)))
    return int(used.value), bool(dr.value)


def noc_sim_stats(h, nbins: int):
    """Returns (counters dict, hist_lat, hist_defl, hist_acc)."""
    cnt = noc_sim_counters()
    hl, hd, ha = (C.c_uint64 * nbins)(), (C.c_uint64 * nbins)(), (C.c_uint64 * nbins)()
    _check(lib().noc_sim_stats(h, C.byref(cnt), hl, hd, ha, nbins))
    d = {"cycle": cnt.cycle}
    for n in COUNTER_NAMES:
        d[n] = getattr(cnt, n)
    for i, k in enumerate(KIND_NAMES):
        d["drops_" + k] = cnt.drops[i]
    for n in L1_COUNTER_NAMES + MIG_COUNTER_NAMES + MEM_COUNTER_NAMES:
        d[n] = getattr(cnt, n)
    # memoryview -> list converts in C (list() over a ctypes array boxes each
    # element through ctypes: 0.7 ms of a 6.6 ms C3 step, measured)
    return d, _u64_list(hl), _u64_list(hd), _u64_list(ha)


def _u64_list(a) -> list:
    return memoryview(a).cast("B").cast("Q").tolist()


def noc_sim_state_hash(h) -> int:
    v = C.c_uint64()
    _check(lib().noc_sim_state_hash(h, C.byref(v)))
    return int(v.value)


def noc_sim_get_info(h) -> dict:
    i = noc_sim_info()
    _check(lib().noc_sim_get_info(h, C.byref(i)))
    return {k: getattr(i, k) for k, _ in noc_sim_info._fields_ if k != "reserved"}


def noc_sim_nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for world_size > 1 (rank 0 calls it)."""
    buf = (C.c_uint8 * 128)()
    _check(lib().noc_sim_nccl_unique_id(buf))
    return bytes(buf)


def noc_sim_destroy(h):
    if h:
        lib().noc_sim_destroy(h)


class NocSim:
    """Object wrapper over one handle."""

    def __init__(self, cfg: dict, script=None, device: int = 0, engine: int = ENGINE_AUTO, **kw):
        self.cfg = dict(cfg)
        self.nbins = int(cfg["hist_bins"])
        self._h = noc_sim_create(cfg, script, device, engine, **kw)

    def close(self):
        if getattr(self, "_h", None):
            noc_sim_destroy(self._h)
            self._h = None

    __del__ = close

    def run(self, n):
        noc_sim_run(self._h, n)

    def run_timed(self, n):
        return noc_sim_run_timed(self._h, n)

    def push_script(self, events):
        """Append scripted events [(cycle, node, value), ...] (NEXT-f3 streamed
        trace replay, noc_sim_push_script, DESIGN R57)."""
        events = list(events)
        ev = (noc_sim_event * max(len(events), 1))()
        for i, (cy, node, val) in enumerate(events):
            ev[i].cycle, ev[i].node, ev[i].value = cy, node, val
        _check(lib().noc_sim_push_script(self._h, ev, len(events)))

    def drain(self, max_cycles):
        return noc_sim_drain(self._h, max_cycles)

    def stats(self):
        return noc_sim_stats(self._h, self.nbins)

    def state_hash(self):
        return noc_sim_state_hash(self._h)

    def info(self):
        return noc_sim_get_info(self._h)
