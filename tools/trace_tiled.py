"""Per-warp cycle trace of the TILED engine (needs the -DNOC_TRACE build:
NOCSIM_DEFS=-DNOC_TRACE NOCSIM_LIB=.../ab/trace.so python -m paper_1508_03235_b200.build --force).
usage: NOCSIM_LIB=.../ab/trace.so python tools/trace_tiled.py [workload] [warm]
Prints where each cycle's time goes: per-CTA cycle length, the arrival of the
last warp at the cycle barrier, and the event mix of the warps that arrive last."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402

TRACE_CYC, TRACE_WARPS = 1024, 1536
wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 6000
cfg = {"c3": W.c3, "c2": W.c2, "c4ur": lambda: W.c4(0.3),
       "ur0": lambda: W.make(mesh_w=208, mesh_h=208, mode=W.MODE_UR, thr_inj=0)}[wl]()
lib = ctypes.CDLL(pkg.LIB_PATH)
lib.noc_trace_ctl.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
s = pkg.NocSim(cfg, engine=pkg.ENGINE_TILED)
s.run(warm)
info = s.info()
lib.noc_trace_ctl(1, None, 0)
ms = s.run_timed(TRACE_CYC)
lib.noc_trace_ctl(0, None, 0)
buf = np.zeros((TRACE_CYC, TRACE_WARPS, 8), dtype=np.uint32)
assert lib.noc_trace_ctl(0, buf.ctypes.data, buf.nbytes) == 0
grid, block = info["grid"], info["block"]
wpc = block // 32
nw = grid * wpc
tr = buf[:, :nw, :].astype(np.int64)
start, arrive, ev, extw = tr[..., 0], tr[..., 1], tr[..., 2], tr[..., 3]
p3w, p1w, pubw = tr[..., 4], tr[..., 5], tr[..., 6]
print("%s: %.3f us/cycle (traced run), grid %d x %d warps" % (wl, ms * 1e3 / TRACE_CYC, grid, wpc))
# per CTA: cycle length from warp 0's start clocks (same SM clock)
st0 = start[:, ::wpc]
clen = (st0[1:] - st0[:-1]) & 0xFFFFFFFF
print("CTA cycle length (clk): median %d  p90 %d  max %d" % (np.median(clen), np.percentile(clen, 90), clen.max()))
arr = arrive.reshape(TRACE_CYC, grid, wpc)
ofs = (start.reshape(TRACE_CYC, grid, wpc) - st0[:, :, None]) & 0xFFFFFFFF
ofs = np.where(ofs > 1 << 31, ofs - (1 << 32), ofs)
fin = ofs + arr                                      # barrier arrival relative to warp 0's start
last = fin.max(axis=2)
print("last-warp arrival (clk): median %d  p90 %d ; barrier release gap median %d" % (
    np.median(last[:-1]), np.percentile(last[:-1], 90), np.median(clen - last[:-1])))
print("warp compute time (clk): median %d  mean %d  p90 %d  p99 %d" % (
    np.median(arr), arr.mean(), np.percentile(arr, 90), np.percentile(arr, 99)))
names = ["phase3", "p1-state", "p1-enq", "refresh", "conflict", "inject", "flits", "boundary"]
# per-warp offsets (clk from the warp's cycle start): ext inputs complete, boundary
# outputs published, Phase 3 done, Phase 1 of the next cycle done, barrier arrival
e3 = ev.reshape(TRACE_CYC, grid, wpc)
print("%-10s %8s %10s %10s %12s" % ("event", "warps%", "time(with)", "time(w/o)", "in last warp%"))
lw = fin.argmax(axis=2)
lastev = np.take_along_axis(e3, lw[..., None], axis=2)[..., 0]
for b, nme in enumerate(names):
    m = (e3 >> b) & 1
    w = arr[m == 1]
    wo = arr[m == 0]
    print("%-10s %7.1f%% %10.0f %10.0f %11.1f%%" % (nme, 100 * m.mean(), w.mean() if w.size else 0,
                                                    wo.mean() if wo.size else 0, 100 * ((lastev >> b) & 1).mean()))
bx = extw.reshape(TRACE_CYC, grid, wpc)
bnd = ((e3 >> 7) & 1) == 1
print("boundary warps: ext-complete offset median %d p90 %d; arrival median %d" % (
    np.median(bx[bnd]), np.percentile(bx[bnd], 90), np.median(arr[bnd])))
print("interior warps arrival median %d" % (np.median(arr[~bnd]) if (~bnd).any() else -1))
for nm, msk in (("boundary", bnd), ("interior", ~bnd)):
    if not msk.any():
        continue
    q = lambda a: "%5d %5d %5d" % (np.percentile(a[msk], 50), np.percentile(a[msk], 90), a[msk].mean())
    print("%s warps (p50 p90 mean clk from cycle start): ext done %s | published %s | phase3 done %s | "
          "phase1 done %s | barrier %s" % (nm, q(bx), q(pubw.reshape(arr.shape)), q(p3w.reshape(arr.shape)),
                                          q(p1w.reshape(arr.shape)), q(arr)))
for par in (0, 1):
    sel = (np.arange(TRACE_CYC - 1) % 2) == par
    print("cycles with cc %% 2 == %d: CTA cycle median %d p90 %d; boundary ext done p50 %d p90 %d; interior phase1-done p50 %d p90 %d; boundary barrier p50 %d; interior barrier p50 %d" % (
        par, np.median(clen[sel]), np.percentile(clen[sel], 90),
        np.percentile(bx[:-1][sel][bnd[:-1][sel]], 50), np.percentile(bx[:-1][sel][bnd[:-1][sel]], 90),
        np.percentile(p1w.reshape(arr.shape)[:-1][sel][~bnd[:-1][sel]], 50), np.percentile(p1w.reshape(arr.shape)[:-1][sel][~bnd[:-1][sel]], 90),
        np.median(arr[:-1][sel][bnd[:-1][sel]]), np.median(arr[:-1][sel][~bnd[:-1][sel]])))
print("last warp is a boundary warp in %.1f%% of CTA-cycles" % (100 * ((lastev >> 7) & 1).mean()))
