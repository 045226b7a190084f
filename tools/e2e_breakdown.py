"""Where the end-to-end step time goes at C3 (public API): run() alone, stats()
alone, run()+stats(), against the device time of the same launches."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
s = pkg.NocSim(W.c3())
s.run(6000)
def tm(f, n=5):
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e3
print("run_timed(2000) device ms: %.3f" % s.run_timed(2000))
print("run(2000) ms:              %.3f" % tm(lambda: s.run(2000)))
print("stats() ms:                %.3f" % tm(lambda: s.stats(), 20))
print("run(2000)+stats() ms:      %.3f" % tm(lambda: (s.run(2000), s.stats())))
h = s._h
nb = s.nbins
def raw():
    cnt = pkg.noc_sim_counters()
    hl, hd, ha = (C.c_uint64 * nb)(), (C.c_uint64 * nb)(), (C.c_uint64 * nb)()
    pkg.lib().noc_sim_stats(h, C.byref(cnt), hl, hd, ha, nb)
print("C noc_sim_stats only ms:   %.3f" % tm(raw, 20))
print("run(1) ms:                 %.3f" % tm(lambda: s.run(1), 20))
