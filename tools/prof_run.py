"""Profiling driver: create a workload, warm up, then advance in launches of
--cycles cycles (run under ncu; never report its numbers as bench values)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c3")
ap.add_argument("--warm", type=int, default=1000)
ap.add_argument("--cycles", type=int, default=200)
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--engine", type=int, default=0)
a = ap.parse_args()
cfg = {"c3": W.c3, "c2": W.c2, "c5": W.c5, "c4ur": lambda: W.c4(0.3),
       "ur0": lambda: W.make(mesh_w=208, mesh_h=208, mode=W.MODE_UR, thr_inj=0)}[a.workload]()
s = pkg.NocSim(cfg, engine=a.engine)
s.run(a.warm)
for _ in range(a.launches):
    ms = s.run_timed(a.cycles)
    print("launch %d cycles %.3f ms -> %.3f us/cycle" % (a.cycles, ms, ms * 1e3 / a.cycles))
print(s.info())
