"""A/B per-cycle timing of library variants (NOCSIM_LIB) at C3 and an idle mesh, 3 repetitions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
eng = int(sys.argv[1]) if len(sys.argv) > 1 else 3
res = []
for name, cfg in (("c3", W.c3()), ("ur208 l=0", W.make(mesh_w=208, mesh_h=208, mode=0, thr_inj=0))):
    s = pkg.NocSim(cfg, engine=eng)
    s.run(6000)
    v = [s.run_timed(2000) * 1e3 / 2000 for _ in range(3)]
    print("%s %-10s %s us/cycle" % (os.path.basename(os.environ.get("NOCSIM_LIB", "default")), name, " ".join("%.3f" % x for x in v)), flush=True)
    s.close()
