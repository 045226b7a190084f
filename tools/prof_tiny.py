import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
cfg = W.make(mode=0, thr_inj=0) if len(sys.argv) < 2 else W.make(mesh_w=int(sys.argv[1]), mesh_h=int(sys.argv[1]), mode=0, thr_inj=0)
s = pkg.NocSim(cfg, engine=3)
s.run(2000)
for _ in range(2):
    ms = s.run_timed(2000)
    print("%.3f us/cycle" % (ms * 1e3 / 2000))
