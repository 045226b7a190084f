"""Debug driver: one small TILED run, prints the error if any."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402
for name, cfg in (("c1b", W.c1b(seed=1)), ("c1a", W.c1a(seed=1)), ("ur64", W.make(mesh_w=64, mesh_h=64, mode=0, thr_inj=0))):
    s = pkg.NocSim(cfg, engine=3)
    try:
        for k in range(10):
            s.run(1000)
        print(name, "ok", s.stats()[0]["ejected"], flush=True)
    except Exception as e:
        print(name, "ERR", e, flush=True)
    s.close()
