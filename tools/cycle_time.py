"""us per simulated cycle for several meshes/engines (after warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
cases = [("ur4x4 l=0", W.make(mode=0, thr_inj=0)), ("ur16x16 l=0", W.make(mesh_w=16, mesh_h=16, mode=0, thr_inj=0)),
         ("ur64 l=0", W.make(mesh_w=64, mesh_h=64, mode=0, thr_inj=0)), ("ur208 l=0", W.make(mesh_w=208, mesh_h=208, mode=0, thr_inj=0)),
         ("c2", W.c2()), ("c3", W.c3()), ("ur208 l=.3", W.c4(0.3))]
engines = [int(a) for a in sys.argv[1:]] or [3]
for name, cfg in cases:
    for e in engines:
        s = pkg.NocSim(cfg, engine=e)
        s.run(2000)
        ms = s.run_timed(2000)
        info = s.info()
        print("%-12s engine %d grid %4d block %4d: %.3f us/cycle" % (name, e, info["grid"], info["block"], ms * 1e3 / 2000), flush=True)
        s.close()
