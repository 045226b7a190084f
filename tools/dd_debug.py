import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
from oracle import Oracle
cfg = W.c3()
o = Oracle(cfg); o.run(1500)
sims = {e: pkg.NocSim(cfg, engine=e) for e in (1, 2, 3)}
for s in sims.values(): s.run(1500)
print("run", {e: s.state_hash() == o.state_hash() for e, s in sims.items()}, flush=True)
for k in (10, 50, 200):
    ro = o.drain(k)
    so = o.stats()[0]
    for e, s in sims.items():
        r = s.drain(k); ss = s.stats()[0]
        print(k, e, r, ro, s.state_hash() == o.state_hash(), {kk: (ss[kk], so[kk]) for kk in ss if ss[kk] != so[kk]}, flush=True)
