import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
from oracle import Oracle
cfg = W.make(mesh_w=16, mesh_h=16, mode=0, lam=0.3)
for seq in ([("run", 305)], [("run", 300), ("run", 5)], [("run", 1), ("run", 1)], [("run", 2), ("run", 2), ("run", 2)], [("run", 300), ("drain", 5)]):
    s = pkg.NocSim(cfg, engine=3)
    o = Oracle(cfg)
    out = []
    for op, arg in seq:
        if op == "run":
            s.run(arg); o.run(arg)
        else:
            s.drain(arg); o.drain(arg)
        gs, os_ = s.stats()[0], o.stats()[0]
        out.append((op, arg, s.state_hash() == o.state_hash(), {k: (gs[k], os_[k]) for k in gs if gs[k] != os_[k]}))
    print(s.info(), flush=True)
    print(out, flush=True)
