"""Per-window rates of a workload on the GPU (h, i, p, a, e per node-cycle) and us/cycle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
win = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
nwin = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfg = {"c3": W.c3, "c2": W.c2, "c5": W.c5}[name]()
s = pkg.NocSim(cfg)
N = cfg["mesh_w"] * cfg["mesh_h"]
prev = s.stats()[0]
for w in range(nwin):
    ms = s.run_timed(win)
    st = s.stats()[0]
    d = {k: (st[k] - prev[k]) / (N * win) for k in st}
    prev = st
    e = d["dir_searches"] + d["requests_received"] + d["installs"] + d["evs_received"]
    print("t=%6d us/cyc=%.3f h=%.3f i=%.4f p=%.4f a=%.4f e=%.4f hit=%.3f defl/hop=%.4f" % (
        (w + 1) * win, ms * 1e3 / win, d["hops"], d["injected"], d["packets_enqueued"], d["accesses"], e,
        d["l2_hits"] / max(d["accesses"], 1e-12), d["deflections"] / max(d["hops"], 1e-12)), flush=True)
