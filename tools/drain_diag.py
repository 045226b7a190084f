"""Diagnose drain at C3: run, drain, report what is still in flight."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402

for eng in (int(a) for a in sys.argv[1:] or ["3", "2"]):
    s = pkg.NocSim(W.c3(), engine=eng)
    s.run(20000)
    for cap in (20000, 100000, 200000):
        used, dr = s.drain(cap)
        st, hl, hd, ha = s.stats()
        inflight = st["injected"] - st["ejected"]
        busy = st["accesses"] - st["completed"]
        maxage = max(b for b, c in enumerate(hd) if c)
        maxlat = max(b for b, c in enumerate(hl) if c)
        print("engine", eng, "drain", cap, "->", used, dr, "inflight", inflight, "cores busy", busy,
              "max age", maxage, "max lat", maxlat, "drops", sum(v for k, v in st.items() if k.startswith("drops")),
              flush=True)
        if dr:
            break
