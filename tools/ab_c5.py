"""A/B per-cycle timing of library variants (NOCSIM_LIB) at C5 (1024x1024 LSPD, PERSIST)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg
from paper_1508_03235_b200 import workloads as W
s = pkg.NocSim(W.c5(), engine=2)
s.run(4000)
v = [s.run_timed(1000) * 1e3 / 1000 for _ in range(3)]
i = s.info()
print("%s c5 grid %d: %s us/cycle" % (os.path.basename(os.environ.get("NOCSIM_LIB", "default")), i["grid"],
                                       " ".join("%.2f" % x for x in v)), flush=True)
