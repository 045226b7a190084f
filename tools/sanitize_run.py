"""Small runs of every engine for compute-sanitizer (memcheck / racecheck /
synccheck): C1b (4x4 LSPD) and a 12x10 LSPD mesh, short runs, plus a drain;
TILED with a forced 2x2 tiling so the cross-tile exchange runs.
usage: compute-sanitizer --tool T python tools/sanitize_run.py [cycles]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 120
cfgs = [("c1b", W.c1b()), ("c1a", W.c1a()),
        ("12x10", W.make(mesh_w=12, mesh_h=10, mode=W.MODE_LSPD, lam=0.2, sendq_cap=32, l2_sets=4, mem_lat=20))]
for name, cfg in cfgs:
    for eng in (pkg.ENGINE_STEP, pkg.ENGINE_PERSIST, pkg.ENGINE_TILED, pkg.ENGINE_TILED4):
        for tiling in ((None, "2x2") if eng == pkg.ENGINE_TILED else (None,)):
            if tiling:
                os.environ["NOCSIM_TILING"] = tiling
            else:
                os.environ.pop("NOCSIM_TILING", None)
            s = pkg.NocSim(cfg, engine=eng)
            s.run(cyc)
            s.drain(5000)
            s.run(cyc // 2)
            h = s.state_hash()
            print("%-6s engine %d tiling %-5s grid %3d hash %016x" % (name, eng, tiling, s.info()["grid"], h), flush=True)
            s.close()
print("sanitize_run done")
