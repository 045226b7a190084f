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
# round-2 features: memory nodes + hub FIFOs, fill-all injection, streamed scripts, migration,
# the opt-in cluster exchange (TILED, 2x2 tiles as one cluster)
extra = [("memctrl", W.make(mesh_w=12, mesh_h=10, mode=W.MODE_LSPD, lam=0.1, sendq_cap=32, l2_sets=4, mem_lat=20,
                            mem_mode=W.MEM_CTRLS, mem_ctrls=3, hub_sendq_cap=256, nfl_b2=5)),
         ("fillall", W.make(mesh_w=12, mesh_h=10, mode=W.MODE_LSPD, lam=0.2, sendq_cap=32, l2_sets=4, mem_lat=20,
                            inject_mode=2)),
         ("mig", W.make(mesh_w=12, mesh_h=10, mode=W.MODE_LSPD, lam=0.2, sendq_cap=64, l2_sets=4, mem_lat=20,
                        mig_hist=6, nfl_b2=16))]
for name, cfg in extra:
    for eng in (pkg.ENGINE_STEP, pkg.ENGINE_PERSIST, pkg.ENGINE_TILED):
        os.environ["NOCSIM_TILING"] = "2x2"
        s = pkg.NocSim(cfg, engine=eng)
        s.run(cyc)
        s.push_script(W.random_script(cfg, 40, cyc * 2, seed=3))
        s.run(cyc)
        s.drain(5000)
        print("%-6s engine %d hash %016x" % (name, eng, s.state_hash()), flush=True)
        s.close()
os.environ["NOCSIM_TILING"] = "2x2"
os.environ["NOCSIM_CLUSTER"] = "1"
os.environ.pop("NOCSIM_TILING", None)
for name, cfg in (("24x20", W.make(mesh_w=24, mesh_h=20, mode=W.MODE_LSPD, lam=0.2, sendq_cap=32, l2_sets=4,
                                   mem_lat=20)),
                  ("ur40x30", W.make(mesh_w=40, mesh_h=30, mode=W.MODE_UR, lam=0.2))):
    s = pkg.NocSim(cfg, engine=pkg.ENGINE_TILED)
    s.run(cyc)
    s.drain(5000)
    print("%-6s cluster %d hash %016x" % (name, s.info()["cluster"], s.state_hash()), flush=True)
    s.close()
print("sanitize_run done")
