"""us per simulated cycle at C2 (64x64 LSPD) and a 40x30 UR mesh: cluster exchange (NOCSIM_CLUSTER=1) vs
LL tiles (the default), TILED engine."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import paper_1508_03235_b200 as pkg
    from paper_1508_03235_b200 import workloads as W
    for name, cfg in (("c2", W.c2()), ("ur40x30 l=.2", W.make(mesh_w=40, mesh_h=30, mode=0, lam=0.2)),
                      ("c2 l=0", W.c2(lam=0.0))):
        s = pkg.NocSim(cfg, engine=3)
        s.run(4000)
        v = [s.run_timed(2000) * 1e3 / 2000 for _ in range(3)]
        i = s.info()
        print("%-8s %-12s grid %4d block %4d cluster %2d: %s us/cycle" % (sys.argv[1], name, i["grid"], i["block"],
              i["cluster"], " ".join("%.3f" % x for x in v)), flush=True)
    sys.exit(0)
for t in ("cluster", "ll"):
    env = dict(os.environ)
    if t == "cluster":
        env["NOCSIM_CLUSTER"] = "1"
    subprocess.run([sys.executable, __file__, t], env=env)
