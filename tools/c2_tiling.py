"""us per simulated cycle of C2 (64x64 LSPD) under forced TILED tilings (NOCSIM_TILING)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import paper_1508_03235_b200 as pkg
    from paper_1508_03235_b200 import workloads as W
    s = pkg.NocSim(W.c2(), engine=3)
    s.run(4000)
    v = [s.run_timed(2000) * 1e3 / 2000 for _ in range(3)]
    i = s.info()
    print("tiling %-8s grid %4d block %4d: %s us/cycle" % (sys.argv[1], i["grid"], i["block"], " ".join("%.3f" % x for x in v)), flush=True)
    sys.exit(0)
for t in ("default", "2x2", "4x2", "4x4", "8x4", "8x8", "16x8"):
    env = dict(os.environ)
    if t != "default":
        env["NOCSIM_TILING"] = t
    subprocess.run([sys.executable, __file__, t], env=env)
