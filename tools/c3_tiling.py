"""C3 per-cycle time for forced tilings (NOCSIM_TILING=TXxTY), steady state (6000 warm-up cycles, 3 x 2000)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    import paper_1508_03235_b200 as pkg
    from paper_1508_03235_b200 import workloads as W
    s = pkg.NocSim(W.c3(), engine=3)
    s.run(6000)
    v = [s.run_timed(2000) * 1e3 / 2000 for _ in range(3)]
    i = s.info()
    print("%-6s grid %3d block %3d: %s us/cycle" % (os.environ.get("NOCSIM_TILING", "auto"), i["grid"], i["block"],
                                                   " ".join("%.3f" % x for x in v)), flush=True)
    sys.exit(0)
for t in ["auto", "7x21", "21x7", "11x13", "13x11", "10x14", "14x10", "9x16", "8x18", "12x12"]:
    env = dict(os.environ)
    if t != "auto":
        env["NOCSIM_TILING"] = t
    r = subprocess.run([sys.executable, __file__, "one"], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout.strip() or ("%s: failed %s" % (t, r.stderr.strip().splitlines()[-1:] if r.stderr else "")), flush=True)
