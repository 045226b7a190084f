"""C4 (BASELINE configs[3]): 208x208 injection-rate sweep on one B200.

For each rate and traffic mode: node-cycles/s (device-timed, AUTO engine),
algorithmic bytes per node-cycle and HBM-roofline fraction (bench.b_alg), and
the network's accepted throughput, mean flit latency and deflections per flit
from the run's own counters / histograms.  Writes one line per point.
usage: python tools/sweep_c4.py [out.txt]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402

WARM, CYC, REPS = 4000, 2000, 2
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
peak, _ = bench.peaks()
print("# C4 sweep, 208x208, seed 1, %d warm-up cycles, %d x %d timed cycles; peak %.1f GB/s" % (WARM, REPS, CYC, peak),
      file=out)
print("%-5s %5s %6s %12s %8s %7s %8s %9s %8s %8s" % ("mode", "lam", "engine", "node-cyc/s", "us/cyc", "B_alg",
                                                    "roofl%", "accepted", "lat", "defl/fl"), file=out, flush=True)
for mode in (W.MODE_UR, W.MODE_LSPD):
    for lam in (0.005, 0.01, 0.05, 0.1, 0.2, 0.3, 0.4, 0.5):
        if mode == W.MODE_LSPD and lam < 0.05:
            continue
        cfg = W.c4(lam, mode=mode)
        s = pkg.NocSim(cfg)
        s.run(WARM)
        st0, h0 = s.stats()[0], s.stats()[1]
        ms = sum(s.run_timed(CYC) for _ in range(REPS))
        st1, h1 = s.stats()[0], s.stats()[1]
        d = {k: st1[k] - st0[k] for k in st1}
        n = cfg["mesh_w"] * cfg["mesh_h"]
        nc = n * CYC * REPS
        B, _ = bench.b_alg(d, nc, cfg["l2_ways"] if mode == W.MODE_LSPD else 2)
        rate = nc / (ms / 1e3)
        ej = d["ejected"]
        hl = [b - a for a, b in zip(h0, h1)]
        lat = sum(i * c for i, c in enumerate(hl)) / max(1, sum(hl))
        print("%-5s %5.3f %6d %12.4g %8.3f %7.1f %8.2f %9.4f %8.1f %8.2f" % (
            "UR" if mode == W.MODE_UR else "LSPD", lam, s.info()["engine"], rate, ms * 1e3 / (CYC * REPS), B,
            100 * B * rate / 1e9 / peak, ej / nc, lat, d["deflections"] / max(1, ej)), file=out, flush=True)
        s.close()
