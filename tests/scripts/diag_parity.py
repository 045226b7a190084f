"""Find the first run() call (then the first 10- / 2-cycle block) after which
the GPU state hash departs from the oracle's, for a failing parity case.
usage: python tools/diag_parity.py [case]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1508_03235_b200 as nb  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402
from oracle import Oracle  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "ur3"
cases = {
    "ur3": (W.make(mesh_w=40, mesh_h=37, mode=W.MODE_UR, lam=0.3, band_streams=1), 3),
    "ur3one": (W.make(mesh_w=40, mesh_h=37, mode=W.MODE_UR, lam=0.3), 3),
    "lspd3": (W.lspd(40, 37, lam=0.2, band_streams=1), 3),
}
cfg, bands = cases[case]
if "drain" in sys.argv:
    g = nb.NocSim(cfg, bands=bands, engine=nb.ENGINE_TILED)
    o = Oracle(cfg)
    for k in (1, 5, 250, 744, 1000):
        g.run(k)
        o.run(k)
    print("before drain", g.state_hash() == o.state_hash(), g.stats()[0]["cycle"])
    print("drain", g.drain(20000), o.drain(20000))
    print("after drain", g.state_hash() == o.state_hash(), g.stats()[0]["cycle"], o.stats()[0]["cycle"])
    for k in [1] * 300:
        g.run(k)
        o.run(k)
        if g.state_hash() != o.state_hash():
            gs, os_ = g.stats()[0], o.stats()[0]
            print("mismatch after", gs["cycle"], {x: (gs[x], os_[x]) for x in gs if gs[x] != os_[x]})
            break
    else:
        print("no mismatch in 300 single-cycle runs after the drain")
    sys.exit(0)
for step in (None, 10, 2):
    g = nb.NocSim(cfg, bands=bands, engine=nb.ENGINE_TILED)
    o = Oracle(cfg)
    splits = [1, 5, 250, 744, 1000, 300] if step is None else [step] * (2300 // step)
    done = 0
    bad = None
    for k in splits:
        g.run(k)
        o.run(k)
        done += k
        if g.state_hash() != o.state_hash():
            gs, os_ = g.stats()[0], o.stats()[0]
            print("step", step, "first mismatch after cycle", done, {x: (gs[x], os_[x]) for x in gs if gs[x] != os_[x]}, flush=True)
            bad = done
            break
    if bad is None:
        print("step", step, "no mismatch through cycle", done, flush=True)
    g.close()
