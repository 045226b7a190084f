"""compute-sanitizer target for the UR split cycle barrier (DESIGN 6.3): UR
meshes on the TILED engine with multi-warp tiles (2x2 forced tiling of 40x30:
300-node tiles, and the default tiling of 64x64), short runs, a drain (drain
launches use BAR.SYNC) and a run after it; hashes checked against the oracle.
usage: compute-sanitizer --tool T python tools/sanitize_split.py [cycles]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1508_03235_b200 as pkg  # noqa: E402
from paper_1508_03235_b200 import workloads as W  # noqa: E402
from oracle import Oracle  # noqa: E402

cyc = int(sys.argv[1]) if len(sys.argv) > 1 else 60
for name, cfg, tiling in (("ur40x30", W.make(mesh_w=40, mesh_h=30, mode=W.MODE_UR, lam=0.3), "2x2"),
                          ("ur64", W.make(mesh_w=64, mesh_h=64, mode=W.MODE_UR, lam=0.2), None)):
    if tiling:
        os.environ["NOCSIM_TILING"] = tiling
    else:
        os.environ.pop("NOCSIM_TILING", None)
    s = pkg.NocSim(cfg, engine=pkg.ENGINE_TILED)
    o = Oracle(cfg)
    for k in (cyc, "drain", cyc // 2):
        if k == "drain":
            assert s.drain(5000) == o.drain(5000)
        else:
            s.run(k)
            o.run(k)
    assert s.state_hash() == o.state_hash(), name
    print("%-8s grid %3d block %3d hash %016x (= oracle)" % (name, s.info()["grid"], s.info()["block"], s.state_hash()),
          flush=True)
    s.close()
print("sanitize_split done")
