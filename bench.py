#!/usr/bin/env python
"""Benchmark: simulated node-cycles/s of the bufferless-NoC + LSPD-L2 hot path
(BASELINE.json metric) on B200, one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c3] [--cycles-per-step C] [--engine auto|step|persist]

A step = C simulated cycles of the whole hot path (all SURVEY 8(a) rows) of
the workload mesh; value = node-cycles of all ranks / max-over-ranks device
time of exactly K steps (CUDA events on the library's stream, L2 flushed
between steps).  --impl reference times the CPU oracle (this tier's reference
arm) on the same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1508_03235_b200 import workloads as W  # noqa: E402

METRIC = "simulated node-cycles/sec (device-timed) at 1/2/4/8 B200; % of HBM roofline"
ENGINES = {"auto": 0, "step": 1, "persist": 2, "tiled": 3, "tiled4": 4}          # NOC_ENGINE_*
KERNELS = {1: "k_step", 2: "k_persist", 3: "k_tiled", 4: "k_tiled4"}
UNIT = "node-cycles/s"
WORKLOADS = {
    "c3": ("208x208 LSPD (BASELINE configs[2], paper's largest mesh)", W.c3),
    "c1a": ("4x4 uniform random lambda 0.1 (BASELINE configs[0], C1a)", W.c1a),
    "c1b": ("4x4 LSPD (BASELINE configs[0], C1b)", W.c1b),
    "c2": ("64x64 LSPD (BASELINE configs[1])", W.c2),
    "c4ur": ("208x208 uniform random lambda 0.3 (BASELINE configs[3])", lambda seed=1: W.c4(0.3, seed=seed)),
    "c5": ("1024x1024 LSPD (BASELINE configs[4])", W.c5),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def b_alg(delta, nodecycles, ways):
    """Algorithmic bytes per node-cycle, SURVEY 8(d.3) / DESIGN 7."""
    h = delta["hops"] / nodecycles
    i = delta["injected"] / nodecycles
    p = delta["packets_enqueued"] / nodecycles
    a = delta["accesses"] / nodecycles
    e = (delta["dir_searches"] + delta["requests_received"] + delta["installs"] + delta["evs_received"]) / nodecycles
    return 12 + 32 * h + 20 * i + 20 * p + (24 + 8 * ways) * a + 24 * e, dict(h=h, i=i, p=p, a=a, e=e)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), "--query-gpu=" + self.FIELDS,
                                       "--format=csv,noheader,nounits", "-lms", "10"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        # start the timed region only once nvidia-smi is sampling
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 3.0:
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.01)

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            try:
                r = [x.strip() for x in r]
                util = float(r[6])
                mx = max(mx, float(r[1]))
                if util > 0:
                    sm.append(float(r[0]))
                for k, v in zip(names, r[2:6]):
                    if v.lower() == "active":
                        reasons.add(k)
            except Exception:
                continue
        if not sm:
            sm = [float(r[0]) for r in rows if r and r[0].strip().replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(rows)}


def flush_l2(buf):
    if buf is not None:
        buf.add_(1)


def oracle_rate(cfg, cycles):
    """CPU oracle (as it stands), one host thread, on a bounded sample."""
    from oracle import Oracle
    o = Oracle(cfg)
    t0 = time.perf_counter()
    o.run(cycles)
    dt = time.perf_counter() - t0
    n = cfg["mesh_w"] * cfg["mesh_h"]
    return n * cycles / dt, dt


def host_cpu():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    desc, fn = WORKLOADS[args.workload]
    cfg = fn(seed=1)
    n = cfg["mesh_w"] * cfg["mesh_h"]
    # a bounded sample per step: about 2e7 node-cycles (C3: 200 cycles, C5: 19)
    cyc = args.ref_cycles_per_step or max(2, min(200, int(2e7 // n)))
    from oracle import Oracle
    o = Oracle(cfg)
    for _ in range(args.warmup):
        o.run(cyc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.run(cyc)
    dt = time.perf_counter() - t0
    v = n * cyc * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (counter-based Philox traffic, seed 1)",
        "config": {"workload": args.workload, "desc": desc, "mesh": [cfg["mesh_w"], cfg["mesh_h"]],
                   "cycles_per_step": cyc, "note": "CPU oracle, 1 host thread"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": "%d steps x %d cycles of %s after %d warm-up steps" % (
                             args.steps, cyc, args.workload, args.warmup)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_1508_03235_b200 as pkg

    rank, world, local = env_rank()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(local)
    dev = torch.cuda.current_device()
    desc, fn = WORKLOADS[args.workload]
    eng = ENGINES[args.engine]
    cfg = fn(seed=1)
    scaling = args.scaling or ("strong" if args.workload == "c5" else "weak")
    if world > 1:
        # row bands (DESIGN 8): weak scaling grows the mesh to W x (H*N), rank
        # r owning rows [r*H, (r+1)*H); strong scaling splits the fixed mesh
        # into N bands.  Edge-row links go to ranks r-1 / r+1 from inside the
        # kernel (CUDA IPC over NVLink)
        from paper_1508_03235_b200 import dist as pdist
        if scaling == "weak":
            cfg["mesh_h"] = cfg["mesh_h"] * world
        sim = pdist.create_band_sim(cfg, dev, engine=eng)
    else:
        sim = pkg.NocSim(cfg, device=dev, engine=eng)
    n = sim.info()["nodes_local"]
    cyc = args.cycles_per_step
    l2buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if not args.no_flush else None

    for _ in range(args.warmup):
        sim.run(cyc)
    st0 = sim.stats()[0]
    info0 = sim.info()
    clocks = Clocks(dev) if rank == 0 else None
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    dev_ms = 0.0
    for _ in range(args.steps):
        flush_l2(l2buf)
        torch.cuda.synchronize()
        dev_ms += sim.run_timed(cyc)
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([dev_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
        dev_ms = float(t.item())
    ck = clocks.stop() if clocks else None
    st1 = sim.stats()[0]
    info1 = sim.info()
    delta = {k: st1[k] - st0[k] for k in st1}
    nodecycles = n * cyc * args.steps
    value = nodecycles * world / (dev_ms / 1e3)

    # roofline of the dominant (only) kernel in the timed region
    peak, peak_src = peaks()
    # stats() sums the counters over all ranks: rates are per node-cycle of the whole job
    B, rates = b_alg(delta, nodecycles * world, cfg["l2_ways"] if cfg["mode"] == W.MODE_LSPD else 2)
    launches = info1["kernel_launches"] - info0["kernel_launches"]
    # the TILED engines also launch the LL-slot refresh kernel before each
    # node-step launch (one per band of this process)
    gpu_launches = launches * (2 if info1["engine"] in (3, 4) and not info1.get("cluster") else 1)
    per_launch_ms = dev_ms / max(launches, 1)
    achieved = B * nodecycles / (dev_ms / 1e3) / 1e9          # per GPU (this rank's nodes)
    traffic, ncu_info = None, None
    tf = os.path.join(ROOT, "profiles", "traffic_%s.json" % args.workload)
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get("dram_bytes_per_launch")
            ncu_info = {k: tj.get(k) for k in ("dram_bytes_per_node_cycle", "lts_bytes_per_node_cycle",
                                              "warp_inst_per_node_cycle", "l2_hit_rate_pct", "summary")}
        except Exception:
            traffic = None

    # end to end through the public API: run + stats copy per step (host wall clock)
    e2e_steps = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sim.run(cyc)
        sim.stats()
    e2e_s = time.perf_counter() - t0
    nb = cfg["hist_bins"]
    d2h = 8 * (31 + 1) + 3 * 8 * nb

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (counter-based Philox traffic keyed on (seed, node, cycle))",
        "config": {"workload": args.workload, "desc": desc, "mesh": [cfg["mesh_w"], cfg["mesh_h"]],
                   "nodes_per_gpu": n, "cycles_per_step": cyc, "engine": info1["engine"],
                   "grid": info1["grid"], "block": info1["block"],
                   "l2_flush": "256 MiB buffer written between timed steps" if l2buf is not None else "none",
                   "parallelism": ("row bands x%d (%s scaling: %dx%d mesh, one %d-row band per GPU, "
                                   "in-kernel NVLink boundary exchange)" % (world, scaling, cfg["mesh_w"], cfg["mesh_h"],
                                                                           cfg["mesh_h"] // world)
                                   if world > 1 else "single GPU")},
        "e2e": {"value": n * cyc * e2e_steps * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": d2h,
                "note": "noc_sim_run + noc_sim_stats per step, host wall clock; traffic is generated on "
                        "device (counter-based), so no per-step input copy"},
        "gpu_launches": gpu_launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": KERNELS.get(info1["engine"], "engine %d" % info1["engine"]),
                     "bytes_per_node_cycle": B, "rates": rates, "per_launch_ms": per_launch_ms,
                     # the dense accounting (every link slot read and written,
                     # 32 B of core state) for transparency, and the ncu measurements of the
                     # same launch (profiles/traffic_<workload>.json) when present
                     "dense": {"bytes_per_node_cycle": 168.0,
                               "frac": 168.0 * nodecycles / (dev_ms / 1e3) / 1e9 / peak},
                     "ncu": ncu_info},
        "clocks": ck,
        "sim": {"hash": None, "drops": sum(v for k, v in delta.items() if k.startswith("drops_"))},
        # the band-edge exchange per cycle of an interior rank (two
        # edges, W links each way, one 32-byte LL slot per link and cycle written
        # across NVLink whether or not it carries a flit)
        "halo": ({"links_per_cycle_per_edge_each_way": cfg["mesh_w"],
                  "bytes_per_cycle_interior_rank": (2 * 2 * cfg["mesh_w"] * 32 if info1["engine"] in (3, 4)
                                                    else None),
                  "engine_exchange": ("TILED: one 32-byte LL slot per band-edge link and cycle, stored into the "
                                      "neighbour rank's memory (CUDA IPC)" if info1["engine"] in (3, 4) else
                                      "PERSIST: 16 B flit + 1 flag byte per crossing flit, stored into the "
                                      "neighbour rank's arrays (CUDA IPC)")}
                 if world > 1 else None),
    }
    # the median over 5 fresh creations (same warm-up, one step each)
    fresh = None
    if world == 1 and args.fresh > 0:
        per = []
        for _ in range(args.fresh):
            f = pkg.NocSim(cfg, device=dev, engine=eng)
            f.run(cyc * args.warmup)
            flush_l2(l2buf)
            torch.cuda.synchronize()
            per.append(f.run_timed(cyc))
            f.close()
        fresh = {"creations": len(per), "median_ms_per_step": statistics.median(per),
                 "median_value": n * cyc / (statistics.median(per) / 1e3),
                 "min_ms_per_step": min(per), "max_ms_per_step": max(per)}
    line["fresh_creations"] = fresh
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample: at most ~1e8 node-cycles of oracle work
        ccyc = max(20, min(args.cpu_cycles, int(1e8 // (cfg["mesh_w"] * cfg["mesh_h"]))))
        v, dt = oracle_rate(cfg, ccyc)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": "%s cycles 0-%d from a fresh state, 1 host thread (%.1f s)" % (
                                    args.workload, ccyc, dt),
                                "host_cpu": host_cpu(), "host_nproc": os.cpu_count()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: c3 on one GPU, c5 (strong scaling) on several")
    ap.add_argument("--cycles-per-step", type=int, default=2000)
    ap.add_argument("--ref-cycles-per-step", type=int, default=0, help="0: ~2e7 node-cycles per step")
    ap.add_argument("--cpu-cycles", type=int, default=2000)
    ap.add_argument("--engine", default="auto", choices=sorted(ENGINES))
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fresh", type=int, default=5, help="fresh creations for the median (SURVEY 8(d.4)); 0 = off")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N>1: weak (mesh height x N, default) or strong (fixed mesh; default for c5)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.workload is None:
        # one GPU: the 208x208 single-B200 configuration (BASELINE configs[2]);
        # several: the 1024x1024 mesh in row bands (configs[4], strong scaling)
        args.workload = "c3" if args.gpus == 1 else "c5"
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_ours(args)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) with
    torch.distributed.run on this node and relay rank 0's line."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write("bench.py: --gpus %d needs %d CUDA devices, this box has %d\n" % (args.gpus, args.gpus, have))
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
