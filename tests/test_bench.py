"""The bench.py contract: one JSON line with the driver's keys."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-cycles-per-step", "5",
                  "--workload", "c2")
    assert KEYS <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_engine_names_cover_the_header():
    sys.path.insert(0, ROOT)
    import bench
    import paper_1508_03235_b200 as pkg
    assert set(bench.ENGINES.values()) == {pkg.ENGINE_AUTO, pkg.ENGINE_STEP, pkg.ENGINE_PERSIST,
                                           pkg.ENGINE_TILED, pkg.ENGINE_TILED4}
    assert set(bench.KERNELS) == set(bench.ENGINES.values()) - {0}


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["auto", "tiled", "persist"])
def test_bench_json_line_on_gpu(engine):
    d = run_bench("--steps", "3", "--warmup", "3", "--cycles-per-step", "200", "--cpu-cycles", "20",
                  "--engine", engine)
    assert KEYS <= set(d) and {"roofline", "cpu_baseline", "clocks", "gpu_launches"} <= set(d)
    assert d["value"] > 0 and d["gpu_launches"] > 0 and 0 < d["roofline"]["frac"] < 1.5


def test_gpus_beyond_the_box_is_an_error():
    """`bench.py --gpus N` outside torchrun spawns N ranks; with fewer than N
    devices it fails with a clear message instead of reporting one GPU."""
    import torch
    n = max(2, torch.cuda.device_count() + 1)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")})
    assert out.returncode == 2 and "needs %d CUDA devices" % n in out.stderr
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
