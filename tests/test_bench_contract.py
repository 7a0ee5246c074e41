"""bench.py keeps the driver's contract: one JSON line with the metric keys.

CPU: the reference arm (`--impl reference`: the reference library on the host
cores, inputs from the C oracle's generators, never the product).
GPU: our arm at N=2 under torch.distributed.run with two ranks on one GPU
(gloo bootstrap; RAS through host-callback collectives) -- the multi-rank
control flow the driver's scaling run uses (one JSON line from rank 0,
max-over-ranks timing, weak scaling).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e"}


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libhecref.so")):
        pytest.skip("oracle/_ref not built")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d) and d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    # the reference arm never loads the product library (bench.py asserts it)
    assert d["product_loaded"] is False


@pytest.mark.gpu
def test_our_arm_two_ranks_one_gpu():
    env = dict(os.environ, HEC_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--config", "c1", "--secondary", "", "--ras-size", "32", "--ras-ref-size", "0"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1, p.stdout
    d = lines[0]
    assert KEYS <= set(d) and d["n_gpus"] == 2 and d["scaling"] == "weak" and d["impl"] == "ours"
    assert d["gpu_launches"] > 0 and d["roofline"]["bound"] == "hbm"
    assert d["ras"]["converged"] and d["ras"]["allreduces"] > 0 and d["ras"]["halo_exchanges"] > 0
