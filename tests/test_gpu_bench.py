"""bench.py contract on the GPU: the single-GPU JSON line, and a functional run of the
multi-rank path (torchrun, 2 ranks) -- on a 1-GPU box both ranks share the device over gloo,
which checks the sharding, the gradient all-reduce hook and the max-over-ranks reporting, not
performance."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline", "cpu_baseline"}


def run(cmd, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_single_gpu_line():
    d = run([sys.executable, "bench.py", "--config", "C2", "--steps", "3", "--warmup", "3", "--cpu-pixels", "16"])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["roofline"]["frac"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.parametrize("balance,port", [("lpt", 29517), ("cyclic", 29518)])
def test_two_ranks_functional(balance, port):
    """Both tile assignments (cyclic tile shards, LPT tile lists), with the end-to-end leg."""
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
             "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--config", "C2", "--steps", "3",
             "--warmup", "3", "--balance", balance], env={"BENCH_SHARE_GPU": "1", "BENCH_DIST_BACKEND": "gloo"})
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "rays2"
    assert d["config"]["balance"] == balance and d["config"]["rays_per_step"] == 8 * 256 * 256
    assert d["e2e"]["value"] > 0 and d["cpu_baseline"] is None


def test_reference_arm():
    d = run([sys.executable, "bench.py", "--impl", "reference", "--config", "C2", "--steps", "1", "--warmup", "1",
             "--ref-pixels", "16"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0


def test_batch_mode_cuda_graph():
    """--batch: the paper's random-ray training iteration, captured into a CUDA graph."""
    d = run([sys.executable, "bench.py", "--config", "C2", "--batch", "500", "--steps", "5", "--warmup", "3"])
    assert d["value"] > 0 and d["config"]["batch"] == 500 and d["config"]["cuda_graph"] is True
    assert d["eager"]["value"] > 0 and d["iterations_per_s"] > 0 and d["gpu_launches"] > 0
