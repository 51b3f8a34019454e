"""bench.py contract parts that need no GPU: the reference arm (the fp64 oracle on a bounded
sample) reports the same metric, unit and workload string as our arm, and under a 2-rank
launch only rank 0 prints a line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _lines(out):
    return [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_line_on_cpu():
    import bench
    from paper_2603_00413_b200 import scenes as S
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "2",
                          "--warmup", "1", "--ref-pixels", "8"], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    (d,) = _lines(out)
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["higher_is_better"] is True
    assert d["config"]["workload"] == bench.workload_name("C1", S.config_c1(), False)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_two_ranks_rank0_only():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--impl", "reference",
                          "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "1", "--ref-pixels", "4"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    (d,) = _lines(out)
    assert d["impl"] == "reference" and d["n_gpus"] == 2
