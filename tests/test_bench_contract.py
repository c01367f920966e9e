"""bench.py's reference arm on CPU (the driver runs `bench.py --impl reference`
beside the GPU arm): one JSON line with the contract's keys, the same
metric / unit / config naming as the GPU arm, e2e with zero copy bytes, and
under torchrun only rank 0 prints (the other ranks exit 0 without work)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "higher_is_better",
        "dtype", "data", "scaling", "config", "cpu_baseline", "e2e"}


def _lines(out: str) -> list[dict]:
    return [json.loads(x) for x in out.splitlines() if x.strip().startswith("{")]


def test_reference_arm_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--config", "tiny_gpt"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _lines(p.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["metric"] == "train samples/s"
    assert d["unit"] == "samples/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == "tiny_gpt" and d["warmup"] >= 3
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("port", "reference") and cb["cores"] >= 1


def test_reference_arm_under_torchrun_prints_once():
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29581",
                        "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "3", "--config", "tiny_gpt"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _lines(p.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    from paper_2411_01075_b200.configs import CONFIGS     # weak scaling: per-GPU batch x N
    assert lines[0]["config"]["global_batch"] == 2 * CONFIGS["tiny_gpt"].batch_per_gpu
