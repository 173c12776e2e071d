"""bench.py's reference arm runs here (CPU only: the oracle port on a small
sample) and prints the one JSON line the driver parses, with the keys the
contract asks for; under torchrun only rank 0 prints."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] +
                         args, cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0",
              "--cpu-n", "48"])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps",
                "warmup", "ms_per_step", "higher_is_better", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1
    assert cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"],
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_uses_all_threads_under_torchrun_env():
    # torchrun sets OMP_NUM_THREADS=1 per rank; the baseline still uses every
    # host thread of its process
    env = dict(os.environ, OMP_NUM_THREADS="1")
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0",
              "--cpu-n", "48"], env=env)
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
