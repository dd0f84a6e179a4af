"""bench.py's GPU arm end to end on a small config (C1): the JSON line carries the contract keys and the
extra objects (roofline, roofline_cg_step, matrix_free, batched_alpha, e2e, clocks)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpu_arm_runs_and_reports():
    r = subprocess.run([sys.executable, "bench.py", "--config", "C1", "--steps", "2", "--warmup", "3",
                        "--no-cpu-baseline", "--e2e-steps", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "roofline_cg_step", "matrix_free",
              "batched_alpha", "e2e", "gpu_launches", "clocks", "status"):
        assert k in line, k
    assert line["status"] == 0 and line["value"] > 0 and line["gpu_launches"] > 0
    assert line["roofline"]["achieved"] > 0 and 0 < line["roofline"]["frac"]
    assert line["matrix_free"]["status"] == 0 and line["matrix_free"]["variant"] == 5
    assert line["batched_alpha"]["seconds"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
