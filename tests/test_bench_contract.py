"""bench.py keeps the driver's JSON contract: the reference arm on CPU, the
B200 arm on the GPU (small sizes)."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    line = _run(["--impl", "reference", "--size", "400", "--steps", "1", "--warmup", "1", "--cpu-blocks", "2"])
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert {"workload", "n", "b", "tau", "seed", "parallelism", "l2"} <= set(line["config"])
    assert line["config"]["n"] == 400 and line["config"]["workload"].startswith("cfg2:")


@pytest.mark.gpu
def test_b200_arm_contract():
    line = _run(["--size", "1500", "--steps", "1", "--warmup", "3", "--e2e-steps", "1", "--cpu-blocks", "2"])
    assert BASE_KEYS <= set(line)
    assert {"roofline", "cpu_baseline", "gpu_launches", "clocks"} <= set(line)
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] <= 1.05 and r["peak"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["result"]["status"] in ("ok", "not_converged", "rank_exhausted")
    # the reference arm names the same workload (the driver compares the two lines' config)
    ref = _run(["--impl", "reference", "--size", "1500", "--steps", "1", "--warmup", "1", "--cpu-blocks", "2"])
    assert ref["config"] == line["config"]
