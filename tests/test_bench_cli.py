"""bench.py's reference arm (CPU only: the reference's own QuadGroup.step from
oracle/_ref, sharded over the host cores, with the float64 C port beside it)
keeps the driver's JSON contract, and under torchrun only rank 0 prints (the
other ranks exit 0 without work)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                           "--warmup", "1", "--substeps", "1", "--agents", "40000", "--cpu-seconds", "0.3"], capture_output=True, text=True, env=env,
                          timeout=600)


def test_reference_arm_json_line():
    p = _run({})
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["value"] == line["value"] and cb["cores"] >= 1 and cb["kind"] in ("port", "reference") and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "workload" in line["config"] and line["config"]["agents_total"] == 40000
    from oracle import ref_runner
    if ref_runner.available():
        # the reference itself, on the whole swarm, with the port beside it
        assert cb["kind"] == "reference" and cb["agents"] == 40000 and len(cb["ms_per_sample"]) == 2
        assert line["port"]["kind"] == "port" and line["port"]["value"] > 0
        assert line["scaling"] == "strong"


def test_reference_arm_non_zero_rank_is_silent():
    p = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip() == ""
