"""bench.py's B200 arm at a small size keeps the driver's JSON contract:
roofline with traffic, cpu_baseline, an end-to-end number with real host
copies, clocks sampled during the timed region and a launch count."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]
ROOT = Path(__file__).resolve().parent.parent


def test_bench_line_contract():
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--agents", "200000", "--steps", "4", "--warmup", "3",
                        "--cpu-seconds", "1", "--cpu-samples", "2"], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ))
    assert p.returncode == 0, p.stderr[-3000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
                "gpu_launches"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["scaling"] == "strong"
    assert d["value"] > 0 and d["config"]["agents_total"] == 200000
    r = d["roofline"]
    assert r["bound"] in ("fp32", "hbm", "tensor") and 0 < r["frac"] <= 1.0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    assert abs(r["frac_nominal"] - r["achieved"] / r["peak_nominal"]) < 1e-9
    k1 = d["roofline_k1"]
    assert k1["bytes_per_agent"] == 182 and abs(k1["frac"] - k1["achieved"] / k1["peak"]) < 1e-9
    from oracle import ref_runner
    if ref_runner.available():       # oracle/_ref travelled with the snapshot
        assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["port"]["kind"] == "port"
    assert d["gpu_launches"] >= d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_bench_two_rank_plumbing():
    """The torchrun path (one JSON line from rank 0, whole-job value, max over
    ranks, cfg4's strong split of one swarm, cpu_baseline on the N > 1 line),
    exercised with the gloo plumbing backend: both ranks share this GPU, so
    the number is not a measurement -- only the contract is checked."""
    env = dict(os.environ, SWARMSTEP_BENCH_BACKEND="gloo")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", str(ROOT / "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--cpu-samples", "1", "--cpu-seconds", "0.3",
                        "--no-k1"], capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    # the default workload is cfg4: 10M agents in total, split over the ranks
    assert d["n_gpus"] == 2 and d["config"]["agents_total"] == 10_000_000 and d["scaling"] == "strong"
    assert d["config"]["agents_per_gpu"] == 5_000_000
    assert d["value"] > 0 and d["cpu_baseline"]["value"] > 0
