"""Single-core timing of the REFERENCE's own `QuadGroup.step` (numpy float64,
core.py:166-202) beside the float64 C oracle port that bench.py's reference arm
and cpu_baseline time on the GPU box (the Python reference cannot travel there).
Build container only: imports swarmstep from /root/reference/pkg/src.

  OMP_NUM_THREADS=1 python tools/ref_vs_port.py [agents] [ticks]

Workload = bench.py's (POS level, random setpoints p0 + U(-1,1)^3, yaw U(-pi,pi),
grid layout, dt 1e-3).  Prints one JSON line.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(v, "1")

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from swarmstep.core import QuadGroup  # noqa: E402
from swarmstep.quad import default_quad_params  # noqa: E402
from swarmstep.state import batch_create as ref_batch_create  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2308_12698_b200.layout import layout_poses  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    ticks = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    dt = 1e-3
    pos, _ = layout_poses({"kind": "grid", "spacing": 3.0, "origin": (0.0, 0.0, 10.0)}, n)
    rng = np.random.default_rng(0)
    sp = np.zeros((n, 7))
    sp[:, :3] = pos + rng.uniform(-1, 1, (n, 3))
    sp[:, 6] = rng.uniform(-np.pi, np.pi, n)

    ref = QuadGroup(0, ref_batch_create(0, n, pos), default_quad_params())
    ref.cmd_values[:] = sp
    ref.step(dt)                                       # warm
    t0 = time.perf_counter()
    for _ in range(ticks):
        ref.step(dt)
    t_ref = time.perf_counter() - t0

    port = orc.OracleGroup(0, ref_batch_create(0, n, pos))
    port.cmd_values[:] = sp
    port.step(dt, nthreads=1)
    t0 = time.perf_counter()
    for _ in range(ticks):
        port.step(dt, nthreads=1)
    t_port = time.perf_counter() - t0
    drift = float(np.max(np.abs(ref.batch.pos - port.state13()[:, :3])))
    print(json.dumps({
        "what": "single-core agent-steps/s, reference numpy QuadGroup.step vs float64 C oracle port",
        "agents": n, "ticks": ticks, "level": "POS", "host": "build container (no GPU), 1 thread",
        "reference_agent_steps_per_s": n * ticks / t_ref, "port_agent_steps_per_s": n * ticks / t_port,
        "port_over_reference": t_ref / t_port, "max_abs_pos_difference_m": drift}))


if __name__ == "__main__":
    main()
