"""Wall time of the World-facing per-tick call, B200QuadGroup.step(dt)
(launch + fault-id readback), for small groups where the host path dominates.

  python tools/step_overhead.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_12698_b200 import B200QuadGroup, batch_create  # noqa: E402

out = {}
for n in (1_000, 10_000):
    g = B200QuadGroup(0, batch_create(0, n, np.random.default_rng(0).uniform(-5, 5, (n, 3))))
    for _ in range(200):
        g.step(1e-3)
    t0 = time.perf_counter()
    for _ in range(2000):
        g.step(1e-3)
    out[f"step_us_n{n}"] = (time.perf_counter() - t0) / 2000 * 1e6
print(json.dumps(out))
