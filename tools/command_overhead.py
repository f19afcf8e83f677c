"""Host cost of the per-agent command path the reference World drives
(core.py:427-443): B200QuadGroup.apply_command for every agent of a 5,000-agent
group (config 2 size), then the batched device scatter at the next step.

  python tools/command_overhead.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2308_12698_b200 import AgentCommand, B200QuadGroup, CommandLevel, batch_create  # noqa: E402

n = 5000
pos = np.random.default_rng(0).uniform(-5, 5, (n, 3))
g = B200QuadGroup(0, batch_create(0, n, pos))
cmds = [AgentCommand(i, CommandLevel.POS, tuple(pos[i]) + (0.0, 0.0, 0.0, 0.1)) for i in range(n)]
for _ in range(3):
    for c in cmds:
        g.apply_command(c)
    g.step(1e-3)
reps = 20
t_apply = t_step = 0.0
for _ in range(reps):
    t0 = time.perf_counter()
    for c in cmds:
        g.apply_command(c)
    t1 = time.perf_counter()
    g.step(1e-3)
    t2 = time.perf_counter()
    t_apply += t1 - t0
    t_step += t2 - t1
print(json.dumps({"n": n, "apply_command_us_per_call": t_apply / reps / n * 1e6,
                  "apply_all_ms": t_apply / reps * 1e3, "step_with_scatter_ms": t_step / reps * 1e3}))
