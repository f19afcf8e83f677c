"""Per-tick time vs ticks per launch at fixed N (tuning aid): separates the
per-launch boundary cost (launch gap, first loads, tail wave) from the
per-tick compute.  python tools/kscale.py N [K ...]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import ClockSampler, _Batch  # noqa: E402
from paper_2308_12698_b200 import B200QuadGroup  # noqa: E402
from paper_2308_12698_b200.synthetic import swarm  # noqa: E402

n = int(sys.argv[1])
ks = [int(x) for x in sys.argv[2:]] or [1, 10, 40, 200]
pos, sp = swarm(n)
g = B200QuadGroup(0, _Batch(n, pos, 0), device="cuda:0")
g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
import time  # noqa: E402
out = {"n": n}
clk = ClockSampler(0).start()
t0 = time.perf_counter()
while time.perf_counter() - t0 < 2.0:     # converge past the transient, warm the clocks
    for _ in range(8):
        g.step_async(1e-3, 10)
    g.collect_faults()
for k in ks:
    launches = max(1, 400 // k)
    for _ in range(2):
        g.step_async(1e-3, k)
    g.collect_faults()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(g.stream)
    for _ in range(launches):
        g.step_async(1e-3, k)
    e1.record(g.stream)
    torch.cuda.synchronize()
    g.collect_faults()
    us_tick = e0.elapsed_time(e1) * 1e3 / (launches * k)
    key = f"K{k}" if f"K{k}_us_per_tick" not in out else f"K{k}_again{sum(x.startswith(f'K{k}_') for x in out)}"
    out[f"{key}_us_per_tick"] = us_tick
    out[f"{key}_frac_nominal"] = n * 705 / (us_tick * 1e-6) / 74.45e12
out["clocks"] = clk.stop()
print(json.dumps(out))
