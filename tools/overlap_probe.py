"""Probe (tuning aid): does overlapping consecutive launches help at 1M agents?
One 1M-agent group vs two 500k groups on their own streams launched
alternately (their launches overlap), K = 10 ticks per launch, same total work."""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import _Batch  # noqa: E402
from paper_2308_12698_b200 import B200QuadGroup  # noqa: E402
from paper_2308_12698_b200.synthetic import swarm  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
K, L = 10, 60
out = {}
for parts in (1, 2, 4):
    groups = []
    for i in range(parts):
        lo, hi = i * N // parts, (i + 1) * N // parts
        pos, sp = swarm(N, lo, hi)
        g = B200QuadGroup(0, _Batch(hi - lo, pos, lo), device="cuda:0")
        g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
        groups.append(g)
    for _ in range(5):
        for g in groups:
            g.step_async(1e-3, K)
    for g in groups:
        g.collect_faults()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for g in groups:
        g.stream.wait_event(e0)
    for _ in range(L):
        for g in groups:
            g.step_async(1e-3, K)
    for g in groups:
        torch.cuda.current_stream().wait_stream(g.stream)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    for g in groups:
        g.collect_faults()
    us_tick = e0.elapsed_time(e1) * 1e3 / (L * K)
    out[f"parts{parts}_us_per_tick"] = us_tick
    out[f"parts{parts}_frac_nominal"] = N * 705 / (us_tick * 1e-6) / 74.45e12
    del groups
    torch.cuda.empty_cache()
print(json.dumps(out))
