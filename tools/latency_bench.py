"""Per-tick latency vs swarm size (config 2 shape, the paper's Table I / Fig. 4 metric).

The paper reports "time per round" -- one tick of dynamics
+ control for all N agents -- of 0.845 ms at N = 1,000 (GTX 1660 SUPER,
PyTorch) and "< 2 ms" at N = 10,000.  This measures the same round on a B200
for the circle-tracking swarm (POS level, device circle feed, client.py:55-73)
three ways:
  * graph:  [circle feed -> fused step] x T ticks captured in one CUDA graph
            (device time per tick, CUDA events);
  * eager:  feed.apply() + group.step(dt) per tick through the Python group
            protocol, i.e. what the reference World loop calls (wall time,
            includes the per-tick fault-id readback);
  * kernel: the fused step kernel alone at K = 1 (device time per launch);
  * fused:  CircleFeed.step_fused(10) -- the circle strategy evaluated per
            tick inside the step kernel, 10 ticks per launch (device time per
            tick): the state stays in registers across the ticks;
  * plain:  step_async(dt, 10) on the same swarm without the feed (fixed
            setpoints), the fused feed's own cost by difference.
Writes JSON to argv[1] (default gpurun_out/latency.json).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2308_12698_b200 import B200QuadGroup  # noqa: E402
from paper_2308_12698_b200.feed import CircleFeed, TickGraph  # noqa: E402
from paper_2308_12698_b200.layout import layout_poses  # noqa: E402
from paper_2308_12698_b200.state import yaw_quat  # noqa: E402


class _B:
    def __init__(self, n):
        pos, yaw = layout_poses({"kind": "circle", "radius": 5.0, "z": 10.0}, n)
        self.type_id, self.agent_ids = 0, np.arange(n, dtype=np.uint64)
        self.pos, self.vel, self.quat = pos, np.zeros((n, 3)), yaw_quat(yaw)
        self.omega, self.alive = np.zeros((n, 3)), np.ones(n, dtype=bool)


def ev_ms(fn, reps, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def measure(n: int, dt: float = 2e-3, T: int = 100) -> dict:
    g = B200QuadGroup(0, _B(n), device="cuda:0")
    feed = CircleFeed(g, dt)
    graph = TickGraph(g, dt, T, feed=feed)
    for _ in range(3):
        graph.replay()
    g.collect_faults()
    reps = max(3, min(50, int(2e7 // (n * T)) + 3))
    graph_ms = ev_ms(graph.replay, reps, g.stream) / T
    g.collect_faults()
    # eager: the World-facing path, one Python call per tick incl. fault readback
    for _ in range(20):
        feed.apply()
        g.step(dt)
    ticks = 200 if n <= 100_000 else 30
    t0 = time.perf_counter()
    for _ in range(ticks):
        feed.apply()
        g.step(dt)
    eager_ms = (time.perf_counter() - t0) / ticks * 1e3
    kern_ms = ev_ms(lambda: g.step_async(dt, 1), 50, g.stream)
    g.collect_faults()
    for _ in range(3):
        feed.step_fused(10)
    g.collect_faults()
    fused_ms = ev_ms(lambda: feed.step_fused(10), 20, g.stream) / 10
    g.collect_faults()
    # the same launches without the feed (the commands the fused launches left)
    plain_ms = ev_ms(lambda: g.step_async(dt, 10), 20, g.stream) / 10
    g.collect_faults()
    return {"n": n, "graph_ms_per_tick": graph_ms, "eager_ms_per_tick": eager_ms, "kernel_ms": kern_ms,
            "fused_k10_ms_per_tick": fused_ms, "plain_k10_ms_per_tick": plain_ms,
            "graph_agent_steps_per_s": n / (graph_ms * 1e-3), "alive": int(g.batch.alive.sum())}


def main():
    out = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "latency.json")
    torch.cuda.set_device(0)
    rows = []
    for n in (1_000, 5_000, 10_000, 50_000, 100_000, 300_000, 1_000_000):
        r = measure(n)
        rows.append(r)
        print(json.dumps(r), flush=True)
    rep = {"paper_round_ms_n1000": 0.8452, "paper_hw": "i7-10700 + GTX 1660 SUPER, PyTorch 1.10 (PAPER.md:151)",
           "rows": rows}
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()
