"""Fused circle launch vs plain launch on the circle swarm, to profile:
python tools/profile_circle.py AGENTS [K]

3 fused launches (CircleFeed.step_fused(K)) then 3 plain step_async(dt, K)
launches, so ``ncu -k regex:quad_step_pair -s 2 -c 2`` captures the third
fused launch and the first plain one back to back.
"""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

from latency_bench import _B  # noqa: E402
from paper_2308_12698_b200 import B200QuadGroup  # noqa: E402
from paper_2308_12698_b200.feed import CircleFeed  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    g = B200QuadGroup(0, _B(n), device="cuda:0")
    feed = CircleFeed(g, 2e-3)
    for _ in range(3):
        feed.step_fused(k)
    for _ in range(3):
        g.step_async(2e-3, k)
    g.collect_faults()
    torch.cuda.synchronize()
    print(f"profiled n={n} K={k}")


if __name__ == "__main__":
    main()
