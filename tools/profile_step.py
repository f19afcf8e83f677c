"""One fused-step launch to profile: python tools/profile_step.py K AGENTS

Runs 3 warm-up launches then exactly one more launch of the step kernel, so
``ncu -k regex:quad_step -s 3 -c 1`` captures a steady-state launch.
"""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from bench import _Batch  # noqa: E402
from paper_2308_12698_b200.synthetic import swarm as workload  # noqa: E402
from paper_2308_12698_b200 import B200QuadGroup  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
    pos, sp = workload(n)
    g = B200QuadGroup(0, _Batch(n, pos, 0), device="cuda:0")
    g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
    for _ in range(4):
        g.step_async(1e-3, k)
    g.collect_faults()
    torch.cuda.synchronize()
    print(f"profiled K={k} n={n}")


if __name__ == "__main__":
    main()
