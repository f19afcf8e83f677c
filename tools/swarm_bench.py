"""Config 5: neighbour-coupled swarm, per-tick cost on one B200 (and per rank
under torchrun).  100k quadrotors per GPU in a box at ~1 agent / 8 m^3, r_sense
2 m, POS level holding their start positions; every tick: pack positions ->
all-gather (NCCL or the fused P2P exchange) -> spatial hash + counting sort + 27-cell scan ->
separation overlay -> fused step (K = 1).  Prints one JSON line (rank 0).

  python tools/swarm_bench.py [agents_per_gpu] [ticks] [nccl|p2p]
  torchrun --nproc-per-node N tools/swarm_bench.py ...

p2p = the position exchange fused into the pack kernel over peer memory
(csrc/exchange.cu; needs a process group even at world 1).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2308_12698_b200 import B200QuadGroup  # noqa: E402
from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard  # noqa: E402


class _B:
    def __init__(self, pos, id_base):
        n = pos.shape[0]
        self.type_id, self.agent_ids = 0, np.arange(id_base, id_base + n, dtype=np.uint64)
        self.pos, self.vel = pos, np.zeros((n, 3))
        self.quat = np.tile([1.0, 0, 0, 0], (n, 1))
        self.omega, self.alive = np.zeros((n, 3)), np.ones(n, dtype=bool)


def main():
    n_per = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    ticks = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    exchange = sys.argv[3] if len(sys.argv) > 3 else "nccl"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1 or exchange == "p2p":
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29555", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
    n_total = n_per * world
    shard = make_shard(n_total, rank, world)
    side = (8.0 * n_total) ** (1 / 3)                   # ~8 m^3 per agent
    rng = np.random.default_rng(1234)
    pos_all = rng.uniform(0, side, (n_total, 3)) + [0, 0, 10]
    g = B200QuadGroup(0, _B(pos_all[shard.lo:shard.hi], shard.lo), device=f"cuda:{local}")
    ns = NeighborSeparation(g, shard, r_sense=2.0, k_sep=0.5, process_group=pg, exchange=exchange)
    for _ in range(10):
        ns.step(1e-3)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    # (a) device time of the exchange + overlay + step chain, CUDA events
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(g.stream)
    for _ in range(ticks):
        ns.apply()
        g.step_async(1e-3, 1)
    e1.record(g.stream)
    torch.cuda.synchronize()
    g.collect_faults()
    dev_ms = e0.elapsed_time(e1) / ticks
    # (b) the same through the group protocol with the per-tick fault readback
    t0 = time.perf_counter()
    for _ in range(ticks):
        ns.step(1e-3)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) / ticks * 1e3
    graph_ms = float("nan")
    if world == 1 or exchange == "p2p":
        # (c) the whole tick chain captured as CUDA graphs of 50 ticks
        from paper_2308_12698_b200.feed import TickGraph
        tg = TickGraph(g, 1e-3, 50, coupling=ns)
        tg.replay()
        g.collect_faults()
        torch.cuda.synchronize()
        e0.record(g.stream)
        reps = max(1, ticks // 50)
        for _ in range(reps):
            tg.replay()
        e1.record(g.stream)
        torch.cuda.synchronize()
        g.collect_faults()
        graph_ms = e0.elapsed_time(e1) / (reps * 50)
    vals = torch.tensor([dev_ms, wall_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"config": "cfg5 neighbour-coupled swarm", "agents_total": n_total, "world": world,
                          "exchange": exchange,
                          "r_sense": 2.0, "ticks": ticks, "device_ms_per_tick": float(vals[0]),
                          "wall_ms_per_tick": float(vals[1]), "graph_ms_per_tick": graph_ms,
                          "agent_steps_per_s_device": n_total / (float(vals[0]) * 1e-3),
                          "alive": int(g.batch.alive.sum())}), flush=True)
    if torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
