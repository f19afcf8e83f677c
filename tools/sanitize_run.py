"""Exercise every kernel of the library once at small sizes -- for
compute-sanitizer where it is available (it is closed on the GPU pool this
repo was built on), and with PyTorch's caching allocator disabled so that an
out-of-bounds access lands on unmapped memory and faults loudly:

  PYTORCH_NO_CUDA_MEMORY_CACHING=1 python tools/sanitize_run.py
  compute-sanitizer --tool memcheck python tools/sanitize_run.py

Covers: the direct / paired / TMA step kernels at every level (K = 1 and 3,
faults, overlay), the rotor-lag and circle-feed kernels, bookkeeping
kernels, wire packing, swarm stats, neighbour overlay (NCCL-free and P2P
exchange on a 1-rank group), collision detection, the unicycle kernel and
the function-level ops.  Prints "sanitize run ok" at the end.
"""

from __future__ import annotations

import socket
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch.distributed as dist

    from paper_2308_12698_b200 import (AgentCommand, B200QuadGroup, CommandLevel, batch_create,
                                       default_outer_gains, default_quad_params, default_rate_gains, functional)
    from paper_2308_12698_b200.collision import CollisionConfig, GpuDetector
    from paper_2308_12698_b200.feed import CircleFeed, TickGraph
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    from paper_2308_12698_b200.unicycle import B200UnicycleGroup
    from paper_2308_12698_b200.wire import snapshot_frame

    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    n = 300
    pos = rng.uniform(-10, 10, (n, 3))

    def fresh(**kw):
        g = B200QuadGroup(0, batch_create(0, n, pos, vel=rng.uniform(-1, 1, (n, 3))), **kw)
        for i in range(0, n, 3):
            g.apply_command(AgentCommand(i, CommandLevel.RATE, (0.1, -0.2, 0.3, 9.0)))
        for i in range(1, n, 7):
            g.apply_command(AgentCommand(i, CommandLevel.MOTOR, (12000.0, 11000.0, 12500.0, 11800.0)))
        g.mark_dead([5, 6])
        return g

    def inject_fault(g, row=2):
        prev = g.pid_state_dict()["prev_omega"]
        prev[row] = np.nan                      # a NaN D-term sample faults the row next tick
        g.set_pid_state(prev_omega=prev)

    for kern in ("direct", "pair", "tma"):
        g = fresh()
        g.kernel = kern
        g.add_velocity_overlay(rng.uniform(-1, 1, (n, 3)))
        g.step_k(1e-3, 3)
        inject_fault(g)
        g.step_k(1e-3, 3)
        g.step(1e-3)
        g.retarget_waypoint([0.0, 0.0, 0.0], 5.0)
        g.step_k(1e-3, 3)
        g.snapshot(0)
        snapshot_frame(0, [g])
        g.swarm_stats()
    g = fresh(motor_tau=0.03)
    g.step_k(1e-3, 3)
    inject_fault(g, 4)
    g.step_k(1e-3, 3)
    g.motor_thrusts()
    # feeds and graphs
    g = fresh()
    feed = CircleFeed(g, 1e-3)
    for kern in ("direct", "pair"):
        g.kernel = kern
        feed.step_fused(3)
    g.collect_faults()
    TickGraph(g, 1e-3, 4, feed=feed).replay()
    g.collect_faults()
    # neighbours: NCCL-free path and the P2P exchange (1-rank group)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    for ex in ("nccl", "p2p"):
        g = fresh()
        ns = NeighborSeparation(g, make_shard(n), r_sense=2.0, k_sep=1.0, exchange=ex)
        ns.step(1e-3)
        ns.step(1e-3)
    dist.destroy_process_group()
    # collision detection over two types
    q = fresh()
    u = B200UnicycleGroup(1, batch_create(1, 50, rng.uniform(-10, 10, (50, 3)), id_base=n))
    u.apply_command(AgentCommand(n + 1, CommandLevel.UNICYCLE, (1.0, 0.5)))
    u.step(1e-2)
    rep = GpuDetector(CollisionConfig(r_collide={0: 0.3, 1: 0.5}, r_sense=2.0, cell=2.0), q.device).detect([q, u], 0)
    len(rep.neighbor_sets)
    # function-level ops
    P = default_quad_params()
    b = batch_create(0, n, pos)
    fc, tau = rng.uniform(0, 30, n), rng.uniform(-0.1, 0.1, (n, 3))
    functional.dynamics_deriv(b, fc, tau, P)
    functional.rk4_step(b, fc, tau, P, 1e-3)
    functional.mix_to_motors(fc, tau, P)
    functional.rotor_thrust_torque(rng.uniform(0, 4e4, (n, 4)), P)
    st = functional.RatePidState(n)
    functional.rate_pid_step(b.omega, functional.RateSetpoint(rng.uniform(-1, 1, (n, 3)), fc), default_rate_gains(),
                             1e-3, st, b.alive)
    functional.position_outer_loop(b.pos, b.vel, b.quat, b.alive,
                                   functional.PosSetpoint(pos + 1.0, np.zeros((n, 3)), np.zeros(n)), P,
                                   default_outer_gains())
    torch.cuda.synchronize()
    print("sanitize run ok", flush=True)


if __name__ == "__main__":
    main()
