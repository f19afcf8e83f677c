"""The sharded multi-GPU code paths executed over REAL B200 groups, checked bit
for bit against one group holding the whole swarm:

* one process per rank (torch.distributed, world size 2): ``ShardedSwarm``
  (index routing, collective-free stepping, fault ids gathered at collect
  time) plus ``NeighborSeparation`` (config 5: per-tick position all-gather
  -> separation overlay) -- both ranks on this one GPU, exchanging through
  the host-staged gloo transport, so no kernel waits on another rank's;
* one process driving several shards (``MultiDeviceQuadGroup`` +
  ``MultiDeviceNeighborSeparation``, the drop-in for the single-process
  World), its pack kernels storing into every shard's gathered buffer
  (csrc/exchange.cu pack_scatter), here with both shards on this GPU.

Overlays sum in fixed point and rows are independent, so the sharded runs
must reproduce the world-1 run exactly: overlays, trajectories, PID state,
fault ids and their ticks."""

import os
import socket

import numpy as np
import pytest

from paper_2308_12698_b200._lib import COL_OVERLAY

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

N, TICKS, DT, R_SENSE, K_SEP = 3001, 12, 2e-3, 2.0, 1.5
FAULT_TICK, FAULT_IDS = 4, (17, 2400)        # one agent on each rank's shard


def _swarm():
    """A dense swarm (neighbours within r_sense everywhere) at POS hold."""
    rng = np.random.default_rng(11)
    pos = rng.uniform(0.0, 14.0, (N, 3)) + [0.0, 0.0, 5.0]
    vel = rng.uniform(-0.5, 0.5, (N, 3))
    omega = rng.uniform(-0.2, 0.2, (N, 3))
    return pos, vel, omega


def _group(lo, hi):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    pos, vel, omega = _swarm()
    b = batch_create(0, hi - lo, pos[lo:hi], vel=vel[lo:hi], omega=omega[lo:hi], id_base=lo)
    return B200QuadGroup(0, b, device="cuda:0")


def _inject_fault(g, ids):
    """A zero quaternion (edited into the host mirror and pushed) faults the
    row at the next tick: its renormalisation has a zero norm (quad.py:404-430)."""
    rows = [g.rows_for(a) for a in ids if g.rows_for(a) is not None]
    if rows:
        g.batch.quat[rows] = 0.0
        g.push_host_state()


def _state(g):
    b = g.batch
    ps = g.pid_state_dict()
    return dict(pos=b.pos.copy(), vel=b.vel.copy(), quat=b.quat.copy(), omega=b.omega.copy(),
                alive=b.alive.copy(), integral=ps["integral"], prev=ps["prev_omega"])


def _overlay(g):
    return g.column_block(COL_OVERLAY, COL_OVERLAY + 3).cpu().numpy()


def _run(g, coupling, step, collect):
    """TICKS coupled ticks; overlays of ticks 0 and TICKS-1, faults per tick."""
    overlays, faults = [], []
    for t in range(TICKS):
        if t == FAULT_TICK:
            _inject_fault(g if not hasattr(g, "shards") else g.shards[0], FAULT_IDS)
            if hasattr(g, "shards"):
                _inject_fault(g.shards[1], FAULT_IDS)
        coupling.apply()
        if t in (0, TICKS - 1):
            overlays.append(np.concatenate([_overlay(s) for s in getattr(g, "shards", [g])]))
        faults.append(step(t))
    return overlays, collect(faults)


def _world1():
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    g = _group(0, N)
    ns = NeighborSeparation(g, make_shard(N), r_sense=R_SENSE, k_sep=K_SEP)
    overlays, faults = _run(g, ns, lambda t: g.step(DT),
                            lambda f: [(t, ids.tolist()) for t, ids in enumerate(f) if len(ids)])
    return overlays, faults, _state(g)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2308_12698_b200.parallel import NeighborSeparation, ShardedSwarm, make_shard
        torch.cuda.set_device(0)
        shard = make_shard(N, rank, world)
        g = _group(shard.lo, shard.hi)
        sw = ShardedSwarm(g, shard)
        ns = NeighborSeparation(g, shard, r_sense=R_SENSE, k_sep=K_SEP, exchange="host")
        # commands route by owner: every rank sees all, exactly one applies each
        from paper_2308_12698_b200 import AgentCommand, CommandLevel
        answers = [sw.apply_command(AgentCommand(a, CommandLevel.POS, (0.0, 0.0, 5.0, 0, 0, 0, 0.0)))
                   for a in (0, N - 1, 10 ** 9)]
        overlays, faults = _run(g, ns, lambda t: sw.step(DT),
                                lambda f: [(t, ids.tolist()) for t, ids in sw.collect()])
        q.put((rank, shard.lo, shard.hi, overlays, faults, _state(g), answers, None))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, 0, 0, None, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_ranks_sharded_swarm_with_neighbour_exchange_equal_world_one():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert o[7] is None, o[7]
    # the world-1 run, with the same commands (routing applied them once)
    from paper_2308_12698_b200 import AgentCommand, CommandLevel  # noqa: F401
    ov1, f1, st1 = _world1_with_commands()
    lo_hi = [(o[1], o[2]) for o in out]
    assert lo_hi == [(0, 1501), (1501, N)]
    for k in range(2):
        ov2 = np.concatenate([o[3][k] for o in out])
        np.testing.assert_array_equal(ov2, ov1[k])
    assert np.abs(ov1[0]).sum() > 0
    # fault ids with their ticks: every rank reports the whole swarm's
    assert out[0][4] == out[1][4] == f1 == [(FAULT_TICK, list(FAULT_IDS))]
    for key in st1:
        got = np.concatenate([o[5][key] for o in out])
        np.testing.assert_array_equal(got, st1[key], err_msg=key)
    # routing answers: True from the owner, None elsewhere; unknown id nowhere
    assert out[0][6] == [True, None, None] and out[1][6] == [None, True, None]


def _world1_with_commands():
    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    g = _group(0, N)
    for a in (0, N - 1):
        assert g.apply_command(AgentCommand(a, CommandLevel.POS, (0.0, 0.0, 5.0, 0, 0, 0, 0.0)))
    ns = NeighborSeparation(g, make_shard(N), r_sense=R_SENSE, k_sep=K_SEP)
    overlays, faults = _run(g, ns, lambda t: g.step(DT),
                            lambda f: [(t, ids.tolist()) for t, ids in enumerate(f) if len(ids)])
    return overlays, faults, _state(g)


def test_single_process_multi_shard_exchange_equals_one_group():
    from paper_2308_12698_b200 import batch_create
    from paper_2308_12698_b200.multidevice import MultiDeviceNeighborSeparation, MultiDeviceQuadGroup
    ov1, f1, st1 = _world1()
    pos, vel, omega = _swarm()
    mg = MultiDeviceQuadGroup(0, batch_create(0, N, pos, vel=vel, omega=omega), devices=["cuda:0", "cuda:0"])
    ns = MultiDeviceNeighborSeparation(mg, r_sense=R_SENSE, k_sep=K_SEP)
    overlays, faults = _run(mg, ns, lambda t: mg.step(DT),
                            lambda f: [(t, ids.tolist()) for t, ids in enumerate(f) if len(ids)])
    for k in range(2):
        np.testing.assert_array_equal(overlays[k], ov1[k])
    assert faults == f1 == [(FAULT_TICK, list(FAULT_IDS))]
    st = {k: np.concatenate([_state(s)[k] for s in mg.shards]) for k in st1}
    for key in st1:
        np.testing.assert_array_equal(st[key], st1[key], err_msg=key)
    # the gathered buffer holds the whole swarm (padding rows NaN)
    gp = ns.gathered_positions(1).cpu().numpy()
    assert np.isnan(gp[:, 0]).sum() == ns.n_all - int(mg.batch.alive.sum())
