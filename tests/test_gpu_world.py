"""The B200 groups, GPU collision detection and device snapshot frames driven
together by a World-style loop (core.py:487-500 phase order, restated here for
the test: events -> commands -> step groups -> in-loop detect -> deaths ->
publish).  Checks the reference's event-triggered-death acceptance criterion
(test_acceptance.py:227-265) and a two-type world."""

import struct

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


class MiniWorld:
    """Just enough of World.tick (core.py:487-500) for integration tests."""

    def __init__(self, groups, dt, collision_config=None):
        self.groups = sorted(groups, key=lambda g: g.type_id)
        self.dt, self.tick_count = dt, 0
        self.cfg = collision_config
        self.inbox, self.events, self.pending = [], [], []
        self.group_of = {int(a): g for g in self.groups for a in g.batch.agent_ids}
        self.frames = []
        if collision_config is not None:
            from paper_2308_12698_b200.collision import GpuDetector
            self.detector = GpuDetector(collision_config, self.groups[0].device)

    def apply_events(self):
        for kind, ids in self.pending:
            killed = []
            for g in self.groups:
                killed += g.mark_dead([i for i in ids if self.group_of.get(i) is g])
            if killed:
                self.events.append((self.tick_count, kind, tuple(killed)))
        self.pending = []

    def tick(self):
        self.apply_events()
        rejected = [c.agent_id for c in self.inbox
                    if self.group_of.get(int(c.agent_id)) is None or not self.group_of[int(c.agent_id)].apply_command(c)]
        if rejected:
            self.events.append((self.tick_count, "agent_command_rejected", tuple(rejected)))
        self.inbox = []
        for g in self.groups:
            faults = g.step(self.dt)
            if faults.size:
                self.events.append((self.tick_count, "fault_death", tuple(int(i) for i in faults)))
        if self.cfg is not None:
            rep = self.detector.detect(self.groups, self.tick_count)
            ids = sorted({i for pair in rep.collisions for i in pair})
            if ids:
                self.pending.append(("collision_death", ids))
                self.apply_events()
        from paper_2308_12698_b200.wire import snapshot_frame
        self.frames.append(snapshot_frame(self.tick_count, self.groups))
        self.tick_count += 1


def test_event_triggered_death_head_on():
    from paper_2308_12698_b200 import AgentCommand, B200QuadGroup, CommandLevel, batch_create
    from paper_2308_12698_b200.collision import CollisionConfig
    r_collide = 0.15
    cfg = CollisionConfig(r_collide={0: r_collide}, r_sense=1.0, cell=0.5)
    g = B200QuadGroup(0, batch_create(0, 2, [[-1.5, 0.0, 5.0], [1.5, 0.0, 5.0]]))
    w = MiniWorld([g], dt=2e-3, collision_config=cfg)
    w.inbox = [AgentCommand(0, CommandLevel.POS, (1.5, 0, 5, 0, 0, 0, 0)),
               AgentCommand(1, CommandLevel.POS, (-1.5, 0, 5, 0, 0, 0, 0))]
    overlap_tick = death_tick = None
    alive_hist = []
    for k in range(3000):
        w.tick()
        b = g.batch
        alive_hist.append(int(b.alive.sum()))
        if overlap_tick is None and np.linalg.norm(b.pos[0] - b.pos[1]) < 2 * r_collide:
            overlap_tick = k
        if death_tick is None and not b.alive.any():
            death_tick = k
            break
    assert overlap_tick is not None and death_tick is not None
    assert death_tick <= overlap_tick + 1                           # in-loop detector: no latency
    assert all(b2 <= b1 for b1, b2 in zip(alive_hist, alive_hist[1:]))
    assert w.events[-1][1] == "collision_death" and set(w.events[-1][2]) == {0, 1}
    frozen = g.batch.pos.copy()
    for _ in range(5):
        w.tick()
    np.testing.assert_array_equal(g.batch.pos, frozen)              # dead rows frozen


def test_two_type_world_and_frames():
    from paper_2308_12698_b200 import AgentCommand, B200QuadGroup, CommandLevel, batch_create
    from paper_2308_12698_b200.unicycle import B200UnicycleGroup
    quad = B200QuadGroup(0, batch_create(0, 2, [[0, 0, 5], [3, 0, 5]]))
    uni = B200UnicycleGroup(1, batch_create(1, 2, [[10, 0, 0], [13, 0, 0]], id_base=2))
    w = MiniWorld([quad, uni], dt=0.01)
    w.inbox = [AgentCommand(2, CommandLevel.UNICYCLE, (1.0, 0.0)), AgentCommand(0, CommandLevel.POS, (0, 0, 6, 0, 0, 0, 0)),
               AgentCommand(3, CommandLevel.POS, (0,) * 7)]     # POS to a unicycle -> rejected
    for _ in range(50):
        w.tick()
    assert uni.batch.pos[0, 0] > 10.4 and quad.batch.pos[0, 2] > 5.01   # test_core.py:98-111
    assert ("agent_command_rejected" in [e[1] for e in w.events])
    frame = w.frames[-1]
    length, mtype = struct.unpack_from("<IB", frame, 0)
    assert mtype == 1 and length == len(frame) - 4
    tick = struct.unpack_from("<Q", frame, 5)[0]
    assert tick == 49
    t0, n0 = struct.unpack_from("<HI", frame, 13)
    assert (t0, n0) == (0, 2)
    off = 13 + 6 + 61 * 2
    assert struct.unpack_from("<HI", frame, off) == (1, 2)


def test_groups_stepped_from_worker_threads_bit_identical():
    """World steps its groups on a thread pool (core.py:455-465, SWARMSTEP_THREADS);
    each B200 group owns its stream, so concurrent stepping from worker threads
    gives the same bits as stepping one after the other (test_core.py:314-339)."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    from paper_2308_12698_b200.unicycle import B200UnicycleGroup

    def make():
        rng = np.random.default_rng(4)
        qa = B200QuadGroup(0, batch_create(0, 5000, rng.uniform(-20, 20, (5000, 3))))
        qb = B200QuadGroup(2, batch_create(2, 3000, rng.uniform(-20, 20, (3000, 3)), id_base=10_000))
        uc = B200UnicycleGroup(1, batch_create(1, 700, rng.uniform(-20, 20, (700, 3)), id_base=20_000))
        qa.set_setpoints(np.hstack([rng.uniform(-20, 20, (5000, 3)), np.zeros((5000, 4))]))
        qb.set_setpoints(np.hstack([rng.uniform(-1, 1, (3000, 3)), np.full((3000, 1), 10.0)]), level="rate")
        return [qa, qb, uc]

    seq = make()
    for _ in range(40):
        for g in seq:
            g.step(2e-3)
    par = make()
    with ThreadPoolExecutor(max_workers=3) as ex:
        for _ in range(40):
            list(ex.map(lambda g: g.step(2e-3), par))
    for a, b in zip(seq, par):
        assert a.batch.pos.tobytes() == b.batch.pos.tobytes()
        assert a.batch.quat.tobytes() == b.batch.quat.tobytes()


def test_batch_view_alive_counts_without_state_pull():
    """World.alive_counts (core.py:370) reads batch.alive every tick: the
    B200 batch view answers from the host (exact after collected faults)
    without pulling the float64 state mirror."""
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    g = B200QuadGroup(0, batch_create(0, 1000, np.zeros((1000, 3))))
    g.mark_dead([1, 2, 3])
    g.step(1e-3)
    assert g._state_stale
    assert int(g.batch.alive.sum()) == 997 and g.batch.n == 1000 and g.batch.type_id == 0
    assert g._state_stale                       # no device read so far
    assert g.batch.pos.shape == (1000, 3) and not g._state_stale
    g.step_async(1e-3, 3)                       # uncollected launches: alive comes from the device
    assert int(g.batch.alive.sum()) == 997
    g.collect_faults()


def test_multi_device_group_equals_single_group():
    """MultiDeviceQuadGroup (one logical group, rows sharded over devices of one
    process, launched concurrently) gives the same bits, faults, commands and
    snapshots as one B200QuadGroup.  Run here with two shards on this GPU."""
    import torch

    from paper_2308_12698_b200 import AgentCommand, B200QuadGroup, CommandLevel, batch_create
    from paper_2308_12698_b200.multidevice import MultiDeviceQuadGroup
    rng = np.random.default_rng(8)
    n = 1001
    pos = rng.uniform(-30, 30, (n, 3))

    def drive(g):
        sp = np.hstack([pos + rng_sp.uniform(-2, 2, (n, 3)), np.zeros((n, 3)), rng_sp.uniform(-3, 3, (n, 1))])
        g.set_setpoints(sp)
        g.apply_command(AgentCommand(10, CommandLevel.RATE, (0.1, 0.0, 0.0, 9.0)))
        g.apply_command(AgentCommand(700, CommandLevel.MOTOR, (1e4, 1.1e4, 1e4, 1.1e4)))
        g.mark_dead([3, 600])
        g.add_velocity_overlay(np.full((n, 3), 0.1))
        faults = [g.step(1e-3).tolist()]
        g.retarget_waypoint(pos[900], 0.5)
        faults.append(g.step_k(1e-3, 5).tolist())
        return faults

    rng_sp = np.random.default_rng(1)
    single = B200QuadGroup(0, batch_create(0, n, pos))
    fa = drive(single)
    rng_sp = np.random.default_rng(1)
    multi = MultiDeviceQuadGroup(0, batch_create(0, n, pos), devices=[torch.device("cuda", 0)] * 2)
    fb = drive(multi)
    assert fa == fb
    for q in ("pos", "vel", "quat", "omega", "alive"):
        np.testing.assert_array_equal(getattr(single.batch, q), getattr(multi.batch, q), err_msg=q)
    np.testing.assert_array_equal(single.cmd_values, multi.cmd_values)
    np.testing.assert_array_equal(single.cmd_level, multi.cmd_level)
    assert multi.rows_for(700) == 700 and multi.alive_count() == n - 2
    assert multi.snapshot(5).pos.tobytes() == single.snapshot(5).pos.tobytes()
