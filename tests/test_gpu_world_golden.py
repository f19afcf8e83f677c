"""The B200 groups inside a World loop, against a recording of the reference's
own ``World`` (tests/golden/world.npz, made by tests/golden/make_golden.py
gen_world from core.py:308-505 with QuadGroup + UnicycleGroup, in-loop
collision detection, commands of every level and viewer inputs of every mode).

``ReplayWorld`` restates World.tick's phase order (core.py:486-500) and the
inbox / event handling (core.py:392-453) around the B200 groups, the GPU
detector and the device viewer influence.  The event log (rejections with
their ids, the collision death tick and ids) must match exactly; the float64
state every 20 ticks within float32 trajectory tolerance."""

import json

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

# float32 state vs the float64 reference after up to 300 ticks of closed-loop
# flight (per-step parity is 1e-5 relative; this bounds the accumulated drift)
TOL = dict(pos=2e-6, vel=2e-5, quat=5e-6, omega=1e-4)   # measured: 1.5e-7, 1.6e-6, 4.1e-7, 8.3e-6


class ReplayWorld:
    def __init__(self, groups, dt, collision_config):
        from paper_2308_12698_b200.collision import GpuDetector
        self.groups = sorted(groups, key=lambda g: g.type_id)
        self.group_of = {int(a): g for g in self.groups for a in g.batch.agent_ids}
        self.dt, self.tick_no = dt, 0
        self.inbox, self.pending, self.event_log = [], [], []
        self.detector = GpuDetector(collision_config, self.groups[0].device)

    def _apply_events(self):                                   # core.py:411-425
        for tick, kind, ids in self.pending:
            killed = []
            for g in self.groups:
                mine = [a for a in ids if self.group_of.get(a) is g]
                if mine:
                    killed += g.mark_dead(mine)
            if killed:
                self.event_log.append([tick, kind, [int(a) for a in killed]])
        self.pending = []

    def _apply_inbox(self):                                    # core.py:427-443
        rejected = []
        for item in self.inbox:
            if hasattr(item, "agent_id"):
                g = self.group_of.get(int(item.agent_id))
                if g is None or not g.apply_command(item):
                    rejected.append(int(item.agent_id))
            else:
                for g in self.groups:                          # core.py:445-453, on the device
                    g.apply_viewer_input(item)
        self.inbox = []
        if rejected:
            self.event_log.append([self.tick_no, "agent_command_rejected", rejected])

    def tick(self):                                            # core.py:486-500
        self._apply_events()
        self._apply_inbox()
        for g in self.groups:
            faults = g.step(self.dt)
            if faults.size:
                self.event_log.append([self.tick_no, "fault_death", [int(i) for i in faults]])
        rep = self.detector.detect(self.groups, self.tick_no)
        ids = sorted({i for pair in rep.collisions for i in pair})
        if ids:
            self.pending.append((self.tick_no, "collision_death", ids))
        self._apply_events()
        self.tick_no += 1


def test_world_replay_matches_reference_world():
    from golden_io import GOLDEN
    from paper_2308_12698_b200 import (AgentCommand, B200QuadGroup, B200UnicycleGroup, CommandLevel,
                                       InfluenceMode, ViewerInputMsg, batch_create)
    from paper_2308_12698_b200.collision import CollisionConfig

    z = dict(np.load(GOLDEN / "world.npz"))
    script = json.loads(str(z["script"]))
    want_events = json.loads(str(z["events"]))
    qpos, upos = z["qpos"], z["upos"]
    n_q, n_u, dt, ticks = qpos.shape[0], upos.shape[0], float(z["dt"]), int(z["ticks"])
    quads = B200QuadGroup(0, batch_create(0, n_q, qpos))
    unis = B200UnicycleGroup(1, batch_create(1, n_u, upos, id_base=n_q))
    cfg = CollisionConfig(r_collide={0: 0.2, 1: 0.3}, r_sense=1.2, cell=1.2)
    w = ReplayWorld([quads, unis], dt, cfg)
    checked = 0
    worst = dict.fromkeys(TOL, 0.0)
    for t in range(ticks):
        for item in script.get(str(t), []):
            if item[0] == "cmd":
                w.inbox.append(AgentCommand(item[1], CommandLevel(item[2]), tuple(item[3])))
            else:
                w.inbox.append(ViewerInputMsg(InfluenceMode(item[1]), tuple(item[2]), item[3], item[4]))
        w.tick()
        if (t + 1) % 20 == 0:
            for g in w.groups:
                b = g.batch
                np.testing.assert_array_equal(b.alive, z[f"t{t}_g{g.type_id}_alive"], err_msg=f"tick {t}")
                for k, tol in TOL.items():
                    got, ref = getattr(b, k), z[f"t{t}_g{g.type_id}_{k}"]
                    err = float(np.max(np.abs(got - ref)))
                    worst[k] = max(worst[k], err)
                    assert err <= tol, f"tick {t} type {g.type_id} {k}: {err:.2e} > {tol:.0e}"
            checked += 1
    print("world replay max |err|:", worst)
    assert checked == ticks // 20
    assert w.event_log == want_events
    assert any(e[1] == "collision_death" for e in want_events)
