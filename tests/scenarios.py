"""Deterministic group scenarios shared by the golden generator and the tests.

A scenario is an initial state plus a script of World-style inputs applied
before given ticks, in World.tick's order (core.py:487-500): deaths
(``_apply_events``) -> commands (``_apply_inbox``) -> waypoint retargets ->
velocity overlays -> ``step(dt)``.  ``run_script`` drives any object with the
reference group protocol (the reference ``QuadGroup``, the float64 oracle
twin, or the B200 group) and records state after chosen ticks.

Pure numpy: importable on the GPU box where /root/reference is absent.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

LEVEL_NAMES = {0: "pos", 1: "rate", 2: "motor", 3: "unicycle"}
HOVER = 1.0 * 9.81


@dataclass
class Scenario:
    name: str
    n: int
    dt: float
    ticks: int
    pos: np.ndarray
    vel: np.ndarray
    quat: np.ndarray
    omega: np.ndarray
    record: list
    cmds: list = field(default_factory=list)       # (tick, agent_id, level_code, values tuple)
    deaths: list = field(default_factory=list)     # (tick, [ids])
    waypoints: list = field(default_factory=list)  # (tick, point(3,), radius)
    overlays: list = field(default_factory=list)   # (tick, offsets (n,3))

    # ---- npz (de)serialisation ----------------------------------------
    def to_arrays(self) -> dict:
        out = dict(name=np.array(self.name), n=np.array(self.n), dt=np.array(self.dt),
                   ticks=np.array(self.ticks), pos=self.pos, vel=self.vel, quat=self.quat,
                   omega=self.omega, record=np.array(self.record, dtype=np.int64))
        m = len(self.cmds)
        out["cmd_tick"] = np.array([c[0] for c in self.cmds], dtype=np.int64).reshape(m)
        out["cmd_id"] = np.array([c[1] for c in self.cmds], dtype=np.int64).reshape(m)
        out["cmd_level"] = np.array([c[2] for c in self.cmds], dtype=np.int64).reshape(m)
        vals = np.zeros((m, 7))
        nv = np.zeros(m, dtype=np.int64)
        for i, c in enumerate(self.cmds):
            vals[i, :len(c[3])] = c[3]
            nv[i] = len(c[3])
        out["cmd_vals"], out["cmd_nvals"] = vals, nv
        out["dead_tick"] = np.array([d[0] for d in self.deaths for _ in d[1]], dtype=np.int64)
        out["dead_id"] = np.array([i for d in self.deaths for i in d[1]], dtype=np.int64)
        out["wp_tick"] = np.array([w[0] for w in self.waypoints], dtype=np.int64)
        out["wp_point"] = np.array([w[1] for w in self.waypoints], dtype=float).reshape(-1, 3)
        out["wp_radius"] = np.array([w[2] for w in self.waypoints], dtype=float)
        out["ov_tick"] = np.array([o[0] for o in self.overlays], dtype=np.int64)
        out["ov_vals"] = np.array([o[1] for o in self.overlays], dtype=float).reshape(-1, self.n, 3)
        return out

    @staticmethod
    def from_arrays(z) -> "Scenario":
        n = int(z["n"])
        cmds = [(int(t), int(a), int(l), tuple(float(x) for x in v[:k]))
                for t, a, l, v, k in zip(z["cmd_tick"], z["cmd_id"], z["cmd_level"], z["cmd_vals"], z["cmd_nvals"])]
        deaths = {}
        for t, a in zip(z["dead_tick"], z["dead_id"]):
            deaths.setdefault(int(t), []).append(int(a))
        return Scenario(name=str(z["name"]), n=n, dt=float(z["dt"]), ticks=int(z["ticks"]),
                        pos=z["pos"], vel=z["vel"], quat=z["quat"], omega=z["omega"],
                        record=[int(r) for r in z["record"]], cmds=cmds,
                        deaths=sorted(deaths.items()),
                        waypoints=[(int(t), p, float(r)) for t, p, r in zip(z["wp_tick"], z["wp_point"], z["wp_radius"])],
                        overlays=[(int(t), v) for t, v in zip(z["ov_tick"], z["ov_vals"])])


class _Cmd:
    """Minimal command object (agent_id, level, values) with a string level."""

    def __init__(self, agent_id, level, values):
        self.agent_id, self.level, self.values = agent_id, level, values


def default_make_cmd(agent_id, level_code, values):
    return _Cmd(agent_id, LEVEL_NAMES[level_code], tuple(values))


def run_script(group, sc: Scenario, make_cmd=default_make_cmd, state_of=None, on_tick=None):
    """Replay ``sc`` on ``group``.  Returns (records, cmd_ok, faults_by_tick).

    ``state_of(group)`` must return a dict of float64 arrays to record;
    faults_by_tick maps tick -> list of fault ids returned by step().
    A step that raises is recorded as faults_by_tick[tick] = "raise:<Type>".
    """
    cmds_at, deaths_at, wps_at, ovs_at = {}, {}, {}, {}
    for i, c in enumerate(sc.cmds):
        cmds_at.setdefault(c[0], []).append((i, c))
    for t, ids in sc.deaths:
        deaths_at.setdefault(t, []).extend(ids)
    for t, p, r in sc.waypoints:
        wps_at.setdefault(t, []).append((p, r))
    for t, v in sc.overlays:
        ovs_at.setdefault(t, []).append(v)
    cmd_ok = np.zeros(len(sc.cmds), dtype=bool)
    records, faults = {}, {}
    for tick in range(sc.ticks):
        if tick in deaths_at:
            group.mark_dead(deaths_at[tick])
        for i, c in cmds_at.get(tick, []):
            cmd_ok[i] = bool(group.apply_command(make_cmd(c[1], c[2], c[3])))
        for p, r in wps_at.get(tick, []):
            group.retarget_waypoint(p, r)
        for v in ovs_at.get(tick, []):
            group.add_velocity_overlay(v)
        try:
            f = group.step(sc.dt)
            faults[tick] = [int(x) for x in np.asarray(f).tolist()]
        except Exception as exc:  # the reference World kills the group here (core.py:467-475)
            faults[tick] = f"raise:{type(exc).__name__}"
            break
        if on_tick is not None:
            on_tick(tick, group)
        if tick in sc.record and state_of is not None:
            records[tick] = state_of(group)
    return records, cmd_ok, faults


# ---------------------------------------------------------------- scenarios
def _unit_quats(rng, n, tilt=None):
    if tilt is None:
        q = rng.standard_normal((n, 4))
    else:
        axis = rng.standard_normal((n, 3))
        axis /= np.linalg.norm(axis, axis=1, keepdims=True)
        ang = rng.uniform(-tilt, tilt, n)
        q = np.concatenate([np.cos(ang / 2)[:, None], np.sin(ang / 2)[:, None] * axis], axis=1)
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _grid(n, spacing, origin):
    cols = max(1, int(np.ceil(np.sqrt(n))))
    idx = np.arange(n)
    return np.stack([(idx % cols) * spacing, (idx // cols) * spacing, np.zeros(n)], axis=1) + np.asarray(origin, float)


def hover_rate(n=64, ticks=300):
    """cfg1 shape: grid (3 m, z=10), RATE (0,0,0,m g), |w0| = 0.5 rad/s (test_control.py:227-233)."""
    rng = np.random.default_rng(0)
    w = rng.standard_normal((n, 3))
    w /= np.linalg.norm(w, axis=1, keepdims=True)
    q = np.zeros((n, 4)); q[:, 0] = 1.0
    sc = Scenario("hover_rate", n, 1e-3, ticks, _grid(n, 3.0, (0, 0, 10)), np.zeros((n, 3)), q, 0.5 * w,
                  record=[0, 1, 49, 99, 199, ticks - 1])
    sc.cmds = [(0, i, 1, (0.0, 0.0, 0.0, HOVER)) for i in range(n)]
    return sc


def pos_random(n=64, ticks=300, seed=1):
    """cfg3 recipe at small n: p_sp = p0 + U(-1,1)^3, v_sp = 0, yaw U(-pi,pi)."""
    rng = np.random.default_rng(seed)
    p0 = rng.uniform(-50, 50, (n, 3)) + np.array([0.0, 0.0, 100.0])
    q = _unit_quats(rng, n, tilt=0.6)
    vel = rng.uniform(-1, 1, (n, 3))
    om = rng.uniform(-0.5, 0.5, (n, 3))
    sc = Scenario("pos_random", n, 1e-3, ticks, p0, vel, q, om, record=[0, 1, 9, 49, 99, 199, ticks - 1])
    sp = p0 + rng.uniform(-1, 1, (n, 3))
    yaw = rng.uniform(-np.pi, np.pi, n)
    sc.cmds = [(0, i, 0, (*sp[i], 0.0, 0.0, 0.0, yaw[i])) for i in range(n)]
    return sc


def mixed(n=48, ticks=200, seed=2):
    """Every level, switches, deaths, overlay, waypoint, saturating commands."""
    rng = np.random.default_rng(seed)
    p0 = _grid(n, 2.0, (0, 0, 5))
    q = _unit_quats(rng, n, tilt=0.3)
    om = rng.uniform(-0.3, 0.3, (n, 3))
    sc = Scenario("mixed", n, 2e-3, ticks, p0, np.zeros((n, 3)), q, om,
                  record=[0, 1, 5, 10, 11, 20, 21, 40, 41, 60, 61, 100, 150, ticks - 1])
    cmds = []
    for i in range(n):
        kind = i % 6
        if kind == 0:   # default POS hold, later a new POS setpoint with velocity feed-forward
            cmds.append((15, i, 0, (p0[i, 0] + 1.0, p0[i, 1] - 0.5, p0[i, 2] + 0.7, 0.2, -0.1, 0.05, 0.4)))
        elif kind == 1:  # RATE, moderate
            cmds.append((0, i, 1, (0.2, -0.1, 0.3, HOVER * 1.05)))
        elif kind == 2:  # RATE, saturating (huge roll demand + over-max thrust)
            cmds.append((0, i, 1, (15.0, -12.0, 8.0, 80.0)))
        elif kind == 3:  # MOTOR, including out-of-range speeds
            cmds.append((0, i, 2, (15000.0, 16000.0, -20.0, 45000.0)))
        elif kind == 4:  # POS -> MOTOR -> POS (stale setpoints feed the PID while MOTOR)
            cmds.append((20, i, 2, (15700.0, 15650.0, 15700.0, 15650.0)))
            cmds.append((60, i, 0, (p0[i, 0], p0[i, 1], p0[i, 2] + 0.5, 0.0, 0.0, 0.0, -0.3)))
        else:            # RATE -> MOTOR -> RATE
            cmds.append((0, i, 1, (-0.3, 0.2, 0.0, HOVER)))
            cmds.append((40, i, 2, (15660.0, 15660.0, 15660.0, 15660.0)))
            cmds.append((100, i, 1, (0.0, 0.0, 0.5, HOVER * 0.95)))
    cmds.append((30, 10_000, 0, (0.0,) * 7))          # unknown agent -> rejected
    cmds.append((31, 3, 3, (1.0, 0.0)))               # non-quad level -> rejected
    cmds.append((12, 9, 1, (0.0, 0.0, 0.0, HOVER)))   # to a row killed at tick 11 -> rejected
    cmds.sort(key=lambda c: c[0])
    sc.cmds = cmds
    sc.deaths = [(0, [7]), (11, [9, 13]), (70, [30, 7])]
    sc.waypoints = [(50, (4.0, 4.0, 5.0), 3.5)]
    ov = np.zeros((n, 3))
    ov[::6] = rng.uniform(-0.5, 0.5, (len(ov[::6]), 3))
    sc.overlays = [(10, ov), (10, 0.5 * ov), (80, -ov)]
    return sc


def fault_nan(n=16, ticks=20):
    """Non-finite commands on RATE / MOTOR rows fault exactly those rows (quad.py:425-436)."""
    q = np.zeros((n, 4)); q[:, 0] = 1.0
    sc = Scenario("fault_nan", n, 1e-3, ticks, _grid(n, 3.0, (0, 0, 10)), np.zeros((n, 3)), q,
                  np.zeros((n, 3)), record=[0, 4, 5, 6, 7, ticks - 1])
    sc.cmds = [(0, i, 1, (0.0, 0.0, 0.0, HOVER)) for i in range(n)]
    sc.cmds += [(5, 3, 1, (0.0, 0.0, 0.0, float("nan"))),
                (7, 11, 2, (float("nan"), 1000.0, 1000.0, 1000.0)),
                (7, 12, 1, (float("inf"), 0.0, 0.0, HOVER))]
    return sc


def crash_nan(n=8, ticks=10):
    """A non-finite POS command makes the reference's outer loop raise (quat.py:84)."""
    q = np.zeros((n, 4)); q[:, 0] = 1.0
    sc = Scenario("crash_nan", n, 1e-3, ticks, _grid(n, 3.0, (0, 0, 10)), np.zeros((n, 3)), q,
                  np.zeros((n, 3)), record=[0, 1, 2, 3])
    sc.cmds = [(4, 2, 0, (0.0, 0.0, float("nan"), 0.0, 0.0, 0.0, 0.0))]
    return sc


def unicycles(n=40, ticks=150, seed=9):
    """UnicycleGroup (core.py:249-289): commands incl. clamped speeds / turn
    rates and straight lines, a death, an overlay tick."""
    rng = np.random.default_rng(seed)
    yaw = rng.uniform(-np.pi, np.pi, n)
    q = np.stack([np.cos(yaw / 2), np.zeros(n), np.zeros(n), np.sin(yaw / 2)], axis=1)
    sc = Scenario("unicycles", n, 0.01, ticks, _grid(n, 2.0, (0, 0, 0)), np.zeros((n, 3)), q, np.zeros((n, 3)),
                  record=[0, 1, 10, 49, 50, 51, 100, ticks - 1])
    cmds = []
    for i in range(n):
        k = i % 4
        if k == 0:
            cmds.append((0, i, 3, (float(rng.uniform(0, 3)), float(rng.uniform(-1, 1)))))
        elif k == 1:
            cmds.append((0, i, 3, (9.0, -7.0)))                    # both clamped
        elif k == 2:
            cmds.append((0, i, 3, (1.5, 0.0)))                     # straight line
        else:
            cmds.append((0, i, 3, (-0.7, 2.0)))
            cmds.append((60, i, 3, (0.4, -0.3)))
    cmds.append((5, 2, 0, (0.0,) * 7))                              # non-unicycle level -> rejected
    cmds.sort(key=lambda c: c[0])
    sc.cmds = cmds
    sc.deaths = [(30, [5])]
    ov = np.zeros((n, 3))
    ov[::3] = rng.uniform(-1, 1, (len(ov[::3]), 3))
    sc.overlays = [(50, ov)]
    return sc


ALL = {"hover_rate": hover_rate, "pos_random": pos_random, "mixed": mixed,
       "fault_nan": fault_nan, "crash_nan": crash_nan}
