"""Generate golden vectors by running the REFERENCE itself (swarmstep, float64).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``swarmstep`` from /root/reference/pkg/src (read-only, via
sys.path), drives its real hot-path functions and ``QuadGroup`` through the
scenarios of tests/scenarios.py, and writes small .npz fixtures next to this
file.  The fixtures are committed; nothing on the GPU box reads the reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import scenarios  # noqa: E402
from swarmstep.control import (PosSetpoint, RatePidState, RateSetpoint, default_outer_gains,  # noqa: E402
                               default_rate_gains, position_outer_loop, rate_pid_step)
from swarmstep.core import QuadGroup  # noqa: E402
from swarmstep.quad import (QuadWorkspace, default_quad_params, dynamics_deriv, mix_to_motors,  # noqa: E402
                            rk4_step)
from swarmstep.state import batch_create  # noqa: E402
from swarmstep.wire import AgentCommand, CommandLevel  # noqa: E402

P = default_quad_params()
LEVELS = {0: CommandLevel.POS, 1: CommandLevel.RATE, 2: CommandLevel.MOTOR, 3: CommandLevel.UNICYCLE}


def make_cmd(agent_id, level_code, values):
    return AgentCommand(int(agent_id), LEVELS[level_code], tuple(values))


def state_of(g: QuadGroup) -> dict:
    b = g.batch
    return dict(pos=b.pos.copy(), vel=b.vel.copy(), quat=b.quat.copy(), omega=b.omega.copy(),
                alive=b.alive.copy(), integral=g.pid_state.integral.copy(),
                prev_omega=g.pid_state.prev_omega.copy(), has_prev=g.pid_state.has_prev.copy(),
                omega_sp=g.omega_sp.copy(), f_c_sp=g.f_c_sp.copy(),
                cmd_level=g.cmd_level.copy(), cmd_values=g.cmd_values.copy())


def gen_scenario(name: str) -> None:
    sc = scenarios.ALL[name]()
    batch = batch_create(0, sc.n, sc.pos, quat=sc.quat, vel=sc.vel, omega=sc.omega)
    init = dict(pos=batch.pos.copy(), vel=batch.vel.copy(), quat=batch.quat.copy(), omega=batch.omega.copy())
    group = QuadGroup(0, batch, P)
    records, cmd_ok, faults = scenarios.run_script(group, sc, make_cmd, state_of)
    out = sc.to_arrays()
    # batch_create renormalises quaternions: store the exact initial state used
    out.update(init)
    ticks = sorted(records)
    out["rec_ticks"] = np.array(ticks, dtype=np.int64)
    for key in records[ticks[0]] if ticks else []:
        out[f"rec_{key}"] = np.stack([records[t][key] for t in ticks])
    out["cmd_ok"] = cmd_ok
    ft, fi, raise_tick = [], [], -1
    for t, f in faults.items():
        if isinstance(f, str):
            raise_tick = t
            continue
        for a in f:
            ft.append(t)
            fi.append(a)
    out["fault_tick"] = np.array(ft, dtype=np.int64)
    out["fault_id"] = np.array(fi, dtype=np.int64)
    out["raise_tick"] = np.array(raise_tick)
    np.savez_compressed(HERE / f"scenario_{name}.npz", **out)
    print(f"{name}: n={sc.n} ticks={sc.ticks} recorded={ticks} faults={len(fi)} raise_tick={raise_tick}")


def gen_functions() -> None:
    rng = np.random.default_rng(2024)
    out = {}
    # --- dynamics_deriv (quad.py:320-335)
    n = 256
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    b = batch_create(0, n, rng.uniform(-5, 5, (n, 3)), quat=q, vel=rng.uniform(-2, 2, (n, 3)),
                     omega=rng.uniform(-3, 3, (n, 3)))
    f_c = rng.uniform(0, 40, n)
    tau = rng.uniform(-0.5, 0.5, (n, 3))
    d = dynamics_deriv(b, f_c, tau, P)
    out["deriv_state"] = np.hstack([b.pos, b.vel, b.quat, b.omega])
    out["deriv_fc"], out["deriv_tau"] = f_c, tau
    out["deriv_out"] = np.hstack([d.pos[:n], d.vel[:n], d.quat[:n], d.omega[:n]])

    # --- rk4_step (quad.py:350-437): 20 steps, piecewise wrench, dead rows
    n = 128
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    b = batch_create(0, n, rng.uniform(-5, 5, (n, 3)), quat=q, vel=rng.uniform(-2, 2, (n, 3)),
                     omega=rng.uniform(-1, 1, (n, 3)))
    b.alive[[5, 77]] = False
    out["rk4_state0"] = np.hstack([b.pos, b.vel, b.quat, b.omega])
    out["rk4_alive0"] = b.alive.copy()
    ws = QuadWorkspace(n)
    fcs, taus = [], []
    for k in range(20):
        if k % 5 == 0:
            f_c = rng.uniform(0.0, 2 * P.m * P.g, n)
            tau = rng.uniform(-0.05, 0.05, (n, 3))
        fcs.append(f_c.copy())
        taus.append(tau.copy())
        rk4_step(b, f_c, tau, P, 1e-3, ws)
    out["rk4_fc"], out["rk4_tau"] = np.stack(fcs), np.stack(taus)
    out["rk4_state20"] = np.hstack([b.pos, b.vel, b.quat, b.omega])
    out["rk4_alive20"] = b.alive.copy()
    # fault case (test_quad.py:171-179)
    bf = batch_create(0, 2, np.zeros((2, 3)))
    fids = rk4_step(bf, np.zeros(2), np.array([[0.0, 0.0, 0.0], [1e308, 0.0, 0.0]]), P, 1e6)
    out["rk4_fault_ids"] = fids.astype(np.int64)
    out["rk4_fault_state"] = np.hstack([bf.pos, bf.vel, bf.quat, bf.omega])
    out["rk4_fault_alive"] = bf.alive.copy()

    # --- mix_to_motors (quad.py:143-168), including saturation
    n = 256
    f_c = rng.uniform(-5, 70, n)
    tau = rng.uniform(-1.0, 1.0, (n, 3)) * np.array([1.0, 1.0, 0.02])
    mx = mix_to_motors(f_c, tau, P)
    out["mix_fc"], out["mix_tau"] = f_c, tau
    out["mix_motors"] = mx.motors.copy()
    out["mix_realized"] = np.hstack([mx.f_c[:, None], mx.tau]).copy()
    out["mix_sat"] = mx.saturated.copy()

    # --- rate_pid_step (control.py:136-187): 30 steps, dead rows appear
    n, steps, dt = 32, 30, 0.013
    st = RatePidState(n)
    alive = np.ones(n, dtype=bool)
    om_s, sp_s, fsp_s, al_s, tau_s, fc_s, int_s = [], [], [], [], [], [], []
    for k in range(steps):
        if k == 10:
            alive[[3, 17]] = False
        om = rng.uniform(-3, 3, (n, 3))
        sp = rng.uniform(-3, 3, (n, 3))
        fsp = rng.uniform(0, 20, n)
        fc, tq = rate_pid_step(om, RateSetpoint(sp, fsp), default_rate_gains(), dt, st, alive)
        om_s.append(om); sp_s.append(sp); fsp_s.append(fsp); al_s.append(alive.copy())
        tau_s.append(tq.copy()); fc_s.append(fc.copy()); int_s.append(st.integral.copy())
    out["pid_omega"], out["pid_sp"], out["pid_fsp"] = np.stack(om_s), np.stack(sp_s), np.stack(fsp_s)
    out["pid_alive"], out["pid_tau"], out["pid_fc"] = np.stack(al_s), np.stack(tau_s), np.stack(fc_s)
    out["pid_integral"], out["pid_dt"] = np.stack(int_s), np.array(dt)

    # --- position_outer_loop (control.py:222-294), incl. every branch
    n = 512
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[:128] = np.array([1.0, 0, 0, 0]) + 0.05 * rng.standard_normal((128, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    pos = rng.uniform(-5, 5, (n, 3))
    vel = rng.uniform(-2, 2, (n, 3))
    p_sp = pos + rng.uniform(-3, 3, (n, 3))
    v_sp = rng.uniform(-1, 1, (n, 3))
    yaw = rng.uniform(-np.pi, np.pi, n)
    alive = rng.random(n) > 0.05
    g = default_outer_gains()
    # low-thrust rows: a_cmd = 0 exactly
    p_sp[500:503] = pos[500:503] + np.array([0.0, 0.0, -P.g / 16.0])
    v_sp[500:503] = vel[500:503]
    # degenerate-yaw rows: z_des parallel to the heading (a = (16,0,0), yaw 0)
    p_sp[503:506] = pos[503:506] + np.array([1.0, 0.0, -P.g / 16.0])
    v_sp[503:506] = vel[503:506]
    yaw[503:506] = 0.0
    alive[500:506] = True
    res = position_outer_loop(pos, vel, q, alive, PosSetpoint(p_sp, v_sp, yaw), P, g)
    for k, v in dict(pos=pos, vel=vel, quat=q, p_sp=p_sp, v_sp=v_sp, yaw=yaw, alive=alive,
                     omega_sp=res.setpoint.omega_sp, f_c=res.setpoint.f_c_sp, low=res.low_thrust).items():
        out[f"outer_{k}"] = np.asarray(v).copy()
    np.savez_compressed(HERE / "functions.npz", **out)
    print("functions: deriv/rk4/mix/pid/outer written")


def gen_collision() -> None:
    """detect() (collision.py:110-176) on random two-type worlds; positions are
    multiples of 2^-10 so they are exact in float32 (the B200 groups hold them
    bit-exactly and the comparison can be exact)."""
    from swarmstep.collision import CollisionConfig, detect
    from swarmstep.state import WorldSnapshot, batch_snapshot
    rng = np.random.default_rng(77)
    out = {}
    worlds = 24
    for w in range(worlds):
        n0, n1 = int(rng.integers(1, 300)), int(rng.integers(0, 60))
        box = float(rng.uniform(3, 15))
        r0, r1 = float(rng.uniform(0.05, 0.4)), float(rng.uniform(0.05, 0.4))
        r_sense = float(rng.uniform(2 * max(r0, r1), 3.0))
        cell = float(rng.uniform(2 * max(r0, r1), 2.5))
        q = lambda a: np.round(a * 1024.0) / 1024.0
        p0, p1 = q(rng.uniform(-box, box, (n0, 3))), q(rng.uniform(-box, box, (n1, 3)))
        a0, a1 = rng.random(n0) > 0.1, rng.random(n1) > 0.1
        batches = []
        b0 = batch_create(0, n0, p0)
        b0.alive[:] = a0
        batches.append(batch_snapshot(b0, w))
        if n1:
            b1 = batch_create(1, n1, p1, id_base=n0)
            b1.alive[:] = a1
            batches.append(batch_snapshot(b1, w))
        cfg = CollisionConfig(r_collide={0: r0, 1: r1}, r_sense=r_sense, cell=cell)
        rep = detect(WorldSnapshot(tick=w, batches=tuple(batches)), cfg)
        pre = f"w{w}_"
        out[pre + "p0"], out[pre + "p1"], out[pre + "a0"], out[pre + "a1"] = p0, p1.reshape(-1, 3), a0, a1
        out[pre + "cfg"] = np.array([r0, r1, r_sense, cell])
        out[pre + "coll"] = np.array(rep.collisions, dtype=np.int64).reshape(-1, 2)
        keys = sorted(rep.neighbor_sets)
        out[pre + "nb_keys"] = np.array(keys, dtype=np.int64)
        out[pre + "nb_len"] = np.array([len(rep.neighbor_sets[k]) for k in keys], dtype=np.int64)
        out[pre + "nb_ids"] = np.array([i for k in keys for i in rep.neighbor_sets[k]], dtype=np.int64)
    out["worlds"] = np.array(worlds)
    np.savez_compressed(HERE / "collision.npz", **out)
    print(f"collision: {worlds} worlds")


def gen_unicycle() -> None:
    from swarmstep.core import UnicycleGroup, UnicycleParams
    sc = scenarios.unicycles()
    batch = batch_create(1, sc.n, sc.pos, quat=sc.quat, vel=sc.vel, omega=sc.omega)
    init = dict(pos=batch.pos.copy(), vel=batch.vel.copy(), quat=batch.quat.copy(), omega=batch.omega.copy())
    group = UnicycleGroup(1, batch, UnicycleParams())

    def state(g):
        b = g.batch
        return dict(pos=b.pos.copy(), vel=b.vel.copy(), quat=b.quat.copy(), omega=b.omega.copy(),
                    alive=b.alive.copy(), cmd=g.cmd.copy())

    records, cmd_ok, faults = scenarios.run_script(group, sc, make_cmd, state)
    out = sc.to_arrays()
    out.update(init)
    ticks = sorted(records)
    out["rec_ticks"] = np.array(ticks, dtype=np.int64)
    for key in records[ticks[0]]:
        out[f"rec_{key}"] = np.stack([records[t][key] for t in ticks])
    out["cmd_ok"] = cmd_ok
    np.savez_compressed(HERE / "scenario_unicycles.npz", **out)
    print(f"unicycles: n={sc.n} ticks={sc.ticks}")


def viewer_cases():
    """(mode, point, radius, strength) messages of the viewer golden set; the
    point of case 3 sits exactly on agent 5 (the d > 1e-12 guard)."""
    return [("attract", (1.0, -2.0, 10.5), 6.0, 1.5), ("repel", (-3.25, 4.0, 9.0), 4.0, 0.75),
            ("attract", (0.0, 0.0, 10.0), 0.0, 2.0), ("repel", None, 5.0, 1.0),
            ("attract", (1.0, 1.0, 10.0), 3.0, 0.0), ("waypoint", (2.0, 2.0, 11.0), 5.0, 1.0),
            ("attract", (50.0, 50.0, 50.0), 2.0, 1.0)]


def gen_viewer() -> None:
    """World._apply_viewer_input (core.py:445-453): viewer_velocity_offsets
    (wire.py:320-340) per message, and the command store after a WAYPOINT
    retarget (core.py:141-149).  Positions are multiples of 2^-20 (exact as a
    float32 hi + lo pair, so the device sees the same float64 positions)."""
    from swarmstep.wire import InfluenceMode, ViewerInputMsg, viewer_velocity_offsets
    rng = np.random.default_rng(31)
    n = 200
    pos = np.round(rng.uniform(-6.0, 6.0, (n, 3)) * 2.0**20) / 2.0**20
    pos[:, 2] += 10.0
    alive = rng.random(n) > 0.15
    alive[5] = True
    quat = rng.normal(size=(n, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    quat = np.round(quat * 2.0**20) / 2.0**20      # exact in float32
    out = {"pos": pos, "alive": alive, "quat": quat}
    for i, (mode, point, radius, strength) in enumerate(viewer_cases()):
        point = tuple(pos[5]) if point is None else point
        msg = ViewerInputMsg(mode=InfluenceMode(mode), world_point=point, radius=radius, strength=strength)
        off = viewer_velocity_offsets(msg, pos, alive)
        out[f"v{i}_point"] = np.array(point, dtype=float)
        out[f"v{i}_msg"] = np.array([mode, radius, strength], dtype=object).astype(str)
        out[f"v{i}_off"] = off
        out[f"v{i}_any"] = np.array(bool(off.any()))
        if mode == "waypoint":
            b = batch_create(0, n, pos, quat=quat)
            b.alive[:] = alive
            g = QuadGroup(0, b, P)
            g.retarget_waypoint(point, radius)
            out[f"v{i}_cmd_level"] = g.cmd_level.copy()
            out[f"v{i}_cmd_values"] = g.cmd_values.copy()
    out["cases"] = np.array(len(viewer_cases()))
    np.savez_compressed(HERE / "viewer.npz", **out)
    print(f"viewer: {len(viewer_cases())} messages over n={n}")


def world_script():
    """Inbox items per tick for the World golden run: commands of every level
    (including rejected ones: unknown id, wrong level, dead agents) and viewer
    inputs of every mode.  Plain data so the GPU test replays it without the
    reference."""
    return {
        "0": [["cmd", 0, "pos", [2.2, 0.0, 5.0, 0.0, 0.0, 0.0, 0.0]],     # agents 0 and 1 fly head on
              ["cmd", 1, "pos", [-0.7, 0.0, 5.0, 0.0, 0.0, 0.0, 0.0]],
              ["cmd", 40, "unicycle", [0.8, 0.3]], ["cmd", 41, "unicycle", [0.5, -0.2]],
              ["cmd", 9999, "pos", [0.0] * 7], ["cmd", 42, "pos", [0.0] * 7]],
        "30": [["viewer", "attract", [6.0, 3.0, 5.5], 3.0, 1.5]],
        "60": [["cmd", 7, "rate", [0.3, -0.2, 0.1, 10.5]], ["cmd", 8, "motor", [11000.0, 10000.0, 11000.0, 10000.0]],
               ["viewer", "repel", [3.0, 4.5, 5.0], 2.5, 2.0]],
        "90": [["viewer", "waypoint", [9.0, 6.0, 5.0], 2.0, 1.0], ["cmd", 20, "pos", [7.0, 7.0, 6.0, 0.5, 0.0, 0.0, 1.0]]],
        "120": [["cmd", 7, "pos", [4.5, 1.5, 5.0, 0.0, 0.0, 0.0, -0.5]], ["cmd", 8, "rate", [0.0, 0.0, 0.0, 9.81]],
                ["viewer", "attract", [1.0, 1.0, 5.0], 0.0, 3.0]],
        "200": [["cmd", 0, "pos", [0.0] * 7], ["cmd", 1, "rate", [0.0, 0.0, 0.0, 9.0]],
                ["viewer", "repel", [7.5, 7.5, 5.0], 4.0, 0.5]],
    }


WORLD_QUADS, WORLD_UNIS, WORLD_TICKS, WORLD_DT = 40, 10, 300, 1.0 / 512.0


def world_layout():
    """Quads on a 1.5 m grid at z = 5 (8 columns), unicycles on a line at y = -3."""
    q = np.array([[1.5 * (i % 8), 1.5 * (i // 8), 5.0] for i in range(WORLD_QUADS)])
    u = np.array([[2.0 * i, -3.0, 0.0] for i in range(WORLD_UNIS)])
    return q, u


def gen_world() -> None:
    """The reference World (core.py:308-505) itself -- events -> inbox ->
    step groups -> in-loop collision detect -> deaths -> publish -- over a
    quad group and a unicycle group for WORLD_TICKS ticks of world_script();
    records the event log and the float64 state every 20 ticks."""
    import json
    from swarmstep.collision import CollisionConfig
    from swarmstep.core import UnicycleGroup, UnicycleParams, World
    from swarmstep.wire import InfluenceMode, ViewerInputMsg
    qpos, upos = world_layout()
    quads = QuadGroup(0, batch_create(0, WORLD_QUADS, qpos), P)
    unis = UnicycleGroup(1, batch_create(1, WORLD_UNIS, upos, id_base=WORLD_QUADS), UnicycleParams())
    cfg = CollisionConfig(r_collide={0: 0.2, 1: 0.3}, r_sense=1.2, cell=1.2)
    world = World([quads, unis], dt=WORLD_DT, collision_config=cfg, collision_in_loop=True)
    script = world_script()
    out = {}
    for t in range(WORLD_TICKS):
        for item in script.get(str(t), []):
            if item[0] == "cmd":
                world.submit_commands([make_cmd(item[1], {"pos": 0, "rate": 1, "motor": 2, "unicycle": 3}[item[2]],
                                                item[3])])
            else:
                world.submit_viewer_input(ViewerInputMsg(mode=InfluenceMode(item[1]), world_point=tuple(item[2]),
                                                         radius=item[3], strength=item[4]))
        world.tick()
        if (t + 1) % 20 == 0:
            for g in world.groups:
                b = g.batch
                for k in ("pos", "vel", "quat", "omega", "alive"):
                    out[f"t{t}_g{g.type_id}_{k}"] = getattr(b, k).copy()
    events = [[e.tick, e.kind.value, list(e.agent_ids)] for e in world.event_log]
    out["events"] = np.array(json.dumps(events))
    out["script"] = np.array(json.dumps(script))
    out["qpos"], out["upos"] = qpos, upos
    out["dt"], out["ticks"] = np.array(WORLD_DT), np.array(WORLD_TICKS)
    np.savez_compressed(HERE / "world.npz", **out)
    print(f"world: {WORLD_TICKS} ticks, events {events}")


CFG1_N, CFG1_TICKS, CFG1_EVERY = 1000, 10_000, 1000


def gen_cfg1() -> None:
    """SURVEY.md 8(d) cfg1 at its stated size and horizon, through the reference
    QuadGroup itself: 1,000 quads on the bench grid (3 m, z = 10), RATE hover
    (0, 0, 0, m g) with initial rates 0.5 unit(N(0, I)) (test_control.py:
    227-233), dt = 1 ms, 10,000 ticks; float64 checkpoints every 1,000 ticks.
    Inputs are float32-representable (initial state, hover thrust, dt), so the
    B200 path starts from the identical state and commands and the recorded
    divergence is arithmetic only (the pattern of test_acceptance.py:38-68)."""
    sc = scenarios.hover_rate(n=CFG1_N, ticks=CFG1_TICKS)

    def f32(a):
        return np.asarray(a, dtype=float).astype(np.float32).astype(np.float64)

    dt = float(np.float32(sc.dt))
    batch = batch_create(0, sc.n, f32(sc.pos), quat=f32(sc.quat), vel=f32(sc.vel), omega=f32(sc.omega))
    init = dict(pos=batch.pos.copy(), vel=batch.vel.copy(), quat=batch.quat.copy(), omega=batch.omega.copy())
    g = QuadGroup(0, batch, P)
    vals = {}
    for _, agent, lvl, v in sc.cmds:
        vals[agent] = tuple(f32(v).tolist())
        assert g.apply_command(make_cmd(agent, lvl, vals[agent]))
    out = {f"init_{k}": v for k, v in init.items()}
    out["cmd_values"] = np.array([vals[i] for i in range(sc.n)])
    out["dt"], out["every"] = np.array(dt), np.array(CFG1_EVERY)
    faults = 0
    for t in range(CFG1_TICKS):
        faults += len(g.step(dt))
        if (t + 1) % CFG1_EVERY == 0:
            b = g.batch
            for k in ("pos", "vel", "quat", "omega"):
                out[f"t{t + 1}_{k}"] = getattr(b, k).copy()
            out[f"t{t + 1}_integral"] = g.pid_state.integral.copy()
    assert faults == 0
    np.savez_compressed(HERE / "cfg1.npz", **out)
    print(f"cfg1: n={sc.n} ticks={CFG1_TICKS} checkpoints every {CFG1_EVERY}")


if __name__ == "__main__":
    if "--cfg1" in sys.argv:
        gen_cfg1()
        sys.exit(0)
    gen_cfg1()
    gen_world()
    gen_viewer()
    gen_unicycle()
    gen_collision()
    gen_functions()
    for name in scenarios.ALL:
        gen_scenario(name)
