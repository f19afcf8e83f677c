"""GPU checks of the device setpoint feed (f1) and CUDA-graph tick loops:
circle setpoints equal circle_reference (control.py:297-315), graph replays are
bit-identical to eager ticks, faults inside a graph keep their tick, and the
closed-loop circle demo meets the reference's acceptance bound
(test_acceptance.py:187-224: RMS < 0.3 m after the 10 s transient)."""

import math

import numpy as np
import pytest

from conftest import cuda_ok
from gpu_util import PER_STEP_TOL, gpu_state, make_group
from oracle import oracle as orc
from scenarios import Scenario

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def circle_reference(t, radius, omega, z, phase):
    """control.py:297-315 in float64 (numpy restatement for the check)."""
    th = omega * t + phase
    p = np.stack([radius * np.cos(th), radius * np.sin(th), np.full_like(th, z)], axis=-1)
    v = np.stack([-radius * omega * np.sin(th), radius * omega * np.cos(th), np.zeros_like(th)], axis=-1)
    return p, v, th + math.copysign(math.pi / 2, omega)


def _circle_group(n, radius=5.0, z=10.0, compensated=True):
    ph = 2 * np.pi * np.arange(n) / n
    pos = np.stack([radius * np.cos(ph), radius * np.sin(ph), np.full(n, z)], axis=1)   # config.py:159-168
    yaw = ph + np.pi / 2
    q = np.stack([np.cos(yaw / 2), np.zeros(n), np.zeros(n), np.sin(yaw / 2)], axis=1)
    return make_group(Scenario("circle", n, 2e-3, 1, pos, np.zeros((n, 3)), q, np.zeros((n, 3)), record=[]),
                      compensated=compensated)


def test_circle_feed_setpoints():
    from paper_2308_12698_b200.feed import CircleFeed
    n, dt = 1000, 2e-3
    g = _circle_group(n)
    feed = CircleFeed(g, dt, radius=5.0, omega=0.3, z=10.0)
    g._tick = 12345
    feed.apply()
    cv = g.cmd_values
    p, v, yaw = circle_reference(12345 * dt, 5.0, 0.3, 10.0, 2 * np.pi * np.arange(n) / n)
    np.testing.assert_allclose(cv[:, :3], p, atol=2e-6)
    np.testing.assert_allclose(cv[:, 3:6], v, atol=2e-6)
    np.testing.assert_allclose(np.cos(cv[:, 6]), np.cos(yaw), atol=1e-6)
    np.testing.assert_allclose(np.sin(cv[:, 6]), np.sin(yaw), atol=1e-6)
    assert np.all(g.cmd_level == 0)


def test_graph_replay_bit_identical_to_eager_ticks():
    from paper_2308_12698_b200.feed import CircleFeed, TickGraph
    n, dt, T = 777, 2e-3, 25
    ga, gb = _circle_group(n), _circle_group(n)
    fa, fb = CircleFeed(ga, dt), CircleFeed(gb, dt)
    graph = TickGraph(ga, dt, T, feed=fa)
    for _ in range(4):
        graph.replay()
    ga.collect_faults()
    for _ in range(4 * T):
        fb.apply()
        gb.step(dt)
    sa, sb = gpu_state(ga), gpu_state(gb)
    for k in ("pos", "vel", "quat", "omega", "integral", "prev_omega"):
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)
    assert ga._tick == gb._tick == 4 * T


def test_graph_fault_keeps_its_tick():
    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    from paper_2308_12698_b200.feed import TickGraph
    n, dt, T = 64, 1e-3, 10
    g = _circle_group(n)
    g.set_setpoints(np.tile([0.0, 0.0, 0.0, 9.81], (n, 1)), level="rate")
    graph = TickGraph(g, dt, T)
    graph.replay()
    assert all(f.size == 0 for f in g.collect_faults())
    assert g.apply_command(AgentCommand(5, CommandLevel.RATE, (0.0, 0.0, 0.0, float("nan"))))
    graph.replay()
    per_tick = g.collect_faults()
    assert len(per_tick) == T and per_tick[0].tolist() == [5]
    assert not g.batch.alive[5] and g.batch.alive.sum() == n - 1


def test_closed_loop_circle_demo_shape():
    """100 quads on 5 m circles (test_acceptance.py:187-224), device feed + graphs,
    and the same run on the float64 oracle with per-tick commands."""
    from paper_2308_12698_b200.feed import CircleFeed, TickGraph
    n, dt, radius, omega, z = 100, 2e-3, 5.0, 0.3, 10.0
    g = _circle_group(n)
    feed = CircleFeed(g, dt, radius=radius, omega=omega, z=z)
    T = 500
    graph = TickGraph(g, dt, T, feed=feed)
    n_ticks = round(40.0 / dt)
    phases = 2 * np.pi * np.arange(n) / n
    st0 = gpu_state(g)
    og = orc.OracleGroup(0, type("B", (), dict(agent_ids=np.arange(n, dtype=np.uint64), pos=st0["pos"],
                                                vel=st0["vel"], quat=st0["quat"], omega=st0["omega"],
                                                alive=np.ones(n, bool)))())
    sq, samples, worst_div = np.zeros(n), 0, 0.0
    for rep in range(n_ticks // T):
        graph.replay()
        for j in range(T):
            k = rep * T + j
            p, v, yaw = circle_reference(k * dt, radius, omega, z, phases)
            og.cmd_level[:] = 0
            og.cmd_values[:, :3], og.cmd_values[:, 3:6], og.cmd_values[:, 6] = p, v, yaw
            og.step(float(np.float32(dt)))
        assert all(f.size == 0 for f in g.collect_faults())
        t = (rep + 1) * T * dt
        pos = g.batch.pos
        worst_div = max(worst_div, float(np.max(np.abs(pos - og.pos))))
        if t > 10.0:
            ref, _, _ = circle_reference(t, radius, omega, z, phases)
            err = np.linalg.norm(pos - ref, axis=1)
            sq += err * err
            samples += 1
    rms = float(np.max(np.sqrt(sq / samples)))
    assert rms < 0.3, rms
    assert worst_div < 1e-3, worst_div     # bounded divergence from the float64 oracle over 40 s


@pytest.mark.parametrize("compensated", [False, True])
@pytest.mark.parametrize("kern", ["direct", "pair"])
@pytest.mark.parametrize("k", [1, 7, 25])
def test_fused_circle_feed_bit_identical(k, kern, compensated):
    """K ticks of the circle strategy evaluated inside one launch vs
    K x (feed kernel + 1-tick step): command columns, levels, faults (row 9
    faults on the first fed tick through a NaN D-term sample) and the tick
    counter identical; the state bit for bit at K = 1, and within FUSION_TOL
    for K > 1 (the fused feed advances the setpoint by rotation after its
    first tick, and the compensated position folds once per launch)."""
    from gpu_util import assert_fusion_close
    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    from paper_2308_12698_b200.feed import CircleFeed
    outs = []
    for fused in (False, True):
        g = _circle_group(300, compensated=compensated)
        g.apply_command(AgentCommand(5, CommandLevel.RATE, (0.0, 0.0, 0.0, 20.0)))   # the feed moves it to POS
        g.mark_dead([7])
        g.step(2e-3)                       # tick 0 outside the feed
        prev = g.pid_state_dict()["prev_omega"]
        prev[9] = np.nan
        g.set_pid_state(prev_omega=prev)
        feed = CircleFeed(g, 2e-3)
        if fused:
            g.kernel = kern
            feed.step_fused(k)
            faults = g.collect_faults()
        else:
            faults = []
            for _ in range(k):
                feed.apply()
                faults.append(g.step(2e-3))
        st = g.batch
        outs.append(dict(pos=st.pos.copy(), vel=st.vel.copy(), quat=st.quat.copy(), omega=st.omega.copy(),
                         alive=st.alive.copy(), cmd=g.cmd_values.copy(), lvl=g.cmd_level.copy(),
                         faults=[np.asarray(f).tolist() for f in faults], tick=g._tick))
    assert outs[0]["faults"][0] == [9]
    for key in outs[0]:
        if key in ("faults", "tick"):
            assert outs[0][key] == outs[1][key], key
        elif k > 1 and key in ("pos", "vel", "quat", "omega"):
            # the rotation-advanced setpoints differ from the direct evaluation
            # by float32 rounding (~1e-7 relative over 25 ticks): the trajectories
            # agree within the per-step parity bar
            assert_fusion_close(outs[0], outs[1], [key], tol=PER_STEP_TOL)
        elif compensated and key in ("pos", "vel", "quat", "omega"):
            assert_fusion_close(outs[0], outs[1], [key])
        else:
            np.testing.assert_array_equal(outs[0][key], outs[1][key], err_msg=key)


def test_command_store_latest_wins_across_device_writers():
    """apply_command (host queue) vs device-side writers (bulk setpoints, the
    circle feed): whichever came last wins (core.py:117-135), and the host
    mirror shows exactly what the device will step on."""
    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    from paper_2308_12698_b200.feed import CircleFeed
    g = _circle_group(200)
    sp = np.tile([1.0, 2.0, 3.0, 0.0, 0.0, 0.0, 0.5], (200, 1))
    g.set_setpoints(sp)                                               # device writer
    g.apply_command(AgentCommand(3, CommandLevel.RATE, (0.1, 0.2, 0.3, 9.0)))   # later: wins for row 3
    cv, lv = g.cmd_values.copy(), g.cmd_level.copy()
    assert lv[3] == 1 and np.allclose(cv[3], [0.1, 0.2, 0.3, 9.0, 0, 0, 0])
    assert np.allclose(cv[4], sp[4]) and lv[4] == 0
    feed = CircleFeed(g, 2e-3)
    g.apply_command(AgentCommand(5, CommandLevel.RATE, (0.0, 0.0, 0.0, 9.0)))   # then the feed: feed wins
    feed.apply()
    assert g.cmd_level[5] == 0 and g.cmd_level[3] == 0
    g.step(2e-3)
    g.apply_command(AgentCommand(6, CommandLevel.MOTOR, (1e4, 1e4, 1e4, 1e4)))   # after the feed: wins
    assert g.cmd_level[6] == 2
    g.step(2e-3)
    assert g.cmd_level[6] == 2 and np.allclose(g.cmd_values[6, :4], 1e4)
