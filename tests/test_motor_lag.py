"""The opt-in first-order rotor lag (north star; ABSENT in the reference, so its
parity is unpinned -- SURVEY.md 8(a)).  CPU checks of the float64 oracle's lag
model against closed forms, plus its tau_m -> 0 limit against the pinned
instantaneous-mixer path.  The GPU kernel is compared with this oracle in
tests/test_gpu_motor_lag.py."""

import math

import numpy as np
import pytest

from oracle import oracle as orc

M, G = 1.0, 9.81


class _B:
    def __init__(self, n, pos=None):
        self.agent_ids = np.arange(n, dtype=np.uint64)
        self.pos = np.zeros((n, 3)) if pos is None else np.asarray(pos, float)
        self.vel, self.omega = np.zeros((n, 3)), np.zeros((n, 3))
        self.quat = np.tile([1.0, 0, 0, 0], (n, 1))
        self.alive = np.ones(n, bool)


def _rate(g, fc, rows=None):
    rows = np.arange(g.n) if rows is None else rows
    g.cmd_level[rows] = 1
    g.cmd_values[rows] = 0.0
    g.cmd_values[rows, 3] = fc


def test_hover_split_is_a_fixed_point():
    g = orc.OracleGroup(0, _B(4), motor_tau=0.03)
    _rate(g, M * G)
    for _ in range(200):
        g.step(1e-3)
    np.testing.assert_allclose(g.motor, M * G / 4, rtol=0, atol=1e-12)
    assert np.abs(g.vel).max() < 1e-12 and np.abs(g.pos).max() < 1e-12


@pytest.mark.parametrize("tau", [0.01, 0.05])
def test_thrust_step_response_closed_form(tau):
    """Vertical thrust step from hover: the rotor thrust follows
    f(t) = u + (f0 - u) e^(-t/tau) exactly, and since each tick integrates the
    tick-mean thrust the climb rate is the exact impulse
    v(t) = int_0^t (4 f(s)/m - g) ds."""
    dt, steps = 1e-3, 300
    g = orc.OracleGroup(0, _B(1), motor_tau=tau)
    u_total = 2.0 * M * G
    _rate(g, u_total)
    for _ in range(steps):
        g.step(dt)
    t = dt * steps
    f0, u = M * G / 4, u_total / 4
    np.testing.assert_allclose(g.motor[0], u + (f0 - u) * math.exp(-t / tau), rtol=1e-12)
    vz = (4 * u / M - G) * t + 4 * (f0 - u) / M * tau * (1 - math.exp(-t / tau))
    assert abs(g.vel[0, 2] - vz) < 1e-11
    # z(t) = int v: the per-tick held mean thrust is second-order accurate
    z = 0.5 * (4 * u / M - G) * t * t + 4 * (f0 - u) / M * tau * (t - tau * (1 - math.exp(-t / tau)))
    assert abs(g.pos[0, 2] - z) < 1e-6
    # the instantaneous mixer climbs faster
    g0 = orc.OracleGroup(0, _B(1))
    _rate(g0, u_total)
    for _ in range(steps):
        g0.step(dt)
    assert abs(g0.vel[0, 2] - (4 * u / M - G) * t) < 1e-9 and g0.vel[0, 2] > g.vel[0, 2]


def test_small_tau_limit_is_the_reference_mixer():
    """tau_m -> 0: the tick-mean thrust is the command, i.e. the (pinned)
    instantaneous mixer of the reference, on a random position-level swarm."""
    rng = np.random.default_rng(3)
    n = 16
    pos = rng.uniform(-5, 5, (n, 3))
    a, b = orc.OracleGroup(0, _B(n, pos)), orc.OracleGroup(0, _B(n, pos), motor_tau=1e-12)
    sp = pos + rng.uniform(-1, 1, (n, 3))
    for g in (a, b):
        g.cmd_values[:, :3] = sp
    for _ in range(100):
        a.step(1e-3)
        b.step(1e-3)
    np.testing.assert_allclose(b.state13(), a.state13(), rtol=0, atol=1e-9)


def test_motor_level_commands_lag_too():
    """MOTOR rows: u = k_t clip(rpm)^2 per rotor (quad.py:134-137); the yaw
    torque builds up through the lag."""
    tau, dt = 0.02, 1e-3
    g = orc.OracleGroup(0, _B(1), motor_tau=tau)
    rpm = np.array([12000.0, 8000.0, 12000.0, 8000.0])
    g.cmd_level[0] = 2
    g.cmd_values[0] = 0.0
    g.cmd_values[0, :4] = rpm
    for _ in range(100):
        g.step(dt)
    u = 1e-8 * rpm ** 2
    want = u + (M * G / 4 - u) * math.exp(-0.1 / tau)
    np.testing.assert_allclose(g.motor[0], want, rtol=1e-12)


def test_dead_and_faulted_rows_keep_thrusts():
    g = orc.OracleGroup(0, _B(3), motor_tau=0.05)
    _rate(g, 2 * M * G)
    g.alive[1] = 0
    g.cmd_values[2, 0] = np.nan           # NaN rate command: row 2 faults
    before = g.motor.copy()
    faults = g.step(1e-3)
    assert faults.tolist() == [2]
    np.testing.assert_array_equal(g.motor[1:], before[1:])
    assert g.motor[0, 0] > before[0, 0]


def test_bad_tau_rejected():
    g = orc.OracleGroup(0, _B(1), motor_tau=0.05)
    g.motor_tau = 0.0
    with pytest.raises(ValueError):
        g.step(1e-3)
