"""The reference's own known-answer tests, run through the fused sm_100a step
(the kernel has no per-function entry points, so each KAT is observed through
one group tick: the outer loop's outputs are the stale inner-loop setpoints the
kernel stores, core.py:178-182).  Tolerances are the reference's, re-derived
for float32."""

import math

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

M, G = 1.0, 9.81


def _group(n=1, quat=None, omega=None, outer=None):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    b = batch_create(0, n, np.zeros((n, 3)), quat=quat, omega=omega)
    return B200QuadGroup(0, b, outer_gains=outer)


def _outer(g, sp):
    """One tick at POS level; returns the outer loop's (omega_sp, f_c_sp)."""
    g.set_setpoints(np.asarray(sp, float).reshape(g.n, 7))
    g.step(1e-3)
    ps = g.pid_state_dict()
    return ps["omega_sp"], ps["f_c_sp"]


def _kat_gains():
    from paper_2308_12698_b200 import OuterGains
    return OuterGains(kp_pos=1.0, kv=0.0, k_att=8.0)


def test_outer_equilibrium():
    # test_control.py:141-147
    w, f = _outer(_group(2), np.zeros((2, 7)))
    np.testing.assert_allclose(f, M * G, rtol=1e-6)
    np.testing.assert_allclose(w, 0.0, atol=1e-6)


def test_outer_unit_position_error():
    # test_control.py:149-155: f_c = m (1 + g)
    w, f = _outer(_group(1, outer=_kat_gains()), [[0, 0, 1.0, 0, 0, 0, 0]])
    assert f[0] == pytest.approx(M * (1.0 + G), rel=1e-6)
    np.testing.assert_allclose(w, 0.0, atol=1e-6)


def test_outer_pure_yaw_error():
    # test_control.py:157-162
    w, _ = _outer(_group(1), [[0, 0, 0, 0, 0, 0, math.pi / 2]])
    assert w[0, 2] > 0.0
    np.testing.assert_allclose(w[0, :2], 0.0, atol=1e-6)


def test_outer_free_fall_floor():
    # test_control.py:164-172: a_cmd ~ 0 -> low-thrust floor m a_min
    gains = _kat_gains()
    w, f = _outer(_group(1, outer=gains), [[0, 0, -G, 0, 0, 0, 0]])
    assert f[0] == pytest.approx(M * gains.a_cmd_min, rel=1e-6)


def test_outer_tilted_thrust_projection():
    # test_control.py:174-180: 45 deg roll -> f_c = m g cos 45
    q = [math.cos(math.pi / 8), math.sin(math.pi / 8), 0.0, 0.0]
    _, f = _outer(_group(1, quat=[q], outer=_kat_gains()), np.zeros((1, 7)))
    assert f[0] == pytest.approx(M * G * math.cos(math.pi / 4), rel=2e-6)


def test_outer_dead_rows_keep_zero():
    # test_control.py:182-189 (dead rows: no outer-loop output, state frozen)
    g = _group(2)
    g.mark_dead([0])
    w, f = _outer(g, np.ones((2, 7)) * [1, 1, 1, 0, 0, 0, 0])
    assert f[0] == 0.0 and np.all(w[0] == 0.0) and f[1] > 0.0


def test_rotor_model_motor_level():
    # test_quad.py:38-42: f(10000 rpm) = k_t 1e8 = 1 N per rotor, no torque;
    # 4 N of thrust < m g: v_z after one tick = (4/m - g) dt, no rotation
    g = _group(1)
    g.set_setpoints(np.array([[1e4, 1e4, 1e4, 1e4]]), level="motor")
    dt = 1e-3
    g.step(dt)
    b = g.batch
    assert b.vel[0, 2] == pytest.approx((4.0 / M - G) * dt, rel=1e-6)
    np.testing.assert_allclose(b.omega[0], 0.0, atol=1e-12)
    np.testing.assert_allclose(b.quat[0], [1, 0, 0, 0], atol=1e-7)


def test_mixer_saturation_clamps():
    # test_quad.py:92-97 through the step: a RATE command demanding more
    # collective thrust than 4 f_max climbs at (4 f_max / m - g)
    g = _group(1)
    g.set_setpoints(np.array([[0, 0, 0, 1000.0]]), level="rate")
    g.step(1e-3)
    assert g.batch.vel[0, 2] == pytest.approx((4 * 16.0 / M - G) * 1e-3, rel=1e-6)


def test_torque_free_momentum_drift():
    # test_quad.py:217-234, float32 tolerance: spin with zero torque (MOTOR
    # level, rotors off) -> world-frame angular momentum conserved
    rng = np.random.default_rng(12)
    n = 64
    g = _group(n, omega=rng.uniform(-0.5, 0.5, (n, 3)))
    g.set_setpoints(np.zeros((n, 4)), level="motor")
    idiag = np.array([0.01, 0.01, 0.02])

    def momentum(b):
        q, w = b.quat, b.omega * idiag
        qw, qx, qy, qz = q.T
        r0 = np.stack([1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz), 2 * (qx * qz + qw * qy)], 1)
        r1 = np.stack([2 * (qx * qy + qw * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx)], 1)
        r2 = np.stack([2 * (qx * qz - qw * qy), 2 * (qy * qz + qw * qx), 1 - 2 * (qx * qx + qy * qy)], 1)
        return np.stack([(r0 * w).sum(1), (r1 * w).sum(1), (r2 * w).sum(1)], 1)

    m0 = momentum(g.batch)
    for _ in range(1000):
        g.step_k(1e-3, 10)
    drift = np.linalg.norm(momentum(g.batch) - m0, axis=1) / np.linalg.norm(m0, axis=1)
    assert drift.max() < 2e-4, drift.max()
    assert np.max(np.abs(np.linalg.norm(g.batch.quat, axis=1) - 1.0)) < 1e-6
