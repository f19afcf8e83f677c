"""The function-level API (paper_2308_12698_b200.functional, csrc/ops.cu)
against the golden vectors produced by running the reference's own functions
(tests/golden/functions.npz) and against the reference's known-answer tests
(test_quad.py, test_control.py), at float32 tolerances.  Mirrors
tests/test_oracle.py, which pins the float64 oracle to the same vectors."""

import math

import numpy as np
import pytest

from conftest import cuda_ok
from golden_io import load_functions

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

TOL = 1e-5   # north_star per-step relative bound


def _rel(got, want, floor):
    scale = np.maximum(np.abs(want), floor)
    return float(np.max(np.abs(np.asarray(got) - want) / scale))


class _Batch:
    def __init__(self, s13, alive=None):
        n = s13.shape[0]
        self.agent_ids = np.arange(n, dtype=np.uint64)
        self.pos, self.vel = s13[:, 0:3].copy(), s13[:, 3:6].copy()
        self.quat, self.omega = s13[:, 6:10].copy(), s13[:, 10:13].copy()
        self.alive = np.ones(n, bool) if alive is None else np.asarray(alive, bool).copy()


@pytest.fixture(scope="module")
def fx():
    return load_functions()


@pytest.fixture(scope="module")
def F():
    from paper_2308_12698_b200 import functional
    return functional


@pytest.fixture(scope="module")
def P():
    from paper_2308_12698_b200 import default_quad_params
    return default_quad_params()


# ------------------------------------------------------------ golden vectors
def test_deriv_golden(F, fx, P):
    b = _Batch(fx["deriv_state"])
    d = F.dynamics_deriv(b, fx["deriv_fc"], fx["deriv_tau"], P)
    got = np.hstack([d.pos, d.vel, d.quat, d.omega])
    assert _rel(got, fx["deriv_out"], 1.0) < TOL


def test_rk4_golden_20_steps(F, fx, P):
    b = _Batch(fx["rk4_state0"], fx["rk4_alive0"])
    for k in range(fx["rk4_fc"].shape[0]):
        assert F.rk4_step(b, fx["rk4_fc"][k], fx["rk4_tau"][k], P, 1e-3).size == 0
    want = fx["rk4_state20"]
    got = np.hstack([b.pos, b.vel, b.quat, b.omega])
    assert _rel(got[:, 0:3], want[:, 0:3], 1.0) < TOL
    assert _rel(got[:, 3:13], want[:, 3:13], 1.0) < 20 * TOL     # 20 steps of float32 rounding
    np.testing.assert_array_equal(b.alive, fx["rk4_alive20"])
    dead = ~fx["rk4_alive0"]
    np.testing.assert_array_equal(got[dead], fx["rk4_state0"][dead])          # dead rows untouched


def test_rk4_fault_revert_golden(F, fx, P):
    # test_quad.py:171-179: a 1e308 torque faults row 1, which keeps its state
    from paper_2308_12698_b200 import batch_create
    b = batch_create(0, 2, np.zeros((2, 3)))
    ids = F.rk4_step(b, np.zeros(2), np.array([[0.0, 0.0, 0.0], [3e38, 0.0, 0.0]]), P, 1e6)
    assert ids.tolist() == fx["rk4_fault_ids"].tolist() == [1]
    np.testing.assert_array_equal(b.alive, fx["rk4_fault_alive"])
    np.testing.assert_array_equal(np.hstack([b.pos, b.vel, b.quat, b.omega])[1], fx["rk4_fault_state"][1])


def test_mixer_golden(F, fx, P):
    mx = F.mix_to_motors(fx["mix_fc"], fx["mix_tau"], P)
    assert _rel(mx.motors, fx["mix_motors"], 1.0) < TOL
    assert _rel(np.hstack([mx.f_c[:, None], mx.tau]), fx["mix_realized"], 1.0) < TOL
    np.testing.assert_array_equal(mx.saturated, fx["mix_sat"])


def test_pid_golden_30_steps(F, fx):
    n = fx["pid_omega"].shape[1]
    st = F.RatePidState(n)
    dt = float(fx["pid_dt"])
    from paper_2308_12698_b200 import default_rate_gains
    for k in range(fx["pid_omega"].shape[0]):
        sp = F.RateSetpoint(fx["pid_sp"][k], fx["pid_fsp"][k])
        f_c, tau = F.rate_pid_step(fx["pid_omega"][k], sp, default_rate_gains(), dt, st, fx["pid_alive"][k])
        assert _rel(tau, fx["pid_tau"][k], 0.1) < TOL, k
        assert _rel(f_c, fx["pid_fc"][k], 1.0) < TOL
        assert _rel(st.integral, fx["pid_integral"][k], 0.2) < TOL


def test_outer_loop_golden(F, fx, P):
    from paper_2308_12698_b200 import default_outer_gains
    sp = F.PosSetpoint(fx["outer_p_sp"], fx["outer_v_sp"], fx["outer_yaw"])
    res = F.position_outer_loop(fx["outer_pos"], fx["outer_vel"], fx["outer_quat"], fx["outer_alive"], sp, P,
                                default_outer_gains())
    assert _rel(res.setpoint.omega_sp, fx["outer_omega_sp"], 1.0) < 5 * TOL
    assert _rel(res.setpoint.f_c_sp, fx["outer_f_c"], 1.0) < TOL
    np.testing.assert_array_equal(res.low_thrust, fx["outer_low"])


# ------------------------------------------------ the reference's own KATs
def test_kat_rotor(F, P):
    # test_quad.py:38-42
    th, tq, sat = F.rotor_thrust_torque(np.array([10000.0, -5.0, 5e4]), P)
    assert th[0] == pytest.approx(1.0, rel=1e-6) and tq[0] == pytest.approx(0.01, rel=1e-6)
    assert th[1] == 0.0 and th[2] == pytest.approx(16.0, rel=1e-6)
    assert sat.tolist() == [False, True, True]


def test_kat_mixer_hover_and_negative_demand(F, P):
    # test_quad.py:78-97
    mx = F.mix_to_motors(np.array([P.m * P.g]), np.zeros((1, 3)), P)
    np.testing.assert_allclose(mx.motors[0], 2.4525, rtol=1e-6)
    assert not mx.saturated[0]
    mx = F.mix_to_motors(np.array([0.0]), np.array([[1.0, 0.0, 0.0]]), P)
    assert mx.saturated[0] and np.all(mx.motors[0] >= 0.0)


def test_kat_derivative(F, P):
    # test_quad.py:110-125: hover is an equilibrium, free fall, principal-axis spin
    from paper_2308_12698_b200 import batch_create
    b = batch_create(0, 3, np.zeros((3, 3)), omega=[[0, 0, 0], [0, 0, 0], [0, 0, 5.0]])
    d = F.dynamics_deriv(b, np.array([P.m * P.g, 0.0, P.m * P.g]), np.zeros((3, 3)), P)
    np.testing.assert_allclose(d.vel[0], 0.0, atol=1e-6)
    np.testing.assert_allclose(d.vel[1], [0, 0, -9.81], rtol=1e-6)
    np.testing.assert_allclose(d.omega[2], 0.0, atol=1e-6)


def test_kat_one_step_free_fall(F, P):
    # test_quad.py:139-144: dt = 0.1 free fall -> v_z = -0.981, p_z = -0.04905
    from paper_2308_12698_b200 import batch_create
    b = batch_create(0, 1, np.zeros((1, 3)))
    F.rk4_step(b, np.zeros(1), np.zeros((1, 3)), P, 0.1)
    assert b.vel[0, 2] == pytest.approx(-0.981, rel=1e-6)
    assert b.pos[0, 2] == pytest.approx(-0.04905, rel=1e-6)


def test_kat_pid(F):
    # test_control.py:36-77: P term, integral clamp, no setpoint kick, D on measurement
    from paper_2308_12698_b200 import PidGains
    g = PidGains(kp=0.1, ki=0.0, kd=0.0, i_limit=1.0)
    st = F.RatePidState(1)
    f_c, tau = F.rate_pid_step(np.zeros((1, 3)), F.RateSetpoint(np.array([[1.0, 0, 0]]), np.array([3.0])), g, 0.01,
                               st, np.array([True]))
    assert tau[0, 0] == pytest.approx(0.1, rel=1e-6) and f_c[0] == 3.0
    g = PidGains(kp=0.0, ki=1.0, kd=0.0, i_limit=0.2)
    st = F.RatePidState(1)
    for _ in range(100):
        F.rate_pid_step(np.zeros((1, 3)), F.RateSetpoint(np.array([[1.0, 0, 0]]), np.zeros(1)), g, 0.01, st,
                        np.array([True]))
    assert st.integral[0, 0] == pytest.approx(0.2, rel=1e-6)
    g = PidGains(kp=0.0, ki=0.0, kd=0.5, i_limit=1.0)
    st = F.RatePidState(1)
    F.rate_pid_step(np.array([[1.0, 0, 0]]), F.RateSetpoint(np.zeros((1, 3)), np.zeros(1)), g, 0.1, st,
                    np.array([True]))                                     # first sample: no D
    _, tau = F.rate_pid_step(np.array([[2.0, 0, 0]]), F.RateSetpoint(np.zeros((1, 3)), np.zeros(1)), g, 0.1, st,
                             np.array([True]))
    assert tau[0, 0] == pytest.approx(-0.5 * (2.0 - 1.0) / 0.1, rel=1e-6)
    # dead rows: zero output, frozen state
    st = F.RatePidState(1)
    f_c, tau = F.rate_pid_step(np.ones((1, 3)), F.RateSetpoint(np.zeros((1, 3)), np.ones(1)), g, 0.1, st,
                               np.array([False]))
    assert f_c[0] == 0.0 and np.all(tau == 0.0) and not st.has_prev[0]


def test_kat_outer_loop(F, P):
    # test_control.py:140-189
    from paper_2308_12698_b200 import OuterGains, default_outer_gains
    z = np.zeros((1, 3))
    q0 = np.array([[1.0, 0, 0, 0]])
    hover = F.PosSetpoint(z, z, np.zeros(1))
    r = F.position_outer_loop(z, z, q0, np.array([True]), hover, P, default_outer_gains())
    assert r.setpoint.f_c_sp[0] == pytest.approx(P.m * P.g, rel=1e-6) and not r.low_thrust[0]
    kat = OuterGains(kp_pos=1.0, kv=0.0, k_att=8.0)
    r = F.position_outer_loop(z, z, q0, np.array([True]), F.PosSetpoint(np.array([[0, 0, 1.0]]), z, np.zeros(1)),
                              P, kat)
    assert r.setpoint.f_c_sp[0] == pytest.approx(P.m * (1.0 + 9.81), rel=1e-6)
    r = F.position_outer_loop(z, z, q0, np.array([True]), F.PosSetpoint(z, z, np.array([np.pi / 2])), P,
                              default_outer_gains())
    assert r.setpoint.omega_sp[0, 2] > 0 and np.allclose(r.setpoint.omega_sp[0, :2], 0.0, atol=1e-6)
    r = F.position_outer_loop(z, z, q0, np.array([True]), F.PosSetpoint(np.array([[0, 0, -9.81]]), z, np.zeros(1)),
                              P, kat)
    assert r.low_thrust[0] and r.setpoint.f_c_sp[0] == pytest.approx(P.m * kat.a_cmd_min, rel=1e-6)
    qt = np.array([[math.cos(math.pi / 8), math.sin(math.pi / 8), 0, 0]])
    r = F.position_outer_loop(z, z, qt, np.array([True]), hover, P, kat)
    assert r.setpoint.f_c_sp[0] == pytest.approx(P.m * P.g * math.cos(math.pi / 4), rel=2e-6)
    r = F.position_outer_loop(np.zeros((2, 3)), np.zeros((2, 3)), np.tile(q0, (2, 1)), np.array([False, True]),
                              F.PosSetpoint(np.ones((2, 3)), np.zeros((2, 3)), np.zeros(2)), P, default_outer_gains())
    assert r.setpoint.f_c_sp[0] == 0.0 and np.all(r.setpoint.omega_sp[0] == 0.0) and r.setpoint.f_c_sp[1] > 0


def test_errors_follow_the_reference(F, P):
    from paper_2308_12698_b200 import InvalidStateError, ValidationError, batch_create, default_outer_gains
    from paper_2308_12698_b200 import default_rate_gains
    b = batch_create(0, 1, np.zeros((1, 3)))
    with pytest.raises(ValidationError):
        F.rk4_step(b, np.zeros(1), np.zeros((1, 3)), P, 0.0)
    with pytest.raises(ValidationError):
        F.rate_pid_step(np.zeros((1, 3)), F.RateSetpoint(np.zeros((1, 3)), np.zeros(1)), default_rate_gains(), -1.0,
                        F.RatePidState(1), np.array([True]))
    with pytest.raises(InvalidStateError):
        F.position_outer_loop(np.zeros((1, 3)), np.zeros((1, 3)), np.array([[np.nan, 0, 0, 0]]), np.array([True]),
                              F.PosSetpoint(np.zeros((1, 3)), np.zeros((1, 3)), np.zeros(1)), P,
                              default_outer_gains())


def test_device_tensors_stay_on_device(F, P):
    import torch
    n = 1000
    rng = np.random.default_rng(5)
    fc = torch.tensor(rng.uniform(0, 60, n), dtype=torch.float32, device="cuda")
    tau = torch.tensor(rng.uniform(-1, 1, (n, 3)), dtype=torch.float32, device="cuda")
    mx = F.mix_to_motors(fc, tau, P)
    assert mx.motors.is_cuda and mx.motors.shape == (n, 4)
    host = F.mix_to_motors(fc.cpu().double().numpy(), tau.cpu().double().numpy(), P)
    np.testing.assert_array_equal(mx.motors.cpu().numpy(), host.motors.astype(np.float32))
