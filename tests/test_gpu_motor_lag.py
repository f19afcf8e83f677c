"""GPU tests of the opt-in first-order rotor lag (swarmstep_quad_step_lag)
against the float64 oracle's lag model (tests/test_motor_lag.py pins that
model to closed forms; the reference has no rotor dynamics, so parity with the
reference itself is unpinned for tau_m > 0 -- SURVEY.md 8(a))."""

import math

import numpy as np
import pytest

from conftest import cuda_ok
from gpu_util import FLOORS, PER_STEP_TOL, f32, gpu_state, make_group, oracle_twin, rel_errors
from scenarios import ALL, Scenario, run_script

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

TAU = 0.03


def _lag_twin(g):
    og = oracle_twin(g)
    og.motor_tau = g.motor_tau
    og.motor = g.motor_thrusts()
    return og


@pytest.mark.parametrize("name", ["mixed", "pos_random", "hover_rate"])
def test_lag_per_step_relative_error(name):
    sc = ALL[name]()
    g = make_group(sc, motor_tau=TAU)
    run_script(g, Scenario(**{**sc.__dict__, "ticks": min(sc.ticks, 25), "record": []}))
    worst = {}
    for _ in range(30):
        og = _lag_twin(g)
        og.step(f32(sc.dt))
        g.step(sc.dt)
        e = rel_errors(gpu_state(g), og)
        alive = og.alive.astype(bool)
        w = og.motor[alive]
        e["motor"] = float(np.max(np.abs(g.motor_thrusts()[alive] - w) / np.maximum(np.abs(w), 1.0))) if w.size else 0.0
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
    for k, v in worst.items():
        assert v <= PER_STEP_TOL, f"{name}: lag per-step {k} rel err {v:.2e} (floors {FLOORS})"


def test_lag_step_response_closed_form():
    """Thrust step from hover: rotor thrust u + (f0 - u) e^(-t/tau), climb
    rate = the exact thrust impulse (tests/test_motor_lag.py), in float32."""
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    n, dt, steps = 256, 1e-3, 300
    g = B200QuadGroup(0, batch_create(0, n, np.zeros((n, 3))), motor_tau=TAU)
    sp = np.zeros((n, 4))
    sp[:, 3] = 2 * 9.81
    g.set_setpoints(sp, level=1)
    for _ in range(steps // 10):
        g.step_k(dt, 10)
    t = dt * steps
    f0, u = 9.81 / 4, 2 * 9.81 / 4
    np.testing.assert_allclose(g.motor_thrusts(), u + (f0 - u) * math.exp(-t / TAU), rtol=2e-6)
    vz = (4 * u - 9.81) * t + 4 * (f0 - u) * TAU * (1 - math.exp(-t / TAU))
    np.testing.assert_allclose(g.batch.vel[:, 2], vz, rtol=1e-5)


def test_lag_fused_equals_single_ticks_bitwise():
    """Plain float32 position: fused ticks are bit-identical to one-tick
    launches (the compensated form is covered in test_gpu_parity)."""
    sc = ALL["mixed"]()
    a, b = make_group(sc, motor_tau=TAU, compensated=False), make_group(sc, motor_tau=TAU, compensated=False)
    for g in (a, b):
        run_script(g, Scenario(**{**sc.__dict__, "ticks": 10, "record": []}))
    a.step_k(sc.dt, 8)
    for _ in range(8):
        b.step(sc.dt)
    sa, sb = gpu_state(a), gpu_state(b)
    for k in ("pos", "vel", "quat", "omega", "integral", "alive"):
        np.testing.assert_array_equal(sa[k], sb[k])
    np.testing.assert_array_equal(a.motor_thrusts(), b.motor_thrusts())


def test_lag_faults_and_dead_rows_keep_thrusts():
    """fault_nan: the NaN RATE / MOTOR commands fault exactly rows 3 and 11 (as
    in the reference; the inf rate command of row 12 saturates the mixer and
    stays finite); a faulted or dead row keeps its rotor thrusts from then on."""
    sc = ALL["fault_nan"]()
    g = make_group(sc, motor_tau=TAU)
    snaps = []
    _, _, faults = run_script(g, sc, on_tick=lambda t, grp: snaps.append((grp.batch.alive.copy(), grp.motor_thrusts())))
    assert sorted(i for f in faults.values() for i in f) == [3, 11]
    for (al0, m0), (al1, m1) in zip(snaps, snaps[1:]):
        np.testing.assert_array_equal(m1[~al0], m0[~al0])     # dead before the tick: frozen
        assert np.all(al1 <= al0)
    assert not snaps[-1][0][[3, 11]].any() and snaps[-1][0][12]


def test_tau_zero_is_the_reference_path():
    from paper_2308_12698_b200 import ValidationError
    sc = ALL["pos_random"]()
    a, b = make_group(sc), make_group(sc, motor_tau=0.0)
    a.step_k(sc.dt, 5)
    b.step_k(sc.dt, 5)
    np.testing.assert_array_equal(gpu_state(a)["pos"], gpu_state(b)["pos"])
    with pytest.raises(ValidationError):
        b.motor_thrusts()
    with pytest.raises(ValidationError):
        make_group(sc, motor_tau=-1.0)


@pytest.mark.parametrize("k", [1, 7])
def test_lag_kernel_variants_bit_identical(k):
    """The paired (FFMA2) rotor-lag kernel == the direct one, bit for bit,
    state and rotor thrusts, all levels and faults included."""
    outs = []
    for kern in ("direct", "pair"):
        sc = ALL["fault_nan"](n=256, ticks=12)
        g = make_group(sc, motor_tau=TAU)
        g.kernel = kern
        run_script(g, Scenario(**{**sc.__dict__, "ticks": 8, "record": []}))
        for _ in range(3):
            g.step_k(sc.dt, k)
        st = gpu_state(g)
        outs.append({**{q: st[q].copy() for q in ("pos", "vel", "quat", "omega", "integral", "alive")},
                     "motor": g.motor_thrusts()})
    for q in outs[0]:
        np.testing.assert_array_equal(outs[0][q], outs[1][q], err_msg=q)


def test_lag_graph_replay_bit_identical():
    """TickGraph (CUDA graph of circle feed + 1-tick steps) drives the rotor-lag
    kernel like eager ticks, bit for bit, rotor thrusts included."""
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    from paper_2308_12698_b200.feed import CircleFeed, TickGraph
    n, dt, T = 300, 2e-3, 20

    def grp():
        ph = 2 * np.pi * np.arange(n) / n
        pos = np.stack([5 * np.cos(ph), 5 * np.sin(ph), np.full(n, 10.0)], axis=1)
        return B200QuadGroup(0, batch_create(0, n, pos), motor_tau=TAU)

    ga, gb = grp(), grp()
    graph = TickGraph(ga, dt, T, feed=CircleFeed(ga, dt))
    for _ in range(3):
        graph.replay()
    ga.collect_faults()
    fb = CircleFeed(gb, dt)
    for _ in range(3 * T):
        fb.apply()
        gb.step(dt)
    assert ga.batch.pos.tobytes() == gb.batch.pos.tobytes()
    np.testing.assert_array_equal(ga.motor_thrusts(), gb.motor_thrusts())
