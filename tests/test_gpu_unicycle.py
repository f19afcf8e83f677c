"""GPU unicycle group (f4) against the reference UnicycleGroup golden run and
the reference's own unicycle known-answer tests (test_core.py:33-60)."""

import numpy as np
import pytest

from conftest import cuda_ok
from golden_io import GOLDEN
from scenarios import Scenario, run_script

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _ugroup(pos, quat=None, params=None, id_base=0):
    from paper_2308_12698_b200 import batch_create
    from paper_2308_12698_b200.unicycle import B200UnicycleGroup
    pos = np.asarray(pos, float).reshape(-1, 3)
    return B200UnicycleGroup(1, batch_create(1, pos.shape[0], pos, quat=quat, id_base=id_base), params)


def _cmd(aid, v, w):
    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    return AgentCommand(aid, CommandLevel.UNICYCLE, (float(v), float(w)))


def test_golden_unicycle_scenario():
    z = dict(np.load(GOLDEN / "scenario_unicycles.npz"))
    sc = Scenario.from_arrays(z)
    g = _ugroup(sc.pos, sc.quat)
    state = lambda g: dict(pos=g.batch.pos.copy(), vel=g.batch.vel.copy(), quat=g.batch.quat.copy(),
                           omega=g.batch.omega.copy(), alive=g.batch.alive.copy(), cmd=g.cmd.copy())
    got, ok, _ = run_script(g, sc, state_of=state)
    np.testing.assert_array_equal(ok, z["cmd_ok"])
    for i, t in enumerate(z["rec_ticks"]):
        a = z["rec_alive"][i]
        np.testing.assert_array_equal(got[int(t)]["alive"], a)
        np.testing.assert_allclose(got[int(t)]["pos"][a], z["rec_pos"][i][a], atol=5e-5)
        np.testing.assert_allclose(got[int(t)]["vel"][a], z["rec_vel"][i][a], atol=5e-5)
        # quaternion sign is fixed by yaw_quat: compare directly
        np.testing.assert_allclose(got[int(t)]["quat"][a], z["rec_quat"][i][a], atol=2e-5)
        np.testing.assert_allclose(got[int(t)]["omega"][a], z["rec_omega"][i][a], atol=1e-6)
        dead = ~a
        if dead.any():   # dead rows untouched
            np.testing.assert_array_equal(got[int(t)]["pos"][dead], got[int(t)]["pos"][dead])


def test_kat_straight_pivot_arc_clamp_dead():
    from paper_2308_12698_b200.unicycle import UnicycleParams
    g = _ugroup([[0, 0, 0]])
    g.apply_command(_cmd(0, 1.0, 0.0))
    g.step(1.0)
    np.testing.assert_allclose(g.batch.pos[0], [1.0, 0.0, 0.0], atol=1e-6)      # test_core.py:34-37
    g = _ugroup([[0, 0, 0]], params=UnicycleParams(omega_max=5.0))
    g.apply_command(_cmd(0, 0.0, np.pi))
    g.step(1.0)
    np.testing.assert_allclose(g.batch.pos[0], 0.0, atol=1e-6)                  # test_core.py:39-43
    from paper_2308_12698_b200.state import quat_yaw
    assert abs(abs(quat_yaw(g.batch.quat[0])) - np.pi) < 1e-5
    g = _ugroup([[0, 0, 0]])
    g.apply_command(_cmd(0, 1.0, 1.0))
    g.step(np.pi)
    np.testing.assert_allclose(g.batch.pos[0], [0.0, 2.0, 0.0], atol=2e-6)      # test_core.py:45-48
    g = _ugroup([[0, 0, 0]], params=UnicycleParams(v_max=2.0))
    g.apply_command(_cmd(0, 100.0, 0.0))
    g.step(1.0)
    np.testing.assert_allclose(g.batch.pos[0], [2.0, 0.0, 0.0], atol=1e-6)      # test_core.py:50-53
    g = _ugroup([[0, 0, 0], [0, 0, 0]])
    g.mark_dead([0])
    assert not g.apply_command(_cmd(0, 1.0, 1.0))
    g.apply_command(_cmd(1, 1.0, 1.0))
    g.step(1.0)
    np.testing.assert_array_equal(g.batch.pos[0], 0.0)                           # test_core.py:55-60
    assert g.batch.pos[1, 0] != 0.0


def test_small_turn_rate_is_accurate():
    """w dt ~ 1e-7: the cancellation-free arc form keeps float32 exact to ~1e-7 m."""
    g = _ugroup([[0, 0, 0]])
    g.apply_command(_cmd(0, 1.0, 1e-5))
    for _ in range(100):
        g.step(0.01)
    np.testing.assert_allclose(g.batch.pos[0, 0], 1.0, atol=1e-5)
    assert abs(g.batch.pos[0, 1] - 0.5 * 1e-5 * 1.0) < 1e-7
