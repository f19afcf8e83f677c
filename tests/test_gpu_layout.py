"""The device layout's compensated position (include/swarmstep_b200.h
COL_POS_LO: three 10-bit low parts in units of ulp(hi) / 512): float64
positions pushed to the device and pulled back keep ~33 significant bits."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def test_packed_position_low_part_round_trip():
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    rng = np.random.default_rng(5)
    n = 4096
    scale = 10.0 ** rng.uniform(-3, 4, (n, 1))          # 1 mm .. 10 km
    pos = rng.uniform(-1, 1, (n, 3)) * scale
    pos[:3] = [[0.0, 0.0, 0.0], [1e-30, -2e-38, 3.0], [2.0 ** 20, -(2.0 ** 20) + 1e-3, 1e-7]]
    g = B200QuadGroup(0, batch_create(0, n, pos))
    back = g.batch.pos
    hi = pos.astype(np.float32)
    unit = np.maximum(np.spacing(np.abs(hi)).astype(np.float64) / 512.0, 2.0 ** -126)
    err = np.abs(back - pos)
    # the stored low part is rounded to the nearest unit (plus the float32
    # rounding of lo itself, 2^-24 relative)
    assert np.all(err <= 0.5 * unit * (1 + 1e-6) + np.abs(pos - hi) * 2.0 ** -23), float(np.max(err / unit))
    # ~33 significant bits: far below the float32 ulp of the coordinate
    # (where ulp(hi) / 512 is a normal float, i.e. |hi| >= 2^-94)
    ulp = np.spacing(np.abs(hi)).astype(np.float64)
    m = ulp >= 2.0 ** -117
    assert np.max(err[m] / ulp[m]) <= 1.0 / 1000


def test_plain_position_mode_has_no_low_part():
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    pos = np.array([[100.0 + 1e-6, -3.25, 7.0]])
    g = B200QuadGroup(0, batch_create(0, 1, pos), compensated=False)
    np.testing.assert_array_equal(g.batch.pos, pos.astype(np.float32).astype(np.float64))


def test_compensated_position_through_the_origin():
    """Agents crossing a coordinate plane at speed, stepped 10 ticks per launch:
    the fold of the launch-local accumulator meets |hi| << |increment| (the
    Fast2Sum precondition fails) and the packed low part sees tiny hi; the
    per-step error stays within the parity bar and the 30-tick trajectory
    within 1e-6 m of the float64 oracle."""
    from gpu_util import PER_STEP_TOL, f32, gpu_state, make_group, oracle_twin, rel_errors
    from scenarios import Scenario
    rng = np.random.default_rng(11)
    n = 256
    pos = rng.uniform(-0.02, 0.02, (n, 3))
    vel = rng.uniform(-20, 20, (n, 3))
    q = np.tile([1.0, 0, 0, 0], (n, 1))
    g = make_group(Scenario("origin", n, 1e-3, 1, pos, vel, q, np.zeros((n, 3)), record=[]))
    og = oracle_twin(g)
    for _ in range(3):
        g.step_k(1e-3, 10)
        for _ in range(10):
            og.step(f32(1e-3))
    st = gpu_state(g)
    assert np.max(np.abs(st["pos"] - og.pos)) < 1e-6
    crossed = np.any(np.sign(st["pos"]) != np.sign(pos), axis=1)
    assert crossed.mean() > 0.5
    og2 = oracle_twin(g)
    g.step(1e-3)
    og2.step(f32(1e-3))
    for k, v in rel_errors(gpu_state(g), og2).items():
        assert v <= PER_STEP_TOL, (k, v)
