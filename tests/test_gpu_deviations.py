"""Pinned behaviour where the float32 device path deliberately differs from the
float64 reference (DESIGN.md 4 "Documented deviations"), and regressions for
host-side ordering bugs (stream order of caller tensors, has_prev across a
host-state push)."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _group(n=64, seed=0):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-20, 20, (n, 3)) + [0, 0, 50]
    b = batch_create(0, n, pos, omega=rng.uniform(-0.3, 0.3, (n, 3)))
    return B200QuadGroup(0, b), pos


def _twin_with(g, overrides):
    """Oracle twin of g's state whose command rows carry the caller's float64
    values (the reference keeps what was commanded; the device holds float32)."""
    from gpu_util import gpu_state, oracle_twin
    st = gpu_state(g)
    og = oracle_twin(g, st)
    for row, vals in overrides.items():
        og.cmd_values[row] = vals
    return st, og


def test_setpoints_beyond_float32_range_follow_the_reference():
    """Finite POS setpoints beyond float32 range (1e39 m, -1e39 m/s) saturate
    at +-FLT_MAX in the device command store, and the outer loop takes the
    direction of the overflowing acceleration command from a scaled copy: the
    rows fly like the float64 reference (which has the range), within the
    per-step tolerance, instead of faulting.  (Residual deviation, DESIGN.md
    4: when several components exceed float32 range by DIFFERENT factors,
    saturating them changes the commanded direction.)"""
    from gpu_util import PER_STEP_TOL, f32, gpu_state, rel_errors

    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    g, pos = _group()
    g.step(1e-3)
    big = {5: (1e39, 0.0, 10.0, 0.0, 0.0, 0.0, 0.0), 6: (0.0, -1e39, 1e39, 0.0, 0.0, 0.0, 0.3),
           7: (pos[7, 0], pos[7, 1], pos[7, 2], -1e39, 0.0, 0.0, -0.2)}
    for row, v in big.items():
        assert g.apply_command(AgentCommand(row, CommandLevel.POS, v))
    for _ in range(3):
        st, og = _twin_with(g, big)
        assert g.step(1e-3).size == 0
        assert og.step(f32(1e-3)).size == 0
        err = rel_errors(gpu_state(g), og)
        assert all(v <= PER_STEP_TOL for v in err.values()), err
    assert g.batch.alive[[5, 6, 7]].all()


def test_large_yaw_setpoints_are_reduced_before_rounding():
    """A yaw setpoint of ~1000 rad is reduced to [-pi, pi] in float64 before
    the float32 command store (a float32 yaw near 1000 carries 3e-5 rad of
    rounding): per-step parity against the reference's float64 yaw holds."""
    from gpu_util import PER_STEP_TOL, f32, gpu_state, rel_errors

    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    g, pos = _group()
    cmds = {i: (pos[i, 0] + 0.5, pos[i, 1], pos[i, 2], 0.0, 0.0, 0.0, 1000.3 + 7.7 * i) for i in range(0, g.n, 3)}
    for row, v in cmds.items():
        assert g.apply_command(AgentCommand(row, CommandLevel.POS, v))
    g.step(1e-3)
    st, og = _twin_with(g, cmds)
    g.step(1e-3)
    og.step(f32(1e-3))
    err = rel_errors(gpu_state(g), og)
    assert all(v <= PER_STEP_TOL for v in err.values()), err


def test_nan_bulk_setpoint_faults_its_row():
    """set_setpoints (the bulk device feed, no reference counterpart) does not
    screen values: a NaN setpoint propagates (NaN-preserving clamps) and faults
    its row at the next step, with its id returned; the same value through
    apply_command raises InvalidStateError before any state changes, like the
    reference (quat.py:84 via the outer loop)."""
    import torch

    from paper_2308_12698_b200 import AgentCommand, CommandLevel, InvalidStateError
    g, pos = _group()
    sp = np.zeros((g.n, 7), dtype=np.float32)
    sp[:, :3] = pos
    sp[9, 0] = np.nan
    sp[11, 6] = np.nan
    g.set_setpoints(torch.from_numpy(sp).cuda())
    assert g.step(1e-3).tolist() == [9, 11]
    assert not g.batch.alive[[9, 11]].any() and g.batch.alive.sum() == g.n - 2
    g2, _ = _group()
    g2.apply_command(AgentCommand(9, CommandLevel.POS, (float("nan"), 0.0, 10.0, 0.0, 0.0, 0.0, 0.0)))
    before = g2.batch.pos.copy()
    with pytest.raises(InvalidStateError):
        g2.step(1e-3)
    np.testing.assert_array_equal(g2.batch.pos, before)


def test_device_setpoints_made_on_the_callers_stream():
    """Setpoints produced by device work on the caller's stream right before
    set_setpoints are read only after that work (the group's stream waits)."""
    import torch

    g, pos = _group(n=200_000 // 128 * 128)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        base = torch.from_numpy(np.asarray(pos, dtype=np.float32)).cuda()
        for _ in range(3):                         # enough device work to race with
            big = torch.randn(4096, 4096, device="cuda")
            big = big @ big
        sp = torch.zeros((g.n, 7), device="cuda")
        sp[:, :3] = base + 1.0
        sp[:, 6] = 0.25
        g.set_setpoints(sp)
    vals = g.cmd_values
    np.testing.assert_allclose(vals[:, :3], np.asarray(pos, dtype=np.float32) + 1.0, rtol=0, atol=1e-5)
    assert np.all(vals[:, 6] == np.float32(0.25))


def test_push_host_state_keeps_the_pid_derivative():
    """Editing the host mirror and pushing it must not reset the PID's
    has_prev (the reference never resets it on state edits): the next tick
    still applies the D term, as the oracle does with has_prev carried over."""
    from gpu_util import PER_STEP_TOL, f32, gpu_state, oracle_twin, rel_errors

    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    g, pos = _group()
    for i in range(g.n):
        g.apply_command(AgentCommand(i, CommandLevel.RATE, (0.2, -0.1, 0.05, 9.81)))
    g.step_k(1e-3, 5)
    assert g.pid_state_dict()["has_prev"].all()
    g.batch.pos[:, 0] += 1.0          # edit the mirror ...
    g.push_host_state()               # ... and push it
    st = gpu_state(g)
    assert st["has_prev"].all()
    og = oracle_twin(g, st)
    g.step(1e-3)
    og.step(f32(1e-3))
    err = rel_errors(gpu_state(g), og)
    assert all(v <= PER_STEP_TOL for v in err.values()), err
