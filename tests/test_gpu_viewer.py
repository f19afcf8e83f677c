"""Viewer influence on the device (World._apply_viewer_input, core.py:445-453):
``B200QuadGroup.apply_viewer_input`` against the reference's own
``viewer_velocity_offsets`` outputs (tests/golden/viewer.npz, wire.py:320-340)
and against the host path it replaces (``add_velocity_overlay`` of host-computed
offsets, which needs a full position pull)."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from conftest import cuda_ok
from golden_io import load_viewer
from gpu_util import PER_STEP_TOL, f32, gpu_state, oracle_twin, rel_errors

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _group(pos, alive, quat, **kw):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    b = batch_create(0, pos.shape[0], pos, quat=quat)
    b.alive[:] = alive
    return B200QuadGroup(0, b, device="cuda:0", **kw)


def _msg(c):
    return SimpleNamespace(mode=c["mode"], world_point=tuple(c["point"]), radius=c["radius"], strength=c["strength"])


def _overlay(g):
    from paper_2308_12698_b200._lib import COL_OVERLAY
    return g.column_block(COL_OVERLAY, COL_OVERLAY + 3).cpu().numpy()


def test_viewer_offsets_match_reference_golden():
    pos, alive, quat, cases = load_viewer()
    for i, c in enumerate(cases):
        g = _group(pos, alive, quat)
        added = g.apply_viewer_input(_msg(c))
        if c["mode"] == "waypoint":
            assert added is False
            np.testing.assert_array_equal(g.cmd_level, c["cmd_level"])
            want = c["cmd_values"].astype(np.float32)
            got = g.cmd_values.astype(np.float32)
            np.testing.assert_array_equal(got[:, :6], want[:, :6])
            # yaw_sp = quat_yaw(q) of the float32-stored (batch_create-renormalised) quaternion
            np.testing.assert_allclose(got[:, 6], want[:, 6], rtol=0, atol=2e-6)
            continue
        assert added == c["any"], i
        assert g._overlay_active == c["any"], i
        if c["any"]:
            # bit-exact: float64 offsets in the reference's order, rounded once
            np.testing.assert_array_equal(_overlay(g), c["off"].astype(np.float32), err_msg=str(i))


def test_viewer_device_path_equals_host_overlay_path():
    """Two stacked messages through the device path step bit-identically to
    add_velocity_overlay of the reference offsets (the World's host path)."""
    pos, alive, quat, cases = load_viewer()
    a, b = _group(pos, alive, quat), _group(pos, alive, quat)
    for c in (cases[0], cases[1], cases[4]):
        a.apply_viewer_input(_msg(c))
        if c["any"]:
            b.add_velocity_overlay(c["off"])
    np.testing.assert_array_equal(_overlay(a), _overlay(b))
    for _ in range(3):
        a.step(1e-3)
        b.step(1e-3)
    assert torch.equal(a.cols, b.cols) and torch.equal(a.flags, b.flags)


def test_viewer_no_hit_leaves_overlay_inactive():
    """The offsets.any() gate: a message that reaches nobody must not activate
    the overlay (v_sp = cmd + 0 would turn -0.0 feed-forward into +0.0)."""
    pos, alive, quat, cases = load_viewer()
    a, b = _group(pos, alive, quat), _group(pos, alive, quat)
    assert not cases[6]["any"]
    assert a.apply_viewer_input(_msg(cases[6])) is False
    assert a.apply_viewer_input(_msg(cases[2])) is False      # radius 0
    a.step(1e-3)
    b.step(1e-3)
    assert torch.equal(a.cols, b.cols)


def test_viewer_step_parity_vs_oracle():
    pos, alive, quat, cases = load_viewer()
    g = _group(pos, alive, quat)
    g.step(1e-3)
    og = oracle_twin(g)
    c = cases[0]
    g.apply_viewer_input(_msg(c))
    st = gpu_state(g)
    from oracle import oracle as orc
    og.add_velocity_overlay(orc.viewer_offsets(c["mode"], c["point"], c["radius"], c["strength"],
                                               st["pos"], st["alive"]))
    g.step(1e-3)
    og.step(f32(1e-3))
    for k, v in rel_errors(gpu_state(g), og).items():
        assert v <= PER_STEP_TOL, f"{k}: {v:.2e}"


def test_viewer_on_unicycles_and_shards():
    from paper_2308_12698_b200 import B200UnicycleGroup, MultiDeviceQuadGroup, batch_create
    pos, alive, quat, cases = load_viewer()
    b = batch_create(1, pos.shape[0], pos, quat=quat)
    b.alive[:] = alive
    u = B200UnicycleGroup(1, b, device="cuda:0")
    assert u.apply_viewer_input(_msg(cases[1])) is True
    np.testing.assert_array_equal(_overlay(u), cases[1]["off"].astype(np.float32))
    m = MultiDeviceQuadGroup(0, b, devices=["cuda:0", "cuda:0"])
    assert m.apply_viewer_input(_msg(cases[0])) is True
    got = np.concatenate([_overlay(s) for s in m.shards])
    np.testing.assert_array_equal(got, cases[0]["off"].astype(np.float32))
