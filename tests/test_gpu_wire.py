"""Device snapshot packing (f2) against the reference's wire format: the golden
snapshot frame documented in PROTOCOL.md ("Golden snapshot fixture") and a
restatement of encode_snapshot (wire.py:162-178) on random groups."""

import struct

import numpy as np
import pytest

from conftest import cuda_ok
from gpu_util import make_group
from scenarios import ALL, Scenario, run_script

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

# PROTOCOL.md, golden snapshot fixture (tests/golden/snapshot_golden.bin of the reference)
GOLDEN_HEX = ("52000000 01 0700000000000000 0000 01000000 2a00000000000000 01 "
              "0000c03f 000000c0 00005040 0000003f 0000803e 000080bf "
              "0000803f 00000000 00000000 00000000 0000803d 000000be 0000803e 0100 00000000")


def encode_section_reference(b) -> bytes:
    """wire.py:162-178 restated with numpy for one batch (float64 mirror)."""
    q = b.quat
    sign = np.where(q[:, :1] < 0.0, -1.0, 1.0)
    qc = q * sign + 0.0                                   # quat.py:52-59
    return (struct.pack("<HI", b.type_id, b.n) + b.agent_ids.astype("<u8").tobytes()
            + b.alive.astype("<u1").tobytes() + b.pos.astype("<f4").tobytes()
            + b.vel.astype("<f4").tobytes() + qc.astype("<f4").tobytes() + b.omega.astype("<f4").tobytes())


def test_golden_snapshot_frame():
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    from paper_2308_12698_b200.wire import snapshot_frame
    b = batch_create(0, 1, [[1.5, -2.0, 3.25]], quat=[[-1.0, 0, 0, 0]], vel=[[0.5, 0.25, -1.0]],
                     omega=[[0.0625, -0.125, 0.25]], agent_ids=[42])
    g = B200QuadGroup(0, b)
    frame = snapshot_frame(7, [g], empty_types=[1])
    assert frame == bytes.fromhex(GOLDEN_HEX.replace(" ", ""))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 128, 1001])
def test_device_section_equals_encode_snapshot(n):
    rng = np.random.default_rng(n)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = Scenario("w", n, 1e-3, 20, rng.uniform(-100, 100, (n, 3)), rng.uniform(-1, 1, (n, 3)), q,
                  rng.uniform(-1, 1, (n, 3)), record=[])
    g = make_group(sc)
    g.mark_dead([n // 2])
    run_script(g, sc)                               # some ticks: hi + lo positions, canonicalisation
    assert g.wire_section() == encode_section_reference(g.batch)


def test_mixed_scenario_frame():
    from paper_2308_12698_b200.wire import snapshot_frame
    sc = ALL["mixed"]()
    g = make_group(sc)
    run_script(g, sc)
    frame = snapshot_frame(200, [g])
    payload = struct.pack("<Q", 200) + encode_section_reference(g.batch)
    assert frame == struct.pack("<IB", 1 + len(payload), 1) + payload
