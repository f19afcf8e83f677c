"""FramePublisher / FrameRecorder (snapshot frames for the
broadcaster and recorder, server.py:292-375): every delivered frame equals the
synchronous ``wire.snapshot_frame`` of the same tick (which test_gpu_wire pins
to the reference's encode_snapshot), for one group, several types with empty
sections, index shards, and the lossy latest-wins mode."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _quads(n, seed, type_id=0, id_base=0):
    from paper_2308_12698_b200 import batch_create
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    b = batch_create(type_id, n, rng.uniform(-50, 50, (n, 3)), quat=q, vel=rng.uniform(-1, 1, (n, 3)),
                     omega=rng.uniform(-1, 1, (n, 3)), id_base=id_base)
    b.alive[::7] = False
    return b


def _twins(n, seed):
    from paper_2308_12698_b200 import B200QuadGroup
    return B200QuadGroup(0, _quads(n, seed)), B200QuadGroup(0, _quads(n, seed))


def _tick_of(frame):
    return int.from_bytes(frame[5:13], "little")


def test_recorder_file_equals_synchronous_frames(tmp_path):
    from paper_2308_12698_b200.publish import FramePublisher, FrameRecorder
    from paper_2308_12698_b200.wire import snapshot_frame
    a, b = _twins(1001, 3)
    rec = FrameRecorder(str(tmp_path / "rec.bin"))
    pub = FramePublisher([a], [rec], slots=2)
    want = []
    for t in range(40):
        a.step(1e-3)
        pub.publish(t)
        b.step(1e-3)
        want.append(snapshot_frame(t, [b]))
    pub.flush()
    pub.close()
    rec.close()
    assert pub.delivered == 40 and pub.dropped == 0 and rec.frames == 40
    assert (tmp_path / "rec.bin").read_bytes() == b"".join(want)


def test_async_ticks_between_publishes():
    """Publishing after step_async (no host sync) captures the state after the
    queued ticks; copies overlap the following launches."""
    from paper_2308_12698_b200.publish import FramePublisher
    from paper_2308_12698_b200.wire import snapshot_frame
    a, b = _twins(20000, 5)
    got = []
    pub = FramePublisher([a], [got.append], slots=3)
    want = []
    for t in range(12):
        a.step_async(1e-3, 3)
        pub.publish(t)
        b.step_k(1e-3, 3)
        want.append(snapshot_frame(t, [b]))
    a.collect_faults()
    pub.flush()
    pub.close()
    assert got == want


def test_multi_type_frames_with_empty_sections():
    from paper_2308_12698_b200 import B200QuadGroup, B200UnicycleGroup
    from paper_2308_12698_b200.publish import FramePublisher
    from paper_2308_12698_b200.wire import snapshot_frame
    q = B200QuadGroup(3, _quads(300, 1, type_id=3))
    u = B200UnicycleGroup(1, _quads(77, 2, type_id=1, id_base=1000))
    got = []
    pub = FramePublisher([q, u], [got.append], empty_types=[2])
    want = []
    for t in range(5):
        q.step(1e-3)
        u.step(1e-3)
        pub.publish(t)
        pub.flush()
        want.append(snapshot_frame(t, [q, u], empty_types=[2]))
    pub.close()
    assert got == want


def test_shards_publish_one_section():
    from paper_2308_12698_b200 import B200QuadGroup, MultiDeviceQuadGroup
    from paper_2308_12698_b200.publish import FramePublisher
    from paper_2308_12698_b200.wire import snapshot_frame
    m = MultiDeviceQuadGroup(0, _quads(999, 4), devices=["cuda:0", "cuda:0", "cuda:0"])
    one = B200QuadGroup(0, _quads(999, 4))
    got = []
    pub = FramePublisher([m], [got.append])
    for t in range(3):
        m.step(1e-3)
        one.step(1e-3)
        pub.publish(t)
    pub.flush()
    pub.close()
    assert got[-1] == snapshot_frame(2, [one])
    assert [_tick_of(f) for f in got] == [0, 1, 2]


def test_latest_wins_mode_delivers_valid_ordered_frames():
    from paper_2308_12698_b200.publish import FramePublisher
    from paper_2308_12698_b200.wire import snapshot_frame
    a, b = _twins(200000, 6)
    got = []
    pub = FramePublisher([a], [got.append], slots=1, drop_when_busy=True)
    want = {}
    ok = 0
    for t in range(30):
        a.step_async(1e-3, 1)
        ok += pub.publish(t)
        b.step(1e-3)
        want[t] = snapshot_frame(t, [b])
    a.collect_faults()
    pub.flush()
    pub.close()
    assert pub.published == ok and pub.delivered + pub.dropped == 30
    assert got and all(f == want[_tick_of(f)] for f in got)
    assert [_tick_of(f) for f in got] == sorted(_tick_of(f) for f in got)


def test_shard_wire_section_equals_single_group():
    from paper_2308_12698_b200 import B200QuadGroup, MultiDeviceQuadGroup
    from paper_2308_12698_b200.wire import snapshot_frame
    m = MultiDeviceQuadGroup(0, _quads(500, 8), devices=["cuda:0", "cuda:0"])
    one = B200QuadGroup(0, _quads(500, 8))
    m.step(1e-3)
    one.step(1e-3)
    assert snapshot_frame(1, [m]) == snapshot_frame(1, [one])


def test_subscriber_error_surfaces_and_slots_recover():
    from paper_2308_12698_b200.publish import FramePublisher
    a, _ = _twins(300, 9)
    calls = []

    def bad(frame):
        calls.append(len(frame))
        raise OSError("socket closed")
    pub = FramePublisher([a], [bad], slots=1)
    a.step(1e-3)
    pub.publish(0)
    with pytest.raises(RuntimeError):
        pub.flush()
    with pytest.raises(RuntimeError):
        pub.publish(1)
    pub.close()
    assert calls == [13 + 6 + 61 * 300]
