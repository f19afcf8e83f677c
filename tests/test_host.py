"""CPU tests of the host-side pieces that need no GPU: parameter packing,
command levels, layouts, wire framing, collision helpers, scenario fixtures,
and property checks with hypothesis."""

import struct

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2308_12698_b200 import (AgentCommand, CommandLevel, OuterGains, PidGains, QuadParams,
                                   ValidationError, batch_create, quat_yaw, yaw_quat)
from paper_2308_12698_b200.collision import CollisionConfig, half_space_offsets
from paper_2308_12698_b200.commands import LEVEL_MOTOR, LEVEL_POS, LEVEL_RATE, level_code
from paper_2308_12698_b200.layout import layout_poses
from paper_2308_12698_b200.params import allocation_matrices, pack_device_params
from paper_2308_12698_b200.parallel import shard_range
from paper_2308_12698_b200.wire import encode_frame, snapshot_frame


def test_params_validation_mirrors_reference():
    # quad.py:56-60, test_quad.py:67-69
    with pytest.raises(ValidationError):
        QuadParams(m=0.0)
    with pytest.raises(ValidationError):
        QuadParams(arm_angle=1e-300)
    with pytest.raises(ValidationError):
        PidGains(kp=-1.0, ki=0.0, kd=0.0, i_limit=1.0)
    assert QuadParams().f_motor_max == pytest.approx(16.0)
    assert QuadParams().hover_thrust == pytest.approx(9.81)


@settings(max_examples=40, deadline=None)
@given(st.floats(0.05, 1.0), st.floats(0.2, 1.3), st.floats(1e-9, 1e-7), st.floats(1e-11, 1e-9))
def test_allocation_inverse_structure(arm, angle, k_t, k_q):
    """G^-1 = sign(G^T) * c holds for every X-geometry the kernel's mixer accepts."""
    p = QuadParams(arm_length=arm, arm_angle=angle, k_t=k_t, k_q=k_q)
    g, gi = allocation_matrices(p)
    np.testing.assert_allclose(gi @ g, np.eye(4), atol=1e-9)
    np.testing.assert_allclose(gi, np.sign(g.T) * np.abs(gi[0]), rtol=1e-9)
    pack_device_params(p, PidGains(kp=0.1, ki=0.1, kd=0.1, i_limit=0.1), OuterGains(kp_pos=1, kv=1, k_att=1))


def test_level_codes():
    assert level_code(CommandLevel.POS) == LEVEL_POS and level_code("rate") == LEVEL_RATE
    assert level_code(CommandLevel.MOTOR) == LEVEL_MOTOR
    assert level_code(CommandLevel.UNICYCLE) is None and level_code(7) is None
    with pytest.raises(ValidationError):
        AgentCommand(1, CommandLevel.POS, (1.0, 2.0))


def test_layouts_match_reference_shapes():
    pos, yaw = layout_poses({"kind": "grid", "spacing": 3.0, "origin": (0, 0, 10)}, 10)
    assert pos.shape == (10, 3) and pos[5].tolist() == [3.0, 3.0, 10.0] and np.all(yaw == 0)
    pos, yaw = layout_poses({"kind": "circle", "radius": 5.0, "z": 2.0}, 4)
    np.testing.assert_allclose(pos[1], [0.0, 5.0, 2.0], atol=1e-12)
    np.testing.assert_allclose(yaw[0], np.pi / 2)
    with pytest.raises(ValidationError):
        layout_poses({"kind": "spiral"}, 3)


@settings(max_examples=50, deadline=None)
@given(st.floats(-3.1, 3.1))
def test_yaw_quat_roundtrip(theta):
    assert quat_yaw(yaw_quat(theta)) == pytest.approx(theta, abs=1e-12)


def test_batch_create_mirrors_reference():
    b = batch_create(0, 3, np.zeros((3, 3)), id_base=100)
    assert b.agent_ids.tolist() == [100, 101, 102] and b.alive.all()
    with pytest.raises(ValidationError):
        batch_create(0, 1, [[0, 0, 0]], quat=[[1.0, 1.0, 0, 0]])
    with pytest.raises(ValidationError):
        batch_create(0, 2, np.zeros((2, 3)), agent_ids=[7, 7])


def test_encode_frame_and_snapshot_frame_layout():
    # PROTOCOL.md framing example: {"op":"stop"} -> 0E 00 00 00 05 + payload
    payload = b'{"op":"stop"}'
    assert encode_frame(5, payload) == bytes.fromhex("0e00000005") + payload

    class G:
        def __init__(self, t, n):
            self.type_id, self.n = t, n

        def wire_section(self):
            return struct.pack("<HI", self.type_id, self.n) + b"x" * (61 * self.n)

    frame = snapshot_frame(9, [G(2, 1), G(0, 2)], empty_types=[1])
    assert frame[4] == 1 and struct.unpack_from("<Q", frame, 5)[0] == 9
    types = []
    off = 13
    while off < len(frame):
        t, n = struct.unpack_from("<HI", frame, off)
        types.append(t)
        off += 6 + 61 * n
    assert types == [0, 1, 2] and off == len(frame)


def test_collision_config_and_offsets_mirror_reference():
    with pytest.raises(ValidationError):
        CollisionConfig(r_collide={0: 0.5}, r_sense=0.4, cell=1.0)    # r_collide > r_sense
    with pytest.raises(ValidationError):
        CollisionConfig(r_collide={0: 0.5}, r_sense=1.0, cell=0.9)    # cell < 2 r
    offs = half_space_offsets(1, 1.0, 1.0)
    assert len(offs) == 13                       # half of the 26 neighbours
    keys = {tuple(o) for o in offs}
    assert all((-a, -b, -c) not in keys for a, b, c in keys)
    offs2 = half_space_offsets(2, 2.0, 1.0)
    assert all(np.sum((np.maximum(np.abs(o) - 1, 0)) ** 2) < 4.0 for o in offs2)


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 10**8), st.integers(1, 64))
def test_shards_partition(n, world):
    rs = [shard_range(n, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= 1


@settings(max_examples=25, deadline=None)
@given(st.integers(1, 40), st.integers(0, 2**31))
def test_oracle_rows_are_independent(n, seed):
    """The float64 oracle's rows do not interact: stepping a subset equals the
    same rows of the full batch (the property the GPU parity tests rely on)."""
    from oracle import oracle as orc
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)

    class B:
        agent_ids = np.arange(n, dtype=np.uint64)
        pos, vel, quat = rng.uniform(-5, 5, (n, 3)), rng.uniform(-1, 1, (n, 3)), q
        omega, alive = rng.uniform(-1, 1, (n, 3)), np.ones(n, bool)

    full = orc.OracleGroup(0, B)
    rows = np.sort(rng.choice(n, max(1, n // 2), replace=False))

    class S:
        agent_ids = B.agent_ids[rows]
        pos, vel, quat, omega, alive = B.pos[rows], B.vel[rows], B.quat[rows], B.omega[rows], B.alive[rows]

    sub = orc.OracleGroup(0, S)
    for _ in range(5):
        full.step(1e-3)
        sub.step(1e-3)
    np.testing.assert_array_equal(full.state13()[rows], sub.state13())


def test_neighbor_sets_from_pair_list():
    """NeighborSets (the report's lazy neighbor_sets) equals the reference's
    dict construction (collision.py:166-175): alive ids in batch order, each
    with its sorted neighbour ids; dead agents absent."""
    from paper_2308_12698_b200.collision import NeighborSets
    rng = np.random.default_rng(0)
    m = 500
    ids = rng.permutation(10_000)[:m].astype(np.int64)
    alive = rng.random(m) > 0.2
    pairs = set()
    while len(pairs) < 2000:
        a, b = rng.integers(0, m, 2)
        if a != b and alive[a] and alive[b]:
            pairs.add((min(a, b), max(a, b)))
    near = np.array(sorted(pairs))
    want = {int(i): [] for i in ids[alive]}
    for a, b in near:
        want[int(ids[a])].append(int(ids[b]))
        want[int(ids[b])].append(int(ids[a]))
    want = {k: tuple(sorted(v)) for k, v in want.items()}
    ns = NeighborSets(alive, ids, near)
    assert len(ns) == len(want)
    assert dict(ns) == want and list(ns) == list(want)
    assert dict(NeighborSets(alive, ids, np.empty((0, 2), np.int64))) == {k: () for k in want}


def test_frame_layout_places_every_shard_block():
    """publish.frame_layout: copying each part's packed columns to the offsets
    it gives reproduces the SnapshotMsg frame built from whole sections
    (wire.py:162-178), for random types, shard splits and empty types."""
    import struct

    from paper_2308_12698_b200.publish import _BLOCKS, frame_layout
    from paper_2308_12698_b200.wire import MSG_SNAPSHOT, encode_frame
    rng = np.random.default_rng(3)

    class Part:
        def __init__(self, n):
            self.n = n

    for _ in range(50):
        types = []
        for t in sorted(rng.choice(20, size=int(rng.integers(1, 4)), replace=False)):
            parts = [Part(int(rng.integers(1, 9))) for _ in range(int(rng.integers(1, 4)))]
            types.append((int(t), parts))
        used = {t for t, _ in types}
        empty = [int(t) for t in rng.choice(20, size=2, replace=False) if int(t) not in used]
        length, headers, copies = frame_layout(types, empty)
        frame = np.zeros(length, dtype=np.uint8)
        hdr = struct.pack("<IBQ", length - 4, MSG_SNAPSHOT, 7)
        frame[:13] = np.frombuffer(hdr, dtype=np.uint8)
        for off, b in headers:
            frame[off:off + len(b)] = np.frombuffer(b, dtype=np.uint8)
        sections = []
        for t, parts in types:
            # per part: its own packed columns (block w of the part is w * n bytes)
            packed = [rng.integers(0, 256, 61 * p.n, dtype=np.uint8) for p in parts]
            for p, buf in zip(parts, packed):
                for src, dst, nb in copies[id(p)]:
                    frame[dst:dst + nb] = buf[src:src + nb]
            # the whole-type section: each column block concatenated across parts
            body, offs = [], [0] * len(parts)
            for w in _BLOCKS:
                for k, (p, buf) in enumerate(zip(parts, packed)):
                    body.append(buf[offs[k]:offs[k] + w * p.n].tobytes())
                    offs[k] += w * p.n
            sections.append((t, struct.pack("<HI", t, sum(p.n for p in parts)) + b"".join(body)))
        sections += [(t, struct.pack("<HI", t, 0)) for t in empty]
        sections.sort(key=lambda s: s[0])
        want = encode_frame(MSG_SNAPSHOT, struct.pack("<Q", 7) + b"".join(s for _, s in sections))
        assert frame.tobytes() == want


def test_f32_commands_reduce_yaw_and_saturate():
    """Host float64 -> float32 command conversion (group.f32_commands)."""
    import math

    from paper_2308_12698_b200.group import f32_commands
    v = np.array([[1.0, 2.0, 3.0, 0.0, 0.0, 0.0, 0.3],            # in range: bit-exact cast
                  [1e39, -2e39, 5.0, 0.0, 0.0, 0.0, 1000.3],       # saturate, reduce yaw
                  [float("nan"), float("inf"), 0.0, 0.0, 0.0, 0.0, -7.0],
                  [0.1, 0.2, 0.3, 9.81, 0.0, 0.0, 0.0],            # a RATE row: no yaw column
                  [1e40, -3.0, 0.0, 0.0, 0.0, 0.0, 0.0]])          # RATE beyond float32: saturates
    out = f32_commands(v, np.array([True, True, True, False, False]))
    assert out.dtype == np.float32
    np.testing.assert_array_equal(out[0], v[0].astype(np.float32))
    fmax = np.finfo(np.float32).max
    # POS position / velocity setpoints scaled together to |.| <= 1e15 (direction kept)
    np.testing.assert_allclose(out[1, :3], np.float32([5e14, -1e15, 2.5e-24]), rtol=1e-7)
    assert np.all(out[1, 3:6] == 0.0)
    assert abs(out[1, 6]) <= math.pi and abs(math.cos(out[1, 6]) - math.cos(1000.3)) < 2e-7
    assert out[4, 0] == fmax and out[4, 1] == -3.0
    assert math.isnan(out[2, 0]) and out[2, 1] == np.inf               # non-finite values pass unchanged
    assert abs(out[2, 6] - (-7.0 + 2 * math.pi)) < 1e-6
    np.testing.assert_array_equal(out[3], v[3].astype(np.float32))


def test_synthetic_swarm_slices_are_shard_independent():
    """Any shard of the bench swarm builds exactly its own rows of one fixed
    workload (bench.py ranks, the reference arm's host processes)."""
    from paper_2308_12698_b200.synthetic import BLOCK, swarm
    n = 3 * BLOCK + 123
    pos, sp = swarm(n)
    want_pos, _ = layout_poses({"kind": "grid", "spacing": 3.0, "origin": (0.0, 0.0, 10.0)}, n)
    np.testing.assert_array_equal(pos, want_pos)
    for w in (2, 3, 7):
        parts = [swarm(n, *shard_range(n, r, w)) for r in range(w)]
        np.testing.assert_array_equal(np.concatenate([p for p, _ in parts]), pos)
        np.testing.assert_array_equal(np.concatenate([s for _, s in parts], axis=1), sp)
    off = sp[:3].T.astype(np.float64) - pos
    assert np.all(np.abs(off) <= 1.0 + 1e-5) and np.all(sp[3:6] == 0.0) and np.all(np.abs(sp[6]) <= np.pi)


def test_pos_lo_decode_layout():
    """The packed compensated-position word (include/swarmstep_b200.h COL_POS_LO):
    10 signed bits per axis in units of ulp(hi) / 512, unit floored at 2^-126."""
    import numpy as np

    from paper_2308_12698_b200._lib import pos_lo_decode

    hi = np.array([[1.0, 100.0, 1e-3], [0.0, -3.5, 2.0 ** -120]], dtype=np.float32)
    q = np.array([[5, -256, 511], [0, 256, -511]])
    words = np.zeros(2, dtype=np.uint32)
    for i in range(3):
        words |= ((q[:, i] & 0x3FF).astype(np.uint32) << np.uint32(10 * i))
    lo = pos_lo_decode(words, hi)
    ulp = np.spacing(np.abs(hi).astype(np.float32)).astype(np.float64)
    unit = np.maximum(ulp / 512.0, 2.0 ** -126)
    unit[1, 0] = 2.0 ** -126          # hi = 0: the floored unit
    assert np.array_equal(lo, q * unit)
    # |lo| <= ulp(hi) / 2 fits the 10-bit field with room to spare
    assert np.all(np.abs(q) <= 511)


def test_overlap_epoch_policy():
    """Which step launches join the overlapped chain (group._overlap_epochs):
    4..4096 ticks, no rotor lag, not forced onto the TMA / direct kernels; the
    epoch chain skips 0 when it wraps (0 means "no wait")."""
    from types import SimpleNamespace

    from paper_2308_12698_b200._lib import STEP_FORCE_DIRECT, STEP_FORCE_PAIR, STEP_FORCE_TMA, STEP_OVERLAY
    from paper_2308_12698_b200.group import B200QuadGroup
    g = SimpleNamespace(overlap_launches=True, _motor=None, _pdl_epoch=0)
    ep = B200QuadGroup._overlap_epochs

    def val(e):
        return None if e is None else (e[0].value, e[1].value)

    assert val(ep(g, 10, 0)) == (0, 1)
    assert val(ep(g, 4, STEP_OVERLAY | STEP_FORCE_PAIR)) == (0, 1)
    assert val(ep(g, 4096, 0)) == (0, 1)
    for k in (1, 2, 3, 4097):
        assert ep(g, k, 0) is None, k
    assert ep(g, 10, STEP_FORCE_TMA) is None and ep(g, 10, STEP_FORCE_DIRECT) is None
    g._pdl_epoch = 0xFFFFFFFF
    assert val(ep(g, 10, 0)) == (0xFFFFFFFF, 1)
    g._pdl_epoch = 41
    assert val(ep(g, 10, 0)) == (41, 42)
    g._motor = object()
    assert ep(g, 10, 0) is None
    g._motor, g.overlap_launches = None, False
    assert ep(g, 10, 0) is None
