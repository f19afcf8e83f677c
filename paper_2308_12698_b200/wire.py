"""Snapshot frames for the viewer / algorithm sides, packed on the device.

Mirrors the reference's framing (wire.py:118-124) and SnapshotMsg layout
(wire.py:162-178, PROTOCOL.md): ``u32 length | u8 type | payload`` with the
payload ``u64 tick`` followed by one section per agent type in ascending
type_id.  Sections of B200 groups come from ``B200QuadGroup.wire_section()``
(device packing + one device->host copy); ``empty_types`` adds header-only
sections for types with no agents.
"""

from __future__ import annotations

import struct

from .errors import ValidationError

MSG_SNAPSHOT = 0x01
MAX_FRAME_LEN = 64 * 1024 * 1024  # wire.py:50


def encode_frame(msg_type: int, payload: bytes) -> bytes:
    """``u32 length (= 1 + payload) | u8 msg_type | payload`` (wire.py:118-124)."""
    length = 1 + len(payload)
    if length > MAX_FRAME_LEN:
        raise ValidationError(f"frame of {length} bytes exceeds the {MAX_FRAME_LEN} cap")
    return struct.pack("<IB", length, msg_type) + payload


def snapshot_frame(tick: int, groups, empty_types=()) -> bytes:
    """A complete SnapshotMsg frame for ``groups`` (objects with ``type_id`` and
    ``wire_section()``) plus header-only sections for ``empty_types``."""
    sections = [(g.type_id, g.wire_section()) for g in groups]
    sections += [(int(t), struct.pack("<HI", int(t), 0)) for t in empty_types]
    sections.sort(key=lambda s: s[0])
    length = 1 + 8 + sum(len(s) for _, s in sections)
    if length > MAX_FRAME_LEN:
        raise ValidationError(f"frame of {length} bytes exceeds the {MAX_FRAME_LEN} cap")
    return b"".join([struct.pack("<IBQ", length, MSG_SNAPSHOT, int(tick))] + [s for _, s in sections])
