"""Snapshot publishing for B200 groups: device packing, pinned copies that
overlap the next ticks, and delivery off the simulation thread.

The reference publishes once per tick (``World._publish``, core.py:477-485):
it deep-copies every group to float64 (``snapshot``), and the broadcaster
thread (server.py:364-369) and ``SnapshotRecorder`` (server.py:292-324) encode
the frames (wire.py:162-178) on the host.  For a B200 group that costs a full
float64 device->host pull per tick plus a host encode.  ``FramePublisher`` does
instead, per published tick:

  1. the wire columns of each group are packed on the device, on the group's
     stream right after its queued ticks (``B200QuadGroup.pack_wire_async``);
  2. a side stream copies the packed bytes into a pinned host slot, so the copy
     overlaps the ticks the loop launches next;
  3. a worker thread waits for the copy, assembles the complete SnapshotMsg
     frame and hands it to the subscribers (callables taking the frame bytes:
     the ``Endpoints`` fan-out, a ``FrameRecorder``, a socket ...).

Frames are the bytes ``wire.snapshot_frame`` returns for the same state.  At
most ``slots`` frames are in flight.  Lossless by default (every frame
delivered, the recorder's semantics: ``publish`` waits for a free slot); with
``drop_when_busy`` it never waits -- a tick with no free slot is dropped, and
a frame with a newer one queued behind it is skipped (the broadcaster
mailbox's latest-wins, server.py:263-289); both count in ``dropped``.
"""

from __future__ import annotations

import contextlib
import queue
import struct
import threading
from collections.abc import Callable, Iterable

import numpy as np
import torch

from . import _lib
from .errors import ValidationError
from .wire import MAX_FRAME_LEN, MSG_SNAPSHOT

# per-agent bytes of the section's column blocks, in wire order (wire.py:166-178):
# ids u64, alive u8, pos 3 f32, vel 3 f32, quat 4 f32, omega 3 f32
_BLOCKS = (8, 1, 12, 12, 16, 12)
_ROW_BYTES = sum(_BLOCKS)   # 61


def _parts_of(group):
    """(type_id, [B200 groups whose sections concatenate into this type's section])."""
    shards = getattr(group, "shards", None)
    return int(group.type_id), (list(shards) if shards is not None else [group])


def frame_layout(types, empty_types=()):
    """Byte layout of a SnapshotMsg frame (wire.py:118-124, 162-178) for the
    given ``[(type_id, [parts])]``: (frame length, header bytes to place at
    their offsets, per part the list of (device byte offset, frame offset,
    bytes) copies that put its packed columns into place)."""
    secs = [(t, parts) for t, parts in types] + [(int(t), []) for t in empty_types]
    secs.sort(key=lambda s: s[0])
    off = 5 + 8                                   # u32 length | u8 type | u64 tick
    headers, copies = [], {}
    for t, parts in secs:
        ns = [g.n for g in parts]
        n = sum(ns)
        headers.append((off, struct.pack("<HI", t, n)))
        off += 6
        if len(parts) == 1:
            copies[id(parts[0])] = [(0, off, _ROW_BYTES * n)]
        for k, g in enumerate(parts if len(parts) > 1 else []):
            # shards: block w of part k follows the previous parts' rows of that block
            cps, src, base = [], 0, off
            for w in _BLOCKS:
                cps.append((src, base + sum(ns[:k]) * w, w * ns[k]))
                src += w * ns[k]
                base += w * n
            copies[id(g)] = cps
        off += _ROW_BYTES * n
    return off, headers, copies


def _on_device(device):
    return contextlib.nullcontext() if torch.cuda.current_device() == device.index else torch.cuda.device(device)


class _Slot:
    def __init__(self, parts, length, headers):
        self.frame = torch.empty(length, dtype=torch.uint8, pin_memory=True)
        self.view = self.frame.numpy()
        hdr = struct.pack("<IB", length - 4, MSG_SNAPSHOT)
        self.view[:5] = np.frombuffer(hdr, dtype=np.uint8)
        for off, b in headers:
            self.view[off:off + len(b)] = np.frombuffer(b, dtype=np.uint8)
        self.dev = [torch.empty(_ROW_BYTES * g.n + 8, dtype=torch.uint8, device=g.device) for g in parts]
        self.packed = [torch.cuda.Event() for _ in parts]
        self.done = [torch.cuda.Event() for _ in parts]


class FramePublisher:
    """Per-tick SnapshotMsg frames of B200 groups, delivered to subscribers on
    a worker thread (see the module docstring)."""

    def __init__(self, groups, subscribers: Iterable[Callable[[bytes], None]] = (), *, slots: int = 2,
                 drop_when_busy: bool = False, empty_types=()):
        if slots < 1:
            raise ValidationError("need at least one slot")
        types = sorted((_parts_of(g) for g in groups), key=lambda t: t[0])
        self._flat = [g for _, parts in types for g in parts]
        length, headers, copies = frame_layout(types, empty_types)
        if length - 4 > MAX_FRAME_LEN:
            raise ValidationError(f"frame of {length - 4} bytes exceeds the {MAX_FRAME_LEN} cap")
        self._copies = [copies[id(g)] for g in self._flat]
        self._subs = list(subscribers)
        self._drop = bool(drop_when_busy)
        self._lib = _lib.load()
        self._copy_streams = {}
        for g in self._flat:
            if g.device not in self._copy_streams:
                self._copy_streams[g.device] = torch.cuda.Stream(g.device)
        self._slots = [_Slot(self._flat, length, headers) for _ in range(slots)]
        self._free: queue.Queue[int] = queue.Queue()
        for i in range(slots):
            self._free.put(i)
        self._work: queue.Queue = queue.Queue()
        self.published = 0
        self.dropped = 0
        self.delivered = 0
        self.error: BaseException | None = None
        self._thread = threading.Thread(target=self._loop, daemon=True, name="b200-publisher")
        self._thread.start()

    def subscribe(self, fn: Callable[[bytes], None]) -> None:
        self._subs.append(fn)

    def publish(self, tick: int) -> bool:
        """Queue the frame of the groups' state after their queued ticks; False
        if it was dropped (``drop_when_busy`` and every slot in flight)."""
        if self.error is not None:
            raise RuntimeError("publisher worker failed") from self.error
        try:
            i = self._free.get_nowait() if self._drop else self._free.get()
        except queue.Empty:
            self.dropped += 1
            return False
        slot = self._slots[i]
        slot.view[5:13] = np.frombuffer(struct.pack("<Q", int(tick)), dtype=np.uint8)
        host = slot.frame.data_ptr()
        for j, g in enumerate(self._flat):
            g.pack_wire_async(slot.dev[j])
            cs = self._copy_streams[g.device]
            slot.packed[j].record(g.stream)
            cs.wait_event(slot.packed[j])
            dev = slot.dev[j].data_ptr()
            with _on_device(g.device):
                for src, dst, nb in self._copies[j]:
                    _lib.check(self._lib.swarmstep_memcpy_async(host + dst, dev + src, nb, cs.cuda_stream))
            slot.done[j].record(cs)
        self.published += 1
        self._work.put((int(tick), i))
        return True

    def _loop(self) -> None:
        while True:
            item = self._work.get()
            if item is None:
                self._work.task_done()
                return
            _, i = item
            slot = self._slots[i]
            try:
                for ev in slot.done:
                    ev.synchronize()
                if self._drop and self._work.qsize() > 0:
                    # a newer frame is already queued: latest wins (server.py:272-277)
                    self.dropped += 1
                    frame = None
                else:
                    frame = slot.view.tobytes()
            except BaseException as e:   # surfaced by the next publish / flush
                self.error = e
                frame = None
            self._free.put(i)
            if frame is None:
                self._work.task_done()
                continue
            try:
                for fn in self._subs:
                    fn(frame)
                self.delivered += 1
            except BaseException as e:
                self.error = e
            self._work.task_done()

    def flush(self) -> None:
        """Wait until every published frame has been delivered."""
        self._work.join()
        if self.error is not None:
            raise RuntimeError("publisher worker failed") from self.error

    def close(self) -> None:
        self._work.put(None)
        self._thread.join(timeout=30.0)


class FrameRecorder:
    """Writes every frame it is given to ``path`` in order: the file
    ``SnapshotRecorder`` (server.py:292-324) writes for the same snapshots.
    Use as a ``FramePublisher`` subscriber (it runs on the publisher's worker
    thread, so frames arrive in publish order)."""

    def __init__(self, path: str):
        self._file = open(path, "wb")
        self.frames = 0

    def __call__(self, frame: bytes) -> None:
        self._file.write(frame)
        self.frames += 1

    publish = __call__

    def close(self) -> None:
        self._file.close()
