"""One homogeneous group spread over several GPUs of ONE process.

The reference's ``World`` is single-process (core.py:308-505) and keys its
bookkeeping by ``type_id`` (alive counts core.py:370, the id map core.py:314-
318), so one agent type cannot simply become eight groups.  ``MultiDeviceQuadGroup``
is one protocol-level group whose rows are sharded by contiguous index over
``devices`` ("contiguous agent-index ranges across 2/4/8
devices, one stream per device, from a single host thread"): ``step`` launches
every shard's fused kernel before waiting on any, so the devices run
concurrently; agents are independent (quad.py:6-7), so stepping needs no
exchange.

The neighbour-coupled controller of config 5 does need every shard's
positions each tick: ``MultiDeviceNeighborSeparation`` is its single-process
form -- each shard's pack kernel stores its rows straight into every shard's
gathered buffer (NVLink peer stores between devices, csrc/exchange.cu
``swarmstep_pack_scatter``), CUDA events order every reader after every
writer, and each shard then computes its overlay against the whole swarm on
its own device (csrc/neighbors.cu), exactly as ``parallel.NeighborSeparation``
does per rank.

(``bench.py`` and ``parallel.ShardedSwarm`` cover the one-process-per-GPU
layout; this class is the drop-in for an unchanged single-process World.)
"""

from __future__ import annotations

import ctypes
from collections.abc import Iterable

import numpy as np
import torch

from . import _lib
from .errors import ValidationError
from .group import B200QuadGroup
from .parallel import shard_range
from .state import AgentBatch, batch_snapshot


class _ShardBatchView:
    """``group.batch`` over the shards: ids / alive / n without a device read,
    state columns concatenated from the shards' float64 mirrors."""

    def __init__(self, mg):
        self._mg = mg

    @property
    def type_id(self) -> int:
        return self._mg.type_id

    @property
    def n(self) -> int:
        return self._mg.n

    @property
    def agent_ids(self) -> np.ndarray:
        return self._mg._ids

    def _cat(self, name):
        return np.concatenate([getattr(s.batch, name) for s in self._mg.shards])

    @property
    def alive(self) -> np.ndarray:
        return self._cat("alive")

    @property
    def pos(self) -> np.ndarray:
        return self._cat("pos")

    @property
    def vel(self) -> np.ndarray:
        return self._cat("vel")

    @property
    def quat(self) -> np.ndarray:
        return self._cat("quat")

    @property
    def omega(self) -> np.ndarray:
        return self._cat("omega")

    def index_of(self, agent_id: int):
        return self._mg.rows_for(agent_id)


class MultiDeviceQuadGroup:
    """A quadrotor group sharded over ``devices`` (same process, one stream each)."""

    kind = "quadrotor"

    def __init__(self, type_id: int, batch, params=None, rate_gains=None, outer_gains=None, *, devices,
                 **group_kw):
        devices = list(devices)
        if not devices:
            raise ValidationError("need at least one device")
        n = int(np.asarray(batch.agent_ids).shape[0])
        if n < len(devices):
            raise ValidationError("fewer agents than devices")
        self.type_id = int(type_id)
        self.n = n
        self._ids = np.array(batch.agent_ids, dtype=np.uint64)
        self.shards: list[B200QuadGroup] = []
        self._lo: list[int] = []
        for i, dev in enumerate(devices):
            lo, hi = shard_range(n, i, len(devices))
            sub = AgentBatch(type_id=int(getattr(batch, "type_id", type_id)), agent_ids=self._ids[lo:hi],
                             pos=np.asarray(batch.pos, float)[lo:hi], vel=np.asarray(batch.vel, float)[lo:hi],
                             quat=np.asarray(batch.quat, float)[lo:hi], omega=np.asarray(batch.omega, float)[lo:hi],
                             alive=np.asarray(batch.alive, bool)[lo:hi])
            self.shards.append(B200QuadGroup(type_id, sub, params, rate_gains, outer_gains, device=dev, **group_kw))
            self._lo.append(lo)
        self._lo_arr = np.array(self._lo + [n])
        self.params = self.shards[0].params
        self._owner = {int(a): i for i, s in enumerate(self.shards) for a in s.agent_ids}
        self._view = _ShardBatchView(self)

    # ------------------------------------------------------------ protocol
    @property
    def batch(self) -> _ShardBatchView:
        return self._view

    def _shard_of(self, agent_id):
        i = self._owner.get(int(agent_id))
        return None if i is None else self.shards[i]

    def rows_for(self, agent_id: int):
        i = self._owner.get(int(agent_id))
        if i is None:
            return None
        return self._lo[i] + self.shards[i].rows_for(agent_id)

    @property
    def cmd_values(self) -> np.ndarray:
        return np.concatenate([s.cmd_values for s in self.shards])

    @property
    def cmd_level(self) -> np.ndarray:
        return np.concatenate([s.cmd_level for s in self.shards])

    def apply_command(self, cmd) -> bool:
        s = self._shard_of(cmd.agent_id)
        return False if s is None else s.apply_command(cmd)

    def mark_dead(self, agent_ids: Iterable[int]) -> list[int]:
        per = [[] for _ in self.shards]
        for a in agent_ids:
            i = self._owner.get(int(a))
            if i is not None:
                per[i].append(a)
        killed = []
        for s, ids in zip(self.shards, per):
            if ids:
                killed += s.mark_dead(ids)
        return killed

    def _split(self, rows_array):
        return [rows_array[lo:hi] for lo, hi in zip(self._lo_arr[:-1], self._lo_arr[1:])]

    def add_velocity_overlay(self, offsets) -> None:
        for s, part in zip(self.shards, self._split(np.asarray(offsets, dtype=float).reshape(self.n, 3))):
            s.add_velocity_overlay(part)

    def retarget_waypoint(self, point, radius: float) -> None:
        for s in self.shards:
            s.retarget_waypoint(point, radius)

    def apply_viewer_input(self, msg) -> bool:
        """Device viewer influence on every shard (core.py:445-453)."""
        return any([s.apply_viewer_input(msg) for s in self.shards])

    def set_setpoints(self, values, level=0, columns: bool = False) -> None:
        v = np.asarray(values)
        if columns:
            v = v.T
        for s, part in zip(self.shards, self._split(v)):
            s.set_setpoints(np.ascontiguousarray(part), level=level)

    def step_async(self, dt: float, k: int = 1) -> None:
        """Queue k fused ticks on every shard's device (no waiting)."""
        for s in self.shards:
            s.step_async(dt, k)

    def collect_faults(self) -> list[np.ndarray]:
        per = [s.collect_faults() for s in self.shards]
        return [np.sort(np.concatenate([p[t] for p in per])) for t in range(len(per[0]))]

    def step_k(self, dt: float, k: int = 1) -> np.ndarray:
        self.step_async(dt, k)
        ticks = self.collect_faults()
        return np.concatenate(ticks) if len(ticks) > 1 else ticks[0]

    def step(self, dt: float) -> np.ndarray:
        """One tick on every device concurrently; the fault ids of all shards."""
        return self.step_k(dt, 1)

    def snapshot(self, tick: int):
        return batch_snapshot(self.batch, tick)

    def wire_section(self) -> bytes:
        """The type's SnapshotMsg section (wire.py:162-178): each column block
        is the concatenation of the shards' blocks."""
        import struct
        secs = [memoryview(s.wire_section())[6:] for s in self.shards]
        ns = [s.n for s in self.shards]
        parts, offs = [struct.pack("<HI", self.type_id, self.n)], [0] * len(secs)
        for w in (8, 1, 12, 12, 16, 12):      # ids, alive, pos, vel, quat, omega
            for k, (b, n) in enumerate(zip(secs, ns)):
                parts.append(b[offs[k]:offs[k] + w * n])
                offs[k] += w * n
        return b"".join(parts)

    def alive_count(self) -> int:
        return sum(s.alive_count() for s in self.shards)


class MultiDeviceNeighborSeparation:
    """Config 5's separation controller over a ``MultiDeviceQuadGroup`` (one process).

    Per tick (``apply()``, or ``step(dt)`` = apply + the group's step): every
    shard packs its alive positions (float4, NaN for dead / padding rows) into
    slot ``tick & 1`` of EVERY shard's gathered buffer -- the pack is the
    all-gather, NVLink stores for shards on other devices -- then each shard's
    stream waits for all packs (CUDA events) and the overlay kernel adds
    v_i += sum_j k_sep (1 - d/r_sense) (p_i - p_j)/d over the whole swarm into
    the shard's one-tick velocity overlay (core.py:137-139, 172-175).  The
    double buffer lets a shard pack tick t+1 while another still reads tick t:
    a pack of tick t+2 is stream-ordered after its shard's overlay of t+1,
    which waited for every pack of t+1, each after its shard's overlay of t.
    Overlays sum in fixed point, so results are bit-identical to one
    ``B200QuadGroup`` under ``parallel.NeighborSeparation`` at world 1.
    """

    def __init__(self, mg: MultiDeviceQuadGroup, r_sense: float = 2.0, k_sep: float = 1.0,
                 cell: float | None = None):
        if not r_sense > 0.0:
            raise ValidationError("r_sense must be positive")
        self.mg = mg
        self.r_sense, self.k_sep = float(r_sense), float(k_sep)
        self.cell = float(cell) if cell is not None else float(r_sense)
        if self.cell < self.r_sense:
            raise ValidationError("cell must be >= r_sense")
        self._lib = _lib.load()
        shards = mg.shards
        self.world = len(shards)
        self.pad = max(s.n for s in shards)
        self.n_all = self.world * self.pad
        devs = sorted({s.device.index for s in shards})
        for d in devs:                      # NVLink peer stores between the shards' devices
            for q in devs:
                _lib.check(self._lib.swarmstep_enable_peer_access(d, q))
        self.bufs, self.ptrs, self.ws, self.events = [], [], [], []
        nbytes = ctypes.c_uint64()
        _lib.check(self._lib.swarmstep_neighbor_workspace_bytes(self.n_all, ctypes.byref(nbytes)))
        for s in shards:
            with torch.cuda.device(s.device), torch.cuda.stream(s.stream):
                self.bufs.append(torch.full((2 * self.n_all, 4), float("nan"), dtype=torch.float32, device=s.device))
                self.ws.append(torch.empty(int(nbytes.value), dtype=torch.uint8, device=s.device))
        for s in shards:
            with torch.cuda.device(s.device), torch.cuda.stream(s.stream):
                self.ptrs.append(torch.tensor([b.data_ptr() for b in self.bufs], dtype=torch.int64, device=s.device))
                self.events.append(torch.cuda.Event())
        for s in shards:
            s.stream.synchronize()
        self.epoch = 0

    def gathered_positions(self, shard: int = 0) -> torch.Tensor:
        """(n_all, 4) positions of the last exchange as seen by ``shard``."""
        s = self.mg.shards[shard]
        s.stream.synchronize()
        slot = (self.epoch - 1) & 1
        return self.bufs[shard][slot * self.n_all:(slot + 1) * self.n_all]

    def apply(self) -> None:
        """This tick's exchange + overlay on every shard (asynchronous)."""
        shards = self.mg.shards
        off = (self.epoch & 1) * self.n_all
        for j, s in enumerate(shards):
            with torch.cuda.device(s.device):
                _lib.check(self._lib.swarmstep_pack_scatter(s._view_ref, ctypes.c_void_p(self.ptrs[j].data_ptr()),
                                                            self.world, j, self.pad, off, s._stream_h))
            self.events[j].record(s.stream)
        for i, s in enumerate(shards):
            for ev in self.events:
                s.stream.wait_event(ev)
            with torch.cuda.device(s.device):
                _lib.check(self._lib.swarmstep_neighbor_overlay(
                    s._view_ref, self.bufs[i].data_ptr() + off * 16, self.n_all, i * self.pad,
                    ctypes.c_float(self.r_sense), ctypes.c_float(self.k_sep), ctypes.c_float(self.cell), 1,
                    self.ws[i].data_ptr(), ctypes.c_uint64(self.ws[i].numel()), None, s._stream_h))
            s._overlay_active = True
        self.epoch += 1

    def step(self, dt: float) -> np.ndarray:
        self.apply()
        return self.mg.step(dt)
