"""B200QuadGroup: the reference's homogeneous quadrotor group, on one B200.

Drop-in for ``swarmstep.core.QuadGroup`` (core.py:76-205): it implements the
duck-typed group protocol the reference ``World`` calls (core.py:308-505) --
``kind``, ``type_id``, ``batch``, ``params``, ``step(dt)``,
``apply_command``, ``mark_dead``, ``add_velocity_overlay``,
``retarget_waypoint``, ``snapshot``, ``rows_for``, ``cmd_values`` /
``cmd_level`` -- and adds the bulk / fused entry points the B200 path is
built for: ``step_k(dt, k)`` (k fused ticks per launch), ``set_setpoints``
(device-resident setpoint feed) and ``step_async`` / ``collect_faults``.

Device layout: one float32 buffer in tiled structure-of-arrays
form -- tiles of 128 agents, each tile holding its ``NCOL`` component columns
contiguously -- plus a uint8 flag column (alive | has_prev | level).  The float64 host views the
reference exposes (``batch.pos`` ...) are mirrors synchronised lazily: a
read after a step packs the device columns to float64 on the device and
copies them down once.  Writes into those mirror arrays do not reach the
device; use ``push_host_state()`` after editing them.
"""

from __future__ import annotations

import ctypes
import math
import os
from typing import Iterable

import numpy as np
import torch

from . import _lib
from ._lib import (COL_CMD, COL_INTEGRAL, COL_OVERLAY, COL_PREV, COL_SP, FLAG_HAS_PREV,
                   LEVEL_MASK, LEVEL_SHIFT, NCOL, STEP_FORCE_DIRECT, STEP_FORCE_PAIR, STEP_FORCE_TMA, STEP_MOTOR,
                   STEP_OVERLAY, TILE, GroupView)
from .commands import LEVEL_MOTOR, LEVEL_POS, LEVEL_RATE, level_code
from .errors import InvalidStateError, NativeLibraryError, ValidationError
from .params import (default_outer_gains, default_quad_params, default_rate_gains,
                     pack_device_params)
from .state import AgentBatch, batch_snapshot, quat_yaw

_ROW_ALIGN = TILE  # row capacity is a whole number of 128-agent tiles
_ZEROS = (0.0,) * 7
_PINNED_MIRROR_MAX = 8_000_000   # agents: 0.83 GB of pinned float64 mirror


_F32_MAX = float(np.finfo(np.float32).max)
_TWO_PI = 2.0 * math.pi
_POS_SCALE_MAX = 1e15


def f32_commands(vals: np.ndarray, pos_rows) -> np.ndarray:
    """float64 command values (rows x 7) -> the float32 device command store.

    Two conversions keep float32 commands faithful to the float64 reference:
    * POS yaw setpoints are reduced to [-pi, pi] in float64 first (the outer
      loop only uses cos / sin of yaw, control.py:252-256): a float32 yaw of
      |yaw| ~ 1000 rad would carry ~6e-5 rad of rounding, far above the 1e-5
      parity budget, the reduced one <= 1.2e-7;
    * POS position / velocity setpoints so large that the acceleration
      command |a| = |kp (p_sp - p) + kv (v_sp - v) + g| would overflow
      float32 when squared (the float64 reference has the range) are scaled
      down together to |.| <= 1e15: the outer loop uses only a's direction and
      the sign of z_body . a (the thrust saturates), and scaling both by one
      factor moves that direction by ~|p| / 1e15 (< 1e-10 rad for any
      position the float32 state can hold precisely);
    * other finite values beyond float32 range saturate at +-FLT_MAX instead
      of becoming inf.
    Non-finite values pass unchanged (they raise or fault like the reference).
    """
    v = np.array(vals, dtype=np.float64, copy=True).reshape(-1, 7)
    pos_rows = np.asarray(pos_rows, dtype=bool).reshape(-1)
    y = v[pos_rows, 6]
    fin = np.isfinite(y)
    y[fin] -= np.round(y[fin] / _TWO_PI) * _TWO_PI
    v[pos_rows, 6] = y
    pv = v[pos_rows, :6]
    big = np.max(np.abs(np.where(np.isfinite(pv), pv, 0.0)), axis=1, initial=0.0) > _POS_SCALE_MAX
    if big.any():
        rows = np.flatnonzero(pos_rows)[big]
        blk = v[rows, :6]
        scale = _POS_SCALE_MAX / np.max(np.abs(np.where(np.isfinite(blk), blk, 0.0)), axis=1)
        v[rows, :6] = blk * scale[:, None]
    fin = np.isfinite(v)
    v[fin] = np.clip(v[fin], -_F32_MAX, _F32_MAX)
    return v.astype(np.float32)


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class DeviceBatchView:
    """``group.batch``: the AgentBatch interface (state.py:43-102) over a B200
    group.  ``type_id``, ``agent_ids``, ``n`` and ``alive`` come from the host
    without a device read (alive changes only through mark_dead and collected
    faults), so the World's per-tick alive counts (core.py:370) stay cheap; the
    float64 ``pos`` / ``vel`` / ``quat`` / ``omega`` mirror is pulled from the
    device on first access after a step."""

    def __init__(self, group):
        self._g = group

    @property
    def type_id(self) -> int:
        return self._g._batch.type_id

    @property
    def agent_ids(self) -> np.ndarray:
        return self._g._batch.agent_ids

    @property
    def n(self) -> int:
        return self._g.n

    @property
    def alive(self) -> np.ndarray:
        if self._g._launched:           # faults of launches not collected yet live on the device
            self._g._pull_state()
        return self._g._alive

    def _full(self) -> AgentBatch:
        self._g._pull_state()
        return self._g._batch

    @property
    def pos(self) -> np.ndarray:
        return self._full().pos

    @property
    def vel(self) -> np.ndarray:
        return self._full().vel

    @property
    def quat(self) -> np.ndarray:
        return self._full().quat

    @property
    def omega(self) -> np.ndarray:
        return self._full().omega

    def validate(self) -> None:
        self._full().validate()

    def index_of(self, agent_id: int):
        return self._g.rows_for(agent_id)


# Overlapped launches from this many ticks per launch: the compute-bound
# paired kernel gains (1M agents, K = 10: +6%, profiles/pdl_r02/), while the
# HBM-bound K = 1 launch loses to the per-tile epoch handshake (0.90 -> 0.81
# of the copy bandwidth), so short launches keep plain stream order.
_OVERLAP_MIN_K = 4
# ... and up to this many: a waiting tile traps after ~18 s (a broken chain
# fails loudly), far beyond one CTA's K <= 4096 ticks; longer launches keep
# plain stream order
_OVERLAP_MAX_K = 4096


class B200QuadGroup:
    """One quadrotor type stepped by the sm_100a fused kernel.

    ``overlap_launches`` (default True; env ``SWARMSTEP_B200_NO_OVERLAP=1``
    turns it off for new groups) lets back-to-back ``step_async`` launches of
    4 to 4096 ticks overlap tile by tile (swarmstep_quad_step_overlapped);
    results are bit-identical either way.
    """

    kind = "quadrotor"

    def __init__(self, type_id: int, batch, params=None, rate_gains=None, outer_gains=None, *,
                 device=None, compensated: bool = True, fault_capacity: int | None = None,
                 motor_tau: float = 0.0):
        lib = _lib.load()
        if not torch.cuda.is_available():
            raise NativeLibraryError("B200QuadGroup needs a CUDA device (there is no CPU fallback)")
        n = int(batch.agent_ids.shape[0])
        if n < 1:
            raise ValidationError("a group needs at least one agent")
        self._lib = lib
        self.type_id = int(type_id)
        self.params = params if params is not None else default_quad_params()
        self.rate_gains = rate_gains if rate_gains is not None else default_rate_gains()
        self.outer_gains = outer_gains if outer_gains is not None else default_outer_gains()
        self._dparams = pack_device_params(self.params, self.rate_gains, self.outer_gains)
        self.compensated = bool(compensated)
        # opt-in first-order rotor lag (north star; absent in the reference):
        # 0 = the reference's instantaneous mixer
        self.motor_tau = float(motor_tau)
        if not (np.isfinite(self.motor_tau) and self.motor_tau >= 0.0):
            raise ValidationError(f"motor_tau must be finite and >= 0, got {motor_tau}")
        self.n = n
        self.stride = _round_up(n, _ROW_ALIGN)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
            with torch.cuda.stream(self.stream):
                self.ntiles = self.stride // TILE
                self._cols = torch.zeros((self.ntiles, NCOL, TILE), dtype=torch.float32, device=self.device)
                self._flags = torch.zeros(self.stride, dtype=torch.uint8, device=self.device)
                self._counters = torch.zeros(4, dtype=torch.int32, device=self.device)
                cap = int(fault_capacity) if fault_capacity is not None else n
                self._fault_cap = max(1, cap)
                self._fault_log = torch.zeros(self._fault_cap, dtype=torch.int64, device=self.device)
                self._motor = None
                if self.motor_tau > 0.0:
                    # rotor thrusts [tiles, 4, 128], starting at the hover split m g / 4
                    self._motor = torch.full((self.ntiles, 4, TILE), self.params.hover_thrust / 4.0,
                                             dtype=torch.float32, device=self.device)
            self._counters_host = torch.zeros(4, dtype=torch.int32, pin_memory=True)
        self._counters_np = self._counters_host.numpy()          # same pinned memory, cheap reads
        self._counters_host_ptr = ctypes.c_void_p(self._counters_host.data_ptr())
        self._view = GroupView(n=n, stride=self.stride, cols=_ptr(self._cols), flags=_ptr(self._flags),
                               counters=_ptr(self._counters), fault_log=_ptr(self._fault_log),
                               fault_cap=self._fault_cap, compensated=int(self.compensated))
        self._view_ref = ctypes.byref(self._view)
        # overlapped step launches (swarmstep_quad_step_overlapped): one epoch
        # word per tile, the chain's last published epoch (0: no launch yet)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self._tile_epoch = torch.zeros(self.ntiles, dtype=torch.int32, device=self.device)
        self._tile_epoch_ptr = _ptr(self._tile_epoch)
        self._pdl_epoch = 0
        self.overlap_launches = os.environ.get("SWARMSTEP_B200_NO_OVERLAP", "") != "1"
        self._dev_idx = self.device.index
        self._stream_h = ctypes.c_void_p(self.stream.cuda_stream)
        self._params_ref = ctypes.byref(self._dparams)

        # host mirrors (the reference's numpy columns); up to _PINNED_MIRROR_MAX
        # agents they live in pinned memory, so a state pull is one DMA per column
        cols = self._mirror_columns(n)
        for name, width, src in (("pos", 3, batch.pos), ("vel", 3, batch.vel), ("quat", 4, batch.quat),
                                 ("omega", 3, batch.omega)):
            cols[name][...] = np.asarray(src, dtype=float).reshape(n, width)
        cols["alive"][...] = np.asarray(batch.alive, dtype=bool).reshape(n)
        self._batch = AgentBatch(type_id=int(getattr(batch, "type_id", type_id)),
                                 agent_ids=np.array(batch.agent_ids, dtype=np.uint64), **cols)
        self._row = {int(a): i for i, a in enumerate(self._batch.agent_ids)}
        self._ids_dev = None             # device copy of agent_ids (wire packing), on demand
        self._wire_bufs = None           # wire_section's device / pinned buffers, on demand
        self._pull_bufs = None           # _pull_state's device staging, on demand
        self._alive = self._batch.alive  # exact: changes only via mark_dead / faults
        self._batch_view = DeviceBatchView(self)
        self._state_stale = False        # device state newer than the host mirror
        # command store (core.py:98-104): position hold at the initial pose
        self._cmd_level = np.full(n, LEVEL_POS, dtype=np.uint8)
        self._cmd_values = np.zeros((n, 7))
        self._cmd_values[:, :3] = self._batch.pos
        self._cmd_values[:, 6] = quat_yaw(self._batch.quat)
        self._cmd_stale = False          # device command store newer than host mirror
        self._pending: dict[int, tuple[int, np.ndarray]] = {}
        self._nonfinite_rows: set[int] = set()
        self._overlay_active = False
        self._overlay_poison = False
        self._motor_possible = False     # sticky: a MOTOR-level row may exist
        self._tick = 0                   # ticks launched so far (fault-log tags)
        self._launched: list[tuple[int, int]] = []  # (first tick, k) not yet collected
        self._fault_seen = 0             # fault-log entries already returned
        self._copy_stream = None         # side stream for host->device setpoint uploads
        self._sp_stage = [None, None]    # double-buffered setpoint staging
        self._sp_consumed = [None, None]
        self._sp_src = [None, None]
        self._sp_slot = 0

        self.push_host_state(upload_commands=True)

    # ------------------------------------------------------------------ utils
    def _mirror_columns(self, n: int) -> dict:
        """Float64 pos / vel / quat / omega and bool alive host columns, laid out
        as the device pack writes them; pinned when small enough (else pageable)."""
        f64 = alive = None
        self._mirror_pinned = None
        if n <= _PINNED_MIRROR_MAX:
            try:
                self._mirror_pinned = (torch.empty(13 * n, dtype=torch.float64, pin_memory=True),
                                       torch.empty(n, dtype=torch.uint8, pin_memory=True))
                f64 = self._mirror_pinned[0].numpy()
                alive = self._mirror_pinned[1].numpy().view(np.bool_)
            except RuntimeError:      # pinned memory exhausted: pageable mirror
                self._mirror_pinned = None
                f64 = None
        if f64 is None:
            f64, alive = np.empty(13 * n), np.empty(n, dtype=bool)
        return dict(pos=f64[:3 * n].reshape(n, 3), vel=f64[3 * n:6 * n].reshape(n, 3),
                    quat=f64[6 * n:10 * n].reshape(n, 4), omega=f64[10 * n:].reshape(n, 3), alive=alive)

    def _call(self, fn, *args) -> None:
        # the device guard costs more than the launch itself on the per-tick
        # path: only switch when the caller's current device differs
        if torch.cuda.current_device() == self._dev_idx:
            _lib.check(fn(self._view_ref, *args))
        else:
            with torch.cuda.device(self.device):
                _lib.check(fn(self._view_ref, *args))

    def _sync(self) -> None:
        _lib.check(self._lib.swarmstep_stream_sync(self._stream_h))

    @property
    def cols(self) -> torch.Tensor:
        """The device tiled-SoA buffer [stride/128, NCOL, 128] (float32)."""
        return self._cols

    def column_block(self, c0: int, c1: int) -> torch.Tensor:
        """Columns [c0, c1) of rows [0, n) as an (n, c1-c0) device tensor (a copy);
        stream-ordered after this group's work."""
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            out = self._cols[:, c0:c1, :].permute(0, 2, 1).reshape(-1, c1 - c0)[:self.n].clone()
        self.stream.synchronize()
        return out

    def _cols_write(self, c0: int, data: torch.Tensor, add: bool = False) -> None:
        """Write (n, k) rows into columns [c0, c0+k) (on the current stream)."""
        k = data.shape[1]
        buf = torch.zeros((self.stride, k), dtype=torch.float32, device=self.device)
        buf[:self.n] = data
        view = self._cols[:, c0:c0 + k, :]
        src = buf.view(self.ntiles, TILE, k).permute(0, 2, 1)
        if add:
            view += src
        else:
            view.copy_(src)

    @property
    def flags(self) -> torch.Tensor:
        return self._flags

    # --------------------------------------------------------- host <-> device
    def push_host_state(self, upload_commands: bool = False) -> None:
        """Upload the host mirror (pos/vel/quat/omega/alive) to the device columns."""
        b = self._batch
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            pos = torch.from_numpy(np.ascontiguousarray(b.pos)).to(self.device, non_blocking=False)
            vel = torch.from_numpy(np.ascontiguousarray(b.vel)).to(self.device)
            quat = torch.from_numpy(np.ascontiguousarray(b.quat)).to(self.device)
            omega = torch.from_numpy(np.ascontiguousarray(b.omega)).to(self.device)
            alive = torch.from_numpy(b.alive.astype(np.uint8)).to(self.device)
            self._call(self._lib.swarmstep_quad_unpack_f64, _ptr(pos), _ptr(vel), _ptr(quat),
                       _ptr(omega), _ptr(alive), ctypes.c_void_p(self.stream.cuda_stream))
            if upload_commands:
                if np.any(self._cmd_level == LEVEL_MOTOR):
                    self._motor_possible = True
                vals = torch.from_numpy(f32_commands(self._cmd_values, self._cmd_level == LEVEL_POS)).to(self.device)
                self._cols_write(COL_CMD, vals)
                lv = torch.from_numpy(self._cmd_level.astype(np.uint8)).to(self.device)
                fl = self._flags[:self.n]
                fl.copy_((fl & (0xFF ^ LEVEL_MASK)) | (lv << LEVEL_SHIFT))
            self._sync()
        self._alive = b.alive
        # the device holds the float32 (hi + lo) image of what was pushed;
        # re-read it so the host mirror always shows the device state
        self._state_stale = True

    def _pull_state(self) -> None:
        if not self._state_stale:
            return
        n = self.n
        b = self._batch
        if self._pull_bufs is None:     # device staging for the float64 pack, reused
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                self._pull_bufs = (torch.empty(n * 13, dtype=torch.float64, device=self.device),
                                   torch.empty(n, dtype=torch.uint8, device=self.device))
        buf, alive = self._pull_bufs
        p = _ptr(buf)
        self._call(self._lib.swarmstep_quad_pack_f64, p, p + n * 3 * 8, p + n * 6 * 8, p + n * 10 * 8,
                   _ptr(alive), self._stream_h)
        # straight into the mirror arrays (no intermediate host buffer); a
        # mirror array that is not a plain contiguous buffer goes via a copy
        for col, off, width in ((b.pos, 0, 3), (b.vel, 3, 3), (b.quat, 6, 4), (b.omega, 10, 3)):
            self._d2h(col, p + off * n * 8, width * n * 8)
        self._d2h(b.alive, _ptr(alive), n)
        self._sync()
        self._state_stale = False

    def _d2h(self, dst: np.ndarray, src: int, nbytes: int) -> None:
        if dst.flags.c_contiguous and dst.flags.writeable and dst.nbytes == nbytes:
            _lib.check(self._lib.swarmstep_memcpy_async(dst.ctypes.data, src, nbytes, self._stream_h))
        else:
            tmp = np.empty(dst.shape, dtype=dst.dtype)
            _lib.check(self._lib.swarmstep_memcpy_async(tmp.ctypes.data, src, nbytes, self._stream_h))
            self._sync()
            dst[...] = tmp

    def _pull_commands(self) -> None:
        if not self._cmd_stale:
            return
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            vals = self._cols[:, COL_CMD:COL_CMD + 7, :].permute(0, 2, 1).reshape(-1, 7)[:self.n].double().cpu().numpy()
            lv = ((self._flags[:self.n] & LEVEL_MASK) >> LEVEL_SHIFT).cpu().numpy()
        self._cmd_values[:] = vals
        self._cmd_level[:] = lv
        # commands queued since the device columns were last written are newer
        for row, (lvl, full) in self._pending.items():
            self._cmd_level[row] = lvl
            self._cmd_values[row] = full
        self._cmd_stale = False

    def _flush_commands(self) -> None:
        if not self._pending:
            return
        count = len(self._pending)
        rows = np.fromiter(self._pending.keys(), dtype=np.int64, count=count)
        pend = list(self._pending.values())
        levels = np.fromiter((lvl for lvl, _ in pend), dtype=np.uint8, count=count)
        vals = f32_commands([v for _, v in pend], levels == LEVEL_POS)   # float64 -> float32
        self._pending.clear()
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            d_rows = torch.from_numpy(rows).to(self.device)
            d_lv = torch.from_numpy(levels).to(self.device)
            d_vals = torch.from_numpy(vals).to(self.device)
            self._call(self._lib.swarmstep_quad_apply_commands, _ptr(d_rows), _ptr(d_lv), _ptr(d_vals),
                       ctypes.c_int64(rows.shape[0]), ctypes.c_void_p(self.stream.cuda_stream))
            # keep the staging tensors alive until the kernel has consumed them
            self._staging = (d_rows, d_lv, d_vals)

    # ------------------------------------------------------- group protocol
    @property
    def batch(self) -> DeviceBatchView:
        """The AgentBatch view of the state table (DeviceBatchView)."""
        return self._batch_view

    @property
    def cmd_values(self) -> np.ndarray:
        self._pull_commands()
        return self._cmd_values

    @property
    def cmd_level(self) -> np.ndarray:
        self._pull_commands()
        return self._cmd_level

    def rows_for(self, agent_id: int) -> int | None:
        return self._row.get(int(agent_id))

    def apply_command(self, cmd) -> bool:
        """Latest-wins command write (core.py:117-135)."""
        row = self._row.get(int(cmd.agent_id))
        if row is None or not self._alive[row]:
            return False
        lvl = level_code(cmd.level)
        if lvl is None:
            return False
        want = 7 if lvl == LEVEL_POS else 4
        try:      # the common case, a flat tuple of numbers: plain Python floats
            vals = tuple(map(float, cmd.values))
        except TypeError:
            vals = tuple(np.asarray(cmd.values, dtype=float).ravel().tolist())
        if len(vals) != want:
            raise ValidationError(f"level takes {want} values, got {len(vals)}")
        # no device read: the row goes to the (possibly stale) host mirror and
        # the pending queue, which _pull_commands re-applies over the device copy
        full = vals + _ZEROS[:7 - want]
        self._cmd_level[row] = lvl
        self._cmd_values[row] = full
        if lvl == LEVEL_MOTOR:
            self._motor_possible = True
        if all(map(math.isfinite, full)):
            self._nonfinite_rows.discard(row)
        else:
            self._nonfinite_rows.add(row)
        self._pending[row] = (lvl, full)
        return True

    def set_setpoints(self, values, level=LEVEL_POS, row0: int = 0, columns: bool = False) -> None:
        """Bulk setpoints for rows [row0, row0 + count) (alive rows only).

        ``values`` is (count, 7|4) -- or (7|4, count) with ``columns=True``,
        the device's own SoA layout -- as numpy, a host tensor (pinned for
        asynchronous upload) or a device tensor.  Host data is copied on a
        side stream into one of two staging buffers, so an upload overlaps
        the group's previous launch; a scatter kernel then writes the command
        columns in stream order.  This is the device-resident setpoint feed
        that replaces per-agent ``apply_command`` calls for whole swarms
        (SURVEY.md 8(f) f1).  Unlike ``apply_command`` it does not screen for
        non-finite values: those fault the affected rows.
        """
        lvl = level_code(level) if not isinstance(level, int) else level
        if lvl not in (LEVEL_POS, LEVEL_RATE, LEVEL_MOTOR):
            raise ValidationError(f"bad level {level!r}")
        want = 7 if lvl == LEVEL_POS else 4
        if isinstance(values, torch.Tensor) and (values.is_cuda or values.dtype == torch.float32):
            t = values
        else:
            # host data in another precision: the same float32 conversion as
            # apply_command (yaw reduction, saturation)
            a = values.numpy() if isinstance(values, torch.Tensor) else np.asarray(values)
            if a.dtype != np.float32 and a.ndim == 2 and (a.shape[0] if columns else a.shape[1]) == want:
                rows = a.T if columns else a
                full = np.zeros((rows.shape[0], 7))
                full[:, :want] = rows
                conv = f32_commands(full, np.full(rows.shape[0], lvl == LEVEL_POS))[:, :want]
                a = conv.T if columns else conv
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
        if t.dim() != 2 or (t.shape[0] if columns else t.shape[1]) != want:
            raise ValidationError(f"setpoints must be ({want}, count) / (count, {want})")
        count = int(t.shape[1] if columns else t.shape[0])
        if row0 < 0 or row0 + count > self.n:
            raise ValidationError("setpoint rows out of range")
        if t.dtype != torch.float32 and not t.is_cuda:
            t = t.float()
        self._flush_commands()
        if t.is_cuda and t.device != self.device:
            raise ValidationError(f"setpoints on {t.device}, group on {self.device}")
        with torch.cuda.device(self.device):
            if t.is_cuda:
                # the caller produced the tensor on its own stream: order this
                # group's (non-blocking) stream after it before any conversion
                # or launch reads it, and tell the allocator the group's stream
                # uses it
                self.stream.wait_stream(torch.cuda.current_stream(t.device))
                with torch.cuda.stream(self.stream):
                    if t.dtype != torch.float32:
                        t = t.float()
                    cols = t if columns else t.T
                    if cols.stride(1) != 1:
                        cols = cols.contiguous()
                    self._call(self._lib.swarmstep_quad_set_setpoints, ctypes.c_int64(row0), ctypes.c_int64(count),
                               int(lvl), _ptr(cols), ctypes.c_int64(cols.stride(0)),
                               ctypes.c_void_p(self.stream.cuda_stream))
                cols.record_stream(self.stream)
                values.record_stream(self.stream)
            else:
                if not columns:
                    t = t.T.contiguous()
                slot = self._sp_slot
                self._sp_slot ^= 1
                if self._sp_stage[slot] is None or self._sp_stage[slot].shape[1] < count:
                    if self._copy_stream is None:
                        self._copy_stream = torch.cuda.Stream(self.device)
                    old = self._sp_stage[slot]
                    if old is not None:
                        # a queued scatter / copy may still use the old buffer:
                        # its memory is reusable only after both streams pass here
                        old.record_stream(self.stream)
                        old.record_stream(self._copy_stream)
                    with torch.cuda.stream(self.stream):
                        self._sp_stage[slot] = torch.empty((7, max(count, 1)), dtype=torch.float32,
                                                           device=self.device)
                    self._sp_stage[slot].record_stream(self._copy_stream)
                    self._sp_consumed[slot] = None
                buf = self._sp_stage[slot][:want, :count]
                with torch.cuda.stream(self._copy_stream):
                    if self._sp_consumed[slot] is not None:
                        self._copy_stream.wait_event(self._sp_consumed[slot])
                    buf.copy_(t, non_blocking=True)
                    copied = torch.cuda.Event()
                    copied.record(self._copy_stream)
                self.stream.wait_event(copied)
                with torch.cuda.stream(self.stream):
                    self._call(self._lib.swarmstep_quad_set_setpoints, ctypes.c_int64(row0), ctypes.c_int64(count),
                               int(lvl), _ptr(buf), ctypes.c_int64(self._sp_stage[slot].shape[1]),
                               ctypes.c_void_p(self.stream.cuda_stream))
                    ev = torch.cuda.Event()
                    ev.record(self.stream)
                    self._sp_consumed[slot] = ev
                # the source must outlive the asynchronous copy
                self._sp_src[slot] = t
        if self._nonfinite_rows:
            self._nonfinite_rows = {r for r in self._nonfinite_rows if not (row0 <= r < row0 + count)}
        if lvl == LEVEL_MOTOR:
            self._motor_possible = True
        self._cmd_stale = True

    def add_velocity_overlay(self, offsets) -> None:
        """One-tick velocity offsets added to v_sp of POS rows (core.py:137-139)."""
        if isinstance(offsets, torch.Tensor) and offsets.is_cuda:
            # produced on the caller's stream: order the group's stream after it
            self.stream.wait_stream(torch.cuda.current_stream(offsets.device))
            offsets.record_stream(self.stream)
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            t = offsets if isinstance(offsets, torch.Tensor) else torch.from_numpy(np.asarray(offsets, dtype=np.float32))
            t = t.to(self.device, torch.float32).reshape(self.n, 3)
            if not bool(torch.isfinite(t).all()):
                self._overlay_poison = True
            if not self._overlay_active:
                self._cols[:, COL_OVERLAY:COL_OVERLAY + 3, :].zero_()
            self._cols_write(COL_OVERLAY, t, add=True)
        self._overlay_active = True

    def apply_viewer_input(self, msg) -> bool:
        """``World._apply_viewer_input`` for this group (core.py:445-453) without
        pulling positions to the host: WAYPOINT retargets (core.py:447-449);
        ATTRACT / REPEL evaluate ``viewer_velocity_offsets`` (wire.py:320-340) on
        the device into the one-tick overlay, which is activated only if some
        offset is non-zero (the reference's ``offsets.any()``).  Returns whether
        an overlay was added.  One 4-byte device read."""
        mode = getattr(msg.mode, "value", msg.mode)
        if mode == "waypoint":
            self.retarget_waypoint(msg.world_point, msg.radius)
            return False
        if mode not in ("attract", "repel"):
            raise ValidationError(f"unknown influence mode {msg.mode!r}")
        radius = float(msg.radius)
        if not radius > 0.0:
            return False
        gain = float(msg.strength) if mode == "attract" else -float(msg.strength)
        pt = (ctypes.c_double * 3)(*[float(x) for x in np.asarray(msg.world_point, dtype=float).ravel()[:3]])
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self._counters[2].zero_()
            if not self._overlay_active:
                self._cols[:, COL_OVERLAY:COL_OVERLAY + 3, :].zero_()
            self._call(self._lib.swarmstep_quad_viewer_overlay, pt, ctypes.c_double(radius), ctypes.c_double(gain),
                       self._stream_h)
            _lib.check(self._lib.swarmstep_memcpy_async(self._counters_host.data_ptr(), self._counters.data_ptr(),
                                                        self._counters.numel() * 4, self._stream_h))
        self._sync()
        if int(self._counters_np[2]) == 0:
            return False
        if not np.isfinite(gain):
            self._overlay_poison = True
        self._overlay_active = True
        return True

    def retarget_waypoint(self, point, radius: float) -> None:
        """Alive rows within ``radius`` of ``point`` go to POS hold there (core.py:141-149)."""
        pt = (ctypes.c_double * 3)(*[float(x) for x in np.asarray(point, dtype=float).ravel()[:3]])
        self._flush_commands()
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self._call(self._lib.swarmstep_quad_retarget_waypoint, pt, ctypes.c_double(float(radius)),
                       ctypes.c_void_p(self.stream.cuda_stream))
        self._cmd_stale = True
        # rows rewritten by the waypoint carry finite values now
        if self._nonfinite_rows:
            self._pull_commands()
            self._nonfinite_rows = {r for r in self._nonfinite_rows
                                    if not np.all(np.isfinite(self._cmd_values[r]))}

    def mark_dead(self, agent_ids: Iterable[int]) -> list[int]:
        """Kill agents; returns the ids that were alive (core.py:151-158)."""
        killed, rows = [], []
        for aid in agent_ids:
            row = self._row.get(int(aid))
            if row is not None and self._alive[row]:
                self._alive[row] = False
                killed.append(int(aid))
                rows.append(row)
        if rows:
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                d_rows = torch.tensor(rows, dtype=torch.int64).to(self.device)
                self._call(self._lib.swarmstep_quad_mark_dead, _ptr(d_rows), None,
                           ctypes.c_int64(len(rows)), ctypes.c_void_p(self.stream.cuda_stream))
                self._staging_dead = d_rows
        return killed

    def snapshot(self, tick: int):
        return batch_snapshot(self.batch, tick)

    def wire_section(self) -> bytes:
        """This group's SnapshotMsg section (wire.py:162-178), packed on the device:
        u16 type_id, u32 n, then 61*n bytes of columns."""
        import struct
        n = self.n
        if self._wire_bufs is None:   # cached: device columns + pinned host copy
            self._wire_bufs = (torch.empty(61 * n + 8, dtype=torch.uint8, device=self.device),
                               torch.empty(61 * n, dtype=torch.uint8, pin_memory=True))
        dev, host = self._wire_bufs
        self.pack_wire_async(dev)
        _lib.check(self._lib.swarmstep_memcpy_async(host.data_ptr(), dev.data_ptr(), 61 * n, self._stream_h))
        self._sync()
        return b"".join((struct.pack("<HI", self._batch.type_id, n), host.numpy().data))

    def pack_wire_async(self, buf: torch.Tensor) -> None:
        """Enqueue the device packing of this group's 61*n section column bytes
        (ids, alive, pos, vel, canonical quat, omega; wire.py:162-178) into the
        device buffer ``buf`` on the group's stream, after its queued ticks."""
        if buf.device != self.device or buf.dtype != torch.uint8 or buf.numel() < 61 * self.n:
            raise ValidationError("pack_wire_async needs a uint8 buffer of >= 61*n bytes on the group's device")
        if self._ids_dev is None:
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                self._ids_dev = torch.from_numpy(self._batch.agent_ids.view(np.int64).copy()).to(self.device)
        self._call(self._lib.swarmstep_quad_pack_wire, _ptr(self._ids_dev), _ptr(buf), self._stream_h)

    # ------------------------------------------------------------ stepping
    def _any_pos_rows(self) -> bool:
        self._pull_commands()
        return bool(np.any(self._cmd_level == LEVEL_POS))

    def step_async(self, dt: float, k: int = 1) -> None:
        """Launch k fused ticks without waiting; ``collect_faults()`` gathers fault ids."""
        if not dt > 0.0:
            raise ValidationError(f"dt must be positive, got {dt}")
        if k < 1:
            raise ValidationError(f"k must be >= 1, got {k}")
        if (self._nonfinite_rows or self._overlay_poison) and self._any_pos_rows():
            # the reference's outer loop runs quat_mul over every row whenever
            # a POS row exists and raises on non-finite input (quat.py:84),
            # before any state changes
            self._overlay_reset()
            raise InvalidStateError("non-finite quaternion input")
        self._flush_commands()
        flags = self._launch_flags()
        ep = self._overlap_epochs(k, flags)
        if ep is not None:
            self._call(self._lib.swarmstep_quad_step_overlapped, self._params_ref, ctypes.c_float(dt), int(k), flags,
                       ctypes.c_uint32(self._tick & 0xFFFFFF), self._tile_epoch_ptr, *ep, self._stream_h)
            self._pdl_epoch = ep[1].value
        else:
            self._launch(dt, k, flags, self._tick & 0xFFFFFF, None)
        self._overlay_reset()
        # no per-launch read-back: back-to-back launches stay back to back on the
        # stream; collect_faults copies the fault counter once (the log entries
        # carry their tick)
        self._launched.append((self._tick, k))
        self._tick += k
        self._state_stale = True

    def _overlap_epochs(self, k: int, flags: int):
        """(wait, set) epochs for an overlapped launch (each tile of the launch
        waits for its own tile of the previous one instead of the whole grid),
        or None for a plain stream-ordered launch; the caller stores set into
        _pdl_epoch once the launch is queued."""
        if not (self.overlap_launches and _OVERLAP_MIN_K <= k <= _OVERLAP_MAX_K and self._motor is None
                and not flags & (STEP_FORCE_TMA | STEP_FORCE_DIRECT)):
            return None
        wait = self._pdl_epoch
        return ctypes.c_uint32(wait), ctypes.c_uint32((wait + 1) & 0xFFFFFFFF or 1)

    def _launch(self, dt: float, k: int, flags: int, tick_base: int, tick_dev) -> None:
        """One step launch on the group's stream (no host bookkeeping)."""
        s = self._stream_h
        if self._motor is None:
            self._call(self._lib.swarmstep_quad_step, self._params_ref, ctypes.c_float(dt), int(k), flags,
                       ctypes.c_uint32(tick_base), tick_dev, s)
        else:
            self._call(self._lib.swarmstep_quad_step_lag, self._params_ref, _ptr(self._motor),
                       ctypes.c_float(self.motor_tau), ctypes.c_float(dt), int(k), flags,
                       ctypes.c_uint32(tick_base), tick_dev, s)

    def swarm_stats(self) -> dict:
        """Swarm-wide reductions on the device (one deterministic launch):
        alive count, centroid, mean and max speed, alive bounding box."""
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            if getattr(self, "_stats_ws", None) is None:
                nb = ctypes.c_uint64(0)
                _lib.check(self._lib.swarmstep_swarm_stats_workspace_bytes(ctypes.byref(nb)))
                self._stats_ws = torch.zeros(int(nb.value), dtype=torch.uint8, device=self.device)
                self._stats_out = torch.zeros(12, dtype=torch.float64, device=self.device)
            self._call(self._lib.swarmstep_quad_swarm_stats, _ptr(self._stats_out), _ptr(self._stats_ws),
                       ctypes.c_uint64(self._stats_ws.numel()), ctypes.c_void_p(self.stream.cuda_stream))
            o = self._stats_out.cpu().numpy()
        alive = int(o[0])
        c = o[1:4] / alive if alive else np.full(3, np.nan)
        return {"alive": alive, "centroid": c, "mean_speed_sq": o[4] / alive if alive else float("nan"),
                "max_speed": float(np.sqrt(o[5])), "bbox_min": o[6:9].copy(), "bbox_max": o[9:12].copy()}

    def motor_thrusts(self) -> np.ndarray:
        """Host float64 copy of the rotor thrusts (n, 4) in newtons (motor_tau > 0)."""
        if self._motor is None:
            raise ValidationError("no rotor state: the group runs the reference's instantaneous mixer (motor_tau = 0)")
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            m = self._motor.permute(0, 2, 1).reshape(-1, 4)[:self.n].double().cpu().numpy()
        return np.ascontiguousarray(m)

    def set_motor_thrusts(self, thrusts) -> None:
        """Load the rotor thrusts (n, 4) in newtons (motor_tau > 0)."""
        if self._motor is None:
            raise ValidationError("no rotor state: the group runs the reference's instantaneous mixer (motor_tau = 0)")
        t = np.asarray(thrusts, dtype=np.float32).reshape(self.n, 4)
        pad = np.zeros((self.stride, 4), dtype=np.float32)
        pad[:self.n] = t
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            src = torch.from_numpy(pad).to(self.device).reshape(self.ntiles, TILE, 4).permute(0, 2, 1)
            self._motor.copy_(src)
            self._sync()

    # kernel selection for tuning: "auto" (the library's choice), "direct",
    # "pair" (two rows per thread on packed FP32x2) or "tma"
    kernel = "auto"

    def _launch_flags(self) -> int:
        f = STEP_OVERLAY if self._overlay_active else 0
        if self._motor_possible:
            f |= STEP_MOTOR
        if self.kernel == "direct":
            f |= STEP_FORCE_DIRECT
        elif self.kernel == "tma":
            f |= STEP_FORCE_TMA
        elif self.kernel == "pair":
            f |= STEP_FORCE_PAIR
        return f

    def _overlay_reset(self) -> None:
        if self._overlay_active:
            with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
                self._cols[:, COL_OVERLAY:COL_OVERLAY + 3, :].zero_()
        self._overlay_active = False
        self._overlay_poison = False

    def collect_faults(self) -> list[np.ndarray]:
        """Wait for the launches since the last call; fault ids per tick, in row order."""
        # the fault counter to pinned host memory, stream-ordered after every launch
        _lib.check(self._lib.swarmstep_memcpy_async(self._counters_host.data_ptr(), self._counters.data_ptr(),
                                                    self._counters.numel() * 4, self._stream_h))
        self._sync()
        launched, self._launched = self._launched, []
        return self._faults_for([t0 + j for t0, k in launched for j in range(k)])

    def _faults_for(self, ticks) -> list[np.ndarray]:
        """Fault ids per tick from the fault log (the counters are on the host)."""
        count = int(self._counters_np[0])
        if count == self._fault_seen:
            return [np.empty(0, dtype=np.uint64) for _ in ticks]
        if count > self._fault_cap:
            raise NativeLibraryError("fault log overflow")
        log = self._fault_log[self._fault_seen:count].cpu().numpy().astype(np.uint64)
        self._fault_seen = count
        tag = (log >> np.uint64(40)).astype(np.int64)
        rows = (log & np.uint64((1 << 40) - 1)).astype(np.int64)
        self._alive[rows] = False
        out = []
        for t in ticks:
            sel = np.sort(rows[tag == (t & 0xFFFFFF)])
            out.append(self._batch.agent_ids[sel].copy())
        return out

    def step_k(self, dt: float, k: int = 1) -> np.ndarray:
        """k fused ticks (== k successive step(dt) calls with fixed commands)."""
        self.step_async(dt, k)
        per = self.collect_faults()
        return np.concatenate(per) if len(per) > 1 else per[0]

    _fast_step = True   # the single-call synchronous tick below applies to this class

    def step(self, dt: float) -> np.ndarray:
        """Advance one tick in place; returns fault ids (core.py:166-202)."""
        if (not self._fast_step or self._launched or self._pending or self._motor is not None
                or self._nonfinite_rows or self._overlay_poison or not dt > 0.0):
            return self.step_k(dt, 1)
        # the World's per-tick call: launch + fault counter readback + wait in
        # one FFI crossing (swarmstep_quad_step_collect)
        self._call(self._lib.swarmstep_quad_step_collect, self._params_ref, ctypes.c_float(dt), 1,
                   self._launch_flags(), ctypes.c_uint32(self._tick & 0xFFFFFF), self._counters_host_ptr,
                   self._stream_h)
        self._overlay_reset()
        tick = self._tick
        self._tick += 1
        self._state_stale = True
        if int(self._counters_np[0]) == self._fault_seen:
            return np.empty(0, dtype=np.uint64)
        return self._faults_for([tick])[0]

    # -------------------------------------------------------------- extras
    def alive_count(self) -> int:
        return int(self._alive.sum())

    def alive_mask(self) -> np.ndarray:
        """Host alive flags as of the last collected step (no device read:
        alive changes only through mark_dead and collected faults)."""
        return self._alive

    @property
    def agent_ids(self) -> np.ndarray:
        """The group's static agent ids (no device read)."""
        return self._batch.agent_ids

    def pid_state_dict(self) -> dict:
        """Host float64 copy of the PID columns (RatePidState, control.py:100-114)
        and the stale inner-loop setpoints (QuadGroup.omega_sp / f_c_sp)."""
        blk = self.column_block(COL_INTEGRAL, COL_PREV + 3).double().cpu().numpy()
        sp = self.column_block(COL_SP, COL_SP + 4).double().cpu().numpy()
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            hp = ((self._flags[:self.n] & FLAG_HAS_PREV) != 0).cpu().numpy()
        return {"integral": blk[:, :3].copy(), "prev_omega": blk[:, 3:6].copy(), "has_prev": hp,
                "omega_sp": sp[:, :3].copy(), "f_c_sp": sp[:, 3].copy()}

    @property
    def pid_state(self):
        """QuadGroup.pid_state (core.py:93): a RatePidState-shaped snapshot
        (integral, prev_omega, has_prev) read from the device; write back with
        set_pid_state."""
        from .functional import RatePidState
        d = self.pid_state_dict()
        st = RatePidState(self.n)
        st.integral[:], st.prev_omega[:], st.has_prev[:] = d["integral"], d["prev_omega"], d["has_prev"]
        return st

    @property
    def omega_sp(self) -> np.ndarray:
        """QuadGroup.omega_sp (core.py:109): last tick's inner-loop rate setpoints."""
        return self.pid_state_dict()["omega_sp"]

    @property
    def f_c_sp(self) -> np.ndarray:
        """QuadGroup.f_c_sp (core.py:110): last tick's collective-thrust setpoints."""
        return self.pid_state_dict()["f_c_sp"]

    def set_pid_state(self, integral=None, prev_omega=None, has_prev=None, omega_sp=None, f_c_sp=None) -> None:
        """Load PID / stale-setpoint columns (test and resume support)."""
        n = self.n
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            def put(c0, arr, k):
                self._cols_write(c0, torch.from_numpy(np.asarray(arr, dtype=np.float32).reshape(n, k)).to(self.device))
            if integral is not None:
                put(COL_INTEGRAL, integral, 3)
            if prev_omega is not None:
                put(COL_PREV, prev_omega, 3)
            if omega_sp is not None:
                put(COL_SP, omega_sp, 3)
            if f_c_sp is not None:
                put(COL_SP + 3, f_c_sp, 1)
            if has_prev is not None:
                hp = torch.from_numpy(np.asarray(has_prev, dtype=np.uint8).reshape(n)).to(self.device)
                fl = self._flags[:n]
                fl.copy_((fl & (0xFF ^ FLAG_HAS_PREV)) | (hp * FLAG_HAS_PREV))
            self._sync()
