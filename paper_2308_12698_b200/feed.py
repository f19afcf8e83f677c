"""Device-resident setpoint feed and CUDA-graph tick loops.

``CircleFeed`` is the reference's in-loop circle strategy (client.py:43-73,
control.py:297-315) as one kernel writing the command columns of every alive
row from a device tick counter -- the reference builds one Python
``AgentCommand`` per agent per tick instead (80% of a 5k-agent tick,
SURVEY.md 3.5).

``TickGraph`` captures ``ticks`` World-style ticks -- [feed ->] fused step --
of one group into a single CUDA graph, so a tick costs one graph node pair
instead of a Python call, a ctypes call and a launch.  Fault ids keep their
exact tick (the step kernel reads the tick from the device counter) and are
gathered by the group's own ``collect_faults()``.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from ._lib import COL_OVERLAY, STEP_OVERLAY
from .errors import InvalidStateError, ValidationError


class CircleFeed:
    """circle_swarm_strategy on the device for one group (all alive rows, POS level).

    Phases follow make_circle_layout (client.py:43-52): phase_r = 2 pi r / n
    over the group's rows, unless ``phase0`` / ``dphase`` are given.
    """

    def __init__(self, group, dt: float, radius: float = 5.0, omega: float = 0.3, z: float = 10.0,
                 phase0: float = 0.0, dphase: float | None = None):
        if not radius > 0.0:
            raise ValidationError("circle radius must be positive")  # control.py:305-306
        self.group, self.dt = group, float(dt)
        self.radius, self.omega, self.z = float(radius), float(omega), float(z)
        self.phase0 = float(phase0)
        self.dphase = float(dphase) if dphase is not None else 2.0 * math.pi / max(group.n, 1)
        self._lib = _lib.load()
        with torch.cuda.device(group.device):
            self.tick = torch.full((1,), group._tick, dtype=torch.int64, device=group.device)
            self._zero = torch.zeros(1, dtype=torch.int64, device=group.device)
        self._zero_ptr = ctypes.c_void_p(self._zero.data_ptr())
        self._tick_ptr = ctypes.c_void_p(self.tick.data_ptr())
        self._fp_key = None

    def apply(self, tick_offset: int = 0, sync_tick: bool = True) -> None:
        """Write the setpoints of the group's current tick (the next one to
        step) + tick_offset; with sync_tick=False, of (*tick + tick_offset)
        with the device tick counter as it stands (the graph-captured form)."""
        g = self.group
        g._flush_commands()          # earlier apply_command calls land first (latest wins)
        if sync_tick:
            # the host knows the tick: pass it as the offset from a zero counter
            # (no device write, no torch launch on the per-tick path)
            tick_ptr, off = self._zero.data_ptr(), g._tick + int(tick_offset)
        else:
            tick_ptr, off = self.tick.data_ptr(), int(tick_offset)
        g._call(self._lib.swarmstep_quad_circle_setpoints, tick_ptr, off, self.dt, self.radius, self.omega,
                self.z, self.phase0, self.dphase, g._stream_h)
        g._cmd_stale = True

    def step_fused(self, k: int) -> None:
        """K ticks of [circle feed -> step] in ONE launch: the kernel evaluates
        the circle setpoint of each tick itself (swarmstep_quad_step_circle),
        bit-identical to K x (apply(); group.step(dt)) but with the state
        register-resident across the K ticks.  Asynchronous like
        group.step_async; collect_faults() gathers the per-tick fault ids."""
        g = self.group
        if k < 1:
            raise ValidationError(f"k must be >= 1, got {k}")
        if g._overlay_active:
            raise ValidationError("the fused circle feed takes no velocity overlay")
        if getattr(g, "_motor", None) is not None:
            raise ValidationError("the fused circle feed runs the reference mixer (motor_tau = 0)")
        g._flush_commands()
        # lean per-launch host path (a launch at <= 100k agents is shorter than
        # the Python around it): the feed struct is rebuilt only when the
        # feed's attributes change, no torch device / stream guards
        key = (self.dt, self.radius, self.omega, self.z, self.phase0, self.dphase)
        if key != self._fp_key:
            self._fp = _lib.CircleFeedParams(*key)
            self._fp_ref, self._fp_key = ctypes.byref(self._fp), key
        if g._tick < (1 << 31):
            # the absolute tick as the launch's base over a device zero: no
            # fill kernel between back-to-back launches
            tick_ptr, base = self._zero_ptr, g._tick
        else:
            with torch.cuda.device(g.device), torch.cuda.stream(g.stream):
                self.tick.fill_(g._tick)
            tick_ptr, base = self._tick_ptr, 0
        flags = g._launch_flags()
        ep = g._overlap_epochs(k, flags)
        if ep is None:
            g._call(self._lib.swarmstep_quad_step_circle, g._params_ref, ctypes.c_float(self.dt), int(k), flags,
                    ctypes.c_uint32(base), tick_ptr, self._fp_ref, g._stream_h)
        else:    # overlapping the group's previous step launch (group.step_async)
            g._call(self._lib.swarmstep_quad_step_circle_overlapped, g._params_ref, ctypes.c_float(self.dt), int(k),
                    flags, ctypes.c_uint32(base), tick_ptr, self._fp_ref, g._tile_epoch_ptr, *ep, g._stream_h)
            g._pdl_epoch = ep[1].value
        g._launched.append((g._tick, k))     # collect_faults reads the fault counter
        g._tick += k
        g._state_stale = True
        g._cmd_stale = True

    def advance(self, k: int) -> None:
        g = self.group
        with torch.cuda.device(g.device):
            _lib.check(self._lib.swarmstep_tick_add(self.tick.data_ptr(), int(k),
                                                    ctypes.c_void_p(g.stream.cuda_stream)))


class TickGraph:
    """``ticks`` ticks of [feed ->] [neighbour coupling ->] fused step (K=1 each)
    as one CUDA graph.  ``coupling`` is a ``parallel.NeighborSeparation`` on a
    single-rank shard or uses the P2P exchange (its exchange is then device-only)."""

    def __init__(self, group, dt: float, ticks: int, feed: CircleFeed | None = None, coupling=None):
        if ticks < 1:
            raise ValidationError("ticks must be >= 1")
        if group._overlay_active:
            raise ValidationError("apply or clear the pending overlay before capturing a graph")
        group._flush_commands()
        self.group, self.dt, self.ticks = group, float(dt), int(ticks)
        self.feed = feed
        if coupling is not None and coupling.shard.world != 1 and coupling.exchange != "p2p":
            raise ValidationError("graph-captured coupling needs a single-rank shard or the P2P exchange "
                                  "(no NCCL call in the graph)")
        self.coupling = coupling
        self._lib = _lib.load()
        with torch.cuda.device(group.device):
            self.tick = feed.tick if feed is not None else torch.full(
                (1,), group._tick, dtype=torch.int64, device=group.device)
        _lib.check(self._lib.swarmstep_preload())   # no lazy module loads inside the capture
        torch.cuda.synchronize(group.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.device(group.device):
            with torch.cuda.graph(self.graph, stream=group.stream):
                self._body()
        torch.cuda.synchronize(group.device)

    def _body(self) -> None:
        g = self.group
        s = ctypes.c_void_p(g.stream.cuda_stream)
        flags = g._launch_flags() | (STEP_OVERLAY if self.coupling is not None else 0)
        for j in range(self.ticks):
            if self.feed is not None:
                self.feed.apply(j, sync_tick=False)
            if self.coupling is not None:
                self.coupling.launch(accumulate=False)     # overwrites the overlay block
            g._launch(self.dt, 1, flags, j, self.tick.data_ptr())
        if self.coupling is not None:
            with torch.cuda.stream(g.stream):
                g._cols[:, COL_OVERLAY:COL_OVERLAY + 3, :].zero_()   # one-tick overlay: leave it clear
        _lib.check(self._lib.swarmstep_tick_add(self.tick.data_ptr(), self.ticks, s))

    def replay(self) -> None:
        """Run the captured ticks (asynchronously on the group's stream)."""
        g = self.group
        # the captured launches have fixed flags: a pending one-tick overlay
        # would be ignored (and land on a later eager tick) or overwritten by
        # the coupling, so it is refused; non-finite POS commands raise like
        # step_async does (quat.py:84), before any state changes
        if g._overlay_active:
            raise ValidationError("a velocity overlay is pending: a graph replay does not apply it "
                                  "(step eagerly or let the coupling compute the overlay)")
        if self.feed is None and g._nonfinite_rows and g._any_pos_rows():
            raise InvalidStateError("non-finite quaternion input")
        if g._pending:
            g._flush_commands()
        with torch.cuda.device(g.device), torch.cuda.stream(g.stream):
            self.tick.fill_(g._tick)       # the graph's tick counter follows the group's
            self.graph.replay()
        g._launched.append((g._tick, self.ticks))
        g._tick += self.ticks
        g._state_stale = True
        if self.feed is not None:
            g._cmd_stale = True
