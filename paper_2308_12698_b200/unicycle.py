"""B200UnicycleGroup: the reference's second homogeneous agent type on the GPU
(core.py:208-289).

Same device layout, host mirrors, id routing, death, overlay and snapshot
machinery as ``B200QuadGroup``; the command store holds (v, omega) per agent
(``CommandLevel.UNICYCLE``, wire.py:63) and ``step`` runs the exact-arc
kinematic kernel (csrc/feed.cu ``unicycle_kernel``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import COL_CMD, STEP_OVERLAY
from .commands import LEVEL_POS
from .errors import ValidationError
from .group import B200QuadGroup


@dataclass(frozen=True)
class UnicycleParams:
    """Unicycle limits (core.py:50-57)."""

    v_max: float = 5.0
    omega_max: float = 3.0

    def __post_init__(self):
        if not (self.v_max > 0.0 and self.omega_max > 0.0):
            raise ValidationError("unicycle limits must be positive")


class B200UnicycleGroup(B200QuadGroup):
    """One unicycle type (drop-in for swarmstep.core.UnicycleGroup)."""

    kind = "unicycle"
    _fast_step = False   # step() goes through this class's step_async

    def __init__(self, type_id: int, batch, params: UnicycleParams | None = None, *, device=None):
        super().__init__(type_id, batch, device=device, compensated=True)
        self.params = params if params is not None else UnicycleParams()
        n = self.n
        self._ucmd = np.zeros((n, 2))
        self._cmd_level = np.full(n, LEVEL_POS, dtype=np.uint8)   # unused by this type
        with torch.cuda.device(self.device), torch.cuda.stream(self.stream):
            self._cols[:, COL_CMD:COL_CMD + 7, :].zero_()
        self._sync()

    @property
    def cmd(self) -> np.ndarray:
        """(n, 2) (v, omega) command columns (core.py:262)."""
        return self._ucmd

    @property
    def cmd_values(self):
        raise AttributeError("unicycle groups carry (v, omega) commands in .cmd")

    def apply_command(self, cmd) -> bool:
        """Accept UNICYCLE-level commands for alive agents (core.py:267-272)."""
        row = self._row.get(int(cmd.agent_id))
        key = getattr(cmd.level, "value", cmd.level)
        if row is None or not self._alive[row] or key != "unicycle":
            return False
        vals = np.asarray(cmd.values, dtype=float).ravel()
        if vals.shape[0] != 2:
            raise ValidationError("unicycle commands take 2 values")
        self._ucmd[row] = vals
        full = np.zeros(7, dtype=np.float32)
        full[:2] = vals
        self._pending[row] = (LEVEL_POS, full)
        return True

    def set_setpoints(self, *a, **k):
        raise ValidationError("unicycle groups take (v, omega) commands through apply_command")

    def retarget_waypoint(self, point, radius: float) -> None:
        pass   # unicycles carry no position controller (core.py:278-279)

    def step_async(self, dt: float, k: int = 1) -> None:
        if not dt > 0.0:
            raise ValidationError(f"dt must be positive, got {dt}")
        if k < 1:
            raise ValidationError(f"k must be >= 1, got {k}")
        self._flush_commands()
        self._call(self._lib.swarmstep_unicycle_step, ctypes.c_float(self.params.v_max),
                   ctypes.c_float(self.params.omega_max), ctypes.c_float(dt), int(k),
                   STEP_OVERLAY if self._overlay_active else 0, self._stream_h)
        self._overlay_reset()
        self._launched.append((self._tick, k))     # collect_faults reads the fault counter
        self._tick += k
        self._state_stale = True
