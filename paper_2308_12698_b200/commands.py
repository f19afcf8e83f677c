"""Command levels, per-agent commands and viewer influence messages, mirroring
wire.py:54-113.

The group accepts these or the reference's own ``AgentCommand`` objects:
only ``agent_id``, ``level`` (an enum whose ``.value`` is "pos" / "rate" /
"motor" / "unicycle", or that string itself) and ``values`` are read.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .errors import ValidationError


class CommandLevel(str, Enum):
    """Command abstraction levels accepted by the central side (wire.py:54-64)."""

    POS = "pos"          # 7 values: p_sp (3), v_sp (3), yaw_sp
    RATE = "rate"        # 4 values: omega_sp (3), f_c
    MOTOR = "motor"      # 4 values: per-rotor speed (RPM)
    UNICYCLE = "unicycle"  # 2 values: v, omega

    @property
    def n_values(self) -> int:
        return {"pos": 7, "rate": 4, "motor": 4, "unicycle": 2}[self.value]


@dataclass(frozen=True)
class AgentCommand:
    agent_id: int
    level: CommandLevel
    values: tuple[float, ...]

    def __post_init__(self):
        if len(self.values) != self.level.n_values:
            raise ValidationError(
                f"level {self.level.value} takes {self.level.n_values} values, got {len(self.values)}")


class InfluenceMode(str, Enum):
    """Viewer influence modes (wire.py:92-95)."""

    ATTRACT = "attract"
    REPEL = "repel"
    WAYPOINT = "waypoint"


@dataclass(frozen=True)
class ViewerInputMsg:
    """A viewer influence message (wire.py:103-113); the groups' device
    ``apply_viewer_input`` also takes the reference's own message objects."""

    mode: InfluenceMode
    world_point: tuple[float, float, float]
    radius: float
    strength: float

    def __post_init__(self):
        if self.radius < 0.0 or self.strength < 0.0:
            raise ValidationError("radius and strength must be non-negative")


# device level codes (core.py:73; include/swarmstep_b200.h SWARMSTEP_LEVEL_*)
LEVEL_POS, LEVEL_RATE, LEVEL_MOTOR = 0, 1, 2
_LEVEL_CODES = {"pos": LEVEL_POS, "rate": LEVEL_RATE, "motor": LEVEL_MOTOR}


def level_code(level) -> int | None:
    """Device level code for a CommandLevel-like value, None for non-quad levels."""
    key = getattr(level, "value", level)
    return _LEVEL_CODES.get(key) if isinstance(key, str) else None
