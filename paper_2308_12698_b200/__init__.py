"""B200-native quadrotor-swarm hot path (Potato / swarmstep, arXiv 2308.12698).

The per-tick batched update of N homogeneous quadrotors -- cascaded position
/ attitude / body-rate controller, saturating mixer, 6-DoF rigid-body model,
RK4 -- as hand-written sm_100a CUDA behind the reference's homogeneous-group
protocol.  See DESIGN.md.
"""

from .commands import AgentCommand, CommandLevel, InfluenceMode, ViewerInputMsg
from .errors import (InvalidStateError, NativeLibraryError, SwarmstepError, ValidationError)
from .params import (OuterGains, PidGains, QuadParams, allocation_matrices, default_outer_gains,
                     default_quad_params, default_rate_gains)
from .state import AgentBatch, BatchSnapshot, SimClock, batch_create, batch_snapshot, quat_yaw, yaw_quat

__all__ = [
    "AgentCommand", "CommandLevel", "InfluenceMode", "ViewerInputMsg", "InvalidStateError", "NativeLibraryError", "SwarmstepError",
    "ValidationError", "OuterGains", "PidGains", "QuadParams", "allocation_matrices",
    "default_outer_gains", "default_quad_params", "default_rate_gains", "AgentBatch",
    "BatchSnapshot", "SimClock", "batch_create", "batch_snapshot", "quat_yaw", "yaw_quat",
    "B200QuadGroup", "B200UnicycleGroup", "MultiDeviceQuadGroup",
]


def __getattr__(name):
    # the group pulls in torch + the native library; import it lazily so the
    # CPU-only parts (params, layouts, commands) stay importable anywhere
    if name == "B200QuadGroup":
        from .group import B200QuadGroup
        return B200QuadGroup
    if name == "B200UnicycleGroup":
        from .unicycle import B200UnicycleGroup
        return B200UnicycleGroup
    if name == "MultiDeviceQuadGroup":
        from .multidevice import MultiDeviceQuadGroup
        return MultiDeviceQuadGroup
    raise AttributeError(name)
