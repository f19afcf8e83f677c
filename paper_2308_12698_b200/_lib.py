"""ctypes binding of libswarmstep_b200.so (declarations: include/swarmstep_b200.h).

There is no fallback: if the library is missing or cannot be loaded, every
product entry point raises ``NativeLibraryError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import NativeLibraryError, ValidationError

LIB_PATH = Path(__file__).resolve().parent / "libswarmstep_b200.so"
# tools/tune.py points this at variant builds; the product always uses LIB_PATH
_OVERRIDE = os.environ.get("SWARMSTEP_B200_LIB_OVERRIDE")
if _OVERRIDE:
    LIB_PATH = Path(_OVERRIDE)

SWARMSTEP_OK, SWARMSTEP_EINVAL, SWARMSTEP_ECUDA, SWARMSTEP_ENODEV = 0, -1, -2, -3
ABI_VERSION = 3

# column block offsets (SWARMSTEP_COL_*)
COL_POS, COL_VEL, COL_QUAT, COL_OMEGA = 0, 3, 6, 10
COL_POS_LO, COL_INTEGRAL, COL_PREV, COL_CMD, COL_SP, COL_OVERLAY = 13, 14, 17, 20, 27, 31
NCOL = 34
TILE = 128   # agents per tile of the tiled SoA layout (SWARMSTEP_TILE)
FLAG_ALIVE, FLAG_HAS_PREV, LEVEL_SHIFT, LEVEL_MASK = 0x01, 0x02, 2, 0x0C
# swarmstep_quad_step launch flags (SWARMSTEP_STEP_*)
STEP_OVERLAY, STEP_MOTOR, STEP_FORCE_DIRECT, STEP_FORCE_TMA, STEP_FORCE_PAIR = 0x1, 0x2, 0x4, 0x8, 0x10

# every symbol include/swarmstep_b200.h declares
EXPORTS = (
    "swarmstep_abi_version", "swarmstep_last_error", "swarmstep_device_info", "swarmstep_preload",
    "swarmstep_memcpy_async", "swarmstep_stream_sync", "swarmstep_quad_params_init",
    "swarmstep_quad_step", "swarmstep_quad_step_overlapped", "swarmstep_quad_step_collect", "swarmstep_quad_step_lag", "swarmstep_quad_step_circle", "swarmstep_quad_step_circle_overlapped",
    "swarmstep_quad_apply_commands", "swarmstep_quad_set_setpoints",
    "swarmstep_quad_mark_dead", "swarmstep_quad_retarget_waypoint", "swarmstep_quad_viewer_overlay",
    "swarmstep_quad_pack_f64", "swarmstep_quad_unpack_f64",
    "swarmstep_pack_positions", "swarmstep_neighbor_workspace_bytes", "swarmstep_neighbor_overlay",
    "swarmstep_quad_circle_setpoints", "swarmstep_tick_add", "swarmstep_quad_pack_wire",
    "swarmstep_pack_collision", "swarmstep_collision_workspace_bytes", "swarmstep_collision_pairs",
    "swarmstep_unicycle_step", "swarmstep_swarm_stats_workspace_bytes", "swarmstep_quad_swarm_stats",
    "swarmstep_p2p_pack_push", "swarmstep_p2p_wait", "swarmstep_pack_scatter", "swarmstep_enable_peer_access",
    "swarmstep_op_deriv", "swarmstep_op_rk4", "swarmstep_op_mix", "swarmstep_op_rotor", "swarmstep_op_pid",
    "swarmstep_op_outer",
)


def pos_lo_decode(words, hi):
    """Low parts (n, 3) float64 of the packed COL_POS_LO words (uint32 (n,))
    against the float32 position words hi (n, 3): the host restatement of
    ssb::pos_lo_decode (csrc/common.cuh; layout in include/swarmstep_b200.h)."""
    import numpy as np

    w = np.asarray(words, dtype=np.uint32)
    e = (np.asarray(hi, dtype=np.float32).view(np.uint32) >> np.uint32(23)) & np.uint32(0xFF)
    unit = np.ldexp(1.0, np.maximum(e.astype(np.int64), 33) - 159)
    out = np.empty(unit.shape, dtype=np.float64)
    for i in range(3):
        q = ((w >> np.uint32(10 * i)) & np.uint32(0x3FF)).astype(np.int64)
        q = np.where(q >= 512, q - 1024, q)
        out[:, i] = q * unit[:, i]
    return out


class CircleFeedParams(ctypes.Structure):
    """swarmstep_circle_feed (include/swarmstep_b200.h)."""
    _fields_ = [(k, ctypes.c_double) for k in ("dt", "radius", "omega", "z", "phase0", "dphase")]


class GroupView(ctypes.Structure):
    """ctypes mirror of ``swarmstep_group_view``."""

    _fields_ = [
        ("n", ctypes.c_int64), ("stride", ctypes.c_int64),
        ("cols", ctypes.c_void_p), ("flags", ctypes.c_void_p),
        ("counters", ctypes.c_void_p), ("fault_log", ctypes.c_void_p),
        ("fault_cap", ctypes.c_int64),
        ("compensated", ctypes.c_int32), ("_pad", ctypes.c_int32),
    ]


_lock = threading.Lock()
_lib = None


def _declare(lib) -> None:
    vp, i64, i32, f32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_double
    view = ctypes.POINTER(GroupView)
    lib.swarmstep_abi_version.restype = i32
    lib.swarmstep_abi_version.argtypes = []
    lib.swarmstep_last_error.restype = ctypes.c_char_p
    lib.swarmstep_last_error.argtypes = []
    lib.swarmstep_preload.restype = i32
    lib.swarmstep_preload.argtypes = []
    lib.swarmstep_quad_params_init.restype = i32
    lib.swarmstep_quad_params_init.argtypes = [vp, vp, vp]
    lib.swarmstep_memcpy_async.restype = i32
    lib.swarmstep_memcpy_async.argtypes = [vp, vp, ctypes.c_uint64, vp]
    lib.swarmstep_stream_sync.restype = i32
    lib.swarmstep_stream_sync.argtypes = [vp]
    lib.swarmstep_device_info.restype = i32
    lib.swarmstep_device_info.argtypes = [ctypes.POINTER(i32)] * 3
    lib.swarmstep_quad_step.restype = i32
    lib.swarmstep_quad_step.argtypes = [view, vp, f32, i32, i32, ctypes.c_uint32, vp, vp]
    lib.swarmstep_quad_step_overlapped.restype = i32
    lib.swarmstep_quad_step_overlapped.argtypes = [view, vp, f32, i32, i32, ctypes.c_uint32, vp,
                                                   ctypes.c_uint32, ctypes.c_uint32, vp]
    lib.swarmstep_quad_step_collect.restype = i32
    lib.swarmstep_quad_step_collect.argtypes = [view, vp, f32, i32, i32, ctypes.c_uint32, vp, vp]
    lib.swarmstep_swarm_stats_workspace_bytes.restype = i32
    lib.swarmstep_swarm_stats_workspace_bytes.argtypes = [vp]
    lib.swarmstep_quad_swarm_stats.restype = i32
    lib.swarmstep_quad_swarm_stats.argtypes = [view, vp, vp, ctypes.c_uint64, vp]
    lib.swarmstep_quad_step_circle.restype = i32
    lib.swarmstep_quad_step_circle.argtypes = [view, vp, f32, i32, i32, ctypes.c_uint32, vp, vp, vp]
    lib.swarmstep_quad_step_circle_overlapped.restype = i32
    lib.swarmstep_quad_step_circle_overlapped.argtypes = [view, vp, f32, i32, i32, ctypes.c_uint32, vp, vp, vp,
                                                          ctypes.c_uint32, ctypes.c_uint32, vp]
    lib.swarmstep_quad_step_lag.restype = i32
    lib.swarmstep_quad_step_lag.argtypes = [view, vp, vp, f32, f32, i32, i32, ctypes.c_uint32, vp, vp]
    lib.swarmstep_quad_apply_commands.restype = i32
    lib.swarmstep_quad_apply_commands.argtypes = [view, vp, vp, vp, i64, vp]
    lib.swarmstep_quad_set_setpoints.restype = i32
    lib.swarmstep_quad_set_setpoints.argtypes = [view, i64, i64, i32, vp, i64, vp]
    lib.swarmstep_quad_mark_dead.restype = i32
    lib.swarmstep_quad_mark_dead.argtypes = [view, vp, vp, i64, vp]
    lib.swarmstep_quad_retarget_waypoint.restype = i32
    lib.swarmstep_quad_retarget_waypoint.argtypes = [view, ctypes.POINTER(f64), f64, vp]
    lib.swarmstep_quad_viewer_overlay.restype = i32
    lib.swarmstep_quad_viewer_overlay.argtypes = [view, ctypes.POINTER(f64), f64, f64, vp]
    lib.swarmstep_quad_pack_f64.restype = i32
    lib.swarmstep_quad_pack_f64.argtypes = [view, vp, vp, vp, vp, vp, vp]
    lib.swarmstep_quad_unpack_f64.restype = i32
    lib.swarmstep_quad_unpack_f64.argtypes = [view, vp, vp, vp, vp, vp, vp]
    lib.swarmstep_pack_positions.restype = i32
    lib.swarmstep_pack_positions.argtypes = [view, vp, i64, vp]
    lib.swarmstep_neighbor_workspace_bytes.restype = i32
    lib.swarmstep_neighbor_workspace_bytes.argtypes = [i64, ctypes.POINTER(ctypes.c_uint64)]
    lib.swarmstep_neighbor_overlay.restype = i32
    lib.swarmstep_neighbor_overlay.argtypes = [view, vp, i64, i64, f32, f32, f32, i32, vp, ctypes.c_uint64, vp, vp]
    lib.swarmstep_p2p_pack_push.restype = i32
    lib.swarmstep_p2p_pack_push.argtypes = [view, vp, i32, i32, i64, vp, vp, vp, vp]
    lib.swarmstep_op_deriv.restype = i32
    lib.swarmstep_op_deriv.argtypes = [i64] + [vp] * 8 + [vp] * 4 + [vp]
    lib.swarmstep_op_rk4.restype = i32
    lib.swarmstep_op_rk4.argtypes = [i64] + [vp] * 9 + [f32, vp, vp]
    lib.swarmstep_op_mix.restype = i32
    lib.swarmstep_op_mix.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp]
    lib.swarmstep_op_rotor.restype = i32
    lib.swarmstep_op_rotor.argtypes = [i64, vp, f32, f32, f32, vp, vp, vp, vp]
    lib.swarmstep_op_pid.restype = i32
    lib.swarmstep_op_pid.argtypes = [i64, vp, vp, vp, vp, f32, vp, vp, vp, vp, vp, vp, vp]
    lib.swarmstep_op_outer.restype = i32
    lib.swarmstep_op_outer.argtypes = [i64] + [vp] * 9 + [vp, vp, vp, vp]
    lib.swarmstep_p2p_wait.restype = i32
    lib.swarmstep_p2p_wait.argtypes = [vp, i32, vp, vp]
    lib.swarmstep_pack_scatter.restype = i32
    lib.swarmstep_pack_scatter.argtypes = [view, vp, i32, i32, i64, i64, vp]
    lib.swarmstep_enable_peer_access.restype = i32
    lib.swarmstep_enable_peer_access.argtypes = [i32, i32]
    lib.swarmstep_quad_circle_setpoints.restype = i32
    lib.swarmstep_quad_circle_setpoints.argtypes = [view, vp, i64, f64, f64, f64, f64, f64, f64, vp]
    lib.swarmstep_quad_pack_wire.restype = i32
    lib.swarmstep_quad_pack_wire.argtypes = [view, vp, vp, vp]
    lib.swarmstep_pack_collision.restype = i32
    lib.swarmstep_pack_collision.argtypes = [view, f64, vp, i64, vp]
    lib.swarmstep_collision_workspace_bytes.restype = i32
    lib.swarmstep_collision_workspace_bytes.argtypes = [i64, ctypes.POINTER(ctypes.c_uint64)]
    lib.swarmstep_collision_pairs.restype = i32
    lib.swarmstep_collision_pairs.argtypes = [vp, i64, f64, vp, i32, f64, vp, ctypes.c_uint64, vp, ctypes.c_uint64,
                                              vp, vp, ctypes.c_uint64, i32, vp]
    lib.swarmstep_unicycle_step.restype = i32
    lib.swarmstep_unicycle_step.argtypes = [view, f32, f32, f32, i32, i32, vp]
    lib.swarmstep_tick_add.restype = i32
    lib.swarmstep_tick_add.argtypes = [vp, i64, vp]


def load():
    """Load (once) and return the native library; raises if it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2308_12698_b200._build` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        _declare(lib)
        if lib.swarmstep_abi_version() != ABI_VERSION:
            raise NativeLibraryError("ABI version mismatch between Python binding and library")
        _lib = lib
        return _lib


def check(status: int) -> None:
    """Map a C-ABI status onto the exception hierarchy."""
    if status == SWARMSTEP_OK:
        return
    msg = (load().swarmstep_last_error() or b"").decode(errors="replace")
    if status == SWARMSTEP_EINVAL:
        raise ValidationError(msg)
    raise NativeLibraryError(f"swarmstep status {status}: {msg}")
