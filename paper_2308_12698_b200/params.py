"""Per-type constants: quadrotor physics and controller gains.

Mirrors the reference's ``QuadParams`` (quad.py:39-69), ``PidGains``
(control.py:40-53), ``OuterGains`` (control.py:56-68) and their default
fixtures (quad.py:72-74, control.py:71-80), and packs them -- together with
the allocation matrix G and its inverse (quad.py:106-127) -- into the
float32 ``swarmstep_quad_params`` struct the kernels take by value.

The group also accepts the reference's own parameter objects: only their
attributes are read.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import ValidationError


@dataclass(frozen=True)
class QuadParams:
    """Physical constants of one quadrotor type (quad.py:39-69)."""

    m: float = 1.0
    i_diag: tuple[float, float, float] = (0.01, 0.01, 0.02)
    g: float = 9.81
    k_t: float = 1e-8
    k_q: float = 1e-10
    arm_length: float = 0.2
    arm_angle: float = float(np.pi / 4)
    omega_max: float = 40000.0

    def __post_init__(self) -> None:
        vals = (self.m, *self.i_diag, self.g, self.k_t, self.k_q,
                self.arm_length, self.arm_angle, self.omega_max)
        if not all(v > 0.0 and np.isfinite(v) for v in vals):
            raise ValidationError("all quadrotor parameters must be strictly positive and finite")
        allocation_matrices(self)  # raises if the geometry is degenerate

    @property
    def f_motor_max(self) -> float:
        return self.k_t * self.omega_max**2

    @property
    def hover_thrust(self) -> float:
        return self.m * self.g


def _vec3(v) -> np.ndarray:
    arr = np.asarray(v, dtype=float) * np.ones(3)
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class PidGains:
    """Per-axis body-rate PID gains with an integral-state clamp (control.py:40-53)."""

    kp: np.ndarray
    ki: np.ndarray
    kd: np.ndarray
    i_limit: np.ndarray

    def __post_init__(self):
        for name in ("kp", "ki", "kd", "i_limit"):
            object.__setattr__(self, name, _vec3(getattr(self, name)))
            if np.any(getattr(self, name) < 0.0):
                raise ValidationError(f"PID gain {name} must be non-negative")


@dataclass(frozen=True)
class OuterGains:
    """Cascaded position/attitude loop gains and limits (control.py:56-68)."""

    kp_pos: np.ndarray
    kv: np.ndarray
    k_att: np.ndarray
    omega_sp_max: float = 20.0
    a_cmd_min: float = 0.5

    def __post_init__(self):
        for name in ("kp_pos", "kv", "k_att"):
            object.__setattr__(self, name, _vec3(getattr(self, name)))


def default_quad_params() -> QuadParams:
    return QuadParams()


def default_rate_gains() -> PidGains:
    # control.py:71-76
    return PidGains(kp=(0.25, 0.25, 0.1), ki=(0.05, 0.05, 0.02),
                    kd=(0.002, 0.002, 0.001), i_limit=0.2)


def default_outer_gains() -> OuterGains:
    # control.py:79-80
    return OuterGains(kp_pos=16.0, kv=8.0, k_att=(12.0, 12.0, 3.0))


def _geometry_key(params) -> tuple:
    return (float(params.arm_length), float(params.arm_angle), float(params.k_q), float(params.k_t))


@lru_cache(maxsize=16)
def _alloc_from_key(key: tuple) -> tuple[np.ndarray, np.ndarray]:
    arm_length, arm_angle, k_q, k_t = key
    ls = arm_length * np.sin(arm_angle)
    lc = arm_length * np.cos(arm_angle)
    kr = k_q / k_t
    g_mat = np.array([
        [1.0, 1.0, 1.0, 1.0],
        [ls, -ls, -ls, ls],
        [-lc, -lc, lc, lc],
        [kr, -kr, kr, -kr],
    ])
    if abs(np.linalg.det(g_mat)) <= 1e-12:
        raise ValidationError("allocation matrix is singular (degenerate arm angle)")
    g_inv = np.linalg.inv(g_mat)
    g_mat.setflags(write=False)
    g_inv.setflags(write=False)
    return g_mat, g_inv


def allocation_matrices(params) -> tuple[np.ndarray, np.ndarray]:
    """(G, G^-1) in float64, as quad.py:106-122 builds them."""
    return _alloc_from_key(_geometry_key(params))


class DeviceParams(ctypes.Structure):
    """ctypes mirror of ``swarmstep_quad_params`` (include/swarmstep_b200.h)."""

    _fields_ = [
        ("m", ctypes.c_float), ("inv_m", ctypes.c_float), ("g", ctypes.c_float),
        ("inv_ixx", ctypes.c_float), ("inv_iyy", ctypes.c_float), ("inv_izz", ctypes.c_float),
        ("ixx", ctypes.c_float), ("iyy", ctypes.c_float), ("izz", ctypes.c_float),
        ("k_t", ctypes.c_float), ("omega_max", ctypes.c_float), ("f_max", ctypes.c_float),
        ("fc_max", ctypes.c_float),
        ("G", ctypes.c_float * 16), ("G_inv", ctypes.c_float * 16),
        ("kp", ctypes.c_float * 3), ("ki", ctypes.c_float * 3), ("kd", ctypes.c_float * 3),
        ("i_limit", ctypes.c_float * 3),
        ("kp_pos", ctypes.c_float * 3), ("kv", ctypes.c_float * 3), ("k_att", ctypes.c_float * 3),
        ("omega_sp_max", ctypes.c_float), ("a_cmd_min", ctypes.c_float),
        ("_pad", ctypes.c_float * 2),
    ]


def pack_device_params(params, rate_gains, outer_gains) -> DeviceParams:
    """Round the float64 per-type constants to the kernel's float32 struct."""
    g_mat, g_inv = allocation_matrices(params)
    # the kernel's mixer uses G^-1 = sign(G^T) * c (csrc/quad_math.cuh mix_row)
    c = np.abs(g_inv[0])
    if not (g_mat[1, 0] > 0 and g_mat[2, 0] < 0 and g_mat[3, 0] > 0
            and np.allclose(g_inv, np.sign(g_mat.T) * c, rtol=1e-9, atol=0.0)):
        raise ValidationError("allocation matrix does not have the quadrotor X structure")
    ixx, iyy, izz = (float(v) for v in params.i_diag)
    f_max = float(params.k_t) * float(params.omega_max) ** 2
    dp = DeviceParams()
    dp.m, dp.inv_m, dp.g = params.m, 1.0 / params.m, params.g
    dp.inv_ixx, dp.inv_iyy, dp.inv_izz = 1.0 / ixx, 1.0 / iyy, 1.0 / izz
    dp.ixx, dp.iyy, dp.izz = ixx, iyy, izz
    dp.k_t, dp.omega_max, dp.f_max, dp.fc_max = params.k_t, params.omega_max, f_max, 4.0 * f_max
    for i, v in enumerate(g_mat.ravel()):
        dp.G[i] = v
    for i, v in enumerate(g_inv.ravel()):
        dp.G_inv[i] = v
    for name in ("kp", "ki", "kd", "i_limit"):
        arr = getattr(dp, name)
        for i, v in enumerate(_vec3(getattr(rate_gains, name))):
            arr[i] = v
    for name in ("kp_pos", "kv", "k_att"):
        arr = getattr(dp, name)
        for i, v in enumerate(_vec3(getattr(outer_gains, name))):
            arr[i] = v
    dp.omega_sp_max = float(outer_gains.omega_sp_max)
    dp.a_cmd_min = float(outer_gains.a_cmd_min)
    return dp
