"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the float64 C oracle.

``oracle/quad_oracle.c`` restates the reference's quadrotor hot path
(swarmstep quad.py / control.py / core.py QuadGroup.step) per agent in
float64.  This module builds/loads it and offers:

* per-function batch wrappers (deriv / rk4 / mix / pid / outer loop), pinned
  against golden vectors from the reference itself (tests/golden/);
* ``OracleGroup``: a float64 twin of ``QuadGroup`` (core.py:76-205) with the
  same command store and group protocol, used as the checker in the parity
  tests and as the CPU baseline arm of bench.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this.  The product package never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"

_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class OracleParams(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_double), ("ixx", ctypes.c_double), ("iyy", ctypes.c_double),
        ("izz", ctypes.c_double), ("g", ctypes.c_double), ("k_t", ctypes.c_double),
        ("k_q", ctypes.c_double), ("arm_length", ctypes.c_double), ("arm_angle", ctypes.c_double),
        ("omega_max", ctypes.c_double), ("f_max", ctypes.c_double),
        ("G", ctypes.c_double * 16), ("Ginv", ctypes.c_double * 16),
        ("kp", ctypes.c_double * 3), ("ki", ctypes.c_double * 3), ("kd", ctypes.c_double * 3),
        ("i_limit", ctypes.c_double * 3),
        ("kp_pos", ctypes.c_double * 3), ("kv", ctypes.c_double * 3), ("k_att", ctypes.c_double * 3),
        ("omega_sp_max", ctypes.c_double), ("a_cmd_min", ctypes.c_double),
    ]


def build(force: bool = False) -> Path:
    src = HERE / "quad_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-B" if force else "build/liboracle.so"],
                       check=True, capture_output=True)
    return LIB_PATH


_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.POINTER(OracleParams)
        i64 = ctypes.c_int64
        lib.oracle_group_step.restype = i64
        lib.oracle_group_step.argtypes = [i64, ctypes.c_double, P, _f64p, _f64p, _f64p, _f64p, _u8p,
                                          _f64p, _f64p, _u8p, _f64p, _f64p, _u8p, _f64p, _f64p, _u8p,
                                          ctypes.c_int]
        lib.oracle_group_step_lag.restype = i64
        lib.oracle_group_step_lag.argtypes = [i64, ctypes.c_double, P, _f64p, _f64p, _f64p, _f64p, _u8p,
                                              _f64p, _f64p, _u8p, _f64p, _f64p, _u8p, _f64p, _f64p, _u8p,
                                              ctypes.c_int, _f64p, ctypes.c_double]
        lib.oracle_deriv_batch.restype = None
        lib.oracle_deriv_batch.argtypes = [i64, _f64p, _f64p, _f64p, P, _f64p]
        lib.oracle_rk4_batch.restype = i64
        lib.oracle_rk4_batch.argtypes = [i64, _f64p, _u8p, _f64p, _f64p, P, ctypes.c_double, _u8p]
        lib.oracle_mix_batch.restype = None
        lib.oracle_mix_batch.argtypes = [i64, _f64p, _f64p, P, _f64p, _f64p, _u8p]
        lib.oracle_pid_batch.restype = None
        lib.oracle_pid_batch.argtypes = [i64, _f64p, _f64p, _f64p, P, ctypes.c_double, _u8p,
                                         _f64p, _f64p, _u8p, _f64p, _f64p]
        lib.oracle_outer_batch.restype = ctypes.c_int
        lib.oracle_outer_batch.argtypes = [i64, _f64p, _f64p, _f64p, _u8p, _f64p, _f64p, _f64p, P,
                                           _f64p, _f64p, _u8p]
        _lib = lib
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_f64p)


def _b(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_u8p)


# reference defaults (quad.py:47-54, control.py:71-80)
DEFAULT_QUAD = dict(m=1.0, i_diag=(0.01, 0.01, 0.02), g=9.81, k_t=1e-8, k_q=1e-10,
                    arm_length=0.2, arm_angle=np.pi / 4, omega_max=40000.0)
DEFAULT_RATE = dict(kp=(0.25, 0.25, 0.1), ki=(0.05, 0.05, 0.02), kd=(0.002, 0.002, 0.001), i_limit=0.2)
DEFAULT_OUTER = dict(kp_pos=16.0, kv=8.0, k_att=(12.0, 12.0, 3.0), omega_sp_max=20.0, a_cmd_min=0.5)


def _get(obj, name, default):
    if obj is None:
        return default[name]
    if isinstance(obj, dict):
        return obj.get(name, default[name])
    return getattr(obj, name)


def make_params(quad=None, rate=None, outer=None) -> OracleParams:
    """Fill the float64 struct from reference-shaped objects (or dicts / defaults)."""
    p = OracleParams()
    p.m = _get(quad, "m", DEFAULT_QUAD)
    p.ixx, p.iyy, p.izz = (float(v) for v in _get(quad, "i_diag", DEFAULT_QUAD))
    p.g = _get(quad, "g", DEFAULT_QUAD)
    p.k_t = _get(quad, "k_t", DEFAULT_QUAD)
    p.k_q = _get(quad, "k_q", DEFAULT_QUAD)
    p.arm_length = _get(quad, "arm_length", DEFAULT_QUAD)
    p.arm_angle = _get(quad, "arm_angle", DEFAULT_QUAD)
    p.omega_max = _get(quad, "omega_max", DEFAULT_QUAD)
    p.f_max = p.k_t * p.omega_max ** 2
    # quad.py:106-122: G and np.linalg.inv(G)
    ls, lc, kr = p.arm_length * np.sin(p.arm_angle), p.arm_length * np.cos(p.arm_angle), p.k_q / p.k_t
    g_mat = np.array([[1.0, 1.0, 1.0, 1.0], [ls, -ls, -ls, ls], [-lc, -lc, lc, lc], [kr, -kr, kr, -kr]])
    g_inv = np.linalg.inv(g_mat)
    for i in range(16):
        p.G[i] = g_mat.ravel()[i]
        p.Ginv[i] = g_inv.ravel()[i]
    for name in ("kp", "ki", "kd", "i_limit"):
        v = np.asarray(_get(rate, name, DEFAULT_RATE), dtype=float) * np.ones(3)
        arr = getattr(p, name)
        for i in range(3):
            arr[i] = v[i]
    for name in ("kp_pos", "kv", "k_att"):
        v = np.asarray(_get(outer, name, DEFAULT_OUTER), dtype=float) * np.ones(3)
        arr = getattr(p, name)
        for i in range(3):
            arr[i] = v[i]
    p.omega_sp_max = _get(outer, "omega_sp_max", DEFAULT_OUTER)
    p.a_cmd_min = _get(outer, "a_cmd_min", DEFAULT_OUTER)
    return p


# ---------------------------------------------------------------- functions
def deriv(state13: np.ndarray, f_c: np.ndarray, tau: np.ndarray, p: OracleParams) -> np.ndarray:
    s = np.ascontiguousarray(state13, dtype=np.float64)
    out = np.empty_like(s)
    load().oracle_deriv_batch(s.shape[0], _d(s), _d(np.ascontiguousarray(f_c, dtype=float)),
                              _d(np.ascontiguousarray(tau, dtype=float)), ctypes.byref(p), _d(out))
    return out


def rk4(state13: np.ndarray, alive: np.ndarray, f_c, tau, p: OracleParams, dt: float):
    """rk4_step semantics on (n,13) rows in place; returns (faulted rows mask)."""
    fault = np.zeros(state13.shape[0], dtype=np.uint8)
    load().oracle_rk4_batch(state13.shape[0], _d(state13), _b(alive),
                            _d(np.ascontiguousarray(f_c, dtype=float)),
                            _d(np.ascontiguousarray(tau, dtype=float)), ctypes.byref(p), dt, _b(fault))
    return fault.astype(bool)


def mix(f_c, tau, p: OracleParams):
    f_c = np.ascontiguousarray(f_c, dtype=float)
    n = f_c.shape[0]
    motors, realized, sat = np.empty((n, 4)), np.empty((n, 4)), np.empty(n, dtype=np.uint8)
    load().oracle_mix_batch(n, _d(f_c), _d(np.ascontiguousarray(tau, dtype=float)), ctypes.byref(p),
                            _d(motors), _d(realized), _b(sat))
    return motors, realized, sat.astype(bool)


def pid(omega, omega_sp, f_c_sp, p: OracleParams, dt: float, alive, integral, prev_omega, has_prev):
    """rate_pid_step; integral / prev_omega / has_prev (uint8) are updated in place."""
    omega = np.ascontiguousarray(omega, dtype=float)
    n = omega.shape[0]
    tau, f_c = np.empty((n, 3)), np.empty(n)
    load().oracle_pid_batch(n, _d(omega), _d(np.ascontiguousarray(omega_sp, dtype=float)),
                            _d(np.ascontiguousarray(f_c_sp, dtype=float)), ctypes.byref(p), dt,
                            _b(np.ascontiguousarray(alive, dtype=np.uint8)), _d(integral), _d(prev_omega),
                            _b(has_prev), _d(tau), _d(f_c))
    return f_c, tau


def outer(pos, vel, quat, alive, p_sp, v_sp, yaw, p: OracleParams):
    pos = np.ascontiguousarray(pos, dtype=float)
    n = pos.shape[0]
    w_sp, f_c, low = np.empty((n, 3)), np.empty(n), np.empty(n, dtype=np.uint8)
    bad = load().oracle_outer_batch(
        n, _d(pos), _d(np.ascontiguousarray(vel, dtype=float)), _d(np.ascontiguousarray(quat, dtype=float)),
        _b(np.ascontiguousarray(alive, dtype=np.uint8)), _d(np.ascontiguousarray(p_sp, dtype=float)),
        _d(np.ascontiguousarray(v_sp, dtype=float)), _d(np.ascontiguousarray(yaw, dtype=float)),
        ctypes.byref(p), _d(w_sp), _d(f_c), _b(low))
    return w_sp, f_c, low.astype(bool), bool(bad)


def quat_yaw(q):
    q = np.asarray(q, dtype=float)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.arctan2(2.0 * (w * z + x * y), 1.0 - 2.0 * (y * y + z * z))


class OracleInvalidState(Exception):
    """quat_mul would have raised InvalidStateError (quat.py:84)."""


_LEVELS = {"pos": 0, "rate": 1, "motor": 2}


class OracleGroup:
    """float64 twin of QuadGroup (core.py:76-205) backed by the C oracle."""

    kind = "quadrotor"

    def __init__(self, type_id, batch, quad=None, rate=None, outer=None, motor_tau: float = 0.0):
        n = int(np.asarray(batch.agent_ids).shape[0])
        self.type_id = type_id
        self.n = n
        self.p = make_params(quad, rate, outer)
        self.agent_ids = np.array(batch.agent_ids, dtype=np.uint64)
        self.pos = np.array(batch.pos, dtype=float).reshape(n, 3).copy()
        self.vel = np.array(batch.vel, dtype=float).reshape(n, 3).copy()
        self.quat = np.array(batch.quat, dtype=float).reshape(n, 4).copy()
        self.omega = np.array(batch.omega, dtype=float).reshape(n, 3).copy()
        self.alive = np.array(batch.alive, dtype=np.uint8).reshape(n).copy()
        self.integral = np.zeros((n, 3))
        self.prev_omega = np.zeros((n, 3))
        self.has_prev = np.zeros(n, dtype=np.uint8)
        self.omega_sp = np.zeros((n, 3))
        self.f_c_sp = np.zeros(n)
        self.cmd_level = np.zeros(n, dtype=np.uint8)
        self.cmd_values = np.zeros((n, 7))
        self.cmd_values[:, :3] = self.pos
        self.cmd_values[:, 6] = quat_yaw(self.quat)
        self.v_overlay = np.zeros((n, 3))
        self.overlay_active = False
        self._row = {int(a): i for i, a in enumerate(self.agent_ids)}
        self.fault_mask = np.zeros(n, dtype=np.uint8)
        # opt-in rotor lag (parity unpinned: absent in the reference); rotor
        # thrusts start at the hover split m g / 4, like B200QuadGroup
        self.motor_tau = float(motor_tau)
        self.motor = np.full((n, 4), self.p.m * self.p.g / 4.0) if self.motor_tau > 0.0 else None

    def rows_for(self, agent_id):
        return self._row.get(int(agent_id))

    def apply_command(self, cmd) -> bool:
        row = self._row.get(int(cmd.agent_id))
        if row is None or not self.alive[row]:
            return False
        key = getattr(cmd.level, "value", cmd.level)
        lvl = _LEVELS.get(key)
        if lvl is None:
            return False
        vals = np.asarray(cmd.values, dtype=float)
        self.cmd_level[row] = lvl
        self.cmd_values[row, :] = 0.0
        self.cmd_values[row, :vals.shape[0]] = vals
        return True

    def add_velocity_overlay(self, offsets):
        self.v_overlay += offsets
        self.overlay_active = True

    def retarget_waypoint(self, point, radius):
        d = np.linalg.norm(self.pos - np.asarray(point, dtype=float), axis=1)
        rows = (d < radius) & self.alive.astype(bool)
        if rows.any():
            self.cmd_level[rows] = 0
            self.cmd_values[rows, :3] = point
            self.cmd_values[rows, 3:6] = 0.0
            self.cmd_values[rows, 6] = quat_yaw(self.quat[rows])

    def mark_dead(self, agent_ids):
        killed = []
        for aid in agent_ids:
            row = self._row.get(int(aid))
            if row is not None and self.alive[row]:
                self.alive[row] = 0
                killed.append(int(aid))
        return killed

    def step(self, dt: float, nthreads: int = 1) -> np.ndarray:
        ov = self.v_overlay if self.overlay_active else None
        args = (self.n, dt, ctypes.byref(self.p), _d(self.pos), _d(self.vel), _d(self.quat), _d(self.omega),
                _b(self.alive), _d(self.integral), _d(self.prev_omega), _b(self.has_prev), _d(self.omega_sp),
                _d(self.f_c_sp), _b(self.cmd_level), _d(self.cmd_values),
                _d(ov) if ov is not None else None, _b(self.fault_mask), int(nthreads))
        if self.motor is None:
            nf = load().oracle_group_step(*args)
        else:
            nf = load().oracle_group_step_lag(*args, _d(self.motor), self.motor_tau)
        if self.overlay_active:
            self.v_overlay[:] = 0.0
            self.overlay_active = False
        if nf == -2:
            raise ValueError("dt must be positive")
        if nf == -1:
            raise OracleInvalidState("non-finite quaternion input")
        return self.agent_ids[self.fault_mask.astype(bool)].copy()

    def state13(self) -> np.ndarray:
        return np.hstack([self.pos, self.vel, self.quat, self.omega])


def unicycle_step(pos, vel, quat, omega, alive, cmd, v_max, omega_max, dt):
    """float64 restatement of unicycle_step (core.py:221-246), in place."""
    alive = np.asarray(alive, dtype=bool)
    v = np.clip(cmd[:, 0], -v_max, v_max)
    w = np.clip(cmd[:, 1], -omega_max, omega_max)
    theta0 = quat_yaw(quat)
    theta1 = theta0 + w * dt
    straight = np.abs(w) <= 1e-9
    w_safe = np.where(straight, 1.0, w)
    dx = np.where(straight, v * np.cos(theta0) * dt, v / w_safe * (np.sin(theta1) - np.sin(theta0)))
    dy = np.where(straight, v * np.sin(theta0) * dt, -v / w_safe * (np.cos(theta1) - np.cos(theta0)))
    pos[alive, 0] += dx[alive]
    pos[alive, 1] += dy[alive]
    yq = np.zeros((theta1.shape[0], 4))
    yq[:, 0], yq[:, 3] = np.cos(0.5 * theta1), np.sin(0.5 * theta1)
    quat[alive] = yq[alive]
    vel[alive, 0] = (v * np.cos(theta1))[alive]
    vel[alive, 1] = (v * np.sin(theta1))[alive]
    vel[alive, 2] = 0.0
    omega[alive, 2] = w[alive]


class OracleUnicycleGroup:
    """float64 twin of UnicycleGroup (core.py:249-289)."""

    kind = "unicycle"

    def __init__(self, type_id, batch, v_max=5.0, omega_max=3.0):
        n = int(np.asarray(batch.agent_ids).shape[0])
        self.type_id, self.n = type_id, n
        self.v_max, self.omega_max = v_max, omega_max
        self.agent_ids = np.array(batch.agent_ids, dtype=np.uint64)
        self.pos = np.array(batch.pos, dtype=float).reshape(n, 3).copy()
        self.vel = np.array(batch.vel, dtype=float).reshape(n, 3).copy()
        self.quat = np.array(batch.quat, dtype=float).reshape(n, 4).copy()
        self.omega = np.array(batch.omega, dtype=float).reshape(n, 3).copy()
        self.alive = np.array(batch.alive, dtype=bool).reshape(n).copy()
        self.cmd = np.zeros((n, 2))
        self.v_overlay = np.zeros((n, 3))
        self.overlay_active = False
        self._row = {int(a): i for i, a in enumerate(self.agent_ids)}

    def apply_command(self, cmd) -> bool:
        row = self._row.get(int(cmd.agent_id))
        if row is None or not self.alive[row] or getattr(cmd.level, "value", cmd.level) != "unicycle":
            return False
        self.cmd[row] = cmd.values
        return True

    def add_velocity_overlay(self, offsets):
        self.v_overlay += offsets
        self.overlay_active = True

    def retarget_waypoint(self, point, radius):
        pass

    def mark_dead(self, agent_ids):
        killed = []
        for aid in agent_ids:
            row = self._row.get(int(aid))
            if row is not None and self.alive[row]:
                self.alive[row] = False
                killed.append(int(aid))
        return killed

    def step(self, dt):
        cmd = self.cmd
        if self.overlay_active:
            heading = quat_yaw(self.quat)
            along = self.v_overlay[:, 0] * np.cos(heading) + self.v_overlay[:, 1] * np.sin(heading)
            cmd = cmd.copy()
            cmd[:, 0] += along
            self.v_overlay[:] = 0.0
            self.overlay_active = False
        unicycle_step(self.pos, self.vel, self.quat, self.omega, self.alive, cmd, self.v_max, self.omega_max, dt)
        return np.empty(0, dtype=np.uint64)


def collide_all_pairs(ids, pos, radii, alive, r_sense: float):
    """All-pairs float64 collision / neighbour oracle (tests/oracles.py:79-102 and
    test_acceptance.py:141-156 restated): (sorted colliding id pairs, dict id ->
    sorted tuple of neighbour ids) over alive agents, strict inequalities."""
    ids, pos, radii, alive = (np.asarray(ids, dtype=np.int64), np.asarray(pos, dtype=float),
                              np.asarray(radii, dtype=float), np.asarray(alive, dtype=bool))
    ids, pos, radii = ids[alive], pos[alive], radii[alive]
    n = ids.shape[0]
    nbrs = {int(i): [] for i in ids}
    pairs = []
    if n >= 2:
        diff = pos[:, None, :] - pos[None, :, :]
        d2 = np.sum(diff * diff, axis=2)
        iu, ju = np.triu_indices(n, k=1)
        rsum = radii[iu] + radii[ju]
        hit = d2[iu, ju] < rsum * rsum
        for a, b in zip(iu[hit], ju[hit]):
            pairs.append((min(int(ids[a]), int(ids[b])), max(int(ids[a]), int(ids[b]))))
        near = d2[iu, ju] < r_sense * r_sense
        for a, b in zip(iu[near], ju[near]):
            nbrs[int(ids[a])].append(int(ids[b]))
            nbrs[int(ids[b])].append(int(ids[a]))
    return sorted(pairs), {k: tuple(sorted(v)) for k, v in nbrs.items()}


def neighbor_overlay(pos, alive, r_sense: float, k_sep: float, rows=None, chunk: int = 2048) -> np.ndarray:
    """All-pairs float64 separation overlay (SURVEY 8(e) controller; the
    wire.py:320-340 repel field applied per neighbour, strict < of
    collision.py:166, zero-distance guard of wire.py:335).  Returns (len(rows), 3)."""
    pos = np.asarray(pos, dtype=float)
    alive = np.asarray(alive, dtype=bool)
    rows = np.arange(pos.shape[0]) if rows is None else np.asarray(rows)
    out = np.zeros((rows.shape[0], 3))
    pa, ia = pos[alive], np.nonzero(alive)[0]
    for s in range(0, rows.shape[0], chunk):
        rr = rows[s:s + chunk]
        diff = pos[rr][:, None, :] - pa[None, :, :]
        d = np.sqrt(np.sum(diff * diff, axis=2))
        m = (d < r_sense) & (d > 1e-12) & (ia[None, :] != rr[:, None]) & alive[rr][:, None]
        w = np.where(m, k_sep * (1.0 - d / r_sense) / np.where(m, d, 1.0), 0.0)
        out[s:s + chunk] = np.einsum("ij,ijk->ik", w, diff)
    return out


def viewer_offsets(mode: str, point, radius: float, strength: float, pos, alive) -> np.ndarray:
    """viewer_velocity_offsets (wire.py:320-340) restated: (n, 3) float64
    attract / repel offsets, zero for WAYPOINT, radius <= 0, dead rows and
    rows outside 1e-12 < d < radius."""
    pos = np.asarray(pos, dtype=float)
    alive = np.asarray(alive, dtype=bool)
    out = np.zeros((pos.shape[0], 3))
    if mode == "waypoint" or not radius > 0.0:
        return out
    delta = np.asarray(point, dtype=float) - pos
    d = np.sqrt((delta[:, 0] * delta[:, 0] + delta[:, 1] * delta[:, 1]) + delta[:, 2] * delta[:, 2])
    inside = (d < radius) & (d > 1e-12) & alive
    sign = 1.0 if mode == "attract" else -1.0
    scale = sign * strength * (1.0 - d[inside] / radius) / d[inside]
    out[inside] = delta[inside] * scale[:, None]
    return out


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
