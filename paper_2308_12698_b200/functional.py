"""The reference's function-level hot-path API, computed by the sm_100a
kernels of csrc/ops.cu ("kernel-level functions").

Same names, arguments and return shapes as the reference's batched numpy
functions, so code and tests written against them switch over unchanged:

  dynamics_deriv(batch, f_c, tau, params)               quad.py:320-335
  rk4_step(batch, f_c, tau, params, dt)  -> fault ids   quad.py:350-437
  mix_to_motors(f_c, tau, params)        -> MixResult   quad.py:143-168
  rotor_thrust_torque(omega_rpm, params)                quad.py:130-140
  rate_pid_step(omega, sp, gains, dt, state, alive)     control.py:136-187
  position_outer_loop(pos, vel, quat, alive, sp, params, gains)
                                         -> OuterResult control.py:222-294

Host (numpy) arguments are copied to the device, computed in float32 on the
GPU and returned as float64 numpy arrays (positions travel as float32 hi +
lo, like the group's columns); CUDA tensors stay on the device and come back
as float32 tensors (mix / pid / outer).  Errors follow the reference:
``ValidationError`` for dt <= 0, ``InvalidStateError`` for a non-finite
outer-loop input (quat.py:84).  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import InvalidStateError, NativeLibraryError, ValidationError
from .params import default_outer_gains, default_quad_params, default_rate_gains, pack_device_params

__all__ = ["StateCols", "MixResult", "RateSetpoint", "PosSetpoint", "OuterResult", "RatePidState",
           "dynamics_deriv", "rk4_step", "mix_to_motors", "rotor_thrust_torque", "rate_pid_step",
           "position_outer_loop"]


@dataclass
class StateCols:
    """Per-quantity derivative / state columns (quad.py _StateCols)."""

    pos: np.ndarray
    vel: np.ndarray
    quat: np.ndarray
    omega: np.ndarray


@dataclass(frozen=True)
class MixResult:
    """Mixer output (quad.py:96-103)."""

    motors: object
    f_c: object
    tau: object
    saturated: object


@dataclass(frozen=True)
class PosSetpoint:
    """Position-level reference (control.py:83-89)."""

    p_sp: object
    v_sp: object
    yaw_sp: object


@dataclass(frozen=True)
class RateSetpoint:
    """Inner-loop reference (control.py:92-97)."""

    omega_sp: object
    f_c_sp: object


@dataclass(frozen=True)
class OuterResult:
    """position_outer_loop output (control.py:216-219)."""

    setpoint: RateSetpoint
    low_thrust: object


class RatePidState:
    """Integral / previous-measurement columns (control.py:100-114)."""

    def __init__(self, n: int) -> None:
        self.integral = np.zeros((n, 3))
        self.prev_omega = np.zeros((n, 3))
        self.has_prev = np.zeros(n, dtype=bool)

    def reset(self, rows=None) -> None:
        if rows is None:
            self.integral[:] = 0.0
            self.has_prev[:] = False
        else:
            self.integral[rows] = 0.0
            self.has_prev[rows] = False


# ----------------------------------------------------------------- plumbing
def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeLibraryError("the function-level API runs on the GPU (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_F32_MAX = float(np.finfo(np.float32).max)


def _p(t: torch.Tensor | None):
    # callers keep every tensor passed here in a local until the launch is
    # queued: a temporary freed inside the argument list would hand its memory
    # to the next allocation of the same call
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _f32(x, shape, dev) -> torch.Tensor:
    """A contiguous float32 device tensor of ``shape`` holding x."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=torch.float32)
    else:
        a = np.asarray(x)
        if a.dtype != np.float32:
            # finite values beyond float32 range saturate (like the group's
            # command store) instead of becoming inf
            a = np.asarray(a, dtype=np.float64)
            fin = np.isfinite(a)
            if not fin.all() or np.abs(a).max(initial=0.0) > _F32_MAX:
                a = np.where(fin, np.clip(a, -_F32_MAX, _F32_MAX), a)
        t = torch.from_numpy(np.array(np.broadcast_to(a.astype(np.float32), shape))).to(dev)
    return t.reshape(shape).contiguous()


def _u8(x, n, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.uint8).reshape(n).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=bool).reshape(n), dtype=np.uint8)).to(dev)


def _hi_lo(x, shape, dev):
    """float64 host positions as float32 hi + lo device tensors."""
    a = np.asarray(x, dtype=np.float64).reshape(shape)
    hi = a.astype(np.float32)
    lo = (a - hi.astype(np.float64)).astype(np.float32)
    return torch.from_numpy(hi).to(dev), torch.from_numpy(lo).to(dev)


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.float64)


def _params(params=None, rate_gains=None, outer_gains=None):
    return pack_device_params(params if params is not None else default_quad_params(),
                              rate_gains if rate_gains is not None else default_rate_gains(),
                              outer_gains if outer_gains is not None else default_outer_gains())


def _check(code: int) -> None:
    _lib.check(code)


# --------------------------------------------------------------- functions
def dynamics_deriv(batch, f_c, tau, params=None, workspace=None, out=None) -> StateCols:
    """State derivative of every alive agent; dead rows get exactly zero."""
    lib, dev = _lib.load(), _device()
    n = int(batch.pos.shape[0])
    P = _params(params)
    ins = [_f32(batch.pos, (n, 3), dev), _f32(batch.vel, (n, 3), dev), _f32(batch.quat, (n, 4), dev),
           _f32(batch.omega, (n, 3), dev)]
    alive = _u8(batch.alive, n, dev)
    fc, tq = _f32(f_c, (n,), dev), _f32(tau, (n, 3), dev)
    outs = [torch.empty((n, 3), device=dev), torch.empty((n, 3), device=dev), torch.empty((n, 4), device=dev),
            torch.empty((n, 3), device=dev)]
    _check(lib.swarmstep_op_deriv(n, *[_p(t) for t in ins], _p(alive), _p(fc), _p(tq), ctypes.byref(P),
                                  *[_p(t) for t in outs], _stream()))
    res = StateCols(*[_host(t) for t in outs])
    if out is not None:
        for name in ("pos", "vel", "quat", "omega"):
            getattr(out, name)[:n] = getattr(res, name)
        return out
    return res


def rk4_step(batch, f_c, tau, params, dt: float, workspace=None) -> np.ndarray:
    """One RK4 step in place on the batch's float64 arrays (wrench held);
    returns the ids of rows that faulted (reverted, marked dead)."""
    if not dt > 0.0:
        raise ValidationError(f"dt must be positive, got {dt}")
    lib, dev = _lib.load(), _device()
    n = int(batch.pos.shape[0])
    P = _params(params)
    hi, lo = _hi_lo(batch.pos, (n, 3), dev)
    vel, quat, om = _f32(batch.vel, (n, 3), dev), _f32(batch.quat, (n, 4), dev), _f32(batch.omega, (n, 3), dev)
    alive = _u8(batch.alive, n, dev)
    fault = torch.empty(n, dtype=torch.uint8, device=dev)
    fc, tq = _f32(f_c, (n,), dev), _f32(tau, (n, 3), dev)
    _check(lib.swarmstep_op_rk4(n, _p(hi), _p(lo), _p(vel), _p(quat), _p(om), _p(alive), _p(fc), _p(tq),
                                ctypes.byref(P), ctypes.c_float(dt), _p(fault), _stream()))
    f = fault.cpu().numpy().astype(bool)
    live = np.asarray(batch.alive, dtype=bool) & ~f
    pos = hi.cpu().numpy().astype(np.float64) + lo.cpu().numpy().astype(np.float64)
    for name, val in (("pos", pos), ("vel", _host(vel)), ("quat", _host(quat)), ("omega", _host(om))):
        arr = getattr(batch, name)
        arr[live] = val[live]
    if f.any():
        batch.alive[f] = False
        return np.asarray(batch.agent_ids)[f].astype(np.uint64)
    return np.empty(0, dtype=np.uint64)


def mix_to_motors(f_c, tau, params, workspace=None) -> MixResult:
    """Clamped motor thrusts and the wrench they realise (quad.py:143-168)."""
    lib, dev = _lib.load(), _device()
    as_torch = isinstance(f_c, torch.Tensor)
    n = int(f_c.numel()) if as_torch else int(np.atleast_1d(np.asarray(f_c)).shape[0])
    fc = _f32(f_c if as_torch else np.atleast_1d(np.asarray(f_c, float)), (n,), dev)
    tq = _f32(tau, (n, 3), dev)
    motors, realized = torch.empty((n, 4), device=dev), torch.empty((n, 4), device=dev)
    sat = torch.empty(n, dtype=torch.uint8, device=dev)
    _check(lib.swarmstep_op_mix(n, _p(fc), _p(tq), ctypes.byref(_params(params)), _p(motors), _p(realized),
                                _p(sat), _stream()))
    if as_torch:
        return MixResult(motors=motors, f_c=realized[:, 0], tau=realized[:, 1:], saturated=sat.bool())
    r = _host(realized)
    return MixResult(motors=_host(motors), f_c=r[:, 0].copy(), tau=r[:, 1:].copy(),
                     saturated=sat.cpu().numpy().astype(bool))


def rotor_thrust_torque(omega_rpm, params):
    """Quadratic rotor fit with clamped speeds: (thrust, torque, saturated)."""
    lib, dev = _lib.load(), _device()
    o = np.asarray(omega_rpm, dtype=float)
    x = _f32(o, o.shape, dev).reshape(-1)
    k = int(x.numel())
    th, tq = torch.empty(k, device=dev), torch.empty(k, device=dev)
    sat = torch.empty(k, dtype=torch.uint8, device=dev)
    _check(lib.swarmstep_op_rotor(k, _p(x), ctypes.c_float(params.k_t), ctypes.c_float(params.k_q),
                                  ctypes.c_float(params.omega_max), _p(th), _p(tq), _p(sat), _stream()))
    return (_host(th).reshape(o.shape), _host(tq).reshape(o.shape),
            sat.cpu().numpy().astype(bool).reshape(o.shape))


def rate_pid_step(omega, sp, gains, dt: float, state, alive, workspace=None, tau_out=None, f_c_out=None):
    """Body-rate PID over a batch; updates ``state`` in place; returns (f_c, tau)."""
    if not dt > 0.0:
        raise ValidationError(f"dt must be positive, got {dt}")
    lib, dev = _lib.load(), _device()
    as_torch = isinstance(omega, torch.Tensor)
    n = int(omega.shape[0])
    P = _params(rate_gains=gains)
    om, osp, fsp = _f32(omega, (n, 3), dev), _f32(sp.omega_sp, (n, 3), dev), _f32(sp.f_c_sp, (n,), dev)
    integ, prev = _f32(state.integral, (n, 3), dev), _f32(state.prev_omega, (n, 3), dev)
    hp, al = _u8(state.has_prev, n, dev), _u8(alive, n, dev)
    tau, fc = torch.empty((n, 3), device=dev), torch.empty(n, device=dev)
    _check(lib.swarmstep_op_pid(n, _p(om), _p(osp), _p(fsp), ctypes.byref(P), ctypes.c_float(dt), _p(integ),
                                _p(prev), _p(hp), _p(al), _p(tau), _p(fc), _stream()))
    if isinstance(state.integral, torch.Tensor):
        state.integral.copy_(integ)
        state.prev_omega.copy_(prev)
        state.has_prev.copy_(hp.bool())
    else:
        state.integral[:] = _host(integ)
        state.prev_omega[:] = _host(prev)
        state.has_prev[:] = hp.cpu().numpy().astype(bool)
    if as_torch:
        return fc, tau
    f, t = _host(fc), _host(tau)
    if tau_out is not None:
        tau_out[:] = t
        t = tau_out
    if f_c_out is not None:
        f_c_out[:] = f
        f = f_c_out
    return f, t


def position_outer_loop(pos, vel, quat, alive, sp, params, gains) -> OuterResult:
    """PD position loop -> desired attitude -> body-rate setpoints."""
    lib, dev = _lib.load(), _device()
    as_torch = isinstance(pos, torch.Tensor)
    n = int(pos.shape[0])
    yaw = sp.yaw_sp
    if as_torch:
        ins = [pos, vel, quat, sp.p_sp, sp.v_sp]
        finite = all(bool(torch.isfinite(t).all()) for t in ins) and bool(torch.isfinite(torch.as_tensor(yaw)).all())
        p_hi, p_lo = _f32(pos, (n, 3), dev), None
    else:
        ins = [pos, vel, quat, sp.p_sp, sp.v_sp, yaw]
        finite = all(np.all(np.isfinite(np.asarray(x, dtype=float))) for x in ins)
        p_hi, p_lo = _hi_lo(pos, (n, 3), dev)
    if not finite:
        # the reference's quat_mul raises before returning anything (quat.py:84)
        raise InvalidStateError("non-finite quaternion input")
    P = _params(params, outer_gains=gains)
    w_sp, f_sp = torch.empty((n, 3), device=dev), torch.empty(n, device=dev)
    low = torch.empty(n, dtype=torch.uint8, device=dev)
    v, q, al = _f32(vel, (n, 3), dev), _f32(quat, (n, 4), dev), _u8(alive, n, dev)
    if as_torch:
        ps, vs, ys = _f32(sp.p_sp, (n, 3), dev), _f32(sp.v_sp, (n, 3), dev), _f32(yaw, (n,), dev)
    else:
        # the group's float32 command conversion (yaw reduced to [-pi, pi],
        # setpoints beyond float32 range scaled: group.f32_commands)
        from .group import f32_commands
        cmd = np.empty((n, 7))
        cmd[:, 0:3] = np.broadcast_to(np.asarray(sp.p_sp, dtype=np.float64), (n, 3))
        cmd[:, 3:6] = np.broadcast_to(np.asarray(sp.v_sp, dtype=np.float64), (n, 3))
        cmd[:, 6] = np.broadcast_to(np.asarray(yaw, dtype=np.float64), (n,))
        c32 = f32_commands(cmd, np.ones(n, dtype=bool))
        ps, vs, ys = (_f32(np.ascontiguousarray(c32[:, 0:3]), (n, 3), dev),
                      _f32(np.ascontiguousarray(c32[:, 3:6]), (n, 3), dev), _f32(c32[:, 6].copy(), (n,), dev))
    _check(lib.swarmstep_op_outer(n, _p(p_hi), _p(p_lo), _p(v), _p(q), _p(al), _p(ps), _p(vs), _p(ys),
                                  ctypes.byref(P), _p(w_sp), _p(f_sp), _p(low), _stream()))
    if as_torch:
        return OuterResult(setpoint=RateSetpoint(omega_sp=w_sp, f_c_sp=f_sp), low_thrust=low.bool())
    return OuterResult(setpoint=RateSetpoint(omega_sp=_host(w_sp), f_c_sp=_host(f_sp)),
                       low_thrust=low.cpu().numpy().astype(bool))
