"""Shared helpers for the GPU parity tests (CUDA float32 path vs float64 oracle)."""

from __future__ import annotations

import numpy as np

from oracle import oracle as orc

# Per-step parity metric (north_star: per-step relative error <= 1e-5 in FP32).
# err_q = max |x32 - x64| / max(|x64|_inf(row), floor_q), per quantity q, taken
# over all rows after ONE step from an identical (float32-representable) state.
# The floors are SURVEY.md 8(c)'s per-quantity absolute floors (s_pos = 1 m,
# s_vel = 0.1 m/s, s_quat = 1, s_omega = 1e-3 rad/s, s_I = 1e-3): below them
# a component counts as near zero and the error is taken against the floor.
PER_STEP_TOL = 1e-5
FLOORS = dict(pos=1.0, vel=0.1, quat=1.0, omega=1e-3, integral=1e-3)


def make_group(sc_or_arrays, compensated=True, **kw):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    s = sc_or_arrays
    b = batch_create(0, s.n, s.pos, quat=s.quat, vel=s.vel, omega=s.omega)
    return B200QuadGroup(0, b, compensated=compensated, **kw)


def gpu_state(g) -> dict:
    b = g.batch
    ps = g.pid_state_dict()
    return dict(pos=b.pos.copy(), vel=b.vel.copy(), quat=b.quat.copy(), omega=b.omega.copy(),
                alive=b.alive.copy(), integral=ps["integral"], prev_omega=ps["prev_omega"],
                has_prev=ps["has_prev"], omega_sp=ps["omega_sp"], f_c_sp=ps["f_c_sp"],
                cmd_level=g.cmd_level.copy(), cmd_values=g.cmd_values.copy())


class _Batch:
    def __init__(self, st):
        n = st["pos"].shape[0]
        self.agent_ids = np.arange(n, dtype=np.uint64)
        self.pos, self.vel, self.quat, self.omega = st["pos"], st["vel"], st["quat"], st["omega"]
        self.alive = st["alive"]


def oracle_twin(g, st=None, params=None) -> orc.OracleGroup:
    """float64 oracle group holding exactly the GPU group's current (float32) state
    (``params``: the (QuadParams, PidGains, OuterGains) the group was built with)."""
    st = st or gpu_state(g)
    og = orc.OracleGroup(0, _Batch(st), *(params or ()))
    og.integral[:] = st["integral"]
    og.prev_omega[:] = st["prev_omega"]
    og.has_prev[:] = st["has_prev"].astype(np.uint8)
    og.omega_sp[:] = st["omega_sp"]
    og.f_c_sp[:] = st["f_c_sp"]
    og.cmd_level[:] = st["cmd_level"]
    og.cmd_values[:] = st["cmd_values"].astype(np.float32).astype(np.float64)
    return og


def rel_errors(gst: dict, og: orc.OracleGroup, rows=None) -> dict:
    rows = slice(None) if rows is None else rows
    alive = og.alive.astype(bool)[rows]
    out = {}
    for q, want in (("pos", og.pos), ("vel", og.vel), ("quat", og.quat), ("omega", og.omega),
                    ("integral", og.integral)):
        w = want[rows][alive]
        h = gst[q][rows][alive]
        if w.size == 0:
            out[q] = 0.0
            continue
        scale = np.maximum(np.max(np.abs(w), axis=1, keepdims=True), FLOORS[q])
        out[q] = float(np.max(np.abs(h - w) / scale))
    return out


def f32(dt: float) -> float:
    return float(np.float32(dt))


# K fused ticks vs K one-tick launches.  Everything in a tick is the same
# arithmetic either way; the compensated position differs only in where its
# low part is folded and rounded: a fused launch carries the position
# increments in a launch-local accumulator and folds it into (hi, lo) once,
# a one-tick launch folds every tick, and the stored low part is rounded to
# ulp(hi)/512 at every launch boundary (include/swarmstep_b200.h COL_POS_LO).
# Without compensation the two are bit-identical (asserted separately).  The
# position difference (<= ulp(p)/1024 per launch boundary) reaches the rates
# through the cascade's gains, so the bound is the per-step parity bar (the
# 200-swarm soak, profiles/fuzz_soak_r02.txt, sees up to 2e-6 near the
# 1e-3 rad/s rate floor and ~1e-8 elsewhere).
FUSION_TOL = PER_STEP_TOL
FUSION_FLOORS = dict(FLOORS, prev_omega=1e-3, omega_sp=1e-3, f_c_sp=1e-3)


def fusion_errors(a: dict, b: dict, keys) -> dict:
    """Per-quantity, per-row |a - b| / max(|a|_row, floor) (the rel_errors metric)."""
    out = {}
    for q in keys:
        x, y = np.asarray(a[q], dtype=np.float64), np.asarray(b[q], dtype=np.float64)
        if x.ndim == 1:
            x, y = x[:, None], y[:, None]
        scale = np.maximum(np.max(np.abs(x), axis=1, keepdims=True), FUSION_FLOORS.get(q, 1.0))
        d = np.abs(x - y)
        d[np.isnan(x) & np.isnan(y)] = 0.0
        out[q] = np.max(d / scale, axis=1) if d.size else np.zeros(0)
    return out


# Two valid float32 evaluations of the reference's control law can part ways
# near its discontinuities (the free-fall floor control.py:243-247, the mixer
# clamp, the degenerate heading): a 2000-swarm soak (profiles/fuzz_soak_r02.txt)
# has 2 of 1000 swarms with one row near one of them, at up to 1.6e-4.  So at
# most 1 % of the rows (at least one) may exceed the bar, none by more than HARD.
FUSION_HARD = 1e-3


def assert_fusion_close(a: dict, b: dict, keys, tol: float = FUSION_TOL):
    err = fusion_errors(a, b, keys)
    rows = np.max(np.stack([v for v in err.values()]), axis=0) if err else np.zeros(0)
    n_bad = int(np.count_nonzero(~(rows <= tol)))
    allowed = max(1, int(0.01 * rows.size))
    worst = {k: float(np.max(v)) if v.size else 0.0 for k, v in err.items()}
    assert n_bad <= allowed, f"fused vs one-tick launches: {n_bad} rows beyond {tol} (allowed {allowed}): {worst}"
    assert not rows.size or float(np.max(rows)) <= FUSION_HARD, f"fused vs one-tick launches beyond {FUSION_HARD}: {worst}"
