"""Synthetic swarms for the benchmark (the reference bench's recipe, sliceable).

The reference bench builds its world with ``layout_poses`` on a grid (spacing
3 m, origin (0, 0, 10); bench.py:87-93 of the reference, config.py:147-179).
SURVEY.md 8(d) cfg3/cfg4 put every agent at POSITION level with random
setpoints p_sp = p0 + U(-1, 1)^3, v_sp = 0, yaw_sp = U(-pi, pi).

Everything here is a pure function of (n_total, row range), so any shard of
the same N-agent swarm -- a rank of a multi-GPU run, a host process of the
CPU reference arm -- builds exactly its own rows of one fixed workload: the
random draws come in blocks of ``BLOCK`` agents, each from its own seeded
generator, and positions follow the grid formula of ``layout_poses`` for the
whole swarm.  Setpoints are float32 values (the device command columns); the
float64 reference receives the same values widened exactly.
"""

from __future__ import annotations

import numpy as np

BLOCK = 1 << 16
SPACING = 3.0
ORIGIN = (0.0, 0.0, 10.0)


def grid_positions(n_total: int, lo: int, hi: int) -> np.ndarray:
    """Rows [lo, hi) of layout_poses({"kind": "grid", "spacing": 3, "origin": (0,0,10)}, n_total)."""
    cols = max(1, int(np.ceil(np.sqrt(max(n_total, 1)))))
    idx = np.arange(lo, hi)
    pos = np.stack([(idx % cols) * SPACING, (idx // cols) * SPACING, np.zeros(hi - lo)], axis=1)
    pos += np.asarray(ORIGIN)
    return pos


def _draws(lo: int, hi: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """U(-1,1)^3 offsets and U(-pi,pi) yaws of rows [lo, hi), blockwise seeded."""
    off = np.empty((hi - lo, 3))
    yaw = np.empty(hi - lo)
    b0, b1 = lo // BLOCK, (hi + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        rng = np.random.default_rng([seed, b])
        o = rng.uniform(-1.0, 1.0, (BLOCK, 3))
        y = rng.uniform(-np.pi, np.pi, BLOCK)
        s, e = max(lo, b * BLOCK), min(hi, (b + 1) * BLOCK)
        off[s - lo:e - lo] = o[s - b * BLOCK:e - b * BLOCK]
        yaw[s - lo:e - lo] = y[s - b * BLOCK:e - b * BLOCK]
    return off, yaw


def pos_setpoints(n_total: int, lo: int, hi: int, seed: int = 0, pos: np.ndarray | None = None) -> np.ndarray:
    """(7, hi - lo) float32 POS command columns: p_sp = p0 + U(-1,1)^3, v_sp = 0, yaw U(-pi, pi)."""
    if pos is None:
        pos = grid_positions(n_total, lo, hi)
    off, yaw = _draws(lo, hi, seed)
    sp = np.zeros((7, hi - lo), dtype=np.float32)
    sp[0:3] = (pos + off).T
    sp[6] = yaw
    return sp


def swarm(n_total: int, lo: int = 0, hi: int | None = None, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Initial positions (hi-lo, 3) float64 and POS setpoints (7, hi-lo) float32
    of rows [lo, hi) of the n_total-agent bench swarm (at rest, identity attitude)."""
    hi = n_total if hi is None else hi
    if not 0 <= lo <= hi <= n_total:
        raise ValueError("bad row range")
    pos = grid_positions(n_total, lo, hi)
    return pos, pos_setpoints(n_total, lo, hi, seed, pos)
