"""GPU sphere-collision and neighbour detection over device-resident groups
(the reference's collision.py).

``detect(groups, config, tick)`` returns the reference's ``CollisionReport``
(collision.py:49-56) for the alive agents of the given B200 groups: all
colliding pairs (``|p_a - p_b| < r_a + r_b``, strict, cross-type included)
and per-agent neighbour sets (strictly within ``r_sense``).  The grid broad
phase and the float64 narrow phase run on the GPU (csrc/collision.cu) with
the reference's arithmetic, so on the same float64 positions the report is
identical to ``swarmstep.collision.detect``; the host only sorts the pair
lists as collision.py:160-175 does.
"""

from __future__ import annotations

import ctypes
import math
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ValidationError


@dataclass(frozen=True)
class CollisionConfig:
    """Per-type collision radii, one sensing radius, and the grid cell size (collision.py:30-46)."""

    r_collide: Mapping[int, float]
    r_sense: float
    cell: float

    def __post_init__(self):
        if not self.r_collide:
            raise ValidationError("r_collide must name at least one agent type")
        rmax = max(self.r_collide.values())
        for tid, r in self.r_collide.items():
            if not 0.0 < r <= self.r_sense:
                raise ValidationError(f"type {tid}: need 0 < r_collide <= r_sense, got {r}")
        if self.cell < 2.0 * rmax:
            raise ValidationError(f"cell size {self.cell} must be >= 2 * max collision radius {2 * rmax}")


@dataclass(frozen=True)
class CollisionReport:
    """Tick-tagged collision pairs and neighbour sets over alive agents (collision.py:49-56)."""

    tick: int
    collisions: tuple = ()
    neighbor_sets: dict = field(default_factory=dict)
    dropped: int = 0


class NeighborSets(Mapping):
    """The report's ``neighbor_sets`` (agent id -> sorted tuple of neighbour
    ids, collision.py:168-175), built from the device pair list on first
    access: an in-loop caller that only needs ``collisions`` (core.py:495-498)
    never pays for the per-agent Python dict.  Compares equal to the plain
    dict the reference returns."""

    def __init__(self, alive_all: np.ndarray, ids_all: np.ndarray, near, n_alive: int | None = None):
        # near: (k, 2) row pairs, numpy or a device tensor (copied on first use)
        self._alive_all, self._ids_all, self._near = alive_all, ids_all, near
        self._n = int(alive_all.sum()) if n_alive is None else int(n_alive)
        self._d = None

    def _dict(self) -> dict:
        if self._d is None:
            ids_all, alive = self._ids_all, self._alive_all
            m = int(ids_all.shape[0])
            rows = np.nonzero(alive)[0]
            near = self._near
            k = (near.numel() // 2) if isinstance(near, torch.Tensor) else int(np.asarray(near).shape[0])
            if k == 0:
                self._d = dict.fromkeys(ids_all[rows].tolist(), ())
                return self._d
            # both directions of every pair, ordered by (row a, id b) through one
            # sort of int64 keys row_a * m + rank(id_b) (on the device when the
            # pairs are there); then one slice of the sorted id list per agent
            by_id = np.argsort(ids_all, kind="stable")
            rank = np.empty(m, dtype=np.int64)
            rank[by_id] = np.arange(m, dtype=np.int64)
            if isinstance(near, torch.Tensor):
                nr = near.reshape(-1, 2).long()
                na, nb = torch.cat([nr[:, 0], nr[:, 1]]), torch.cat([nr[:, 1], nr[:, 0]])
                key = na * m + torch.from_numpy(rank).to(near.device)[nb]
                key = torch.sort(key).values.cpu().numpy()
            else:
                nr = np.asarray(near, dtype=np.int64).reshape(-1, 2)
                na, nb = np.concatenate([nr[:, 0], nr[:, 1]]), np.concatenate([nr[:, 1], nr[:, 0]])
                key = np.sort(na * m + rank[nb])
            row_a = key // m
            nb_ids = ids_all[by_id[key - row_a * m]].tolist()
            offs = np.searchsorted(row_a, np.arange(m + 1)).tolist()
            self._d = {i: tuple(nb_ids[offs[r]:offs[r + 1]]) for r, i in zip(rows.tolist(), ids_all[rows].tolist())}
        return self._d

    def __getitem__(self, key):
        return self._dict()[key]

    def __iter__(self):
        return iter(self._dict())

    def __len__(self) -> int:
        return self._n

    def __repr__(self) -> str:
        return repr(self._dict())


def half_space_offsets(d_max: int, reach: float, cell: float) -> np.ndarray:
    """Cell offsets o > (0,0,0) lexicographically whose closest corners can be
    within ``reach`` (collision.py:86-95)."""
    rng = np.arange(-d_max, d_max + 1)
    grid = np.stack(np.meshgrid(rng, rng, rng, indexing="ij"), axis=-1).reshape(-1, 3)
    k0, k1, k2 = grid[:, 0], grid[:, 1], grid[:, 2]
    lex_positive = (k0 > 0) | ((k0 == 0) & ((k1 > 0) | ((k1 == 0) & (k2 > 0))))
    min_sep = np.maximum(np.abs(grid) - 1, 0) * cell
    reachable = np.sum(min_sep * min_sep, axis=1) < reach * reach
    return grid[lex_positive & reachable]


class GpuDetector:
    """Reusable device buffers for ``detect`` on one device."""

    def __init__(self, config: CollisionConfig, device=None):
        self.config = config
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._lib = _lib.load()
        self._counts = torch.zeros(4, dtype=torch.int64, device=self.device)
        self._ids_key, self._ids_all, self._n_alive = None, None, 0
        self._offs_key, self._offs, self._offs_d = None, None, None

    def detect(self, groups, tick: int, dropped: int = 0) -> CollisionReport:
        ids_all, alive_all, coll_h, near_h = self.pairs(groups)
        if coll_h is None:
            return CollisionReport(tick=tick, collisions=(), neighbor_sets={int(i): () for i in ids_all[alive_all]},
                                   dropped=dropped)
        # host post-processing exactly as collision.py:160-175
        src, dst = coll_h[:, 0], coll_h[:, 1]
        ids_a = np.minimum(ids_all[src], ids_all[dst])
        ids_b = np.maximum(ids_all[src], ids_all[dst])
        order = np.lexsort((ids_b, ids_a))
        collisions = tuple(zip(ids_a[order].tolist(), ids_b[order].tolist()))
        return CollisionReport(tick=tick, collisions=collisions,
                               neighbor_sets=NeighborSets(alive_all, ids_all, near_h, self._n_alive), dropped=dropped)

    def pairs(self, groups):
        """Device broad + narrow phase: (ids_all, alive_all, colliding row
        pairs (k, 2) numpy, neighbour row pairs (k, 2) as a device int32
        tensor) -- rows index ids_all; None when fewer than two agents are
        alive.  Only the collision pairs cross PCIe here; the (large)
        neighbour list is copied when the report's neighbor_sets is read."""
        cfg = self.config
        groups = sorted(groups, key=lambda g: g.type_id)
        for g in groups:
            if g.type_id not in cfg.r_collide:
                raise ValidationError(f"no collision radius configured for type {g.type_id}")
            if g.device != self.device:
                raise ValidationError("all groups must live on the detector's device")
        # host alive flags / ids without pulling the float64 state mirror: the
        # device rows carry the same alive flags (dead rows are packed with
        # a NaN radius and never paired)
        alive = [g.alive_mask() for g in groups]
        key = tuple(id(g) for g in groups)
        if self._ids_key != key:                 # ids are static per group: concatenate once
            self._ids_key = key
            self._ids_all = (np.concatenate([g.agent_ids.astype(np.int64) for g in groups]) if groups
                             else np.empty(0, np.int64))
        ids_all = self._ids_all
        alive_all = np.concatenate(alive) if groups else np.empty(0, bool)
        counts_alive = [g.alive_count() for g in groups]
        self._n_alive = sum(counts_alive)
        if self._n_alive < 2:
            return ids_all, alive_all, None, None
        rmax = max(cfg.r_collide[g.type_id] for g, c in zip(groups, counts_alive) if c)
        m = int(ids_all.shape[0])
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            xyzr = torch.empty((m, 4), dtype=torch.float64, device=self.device)
            off = 0
            for g in groups:
                g.stream.synchronize()   # positions of the group's last step
                _lib.check(self._lib.swarmstep_pack_collision(g._view_ref, float(cfg.r_collide[g.type_id]),
                                                              xyzr.data_ptr(), off, ctypes.c_void_p(stream.cuda_stream)))
                off += g.n
        coll_h, near = self._pairs_xyzr(xyzr, float(rmax))
        return ids_all, alive_all, coll_h, near

    def _pairs_xyzr(self, xyzr: torch.Tensor, rmax: float):
        """Broad + narrow phase over packed (m, 4) float64 rows (x, y, z, radius;
        NaN radius = dead): (colliding row pairs numpy, neighbour row pairs device)."""
        cfg = self.config
        reach = max(cfg.r_sense, 2.0 * rmax)
        d_max = int(math.ceil(reach / cfg.cell))
        okey = (d_max, reach, cfg.cell)
        if self._offs_key != okey:
            self._offs_key = okey
            self._offs = half_space_offsets(d_max, reach, cfg.cell).astype(np.int32)
            self._offs_d = (torch.from_numpy(self._offs.reshape(-1)).to(self.device) if self._offs.size
                            else torch.zeros(3, dtype=torch.int32, device=self.device))
        offs, offs_d = self._offs, self._offs_d
        m = int(xyzr.shape[0])
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            nbytes = ctypes.c_uint64()
            _lib.check(self._lib.swarmstep_collision_workspace_bytes(m, ctypes.byref(nbytes)))
            ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)

            def run(coll, cc, near, nc, fill):
                _lib.check(self._lib.swarmstep_collision_pairs(
                    xyzr.data_ptr(), m, float(cfg.cell), offs_d.data_ptr(), int(offs.shape[0]), float(cfg.r_sense),
                    coll, cc, near, nc, self._counts.data_ptr(), ws.data_ptr(), nbytes.value, fill,
                    ctypes.c_void_p(stream.cuda_stream)))
                return self._counts.cpu().numpy()

            counts = run(None, 0, None, 0, 0)
            if counts[2]:
                raise ValidationError("world extent exceeds the supported grid range")
            n_coll, n_near = int(counts[0]), int(counts[1])
            coll = torch.empty(max(2 * n_coll, 2), dtype=torch.int32, device=self.device)
            near = torch.empty(max(2 * n_near, 2), dtype=torch.int32, device=self.device)
            if n_coll or n_near:
                run(coll.data_ptr(), n_coll, near.data_ptr(), n_near, 1)
            coll_h = coll[:2 * n_coll].cpu().numpy().astype(np.int64).reshape(-1, 2)
        return coll_h, near[:2 * n_near]

    def detect_snapshot(self, snapshot, dropped: int = 0) -> CollisionReport:
        """``swarmstep.collision.detect(snapshot, config, dropped)``
        (collision.py:110-176) on the GPU for a host ``WorldSnapshot`` of any
        groups (the out-of-loop detector's input): same validation, same
        report.  The float64 positions are uploaded as they are."""
        cfg = self.config
        ids, pos, rad, alive = [], [], [], []
        for b in snapshot.batches:                    # collision.py:66-80
            if b.tick != snapshot.tick:
                raise ValidationError("snapshot sections disagree on tick")
            if b.type_id not in cfg.r_collide:
                raise ValidationError(f"no collision radius configured for type {b.type_id}")
            ids.append(np.asarray(b.agent_ids).astype(np.int64))
            pos.append(np.asarray(b.pos, dtype=np.float64).reshape(-1, 3))
            live = np.asarray(b.alive, dtype=bool)
            alive.append(live)
            rad.append(np.where(live, float(cfg.r_collide[b.type_id]), np.nan))
        ids_all = np.concatenate(ids) if ids else np.empty(0, np.int64)
        alive_all = np.concatenate(alive) if alive else np.empty(0, bool)
        n_alive = int(alive_all.sum())
        if n_alive < 2:
            return CollisionReport(tick=snapshot.tick, collisions=(),
                                   neighbor_sets={int(i): () for i in ids_all[alive_all]}, dropped=dropped)
        rmax = max(float(cfg.r_collide[b.type_id]) for b, a in zip(snapshot.batches, alive) if a.any())
        host = np.empty((ids_all.shape[0], 4))
        host[:, :3] = np.concatenate(pos)
        host[:, 3] = np.concatenate(rad)
        xyzr = torch.from_numpy(host).to(self.device)
        coll_h, near = self._pairs_xyzr(xyzr, rmax)
        self._n_alive = n_alive
        src, dst = coll_h[:, 0], coll_h[:, 1]
        ids_a = np.minimum(ids_all[src], ids_all[dst])
        ids_b = np.maximum(ids_all[src], ids_all[dst])
        order = np.lexsort((ids_b, ids_a))
        collisions = tuple(zip(ids_a[order].tolist(), ids_b[order].tolist()))
        return CollisionReport(tick=snapshot.tick, collisions=collisions,
                               neighbor_sets=NeighborSets(alive_all, ids_all, near, n_alive), dropped=dropped)


def run_detector(in_q, out_q, config: CollisionConfig, device=None) -> None:
    """The out-of-loop detector task (collision.py:179-215) on the GPU: consume
    tick-ordered WorldSnapshots, emit one report per consumed snapshot, jump to
    the newest pending snapshot when behind (skips counted in the next
    report's ``dropped``), echo the ``None`` sentinel downstream."""
    import queue
    det = GpuDetector(config, device)
    try:
        pending_drops = 0
        closing = False
        item = in_q.get()
        while item is not None:
            out_q.put(det.detect_snapshot(item, dropped=pending_drops))
            pending_drops = 0
            if closing:
                break
            item = in_q.get()
            while item is not None:
                try:
                    nxt = in_q.get_nowait()
                except queue.Empty:
                    break
                if nxt is None:
                    closing = True
                    break
                item = nxt
                pending_drops += 1
    finally:
        out_q.put(None)


def detect(groups, config: CollisionConfig, tick: int, dropped: int = 0) -> CollisionReport:
    """One-shot detection over B200 groups (see GpuDetector)."""
    groups = list(groups)
    dev = groups[0].device if groups else None
    return GpuDetector(config, dev).detect(groups, tick, dropped)
