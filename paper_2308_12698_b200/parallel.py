"""Agent sharding across GPUs and the neighbour-coupled swarm controller.

One process per GPU (torchrun / torch.distributed).  Agents are independent
in the reference (quad.py:6-7), so a swarm of N agents shards by
contiguous agent index: rank r owns ids [lo_r, hi_r) in its own
``B200QuadGroup`` and steps them with no data-path collective
(``shard_range``, ``ShardedSwarm``).

The only exchange is for the neighbour-coupled controller of config 5
(``NeighborSeparation``): every tick each rank packs its alive positions
(float4, NaN for dead rows) and the ranks all-gather them -- either fused
into the pack kernel over peer memory (``exchange="p2p"``: NVLink stores
into every rank's symmetric buffer plus release/acquire signals,
csrc/exchange.cu) or with NCCL (``exchange="nccl"``, the baseline) -- and
each rank computes the separation overlay of its own agents
against the whole swarm on its GPU (csrc/neighbors.cu), which enters the
next tick through the group's one-tick velocity overlay (core.py:137-139,
172-175).  The reference defines no such controller; its form follows
SURVEY.md 8(e) (the viewer repel field of wire.py:320-340 per neighbour,
strict < of collision.py:166).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ValidationError


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) agent-index range of ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValidationError("bad shard arguments")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_sizes(n_total: int, world: int) -> list[int]:
    return [hi - lo for lo, hi in (shard_range(n_total, r, world) for r in range(world))]


@dataclass
class ShardInfo:
    rank: int
    world: int
    n_total: int
    lo: int
    hi: int
    pad: int          # per-rank slot count in the all-gather (max shard size)

    @property
    def n_local(self) -> int:
        return self.hi - self.lo

    @property
    def self_offset(self) -> int:
        """Row of this rank's first agent in the gathered position buffer."""
        return self.rank * self.pad

    @property
    def n_gathered(self) -> int:
        return self.world * self.pad


def make_shard(n_total: int, rank: int = 0, world: int = 1) -> ShardInfo:
    lo, hi = shard_range(n_total, rank, world)
    return ShardInfo(rank, world, n_total, lo, hi, max(shard_sizes(n_total, world)))


class ShardedSwarm:
    """This rank's shard of one homogeneous swarm: id routing and fault gathering.

    ``group`` is the rank-local group (a ``B200QuadGroup`` holding ids
    [lo, hi)); commands for ids outside the shard are ignored locally (every
    rank sees the full command stream and applies its own).  Stepping is
    collective-free (no per-tick exchange on the uncoupled
    path): ``step`` / ``step_k`` return this rank's fault ids and log them
    with their tick; ``collect()`` exchanges the logged ids of every rank in
    ONE all-gather, so every rank can emit the same FAULT_DEATH events
    (core.py:460-465) at the cadence the caller chooses (every tick, every
    K ticks, or at the end).
    """

    def __init__(self, group, shard: ShardInfo, process_group=None):
        self.group = group
        self.shard = shard
        self.pg = process_group
        self.tick = 0
        self._log: list[tuple[int, np.ndarray]] = []    # (tick, local fault ids) not yet collected

    def owns(self, agent_id: int) -> bool:
        return self.shard.lo <= int(agent_id) < self.shard.hi

    def apply_command(self, cmd) -> bool | None:
        """True/False from the owning rank; None on ranks that do not own the id."""
        if not self.owns(cmd.agent_id):
            return None
        return self.group.apply_command(cmd)

    def mark_dead(self, agent_ids) -> list[int]:
        return self.group.mark_dead([a for a in agent_ids if self.owns(a)])

    def _log_faults(self, per_tick) -> None:
        for j, ids in enumerate(per_tick):
            if len(ids):
                self._log.append((self.tick + j, np.asarray(ids, dtype=np.uint64)))
        self.tick += len(per_tick)

    def step(self, dt: float) -> np.ndarray:
        """One tick of this rank's shard; returns its local fault ids (no collective)."""
        local = np.asarray(self.group.step(dt), dtype=np.uint64)
        self._log_faults([local])
        return local

    def step_k(self, dt: float, k: int = 1) -> np.ndarray:
        """k fused ticks of this rank's shard (one launch); local fault ids."""
        self.group.step_async(dt, k)
        per = self.group.collect_faults()
        self._log_faults(per)
        return np.concatenate(per) if per else np.empty(0, dtype=np.uint64)

    def collect(self) -> list[tuple[int, np.ndarray]]:
        """Every rank's fault ids since the last collect, as (tick, sorted ids)
        in tick order -- one all-gather of the logs (the only collective on
        the uncoupled path; the caller decides how often)."""
        log, self._log = self._log, []
        if self.shard.world == 1:
            parts = [log]
        else:
            import torch.distributed as dist
            parts = [None] * self.shard.world
            dist.all_gather_object(parts, [(t, ids.tolist()) for t, ids in log], group=self.pg)
        by_tick: dict[int, list[int]] = {}
        for part in parts:
            for t, ids in part:
                by_tick.setdefault(int(t), []).extend(int(i) for i in ids)
        return [(t, np.sort(np.array(v, dtype=np.uint64))) for t, v in sorted(by_tick.items())]

    def gather_ids(self, local: np.ndarray) -> np.ndarray:
        """All ranks' ids of ``local`` (collective; sorted)."""
        if self.shard.world == 1:
            return np.sort(np.asarray(local, dtype=np.uint64))
        import torch.distributed as dist
        out = [None] * self.shard.world
        dist.all_gather_object(out, np.asarray(local, dtype=np.int64).tolist(), group=self.pg)
        return np.sort(np.array([i for part in out for i in part], dtype=np.int64)).astype(np.uint64)


class NeighborSeparation:
    """Neighbour-coupled separation controller over a sharded swarm (config 5).

    ``apply()`` performs one exchange + overlay computation; call it right
    before ``group.step(dt)`` (``step()`` does both).  With world == 1 the
    all-gather is skipped (the local buffer is the whole swarm).
    """

    def __init__(self, group, shard: ShardInfo, r_sense: float = 2.0, k_sep: float = 1.0,
                 cell: float | None = None, process_group=None, exchange: str = "nccl"):
        if not r_sense > 0.0:
            raise ValidationError("r_sense must be positive")
        self.group, self.shard = group, shard
        self.r_sense, self.k_sep = float(r_sense), float(k_sep)
        self.cell = float(cell) if cell is not None else float(r_sense)
        if self.cell < self.r_sense:
            raise ValidationError("cell must be >= r_sense")
        self.pg = process_group
        if exchange not in ("nccl", "p2p", "host"):
            raise ValidationError(f"exchange must be 'nccl', 'p2p' or 'host', got {exchange!r}")
        self.exchange = exchange
        self._lib = _lib.load()
        dev = group.device
        n_all = shard.n_gathered
        self.n_all = n_all
        self._epoch = None
        if exchange == "p2p":
            self._init_p2p(dev)
        elif exchange == "host":
            # host-staged transport for CPU (gloo) process groups: the test
            # harness of the multi-rank path on a one-GPU box, not a
            # performance path (the device packs, the host gathers, the
            # device computes the overlay)
            self.local = torch.empty((shard.pad, 4), dtype=torch.float32, device=dev)
            self.all = torch.empty((n_all, 4), dtype=torch.float32, device=dev)
            self._h_parts = [torch.empty((shard.pad, 4), dtype=torch.float32) for _ in range(shard.world)]
        else:
            self.local = torch.empty((shard.pad, 4), dtype=torch.float32, device=dev)
            self.all = self.local if shard.world == 1 else torch.empty((n_all, 4), dtype=torch.float32, device=dev)
        nbytes = ctypes.c_uint64()
        _lib.check(self._lib.swarmstep_neighbor_workspace_bytes(n_all, ctypes.byref(nbytes)))
        self.workspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device=dev)

    def _init_p2p(self, dev) -> None:
        """Symmetric double buffer + signal pads across the process group
        (torch.distributed._symmetric_memory: cuMem / IPC peer mappings)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        if not dist.is_initialized():
            raise ValidationError("exchange='p2p' needs an initialised torch.distributed process group")
        pg = self.pg if self.pg is not None else dist.group.WORLD
        if dist.get_world_size(pg) != self.shard.world or dist.get_rank(pg) != self.shard.rank:
            raise ValidationError("shard does not match the process group")
        with torch.cuda.device(dev):
            self._buf = symm.empty((2 * self.n_all, 4), dtype=torch.float32, device=dev)
            self._buf.fill_(float("nan"))
            self._hdl = symm.rendezvous(self._buf, pg.group_name)
            self._epoch = torch.zeros(1, dtype=torch.int32, device=dev)
            self._arrive = torch.zeros(1, dtype=torch.int32, device=dev)
            torch.cuda.synchronize(dev)
        self._hdl.barrier()
        self.all = self._buf
        self._sig_local = int(self._hdl.signal_pad_ptrs[self.shard.rank])

    def gather(self) -> torch.Tensor:
        g = self.group
        if self.exchange == "p2p":
            s = ctypes.c_void_p(g.stream.cuda_stream)
            with torch.cuda.device(g.device):
                _lib.check(self._lib.swarmstep_p2p_pack_push(
                    g._view_ref, ctypes.c_void_p(int(self._hdl.buffer_ptrs_dev)), self.shard.world,
                    self.shard.rank, self.shard.pad, ctypes.c_void_p(int(self._hdl.signal_pad_ptrs_dev)),
                    self._epoch.data_ptr(), self._arrive.data_ptr(), s))
                _lib.check(self._lib.swarmstep_p2p_wait(ctypes.c_void_p(self._sig_local), self.shard.world,
                                                        self._epoch.data_ptr(), s))
            return self.all
        with torch.cuda.device(g.device), torch.cuda.stream(g.stream):
            _lib.check(self._lib.swarmstep_pack_positions(g._view_ref, self.local.data_ptr(), self.shard.pad,
                                                          ctypes.c_void_p(g.stream.cuda_stream)))
            if self.exchange == "host":
                import torch.distributed as dist
                mine = self.local.cpu()                       # waits for the pack (stream order)
                if self.shard.world > 1:
                    dist.all_gather(self._h_parts, mine, group=self.pg)
                else:
                    self._h_parts[0].copy_(mine)
                self.all.copy_(torch.cat(self._h_parts))
            elif self.shard.world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(self.all, self.local, group=self.pg)
        return self.all

    def gathered_positions(self) -> torch.Tensor:
        """The (n_all, 4) positions of the last exchange (the slot of the
        current epoch for the P2P double buffer)."""
        if self.exchange != "p2p":
            if self.shard.world == 1:
                self.gather()          # the single-rank launch reads the columns directly
            torch.cuda.synchronize(self.group.device)
            return self.all
        torch.cuda.synchronize(self.group.device)
        e = int(self._epoch.item())
        return self._buf[(e & 1) * self.n_all:((e & 1) + 1) * self.n_all]

    def launch(self, accumulate: bool = True) -> None:
        """Device work of one exchange: pack -> all-gather -> overlay kernel (no
        host state change; graph-capturable when world == 1 or with the P2P
        exchange, whose slot selection happens on the device)."""
        g = self.group
        single = self.shard.world == 1 and self.exchange == "nccl"
        if not single:
            self.gather()
        with torch.cuda.device(g.device), torch.cuda.stream(g.stream):
            _lib.check(self._lib.swarmstep_neighbor_overlay(
                g._view_ref, None if single else self.all.data_ptr(), self.n_all, self.shard.self_offset,
                ctypes.c_float(self.r_sense), ctypes.c_float(self.k_sep), ctypes.c_float(self.cell),
                1 if accumulate else 0, self.workspace.data_ptr(), ctypes.c_uint64(self.workspace.numel()),
                self._epoch.data_ptr() if self._epoch is not None else None,
                ctypes.c_void_p(g.stream.cuda_stream)))

    def apply(self) -> None:
        """Compute this tick's separation overlay into the group's one-tick
        overlay input (added to any overlay already pending)."""
        # the overlay block is all-zero whenever no overlay is pending (the
        # group clears it after every step), so accumulating is always right
        self.launch(accumulate=True)
        self.group._overlay_active = True

    def step(self, dt: float) -> np.ndarray:
        self.apply()
        return self.group.step(dt)
